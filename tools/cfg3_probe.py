"""Config-3 probe: setup time, one all-at-once fine sweep over the 128 intervals, one
parareal iteration (bench step), GPU memory."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_09244_b200 as P  # noqa: E402

t0 = time.time()
z = np.load(os.path.join(ROOT, "data", "sys_cfg3.npz"))
s = P.CoarseSystem(*(np.ascontiguousarray(z[k]) for k in ("M11", "A11", "M12", "A12", "M22", "A22")))
ld = P.ConstantLoads(z["f1"], z["f2"])
print("load", round(time.time() - t0, 1), "s", s.d1, s.d2, flush=True)
N, J, T = 128, 100, 2.0
ctx = P.PeContext([s], [ld], J)
torch.cuda.synchronize()
t0 = time.time()
ctx.prepare_coarse(T / N)
torch.cuda.synchronize()
t1 = time.time()
ctx.prepare_allatonce(T / N / J, 0.1, 1e-12, 400)
torch.cuda.synchronize()
t2 = time.time()
print(f"setup coarse {t1 - t0:.1f} s, all-at-once {t2 - t1:.1f} s, mem {torch.cuda.memory_allocated() / 1e9:.1f} GB (torch)", flush=True)
d = s.d1 + s.d2
A = torch.zeros(1, N + 1, d, dtype=torch.float64, device="cuda")
B = torch.zeros_like(A)
Gc = torch.zeros(1, N, d, dtype=torch.float64, device="cuda")
diff = torch.zeros(1, 2, dtype=torch.float64, device="cuda")
t0 = time.time()
ctx.coarse_correct(N, A, None, Gc, A)
torch.cuda.synchronize()
print(f"initial coarse sweep {1e3 * (time.time() - t0):.1f} ms", flush=True)
sw = torch.zeros(1, N, dtype=torch.int32, device="cuda")
rs = torch.zeros(1, N, dtype=torch.int32, device="cuda")
for it in range(int(os.environ.get("ITERS", "2"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.iterate("all-at-once", N, A, B, Gc, diff, wr_sweeps=sw, wr_reasons=rs)
    e1.record()
    torch.cuda.synchronize()
    A, B = B, A
    swn = sw.cpu().numpy()[0]
    rsn = rs.cpu().numpy()[0]
    dd = diff.cpu().numpy()[0]
    print(f"iteration {it + 1}: {e0.elapsed_time(e1):.0f} ms, sweeps min/mean/max "
          f"{swn.min()}/{swn.mean():.1f}/{swn.max()}, reasons {np.bincount(rsn, minlength=4)}, "
          f"diff {dd[0]:.3e} rel {dd[0] / dd[1]:.3e}", flush=True)
print(json.dumps(ctx.fine_stats()))
