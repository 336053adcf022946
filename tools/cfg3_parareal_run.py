"""Config 3 parareal run to its stop (relative 1e-8) on one B200.

Parareal needs ~50 iterations here (relative increment ~0.78x per iteration,
tools/cfg3_wr_probe.py), each 502 WR sweeps (~32 s), so the run takes ~25-30 minutes.
Iterations are run one `ctx.iterate` at a time so that progress is written after each:
gpurun_out/cfg3_parareal.json (iteration count, relative increments, WR sweep statistics,
seconds per iteration) and gpurun_out/cfg3_parareal.npz (history rows of sampled
intervals).  The device loop is the one `run_parareal` uses (pe_parareal_iterate).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_09244_b200 as P  # noqa: E402
from paper_2411_09244_b200.sysdata import load_system  # noqa: E402

K_MAX = int(sys.argv[1]) if len(sys.argv) > 1 else 128
EPS, MAX_ITER = 1e-8, 600
SAMPLE = [0, 1, 32, 64, 96, 127, 128]
blocks, f1, f2, meta = load_system(os.path.join(ROOT, "data", "cfg3"))
s = P.CoarseSystem(**blocks)
N, J, T = 128, 100, 2.0
ctx = P.PeContext([s], [P.ConstantLoads(f1, f2)], J)
ctx.prepare_coarse(T / N)
ctx.prepare_allatonce(T / N / J, 0.1, 1e-12, MAX_ITER)
d = s.d1 + s.d2
A = torch.zeros(1, N + 1, d, dtype=torch.float64, device="cuda")
B = torch.zeros_like(A)
Gc = torch.zeros(1, N, d, dtype=torch.float64, device="cuda")
diff = torch.zeros(1, 2, dtype=torch.float64, device="cuda")
sw = torch.zeros(1, N, dtype=torch.int32, device="cuda")
rs = torch.zeros(1, N, dtype=torch.int32, device="cuda")
ctx.coarse_correct(N, A, None, Gc, A)
torch.cuda.synchronize()
hist = [A[0, SAMPLE].cpu().numpy()]
rec = dict(config="cfg3-aao", fine_max_iter=MAX_ITER, epsilon=EPS, rule="relative",
           rel_increments=[], abs_increments=[], sweeps_min=[], sweeps_max=[], sweeps_mean=[],
           reasons=[], seconds=[], converged=False, iterations=0)
out_json = os.path.join(ROOT, "gpurun_out", "cfg3_parareal.json")
os.makedirs(os.path.dirname(out_json), exist_ok=True)
for k in range(1, K_MAX + 1):
    t0 = time.perf_counter()
    ctx.iterate("all-at-once", N, A, B, Gc, diff, wr_sweeps=sw, wr_reasons=rs)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    A, B = B, A
    dv = diff[0].cpu().numpy()
    rel = float(dv[0] / dv[1]) if dv[1] > 0 else float(dv[0])
    s_np, r_np = sw[0].cpu().numpy(), rs[0].cpu().numpy()
    hist.append(A[0, SAMPLE].cpu().numpy())
    rec["rel_increments"].append(rel)
    rec["abs_increments"].append(float(dv[0]))
    rec["sweeps_min"].append(int(s_np.min()))
    rec["sweeps_max"].append(int(s_np.max()))
    rec["sweeps_mean"].append(float(s_np.mean()))
    rec["reasons"].append(np.bincount(r_np, minlength=4).tolist())
    rec["seconds"].append(dt)
    rec["iterations"] = k
    print(f"k={k}: rel {rel:.3e} sweeps {s_np.min()}-{s_np.max()} {dt:.1f} s", flush=True)
    if rel < EPS:
        rec["converged"] = True
    with open(out_json, "w") as f:
        json.dump(rec, f, indent=1)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", "cfg3_parareal.npz"),
                        sample=np.array(SAMPLE), history=np.array(hist))
    if rec["converged"]:
        break
print(json.dumps({k: rec[k] for k in ("iterations", "converged")}))
