"""cfg1 WR fine solve on the fused tiny path: sweeps per interval and event time per call,
tiny path vs graph path (set_recurrence(False) disables the fused kernel)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_09244_b200 as P  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg1-aao"]
blocks, f1, f2, meta = bench.load_system(wl["sys"])
s = P.CoarseSystem(**blocks)
ctx = P.PeContext([s], [P.ConstantLoads(f1, f2)], wl["J"])
N, J, T = wl["N"], wl["J"], wl["T"]
ctx.prepare_coarse(T / N)
ctx.prepare_allatonce(T / N / J, wl["alpha"], bench.FINE_TOL, bench.MAX_ITER)
d = s.d1 + s.d2
g = torch.Generator().manual_seed(0)
X = torch.randn(1, N, d, dtype=torch.float64, generator=g).cuda()
for tiny in (True, False):
    ctx.set_recurrence(tiny)
    for _ in range(3):
        Y, sw, rs, rh = ctx.fine_allatonce(X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        Y, sw, rs, rh = ctx.fine_allatonce(X)
    e1.record()
    torch.cuda.synchronize()
    print("tiny" if tiny else "graph", "ms/call %.4f" % (e0.elapsed_time(e1) / 10),
          "sweeps", sw.flatten().tolist(), "reasons", rs.flatten().tolist(), flush=True)
