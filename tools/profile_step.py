"""Run setup + one warm parareal iteration, then ONE profiled iteration inside a
cudaProfilerStart/Stop range (ncu --profile-from-start off captures exactly one step)."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_09244_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2-aao")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--max-iter", type=int, default=0,
                help="cap the WR sweeps per solve (shares of a sweep do not depend on it)")
args = ap.parse_args()
wl = bench.WORKLOADS[args.workload]
mem, meta = bench.load_workload(wl)
systems = [P.CoarseSystem(**b) for b, _, _ in mem]
s = systems[0]
E = len(systems)
ctx = P.PeContext(systems, [P.ConstantLoads(a, b) for _, a, b in mem], wl["J"])
N, J, T, kind = wl["N"], wl["J"], wl["T"], wl["kind"]
ctx.prepare_coarse(T / N)
if kind == "sequential":
    ctx.prepare_sequential(T / N / J)
else:
    ctx.prepare_allatonce(T / N / J, wl["alpha"], bench.FINE_TOL,
                          args.max_iter or wl["max_iter"])
d = s.d1 + s.d2
A = torch.zeros(E, N + 1, d, dtype=torch.float64, device="cuda")
B = torch.zeros_like(A)
Gc = torch.zeros(E, N, d, dtype=torch.float64, device="cuda")
diff = torch.zeros(E, 2, dtype=torch.float64, device="cuda")
ctx.coarse_correct(N, A, None, Gc, A)
ctx.iterate(kind, N, A, B, Gc, diff)
A, B = B, A
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.steps):
    ctx.iterate(kind, N, A, B, Gc, diff)
    A, B = B, A
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", args.workload, "launches", ctx.launch_count())
