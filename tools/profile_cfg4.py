"""Setup + one warm iteration of the cfg4 ensemble, then ONE profiled iteration."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_09244_b200 as P  # noqa: E402

wl = bench.WORKLOADS["cfg4-seq"]
mem, meta = bench.load_workload(wl)
systems = [P.CoarseSystem(**b) for b, _, _ in mem]
loads = [P.ConstantLoads(a, b) for _, a, b in mem]
E, N, J, T = len(mem), 32, 32, 1.0
ctx = P.PeContext(systems, loads, J)
ctx.prepare_coarse(T / N)
ctx.prepare_sequential(T / N / J)
d = systems[0].d1 + systems[0].d2
A = torch.zeros(E, N + 1, d, dtype=torch.float64, device="cuda")
B = torch.zeros_like(A)
Gc = torch.zeros(E, N, d, dtype=torch.float64, device="cuda")
diff = torch.zeros(E, 2, dtype=torch.float64, device="cuda")
ctx.coarse_correct(N, A, None, Gc, A)
ctx.iterate("sequential", N, A, B, Gc, diff)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ctx.iterate("sequential", N, B, A, Gc, diff)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
