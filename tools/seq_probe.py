"""Event-time the pieces of one sequential parareal iteration (fine chain, coarse sweep,
whole iterate) for a bench workload, with and without an L2 flush in front."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_09244_b200 as P  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2-seq"]
mem, meta = bench.load_workload(wl)
blocks, f1, f2 = mem[0]
s = P.CoarseSystem(**blocks)
ctx = P.PeContext([s], [P.ConstantLoads(f1, f2)], wl["J"])
N, J, T = wl["N"], wl["J"], wl["T"]
ctx.prepare_coarse(T / N)
ctx.prepare_sequential(T / N / J)
d = s.d1 + s.d2
A = torch.randn(1, N + 1, d, dtype=torch.float64, device="cuda") * 0.1
B = torch.zeros_like(A)
Gc = torch.zeros(1, N, d, dtype=torch.float64, device="cuda")
diff = torch.zeros(1, 2, dtype=torch.float64, device="cuda")
X = A[:, :N].contiguous()
flush = torch.empty(40 * 1024 * 1024, dtype=torch.float64, device="cuda")


def timed(fn, reps=10, fl=False):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        if fl:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return 1e3 * tot / reps


for fl in (False, True):
    tag = "flushed" if fl else "warm"
    print(tag, "fine_sequential %.1f us" % timed(lambda: ctx.fine_sequential(X), fl=fl),
          "coarse_correct %.1f us" % timed(lambda: ctx.coarse_correct(N, A, None, Gc, B, diff), fl=fl),
          "iterate %.1f us" % timed(lambda: ctx.iterate("sequential", N, A, B, Gc, diff), fl=fl),
          flush=True)
