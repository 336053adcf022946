"""Config-3 waveform-relaxation convergence probe (GPU).

1. Iteration 1 (inputs: the initial coarse sweep): WR on all 128 intervals with a large
   sweep cap; per-interval sweep counts, stop reasons and full residual histories.
2. The full parareal run (relative 1e-8 stop) with that cap: iteration count,
   max_diffs, per-(k, n) sweep counts / reasons, and the history rows of sampled
   intervals (inputs for the CPU oracle comparison, oracle/make_cfg3_golden.py).

Writes gpurun_out/cfg3_wr_probe.npz and prints a summary.
    python tools/cfg3_wr_probe.py [max_iter] [k_max]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_09244_b200 as P  # noqa: E402
from paper_2411_09244_b200.sysdata import load_system  # noqa: E402

MAX_ITER = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
K_MAX = int(sys.argv[2]) if len(sys.argv) > 2 else 16
SAMPLE = (0, 1, 2, 63, 64, 127)

t0 = time.time()
blocks, f1, f2, meta = load_system(os.path.join(ROOT, "data", "cfg3"))
s = P.CoarseSystem(**blocks)
ld = P.ConstantLoads(f1, f2)
print("load", round(time.time() - t0, 1), "s", s.d1, s.d2, flush=True)
N, J, T = 128, 100, 2.0
ctx = P.PeContext([s], [ld], J)
ctx.prepare_coarse(T / N)
ctx.prepare_allatonce(T / N / J, 0.1, 1e-12, MAX_ITER)
d = s.d1 + s.d2
A = torch.zeros(1, N + 1, d, dtype=torch.float64, device="cuda")
Gc = torch.zeros(1, N, d, dtype=torch.float64, device="cuda")
ctx.coarse_correct(N, A, None, Gc, A)
torch.cuda.synchronize()
out = {"x0_it1": A[0].cpu().numpy()[list(SAMPLE)], "sample": np.array(SAMPLE),
       "max_iter": np.array(MAX_ITER)}
t1 = time.time()
Y, sw, rs, rh = ctx.fine_allatonce(A[:, :N].contiguous())
torch.cuda.synchronize()
t_it1 = time.time() - t1
sw = sw[0].cpu().numpy()
rs = rs[0].cpu().numpy()
rh = rh[0].cpu().numpy()
out.update(it1_sweeps=sw, it1_reasons=rs, it1_resid=rh[:, : int(sw.max())],
           it1_final=Y[0].cpu().numpy()[list(SAMPLE)])
print(f"iteration-1 fine sweep: {t_it1:.1f} s; sweeps min/mean/max {sw.min()}/{sw.mean():.1f}/"
      f"{sw.max()}; reasons (tol, diverged, floor, max_iter) {np.bincount(rs, minlength=4)}",
      flush=True)
for n in (0, 1, 64, 127):
    r = rh[n, : sw[n]]
    marks = [r[i] for i in range(0, len(r), max(1, len(r) // 12))]
    print(f"  interval {n}: " + " ".join(f"{v:.2e}" for v in marks) + f" ... {r[-1]:.2e}",
          flush=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "cfg3_wr_probe.npz"), **out)

cfg = P.ParerealConfig(time_grid=P.TimeGrid(T, N, J), alpha=0.1, epsilon=1e-8, k_max=K_MAX,
                       fine_kind="all-at-once", fine_tol=1e-12, fine_max_iter=MAX_ITER,
                       stop_rule="relative")
props = P.SplitPropagators(s, ld)
props._ctx[J] = ctx
fine = P.build_fine_propagator(cfg, props, ld)
t1 = time.time()
run = P.run_parareal(cfg, props, fine, P.SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2)))
t_run = time.time() - t1
hist = np.array(run.history)
sweeps = np.array([[i["iterations"] for i in k] for k in run.fine_info])
reasons = np.array([[i["stop_reason"] for i in k] for k in run.fine_info])
out.update(iterations=np.array(run.iterations), max_diffs=np.array(run.max_diffs),
           sweeps=sweeps, hist_sample=hist[:, list(SAMPLE)],
           fine_seconds=np.array(run.fine_seconds), converged=np.array(run.converged))
for k in range(len(run.fine_info)):
    u, c = np.unique(reasons[k], return_counts=True)
    print(f"  k={k + 1}: max_diff {run.max_diffs[k]:.3e}, sweeps {sweeps[k].min()}-"
          f"{sweeps[k].max()} (mean {sweeps[k].mean():.1f}), reasons {dict(zip(u, c))}, "
          f"fine {run.fine_seconds[k]:.1f} s", flush=True)
print(f"parareal: {run.iterations} iterations, converged {run.converged}, {t_run:.0f} s",
      flush=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "cfg3_wr_probe.npz"), **out)
