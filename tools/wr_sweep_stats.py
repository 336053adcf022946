"""cfg2 all-at-once parareal on the GPU vs the reference golden run: iteration count, max
history deviation and the WR sweep-count statistics per (iteration, interval)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_09244_b200 as P  # noqa: E402

z = np.load(os.path.join(ROOT, "tests", "golden", "sys_cfg2.npz"))
g = np.load(os.path.join(ROOT, "tests", "golden", "run_cfg2_aao.npz"))
s = P.CoarseSystem(*(z[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")))
ld = P.ConstantLoads(z["f1"], z["f2"])
cfg = P.ParerealConfig(time_grid=P.TimeGrid(1.0, 64, 64), alpha=0.1, epsilon=1e-8, k_max=64,
                       fine_kind="all-at-once", fine_tol=1e-12, stop_rule="relative")
props = P.SplitPropagators(s, ld)
fine = P.build_fine_propagator(cfg, props, ld)
run = P.run_parareal(cfg, props, fine, P.SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2)))
h, r = np.array(run.history), g["history"]
rel = (np.linalg.norm(h - r, axis=-1) / np.maximum(np.linalg.norm(r, axis=-1), 1e-300)).max()
its = np.array([[i["iterations"] for i in sw] for sw in run.fine_info])
reasons = [i["stop_reason"] for sw in run.fine_info for i in sw]
ref = g["wr_iterations"]
print(f"modal level {fine.ctx.modal_level()}: parareal iterations {run.iterations} (reference "
      f"{int(g['iterations'])}), max history rel L2 {rel:.2e}")
print(f"WR sweeps: GPU mean {its.mean():.1f} [{its.min()}, {its.max()}], reference mean "
      f"{ref.mean():.1f} [{ref.min()}, {ref.max()}], mean rel dev "
      f"{(its.mean() - ref.mean()) / ref.mean():+.3%}, max |dev| {np.abs(its - ref).max()}")
print("GPU stop reasons:", {k: reasons.count(k) for k in set(reasons)})
