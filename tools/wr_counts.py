"""GPU WR sweep counts / residual tails for cfg2 iteration-1 intervals vs the oracle."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_09244_b200 as P
from oracle import pe_oracle as po
z = np.load(os.path.join(ROOT, "tests/golden/sys_cfg2.npz"))
run = np.load(os.path.join(ROOT, "tests/golden/run_cfg2_aao.npz"))
s = P.CoarseSystem(*(z[k] for k in ["M11", "A11", "M12", "A12", "M22", "A22"]))
ld = P.ConstantLoads(z["f1"], z["f2"])
wr = P.WaveformRelaxation(s, 64, 1 / 64, 0.1, ld, tol=1e-12, max_iter=400)
for k in (0, 3):
    X = run["history"][k]
    states = [P.SplitState.fresh(X[n, :300], X[n, 300:], n / 64) for n in range(64)]
    res = wr.solve_all(states, trajectories=False)
    g = np.array([r.iterations for r in res])
    ref = run["wr_iterations"][k]
    print("iter", k + 1, "gpu sweeps", g[:12], "ref", ref[:12], "maxdiff", np.abs(g - ref).max())
    print("   reasons", [r.stop_reason for r in res[:6]], "tail", res[1].residuals[-4:])
