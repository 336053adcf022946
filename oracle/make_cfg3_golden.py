"""Config-3 sampled-interval golden vectors (TEST INFRASTRUCTURE, SURVEY §8c "Config-3
parity": a full reference run is infeasible, F7).

Runs the CPU oracle (pinned bitwise to the reference in tests/test_oracle_pins.py) on
data/sys_cfg3.npz: the initial coarse sweep, then waveform relaxation with a small sweep
cap on sampled intervals of iteration 1.  The shifted inverses are formed one mode at a
time into a preallocated array (the reference's stacked np.linalg.inv would need 2 x 26.8
GB), which changes nothing numerically: each mode is an independent LAPACK inverse.

Output: tests/golden/cfg3_sample.npz (small; the GPU test skips without data/sys_cfg3.npz).
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pe_oracle as po  # noqa: E402

SAMPLE = (1, 64)   # interval indices of iteration 1
SWEEPS = 3         # WR sweep cap for the sample


def main():
    z = np.load(os.path.join(ROOT, "data", "sys_cfg3.npz"))
    s = po.OSystem.from_arrays(z)
    N, J, T, alpha = 128, 100, 2.0, 0.1
    dt = T / N
    t0 = time.time()
    sp = po.OracleSplit(s)
    states = [np.zeros(s.d1 + s.d2)]
    for _ in range(max(SAMPLE)):
        states.append(sp.coarse_step(states[-1], dt))
    print("coarse sweep", time.time() - t0, flush=True)

    class WR(po.OracleWR):
        def __init__(self):  # noqa: D401 - per-mode inverses, same arithmetic
            self.s, self.J, self.dt_interval, self.dt = s, J, dt, dt / J
            self.alpha, self.tol, self.max_iter = alpha, 1e-12, SWEEPS
            d = po.time_eigenvalues(J, self.dt, alpha)
            self.inv_shifted = np.empty((J, s.d1, s.d1), dtype=complex)
            for k in range(J):
                self.inv_shifted[k] = np.linalg.inv(d[k] * s.M11 + s.A11.astype(complex))
                if k % 10 == 0:
                    print("  inverse", k, round(time.time() - t0), flush=True)
            from scipy.linalg import cho_factor, cho_solve
            self.m22_inv = cho_solve(cho_factor(s.M22), np.eye(s.d2))
            self.e_mat = np.eye(s.d2) - self.dt * self.m22_inv @ s.A22

    wr = WR()
    out = {"sample": np.array(SAMPLE), "sweeps": np.array(SWEEPS)}
    for n in SAMPLE:
        x = states[n]
        r = wr.solve(x[: s.d1], x[s.d1:])
        out[f"x_{n}"] = x
        out[f"final_{n}"] = np.concatenate([r["U"][-1], r["W"][-1]])
        out[f"U5_{n}"] = r["U"][5]
        out[f"res_{n}"] = np.array(r["residuals"])
        print("interval", n, "residuals", r["residuals"], round(time.time() - t0), flush=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cfg3_sample.npz"), **out)


if __name__ == "__main__":
    main()
