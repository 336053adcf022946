"""Golden vectors for the reference's Example-1 acceptance test (TEST INFRASTRUCTURE).

`pkg/tests/test_acceptance.py:82-93` runs `run_single(example1_pipeline, n)` for
N = 20..60 (the paper's Example 1 analog: 100x100 mesh, 10x10 coarse blocks, 4 layers,
one channel (5, 95, 44, 46) at 1e4, box source, NLMC split space, T = 0.005, J = N,
all-at-once fine solver, alpha = 0.5, absolute stop 1e-14) and asserts the iteration
counts stay in [8, 25] with count(60) <= count(20) + 2; measured here: 19, 15, 12, 12, 12.

Records, from the UNMODIFIED reference imported read-only: the reduced system and loads
of the example-1 pipeline, and per N the parareal iteration count, max_diffs, history
and per-(k, n) WR sweep counts.  Output: tests/golden/example1.npz.
"""

import os
import sys
from dataclasses import replace

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402
from paradiff.experiment import build_pipeline, example1_config, run_single  # noqa: E402

NS = (20, 30, 40, 50, 60)


def main():
    cfg = replace(example1_config(), compute_reference=False, export_solution=False)
    pipe = build_pipeline(cfg)
    s = pipe.space.system
    out = {k: getattr(s, k) for k in ("M11", "A11", "M12", "A12", "M22", "A22")}
    out["f1"], out["f2"] = pipe.loads.f1, pipe.loads.f2
    out["ns"] = np.array(NS)
    out["t_end"] = np.array(cfg.t_end)
    out["alpha"] = np.array(cfg.alpha)
    out["epsilon"] = np.array(cfg.epsilon)
    for n in NS:
        r = run_single(pipe, n).run
        out[f"iters_{n}"] = np.array(r.iterations)
        out[f"diffs_{n}"] = np.array(r.max_diffs)
        out[f"hist_{n}"] = np.array(r.history)
        out[f"wr_{n}"] = np.array([[i["iterations"] for i in k] for k in r.fine_info])
        print(n, r.iterations, r.max_diffs[-3:], flush=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "example1.npz"), **out)
    print("d1, d2 =", s.d1, s.d2)


if __name__ == "__main__":
    main()
