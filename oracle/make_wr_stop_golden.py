"""Golden vectors for the waveform-relaxation stop branches (TEST INFRASTRUCTURE).

Runs the UNMODIFIED reference (`WaveformRelaxation.solve`, allatonce.py:232-298) in the
build container on the reference test fixture system `channel.npz` (the channel pipeline
of pkg/tests/conftest.py:7-28, recorded by make_golden.py) for windows that end in each
stop reason of allatonce.py:258-271:

* `diverged`: dt_interval 1e-2, J = 10, alpha = 0.9 (the alpha-corner recycles the error
  at a rate > 1 on this window: the residual grows ~9 % per sweep past 1e8 * r0);
* `floor`:    dt_interval 5e-4, J = 10, alpha = 0.99, tol 1e-13 (the residual stalls
  between tol and 1e3 tol);
* `max_iter`: dt_interval 5e-3, J = 10, alpha = 0.9, 300-sweep cap;
* `tol`:      dt_interval 5e-3, J = 10, alpha = 0.5.

For each: sweep count, stop reason, full residual history and the final waveform rows.
Output: tests/golden/wr_stop.npz.
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402
from paradiff.allatonce import WaveformRelaxation  # noqa: E402
from paradiff.msbasis import CoarseSystem  # noqa: E402
from paradiff.stepping import ConstantLoads, SplitState  # noqa: E402

CASES = {  # name: (dt_interval, J, alpha, tol, max_iter)
    "diverged": (1e-2, 10, 0.9, 1e-13, 400),
    "floor": (5e-4, 10, 0.99, 1e-13, 400),
    "max_iter": (5e-3, 10, 0.9, 1e-13, 300),
    "tol": (5e-3, 10, 0.5, 1e-13, 400),
}
REASON_CODE = {"tol": 0, "diverged": 1, "floor": 2, "max_iter": 3}


def main():
    z = np.load(os.path.join(ROOT, "tests", "golden", "channel.npz"))
    s = CoarseSystem(*(z[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")))
    loads = ConstantLoads(z["f1"], z["f2"])
    out = {}
    for name, (dti, J, alpha, tol, cap) in CASES.items():
        wr = WaveformRelaxation(s, J, dti, alpha, loads, tol=tol, max_iter=cap)
        r = wr.solve(SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2)))
        assert r.stop_reason == name, (name, r.stop_reason)
        out[f"{name}_params"] = np.array([dti, J, alpha, tol, cap])
        out[f"{name}_meta"] = np.array([r.iterations, REASON_CODE[r.stop_reason]])
        out[f"{name}_res"] = np.array(r.residuals)
        out[f"{name}_U"] = r.trajectory.U
        out[f"{name}_W"] = r.trajectory.W
        print(name, r.iterations, r.stop_reason, r.residuals[-1])
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "wr_stop.npz"), **out)


if __name__ == "__main__":
    main()
