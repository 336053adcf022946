"""Golden vectors with time-dependent loads (TEST INFRASTRUCTURE).

The reference evaluates loads at the step's end time, `loads.at(state.t + dt)`, in
split_step and coarse_step (stepping.py:125,164) and at t0 + dt (1..J) in the waveform
relaxation (allatonce.py:212-218); every ConstantLoads config hides this.  This runs the
UNMODIFIED reference with a time-dependent load on the config-0 reduced system:

    f1(t) = f1 (1 + 0.5 sin(2 pi t)),  f2(t) = f2 (1 - 0.3 cos(2 pi t)) + 0.01 t

and records one split step / coarse step / fine interval / WR solve starting at t = 0.37,
and full parareal runs (sequential and all-at-once, alpha = 0.1, T = 1, N = J = 10,
relative 1e-8 stop, fine_tol 1e-12) with their histories.  Output: tests/golden/tv_loads.npz.
"""

import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import paradiff.parareal as pp  # noqa: E402
from paradiff.allatonce import WaveformRelaxation  # noqa: E402
from paradiff.msbasis import CoarseSystem  # noqa: E402
from paradiff.parareal import ParerealConfig, build_fine_propagator, run_parareal  # noqa: E402
from paradiff.stepping import SplitPropagators, SplitState, TimeGrid  # noqa: E402

from oracle.make_golden import _relative_check  # noqa: E402


class WaveLoads:
    constant = False

    def __init__(self, f1, f2):
        self.f1, self.f2 = np.asarray(f1, float), np.asarray(f2, float)

    def at(self, t):
        return (self.f1 * (1.0 + 0.5 * np.sin(2.0 * np.pi * t)),
                self.f2 * (1.0 - 0.3 * np.cos(2.0 * np.pi * t)) + 0.01 * t)


def main():
    z = np.load(os.path.join(ROOT, "tests", "golden", "sys_cfg0.npz"))
    s = CoarseSystem(*(z[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")))
    loads = WaveLoads(z["f1"], z["f2"])
    props = SplitPropagators(s, loads)
    rng = np.random.default_rng(17)
    x = rng.standard_normal(s.d1 + s.d2) * 1e-3
    st = SplitState(x[: s.d1], x[s.d1:], x[: s.d1] * 0.9, x[s.d1:] * 1.1, 0.37)
    out = {}
    a = props.split_step(st, 0.01)
    out["split"] = a.stacked()
    out["coarse"] = props.coarse_step(st, 0.1).stacked()
    tr = props.fine_interval(st, 0.1, 10)
    out["fine_U"], out["fine_W"], out["fine_t"] = tr.U, tr.W, np.array(tr.final.t)
    wr = WaveformRelaxation(s, 10, 0.1, 0.1, loads, tol=1e-12, max_iter=400)
    r = wr.solve(SplitState.fresh(x[: s.d1], x[s.d1:], 0.37))
    out["wr_U"], out["wr_W"] = r.trajectory.U, r.trajectory.W
    out["wr_meta"] = np.array([r.iterations])
    out["x"] = x
    saved = pp.check_stop
    pp.check_stop = _relative_check
    try:
        for kind, tag in (("sequential", "seq"), ("all-at-once", "aao")):
            cfg = ParerealConfig(time_grid=TimeGrid(1.0, 10, 10), alpha=0.1, epsilon=1e-8,
                                 k_max=10, fine_kind=kind, fine_tol=1e-12)
            fine = build_fine_propagator(cfg, props, loads)
            run = run_parareal(cfg, props, fine, SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2)))
            out[f"{tag}_hist"] = np.array(run.history)
            out[f"{tag}_iters"] = np.array(run.iterations)
            print(tag, run.iterations, run.max_diffs[-1])
    finally:
        pp.check_stop = saved
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "tv_loads.npz"), **out)


if __name__ == "__main__":
    main()
