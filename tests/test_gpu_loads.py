"""Time-dependent loads on the GPU path (the reference's `loads.at(t)`: stepping.py:125,164,
allatonce.py:212-218) against the unmodified reference's own runs
(tests/golden/tv_loads.npz, oracle/make_tv_golden.py) and the CPU oracle.

Load: f1(t) = f1 (1 + 0.5 sin 2 pi t), f2(t) = f2 (1 - 0.3 cos 2 pi t) + 0.01 t on the
config-0 reduced system.
"""

import dataclasses

import numpy as np
import pytest

from oracle import pe_oracle as po
from tests.conftest import golden

pytestmark = pytest.mark.gpu
BLOCKS = ("M11", "A11", "M12", "A12", "M22", "A22")


class WaveLoads:
    constant = False

    def __init__(self, f1, f2):
        self.f1, self.f2 = np.asarray(f1, float), np.asarray(f2, float)

    def at(self, t):
        return (self.f1 * (1.0 + 0.5 * np.sin(2.0 * np.pi * t)),
                self.f2 * (1.0 - 0.3 * np.cos(2.0 * np.pi * t)) + 0.01 * t)


def _setup():
    import paper_2411_09244_b200 as P

    z = golden("sys_cfg0.npz")
    s = P.CoarseSystem(*(z[k] for k in BLOCKS))
    ld = WaveLoads(z["f1"], z["f2"])
    return P, z, s, ld


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_steps_with_time_dependent_loads_match_reference():
    P, z, s, ld = _setup()
    g = golden("tv_loads.npz")
    x = g["x"]
    d1 = s.d1
    props = P.SplitPropagators(s, ld)
    st = P.SplitState(x[:d1], x[d1:], x[:d1] * 0.9, x[d1:] * 1.1, 0.37)
    assert _rel(props.split_step(st, 0.01).stacked(), g["split"]) < 1e-11
    assert _rel(props.coarse_step(st, 0.1).stacked(), g["coarse"]) < 1e-11
    tr = props.fine_interval(st, 0.1, 10)
    assert _rel(tr.U, g["fine_U"]) < 1e-10 and _rel(tr.W, g["fine_W"]) < 1e-10
    assert tr.final.t == float(g["fine_t"])
    # the batched sequential propagator (per-step GEMMs with per-column load terms)
    cfg = P.ParerealConfig(time_grid=P.TimeGrid(1.0, 10, 10), alpha=0.1, fine_kind="sequential")
    fine = P.build_fine_propagator(cfg, props, ld)
    out, _ = fine.propagate(P.SplitState.fresh(x[:d1], x[d1:], 0.37))
    assert _rel(out.stacked(), np.concatenate([g["fine_U"][-1], g["fine_W"][-1]])) < 1e-10


def test_waveform_relaxation_with_time_dependent_loads_matches_reference():
    P, z, s, ld = _setup()
    g = golden("tv_loads.npz")
    x = g["x"]
    d1 = s.d1
    wr = P.WaveformRelaxation(s, 10, 0.1, 0.1, ld, tol=1e-12, max_iter=400)
    r = wr.solve(P.SplitState.fresh(x[:d1], x[d1:], 0.37))
    assert r.converged
    assert abs(r.iterations - int(g["wr_meta"][0])) <= 1
    assert _rel(r.trajectory.U, g["wr_U"]) < 1e-10 and _rel(r.trajectory.W, g["wr_W"]) < 1e-10


@pytest.mark.parametrize("kind,tag", [("sequential", "seq"), ("all-at-once", "aao")])
def test_parareal_with_time_dependent_loads_matches_reference(kind, tag):
    P, z, s, ld = _setup()
    g = golden("tv_loads.npz")
    props = P.SplitPropagators(s, ld)
    cfg = P.ParerealConfig(time_grid=P.TimeGrid(1.0, 10, 10), alpha=0.1, epsilon=1e-8, k_max=10,
                           fine_kind=kind, fine_tol=1e-12, stop_rule="relative")
    run = P.run_parareal(cfg, props, P.build_fine_propagator(cfg, props, ld),
                         P.SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2)))
    assert run.iterations == int(g[f"{tag}_iters"])
    h = np.array(run.history)
    ref = g[f"{tag}_hist"]
    rel = (np.linalg.norm(h - ref, axis=-1)
           / np.maximum(np.linalg.norm(ref, axis=-1), 1e-300)).max()
    assert rel < 1e-10


def test_constant_rows_reproduce_the_constant_path():
    """A load series whose rows all equal (f1, f2) gives the constant-load results: the
    per-column load terms are the same arithmetic as the baked bias, up to rounding."""
    P, z, s, _ = _setup()
    ld = P.ConstantLoads(z["f1"], z["f2"])

    class Same:
        constant = False

        def at(self, t):
            return z["f1"], z["f2"]

    cfg = P.ParerealConfig(time_grid=P.TimeGrid(1.0, 10, 10), alpha=0.1, epsilon=1e-8, k_max=10,
                           fine_kind="all-at-once", fine_tol=1e-12, stop_rule="relative")
    init = P.SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2))
    a = P.SplitPropagators(s, ld)
    b = P.SplitPropagators(s, Same())
    ra = P.run_parareal(cfg, a, P.build_fine_propagator(cfg, a, ld), init)
    rb = P.run_parareal(cfg, b, P.build_fine_propagator(cfg, b, Same()), init)
    assert ra.iterations == rb.iterations
    assert _rel(np.array(rb.history), np.array(ra.history)) < 1e-11


def test_oracle_agrees_on_a_larger_system():
    """Time-dependent loads at config-2 size (d = 300 + 300, J = 16) against the oracle."""
    import paper_2411_09244_b200 as P

    z = golden("sys_cfg2.npz")
    s = P.CoarseSystem(*(z[k] for k in BLOCKS))
    ld = WaveLoads(z["f1"], z["f2"])
    f1, f2 = z["f1"], z["f2"]
    osys = dataclasses.replace(po.OSystem(*(z[k] for k in BLOCKS), f1, f2),
                               loads_at=ld.at)
    props = P.SplitPropagators(s, ld)
    for kind in ("sequential", "all-at-once"):
        cfg = P.ParerealConfig(time_grid=P.TimeGrid(0.25, 16, 16), alpha=0.1, epsilon=1e-8,
                               k_max=3, fine_kind=kind, fine_tol=1e-12, stop_rule="relative")
        run = P.run_parareal(cfg, props, P.build_fine_propagator(cfg, props, ld),
                             P.SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2)))
        ref = po.run_parareal(osys, np.zeros(s.d1 + s.d2), 0.25, 16, 16, kind=kind, alpha=0.1,
                              epsilon=1e-8, k_max=3, stop="relative", fine_tol=1e-12)
        assert run.iterations == ref["iterations"]
        assert _rel(np.array(run.history), np.array(ref["history"])) < 1e-10, kind
