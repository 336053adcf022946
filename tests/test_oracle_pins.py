"""Pin the CPU oracle to golden vectors produced by the unmodified reference.

The fixtures in tests/golden/ were written by oracle/make_golden.py, which imports the
reference (`/root/reference/pkg/src/paradiff`) in the build container and runs it on
seeded inputs.  If the oracle restatement drifts from the reference these fail.
"""

import json

import numpy as np
import pytest

from oracle import pe_oracle as po
from tests.conftest import golden


def _sys(z, prefix=""):
    g = lambda k: z[prefix + k]  # noqa: E731
    return po.OSystem(g("M11"), g("A11"), g("M12"), g("A12"), g("M22"), g("A22"),
                      g("f1"), g("f2"))


def tiny(f1=(0.3,), f2=(-0.2,)):
    return po.OSystem(np.array([[2.0]]), np.array([[3.0]]), np.array([[0.5]]),
                      np.array([[0.4]]), np.array([[1.5]]), np.array([[0.7]]),
                      np.array(f1), np.array(f2))


def test_split_and_coarse_step_tiny():
    z = golden("units.npz")
    o = po.OracleSplit(tiny())
    u, w = o.split_step(np.array([1.0]), np.array([2.0]), np.array([0.8]), np.array([1.5]), 0.01)
    np.testing.assert_allclose(np.concatenate([u, w]), z["tiny_split"], rtol=1e-14)
    o2 = po.OracleSplit(tiny((0.3,), (-0.2,)))
    g = o2.coarse_step(np.array([0.7, -0.3]), 0.02)
    np.testing.assert_allclose(g, z["tiny_coarse"], rtol=1e-14)
    U, W = o.fine_interval(np.array([1.0]), np.array([2.0]), 0.05, 7)
    np.testing.assert_allclose(U, z["tiny_fine_U"], rtol=1e-14)
    np.testing.assert_allclose(W, z["tiny_fine_W"], rtol=1e-14)


def test_build_rhs_hand_values():
    z = golden("units.npz")
    s = tiny((0.2,), (0.0,))
    rhs = po.build_rhs(s, np.array([[0.2], [0.2]]), np.array([1.0]), np.array([2.0]),
                       np.array([2.0]), np.array([[2.5], [3.0]]), np.array([0.9]), 0.1, 0.3)
    np.testing.assert_allclose(rhs, [[14.0], [-3.3]], atol=1e-13)
    np.testing.assert_array_equal(rhs, z["rhs_hand"])


def test_max_state_diff_known_answer():
    prev = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 2.0]])
    new = np.array([[9.0, 9.0], [1.0, 3.0], [0.0, 2.0]])
    assert po.max_state_diff(prev, new) == 3.0


def test_random_system_functions_bitwise():
    z = golden("units.npz")
    s = _sys(z, "rand_")
    o = po.OracleSplit(s)
    x0 = z["rand_x0"]
    u, w = o.split_step(x0[:5], x0[5:], x0[:5] * 0.9, x0[5:] * 1.1, 1e-3)
    np.testing.assert_array_equal(np.concatenate([u, w]), z["rand_split"])
    np.testing.assert_array_equal(o.coarse_step(x0, 0.04), z["rand_coarse"])
    U, W = o.fine_interval(x0[:5], x0[5:], 0.04, 16)
    np.testing.assert_array_equal(U, z["rand_fine_U"])
    np.testing.assert_array_equal(W, z["rand_fine_W"])
    r = po.OracleWR(s, 16, 0.04, 0.3, tol=1e-13, max_iter=400).solve(x0[:5], x0[5:])
    np.testing.assert_array_equal(r["U"], z["rand_wr_U"])
    np.testing.assert_array_equal(r["W"], z["rand_wr_W"])
    np.testing.assert_array_equal(np.array(r["residuals"]), z["rand_wr_res"])
    assert r["iterations"] == z["rand_wr_meta"][0]


@pytest.mark.parametrize("kind,tag", [("sequential", "seq"), ("all-at-once", "aao")])
def test_random_system_parareal(kind, tag):
    z = golden("units.npz")
    s = _sys(z, "rand_")
    r = po.run_parareal(s, z["rand_x0"], 0.32, 8, 16, kind=kind, alpha=0.3, epsilon=1e-10,
                        k_max=8, fine_tol=1e-13)
    assert r["iterations"] == int(z[f"rand_par_{tag}_iters"])
    np.testing.assert_array_equal(np.array(r["history"]), z[f"rand_par_{tag}_hist"])
    r = po.run_parareal(s, z["rand_x0"], 0.32, 8, 16, kind=kind, alpha=0.3, epsilon=0.0,
                        k_max=8, fine_tol=1e-13)
    np.testing.assert_array_equal(np.array(r["history"]), z[f"rand_exact_{tag}_hist"])


def test_lowgamma_and_floor_stop():
    z = golden("units.npz")
    g = po.OSystem(np.eye(2), np.diag([200.0, 100.0]), np.diag([0.3, 0.1]), np.zeros((2, 2)),
                   np.eye(2), np.diag([0.5, 0.5]), np.array([1.0, 1.0]), np.array([1.0, -1.0]))
    r = po.OracleWR(g, 8, 0.01, 0.1, tol=1e-13, max_iter=200).solve(np.zeros(2), np.zeros(2))
    np.testing.assert_array_equal(np.array(r["residuals"]), z["lowgamma_res"])
    g2 = po.OSystem(*[getattr(g, k) for k in ("M11", "A11", "M12", "A12", "M22", "A22")],
                    np.array([1.0, 0.0]), np.array([0.0, 1.0]))
    r = po.OracleWR(g2, 8, 0.01, 0.1, tol=1e-18, max_iter=500).solve(np.zeros(2), np.zeros(2))
    assert r["iterations"] == z["floor_meta"][0]
    assert po.STOP_REASONS.index(r["stop_reason"]) == z["floor_meta"][1]


def test_degenerate_spaces():
    z = golden("units.npz")
    us = po.OSystem(np.array([[1.0]]), np.array([[6.0]]), np.zeros((1, 0)), np.zeros((1, 0)),
                    np.zeros((0, 0)), np.zeros((0, 0)), np.array([2.4]), np.zeros(0))
    r = po.run_parareal(us, np.array([1.0]), 0.8, 8, 16, epsilon=1e-15, k_max=50)
    np.testing.assert_array_equal(np.array(r["history"]), z["uonly_hist"])
    kappa = 1.0 / (1.0 + 0.8 / 128 * 6.0)
    assert np.isclose(r["history"][-1][-1][0], 0.4 + kappa ** 128 * 0.6, rtol=1e-12)
    ws = po.OSystem(np.zeros((0, 0)), np.zeros((0, 0)), np.zeros((0, 1)), np.zeros((0, 1)),
                    np.array([[2.0]]), np.array([[3.0]]), np.zeros(0), np.array([0.6]))
    for kind, tag in (("sequential", "seq"), ("all-at-once", "aao")):
        r = po.run_parareal(ws, np.array([1.0]), 0.4, 5, 4, kind=kind, alpha=0.5,
                            epsilon=1e-15, k_max=5, fine_tol=1e-13)
        np.testing.assert_array_equal(np.array(r["history"]), z[f"wonly_{tag}_hist"])


@pytest.mark.parametrize("tag,n,J,kind", [("seq", 6, 4, "sequential"),
                                          ("aao", 5, 6, "all-at-once")])
def test_channel_fixture_exactness(tag, n, J, kind):
    z = golden("channel.npz")
    s = _sys(z)
    r = po.run_parareal(s, np.zeros(s.d1 + s.d2), 0.005, n, J, kind=kind, alpha=0.5,
                        epsilon=0.0, k_max=n, fine_tol=1e-13)
    np.testing.assert_array_equal(np.array(r["history"]), z[f"{tag}_hist"])


@pytest.mark.parametrize("run_name", ["run_cfg0_seq.npz", "run_cfg1_aao.npz"])
def test_config_runs_match_reference(run_name):
    z = golden(run_name)
    sz = golden("sys_cfg0.npz")
    meta = json.loads(str(sz["meta"]))
    assert abs(meta["dt_over_bound"] - 0.4) < 1e-6
    s = _sys(sz)
    kind = str(z["kind"])
    r = po.run_parareal(s, np.zeros(s.d1 + s.d2), 1.0, 10, 10, kind=kind, alpha=0.1,
                        epsilon=1e-8, k_max=10, stop="relative", fine_tol=1e-12)
    assert r["iterations"] == int(z["iterations"])
    h = np.array(r["history"])
    ref = z["history"]
    num = np.linalg.norm(h - ref, axis=-1)
    den = np.maximum(np.linalg.norm(ref, axis=-1), 1e-300)
    assert (num / den).max() < 1e-12
    np.testing.assert_allclose(r["max_diffs"], z["max_diffs"], rtol=1e-8)
    if kind == "all-at-once":
        its = np.array([[i["iterations"] for i in sw] for sw in r["fine_info"]])
        np.testing.assert_array_equal(its, z["wr_iterations"])


def test_config_kappa_and_fine_assembly_pinned():
    """The harness's kappa generator and Q1 assembly (oracle/configs.py) reproduce the
    reference's fine operators of config 0 (fine_cfg0.npz: M and the kappa-rescaled A)."""
    import json

    import scipy.sparse as sp

    from oracle.configs import assemble_fine, kappa_field

    z = golden("fine_cfg0.npz")
    scale = json.loads(str(golden("sys_cfg0.npz")["meta"]))["kappa_scale"]
    M, A = assemble_fine(40, kappa_field("cfg0"))

    def ref(prefix):
        return sp.csr_matrix((z[prefix + "_val"], z[prefix + "_idx"], z[prefix + "_ptr"]),
                             shape=tuple(z[prefix + "_shape"]))

    assert abs(M - ref("M")).max() <= 1e-15 * abs(ref("M")).max()
    assert abs(A * scale - ref("A")).max() <= 1e-14 * abs(ref("A")).max()


def _wave(z):
    f1, f2 = z["f1"], z["f2"]
    return lambda t: (f1 * (1.0 + 0.5 * np.sin(2.0 * np.pi * t)),
                      f2 * (1.0 - 0.3 * np.cos(2.0 * np.pi * t)) + 0.01 * t)


def test_oracle_time_dependent_loads_pinned():
    """The oracle's time-dependent-load paths (loads at t + dt in the split / coarse steps,
    at t0 + s dt in the WR rows, state times carried through parareal) against the
    unmodified reference (tests/golden/tv_loads.npz, oracle/make_tv_golden.py)."""
    import dataclasses

    g = golden("tv_loads.npz")
    z = golden("sys_cfg0.npz")
    s = dataclasses.replace(_sys(z), loads_at=_wave(z))
    o = po.OracleSplit(s)
    x = g["x"]
    d1 = s.d1
    un, wn = o.split_step(x[:d1], x[d1:], x[:d1] * 0.9, x[d1:] * 1.1, 0.01, 0.37)
    np.testing.assert_allclose(np.concatenate([un, wn]), g["split"], rtol=1e-12, atol=1e-18)
    # coarse_step reads the current state only
    np.testing.assert_allclose(o.coarse_step(x, 0.1, 0.37), g["coarse"], rtol=1e-12, atol=1e-18)
    U, W, t1 = o.fine_interval(x[:d1], x[d1:], 0.1, 10, 0.37, return_t=True)
    np.testing.assert_allclose(U, g["fine_U"], rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(W, g["fine_W"], rtol=1e-12, atol=1e-18)
    assert t1 == float(g["fine_t"])
    r = po.OracleWR(s, 10, 0.1, 0.1, tol=1e-12, max_iter=400).solve(x[:d1], x[d1:], 0.37)
    assert r["iterations"] == int(g["wr_meta"][0])
    np.testing.assert_allclose(r["U"], g["wr_U"], rtol=1e-10, atol=1e-16)
    for kind, tag in (("sequential", "seq"), ("all-at-once", "aao")):
        ref = po.run_parareal(s, np.zeros(s.d1 + s.d2), 1.0, 10, 10, kind=kind, alpha=0.1,
                              epsilon=1e-8, k_max=10, stop="relative", fine_tol=1e-12)
        assert ref["iterations"] == int(g[f"{tag}_iters"])
        h = np.array(ref["history"])
        assert np.abs(h - g[f"{tag}_hist"]).max() <= 1e-10 * np.abs(g[f"{tag}_hist"]).max()
