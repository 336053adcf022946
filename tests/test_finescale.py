"""Fine-scale accuracy path: the GPU backward-Euler reference solve
and Eq (31) error series against the reference's golden vectors (tests/golden/
fine_cfg0.npz, written by oracle/make_fine_golden.py from the unmodified reference), and
the artifact writers byte-for-byte against the reference's own CSV output.

Tolerances.  The GPU reference solve applies an explicit inverse (R = K^-1 M / dt,
c = K^-1 b) where the reference back-substitutes a sparse LU each step: rounding differs
at cond(K) * eps per step, so trajectory rows are compared at 1e-10 relative L2.  The
error series differs from the reference only in summation order: 1e-12 relative.
"""

import json
import types

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pe_oracle as po
from tests.conftest import golden

REL_TRAJ = 1e-10
REL_SERIES = 1e-12


def _csr(z, p):
    return sp.csr_matrix((z[f"{p}_val"], z[f"{p}_idx"], z[f"{p}_ptr"]), shape=tuple(z[f"{p}_shape"]))


def _fixture():
    z = golden("fine_cfg0.npz")
    ops = types.SimpleNamespace(M=_csr(z, "M"), A=_csr(z, "A"))
    space = types.SimpleNamespace(Psi1=_csr(z, "P1"), Psi2=_csr(z, "P2"))
    return z, ops, space


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ------------------------------------------------------------------ CPU: oracle pins


def test_oracle_reference_solve_pinned():
    z, ops, _ = _fixture()
    traj = po.fine_reference_solve(ops.M, ops.A, z["b"], 1.0, 100)
    assert np.array_equal(traj[::10], z["traj"])
    short = po.fine_reference_solve(ops.M, ops.A, z["b"], 0.05, 7, u0=z["u0"],
                                    keep_trajectory=False)
    assert np.array_equal(short, z["short"])


def test_oracle_error_series_pinned():
    z, ops, space = _fixture()
    hist = golden("run_cfg0_seq.npz")["history"]
    s = po.error_series(ops.M, space.Psi1.tocsc(), space.Psi2.tocsc(), z["traj"][-1], hist)
    np.testing.assert_allclose(s, z["series"], rtol=1e-14)
    assert po.relative_error(ops.M, np.zeros(ops.M.shape[0]), np.zeros(ops.M.shape[0])) == 0.0
    assert po.relative_error(ops.M, np.zeros(ops.M.shape[0]), np.ones(ops.M.shape[0])) == np.inf


def test_writers_match_reference_bytes(tmp_path):
    """conv / timings / wr_residuals CSVs are byte-identical to the reference's writers
    (util.py:36-50 via experiment.py:418-441) for the same run record."""
    from paper_2411_09244_b200.experiment import write_run_artifacts

    z, _, _ = _fixture()
    fine_info = [[{"residuals": r} for r in sw] for sw in json.loads(str(z["w_residuals"]))]
    run = types.SimpleNamespace(max_diffs=list(z["w_max_diffs"]),
                                fine_seconds=list(z["w_fine_seconds"]),
                                coarse_seconds=list(z["w_coarse_seconds"]), fine_info=fine_info)
    files = write_run_artifacts(tmp_path, 10, run, list(z["series"]),
                                solution_grid=np.arange(6.0).reshape(2, 3) / 7)
    assert [f.name for f in files] == ["conv_N10.csv", "timings_N10.csv", "wr_residuals_N10.csv",
                                       "solution_N10.txt"]
    assert (tmp_path / "conv_N10.csv").read_text() == str(z["csv_conv"])
    assert (tmp_path / "timings_N10.csv").read_text() == str(z["csv_timings"])
    assert (tmp_path / "wr_residuals_N10.csv").read_text() == str(z["csv_wr"])
    back = np.loadtxt(tmp_path / "solution_N10.txt")
    assert np.array_equal(back, np.arange(6.0).reshape(2, 3) / 7)


def test_node_values_on_grid():
    from paper_2411_09244_b200.fem import node_values_on_grid

    z, _, _ = _fixture()
    nx = int(z["nx"])
    grid = types.SimpleNamespace(n_nodes=(nx + 1) ** 2, interior=z["interior"], nx=nx, ny=nx)
    full = node_values_on_grid(grid, np.arange(int(z["n_interior"]), dtype=float) + 1)
    assert full.shape == (nx + 1, nx + 1)
    assert full[0].sum() == 0 and full[:, 0].sum() == 0 and full[-1].sum() == 0
    assert full[1, 1] == 1.0


# ------------------------------------------------------------------ GPU parity


@pytest.mark.gpu
def test_gpu_reference_solve_matches_reference():
    from paper_2411_09244_b200 import fem

    z, ops, _ = _fixture()
    tm = {}
    times, traj = fem.reference_solve(ops, z["b"], 1.0, 100, timing=tm)
    assert traj.shape == (101, ops.M.shape[0]) and times[-1] == 1.0
    for r, g in zip(traj[::10], z["traj"]):
        assert _rel(r, g) < REL_TRAJ or np.linalg.norm(g) == 0
    assert tm["step_ms"] > 0
    times, short = fem.reference_solve(ops, z["b"], 0.05, 7, u0=z["u0"], keep_trajectory=False)
    assert short.shape == (2, ops.M.shape[0]) and list(times) == [0.0, 0.05]
    assert np.array_equal(short[0], z["u0"])
    assert _rel(short[1], z["short"][1]) < REL_TRAJ


@pytest.mark.gpu
def test_gpu_reference_solve_odd_sizes_vs_oracle(rng):
    """Odd n (unaligned rows), n < 32 and n_steps = 1 against the oracle's splu."""
    from paper_2411_09244_b200 import fem

    for n, steps in ((1, 3), (7, 1), (33, 5), (257, 9)):
        T = sp.random(n, n, density=0.3, random_state=int(rng.integers(1 << 30))).toarray()
        Mm = sp.csr_matrix(np.eye(n) * 2 + 0.1 * (T + T.T) / max(1, n) ** 0.5)
        Am = sp.csr_matrix(np.eye(n) + np.diag(np.full(n - 1, -0.3), 1) + np.diag(np.full(n - 1, -0.3), -1))
        b = rng.standard_normal(n)
        u0 = rng.standard_normal(n)
        ops = types.SimpleNamespace(M=Mm, A=Am)
        ref = po.fine_reference_solve(Mm, Am, b, 0.3, steps, u0=u0)
        _, got = fem.reference_solve(ops, b, 0.3, steps, u0=u0)
        for r, g in zip(got, ref):
            assert _rel(r, g) < 1e-12, (n, steps)


def _fem_like(m, seed):
    """Mass / stiffness with the fine operators' structure on an m x m interior grid."""
    rng = np.random.default_rng(seed)
    one = np.ones(m)
    T1 = sp.diags([one[:-1], 4 * one, one[:-1]], [-1, 0, 1])
    M = (sp.kron(T1, T1) / (36.0 * (m + 1) ** 2)).tocsr()
    G1 = sp.diags([np.ones(m), -np.ones(m)], [0, -1], shape=(m + 1, m))
    I = sp.identity(m)
    Gx, Gy = sp.kron(I, G1).tocsr(), sp.kron(G1, I).tocsr()
    kx = np.where(rng.random(Gx.shape[0]) < 0.1, 1e4, 1.0)
    ky = np.where(rng.random(Gy.shape[0]) < 0.1, 1e4, 1.0)
    A = (Gx.T @ sp.diags(kx) @ Gx + Gy.T @ sp.diags(ky) @ Gy).tocsr() * 1e-3
    return M, A, rng.standard_normal(m * m)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [64, 67, 90])
def test_gpu_reference_solve_packed_symmetric_path(m, monkeypatch):
    """n = m^2 >= 4096 takes the packed lower-triangle path (partial last tile for m = 67,
    90): equal to the oracle's splu and to the dense-R path within 1e-12."""
    from paper_2411_09244_b200 import fem

    M, A, u0 = _fem_like(m, m)
    b = np.full(m * m, 1.0 / (m + 1) ** 2)
    ops = types.SimpleNamespace(M=M, A=A)
    ref = po.fine_reference_solve(M, A, b, 0.02, 6, u0=u0)
    _, got = fem.reference_solve(ops, b, 0.02, 6, u0=u0)
    for r, g in zip(got, ref):
        assert _rel(r, g) < 1e-12
    _, ends = fem.reference_solve(ops, b, 0.02, 6, u0=u0, keep_trajectory=False)
    assert np.array_equal(ends[0], u0) and np.array_equal(ends[1], got[-1])  # same kernels
    monkeypatch.setenv("PE_FINE_NO_TMA", "1")  # per-tile CTAs instead of the TMA ring
    _, plain = fem.reference_solve(ops, b, 0.02, 6, u0=u0)
    assert _rel(plain[-1], got[-1]) < 1e-13
    monkeypatch.setenv("PE_FINE_NO_SYM", "1")
    _, dense = fem.reference_solve(ops, b, 0.02, 6, u0=u0)
    assert _rel(dense[-1], got[-1]) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("m,steps", [(20, 5), (63, 6), (64, 4), (100, 7), (150, 3)])
def test_gpu_reference_solve_chain_solver(m, steps, monkeypatch):
    """The block-tridiagonal chain solver (finechain.cu; default above 16384 nodes, forced
    here): block sizes 64 .. 192, partial last block, one and several ring chunks, against
    the oracle's splu (fem.py:292-318) and the dense path."""
    from paper_2411_09244_b200 import fem

    M, A, u0 = _fem_like(m, 100 + m)
    b = np.full(m * m, 1.0 / (m + 1) ** 2)
    ops = types.SimpleNamespace(M=M, A=A)
    ref = po.fine_reference_solve(M, A, b, 0.02, steps, u0=u0)
    monkeypatch.setenv("PE_FINE_CHAIN", "1")
    tm = {}
    _, got = fem.reference_solve(ops, b, 0.02, steps, u0=u0, timing=tm)
    assert got.shape == ref.shape and tm["step_ms"] > 0
    for r, g in zip(got, ref):
        assert _rel(r, g) < 1e-11, (m, steps)
    _, ends = fem.reference_solve(ops, b, 0.02, steps, u0=u0, keep_trajectory=False)
    assert np.array_equal(ends[0], u0) and np.array_equal(ends[1], got[-1])
    monkeypatch.setenv("PE_FINE_CHAIN", "0")
    _, dense = fem.reference_solve(ops, b, 0.02, steps, u0=u0)
    assert _rel(dense[-1], got[-1]) < 1e-11


@pytest.mark.gpu
def test_gpu_reference_solve_chain_solver_is_default_for_large_grids():
    """n = 150^2 = 22500 > 16384 takes the chain solver without any switch, and a grid
    above the dense path's 65535-node cap (257^2) runs at all."""
    from paper_2411_09244_b200 import fem

    for m, steps in ((150, 2), (257, 2)):
        M, A, u0 = _fem_like(m, 7)
        b = np.full(m * m, 1.0 / (m + 1) ** 2)
        ops = types.SimpleNamespace(M=M, A=A)
        ref = po.fine_reference_solve(M, A, b, 0.01, steps, u0=u0)
        _, got = fem.reference_solve(ops, b, 0.01, steps, u0=u0)
        assert _rel(got[-1], ref[-1]) < 1e-11, m


@pytest.mark.gpu
def test_gpu_error_series_matches_reference():
    from paper_2411_09244_b200 import fem

    z, ops, space = _fixture()
    hist = golden("run_cfg0_seq.npz")["history"]
    got = fem.error_series(ops, space, z["traj"][-1], hist[:, -1, :])
    np.testing.assert_allclose(got, z["series"], rtol=REL_SERIES)
    # one endpoint through relative_error on fine vectors
    x = hist[-1, -1]
    d1 = space.Psi1.shape[1]
    y = space.Psi1 @ x[:d1] + space.Psi2 @ x[d1:]
    assert abs(fem.relative_error(ops, z["traj"][-1], y) - z["series"][-1]) < REL_SERIES * z["series"][-1]


@pytest.mark.gpu
def test_gpu_error_edge_cases():
    from paper_2411_09244_b200 import fem
    from paper_2411_09244_b200._lib import PeError

    z, ops, space = _fixture()
    n = ops.M.shape[0]
    assert fem.relative_error(ops, np.zeros(n), np.zeros(n)) == 0.0
    assert fem.relative_error(ops, np.zeros(n), np.ones(n)) == np.inf
    assert fem.error_series(ops, space, z["traj"][-1], np.zeros((0, 64))) == []
    with pytest.raises(ValueError):
        fem.reference_solve(ops, z["b"], 1.0, 0)
    with pytest.raises(ValueError):
        fem.reference_solve(ops, z["b"][:-1], 1.0, 5)
    bad = types.SimpleNamespace(M=sp.csr_matrix(np.eye(3)), A=sp.csr_matrix(-5 * np.eye(3)))
    with pytest.raises(PeError):
        fem.reference_solve(bad, np.ones(3), 1.0, 1)


@pytest.mark.gpu
def test_gpu_project_coarse_matches_reference_blocks():
    """Galerkin projection (msbasis.py:545-572) against the reference's cfg0 CoarseSystem
    (sys_cfg0.npz: M blocks as projected; A blocks projected then scaled by kappa_scale,
    here the fine A is scaled first) and its loads: 1e-12 relative to the block's max."""
    import paper_2411_09244_b200 as P

    z, ops, space = _fixture()
    ref = golden("sys_cfg0.npz")
    cs = P.project_coarse(space.Psi1, space.Psi2, ops)
    for k in ("M11", "A11", "M12", "A12", "M22", "A22"):
        g, r = getattr(cs, k), ref[k]
        assert g.shape == r.shape
        assert np.abs(g - r).max() <= 1e-12 * np.abs(r).max(), k
    assert np.array_equal(cs.M11, cs.M11.T) and np.array_equal(cs.A22, cs.A22.T)
    f1, f2 = P.project_load(space, z["b"])  # reference signature (no ops)
    g1, g2 = P.project_load(space, z["b"], ops)  # round-1 signature still accepted
    assert np.array_equal(f1, g1) and np.array_equal(f2, g2)
    np.testing.assert_allclose(f1, ref["f1"], rtol=1e-12, atol=1e-14 * np.abs(ref["f1"]).max())
    np.testing.assert_allclose(f2, ref["f2"], rtol=1e-12, atol=1e-14 * np.abs(ref["f2"]).max())
    # degenerate split (d2 = 0) and a bad basis
    cs0 = P.project_coarse(sp.hstack([space.Psi1, space.Psi2]).tocsr(), sp.csr_matrix((ops.M.shape[0], 0)), ops)
    assert cs0.M22.shape == (0, 0) and cs0.M11.shape == (64, 64)
    with pytest.raises(ValueError):
        P.project_coarse(space.Psi1[:-1], space.Psi2[:-1], ops)


@pytest.mark.gpu
def test_gpu_run_single_accuracy_matches_reference(tmp_path):
    """experiment.run_single (experiment.py:328-360) on config 0: parareal iterations and
    history as the reference run, error series as the reference's within 1e-10, and the
    writers on its record."""
    import paper_2411_09244_b200 as P
    from paper_2411_09244_b200.experiment import run_single, write_run_artifacts

    z, ops, space = _fixture()
    sysz = golden("sys_cfg0.npz")
    gold = golden("run_cfg0_seq.npz")
    space.system = P.CoarseSystem(*[sysz[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")])
    cfg = types.SimpleNamespace(time_grid=lambda n: P.TimeGrid(1.0, n, n), alpha=0.1,
                                epsilon=1e-8, k_max=10, fine_kind="sequential", workers=1,
                                compute_reference=True, to_source=lambda: z["b"], t_end=1.0)
    pipe = types.SimpleNamespace(config=cfg, space=space, ops=ops,
                                 loads=P.ConstantLoads(sysz["f1"], sysz["f2"]))
    res = run_single(pipe, 10, stop_rule="relative")
    assert res.run.iterations == int(gold["iterations"])
    h = np.array(res.run.history)
    assert max(_rel(a, b) for a, b in zip(h.reshape(len(h), -1), gold["history"].reshape(len(h), -1))) < 1e-10
    np.testing.assert_allclose(res.error_series, z["series"], rtol=1e-10)
    assert res.relative_error == res.error_series[-1] and res.dt_sub == 0.01
    files = write_run_artifacts(tmp_path, 10, res.run, res.error_series)
    assert len(files) == 3 and (tmp_path / "conv_N10.csv").read_text().startswith("iteration,")
