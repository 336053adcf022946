"""CPU check of the modal WR formulation that libpe's all-at-once path implements
(paper_2411_09244_b200/csrc/wr_modal.cu).

The reference sweep (allatonce.py:220-298, restated in oracle/pe_oracle.py) is re-derived
here in the generalized eigenbases of (A11, M11) and (A22, M22): the shifted solves become
one scalar time recurrence per mode with a corner closure, the w recursion a scalar
recurrence per mode, and the residual norms use U = chol(V^T V)^T.  This NumPy model of
the GPU arithmetic must reproduce the oracle's iterates: same sweep counts (to within the
round-off floor) and final states to 1e-12.  It documents that the reformulation is exact
algebra, not an approximation; the GPU kernels are checked against the oracle in
tests/test_gpu_parity.py.
"""

import numpy as np
import pytest
from scipy.linalg import cholesky, eigh

from oracle import pe_oracle as po
from tests.conftest import golden


def modal_wr_solve(s: po.OSystem, u0, w0, J, dt_interval, alpha, tol, max_iter):
    dt = dt_interval / J
    mu1, V1 = eigh(s.A11, s.M11)
    mu2, V2 = eigh(s.A22, s.M22)
    U1 = cholesky(V1.T @ V1)  # upper: ||U1 e|| = ||V1 e||
    U2 = cholesky(V2.T @ V2)
    Rz = -V1.T @ s.A12 @ V2
    Rd = -V1.T @ s.M12 @ V2 / dt
    f1t = V1.T @ s.f1
    Gu = -dt * V2.T @ s.A12.T @ V1
    Gd = -V2.T @ s.M12.T @ V1
    cg = dt * V2.T @ s.f2
    a = 1.0 / (1.0 + mu1 * dt)
    cden = 1.0 / (1.0 - alpha * a ** J)
    lam = 1.0 - dt * mu2
    y0 = V1.T @ s.M11 @ u0
    z0 = V2.T @ s.M22 @ w0
    Y = np.tile(y0, (J, 1))
    Z = np.tile(z0, (J, 1))
    res, stall, prev, reason, it = [], 0, np.inf, "max_iter", 0
    for _ in range(max_iter):
        it += 1
        zh = np.vstack([z0, z0, Z[:-1]])
        R = zh[1:] @ Rz.T + (zh[1:] - zh[:-1]) @ Rd.T + f1t
        R[0] += (y0 - alpha * Y[-1]) / dt
        c = np.zeros_like(y0)
        for t in range(1, J):
            c = a * (c + dt * R[t])
        Yn = np.empty_like(Y)
        Yn[0] = a * (alpha * c + dt * R[0]) * cden
        for t in range(1, J):
            Yn[t] = a * (Yn[t - 1] + dt * R[t])
        yh = np.vstack([y0, y0, Yn[:-1]])
        H = Yn @ Gu.T + (yh[1:] - yh[:-1]) @ Gd.T + cg
        Zn = np.empty_like(Z)
        z = z0
        for t in range(J):
            z = lam * z + H[t]
            Zn[t] = z
        r = (np.linalg.norm((Yn - Y) @ U1.T, axis=1).max()
             + np.linalg.norm((Zn - Z) @ U2.T, axis=1).max())
        res.append(r)
        Y, Z = Yn, Zn
        if r <= tol:
            reason = "tol"
            break
        if not np.isfinite(r) or r > 1e8 * max(1.0, res[0]):
            reason = "diverged"
            break
        stall = stall + 1 if r >= prev else 0
        if stall >= 2 and r <= 1e3 * tol:
            reason = "floor"
            break
        prev = r
    return V1 @ Y[-1], V2 @ Z[-1], it, reason, res


def _random_spd_system(d1, d2, seed):
    rng = np.random.default_rng(seed)
    n = d1 + d2
    q = rng.standard_normal((2 * n, n))
    mass = q.T @ q / (2 * n) + 0.5 * np.eye(n)
    r = rng.standard_normal((2 * n, n))
    stiff = r.T @ r / (2 * n) + 0.1 * np.eye(n)
    f = rng.standard_normal(n)
    return po.OSystem(mass[:d1, :d1], stiff[:d1, :d1], mass[:d1, d1:], stiff[:d1, d1:],
                      mass[d1:, d1:], stiff[d1:, d1:], f[:d1], f[d1:])


@pytest.mark.parametrize("d1,d2,J,alpha", [(6, 5, 8, 0.2), (12, 12, 16, 0.1), (9, 14, 5, 0.5)])
def test_modal_sweep_equals_reference_sweep_random(d1, d2, J, alpha):
    s = _random_spd_system(d1, d2, 100 * d1 + d2)
    rng = np.random.default_rng(J)
    u0, w0 = rng.standard_normal(d1), rng.standard_normal(d2)
    ref = po.OracleWR(s, J, 0.05, alpha, tol=1e-13, max_iter=400).solve(u0, w0)
    u, w, it, reason, res = modal_wr_solve(s, u0, w0, J, 0.05, alpha, 1e-13, 400)
    assert abs(it - ref["iterations"]) <= 2
    np.testing.assert_allclose(res[:5], ref["residuals"][:5], rtol=1e-9)
    fin = np.concatenate([ref["U"][-1], ref["W"][-1]])
    assert np.linalg.norm(np.concatenate([u, w]) - fin) <= 1e-12 * np.linalg.norm(fin)


def test_modal_sweep_equals_reference_sweep_cfg0():
    """The reference-built cfg0 operators (d = 32 + 32, J = 10, alpha = 0.1)."""
    z = golden("sys_cfg0.npz")
    s = po.OSystem.from_arrays(z)
    rng = np.random.default_rng(0)
    u0, w0 = 0.1 * rng.standard_normal(s.d1), 0.1 * rng.standard_normal(s.d2)
    ref = po.OracleWR(s, 10, 0.1, 0.1, tol=1e-12, max_iter=400).solve(u0, w0)
    u, w, it, reason, res = modal_wr_solve(s, u0, w0, 10, 0.1, 0.1, 1e-12, 400)
    assert abs(it - ref["iterations"]) <= 2
    fin = np.concatenate([ref["U"][-1], ref["W"][-1]])
    assert np.linalg.norm(np.concatenate([u, w]) - fin) <= 1e-12 * np.linalg.norm(fin)


def test_corner_closure_solves_shifted_time_system():
    """(B + mu) y = r with B the alpha-corner time matrix (allatonce.py:36-67): the scalar
    recurrence with the corner closure equals a dense solve."""
    J, dt, alpha = 12, 0.01, 0.3
    B = po.time_matrix_dense(J, dt, alpha)
    rng = np.random.default_rng(1)
    for mu in (0.0, 3.7, 250.0):
        r = rng.standard_normal(J)
        a = 1.0 / (1.0 + mu * dt)
        c = 0.0
        for t in range(1, J):
            c = a * (c + dt * r[t])
        y = np.empty(J)
        y[0] = a * (alpha * c + dt * r[0]) / (1.0 - alpha * a ** J)
        for t in range(1, J):
            y[t] = a * (y[t - 1] + dt * r[t])
        np.testing.assert_allclose(y, np.linalg.solve(B + mu * np.eye(J), r), rtol=1e-12)
