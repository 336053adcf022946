"""libpe's batched LU inversion (batchlu.cu, SURVEY kernel K3) against LAPACK (numpy).

`pe_shifted_inverses` restates ImplicitAllAtOnce.__init__'s per-mode inverses
(/root/reference/pkg/src/paradiff/allatonce.py:100-110): inv(d_k M11 + A11) for every time
mode, here in one batched pass over the real block forms."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inverse(A):
    import torch

    from paper_2411_09244_b200 import _lib

    lib = _lib.require_cuda()
    batch, n, _ = A.shape
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    dX = torch.full((batch, n, n), float("nan"), dtype=torch.float64, device="cuda")
    info = (C.c_int * batch)()
    _lib.check(lib.pe_batched_inverse(n, batch, C.c_void_p(dA.data_ptr()),
                                      C.c_void_p(dX.data_ptr()), info, None))
    torch.cuda.synchronize()
    assert np.array_equal(dA.cpu().numpy(), A), "input must not be modified"
    return dX.cpu().numpy(), np.array(list(info))


@pytest.mark.parametrize("n,batch", [(1, 1), (2, 3), (5, 2), (31, 2), (32, 1), (33, 3), (64, 2),
                                     (97, 3), (300, 4), (600, 5), (801, 2), (1500, 2), (3100, 2),
                                     (6500, 1)])
def test_batched_inverse_matches_lapack(n, batch):
    """General (non-symmetric, pivoting-needed) matrices: residual at round-off and the
    inverse within cond * eps of numpy's (LAPACK getrf / getri)."""
    rng = np.random.default_rng(n * 1009 + batch)
    A = rng.standard_normal((batch, n, n))
    # make partial pivoting matter: tiny leading entries, one matrix with a zero corner
    A[:, 0, 0] *= 1e-14
    if n > 1:
        A[0, 0, 0] = 0.0
    X, info = _inverse(A)
    assert np.all(info == 0)
    for b in range(batch):
        ref = np.linalg.inv(A[b])
        cond = np.linalg.cond(A[b])
        # rows of the inverse are backward stable: X A = I to round-off, not cond * eps
        res = np.abs(X[b] @ A[b] - np.eye(n)).max()
        assert res < 2e-16 * n * np.abs(X[b]).max() * np.abs(A[b]).max() * 4, (b, res, cond)
        err = np.abs(X[b] - ref).max() / np.abs(ref).max()
        assert err < 1e-15 * cond * n + 1e-13, (b, err, cond)


def test_batched_inverse_is_deterministic_and_batch_invariant():
    """A matrix alone and inside a batch gives the same bits (same pivots, fixed k order)."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((4, 200, 200))
    X1, _ = _inverse(A)
    X2, _ = _inverse(A)
    assert np.array_equal(X1, X2)
    Xs, _ = _inverse(A[2:3])
    assert np.array_equal(Xs[0], X1[2])


def test_tall_panel_cluster_kernel_equals_single_cta_panel(monkeypatch):
    """Panels too tall for one CTA's shared memory run on a thread-block cluster (rows
    split over the CTAs, pivot exchange through distributed shared memory); the
    global-memory single-CTA panel does the same arithmetic: equal bits."""
    rng = np.random.default_rng(8)
    A = rng.standard_normal((3, 1700, 1700))
    X1, i1 = _inverse(A)
    monkeypatch.setenv("PE_LU_CLUSTER", "0")
    X0, i0 = _inverse(A)
    monkeypatch.setenv("PE_LU_CLUSTER", "4")
    X4, _ = _inverse(A)
    assert np.array_equal(X0, X1) and np.array_equal(X4, X1)
    assert np.all(i0 == 0) and np.all(i1 == 0)


def test_batched_inverse_reports_singular_matrices():
    rng = np.random.default_rng(4)
    A = rng.standard_normal((3, 40, 40))
    A[1, 7, :] = 0.0  # an exactly zero row: the factorisation (of A^T) meets a zero pivot 8
    _, info = _inverse(A)
    assert info[0] == 0 and info[2] == 0
    assert info[1] == 8


def _spd(rng, n, scale=1.0):
    Q = rng.standard_normal((n, n))
    return scale * (Q @ Q.T / n + np.eye(n))


@pytest.mark.parametrize("d1,J,sym", [(40, 10, True), (33, 7, True), (64, 1, True),
                                      (50, 12, False), (300, 64, True)])
def test_shifted_inverses_match_reference_formula(d1, J, sym):
    """inv(d_k M11 + A11), d_k = (1 - alpha^(1/J) e^(-2 pi i k / J)) / dt, for all k
    (allatonce.py:58-62, 100-110), against numpy's complex inverses."""
    import torch

    from paper_2411_09244_b200 import _lib

    lib = _lib.require_cuda()
    rng = np.random.default_rng(d1 + J)
    M = _spd(rng, d1)
    A = _spd(rng, d1, 30.0)
    if not sym:
        A = A + 3.0 * rng.standard_normal((d1, d1))
    dt, alpha = 0.01, 0.1
    dM, dA = torch.from_numpy(M).cuda(), torch.from_numpy(A).cuda()
    re = torch.empty((J, d1, d1), dtype=torch.float64, device="cuda")
    im = torch.empty_like(re)
    _lib.check(lib.pe_shifted_inverses(d1, J, dt, alpha, C.c_void_p(dM.data_ptr()),
                                       C.c_void_p(dA.data_ptr()), C.c_void_p(re.data_ptr()),
                                       C.c_void_p(im.data_ptr()), None))
    got = re.cpu().numpy() + 1j * im.cpu().numpy()
    k = np.arange(J)
    dk = (1.0 - alpha ** (1.0 / J) * np.exp(-2j * np.pi * k / J)) / dt
    for q in range(J):
        S = dk[q] * M + A
        ref = np.linalg.inv(S)
        err = np.abs(got[q] - ref).max() / np.abs(ref).max()
        assert err < 1e-12, (q, err)
        assert np.abs(S @ got[q] - np.eye(d1)).max() < 1e-11


def test_shifted_inverses_singular_pencil_raises():
    import torch

    from paper_2411_09244_b200 import _lib

    lib = _lib.require_cuda()
    d1 = 8
    M = torch.zeros((d1, d1), dtype=torch.float64, device="cuda")
    A = torch.zeros((d1, d1), dtype=torch.float64, device="cuda")
    out = torch.empty((4, d1, d1), dtype=torch.float64, device="cuda")
    rc = lib.pe_shifted_inverses(d1, 4, 0.1, 0.1, C.c_void_p(M.data_ptr()),
                                 C.c_void_p(A.data_ptr()), C.c_void_p(out.data_ptr()),
                                 C.c_void_p(out.data_ptr()), None)
    assert rc != 0
    assert b"singular" in lib.pe_last_error()
