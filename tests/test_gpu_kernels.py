"""Kernel-level GPU tests: the FP64 DMMA GEMM against a torch FP64 reference."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(A, B, a_str, b_str, M, N, K, c_layout="col"):
    import torch

    from paper_2411_09244_b200 import _lib

    lib = _lib.require_cuda()
    Cm = torch.full((M * N + 1,), float("nan"), dtype=torch.float64, device="cuda")
    ci, cj = (1, M) if c_layout == "col" else (N, 1)
    _lib.check(lib.pe_gemm_f64(M, N, K, 1, C.c_void_p(A.data_ptr()), a_str[0], a_str[1], 0,
                               C.c_void_p(B.data_ptr()), b_str[0], b_str[1], 0,
                               C.c_void_p(Cm.data_ptr()), ci, cj, 0, None))
    torch.cuda.synchronize()
    out = Cm[: M * N].reshape(N, M).T if c_layout == "col" else Cm[: M * N].reshape(M, N)
    return out.cpu().numpy()


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (65, 33, 129),
                                   (300, 64, 600), (600, 4096, 300), (128, 19200, 64)])
@pytest.mark.parametrize("a_rowmajor,b_colmajor", [(True, True), (True, False),
                                                   (False, True), (False, False)])
def test_gemm_matches_torch_fp64(M, N, K, a_rowmajor, b_colmajor):
    import torch

    if M * N * K > 2e8 and not (a_rowmajor and b_colmajor):
        pytest.skip("large shape checked once")
    g = torch.Generator(device="cuda").manual_seed(M * 7919 + N * 31 + K)
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    ref = (A @ B).cpu().numpy()
    Ab = A.contiguous() if a_rowmajor else A.T.contiguous()
    a_str = (K, 1) if a_rowmajor else (1, M)
    Bb = B.T.contiguous() if b_colmajor else B.contiguous()
    b_str = (1, K) if b_colmajor else (N, 1)
    for layout in ("col", "row"):
        out = _gemm(Ab, Bb, a_str, b_str, M, N, K, layout)
        err = np.abs(out - ref).max() / max(1.0, np.abs(ref).max())
        assert err < 1e-13 * max(1, K) ** 0.5, (layout, err)


def test_gemm_zero_k_and_batch_invariance():
    """Column j of A@B does not depend on how many columns are in the launch."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(5)
    M, K = 300, 601
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(K, 200, dtype=torch.float64, device="cuda", generator=g)
    Bc = B.T.contiguous()
    full = _gemm(A, Bc, (K, 1), (1, K), M, 200, K)
    for j in (0, 7, 199):
        one = _gemm(A, Bc[j:j + 1].contiguous(), (K, 1), (1, K), M, 1, K)
        assert np.array_equal(one[:, 0], full[:, j])
    z = _gemm(A, Bc, (K, 1), (1, K), M, 3, 0)
    assert np.array_equal(z, np.zeros((M, 3)))


def test_fast_and_generic_gemm_paths_bitwise_equal():
    """The 16-byte cp.async fast GEMM (large launches) and the generic kernel (small
    launches) share the k reduction order: a column computed alone (generic) equals the
    same column inside a fast-path batch, bit for bit, for both B layouts."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(11)
    M, K, N = 300, 600, 2048
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    Bt = torch.randn(N, K, dtype=torch.float64, device="cuda", generator=g)  # k-contiguous
    full = _gemm(A, Bt, (K, 1), (1, K), M, N, K)
    ref = (A @ Bt.T).cpu().numpy()
    assert np.abs(full - ref).max() / np.abs(ref).max() < 1e-13
    for j in (0, 777, N - 1):
        one = _gemm(A, Bt[j:j + 1].contiguous(), (K, 1), (1, K), M, 1, K)
        assert np.array_equal(one[:, 0], full[:, j])
    Bj = Bt.T.contiguous()  # j-contiguous (time-transform layout), row-major C
    full2 = _gemm(A, Bj, (K, 1), (N, 1), M, N, K, "row")
    assert np.array_equal(full2, full)
