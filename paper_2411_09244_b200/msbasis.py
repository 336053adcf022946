"""The offline -> online handoff type (msbasis.py:397-418 of the reference) and the
Galerkin projection that produces it (msbasis.py:545-572), on the GPU.

The multiscale basis itself (CEM/NLMC eigenproblems and saddle solves) is built by the
reference's own offline code; `project_coarse` / `project_load` take its
Psi1, Psi2 and the fine operators and run the projection in libpe (`project.cu`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class CoarseSystem:
    """Galerkin projections of the fine mass/stiffness onto the split basis."""

    M11: np.ndarray
    A11: np.ndarray
    M12: np.ndarray
    A12: np.ndarray
    M22: np.ndarray
    A22: np.ndarray

    @property
    def d1(self) -> int:
        return self.M11.shape[0]

    @property
    def d2(self) -> int:
        return self.M22.shape[0]

    def mass_block(self) -> np.ndarray:
        """Full coarse mass [[M11, M12], [M12^T, M22]]."""
        return np.block([[self.M11, self.M12], [self.M12.T, self.M22]])

    @classmethod
    def from_any(cls, s) -> "CoarseSystem":
        """Accept the reference's CoarseSystem (or any object with the six blocks)."""
        g = lambda k: np.ascontiguousarray(np.asarray(getattr(s, k), dtype=float))  # noqa: E731
        return cls(g("M11"), g("A11"), g("M12"), g("A12"), g("M22"), g("A22"))


def _proj(psi1, psi2, ops, b=None, stream=None):
    import ctypes as C

    import scipy.sparse as sp

    from ._lib import check, require_cuda
    from .fem import _csr, _dp, _ip, _stream_ptr

    lib = require_cuda()
    n = ops.M.shape[0]
    d1, d2 = psi1.shape[1], psi2.shape[1]
    if psi1.shape[0] != n or psi2.shape[0] != n:
        raise ValueError("basis rows do not match the fine space")
    pp, pi, pv = _csr(sp.hstack([sp.csr_matrix(psi1), sp.csr_matrix(psi2)]).tocsr())
    mp, mi, mv = _csr(ops.M, n)
    ap, ai, av = _csr(ops.A, n)
    d = d1 + d2
    Mc, Ac, asym = np.empty((d, d)), np.empty((d, d)), np.empty(2)
    bb = None if b is None else np.ascontiguousarray(np.asarray(b, dtype=float))
    if bb is not None and bb.shape != (n,):
        raise ValueError(f"load has shape {bb.shape}, expected ({n},)")
    f = np.empty(d)
    check(lib.pe_project_coarse(n, d1, d2, _ip(pp), _ip(pi), _dp(pv), _ip(mp), _ip(mi), _dp(mv),
                                _ip(ap), _ip(ai), _dp(av), None if bb is None else _dp(bb),
                                _dp(Mc), _dp(Ac), _dp(f) if bb is not None else None,
                                asym.ctypes.data_as(C.POINTER(C.c_double)), _stream_ptr(stream)))
    return Mc, Ac, f, asym, d1


def project_coarse(psi1, psi2, ops, *, stream=None) -> CoarseSystem:
    """Dense Galerkin blocks Psi_i^T X Psi_j for X in {M, A} (msbasis.py:545-567):
    diagonal blocks symmetrised, B12 = Psi1^T X Psi2.  One SpMM + one DMMA GEMM per X."""
    Mc, Ac, _, _, d1 = _proj(psi1, psi2, ops, stream=stream)
    c = lambda X: (np.ascontiguousarray(X[:d1, :d1]), np.ascontiguousarray(X[:d1, d1:]),  # noqa: E731
                   np.ascontiguousarray(X[d1:, d1:]))
    m11, m12, m22 = c(Mc)
    a11, a12, a22 = c(Ac)
    return CoarseSystem(M11=m11, A11=a11, M12=m12, A12=a12, M22=m22, A22=a22)


def project_load(space, b_fine, ops=None, *, stream=None):
    """Coarse load pair (Psi1^T b, Psi2^T b) (msbasis.py:570-572), same signature as the
    reference (`ops` is accepted for backward compatibility and ignored).  One warp per
    basis column over the CSC of [Psi1 Psi2] (`pe_project_load`); no operator products."""
    import scipy.sparse as sp

    from ._lib import check, require_cuda
    from .fem import _dp, _ip, _stream_ptr

    lib = require_cuda()
    psi = sp.hstack([sp.csc_matrix(space.Psi1), sp.csc_matrix(space.Psi2)]).tocsc()
    psi.sort_indices()
    n, d = psi.shape
    d1 = space.Psi1.shape[1]
    b = np.ascontiguousarray(np.asarray(b_fine, dtype=float))
    if b.shape != (n,):
        raise ValueError(f"load has shape {b.shape}, expected ({n},)")
    cp = np.ascontiguousarray(psi.indptr, dtype=np.int32)
    ci = np.ascontiguousarray(psi.indices, dtype=np.int32)
    cv = np.ascontiguousarray(psi.data, dtype=np.float64)
    f = np.empty(d)
    check(lib.pe_project_load(n, d, _ip(cp), _ip(ci), _dp(cv), _dp(b), _dp(f),
                              _stream_ptr(stream)))
    return f[:d1].copy(), f[d1:].copy()
