"""The offline -> online handoff type (msbasis.py:397-418 of the reference), the CEM-GMsFEM
basis build (msbasis.py:296-394) and the Galerkin projection that produces the handoff
(msbasis.py:545-572), on the GPU.

`build_cem_space` builds the split CEM basis of every coarse block in libpe (`cem.cu`:
batched auxiliary eigenproblems, per-block constrained energy minimisation);
`project_coarse` / `project_load` take Psi1, Psi2 and the fine operators and run the
projection in libpe (`project.cu`).  The NLMC basis (msbasis.py:181-252) stays out of
scope (no reference config uses it).
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


@dataclass
class CemSpace:
    """Split CEM space: Psi1 (dominant, n_dom per block) and Psi2 (complementary), CSR on
    the interior nodes, columns block-major as the reference's per-block stacking."""

    Psi1: object
    Psi2: object
    eigenvalues: np.ndarray  # (blocks, n_dom + n_comp) auxiliary eigenvalues
    constraint_residual: float
    seconds: float


def build_cem_space(nx: int, nb: int, layers: int, kappa, n_dom: int, n_comp: int,
                    weight: str = "kappa_h2", *, stream=None) -> CemSpace:
    """CEM basis of every block of a uniform nx x nx Q1 grid with nb x nb blocks, on the GPU.

    Same construction as the reference's `build_cem_basis(part, ops, field, b, n_dom +
    n_comp)` for b = 0 .. nb^2 - 1 (msbasis.py:331-394, with `aux_eigen_cem`, :296-328):
    the first n_dom columns of each block go to Psi1, the next n_comp to Psi2.
    `kappa`: cell values, row-major (cell (cx, cy) at cy * nx + cx).  Only the
    reference's default weight "kappa_h2" (kt = kappa nb^2) is supported.
    """
    import ctypes as C
    import time

    import scipy.sparse as sp

    from ._lib import check, require_cuda
    from .fem import _dp, _stream_ptr

    if weight != "kappa_h2":
        raise ValueError(f"unsupported aux weight {weight!r} (libpe builds 'kappa_h2')")
    if nx % nb:
        raise ValueError(f"{nb} blocks do not divide {nx} cells")
    lib = require_cuda()
    kap = np.ascontiguousarray(np.asarray(kappa, dtype=np.float64).ravel())
    if kap.size != nx * nx:
        raise ValueError(f"kappa has {kap.size} cells, expected {nx * nx}")
    ne = n_dom + n_comp
    nblk = nb * nb
    total = lib.pe_cem_basis_size(nx, nb, layers, ne)
    if total < 0:
        raise ValueError("invalid CEM geometry")
    vals = np.empty(total)
    offs = np.empty(nblk + 1, dtype=np.int64)
    eig = np.empty((nblk, ne))
    worst = C.c_double(0.0)
    t0 = time.perf_counter()
    check(lib.pe_cem_basis(nx, nb, layers, ne, _dp(kap), float(nb * nb), _dp(vals),
                           offs.ctypes.data_as(C.POINTER(C.c_longlong)), _dp(eig),
                           C.byref(worst), _stream_ptr(stream)))
    secs = time.perf_counter() - t0
    s = nx // nb
    n_int = (nx - 1) * (nx - 1)
    rows1, cols1, v1, rows2, cols2, v2 = [], [], [], [], [], []
    for b in range(nblk):
        bx, by = b % nb, b // nb
        x0 = max(bx - layers, 0) * s + 1
        x1 = min(bx + layers + 1, nb) * s - 1
        y0 = max(by - layers, 0) * s + 1
        y1 = min(by + layers + 1, nb) * s - 1
        xs, ys = np.meshgrid(np.arange(x0, x1 + 1), np.arange(y0, y1 + 1))
        rows = ((ys - 1) * (nx - 1) + (xs - 1)).ravel()
        nl = rows.size
        block = vals[offs[b]: offs[b + 1]].reshape(ne, nl)
        for k in range(ne):
            col = block[k]
            nz = np.nonzero(col)[0]
            if k < n_dom:
                rows1.append(rows[nz]); cols1.append(np.full(nz.size, b * n_dom + k))
                v1.append(col[nz])
            else:
                rows2.append(rows[nz]); cols2.append(np.full(nz.size, b * n_comp + k - n_dom))
                v2.append(col[nz])
    cat = lambda x: np.concatenate(x) if x else np.zeros(0)  # noqa: E731
    psi1 = sp.csr_matrix((cat(v1), (cat(rows1).astype(np.int64), cat(cols1).astype(np.int64))),
                         shape=(n_int, nblk * n_dom))
    psi2 = sp.csr_matrix((cat(v2), (cat(rows2).astype(np.int64), cat(cols2).astype(np.int64))),
                         shape=(n_int, nblk * n_comp))
    return CemSpace(psi1, psi2, eig, float(worst.value), secs)
