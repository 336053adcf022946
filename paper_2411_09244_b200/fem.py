"""Fine-scale accuracy path on the GPU.

Mirrors the reference's accuracy reporting around a parareal run:
  * `reference_solve`  — fem.py:292-318 (backward Euler on the fine interior nodes);
  * `relative_error`   — experiment.py:320-325 (relative discrete L2 distance);
  * `error_series`     — experiment.py:348-354 (one relative error per parareal iterate,
    the coarse endpoint reconstructed through the split basis, msbasis.py:448-450);
  * `node_values_on_grid` — fem.py:321-330 (pure index bookkeeping for the writers).

The fine operators come from the reference's own offline assembly (out of scope here,
SURVEY §2): any object with scipy-sparse `M`, `A` (interior nodes) works, and the load is
either an ndarray or, when `ops` has a `load(source)` method, a source spec.  All
arithmetic runs in libpe (`finescale.cu`); there is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, require_cuda


SYM_MIN = 4096  # finescale.cu kSymMin: packed symmetric K^-1 tiles from this size on


def _csr(mat, n_rows=None):
    """(indptr int32, indices int32, data float64) of a scipy sparse / dense matrix."""
    import scipy.sparse as sp

    m = sp.csr_matrix(mat, dtype=float)
    m.sort_indices()
    if n_rows is not None and m.shape[0] != n_rows:
        raise ValueError(f"operator has {m.shape[0]} rows, expected {n_rows}")
    return (np.ascontiguousarray(m.indptr, dtype=np.int32),
            np.ascontiguousarray(m.indices, dtype=np.int32),
            np.ascontiguousarray(m.data, dtype=np.float64))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _stream_ptr(stream):
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _load_vector(ops, source, n):
    if isinstance(source, (np.ndarray, list, tuple)):
        b = np.ascontiguousarray(np.asarray(source, dtype=float))
    else:  # a source spec: the reference's own (offline) load assembly
        b = np.ascontiguousarray(np.asarray(ops.load(source), dtype=float))
    if b.shape != (n,):
        raise ValueError(f"load has shape {b.shape}, expected ({n},)")
    return b


MAX_DENSE_NODES = 65535      # dense (packed) K^-1 formulation limit (finescale.cu)
MAX_CHAIN_BANDWIDTH = 512    # block-tridiagonal chain solver limit (finechain.cu)


def _half_bandwidth(A) -> int:
    A = A.tocsr()
    rows = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
    return int(np.abs(A.indices - rows).max()) if A.nnz else 0


def check_reference_size(ops) -> None:
    """Up to 65535 interior nodes the GPU fine reference solve can keep a dense (packed)
    K^-1; larger grids need a banded operator (half-bandwidth <= 512: the chain solver of
    finechain.cu, which any row-ordered Q1 grid up to 511^2 nodes satisfies).  Raised before
    any work, so `run_single` fails before its parareal run rather than after it."""
    n = ops.M.shape[0]
    if n <= MAX_DENSE_NODES:
        return
    w = max(_half_bandwidth(ops.M), _half_bandwidth(ops.A))
    if w > MAX_CHAIN_BANDWIDTH:
        raise ValueError(f"fine reference solve: {n} interior nodes exceed the dense K^-1 limit "
                         f"({MAX_DENSE_NODES}) and the operator's half-bandwidth {w} exceeds the "
                         f"chain solver's ({MAX_CHAIN_BANDWIDTH})")


def reference_solve(ops, source, t_end: float, n_steps: int, u0=None,
                    keep_trajectory: bool = True, *, stream=None, timing: dict | None = None):
    """Backward Euler on the full fine space: (M/dt + A) u_{n+1} = M u_n/dt + b.

    Same contract as the reference (fem.py:292-318): returns (times, states), with every
    step when `keep_trajectory`, otherwise the initial and final vectors and
    times = [0, t_end].  `timing`, if given, receives the device time of the step loop.
    """
    n = ops.M.shape[0]
    check_reference_size(ops)
    lib = require_cuda()
    if n_steps <= 0 or not t_end > 0:
        raise ValueError("need n_steps > 0 and t_end > 0")
    mp, mi, mv = _csr(ops.M, n)
    ap, ai, av = _csr(ops.A, n)
    b = _load_vector(ops, source, n)
    u = None if u0 is None else np.ascontiguousarray(np.asarray(u0, dtype=float))
    if u is not None and u.shape != (n,):
        raise ValueError(f"u0 has shape {u.shape}, expected ({n},)")
    rows = n_steps + 1 if keep_trajectory else 2
    states = np.empty((rows, n))
    ms = C.c_float(0.0)
    check(lib.pe_fine_reference_solve(
        n, _ip(mp), _ip(mi), _dp(mv), _ip(ap), _ip(ai), _dp(av), _dp(b),
        None if u is None else _dp(u), float(t_end), int(n_steps), int(bool(keep_trajectory)),
        _dp(states), C.byref(ms), _stream_ptr(stream)))
    if timing is not None:
        timing["step_ms"] = float(ms.value)
        # algorithmic HBM bytes per step: R once + u, c, u' (n < 4096); from n = 4096 on the
        # lower triangle of the symmetric K^-1 once + M, u, b, v, u' (finescale.cu)
        blk = C.c_int(0)
        kind = lib.pe_fine_solver_kind(n, _ip(mp), _ip(mi), _ip(ap), _ip(ai), C.byref(blk))
        timing["solver"] = {0: "dense-gemv", 1: "packed-tiles", 2: "block-chain"}.get(kind, "?")
        if kind == 2:
            # chain solver: the nb dense block inverses twice (forward and backward sweep,
            # the last block once) + the sparse couplings and vectors (finechain.cu)
            bs = blk.value
            nblk = -(-n // bs)
            timing["block"] = bs
            timing["bytes_per_step"] = (8.0 * (2 * nblk - 1) * bs * bs + 12.0 * ops.M.nnz
                                        + 12.0 * (ops.M.nnz + ops.A.nnz) / 2 + 8.0 * 5 * n)
        else:
            timing["bytes_per_step"] = (8.0 * n * (n + 2) if n < SYM_MIN
                                        else 8.0 * (n * (n + 1) / 2 + 4 * n) + 12.0 * ops.M.nnz)
    times = np.linspace(0.0, t_end, n_steps + 1) if keep_trajectory else np.array([0.0, t_end])
    return times, states


def _error_norms(ops, psi1, psi2, ref, X, stream=None):
    import scipy.sparse as sp

    lib = require_cuda()
    n = ops.M.shape[0]
    P = sp.hstack([sp.csr_matrix(psi1), sp.csr_matrix(psi2)]).tocsr()
    if P.shape[0] != n:
        raise ValueError(f"basis has {P.shape[0]} rows, fine space has {n}")
    d = P.shape[1]
    pp, pi, pv = _csr(P)
    mp, mi, mv = _csr(ops.M, n)
    ref = np.ascontiguousarray(np.asarray(ref, dtype=float))
    X = np.ascontiguousarray(np.asarray(X, dtype=float).reshape(-1, d))
    K = X.shape[0]
    norms = np.empty(K + 1)
    check(lib.pe_relative_error_series(
        n, d, _ip(pp), _ip(pi), _dp(pv), _ip(mp), _ip(mi), _dp(mv), _dp(ref), K,
        _dp(X) if K else None, _dp(norms), _stream_ptr(stream)))
    return norms[:K], float(norms[K])


def _ratio(num, den, coarse_norm):
    # experiment.py:322-325: zero reference -> inf unless the coarse state is zero too
    if den == 0.0:
        return float(np.inf) if coarse_norm > 0 else 0.0
    return float(num / den)


def error_series(ops, space, ref_final, endpoints, *, stream=None) -> list[float]:
    """Relative errors of every coarse endpoint (K, d1 + d2) against `ref_final`.

    `space` is any object with `Psi1`, `Psi2` (the reference MultiscaleSpace,
    msbasis.py:421-450).  One launch chain for all K iterates.
    """
    X = np.asarray(endpoints, dtype=float)
    X = X.reshape(-1, space.Psi1.shape[1] + space.Psi2.shape[1])
    num, den = _error_norms(ops, space.Psi1, space.Psi2, ref_final, X, stream)
    # with ||ref||_M = 0, ||ref - y||_M is ||y||_M
    return [_ratio(v, den, v) for v in num]


def relative_error(ops, fine_final, coarse_final, *, stream=None) -> float:
    """Relative discrete L2 distance at the final time (experiment.py:320-325), where
    `coarse_final` is already a fine-space vector."""
    import scipy.sparse as sp

    n = ops.M.shape[0]
    eye = sp.identity(n, format="csr")
    num, den = _error_norms(ops, eye, sp.csr_matrix((n, 0)), fine_final,
                            np.asarray(coarse_final, dtype=float).reshape(1, n), stream)
    return _ratio(float(num[0]), den, float(num[0]))


def node_values_on_grid(grid, interior_values) -> np.ndarray:
    """Expand an interior-node vector to the (ny+1, nx+1) node lattice (fem.py:321-330)."""
    full = np.zeros(grid.n_nodes)
    full[grid.interior] = interior_values
    return full.reshape(grid.ny + 1, grid.nx + 1)
