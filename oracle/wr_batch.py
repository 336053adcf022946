"""Batched restatement of the reference waveform relaxation for large systems (TEST
INFRASTRUCTURE; config-3 parity).

`WaveformRelaxation.solve` (allatonce.py:232-298) handles one interval and applies its
J shifted inverses with a single-threaded `einsum` (allatonce.py:118): at config 3
(d1 = 4096, J = 100) that is ~5 s per sweep per interval, and a full solve takes hundreds
of sweeps.  This module runs the same per-interval algorithm for B intervals at once:

* the same seeds, build_rhs rows, S^{-1} / S transforms (numpy FFT along the time axis),
  explicit shifted inverses, w recursion, residual (sum of the two max row norms) and
  stop logic (tol / diverged / floor / max_iter) as allatonce.py:239-289, per interval;
* the shifted apply q_k = inv_k p_k becomes one (d1 x d1)(d1 x B) product per mode, so
  the 26.8 GB of inverses stream once per sweep for all B intervals (multithreaded BLAS);
* an interval that has stopped keeps the waveforms of its stopping sweep (its columns are
  still computed, then discarded), exactly like a sequence of independent solves.

The inverses are formed one mode at a time into a preallocated array (the reference's
stacked `np.linalg.inv` would transiently need twice the 26.8 GB).  Matmul instead of
einsum only reorders the floating-point sums of the shifted apply (~1e-16 relative).
"""

from __future__ import annotations

import time

import numpy as np
from scipy.linalg import cho_factor, cho_solve

from oracle.pe_oracle import apply_S, apply_S_inverse, time_eigenvalues


def _apply(A, X):
    """A @ X[s] for every s of X (S, n, B) as ONE GEMM (A is read once, not S times)."""
    S, n, B = X.shape
    Y = A @ np.ascontiguousarray(X.transpose(1, 0, 2)).reshape(n, S * B)
    return np.ascontiguousarray(Y.reshape(A.shape[0], S, B).transpose(1, 0, 2))


class BatchWR:
    def __init__(self, s, J, dt_interval, alpha, tol=1e-12, max_iter=400, verbose=False):
        self.s, self.J, self.dt = s, J, dt_interval / J
        self.alpha, self.tol, self.max_iter = alpha, tol, max_iter
        t0 = time.time()
        d = time_eigenvalues(J, self.dt, alpha)
        self.inv = np.empty((J, s.d1, s.d1), dtype=complex)
        a11 = s.A11.astype(complex)
        for k in range(J):
            self.inv[k] = np.linalg.inv(d[k] * s.M11 + a11)
            if verbose and k % 10 == 0:
                print(f"  inverse {k}/{J} ({time.time() - t0:.0f} s)", flush=True)
        self.m22_inv = cho_solve(cho_factor(s.M22), np.eye(s.d2))
        self.e_mat = np.eye(s.d2) - self.dt * self.m22_inv @ s.A22

    def solve(self, X0, verbose=False):
        """X0: (B, d1 + d2) interval start states.  Returns per-interval dicts like
        `OracleWR.solve` (U, W with the start row, residuals, iterations, stop_reason)."""
        s, J, dt, al = self.s, self.J, self.dt, self.alpha
        d1 = s.d1
        X0 = np.asarray(X0, dtype=float)
        B = X0.shape[0]
        u0 = X0[:, :d1].T  # (d1, B)
        w0 = X0[:, d1:].T
        U = np.repeat(u0[None], J, axis=0)  # (J, d1, B)
        W = np.repeat(w0[None], J, axis=0)
        ufp = u0.copy()
        f1 = s.f1[:, None]
        f2 = s.f2[:, None]
        res = [[] for _ in range(B)]
        stall = np.zeros(B, dtype=int)
        prev = np.full(B, np.inf)
        active = np.ones(B, dtype=bool)
        reason = ["max_iter"] * B
        iters = np.zeros(B, dtype=int)
        outU = np.empty((B, J + 1, d1))
        outW = np.empty((B, J + 1, s.d2))
        t0 = time.time()
        for sweep in range(1, self.max_iter + 1):
            # build_rhs (allatonce.py:154-157): w_hist = [w_lag, w_start, W[:-1]]
            wh = np.concatenate([w0[None], w0[None], W[:-1]], axis=0)
            dw = (wh[1:] - wh[:-1]) / dt
            rhs = f1[None] - _apply(s.M12, dw) - _apply(s.A12, wh[1:])
            rhs[0] += s.M11 @ (u0 - al * ufp) / dt
            # u solve (allatonce.py:117-119): p = S^-1 rhs, q_k = inv_k p_k, u = Re(S q)
            p = apply_S_inverse(rhs, al)
            q = np.empty_like(p)
            for k in range(J):
                q[k] = self.inv[k] @ p[k]
            Un = apply_S(q, al).real
            # w sweep (allatonce.py:222-229)
            uh = np.concatenate([u0[None], u0[None], Un[:-1]], axis=0)
            du = (uh[1:] - uh[:-1]) / dt
            g = dt * _apply(self.m22_inv.T, f2[None] - _apply(s.M12.T, du) - _apply(s.A12.T, Un))
            Wn = np.empty_like(W)
            w = w0
            for i in range(J):
                w = self.e_mat @ w + g[i]
                Wn[i] = w
            r = (np.linalg.norm(Un - U, axis=1).max(axis=0)
                 + np.linalg.norm(Wn - W, axis=1).max(axis=0))
            U, W = Un, Wn
            ufp = U[-1]
            for b in np.nonzero(active)[0]:
                rb = float(r[b])
                res[b].append(rb)
                iters[b] = sweep
                stop = None
                if rb <= self.tol:
                    stop = "tol"
                elif not np.isfinite(rb) or rb > 1e8 * max(1.0, res[b][0]):
                    stop = "diverged"
                else:
                    stall[b] = stall[b] + 1 if rb >= prev[b] else 0
                    if stall[b] >= 2 and rb <= 1e3 * self.tol:
                        stop = "floor"
                    prev[b] = rb
                if stop is not None or sweep == self.max_iter:
                    reason[b] = stop or "max_iter"
                    active[b] = False
                    outU[b, 0], outW[b, 0] = u0[:, b], w0[:, b]
                    outU[b, 1:], outW[b, 1:] = U[:, :, b], W[:, :, b]
            if verbose and (sweep % 25 == 0 or not active.any()):
                print(f"  sweep {sweep}: active {active.sum()}/{B}, resid "
                      + " ".join(f"{float(v):.2e}" for v in r) + f" ({time.time() - t0:.0f} s)",
                      flush=True)
            if not active.any():
                break
        return [dict(U=outU[b], W=outW[b], residuals=res[b], iterations=int(iters[b]),
                     converged=reason[b] in ("tol", "floor"), stop_reason=reason[b])
                for b in range(B)]
