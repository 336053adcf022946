"""CPU oracle for the parareal hot path — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import this module, and only as the checker / the timed CPU
reference arm.  The product path (`paper_2411_09244_b200`) never imports it.

This is a NumPy/SciPy restatement of the reference's online algorithm
(`/root/reference/pkg/src/paradiff/`, cited below as `stepping.py:L`,
`allatonce.py:L`, `parareal.py:L`).  It uses the same dense LAPACK building blocks
the reference calls (Cholesky `cho_solve`, LU `lu_solve`, explicit complex
inverses + FFT + einsum), so that its timing is representative of the reference and
its rounding follows the reference's arithmetic order.

Pinning: `tests/test_oracle_pins.py` checks this restatement against golden vectors
produced by running the unmodified reference in the build container
(`oracle/make_golden.py`, fixtures in `tests/golden/`) and against the reference
tests' hand values (build_rhs -> [[14.0], [-3.3]], max_state_diff -> 3.0, closed forms).
"""

from __future__ import annotations

import logging
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
from scipy.linalg import cho_factor, cho_solve, lu_factor, lu_solve

log = logging.getLogger(__name__)

STOP_REASONS = ("tol", "diverged", "floor", "max_iter")


@dataclass(frozen=True)
class OSystem:
    """Dense reduced blocks + constant loads (msbasis.py:397-418, stepping.py:77-91)."""

    M11: np.ndarray
    A11: np.ndarray
    M12: np.ndarray
    A12: np.ndarray
    M22: np.ndarray
    A22: np.ndarray
    f1: np.ndarray
    f2: np.ndarray
    # time-dependent loads (stepping.py:125,164 `loads.at(t + dt)`; allatonce.py:212-218):
    # t -> (f1(t), f2(t)); None = the constant pair (f1, f2)
    loads_at: object = None

    def f_at(self, t):
        return (self.f1, self.f2) if self.loads_at is None else self.loads_at(t)

    @property
    def d1(self) -> int:
        return self.M11.shape[0]

    @property
    def d2(self) -> int:
        return self.M22.shape[0]

    @staticmethod
    def from_arrays(arrs) -> "OSystem":
        g = (lambda k: np.asarray(arrs[k], dtype=float))
        return OSystem(g("M11"), g("A11"), g("M12"), g("A12"), g("M22"), g("A22"),
                       g("f1"), g("f2"))


class OracleSplit:
    """Fine split step, coarse step G and the J-substep interval map.

    stepping.py:109-120 (factor caches), 122-147 (split_step), 149-176 (G),
    178-189 (fine_interval with lag reset), 191-207 (stability bound).
    """

    def __init__(self, s: OSystem):
        self.s = s
        self._kchol = {}
        self._glu = {}
        self._m22 = cho_factor(s.M22) if s.d2 else None

    def _k(self, dt):
        if dt not in self._kchol:
            self._kchol[dt] = cho_factor(self.s.M11 / dt + self.s.A11)
        return self._kchol[dt]

    def split_step(self, u, w, up, wp, dt, t=0.0):
        """One substep from time t (loads at t + dt, stepping.py:125)."""
        s = self.s
        f1, f2 = s.f_at(t + dt)
        if s.d1:
            r = s.M11 @ u / dt - s.M12 @ (w - wp) / dt - s.A12 @ w + f1
            un = cho_solve(self._k(dt), r)
        else:
            un = u.copy()
        if s.d2:
            r = (s.M22 @ w / dt - s.M12.T @ (u - up) / dt - s.A12.T @ un
                 - s.A22 @ w + f2)
            wn = cho_solve(self._m22, dt * r)
        else:
            wn = w.copy()
        return un, wn

    def fine_interval(self, u, w, dt_interval, substeps, t=0.0, return_t=False):
        """Returns (U, W) trajectories of shape (J+1, d1), (J+1, d2); lags reset.
        The substep time accumulates as the reference's SplitState.t (stepping.py:147)."""
        dt = dt_interval / substeps
        u = np.array(u, dtype=float)
        w = np.array(w, dtype=float)
        up, wp = u.copy(), w.copy()
        us, ws = [u.copy()], [w.copy()]
        for _ in range(substeps):
            un, wn = self.split_step(u, w, up, wp, dt, t)
            up, wp, u, w = u, w, un, wn
            t = t + dt
            us.append(u.copy())
            ws.append(w.copy())
        if return_t:
            return np.array(us), np.array(ws), t
        return np.array(us), np.array(ws)

    def _g(self, dt):
        if dt not in self._glu:
            s = self.s
            k = np.block([[s.M11 / dt + s.A11, s.M12 / dt],
                          [s.M12.T / dt + s.A12.T, s.M22 / dt]])
            self._glu[dt] = lu_factor(k)
        return self._glu[dt]

    def coarse_step(self, x, dt, t=0.0):
        """G from time t (loads at t + dt, stepping.py:164)."""
        s = self.s
        f1, f2 = s.f_at(t + dt)
        u, w = x[: s.d1], x[s.d1:]
        rhs = np.concatenate([
            f1 + s.M11 @ u / dt + s.M12 @ w / dt - s.A12 @ w,
            f2 + s.M12.T @ u / dt + s.M22 @ w / dt - s.A22 @ w,
        ])
        return lu_solve(self._g(dt), rhs)

    def stability_max_step(self, tol=1e-10, max_iter=10000):
        s = self.s
        if s.d2 == 0 or np.abs(s.A22).max() == 0.0:
            return np.inf
        v = np.ones(s.d2) / np.sqrt(s.d2)
        lam = 0.0
        for _ in range(max_iter):
            z = cho_solve(self._m22, s.A22 @ v)
            z /= np.linalg.norm(z)
            new = float((z @ (s.A22 @ z)) / (z @ (s.M22 @ z)))
            done = abs(new - lam) <= tol * abs(new)
            v, lam = z, new
            if done:
                break
        return 2.0 / lam


# ---------------------------------------------------------------- all-at-once (allatonce.py)

def time_eigenvalues(J, dt, alpha):
    """d_k = (1 - alpha^{1/J} e^{-2 pi i k/J}) / dt   (allatonce.py:58-62)."""
    om = np.exp(-2j * np.pi * np.arange(J) / J)
    return (1.0 - alpha ** (1.0 / J) * om) / dt


def time_matrix_dense(J, dt, alpha):
    """alpha-circulant backward difference B (allatonce.py:50-56)."""
    b = np.eye(J)
    if J > 1:
        b[np.arange(1, J), np.arange(J - 1)] = -1.0
    b[0, J - 1] -= alpha
    return b / dt


def _lam(alpha, J, ndim):
    return (alpha ** (-np.arange(J) / J)).reshape((J,) + (1,) * (ndim - 1))


def apply_S(x, alpha):
    """S x = Lambda J ifft(x) along axis 0 (allatonce.py:79-82)."""
    J = x.shape[0]
    return _lam(alpha, J, x.ndim) * (J * np.fft.ifft(x, axis=0))


def apply_S_inverse(x, alpha):
    """S^{-1} x = fft(Lambda^{-1} x)/J along axis 0 (allatonce.py:85-88)."""
    J = x.shape[0]
    return np.fft.fft(x / _lam(alpha, J, x.ndim), axis=0) / J


def build_rhs(s: OSystem, f1_rows, u_start, w_start, w_lag, w_rows_prev, u_final_prev, dt, alpha):
    """Lagged-w right-hand side of the u all-at-once system (allatonce.py:136-158)."""
    wh = np.vstack([w_lag, w_start, w_rows_prev[:-1]])
    dw = (wh[1:] - wh[:-1]) / dt
    rhs = f1_rows - dw @ s.M12.T - wh[1:] @ s.A12.T
    rhs[0] += s.M11 @ (u_start - alpha * u_final_prev) / dt
    return rhs


class OracleWR:
    """Waveform relaxation over one coarse interval (allatonce.py:172-298)."""

    def __init__(self, s: OSystem, substeps, dt_interval, alpha, tol=1e-12, max_iter=50):
        if substeps < 1 or dt_interval <= 0:
            raise ValueError("need substeps >= 1 and dt > 0")
        if not 0.0 < alpha < 1.0:
            raise ValueError(f"alpha must lie in (0, 1), got {alpha}")
        self.s = s
        self.J = substeps
        self.dt_interval = dt_interval
        self.dt = dt_interval / substeps
        self.alpha = alpha
        self.tol = tol
        self.max_iter = max_iter
        d = time_eigenvalues(substeps, self.dt, alpha)
        if s.d1:
            shifted = d[:, None, None] * s.M11[None] + s.A11[None].astype(complex)
            self.inv_shifted = np.linalg.inv(shifted)
        else:
            self.inv_shifted = np.zeros((substeps, 0, 0), dtype=complex)
        if s.d2:
            self.m22_inv = cho_solve(cho_factor(s.M22), np.eye(s.d2))
            self.e_mat = np.eye(s.d2) - self.dt * self.m22_inv @ s.A22
        else:
            self.m22_inv = np.zeros((0, 0))
            self.e_mat = np.zeros((0, 0))

    def u_solve(self, rhs):
        if self.s.d1 == 0:
            return np.zeros((self.J, 0))
        p = apply_S_inverse(rhs, self.alpha)
        q = np.einsum("kij,kj->ki", self.inv_shifted, p)
        return apply_S(q, self.alpha).real

    def w_sweep(self, u_rows, u0, w0, f2_rows):
        s = self.s
        uh = np.vstack([u0, u0, u_rows[:-1]])
        du = (uh[1:] - uh[:-1]) / self.dt
        g = self.dt * (f2_rows - du @ s.M12 - u_rows @ s.A12) @ self.m22_inv
        out = np.empty((self.J, s.d2))
        w = w0
        for i in range(self.J):
            w = self.e_mat @ w + g[i]
            out[i] = w
        return out

    def solve(self, u0, w0, t0=0.0):
        s, J = self.s, self.J
        if s.loads_at is None:
            f1_rows = np.tile(s.f1, (J, 1))
            f2_rows = np.tile(s.f2, (J, 1))
        else:  # _load_rows (allatonce.py:212-218)
            pairs = [s.loads_at(t) for t in t0 + self.dt * np.arange(1, J + 1)]
            f1_rows = np.array([q[0] for q in pairs])
            f2_rows = np.array([q[1] for q in pairs])
        U = np.tile(u0, (J, 1))
        W = np.tile(w0, (J, 1))
        ufp = np.array(u0, dtype=float).copy()
        res = []
        converged, reason, stall, prev = False, "max_iter", 0, np.inf
        it = 0
        for _ in range(self.max_iter):
            it += 1
            rhs = build_rhs(s, f1_rows, u0, w0, w0, W, ufp, self.dt, self.alpha)
            Un = self.u_solve(rhs)
            Wn = self.w_sweep(Un, u0, w0, f2_rows)
            r = 0.0
            if s.d1:
                r += float(np.linalg.norm(Un - U, axis=1).max())
            if s.d2:
                r += float(np.linalg.norm(Wn - W, axis=1).max())
            res.append(r)
            U, W = Un, Wn
            ufp = U[-1] if s.d1 else np.asarray(u0, dtype=float)
            if r <= self.tol:
                converged, reason = True, "tol"
                break
            if not np.isfinite(r) or r > 1e8 * max(1.0, res[0]):
                reason = "diverged"
                break
            stall = stall + 1 if r >= prev else 0
            if stall >= 2 and r <= 1e3 * self.tol:
                converged, reason = True, "floor"
                break
            prev = r
        Uf = np.vstack([u0, U])
        Wf = np.vstack([w0, W])
        return dict(U=Uf, W=Wf, residuals=res, iterations=it, converged=converged,
                    stop_reason=reason)


# ---------------------------------------------------------------- parareal (parareal.py)

def max_state_diff(prev, new):
    """max over n = 1..N of ||new_n - prev_n||_2 (parareal.py:140-142)."""
    return float(np.linalg.norm(new[1:] - prev[1:], axis=1).max())


def rel_state_diff(prev, new):
    """Relative increment max_n ||dx_n|| / max_n ||x_n^k||, n = 1..N."""
    num = np.linalg.norm(new[1:] - prev[1:], axis=1).max()
    den = np.linalg.norm(new[1:], axis=1).max()
    return float(num / den) if den > 0 else float(num)


def resolved_fine_tol(epsilon, fine_tol=None):
    """parareal.py:42-50."""
    if fine_tol is not None:
        return fine_tol
    return min(1e-12, max(0.01 * epsilon, 1e-14))


def run_parareal(s: OSystem, x0, t_end, n_intervals, substeps, *, kind="sequential",
                 alpha=0.5, epsilon=1e-14, k_max=100, stop="absolute", fine_tol=None,
                 fine_max_iter=400, workers=1, t0=0.0):
    """Algorithm 1 (parareal.py:160-236) with the stop rule selectable.

    stop="absolute" is the reference check_stop (parareal.py:145-147);
    stop="relative" is the harness rule of SURVEY §0 F5.
    Returns a dict with history, max_diffs, iterations, converged, fine_info,
    fine_seconds, coarse_seconds.
    """
    if t_end <= 0 or n_intervals < 1 or substeps < 1:
        raise ValueError("need t_end > 0, n_intervals >= 1, substeps >= 1")
    d1 = s.d1
    dt = t_end / n_intervals
    sp_ = OracleSplit(s)
    if kind == "sequential":
        def fine(xt):
            x, t = xt
            U, W, t1 = sp_.fine_interval(x[:d1], x[d1:], dt, substeps, t, return_t=True)
            return np.concatenate([U[-1], W[-1]]), {"converged": True}, t1
    elif kind == "all-at-once":
        wr = OracleWR(s, substeps, dt, alpha, tol=resolved_fine_tol(epsilon, fine_tol),
                      max_iter=fine_max_iter)

        def fine(xt):
            x, t = xt
            r = wr.solve(x[:d1], x[d1:], t)
            return np.concatenate([r["U"][-1], r["W"][-1]]), {
                "converged": r["converged"], "iterations": r["iterations"],
                "residuals": r["residuals"], "stop_reason": r["stop_reason"]}, t + dt
    else:
        raise ValueError(f"unknown fine propagator kind {kind!r}")
    check = rel_state_diff if stop == "relative" else max_state_diff

    x0 = np.asarray(x0, dtype=float)
    states = [x0.copy()]
    times = [float(t0)]  # SplitState.t of each state (parareal.py:150-157, 210)
    for _ in range(n_intervals):
        states.append(sp_.coarse_step(states[-1], dt, times[-1]))
        times.append(times[-1] + dt)
    gold = [sp_.coarse_step(x, dt, t) for x, t in zip(states[:-1], times[:-1])]
    history = [np.array(states)]
    max_diffs, fine_info, fsec, csec = [], [], [], []
    converged, iterations = False, 0
    pool = ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
    try:
        for _ in range(k_max):
            iterations += 1
            tic = time.perf_counter()
            args = [(states[n], times[n]) for n in range(n_intervals)]
            if pool is None:
                fr = [fine(a) for a in args]
            else:
                fr = list(pool.map(fine, args))
            fsec.append(time.perf_counter() - tic)
            fine_info.append([info for _, info, _ in fr])
            tic = time.perf_counter()
            new = [x0.copy()]
            gnew = []
            for n in range(n_intervals):
                g = sp_.coarse_step(new[n], dt, times[n])
                gnew.append(g)
                new.append(fr[n][0] + (g - gold[n]))
            times = [float(t0)] + [fr[n][2] for n in range(n_intervals)]
            csec.append(time.perf_counter() - tic)
            history.append(np.array(new))
            diff = check(history[-2], history[-1])
            max_diffs.append(diff)
            states, gold = new, gnew
            if diff < epsilon:
                converged = True
                break
    finally:
        if pool is not None:
            pool.shutdown()
    return dict(history=history, max_diffs=max_diffs, iterations=iterations,
                converged=converged, fine_info=fine_info, fine_seconds=fsec,
                coarse_seconds=csec)


# ------------------------------------------------------------------ fine-scale accuracy
# restated from fem.py:292-318, fem.py:272-274 and experiment.py:320-325.


def fine_reference_solve(M, A, b, t_end, n_steps, u0=None, keep_trajectory=True):
    """Backward Euler (M/dt + A) u_{n+1} = M u_n / dt + b with a sparse LU, as
    fem.py:292-318 (`splu` of the CSC matrix, one `lu.solve` per step)."""
    from scipy.sparse.linalg import splu

    n = M.shape[0]
    dt = t_end / n_steps
    u = np.zeros(n) if u0 is None else np.asarray(u0, dtype=float).copy()
    lu = splu((M / dt + A).tocsc())
    states = [u.copy()]
    for _ in range(n_steps):
        u = lu.solve(M @ u / dt + b)
        if keep_trajectory:
            states.append(u.copy())
    if not keep_trajectory:
        states.append(u.copy())
    return np.array(states)


def m_norm(M, v):
    """sqrt(v^T M v), fem.py:272-274."""
    return float(np.sqrt(v @ (M @ v)))


def relative_error(M, fine_final, coarse_final):
    """experiment.py:320-325."""
    denom = m_norm(M, fine_final)
    if denom == 0.0:
        return float(np.inf) if m_norm(M, coarse_final) > 0 else 0.0
    return m_norm(M, fine_final - coarse_final) / denom


def error_series(M, psi1, psi2, ref_final, history):
    """experiment.py:348-354: one relative error per iterate, endpoint reconstructed
    through Psi1 u + Psi2 w (msbasis.py:448-450)."""
    d1 = psi1.shape[1]
    out = []
    for rows in history:
        x = np.asarray(rows)[-1]
        out.append(relative_error(M, ref_final, psi1 @ x[:d1] + psi2 @ x[d1:]))
    return out
