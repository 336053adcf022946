"""Partially explicit splitting propagators on the GPU (drop-in for paradiff.stepping).

Same names, argument meaning and error behaviour as the reference
(`/root/reference/pkg/src/paradiff/stepping.py`): `SplitState` (:32-50), `TimeGrid`
(:53-74), `ConstantLoads` (:77-91), `SplitTrajectory` (:94-99) and `SplitPropagators`
(:102-213).  Every arithmetic step runs in libpe (sm_100a); the host side only moves
states in and out.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np
import torch

from .engine import PeContext
from .msbasis import CoarseSystem

log = logging.getLogger(__name__)


@dataclass
class SplitState:
    """Coarse coefficients at one time level plus the lagged previous level."""

    u: np.ndarray
    w: np.ndarray
    u_prev: np.ndarray
    w_prev: np.ndarray
    t: float

    @classmethod
    def fresh(cls, u, w, t: float = 0.0) -> "SplitState":
        """State with lag values equal to the current ones (interval start)."""
        u = np.asarray(u, dtype=float)
        w = np.asarray(w, dtype=float)
        return cls(u.copy(), w.copy(), u.copy(), w.copy(), t)

    def stacked(self) -> np.ndarray:
        return np.concatenate([self.u, self.w])


@dataclass(frozen=True)
class TimeGrid:
    """T split into n_intervals coarse steps of `substeps` fine steps each."""

    t_end: float
    n_intervals: int
    substeps: int

    def __post_init__(self):
        if self.t_end <= 0 or self.n_intervals < 1 or self.substeps < 1:
            raise ValueError("need t_end > 0, n_intervals >= 1, substeps >= 1")

    @property
    def dt(self) -> float:
        return self.t_end / self.n_intervals

    @property
    def dt_sub(self) -> float:
        return self.dt / self.substeps

    def interval_starts(self) -> np.ndarray:
        return np.arange(self.n_intervals) * self.dt


class ConstantLoads:
    """Time-constant coarse load pair; the provider interface is at(t)."""

    constant = True

    def __init__(self, f1, f2):
        self.f1 = np.asarray(f1, dtype=float)
        self.f2 = np.asarray(f2, dtype=float)

    @classmethod
    def zero(cls, system: CoarseSystem) -> "ConstantLoads":
        return cls(np.zeros(system.d1), np.zeros(system.d2))

    def at(self, t: float):
        return self.f1, self.f2


@dataclass
class SplitTrajectory:
    times: np.ndarray
    U: np.ndarray  # (n_steps + 1, d1)
    W: np.ndarray  # (n_steps + 1, d2)
    final: SplitState


def _stack_states(states, lag: bool = False) -> np.ndarray:
    if lag:
        return np.array([np.concatenate([s.u_prev, s.w_prev]) for s in states])
    return np.array([s.stacked() for s in states])


class SplitPropagators:
    """Fine substep, coarse step G and interval map for one reduced system, on the GPU.

    The reference caches a Cholesky / LU per step size (stepping.py:109-120,
    149-159); here the corresponding composite operators live in HBM inside a libpe
    context, built once per step size.
    """

    def __init__(self, system: CoarseSystem, loads, device: int | None = None):
        self.system = system
        self.loads = loads
        self.device = device
        self._ctx: dict[int, PeContext] = {}

    @property
    def constant_loads(self) -> bool:
        return bool(getattr(self.loads, "constant", False))

    def context(self, substeps: int) -> PeContext:
        if substeps not in self._ctx:
            base = self.loads if self.constant_loads else ConstantLoads.zero(self.system)
            self._ctx[substeps] = PeContext([self.system], [base], substeps, self.device)
        return self._ctx[substeps]

    def load_rows(self, times) -> np.ndarray:
        """[f1(t); f2(t)] for every t (the reference's `loads.at`), shape (len(times), d)."""
        rows = []
        for t in times:
            f1, f2 = self.loads.at(float(t))
            rows.append(np.concatenate([np.asarray(f1, dtype=float).ravel(),
                                        np.asarray(f2, dtype=float).ravel()]))
        return np.array(rows).reshape(len(rows), self.system.d1 + self.system.d2)

    def fine_load_series(self, starts, dt: float, substeps: int) -> np.ndarray:
        """Loads of a sequential fine interval from each start time: substep s at the
        reference's accumulated SplitState.t + dt (stepping.py:125,147), (nc, J, d)."""
        out = []
        for t in starts:
            times = []
            tt = float(t)
            for _ in range(substeps):
                times.append(tt + dt)
                tt = tt + dt
            out.append(self.load_rows(times))
        return np.array(out)

    # ------------------------------------------------------------------ reference API
    def split_step(self, state: SplitState, dt: float) -> SplitState:
        """One substep of the partially explicit scheme (stepping.py:122-147)."""
        ctx = self.context(1)
        with ctx.lock:
            ctx.prepare_sequential(dt)
            x = ctx.to_dev(state.stacked()[None, None])
            xp = ctx.to_dev(np.concatenate([state.u_prev, state.w_prev])[None, None])
            if self.constant_loads:
                y = ctx.split_step(x, xp)[0, 0].cpu().numpy()
            else:  # loads at state.t + dt (stepping.py:125)
                F = ctx.to_dev(self.load_rows([state.t + dt])[None, None])
                y = ctx.split_step_loads(x, xp, F)[0, 0].cpu().numpy()
        d1 = self.system.d1
        return SplitState(y[:d1].copy(), y[d1:].copy(), state.u.copy(), state.w.copy(),
                          state.t + dt)

    def coarse_step(self, state: SplitState, dt: float) -> SplitState:
        """Coupled one-step solve G (stepping.py:161-176)."""
        return self.coarse_step_all([state], dt)[0]

    def coarse_step_all(self, states, dt: float):
        ctx = self.context(1)
        with ctx.lock:
            ctx.prepare_coarse(dt)
            X = ctx.to_dev(_stack_states(states)[None])
            if self.constant_loads:
                y = ctx.coarse_apply(X)[0].cpu().numpy()
            else:  # loads at state.t + dt (stepping.py:164)
                Fc = ctx.to_dev(self.load_rows([s.t + dt for s in states])[None])
                y = ctx.coarse_apply_loads(X, Fc)[0].cpu().numpy()
        d1 = self.system.d1
        return [SplitState(r[:d1].copy(), r[d1:].copy(), s.u.copy(), s.w.copy(), s.t + dt)
                for r, s in zip(y, states)]

    def fine_interval(self, state: SplitState, dt_interval: float,
                      substeps: int) -> SplitTrajectory:
        """`substeps` split steps with lags reset (stepping.py:178-189), full trajectory."""
        ctx = self.context(1)
        dt = dt_interval / substeps
        d1 = self.system.d1
        Fs = None if self.constant_loads else self.fine_load_series([state.t], dt, substeps)[0]
        with ctx.lock:
            ctx.prepare_sequential(dt)
            x = ctx.to_dev(state.stacked()[None, None])
            xp = x.clone()
            rows = [x[0, 0]]
            for s in range(substeps):
                if Fs is None:
                    y = ctx.split_step(x, xp)
                else:
                    y = ctx.split_step_loads(x, xp, ctx.to_dev(Fs[s][None, None]))
                xp, x = x, y
                rows.append(y[0, 0])
            traj = torch.stack(rows).cpu().numpy()
        t_end = state.t
        for _ in range(substeps):  # SplitState.t accumulates per substep (stepping.py:147)
            t_end = t_end + dt
        cur = SplitState(traj[-1, :d1].copy(), traj[-1, d1:].copy(), traj[-2, :d1].copy(),
                         traj[-2, d1:].copy(), t_end)
        times = state.t + dt * np.arange(substeps + 1)
        return SplitTrajectory(times, traj[:, :d1].copy(), traj[:, d1:].copy(), cur)

    def stability_max_step(self, tol: float = 1e-10, max_iter: int = 10000) -> float:
        """2 / lambda_max(M22^{-1} A22) by power iteration (stepping.py:191-207), in libpe
        (pe_stability_max_step: the reference's start vector, Rayleigh quotient and stop)."""
        import ctypes as C

        from ._lib import check

        s = self.system
        if s.d2 == 0:
            return np.inf
        ctx = self.context(1)
        out, its = C.c_double(0.0), C.c_int(0)
        with ctx.lock:
            check(ctx.lib.pe_stability_max_step(ctx.ptr, 0, float(tol), int(max_iter),
                                                C.byref(out), C.byref(its), ctx.stream()))
        if its.value < 0:
            log.warning("stability power iteration hit %d iterations, last rayleigh %.6e",
                        max_iter, 2.0 / out.value)
        return float(out.value)

    def check_substep(self, dt: float) -> None:
        bound = self.stability_max_step()
        if dt > bound:
            log.warning("substep %.3e exceeds stability bound %.3e", dt, bound)


def project_initial(u0_fine, space, ops, *, stream=None) -> SplitState:
    """Mass-orthogonal projection of a fine initial value onto each subspace
    (stepping.py:216-226): M11 u = Psi1^T M u0, M22 w = Psi2^T M u0, lags equal to the
    projections.  On the GPU (pe_project_initial): CSR SpMV, one warp per basis column,
    LU solves of the two coarse mass blocks."""
    import ctypes as C

    import scipy.sparse as sp

    from ._lib import check, require_cuda
    from .fem import _csr, _dp, _ip, _stream_ptr

    lib = require_cuda()
    s = space.system
    d1, d2 = s.M11.shape[0], s.M22.shape[0]
    n = ops.M.shape[0]
    u0 = np.ascontiguousarray(np.asarray(u0_fine, dtype=float))
    if u0.shape != (n,):
        raise ValueError(f"u0 has shape {u0.shape}, expected ({n},)")
    mp, mi, mv = _csr(ops.M, n)
    psi = sp.hstack([sp.csc_matrix(space.Psi1), sp.csc_matrix(space.Psi2)]).tocsc()
    psi.sort_indices()
    cp = np.ascontiguousarray(psi.indptr, dtype=np.int32)
    ci = np.ascontiguousarray(psi.indices, dtype=np.int32)
    cv = np.ascontiguousarray(psi.data, dtype=np.float64)
    m11 = np.ascontiguousarray(s.M11, dtype=float)
    m22 = np.ascontiguousarray(s.M22, dtype=float)
    u, w = np.zeros(d1), np.zeros(d2)
    check(lib.pe_project_initial(n, d1, d2, _ip(mp), _ip(mi), _dp(mv), _ip(cp), _ip(ci),
                                 _dp(cv), _dp(m11) if d1 else None, _dp(m22) if d2 else None,
                                 _dp(u0), _dp(u) if d1 else None, _dp(w) if d2 else None,
                                 _stream_ptr(stream)))
    return SplitState.fresh(u, w, 0.0)


def split_energy(system: CoarseSystem, state: SplitState) -> float:
    """Squared fine-space L2 norm of the represented function (stepping.py:229-232)."""
    x = state.stacked()
    return float(x @ (system.mass_block() @ x))
