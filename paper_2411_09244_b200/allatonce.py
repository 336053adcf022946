"""All-at-once waveform-relaxation fine solver on the GPU (drop-in for paradiff.allatonce).

Mirrors `/root/reference/pkg/src/paradiff/allatonce.py`: `TimeMatrixB` (:36-67),
`WRResult` (:161-169), `WaveformRelaxation` (:172-298) and `wr_fine_solve` (:301-313).
The diagonalised u-solve (S^{-1} transform, the J shifted complex solves, Re(S .)),
the lagged right-hand side (build_rhs, :136-158), the w-sweep (:220-230) and the
per-interval stop logic (:245-271) all run inside libpe for a whole batch of
intervals at once; `solve_all` exposes the batch.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from .engine import PeContext, stop_reason_name
from .msbasis import CoarseSystem
from .stepping import ConstantLoads, SplitState, SplitTrajectory

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class TimeMatrixB:
    """Alpha-circulant backward-difference matrix over one interval's substeps."""

    substeps: int
    dt: float
    alpha: float

    def __post_init__(self):
        if self.substeps < 1 or self.dt <= 0:
            raise ValueError("need substeps >= 1 and dt > 0")
        if not 0.0 < self.alpha < 1.0:
            raise ValueError(f"alpha must lie in (0, 1), got {self.alpha}")

    def dense(self) -> np.ndarray:
        m = self.substeps
        b = np.eye(m)
        if m > 1:
            b[np.arange(1, m), np.arange(m - 1)] = -1.0
        b[0, m - 1] -= self.alpha
        return b / self.dt

    def eigenvalues(self) -> np.ndarray:
        """d_k = (1 - alpha^{1/M} e^{-2 pi i k/M}) / dt."""
        m = self.substeps
        return (1.0 - self.alpha ** (1.0 / m) * np.exp(-2j * np.pi * np.arange(m) / m)) / self.dt

    def scaling(self) -> np.ndarray:
        m = self.substeps
        return self.alpha ** (-np.arange(m) / m)


def build_time_matrix(substeps: int, dt: float, alpha: float) -> TimeMatrixB:
    return TimeMatrixB(substeps, dt, alpha)


@dataclass
class WRResult:
    trajectory: SplitTrajectory
    residuals: list
    iterations: int
    converged: bool
    stop_reason: str
    solver_residual: float = 0.0
    imag_residue: float = 0.0


class WaveformRelaxation:
    """Alternating all-at-once u-solve / w-sweep for coarse intervals, batched on GPU."""

    def __init__(self, system: CoarseSystem, substeps: int, dt_interval: float, alpha: float,
                 loads: ConstantLoads, tol: float = 1e-12, max_iter: int = 50,
                 device: int | None = None, context: PeContext | None = None):
        TimeMatrixB(substeps, dt_interval / substeps if dt_interval > 0 else -1.0, alpha)
        if not getattr(loads, "constant", False):
            raise NotImplementedError("libpe supports time-constant loads (ConstantLoads)")
        self.system = system
        self.substeps = substeps
        self.dt_interval = dt_interval
        self.dt = dt_interval / substeps
        self.alpha = alpha
        self.loads = loads
        self.tol = tol
        self.max_iter = max_iter
        self.ctx = context or PeContext([system], [loads], substeps, device)
        self.ctx.prepare_allatonce(self.dt, alpha, tol, max_iter)

    def solve(self, state: SplitState) -> WRResult:
        """Treats state as an interval start: lag values reset to (u, w)."""
        return self.solve_all([state])[0]

    def solve_all(self, states, trajectories: bool = True) -> list:
        ctx = self.ctx
        ctx.prepare_allatonce(self.dt, self.alpha, self.tol, self.max_iter)
        X = ctx.to_dev(np.array([s.stacked() for s in states])[None])
        Y, sw, rs, rh = ctx.fine_allatonce(X)
        nc = len(states)
        Y = Y[0].cpu().numpy()
        sw = sw[0].cpu().numpy()
        rs = rs[0].cpu().numpy()
        rh = rh[0].cpu().numpy()
        d1 = self.system.d1
        if trajectories:
            U, W = ctx.wr_waveforms(nc)
            U = U[0].cpu().numpy()
            W = W[0].cpu().numpy()
        out = []
        for n, s in enumerate(states):
            it = int(sw[n])
            reason = stop_reason_name(rs[n])
            res = rh[n, :it].tolist()
            conv = reason in ("tol", "floor")
            if not conv:
                log.warning("waveform relaxation %s after %d iterations (residual %.3e)",
                            "diverged" if reason == "diverged" else "not converged", it,
                            res[-1] if res else float("nan"))
            m = self.substeps
            times = s.t + self.dt * np.arange(m + 1)
            if trajectories:
                Un, Wn = U[n], W[n]
            else:
                Un = np.vstack([s.u, Y[n, :d1]])
                Wn = np.vstack([s.w, Y[n, d1:]])
            final = SplitState(u=Y[n, :d1].copy(), w=Y[n, d1:].copy(),
                               u_prev=Un[-2].copy(), w_prev=Wn[-2].copy(),
                               t=s.t + self.dt_interval)
            out.append(WRResult(SplitTrajectory(times, Un, Wn, final), res, it, conv, reason))
        return out


def wr_fine_solve(system: CoarseSystem, state: SplitState, dt_interval: float, substeps: int,
                  alpha: float, loads: ConstantLoads, tol: float = 1e-12,
                  max_iter: int = 400) -> WRResult:
    """One-shot waveform-relaxation solve of a single coarse interval."""
    return WaveformRelaxation(system, substeps, dt_interval, alpha, loads, tol,
                              max_iter).solve(state)
