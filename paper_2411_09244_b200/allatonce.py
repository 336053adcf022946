"""All-at-once waveform-relaxation fine solver on the GPU (drop-in for paradiff.allatonce).

Mirrors `/root/reference/pkg/src/paradiff/allatonce.py`: `TimeMatrixB` (:36-67),
`apply_S` / `apply_S_inverse` (:74-88), `ImplicitAllAtOnce` (:91-133), `build_rhs`
(:136-158), `WRResult` (:161-169), `WaveformRelaxation` (:172-298) and `wr_fine_solve`
(:301-313).
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


def _device():
    import torch

    from ._lib import require_cuda

    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    import ctypes as C

    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _apply(x, alpha: float, inverse: int) -> np.ndarray:
    import ctypes as C

    import torch

    from ._lib import check, load

    if not 0.0 < alpha < 1.0:
        raise ValueError(f"alpha must lie in (0, 1), got {alpha}")
    dev = _device()
    x = np.asarray(x)
    shape = x.shape
    J = shape[0]
    cols = int(np.prod(shape[1:], dtype=np.int64)) if x.ndim > 1 else 1
    xr = torch.as_tensor(np.ascontiguousarray(x.real, dtype=np.float64).reshape(J, cols),
                         device=dev)
    xi = (torch.as_tensor(np.ascontiguousarray(x.imag, dtype=np.float64).reshape(J, cols),
                          device=dev) if np.iscomplexobj(x) else None)
    yr = torch.empty_like(xr)
    yi = torch.empty_like(xr)
    p = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
    check(load().pe_apply_S(J, cols, float(alpha), inverse, p(xr), p(xi), p(yr), p(yi),
                            _stream()))
    return (yr.cpu().numpy() + 1j * yi.cpu().numpy()).reshape(shape)


def apply_S(x: np.ndarray, alpha: float) -> np.ndarray:
    """S x = Lambda (M ifft(x)) along axis 0 (allatonce.py:79-82), on the GPU (libpe
    direct DFT, pe_apply_S).  Returns complex128 like the reference."""
    return _apply(x, alpha, 0)


def apply_S_inverse(x: np.ndarray, alpha: float) -> np.ndarray:
    """S^{-1} x = fft(Lambda^{-1} x)/M along axis 0 (allatonce.py:85-88), on the GPU."""
    return _apply(x, alpha, 1)


def build_rhs(system: CoarseSystem, f1_rows, u_start, w_start, w_lag, w_rows_prev,
              u_final_prev, dt: float, alpha: float) -> np.ndarray:
    """Stacked right-hand side of the u all-at-once system (allatonce.py:136-158), on the
    GPU (pe_build_rhs): row s = f1^s - M12 (w_{s-1} - w_{s-2})/dt - A12 w_{s-1}, plus
    M11 (u_0 - alpha u_M^prev)/dt on the first row; w_0 = w_start, w_{-1} = w_lag."""
    import ctypes as C

    import torch

    from ._lib import check, load

    dev = _device()
    f1_rows = np.asarray(f1_rows, dtype=np.float64)
    J = f1_rows.shape[0]
    d1, d2 = system.d1, system.d2
    t = lambda a, shp: torch.as_tensor(  # noqa: E731
        np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(shp)), device=dev)
    args = [t(system.M11, (d1, d1)), t(system.M12, (d1, d2)), t(system.A12, (d1, d2)),
            t(f1_rows, (J, d1)), t(u_start, (d1,)), t(w_start, (d2,)), t(w_lag, (d2,)),
            t(w_rows_prev, (J, d2)), t(u_final_prev, (d1,))]
    out = torch.empty(J, d1, dtype=torch.float64, device=dev)
    check(load().pe_build_rhs(d1, d2, J, *[C.c_void_p(a.data_ptr()) for a in args],
                              float(dt), float(alpha), C.c_void_p(out.data_ptr()), _stream()))
    return out.cpu().numpy()


class ImplicitAllAtOnce:
    """Solver for (B kron M11 + I kron A11) U = F (allatonce.py:91-133), on the GPU.

    The reference inverts the M shifted matrices d_k M11 + A11 at construction and solves
    by FFT / einsum / inverse FFT.  libpe diagonalises the space pencil (A11, M11) once
    instead when it is symmetric-definite (every reference system), so each solve is two
    basis GEMMs around one scalar alpha-circulant recurrence per mode; otherwise it
    applies the half-spectrum shifted inverses between two time-transform GEMMs.
    `last_residual` is the reference's conditioning guard (the relative residual of the
    stacked system, :125-131), computed on the GPU for every solve.  `last_imag_residue`
    is 0.0: both formulations run in real arithmetic (the conjugate-symmetric half
    spectrum is folded into real operators), so no imaginary part is discarded.
    """

    def __init__(self, system: CoarseSystem, substeps: int, dt: float, alpha: float,
                 device: int | None = None):
        self.system = system
        self.time_matrix = TimeMatrixB(substeps, dt, alpha)
        self.last_residual = 0.0
        self.last_imag_residue = 0.0
        self.ctx = None
        if system.d1:
            # the load does not enter the u solve; the w block is carried along unused
            self.ctx = PeContext([system], [ConstantLoads.zero(system)], substeps, device)
            self.ctx.prepare_allatonce(dt, alpha, 1e-12, 1)

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        """rhs has one row per substep, shape (M, d1)."""
        return self.solve_all(np.asarray(rhs)[None])[0]

    def solve_all(self, rhs: np.ndarray) -> np.ndarray:
        """Batch of right-hand sides (nc, M, d1) -> (nc, M, d1)."""
        import ctypes as C

        from ._lib import check

        tm = self.time_matrix
        rhs = np.asarray(rhs, dtype=np.float64)
        if self.system.d1 == 0:
            return np.zeros((rhs.shape[0], tm.substeps, 0))
        if rhs.shape[1:] != (tm.substeps, self.system.d1):
            raise ValueError(f"rhs has shape {rhs.shape}, expected (nc, {tm.substeps}, "
                             f"{self.system.d1})")
        ctx = self.ctx
        nc = rhs.shape[0]
        with ctx.lock:
            R = ctx.to_dev(rhs[None])
            U = ctx.empty(1, nc, tm.substeps, self.system.d1)
            res = ctx.empty(nc)
            check(ctx.lib.pe_allatonce_usolve(ctx.ptr, C.c_void_p(R.data_ptr()),
                                              C.c_void_p(U.data_ptr()), nc,
                                              C.c_void_p(res.data_ptr()), ctx.stream()))
            self.last_residual = float(res[-1].item())
            U = U[0].cpu().numpy()
        self.last_imag_residue = 0.0
        log.debug("all-at-once residual %.3e", self.last_residual)
        return U


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
        self.constant_loads = bool(getattr(loads, "constant", False))
        self.system = system
        self.substeps = substeps
        self.dt_interval = dt_interval
        self.dt = dt_interval / substeps
        self.alpha = alpha
        self.loads = loads
        self.tol = tol
        self.max_iter = max_iter
        self.ctx = context or PeContext(
            [system], [loads if self.constant_loads else ConstantLoads.zero(system)], substeps,
            device)
        self.ctx.prepare_allatonce(self.dt, alpha, tol, max_iter)

    def solve(self, state: SplitState) -> WRResult:
        """Treats state as an interval start: lag values reset to (u, w)."""
        return self.solve_all([state])[0]

    def solve_all(self, states, trajectories: bool = True) -> list:
        ctx = self.ctx
        nc = len(states)
        F = None
        if not self.constant_loads:  # _load_rows: t0 + dt (1..J) (allatonce.py:212-218)
            rows = []
            for s in states:
                pairs = [self.loads.at(float(t))
                         for t in s.t + self.dt * np.arange(1, self.substeps + 1)]
                rows.append(np.array([np.concatenate([np.ravel(a), np.ravel(b)])
                                      for a, b in pairs]))
            F = np.array(rows)
        with ctx.lock:
            ctx.prepare_allatonce(self.dt, self.alpha, self.tol, self.max_iter)
            X = ctx.to_dev(np.array([s.stacked() for s in states])[None])
            if F is None:
                Y, sw, rs, rh = ctx.fine_allatonce(X)
            else:
                Y, sw, rs, rh = ctx.fine_allatonce_loads(X, ctx.to_dev(F[None]))
            Y = Y[0].cpu().numpy()
            sw = sw[0].cpu().numpy()
            rs = rs[0].cpu().numpy()
            rh = rh[0].cpu().numpy()
            if trajectories:
                U, W = ctx.wr_waveforms(nc)
                U = U[0].cpu().numpy()
                W = W[0].cpu().numpy()
            sres = ctx.wr_solver_residual(nc)[0].cpu().numpy()
        d1 = self.system.d1
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
            # solver_residual: the u-solve's relative residual (allatonce.py:125-131, :296);
            # imag_residue is 0.0: the solves run in real arithmetic (ImplicitAllAtOnce above)
            log.debug("all-at-once residual %.3e", sres[n])
            out.append(WRResult(SplitTrajectory(times, Un, Wn, final), res, it, conv, reason,
                                solver_residual=float(sres[n]), imag_residue=0.0))
        return out


def wr_fine_solve(system: CoarseSystem, state: SplitState, dt_interval: float, substeps: int,
                  alpha: float, loads: ConstantLoads, tol: float = 1e-12,
                  max_iter: int = 400) -> WRResult:
    """One-shot waveform-relaxation solve of a single coarse interval."""
    return WaveformRelaxation(system, substeps, dt_interval, alpha, loads, tol,
                              max_iter).solve(state)
