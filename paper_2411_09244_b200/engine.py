"""Device-side engine: one libpe context per (members, substeps J) holding the reduced
operators in HBM, with torch tensors as the device buffers passed across the C ABI.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib
from ._lib import PE_KIND, PE_RULE, PE_STOP, check

_D = C.POINTER(C.c_double)


def _host(a) -> tuple:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return arr, (arr.ctypes.data_as(_D) if arr.size else None)


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


class PeContext:
    """Owns a `pe_ctx` for E members of one reduced size and J fine substeps."""

    def __init__(self, systems, loads, J: int, device: int | None = None):
        self.lib = _lib.require_cuda()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self.E = len(systems)
        s0 = systems[0]
        self.d1, self.d2 = int(s0.d1), int(s0.d2)
        self.d = self.d1 + self.d2
        self.J = int(J)
        ptr = C.c_void_p()
        check(self.lib.pe_create(C.byref(ptr), self.E, self.d1, self.d2, 1 << 24, self.J,
                                 device))
        self.ptr = ptr
        # one libpe context is not thread-safe (shared work buffers); the reference lets
        # callers invoke propagators from a thread pool (parareal.py:191-193), so every
        # host-side use of the context is serialised (the GPU work is ordered anyway)
        self.lock = threading.RLock()
        self._keep = []
        for m, (s, ld) in enumerate(zip(systems, loads)):
            if (s.d1, s.d2) != (self.d1, self.d2):
                raise ValueError("all ensemble members need the same (d1, d2)")
            blocks = [_host(x) for x in (s.M11, s.A11, s.M12, s.A12, s.M22, s.A22,
                                         ld.f1, ld.f2)]
            check(self.lib.pe_set_system(self.ptr, m, *[b[1] for b in blocks]))
        self.seq_dt = self.coarse_dt = None
        self.wr_key = None

    def __del__(self):
        try:
            if getattr(self, "ptr", None) is not None and self.ptr.value:
                self.lib.pe_destroy(self.ptr)
                self.ptr = None
        except Exception:
            pass

    # ------------------------------------------------------------------ setup
    def prepare_sequential(self, dt_sub: float):
        if self.seq_dt != dt_sub:
            check(self.lib.pe_prepare_sequential(self.ptr, float(dt_sub)))
            self.seq_dt = dt_sub

    def prepare_coarse(self, dt: float):
        if self.coarse_dt != dt:
            check(self.lib.pe_prepare_coarse(self.ptr, float(dt)))
            self.coarse_dt = dt

    def prepare_allatonce(self, dt_sub: float, alpha: float, tol: float, max_iter: int):
        key = (dt_sub, alpha, tol, max_iter)
        if self.wr_key != key:
            check(self.lib.pe_prepare_allatonce(self.ptr, float(dt_sub), float(alpha),
                                                float(tol), int(max_iter)))
            self.wr_key = key
            self.max_iter = int(max_iter)

    # ------------------------------------------------------------------ helpers
    def stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def to_dev(self, x) -> torch.Tensor:
        return torch.as_tensor(np.asarray(x, dtype=np.float64)).to(self.device).contiguous()

    def empty(self, *shape, dtype=torch.float64):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def reserve_history(self, k_max: int, N: int, pinned: bool = True):
        """Device buffer (+ pinned host staging) for the (k_max + 1, E, N + 1, d) history of
        `parareal`.  Called at setup by the ensemble driver: the pinned copy runs at PCIe
        rate, where a pageable `.cpu()` of the config-4 history (200 MB) took longer than the
        solve.  `parareal` itself only reserves the device buffer (a pinned allocation inside
        a run costs more than the pageable copy of a small history)."""
        shape = (k_max + 1, self.E, N + 1, self.d)
        if getattr(self, "_hist_shape", None) != shape:
            self._hist_dev = self.empty(*shape)
            self._hist_pin = None
            self._hist_shape = shape
        if pinned and self._hist_pin is None:
            try:
                self._hist_pin = torch.empty(shape, dtype=torch.float64, pin_memory=True)
            except RuntimeError:  # no pinned memory left: pageable copies
                self._hist_pin = None
        return self._hist_dev

    # ------------------------------------------------------------------ hot path
    def fine_sequential(self, X: torch.Tensor) -> torch.Tensor:
        """X: (E, nc, d) device -> F(X) over one interval (lags reset)."""
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        check(self.lib.pe_fine_sequential(self.ptr, _ptr(X), _ptr(Y), nc, self.stream()))
        return Y

    def split_step(self, X: torch.Tensor, Xp: torch.Tensor) -> torch.Tensor:
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        check(self.lib.pe_split_step(self.ptr, _ptr(X), _ptr(Xp), _ptr(Y), nc, self.stream()))
        return Y

    def fine_allatonce(self, X: torch.Tensor, record: bool = True):
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        sw = self.empty(self.E, nc, dtype=torch.int32)
        rs = self.empty(self.E, nc, dtype=torch.int32)
        rh = self.empty(self.E, nc, self.max_iter) if record else None
        check(self.lib.pe_fine_allatonce(self.ptr, _ptr(X), _ptr(Y), nc, _ptr(sw), _ptr(rs),
                                         _ptr(rh), self.stream()))
        return Y, sw, rs, rh

    # ------------------------------------------------------------------ time-dependent loads
    def fine_sequential_loads(self, X: torch.Tensor, F: torch.Tensor) -> torch.Tensor:
        """F: (E, nc, J, d) loads [f1; f2] at each substep's end time."""
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        check(self.lib.pe_fine_sequential_loads(self.ptr, _ptr(X), _ptr(Y), nc, _ptr(F),
                                                self.stream()))
        return Y

    def split_step_loads(self, X, Xp, F) -> torch.Tensor:
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        check(self.lib.pe_split_step_loads(self.ptr, _ptr(X), _ptr(Xp), _ptr(Y), nc, _ptr(F),
                                           self.stream()))
        return Y

    def fine_allatonce_loads(self, X: torch.Tensor, F: torch.Tensor, record: bool = True):
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        sw = self.empty(self.E, nc, dtype=torch.int32)
        rs = self.empty(self.E, nc, dtype=torch.int32)
        rh = self.empty(self.E, nc, self.max_iter) if record else None
        check(self.lib.pe_fine_allatonce_loads(self.ptr, _ptr(X), _ptr(Y), nc, _ptr(F),
                                               _ptr(sw), _ptr(rs), _ptr(rh), self.stream()))
        return Y, sw, rs, rh

    def coarse_correct_loads(self, N, X_old, F_hat, G_cache, X_new, Fc, diff=None, active=None):
        check(self.lib.pe_coarse_correct_loads(self.ptr, N, _ptr(X_old), _ptr(F_hat),
                                               _ptr(G_cache), _ptr(X_new), _ptr(diff),
                                               _ptr(active), _ptr(Fc), self.stream()))

    def coarse_apply_loads(self, X: torch.Tensor, Fc: torch.Tensor) -> torch.Tensor:
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        check(self.lib.pe_coarse_apply_loads(self.ptr, _ptr(X), _ptr(Y), nc, _ptr(Fc),
                                             self.stream()))
        return Y

    def wr_waveforms(self, nc: int):
        U = self.empty(self.E, nc, self.J + 1, self.d1)
        W = self.empty(self.E, nc, self.J + 1, self.d2)
        check(self.lib.pe_wr_waveforms(self.ptr, _ptr(U), _ptr(W), nc, self.stream()))
        return U, W

    def wr_solver_residual(self, nc: int) -> torch.Tensor:
        """(E, nc) ImplicitAllAtOnce residual guard of the last all-at-once solve."""
        out = self.empty(self.E, nc)
        check(self.lib.pe_wr_solver_residual(self.ptr, _ptr(out), self.stream()))
        return out

    def coarse_apply(self, X: torch.Tensor) -> torch.Tensor:
        nc = X.shape[1]
        Y = self.empty(self.E, nc, self.d)
        check(self.lib.pe_coarse_apply(self.ptr, _ptr(X), _ptr(Y), nc, self.stream()))
        return Y

    def coarse_correct(self, N, X_old, F_hat, G_cache, X_new, diff=None, active=None):
        check(self.lib.pe_coarse_correct(self.ptr, N, _ptr(X_old), _ptr(F_hat), _ptr(G_cache),
                                         _ptr(X_new), _ptr(diff), _ptr(active), self.stream()))

    def parareal(self, kind: str, N: int, X0: torch.Tensor, k_max: int, epsilon: float,
                 rule: str = "absolute", record_wr: bool = True):
        """Device-resident parareal loop; returns host numpy results per member."""
        E, d = self.E, self.d
        hist = self.reserve_history(k_max, N, pinned=False)
        diffs = np.full((max(k_max, 1), E), np.nan)
        iters = np.zeros(E, dtype=np.int32)
        conv = np.zeros(E, dtype=np.int32)
        fine_ms = np.zeros(max(k_max, 1), dtype=np.float32)
        coarse_ms = np.zeros(max(k_max, 1), dtype=np.float32)
        aao = kind == "all-at-once"
        wsw = self.empty(max(k_max, 1), E, N, dtype=torch.int32) if aao else None
        wrs = self.empty(max(k_max, 1), E, N, dtype=torch.int32) if aao else None
        wrh = self.empty(max(k_max, 1), E, N, self.max_iter) if (aao and record_wr) else None
        k_done = C.c_int(0)
        I = C.POINTER(C.c_int)  # noqa: E741
        F = C.POINTER(C.c_float)
        check(self.lib.pe_parareal_run(
            self.ptr, PE_KIND[kind], N, _ptr(X0), k_max, float(epsilon), PE_RULE[rule],
            _ptr(hist), diffs.ctypes.data_as(_D), iters.ctypes.data_as(I),
            conv.ctypes.data_as(I), _ptr(wsw), _ptr(wrs), _ptr(wrh),
            fine_ms.ctypes.data_as(F), coarse_ms.ctypes.data_as(F), C.byref(k_done),
            self.stream()))
        K = k_done.value
        if self._hist_pin is not None:
            # view of the context's staging buffer: valid until the next `parareal` call
            # (`_runs_from` copies every slab into the ParerealRun it returns)
            self._hist_pin[: K + 1].copy_(hist[: K + 1], non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()
            history = self._hist_pin[: K + 1].numpy()
        else:
            history = hist[: K + 1].cpu().numpy()
        out = dict(history=history, diffs=diffs[:K], iterations=iters,
                   converged=conv.astype(bool), fine_ms=fine_ms[:K], coarse_ms=coarse_ms[:K],
                   k_done=K)
        if aao:
            out["wr_sweeps"] = wsw[:K].cpu().numpy()
            out["wr_reasons"] = wrs[:K].cpu().numpy()
            out["wr_resid"] = wrh[:K].cpu().numpy() if wrh is not None else None
        return out

    def iterate(self, kind: str, N: int, X_old, X_new, G_cache, diff, active=None,
                wr_sweeps=None, wr_reasons=None, wr_resid=None):
        """One parareal iteration X_old -> X_new (the bench "step")."""
        check(self.lib.pe_parareal_iterate(
            self.ptr, PE_KIND[kind], N, _ptr(X_old), _ptr(X_new), _ptr(G_cache), _ptr(diff),
            _ptr(active), _ptr(wr_sweeps), _ptr(wr_reasons), _ptr(wr_resid), self.stream()))

    def set_recurrence(self, on: bool):
        check(self.lib.pe_set_recurrence(self.ptr, 1 if on else 0))

    def set_modal(self, on: bool):
        """Modal (diagonalised) w recursion for the all-at-once solver (pe_set_modal)."""
        check(self.lib.pe_set_modal(self.ptr, 1 if on else 0))

    def modal_level(self) -> int:
        """2: full modal WR sweep, 1: modal w recursion only, 0: direct (pe_wr_is_modal)."""
        rc = self.lib.pe_wr_is_modal(self.ptr)
        check(min(rc, 0))
        return int(rc)

    def is_modal(self) -> bool:
        return self.modal_level() > 0

    def set_profiling(self, on: bool):
        check(self.lib.pe_set_profiling(self.ptr, 1 if on else 0))

    def launch_count(self) -> int:
        return int(self.lib.pe_launch_count(self.ptr))

    def fine_stats(self):
        ms, fl, n = C.c_double(), C.c_double(), C.c_int()
        check(self.lib.pe_last_fine_stats(self.ptr, C.byref(ms), C.byref(fl), C.byref(n)))
        other = C.c_double()
        check(self.lib.pe_last_fine_other_ms(self.ptr, C.byref(other)))
        return dict(gemm_ms=ms.value, gemm_flops=fl.value, launches=n.value,
                    other_ms=other.value)


def stop_reason_name(code: int) -> str:
    return PE_STOP[int(code)]
