"""ctypes binding of libpe (include/pe.h).  Loads the in-tree .so; fails loudly.

There is no CPU fallback: if the library or a CUDA device is missing, every solver
entry point raises `NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpe.so")

PE_STOP = ("tol", "diverged", "floor", "max_iter")
PE_RULE = {"absolute": 0, "relative": 1}
PE_KIND = {"sequential": 0, "all-at-once": 1}


class NativeUnavailable(RuntimeError):
    """libpe.so is not built or no CUDA device is visible."""


class PeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libpe error {code}: {msg}")
        self.code = code


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_F = C.POINTER(C.c_float)

# name -> (restype, argtypes)
SIGNATURES = {
    "pe_last_error": (C.c_char_p, []),
    "pe_version": (C.c_char_p, []),
    "pe_create": (C.c_int, [C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "pe_destroy": (C.c_int, [_P]),
    "pe_set_system": (C.c_int, [_P, C.c_int] + [_D] * 8),
    "pe_prepare_sequential": (C.c_int, [_P, C.c_double]),
    "pe_prepare_coarse": (C.c_int, [_P, C.c_double]),
    "pe_prepare_allatonce": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_int]),
    "pe_fine_sequential": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "pe_split_step": (C.c_int, [_P, _P, _P, _P, C.c_int, _P]),
    "pe_fine_allatonce": (C.c_int, [_P, _P, _P, C.c_int, _P, _P, _P, _P]),
    "pe_wr_waveforms": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "pe_coarse_apply": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "pe_coarse_correct": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _P, _P, _P]),
    "pe_parareal_run": (C.c_int, [_P, C.c_int, C.c_int, _P, C.c_int, C.c_double, C.c_int, _P,
                                  _D, _I, _I, _P, _P, _P, _F, _F, _I, _P]),
    "pe_gemm_f64": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _P, C.c_longlong,
                              C.c_longlong, C.c_longlong, _P, C.c_longlong, C.c_longlong,
                              C.c_longlong, _P, C.c_longlong, C.c_longlong, C.c_longlong, _P]),
    "pe_parareal_iterate": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, _P, _P, _P, _P, _P, _P,
                                      _P]),
    "pe_set_profiling": (C.c_int, [_P, C.c_int]),
    "pe_set_recurrence": (C.c_int, [_P, C.c_int]),
    "pe_set_modal": (C.c_int, [_P, C.c_int]),
    "pe_last_fine_other_ms": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "pe_wr_is_modal": (C.c_int, [_P]),
    "pe_launch_count": (C.c_longlong, [_P]),
    "pe_last_fine_stats": (C.c_int, [_P, _D, _D, _I]),
    "pe_fine_reference_solve": (C.c_int, [C.c_int, _I, _I, _D, _I, _I, _D, _D, _D, C.c_double,
                                          C.c_int, C.c_int, _D, _F, _P]),
    "pe_fine_solver_kind": (C.c_int, [C.c_int, _I, _I, _I, _I, _I]),
    "pe_relative_error_series": (C.c_int, [C.c_int, C.c_int, _I, _I, _D, _I, _I, _D, _D,
                                           C.c_int, _D, _D, _P]),
    "pe_project_coarse": (C.c_int, [C.c_int, C.c_int, C.c_int, _I, _I, _D, _I, _I, _D, _I, _I,
                                    _D, _D, _D, _D, _D, _D, _P]),
    "pe_project_load": (C.c_int, [C.c_int, C.c_int, _I, _I, _D, _D, _D, _P]),
    "pe_apply_S": (C.c_int, [C.c_int, C.c_longlong, C.c_double, C.c_int, _P, _P, _P, _P, _P]),
    "pe_build_rhs": (C.c_int, [C.c_int, C.c_int, C.c_int] + [_P] * 9 + [C.c_double, C.c_double,
                                                                       _P, _P]),
    "pe_allatonce_usolve": (C.c_int, [_P, _P, _P, C.c_int, _P, _P]),
    "pe_wr_solver_residual": (C.c_int, [_P, _P, _P]),
    "pe_project_initial": (C.c_int, [C.c_int, C.c_int, C.c_int, _I, _I, _D, _I, _I, _D, _D, _D,
                                     _D, _D, _D, _P]),
    "pe_stability_max_step": (C.c_int, [_P, C.c_int, C.c_double, C.c_int, _D, _I, _P]),
    "pe_cem_basis": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _D, C.c_double, _D,
                               C.POINTER(C.c_longlong), _D, _D, _P]),
    "pe_cem_basis_size": (C.c_longlong, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "pe_fine_sequential_loads": (C.c_int, [_P, _P, _P, C.c_int, _P, _P]),
    "pe_split_step_loads": (C.c_int, [_P, _P, _P, _P, C.c_int, _P, _P]),
    "pe_fine_allatonce_loads": (C.c_int, [_P, _P, _P, C.c_int, _P, _P, _P, _P, _P]),
    "pe_coarse_correct_loads": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pe_coarse_apply_loads": (C.c_int, [_P, _P, _P, C.c_int, _P, _P]),
    "pe_batched_inverse": (C.c_int, [C.c_int, C.c_int, _P, _P, _I, _P]),
    "pe_shifted_inverses": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, _P, _P, _P, _P,
                                      _P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libpe and bind every exported symbol of include/pe.h (no GPU needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is not built; run `make` (or __graft_entry__.build()) first")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib


def check(rc: int):
    if rc != 0:
        msg = _lib.pe_last_error().decode(errors="replace") if _lib else "?"
        raise PeError(rc, msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; libpe has no CPU path")
    return load()
