"""CPU-side checks of the C ABI and the host mirror (no GPU needed)."""

import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pe.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pe_[A-Za-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2411_09244_b200 import _lib

    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), f"{n} declared in pe.h but not exported"
        assert n in _lib.SIGNATURES, f"{n} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(names)
    assert b"sm_100a" in lib.pe_version()


def test_library_is_sm100a_dmma():
    """The built cubin targets sm_100a and its GEMM uses FP64 tensor-core DMMA."""
    import shutil
    import subprocess

    from paper_2411_09244_b200 import _lib

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True, check=True).stdout
    assert "sm_100a" in sass
    assert "DMMA" in sass


def test_create_fails_cleanly_without_device_or_with_bad_args():
    import ctypes as C

    from paper_2411_09244_b200 import _lib

    lib = _lib.load()
    p = C.c_void_p()
    rc = lib.pe_create(C.byref(p), 1, 2, 2, 4, 0, 0)  # J = 0 is rejected before any CUDA call
    assert rc == -1
    assert b"J >= 1" in lib.pe_last_error()


def test_host_validation_matches_reference():
    from paper_2411_09244_b200 import ParerealConfig, TimeGrid, TimeMatrixB

    for bad in [(0.0, 1, 1), (1.0, 0, 1), (1.0, 1, 0)]:
        with pytest.raises(ValueError):
            TimeGrid(*bad)
    with pytest.raises(ValueError):
        TimeMatrixB(0, 0.1, 0.5)
    for alpha in (0.0, 1.0, 1.5):
        with pytest.raises(ValueError):
            TimeMatrixB(4, 0.1, alpha)
    tg = TimeGrid(0.005, 2, 2)
    assert ParerealConfig(time_grid=tg, alpha=0.5, epsilon=1e-8).resolved_fine_tol() == 1e-12
    assert ParerealConfig(time_grid=tg, alpha=0.5, epsilon=0.0).resolved_fine_tol() == 1e-14
    assert ParerealConfig(time_grid=tg, alpha=0.5, fine_tol=1e-9).resolved_fine_tol() == 1e-9


def test_time_matrix_closed_forms():
    from paper_2411_09244_b200 import TimeMatrixB

    tm = TimeMatrixB(4, 0.25, 0.3)
    expect = np.array([[1.0, 0, 0, -0.3], [-1, 1, 0, 0], [0, -1, 1, 0], [0, 0, -1, 1]]) / 0.25
    assert np.array_equal(tm.dense(), expect)
    for m in (1, 2, 3, 8, 17):
        t = TimeMatrixB(m, 0.05, 0.4)
        ref = list(np.linalg.eigvals(t.dense()))
        for a in t.eigenvalues():  # greedy multiset match (conjugate pairs)
            dist = [abs(a - b) for b in ref]
            j = int(np.argmin(dist))
            assert dist[j] < 1e-9
            ref.pop(j)


def test_max_state_diff_known_answer():
    from paper_2411_09244_b200 import max_state_diff

    prev = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 2.0]])
    new = np.array([[9.0, 9.0], [1.0, 3.0], [0.0, 2.0]])
    assert max_state_diff(prev, new) == 3.0


def test_solvers_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2411_09244_b200 import (CoarseSystem, ConstantLoads, NativeUnavailable,
                                       SplitPropagators, SplitState)

    s = CoarseSystem(*(np.eye(1) for _ in range(6)))
    props = SplitPropagators(s, ConstantLoads(np.zeros(1), np.zeros(1)))
    with pytest.raises(NativeUnavailable):
        props.coarse_step(SplitState.fresh(np.ones(1), np.ones(1)), 0.1)


def test_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2411_09244_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert "oracle" not in open(os.path.join(pkg, fn)).read().replace(
                "# noqa", ""), fn
