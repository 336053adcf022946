"""Measure the FP64 roofline denominators on the box: cuBLAS DGEMM (torch float64 matmul)
and libpe's DMMA GEMM on the same shapes.  MEASURED_PEAKS.json has no FP64 entry
(SURVEY §0 F8), so bench.py uses profiles/fp64_peak.json written by this script."""

import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_09244_b200 import _lib  # noqa: E402


def time_it(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    lib = _lib.require_cuda()
    out = {"gpu": torch.cuda.get_device_name(0)}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, n, dtype=torch.float64, device="cuda")
        c = torch.empty(n, n, dtype=torch.float64, device="cuda")
        ms = time_it(lambda: torch.matmul(a, b, out=c))
        out[f"cublas_dgemm_{n}_tflops"] = 2 * n ** 3 / ms / 1e9
        bt = b.T.contiguous()
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

        def mine():
            _lib.check(lib.pe_gemm_f64(n, n, n, 1, C.c_void_p(a.data_ptr()), n, 1, 0,
                                       C.c_void_p(bt.data_ptr()), 1, n, 0,
                                       C.c_void_p(c.data_ptr()), 1, n, 0, st))

        ms = time_it(mine, reps=5)
        out[f"libpe_dmma_{n}_tflops"] = 2 * n ** 3 / ms / 1e9
        ref = a @ b
        out[f"libpe_dmma_{n}_maxerr"] = float(((c.T - ref).abs().max() / ref.abs().max()))
        print(json.dumps(out), flush=True)
    x = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ms = time_it(lambda: y.copy_(x))
    out["copy_gbs"] = 2 * x.numel() * 8 / ms / 1e6
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fp64_peak.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
