"""Time libpe's DMMA GEMM (pe_gemm_f64, col-major C) against cuBLAS on the hot-path
shapes.  PE_GEMM_VARIANT=<id> forces a fast-path tile variant (tuning only);
PE_GEMM_TRACE=1 prints the variant the cost model picks."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_09244_b200 import _lib  # noqa: E402

SHAPES = [  # (M, N, K, batch, label); label ending in "jc": B stored j-contiguous (K x N)
    (64, 19200, 64, 1, "cfg2 time transform jc"),
    (300, 4096, 600, 1, "cfg2 rhs/g"),
    (300, 4096, 300, 2, "cfg2 modal norms"),
    (300, 64, 300, 16, "cfg2 blocked-w H step"),
    (300, 64, 300, 48, "cfg2 blocked-w fill"),
    (300, 64, 600, 66, "cfg2 shifted (batched)"),
    (600, 64, 1200, 1, "cfg2 seq step"),
    (600, 32, 1200, 64, "cfg4 seq step"),
    (600, 32, 1200, 32, "cfg4 seq step chunk"),
    (4096, 12800, 8192, 1, "cfg3 rhs/g"),
    (4096, 128, 8192, 50, "cfg3 shifted (batched)"),
    (8192, 8192, 8192, 1, "square"),
]


def main():
    lib = _lib.require_cuda()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    only = os.environ.get("GEMM_BENCH_ONLY")
    for M, N, K, b, label in SHAPES:
        if only and only not in label:
            continue
        A = torch.randn(b, M, K, dtype=torch.float64, device="cuda")
        jc = label.endswith("jc")
        if jc:
            B = torch.randn(b, K, N, dtype=torch.float64, device="cuda")  # j-contiguous rows
            bk, bj = N, 1
        else:
            B = torch.randn(b, N, K, dtype=torch.float64, device="cuda")  # k-contiguous columns
            bk, bj = 1, K
        Cm = torch.empty(b, N, M, dtype=torch.float64, device="cuda")

        def mine():
            _lib.check(lib.pe_gemm_f64(M, N, K, b, C.c_void_p(A.data_ptr()), K, 1, M * K,
                                       C.c_void_p(B.data_ptr()), bk, bj, N * K,
                                       C.c_void_p(Cm.data_ptr()), 1, M, M * N, st))

        def cublas():
            torch.bmm(A, B if jc else B.transpose(1, 2))

        res = {}
        for name, fn in (("libpe", mine), ("cublas", cublas)):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res[name] = (ms, 2.0 * M * N * K * b / ms / 1e9)
        print(f"{label:24s} M={M:5d} N={N:5d} K={K:5d} b={b:3d}  libpe {res['libpe'][0]*1e3:9.1f} us "
              f"{res['libpe'][1]:6.2f} TF/s   cuBLAS {res['cublas'][0]*1e3:9.1f} us {res['cublas'][1]:6.2f} TF/s",
              flush=True)


if __name__ == "__main__":
    main()
