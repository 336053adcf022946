"""Time libpe's batched shifted inversion (pe_shifted_inverses, batchlu.cu) against
torch.linalg.inv on the same complex batch (cuSOLVER / MAGMA batched getrf + getri)."""
import ctypes as C
import json
import sys

import numpy as np
import torch

from paper_2411_09244_b200 import _lib

lib = _lib.require_cuda()


def bench(d1, J, reps=3):
    rng = np.random.default_rng(0)
    Q = rng.standard_normal((d1, d1))
    M = torch.from_numpy(Q @ Q.T / d1 + np.eye(d1)).cuda()
    Q = rng.standard_normal((d1, d1))
    A = torch.from_numpy(30 * (Q @ Q.T / d1 + np.eye(d1))).cuda()
    dt, alpha = 0.01, 0.1
    re = torch.empty((J, d1, d1), dtype=torch.float64, device="cuda")
    im = torch.empty_like(re)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def ours():
        _lib.check(lib.pe_shifted_inverses(d1, J, dt, alpha, C.c_void_p(M.data_ptr()),
                                           C.c_void_p(A.data_ptr()), C.c_void_p(re.data_ptr()),
                                           C.c_void_p(im.data_ptr()), None))

    k = np.arange(J // 2 + 1)
    dk = torch.from_numpy((1.0 - alpha ** (1.0 / J) * np.exp(-2j * np.pi * k / J)) / dt).cuda()
    S = dk[:, None, None] * M.to(torch.complex128) + A.to(torch.complex128)

    def lib_inv():
        return torch.linalg.inv(S)

    out = {}
    for name, fn in (("libpe_ms", ours), ("torch_linalg_inv_ms", lib_inv)):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            ev[0].record()
            fn()
            ev[1].record()
            torch.cuda.synchronize()
            best = min(best, ev[0].elapsed_time(ev[1]))
        out[name] = best
    ref = lib_inv()
    got = (re + 1j * im)[: J // 2 + 1]
    out["max_rel_diff"] = float((got - ref).abs().max() / ref.abs().max())
    out.update(d1=d1, J=J, modes_factored=J // 2 + 1, block_form_n=2 * d1)
    return out


cases = ((32, 10), (300, 64), (1024, 32), (4096, 8))
if len(sys.argv) > 2:
    cases = ((int(sys.argv[1]), int(sys.argv[2])),)
for d1, J in cases:
    print(json.dumps(bench(d1, J, reps=1 if len(sys.argv) > 2 else 3)), flush=True)
