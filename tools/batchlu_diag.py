import ctypes as C, sys, numpy as np, torch
from paper_2411_09244_b200 import _lib
lib = _lib.require_cuda()
def ours(A):
    b, n, _ = A.shape
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    dX = torch.empty((b, n, n), dtype=torch.float64, device="cuda")
    info = (C.c_int * b)()
    _lib.check(lib.pe_batched_inverse(n, b, C.c_void_p(dA.data_ptr()), C.c_void_p(dX.data_ptr()), info, None))
    return dX.cpu().numpy()
def report(name, A):
    ld = np.longdouble if A.shape[0] <= 300 else np.float64
    Al = A.astype(ld)
    X1 = ours(A[None])[0]
    X2 = torch.linalg.inv(torch.from_numpy(A).cuda()).cpu().numpy()
    X3 = np.linalg.inv(A)
    n = A.shape[0]
    I = np.eye(n)
    out = {}
    for k, X in (("libpe", X1), ("torch", X2), ("numpy", X3)):
        Xl = X.astype(ld)
        out[k] = (float(np.abs(Al @ Xl - I).max()), float(np.abs(Xl @ Al - I).max()), float(np.abs(X - X3).max() / np.abs(X3).max()))
    print(name, n, "cond %.2e" % np.linalg.cond(A), {k: tuple("%.1e" % v for v in t) for k, t in out.items()}, flush=True)
rng = np.random.default_rng(0)
for n in (64, 300, 2048):
    Q = rng.standard_normal((n, n)); report("spd", Q @ Q.T / n + np.eye(n))
    report("gauss", rng.standard_normal((n, n)))
from paper_2411_09244_b200 import sysdata
for m in (0, 20, 45):
    blocks, f1, f2, meta = sysdata.load_system("data/cfg4/m%02d.npz" % m)
    dt = 1.0 / 32 / 32
    report("cfg4 m%d K11" % m, blocks["M11"] / dt + blocks["A11"])
    report("cfg4 m%d M22" % m, blocks["M22"])
    d1 = blocks["M11"].shape[0]
    M = np.block([[blocks["M11"], blocks["M12"]], [blocks["M12"].T, blocks["M22"]]])
    Ab = np.block([[blocks["A11"], blocks["A12"]], [blocks["A12"].T, blocks["A22"]]])
    report("cfg4 m%d KG" % m, M * 32 + Ab)
