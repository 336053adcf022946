"""Offline build on the GPU: CEM basis + Galerkin projection of a
config, timed, and compared with the reference-built operators committed in the repo.

    python tools/cem_build_bench.py [cfg3|cfg2|cfg0]

Writes gpurun_out/cem_<cfg>.json: seconds for the basis build and the projection, the
constraint residual, and the max block deviation from the reference's CoarseSystem
(relative to each block's max).  The reference's own build of config 3 takes ~6 min on 8
processes (oracle/build_cfg3.py; 2.5-6 s per block single-threaded).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_09244_b200 as P  # noqa: E402
from oracle.configs import CONFIGS, assemble_fine, corner_load, gaussian_cell_values, \
    kappa_field, rectangles  # noqa: E402
from paper_2411_09244_b200.sysdata import load_system  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
c = CONFIGS[name]
kap = kappa_field(name)
t0 = time.perf_counter()
M, A = assemble_fine(c["nx"], kap)
t_asm = time.perf_counter() - t0
P.build_cem_space(8, 2, 1, np.ones(64), 2, 2)  # warm-up: handles, module load
t0 = time.perf_counter()
space = P.build_cem_space(c["nx"], c["nb"], c["layers"], kap, c["n_dom"], c["n_comp"])
t_basis = time.perf_counter() - t0
if name == "cfg3":
    blocks, f1, f2, meta = load_system(os.path.join(ROOT, "data", "cfg3"))
else:
    z = np.load(os.path.join(ROOT, "tests", "golden", f"sys_{name}.npz"))
    blocks = {k: z[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")}
    f1, f2, meta = z["f1"], z["f2"], json.loads(str(z["meta"]))
ops = type("Ops", (), {})()
ops.M, ops.A = M, A * meta["kappa_scale"]
t0 = time.perf_counter()
cs = P.project_coarse(space.Psi1, space.Psi2, ops)
t_proj = time.perf_counter() - t0
dev = {k: float(np.abs(getattr(cs, k) - blocks[k]).max() / np.abs(blocks[k]).max())
       for k in blocks}


def invariants(s, f1, f2):
    """Unchanged by orthogonal transforms within Psi1 / Psi2 (eigenvector sign ties and
    repeated eigenvalues of the aux problems, tests/test_gpu_cem.py)."""
    import scipy.linalg as sla

    out = {"eig11": np.sort(sla.eigh(s["A11"], s["M11"], eigvals_only=True)),
           "eig22": np.sort(sla.eigh(s["A22"], s["M22"], eigvals_only=True))}
    l1, l2 = np.linalg.cholesky(s["M11"]), np.linalg.cholesky(s["M22"])
    cm = sla.solve_triangular(l1, sla.solve_triangular(l2, s["M12"].T, lower=True).T, lower=True)
    out["mass_angles"] = np.linalg.svd(cm, compute_uv=False)
    out["f1"] = np.array([f1 @ np.linalg.solve(s["M11"], f1)])
    out["f2"] = np.array([f2 @ np.linalg.solve(s["M22"], f2)])
    return out
_, _, src = rectangles(name)
if src == "constant":
    fc = np.ones(c["nx"] * c["nx"])
else:
    fc = gaussian_cell_values(c["nx"], *src[1:])
g1, g2 = P.project_load(space, corner_load(c["nx"], fc))
load_dev = max(float(np.abs(g1 - f1).max() / np.abs(f1).max()),
               float(np.abs(g2 - f2).max() / np.abs(f2).max()))
t0 = time.perf_counter()
mine = invariants({k: getattr(cs, k) for k in blocks}, g1, g2)
ref = invariants(blocks, f1, f2)
inv_dev = {k: float(np.abs(mine[k] - ref[k]).max() / np.abs(ref[k]).max()) for k in ref}
t_inv = time.perf_counter() - t0
out = dict(config=name, basis_seconds=t_basis, projection_seconds=t_proj,
           invariant_rel_dev=inv_dev, invariant_seconds=t_inv,
           host_assembly_seconds=t_asm, constraint_residual=space.constraint_residual,
           max_block_rel_dev=max(dev.values()), block_rel_dev=dev, load_rel_dev=load_dev,
           d1=space.Psi1.shape[1], d2=space.Psi2.shape[1], basis_nnz=int(space.Psi1.nnz + space.Psi2.nnz),
           reference_build_seconds=meta.get("build_seconds"),
           reference_build_workers=meta.get("workers"))
print(json.dumps(out, indent=1))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"cem_{name}.json"), "w") as f:
    json.dump(out, f, indent=1)
