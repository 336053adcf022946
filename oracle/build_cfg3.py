"""Parallel offline build of the BASELINE config-3 reduced system with the reference's
own CEM code (TEST / BENCH INFRASTRUCTURE; needs /root/reference in this container).

1024 coarse blocks x `build_cem_basis` (2.5-6 s each single-threaded) are
split over worker processes by contiguous block ranges; each worker keeps its own
aux-eigenproblem cache (boundary blocks of a range are solved twice, which is harmless:
`aux_eigen_cem` is deterministic).  Columns are stacked in ascending block order exactly
as `make_golden.build_system` does, then `project_coarse` and the F2 rescaling.

Output: data/cfg3/ (committed): one packed file per block (paper_2411_09244_b200.sysdata:
nonzero mask + byte-shuffled zlib values, upper triangle of the symmetric blocks; the
blocks are 13 % nonzero, 63 MB in total instead of 0.8 GB dense) plus loads.npz with the
loads and the build meta.  Decoding is bitwise exact.
"""

from __future__ import annotations

import json
import os
import sys
import time
from multiprocessing import Pool

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

CFG = "cfg3"
_state = {}


def _setup():
    from paradiff.fem import Channel, assemble_fine, build_fine_grid, generate_field
    from paradiff.msbasis import build_coarse_partition

    from oracle.configs import CONFIGS, rectangles

    c = CONFIGS[CFG]
    rects, contrast, src = rectangles(CFG)
    grid = build_fine_grid(c["nx"])
    fld = generate_field(grid, 1.0, contrast, [Channel(*r) for r in rects])
    ops = assemble_fine(grid, fld)
    part = build_coarse_partition(grid, c["nb"], c["layers"])
    return c, grid, fld, ops, part, src, len(rects), contrast


def _work(block_range):
    from paradiff.msbasis import build_cem_basis

    if "ctx" not in _state:
        _state["ctx"] = _setup()
        _state["cache"] = {}
    c, grid, fld, ops, part, _, _, _ = _state["ctx"]
    out = []
    for b in block_range:
        bb = build_cem_basis(part, ops, fld, b, c["n_dom"] + c["n_comp"],
                             aux_cache=_state["cache"])
        cols = bb.columns
        nz = np.nonzero(np.abs(cols).sum(axis=1))[0]
        out.append((b, nz, cols[nz]))
    return out


def main():
    import scipy.sparse as sp
    from paradiff.msbasis import CoarseSystem, project_coarse
    from paradiff.stepping import ConstantLoads, SplitPropagators

    from oracle.configs import R_STABILITY, corner_load, gaussian_cell_values

    workers = int(os.environ.get("BUILD_WORKERS", "8"))
    t0 = time.time()
    c, grid, fld, ops, part, src, n_rects, contrast = _setup()
    nblk = part.n_blocks
    chunk = 16
    ranges = [range(i, min(i + chunk, nblk)) for i in range(0, nblk, chunk)]
    with Pool(workers) as pool:
        parts = []
        for i, res in enumerate(pool.imap(_work, ranges)):
            parts.extend(res)
            print(f"  blocks done {min((i + 1) * chunk, nblk)}/{nblk} "
                  f"({time.time() - t0:.0f} s)", flush=True)
    parts.sort(key=lambda x: x[0])
    nd = c["n_dom"]
    n_int = grid.n_interior
    rows1, cols1, vals1, rows2, cols2, vals2 = [], [], [], [], [], []
    for b, nz, cb in parts:
        for j in range(cb.shape[1]):
            if j < nd:
                rows1.append(nz); cols1.append(np.full(nz.size, b * nd + j)); vals1.append(cb[:, j])
            else:
                k = b * (cb.shape[1] - nd) + (j - nd)
                rows2.append(nz); cols2.append(np.full(nz.size, k)); vals2.append(cb[:, j])
    d1 = nblk * nd
    d2 = nblk * c["n_comp"]
    psi1 = sp.csc_matrix((np.concatenate(vals1), (np.concatenate(rows1), np.concatenate(cols1))),
                         shape=(n_int, d1))
    psi2 = sp.csc_matrix((np.concatenate(vals2), (np.concatenate(rows2), np.concatenate(cols2))),
                         shape=(n_int, d2))
    system = project_coarse(psi1, psi2, ops)
    _, x, y, sig = src
    bload = corner_load(c["nx"], gaussian_cell_values(c["nx"], x, y, sig))
    f1 = np.asarray(psi1.T @ bload)
    f2 = np.asarray(psi2.T @ bload)
    build_s = time.time() - t0
    bound = SplitPropagators(system, ConstantLoads(f1, f2)).stability_max_step()
    scale = R_STABILITY * bound * c["N"] / c["T"]
    meta = dict(name=CFG, contrast=contrast, kappa_scale=scale, bound_before=bound,
                dt_over_bound=R_STABILITY, d1=d1, d2=d2, n_rects=n_rects,
                build_seconds=build_s, workers=workers)
    from paper_2411_09244_b200.sysdata import save_system

    blocks = dict(M11=system.M11, A11=scale * system.A11, M12=system.M12,
                  A12=scale * system.A12, M22=system.M22, A22=scale * system.A22)
    save_system(os.path.join("data", "cfg3"), blocks, f1, f2, meta, split=True)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
