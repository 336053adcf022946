"""BASELINE config 4: 64 ensemble members built by the reference's offline CEM code, plus
reference parareal runs per member (TEST / BENCH INFRASTRUCTURE; needs /root/reference).

Member m uses default_rng(m) for the contrast 10^U(2,8), 8 channel rows and 10 %
2x2 inclusions (oracle/configs.py); 100x100 mesh, 10x10 blocks, layers 3, CEM 3+3;
per-member diffusion rescaling c_m; N = J = 32, T = 1; sequential fine
solver; relative 1e-8 stop (F5).

Output (committed): data/cfg4/mNN.npz, one packed system per member
(paper_2411_09244_b200.sysdata, bitwise-exact decoding) with its meta, and
data/cfg4/runs.npz (reference iteration counts of all members, full histories of four).
"""

import json
import os
import sys
import time
from multiprocessing import Pool

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

E = 64
HIST_MEMBERS = (0, 1, 2, 3)


def build(m):
    from oracle.make_golden import BLOCKS, build_system, reference_run

    system, f1, f2, meta = build_system("cfg4", member=m)
    r = reference_run(system, f1, f2, 1.0, 32, 32, "sequential", 0.1, epsilon=1e-8,
                      k_max=32, stop="relative", fine_tol=1e-12)
    blocks = {k: getattr(system, k) for k in BLOCKS}
    return m, blocks, f1, f2, meta, r["iterations"], r["history"], r["seconds"]


def main():
    t0 = time.time()
    workers = int(os.environ.get("BUILD_WORKERS", "8"))
    with Pool(workers) as pool:
        res = []
        for out in pool.imap_unordered(build, range(E)):
            res.append(out)
            print(f"member {out[0]} iterations {out[5]} contrast {out[4]['contrast']:.3g} "
                  f"({time.time() - t0:.0f} s)", flush=True)
    res.sort(key=lambda x: x[0])
    from paper_2411_09244_b200.sysdata import save_system

    out = os.path.join(ROOT, "data", "cfg4")
    os.makedirs(out, exist_ok=True)
    for r in res:
        save_system(os.path.join(out, f"m{r[0]:02d}.npz"), r[1], r[2], r[3], r[4])
    runs = {"iterations": np.array([r[5] for r in res]),
            "contrast": np.array([r[4]["contrast"] for r in res]),
            "kappa_scale": np.array([r[4]["kappa_scale"] for r in res]),
            "ref_seconds": np.array([r[7] for r in res])}
    for m in HIST_MEMBERS:
        runs[f"hist_{m}"] = res[m][6]
    np.savez_compressed(os.path.join(out, "runs.npz"), **runs)
    print("iterations per member:", runs["iterations"].tolist())


if __name__ == "__main__":
    main()
