"""Time the GPU fine-scale reference solve (fem.reference_solve).

Synthetic fine operators with the reference's structure on an nx x nx cell grid
(interior nodes (nx-1)^2): bilinear-FEM-like 9-point mass and a 5-point stiffness with a
two-valued kappa (contrast 1e4 channels); the step cost depends only on n.  Prints one
JSON line per size: step time, HBM GB/s over the algorithmic bytes (R once + u, c, u'
per step) and the fraction of the measured copy bandwidth; plus the CPU splu step time
(the reference's algorithm, oracle restatement) on a bounded sample of steps.

    python tools/bench_finescale.py [--nx 100 256] [--steps 400]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
import types

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def operators(nx, seed=0):
    m = nx - 1
    h = 1.0 / nx
    rng = np.random.default_rng(seed)
    one = np.ones(m)
    T = sp.diags([one[:-1], 4 * one, one[:-1]], [-1, 0, 1])
    M = (sp.kron(T, T) * (h * h / 36.0)).tocsr()
    # stiffness G^T diag(kappa_edge) G on the x and y edges: SPD, two-valued kappa
    G1 = sp.diags([np.ones(m), -np.ones(m)], [0, -1], shape=(m + 1, m))
    I = sp.identity(m)
    Gx, Gy = sp.kron(I, G1).tocsr(), sp.kron(G1, I).tocsr()
    kx = np.where(rng.random(Gx.shape[0]) < 0.1, 1e4, 1.0)
    ky = np.where(rng.random(Gy.shape[0]) < 0.1, 1e4, 1.0)
    A = (Gx.T @ sp.diags(kx) @ Gx + Gy.T @ sp.diags(ky) @ Gy).tocsr() * 1e-3
    return M, A, np.full(m * m, h * h)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, nargs="+", default=[100, 256])
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--project", type=str, default="", help="nx:d:density[:gpuonly][,...] projection runs")
    args = ap.parse_args()
    for spec in filter(None, args.project.split(",")):
        nx, d, dens, *flag = spec.split(":")
        bench_project(int(nx), int(d), float(dens), cpu=not flag)
    if args.project:
        return
    from paper_2411_09244_b200 import fem
    from oracle import pe_oracle as po

    peak = None
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        try:
            peak = float(json.load(open(mp)).get("hbm_gbs") or 0) or None
        except Exception:
            peak = None
    for nx in args.nx:
        M, A, b = operators(nx)
        n = M.shape[0]
        ops = types.SimpleNamespace(M=M, A=A)
        fem.reference_solve(ops, b, 1.0, 4, keep_trajectory=False)  # warm-up (same sizes)
        t0 = time.perf_counter()
        tm = {}
        _, st = fem.reference_solve(ops, b, 1.0, args.steps, keep_trajectory=False, timing=tm)
        wall = time.perf_counter() - t0
        step_ms = tm["step_ms"] / args.steps
        gbs = tm["bytes_per_step"] / (step_ms * 1e-3) / 1e9
        t1 = time.perf_counter()
        ref = po.fine_reference_solve(M, A, b, 1.0 * args.cpu_steps / args.steps, args.cpu_steps,
                                      keep_trajectory=False)
        cpu_ms = (time.perf_counter() - t1) * 1e3 / args.cpu_steps
        _, chk = fem.reference_solve(ops, b, 1.0 * args.cpu_steps / args.steps, args.cpu_steps,
                                     keep_trajectory=False)
        rel = float(np.linalg.norm(chk[1] - ref[1]) / np.linalg.norm(ref[1]))
        print(json.dumps(dict(nx=nx, n=n, solver=tm.get("solver"), block=tm.get("block"),
                              steps=args.steps, step_ms=step_ms, hbm_gbs=gbs,
                              peak_gbs=peak, frac=(gbs / peak if peak else None),
                              bytes_per_step=tm["bytes_per_step"], wall_s_incl_setup=wall,
                              cpu_splu_step_ms=cpu_ms, speedup_per_step=cpu_ms / step_ms,
                              rel_vs_splu=rel, final_norm=float(np.linalg.norm(st[1])))))



def bench_project(nx, d, density, seed=0, cpu=True):
    """GPU project_coarse vs the reference's sparse products (msbasis.py:552-562) on a
    random basis of the given density (cfg3: d = 8192, ~13 % nonzero)."""
    import paper_2411_09244_b200 as P

    M, A, b = operators(nx)
    n = M.shape[0]
    psi = sp.random(n, d, density=density, random_state=seed, format="csc")
    p1, p2 = psi[:, : d // 2], psi[:, d // 2:]
    ops = types.SimpleNamespace(M=M, A=A)
    P.project_coarse(p1[:, :8], p2[:, :8], ops)  # warm-up
    t0 = time.perf_counter()
    cs = P.project_coarse(p1, p2, ops)
    gpu = time.perf_counter() - t0
    if not cpu:
        print(json.dumps(dict(kind="project_coarse", nx=nx, n=n, d=d, density=density,
                              gpu_s_both_operators_incl_upload=gpu)))
        return
    t1 = time.perf_counter()
    xp1, xp2 = M @ p1, M @ p2
    b11 = (p1.T @ xp1).toarray()
    b12 = (p1.T @ xp2).toarray()
    b22 = (p2.T @ xp2).toarray()
    cpu_m = time.perf_counter() - t1
    err = max(np.abs(cs.M11 - (b11 + b11.T) / 2).max(), np.abs(cs.M12 - b12).max(),
              np.abs(cs.M22 - (b22 + b22.T) / 2).max()) / np.abs(b11).max()
    print(json.dumps(dict(kind="project_coarse", nx=nx, n=n, d=d, density=density,
                          gpu_s_both_operators_incl_upload=gpu,
                          cpu_s_mass_only_reference_sparse=cpu_m, rel_err_vs_sparse=float(err))))


if __name__ == "__main__":
    main()
