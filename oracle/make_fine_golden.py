"""Golden fixture for the fine-scale accuracy path.

TEST INFRASTRUCTURE: runs the UNMODIFIED reference in the build container
(`/root/reference/pkg/src`, read-only import) on config 0 and writes
`tests/golden/fine_cfg0.npz`:
  * the fine interior operators M, A (A after the kappa rescaling c of sys_cfg0.npz),
    the interior load b and the split basis Psi1, Psi2, all as CSR arrays;
  * `reference_solve` trajectory rows 0, 10, ..., 100 (fem.py:292-318) at n_steps = N*J = 100, a short
    run with a non-zero u0;
  * the per-iteration relative-error series of run_cfg0_seq's history computed with the
    reference's own `relative_error` / `reconstruct` (experiment.py:320-354);
  * the reference writers' bytes (util.write_csv) for conv / timings / wr_residuals of a
    config-1 all-at-once run, plus that run's fields, so writer parity is byte-checked.

Usage:  python oracle/make_fine_golden.py
"""

from __future__ import annotations

import dataclasses
import io
import json
import os
import sys
import tempfile

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.path.insert(0, "/root/reference/pkg/src")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

from paradiff.experiment import relative_error  # noqa: E402
from paradiff.fem import (Channel, SourceSpec, assemble_fine, build_fine_grid,  # noqa: E402
                          generate_field, reference_solve)
from paradiff.msbasis import build_cem_basis, build_coarse_partition  # noqa: E402
from paradiff.parareal import ParerealConfig, build_fine_propagator, run_parareal  # noqa: E402
from paradiff.stepping import ConstantLoads, SplitPropagators, SplitState, TimeGrid  # noqa: E402
from paradiff.util import write_csv  # noqa: E402

from oracle.configs import CONFIGS, rectangles  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def csr_parts(prefix, m):
    m = sp.csr_matrix(m)
    m.sort_indices()
    return {f"{prefix}_ptr": m.indptr.astype(np.int32), f"{prefix}_idx": m.indices.astype(np.int32),
            f"{prefix}_val": m.data.astype(float), f"{prefix}_shape": np.array(m.shape)}


def main():
    c = CONFIGS["cfg0"]
    z = np.load(os.path.join(OUT, "sys_cfg0.npz"))
    meta = json.loads(str(z["meta"]))
    scale = meta["kappa_scale"]
    rects, contrast, _ = rectangles("cfg0", 0)
    grid = build_fine_grid(c["nx"])
    fld = generate_field(grid, 1.0, contrast, [Channel(*r) for r in rects])
    ops = assemble_fine(grid, fld)
    part = build_coarse_partition(grid, c["nb"], c["layers"])
    cache, c1, c2 = {}, [], []
    nd = c["n_dom"]
    for blk in range(part.n_blocks):
        bb = build_cem_basis(part, ops, fld, blk, nd + c["n_comp"], aux_cache=cache)
        c1.append(bb.columns[:, :nd])
        c2.append(bb.columns[:, nd:])
    psi1, psi2 = sp.csc_matrix(np.hstack(c1)), sp.csc_matrix(np.hstack(c2))
    ops_s = dataclasses.replace(ops, A=(scale * ops.A).tocsr())
    src = SourceSpec("constant", 1.0)
    b = ops_s.load(src)
    # consistency with the committed reduced system
    assert np.allclose(psi1.T @ (ops_s.A @ psi1).toarray(), z["A11"], rtol=1e-12, atol=1e-12 * abs(z["A11"]).max())
    assert np.allclose(psi1.T @ b, z["f1"], rtol=1e-13)
    n_steps = c["N"] * c["J"]
    _, traj = reference_solve(ops_s, src, c["T"], n_steps, keep_trajectory=True)
    rng = np.random.default_rng(5)
    u0 = rng.standard_normal(grid.n_interior)
    _, short = reference_solve(ops_s, src, 0.05, 7, u0=u0, keep_trajectory=False)
    run = np.load(os.path.join(OUT, "run_cfg0_seq.npz"))
    hist = run["history"]
    series = []
    for k in range(len(hist)):
        x = hist[k][-1]
        series.append(relative_error(ops_s, traj[-1], psi1 @ x[:psi1.shape[1]] + psi2 @ x[psi1.shape[1]:]))
    # writer bytes from a config-1 all-at-once reference run
    props = SplitPropagators(__import__("paradiff.msbasis", fromlist=["CoarseSystem"]).CoarseSystem(
        **{k: z[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")}), ConstantLoads(z["f1"], z["f2"]))
    cfg = ParerealConfig(time_grid=TimeGrid(1.0, 10, 10), alpha=0.1, epsilon=1e-6, k_max=4,
                         fine_kind="all-at-once", fine_tol=1e-12)
    fine = build_fine_propagator(cfg, props, ConstantLoads(z["f1"], z["f2"]))
    r = run_parareal(cfg, props, fine, SplitState.fresh(np.zeros(z["f1"].size), np.zeros(z["f2"].size)))
    with tempfile.TemporaryDirectory() as td:
        rows = [(k, d, series[k] if k < len(series) else float("nan")) for k, d in enumerate(r.max_diffs, start=1)]
        write_csv(os.path.join(td, "conv.csv"), ["iteration", "max_diff", "relative_error"], rows)
        write_csv(os.path.join(td, "tim.csv"), ["iteration", "fine_seconds", "coarse_seconds"],
                  [(k + 1, r.fine_seconds[k], r.coarse_seconds[k]) for k in range(len(r.fine_seconds))])
        wr = [(k, i, j, res) for k, sw in enumerate(r.fine_info, start=1) for i, info in enumerate(sw)
              for j, res in enumerate(info.get("residuals", []), start=1)]
        write_csv(os.path.join(td, "wr.csv"), ["sweep", "interval", "iteration", "residual"], wr)
        texts = {k: open(os.path.join(td, f)).read() for k, f in
                 (("csv_conv", "conv.csv"), ("csv_timings", "tim.csv"), ("csv_wr", "wr.csv"))}
    resid = [[list(info["residuals"]) for info in sw] for sw in r.fine_info]
    np.savez_compressed(
        os.path.join(OUT, "fine_cfg0.npz"),
        b=b, traj=traj[::10], u0=u0, short=short, series=np.array(series), nx=c["nx"],
        n_interior=grid.n_interior, interior=np.asarray(grid.interior),
        w_max_diffs=np.array(r.max_diffs), w_fine_seconds=np.array(r.fine_seconds),
        w_coarse_seconds=np.array(r.coarse_seconds), w_residuals=json.dumps(resid),
        **texts, **csr_parts("M", ops_s.M), **csr_parts("A", ops_s.A),
        **csr_parts("P1", psi1), **csr_parts("P2", psi2))
    print("n_interior", grid.n_interior, "series", np.array(series))


if __name__ == "__main__":
    main()
