"""Artifact writers for GPU parareal runs (output compatibility).

Byte-compatible with the reference's experiment outputs so downstream scripts read a
GPU run unchanged: `write_csv` / `save_matrix_txt` follow util.py:26-50, and
`write_run_artifacts` writes the per-N files of `_emit_all` (experiment.py:398-450):
runs.csv rows, conv_N*.csv, timings_N*.csv, wr_residuals_N*.csv and, optionally, the
solution / reference node grids.  The accuracy numbers come from `fem.error_series`
(GPU); nothing here computes on the CPU beyond formatting.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path

import numpy as np


def _fmt(value):
    # util.py:46-50: floats at full round-trip precision, everything else via str()
    if isinstance(value, (float, np.floating)):
        return format(float(value), ".17g")
    return value


def write_csv(path, header, rows) -> None:
    """Rows of mixed scalars as CSV (util.py:36-43)."""
    with Path(path).open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        for row in rows:
            w.writerow([_fmt(v) for v in row])


def save_matrix_txt(path, array) -> None:
    """A matrix as plain text, one row per line, full precision (util.py:26-29)."""
    np.savetxt(path, np.atleast_2d(np.asarray(array)), fmt="%.17g")


def runs_rows(results, gamma):
    """runs.csv rows (experiment.py:410-417) from (n, run, relative_error) triples."""
    return [(n, run.iterations, int(run.converged), err, gamma, run.total_seconds)
            for n, run, err in results]


RUNS_HEADER = ["n", "iterations", "converged", "relative_error", "gamma", "wall_seconds"]


def write_run_artifacts(out_dir, n, run, error_series=(), *, solution_grid=None,
                        reference_grid=None) -> list[Path]:
    """The per-N files of the reference's `_emit_all` (experiment.py:418-450).

    `run` is a ParerealRun (ours or the reference's); `error_series[k]` is the relative
    error of iterate k (index 0 = the initial coarse sweep), NaN where absent.
    Returns the written paths.
    """
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    written = []

    def path(name):
        p = out / name
        written.append(p)
        return p

    rows = []
    for k, diff in enumerate(run.max_diffs, start=1):
        err_k = error_series[k] if k < len(error_series) else float("nan")
        rows.append((k, diff, err_k))
    write_csv(path(f"conv_N{n}.csv"), ["iteration", "max_diff", "relative_error"], rows)
    write_csv(path(f"timings_N{n}.csv"), ["iteration", "fine_seconds", "coarse_seconds"],
              [(k + 1, run.fine_seconds[k], run.coarse_seconds[k])
               for k in range(len(run.fine_seconds))])
    wr_rows = []
    for k, sweep in enumerate(run.fine_info, start=1):
        for interval, info in enumerate(sweep):
            for j, res in enumerate(info.get("residuals", []), start=1):
                wr_rows.append((k, interval, j, res))
    write_csv(path(f"wr_residuals_N{n}.csv"), ["sweep", "interval", "iteration", "residual"],
              wr_rows)
    if solution_grid is not None:
        save_matrix_txt(path(f"solution_N{n}.txt"), solution_grid)
    if reference_grid is not None:
        save_matrix_txt(path(f"reference_N{n}.txt"), reference_grid)
    return written


# ------------------------------------------------------------------ run_single on the GPU


@dataclass
class RunResult:
    """experiment.py:309-317."""

    n: int
    run: object
    relative_error: float
    error_series: list
    reference_final: np.ndarray | None
    stability_bound: float
    dt_sub: float


def run_single(pipe, n: int, *, stop_rule: str = "absolute") -> RunResult:
    """One parareal run plus its Eq (31) accuracy series, all on the GPU
    (experiment.py:328-360).

    `pipe` is the reference's `Pipeline` (or any object with `config`, `space` (system,
    Psi1, Psi2), `loads`, `ops`, `grid`): the offline build stays in the reference.  The
    initial state is the projection of the zero fine field (`project_initial` of zeros is
    exactly zero).  Only the time-grid fields of `pipe.config` are read, plus
    `compute_reference` and `to_source()`.
    """
    import logging

    from .fem import error_series, reference_solve
    from .parareal import ParerealConfig, build_fine_propagator, run_parareal
    from .stepping import ConstantLoads, SplitPropagators, SplitState, TimeGrid

    cfg = pipe.config
    tg = cfg.time_grid(n)
    tg = TimeGrid(tg.t_end, tg.n_intervals, tg.substeps)
    loads = pipe.loads
    if getattr(loads, "constant", False):
        loads = ConstantLoads(*loads.at(0.0))
    # otherwise a time-dependent provider with at(t), used as given (stepping.py:125,164)
    if getattr(cfg, "compute_reference", False):
        from .fem import check_reference_size

        check_reference_size(pipe.ops)
    props = SplitPropagators(pipe.space.system, loads)
    bound = props.stability_max_step()
    if tg.dt_sub > bound:
        logging.getLogger(__name__).warning(
            "N=%d substep %.3e exceeds stability bound %.3e", n, tg.dt_sub, bound)
    pconfig = ParerealConfig(time_grid=tg, alpha=cfg.alpha, epsilon=cfg.epsilon,
                             k_max=cfg.k_max, fine_kind=cfg.fine_kind, workers=cfg.workers,
                             stop_rule=stop_rule)
    fine = build_fine_propagator(pconfig, props, loads)
    s = pipe.space.system
    initial = SplitState.fresh(np.zeros(s.M11.shape[0]), np.zeros(s.M22.shape[0]))
    run = run_parareal(pconfig, props, fine, initial)
    ref_final, err, series = None, float("nan"), []
    if getattr(cfg, "compute_reference", False):
        _, states = reference_solve(pipe.ops, cfg.to_source(), cfg.t_end,
                                    tg.n_intervals * tg.substeps, keep_trajectory=False)
        ref_final = states[-1]
        series = error_series(pipe.ops, pipe.space, ref_final,
                              [np.asarray(h)[-1] for h in run.history])
        err = series[-1]
    return RunResult(n, run, err, series, ref_final, bound, tg.dt_sub)
