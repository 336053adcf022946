"""Parareal driver on the GPU (drop-in for paradiff.parareal).

Mirrors `/root/reference/pkg/src/paradiff/parareal.py`: `ParerealConfig` (:31-50),
`SequentialFine` (:53-66), `AllAtOnceFine` (:69-84), `build_fine_propagator` (:87-106),
`ParerealRun` (:109-137), `max_state_diff` / `check_stop` (:140-147), `initial_sweep`
(:150-157) and `run_parareal` (:160-236).

`run_parareal` runs device-resident: the fine sweep over all N intervals is one
batched libpe call (the reference's thread-pool `parallel_map`, util.py:12-23, becomes
the column dimension), and the coarse sweep + correction F + (G_new - G_old) + the
convergence norm is one fused kernel; the host reads one stop flag per iteration.
The stop rule defaults to the reference's absolute max-norm; `stop_rule="relative"`
selects the relative increment of BASELINE.json.
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass, field

import numpy as np

from .allatonce import WaveformRelaxation
from .engine import PeContext, stop_reason_name
from .stepping import ConstantLoads, SplitPropagators, SplitState, TimeGrid

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class ParerealConfig:
    time_grid: TimeGrid
    alpha: float
    epsilon: float = 1e-14
    k_max: int = 100
    fine_kind: str = "all-at-once"
    workers: int = 1
    fine_max_iter: int = 400
    fine_tol: float | None = None
    stop_rule: str = "absolute"

    def resolved_fine_tol(self) -> float:
        """Keep the inner solver's accuracy below the outer stopping regime."""
        if self.fine_tol is not None:
            return self.fine_tol
        return min(1e-12, max(0.01 * self.epsilon, 1e-14))


class SequentialFine:
    """Fine propagator: `substeps` split steps per interval, all intervals batched."""

    kind = "sequential"

    def __init__(self, propagators: SplitPropagators, time_grid: TimeGrid):
        self.propagators = propagators
        self.time_grid = time_grid
        self.ctx = propagators.context(time_grid.substeps)
        self.ctx.prepare_sequential(time_grid.dt_sub)

    def propagate(self, state: SplitState):
        return self.propagate_all([state])[0]

    def propagate_all(self, states):
        ctx = self.ctx
        tg = self.time_grid
        props = self.propagators
        F = (None if props.constant_loads else
             props.fine_load_series([s.t for s in states], tg.dt_sub, tg.substeps))
        with ctx.lock:
            ctx.prepare_sequential(tg.dt_sub)
            X = ctx.to_dev(np.array([s.stacked() for s in states])[None])
            if F is None:
                Y = ctx.fine_sequential(X)[0].cpu().numpy()
            else:
                Y = ctx.fine_sequential_loads(X, ctx.to_dev(F[None]))[0].cpu().numpy()
        d1 = props.system.d1
        out = []
        for y, s in zip(Y, states):
            t = s.t
            for _ in range(tg.substeps):  # the reference's accumulated SplitState.t
                t = t + tg.dt_sub
            out.append((SplitState.fresh(y[:d1], y[d1:], t), {"converged": True}))
        return out


class AllAtOnceFine:
    """Fine propagator backed by the batched waveform-relaxation solver."""

    kind = "all-at-once"

    def __init__(self, wr: WaveformRelaxation):
        self.wr = wr
        self.ctx = wr.ctx

    def propagate(self, state: SplitState):
        return self.propagate_all([state])[0]

    def propagate_all(self, states):
        out = []
        for res in self.wr.solve_all(states, trajectories=False):
            out.append((res.trajectory.final, {
                "converged": res.converged, "iterations": res.iterations,
                "residuals": res.residuals, "stop_reason": res.stop_reason}))
        return out


def build_fine_propagator(config: ParerealConfig, propagators: SplitPropagators,
                          loads: ConstantLoads):
    tg = config.time_grid
    if config.fine_kind == "sequential":
        return SequentialFine(propagators, tg)
    if config.fine_kind == "all-at-once":
        ctx = propagators.context(tg.substeps)
        wr = WaveformRelaxation(propagators.system, tg.substeps, tg.dt, config.alpha, loads,
                                tol=config.resolved_fine_tol(), max_iter=config.fine_max_iter,
                                context=ctx)
        return AllAtOnceFine(wr)
    raise ValueError(f"unknown fine propagator kind {config.fine_kind!r}")


@dataclass
class ParerealRun:
    config: ParerealConfig
    d1: int
    history: list  # per iteration: (N+1, d1+d2) endpoint coefficients
    max_diffs: list
    iterations: int
    converged: bool
    fine_info: list
    fine_seconds: list = field(default_factory=list)
    coarse_seconds: list = field(default_factory=list)
    total_seconds: float = 0.0

    def states_at(self, k: int = -1) -> np.ndarray:
        return self.history[k]

    def endpoint(self, k: int = -1):
        row = self.history[k][-1]
        return row[: self.d1], row[self.d1:]

    def wr_nonconverged(self):
        bad = []
        for k, sweep in enumerate(self.fine_info):
            for n, info in enumerate(sweep):
                if not info.get("converged", True):
                    bad.append((k + 1, n))
        return bad


def max_state_diff(prev: np.ndarray, new: np.ndarray) -> float:
    """Largest Euclidean update over interval endpoints n = 1..N."""
    return float(np.linalg.norm(new[1:] - prev[1:], axis=1).max())


def check_stop(prev: np.ndarray, new: np.ndarray, epsilon: float):
    diff = max_state_diff(prev, new)
    return diff, diff < epsilon


def initial_sweep(propagators: SplitPropagators, initial: SplitState, time_grid: TimeGrid):
    """Sequential coarse pass producing the iteration-0 states (G on the GPU)."""
    states = [initial]
    for _ in range(time_grid.n_intervals):
        states.append(propagators.coarse_step(states[-1], time_grid.dt))
    return states


def _wr_info(res: dict, k: int, e: int, n: int) -> dict:
    it = int(res["wr_sweeps"][k, e, n])
    reason = stop_reason_name(res["wr_reasons"][k, e, n])
    rh = res.get("wr_resid")
    resid = rh[k, e, n, :it].tolist() if rh is not None else []  # C-level float conversion
    return {"converged": reason in ("tol", "floor"), "iterations": it, "residuals": resid,
            "stop_reason": reason}


def _runs_from(res: dict, config: ParerealConfig, d1: int, kind: str, t_total: float):
    E = res["history"].shape[1]
    runs = []
    for e in range(E):
        K = int(res["iterations"][e])
        hist = [res["history"][k, e].copy() for k in range(K + 1)]
        if kind == "all-at-once":
            info = [[_wr_info(res, k, e, n) for n in range(hist[0].shape[0] - 1)]
                    for k in range(K)]
        else:
            info = [[{"converged": True} for _ in range(hist[0].shape[0] - 1)]
                    for _ in range(K)]
        run = ParerealRun(config=config, d1=d1, history=hist,
                          max_diffs=[float(v) for v in res["diffs"][:K, e]], iterations=K,
                          converged=bool(res["converged"][e]), fine_info=info,
                          fine_seconds=[float(v) / 1e3 for v in res["fine_ms"][:K]],
                          coarse_seconds=[float(v) / 1e3 for v in res["coarse_ms"][:K]],
                          total_seconds=t_total)
        bad = run.wr_nonconverged()
        if bad:
            log.warning("fine solver hit max_iter on %d (iteration, interval) pairs", len(bad))
        runs.append(run)
    return runs


def _libpe_context(fine):
    """The libpe context of a fine propagator built by this package, else None."""
    ctx = getattr(fine, "ctx", None)
    return ctx if isinstance(ctx, PeContext) else None


def _parallel_map(fn, items, workers: int = 1) -> list:
    """Ordered map, optionally on a thread pool (util.py:12-23): results are merged in input
    order, so the output does not depend on the worker count."""
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(it) for it in items]
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(fn, items))


def _run_parareal_plugin(config: ParerealConfig, propagators: SplitPropagators, fine,
                         initial: SplitState) -> ParerealRun:
    """`run_parareal` with a user fine propagator (the reference's duck-typed plugin
    contract, parareal.py:53-106,191-193): any object with `propagate(state) -> (state,
    info)`, optionally `propagate_all(states)` for a batch.  The fine sweep calls it once
    per interval (through an ordered thread pool of `config.workers`, util.py:12-23) or
    once per iteration with the batch; the initial coarse sweep, the correction
    F + (G_new - G_old) and the convergence norm stay fused on the GPU (pe_coarse_correct),
    one launch per iteration.  The stop rules and the record are those of the device loop."""
    tg = config.time_grid
    N, d1 = tg.n_intervals, propagators.system.d1
    t_start = time.perf_counter()
    ctx = propagators.context(tg.substeps)
    ctx.prepare_coarse(tg.dt)
    d = ctx.d
    const = propagators.constant_loads
    x0 = initial.stacked()
    X = ctx.to_dev(np.zeros((1, N + 1, d)))
    X[0, 0] = ctx.to_dev(x0)
    G = ctx.empty(1, N, d)
    diff = ctx.empty(1, 2)
    times = [initial.t]  # state times as the reference carries them (t + dt per step)
    for _ in range(N):
        times.append(times[-1] + tg.dt)

    def coarse(X_old, F_hat, X_new, dif):
        if const:
            ctx.coarse_correct(N, X_old, F_hat, G, X_new, dif)
        else:  # G from state n at times[n]: loads at times[n] + dt (stepping.py:164)
            Fc = ctx.to_dev(propagators.load_rows([times[n] + tg.dt for n in range(N)])[None])
            ctx.coarse_correct_loads(N, X_old, F_hat, G, X_new, Fc, dif)

    coarse(X, None, X, None)  # initial_sweep + cached G (parareal.py:178-179)
    hist_rows = X[0].cpu().numpy()
    history = [hist_rows.copy()]
    max_diffs, fine_info, fine_seconds, coarse_seconds = [], [], [], []
    converged = False
    iterations = 0
    for _ in range(config.k_max):
        iterations += 1
        tic = time.perf_counter()
        states = [initial] + [SplitState.fresh(r[:d1], r[d1:], times[n])
                              for n, r in enumerate(hist_rows[1:N], start=1)]
        if hasattr(fine, "propagate_all"):
            results = fine.propagate_all(states)
        else:
            results = _parallel_map(fine.propagate, states, config.workers)
        fine_seconds.append(time.perf_counter() - tic)
        fine_info.append([info for _, info in results])
        times = [initial.t] + [st.t for st, _ in results]
        tic = time.perf_counter()
        F = ctx.to_dev(np.array([st.stacked() for st, _ in results])[None])
        X_new = ctx.empty(1, N + 1, d)
        coarse(X, F, X_new, diff)
        X = X_new
        hist_rows = X[0].cpu().numpy()
        dv = diff[0].cpu().numpy()
        coarse_seconds.append(time.perf_counter() - tic)
        history.append(hist_rows.copy())
        v = float(dv[0]) if config.stop_rule == "absolute" else (
            float(dv[0] / dv[1]) if dv[1] > 0 else float(dv[0]))
        max_diffs.append(v)
        if v < config.epsilon:
            converged = True
            break
    run = ParerealRun(config=config, d1=d1, history=history, max_diffs=max_diffs,
                      iterations=iterations, converged=converged, fine_info=fine_info,
                      fine_seconds=fine_seconds, coarse_seconds=coarse_seconds,
                      total_seconds=time.perf_counter() - t_start)
    bad = run.wr_nonconverged()
    if bad:
        log.warning("fine solver hit max_iter on %d (iteration, interval) pairs", len(bad))
    return run


def run_parareal(config: ParerealConfig, propagators: SplitPropagators, fine,
                 initial: SplitState) -> ParerealRun:
    """Full parareal run on the device; deterministic (fixed reduction order).

    `fine` is a propagator from `build_fine_propagator` (the whole loop then runs
    device-resident in libpe, one host sync per iteration) or any user object following
    the reference's fine-propagator contract (`propagate(state) -> (state, info)`); the
    latter is called per interval and the coarse sweep / correction / norm run on the GPU.
    """
    if config.stop_rule not in ("absolute", "relative"):
        raise ValueError(f"unknown stop rule {config.stop_rule!r}")
    ctx = _libpe_context(fine)
    if ctx is None or not propagators.constant_loads:
        # user propagators, and time-dependent loads (whose per-iteration load series come
        # from the host): host loop over iterations, fine + coarse on the GPU
        if not callable(getattr(fine, "propagate", None)):
            raise TypeError("fine propagator needs a propagate(state) -> (state, info) method")
        return _run_parareal_plugin(config, propagators, fine, initial)
    tg = config.time_grid
    t0 = time.perf_counter()
    ctx.prepare_coarse(tg.dt)
    if fine.kind == "sequential":
        ctx.prepare_sequential(tg.dt_sub)
    else:
        w = fine.wr
        ctx.prepare_allatonce(w.dt, w.alpha, w.tol, w.max_iter)
    X0 = ctx.to_dev(initial.stacked()[None])
    res = ctx.parareal(fine.kind, tg.n_intervals, X0, config.k_max, config.epsilon,
                       config.stop_rule)
    return _runs_from(res, config, propagators.system.d1, fine.kind,
                      time.perf_counter() - t0)[0]


class ParerealEnsemble:
    """E independent problems of equal (d1, d2) solved as one batch (BASELINE config 4).

    Construction uploads the members and factorises (setup, outside any timed region);
    `run(initials)` runs the device-resident parareal loop for all members at once.  Each
    member stops on its own rule and its iterate is frozen afterwards, so every run equals
    the single-member run.
    """

    def __init__(self, config: ParerealConfig, systems, loads, device: int | None = None):
        if config.fine_kind not in ("sequential", "all-at-once"):
            raise ValueError(f"unknown fine propagator kind {config.fine_kind!r}")
        if config.stop_rule not in ("absolute", "relative"):
            raise ValueError(f"unknown stop rule {config.stop_rule!r}")
        self.config = config
        self.d1 = systems[0].d1
        tg = config.time_grid
        self.ctx = PeContext(systems, loads, tg.substeps, device)
        self.ctx.prepare_coarse(tg.dt)
        if config.fine_kind == "sequential":
            self.ctx.prepare_sequential(tg.dt_sub)
        else:
            self.ctx.prepare_allatonce(tg.dt_sub, config.alpha, config.resolved_fine_tol(),
                                       config.fine_max_iter)
        self.ctx.reserve_history(config.k_max, tg.n_intervals)

    def run(self, initials):
        cfg = self.config
        t0 = time.perf_counter()
        X0 = self.ctx.to_dev(np.array([s.stacked() for s in initials]))
        res = self.ctx.parareal(cfg.fine_kind, cfg.time_grid.n_intervals, X0, cfg.k_max,
                                cfg.epsilon, cfg.stop_rule)
        return _runs_from(res, cfg, self.d1, cfg.fine_kind, time.perf_counter() - t0)


def run_parareal_ensemble(config: ParerealConfig, systems, loads, initials,
                          device: int | None = None):
    """One-shot ensemble solve (setup + run); see ParerealEnsemble."""
    return ParerealEnsemble(config, systems, loads, device).run(initials)
