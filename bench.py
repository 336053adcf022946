"""Benchmark: reduced-DOF x fine-steps per second per parareal iteration (FP64).

A "step" is one parareal iteration of the hot path (parareal.py:188-215): the fine
sweep over all N coarse intervals (the all-at-once waveform-relaxation solver for the
default workload) plus the fused coarse sweep / correction / convergence norm, on one
batch of seeded inputs already resident in HBM.  units/step = E * (d1+d2) * N * J.

    python bench.py [--gpus N --steps K --warmup W] [--workload cfg3-aao] [--impl reference]

Default workload: BASELINE config 3 (256x256 mesh, CEM 4+4 -> d = 4096+4096, N = 128,
J = 100, channels + inclusions at 1e4, all-at-once fine solver, alpha = 0.1), the
largest single-GPU configuration, with the reduced operators built by the reference's own
offline CEM code (data/cfg3: oracle/build_cfg3.py, packed by paper_2411_09244_b200.sysdata).

--gpus N > 1 (re-executed under torchrun when WORLD_SIZE is unset): one process per GPU
over NCCL.  Default: the intervals of the one problem are sharded across the ranks, one
all-gather of the fine endpoints per iteration (sharded.py, strong scaling);
`--shard replicas` runs independent replicas instead (weak scaling, no collective).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
METRIC = "reduced-DOF·fine-steps/s per parareal iteration (FP64); % of roofline"
UNIT = "reduced-DOF*fine-steps/s"
FINE_TOL = 1e-12
STOP_EPS = 1e-8  # relative-increment stop of BASELINE.json

WORKLOADS = {
    # BASELINE config 3.  WR contracts at 0.943 per sweep here and needs ~502 sweeps to reach
    # tol = 1e-12, so the reference's default 400-sweep cap (ParerealConfig.fine_max_iter)
    # would stop every interval unconverged: the cap is raised to 600.
    # Parareal itself needs ~50 iterations at this config, so the e2e leg runs a fixed 3.
    "cfg3-aao": dict(data="data/cfg3", T=2.0, N=128, J=100, kind="all-at-once", alpha=0.1,
                     max_iter=600, golden="cfg3_sample.npz", e2e_iters=3),
    "cfg2-aao": dict(data="tests/golden/sys_cfg2.npz", T=1.0, N=64, J=64, kind="all-at-once",
                     alpha=0.1, max_iter=400, golden="run_cfg2_aao.npz"),
    "cfg2-seq": dict(data="tests/golden/sys_cfg2.npz", T=1.0, N=64, J=64, kind="sequential",
                     alpha=0.1, max_iter=400, golden="run_cfg2_seq.npz"),
    "cfg0-seq": dict(data="tests/golden/sys_cfg0.npz", T=1.0, N=10, J=10, kind="sequential",
                     alpha=0.1, max_iter=400, golden="run_cfg0_seq.npz"),
    "cfg1-aao": dict(data="tests/golden/sys_cfg0.npz", T=1.0, N=10, J=10, kind="all-at-once",
                     alpha=0.1, max_iter=400, golden="run_cfg1_aao.npz"),
    # BASELINE config 4: 64 seeded members (own contrast 10^U(2,8), own kappa rescaling)
    "cfg4-seq": dict(data="data/cfg4", T=1.0, N=32, J=32, kind="sequential", alpha=0.1,
                     max_iter=400, members=64, golden="data/cfg4/runs.npz"),
}
DEFAULT_WORKLOAD = "cfg3-aao"
BLOCKS = ("M11", "A11", "M12", "A12", "M22", "A22")


# ---------------------------------------------------------------------- inputs

def load_workload(wl):
    """[(blocks, f1, f2)] per member and a representative meta dict."""
    from paper_2411_09244_b200.sysdata import load_system

    path = os.path.join(ROOT, wl["data"])
    if not os.path.exists(path):
        raise SystemExit(f"bench: workload data {wl['data']} is missing")
    if wl.get("members"):
        mem, metas = [], []
        for m in range(wl["members"]):
            b, f1, f2, meta = load_system(os.path.join(path, f"m{m:02d}.npz"))
            mem.append((b, f1, f2))
            metas.append(meta)
        meta = dict(metas[0])
        meta["members"] = len(mem)
        meta["contrast"] = [min(x["contrast"] for x in metas), max(x["contrast"] for x in metas)]
        meta["kappa_scale"] = [min(x["kappa_scale"] for x in metas),
                               max(x["kappa_scale"] for x in metas)]
        return mem, meta
    if os.path.isdir(path):
        b, f1, f2, meta = load_system(path)
        return [(b, f1, f2)], meta
    z = np.load(path)
    return ([({k: np.ascontiguousarray(z[k]) for k in BLOCKS}, z["f1"], z["f2"])],
            json.loads(str(z["meta"])))


def golden(wl):
    name = wl.get("golden")
    if not name:
        return None
    p = os.path.join(ROOT, name) if "/" in name else os.path.join(ROOT, "tests", "golden", name)
    return np.load(p) if os.path.exists(p) else None


def config_dict(args, wl, meta, d1, d2, E):
    """The `config` object; identical for the libpe arm and the reference arm."""
    return dict(workload=args.workload, d1=d1, d2=d2, N=wl["N"], J=wl["J"], E=E,
                kind=wl["kind"], alpha=wl["alpha"], fine_tol=FINE_TOL,
                fine_max_iter=wl["max_iter"], stop=f"relative increment < {STOP_EPS:g}",
                kappa_scale=meta["kappa_scale"], contrast=meta.get("contrast"),
                units_per_step=E * (d1 + d2) * wl["N"] * wl["J"],
                step="one parareal iteration: fine sweep over N intervals + coarse sweep / "
                     "correction / convergence norm",
                l2="GPU arm: L2 flushed (320 MB write) before every timed step")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.result = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if sm:
            busy = [v for v in sm if smax and v > 0.5 * smax] or sm
            self.result = {"sm_mhz": statistics.median(busy), "sm_max_mhz": smax,
                           "samples": len(sm), "reasons": sorted(reasons)}


def fp64_peak_tflops(torch):
    """cuBLAS DGEMM 8192^3 burst, measured in this run (MEASURED_PEAKS.json has no FP64)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b, c
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / best / 1e9


class CudaBackend:
    """The real arm: libpe on one GPU per rank, NCCL, CUDA events on the launch stream."""

    name = "cuda"
    dist_backend = "nccl"

    def __init__(self, local):
        import torch

        self.torch = torch
        torch.cuda.set_device(local)
        self.local = local
        self.device = torch.device("cuda", local)

    def init_dist(self, dist):
        dist.init_process_group("nccl", device_id=self.device)

    def sync(self):
        self.torch.cuda.synchronize()

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)

    def make_context(self, P, systems, loads, J):
        return P.PeContext(systems, loads, J, self.local)

    def clocks(self):
        return ClockSampler(self.local)

    def flush_buffer(self):
        return self.torch.empty(320 * 1024 * 1024 // 8, dtype=self.torch.float64,
                                device=self.device)

    def fp64_peak(self):
        return fp64_peak_tflops(self.torch)


def make_backend(local):
    """CudaBackend, or (dry runs of the multi-process logic from the tests only) the class
    named by PE_BENCH_BACKEND=module:attr, constructed with the local rank."""
    spec = os.environ.get("PE_BENCH_BACKEND")
    if not spec:
        return CudaBackend(local)
    import importlib

    mod, attr = spec.split(":")
    return getattr(importlib.import_module(mod), attr)(local)


# ---------------------------------------------------------------------- CPU arms

def _osys(blocks, f1, f2):
    from oracle import pe_oracle as po

    return po.OSystem(*(blocks[k] for k in BLOCKS), f1, f2)


def _initial_states(s, wl):
    """Iteration-0 states by the oracle's coarse sweep (also times one coarse sweep)."""
    from oracle import pe_oracle as po

    sp = po.OracleSplit(s)
    N, T = wl["N"], wl["T"]
    states = [np.zeros(s.d1 + s.d2)]
    t0 = time.perf_counter()
    for _ in range(N):
        states.append(sp.coarse_step(states[-1], T / N))
    return states, time.perf_counter() - t0


class CpuSampler:
    """Times the CPU restatement of the reference path (oracle/pe_oracle.py, the same
    NumPy/LAPACK calls as the reference) on a bounded sample of one parareal iteration
    of the workload, on the host's cores; `sample()` is one bounded step and returns
    (extrapolated seconds per parareal iteration, measured seconds of this sample)."""

    def __init__(self, wl, blocks, f1, f2, cores):
        from threadpoolctl import threadpool_limits

        from oracle import pe_oracle as po

        self.wl, self.cores = wl, cores
        self.s = s = _osys(blocks, f1, f2)
        N, J, T = wl["N"], wl["J"], wl["T"]
        self.large = s.d1 > 2048
        t0 = time.perf_counter()
        with threadpool_limits(cores):
            self.states, self.t_coarse = _initial_states(s, wl)
            if self.large:
                # config 3: the reference's setup stores J = 100 complex inverses of
                # 4096^2 (26.8 GB, hours with the stacked np.linalg.inv); two
                # modes are formed and the shifted apply is timed per mode
                dt = T / N / J
                lam = po.time_eigenvalues(J, dt, wl["alpha"])
                self.invs = [np.linalg.inv(lam[k] * s.M11 + s.A11.astype(complex))
                             for k in (1, 2)]
                self.m22_inv = np.linalg.inv(s.M22)
                self.e_mat = np.eye(s.d2) - dt * self.m22_inv @ s.A22
                g = golden(wl)
                self.sweeps = (float(np.mean(g["oracle_sweeps"])) if g is not None and
                               "oracle_sweeps" in g else float(wl["max_iter"]))
            elif wl["kind"] == "all-at-once":
                self.wr = po.OracleWR(s, J, T / N, wl["alpha"], tol=FINE_TOL,
                                      max_iter=wl["max_iter"])
            else:
                self.sp = po.OracleSplit(s)
        self.setup_s = time.perf_counter() - t0
        self.next = 0

    def sample(self):
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits

        from oracle import pe_oracle as po

        s, wl, cores = self.s, self.wl, self.cores
        N, J, T = wl["N"], wl["J"], wl["T"]
        d1 = s.d1
        t_start = time.perf_counter()
        if self.large:
            rng = np.random.default_rng(0)
            p = rng.standard_normal((1, d1)) + 1j * rng.standard_normal((1, d1))
            with threadpool_limits(1):
                def apply(_):
                    t0 = time.perf_counter()
                    for inv in self.invs:
                        np.einsum("kij,kj->ki", inv[None], p)
                    return time.perf_counter() - t0
                with ThreadPoolExecutor(max_workers=cores) as pool:
                    t_modes = max(pool.map(apply, range(cores)))
                t_mode = t_modes / (2 * cores)  # per mode-apply, pool aggregate
                u0 = np.zeros(d1)
                w0 = np.zeros(s.d2)
                W = rng.standard_normal((J, s.d2)) * 1e-3
                dt = T / N / J
                t0 = time.perf_counter()
                rhs = po.build_rhs(s, np.tile(s.f1, (J, 1)), u0, w0, w0, W, u0, dt, wl["alpha"])
                q = po.apply_S(po.apply_S_inverse(rhs, wl["alpha"]), wl["alpha"]).real
                uh = np.vstack([u0, u0, q[:-1]])
                g = dt * (np.tile(s.f2, (J, 1)) - (uh[1:] - uh[:-1]) / dt @ s.M12
                          - q @ s.A12) @ self.m22_inv
                w = w0
                for i in range(J):
                    w = self.e_mat @ w + g[i]
                t_rest = time.perf_counter() - t0
            t_sweep = J * t_mode + t_rest / cores
            t_iter = N * self.sweeps * t_sweep + self.t_coarse
            info = dict(extrapolated=True, sample=(
                f"per step: the einsum shifted apply (allatonce.py:118) on 2 of J={J} modes on "
                f"{cores} threads ({t_mode * 1e3:.1f} ms per mode-apply, pool aggregate) + one "
                f"build_rhs / FFT pair / w-sweep ({t_rest:.2f} s); extrapolated x J modes x "
                f"{self.sweeps:.1f} sweeps (the CPU oracle's mean on sampled intervals, "
                f"tests/golden/cfg3_sample.npz) x N={N} intervals + one measured coarse sweep "
                f"({self.t_coarse:.2f} s); setup (26.8 GB of inverses) excluded"))
        elif wl["kind"] == "all-at-once":
            # one round of `cores` concurrent WR interval solves (workers = cores, BLAS 1
            # thread: the reference's best setting) x ceil(N / cores) rounds
            n0 = self.next
            idx = [(n0 + i) % N for i in range(min(N, cores))]
            self.next = (n0 + len(idx)) % N
            with threadpool_limits(1):
                with ThreadPoolExecutor(max_workers=cores) as pool:
                    res = list(pool.map(
                        lambda n: self.wr.solve(self.states[n][:d1], self.states[n][d1:]), idx))
            t_round = time.perf_counter() - t_start
            rounds = math.ceil(N / len(idx))
            t_iter = t_round * rounds + self.t_coarse
            sw = [r["iterations"] for r in res]
            info = dict(extrapolated=rounds > 1, sample=(
                f"per step: WR solves of intervals {idx[0]}..{idx[-1]} (iteration-1 inputs, "
                f"{min(sw)}-{max(sw)} sweeps) concurrently on {len(idx)} threads, BLAS 1 "
                f"thread ({t_round:.2f} s) x {rounds} rounds for the N={N} intervals + one "
                f"measured coarse sweep ({self.t_coarse:.3f} s)"))
        else:
            # sequential fine intervals, workers = 1, BLAS 1 thread (the reference's best
            # setting: the GIL-bound pool does not help this kind)
            budget = 8.0
            with threadpool_limits(1):
                n_s = 0
                while n_s < N:
                    v = self.states[(self.next + n_s) % N]
                    self.sp.fine_interval(v[:d1], v[d1:], T / N, J)
                    n_s += 1
                    if time.perf_counter() - t_start > budget:
                        break
            self.next = (self.next + n_s) % N
            t_f = time.perf_counter() - t_start
            t_iter = t_f * N / n_s + self.t_coarse
            info = dict(extrapolated=n_s < N, sample=(
                f"per step: {n_s} of {N} sequential fine intervals (workers=1, BLAS 1 thread) "
                f"({t_f:.2f} s) x N/{n_s} + one measured coarse sweep ({self.t_coarse:.3f} s)"))
            cores = 1
        info["cores"] = cores
        return t_iter, time.perf_counter() - t_start, info


def reference_arm(args, wl):
    """`--impl reference`: the reference's CPU path (its restatement in oracle/, the same
    NumPy/LAPACK calls) on the box's host cores, W + K bounded steps."""
    mem, meta = load_workload(wl)
    E = len(mem)
    blocks, f1, f2 = mem[0]
    d1, d2 = blocks["M11"].shape[0], blocks["M22"].shape[0]
    units = E * (d1 + d2) * wl["N"] * wl["J"]
    cores = len(os.sched_getaffinity(0))
    sampler = CpuSampler(wl, blocks, f1, f2, cores)
    vals, measured = [], []
    info = {}
    for i in range(args.warmup + args.steps):
        t_iter, t_meas, info = sampler.sample()
        if i >= args.warmup:
            vals.append(units / (E * t_iter))  # members run one after the other
            measured.append(t_meas)
    v = statistics.median(vals)
    cpu = dict(value=v, unit=UNIT, cores=info["cores"], kind="port", sample=info["sample"],
               extrapolated=info["extrapolated"],
               measured_s_per_step=statistics.mean(measured), setup_s=sampler.setup_s)
    if E > 1:
        cpu["sample"] += f"; member 0 of {E} timed, x{E} members (run one after the other)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(measured) * 1e3,
            "ms_per_step_note": ("measured wall time of one bounded CPU sample step; `value` "
                                 "is the extrapolated full-iteration throughput (cpu_baseline)"),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded kappa field per BASELINE config; reduced operators built "
                    "by the reference's offline CEM code)",
            "config": config_dict(args, wl, meta, d1, d2, E),
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- GPU arm

def _recorded_cfg3_iterations():
    path = os.path.join(ROOT, "profiles", "r02", "cfg3_parareal.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        rec = json.load(f)
    return int(rec["iterations"]) if rec.get("converged") else None


def parity_check(P, wl, ctx, system, loads, run_history, run_iterations, kind):
    """Parity of this run against the committed reference / oracle vectors."""
    g = golden(wl)
    if g is None:
        return {"status": "no golden for this workload"}
    d1 = system.d1
    rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))  # noqa
    if "sample" in g:  # config 3: sampled intervals vs the full-sweep CPU oracle
        res = []
        ok_sweeps = 0
        for key in ("it1",) + tuple(k[:-len("_x")] for k in g.files
                                    if k.startswith("k") and k.endswith("_x")):
            X = g[f"{key}_x"]
            wr = P.WaveformRelaxation(system, wl["J"], wl["T"] / wl["N"], wl["alpha"], loads,
                                      tol=FINE_TOL, max_iter=wl["max_iter"], context=ctx)
            out = wr.solve_all([P.SplitState.fresh(x[:d1], x[d1:]) for x in X],
                               trajectories=False)
            for i, r in enumerate(out):
                res.append(rel(r.trajectory.final.stacked(), g[f"{key}_final"][i]))
                ok_sweeps += int(r.iterations == int(g[f"{key}_sweeps"][i]))
        return {"what": "WR finals on sampled (iteration, interval) inputs vs the CPU oracle's "
                        "full-sweep solves (tests/golden/cfg3_sample.npz); a full reference "
                        "run is infeasible at config 3 (SURVEY F7)",
                "intervals": len(res), "max_rel_l2": max(res),
                "sweeps_equal": f"{ok_sweeps}/{len(res)}",
                "iterations_gpu": _recorded_cfg3_iterations(), "iterations_ref": None,
                "iterations_note": "iterations_gpu is the recorded full run to the relative "
                                   "1e-8 stop (tools/cfg3_parareal_run.py, "
                                   "profiles/r02/cfg3_parareal.json: ~18 min on one B200), not "
                                   "re-run by the bench; the reference needs ~7 hours per "
                                   "iteration on the CPU (cpu_baseline), so iterations_ref "
                                   "does not exist"}
    if "history" in g and g["history"].ndim == 3:  # full reference run (cfg0/1/2)
        K = min(len(run_history), g["history"].shape[0])
        return {"what": "full parareal run vs the unmodified reference's run on the same inputs",
                "iterations_gpu": run_iterations, "iterations_ref": int(g["iterations"]),
                "max_rel_l2": max(rel(run_history[k], g["history"][k]) for k in range(K))}
    if "iterations" in g:  # cfg4 per-member counts
        return {"what": "per-member parareal iteration counts vs the reference's runs",
                "iterations_gpu": run_iterations, "iterations_ref": g["iterations"].tolist(),
                "members_equal": int(np.sum(np.array(run_iterations) == g["iterations"])),
                "max_rel_l2_members_0_3": max(rel(run_history[m], g[f"hist_{m}"])
                                              for m in range(4))}
    return {"status": "golden has no comparable fields"}


def gpu_arm(args, wl):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    be = make_backend(local)
    be.workload = args.workload
    dev = be.device
    dist = None
    if world > 1:
        import torch.distributed as dist

        be.init_dist(dist)
    import paper_2411_09244_b200 as P

    mem, meta = load_workload(wl)
    systems = [P.CoarseSystem(**b) for b, _, _ in mem]
    loads_l = [P.ConstantLoads(a, b) for _, a, b in mem]
    system, loads = systems[0], loads_l[0]
    shard = args.shard == "intervals" and world > 1
    E = len(mem)
    N, J, T, kind = wl["N"], wl["J"], wl["T"], wl["kind"]
    max_iter = wl["max_iter"]
    d = system.d1 + system.d2
    units = E * d * N * J  # per replica / per problem
    be.sync()
    t_setup = time.perf_counter()
    ctx = be.make_context(P, systems, loads_l, J)
    be.sync()
    t_upload = time.perf_counter() - t_setup
    ctx.prepare_coarse(T / N)
    if kind == "sequential":
        ctx.prepare_sequential(T / N / J)
    else:
        ctx.prepare_allatonce(T / N / J, wl["alpha"], FINE_TOL, max_iter)
    be.sync()
    t_setup = time.perf_counter() - t_setup
    modal = ctx.modal_level() if kind == "all-at-once" else None

    A = torch.zeros(E, N + 1, d, dtype=torch.float64, device=dev)
    B = torch.zeros_like(A)
    Gc = torch.zeros(E, N, d, dtype=torch.float64, device=dev)
    diff = torch.zeros(E, 2, dtype=torch.float64, device=dev)
    ctx.coarse_correct(N, A, None, Gc, A)  # initial coarse sweep (x_0 = 0, u0 = 0 projection)
    flush = be.flush_buffer()
    sweeps_buf = torch.zeros(E, N, dtype=torch.int32, device=dev) if kind != "sequential" \
        else None
    sweeps_seen = []

    if shard:
        from paper_2411_09244_b200.dist import shard_members

        ranges = [shard_members(N, r, world) for r in range(world)]
        mine = ranges[rank]
        m_loc = max(len(r) for r in ranges)
        F_loc = torch.zeros(E, m_loc, d, dtype=torch.float64, device=dev)
        parts = [torch.empty_like(F_loc) for _ in range(world)]

        def step(x_old, x_new):
            if len(mine):
                Xs = x_old[:, mine.start:mine.stop].contiguous()
                if kind == "sequential":
                    F_loc[:, : len(mine)] = ctx.fine_sequential(Xs)
                else:
                    Y, sw, _, _ = ctx.fine_allatonce(Xs, record=False)
                    F_loc[:, : len(mine)] = Y
                    sweeps_seen.append(sw)
            dist.all_gather(parts, F_loc)  # the one exchange per iteration (NCCL)
            F = torch.cat([p[:, : len(r)] for p, r in zip(parts, ranges)], dim=1)
            ctx.coarse_correct(N, x_old, F.contiguous(), Gc, x_new, diff)
    else:
        def step(x_old, x_new):
            ctx.iterate(kind, N, x_old, x_new, Gc, diff, wr_sweeps=sweeps_buf)
            if sweeps_buf is not None:
                sweeps_seen.append(sweeps_buf.clone())

    for _ in range(args.warmup):
        step(A, B)
        A, B = B, A
    be.sync()
    sweeps_seen.clear()
    if dist:
        dist.barrier()
    launches0 = ctx.launch_count()
    starts = [be.event() for _ in range(args.steps)]
    ends = [be.event() for _ in range(args.steps)]
    with be.clocks() as clk:
        be.sync()
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))  # evict L2 (320 MB > 126 MB) between timed steps
            starts[i].record()
            step(A, B)
            ends[i].record()
            A, B = B, A
        be.sync()
        t_wall = time.perf_counter() - t_wall
    if dist:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    launches = ctx.launch_count() - launches0
    total_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # whole job: one problem (sharded) or `world` replicas
    value = (1 if shard else world) * units * args.steps / (total_ms / 1e3)
    sw_all = (torch.cat([s.reshape(-1) for s in sweeps_seen]).cpu().numpy()
              if sweeps_seen else None)

    # roofline pass: one extra instrumented step, every DMMA launch bracketed by events
    ctx.set_profiling(True)
    flush.fill_(0.0)
    step(A, B)
    be.sync()
    st = ctx.fine_stats()
    ctx.set_profiling(False)
    peak = be.fp64_peak()
    achieved = st["gemm_flops"] / (st["gemm_ms"] / 1e3) / 1e12 if st["gemm_ms"] > 0 else 0.0
    step_avg = total_ms / args.steps

    # end to end through the public API: host initial state in, full host history out,
    # run to the BASELINE stop rule (relative increment < 1e-8) -> the GPU iteration count;
    # config 3 (~50 parareal iterations of ~32 s) runs a fixed number of iterations instead
    fixed = wl.get("e2e_iters")
    cfg = P.ParerealConfig(time_grid=P.TimeGrid(T, N, J), alpha=wl["alpha"],
                           epsilon=0.0 if fixed else STOP_EPS,
                           k_max=fixed or min(N, 40), fine_kind=kind, fine_tol=FINE_TOL,
                           fine_max_iter=max_iter, stop_rule="relative")
    zeros = P.SplitState.fresh(np.zeros(system.d1), np.zeros(system.d2))
    if dist:
        dist.barrier()
    be.sync()
    if shard:
        from paper_2411_09244_b200.sharded import LibpeShardOps, run_parareal_sharded

        ops = LibpeShardOps(ctx, kind)
        t0 = time.perf_counter()
        res = run_parareal_sharded(N, np.zeros(d), ops, cfg.k_max, cfg.epsilon, "relative")
        be.sync()
        e2e_s = time.perf_counter() - t0
        K, hist = res["iterations"], list(res["history"])
        iters = K
        path = (f"paper_2411_09244_b200.run_parareal_sharded ({world} ranks, intervals sharded, "
                "host arrays in/out)")
    elif E == 1:
        props = P.SplitPropagators(system, loads)
        props._ctx[J] = ctx  # reuse the factorised context (setup stays out of e2e)
        fine = P.build_fine_propagator(cfg, props, loads)
        t0 = time.perf_counter()
        run = P.run_parareal(cfg, props, fine, zeros)
        be.sync()
        e2e_s = time.perf_counter() - t0
        K, hist, iters = run.iterations, run.history, run.iterations
        path = "paper_2411_09244_b200.run_parareal (host arrays in/out)"
    else:
        ens = P.ParerealEnsemble(cfg, systems, loads_l)  # setup stays out of e2e
        be.sync()
        t0 = time.perf_counter()
        runs = ens.run([zeros] * E)
        be.sync()
        e2e_s = time.perf_counter() - t0
        K = max(r.iterations for r in runs)
        iters = [r.iterations for r in runs]
        hist = [np.array(r.history) for r in runs]
        path = f"paper_2411_09244_b200.ParerealEnsemble.run ({E} members, host arrays in/out)"
    wr_bytes = K * N * (4 + 4 + 8 * max_iter) if kind == "all-at-once" else 0
    e2e = {"value": units * K / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": E * d * 8 / K,
           "d2h_bytes_per_step": E * ((K + 1) * (N + 1) * d * 8 + wr_bytes) / K,
           "path": path, "iterations": K, "seconds": e2e_s,
           "run": (f"fixed {fixed} iterations (epsilon 0)" if fixed else
                   f"to the relative {STOP_EPS:g} stop")}

    line = None
    if rank == 0:
        parity = (parity_check(P, wl, ctx, system, loads, hist, iters, kind) if be.name == "cuda"
                  else {"status": f"dry run ({be.name} backend): no parity check"})
        cpu = None
        if world == 1 and not args.no_cpu and be.name == "cuda":
            blocks, f1, f2 = mem[0]
            sampler = CpuSampler(wl, blocks, f1, f2, len(os.sched_getaffinity(0)))
            t_iter, t_meas, info = sampler.sample()
            cpu = dict(value=units / (E * t_iter), unit=UNIT, cores=info["cores"], kind="port",
                       sample=info["sample"], extrapolated=info["extrapolated"],
                       measured_s=t_meas)
        wr = None
        if sw_all is not None:
            wr = {"sweeps_min": int(sw_all.min()), "sweeps_mean": float(sw_all.mean()),
                  "sweeps_max": int(sw_all.max()),
                  "at_cap": int(np.sum(sw_all >= max_iter)), "solves": int(sw_all.size)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_avg,
            "higher_is_better": True, "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded kappa field per BASELINE config; reduced operators built "
                    "by the reference's offline CEM code, " + wl["data"] + ")",
            "config": config_dict(args, wl, meta, system.d1, system.d2, E),
            "parallelism": (f"intervals sharded over {world} ranks, one NCCL all-gather of the "
                            "fine endpoints per iteration" if shard else
                            f"{world} independent replica(s), no collective"),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": None,
                         "kernel": "every FP64 DMMA (m8n8k4) launch of one instrumented step: "
                                   "GEMMs + recurrence / all-SM chains; algorithmic flops "
                                   "(structural zeros and re-associated work not counted)",
                         "gemm_launches": st["launches"], "gemm_ms": st["gemm_ms"],
                         "gemm_flops": st["gemm_flops"],
                         "gemm_share_of_step": st["gemm_ms"] / step_avg,
                         "other_kernels_ms": st.get("other_ms", 0.0),
                         "other_share_of_step": st.get("other_ms", 0.0) / step_avg,
                         "peak_source": "cuBLAS DGEMM 8192^3 burst measured in this run "
                                        "(MEASURED_PEAKS.json has no FP64 entry)"},
            "wr_sweeps_timed": wr,
            "parity": parity,
            "cpu_baseline": cpu,
            "setup": {"upload_s": t_upload, "factorisations_s": t_setup - t_upload,
                      "what": ("pe_create + pe_set_system uploads; G, sequential operator T or "
                               "the all-at-once pencil eigendecompositions (modal level "
                               f"{modal}) on the GPU; excluded from the step")},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.result,
            "wall_s_timed": t_wall,
        }
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            tr = json.load(open(tpath)).get(args.workload)
            if tr:
                line["roofline"]["traffic"] = tr.get("dram_bytes_per_launch")
                line["roofline"]["traffic_detail"] = tr
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return line


def relaunch_under_torchrun(n):
    """`--gpus N` without a torchrun environment: one process per GPU on this node."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libpe", choices=["libpe", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--shard", default="intervals", choices=["replicas", "intervals"],
                    help="N > 1: one problem with its intervals sharded across the ranks "
                         "(strong scaling, default) or independent replicas (weak scaling)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("bench: at least 3 warm-up steps")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch_under_torchrun(args.gpus))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        reference_arm(args, wl)
        return
    gpu_arm(args, wl)


if __name__ == "__main__":
    main()
