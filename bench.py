"""Benchmark: reduced-DOF x fine-steps per second per parareal iteration (FP64).

A "step" is one parareal iteration of the hot path (parareal.py:188-215): the fine
sweep over all N coarse intervals (the all-at-once waveform-relaxation solver by
default) plus the fused coarse sweep / correction / convergence norm, on one batch of
seeded inputs already resident in HBM.  units/step = E * (d1+d2) * N * J.

    python bench.py [--gpus N --steps K --warmup W] [--workload cfg2-aao] [--impl reference]

Default workload: BASELINE config 2 (100x100 mesh, CEM 3+3 -> d = 300+300, N = J = 64,
kappa inclusions at 1e6, all-at-once fine solver, alpha = 0.1), with the reduced
operators built by the reference's own offline CEM code (tests/golden/sys_cfg2.npz,
written by oracle/make_golden.py).  Under torchrun every rank runs an independent
replica (ensemble member): the units shard with no data-path collective (weak scaling).
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
GOLDEN = os.path.join(ROOT, "tests", "golden")
METRIC = "reduced-DOF·fine-steps/s per parareal iteration (FP64); % of roofline"
UNIT = "reduced-DOF*fine-steps/s"

WORKLOADS = {
    "cfg2-aao": dict(sys="sys_cfg2.npz", T=1.0, N=64, J=64, kind="all-at-once", alpha=0.1),
    "cfg2-seq": dict(sys="sys_cfg2.npz", T=1.0, N=64, J=64, kind="sequential", alpha=0.1),
    "cfg0-seq": dict(sys="sys_cfg0.npz", T=1.0, N=10, J=10, kind="sequential", alpha=0.1),
    "cfg1-aao": dict(sys="sys_cfg0.npz", T=1.0, N=10, J=10, kind="all-at-once", alpha=0.1),
    # config 3 (d = 4096+4096, N = 128, J = 100): operators from oracle/build_cfg3.py
    # (0.8 GB, not committed; data/ travels to the GPU box with the repo snapshot)
    "cfg3-aao": dict(sys="../../data/sys_cfg3.npz", T=2.0, N=128, J=100, kind="all-at-once",
                     alpha=0.1),
    # config 4: 64 seeded members (own contrast 10^U(2,8), own kappa rescaling), one batch;
    # operators from oracle/build_cfg4.py (data/, travels with the repo snapshot)
    "cfg4-seq": dict(members="../../data/cfg4_members.npz", T=1.0, N=32, J=32,
                     kind="sequential", alpha=0.1),
}
FINE_TOL, MAX_ITER = 1e-12, 400


BLOCKS = ("M11", "A11", "M12", "A12", "M22", "A22")


def load_system(name):
    z = np.load(os.path.join(GOLDEN, name))
    blocks = {k: np.ascontiguousarray(z[k]) for k in BLOCKS}
    return blocks, z["f1"], z["f2"], json.loads(str(z["meta"]))


def load_workload(wl, n_replicas=1):
    """[(blocks, f1, f2)] per member and a representative meta dict."""
    if "members" in wl:
        z = np.load(os.path.join(GOLDEN, wl["members"]))
        metas = json.loads(str(z["meta"]))
        mem = [({k: np.ascontiguousarray(z[k][m]) for k in BLOCKS}, z["f1"][m], z["f2"][m])
               for m in range(z["f1"].shape[0])]
        meta = dict(metas[0])
        meta["members"] = len(mem)
        meta["contrast_range"] = [min(x["contrast"] for x in metas),
                                  max(x["contrast"] for x in metas)]
        meta["kappa_scale"] = [x["kappa_scale"] for x in metas]
        return mem, meta
    blocks, f1, f2, meta = load_system(wl["sys"])
    return [(blocks, f1, f2)] * n_replicas, meta


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.result = None
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


# ---------------------------------------------------------------------- CPU arms

def cpu_sample_large(wl, s, sweeps_hint, cores):
    """Config 3 (d1 = d2 = 4096, J = 100): a full reference iteration needs 26.8 GB of
    complex inverses and hours, so time the reference's per-sweep operations
    on a bounded subset and extrapolate: the `einsum("kij,kj->ki")` shifted apply on 2
    modes per thread of a `cores`-thread pool (the dominant, memory-bound term), plus
    build_rhs + both FFTs + the w-sweep of one interval once, times J modes, the sweep
    count the GPU measured on the same iteration, and N intervals."""
    from concurrent.futures import ThreadPoolExecutor

    from threadpoolctl import threadpool_limits

    from oracle import pe_oracle as po

    N, J, T = wl["N"], wl["J"], wl["T"]
    dt = T / N / J
    d1, d2 = s.d1, s.d2
    lam = po.time_eigenvalues(J, dt, wl["alpha"])
    rng = np.random.default_rng(0)
    with threadpool_limits(cores):
        invs = [np.linalg.inv(lam[k] * s.M11 + s.A11.astype(complex)) for k in (1, 2)]
        m22_inv = np.linalg.inv(s.M22)
        e_mat = np.eye(d2) - dt * m22_inv @ s.A22
    p = (rng.standard_normal((1, d1)) + 1j * rng.standard_normal((1, d1)))
    with threadpool_limits(1):
        def apply(i):
            t0 = time.perf_counter()
            for inv in invs:
                np.einsum("kij,kj->ki", inv[None], p)
            return time.perf_counter() - t0
        with ThreadPoolExecutor(max_workers=cores) as pool:
            times = list(pool.map(apply, range(cores)))
        t_mode_pool = max(times) / (2 * cores)  # seconds per mode-apply, pool aggregate
        u0 = np.zeros(d1)
        w0 = np.zeros(d2)
        W = rng.standard_normal((J, d2)) * 1e-3
        t0 = time.perf_counter()
        rhs = po.build_rhs(s, np.tile(s.f1, (J, 1)), u0, w0, w0, W, u0, dt, wl["alpha"])
        q = po.apply_S(po.apply_S_inverse(rhs, wl["alpha"]), wl["alpha"]).real
        uh = np.vstack([u0, u0, q[:-1]])
        g = dt * (np.tile(s.f2, (J, 1)) - (uh[1:] - uh[:-1]) / dt @ s.M12 - q @ s.A12) @ m22_inv
        w = w0
        for i in range(J):
            w = e_mat @ w + g[i]
        t_rest = time.perf_counter() - t0
    t_sweep = J * t_mode_pool + t_rest / cores
    t_iter = N * sweeps_hint * t_sweep
    return t_iter, dict(cores=cores, extrapolated=True, sample=(
        f"extrapolated: einsum shifted apply timed on 2 modes x {cores} threads "
        f"({t_mode_pool * 1e3:.1f} ms per mode-apply, pool aggregate) + one build_rhs/FFT/"
        f"w-sweep ({t_rest:.2f} s); x J={J} modes x {sweeps_hint:.1f} sweeps (GPU-measured "
        f"mean on the same iteration) x N={N} intervals; setup (26.8 GB inverses) excluded"))


def cpu_sample(wl, blocks, f1, f2, budget_s=20.0, sweeps_hint=None):
    """Time the CPU oracle port (restatement of the reference, same LAPACK calls) on a
    bounded sample of one parareal iteration; returns (seconds_per_iteration, info)."""
    from threadpoolctl import threadpool_limits

    from oracle import pe_oracle as po

    cores = len(os.sched_getaffinity(0))
    s = po.OSystem(*(blocks[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")), f1, f2)
    if s.d1 > 2048:
        return cpu_sample_large(wl, s, sweeps_hint or 200.0, cores)
    N, J, T = wl["N"], wl["J"], wl["T"]
    dt = T / N
    sp = po.OracleSplit(s)
    x = np.zeros(s.d1 + s.d2)
    states = [x]
    t0 = time.perf_counter()
    for _ in range(N):
        states.append(sp.coarse_step(states[-1], dt))
    t_coarse = time.perf_counter() - t0  # one coarse sweep (correction sweep has the same N G-solves)
    from concurrent.futures import ThreadPoolExecutor

    if wl["kind"] == "all-at-once":
        # best of workers in {1, cores} with 1 BLAS thread
        with threadpool_limits(1):
            wr = po.OracleWR(s, J, dt, wl["alpha"], tol=FINE_TOL, max_iter=MAX_ITER)
            n_s, t0 = 0, time.perf_counter()
            while n_s < N:
                v = states[n_s]
                wr.solve(v[: s.d1], v[s.d1:])
                n_s += 1
                if time.perf_counter() - t0 > budget_s / 2:
                    break
            t_serial = (time.perf_counter() - t0) * N / n_s
            sample = states[:min(N, cores)]
            t0 = time.perf_counter()
            with ThreadPoolExecutor(max_workers=cores) as pool:
                res = list(pool.map(lambda v: wr.solve(v[: s.d1], v[s.d1:]), sample))
            t_round = time.perf_counter() - t0
        rounds = math.ceil(N / cores)
        t_par = t_round * rounds
        sweeps = [r["iterations"] for r in res]
        if t_par < t_serial:
            t_iter = t_par + t_coarse
            info = dict(cores=cores, sample=(
                f"WR solves of {len(sample)} intervals (iteration-1 inputs, {min(sweeps)}-"
                f"{max(sweeps)} sweeps) on a {cores}-thread pool, BLAS 1 thread, x{rounds} "
                f"rounds + 1 measured coarse sweep (beat workers=1: {t_serial:.3g} s)"))
        else:
            t_iter = t_serial + t_coarse
            info = dict(cores=1, sample=(
                f"WR solves of {n_s} of {N} intervals serially (workers=1, BLAS 1 thread, "
                f"{min(sweeps)}-{max(sweeps)} sweeps) x N/{n_s} + 1 measured coarse sweep "
                f"(beat the {cores}-thread pool: {t_par:.3g} s)"))
    else:
        with threadpool_limits(1):
            n_s, t0 = 0, time.perf_counter()
            while n_s < N:
                v = states[n_s]
                sp.fine_interval(v[: s.d1], v[s.d1:], dt, J)
                n_s += 1
                if time.perf_counter() - t0 > budget_s:
                    break
            t_f = time.perf_counter() - t0
        t_iter = t_f * N / n_s + t_coarse
        info = dict(cores=1, sample=(f"{n_s} of {N} sequential fine intervals (workers=1, BLAS 1 "
                                     f"thread, the reference's best setting) + 1 coarse sweep"))
    return t_iter, info


def reference_arm(args, wl, units):
    mem, meta = load_workload(wl)
    blocks, f1, f2 = mem[0]
    vals = []
    for i in range(args.warmup + args.steps):
        t_iter, info = cpu_sample(wl, blocks, f1, f2, budget_s=5.0)
        if i >= args.warmup:
            vals.append(units / t_iter)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": units / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded kappa field; reduced operators from the reference's "
                    "offline CEM code)",
            "config": dict(workload=args.workload, d1=meta["d1"], d2=meta["d2"], N=wl["N"],
                           J=wl["J"], E=1, kind=wl["kind"], alpha=wl["alpha"]),
            "cpu_baseline": dict(value=v, unit=UNIT, cores=info["cores"], kind="port",
                                 sample=info["sample"]),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- GPU arm

def gpu_arm(args, wl, units_member):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2411_09244_b200 as P

    mem, meta = load_workload(wl, args.members)
    blocks, f1, f2 = mem[0]
    systems = [P.CoarseSystem(**b) for b, _, _ in mem]
    loads_l = [P.ConstantLoads(a, b) for _, a, b in mem]
    system, loads = systems[0], loads_l[0]
    E = len(mem)
    N, J, T, kind = wl["N"], wl["J"], wl["T"], wl["kind"]
    d = system.d1 + system.d2
    units = units_member * E
    # upload + setup factorisations, timed separately (outside the step)
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    ctx = P.PeContext(systems, loads_l, J, local)
    torch.cuda.synchronize()
    t_upload = time.perf_counter() - t_setup
    ctx.prepare_coarse(T / N)
    if kind == "sequential":
        ctx.prepare_sequential(T / N / J)
    else:
        ctx.prepare_allatonce(T / N / J, wl["alpha"], FINE_TOL, MAX_ITER)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    modal = ctx.modal_level() if kind == "all-at-once" else None

    A = torch.zeros(E, N + 1, d, dtype=torch.float64, device="cuda")
    B = torch.zeros_like(A)
    Gc = torch.zeros(E, N, d, dtype=torch.float64, device="cuda")
    diff = torch.zeros(E, 2, dtype=torch.float64, device="cuda")
    ctx.coarse_correct(N, A, None, Gc, A)  # initial coarse sweep (x_0 = 0, u0 = 0 projection)
    flush = torch.empty(320 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    sweeps_buf = (torch.zeros(E, N, dtype=torch.int32, device="cuda")
                  if kind == "all-at-once" else None)

    shard = args.shard == "intervals"
    if shard:
        # one problem, intervals sharded across ranks (strong scaling): fine on the local
        # slice, one all-gather of the F endpoints, replicated coarse correction
        # (paper_2411_09244_b200/sharded.py)
        from paper_2411_09244_b200.dist import shard_members

        ranges = [shard_members(N, r, world) for r in range(world)]
        mine = ranges[rank]
        m_loc = max(len(r) for r in ranges)
        F_loc = torch.zeros(E, m_loc, d, dtype=torch.float64, device="cuda")
        parts = [torch.empty_like(F_loc) for _ in range(world)]

        def step(x_old, x_new):
            if len(mine):
                Xs = x_old[:, mine.start:mine.stop].contiguous()
                if kind == "sequential":
                    F_loc[:, : len(mine)] = ctx.fine_sequential(Xs)
                else:
                    F_loc[:, : len(mine)] = ctx.fine_allatonce(Xs, record=False)[0]
            if dist:
                dist.all_gather(parts, F_loc)
                F = torch.cat([p[:, : len(r)] for p, r in zip(parts, ranges)], dim=1)
            else:
                F = F_loc[:, :N]
            ctx.coarse_correct(N, x_old, F.contiguous(), Gc, x_new, diff)
    else:
        def step(x_old, x_new):
            ctx.iterate(kind, N, x_old, x_new, Gc, diff, wr_sweeps=sweeps_buf)

    for _ in range(args.warmup):
        step(A, B)
        A, B = B, A
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = ctx.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))  # evict L2 (320 MB > 126 MB) between timed steps
            starts[i].record()
            step(A, B)
            ends[i].record()
            A, B = B, A
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    launches = ctx.launch_count() - launches0
    total_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    value = (1 if shard else world) * units * args.steps / (total_ms / 1e3)

    # roofline pass: one extra instrumented step, every GEMM launch bracketed by events
    ctx.set_profiling(True)
    flush.fill_(0.0)
    step(A, B)
    torch.cuda.synchronize()
    st = ctx.fine_stats()
    ctx.set_profiling(False)
    peak = fp64_peak_tflops(torch)
    achieved = st["gemm_flops"] / (st["gemm_ms"] / 1e3) / 1e12 if st["gemm_ms"] > 0 else 0.0
    gemm_share = st["gemm_ms"] / (total_ms / args.steps)

    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "r01", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.workload, {})
    line = None
    if rank == 0:
        # end to end through the public API: run_parareal with host initial state in and
        # the full history (host numpy) out, K iterations, epsilon = 0 (no early stop)
        cfg = P.ParerealConfig(time_grid=P.TimeGrid(T, N, J), alpha=wl["alpha"], epsilon=0.0,
                               k_max=args.steps, fine_kind=kind, fine_tol=FINE_TOL,
                               fine_max_iter=MAX_ITER)
        warm = P.ParerealConfig(time_grid=cfg.time_grid, alpha=cfg.alpha, epsilon=0.0, k_max=1,
                                fine_kind=kind, fine_tol=FINE_TOL, fine_max_iter=MAX_ITER)
        if shard:
            from paper_2411_09244_b200.sharded import LibpeShardOps, run_parareal_sharded

            ops = LibpeShardOps(ctx, kind)
            run_parareal_sharded(N, np.zeros(d), ops, 1, 0.0)  # warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = run_parareal_sharded(N, np.zeros(d), ops, args.steps, 0.0)
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
            K = res["iterations"]
            path = (f"paper_2411_09244_b200.run_parareal_sharded ({world} ranks, intervals "
                    "sharded, host arrays in/out)")
        elif E == 1:
            props = P.SplitPropagators(system, loads)
            fine = P.build_fine_propagator(cfg, props, loads)
            init = P.SplitState.fresh(np.zeros(system.d1), np.zeros(system.d2))
            P.run_parareal(warm, props, fine, init)  # setup (factorisations) stays out of e2e
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run = P.run_parareal(cfg, props, fine, init)
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
            K = run.iterations
            path = "paper_2411_09244_b200.run_parareal (host arrays in/out, 1 member)"
        else:
            inits = [P.SplitState.fresh(np.zeros(system.d1), np.zeros(system.d2))] * E
            ens = P.ParerealEnsemble(cfg, systems, loads_l)  # setup stays out of e2e
            ens.run(inits)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            runs = ens.run(inits)
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
            K = runs[0].iterations
            path = (f"paper_2411_09244_b200.ParerealEnsemble.run ({E} members, host arrays "
                    "in/out)")
        wr_bytes = K * N * (4 + 4 + 8 * MAX_ITER) if kind == "all-at-once" else 0
        e2e = {"value": units_member * E * K / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": E * d * 8 / K,
               "d2h_bytes_per_step": E * ((K + 1) * (N + 1) * d * 8 + wr_bytes) / K,
               "path": path}
        cpu = None
        if world == 1 and not args.no_cpu:
            hint = float(sweeps_buf.float().mean()) if sweeps_buf is not None else None
            t_iter, info = cpu_sample(wl, blocks, f1, f2, sweeps_hint=hint)
            cpu = dict(value=units_member / t_iter, unit=UNIT, cores=info["cores"], kind="port",
                       sample=info["sample"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded kappa field per BASELINE config; reduced operators built "
                    "by the reference's offline CEM code, " + (wl.get("sys") or wl["members"]) +
                    ")",
            "config": dict(workload=args.workload, d1=system.d1, d2=system.d2, N=N, J=J,
                           E_per_gpu=E, kind=kind, alpha=wl["alpha"], fine_tol=FINE_TOL,
                           parallelism=(f"intervals sharded over {world} ranks, one NCCL "
                                        "all-gather of the F endpoints per iteration" if shard
                                        else f"{world} independent replicas (no collective)"),
                           kappa_scale=meta["kappa_scale"],
                           contrast=meta.get("contrast_range", meta.get("contrast")),
                           l2="L2 flushed (320 MB write) before every timed step",
                           step="one parareal iteration: fine sweep over N intervals + fused "
                                "coarse sweep/correction/norm"),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic.get("dram_bytes_per_launch"),
                         "traffic_kernel": traffic.get("kernel"),
                         "traffic_algorithmic_bytes": traffic.get("algorithmic_bytes_per_launch"),
                         "traffic_source": traffic.get("source"),
                         "kernel": "every FP64 DMMA (m8n8k4) launch of one instrumented step: "
                                   "GEMMs + recurrence / all-SM chains; algorithmic flops "
                                   "(structural zeros and re-associated work not counted)",
                         "gemm_launches": st["launches"], "gemm_ms": st["gemm_ms"],
                         "gemm_flops": st["gemm_flops"], "gemm_share_of_step": gemm_share,
                         "other_kernels_ms": st.get("other_ms", 0.0),
                         "other_share_of_step": st.get("other_ms", 0.0) / (total_ms / args.steps),
                         "peak_source": "cuBLAS DGEMM 8192^3 burst measured in this run "
                                        "(MEASURED_PEAKS.json has no FP64 entry)"},
            "cpu_baseline": cpu,
            "setup": {"upload_s": t_upload, "factorisations_s": t_setup - t_upload,
                      "what": ("pe_create + pe_set_system uploads; G, sequential operator T or the "
                               "all-at-once pencil eigendecompositions (modal level "
                               f"{modal}) on the GPU; excluded from the step")},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.result,
            "wall_s_timed": t_wall,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="libpe", choices=["libpe", "reference"])
    ap.add_argument("--workload", default="cfg2-aao", choices=sorted(WORKLOADS))
    ap.add_argument("--members", type=int, default=1, help="ensemble members per GPU")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "intervals"],
                    help="N > 1: independent replicas (weak scaling, default) or one problem "
                         "with its intervals sharded across the ranks (strong scaling)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if "members" in wl:
        z = np.load(os.path.join(GOLDEN, wl["members"]))
        dd = z["M11"].shape[1] + z["M22"].shape[1]
    else:
        _, _, _, meta = load_system(wl["sys"])
        dd = meta["d1"] + meta["d2"]
    units = dd * wl["N"] * wl["J"]
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        reference_arm(args, wl, units)
        return
    gpu_arm(args, wl, units)


if __name__ == "__main__":
    main()
