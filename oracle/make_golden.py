"""Generate golden fixtures by running the UNMODIFIED reference in the build container.

TEST INFRASTRUCTURE.  Needs `/root/reference/pkg/src` (read-only import; the reference
is never copied).  Writes `tests/golden/*.npz`; those small fixtures travel to the GPU
box, the reference does not.

What it records:
  * `sys_<cfg>.npz`: the reduced `CoarseSystem` blocks and loads built by the
    reference's own offline CEM code (`build_cem_basis` per block in ascending
    order, columns [:n_dom] -> Psi1, [n_dom:] -> Psi2, `project_coarse`,
    `Psi^T b`), after the diffusion-time rescaling A <- c A with
    c = 0.4 * dt_max * N / T (`SplitPropagators.stability_max_step`).
  * `run_<cfg>.npz`: `run_parareal` history / max_diffs / iterations under the
    relative 1e-8 stop rule (the reference's `check_stop` monkeypatched, F5),
    the fine outputs F(x_n^k) captured around `fine.propagate`, and the WR sweep
    counts / stop reasons / residual histories per (k, n).
  * `units.npz`: reference outputs of the hot-path functions on hand-built
    systems (split_step, coarse_step, fine_interval, build_rhs, WR solve,
    parareal runs of both kinds, degenerate d1=0 / d2=0 systems).

Usage:  python oracle/make_golden.py [cfg0 cfg1 cfg2 units channel ...]
"""

from __future__ import annotations

import json
import os
import sys
import time

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

import paradiff.parareal as pp  # noqa: E402
from paradiff.allatonce import WaveformRelaxation, build_rhs, wr_fine_solve  # noqa: E402
from paradiff.fem import (Channel, SourceSpec, assemble_fine, build_fine_grid,  # noqa: E402
                          generate_field)
from paradiff.msbasis import (CoarseSystem, build_cem_basis,  # noqa: E402
                              build_coarse_partition, project_coarse, subspace_angle)
from paradiff.parareal import ParerealConfig, build_fine_propagator, run_parareal  # noqa: E402
from paradiff.stepping import (ConstantLoads, SplitPropagators, SplitState,  # noqa: E402
                               TimeGrid)

from oracle.configs import (CONFIGS, FINE_TOL, R_STABILITY, STOP_REL_EPS,  # noqa: E402
                            corner_load, gaussian_cell_values, rectangles)

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")
BLOCKS = ("M11", "A11", "M12", "A12", "M22", "A22")
REASON_CODE = {"tol": 0, "diverged": 1, "floor": 2, "max_iter": 3}


def build_system(name, member=0):
    """Reference offline CEM build + F2 rescaling.  Returns (CoarseSystem, f1, f2, meta)."""
    c = CONFIGS[name]
    rects, contrast, src = rectangles(name, member)
    t0 = time.time()
    grid = build_fine_grid(c["nx"])
    fld = generate_field(grid, 1.0, contrast, [Channel(*r) for r in rects])
    ops = assemble_fine(grid, fld)
    part = build_coarse_partition(grid, c["nb"], c["layers"])
    cache = {}
    c1, c2 = [], []
    nd = c["n_dom"]
    for b in range(part.n_blocks):
        bb = build_cem_basis(part, ops, fld, b, nd + c["n_comp"], aux_cache=cache)
        c1.append(bb.columns[:, :nd])
        c2.append(bb.columns[:, nd:])
    psi1 = sp.csc_matrix(np.hstack(c1))
    psi2 = sp.csc_matrix(np.hstack(c2))
    system = project_coarse(psi1, psi2, ops)
    if src == "constant":
        b = ops.load(SourceSpec("constant", 1.0))
    else:
        _, x, y, sig = src
        b = corner_load(c["nx"], gaussian_cell_values(c["nx"], x, y, sig))
    f1 = np.asarray(psi1.T @ b)
    f2 = np.asarray(psi2.T @ b)
    build_s = time.time() - t0
    bound = SplitPropagators(system, ConstantLoads(f1, f2)).stability_max_step()
    scale = R_STABILITY * bound * c["N"] / c["T"]
    scaled = CoarseSystem(M11=system.M11, A11=scale * system.A11, M12=system.M12,
                          A12=scale * system.A12, M22=system.M22, A22=scale * system.A22)
    new_bound = SplitPropagators(scaled, ConstantLoads(f1, f2)).stability_max_step()
    meta = dict(name=name, member=member, contrast=contrast, kappa_scale=scale,
                bound_before=bound, bound_after=new_bound,
                dt_over_bound=(c["T"] / c["N"]) / new_bound,
                gamma=subspace_angle(scaled), build_seconds=build_s,
                d1=scaled.d1, d2=scaled.d2, n_rects=len(rects))
    return scaled, f1, f2, meta


def save_system(path, system, f1, f2, meta):
    np.savez_compressed(path, f1=f1, f2=f2, meta=json.dumps(meta),
                        **{k: getattr(system, k) for k in BLOCKS})


def load_system(path):
    z = np.load(path)
    system = CoarseSystem(**{k: z[k] for k in BLOCKS})
    return system, z["f1"], z["f2"], json.loads(str(z["meta"]))


def _relative_check(prev, new, epsilon):
    num = np.linalg.norm(new[1:] - prev[1:], axis=1).max()
    den = np.linalg.norm(new[1:], axis=1).max()
    rel = float(num / den) if den > 0 else float(num)
    return rel, rel < epsilon


def reference_run(system, f1, f2, T, N, J, kind, alpha, *, epsilon, k_max, stop,
                  fine_tol, fine_max_iter=400, workers=1, x0=None):
    """Run the unmodified reference parareal; record F outputs around propagate."""
    loads = ConstantLoads(f1, f2)
    props = SplitPropagators(system, loads)
    cfg = ParerealConfig(time_grid=TimeGrid(T, N, J), alpha=alpha, epsilon=epsilon,
                         k_max=k_max, fine_kind=kind, workers=workers,
                         fine_tol=fine_tol, fine_max_iter=fine_max_iter)
    fine = build_fine_propagator(cfg, props, loads)
    captured = {}
    inner = fine.propagate

    def recording(state):
        out, info = inner(state)
        captured[(round(state.t, 12), state.stacked().tobytes())] = out.stacked()
        return out, info

    fine.propagate = recording
    if x0 is None:
        initial = SplitState.fresh(np.zeros(system.d1), np.zeros(system.d2))
    else:
        initial = SplitState.fresh(x0[: system.d1], x0[system.d1:])
    saved = pp.check_stop
    if stop == "relative":
        pp.check_stop = _relative_check
    try:
        t0 = time.time()
        run = run_parareal(cfg, props, fine, initial)
        secs = time.time() - t0
    finally:
        pp.check_stop = saved
    hist = np.array(run.history)
    K = run.iterations
    # F(x_n^{k-1}) for k = 1..K: re-key by the input state rows of history[k-1]
    dt = T / N
    fhat = np.zeros((K, N, system.d1 + system.d2))
    for k in range(K):
        for n in range(N):
            key = (round(n * dt, 12), hist[k][n].tobytes())
            fhat[k, n] = captured[key]
    out = dict(history=hist, max_diffs=np.array(run.max_diffs), iterations=K,
               converged=run.converged, fhat=fhat, seconds=secs,
               fine_seconds=np.array(run.fine_seconds),
               coarse_seconds=np.array(run.coarse_seconds))
    if kind == "all-at-once":
        it = np.array([[info["iterations"] for info in sweep] for sweep in run.fine_info])
        rc = np.array([[REASON_CODE[info["stop_reason"]] for info in sweep]
                       for sweep in run.fine_info])
        mx = int(it.max())
        res = np.full((K, N, mx), np.nan)
        for k, sweep in enumerate(run.fine_info):
            for n, info in enumerate(sweep):
                res[k, n, : len(info["residuals"])] = info["residuals"]
        out.update(wr_iterations=it, wr_reasons=rc, wr_residuals=res)
    return out


def make_config(name, workers=1):
    c = CONFIGS[name]
    sys_path = os.path.join(OUT, f"sys_{'cfg0' if name == 'cfg1' else name}.npz")
    if os.path.exists(sys_path):
        system, f1, f2, meta = load_system(sys_path)
    else:
        system, f1, f2, meta = build_system(name)
        save_system(sys_path, system, f1, f2, meta)
    print(name, json.dumps(meta))
    kinds = ["sequential", "all-at-once"] if name == "cfg2" else [c["kind"]]
    for kind in kinds:
        r = reference_run(system, f1, f2, c["T"], c["N"], c["J"], kind, c["alpha"],
                          epsilon=STOP_REL_EPS, k_max=c["N"], stop="relative",
                          fine_tol=FINE_TOL, workers=workers)
        tag = f"{name}_{'seq' if kind == 'sequential' else 'aao'}"
        print(tag, "iterations", r["iterations"], "converged", r["converged"],
              "seconds", round(r["seconds"], 2), "max_diffs", r["max_diffs"])
        if "wr_iterations" in r:
            print("   wr sweeps", r["wr_iterations"].min(), r["wr_iterations"].max())
        if c["N"] >= 64:  # keep committed fixtures small: history is the parity target
            r.pop("fhat", None)
            res = r.pop("wr_residuals", None)
            if res is not None:  # per-(k, n) WR residual histories: the stop-logic comparison
                np.savez_compressed(os.path.join(OUT, f"run_{tag}_wr.npz"),
                                    wr_iterations=r["wr_iterations"],
                                    wr_reasons=r["wr_reasons"], wr_residuals=res)
        np.savez_compressed(os.path.join(OUT, f"run_{tag}.npz"), kind=kind,
                            **{k: v for k, v in r.items()})


# ------------------------------------------------------------------ hand systems

def tiny_system():
    """1+1, every block nonzero (test_stepping.py:16-26)."""
    return CoarseSystem(M11=np.array([[2.0]]), A11=np.array([[3.0]]),
                        M12=np.array([[0.5]]), A12=np.array([[0.4]]),
                        M22=np.array([[1.5]]), A22=np.array([[0.7]]))


def random_system(d1, d2, seed, a_scale=1.0, m_cond=1.0):
    """Seeded SPD-mass / SPD-stiffness coupled system (Galerkin-like Gram blocks)."""
    rng = np.random.default_rng(seed)
    n = d1 + d2
    q = rng.standard_normal((3 * n, n))
    mass = q.T @ q / (3 * n) + m_cond * 0.1 * np.eye(n)
    r = rng.standard_normal((3 * n, n))
    stiff = a_scale * (r.T @ r / (3 * n) + 0.05 * np.eye(n))
    mass = (mass + mass.T) / 2
    stiff = (stiff + stiff.T) / 2
    return CoarseSystem(M11=mass[:d1, :d1], A11=stiff[:d1, :d1], M12=mass[:d1, d1:],
                        A12=stiff[:d1, d1:], M22=mass[d1:, d1:], A22=stiff[d1:, d1:])


def make_units():
    out = {}
    # split_step on the tiny system (test_stepping.py:117-147)
    sysb = tiny_system()
    loads = ConstantLoads(np.array([0.3]), np.array([-0.2]))
    props = SplitPropagators(sysb, loads)
    st = SplitState(u=np.array([1.0]), w=np.array([2.0]), u_prev=np.array([0.8]),
                    w_prev=np.array([1.5]), t=0.0)
    o = props.split_step(st, 0.01)
    out["tiny_split"] = np.concatenate([o.u, o.w])
    out["tiny_coarse"] = props.coarse_step(SplitState.fresh(np.array([0.7]), np.array([-0.3])),
                                           0.02).stacked()
    tr = props.fine_interval(SplitState.fresh(np.array([1.0]), np.array([2.0])), 0.05, 7)
    out["tiny_fine_U"], out["tiny_fine_W"] = tr.U, tr.W
    # build_rhs hand values (test_allatonce.py:100-124)
    out["rhs_hand"] = build_rhs(sysb, np.array([[0.2], [0.2]]), np.array([1.0]),
                                np.array([2.0]), np.array([2.0]), np.array([[2.5], [3.0]]),
                                np.array([0.9]), 0.1, 0.3)
    # random coupled system: every hot-path function
    rs = random_system(5, 4, seed=7, a_scale=3.0)
    rng = np.random.default_rng(11)
    f1, f2 = rng.standard_normal(5), rng.standard_normal(4)
    for k in ("M11", "A11", "M12", "A12", "M22", "A22"):
        out[f"rand_{k}"] = getattr(rs, k)
    out["rand_f1"], out["rand_f2"] = f1, f2
    rl = ConstantLoads(f1, f2)
    rp = SplitPropagators(rs, rl)
    x0 = rng.standard_normal(9)
    out["rand_x0"] = x0
    st = SplitState(u=x0[:5], w=x0[5:], u_prev=x0[:5] * 0.9, w_prev=x0[5:] * 1.1, t=0.0)
    o = rp.split_step(st, 1e-3)
    out["rand_split"] = np.concatenate([o.u, o.w])
    out["rand_coarse"] = rp.coarse_step(SplitState.fresh(x0[:5], x0[5:]), 0.04).stacked()
    tr = rp.fine_interval(SplitState.fresh(x0[:5], x0[5:]), 0.04, 16)
    out["rand_fine_U"], out["rand_fine_W"] = tr.U, tr.W
    wr = wr_fine_solve(rs, SplitState.fresh(x0[:5], x0[5:]), 0.04, 16, 0.3, rl,
                       tol=1e-13, max_iter=400)
    out["rand_wr_U"], out["rand_wr_W"] = wr.trajectory.U, wr.trajectory.W
    out["rand_wr_res"] = np.array(wr.residuals)
    out["rand_wr_meta"] = np.array([wr.iterations, REASON_CODE[wr.stop_reason]])
    for kind, tag in (("sequential", "seq"), ("all-at-once", "aao")):
        r = reference_run(rs, f1, f2, 0.32, 8, 16, kind, 0.3, epsilon=1e-10, k_max=8,
                          stop="absolute", fine_tol=1e-13, x0=x0)
        out[f"rand_par_{tag}_hist"] = r["history"]
        out[f"rand_par_{tag}_diffs"] = r["max_diffs"]
        out[f"rand_par_{tag}_iters"] = np.array(r["iterations"])
        # forced k = N: exactness vs sequential composition
        r = reference_run(rs, f1, f2, 0.32, 8, 16, kind, 0.3, epsilon=0.0, k_max=8,
                          stop="absolute", fine_tol=1e-13, x0=x0)
        out[f"rand_exact_{tag}_hist"] = r["history"]
    # synthetic low-gamma system (test_allatonce.py:179-217)
    g = CoarseSystem(M11=np.eye(2), A11=np.diag([200.0, 100.0]), M12=np.diag([0.3, 0.1]),
                     A12=np.zeros((2, 2)), M22=np.eye(2), A22=np.diag([0.5, 0.5]))
    gl = ConstantLoads(np.array([1.0, 1.0]), np.array([1.0, -1.0]))
    res = wr_fine_solve(g, SplitState.fresh(np.zeros(2), np.zeros(2)), 0.01, 8, 0.1, gl,
                        tol=1e-13, max_iter=200)
    out["lowgamma_res"] = np.array(res.residuals)
    out["lowgamma_U"], out["lowgamma_W"] = res.trajectory.U, res.trajectory.W
    floor = WaveformRelaxation(g, 8, 0.01, 0.1, ConstantLoads(np.array([1.0, 0.0]),
                                                              np.array([0.0, 1.0])),
                               tol=1e-18, max_iter=500).solve(
        SplitState.fresh(np.zeros(2), np.zeros(2)))
    out["floor_meta"] = np.array([floor.iterations, REASON_CODE[floor.stop_reason]])
    out["floor_res"] = np.array(floor.residuals)
    # degenerate spaces: u-only scalar parareal (test_parareal.py:100-114), w-only
    us = CoarseSystem(M11=np.array([[1.0]]), A11=np.array([[6.0]]), M12=np.zeros((1, 0)),
                      A12=np.zeros((1, 0)), M22=np.zeros((0, 0)), A22=np.zeros((0, 0)))
    r = reference_run(us, np.array([2.4]), np.zeros(0), 0.8, 8, 16, "sequential", 0.5,
                      epsilon=1e-15, k_max=50, stop="absolute", fine_tol=None,
                      x0=np.array([1.0]))
    out["uonly_hist"], out["uonly_iters"] = r["history"], np.array(r["iterations"])
    ws = CoarseSystem(M11=np.zeros((0, 0)), A11=np.zeros((0, 0)), M12=np.zeros((0, 1)),
                      A12=np.zeros((0, 1)), M22=np.array([[2.0]]), A22=np.array([[3.0]]))
    for kind, tag in (("sequential", "seq"), ("all-at-once", "aao")):
        r = reference_run(ws, np.zeros(0), np.array([0.6]), 0.4, 5, 4, kind, 0.5,
                          epsilon=1e-15, k_max=5, stop="absolute", fine_tol=1e-13,
                          x0=np.array([1.0]))
        out[f"wonly_{tag}_hist"] = r["history"]
        out[f"wonly_{tag}_iters"] = np.array(r["iterations"])
    np.savez_compressed(os.path.join(OUT, "units.npz"), **out)
    print("units:", sorted(out))


def make_channel():
    """The reference test fixture `channel_pipeline` (conftest.py:7-33) runs."""
    from paradiff.experiment import ExperimentConfig, build_pipeline
    cfg = ExperimentConfig(nx=20, blocks=4, layers=2, contrast=1e4, channels=[(1, 19, 8, 10)],
                           source_kind="box", source_amplitude=1.0,
                           source_region=(0.3, 0.7, 0.3, 0.7), n_values=(10,), alpha=0.5,
                           compute_reference=False, export_solution=False)
    pipe = build_pipeline(cfg)
    s = pipe.space.system
    out = {k: getattr(s, k) for k in BLOCKS}
    out["f1"], out["f2"] = pipe.loads.f1, pipe.loads.f2
    for kind, tag, n, J in (("sequential", "seq", 6, 4), ("all-at-once", "aao", 5, 6)):
        r = reference_run(s, pipe.loads.f1, pipe.loads.f2, 0.005, n, J, kind, 0.5,
                          epsilon=0.0, k_max=n, stop="absolute", fine_tol=1e-13)
        out[f"{tag}_hist"] = r["history"]
        out[f"{tag}_fhat"] = r["fhat"]
        if "wr_iterations" in r:
            out[f"{tag}_wr_iters"] = r["wr_iterations"]
    r = reference_run(s, pipe.loads.f1, pipe.loads.f2, 0.005, 10, 10, "all-at-once", 0.5,
                      epsilon=1e-14, k_max=100, stop="absolute", fine_tol=1e-13)
    out["conv_hist"], out["conv_diffs"] = r["history"], r["max_diffs"]
    out["conv_iters"] = np.array(r["iterations"])
    out["conv_wr_iters"] = r["wr_iterations"]
    np.savez_compressed(os.path.join(OUT, "channel.npz"), **out)
    print("channel d1,d2", s.d1, s.d2, "conv iterations", r["iterations"])


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    targets = sys.argv[1:] or ["units", "channel", "cfg0", "cfg1"]
    workers = int(os.environ.get("GOLDEN_WORKERS", "1"))
    for t in targets:
        if t == "units":
            make_units()
        elif t == "channel":
            make_channel()
        else:
            make_config(t, workers=workers)
