"""Config-2 all-at-once parareal on the GPU vs the reference's run: per (iteration,
interval) WR sweep count, stop reason and the sweep at which the two residual histories
first differ by more than 1e-3 (relative), with both residuals there.

Writes gpurun_out/wr_stop_cfg2.json (summary + every mismatching pair) and prints the
summary.  Reference data: tests/golden/run_cfg2_aao.npz, run_cfg2_aao_wr.npz
(oracle/make_golden.py cfg2).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_09244_b200 as P  # noqa: E402

REASONS = ("tol", "diverged", "floor", "max_iter")
z = np.load(os.path.join(ROOT, "tests", "golden", "sys_cfg2.npz"))
g = np.load(os.path.join(ROOT, "tests", "golden", "run_cfg2_aao.npz"))
gw = np.load(os.path.join(ROOT, "tests", "golden", "run_cfg2_aao_wr.npz"))
s = P.CoarseSystem(*(z[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")))
ld = P.ConstantLoads(z["f1"], z["f2"])
cfg = P.ParerealConfig(time_grid=P.TimeGrid(1.0, 64, 64), alpha=0.1, epsilon=1e-8, k_max=64,
                       fine_kind="all-at-once", fine_tol=1e-12, stop_rule="relative")
props = P.SplitPropagators(s, ld)
run = P.run_parareal(cfg, props, P.build_fine_propagator(cfg, props, ld),
                     P.SplitState.fresh(np.zeros(s.d1), np.zeros(s.d2)))
h, r = np.array(run.history), g["history"]
rel = float((np.linalg.norm(h - r, axis=-1) / np.maximum(np.linalg.norm(r, axis=-1), 1e-300)).max())
pairs, same = [], 0
worst_excess = -1.0  # max over sweeps of |r_gpu - r_ref| - 1e-3 r_ref (the test allows 1e-11)
cnt = {}
for k, sw in enumerate(run.fine_info):
    for n, info in enumerate(sw):
        ref_it = int(gw["wr_iterations"][k, n])
        ref_reason = REASONS[int(gw["wr_reasons"][k, n])]
        rr = gw["wr_residuals"][k, n, :ref_it]
        rg = np.array(info["residuals"])
        m = min(len(rr), len(rg))
        dev = np.nonzero(np.abs(rg[:m] - rr[:m]) > 1e-3 * rr[:m])[0]
        worst_excess = max(worst_excess, float(np.max(np.abs(rg[:m] - rr[:m]) - 1e-3 * rr[:m])))
        first = int(dev[0]) if dev.size else None
        key = f"{ref_reason}->{info['stop_reason']}"
        cnt[key] = cnt.get(key, 0) + 1
        if info["iterations"] == ref_it and info["stop_reason"] == ref_reason:
            same += 1
            continue
        pairs.append(dict(k=k + 1, n=n, gpu_sweeps=info["iterations"],
                          gpu_reason=info["stop_reason"], ref_sweeps=ref_it,
                          ref_reason=ref_reason, first_dev_sweep=None if first is None else first + 1,
                          ref_resid_at_dev=None if first is None else float(rr[first]),
                          gpu_resid_at_dev=None if first is None else float(rg[first]),
                          ref_final_resid=float(rr[-1]), gpu_final_resid=float(rg[-1])))
devs = [p["ref_resid_at_dev"] for p in pairs if p["ref_resid_at_dev"] is not None]
summary = dict(parareal_iterations=run.iterations, reference_iterations=int(g["iterations"]),
               max_history_rel_l2=rel, pairs=len(pairs) + same, identical=same,
               reason_transitions=cnt,
               max_ref_resid_at_first_deviation=max(devs) if devs else None,
               max_abs_excess_over_1e3_rel=worst_excess,
               tol=1e-12, floor_band=1e-9,
               gpu_sweeps_mean=float(np.mean([i["iterations"] for sw in run.fine_info for i in sw])),
               ref_sweeps_mean=float(gw["wr_iterations"].mean()))
print(json.dumps(summary, indent=1))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "wr_stop_cfg2.json"), "w") as f:
    json.dump(dict(summary=summary, mismatches=pairs), f, indent=1)
