"""Config-3 sampled-interval golden vectors (TEST INFRASTRUCTURE, SURVEY §8c "Config-3
parity": a full reference run is infeasible, F7).

Full waveform-relaxation solves (the reference stop logic, allatonce.py:245-271, to its
own stop; cap 600 sweeps) by the CPU oracle's batched restatement
(oracle/wr_batch.py, pinned to the reference's per-interval solve in
tests/test_oracle_pins.py) on sampled (iteration, interval) inputs of a config-3 parareal
run:

* it1: iteration 1, intervals 0, 1, 64, 127 (inputs: the initial coarse sweep);
* k2:  iteration 2, intervals 2, 63;
* k8:  iteration 8, intervals 1, 127;

all inputs taken from the GPU run recorded by tools/cfg3_wr_probe.py
(gpurun_out/cfg3_wr_probe.npz); the iteration-1 inputs are also checked against the
oracle's own coarse sweep.  Records per sample the input, the final state, the sweep
count, the stop reason and the residual history.  ~25 min on 8 cores (26.8 GB of complex
inverses, formed one mode at a time).

Output: tests/golden/cfg3_sample.npz.
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pe_oracle as po  # noqa: E402
from oracle.wr_batch import BatchWR  # noqa: E402
from paper_2411_09244_b200.sysdata import load_system  # noqa: E402

MAX_ITER = 600
PICK = {"it1": (0, [0, 1, 64, 127]), "k2": (1, [2, 63]), "k8": (7, [1, 127])}


def main():
    blocks, f1, f2, meta = load_system(os.path.join(ROOT, "data", "cfg3"))
    s = po.OSystem(*(blocks[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")), f1, f2)
    probe = np.load(os.path.join(ROOT, "gpurun_out", "cfg3_wr_probe.npz"))
    sample = list(probe["sample"])
    hist = probe["hist_sample"]  # (K+1, len(sample), d): history rows of the GPU run
    N, J, T, alpha = 128, 100, 2.0, 0.1
    t0 = time.time()
    # the oracle's own coarse sweep vs the GPU's iteration-1 inputs
    sp = po.OracleSplit(s)
    x = np.zeros(s.d1 + s.d2)
    co = {0: x}
    for n in range(1, max(PICK["it1"][1]) + 1):
        x = sp.coarse_step(x, T / N)
        co[n] = x
    dev = max(np.linalg.norm(co[n] - hist[0, sample.index(n)]) /
              max(np.linalg.norm(co[n]), 1e-300) for n in PICK["it1"][1])
    print(f"coarse sweep: GPU vs oracle max rel L2 {dev:.2e} ({time.time() - t0:.0f} s)", flush=True)
    X, tags = [], []
    for key, (k, ns) in PICK.items():
        for n in ns:
            X.append(hist[k, sample.index(n)])
            tags.append((key, n))
    wr = BatchWR(s, J, T / N, alpha, tol=1e-12, max_iter=MAX_ITER, verbose=True)
    print(f"inverses done ({time.time() - t0:.0f} s)", flush=True)
    res = wr.solve(np.array(X), verbose=True)
    out = {"sample": np.array(sample), "max_iter": np.array(MAX_ITER),
           "coarse_dev": np.array(dev)}
    for key in PICK:
        idx = [i for i, t in enumerate(tags) if t[0] == key]
        r = [res[i] for i in idx]
        mx = max(len(q["residuals"]) for q in r)
        out[f"{key}_n"] = np.array([tags[i][1] for i in idx])
        out[f"{key}_x"] = np.array([X[i] for i in idx])
        out[f"{key}_final"] = np.array([np.concatenate([q["U"][-1], q["W"][-1]]) for q in r])
        out[f"{key}_sweeps"] = np.array([q["iterations"] for q in r])
        out[f"{key}_reasons"] = np.array([q["stop_reason"] for q in r])
        rh = np.full((len(r), mx), np.nan)
        for j, q in enumerate(r):
            rh[j, : len(q["residuals"])] = q["residuals"]
        out[f"{key}_resid"] = rh
    out["oracle_sweeps"] = np.array([q["iterations"] for q in res])
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cfg3_sample.npz"), **out)
    print("sweeps", out["oracle_sweeps"].tolist(), "reasons",
          [q["stop_reason"] for q in res], f"({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
