"""World-size-2 gloo test of the interval-sharded parareal driver (CPU only).

`paper_2411_09244_b200.sharded.run_parareal_sharded` shards the fine sweep by intervals
and all-gathers the fine endpoints once per iteration; the coarse correction is
replicated.  Here the device operations are a CPU stand-in built on the oracle (the same
role libpe plays on the GPU box), so the test checks the host logic: interval ranges,
padding of uneven shards, the all-gather order, the replicated correction and the stop
rule.  The sharded history must equal the single-process history bitwise and the
oracle's own parareal driver.
"""

import os
import socket

import numpy as np
import pytest

from oracle import pe_oracle as po
from tests.conftest import GOLDEN


class OracleOps:
    """CPU stand-in for LibpeShardOps: oracle fine propagators and the reference correction
    `x_{n+1} = F_n + (G(x_n^new) - G_old_n)` (parareal.py:198-215)."""

    def __init__(self, s, T, N, J, kind, alpha=0.1, fine_tol=1e-12):
        import torch

        self.torch = torch
        self.s, self.dt, self.J, self.kind = s, T / N, J, kind
        self.sp = po.OracleSplit(s)
        self.wr = po.OracleWR(s, J, T / N, alpha, tol=fine_tol, max_iter=400)

    def to_dev(self, x):
        return self.torch.as_tensor(np.array(x, dtype=np.float64))

    def fine(self, X):
        d1 = self.s.d1
        out, sw = [], []
        for x in X[0].numpy():
            if self.kind == "sequential":
                U, W = self.sp.fine_interval(x[:d1], x[d1:], self.dt, self.J)
                out.append(np.concatenate([U[-1], W[-1]]))
            else:
                r = self.wr.solve(x[:d1], x[d1:])
                out.append(np.concatenate([r["U"][-1], r["W"][-1]]))
                sw.append(r["iterations"])
        Y = self.to_dev(np.array(out)[None])
        return Y, (self.torch.as_tensor(np.array(sw, dtype=np.int32)) if sw else None)

    def coarse_correct(self, N, X_old, F_hat, G_cache, X_new, diff):
        xo = X_old[0].numpy().copy()
        xn = xo.copy()
        G = G_cache[0].numpy()
        for n in range(N):
            g = self.sp.coarse_step(xn[n], self.dt)
            xn[n + 1] = g if F_hat is None else F_hat[0, n].numpy() + (g - G[n])
            G[n] = g
        X_new[0] = self.to_dev(xn)
        G_cache[0] = self.to_dev(G)
        if diff is not None:
            diff[0, 0] = float(np.linalg.norm(xn[1:] - xo[1:], axis=1).max())
            diff[0, 1] = float(np.linalg.norm(xn[1:], axis=1).max())


def _system():
    z = np.load(os.path.join(GOLDEN, "sys_cfg0.npz"))
    return po.OSystem.from_arrays(z)


def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def _worker(rank, world, port, out_dir, kind, N):
    import torch.distributed as dist

    from paper_2411_09244_b200.sharded import run_parareal_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = _system()
    ops = OracleOps(s, 1.0, N, 10, kind)
    r = run_parareal_sharded(N, np.zeros(s.d1 + s.d2), ops, k_max=N, epsilon=1e-8,
                             rule="relative")
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), history=r["history"], diffs=r["diffs"],
             iterations=r["iterations"], sweeps=r["wr_sweeps"], lo=r["intervals"][0],
             hi=r["intervals"][1])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,N", [("sequential", 10), ("all-at-once", 7)])
def test_two_rank_interval_sharding_equals_single_process(tmp_path, kind, N):
    import torch.multiprocessing as mp

    from paper_2411_09244_b200.sharded import run_parareal_sharded

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), kind, N), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"rank{r}.npz") for r in (0, 1))
    # uneven shards when N is odd; contiguous and covering
    assert (int(r0["lo"]), int(r0["hi"]), int(r1["lo"]), int(r1["hi"])) == (0, (N + 1) // 2, (N + 1) // 2, N)
    # the replicated correction gives every rank the same history, bitwise
    assert np.array_equal(r0["history"], r1["history"])
    s = _system()
    single = run_parareal_sharded(N, np.zeros(s.d1 + s.d2), OracleOps(s, 1.0, N, 10, kind),
                                  k_max=N, epsilon=1e-8, rule="relative")
    assert int(r0["iterations"]) == single["iterations"]
    assert np.array_equal(r0["history"], single["history"])
    assert np.array_equal(r0["diffs"], single["diffs"])
    if kind == "all-at-once":
        assert np.array_equal(r0["sweeps"], single["wr_sweeps"])
    # and the oracle's own driver (parareal.py:160-236 restated)
    ref = po.run_parareal(s, np.zeros(s.d1 + s.d2), 1.0, N, 10, kind=kind, alpha=0.1,
                          epsilon=1e-8, k_max=N, stop="relative", fine_tol=1e-12)
    assert ref["iterations"] == single["iterations"]
    np.testing.assert_allclose(single["history"], np.array(ref["history"]), rtol=0, atol=1e-12)


def test_sharded_driver_rejects_unknown_rule():
    from paper_2411_09244_b200.sharded import run_parareal_sharded

    s = _system()
    with pytest.raises(ValueError):
        run_parareal_sharded(4, np.zeros(s.d1 + s.d2), OracleOps(s, 1.0, 4, 10, "sequential"),
                             k_max=1, epsilon=0.0, rule="bogus")


def test_bench_two_rank_dry_run_reports_the_job(tmp_path):
    """`bench.py --gpus 2` re-executes itself under torchrun (one process per device), shards
    the intervals, all-gathers the fine endpoints once per iteration and prints ONE line from
    rank 0 with n_gpus 2 and the strong-scaling tag -- here on CPU under gloo with the oracle
    stand-in context (PE_BENCH_BACKEND), so only the multi-process logic is exercised."""
    import json
    import subprocess
    import sys

    from tests.conftest import ROOT

    env = dict(os.environ, PE_BENCH_BACKEND="tests.bench_cpu_backend:CpuBackend",
               PYTHONPATH=ROOT, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--workload", "cfg0-seq", "--steps", "2", "--warmup", "3"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["steps"] == 2
    assert d["parallelism"].startswith("intervals sharded over 2 ranks")
    assert d["config"]["workload"] == "cfg0-seq" and d["value"] > 0
    assert d["e2e"]["iterations"] >= 1
