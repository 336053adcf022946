"""Interval-sharded parareal over several GPUs.

The fine sweep of one parareal iteration is N independent interval solves
(`parareal.py:191-193`, `util.parallel_map`), so ranks own contiguous interval ranges and
run their fine propagators locally.  The one exchange per iteration is an all-gather of
the N x (d1 + d2) FP64 fine endpoints F(x_n^k); every rank then runs the cheap sequential
coarse sweep / correction / convergence norm (`parareal.py:198-215`) on the full set,
replicated, so no broadcast is needed and every rank holds the same history.

Because libpe's fine propagators are batch invariant (an interval's result does not
depend on which other intervals share the launch, bitwise-tested), the sharded run is
bitwise identical to the single-GPU run for any world size.

One process per GPU, `torch.distributed` for the plumbing: NCCL on the GPU box (device
tensors), gloo in the CPU tests.  The device work goes through a small ops object so the
same driver runs libpe (`LibpeShardOps`) or a CPU stand-in in the tests.
"""

from __future__ import annotations

import time

import numpy as np

from .dist import shard_members


class LibpeShardOps:
    """The three device operations of the driver, on one libpe context (one member)."""

    def __init__(self, ctx, kind: str):
        if kind not in ("sequential", "all-at-once"):
            raise ValueError(f"unknown fine propagator kind {kind!r}")
        self.ctx = ctx
        self.kind = kind

    def to_dev(self, x):
        return self.ctx.to_dev(x)

    def fine(self, X):
        """F on the (1, nc, d) states X -> ((1, nc, d) endpoints, (nc,) WR sweeps or None)."""
        if self.kind == "sequential":
            return self.ctx.fine_sequential(X), None
        Y, sw, _, _ = self.ctx.fine_allatonce(X, record=False)
        return Y, sw

    def coarse_correct(self, N, X_old, F_hat, G_cache, X_new, diff):
        self.ctx.coarse_correct(N, X_old, F_hat, G_cache, X_new, diff)


def run_parareal_sharded(N: int, x0: np.ndarray, ops, k_max: int, epsilon: float,
                         rule: str = "absolute", group=None):
    """Parareal with the fine sweep sharded by intervals across the ranks of `group`.

    x0: initial state (d,).  Returns a dict with the replicated `history` (K+1, N+1, d),
    `diffs` (K,), `iterations`, `converged`, per-iteration `wr_sweeps` (K, N) for the
    all-at-once kind, `fine_seconds` / `exchange_seconds` per iteration.  Stop rules as in
    `pe_parareal_run`: absolute max_n ||dx_n|| or relative (/ max_n ||x_n||), n = 1..N.
    """
    import torch
    import torch.distributed as dist

    if rule not in ("absolute", "relative"):
        raise ValueError(f"unknown stop rule {rule!r}")
    sharded = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if sharded else 0
    world = dist.get_world_size(group) if sharded else 1
    ranges = [shard_members(N, r, world) for r in range(world)]
    mine = ranges[rank]
    m = max(len(r) for r in ranges)
    d = x0.shape[-1]

    X = ops.to_dev(np.zeros((1, N + 1, d)))
    X[0, 0] = ops.to_dev(np.asarray(x0, dtype=np.float64))
    G = ops.to_dev(np.zeros((1, N, d)))
    diff = ops.to_dev(np.zeros((1, 2)))
    ops.coarse_correct(N, X, None, G, X, None)  # initial coarse sweep (parareal.py:150-157)
    history = [X[0].cpu().numpy().copy()]
    diffs, sweeps, fine_s, xchg_s = [], [], [], []
    converged = False
    k = 0
    for k in range(1, k_max + 1):
        t0 = time.perf_counter()
        F_loc = ops.to_dev(np.zeros((1, m, d)))
        sw_loc = ops.to_dev(np.zeros(m)).to(torch.int32)
        if len(mine):
            Xs = X[:, mine.start:mine.stop].contiguous()
            Y, sw = ops.fine(Xs)
            F_loc[:, : len(mine)] = Y
            if sw is not None:
                sw_loc[: len(mine)] = sw.reshape(-1)
        t1 = time.perf_counter()
        if sharded:
            parts = [torch.empty_like(F_loc) for _ in range(world)]
            dist.all_gather(parts, F_loc, group=group)
            sparts = [torch.empty_like(sw_loc) for _ in range(world)]
            dist.all_gather(sparts, sw_loc, group=group)
        else:
            parts, sparts = [F_loc], [sw_loc]
        F_hat = torch.cat([p[:, : len(r)] for p, r in zip(parts, ranges)], dim=1).contiguous()
        sw_all = torch.cat([p[: len(r)] for p, r in zip(sparts, ranges)])
        t2 = time.perf_counter()
        X_new = torch.empty_like(X)
        ops.coarse_correct(N, X, F_hat, G, X_new, diff)
        X = X_new
        dv = diff[0].cpu().numpy()
        v = float(dv[0]) if rule == "absolute" else (float(dv[0] / dv[1]) if dv[1] > 0 else float(dv[0]))
        history.append(X[0].cpu().numpy().copy())
        diffs.append(v)
        sweeps.append(sw_all.cpu().numpy())
        fine_s.append(t1 - t0)
        xchg_s.append(t2 - t1)
        if v < epsilon:
            converged = True
            break
    return dict(history=np.array(history), diffs=np.array(diffs), iterations=k,
                converged=converged, wr_sweeps=np.array(sweeps), fine_seconds=fine_s,
                exchange_seconds=xchg_s, intervals=(mine.start, mine.stop), world=world)
