"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

Ranks own disjoint ensemble members (no data-path collective); the step time is the
max over ranks and units add up across ranks.  The per-member solves here use the CPU
oracle as a stand-in workload; on the GPU box the same logic drives libpe (bench.py).
"""

import os
import socket

import numpy as np
import pytest

from paper_2411_09244_b200.dist import shard_members


def test_shard_members_balanced_and_disjoint():
    for n in (0, 1, 7, 64):
        for w in (1, 2, 3, 8):
            ranges = [shard_members(n, r, w) for r in range(w)]
            flat = [m for rg in ranges for m in rg]
            assert flat == list(range(n))
            sizes = [len(rg) for rg in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_members(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from oracle import pe_oracle as po
    from paper_2411_09244_b200.dist import (gather_member_results, max_over_ranks,
                                            shard_members, sum_over_ranks)
    from tests.conftest import GOLDEN

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(os.path.join(GOLDEN, "sys_cfg0.npz"))
    blocks = [z[k] for k in ("M11", "A11", "M12", "A12", "M22", "A22")]
    local_iters, local_units, t_local = {}, 0, 0.0
    for m in shard_members(4, rank, world):
        scale = 0.5 ** m  # member-specific diffusion (kappa) scaling
        s = po.OSystem(blocks[0], blocks[1] * scale, blocks[2], blocks[3] * scale, blocks[4],
                       blocks[5] * scale, z["f1"], z["f2"])
        r = po.run_parareal(s, np.zeros(64), 1.0, 10, 10, epsilon=1e-8, k_max=10,
                            stop="relative")
        local_iters[m] = r["iterations"]
        local_units += 64 * 10 * 10 * r["iterations"]
        t_local += sum(r["fine_seconds"]) + sum(r["coarse_seconds"])
    t_max = max_over_ranks(t_local)
    units = sum_over_ranks(local_units)
    merged = gather_member_results(local_iters)
    if rank == 0:
        np.save(os.path.join(out_dir, "result.npy"),
                np.array([t_max, t_local, units] + [merged[m] for m in range(4)]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_ensemble_sharding(tmp_path):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    res = np.load(tmp_path / "result.npy")
    t_max, t0, units = res[:3]
    iters = res[3:].astype(int)
    assert t_max >= t0 > 0
    assert units == 64 * 100 * iters.sum()
    # every member converges, and matches a single-process run of the same member
    from oracle import pe_oracle as po
    from tests.conftest import GOLDEN

    z = np.load(os.path.join(GOLDEN, "sys_cfg0.npz"))
    for m in range(4):
        sc = 0.5 ** m
        s = po.OSystem(z["M11"], z["A11"] * sc, z["M12"], z["A12"] * sc, z["M22"],
                       z["A22"] * sc, z["f1"], z["f2"])
        r = po.run_parareal(s, np.zeros(64), 1.0, 10, 10, epsilon=1e-8, k_max=10, stop="relative")
        assert r["iterations"] == iters[m]
