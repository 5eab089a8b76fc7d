"""Sharding plan for N beyond one GPU, on CPU
(-m "not gpu"): the partition, the pairwise halo exchange and the exact cross-rank sums,
world_size 2 over gloo.  Data movement and integer sums only: the sweep stays in the kernels."""
import math
import os
import socket
import sys
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_03019_b200 import shard  # noqa: E402

N = 12
XE = 12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _global_class():
    return np.random.default_rng(5).random(1 << (N - 1))


def _layer_sums(rank):
    return np.random.default_rng(100 + rank).random((N + 1, 3)) * 7.0


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = shard.ShardPlan(N, world, rank)
    glob = _global_class()
    lo = rank * plan.local_states
    mine = torch.from_numpy(glob[lo:lo + plan.local_states].copy())
    halo = shard.exchange_halo(plan, mine)
    # every top-unit neighbour of every local state, from the partner's slice
    ok = True
    local = np.arange(plan.local_states, dtype=np.uint64)
    gidx = plan.global_index(local)
    for u, _ in plan.top_units:
        want = glob[(gidx ^ np.uint64(1 << (u - 1))).astype(np.int64)]   # compressed bit u - 1
        ok = ok and np.array_equal(halo[u].numpy(), want)
    # exact per-layer sums across ranks
    limbs = torch.from_numpy(np.stack([[shard.to_limbs(x, XE) for x in row] for row in _layer_sums(rank)]))
    shard.allreduce_exact(limbs)
    out[rank] = (ok, limbs.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_halo_exchange_and_exact_sums_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, start_method="spawn", join=True)
    assert out[0][0] and out[1][0], "halo slices differ from the neighbours' values"
    # both ranks hold the same bits, equal to the exact sum of the truncated addends
    assert np.array_equal(out[0][1], out[1][1])
    unit = Fraction(2) ** (XE - 32 * shard.HQ_XL)
    for L in range(N + 1):
        for v in range(3):
            exact = sum(Fraction(math.floor(Fraction(_layer_sums(r)[L, v]) / unit)) for r in range(world))
            got = sum(int(out[0][1][L, v, k]) << (32 * k) for k in range(shard.HQ_XL))
            assert got == exact
            assert abs(shard.from_limbs(out[0][1][L, v], XE) - sum(_layer_sums(r)[L, v] for r in range(world))) <= 1e-13


def test_plan_partition_and_memory():
    for world in (1, 2, 4):
        plans = [shard.ShardPlan(N, world, r) for r in range(world)]
        assert sum(p.local_states for p in plans) == 1 << (N - 1)
        for p in plans:
            assert len(p.top_units) == p.s
            for u, partner in p.top_units:
                assert 0 <= partner < world and partner != p.rank
            j = np.uint64(p.rank * p.local_states + 5)
            assert p.owner(int(j)) == (p.rank, 5)
    with pytest.raises(ValueError):
        shard.ShardPlan(N, 3, 0).s
    # the memory budget that makes sharding necessary: 180 GB per B200
    assert shard.ShardPlan(31, 1, 0).rank_bytes() < 100e9
    assert shard.ShardPlan(33, 1, 0).rank_bytes() > 180e9
    assert shard.ShardPlan(33, 2, 0).rank_bytes() < 180e9
