"""Multi-GPU host logic on CPU (-m "not gpu"): world_size 2 over gloo (replicas
only).  bench.py's cross-rank reduction gives the job time (max over ranks) and the work of all
ranks (sum), and the reference arm does its work on rank 0 only."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    t, w = bench.reduce_over_ranks(10.0 + rank, 100.0 * (rank + 1), torch.device("cpu"))
    out[rank] = (t, w)

    class A:
        pass

    a = A()
    if rank != 0:   # the reference arm: ranks other than 0 exit 0 without work
        out[world + rank] = bench.run_reference(a, rank, world)
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_over_ranks_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, start_method="spawn", join=True)
    for r in range(world):
        assert out[r] == (11.0, 300.0)   # max time, summed work
    assert out[world + 1] == 0
