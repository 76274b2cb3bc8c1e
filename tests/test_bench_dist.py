"""Multi-process (world_size 2, gloo, CPU) check of the replica aggregation bench.py uses for
--gpus N under torchrun: times are max-reduced, work units sum-reduced."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, work = bench.replica_aggregate(10.0 + rank, 7 + rank)
    out[rank] = (ms, work)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregate_two_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1] == (11.0, 15.0)


def test_replica_aggregate_single_process_is_identity():
    import bench
    assert bench.replica_aggregate(3.5, 9) == (3.5, 9.0)
