"""N>1 path of bench.py on the CPU: two gloo ranks, the job time is the max
over ranks and the whole-job value counts every rank's replica."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = bench.max_over_ranks(10.0 + 5.0 * rank, world, "cpu")
    out[rank] = (ms, bench.replica_throughput(world, 1, ms))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_aggregation():
    world = 2
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
        got = dict(out)
    for rank in range(world):
        ms, value = got[rank]
        assert ms == pytest.approx(15.0)  # slowest rank
        assert value == pytest.approx(2 / 15e-3)  # both replicas' matvecs over the job time
