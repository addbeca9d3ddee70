"""Multi-process (world size 2, gloo on CPU) coverage of bench.py's replica
path: barrier, max-over-ranks timing and the whole-job aggregate value."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    bench.barrier(world)
    t_rank = 1.5 + rank  # rank 1 is the slow one
    t_max = bench.max_over_ranks(t_rank, world, "cpu")
    value = bench.replica_value(world, 10, 1000, t_max)
    bench.barrier(world)
    q.put((rank, t_max, value))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replicas_take_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(90)
        assert p.exitcode == 0
    out = sorted(q.get(timeout=5) for _ in range(world))
    for rank, t_max, value in out:
        assert t_max == 2.5  # the slowest rank's time, seen by every rank
        assert value == pytest.approx(2 * 10 * 1000 / 2.5)


def test_single_rank_is_identity():
    import bench

    assert bench.max_over_ranks(3.25, 1, "cpu") == 3.25
    assert bench.replica_value(1, 4, 100, 2.0) == 200.0
