"""The N > 1 path on CPU: world_size-2 gloo process group over 127.0.0.1 (bench.py's replica
plumbing -- independent products per rank, max-over-ranks job time, whole-job throughput)."""
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


def _worker(rank, world, port, times, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        ms_max = bench.max_over_ranks(times[rank], world, torch.device("cpu"))
        value = bench.job_throughput(5, world, ms_max * 1e-3)
        seeds = [None] * world
        dist.all_gather_object(seeds, bench.replica_seed(rank))
        q.put((rank, ms_max, value, seeds))
    finally:
        dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world, port = 2, _free_port()
    times = [12.5, 17.25]  # per-rank device ms for 5 steps
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, times, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms_max, value, seeds in out:
        assert ms_max == max(times)                      # slowest rank sets the job time
        assert value == pytest.approx(world * 5 / (max(times) * 1e-3))
        assert len(set(seeds)) == world                  # independent replica inputs


def test_single_rank_no_collective():
    import bench
    assert bench.max_over_ranks(3.5, 1, torch.device("cpu")) == 3.5
    assert bench.job_throughput(4, 1, 2.0) == 2.0
