"""The N>1 bench plumbing on CPU: world_size-2 gloo process group (the
driver launches bench.py under torchrun with 127.0.0.1).  Checks the
max-over-ranks timing reduction, the batch sharding and whole-job TOPS, and
that the reference arm does no work on ranks != 0."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = bench.max_over_ranks(10.0 + 5.0 * rank, world, torch.device("cpu"))
        r, w, lr = bench.dist_env()
        bpg = bench.shard_batch(256, w)

        class A:  # bench.run_reference args; rank != 0 must return at once
            layers, cpu_seconds, steps, warmup, batch = "", 1.0, 1, 1, 256
        ref = bench.run_reference(A, r, w) if r != 0 else None
        q.put((rank, got, r, w, bpg, ref))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, r, w, bpg, ref in res:
        assert got == 15.0          # the slower rank's time on every rank
        assert (r, w) == (rank, 2)
        assert bpg == 128           # 256 images sharded over 2 ranks
        assert ref is None


def test_job_tops_and_sharding():
    assert bench.job_tops(10**12, 2, 1000.0) == pytest.approx(2.0)
    assert bench.shard_batch(256, 8) == 32
    with pytest.raises(ValueError):
        bench.shard_batch(256, 3)
