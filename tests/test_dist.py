"""N > 1 host logic on CPU: world-size-2 gloo process group exercising bench.py's
replica-mode helpers (barrier, max-over-ranks timing, RHS dealing)."""
import os
import socket

import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    bench.barrier(world)
    m = bench.max_over_ranks(1.5 + rank, world)
    plan = bench.replica_plan(world, rank, n_rhs=8)
    q.put((rank, m, plan))
    dist.destroy_process_group()


def test_replica_helpers_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [m for _, m, _ in out] == [2.5, 2.5]
    assert out[0][2] == [0, 2, 4, 6] and out[1][2] == [1, 3, 5, 7]
    assert sorted(out[0][2] + out[1][2]) == list(range(8))
