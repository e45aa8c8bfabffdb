"""N > 1 host logic on CPU: world-size-2 gloo process group exercising bench.py's
multi-rank helpers (barrier, max-over-ranks timing) and the subtree partition,
which every rank must compute identically without talking to the others."""
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
    import torch
    import bench
    import paper_1410_2697_b200 as P
    from paper_1410_2697_b200.sharded import SubtreePartition
    bench.barrier(world)
    m = bench.max_over_ranks(1.5 + rank, world)
    A, _ = P.gen_poisson7(14, 13, 12)
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 32), A)
    own = torch.from_numpy(SubtreePartition(et, world).owners().astype("int64"))
    got = [torch.zeros_like(own) for _ in range(world)]
    dist.all_gather(got, own)
    plan = [bool(torch.equal(g, own)) for g in got] + [int((own == rank).sum())]
    q.put((rank, m, plan))
    dist.destroy_process_group()


def test_multirank_helpers_world2():
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
    for _, _, plan in out:
        assert plan[:2] == [True, True] and plan[2] > 0  # same owners everywhere, work on both ranks
