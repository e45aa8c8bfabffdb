"""Subtree partition for the sharded factorization on CPU: cut
properties, determinism across a world-size-2 gloo group, and exactness of
the disjoint-support all-reduce the exchange step relies on."""
import os
import socket

import numpy as np
import pytest


def _tree(n=20):
    import paper_1410_2697_b200 as P
    from paper_1410_2697_b200 import problems as PR
    A, _ = PR.gen_poisson7(n, n, n)
    return P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 32), A)


def _check_partition(tree, part, world):
    nodes = tree.nodes
    owner = part.owners()
    assert owner.dtype == np.int32 and owner.min() >= 0 and owner.max() < world
    top = set(part.top)
    for v in tree.post_order:
        nd = nodes[v]
        if v in top:
            if nd.parent is not None:
                assert nd.parent in top  # the top is closed upward
        else:
            for c in nd.children:
                assert owner[c] == owner[v]  # subtrees are whole
                assert c not in top


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_cut_properties(world):
    from paper_1410_2697_b200.sharded import SubtreePartition
    tree = _tree()
    part = SubtreePartition(tree, world)
    _check_partition(tree, part, world)
    if world == 1:
        assert part.top == [] and set(part.owners()) == {0}
    else:
        assert all(l > 0 for l in part.load)  # every rank factors something
        assert max(part.load) <= 2.0 * (sum(part.load) / world)
        # sibling top fronts at one height go to different ranks when there are enough ranks
        assert len(set(part.owners()[part.top])) == min(world, len(part.top))
    # deterministic
    again = SubtreePartition(tree, world)
    assert again.top == part.top and np.array_equal(again.node_owner, part.node_owner)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1410_2697_b200.sharded import SubtreePartition
    part = SubtreePartition(_tree(16), world)
    owners = [None] * world
    dist.all_gather_object(owners, part.owners().tolist())
    # the exchange premise: every slot written by one rank, zero elsewhere -> exact sum
    rng = np.random.default_rng(5)
    vals = rng.standard_normal(4096) * np.exp(rng.uniform(-700, 700, 4096))
    vals[:4] = [5e-324, -5e-324, 1.7e308, -0.0]
    mine = np.where(np.arange(4096) % world == rank, vals, 0.0)
    t = torch.from_numpy(mine.copy())
    dist.all_reduce(t)
    exact = bool(np.array_equal(t.numpy(), vals + 0.0))
    q.put((rank, owners[0] == owners[1], exact))
    dist.destroy_process_group()


def test_partition_and_exchange_world2_gloo():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(same for _, same, _ in out)
    assert all(exact for _, _, exact in out)
