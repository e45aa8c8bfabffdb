"""Subtree-sharded factorization on the GPU: world-size-2 and -3
gloo groups of processes sharing one GPU (the exchanges are host-side between
launches, so no kernel waits on another rank). With the compressed
point-to-point update exchange and with the dense all-reduce fallback, the
sharded preconditioner's apply, GMRES solution and iteration count, stats and
records must be bitwise equal to the single-GPU factorization's."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    "p7_16": (lambda PR: PR.gen_poisson7(16, 16, 16)[0], 32, dict(n_c=96, eps=1e-5, d=1, n_leaf=32)),
    "hex_8": (lambda PR: PR.gen_hex_q1(8, seed=3)[0], 32, dict(n_c=96, eps=1e-4, d=1, n_leaf=32)),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _recs(F):
    return [(r.node_id, r.front_size, r.n_pivot, r.path, r.max_offdiag_rank, r.stored_reals)
            for r in F.stats.records]


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1410_2697_b200 as P
        from paper_1410_2697_b200 import problems as PR
        from paper_1410_2697_b200.sharded import gmres_sharded, mf_factorize_sharded
        gen, leaf, kw = CASES[case]
        A = gen(PR)
        tree = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), leaf), A)
        params = P.MfParams(**kw)
        b = np.random.default_rng(0).standard_normal(A.n_rows)
        out = dict(rank=rank)
        for compressed in (True, False):
            F = mf_factorize_sharded(A, tree, P.ACCELERATED, params, compressed=compressed)
            x = P.mf_solve(F, b)
            xg, h = P.gmres(A, b, M=P.mf_preconditioner(F), tol=1e-10, restart=30)
            xd, hd = gmres_sharded(A, b, F, tol=1e-10, restart=30) if compressed else (None, None)
            if compressed:
                out["dist"] = dict(x=xd, its=hd.iterations, conv=hd.converged,
                                   res=float(np.linalg.norm(A._csc @ xd - b) / np.linalg.norm(b)))
            out[compressed] = dict(x=x, xg=xg, its=h.iterations, hist=np.asarray(h.residuals), recs=_recs(F),
                                   peak=F.stats.peak_stored_reals,
                                   counts=(F.stats.structured_fronts, F.stats.dense_fronts),
                                   calls=F.exchange.calls, p2p=F.exchange.p2p_calls, p2p_bytes=F.exchange.p2p_bytes,
                                   owners=F.partition.owners())
            F = None
        if rank == 0:
            F1 = P.mf_factorize(A, tree, P.ACCELERATED, params)
            x1g, h1 = P.gmres(A, b, M=P.mf_preconditioner(F1), tol=1e-10, restart=30)
            out.update(x1=P.mf_solve(F1, b), x1g=x1g, its1=h1.iterations, hist1=np.asarray(h1.residuals),
                       recs1=_recs(F1), peak1=F1.stats.peak_stored_reals,
                       counts1=(F1.stats.structured_fronts, F1.stats.dense_fronts))
        dist.barrier()
        q.put(out)
        dist.destroy_process_group()
    except Exception as e:  # surfaced by the parent
        import traceback
        q.put(dict(rank=rank, error=traceback.format_exc()))


@pytest.mark.parametrize("world,case", [(2, "p7_16"), (3, "p7_16"), (2, "hex_8")])
def test_sharded_factor_bitwise_equals_single(world, case):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in ps:
        p.start()
    outs = sorted((q.get(timeout=240) for _ in ps), key=lambda o: o["rank"])
    for p in ps:
        p.join(timeout=60)
    for o in outs:
        assert "error" not in o, o.get("error")
    r0 = outs[0]
    assert len(set(r0[True]["owners"].tolist())) == world  # every rank owns fronts
    # compressed point-to-point update exchange (UpdateRep form) and the dense
    # all-reduce fallback: both bitwise the single-GPU factorization
    for compressed in (True, False):
        for o in outs:
            c = o[compressed]
            assert c["calls"] > 0
            np.testing.assert_array_equal(c["x"], r0["x1"])
            np.testing.assert_array_equal(c["xg"], r0["x1g"])
            assert c["its"] == r0["its1"]
            np.testing.assert_array_equal(c["hist"], r0["hist1"])
            assert c["recs"] == r0["recs1"]
            assert c["peak"] == r0["peak1"] and c["counts"] == r0["counts1"]
    assert sum(o[True]["p2p"] for o in outs) > 0 and sum(o[True]["p2p_bytes"] for o in outs) > 0
    # distributed GMRES (rank-local vectors, halo SpMV, CGS2): every rank gets
    # the same solution, iterations within one of the replicated solve
    for o in outs:
        d = o["dist"]
        assert d["conv"] and abs(d["its"] - r0["its1"]) <= 1 and d["res"] <= 1e-9
        np.testing.assert_array_equal(d["x"], outs[0]["dist"]["x"])
        assert np.linalg.norm(d["x"] - r0["x1g"]) <= 1e-7 * np.linalg.norm(r0["x1g"])
    assert all(o[False]["p2p"] == 0 for o in outs)
