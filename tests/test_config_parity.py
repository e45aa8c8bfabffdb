"""Parity at BASELINE.json's own configurations: configs[0] (C1, 2D Q1 128^2)
and configs[1] (C2, 3D 7-point 48^3, the bench workload), against fixtures
the REFERENCE produced (tests/golden/make_golden_configs.py ->
tests/golden/cfg_c1.npz, cfg_c2.npz).

CPU tests pin the oracle to those fixtures bit for bit (integer structure and
pivot sequences) and to 1e-12 (mf_solve). GPU tests hold the device path to:
  * front records and FactorStats counters: exact
  * every block's |I| and |J| (BDLR selections): exact
  * pivot sequences: the match rate is reported; the mismatches may be at
    most twice the reference's OWN under a 1-ulp perturbation of its dense
    solves (env_pivot_rate, measured by the fixture script): on a
    configuration where the reference itself re-picks pivots under 1-ulp
    noise, exact equality is not a property of the reference
  * mf_solve: within max(1e-8, 10 x the reference's own 1-ulp envelope)
  * GMRES(restart) to 1e-10: iterations within +-1, converged, and the final
    residual <= tol like the reference's
The reference's envelopes are recorded in BASELINE.md (C1 4.5e-10, C2 3.0e-5).
"""
import numpy as np
import pytest

from paper_1410_2697_b200 import problems as PR

CFG = {
    "c1": (lambda: PR.gen_q1_2d(128), 64, dict(n_c=256, eps=1e-6, d=1, n_leaf=32), "uniform", 30),
    "c2": (lambda: PR.gen_poisson7(48, 48, 48), 64, dict(n_c=1024, eps=1e-5, d=1, n_leaf=64), "normal", 30),
}


def _records(recs):
    return np.array([[r[0], r[1], r[2], {"empty": 0, "dense": 1, "structured": 2}[r[3]], r[4], r[5]]
                     for r in recs], dtype=np.int64)


@pytest.mark.parametrize("name", ["c1", pytest.param("c2", marks=pytest.mark.slow)])
def test_oracle_matches_reference_at_config(golden, oracle, name):
    """The CPU oracle is the reference at config scale: identical records,
    selections, ranks and pivot sequences; mf_solve to 1e-12."""
    from threadpoolctl import threadpool_limits
    g = golden(f"cfg_{name}.npz")
    gen, leaf, kw, dist, restart = CFG[name]
    A, _ = gen()
    b = PR.seeded_rhs(A.n_rows, 0, dist)
    # the fixtures were made with one BLAS thread; at C2 the reference itself
    # picks different pivots with 8 OpenBLAS threads (rounding-chaotic config)
    with threadpool_limits(1):
        _oracle_check(oracle, g, A, b, leaf, kw)


def _oracle_check(oracle, g, A, b, leaf, kw):
    np.testing.assert_array_equal(b, g["b"])
    ip, ix = oracle.adjacency(A._csc)
    et = oracle.build_elimination_tree(oracle.nested_dissection(ip, ix, A.n_rows, leaf), A._csc)
    log = {}
    F = oracle.factorize(A._csc, et, "accelerated", block_log=log, **kw)
    np.testing.assert_array_equal(_records(F.stats.records), g["records"])
    st = F.stats
    stored = sum(f.stored() for f in F.factors.values() if f is not None)
    np.testing.assert_array_equal([st.peak, st.structured, st.dense, st.full_square, stored], g["counters"])
    blocks = [d for p in et.post_order for d in log.get(p, [])]
    ref, perms = g["blk"], g["blkperm"]
    assert len(blocks) == len(ref)
    q = 0
    for d, (m, n, r) in zip(blocks, ref):
        assert (d["nI"], d["nJ"], d["rank"]) == (m, n, r)
        np.testing.assert_array_equal(d["row_perm"], perms[q:q + r, 0])
        np.testing.assert_array_equal(d["col_perm"], perms[q:q + r, 1])
        q += r
    x = oracle.solve(F, b)
    assert np.linalg.norm(x - g["x"]) <= 1e-12 * np.linalg.norm(g["x"])


def test_config_fixtures_are_consistent(golden):
    """The fixtures describe converged reference runs (these are the
    (d, n_c) at which the reference converges)."""
    for name in CFG:
        g = golden(f"cfg_{name}.npz")
        its, conv, tol, restart = g["gmres_meta"]
        assert bool(conv) and g["gmres_hist"][-1] <= tol
        assert float(g["true_res"]) <= 10 * tol
        assert len(g["blk"]) > 0 and int(g["counters"][1]) > 0
        assert 0.9 <= float(g["env_pivot_rate"]) <= 1.0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_device_matches_reference_at_config(golden, name):
    import paper_1410_2697_b200 as P
    g = golden(f"cfg_{name}.npz")
    gen, leaf, kw, dist, restart = CFG[name]
    A, _ = gen()
    b = g["b"]
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), leaf), A)
    F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(**kw))
    recs = np.array([[r.node_id, r.front_size, r.n_pivot, {"empty": 0, "dense": 1, "structured": 2}[r.path],
                      r.max_offdiag_rank, r.stored_reals] for r in F.stats.records], dtype=np.int64)
    ref_recs = g["records"]
    # the integer structure of every front: exact
    np.testing.assert_array_equal(recs[:, :4], ref_recs[:, :4])
    log = F.block_log()
    ref, perms = g["blk"], g["blkperm"]
    assert len(log) == len(ref)
    q = same = 0
    shifted = set()  # fronts with a block whose rank differs from the reference's
    for d, (m, n, r) in zip(log, ref):
        assert (d["nI"], d["nJ"]) == (m, n)  # BDLR selections: exact
        if d["rank"] != r:
            shifted.add(d["node"])
        if d["rank"] == r and np.array_equal(d["row_perm"], perms[q:q + r, 0]) and \
                np.array_equal(d["col_perm"], perms[q:q + r, 1]):
            same += 1
        q += r
    rate = same / len(log)
    env_rate = float(g["env_pivot_rate"])
    print(f"{name}: pivot-sequence match {same}/{len(log)} = {rate:.4f} (reference 1-ulp self-match {env_rate:.4f}); "
          f"fronts with a shifted rank {len(shifted)} (reference 1-ulp: {int(g['env_records_mismatch'])} records move)")
    # the reference itself re-picks (1 - env_rate) of its pivot sequences under
    # 1-ulp noise; an implementation with different (equally valid) rounding
    # must stay within the same order: at most twice that many, plus one block
    assert (1.0 - rate) <= 2.0 * (1.0 - env_rate) + 1.0 / len(log), (rate, env_rate)
    # ranks / stored reals: exact on every front whose block ranks all match;
    # a shifted rank moves that front's accounting exactly as it moves the
    # reference's own under 1-ulp noise
    keep = np.array([int(nd) not in shifted for nd in recs[:, 0]])
    np.testing.assert_array_equal(recs[keep], ref_recs[keep])
    assert len(shifted) <= max(2, 2 * int(g["env_records_mismatch"]))
    cnt = [F.stats.peak_stored_reals, F.stats.structured_fronts, F.stats.dense_fronts, F.stats.full_square_allocs,
           F.stored_reals()]
    np.testing.assert_array_equal(cnt[1:4], g["counters"][1:4])
    if not shifted:
        np.testing.assert_array_equal(cnt, g["counters"])
    else:
        for k in (0, 4):
            assert abs(cnt[k] - g["counters"][k]) <= max(abs(g["env_counters"][k] - g["counters"][k]),
                                                         1e-3 * g["counters"][k]), (k, cnt[k], g["counters"][k])
    x = P.mf_solve(F, b)
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    env = float(g["env_rel"])
    print(f"{name}: mf_solve rel diff {rel:.3e} (reference 1-ulp envelope {env:.3e})")
    assert rel <= max(1e-8, 10 * env), (rel, env)
    its, conv, tol, _ = g["gmres_meta"]
    xg, h = P.gmres(A, b, M=P.mf_preconditioner(F), tol=float(tol), restart=restart)
    print(f"{name}: GMRES {h.iterations} iterations (reference {int(its)}), final {h.residuals[-1]:.3e} "
          f"(reference {g['gmres_hist'][-1]:.3e})")
    assert h.converged and abs(h.iterations - int(its)) <= 1
    assert h.residuals[-1] <= tol
    true_res = np.linalg.norm(A._csc @ xg - b) / np.linalg.norm(b)
    assert true_res <= 10 * tol
