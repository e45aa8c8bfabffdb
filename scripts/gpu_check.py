"""Quick GPU parity sweep (development helper): device path vs the CPU oracle."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, '.')
import paper_1410_2697_b200 as P
from oracle import mfh_oracle as O

def log(*a):
    print(*a, flush=True)

# 1. full pivot LU
rng = np.random.default_rng(0)
blocks, caps, epss = [], [], []
for t in range(40):
    m = int(rng.integers(1, 40)); n = int(rng.integers(1, 40)); r = int(rng.integers(1, min(m, n) + 1))
    B = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    blocks.append(B); caps.append(int(rng.integers(1, min(m, n) + 1)))
ok = 0
for B, cap in zip(blocks, caps):
    eps = 1e-6
    g = P.full_pivot_lu(B, eps, cap)
    o = O.full_pivot_lu(B, eps, cap)
    same = g[3] == o[3] and np.array_equal(g[1], o[1]) and np.array_equal(g[2], o[2]) and np.array_equal(g[0], o[0]) and g[4] == o[4]
    ok += same
    if not same:
        log("FPLU mismatch", B.shape, cap, g[3], o[3], np.abs(g[0]-o[0]).max())
log("fplu parity", ok, "/", len(blocks))

def run(name, A, leaf, mode, **kw):
    t = time.time()
    g = P.adjacency_graph(A); st = P.nested_dissection(g, leaf); et = P.build_elimination_tree(st, A)
    ip, ix = O.adjacency(A._csc); ost = O.nested_dissection(ip, ix, A.n_rows, leaf); ot = O.build_elimination_tree(ost, A._csc)
    b = np.random.default_rng(1).standard_normal(A.n_rows)
    params = P.MfParams(**kw)
    t0 = time.time()
    F = P.mf_factorize(A, et, mode, params)
    tf = time.time() - t0
    x = P.mf_solve(F, b)
    log_ = {}
    OF = O.factorize(A._csc, ot, mode, block_log=log_, **kw)
    ox = O.solve(OF, b)
    rel = np.linalg.norm(x - ox) / np.linalg.norm(ox)
    recs = [(r.node_id, r.front_size, r.n_pivot, r.path, r.max_offdiag_rank, r.stored_reals) for r in F.stats.records]
    rec_ok = recs == OF.stats.records
    bl = F.block_log()
    obl = [d for p in ot.post_order for d in log_.get(p, [])]
    nb_ok = len(bl) == len(obl)
    piv_ok = sum(1 for a, b2 in zip(bl, obl) if a['rank'] == b2['rank'] and np.array_equal(a['row_perm'], b2['row_perm']) and np.array_equal(a['col_perm'], b2['col_perm']) and a['dense'] == b2['dense'] and a['nI']==b2['nI'] and a['nJ']==b2['nJ'])
    log(f"{name}: rel(mf_solve vs oracle)={rel:.2e} records={rec_ok} peak={F.stats.peak_stored_reals}/{OF.stats.peak} "
        f"struct={F.stats.structured_fronts} blocks={len(bl)}/{len(obl)} pivots_match={piv_ok} fsq={F.stats.full_square_allocs}/{OF.stats.full_square} factor {tf*1e3:.1f} ms")
    return F, et

for name, A, leaf, mode, kw in [
    ("p7 6^3 conv", P.gen_poisson7(6,6,6)[0], 16, "conventional", {}),
    ("p7 8^3 acc", P.gen_poisson7(8,8,8)[0], 16, "accelerated", dict(n_c=32, eps=1e-5, d=1, n_leaf=16)),
    ("p7 12^3 acc", P.gen_poisson7(12,12,12)[0], 64, "accelerated", dict(n_c=64, eps=1e-5, d=1, n_leaf=16)),
    ("p7 10^3 acc d2", P.gen_poisson7(10,10,10)[0], 32, "accelerated", dict(n_c=64, eps=1e-3, d=2, n_leaf=32)),
    ("q1 64^2 acc", P.gen_q1_2d(64)[0], 64, "accelerated", dict(n_c=128, eps=1e-6, d=1, n_leaf=32)),
    ("p7 16^3 acc", P.gen_poisson7(16,16,16)[0], 64, "accelerated", dict(n_c=256, eps=1e-5, d=1, n_leaf=64)),
]:
    try:
        run(name, A, leaf, mode, **kw)
    except Exception:
        traceback.print_exc()

# gmres
try:
    A, _ = P.gen_poisson7(16, 16, 16)
    b = np.random.default_rng(0).standard_normal(A.n_rows)
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 64), A)
    F = P.mf_factorize(A, et, "accelerated", P.MfParams(n_c=256, eps=1e-5, d=1, n_leaf=64))
    M = P.mf_preconditioner(F)
    x, h = P.gmres(P.LinearOperator.from_matrix(A), b, M=M, tol=1e-10, restart=30)
    ip, ix = O.adjacency(A._csc); ot = O.build_elimination_tree(O.nested_dissection(ip, ix, A.n_rows, 64), A._csc)
    OF = O.factorize(A._csc, ot, "accelerated", n_c=256, eps=1e-5, d=1, n_leaf=64)
    ox, ores, oits, oconv = O.gmres(lambda v: A._csc @ v, b, lambda v: O.solve(OF, v), tol=1e-10, restart=30)
    log("gmres its", h.iterations, "oracle", oits, "res", h.residuals[-1], ores[-1], "x rel", np.linalg.norm(x-ox)/np.linalg.norm(ox))
    ms, by = F.apply_bench(20)
    log("apply", ms, "ms", by/1e6, "MB")
    log("timing", F.timing())
except Exception:
    traceback.print_exc()
