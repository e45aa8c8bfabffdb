/*
 * mfh.h — C-ABI of the B200-native HODLR-multifrontal hot path (libmfh.so).
 *
 * This is the drop-in boundary. Plain pointers, sizes and opaque handles only;
 * no torch / numpy types. Every entry point returns 0 on success and a nonzero
 * error kind on failure, with the message (reference text) in mfh_last_error():
 *
 *   MFH_EVALUE  -> Python ValueError              (reference raises ValueError)
 *   MFH_EPIVOT  -> PivotMonotonicityError          (_kernels/_core.pyx:17)
 *   MFH_ERUNTIME-> RuntimeError (CUDA failure, bad handle, internal error)
 *
 * Each entry point cites the reference interface it replaces
 * (/root/reference/pkg/src/mfhodlr/<file>:<line>). The Python binding that a
 * maintainer adds on the reference side is shown in INTEGRATION.md.
 *
 * Threading: calls that use a context are serialized per context (a
 * recursive lock: a GMRES host-callback operator may call back into the
 * library on the same thread). Distinct contexts run independently.
 * Lifetimes: an mfh_etree may be freed while factors built on it live on.
 */
#ifndef MFH_H_
#define MFH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFH_OK 0
#define MFH_EVALUE 1
#define MFH_EPIVOT 2
#define MFH_ERUNTIME 3

typedef struct mfh_ctx mfh_ctx;          /* device + stream + workspaces          */
typedef struct mfh_nd mfh_nd;            /* separator tree (ordering.py:32-56)    */
typedef struct mfh_etree mfh_etree;      /* elimination tree (ordering.py:238-261)*/
typedef struct mfh_factor mfh_factor;    /* MfFactorization (multifrontal.py:227) */
typedef struct mfh_csr mfh_csr;          /* device CSR operator (krylov.py:21-33) */
typedef struct mfh_precond mfh_precond;  /* baseline preconditioners (krylov.py:164-204) */

/* MfParams (multifrontal.py:34-48); max_rank < 0 means None. */
typedef struct {
  int64_t n_c;
  double eps;
  int64_t d;
  int64_t n_leaf;
  int64_t max_rank;
} mfh_params;

/* mode (multifrontal.py:30-31, 459-470) */
#define MFH_CONVENTIONAL 0
#define MFH_ACCELERATED 1

/* FactorStats counters (multifrontal.py:61-103) */
typedef struct {
  int64_t peak_stored_reals;
  int64_t retained_reals;
  int64_t structured_fronts;
  int64_t dense_fronts;
  int64_t full_square_allocs;
  int64_t n_records;
  int64_t stored_reals; /* MfFactorization.stored_reals() (multifrontal.py:239) */
  /* device-side truth, not in the reference */
  int64_t device_bytes_peak;
  int64_t n_blocks;    /* compressed off-diagonal blocks */
  int64_t n_dense_fallback;
} mfh_stats_t;

/* one FrontRecord (multifrontal.py:51-58); path: 0 empty, 1 dense, 2 structured */
typedef struct {
  int64_t node_id, front_size, n_pivot, path, max_offdiag_rank, stored_reals;
} mfh_record_t;

/* per-phase device timing of the last mfh_factorize (ms, CUDA events) */
typedef struct {
  double total_ms;
  double sample_ms, pivot_lu_ms, skeleton_ms, hodlr_factor_ms, dense_front_ms, eliminate_ms;
  double host_ms;        /* host work before the first launch + BDLR selection */
  double host_preamble_ms, host_select_ms, host_sync_wait_ms, wall_ms;
  double apply_build_ms, apply_instantiate_ms; /* first-use CUDA-graph construction */
  double gmres_ms, gmres_apply_ms, gmres_sync_ms; /* last GMRES using this factor (host clock) */
  int64_t kernel_launches;
  double pivot_lu_visits; /* algorithmic trailing-entry visits */
  double sample_entries;
  /* algorithmic counts of the REFERENCE's algorithm on this factor's structure
   * (SURVEY 8d), the numerators of the per-phase rooflines */
  double hodlr_flops;     /* a14 hodlr_factorize: leaf getrf + Woodbury (hodlr.py:312-357) */
  double elim_flops;      /* a16 eliminate_hodlr: x = H^{-1} col_pf, core, W / V (multifrontal.py:424-438) */
  double dense_flops;     /* a5 dense fronts: (2/3) n_p^3 + 2 n_p^2 nf + 2 n_p nf^2 */
  double skeleton_flops;  /* a9 the two triangular solves: r^2 (m + n) per low-rank block */
  double sample_lr_flops; /* a7 2 r per sampled entry per low-rank child term W V^T it meets */
  double pivot_lu_crit_steps; /* sum over structured heights of the longest core's steps */
  double apply_ref_bytes; /* one mf_solve by SURVEY 8d's count: 8 sum(2 S_pp + S_pf + S_fp) + 32 N */
  /* flops this engine executed per phase (GEMMs 2mnk, register inverses 2n^3):
   * the numerators of the achieved-throughput rooflines (the reference's own
   * counts above can be lower or higher than the work this form does) */
  double exec_flops_skeleton, exec_flops_hodlr, exec_flops_elim, exec_flops_dense;
  /* child updates written out as dense blocks before their parent's height samples them
   * (HODLR leaves and low-rank blocks, minus W V^T): device time, executed flops, and the
   * rest of the time between a height's sampling and the previous height's end, in which
   * the GPU waits for the host (planning, request building) */
  double materialize_ms, exec_flops_materialize, idle_gap_ms;
} mfh_timing_t;

/* ---- errors --------------------------------------------------------------- */
const char *mfh_last_error(void);
int mfh_version(void);

/* ---- context -------------------------------------------------------------- */
int mfh_ctx_create(int device, mfh_ctx **out);
void mfh_ctx_destroy(mfh_ctx *ctx);
int mfh_ctx_sync(mfh_ctx *ctx);
/* the context's cudaStream_t (for event timing by the caller) and the number
 * of kernels this context has launched so far (graph replays count nodes) */
int mfh_ctx_info(mfh_ctx *ctx, void **stream, int64_t *launches);

/* ---- host symbolic analysis (bit-identical to the reference) -------------- */
/* AdjGraph.from_pattern (sparse.py:102-111): symmetrized pattern of the
 * nonzero-valued entries, diagonal removed, rows sorted. Two-call protocol:
 * pass indices_out == NULL to get nnz_out, then call again with buffers. */
int mfh_adjacency(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
                  int64_t *indptr_out, int64_t *indices_out, int64_t *nnz_out);

/* nested_dissection (ordering.py:157-208) */
int mfh_nd_create(int64_t n, const int64_t *g_indptr, const int64_t *g_indices, int64_t leaf_size,
                  mfh_nd **out);
int mfh_nd_sizes(const mfh_nd *nd, int64_t *n_nodes, int64_t *n_vertices, int64_t *root);
int mfh_nd_fetch(const mfh_nd *nd, int64_t *perm, int64_t *vptr, int64_t *verts, int64_t *left,
                 int64_t *right, int64_t *parent);
void mfh_nd_free(mfh_nd *nd);

/* build_elimination_tree (ordering.py:264-312). A given as CSR (rows sorted). */
int mfh_etree_create(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
                     const mfh_nd *nd, mfh_etree **out);
int mfh_etree_sizes(const mfh_etree *t, int64_t *n_nodes, int64_t *n_piv_total,
                    int64_t *n_frontal_total, int64_t *root);
int mfh_etree_fetch(const mfh_etree *t, int64_t *post_order, int64_t *piv_ptr, int64_t *piv,
                    int64_t *fr_ptr, int64_t *fr, int64_t *parent);
/* The CALLER's elimination tree (replaces passing the reference's
 * EliminationTree, ordering.py:238-261, to mf_factorize, multifrontal.py:459),
 * flattened: permutation (old -> new), n_nodes nodes, root, parent (-1 at the
 * root), children in node.children order (child_ptr / child), post order, and
 * per node the pivot ids (a contiguous run) and sorted frontal ids, all in the
 * permuted numbering. Validated (permutation, tree shape, post order children
 * first, pivots covering 0..n-1 once); a frontal id at or below its node's
 * pivots raises the reference's "node {id}: frontal index below the pivot
 * block" (ordering.py:303-306). Nothing is recomputed: the factorization uses
 * exactly this tree. */
int mfh_etree_from_arrays(int64_t n, const int64_t *perm, int64_t n_nodes, int64_t root, const int64_t *parent,
                          const int64_t *child_ptr, const int64_t *child, int64_t n_post,
                          const int64_t *post_order, const int64_t *piv_ptr, const int64_t *piv,
                          const int64_t *fr_ptr, const int64_t *fr, mfh_etree **out);
void mfh_etree_free(mfh_etree *t);

/* ---- numeric factorization (mf_factorize, multifrontal.py:459-530) --------- */
/* A is the ORIGINAL matrix as CSR (rows sorted, no duplicates); the etree
 * carries the permutation. The numeric work runs on the context's GPU. */
int mfh_factorize(mfh_ctx *ctx, const mfh_etree *t, int64_t n, const int64_t *indptr,
                  const int64_t *indices, const double *values, int mode, const mfh_params *params,
                  mfh_factor **out);
/* ---- subtree-sharded factorization (one process per GPU) ------- */
/* The exchange callback sums `count` doubles of the DEVICE buffer `d_buf` in
 * place over all ranks (an all-reduce SUM). Work producing d_buf is enqueued on
 * the context stream (mfh_ctx_info); the callback must order its collective
 * after it (NCCL on that stream) or synchronize (host staging). Every slot is
 * written by exactly one rank and is zero elsewhere, so the sum is exact.
 * Returns 0 on success. */
typedef int (*mfh_exchange_fn)(void *user, double *d_buf, int64_t count);
/* Point-to-point transfers of DEVICE buffers posted as one group (NCCL group
 * semantics: no ordering among the ops): op i sends (is_send[i] = 1) or
 * receives counts[i] doubles of bufs[i] to / from rank peers[i]. Ordered after
 * the work on the context stream, like mfh_exchange_fn. Returns 0 on success. */
typedef int (*mfh_p2p_fn)(void *user, int64_t nops, double *const *bufs, const int64_t *counts,
                          const int32_t *peers, const int32_t *is_send);
typedef struct {
  const int32_t *owner; /* per etree node id: the rank that factors it (subtrees whole) */
  int rank;             /* this rank */
  mfh_exchange_fn exchange;
  void *user;
  /* optional: with it, a child update crossing ranks travels in its own
   * compressed form (the update HODLR's leaves and blocks, W, V^T: the
   * reference's UpdateRep, hodlr.py:429-470) from the child's owner to the
   * parent's owner only; without it, every cut update is densified and
   * all-reduced to every rank */
  mfh_p2p_fn p2p;
} mfh_shard_t;
/* mf_factorize over the nodes this rank owns, in global height order. After
 * each height with a child -> parent edge between ranks, the children's
 * updates go to the parents' owners: serialized in their compressed form and
 * sent point to point (shard->p2p), or densified (bitwise the per-child term
 * of the parent's sampler) and all-reduced (no p2p callback). The factor's stats
 * cover the whole tree (per-node accounting exchanged). mfh_apply /
 * mfh_gmres on it run the global apply levels on this rank's fronts, with the
 * contribution buffer (upward) and x (downward) exchanged at the level
 * boundaries where a dependency crosses ranks and x exchanged at the end:
 * every rank gets the full solution, bitwise equal to the single-GPU one. */
int mfh_factorize_sharded(mfh_ctx *ctx, const mfh_etree *t, int64_t n, const int64_t *indptr,
                          const int64_t *indices, const double *values, int mode, const mfh_params *params,
                          const mfh_shard_t *shard, mfh_factor **out);
int mfh_factor_stats(const mfh_factor *f, mfh_stats_t *out);
/* Per-node solve operators of MfFactorization.node_factors (DenseNodeFactor /
 * StructuredNodeFactor, multifrontal.py:160-216) on host vectors: op 0 =
 * pp_solve (y = F_pp^{-1} x, n_pivot -> n_pivot), 1 = apply_pf (y = F_pf x,
 * frontal -> n_pivot), 2 = apply_fp (y = F_fp x, n_pivot -> frontal). */
int mfh_node_op(mfh_factor *f, int64_t node, int op, const double *x, double *y);
int mfh_factor_records(const mfh_factor *f, mfh_record_t *out /* n_records */);
int mfh_factor_timing(const mfh_factor *f, mfh_timing_t *out);
/* integer parity record of every compressed block, in the reference's visiting
 * order: per block (node_id, m, n, |I|, |J|, rank, dense_fallback) and the
 * pivot sequences row_perm[:rank], col_perm[:rank] concatenated. Two-call. */
int mfh_factor_blocks(const mfh_factor *f, int64_t *n_blocks, int64_t *n_perm, int64_t *info /*7*n*/,
                      int64_t *perms /* 2*n_perm */, double *ratios /* n */);
void mfh_factor_free(mfh_factor *f);

/* ---- preconditioner apply (mf_solve, multifrontal.py:533-560) ------------- */
/* b, x: host (on_device == 0) or device (on_device == 1) arrays of n*nrhs,
 * column-major per right-hand side. */
int mfh_apply(mfh_factor *f, const double *b, double *x, int64_t nrhs, int on_device);
/* time `reps` device-resident applies; returns mean ms and algorithmic bytes/apply */
int mfh_apply_bench(mfh_factor *f, int64_t reps, double *ms_per_apply, double *bytes_per_apply);

/* ---- sparse operator (spmv, sparse.py:277-284; LinearOperator.from_matrix) */
int mfh_csr_create(mfh_ctx *ctx, int64_t n_rows, int64_t n_cols, const int64_t *indptr,
                   const int64_t *indices, const double *values, mfh_csr **out);
int mfh_spmv(mfh_csr *A, const double *x, double *y, int on_device);
/* time `reps` device-resident SpMVs back to back (CUDA events); mean ms */
int mfh_spmv_bench(mfh_csr *A, int64_t reps, double *ms_per_spmv);
void mfh_csr_free(mfh_csr *A);
/* dense operator (LinearOperator.from_matrix(ndarray), krylov.py:32-33): row-major n x n */
int mfh_dense_create(mfh_ctx *ctx, int64_t n, const double *values, mfh_csr **out);

/* ---- GMRES (gmres, krylov.py:68-161) -------------------------------------- */
/* host callback operator: y = op(x), both host arrays of length n */
typedef void (*mfh_host_op)(void *user, const double *x, double *y);

typedef struct {
  mfh_csr *A;          /* device operator, or NULL to use A_cb */
  mfh_host_op A_cb;
  void *A_user;
  mfh_factor *M;       /* device preconditioner (accelerated-mf), or NULL */
  mfh_host_op M_cb;    /* host preconditioner callback when M == NULL; NULL = identity */
  void *M_user;
  mfh_precond *P;      /* device baseline preconditioner (diagonal / ILUT); takes precedence over M */
} mfh_gmres_ops;

/* b, x host arrays of n; hist receives up to max_iter residuals (or 1 when
 * ||b|| == 0). Returns iterations, converged, n_hist. */
int mfh_gmres(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, const double *b, double *x,
              double tol, int64_t max_iter, int64_t restart, double *hist, int64_t *n_hist,
              int64_t *iterations, int *converged);
/* same, b/x already on the device (x overwritten); used by the benchmark */
int mfh_gmres_device(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, const double *d_b,
                     double *d_x, double tol, int64_t max_iter, int64_t restart, double *hist,
                     int64_t *n_hist, int64_t *iterations, int *converged);
/* GMRES distributed over the ranks of a sharded factorization:
 * every rank holds the rows and vector entries of the pivots it owns; SpMV
 * reads the entries of other ranks it couples to (ancestor separators) from an
 * all-reduced halo buffer; Gram-Schmidt is classical and repeated once (CGS2:
 * one all-reduce of the j + 1 dot products per pass), norms all-reduced, the
 * preconditioner is the sharded apply. All through the factor's exchange
 * callback. Collective: every rank calls it with the same ORIGINAL matrix
 * (CSR), the same host b, and receives the whole solution in x. Iteration
 * counts agree with mfh_gmres to +-1 (CGS2 instead of MGS). */
int mfh_gmres_sharded(mfh_factor *F, int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
                      const double *b, double *x, double tol, int64_t max_iter, int64_t restart, double *hist,
                      int64_t *n_hist, int64_t *iterations, int *converged);
/* Several right-hand sides with one device factorization (BASELINE C5: 8
 * RHS). Replaces the caller's loop of gmres(A, b_r, M) calls (the reference
 * has no batched entry; krylov.py:68-161 per column): right-hand side r is
 * b + r*n, its solution x + r*n; groups of up to eight run in lockstep and
 * share each preconditioner apply, so the factor is read once per Arnoldi step
 * for the group. Per right-hand side: history row r of hist (hist_cap
 * entries), n_hist[r], iterations[r], converged[r]. The shared apply runs
 * on the FP64 tensor cores (several vectors per matrix element), the
 * one-vector apply of mfh_gmres as a warp per row: a column equals its
 * mfh_gmres solve to rounding (iteration counts within one); a column never
 * depends on the other columns of its group. ops->A and ops->M must be device
 * objects (no host callbacks). Host arrays / device arrays respectively. */
int mfh_gmres_batched(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, int64_t nrhs, const double *b,
                      double *x, double tol, int64_t max_iter, int64_t restart, double *hist,
                      int64_t hist_cap, int64_t *n_hist, int64_t *iterations, int *converged);
int mfh_gmres_batched_device(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, int64_t nrhs,
                             const double *d_b, double *d_x, double tol, int64_t max_iter,
                             int64_t restart, double *hist, int64_t hist_cap, int64_t *n_hist,
                             int64_t *iterations, int *converged);

/* ---- baseline preconditioners (krylov.py:164-204) ------------------------ */
/* diagonal_preconditioner (krylov.py:164-170): y = x / diag(A); A as CSR.
 * ValueError "zero diagonal entry at index i". */
int mfh_precond_diag_create(mfh_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                            const double *values, mfh_precond **out);
/* ilut (krylov.py:173-204): dual-threshold ILU, per-row fill cap
 * floor(k nnz / n) + 1, drop_tol relative to the row 2-norm; the factors are
 * bit-identical to the reference's ilut_factor (_core.pyx:145-269), computed on
 * the host (a row-sequential recurrence). The apply (two triangular solves,
 * _core.pyx:272-305) runs on the GPU by level sets, one graph replay, and is
 * bit-identical to the reference's scalar loops. A as CSR with sorted rows.
 * ValueError texts: "k must be at least 1", "drop_tol must be nonnegative",
 * "ILUT zero pivot in row i". */
int mfh_precond_ilut_create(mfh_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                            const double *values, int64_t k, double drop_tol, mfh_precond **out);
/* the ILUT factorization alone, on the host (no context): two-call protocol,
 * li == NULL returns lnz / unz only (ilut_factor, _core.pyx:145-269) */
int mfh_ilut_factor(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values, int64_t k,
                    double drop_tol, int64_t *lnz, int64_t *unz, int64_t *lp, int64_t *li, double *lv,
                    int64_t *up, int64_t *ui, double *uv);
/* stored reals (Preconditioner.stored_reals), nnz of L and U, triangular-solve levels */
int mfh_precond_info(const mfh_precond *P, int64_t *stored_reals, int64_t *lnz, int64_t *unz, int64_t *levels);
/* the ILUT factors (lp n+1, li/lv lnz; up n+1, ui/uv unz), as ilut_factor returns them */
int mfh_precond_ilut_factors(const mfh_precond *P, int64_t *lp, int64_t *li, double *lv, int64_t *up,
                             int64_t *ui, double *uv);
int mfh_precond_apply(mfh_precond *P, const double *b, double *x, int on_device);
void mfh_precond_free(mfh_precond *P);

/* ---- kernel plugin (full_pivot_lu, _kernels/__init__.py:25; _core.pyx:23) - */
/* Batched complete-pivot LU on the device. Blocks are row-major, packed at
 * offs[i] (doubles) in `blocks` (host); shapes ms[i] x ns[i]. Outputs: lu
 * overwritten in place in the reference's (physically permuted) layout;
 * row_perm packed at sum(ms[:i]), col_perm at sum(ns[:i]); ranks; next
 * ratios; status 1 = PivotMonotonicityError with err[3i..3i+2] = (k, pivot,
 * previous pivot), for the exact reference message. */
int mfh_full_pivot_lu_batched(mfh_ctx *ctx, int64_t batch, const int64_t *offs, const int64_t *ms,
                              const int64_t *ns, double *blocks, int64_t total, double eps,
                              const int64_t *max_ranks, int64_t *row_perm, int64_t *col_perm,
                              int64_t *ranks, double *ratios, int64_t *status, double *err);

/* ---- test hook (no reference counterpart) ------------------------------ */
/* The factorization's explicit-inverse dispatch (register-tiled Gauss-Jordan
 * for n <= 128, blocked LU + triangular inverses above) on a host batch of
 * square row-major blocks packed at offs[i]; blocks are overwritten with the
 * inverses; singular[i] = 1 where a pivot was zero or non-finite. */
int mfh_test_inverse_batched(mfh_ctx *ctx, int64_t batch, const int64_t *offs, const int64_t *ns,
                             double *blocks, int64_t total, int *singular);

/* The factorization's batched GEMM dispatch (DMMA tiles, identity strips,
 * split-K, cuBLAS for large plain GEMMs) on one host workspace: job q is
 * desc[9q..9q+8] = (m, n, k, A offset, B offset, C offset, lda, ldb, ldc) into
 * buf, C = alpha A B + beta C with (alpha, beta) = ab[2q], ab[2q+1]; an A or B
 * offset of -1 is the identity strip (leading dimension -1). split_k > 0
 * splits long k for <= 32-tile jobs into chunks of split_k (deterministic). */
int mfh_test_gemm_batched(mfh_ctx *ctx, int64_t batch, const int64_t *desc, const double *ab, double *buf,
                          int64_t total, int split_k);

/* The apply's batched GEMV (k_gemv_tc: rows in groups of 8 on the FP64 tensor
 * cores, 1..8 right-hand sides) on one host workspace: job q is
 * desc[16q..16q+15] = (m, k1, k2, y, y0, A1, lda1, x1, A2, lda2, x2, idx2, ys,
 * y0s, x1s, x2s) with offsets into buf (y0, A2, x2, idx2 = -1: none; idx2 is
 * an offset into idx) and (a1, a2) = ab[2q], ab[2q+1]:
 *   y[v][i] = (y0[v][i] or 0) + a1 A1[i,:] . x1[v] + a2 A2[i,:] . x2[v][idx2]. */
int mfh_test_gemv_batched(mfh_ctx *ctx, int64_t batch, const int64_t *desc, const double *ab, double *buf,
                          int64_t total, const int64_t *idx, int64_t nidx, int nv);

#ifdef __cplusplus
}
#endif
#endif /* MFH_H_ */
