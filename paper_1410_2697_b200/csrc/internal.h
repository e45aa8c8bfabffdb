// Internal declarations shared by the host symbolic code and the CUDA engine.
#pragma once
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mfh.h"

namespace mfh {

// Exceptions carry the C-ABI error kind; the C entry points translate them.
struct Error : public std::runtime_error {
  int kind;
  Error(int k, const std::string &m) : std::runtime_error(m), kind(k) {}
};
inline Error value_error(const std::string &m) { return Error(MFH_EVALUE, m); }
inline Error runtime_error(const std::string &m) { return Error(MFH_ERUNTIME, m); }

void set_last_error(const std::string &m);

// Undirected graph in CSR, neighbours sorted, no self loops.
struct Graph {
  int64_t n = 0;
  std::vector<int64_t> ptr, idx;
  int64_t degree(int64_t v) const { return ptr[v + 1] - ptr[v]; }
};

// Host CSR of a square matrix (rows sorted, no duplicates).
struct HostCsr {
  int64_t n = 0;
  std::vector<int64_t> ptr, idx;
  std::vector<double> val;
};

Graph adjacency_from_csr(int64_t n, const int64_t *indptr, const int64_t *indices,
                         const double *values);

// Dual-threshold incomplete LU (ILUT) of a CSR matrix with sorted rows: the
// comparison-baseline preconditioner (krylov.py:173-204, _core.pyx:145-269).
// L is unit lower (diagonal not stored), U upper with the diagonal first in
// every row. Throws value_error("ILUT zero pivot in row i").
struct IlutFactors {
  std::vector<int64_t> lp, li, up, ui;
  std::vector<double> lv, uv;
};
IlutFactors ilut_factor(int64_t n, const int64_t *ap, const int64_t *aj, const double *ax, int64_t cap,
                        double drop_tol);

}  // namespace mfh

// Separator tree produced by nested dissection (ordering.py:19-56).
struct mfh_nd {
  int64_t n = 0;
  int64_t root = -1;
  std::vector<int64_t> perm;
  std::vector<int64_t> vptr, verts;  // per node vertex list (creation order ids)
  std::vector<int64_t> left, right, parent;
  std::vector<int64_t> post_order() const;
};

// Symbolic data derived from (pattern of A, permutation, zero pattern): the
// permuted CSR pattern of P A P^T with a value-gather map, and the BDLR graph.
struct mfh_symcache {
  uint64_t key = 0;
  bool valid = false;
  // exact validation of the cached pattern (no hashing of the whole pattern per call)
  std::vector<int64_t> pat_ptr, pat_idx, pat_zero;
  bool pat_accel = false;
  uint64_t gen = 0;  // process-unique generation (device copies are keyed by it)
  std::vector<int64_t> ap_ptr, src;  // src[r]: position in A's CSR values of Ap entry r
  std::vector<int> ap_col;
  mfh::Graph graph;
  bool has_graph = false;
};

// Extend-add index maps (multifrontal.py:270-280, 321-327) are symbolic: one
// flat array per tree, map of child c (post index) at [off[c], off[c] + parent nh)
struct mfh_mapcache {
  bool valid = false;
  std::vector<int> maps;
  std::vector<int64_t> off;  // per post index, -1 when the child passes no update
  // front id lists (pivots then frontal ids) of every node in post order, flat
  bool ids_valid = false;
  std::vector<int64_t> ids_flat, ids_off;
};

// Elimination tree in the permuted numbering (ordering.py:211-261).
struct mfh_etree {
  mutable mfh_symcache cache;
  mutable mfh_mapcache mapcache;
  uint64_t uid = 0;  // process-unique id (device-side caches are keyed by it)
  int64_t n = 0;
  int64_t root = -1;
  std::vector<int64_t> perm;
  std::vector<int64_t> post;               // node ids in post order
  std::vector<int64_t> piv_ptr, piv;       // pivot ids (sorted, contiguous run)
  std::vector<int64_t> fr_ptr, fr;         // frontal ids (sorted, > pivots)
  std::vector<int64_t> parent;             // -1 for root
  std::vector<std::vector<int64_t>> children;  // (left, right) order
};
