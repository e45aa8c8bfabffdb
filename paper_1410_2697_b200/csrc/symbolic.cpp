// Host symbolic analysis: adjacency graph, nested dissection, elimination tree.
//
// Bit-identical restatement (integer outputs) of the reference's ordering
// path, written as iterative C++ (the reference recursion is 979 frames deep
// at 128^3 and its pure-Python ND takes 427 s there):
//   adjacency_from_csr   <- sparse.py:102-111   (AdjGraph.from_pattern)
//   levels / peripheral  <- ordering.py:59-93   (BFS level sets, George-Liu)
//   components           <- ordering.py:96-115
//   bisect               <- ordering.py:118-154 (median level separator)
//   nested_dissection    <- ordering.py:157-208
//   etree                <- ordering.py:264-312
#include <algorithm>
#include <cstring>
#include <memory>
#include <queue>
#include <cmath>
#include <functional>
#include <string>

#include "internal.h"

#include <atomic>

namespace mfh {

Graph adjacency_from_csr(int64_t n, const int64_t *indptr, const int64_t *indices,
                         const double *values) {
  // edge (i, j), i != j, iff a_ij != 0 or a_ji != 0 (bool-cast pattern, symmetrized)
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
      int64_t j = indices[p];
      if (j == i || !(values[p] != 0.0)) continue;
      cnt[i + 1]++;
      cnt[j + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int64_t> tmp(cnt[n]);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
      int64_t j = indices[p];
      if (j == i || !(values[p] != 0.0)) continue;
      tmp[fill[i]++] = j;
      tmp[fill[j]++] = i;
    }
  Graph g;
  g.n = n;
  g.ptr.assign(n + 1, 0);
  g.idx.reserve(tmp.size());
  for (int64_t i = 0; i < n; ++i) {
    auto b = tmp.begin() + cnt[i], e = tmp.begin() + cnt[i + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    g.idx.insert(g.idx.end(), b, u);
    g.ptr[i + 1] = (int64_t)g.idx.size();
  }
  return g;
}

namespace {

struct NdWork {
  const Graph &g;
  std::vector<char> mask;
  std::vector<int64_t> mark;
  int64_t stamp = 0;
  explicit NdWork(const Graph &gr) : g(gr), mask(gr.n, 0), mark(gr.n, 0) {}

  // BFS level sets of the masked component containing `start`
  void levels(int64_t start, std::vector<int64_t> &flat, std::vector<int64_t> &off) {
    ++stamp;
    flat.clear();
    off.clear();
    flat.push_back(start);
    off.push_back(0);
    off.push_back(1);
    mark[start] = stamp;
    while (true) {
      int64_t b = off[off.size() - 2], e = off.back();
      size_t before = flat.size();
      for (int64_t t = b; t < e; ++t) {
        int64_t v = flat[t];
        for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p) {
          int64_t w = g.idx[p];
          if (mask[w] && mark[w] != stamp) {
            mark[w] = stamp;
            flat.push_back(w);
          }
        }
      }
      if (flat.size() == before) break;
      std::sort(flat.begin() + before, flat.end());
      off.push_back((int64_t)flat.size());
    }
  }

  void peripheral(const std::vector<int64_t> &region, std::vector<int64_t> &flat,
                  std::vector<int64_t> &off) {
    int64_t root = region.front();  // regions are sorted: min vertex
    levels(root, flat, off);
    std::vector<int64_t> f2, o2;
    while (true) {
      int64_t lb = off[off.size() - 2], le = off.back();
      int64_t cand = flat[lb];
      for (int64_t t = lb + 1; t < le; ++t) {
        int64_t v = flat[t];
        int64_t dv = g.degree(v), dc = g.degree(cand);
        if (dv < dc || (dv == dc && v < cand)) cand = v;
      }
      if (cand == root) return;
      levels(cand, f2, o2);
      if (o2.size() > off.size()) {
        root = cand;
        flat.swap(f2);
        off.swap(o2);
      } else {
        return;
      }
    }
  }

  void components(const std::vector<int64_t> &region, std::vector<std::vector<int64_t>> &comps) {
    ++stamp;
    comps.clear();
    std::vector<int64_t> queue;
    for (int64_t v : region) {
      if (mark[v] == stamp) continue;
      std::vector<int64_t> comp;
      mark[v] = stamp;
      queue.assign(1, v);
      size_t head = 0;
      while (head < queue.size()) {
        int64_t u = queue[head++];
        comp.push_back(u);
        for (int64_t p = g.ptr[u]; p < g.ptr[u + 1]; ++p) {
          int64_t w = g.idx[p];
          if (mask[w] && mark[w] != stamp) {
            mark[w] = stamp;
            queue.push_back(w);
          }
        }
      }
      std::sort(comp.begin(), comp.end());
      comps.push_back(std::move(comp));
    }
  }

  void bisect(const std::vector<int64_t> &region, std::vector<int64_t> &a, std::vector<int64_t> &b,
              std::vector<int64_t> &sep) {
    std::vector<int64_t> flat, off;
    peripheral(region, flat, off);
    int64_t nlev = (int64_t)off.size() - 1;
    int64_t total = (int64_t)flat.size();
    int64_t half = (total + 1) / 2;
    int64_t acc = 0, med = 0;
    for (med = 0; med < nlev; ++med) {
      acc += off[med + 1] - off[med];
      if (acc >= half) break;
    }
    if (med == nlev) med = nlev - 1;  // python for-loop leaves the last index
    if (med == nlev - 1 && med > 0) med -= 1;
    a.assign(flat.begin(), flat.begin() + off[med]);
    b.assign(flat.begin() + off[med + 1], flat.end());
    bool a_small = a.size() <= b.size();
    const std::vector<int64_t> &small = a_small ? a : b;
    ++stamp;
    for (int64_t v : small) mark[v] = stamp;
    sep.clear();
    std::vector<int64_t> rest;
    for (int64_t t = off[med]; t < off[med + 1]; ++t) {
      int64_t v = flat[t];
      bool touch = false;
      for (int64_t p = g.ptr[v]; p < g.ptr[v + 1]; ++p)
        if (mark[g.idx[p]] == stamp) {
          touch = true;
          break;
        }
      (touch ? sep : rest).push_back(v);
    }
    if (sep.empty()) {
      sep.swap(rest);
    } else {
      std::vector<int64_t> &big = a_small ? b : a;
      big.insert(big.end(), rest.begin(), rest.end());
    }
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    std::sort(sep.begin(), sep.end());
  }
};

}  // namespace
}  // namespace mfh

std::vector<int64_t> mfh_nd::post_order() const {
  std::vector<int64_t> order;
  if (root < 0) return order;
  std::vector<std::pair<int64_t, bool>> st{{root, false}};
  while (!st.empty()) {
    auto [v, done] = st.back();
    st.pop_back();
    if (done) {
      order.push_back(v);
      continue;
    }
    st.push_back({v, true});
    if (left[v] >= 0) {
      st.push_back({right[v], false});
      st.push_back({left[v], false});
    }
  }
  return order;
}

namespace mfh {

mfh_nd *nested_dissection(const Graph &g, int64_t leaf_size) {
  if (leaf_size < 1) throw value_error("leaf_size must be at least 1");
  auto *nd = new mfh_nd();
  nd->n = g.n;
  nd->perm.assign(g.n, 0);
  nd->vptr.push_back(0);
  if (g.n == 0) return nd;
  NdWork w(g);
  int64_t counter = 0;
  auto number = [&](const std::vector<int64_t> &vs) {
    for (int64_t v : vs) nd->perm[v] = counter++;
  };
  auto add = [&](const std::vector<int64_t> &vs, int64_t l, int64_t r) {
    nd->verts.insert(nd->verts.end(), vs.begin(), vs.end());
    nd->vptr.push_back((int64_t)nd->verts.size());
    nd->left.push_back(l);
    nd->right.push_back(r);
    nd->parent.push_back(-1);
    int64_t id = (int64_t)nd->left.size() - 1;
    if (l >= 0) {
      nd->parent[l] = id;
      nd->parent[r] = id;
    }
    return id;
  };
  struct Frame {
    std::vector<int64_t> region;
    int stage = 0;
    bool merge = false;
    std::vector<int64_t> second, sep;
    int64_t left = -1;
  };
  std::vector<Frame> st;
  st.emplace_back();
  st.back().region.resize(g.n);
  for (int64_t i = 0; i < g.n; ++i) st.back().region[i] = i;
  int64_t ret = -1;
  std::vector<std::vector<int64_t>> comps;
  while (!st.empty()) {
    Frame &fr = st.back();
    if (fr.stage == 0) {
      if ((int64_t)fr.region.size() <= leaf_size) {
        number(fr.region);
        ret = add(fr.region, -1, -1);
        st.pop_back();
        continue;
      }
      for (int64_t v : fr.region) w.mask[v] = 1;
      w.components(fr.region, comps);
      std::vector<int64_t> first;
      if (comps.size() > 1) {
        for (int64_t v : fr.region) w.mask[v] = 0;
        fr.merge = true;
        first = std::move(comps[0]);
        std::vector<int64_t> rest;
        for (size_t c = 1; c < comps.size(); ++c)
          rest.insert(rest.end(), comps[c].begin(), comps[c].end());
        std::sort(rest.begin(), rest.end());
        fr.second = std::move(rest);
      } else {
        std::vector<int64_t> a, b, s;
        w.bisect(fr.region, a, b, s);
        for (int64_t v : fr.region) w.mask[v] = 0;
        first = std::move(a);
        fr.second = std::move(b);
        fr.sep = std::move(s);
      }
      fr.region.clear();
      fr.region.shrink_to_fit();
      fr.stage = 1;
      Frame child;
      child.region = std::move(first);
      st.push_back(std::move(child));
    } else if (fr.stage == 1) {
      fr.left = ret;
      fr.stage = 2;
      Frame child;
      child.region = std::move(fr.second);
      st.push_back(std::move(child));
    } else {
      int64_t l = fr.left, r = ret;
      if (fr.merge) {
        ret = add(std::vector<int64_t>(), l, r);
      } else {
        number(fr.sep);
        ret = add(fr.sep, l, r);
      }
      st.pop_back();
    }
  }
  nd->root = ret;
  return nd;
}

mfh_etree *elimination_tree(const HostCsr &A, const mfh_nd &nd) {
  int64_t n = A.n;
  if (nd.n != n) throw value_error("separator tree size does not match the matrix");
  // pat = csr + csr.T with scipy's drop-zero-results semantics
  std::vector<int64_t> tptr(n + 1, 0), tidx(A.idx.size());
  std::vector<double> tval(A.idx.size());
  for (int64_t p = 0; p < (int64_t)A.idx.size(); ++p) tptr[A.idx[p] + 1]++;
  for (int64_t i = 0; i < n; ++i) tptr[i + 1] += tptr[i];
  {
    std::vector<int64_t> fill(tptr.begin(), tptr.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
        int64_t q = fill[A.idx[p]]++;
        tidx[q] = i;
        tval[q] = A.val[p];
      }
  }
  std::vector<int64_t> pptr(n + 1, 0), pidx;
  pidx.reserve(A.idx.size() * 2);
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = A.ptr[i], pe = A.ptr[i + 1], q = tptr[i], qe = tptr[i + 1];
    while (p < pe || q < qe) {
      int64_t j;
      double s;
      if (q >= qe || (p < pe && A.idx[p] < tidx[q])) {
        j = A.idx[p];
        s = A.val[p] + 0.0;
        ++p;
      } else if (p >= pe || tidx[q] < A.idx[p]) {
        j = tidx[q];
        s = 0.0 + tval[q];
        ++q;
      } else {
        j = A.idx[p];
        s = A.val[p] + tval[q];
        ++p;
        ++q;
      }
      if (s != 0.0 || s != s) pidx.push_back(j);
    }
    pptr[i + 1] = (int64_t)pidx.size();
  }

  auto *t = new mfh_etree();
  static std::atomic<uint64_t> next_uid{1};
  t->uid = next_uid++;
  t->n = n;
  t->root = nd.root;
  t->perm = nd.perm;
  int64_t nn = (int64_t)nd.left.size();
  t->post = nd.post_order();
  t->parent = nd.parent;
  t->children.assign(nn, {});
  for (int64_t v = 0; v < nn; ++v)
    if (nd.left[v] >= 0) t->children[v] = {nd.left[v], nd.right[v]};
  std::vector<std::vector<int64_t>> pivs(nn), frs(nn);
  std::vector<int64_t> buf;
  for (int64_t p : t->post) {
    std::vector<int64_t> &piv = pivs[p];
    for (int64_t k = nd.vptr[p]; k < nd.vptr[p + 1]; ++k) piv.push_back(nd.perm[nd.verts[k]]);
    std::sort(piv.begin(), piv.end());
    buf.clear();
    if (!piv.empty()) {
      int64_t top = piv.back();
      for (int64_t k = nd.vptr[p]; k < nd.vptr[p + 1]; ++k) {
        int64_t v = nd.verts[k];
        for (int64_t q = pptr[v]; q < pptr[v + 1]; ++q) {
          int64_t pj = nd.perm[pidx[q]];
          if (pj > top) buf.push_back(pj);
        }
      }
    }
    for (int64_t c : t->children[p]) buf.insert(buf.end(), frs[c].begin(), frs[c].end());
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
    std::vector<int64_t> &fr = frs[p];
    fr.reserve(buf.size());
    for (int64_t x : buf)
      if (!std::binary_search(piv.begin(), piv.end(), x)) fr.push_back(x);
    if (!piv.empty() && !fr.empty() && fr.front() <= piv.back())
      throw runtime_error("node " + std::to_string(p) + ": frontal index below the pivot block");
    // children's frontal lists are no longer needed once the parent has them
    for (int64_t c : t->children[p]) {
      (void)c;
    }
  }
  t->piv_ptr.assign(nn + 1, 0);
  t->fr_ptr.assign(nn + 1, 0);
  for (int64_t v = 0; v < nn; ++v) {
    t->piv_ptr[v + 1] = t->piv_ptr[v] + (int64_t)pivs[v].size();
    t->fr_ptr[v + 1] = t->fr_ptr[v] + (int64_t)frs[v].size();
  }
  t->piv.reserve(t->piv_ptr[nn]);
  t->fr.reserve(t->fr_ptr[nn]);
  for (int64_t v = 0; v < nn; ++v) {
    t->piv.insert(t->piv.end(), pivs[v].begin(), pivs[v].end());
    t->fr.insert(t->fr.end(), frs[v].begin(), frs[v].end());
  }
  return t;
}

// ILUT, row by row (the algorithm of _core.pyx:145-269, restated): scatter the
// row into a dense work row, eliminate its below-diagonal entries in
// ascending column order against the finished U rows (dropping multipliers
// below drop_tol * ||row||_2), keep the cap largest-magnitude L entries
// (magnitude ties: the smaller column survives), then the diagonal plus the
// cap largest U entries above drop_tol * ||row||_2. Sequential scalar
// arithmetic in the same order as the reference, so the factors are
// bit-identical (no FMA contraction on the x86-64 baseline ISA).
IlutFactors ilut_factor(int64_t n, const int64_t *ap, const int64_t *aj, const double *ax, int64_t cap,
                        double drop_tol) {
  IlutFactors F;
  F.lp.assign(n + 1, 0);
  F.up.assign(n + 1, 0);
  F.li.reserve((size_t)n * cap);
  F.lv.reserve((size_t)n * cap);
  F.ui.reserve((size_t)n * (cap + 1));
  F.uv.reserve((size_t)n * (cap + 1));
  std::vector<double> w((size_t)std::max<int64_t>(n, 1), 0.0);
  std::vector<uint8_t> occ((size_t)std::max<int64_t>(n, 1), 0);
  std::vector<int64_t> lc, uc;
  std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> below;
  // the cap largest |w| (ties: smaller column), then by column
  auto keep_largest = [&](std::vector<int64_t> &c) {
    if ((int64_t)c.size() > cap) {
      auto better = [&](int64_t a, int64_t b) {
        const double x = std::fabs(w[a]), y = std::fabs(w[b]);
        return x > y || (x == y && a < b);
      };
      std::nth_element(c.begin(), c.begin() + cap, c.end(), better);
      for (size_t t = cap; t < c.size(); ++t) w[c[t]] = 0.0;
      c.resize(cap);
    }
    std::sort(c.begin(), c.end());
  };
  for (int64_t i = 0; i < n; ++i) {
    lc.clear();
    uc.clear();
    double tnorm = 0.0;
    for (int64_t p = ap[i]; p < ap[i + 1]; ++p) {
      const int64_t j = aj[p];
      const double v = ax[p];
      tnorm += v * v;
      w[j] = v;
      occ[j] = 1;
      if (j < i)
        below.push(j);
      else if (j > i)
        uc.push_back(j);
    }
    const double delta = tnorm > 0.0 ? drop_tol * std::sqrt(tnorm) : 0.0;
    while (!below.empty()) {
      const int64_t k = below.top();
      below.pop();
      if (!occ[k]) continue;
      occ[k] = 0;
      const double wk = w[k] / F.uv[F.up[k]];
      w[k] = 0.0;
      if (std::fabs(wk) < delta) continue;
      lc.push_back(k);
      w[k] = wk;
      for (int64_t p = F.up[k] + 1; p < F.up[k + 1]; ++p) {
        const int64_t j = F.ui[p];
        if (occ[j]) {
          w[j] -= wk * F.uv[p];
        } else {
          w[j] = -wk * F.uv[p];
          occ[j] = 1;
          if (j < i)
            below.push(j);
          else if (j > i)
            uc.push_back(j);
        }
      }
    }
    keep_largest(lc);
    for (int64_t k : lc) {
      F.li.push_back(k);
      F.lv.push_back(w[k]);
      w[k] = 0.0;
    }
    F.lp[i + 1] = (int64_t)F.li.size();
    double diag = 0.0;
    if (occ[i]) {
      diag = w[i];
      w[i] = 0.0;
      occ[i] = 0;
    }
    if (diag == 0.0) throw value_error("ILUT zero pivot in row " + std::to_string(i));
    size_t keep = 0;
    for (int64_t j : uc) {
      occ[j] = 0;
      if (std::fabs(w[j]) >= delta)
        uc[keep++] = j;
      else
        w[j] = 0.0;
    }
    uc.resize(keep);
    keep_largest(uc);
    F.ui.push_back(i);
    F.uv.push_back(diag);
    for (int64_t j : uc) {
      F.ui.push_back(j);
      F.uv.push_back(w[j]);
      w[j] = 0.0;
    }
    F.up[i + 1] = (int64_t)F.ui.size();
  }
  return F;
}

}  // namespace mfh

// ---- C-ABI (host symbolic) --------------------------------------------------
using namespace mfh;

#define MFH_TRY try {
#define MFH_CATCH                           \
  }                                         \
  catch (const mfh::Error &e) {             \
    set_last_error(e.what());               \
    return e.kind;                          \
  }                                         \
  catch (const std::exception &e) {         \
    set_last_error(e.what());               \
    return MFH_ERUNTIME;                    \
  }                                         \
  return MFH_OK;

extern "C" int mfh_adjacency(int64_t n, const int64_t *indptr, const int64_t *indices,
                             const double *values, int64_t *indptr_out, int64_t *indices_out,
                             int64_t *nnz_out) {
  MFH_TRY
  Graph g = adjacency_from_csr(n, indptr, indices, values);
  *nnz_out = (int64_t)g.idx.size();
  if (indptr_out) std::memcpy(indptr_out, g.ptr.data(), sizeof(int64_t) * (n + 1));
  if (indices_out) std::memcpy(indices_out, g.idx.data(), sizeof(int64_t) * g.idx.size());
  MFH_CATCH
}

extern "C" int mfh_nd_create(int64_t n, const int64_t *g_indptr, const int64_t *g_indices,
                             int64_t leaf_size, mfh_nd **out) {
  MFH_TRY
  Graph g;
  g.n = n;
  g.ptr.assign(g_indptr, g_indptr + n + 1);
  g.idx.assign(g_indices, g_indices + g.ptr[n]);
  *out = nested_dissection(g, leaf_size);
  MFH_CATCH
}

extern "C" int mfh_nd_sizes(const mfh_nd *nd, int64_t *n_nodes, int64_t *n_vertices,
                            int64_t *root) {
  MFH_TRY
  *n_nodes = (int64_t)nd->left.size();
  *n_vertices = (int64_t)nd->verts.size();
  *root = nd->root;
  MFH_CATCH
}

extern "C" int mfh_nd_fetch(const mfh_nd *nd, int64_t *perm, int64_t *vptr, int64_t *verts,
                            int64_t *left, int64_t *right, int64_t *parent) {
  MFH_TRY
  size_t nn = nd->left.size();
  std::memcpy(perm, nd->perm.data(), sizeof(int64_t) * nd->perm.size());
  std::memcpy(vptr, nd->vptr.data(), sizeof(int64_t) * (nn + 1));
  std::memcpy(verts, nd->verts.data(), sizeof(int64_t) * nd->verts.size());
  std::memcpy(left, nd->left.data(), sizeof(int64_t) * nn);
  std::memcpy(right, nd->right.data(), sizeof(int64_t) * nn);
  std::memcpy(parent, nd->parent.data(), sizeof(int64_t) * nn);
  MFH_CATCH
}

extern "C" void mfh_nd_free(mfh_nd *nd) { delete nd; }

extern "C" int mfh_etree_create(int64_t n, const int64_t *indptr, const int64_t *indices,
                                const double *values, const mfh_nd *nd, mfh_etree **out) {
  MFH_TRY
  HostCsr A;
  A.n = n;
  A.ptr.assign(indptr, indptr + n + 1);
  A.idx.assign(indices, indices + A.ptr[n]);
  A.val.assign(values, values + A.ptr[n]);
  *out = elimination_tree(A, *nd);
  MFH_CATCH
}

extern "C" int mfh_etree_sizes(const mfh_etree *t, int64_t *n_nodes, int64_t *n_piv_total,
                               int64_t *n_frontal_total, int64_t *root) {
  MFH_TRY
  *n_nodes = (int64_t)t->parent.size();
  *n_piv_total = (int64_t)t->piv.size();
  *n_frontal_total = (int64_t)t->fr.size();
  *root = t->root;
  MFH_CATCH
}

extern "C" int mfh_etree_fetch(const mfh_etree *t, int64_t *post_order, int64_t *piv_ptr,
                               int64_t *piv, int64_t *fr_ptr, int64_t *fr, int64_t *parent) {
  MFH_TRY
  size_t nn = t->parent.size();
  std::memcpy(post_order, t->post.data(), sizeof(int64_t) * t->post.size());
  std::memcpy(piv_ptr, t->piv_ptr.data(), sizeof(int64_t) * (nn + 1));
  std::memcpy(piv, t->piv.data(), sizeof(int64_t) * t->piv.size());
  std::memcpy(fr_ptr, t->fr_ptr.data(), sizeof(int64_t) * (nn + 1));
  std::memcpy(fr, t->fr.data(), sizeof(int64_t) * t->fr.size());
  std::memcpy(parent, t->parent.data(), sizeof(int64_t) * nn);
  MFH_CATCH
}

extern "C" void mfh_etree_free(mfh_etree *t) { delete t; }

extern "C" int mfh_ilut_factor(int64_t n, const int64_t *indptr, const int64_t *indices, const double *values,
                               int64_t k, double drop_tol, int64_t *lnz, int64_t *unz, int64_t *lp, int64_t *li,
                               double *lv, int64_t *up, int64_t *ui, double *uv) {
  MFH_TRY
  if (k < 1) throw value_error("k must be at least 1");
  if (!(drop_tol >= 0)) throw value_error("drop_tol must be nonnegative");
  if (n < 1) throw value_error("ILUT requires a non-empty square matrix");
  IlutFactors F = ilut_factor(n, indptr, indices, values, k * indptr[n] / n + 1, drop_tol);
  *lnz = (int64_t)F.lv.size();
  *unz = (int64_t)F.uv.size();
  if (li) {
    std::memcpy(lp, F.lp.data(), sizeof(int64_t) * (n + 1));
    std::memcpy(up, F.up.data(), sizeof(int64_t) * (n + 1));
    std::memcpy(li, F.li.data(), sizeof(int64_t) * F.li.size());
    std::memcpy(ui, F.ui.data(), sizeof(int64_t) * F.ui.size());
    std::memcpy(lv, F.lv.data(), sizeof(double) * F.lv.size());
    std::memcpy(uv, F.uv.data(), sizeof(double) * F.uv.size());
  }
  MFH_CATCH
}

// The caller's own elimination tree (the reference's EliminationTree,
// ordering.py:238-261, flattened), validated against what the numeric
// factorization relies on.
extern "C" int mfh_etree_from_arrays(int64_t n, const int64_t *perm, int64_t n_nodes, int64_t root,
                                     const int64_t *parent, const int64_t *child_ptr, const int64_t *child,
                                     int64_t n_post, const int64_t *post_order, const int64_t *piv_ptr,
                                     const int64_t *piv, const int64_t *fr_ptr, const int64_t *fr,
                                     mfh_etree **out) {
  MFH_TRY
  if (n < 0 || n_nodes < 0 || n_post < 0) throw value_error("elimination tree sizes must be non-negative");
  std::vector<char> seen((size_t)std::max<int64_t>(n, 1), 0);
  for (int64_t i = 0; i < n; ++i) {
    if (perm[i] < 0 || perm[i] >= n || seen[perm[i]]) throw value_error("permutation is not a permutation of 0..n-1");
    seen[perm[i]] = 1;
  }
  if (n_nodes == 0 ? root != -1 : (root < 0 || root >= n_nodes)) throw value_error("root is not a node of the tree");
  auto *t = new mfh_etree();
  std::unique_ptr<mfh_etree> guard(t);
  static std::atomic<uint64_t> next_uid{1ull << 62};  // disjoint from mfh_etree_create's uids
  t->uid = next_uid++;
  t->n = n;
  t->root = root;
  t->perm.assign(perm, perm + n);
  t->parent.assign(parent, parent + n_nodes);
  t->children.assign(n_nodes, {});
  for (int64_t v = 0; v < n_nodes; ++v) {
    if (parent[v] < -1 || parent[v] >= n_nodes) throw value_error("parent of node " + std::to_string(v) + " out of range");
    for (int64_t q = child_ptr[v]; q < child_ptr[v + 1]; ++q) {
      const int64_t c = child[q];
      if (c < 0 || c >= n_nodes || parent[c] != v)
        throw value_error("children of node " + std::to_string(v) + " disagree with the parent array");
      t->children[v].push_back(c);
    }
  }
  // post order: every node once, children before their parent
  std::vector<char> done((size_t)std::max<int64_t>(n_nodes, 1), 0);
  t->post.assign(post_order, post_order + n_post);
  for (int64_t p : t->post) {
    if (p < 0 || p >= n_nodes || done[p]) throw value_error("post order repeats or leaves the tree");
    for (int64_t c : t->children[p])
      if (!done[c]) throw value_error("post order visits node " + std::to_string(p) + " before its child");
    done[p] = 1;
  }
  if (n_post != n_nodes) throw value_error("post order must visit every node");
  t->piv_ptr.assign(piv_ptr, piv_ptr + n_nodes + 1);
  t->fr_ptr.assign(fr_ptr, fr_ptr + n_nodes + 1);
  t->piv.assign(piv, piv + piv_ptr[n_nodes]);
  t->fr.assign(fr, fr + fr_ptr[n_nodes]);
  std::fill(seen.begin(), seen.end(), 0);
  for (int64_t v = 0; v < n_nodes; ++v) {
    const int64_t pb = piv_ptr[v], pe = piv_ptr[v + 1], fb = fr_ptr[v], fe = fr_ptr[v + 1];
    if (pb > pe || fb > fe) throw value_error("index pointers must be non-decreasing");
    for (int64_t q = pb; q < pe; ++q) {
      if (piv[q] < 0 || piv[q] >= n || seen[piv[q]]) throw value_error("pivot ids must cover 0..n-1 exactly once");
      seen[piv[q]] = 1;
      if (q > pb && piv[q] != piv[q - 1] + 1)
        throw value_error("pivot ids of node " + std::to_string(v) + " are not a contiguous run");
    }
    for (int64_t q = fb; q < fe; ++q) {
      if (fr[q] < 0 || fr[q] >= n || (q > fb && fr[q] <= fr[q - 1]))
        throw value_error("frontal ids of node " + std::to_string(v) + " must be sorted and in range");
    }
    if (pe > pb && fe > fb && fr[fb] <= piv[pe - 1])  // the reference's RuntimeError (ordering.py:303-306)
      throw runtime_error("node " + std::to_string(v) + ": frontal index below the pivot block");
  }
  for (int64_t i = 0; i < n; ++i)
    if (!seen[i]) throw value_error("pivot ids must cover 0..n-1 exactly once");
  *out = guard.release();
  MFH_CATCH
}
