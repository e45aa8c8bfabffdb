// Batched FP64 kernels for the HODLR-multifrontal hot path (sm_100a).
//
// Everything is row-major with explicit leading dimensions, like the
// reference's C-ordered numpy arrays. Each kernel processes a whole batch of
// variable-size problems (one etree height, one HODLR level) per launch; the
// host builds the descriptor arrays.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

namespace mfh {

// Programmatic dependent launch (the apply graph's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): wait until the
// preceding grid has completed and its writes are visible, then let the next
// grid start launching its CTAs (they block in their own wait), so the
// launch latency between dependent levels overlaps the running level. Both
// are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


constexpr int kZeroPivotNum = 1;  // marker
#define MFH_ZERO_PIVOT_RATIO 1e-14
#define MFH_PIVOT_GROWTH_BOUND (2.0 * (1.0 + 1e-10))

// ---------------------------------------------------------------------------
// descriptors
// ---------------------------------------------------------------------------

// off-diagonal HODLR block as stored on the device
struct HBlk {
  const double *a;  // LR: col factor (m x rank, lda); dense: values (m x n, lda)
  const double *b;  // LR: row factor (rank x n, ldb)
  int rank, kind;   // kind 0 = low rank, 1 = dense
  int lda, ldb;
};

// heap-indexed HODLR node (children 2i+1, 2i+2); leaf != nullptr marks a leaf
struct HNode {
  const double *leaf;  // (hi-lo)^2 row-major
  HBlk up, lw;         // rows lo:mid x cols mid:hi ; rows mid:hi x cols lo:mid
};

// a serialized update HODLR (sharded exchange): the table's pointers are
// offsets in doubles from the payload base (0 = null); make them addresses
__global__ void k_rebase_hnodes(HNode *__restrict__ t, int n, const double *base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  HNode h = t[i];
  auto fix = [&](const double *&p) {
    if (p) p = base + (unsigned long long)p;
  };
  fix(h.leaf);
  fix(h.up.a);
  fix(h.up.b);
  fix(h.lw.a);
  fix(h.lw.b);
  t[i] = h;
}

// child update as seen by the parent's entry sampler
struct DChild {
  const int *to_child;  // parent front position -> child position or -1
  int kind;             // 0 dense (Schur block), 1 HODLR - W Vt
  int n;                // update dimension
  const double *dense;
  int ldd;
  const HNode *hn;
  const double *W;   // n x rw (ldw)
  const double *Vt;  // rw x n (ldv)
  int rw, ldw, ldv;
};

struct DFront {
  const long long *ids;  // front global ids (permuted numbering), sorted
  int nh, npv;
  int child_begin, child_end;
};

// one entry-sampling request F(rows, cols) -> out (nr x nc, ld)
struct SReq {
  int front;
  int nr, nc;
  const int *rows;  // front-local positions, or nullptr for r0..r0+nr-1
  const int *cols;
  int r0, c0;
  double *out;
  int ld;
};

struct GemmJob {  // C = alpha * A(m x k) * B(k x n) + beta * C
  const double *A;
  const double *B;
  double *C;
  int m, n, k, lda, ldb, ldc;
  double alpha, beta;
};

struct LuJob {  // partial-pivot LU (getrf) of n x n in place
  double *a;
  int n, lda;
  int *piv;
  int *flag;  // set to 1 when singular / non-finite (reference diag checks)
};


struct CopyJob {  // dst (m x n, ldd) = src (m x n, lds); optional row/col maps on src
  const double *src;
  double *dst;
  int m, n, lds, ldd;
  const int *rmap;
  const int *cmap;
};

struct PluJob {  // complete-pivot partial LU of an m x n core (logical permutation)
  double *a;
  int m, n, ld;
  int kmax;
  int *rowAt, *colAt;  // position -> original index (outputs: row_perm, col_perm)
  int *posR, *posC;    // original index -> position
  int *actR, *actC;    // active original indices
  int *idxR, *idxC;    // original index -> slot in the active list
  double *mult, *prow; // scratch m and n
  int *out;            // [0]=rank [1]=status [2]=err_k
  double *outd;        // [0]=ratio [1]=err_piv [2]=err_prev
};

struct SkelJob {  // skeleton factors from a factored core
  const double *lu;  // compact r x r (L unit-lower strict, U upper), ld r
  int r;
  const double *R;  // |I| x n panel, ldR
  int ldR, n;
  const int *rp;  // rowAt (first r entries used)
  const double *C;  // m x |J| panel, ldC
  int ldC, m;
  const int *cp;  // colAt
  double *row_out;  // r x n
  double *col_out;  // m x r
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ double blk_entry(const HBlk &b, int rr, int cc) {
  if (b.kind == 1) return b.a[(long long)rr * b.lda + cc];
  double s = 0.0;
  const double *a = b.a + (long long)rr * b.lda;
  const double *bb = b.b + cc;
  for (int t = 0; t < b.rank; ++t) s = fma(a[t], bb[(long long)t * b.ldb], s);
  return s;
}

// entry (r, c) of a HODLR matrix of size n at local positions (hodlr.py:386-426)
__device__ __forceinline__ double hodlr_entry(const HNode *hn, int n, int r, int c) {
  int idx = 0, lo = 0, hi = n;
  while (true) {
    const HNode &nd = hn[idx];
    if (nd.leaf) return nd.leaf[(long long)(r - lo) * (hi - lo) + (c - lo)];
    int mid = (lo + hi) >> 1;
    if (r < mid) {
      if (c < mid) {
        idx = 2 * idx + 1;
        hi = mid;
        continue;
      }
      return blk_entry(nd.up, r - lo, c - mid);
    }
    if (c >= mid) {
      idx = 2 * idx + 2;
      lo = mid;
      continue;
    }
    return blk_entry(nd.lw, r - mid, c - lo);
  }
}

__device__ __forceinline__ double seed_entry(const long long *Ap_ptr, const int *Ap_col,
                                             const double *Ap_val, long long gr, long long gc) {
  long long lo = Ap_ptr[gr], hi = Ap_ptr[gr + 1];
  int key = (int)gc;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    int v = Ap_col[mid];
    if (v < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < Ap_ptr[gr + 1] && Ap_col[lo] == key) return Ap_val[lo];
  return 0.0;
}

// ---------------------------------------------------------------------------
// extend-add sampler (multifrontal.py:313-350 + hodlr.py:386-463)
// value = seed(r,c) [+ child_1] [+ child_2] ... in node.children order;
// child value = HODLR entry - W[r,:] . V[c,:]
// ---------------------------------------------------------------------------
// a tile is SAMPLE_TR x SAMPLE_TC entries for a block of SAMPLE_TRB x SAMPLE_TC threads: a thread
// keeps its column (and the column's position in the first children) over SAMPLE_TR / SAMPLE_TRB
// rows, and the tile decode and descriptor loads are paid once per tile
constexpr int SAMPLE_TR = 64, SAMPLE_TRB = 8, SAMPLE_TC = 32;

// Tile t of a sampling batch: request rids[p] with tpre[p] <= t < tpre[p + 1]
// (the host sends the per-request tile prefix, not one descriptor per tile)
struct SampleTiles {
  const int *rids;
  const long long *tpre;
  int nr;
  long long ntiles;
};
__device__ __forceinline__ int2 sample_tile(const SampleTiles &T, long long t) {
  int lo = 0, hi = T.nr - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (T.tpre[mid] <= t)
      lo = mid;
    else
      hi = mid - 1;
  }
  return make_int2(T.rids[lo], (int)(t - T.tpre[lo]));
}

__global__ void __launch_bounds__(256, 6) k_sample(const SReq *__restrict__ reqs, SampleTiles tiles,
                         const DFront *__restrict__ fronts, const DChild *__restrict__ kids,
                         const long long *__restrict__ Ap_ptr, const int *__restrict__ Ap_col,
                         const double *__restrict__ Ap_val) {
  pdl_wait();
  pdl_trigger();
  for (long long t = blockIdx.x; t < tiles.ntiles; t += gridDim.x) {
    const int2 tl = sample_tile(tiles, t);
    const SReq rq = reqs[tl.x];
    const int tpr = (rq.nc + SAMPLE_TC - 1) / SAMPLE_TC;
    const int i0 = (tl.y / tpr) * SAMPLE_TR;
    const int j = (tl.y % tpr) * SAMPLE_TC + threadIdx.x;
    if (j >= rq.nc) continue;
    const int c = rq.cols ? rq.cols[j] : rq.c0 + j;
    const DFront F = fronts[rq.front];
    // the column's position in the first two children (most fronts have two)
    const int nch = F.child_end - F.child_begin;
    const int cc0 = nch > 0 ? kids[F.child_begin].to_child[c] : -1;
    const int cc1 = nch > 1 ? kids[F.child_begin + 1].to_child[c] : -1;
    const long long gc = F.ids[c];
    for (int ii = threadIdx.y; ii < SAMPLE_TR; ii += SAMPLE_TRB) {
      const int i = i0 + ii;
      if (i >= rq.nr) break;
      const int r = rq.rows ? rq.rows[i] : rq.r0 + i;
      double v = 0.0;
      if (r < F.npv || c < F.npv) v = seed_entry(Ap_ptr, Ap_col, Ap_val, F.ids[r], gc);
      for (int q = F.child_begin; q < F.child_end; ++q) {
        const DChild &ch = kids[q];
        const int cc = (q == F.child_begin) ? cc0 : (q == F.child_begin + 1 ? cc1 : ch.to_child[c]);
        if (cc < 0) continue;
        const int cr = ch.to_child[r];
        if (cr < 0) continue;
        double sub;
        if (ch.kind == 0) {
          sub = ch.dense[(long long)cr * ch.ldd + cc];
        } else {
          sub = hodlr_entry(ch.hn, ch.n, cr, cc);
          if (ch.rw) {
            double s = 0.0;
            const double *w = ch.W + (long long)cr * ch.ldw;
            for (int u = 0; u < ch.rw; ++u) s = fma(w[u], ch.Vt[(long long)u * ch.ldv + cc], s);
            sub = sub - s;
          }
        }
        v = v + sub;
      }
      rq.out[(long long)i * rq.ld + j] = v;
    }
  }
}

// dst = mask ? src : 0 (a select: no arithmetic on the dropped values)
__global__ void k_mask_select(const double *__restrict__ src, const int8_t *__restrict__ mask,
                              double *__restrict__ dst, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = mask[i] ? src[i] : 0.0;
}

// descend to the block holding (r, c), also returning the block's rectangle
// in HODLR-local coordinates (rows [rlo, rhi), cols [clo, chi)); nullptr for a leaf
__device__ __forceinline__ const HBlk *hodlr_locate_rect(const HNode *hn, int n, int r, int c, int &rlo, int &rhi,
                                                         int &clo, int &chi) {
  int idx = 0, lo = 0, hi = n;
  while (true) {
    const HNode &nd = hn[idx];
    if (nd.leaf) return nullptr;
    int mid = (lo + hi) >> 1;
    if (r < mid) {
      if (c < mid) {
        idx = 2 * idx + 1;
        hi = mid;
        continue;
      }
      rlo = lo, rhi = mid, clo = mid, chi = hi;
      return &nd.up;
    }
    if (c >= mid) {
      idx = 2 * idx + 2;
      lo = mid;
      continue;
    }
    rlo = mid, rhi = hi, clo = lo, chi = mid;
    return &nd.lw;
  }
}

// Register-blocked extend-add sampler for fronts whose children carry a
// low-rank update W Vt of meaningful rank: 64 x 64 tiles, 256 threads. The
// rank-r dot products run on the FP64 tensor cores (mma.sync m8n8k4): warp w
// owns a 16 x 32 sub-tile (two 8-row by four 8-column MMA tiles), the factors
// stream through shared memory in 16-wide chunks (next chunk prefetched into
// registers). An m8n8k4 FP64 MMA equals the k-ascending FMA chain bit for bit
// (scripts/probe/dmma_order.cu: 0 differences in 1.28M entries on B200), so
// per entry the arithmetic is exactly k_sample's: seed, then per child in
// order sub = (HODLR or dense entry) - (u-ascending FMA chain of W[cr,u]
// Vt[u,cc]), v = v + sub (the HODLR low-rank entry is itself a t-ascending
// FMA chain). The W Vt term always uses the MMA path, the HODLR term when the
// tile's child rows x cols rectangle lies inside one low-rank block.
constexpr int RB_T = 64, RB_K = 16, RB_LD = RB_T + 4;  // RB_LD: conflict-free fragment loads
constexpr size_t RB_DYN = sizeof(double) * RB_T * (RB_T + 1);

// thread entry (a, b), a in {0, 1}, b in 0..7: tile row / column
__device__ __forceinline__ int rb_row(int a, int wr, int g) { return 16 * wr + 8 * a + g; }
__device__ __forceinline__ int rb_col(int b, int wc, int q) { return 32 * wc + 8 * (b >> 1) + 2 * q + (b & 1); }

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// acc[a][b] = sum_u X[sx[row], u] * Y[u, sy[col]] (u ascending from 0) for the
// thread's entries; rows / cols with index -1 contribute zero
// cp.async (LDGSTS) 8-byte element copies into shared memory; src_size 0
// writes zeros (padding) without reading
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void rb_dot(double (&acc)[2][8], const double *__restrict__ X, int ldx, const int *sx,
                                       const double *__restrict__ Y, int ldy, const int *sy, int K,
                                       double (*Ws)[RB_LD], double (*Vs)[RB_LD], int tid, int wr, int wc, int g,
                                       int q) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  double pw[4], pv[4];
  auto fetch = [&](int u0) {
    const int kc = min(RB_K, K - u0);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int e = tid + 256 * m;
      const int row = e >> 4, k = e & 15;
      const int xr = sx[row];
      pw[m] = (xr >= 0 && k < kc) ? X[(long long)xr * ldx + u0 + k] : 0.0;
      const int k2 = e >> 6, col = e & 63;
      const int yc = sy[col];
      pv[m] = (yc >= 0 && k2 < kc) ? Y[(long long)(u0 + k2) * ldy + yc] : 0.0;
    }
  };
  fetch(0);
  for (int u0 = 0; u0 < K; u0 += RB_K) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int e = tid + 256 * m;
      Ws[e & 15][e >> 4] = pw[m];
      Vs[e >> 6][e & 63] = pv[m];
    }
    __syncthreads();
    if (u0 + RB_K < K) fetch(u0 + RB_K);  // in flight during the MMAs
    // full chunk: padded ranks are zeros in both operands and fma(0, 0, acc)
    // == acc, so the chain is unchanged
#pragma unroll
    for (int kb = 0; kb < RB_K / 4; ++kb) {
      double fa[2], fb[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) fa[a] = Ws[4 * kb + q][16 * wr + 8 * a + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = Vs[4 * kb + q][32 * wc + 8 * j + g];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[a][2 * j], acc[a][2 * j + 1], fa[a], fb[j]);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_sample_rb(const SReq *__restrict__ reqs, SampleTiles tiles,
                                                   const DFront *__restrict__ fronts,
                                                   const DChild *__restrict__ kids,
                                                   const long long *__restrict__ Ap_ptr,
                                                   const int *__restrict__ Ap_col,
                                                   const double *__restrict__ Ap_val) {
  pdl_wait();
  pdl_trigger();
  __shared__ double Ws[RB_K][RB_LD];
  __shared__ double Vs[RB_K][RB_LD];
  __shared__ int s_r[RB_T], s_c[RB_T], s_cr[RB_T], s_cc[RB_T], s_br[RB_T], s_bc[RB_T];
  __shared__ const HBlk *s_blk;
  __shared__ int s_rlo, s_clo;
  extern __shared__ double rb_dyn[];  // running entry values s_v[RB_T][RB_T + 1] (keeps registers for the dots)
  double(*s_v)[RB_T + 1] = reinterpret_cast<double(*)[RB_T + 1]>(rb_dyn);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1, g = lane >> 2, q = lane & 3;
  for (long long t = blockIdx.x; t < tiles.ntiles; t += gridDim.x) {
    const int2 tl = sample_tile(tiles, t);
    const SReq rq = reqs[tl.x];
    const int tpr = (rq.nc + RB_T - 1) / RB_T;
    const int bi = (tl.y / tpr) * RB_T, bj = (tl.y % tpr) * RB_T;
    const DFront F = fronts[rq.front];
    if (tid < RB_T) {
      int i = bi + tid;
      s_r[tid] = i < rq.nr ? (rq.rows ? rq.rows[i] : rq.r0 + i) : -1;
    } else if (tid < 2 * RB_T) {
      int j = bj + tid - RB_T;
      s_c[tid - RB_T] = j < rq.nc ? (rq.cols ? rq.cols[j] : rq.c0 + j) : -1;
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int ra = rb_row(a, wr, g), cb = rb_col(b, wc, q);
        const int r = s_r[ra], c = s_c[cb];
        s_v[ra][cb] = (r >= 0 && c >= 0 && (r < F.npv || c < F.npv))
                          ? seed_entry(Ap_ptr, Ap_col, Ap_val, F.ids[r], F.ids[c])
                          : 0.0;
      }
    for (int qq = F.child_begin; qq < F.child_end; ++qq) {
      const DChild &ch = kids[qq];
      if (tid < RB_T) {
        int r = s_r[tid];
        s_cr[tid] = r >= 0 ? ch.to_child[r] : -1;
      } else if (tid < 2 * RB_T) {
        int c = s_c[tid - RB_T];
        s_cc[tid - RB_T] = c >= 0 ? ch.to_child[c] : -1;
      }
      __syncthreads();
      bool uni = false;
      if (ch.kind == 1) {
        // does the tile's child rectangle sit inside one low-rank block?
        if (tid < 32) {
          int rmin = 0x7fffffff, rmax = -1, cmin = 0x7fffffff, cmax = -1;
          for (int e = tid; e < RB_T; e += 32) {
            int x = s_cr[e], y = s_cc[e];
            if (x >= 0) rmin = min(rmin, x), rmax = max(rmax, x);
            if (y >= 0) cmin = min(cmin, y), cmax = max(cmax, y);
          }
          for (int o = 16; o > 0; o >>= 1) {
            rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
            rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
            cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
            cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
          }
          if (tid == 0) {
            const HBlk *blk = nullptr;
            if (rmax >= 0 && cmax >= 0) {
              int rlo, rhi, clo, chi;
              blk = hodlr_locate_rect(ch.hn, ch.n, rmin, cmin, rlo, rhi, clo, chi);
              if (blk && !(blk->kind == 0 && blk->rank > 0 && rmax < rhi && cmax < chi)) blk = nullptr;
              s_rlo = rlo;
              s_clo = clo;
            }
            s_blk = blk;
          }
        }
        __syncthreads();
        uni = s_blk != nullptr;
      }
      double sub[2][8];
      if (uni) {
        const HBlk B = *s_blk;
        if (tid < RB_T) {
          int x = s_cr[tid];
          s_br[tid] = x >= 0 ? x - s_rlo : -1;
        } else if (tid < 2 * RB_T) {
          int y = s_cc[tid - RB_T];
          s_bc[tid - RB_T] = y >= 0 ? y - s_clo : -1;
        }
        __syncthreads();
        rb_dot(sub, B.a, B.lda, s_br, B.b, B.ldb, s_bc, B.rank, Ws, Vs, tid, wr, wc, g, q);
      } else {
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            const int cr = s_cr[rb_row(a, wr, g)], cc = s_cc[rb_col(b, wc, q)];
            double x = 0.0;
            if (cr >= 0 && cc >= 0)
              x = ch.kind == 0 ? ch.dense[(long long)cr * ch.ldd + cc] : hodlr_entry(ch.hn, ch.n, cr, cc);
            sub[a][b] = x;
          }
      }
      if (ch.kind == 1 && ch.rw) {
        double acc[2][8];
        rb_dot(acc, ch.W, ch.ldw, s_cr, ch.Vt, ch.ldv, s_cc, ch.rw, Ws, Vs, tid, wr, wc, g, q);
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) sub[a][b] = sub[a][b] - acc[a][b];
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const int ra = rb_row(a, wr, g), cb = rb_col(b, wc, q);
          if (s_cr[ra] >= 0 && s_cc[cb] >= 0) s_v[ra][cb] = s_v[ra][cb] + sub[a][b];
        }
      __syncthreads();  // s_cr / s_cc / s_blk are rewritten for the next child
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int ra = rb_row(a, wr, g), cb = rb_col(b, wc, q);
        const int i = bi + ra, j = bj + cb;
        if (i < rq.nr && j < rq.nc) rq.out[(long long)i * rq.ld + j] = s_v[ra][cb];
      }
    __syncthreads();  // s_r / s_c are rewritten for the next tile
  }
}

// ---------------------------------------------------------------------------
// batched 2-D copy / gather
// ---------------------------------------------------------------------------
__global__ void k_copy(const CopyJob *__restrict__ jobs, int njobs) {
  pdl_wait();
  pdl_trigger();
  const CopyJob J = jobs[blockIdx.y];
  long long total = (long long)J.m * J.n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / J.n), j = (int)(e % J.n);
    int si = J.rmap ? J.rmap[i] : i;
    int sj = J.cmap ? J.cmap[j] : j;
    J.dst[(long long)i * J.ldd + j] = J.src[(long long)si * J.lds + sj];
  }
}

// C = alpha X + beta C (m x n): a GEMM whose other operand is an identity
// (DenseBlock.as_factors' eye, stored as a strip with leading dimension -1).
// Same epilogue expression as k_gemm, and the identity product is exact there,
// so the result is the GEMM's bit for bit.
__global__ void k_axpby(const GemmJob *__restrict__ jobs, const int *__restrict__ which) {
  pdl_wait();
  pdl_trigger();
  const GemmJob J = jobs[blockIdx.y];
  const bool a_is_eye = which[blockIdx.y] == 0;
  const double *X = a_is_eye ? J.B : J.A;
  const long long ldx = a_is_eye ? J.ldb : J.lda;
  const long long total = (long long)J.m * J.n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / J.n), j = (int)(e % J.n);
    double *cp = J.C + (long long)i * J.ldc + j;
    const double v = J.alpha * X[(long long)i * ldx + j];
    *cp = (J.beta == 0.0) ? v : J.beta * (*cp) + v;
  }
}

// identity in an m x m block (ld)
__global__ void k_identity(double *const *__restrict__ ptrs, const int *__restrict__ dims,
                           const int *__restrict__ lds) {
  pdl_wait();
  pdl_trigger();
  double *p = ptrs[blockIdx.y];
  int m = dims[blockIdx.y], ld = lds[blockIdx.y];
  long long total = (long long)m * m;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / m), j = (int)(e % m);
    p[(long long)i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// vbatched GEMM, NN, row-major: 64x64 tiles, BK 16, 256 threads. The dot
// products run on the FP64 tensor cores (mma.sync m8n8k4, the sampler's
// fragment layout: warp w owns a 16 x 32 sub-tile); an m8n8k4 FP64 MMA equals
// the k-ascending FMA chain bit for bit (scripts/probe/dmma_order.cu), and the
// zero padding of a short last slab leaves the chain unchanged. The next k
// slab is prefetched into registers while the current one is multiplied.
// Deterministic split-K (off by default, see run_gemm): each split tile writes
// its partial (valid rows/columns only) to a workspace slot, and k_gemm_reduce
// sums the partials in split order 0..S-1 and applies alpha/beta.
// ---------------------------------------------------------------------------
constexpr int GEMM_BM = 64, GEMM_BN = 64, GEMM_BK = 16;

struct GemmTile {
  int job, mt, nt, k0, k1;
  int ws;  // split-K: workspace slot of this partial, -1 = write C directly
};

struct GemmSplit {  // one split output tile: partials ws .. ws+ns-1
  int job, mt, nt, ws, ns;
};

constexpr int GEMM_STG = 3;  // cp.async stages of (A slab, B slab)
constexpr size_t GEMM_DYN = sizeof(double) * GEMM_STG * 2 * GEMM_BK * RB_LD;
__global__ void __launch_bounds__(256) k_gemm(const GemmJob *__restrict__ jobs,
                                              const GemmTile *__restrict__ tiles, int ntiles,
                                              double *__restrict__ ws) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double gemm_stg[];  // GEMM_STG x (As[GEMM_BK][RB_LD], Bs[GEMM_BK][RB_LD])
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1, g = lane >> 2, q = lane & 3;
  auto Ast = [&](int sidx) { return reinterpret_cast<double(*)[RB_LD]>(gemm_stg + (size_t)sidx * 2 * GEMM_BK * RB_LD); };
  auto Bst = [&](int sidx) {
    return reinterpret_cast<double(*)[RB_LD]>(gemm_stg + (size_t)sidx * 2 * GEMM_BK * RB_LD + GEMM_BK * RB_LD);
  };
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const GemmTile tl = tiles[t];
    const GemmJob J = jobs[tl.job];
    const int m0 = tl.mt * GEMM_BM, n0 = tl.nt * GEMM_BN;
    const int k1 = tl.k1;
    double acc[2][8];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
    const int nsl = tl.k0 < k1 ? (k1 - tl.k0 + GEMM_BK - 1) / GEMM_BK : 0;
    // slab c gathered straight into stage c % GEMM_STG (zeros outside the job)
    auto issue = [&](int c) {
      if (c < nsl) {
        const int k0 = tl.k0 + c * GEMM_BK;
        double(*As)[RB_LD] = Ast(c % GEMM_STG);
        double(*Bs)[RB_LD] = Bst(c % GEMM_STG);
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int e = tid + 256 * m;
          const int mm = e >> 4, kk = e & 15;  // A: 64 rows x 16 k
          const int gm = m0 + mm, gk = k0 + kk;
          const bool oka = gm < J.m && gk < k1;
          cp_async8(&As[kk][mm], oka ? J.A + (long long)gm * J.lda + gk : J.A, oka);
          const int k2 = e >> 6, nn = e & 63;  // B: 16 k x 64 cols
          const int gk2 = k0 + k2, gn = n0 + nn;
          const bool okb = gk2 < k1 && gn < J.n;
          cp_async8(&Bs[k2][nn], okb ? J.B + (long long)gk2 * J.ldb + gn : J.B, okb);
        }
      }
      cp_async_commit();
    };
    issue(0);
    issue(1);
    for (int c = 0; c < nsl; ++c) {
      cp_async_wait<1>();
      __syncthreads();  // slab c visible to all; slab c - 1's stage no longer read
      issue(c + 2);
      double(*As)[RB_LD] = Ast(c % GEMM_STG);
      double(*Bs)[RB_LD] = Bst(c % GEMM_STG);
#pragma unroll
      for (int kb = 0; kb < GEMM_BK / 4; ++kb) {
        double fa[2], fb[4];
#pragma unroll
        for (int a = 0; a < 2; ++a) fa[a] = As[4 * kb + q][16 * wr + 8 * a + g];
#pragma unroll
        for (int j = 0; j < 4; ++j) fb[j] = Bs[4 * kb + q][32 * wc + 8 * j + g];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[a][2 * j], acc[a][2 * j + 1], fa[a], fb[j]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // stages free for the next tile
    double *part = tl.ws >= 0 ? ws + (long long)tl.ws * (GEMM_BM * GEMM_BN) : nullptr;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int r = rb_row(a, wr, g), gm = m0 + r;
      if (gm >= J.m) continue;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int c = rb_col(b, wc, q), gn = n0 + c;
        if (gn >= J.n) continue;
        if (part) {
          part[r * GEMM_BN + c] = acc[a][b];
          continue;
        }
        double *cp = J.C + (long long)gm * J.ldc + gn;
        double v = J.alpha * acc[a][b];
        *cp = (J.beta == 0.0) ? v : J.beta * (*cp) + v;
      }
    }
  }
}

// split-K epilogue: C = alpha * (((p0 + p1) + p2) + ...) + beta * C
__global__ void __launch_bounds__(256) k_gemm_reduce(const GemmJob *__restrict__ jobs,
                                                     const GemmSplit *__restrict__ splits,
                                                     const double *__restrict__ ws) {
  pdl_wait();
  pdl_trigger();
  const GemmSplit sp = splits[blockIdx.x];
  const GemmJob J = jobs[sp.job];
  const int m0 = sp.mt * GEMM_BM, n0 = sp.nt * GEMM_BN;
  const double *w0 = ws + (long long)sp.ws * (GEMM_BM * GEMM_BN);
  for (int e = threadIdx.x; e < GEMM_BM * GEMM_BN; e += blockDim.x) {
    int r = e >> 6, c = e & 63;
    int gm = m0 + r, gn = n0 + c;
    if (gm >= J.m || gn >= J.n) continue;
    double v = w0[e];
    for (int s = 1; s < sp.ns; ++s) v += w0[(long long)s * (GEMM_BM * GEMM_BN) + e];
    double *cp = J.C + (long long)gm * J.ldc + gn;
    v = J.alpha * v;
    *cp = (J.beta == 0.0) ? v : J.beta * (*cp) + v;
  }
}

// ---------------------------------------------------------------------------
// block reductions
// ---------------------------------------------------------------------------
struct MaxLoc {
  double v;
  long long key;
};

__device__ __forceinline__ bool better(double v, long long k, double bv, long long bk) {
  return v > bv || (v == bv && k < bk);
}

__device__ __forceinline__ MaxLoc block_maxloc(double v, long long key, MaxLoc *sh) {
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, v, o);
    long long ok = __shfl_down_sync(0xffffffffu, key, o);
    if (better(ov, ok, v, key)) {
      v = ov;
      key = ok;
    }
  }
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) sh[w] = MaxLoc{v, key};
  __syncthreads();
  if (w == 0) {
    MaxLoc m = lane < nw ? sh[lane] : MaxLoc{-2.0, 0x7fffffffffffffffLL};
    v = m.v;
    key = m.key;
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, v, o);
      long long ok = __shfl_down_sync(0xffffffffu, key, o);
      if (better(ov, ok, v, key)) {
        v = ov;
        key = ok;
      }
    }
    if (lane == 0) sh[32] = MaxLoc{v, key};
  }
  __syncthreads();
  MaxLoc r = sh[32];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// complete-pivot partial LU with rank cut (_core.pyx:23-86): shared state and
// the cross-CTA candidate buffers; the kernels are the v2 family below.
// ---------------------------------------------------------------------------
struct PluState {
  int done, bi, bj, ar, ac, rank, status, errk;
  double akk, u11, prev, ratio, errpiv, errprev;
};

constexpr int GRID_MAX = 160;  // CTAs per cooperative group (>= SM count)

struct GridScratch {
  MaxLoc *best;    // 2 x G
  double *cand;    // 2 x G x nmax
  int nmax;
  unsigned *bar;   // group barrier arrival counter (zeroed before the launch); nullptr = whole-grid sync
  unsigned epoch;  // barriers this CTA has passed (thread 0's copy)
};

// Barrier over the G CTAs of one group of a cooperative launch (all CTAs are
// co-resident). The counter only grows: barrier e is complete once it reaches
// G * e, so an arrival is one acq_rel atomic and the wait an acquire-load
// spin (the release publishes the CTA's candidate slot and row, ordered
// after the block's writes by the __syncthreads; the acquire makes the other
// CTAs' visible before the closing __syncthreads).
__device__ __forceinline__ void group_barrier(GridScratch *gs, int G) {
  if (!gs->bar) {
    cg::this_grid().sync();
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (unsigned)G * ++gs->epoch;
    unsigned v;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(gs->bar) : "memory");
    unsigned cur = v + 1;
    while ((int)(cur - target) < 0)  // not the last arriver: wait for the rest
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gs->bar) : "memory");
  }
  __syncthreads();
}

// ===========================================================================
// v2 complete-pivot LU kernels: the reference's physical column swaps are
// reproduced, so the trailing columns of step k are the contiguous range
// (k, n) and the tie-break key of a candidate is (row position) * n + column
// -- no per-entry indirection. Rows are physically swapped in the single-CTA
// kernel and kept logical (owned rows + position table) in the distributed
// kernels. One reduction barrier, one decision barrier and one pivot-row
// barrier per step.
// ===========================================================================
__device__ __forceinline__ MaxLoc reduce_to0(double v, long long key, MaxLoc *red) {
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, v, o);
    long long ok = __shfl_down_sync(0xffffffffu, key, o);
    if (better(ov, ok, v, key)) {
      v = ov;
      key = ok;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) red[w] = MaxLoc{v, key};
  __syncthreads();
  MaxLoc r{-2.0, 0x7fffffffffffffffLL};
  if (w == 0) {
    r = lane < nw ? red[lane] : MaxLoc{-2.0, 0x7fffffffffffffffLL};
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, r.v, o);
      long long ok = __shfl_down_sync(0xffffffffu, r.key, o);
      if (better(ov, ok, r.v, r.key)) {
        r.v = ov;
        r.key = ok;
      }
    }
  }
  return r;  // valid in thread 0
}

// stop/continue rule of _core.pyx:49-62; returns true when elimination stops
__device__ __forceinline__ bool plu_stop(PluState &st, int k, int kmax, double eps, double piv) {
  if (k == 0) {
    st.u11 = piv;
    if (piv == 0.0) {
      st.rank = 0;
      st.ratio = 0.0;
      return true;
    }
  } else {
    if (piv > st.prev * MFH_PIVOT_GROWTH_BOUND) {
      st.status = 1;
      st.errk = k;
      st.errpiv = piv;
      st.errprev = st.prev;
      return true;
    }
    double ratio = piv / st.u11;
    if (ratio < eps || piv <= MFH_ZERO_PIVOT_RATIO * st.u11) {
      st.rank = k;
      st.ratio = ratio;
      return true;
    }
  }
  if (k == kmax) {
    st.rank = kmax;
    st.ratio = piv / st.u11;
    return true;
  }
  return false;
}

__device__ __forceinline__ void plu_out(const PluJob &J, const PluState &st) {
  J.out[0] = st.rank;
  J.out[1] = st.status;
  J.out[2] = st.errk;
  J.outd[0] = st.ratio;
  J.outd[1] = st.errpiv;
  J.outd[2] = st.errprev;
}

// One trailing-update row of the complete-pivot LU: a[j] -= l * p[j] for the
// lane's columns j = j0 + lane + 32 t, t ascending, with f(v, j) called in
// that order (the caller's strict '>' running max keeps the first max). Four
// columns' loads are issued before their arithmetic: the same per-element
// operations, more bytes in flight per lane.
template <class F>
__device__ __forceinline__ void plu_row_update(double *__restrict__ row, const double *__restrict__ prow, double l,
                                               int j0, int n, int lane, F &&f) {
  int j = j0 + lane;
  for (; j + 96 < n; j += 128) {
    const double a0 = row[j], a1 = row[j + 32], a2 = row[j + 64], a3 = row[j + 96];
    const double p0 = prow[j], p1 = prow[j + 32], p2 = prow[j + 64], p3 = prow[j + 96];
    const double v0 = __dsub_rn(a0, __dmul_rn(l, p0)), v1 = __dsub_rn(a1, __dmul_rn(l, p1));
    const double v2 = __dsub_rn(a2, __dmul_rn(l, p2)), v3 = __dsub_rn(a3, __dmul_rn(l, p3));
    row[j] = v0;
    row[j + 32] = v1;
    row[j + 64] = v2;
    row[j + 96] = v3;
    f(v0, j);
    f(v1, j + 32);
    f(v2, j + 64);
    f(v3, j + 96);
  }
  for (; j < n; j += 32) {
    const double v = __dsub_rn(row[j], __dmul_rn(l, prow[j]));
    row[j] = v;
    f(v, j);
  }
}

template <bool SMEM_CORE, int NT = 512>
__global__ void __launch_bounds__(NT) k_plu_cta2(const PluJob *__restrict__ jobs, const int *__restrict__ ids,
                                                 double eps) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) char dsm[];
  __shared__ MaxLoc red[32];
  __shared__ PluState st;
  const PluJob J = jobs[ids[blockIdx.x]];
  const int m = J.m, n = J.n, tid = threadIdx.x, nt = blockDim.x;
  double *a = J.a;
  int ld = J.ld;
  char *base = dsm;
  if (SMEM_CORE) {
    double *sa = (double *)dsm;
    for (long long e = tid; e < (long long)m * n; e += nt) sa[e] = J.a[(e / n) * J.ld + (e % n)];
    a = sa;
    ld = n;
    base = dsm + sizeof(double) * (size_t)m * n;
  }
  int *rowAt = (int *)base, *colAt = rowAt + m;
  for (int i = tid; i < m; i += nt) rowAt[i] = i;
  for (int j = tid; j < n; j += nt) colAt[j] = j;
  if (tid == 0) {
    st = PluState{};
  }
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  double bv = -1.0;
  long long bk = 0x7fffffffffffffffLL;
  __syncthreads();
  for (int i = warp; i < m; i += nw) {
    const double *row = a + (long long)i * ld;
    for (int j = lane; j < n; j += 32) {
      double v = fabs(row[j]);
      if (better(v, (long long)i * n + j, bv, bk)) {
        bv = v;
        bk = (long long)i * n + j;
      }
    }
  }
  const int kmin = min(m, n);
  for (int k = 0; k < kmin; ++k) {
    MaxLoc best = reduce_to0(bv, bk, red);
    if (tid == 0) {
      double piv = best.v;
      int bi = k, bj = k;
      if (best.key != 0x7fffffffffffffffLL) {
        bi = (int)(best.key / n);
        bj = (int)(best.key % n);
      } else {
        piv = -1.0;
      }
      bool stop = plu_stop(st, k, J.kmax, eps, piv);
      st.done = stop ? 1 : 0;
      if (!stop) {
        st.bi = bi;
        st.bj = bj;
        st.akk = a[(long long)bi * ld + bj];
        st.prev = fabs(st.akk);
        st.rank = k + 1;
        int t = rowAt[k];
        rowAt[k] = rowAt[bi];
        rowAt[bi] = t;
        t = colAt[k];
        colAt[k] = colAt[bj];
        colAt[bj] = t;
      }
    }
    __syncthreads();
    if (st.done) break;
    const int bi = st.bi, bj = st.bj;
    const double akk = st.akk;
    // physical swaps: rows k <-> bi and columns k <-> bj in one conflict-free pass
    if (bi != k)
      for (int t = tid; t < n; t += nt) {
        if (t == k || t == bj) continue;
        double x = a[(long long)k * ld + t];
        a[(long long)k * ld + t] = a[(long long)bi * ld + t];
        a[(long long)bi * ld + t] = x;
      }
    if (bj != k)
      for (int t = tid; t < m; t += nt) {
        if (t == k || t == bi) continue;
        double x = a[(long long)t * ld + k];
        a[(long long)t * ld + k] = a[(long long)t * ld + bj];
        a[(long long)t * ld + bj] = x;
      }
    if (tid == 0) {
      double okk = a[(long long)k * ld + k], okb = a[(long long)k * ld + bj];
      double oik = a[(long long)bi * ld + k], oib = a[(long long)bi * ld + bj];
      a[(long long)k * ld + k] = oib;
      a[(long long)k * ld + bj] = oik;
      a[(long long)bi * ld + k] = okb;
      a[(long long)bi * ld + bj] = okk;
    }
    __syncthreads();
    bv = -1.0;
    // each thread scans rows ascending and, within a row, columns ascending:
    // scan order = key order, so a strict '>' keeps the first (lowest-key) max
    int bi_ = -1, bj_ = 0;
    const double *prow = a + (long long)k * ld;
    for (int i = k + 1 + warp; i < m; i += nw) {
      double *row = a + (long long)i * ld;
      const double l = row[k] / akk;
      __syncwarp();
      if (lane == 0) row[k] = l;
      plu_row_update(row, prow, l, k + 1, n, lane, [&](double v, int j) {
        const double av = fabs(v);
        if (av > bv) {
          bv = av;
          bi_ = i;
          bj_ = j;
        }
      });
    }
    bk = bi_ >= 0 ? (long long)bi_ * n + bj_ : 0x7fffffffffffffffLL;
  }
  __syncthreads();
  if (SMEM_CORE)
    for (long long e = tid; e < (long long)m * n; e += nt) J.a[(e / n) * J.ld + (e % n)] = a[e];
  // physically permuted rows: the caller's row_perm is rowAt; report the layout as
  // "rows already permuted" by storing rowAt and flagging it in out[3]
  for (int i = tid; i < m; i += nt) J.rowAt[i] = rowAt[i];
  for (int j = tid; j < n; j += nt) J.colAt[j] = colAt[j];
  if (tid == 0) {
    plu_out(J, st);
    J.out[3] = 1;  // rows physically permuted
  }
}

// distributed over CTAs (cluster: DSMEM; grid: global candidates): original
// row i lives in CTA (i % G) at local row (i / G); columns are physical
template <bool GRID, bool ROWS_SMEM>
__device__ __forceinline__ void plu_dist_body(const PluJob &J, double eps, int G, int g, char *dsm, MaxLoc *red,
                                              PluState &st, int &s_nact, cg::cluster_group *clp,
                                              MaxLoc *slot, GridScratch *gs, int *s_win) {
  const int m = J.m, n = J.n, tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const int nl_max = (m + G - 1) / G;
  const int nl = (m - g + G - 1) / G;
  double *rows = (double *)dsm;  // ROWS_SMEM: nl_max x n
  double *prow = ROWS_SMEM ? rows + (size_t)nl_max * n : rows;
  int *rowAt = (int *)(prow + n);
  int *colAt = rowAt + m;
  int *posRl = colAt + n;
  int *actRl = posRl + nl_max;
  int *idxRl = actRl + nl_max;
  int *defer = idxRl + nl_max;  // deferred column swap of this CTA's last pivot row: (li, k, bj)
  auto row_ptr = [&](int li) -> double * {
    return ROWS_SMEM ? rows + (size_t)li * n : J.a + (long long)(li * G + g) * J.ld;
  };
  if (ROWS_SMEM)
    for (long long e = tid; e < (long long)nl * n; e += nt) {
      int li = (int)(e / n), j = (int)(e % n);
      rows[e] = J.a[(long long)(li * G + g) * J.ld + j];
    }
  for (int i = tid; i < m; i += nt) rowAt[i] = i;
  for (int j = tid; j < n; j += nt) colAt[j] = j;
  for (int li = tid; li < nl; li += nt) {
    posRl[li] = li * G + g;
    actRl[li] = li;
    idxRl[li] = li;
  }
  if (tid == 0) {
    st = PluState{};
    s_nact = nl;
    defer[0] = -1;
  }
  __syncthreads();
  double bv = -1.0;
  long long bk = 0x7fffffffffffffffLL;
  for (int li = warp; li < nl; li += nw) {
    const double *row = row_ptr(li);
    const long long pr = (long long)(li * G + g) * n;
    for (int j = lane; j < n; j += 32) {
      double v = fabs(row[j]);
      if (better(v, pr + j, bv, bk)) {
        bv = v;
        bk = pr + j;
      }
    }
  }
  const int kmin = min(m, n);
  for (int k = 0; k < kmin; ++k) {
    const int par = k & 1;
    MaxLoc best = reduce_to0(bv, bk, red);
    if (GRID) {
      // publish the candidate and its row (pre-swap values of this step)
      __shared__ int s_cand;
      if (tid == 0) {
        gs->best[par * G + g] = best;
        s_cand = best.key == 0x7fffffffffffffffLL ? -1 : rowAt[(int)(best.key / n)] / G;
      }
      __syncthreads();
      if (s_cand >= 0) {
        const double *src = row_ptr(s_cand);
        double *dst = gs->cand + ((size_t)par * G + g) * gs->nmax;
        for (int j = tid; j < n; j += nt) dst[j] = src[j];
      }
      group_barrier(gs, G);
    } else {
      if (tid == 0) slot[par] = best;
      clp->sync();
    }
    if (tid < 32) {
      MaxLoc gb{-2.0, 0x7fffffffffffffffLL};
      int who = -1;
      if (GRID) {
        // all loads first (independent), then the in-lane reduction
        MaxLoc o[GRID_MAX / 32];
#pragma unroll
        for (int u = 0; u < GRID_MAX / 32; ++u) {
          int q = lane + 32 * u;
          o[u] = q < G ? gs->best[par * G + q] : MaxLoc{-2.0, 0x7fffffffffffffffLL};
        }
#pragma unroll
        for (int u = 0; u < GRID_MAX / 32; ++u)
          if (better(o[u].v, o[u].key, gb.v, gb.key)) {
            gb = o[u];
            who = lane + 32 * u;
          }
      } else if (lane < G) {
        gb = *clp->map_shared_rank(&slot[par], lane);
        who = lane;
      }
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, gb.v, o);
        long long ok = __shfl_down_sync(0xffffffffu, gb.key, o);
        int ow = __shfl_down_sync(0xffffffffu, who, o);
        if (better(ov, ok, gb.v, gb.key)) {
          gb.v = ov;
          gb.key = ok;
          who = ow;
        }
      }
      if (tid == 0) {
        // previous deferred pivot-row swap (nobody reads that row any more)
        if (!GRID && defer[0] >= 0) {
          double *r = row_ptr(defer[0]);
          double x = r[defer[1]];
          r[defer[1]] = r[defer[2]];
          r[defer[2]] = x;
          defer[0] = -1;
        }
        double piv = gb.v;
        int pr = k, bj = k;
        if (gb.key != 0x7fffffffffffffffLL) {
          pr = (int)(gb.key / n);
          bj = (int)(gb.key % n);
        } else {
          piv = -1.0;
        }
        if (pr < 0 || pr >= m || bj < 0 || bj >= n) {  // defensive: corrupt candidate
          st.status = 2;
          piv = -1.0;
          pr = k;
          bj = k;
        }
        bool stop = st.status == 2 || plu_stop(st, k, J.kmax, eps, piv);
        st.done = stop ? 1 : 0;
        if (!stop) {
          const int bi = rowAt[pr], ak = rowAt[k];
          const int owner = bi % G;
          rowAt[k] = bi;
          rowAt[pr] = ak;
          if (bi % G == g) {
            int li = bi / G;
            posRl[li] = k;
            int s2 = idxRl[li], l2 = actRl[s_nact - 1];
            actRl[s2] = l2;
            idxRl[l2] = s2;
            idxRl[li] = 0x7fffffff;  // inactive
            s_nact -= 1;
            if (!GRID) {
              defer[0] = li;
              defer[1] = k;
              defer[2] = bj;
            }
          }
          if (ak % G == g && ak != bi) posRl[ak / G] = pr;
          int t = colAt[k];
          colAt[k] = colAt[bj];
          colAt[bj] = t;
          const double *orow;
          if (GRID)
            orow = gs->cand + ((size_t)par * G + who) * gs->nmax;
          else
            orow = ROWS_SMEM ? clp->map_shared_rank(rows, owner) + (size_t)(bi / G) * n : J.a + (long long)bi * J.ld;
          st.akk = orow[bj];
          st.prev = fabs(st.akk);
          st.rank = k + 1;
          st.bi = bi;
          st.bj = bj;
          *s_win = owner;
          (void)who;
        }
      }
    }
    __syncthreads();
    if (st.done) break;
    const int bi = st.bi, bj = st.bj, na = s_nact;
    const double akk = st.akk;
    // pivot row at physical columns after this step's swap: prow[j] = orow[j], prow[bj] = orow[k]
    {
      const double *orow;
      if (GRID) {
        // the winner CTA published bi's row (keys are unique: winner = owner)
        orow = gs->cand + ((size_t)par * G + (bi % G)) * gs->nmax;
      } else {
        orow = ROWS_SMEM ? clp->map_shared_rank(rows, bi % G) + (size_t)(bi / G) * n : J.a + (long long)bi * J.ld;
      }
      for (int j = k + 1 + tid; j < n; j += nt) prow[j] = (j == bj) ? orow[k] : orow[j];
    }
    // inactive owned rows (earlier pivots): physical column swap k <-> bj
    if (bj != k)
      for (int li = tid; li < nl; li += nt) {
        if (idxRl[li] != 0x7fffffff) continue;  // still active (handled below)
        if (!GRID && li * G + g == bi) continue;  // current pivot row: deferred (peers read it)
        double *r = row_ptr(li);
        double x = r[k];
        r[k] = r[bj];
        r[bj] = x;
      }
    __syncthreads();
    bv = -1.0;
    bk = 0x7fffffffffffffffLL;
    for (int q = warp; q < na; q += nw) {
      const int li = actRl[q];
      double *row = row_ptr(li);
      const double ok_ = row[k], ob = row[bj];
      const double l = ob / akk;
      __syncwarp();
      if (lane == 0) {
        row[k] = l;
        if (bj != k) row[bj] = ok_;  // the physical column swap, before the sweep
      }
      __syncwarp();
      const long long rk = (long long)posRl[li] * n;
      // within one row the lane's columns ascend, so key order = scan order:
      // a strict '>' with the column index is exact; the (value, key) merge
      // with the thread's best happens once per row
      double rbv = -1.0;
      int rj = 0x7fffffff;
      plu_row_update(row, prow, l, k + 1, n, lane, [&](double v, int j) {
        const double av = fabs(v);
        if (av > rbv) {
          rbv = av;
          rj = j;
        }
      });
      if (rj != 0x7fffffff && better(rbv, rk + rj, bv, bk)) {
        bv = rbv;
        bk = rk + rj;
      }
    }
  }
  __syncthreads();
  if (tid == 0 && !GRID && defer[0] >= 0) {
    double *r = row_ptr(defer[0]);
    double x = r[defer[1]];
    r[defer[1]] = r[defer[2]];
    r[defer[2]] = x;
  }
  __syncthreads();
  if (ROWS_SMEM)
    for (long long e = tid; e < (long long)nl * n; e += nt) {
      int li = (int)(e / n), j = (int)(e % n);
      J.a[(long long)(li * G + g) * J.ld + j] = rows[e];
    }
  if (g == 0) {
    for (int i = tid; i < m; i += nt) J.rowAt[i] = rowAt[i];
    for (int j = tid; j < n; j += nt) J.colAt[j] = colAt[j];
    if (tid == 0) {
      plu_out(J, st);
      J.out[3] = 0;  // rows logical: row p of the factor is original row rowAt[p]
    }
  }
}

__host__ __device__ inline size_t plu_dist_bytes(int m, int n, int G, bool rows_smem) {
  size_t nl = (size_t)((m + G - 1) / G);
  size_t b = sizeof(double) * ((rows_smem ? nl * (size_t)n : 0) + (size_t)n);
  b += sizeof(int) * ((size_t)m + (size_t)n + 3 * nl + 4);
  return (b + 15) & ~size_t(15);
}


// ---------------------------------------------------------------------------
// Cluster complete-pivot LU, one cluster barrier per step (rows in DSMEM)
//   * every CTA publishes its best candidate (|v|, key, signed v, local row);
//     after the cluster barrier EVERY warp reduces the G slots itself, so all
//     threads know the pivot without a broadcast
//   * the stop / rank state (plu_stop) is evaluated identically in every
//     thread's registers
//   * rows are dealt round-robin (original row i -> CTA i % G, local i / G), so
//     the pivot's original row is (local row, CTA); each row's logical position
//     is kept by the warp that updates it; active rows carry a flag instead of
//     a compacted list
//   * the column swap k <-> bj is fused into the update for active rows;
//     pivoted rows receive all their later swaps in one pass at the end
// Same arithmetic and the same (|v|, row-major key) first-max rule as
// k_plu_cta2 / plu_dist_body: bit-identical factors, pivots, rank, ratio.
// ---------------------------------------------------------------------------
struct PluCand {
  double v, sv;
  long long key;
  int li;
};
__device__ __forceinline__ PluCand cand_none() { return PluCand{-1.0, 0.0, 0x7fffffffffffffffLL, -1}; }
// warp argmax under better(): max |v| (NaN and "none" never win), then the
// lowest key, with hardware redux on 32-bit halves of a monotone encoding;
// every lane returns the winner (payload broadcast from the winning lane)
__device__ __forceinline__ PluCand warp_best(PluCand c, int &who) {
  const unsigned long long u = (c.v >= 0.0) ? (unsigned long long)__double_as_longlong(c.v) + 1ull : 0ull;
  const unsigned uh = (unsigned)(u >> 32), ul = (unsigned)u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, uh);
  const unsigned ml = __reduce_max_sync(0xffffffffu, uh == mh ? ul : 0u);
  const bool top = uh == mh && ul == ml;
  const unsigned long long key = (unsigned long long)c.key;
  const unsigned kh = (unsigned)(key >> 32), kl = (unsigned)key;
  const unsigned mkh = __reduce_min_sync(0xffffffffu, top ? kh : 0xffffffffu);
  const unsigned mkl = __reduce_min_sync(0xffffffffu, (top && kh == mkh) ? kl : 0xffffffffu);
  const unsigned win = __ballot_sync(0xffffffffu, top && kh == mkh && kl == mkl);
  const int src = __ffs(win) - 1;
  PluCand r;
  r.v = __shfl_sync(0xffffffffu, c.v, src);
  r.sv = __shfl_sync(0xffffffffu, c.sv, src);
  r.key = (long long)(((unsigned long long)mkh << 32) | mkl);
  r.li = __shfl_sync(0xffffffffu, c.li, src);
  who = __shfl_sync(0xffffffffu, who, src);
  return r;
}

__host__ __device__ inline size_t plu_cl3_bytes(int m, int n, int G) {
  size_t nl = (size_t)((m + G - 1) / G), kmin = (size_t)(m < n ? m : n);
  size_t b = sizeof(double) * (nl * (size_t)n + (size_t)n);
  b += sizeof(int) * (3 * nl + kmin + (size_t)n + 4);
  return (b + 15) & ~size_t(15);
}

template <int NT>
__global__ void __launch_bounds__(NT) k_plu_cluster3(const PluJob *__restrict__ jobs, const int *__restrict__ ids,
                                                     double eps) {
  extern __shared__ __align__(16) char dsm[];
  __shared__ PluCand red[NT / 32];
  __shared__ PluCand slots[2][16];  // [parity][source CTA]: pushed by every CTA before the barrier
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks(), g = (int)cl.block_rank();
  const PluJob J = jobs[ids[blockIdx.x / G]];
  const int m = J.m, n = J.n, tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const int nl_max = (m + G - 1) / G, nl = (m - g + G - 1) / G, kmin = min(m, n);
  double *rows = (double *)dsm;
  double *prow = rows + (size_t)nl_max * n;
  int *posR = (int *)(prow + n);
  int *act = posR + nl_max;
  int *pstep = act + nl_max;
  int *swp = pstep + nl_max;
  int *colAt = swp + kmin;
  for (long long e = tid; e < (long long)nl * n; e += nt) {
    int li = (int)(e / n), j = (int)(e % n);
    rows[e] = J.a[(long long)(li * G + g) * J.ld + j];
  }
  for (int li = tid; li < nl; li += nt) {
    posR[li] = li * G + g;
    act[li] = 1;
    pstep[li] = -1;
  }
  for (int j = tid; j < n; j += nt) colAt[j] = j;
  __syncthreads();
  // initial candidates: first max of |a| in row-major (original) order
  PluCand best = cand_none();
  for (int li = warp; li < nl; li += nw) {
    const double *row = rows + (size_t)li * n;
    double rbv = -1.0, rsv = 0.0;
    int rj = 0x7fffffff;
    for (int j = lane; j < n; j += 32) {
      double x = row[j], av = fabs(x);
      if (av > rbv) {
        rbv = av;
        rsv = x;
        rj = j;
      }
    }
    const long long key = (long long)(li * G + g) * n + rj;
    if (rj != 0x7fffffff && better(rbv, key, best.v, best.key)) best = PluCand{rbv, rsv, key, li};
  }
  PluState my{};
  int steps = 0;
  for (int k = 0; k < kmin; ++k) {
    const int par = k & 1;
    {
      int who = 0;
      PluCand c = warp_best(best, who);
      if (lane == 0) red[warp] = c;
      __syncthreads();
      if (warp == 0) {
        PluCand x = lane < nw ? red[lane] : cand_none();
        x = warp_best(x, who);
        // push this CTA's candidate into every CTA's local slot array
        if (lane < G) *cl.map_shared_rank(&slots[par][g], lane) = x;
      }
    }
    cl.sync();
    // every warp reduces the cluster's candidates from local shared memory
    int who = lane;
    PluCand gb = lane < G ? slots[par][lane] : cand_none();
    gb = warp_best(gb, who);
    double piv = gb.v;
    int pr = k, bj = k;
    if (gb.key != 0x7fffffffffffffffLL) {
      if (gb.key < 0xffffffffLL) {  // keys of cluster-sized cores fit 32 bits: cheap division
        const unsigned k32 = (unsigned)gb.key, q32 = k32 / (unsigned)n;
        pr = (int)q32;
        bj = (int)(k32 - q32 * (unsigned)n);
      } else {
        pr = (int)(gb.key / n);
        bj = (int)(gb.key % n);
      }
    } else {
      piv = -1.0;
    }
    if (plu_stop(my, k, J.kmax, eps, piv)) break;
    my.prev = fabs(gb.sv);
    my.rank = k + 1;
    steps = k + 1;
    const double akk = gb.sv;
    // pivot row (after this step's column swap) from the winner's DSMEM
    {
      const double *orow = cl.map_shared_rank(rows, who) + (size_t)gb.li * n;
      for (int j = k + 1 + tid; j < n; j += nt) prow[j] = (j == bj) ? orow[k] : orow[j];
    }
    if (tid == 0) {
      int t = colAt[k];
      colAt[k] = colAt[bj];
      colAt[bj] = t;
      swp[k] = bj;
      if (who == g) {
        act[gb.li] = 0;
        pstep[gb.li] = k;
        posR[gb.li] = k;
      }
    }
    __syncthreads();
    best = cand_none();
    for (int li = warp; li < nl; li += nw) {
      if (!act[li]) continue;
      double *row = rows + (size_t)li * n;
      const double ok_ = row[k], ob = row[bj];
      int pos = posR[li];
      const double l = ob / akk;
      __syncwarp();
      if (lane == 0) {
        row[k] = l;
        if (bj != k) row[bj] = ok_;
        if (pos == k) posR[li] = pr;  // the row at position k moves to the pivot's old position
      }
      __syncwarp();
      if (pos == k) pos = pr;
      double rbv = -1.0, rsv = 0.0;
      int rj = 0x7fffffff;
      plu_row_update(row, prow, l, k + 1, n, lane, [&](double v, int j) {
        const double av = fabs(v);
        if (av > rbv) {
          rbv = av;
          rsv = v;
          rj = j;
        }
      });
      const long long key = (long long)pos * n + rj;
      if (rj != 0x7fffffff && better(rbv, key, best.v, best.key)) best = PluCand{rbv, rsv, key, li};
    }
  }
  __syncthreads();
  // pivoted rows: the column swaps of their own step and every later step
  for (int li = tid; li < nl; li += nt) {
    const int p = pstep[li];
    if (p < 0) continue;
    double *row = rows + (size_t)li * n;
    for (int s2 = p; s2 < steps; ++s2) {
      const int b2 = swp[s2];
      if (b2 != s2) {
        double x = row[s2];
        row[s2] = row[b2];
        row[b2] = x;
      }
    }
  }
  __syncthreads();
  for (long long e = tid; e < (long long)nl * n; e += nt) {
    int li = (int)(e / n), j = (int)(e % n);
    J.a[(long long)(li * G + g) * J.ld + j] = rows[e];
  }
  for (int li = tid; li < nl; li += nt) J.rowAt[posR[li]] = li * G + g;
  if (g == 0) {
    for (int j = tid; j < n; j += nt) J.colAt[j] = colAt[j];
    if (tid == 0) {
      plu_out(J, my);
      J.out[3] = 0;  // rows logical: row p of the factor is original row rowAt[p]
    }
  }
  cl.sync();  // DSMEM lifetime: peers may still read this CTA's rows
}

// Grouped cooperative complete-pivot LU with the cluster kernel's per-step
// structure (k_plu_cluster3), candidates exchanged through global memory:
// every CTA publishes (|v|, key, signed v, local row) and its candidate row
// before the group barrier; after it EVERY warp reduces the group's
// candidates (L2 reads, __ldcg) and copies the winner's published row. The
// stop / rank state lives in every thread's registers, row positions with the
// warp that owns the row, pivoted rows get their column swaps at the end.
// Same arithmetic and first-max rule: bit-identical results.
__device__ __forceinline__ PluCand ldcg_cand(const PluCand *p) {
  PluCand c;
  c.v = __ldcg(&p->v);
  c.sv = __ldcg(&p->sv);
  c.key = __ldcg(&p->key);
  c.li = __ldcg(&p->li);
  return c;
}

__global__ void __launch_bounds__(512) k_plu_groups3(const PluJob *__restrict__ jobs, const int *__restrict__ ids,
                                                     const int *__restrict__ first, const int *__restrict__ cptr,
                                                     int ngroups, double eps, GridScratch gs) {
  extern __shared__ __align__(16) char dsm[];
  __shared__ PluCand red[16];
  __shared__ PluCand s_best;
  __shared__ int s_who, s_myli;
  int gq = 0;
  while (gq < ngroups && !((int)blockIdx.x >= first[2 * gq] && (int)blockIdx.x < first[2 * gq + 1])) ++gq;
  if (gq >= ngroups) return;  // CTA of no group in this launch
  const int f0 = first[2 * gq], G = first[2 * gq + 1] - f0, g = blockIdx.x - f0;
  GridScratch mine = gs;
  // 16-byte slots {signed pivot value, key}: |value| orders, the sign rides along
  MaxLoc *slots = gs.best + 2 * (size_t)f0;  // [parity][G]
  double *cand = gs.cand + 2 * (size_t)f0 * gs.nmax;                       // [parity][G][nmax]
  mine.bar = gs.bar + 2 * gq;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int cc = cptr[gq]; cc < cptr[gq + 1]; ++cc) {
    const PluJob J = jobs[ids[cc]];
    const int m = J.m, n = J.n;
    const int nl_max = (m + G - 1) / G, nl = (m - g + G - 1) / G, kmin = min(m, n);
    double *rows = (double *)dsm;
    double *prow = rows + (size_t)nl_max * n;
    int *posR = (int *)(prow + n);
    int *act = posR + nl_max;
    int *pstep = act + nl_max;
    int *swp = pstep + nl_max;
    int *colAt = swp + kmin;
    for (long long e = tid; e < (long long)nl * n; e += nt) {
      int li = (int)(e / n), j = (int)(e % n);
      rows[e] = J.a[(long long)(li * G + g) * J.ld + j];
    }
    for (int li = tid; li < nl; li += nt) {
      posR[li] = li * G + g;
      act[li] = 1;
      pstep[li] = -1;
    }
    for (int j = tid; j < n; j += nt) colAt[j] = j;
    __syncthreads();
    PluCand best = cand_none();
    for (int li = warp; li < nl; li += nw) {
      const double *row = rows + (size_t)li * n;
      double rbv = -1.0, rsv = 0.0;
      int rj = 0x7fffffff;
      for (int j = lane; j < n; j += 32) {
        double x = row[j], av = fabs(x);
        if (av > rbv) {
          rbv = av;
          rsv = x;
          rj = j;
        }
      }
      const long long key = (long long)(li * G + g) * n + rj;
      if (rj != 0x7fffffff && better(rbv, key, best.v, best.key)) best = PluCand{rbv, rsv, key, li};
    }
    PluState my{};
    int steps = 0;
    for (int k = 0; k < kmin; ++k) {
      const int par = k & 1;
      {
        int who = 0;
        PluCand c = warp_best(best, who);
        if (lane == 0) red[warp] = c;
        __syncthreads();
        if (warp == 0) {
          PluCand x = lane < nw ? red[lane] : cand_none();
          x = warp_best(x, who);
          if (lane == 0) {
            s_best = x;
            slots[par * G + g] = MaxLoc{x.key == 0x7fffffffffffffffLL ? -1.0 : x.sv, x.key};
          }
        }
        __syncthreads();
        const int bl = s_best.li;
        if (tid == 0) s_myli = bl;
        if (bl >= 0) {
          const double *src = rows + (size_t)bl * n;
          double *dst = cand + ((size_t)par * G + g) * gs.nmax;
          for (int j = tid; j < n; j += nt) dst[j] = src[j];
        }
      }
      group_barrier(&mine, G);
      // warp 0 reduces the group's candidates (L2, bypassing L1) and broadcasts
      // the winner through shared memory (every warp reading them would put
      // G x warps x CTAs requests on the same lines)
      if (warp == 0) {
        double ov[GRID_MAX / 32];
        long long ok[GRID_MAX / 32];
#pragma unroll
        for (int u = 0; u < GRID_MAX / 32; ++u) {  // all loads first, then the in-lane reduction
          const int q = lane + 32 * u;
          ov[u] = q < G ? __ldcg(&slots[par * G + q].v) : 0.0;
          ok[u] = q < G ? __ldcg(&slots[par * G + q].key) : 0x7fffffffffffffffLL;
        }
        PluCand gb0 = cand_none();
        int who0 = 0x7fffffff;
#pragma unroll
        for (int u = 0; u < GRID_MAX / 32; ++u) {
          const double av = ok[u] == 0x7fffffffffffffffLL ? -1.0 : fabs(ov[u]);
          if (better(av, ok[u], gb0.v, gb0.key)) {
            gb0 = PluCand{av, ov[u], ok[u], -1};
            who0 = lane + 32 * u;
          }
        }
        gb0 = warp_best(gb0, who0);
        if (lane == 0) {
          s_best = gb0;
          s_who = who0;
        }
      }
      __syncthreads();
      const PluCand gb = s_best;
      const int who = s_who;
      double piv = gb.v;
      int pr = k, bj = k;
      if (gb.key != 0x7fffffffffffffffLL) {
        if (gb.key < 0xffffffffLL) {
          const unsigned k32 = (unsigned)gb.key, q32 = k32 / (unsigned)n;
          pr = (int)q32;
          bj = (int)(k32 - q32 * (unsigned)n);
        } else {
          pr = (int)(gb.key / n);
          bj = (int)(gb.key % n);
        }
      } else {
        piv = -1.0;
      }
      if (plu_stop(my, k, J.kmax, eps, piv)) break;
      my.prev = fabs(gb.sv);
      my.rank = k + 1;
      steps = k + 1;
      const double akk = gb.sv;
      {
        const double *orow = cand + ((size_t)par * G + who) * gs.nmax;
        for (int j = k + 1 + tid; j < n; j += nt) prow[j] = (j == bj) ? __ldcg(orow + k) : __ldcg(orow + j);
      }
      if (tid == 0) {
        int t = colAt[k];
        colAt[k] = colAt[bj];
        colAt[bj] = t;
        swp[k] = bj;
        if (who == g) {
          const int wl = s_myli;  // this CTA won: its published candidate row
          act[wl] = 0;
          pstep[wl] = k;
          posR[wl] = k;
        }
      }
      __syncthreads();
      best = cand_none();
      for (int li = warp; li < nl; li += nw) {
        if (!act[li]) continue;
        double *row = rows + (size_t)li * n;
        const double ok_ = row[k], ob = row[bj];
        int pos = posR[li];
        const double l = ob / akk;
        __syncwarp();
        if (lane == 0) {
          row[k] = l;
          if (bj != k) row[bj] = ok_;
          if (pos == k) posR[li] = pr;
        }
        __syncwarp();
        if (pos == k) pos = pr;
        double rbv = -1.0, rsv = 0.0;
        int rj = 0x7fffffff;
        plu_row_update(row, prow, l, k + 1, n, lane, [&](double v, int j) {
          const double av = fabs(v);
          if (av > rbv) {
            rbv = av;
            rsv = v;
            rj = j;
          }
        });
        const long long key = (long long)pos * n + rj;
        if (rj != 0x7fffffff && better(rbv, key, best.v, best.key)) best = PluCand{rbv, rsv, key, li};
      }
    }
    __syncthreads();
    for (int li = tid; li < nl; li += nt) {
      const int p = pstep[li];
      if (p < 0) continue;
      double *row = rows + (size_t)li * n;
      for (int s2 = p; s2 < steps; ++s2) {
        const int b2 = swp[s2];
        if (b2 != s2) {
          double x = row[s2];
          row[s2] = row[b2];
          row[b2] = x;
        }
      }
    }
    __syncthreads();
    for (long long e = tid; e < (long long)nl * n; e += nt) {
      int li = (int)(e / n), j = (int)(e % n);
      J.a[(long long)(li * G + g) * J.ld + j] = rows[e];
    }
    for (int li = tid; li < nl; li += nt) J.rowAt[posR[li]] = li * G + g;
    if (g == 0) {
      for (int j = tid; j < n; j += nt) J.colAt[j] = colAt[j];
      if (tid == 0) {
        plu_out(J, my);
        J.out[3] = 0;
      }
    }
    group_barrier(&mine, G);  // candidate buffers are reused by the next core
  }
}

// Cooperative launch split into groups of CTAs: group q = CTAs
// [range[2q], range[2q+1]) factors cores ids[cptr[q] .. cptr[q+1]) one after
// another with its own barrier and candidate buffers, concurrently with the
// other groups (the per-step latency, not the trailing update, bounds a core).
template <bool ROWS_SMEM>
__global__ void __launch_bounds__(512) k_plu_groups(const PluJob *__restrict__ jobs, const int *__restrict__ ids,
                                                    const int *__restrict__ first, const int *__restrict__ cptr,
                                                    int ngroups, double eps, GridScratch gs) {
  extern __shared__ __align__(16) char dsm[];
  __shared__ MaxLoc red[32];
  __shared__ PluState st;
  __shared__ int s_nact, s_win;
  int q = 0;
  while (q < ngroups && !((int)blockIdx.x >= first[2 * q] && (int)blockIdx.x < first[2 * q + 1])) ++q;
  if (q >= ngroups) return;  // CTA of no group in this launch
  const int f0 = first[2 * q], G = first[2 * q + 1] - f0, g = blockIdx.x - f0;
  GridScratch mine = gs;
  mine.best = gs.best + 2 * (size_t)f0;
  mine.cand = gs.cand + 2 * (size_t)f0 * gs.nmax;
  mine.bar = gs.bar + 2 * q;
  for (int c = cptr[q]; c < cptr[q + 1]; ++c) {
    const PluJob J = jobs[ids[c]];
    plu_dist_body<true, ROWS_SMEM>(J, eps, G, g, dsm, red, st, s_nact, nullptr, nullptr, &mine, &s_win);
    group_barrier(&mine, G);  // candidate buffers are reused by the next core
  }
}

// compact r x r LU of a factored core: lu[i][j] = a[rowAt[i]][colAt[j]]
struct LuExtractJob {
  const double *a;
  int ld, r;
  const int *rowAt, *colAt;
  double *out;
};
__global__ void k_lu_extract(const LuExtractJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  const LuExtractJob J = jobs[blockIdx.y];
  long long total = (long long)J.r * J.r;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / J.r), j = (int)(e % J.r);
    J.out[e] = J.a[(long long)(J.rowAt ? J.rowAt[i] : i) * J.ld + (J.colAt ? J.colAt[j] : j)];
  }
}



// ---------------------------------------------------------------------------
// getrf (partial pivoting, LAPACK dgetf2 semantics: first max |a|, row swaps
// of whole rows, reciprocal scaling), one CTA per matrix, in place.
// flag: 1 if a zero / non-finite diagonal (reference singular checks) or a
// non-finite input (hodlr.py:346).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_getrf(const LuJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  __shared__ MaxLoc red[33];
  __shared__ int s_p;
  const LuJob J = jobs[blockIdx.x];
  const int n = J.n, lda = J.lda, tid = threadIdx.x, nt = blockDim.x;
  double *a = J.a;
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (int i = k + tid; i < n; i += nt) {
      double v = fabs(a[(long long)i * lda + k]);
      if (better(v, i, bv, bk)) {
        bv = v;
        bk = i;
      }
    }
    MaxLoc best = block_maxloc(bv, bk, red);
    if (tid == 0) {
      int p = (best.key == 0x7fffffffffffffffLL) ? k : (int)best.key;
      J.piv[k] = p;
      s_p = p;
    }
    __syncthreads();
    const int p = s_p;
    const double pv = a[(long long)p * lda + k];
    if (pv != 0.0) {
      if (p != k)
        for (int j = tid; j < n; j += nt) {
          double t = a[(long long)k * lda + j];
          a[(long long)k * lda + j] = a[(long long)p * lda + j];
          a[(long long)p * lda + j] = t;
        }
      __syncthreads();
      const double rinv = 1.0 / pv;
      for (int i = k + 1 + tid; i < n; i += nt) a[(long long)i * lda + k] *= rinv;
    }
    __syncthreads();
    const int w = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int i = k + 1 + w; i < n; i += nw) {
      const double l = a[(long long)i * lda + k];
      double *ri = a + (long long)i * lda;
      const double *rk = a + (long long)k * lda;
      for (int j = k + 1 + lane; j < n; j += 32) ri[j] = fma(-l, rk[j], ri[j]);
    }
    __syncthreads();
  }
  if (tid == 0 && J.flag) {
    int bad = 0;
    for (int k = 0; k < n; ++k) {
      double d = fabs(a[(long long)k * lda + k]);
      if (d == 0.0 || !isfinite(d)) bad = 1;
    }
    if (bad) *J.flag = 1;
  }
}

// ---------------------------------------------------------------------------
// blocked getrf / getrs building blocks for large matrices (right-looking,
// panel width PNB; the trailing update is k_gemm across the whole GPU)
// ---------------------------------------------------------------------------
constexpr int PNB = 64;

struct PanelJob {  // panel columns [c0, c0+w) of an n x n matrix, rows c0..n-1
  double *a;
  int n, lda, c0, w;
  int *piv;
  int *flag;
};


// Panel LU (partial pivoting, LAPACK rule) with the panel resident in shared
// memory (stride PNB+1: conflict-free column scans), one thread per row.
constexpr int PLD = PNB + 1;
constexpr int PANEL_ROWS_MAX = 416;  // rows per CTA (416 * 65 * 8 = 216 KB)
// Panel LU across a cluster of CS CTAs (panel rows in distributed shared
// memory), ONE cluster barrier per column step: every CTA pushes its block
// candidate (|a|, row) and that candidate's row into a slot of EVERY CTA's
// shared memory, and the CTA owning panel row kk pushes row kk; after the
// barrier each CTA reduces the CS candidates locally and has the pivot row and
// row kk in its own shared memory, so the swap and the trailing update need no
// remote reads. Slots are parity double-buffered (a CTA pushes step kk + 2
// only after every CTA passed step kk + 1's barrier). Same pivot rule and
// arithmetic as k_getrf_panel_cta.
constexpr int PANEL_ROWS_CL = 384;  // rows per cluster CTA (panel + slots fit the opt-in)
constexpr int PSLOT = PNB + 2;      // candidate row, |a|, key bits
constexpr size_t PANEL_CL_SLOTS = sizeof(double) * (2 * 16 * PSLOT + 2 * PNB);
__global__ void __launch_bounds__(512) k_getrf_panel_cl(const PanelJob *__restrict__ jobs) {
  extern __shared__ double sh_panel[];
  __shared__ MaxLoc red[33];
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), q = (int)cl.block_rank();
  const PanelJob J = jobs[blockIdx.x / CS];
  const int n = J.n, lda = J.lda, c0 = J.c0, w = J.w, tid = threadIdx.x;
  const int m = n - c0, rp = (m + CS - 1) / CS, r0 = q * rp, nr = max(0, min(m, r0 + rp) - r0);
  double *slots = sh_panel + (size_t)rp * PLD;  // [2][16][PSLOT]
  double *rowk = slots + 2 * 16 * PSLOT;        // [2][PNB]
  double *a = J.a;
  // load my slab: panel row t (global row c0 + r0 + t), columns c0 .. c0+w-1
  for (int e = tid; e < nr * w; e += blockDim.x) {
    int t = e / w, j = e - t * w;
    sh_panel[t * PLD + j] = a[(long long)(c0 + r0 + t) * lda + c0 + j];
  }
  __syncthreads();
  double *myrow = tid < nr ? sh_panel + tid * PLD : nullptr;
  const int lane = tid & 31;
  for (int kk = 0; kk < w; ++kk) {
    const int par = kk & 1;
    // local candidate over my rows with panel index >= kk (block_maxloc's
    // barriers also order the previous step's row updates before the pushes)
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    if (myrow && r0 + tid >= kk) {
      bv = fabs(myrow[kk]);
      bk = r0 + tid;
    }
    const MaxLoc b = block_maxloc(bv, bk, red);
    const int li = b.key == 0x7fffffffffffffffLL ? -1 : (int)(b.key - r0);
    for (int e = tid; e < CS * PSLOT; e += blockDim.x) {
      const int dst = e / PSLOT, idx = e - dst * PSLOT;
      double val;
      if (idx < PNB)
        val = (li >= 0 && idx < w) ? sh_panel[li * PLD + idx] : 0.0;
      else if (idx == PNB)
        val = b.v;
      else
        val = __longlong_as_double(b.key);
      cl.map_shared_rank(slots, dst)[(par * 16 + q) * PSLOT + idx] = val;
    }
    const int okk = kk / rp;  // CTA holding panel row kk
    if (q == okk)
      for (int e = tid; e < CS * w; e += blockDim.x) {
        const int dst = e / w, j = e - dst * w;
        cl.map_shared_rank(rowk, dst)[par * PNB + j] = sh_panel[(kk - r0) * PLD + j];
      }
    cl.sync();
    // every warp reduces the CS candidates from its own shared memory
    double gv = -2.0;
    long long gk = 0x7fffffffffffffffLL;
    int who = 0;
    if (lane < CS) {
      gv = slots[(par * 16 + lane) * PSLOT + PNB];
      gk = __double_as_longlong(slots[(par * 16 + lane) * PSLOT + PNB + 1]);
      who = lane;
    }
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, gv, off);
      const long long ok = __shfl_xor_sync(0xffffffffu, gk, off);
      const int ow = __shfl_xor_sync(0xffffffffu, who, off);
      if (better(ov, ok, gv, gk) || (ov == gv && ok == gk && ow < who)) {
        gv = ov;
        gk = ok;
        who = ow;
      }
    }
    const int p = gk == 0x7fffffffffffffffLL ? kk : (int)gk;  // panel row index
    const double *prow = slots + (par * 16 + who) * PSLOT;  // row p before the swap
    const double *told = rowk + par * PNB;                  // row kk before the swap
    const double pv = prow[kk];
    if (q == 0 && tid == 0) J.piv[c0 + kk] = c0 + p;
    if (myrow) {  // each row by its own thread: swap, then the update
      const int gr = r0 + tid;
      if (p != kk && pv != 0.0) {
        if (gr == kk)
          for (int j = 0; j < w; ++j) myrow[j] = prow[j];
        else if (gr == p)
          for (int j = 0; j < w; ++j) myrow[j] = told[j];
      }
      if (gr > kk) {
        double l = myrow[kk];
        if (pv != 0.0) {
          l *= 1.0 / pv;
          myrow[kk] = l;
        }
        for (int j = kk + 1; j < w; ++j) myrow[j] = fma(-l, prow[j], myrow[j]);
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < nr * w; e += blockDim.x) {
    int t = e / w, j = e - t * w;
    a[(long long)(c0 + r0 + t) * lda + c0 + j] = sh_panel[t * PLD + j];
  }
  cl.sync();  // no CTA exits while a peer may still push into its shared memory
}

// panel LU with the panel in global memory: fallback for panels taller than a
// cluster's shared memory holds (16 x PANEL_ROWS_MAX rows)
__global__ void __launch_bounds__(512) k_getrf_panel(const PanelJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  __shared__ MaxLoc red[33];
  __shared__ int s_p;
  const PanelJob J = jobs[blockIdx.x];
  const int n = J.n, lda = J.lda, c0 = J.c0, w = J.w, tid = threadIdx.x, nt = blockDim.x;
  double *a = J.a;
  for (int k = c0; k < c0 + w; ++k) {
    double bv = -1.0;
    long long bk = 0x7fffffffffffffffLL;
    for (int i = k + tid; i < n; i += nt) {
      double v = fabs(a[(long long)i * lda + k]);
      if (better(v, i, bv, bk)) {
        bv = v;
        bk = i;
      }
    }
    MaxLoc best = block_maxloc(bv, bk, red);
    if (tid == 0) {
      int p = (best.key == 0x7fffffffffffffffLL) ? k : (int)best.key;
      J.piv[k] = p;
      s_p = p;
    }
    __syncthreads();
    const int p = s_p;
    const double pv = a[(long long)p * lda + k];
    if (pv != 0.0) {
      if (p != k)
        for (int j = c0 + tid; j < c0 + w; j += nt) {
          double t = a[(long long)k * lda + j];
          a[(long long)k * lda + j] = a[(long long)p * lda + j];
          a[(long long)p * lda + j] = t;
        }
      __syncthreads();
      const double rinv = 1.0 / pv;
      for (int i = k + 1 + tid; i < n; i += nt) a[(long long)i * lda + k] *= rinv;
    }
    __syncthreads();
    const int wp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int i = k + 1 + wp; i < n; i += nw) {
      const double l = a[(long long)i * lda + k];
      double *ri = a + (long long)i * lda;
      const double *rk = a + (long long)k * lda;
      for (int j = k + 1 + lane; j < c0 + w; j += 32) ri[j] = fma(-l, rk[j], ri[j]);
    }
    __syncthreads();
  }
}

// Panel LU in ONE CTA (panel rows <= PANEL_ROWS_MAX): rows in shared memory,
// thread per row, warp argmax by redux (first max |a|, NaN never wins, ties to
// the lower row), two or three block barriers per column. Same arithmetic as
// k_getrf_panel_cl / k_getrf_panel (multiply by 1/pv, FMA update).
__device__ __forceinline__ void warp_argmax_row(double v, int row, unsigned &uh_out, unsigned &ul_out,
                                                int &row_out) {
  const unsigned long long u = (v >= 0.0) ? (unsigned long long)__double_as_longlong(v) + 1ull : 0ull;
  const unsigned uh = (unsigned)(u >> 32), ul = (unsigned)u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, uh);
  const unsigned ml = __reduce_max_sync(0xffffffffu, uh == mh ? ul : 0u);
  const bool top = uh == mh && ul == ml;
  const unsigned r = (unsigned)__reduce_min_sync(0xffffffffu, top ? (unsigned)row : 0x7fffffffu);
  uh_out = mh;
  ul_out = ml;
  row_out = (int)r;
}

__global__ void __launch_bounds__(512) k_getrf_panel_cta(const PanelJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double sh_panel[];
  __shared__ unsigned s_uh[16], s_ul[16];
  __shared__ int s_row[16];
  const PanelJob J = jobs[blockIdx.x];
  const int n = J.n, lda = J.lda, c0 = J.c0, w = J.w, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = n - c0;
  double *a = J.a;
  for (int e = tid; e < m * w; e += blockDim.x) {
    int t = e / w, j = e - t * w;
    sh_panel[t * PLD + j] = a[(long long)(c0 + t) * lda + c0 + j];
  }
  __syncthreads();
  double *myrow = tid < m ? sh_panel + tid * PLD : nullptr;
  for (int kk = 0; kk < w; ++kk) {
    const double v = (myrow && tid >= kk) ? fabs(myrow[kk]) : -1.0;
    unsigned uh, ul;
    int r;
    warp_argmax_row(v, tid, uh, ul, r);
    if (lane == 0) {
      s_uh[warp] = uh;
      s_ul[warp] = ul;
      s_row[warp] = r;
    }
    __syncthreads();
    {  // every warp reduces the 16 warp candidates (warps ascend in rows)
      const unsigned xh = lane < 16 ? s_uh[lane] : 0u, xl = lane < 16 ? s_ul[lane] : 0u;
      const int xr = lane < 16 ? s_row[lane] : 0x7fffffff;
      const unsigned mh = __reduce_max_sync(0xffffffffu, xh);
      const unsigned ml = __reduce_max_sync(0xffffffffu, xh == mh ? xl : 0u);
      r = (int)__reduce_min_sync(0xffffffffu, (xh == mh && xl == ml) ? (unsigned)xr : 0x7fffffffu);
      if (mh == 0u && ml == 0u) r = kk;  // no candidate: keep row kk
    }
    const int p = r;
    const double pv = sh_panel[p * PLD + kk];
    if (tid == 0) J.piv[c0 + kk] = c0 + p;
    if (p != kk && pv != 0.0) {
      if (tid < w) {
        double t = sh_panel[kk * PLD + tid];
        sh_panel[kk * PLD + tid] = sh_panel[p * PLD + tid];
        sh_panel[p * PLD + tid] = t;
      }
      __syncthreads();
    }
    if (myrow && tid > kk) {
      double l = myrow[kk];
      if (pv != 0.0) {
        l *= 1.0 / pv;
        myrow[kk] = l;
      }
      const double *prow = sh_panel + kk * PLD;
      for (int j = kk + 1; j < w; ++j) myrow[j] = fma(-l, prow[j], myrow[j]);
    }
    __syncthreads();
  }
  for (int e = tid; e < m * w; e += blockDim.x) {
    int t = e / w, j = e - t * w;
    a[(long long)(c0 + t) * lda + c0 + j] = sh_panel[t * PLD + j];
  }
}

// apply the panel's row swaps to the columns outside the panel
struct SwapJob {
  double *a;
  int lda, ncols;  // columns 0..ncols-1 of a
  const int *piv;
  int k0, k1;      // swaps k0..k1-1 (piv[k] = row swapped with row k)
  int skip0, skip1;  // columns [skip0, skip1) are left alone
};
__global__ void k_laswp(const SwapJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  const SwapJob J = jobs[blockIdx.y];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < J.ncols; j += gridDim.x * blockDim.x) {
    if (j >= J.skip0 && j < J.skip1) continue;
    for (int k = J.k0; k < J.k1; ++k) {
      int p = J.piv[k];
      if (p != k) {
        double t = J.a[(long long)k * J.lda + j];
        J.a[(long long)k * J.lda + j] = J.a[(long long)p * J.lda + j];
        J.a[(long long)p * J.lda + j] = t;
      }
    }
  }
}

// B (w x ncols, ldb) <- T^{-1} B with T = w x w diagonal block (unit lower, or
// non-unit upper), thread per column, T staged in shared memory
struct TrsmJob {
  const double *T;
  int ldt, w;
  double *B;
  int ldb, ncols;
  int upper;
};

// ---------------------------------------------------------------------------
// explicit inverses (GPU-native replacement for the reference's lu_factor +
// lu_solve: every later solve becomes a GEMM / GEMV)
// ---------------------------------------------------------------------------
constexpr int INV_SMALL = 128;

struct InvJob {  // in-place inverse of an n x n block (n <= INV_SMALL)
  double *a;
  int n, lda;
  int *flag;  // set when a pivot is zero / non-finite (== reference's LU diagonal checks)
};


// Register-tiled Gauss-Jordan inverse for n <= NW*8 (<= 32*CPL) with partial
// pivoting (max |a| in the pivot column among the rows not yet used as pivot
// rows, lowest row on ties) and implicit row interchanges: warp w owns rows
// [8w, 8w+8), lane l owns columns {l, l+32, ...}; each thread keeps its
// 8 x CPL tile in registers. Per step the lane holding column k publishes the
// column of its warp's rows and the warp's candidate, the warp publishes its
// candidate row; after the step's only barrier every warp reduces the
// candidates redundantly and updates its tile in place (column k becomes the
// inverse's column: -a_ik / a_pk, and 1 / a_pk in the pivot row). The row /
// column scrambling of the implicit interchanges is undone by the final store:
// inv[step(r)][pivot_row(l)] = tile[r][l].
template <int NW, int CPL>
__global__ void __launch_bounds__(NW * 32) k_inv_reg(const InvJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  constexpr int NR = NW * 8, NC = 32 * CPL;
  static_assert(NW <= 32, "candidate reduction is one warp wide");
  // parity double buffers: step k writes buffer k & 1 before its only barrier;
  // a warp cannot reach step k + 2's writes before every warp has passed step
  // k + 1's barrier, i.e. finished reading step k's buffers
  __shared__ double colkb[2][NR];
  __shared__ double candrow[2][NW][NC];
  __shared__ double cv[2][NW];
  __shared__ int ci[2][NW];
  __shared__ int stepof[NR], prow[NC];
  __shared__ int bad;
  const InvJob J = jobs[blockIdx.x];
  const int n = J.n, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a[8][CPL];
  unsigned used = 0;  // bit r: row 8 warp + r is a pivot row already (or beyond n)
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = warp * 8 + r;
    if (i >= n) used |= 1u << r;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = lane + 32 * c;
      a[r][c] = (i < n && j < n) ? J.a[(long long)i * J.lda + j] : 0.0;
    }
  }
  if (threadIdx.x == 0) bad = 0;
  bool stop = false;
  // step k = 32 kc + kl: the column group kc is a compile-time register index
#pragma unroll
  for (int kc = 0; kc < CPL; ++kc) {
    if (stop) break;
    for (int kl = 0; kl < 32; ++kl) {
      const int k = kc * 32 + kl;
      if (k >= n) {
        stop = true;
        break;
      }
      const int par = k & 1;
      int wr = -1;  // this warp's candidate (local row), -1 = none
      if (lane == kl) {
        double bv = -1.0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const double v = a[r][kc];
          colkb[par][warp * 8 + r] = v;
          const double av = fabs(v);
          if (!((used >> r) & 1u) && av > bv) {  // rows ascend: strict '>' keeps the first maximum
            bv = av;
            wr = r;
          }
        }
        cv[par][warp] = bv;
        ci[par][warp] = wr < 0 ? 0x7fffffff : warp * 8 + wr;
      }
      wr = __shfl_sync(0xffffffffu, wr, kl);
      switch (wr) {  // warp-uniform: publish the candidate row
#pragma unroll
        case 0: case 1: case 2: case 3: case 4: case 5: case 6: case 7:
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (r == wr)
#pragma unroll
              for (int c = 0; c < CPL; ++c) candrow[par][warp][lane + 32 * c] = a[r][c];
          break;
        default: break;
      }
      __syncthreads();  // the only barrier of the step
      double bv = lane < NW ? cv[par][lane] : -1.0;
      int bi = lane < NW ? ci[par][lane] : 0x7fffffff;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        if (off >= NW) continue;
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      const int p = __shfl_sync(0xffffffffu, bi, 0);
      const double pv = p == 0x7fffffff ? 0.0 : colkb[par][p];
      if (pv == 0.0 || !isfinite(pv)) {
        if (threadIdx.x == 0) bad = 1;
        stop = true;
        break;
      }
      if (threadIdx.x == 0) {
        stepof[p] = k;
        prow[k] = p;
      }
      const double rinv = 1.0 / pv;
      const double *rowP = candrow[par][p >> 3];
      double pj[CPL];  // the new pivot row: a_pj / a_pk, and 1 / a_pk in column k
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int j = lane + 32 * c;
        pj[c] = ((c == kc && lane == kl) ? 1.0 : rowP[j]) * rinv;
      }
      if (lane == kl) {
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r][kc] = 0.0;  // column k: 0 - a_ik / a_pk after the update
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const double f = colkb[par][warp * 8 + r];
#pragma unroll
        for (int c = 0; c < CPL; ++c) a[r][c] = fma(-f, pj[c], a[r][c]);
      }
      if (warp == (p >> 3)) {
        const int pr = p & 7;
        used |= 1u << pr;
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r == pr)
#pragma unroll
            for (int c = 0; c < CPL; ++c) a[r][c] = pj[c];
      }
    }
  }
  __syncthreads();
  if (!bad) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int i = warp * 8 + r, l = lane + 32 * c;
        if (i < n && l < n) J.a[(long long)stepof[i] * J.lda + prow[l]] = a[r][c];
      }
  }
  if (threadIdx.x == 0 && bad && J.flag) *J.flag = 1;
}

// inverse of a w x w (w <= 64) diagonal block: unit lower (upper = 0) or
// non-unit upper (upper = 1); out is w x w, ld w
struct TrinvJob {
  const double *T;
  int ldt, w, upper;
  double *out;
  int ldo;  // leading dimension of out (w when 0)
};
constexpr size_t TRINV_SMEM = sizeof(double) * (64 * 64 + 2 * 64 * 65);
// Triangular inverse by recursive doubling: with the inverses of the two s x s
// diagonal blocks known, the 2s x 2s inverse only needs its off-diagonal block:
//   lower [[A,0],[C,B]]^-1 = [[Ai,0],[-Bi C Ai, Bi]]
//   upper [[A,C],[0,B]]^-1 = [[Ai,-Ai C Bi],[0,Bi]]
// All pairs of a stage are formed in parallel (log2(64) = 6 stages of small
// shared-memory GEMMs, instead of 64 dependent substitution rows).
__global__ void __launch_bounds__(256) k_trinv(const TrinvJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double tdyn[];
  double *Ts = tdyn;              // w x w (ld w)
  double *X = tdyn + 64 * 64;     // inverse, ld 65
  double *Tm = X + 64 * 65;       // temporary, ld 65
  const TrinvJob J = jobs[blockIdx.x];
  const int w = J.w, tid = threadIdx.x, nt = blockDim.x;
  const bool up = J.upper != 0;
  for (int e = tid; e < w * w; e += nt) {
    int i = e / w, j = e % w;
    double t = J.T[(long long)i * J.ldt + j];
    Ts[e] = t;
    X[i * 65 + j] = (i == j) ? (up ? 1.0 / t : 1.0) : 0.0;
  }
  __syncthreads();
  for (int sz = 1; sz < w; sz <<= 1) {
    const int npair = (w + 2 * sz - 1) / (2 * sz);
    // Tm = C * Bi (upper) or C * Ai (lower) for every pair; C is |B| x s (lower) or s x |B| (upper)
    for (int e = tid; e < npair * sz * sz; e += nt) {
      int p = e / (sz * sz), r = (e / sz) % sz, c = e % sz;
      int k0 = p * 2 * sz, k1 = k0 + sz, nb = min(sz, w - k1);
      if (nb <= 0) continue;
      double acc = 0.0;
      if (!up) {  // rows of B (r < nb), cols of A (c)
        if (r >= nb) continue;
        for (int t = 0; t < sz; ++t) acc = fma(Ts[(k1 + r) * w + k0 + t], X[(k0 + t) * 65 + k0 + c], acc);
        Tm[(k1 + r) * 65 + k0 + c] = acc;
      } else {    // rows of A (r), cols of B (c < nb)
        if (c >= nb) continue;
        for (int t = 0; t < nb; ++t) acc = fma(Ts[(k0 + r) * w + k1 + t], X[(k1 + t) * 65 + k1 + c], acc);
        Tm[(k0 + r) * 65 + k1 + c] = acc;
      }
    }
    __syncthreads();
    for (int e = tid; e < npair * sz * sz; e += nt) {
      int p = e / (sz * sz), r = (e / sz) % sz, c = e % sz;
      int k0 = p * 2 * sz, k1 = k0 + sz, nb = min(sz, w - k1);
      if (nb <= 0) continue;
      double acc = 0.0;
      if (!up) {  // X[B rows, A cols] = -Bi * Tm
        if (r >= nb) continue;
        for (int t = 0; t < nb; ++t) acc = fma(X[(k1 + r) * 65 + k1 + t], Tm[(k1 + t) * 65 + k0 + c], acc);
        X[(k1 + r) * 65 + k0 + c] = -acc;
      } else {    // X[A rows, B cols] = -Ai * Tm
        if (c >= nb) continue;
        for (int t = 0; t < sz; ++t) acc = fma(X[(k0 + r) * 65 + k0 + t], Tm[(k0 + t) * 65 + k1 + c], acc);
        X[(k0 + r) * 65 + k1 + c] = -acc;
      }
    }
    __syncthreads();
  }
  const int ldo = J.ldo > 0 ? J.ldo : w;
  for (int e = tid; e < w * w; e += nt) J.out[(long long)(e / w) * ldo + (e % w)] = X[(e / w) * 65 + (e % w)];
}

// diagonal check after a blocked LU
__global__ void k_diag_check(const LuJob *__restrict__ jobs) {
  pdl_wait();
  pdl_trigger();
  const LuJob J = jobs[blockIdx.x];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int k = threadIdx.x; k < J.n; k += blockDim.x) {
    double d = fabs(J.a[(long long)k * J.lda + k]);
    if (d == 0.0 || !isfinite(d)) bad = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && bad && J.flag) *J.flag = 1;
}

// non-finite scan of a square block (hodlr.py:346 check before the core LU)
__global__ void k_check_finite(const LuJob *__restrict__ jobs) {
  const LuJob J = jobs[blockIdx.y];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  long long total = (long long)J.n * J.n;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int i = (int)(e / J.n), j = (int)(e % J.n);
    if (!isfinite(J.a[(long long)i * J.lda + j])) bad = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && bad && J.flag) *J.flag = 1;
}

// ---------------------------------------------------------------------------
// batched two-term GEMV for the preconditioner apply, 1..8 right-hand sides:
//   y[v][i] = (y0 ? y0[v][i] : 0) + a1 * A1[i,:] . x1[v] + a2 * A2[i,:] . x2[v][idx2]
// ---------------------------------------------------------------------------
struct GemvJob {
  double *y;
  const double *y0;
  int m;
  const double *A1;
  int lda1, k1;
  const double *x1;
  double a1;
  const double *A2;
  int lda2, k2;
  const double *x2;
  const long long *idx2;
  double a2;
  // several right-hand sides: vector v reads / writes at p + v * stride
  long long ys, y0s, x1s, x2s;
};

// ---------------------------------------------------------------------------
// one right-hand side: warp per output row (k_gemv2)
// ---------------------------------------------------------------------------
// Row t belongs to job q with start[q] <= t < start[q + 1] (rows at or past
// start[q] + m are padding of a plan shared with k_gemv_tc and are skipped).
// Each warp takes a contiguous chunk of rows: one binary search, then a walk.
// Every row is summed in the same order (lane-strided, k ascending per lane,
// then a shuffle tree) however rows are grouped, so a row's bits do not depend
// on the batch it is in (the sharded apply relies on that). Loads are issued
// ahead of the FMAs (GV_U per lane per row, GV_R rows of one job at a time)
// to keep enough bytes in flight for HBM.
constexpr int GV_R = 4;
template <int U, typename Ld>
__device__ __forceinline__ void gv_run(const double *__restrict__ a, const Ld &xv, int k, int &kk, double &s) {
  for (; kk + 32 * (U - 1) < k; kk += 32 * U) {
    double v[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = a[kk + 32 * u];
      w[u] = xv(kk + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(v[u], w[u], s);
  }
}
// lane-strided dot, k ascending per lane (8 then 2 then 1 loads in flight)
template <typename Ld>
__device__ __forceinline__ double gv_dot_t(const double *__restrict__ a, const Ld &xv, int k, int lane) {
  double s = 0.0;
  int kk = lane;
  gv_run<8>(a, xv, k, kk, s);
  gv_run<2>(a, xv, k, kk, s);
  gv_run<1>(a, xv, k, kk, s);
  return s;
}
__device__ __forceinline__ double gv_dot(const double *__restrict__ a, const double *__restrict__ x, int k, int lane) {
  return gv_dot_t(a, [x](int q) { return x[q]; }, k, lane);
}
__device__ __forceinline__ double gv_dot_idx(const double *__restrict__ a, const double *__restrict__ x,
                                             const long long *__restrict__ idx, int k, int lane) {
  return gv_dot_t(a, [x, idx](int q) { return x[idx[q]]; }, k, lane);
}
__device__ __forceinline__ double warp_sum_down(double s) {
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  return s;
}
__device__ __forceinline__ void gemv_rows(const GemvJob *__restrict__ jobs, const int *__restrict__ start, int q,
                                          int t0, int t1, int lane) {
  if (t0 >= t1) return;
  int qend = start[q + 1];
  for (int t = t0; t < t1;) {
    while (t >= qend) {
      ++q;
      qend = start[q + 1];
    }
    const GemvJob &J = jobs[q];
    const int i = t - start[q], mend = start[q] + J.m;  // rows past m: padding of a shared plan
    if (t >= mend) {
      t = min(t1, qend);
      continue;
    }
    if (J.k2 == 0 && J.k1 <= 16) {
      // short rows: W >= k1 lanes per row (W = 4, 8, 16 from k1 alone: one
      // element per lane), 32 / W rows per pass, GV_R passes' loads in flight,
      // xor tree inside the W lanes
      const int W = J.k1 <= 4 ? 4 : (J.k1 <= 8 ? 8 : 16);
      const int G = 32 / W, g = lane / W, l = lane & (W - 1);
      const int tend = min(t1, mend), s0 = start[q];
      for (int tb = t; tb < tend; tb += G * GV_R) {
        double sr[GV_R];
#pragma unroll
        for (int r = 0; r < GV_R; ++r) {
          const int tr = tb + g + G * r;
          sr[r] = (tr < tend && l < J.k1) ? J.A1[(long long)(tr - s0) * J.lda1 + l] * J.x1[l] : 0.0;
        }
        for (int o = W >> 1; o > 0; o >>= 1)
#pragma unroll
          for (int r = 0; r < GV_R; ++r) sr[r] += __shfl_xor_sync(0xffffffffu, sr[r], o);
        if (l == 0) {
#pragma unroll
          for (int r = 0; r < GV_R; ++r) {
            const int tr = tb + g + G * r;
            if (tr < tend) {
              double v = J.y0 ? J.y0[tr - s0] : 0.0;
              J.y[tr - s0] = v + J.a1 * sr[r];
            }
          }
        }
      }
      t = tend;
      continue;
    }
    if (t + GV_R <= min(t1, mend)) {
      // GV_R rows of one job: the same per-row order as below, loads of all rows in flight
      double s1[GV_R], s2[GV_R];
#pragma unroll
      for (int r = 0; r < GV_R; ++r) s1[r] = s2[r] = 0.0;
      if (J.k1) {
        const double *a = J.A1 + (long long)i * J.lda1;
        for (int kk = lane; kk < J.k1; kk += 32) {
          const double xv = J.x1[kk];
          double v[GV_R];
#pragma unroll
          for (int r = 0; r < GV_R; ++r) v[r] = a[(long long)r * J.lda1 + kk];
#pragma unroll
          for (int r = 0; r < GV_R; ++r) s1[r] = fma(v[r], xv, s1[r]);
        }
      }
      if (J.k2) {
        const double *a = J.A2 + (long long)i * J.lda2;
        for (int kk = lane; kk < J.k2; kk += 32) {
          const double xv = J.idx2 ? J.x2[J.idx2[kk]] : J.x2[kk];
          double v[GV_R];
#pragma unroll
          for (int r = 0; r < GV_R; ++r) v[r] = a[(long long)r * J.lda2 + kk];
#pragma unroll
          for (int r = 0; r < GV_R; ++r) s2[r] = fma(v[r], xv, s2[r]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < GV_R; ++r) {
          s1[r] += __shfl_down_sync(0xffffffffu, s1[r], o);
          s2[r] += __shfl_down_sync(0xffffffffu, s2[r], o);
        }
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < GV_R; ++r) {
          double v = J.y0 ? J.y0[i + r] : 0.0;
          if (J.k1) v += J.a1 * s1[r];
          if (J.k2) v += J.a2 * s2[r];
          J.y[i + r] = v;
        }
      }
      t += GV_R;
      continue;
    }
    double s1 = 0.0, s2 = 0.0;
    if (J.k1) s1 = gv_dot(J.A1 + (long long)i * J.lda1, J.x1, J.k1, lane);
    if (J.k2) {
      const double *a = J.A2 + (long long)i * J.lda2;
      s2 = J.idx2 ? gv_dot_idx(a, J.x2, J.idx2, J.k2, lane) : gv_dot(a, J.x2, J.k2, lane);
    }
    s1 = warp_sum_down(s1);
    s2 = warp_sum_down(s2);
    if (lane == 0) {
      double v = J.y0 ? J.y0[i] : 0.0;
      if (J.k1) v += J.a1 * s1;
      if (J.k2) v += J.a2 * s2;
      J.y[i] = v;
    }
    ++t;
  }
}

// warp per output row; each warp takes a contiguous chunk of rows, starting in
// job wq[warp] (computed on the host: no search through start[] on the device)
__global__ void __launch_bounds__(256) k_gemv2(const GemvJob *__restrict__ jobs, const int *__restrict__ start,
                                               const int *__restrict__ wq, int chunk, int nrows) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int t0 = warp * chunk;
  if (t0 >= nrows) return;
  gemv_rows(jobs, start, wq[warp], t0, min(nrows, t0 + chunk), lane);
}


// ---------------------------------------------------------------------------
// several right-hand sides (2..8): k_gemv_tc
// ---------------------------------------------------------------------------
// Rows in groups of 8 on the FP64 tensor cores (mma.sync m8n8k4): the A
// fragment is 8 rows x 4 consecutive columns of the matrix, the B fragment the
// same 4 entries of up to 8 right-hand sides (vector v in column v, unused
// columns zero), so a matrix element is loaded once for every vector and every
// load instruction reads 32 contiguous bytes per row.
// Arithmetic of a row (a function of the job's shape only): a term's k columns
// are cut into ws(k) = ceil(k / 256) (at most 8) segments of whole 16-column
// steps; a segment's partial is four interleaved k-ascending chains of
// correctly rounded FMAs (what m8n8k4 computes, see the GEMV test) summed as
// (c0 + c1) + (c2 + c3), and the term is p_0 + p_1 + ... left to right. A column of a
// several-vector apply is therefore bitwise the one-vector apply, and a row's
// bits do not depend on the launch it is in (the sharded apply and the subtree
// kernel rely on that). Long rows use several warps of one CTA (the segments),
// so a matrix with few rows still keeps many warps' loads in flight.
__device__ __forceinline__ int gv_ws(int k) { return k <= 256 ? 1 : min(8, (k + 255) >> 8); }
__device__ __forceinline__ int gv_seglen(int k, int ws) { return ((((k + ws - 1) / ws) + 15) >> 4) << 4; }
// partial of one segment [kb, ke) for rows i0 .. i0 + 7 (D fragment: rows
// i0 + g, vectors 2c, 2c + 1): four interleaved chains (chain j takes columns
// 4j .. 4j + 3 of every 16-column step, k ascending), then (c0 + c1) + (c2 + c3)
template <int NV, int RGN>
__device__ __forceinline__ void gv_segn(const double *__restrict__ A, long long lda,
                                        const double *__restrict__ x, long long xs,
                                        const long long *__restrict__ idx, int kb, int ke, const int (&i0)[RGN],
                                        int m, int g, int c, double (&d)[RGN][2]) {
  double acc[RGN][4][2];
#pragma unroll
  for (int r = 0; r < RGN; ++r)
#pragma unroll
    for (int h = 0; h < 4; ++h) acc[r][h][0] = acc[r][h][1] = 0.0;
  bool rok[RGN];
  const double *ar[RGN];
#pragma unroll
  for (int r = 0; r < RGN; ++r) {
    const int row = i0[r] + g;
    rok[r] = row < m;
    ar[r] = A + (long long)(rok[r] ? row : 0) * lda;
  }
  const bool xok = g < NV;
  const double *xr = x + (long long)(xok ? g : 0) * xs;
  int k0 = kb;
  for (; k0 + 32 <= ke; k0 += 32) {  // two 16-column steps per pass, every load issued first
    double av[RGN][8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int kk = k0 + 4 * u + c;
#pragma unroll
      for (int r = 0; r < RGN; ++r) av[r][u] = rok[r] ? ar[r][kk] : 0.0;
      xv[u] = xok ? (idx ? xr[idx[kk]] : xr[kk]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int r = 0; r < RGN; ++r) dmma884(acc[r][u & 3][0], acc[r][u & 3][1], av[r][u], xv[u]);
  }
  if (k0 < ke) {  // the last < 32 columns (masked)
    double av[RGN][8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int kk = k0 + 4 * u + c;
      const bool kin = kk < ke;
#pragma unroll
      for (int r = 0; r < RGN; ++r) av[r][u] = (rok[r] && kin) ? ar[r][kk] : 0.0;
      xv[u] = (xok && kin) ? (idx ? xr[idx[kk]] : xr[kk]) : 0.0;
    }
    const bool two = ke - k0 > 16;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < 4 || two)
#pragma unroll
        for (int r = 0; r < RGN; ++r) dmma884(acc[r][u & 3][0], acc[r][u & 3][1], av[r][u], xv[u]);
  }
#pragma unroll
  for (int r = 0; r < RGN; ++r) {
    d[r][0] = (acc[r][0][0] + acc[r][1][0]) + (acc[r][2][0] + acc[r][3][0]);
    d[r][1] = (acc[r][0][1] + acc[r][1][1]) + (acc[r][2][1] + acc[r][3][1]);
  }
}
template <int NV>
__device__ __forceinline__ void gv_seg(const double *__restrict__ A, long long lda,
                                       const double *__restrict__ x, long long xs,
                                       const long long *__restrict__ idx, int kb, int ke, int i0, int m, int g,
                                       int c, double &d0, double &d1) {
  const int i0s[1] = {i0};
  double d[1][2];
  gv_segn<NV, 1>(A, lda, x, xs, idx, kb, ke, i0s, m, g, c, d);
  d0 = d[0][0];
  d1 = d[0][1];
}
template <int NV>
__device__ __forceinline__ void gv_term_seg(const GemvJob &J, int part, int seg, int i0, int g, int c, double &d0,
                                            double &d1) {
  const int k = part == 0 ? J.k1 : J.k2, ws = gv_ws(k), sl = gv_seglen(k, ws);
  const int kb = seg * sl, ke = min(k, kb + sl);
  d0 = d1 = 0.0;
  if (seg >= ws || kb >= ke) return;
  if (part == 0)
    gv_seg<NV>(J.A1, J.lda1, J.x1, J.x1s, nullptr, kb, ke, i0, J.m, g, c, d0, d1);
  else
    gv_seg<NV>(J.A2, J.lda2, J.x2, J.x2s, J.idx2, kb, ke, i0, J.m, g, c, d0, d1);
}
// two row groups sharing each x fragment (k_gemv_tc): the same per-row chains
template <int NV>
__device__ __forceinline__ void gv_term_seg2(const GemvJob &J, int part, int seg, const int (&i0)[2], int g, int c,
                                             double (&d)[2][2]) {
  const int k = part == 0 ? J.k1 : J.k2, ws = gv_ws(k), sl = gv_seglen(k, ws);
  const int kb = seg * sl, ke = min(k, kb + sl);
  d[0][0] = d[0][1] = d[1][0] = d[1][1] = 0.0;
  if (seg >= ws || kb >= ke) return;
  if (part == 0)
    gv_segn<NV, 2>(J.A1, J.lda1, J.x1, J.x1s, nullptr, kb, ke, i0, J.m, g, c, d);
  else
    gv_segn<NV, 2>(J.A2, J.lda2, J.x2, J.x2s, J.idx2, kb, ke, i0, J.m, g, c, d);
}
// y = y0; y += a1 S1; y += a2 S2 for the lane's rows / vectors
template <int NV>
__device__ __forceinline__ void gv_epilogue(const GemvJob &J, int i0, int g, int c, const double (&s1)[2],
                                            const double (&s2)[2]) {
  const int row = i0 + g;
  if (row >= J.m) return;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int v = 2 * c + e;
    if (v >= NV) continue;
    double y = J.y0 ? J.y0[v * J.y0s + row] : 0.0;
    if (J.k1) y += J.a1 * s1[e];
    if (J.k2) y += J.a2 * s2[e];
    J.y[v * J.ys + row] = y;
  }
}
// one warp, whole row groups: every segment in turn, summed in order (the
// subtree kernel's path; the same bits as k_gemv_tc's CTA-split rows)
template <int NV>
__device__ __forceinline__ void gemv_rows_tc(const GemvJob *__restrict__ jobs, const int *__restrict__ start, int q,
                                             int t0, int t1, int lane) {
  if (t0 >= t1) return;
  const int g = lane >> 2, c = lane & 3;
  int qend = start[q + 1];
  for (int t = t0; t < t1;) {
    while (t >= qend) {
      ++q;
      qend = start[q + 1];
    }
    const GemvJob &J = jobs[q];
    const int s0 = start[q], tend = min(t1, qend);
    for (int tg = t; tg < tend; tg += 8) {
      const int i0 = tg - s0;
      double S[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      for (int part = 0; part < 2; ++part) {
        const int k = part == 0 ? J.k1 : J.k2;
        if (!k) continue;
        const int ws = gv_ws(k);
        for (int seg = 0; seg < ws; ++seg) {
          double d0, d1;
          gv_term_seg<NV>(J, part, seg, i0, g, c, d0, d1);
          if (seg == 0) {
            S[part][0] = d0;
            S[part][1] = d1;
          } else {
            S[part][0] += d0;
            S[part][1] += d1;
          }
        }
      }
      gv_epilogue<NV>(J, i0, g, c, S[0], S[1]);
    }
    t = tend;
  }
}

// One CTA (8 warps) per work item (job, first row group): a job whose longer
// term has ws segments gives each of 8 / ws warp slots ws warps, a warp slot
// covers two row groups sharing every x fragment (half the vector loads per
// matrix element); the partials meet in shared memory and the segment-0 warp
// sums them in order.
struct GvItem {
  int q, g0;
};
template <int NV>
__global__ void __launch_bounds__(256) k_gemv_tc(const GemvJob *__restrict__ jobs, const GvItem *__restrict__ items) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[8][2][2][2][32];  // [warp][group][term][e][lane]
  const GvItem it = items[blockIdx.x];
  const GemvJob &J = jobs[it.q];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  const int ws = max(J.k1 ? gv_ws(J.k1) : 1, J.k2 ? gv_ws(J.k2) : 1), gpc = 8 / ws;
  const int gi = warp / ws, seg = warp % ws;
  // this warp's two row groups (they share every x fragment)
  const int i0[2] = {(it.g0 + 2 * gi) * 8, (it.g0 + 2 * gi + 1) * 8};
  const bool live = gi < gpc && i0[0] < J.m;
  double p[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};  // [term][group][e]
  if (live) {
    if (J.k1) gv_term_seg2<NV>(J, 0, seg, i0, g, c, p[0]);
    if (J.k2) gv_term_seg2<NV>(J, 1, seg, i0, g, c, p[1]);
  }
  if (ws > 1) {
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int e = 0; e < 2; ++e) red[warp][r][a][e][lane] = p[a][r][e];
    __syncthreads();
  }
  if (!live || seg != 0) return;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (i0[r] >= J.m) continue;
    double S[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int k = a == 0 ? J.k1 : J.k2, wk = k ? gv_ws(k) : 1;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double s = p[a][r][e];
        for (int sg = 1; sg < wk; ++sg) s += red[warp + sg][r][a][e][lane];
        S[a][e] = s;
      }
    }
    gv_epilogue<NV>(J, i0[r], g, c, S[0], S[1]);
  }
}

// ---------------------------------------------------------------------------
// apply, low levels: one CTA per group of whole dense subtrees, both passes
// ---------------------------------------------------------------------------
// The fronts below the first level holding a structured front form
// independent subtrees. A CTA owns whole subtrees and walks their levels with
// CTA barriers instead of kernel boundaries: per level, the contribution
// gathers of all its fronts' pivots (upward), then all their GEMV rows, warps
// spread over the rows of every front of the level. Every row is computed by
// gemv_rows_tc and every gather in k_contrib_gather's order, so the results
// are bitwise the per-level graph's; one launch per pass.
struct SubSeg {   // one level of one CTA
  int jb, je;     // GEMV jobs [jb, je) (rows numbered by start[jb .. je])
  int gb, ge;     // pivot ids to gather, gids[gb .. ge)
};
struct SubApply {
  const SubSeg *seg;
  const int *cta_seg;      // segments [cta_seg[c], cta_seg[c + 1]) in level order
  const GemvJob *job;      // upward (t = Gfp b_piv) or downward (x = Pinv b - Gpf x_fro) jobs
  const int *start;        // row prefix per job (global numbering)
  const long long *gids;   // pivot ids gathered before each upward level
  const long long *cptr, *coff;
  double *cbuf, *bu;
  long long cst, nst;      // vector strides (several right-hand sides)
};
template <int NV>
__device__ __forceinline__ void sub_level_rows(const SubApply &S, const SubSeg &g, int warp, int nw, int lane) {
  const int r0 = S.start[g.jb], r1 = S.start[g.je];
  // k_gemv_tc works on whole row groups (start[] is padded to them)
  const int chunk = NV == 1 ? (r1 - r0 + nw - 1) / nw : (((r1 - r0 + nw - 1) / nw) + 7) & ~7;
  const int t0 = r0 + warp * chunk, t1 = min(r1, t0 + chunk);
  if (t0 >= t1) return;
  int lo = g.jb, hi = g.je - 1;  // last job with start <= t0
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (S.start[mid] <= t0) lo = mid; else hi = mid - 1;
  }
  if (NV == 1)
    gemv_rows(S.job, S.start, lo, t0, t1, lane);
  else
    gemv_rows_tc<NV>(S.job, S.start, lo, t0, t1, lane);
}
template <int NV>
__global__ void __launch_bounds__(512) k_apply_sub(SubApply S, int up) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int s0 = S.cta_seg[blockIdx.x], s1 = S.cta_seg[blockIdx.x + 1];
  for (int k = 0; k < s1 - s0; ++k) {
    const SubSeg g = S.seg[up ? s0 + k : s1 - 1 - k];
    if (up && g.ge > g.gb) {
      // b_u[piv] -= contributions of the descendants, in post order
      for (int t = g.gb + warp; t < g.ge; t += nw) {
        const long long gg = S.gids[t], b = S.cptr[gg], e = S.cptr[gg + 1];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double *cb = S.cbuf + v * S.cst;
          double acc = S.bu[v * S.nst + gg];
          for (long long q0 = b; q0 < e; q0 += 32) {
            const double x = q0 + lane < e ? cb[S.coff[q0 + lane]] : 0.0;
            const int mm = (int)(e - q0 < 32 ? e - q0 : 32);
            for (int r = 0; r < mm; ++r) acc = acc - __shfl_sync(0xffffffffu, x, r);
          }
          if (lane == 0) S.bu[v * S.nst + gg] = acc;
        }
      }
      __syncthreads();  // gathered b_piv visible to every warp
    }
    sub_level_rows<NV>(S, g, warp, nw, lane);
    __syncthreads();  // this level's results visible to the next level (same CTA)
  }
}

// ---------------------------------------------------------------------------
// solve-phase vector kernels
// ---------------------------------------------------------------------------
__global__ void k_scatter_perm(const double *__restrict__ b, const long long *__restrict__ perm,
                               double *__restrict__ bu, long long n) {
  pdl_wait();
  pdl_trigger();
  b += blockIdx.y * n;  // right-hand side blockIdx.y
  bu += blockIdx.y * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bu[perm[i]] = b[i];
}
__global__ void k_gather_perm(const double *__restrict__ x, const long long *__restrict__ perm,
                              double *__restrict__ out, long long n) {
  pdl_wait();
  pdl_trigger();
  x += blockIdx.y * n;  // right-hand side blockIdx.y
  out += blockIdx.y * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = x[perm[i]];
}
// b_u[g] -= contributions in post order (multifrontal.py:549 applied lazily)
// Warp per pivot: the lanes load 32 contributions at once, then the sum runs
// in list order through shuffles (the same bits as a sequential loop).
__global__ void __launch_bounds__(256) k_contrib_gather(const long long *__restrict__ gl, int cnt,
                                                        const long long *__restrict__ cptr,
                                                        const long long *__restrict__ coff,
                                                        const double *__restrict__ cbuf, double *__restrict__ bu,
                                                        double *__restrict__ y, long long cstride, long long bstride) {
  pdl_wait();
  pdl_trigger();
  cbuf += blockIdx.y * cstride;  // right-hand side blockIdx.y
  bu += blockIdx.y * bstride;
  if (y) y += blockIdx.y * bstride;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < cnt; t += nw) {
    const long long g = gl[t];
    const long long b = cptr[g], e = cptr[g + 1];
    double acc = bu[g];
    for (long long q0 = b; q0 < e; q0 += 32) {
      const double v = q0 + lane < e ? cbuf[coff[q0 + lane]] : 0.0;
      const int m = (int)(e - q0 < 32 ? e - q0 : 32);
      for (int r = 0; r < m; ++r) acc = acc - __shfl_sync(0xffffffffu, v, r);
    }
    if (lane == 0) {
      bu[g] = acc;
      if (y) y[g] = acc;
    }
  }
}
// xf[off + j] = x[fro[j]] for all (off, fro) of a height
__global__ void k_gather_idx(const long long *__restrict__ src_idx, const double *__restrict__ x,
                             double *__restrict__ dst, long long cnt) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < cnt;
       t += (long long)gridDim.x * blockDim.x)
    dst[t] = x[src_idx[t]];
}

// ---------------------------------------------------------------------------
// Krylov vector kernels (deterministic reductions: fixed grid, ordered final sum)
// ---------------------------------------------------------------------------
constexpr int RED_BLOCKS = 296, RED_THREADS = 256;
constexpr int MGS_MAX_GRID = 1024;  // MGS partials: 2 * grid doubles of the context's d_part

__device__ __forceinline__ double block_sum(double v, double *sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) r += sh[q];
    sh[32] = r;
  }
  __syncthreads();
  r = sh[32];
  __syncthreads();
  return r;
}

// partial[b] = sum over block b of x.y
__global__ void __launch_bounds__(RED_THREADS) k_dot_part(const double *__restrict__ x,
                                                          const double *__restrict__ y,
                                                          long long n, double *__restrict__ part) {
  __shared__ double sh[33];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__device__ __forceinline__ double sum_parts(const double *part) {
  double s = 0.0;
  for (int q = 0; q < RED_BLOCKS; ++q) s += part[q];
  return s;
}
// out = sum(part) (single thread), optionally sqrt
__global__ void k_finish(const double *__restrict__ part, double *__restrict__ out, int do_sqrt) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = sum_parts(part);
    *out = do_sqrt ? sqrt(s) : s;
  }
}
// y = a*x (a = 1/s with s read on device)  : V[:, j] = w / h
__global__ void k_scale_inv(const double *__restrict__ s, const double *__restrict__ x,
                            double *__restrict__ y, long long n) {
  const double d = *s;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}
__global__ void k_sub(const double *__restrict__ a, const double *__restrict__ b,
                      double *__restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = a[i] - b[i];
}
__global__ void k_add(const double *__restrict__ a, double *__restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = y[i] + a[i];
}
// y = sum_i c[i] * V_i   (V_i = V + i*n), fixed order i = 0..j-1
__global__ void k_combine(const double *__restrict__ V, const double *__restrict__ c, int j,
                          long long n, double *__restrict__ y) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < j; ++i) s = fma(V[(long long)i * n + r], c[i], s);
    y[r] = s;
  }
}

// ---- distributed GMRES (sharded factor): rank-local vectors ----
// local SpMV over this rank's rows; column c < nl reads the local vector,
// c >= nl the all-reduced halo buffer (top-separator values of other ranks)
template <int W>
__global__ void __launch_bounds__(256) k_spmv_dist(long long nrows, const long long *__restrict__ ptr,
                                                   const int *__restrict__ col, const double *__restrict__ val,
                                                   const double *__restrict__ x, const double *__restrict__ halo,
                                                   int nl, double *__restrict__ y) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int l = threadIdx.x & (W - 1);
  const long long ng = ((long long)gridDim.x * blockDim.x) / W;
  for (long long r = t / W; r < nrows; r += ng) {
    double s = 0.0;
    for (long long p = ptr[r] + l; p < ptr[r + 1]; p += W) {
      const int c = col[p];
      s = fma(val[p], c < nl ? x[c] : halo[c - nl], s);
    }
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, W);
    if (l == 0) y[r] = s;
  }
}
// dst[idx[i]] = src[i] (dst zeroed by the caller where nothing lands)
__global__ void k_scatter_to(const long long *__restrict__ idx, const double *__restrict__ src,
                             double *__restrict__ dst, long long cnt) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x)
    dst[idx[i]] = src[i];
}
// dst[i] = src[idx[i]]
__global__ void k_gather_from(const long long *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst, long long cnt) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
// classical Gram-Schmidt projection: w -= sum_i h[i] V_i (i ascending)
__global__ void k_sub_vh(const double *__restrict__ V, const double *__restrict__ h, int j, long long n,
                         double *__restrict__ w) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    double s = w[r];
    for (int i = 0; i < j; ++i) s = s - h[i] * V[(long long)i * n + r];
    w[r] = s;
  }
}
// h[i] (+)= V_i . w for i < j: one block per basis vector, deterministic
__global__ void __launch_bounds__(256) k_multi_dot(const double *__restrict__ V, const double *__restrict__ w,
                                                   long long n, double *__restrict__ h, int accumulate) {
  __shared__ double sh[33];
  const double *v = V + (long long)blockIdx.x * n;
  double s = 0.0;
  for (long long r = threadIdx.x; r < n; r += blockDim.x) s = fma(v[r], w[r], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) h[blockIdx.x] = accumulate ? h[blockIdx.x] + s : s;
}

// Whole modified Gram-Schmidt sweep + norm of one Arnoldi step in one
// cooperative launch (krylov.py:116-120): for i = 0..j, H[i] = V_i . w then
// w -= H[i] V_i (numpy: w - (h * V_i), no FMA); finally H[j+1] = ||w||.
// Each block owns a fixed slice of w, so the axpy of projection i-1 and the
// dot of projection i run back to back on that slice; one grid barrier per
// projection, and every block sums the partials in the same fixed order
// (lane-strided, then an xor butterfly: a+b == b+a, so all lanes agree).
__global__ void __launch_bounds__(256) k_mgs_coop(const double *__restrict__ V, double *__restrict__ w, long long n,
                                                  int j, double *__restrict__ H, double *__restrict__ part) {
  __shared__ double sh[33];
  __shared__ double s_h;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const long long chunk = (n + G - 1) / G;
  const long long lo = (long long)b * chunk, hi = min(n, lo + chunk);
  double h = 0.0;
  for (int i = 0; i <= j + 1; ++i) {
    const double *Vp = V + (long long)(i - 1) * n;
    const double *Vi = V + (long long)i * n;
    double s = 0.0;
    for (long long k = lo + threadIdx.x; k < hi; k += blockDim.x) {
      double wk = w[k];
      if (i > 0) {
        wk = __dsub_rn(wk, __dmul_rn(h, Vp[k]));
        w[k] = wk;
      }
      s = (i <= j) ? fma(Vi[k], wk, s) : fma(wk, wk, s);
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[(i & 1) * G + b] = s;
    grid.sync();
    if (threadIdx.x < 32) {  // lane-strided partials + xor butterfly: every block gets the same bits
      double t = 0.0;
      for (int q = threadIdx.x; q < G; q += 32) t += __ldcg(part + (i & 1) * G + q);
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) s_h = t;
    }
    __syncthreads();
    h = s_h;
    if (b == 0 && threadIdx.x == 0) H[i] = (i <= j) ? h : sqrt(h);
  }
}

// k_mgs_coop with the block's slice of w held in registers and its slice of
// the previous basis vector in shared memory (R elements per thread, the same
// elements in the same order, so the same bits): one read of V_0 .. V_j and of
// w and one write of w, instead of reading V_{i-1}, V_i and w and writing w for
// every projection. Dynamic shared memory: R * 256 doubles.
template <int R>
__global__ void __launch_bounds__(256, R >= 16 ? 2 : 1) k_mgs_reg(const double *__restrict__ V, double *__restrict__ w,
                                                                  long long n, int j, double *__restrict__ H,
                                                                  double *__restrict__ part) {
  extern __shared__ double vps[];  // [R][256]: this thread's V_{i-1} entries
  __shared__ double sh[33];
  __shared__ double s_h;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const long long chunk = (n + G - 1) / G;
  const long long lo = (long long)b * chunk, hi = min(n, lo + chunk);
  // this thread's elements: lo + tid + 256 u for u < cnt (ascending, as k_mgs_coop)
  const int cnt = hi > lo + threadIdx.x ? (int)((hi - lo - threadIdx.x + 255) / 256) : 0;
  double *wb = w + lo + threadIdx.x;
  double wv[R];
#pragma unroll
  for (int u = 0; u < R; ++u) wv[u] = u < cnt ? wb[256 * u] : 0.0;
  double h = 0.0;
  for (int i = 0; i <= j + 1; ++i) {
    const double *vb = V + (long long)i * n + lo + threadIdx.x;
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < R; ++u) {
      if (u < cnt) {
        double wk = wv[u];
        if (i > 0) {
          wk = __dsub_rn(wk, __dmul_rn(h, vps[u * 256 + threadIdx.x]));
          wv[u] = wk;
        }
        if (i <= j) {
          const double vi = vb[256 * u];
          vps[u * 256 + threadIdx.x] = vi;
          s = fma(vi, wk, s);
        } else {
          s = fma(wk, wk, s);
        }
      }
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[(i & 1) * G + b] = s;
    grid.sync();
    if (threadIdx.x < 32) {
      double t = 0.0;
      for (int q = threadIdx.x; q < G; q += 32) t += __ldcg(part + (i & 1) * G + q);
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) s_h = t;
    }
    __syncthreads();
    h = s_h;
    if (b == 0 && threadIdx.x == 0) H[i] = (i <= j) ? h : sqrt(h);
  }
#pragma unroll
  for (int u = 0; u < R; ++u)
    if (u < cnt) wb[256 * u] = wv[u];
}

// CSR SpMV, one warp per row (A @ x, sparse.py:277-284)
// CSR SpMV with W lanes per row (W = 4, 8, 16: the power of two at or above
// the average row length), so short stencil rows (7 / 9 / 27 nonzeros) keep
// every lane busy: lane-strided partial sums, then an xor tree in the group
template <int W>
__global__ void __launch_bounds__(256) k_spmv_sub(long long nrows, const long long *__restrict__ ptr,
                                                  const int *__restrict__ col, const double *__restrict__ val,
                                                  const double *__restrict__ x, double *__restrict__ y) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int l = threadIdx.x & (W - 1);
  const long long ng = ((long long)gridDim.x * blockDim.x) / W;
  for (long long r = t / W; r < nrows; r += ng) {
    double s = 0.0;
    const long long p1 = __ldg(ptr + r + 1);
    for (long long p = __ldg(ptr + r) + l; p < p1; p += W) s = fma(__ldg(val + p), __ldg(x + __ldg(col + p)), s);
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, W);
    if (l == 0) y[r] = s;
  }
}

__global__ void __launch_bounds__(256) k_spmv(long long nrows, const long long *__restrict__ ptr,
                                              const int *__restrict__ col,
                                              const double *__restrict__ val,
                                              const double *__restrict__ x, double *__restrict__ y) {
  long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = warp; r < nrows; r += nw) {
    double s = 0.0;
    for (long long p = ptr[r] + lane; p < ptr[r + 1]; p += 32) s = fma(val[p], x[col[p]], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = s;
  }
}

// ---------------------------------------------------------------------------
// Streamed CSR SpMV (A @ x, sparse.py:277-284): the matrix streams through
// shared memory by TMA bulk copies (cp.async.bulk + mbarrier complete_tx), two
// stages per CTA, persistent CTAs over chunks of R consecutive rows.
//   stage  = row pointers [r0, r0 + rows], values and columns [p0, p1) of the chunk
//   pass A = every thread turns entries into products val * x[col] in place
//            (entry-strided: the x gathers of a chunk are all in flight at once)
//   pass B = one thread per row adds its products in ascending entry order from 0
// The arithmetic is the reference's scipy CSC product (y[i] += a_ij * x_j over
// ascending j, a rounded product then a rounded add): bit-identical for a CSR
// with ascending columns. Bulk copies need 16-byte aligned ends: the copied
// ranges are widened to even (double) / multiple-of-4 (int) entry offsets, and
// the arrays carry that much slack (mfh_csr_create).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra D_%=;\n"
      "bra W_%=;\n"
      "D_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void *smem_dst, const void *gsrc, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int SPMV_MAX_STG = 4;
// shared-memory bytes of one stage: values (cap + 2), row pointers (R + 4, 4 or 8 bytes each),
// columns (cap + 8); R a multiple of 4, cap even
__host__ __device__ inline size_t spmv_stage_bytes(int R, int cap, int ptr_bytes) {
  return (size_t)8 * (cap + 2) + (size_t)ptr_bytes * (R + 4) + (((size_t)4 * (cap + 8) + 15) & ~(size_t)15);
}

// PT: the row-pointer type streamed (int when nnz < 2^31: the 4-byte pointers of the byte count)
template <typename PT, bool HALO>
__global__ void __launch_bounds__(256) k_spmv_stream(long long nrows, int R, int cap, int nst, long long nchunks,
                                                     const PT *__restrict__ ptr, const int *__restrict__ col,
                                                     const double *__restrict__ val, const double *__restrict__ x,
                                                     const double *__restrict__ halo, int nl, double *__restrict__ y) {
  // HALO: column j < nl reads x[j], j >= nl the halo buffer (distributed SpMV: other ranks'
  // separator values)
  extern __shared__ __align__(128) unsigned char spmv_smem[];
  __shared__ unsigned long long bar[SPMV_MAX_STG];
  constexpr int PB = (int)sizeof(PT), PA = 16 / PB;  // pointers per 16 bytes
  const size_t stb = spmv_stage_bytes(R, cap, PB);
  auto sval = [&](int s) { return reinterpret_cast<double *>(spmv_smem + stb * s); };
  auto sptr = [&](int s) { return reinterpret_cast<PT *>(spmv_smem + stb * s + (size_t)8 * (cap + 2)); };
  auto scol = [&](int s) {
    return reinterpret_cast<int *>(spmv_smem + stb * s + (size_t)8 * (cap + 2) + (size_t)PB * (R + 4));
  };
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // thread 0 issues the three bulk copies of chunk c into stage s
  auto issue = [&](long long c, int s, long long p0, long long p1) {
    const long long r0 = c * R;
    const int rows = (int)min((long long)R, nrows - r0);
    const long long v0 = p0 & ~1LL, v1 = (p1 + 1) & ~1LL;
    const long long c0 = p0 & ~3LL, c1 = (p1 + 3) & ~3LL;
    const unsigned bp = (unsigned)(PB * ((rows + PA) & ~(PA - 1)));  // rows + 1 pointers, rounded up to 16 bytes
    const unsigned bv = (unsigned)(8 * (v1 - v0)), bc = (unsigned)(4 * (c1 - c0));
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    mbar_expect_tx(&bar[s], bp + bv + bc);
    tma_bulk_g2s(sptr(s), ptr + r0, bp, &bar[s]);
    if (bv) tma_bulk_g2s(sval(s), val + v0, bv, &bar[s]);
    if (bc) tma_bulk_g2s(scol(s), col + c0, bc, &bar[s]);
  };
  auto xin = [&](int j) { return (!HALO || j < nl) ? __ldg(x + j) : __ldg(halo + (j - nl)); };
  const long long G = gridDim.x;
  long long np0 = 0, np1 = 0;  // thread 0: entry range of the chunk it issues next
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      const long long c = blockIdx.x + s * G;
      if (c < nchunks) issue(c, s, (long long)__ldg(ptr + c * R), (long long)__ldg(ptr + min(nrows, (c + 1) * R)));
    }
  }
  // programmatic dependent launch: the matrix never changes, so the first stages are already
  // streaming in while the preceding kernel (the producer of x) drains; x and y only after the wait
  pdl_wait();
  pdl_trigger();
  int s = 0;
  unsigned par = 0;
  for (long long c = blockIdx.x; c < nchunks; c += G) {
    const long long cn = c + nst * G;  // the chunk that reuses this stage
    if (tid == 0 && cn < nchunks) {
      np0 = (long long)__ldg(ptr + cn * R);
      np1 = (long long)__ldg(ptr + min(nrows, (cn + 1) * R));
    }
    mbar_wait(&bar[s], par);
    const long long r0 = c * R;
    const int rows = (int)min((long long)R, nrows - r0);
    const PT *sp = sptr(s);
    const long long p0 = sp[0], p1 = sp[rows];
    double *sv = sval(s) - (p0 & ~1LL);  // entry p at sv[p]
    const int *sc = scol(s) - (p0 & ~3LL);
    {
      long long p = p0 + tid;
      for (; p + 768 < p1; p += 1024) {  // four independent gathers in flight per thread
        const int j0 = sc[p], j1 = sc[p + 256], j2 = sc[p + 512], j3 = sc[p + 768];
        const double x0 = xin(j0), x1 = xin(j1), x2 = xin(j2), x3 = xin(j3);
        sv[p] = __dmul_rn(sv[p], x0);
        sv[p + 256] = __dmul_rn(sv[p + 256], x1);
        sv[p + 512] = __dmul_rn(sv[p + 512], x2);
        sv[p + 768] = __dmul_rn(sv[p + 768], x3);
      }
      for (; p < p1; p += 256) sv[p] = __dmul_rn(sv[p], xin(sc[p]));
    }
    __syncthreads();
    for (int r = tid; r < rows; r += 256) {
      double acc = 0.0;
      const long long e = sp[r + 1];
      for (long long p = sp[r]; p < e; ++p) acc = __dadd_rn(acc, sv[p]);
      y[r0 + r] = acc;
    }
    __syncthreads();
    if (tid == 0 && cn < nchunks) issue(cn, s, np0, np1);
    if (++s == nst) { s = 0; par ^= 1u; }
  }
}

// ---------------------------------------------------------------------------
// baseline preconditioners (krylov.py:164-204)
// ---------------------------------------------------------------------------
// y = x / d (diagonal_preconditioner: v / diag, IEEE division, bit-exact)
__global__ void k_diag_div(long long n, const double *__restrict__ d, const double *__restrict__ x,
                           double *__restrict__ y) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i] / d[i];
}

// One level of a sparse triangular solve (ILUT apply), one thread per row of
// the level: lower unit (x_i = b_i - sum_p v_p x_{j_p}) or upper with the
// diagonal first in the row (x_i = (b_i - sum_{p > first} v_p x_{j_p}) / v_first).
// The products and differences are rounded separately in the row's entry
// order (__dmul_rn / __dsub_rn: no FMA contraction), exactly like the
// reference's scalar loops (_core.pyx:272-305), so the apply is bit-identical.
__global__ void k_trsv_level(const int *__restrict__ rows, int nrows, const long long *__restrict__ ptr,
                             const int *__restrict__ idx, const double *__restrict__ val, const double *__restrict__ b,
                             double *__restrict__ x, int upper) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int i = rows[t];
  double s = b[i];
  const long long p0 = ptr[i] + (upper ? 1 : 0), p1 = ptr[i + 1];
  for (long long p = p0; p < p1; ++p) s = __dsub_rn(s, __dmul_rn(val[p], x[idx[p]]));
  x[i] = upper ? s / val[ptr[i]] : s;
}

}  // namespace mfh

#include "gemm_big.cuh"
