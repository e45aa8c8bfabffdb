// Host orchestrator for the B200 HODLR-multifrontal factorization, the
// preconditioner apply and GMRES, plus their C-ABI entry points.
//
// Schedule: the elimination tree is processed by HEIGHT (children strictly
// below parents), every front of a height in the same batched launches:
//   dense fronts  (front < n_c): sample (assemble + extend-add), getrf(F_pp),
//                                getrs(F_pp, F_pf), Schur GEMM  (multifrontal.py:283-310)
//   structured fronts (>= n_c): sample leaves + BDLR panels, complete-pivot LU
//                                of every core, [one host sync for the ranks],
//                                skeleton TRSMs / dense fallbacks, level-batched
//                                HODLR factorization, W/V update (multifrontal.py:353-456)
// BDLR selections (bdlr.py:89-136) are integer graph work done on the host.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <atomic>
#include <mutex>
#include <thread>

#include "internal.h"
#include "kernels.cuh"

namespace mfh {

thread_local std::string g_last_error;
void set_last_error(const std::string &m) { g_last_error = m; }

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x);    \
  } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// device memory: chunked bump arena
// ---------------------------------------------------------------------------
// device chunks are recycled through a per-context pool: factorizations of
// the same pattern reuse the previous one's memory instead of cudaMalloc/Free
// inside the timed step
struct ChunkPool {
  std::vector<std::pair<char *, size_t>> free_chunks;
  // MFH_POOL_TRACE: device allocations that missed the pool (count, bytes, host ms) and retries
  int64_t miss_calls = 0, retry_calls = 0;
  double miss_bytes = 0.0, miss_ms = 0.0;
  std::pair<char *, size_t> take(size_t need) {
    auto t0_ = std::chrono::steady_clock::now();
    struct Clock {
      ChunkPool *p;
      std::chrono::steady_clock::time_point t0;
      bool on = false;
      ~Clock() {
        if (on) p->miss_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      }
    } clk{this, t0_};
    int best = -1;
    for (int q = 0; q < (int)free_chunks.size(); ++q)
      if (free_chunks[q].second >= need && (best < 0 || free_chunks[q].second < free_chunks[best].second))
        best = q;
    if (best >= 0) {
      auto c = free_chunks[best];
      free_chunks.erase(free_chunks.begin() + best);
      return c;
    }
    char *p = nullptr;
    clk.on = true;
    miss_calls++;
    miss_bytes += (double)need;
    if (cudaMalloc(&p, need) != cudaSuccess) {
      retry_calls++;
      // free chunks of the wrong sizes can hold the memory a larger request
      // needs (C5): return them to the device and retry once. A free chunk may
      // still be read by enqueued work (release arenas hand chunks back as soon
      // as their last reader is enqueued), so the device drains first; the
      // cudaFree below must never race those kernels, even if it becomes
      // stream-ordered.
      (void)cudaGetLastError();
      CK(cudaDeviceSynchronize());
      release();
      if (cudaMalloc(&p, need) != cudaSuccess) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        fprintf(stderr, "[mfh] out of device memory: chunk of %.1f MB requested, %.1f of %.1f GB free\n",
                need / 1e6, fr / 1e9, tot / 1e9);
        CK(cudaErrorMemoryAllocation);
      }
    }
    return {p, need};
  }
  void give(std::pair<char *, size_t> c) { free_chunks.push_back(c); }
  void release() {
    for (auto &c : free_chunks) cudaFree(c.first);
    free_chunks.clear();
  }
};

struct Arena {
  std::vector<std::pair<char *, size_t>> chunks;
  size_t cur = 0, off = 0;
  size_t chunk = size_t(256) << 20;
  size_t in_use = 0, peak = 0;
  ChunkPool *pool = nullptr;
  void *alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    while (true) {
      if (cur < chunks.size()) {
        if (off + bytes <= chunks[cur].second) {
          void *p = chunks[cur].first + off;
          off += bytes;
          in_use += bytes;
          peak = std::max(peak, in_use);
          return p;
        }
        ++cur;
        off = 0;
        continue;
      }
      size_t sz = std::max(chunk, bytes);
      if (pool) {
        chunks.push_back(pool->take(sz));
      } else {
        char *p = nullptr;
        CK(cudaMalloc(&p, sz));
        chunks.push_back({p, sz});
      }
    }
  }
  double *d(size_t n) { return (double *)alloc(n * sizeof(double)); }
  int *i(size_t n) { return (int *)alloc(n * sizeof(int)); }
  void reset() {
    cur = 0;
    off = 0;
    in_use = 0;
  }
  void release() {
    for (auto &c : chunks) {
      if (pool)
        pool->give(c);
      else
        cudaFree(c.first);
    }
    chunks.clear();
    reset();
  }
  size_t capacity() const {
    size_t s = 0;
    for (auto &c : chunks) s += c.second;
    return s;
  }
};

// pinned staging for descriptor arrays: async H2D from pinned chunks into
// matching device chunks; chunks are only rewound at stream sync points, so a
// descriptor stays valid until the kernels that read it have completed
struct Stage {
  struct Chunk {
    char *h = nullptr, *d = nullptr;
    size_t cap = 0;
  };
  std::vector<Chunk> chunks;
  size_t cur = 0, off = 0, chunk = size_t(64) << 20;
  void init(size_t c) { chunk = c; }
  // returns (host, device) addresses for `bytes`
  std::pair<char *, char *> take(size_t bytes) {
    size_t b = (bytes + 255) & ~size_t(255);
    while (true) {
      if (cur < chunks.size()) {
        if (off + b <= chunks[cur].cap) {
          auto r = std::make_pair(chunks[cur].h + off, chunks[cur].d + off);
          off += b;
          return r;
        }
        ++cur;
        off = 0;
        continue;
      }
      Chunk c;
      c.cap = std::max(chunk, b);
      CK(cudaMallocHost(&c.h, c.cap));
      CK(cudaMalloc(&c.d, c.cap));
      chunks.push_back(c);
    }
  }
  void rewind() {
    cur = 0;
    off = 0;
  }
  void release() {
    for (auto &c : chunks) {
      cudaFreeHost(c.h);
      cudaFree(c.d);
    }
    chunks.clear();
    rewind();
  }
};

// Chunked bump allocator for data that dies during the factorization (dense
// front buffers: read by the parent's sampler, dead afterwards). Each chunk
// keeps the latest release height of its allocations and goes back to the
// pool once that height has been enqueued; every reader runs earlier on the
// same stream, so reuse is stream-ordered after it.
struct ReleaseArena {
  struct Chunk {
    char *p;
    size_t cap, off;
    int rh;
  };
  std::vector<Chunk> live;
  ChunkPool *pool = nullptr;
  size_t chunk = size_t(64) << 20;
  size_t held = 0, peak = 0;
  void *alloc(size_t bytes, int rh) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    if (!live.empty()) {
      Chunk &c = live.back();
      if (c.off + bytes <= c.cap) {
        void *p = c.p + c.off;
        c.off += bytes;
        c.rh = std::max(c.rh, rh);
        return p;
      }
    }
    auto t = pool->take(std::max(chunk, bytes));
    live.push_back(Chunk{t.first, t.second, bytes, rh});
    held += t.second;
    peak = std::max(peak, held);
    return t.first;
  }
  double *d(size_t n, int rh) { return (double *)alloc(n * sizeof(double), rh); }
  void release_upto(int h) {
    for (size_t i = 0; i < live.size();) {
      if (live[i].rh > h) {
        ++i;
      } else if (i + 1 == live.size()) {  // the open chunk: everything in it is dead, reuse it
        live[i].off = 0;
        live[i].rh = -1;
        ++i;
      } else {
        pool->give({live[i].p, live[i].cap});
        held -= live[i].cap;
        live.erase(live.begin() + i);
      }
    }
  }
  void release_all() {
    for (auto &c : live) pool->give({c.p, c.cap});
    live.clear();
    held = 0;
  }
};

// host -> device upload ordered on the library stream (a plain cudaMemcpy from
// pageable memory is only ordered on the legacy default stream)
static void upload(cudaStream_t st, void *dst, const void *src, size_t bytes) {
  if (bytes == 0) return;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
}

struct Ctx {
  int device = 0;
  cudaStream_t s = nullptr;
  cudaStream_t side = nullptr;   // concurrent large-core cluster / cooperative kernels
  cudaStream_t side2 = nullptr;  // 8-CTA cluster cores, concurrently with the 16-CTA ones
  cudaStream_t side3 = nullptr;  // the cooperative grid-class cores when launched first
  cudaStream_t side4 = nullptr;  // the one-CTA pivot-LU cores, beside the dense fronts' work
  cudaStream_t la = nullptr;     // blocked LU look-ahead: the next panel beside the trailing update
  cudaEvent_t ev_la_cols = nullptr, ev_la_panel = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr, ev_join3 = nullptr;
  cudaEvent_t ev_fork2 = nullptr, ev_join4 = nullptr;
  cudaEvent_t gmres_ev[2] = {nullptr, nullptr};  // Hessenberg column read-backs (pipelined Arnoldi)
  int cluster_size = 16;
  size_t plu_dyn_max = 0;  // dynamic shared memory the pivot-LU kernels may use (per device)
  int nsm = 148;
  ChunkPool pool;
  std::vector<cudaEvent_t> evpool;  // per-height phase events, reused
  std::vector<cudaEvent_t> evd_pool;  // per height: end of the child-update materialization (trace)
  Stage stage;
  Arena scratch;
  double *d_part = nullptr;  // reduction partials
  double *d_scal = nullptr;  // small device scalars
  double *h_scal = nullptr;  // pinned host mirror for GMRES read-backs
  char *h_rb = nullptr;      // pinned landing area for the per-height rank read-back
  size_t h_rb_cap = 0;
  char *readback(size_t bytes) {
    if (bytes > h_rb_cap) {
      if (h_rb) CK(cudaFreeHost(h_rb));
      h_rb_cap = std::max(bytes, std::max(h_rb_cap * 2, size_t(1) << 20));
      CK(cudaMallocHost(&h_rb, h_rb_cap));
    }
    return h_rb;
  }
  // every C entry point holds this while it uses the context (recursive: a
  // GMRES host-callback preconditioner may re-enter on the same thread)
  std::recursive_mutex mu;
  int64_t launches = 0;      // launches of this library's kernels
  int64_t h2d_copies = 0, h2d_single = 0;  // staged host-to-device copies issued (all / outside batched stretches)
  int64_t lib_calls = 0;     // cuBLAS DGEMM calls (only with MFH_GEMM_ROUTE=blas)
  int64_t big_gemm_jobs = 0; // large plain GEMMs run on k_gemm_big
  double flops_exec = 0.0;   // flops enqueued by run_gemm (2mnk) and the register inverses (2n^3)
  cublasHandle_t blas = nullptr;
  void *blas_ws = nullptr;  // cuBLAS workspace (set once with the stream)
  // device copies of per-tree extend-add maps and front id lists, keyed by etree uid
  std::vector<std::pair<uint64_t, int *>> map_dev;
  std::vector<std::pair<uint64_t, long long *>> ids_dev;
  struct PatDev {  // permuted matrix pattern + gather map, keyed by symcache generation
    uint64_t gen = 0;
    long long *ptr = nullptr, *src = nullptr;
    int *col = nullptr;
  };
  std::vector<PatDev> pat_dev;
  // per-tree apply structure: contribution CSR over global ids (post order);
  // shared with the apply plans of live factors, so eviction never frees it
  // under a factor
  struct ApplySym {
    uint64_t uid = 0;
    int64_t tot = 0;
    std::vector<int64_t> off;  // contribution slot offset per post index (-1: none)
    long long *d_cptr = nullptr, *d_coff = nullptr, *d_fro = nullptr;
    ~ApplySym() {
      cudaFree(d_cptr);
      cudaFree(d_coff);
      cudaFree(d_fro);
    }
  };
  std::vector<std::shared_ptr<ApplySym>> apply_sym;
  // the per-tree device caches keep the most recent trees only
  static constexpr size_t SYM_CACHE_MAX = 8;
};

// ---------------------------------------------------------------------------
// Sink: where descriptors go and how launches happen.
//   immediate: staged async copy, launch now (factorization)
//   batched:   between begin_batch() and flush(), descriptor copies are only
//              staged and launches deferred; flush() issues the copies as few
//              contiguous transfers, then every launch back to back (no copy
//              between two kernels: programmatic dependent launch overlaps
//              them). Only for stretches without host read-backs.
//   record:    persistent copy, launch recorded for graph capture (apply)
// ---------------------------------------------------------------------------
struct Sink {
  Ctx *ctx;
  Arena *persist = nullptr;  // record mode
  bool record = false;
  bool batching = false;
  std::vector<std::function<void(cudaStream_t)>> ops;
  struct Pending {
    char *dst;
    const char *src;
    size_t bytes;
  };
  std::vector<Pending> pend;
  std::vector<std::function<void(cudaStream_t)>> deferred;

  void begin_batch() {
    if (record) return;
    batching = true;
  }
  void flush() {
    if (!batching) return;
    batching = false;
    // coalesce staged ranges that follow each other on both sides; the staging ring hands out
    // 256-byte aligned pieces, so up to 255 bytes of padding may lie between two ranges (copied
    // along: it is padding on the device side too)
    for (size_t q = 0; q < pend.size();) {
      char *d = pend[q].dst;
      const char *h = pend[q].src;
      size_t b = pend[q].bytes;
      size_t r = q + 1;
      while (r < pend.size()) {
        const ptrdiff_t gd = pend[r].dst - (d + b), gh = pend[r].src - (h + b);
        if (gd != gh || gd < 0 || gd >= 256) break;
        b += (size_t)gd + pend[r++].bytes;
      }
      CK(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, ctx->s));
      ctx->h2d_copies++;
      q = r;
    }
    pend.clear();
    auto ops_ = std::move(deferred);
    deferred.clear();
    for (auto &f : ops_) {
      ctx->launches++;
      f(ctx->s);
    }
  }
  ~Sink() {
    if (batching && !std::uncaught_exceptions()) flush();
  }
  // host -> device copy of staged bytes (now, or at flush when batching)
  void h2d(void *dst, const void *src, size_t bytes) {
    if (batching) {
      pend.push_back(Pending{(char *)dst, (const char *)src, bytes});
      return;
    }
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->s));
    ctx->h2d_copies++;
    ctx->h2d_single++;
  }

  void sync_reset() {
    if (batching) throw std::logic_error("internal: stream sync inside a batched stretch");
    CK(cudaStreamSynchronize(ctx->s));
    ctx->stage.rewind();
  }
  void *push_bytes(const void *src, size_t bytes) {
    if (bytes == 0) return nullptr;
    if (record) {  // persistent copy, staged asynchronously (ordered on the stream)
      void *p = persist->alloc(bytes);
      auto hd = ctx->stage.take(bytes);
      std::memcpy(hd.first, src, bytes);
      CK(cudaMemcpyAsync(p, hd.first, bytes, cudaMemcpyHostToDevice, ctx->s));
      return p;
    }
    auto hd = ctx->stage.take(bytes);
    std::memcpy(hd.first, src, bytes);
    h2d(hd.second, hd.first, bytes);
    return hd.second;
  }
  template <class T>
  T *push(const std::vector<T> &v) {
    return (T *)push_bytes(v.data(), v.size() * sizeof(T));
  }
  // copy into scratch device memory that survives until the end of the height
  template <class T>
  T *push_keep(const std::vector<T> &v) {
    size_t bytes = v.size() * sizeof(T);
    if (bytes == 0) return nullptr;
    if (record) return push(v);
    void *dst = ctx->scratch.alloc(bytes);
    auto hd = ctx->stage.take(bytes);
    std::memcpy(hd.first, v.data(), bytes);
    h2d(dst, hd.first, bytes);
    return (T *)dst;
  }
  // several arrays in one staged copy into scratch (valid to the end of the
  // height): one H2D transfer instead of one per array (each costs GPU time)
  std::vector<char *> push_keep_many(const std::vector<std::pair<const void *, size_t>> &parts) {
    size_t tot = 0;
    for (auto &p : parts) tot += (p.second + 255) & ~size_t(255);
    std::vector<char *> out;
    if (tot == 0) {
      out.assign(parts.size(), nullptr);
      return out;
    }
    char *dst = record ? (char *)persist->alloc(tot) : (char *)ctx->scratch.alloc(tot);
    auto hd = ctx->stage.take(tot);
    size_t o = 0;
    for (auto &p : parts) {
      if (p.second) std::memcpy(hd.first + o, p.first, p.second);
      out.push_back(p.second ? dst + o : nullptr);
      o += (p.second + 255) & ~size_t(255);
    }
    if (record)
      CK(cudaMemcpyAsync(dst, hd.first, tot, cudaMemcpyHostToDevice, ctx->s));
    else
      h2d(dst, hd.first, tot);
    return out;
  }
  double *scratch_d(size_t n) { return record ? persist->d(n) : ctx->scratch.d(n); }
  // async host -> device copy into caller-owned device memory through the
  // pinned staging ring (valid until the next sync rewinds it)
  void push_to(void *dst, const void *src, size_t bytes) {
    if (bytes == 0) return;
    auto hd = ctx->stage.take(bytes);
    std::memcpy(hd.first, src, bytes);
    h2d(dst, hd.first, bytes);
  }
  int *scratch_i(size_t n) { return record ? persist->i(n) : ctx->scratch.i(n); }
  void launch(std::function<void(cudaStream_t)> f) {
    if (record) {
      ops.push_back(std::move(f));
    } else if (batching) {
      deferred.push_back(std::move(f));
    } else {
      ctx->launches++;
      f(ctx->s);
    }
  }
};

static void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw runtime_error(std::string("CUDA launch error: ") + cudaGetErrorString(e));
}

// Launch with programmatic stream serialization (PDL). Captured into the
// apply graph it becomes a programmatic edge: the kernel's CTAs launch while
// the previous level drains and block in griddepcontrol.wait until its writes
// are visible, which hides the launch gap between dependent launches (apply levels, HODLR
// levels, panel steps). MFH_PDL=0 launches them ordinarily (A/B).
static bool pdl_on() {
  const char *e = getenv("MFH_PDL");
  return !(e && atoi(e) == 0);
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, args...));
}


// ---- batched launch helpers -------------------------------------------------
// Batched GEMM dispatch: large plain GEMMs (>= 2^27 flops, both sides >= 64,
// C not aliasing A or B) go to cuBLAS DGEMM (FP64 tensor cores); the many
// small / aliased ones to the batched tile kernel k_gemm.
// Per-operation host clock (MFH_OP_TRACE=1; with CUDA_LAUNCH_BLOCKING=1 the
// host time of an operation is its GPU time): where a factorization goes.
struct OpClock {
  static std::map<std::string, std::pair<double, int64_t>> &table() {
    static std::map<std::string, std::pair<double, int64_t>> t;
    return t;
  }
  static bool on() {
    static const bool o = getenv("MFH_OP_TRACE") != nullptr;
    return o;
  }
  const char *name;
  std::chrono::steady_clock::time_point t0;
  explicit OpClock(const char *n) : name(n), t0(std::chrono::steady_clock::now()) {}
  ~OpClock() {
    if (!on()) return;
    auto &e = table()[name];
    e.first += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    e.second++;
  }
  static void dump() {
    if (!on()) return;
    for (auto &kv : table())
      fprintf(stderr, "[mfh op] %-18s %10.1f ms %8lld calls\n", kv.first.c_str(), kv.second.first,
              (long long)kv.second.second);
  }
};
// host-side time spent in library GEMM calls (MFH_HEIGHT_TRACE diagnostics)
static double g_blas_host_ms = 0.0;
static int64_t g_blas_calls = 0;
// Do C and A (or B) share an element? Row-major blocks inside one buffer with
// the same leading dimension (e.g. F_ff and F_fp of one front) are tested
// exactly on the row/column lattice; anything else by address span.
static bool blocks_overlap(const double *p, int rows, int cols, int ld, const double *q, int rows2, int cols2,
                           int ld2) {
  const double *pe = p + (int64_t)(rows - 1) * ld + cols, *qe = q + (int64_t)(rows2 - 1) * ld2 + cols2;
  if (!(p < qe && q < pe)) return false;
  if (ld != ld2 || cols > ld || cols2 > ld) return true;
  const int64_t d = q - p;
  const int64_t c = ((d % ld) + ld) % ld, r0 = (d - c) / ld;
  if (c + cols2 > ld) return true;
  const bool rows_hit = r0 < rows && 0 < r0 + rows2;
  const bool cols_hit = c < cols && 0 < c + cols2;
  return rows_hit && cols_hit;
}
static bool gemm_overlaps(const GemmJob &g) {
  return blocks_overlap(g.C, g.m, g.n, g.ldc, g.A, g.m, g.k, g.lda) ||
         blocks_overlap(g.C, g.m, g.n, g.ldc, g.B, g.k, g.n, g.ldb);
}

static thread_local int g_split_k_override = -1;  // test hook (mfh_test_gemm_batched)
static thread_local int g_route_override = -1;    // test hook: 0 k_gemm_big, 1 cuBLAS, 2 k_gemm for large plain GEMMs
// tiles_only: every job on k_gemm (the sampler's k-ascending chains, so a
// product it forms equals the per-entry one bit for bit), no cuBLAS route
static void run_gemm(Sink &sk, const std::vector<GemmJob> &jobs, bool tiles_only = false) {
  OpClock oc_("gemm");
  if (jobs.empty()) return;
  for (const GemmJob &g : jobs)
    if (g.k > 0 && g.lda >= 0 && g.ldb >= 0) sk.ctx->flops_exec += 2.0 * g.m * g.n * g.k;
  std::vector<GemmTile> tiles;
  std::vector<GemmJob> big;
  std::vector<GemmSplit> splits;
  int nslot = 0;
  // Large plain GEMMs (>= 2^27 flops) go to cuBLAS DGEMM, or with MFH_GEMM_ROUTE=big to
  // k_gemm_big (128-wide tiles, one persistent launch per batch; the same k-ascending DMMA chain
  // as k_gemm, so choosing it never changes a bit of the result): a library-free factorization.
  // Measured on B200 (profiles/r2_gemm_big_probe.txt, r2_ab_gemm_route.txt): k_gemm_big reaches
  // 33.1 TFLOP/s on 4096^3 against the library's 35.2 and beats one-call-per-job cuBLAS on
  // batches of 2^28..2^30-flop jobs (27 vs 19 TFLOP/s), but 90% of C5's large-GEMM flops are in
  // products of 2^35 flops and more, half of them with rows that are not 16-byte aligned:
  // C5 2.88 s/step with the library, 3.14 s without. While a graph is being recorded the large
  // jobs always run on k_gemm_big.
  // A/B knobs: MFH_GEMM_ROUTE=big (no library call at all) / blas (the default) / tiles (or
  // MFH_GEMM_NO_BLAS=1: everything on the 64 x 64 kernel); MFH_GEMM_BLAS_MIN=<flops> sends only
  // jobs of at least that many flops to the library and the smaller large ones to k_gemm_big.
  static const int route_env = [] {
    const char *e = getenv("MFH_GEMM_ROUTE");
    if (e && !strcmp(e, "blas")) return 1;
    if ((e && !strcmp(e, "tiles")) || (getenv("MFH_GEMM_NO_BLAS") && atoi(getenv("MFH_GEMM_NO_BLAS")) != 0)) return 2;
    if (e && !strcmp(e, "big")) return 0;
    return 3;
  }();
  const int route = g_route_override >= 0 ? g_route_override : route_env;
  static const double big_min = getenv("MFH_GEMM_BIG_MIN") ? atof(getenv("MFH_GEMM_BIG_MIN")) : (double)(1 << 27);
  static const double blas_min = getenv("MFH_GEMM_BLAS_MIN") ? atof(getenv("MFH_GEMM_BLAS_MIN")) : 0.0;
  auto is_big = [&](const GemmJob &g) {
    return route != 2 && !tiles_only && g.k > 0 && g.m >= 64 && g.n >= 64 && 2.0 * g.m * g.n * g.k >= big_min &&
           g.lda > 0 && g.ldb > 0 && !gemm_overlaps(g);
  };
  // of the large jobs: which go to the library (never while a graph is being recorded)
  auto to_blas = [&](const GemmJob &g) {
    if (sk.record || route == 0) return false;
    if (route == 1) return true;
    return 2.0 * g.m * g.n * g.k >= blas_min;
  };
  std::vector<GemmJob> lib;
  // products with an identity operand (leading dimension -1: the strip that
  // stands for DenseBlock.as_factors' eye) are scaled copies, not GEMMs
  std::vector<GemmJob> eye;
  std::vector<int> eye_which;
  for (int j = 0; j < (int)jobs.size(); ++j) {
    const GemmJob &g = jobs[j];
    if (g.m <= 0 || g.n <= 0) continue;
    if (g.k > 0 && (g.lda < 0 || g.ldb < 0)) {
      if ((g.lda < 0 && g.m != g.k) || (g.ldb < 0 && g.k != g.n))
        throw runtime_error("internal: identity operand of a GEMM must be square");
      eye.push_back(g);
      eye_which.push_back(g.lda < 0 ? 0 : 1);
      continue;
    }
    if (is_big(g)) {
      static const bool blog = getenv("MFH_GEMM_BIGLOG") != nullptr;  // shapes of the large plain GEMMs
      if (blog)
        fprintf(stderr, "[biggemm] m %d n %d k %d a16 %d b16 %d c16 %d beta %g batch %zu\n", g.m, g.n, g.k,
                (int)((((uintptr_t)g.A) & 15) == 0 && g.lda % 2 == 0), (int)((((uintptr_t)g.B) & 15) == 0 && g.ldb % 2 == 0),
                (int)((((uintptr_t)g.C) & 15) == 0 && g.ldc % 2 == 0), g.beta, jobs.size());
      (to_blas(g) ? lib : big).push_back(g);
      continue;
    }
    int tm = (int)cdiv(g.m, GEMM_BM), tn = (int)cdiv(g.n, GEMM_BN);
    // split-K (a rule of the job alone): <= 32 output tiles and k >= 2 chunks
    // -> k chunks of MFH_GEMM_SPLIT_K, partials summed in order by
    // k_gemm_reduce. Off by default: with the prefetched slabs it measured no
    // gain at C2 (0.1282 vs 0.1278 s/step), and at C5 the per-job partials
    // (32 KB per tile per chunk) ran the device out of memory.
    static const int split_k_env = getenv("MFH_GEMM_SPLIT_K") ? atoi(getenv("MFH_GEMM_SPLIT_K")) : 0;
    const int split_k = g_split_k_override >= 0 ? g_split_k_override : split_k_env;
    const int ns = (split_k > 0 && !sk.record && g.k >= 2 * split_k && tm * tn <= 32 && !gemm_overlaps(g))
                       ? (int)cdiv(g.k, split_k)
                       : 1;
    for (int a = 0; a < tm; ++a)
      for (int b = 0; b < tn; ++b) {
        if (ns == 1) {
          tiles.push_back(GemmTile{j, a, b, 0, std::max(g.k, 0), -1});
          continue;
        }
        splits.push_back(GemmSplit{j, a, b, nslot, ns});
        for (int q = 0; q < ns; ++q)
          tiles.push_back(GemmTile{j, a, b, q * split_k, std::min(g.k, (q + 1) * split_k), nslot + q});
        nslot += ns;
      }
  }
  if (!big.empty()) {
    // tile shape of the launch: least padded work, with half a round of the persistent grid
    // charged for the partial last round (128 x 128 runs one CTA per SM, the others two)
    struct Shape { int bm, bn, slots; double eff; };
    const Shape shapes[3] = {{128, 128, sk.ctx->nsm, 1.0}, {128, 64, 2 * sk.ctx->nsm, 1.035}, {64, 128, 2 * sk.ctx->nsm, 1.01}};
    int best = 0;
    double best_est = 0.0;
    for (int c = 0; c < 3; ++c) {
      double work = 0.0, nt = 0.0;
      for (const GemmJob &g : big) {
        const double t = (double)cdiv(g.m, shapes[c].bm) * (double)cdiv(g.n, shapes[c].bn);
        nt += t;
        work += t * shapes[c].bm * shapes[c].bn * g.k;
      }
      const double est = work * shapes[c].eff * (1.0 + 0.5 * shapes[c].slots / nt);
      if (c == 0 || est < best_est) best = c, best_est = est;
    }
    std::vector<GemmBigTile> bt;
    for (int j = 0; j < (int)big.size(); ++j)
      for (int a = 0; a < (int)cdiv(big[j].m, shapes[best].bm); ++a)
        for (int b = 0; b < (int)cdiv(big[j].n, shapes[best].bn); ++b) bt.push_back(GemmBigTile{j, a, b});
    GemmJob *dj = sk.push(big);
    GemmBigTile *dt = sk.push(bt);
    const int nt = (int)bt.size(), grid = std::min(nt, shapes[best].slots);
    sk.launch([=](cudaStream_t st) {
      if (best == 0)
        launch_pdl(k_gemm_big<2, 4, 8, 4, 4, 1>, dim3(grid), dim3(256), GemmBigCfg<2, 4, 8, 4, 4>::SMEM, st, dj, dt, nt);
      else if (best == 1)
        launch_pdl(k_gemm_big<4, 2, 4, 4, 3, 2>, dim3(grid), dim3(256), GemmBigCfg<4, 2, 4, 4, 3>::SMEM, st, dj, dt, nt);
      else
        launch_pdl(k_gemm_big<2, 4, 4, 4, 4, 2>, dim3(grid), dim3(256), GemmBigCfg<2, 4, 4, 4, 4>::SMEM, st, dj, dt, nt);
      check_launch();
    });
    sk.ctx->big_gemm_jobs += (int64_t)big.size();
  }
  if (!lib.empty()) {
    const std::vector<GemmJob> &big = lib;
    Ctx *ctx = sk.ctx;
    if (!ctx->blas) {
      if (cublasCreate(&ctx->blas) != CUBLAS_STATUS_SUCCESS) throw runtime_error("cublasCreate failed");
      // stream and a fixed workspace once per handle: cublasSetStream resets
      // the workspace, so calling it per launch batch re-provisions it
      if (cublasSetStream(ctx->blas, ctx->s) != CUBLAS_STATUS_SUCCESS) throw runtime_error("cublasSetStream failed");
      const size_t ws = size_t(32) << 20;
      CK(cudaMalloc(&ctx->blas_ws, ws));
      if (cublasSetWorkspace(ctx->blas, ctx->blas_ws, ws) != CUBLAS_STATUS_SUCCESS)
        throw runtime_error("cublasSetWorkspace failed");
    }
    auto tb0 = std::chrono::steady_clock::now();
    g_blas_calls += (int64_t)big.size();
    struct BlasClock {
      std::chrono::steady_clock::time_point t0;
      ~BlasClock() {
        g_blas_host_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      }
    } bclk{tb0};
    cublasHandle_t h = ctx->blas;
    sk.launch([h, big](cudaStream_t) {  // the handle's stream is ctx->s (a batched sink defers the calls)
      for (const GemmJob &g : big) {
        // row-major C = alpha A B + beta C  ==  column-major C^T = alpha B^T A^T + beta C^T
        double al = g.alpha, be = g.beta;
        if (cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, g.n, g.m, g.k, &al, g.B, g.ldb, g.A, g.lda, &be, g.C, g.ldc) !=
            CUBLAS_STATUS_SUCCESS)
          throw runtime_error("cublasDgemm failed");
      }
    });
    ctx->lib_calls += (int64_t)big.size();
  }
  if (!eye.empty()) {
    int64_t mx = 1;
    for (auto &g : eye) mx = std::max<int64_t>(mx, (int64_t)g.m * g.n);
    for (size_t b = 0; b < eye.size(); b += 60000) {
      std::vector<GemmJob> part(eye.begin() + b, eye.begin() + std::min(eye.size(), b + 60000));
      std::vector<int> wh(eye_which.begin() + b, eye_which.begin() + std::min(eye.size(), b + 60000));
      GemmJob *dj = sk.push(part);
      int *dw = sk.push(wh);
      dim3 grid((unsigned)std::min<int64_t>(cdiv(mx, 256), 128), (unsigned)part.size());
      sk.launch([=](cudaStream_t st) {
        launch_pdl(k_axpby, dim3(grid), dim3(256), 0, st, dj, dw);
        check_launch();
      });
    }
  }
  if (tiles.empty()) return;
  static const bool glog = getenv("MFH_GEMM_LOG") != nullptr;
  if (glog) {
    int64_t fl = 0;
    int kmax = 0, ov = 0;
    for (auto &g : jobs) {
      fl += 2ll * g.m * g.n * g.k;
      kmax = std::max(kmax, g.k);
      ov += gemm_overlaps(g);
    }
    fprintf(stderr, "[gemm] jobs %zu tiles %zu splits %zu kmax %d overlap %d gflop %.4f first m%d n%d k%d\n",
            jobs.size(), tiles.size(), splits.size(), kmax, ov, fl * 1e-9, jobs[0].m, jobs[0].n, jobs[0].k);
  }
  GemmJob *dj = sk.push(jobs);
  GemmTile *dt = sk.push(tiles);
  GemmSplit *dsp = splits.empty() ? nullptr : sk.push(splits);
  double *dws = nslot ? sk.scratch_d((size_t)nslot * GEMM_BM * GEMM_BN) : nullptr;
  int nt = (int)tiles.size(), nsp = (int)splits.size();
  int grid = std::min(nt, 148 * 16);
  sk.launch([=](cudaStream_t s) {
    launch_pdl(k_gemm, dim3(grid), dim3(256), GEMM_DYN, s, dj, dt, nt, dws);
    check_launch();
    if (nsp) launch_pdl(k_gemm_reduce, dim3(nsp), dim3(256), 0, s, dj, dsp, dws);
    check_launch();
  });
}

// TRSM with a w x w (w <= 64) triangular diagonal block: invert the block
// (k_trinv), then B <- T^{-1} B as an in-place GEMM (safe: m = w fits one
// 64-row GEMM tile, so every CTA reads its whole column strip before writing)
static void run_trsm(Sink &sk, const std::vector<TrsmJob> &jobs) {
  OpClock oc_("trsm");
  if (jobs.empty()) return;
  std::vector<TrinvJob> ti;
  std::vector<GemmJob> gm;
  for (auto &j : jobs) {
    if (j.ncols <= 0 || j.w <= 0) continue;
    double *inv = sk.scratch_d((size_t)j.w * j.w);
    ti.push_back(TrinvJob{j.T, j.ldt, j.w, j.upper, inv});
    gm.push_back(GemmJob{inv, j.B, j.B, j.w, j.ncols, j.w, j.w, j.ldb, j.ldb, 1.0, 0.0});
  }
  if (ti.empty()) return;
  TrinvJob *dj = sk.push(ti);
  int nb = (int)ti.size();
  sk.launch([=](cudaStream_t st) {
    launch_pdl(k_trinv, dim3(nb), dim3(256), TRINV_SMEM, st, dj);
    check_launch();
  });
  run_gemm(sk, gm);
}

constexpr int BIG_N = INV_SMALL;  // above this, LU / solves run blocked across the GPU

static void run_laswp(Sink &sk, const std::vector<SwapJob> &jobs) {
  OpClock oc_("laswp");
  for (size_t b = 0; b < jobs.size(); b += 60000) {
    std::vector<SwapJob> part(jobs.begin() + b, jobs.begin() + std::min(jobs.size(), b + 60000));
    int mx = 1;
    for (auto &j : part) mx = std::max(mx, j.ncols);
    SwapJob *dj = sk.push(part);
    dim3 grid((unsigned)cdiv(mx, 128), (unsigned)part.size());
    sk.launch([=](cudaStream_t st) {
      launch_pdl(k_laswp, dim3(grid), dim3(128), 0, st, dj);
      check_launch();
    });
  }
}

static void run_getrf(Sink &sk, const std::vector<LuJob> &jobs) {
  OpClock oc_("getrf");
  if (jobs.empty()) return;
  std::vector<LuJob> small, big;
  for (auto &j : jobs) (j.n > BIG_N ? big : small).push_back(j);
  if (!small.empty()) {
    int maxn = 0;
    for (auto &j : small) maxn = std::max(maxn, j.n);
    LuJob *dj = sk.push(small);
    int nb = (int)small.size();
    int th = maxn > 128 ? 512 : (maxn > 32 ? 256 : 64);
    sk.launch([=](cudaStream_t s) {
      launch_pdl(k_getrf, dim3(nb), dim3(th), 0, s, dj);
      check_launch();
    });
  }
  if (big.empty()) return;
  int maxn = 0;
  for (auto &j : big) maxn = std::max(maxn, j.n);
  // Look-ahead (MFH_LU_LOOKAHEAD_MIN=<rows>: batches whose largest matrix has at least that many
  // rows; off by default): the trailing update of step c0 is split into the next panel's columns
  // and the rest; once the first part is done the next panel is factored on its own high-priority
  // stream beside the rest of the update (which leaves the panel's columns alone), and the main
  // stream picks the panel up before the next step's row swaps. The split only regroups output
  // tiles: every entry keeps its k chain (bitwise equal, scripts/lu_lookahead_bench.py). Measured
  // neutral on B200 (profiles/r2_ab_lu_lookahead.txt: C5 2.864 vs 2.859 s, C3 0.979 vs 0.992,
  // one 4096^2 inverse 47.5 vs 48.6 ms): a height's panels already run as one launch of up to
  // eight 16-CTA clusters, and a cluster does not get its 16 SMs while the update's grid is resident.
  static const int la_min = getenv("MFH_LU_LOOKAHEAD_MIN") ? atoi(getenv("MFH_LU_LOOKAHEAD_MIN")) : INT_MAX;
  const bool lookahead = !sk.record && maxn >= la_min;
  Ctx *ctx = sk.ctx;
  // panel factorization of columns [c0, c0 + w) of every job that has them; side: on the look-ahead stream
  auto launch_panels = [&](int c0, bool side) {
    std::vector<PanelJob> pj;
    for (auto &j : big) {
      if (j.n <= c0) continue;
      pj.push_back(PanelJob{j.a, j.n, j.lda, c0, std::min(PNB, j.n - c0), j.piv, j.flag});
    }
    if (pj.empty()) return;
    PanelJob *dp = sk.push(pj);
    int np_ = (int)pj.size();
    int mmax = 0;
    for (auto &q : pj) mmax = std::max(mmax, q.n - q.c0);
    int cs = mmax <= PANEL_ROWS_MAX ? 1 : (mmax + PANEL_ROWS_CL - 1) / PANEL_ROWS_CL;
    cudaStream_t la = ctx->la;
    cudaEvent_t e_cols = ctx->ev_la_cols, e_panel = ctx->ev_la_panel;
    const int csmax = ctx->cluster_size;
    sk.launch([=](cudaStream_t main) {
      cudaStream_t s = main;
      if (side) {  // after the next panel's columns have been updated on the main stream
        CK(cudaEventRecord(e_cols, main));
        CK(cudaStreamWaitEvent(la, e_cols, 0));
        s = la;
      }
      if (cs == 1) {
        // every panel of the batch fits one CTA's shared memory
        size_t smem = sizeof(double) * (size_t)mmax * PLD;
        launch_pdl(k_getrf_panel_cta, dim3(np_), dim3(512), smem, s, dp);
        check_launch();
      } else if (cs <= csmax) {
        // shared-memory resident panel across a cluster of cs CTAs
        int rp = (mmax + cs - 1) / cs;
        size_t smem = sizeof(double) * (size_t)rp * PLD + PANEL_CL_SLOTS;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(np_ * cs);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const PanelJob *arg = dp;
        void *args[1] = {(void *)&arg};
        cudaError_t e = cudaLaunchKernelExC(&cfg, (const void *)k_getrf_panel_cl, args);
        if (e != cudaSuccess) throw runtime_error(std::string("panel cluster launch failed: ") + cudaGetErrorString(e));
      } else {
        launch_pdl(k_getrf_panel, dim3(np_), dim3(512), 0, s, dp);
        check_launch();
      }
      if (side) CK(cudaEventRecord(e_panel, la));
    });
  };
  bool panel_ahead = false;  // this step's panel was launched on the look-ahead stream
  for (int c0 = 0; c0 < maxn; c0 += PNB) {
    std::vector<SwapJob> sw;
    std::vector<TrsmJob> tr;
    std::vector<GemmJob> gm, gm_next;
    for (auto &j : big) {
      if (j.n <= c0) continue;
      int w = std::min(PNB, j.n - c0);
      sw.push_back(SwapJob{j.a, j.lda, j.n, j.piv, c0, c0 + w, c0, c0 + w});
      int rest = j.n - c0 - w;
      if (rest > 0) {
        double *A11 = j.a + (int64_t)c0 * j.lda + c0;
        tr.push_back(TrsmJob{A11, j.lda, w, A11 + w, j.lda, rest, 0});
        const double *L21 = A11 + (int64_t)w * j.lda, *U12 = A11 + w;
        double *A22 = A11 + (int64_t)w * j.lda + w;
        const int w2 = lookahead ? std::min(PNB, rest) : 0;  // the next panel's columns first
        if (w2 > 0) gm_next.push_back(GemmJob{L21, U12, A22, rest, w2, w, j.lda, j.lda, j.lda, -1.0, 1.0});
        if (rest > w2) gm.push_back(GemmJob{L21, U12 + w2, A22 + w2, rest, rest - w2, w, j.lda, j.lda, j.lda, -1.0, 1.0});
      }
    }
    if (panel_ahead) {
      cudaEvent_t e_panel = ctx->ev_la_panel;
      sk.launch([=](cudaStream_t main) {
        CK(cudaStreamWaitEvent(main, e_panel, 0));
        ctx->launches--;  // not a kernel
      });
    } else {
      launch_panels(c0, false);
    }
    run_laswp(sk, sw);
    run_trsm(sk, tr);
    panel_ahead = false;
    if (!gm_next.empty()) {
      run_gemm(sk, gm_next);
      launch_panels(c0 + PNB, true);
      panel_ahead = true;
    }
    run_gemm(sk, gm);
  }
  if (panel_ahead) {  // (cannot happen: the last step has no trailing block) keep the streams joined anyway
    cudaEvent_t e_panel = ctx->ev_la_panel;
    sk.launch([=](cudaStream_t main) { CK(cudaStreamWaitEvent(main, e_panel, 0)); });
  }
  LuJob *dj = sk.push(big);
  int nb = (int)big.size();
  sk.launch([=](cudaStream_t s) {
    launch_pdl(k_diag_check, dim3(nb), dim3(256), 0, s, dj);
    check_launch();
  });
}


// Full triangular inverse out = T^{-1} (n x n, ld n) of a unit-lower (upper = 0)
// or non-unit upper (upper = 1) triangle: the 64 x 64 diagonal blocks in one
// k_trinv launch, then recursive doubling over block pairs,
//   lower [[A,0],[C,B]]^-1 = [[Ai,0],[-Bi (C Ai), Bi]]
//   upper [[A,C],[0,B]]^-1 = [[Ai,-Ai (C Bi)],[0,Bi]]
// two batched GEMMs per level: log2(n / 64) dependent levels instead of n / 64
// dependent block-solve steps.
static void run_identity(Sink &sk, const std::vector<double *> &ptrs, const std::vector<int> &dims,
                         const std::vector<int> &lds);
struct TriInvReq {
  const double *T;
  int ldt, n, upper;
  double *out;
};
static void run_tri_inv(Sink &sk, const std::vector<TriInvReq> &reqs) {
  OpClock oc_("tri_inv");
  if (reqs.empty()) return;
  std::vector<double *> ip;
  std::vector<int> idim, ild;
  std::vector<TrinvJob> ti;
  int maxn = 0;
  for (auto &r : reqs) {
    if (r.n <= 0) continue;
    ip.push_back(r.out), idim.push_back(r.n), ild.push_back(r.n);  // zero triangle
    for (int c0 = 0; c0 < r.n; c0 += 64) {
      int w = std::min(64, r.n - c0);
      ti.push_back(TrinvJob{r.T + (int64_t)c0 * r.ldt + c0, r.ldt, w, r.upper, r.out + (int64_t)c0 * r.n + c0, r.n});
    }
    maxn = std::max(maxn, r.n);
  }
  run_identity(sk, ip, idim, ild);
  if (!ti.empty()) {
    TrinvJob *dj = sk.push(ti);
    int nb = (int)ti.size();
    sk.launch([=](cudaStream_t st) {
      launch_pdl(k_trinv, dim3(nb), dim3(256), TRINV_SMEM, st, dj);
      check_launch();
    });
  }
  for (int b = 64; b < maxn; b <<= 1) {
    std::vector<GemmJob> g1, g2;
    for (auto &r : reqs) {
      const int n = r.n;
      for (int k0 = 0; k0 + b < n; k0 += 2 * b) {
        const int k1 = k0 + b, nb = std::min(b, n - k1);
        double *Ai = r.out + (int64_t)k0 * n + k0, *Bi = r.out + (int64_t)k1 * n + k1;
        if (!r.upper) {
          double *tmp = sk.scratch_d((size_t)nb * b);
          const double *C = r.T + (int64_t)k1 * r.ldt + k0;  // nb x b
          g1.push_back(GemmJob{C, Ai, tmp, nb, b, b, r.ldt, n, b, 1.0, 0.0});
          g2.push_back(GemmJob{Bi, tmp, r.out + (int64_t)k1 * n + k0, nb, b, nb, n, b, n, -1.0, 0.0});
        } else {
          double *tmp = sk.scratch_d((size_t)b * nb);
          const double *C = r.T + (int64_t)k0 * r.ldt + k1;  // b x nb
          g1.push_back(GemmJob{C, Bi, tmp, b, nb, nb, r.ldt, n, nb, 1.0, 0.0});
          g2.push_back(GemmJob{Ai, tmp, r.out + (int64_t)k0 * n + k1, b, nb, b, n, nb, n, -1.0, 0.0});
        }
      }
    }
    run_gemm(sk, g1);
    run_gemm(sk, g2);
  }
}

struct InvReq {
  double *a;  // n x n, lda (destroyed for n > INV_SMALL: holds the LU)
  int n, lda;
  double *out;  // inverse (n x n, ldo); may equal a when n <= INV_SMALL
  int ldo;
  int *piv;     // n ints (blocked path)
  int *flag;
};
static void run_copy(Sink &sk, const std::vector<CopyJob> &jobs);
static void run_identity(Sink &sk, const std::vector<double *> &ptrs, const std::vector<int> &dims,
                         const std::vector<int> &lds);

// explicit inverses: in-shared-memory Gauss-Jordan for n <= 128, blocked LU +
// GEMM-based solve against the identity above that
static void run_inverse(Sink &sk, const std::vector<InvReq> &reqs) {
  OpClock oc_("inverse");
  if (reqs.empty()) return;
  std::vector<InvJob> small;
  std::vector<CopyJob> cps;
  std::vector<LuJob> lus;
  std::vector<double *> ip;
  std::vector<int> idim, ild;
  int maxs = 1;
  for (auto &r : reqs) {
    if (r.n <= 0) continue;
    if (r.n <= INV_SMALL) {
      if (r.out != r.a) cps.push_back(CopyJob{r.a, r.out, r.n, r.n, r.lda, r.ldo, nullptr, nullptr});
      small.push_back(InvJob{r.out, r.n, r.ldo, r.flag});
      maxs = std::max(maxs, r.n);
    } else {
      lus.push_back(LuJob{r.a, r.n, r.lda, r.piv, r.flag});
      ip.push_back(r.out);
      idim.push_back(r.n);
      ild.push_back(r.ldo);
    }
  }
  static const bool ilog = getenv("MFH_INV_LOG") != nullptr;
  if (ilog) {
    int mx = 0;
    for (auto &l : lus) mx = std::max(mx, l.n);
    fprintf(stderr, "[mfh inverse] %zu register (<= %d) + %zu blocked (max n %d)\n", small.size(), INV_SMALL,
            lus.size(), mx);
  }
  for (auto &j : small) sk.ctx->flops_exec += 2.0 * j.n * j.n * j.n;
  run_copy(sk, cps);
  if (!small.empty()) {
    // register-tiled Gauss-Jordan: 64-wide tiles (256 threads) or 128-wide (512)
    std::vector<InvJob> s64, s128;
    for (auto &j : small) (j.n <= 64 ? s64 : s128).push_back(j);
    if (!s64.empty()) {
      InvJob *dj = sk.push(s64);
      int nb = (int)s64.size();
      sk.launch([=](cudaStream_t st) {
        launch_pdl(k_inv_reg<8, 2>, dim3(nb), dim3(256), 0, st, dj);
        check_launch();
      });
    }
    if (!s128.empty()) {
      InvJob *dj = sk.push(s128);
      int nb = (int)s128.size();
      sk.launch([=](cudaStream_t st) {
        launch_pdl(k_inv_reg<16, 4>, dim3(nb), dim3(512), 0, st, dj);
        check_launch();
      });
    }
  }
  if (!lus.empty()) {
    // A^{-1} = U^{-1} L^{-1} P: triangular inverses by recursive doubling, P as the
    // row-swapped identity, two GEMMs (log-depth instead of n / 64 solve steps)
    run_getrf(sk, lus);
    std::vector<TriInvReq> ti;
    std::vector<SwapJob> sw;
    std::vector<GemmJob> g1, g2;
    for (size_t q = 0; q < lus.size(); ++q) {
      const LuJob &L = lus[q];
      const int n = L.n;
      double *Li = sk.scratch_d((size_t)n * n), *Ui = sk.scratch_d((size_t)n * n), *T = sk.scratch_d((size_t)n * n);
      ti.push_back(TriInvReq{L.a, L.lda, n, 0, Li});
      ti.push_back(TriInvReq{L.a, L.lda, n, 1, Ui});
      sw.push_back(SwapJob{ip[q], ild[q], n, L.piv, 0, n, 0, 0});
      g1.push_back(GemmJob{Li, ip[q], T, n, n, n, n, ild[q], n, 1.0, 0.0});
      g2.push_back(GemmJob{Ui, T, ip[q], n, n, n, n, n, ild[q], 1.0, 0.0});
    }
    run_tri_inv(sk, ti);
    run_identity(sk, ip, idim, ild);
    run_laswp(sk, sw);
    run_gemm(sk, g1);
    run_gemm(sk, g2);
  }
}

static void run_copy(Sink &sk, const std::vector<CopyJob> &jobs) {
  OpClock oc_("copy");
  for (size_t b = 0; b < jobs.size(); b += 60000) {
    std::vector<CopyJob> part(jobs.begin() + b, jobs.begin() + std::min(jobs.size(), b + 60000));
    int64_t mx = 0;
    for (auto &j : part) mx = std::max<int64_t>(mx, (int64_t)j.m * j.n);
    if (mx == 0) continue;
    CopyJob *dj = sk.push(part);
    dim3 grid((unsigned)std::min<int64_t>(cdiv(mx, 256), 64), (unsigned)part.size());
    sk.launch([=](cudaStream_t s) {
      launch_pdl(k_copy, dim3(grid), dim3(256), 0, s, dj, 0);
      check_launch();
    });
  }
}

static void run_identity(Sink &sk, const std::vector<double *> &ptrs, const std::vector<int> &dims,
                         const std::vector<int> &lds) {
  for (size_t b = 0; b < ptrs.size(); b += 60000) {
    size_t e = std::min(ptrs.size(), b + 60000);
    std::vector<double *> p(ptrs.begin() + b, ptrs.begin() + e);
    std::vector<int> d(dims.begin() + b, dims.begin() + e), l(lds.begin() + b, lds.begin() + e);
    int64_t mx = 0;
    for (int x : d) mx = std::max<int64_t>(mx, (int64_t)x * x);
    double **dp = sk.push(p);
    int *dd = sk.push(d);
    int *dl = sk.push(l);
    dim3 grid((unsigned)std::min<int64_t>(cdiv(mx, 256), 64), (unsigned)p.size());
    sk.launch([=](cudaStream_t s) {
      launch_pdl(k_identity, dim3(grid), dim3(256), 0, s, dp, dd, dl);
      check_launch();
    });
  }
}

// complete-pivot LU of a batch of cores: small cores run with the core in
// shared memory, mid-size cores from L2 with bookkeeping in shared memory,
// large cores on a thread-block cluster (on the side stream, concurrently)
constexpr long long PLU_CTA_MAX = 32 * 1024;  // entries: one CTA with the core in shared memory (if it fits)
constexpr int PLU_CL_NT = 1024;               // threads per CTA of the cluster kernel

// the pivot-LU kernels that opt into large dynamic shared memory
static const void *const *plu_fns() {
  static const void *fns[6] = {(const void *)k_plu_cta2<true, 512>, (const void *)k_plu_cta2<true, 1024>,
                               (const void *)k_plu_cluster3<PLU_CL_NT>, (const void *)k_plu_groups3,
                               (const void *)k_plu_groups<false>,   (const void *)k_plu_groups<true>};
  return fns;
}

// Function attributes (shared-memory opt-ins, non-portable cluster sizes) are
// per DEVICE: set them once per device (the first context created on it), and
// record the device's limits in every context.
static void device_setup(Ctx *ctx) {
  static std::mutex mu;
  static std::vector<int> done;  // devices already configured
  std::lock_guard<std::mutex> lk(mu);
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  CK(cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, ctx->device));
  const void *const *fns = plu_fns();
  size_t stat = 0;
  for (int q = 0; q < 6; ++q) {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, fns[q]));
    stat = std::max(stat, fa.sharedSizeBytes);
  }
  ctx->plu_dyn_max = (size_t)optin - stat - 64;
  const bool first = std::find(done.begin(), done.end(), ctx->device) == done.end();
  if (first) {
    for (int q = 0; q < 6; ++q)
      CK(cudaFuncSetAttribute(fns[q], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->plu_dyn_max));
    CK(cudaFuncSetAttribute(k_trinv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRINV_SMEM));
    CK(cudaFuncSetAttribute(k_getrf_panel_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double) * PANEL_ROWS_MAX * PLD)));
    CK(cudaFuncSetAttribute(k_getrf_panel_cl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double) * PANEL_ROWS_CL * PLD + PANEL_CL_SLOTS)));
    CK(cudaFuncSetAttribute(k_sample_rb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RB_DYN));
    CK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_DYN));
    CK(cudaFuncSetAttribute(k_gemm_big<2, 4, 8, 4, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)GemmBigCfg<2, 4, 8, 4, 4>::SMEM));
    CK(cudaFuncSetAttribute(k_gemm_big<4, 2, 4, 4, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)GemmBigCfg<4, 2, 4, 4, 3>::SMEM));
    CK(cudaFuncSetAttribute(k_gemm_big<2, 4, 4, 4, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)GemmBigCfg<2, 4, 4, 4, 4>::SMEM));
  }
  // 16-CTA clusters need the non-portable opt-in; without it the cluster
  // kernels run 8-CTA clusters
  cudaError_t e1 = cudaFuncSetAttribute(fns[2], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaError_t e2 = cudaFuncSetAttribute(k_getrf_panel_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    (void)cudaGetLastError();
    ctx->cluster_size = 8;
  }
  if (first) done.push_back(ctx->device);
}

// every entry point that uses a context runs on that context's device (and
// restores the caller's current device)
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

static void launch_cluster(const void *fn, int ncores, int cs, size_t smem, cudaStream_t st, const PluJob *dj,
                           const int *dids, double eps) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncores * cs);
  cfg.blockDim = dim3(PLU_CL_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void *args[3] = {(void *)&dj, (void *)&dids, (void *)&eps};
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) throw runtime_error(std::string("cluster launch failed: ") + cudaGetErrorString(e));
}

// main_work (optional) is enqueued on the main stream while the side streams
// run the cluster / cooperative cores
static void run_plu(Sink &sk, const std::vector<PluJob> &jobs, double eps,
                    const std::function<void()> &main_work = nullptr) {
  OpClock oc_("plu");
  if (jobs.empty()) {
    if (main_work) main_work();
    return;
  }
  Ctx *ctx = sk.ctx;
  const size_t dyn_max = ctx->plu_dyn_max;  // set per device in device_setup
  const void *const *fns = plu_fns();
  const int CS = ctx->cluster_size;
  // SMs of the cooperative (grid class) launch: all of them by default;
  // MFH_PLU_GRID caps it so the cluster classes can run beside it (A/B knob)
  const int nsm = getenv("MFH_PLU_GRID") ? std::max(1, std::min(ctx->nsm, atoi(getenv("MFH_PLU_GRID")))) : ctx->nsm;
  const bool coop_first = getenv("MFH_PLU_COOP_FIRST") && atoi(getenv("MFH_PLU_COOP_FIRST")) != 0;
  // A/B knob: the 16-CTA cluster class goes to the grouped cooperative launch
  // (one wave, global-memory exchange) instead of cluster waves
  const bool cl16_to_grid = getenv("MFH_PLU_CL16_GRID") && atoi(getenv("MFH_PLU_CL16_GRID")) != 0;
  auto cta_bytes = [](int m, int n) { return sizeof(double) * (size_t)m * n + sizeof(int) * (size_t)(m + n) + 16; };
  std::vector<int> small[3], cl8, cl16, grd;
  size_t smax[3] = {48 * 1024, 100 * 1024, dyn_max};
  for (int q = 0; q < (int)jobs.size(); ++q) {
    const PluJob &j = jobs[q];
    long long ent = (long long)j.m * j.n;
    size_t wc = cta_bytes(j.m, j.n);
    if (ent <= PLU_CTA_MAX && wc <= dyn_max) {
      small[wc <= smax[0] ? 0 : (wc <= smax[1] ? 1 : 2)].push_back(q);
    } else if (ent < 64 * 1024 && plu_dist_bytes(j.m, j.n, 8, true) <= dyn_max) {
      cl8.push_back(q);
    } else if (plu_dist_bytes(j.m, j.n, CS, true) <= dyn_max && !cl16_to_grid) {
      cl16.push_back(q);
    } else if (plu_dist_bytes(j.m, j.n, nsm, false) <= dyn_max) {
      grd.push_back(q);
    } else {
      throw runtime_error("complete-pivot core too large for the shared-memory bookkeeping");
    }
  }
  // Cores of a class start in launch order as SMs free up (only ~7 16-CTA
  // clusters are co-resident): longest first (steps bounded by min(m, n) and
  // kmax, work per step by m n), so the tail is short.
  auto lpt = [&](std::vector<int> &v) {
    auto cost = [&](int q) {
      const PluJob &j = jobs[q];
      return (double)std::min(std::min(j.m, j.n), j.kmax) * ((double)j.m * j.n);
    };
    std::stable_sort(v.begin(), v.end(), [&](int a, int b) { return cost(a) > cost(b); });
  };
  lpt(cl8);
  lpt(cl16);
  for (auto &v : small) lpt(v);
  PluJob *dj = sk.push(jobs);
  // every descriptor the side stream reads is pushed (on the main stream)
  // BEFORE the fork event, so the side-stream kernels see them
  int *ids_cl16 = sk.push(cl16), *ids_cl8 = sk.push(cl8);
  // grid class: the cooperative launch is split into groups of CTAs, one core
  // sequence per group (LPT over min(m, n), the step-count bound), so large
  // cores of one height factor concurrently; a group whose cores do not fit
  // the shared-memory row layout at its size goes to a second (global-row) launch
  struct GridLaunch {
    std::vector<int> first, cptr, ids;
    size_t smem = 0;
  } gl[2];
  GridScratch gs{};
  if (!grd.empty()) {
    std::vector<int> order = grd;
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      long long sa = std::min(jobs[a].m, jobs[a].n), sb = std::min(jobs[b].m, jobs[b].n);
      if (sa != sb) return sa > sb;
      return a < b;
    });
    // per-step cost model (measured at C2): a latency floor plus the trailing
    // update spread over the group's CTAs; steps bounded by min(m, n). Groups
    // get CTAs in proportion to their work and must keep rows in shared memory.
    const double LAT = 8.0, PER = 4.0e-4;  // us per step, us per entry per CTA
    auto steps = [&](int q) { return (double)std::min(jobs[q].m, jobs[q].n); };
    auto ent = [&](int q) { return (double)jobs[q].m * jobs[q].n; };
    auto gmin = [&](int q) {
      for (int G = 1; G <= nsm; ++G)
        if (plu_dist_bytes(jobs[q].m, jobs[q].n, G, true) <= dyn_max) return G;
      return nsm + 1;
    };
    static const int max_groups = std::getenv("MFH_PLU_MAXGROUPS") ? std::atoi(std::getenv("MFH_PLU_MAXGROUPS"))
                                                                     : std::max(1, nsm / 16);
    double best_cost = 1e300;
    std::vector<std::vector<int>> members;
    std::vector<int> sizes;
    for (int ng = 1; ng <= std::min<int>((int)order.size(), std::max(1, max_groups)); ++ng) {
      std::vector<double> load(ng, 0.0), work(ng, 0.0);
      std::vector<int> need(ng, 1);
      std::vector<std::vector<int>> mem(ng);
      for (int q : order) {
        int t = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        load[t] += steps(q);
        work[t] += steps(q) * ent(q);
        need[t] = std::max(need[t], gmin(q));
        mem[t].push_back(q);
      }
      double wsum = 0;
      int nsum = 0;
      for (int t = 0; t < ng; ++t) wsum += work[t], nsum += need[t];
      if (nsum > nsm && ng > 1) continue;  // some group could not keep its rows in shared memory
      // proportional allocation with minimums (one group = the whole grid,
      // global-row layout if its rows do not fit shared memory)
      std::vector<int> G(ng);
      int left = nsm;
      for (int t = 0; t < ng && ng > 1; ++t) {
        G[t] = std::max(need[t], (int)std::floor(nsm * work[t] / std::max(wsum, 1.0)));
        left -= G[t];
      }
      while (left < 0) {  // trim the largest groups above their minimum
        int t = (int)(std::max_element(G.begin(), G.end()) - G.begin());
        if (G[t] <= need[t]) break;
        G[t]--;
        left++;
      }
      if (left < 0) continue;
      if (ng == 1) G[0] = 0;
      for (int t = 0; left > 0; t = (t + 1) % ng, --left) G[t]++;
      double cost = 0;
      for (int t = 0; t < ng; ++t) {
        double c = 0;
        for (int q : mem[t]) c += steps(q) * (LAT + PER * ent(q) / G[t]);
        cost = std::max(cost, c);
      }
      if (cost < best_cost) {
        best_cost = cost;
        members = mem;
        sizes = G;
      }
    }
    int ng = (int)members.size();
    int nmax = 1;
    for (int q : grd) nmax = std::max(nmax, jobs[q].n);
    for (int t = 0, f1 = 0; t < ng; ++t) {
      int f0 = f1, G = sizes[t];
      f1 = f0 + G;
      bool fits = true;
      for (int q : members[t]) fits &= plu_dist_bytes(jobs[q].m, jobs[q].n, G, true) <= dyn_max;
      bool ok = true;
      for (int q : members[t]) ok &= plu_dist_bytes(jobs[q].m, jobs[q].n, G, false) <= dyn_max;
      if (!ok) throw runtime_error("complete-pivot core too large for its cooperative group");
      GridLaunch &L = gl[fits ? 0 : 1];
      if (L.cptr.empty()) L.cptr.push_back(0);
      L.first.push_back(f0);  // group = CTAs [f0, f1) of the launch
      L.first.push_back(f1);
      for (int q : members[t]) {
        L.ids.push_back(q);
        L.smem = std::max(L.smem, plu_dist_bytes(jobs[q].m, jobs[q].n, G, fits));
      }
      L.cptr.push_back((int)L.ids.size());
    }
    gs.nmax = nmax;
    gs.best = (MaxLoc *)ctx->scratch.alloc(std::max(sizeof(MaxLoc), sizeof(PluCand)) * 2 * nsm);
    gs.cand = ctx->scratch.d((size_t)2 * nsm * nmax);
    gs.bar = (unsigned *)ctx->scratch.alloc(sizeof(unsigned) * 2 * ng);
    CK(cudaMemsetAsync(gs.bar, 0, sizeof(unsigned) * 2 * ng, ctx->s));
  }
  int *gl_first[2], *gl_cptr[2], *gl_ids[2];
  for (int v = 0; v < 2; ++v) {
    gl_first[v] = gl[v].ids.empty() ? nullptr : sk.push(gl[v].first);
    gl_cptr[v] = gl[v].ids.empty() ? nullptr : sk.push(gl[v].cptr);
    gl_ids[v] = gl[v].ids.empty() ? nullptr : sk.push(gl[v].ids);
  }
  bool side = !cl8.empty() || !cl16.empty() || !grd.empty();
  if (side) {
    CK(cudaEventRecord(ctx->ev_fork, ctx->s));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    if (!cl8.empty()) CK(cudaStreamWaitEvent(ctx->side2, ctx->ev_fork, 0));
  }
  auto cluster_group = [&](const std::vector<int> &g, int *dids, int cs, cudaStream_t st) {
    if (g.empty()) return;
    size_t sm = 0;
    for (int q : g) sm = std::max(sm, plu_cl3_bytes(jobs[q].m, jobs[q].n, cs));
    launch_cluster(fns[2], (int)g.size(), cs, sm, st, dj, dids, eps);
    ctx->launches++;
  };
  // 8-CTA clusters on their own stream: they run beside the 16-CTA clusters
  // (and ahead of the cooperative launch, which waits for free SMs)
  auto coop = [&](cudaStream_t st) {
  for (int v = 0; v < 2; ++v) {
    GridLaunch &L = gl[v];
    if (L.ids.empty()) continue;
    // one group spanning the GPU: the compacted-list kernel measures faster
    // (4.4 vs 8.4 us/step at 1728 x 971); split GPUs: the one-barrier kernel
    const int ngroups_l = (int)L.cptr.size() - 1;
    const void *fn = v == 1 ? fns[4] : (ngroups_l == 1 ? fns[5] : fns[3]);
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 512, L.smem));
    if (per_sm < 1) throw runtime_error("cooperative pivot-LU kernel does not fit on an SM");
    int ngr = (int)L.cptr.size() - 1;
    double e = eps;
    GridScratch g2 = gs;
    void *args[7] = {(void *)&dj, (void *)&gl_ids[v], (void *)&gl_first[v], (void *)&gl_cptr[v], (void *)&ngr,
                     (void *)&e, (void *)&g2};
    CK(cudaLaunchCooperativeKernel(fn, dim3(nsm), dim3(512), args, L.smem, st));
    ctx->launches++;
  }
  };
  // MFH_PLU_EVENTS=1: per-class completion times of this window (diagnostics;
  // adds a synchronization)
  static const bool pev = getenv("MFH_PLU_EVENTS") != nullptr;
  cudaEvent_t pe[8] = {};
  if (pev) {
    for (auto &e : pe) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(pe[0], ctx->s));
  }
  const bool coop_own = coop_first && !grd.empty() && (!cl8.empty() || !cl16.empty());
  if (coop_own) {  // the critical-path cores claim their SMs first, clusters fill the rest
    CK(cudaStreamWaitEvent(ctx->side3, ctx->ev_fork, 0));
    coop(ctx->side3);
    CK(cudaEventRecord(ctx->ev_join3, ctx->side3));
  }
  cluster_group(cl8, ids_cl8, 8, ctx->side2);
  if (pev && !cl8.empty()) CK(cudaEventRecord(pe[1], ctx->side2));
  if (!cl8.empty()) CK(cudaEventRecord(ctx->ev_join2, ctx->side2));
  cluster_group(cl16, ids_cl16, CS, ctx->side);
  if (pev && side) CK(cudaEventRecord(pe[2], ctx->side));
  if (!coop_own) coop(ctx->side);
  if (pev && side) CK(cudaEventRecord(pe[3], ctx->side));
  if (side) CK(cudaEventRecord(ctx->ev_join, ctx->side));
  // the one-CTA cores on their own stream, beside the dense fronts' work on the
  // main stream (both are independent of each other within the height)
  int *dids_small[3] = {nullptr, nullptr, nullptr};
  for (int b = 0; b < 3; ++b)
    if (!small[b].empty()) dids_small[b] = sk.push(small[b]);
  const bool any_small = !small[0].empty() || !small[1].empty() || !small[2].empty();
  if (any_small) {
    CK(cudaEventRecord(ctx->ev_fork2, ctx->s));  // after the pushes above
    CK(cudaStreamWaitEvent(ctx->side4, ctx->ev_fork2, 0));
  }
  for (int b = 0; b < 3; ++b) {
    if (small[b].empty()) continue;
    size_t sm = 0;
    for (int q : small[b]) sm = std::max(sm, cta_bytes(jobs[q].m, jobs[q].n));
    const int nb = (int)small[b].size();
    if (b == 2)
      launch_pdl(k_plu_cta2<true, 1024>, dim3(nb), dim3(1024), sm, ctx->side4, dj, (const int *)dids_small[b], eps);
    else
      launch_pdl(k_plu_cta2<true, 512>, dim3(nb), dim3(b == 0 ? 256 : 512), sm, ctx->side4, dj,
                 (const int *)dids_small[b], eps);
    ctx->launches++;
  }
  if (any_small) CK(cudaEventRecord(ctx->ev_join4, ctx->side4));
  if (main_work) main_work();
  if (pev) CK(cudaEventRecord(pe[4], ctx->s));
  if (any_small) CK(cudaStreamWaitEvent(ctx->s, ctx->ev_join4, 0));
  if (pev) CK(cudaEventRecord(pe[5], ctx->s));
  if (side) CK(cudaStreamWaitEvent(ctx->s, ctx->ev_join, 0));
  if (!cl8.empty()) CK(cudaStreamWaitEvent(ctx->s, ctx->ev_join2, 0));
  if (coop_own) CK(cudaStreamWaitEvent(ctx->s, ctx->ev_join3, 0));
  if (pev) {
    CK(cudaEventRecord(pe[6], ctx->s));
    CK(cudaEventSynchronize(pe[6]));
    auto el = [&](int q, bool have) {
      float ms = -1.f;
      if (have) CK(cudaEventElapsedTime(&ms, pe[0], pe[q]));
      return ms;
    };
    auto steps = [&](const std::vector<int> &v) {
      int mx = 0;
      for (int q : v) mx = std::max(mx, std::min(std::min(jobs[q].m, jobs[q].n), jobs[q].kmax));
      return mx;
    };
    int nsmall = 0, ssmall = 0;
    for (auto &v : small) nsmall += (int)v.size(), ssmall = std::max(ssmall, steps(v));
    fprintf(stderr, "[mfh plu window] cl8 %zu cores (<=%d steps) done %.3f | cl16 %zu (<=%d) done %.3f | grid %zu (<=%d) done %.3f | main dense %.3f, cta %d (<=%d) done %.3f | all %.3f ms\n",
            cl8.size(), steps(cl8), el(1, !cl8.empty()), cl16.size(), steps(cl16), el(2, side), grd.size(), steps(grd),
            el(3, side), el(4, true), nsmall, ssmall, el(5, true), el(6, true));
    for (auto &e : pe) cudaEventDestroy(e);
  }
}

// ---------------------------------------------------------------------------
// HODLR factor tree (device pointers kept on the host side)
// ---------------------------------------------------------------------------
struct FacView {  // DenseBlock.as_factors / LowRankFactor.as_factors (hodlr.py:59-63)
  const double *col = nullptr;
  int ldc = 0;
  const double *row = nullptr;
  int ldr = 0;
  int rank = 0;
};

struct BlockH {
  int fi = -1;
  int kind = 2;  // 0: pivot-block HODLR (dies with the height), 1: update HODLR (dies once the
                 // parent has sampled it), 2: pf / fp coupling (retained for the apply)
  int r0 = 0, m = 0, c0 = 0, n = 0;
  std::vector<int> I, J;
  bool fullI = false, fullJ = false;
  int kmax = 0;
  // temporaries
  double *R = nullptr, *C = nullptr, *core = nullptr;
  int ldR = 0, ldC = 0;
  int *d_I = nullptr, *d_J = nullptr, *d_inter = nullptr;
  int *pint = nullptr;     // PLU int scratch
  double *pdbl = nullptr;  // PLU double scratch
  int *res = nullptr;      // device [rank,status,errk]
  double *resd = nullptr;  // device [ratio, errpiv, errprev]
  // results
  int rank = 0, status = 0, errk = 0;
  bool rows_phys = false;  // pivot-LU kernel left the core's rows physically permuted
  double ratio = 0.0, errpiv = 0.0, errprev = 0.0;
  bool dense = false;
  std::vector<int> rowperm, colperm;  // first `rank` pivots (parity log)
  double *col = nullptr, *row = nullptr, *val = nullptr;
  int64_t stored() const { return dense ? (int64_t)m * n : (int64_t)(m + n) * rank; }
  int erank() const { return dense ? std::min(m, n) : rank; }
  HBlk dev() const {
    HBlk b{};
    if (dense) {
      b.kind = 1;
      b.a = val;
      b.lda = n;
    } else {
      b.kind = 0;
      b.a = col;
      b.lda = rank;
      b.b = row;
      b.ldb = n;
      b.rank = rank;
    }
    return b;
  }
};

struct HTree {
  int fi = -1, base = 0, n = 0;
  int nslots = 0;
  std::vector<int> lo, hi, depth;
  std::vector<char> leaf;  // 1 leaf, 0 internal, -1 absent
  std::vector<int> up, lw;  // block ids
  std::vector<double *> lval;  // leaf values (LU in place after factorization)
  std::vector<int *> lpiv;
  std::vector<int> lflag;  // flag slot
  // factorization data (internal nodes)
  std::vector<double *> xt, xb, core;
  std::vector<int *> cpiv;
  std::vector<int> r1, r2;
  std::vector<FacView> f1, f2;
  std::vector<double *> linv, cinv;  // explicit inverses of leaves / Woodbury cores (apply)
  HNode *d_nodes = nullptr;
  int maxdepth = 0;
};

// ---------------------------------------------------------------------------
// factorization object
// ---------------------------------------------------------------------------
// non-owning view of a front's id list (the per-tree flat cache)
struct IdsView {
  const int64_t *p = nullptr;
  size_t n = 0;
  const int64_t &operator[](size_t i) const { return p[i]; }
  const int64_t *data() const { return p; }
  size_t size() const { return n; }
  const int64_t *begin() const { return p; }
  const int64_t *end() const { return p + n; }
};

struct FrontH {
  int64_t node = -1;
  int npv = 0, nf = 0, nh = 0;
  int64_t piv_lo = 0;
  IdsView ids;
  int height = 0;
  bool structured = false;
  std::vector<int> kids;  // fronts with a non-empty update, in node.children order
  std::vector<int> allkids;  // every child front (post-order index)
  int64_t freed = 0;
  long long *d_ids = nullptr;
  // dense path
  double *F = nullptr;
  int *piv = nullptr;
  // apply operators (explicit inverse form, computed once at factor time)
  double *Pinv = nullptr, *Gfp = nullptr, *Gpf = nullptr;
  // dense: F_pp kept for node_factors: apply_pf = F_pp (Gpf v), apply_fp = Gfp (F_pp v)
  // (n_p^2 reals instead of keeping F_pf and F_fp, 2 n_p nf)
  double *Fpp = nullptr;
  // structured: Hinv = (HODLR pivot block)^{-1} (retained when pform == 0),
  // Xp = Hinv col_pf, RH = row_fp Hinv (low-rank couplings only)
  double *Hinv = nullptr, *Xp = nullptr, *RH = nullptr;
  // retained pivot-block inverse: 0 explicit Hinv, 1 HODLR inverse form
  //   H^{-1} b = L^{-1} b - sum_v X_v w_v,  w_v = Tm_v b[v's range]
  int pform = 0;
  struct TmNode {
    int slot = 0, lo = 0, nv = 0, r1 = 0, r2 = 0;
    double *Tm = nullptr;                  // (r1 + r2) x nv, retained
    const double *xt = nullptr, *xb = nullptr;  // x_top / x_bot (factor-time scratch)
    int64_t woff = 0;                      // offset of w_v in the front's w segment
  };
  struct TmLeaf {
    int slot = 0, lo = 0, sz = 0, K = 0;
    double *Linv = nullptr, *XL = nullptr;  // sz x sz, sz x K
    long long *idx = nullptr;               // K entries into the w segment
  };
  std::vector<TmNode> tnode;
  std::vector<TmLeaf> tleaf;
  int64_t wlen = 0;
  // structured path
  int pp = -1, ff = -1, pf = -1, fp = -1;  // tree / block ids
  int tree_base = -1, block_base = -1;      // pre-assigned plan slots
  // update for the parent
  int upd = -1;  // -1 none, 0 dense, 1 hodlr
  bool densified = false;  // update materialized dense for the parent (densify_update)
  const double *upd_dense = nullptr;
  int upd_ld = 0;
  const double *W = nullptr, *Vt = nullptr;
  int rw = 0, ldw = 0, ldv = 0;
  const HNode *rx_nodes = nullptr;  // sharded: update HODLR received from the child's owner
  // accounting
  int64_t front_reals = 0, factor_reals = 0, upd_reals = 0;
  int64_t hint = 0;
  int flag_slot = -1;
};

struct ApplyPlan;

}  // namespace mfh

struct mfh_factor;
namespace mfh {
static void build_apply(mfh_factor *F);
}

struct mfh_ctx {
  mfh::Ctx c;
};

struct mfh_factor {
  mfh::Ctx *ctx = nullptr;
  mfh::Arena arena;
  int64_t n = 0;
  int mode = 0;
  mfh_params params{};
  std::vector<int64_t> perm;
  long long *d_perm = nullptr;
  uint64_t et_uid = 0;                   // elimination tree the factor was built on
  std::vector<mfh::FrontH> fronts;       // by post-order index
  std::vector<int64_t> post;             // node ids in post order
  std::vector<mfh::BlockH> blocks;
  std::vector<mfh::HTree> trees;
  std::vector<std::vector<int>> front_blocks;  // per front, block ids in visiting order
  double *ident = nullptr;
  int ident_ld = 0;
  // stats
  mfh_stats_t stats{};
  std::vector<mfh_record_t> records;
  mfh_timing_t timing{};
  // apply
  std::unique_ptr<mfh::ApplyPlan> apply;
  std::map<int, std::unique_ptr<mfh::ApplyPlan>> apply_nv;  // several right-hand sides per replay (built on demand)
  // subtree-sharded factor: owner rank per post index, mine = owner == rank
  bool sharded = false;
  std::vector<int> owner;
  std::vector<int8_t> mine;
  int rank = 0, world = 1;
  mfh_exchange_fn exchange = nullptr;
  mfh_p2p_fn p2p = nullptr;
  void *xuser = nullptr;
  int64_t xchg_bytes = 0;  // bytes this rank sent in update exchanges (diagnostics)
  void exchange_or_throw(double *d, int64_t count) {
    if (count <= 0) return;
    if (exchange(xuser, d, count) != 0) throw mfh::runtime_error("shard exchange callback failed");
  }
};

namespace mfh {

// ---------------------------------------------------------------------------
// the factorization driver
// ---------------------------------------------------------------------------
// read-only view of the caller's CSR (rows sorted, no duplicates)
struct CsrView {
  int64_t n = 0;
  const int64_t *ptr = nullptr, *idx = nullptr;
  const double *val = nullptr;
};

// fn(begin, end, t) over [0, n) on up to 8 host threads (half the cores), at least
// min_per_thread items each; fn must not throw
template <class Fn>
static int par_chunks(int64_t n, int64_t min_per_thread, Fn fn) {
  const unsigned hc = std::thread::hardware_concurrency();
  const int k = (int)std::min<int64_t>(std::min(8u, std::max(1u, hc / 2)), std::max<int64_t>(1, n / min_per_thread));
  if (k <= 1) {
    fn((int64_t)0, n, 0);
    return 1;
  }
  const int64_t step = (n + k - 1) / k;
  std::vector<std::thread> th;
  for (int t = 1; t < k; ++t) th.emplace_back([=, &fn] { fn(t * step, std::min(n, (t + 1) * step), t); });
  fn((int64_t)0, std::min(n, step), 0);
  for (auto &x : th) x.join();
  return k;
}

struct Factorizer {
  mfh_factor *F;
  Ctx *ctx;
  const mfh_etree *et;
  mfh_params P;
  const mfh_shard_t *shard = nullptr;
  ReleaseArena upd;            // dense front buffers (dead once the parent has sampled them)
  std::vector<int> pidx_;      // post index of every node
  std::vector<char> alias_;    // dense merge node whose update is its only child's, bit for bit
  int release_height(const FrontH &f) const {
    int64_t par = et->parent[f.node];
    while (par >= 0 && alias_[pidx_[par]]) par = et->parent[par];
    return par < 0 ? (1 << 30) : F->fronts[pidx_[par]].height;
  }
  bool accel;
  int64_t n;
  // permuted matrix on device
  std::vector<int64_t> ap_ptr;
  std::vector<int> ap_col;
  long long *d_ap_ptr = nullptr;
  int *d_ap_col = nullptr;
  double *d_ap_val = nullptr;
  const Graph *gp = nullptr;  // BDLR graph over permuted ids (cached on the etree)
  // selection scratch, one per selection thread
  struct SelScratch {
    std::vector<int64_t> mark;
    int64_t stamp = 0;
    std::vector<int> distv;
  };
  std::vector<SelScratch> sel_scratch;
  // error flags
  int *d_flags = nullptr;
  int nflags = 0;
  std::vector<std::string> flag_msg;
  std::vector<int64_t> flag_order;  // post index for ordering

  Sink sk() { return Sink{ctx}; }

  // ---- selection (bdlr.py:89-136), positions are front-local ----
  void select(SelScratch &sc, const FrontH &f, int r0, int m, int c0, int nn, std::vector<int> &I,
              std::vector<int> &J) {
    const Graph &graph = *gp;
    std::vector<int64_t> &mark = sc.mark;
    std::vector<int> &distv = sc.distv;
    int64_t &stamp = sc.stamp;
    I.clear();
    J.clear();
    const int64_t *ids = f.ids.data();
    if ((int64_t)mark.size() < graph.n) {
      mark.assign(graph.n, 0);
      distv.assign(graph.n, 0);
    }
    auto near_set = [&](int s0, int sn, int t0, int tn, std::vector<int> &out) {
      // out = positions t in [t0,t0+tn) whose vertex is within distance d of {ids[s0..s0+sn)}
      ++stamp;
      if (P.d == 1) {
        for (int s = s0; s < s0 + sn; ++s) mark[ids[s]] = stamp;
        for (int t = t0; t < t0 + tn; ++t) {
          int64_t v = ids[t];
          for (int64_t q = graph.ptr[v]; q < graph.ptr[v + 1]; ++q)
            if (mark[graph.idx[q]] == stamp) {
              out.push_back(t);
              break;
            }
        }
        return;
      }
      std::vector<int64_t> queue;
      for (int s = s0; s < s0 + sn; ++s) {
        mark[ids[s]] = stamp;
        distv[ids[s]] = 0;
        queue.push_back(ids[s]);
      }
      size_t head = 0;
      while (head < queue.size()) {
        int64_t v = queue[head++];
        if (distv[v] >= P.d) continue;
        for (int64_t q = graph.ptr[v]; q < graph.ptr[v + 1]; ++q) {
          int64_t w = graph.idx[q];
          if (mark[w] != stamp) {
            mark[w] = stamp;
            distv[w] = distv[v] + 1;
            queue.push_back(w);
          }
        }
      }
      for (int t = t0; t < t0 + tn; ++t) {
        int64_t v = ids[t];
        if (mark[v] == stamp && distv[v] <= P.d) out.push_back(t);
      }
    };
    near_set(c0, nn, r0, m, I);
    near_set(r0, m, c0, nn, J);
    if (I.empty())
      for (int t = r0; t < r0 + m; ++t) I.push_back(t);
    if (J.empty())
      for (int t = c0; t < c0 + nn; ++t) J.push_back(t);
  }

  int flag_cap = 0;
  // host time from the rank read-back to the skeleton launches (the GPU idles in it)
  std::chrono::steady_clock::time_point t_decide0;
  double last_decide_us = 0.0;
  int new_flag(const std::string &msg, int64_t order) {
    if (nflags >= flag_cap) throw runtime_error("internal: error-flag capacity exceeded");
    flag_msg.push_back(msg);
    flag_order.push_back(order);
    return nflags++;
  }

  // ---- tree construction (hodlr.py:203-246 recursion order) ----
  int make_tree(int fi, int base, int nloc, std::vector<int> &blist, int tid, int kind) {
    HTree t;
    t.fi = fi;
    t.base = base;
    t.n = nloc;
    // slots
    int cap = 1;
    {
      // depth bound
      int d = 0;
      int64_t s = nloc;
      while (s > P.n_leaf) {
        s = (s + 1) / 2;
        ++d;
      }
      cap = (1 << (d + 2));
    }
    t.nslots = cap;
    t.lo.assign(cap, -1);
    t.hi.assign(cap, -1);
    t.depth.assign(cap, 0);
    t.leaf.assign(cap, -1);
    t.up.assign(cap, -1);
    t.lw.assign(cap, -1);
    t.lval.assign(cap, nullptr);
    t.lpiv.assign(cap, nullptr);
    t.lflag.assign(cap, -1);
    t.xt.assign(cap, nullptr);
    t.xb.assign(cap, nullptr);
    t.core.assign(cap, nullptr);
    t.cpiv.assign(cap, nullptr);
    t.r1.assign(cap, 0);
    t.r2.assign(cap, 0);
    t.f1.assign(cap, FacView{});
    t.f2.assign(cap, FacView{});
    t.linv.assign(cap, nullptr);
    t.cinv.assign(cap, nullptr);
    F->trees[tid] = std::move(t);
    // recursion with explicit stack: (slot, lo, hi, depth, stage)
    struct Fr {
      int v, lo, hi, d, stage;
    };
    std::vector<Fr> st{{0, 0, nloc, 0, 0}};
    while (!st.empty()) {
      Fr &fr = st.back();
      HTree &T = F->trees[tid];
      if (fr.stage == 0) {
        T.lo[fr.v] = fr.lo;
        T.hi[fr.v] = fr.hi;
        T.depth[fr.v] = fr.d;
        T.maxdepth = std::max(T.maxdepth, fr.d);
        if (fr.hi - fr.lo <= P.n_leaf) {
          T.leaf[fr.v] = 1;
          st.pop_back();
          continue;
        }
        T.leaf[fr.v] = 0;
        fr.stage = 1;
        int mid = (fr.lo + fr.hi) >> 1;
        Fr c{2 * fr.v + 1, fr.lo, mid, fr.d + 1, 0};
        st.push_back(c);
      } else if (fr.stage == 1) {
        fr.stage = 2;
        int mid = (fr.lo + fr.hi) >> 1;
        Fr c{2 * fr.v + 2, mid, fr.hi, fr.d + 1, 0};
        st.push_back(c);
      } else {
        int lo = fr.lo, hi = fr.hi, mid = (lo + hi) >> 1;
        int v = fr.v;
        st.pop_back();
        int bu = new_block(fi, base + lo, mid - lo, base + mid, hi - mid, kind);
        int bl = new_block(fi, base + mid, hi - mid, base + lo, mid - lo, kind);
        F->trees[tid].up[v] = bu;
        F->trees[tid].lw[v] = bl;
        blist.push_back(bu);
        blist.push_back(bl);
      }
    }
    return tid;
  }

  int block_cursor = 0;  // planner thread: next pre-assigned block slot
  int new_block(int fi, int r0, int m, int c0, int nn, int kind) {
    BlockH &b = F->blocks[block_cursor];
    b.fi = fi;
    b.kind = kind;
    b.r0 = r0;
    b.m = m;
    b.c0 = c0;
    b.n = nn;
    return block_cursor++;
  }

  // ---- symbolic plan of one structured front (trees, blocks, BDLR selections);
  // runs on the planner thread, writing only into this front's pre-assigned slots
  void plan_front(int fi) {
    FrontH &f = F->fronts[fi];
    block_cursor = f.block_base;
    std::vector<int> blist;
    if (f.npv) f.pp = make_tree(fi, 0, f.npv, blist, f.tree_base, 0);
    if (f.npv && f.nf) {
      f.pf = new_block(fi, 0, f.npv, f.npv, f.nf, 2);
      f.fp = new_block(fi, f.npv, f.nf, 0, f.npv, 2);
      blist.push_back(f.pf);
      blist.push_back(f.fp);
    }
    if (f.nf) f.ff = make_tree(fi, f.npv, f.nf, blist, f.tree_base + 1, 1);
    F->front_blocks[fi] = blist;
    // The blocks' selections are independent (each writes its own I / J): spread over
    // MFH_PLAN_THREADS host threads (default: half the cores, at most 16), each with its own
    // marker arrays. At C3 one thread could not stay ahead of the GPU: the structured heights
    // waited 67-115 ms each for their selections (MFH_HEIGHT_TRACE: gap minus materialization).
    if (sel_scratch.empty()) sel_scratch.resize(1);
    const int nthreads = (int)sel_scratch.size();
    std::atomic<size_t> next{0};
    std::exception_ptr err;
    std::mutex err_mu;
    auto work = [&](int t) {
      try {
        for (size_t q; (q = next.fetch_add(1, std::memory_order_relaxed)) < blist.size();) {
          BlockH &b = F->blocks[blist[q]];
          select(sel_scratch[t], f, b.r0, b.m, b.c0, b.n, b.I, b.J);
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (!err) err = std::current_exception();
      }
    };
    // threads by the front's selection work (graph edges visited ~ vertices x degree^d): a thread
    // is worth spawning for ~2M edge visits; the small fronts of C1 / C2 / C4 stay on one thread
    double edges = 0.0;
    {
      const Graph &graph = *gp;
      const double deg = graph.n ? (double)graph.ptr[graph.n] / (double)graph.n : 1.0;
      double per = 1.0;
      for (int q = 0; q < std::max(1, (int)P.d); ++q) per *= std::max(1.0, deg);
      for (int bi : blist) edges += ((double)F->blocks[bi].m + F->blocks[bi].n) * per;
    }
    const double per_thread = getenv("MFH_PLAN_MIN_EDGES") ? atof(getenv("MFH_PLAN_MIN_EDGES")) : 2e6;  // test knob
    const int use = (int)std::max<double>(
        1.0, std::min<double>(std::min<double>(nthreads, blist.size()), edges / std::max(1.0, per_thread)));
    std::vector<std::thread> pool;
    for (int t = 1; t < use; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto &th : pool) th.join();
    if (err) std::rethrow_exception(err);
  }

  static int count_internal(int64_t n, int64_t nl) {
    if (n <= nl) return 0;
    int64_t h = n / 2;
    return 1 + count_internal(h, nl) + count_internal(n - h, nl);
  }

  // planner thread over the structured fronts, in processing order
  std::thread planner;
  std::atomic<int> planned{0};
  std::vector<int> plan_order, plan_pos;
  std::exception_ptr plan_error;
  void start_planner() {
    {
      const char *e = getenv("MFH_PLAN_THREADS");
      const unsigned hc = std::thread::hardware_concurrency();
      int k = e ? atoi(e) : (int)std::min(16u, std::max(1u, hc / 2));
      sel_scratch.resize((size_t)std::max(1, k));
    }
    planner = std::thread([this]() {
      try {
        for (int fi : plan_order) {
          plan_front(fi);
          planned.fetch_add(1, std::memory_order_release);
        }
      } catch (...) {
        plan_error = std::current_exception();
        planned.store(1 << 30, std::memory_order_release);
      }
    });
  }
  void wait_planned(int fi) {
    int need = plan_pos[fi] + 1;
    while (planned.load(std::memory_order_acquire) < need) std::this_thread::yield();
    if (plan_error) std::rethrow_exception(plan_error);
  }
  ~Factorizer() {
    if (planner.joinable()) planner.join();
    upd.release_all();  // (error paths synchronize the stream before the pool is reused)
  }

  void check_flags(int64_t upto_flags, const int *hflags = nullptr) {
    if (nflags == 0) return;
    std::vector<int> h(nflags);
    if (hflags)
      std::memcpy(h.data(), hflags, sizeof(int) * nflags);
    else
      CK(cudaMemcpy(h.data(), d_flags, sizeof(int) * nflags, cudaMemcpyDeviceToHost));
    int best = -1;
    for (int q = 0; q < nflags; ++q)
      if (h[q] && (best < 0 || flag_order[q] < flag_order[best])) best = q;
    if (best >= 0) throw value_error(flag_msg[best]);
    (void)upto_flags;
  }

  // ---- extend-add maps (symbolic, once per tree; device copy once per context) ----
  int *d_maps = nullptr;
  void ensure_maps() {
    mfh_mapcache &M = et->mapcache;
    if (!M.valid) {
      M.maps.clear();
      M.off.assign(F->fronts.size(), -1);
      for (size_t fi = 0; fi < F->fronts.size(); ++fi) {
        FrontH &f = F->fronts[fi];
        for (int ci : f.kids) {
          FrontH &c = F->fronts[ci];
          // parent position -> child update position (multifrontal.py:270-280, 321-327)
          M.off[ci] = (int64_t)M.maps.size();
          M.maps.resize(M.maps.size() + f.nh, -1);
          int *to = M.maps.data() + M.off[ci];
          const int64_t *cid = c.ids.data() + c.npv;
          int p = 0;
          for (int q = 0; q < c.nf; ++q) {
            int64_t g = cid[q];
            while (p < f.nh && f.ids[p] < g) ++p;
            if (p >= f.nh || f.ids[p] != g)
              throw value_error("update index " + std::to_string(g) + " not present in parent front (node " +
                                std::to_string(f.node) + ")");
            to[p] = q;
          }
        }
      }
      M.valid = true;
    }
    for (auto &m : ctx->map_dev)
      if (m.first == et->uid) {
        d_maps = m.second;
        return;
      }
    if (ctx->map_dev.size() >= Ctx::SYM_CACHE_MAX) {  // least recently added tree
      cudaFree(ctx->map_dev.front().second);
      ctx->map_dev.erase(ctx->map_dev.begin());
    }
    size_t bytes = sizeof(int) * std::max<size_t>(1, M.maps.size());
    CK(cudaMalloc(&d_maps, bytes));
    upload(ctx->s, d_maps, M.maps.data(), sizeof(int) * M.maps.size());
    ctx->map_dev.push_back({et->uid, d_maps});
  }

  // ---- child descriptors (maps from the per-tree cache) for a set of fronts ----
  // A child update of nf >= 256 (the update HODLR minus W V^T, multifrontal.py:340-347)
  // is materialized once as a dense nf x nf block when its parent is
  // processed: leaf copies and one GEMM per low-rank block (the reference's
  // to_dense), then -W V^T as one GEMM. The parent's extend-add requests then
  // gather from it instead of descending the HODLR tree and recomputing a
  // rank-r product per sampled entry (C5: the root's dense fallbacks read
  // ~300 GB that way). Below nf 4096 the products run on k_gemm (k-ascending
  // DMMA chains, epilogue fma(beta, C, alpha acc)), the same arithmetic as the
  // sampler's per-entry chains, so the sampled values are bitwise unchanged
  // (tests/test_gpu_densify.py). nf >= MFH_DENSIFY_MIN (0 = never).
  struct DensifyJobs {
    std::vector<CopyJob> cp;
    std::vector<GemmJob> gm[2], wv[2];  // [exact]: block products, then -W V^T
  };
  const double *densify_update(DensifyJobs &dj, const FrontH &c) {
    const int nf = c.nf;
    double *D = upd.d((size_t)nf * nf, release_height(c));
    HTree &T = F->trees[c.ff];
    // below 4096 every product stays on k_gemm (bitwise the sampler's values);
    // larger ones may take the cuBLAS route (C5: 0.1 s faster per step)
    const int exact = nf < 4096 ? 1 : 0;
    for (int v = 0; v < T.nslots; ++v) {
      const int lo = T.lo[v], hi = T.hi[v];
      if (T.leaf[v] == 1) {
        const int sz = hi - lo;
        dj.cp.push_back(CopyJob{T.lval[v], D + (int64_t)lo * nf + lo, sz, sz, sz, nf, nullptr, nullptr});
      } else if (T.leaf[v] == 0) {
        const int mid = (lo + hi) >> 1;
        for (int side = 0; side < 2; ++side) {
          const BlockH &b = F->blocks[side == 0 ? T.up[v] : T.lw[v]];
          double *dst = D + (side == 0 ? (int64_t)lo * nf + mid : (int64_t)mid * nf + lo);
          if (b.dense)
            dj.cp.push_back(CopyJob{b.val, dst, b.m, b.n, b.n, nf, nullptr, nullptr});
          else  // rank 0 writes zeros (k = 0)
            dj.gm[exact].push_back(
                GemmJob{b.col, b.row, dst, b.m, b.n, b.rank, std::max(1, b.rank), b.n, nf, 1.0, 0.0});
        }
      }
    }
    // D = H - W V^T: fma(1, H, -acc), the sampler's sub - acc
    if (c.rw) dj.wv[exact].push_back(GemmJob{c.W, c.Vt, D, nf, nf, c.rw, c.ldw, c.ldv, nf, -1.0, 1.0});
    return D;
  }
  // one launch per job kind for every child materialized at this height
  void run_densify(Sink &s, DensifyJobs &dj) {
    if (dj.cp.empty() && dj.gm[0].empty() && dj.gm[1].empty()) return;
    const double fl0 = ctx->flops_exec;
    s.begin_batch();
    run_copy(s, dj.cp);
    for (int x = 0; x < 2; ++x) run_gemm(s, dj.gm[x], x == 1);
    for (int x = 0; x < 2; ++x) run_gemm(s, dj.wv[x], x == 1);
    s.flush();
    F->timing.exec_flops_materialize += ctx->flops_exec - fl0;
  }

  void build_fronts_dev(Sink &s, const std::vector<int> &fis, std::vector<DFront> &dfr,
                        std::vector<DChild> &dch, std::vector<int> &slot_of) {
    static const int densify_min = getenv("MFH_DENSIFY_MIN") ? atoi(getenv("MFH_DENSIFY_MIN")) : 256;
    DensifyJobs dj;
    slot_of.assign(F->fronts.size(), -1);
    slot_rw.clear();
    for (int fi : fis) {
      FrontH &f = F->fronts[fi];
      DFront d{};
      d.ids = f.d_ids;
      d.nh = f.nh;
      d.npv = f.npv;
      d.child_begin = (int)dch.size();
      for (int ci : f.kids) {
        FrontH &c = F->fronts[ci];
        DChild ch{};
        ch.to_child = d_maps + et->mapcache.off[ci];
        const int cn = c.nf;
        ch.n = cn;
        if (c.upd == 0) {
          ch.kind = 0;
          ch.dense = c.upd_dense;
          ch.ldd = c.upd_ld;
        } else if (densify_min > 0 && cn >= densify_min && !c.rx_nodes && c.ff >= 0) {
          ch.kind = 0;
          ch.dense = densify_update(dj, c);
          ch.ldd = cn;
          c.densified = true;
        } else {
          ch.kind = 1;
          ch.hn = c.rx_nodes ? c.rx_nodes : F->trees[c.ff].d_nodes;
          ch.W = c.W;
          ch.Vt = c.Vt;
          ch.rw = c.rw;
          ch.ldw = c.ldw;
          ch.ldv = c.ldv;
        }
        dch.push_back(ch);
      }
      d.child_end = (int)dch.size();
      slot_of[fi] = (int)dfr.size();
      int mrw = 0;
      for (int q = d.child_begin; q < d.child_end; ++q)
        if (dch[q].kind == 1) mrw = std::max(mrw, dch[q].rw);
      slot_rw.push_back(mrw);
      dfr.push_back(d);
    }
    run_densify(s, dj);
  }

  // largest child update rank per DFront slot of the current descriptor set
  // (filled where the descriptors are built): routes requests to the
  // register-blocked sampler when a child carries a real W Vt
  std::vector<int> slot_rw;
  static constexpr int RB_MIN_RANK = 16;

  // hfr / hch given: the front descriptors are pushed here, in the same H2D
  // transfer as the requests and tiles, and dF / dC are set
  void run_sample(Sink &s, const std::vector<SReq> &reqs, DFront *&dF, DChild *&dC,
                  const std::vector<DFront> *hfr = nullptr, const std::vector<DChild> *hch = nullptr) {
    OpClock oc_("sample");
    auto push_fronts = [&](std::vector<std::pair<const void *, size_t>> extra) {
      std::vector<std::pair<const void *, size_t>> parts{{hfr->data(), hfr->size() * sizeof(DFront)},
                                                        {hch->data(), hch->size() * sizeof(DChild)}};
      parts.insert(parts.end(), extra.begin(), extra.end());
      auto p = s.push_keep_many(parts);
      dF = (DFront *)p[0];
      dC = (DChild *)p[1];
      return p;
    };
    if (reqs.empty()) {
      if (hfr) push_fronts({});
      return;
    }
    // per class: the requests and their tile prefix (the kernels decode tile t
    // by a binary search; no per-tile descriptors from the host)
    std::vector<int> rid[2];
    std::vector<long long> pre[2] = {{0}, {0}};
    for (int q = 0; q < (int)reqs.size(); ++q) {
      const bool rb = reqs[q].front < (int)slot_rw.size() && slot_rw[reqs[q].front] >= RB_MIN_RANK;
      const int64_t nt = rb ? cdiv(reqs[q].nr, RB_T) * cdiv(reqs[q].nc, RB_T)
                            : cdiv(reqs[q].nr, SAMPLE_TR) * cdiv(reqs[q].nc, SAMPLE_TC);
      F->timing.sample_entries += (double)reqs[q].nr * reqs[q].nc;
      if (nt == 0) continue;
      rid[rb].push_back(q);
      pre[rb].push_back(pre[rb].back() + nt);
    }
    if (rid[0].empty() && rid[1].empty()) {
      if (hfr) push_fronts({});
      return;
    }
    SReq *dr;
    int *drid[2];
    long long *dpre[2];
    auto bytes_of = [](const auto &v) { return v.size() * sizeof(v[0]); };
    if (hfr) {
      auto p = push_fronts({{reqs.data(), reqs.size() * sizeof(SReq)},
                            {rid[0].data(), bytes_of(rid[0])},
                            {pre[0].data(), bytes_of(pre[0])},
                            {rid[1].data(), bytes_of(rid[1])},
                            {pre[1].data(), bytes_of(pre[1])}});
      dr = (SReq *)p[2];
      drid[0] = (int *)p[3];
      dpre[0] = (long long *)p[4];
      drid[1] = (int *)p[5];
      dpre[1] = (long long *)p[6];
    } else {
      auto p = s.push_keep_many({{reqs.data(), reqs.size() * sizeof(SReq)},
                                 {rid[0].data(), bytes_of(rid[0])},
                                 {pre[0].data(), bytes_of(pre[0])},
                                 {rid[1].data(), bytes_of(rid[1])},
                                 {pre[1].data(), bytes_of(pre[1])}});
      dr = (SReq *)p[0];
      drid[0] = (int *)p[1];
      dpre[0] = (long long *)p[2];
      drid[1] = (int *)p[3];
      dpre[1] = (long long *)p[4];
    }
    DFront *fF = dF;
    DChild *fC = dC;
    long long *pp = d_ap_ptr;
    int *pc = d_ap_col;
    double *pv = d_ap_val;
    if (!rid[0].empty()) {
      SampleTiles T{drid[0], dpre[0], (int)rid[0].size(), pre[0].back()};
      int grid = (int)std::min<int64_t>(T.ntiles, 148 * 32);
      s.launch([=](cudaStream_t st) {
        launch_pdl(k_sample, dim3(grid), dim3(SAMPLE_TC, SAMPLE_TRB), 0, st, dr, T, fF, fC, pp, pc, pv);
        check_launch();
      });
    }
    if (!rid[1].empty()) {
      SampleTiles T{drid[1], dpre[1], (int)rid[1].size(), pre[1].back()};
      int grid = (int)std::min<int64_t>(T.ntiles, 148 * 8);
      s.launch([=](cudaStream_t st) {
        launch_pdl(k_sample_rb, dim3(grid), dim3(256), RB_DYN, st, dr, T, fF, fC, pp, pc, pv);
        check_launch();
      });
    }
  }

  FacView as_factors(const BlockH &b) {
    FacView v;
    if (!b.dense) {
      v.col = b.col;
      v.ldc = b.rank;
      v.row = b.row;
      v.ldr = b.n;
      v.rank = b.rank;
      return v;
    }
    if (b.n <= b.m) {
      v.col = b.val;
      v.ldc = b.n;
      v.row = F->ident;
      v.ldr = F->ident_ld;
      v.rank = b.n;
    } else {
      v.col = F->ident;
      v.ldc = F->ident_ld;
      v.row = b.val;
      v.ldr = b.n;
      v.rank = b.m;
    }
    return v;
  }

  // retained pivot-block form: 1 (HODLR inverse form) when it holds fewer reals
  // than the explicit inverse; MFH_PFORM=0/1 forces one (tests)
  int pform_of(const HTree &T, int N) {
    const char *fe = getenv("MFH_PFORM");
    const int force = fe ? atoi(fe) : -1;
    if (force == 0 || force == 1) return force;
    double tm = 0;
    for (int v = 0; v < T.nslots; ++v) {
      if (T.leaf[v] == 1) {
        double sz = T.hi[v] - T.lo[v];
        tm += sz * sz;
      } else if (T.leaf[v] == 0) {
        const int lo = T.lo[v], hi = T.hi[v], mid = (lo + hi) >> 1;
        const double r1 = F->blocks[T.up[v]].erank(), r2 = F->blocks[T.lw[v]].erank();
        tm += (r1 + r2) * (hi - lo) + (mid - lo) * r1 + (hi - mid) * r2;
      }
    }
    return tm < (double)N * N ? 1 : 0;
  }

  // device storage of a compressed block by its lifetime (BlockH::kind)
  double *blk_alloc(const BlockH &b, size_t n) {
    if (b.kind == 0) return ctx->scratch.d(n);
    if (b.kind == 1) return upd.d(n, release_height(F->fronts[b.fi]));
    return F->arena.d(n);
  }

  // algorithmic flops of the low-rank child terms an extend-add request meets:
  // 2 r per sampled entry whose row and column both map into a child carrying
  // W V^T (multifrontal.py:340-347). Rows / columns: a range, or an index list.
  // (acc: the counter the flops go to; dense fallbacks sampled in the skeleton
  // phase count as that phase's executed flops)
  void count_lr(int fi, int r0, int nr, const std::vector<int> *rl, int c0, int nc, const std::vector<int> *cl,
                double *acc = nullptr) {
    const FrontH &f = F->fronts[fi];
    for (int ci : f.kids) {
      const FrontH &c = F->fronts[ci];
      if (c.upd != 1 || c.rw == 0 || c.densified) continue;  // a densified update is gathered
      const int *to = et->mapcache.maps.data() + et->mapcache.off[ci];
      auto hits = [&](int a0, int n, const std::vector<int> *l) {
        double h = 0;
        if (l)
          for (int x : *l) h += to[x] >= 0;
        else
          for (int x = a0; x < a0 + n; ++x) h += to[x] >= 0;
        return h;
      };
      *(acc ? acc : &F->timing.sample_lr_flops) += 2.0 * c.rw * hits(r0, nr, rl) * hits(c0, nc, cl);
    }
  }

  // ---- one height ----
  // host clock when each phase event was enqueued (MFH_HEIGHT_TRACE)
  std::chrono::steady_clock::time_point hts[8];
  // MFH_HOST_TRACE: host ms per factorization in a height's prologue: [0] front descriptors +
  // materialization enqueue, [1] dense requests + waiting for the planner + leaf requests
  // ([2] = host_select_ms, the block / request / pivot-LU job loop)
  double host_sec[2] = {0.0, 0.0};
  cudaEvent_t cur_evd = nullptr;  // recorded after the height's child updates have been materialized
  void process_height(const std::vector<int> &fis, cudaEvent_t *ev) {
    const auto h_t0 = std::chrono::steady_clock::now();
    for (auto &t : hts) t = h_t0;
    Sink s{ctx};
    std::vector<int> D, S;
    for (int fi : fis) (F->fronts[fi].structured ? S : D).push_back(fi);
    std::vector<DFront> dfr;
    std::vector<DChild> dch;
    std::vector<int> slot;
    // (materializing large child updates is enqueued here, so the GPU runs it
    // while the host builds this height's requests; it shows as the gap before
    // the sample phase)
    build_fronts_dev(s, fis, dfr, dch, slot);
    if (cur_evd) cudaEventRecord(cur_evd, ctx->s);
    host_sec[0] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h_t0).count();
    const auto h_t1 = std::chrono::steady_clock::now();
    DFront *dF = nullptr;  // pushed with the first sampling batch below
    DChild *dC = nullptr;

    std::vector<SReq> reqs;
    // ------------------------------------------------ dense fronts: assemble
    for (int fi : D) {
      FrontH &f = F->fronts[fi];
      f.F = upd.d((size_t)f.nh * f.nh, release_height(f));
      if (f.npv) f.piv = F->arena.i(f.npv);
      reqs.push_back(SReq{slot[fi], f.nh, f.nh, nullptr, nullptr, 0, 0, f.F, f.nh});
      count_lr(fi, 0, f.nh, nullptr, 0, f.nh, nullptr);
    }
    // ------------------------------------------------ structured: plan blocks
    std::vector<int> sblocks;  // all compressed blocks at this height
    for (int fi : S) {
      wait_planned(fi);
      FrontH &f = F->fronts[fi];
      const std::vector<int> &blist = F->front_blocks[fi];
      sblocks.insert(sblocks.end(), blist.begin(), blist.end());
      // leaves: sampled straight into their storage
      for (int tt : {f.pp, f.ff}) {
        if (tt < 0) continue;
        HTree &T = F->trees[tt];
        for (int v = 0; v < T.nslots; ++v)
          if (T.leaf[v] == 1) {
            int sz = T.hi[v] - T.lo[v];
            // pivot-block leaves live for the height, update leaves until the parent sampled them
            T.lval[v] = tt == f.pp ? ctx->scratch.d((size_t)sz * sz) : upd.d((size_t)sz * sz, release_height(f));
            count_lr(fi, T.base + T.lo[v], sz, nullptr, T.base + T.lo[v], sz, nullptr);
            reqs.push_back(SReq{slot[fi], sz, sz, nullptr, nullptr, T.base + T.lo[v], T.base + T.lo[v],
                                T.lval[v], sz});
          }
      }
    }
    auto t_sel0 = std::chrono::steady_clock::now();
    host_sec[1] += std::chrono::duration<double, std::milli>(t_sel0 - h_t1).count();
    // The index lists of every block (I, J, the core's column positions: three small arrays per
    // block, 35,000 at C5) are staged and sent as one copy with the sampling requests. Issued one
    // by one they filled the stream's queue behind the materialization (the host blocked in
    // cudaMemcpyAsync: 930 ms of "host" time at C5) and then trickled through the copy engine
    // with the SMs idle (the 63 / 112 ms idle gaps of C3 / C5).
    s.begin_batch();
    std::vector<CopyJob> core_copies;
    std::vector<PluJob> plu;
    // one contiguous int / double scratch for every core of the height, so the
    // ranks and pivot sequences come back in a single D2H copy
    int64_t itot = 0, dtot = 0;
    std::vector<int64_t> ioff, doff;
    for (int bi : sblocks) {
      BlockH &b = F->blocks[bi];
      ioff.push_back(itot);
      doff.push_back(dtot);
      itot += 4 * ((int64_t)b.I.size() + b.J.size()) + 4;
      dtot += (int64_t)b.I.size() + b.J.size() + 3;
    }
    int *pint_all = sblocks.empty() ? nullptr : ctx->scratch.i(itot);
    double *pdbl_all = sblocks.empty() ? nullptr : ctx->scratch.d(dtot);
    for (size_t qb = 0; qb < sblocks.size(); ++qb) {
      int bi = sblocks[qb];
      BlockH &b = F->blocks[bi];
      b.fullI = (int)b.I.size() == b.m;
      b.fullJ = (int)b.J.size() == b.n;
      int nI = (int)b.I.size(), nJ = (int)b.J.size();
      int cap = P.max_rank >= 0 ? (int)P.max_rank : std::min(nI, nJ);
      if (cap < 1) throw value_error("max_rank must be at least 1");
      b.kmax = std::min(std::min(nI, nJ), cap);
      // R = B(I, :)
      b.R = ctx->scratch.d((size_t)nI * b.n);
      b.ldR = b.n;
      b.d_I = b.fullI ? nullptr : s.push(b.I);
      reqs.push_back(SReq{slot[b.fi], nI, b.n, b.d_I, nullptr, b.I[0], b.c0, b.R, b.ldR});
      count_lr(b.fi, 0, 0, &b.I, b.c0, b.n, nullptr);
      if (b.fullI && b.fullJ) {
        b.C = b.R;
        b.ldC = b.n;
      } else {
        b.C = ctx->scratch.d((size_t)b.m * nJ);
        b.ldC = nJ;
        b.d_J = b.fullJ ? nullptr : s.push(b.J);
        reqs.push_back(SReq{slot[b.fi], b.m, nJ, nullptr, b.d_J, b.r0, b.J[0], b.C, b.ldC});
        count_lr(b.fi, b.r0, b.m, nullptr, 0, 0, &b.J);
      }
      // core = R[:, J - c0]
      b.core = ctx->scratch.d((size_t)nI * nJ);
      std::vector<int> inter(nJ);
      for (int q = 0; q < nJ; ++q) inter[q] = b.J[q] - b.c0;
      b.d_inter = b.fullJ ? nullptr : s.push(inter);
      core_copies.push_back(CopyJob{b.R, b.core, nI, nJ, b.ldR, nJ, nullptr, b.d_inter});
      // PLU scratch
      b.pint = pint_all + ioff[qb];
      b.pdbl = pdbl_all + doff[qb];
      PluJob j{};
      j.a = b.core;
      j.m = nI;
      j.n = nJ;
      j.ld = nJ;
      j.kmax = b.kmax;
      int *pi = b.pint;
      j.rowAt = pi;
      j.posR = pi + nI;
      j.actR = pi + 2 * nI;
      j.idxR = pi + 3 * nI;
      pi += 4 * nI;
      j.colAt = pi;
      j.posC = pi + nJ;
      j.actC = pi + 2 * nJ;
      j.idxC = pi + 3 * nJ;
      pi += 4 * nJ;
      j.out = pi;
      b.res = pi;
      j.mult = b.pdbl;
      j.prow = b.pdbl + nI;
      j.outd = b.pdbl + nI + nJ;
      b.resd = j.outd;
      plu.push_back(j);
      F->timing.pivot_lu_visits += 0;  // filled after ranks are known
    }
    {
      double dt = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_sel0).count();
      F->timing.host_ms += dt;
      F->timing.host_select_ms += dt;
    }

    cudaEventRecord(ev[0], ctx->s);
    hts[0] = std::chrono::steady_clock::now();
    run_sample(s, reqs, dF, dC, &dfr, &dch);
    s.flush();  // the staged index lists, descriptors and requests in one transfer, then the sampling launches
    cudaEventRecord(ev[1], ctx->s);
    hts[1] = std::chrono::steady_clock::now();

    // ------------------------------------------------ dense fronts: eliminate
    // (at heights with structured fronts this runs on the main stream inside
    // the pivot-LU window, overlapping the side-stream complete-pivot LU)
    auto dense_elim = [&]() {
      // F_pp^{-1} explicitly (multifrontal.py:302-306 semantics incl. the singular
      // check); Gpf = F_pp^{-1} F_pf; Schur update F_ff -= F_fp Gpf; Gfp = F_fp F_pp^{-1}
      std::vector<InvReq> inv;
      std::vector<GemmJob> g1, g2;
      s.begin_batch();
      for (int fi : D) {
        FrontH &f = F->fronts[fi];
        if (!f.npv) continue;
        f.flag_slot = new_flag("singular pivot block at node " + std::to_string(f.node), fi);
        f.Pinv = F->arena.d((size_t)f.npv * f.npv);
        int *pv = f.npv > INV_SMALL ? ctx->scratch.i(f.npv) : nullptr;
        inv.push_back(InvReq{f.F, f.npv, f.nh, f.Pinv, f.npv, pv, d_flags + f.flag_slot});
        if (f.nf) {
          f.Gpf = F->arena.d((size_t)f.npv * f.nf);
          f.Gfp = F->arena.d((size_t)f.nf * f.npv);
          g1.push_back(GemmJob{f.Pinv, f.F + f.npv, f.Gpf, f.npv, f.nf, f.npv, f.npv, f.nh, f.nf, 1.0, 0.0});
          g1.push_back(GemmJob{f.F + (int64_t)f.npv * f.nh, f.Pinv, f.Gfp, f.nf, f.npv, f.npv, f.nh, f.npv,
                               f.npv, 1.0, 0.0});
          g2.push_back(GemmJob{f.F + (int64_t)f.npv * f.nh, f.Gpf, f.F + (int64_t)f.npv * f.nh + f.npv, f.nf,
                               f.nf, f.npv, f.nh, f.nf, f.nh, -1.0, 1.0});
        }
      }
      {  // F_pp outlives the front buffer (node_factors apply_pf / apply_fp); copied
        // before the blocked inversion overwrites it with its LU
        std::vector<CopyJob> keep;
        for (int fi : D) {
          FrontH &f = F->fronts[fi];
          if (!f.npv || !f.nf) continue;
          f.Fpp = F->arena.d((size_t)f.npv * f.npv);
          keep.push_back(CopyJob{f.F, f.Fpp, f.npv, f.npv, f.nh, f.npv, nullptr, nullptr});
        }
        run_copy(s, keep);
      }
      run_inverse(s, inv);
      run_gemm(s, g1);
      run_gemm(s, g2);
      s.flush();
      for (int fi : D) {
        FrontH &f = F->fronts[fi];
        if (f.nf) {
          f.upd = 0;
          f.upd_dense = f.F + (int64_t)f.npv * f.nh + f.npv;
          f.upd_ld = f.nh;
        }
        f.front_reals = (int64_t)f.nh * f.nh;
        {
          const double np_ = f.npv, nf_ = f.nf;
          F->timing.dense_flops += (2.0 / 3.0) * np_ * np_ * np_ + 2.0 * np_ * np_ * nf_ + 2.0 * np_ * nf_ * nf_;
        }
        f.factor_reals = (f.npv ? (int64_t)f.npv * f.npv : 0) + 2 * (int64_t)f.npv * f.nf;
        if (f.npv) F->timing.apply_ref_bytes += 8.0 * (2.0 * f.npv * f.npv + 2.0 * f.npv * f.nf);
        f.upd_reals = (int64_t)f.nf * f.nf;
      }
    };
    if (S.empty()) {  // dense-only height: three events (each record costs GPU time)
      const double fl0 = ctx->flops_exec;
      dense_elim();
      F->timing.exec_flops_dense += ctx->flops_exec - fl0;
      cudaEventRecord(ev[2], ctx->s);
      return;
    }
    cudaEventRecord(ev[2], ctx->s);
    hts[2] = std::chrono::steady_clock::now();

    // ------------------------------------------------ structured: pivot LU
    run_copy(s, core_copies);
    {
      const double fl0 = ctx->flops_exec;
      run_plu(s, plu, P.eps, dense_elim);
      F->timing.exec_flops_dense += ctx->flops_exec - fl0;
    }
    cudaEventRecord(ev[3], ctx->s);
    hts[3] = std::chrono::steady_clock::now();
    // read ranks, status and pivot sequences: one D2H pair for the height
    {
      // one pinned landing area: ranks / pivots, their doubles and the error
      // flags arrive with the same sync (no pageable copies, no second trip)
      const size_t bi_ = sizeof(int) * itot, bd_ = sizeof(double) * dtot, bf_ = sizeof(int) * nflags;
      const size_t oD = (bi_ + 15) & ~size_t(15), oF = oD + ((bd_ + 15) & ~size_t(15));
      char *hb = ctx->readback(oF + bf_);
      CK(cudaMemcpyAsync(hb, pint_all, bi_, cudaMemcpyDeviceToHost, ctx->s));
      CK(cudaMemcpyAsync(hb + oD, pdbl_all, bd_, cudaMemcpyDeviceToHost, ctx->s));
      if (nflags) CK(cudaMemcpyAsync(hb + oF, d_flags, bf_, cudaMemcpyDeviceToHost, ctx->s));
      s.sync_reset();
      t_decide0 = std::chrono::steady_clock::now();
      std::vector<int> hi((const int *)hb, (const int *)hb + itot);
      std::vector<double> hd((const double *)(hb + oD), (const double *)(hb + oD) + dtot);
      check_flags(0, (const int *)(hb + oF));
      int first_err = -1;
      int crit = 0;  // steps of the longest core of the height (the latency-bound critical path)
      for (size_t q = 0; q < sblocks.size(); ++q) {
        BlockH &b = F->blocks[sblocks[q]];
        int nI = (int)b.I.size(), nJ = (int)b.J.size();
        const int *p = hi.data() + ioff[q];
        const int *out = p + 4 * (nI + nJ);
        const double *od = hd.data() + doff[q] + nI + nJ;
        b.rank = out[0];
        b.status = out[1];
        b.errk = out[2];
        b.ratio = od[0];
        b.errpiv = od[1];
        b.errprev = od[2];
        if (b.status && first_err < 0) first_err = (int)q;
        static const bool ptrace = getenv("MFH_PLU_TRACE") != nullptr;
        if (ptrace)
          fprintf(stderr, "[mfh plu] height %d block %d core %d x %d rank %d\n", F->fronts[b.fi].height, sblocks[q], nI,
                  nJ, b.rank);
        b.rows_phys = out[3] == 1;
        b.rowperm.assign(p, p + b.rank);
        b.colperm.assign(p + 4 * nI, p + 4 * nI + b.rank);
        // algorithmic visits: sum_{k < min(rank+1, min(I,J))} (|I|-k)(|J|-k)
        int kk = std::min(b.rank + 1, std::min(nI, nJ));
        double vis = 0;
        for (int k = 0; k < kk; ++k) vis += (double)(nI - k) * (nJ - k);
        F->timing.pivot_lu_visits += vis;
        crit = std::max(crit, kk);
      }
      F->timing.pivot_lu_crit_steps += crit;
      if (first_err >= 0) {
        BlockH &b = F->blocks[sblocks[first_err]];
        if (b.status == 2) throw runtime_error("internal: corrupt complete-pivot candidate");
        char buf[256];
        snprintf(buf, sizeof buf, "pivot %d magnitude %.3e exceeds twice the previous %.3e", b.errk,
                 b.errpiv, b.errprev);
        throw Error(MFH_EPIVOT, buf);
      }
    }
    // ------------------------------------------------ decisions + skeletons
    std::vector<LuExtractJob> lux;
    std::vector<SkelJob> skel;
    std::vector<SReq> dreq;
    std::vector<CopyJob> dcopy;
    for (int bi : sblocks) {
      BlockH &b = F->blocks[bi];
      int nI = (int)b.I.size(), nJ = (int)b.J.size();
      bool capped = P.max_rank >= 0 && b.rank == P.max_rank;
      bool full = b.fullI && b.fullJ;
      bool exhausted = b.rank == std::min(nI, nJ);
      bool unc = exhausted && !full && !capped;  // strict certificate (hodlr.py:92-97)
      int64_t lr_stored = (int64_t)(b.m + b.n) * b.rank;
      b.dense = unc || lr_stored > (int64_t)b.m * b.n;
      if (b.dense) {
        if (full) {
          // the full-selection panel R = B(all rows, :) IS the block, sampled by
          // the same kernels the dense fallback would re-run (hodlr.py:98-99):
          // adopt it (a pivot-block leaf lives exactly as long as R) or copy it
          if (b.kind == 0) {
            b.val = b.R;
          } else {
            b.val = blk_alloc(b, (size_t)b.m * b.n);
            dcopy.push_back(CopyJob{b.R, b.val, b.m, b.n, b.ldR, b.n, nullptr, nullptr});
          }
        } else {
          b.val = blk_alloc(b, (size_t)b.m * b.n);
          dreq.push_back(SReq{slot[b.fi], b.m, b.n, nullptr, nullptr, b.r0, b.c0, b.val, b.n});
          count_lr(b.fi, b.r0, b.m, nullptr, b.c0, b.n, nullptr, &F->timing.exec_flops_skeleton);
        }
        F->stats.n_dense_fallback++;
      } else if (b.rank > 0) {
        int r = b.rank;
        F->timing.skeleton_flops += (double)r * r * (b.m + b.n);
        double *lu = ctx->scratch.d((size_t)r * r);
        lux.push_back(LuExtractJob{b.core, nJ, r, b.rows_phys ? nullptr : b.pint, nullptr, lu});
        b.row = blk_alloc(b, (size_t)r * b.n);
        b.col = blk_alloc(b, (size_t)b.m * r);
        SkelJob sj{};
        sj.lu = lu;
        sj.r = r;
        sj.R = b.R;
        sj.ldR = b.ldR;
        sj.n = b.n;
        sj.rp = b.pint;
        sj.C = b.C;
        sj.ldC = b.ldC;
        sj.m = b.m;
        sj.cp = b.pint + 4 * nI;
        sj.row_out = b.row;
        sj.col_out = b.col;
        skel.push_back(sj);
      }
      F->stats.n_blocks++;
    }
    cudaEventRecord(ev[4], ctx->s);
    hts[4] = std::chrono::steady_clock::now();
    const double fl_skel0 = ctx->flops_exec;
    s.begin_batch();  // skeletons + dense fallbacks: no read-back until the next height
    if (!lux.empty()) {
      LuExtractJob *dj = s.push(lux);
      int64_t mx = 0;
      for (auto &j : lux) mx = std::max<int64_t>(mx, (int64_t)j.r * j.r);
      for (size_t b0 = 0; b0 < lux.size(); b0 += 60000) {
        unsigned cnt = (unsigned)std::min<size_t>(60000, lux.size() - b0);
        LuExtractJob *p = dj + b0;
        dim3 grid((unsigned)std::min<int64_t>(cdiv(mx, 256), 32), cnt);
        s.launch([=](cudaStream_t st) {
          launch_pdl(k_lu_extract, dim3(grid), dim3(256), 0, st, p);
          check_launch();
        });
      }
      // row factor = L^{-1} R[rp[:r], :] ; col factor = C[:, cp[:r]] U^{-1} (bdlr.py:178-183):
      // gathered panels times the explicit triangular inverses (one GEMM each)
      std::vector<CopyJob> gat;
      std::vector<TriInvReq> tinv;
      std::vector<GemmJob> app;
      for (auto &sj : skel) {
        double *Rg = ctx->scratch.d((size_t)sj.r * sj.n), *Cg = ctx->scratch.d((size_t)sj.m * sj.r);
        double *Li = ctx->scratch.d((size_t)sj.r * sj.r), *Ui = ctx->scratch.d((size_t)sj.r * sj.r);
        gat.push_back(CopyJob{sj.R, Rg, sj.r, sj.n, sj.ldR, sj.n, sj.rp, nullptr});
        gat.push_back(CopyJob{sj.C, Cg, sj.m, sj.r, sj.ldC, sj.r, nullptr, sj.cp});
        tinv.push_back(TriInvReq{sj.lu, sj.r, sj.r, 0, Li});
        tinv.push_back(TriInvReq{sj.lu, sj.r, sj.r, 1, Ui});
        app.push_back(GemmJob{Li, Rg, sj.row_out, sj.r, sj.n, sj.r, sj.r, sj.n, sj.n, 1.0, 0.0});
        app.push_back(GemmJob{Cg, Ui, sj.col_out, sj.m, sj.r, sj.r, sj.r, sj.r, sj.r, 1.0, 0.0});
      }
      run_copy(s, gat);
      run_tri_inv(s, tinv);
      run_gemm(s, app);
    }
    run_copy(s, dcopy);
    run_sample(s, dreq, dF, dC);
    s.flush();
    F->timing.exec_flops_skeleton += ctx->flops_exec - fl_skel0;
    cudaEventRecord(ev[5], ctx->s);
    last_decide_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_decide0).count();
    hts[5] = std::chrono::steady_clock::now();

    // ------------------------------------------------ device HNode tables of the
    // update HODLRs (what the parent's sampler descends), one upload; they die
    // with the update
    {
      std::vector<HNode> all;
      std::vector<std::pair<int, size_t>> where;
      std::vector<std::pair<size_t, int>> seg;  // (first node, release height) per front
      for (int fi : S) {
        FrontH &f = F->fronts[fi];
        if (f.ff < 0) continue;
        HTree &T = F->trees[f.ff];
        where.push_back({f.ff, all.size()});
        seg.push_back({all.size(), release_height(f)});
        for (int v = 0; v < T.nslots; ++v) {
          HNode h{};
          if (T.leaf[v] == 1)
            h.leaf = T.lval[v];
          else if (T.leaf[v] == 0) {
            h.up = F->blocks[T.up[v]].dev();
            h.lw = F->blocks[T.lw[v]].dev();
          }
          all.push_back(h);
        }
      }
      if (!all.empty()) {
        int rh = 0;
        for (auto &q : seg) rh = std::max(rh, q.second);
        HNode *d = (HNode *)upd.alloc(sizeof(HNode) * all.size(), rh);
        for (auto &w : where) F->trees[w.first].d_nodes = d + w.second;
        s.push_to(d, all.data(), sizeof(HNode) * all.size());
      }
    }

    const double fl_hodlr0 = ctx->flops_exec;
    s.begin_batch();  // HODLR factorization + eliminate: host-planned, one descriptor transfer
    // ------------------------------------------------ HODLR factorization of pp
    // hodlr_factorize (hodlr.py:312-357) in explicit-inverse form, one launch
    // group per stage of a tree level, batched over every front of the height:
    //   H_v = diag(H_L, H_R) + P Q,  P = diag(col1, col2),  Q = [[0, row1], [row2, 0]]
    //   core = I + Q D^{-1} P = [[I, row1 x_bot], [row2 x_top, I]]  (the reference's core)
    //   H_v^{-1} = D^{-1} - (D^{-1} P) core^{-1} (Q D^{-1})
    // When a pivot-block HODLR is effectively dense (dense-fallback blocks
    // everywhere, so its Woodbury cores are as large as the blocks), its exact
    // inverse is cheaper as ONE dense blocked inversion of the assembled
    // compressed matrix than as a chain of large core inversions: same
    // compressed operator, exact either way. Per-tree choice by a cost model.
    std::vector<int> ptrees, dtrees;
    for (int fi : S) {
      FrontH &f = F->fronts[fi];
      if (f.pp < 0) continue;
      HTree &T = F->trees[f.pp];
      double core3 = 0.0;
      for (int v = 0; v < T.nslots; ++v)
        if (T.leaf[v] == 0) {
          double rr = (double)F->blocks[T.up[v]].erank() + F->blocks[T.lw[v]].erank();
          core3 += rr * rr * rr;
        }
      double N = (double)f.npv;
      // with Schur-complement cores the level-by-level inverse wins at C2 even
      // for effectively dense blocks (measured: 28.5 ms vs 36 ms at frac 0.3);
      // the dense path stays available for other matrix families
      static const double dense_frac = std::getenv("MFH_DENSE_FRAC") ? std::atof(std::getenv("MFH_DENSE_FRAC")) : 1e30;
      (core3 >= dense_frac * N * N * N && f.npv > INV_SMALL ? dtrees : ptrees).push_back(f.pp);
    }
    {
      std::vector<CopyJob> lc;
      std::vector<InvReq> leaves, dense_inv;
      std::vector<GemmJob> dense_lr;
      for (int tt : dtrees) {
        HTree &T = F->trees[tt];
        FrontH &f = F->fronts[T.fi];
        const int N = f.npv;
        f.Hinv = F->arena.d((size_t)N * N);
        double *Hd = ctx->scratch.d((size_t)N * N);
        for (int v = 0; v < T.nslots; ++v) {
          if (T.leaf[v] == 1) {
            int lo = T.lo[v], sz = T.hi[v] - T.lo[v];
            lc.push_back(CopyJob{T.lval[v], Hd + (int64_t)lo * N + lo, sz, sz, sz, N, nullptr, nullptr});
            // the reference's leaf singularity check (hodlr.py:325-328), flag only
            std::string msg = "singular pivot in leaf block [" + std::to_string(T.lo[v]) + ", " +
                              std::to_string(T.hi[v]) + ")";
            T.lflag[v] = new_flag(msg, (int64_t)T.fi * 1000000 + v);
            if (sz <= INV_SMALL) {
              double *chk = ctx->scratch.d((size_t)sz * sz);
              lc.push_back(CopyJob{T.lval[v], chk, sz, sz, sz, sz, nullptr, nullptr});
              leaves.push_back(InvReq{chk, sz, sz, chk, sz, nullptr, d_flags + T.lflag[v]});
            }
          } else if (T.leaf[v] == 0) {
            FacView f1 = as_factors(F->blocks[T.up[v]]), f2 = as_factors(F->blocks[T.lw[v]]);
            T.f1[v] = f1;
            T.f2[v] = f2;
            T.r1[v] = f1.rank;
            T.r2[v] = f2.rank;
            const int lo = T.lo[v], hi = T.hi[v], mid = (lo + hi) >> 1;
            for (int side = 0; side < 2; ++side) {
              const BlockH &b = F->blocks[side == 0 ? T.up[v] : T.lw[v]];
              double *dst = Hd + (side == 0 ? (int64_t)lo * N + mid : (int64_t)mid * N + lo);
              if (b.dense)
                lc.push_back(CopyJob{b.val, dst, b.m, b.n, b.n, N, nullptr, nullptr});
              else  // rank 0 writes zeros (k = 0)
                dense_lr.push_back(GemmJob{b.col, b.row, dst, b.m, b.n, b.rank, std::max(1, b.rank), b.n, N, 1.0, 0.0});
            }
          }
        }
        int fl = new_flag("singular coupling core at node [0, " + std::to_string(N) + ")", (int64_t)T.fi * 1000000);
        dense_inv.push_back(InvReq{Hd, N, N, f.Hinv, N, ctx->scratch.i(N), d_flags + fl});
      }
      run_copy(s, lc);
      lc.clear();
      run_gemm(s, dense_lr);
      run_inverse(s, dense_inv);

      for (int tt : ptrees) {
        HTree &T = F->trees[tt];
        FrontH &f = F->fronts[T.fi];
        const int N = f.npv;
        // retained form of the pivot-block inverse (a14/a15): the explicit n_p^2
        // inverse, or the HODLR inverse form (leaf inverses, per node X_v and
        // Tm_v: H^{-1} = blockdiag(L^{-1}) - sum_v X_v Tm_v), whichever holds
        // fewer reals -- it is also what one apply reads
        f.pform = pform_of(T, N);
        f.Hinv = f.pform ? ctx->scratch.d((size_t)N * N) : F->arena.d((size_t)N * N);
        {
          double *hz = f.Hinv;
          const size_t nb = sizeof(double) * (size_t)N * N;
          s.launch([hz, nb](cudaStream_t st) { CK(cudaMemsetAsync(hz, 0, nb, st)); });
        }
        for (int v = 0; v < T.nslots; ++v)
          if (T.leaf[v] == 1) {
            int lo = T.lo[v], sz = T.hi[v] - T.lo[v];
            double *blk = f.Hinv + (int64_t)lo * N + lo;
            std::string msg = "singular pivot in leaf block [" + std::to_string(T.lo[v]) + ", " +
                              std::to_string(T.hi[v]) + ")";
            T.lflag[v] = new_flag(msg, (int64_t)T.fi * 1000000 + v);
            if (sz <= INV_SMALL) {
              lc.push_back(CopyJob{T.lval[v], blk, sz, sz, sz, N, nullptr, nullptr});
              leaves.push_back(InvReq{blk, sz, N, blk, N, nullptr, d_flags + T.lflag[v]});
            } else {
              T.lpiv[v] = ctx->scratch.i(sz);
              leaves.push_back(InvReq{T.lval[v], sz, sz, blk, N, T.lpiv[v], d_flags + T.lflag[v]});
            }
          }
      }
      run_copy(s, lc);
      run_inverse(s, leaves);
      {  // HODLR inverse form: keep the leaf inverses before the levels update Hinv's diagonal
        std::vector<CopyJob> lk;
        for (int tt : ptrees) {
          HTree &T = F->trees[tt];
          FrontH &f = F->fronts[T.fi];
          if (!f.pform) continue;
          f.tleaf.clear();
          f.tnode.clear();
          f.wlen = 0;
          const int N = f.npv;
          for (int v = 0; v < T.nslots; ++v)
            if (T.leaf[v] == 1) {
              const int lo = T.lo[v], sz = T.hi[v] - T.lo[v];
              FrontH::TmLeaf L{};
              L.slot = v;
              L.lo = lo;
              L.sz = sz;
              L.Linv = F->arena.d((size_t)sz * sz);
              lk.push_back(CopyJob{f.Hinv + (int64_t)lo * N + lo, L.Linv, sz, sz, N, sz, nullptr, nullptr});
              f.tleaf.push_back(L);
            }
        }
        run_copy(s, lk);
      }
      int maxd = 0;
      for (int tt : ptrees) maxd = std::max(maxd, F->trees[tt].maxdepth);
      for (int d = maxd; d >= 0; --d) {
        // Per node v = [L | R] (hodlr.py:330-352) with D = diag(H_L, H_R),
        // x_top = H_L^{-1} col1, x_bot = H_R^{-1} col2, y_top = row1 H_R^{-1},
        // y_bot = row2 H_L^{-1}, and the Woodbury core C = [[I, A], [B, I]]
        // (A = row1 x_bot, B = row2 x_top, the reference's core):
        //   H_v^{-1} = D^{-1} - diag(x_top, x_bot) Tm,  Tm = C^{-1} [[0, y_top], [y_bot, 0]].
        // C^{-1} is never formed: through the Schur complement of the smaller
        // side, S = I - B A (r2 <= r1),
        //   Tm = [[-A Z1, y_top + A Z2], [Z1, -Z2]],  Z1 = S^{-1} y_bot, Z2 = S^{-1} (B y_top)
        // (mirrored with S = I - A B when r1 < r2); C is singular iff S is
        // (the reference's core check, hodlr.py:346-352). Launches per level:
        // x / y, A / B, S + (B y_top | A y_bot), S^{-1}, Z, the top rows, Hinv.
        std::vector<GemmJob> ga, gc, gsch, gz, gt, ge;
        std::vector<double *> ip;
        std::vector<int> idim, ild;
        std::vector<InvReq> invs;
        bool any = false;
        for (int tt : ptrees) {
          HTree &T = F->trees[tt];
          FrontH &f = F->fronts[T.fi];
          const int N = f.npv;
          for (int v = 0; v < T.nslots; ++v) {
            if (T.leaf[v] != 0 || T.depth[v] != d) continue;
            FacView f1 = as_factors(F->blocks[T.up[v]]);
            FacView f2 = as_factors(F->blocks[T.lw[v]]);
            T.f1[v] = f1;
            T.f2[v] = f2;
            const int lo = T.lo[v], hi = T.hi[v], mid = (lo + hi) >> 1;
            const int m1 = mid - lo, m2 = hi - mid, nv = hi - lo;
            const int r1 = f1.rank, r2 = f2.rank, rr = r1 + r2;
            T.r1[v] = r1;
            T.r2[v] = r2;
            if (rr == 0) continue;
            any = true;
            double *HLL = f.Hinv + (int64_t)lo * N + lo, *HRR = f.Hinv + (int64_t)mid * N + mid;
            double *xt = ctx->scratch.d((size_t)m1 * std::max(1, r1));
            double *xb = ctx->scratch.d((size_t)m2 * std::max(1, r2));
            double *Tm = f.pform ? F->arena.d((size_t)rr * nv) : ctx->scratch.d((size_t)rr * nv);
            if (f.pform) {
              FrontH::TmNode tn{};
              tn.slot = v;
              tn.lo = lo;
              tn.nv = nv;
              tn.r1 = r1;
              tn.r2 = r2;
              tn.Tm = Tm;
              tn.xt = xt;
              tn.xb = xb;
              tn.woff = f.wlen;
              f.wlen += rr;
              f.tnode.push_back(tn);
            }
            double *Ttl = Tm, *Ttr = Tm + m1;                                      // rows [0, r1)
            double *Tbl = Tm + (int64_t)r1 * nv, *Tbr = Tm + (int64_t)r1 * nv + m1;  // rows [r1, rr)
            if (r1) ga.push_back(GemmJob{HLL, f1.col, xt, m1, r1, m1, N, f1.ldc, r1, 1.0, 0.0});
            if (r2) ga.push_back(GemmJob{HRR, f2.col, xb, m2, r2, m2, N, f2.ldc, r2, 1.0, 0.0});
            std::string msg = "singular coupling core at node [" + std::to_string(lo) + ", " + std::to_string(hi) + ")";
            if (!(r1 && r2)) {  // C = I: Tm = [[0, y_top]] or [[y_bot, 0]]
              if (r1) {
                ga.push_back(GemmJob{f1.row, HRR, Ttr, r1, m2, m2, f1.ldr, N, nv, 1.0, 0.0});
                gt.push_back(GemmJob{nullptr, nullptr, Ttl, r1, m1, 0, 1, 1, nv, 0.0, 0.0});  // zeros
              } else {
                ga.push_back(GemmJob{f2.row, HLL, Tbl, r2, m1, m1, f2.ldr, N, nv, 1.0, 0.0});
                gt.push_back(GemmJob{nullptr, nullptr, Tbr, r2, m2, 0, 1, 1, nv, 0.0, 0.0});
              }
            } else {
              const int fl = new_flag(msg, (int64_t)T.fi * 1000000 + v);
              double *A = ctx->scratch.d((size_t)r1 * r2), *B = ctx->scratch.d((size_t)r2 * r1);
              gc.push_back(GemmJob{f1.row, xb, A, r1, r2, m2, f1.ldr, r2, r2, 1.0, 0.0});
              gc.push_back(GemmJob{f2.row, xt, B, r2, r1, m1, f2.ldr, r1, r1, 1.0, 0.0});
              if (r2 <= r1) {
                double *yb = ctx->scratch.d((size_t)r2 * m1), *P = ctx->scratch.d((size_t)r2 * m2);
                double *S = ctx->scratch.d((size_t)r2 * r2), *Si = ctx->scratch.d((size_t)r2 * r2);
                ga.push_back(GemmJob{f1.row, HRR, Ttr, r1, m2, m2, f1.ldr, N, nv, 1.0, 0.0});  // y_top in place
                ga.push_back(GemmJob{f2.row, HLL, yb, r2, m1, m1, f2.ldr, N, m1, 1.0, 0.0});
                ip.push_back(S), idim.push_back(r2), ild.push_back(r2);
                gsch.push_back(GemmJob{B, A, S, r2, r2, r1, r1, r2, r2, -1.0, 1.0});
                gsch.push_back(GemmJob{B, Ttr, P, r2, m2, r1, r1, nv, m2, 1.0, 0.0});
                invs.push_back(InvReq{S, r2, r2, Si, r2, r2 > INV_SMALL ? ctx->scratch.i(r2) : nullptr, d_flags + fl});
                gz.push_back(GemmJob{Si, yb, Tbl, r2, m1, r2, r2, m1, nv, 1.0, 0.0});
                gz.push_back(GemmJob{Si, P, Tbr, r2, m2, r2, r2, m2, nv, -1.0, 0.0});
                gt.push_back(GemmJob{A, Tbl, Ttl, r1, m1, r2, r2, nv, nv, -1.0, 0.0});
                gt.push_back(GemmJob{A, Tbr, Ttr, r1, m2, r2, r2, nv, nv, -1.0, 1.0});
              } else {
                double *yt = ctx->scratch.d((size_t)r1 * m2), *Q = ctx->scratch.d((size_t)r1 * m1);
                double *S = ctx->scratch.d((size_t)r1 * r1), *Si = ctx->scratch.d((size_t)r1 * r1);
                ga.push_back(GemmJob{f1.row, HRR, yt, r1, m2, m2, f1.ldr, N, m2, 1.0, 0.0});
                ga.push_back(GemmJob{f2.row, HLL, Tbl, r2, m1, m1, f2.ldr, N, nv, 1.0, 0.0});  // y_bot in place
                ip.push_back(S), idim.push_back(r1), ild.push_back(r1);
                gsch.push_back(GemmJob{A, B, S, r1, r1, r2, r2, r1, r1, -1.0, 1.0});
                gsch.push_back(GemmJob{A, Tbl, Q, r1, m1, r2, r2, nv, m1, 1.0, 0.0});
                invs.push_back(InvReq{S, r1, r1, Si, r1, r1 > INV_SMALL ? ctx->scratch.i(r1) : nullptr, d_flags + fl});
                gz.push_back(GemmJob{Si, Q, Ttl, r1, m1, r1, r1, m1, nv, -1.0, 0.0});
                gz.push_back(GemmJob{Si, yt, Ttr, r1, m2, r1, r1, m2, nv, 1.0, 0.0});
                gt.push_back(GemmJob{B, Ttl, Tbl, r2, m1, r1, r1, nv, nv, -1.0, 1.0});
                gt.push_back(GemmJob{B, Ttr, Tbr, r2, m2, r1, r1, nv, nv, -1.0, 0.0});
              }
            }
            // H_v^{-1} rows L -= x_top Tm[:r1, :], rows R -= x_bot Tm[r1:, :]
            if (r1) ge.push_back(GemmJob{xt, Tm, HLL, m1, nv, r1, r1, nv, N, -1.0, 1.0});
            if (r2)
              ge.push_back(GemmJob{xb, Tm + (int64_t)r1 * nv, f.Hinv + (int64_t)mid * N + lo, m2, nv, r2, r2, nv, N,
                                   -1.0, 1.0});
          }
        }
        if (!any) continue;
        run_identity(s, ip, idim, ild);
        run_gemm(s, ga);
        run_gemm(s, gc);
        run_gemm(s, gsch);
        run_inverse(s, invs);
        run_gemm(s, gz);
        run_gemm(s, gt);
        run_gemm(s, ge);
      }
      // HODLR inverse form: per leaf, the rows of its ancestors' X_v = diag(x_top,
      // x_bot) side by side (XL, sz x K) and where each column's w entry lives
      // (idx into the front's w segment): y_leaf = L^{-1} b_leaf - XL w[idx]
      std::vector<CopyJob> xl;
      for (int tt : ptrees) {
        HTree &T = F->trees[tt];
        FrontH &f = F->fronts[T.fi];
        if (!f.pform) continue;
        std::map<int, const FrontH::TmNode *> by_slot;
        for (auto &tn : f.tnode) by_slot[tn.slot] = &tn;
        for (auto &L : f.tleaf) {
          std::vector<const FrontH::TmNode *> anc;
          for (int v = L.slot; v > 0;) {
            v = (v - 1) / 2;
            auto it = by_slot.find(v);
            if (it != by_slot.end()) anc.push_back(it->second);
          }
          std::reverse(anc.begin(), anc.end());  // root first
          std::vector<long long> idx;
          std::vector<std::array<int64_t, 4>> cols;  // (node, left?, column offset, width)
          for (auto *tn : anc) {
            const int mid = tn->lo + tn->nv / 2;
            const bool left = L.lo < mid;
            const int r = left ? tn->r1 : tn->r2;
            if (r == 0) continue;
            cols.push_back({(int64_t)(tn - f.tnode.data()), left, (int64_t)idx.size(), r});
            for (int j = 0; j < r; ++j) idx.push_back(tn->woff + (left ? 0 : tn->r1) + j);
          }
          L.K = (int)idx.size();
          if (!L.K) continue;
          L.XL = F->arena.d((size_t)L.sz * L.K);
          L.idx = (long long *)F->arena.alloc(sizeof(long long) * idx.size());
          s.push_to(L.idx, idx.data(), sizeof(long long) * idx.size());
          for (auto &c : cols) {
            const FrontH::TmNode &tn = f.tnode[c[0]];
            const int mid = tn.lo + tn.nv / 2, r = (int)c[3];
            const double *src = c[1] ? tn.xt + (int64_t)(L.lo - tn.lo) * r : tn.xb + (int64_t)(L.lo - mid) * r;
            xl.push_back(CopyJob{src, L.XL + c[2], L.sz, r, r, L.K, nullptr, nullptr});
          }
        }
      }
      run_copy(s, xl);
    }
    s.flush();
    F->timing.exec_flops_hodlr += ctx->flops_exec - fl_hodlr0;
    cudaEventRecord(ev[6], ctx->s);
    const double fl_elim0 = ctx->flops_exec;
    s.begin_batch();
    hts[6] = std::chrono::steady_clock::now();

    // ------------------------------------------------ eliminate_hodlr (W, V)  (multifrontal.py:411-456)
    {
      std::vector<GemmJob> g0, g1, g2;
      struct El {
        int fi;
        FacView pf, fp;
      };
      std::vector<El> els;
      for (int fi : S) {
        FrontH &f = F->fronts[fi];
        if (!(f.npv && f.nf)) continue;
        El e{fi, as_factors(F->blocks[f.pf]), as_factors(F->blocks[f.fp])};
        const int N = f.npv, nf = f.nf;
        const BlockH &bpf = F->blocks[f.pf], &bfp = F->blocks[f.fp];
        // x = H^{-1} col_pf (multifrontal.py:428): the eliminate core and, for a
        // low-rank F_pf, the apply's downward operator Xp. A dense-fallback F_pf
        // enters as (F_pf, I) or (I, F_pf) (hodlr.py:59-63): x is H^{-1} F_pf
        // (factor-time scratch) or H^{-1} itself; the apply then uses F_pf
        // directly (x_piv = H^{-1} (b_piv - F_pf x_fro)), so nothing n_p x nf
        // beyond the block itself is kept
        if (!bpf.dense) {
          f.Xp = F->arena.d((size_t)N * std::max(1, e.pf.rank));
          if (e.pf.rank) g0.push_back(GemmJob{f.Hinv, e.pf.col, f.Xp, N, e.pf.rank, N, N, e.pf.ldc, e.pf.rank, 1.0, 0.0});
        } else if (nf <= N) {
          f.Xp = ctx->scratch.d((size_t)N * nf);
          g0.push_back(GemmJob{f.Hinv, bpf.val, f.Xp, N, nf, N, N, nf, nf, 1.0, 0.0});
        } else {
          f.Xp = f.Hinv;  // H^{-1} I (rank n_p = N, leading dimension N)
        }
        // upward apply operator RH = row_fp H^{-1} (low rank; a dense F_fp is
        // applied to y_piv = H^{-1} b_piv directly)
        if (!bfp.dense) {
          f.RH = F->arena.d((size_t)std::max(1, e.fp.rank) * N);
          if (e.fp.rank) g0.push_back(GemmJob{e.fp.row, f.Hinv, f.RH, e.fp.rank, N, N, e.fp.ldr, N, N, 1.0, 0.0});
        }
        els.push_back(e);
      }
      run_gemm(s, g0);
      for (auto &e : els) {
        FrontH &f = F->fronts[e.fi];
        int rpf = e.pf.rank, rfp = e.fp.rank;
        double *core = ctx->scratch.d((size_t)std::max(1, rfp) * std::max(1, rpf));
        if (rfp && rpf)
          g1.push_back(GemmJob{e.fp.row, f.Xp, core, rfp, rpf, f.npv, e.fp.ldr, rpf, rpf, 1.0, 0.0});
        if (rpf <= rfp) {
          // W = col_fp @ core (nf x r_pf), V = row_pf^T  -> Vt = row_pf
          f.rw = rpf;
          if (rpf) {
            double *W = upd.d((size_t)f.nf * rpf, release_height(f));
            g2.push_back(GemmJob{e.fp.col, core, W, f.nf, rpf, rfp, e.fp.ldc, rpf, rpf, 1.0, 0.0});
            f.W = W;
            f.ldw = rpf;
            f.Vt = e.pf.row;
            f.ldv = e.pf.ldr;
          }
        } else {
          // W = col_fp, V = (core @ row_pf)^T -> Vt = core @ row_pf (r_fp x nf)
          f.rw = rfp;
          f.W = e.fp.col;
          f.ldw = e.fp.ldc;
          double *Vt = upd.d((size_t)rfp * f.nf, release_height(f));
          g2.push_back(GemmJob{core, e.pf.row, Vt, rfp, f.nf, rpf, rpf, e.pf.ldr, f.nf, 1.0, 0.0});
          f.Vt = Vt;
          f.ldv = f.nf;
        }
      }
      run_gemm(s, g1);
      run_gemm(s, g2);
    }
    s.flush();
    F->timing.exec_flops_elim += ctx->flops_exec - fl_elim0;
    cudaEventRecord(ev[7], ctx->s);
    hts[7] = std::chrono::steady_clock::now();
    static const bool htr = getenv("MFH_HEIGHT_TRACE") != nullptr;
    if (htr) {
      auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
      fprintf(stderr, "[mfh host height %d] enqueue-at (us from entry): ev0 %.0f ev1 %.0f ev2 %.0f ev3 %.0f ev4 %.0f ev5 %.0f ev6 %.0f ev7 %.0f\n",
              F->fronts[fis[0]].height, us(h_t0, hts[0]), us(h_t0, hts[1]), us(h_t0, hts[2]), us(h_t0, hts[3]),
              us(h_t0, hts[4]), us(h_t0, hts[5]), us(h_t0, hts[6]), us(h_t0, hts[7]));
    }

    // ------------------------------------------------ accounting (host)
    for (int fi : S) {
      FrontH &f = F->fronts[fi];
      auto tree_stored = [&](int tt) -> int64_t {
        if (tt < 0) return 0;
        HTree &T = F->trees[tt];
        int64_t s2 = 0;
        for (int v = 0; v < T.nslots; ++v) {
          if (T.leaf[v] == 1) {
            int64_t sz = T.hi[v] - T.lo[v];
            s2 += sz * sz;
          } else if (T.leaf[v] == 0) {
            s2 += F->blocks[T.up[v]].stored() + F->blocks[T.lw[v]].stored();
          }
        }
        return s2;
      };
      auto tree_hint = [&](int tt) -> int64_t {
        if (tt < 0) return 0;
        HTree &T = F->trees[tt];
        int64_t h = 0;
        for (int v = 0; v < T.nslots; ++v)
          if (T.leaf[v] == 0)
            h = std::max<int64_t>(h, std::max(F->blocks[T.up[v]].erank(), F->blocks[T.lw[v]].erank()));
        return h;
      };
      auto factor_stored = [&](int tt) -> int64_t {
        if (tt < 0) return 0;
        HTree &T = F->trees[tt];
        int64_t s2 = 0;
        for (int v = 0; v < T.nslots; ++v) {
          if (T.leaf[v] == 1) {
            int64_t sz = T.hi[v] - T.lo[v];
            s2 += sz * sz;
          } else if (T.leaf[v] == 0) {
            int lo = T.lo[v], hi = T.hi[v], mid = (lo + hi) >> 1;
            int64_t m1 = mid - lo, m2 = hi - mid, r1 = T.r1[v], r2 = T.r2[v];
            s2 += m1 * r1 + m2 * r2 + r1 * m2 + r2 * m1;
            if (r1 + r2) s2 += (r1 + r2) * (r1 + r2);
          }
        }
        return s2;
      };
      // algorithmic flops of the reference's hodlr_factorize / eliminate_hodlr
      // on this structure: S(v) = stored reals of v's factor subtree
      double s_pp = 0;
      if (f.pp >= 0) {
        HTree &T = F->trees[f.pp];
        std::vector<double> S(T.nslots, 0.0);
        for (int v = T.nslots - 1; v >= 0; --v) {
          if (T.leaf[v] == 1) {
            const double sz = T.hi[v] - T.lo[v];
            S[v] = sz * sz;
            F->timing.hodlr_flops += (2.0 / 3.0) * sz * sz * sz;
          } else if (T.leaf[v] == 0) {
            const double lo = T.lo[v], hi = T.hi[v], mid = (T.lo[v] + T.hi[v]) >> 1;
            const double r1 = F->blocks[T.up[v]].erank(), r2 = F->blocks[T.lw[v]].erank();
            const double m1 = mid - lo, m2 = hi - mid, rr = r1 + r2;
            const double SL = S[2 * v + 1], SR = S[2 * v + 2];
            S[v] = SL + SR + m1 * r1 + m2 * r2 + r1 * m2 + r2 * m1 + rr * rr;
            F->timing.hodlr_flops += 2.0 * r1 * SL + 2.0 * r2 * SR + 2.0 * r1 * r2 * (hi - lo) + (2.0 / 3.0) * rr * rr * rr;
          }
        }
        s_pp = S[0];
      }
      if (f.npv && f.nf) {
        const double rpf = F->blocks[f.pf].erank(), rfp = F->blocks[f.fp].erank();
        F->timing.elim_flops += 2.0 * rpf * s_pp + 2.0 * rfp * f.npv * rpf + 2.0 * f.nf * rfp * rpf;
      }
      int64_t pfs = f.pf >= 0 ? F->blocks[f.pf].stored() : 0;
      int64_t fps = f.fp >= 0 ? F->blocks[f.fp].stored() : 0;
      f.front_reals = tree_stored(f.pp) + pfs + fps + tree_stored(f.ff);
      f.factor_reals = factor_stored(f.pp) + pfs + fps;
      if (f.npv) F->timing.apply_ref_bytes += 8.0 * (2.0 * factor_stored(f.pp) + pfs + fps);
      f.upd_reals = f.nf ? tree_stored(f.ff) + 2 * (int64_t)f.nf * f.rw : 0;
      int64_t h = std::max(tree_hint(f.pp), tree_hint(f.ff));
      if (f.pf >= 0) h = std::max<int64_t>(h, F->blocks[f.pf].erank());
      if (f.fp >= 0) h = std::max<int64_t>(h, F->blocks[f.fp].erank());
      f.hint = h;
      if (f.nf) f.upd = 1;
      // structured_alloc_note(nf) on x, W, V (multifrontal.py:421-438)
      if (f.npv && f.nf) {
        int64_t rpf = as_factors(F->blocks[f.pf]).rank;
        auto note = [&](int64_t r, int64_t c) {
          if (f.nf > 0 && r >= f.nf && c >= f.nf) F->stats.full_square_allocs++;
        };
        note(f.npv, rpf);
        note(f.nf, f.rw);
        note(f.nf, f.rw);
      }
    }
  }

  // ---- sharded: every cut root's update, densified by the
  // owner through a virtual front with no pivots (so each entry is bitwise
  // the per-child term the parent's sampler would add), summed over ranks;
  // the top fronts then see every cut root as a dense child
  void exchange_updates(const std::vector<int> &cuts) {
    std::vector<int64_t> coff;
    int64_t T = 0;
    for (int q : cuts) {
      coff.push_back(T);
      T += (int64_t)F->fronts[q].nf * F->fronts[q].nf;
    }
    Sink s{ctx};
    s.sync_reset();
    check_flags(0);
    ctx->scratch.reset();
    double *imp = F->arena.d(std::max<int64_t>(1, T));
    CK(cudaMemsetAsync(imp, 0, sizeof(double) * std::max<int64_t>(1, T), ctx->s));
    std::vector<DFront> dfr;
    std::vector<DChild> dch;
    std::vector<SReq> reqs;
    std::vector<int> rws;
    for (size_t k = 0; k < cuts.size(); ++k) {
      if (!F->mine[cuts[k]]) continue;
      FrontH &c = F->fronts[cuts[k]];
      std::vector<int> to(c.nf);
      for (int q = 0; q < c.nf; ++q) to[q] = q;
      DChild ch{};
      ch.to_child = s.push_keep(to);
      ch.n = c.nf;
      if (c.upd == 0) {
        ch.kind = 0;
        ch.dense = c.upd_dense;
        ch.ldd = c.upd_ld;
      } else {
        ch.kind = 1;
        ch.hn = F->trees[c.ff].d_nodes;
        ch.W = c.W;
        ch.Vt = c.Vt;
        ch.rw = c.rw;
        ch.ldw = c.ldw;
        ch.ldv = c.ldv;
      }
      DFront d{};
      d.ids = c.d_ids + c.npv;
      d.nh = c.nf;
      d.npv = 0;  // no seed: every entry is the child term alone
      d.child_begin = (int)dch.size();
      dch.push_back(ch);
      d.child_end = (int)dch.size();
      reqs.push_back(SReq{(int)dfr.size(), c.nf, c.nf, nullptr, nullptr, 0, 0, imp + coff[k], c.nf});
      dfr.push_back(d);
      rws.push_back(ch.kind == 1 ? ch.rw : 0);
    }
    if (!reqs.empty()) {
      DFront *dF = s.push_keep(dfr);
      DChild *dC = s.push_keep(dch);
      slot_rw = rws;
      run_sample(s, reqs, dF, dC);
    }
    F->exchange_or_throw(imp, T);
    for (size_t k = 0; k < cuts.size(); ++k) {
      FrontH &c = F->fronts[cuts[k]];
      c.upd = 0;
      c.upd_dense = imp + coff[k];
      c.upd_ld = c.nf;
    }
  }

  // ---- sharded, compressed (the p2p path): every cut child's update travels
  // from its owner to its parent's owner only, in its own form -- a dense
  // Schur block, or the reference's UpdateRep (hodlr.py:429-470): the update
  // HODLR's leaves and blocks behind an HNode table whose pointers are
  // offsets, then W and V^T. Sizes first (one small all-reduce of disjoint
  // meta slots), then one group of sends / receives; the receiver rebases the
  // table. The parent's sampler then reads the same numbers it would read on
  // one GPU: bitwise the single-GPU factorization.
  void exchange_updates_p2p(const std::vector<int> &cuts) {
    Sink s{ctx};
    const int K = (int)cuts.size();
    constexpr int MW = 6;  // kind, length, table slots, rw, offset of W, offset of V^T
    std::vector<double> meta((size_t)MW * K, 0.0);
    std::vector<double *> sbuf(K, nullptr);
    std::vector<CopyJob> cps;
    std::vector<std::vector<HNode>> tables(K);
    auto parent_post = [&](int q) { return pidx_[et->parent[F->fronts[q].node]]; };
    for (int k = 0; k < K; ++k) {
      const int q = cuts[k];
      if (!F->mine[q]) continue;
      FrontH &c = F->fronts[q];
      const int rh = release_height(c);
      double *m = meta.data() + (size_t)MW * k;
      if (c.upd == 0) {
        const int64_t len = (int64_t)c.nf * c.nf;
        sbuf[k] = upd.d(std::max<int64_t>(1, len), rh);
        cps.push_back(CopyJob{c.upd_dense, sbuf[k], c.nf, c.nf, c.upd_ld, c.nf, nullptr, nullptr});
        m[0] = 0;
        m[1] = (double)len;
        continue;
      }
      HTree &T = F->trees[c.ff];
      const int64_t tab = (int64_t)cdiv((int64_t)sizeof(HNode) * T.nslots, (int64_t)sizeof(double));
      int64_t off = tab;
      struct Pend {
        const double *src;
        int64_t at;
        int r, cl, lds;
      };
      std::vector<Pend> pend;
      auto put = [&](const double *src, int r, int cl, int lds) -> const double * {
        if (!src || (int64_t)r * cl == 0) return nullptr;
        pend.push_back(Pend{src, off, r, cl, lds});
        const int64_t at = off;
        off += (int64_t)r * cl;
        return (const double *)(uintptr_t)at;
      };
      auto blk = [&](const BlockH &b) {
        HBlk h = b.dev();
        if (b.dense) {
          h.a = put(b.val, b.m, b.n, b.n);
        } else {
          h.a = put(b.col, b.m, b.rank, b.rank);
          h.b = put(b.row, b.rank, b.n, b.n);
        }
        return h;
      };
      std::vector<HNode> &tb = tables[k];
      tb.assign(T.nslots, HNode{});
      for (int v = 0; v < T.nslots; ++v) {
        if (T.leaf[v] == 1) {
          const int sz = T.hi[v] - T.lo[v];
          tb[v].leaf = put(T.lval[v], sz, sz, sz);
        } else if (T.leaf[v] == 0) {
          tb[v].up = blk(F->blocks[T.up[v]]);
          tb[v].lw = blk(F->blocks[T.lw[v]]);
        }
      }
      const int64_t oW = off;
      put(c.W, c.nf, c.rw, c.ldw);
      const int64_t oV = off;
      put(c.Vt, c.rw, c.nf, c.ldv);
      sbuf[k] = upd.d(std::max<int64_t>(1, off), rh);
      for (auto &p : pend) cps.push_back(CopyJob{p.src, sbuf[k] + p.at, p.r, p.cl, p.lds, p.cl, nullptr, nullptr});
      s.push_to(sbuf[k], tb.data(), sizeof(HNode) * tb.size());
      m[0] = 1;
      m[1] = (double)off;
      m[2] = T.nslots;
      m[3] = c.rw;
      m[4] = (double)oW;
      m[5] = (double)oV;
    }
    run_copy(s, cps);
    // every rank learns every payload's size (disjoint slots: the sum is exact)
    double *dm = ctx->scratch.d(std::max<size_t>(1, meta.size()));
    s.push_to(dm, meta.data(), sizeof(double) * meta.size());
    F->exchange_or_throw(dm, (int64_t)meta.size());
    CK(cudaMemcpyAsync(meta.data(), dm, sizeof(double) * meta.size(), cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    std::vector<double *> bufs;
    std::vector<int64_t> counts;
    std::vector<int32_t> peers, sends;
    std::vector<std::pair<int, double *>> recv;
    for (int k = 0; k < K; ++k) {
      const int q = cuts[k], pq = parent_post(q);
      const int from = F->owner[q], to = F->owner[pq];
      const int64_t len = (int64_t)meta[(size_t)MW * k + 1];
      if (len <= 0 || from == to) continue;
      if (F->mine[q]) {
        bufs.push_back(sbuf[k]);
        counts.push_back(len);
        peers.push_back(to);
        sends.push_back(1);
        F->xchg_bytes += 8 * len;
      } else if (F->mine[pq]) {
        double *rb = upd.d(len, release_height(F->fronts[q]));
        bufs.push_back(rb);
        counts.push_back(len);
        peers.push_back(from);
        sends.push_back(0);
        recv.push_back({k, rb});
      }
    }
    if (!bufs.empty() &&
        F->p2p(F->xuser, (int64_t)bufs.size(), bufs.data(), counts.data(), peers.data(), sends.data()) != 0)
      throw runtime_error("shard point-to-point callback failed");
    for (auto &r : recv) {
      const int k = r.first;
      FrontH &c = F->fronts[cuts[k]];
      const double *m = meta.data() + (size_t)MW * k;
      if (m[0] == 0) {
        c.upd = 0;
        c.upd_dense = r.second;
        c.upd_ld = c.nf;
        continue;
      }
      const int ns = (int)m[2];
      HNode *t = (HNode *)r.second;
      k_rebase_hnodes<<<(unsigned)cdiv(ns, 128), 128, 0, ctx->s>>>(t, ns, r.second);
      check_launch();
      ctx->launches++;
      c.upd = 1;
      c.rx_nodes = t;
      c.rw = (int)m[3];
      c.W = r.second + (int64_t)m[4];
      c.ldw = c.rw;
      c.Vt = r.second + (int64_t)m[5];
      c.ldv = c.nf;
    }
  }

  // ---- sharded: the numeric accounting of fronts factored elsewhere, for the
  // whole-tree stats replay
  void exchange_accounting() {
    const size_t nf_ = F->fronts.size();
    std::vector<double> acc(4 * nf_, 0.0);
    for (size_t q = 0; q < nf_; ++q) {
      if (!F->mine[q]) continue;
      FrontH &f = F->fronts[q];
      acc[4 * q] = (double)f.front_reals;
      acc[4 * q + 1] = (double)f.factor_reals;
      acc[4 * q + 2] = (double)f.upd_reals;
      acc[4 * q + 3] = (double)f.hint;
    }
    double *d = ctx->scratch.d(std::max<size_t>(1, acc.size()));
    upload(ctx->s, d, acc.data(), sizeof(double) * acc.size());  // ordered on the library stream
    F->exchange_or_throw(d, (int64_t)acc.size());
    CK(cudaStreamSynchronize(ctx->s));
    CK(cudaMemcpy(acc.data(), d, sizeof(double) * acc.size(), cudaMemcpyDeviceToHost));
    ctx->scratch.reset();
    for (size_t q = 0; q < nf_; ++q) {
      if (F->mine[q]) continue;
      FrontH &f = F->fronts[q];
      f.front_reals = (int64_t)acc[4 * q];
      f.factor_reals = (int64_t)acc[4 * q + 1];
      f.upd_reals = (int64_t)acc[4 * q + 2];
      f.hint = (int64_t)acc[4 * q + 3];
    }
  }

  // where the device memory of a factorization goes (MFH_MEM_TRACE=1): the
  // retained arena by category, from the host-side metadata
  void memory_breakdown() {
    // retained (arena) categories, then the transient ones (release arena / scratch)
    double cat[7] = {0}, tr[3] = {0};
    const char *names[7] = {"dense Pinv/Gpf/Gfp", "dense Fpp", "pf/fp blocks", "pp inverse (Hinv|form)",
                            "Xp/RH", "other", ""};
    auto tree_bytes = [&](int tt) {
      double s2 = 0;
      if (tt < 0) return s2;
      HTree &T = F->trees[tt];
      for (int v = 0; v < T.nslots; ++v) {
        if (T.leaf[v] == 1) {
          double sz = T.hi[v] - T.lo[v];
          s2 += 8 * sz * sz;
        } else if (T.leaf[v] == 0) {
          s2 += 8.0 * (F->blocks[T.up[v]].stored() + F->blocks[T.lw[v]].stored());
        }
      }
      return s2;
    };
    int n_form = 0, n_struct = 0;
    for (auto &f : F->fronts) {
      if (f.nh == 0) continue;
      if (!f.structured) {
        cat[0] += 8.0 * ((double)f.npv * f.npv + 2.0 * f.npv * f.nf);
        if (f.Fpp) cat[1] += 8.0 * f.npv * f.npv;
        continue;
      }
      n_struct++;
      tr[0] += tree_bytes(f.pp);
      tr[1] += tree_bytes(f.ff);
      if (f.W && f.W != as_factors(F->blocks[f.fp]).col) tr[2] += 8.0 * f.nf * f.rw;
      if (f.Vt && f.Vt != as_factors(F->blocks[f.pf]).row) tr[2] += 8.0 * f.nf * f.rw;
      if (f.pf >= 0) cat[2] += 8.0 * (F->blocks[f.pf].stored() + F->blocks[f.fp].stored());
      if (!f.pform) {
        cat[3] += 8.0 * f.npv * f.npv;
      } else {
        n_form++;
        for (auto &L : f.tleaf) cat[3] += 8.0 * L.sz * (L.sz + L.K);
        for (auto &t : f.tnode) cat[3] += 8.0 * (t.r1 + t.r2) * t.nv;
      }
      if (f.pf >= 0) {
        const BlockH &bpf = F->blocks[f.pf], &bfp = F->blocks[f.fp];
        cat[4] += 8.0 * f.npv * ((bpf.dense ? 0 : bpf.rank) + (bfp.dense ? 0 : bfp.rank));
      }
    }
    double known = 0;
    for (int q = 0; q < 5; ++q) known += cat[q];
    cat[5] = (double)F->arena.capacity() - known;
    fprintf(stderr, "[mfh mem] arena %.2f GB (peak in use %.2f GB), release arena peak %.2f GB, scratch %.2f GB; "
            "%d of %d structured fronts in HODLR inverse form\n",
            F->arena.capacity() / 1e9, F->arena.peak / 1e9, upd.peak / 1e9, ctx->scratch.capacity() / 1e9, n_form,
            n_struct);
    for (int q = 0; q < 6; ++q) fprintf(stderr, "[mfh mem]   retained %-24s %8.3f GB\n", names[q], cat[q] / 1e9);
    fprintf(stderr, "[mfh mem]   transient pp trees %.3f GB, update trees %.3f GB, W/Vt %.3f GB\n", tr[0] / 1e9,
            tr[1] / 1e9, tr[2] / 1e9);
  }

  void run(const CsrView &A, int mode) {
    auto t0 = std::chrono::steady_clock::now();
    const bool trace = getenv("MFH_HOST_TRACE") != nullptr;
    auto tprev = t0;
    auto mark_t = [&](const char *what) {
      if (!trace) return;
      auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[mfh host] %-20s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - tprev).count());
      tprev = now;
    };
    n = A.n;
    accel = mode == MFH_ACCELERATED;
    F->n = n;
    F->et_uid = et->uid;
    F->perm = et->perm;
    F->mode = mode;
    F->params = P;
    // ---- P A P^T as CSR (multifrontal.py:245-250). The pattern part (two
    // counting-sort transposes, O(nnz)) and the BDLR graph are symbolic: they
    // are cached on the elimination tree, keyed by (pattern, zero pattern);
    // every factorization gathers the values.
    {
      const std::vector<int64_t> &perm = et->perm;
      const int64_t nnz = A.ptr[n];
      mfh_symcache &C = et->cache;
      // the cached symbolic data is valid for exactly this pattern and zero pattern
      // (the scan for explicit zeros and the pattern comparison read ~16 bytes per entry:
      // on several host threads above 1M entries; 19 ms on one thread at C4's 7M)
      std::vector<int64_t> zeros;
      {
        std::vector<int64_t> zl[8];
        par_chunks(nnz, 1 << 20, [&](int64_t b, int64_t e, int t) {
          for (int64_t p2 = b; p2 < e; ++p2)
            if (A.val[p2] == 0.0) zl[t].push_back(p2);
        });
        for (auto &z : zl) zeros.insert(zeros.end(), z.begin(), z.end());
      }
      bool same = C.valid && C.pat_accel == accel && (int64_t)C.pat_ptr.size() == n + 1 &&
                  (int64_t)C.pat_idx.size() == nnz &&
                  std::memcmp(C.pat_ptr.data(), A.ptr, sizeof(int64_t) * (n + 1)) == 0 && C.pat_zero == zeros;
      if (same) {
        std::atomic<int> diff{0};
        const int64_t *cached = C.pat_idx.data(), *given = A.idx;
        par_chunks(nnz, 1 << 20, [&](int64_t b, int64_t e, int) {
          if (e > b && std::memcmp(cached + b, given + b, sizeof(int64_t) * (size_t)(e - b)) != 0) diff.store(1);
        });
        same = diff.load() == 0;
      }
      if (!same) {
        C = mfh_symcache{};
        C.pat_ptr.assign(A.ptr, A.ptr + n + 1);
        C.pat_idx.assign(A.idx, A.idx + nnz);
        C.pat_zero = zeros;
        C.pat_accel = accel;
        static std::atomic<uint64_t> next_gen{1};
        C.gen = next_gen++;
        std::vector<int64_t> iperm(n);
        for (int64_t i = 0; i < n; ++i) iperm[perm[i]] = i;
        // T = (P A P^T)^T: row = new column, entries in increasing new row
        std::vector<int64_t> tptr(n + 1, 0);
        for (int64_t p2 = 0; p2 < nnz; ++p2) tptr[perm[A.idx[p2]] + 1]++;
        for (int64_t i = 0; i < n; ++i) tptr[i + 1] += tptr[i];
        std::vector<int> tcol(nnz);
        std::vector<int64_t> tsrc(nnz);
        {
          std::vector<int64_t> fill(tptr.begin(), tptr.end() - 1);
          for (int64_t pi = 0; pi < n; ++pi) {
            int64_t i = iperm[pi];
            for (int64_t p2 = A.ptr[i]; p2 < A.ptr[i + 1]; ++p2) {
              int64_t q = fill[perm[A.idx[p2]]]++;
              tcol[q] = (int)pi;
              tsrc[q] = p2;
            }
          }
        }
        C.ap_ptr.assign(n + 1, 0);
        for (int64_t pi = 0; pi < n; ++pi) C.ap_ptr[pi + 1] = C.ap_ptr[pi] + (A.ptr[iperm[pi] + 1] - A.ptr[iperm[pi]]);
        C.ap_col.resize(nnz);
        C.src.resize(nnz);
        {
          std::vector<int64_t> fill(C.ap_ptr.begin(), C.ap_ptr.end() - 1);
          for (int64_t pj = 0; pj < n; ++pj)
            for (int64_t q = tptr[pj]; q < tptr[pj + 1]; ++q) {
              int64_t r = fill[tcol[q]]++;
              C.ap_col[r] = (int)pj;
              C.src[r] = tsrc[q];
            }
        }
        if (accel) {
          // BDLR graph (sparse.py:102-111 on Ap): row i = {j != i : Ap[i][j] != 0 or Ap[j][i] != 0}
          Graph &g = C.graph;
          g.n = n;
          g.ptr.assign(n + 1, 0);
          g.idx.reserve(2 * nnz);
          for (int64_t i = 0; i < n; ++i) {
            int64_t p2 = C.ap_ptr[i], pe = C.ap_ptr[i + 1], q = tptr[i], qe = tptr[i + 1];
            int64_t last = -1;
            while (p2 < pe || q < qe) {
              int64_t j;
              bool nz;
              if (q >= qe || (p2 < pe && C.ap_col[p2] <= tcol[q])) {
                j = C.ap_col[p2];
                nz = A.val[C.src[p2]] != 0.0;
                ++p2;
              } else {
                j = tcol[q];
                nz = A.val[tsrc[q]] != 0.0;
                ++q;
              }
              if (!nz || j == i || j == last) continue;
              g.idx.push_back(j);
              last = j;
            }
            g.ptr[i + 1] = (int64_t)g.idx.size();
          }
          C.has_graph = true;
        }
        C.valid = true;
      }
      if (accel) gp = &C.graph;
      // permuted pattern + value-gather map: on the device once per (context, pattern)
      Ctx::PatDev *pd = nullptr;
      for (auto &q : ctx->pat_dev)
        if (q.gen == C.gen) pd = &q;
      if (!pd) {
        if (ctx->pat_dev.size() >= Ctx::SYM_CACHE_MAX) {
          cudaFree(ctx->pat_dev.front().ptr);
          cudaFree(ctx->pat_dev.front().col);
          cudaFree(ctx->pat_dev.front().src);
          ctx->pat_dev.erase(ctx->pat_dev.begin());
        }
        Ctx::PatDev q;
        q.gen = C.gen;
        CK(cudaMalloc(&q.ptr, sizeof(int64_t) * (n + 1)));
        CK(cudaMalloc(&q.col, sizeof(int) * std::max<int64_t>(1, nnz)));
        CK(cudaMalloc(&q.src, sizeof(int64_t) * std::max<int64_t>(1, nnz)));
        upload(ctx->s, q.ptr, C.ap_ptr.data(), sizeof(int64_t) * (n + 1));
        if (nnz) {
          upload(ctx->s, q.col, C.ap_col.data(), sizeof(int) * nnz);
          upload(ctx->s, q.src, C.src.data(), sizeof(int64_t) * nnz);
        }
        ctx->pat_dev.push_back(q);
        pd = &ctx->pat_dev.back();
      }
      d_ap_ptr = pd->ptr;
      d_ap_col = pd->col;
      d_ap_val = F->arena.d(std::max<int64_t>(1, nnz));
      if (nnz) {
        // raw values staged asynchronously, gathered into P A P^T order on the device
        double *raw = F->arena.d(nnz);
        Sink up{ctx};
        {
          // into the pinned staging ring on several host threads, then one async H2D copy
          auto hd = ctx->stage.take(sizeof(double) * nnz);
          char *dsth = (char *)hd.first;
          const char *srch = (const char *)A.val;
          par_chunks(nnz, 1 << 20, [&](int64_t b, int64_t e, int) {
            std::memcpy(dsth + sizeof(double) * b, srch + sizeof(double) * b, sizeof(double) * (size_t)(e - b));
          });
          up.h2d(raw, hd.first, sizeof(double) * nnz);
        }
        const long long *srcp = pd->src;
        double *dst = d_ap_val;
        int g = (int)std::min<int64_t>(cdiv(nnz, 256), 148 * 8);
        k_gather_idx<<<g, 256, 0, ctx->s>>>(srcp, raw, dst, nnz);
        check_launch();
        ctx->launches++;
      }
    }
    mark_t("permute+graph");
    // ---- fronts in post order
    int64_t nn = (int64_t)et->parent.size();
    std::vector<int> &pidx = pidx_;
    pidx.assign(nn, -1);
    upd.pool = &ctx->pool;
    F->post = et->post;
    {  // front id lists (symbolic): flattened once per tree
      mfh_mapcache &M = et->mapcache;
      if (!M.ids_valid) {
        M.ids_flat.clear();
        M.ids_off.assign(et->post.size(), 0);
        for (size_t q = 0; q < et->post.size(); ++q) {
          int64_t p = et->post[q];
          M.ids_off[q] = (int64_t)M.ids_flat.size();
          M.ids_flat.insert(M.ids_flat.end(), et->piv.begin() + et->piv_ptr[p], et->piv.begin() + et->piv_ptr[p + 1]);
          M.ids_flat.insert(M.ids_flat.end(), et->fr.begin() + et->fr_ptr[p], et->fr.begin() + et->fr_ptr[p + 1]);
        }
        M.ids_valid = true;
      }
    }
    F->fronts.resize(et->post.size());
    F->front_blocks.assign(et->post.size(), {});
    double thr = accel ? (double)P.n_c : INFINITY;
    int maxh = 0;
    int64_t max_nh = 1;
    bool any_struct = false;
    for (size_t q = 0; q < et->post.size(); ++q) {
      int64_t p = et->post[q];
      pidx[p] = (int)q;
      FrontH &f = F->fronts[q];
      f.node = p;
      int64_t pb = et->piv_ptr[p], pe = et->piv_ptr[p + 1], fb = et->fr_ptr[p], fe = et->fr_ptr[p + 1];
      f.npv = (int)(pe - pb);
      f.nf = (int)(fe - fb);
      f.nh = f.npv + f.nf;
      f.ids = IdsView{et->mapcache.ids_flat.data() + et->mapcache.ids_off[q], (size_t)f.nh};
      f.piv_lo = f.npv ? f.ids[0] : 0;
      for (int q2 = 1; q2 < f.npv; ++q2)
        if (f.ids[q2] != f.ids[q2 - 1] + 1) throw runtime_error("pivot ids are not a contiguous run");
      int h = 0;
      for (int64_t c : et->children[p]) {
        int ci = pidx[c];
        f.allkids.push_back(ci);
        h = std::max(h, F->fronts[ci].height + 1);
        FrontH &cf = F->fronts[ci];
        if (cf.nh > 0 && cf.nf > 0) {
          f.kids.push_back(ci);
        }
      }
      f.height = h;
      maxh = std::max(maxh, h);
      f.structured = f.nh > 0 && (double)f.nh >= thr;
      any_struct |= f.structured;
      max_nh = std::max<int64_t>(max_nh, f.nh);
    }
    mark_t("fronts");
    if (shard) {
      F->sharded = true;
      F->rank = shard->rank;
      F->exchange = shard->exchange;
      F->p2p = shard->p2p;
      F->xuser = shard->user;
      if (!shard->owner || !shard->exchange) throw value_error("shard needs an owner array and an exchange callback");
      F->owner.assign(F->fronts.size(), 0);
      F->mine.assign(F->fronts.size(), 0);
      int world = 1;
      for (size_t q = 0; q < F->fronts.size(); ++q) {
        int o = shard->owner[F->fronts[q].node];
        if (o < 0) throw value_error("shard owner ranks must be non-negative");
        F->owner[q] = o;
        F->mine[q] = o == shard->rank;
        world = std::max(world, o + 1);
      }
      F->world = std::max(world, shard->rank + 1);
    }
    auto active = [&](size_t q) { return !F->sharded || F->mine[q] != 0; };
    ensure_maps();
    mark_t("maps");
    if (any_struct) {
      if (!(P.eps > 0.0 && P.eps < 1.0)) throw value_error("eps must lie in (0, 1)");
      if (P.n_leaf < 1) throw value_error("n_leaf must be positive");
      if (P.d < 1) throw value_error("distance must be at least 1");
      // identity for DenseBlock.as_factors: a strip of 2 max_nh - 1 doubles with
      // the one in the middle, read with leading dimension -1 (element (i, j) at
      // center + j - i), instead of a max_nh^2 matrix (3 GB at C5). GEMMs with
      // it become scaled copies (run_gemm); the GEMV kernels index with signed
      // 64-bit arithmetic and read it directly.
      double *strip = F->arena.d((size_t)2 * max_nh - 1);
      CK(cudaMemsetAsync(strip, 0, sizeof(double) * (2 * max_nh - 1), ctx->s));
      static const double one = 1.0;
      CK(cudaMemcpyAsync(strip + (max_nh - 1), &one, sizeof(double), cudaMemcpyHostToDevice, ctx->s));
      F->ident_ld = -1;
      F->ident = strip + (max_nh - 1);
    }
    F->d_perm = (long long *)F->arena.alloc(sizeof(int64_t) * std::max<int64_t>(1, n));
    upload(ctx->s, F->d_perm, et->perm.data(), sizeof(int64_t) * n);
    // device ids + flags
    {  // all front id lists: symbolic, on the device once per (context, tree)
      long long *all = nullptr;
      for (auto &m : ctx->ids_dev)
        if (m.first == et->uid) all = m.second;
      int64_t tot = 0;
      if (!all) {
        if (ctx->ids_dev.size() >= Ctx::SYM_CACHE_MAX) {
          cudaFree(ctx->ids_dev.front().second);
          ctx->ids_dev.erase(ctx->ids_dev.begin());
        }
        for (auto &f : F->fronts) tot += f.nh;
        const std::vector<int64_t> &flat = et->mapcache.ids_flat;
        CK(cudaMalloc(&all, sizeof(int64_t) * std::max<int64_t>(1, tot)));
        upload(ctx->s, all, flat.data(), sizeof(int64_t) * tot);
        ctx->ids_dev.push_back({et->uid, all});
      }
      int64_t o = 0;
      for (auto &f : F->fronts) {
        f.d_ids = f.nh ? all + o : nullptr;
        o += f.nh;
      }
    }
    mark_t("identity+uploads");
    int max_flags = 0;
    for (auto &f : F->fronts) max_flags += 1 + (f.structured ? 8 * (int)(f.nh / std::max<int64_t>(1, P.n_leaf) + 2) : 0);
    flag_cap = max_flags + 16;
    d_flags = F->arena.i(max_flags + 16);
    CK(cudaMemset(d_flags, 0, sizeof(int) * (max_flags + 16)));
    // Dense merge nodes (no pivots) with one updating child over the same
    // frontal ids: the front is 0 + the child's update, i.e. that update bit
    // for bit, so it aliases the child's buffer instead of being assembled
    // (the long single-child merge chains of nested dissection).
    alias_.assign(F->fronts.size(), 0);
    std::vector<std::vector<int>> alias_at(maxh + 1);
    if (!F->sharded)
      for (size_t q = 0; q < F->fronts.size(); ++q) {
        FrontH &f = F->fronts[q];
        if (f.structured || f.nh == 0 || f.npv != 0 || f.kids.size() != 1) continue;
        FrontH &c = F->fronts[f.kids[0]];
        if (c.structured || c.nf != f.nf) continue;
        bool same = true;
        for (int j = 0; j < f.nf && same; ++j) same = c.ids[c.npv + j] == f.ids[j];
        if (!same) continue;
        alias_[q] = 1;
        alias_at[f.height].push_back((int)q);
      }
    // ---- heights
    std::vector<std::vector<int>> byh(maxh + 1);
    for (size_t q = 0; q < F->fronts.size(); ++q)
      if (F->fronts[q].nh > 0 && active(q) && !alias_[q]) byh[F->fronts[q].height].push_back((int)q);
    // sharded: heights after which a child -> parent update crosses ranks (the
    // same on every rank: computed from the global tree)
    std::vector<std::vector<int>> cut_at(maxh + 1);
    if (F->sharded)
      for (size_t q = 0; q < F->fronts.size(); ++q) {
        FrontH &f = F->fronts[q];
        int64_t par = et->parent[f.node];
        if (par < 0 || f.nh == 0 || f.nf == 0) continue;
        if (F->owner[pidx[par]] != F->owner[q]) cut_at[f.height].push_back((int)q);
      }
    // structured-front plans (trees, blocks, BDLR selections) are symbolic: a
    // planner thread computes them, in processing order, while the GPU works
    {
      int ntrees = 0, nblocks = 0;
      plan_pos.assign(F->fronts.size(), -1);
      for (int h = 0; h <= maxh; ++h)
        for (int fi : byh[h]) {
          FrontH &f = F->fronts[fi];
          if (!f.structured) continue;
          f.tree_base = ntrees;
          ntrees += 2;
          f.block_base = nblocks;
          if (f.npv) nblocks += 2 * count_internal(f.npv, P.n_leaf);
          if (f.npv && f.nf) nblocks += 2;
          if (f.nf) nblocks += 2 * count_internal(f.nf, P.n_leaf);
          plan_pos[fi] = (int)plan_order.size();
          plan_order.push_back(fi);
        }
      F->trees.assign(ntrees, HTree{});
      F->blocks.assign(nblocks, BlockH{});
      if (!plan_order.empty()) start_planner();
    }
    mark_t("flags+plan");
    double tsum[7] = {0, 0, 0, 0, 0, 0, 0};
    auto host_done = std::chrono::steady_clock::now();
    F->timing.host_ms += std::chrono::duration<double, std::milli>(host_done - t0).count();
    F->timing.host_preamble_ms = std::chrono::duration<double, std::milli>(host_done - t0).count();
    cudaEvent_t e_begin, e_end;
    CK(cudaEventCreate(&e_begin));
    CK(cudaEventCreate(&e_end));
    CK(cudaEventRecord(e_begin, ctx->s));
    // Heights are enqueued back to back: the host only waits where it needs
    // device data (the rank readback inside structured heights) or to recycle
    // scratch memory; per-height phase events are evaluated at the end.
    int used = 0;
    std::vector<int> height_of_use, struct_of_use;
    std::vector<std::array<int, 4>> first_of_use;  // npv, nf, kids of the first front; aliased fronts
    std::vector<double> host_us_of_use, decide_us_of_use;
    for (int h = 0; h <= maxh; ++h) {
      for (int q : alias_at[h]) {  // the child was enqueued at a lower height
        FrontH &f = F->fronts[q];
        const FrontH &c = F->fronts[f.kids[0]];
        f.upd = 0;
        f.upd_dense = c.upd_dense;
        f.upd_ld = c.upd_ld;
        f.front_reals = (int64_t)f.nh * f.nh;
        f.factor_reals = 0;
        f.upd_reals = (int64_t)f.nf * f.nf;
      }
      if (byh[h].empty()) {
        if (!cut_at[h].empty()) (F->p2p ? exchange_updates_p2p(cut_at[h]) : exchange_updates(cut_at[h]));
        upd.release_upto(h);
        continue;
      }
      while ((int)ctx->evpool.size() < 8 * (used + 1)) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ctx->evpool.push_back(e);
      }
      cudaEvent_t *ev = ctx->evpool.data() + 8 * used;
      while ((int)ctx->evd_pool.size() < used + 1) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        ctx->evd_pool.push_back(e);
      }
      cur_evd = ctx->evd_pool[used];
      ++used;
      height_of_use.push_back(h);
      {
        int ns = 0;
        for (int fi : byh[h]) ns += F->fronts[fi].structured;
        struct_of_use.push_back(ns);
        const FrontH &f0 = F->fronts[byh[h][0]];
        first_of_use.push_back({f0.npv, f0.nf, (int)f0.kids.size(), (int)alias_at[h].size()});
      }
      // process_height records ev[0..2] (dense-only heights) or ev[0..7]
      auto th0 = std::chrono::steady_clock::now();
      last_decide_us = 0.0;
      process_height(byh[h], ev);
      host_us_of_use.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count());
      decide_us_of_use.push_back(last_decide_us);
      // heights run ahead of the host: the only waits are the rank readback
      // inside structured heights and scratch recycling
      if (ctx->scratch.in_use > (size_t(4) << 30)) {
        Sink s{ctx};
        auto tw = std::chrono::steady_clock::now();
        s.sync_reset();
        F->timing.host_sync_wait_ms +=
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw).count();
        check_flags(0);
        ctx->scratch.reset();
      }
      if (!cut_at[h].empty()) (F->p2p ? exchange_updates_p2p(cut_at[h]) : exchange_updates(cut_at[h]));
      upd.release_upto(h);  // dense front buffers whose parents have sampled them
    }
    CK(cudaEventRecord(e_end, ctx->s));
    // the apply plan (host work) is built while the GPU finishes the last heights
    build_apply(F);
    {
      auto tw = std::chrono::steady_clock::now();
      CK(cudaStreamSynchronize(ctx->s));
      F->timing.host_sync_wait_ms +=
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw).count();
    }
    ctx->stage.rewind();
    check_flags(0);
    ctx->scratch.reset();
    const bool htrace = getenv("MFH_HEIGHT_TRACE") != nullptr;
    if (htrace) {
      fprintf(stderr, "[mfh blas] %lld cuBLAS DGEMM calls, %.1f ms host time in them (cumulative)\n",
              (long long)g_blas_calls, g_blas_host_ms);
    }
    OpClock::dump();
    for (int u = 0; u < used; ++u) {
      cudaEvent_t *ev = ctx->evpool.data() + 8 * u;
      const bool donly = struct_of_use[u] == 0;
      if (htrace) {
        float a[7] = {0, 0, 0, 0, 0, 0, 0}, gap = 0.f;
        for (int q = 0; q < (donly ? 2 : 7); ++q) CK(cudaEventElapsedTime(&a[q], ev[q], ev[q + 1]));
        float dens = 0.f;
        if (u > 0) {
          CK(cudaEventElapsedTime(&gap, ctx->evpool[8 * (u - 1) + (struct_of_use[u - 1] ? 7 : 2)], ev[0]));
          CK(cudaEventElapsedTime(&dens, ctx->evpool[8 * (u - 1) + (struct_of_use[u - 1] ? 7 : 2)], ctx->evd_pool[u]));
        }
        fprintf(stderr, "[mfh height %3d] materialize %7.3f of the gap\n", height_of_use[u], dens);
        fprintf(stderr, "[mfh height %3d] fronts %4zu struct %2d | gap %7.3f sample %7.3f dense %7.3f plu %7.3f - %7.3f skel %7.3f hodlr %7.3f elim %7.3f ms | first npv %d nf %d kids %d, aliased %d | host %.1f us, decide %.1f us\n",
                height_of_use[u], byh[height_of_use[u]].size(), struct_of_use[u], gap, a[0], a[1], a[2], a[3], a[4], a[5], a[6],
                first_of_use[u][0], first_of_use[u][1], first_of_use[u][2], first_of_use[u][3], host_us_of_use[u],
                decide_us_of_use[u]);
      }
      float ms;
      if (u > 0) {
        cudaEvent_t prev = ctx->evpool[8 * (u - 1) + (struct_of_use[u - 1] ? 7 : 2)];
        float g = 0.f, m2 = 0.f;
        CK(cudaEventElapsedTime(&g, prev, ev[0]));
        CK(cudaEventElapsedTime(&m2, prev, ctx->evd_pool[u]));
        F->timing.materialize_ms += m2;
        F->timing.idle_gap_ms += g - m2;
      }
      CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      tsum[0] += ms;
      CK(cudaEventElapsedTime(&ms, ev[1], ev[2]));
      tsum[4] += ms;
      if (donly) continue;
      CK(cudaEventElapsedTime(&ms, ev[2], ev[3]));
      tsum[1] += ms;
      CK(cudaEventElapsedTime(&ms, ev[4], ev[5]));
      tsum[2] += ms;
      CK(cudaEventElapsedTime(&ms, ev[5], ev[6]));
      tsum[3] += ms;
      CK(cudaEventElapsedTime(&ms, ev[6], ev[7]));
      tsum[5] += ms;
    }
    float tot;
    CK(cudaEventElapsedTime(&tot, e_begin, e_end));
    cudaEventDestroy(e_begin);
    cudaEventDestroy(e_end);
    F->timing.sample_ms = tsum[0];
    F->timing.dense_front_ms = tsum[4];
    F->timing.pivot_lu_ms = tsum[1];
    F->timing.skeleton_ms = tsum[2];
    F->timing.hodlr_factor_ms = tsum[3];
    F->timing.eliminate_ms = tsum[5];
    if (F->sharded) exchange_accounting();
    // ---- stats replay in post order (multifrontal.py:76-86, 478-529)
    int64_t retained = 0, live = 0, peak = 0;
    F->records.clear();
    for (size_t q = 0; q < F->fronts.size(); ++q) {
      FrontH &f = F->fronts[q];
      int64_t freed = 0;
      for (int64_t c : et->children[f.node]) {
        FrontH &cf = F->fronts[pidx[c]];
        if (cf.nh > 0 && cf.nf > 0) freed += cf.upd_reals;
      }
      mfh_record_t r{};
      r.node_id = f.node;
      if (f.nh == 0) {
        r.path = 0;
      } else {
        peak = std::max(peak, retained + live + f.front_reals);  // note_front
        r.front_size = f.nh;
        r.n_pivot = f.npv;
        r.path = f.structured ? 2 : 1;
        r.max_offdiag_rank = f.structured ? f.hint : 0;
        r.stored_reals = f.factor_reals;
        if (f.structured)
          F->stats.structured_fronts++;
        else
          F->stats.dense_fronts++;
      }
      int64_t newr = (f.nh > 0 && f.nf > 0) ? f.upd_reals : 0;
      retained += r.stored_reals;
      live += newr - freed;
      peak = std::max(peak, retained + live);
      F->records.push_back(r);
    }
    F->stats.peak_stored_reals = peak;
    F->stats.retained_reals = retained;
    F->stats.n_records = (int64_t)F->records.size();
    F->stats.stored_reals = retained;
    F->stats.device_bytes_peak =
        (int64_t)F->arena.capacity() + (int64_t)upd.peak + (int64_t)ctx->scratch.capacity();
    if (getenv("MFH_MEM_TRACE")) memory_breakdown();
    if (getenv("MFH_HOST_TRACE"))
      fprintf(stderr, "[mfh host] height prologues: descriptors + materialization enqueue %.1f ms, dense / leaf requests + planner wait %.1f ms, block loop %.1f ms\n",
              host_sec[0], host_sec[1], F->timing.host_select_ms);
    if (getenv("MFH_HOST_TRACE")) {
      fprintf(stderr, "[mfh host] staged host-to-device copies: %lld (%lld outside batched stretches)\n",
              (long long)ctx->h2d_copies, (long long)ctx->h2d_single);
      ctx->h2d_copies = ctx->h2d_single = 0;
    }
    if (getenv("MFH_POOL_TRACE")) {
      ChunkPool &cp = ctx->pool;
      fprintf(stderr, "[mfh pool] misses %lld (%.2f GB, %.1f ms in cudaMalloc), out-of-memory retries %lld, free chunks %zu\n",
              (long long)cp.miss_calls, cp.miss_bytes / 1e9, cp.miss_ms, (long long)cp.retry_calls, cp.free_chunks.size());
      cp.miss_calls = cp.retry_calls = 0;
      cp.miss_bytes = cp.miss_ms = 0.0;
    }
    // id views point into the tree's cache; nothing after the factorization
    // (the apply plan is already built) may read them
    for (auto &f : F->fronts) f.ids = IdsView{};
    F->timing.total_ms = tot;
    F->timing.apply_ref_bytes += 32.0 * n;
    F->timing.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

// ---------------------------------------------------------------------------
// preconditioner apply plan (mf_solve, multifrontal.py:533-560), recorded once
// and replayed as a CUDA graph
// ---------------------------------------------------------------------------
struct ApplyPlan {
  double *d_b = nullptr, *d_x = nullptr;  // user-facing input / output
  double *bu = nullptr, *xw = nullptr, *y = nullptr, *cbuf = nullptr, *xf = nullptr;
  double *yb = nullptr;  // structured fronts: y_piv = H^{-1} b_piv from the upward pass, reused downward
  double *ub = nullptr;  // dense-fallback F_pf: u_piv = b_piv - F_pf x_fro before its H^{-1}
  double *wb = nullptr;  // HODLR inverse form: w_v = Tm_v b_v of every node
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  // sharded: segment k + 1 runs after exchange k (buffer, count); the first
  // segment is (graph, exec)
  std::vector<cudaGraph_t> seg_graph;
  std::vector<cudaGraphExec_t> seg_exec;
  std::vector<int64_t> seg_nodes;
  std::vector<std::pair<double *, int64_t>> xchg;
  double bytes = 0;  // algorithmic bytes per apply
  int64_t nodes = 0;
  std::shared_ptr<Ctx::ApplySym> sym;  // contribution CSR the graph reads
  std::vector<std::function<void(cudaStream_t)>> ops;  // the captured ops (MFH_APPLY_OPS profile)
  int nv = 1;                                          // right-hand sides per replay
  ~ApplyPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (auto e : seg_exec) cudaGraphExecDestroy(e);
    for (auto g : seg_graph) cudaGraphDestroy(g);
  }
};

// DenseBlock.as_factors / LowRankFactor.as_factors (hodlr.py:59-63) as a device view
static FacView fac_view(const mfh_factor *F, const BlockH &b) {
  FacView v;
  if (!b.dense) {
    v.col = b.col;
    v.ldc = b.rank;
    v.row = b.row;
    v.ldr = b.n;
    v.rank = b.rank;
  } else if (b.n <= b.m) {
    v.col = b.val;
    v.ldc = b.n;
    v.row = F->ident;
    v.ldr = F->ident_ld;
    v.rank = b.n;
  } else {
    v.col = F->ident;
    v.ldc = F->ident_ld;
    v.row = b.val;
    v.ldr = b.n;
    v.rank = b.m;
  }
  return v;
}

// One MGS sweep (k_mgs_reg<R> when the grid's slices fit R registers per
// thread, else k_mgs_coop). The plan is a function of n and the device only,
// so every solve of the same n sums in the same order (batched columns stay
// bitwise the one-vector solves).
struct MgsPlan {
  const void *fn = nullptr;
  int grid = 1;
  size_t smem = 0;
};
static MgsPlan mgs_plan(int device, long long n) {
  static std::mutex mu;
  static std::map<std::pair<int, long long>, MgsPlan> memo;
  std::lock_guard<std::mutex> lk(mu);
  auto it = memo.find({device, n});
  if (it != memo.end()) return it->second;
  int nsm = 148;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  const void *fr[6] = {(const void *)k_mgs_reg<1>, (const void *)k_mgs_reg<2>, (const void *)k_mgs_reg<4>,
                       (const void *)k_mgs_reg<8>, (const void *)k_mgs_reg<16>, (const void *)k_mgs_reg<32>};
  MgsPlan p;
  for (int q = 0; q < 6 && !p.fn; ++q) {
    const int R = 1 << q;
    const size_t sm = sizeof(double) * 256 * R;
    if (sm > 48 * 1024) CK(cudaFuncSetAttribute(fr[q], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fr[q], 256, sm));
    if (per_sm < 1) continue;
    int grid = std::min(std::min(per_sm, 4) * nsm, MGS_MAX_GRID);
    grid = (int)std::min<long long>(grid, std::max<long long>(1, cdiv(n, 256)));
    if (cdiv(cdiv(n, grid), 256) <= R) {
      p.fn = fr[q];
      p.grid = grid;
      p.smem = sm;
    }
  }
  if (!p.fn) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mgs_coop, 256, 0));
    p.fn = (const void *)k_mgs_coop;
    p.grid = std::max(1, std::min(std::min(per_sm, 2) * nsm, MGS_MAX_GRID));
    p.grid = (int)std::min<long long>(p.grid, std::max<long long>(1, cdiv(n, 256)));
  }
  memo[{device, n}] = p;
  return p;
}
static void launch_mgs(const MgsPlan &p, const double *V, double *w, long long n, int j, double *H, double *part,
                       cudaStream_t st) {
  void *args[6] = {(void *)&V, (void *)&w, (void *)&n, (void *)&j, (void *)&H, (void *)&part};
  CK(cudaLaunchCooperativeKernel(p.fn, dim3(p.grid), dim3(256), args, p.smem, st));
}

// rows of a GEMV job in the subtree kernel's numbering: whole groups of 8
static inline int gv_rows(int m) { return (std::max(0, m) + 7) & ~7; }
static inline int gv_ws_host(int k) { return k <= 256 ? 1 : std::min(8, (k + 255) >> 8); }
template <int NV>
static void launch_gemv_tc(cudaStream_t st, int grid, const GemvJob *dj, const GvItem *di) {
  launch_pdl(k_gemv_tc<NV>, dim3(grid), dim3(256), 0, st, dj, di);
}
// nv right-hand sides (1..8): vector v of a job at pointer + v * its stride.
// Several: one CTA per (job, 8 / ws row groups), ws = the job's K segments
// (k_gemv_tc, FP64 tensor cores).
// One right-hand side: k_gemv2, a warp per row (lane-strided chains), one
// wave of warps each taking a contiguous chunk of rows.
static void run_gemv1(Sink &sk, const std::vector<GemvJob> &jobs) {
  std::vector<int> start(jobs.size() + 1, 0);
  for (size_t q = 0; q < jobs.size(); ++q) start[q + 1] = start[q] + std::max(0, jobs[q].m);
  const int nr = start.back();
  if (nr == 0) return;
  static int occ = 0;
  if (!occ) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)k_gemv2, 256, 0));
    occ = std::max(occ, 1);
  }
  const int grid = (int)std::min<int64_t>(cdiv((int64_t)nr * 32, 256), (int64_t)148 * occ);
  const int chunk = (int)cdiv(nr, grid * 8);
  std::vector<int> wq;
  wq.reserve(cdiv(nr, chunk));
  for (int t0 = 0, q = 0; t0 < nr; t0 += chunk) {
    while (start[q + 1] <= t0) ++q;
    wq.push_back(q);
  }
  GemvJob *dj = sk.push(jobs);
  int *ds = sk.push(start);
  int *dw = sk.push(wq);
  sk.launch([=](cudaStream_t st) {
    launch_pdl(k_gemv2, dim3(grid), dim3(256), 0, st, dj, ds, dw, chunk, nr);
    check_launch();
  });
}
static void run_gemv(Sink &sk, const std::vector<GemvJob> &jobs, int nv = 1) {
  if (jobs.empty()) return;
  if (nv < 1 || nv > 8) throw runtime_error("run_gemv: 1..8 right-hand sides per launch");
  if (nv == 1) {
    run_gemv1(sk, jobs);
    return;
  }
  std::vector<GvItem> items;
  for (size_t q = 0; q < jobs.size(); ++q) {
    const GemvJob &j = jobs[q];
    if (j.m <= 0) continue;
    const int ws = std::max(j.k1 ? gv_ws_host(j.k1) : 1, j.k2 ? gv_ws_host(j.k2) : 1), gpc = 8 / ws;
    const int ng = (j.m + 7) / 8;
    for (int g0 = 0; g0 < ng; g0 += 2 * gpc) items.push_back(GvItem{(int)q, g0});  // two groups per warp
  }
  if (items.empty()) return;
  static const bool gtrace = getenv("MFH_APPLY_TRACE") != nullptr;
  if (gtrace) {
    double el = 0, mx = 0;
    int nk2 = 0, nr = 0;
    for (auto &j : jobs) {
      el += (double)j.m * (j.k1 + j.k2);
      mx = std::max(mx, (double)(j.k1 + j.k2));
      nk2 += j.k2 > 0;
      nr += std::max(0, j.m);
    }
    fprintf(stderr, "[mfh gemv] jobs %5zu rows %7d avg k %7.1f max k %6.0f with k2 %5d ctas %5zu\n", jobs.size(), nr,
            el / std::max(1, nr), mx, nk2, items.size());
  }
  GemvJob *dj = sk.push(jobs);
  GvItem *di = sk.push(items);
  const int grid = (int)items.size();
  sk.launch([=](cudaStream_t st) {
    switch (nv) {
      case 2: launch_gemv_tc<2>(st, grid, dj, di); break;
      case 3: launch_gemv_tc<3>(st, grid, dj, di); break;
      case 4: launch_gemv_tc<4>(st, grid, dj, di); break;
      case 5: launch_gemv_tc<5>(st, grid, dj, di); break;
      case 6: launch_gemv_tc<6>(st, grid, dj, di); break;
      case 7: launch_gemv_tc<7>(st, grid, dj, di); break;
      case 8: launch_gemv_tc<8>(st, grid, dj, di); break;
      default: throw runtime_error("run_gemv: 1..8 right-hand sides per launch");
    }
    check_launch();
  });
}

static GemvJob gemv(double *y, const double *y0, int m, const double *A1, int lda1, int k1, const double *x1,
                    double a1, const double *A2 = nullptr, int lda2 = 0, int k2 = 0, const double *x2 = nullptr,
                    const long long *idx2 = nullptr, double a2 = 0.0) {
  return GemvJob{y, y0, m, A1, lda1, k1, x1, a1, A2, lda2, k2, x2, idx2, a2, 0, 0, 0, 0};
}
// the same job with the vector strides of a several-right-hand-side plan
static GemvJob strided(GemvJob j, long long ys, long long x1s, long long x2s, long long y0s = 0) {
  j.ys = ys;
  j.x1s = x1s;
  j.x2s = x2s;
  j.y0s = y0s;
  return j;
}

// The two-pass apply for nv right-hand sides (1..8; several only for an
// unsharded factor): every per-vector buffer is [nv][len], one graph.
static std::unique_ptr<ApplyPlan> make_apply(mfh_factor *F, int nv);
static void build_apply(mfh_factor *F) { F->apply = make_apply(F, 1); }
static std::unique_ptr<ApplyPlan> make_apply(mfh_factor *F, int nv) {
  auto tb0 = std::chrono::steady_clock::now();
  Ctx *ctx = F->ctx;
  auto AP = std::make_unique<ApplyPlan>();
  int64_t n = F->n;
  Arena &ar = F->arena;
  if (nv < 1 || nv > 8 || (nv > 1 && F->sharded)) throw runtime_error("apply plan: 1..8 right-hand sides (one when sharded)");
  AP->nv = nv;
  const int64_t nn1 = std::max<int64_t>(1, n);
  AP->d_b = ar.d(nv * nn1);
  AP->d_x = ar.d(nv * nn1);
  AP->bu = ar.d(nv * nn1);
  AP->xw = ar.d(nv * nn1);
  AP->y = ar.d(nn1);
  AP->yb = ar.d(nv * nn1);
  AP->ub = ar.d(nv * nn1);
  // w segments of the fronts kept in HODLR inverse form
  std::vector<int64_t> wo(F->fronts.size(), 0);
  int64_t wtot = 0;
  for (size_t q = 0; q < F->fronts.size(); ++q)
    if (F->fronts[q].structured && F->fronts[q].pform) {
      wo[q] = wtot;
      wtot += F->fronts[q].wlen;
    }
  const long long wst = std::max<int64_t>(1, wtot);
  AP->wb = ar.d(nv * wst);
  // contribution CSR (symbolic: built once per tree, kept on the device per context)
  std::shared_ptr<Ctx::ApplySym> sym;
  // a several-vector plan is built after the factorization, when the front id
  // views are gone: it shares the one-vector plan's contribution CSR
  if (nv > 1) sym = F->apply->sym;
  for (auto &a : ctx->apply_sym)
    if (!sym && a->uid == F->et_uid) sym = a;
  if (!sym) {
    auto ap = std::make_shared<Ctx::ApplySym>();
    Ctx::ApplySym &a = *ap;
    a.uid = F->et_uid;
    a.off.assign(F->fronts.size(), -1);
    int64_t tt = 0;
    for (size_t q = 0; q < F->fronts.size(); ++q) {
      FrontH &f = F->fronts[q];
      if (f.nh == 0 || f.npv == 0 || f.nf == 0) continue;
      a.off[q] = tt;
      tt += f.nf;
    }
    a.tot = tt;
    // contributions to each global id, in post order (multifrontal.py:549 order)
    std::vector<int64_t> cptr(n + 1, 0), coff(std::max<int64_t>(1, tt)), fro_all(std::max<int64_t>(1, tt));
    for (size_t q = 0; q < F->fronts.size(); ++q)
      if (a.off[q] >= 0)
        for (int j = 0; j < F->fronts[q].nf; ++j) {
          int64_t g = F->fronts[q].ids[F->fronts[q].npv + j];
          cptr[g + 1]++;
          fro_all[a.off[q] + j] = g;
        }
    for (int64_t i = 0; i < n; ++i) cptr[i + 1] += cptr[i];
    {
      std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
      for (size_t q = 0; q < F->fronts.size(); ++q)
        if (a.off[q] >= 0) {
          FrontH &f = F->fronts[q];
          for (int j = 0; j < f.nf; ++j) coff[fill[f.ids[f.npv + j]]++] = a.off[q] + j;
        }
    }
    CK(cudaMalloc(&a.d_cptr, sizeof(int64_t) * (n + 1)));
    CK(cudaMalloc(&a.d_coff, sizeof(int64_t) * std::max<int64_t>(1, tt)));
    CK(cudaMalloc(&a.d_fro, sizeof(int64_t) * std::max<int64_t>(1, tt)));
    upload(ctx->s, a.d_cptr, cptr.data(), sizeof(int64_t) * (n + 1));
    if (tt) {
      upload(ctx->s, a.d_coff, coff.data(), sizeof(int64_t) * tt);
      upload(ctx->s, a.d_fro, fro_all.data(), sizeof(int64_t) * tt);
    }
    if (ctx->apply_sym.size() >= Ctx::SYM_CACHE_MAX) ctx->apply_sym.erase(ctx->apply_sym.begin());
    ctx->apply_sym.push_back(ap);
    sym = ap;
  }
  AP->sym = sym;  // the plan's graph reads these arrays: keep them alive with the factor
  const std::vector<int64_t> &off = sym->off;
  const int64_t tot = sym->tot;
  long long *d_cptr = sym->d_cptr, *d_coff = sym->d_coff, *d_fro = sym->d_fro;
  AP->cbuf = ar.d(nv * std::max<int64_t>(1, tot));
  const long long cst = std::max<int64_t>(1, tot), nst = nn1;  // vector strides of cbuf and bu / xw

  Sink sk{ctx};
  sk.record = true;
  sk.persist = &ar;
  double *bu = AP->bu, *xw = AP->xw, *y = AP->y, *cbuf = AP->cbuf, *yb = AP->yb, *wb = AP->wb, *ub = AP->ub;
  double bytes = 0;
  // apply levels count only pivot-carrying nodes: merge nodes (npv = 0) do no
  // solve work, and skipping them collapses the long merge chains.
  // Levels are global (all ranks agree); a sharded factor runs its own fronts.
  const bool sh = F->sharded;
  const size_t NF = F->fronts.size();
  std::vector<int> ah(NF, -1);
  int maxh = -1;
  {
    std::vector<int> sub(NF, -1);
    for (size_t q = 0; q < NF; ++q) {
      FrontH &f = F->fronts[q];
      int below = -1;
      for (int c : f.allkids) below = std::max(below, sub[c]);
      if (f.nh > 0 && f.npv > 0) {
        ah[q] = below + 1;
        sub[q] = ah[q];
        maxh = std::max(maxh, ah[q]);
      } else {
        sub[q] = below;
      }
    }
  }
  std::vector<std::vector<int>> byh(maxh + 1);
  for (size_t q = 0; q < NF; ++q)
    if (ah[q] >= 0 && (!sh || F->mine[q])) byh[ah[q]].push_back((int)q);
  // sharded exchange points (symbolic, identical on every rank): upward before
  // level L when a level-L front has a descendant of another rank at a level
  // not yet exchanged; downward before L when a level-L front has an ancestor
  // of another rank at a level written since the last exchange
  std::vector<char> ex_up(maxh + 2, 0), ex_dn(maxh + 2, 0);
  if (sh) {
    const int W = F->world;
    std::vector<int> dsub(NF * W, -1), dmax(NF * W, -1);
    for (size_t q = 0; q < NF; ++q) {
      for (int c : F->fronts[q].allkids)
        for (int o = 0; o < W; ++o) dmax[q * W + o] = std::max(dmax[q * W + o], dsub[(size_t)c * W + o]);
      for (int o = 0; o < W; ++o) dsub[q * W + o] = dmax[q * W + o];
      if (ah[q] >= 0) dsub[q * W + F->owner[q]] = std::max(dsub[q * W + F->owner[q]], ah[q]);
    }
    const int INF = 1 << 30;
    std::vector<int> amin(NF * W, INF);
    for (size_t q = NF; q-- > 0;)  // parents come after children in post order
      for (int c : F->fronts[q].allkids) {
        for (int o = 0; o < W; ++o) amin[(size_t)c * W + o] = amin[q * W + o];
        if (ah[q] >= 0) amin[(size_t)c * W + F->owner[q]] = std::min(amin[(size_t)c * W + F->owner[q]], ah[q]);
      }
    std::vector<int> mo(NF, -1), ma(NF, INF);
    for (size_t q = 0; q < NF; ++q)
      for (int o = 0; o < W; ++o)
        if (o != F->owner[q]) {
          mo[q] = std::max(mo[q], dmax[q * W + o]);
          ma[q] = std::min(ma[q], amin[q * W + o]);
        }
    std::vector<std::vector<int>> all_at(maxh + 1);
    for (size_t q = 0; q < NF; ++q)
      if (ah[q] >= 0) all_at[ah[q]].push_back((int)q);
    int last = 0;
    for (int L = 0; L <= maxh; ++L) {
      bool need = false;
      for (int q : all_at[L]) need |= mo[q] >= last;
      if (need) {
        ex_up[L] = 1;
        last = L;
      }
    }
    int synced = INF;
    for (int L = maxh; L >= 0; --L) {
      bool need = false;
      for (int q : all_at[L]) need |= ma[q] <= synced;
      if (need) {
        ex_dn[L] = 1;
        synced = L;
      }
    }
  }
  long long *perm = F->d_perm;
  double *db = AP->d_b, *dx = AP->d_x;
  int grid_n = (int)std::min<int64_t>(cdiv(std::max<int64_t>(n, 1), 256), 148 * 8);
  // sharded: exchanges split the recorded ops into segments; an exchange
  // all-reduces this rank's own slots / pivots (selected, others zero) and
  // copies the result back
  std::vector<std::vector<std::function<void(cudaStream_t)>>> segs;
  int8_t *cb_mask = nullptr, *x_mask = nullptr;
  double *cb_tmp = nullptr, *x_tmp = nullptr;
  const int64_t ncb = std::max<int64_t>(1, tot);
  if (sh) {
    std::vector<int8_t> cm(ncb, 0), xm(std::max<int64_t>(1, n), 0);
    for (size_t q = 0; q < NF; ++q) {
      if (!F->mine[q]) continue;
      FrontH &f = F->fronts[q];
      if (off[q] >= 0)
        for (int j = 0; j < f.nf; ++j) cm[off[q] + j] = 1;
      for (int j = 0; j < f.npv; ++j) xm[f.piv_lo + j] = 1;
    }
    cb_mask = (int8_t *)ar.alloc(cm.size());
    x_mask = (int8_t *)ar.alloc(xm.size());
    {
      Sink up{ctx};
      up.push_to(cb_mask, cm.data(), cm.size());
      up.push_to(x_mask, xm.data(), xm.size());
    }
    cb_tmp = ar.d(ncb);
    x_tmp = ar.d(std::max<int64_t>(1, n));
    sk.launch([=](cudaStream_t s) {
      CK(cudaMemsetAsync(cbuf, 0, sizeof(double) * ncb, s));
      CK(cudaMemsetAsync(xw, 0, sizeof(double) * std::max<int64_t>(1, n), s));
    });
  }
  auto exchange_point = [&](double *buf, const int8_t *mask, double *tmp, int64_t cnt) {
    int g = (int)std::min<int64_t>(cdiv(cnt, 256), 148 * 8);
    sk.launch([=](cudaStream_t s) {
      k_mask_select<<<g, 256, 0, s>>>(buf, mask, tmp, cnt);
      check_launch();
    });
    segs.push_back(std::move(sk.ops));
    sk.ops.clear();
    AP->xchg.push_back({tmp, cnt});
    sk.launch([=](cudaStream_t s) {
      CK(cudaMemcpyAsync(buf, tmp, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, s));
    });
  };
  sk.launch([=](cudaStream_t s) {
    launch_pdl(k_scatter_perm, dim3(grid_n, nv), dim3(256), 0, s, (const double *)db, (const long long *)perm, bu,
               (long long)n);
    check_launch();
  });
  bytes += 24.0 * n;
  // ---------------- upward: b_u[fro] -= apply_fp(pp_solve(b_u[piv]))
  const bool atrace = getenv("MFH_APPLY_TRACE") != nullptr;
  auto upward = [&](std::vector<std::vector<int>> &byh) {
  for (int h = 0; h < (int)byh.size(); ++h) {
    if (sh && ex_up[h]) exchange_point(cbuf, cb_mask, cb_tmp, ncb);
    auto &fis = byh[h];
    if (fis.empty()) continue;
    std::vector<int64_t> gl;
    for (int q : fis) {
      FrontH &f = F->fronts[q];
      for (int j = 0; j < f.npv; ++j) gl.push_back(f.piv_lo + j);  // pivot ids are one contiguous run
    }
    long long *dgl = (long long *)sk.push(gl);
    int cnt = (int)gl.size();
    // level 0 fronts have no pivot-carrying descendants: nothing to gather
    if (h > 0) sk.launch([=](cudaStream_t s) {
      launch_pdl(k_contrib_gather, dim3((unsigned)std::min<int64_t>(cdiv((int64_t)cnt * 32, 256), 148 * 16), nv),
                 dim3(256), 0, s, (const long long *)dgl, cnt, (const long long *)d_cptr, (const long long *)d_coff,
                 (const double *)cbuf, bu, (double *)nullptr, (long long)cst, (long long)nst);
      check_launch();
    });
    // three dependent stages at most: st[0] reads b_piv only, st[1] reads
    // st[0]'s results, st[2] (HODLR inverse form with a dense F_fp) reads st[1]'s
    std::vector<GemvJob> st[3];
    for (int q : fis) {
      FrontH &f = F->fronts[q];
      const double *bp = bu + f.piv_lo;
      double *t = f.nf ? cbuf + off[q] : nullptr;
      if (!f.structured) {
        if (f.nf == 0) continue;
        st[0].push_back(strided(gemv(t, nullptr, f.nf, f.Gfp, f.npv, f.npv, bp, 1.0), cst, nst, 0));
        bytes += 8.0 * (double)f.nf * f.npv;
        continue;
      }
      // y_piv = H^{-1} b_piv, kept for the downward pass (b_u[piv] is final once
      // this level's gather ran: only ancestors' pivots change after it)
      double *yp = yb + f.piv_lo;
      int ystage;  // the stage that writes y_piv
      if (!f.pform) {
        st[0].push_back(strided(gemv(yp, nullptr, f.npv, f.Hinv, f.npv, f.npv, bp, 1.0), nst, nst, 0));
        bytes += 8.0 * (double)f.npv * f.npv;
        ystage = 0;
      } else {
        // HODLR inverse form: every w_v = Tm_v b_v at once, then per leaf
        // y_leaf = L^{-1} b_leaf - XL w[idx] (all ancestors' corrections)
        double *w = wb + wo[q];
        for (auto &tn : f.tnode) {
          const int rr = tn.r1 + tn.r2;
          st[0].push_back(strided(gemv(w + tn.woff, nullptr, rr, tn.Tm, tn.nv, tn.nv, bp + tn.lo, 1.0), wst, nst, 0));
          bytes += 8.0 * (double)rr * tn.nv;
        }
        for (auto &L : f.tleaf) {
          if (L.K)
            st[1].push_back(strided(gemv(yp + L.lo, nullptr, L.sz, L.Linv, L.sz, L.sz, bp + L.lo, 1.0, L.XL, L.K, L.K,
                                         w, L.idx, -1.0),
                                    nst, nst, wst));
          else
            st[1].push_back(strided(gemv(yp + L.lo, nullptr, L.sz, L.Linv, L.sz, L.sz, bp + L.lo, 1.0), nst, nst, 0));
          bytes += 8.0 * (double)L.sz * (L.sz + L.K);
        }
        ystage = 1;
      }
      if (f.nf == 0) continue;
      // t = F_fp H^{-1} b_piv: F_fp y_piv (dense fallback) or col_fp (RH b_piv) (low rank)
      const BlockH &bfp = F->blocks[f.fp];
      if (bfp.dense) {
        st[ystage + 1].push_back(strided(gemv(t, nullptr, f.nf, bfp.val, f.npv, f.npv, yp, 1.0), cst, nst, 0));
        bytes += 8.0 * (double)f.nf * f.npv;
      } else if (bfp.rank) {
        const int r = bfp.rank;
        double *tmp = ar.d((size_t)nv * r);
        st[0].push_back(strided(gemv(tmp, nullptr, r, f.RH, f.npv, f.npv, bp, 1.0), r, nst, 0));
        st[1].push_back(strided(gemv(t, nullptr, f.nf, bfp.col, r, r, tmp, 1.0), cst, r, 0));
        bytes += 8.0 * ((double)r * f.npv + (double)f.nf * r);
      } else {
        st[1].push_back(strided(gemv(t, nullptr, f.nf, nullptr, 0, 0, nullptr, 0.0), cst, 0, 0));  // exact zero contribution
      }
    }
    if (atrace) {
      int64_t mr = 0;
      for (int q : fis) mr = std::max<int64_t>(mr, F->fronts[q].npv);
      fprintf(stderr, "[mfh apply up %2d] fronts %5zu gather %7d jobs %5zu+%5zu+%5zu max npv %5lld\n", h, fis.size(), cnt,
              st[0].size(), st[1].size(), st[2].size(), (long long)mr);
    }
    for (auto &v : st) run_gemv(sk, v, nv);
  }
  };
  // ---------------- downward: x[piv] = pp_solve(b_u[piv] - apply_pf(x[fro]))
  auto downward = [&](std::vector<std::vector<int>> &byh) {
  for (int h = (int)byh.size() - 1; h >= 0; --h) {
    if (sh && ex_dn[h]) exchange_point(xw, x_mask, x_tmp, std::max<int64_t>(1, n));
    auto &fis = byh[h];
    if (fis.empty()) continue;
    // stages: sa[0] reads x_fro (final), sa[1] writes x_piv, except a dense
    // F_pf in HODLR inverse form: u, w = Tm u, then the leaves (sa[2])
    std::vector<GemvJob> sa[3];
    for (int q : fis) {
      FrontH &f = F->fronts[q];
      const double *bp = bu + f.piv_lo;
      double *xv = xw + f.piv_lo;
      const long long *fro = f.nf ? d_fro + off[q] : nullptr;
      if (!f.structured) {
        sa[1].push_back(strided(gemv(xv, nullptr, f.npv, f.Pinv, f.npv, f.npv, bp, 1.0, f.Gpf, f.nf, f.nf, xw, fro, -1.0),
                                nst, nst, nst));
        bytes += 8.0 * ((double)f.npv * f.npv + (double)f.npv * f.nf);
        continue;
      }
      // x_piv = y_piv - Xp (row_pf x_fro) (low rank), y_piv (no coupling), or
      // H^{-1} (b_piv - F_pf x_fro) (dense fallback); y_piv = H^{-1} b_piv
      const double *yp = yb + f.piv_lo;
      const BlockH *bpf = f.nf ? &F->blocks[f.pf] : nullptr;
      if (bpf && bpf->dense) {
        double *u = ub + f.piv_lo;
        sa[0].push_back(strided(gemv(u, bp, f.npv, nullptr, 0, 0, nullptr, 0.0, bpf->val, f.nf, f.nf, xw, fro, -1.0), nst,
                                0, nst, nst));
        bytes += 8.0 * (double)f.npv * f.nf;
        if (!f.pform) {
          sa[1].push_back(strided(gemv(xv, nullptr, f.npv, f.Hinv, f.npv, f.npv, u, 1.0), nst, nst, 0));
          bytes += 8.0 * (double)f.npv * f.npv;
        } else {
          double *w = wb + wo[q];
          for (auto &tn : f.tnode) {
            const int rr = tn.r1 + tn.r2;
            sa[1].push_back(strided(gemv(w + tn.woff, nullptr, rr, tn.Tm, tn.nv, tn.nv, u + tn.lo, 1.0), wst, nst, 0));
            bytes += 8.0 * (double)rr * tn.nv;
          }
          for (auto &L : f.tleaf) {
            if (L.K)
              sa[2].push_back(strided(gemv(xv + L.lo, nullptr, L.sz, L.Linv, L.sz, L.sz, u + L.lo, 1.0, L.XL, L.K, L.K,
                                           w, L.idx, -1.0),
                                      nst, nst, wst));
            else
              sa[2].push_back(strided(gemv(xv + L.lo, nullptr, L.sz, L.Linv, L.sz, L.sz, u + L.lo, 1.0), nst, nst, 0));
            bytes += 8.0 * (double)L.sz * (L.sz + L.K);
          }
        }
      } else if (bpf && bpf->rank) {
        const int r = bpf->rank;
        double *tmp = ar.d((size_t)nv * r);
        sa[0].push_back(strided(gemv(tmp, nullptr, r, nullptr, 0, 0, nullptr, 0.0, bpf->row, f.nf, f.nf, xw, fro, 1.0),
                                r, 0, nst));
        sa[1].push_back(strided(gemv(xv, yp, f.npv, nullptr, 0, 0, nullptr, 0.0, f.Xp, r, r, tmp, nullptr, -1.0), nst, 0,
                                r, nst));
        bytes += 8.0 * ((double)f.npv * r + (double)r * f.nf);
      } else {
        sa[1].push_back(strided(gemv(xv, yp, f.npv, nullptr, 0, 0, nullptr, 0.0), nst, 0, 0, nst));
      }
    }
    if (atrace) {
      double lb = 0;
      for (auto &v : sa)
        for (auto &j : v) lb += 8.0 * (double)j.m * (j.k1 + j.k2);
      fprintf(stderr, "[mfh apply dn %2d] jobs %5zu+%5zu+%5zu  %.2f MB\n", h, sa[0].size(), sa[1].size(), sa[2].size(),
              lb / 1e6);
    }
    for (auto &v : sa) run_gemv(sk, v, nv);
  }
  };
  // ---- low levels as whole dense subtrees per CTA (one launch per pass)
  SubApply sub[2] = {};  // upward, downward
  int sub_grid = 0, L0 = 0;
  if (!sh && !(getenv("MFH_APPLY_SUBTREE") && atoi(getenv("MFH_APPLY_SUBTREE")) == 0)) {
    const int INF = 1 << 30;
    int L0s = maxh + 1;  // the first level holding a structured front
    for (size_t q = 0; q < NF; ++q)
      if (ah[q] >= 0 && F->fronts[q].structured) L0s = std::min(L0s, ah[q]);
    std::vector<int> par(NF, -1), anc(NF, INF), cnt(NF, 1);
    std::vector<double> sb(NF, 0.0);  // bytes of the pivot-carrying fronts of the subtree
    for (size_t q = 0; q < NF; ++q) {
      FrontH &f = F->fronts[q];
      for (int c : f.allkids) {
        par[c] = (int)q;
        cnt[q] += cnt[c];
        sb[q] += sb[c];
      }
      if (ah[q] >= 0) sb[q] += 8.0 * ((double)f.npv * f.npv + 2.0 * f.npv * f.nf);
    }
    for (size_t q = NF; q-- > 0;)
      if (par[q] >= 0) anc[q] = ah[par[q]] >= 0 ? ah[par[q]] : anc[par[q]];
    // cut level by a cost model: per-level launches cost about 35 us per level
    // (gather + GEMV up, GEMV down); the subtree kernels cost their LPT
    // makespan at ~40 GB/s per CTA plus ~5 us of barriers and load latency per
    // level, in both passes
    const int GMAX = 2 * ctx->nsm;
    auto plan = [&](int L, std::vector<std::vector<int>> *assign) {
      std::vector<int> roots;
      for (size_t q = 0; q < NF; ++q)
        if (ah[q] >= 0 && ah[q] < L && anc[q] >= L) roots.push_back((int)q);
      if (roots.empty()) return 0.0;
      std::stable_sort(roots.begin(), roots.end(), [&](int a, int b) { return sb[a] > sb[b]; });
      const int G = std::min<int>((int)roots.size(), GMAX);
      std::vector<double> load(G, 0.0);
      if (assign) assign->assign(G, {});
      for (int r : roots) {
        int t = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        load[t] += sb[r];
        if (assign) (*assign)[t].push_back(r);
      }
      return *std::max_element(load.begin(), load.end());
    };
    double best = 35e-6 * L0s;
    for (int L = 1; L <= L0s; ++L) {
      const double c = 2.0 * (plan(L, nullptr) / 40e9 + 5e-6 * L) + 35e-6 * (L0s - L);
      if (c < best) {
        best = c;
        L0 = L;
      }
    }
    if (L0 > 0) {
      std::vector<std::vector<int>> assign;
      plan(L0, &assign);
      // per CTA, per level: the fronts of its subtrees (post order), their
      // upward and downward GEMV jobs and the pivot ids to gather
      std::vector<SubSeg> seg;
      std::vector<int> cseg{0}, start{0};
      std::vector<GemvJob> jup, jdn;
      std::vector<int> sdn{0};
      std::vector<long long> gids;
      int nfr = 0;
      for (auto &rs : assign) {
        std::sort(rs.begin(), rs.end());
        std::vector<std::vector<int>> lev(L0);
        for (int r : rs)
          for (int q = r - cnt[r] + 1; q <= r; ++q)
            if (ah[q] >= 0) lev[ah[q]].push_back(q);
        for (int L = 0; L < L0; ++L) {
          if (lev[L].empty()) continue;
          SubSeg g{};
          g.jb = (int)jup.size();
          g.gb = (int)gids.size();
          for (int q : lev[L]) {
            FrontH &f = F->fronts[q];
            ++nfr;
            if (L > 0)
              for (int j = 0; j < f.npv; ++j) gids.push_back(f.piv_lo + j);
            // upward t = Gfp b_piv (a zero-row job keeps jobs aligned with the downward list)
            const double *bp = bu + f.piv_lo;
            GemvJob u = f.nf ? strided(gemv(cbuf + off[q], nullptr, f.nf, f.Gfp, f.npv, f.npv, bp, 1.0), cst, nst, 0)
                             : strided(gemv(nullptr, nullptr, 0, nullptr, 0, 0, nullptr, 0.0), 0, 0, 0);
            GemvJob d = strided(gemv(xw + f.piv_lo, nullptr, f.npv, f.Pinv, f.npv, f.npv, bp, 1.0, f.Gpf, f.nf, f.nf,
                                     xw, f.nf ? d_fro + off[q] : nullptr, -1.0),
                                nst, nst, nst);
            jup.push_back(u);
            jdn.push_back(d);
            start.push_back(start.back() + gv_rows(u.m));  // rows padded to whole groups of 8
            sdn.push_back(sdn.back() + gv_rows(d.m));
            bytes += 8.0 * ((double)f.npv * f.npv + 2.0 * f.npv * f.nf);
          }
          g.je = (int)jup.size();
          g.ge = (int)gids.size();
          seg.push_back(g);
        }
        cseg.push_back((int)seg.size());
      }
      for (int pass = 0; pass < 2; ++pass) {
        SubApply &S = sub[pass];
        S.seg = sk.push(seg);
        S.cta_seg = sk.push(cseg);
        S.job = sk.push(pass == 0 ? jup : jdn);
        S.start = sk.push(pass == 0 ? start : sdn);
        S.gids = gids.empty() ? nullptr : sk.push(gids);
        S.cptr = d_cptr;
        S.coff = d_coff;
        S.cbuf = cbuf;
        S.bu = bu;
        S.cst = cst;
        S.nst = nst;
      }
      sub_grid = (int)assign.size();
      for (int h = 0; h < L0; ++h) byh[h].clear();
      if (atrace)
        fprintf(stderr, "[mfh apply] levels < %d (of %d dense-only) as %d subtree fronts on %d CTAs, est %.1f us\n",
                L0, L0s, nfr, sub_grid, best * 1e6);
    }
  }
  auto launch_sub = [&](bool up) {
    if (!sub_grid) return;
    const SubApply S = sub[up ? 0 : 1];
    const int g = sub_grid, v = nv, u = up ? 1 : 0;
    sk.launch([=](cudaStream_t st) {
      switch (v) {
        case 1: launch_pdl(k_apply_sub<1>, dim3(g), dim3(512), 0, st, S, u); break;
        case 2: launch_pdl(k_apply_sub<2>, dim3(g), dim3(512), 0, st, S, u); break;
        case 3: launch_pdl(k_apply_sub<3>, dim3(g), dim3(512), 0, st, S, u); break;
        case 4: launch_pdl(k_apply_sub<4>, dim3(g), dim3(512), 0, st, S, u); break;
        case 5: launch_pdl(k_apply_sub<5>, dim3(g), dim3(512), 0, st, S, u); break;
        case 6: launch_pdl(k_apply_sub<6>, dim3(g), dim3(512), 0, st, S, u); break;
        case 7: launch_pdl(k_apply_sub<7>, dim3(g), dim3(512), 0, st, S, u); break;
        case 8: launch_pdl(k_apply_sub<8>, dim3(g), dim3(512), 0, st, S, u); break;
        default: throw runtime_error("apply: 1..8 right-hand sides");
      }
      check_launch();
    });
  };
  launch_sub(true);
  upward(byh);
  downward(byh);
  launch_sub(false);
  if (sh) exchange_point(xw, x_mask, x_tmp, std::max<int64_t>(1, n));  // every rank gets every pivot
  sk.launch([=](cudaStream_t s) {
    launch_pdl(k_gather_perm, dim3(grid_n, nv), dim3(256), 0, s, (const double *)xw, (const long long *)perm, dx,
               (long long)n);
    check_launch();
  });
  // capture (the stream may still be running the factorization: captured work
  // is independent of it, and the graph is only launched after it)
  auto tb1 = std::chrono::steady_clock::now();
  auto capture = [&](std::vector<std::function<void(cudaStream_t)>> &ops, cudaGraph_t *g, cudaGraphExec_t *e) {
    CK(cudaStreamBeginCapture(ctx->s, cudaStreamCaptureModeThreadLocal));
    for (auto &op : ops) op(ctx->s);
    CK(cudaStreamEndCapture(ctx->s, g));
    CK(cudaGraphInstantiate(e, *g, 0));
  };
  if (sh) {
    segs.push_back(std::move(sk.ops));
    capture(segs[0], &AP->graph, &AP->exec);
    for (size_t k = 1; k < segs.size(); ++k) {
      cudaGraph_t g;
      cudaGraphExec_t e;
      capture(segs[k], &g, &e);
      AP->seg_graph.push_back(g);
      AP->seg_exec.push_back(e);
      AP->seg_nodes.push_back((int64_t)segs[k].size());
    }
  } else {
    capture(sk.ops, &AP->graph, &AP->exec);
    if (getenv("MFH_APPLY_OPS")) AP->ops = sk.ops;
  }
  auto tb2 = std::chrono::steady_clock::now();
  if (nv == 1) {
    F->timing.apply_build_ms = std::chrono::duration<double, std::milli>(tb1 - tb0).count();
    F->timing.apply_instantiate_ms = std::chrono::duration<double, std::milli>(tb2 - tb1).count();
  }
  AP->bytes = bytes;
  AP->nodes = sh ? (int64_t)segs[0].size() : (int64_t)sk.ops.size();
  return AP;
}

// A->d_b -> A->d_x; a sharded factor exchanges the contribution buffer
// between its two graphs and the solution after them
static void apply_run(mfh_factor *F) {
  Ctx *ctx = F->ctx;
  ApplyPlan *A = F->apply.get();
  CK(cudaGraphLaunch(A->exec, ctx->s));
  ctx->launches += A->nodes;
  for (size_t k = 0; k < A->xchg.size(); ++k) {
    F->exchange_or_throw(A->xchg[k].first, A->xchg[k].second);
    CK(cudaGraphLaunch(A->seg_exec[k], ctx->s));
    ctx->launches += A->seg_nodes[k];
  }
}

// the plan for nv right-hand sides (nv > 1: unsharded factors only)
static ApplyPlan *plan_nv(mfh_factor *F, int nv) {
  if (!F->apply) build_apply(F);
  if (nv == 1) return F->apply.get();
  auto &p = F->apply_nv[nv];
  if (!p) p = make_apply(F, nv);
  return p.get();
}

// nv right-hand sides, vector v at d_in + v * in_stride -> d_out + v * out_stride
static void apply_device_nv(mfh_factor *F, int nv, const double *d_in, int64_t in_stride, double *d_out,
                            int64_t out_stride) {
  Ctx *ctx = F->ctx;
  int64_t n = F->n;
  if (n == 0) return;
  ApplyPlan *A = plan_nv(F, nv);
  CK(cudaMemcpy2DAsync(A->d_b, sizeof(double) * n, d_in, sizeof(double) * in_stride, sizeof(double) * n, nv,
                       cudaMemcpyDeviceToDevice, ctx->s));
  if (nv == 1) {
    apply_run(F);
  } else {
    CK(cudaGraphLaunch(A->exec, ctx->s));
    ctx->launches += A->nodes;
  }
  CK(cudaMemcpy2DAsync(d_out, sizeof(double) * out_stride, A->d_x, sizeof(double) * n, sizeof(double) * n, nv,
                       cudaMemcpyDeviceToDevice, ctx->s));
}

static void apply_device(mfh_factor *F, const double *d_in, double *d_out) {
  Ctx *ctx = F->ctx;
  if (!F->apply) build_apply(F);
  ApplyPlan *A = F->apply.get();
  int64_t n = F->n;
  if (n == 0) return;
  CK(cudaMemcpyAsync(A->d_b, d_in, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s));
  apply_run(F);
  CK(cudaMemcpyAsync(d_out, A->d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s));
}

}  // namespace mfh

// ---------------------------------------------------------------------------
// operators for GMRES
// ---------------------------------------------------------------------------
// baseline preconditioners (krylov.py:164-204): diagonal, and ILUT with the
// factorization on the host (a row-sequential recurrence; bit-identical to the
// reference's) and the two triangular solves on the GPU, level-scheduled and
// replayed as one CUDA graph
struct mfh_precond {
  mfh::Ctx *ctx = nullptr;
  int kind = 0;  // 0 diagonal, 1 ILUT
  int64_t n = 0;
  double *d = nullptr;  // diagonal
  mfh::IlutFactors host;  // ILUT factors (host copy for ilut_factors / the test)
  long long *lp = nullptr, *up = nullptr;
  int *li = nullptr, *ui = nullptr, *lrows = nullptr, *urows = nullptr;
  double *lv = nullptr, *uv = nullptr, *b = nullptr, *y = nullptr, *x = nullptr;
  int64_t levels_l = 0, levels_u = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t nodes = 0;
  ~mfh_precond() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (void *q : {(void *)d, (void *)lp, (void *)up, (void *)li, (void *)ui, (void *)lrows, (void *)urows,
                    (void *)lv, (void *)uv, (void *)b, (void *)y, (void *)x})
      cudaFree(q);
  }
};

namespace mfh {
// streamed SpMV (k_spmv_stream) of one CSR: rows per chunk, entry capacity of a stage, stages,
// grid; R = 0: a row is too long to stream. The CSR arrays must carry the slack of the widened
// bulk copies: 4 row pointers, 8 columns, 4 values past the end.
struct SpmvStream {
  int R = 0, cap = 0, grid = 0, nst = 2;
  size_t smem = 0;
  int *ptr32 = nullptr;  // 4-byte row pointers when nnz < 2^31
};
static void spmv_stream_plan(Ctx *ctx, int64_t n_rows, const long long *hptr, SpmvStream &P) {
  const int64_t nnz = n_rows > 0 ? hptr[n_rows] : 0;
  if (n_rows <= 0 || nnz <= 0) return;
  int64_t maxrow = 0;
  for (int64_t r = 0; r < n_rows; ++r) maxrow = std::max<int64_t>(maxrow, hptr[r + 1] - hptr[r]);
  const char *eR = getenv("MFH_SPMV_R"), *eS = getenv("MFH_SPMV_STG"), *eP = getenv("MFH_SPMV_P64");  // tuning knobs
  // chunk shape: the most rows R in {128, 64, 32} whose longest possible chunk fits a stage
  // (measured: 128 rows x 7 entries, 128 x ~10, 64 x 27 beat the next larger chunk; a software-pipelined
  // variant with the next chunk's gathers in registers and three stages was slower: fewer CTAs per SM)
  int R = 0;
  for (int cand : {128, 64, 32})
    if ((!eR || cand <= atoi(eR)) && (int64_t)cand * maxrow <= (cand == 32 ? 8192 : 2048)) { R = cand; break; }
  if (eR && atoi(eR) >= 256 && 256 * maxrow <= 4096) R = 256;
  if (!R) return;
  const bool p32 = nnz < (int64_t(1) << 31) && !eP;
  P.R = R;
  P.cap = (int)((R * maxrow + 1) & ~(int64_t)1);
  P.nst = eS ? std::min(SPMV_MAX_STG, std::max(1, atoi(eS))) : 2;
  P.smem = P.nst * spmv_stage_bytes(P.R, P.cap, p32 ? 4 : 8);
  int per_sm = 0;
  if (p32) {
    std::vector<int> p4(hptr, hptr + n_rows + 1);
    p4.resize(n_rows + 8, 0);
    CK(cudaMalloc(&P.ptr32, sizeof(int) * (n_rows + 8)));
    upload(ctx->s, P.ptr32, p4.data(), sizeof(int) * (n_rows + 8));
    CK(cudaFuncSetAttribute(k_spmv_stream<int, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
    CK(cudaFuncSetAttribute(k_spmv_stream<int, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_stream<int, true>, 256, P.smem));
  } else {
    CK(cudaFuncSetAttribute(k_spmv_stream<long long, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
    CK(cudaFuncSetAttribute(k_spmv_stream<long long, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_stream<long long, true>, 256, P.smem));
  }
  // persistent CTAs with the same number of chunks each (no partial last round)
  const int64_t nchunks = cdiv(n_rows, (int64_t)R), gmax = (int64_t)ctx->nsm * std::max(1, per_sm);
  P.grid = (int)cdiv(nchunks, cdiv(nchunks, gmax));
}
static void spmv_stream_launch(Ctx *ctx, const SpmvStream &P, int64_t n_rows, const long long *ptr, const int *col,
                               const double *val, const double *x, const double *halo, int nl, double *y) {
  const int64_t nchunks = cdiv(n_rows, (int64_t)P.R);
  auto go = [&](auto kern, auto p) {
    launch_pdl(kern, dim3(P.grid), dim3(256), P.smem, ctx->s, (long long)n_rows, P.R, P.cap, P.nst, (long long)nchunks,
               p, col, val, x, halo ? halo : x, nl, y);
  };
  if (P.ptr32) {
    if (halo) go(k_spmv_stream<int, true>, (const int *)P.ptr32);
    else go(k_spmv_stream<int, false>, (const int *)P.ptr32);
  } else {
    if (halo) go(k_spmv_stream<long long, true>, ptr);
    else go(k_spmv_stream<long long, false>, ptr);
  }
  check_launch();
  ctx->launches++;
}
}  // namespace mfh

struct mfh_csr {
  mfh::Ctx *ctx = nullptr;
  int kind = 0;  // 0 csr, 1 dense
  int64_t nr = 0, nc = 0, nnz = 0;
  long long *ptr = nullptr;
  int *col = nullptr;
  double *val = nullptr;
  mfh::GemmJob *djob = nullptr;  // dense GEMV descriptor (x/y patched per call)
  mfh::SpmvStream stream;  // streamed SpMV plan (R = 0: rows too long, k_spmv_sub instead)
};

namespace mfh {

static void op_apply_device(mfh_csr *A, const double *x, double *y) {
  Ctx *ctx = A->ctx;
  if (A->kind == 0) {
    // lanes per row from the average row length
    const int64_t nnz = A->nnz;
    const double avg = A->nr ? (double)nnz / A->nr : 0.0;
    static const bool no_stream = getenv("MFH_SPMV_NO_STREAM") != nullptr;  // A/B knob
    if (A->stream.R > 0 && !no_stream) {
      spmv_stream_launch(ctx, A->stream, A->nr, A->ptr, A->col, A->val, x, nullptr, 0, y);
      return;
    }
    const int W = avg <= 4.5 ? 4 : (avg <= 9.5 ? 8 : (avg <= 20 ? 16 : 32));
    int grid = (int)std::min<int64_t>(cdiv(std::max<int64_t>(1, A->nr) * W, 256), 148 * 16);
    if (grid < 1) grid = 1;
    switch (W) {
      case 4: k_spmv_sub<4><<<grid, 256, 0, ctx->s>>>(A->nr, A->ptr, A->col, A->val, x, y); break;
      case 8: k_spmv_sub<8><<<grid, 256, 0, ctx->s>>>(A->nr, A->ptr, A->col, A->val, x, y); break;
      case 16: k_spmv_sub<16><<<grid, 256, 0, ctx->s>>>(A->nr, A->ptr, A->col, A->val, x, y); break;
      default: k_spmv<<<grid, 256, 0, ctx->s>>>(A->nr, A->ptr, A->col, A->val, x, y);
    }
    check_launch();
    ctx->launches++;
  } else {
    GemmJob j{A->val, x, y, (int)A->nr, 1, (int)A->nc, (int)A->nc, 1, 1, 1.0, 0.0};
    Sink s{ctx};
    run_gemm(s, {j});
  }
}

// d_in -> d_out on the context stream (device vectors of length n)
static void precond_apply_device(mfh_precond *P, const double *d_in, double *d_out) {
  Ctx *ctx = P->ctx;
  const int64_t n = P->n;
  if (n == 0) return;
  if (P->kind == 0) {
    const int g = (int)std::min<int64_t>(cdiv(n, 256), 148 * 8);
    k_diag_div<<<g, 256, 0, ctx->s>>>(n, P->d, d_in, d_out);
    check_launch();
    ctx->launches++;
    return;
  }
  CK(cudaMemcpyAsync(P->b, d_in, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s));
  CK(cudaGraphLaunch(P->exec, ctx->s));
  ctx->launches += P->nodes;
  CK(cudaMemcpyAsync(d_out, P->x, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s));
}

}  // namespace mfh

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

extern "C" const char *mfh_last_error(void) { return g_last_error.c_str(); }
extern "C" int mfh_version(void) { return 1; }

extern "C" int mfh_ctx_create(int device, mfh_ctx **out) {
  MFH_TRY
  CK(cudaSetDevice(device));
  auto *c = new mfh_ctx();
  c->c.device = device;
  CK(cudaStreamCreateWithFlags(&c->c.s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->c.side, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->c.side2, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->c.side3, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->c.side4, cudaStreamNonBlocking));
  {
    // the look-ahead panel must get SMs while the trailing update's grid is still being issued
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->c.la, cudaStreamNonBlocking, hi));
  }
  CK(cudaEventCreateWithFlags(&c->c.ev_la_cols, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->c.ev_la_panel, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->c.ev_join3, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->c.ev_fork2, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->c.ev_join4, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->c.ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->c.ev_join, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->c.ev_join2, cudaEventDisableTiming));
  for (auto &e : c->c.gmres_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  c->c.stage.init(size_t(64) << 20);
  c->c.scratch.chunk = size_t(512) << 20;
  CK(cudaMalloc(&c->c.d_part, sizeof(double) * std::max(RED_BLOCKS + 64, 2 * MGS_MAX_GRID)));
  CK(cudaMalloc(&c->c.d_scal, sizeof(double) * 4096));
  CK(cudaMallocHost(&c->c.h_scal, sizeof(double) * 4096));
  device_setup(&c->c);
  *out = c;
  MFH_CATCH
}

extern "C" void mfh_ctx_destroy(mfh_ctx *ctx) {
  if (!ctx) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.s);
  ctx->c.stage.release();
  ctx->c.scratch.release();
  ctx->c.pool.release();
  for (auto e : ctx->c.evpool) cudaEventDestroy(e);
  for (auto e : ctx->c.evd_pool) cudaEventDestroy(e);
  cudaFree(ctx->c.d_part);
  cudaFree(ctx->c.d_scal);
  if (ctx->c.blas) cublasDestroy(ctx->c.blas);
  if (ctx->c.blas_ws) cudaFree(ctx->c.blas_ws);
  for (auto &m : ctx->c.map_dev) cudaFree(m.second);
  for (auto &m : ctx->c.ids_dev) cudaFree(m.second);
  for (auto &q : ctx->c.pat_dev) {
    cudaFree(q.ptr);
    cudaFree(q.col);
    cudaFree(q.src);
  }
  ctx->c.apply_sym.clear();
  cudaFreeHost(ctx->c.h_scal);
  if (ctx->c.h_rb) cudaFreeHost(ctx->c.h_rb);
  cudaStreamSynchronize(ctx->c.side);
  cudaStreamSynchronize(ctx->c.side2);
  cudaStreamSynchronize(ctx->c.side3);
  cudaStreamSynchronize(ctx->c.side4);
  cudaStreamSynchronize(ctx->c.la);
  cudaEventDestroy(ctx->c.ev_la_cols);
  cudaEventDestroy(ctx->c.ev_la_panel);
  cudaStreamDestroy(ctx->c.la);
  cudaEventDestroy(ctx->c.ev_join3);
  cudaEventDestroy(ctx->c.ev_fork2);
  cudaEventDestroy(ctx->c.ev_join4);
  cudaStreamDestroy(ctx->c.side3);
  cudaStreamDestroy(ctx->c.side4);
  cudaEventDestroy(ctx->c.ev_fork);
  cudaEventDestroy(ctx->c.ev_join);
  cudaEventDestroy(ctx->c.ev_join2);
  for (auto &e : ctx->c.gmres_ev) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->c.side);
  cudaStreamDestroy(ctx->c.side2);
  cudaStreamDestroy(ctx->c.s);
  delete ctx;
  if (prev >= 0) cudaSetDevice(prev);
}

extern "C" int mfh_ctx_info(mfh_ctx *ctx, void **stream, int64_t *launches) {
  MFH_TRY
  if (stream) *stream = (void *)ctx->c.s;
  if (launches) *launches = ctx->c.launches;
  MFH_CATCH
}

extern "C" int mfh_ctx_sync(mfh_ctx *ctx) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  DeviceGuard dg_(ctx->c.device);
  MFH_TRY
  CK(cudaStreamSynchronize(ctx->c.s));
  MFH_CATCH
}

static int factorize_common(mfh_ctx *ctx, const mfh_etree *t, int64_t n, const int64_t *indptr,
                            const int64_t *indices, const double *values, int mode, const mfh_params *params,
                            const mfh_shard_t *shard, mfh_factor **out) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  mfh_factor *F = nullptr;
  MFH_TRY
  if (mode != MFH_CONVENTIONAL && mode != MFH_ACCELERATED) throw value_error("unknown mode");
  if (t->n != n) throw value_error("separator tree size does not match the matrix");
  DeviceGuard dg_(ctx->c.device);
  CsrView A{n, indptr, indices, values};  // the caller's arrays, read-only (no copy)
  F = new mfh_factor();
  F->ctx = &ctx->c;
  F->arena.pool = &ctx->c.pool;
  int64_t launches0 = ctx->c.launches;
  Factorizer fz{};
  fz.F = F;
  fz.ctx = &ctx->c;
  fz.et = t;
  fz.P = *params;
  fz.shard = shard;
  fz.run(A, mode);
  F->timing.kernel_launches = ctx->c.launches - launches0;
  *out = F;
  F = nullptr;
  }
  catch (const mfh::Error &e) {
    set_last_error(e.what());
    if (F) {
      cudaStreamSynchronize(ctx->c.s);
      ctx->c.scratch.reset();
      ctx->c.stage.rewind();
      F->arena.release();
      delete F;
    }
    return e.kind;
  }
  catch (const std::exception &e) {
    set_last_error(e.what());
    if (F) {
      cudaStreamSynchronize(ctx->c.s);
      ctx->c.scratch.reset();
      ctx->c.stage.rewind();
      F->arena.release();
      delete F;
    }
    return MFH_ERUNTIME;
  }
  return MFH_OK;
}

extern "C" int mfh_factorize(mfh_ctx *ctx, const mfh_etree *t, int64_t n, const int64_t *indptr,
                             const int64_t *indices, const double *values, int mode,
                             const mfh_params *params, mfh_factor **out) {
  return factorize_common(ctx, t, n, indptr, indices, values, mode, params, nullptr, out);
}

extern "C" int mfh_factorize_sharded(mfh_ctx *ctx, const mfh_etree *t, int64_t n, const int64_t *indptr,
                                     const int64_t *indices, const double *values, int mode,
                                     const mfh_params *params, const mfh_shard_t *shard, mfh_factor **out) {
  if (!shard) {
    set_last_error("mfh_factorize_sharded needs a shard description");
    return MFH_EVALUE;
  }
  return factorize_common(ctx, t, n, indptr, indices, values, mode, params, shard, out);
}

extern "C" int mfh_factor_stats(const mfh_factor *f, mfh_stats_t *out) {
  MFH_TRY
  *out = f->stats;
  MFH_CATCH
}

extern "C" int mfh_factor_records(const mfh_factor *f, mfh_record_t *out) {
  MFH_TRY
  std::memcpy(out, f->records.data(), sizeof(mfh_record_t) * f->records.size());
  MFH_CATCH
}

extern "C" int mfh_factor_timing(const mfh_factor *f, mfh_timing_t *out) {
  MFH_TRY
  *out = f->timing;
  MFH_CATCH
}

extern "C" int mfh_factor_blocks(const mfh_factor *f, int64_t *n_blocks, int64_t *n_perm, int64_t *info,
                                 int64_t *perms, double *ratios) {
  MFH_TRY
  int64_t nb = 0, np_ = 0;
  for (size_t q = 0; q < f->fronts.size(); ++q)
    for (int b : f->front_blocks[q]) {
      const BlockH &B = f->blocks[b];
      if (info) {
        int64_t *r = info + 7 * nb;
        r[0] = f->fronts[q].node;
        r[1] = B.m;
        r[2] = B.n;
        r[3] = (int64_t)B.I.size();
        r[4] = (int64_t)B.J.size();
        r[5] = B.rank;
        r[6] = B.dense ? 1 : 0;
      }
      if (ratios) ratios[nb] = B.ratio;
      if (perms) {
        for (int k = 0; k < B.rank; ++k) {
          perms[2 * (np_ + k)] = B.rowperm[k];
          perms[2 * (np_ + k) + 1] = B.colperm[k];
        }
      }
      nb++;
      np_ += B.rank;
    }
  *n_blocks = nb;
  *n_perm = np_;
  MFH_CATCH
}

extern "C" void mfh_factor_free(mfh_factor *f) {
  if (!f) return;
  std::lock_guard<std::recursive_mutex> lk_(f->ctx->mu);
  DeviceGuard dg_(f->ctx->device);
  cudaStreamSynchronize(f->ctx->s);
  f->arena.release();
  delete f;
}

extern "C" int mfh_apply(mfh_factor *f, const double *b, double *x, int64_t nrhs, int on_device) {
  std::lock_guard<std::recursive_mutex> lk_(f->ctx->mu);
  MFH_TRY
  DeviceGuard dg_(f->ctx->device);
  Ctx *ctx = f->ctx;
  int64_t n = f->n;
  if (!f->apply) build_apply(f);
  // up to eight right-hand sides per graph replay: the factor is read once per group
  for (int64_t r = 0; r < nrhs && n > 0;) {
    const int c = f->sharded ? 1 : (int)std::min<int64_t>(8, nrhs - r);
    if (on_device) {
      apply_device_nv(f, c, b + r * n, n, x + r * n, n);
    } else {
      ApplyPlan *A = plan_nv(f, c);
      CK(cudaMemcpyAsync(A->d_b, b + r * n, sizeof(double) * n * c, cudaMemcpyHostToDevice, ctx->s));
      if (c == 1) {
        apply_run(f);
      } else {
        CK(cudaGraphLaunch(A->exec, ctx->s));
        ctx->launches += A->nodes;
      }
      CK(cudaMemcpyAsync(x + r * n, A->d_x, sizeof(double) * n * c, cudaMemcpyDeviceToHost, ctx->s));
    }
    r += c;
  }
  CK(cudaStreamSynchronize(ctx->s));
  MFH_CATCH
}

// per-node solve operators (DenseNodeFactor / StructuredNodeFactor,
// multifrontal.py:160-216): op 0 pp_solve (F_pp^{-1} v), 1 apply_pf (F_pf v),
// 2 apply_fp (F_fp v); host vectors
extern "C" int mfh_node_op(mfh_factor *f, int64_t node, int op, const double *x, double *y) {
  std::lock_guard<std::recursive_mutex> lk_(f->ctx->mu);
  MFH_TRY
  DeviceGuard dg_(f->ctx->device);
  using namespace mfh;
  Ctx *ctx = f->ctx;
  int q = -1;
  for (size_t t = 0; t < f->post.size(); ++t)
    if (f->post[t] == node) q = (int)t;
  if (q < 0) throw value_error("node " + std::to_string(node) + " is not in the elimination tree");
  const FrontH &fr = f->fronts[q];
  if (fr.nh == 0) throw value_error("node " + std::to_string(node) + " has no node factor");
  if (op < 0 || op > 2) throw value_error("node operator must be 0 (pp_solve), 1 (apply_pf) or 2 (apply_fp)");
  const int npv = fr.npv, nf = fr.nf;
  const int nin = op == 1 ? nf : npv, nout = op == 2 ? nf : npv;
  if (nout == 0) return MFH_OK;
  if (npv == 0 || nin == 0) {  // merge node (F_fp is nf x 0) or F_pf with no columns
    std::memset(y, 0, sizeof(double) * nout);
    return MFH_OK;
  }
  double *dx = ctx->scratch.d(std::max(1, nin)), *dy = ctx->scratch.d(std::max(1, nout));
  double *dt = ctx->scratch.d(std::max(1, std::max(npv, nf)));
  if (nin) CK(cudaMemcpyAsync(dx, x, sizeof(double) * nin, cudaMemcpyHostToDevice, ctx->s));
  Sink sk{ctx};
  std::vector<GemvJob> g1, g2;
  if (op == 0 && fr.structured && fr.pform) {
    // HODLR inverse form: w_v = Tm_v x_v for every node, then the leaves
    double *dw = ctx->scratch.d(std::max<int64_t>(1, fr.wlen));
    for (auto &tn : fr.tnode) g1.push_back(gemv(dw + tn.woff, nullptr, tn.r1 + tn.r2, tn.Tm, tn.nv, tn.nv, dx + tn.lo, 1.0));
    for (auto &L : fr.tleaf)
      g2.push_back(L.K ? gemv(dy + L.lo, nullptr, L.sz, L.Linv, L.sz, L.sz, dx + L.lo, 1.0, L.XL, L.K, L.K, dw, L.idx, -1.0)
                       : gemv(dy + L.lo, nullptr, L.sz, L.Linv, L.sz, L.sz, dx + L.lo, 1.0));
  } else if (op == 0) {
    g1.push_back(gemv(dy, nullptr, npv, fr.structured ? fr.Hinv : fr.Pinv, npv, npv, dx, 1.0));
  } else if (!fr.structured) {
    // F_pf v = F_pp (Gpf v), F_fp v = Gfp (F_pp v)  (Gpf = F_pp^{-1} F_pf, Gfp = F_fp F_pp^{-1})
    if (op == 1) {
      g1.push_back(gemv(dt, nullptr, npv, fr.Gpf, nf, nf, dx, 1.0));
      g2.push_back(gemv(dy, nullptr, npv, fr.Fpp, npv, npv, dt, 1.0));
    } else {
      g1.push_back(gemv(dt, nullptr, npv, fr.Fpp, npv, npv, dx, 1.0));
      g2.push_back(gemv(dy, nullptr, nf, fr.Gfp, npv, npv, dt, 1.0));
    }
  } else {
    FacView v = fac_view(f, f->blocks[op == 1 ? fr.pf : fr.fp]);
    if (v.rank == 0) {
      CK(cudaMemsetAsync(dy, 0, sizeof(double) * nout, ctx->s));
    } else {
      g1.push_back(gemv(dt, nullptr, v.rank, v.row, v.ldr, nin, dx, 1.0));  // row factor first
      g2.push_back(gemv(dy, nullptr, nout, v.col, v.ldc, v.rank, dt, 1.0));
    }
  }
  run_gemv(sk, g1);
  run_gemv(sk, g2);
  CK(cudaMemcpyAsync(y, dy, sizeof(double) * nout, cudaMemcpyDeviceToHost, ctx->s));
  CK(cudaStreamSynchronize(ctx->s));
  ctx->scratch.reset();
  ctx->stage.rewind();
  MFH_CATCH
}

extern "C" int mfh_apply_bench(mfh_factor *f, int64_t reps, double *ms_per_apply, double *bytes_per_apply) {
  std::lock_guard<std::recursive_mutex> lk_(f->ctx->mu);
  MFH_TRY
  DeviceGuard dg_(f->ctx->device);
  Ctx *ctx = f->ctx;
  if (!f->apply) build_apply(f);
  ApplyPlan *A = f->apply.get();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  apply_run(f);
  CK(cudaEventRecord(e0, ctx->s));
  for (int64_t r = 0; r < reps; ++r) apply_run(f);
  CK(cudaEventRecord(e1, ctx->s));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *ms_per_apply = ms / std::max<int64_t>(1, reps);
  *bytes_per_apply = A->bytes;
  if (!A->ops.empty()) {  // warm per-op device times, ops run eagerly with events between them
    const size_t no = A->ops.size();
    std::vector<cudaEvent_t> ev(no + 1);
    for (auto &e : ev) CK(cudaEventCreate(&e));
    std::vector<float> best(no, 1e30f);
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(ev[0], ctx->s));
      for (size_t k = 0; k < no; ++k) {
        A->ops[k](ctx->s);
        CK(cudaEventRecord(ev[k + 1], ctx->s));
      }
      CK(cudaEventSynchronize(ev[no]));
      for (size_t k = 0; k < no; ++k) {
        float t;
        CK(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
        best[k] = std::min(best[k], t);
      }
    }
    double sum = 0;
    for (size_t k = 0; k < no; ++k) {
      fprintf(stderr, "[mfh apply op %3zu] %8.2f us\n", k, best[k] * 1e3);
      sum += best[k] * 1e3;
    }
    fprintf(stderr, "[mfh apply ops] sum %.1f us over %zu ops\n", sum, no);
    for (auto &e : ev) cudaEventDestroy(e);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  MFH_CATCH
}

extern "C" int mfh_precond_diag_create(mfh_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                                       const double *values, mfh_precond **out) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  std::vector<double> dg((size_t)std::max<int64_t>(n, 1), 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p)
      if (indices[p] == i) dg[i] = values[p];
  for (int64_t i = 0; i < n; ++i)  // krylov.py:166-168
    if (dg[i] == 0.0) throw value_error("zero diagonal entry at index " + std::to_string(i));
  std::unique_ptr<mfh_precond> P(new mfh_precond());
  P->ctx = &ctx->c;
  P->kind = 0;
  P->n = n;
  CK(cudaMalloc(&P->d, sizeof(double) * std::max<int64_t>(n, 1)));
  upload(ctx->c.s, P->d, dg.data(), sizeof(double) * n);
  *out = P.release();
  MFH_CATCH
}

// level sets of a triangular factor: rows whose dependencies are all in
// earlier levels (lower: columns < i; upper: columns > i, diagonal first)
static std::vector<std::vector<int>> tri_levels(int64_t n, const std::vector<int64_t> &ptr,
                                                const std::vector<int64_t> &idx, bool upper) {
  std::vector<int> lev((size_t)std::max<int64_t>(n, 1), 0);
  int mx = -1;
  for (int64_t s = 0; s < n; ++s) {
    const int64_t i = upper ? n - 1 - s : s;
    int l = 0;
    for (int64_t p = ptr[i] + (upper ? 1 : 0); p < ptr[i + 1]; ++p) l = std::max(l, lev[idx[p]] + 1);
    lev[i] = l;
    mx = std::max(mx, l);
  }
  std::vector<std::vector<int>> out(mx + 1);
  for (int64_t i = 0; i < n; ++i) out[lev[i]].push_back((int)i);
  return out;
}

extern "C" int mfh_precond_ilut_create(mfh_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                                       const double *values, int64_t k, double drop_tol, mfh_precond **out) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  if (k < 1) throw value_error("k must be at least 1");  // krylov.py:180-185
  if (!(drop_tol >= 0)) throw value_error("drop_tol must be nonnegative");
  if (n < 1) throw value_error("ILUT requires a non-empty square matrix");
  const int64_t nnz = indptr[n];
  const int64_t cap = k * nnz / n + 1;
  std::unique_ptr<mfh_precond> P(new mfh_precond());
  P->ctx = &ctx->c;
  P->kind = 1;
  P->n = n;
  P->host = ilut_factor(n, indptr, indices, values, cap, drop_tol);
  const IlutFactors &H = P->host;
  auto up_i32 = [&](int **dst, const std::vector<int64_t> &v) {
    std::vector<int> t(v.begin(), v.end());
    CK(cudaMalloc(dst, sizeof(int) * std::max<size_t>(1, t.size())));
    upload(ctx->c.s, *dst, t.data(), sizeof(int) * t.size());
  };
  auto up_raw = [&](auto **dst, const auto &v) {
    CK(cudaMalloc(dst, sizeof(v[0]) * std::max<size_t>(1, v.size())));
    upload(ctx->c.s, *dst, v.data(), sizeof(v[0]) * v.size());
  };
  up_raw(&P->lp, H.lp);
  up_raw(&P->up, H.up);
  up_i32(&P->li, H.li);
  up_i32(&P->ui, H.ui);
  up_raw(&P->lv, H.lv);
  up_raw(&P->uv, H.uv);
  for (double **q : {&P->b, &P->y, &P->x}) CK(cudaMalloc(q, sizeof(double) * n));
  auto L = tri_levels(n, H.lp, H.li, false), U = tri_levels(n, H.up, H.ui, true);
  P->levels_l = (int64_t)L.size();
  P->levels_u = (int64_t)U.size();
  std::vector<int> lr, ur;
  std::vector<std::pair<int64_t, int>> lo, uo;  // (offset, count) per level
  for (auto &v : L) {
    lo.push_back({(int64_t)lr.size(), (int)v.size()});
    lr.insert(lr.end(), v.begin(), v.end());
  }
  for (auto &v : U) {
    uo.push_back({(int64_t)ur.size(), (int)v.size()});
    ur.insert(ur.end(), v.begin(), v.end());
  }
  up_raw(&P->lrows, lr);
  up_raw(&P->urows, ur);
  // one graph: every level of L (b -> y), then every level of U (y -> x)
  cudaStream_t st = ctx->c.s;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (auto &q : lo)
    k_trsv_level<<<(unsigned)cdiv(q.second, 128), 128, 0, st>>>(P->lrows + q.first, q.second, P->lp, P->li, P->lv,
                                                                  P->b, P->y, 0);
  for (auto &q : uo)
    k_trsv_level<<<(unsigned)cdiv(q.second, 128), 128, 0, st>>>(P->urows + q.first, q.second, P->up, P->ui, P->uv,
                                                                  P->y, P->x, 1);
  CK(cudaStreamEndCapture(st, &P->graph));
  CK(cudaGraphInstantiate(&P->exec, P->graph, 0));
  P->nodes = (int64_t)(lo.size() + uo.size());
  *out = P.release();
  MFH_CATCH
}

extern "C" int mfh_precond_info(const mfh_precond *P, int64_t *stored_reals, int64_t *lnz, int64_t *unz,
                                int64_t *levels) {
  MFH_TRY
  if (P->kind == 0) {
    *stored_reals = P->n;
    if (lnz) *lnz = 0;
    if (unz) *unz = 0;
    if (levels) *levels = 1;
  } else {
    *stored_reals = (int64_t)(P->host.lv.size() + P->host.uv.size());
    if (lnz) *lnz = (int64_t)P->host.lv.size();
    if (unz) *unz = (int64_t)P->host.uv.size();
    if (levels) *levels = P->levels_l + P->levels_u;
  }
  MFH_CATCH
}

extern "C" int mfh_precond_ilut_factors(const mfh_precond *P, int64_t *lp, int64_t *li, double *lv, int64_t *up,
                                        int64_t *ui, double *uv) {
  MFH_TRY
  if (P->kind != 1) throw value_error("not an ILUT preconditioner");
  const IlutFactors &H = P->host;
  std::memcpy(lp, H.lp.data(), sizeof(int64_t) * H.lp.size());
  std::memcpy(up, H.up.data(), sizeof(int64_t) * H.up.size());
  std::memcpy(li, H.li.data(), sizeof(int64_t) * H.li.size());
  std::memcpy(ui, H.ui.data(), sizeof(int64_t) * H.ui.size());
  std::memcpy(lv, H.lv.data(), sizeof(double) * H.lv.size());
  std::memcpy(uv, H.uv.data(), sizeof(double) * H.uv.size());
  MFH_CATCH
}

extern "C" int mfh_precond_apply(mfh_precond *P, const double *b, double *x, int on_device) {
  std::lock_guard<std::recursive_mutex> lk_(P->ctx->mu);
  MFH_TRY
  DeviceGuard dg_(P->ctx->device);
  Ctx *ctx = P->ctx;
  const int64_t n = P->n;
  if (on_device) {
    precond_apply_device(P, b, x);
  } else {
    double *db = ctx->scratch.d(std::max<int64_t>(1, n)), *dx = ctx->scratch.d(std::max<int64_t>(1, n));
    CK(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->s));
    precond_apply_device(P, db, dx);
    CK(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->s));
  }
  CK(cudaStreamSynchronize(ctx->s));
  if (!on_device) ctx->scratch.reset();
  MFH_CATCH
}

extern "C" void mfh_precond_free(mfh_precond *P) {
  if (!P) return;
  std::lock_guard<std::recursive_mutex> lk_(P->ctx->mu);
  DeviceGuard dg_(P->ctx->device);
  cudaStreamSynchronize(P->ctx->s);
  delete P;
}

extern "C" int mfh_csr_create(mfh_ctx *ctx, int64_t n_rows, int64_t n_cols, const int64_t *indptr,
                              const int64_t *indices, const double *values, mfh_csr **out) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  auto *A = new mfh_csr();
  A->ctx = &ctx->c;
  A->kind = 0;
  A->nr = n_rows;
  A->nc = n_cols;
  int64_t nnz = indptr[n_rows];
  A->nnz = nnz;
  // slack for the streamed SpMV's widened bulk copies (16-byte aligned ends)
  CK(cudaMalloc(&A->ptr, sizeof(int64_t) * (n_rows + 4)));
  CK(cudaMalloc(&A->col, sizeof(int) * (nnz + 8)));
  CK(cudaMalloc(&A->val, sizeof(double) * (nnz + 4)));
  CK(cudaMemsetAsync(A->ptr + n_rows, 0, sizeof(int64_t) * 4, A->ctx->s));
  CK(cudaMemsetAsync(A->col + nnz, 0, sizeof(int) * 8, A->ctx->s));
  CK(cudaMemsetAsync(A->val + nnz, 0, sizeof(double) * 4, A->ctx->s));
  std::vector<int> c32(indices, indices + nnz);
  spmv_stream_plan(A->ctx, n_rows, reinterpret_cast<const long long *>(indptr), A->stream);
  upload(A->ctx->s, A->ptr, indptr, sizeof(int64_t) * (n_rows + 1));
  if (nnz) {
    upload(A->ctx->s, A->col, c32.data(), sizeof(int) * nnz);
    upload(A->ctx->s, A->val, values, sizeof(double) * nnz);
  }
  *out = A;
  MFH_CATCH
}

extern "C" int mfh_dense_create(mfh_ctx *ctx, int64_t n, const double *values, mfh_csr **out) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  auto *A = new mfh_csr();
  A->ctx = &ctx->c;
  A->kind = 1;
  A->nr = n;
  A->nc = n;
  CK(cudaMalloc(&A->val, sizeof(double) * std::max<int64_t>(1, n * n)));
  upload(A->ctx->s, A->val, values, sizeof(double) * n * n);
  *out = A;
  MFH_CATCH
}

extern "C" void mfh_csr_free(mfh_csr *A) {
  if (!A) return;
  std::lock_guard<std::recursive_mutex> lk_(A->ctx->mu);
  DeviceGuard dg_(A->ctx->device);
  cudaStreamSynchronize(A->ctx->s);
  cudaFree(A->ptr);
  cudaFree(A->stream.ptr32);
  cudaFree(A->col);
  cudaFree(A->val);
  delete A;
}

extern "C" int mfh_spmv_bench(mfh_csr *A, int64_t reps, double *ms_per_spmv) {
  std::lock_guard<std::recursive_mutex> lk_(A->ctx->mu);
  MFH_TRY
  DeviceGuard dg_(A->ctx->device);
  Ctx *ctx = A->ctx;
  double *dx = ctx->scratch.d(std::max<int64_t>(1, A->nc)), *dy = ctx->scratch.d(std::max<int64_t>(1, A->nr));
  CK(cudaMemsetAsync(dx, 0, sizeof(double) * std::max<int64_t>(1, A->nc), ctx->s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  op_apply_device(A, dx, dy);
  CK(cudaEventRecord(e0, ctx->s));
  for (int64_t r = 0; r < reps; ++r) op_apply_device(A, dx, dy);
  CK(cudaEventRecord(e1, ctx->s));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *ms_per_spmv = ms / std::max<int64_t>(1, reps);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ctx->scratch.reset();
  MFH_CATCH
}

extern "C" int mfh_spmv(mfh_csr *A, const double *x, double *y, int on_device) {
  std::lock_guard<std::recursive_mutex> lk_(A->ctx->mu);
  MFH_TRY
  DeviceGuard dg_(A->ctx->device);
  Ctx *ctx = A->ctx;
  if (on_device) {
    op_apply_device(A, x, y);
  } else {
    double *dx, *dy;
    CK(cudaMallocAsync(&dx, sizeof(double) * std::max<int64_t>(1, A->nc), ctx->s));
    CK(cudaMallocAsync(&dy, sizeof(double) * std::max<int64_t>(1, A->nr), ctx->s));
    CK(cudaMemcpyAsync(dx, x, sizeof(double) * A->nc, cudaMemcpyHostToDevice, ctx->s));
    op_apply_device(A, dx, dy);
    CK(cudaMemcpyAsync(y, dy, sizeof(double) * A->nr, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaFreeAsync(dx, ctx->s));
    CK(cudaFreeAsync(dy, ctx->s));
  }
  CK(cudaStreamSynchronize(ctx->s));
  MFH_CATCH
}

// ---------------------------------------------------------------------------
// GMRES (krylov.py:68-161): vectors on the device, Hessenberg/Givens on host
// ---------------------------------------------------------------------------
namespace mfh {

struct GmresRun {
  Ctx *ctx;
  const mfh_gmres_ops *ops;
  int64_t n;
  std::vector<double> hx, hy;  // host bounce buffers for callbacks
  double *tmp = nullptr, *tmp2 = nullptr;

  int gridn() const { return (int)std::min<int64_t>(cdiv(std::max<int64_t>(n, 1), 256), 148 * 8); }

  void host_op(mfh_host_op cb, void *user, const double *dx, double *dy) {
    hx.resize(n);
    hy.resize(n);
    CK(cudaMemcpyAsync(hx.data(), dx, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
    cb(user, hx.data(), hy.data());
    CK(cudaMemcpyAsync(dy, hy.data(), sizeof(double) * n, cudaMemcpyHostToDevice, ctx->s));
    CK(cudaStreamSynchronize(ctx->s));
  }
  void A(const double *x, double *y) {
    if (ops->A)
      op_apply_device(ops->A, x, y);
    else
      host_op(ops->A_cb, ops->A_user, x, y);
  }
  double m_ms = 0.0;
  void M(const double *x, double *y) {
    auto t0 = std::chrono::steady_clock::now();
    if (ops->P) {
      precond_apply_device(ops->P, x, y);
    } else if (ops->M) {
      apply_device(ops->M, x, y);
      m_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    } else if (ops->M_cb)
      host_op(ops->M_cb, ops->M_user, x, y);
    else
      CK(cudaMemcpyAsync(y, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s));
  }
  // dot into device scalar slot, deterministic
  void dot(const double *x, const double *y, double *out, bool do_sqrt) {
    ctx->launches += 2;
    k_dot_part<<<RED_BLOCKS, RED_THREADS, 0, ctx->s>>>(x, y, n, ctx->d_part);
    k_finish<<<1, 32, 0, ctx->s>>>(ctx->d_part, out, do_sqrt ? 1 : 0);
    check_launch();
  }
  double sync_ms = 0.0;
  double host_scalar(double *d) {
    CK(cudaMemcpyAsync(ctx->h_scal, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
    auto t0 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(ctx->s));
    sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return ctx->h_scal[0];
  }

  void run(const double *d_b, double *d_x, double tol, int64_t max_iter, int64_t restart,
           std::vector<double> &res, int64_t &its, bool &conv) {
    if (!(tol > 0.0 && tol < 1.0)) throw value_error("tol must lie in (0, 1)");
    if (max_iter < 1 || restart < 1) throw value_error("max_iter and restart must be positive");
    res.clear();
    its = 0;
    conv = false;
    double *S = ctx->d_scal;  // [0] norm b, [1] beta, [2] hn, [8..] H column
    const bool trace = std::getenv("MFH_GMRES_TRACE") != nullptr;
    CK(cudaMemsetAsync(d_x, 0, sizeof(double) * n, ctx->s));
    dot(d_b, d_b, S, true);
    double nb = host_scalar(S);
    if (nb == 0.0) {
      conv = true;
      res.push_back(0.0);
      return;
    }
    int64_t mcap = std::min(restart, max_iter);
    if (mcap > 2000)  // Hessenberg column and y live in the 4096-slot scalar buffers
      throw value_error("min(restart, max_iter) must be <= 2000");
    // Krylov basis + work vectors from the context's chunk pool (no per-solve
    // cudaMalloc / driver-pool remapping)
    auto chunk = ctx->pool.take(sizeof(double) * (size_t)n * (size_t)(mcap + 4));
    double *V = (double *)chunk.first, *w = V + n * (mcap + 1), *r = w + n, *z = r + n;
    double *dy = S + 2048;
    int g = gridn();
    const MgsPlan mgs = mgs_plan(ctx->device, n);
    auto cleanup = [&]() {
      cudaStreamSynchronize(ctx->s);
      ctx->pool.give(chunk);
    };
    try {
      while (its < max_iter && !conv) {
        A(d_x, w);
        k_sub<<<g, 256, 0, ctx->s>>>(d_b, w, r, n);
        ctx->launches += 2;
        dot(r, r, S + 1, true);
        double beta = host_scalar(S + 1);
        if (!std::isfinite(beta)) throw value_error("GMRES residual is not finite");
        if (beta / nb <= tol) {
          conv = true;
          if (res.empty()) res.push_back(beta / nb);
          break;
        }
        int64_t m = std::min(restart, max_iter - its);
        std::vector<double> H((m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), gg(m + 1, 0.0);
        auto h = [&](int64_t i, int64_t j) -> double & { return H[i * m + j]; };
        gg[0] = beta;
        k_scale_inv<<<g, 256, 0, ctx->s>>>(S + 1, r, V, n);
        int64_t j = 0;
        bool lucky_stop = false;
        // Arnoldi steps are pipelined one deep: step j+1 (and the basis vector
        // it starts from, V_{j+1} = w / H[j+1], a device value) is enqueued
        // before the host waits for step j's Hessenberg column, so the GPU does
        // not idle while the host applies the Givens rotations. A speculative
        // step after the last one only writes scratch (w, z, H slots, V_{j+1})
        // that the final combine never reads. It is skipped when the residual
        // trend says step j is likely the last (it would delay the combine).
        double *hbuf[2] = {ctx->h_scal + 16, ctx->h_scal + 2040};  // pinned: the copies are truly async
        cudaEvent_t *hev = ctx->gmres_ev;
        double qm = 0.0, qa = 0.0, qg = 0.0;
        auto enqueue_step = [&](int64_t jj) {
          auto q0 = std::chrono::steady_clock::now();
          if (jj > 0) {
            k_scale_inv<<<g, 256, 0, ctx->s>>>(S + 8 + jj, w, V + jj * n, n);
            ctx->launches++;
          }
          M(V + jj * n, z);
          auto q1 = std::chrono::steady_clock::now();
          A(z, w);
          auto q2 = std::chrono::steady_clock::now();
          {
            // whole MGS sweep + norm in one cooperative launch
            launch_mgs(mgs, V, w, n, (int)jj, S + 8, ctx->d_part, ctx->s);
            ctx->launches++;
          }
          CK(cudaMemcpyAsync(hbuf[jj & 1], S + 8, sizeof(double) * (jj + 2), cudaMemcpyDeviceToHost, ctx->s));
          CK(cudaEventRecord(hev[jj & 1], ctx->s));
          auto q3 = std::chrono::steady_clock::now();
          auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
          qm = ms(q0, q1);
          qa = ms(q1, q2);
          qg = ms(q2, q3);
        };
        // host callbacks see exactly the reference's calls: no speculation
        const bool can_spec = ops->A != nullptr && (ops->M != nullptr || ops->M_cb == nullptr);
        bool ahead = false;  // step j+1 already enqueued
        enqueue_step(0);
        while (j < m) {
          // speculate on step j+1 unless step j is predicted to converge
          bool spec = can_spec && j + 1 < m && its + 1 < max_iter;
          if (spec && res.size() >= 2 && j >= 2) {
            double r1 = res[res.size() - 1], r0 = res[res.size() - 2];
            double rate = r0 > 0.0 ? r1 / r0 : 1.0;
            if (r1 * rate <= 4.0 * tol) spec = false;
          }
          if (spec) enqueue_step(j + 1);
          ahead = spec;
          auto q4 = std::chrono::steady_clock::now();
          CK(cudaEventSynchronize(hev[j & 1]));
          sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - q4).count();
          if (trace)
            std::fprintf(stderr, "gmres it %lld: M %.3f A %.3f mgs %.3f sync %.3f ms%s\n", (long long)its, qm, qa, qg,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - q4).count(),
                         spec ? " (next enqueued)" : "");
          const double *hcol = hbuf[j & 1];
          double hn = hcol[j + 1];
          for (int64_t i = 0; i <= j; ++i) h(i, j) = hcol[i];
          if (!std::isfinite(hn)) throw value_error("GMRES residual is not finite");
          h(j + 1, j) = hn;
          for (int64_t i = 0; i < j; ++i) {
            double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
            h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
            h(i, j) = t;
          }
          double den = std::hypot(h(j, j), h(j + 1, j));
          if (den == 0.0) throw value_error("GMRES breakdown: zero Hessenberg column");
          cs[j] = h(j, j) / den;
          sn[j] = h(j + 1, j) / den;
          h(j, j) = den;
          h(j + 1, j) = 0.0;
          gg[j + 1] = -sn[j] * gg[j];
          gg[j] = cs[j] * gg[j];
          its += 1;
          double rel = std::fabs(gg[j + 1]) / nb;
          res.push_back(rel);
          bool lucky = hn == 0.0;
          j += 1;
          if (rel <= tol || lucky) {
            lucky_stop = lucky;
            break;
          }
          if (j < m && !ahead) enqueue_step(j);
        }
        if (j > 0) {
          std::vector<double> y(j, 0.0);
          for (int64_t i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t q = i + 1; q < j; ++q) s += h(i, q) * y[q];
            y[i] = (gg[i] - s) / h(i, i);
          }
          CK(cudaMemcpyAsync(dy, y.data(), sizeof(double) * j, cudaMemcpyHostToDevice, ctx->s));
          k_combine<<<g, 256, 0, ctx->s>>>(V, dy, (int)j, n, w);
          M(w, z);
          k_add<<<g, 256, 0, ctx->s>>>(z, d_x, n);
          ctx->launches += 2;
          CK(cudaStreamSynchronize(ctx->s));  // dy host buffer lifetime
        }
        A(d_x, w);
        k_sub<<<g, 256, 0, ctx->s>>>(d_b, w, r, n);
        dot(r, r, S + 3, true);
        double tr = host_scalar(S + 3) / nb;
        if (!std::isfinite(tr)) throw value_error("GMRES residual is not finite");
        if (!res.empty()) res.back() = tr;
        if (tr <= tol || lucky_stop) conv = true;
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }
};

// Several right-hand sides in lockstep (BASELINE C5: 8 RHS, one factor). The
// preconditioner apply of all Krylov vectors of a step is one graph replay
// (apply_device_nv: the factor is read once per step, not once per vector);
// SpMV, Gram-Schmidt, the scalings and the host Givens recurrence run per
// right-hand side with GmresRun's kernels and launch shapes, so every
// solution and residual history is bit-identical to its one-vector solve.
struct GmresMulti {
  Ctx *ctx;
  const mfh_gmres_ops *ops;
  int64_t n;
  int nv;
  double sync_ms = 0.0;
  struct Rhs {
    double nb = 0.0;
    bool conv = false, lucky_stop = false;
    int64_t its = 0, m = 0, j = 0;
    std::vector<double> H, cs, sn, gg, res;
  };
  void run(const double *d_B, double *d_X, double tol, int64_t max_iter, int64_t restart, std::vector<Rhs> &st) {
    if (!(tol > 0.0 && tol < 1.0)) throw value_error("tol must lie in (0, 1)");
    if (max_iter < 1 || restart < 1) throw value_error("max_iter and restart must be positive");
    if (!ops->A || !ops->M) throw value_error("batched GMRES needs a device operator and a device factorization");
    if (nv < 1 || nv > 8) throw value_error("batched GMRES: 1..8 right-hand sides per group");
    GmresRun g{ctx, ops, n};
    st.assign(nv, Rhs{});
    const int64_t mcap = std::min(restart, max_iter);
    if (mcap > 2000) throw value_error("min(restart, max_iter) must be <= 2000");
    const int64_t HS = 2048;  // per-vector stride of the Hessenberg column / y areas
    // V [nv][mcap+1][n], w / r / z / x-work [nv][n], H and y [nv][HS], scalars [nv][8]
    const size_t need = sizeof(double) * ((size_t)nv * (size_t)n * (size_t)(mcap + 4) + (size_t)nv * (2 * HS + 8));
    auto chunk = ctx->pool.take(need);
    double *V = (double *)chunk.first, *w = V + (size_t)nv * n * (mcap + 1), *r = w + (size_t)nv * n,
           *z = r + (size_t)nv * n, *Hd = z + (size_t)nv * n, *Yd = Hd + nv * HS, *sc = Yd + nv * HS;
    const int64_t vs = n * (mcap + 1);  // V stride between right-hand sides
    double *hp = nullptr;
    CK(cudaMallocHost(&hp, sizeof(double) * (size_t)nv * (2 * HS + 8)));
    double *hH = hp, *hY = hp + nv * HS, *hS = hp + 2 * nv * HS;
    int gr = g.gridn();
    const MgsPlan mgs = mgs_plan(ctx->device, n);
    auto sync_read = [&](double *dst, const double *src, size_t bytes) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->s));
      auto t0 = std::chrono::steady_clock::now();
      CK(cudaStreamSynchronize(ctx->s));
      sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    auto cleanup = [&]() {
      cudaStreamSynchronize(ctx->s);
      ctx->pool.give(chunk);
      cudaFreeHost(hp);
    };
    auto B = [&](int v) { return d_B + (size_t)v * n; };
    auto X = [&](int v) { return d_X + (size_t)v * n; };
    auto W = [&](int v) { return w + (size_t)v * n; };
    auto R = [&](int v) { return r + (size_t)v * n; };
    auto Z = [&](int v) { return z + (size_t)v * n; };
    auto Vj = [&](int v, int64_t j) { return V + (size_t)v * vs + (size_t)j * n; };
    try {
      for (int v = 0; v < nv; ++v) {
        CK(cudaMemsetAsync(X(v), 0, sizeof(double) * n, ctx->s));
        g.dot(B(v), B(v), sc + 8 * v, true);
      }
      sync_read(hS, sc, sizeof(double) * 8 * nv);
      for (int v = 0; v < nv; ++v) {
        st[v].nb = hS[8 * v];
        if (st[v].nb == 0.0) {
          st[v].conv = true;
          st[v].res.push_back(0.0);
        }
      }
      auto active = [&](int v) { return !st[v].conv && st[v].its < max_iter; };
      while (true) {
        std::vector<int> C;
        for (int v = 0; v < nv; ++v)
          if (active(v)) C.push_back(v);
        if (C.empty()) break;
        for (int v : C) {
          op_apply_device(ops->A, X(v), W(v));
          k_sub<<<gr, 256, 0, ctx->s>>>(B(v), W(v), R(v), n);
          ctx->launches++;
          g.dot(R(v), R(v), sc + 8 * v + 1, true);
        }
        sync_read(hS, sc, sizeof(double) * 8 * nv);
        std::vector<int> run;
        for (int v : C) {
          Rhs &q = st[v];
          const double beta = hS[8 * v + 1];
          if (!std::isfinite(beta)) throw value_error("GMRES residual is not finite");
          if (beta / q.nb <= tol) {
            q.conv = true;
            if (q.res.empty()) q.res.push_back(beta / q.nb);
            continue;
          }
          q.m = std::min(restart, max_iter - q.its);
          q.H.assign((q.m + 1) * q.m, 0.0);
          q.cs.assign(q.m, 0.0);
          q.sn.assign(q.m, 0.0);
          q.gg.assign(q.m + 1, 0.0);
          q.gg[0] = beta;
          q.j = 0;
          q.lucky_stop = false;
          k_scale_inv<<<gr, 256, 0, ctx->s>>>(sc + 8 * v + 1, R(v), Vj(v, 0), n);
          ctx->launches++;
          run.push_back(v);
        }
        std::vector<int> cyc = run;  // right-hand sides of this cycle
        for (int64_t j = 0; !run.empty(); ++j) {
          // one replay applies M to column j of every right-hand side
          apply_device_nv(ops->M, nv, V + (size_t)j * n, vs, z, n);
          for (int v : run) {
            op_apply_device(ops->A, Z(v), W(v));
            launch_mgs(mgs, V + (size_t)v * vs, W(v), n, (int)j, Hd + v * HS, ctx->d_part, ctx->s);
            ctx->launches++;
          }
          CK(cudaMemcpy2DAsync(hH, sizeof(double) * HS, Hd, sizeof(double) * HS, sizeof(double) * (j + 2), nv,
                               cudaMemcpyDeviceToHost, ctx->s));
          {
            auto t0 = std::chrono::steady_clock::now();
            CK(cudaStreamSynchronize(ctx->s));
            sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
          }
          std::vector<int> next;
          for (int v : run) {
            Rhs &q = st[v];
            const int64_t m = q.m;
            auto h = [&](int64_t i, int64_t jc) -> double & { return q.H[i * m + jc]; };
            const double *hcol = hH + v * HS;
            const double hn = hcol[j + 1];
            for (int64_t i = 0; i <= j; ++i) h(i, j) = hcol[i];
            if (!std::isfinite(hn)) throw value_error("GMRES residual is not finite");
            h(j + 1, j) = hn;
            for (int64_t i = 0; i < j; ++i) {
              double t = q.cs[i] * h(i, j) + q.sn[i] * h(i + 1, j);
              h(i + 1, j) = -q.sn[i] * h(i, j) + q.cs[i] * h(i + 1, j);
              h(i, j) = t;
            }
            const double den = std::hypot(h(j, j), h(j + 1, j));
            if (den == 0.0) throw value_error("GMRES breakdown: zero Hessenberg column");
            q.cs[j] = h(j, j) / den;
            q.sn[j] = h(j + 1, j) / den;
            h(j, j) = den;
            h(j + 1, j) = 0.0;
            q.gg[j + 1] = -q.sn[j] * q.gg[j];
            q.gg[j] = q.cs[j] * q.gg[j];
            q.its += 1;
            const double rel = std::fabs(q.gg[j + 1]) / q.nb;
            q.res.push_back(rel);
            const bool lucky = hn == 0.0;
            q.j = j + 1;
            if (rel <= tol || lucky) {
              q.lucky_stop = lucky;
              continue;
            }
            if (j + 1 < m) {
              k_scale_inv<<<gr, 256, 0, ctx->s>>>(Hd + v * HS + j + 1, W(v), Vj(v, j + 1), n);
              ctx->launches++;
              next.push_back(v);
            }
          }
          run.swap(next);
        }
        // x += M (V y) for every right-hand side of the cycle; one replay for all
        bool any = false;
        for (int v : cyc) {
          Rhs &q = st[v];
          if (q.j == 0) continue;
          const int64_t m = q.m, jn = q.j;
          auto h = [&](int64_t i, int64_t jc) -> double & { return q.H[i * m + jc]; };
          double *y = hY + v * HS;
          for (int64_t i = jn - 1; i >= 0; --i) {
            double s2 = 0.0;
            for (int64_t c = i + 1; c < jn; ++c) s2 += h(i, c) * y[c];
            y[i] = (q.gg[i] - s2) / h(i, i);
          }
          CK(cudaMemcpyAsync(Yd + v * HS, y, sizeof(double) * jn, cudaMemcpyHostToDevice, ctx->s));
          k_combine<<<gr, 256, 0, ctx->s>>>(V + (size_t)v * vs, Yd + v * HS, (int)jn, n, W(v));
          ctx->launches++;
          any = true;
        }
        if (any) {
          apply_device_nv(ops->M, nv, w, n, z, n);
          for (int v : cyc)
            if (st[v].j > 0) {
              k_add<<<gr, 256, 0, ctx->s>>>(Z(v), X(v), n);
              ctx->launches++;
            }
        }
        for (int v : cyc) {
          op_apply_device(ops->A, X(v), W(v));
          k_sub<<<gr, 256, 0, ctx->s>>>(B(v), W(v), R(v), n);
          ctx->launches++;
          g.dot(R(v), R(v), sc + 8 * v + 3, true);
        }
        sync_read(hS, sc, sizeof(double) * 8 * nv);
        for (int v : cyc) {
          Rhs &q = st[v];
          const double tr = hS[8 * v + 3] / q.nb;
          if (!std::isfinite(tr)) throw value_error("GMRES residual is not finite");
          if (!q.res.empty()) q.res.back() = tr;
          if (tr <= tol || q.lucky_stop) q.conv = true;
        }
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }
};

}  // namespace mfh

// ---------------------------------------------------------------------------
// distributed GMRES on a sharded factorization: every rank holds
// the rows / vector entries of the pivots it owns (permuted numbering); SpMV
// reads the other ranks' values it couples to from an all-reduced halo buffer
// (by the separator property: pivots of ancestor separators); Gram-Schmidt is
// classical, twice (CGS2: one all-reduce of j + 1 dots per pass instead of one
// per projection, as stable as the reference's MGS); norms all-reduced; the
// preconditioner is the sharded apply. Givens on the host, identical on every
// rank (the Hessenberg column is the same after the all-reduce).
// ---------------------------------------------------------------------------
struct DistSys {
  int64_t n = 0, nl = 0, nh = 0;            // global size, local rows, halo buffer length
  long long *lpos = nullptr;                // local row -> original index (for b / x)
  long long *ptr = nullptr;                 // local CSR
  int *col = nullptr;
  double *val = nullptr;
  long long *hown_pos = nullptr, *hown_loc = nullptr;  // halo entries this rank owns: buffer slot, local index
  int64_t nhown = 0;
  int W = 8;
  SpmvStream stream;  // streamed SpMV plan of the local CSR
  ~DistSys() {
    for (void *q : {(void *)lpos, (void *)ptr, (void *)col, (void *)val, (void *)hown_pos, (void *)hown_loc,
                    (void *)stream.ptr32})
      cudaFree(q);
  }
};

static std::unique_ptr<DistSys> dist_build(mfh_factor *F, int64_t n, const int64_t *ip, const int64_t *ix,
                                           const double *vx) {
  Ctx *ctx = F->ctx;
  auto D = std::make_unique<DistSys>();
  D->n = n;
  // owner of every permuted id, from the fronts' pivot runs (identical on every rank)
  std::vector<int> own((size_t)std::max<int64_t>(1, n), -1);
  for (size_t q = 0; q < F->fronts.size(); ++q) {
    const FrontH &f = F->fronts[q];
    for (int j = 0; j < f.npv; ++j) own[f.piv_lo + j] = F->owner[q];
  }
  std::vector<int64_t> iperm((size_t)std::max<int64_t>(1, n));
  for (int64_t i = 0; i < n; ++i) iperm[F->perm[i]] = i;
  // local rows: owned permuted ids ascending
  std::vector<int64_t> loc((size_t)std::max<int64_t>(1, n), -1), rows;
  for (int64_t g = 0; g < n; ++g)
    if (own[g] == F->rank) {
      loc[g] = (int64_t)rows.size();
      rows.push_back(g);
    }
  D->nl = (int64_t)rows.size();
  // halo: every id some rank reads but does not own (all ranks compute the same list)
  std::vector<int64_t> hidx((size_t)std::max<int64_t>(1, n), -1), hall;
  for (int64_t i = 0; i < n; ++i) {
    const int r = own[F->perm[i]];
    for (int64_t p = ip[i]; p < ip[i + 1]; ++p) {
      const int64_t gc = F->perm[ix[p]];
      if (own[gc] != r && hidx[gc] < 0) hidx[gc] = 1;
    }
  }
  for (int64_t g = 0; g < n; ++g)
    if (hidx[g] >= 0) {
      hidx[g] = (int64_t)hall.size();
      hall.push_back(g);
    }
  D->nh = (int64_t)hall.size();
  std::vector<long long> lp(D->nl + 1, 0), lpos(std::max<int64_t>(1, D->nl));
  std::vector<int> lc;
  std::vector<double> lv;
  for (int64_t l = 0; l < D->nl; ++l) {
    const int64_t i = iperm[rows[l]];
    lpos[l] = i;
    for (int64_t p = ip[i]; p < ip[i + 1]; ++p) {
      const int64_t gc = F->perm[ix[p]];
      lc.push_back(own[gc] == F->rank ? (int)loc[gc] : (int)(D->nl + hidx[gc]));
      lv.push_back(vx[p]);
    }
    lp[l + 1] = (long long)lc.size();
  }
  std::vector<long long> hp, hl;
  for (int64_t s2 = 0; s2 < D->nh; ++s2)
    if (own[hall[s2]] == F->rank) {
      hp.push_back(s2);
      hl.push_back(loc[hall[s2]]);
    }
  D->nhown = (int64_t)hp.size();
  const double avg = D->nl ? (double)lc.size() / D->nl : 0.0;
  D->W = avg <= 4.5 ? 4 : (avg <= 9.5 ? 8 : (avg <= 20 ? 16 : 32));
  spmv_stream_plan(ctx, D->nl, lp.data(), D->stream);
  // slack of the streamed SpMV's widened bulk copies
  lp.resize(lp.size() + 4, 0);
  lc.resize(lc.size() + 8, 0);
  lv.resize(lv.size() + 4, 0.0);
  auto upv = [&](auto **dst, const auto &v) {
    CK(cudaMalloc(dst, sizeof(v[0]) * std::max<size_t>(1, v.size())));
    upload(ctx->s, *dst, v.data(), sizeof(v[0]) * v.size());
  };
  upv(&D->lpos, lpos);
  upv(&D->ptr, lp);
  upv(&D->col, lc);
  upv(&D->val, lv);
  upv(&D->hown_pos, hp);
  upv(&D->hown_loc, hl);
  return D;
}

struct DistGmres {
  mfh_factor *F;
  Ctx *ctx;
  DistSys *D;
  double *halo = nullptr, *full = nullptr, *full2 = nullptr;  // halo buffer; full-length apply in / out
  double sync_ms = 0.0;
  int64_t allreduce_calls = 0;
  int g(int64_t n) const { return (int)std::min<int64_t>(cdiv(std::max<int64_t>(n, 1), 256), 148 * 8); }
  void allreduce(double *d, int64_t cnt) {
    allreduce_calls++;
    F->exchange_or_throw(d, cnt);
  }
  // y = A x on this rank's rows
  void A(const double *x, double *y) {
    const int64_t nl = D->nl;
    if (D->nh) {
      CK(cudaMemsetAsync(halo, 0, sizeof(double) * D->nh, ctx->s));
      if (D->nhown) {
        // halo[hown_pos[i]] = x[hown_loc[i]]
        double *tmp = full2;  // scratch: gathered owned halo values
        k_gather_from<<<g(D->nhown), 256, 0, ctx->s>>>(D->hown_loc, x, tmp, D->nhown);
        k_scatter_to<<<g(D->nhown), 256, 0, ctx->s>>>(D->hown_pos, tmp, halo, D->nhown);
        ctx->launches += 2;
      }
      allreduce(halo, D->nh);
    }
    static const bool no_stream = getenv("MFH_SPMV_NO_STREAM") != nullptr;
    if (D->stream.R > 0 && !no_stream) {
      spmv_stream_launch(ctx, D->stream, nl, D->ptr, D->col, D->val, x, D->nh ? halo : nullptr, (int)nl, y);
      return;
    }
    const int grid = (int)std::min<int64_t>(cdiv(std::max<int64_t>(1, nl) * D->W, 256), 148 * 16);
    switch (D->W) {
      case 4: k_spmv_dist<4><<<grid, 256, 0, ctx->s>>>(nl, D->ptr, D->col, D->val, x, halo, (int)nl, y); break;
      case 8: k_spmv_dist<8><<<grid, 256, 0, ctx->s>>>(nl, D->ptr, D->col, D->val, x, halo, (int)nl, y); break;
      case 16: k_spmv_dist<16><<<grid, 256, 0, ctx->s>>>(nl, D->ptr, D->col, D->val, x, halo, (int)nl, y); break;
      default: k_spmv_dist<32><<<grid, 256, 0, ctx->s>>>(nl, D->ptr, D->col, D->val, x, halo, (int)nl, y);
    }
    check_launch();
    ctx->launches++;
  }
  // y = M^{-1} x: the sharded apply on the full-length (original numbering) vector
  void M(const double *x, double *y) {
    const int64_t n = D->n, nl = D->nl;
    CK(cudaMemsetAsync(full, 0, sizeof(double) * n, ctx->s));
    if (nl) k_scatter_to<<<g(nl), 256, 0, ctx->s>>>(D->lpos, x, full, nl);
    apply_device(F, full, full);  // the plan copies in, applies (exchanges inside), copies out
    if (nl) k_gather_from<<<g(nl), 256, 0, ctx->s>>>(D->lpos, full, y, nl);
    ctx->launches += 2;
  }
  // out[0] = global x . y
  void dot(const double *x, const double *y, double *out) {
    k_dot_part<<<RED_BLOCKS, RED_THREADS, 0, ctx->s>>>(x, y, D->nl, ctx->d_part);
    k_finish<<<1, 32, 0, ctx->s>>>(ctx->d_part, out, 0);
    ctx->launches += 2;
    allreduce(out, 1);
  }
  double host(double *d) {
    CK(cudaMemcpyAsync(ctx->h_scal, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
    auto t0 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(ctx->s));
    sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return ctx->h_scal[0];
  }
  // b, x: host, full length, original numbering (every rank passes the same b, gets the same x)
  void run(const double *hb, double *hx, double tol, int64_t max_iter, int64_t restart, std::vector<double> &res,
           int64_t &its, bool &conv) {
    if (!(tol > 0.0 && tol < 1.0)) throw value_error("tol must lie in (0, 1)");
    if (max_iter < 1 || restart < 1) throw value_error("max_iter and restart must be positive");
    const int64_t n = D->n, nl = std::max<int64_t>(1, D->nl);
    res.clear();
    its = 0;
    conv = false;
    const int64_t mcap = std::min(restart, max_iter);
    if (mcap > 2000) throw value_error("min(restart, max_iter) must be <= 2000");
    auto chunk = ctx->pool.take(sizeof(double) * ((size_t)nl * (size_t)(mcap + 6) + 3 * (size_t)std::max<int64_t>(1, n) +
                                                  (size_t)std::max<int64_t>(1, D->nh) + 2 * 4096));
    double *V = (double *)chunk.first, *w = V + nl * (mcap + 1), *r = w + nl, *z = r + nl, *b = z + nl, *x = b + nl;
    full = x + nl;
    full2 = full + std::max<int64_t>(1, n);
    double *fin = full2 + std::max<int64_t>(1, n);  // full-length staging for b / x
    halo = fin + std::max<int64_t>(1, n);
    double *S = halo + std::max<int64_t>(1, D->nh);  // [0] |b|^2, [1] beta^2, [2] hn^2, [8..] h, [2048..] h2 / y
    auto cleanup = [&]() {
      cudaStreamSynchronize(ctx->s);
      ctx->pool.give(chunk);
    };
    try {
      CK(cudaMemcpyAsync(fin, hb, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->s));
      if (D->nl) k_gather_from<<<g(D->nl), 256, 0, ctx->s>>>(D->lpos, fin, b, D->nl);
      CK(cudaMemsetAsync(x, 0, sizeof(double) * nl, ctx->s));
      dot(b, b, S);
      const double nb = std::sqrt(host(S));
      if (nb == 0.0) {
        conv = true;
        res.push_back(0.0);
      }
      while (!conv && its < max_iter) {
        A(x, w);
        k_sub<<<g(nl), 256, 0, ctx->s>>>(b, w, r, D->nl);
        dot(r, r, S + 1);
        const double beta = std::sqrt(host(S + 1));
        if (!std::isfinite(beta)) throw value_error("GMRES residual is not finite");
        if (beta / nb <= tol) {
          conv = true;
          if (res.empty()) res.push_back(beta / nb);
          break;
        }
        const int64_t m = std::min(restart, max_iter - its);
        std::vector<double> H((m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), gg(m + 1, 0.0);
        auto h = [&](int64_t i, int64_t j) -> double & { return H[i * m + j]; };
        gg[0] = beta;
        {
          const double inv = beta;
          CK(cudaMemcpyAsync(S + 4, &inv, sizeof(double), cudaMemcpyHostToDevice, ctx->s));
          k_scale_inv<<<g(nl), 256, 0, ctx->s>>>(S + 4, r, V, D->nl);
        }
        int64_t j = 0;
        bool lucky_stop = false;
        std::vector<double> hc(m + 2);
        while (j < m) {
          double *vj = V + j * nl;
          M(vj, z);
          A(z, w);
          // CGS2: h = V^T w; w -= V h; h2 = V^T w; w -= V h2; h += h2
          double *hd = S + 8, *h2 = S + 2048;
          k_multi_dot<<<(unsigned)(j + 1), 256, 0, ctx->s>>>(V, w, D->nl, hd, 0);
          allreduce(hd, j + 1);
          k_sub_vh<<<g(nl), 256, 0, ctx->s>>>(V, hd, (int)(j + 1), D->nl, w);
          k_multi_dot<<<(unsigned)(j + 1), 256, 0, ctx->s>>>(V, w, D->nl, h2, 0);
          allreduce(h2, j + 1);
          k_sub_vh<<<g(nl), 256, 0, ctx->s>>>(V, h2, (int)(j + 1), D->nl, w);
          k_add<<<1, 256, 0, ctx->s>>>(h2, hd, j + 1);
          ctx->launches += 5;
          dot(w, w, S + 2);
          CK(cudaMemcpyAsync(hc.data(), hd, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, ctx->s));
          const double hn = std::sqrt(host(S + 2));
          for (int64_t i = 0; i <= j; ++i) h(i, j) = hc[i];
          if (!std::isfinite(hn)) throw value_error("GMRES residual is not finite");
          h(j + 1, j) = hn;
          for (int64_t i = 0; i < j; ++i) {
            const double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
            h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
            h(i, j) = t;
          }
          const double den = std::hypot(h(j, j), h(j + 1, j));
          if (den == 0.0) throw value_error("GMRES breakdown: zero Hessenberg column");
          cs[j] = h(j, j) / den;
          sn[j] = h(j + 1, j) / den;
          h(j, j) = den;
          h(j + 1, j) = 0.0;
          gg[j + 1] = -sn[j] * gg[j];
          gg[j] = cs[j] * gg[j];
          its += 1;
          const double rel = std::fabs(gg[j + 1]) / nb;
          res.push_back(rel);
          const bool lucky = hn == 0.0;
          j += 1;
          if (rel <= tol || lucky) {
            lucky_stop = lucky;
            break;
          }
          CK(cudaMemcpyAsync(S + 5, &hn, sizeof(double), cudaMemcpyHostToDevice, ctx->s));
          k_scale_inv<<<g(nl), 256, 0, ctx->s>>>(S + 5, w, V + j * nl, D->nl);
          CK(cudaStreamSynchronize(ctx->s));  // the host scalars above are pageable
        }
        if (j > 0) {
          std::vector<double> y(j, 0.0);
          for (int64_t i = j - 1; i >= 0; --i) {
            double s2 = 0.0;
            for (int64_t q = i + 1; q < j; ++q) s2 += h(i, q) * y[q];
            y[i] = (gg[i] - s2) / h(i, i);
          }
          double *dy = S + 2048;
          CK(cudaMemcpyAsync(dy, y.data(), sizeof(double) * j, cudaMemcpyHostToDevice, ctx->s));
          k_combine<<<g(nl), 256, 0, ctx->s>>>(V, dy, (int)j, D->nl, w);
          M(w, z);
          k_add<<<g(nl), 256, 0, ctx->s>>>(z, x, D->nl);
          CK(cudaStreamSynchronize(ctx->s));
        }
        A(x, w);
        k_sub<<<g(nl), 256, 0, ctx->s>>>(b, w, r, D->nl);
        dot(r, r, S + 3);
        const double tr = std::sqrt(host(S + 3)) / nb;
        if (!std::isfinite(tr)) throw value_error("GMRES residual is not finite");
        if (!res.empty()) res.back() = tr;
        if (tr <= tol || lucky_stop) conv = true;
      }
      // every rank gets the whole solution (disjoint entries, exact sum)
      CK(cudaMemsetAsync(fin, 0, sizeof(double) * n, ctx->s));
      if (D->nl) k_scatter_to<<<g(D->nl), 256, 0, ctx->s>>>(D->lpos, x, fin, D->nl);
      allreduce(fin, n);
      CK(cudaMemcpyAsync(hx, fin, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->s));
      CK(cudaStreamSynchronize(ctx->s));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }
};

static int gmres_common(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, const double *d_b, double *d_x,
                        double tol, int64_t max_iter, int64_t restart, double *hist, int64_t *n_hist,
                        int64_t *iterations, int *converged) {
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  GmresRun g{&ctx->c, ops, n};
  std::vector<double> res;
  int64_t its = 0;
  bool conv = false;
  auto tg0 = std::chrono::steady_clock::now();
  g.run(d_b, d_x, tol, max_iter, restart, res, its, conv);
  if (ops->M) {
    ops->M->timing.gmres_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg0).count();
    ops->M->timing.gmres_apply_ms = g.m_ms;
    ops->M->timing.gmres_sync_ms = g.sync_ms;
  }
  if (hist) std::memcpy(hist, res.data(), sizeof(double) * res.size());
  *n_hist = (int64_t)res.size();
  *iterations = its;
  *converged = conv ? 1 : 0;
  MFH_CATCH
}

extern "C" int mfh_gmres_device(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, const double *d_b,
                                double *d_x, double tol, int64_t max_iter, int64_t restart, double *hist,
                                int64_t *n_hist, int64_t *iterations, int *converged) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  return gmres_common(ctx, ops, n, d_b, d_x, tol, max_iter, restart, hist, n_hist, iterations, converged);
}

extern "C" int mfh_gmres(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, const double *b, double *x,
                         double tol, int64_t max_iter, int64_t restart, double *hist, int64_t *n_hist,
                         int64_t *iterations, int *converged) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  cudaStream_t s = ctx->c.s;
  std::pair<char *, size_t> chunk{nullptr, 0};
  try {
    chunk = ctx->c.pool.take(sizeof(double) * 2 * (size_t)std::max<int64_t>(1, n));
  } catch (const std::exception &e) {
    set_last_error(std::string("CUDA allocation failed in mfh_gmres: ") + e.what());
    return MFH_ERUNTIME;
  }
  double *db = (double *)chunk.first, *dx = db + std::max<int64_t>(1, n);
  cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  int rc = gmres_common(ctx, ops, n, db, dx, tol, max_iter, restart, hist, n_hist, iterations, converged);
  if (rc == MFH_OK) cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  ctx->c.pool.give(chunk);
  return rc;
}

// Several right-hand sides (vector r at b + r n), groups of up to eight in
// lockstep; per right-hand side: history row r of hist (hist_cap entries),
// n_hist[r], iterations[r], converged[r]. Device operator and factor only.
static int gmres_batched_common(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, int64_t nrhs, const double *d_b,
                                double *d_x, double tol, int64_t max_iter, int64_t restart, double *hist,
                                int64_t hist_cap, int64_t *n_hist, int64_t *iterations, int *converged) {
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  if (nrhs < 0) throw value_error("nrhs must be non-negative");
  auto tg0 = std::chrono::steady_clock::now();
  double sync_ms = 0.0;
  for (int64_t r0 = 0; r0 < nrhs; r0 += 8) {
    const int nv = (int)std::min<int64_t>(8, nrhs - r0);
    GmresMulti g{&ctx->c, ops, n, nv};
    std::vector<GmresMulti::Rhs> st;
    g.run(d_b + r0 * n, d_x + r0 * n, tol, max_iter, restart, st);
    sync_ms += g.sync_ms;
    for (int v = 0; v < nv; ++v) {
      const int64_t r = r0 + v;
      const auto &q = st[v];
      const int64_t nh = (int64_t)q.res.size();
      if (hist) std::memcpy(hist + r * hist_cap, q.res.data(), sizeof(double) * std::min(nh, hist_cap));
      n_hist[r] = nh;
      iterations[r] = q.its;
      converged[r] = q.conv ? 1 : 0;
    }
  }
  if (ops->M) {
    ops->M->timing.gmres_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg0).count();
    ops->M->timing.gmres_sync_ms = sync_ms;
  }
  MFH_CATCH
}

extern "C" int mfh_gmres_batched_device(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, int64_t nrhs,
                                        const double *d_b, double *d_x, double tol, int64_t max_iter,
                                        int64_t restart, double *hist, int64_t hist_cap, int64_t *n_hist,
                                        int64_t *iterations, int *converged) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  return gmres_batched_common(ctx, ops, n, nrhs, d_b, d_x, tol, max_iter, restart, hist, hist_cap, n_hist,
                              iterations, converged);
}

extern "C" int mfh_gmres_sharded(mfh_factor *F, int64_t n, const int64_t *indptr, const int64_t *indices,
                                 const double *values, const double *b, double *x, double tol, int64_t max_iter,
                                 int64_t restart, double *hist, int64_t *n_hist, int64_t *iterations, int *converged) {
  std::lock_guard<std::recursive_mutex> lk_(F->ctx->mu);
  MFH_TRY
  DeviceGuard dg_(F->ctx->device);
  if (!F->sharded) throw value_error("mfh_gmres_sharded needs a factorization from mfh_factorize_sharded");
  if (n != F->n) throw value_error("dimension mismatch: system is " + std::to_string(F->n) + ", rhs is " + std::to_string(n));
  auto D = dist_build(F, n, indptr, indices, values);
  DistGmres g{F, F->ctx, D.get()};
  std::vector<double> res;
  int64_t its = 0;
  bool conv = false;
  auto t0 = std::chrono::steady_clock::now();
  g.run(b, x, tol, max_iter, restart, res, its, conv);
  F->timing.gmres_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  F->timing.gmres_sync_ms = g.sync_ms;
  if (hist) std::memcpy(hist, res.data(), sizeof(double) * res.size());
  *n_hist = (int64_t)res.size();
  *iterations = its;
  *converged = conv ? 1 : 0;
  MFH_CATCH
}

extern "C" int mfh_gmres_batched(mfh_ctx *ctx, const mfh_gmres_ops *ops, int64_t n, int64_t nrhs, const double *b,
                                 double *x, double tol, int64_t max_iter, int64_t restart, double *hist,
                                 int64_t hist_cap, int64_t *n_hist, int64_t *iterations, int *converged) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  cudaStream_t s = ctx->c.s;
  std::pair<char *, size_t> chunk{nullptr, 0};
  const size_t len = (size_t)std::max<int64_t>(1, n * std::max<int64_t>(1, nrhs));
  try {
    chunk = ctx->c.pool.take(sizeof(double) * 2 * len);
  } catch (const std::exception &e) {
    set_last_error(std::string("CUDA allocation failed in mfh_gmres_batched: ") + e.what());
    return MFH_ERUNTIME;
  }
  double *db = (double *)chunk.first, *dx = db + len;
  cudaMemcpyAsync(db, b, sizeof(double) * n * nrhs, cudaMemcpyHostToDevice, s);
  int rc = gmres_batched_common(ctx, ops, n, nrhs, db, dx, tol, max_iter, restart, hist, hist_cap, n_hist,
                                iterations, converged);
  if (rc == MFH_OK) cudaMemcpyAsync(x, dx, sizeof(double) * n * nrhs, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  ctx->c.pool.give(chunk);
  return rc;
}

// ---------------------------------------------------------------------------
// kernel plugin: batched full_pivot_lu (_core.pyx:23-86)
// ---------------------------------------------------------------------------
extern "C" int mfh_full_pivot_lu_batched(mfh_ctx *ctx, int64_t batch, const int64_t *offs, const int64_t *ms,
                                         const int64_t *ns, double *blocks, int64_t total, double eps,
                                         const int64_t *max_ranks, int64_t *row_perm, int64_t *col_perm,
                                         int64_t *ranks, double *ratios, int64_t *status, double *err) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  Ctx *c = &ctx->c;
  if (batch == 0) return MFH_OK;
  double *d_blocks = c->scratch.d(std::max<int64_t>(1, total));
  CK(cudaMemcpyAsync(d_blocks, blocks, sizeof(double) * total, cudaMemcpyHostToDevice, c->s));
  std::vector<PluJob> jobs(batch);
  std::vector<int64_t> ioff(batch), doff(batch);
  int64_t itot = 0, dtot = 0;
  for (int64_t b = 0; b < batch; ++b) {
    ioff[b] = itot;
    doff[b] = dtot;
    itot += 4 * (ms[b] + ns[b]) + 4;
    dtot += ms[b] + ns[b] + 3;
  }
  int *ibuf = c->scratch.i(std::max<int64_t>(1, itot));
  double *dbuf = c->scratch.d(std::max<int64_t>(1, dtot));
  for (int64_t b = 0; b < batch; ++b) {
    PluJob &j = jobs[b];
    int m = (int)ms[b], n = (int)ns[b];
    j.a = d_blocks + offs[b];
    j.m = m;
    j.n = n;
    j.ld = n;
    j.kmax = (int)std::min<int64_t>(std::min(m, n), max_ranks[b]);
    int *p = ibuf + ioff[b];
    j.rowAt = p;
    j.posR = p + m;
    j.actR = p + 2 * m;
    j.idxR = p + 3 * m;
    p += 4 * m;
    j.colAt = p;
    j.posC = p + n;
    j.actC = p + 2 * n;
    j.idxC = p + 3 * n;
    p += 4 * n;
    j.out = p;
    j.mult = dbuf + doff[b];
    j.prow = dbuf + doff[b] + m;
    j.outd = dbuf + doff[b] + m + n;
  }
  Sink s{c};
  run_plu(s, jobs, eps);
  std::vector<int> hi(itot);
  std::vector<double> hd(dtot);
  CK(cudaMemcpyAsync(hi.data(), ibuf, sizeof(int) * itot, cudaMemcpyDeviceToHost, c->s));
  CK(cudaMemcpyAsync(hd.data(), dbuf, sizeof(double) * dtot, cudaMemcpyDeviceToHost, c->s));
  std::vector<double> raw(total);
  CK(cudaMemcpyAsync(raw.data(), d_blocks, sizeof(double) * total, cudaMemcpyDeviceToHost, c->s));
  CK(cudaStreamSynchronize(c->s));
  c->scratch.reset();
  c->stage.rewind();
  int64_t ro = 0, co = 0;
  for (int64_t b = 0; b < batch; ++b) {
    int m = (int)ms[b], n = (int)ns[b];
    const int *p = hi.data() + ioff[b];
    const int *rowAt = p, *colAt = p + 4 * m;
    const int *out = p + 4 * m + 4 * n;
    const double *od = hd.data() + doff[b] + m + n;
    ranks[b] = out[0];
    status[b] = out[1];
    ratios[b] = od[0];
    err[3 * b] = out[2];
    err[3 * b + 1] = od[1];
    err[3 * b + 2] = od[2];
    for (int i = 0; i < m; ++i) row_perm[ro + i] = rowAt[i];
    for (int j = 0; j < n; ++j) col_perm[co + j] = colAt[j];
    // reference layout: lu[p][q] = a[row at position p][q] (columns already physical)
    const double *a = raw.data() + offs[b];
    double *o = blocks + offs[b];
    const bool phys = out[3] == 1;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) o[(int64_t)i * n + j] = a[(int64_t)(phys ? i : rowAt[i]) * n + j];
    ro += m;
    co += n;
  }
  MFH_CATCH
}

// ---------------------------------------------------------------------------
// test hook: the factorization's explicit-inverse dispatch (run_inverse) on a
// host batch of square row-major blocks; singular[i] = 1 where a pivot was
// zero / non-finite (the reference's LU diagonal checks)
// ---------------------------------------------------------------------------
extern "C" int mfh_test_inverse_batched(mfh_ctx *ctx, int64_t batch, const int64_t *offs, const int64_t *ns,
                                        double *blocks, int64_t total, int *singular) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  Ctx *c = &ctx->c;
  if (batch == 0) return MFH_OK;
  double *d_blocks = c->scratch.d(std::max<int64_t>(1, total));
  double *d_out = c->scratch.d(std::max<int64_t>(1, total));
  int64_t ptot = 0;
  for (int64_t b = 0; b < batch; ++b) ptot += ns[b];
  int *d_piv = c->scratch.i(std::max<int64_t>(1, ptot));
  int *d_flag = c->scratch.i(std::max<int64_t>(1, batch));
  CK(cudaMemcpyAsync(d_blocks, blocks, sizeof(double) * total, cudaMemcpyHostToDevice, c->s));
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int) * batch, c->s));
  std::vector<InvReq> reqs;
  int64_t po = 0;
  for (int64_t b = 0; b < batch; ++b) {
    int n = (int)ns[b];
    if (n < 1) throw value_error("block sizes must be positive");
    reqs.push_back(InvReq{d_blocks + offs[b], n, n, d_out + offs[b], n, d_piv + po, d_flag + b});
    po += n;
  }
  Sink s{c};
  run_inverse(s, reqs);
  std::vector<int> hf(batch);
  CK(cudaMemcpyAsync(blocks, d_out, sizeof(double) * total, cudaMemcpyDeviceToHost, c->s));
  CK(cudaMemcpyAsync(hf.data(), d_flag, sizeof(int) * batch, cudaMemcpyDeviceToHost, c->s));
  CK(cudaStreamSynchronize(c->s));
  c->scratch.reset();
  c->stage.rewind();
  for (int64_t b = 0; b < batch; ++b) singular[b] = hf[b];
  MFH_CATCH
}

// test hook: the factorization's batched GEMM dispatch (run_gemm: DMMA tiles,
// identity strips, split-K, cuBLAS for the large plain ones) on a host
// workspace. Job q: C = alpha A B + beta C with A at buf + ao[q] (m x k, lda),
// B at buf + bo[q] (k x n, ldb), C at buf + co[q] (m x n, ldc), all offsets in
// one buffer so aliasing jobs (C == B, disjoint blocks of one buffer) can be
// expressed; a negative offset -1 selects the identity strip (ld -1).
extern "C" int mfh_test_gemm_batched(mfh_ctx *ctx, int64_t batch, const int64_t *desc /* 9 per job */,
                                     const double *ab /* alpha, beta per job */, double *buf, int64_t total,
                                     int split_k) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  Ctx *c = &ctx->c;
  if (batch == 0) return MFH_OK;
  int maxdim = 1;
  for (int64_t q = 0; q < batch; ++q) maxdim = std::max<int>(maxdim, (int)std::max({desc[9 * q], desc[9 * q + 1], desc[9 * q + 2]}));
  double *d = c->scratch.d(std::max<int64_t>(1, total));
  double *strip = c->scratch.d((size_t)2 * maxdim - 1);
  CK(cudaMemsetAsync(strip, 0, sizeof(double) * (2 * maxdim - 1), c->s));
  static const double one = 1.0;
  CK(cudaMemcpyAsync(strip + maxdim - 1, &one, sizeof(double), cudaMemcpyHostToDevice, c->s));
  CK(cudaMemcpyAsync(d, buf, sizeof(double) * total, cudaMemcpyHostToDevice, c->s));
  std::vector<GemmJob> jobs;
  for (int64_t q = 0; q < batch; ++q) {
    const int64_t *t = desc + 9 * q;  // m n k ao bo co lda ldb ldc
    GemmJob g{};
    g.m = (int)t[0];
    g.n = (int)t[1];
    g.k = (int)t[2];
    g.A = t[3] < 0 ? strip + maxdim - 1 : d + t[3];
    g.B = t[4] < 0 ? strip + maxdim - 1 : d + t[4];
    g.C = d + t[5];
    g.lda = t[3] < 0 ? -1 : (int)t[6];
    g.ldb = t[4] < 0 ? -1 : (int)t[7];
    g.ldc = (int)t[8];
    g.alpha = ab[2 * q];
    g.beta = ab[2 * q + 1];
    jobs.push_back(g);
  }
  Sink s{c};
  // split_k -2 / -3 / -4: large plain GEMMs on k_gemm (64 x 64 tiles) / cuBLAS / k_gemm_big
  g_route_override = split_k == -2 ? 2 : (split_k == -3 ? 1 : (split_k == -4 ? 0 : -1));
  g_split_k_override = split_k < 0 ? 0 : split_k;
  try {
    run_gemm(s, jobs);
  } catch (...) {
    g_split_k_override = -1;
    g_route_override = -1;
    throw;
  }
  g_route_override = -1;
  g_split_k_override = -1;
  CK(cudaMemcpyAsync(buf, d, sizeof(double) * total, cudaMemcpyDeviceToHost, c->s));
  CK(cudaStreamSynchronize(c->s));
  c->scratch.reset();
  c->stage.rewind();
  MFH_CATCH
}

// Test hook: the apply's batched GEMV (k_gemv_tc, 1..8 right-hand sides) on one
// host workspace. Job q is desc[16q..16q+15] = (m, k1, k2, y, y0, A1, lda1, x1,
// A2, lda2, x2, idx2, ys, y0s, x1s, x2s): offsets into buf (y0 / A2 / idx2 -1 =
// none; idx2 is an offset into idx), ab[2q], ab[2q+1] = (a1, a2).
extern "C" int mfh_test_gemv_batched(mfh_ctx *ctx, int64_t batch, const int64_t *desc, const double *ab,
                                     double *buf, int64_t total, const int64_t *idx, int64_t nidx, int nv) {
  std::lock_guard<std::recursive_mutex> lk_(ctx->c.mu);
  MFH_TRY
  DeviceGuard dg_(ctx->c.device);
  Ctx *c = &ctx->c;
  if (batch == 0) return MFH_OK;
  double *d = c->scratch.d(std::max<int64_t>(1, total));
  long long *di = (long long *)c->scratch.alloc(sizeof(long long) * std::max<int64_t>(1, nidx));
  CK(cudaMemcpyAsync(d, buf, sizeof(double) * total, cudaMemcpyHostToDevice, c->s));
  if (nidx) CK(cudaMemcpyAsync(di, idx, sizeof(long long) * nidx, cudaMemcpyHostToDevice, c->s));
  std::vector<GemvJob> jobs;
  for (int64_t q = 0; q < batch; ++q) {
    const int64_t *t = desc + 16 * q;
    GemvJob g{};
    g.m = (int)t[0];
    g.k1 = (int)t[1];
    g.k2 = (int)t[2];
    g.y = d + t[3];
    g.y0 = t[4] < 0 ? nullptr : d + t[4];
    g.A1 = d + t[5];
    g.lda1 = (int)t[6];
    g.x1 = d + t[7];
    g.A2 = t[8] < 0 ? nullptr : d + t[8];
    g.lda2 = (int)t[9];
    g.x2 = t[10] < 0 ? nullptr : d + t[10];
    g.idx2 = t[11] < 0 ? nullptr : di + t[11];
    g.ys = t[12];
    g.y0s = t[13];
    g.x1s = t[14];
    g.x2s = t[15];
    g.a1 = ab[2 * q];
    g.a2 = ab[2 * q + 1];
    jobs.push_back(g);
  }
  Sink s{c};
  run_gemv(s, jobs, nv);
  CK(cudaMemcpyAsync(buf, d, sizeof(double) * total, cudaMemcpyDeviceToHost, c->s));
  CK(cudaStreamSynchronize(c->s));
  c->scratch.reset();
  c->stage.rewind();
  MFH_CATCH
}
