// Large-tile batched FP64 GEMM on the tensor cores (sm_100a; included by kernels.cuh).
//
// C = alpha * A (m x k) * B (k x n) + beta * C, row-major with leading dimensions, for the plain
// GEMMs of the HODLR levels, eliminations and dense fronts whose size used to send them to the
// library (hodlr.py:330-352, multifrontal.py:283-310, 411-456). One persistent launch covers every
// job of a batch: CTAs walk a host-built tile list, so a level's few medium products fill the GPU
// together instead of running one library call after another.
//
//   CTA tile  BM x BN = (WM * FA * 8) x (WN * FB * 8), 8 warps as WM x WN, warp tile (FA * 8) x (FB * 8)
//   k slab    16, STG - 2 slabs in flight by 16-byte cp.async (8-byte copies when an operand's
//             rows are not 16-byte aligned); src-size clamps zero-fill rows / columns / k outside the
//             job; per-stage full / empty mbarriers, no CTA barrier in the k loop
//   A slab    [BM][16 + 4], B slab [16][BN + 4]: the m8n8k4 fragment loads (lane = 4 g + q reads
//             A[g][q], B[q][g]) are bank-conflict free with these pitches
//   math      mma.sync m8n8k4 f64: per output entry one k-ascending chain of fused 4-term steps, the
//             same chain k_gemm and the sampler run, so the three agree bit for bit on a job
#pragma once

namespace mfh {

constexpr int GB_BK = 16, GB_LDA = GB_BK + 4;

struct GemmBigTile {
  int job, mt, nt;
};

template <int WM, int WN, int FA, int FB, int STG>
struct GemmBigCfg {
  static constexpr int BM = WM * FA * 8, BN = WN * FB * 8, LDB = BN + 4;
  static constexpr int A_ELEMS = BM * GB_LDA, B_ELEMS = GB_BK * LDB;
  static constexpr size_t SMEM = sizeof(double) * STG * (A_ELEMS + B_ELEMS);
};

// 16-byte cp.async with a source size of 0, 8 or 16 bytes (the rest of the 16 is zero-filled)
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gsrc), "r"(src_bytes) : "memory");
}

// every cp.async this thread issued so far arrives on the barrier when it lands (.noinc: it
// counts against the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int WM, int WN, int FA, int FB, int STG, int MINB>
__global__ void __launch_bounds__(WM * WN * 32, MINB) k_gemm_big(const GemmJob *__restrict__ jobs,
                                                                 const GemmBigTile *__restrict__ tiles, int ntiles) {
  using Cfg = GemmBigCfg<WM, WN, FA, FB, STG>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, LDB = Cfg::LDB, GB_STG = STG;
  constexpr int NT = WM * WN * 32;  // 8 or 16 warps
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double gb_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN, g = lane >> 2, q = lane & 3;
  auto Ast = [&](int s) { return gb_smem + (size_t)s * (Cfg::A_ELEMS + Cfg::B_ELEMS); };
  auto Bst = [&](int s) { return gb_smem + (size_t)s * (Cfg::A_ELEMS + Cfg::B_ELEMS) + Cfg::A_ELEMS; };
  // Slab pipeline without CTA barriers: full[s] completes when every thread's copies of the slab
  // in stage s have landed, empty[s] when every warp has multiplied it. Slabs are prefetched
  // GB_PD = STG - 2 ahead, so the stage a warp overwrites was released a whole slab earlier and
  // warps drift up to a slab apart instead of meeting at a barrier every 16 k. The slab counter
  // runs across the CTA's tiles (stage = counter % STG, parity = (counter / STG) & 1).
  // (Measured alternatives on B200, 4096^3: CTA barrier per slab 32.4 TFLOP/s, this 33.1; one
  // dedicated copy warp 22.3 (it cannot issue a slab's 128 copies per lane in a slab's time);
  // 16 warps with 32 x 32 warp tiles 31.3; cuBLAS 35.2.)
  constexpr int GB_PD = STG - 2;
  static_assert(GB_PD >= 1, "at least three stages");
  __shared__ unsigned long long full_bar[STG], empty_bar[STG];
  if (tid == 0) {
    for (int i = 0; i < STG; ++i) {
      mbar_init(&full_bar[i], NT);
      mbar_init(&empty_bar[i], WM * WN);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned gc = 0;  // slabs this CTA has consumed before the current tile
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const GemmBigTile tl = tiles[t];
    const GemmJob J = jobs[tl.job];
    const int m0 = tl.mt * BM, n0 = tl.nt * BN, K = J.k;
    const bool a16 = ((((unsigned long long)J.A) & 15) == 0) && (J.lda % 2 == 0);
    const bool b16 = ((((unsigned long long)J.B) & 15) == 0) && (J.ldb % 2 == 0);
    double acc[FA][FB][2];
#pragma unroll
    for (int a = 0; a < FA; ++a)
#pragma unroll
      for (int j = 0; j < FB; ++j) acc[a][j][0] = acc[a][j][1] = 0.0;
    const int nsl = (K + GB_BK - 1) / GB_BK;
    // Copies of a slab, one part per fragment step (part i = the thread's i-th A chunk and B chunk),
    // so the address arithmetic and the cp.async issue sit between the DMMA groups instead of in
    // front of them. Per thread: A chunk (row (tid >> 3) + RSTEP i, k pair tid & 7), B chunk
    // (k row (tid / (BN / 2)) + KSTEP i, column pair tid % (BN / 2)).
    constexpr int NA = BM * 8 / NT, NB = GB_BK * (BN / 2) / NT, KSTEP = 2 * NT / BN, RSTEP = NT / 8;
    static_assert(NA <= GB_BK / 4 && NB <= GB_BK / 4, "one chunk of each operand per fragment step");
    const int ar = tid >> 3, ach = tid & 7, bk = tid / (BN / 2), bch = tid % (BN / 2);
    const double *pa = J.A + (long long)(m0 + ar) * J.lda + 2 * ach;
    const double *pb = J.B + (long long)bk * J.ldb + n0 + 2 * bch;
    const long long sa = (long long)RSTEP * J.lda, sb = (long long)KSTEP * J.ldb;
    const int bleft = min(max(J.n - (n0 + 2 * bch), 0), 2);
    unsigned avalid = 0;  // bit i: the thread's i-th A row lies inside the job
#pragma unroll
    for (int i = 0; i < NA; ++i) avalid |= (m0 + ar + RSTEP * i < J.m) ? (1u << i) : 0u;
    auto issue_part = [&](int c, int i) {
      const int k0 = c * GB_BK;
      const bool full = k0 + GB_BK <= K;  // only the last slab of a job clamps in k
      const unsigned st = (gc + c) % GB_STG;
      double *As = Ast(st), *Bs = Bst(st);
      if (i < NA) {
        int left = ((avalid >> i) & 1u) ? 2 : 0;
        if (!full) left = min(max(K - (k0 + 2 * ach), 0), left);
        const double *src = left ? pa + i * sa + k0 : J.A;
        double *dst = As + (ar + RSTEP * i) * GB_LDA + 2 * ach;
        if (a16) {
          cp_async16(dst, src, 8 * left);
        } else {
          cp_async8(dst, src, left >= 1);
          cp_async8(dst + 1, left >= 2 ? src + 1 : J.A, left >= 2);
        }
      }
      if (i < NB) {
        const int kk = bk + KSTEP * i;
        const int left = (full || k0 + kk < K) ? bleft : 0;
        const double *src = left ? pb + i * sb + (long long)k0 * J.ldb : J.B;
        double *dst = Bs + kk * LDB + 2 * bch;
        if (b16) {
          cp_async16(dst, src, 8 * left);
        } else {
          cp_async8(dst, src, left >= 1);
          cp_async8(dst + 1, left >= 2 ? src + 1 : J.B, left >= 2);
        }
      }
    };
    // wait until the stage slab c goes into has been released by every warp
    auto wait_empty = [&](int c) {
      const unsigned u = gc + c;
      if (u >= GB_STG) mbar_wait(&empty_bar[u % GB_STG], ((u / GB_STG) + 1) & 1);
    };
#pragma unroll
    for (int c = 0; c < GB_PD; ++c) {
      if (c < nsl) {
        wait_empty(c);
#pragma unroll
        for (int i = 0; i < GB_BK / 4; ++i) issue_part(c, i);
        cp_async_mbar_arrive(&full_bar[(gc + c) % GB_STG]);
      }
    }
    // The warps of a scheduler (warp, warp + 4, ...) run out of phase: one issues its copies
    // before a DMMA group, the other after it, so one of them always feeds the FP64 tensor pipe.
    const bool late = (warp >> 2) & 1;
    for (int c = 0; c < nsl; ++c) {
      const unsigned u = gc + c, st = u % GB_STG;
      const bool produce = c + GB_PD < nsl;
      mbar_wait(&full_bar[st], (u / GB_STG) & 1);
      if (produce) wait_empty(c + GB_PD);
      const double *As = Ast(st) + (wm * FA * 8 + g) * GB_LDA + q;
      const double *Bs = Bst(st) + q * LDB + wn * FB * 8 + g;
#pragma unroll
      for (int kb = 0; kb < GB_BK / 4; ++kb) {
        double fa[FA], fb[FB];
#pragma unroll
        for (int a = 0; a < FA; ++a) fa[a] = As[a * 8 * GB_LDA + 4 * kb];
#pragma unroll
        for (int j = 0; j < FB; ++j) fb[j] = Bs[4 * kb * LDB + 8 * j];
        if (produce && !late) issue_part(c + GB_PD, kb);
#pragma unroll
        for (int a = 0; a < FA; ++a)
#pragma unroll
          for (int j = 0; j < FB; ++j) dmma884(acc[a][j][0], acc[a][j][1], fa[a], fb[j]);
        if (produce && late) issue_part(c + GB_PD, kb);
      }
      if (produce) cp_async_mbar_arrive(&full_bar[(u + GB_PD) % GB_STG]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[st]);  // after the DMMAs that consumed the slab's last fragments
    }
    gc += (unsigned)nsl;
    const bool c16 = ((((unsigned long long)J.C) & 15) == 0) && (J.ldc % 2 == 0);
#pragma unroll
    for (int a = 0; a < FA; ++a) {
      const int gm = m0 + wm * FA * 8 + a * 8 + g;
      if (gm >= J.m) continue;
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        const int gn = n0 + wn * FB * 8 + j * 8 + 2 * q;
        if (gn >= J.n) continue;
        double *cp = J.C + (long long)gm * J.ldc + gn;
        const double v0 = J.alpha * acc[a][j][0], v1 = J.alpha * acc[a][j][1];
        if (c16 && gn + 1 < J.n) {
          double2 o;
          if (J.beta == 0.0) {
            o.x = v0;
            o.y = v1;
          } else {
            const double2 old = *reinterpret_cast<const double2 *>(cp);
            o.x = J.beta * old.x + v0;
            o.y = J.beta * old.y + v1;
          }
          *reinterpret_cast<double2 *>(cp) = o;
        } else {
          cp[0] = (J.beta == 0.0) ? v0 : J.beta * cp[0] + v0;
          if (gn + 1 < J.n) cp[1] = (J.beta == 0.0) ? v1 : J.beta * cp[1] + v1;
        }
      }
    }
  }
}

}  // namespace mfh
