// Per-step communication floor of a grid-distributed complete-pivot step (probe).
// G CTAs x 512 threads run K steps of: block argmax -> publish (slot + candidate
// row of n doubles) -> exchange -> every CTA reads the winner's row. Variants:
//   0: atomic arrival counter + spin, then the slots (one L2 read), then the row
//   1: tagged slots (|v| bits + step tag in one 64-bit word, st.release), every
//      CTA polls all G slots (the exchange IS the barrier), then the row
//   2: variant 1 with the row published into a per-step ring and the winner's
//      row read straight after the poll (same as 1; measures the same path)
//   3: barrier only (atomic counter), no slots, no row
// Output: microseconds per step for each variant and G.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Scratch {
  unsigned *bar;
  unsigned long long *tag;  // [2][G]
  long long *key;           // [2][G]
  double *rows;             // [2][G][n]
};

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int VAR>
__global__ void __launch_bounds__(512) k_probe(Scratch s, int n, int K, double *sink, int nl) {
  extern __shared__ double rowsm[];  // nl x n (variant 4)
  __shared__ double prow[4096];
  __shared__ double red[16];
  __shared__ int s_who;
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned epoch = 0;
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    const int par = k & 1;
    // fake local candidate: value depends on (g, k) so the winner moves
    double v = (double)((g * 7919 + k * 104729) % 1000003) + tid * 1e-9;
    if (VAR == 4) {  // trailing update + running argmax over this CTA's rows (as the PLU kernels)
      double bv = -1.0;
      int bj = 0;
      for (int li = warp; li < nl; li += 16) {
        double *row = rowsm + (size_t)li * n;
        const double l = row[k % n] / (1.0 + prow[(k + 1) % n] * 1e-30);
        for (int j = k % 7 + 1 + lane; j < n; j += 32) {
          const double x = __dsub_rn(row[j], __dmul_rn(l * 1e-30, prow[j]));
          row[j] = x;
          const double ax = fabs(x);
          if (ax > bv) {
            bv = ax;
            bj = j;
          }
        }
      }
      v += bv * 1e-300 + bj * 1e-300;
    }
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
      double x = lane < 16 ? red[lane] : -1.0;
      for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == 0) red[0] = x;
    }
    __syncthreads();
    const double best = red[0];
    if (VAR != 3) {
      double *myrow = s.rows + ((size_t)par * G + g) * n;
      for (int j = tid; j < n; j += 512) myrow[j] = best + j;
    }
    if (VAR == 0 || VAR == 3 || VAR == 4) {
      if ((VAR == 0 || VAR == 4) && tid == 0) {
        s.key[par * G + g] = (long long)best;
      }
      __syncthreads();
      if (tid == 0) {
        const unsigned target = (unsigned)G * ++epoch;
        unsigned w;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(w) : "l"(s.bar) : "memory");
        unsigned cur = w + 1;
        while ((int)(cur - target) < 0) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(s.bar) : "memory");
      }
      __syncthreads();
      if (VAR == 0 || VAR == 4) {
        if (warp == 0) {
          long long bk = -1;
          int who = 0;
          for (int q = lane; q < G; q += 32) {
            long long kk = __ldcg(s.key + par * G + q);
            if (kk > bk) bk = kk, who = q;
          }
          for (int o = 16; o > 0; o >>= 1) {
            long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
            int ow = __shfl_xor_sync(0xffffffffu, who, o);
            if (ok > bk || (ok == bk && ow < who)) bk = ok, who = ow;
          }
          if (lane == 0) s_who = who;
        }
        __syncthreads();
      }
    } else {
      // tagged slot: bit 63 = (k >> 1) & 1, low bits = |v| (non-negative double bits)
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        const unsigned long long w =
            ((unsigned long long)((k >> 1) & 1) << 63) | (unsigned long long)__double_as_longlong(best);
        st_rel(s.tag + par * G + g, w);
      }
      if (warp == 0) {
        const unsigned long long want = (unsigned long long)((k >> 1) & 1);
        unsigned long long bw = 0;
        int who = 0x7fffffff;
        for (int q = lane; q < G; q += 32) {
          unsigned long long t;
          do {
            t = ld_acq(s.tag + par * G + q);
          } while ((t >> 63) != want);
          t &= 0x7fffffffffffffffull;
          if (t > bw || (t == bw && q < who)) bw = t, who = q;
        }
        for (int o = 16; o > 0; o >>= 1) {
          unsigned long long ob = __shfl_xor_sync(0xffffffffu, bw, o);
          int ow = __shfl_xor_sync(0xffffffffu, who, o);
          if (ob > bw || (ob == bw && ow < who)) bw = ob, who = ow;
        }
        if (lane == 0) s_who = who;
      }
      __syncthreads();
    }
    if (VAR != 3) {
      const double *orow = s.rows + ((size_t)par * G + s_who) * n;
      for (int j = tid; j < n; j += 512) prow[j] = __ldcg(orow + j);
      __syncthreads();
      acc += prow[(k * 31 + tid) % n];
    }
  }
  if (tid == 0) sink[g] = acc;
}

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1000, K = 2000;
  const int m = argc > 2 ? atoi(argv[2]) : 1728;
  int Gs[] = {37, 74, 148};
  double *sink;
  cudaMalloc(&sink, sizeof(double) * 148);
  cudaFuncSetAttribute((const void *)k_probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024);
  cudaGetLastError();
  for (int var = 0; var < 5; ++var) {
    if (var == 1 || var == 2) continue;
    for (int G : Gs) {
      Scratch s;
      cudaMalloc(&s.bar, 4);
      cudaMalloc(&s.tag, 8 * 2 * G);
      cudaMalloc(&s.key, 8 * 2 * G);
      cudaMalloc(&s.rows, sizeof(double) * 2 * G * n);
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(s.bar, 0, 4);
        // tags start "one parity behind": bit 63 = 1 for both buffers (step 0/1 want 0)
        cudaMemset(s.tag, 0xff, 8 * 2 * G);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        int nn = n, KK = K, nl = (m + G - 1) / G;
        size_t dyn = var == 4 ? sizeof(double) * nl * n : 0;
        if (dyn > 190 * 1024) { printf("variant %d G %d: rows do not fit\n", var, G); break; }
        void *args[5] = {&s, &nn, &KK, &sink, &nl};
        const void *fn = var == 0 ? (const void *)k_probe<0>
                                  : var == 3 ? (const void *)k_probe<3> : (const void *)k_probe<4>;
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(G), dim3(512), args, dyn, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
          printf("launch failed %s\n", cudaGetErrorString(e));
          return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("variant %d G %3d n %d m %d: %.2f us/step\n", var, G, n, m, best * 1e3 / K);
      cudaFree(s.bar);
      cudaFree(s.tag);
      cudaFree(s.key);
      cudaFree(s.rows);
    }
  }
  return 0;
}
