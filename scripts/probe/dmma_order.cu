// Does mma.sync m8n8k4 f64 equal the k-ascending FMA chain bit for bit? (probe)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double *A, const double *B, const double *C, double *D, double *E, int trials) {
  int lane = threadIdx.x;
  for (int t = 0; t < trials; ++t) {
    const double *a = A + t * 32, *b = B + t * 32, *c = C + t * 64;
    int g = lane >> 2, q = lane & 3;
    double a0 = a[g * 4 + q];      // A 8x4 row-major
    double b0 = b[q * 8 + g];      // B 4x8 row-major: B[k][n], k = q, n = g
    double c0 = c[g * 8 + 2 * q], c1 = c[g * 8 + 2 * q + 1];
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d0), "=d"(d1) : "d"(a0), "d"(b0), "d"(c0), "d"(c1));
    D[t * 64 + g * 8 + 2 * q] = d0;
    D[t * 64 + g * 8 + 2 * q + 1] = d1;
    // reference chains
    for (int e = lane; e < 64; e += 32) {
      int i = e / 8, j = e % 8;
      double s = c[e];
      for (int kk = 0; kk < 4; ++kk) s = fma(a[i * 4 + kk], b[kk * 8 + j], s);
      E[t * 64 + e] = s;
    }
  }
}
int main() {
  const int T = 20000;
  double *A, *B, *C, *D, *E;
  cudaMallocManaged(&A, sizeof(double) * 32 * T);
  cudaMallocManaged(&B, sizeof(double) * 32 * T);
  cudaMallocManaged(&C, sizeof(double) * 64 * T);
  cudaMallocManaged(&D, sizeof(double) * 64 * T);
  cudaMallocManaged(&E, sizeof(double) * 64 * T);
  srand(1);
  auto rnd = [] { double m = (rand() / (double)RAND_MAX) * 2 - 1; int ex = rand() % 40 - 20; return ldexp(m, ex); };
  for (int i = 0; i < 32 * T; ++i) A[i] = rnd(), B[i] = rnd();
  for (int i = 0; i < 64 * T; ++i) C[i] = rnd();
  k<<<1, 32>>>(A, B, C, D, E, T);
  cudaDeviceSynchronize();
  long diff = 0, diff_sum = 0;
  for (int i = 0; i < 64 * T; ++i) {
    if (memcmp(&D[i], &E[i], 8)) ++diff;
  }
  // also compare with an unfused product sum
  printf("entries %d, bit differences vs k-ascending fma chain: %ld\n", 64 * T, diff);
  return 0;
}
