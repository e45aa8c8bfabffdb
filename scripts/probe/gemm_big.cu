// k_gemm_big against cuBLAS DGEMM on the shapes of the HODLR levels / eliminations (probe).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1410_2697_b200/csrc
//      scripts/probe/gemm_big.cu -o /tmp/gemm_big -lcublas
#include <cublas_v2.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "kernels.cuh"
using namespace mfh;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("cuda error %s line %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

template <int WM, int WN, int FA, int FB, int STG, int MINB>
static float run_big(const std::vector<GemmJob> &jobs, int reps, int ctas_per_sm) {
  using Cfg = GemmBigCfg<WM, WN, FA, FB, STG>;
  std::vector<GemmBigTile> tiles;
  for (int j = 0; j < (int)jobs.size(); ++j)
    for (int a = 0; a < (jobs[j].m + Cfg::BM - 1) / Cfg::BM; ++a)
      for (int b = 0; b < (jobs[j].n + Cfg::BN - 1) / Cfg::BN; ++b) tiles.push_back({j, a, b});
  GemmJob *dj;
  GemmBigTile *dt;
  CK(cudaMalloc(&dj, sizeof(GemmJob) * jobs.size()));
  CK(cudaMalloc(&dt, sizeof(GemmBigTile) * tiles.size()));
  CK(cudaMemcpy(dj, jobs.data(), sizeof(GemmJob) * jobs.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dt, tiles.data(), sizeof(GemmBigTile) * tiles.size(), cudaMemcpyHostToDevice));
  auto kern = k_gemm_big<WM, WN, FA, FB, STG, MINB>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  int grid = std::min((int)tiles.size(), 148 * ctas_per_sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, WM * WN * 32, Cfg::SMEM>>>(dj, dt, (int)tiles.size());
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<grid, WM * WN * 32, Cfg::SMEM>>>(dj, dt, (int)tiles.size());
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(dj);
  cudaFree(dt);
  return ms / reps;
}

int main() {
  cublasHandle_t h;
  cublasCreate(&h);
  struct Shape { int m, n, k, pad, cnt; };  // pad: extra leading-dimension entries (odd: unaligned rows); cnt: jobs in the batch
  std::vector<Shape> shapes = {{4096, 4096, 4096, 0, 1}, {8192, 1024, 8192, 0, 1}, {8192, 700, 8192, 0, 1}, {4096, 512, 4096, 0, 2},
                               {2048, 2048, 2048, 0, 1}, {2048, 300, 2048, 0, 4}, {1024, 256, 1024, 0, 8}, {1024, 1024, 1024, 0, 4},
                               {6000, 301, 6000, 1, 1}, {3000, 3000, 333, 0, 1}, {6144, 6144, 640, 0, 1}, {12288, 12288, 1000, 0, 1},
                               {512, 512, 512, 0, 16}, {1000, 129, 4000, 3, 6}};
  for (auto s : shapes) {
    const int lda = s.k + s.pad, ldb = s.n + s.pad, ldc = s.n + s.pad;
    std::vector<GemmJob> jobs;
    std::vector<double *> Cref;
    std::vector<double> hA((size_t)s.m * lda), hB((size_t)s.k * ldb);
    for (auto &v : hA) v = (double)rand() / RAND_MAX - 0.5;
    for (auto &v : hB) v = (double)rand() / RAND_MAX - 0.5;
    for (int c = 0; c < s.cnt; ++c) {
      double *A, *B, *C, *C2;
      CK(cudaMalloc(&A, sizeof(double) * hA.size()));
      CK(cudaMalloc(&B, sizeof(double) * hB.size()));
      CK(cudaMalloc(&C, sizeof(double) * s.m * ldc));
      CK(cudaMalloc(&C2, sizeof(double) * s.m * ldc));
      CK(cudaMemcpy(A, hA.data(), sizeof(double) * hA.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(B, hB.data(), sizeof(double) * hB.size(), cudaMemcpyHostToDevice));
      CK(cudaMemset(C, 0, sizeof(double) * s.m * ldc));
      CK(cudaMemset(C2, 0, sizeof(double) * s.m * ldc));
      jobs.push_back(GemmJob{A, B, C, s.m, s.n, s.k, lda, ldb, ldc, 1.0, 0.0});
      Cref.push_back(C2);
    }
    const double flops = 2.0 * s.m * s.n * s.k * s.cnt;
    const int reps = flops > 5e10 ? 5 : 20;
    // cuBLAS, one call per job (the engine's route)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double al = 1.0, be = 0.0;
    auto blas = [&]() {
      for (int c = 0; c < s.cnt; ++c)
        cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, s.n, s.m, s.k, &al, jobs[c].B, ldb, jobs[c].A, lda, &be, Cref[c], ldc);
    };
    blas();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) blas();
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float msb;
    cudaEventElapsedTime(&msb, e0, e1);
    msb /= reps;
    const float m1 = run_big<2, 4, 8, 4, 4, 1>(jobs, reps, 1);   // 128 x 128
    const float m2 = run_big<2, 4, 8, 4, 5, 1>(jobs, reps, 1);   // 128 x 128, 5 stages (3 slabs ahead)
    const float m3 = run_big<2, 4, 4, 4, 4, 2>(jobs, reps, 2);   // 64 x 128
    // check job 0 against cuBLAS (last config ran last)
    std::vector<double> c1((size_t)s.m * ldc), c2((size_t)s.m * ldc);
    CK(cudaMemcpy(c1.data(), jobs[0].C, sizeof(double) * c1.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c2.data(), Cref[0], sizeof(double) * c2.size(), cudaMemcpyDeviceToHost));
    double md = 0, mx = 0;
    for (int i = 0; i < s.m; ++i)
      for (int j = 0; j < s.n; ++j) {
        md = fmax(md, fabs(c1[(size_t)i * ldc + j] - c2[(size_t)i * ldc + j]));
        mx = fmax(mx, fabs(c2[(size_t)i * ldc + j]));
      }
    printf("%5d x %5d x %5d  ld+%d  x%-2d | cuBLAS %8.3f ms %5.1f TF | 128x128 %8.3f ms %5.1f TF | 128x128s5 %8.3f ms %5.1f TF | 64x128 %8.3f ms %5.1f TF | maxdiff %.2e / %.2e\n",
           s.m, s.n, s.k, s.pad, s.cnt, msb, flops / msb * 1e-9, m1, flops / m1 * 1e-9, m2, flops / m2 * 1e-9, m3, flops / m3 * 1e-9, md, mx);
    fflush(stdout);
    for (auto &j : jobs) { cudaFree((void *)j.A); cudaFree((void *)j.B); cudaFree(j.C); }
    for (auto p : Cref) cudaFree(p);
  }
  return 0;
}
