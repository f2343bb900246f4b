// Tile-configuration sweep of the DMMA GEMM (csrc/dgemm.cuh) on the c2
// shapes: B = Y·W (M = 200000, N = 304, K = 256) and Yᵀ·ES (M = 256, N = 304,
// K = 200000, split-K). Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// -I paper_1908_06843_b200/csrc tools/gemm_bench.cu -o tools/gemm_bench
#include <cstdio>
#include <vector>

#include "dgemm.cuh"

using namespace bscgpu;

template <int BM, int BN, int BK, int WM, int WN, bool AR, bool BR, int ST>
float time_cfg(const GemmArgs& g, int splits, cudaStream_t s, int reps = 10) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) launch_dgemm<BM, BN, BK, WM, WN, AR, BR, ST>(g, splits, s);
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) launch_dgemm<BM, BN, BK, WM, WN, AR, BR, ST>(g, splits, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
  return ms / reps;
}

#define RUN1(name, ...)                                                                    \
  {                                                                                       \
    const float ms = time_cfg<__VA_ARGS__>(g1, 1, s);                                     \
    printf("gemm1 %-34s %.4f ms  %.2f TF\n", name, ms, 2.0 * M * Nr * K / (ms * 1e9));    \
  }
#define RUN2(name, ...)                                                                   \
  {                                                                                      \
    const float ms = time_cfg<__VA_ARGS__>(g2, splits, s);                               \
    printf("gemm2 %-34s %.4f ms  %.2f TF\n", name, ms, 2.0 * M * Nr * K / (ms * 1e9));   \
  }

int main() {
  const int M = 200000, Np = 304, Nr = 300, K = 256, Kp = 256;
  double *y, *w, *b, *es, *part, *cs;
  cudaMalloc(&y, sizeof(double) * M * Kp);
  cudaMalloc(&w, sizeof(double) * Kp * Np);
  cudaMalloc(&b, sizeof(double) * M * Np);
  cudaMalloc(&es, sizeof(double) * M * Np);
  cudaMemset(y, 0, sizeof(double) * M * Kp);
  cudaMemset(w, 0, sizeof(double) * Kp * Np);
  cudaMemset(es, 0, sizeof(double) * M * Np);
  const int splits = 59;
  cudaMalloc(&part, sizeof(double) * splits * Kp * Np);
  cudaMalloc(&cs, sizeof(double) * splits * Np);
  cudaStream_t s;
  cudaStreamCreate(&s);
  GemmArgs g1{M, Np, Kp, y, Kp, w, Np, b, Np, 1.0, 0.0, Kp, 0};
  RUN1("64x64x16 w32x32 s2", 64, 64, 16, 32, 32, true, true, 2);
  RUN1("64x64x16 w64x16 s2", 64, 64, 16, 64, 16, true, true, 2);
  RUN1("64x64x16 w16x64 s2", 64, 64, 16, 16, 64, true, true, 2);
  RUN1("64x32x16 w32x32 s2", 64, 32, 16, 32, 32, true, true, 2);
  RUN1("64x32x16 w32x32 s3", 64, 32, 16, 32, 32, true, true, 3);
  RUN1("32x64x16 w32x32 s3", 32, 64, 16, 32, 32, true, true, 3);
  RUN1("128x64x16 w64x32 s2", 128, 64, 16, 64, 32, true, true, 2);
  RUN1("64x64x32 w32x32 s2", 64, 64, 32, 32, 32, true, true, 2);
  const int krows = M;
  int kchunk = (krows + splits - 1) / splits;
  kchunk = (kchunk + 1) & ~1;
  GemmArgs g2{Kp, Np, krows, y, Kp, es, Np, part, Np, 1.0, 0.0, kchunk, (long long)Kp * Np, cs};
  RUN2("128x64x16 w64x16 s3", 128, 64, 16, 64, 16, false, true, 3);
  RUN2("128x64x16 w64x16 s2", 128, 64, 16, 64, 16, false, true, 2);
  RUN2("128x64x16 w64x32 s3", 128, 64, 16, 64, 32, false, true, 3);
  RUN2("128x64x16 w128x16 s3", 128, 64, 16, 128, 16, false, true, 3);
  RUN2("128x32x16 w64x16 s3", 128, 32, 16, 64, 16, false, true, 3);
  RUN2("64x64x16 w64x16 s3", 64, 64, 16, 64, 16, false, true, 3);
  RUN2("128x64x32 w64x16 s2", 128, 64, 32, 64, 16, false, true, 2);
  return 0;
}
