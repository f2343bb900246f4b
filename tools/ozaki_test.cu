// Standalone check + timing of the int8-sliced tcgen05 fp64 GEMM (csrc/ozaki_gemm.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1908_06843_b200/csrc \
//        tools/ozaki_test.cu -o tools/ozaki_test
//   tools/ozaki_test [M N K [P]]   (GEMM1 shape: C = Y·W;  GEMM2 shape: C = Yᵀ·E, split-K over P points)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "ozaki_gemm.cuh"

using namespace bscgpu;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

static long long rup(long long x, long long m) { return (x + m - 1) / m * m; }

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 200000, N = argc > 2 ? atoi(argv[2]) : 300,
            K = argc > 3 ? atoi(argv[3]) : 256;
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud;

  // ---------------- GEMM1: C[M×N] = Y[M×K] · W[K×N]
  {
    std::vector<double> Y((size_t)M * K), W((size_t)K * N);
    for (auto& v : Y) v = nd(rng) * 2.0 + 0.3;
    for (auto& v : W) v = nd(rng) * 0.3;
    const long long Kp = rup(K, 16), Np = rup(N, 8);
    double *dY, *dW, *dC, *dsa, *dsb;
    unsigned long long* dmax;
    int8_t *dYs, *dWs;
    CK(cudaMalloc(&dY, Y.size() * 8));
    CK(cudaMalloc(&dW, W.size() * 8));
    CK(cudaMalloc(&dC, (size_t)M * Np * 8));
    CK(cudaMalloc(&dsa, (size_t)M * 8));
    CK(cudaMalloc(&dsb, (size_t)Np * 8));
    CK(cudaMalloc(&dmax, (size_t)Np * 8));
    CK(cudaMalloc(&dYs, (size_t)oz::S * M * Kp));
    CK(cudaMalloc(&dWs, (size_t)oz::S * Np * rup(K, 64)));
    CK(cudaMemcpy(dY, Y.data(), Y.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dW, W.data(), W.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(dmax, 0, Np * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    CK(oz::slice_rows(dY, K, M, K, (int)Kp, dYs, (long long)M * Kp, dsa, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms_slice;
    cudaEventElapsedTime(&ms_slice, e0, e1);
    oz::oz_colmax_kernel<<<dim3((N + 31) / 32, 8), 256>>>(dW, N, K, N, dmax);
    oz::oz_scale_from_max_kernel<<<(Np + 255) / 256, 256>>>(dmax, N, (int)Np, 0.0, dsb);
    oz::oz_slice_cols_kernel<<<dim3((Np + 31) / 32, (rup(K, 64) + 127) / 128), 256>>>(dW, N, K, N, (int)Np, rup(K, 64),
                                                                                      dsb, dWs, Np * rup(K, 64), nullptr);
    const oz::Operand opA{dYs, (long long)M * Kp, Kp, M, 0}, opB{dWs, Np * rup(K, 64), Np, (int)Np, 1};
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    oz::Args a{};
    a.sa = dsa;
    a.sb = dsb;
    a.C = dC;
    a.ldc = Np;
    CK(oz::launch_gemm(opA, opB, M, N, (int)Kp, a, sms, 0));
    CK(cudaDeviceSynchronize());
    std::vector<double> C((size_t)M * Np);
    CK(cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost));
    double worst = 0, worst_rel = 0;
    for (int m = 0; m < M; m += (M > 4000 ? M / 2000 : 1)) {
      double ma = 0;
      for (int k = 0; k < K; ++k) ma = fmax(ma, fabs(Y[(size_t)m * K + k]));
      for (int n = 0; n < N; ++n) {
        long double ref = 0, absum = 0;
        double mb = 0;
        for (int k = 0; k < K; ++k) {
          ref += (long double)Y[(size_t)m * K + k] * W[(size_t)k * N + n];
          absum += fabsl((long double)Y[(size_t)m * K + k] * W[(size_t)k * N + n]);
          mb = fmax(mb, fabs(W[(size_t)k * N + n]));
        }
        const double err = fabs((double)(C[(size_t)m * Np + n] - ref));
        worst = fmax(worst, err / (K * ma * mb));
        worst_rel = fmax(worst_rel, err / (double)absum);
      }
    }
    for (int it = 0; it < 3; ++it) CK(oz::launch_gemm(opA, opB, M, N, (int)Kp, a, sms, 0));
    cudaEventRecord(e0);
    const int reps = 10;
    for (int it = 0; it < reps; ++it)
      CK(oz::launch_gemm(opA, opB, M, N, (int)Kp, a, sms, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("GEMM1 M=%d N=%d K=%d: err/(K·max|a|·max|b|) = %.3g (2^%.1f), err/Σ|ab| = %.3g;  %.3f ms, "
           "%.1f fp64-equiv TFLOP/s; slice Y %.3f ms\n",
           M, N, K, worst, log2(worst + 1e-300), worst_rel, ms, 2.0 * M * N * K / ms / 1e9, ms_slice);
    cudaFree(dY); cudaFree(dW); cudaFree(dC); cudaFree(dsa); cudaFree(dsb); cudaFree(dmax); cudaFree(dYs); cudaFree(dWs);
  }

  // ---------------- GEMM2: C[D×H] = Yᵀ·E with Y [P×D], E [P×H] ∈ [0,1], split-K partials
  const int P0 = argc > 4 ? atoi(argv[4]) : 0;  // one checked GEMM2 size (tests) instead of 20k + 200k
  for (int P : {P0 ? P0 : 20000, P0 ? 0 : 200000}) {
    if (P == 0) continue;
    const int D = K, H = N;
    const long long Dp = rup(D, 8), Hp = rup(H, 8), Pp = rup(P, 128);
    std::vector<double> Y((size_t)P * D), E((size_t)P * H);
    for (auto& v : Y) v = nd(rng) * 2.0 + 0.3;
    for (auto& v : E) { double u = ud(rng); v = u < 0.05 ? u * 20 : exp(-40 * u); }
    double *dY, *dE, *dC, *dsa, *dsb, *dcs;
    unsigned long long* dmax;
    int8_t *dYs, *dEs;
    CK(cudaMalloc(&dY, Y.size() * 8));
    CK(cudaMalloc(&dE, E.size() * 8));
    CK(cudaMalloc(&dsa, Dp * 8));
    CK(cudaMalloc(&dsb, Hp * 8));
    CK(cudaMalloc(&dmax, Dp * 8));
    CK(cudaMalloc(&dYs, (size_t)oz::S * Dp * Pp));
    CK(cudaMalloc(&dEs, (size_t)oz::S * Hp * Pp));
    CK(cudaMalloc(&dcs, (size_t)(Pp / 128) * Hp * 8));
    CK(cudaMemcpy(dY, Y.data(), Y.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dE, E.data(), E.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(dmax, 0, Dp * 8));
    oz::oz_colmax_kernel<<<dim3((D + 31) / 32, 64), 256>>>(dY, D, P, D, dmax);
    oz::oz_scale_from_max_kernel<<<(Dp + 255) / 256, 256>>>(dmax, D, (int)Dp, 0.0, dsa);
    oz::oz_slice_cols_kernel<<<dim3((Dp + 31) / 32, Pp / 128), 256>>>(dY, D, P, D, (int)Dp, Pp, dsa, dYs, Dp * Pp,
                                                                     nullptr);
    oz::oz_scale_from_max_kernel<<<(Hp + 255) / 256, 256>>>(dmax, H, (int)Hp, 2.0, dsb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    oz::oz_slice_cols_kernel<<<dim3((Hp + 31) / 32, Pp / 128), 256>>>(dE, H, P, H, (int)Hp, Pp, dsb, dEs, Hp * Pp,
                                                                     dcs);
    cudaEventRecord(e1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    float ms_slice;
    cudaEventElapsedTime(&ms_slice, e0, e1);
    const int kchunk = 128 * (int)std::min<long long>(oz::MAX_KJOB / 128, (Pp / 128 + 23) / 24);
    const oz::Operand opA{dYs, Dp * Pp, Dp, (int)Dp, 1}, opB{dEs, Hp * Pp, Hp, (int)Hp, 1};
    const int splits = (P + kchunk - 1) / kchunk;
    CK(cudaMalloc(&dC, (size_t)splits * Dp * Hp * 8));
    oz::Args a{};
    a.sa = dsa;
    a.sb = dsb;
    a.C = dC;
    a.ldc = Hp;
    a.kchunk = kchunk;
    a.c_split_stride = Dp * Hp;
    CK(oz::launch_gemm(opA, opB, D, H, P, a, sms, 0));
    CK(cudaDeviceSynchronize());
    std::vector<double> Cp((size_t)splits * Dp * Hp);
    CK(cudaMemcpy(Cp.data(), dC, Cp.size() * 8, cudaMemcpyDeviceToHost));
    double worst = 0, worst_rel = 0;
    if (P <= 20000) {
      for (int d = 0; d < D; d += 3)
        for (int h = 0; h < H; h += 2) {
          long double ref = 0, absum = 0;
          double ma = 0, mb = 0;
          for (int p = 0; p < P; ++p) {
            ref += (long double)Y[(size_t)p * D + d] * E[(size_t)p * H + h];
            absum += fabsl((long double)Y[(size_t)p * D + d] * E[(size_t)p * H + h]);
            ma = fmax(ma, fabs(Y[(size_t)p * D + d]));
            mb = fmax(mb, E[(size_t)p * H + h]);
          }
          double c = 0;
          for (int s = 0; s < splits; ++s) c += Cp[(size_t)s * Dp * Hp + (size_t)d * Hp + h];
          const double err = fabs((double)(c - ref));
          worst = fmax(worst, err / (P * ma * mb));
          worst_rel = fmax(worst_rel, err / (double)absum);
        }
    }
    cudaEventRecord(e0);
    const int reps = 10;
    for (int it = 0; it < reps; ++it)
      CK(oz::launch_gemm(opA, opB, D, H, P, a, sms, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("GEMM2 D=%d H=%d P=%d (kchunk %d, %d splits): err/(P·max|a|·max|b|) = %.3g (2^%.1f), err/Σ|ab| = %.3g;"
           "  %.3f ms, %.1f fp64-equiv TFLOP/s; slice E %.3f ms\n",
           D, H, P, kchunk, splits, worst, log2(worst + 1e-300), worst_rel, ms, 2.0 * D * H * P / ms / 1e9,
           ms_slice);
    cudaFree(dY); cudaFree(dE); cudaFree(dC); cudaFree(dsa); cudaFree(dsb); cudaFree(dmax); cudaFree(dYs); cudaFree(dEs); cudaFree(dcs);
  }
  return 0;
}
