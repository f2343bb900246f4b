// FP64 pipe microbenchmarks for the B200 roofline denominators (DFMA, DMMA,
// double exp, fp64 atomics). Not product code: run once per box to measure the
// peaks the BSC kernels are judged against.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = i + 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void dmma16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void exp_kernel(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = -1.0 - threadIdx.x * 1e-4 - i * 0.1;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { s += exp(x[i]); x[i] -= 1e-7; }
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void red_kernel(double* buf, int n, int iters) {
  unsigned idx = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    unsigned a = (idx * 2654435761u + it * 40503u) % n;
    atomicAdd(buf + a, 1.0);
  }
}

__global__ void reds_kernel(double* out, int iters) {
  __shared__ double sb[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    unsigned a = (threadIdx.x * 97u + it * 31u) & 4095u;
    atomicAdd(sb + a, 1.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sb[5];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  auto timeit = [&](auto launch) { launch(); cudaDeviceSynchronize(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); return ms; };
  {
    int iters = 20000, blocks = sms * 8, threads = 256;
    timeit([&] { dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); });
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_tflops\": %.2f", flops / ms / 1e9);
  }
  {
    int iters = 4000, blocks = sms * 8, threads = 256;
    timeit([&] { dmma_kernel<8><<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf(", \"dmma_m8n8k4_tflops\": %.2f", flops / ms / 1e9);
  }
  {
    int iters = 1000, blocks = sms * 8, threads = 256;
    timeit([&] { dmma16_kernel<4><<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * blocks * (threads / 32);
    printf(", \"dmma_m16n8k16_tflops\": %.2f", flops / ms / 1e9);
  }
  {
    int iters = 2000, blocks = sms * 8, threads = 256;
    timeit([&] { exp_kernel<<<blocks, threads>>>(out, iters); });
    double n = 8.0 * iters * blocks * threads;
    printf(", \"dexp_gps\": %.2f", n / ms / 1e6);
  }
  {
    int n = 1 << 24; double* buf; CK(cudaMalloc(&buf, n * 8)); cudaMemset(buf, 0, n * 8);
    int iters = 64, blocks = sms * 16, threads = 256;
    timeit([&] { red_kernel<<<blocks, threads>>>(buf, n, iters); });
    printf(", \"red_f64_global_gops\": %.2f", (double)iters * blocks * threads / ms / 1e6);
    cudaFree(buf);
  }
  {
    int iters = 2000, blocks = sms * 8, threads = 256;
    timeit([&] { reds_kernel<<<blocks, threads>>>(out, iters); });
    printf(", \"atom_f64_shared_gops\": %.2f", (double)iters * blocks * threads / ms / 1e6);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
