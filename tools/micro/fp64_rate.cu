// Throughput of independent DADD / DFMA / FADD2 (packed f32x2) per SM (dev tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu
#include <cstdio>

template <int K>
__global__ void k_dadd(double* out, int iters, double s) {
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __dadd_rn(v[k], s);
  }
  double t = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) t += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int K>
__global__ void k_dfma(double* out, int iters, double s) {
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = fma(v[k], s, 1e-7);
  }
  double t = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) t += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int K>
__global__ void k_fadd2(double* out, int iters, float s) {
  unsigned long long v[K];
  unsigned long long ss = ((unsigned long long)__float_as_uint(s) << 32) | __float_as_uint(s);
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v[k]) : "l"(ss));
  }
  unsigned long long t = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) t ^= v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (double)t;
}

int main() {
  double* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, K = 8;
  for (int nt : {256, 512, 1024}) {
    const int grid = 148 * (2048 / nt);
    for (int which = 0; which < 3; ++which) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (which == 0) k_dadd<K><<<grid, nt>>>(o, iters, 1e-9);
        if (which == 1) k_dfma<K><<<grid, nt>>>(o, iters, 1.0000001);
        if (which == 2) k_fadd2<K><<<grid, nt>>>(o, iters, 1e-9f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) {
          const double ops = (double)grid * nt * iters * K;
          const double per_clk_sm = ops / (ms * 1e-3) / 148 / (clk * 1e3);
          printf("nt %4d %-6s %.3f ms  %.1f ops/clk/SM (at %d MHz max)  %.2f Tops/s\n", nt,
                 which == 0 ? "dadd" : which == 1 ? "dfma" : "fadd2", ms, per_clk_sm, clk / 1000, ops / ms / 1e9);
        }
      }
    }
  }
  return 0;
}
