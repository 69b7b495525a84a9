// Throughput of the special-function unit ops used by the Box-Muller
// generator (sin / cos / lg2 / sqrt approx) versus FMA, cycles per warp op.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_bench mufu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, long long* cyc, int iters) {
  float a = threadIdx.x * 1e-3f + 0.5f, b = a * 0.7f, c = a * 0.3f, e = a * 0.9f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) { a = __sinf(a); b = __sinf(b); c = __sinf(c); e = __sinf(e); }
      if (OP == 1) { asm("lg2.approx.ftz.f32 %0, %0;" : "+f"(a)); asm("lg2.approx.ftz.f32 %0, %0;" : "+f"(b));
                     asm("lg2.approx.ftz.f32 %0, %0;" : "+f"(c)); asm("lg2.approx.ftz.f32 %0, %0;" : "+f"(e)); }
      if (OP == 2) { asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(a)); asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(b));
                     asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(c)); asm("sqrt.approx.ftz.f32 %0, %0;" : "+f"(e)); }
      if (OP == 3) { a = fmaf(a, 1.0001f, 0.1f); b = fmaf(b, 1.0001f, 0.1f); c = fmaf(c, 1.0001f, 0.1f); e = fmaf(e, 1.0001f, 0.1f); }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + e;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4 * 8);
  cudaMalloc(&c, 8);
  const int iters = 1000;
  const char* names[] = {"sin.approx", "lg2.approx", "sqrt.approx", "fma"};
  for (int op = 0; op < 4; ++op) {
    for (int warps : {4, 16, 32}) {
      long long h = 0;
      auto run = [&](auto kern) { kern<<<148, warps * 32>>>(o, c, iters); cudaDeviceSynchronize(); };
      if (op == 0) run(k<0>); if (op == 1) run(k<1>); if (op == 2) run(k<2>); if (op == 3) run(k<3>);
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)iters * 8 * 4 * warps * 32;  // per SM (one CTA per SM)
      printf("%-12s warps/SM=%2d: %.2f ops/clk/SM\n", names[op], warps, ops / h);
    }
  }
  return 0;
}
