// Micro-benchmark: cost of cooperative-groups grid.sync() vs a hand-rolled
// release/acquire counter barrier on 148 CTAs (dev tool).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_cg(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}
__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;
__device__ __forceinline__ void my_sync(unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int target = gen + 1;
    unsigned int old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(&g_count) : "memory");
    if (old == target * nblocks - 1) {
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&g_gen), "r"(target) : "memory");
    } else {
      unsigned int v;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&g_gen) : "memory"); } while (v < target);
    }
    gen = target;
  }
  __syncthreads();
}
__global__ void k_my(int iters, long long* out) {
  unsigned int gen = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) my_sync(gridDim.x, gen);
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}
int main() {
  long long* o; cudaMalloc(&o, 16);
  int iters = 1000;
  for (int grid : {148, 296}) {
    void* a1[] = {&iters, &o};
    cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, a1, 0, 0);
    long long h; cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("grid %d cg::grid.sync: %.0f cycles/sync\n", grid, (double)h / iters);
    unsigned int z = 0; cudaMemcpyToSymbol(g_count, &z, 4); cudaMemcpyToSymbol(g_gen, &z, 4);
    cudaLaunchCooperativeKernel((void*)k_my, grid, 256, a1, 0, 0);
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("grid %d custom barrier: %.0f cycles/sync (%s)\n", grid, (double)h / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
