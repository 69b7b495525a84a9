// Probe of tcgen05.mma kind::tf32 operand layouts: one 128 x 256 x 8 MMA with
// operands written by threads into shared memory under several layout /
// descriptor hypotheses; D is read back from TMEM and compared on the host.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2104_14101_b200/csrc/umma.cuh"

using namespace adask;

constexpr int M = 128, N = 256, K = 8;

// layout ids: 0 = K-major SW128 (rows of 128 B along K), 1 = MN-major SW128
__device__ uint32_t off_kmajor(int i, int k) {  // i = M/N index, k < 32
  return (i / 8) * 1024 + (i % 8) * 128 + ((((k / 4) ^ (i % 8)) & 7) * 16) + (k % 4) * 4;
}
__device__ uint32_t off_mnmajor(int i, int k, int lbo, int sbo) {
  return (i / 32) * lbo + (k / 8) * sbo + (k % 8) * 128 + (((((i % 32) / 4) ^ (k % 8)) & 7) * 16) + (i % 4) * 4;
}

// MN-major SWIZZLE_128B_BASE32B: 32 MN per 128 B row, K rows at 128 B, K
// groups of 4 rows at sbo, MN groups at lbo, 32-byte chunk ^= (row & 3)
__device__ uint32_t off_mn32(int i, int k, int lbo, int sbo) {
  return (i / 32) * lbo + (k / 4) * sbo + (k % 4) * 128 + (((((i % 32) / 8) ^ (k % 4)) & 3) * 32) + (i % 8) * 4;
}

__global__ void k_probe(int amode, int bmode, int alb, int asb, int blb, int bsb, int swap_a, int swap_b,
                        const float* Ag, const float* Bg, float* D) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                // up to 64 KB
  uint8_t* sB = sm + 64 * 1024;    // up to 64 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int e = threadIdx.x; e < 16384; e += blockDim.x) {
    ((float*)sA)[e] = 0.f;
    ((float*)sB)[e] = 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    int i = e / K, k = e % K;
    uint32_t o = amode == 0 ? off_kmajor(i, k) : amode == 1 ? off_mnmajor(i, k, alb, asb) : off_mn32(i, k, alb, asb);
    *(float*)(sA + o) = Ag[i * K + k];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    int j = e / K, k = e % K;
    uint32_t o = bmode == 0 ? off_kmajor(j, k) : bmode == 1 ? off_mnmajor(j, k, blb, bsb) : off_mn32(j, k, blb, bsb);
    *(float*)(sB + o) = Bg[j * K + k];
  }
  umma::fence_proxy_async_smem();
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) umma::tmem_alloc(&tslot, 256);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    uint32_t la = amode == 0 ? 16 : alb, sa_ = amode == 0 ? 1024 : asb;
    uint32_t lb = bmode == 0 ? 16 : blb, sb_ = bmode == 0 ? 1024 : bsb;
    if (swap_a) { uint32_t t = la; la = sa_; sa_ = t; }
    if (swap_b) { uint32_t t = lb; lb = sb_; sb_ = t; }
    uint64_t ad = umma::sdesc(smem_u32(sA), la, sa_, amode == 2 ? 1 : 2);
    uint64_t bd = umma::sdesc(smem_u32(sB), lb, sb_, bmode == 2 ? 1 : 2);
    uint32_t idesc = umma::idesc_tf32(M, N, amode != 0, bmode != 0);
    umma::mma_tf32(tb, ad, bd, idesc, 0u);
    umma::mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  umma::fence_after_sync();
  if (warp < 4) {
    int row = warp * 32 + (threadIdx.x & 31);
    for (int c = 0; c < N; c += 16) {
      float v[16];
      umma::tmem_ld16(tb + ((uint32_t)(warp * 32) << 16) + c, v);
      for (int j = 0; j < 16; ++j) D[row * N + c + j] = v[j];
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tb, 256);
}

int main() {
  std::vector<float> A(M * K), B(N * K), ref(M * N);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 7 - 3);
  for (auto& x : B) x = (float)(rand() % 7 - 3);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += A[i * K + k] * B[j * K + k];
      ref[i * N + j] = s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, ref.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  struct Cfg { int am, bm, alb, asb, blb, bsb, swa, swb; const char* name; };
  Cfg cfgs[] = {
      {0, 0, 0, 0, 0, 0, 0, 0, "A K-major, B K-major"},
      {1, 0, 1024, 4096, 0, 0, 0, 0, "A MN-major (lbo=1024 sbo=4096), B K"},
      {1, 0, 1024, 4096, 0, 0, 1, 0, "A MN-major swapped desc, B K"},
      {0, 1, 0, 0, 1024, 8192, 0, 0, "A K, B MN-major (lbo=1024 sbo=8192)"},
      {0, 1, 0, 0, 1024, 8192, 0, 1, "A K, B MN-major swapped desc"},
      {1, 1, 1024, 4096, 1024, 8192, 0, 0, "A MN, B MN"},
      {1, 1, 1024, 4096, 1024, 8192, 1, 1, "A MN, B MN swapped desc"},
      {1, 1, 2048, 1024, 2048, 1024, 0, 0, "A MN, B MN (lbo=2048 sbo=1024, kernel layout)"},
      {1, 1, 2048, 1024, 2048, 1024, 1, 1, "A MN, B MN (kernel layout) swapped desc"},
      {0, 2, 0, 0, 1024, 512, 0, 0, "A K, B MN32 (lbo=1024 sbo=512)"},
      {0, 2, 0, 0, 1024, 512, 0, 1, "A K, B MN32 swapped"},
      {2, 2, 1024, 512, 1024, 512, 0, 0, "A MN32, B MN32 (lbo=1024 sbo=512)"},
      {2, 2, 1024, 512, 1024, 512, 1, 1, "A MN32, B MN32 swapped"},
      {2, 2, 2048, 512, 2048, 512, 0, 0, "A MN32, B MN32 (lbo=2048 sbo=512)"},
      {2, 2, 4096, 1024, 4096, 1024, 0, 0, "A MN32, B MN32 (lbo=4096 sbo=1024)"},
  };
  for (auto& c : cfgs) {
    cudaMemset(dD, 0, ref.size() * 4);
    k_probe<<<1, 256, 140 * 1024>>>(c.am, c.bm, c.alb, c.asb, c.blb, c.bsb, c.swa, c.swb, dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(M * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, nz = 0;
    int first_bad = -1;
    for (int t = 0; t < M * N; ++t) {
      double df = fabs(D[t] - ref[t]);
      if (df > err) err = df;
      if (df > 0.5 && first_bad < 0) first_bad = t;
      nz += D[t] != 0;
    }
    printf("%-50s err=%8.2f nonzero=%6.0f first_bad=%d (%s)\n", c.name, err, nz, first_bad,
           cudaGetErrorString(e));
    if (first_bad >= 0 && first_bad < 2 * N) {
      printf("   row0 got:");
      for (int j = 0; j < 12; ++j) printf(" %g", D[j]);
      printf("\n   row0 ref:");
      for (int j = 0; j < 12; ++j) printf(" %g", ref[j]);
      printf("\n");
    }
  }
  return 0;
}
