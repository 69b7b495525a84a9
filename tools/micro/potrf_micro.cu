// Micro-benchmark: latency of the 32x32 diagonal-tile Cholesky variants and of
// the primitives on its dependency chain (double shuffle, rsqrt, DFMA), one
// CTA, clock64.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o potrf_micro tools/micro/potrf_micro.cu && ./potrf_micro
#include <cstdio>
#include <cmath>

constexpr int NB = 32, PT = 36;

__global__ void k_prims(double* out, long long* cyc, double seed) {
  const int lane = threadIdx.x & 31;
  double v = seed + lane;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31) + 1e-3;
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) v = rsqrt(v * v + 1.0);
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) v = fma(v, 0.999, 1e-3);
  long long t3 = clock64();
  float f = (float)v;
#pragma unroll 1
  for (int i = 0; i < 64; ++i) f = rsqrtf(f * f + 1.0f);
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
    __syncthreads();
  }
  long long t5 = clock64();
  out[threadIdx.x] = v + f;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 64;
    cyc[1] = (t2 - t1) / 64;
    cyc[2] = (t3 - t2) / 64;
    cyc[3] = (t4 - t3) / 64;
    cyc[4] = (t5 - t4) / 64;
  }
}

// variant A: whole tile in warp 0's registers, lane = row, fully unrolled
__device__ void potrf_regs(double* S) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  double r[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) r[q] = S[lane * PT + q];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const double d = __shfl_sync(0xffffffffu, r[j], j);
    const double rs = rsqrt(d);
    const double l = lane > j ? r[j] * rs : (lane == j ? d * rs : 0.0);
    r[j] = l;
#pragma unroll
    for (int q = j + 1; q < NB; ++q) {
      const double lq = __shfl_sync(0xffffffffu, l, q);
      r[q] = fma(-l, lq, r[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NB; ++q) S[lane * PT + q] = r[q];
}

// variant B: panels of PW (warp 0 registers) + CTA-wide trailing update
template <int PW>
__device__ void potrf_panels(double* S) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll 1
  for (int jb = 0; jb < NB; jb += PW) {
    if (w == 0) {
      double r[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) r[q] = S[lane * PT + jb + q];
#pragma unroll
      for (int p = 0; p < PW; ++p) {
        const int j = jb + p;
        const double d = __shfl_sync(0xffffffffu, r[p], j);
        const double rs = rsqrt(d);
        const double l = lane > j ? r[p] * rs : (lane == j ? d * rs : 0.0);
        r[p] = l;
#pragma unroll
        for (int q = p + 1; q < PW; ++q) {
          const double lq = __shfl_sync(0xffffffffu, l, jb + q);
          if (lane > j) r[q] = fma(-l, lq, r[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < PW; ++q) S[lane * PT + jb + q] = r[q];
    }
    __syncthreads();
    const int base = jb + PW;
    for (int i = base + (t >> 4); i < NB; i += 16)
      for (int l = base + (t & 15); l <= i; l += 16) {
        double v = S[i * PT + l];
#pragma unroll
        for (int p = 0; p < PW; ++p) v = fma(-S[i * PT + jb + p], S[l * PT + jb + p], v);
        S[i * PT + l] = v;
      }
    __syncthreads();
  }
}

// variant C: smem, lane = row, rolled loops, warp 0 only (no CTA barriers)
__device__ void potrf_warp_smem(double* S) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const double d = S[j * 33 + j];
    const double rs = rsqrt(d);
    double l = 0.0;
    if (lane > j) {
      l = S[lane * 33 + j] * rs;
      S[lane * 33 + j] = l;
    }
    __syncwarp();
    if (lane == j) S[j * 33 + j] = d * rs;
    if (lane > j) {
#pragma unroll 4
      for (int q = j + 1; q <= lane; ++q) S[lane * 33 + q] = fma(-l, S[q * 33 + j], S[lane * 33 + q]);
    }
    __syncwarp();
  }
}

__global__ void k_potrf(const double* Min, double* out, long long* cyc, int variant) {
  __shared__ double S[NB * PT];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int i = e / NB, j = e % NB;
    S[i * (variant == 3 ? 33 : PT) + j] = Min[e];
  }
  __syncthreads();
  long long best = 1ll << 60;
  for (int rep = 0; rep < 3; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    if (variant == 0) potrf_regs(S);
    else if (variant == 1) potrf_panels<8>(S);
    else if (variant == 2) potrf_panels<4>(S);
    else potrf_warp_smem(S);
    __syncthreads();
    long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
    // reload for the next repetition
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
      const int i = e / NB, j = e % NB;
      if (rep < 2) S[i * (variant == 3 ? 33 : PT) + j] = Min[e];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) out[e] = S[(e / NB) * (variant == 3 ? 33 : PT) + e % NB];
  if (threadIdx.x == 0) cyc[0] = best;
}

int main() {
  double* M;
  double* o;
  long long* c;
  cudaMallocManaged(&M, NB * NB * 8);
  cudaMallocManaged(&o, NB * NB * 8);
  cudaMallocManaged(&c, 64);
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < NB; ++j) M[i * NB + j] = (i == j ? NB + 1.0 : 1.0 / (1 + i + j));
  k_prims<<<1, 256>>>(o, c, 0.5);
  cudaDeviceSynchronize();
  printf("latency cycles: shfl.f64 %lld  rsqrt.f64 %lld  dfma %lld  rsqrtf %lld  syncthreads(256) %lld\n", c[0], c[1],
         c[2], c[3], c[4]);
  const char* names[] = {"registers (full unroll)", "panels PW=8", "panels PW=4", "warp smem rolled"};
  for (int v = 0; v < 4; ++v) {
    k_potrf<<<1, 256>>>(M, o, c, v);
    cudaError_t e = cudaDeviceSynchronize();
    double l00 = o[0], l10 = o[NB];
    printf("potrf %-26s %lld cycles  (L00 %.6f L10 %.6f) %s\n", names[v], c[0], l00, l10, cudaGetErrorString(e));
  }
  return 0;
}
