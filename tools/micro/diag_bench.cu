// Micro-benchmark of the 64x64 diagonal-factor pivot loop variants (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NB = 64, NBP = 65, NT = 256;
__device__ void build_tab(unsigned short* tab) {
  for (int e = threadIdx.x; e < NB * (NB - 1) / 2; e += blockDim.x) {
    int l = NB - 1, base = 0;
    while (e >= base + (NB - l)) { base += NB - l; --l; }
    tab[e] = (unsigned short)((l + (e - base)) | (l << 8));
  }
}
template <int V>
__global__ void k(double* out, long long* cyc) {
  extern __shared__ double dsm[];
  double (*S)[NBP] = (double(*)[NBP])dsm; double (*X)[NBP] = (double(*)[NBP])(dsm + NB*NBP);
  __shared__ unsigned short tab[NB * (NB - 1) / 2];
  const int t = threadIdx.x;
  build_tab(tab);
  for (int e = t; e < NB * NB; e += NT) { int i = e / NB, j = e % NB; S[i][j] = (i == j) ? 100.0 + i : 0.01 * ((i * 7 + j * 3) % 11); }
  __syncthreads();
  long long c0 = clock64();
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const double pj = S[j][j];
    double rd = (V == 1) ? 0.1 : rsqrt(pj);
    const double rd2 = rd * rd;
    if (t >= j && t < NB) X[t][j] = (t == j) ? pj * rd : S[t][j] * rd;
    if (V != 2) {
      const int T = (NB - 1 - j) * (NB - j) / 2;
      for (int e0 = t; e0 < T; e0 += NT * 8) {
        int ii[8], ll[8]; double a[8], b[8], c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { const int e = e0 + u * NT; const int il = e < T ? tab[e] : 0x0101; ii[u] = il & 0xff; ll[u] = il >> 8; }
#pragma unroll
        for (int u = 0; u < 8; ++u) { a[u] = S[ii[u]][j]; b[u] = S[ll[u]][j]; c[u] = S[ii[u]][ll[u]]; }
#pragma unroll
        for (int u = 0; u < 8; ++u) if (e0 + u * NT < T) S[ii[u]][ll[u]] = fma(-(a[u] * rd2), b[u], c[u]);
      }
    }
    if (V != 3) __syncthreads();
  }
  long long c1 = clock64();
  if (t == 0) { cyc[V] = c1 - c0; out[V] = X[63][63]; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  for (int rep = 0; rep < 2; ++rep) {
    int sm = 2*NB*NBP*8; cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    k<0><<<1, NT, sm>>>(o, c); k<1><<<1, NT, sm>>>(o, c); k<2><<<1, NT, sm>>>(o, c); k<3><<<1, NT, sm>>>(o, c);
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("full %lld  no-rsqrt %lld  no-update %lld  no-barrier %lld cycles (64 steps)\n", h[0], h[1], h[2], h[3]);
  }
  return 0;
}
