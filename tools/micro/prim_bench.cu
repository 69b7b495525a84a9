// Micro-benchmark of primitive costs inside one CTA (dev tool): barrier,
// fp64 rsqrt chain, shared-memory dependent load chain, shuffle chain.
#include <cstdio>
__global__ void k(double* out, long long* cyc) {
  __shared__ double S[64][65];
  const int t = threadIdx.x;
  for (int e = t; e < 64 * 65; e += blockDim.x) (&S[0][0])[e] = 1.0 + 1e-3 * e;
  __syncthreads();
  long long c0 = clock64();
  for (int i = 0; i < 1000; ++i) __syncthreads();
  long long c1 = clock64();
  double x = S[t & 63][t & 63];
  for (int i = 0; i < 1000; ++i) x = rsqrt(x + 1.0);
  long long c2 = clock64();
  double y = 0; int idx = t & 63;
  for (int i = 0; i < 1000; ++i) { y += S[idx][i & 63]; idx = ((int)y) & 63; }
  long long c3 = clock64();
  double z = x;
  for (int i = 0; i < 1000; ++i) z = __shfl_sync(0xffffffffu, z, (i + t) & 31) + 1.0;
  long long c4 = clock64();
  double w = z;
  for (int i = 0; i < 1000; ++i) w = fma(w, 1.0000001, 1e-9);
  long long c5 = clock64();
  if (t == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4; }
  out[t] = x + y + z + w;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64);
  for (int nt : {32, 256}) {
    k<<<1, nt>>>(o, c); k<<<1, nt>>>(o, c);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("threads %d: bar %.1f  rsqrt %.1f  lds-chain %.1f  shfl-chain %.1f  dfma-chain %.1f cycles/op\n", nt,
           h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0, h[4] / 1000.0);
  }
}
