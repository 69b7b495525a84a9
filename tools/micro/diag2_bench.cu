// Micro-benchmark: register-owned lower-triangle right-looking 64x64 Cholesky + inverse (dev tool).
#include <cstdio>
#include <cmath>
constexpr int NB = 64, NBP = 65, NT = 256, NE = NB * (NB + 1) / 2, PER = (NE + NT - 1) / NT;  // 2080, 9
__global__ void k(const double* Min, double* Lout, double* Xout, long long* cyc) {
  __shared__ double S[NB][NBP];
  __shared__ double colbuf[2][NB], piv[2], xbuf[2][NB], rinv[NB];
  const int t = threadIdx.x;
  // element e -> (i, l), lower triangle row-major: e = i(i+1)/2 + l
  int ei[PER], el[PER];
  double a[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = t + q * NT;
    int i = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    while (i * (i + 1) / 2 > e) --i;
    ei[q] = e < NE ? i : -1;
    el[q] = e < NE ? e - i * (i + 1) / 2 : -1;
    a[q] = e < NE ? Min[i * NB + el[q]] : 0.0;
    if (e < NE && i == 0 && el[q] == 0) piv[0] = a[q];
  }
  __syncthreads();
  long long c0 = clock64();
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const double pj = piv[j & 1];
    const double rd = rsqrt(pj);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const bool cj = el[q] == j;
      const double v = (ei[q] == j) ? pj * rd : a[q] * rd;
      a[q] = cj ? v : a[q];
      if (cj) colbuf[j & 1][ei[q]] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const bool act = el[q] > j;
      const int ii = act ? ei[q] : 0, ll = act ? el[q] : 0;
      const double u = fma(-colbuf[j & 1][ii], colbuf[j & 1][ll], a[q]);
      a[q] = act ? u : a[q];
      if (act && ii == j + 1 && ll == j + 1) piv[(j + 1) & 1] = u;
    }
    __syncthreads();
  }
  long long c1 = clock64();
  // L -> S
#pragma unroll
  for (int q = 0; q < PER; ++q) if (ei[q] >= 0) S[ei[q]][el[q]] = a[q];
  if (t < NB) rinv[t] = 0;  // placeholder
  __syncthreads();
  if (t < NB) rinv[t] = 1.0 / S[t][t];
  // inverse: acc init identity on owned elements
#pragma unroll
  for (int q = 0; q < PER; ++q) a[q] = (ei[q] == el[q]) ? 1.0 : 0.0;
  __syncthreads();
  long long c2 = clock64();
#pragma unroll 1
  for (int i = 0; i < NB; ++i) {
    const double ri = rinv[i];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const bool ci = ei[q] == i;
      const double v = a[q] * ri;
      a[q] = ci ? v : a[q];
      if (ci) xbuf[i & 1][el[q]] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const bool act = ei[q] > i && el[q] <= i;
      const int ii = act ? ei[q] : 0, ll = act ? el[q] : 0;
      const double u = fma(-S[ii][i], xbuf[i & 1][ll], a[q]);
      a[q] = act ? u : a[q];
    }
  }
  long long c3 = clock64();
#pragma unroll
  for (int q = 0; q < PER; ++q) if (ei[q] >= 0) { Lout[ei[q] * NB + el[q]] = S[ei[q]][el[q]]; Xout[ei[q] * NB + el[q]] = a[q]; }
  if (t == 0) { cyc[0] = c1 - c0; cyc[1] = c3 - c2; }
}
int main() {
  double h[NB * NB];
  for (int i = 0; i < NB; ++i) for (int j = 0; j < NB; ++j) h[i * NB + j] = (i == j ? 64.0 : 0.0) + 1.0 / (1 + i + j);
  double *M, *L, *X; long long* c;
  cudaMalloc(&M, sizeof h); cudaMalloc(&L, sizeof h); cudaMalloc(&X, sizeof h); cudaMalloc(&c, 16);
  cudaMemset(L, 0, sizeof h); cudaMemset(X, 0, sizeof h);
  cudaMemcpy(M, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) k<<<1, NT>>>(M, L, X, c);
  long long cy[2]; cudaMemcpy(cy, c, 16, cudaMemcpyDeviceToHost);
  double Lh[NB * NB], Xh[NB * NB];
  cudaMemcpy(Lh, L, sizeof h, cudaMemcpyDeviceToHost); cudaMemcpy(Xh, X, sizeof h, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < NB; ++i) for (int j = 0; j <= i; ++j) {
    double s = 0; for (int p = 0; p <= j; ++p) s += Lh[i * NB + p] * Lh[j * NB + p];
    e1 = fmax(e1, fabs(s - h[i * NB + j]));
    double u = 0; for (int p = j; p <= i; ++p) u += Lh[i * NB + p] * Xh[p * NB + j];
    e2 = fmax(e2, fabs(u - (i == j)));
  }
  printf("factor %lld cycles, inverse %lld cycles; |LL^T-M| %.2e |LX-I| %.2e (%s)\n", cy[0], cy[1], e1, e2, cudaGetErrorString(cudaGetLastError()));
}
