// Micro-benchmark: read bandwidth of the SRHT pass-1 access pattern
// (CTA = B rows x C columns of a row-major n x d fp64 matrix) vs row-contiguous
// streaming (dev tool).
#include <cstdio>
template <int B, int C, int TPB>
__global__ void __launch_bounds__(TPB) k_tile(const double* __restrict__ A, long d, double* out) {
  constexpr int NCW = C / 2;               // 16B vectors per row
  constexpr int ROWS = B * NCW / TPB;       // rows per thread
  const long blk = blockIdx.y, c0 = (long)blockIdx.x * C;
  const int cw = threadIdx.x % NCW, q = threadIdx.x / NCW;
  const double* p = A + (blk * B + (long)q * ROWS) * d + c0 + cw * 2;
  double s = 0;
  double2 v[ROWS];
#pragma unroll
  for (int e = 0; e < ROWS; ++e) { v[e] = __ldg(reinterpret_cast<const double2*>(p)); p += d; }
#pragma unroll
  for (int e = 0; e < ROWS; ++e) s += v[e].x + v[e].y;
  if (s == 12345.678) out[0] = s;
}
__global__ void k_stream(const double2* __restrict__ A, long n2, double* out) {
  double s = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    double2 v = __ldg(A + i); s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}
template <int B, int C, int TPB>
void run(const double* A, long n, long d, double* o) {
  dim3 g(d / C, n / B);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) k_tile<B, C, TPB><<<g, TPB>>>(A, d, o);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) k_tile<B, C, TPB><<<g, TPB>>>(A, d, o);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
  printf("tile B=%4d C=%3d TPB=%d: %.1f us  %.0f GB/s\n", B, C, TPB, ms * 1e3, n * d * 8 / ms / 1e6);
}
int main() {
  long n = 1 << 16, d = 1024;
  double *A, *o; cudaMalloc(&A, n * d * 8); cudaMalloc(&o, 8); cudaMemset(A, 0, n * d * 8);
  run<1024, 8, 128>(A, n, d, o);
  run<1024, 8, 256>(A, n, d, o);
  run<512, 16, 128>(A, n, d, o);
  run<256, 32, 128>(A, n, d, o);
  run<128, 64, 128>(A, n, d, o);
  run<64, 128, 128>(A, n, d, o);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_stream<<<148 * 8, 256>>>((const double2*)A, n * d / 2, o);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) k_stream<<<148 * 8, 256>>>((const double2*)A, n * d / 2, o);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
  printf("stream: %.1f us  %.0f GB/s\n", ms * 1e3, n * d * 8 / ms / 1e6);
}
