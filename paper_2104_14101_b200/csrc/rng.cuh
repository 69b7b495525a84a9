// Device-side views of the PCG64 stream and the Gaussian entry definition.
#pragma once
#include "common.cuh"
#include "pcg64.cuh"

namespace adask {

// Generator snapshot passed by value to kernels.
struct GenState {
  u128 st, inc;
  int has;
  uint32_t buf;
  static GenState from(const adask_pcg64& g) {
    GenState s;
    s.st = u128{g.state_hi, g.state_lo};
    s.inc = u128{g.inc_hi, g.inc_lo};
    s.has = g.has_uint32;
    s.buf = g.uinteger;
    return s;
  }
};

// Sequential reader of 32-bit draws starting at absolute draw index j of a
// generator snapshot (numpy next_uint32 semantics, buffered half first).
struct U32Stream {
  u128 st, inc;
  uint32_t hi_pending;
  bool have_hi;
  bool first_buf;
  uint32_t buf;
  __device__ U32Stream(const GenState& g, uint64_t j) : inc(g.inc) {
    first_buf = false;
    have_hi = false;
    buf = g.buf;
    st = g.st;
    if (g.has) {
      if (j == 0) {
        first_buf = true;
        return;
      }
      j -= 1;
    }
    // draw j of the unbuffered stream = half (j & 1) of 64-bit output j >> 1
    st = pcg_jump(g.st, inc, j >> 1);  // state before output j>>1
    if (j & 1) {
      st = pcg_step(st, inc);
      uint64_t v = pcg_output(st);
      hi_pending = (uint32_t)(v >> 32);
      have_hi = true;
    }
  }
  __device__ __forceinline__ uint32_t next() {
    if (first_buf) {
      first_buf = false;
      return buf;
    }
    if (have_hi) {
      have_hi = false;
      return hi_pending;
    }
    st = pcg_step(st, inc);
    uint64_t v = pcg_output(st);
    hi_pending = (uint32_t)(v >> 32);
    have_hi = true;
    return (uint32_t)v;
  }
};

// Gaussian sketch entries (the product's definition; oracle/philox_gaussian
// restates it).  For global A row i and sketch-row group g = k >> 2:
//   (o0, o1, o2, o3) = Philox4x32-10(counter = (i_lo, i_hi, g, 0), key = seed)
//   u_j = (o_j >> 9) * 2^-23                      (23-bit uniforms in [0, 1))
//   z0, z1 = sqrt(-2 ln(1 - u0)) * (cos, sin)(2 pi u1)
//   z2, z3 = sqrt(-2 ln(1 - u2)) * (cos, sin)(2 pi u3)
//   S[k, i] = z_{k & 3} / sqrt(m)
// One Philox call feeds four consecutive sketch rows of one column, so the
// tensor-core kernel (gauss_tc.cu) writes one 16-byte chunk per call.
__host__ __device__ inline void gaussian_quad_f64(uint64_t i, uint32_t g, uint32_t k0, uint32_t k1,
                                                  double z[4]) {
  philox4 c{(uint32_t)i, (uint32_t)(i >> 32), g, 0u};
  philox4 r = philox4x32_10(c, k0, k1);
  const double two_m23 = 1.1920928955078125e-07;  // 2^-23
  const uint32_t o[4] = {r.x, r.y, r.z, r.w};
  for (int p = 0; p < 2; ++p) {
    double ua = (double)(o[2 * p] >> 9) * two_m23;
    double ub = (double)(o[2 * p + 1] >> 9) * two_m23;
    double rad = sqrt(-2.0 * log(1.0 - ua));
    double th = 6.283185307179586 * ub;
    double s, co;
#if defined(__CUDA_ARCH__)
    sincos(th, &s, &co);
#else
    s = sin(th);
    co = cos(th);
#endif
    z[2 * p] = rad * co;
    z[2 * p + 1] = rad * s;
  }
}

// Rows [krow0, krow0 + mk) of the m_total-row Gaussian S (scale 1/sqrt(m_total)),
// columns [col0, col0 + ncols), row-major with leading dimension ldo.
int philox_gaussian_rows(adask_ctx* ctx, int dtype, int64_t krow0, int64_t mk, int64_t m_total, int64_t col0,
                         int64_t ncols, uint64_t key, void* out, int64_t ldo, cudaStream_t st);

// The same rows stored transposed (out[(i - col0) * ldo + (k - krow0)] = S[k, i], ldo >= mk).
int philox_gaussian_rows_t(adask_ctx* ctx, int dtype, int64_t krow0, int64_t mk, int64_t m_total, int64_t col0,
                           int64_t ncols, uint64_t key, void* out, int64_t ldo, cudaStream_t st);

// Items [item0, item0 + count) of Generator.integers(0, m, size=total_items)
// whose draws start at index `first`; *next = draw index after the last item
// of the whole call (total_items).
int pcg_integers_impl(adask_ctx* ctx, const adask_pcg64* g, uint64_t first, int64_t item0,
                      int64_t count, int64_t total_items, uint32_t m, int32_t* out, uint64_t* next,
                      cudaStream_t st);

// Packed sign bits (bit = 1 -> +1) of integers(0, 2, size=count) from draw `first`.
int pcg_sign_bits_impl(adask_ctx* ctx, const adask_pcg64* g, uint64_t first, int64_t count,
                       uint32_t* words, cudaStream_t st);

}  // namespace adask
