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

// Gaussian sketch entry pair for global column pair q = i >> 1 and sketch row
// k: Philox4x32-10(counter = (q_lo, q_hi, k, 0), key = (k0, k1)) -> two 53-bit
// uniforms u = (hi:lo >> 11) * 2^-53; Box-Muller with u1 = 1 - u_a in (0, 1]:
// z0 = sqrt(-2 ln u1) cos(2 pi u_b) (even column), z1 = ... sin(...) (odd).
__host__ __device__ inline void gaussian_pair_f64(uint64_t q, uint32_t k, uint32_t k0, uint32_t k1,
                                                  double& z0, double& z1) {
  philox4 c{(uint32_t)q, (uint32_t)(q >> 32), k, 0u};
  philox4 r = philox4x32_10(c, k0, k1);
  uint64_t a = ((uint64_t)r.y << 32) | r.x;
  uint64_t b = ((uint64_t)r.w << 32) | r.z;
  const double two_m53 = 1.1102230246251565e-16;  // 2^-53
  double ua = (double)(a >> 11) * two_m53;
  double ub = (double)(b >> 11) * two_m53;
  double u1 = 1.0 - ua;
  double rad = sqrt(-2.0 * log(u1));
  double th = 6.283185307179586 * ub;
  double s, co;
#if defined(__CUDA_ARCH__)
  sincos(th, &s, &co);
#else
  s = sin(th);
  co = cos(th);
#endif
  z0 = rad * co;
  z1 = rad * s;
}

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
