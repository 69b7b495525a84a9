// PCG64 (XSL-RR 128/64, numpy.random.PCG64) and Philox4x32-10 for host and
// device.  The PCG64 stream is the one numpy's Generator consumes in the
// reference's sketches (embeddings.py:95-100, 117-124); it is restated here so
// the device can jump ahead to any draw index and generate signs / buckets
// in parallel, bit-exactly.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define ADASK_HD __host__ __device__ __forceinline__
#else
#define ADASK_HD inline
#endif

namespace adask {

struct u128 {
  uint64_t hi, lo;
};

ADASK_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

ADASK_HD u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
  return r;
}

ADASK_HD u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

// PCG64 multiplier 0x2360ED051FC65DA4_4385DF649FCCF645 (numpy pcg64.h).
ADASK_HD u128 pcg_mult() { return u128{0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}; }

ADASK_HD u128 pcg_step(u128 s, u128 inc) { return add128(mul128(s, pcg_mult()), inc); }

// XSL-RR output of a (new) state.
ADASK_HD uint64_t pcg_output(u128 s) {
  uint64_t x = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// State after `delta` LCG steps (O(log delta) jump-ahead).
ADASK_HD u128 pcg_jump(u128 s, u128 inc, uint64_t delta) {
  u128 acc_mult{0, 1}, acc_plus{0, 0};
  u128 cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, u128{0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, s), acc_plus);
}

// 64-bit output number k (0-based) of a generator whose current state is s:
// numpy steps first, then outputs, so output k is output(state after k+1 steps).
ADASK_HD uint64_t pcg_output_at(u128 s, u128 inc, uint64_t k) {
  return pcg_output(pcg_jump(s, inc, k + 1));
}

// Lemire bounded draw in [0, m) from one u32 (numpy buffered_bounded_lemire_uint32
// with rng = m-1): accepted iff low word >= (2^32 - m) mod m.
ADASK_HD uint32_t lemire_threshold(uint32_t m) { return (uint32_t)(0u - m) % m; }
ADASK_HD bool lemire_reject(uint32_t u, uint32_t m, uint32_t thr) {
  return (uint32_t)((uint64_t)u * m) < thr;
}
ADASK_HD uint32_t lemire_value(uint32_t u, uint32_t m) {
  return (uint32_t)(((uint64_t)u * m) >> 32);
}

// ---------------------------------------------------------------- Philox4x32-10
struct philox4 {
  uint32_t x, y, z, w;
};

ADASK_HD philox4 philox4x32_10(philox4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int i = 0; i < 10; ++i) {
    uint64_t p0 = (uint64_t)M0 * c.x;
    uint64_t p1 = (uint64_t)M1 * c.z;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    philox4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
    k0 += W0;
    k1 += W1;
  }
  return c;
}

}  // namespace adask
