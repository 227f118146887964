// ccg_rng.cuh -- device side of the reference's per-worker random streams.
//
// Reference: rng.py:58-97 (WorkerRng) wraps numpy.random.Generator(Philox(key=[seed, stream])).
// numpy's Philox is Philox4x64-10 with a 256-bit counter that is incremented BEFORE each
// block is generated (so block b of a stream uses counter b+1), and Generator.random()
// maps one 64-bit word x to (x >> 11) * 2^-53.  next_int_below(bound) is int(u * bound)
// (rng.py:43-47): an IEEE-754 double multiply, rounded to nearest-even, then truncated.
//
// Device design (B200): draws are produced a warp at a time -- a refill makes each lane
// compute ONE Philox block (4 words), so a warp produces 128 consecutive draws at once.
// The consumers keep them as letters in registers (ccg_mas_common.cuh ByteWindow /
// LetterWindow) or pre-shifted in shared memory (ccg_sct.cu Draws).
//
// int(u*bound) is emulated exactly in integer arithmetic (no FP64 pipe): with m = x>>11
// and P = m*bound (exact), the double product is P*2^-53 rounded to 53 significant bits;
// truncation differs from P>>53 only when that rounding carries into the next multiple of
// 2^53, i.e. when 2^53 - (P mod 2^53) <= 2^(s-1) with s = bitlen(P) - 53 (ties round up
// because the carried value has an even mantissa).  Verified against numpy in
// tests/test_oracle_golden.py and on device in tests/test_gpu_parity.py.
#pragma once
#include <stdint.h>

namespace ccg {

constexpr uint64_t kPhiloxM0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t kPhiloxM1 = 0xCA5A826395121157ULL;
constexpr uint64_t kPhiloxW0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kPhiloxW1 = 0xBB67AE8584CAA73BULL;

// Philox4x64-10 for counter (c0, 0, 0, 0) under key (k0, k1).
__device__ __forceinline__ void philox4x64_10(uint64_t k0, uint64_t k1, uint64_t c0,
                                              uint64_t& o0, uint64_t& o1, uint64_t& o2,
                                              uint64_t& o3) {
  uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = kPhiloxM0 * x0, hi0 = __umul64hi(kPhiloxM0, x0);
    const uint64_t lo1 = kPhiloxM1 * x2, hi1 = __umul64hi(kPhiloxM1, x2);
    const uint64_t n0 = hi1 ^ x1 ^ k0;
    const uint64_t n2 = hi0 ^ x3 ^ k1;
    x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  o0 = x0; o1 = x1; o2 = x2; o3 = x3;
}

// int((x >> 11) * 2^-53 * bound) exactly as CPython/numpy compute it, for 1 <= bound < 2^32.
__device__ __forceinline__ uint32_t int_below(uint64_t x, uint32_t bound) {
  const uint64_t m = x >> 11;
  const uint64_t lo = m * (uint64_t)bound;
  const uint64_t hi = __umul64hi(m, (uint64_t)bound);
  uint32_t q = (uint32_t)((lo >> 53) | (hi << 11));
  if (hi != 0 || lo >= (1ULL << 53)) {
    const int bitlen = hi ? 128 - __clzll(hi) : 64 - __clzll(lo);
    const int s = bitlen - 53;  // 1 <= s <= 32
    const uint64_t r = lo & ((1ULL << 53) - 1);
    if ((1ULL << 53) - r <= (1ULL << (s - 1))) ++q;
  }
  return q;
}

// Same for 1 <= bound < 2^11, where m*bound < 2^64 needs no high product word.
__device__ __forceinline__ uint32_t int_below_small(uint64_t x, uint32_t bound) {
  const uint64_t P = (x >> 11) * (uint64_t)bound;
  uint32_t q = (uint32_t)(P >> 53);
  if (P >= (1ULL << 53)) {
    const int s = (64 - __clzll(P)) - 53;
    if ((1ULL << 53) - (P & ((1ULL << 53) - 1)) <= (1ULL << (s - 1))) ++q;
  }
  return q;
}

// Same for 1 <= bound < 2^11 from the top 32 bits: with A = (x >> 32) * bound, the product
// m * bound (m = x >> 11) lies in [A, A + bound) * 2^21, so int(u*bound) = A >> 32 exactly --
// including the float rounding, whose carry needs a fraction within 2^10 of 1 -- unless the
// low word of A is within `bound` of wrapping (probability bound / 2^32), where the exact
// test above decides.
__device__ __forceinline__ uint32_t int_below_tiny(uint64_t x, uint32_t bound) {
  const uint64_t A = (uint64_t)(uint32_t)(x >> 32) * bound;
  if ((uint32_t)A < 0u - bound) return (uint32_t)(A >> 32);
  return int_below_small(x, bound);
}

// Philox4x64-10 with the ten round keys (k0 + r*W0, k1 + r*W1) precomputed in shared memory
// at `rk` (22 x u64, see philox_round_keys): one broadcast LDS.128 per round instead of two
// 64-bit key additions.  The counter is (c0, 0, 0, 0), so round 1 multiplies only x0 and
// leaves x0 = k0 for round 2, whose M0*k0 product is the same for every block of the stream:
// rk[20..21] hold it (one 64x64 multiply of twenty saved per block).
__device__ __forceinline__ void philox_round_keys(uint64_t* rk, uint64_t k0, uint64_t k1,
                                                  int lane) {
  if (lane < 10) {
    rk[2 * lane] = k0 + (uint64_t)lane * kPhiloxW0;
    rk[2 * lane + 1] = k1 + (uint64_t)lane * kPhiloxW1;
  }
  if (lane == 10) rk[20] = kPhiloxM0 * k0;
  if (lane == 11) rk[21] = __umul64hi(kPhiloxM0, k0);
}
__device__ __forceinline__ void philox4x64_10_rk(uint32_t rk, uint64_t c0, uint64_t& o0,
                                                 uint64_t& o1, uint64_t& o2, uint64_t& o3) {
  uint64_t k0, k1, pl, ph;
  // round 1: x = (c0, 0, 0, 0)
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(k0), "=l"(k1) : "r"(rk));
  const uint64_t lo0 = kPhiloxM0 * c0, hi0 = __umul64hi(kPhiloxM0, c0);
  uint64_t x2 = hi0 ^ k1, x3 = lo0;
  // round 2: x = (k0, 0, x2, x3) with M0*k0 precomputed
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(k0), "=l"(k1) : "r"(rk + 16u));
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(pl), "=l"(ph) : "r"(rk + 160u));
  const uint64_t lo1 = kPhiloxM1 * x2, hi1 = __umul64hi(kPhiloxM1, x2);
  uint64_t x0 = hi1 ^ k0, x1 = lo1;
  x2 = ph ^ x3 ^ k1;
  x3 = pl;
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(k0), "=l"(k1) : "r"(rk + 16u * r));
    const uint64_t a0 = kPhiloxM0 * x0, b0 = __umul64hi(kPhiloxM0, x0);
    const uint64_t a1 = kPhiloxM1 * x2, b1 = __umul64hi(kPhiloxM1, x2);
    const uint64_t n0 = b1 ^ x1 ^ k0;
    const uint64_t n2 = b0 ^ x3 ^ k1;
    x0 = n0; x1 = a1; x2 = n2; x3 = a0;
  }
  o0 = x0; o1 = x1; o2 = x2; o3 = x3;
}

// u in [0,1) exactly as numpy: (x >> 11) * 2^-53.
__device__ __forceinline__ double to_uniform(uint64_t x) {
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}

}  // namespace ccg
