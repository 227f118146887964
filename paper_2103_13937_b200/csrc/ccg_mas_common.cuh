// ccg_mas_common.cuh -- device helpers shared by the MAS climb kernels (ccg_mas.cu,
// ccg_mas_tform.cu, ccg_mas_dform.cu, ccg_mas_ngram.cu): the per-worker letter windows over
// the numpy Philox stream (rng.py:81-89 next_distinct_pair(26)) and raw shared-memory
// accessors.
#pragma once
#include "ccg_internal.h"
#include "ccg_rng.cuh"

namespace ccg {

constexpr unsigned kFull = 0xffffffffu;

// full-warp shfl.sync.idx with clamp 0x1f: the source lane is bits [4:0] of `src_lane`
// (callers pass unmasked indices; __shfl_sync would mask them again)
__device__ __forceinline__ uint32_t shfl_idx_raw(uint32_t v, uint32_t src_lane) {
  uint32_t r;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v), "r"(src_lane));
  return r;
}

// 128 draws of one stream as letters int(u*26), 5 bits each.  Lane L holds the letters of
// draws base+4L .. base+4L+7 (its own Philox block plus lane L+1's), so the next FOUR
// letters -- two tries' pairs in the common no-redraw case -- come out of one 64-bit
// shuffle.  Offsets are 32-bit; the Philox key is re-read from global memory at refill
// time (keeps it out of registers).
struct LetterWindow {
  const uint64_t* key;  // &keys[2*w] (global)
  uint64_t base;        // stream index of window draw 0 (multiple of 4)
  uint64_t packed;
  uint32_t o;           // window offset of the next draw

  __device__ __forceinline__ void refill(int lane) {
    const uint64_t pos = base + o;
    base = pos & ~3ULL;
    o = (uint32_t)(pos & 3);
    uint64_t v0, v1, v2, v3;
    philox4x64_10(__ldg(key), __ldg(key + 1), (base >> 2) + 1 + (uint64_t)lane, v0, v1, v2, v3);
    const uint32_t p4 = int_below_small(v0, 26) | (int_below_small(v1, 26) << 5) |
                        (int_below_small(v2, 26) << 10) | (int_below_small(v3, 26) << 15);
    const uint32_t nxt = __shfl_down_sync(kFull, p4, 1);
    packed = (uint64_t)p4 | ((uint64_t)nxt << 20);
  }
  // letters of draws o .. o+3 in 5-bit fields; valid when o <= 124
  __device__ __forceinline__ uint32_t peek4() const {
    return (uint32_t)(shfl64(packed, (int)(o >> 2)) >> ((o & 3) * 5)) & 0xfffffu;
  }
  __device__ __forceinline__ int next(int lane) {
    if (o > 127) refill(lane);
    const uint32_t w = (uint32_t)(shfl64(packed, (int)(o >> 2)) >> ((o & 3) * 5));
    ++o;
    return (int)(w & 31u);
  }
  // rng.py:81-89 next_distinct_pair(26)
  __device__ __forceinline__ void pair(int lane, int& a, int& b) {
    a = next(lane);
    b = next(lane);
    while (b == a) b = next(lane);
  }
  __device__ __forceinline__ uint64_t position() const { return base + o; }
};

// 128 draws of one stream as letters int(u*26), one byte each.  Lane L holds the letters
// of draws base+4L .. base+4L+3 (its own Philox block) in `lo` and lane L+1's in `hi`,
// so the next four letters -- two tries' pairs when no redraw happens -- come out of two
// 32-bit shuffles and one funnel shift.  The Philox key is re-read from global memory at
// refill time (keeps it out of registers).
struct ByteWindow {
  const uint64_t* key;
  uint64_t base;  // stream index of window draw 0 (multiple of 4)
  uint32_t lo, hi;
  uint32_t o;     // window offset of the next draw
  uint32_t rk = 0;  // shared address of precomputed round keys (philox_round_keys), or 0

  __device__ __forceinline__ void refill(int lane) {
    const uint64_t pos = base + o;
    base = pos & ~3ULL;
    o = (uint32_t)(pos & 3);
    uint64_t v0, v1, v2, v3;
    const uint64_t ctr = (base >> 2) + 1 + (uint64_t)lane;
    if (rk)
      philox4x64_10_rk(rk, ctr, v0, v1, v2, v3);
    else
      philox4x64_10(__ldg(key), __ldg(key + 1), ctr, v0, v1, v2, v3);
    lo = int_below_tiny(v0, 26) | (int_below_tiny(v1, 26) << 8) |
         (int_below_tiny(v2, 26) << 16) | (int_below_tiny(v3, 26) << 24);
    hi = __shfl_down_sync(kFull, lo, 1);
  }
  // letters of draws o .. o+3, one per byte; valid when o <= 124
  __device__ __forceinline__ uint32_t peek4() const {
    const int src = (int)(o >> 2);
    const uint32_t x = __shfl_sync(kFull, lo, src), y = __shfl_sync(kFull, hi, src);
    return __funnelshift_r(x, y, (o & 3u) * 8u);
  }
  // letters of draws o .. o+7 (La: o..o+3, Lb: o+4..o+7); valid when o <= 120
  __device__ __forceinline__ void peek8(uint32_t& La, uint32_t& Lb) const {
    const int src = (int)(o >> 2);
    const uint32_t x0 = __shfl_sync(kFull, lo, src), x1 = __shfl_sync(kFull, hi, src);
    const uint32_t x2 = __shfl_sync(kFull, hi, src + 1);
    La = __funnelshift_r(x0, x1, (o & 3u) * 8u);
    Lb = __funnelshift_r(x1, x2, (o & 3u) * 8u);
  }
  __device__ __forceinline__ int next(int lane) {
    if (o > 127) refill(lane);
    const uint32_t x = __shfl_sync(kFull, lo, (int)(o >> 2));
    const int v = (int)((x >> ((o & 3u) * 8u)) & 0xffu);
    ++o;
    return v;
  }
  // rng.py:81-89 next_distinct_pair(26)
  __device__ __forceinline__ void pair(int lane, int& a, int& b) {
    a = next(lane);
    b = next(lane);
    while (b == a) b = next(lane);
  }
  __device__ __forceinline__ uint64_t position() const { return base + o; }
};

// 256 draws of one stream as letters int(u*26), one byte each, in two halves: lane L holds
// draws base+4L .. base+4L+3 in `A` and base+128+4L .. +3 in `B`.  A round that starts at
// offset o < 128 reads at most 66 draws from o on, so it always finds its 32 pairs in the
// window (a 128-draw window truncates about a third of the rounds); when o passes 128 the
// halves shift by one Philox block per lane.
struct ByteWindow2 {
  const uint64_t* key;
  uint64_t base;    // stream index of draw 0 of half A (multiple of 4)
  uint32_t A, B;
  uint32_t o;       // window offset of the next draw (0 .. 255)
  uint32_t rk = 0;  // shared address of precomputed round keys (philox_round_keys), or 0

  __device__ __forceinline__ uint32_t letters(uint64_t block) const {
    uint64_t v0, v1, v2, v3;
    if (rk)
      philox4x64_10_rk(rk, block + 1, v0, v1, v2, v3);
    else
      philox4x64_10(__ldg(key), __ldg(key + 1), block + 1, v0, v1, v2, v3);
    return letters4(v0, v1, v2, v3);
  }
  // int(u*26) of four words, one byte each: the 32-bit products decide all four unless one
  // lies within 26 of wrapping (probability ~2^-25 per word), when the exact path runs
  __device__ __forceinline__ static uint32_t letters4(uint64_t v0, uint64_t v1, uint64_t v2,
                                                      uint64_t v3) {
    const uint64_t A0 = (uint64_t)(uint32_t)(v0 >> 32) * 26u, A1 = (uint64_t)(uint32_t)(v1 >> 32) * 26u;
    const uint64_t A2 = (uint64_t)(uint32_t)(v2 >> 32) * 26u, A3 = (uint64_t)(uint32_t)(v3 >> 32) * 26u;
    const uint32_t hi = max(max((uint32_t)A0, (uint32_t)A1), max((uint32_t)A2, (uint32_t)A3));
    if (hi >= 0u - 26u)
      return int_below_tiny(v0, 26) | (int_below_tiny(v1, 26) << 8) |
             (int_below_tiny(v2, 26) << 16) | (int_below_tiny(v3, 26) << 24);
    const uint32_t q01 = __byte_perm((uint32_t)(A0 >> 32), (uint32_t)(A1 >> 32), 0x0040);
    const uint32_t q23 = __byte_perm((uint32_t)(A2 >> 32), (uint32_t)(A3 >> 32), 0x0040);
    return __byte_perm(q01, q23, 0x5410);
  }
  __device__ __forceinline__ void start(uint64_t pos, int lane) {
    base = pos & ~3ULL;
    o = (uint32_t)(pos & 3);
    A = letters((base >> 2) + (uint64_t)lane);
    B = letters((base >> 2) + 32 + (uint64_t)lane);
  }
  __device__ __forceinline__ void advance(int lane) {
    base += 128;
    o -= 128;
    A = B;
    B = letters((base >> 2) + 32 + (uint64_t)lane);
  }
  // Lane j's three letters at draws o+2j .. o+2j+2 (o < 128; byte 0 = draw o+2j).  The words
  // a round needs span 18 < 32 lanes, so each source lane offers the one half it is asked for.
  __device__ __forceinline__ uint32_t round_letters(int lane) const {
    const uint32_t src = (uint32_t)lane >= (o >> 2) ? A : B;
    const uint32_t pos = o + 2u * (uint32_t)lane;
    const uint32_t w = pos >> 2;
    // shfl.idx takes the source lane from bits [4:0] of the index (clamp 0x1f), and the
    // funnel shift's amount is taken mod 32: no masking needed
    const uint32_t x0 = shfl_idx_raw(src, w), x1 = shfl_idx_raw(src, w + 1u);
    return __funnelshift_r(x0, x1, pos * 8u);
  }
  __device__ __forceinline__ int next(int lane) {
    if (o > 255u) advance(lane);
    const uint32_t x = __shfl_sync(kFull, o < 128u ? A : B, (int)((o >> 2) & 31u));
    const int v = (int)((x >> ((o & 3u) * 8u)) & 0xffu);
    ++o;
    return v;
  }
  // rng.py:81-89 next_distinct_pair(26)
  __device__ __forceinline__ void pair(int lane, int& a, int& b) {
    a = next(lane);
    b = next(lane);
    while (b == a) b = next(lane);
  }
  __device__ __forceinline__ uint64_t position() const { return base + o; }
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return (int)v;
}

__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint2 lds_u64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

}  // namespace ccg
