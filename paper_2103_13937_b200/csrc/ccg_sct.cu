// ccg_sct.cu -- single-columnar-transposition (SCT) kernels for sm_100a.
//
// Reference path: sct.py:148-170 sct_worker.  n-gram extension: ORDER-letter windows
// (trigram/quadgram log tables, BASELINE.json config 3); ORDER 2 is the reference.  Start from permutation(k) (rng.py:91-97),
// then per try draw an operator (sct.py:69-79: element swaps, block swaps, block shift,
// sct.py:82-135), decrypt the whole ciphertext with the candidate key
// (ciphers.py:71-86 transposition_gather_map, irregular grid), score it as the float64
// sum of log2 bigram probabilities in NUMPY'S PAIRWISE ORDER (ngrams.py:172 / sct.py:160:
// `logs[idx].sum()`), and accept iff the candidate score is strictly greater.
//
// B200 design (warp per worker):
//  * The key is lane-distributed (lane l holds key positions l and l+32).  Every
//    operator is a gather cand[l] = key[src(l)] with src computed from warp-uniform draw
//    values, done with shuffles -- no key arrays in memory.
//  * Decryption is never materialised.  Plaintext position t sits in grid column c = t%k,
//    row r = t/k, and plain[t] = cipher[colstart[c] + r] where colstart[key[j]] is the
//    exclusive prefix sum of the segment lengths in key order (one warp scan per
//    candidate; column c has ceil(n/k) letters iff c < n%k, ciphers.py:79-81).
//  * numpy's pairwise sum (n <= 128: 8 strided accumulators, tree
//    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8 tail in order; n > 128: split at
//    n/2 rounded down to a multiple of 8 and recurse) is laid onto the warp: each leaf's 8
//    accumulators are 8 lanes (4 leaves per 32-lane "slot", up to 8 slots), the tree is
//    a 3-step xor butterfly (fp add is commutative, so every lane of the group holds the
//    identical rounded value), the tail is added in order, and the host-computed
//    post-order merge list (SumPlan) replays the recursion with shuffles.  The result is
//    bit-identical to numpy's float64 sum, so accept decisions match the reference.
//  * Tables: the 676 float64 log2 probabilities and each warp's ciphertext are staged in
//    shared memory; colstart is a per-warp 64-entry u16 array (conflict-free).
#include <cooperative_groups.h>
#include <cstdio>

#include "ccg_internal.h"
#include "ccg_rng.cuh"

namespace ccg {
namespace {
namespace cg = cooperative_groups;

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSctWarps = 8;

// raw shared-memory accessors on 32-bit shared addresses (ld/st.shared): the evaluator keeps
// its buffers' addresses in registers instead of letting the compiler rebuild the shared
// window base (S2R + uniform arithmetic) at every access
__device__ __forceinline__ uint32_t pin_smem(const void* p) {
  uint32_t a;
  asm volatile("mov.u32 %0, %1;" : "=r"(a) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return a;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double ldsf64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// The worker's draw window: 128 consecutive raw draws of its stream in shared memory
// (one Philox4x64-10 block per lane per refill, rng.py:68-75), so a scalar draw is one
// broadcast 64-bit shared load.  Every SCT bound is < 2^11 (100, hops, k <= 64, ...), so
// int(u*bound) uses the single-product exact conversion (ccg_rng.cuh int_below_small).
__device__ __noinline__ int slow_below(uint64_t m, uint32_t bound) {
  return (int)int_below_small(m << 11, bound);
}

struct Draws {
  const uint64_t* key;  // &keys[2*w] (global; re-read at refill)
  uint32_t win;         // shared address of the 128-slot window; slot j holds draw base+j >> 11
  uint64_t base;        // stream index of window slot 0 (multiple of 4)
  uint32_t o;           // window slot of the next draw

  // out of line: one copy of the Philox block instead of one per draw site (the climb loop
  // was instruction-fetch bound with it inlined everywhere)
  __device__ __noinline__ void refill(int lane) {
    base += o & ~3u;
    o &= 3u;
    uint64_t v0, v1, v2, v3;
    philox4x64_10(__ldg(key), __ldg(key + 1), (base >> 2) + 1 + (uint64_t)lane, v0, v1, v2, v3);
    __syncwarp();
    const uint32_t a = win + 32u * (uint32_t)lane;
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(v0 >> 11), "l"(v1 >> 11)
                 : "memory");
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a + 16u), "l"(v2 >> 11), "l"(v3 >> 11)
                 : "memory");
    __syncwarp();
  }
  __device__ __forceinline__ void start(uint64_t pos, int lane) {
    base = pos & ~3ULL;
    o = 0;
    refill(lane);
    o = (uint32_t)(pos & 3);
  }
  __device__ __forceinline__ uint64_t position() const { return base + o; }
  // rng.py:77-79: int(u * bound) for the next draw, 1 <= bound < 2^11, m = x >> 11.  The top
  // 32 bits of the draw give it with one 32x32 product unless the product's low word is
  // within `bound` of wrapping (probability < 2^-21), when the exact 64-bit conversion runs.
  __device__ __forceinline__ int below(uint32_t bound, int lane) {
    if (o > 127u) refill(lane);
    uint64_t m;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(m) : "r"(win + 8u * o));
    ++o;
    const uint64_t A = (uint64_t)(uint32_t)(m >> 21) * bound;
    if ((uint32_t)A < 0u - bound) return (int)(A >> 32);
    return slow_below(m, bound);
  }
  // rng.py:81-89
  __device__ __forceinline__ void pair(uint32_t bound, int lane, int& a, int& b) {
    a = below(bound, lane);
    b = below(bound, lane);
    while (b == a) b = below(bound, lane);
  }
};

// Lane-distributed key of length k <= 64: v0 = key[lane], v1 = key[lane + 32].
struct Key {
  int v0, v1;
  __device__ __forceinline__ int at(int i) const {  // i warp-uniform
    return i < 32 ? __shfl_sync(kFull, v0, i) : __shfl_sync(kFull, v1, i - 32);
  }
  // out[l] = this[src(l)] for the two positions owned by the lane
  __device__ __forceinline__ Key gather(int s0, int s1, bool wide) const {
    Key o;
    const int a0 = __shfl_sync(kFull, v0, s0 & 31);
    if (!wide) {
      o.v0 = a0;
      o.v1 = v1;
      return o;
    }
    const int b0 = __shfl_sync(kFull, v1, s0 & 31);
    const int a1 = __shfl_sync(kFull, v0, s1 & 31);
    const int b1 = __shfl_sync(kFull, v1, s1 & 31);
    o.v0 = s0 < 32 ? a0 : b0;
    o.v1 = s1 < 32 ? a1 : b1;
    return o;
  }
  template <bool MAYBE_WIDE = true>
  __device__ __forceinline__ void swap_pos(int i, int j, int lane) {
    if (!MAYBE_WIDE) {  // k <= 32: positions live in v0 only
      const int vi = __shfl_sync(kFull, v0, i), vj = __shfl_sync(kFull, v0, j);
      if (lane == i) v0 = vj;
      if (lane == j) v0 = vi;
      return;
    }
    const int vi = at(i), vj = at(j);
    if (lane == i) v0 = vj;
    if (lane == j) v0 = vi;
    if (lane + 32 == i) v1 = vj;
    if (lane + 32 == j) v1 = vi;
  }
};

// Per-lane static part of the sum plan for one slot.
struct SlotPlan {
  int leaf;       // leaf id handled by this lane's 8-lane group in this slot (-1: none)
  int count;      // strided terms per accumulator (len/8, 0 for a sequential leaf)
  int tail;       // terms added in order after the tree
  int mtail;      // the largest tail in the warp (warp-uniform loop bound)
  int p0;         // plaintext position of this lane's first strided term
  int pt;         // position of the first tail term
};

template <int SLOTS, int ORDER>
struct Evaluator {
  SlotPlan sp[SLOTS];
  int k, n, base, rem;
  int c0, r0, qs, rs;  // grid position of plaintext position 4*lane; 128 = qs*k + rs
  int n4, tc, tr;      // n rounded down to 128; grid position of plaintext position n4+lane
  const SumPlan* plan;

  // the key length may change per worker (ragged SCT batches)
  __device__ __forceinline__ void set_k(int k_, int lane) {
    k = k_;
    base = n / k;
    rem = n - base * k;
    qs = 128 / k;
    rs = 128 - qs * k;
    r0 = 4 * lane / k;
    c0 = 4 * lane - r0 * k;
    n4 = n & ~127;
    tr = (n4 + lane) / k;
    tc = n4 + lane - tr * k;
  }

  __device__ void init(const SumPlan& P, int k_, int n_, int lane) {
    plan = &P;
    n = n_;
    set_k(k_, lane);
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int leaf = 4 * s + (lane >> 3);
      SlotPlan& q = sp[s];
      if (leaf < P.n_leaves) {
        const int len = P.leaf_len[leaf], start = P.leaf_start[leaf];
        q.leaf = leaf;
        q.count = len >= 8 ? len / 8 : 0;
        q.tail = len >= 8 ? len % 8 : len;
        q.p0 = start + (lane & 7);
        q.pt = start + 8 * q.count;
      } else {
        q.leaf = -1;
        q.count = 0;
        q.tail = 0;
        q.p0 = q.pt = 0;
      }
      q.mtail = (int)__reduce_max_sync(kFull, (unsigned)q.tail);
    }
  }

  // log-probability of the window of ORDER plaintext letters starting at position t
  __device__ __forceinline__ double term(uint32_t plain, uint32_t slogs, const double* logs,
                                        int t) const {
    int idx = (int)lds8(plain + (uint32_t)t);
#pragma unroll
    for (int j = 1; j < ORDER; ++j) idx = idx * kAlpha + (int)lds8(plain + (uint32_t)(t + j));
    if (ORDER == 2) return ldsf64(slogs + 8u * (uint32_t)idx);
    return __ldg(logs + idx);  // trigram/quadgram tables are read through L1/L2
  }

  // Score of decrypting txt with the lane-distributed key.
  // MAYBE_WIDE = false: the caller guarantees k <= 32 (no second key register)
  template <bool MAYBE_WIDE = true>
  __device__ double score(const Key& key, const uint8_t* txt_p, uint16_t* colstart_p,
                          uint8_t* plain_p, const double* logs, int lane) const {
    const uint32_t txt = pin_smem(txt_p), colstart = pin_smem(colstart_p);
    const uint32_t plain = pin_smem(plain_p);
    const uint32_t slogs = ORDER == 2 ? pin_smem(logs) : 0u;
    // colstart[key[j]] = sum of segment lengths of key positions < j (ciphers.py:79-86)
    const bool wide = MAYBE_WIDE && k > 32;
    const int len0 = lane < k ? base + (key.v0 < rem ? 1 : 0) : 0;
    const int len1 = lane + 32 < k ? base + (key.v1 < rem ? 1 : 0) : 0;
    int inc0 = len0, inc1 = len1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u0 = __shfl_up_sync(kFull, inc0, o);
      if (lane >= o) inc0 += u0;
      if (wide) {
        const int u1 = __shfl_up_sync(kFull, inc1, o);
        if (lane >= o) inc1 += u1;
      }
    }
    __syncwarp();
    if (lane < k) sts16(colstart + 2u * (uint32_t)key.v0, (uint32_t)(inc0 - len0));
    if (wide) {
      const int tot0 = __shfl_sync(kFull, inc0, 31);
      if (lane + 32 < k) sts16(colstart + 2u * (uint32_t)key.v1, (uint32_t)(tot0 + inc1 - len1));
    }
    __syncwarp();
    // decrypt (ciphers.py:107-113): plain[t] = cipher[colstart[t % k] + t / k], four
    // consecutive positions per lane and one 32-bit store (positions past n land in the
    // buffer's padding and are never read)
    {
      int c = c0, r = r0;
      // a remainder of at most 32 positions is one position per lane, not a 4-wide round
      const int end = n - n4 <= 32 ? n4 : n;
      for (int t = 4 * lane; t < end; t += 128) {
        uint32_t wd = 0;
        int cc = c, rr = r;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          wd |= lds8(txt + lds16(colstart + 2u * (uint32_t)cc) + (uint32_t)rr) << (8 * q);
          if (++cc == k) {
            cc = 0;
            ++rr;
          }
        }
        sts32(plain + (uint32_t)t, wd);
        c += rs;
        r += qs;
        if (c >= k) {
          c -= k;
          ++r;
        }
      }
      if (end == n4 && n4 + lane < n)
        sts8(plain + (uint32_t)(n4 + lane), lds8(txt + lds16(colstart + 2u * (uint32_t)tc) + (uint32_t)tr));
    }
    __syncwarp();

    double res[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const SlotPlan& q = sp[s];
      double acc = 0.0;
      int t = q.p0;
      for (int i = 0; i < q.count; ++i, t += 8) {
        const double v = term(plain, slogs, logs, t);
        acc = i == 0 ? v : acc + v;
      }
      // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) as an xor butterfly over the 8-lane group
      acc += __shfl_xor_sync(kFull, acc, 1);
      acc += __shfl_xor_sync(kFull, acc, 2);
      acc += __shfl_xor_sync(kFull, acc, 4);
      // the tail terms follow in order (numpy pairwise_sum): lane j of the group evaluates
      // tail term j, the additions run through shuffles
      double tv = 0.0;
      if ((lane & 7) < q.tail) tv = term(plain, slogs, logs, q.pt + (lane & 7));
      for (int u = 0; u < q.mtail; ++u) {
        const double v = __shfl_sync(kFull, tv, (lane & ~7) | u);
        if (u < q.tail) acc += v;
      }
      res[s] = acc;
    }
    // leaf sums to lanes: lane L gets leaf L (slot L / 4, 8-lane group L % 4)
    double lv = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const double v = __shfl_sync(kFull, res[s], 8 * (lane & 3));
      if ((lane >> 2) == s) lv = v;
    }
    // replay the recursion's merges (post-order): leaf[dst] = leaf[dst] + leaf[src]
    const SumPlan& P = *plan;
    for (int m = 0; m < P.n_merges; ++m) {
      const double sv = __shfl_sync(kFull, lv, P.merge_src[m]);
      if (lane == P.merge_dst[m]) lv = lv + sv;
    }
    const double out = __shfl_sync(kFull, lv, 0);
    __syncwarp();  // plain / colstart are rewritten by the next candidate
    return out;
  }
};

__device__ __forceinline__ void stage_text(uint8_t* dst, const uint8_t* __restrict__ src, int n,
                                           int lane) {
  for (int i = lane; i < n; i += 32) dst[i] = src[i];
  __syncwarp();
}

// the bigram table is staged in shared memory; higher orders stay in global memory
template <int ORDER>
__device__ __forceinline__ const double* stage_logs(double* logs, const double* __restrict__ g) {
  if (ORDER != 2) return g;
  for (int i = threadIdx.x; i < kAlpha * kAlpha; i += blockDim.x) logs[i] = g[i];
  __syncthreads();
  return logs;
}

__host__ __device__ __forceinline__ size_t text_stride(int n) { return ((size_t)n + 15) & ~(size_t)15; }

// Shared layout: [bigram log table 676 x f64] then per warp
// [draw window 128 x u64][colstart 64 x u16][ciphertext][decrypted candidate].
constexpr size_t kLogsBytes = kAlpha * kAlpha * sizeof(double);
constexpr size_t kWinBytes = 128 * sizeof(uint64_t);
__host__ __device__ __forceinline__ size_t sct_warp_bytes(int n) {
  return kWinBytes + kSctMaxKey * 2 + 2 * text_stride(n);
}
struct WarpSmem {
  uint32_t win;
  uint16_t* colstart;
  uint8_t* txt;
  uint8_t* plain;
  __device__ WarpSmem(unsigned char* smem, int warp, int n) {
    unsigned char* b = smem + kLogsBytes + (size_t)warp * sct_warp_bytes(n);
    win = (uint32_t)__cvta_generic_to_shared(b);
    colstart = reinterpret_cast<uint16_t*>(b + kWinBytes);
    txt = b + kWinBytes + kSctMaxKey * 2;
    plain = txt + text_stride(n);
  }
};

// sct.py:82-89 apply_element_swaps
template <bool MAYBE_WIDE = true>
__device__ __forceinline__ void op_element_swaps(Key& c, Draws& d, int k, int max_hops, int lane) {
  const int hops = 1 + d.below((uint32_t)max_hops, lane);
  for (int h = 0; h < hops; ++h) {
    int i, j;
    d.pair((uint32_t)k, lane, i, j);
    c.template swap_pos<MAYBE_WIDE>(i, j, lane);
  }
}

// sct.py:92-112 apply_block_swaps
template <bool MAYBE_WIDE = true>
__device__ __forceinline__ void op_block_swaps(Key& c, Draws& d, int k, int max_hops, int lane) {
  const int hops = 1 + d.below((uint32_t)max_hops, lane);
  for (int h = 0; h < hops; ++h) {
    const int len = 1 + d.below((uint32_t)(k / 2), lane);
    int p, q;
    d.pair((uint32_t)(k - len + 1), lane, p, q);
    while (abs(p - q) < len) d.pair((uint32_t)(k - len + 1), lane, p, q);
    if (p > q) { const int t = p; p = q; q = t; }
    auto src = [&](int l) {
      if (l >= p && l < p + len) return l - p + q;
      if (l >= q && l < q + len) return l - q + p;
      return l;
    };
    c = c.gather(src(lane), src(lane + 32), MAYBE_WIDE && k > 32);
  }
}

// sct.py:115-135 apply_block_shift
template <bool MAYBE_WIDE = true>
__device__ __forceinline__ void op_block_shift(Key& c, Draws& d, int k, int lane) {
  const int len = 1 + d.below((uint32_t)(k - 1), lane);
  const int starts = k - len + 1;
  const int p = d.below((uint32_t)starts, lane);
  int dest = d.below((uint32_t)starts, lane);
  while (dest == p) dest = d.below((uint32_t)starts, lane);
  const int lo = min(p, dest), hi = max(p, dest) + len, w = hi - lo;
  const int sh = dest > p ? len : w - len;  // window[len:]+window[:len]  /  window[-len:]+window[:-len]
  auto src = [&](int l) {
    if (l >= lo && l < hi) {
      int i = l - lo + sh;
      if (i >= w) i -= w;
      return lo + i;
    }
    return l;
  };
  c = c.gather(src(lane), src(lane + 32), MAYBE_WIDE && k > 32);
}

// The draws of one proposal without building it (sct.py:69-135: the operator choice and
// every operator's draws depend only on the stream and k, never on the key).
__device__ __forceinline__ void skip_proposal(Draws& d, int k, int p1, int p2, int hop1, int hop2,
                                           int lane) {
  const int u = d.below(100u, lane);
  int a, b;
  if (u < p1) {
    const int hops = 1 + d.below((uint32_t)hop1, lane);
    for (int h = 0; h < hops; ++h) d.pair((uint32_t)k, lane, a, b);
  } else if (u < p2) {
    const int hops = 1 + d.below((uint32_t)hop2, lane);
    for (int h = 0; h < hops; ++h) {
      const int len = 1 + d.below((uint32_t)(k / 2), lane);
      d.pair((uint32_t)(k - len + 1), lane, a, b);
      while (abs(a - b) < len) d.pair((uint32_t)(k - len + 1), lane, a, b);
    }
  } else {
    const int len = 1 + d.below((uint32_t)(k - 1), lane);
    const int starts = k - len + 1;
    a = d.below((uint32_t)starts, lane);
    b = d.below((uint32_t)starts, lane);
    while (b == a) b = d.below((uint32_t)starts, lane);
  }
}

template <int SLOTS, int ORDER, bool MAYBE_WIDE>
__global__ void __launch_bounds__(kSctWarps * 32, 4)
    sct_climb_kernel(const SctLaunch p, const __grid_constant__ SumPlan plan) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const WarpSmem ws(smem, warp, p.n);
  const double* logs = stage_logs<ORDER>(reinterpret_cast<double*>(smem), p.logs);

  Evaluator<SLOTS, ORDER> ev;
  ev.init(plan, p.k, p.n, lane);
  const int kmax = p.k;  // keys_out stride
  const int64_t stride = (int64_t)gridDim.x * kSctWarps;

  const WorkerTickets tk{p.tickets, stride};
  for (int64_t w = (int64_t)blockIdx.x * kSctWarps + warp; w < p.n_workers; w = tk.next(w, lane)) {
    const int32_t cid = p.cipher_of[w];
    const int k = p.key_lengths ? p.key_lengths[w] : kmax;
    if (p.key_lengths) ev.set_k(k, lane);
    stage_text(ws.txt, p.ciphers + p.offsets[cid], p.n, lane);
    Draws d;
    d.key = p.keys + 2 * w;
    d.win = ws.win;
    d.start(p.skips ? p.skips[w] : 0, lane);

    // rng.py:91-97 permutation(k): Fisher-Yates from the top
    Key key;
    key.v0 = lane;
    key.v1 = lane + 32;
    for (int i = k - 1; i > 0; --i) {
      const int j = d.below((uint32_t)(i + 1), lane);
      key.template swap_pos<MAYBE_WIDE>(i, j, lane);
    }
    // t = -1 scores the start key (sct.py:157); one call site keeps a single inlined copy of
    // the evaluator in the loop (the kernel is instruction-fetch sensitive)
    double score = 0.0;
    int64_t last = -1, t = -1;
    for (; t < p.climbings; ++t) {
      Key cand = key;
      if (t >= 0) {
        const int u = d.below(100u, lane);
        if (u < p.p1)
          op_element_swaps<MAYBE_WIDE>(cand, d, k, p.op1_hop, lane);
        else if (u < p.p2)
          op_block_swaps<MAYBE_WIDE>(cand, d, k, p.op2_hop, lane);
        else
          op_block_shift<MAYBE_WIDE>(cand, d, k, lane);
      }
      const double cs = ev.template score<MAYBE_WIDE>(cand, ws.txt, ws.colstart, ws.plain, logs, lane);
      if (t < 0) {
        score = cs;
      } else if (cs > score) {
        key = cand;
        score = cs;
        last = t;
      }
    }
    if (lane < k) p.keys_out[w * kmax + lane] = (uint8_t)key.v0;
    if (lane + 32 < k) p.keys_out[w * kmax + lane + 32] = (uint8_t)key.v1;
    if (lane == 0) {
      p.scores[w] = score;
      if (p.draws_used) p.draws_used[w] = d.position();
      if (p.last_accept) p.last_accept[w] = last;
      if (p.tries_done) p.tries_done[w] = t;
    }
    __syncwarp();
  }
}

// Latency mode (few workers: a time-to-recover solve runs 64): one CTA of P warps per
// worker, evaluating P consecutive proposals at once.  Proposals never read the key to
// choose their draws, and a rejected proposal leaves the key unchanged, so warp j builds
// proposal t+j from the current key after replaying the draws of proposals t..t+j-1; the
// first proposal whose score beats the current one is accepted (exactly the sequential
// outcome), everything after it is discarded and the stream resumes right after it.
struct SpecExchange {
  double score[16];
  uint64_t end[16];  // draw position after each warp's proposal
  uint8_t key[kSctMaxKey];
};

template <int SLOTS, int ORDER, int P>
__global__ void __launch_bounds__(P * 32, P >= 32 ? 1 : 32 / P)
    sct_climb_spec_kernel(const SctLaunch p, const __grid_constant__ SumPlan plan) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const WarpSmem ws(smem, warp, p.n);
  const double* logs = stage_logs<ORDER>(reinterpret_cast<double*>(smem), p.logs);
  // two exchange buffers, alternated by round: a round's writes never meet the previous
  // round's reads, so a round needs one block barrier (two when it accepts)
  SpecExchange* exb = reinterpret_cast<SpecExchange*>(smem + kLogsBytes + P * sct_warp_bytes(p.n));

  Evaluator<SLOTS, ORDER> ev;
  ev.init(plan, p.k, p.n, lane);
  const int kmax = p.k;
  const int64_t climbings = p.climbings;

  for (int64_t w = blockIdx.x; w < p.n_workers; w += gridDim.x) {
    const int32_t cid = p.cipher_of[w];
    const int k = p.key_lengths ? p.key_lengths[w] : kmax;
    if (p.key_lengths) ev.set_k(k, lane);
    stage_text(ws.txt, p.ciphers + p.offsets[cid], p.n, lane);
    Draws d;
    d.key = p.keys + 2 * w;
    d.win = ws.win;
    d.start(p.skips ? p.skips[w] : 0, lane);
    Key key;
    key.v0 = lane;
    key.v1 = lane + 32;
    for (int i = k - 1; i > 0; --i) {  // rng.py:91-97
      const int j = d.below((uint32_t)(i + 1), lane);
      key.swap_pos(i, j, lane);
    }
    double score = 0.0;
    int64_t last = -1, t = 0;
    uint32_t rnd = 0;
    bool first = true;  // the first pass scores the start key (one evaluator call site)
    while (first || t < climbings) {
      Key cand = key;
      const bool mine = !first && t + warp < climbings;
      if (mine) {
        for (int j = 0; j < warp; ++j) skip_proposal(d, k, p.p1, p.p2, p.op1_hop, p.op2_hop, lane);
        const int u = d.below(100u, lane);
        if (u < p.p1)
          op_element_swaps(cand, d, k, p.op1_hop, lane);
        else if (u < p.p2)
          op_block_swaps(cand, d, k, p.op2_hop, lane);
        else
          op_block_shift(cand, d, k, lane);
      }
      double cs = 0.0;
      if (first || mine) cs = ev.score(cand, ws.txt, ws.colstart, ws.plain, logs, lane);
      if (first) {
        score = cs;
        first = false;
        continue;
      }
      SpecExchange& ex = exb[rnd++ & 1u];
      if (lane == 0) {
        ex.score[warp] = cs;
        ex.end[warp] = d.position();
      }
      __syncthreads();
      const int avail = climbings - t < P ? (int)(climbings - t) : P;
      int acc = -1;
      for (int j = 0; j < avail; ++j)
        if (ex.score[j] > score) {
          acc = j;
          break;
        }
      const int used = acc >= 0 ? acc : avail - 1;  // the last proposal consumed
      const uint64_t pos = ex.end[used];
      if (acc >= 0) {  // block-uniform: every thread read the same scores
        if (warp == acc) {
          if (lane < k) ex.key[lane] = (uint8_t)cand.v0;
          if (lane + 32 < k) ex.key[lane + 32] = (uint8_t)cand.v1;
        }
        const double next_score = ex.score[acc];
        __syncthreads();
        key.v0 = lane < k ? ex.key[lane] : lane;
        key.v1 = lane + 32 < k ? ex.key[lane + 32] : lane + 32;
        score = next_score;
        last = t + acc;
      }
      t += used + 1;
      // resume every warp's stream right after the last proposal consumed
      if (pos >= d.base && pos - d.base < 128)
        d.o = (uint32_t)(pos - d.base);
      else
        d.start(pos, lane);
    }
    if (warp == 0) {
      if (lane < k) p.keys_out[w * kmax + lane] = (uint8_t)key.v0;
      if (lane + 32 < k) p.keys_out[w * kmax + lane + 32] = (uint8_t)key.v1;
      if (lane == 0) {
        p.scores[w] = score;
        if (p.draws_used) p.draws_used[w] = d.position();
        if (p.last_accept) p.last_accept[w] = last;
        if (p.tries_done) p.tries_done[w] = t;
      }
    }
    __syncthreads();
  }
}

// ---- Latency mode, chain-parsed (sct_climb_chain_kernel) ----
// The speculative kernel above makes warp j replay the draws of j proposals before it can
// build its own, every round: the round lasts as long as warp P-1's serial replay.  But the
// proposal sequence is a pure function of the stream (sct.py:69-135 never read the key, and
// an accepted proposal is followed by exactly the proposal that follows it in the stream),
// so it can be parsed once, ahead of the climb, and in parallel:
//   1. the CTA generates a chunk of kChainDraws consecutive draws into shared memory;
//   2. every thread parses the proposal that WOULD start at each of its draw offsets and
//      records where it ends (one table of end offsets for the whole chunk);
//   3. one thread follows end[] from the chunk's entry offset: the chain of true proposal
//      starts (one shared load per proposal);
//   4. the chain's proposals are parsed again, one per thread, into 16-byte descriptors
//      (operator + up to kSctLaneMaxHops position events).
// A round is then: warp j applies descriptor t+j to the current key and scores it; the first
// improvement is accepted (sct.py:168) and the next round starts at the proposal after it.
constexpr int kChainDraws = 4096;               // draws per parsed chunk
constexpr int kChainMaxProps = kChainDraws / 4;  // every proposal reads at least 4 draws
constexpr uint16_t kChainOvf = 0xffffu;          // the proposal runs past the chunk
constexpr int kChainJumps = 5;
constexpr int kChainBudget = 24;                 // draws per proposal in the first parse pass
#ifndef CCG_CHAIN_STEPS
#define CCG_CHAIN_STEPS 4
#endif
constexpr int kChainSteps = CCG_CHAIN_STEPS;     // first-pass automaton steps per bookkeeping round
constexpr size_t kMaxSmemPerBlock = 227 * 1024;  // sm_100 opt-in dynamic shared memory per block                   // jump tables of 1, 2, 4, 8, 16 proposals

struct ChainSmem {
  uint32_t hi[kChainDraws];            // top 32 bits of each draw of the chunk (rng.py:68-75)
  uint16_t jump[kChainJumps][kChainDraws];  // jump[b][i]: offset 2^b proposals after i (>= kChainDraws: none)
  uint16_t start[kChainMaxProps];      // the chain: start offsets of consecutive proposals
  uint4 desc[kChainDraws];             // the proposal at each offset: x = op | events << 4,
                                       // y, z, w = events (a | b << 8 | len << 16)
  double score[2][32];                 // round exchange, alternated by round
  uint8_t key[kSctMaxKey];
  int n, next;                         // proposals in the chain; offset of the one after them
  uint16_t queue[kChainDraws];         // offsets whose proposal outran the first pass's budget
  int ticket, n_queued;                // next item to parse; queue length (chain_parse_lockstep)
  uint32_t ptab[20];                   // parse automaton table (chain_parse_table)
#ifdef CCG_CHAIN_PROFILE
  long long prof[5];                   // cycles per parse phase (CCG_CHAIN_PROFILE builds)
#endif
};

// int(u*bound) of stream draw `pos` from its full 53-bit mantissa (the 32-bit test failed)
__device__ __noinline__ int chain_exact_below(uint64_t k0, uint64_t k1, uint64_t pos, uint32_t bound) {
  uint64_t v[4];
  philox4x64_10(k0, k1, (pos >> 2) + 1, v[0], v[1], v[2], v[3]);
  return (int)int_below_small(v[pos & 3], bound);
}
__device__ __noinline__ uint32_t chain_direct_hi(uint64_t k0, uint64_t k1, uint64_t pos) {
  uint64_t v[4];
  philox4x64_10(k0, k1, (pos >> 2) + 1, v[0], v[1], v[2], v[3]);
  return (uint32_t)(v[pos & 3] >> 32);
}

// The proposal starting at draw offset i of the chunk whose draw 0 is stream index `base`
// (sct.py:69-135; the same draws as skip_proposal / op_*): returns its end offset, or -1 when
// it needs a draw at or past `lim`.  hi == nullptr reads the stream directly (no limit).
__device__ __noinline__ int chain_parse(const uint32_t* hi, int lim, int i, uint64_t base,
                                        uint64_t k0, uint64_t k1, int k, int p1, int p2, int h1,
                                        int h2, uint4* out) {
  auto draw = [&](uint32_t bound, int& v) -> bool {
    uint32_t h;
    if (hi) {
      if (i >= lim) return false;
      h = hi[i];
    } else {
      h = chain_direct_hi(k0, k1, base + (uint64_t)i);
    }
    const uint64_t A = (uint64_t)h * bound;
    v = (uint32_t)A < 0u - bound ? (int)(A >> 32) : chain_exact_below(k0, k1, base + (uint64_t)i, bound);
    ++i;
    return true;
  };
  uint32_t e0 = 0u, e1 = 0u, e2 = 0u;  // the events (registers, not a local array)
  int v, op, nev = 0;
  auto put = [&](uint32_t x) {
    if (nev == 0) e0 = x; else if (nev == 1) e1 = x; else e2 = x;
    ++nev;
  };
  if (!draw(100u, v)) return -1;  // sct.py:69-79 select_operator
  if (v < p1) {                   // sct.py:82-89 apply_element_swaps
    op = 1;
    if (!draw((uint32_t)h1, v)) return -1;
    for (int h = 1 + v; h > 0; --h) {
      int a;
      if (!draw((uint32_t)k, a)) return -1;
      do {
        if (!draw((uint32_t)k, v)) return -1;
      } while (v == a);
      put((uint32_t)a | ((uint32_t)v << 8));
    }
  } else if (v < p2) {  // sct.py:92-112 apply_block_swaps
    op = 2;
    if (!draw((uint32_t)h2, v)) return -1;
    for (int h = 1 + v; h > 0; --h) {
      int len, a;
      if (!draw((uint32_t)(k / 2), len)) return -1;
      ++len;
      const uint32_t m = (uint32_t)(k - len + 1);
      for (;;) {  // the whole pair is redrawn while |p - q| < len
        if (!draw(m, a)) return -1;
        do {
          if (!draw(m, v)) return -1;
        } while (v == a);
        if (abs(a - v) >= len) break;
      }
      put((uint32_t)min(a, v) | ((uint32_t)max(a, v) << 8) | ((uint32_t)len << 16));
    }
  } else {  // sct.py:115-135 apply_block_shift
    op = 3;
    int len, a;
    if (!draw((uint32_t)(k - 1), len)) return -1;
    ++len;
    const uint32_t m = (uint32_t)(k - len + 1);
    if (!draw(m, a)) return -1;
    do {
      if (!draw(m, v)) return -1;
    } while (v == a);
    put((uint32_t)a | ((uint32_t)v << 8) | ((uint32_t)len << 16));
  }
  if (out) *out = make_uint4((uint32_t)op | ((uint32_t)nev << 4), e0, e1, e2);
  return i;
}

// The same parse as a one-draw-per-step automaton, table-driven so that the lanes of a warp
// parse different proposals in lockstep without branching on their states: a proposal with a
// long rejection loop costs its lane more steps instead of serialising the warp.
// State s = 4 * phase + op: phase 0 = operator draw (select_operator), 1 = hop count, 2 = block
// length, 3 = first position of a pair, 4 = second position (redrawn while equal; for block
// swaps the whole pair is redrawn while |p - q| < len); op 1 = element swaps (0 5 (13 17)+),
// 2 = block swaps (0 6 (10 14 18)+), 3 = block shift (0 11 15 19).  C.ptab[s] = the draw's
// bound (0xffff: k - len + 1, the current block's position count) | the next state << 16.
__device__ __forceinline__ void chain_parse_table(uint32_t* t, int k, int h1, int h2) {
  for (int i = 0; i < 20; ++i) t[i] = 0u;
  t[5] = (uint32_t)h1 | (13u << 16);
  t[6] = (uint32_t)h2 | (10u << 16);
  t[10] = (uint32_t)(k / 2) | (14u << 16);
  t[11] = (uint32_t)(k - 1) | (15u << 16);
  t[13] = (uint32_t)k | (17u << 16);
  t[14] = 0xffffu | (18u << 16);
  t[15] = 0xffffu | (19u << 16);
  t[17] = (uint32_t)k | (13u << 16);
  t[18] = 0xffffu | (10u << 16);
  t[19] = 0xffffu;
  t[0] = 100u;
}

// Parse, in lockstep, the proposal that would start at every offset of the chunk (draw values
// C.hi, draw 0 = stream index base): C.jump[0][i] = its end offset (kChainOvf when it runs
// past the chunk) and C.desc[i] = the proposal.  Thread t starts with offset t; a lane that
// finishes takes the next offset from C.ticket (= the thread count at entry), so lanes with
// long proposals do not leave the rest of their warp idle.  Every lane runs every step
// (inactive lanes with their state frozen), so the warp stays converged: only the rare exact
// conversion and the stores are predicated branches.
//
// Proposal lengths are heavy-tailed (block swaps redraw whole pairs while |p - q| < len: ~2 %
// of k = 10 proposals read more than 64 draws, a few several hundred), and a warp runs until
// its slowest lane is done.  So the first pass gives each proposal kChainBudget draws and
// queues the offsets that need more; the second pass (PASS2) parses the queued offsets in
// full, from their start.
// One automaton step of the proposal at offset o (state s, hops, plen, pm, pa, events): reads
// draw cur; returns true when the proposal is complete or ran past the chunk (ovf).
struct ChainStep {
  int s = 0, hops = 1, plen = 1, pm = 2, pa = 0, nev = 0, op = 0;
  uint32_t e0 = 0u, e1 = 0u, e2 = 0u;
  __device__ __forceinline__ void reset() {
    s = 0;
    nev = 0;
  }
  __device__ __forceinline__ bool step(const ChainSmem& C, int& cur, bool& ovf, uint64_t base,
                                       uint64_t k0, uint64_t k1, int k, int p1, int p2) {
    ovf = cur >= kChainDraws;
    if (ovf) return true;
    const uint32_t te = C.ptab[s];
    const uint32_t bt = te & 0xffffu;
    const uint32_t bound = bt == 0xffffu ? (uint32_t)pm : bt;
    const uint64_t A = (uint64_t)C.hi[cur] * bound;
    int v = (int)(A >> 32);
    if ((uint32_t)A >= 0u - bound) v = chain_exact_below(k0, k1, base + (uint64_t)cur, bound);
    ++cur;
    const int ph = s >> 2;
    const bool same = v == pa;
    const bool pb = ph == 4 && !same;
    const bool rej = pb && s == 18 && abs(pa - v) < plen;
    const bool pair_done = pb && !rej;
    const uint32_t lo = (uint32_t)min(pa, v), hi = (uint32_t)max(pa, v);
    const uint32_t x = s == 18 ? lo | (hi << 8) | ((uint32_t)plen << 16)
                               : (uint32_t)pa | ((uint32_t)v << 8) | (s == 19 ? (uint32_t)plen << 16 : 0u);
    e0 = pair_done && nev == 0 ? x : e0;
    e1 = pair_done && nev == 1 ? x : e1;
    e2 = pair_done && nev == 2 ? x : e2;
    nev += pair_done ? 1 : 0;
    const int nop = v < p1 ? 1 : v < p2 ? 2 : 3;
    int ns = (int)(te >> 16);
    ns = s == 0 ? (nop == 3 ? 11 : 4 + nop) : ns;
    ns = ph == 4 && same ? s : ns;
    ns = rej ? 14 : ns;
    op = s & 3;
    hops = s == 0 ? 1 : ph == 1 ? 1 + v : hops - (pair_done ? 1 : 0);
    plen = ph == 2 ? 1 + v : plen;
    pm = ph == 2 ? k - v : pm;  // k - len + 1 positions
    pa = ph == 3 ? v : pa;
    s = ns;
    return pair_done && hops == 0;
  }
  __device__ __forceinline__ void record(ChainSmem& C, int o, int cur, bool ovf) const {
    C.jump[0][o] = ovf ? kChainOvf : (uint16_t)cur;
    if (!ovf) C.desc[o] = make_uint4((uint32_t)op | ((uint32_t)nev << 4), e0, e1, e2);
  }
};

template <bool PASS2>
__device__ __forceinline__ void chain_parse_lockstep(ChainSmem& C, uint64_t base, uint64_t k0,
                                                     uint64_t k1, int k, int p1, int p2) {
  if (PASS2) {
    // the few deferred offsets, one (or a few) per thread, each parsed to its end with no
    // warp-collective step: a lone long proposal runs at one shared load per draw
    const int nt = blockDim.x;
    for (int j = threadIdx.x; j < C.n_queued; j += nt) {
      const int o = C.queue[j];
      int cur = o;
      bool ovf = false;
      ChainStep ps;
      while (!ps.step(C, cur, ovf, base, k0, k1, k, p1, p2)) {
      }
      ps.record(C, o, cur, ovf);
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const int lim = kChainDraws;
  int j = threadIdx.x;
  int o = j;  // the offset being parsed
  int cur = o;
  ChainStep ps;
  for (;;) {
    const bool active = j < lim;
    if (!__any_sync(kFull, active)) break;
    bool done = false, ovf = false;
    // kChainSteps automaton steps per round of warp-collective bookkeeping
    if (active) {
      done = ps.step(C, cur, ovf, base, k0, k1, k, p1, p2);
#pragma unroll
      for (int r = 1; r < kChainSteps; ++r)
        if (!done && cur - o < kChainBudget) done = ps.step(C, cur, ovf, base, k0, k1, k, p1, p2);
    }
    const bool defer = active && !done && cur - o >= kChainBudget;  // to the second pass
    if (done) ps.record(C, o, cur, ovf);
    // warp-aggregated push of the deferred offsets
    const unsigned dm = __ballot_sync(kFull, defer);
    if (dm) {
      const int leader = __ffs(dm) - 1;
      int q0 = 0;
      if (lane == leader) q0 = atomicAdd(&C.n_queued, __popc(dm));
      q0 = __shfl_sync(kFull, q0, leader);
      if (defer) C.queue[q0 + __popc(dm & ((1u << lane) - 1u))] = (uint16_t)o;
    }
    const bool fin = done || defer;
    const unsigned fm = __ballot_sync(kFull, fin);
    if (fm) {  // warp-aggregated ticket
      const int leader = __ffs(fm) - 1;
      int t0 = 0;
      if (lane == leader) t0 = atomicAdd(&C.ticket, __popc(fm));
      t0 = __shfl_sync(kFull, t0, leader);
      if (fin) {
        j = t0 + __popc(fm & ((1u << lane) - 1u));
        o = j;
        cur = o;
        ps.reset();
      }
    }
  }
}

// The chain from entry offset e, by one warp: lane l composes the jump tables along the
// binary digits of l to find the node l proposals ahead, so 32 nodes cost five dependent
// shared loads.  Writes C.start[0 .. n), C.n (0: the first proposal overflows the chunk) and
// C.next = the offset after the last node.
__device__ __forceinline__ void chain_follow(ChainSmem& C, int e, int64_t need, int lane) {
  int x = e, n = 0, next = e;
  for (;;) {
    int y = x;
#pragma unroll
    for (int b = 0; b < kChainJumps; ++b)
      if ((lane >> b) & 1) y = y < kChainDraws ? (int)C.jump[b][y] : y;
    // node y is in the chain iff its proposal ends inside the chunk; nodes past the first
    // failure fail too, so the valid lanes are a prefix
    const bool ok = y < kChainDraws && C.jump[0][y] != kChainOvf;
    int cnt = __popc(__ballot_sync(kFull, ok));
    if ((int64_t)cnt > need - n) cnt = (int)(need - n);
    if (lane < cnt) C.start[n + lane] = (uint16_t)y;
    n += cnt;
    const int last = __shfl_sync(kFull, y, cnt > 0 ? cnt - 1 : 0);
    if (cnt > 0) next = C.jump[0][last];
    if (cnt < 32 || n >= need) break;
    x = next;
  }
  if (lane == 0) {
    C.n = n;
    C.next = next;
  }
}

// cand = the proposal `d` applied to the lane-distributed key (op_element_swaps /
// op_block_swaps / op_block_shift with the parsed positions)
__device__ __forceinline__ void chain_apply(Key& c, const uint4 d, int k, int lane) {
  const int op = (int)(d.x & 15u), ne = (int)(d.x >> 4);
  const bool wide = k > 32;
#pragma unroll 1
  for (int e = 0; e < ne; ++e) {
    const uint32_t ev = e == 0 ? d.y : e == 1 ? d.z : d.w;
    const int x = (int)(ev & 255u), y = (int)((ev >> 8) & 255u), len = (int)(ev >> 16);
    if (op == 1) {
      c.swap_pos(x, y, lane);
    } else if (op == 2) {  // x < y
      auto src = [&](int l) {
        if (l >= x && l < x + len) return l - x + y;
        if (l >= y && l < y + len) return l - y + x;
        return l;
      };
      c = c.gather(src(lane), src(lane + 32), wide);
    } else {
      const int lo = min(x, y), hi = max(x, y) + len, w = hi - lo;
      const int sh = y > x ? len : w - len;
      auto src = [&](int l) {
        if (l >= lo && l < hi) {
          int i = l - lo + sh;
          if (i >= w) i -= w;
          return lo + i;
        }
        return l;
      };
      c = c.gather(src(lane), src(lane + 32), wide);
    }
  }
}

// One chunk of the proposal chain, by the whole CTA (nt threads): the draws from stream
// index `entry` on, every offset's proposal (two lockstep passes), the jump tables and the
// chain of at most `need` proposals from the entry.  Ends with a barrier; then C.n proposals
// start at C.start[j] (descriptors C.desc[C.start[j]]) and the next chunk's entry is
// (entry & ~3) + C.next.
__device__ __forceinline__ void chain_parse_chunk(ChainSmem& C, uint64_t entry, int64_t need,
                                                  uint64_t k0, uint64_t k1, int k, int p1, int p2,
                                                  int h1, int h2, int nt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t base = entry & ~3ULL;
  const int e = (int)(entry - base);
#ifdef CCG_CHAIN_PROFILE  // per-phase cycle counts (make NVFLAGS="... -DCCG_CHAIN_PROFILE")
  long long c0 = clock64();
#define CHAIN_T(i) do { __syncthreads(); const long long c1 = clock64(); if (tid == 0) C.prof[i] += c1 - c0; c0 = c1; } while (0)
#else
#define CHAIN_T(i) __syncthreads()
#endif
  if (tid == 0) {
    C.ticket = nt;
    C.n_queued = 0;
    chain_parse_table(C.ptab, k, h1, h2);
  }
  for (int j = tid; j < kChainDraws / 4; j += nt) {
    uint64_t v0, v1, v2, v3;
    philox4x64_10(k0, k1, (base >> 2) + 1 + (uint64_t)j, v0, v1, v2, v3);
    *reinterpret_cast<uint4*>(C.hi + 4 * j) =
        make_uint4((uint32_t)(v0 >> 32), (uint32_t)(v1 >> 32), (uint32_t)(v2 >> 32), (uint32_t)(v3 >> 32));
  }
  CHAIN_T(0);
  chain_parse_lockstep<false>(C, base, k0, k1, k, p1, p2);
  CHAIN_T(1);
  if (tid == 0) C.ticket = nt;
  __syncthreads();
  chain_parse_lockstep<true>(C, base, k0, k1, k, p1, p2);
  CHAIN_T(2);
  // jump tables: 2^b proposals ahead (entries >= kChainDraws are terminal)
#pragma unroll 1
  for (int b = 1; b < kChainJumps; ++b) {
    for (int i = tid; i < kChainDraws; i += nt) {
      const int x = C.jump[b - 1][i];
      C.jump[b][i] = x < kChainDraws ? C.jump[b - 1][x] : (uint16_t)x;
    }
    __syncthreads();
  }
  CHAIN_T(3);
  if (warp == 0) {
    chain_follow(C, e, need, lane);
    if (lane == 0 && C.n == 0) {  // a proposal longer than the chunk: parse it from the stream
      C.start[0] = (uint16_t)e;
      C.next = chain_parse(nullptr, 0, e, base, k0, k1, k, p1, p2, h1, h2, &C.desc[e]);
      C.n = 1;
    }
  }
  CHAIN_T(4);
}

template <int SLOTS, int ORDER, int P>
__global__ void __launch_bounds__(P * 32, P >= 32 ? 1 : 32 / P)
    sct_climb_chain_kernel(const SctLaunch p, const __grid_constant__ SumPlan plan) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NT = P * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const WarpSmem ws(smem, warp, p.n);
  const double* logs = stage_logs<ORDER>(reinterpret_cast<double*>(smem), p.logs);
  ChainSmem& C = *reinterpret_cast<ChainSmem*>(smem + kLogsBytes + P * sct_warp_bytes(p.n));

  Evaluator<SLOTS, ORDER> ev;
  ev.init(plan, p.k, p.n, lane);
  const int kmax = p.k;
  const int64_t climbings = p.climbings;

  for (int64_t w = blockIdx.x; w < p.n_workers; w += gridDim.x) {
    const int32_t cid = p.cipher_of[w];
    const int k = p.key_lengths ? p.key_lengths[w] : kmax;
    if (p.key_lengths) ev.set_k(k, lane);
    stage_text(ws.txt, p.ciphers + p.offsets[cid], p.n, lane);
    const uint64_t k0 = p.keys[2 * w], k1 = p.keys[2 * w + 1];
    Draws d;
    d.key = p.keys + 2 * w;
    d.win = ws.win;
    d.start(p.skips ? p.skips[w] : 0, lane);
    Key key;
    key.v0 = lane;
    key.v1 = lane + 32;
    for (int i = k - 1; i > 0; --i) {  // rng.py:91-97
      const int j = d.below((uint32_t)(i + 1), lane);
      key.swap_pos(i, j, lane);
    }
    uint64_t entry = d.position();  // the first proposal's first draw
    double score = ev.score(key, ws.txt, ws.colstart, ws.plain, logs, lane);
    int64_t last = -1, t = 0;
    uint32_t rnd = 0;
    while (t < climbings) {
      // ---- parse the proposals of the next chunk of draws ----
      __syncthreads();  // the previous chunk's descriptors are consumed
      chain_parse_chunk(C, entry, climbings - t, k0, k1, k, p.p1, p.p2, p.op1_hop, p.op2_hop, NT);
      const int n = C.n;
      entry = (entry & ~3ULL) + (uint64_t)C.next;
      // ---- speculative rounds over the chain ----
      for (int tl = 0; tl < n;) {
        const int avail = n - tl < P ? n - tl : P;
        Key cand = key;
        double cs = 0.0;
        if (warp < avail) {
          chain_apply(cand, C.desc[C.start[tl + warp]], k, lane);
          cs = ev.score(cand, ws.txt, ws.colstart, ws.plain, logs, lane);
        }
        double* ex = C.score[rnd++ & 1u];
        if (lane == 0) ex[warp] = cs;
        __syncthreads();
        // the first improvement (sct.py:168): lane j tests proposal t+j, one ballot
        const unsigned better = __ballot_sync(kFull, lane < avail && ex[lane] > score);
        const int acc = better ? __ffs(better) - 1 : -1;
        const int used = acc >= 0 ? acc : avail - 1;
        if (acc >= 0) {  // block-uniform: every warp read the same scores
          if (warp == acc) {
            if (lane < k) C.key[lane] = (uint8_t)cand.v0;
            if (lane + 32 < k) C.key[lane + 32] = (uint8_t)cand.v1;
          }
          const double next_score = ex[acc];
          __syncthreads();
          key.v0 = lane < k ? C.key[lane] : lane;
          key.v1 = lane + 32 < k ? C.key[lane + 32] : lane + 32;
          score = next_score;
          last = t + acc;
        }
        tl += used + 1;
        t += used + 1;
      }
    }
    if (warp == 0) {
      if (lane < k) p.keys_out[w * kmax + lane] = (uint8_t)key.v0;
      if (lane + 32 < k) p.keys_out[w * kmax + lane + 32] = (uint8_t)key.v1;
      if (lane == 0) {
        p.scores[w] = score;
        if (p.draws_used) p.draws_used[w] = entry;
        if (p.last_accept) p.last_accept[w] = last;
        if (p.tries_done) p.tries_done[w] = t;
      }
    }
    __syncthreads();
  }
}

// ---- Latency mode on a pair of SMs (sct_climb_pair_kernel) ----
// A restart is 64 workers, so in latency mode most of the GPU's 148 SMs idle.  Here each
// worker gets a cluster of two CTAs: CTA 1 parses the worker's proposal chain chunk by chunk
// (chain_parse_chunk, as above) and copies each chunk's descriptors into CTA 0's shared
// memory (distributed shared memory); CTA 0 runs the speculative scoring rounds.  Double
// buffering lets CTA 1 parse chunk c+1 while CTA 0 scores chunk c; one cluster barrier per
// chunk hands the buffers over.
struct PairBuf {  // in the scoring CTA
  uint4 desc[2][kChainMaxProps];
  int n[2];
  double score[2][32];
  uint8_t key[kSctMaxKey];
};
constexpr int kPairWarps = 32;

__host__ __device__ inline size_t pair_buf_offset(int n) {
  return kLogsBytes + kPairWarps * sct_warp_bytes(n);
}
__host__ __device__ inline size_t pair_smem_bytes(int n) {
  const size_t scorer = pair_buf_offset(n) + sizeof(PairBuf);
  return scorer > sizeof(ChainSmem) ? scorer : sizeof(ChainSmem);
}

template <int SLOTS, int ORDER>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairWarps * 32, 1)
    sct_climb_pair_kernel(const SctLaunch p, const __grid_constant__ SumPlan plan) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int P = kPairWarps, NT = kPairWarps * 32;
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kmax = p.k;
  const int64_t climbings = p.climbings;
  const int64_t n_pairs = gridDim.x / 2;
  PairBuf* buf_view = reinterpret_cast<PairBuf*>(smem + pair_buf_offset(p.n));
  cluster.sync();  // both CTAs are running before either touches the other's shared memory

  if (rank == 1) {
    // ---- the parsing CTA ----
    ChainSmem& C = *reinterpret_cast<ChainSmem*>(smem);
    PairBuf* remote = cluster.map_shared_rank(buf_view, 0);
#ifdef CCG_CHAIN_PROFILE
    if (tid < 5) C.prof[tid] = 0;
#endif
    for (int64_t w = blockIdx.x / 2; w < p.n_workers; w += n_pairs) {
      const int k = p.key_lengths ? p.key_lengths[w] : kmax;
      const uint64_t k0 = p.keys[2 * w], k1 = p.keys[2 * w + 1];
      // the first proposal follows permutation(k)'s k - 1 draws (rng.py:91-97)
      uint64_t entry = (p.skips ? p.skips[w] : 0) + (uint64_t)(k - 1);
      int64_t produced = 0;
      int b = 0;
      while (produced < climbings) {
        chain_parse_chunk(C, entry, climbings - produced, k0, k1, k, p.p1, p.p2, p.op1_hop,
                          p.op2_hop, NT);
        const int n = C.n;
        for (int j = tid; j < n; j += NT) remote->desc[b][j] = C.desc[C.start[j]];
        if (tid == 0) remote->n[b] = n;
        entry = (entry & ~3ULL) + (uint64_t)C.next;
        produced += n;
        cluster.sync();  // chunk ready; the scorers are done with the buffer written next
        b ^= 1;
      }
      if (tid == 0 && p.draws_used) p.draws_used[w] = entry;
#ifdef CCG_CHAIN_PROFILE
      if (tid == 0 && w < 2) {
        printf("parse profile w=%lld: gen %lld pass1 %lld pass2 %lld jumps %lld follow %lld\n", (long long)w,
               C.prof[0], C.prof[1], C.prof[2], C.prof[3], C.prof[4]);
        for (int i = 0; i < 5; ++i) C.prof[i] = 0;
      }
#endif
      cluster.sync();  // end of the worker
    }
    return;
  }

  // ---- the scoring CTA ----
  const WarpSmem ws(smem, warp, p.n);
  const double* logs = stage_logs<ORDER>(reinterpret_cast<double*>(smem), p.logs);
  PairBuf& B = *buf_view;
  Evaluator<SLOTS, ORDER> ev;
  ev.init(plan, p.k, p.n, lane);
  for (int64_t w = blockIdx.x / 2; w < p.n_workers; w += n_pairs) {
    const int32_t cid = p.cipher_of[w];
    const int k = p.key_lengths ? p.key_lengths[w] : kmax;
    if (p.key_lengths) ev.set_k(k, lane);
    stage_text(ws.txt, p.ciphers + p.offsets[cid], p.n, lane);
    Draws d;
    d.key = p.keys + 2 * w;
    d.win = ws.win;
    d.start(p.skips ? p.skips[w] : 0, lane);
    Key key;
    key.v0 = lane;
    key.v1 = lane + 32;
    for (int i = k - 1; i > 0; --i) {  // rng.py:91-97
      const int j = d.below((uint32_t)(i + 1), lane);
      key.swap_pos(i, j, lane);
    }
    double score = ev.score(key, ws.txt, ws.colstart, ws.plain, logs, lane);
    int64_t last = -1, t = 0;
    uint32_t rnd = 0;
    int b = 0;
    while (t < climbings) {
      cluster.sync();  // the parser's chunk is in buffer b
      const int n = B.n[b];
      for (int tl = 0; tl < n;) {
        const int avail = n - tl < P ? n - tl : P;
        Key cand = key;
        double cs = 0.0;
        if (warp < avail) {
          chain_apply(cand, B.desc[b][tl + warp], k, lane);
          cs = ev.score(cand, ws.txt, ws.colstart, ws.plain, logs, lane);
        }
        double* ex = B.score[rnd++ & 1u];
        if (lane == 0) ex[warp] = cs;
        __syncthreads();
        // the first improvement (sct.py:168): lane j tests proposal t+j, one ballot
        const unsigned better = __ballot_sync(kFull, lane < avail && ex[lane] > score);
        const int acc = better ? __ffs(better) - 1 : -1;
        const int used = acc >= 0 ? acc : avail - 1;
        if (acc >= 0) {  // block-uniform: every warp read the same scores
          if (warp == acc) {
            if (lane < k) B.key[lane] = (uint8_t)cand.v0;
            if (lane + 32 < k) B.key[lane + 32] = (uint8_t)cand.v1;
          }
          const double next_score = ex[acc];
          __syncthreads();
          key.v0 = lane < k ? B.key[lane] : lane;
          key.v1 = lane + 32 < k ? B.key[lane + 32] : lane + 32;
          score = next_score;
          last = t + acc;
        }
        tl += used + 1;
        t += used + 1;
      }
      b ^= 1;
    }
    if (warp == 0) {
      if (lane < k) p.keys_out[w * kmax + lane] = (uint8_t)key.v0;
      if (lane + 32 < k) p.keys_out[w * kmax + lane + 32] = (uint8_t)key.v1;
      if (lane == 0) {
        p.scores[w] = score;
        if (p.last_accept) p.last_accept[w] = last;
        if (p.tries_done) p.tries_done[w] = t;
      }
    }
    cluster.sync();  // end of the worker
  }
}

// Score given (cipher, key) pairs with the same evaluator (sct.py:158-160).
template <int SLOTS, int ORDER>
__global__ void __launch_bounds__(kSctWarps * 32)
    sct_score_kernel(const uint8_t* __restrict__ ciphers, const int64_t* __restrict__ offsets,
                     const int32_t* __restrict__ cipher_of, const uint8_t* __restrict__ keys,
                     int32_t k, int64_t n_keys, const double* __restrict__ glogs,
                     double* __restrict__ out, int32_t n, const __grid_constant__ SumPlan plan) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const WarpSmem ws(smem, warp, n);
  const double* logs = stage_logs<ORDER>(reinterpret_cast<double*>(smem), glogs);
  const int64_t w = (int64_t)blockIdx.x * kSctWarps + warp;
  if (w >= n_keys) return;
  Evaluator<SLOTS, ORDER> ev;
  ev.init(plan, k, n, lane);
  stage_text(ws.txt, ciphers + offsets[cipher_of[w]], n, lane);
  Key key;
  key.v0 = lane < k ? keys[w * k + lane] : lane;
  key.v1 = lane + 32 < k ? keys[w * k + lane + 32] : lane + 32;
  const double s = ev.score(key, ws.txt, ws.colstart, ws.plain, logs, lane);
  if (lane == 0) out[w] = s;
}

// Any-length scoring: one thread per (cipher, key), numpy's pairwise recursion done by a
// recursive device function over on-the-fly decryption.  Used by the fitness API for texts
// beyond the warp evaluator's plan budget (the climb kernels never take this path).
struct LongText {
  const uint8_t* txt;
  const double* logs;
  const int32_t* colstart;
  int k;
  int order;
  __device__ __forceinline__ int at(int64_t t) const {
    const int64_t r = t / k;
    return txt[colstart[t - r * k] + r];
  }
  __device__ __forceinline__ double term(int64_t t) const {
    int64_t idx = 0;
    for (int j = 0; j < order; ++j) idx = idx * kAlpha + at(t + j);
    return logs[idx];
  }
};

__device__ double pairwise_leaf(const LongText& L, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += L.term(lo + i);
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = L.term(lo + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += L.term(lo + i + j);
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += L.term(lo + i);
  return res;
}

// numpy's recursion (split at n/2 rounded down to a multiple of 8) with an explicit stack.
__device__ double pairwise_iter(const LongText& L, int64_t n_terms) {
  struct Frame { int64_t lo, n; double left; int state; };
  Frame st[48];  // depth <= log2(n / 64) + 1
  int sp = 0;
  st[0] = {0, n_terms, 0.0, 0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    const int64_t half = (f.n / 2) - (f.n / 2) % 8;
    if (f.state == 0) {
      if (f.n <= 128) {
        ret = pairwise_leaf(L, f.lo, f.n);
        --sp;
      } else {
        f.state = 1;
        st[sp + 1] = {f.lo, half, 0.0, 0};
        ++sp;
      }
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.lo + half, f.n - half, 0.0, 0};
      ++sp;
    } else {
      ret = f.left + ret;
      --sp;
    }
  }
  return ret;
}

__global__ void sct_score_long_kernel(const uint8_t* __restrict__ ciphers,
                                      const int64_t* __restrict__ offsets,
                                      const int32_t* __restrict__ cipher_of,
                                      const uint8_t* __restrict__ keys, int32_t k, int64_t n_keys,
                                      int order, const double* __restrict__ logs,
                                      double* __restrict__ out) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_keys) return;
  const int32_t c = cipher_of[w];
  const int64_t n = offsets[c + 1] - offsets[c];
  int32_t colstart[kSctMaxKey];
  const int64_t base = n / k, rem = n - base * k;
  int64_t acc = 0;
  for (int j = 0; j < k; ++j) {
    const int col = keys[w * k + j];
    colstart[col] = (int32_t)acc;
    acc += base + (col < rem ? 1 : 0);
  }
  LongText L{ciphers + offsets[c], logs, colstart, k, order};
  out[w] = n < order ? 0.0 : pairwise_iter(L, n - order + 1);
}

size_t sct_smem_bytes(int n) { return kLogsBytes + kSctWarps * sct_warp_bytes(n); }

template <typename K>
cudaError_t prep_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

int slots_for(const SumPlan& plan) {
  const int s = (plan.n_leaves + 3) / 4;
  return s <= 1 ? 1 : s <= 2 ? 2 : s <= 4 ? 4 : 8;
}

template <int SLOTS, int ORDER>
cudaError_t climb_slots(cudaStream_t s, const SctLaunch& p, const SumPlan& plan, int sm_count) {
  // keys of at most 32 positions (every worker: p.k is the batch maximum) skip the second
  // key register in every operator and in the segment scan
  auto kern = p.k > 32 ? sct_climb_kernel<SLOTS, ORDER, true> : sct_climb_kernel<SLOTS, ORDER, false>;
  const size_t bytes = sct_smem_bytes(p.n);
  cudaError_t e = prep_smem(kern, bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSctWarps * 32, bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (p.n_workers + kSctWarps - 1) / kSctWarps;
  const int64_t resident = (int64_t)per_sm * sm_count;
  const int grid = (int)(need < resident ? need : resident);
  kern<<<grid, kSctWarps * 32, bytes, s>>>(p, plan);
  return cudaGetLastError();
}

template <int SLOTS, int ORDER, int P>
cudaError_t spec_launch(cudaStream_t s, const SctLaunch& p, const SumPlan& plan, int sm_count,
                        bool* launched) {
  *launched = false;
  auto kern = sct_climb_spec_kernel<SLOTS, ORDER, P>;
  const size_t bytes = kLogsBytes + P * sct_warp_bytes(p.n) + 2 * sizeof(SpecExchange);
  cudaError_t e = prep_smem(kern, bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P * 32, bytes);
  if (e != cudaSuccess) return e;
  if ((int64_t)per_sm * sm_count < p.n_workers) return cudaSuccess;  // more than one wave
  kern<<<(unsigned)p.n_workers, P * 32, bytes, s>>>(p, plan);
  *launched = true;
  return cudaGetLastError();
}

// Latency mode: the deepest speculation (16, 8, 4 or 2 warps per worker) whose CTAs all fit
// on the GPU at once -- one restart of the #08 shape (64 workers) takes 21 ms with 16 warps,
// 23 ms with 8, 28 ms with 4, 61 ms with one warp per worker.  *launched = false: none fits,
// use the one-warp kernel.
template <int SLOTS, int ORDER>
cudaError_t climb_spec_slots(cudaStream_t s, const SctLaunch& p, const SumPlan& plan, int sm_count,
                             bool* launched) {
  cudaError_t e = spec_launch<SLOTS, ORDER, 16>(s, p, plan, sm_count, launched);
  if (e != cudaSuccess || *launched) return e;
  e = spec_launch<SLOTS, ORDER, 8>(s, p, plan, sm_count, launched);
  if (e != cudaSuccess || *launched) return e;
  e = spec_launch<SLOTS, ORDER, 4>(s, p, plan, sm_count, launched);
  if (e != cudaSuccess || *launched) return e;
  return spec_launch<SLOTS, ORDER, 2>(s, p, plan, sm_count, launched);
}

template <int SLOTS, int ORDER, int P>
cudaError_t chain_launch(cudaStream_t s, const SctLaunch& p, const SumPlan& plan, int sm_count,
                         bool* launched) {
  *launched = false;
  auto kern = sct_climb_chain_kernel<SLOTS, ORDER, P>;
  const size_t bytes = kLogsBytes + P * sct_warp_bytes(p.n) + sizeof(ChainSmem);
  if (bytes > kMaxSmemPerBlock) return cudaSuccess;  // long texts: fewer warps per worker
  cudaError_t e = prep_smem(kern, bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, P * 32, bytes);
  if (e != cudaSuccess) return e;
  if ((int64_t)per_sm * sm_count < p.n_workers) return cudaSuccess;  // more than one wave
  kern<<<(unsigned)p.n_workers, P * 32, bytes, s>>>(p, plan);
  *launched = true;
  return cudaGetLastError();
}

template <int SLOTS, int ORDER>
cudaError_t pair_launch(cudaStream_t s, const SctLaunch& p, const SumPlan& plan, int sm_count,
                        bool* launched) {
  *launched = false;
  auto kern = sct_climb_pair_kernel<SLOTS, ORDER>;
  const size_t bytes = pair_smem_bytes(p.n);
  if (bytes > kMaxSmemPerBlock || 2 * p.n_workers > sm_count) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * p.n_workers));
  cfg.blockDim = dim3(kPairWarps * 32);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  int clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg);
  if (e != cudaSuccess) return e;
  if (clusters < p.n_workers) return cudaSuccess;  // not all workers at once
  kern<<<cfg.gridDim, cfg.blockDim, bytes, s>>>(p, plan);
  *launched = true;
  return cudaGetLastError();
}

// Chain-parsed latency mode: the deepest speculation (32, 16, 8 or 4 warps per worker) whose
// CTAs all fit at once.  *launched = false: none fits.
template <int SLOTS, int ORDER>
cudaError_t climb_chain_slots(cudaStream_t s, const SctLaunch& p, const SumPlan& plan, int sm_count,
                              bool* launched) {
  cudaError_t e = chain_launch<SLOTS, ORDER, 32>(s, p, plan, sm_count, launched);
  if (e != cudaSuccess || *launched) return e;
  e = chain_launch<SLOTS, ORDER, 16>(s, p, plan, sm_count, launched);
  if (e != cudaSuccess || *launched) return e;
  e = chain_launch<SLOTS, ORDER, 8>(s, p, plan, sm_count, launched);
  if (e != cudaSuccess || *launched) return e;
  return chain_launch<SLOTS, ORDER, 4>(s, p, plan, sm_count, launched);
}

template <int SLOTS, int ORDER>
cudaError_t score_slots(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                        const int32_t* cipher_of, const uint8_t* keys, int32_t k, int64_t n_keys,
                        const double* logs, double* out, int32_t n, const SumPlan& plan) {
  auto kern = sct_score_kernel<SLOTS, ORDER>;
  const size_t bytes = sct_smem_bytes(n);
  cudaError_t e = prep_smem(kern, bytes);
  if (e != cudaSuccess) return e;
  const int grid = (int)((n_keys + kSctWarps - 1) / kSctWarps);
  kern<<<grid, kSctWarps * 32, bytes, s>>>(ciphers, offsets, cipher_of, keys, k, n_keys, logs,
                                           out, n, plan);
  return cudaGetLastError();
}

}  // namespace

// numpy pairwise_sum recursion -> leaves + post-order merges.
static int plan_rec(SumPlan* P, int start, int n) {
  if (n <= 128) {
    const int id = P->n_leaves++;
    P->leaf_start[id] = start;
    P->leaf_len[id] = n;
    return id;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  const int L = plan_rec(P, start, n2);
  const int R = plan_rec(P, start + n2, n - n2);
  P->merge_dst[P->n_merges] = (int8_t)L;
  P->merge_src[P->n_merges] = (int8_t)R;
  ++P->n_merges;
  return L;
}

void build_sum_plan(int64_t n_terms, SumPlan* plan) {
  *plan = SumPlan{};
  plan->n_terms = (int32_t)n_terms;
  plan->seq = n_terms < 8;
  plan_rec(plan, 0, (int)n_terms);
}

cudaError_t launch_sct_score_long(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                                  const int32_t* cipher_of, const uint8_t* keys, int32_t k,
                                  int64_t n_keys, int order, const double* logs, double* out) {
  if (n_keys <= 0) return cudaSuccess;
  const int grid = (int)((n_keys + 127) / 128);
  sct_score_long_kernel<<<grid, 128, 0, s>>>(ciphers, offsets, cipher_of, keys, k, n_keys, order,
                                              logs, out);
  return cudaGetLastError();
}

template <int ORDER>
static cudaError_t climb_order(cudaStream_t s, const SctLaunch& p, const SumPlan& plan,
                               int sm_count) {
  // latency mode: few enough workers that each can get a CTA of speculating warps
  if (p.n_workers <= 16 * (int64_t)sm_count && !(p.flags & CCG_FLAG_SCT_NO_SPEC)) {
    bool launched = false;
    cudaError_t e = cudaSuccess;
    // the chain-parsed kernel's descriptors hold up to kSctLaneMaxHops events per proposal
    if (!(p.flags & CCG_FLAG_SCT_SPEC_REPLAY) && p.op1_hop <= kSctLaneMaxHops &&
        p.op2_hop <= kSctLaneMaxHops) {
      switch (slots_for(plan)) {  // two SMs per worker when the GPU has them
        case 1: e = pair_launch<1, ORDER>(s, p, plan, sm_count, &launched); break;
        case 2: e = pair_launch<2, ORDER>(s, p, plan, sm_count, &launched); break;
        case 4: e = pair_launch<4, ORDER>(s, p, plan, sm_count, &launched); break;
        default: e = pair_launch<8, ORDER>(s, p, plan, sm_count, &launched); break;
      }
      if (e != cudaSuccess || launched) return e;
      switch (slots_for(plan)) {
        case 1: e = climb_chain_slots<1, ORDER>(s, p, plan, sm_count, &launched); break;
        case 2: e = climb_chain_slots<2, ORDER>(s, p, plan, sm_count, &launched); break;
        case 4: e = climb_chain_slots<4, ORDER>(s, p, plan, sm_count, &launched); break;
        default: e = climb_chain_slots<8, ORDER>(s, p, plan, sm_count, &launched); break;
      }
      if (e != cudaSuccess || launched) return e;
    }
    switch (slots_for(plan)) {
      case 1: e = climb_spec_slots<1, ORDER>(s, p, plan, sm_count, &launched); break;
      case 2: e = climb_spec_slots<2, ORDER>(s, p, plan, sm_count, &launched); break;
      case 4: e = climb_spec_slots<4, ORDER>(s, p, plan, sm_count, &launched); break;
      default: e = climb_spec_slots<8, ORDER>(s, p, plan, sm_count, &launched); break;
    }
    if (e != cudaSuccess || launched) return e;
  }
  switch (slots_for(plan)) {
    case 1: return climb_slots<1, ORDER>(s, p, plan, sm_count);
    case 2: return climb_slots<2, ORDER>(s, p, plan, sm_count);
    case 4: return climb_slots<4, ORDER>(s, p, plan, sm_count);
    default: return climb_slots<8, ORDER>(s, p, plan, sm_count);
  }
}

cudaError_t launch_sct_climb(cudaStream_t s, const SctLaunch& p, const SumPlan& plan,
                             int sm_count) {
  if (p.n_workers <= 0) return cudaSuccess;
  switch (p.order) {
    case 2: return climb_order<2>(s, p, plan, sm_count);
    case 3: return climb_order<3>(s, p, plan, sm_count);
    case 4: return climb_order<4>(s, p, plan, sm_count);
    default: return cudaErrorInvalidValue;
  }
}

template <int ORDER>
static cudaError_t score_order(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                               const int32_t* cipher_of, const uint8_t* keys, int32_t k,
                               int64_t n_keys, const double* logs, double* out, int32_t n_common,
                               const SumPlan& plan) {
  switch (slots_for(plan)) {
    case 1: return score_slots<1, ORDER>(s, ciphers, offsets, cipher_of, keys, k, n_keys, logs, out, n_common, plan);
    case 2: return score_slots<2, ORDER>(s, ciphers, offsets, cipher_of, keys, k, n_keys, logs, out, n_common, plan);
    case 4: return score_slots<4, ORDER>(s, ciphers, offsets, cipher_of, keys, k, n_keys, logs, out, n_common, plan);
    default: return score_slots<8, ORDER>(s, ciphers, offsets, cipher_of, keys, k, n_keys, logs, out, n_common, plan);
  }
}

cudaError_t launch_sct_score(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                             const int32_t* cipher_of, const uint8_t* keys, int32_t k,
                             int64_t n_keys, int order, const double* logs, double* out,
                             int32_t n_common, const SumPlan& plan) {
  if (n_keys <= 0) return cudaSuccess;
  switch (order) {
    case 2: return score_order<2>(s, ciphers, offsets, cipher_of, keys, k, n_keys, logs, out, n_common, plan);
    case 3: return score_order<3>(s, ciphers, offsets, cipher_of, keys, k, n_keys, logs, out, n_common, plan);
    case 4: return score_order<4>(s, ciphers, offsets, cipher_of, keys, k, n_keys, logs, out, n_common, plan);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ccg
