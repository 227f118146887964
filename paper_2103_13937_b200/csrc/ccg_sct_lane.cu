// ccg_sct_lane.cu -- SCT climb with one worker per LANE (sm_100a).
//
// Reference path: sct.py:148-170 sct_worker (start key permutation(k), rng.py:91-97; per try
// select_operator sct.py:69-79 and apply_element_swaps / apply_block_swaps /
// apply_block_shift sct.py:82-135; candidate_score sct.py:158-160 over the irregular-grid
// decryption ciphers.py:71-86; accept iff strictly greater, sct.py:168).
//
// Two scoring modes share the climb:
//  * PARITY (MODE 0): the reference's float64 score, numpy's pairwise summation order
//    (ngrams.py:172 `logs[idx].sum()`), bit-exact -- the default path of ccg_sct_climb.
//  * FAST (MODE 1, opt-in, ccg_sct_fast_climb): an int32-quantised log table (exactly
//    associative), so a candidate is scored INCREMENTALLY: only the n-gram windows that touch
//    a column whose content moved are re-read (north_star: "incremental (delta) ... scoring,
//    which re-scores only the positions touched by a swap").  Its own oracle is
//    oracle/cc_oracle.c cco_sct_fast_worker (full rescore of the same integer fitness).
//
// Why a lane per worker.  The warp-per-worker kernel (ccg_sct.cu) spends ~950 warp
// instructions per try, most of it scalar work every lane repeats (draws, operators, the
// segment scan, the pairwise plan replay).  Here each lane runs its own worker, so that work
// is done once per worker, and the score is a plain sequential loop per lane: the decryption
// walk plain[t] = cipher[colstart[t % k] + t / k] (ciphers.py:79-86 via the exclusive prefix
// sum of the segment lengths in key order) feeding numpy's pairwise recursion term by term
// (leaves of <= 128 terms with 8 strided accumulators, merged in post-order), or the
// windows of the moved columns.  The 32 workers of a warp share one ciphertext (workers of a
// chunk with other ciphertexts run in further passes), staged once in shared memory.
//
// Proposals (sct.py:69-135) never read the key, so each lane parses its stream ahead, one
// draw per step in every lane, into a small queue of position events (swap / block swap /
// shift); a round = a fixed number of parse steps, then one evaluation per lane.  Long
// rejection loops (apply_block_swaps) cost the lane that has them extra steps instead of
// stalling the warp.
//
// Shared memory per warp, lane-interleaved so a lane's own arrays sit in its own banks:
//   draw ring  u32[ring][32 lanes]: top 32 bits of each Philox word (rng.py:68-75), topped
//              up warp-collectively once per round, so the lanes' Philox blocks are
//              generated together instead of diverging at every draw
//   queue      parsed proposals: a header word + up to kSctLaneMaxHops events each
//   key, cand  u8[KMAX][32];  colstart u16[KMAX + 8][32] (+8: next-row copies);  window sums i32[KMAX][32] (FAST)
//   plan       the numpy pairwise recursion of this pass's text length (PARITY)
//   text       the pass's ciphertext
// The log table is staged per block: bigram directly (676 f64 / i32); trigram as a byte index
// into its distinct values when it has at most 256 (exact, 17.6 KB -- the host finds them),
// else directly when it fits, else through L1/L2; quadgram tables are read through L2.
#include <type_traits>

#include "ccg_internal.h"
#include "ccg_rng.cuh"
#include "ccg_smem.cuh"

namespace ccg {
namespace {

constexpr unsigned kFull = 0xffffffffu;
// draws buffered per lane (power of two) and proposal-parser steps per lane per round
// (< ring - 3).  The fast mode trades ring depth for a third block per SM (its registers
// fit 80); the parity mode's pairwise stack needs more registers and keeps two blocks.
#ifndef CCG_LANE_RING0
#define CCG_LANE_RING0 32
#endif
#ifndef CCG_LANE_PARSE0
#define CCG_LANE_PARSE0 16
#endif
#ifndef CCG_LANE_MINB0
#define CCG_LANE_MINB0 1
#endif
#ifndef CCG_LANE_ILP
#define CCG_LANE_ILP 8
#endif
constexpr int ring_of(int mode) { return mode == 1 ? 16 : CCG_LANE_RING0; }
constexpr int parse_steps_of(int mode) { return mode == 1 ? 12 : CCG_LANE_PARSE0; }
// parsed-proposal queue per lane: kQSlots proposals of a header word + up to kSctLaneMaxHops
// position events (one per swap / block swap; a shift is one event)
constexpr int kQSlots = 2;
constexpr int kQWords = 1 + kSctLaneMaxHops;
constexpr int kQueueBytes = kQSlots * kQWords * 4 * 32;

constexpr int pow26(int o) { return o == 2 ? 676 : o == 3 ? 17576 : 456976; }

__host__ __device__ constexpr size_t round16(size_t b) { return (b + 15) & ~(size_t)15; }

// colstart has kCsExt extra entries per lane: cs[m] = cs[m mod k] + m div k for
// k <= m < k + kCsExt (the columns of the following rows), so the letter of any of the next
// kCsExt positions -- in this row or past its end -- is txt[cs[c + j] + r] with no
// per-position row select (ParityTerms::letters)
constexpr int kCsExt = 8;
constexpr int cs_ext_of(int mode) { return mode == 0 ? kCsExt : 0; }  // (parity mode only)
// the extended entries of column c (segment start s): cs[c + q k] = s + q, q >= 1
__device__ __forceinline__ void set_cs_ext(uint16_t* csp, int k, int c, int s) {
  for (int m = c + k, q = 1; m < k + kCsExt; m += k, ++q) csp[32 * m] = (uint16_t)(s + q);
}

template <int MODE, int KMAX>
__host__ __device__ constexpr size_t lane_fixed_bytes() {
  return (size_t)ring_of(MODE) * 128 + kQueueBytes + 2 * KMAX * 32 + (KMAX + cs_ext_of(MODE)) * 64 +
         (MODE == 1 ? KMAX * 128 : 256);
}
template <int MODE, int ORDER, bool TSMEM, bool CIDX>
__host__ __device__ constexpr size_t lane_tab_bytes() {
  using Tab = typename std::conditional<MODE == 0, double, int32_t>::type;
  return CIDX ? round16(256 * sizeof(Tab)) + round16((size_t)pow26(ORDER))
              : TSMEM ? round16((size_t)pow26(ORDER) * sizeof(Tab)) : 0;
}

template <int MODE, int KMAX>
__host__ __device__ size_t lane_warp_bytes(int max_len) {
  return lane_fixed_bytes<MODE, KMAX>() + round16((size_t)max_len + 16);
}

// The exact int(u*bound) when the 32-bit fast path cannot decide (probability < 2^-21):
// regenerate the Philox block of draw `pos` and convert the full 53-bit mantissa.
__device__ __noinline__ int lane_exact_below(uint64_t k0, uint64_t k1, uint64_t pos, uint32_t bound) {
  uint64_t v[4];
  philox4x64_10(k0, k1, (pos >> 2) + 1, v[0], v[1], v[2], v[3]);
  return (int)int_below_small(v[pos & 3], bound);
}

// Philox4x64-10 block `prod/4` of stream (k0, k1) (numpy increments the counter before each
// block, rng.py:68-75), top 32 bits of its four words into the ring slots at a, a+128, ...
__device__ __noinline__ void lane_gen_block(uint64_t k0, uint64_t k1, uint64_t prod, uint32_t a) {
  uint64_t v0, v1, v2, v3;
  philox4x64_10(k0, k1, (prod >> 2) + 1, v0, v1, v2, v3);
  sm::st32(a, (uint32_t)(v0 >> 32));
  sm::st32(a + 128u, (uint32_t)(v1 >> 32));
  sm::st32(a + 256u, (uint32_t)(v2 >> 32));
  sm::st32(a + 384u, (uint32_t)(v3 >> 32));
}

// One lane's draw stream: WorkerRng(seed, stream) (rng.py:58-79), ring-buffered in shared memory.
template <int kRing>
struct LaneRing {
  uint64_t k0, k1;
  uint64_t cons;  // stream index of the next draw
  uint64_t prod;  // stream index one past the last generated draw (multiple of 4)
  uint32_t slot0; // shared address of this lane's slot 0; slot s at +128*s

  // the Philox block is generated out of line by value (a member call would force the ring
  // state into local memory)
  __device__ __forceinline__ void gen() {
    lane_gen_block(k0, k1, prod, slot0 + 128u * (uint32_t)(prod & (kRing - 1)));
    prod += 4;
  }
  __device__ void start(uint64_t pos) {
    prod = pos & ~3ULL;
    cons = pos;
    gen();
  }
  // warp-collective: every active lane refills to more than kRing - 4 buffered draws
  __device__ __forceinline__ void top_up(bool active) {
    for (;;) {
      const bool need = active && prod - cons <= (uint64_t)(kRing - 4);
      if (!__any_sync(kFull, need)) break;
      if (need) gen();
    }
  }
  // rng.py:77-79 int(u * bound), 1 <= bound < 2^11: A = (x >> 32) * bound gives it exactly
  // unless A's low word is within `bound` of wrapping (ccg_rng.cuh int_below_tiny)
  __device__ __forceinline__ int below(uint32_t bound) {
    // Used for the start key's Fisher-Yates draws (up to 63, more than the ring holds): a
    // lane whose ring ran dry refills together with every lane of its branch that has room,
    // so one Philox pass serves all of them.
    if (__any_sync(__activemask(), prod == cons) && prod - cons <= (uint64_t)(kRing - 4)) gen();
    const uint32_t hi = sm::ld32(slot0 + 128u * (uint32_t)(cons & (kRing - 1)));
    const uint64_t A = (uint64_t)hi * bound;
    ++cons;
    if ((uint32_t)A < 0u - bound) return (int)(A >> 32);
    return lane_exact_below(k0, k1, cons - 1, bound);
  }
  // the same when the caller guarantees a buffered draw (after top_up)
  __device__ __forceinline__ int below_buffered(uint32_t bound) {
    const uint32_t hi = sm::ld32(slot0 + 128u * (uint32_t)(cons & (kRing - 1)));
    const uint64_t A = (uint64_t)hi * bound;
    ++cons;
    if ((uint32_t)A < 0u - bound) return (int)(A >> 32);
    return lane_exact_below(k0, k1, cons - 1, bound);
  }
};

// numpy pairwise_sum recursion of n_terms terms as a post-order op list: op >= 0 is a leaf of
// that many terms (leaves are consecutive, so no start is needed), op = -1 merges the top two
// partial sums (left + right).
__device__ int build_plan(uint32_t plan, int n_terms) {
  if (n_terms <= 0) return 0;
  int len[16], state[16];
  int sp = 1, nops = 0;
  len[0] = n_terms;
  state[0] = 0;
  while (sp > 0) {
    const int L = len[sp - 1];
    if (L <= 128) {
      sm::st32(plan + 4u * nops++, (uint32_t)L);
      --sp;
      continue;
    }
    const int n2 = L / 2 - (L / 2) % 8;
    if (state[sp - 1] == 0) {
      state[sp - 1] = 1;
      len[sp] = n2;
      state[sp] = 0;
      ++sp;
    } else if (state[sp - 1] == 1) {
      state[sp - 1] = 2;
      len[sp] = L - n2;
      state[sp] = 0;
      ++sp;
    } else {
      sm::st32(plan + 4u * nops++, 0xffffffffu);
      --sp;
    }
  }
  return nops;
}

// A log table in shared or global memory: direct entries, or (CIDX) a byte index per entry
// into at most 256 distinct values -- an n-gram log table built from counts has few distinct
// entries (65 for the corpus trigram table), so the exact float64 / int32 values of a
// 17,576-entry trigram table fit in 17.6 KB of shared memory instead of 140 / 70 KB.
template <typename V, bool CIDX>
struct TabRef {
  const V* v;
  const uint8_t* ix;
  __device__ __forceinline__ V operator[](int i) const { return CIDX ? v[ix[i]] : v[i]; }
};

// The decryption walk of one lane: the letters of plain[0], plain[1], ... in order
// (plain[t] = cipher[colstart[t % k] + t / k]).  Plain shared-memory pointers (no volatile
// asm) so the compiler can issue the loads of eight consecutive positions back to back:
// a position's letter needs two dependent loads (its column's start, then the letter) and
// the term a third (the table), so the throughput of one lane depends on that overlap.
struct Walk {
  const uint8_t* txt;
  const uint16_t* cs;  // this lane's colstart: column c at cs[32 * c]
  int k, c, r;
  __device__ __forceinline__ void pos(int& cc, int& rr) {
    cc = c;
    rr = r;
    if (++c == k) {
      c = 0;
      ++r;
    }
  }
  __device__ __forceinline__ int at(int cc, int rr) const { return txt[cs[32 * cc] + rr]; }
};

template <int ORDER, typename Tab>
struct ParityTerms {
  Walk wk;
  int h[3];  // the previous ORDER-1 letters, oldest first
  Tab tab;
  __device__ __forceinline__ void prime() {
#pragma unroll
    for (int i = 0; i < ORDER - 1; ++i) {
      int cc, rr;
      wk.pos(cc, rr);
      h[i] = wk.at(cc, rr);
    }
  }
  // the letters of the next G positions, loaded before any is used.  For G >= 4, positions
  // past the row's end read the extended colstart (cs[m] = cs[m mod k] + m div k, m < k + 8),
  // so every letter is txt[cs[c + j] + r] -- one base pointer with immediate offsets, no
  // per-position select, for any key length.
  template <int G>
  __device__ __forceinline__ void letters(int (&L)[ORDER - 1 + G]) {
    static_assert(G <= kCsExt, "the extended colstart covers one row wrap of G positions");
    if (G >= 4) {
      const int k = wk.k, c = wk.c, r = wk.r;
      const uint16_t* cb = wk.cs + 32 * c;
      const uint8_t* tr = wk.txt + r;
#pragma unroll
      for (int j = 0; j < G; ++j) L[ORDER - 1 + j] = tr[cb[32 * j]];
      int nc = c + G, nr = r;
      while (nc >= k) {  // once for k >= G
        nc -= k;
        ++nr;
      }
      wk.c = nc;
      wk.r = nr;
      return;
    }
    int cc[G], rr[G];
#pragma unroll
    for (int j = 0; j < G; ++j) wk.pos(cc[j], rr[j]);
#pragma unroll
    for (int j = 0; j < G; ++j) L[ORDER - 1 + j] = wk.at(cc[j], rr[j]);
  }
  // the next G window terms (G = 1 or 8)
  template <int G>
  __device__ __forceinline__ void terms(double (&v)[G]) {
    int L[ORDER - 1 + G];
    letters<G>(L);
#pragma unroll
    for (int i = 0; i < ORDER - 1; ++i) L[i] = h[i];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      int idx = L[j];
#pragma unroll
      for (int i = 1; i < ORDER; ++i) idx = idx * kAlpha + L[j + i];
      v[j] = tab[idx];
    }
#pragma unroll
    for (int i = 0; i < ORDER - 1; ++i) h[i] = L[G + i];
  }
  __device__ __forceinline__ double term() {
    double v[1];
    terms<1>(v);
    return v[0];
  }
};

// sct.py:158-160 candidate_score: numpy's pairwise float64 sum of the window log-probabilities
// in plaintext order, bit for bit (the oracle's cco_pairwise_sum).
template <int ORDER, typename Tab>
__device__ double parity_score(ParityTerms<ORDER, Tab>& T, const int32_t* plan, int nops) {
  if (nops == 0) return 0.0;
  T.wk.c = 0;
  T.wk.r = 0;
  T.prime();
  double stk[8];
  int sp = 0;
  for (int i = 0; i < nops; ++i) {
    const int op = plan[i];
    if (op < 0) {
      const double b = stk[--sp];
      const double a = stk[--sp];
      stk[sp++] = a + b;
      continue;
    }
    double res;
    if (op < 8) {
      res = 0.0;
      for (int j = 0; j < op; ++j) res += T.term();
    } else {
      double r[8];
      const int blocks = op / 8;
      if (CCG_LANE_ILP == 8) {
        double v[8];
        T.template terms<8>(r);
        for (int b = 1; b < blocks; ++b) {
          T.template terms<8>(v);
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] += v[j];
        }
      } else {  // four terms in flight (fewer live registers)
        double v[4];
        T.template terms<4>(v);
        r[0] = v[0]; r[1] = v[1]; r[2] = v[2]; r[3] = v[3];
        T.template terms<4>(v);
        r[4] = v[0]; r[5] = v[1]; r[6] = v[2]; r[7] = v[3];
        for (int b = 1; b < blocks; ++b) {
          T.template terms<4>(v);
#pragma unroll
          for (int j = 0; j < 4; ++j) r[j] += v[j];
          T.template terms<4>(v);
#pragma unroll
          for (int j = 0; j < 4; ++j) r[4 + j] += v[j];
        }
      }
      res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (int j = 8 * blocks; j < op; ++j) res += T.term();
    }
    stk[sp++] = res;
  }
  return stk[0];
}

// FAST mode: integer sum of the windows whose first letter lies in grid column w
// (positions t = w + r*k, t <= n - ORDER), read column-wise from the ciphertext.
template <int ORDER, typename Tab>
__device__ __forceinline__ int32_t window_sum(int w, int k, int rows, const uint8_t* txt,
                                              const uint16_t* cs, Tab tab) {
  const uint8_t* b[ORDER];
#pragma unroll
  for (int i = 0; i < ORDER; ++i) {
    int cc = w + i, dr = 0;
    while (cc >= k) {
      cc -= k;
      ++dr;
    }
    b[i] = txt + cs[32 * cc] + dr;
  }
  auto one = [&](int rr) {
    int idx = b[0][rr];
#pragma unroll
    for (int i = 1; i < ORDER; ++i) idx = idx * kAlpha + b[i][rr];
    return tab[idx];
  };
  int32_t acc = 0;
  int r = 0;
  for (; r + 8 <= rows; r += 8) {
    int32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = one(r + j);
    acc += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
  }
  for (; r < rows; ++r) acc += one(r);
  return acc;
}

template <int MODE, int ORDER, int KMAX, bool TSMEM, bool CIDX>
__global__ void __launch_bounds__(kSctLaneWarps * 32, MODE == 1 ? 3 : CCG_LANE_MINB0)
    sct_lane_kernel(const SctLaneLaunch p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  using Tab = typename std::conditional<MODE == 0, double, int32_t>::type;
  constexpr int T = pow26(ORDER);
  const Tab* gtab = MODE == 0 ? (const Tab*)p.logs : (const Tab*)p.qtable;
  const size_t tab_bytes = lane_tab_bytes<MODE, ORDER, TSMEM, CIDX>();
  TabRef<Tab, CIDX> tab{gtab, nullptr};
  if (CIDX) {  // distinct values, then the byte index
    Tab* sv = reinterpret_cast<Tab*>(smem);
    uint8_t* si = smem + round16(256 * sizeof(Tab));
    for (int i = threadIdx.x; i < p.n_cvals; i += blockDim.x) sv[i] = reinterpret_cast<const Tab*>(p.cvals)[i];
    for (int i = threadIdx.x; i < T; i += blockDim.x) si[i] = p.cidx[i];
    __syncthreads();
    tab.v = sv;
    tab.ix = si;
  } else if (TSMEM) {
    Tab* st = reinterpret_cast<Tab*>(smem);
    for (int i = threadIdx.x; i < T; i += blockDim.x) st[i] = gtab[i];
    __syncthreads();
    tab.v = st;
  }
  unsigned char* wb = smem + tab_bytes + (size_t)warp * lane_warp_bytes<MODE, KMAX>(p.max_len);
  const uint32_t ring = sm::addr(wb);
  constexpr int kRing = ring_of(MODE), kParseSteps = parse_steps_of(MODE);
  uint32_t* qp = reinterpret_cast<uint32_t*>(wb + kRing * 128) + lane;  // [32 (4 slot + word)]
  unsigned char* kb = wb + kRing * 128 + kQueueBytes;
  uint8_t* keyp = kb + lane;                                  // key[q] at keyp[32 q]
  uint8_t* candp = keyp + 32 * KMAX;                          // cand[q] at candp[32 q]
  uint16_t* csp = reinterpret_cast<uint16_t*>(kb + 64 * KMAX) + lane;  // colstart[c] at [32 c]
  unsigned char* aux = kb + 128 * KMAX + 64 * cs_ext_of(MODE);
  int32_t* gp = reinterpret_cast<int32_t*>(aux) + lane;       // FAST: G[w] at gp[32 w]
  int32_t* plan = reinterpret_cast<int32_t*>(aux);            // PARITY
  uint8_t* txt = aux + (MODE == 1 ? 128 * KMAX : 256);

  const int64_t n_chunks = (p.n_workers + 31) / 32;
  const WorkerTickets tk{p.tickets, (int64_t)gridDim.x * kSctLaneWarps};
  for (int64_t ch = (int64_t)blockIdx.x * kSctLaneWarps + warp; ch < n_chunks; ch = tk.next(ch, lane)) {
    const int64_t w = ch * 32 + lane;
    const bool valid = w < p.n_workers;
    const int32_t cid = valid ? p.cipher_of[w] : -1;
    unsigned todo = __ballot_sync(kFull, valid);
    while (todo) {  // one pass per ciphertext among the chunk's workers
      const int leader = __ffs(todo) - 1;
      const int32_t pc = __shfl_sync(kFull, cid, leader);
      const bool mine = ((todo >> lane) & 1u) && cid == pc;
      todo &= ~__ballot_sync(kFull, mine);
      const int64_t toff = p.offsets[pc];
      const int n = (int)(p.offsets[pc + 1] - toff);
      __syncwarp();
      for (int i = lane; i < n; i += 32) txt[i] = p.ciphers[toff + i];
      int nops = 0;
      if (MODE == 0 && lane == 0) nops = build_plan(sm::addr(plan), n >= ORDER ? n - ORDER + 1 : 0);
      nops = __shfl_sync(kFull, nops, 0);
      __syncwarp();

      const int k = mine ? (p.key_lengths ? p.key_lengths[w] : p.kmax) : 2;
      const int base = n / k, rem = n - base * k;
      auto seglen = [&](int c) { return c < rem ? base + 1 : base; };
      LaneRing<kRing> d;
      d.slot0 = ring + 4u * (uint32_t)lane;
      d.k0 = d.k1 = 0;
      d.cons = d.prod = 0;
      if (mine) {
        d.k0 = p.keys[2 * w];
        d.k1 = p.keys[2 * w + 1];
        d.start(p.skips ? p.skips[w] : 0);
      }
      // FAST: window rows = rows_q + (w <= rows_s), from n - ORDER = rows_q * k + rows_s
      const int no = n - ORDER;
      const int rows_q = no >= 0 ? no / k : 0, rows_s = no >= 0 ? no - rows_q * k : -1;
      auto rows_of = [&](int ww) { return no < 0 ? 0 : rows_q + (ww <= rows_s ? 1 : 0); };
      ParityTerms<ORDER, TabRef<Tab, CIDX>> pt;
      pt.wk.txt = txt;
      pt.wk.cs = csp;
      pt.wk.k = k;
      pt.tab = tab;
      // regular grid with a tabulated window sum (fast mode): segment c starts at rank(c) * L,
      // so a window's sum is a function of its columns' ranks (sct_ftab_kernel)
      const int32_t* F = nullptr;
      uint32_t rank_mul = 0;
      if (MODE == 1 && p.ftab && mine) {
        const int64_t fo = p.f_off[w];
        if (fo >= 0) {
          F = p.ftab + fo;
          rank_mul = (uint32_t)((0x100000000ULL + (uint64_t)base - 1) / (uint64_t)base);  // ceil(2^32 / L)
        }
      }
      int kpow = 1;
#pragma unroll
      for (int i = 0; i < ORDER; ++i) kpow *= k;
      auto wsum = [&](int ww) -> int32_t {
        if (MODE == 1 && F) {
          const int kind = ww > k - ORDER ? ww - (k - ORDER) : 0;
          int e = 0;
#pragma unroll
          for (int i = 0; i < ORDER; ++i) {
            int cc = ww + i;
            if (cc >= k) cc -= k;
            e = e * k + (int)__umulhi((uint32_t)csp[32 * cc], rank_mul);
          }
          return __ldg(F + (int64_t)kind * kpow + e);
        }
        return window_sum<ORDER>(ww, k, rows_of(ww), txt, csp, tab);
      };
      int64_t lookups = 0;

      double fscore = 0.0;
      int32_t iscore = 0;
      if (mine) {
        // rng.py:91-97 permutation(k): Fisher-Yates from the top
        for (int q = 0; q < k; ++q) keyp[32 * q] = (uint8_t)q;
        for (int i = k - 1; i > 0; --i) {
          const int j = d.below((uint32_t)(i + 1));
          const uint8_t a = keyp[32 * i], b = keyp[32 * j];
          keyp[32 * i] = b;
          keyp[32 * j] = a;
        }
        int s = 0;
        for (int q = 0; q < k; ++q) {
          const int c = keyp[32 * q];
          candp[32 * q] = (uint8_t)c;
          csp[32 * c] = (uint16_t)s;
          if (MODE == 0) set_cs_ext(csp, k, c, s);
          s += seglen(c);
        }
        if (MODE == 0) {
          fscore = parity_score(pt, plan, nops);
        } else {
          for (int ww = 0; ww < k; ++ww) {
            const int32_t g = wsum(ww);
            gp[32 * ww] = g;
            iscore += g;
          }
        }
      }
      const uint64_t kmask = k >= 64 ? ~0ULL : ((1ULL << k) - 1);
      // ---- the proposal stream (sct.py:69-135) as a one-draw-per-step automaton ----
      // Proposals never read the key: the operator choice and every operator's
      // draws depend on the stream and k only, so they are parsed ahead into a small queue of
      // position events, and a step consumes exactly one draw in every lane.  Rejection loops
      // (apply_block_swaps redraws whole pairs while |p - q| < len, sct.py:100-104) then cost
      // one step per draw in the lane that needs them instead of stalling the warp.
      // State stt = 4 * phase + op, as in ccg_sct.cu ChainStep: phase 0 = operator draw
      // (select_operator), 1 = hop count, 2 = block length, 3 = first position of a pair, 4 =
      // second position (redrawn while equal; block swaps redraw the whole pair while
      // |p - q| < len); op 1 = element swaps, 2 = block swaps, 3 = block shift.  Written with
      // selects: the lanes of a warp are in different states, and a switch would serialise
      // them.  A proposal's events collect in registers and go to the queue when it completes.
      int stt = 0, hops = 1, pa = 0, plen = 1, pm = 2, nev = 0;
      uint32_t e0 = 0u, e1 = 0u, e2 = 0u;
      int q_head = 0, q_cnt = 0;
      int64_t parsed = 0, done_t = 0, last = -1;
      auto qword = [&](int slot, int word) -> uint32_t& { return qp[32 * (kQWords * slot + word)]; };
      const uint32_t kh = (uint32_t)(k / 2), km1 = (uint32_t)(k - 1);
      const uint32_t h1 = (uint32_t)p.op1_hop, h2 = (uint32_t)p.op2_hop;
      auto step = [&]() {
        const int ph = stt >> 2, op = stt & 3;
        uint32_t bound = op == 1 ? (uint32_t)k : (uint32_t)pm;  // pairs / positions within k - len + 1
        bound = ph == 2 ? (op == 2 ? kh : km1) : bound;
        bound = ph == 1 ? (op == 1 ? h1 : h2) : bound;
        bound = ph == 0 ? 100u : bound;
        const int v = d.below_buffered(bound);
        const bool same = v == pa;
        const bool pb = ph == 4 && !same;
        const bool rej = pb && op == 2 && abs(pa - v) < plen;
        const bool pair_done = pb && !rej;
        const uint32_t lo = (uint32_t)min(pa, v), hi = (uint32_t)max(pa, v);
        const uint32_t x = op == 2 ? lo | (hi << 8) | ((uint32_t)plen << 16)
                                   : (uint32_t)pa | ((uint32_t)v << 8) | (op == 3 ? (uint32_t)plen << 16 : 0u);
        e0 = pair_done && nev == 0 ? x : e0;
        e1 = pair_done && nev == 1 ? x : e1;
        e2 = pair_done && nev == 2 ? x : e2;
        nev += pair_done ? 1 : 0;
        const int nop = v < p.p1 ? 1 : v < p.p2 ? 2 : 3;
        int ns = same ? stt : rej ? 14 : (op == 1 ? 13 : 10);  // phase 4
        ns = ph == 3 ? 16 + op : ns;
        ns = ph == 2 ? 12 + op : ns;
        ns = ph == 1 ? (op == 1 ? 13 : 10) : ns;
        ns = ph == 0 ? (nop == 3 ? 11 : 4 + nop) : ns;
        hops = ph == 0 ? 1 : ph == 1 ? 1 + v : hops - (pair_done ? 1 : 0);
        plen = ph == 2 ? 1 + v : plen;
        pm = ph == 2 ? k - v : pm;
        pa = ph == 3 ? v : pa;
        stt = ns;
        if (pair_done && hops == 0) {  // the proposal is complete: queue it
          const int slot = (q_head + q_cnt) % kQSlots;
          qword(slot, 0) = (uint32_t)op | ((uint32_t)nev << 4);
          qword(slot, 1) = e0;
          qword(slot, 2) = e1;
          qword(slot, 3) = e2;
          ++q_cnt;
          ++parsed;
          stt = 0;
          nev = 0;
        }
      };

      const int64_t climbings = p.climbings;
      while (__any_sync(kFull, mine && done_t < climbings)) {
        // parse: up to kParseSteps draws per lane (the ring holds more than that after top_up)
        d.top_up(mine && parsed < climbings);
        for (int s = 0; s < kParseSteps; ++s)
          if (mine && parsed < climbings && q_cnt < kQSlots) step();
        if (!(mine && done_t < climbings && q_cnt > 0)) continue;
        // evaluate the oldest parsed proposal: apply its events to cand
        const uint32_t hdr = qword(q_head, 0);
        const int op = (int)(hdr & 15u), ne = (int)(hdr >> 4);
        int lo = k, hi = 0;
        for (int e = 0; e < ne; ++e) {
          const uint32_t ev = qword(q_head, 1 + e);
          const int x = (int)(ev & 255u), y = (int)((ev >> 8) & 255u), len = (int)(ev >> 16);
          if (op == 1) {  // element swap
            const uint8_t a = candp[32 * x], b = candp[32 * y];
            candp[32 * x] = b;
            candp[32 * y] = a;
            lo = min(lo, min(x, y));
            hi = max(hi, max(x, y) + 1);
          } else if (op == 2) {  // block swap, x < y
            for (int q = 0; q < len; ++q) {
              const uint8_t a = candp[32 * (x + q)], b = candp[32 * (y + q)];
              candp[32 * (x + q)] = b;
              candp[32 * (y + q)] = a;
            }
            lo = min(lo, x);
            hi = max(hi, y + len);
          } else {  // block shift of len positions from x to y
            lo = min(x, y);
            hi = max(x, y) + len;
            const int wn = hi - lo;
            const int sh = y > x ? len : wn - len;
            for (int i = 0; i < wn; ++i) {
              int q = i + sh;
              if (q >= wn) q -= wn;
              candp[32 * (lo + i)] = keyp[32 * (lo + q)];
            }
          }
        }
        q_head = (q_head + 1) % kQSlots;
        --q_cnt;
        const int64_t t = done_t++;
        // colstart of the candidate: only key positions in [lo, hi) move (the candidate
        // permutes that range, so the segment offsets outside it are unchanged)
        const int s0 = csp[32 * keyp[32 * lo]];
        uint64_t dirty = 0;
        {
          int s = s0;
          for (int q = lo; q < hi; ++q) {
            const int c = candp[32 * q];
            if (MODE == 1 && csp[32 * c] != s) dirty |= 1ULL << c;
            csp[32 * c] = (uint16_t)s;
            if (MODE == 0) set_cs_ext(csp, k, c, s);
            s += seglen(c);
          }
        }
        bool accept;
        double fcand = 0.0;
        int32_t delta = 0;
        uint64_t wd = 0;
        if (MODE == 0) {
          fcand = parity_score(pt, plan, nops);
          accept = fcand > fscore;  // sct.py:168
        } else {
          // windows touching a moved column: w = c - i (mod k), i < ORDER
          wd = dirty;
#pragma unroll
          for (int i = 1; i < ORDER; ++i) {
            int sft = i;
            while (sft >= k) sft -= k;
            if (sft) wd |= ((dirty >> sft) | (dirty << (k - sft))) & kmask;
          }
          uint64_t m = wd;
          while (m) {
            const int ww = __ffsll((long long)m) - 1;
            m &= m - 1;
            lookups += F ? 1 : rows_of(ww);
            delta += wsum(ww) - gp[32 * ww];
          }
          accept = delta > 0;  // sct.py:168, on the quantised fitness
        }
        if (accept) {
          for (int q = lo; q < hi; ++q) keyp[32 * q] = candp[32 * q];
          last = t;
          if (MODE == 0) {
            fscore = fcand;
          } else {
            iscore += delta;
            uint64_t m = wd;
            while (m) {
              const int ww = __ffsll((long long)m) - 1;
              m &= m - 1;
              gp[32 * ww] = wsum(ww);
            }
          }
        } else {
          int s = s0;
          for (int q = lo; q < hi; ++q) {
            const int c = keyp[32 * q];
            candp[32 * q] = (uint8_t)c;
            csp[32 * c] = (uint16_t)s;
            if (MODE == 0) set_cs_ext(csp, k, c, s);
            s += seglen(c);
          }
        }
      }
      if (mine) {
        for (int q = 0; q < k; ++q) p.keys_out[w * p.kmax + q] = keyp[32 * q];
        if (MODE == 0)
          p.scores[w] = fscore;
        else
          p.iscores[w] = iscore;
        if (p.draws_used) p.draws_used[w] = d.cons;
        if (p.last_accept) p.last_accept[w] = last;
        if (p.tries_done) p.tries_done[w] = done_t;
        if (MODE == 1 && p.lookups) p.lookups[w] = lookups;
      }
      __syncwarp();
    }
  }
}

// Fast mode on a regular grid (n = L * k): segment j of the ciphertext is cipher[jL, jL + L)
// and plaintext column c reads segment rank(c), so the integer sum of the windows starting in
// column w is F[kind][rank(w)][rank(w+1)]...[rank(w+ORDER-1)] with kind = the number of the
// window's letters that wrap to the next row (w > k - ORDER) and L (kind 0) or L - 1 rows.
// One CTA per (ciphertext, k): the text in shared memory, one table entry per thread.  A
// candidate then costs one table read per changed window instead of a column walk.
__global__ void __launch_bounds__(256) sct_ftab_kernel(const uint8_t* __restrict__ ciphers,
                                                        const int64_t* __restrict__ offsets,
                                                        const SctFPair* __restrict__ pairs,
                                                        const int32_t* __restrict__ qt, int order,
                                                        int32_t* __restrict__ F) {
  extern __shared__ uint8_t ftxt[];
  const SctFPair P = pairs[blockIdx.x];
  const int64_t off = offsets[P.cipher];
  const int n = (int)(offsets[P.cipher + 1] - off), k = P.k, L = n / k;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ftxt[i] = ciphers[off + i];
  __syncthreads();
  int kpow = 1;
  for (int i = 0; i < order; ++i) kpow *= k;
  for (int e = threadIdx.x; e < order * kpow; e += blockDim.x) {
    const int kind = e / kpow;
    int rem = e - kind * kpow;
    int start[4];
    for (int i = order - 1; i >= 0; --i) {
      const int r = rem % k;
      rem /= k;
      start[i] = r * L + (i >= order - kind ? 1 : 0);  // wrapped letters read the next row
    }
    const int rows = kind == 0 ? L : L - 1;
    int32_t acc = 0;
    for (int r = 0; r < rows; ++r) {
      int idx = 0;
      for (int i = 0; i < order; ++i) idx = idx * kAlpha + ftxt[start[i] + r];
      acc += __ldg(qt + idx);
    }
    F[P.off + e] = acc;
  }
}

template <typename K>
cudaError_t lane_smem_attr(K kern, size_t bytes) {
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

template <int MODE, int ORDER, int KMAX, bool TSMEM, bool CIDX = false>
cudaError_t lane_launch(cudaStream_t s, const SctLaneLaunch& p, int sm_count) {
  auto kern = sct_lane_kernel<MODE, ORDER, KMAX, TSMEM, CIDX>;
  const size_t bytes =
      lane_tab_bytes<MODE, ORDER, TSMEM, CIDX>() + kSctLaneWarps * lane_warp_bytes<MODE, KMAX>(p.max_len);
  cudaError_t e = lane_smem_attr(kern, bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSctLaneWarps * 32, bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int64_t chunks = (p.n_workers + 31) / 32;
  const int64_t need = (chunks + kSctLaneWarps - 1) / kSctLaneWarps;
  const int64_t resident = (int64_t)per_sm * sm_count;
  const int grid = (int)(need < resident ? need : resident);
  kern<<<grid, kSctLaneWarps * 32, bytes, s>>>(p);
  return cudaGetLastError();
}

// Where the table lives: bigram in shared memory; trigram as a byte index + distinct values
// in shared memory when the host found at most 256 distinct entries (p.cidx), else in shared
// memory when it fits beside the warps' arrays, else read through L1/L2; quadgram via L2.
template <int MODE, int ORDER, int KMAX>
cudaError_t lane_table(cudaStream_t s, const SctLaneLaunch& p, int sm_count) {
  if (ORDER == 4) return lane_launch<MODE, 4, KMAX, false>(s, p, sm_count);
  if (ORDER == 3 && p.cidx && !(p.flags & CCG_FLAG_SCT_TABLE_L2))
    return lane_launch<MODE, 3, KMAX, true, true>(s, p, sm_count);
  const size_t bytes =
      lane_tab_bytes<MODE, ORDER, true, false>() + kSctLaneWarps * lane_warp_bytes<MODE, KMAX>(p.max_len);
  if (ORDER == 2 || (bytes <= 200 * 1024 && !(p.flags & CCG_FLAG_SCT_TABLE_L2)))
    return lane_launch<MODE, ORDER, KMAX, true>(s, p, sm_count);
  return lane_launch<MODE, ORDER, KMAX, false>(s, p, sm_count);
}

template <int MODE, int ORDER>
cudaError_t lane_kmax(cudaStream_t s, const SctLaneLaunch& p, int sm_count) {
  if (p.kmax <= 32) return lane_table<MODE, ORDER, 32>(s, p, sm_count);
  return lane_table<MODE, ORDER, 64>(s, p, sm_count);
}

template <int MODE>
cudaError_t lane_order(cudaStream_t s, const SctLaneLaunch& p, int sm_count) {
  switch (p.order) {
    case 2: return lane_kmax<MODE, 2>(s, p, sm_count);
    case 3: return lane_kmax<MODE, 3>(s, p, sm_count);
    case 4: return lane_kmax<MODE, 4>(s, p, sm_count);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

size_t sct_lane_smem_bytes(int mode, int kmax, int64_t max_len) {
  if (mode == 0)
    return kmax <= 32 ? kSctLaneWarps * lane_warp_bytes<0, 32>((int)max_len)
                      : kSctLaneWarps * lane_warp_bytes<0, 64>((int)max_len);
  return kmax <= 32 ? kSctLaneWarps * lane_warp_bytes<1, 32>((int)max_len)
                    : kSctLaneWarps * lane_warp_bytes<1, 64>((int)max_len);
}

cudaError_t launch_sct_lane(cudaStream_t s, const SctLaneLaunch& p, int sm_count) {
  if (p.n_workers <= 0) return cudaSuccess;
  return p.mode == 0 ? lane_order<0>(s, p, sm_count) : lane_order<1>(s, p, sm_count);
}

cudaError_t launch_sct_ftab(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                            const SctFPair* pairs, int64_t n_pairs, const int32_t* qtable,
                            int order, int max_len, int32_t* ftab) {
  if (n_pairs <= 0) return cudaSuccess;
  sct_ftab_kernel<<<(unsigned)n_pairs, 256, (size_t)max_len, s>>>(ciphers, offsets, pairs, qtable,
                                                                    order, ftab);
  return cudaGetLastError();
}

}  // namespace ccg
