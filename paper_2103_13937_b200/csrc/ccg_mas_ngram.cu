// ccg_mas_ngram.cu -- the MAS stochastic climb with an order-G n-gram table (G = 2, 3, 4):
// stochastic_worker (mas.py:218-244) generalised from bigrams to windows of G letters
// (BASELINE.json configs 4-5; the reference itself has bigrams only).
//
// Fitness = sum over the n-G+1 windows of table[sum_j 26^(G-1-j) t_{s+j}] (integer, uint16
// entries).  The proposal stream, the accept rule (exact score change > 0) and the result
// are those of stochastic_worker; the oracle is oracle/cc_oracle.c cco_ngram_worker, which
// reduces to the reference at G = 2 (tests/test_oracle_golden.py).
//
// Position-based delta.  A 26x26 count-matrix delta (mas.py:181-210) does not extend to
// G > 2, so the warp keeps the current PLAINTEXT in shared memory together with the
// per-ciphertext occurrence lists (positions grouped by cipher letter).  Interchanging
// plaintext letters a, b touches exactly the positions of cipher letters xa = pi^-1(a) and
// xb = pi^-1(b); each such position i re-scores the windows that contain it and whose
// FIRST touched position is i (so a window holding several touched positions is counted
// once).  Cost per evaluation ~ (occurrences of a and b) x G x 2 lookups instead of O(n).
//
// Delta cache.  A rejected proposal leaves the state unchanged, so every computed delta is
// kept (per letter pair, tagged with an epoch that each accept advances): after the last
// accept of a climb -- typically within its first ~20 % of tries -- almost every proposal
// is a cache hit.
//
// Warp rounds.  A round pairs up to 32 proposals, one per lane, exactly as the D-form
// kernel does (rng.py:81-89), and reads their cached deltas: the cache-hit prefix before the
// first miss decides it (first positive delta accepted, else all rejected).  On a miss the
// first four misses of the round are walked at once, one per 8-lane group, into the cache,
// and the round is re-run -- proposals never read the state (rng.py:81-89), so computing
// deltas ahead of the sequential order is exact; after an accept they are simply stale.
// The window bytes around a position come from three 32-bit shared loads and two funnel
// shifts; the a/b tests and the swapped copy are SWAR byte operations on those words.  The
// table score of every window of the current plaintext is kept in shared memory (refreshed
// around the touched positions on accept), so a walk looks up only the new windows.
//
// Tables: G <= 3 are staged in shared memory (1.3 KB / 34 KB of uint16); the quadgram
// table (914 KB uint16) is read through L1/L2 with __ldg.
#include "ccg_mas_common.cuh"

namespace ccg {
namespace {



__host__ __device__ constexpr int pow26(int g) { return g == 0 ? 1 : 26 * pow26(g - 1); }

// per-warp shared layout (bytes)
__host__ __device__ inline uint32_t ng_text_stride(int max_len) {
  return ((uint32_t)max_len + 12u + 15u) & ~15u;  // plaintext at +4, >= 8 bytes of slack after
}
constexpr uint32_t kCacheBytes = 676u * 4u + 676u * 2u + 8u;  // delta cache + epoch tags
__host__ __device__ inline uint32_t ng_u16_bytes(int max_len) {
  return (2u * (uint32_t)max_len + 15u) & ~15u;
}
constexpr uint32_t kRoundKeyBytes = 22u * 8u;  // Philox round keys (philox_round_keys)
// plaintext | occurrence lists | start | cursor | delta cache + tags | window scores | round keys
__host__ __device__ inline uint32_t ng_warp_bytes(int max_len) {
  return ng_text_stride(max_len) + ng_u16_bytes(max_len) + 32u * 2u + 32u * 4u + kCacheBytes +
         ng_u16_bytes(max_len) + kRoundKeyBytes;
}

// per-byte equality mask (0x80 in each byte of x equal to the byte in rep), exact for bytes < 0x80
__device__ __forceinline__ uint32_t eq_bytes(uint32_t x, uint32_t rep) {
  const uint32_t d = x ^ rep;
  const uint32_t t = (d & 0x7f7f7f7fu) + 0x7f7f7f7fu;
  return ~(t | d) & 0x80808080u;
}
__device__ __forceinline__ uint32_t expand_mask(uint32_t m80) { return (m80 >> 7) * 0xffu; }

template <int G, bool SMEM_TAB>
struct NgState {
  const uint16_t* tab;   // global table (G = 4)
  uint32_t tab_s;        // shared address of the staged table (G <= 3)
  uint32_t text_base;    // shared address of the plaintext buffer (plain[i] at +4+i)
  const uint16_t* occ;   // occurrence lists (shared)
  const uint16_t* start; // start[x] .. start[x+1] (shared)
  uint32_t ws_base;      // shared address of the window scores
  int n;

  __device__ __forceinline__ int lookup(int idx) const {
    if (SMEM_TAB) return lds_u16(tab_s + 2u * (uint32_t)idx);
    return (int)__ldg(tab + idx);
  }

  // Score change contributed by position i for the interchange a<->b (a, b plaintext
  // letters, i holds a or b): windows containing i whose first touched position is i.
  __device__ __forceinline__ int position_delta(int i, uint32_t arep, uint32_t brep) const {
    // bytes plain[i-(G-1)] .. plain[i+(G-1)] as lo (bytes 0..3) and hi (bytes 4..7),
    // starting at buffer offset 4 + i - 3 = i + 1 (G = 4; smaller G use a subset)
    const uint32_t off = (uint32_t)(i + 1);
    const uint32_t wa = text_base + (off & ~3u);
    const uint32_t w0 = lds_u32(wa), w1 = lds_u32(wa + 4), w2 = lds_u32(wa + 8);
    const uint32_t sh = (off & 3u) * 8u;
    const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
    // byte j of (lo,hi) is plain[i - 3 + j]; the centre is byte 3.  Bytes equal to a or b
    // are exchanged by XOR with a^b.
    const uint32_t m_lo = eq_bytes(lo, arep) | eq_bytes(lo, brep);
    const uint32_t m_hi = eq_bytes(hi, arep) | eq_bytes(hi, brep);
    const uint32_t abx = arep ^ brep;
    const uint32_t nlo = lo ^ (expand_mask(m_lo) & abx), nhi = hi ^ (expand_mask(m_hi) & abx);
    const uint32_t touched_lo = m_lo >> 7;  // bit 8j set for touched byte j
    int delta = 0;
    // window k covers bytes 3-(G-1)+k .. 3+k (k = 0..G-1), start s = i-(G-1)+k; it is
    // counted here when no byte before the centre in it is touched (positions s .. i-1)
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const int s = i - (G - 1) + k;
      const int first = 3 - (G - 1) + k;  // first byte of the window
      uint32_t before = 0;
#pragma unroll
      for (int j = first; j < 3; ++j) before |= touched_lo & (1u << (8 * j));
      const bool valid = s >= 0 && s + G <= n && before == 0;
      int in = 0;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int b = first + j;
        const uint32_t nb = b < 4 ? __byte_perm(nlo, 0u, 0x4440u + (uint32_t)b)
                                  : __byte_perm(nhi, 0u, 0x4440u + (uint32_t)(b - 4));
        in = in * kAlpha + (int)nb;
      }
      // invalid windows read entry 0 and a neighbouring score; both are discarded
      const int v = lookup(valid ? in : 0) - lds_u16(ws_base + 2u * (uint32_t)s);
      delta += valid ? v : 0;
    }
    return delta;
  }

  // touched position j (0 <= j < na + nb) of the interchange with cipher letters xa, xb
  __device__ __forceinline__ int touched(int j, int sa, int na, int sb) const {
    return j < na ? (int)occ[sa + j] : (int)occ[sb + j - na];
  }
};

// kMissBatch: cache misses walked together, one per lane group (8 for short texts, whose
// walks are a few positions each; 4 for long texts read through L2)
template <int G, bool SMEM_TAB, int kNgWarps, int kMissBatch>
__global__ void __launch_bounds__(kNgWarps * 32, 512 / (kNgWarps * 16)) mas_ngram_kernel(const MasNgramLaunch p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kTab = pow26(G);
  uint32_t tab_bytes = 0;
  if (SMEM_TAB) {
    uint16_t* stab = reinterpret_cast<uint16_t*>(smem_raw);
    for (int i = threadIdx.x; i < kTab; i += blockDim.x) stab[i] = p.table[i];
    tab_bytes = ((uint32_t)kTab * 2u + 15u) & ~15u;
    __syncthreads();
  }
  const int max_len = (int)p.max_len;
  unsigned char* wb = smem_raw + tab_bytes + (size_t)warp * ng_warp_bytes(max_len);
  uint8_t* text = wb;  // plain[i] at text[4 + i]
  uint16_t* occ = reinterpret_cast<uint16_t*>(wb + ng_text_stride(max_len));
  uint16_t* start = reinterpret_cast<uint16_t*>(wb + ng_text_stride(max_len) + ng_u16_bytes(max_len));
  uint32_t* cursor = reinterpret_cast<uint32_t*>(start + 32);
  // exact deltas of the current state already computed, keyed by the letter pair (a < b):
  // valid while dtag == epoch, and every accept starts a new epoch (a rejected proposal leaves
  // the state unchanged, so late in a climb almost every proposal is a cache hit)
  int* dcache = reinterpret_cast<int*>(cursor + 32);
  uint16_t* dtag = reinterpret_cast<uint16_t*>(dcache + 676);
  // table score of every window of the current plaintext (ws[s] for the window starting at s)
  uint16_t* ws = reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(dcache) + kCacheBytes);
  uint64_t* rk = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(ws) + ng_u16_bytes(max_len));

  NgState<G, SMEM_TAB> st;
  st.tab = p.table;
  // held in a register (an opaque copy: the compiler would otherwise rebuild the shared
  // window address with uniform-datapath instructions at every lookup)
  asm volatile("mov.u32 %0, %1;" : "=r"(st.tab_s) : "r"(smem_addr(smem_raw)));
  st.text_base = smem_addr(text);
  st.occ = occ;
  st.start = start;
  st.ws_base = smem_addr(ws);

  const int64_t stride = (int64_t)gridDim.x * kNgWarps;
  const uint32_t climbings = (uint32_t)p.climbings;

  const WorkerTickets tk{p.tickets, stride};
  for (int64_t w = (int64_t)blockIdx.x * kNgWarps + warp; w < p.n_workers; w = tk.next(w, lane)) {
    const int32_t cid = p.cipher_of[w];
    const int64_t off = p.offsets[cid];
    const int n = (int)(p.offsets[cid + 1] - off);
    const uint8_t* ct = p.ciphers + off;
    st.n = n;

    // plaintext := ciphertext (the worker starts at the ciphertext, mas.py:229)
    for (int i = lane; i < n + 12; i += 32) text[i] = (i >= 4 && i < n + 4) ? ct[i - 4] : 0xff;
    cursor[lane] = 0;
    __syncwarp();
    // occurrence lists: counting sort of positions by cipher letter
    for (int i = lane; i < n; i += 32) atomicAdd(&cursor[ct[i]], 1u);
    __syncwarp();
    {
      const int c = (int)cursor[lane];
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += u;
      }
      start[lane] = (uint16_t)(inc - c);  // lanes >= 26: start = n
      cursor[lane] = (uint32_t)(inc - c);
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) occ[atomicAdd(&cursor[ct[i]], 1u)] = (uint16_t)i;
    __syncwarp();

    // initial score (mas.py:232)
    int64_t score = 0;
    {
      int part = 0;
      for (int s = lane; s + G <= n; s += 32) {
        int idx = 0;
#pragma unroll
        for (int j = 0; j < G; ++j) idx = idx * kAlpha + text[4 + s + j];
        const int v = st.lookup(idx);
        ws[s] = (uint16_t)v;
        part += v;
      }
      // partial sums < 32 x ceil(n/32) x 65535 < 2^31 for n <= 32768
      score = (int64_t)(int)__reduce_add_sync(kFull, (uint32_t)part);
    }
    int pinv = lane < kAlpha ? lane : 0;  // pi^-1(lane): the cipher letter holding plaintext lane
    for (int i = lane; i < 676 / 2; i += 32) reinterpret_cast<uint32_t*>(dtag)[i] = 0u;
    uint32_t epoch = 1;
    int64_t walks = 0;  // deltas computed by a position walk (the rest came from the cache)
    uint32_t reads = 0;  // this lane's table reads (G per walked position / refreshed window)
    __syncwarp();

    ByteWindow2 win;
    win.key = p.keys + 2 * w;
    philox_round_keys(rk, __ldg(win.key), __ldg(win.key + 1), lane);
    __syncwarp();
    win.rk = smem_addr(rk);
    win.start(p.skips ? p.skips[w] : 0, lane);

    // Exact deltas of up to four interchanges (lane g < 4 holds pair g in ga, gb; valid: it
    // is a miss to compute) into the cache.  The warp's lanes are split between the four
    // walks in proportion to their touched-position counts (at least one lane each), so
    // uneven letter frequencies do not idle lanes.
    auto eval_misses = [&](uint32_t ga, uint32_t gb, bool valid) {
      const int xa = __shfl_sync(kFull, pinv, (int)ga), xb = __shfl_sync(kFull, pinv, (int)gb);
      const int sa = start[xa], na = (int)start[xa + 1] - sa;
      const int sb = start[xb], nb = (int)start[xb + 1] - sb;
      const int cnt = valid ? na + nb : 0;
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < kMissBatch; o <<= 1) {
        const int u = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += u;
      }
      const int total = max(__shfl_sync(kFull, incl, kMissBatch - 1), 1);
      // first lane of walk g: ~floor((33 - MB) * positions before g / total) + g, monotone
      // with steps >= 1 and < 32 for the last walk (any such split is exact; it only
      // balances the work).  The walks' first lanes as a bit mask give each lane its walk.
      float rt;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rt) : "f"((float)total));
      constexpr int kSpread = 33 - kMissBatch;
      const int first = min((int)((float)kSpread * (float)(incl - cnt) * rt), kSpread - 1) + lane;
      const uint32_t starts = __reduce_or_sync(kFull, lane < kMissBatch ? 1u << first : 0u);
      const uint32_t upto = starts & (0xffffffffu >> (31 - lane));  // starts at lanes <= lane
      const int g = __popc(upto) - 1;
      const int lo_lane = 31 - __clz(upto);
      const uint32_t above = starts & ~(0xffffffffu >> (31 - lane));
      const int hi_lane = above ? __ffs(above) - 1 : 32;
      const int msa = __shfl_sync(kFull, sa, g), mna = __shfl_sync(kFull, na, g);
      const int msb = __shfl_sync(kFull, sb, g), mcnt = __shfl_sync(kFull, cnt, g);
      const uint32_t ma = (uint32_t)__shfl_sync(kFull, (int)ga, g);
      const uint32_t mb = (uint32_t)__shfl_sync(kFull, (int)gb, g);
      const uint32_t arep = ma * 0x01010101u, brep = mb * 0x01010101u;
      walks += __popc(__ballot_sync(kFull, valid));
      int d = 0;
      for (int j = lane - lo_lane; j < mcnt; j += hi_lane - lo_lane) {
        d += st.position_delta(st.touched(j, msa, mna, msb), arep, brep);
        reads += G;
      }
      // per-walk sums: an inclusive warp scan, differenced at each walk's lane range
      int sc = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(kFull, sc, o);
        if (lane >= o) sc += u;
      }
      const int nxt = __shfl_down_sync(kFull, first, 1);  // every lane takes part
      const int my_first = lane < kMissBatch ? first : 0;
      const int my_last = lane + 1 < kMissBatch ? nxt - 1 : 31;
      const int s_hi = __shfl_sync(kFull, sc, my_last);
      const int s_lo = __shfl_sync(kFull, sc, (my_first + 31) & 31);
      const int dsum = s_hi - (my_first > 0 ? s_lo : 0);
      __syncwarp();  // the round's cache reads precede these writes
      if (valid) {
        const int key = (int)(min(ga, gb) * kAlpha + max(ga, gb));
        dcache[key] = dsum;
        dtag[key] = (uint16_t)epoch;
      }
      __syncwarp();
    };
    auto eval_one = [&](uint32_t a, uint32_t b) -> int {
      const int xa = __shfl_sync(kFull, pinv, (int)a), xb = __shfl_sync(kFull, pinv, (int)b);
      const int sa = start[xa], na = (int)start[xa + 1] - sa;
      const int sb = start[xb], nb = (int)start[xb + 1] - sb;
      const uint32_t arep = a * 0x01010101u, brep = b * 0x01010101u;
      const int key = (int)(min(a, b) * kAlpha + max(a, b));
      if (dtag[key] == epoch) return dcache[key];
      ++walks;
      int d = 0;
      for (int j = lane; j < na + nb; j += 32) {
        d += st.position_delta(st.touched(j, sa, na, sb), arep, brep);
        reads += G;
      }
      d = (int)__reduce_add_sync(kFull, (uint32_t)d);
      __syncwarp();  // every lane's tag read precedes the write
      if (lane == 0) {
        dcache[key] = d;
        dtag[key] = (uint16_t)epoch;
      }
      __syncwarp();
      return d;
    };
    // commit a<->b (mas.py:237-243)
    auto accept = [&](int a, int b, int d) {
      score += d;
      const int xa = __shfl_sync(kFull, pinv, a), xb = __shfl_sync(kFull, pinv, b);
      const int sa = start[xa], na = (int)start[xa + 1] - sa;
      const int sb = start[xb], nb = (int)start[xb + 1] - sb;
      __syncwarp();
      for (int j = lane; j < na + nb; j += 32) {
        const int i = st.touched(j, sa, na, sb);
        text[4 + i] = (uint8_t)(j < na ? b : a);
      }
      __syncwarp();
      for (int j = lane; j < na + nb; j += 32) {  // windows holding a touched position
        const int i = st.touched(j, sa, na, sb);
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int s0 = i - (G - 1) + k;
          if (s0 >= 0 && s0 + G <= st.n) {
            int idx = 0;
#pragma unroll
            for (int q = 0; q < G; ++q) idx = idx * kAlpha + text[4 + s0 + q];
            ws[s0] = (uint16_t)st.lookup(idx);
            ++reads;
          }
        }
      }
      if (lane == a) pinv = xb;
      if (lane == b) pinv = xa;
      if (++epoch == 0x10000u) {  // tags wrap: clear them
        for (int i = lane; i < 676 / 2; i += 32) reinterpret_cast<uint32_t*>(dtag)[i] = 0u;
        epoch = 1;
      }
      __syncwarp();
    };
    auto improvable = [&]() {
      for (uint32_t a2 = 0; a2 < kAlpha - 1; ++a2)
        for (uint32_t b2 = a2 + 1; b2 < kAlpha; ++b2)
          if (eval_one(a2, b2) > 0) return true;
      return false;
    };

    int last = -1;
    uint32_t t = 0, since = 0, next_check = 256;
    auto check_exit = [&]() {  // true: the climb is at a local optimum (early-exit mode)
      if (!(p.flags & CCG_FLAG_EARLY_EXIT) || since < next_check) return false;
      if (!improvable()) return true;
      next_check *= 4;
      return false;
    };
    while (t < climbings) {
      if (win.o >= 128u) win.advance(lane);  // o <= 128 at every round start
      // Round: up to 32 proposals, one per lane, paired exactly as in ccg_mas_dform.cu
      // (aligned pairs, one redraw, shifted pairs; rng.py:81-89).  The cached deltas of the
      // prefix before the first cache miss decide it: the first positive one is accepted,
      // otherwise the prefix is rejected.  On a miss, the first four misses of the round are
      // computed (one per 8-lane group) into the cache and the round is re-run from the
      // first miss -- proposals never read the state, so computing ahead is exact.
      const uint32_t o = win.o;
      const uint32_t wd = win.round_letters(lane);
      const uint32_t c0 = wd & 0xffu, c1 = __byte_perm(wd, 0u, 0x4441u), c2 = __byte_perm(wd, 0u, 0x4442u);
      // (o <= 128, so all 32 pairs and their redraw partners lie in the 256-draw window)
      // lane j + 1's first two letters: after a second redraw the pairs realign on even draws
      // one lane further on (three segments, as in ccg_mas_dform.cu)
      const uint32_t wn = __shfl_down_sync(kFull, wd, 1);
      const uint32_t n0 = wn & 0xffu, n1 = __byte_perm(wn, 0u, 0x4441u);
      const uint32_t eqA = __ballot_sync(kFull, c0 == c1);
      const uint32_t r0 = eqA ? (uint32_t)(__ffs(eqA) - 1) : 32u;
      uint32_t R = 32u;    // pairs in this round
      uint32_t r1 = 32u;   // the second redraw pair, if handled
      bool seq = false;    // the round stopped at a pair that needs the sequential path
      if (eqA != 0u) {  // (r0 < 32)
        const uint32_t c2r = __shfl_sync(kFull, c2, (int)r0), c0r = __shfl_sync(kFull, c0, (int)r0);
        if (c2r == c0r) {
          R = r0;
          seq = true;
        } else {
          const uint32_t eqB = __ballot_sync(kFull, c1 == c2) & ~((2u << r0) - 1u);
          if (eqB) {
            const uint32_t rb = (uint32_t)(__ffs(eqB) - 1);
            const uint32_t a1 = __shfl_sync(kFull, c1, (int)rb), b1 = __shfl_sync(kFull, n1, (int)rb);
            if (rb == 31u || b1 == a1) {
              R = rb;  // the next round handles it as its first-segment redraw
            } else {
              r1 = rb;
              const uint32_t eqC = __ballot_sync(kFull, n0 == n1) & ~((2u << r1) - 1u);
              R = eqC ? min((uint32_t)(__ffs(eqC) - 1), 31u) : 31u;
            }
          }
        }
      }
      if (R > climbings - t) {
        R = climbings - t;
        seq = false;
      }
      const uint32_t j = (uint32_t)lane;
      const uint32_t pa = j <= r0 ? c0 : (j <= r1 ? c1 : n0);
      const uint32_t pb = j < r0 ? c1 : (j < r1 ? c2 : n1);
      const int key = (int)(min(pa, pb) * kAlpha + max(pa, pb));
      const bool in = j < R;
      const bool hit = in && dtag[key] == epoch;
      const int d = hit ? dcache[key] : 0;
      const uint32_t miss = __ballot_sync(kFull, in && !hit);
      const uint32_t f = miss ? (uint32_t)(__ffs(miss) - 1) : R;
      const uint32_t acc = __ballot_sync(kFull, j < f && d > 0);
      if (acc) {
        const uint32_t k = (uint32_t)(__ffs(acc) - 1);
        const int ak = __shfl_sync(kFull, (int)pa, (int)k), bk = __shfl_sync(kFull, (int)pb, (int)k);
        const int dk = __shfl_sync(kFull, d, (int)k);
        t += k;
        win.o += 2u * (k + 1u) + ((r0 - (k + 1u)) >> 31) + ((r1 - (k + 1u)) >> 31);  // + redraws
        accept(ak, bk, dk);
        last = (int)t;
        since = 0;
        next_check = 256;
        ++t;
        continue;
      }
      t += f;
      since += f;
      win.o += 2u * f + ((r0 - f) >> 31) + ((r1 - f) >> 31);  // + (f > r0) + (f > r1)
      if (f < R) {
        // lane g < kMissBatch takes the g-th miss of the round
        uint32_t m = miss, mg = 32u;
#pragma unroll
        for (int g = 0; g < kMissBatch; ++g) {
          const uint32_t q = m ? (uint32_t)(__ffs(m) - 1) : 32u;
          if (g == lane) mg = q;
          m &= m - 1u;
        }
        const int ga = __shfl_sync(kFull, (int)pa, (int)(mg & 31u));
        const int gb = __shfl_sync(kFull, (int)pb, (int)(mg & 31u));
        eval_misses((uint32_t)ga, (uint32_t)gb, mg < 32u);
        continue;
      }
      if (check_exit()) break;
      if (seq && t < climbings) {  // one try through the sequential redraw path
        int a2, b2;
        win.pair(lane, a2, b2);
        const int d2 = eval_one((uint32_t)a2, (uint32_t)b2);
        if (d2 > 0) {
          accept(a2, b2, d2);
          last = (int)t;
          since = 0;
          next_check = 256;
        } else {
          ++since;
        }
        ++t;
        if (check_exit()) break;
      }
    }
    if (lane < kAlpha && p.maps) p.maps[w * kAlpha + pinv] = (uint8_t)lane;
    const uint32_t all_reads = p.lookups ? __reduce_add_sync(kFull, reads) : 0u;
    if (lane == 0) {
      if (p.lookups) p.lookups[w] = (int64_t)all_reads;
      p.scores[w] = score;
      if (p.draws_used) p.draws_used[w] = win.position();
      if (p.last_accept) p.last_accept[w] = last;
      if (p.tries_done) p.tries_done[w] = t;
      if (p.computed) p.computed[w] = walks;
    }
    __syncwarp();
  }
}

template <int G, bool SMEM_TAB, int kNgWarps>
cudaError_t launch_ng_w(cudaStream_t s, const MasNgramLaunch& p, int sm_count) {
  // measured: 8 misses per batch +10 % on 60-100-letter quadgram climbs and +4 % on
  // 300-letter trigram ones, -5 % on 300-letter quadgram (L2-bound) ones
  auto kern = (G == 4 && p.max_len > 128) ? mas_ngram_kernel<G, SMEM_TAB, kNgWarps, 4>
                                          : mas_ngram_kernel<G, SMEM_TAB, kNgWarps, 8>;
  const size_t tab = SMEM_TAB ? (((size_t)pow26(G) * 2 + 15) & ~(size_t)15) : 0;
  const size_t bytes = tab + (size_t)kNgWarps * ng_warp_bytes((int)p.max_len);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNgWarps * 32, bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (p.n_workers + kNgWarps - 1) / kNgWarps;
  const int64_t resident = (int64_t)per_sm * sm_count;
  const int grid = (int)(need < resident ? need : resident);
  kern<<<grid, kNgWarps * 32, bytes, s>>>(p);
  return cudaGetLastError();
}

// The largest block the shared-memory layout allows: 32 warps when a staged table is shared
// by a whole SM, else 16, 8 or 4 (more warps hide the table-lookup latency).
template <int G, bool SMEM_TAB>
cudaError_t launch_ng(cudaStream_t s, const MasNgramLaunch& p, int sm_count) {
  const size_t tab = SMEM_TAB ? (((size_t)pow26(G) * 2 + 15) & ~(size_t)15) : 0;
  const size_t wb = ng_warp_bytes((int)p.max_len);
  if (SMEM_TAB && tab + 32 * wb <= 227 * 1024)  // one 32-warp block per SM shares the table (opt-in max)
    return launch_ng_w<G, SMEM_TAB, 32>(s, p, sm_count);
  if (tab + 16 * wb <= 200 * 1024) return launch_ng_w<G, SMEM_TAB, 16>(s, p, sm_count);
  if (tab + 8 * wb <= 200 * 1024) return launch_ng_w<G, SMEM_TAB, 8>(s, p, sm_count);
  return launch_ng_w<G, SMEM_TAB, 4>(s, p, sm_count);
}

// ngrams.py:134-140 generalised to order G: one warp per text, int64 sum.
__global__ void ngram_score_kernel(const uint8_t* __restrict__ texts, const int64_t* __restrict__ offsets,
                                   int64_t n_texts, int order, const int64_t* __restrict__ table,
                                   int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= n_texts) return;
  const int64_t off = offsets[j], n = offsets[j + 1] - off;
  long long part = 0;
  for (int64_t s = lane; s + order <= n; s += 32) {
    int64_t idx = 0;
    for (int q = 0; q < order; ++q) idx = idx * kAlpha + texts[off + s + q];
    part += table[idx];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
  if (lane == 0) out[j] = part;
}

}  // namespace

cudaError_t launch_mas_ngram_climb(cudaStream_t s, const MasNgramLaunch& p, int sm_count) {
  if (p.n_workers <= 0) return cudaSuccess;
  switch (p.order) {
    case 2: return launch_ng<2, true>(s, p, sm_count);
    case 3: return launch_ng<3, true>(s, p, sm_count);
    case 4: return launch_ng<4, false>(s, p, sm_count);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ngram_score(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                               int64_t n, int order, const int64_t* table, int64_t* out) {
  if (n <= 0) return cudaSuccess;
  const int64_t threads = n * 32;
  ngram_score_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(texts, offsets, n, order,
                                                                        table, out);
  return cudaGetLastError();
}

}  // namespace ccg
