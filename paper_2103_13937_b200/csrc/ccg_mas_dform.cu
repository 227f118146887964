// ccg_mas_dform.cu -- the MAS stochastic climb from maintained aggregates that give every
// exact swap delta in O(1) ("D-form"): the sm_100a fast path of mas.py:218-244
// stochastic_worker.  Default: deltas computed on demand from T, N (five reads); variant
// CCG_FLAG_KERNEL_DTABLE keeps the full 325-entry delta table instead.
//
// Why.  A rejected proposal does not change the state, and ~99% of proposals are rejected
// (the reference accepts ~70 of 10,000 tries, mas.py:237).  The reference recomputes
// swap_delta (mas.py:181-210, 208 lookups) for every try; between two accepts the same
// state is re-scored over and over.  Here the warp keeps ALL 325 exact deltas of the
// current state in shared memory,
//     D[a][b] = swap_delta(counts, a, b, S),
// and rebuilds them only when a proposal is accepted.  Evaluating a proposal is one lookup,
// so 32 proposals are evaluated by one warp instruction (lane j takes proposal t+j) and a
// ballot finds the first accepted one -- exactly the sequential outcome, because proposals
// never read the state (rng.py:81-89).
//
// Algebra (all exact integers).  With T the bigram counts of the current plaintext:
//   D[a][b] = kt(a,b) * ks(a,b) - (N[a][a] + N[b][b] - N[a][b] - N[b][a])
//   kt = T[a][a] + T[b][b] - T[a][b] - T[b][a],  ks = the same on S (static),
//   N[x][y] = sum_q T[x][q] S[y][q] + T[q][x] S[q][y],
// which is the T-form identity of ccg_mas_tform.cu expanded over rows/columns.  Accepting
// the interchange sigma = (a b) maps T'[x][y] = T[sigma x][sigma y], and
//   N'[x][y] = N[sigma x][y] + (T[sx][a] - T[sx][b]) (S[y][b] - S[y][a])
//                             + (T[a][sx] - T[b][sx]) (S[b][y] - S[a][y]),   sx = sigma x,
// an O(676) update; D is then rebuilt from N, T and ks (325 pairs).
//
// Proposal stream.  The letter window is the byte window of ccg_mas_common.cuh (one
// Philox4x64-10 block per lane per refill, int(u*26) exact).  A pair with equal letters
// needs a redraw (rng.py:85-86) and shifts the pairing by one draw, so each lane reads
// three letters and a round covers the aligned pairs before the first redraw, the redraw
// pair itself, and the shifted pairs up to the next redraw (two ballots) -- ~30 tries per
// round; anything rarer (a double redraw) goes through the sequential path.
//
// Gate: max(S) <= 32767, n <= 32768 and (n-1)*max(S) < 2^27 keep every N and D entry in
// int32 (|D| < 12 (n-1) max(S)); the host falls back to the T-form / packed kernels.
#include "ccg_mas_common.cuh"

namespace ccg {
namespace {

constexpr int kDWarps = 8;
// T row stride (int16) = N's row stride (kNT): T[a][b] and NT[a][b] (= N[b][a]) share the index
// a * 36 + b, so an on-demand delta computes two indices for its four T/N reads (and KS uses
// the same stride for the fifth)
constexpr int kTS = 36;
constexpr int kNS = 33;  // S row stride (int32)
// N is stored TRANSPOSED: lane y's column N[.][y] is the contiguous row NT[y][.], stride 36
// words (16-byte aligned), so the accept's rank-2 update streams it with 128-bit loads and
// stores (each 8-lane phase of an LDS.128 hits distinct banks: 4y + x mod 32)
constexpr int kNT = 36;
constexpr int kDS = 32;  // D row stride (int32): D[a][b] sits in bank b
constexpr int kKS = 36;  // KS row stride (int32), = kTS

// TABLE = true keeps D in shared memory (rebuilt on every accept); TABLE = false computes
// each looked-up delta from T, N and ks on demand (no rebuild, 3.3 KB less per warp).
template <bool TABLE>
struct alignas(16) DWarp {
  uint64_t rk[22];  // Philox round keys of the current worker's stream (+ M0*k0)
  int2 uv[28];      // accept: the (u_x, v_x) row factors of the N update (x < 26; 26, 27 pad)
  int16_t T[kAlpha * kTS];  // (936 int16: N starts 16-byte aligned)
  int N[kAlpha * kNT];      // N[x][y] at N[y * kNT + x]
  int D[TABLE ? kAlpha * kDS : 4];
};
template <bool TABLE>
struct DBlock {
  int S[kAlpha * kNS];
  int KS[kAlpha * kKS];
  DWarp<TABLE> w[kDWarps];
};

// Initial state of a ciphertext's workers (identical for all of them: they start at the
// ciphertext), computed once per ciphertext by dform_init_kernel when several workers share
// a ciphertext: T and N in the shared-memory layout, and the score.
struct alignas(16) CipherInit {
  int16_t T[kAlpha * kTS];
  int N[kAlpha * kNT];
  int score;
  int pad_[3];
};
constexpr int kInitVec = (int)(sizeof(CipherInit) / 16);

template <class WT>
__device__ __forceinline__ int t_at(const WT& W, int x, int y) { return W.T[x * kTS + y]; }

// T[x][y] += 1 via a 32-bit shared atomic on the containing word (no 16-bit atomics)
template <class WT>
__device__ __forceinline__ void t_inc(WT& W, int x, int y) {
  const uint32_t idx = (uint32_t)(x * kTS + y);
  uint32_t* word = reinterpret_cast<uint32_t*>(W.T) + (idx >> 1);
  atomicAdd(word, 1u << (16u * (idx & 1u)));
}

// D[x][y] for all x != y from the current T, N (and the static ks).  Lane y builds column
// y, so every shared access is either a broadcast (diagonals, via shuffles) or lands in a
// distinct bank (row strides 17, 33 and 32 words): no bank conflicts.
template <class BT, class WT>
__device__ __forceinline__ void rebuild_D(const BT& B, WT& W, int lane) {
  __syncwarp();
  const int y = lane < kAlpha ? lane : 0;
  const int tyy = t_at(W, y, y), nyy = W.N[y * kNT + y];
#pragma unroll
  for (int x = 0; x < kAlpha; ++x) {
    const int txx = __shfl_sync(kFull, tyy, x), nxx = __shfl_sync(kFull, nyy, x);
    const int kt = txx + tyy - t_at(W, x, y) - t_at(W, y, x);
    const int dv = kt * B.KS[x * kKS + y] - nxx - nyy + W.N[y * kNT + x] + W.N[x * kNT + y];
    if (lane < kAlpha) W.D[x * kDS + y] = dv;
  }
  __syncwarp();
}

// D[a][b] from T, N and ks; tdg / ndg hold T[lane][lane] / N[lane][lane] (all lanes call).
// ks_s: 32-bit shared address of B.KS.  With i1 = a*36 + b, i2 = b*36 + a:
// T[a][b] = T[i1], T[b][a] = T[i2], N[b][a] = NT[i1], N[a][b] = NT[i2], ks = KS[i1].
template <class WT>
__device__ __forceinline__ int delta_at(uint32_t ks_s, const WT& W, int tdg, int ndg, int a, int b) {
  static_assert(kTS == kNT && kKS == kNT, "delta_at shares one index across T, N and KS");
  const int ta = __shfl_sync(kFull, tdg, a), tb = __shfl_sync(kFull, tdg, b);
  const int na = __shfl_sync(kFull, ndg, a), nb = __shfl_sync(kFull, ndg, b);
  const uint32_t i1 = (uint32_t)(a * kTS + b), i2 = (uint32_t)(b * kTS + a);
  const int kt = ta + tb - W.T[i1] - W.T[i2];
  // ks through a 32-bit shared address (a generic B.KS access recomputes the window base)
  const int ks = (int)lds_u32(ks_s + 4u * i1);
  return kt * ks - na - nb + W.N[i2] + W.N[i1];
}

// max over the 325 on-demand deltas; lane y scans column y
template <class WT>
__device__ __forceinline__ int max_delta(uint32_t ks_s, const WT& W, int tdg, int ndg, int lane) {
  int m = (int)0x80000000;
  const int y = lane < kAlpha ? lane : 0;
  for (int x = 0; x < kAlpha; ++x) {
    const int dv = delta_at(ks_s, W, tdg, ndg, x, y);
    if (lane < kAlpha && x != lane) m = max(m, dv);
  }
  return __reduce_max_sync(kFull, m);
}

// max over the 325 deltas (exact local-optimum test); lane y scans column y
template <class WT>
__device__ __forceinline__ int max_D(const WT& W, int lane) {
  int m = (int)0x80000000;
  if (lane < kAlpha)
    for (int x = 0; x < kAlpha; ++x)
      if (x != lane) m = max(m, W.D[x * kDS + lane]);
  return __reduce_max_sync(kFull, m);
}

// T = bigram counts of the ciphertext (the worker starts at the ciphertext, mas.py:229-230),
// N from scratch (lane y owns column y), returns the score (mas.py:232)
template <class BT, class WT>
__device__ __forceinline__ int64_t initial_state(const BT& B, WT& W, const uint8_t* text,
                                                 int64_t n, int lane, int y) {
  for (int i = lane; i < kAlpha * kTS / 2; i += 32) reinterpret_cast<uint32_t*>(W.T)[i] = 0u;
  __syncwarp();
  for (int64_t i = lane; i + 1 < n; i += 32) t_inc(W, text[i], text[i + 1]);
  __syncwarp();
  int part = 0;
  if (lane < kAlpha) {
    for (int x = 0; x < kAlpha; ++x) {
      int acc = 0;
      for (int q = 0; q < kAlpha; ++q)
        acc += t_at(W, x, q) * B.S[y * kNS + q] + t_at(W, q, x) * B.S[q * kNS + y];
      W.N[y * kNT + x] = acc;
      part += t_at(W, x, y) * B.S[x * kNS + y];
    }
  }
  const int64_t score = (int64_t)(int)__reduce_add_sync(kFull, (uint32_t)part);
  __syncwarp();
  return score;
}

template <bool TABLE>
__device__ __forceinline__ void stage_block_tables(DBlock<TABLE>& B, const int64_t* table) {
  for (int i = threadIdx.x; i < kAlpha * kAlpha; i += blockDim.x) {
    const int x = i / kAlpha, y = i - x * kAlpha;
    B.S[x * kNS + y] = (int)table[i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kAlpha * kAlpha; i += blockDim.x) {
    const int x = i / kAlpha, y = i - x * kAlpha;
    B.KS[x * kKS + y] =
        B.S[x * kNS + x] + B.S[y * kNS + y] - B.S[x * kNS + y] - B.S[y * kNS + x];
  }
  __syncthreads();
}

// One warp per ciphertext: its workers' common initial state.
__global__ void __launch_bounds__(kDWarps * 32) dform_init_kernel(const MasLaunch p, int64_t n_ciphers,
                                                                  CipherInit* out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DBlock<false>& B = *reinterpret_cast<DBlock<false>*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  DWarp<false>& W = B.w[warp];
  stage_block_tables(B, p.table);
  const int y = lane < kAlpha ? lane : 0;
  for (int64_t c = (int64_t)blockIdx.x * kDWarps + warp; c < n_ciphers;
       c += (int64_t)gridDim.x * kDWarps) {
    const int64_t off = p.offsets[c], n = p.offsets[c + 1] - off;
    const int64_t score = initial_state(B, W, p.ciphers + off, n, lane, y);
    const uint4* src = reinterpret_cast<const uint4*>(W.T);
    uint4* dst = reinterpret_cast<uint4*>(out + c);
    for (int i = lane; i < kInitVec - 1; i += 32) dst[i] = src[i];
    if (lane == 0) out[c].score = (int)score;
    __syncwarp();
  }
}

template <bool EARLY, bool TABLE>
__global__ void __launch_bounds__(kDWarps * 32, TABLE ? 3 : 4) mas_climb_dform_kernel(const MasLaunch p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DBlock<TABLE>& B = *reinterpret_cast<DBlock<TABLE>*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  DWarp<TABLE>& W = B.w[warp];

  stage_block_tables(B, p.table);

  const int64_t stride = (int64_t)gridDim.x * kDWarps;
  const uint32_t climbings = (uint32_t)p.climbings;
  const int y = lane < kAlpha ? lane : 0;  // the column this lane owns in N updates
  // held in a register (an opaque copy: otherwise the shared window address is rebuilt with
  // S2R/uniform instructions in every round)
  uint32_t ks_s;
  asm volatile("mov.u32 %0, %1;" : "=r"(ks_s) : "r"(smem_addr(B.KS)));

  const WorkerTickets tk{p.tickets, stride};
  for (int64_t w = (int64_t)blockIdx.x * kDWarps + warp; w < p.n_workers; w = tk.next(w, lane)) {
    const int32_t cid = p.cipher_of[w];
    const int64_t off = p.offsets[cid], n = p.offsets[cid + 1] - off;
    const uint8_t* text = p.ciphers + off;

    int64_t score;
    if (p.init) {  // the ciphertext's initial state, computed once by dform_init_kernel
      const uint4* src = reinterpret_cast<const uint4*>(p.init) + (int64_t)cid * kInitVec;
      uint4* dst = reinterpret_cast<uint4*>(W.T);  // T, N are contiguous like CipherInit
      for (int i = lane; i < kInitVec - 1; i += 32) dst[i] = src[i];
      score = reinterpret_cast<const CipherInit*>(p.init)[cid].score;
      __syncwarp();
    } else {
      score = initial_state(B, W, text, n, lane, y);
    }
    int tdg = 0, ndg = 0;  // T[lane][lane], N[lane][lane] (on-demand deltas)
    if (TABLE) {
      rebuild_D(B, W, lane);
    } else {
      __syncwarp();
      tdg = t_at(W, y, y);
      ndg = W.N[y * kNT + y];
    }

    int pv = lane < kAlpha ? lane : 0;  // pi(lane): cipher letter -> plaintext letter
    ByteWindow2 win;
    win.key = p.keys + 2 * w;
    philox_round_keys(W.rk, __ldg(win.key), __ldg(win.key + 1), lane);
    __syncwarp();
    win.rk = smem_addr(W.rk);
    win.start(p.skips ? p.skips[w] : 0, lane);

    // commit the interchange a<->b (mas.py:237-243)
    auto accept = [&](int a, int b, int d) {
      score += d;
      pv = pv == a ? b : (pv == b ? a : pv);
      // lane x: u_x = T[sx][a] - T[sx][b], v_x = T[a][sx] - T[b][sx] (old T, sx = sigma x)
      const int x = lane < kAlpha ? lane : 0;
      const int sx = x == a ? b : (x == b ? a : x);
      const int u = t_at(W, sx, a) - t_at(W, sx, b);
      const int v = t_at(W, a, sx) - t_at(W, b, sx);
      // lane y: S-column factors of its N column
      const int sb = B.S[y * kNS + b] - B.S[y * kNS + a];
      const int sc = B.S[b * kNS + y] - B.S[a * kNS + y];
      const int na = W.N[y * kNT + a], nb = W.N[y * kNT + b];
      const int ua = __shfl_sync(kFull, u, a), va = __shfl_sync(kFull, v, a);
      const int ub = __shfl_sync(kFull, u, b), vb = __shfl_sync(kFull, v, b);
      if (lane < 28) W.uv[lane] = lane < kAlpha ? make_int2(u, v) : make_int2(0, 0);
      __syncwarp();
      // N'[x][y] = N[sigma x][y] + u_x sb_y + v_x sc_y: lane y streams its column 4 entries
      // at a time (entries a, b are rewritten below from the saved old values)
      if (lane < kAlpha) {
        int4* col = reinterpret_cast<int4*>(W.N + y * kNT);
        const int4* f = reinterpret_cast<const int4*>(W.uv);
#pragma unroll
        for (int c = 0; c < 7; ++c) {
          int4 nv = col[c];
          const int4 q0 = f[2 * c], q1 = f[2 * c + 1];
          nv.x += q0.x * sb + q0.y * sc;
          nv.y += q0.z * sb + q0.w * sc;
          nv.z += q1.x * sb + q1.y * sc;
          nv.w += q1.z * sb + q1.w * sc;
          col[c] = nv;
        }
        W.N[y * kNT + a] = nb + ua * sb + va * sc;
        W.N[y * kNT + b] = na + ub * sb + vb * sc;
      }
      // swap rows a, b then columns a, b of T
      int16_t ra = 0, rb = 0;
      if (lane < kAlpha) {
        ra = W.T[a * kTS + lane];
        rb = W.T[b * kTS + lane];
      }
      __syncwarp();
      if (lane < kAlpha) {
        W.T[a * kTS + lane] = rb;
        W.T[b * kTS + lane] = ra;
      }
      __syncwarp();
      if (lane < kAlpha) {
        ra = W.T[lane * kTS + a];
        rb = W.T[lane * kTS + b];
      }
      __syncwarp();
      if (lane < kAlpha) {
        W.T[lane * kTS + a] = rb;
        W.T[lane * kTS + b] = ra;
      }
      if (TABLE) {
        rebuild_D(B, W, lane);
      } else {
        __syncwarp();
        tdg = t_at(W, y, y);
        ndg = W.N[y * kNT + y];
      }
    };
    auto optimum = [&]() {
      return TABLE ? max_D(W, lane) <= 0 : max_delta(ks_s, W, tdg, ndg, lane) <= 0;
    };

    int last = -1, nacc = 0;
    uint32_t t = 0;
    bool done = EARLY && optimum();
    while (!done && t < climbings) {
      if (win.o >= 128u) win.advance(lane);  // o <= 128 at every round start
      const uint32_t o = win.o;
      // Lane j reads letters c0, c1, c2 = L[o+2j], L[o+2j+1], L[o+2j+2].  Pairs j < r0 are
      // aligned (c0, c1); r0 is the first pair needing a redraw (c0 == c1); its partner is
      // c2 of lane r0 unless that equals c0 too; the pairs after it are shifted by one draw
      // (c1, c2) up to the next redraw.  rng.py:81-89 exactly.
      const uint32_t wd = win.round_letters(lane);
      // (one PRMT per byte: __byte_perm(x, 0, 0x444k) = byte k of x, zero-extended)
      const int c0 = (int)(wd & 0xffu), c1 = (int)__byte_perm(wd, 0u, 0x4441u), c2 = (int)__byte_perm(wd, 0u, 0x4442u);
      // (o <= 128, so all 32 pairs and their redraw partners lie in the 256-draw window)
      // Lane j + 1's first two letters: after a second redraw the pairs realign on even
      // draws again, one lane further on (lane 31 has no successor: R <= 31 then).
      const uint32_t wn = __shfl_down_sync(kFull, wd, 1);
      const int n0 = (int)(wn & 0xffu), n1 = (int)__byte_perm(wn, 0u, 0x4441u);
      const uint32_t eqA = __ballot_sync(kFull, c0 == c1);
      const uint32_t r0 = eqA ? (uint32_t)(__ffs(eqA) - 1) : 32u;  // (< 32 iff eqA != 0)
      uint32_t R = 32u;    // pairs in this round
      uint32_t r1 = 32u;   // the second redraw pair (shifted alignment), if handled
      bool seq = false;    // the round stopped at a pair that needs the sequential path
      if (eqA != 0u) {
        const int c2r = __shfl_sync(kFull, c2, (int)r0), c0r = __shfl_sync(kFull, c0, (int)r0);
        if (c2r == c0r) {
          R = r0;
          seq = true;
        } else {
          const uint32_t eqB = __ballot_sync(kFull, c1 == c2) & ~((2u << r0) - 1u);
          if (eqB) {
            // the second redraw: pair rb = (c1[rb], c1[rb + 1]) unless that is a double
            // redraw or rb is lane 31 -- then the round ends at rb and the next round
            // handles it as its first-segment redraw
            const uint32_t rb = (uint32_t)(__ffs(eqB) - 1);
            const int a1 = __shfl_sync(kFull, c1, (int)rb), b1 = __shfl_sync(kFull, n1, (int)rb);
            if (rb == 31u || b1 == a1) {
              R = rb;
            } else {
              r1 = rb;
              // third segment: lane j > r1 pairs (n0, n1) up to the next redraw
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
      const int pa = j <= r0 ? c0 : (j <= r1 ? c1 : n0);
      const int pb = j < r0 ? c1 : (j < r1 ? c2 : n1);
      int d;
      if (TABLE) {
        d = j < R ? W.D[pa * kDS + pb] : 0;
      } else {
        d = delta_at(ks_s, W, tdg, ndg, pa, pb);
        d = j < R ? d : 0;
      }
      const uint32_t acc = __ballot_sync(kFull, d > 0);
      if (acc == 0) {  // the common case: R rejections
        t += R;
        // + (R > r0) + (R > r1), the redraws consumed (all values <= 32: the sign bit of the
        // difference is the comparison, one LEA.HI each)
        win.o += 2u * R + ((r0 - R) >> 31) + ((r1 - R) >> 31);
        if (seq && t < climbings) {  // one try through the sequential redraw path
          int a2, b2;
          win.pair(lane, a2, b2);
          const int d2 = TABLE ? W.D[a2 * kDS + b2] : delta_at(ks_s, W, tdg, ndg, a2, b2);
          if (d2 > 0) {
            accept(a2, b2, d2);
            last = (int)t;
            ++nacc;
            if (EARLY) done = optimum();
          }
          ++t;
        }
        continue;
      }
      const uint32_t k = (uint32_t)(__ffs(acc) - 1);  // the first accepted proposal
      const int ak = __shfl_sync(kFull, pa, (int)k), bk = __shfl_sync(kFull, pb, (int)k);
      const int dk = __shfl_sync(kFull, d, (int)k);
      t += k;
      win.o += 2u * (k + 1u) + ((r0 - (k + 1u)) >> 31) + ((r1 - (k + 1u)) >> 31);
      accept(ak, bk, dk);
      last = (int)t;
      ++nacc;
      ++t;
      if (EARLY) done = optimum();
    }

    if (lane < kAlpha && p.maps) p.maps[w * kAlpha + lane] = (uint8_t)pv;
    if (lane == 0) {
      p.scores[w] = score;
      if (p.draws_used) p.draws_used[w] = win.position();
      if (p.last_accept) p.last_accept[w] = last;
      if (p.accepts) p.accepts[w] = nacc;
      if (p.tries_done) p.tries_done[w] = t;
    }
    __syncwarp();
  }
}

}  // namespace

bool mas_dform_ok(int64_t max_len, int64_t table_max) {
  if (table_max > 32767 || max_len > 32768) return false;
  const int64_t n1 = max_len > 0 ? max_len - 1 : 0;
  return n1 * table_max < (int64_t(1) << 27);
}

size_t dform_init_bytes(int64_t n_ciphers) { return (size_t)n_ciphers * sizeof(CipherInit); }

cudaError_t launch_dform_init(cudaStream_t s, const MasLaunch& p, int64_t n_ciphers, void* out,
                              int sm_count) {
  if (n_ciphers <= 0) return cudaSuccess;
  const int smem = (int)sizeof(DBlock<false>);
  cudaError_t e = cudaFuncSetAttribute(dform_init_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t need = (n_ciphers + kDWarps - 1) / kDWarps;
  const int grid = (int)(need < 4 * (int64_t)sm_count ? need : 4 * (int64_t)sm_count);
  dform_init_kernel<<<grid, kDWarps * 32, smem, s>>>(p, n_ciphers, (CipherInit*)out);
  return cudaGetLastError();
}

cudaError_t launch_mas_climb_dform(cudaStream_t s, const MasLaunch& p, int sm_count) {
  if (p.n_workers <= 0) return cudaSuccess;
  const bool table = (p.flags & CCG_FLAG_KERNEL_MASK) == CCG_FLAG_KERNEL_DTABLE;
  auto kern = (p.flags & CCG_FLAG_EARLY_EXIT)
                  ? (table ? mas_climb_dform_kernel<true, true> : mas_climb_dform_kernel<true, false>)
                  : (table ? mas_climb_dform_kernel<false, true> : mas_climb_dform_kernel<false, false>);
  const int smem = table ? (int)sizeof(DBlock<true>) : (int)sizeof(DBlock<false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDWarps * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (p.n_workers + kDWarps - 1) / kDWarps;
  const int64_t resident = (int64_t)per_sm * sm_count;
  const int grid = (int)(need < resident ? need : resident);
  kern<<<grid, kDWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ccg
