// ccg_mas_tform.cu -- the MAS climb in "T-form": mas.py:218-244 stochastic_worker (driven
// by mas.py:253-278 solve_stochastic) for tables beyond the D-form gate (ccg_mas_dform.cu
// is the fast path; this kernel was the round-1 headline before it).
//
// State.  Like the reference, the warp keeps the bigram-count matrix T of the CURRENT
// plaintext (mas.py:230, rows/columns swapped on accept at mas.py:239-240), not the
// ciphertext's.  Lane q owns column q of packed 16-bit tables in shared memory:
//     TS[u][q].x = T[u][q] | T[q][u] << 16      (per warp, changes on accept)
//     TS[u][q].y = S[u][q] | S[q][u] << 16      (static, copied per warp so one
//                                                 LDS.64 fetches T and S together)
// Delta.  For a plaintext interchange a<->b the reference's swap_delta (mas.py:181-210)
// equals, exactly,
//     delta = K(a,b) - sum_q [ (T[a][q]-T[b][q])(S[a][q]-S[b][q])
//                             + (T[q][a]-T[q][b])(S[q][a]-S[q][b]) ]
//     K(a,b) = (T[a][a]+T[b][b]-T[a][b]-T[b][a]) * (S[a][a]+S[b][b]-S[a][b]-S[b][a])
// (the rank-one K term is the 2x2 corner the reference removes).  Lane q's term is a
// two-way dot product of the packed differences TS[a][q]-TS[b][q], so a try costs two
// conflict-free LDS.64 (rows a and b), one broadcast LDS of K(a,b) from a per-warp
// 26x32 table, eight integer instructions and one REDUX -- no shuffles of the state,
// no per-lane select for the two moving letters.  K is kept up to date on accept
// (only the rows and columns of the two swapped letters change).
//
// Exactness.  Differences of 16-bit halves are sign-extended, so this path requires
// max(S) <= 32767, n <= 32768 and (n-1)*max(S) < 2^29 (every partial sum and K fit in
// int32); the host falls back to the packed/wide kernels of ccg_mas.cu otherwise.
// Accept decisions (delta > 0), the proposal stream and the final score are those of
// the reference; pinned by tests/test_gpu_parity.py against the oracle and the golden
// stochastic_worker runs.
#include "ccg_mas_common.cuh"

namespace ccg {
namespace {

constexpr int kTWarps = 4;     // warps (workers in flight) per block
constexpr uint32_t kRowB = 392;  // bytes per table row: 32 x uint2 (T,S), 32 x int32 K, pad
                                 // (98 words: column walks hit 2-way, not 26-way, conflicts)
constexpr uint32_t kKOff = 256;  // offset of the K part inside a row

// Per warp: 26 rows u of kRowB bytes,
//   [u][q].x = T[u][q] | T[q][u] << 16, [u][q].y = S[u][q] | S[q][u] << 16  (q < 32)
//   K[u][v]  = K(u, v) (symmetric)                                           (v < 32)
constexpr uint32_t kTWarpBytes = kAlpha * kRowB;  // 10192

__device__ __forceinline__ int sext16(uint32_t v) { return (int)(int16_t)(v & 0xffffu); }
__device__ __forceinline__ int lo16u(uint32_t v) { return (int)(v & 0xffffu); }
__device__ __forceinline__ int hi16u(uint32_t v) { return (int)(v >> 16); }

template <bool EARLY>
__global__ void __launch_bounds__(kTWarps * 32) mas_climb_tform_kernel(const MasLaunch p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wb = smem_raw + (size_t)warp * kTWarpBytes;
  const uint32_t wbase = smem_addr(wb);
  const uint32_t tsl = wbase + 8u * (uint32_t)lane;                  // [0][lane]
  const uint32_t tsr = wbase + kRowB * (uint32_t)min(lane, kAlpha - 1);  // [lane][0]
  auto T_at = [&](int u, int q) -> uint32_t* {
    return reinterpret_cast<uint32_t*>(wb + (uint32_t)u * kRowB + 8u * (uint32_t)q);
  };

  // static S halves and S diagonal (lane q: S[q][q])
  for (int u = 0; u < kAlpha; ++u) {
    uint32_t s = 0;
    if (lane < kAlpha)
      s = (uint32_t)p.table[u * kAlpha + lane] | ((uint32_t)p.table[lane * kAlpha + u] << 16);
    T_at(u, lane)[1] = s;
  }
  const int sdiag = lane < kAlpha ? (int)p.table[lane * (kAlpha + 1)] : 0;
  __syncwarp();

  const int64_t stride = (int64_t)gridDim.x * kTWarps;
  const uint32_t climbings = (uint32_t)p.climbings;

  // K(r, lane) for the current T, written to K[r][lane] and K[lane][r]
  auto k_row = [&](int r, int tdiag) {
    const uint2 e = lds_u64(tsl + kRowB * (uint32_t)r);
    const int kt = __shfl_sync(kFull, tdiag, r) + tdiag - lo16u(e.x) - hi16u(e.x);
    const int ks = __shfl_sync(kFull, sdiag, r) + sdiag - lo16u(e.y) - hi16u(e.y);
    if (lane < kAlpha) {
      sts_u32(wbase + kRowB * (uint32_t)r + kKOff + 4u * (uint32_t)lane, (uint32_t)(kt * ks));
      sts_u32(wbase + kRowB * (uint32_t)lane + kKOff + 4u * (uint32_t)r, (uint32_t)(kt * ks));
    }
  };

  const WorkerTickets tk{p.tickets, stride};
  for (int64_t w = (int64_t)blockIdx.x * kTWarps + warp; w < p.n_workers; w = tk.next(w, lane)) {
    const int32_t cid = p.cipher_of[w];
    const int64_t off = p.offsets[cid], n = p.offsets[cid + 1] - off;
    const uint8_t* text = p.ciphers + off;

    // T = bigram counts of the ciphertext (mas.py:230; the worker starts at the cipher)
    for (int u = 0; u < kAlpha; ++u) T_at(u, lane)[0] = 0u;
    __syncwarp();
    for (int64_t i = lane; i + 1 < n; i += 32) {
      const int x = text[i], y = text[i + 1];
      atomicAdd(T_at(x, y), 1u);
      atomicAdd(T_at(y, x), 1u << 16);
    }
    __syncwarp();

    // initial score (mas.py:232) and the K table
    int part = 0;
    for (int u = 0; u < kAlpha; ++u) {
      const uint2 e = lds_u64(tsl + kRowB * (uint32_t)u);
      part += lo16u(e.x) * lo16u(e.y);
    }
    int64_t score = (int64_t)(int)__reduce_add_sync(kFull, (uint32_t)part);  // < 2^29 by the gate
    int tdiag = lo16u(lds_u32(tsr + 8u * (uint32_t)lane));
    for (int r = 0; r < kAlpha; ++r) k_row(r, tdiag);
    __syncwarp();

    int pv = lane < kAlpha ? lane : 0;  // pi(lane): cipher letter -> plaintext letter
    ByteWindow win;
    win.key = p.keys + 2 * w;
    win.base = p.skips ? p.skips[w] : 0;
    win.o = 0;
    win.refill(lane);

    // exact swap_delta(a, b) of the current state (see the file header)
    auto eval = [&](uint32_t a, uint32_t b) -> int {
      const uint2 A = lds_u64(tsl + kRowB * a);
      const uint2 B = lds_u64(tsl + kRowB * b);
      const int k = (int)lds_u32(wbase + kRowB * a + kKOff + 4u * b);
      const int dT = (int)(A.x - B.x), dS = (int)(A.y - B.y);
      const int lT = sext16((uint32_t)dT), lS = sext16((uint32_t)dS);
      // (dT - lT) = hi(dT) * 2^16 exactly, so the high word of the product is hi*hi
      const int v = lT * lS + __mulhi(dT - lT, dS - lS);
      return k - (int)__reduce_add_sync(kFull, (uint32_t)v);
    };
    // commit the interchange a<->b (mas.py:237-243): swap rows a,b and columns a,b of T,
    // refresh the K rows/columns of a and b
    auto accept = [&](int a, int b, int d) {
      score += d;
      pv = pv == a ? b : (pv == b ? a : pv);
      const uint32_t ra = tsl + kRowB * (uint32_t)a, rb = tsl + kRowB * (uint32_t)b;
      const uint32_t xa = lds_u32(ra), xb = lds_u32(rb);
      sts_u32(ra, xb);
      sts_u32(rb, xa);
      __syncwarp();
      if (lane < kAlpha) {
        const uint32_t ca = tsr + 8u * (uint32_t)a, cb = tsr + 8u * (uint32_t)b;
        const uint32_t ya = lds_u32(ca), yb = lds_u32(cb);
        sts_u32(ca, yb);
        sts_u32(cb, ya);
      }
      __syncwarp();
      tdiag = lo16u(lds_u32(tsr + 8u * (uint32_t)lane));
      k_row(a, tdiag);
      k_row(b, tdiag);
      __syncwarp();
    };
    // exact local-optimum test over all 325 interchanges (CCG_FLAG_EARLY_EXIT)
    auto improvable = [&]() {
      for (uint32_t a2 = 0; a2 < kAlpha - 1; ++a2)
        for (uint32_t b2 = a2 + 1; b2 < kAlpha; ++b2)
          if (eval(a2, b2) > 0) return true;
      return false;
    };

    int last = -1, nacc = 0;
    uint32_t t = 0;
    uint32_t since = 0, next_check = 256;
    // Four proposals per iteration.  Proposals never depend on the state (rng.py:81-89
    // draws only), so tries t..t+3 are all evaluated against the state before try t.  If
    // none is accepted (the common case) that is exactly the sequential outcome; otherwise
    // they are replayed in order, re-evaluating every try after the first accept against
    // the new state.  A pair with a == b (a redraw is due) evaluates to 0 and routes the
    // batch through the sequential path from that try on.
    bool dirty = false;
    auto step = [&](uint32_t a, uint32_t b, int dd) -> bool {
      if (a == b) return false;
      const int d = dirty ? eval(a, b) : dd;
      win.o += 2;
      if (d > 0) {
        accept((int)a, (int)b, d);
        last = (int)t;
        ++nacc;
        dirty = true;
        since = 0;
        next_check = 256;
      } else {
        ++since;
      }
      ++t;
      return true;
    };
    while (t + 3 < climbings) {
      if (win.o > 120) win.refill(lane);
      uint32_t La, Lb;
      win.peek8(La, Lb);
      const uint32_t a1 = __byte_perm(La, 0, 0x4440), b1 = __byte_perm(La, 0, 0x4441);
      const uint32_t a2 = __byte_perm(La, 0, 0x4442), b2 = __byte_perm(La, 0, 0x4443);
      const uint32_t a3 = __byte_perm(Lb, 0, 0x4440), b3 = __byte_perm(Lb, 0, 0x4441);
      const uint32_t a4 = __byte_perm(Lb, 0, 0x4442), b4 = __byte_perm(Lb, 0, 0x4443);
      const int d1 = eval(a1, b1), d2 = eval(a2, b2), d3 = eval(a3, b3), d4 = eval(a4, b4);
      const bool ok = a1 != b1 && a2 != b2 && a3 != b3 && a4 != b4;
      if (ok && max(max(d1, d2), max(d3, d4)) <= 0) {  // the common case: four rejections
        win.o += 8;
        t += 4;
        if (EARLY) {
          since += 4;
          if (since >= next_check) {
            if (!improvable()) break;
            next_check *= 4;
          }
        }
        continue;
      }
      dirty = false;
      if (!(step(a1, b1, d1) && step(a2, b2, d2) && step(a3, b3, d3) && step(a4, b4, d4))) {
        // a redraw is due: one sequential try (rng.py:81-89)
        int a, b;
        win.pair(lane, a, b);
        const int d = eval((uint32_t)a, (uint32_t)b);
        if (d > 0) {
          accept(a, b, d);
          last = (int)t;
          ++nacc;
          since = 0;
          next_check = 256;
        } else {
          ++since;
        }
        ++t;
      }
      if (EARLY && since >= next_check) {
        if (!improvable()) break;
        next_check *= 4;
      }
    }
    // the last tries of the budget (fewer than four left)
    bool done = EARLY && t + 3 < climbings;  // early exit taken
    while (!done && t < climbings) {
      int a, b;
      win.pair(lane, a, b);
      const int d = eval((uint32_t)a, (uint32_t)b);
      if (d > 0) {
        accept(a, b, d);
        last = (int)t;
        ++nacc;
      }
      ++t;
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

bool mas_tform_ok(int64_t max_len, int64_t table_max) {
  if (table_max > 32767 || max_len > 32768) return false;
  const int64_t n1 = max_len > 0 ? max_len - 1 : 0;
  return n1 * table_max < (int64_t(1) << 29);
}

cudaError_t launch_mas_climb_tform(cudaStream_t s, const MasLaunch& p, int sm_count) {
  if (p.n_workers <= 0) return cudaSuccess;
  auto kern = (p.flags & CCG_FLAG_EARLY_EXIT) ? mas_climb_tform_kernel<true>
                                              : mas_climb_tform_kernel<false>;
  const int smem = kTWarps * (int)kTWarpBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTWarps * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (p.n_workers + kTWarps - 1) / kTWarps;
  const int64_t resident = (int64_t)per_sm * sm_count;
  const int grid = (int)(need < resident ? need : resident);
  kern<<<grid, kTWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ccg
