// ccg_mas.cu -- monoalphabetic-substitution (MAS) kernels for sm_100a: the pi-form climb
// (packed 16-bit and wide int64 variants -- the engine's exact fallback for tables past the
// D-form / T-form gates: max(S) > 32767 or very long texts), the fitness-oracle kernels
// (score_text, swap_delta batches), Philox draws and the per-group first-max.
//
// Reference path: mas.py:218-244 stochastic_worker (per try: draw a distinct letter pair,
// exact score delta of interchanging the two letters in the current text via the
// bigram-count matrix, mas.py:181-210, commit iff delta > 0), driven by
// mas.py:253-278 solve_stochastic over W workers with streams (restart<<32)|w.
//
// B200 design ("pi-form", warp per worker, lane per letter):
//  * The climb never rewrites text or counts.  C = bigram counts of the CIPHERTEXT is fixed;
//    the state is the letter map pi (cipher letter -> plaintext letter), lane y holding
//    p_y = pi(y) and inv_y = pi^-1(y).  Swapping plaintext letters a,b is swapping pi at
//    xa = pi^-1(a), xb = pi^-1(b), and the reference's delta becomes, per lane y,
//      A_y = C[xa][y](S[b][p'_y] - S[a][p_y]) + C[xb][y](S[a][p'_y] - S[b][p_y])
//      B_y = [y not in {xa,xb}] (C[y][xa] - C[y][xb])(S[p_y][b] - S[p_y][a])
//    (p' = pi after the swap), summed with one REDUX.  This is the same integer as
//    swap_delta on the current text's counts, so accept decisions are identical.
//  * Both 26x26 tables live in shared memory as 26 rows x 32 banks of packed u32:
//      CC[x][y] = C[x][y] | C[y][x] << 16   (per warp: its worker's ciphertext)
//      SS[a][q] = S[a][q] | S[q][a] << 16   (per block)
//    so each try is 4 conflict-free LDS (row reads; p_y is a permutation, hence distinct
//    banks) + 2 for the two lanes whose letter moves.  The wide variant (S > 65535 or
//    (n-1)*max(S) >= 2^31) keeps S as int64 and reduces in 64 bits.
//  * Draws: a warp refill computes 32 Philox blocks (one per lane) = 128 draws and converts
//    them to letters int(u*26) in parallel; the sequential consumer reads one byte per draw
//    with a shuffle.  The stream is bit-identical to numpy's (ccg_rng.cuh).
//  * Optional exact early exit (CCG_FLAG_EARLY_EXIT): after a run of rejections the warp
//    evaluates all 325 pair deltas; if none is positive no future proposal can be accepted
//    (proposals never depend on the state), so the remaining tries are all rejections and
//    the worker's result is final.
#include "ccg_mas_common.cuh"

namespace ccg {
namespace {

constexpr int kMasWarps = 8;  // warps (workers in flight) per block

__device__ __forceinline__ int lo16(uint32_t v) { return (int)(v & 0xffffu); }
__device__ __forceinline__ int hi16(uint32_t v) { return (int)(v >> 16); }

// Lane y's share of the swap delta (fast variant: packed 16-bit tables, int32 math).
__device__ __forceinline__ int delta_lane_fast(const uint32_t* __restrict__ C,
                                               const uint32_t* __restrict__ SS, int lane, int p,
                                               int xa, int xb, int a, int b) {
  const uint32_t ca = C[xa * kRow + lane], cb = C[xb * kRow + lane];
  const int p2 = lane == xa ? b : (lane == xb ? a : p);
  const uint32_t sa = SS[a * kRow + p], sb = SS[b * kRow + p];
  const uint32_t sa2 = SS[a * kRow + p2], sb2 = SS[b * kRow + p2];
  int v = lo16(ca) * (lo16(sb2) - lo16(sa)) + lo16(cb) * (lo16(sa2) - lo16(sb));
  if (lane != xa && lane != xb) v += (hi16(ca) - hi16(cb)) * (hi16(sb) - hi16(sa));
  return v;
}

// Wide variant: S as int64[26*26], 64-bit accumulation.
__device__ __forceinline__ int64_t delta_lane_wide(const uint32_t* __restrict__ C,
                                                   const int64_t* __restrict__ S, int lane, int p,
                                                   int xa, int xb, int a, int b) {
  const uint32_t ca = C[xa * kRow + lane], cb = C[xb * kRow + lane];
  const int p2 = lane == xa ? b : (lane == xb ? a : p);
  int64_t v = (int64_t)lo16(ca) * (S[b * kAlpha + p2] - S[a * kAlpha + p]) +
              (int64_t)lo16(cb) * (S[a * kAlpha + p2] - S[b * kAlpha + p]);
  if (lane != xa && lane != xb)
    v += (int64_t)(hi16(ca) - hi16(cb)) * (S[p * kAlpha + b] - S[p * kAlpha + a]);
  return v;
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += (int64_t)shfl64((uint64_t)v, (threadIdx.x & 31) ^ o);
  return v;
}

template <bool WIDE>
struct Tables;

template <>
struct Tables<false> {
  uint32_t ss[kAlpha * kRow];
  __device__ void load(const int64_t* __restrict__ t) {
    for (int i = threadIdx.x; i < kAlpha * kRow; i += blockDim.x) {
      const int a = i / kRow, q = i % kRow;
      ss[i] = q < kAlpha ? ((uint32_t)t[a * kAlpha + q] | ((uint32_t)t[q * kAlpha + a] << 16)) : 0u;
    }
  }
  __device__ __forceinline__ int64_t delta(const uint32_t* C, int lane, int p, int xa, int xb,
                                           int a, int b) const {
    return (int64_t)__reduce_add_sync(kFull, delta_lane_fast(C, ss, lane, p, xa, xb, a, b));
  }
  __device__ __forceinline__ int64_t s(int x, int y) const {
    return (int64_t)(ss[x * kRow + y] & 0xffffu);
  }
};

template <>
struct Tables<true> {
  int64_t s64[kAlpha * kAlpha];
  __device__ void load(const int64_t* __restrict__ t) {
    for (int i = threadIdx.x; i < kAlpha * kAlpha; i += blockDim.x) s64[i] = t[i];
  }
  __device__ __forceinline__ int64_t delta(const uint32_t* C, int lane, int p, int xa, int xb,
                                           int a, int b) const {
    return warp_sum_i64(delta_lane_wide(C, s64, lane, p, xa, xb, a, b));
  }
  __device__ __forceinline__ int64_t s(int x, int y) const { return s64[x * kAlpha + y]; }
};

// Build this warp's packed count table CC for text[0..n) (mas.py:172-178 bigram_count_matrix).
__device__ __forceinline__ void build_counts(uint32_t* C, const uint8_t* __restrict__ text,
                                             int64_t n, int lane) {
  for (int i = lane; i < kAlpha * kRow; i += 32) C[i] = 0u;
  __syncwarp();
  for (int64_t i = lane; i + 1 < n; i += 32) {
    const int x = text[i], y = text[i + 1];
    atomicAdd(&C[x * kRow + y], 1u);
    atomicAdd(&C[y * kRow + x], 1u << 16);
  }
  __syncwarp();
}

template <bool WIDE, bool EARLY>
__global__ void __launch_bounds__(kMasWarps * 32, 4)
    mas_climb_kernel(const MasLaunch p) {
  __shared__ Tables<WIDE> tab;
  __shared__ uint32_t counts[kMasWarps][kAlpha * kRow];
  tab.load(p.table);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* C = counts[warp];
  const int64_t stride = (int64_t)gridDim.x * kMasWarps;
  const uint32_t climbings = (uint32_t)p.climbings;

  const WorkerTickets tk{p.tickets, stride};
  for (int64_t w = (int64_t)blockIdx.x * kMasWarps + warp; w < p.n_workers; w = tk.next(w, lane)) {
    const int32_t cid = p.cipher_of[w];
    const int64_t off = p.offsets[cid], n = p.offsets[cid + 1] - off;
    build_counts(C, p.ciphers + off, n, lane);

    // initial score (mas.py:234): sum over bigram types of C[x][y] * S[x][y]
    int64_t part = 0;
    if (lane < kAlpha)
      for (int x = 0; x < kAlpha; ++x) part += (int64_t)(C[x * kRow + lane] & 0xffffu) * tab.s(x, lane);
    int64_t score = warp_sum_i64(part);

    int pv = lane < kAlpha ? lane : 0;  // pi(y)
    int inv = lane;                     // pi^-1(y)
    LetterWindow win;
    win.key = p.keys + 2 * w;
    win.base = p.skips ? p.skips[w] : 0;
    win.o = 0;
    win.refill(lane);

    int last = -1, nacc = 0;
    uint32_t t = 0;
    uint32_t since = 0, next_check = 256;
    // exact local-optimum test over all 325 interchanges (CCG_FLAG_EARLY_EXIT)
    auto improvable = [&]() {
      for (int a2 = 0; a2 < kAlpha - 1; ++a2) {
        const int x1 = __shfl_sync(kFull, inv, a2);
        for (int b2 = a2 + 1; b2 < kAlpha; ++b2) {
          const int x2 = __shfl_sync(kFull, inv, b2);
          if (tab.delta(C, lane, pv, x1, x2, a2, b2) > 0) return true;
        }
      }
      return false;
    };
    bool done = false;
    if constexpr (!WIDE) {
      // Fast path: two proposals per iteration.  Proposals never depend on the state
      // (rng.py:81-89 draws only), so try t+1 is evaluated against the state before try t;
      // if try t is accepted, try t+1 is re-evaluated against the new state.  Decisions
      // are therefore exactly the sequential ones.
      const uint32_t cl = smem_addr(&C[lane]);
      const uint32_t ss0 = smem_addr(&tab.ss[0]);
      uint32_t pofs = ss0 + 4u * (uint32_t)pv;
      auto eval = [&](int a, int b, int xa, int xb) -> int {
        const uint32_t ca = lds_u32(cl + 128u * (uint32_t)xa);
        const uint32_t cb = lds_u32(cl + 128u * (uint32_t)xb);
        const uint32_t sa = lds_u32(pofs + 128u * (uint32_t)a);
        const uint32_t sb = lds_u32(pofs + 128u * (uint32_t)b);
        const bool in_x = lane == xa || lane == xb;
        const int p2 = lane == xa ? b : (lane == xb ? a : pv);
        const uint32_t q2 = ss0 + 4u * (uint32_t)p2;
        const int sa2 = lds_u16(q2 + 128u * (uint32_t)a);
        const int sb2 = lds_u16(q2 + 128u * (uint32_t)b);
        int v = lo16(ca) * (sb2 - lo16(sa)) + lo16(cb) * (sa2 - lo16(sb));
        if (!in_x) v += (hi16(ca) - hi16(cb)) * (hi16(sb) - hi16(sa));
        return __reduce_add_sync(kFull, v);
      };
      auto accept = [&](int a, int b, int xa, int xb, int d) {
        score += d;
        pv = lane == xa ? b : (lane == xb ? a : pv);
        inv = lane == a ? xb : (lane == b ? xa : inv);
        pofs = ss0 + 4u * (uint32_t)pv;
      };
      while (t < climbings && !done) {
        int a1, b1, a2, b2;
        bool two = false;
        if (t + 1 < climbings) {
          if (win.o > 124) win.refill(lane);
          const uint32_t L4 = win.peek4();
          a1 = (int)(L4 & 31u);
          b1 = (int)((L4 >> 5) & 31u);
          a2 = (int)((L4 >> 10) & 31u);
          b2 = (int)((L4 >> 15) & 31u);
          two = a1 != b1 && a2 != b2;
        }
        if (two) {
          win.o += 4;
          const int xa1 = __shfl_sync(kFull, inv, a1), xb1 = __shfl_sync(kFull, inv, b1);
          const int xa2 = __shfl_sync(kFull, inv, a2), xb2 = __shfl_sync(kFull, inv, b2);
          const int d1 = eval(a1, b1, xa1, xb1);
          int d2 = eval(a2, b2, xa2, xb2);
          if (d1 > 0) {
            accept(a1, b1, xa1, xb1, d1);
            last = (int)t;
            ++nacc;
            const int ya = __shfl_sync(kFull, inv, a2), yb = __shfl_sync(kFull, inv, b2);
            d2 = eval(a2, b2, ya, yb);
            if (d2 > 0) {
              accept(a2, b2, ya, yb, d2);
              last = (int)t + 1;
              ++nacc;
            }
          } else if (d2 > 0) {
            accept(a2, b2, xa2, xb2, d2);
            last = (int)t + 1;
            ++nacc;
          }
          t += 2;
          if (EARLY) {
            since = last >= (int)t - 2 ? (uint32_t)((int)t - 1 - last) : since + 2;
            if (last >= (int)t - 2) next_check = 256;
          }
        } else {
          int a, b;
          win.pair(lane, a, b);
          const int xa = __shfl_sync(kFull, inv, a), xb = __shfl_sync(kFull, inv, b);
          const int d = eval(a, b, xa, xb);
          if (d > 0) {
            accept(a, b, xa, xb, d);
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
          if (!improvable()) done = true;
          next_check *= 4;
        }
      }
    } else {
      for (; t < climbings; ++t) {
        int a, b;
        win.pair(lane, a, b);
        const int xa = __shfl_sync(kFull, inv, a);
        const int xb = __shfl_sync(kFull, inv, b);
        const int64_t d = tab.delta(C, lane, pv, xa, xb, a, b);
        if (d > 0) {
          score += d;
          pv = lane == xa ? b : (lane == xb ? a : pv);
          inv = lane == a ? xb : (lane == b ? xa : inv);
          last = (int)t;
          ++nacc;
          since = 0;
          next_check = 256;
        } else if (EARLY && ++since >= next_check) {
          if (!improvable()) {
            ++t;
            break;
          }
          next_check *= 4;
        }
      }
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

// ---------------------------------------------------------------- fitness batches
__global__ void score_text_kernel(const uint8_t* __restrict__ texts,
                                  const int64_t* __restrict__ offsets, int64_t n,
                                  const int64_t* __restrict__ table, int64_t* __restrict__ out) {
  __shared__ int64_t s[kAlpha * kAlpha];
  for (int i = threadIdx.x; i < kAlpha * kAlpha; i += blockDim.x) s[i] = table[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wid >= n) return;
  const uint8_t* t = texts + offsets[wid];
  const int64_t len = offsets[wid + 1] - offsets[wid];
  int64_t acc = 0;
  for (int64_t i = lane; i + 1 < len; i += 32) acc += s[kAlpha * t[i] + t[i + 1]];
  acc = warp_sum_i64(acc);
  if (lane == 0) out[wid] = acc;
}

// swap_delta on each text's own count matrix with pi = identity (xa = a, xb = b).
template <bool WIDE>
__global__ void mas_delta_kernel(const uint8_t* __restrict__ texts,
                                 const int64_t* __restrict__ offsets, int64_t n,
                                 const int32_t* __restrict__ ab, const int64_t* __restrict__ table,
                                 int64_t* __restrict__ out) {
  __shared__ Tables<WIDE> tab;
  __shared__ uint32_t counts[kMasWarps][kAlpha * kRow];
  tab.load(table);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wid = (int64_t)blockIdx.x * kMasWarps + warp;
  if (wid >= n) return;
  uint32_t* C = counts[warp];
  build_counts(C, texts + offsets[wid], offsets[wid + 1] - offsets[wid], lane);
  const int a = ab[2 * wid], b = ab[2 * wid + 1];
  const int pv = lane < kAlpha ? lane : 0;
  const int64_t d = tab.delta(C, lane, pv, a, b, a, b);
  if (lane == 0) out[wid] = d;
}

// swap_delta on explicit count matrices (entries 0..65535) with pi = identity.
template <bool WIDE>
__global__ void mas_delta_counts_kernel(const int64_t* __restrict__ counts, int64_t n,
                                        const int32_t* __restrict__ ab,
                                        const int64_t* __restrict__ table,
                                        int64_t* __restrict__ out) {
  __shared__ Tables<WIDE> tab;
  __shared__ uint32_t cc[kMasWarps][kAlpha * kRow];
  tab.load(table);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wid = (int64_t)blockIdx.x * kMasWarps + warp;
  if (wid >= n) return;
  uint32_t* C = cc[warp];
  const int64_t* m = counts + wid * kAlpha * kAlpha;
  for (int i = lane; i < kAlpha * kRow; i += 32) {
    const int x = i / kRow, y = i % kRow;
    C[i] = y < kAlpha ? ((uint32_t)m[x * kAlpha + y] | ((uint32_t)m[y * kAlpha + x] << 16)) : 0u;
  }
  __syncwarp();
  const int a = ab[2 * wid], b = ab[2 * wid + 1];
  const int pv = lane < kAlpha ? lane : 0;
  const int64_t d = tab.delta(C, lane, pv, a, b, a, b);
  if (lane == 0) out[wid] = d;
}

// search.py:19-25 max_element per group of consecutive workers: first maximum.
template <typename T>
__global__ void group_best_kernel(const T* __restrict__ scores, int64_t n_groups, int32_t gs,
                                  int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= n_groups) return;
  const T* s = scores + g * gs;
  T best = s[0];
  int32_t bi = 0;
  for (int32_t i = lane; i < gs; i += 32) {
    const T v = s[i];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T ov;
    if constexpr (sizeof(T) == 8) {
      uint64_t bits;
      memcpy(&bits, &best, 8);
      bits = shfl64(bits, lane ^ o);
      memcpy(&ov, &bits, 8);
    }
    const int32_t oi = __shfl_xor_sync(kFull, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (lane == 0) out[g] = bi;
}

__global__ void philox_kernel(uint64_t k0, uint64_t k1, uint64_t skip, int64_t count,
                              uint32_t bound, double* __restrict__ out_u,
                              int64_t* __restrict__ out_i) {
  const uint64_t blk = (skip >> 2) + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t v[4];
  philox4x64_10(k0, k1, blk + 1, v[0], v[1], v[2], v[3]);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t g = blk * 4 + j;
    if (g < skip || g >= skip + (uint64_t)count) continue;
    const uint64_t o = g - skip;
    if (out_u) out_u[o] = to_uniform(v[j]);
    if (out_i) out_i[o] = (int64_t)int_below(v[j], bound);
  }
}

}  // namespace

cudaError_t launch_mas_climb(cudaStream_t s, const MasLaunch& p, bool wide, int sm_count) {
  if (p.n_workers <= 0) return cudaSuccess;
  auto kern = wide ? ((p.flags & CCG_FLAG_EARLY_EXIT) ? mas_climb_kernel<true, true>
                                                       : mas_climb_kernel<true, false>)
                   : ((p.flags & CCG_FLAG_EARLY_EXIT) ? mas_climb_kernel<false, true>
                                                       : mas_climb_kernel<false, false>);
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMasWarps * 32, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (p.n_workers + kMasWarps - 1) / kMasWarps;
  const int64_t resident = (int64_t)per_sm * sm_count;
  // persistent grid: at most one full wave of resident blocks, workers strided over warps
  const int grid = (int)(need < resident ? need : resident);
  kern<<<grid, kMasWarps * 32, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_mas_delta(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                             int64_t n, const int32_t* ab, const int64_t* table, bool wide,
                             int64_t* out) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)((n + kMasWarps - 1) / kMasWarps);
  if (wide)
    mas_delta_kernel<true><<<grid, kMasWarps * 32, 0, s>>>(texts, offsets, n, ab, table, out);
  else
    mas_delta_kernel<false><<<grid, kMasWarps * 32, 0, s>>>(texts, offsets, n, ab, table, out);
  return cudaGetLastError();
}

cudaError_t launch_mas_delta_counts(cudaStream_t s, const int64_t* counts, int64_t n,
                                    const int32_t* ab, const int64_t* table, bool wide,
                                    int64_t* out) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)((n + kMasWarps - 1) / kMasWarps);
  if (wide)
    mas_delta_counts_kernel<true><<<grid, kMasWarps * 32, 0, s>>>(counts, n, ab, table, out);
  else
    mas_delta_counts_kernel<false><<<grid, kMasWarps * 32, 0, s>>>(counts, n, ab, table, out);
  return cudaGetLastError();
}

cudaError_t launch_score_text(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                              int64_t n, const int64_t* table, int64_t* out) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)((n * 32 + 255) / 256);
  score_text_kernel<<<grid, 256, 0, s>>>(texts, offsets, n, table, out);
  return cudaGetLastError();
}

cudaError_t launch_group_best_i64(cudaStream_t s, const int64_t* scores, int64_t n_groups,
                                  int32_t group_size, int64_t* out) {
  if (n_groups <= 0) return cudaSuccess;
  const int grid = (int)((n_groups * 32 + 255) / 256);
  group_best_kernel<int64_t><<<grid, 256, 0, s>>>(scores, n_groups, group_size, out);
  return cudaGetLastError();
}

cudaError_t launch_group_best_f64(cudaStream_t s, const double* scores, int64_t n_groups,
                                  int32_t group_size, int64_t* out) {
  if (n_groups <= 0) return cudaSuccess;
  const int grid = (int)((n_groups * 32 + 255) / 256);
  group_best_kernel<double><<<grid, 256, 0, s>>>(scores, n_groups, group_size, out);
  return cudaGetLastError();
}

cudaError_t launch_philox_uniform(cudaStream_t s, uint64_t k0, uint64_t k1, uint64_t skip,
                                  int64_t count, uint32_t bound, double* out_u, int64_t* out_i) {
  if (count <= 0) return cudaSuccess;
  const uint64_t first = skip >> 2, last = (skip + count - 1) >> 2;
  const int64_t blocks = (int64_t)(last - first + 1);
  const int grid = (int)((blocks + 255) / 256);
  philox_kernel<<<grid, 256, 0, s>>>(k0, k1, skip, count, bound, out_u, out_i);
  return cudaGetLastError();
}

}  // namespace ccg
