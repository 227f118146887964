// ccg_mas_det.cu -- the deterministic best-neighbour MAS climb on the GPU
// (reference mas.py:84-169: deterministic_step, climb, _draw_present_letter,
// solve_deterministic; pairs.py:27-35 for the worker <-> letter-pair numbering).
//
// Layout: one CTA per job (a ciphertext x restart), 352 threads; thread t < 325 is the
// reference's pair-worker t = (L, R) (lexicographic, pairs.py).  The whole 500-iteration
// loop stays on the device -- the per-iteration host round trip that the paper names as
// its first bottleneck is gone.
//
// State: the bigram-count matrix T of the CURRENT plaintext (int32, 26x26, shared), the
// score table S and the row/column aggregates R = T S^T, C = T^T S (shared, in the
// accumulator type; rebuilt after every accept).  Worker t's candidate applies the letter
// map m = (pr R) o (pl L) (mas.py:75-81) to the text; its score is the current score plus
// the exact change over the letters D = {pl, L, pr, R} that m moves (candidate_delta: ~100
// table reads from R, C, T, S), which equals the reference's full rescore (mas.py:114-116)
// as an integer.  Crosswise
// workers (R == pl or L == pr) score 0 (mas.py:117); the best is the FIRST maximum
// (search.py:19-25), accepted iff strictly greater (mas.py:161).
//
// Pivot draws (mas.py:133-137, 155-158) come from the PIVOT stream on thread 0 (scalar
// numpy-exact Philox, ccg_rng.cuh); the letters present in the current text are a 26-bit
// mask that is permuted with the text on every accept.
#include "ccg_internal.h"
#include "ccg_rng.cuh"

namespace ccg {
namespace {

constexpr int kDetThreads = 352;  // 11 warps: 325 pair-workers + idle lanes
constexpr int kPairs = 325;

// pair index t -> (L, R), L < R, lexicographic (pairs.py:27-35)
__device__ __forceinline__ void pair_of(int t, int& L, int& R) {
  int l = 0, rem = t;
  while (rem >= kAlpha - 1 - l) {
    rem -= kAlpha - 1 - l;
    ++l;
  }
  L = l;
  R = l + 1 + rem;
}

// m = second o first: first swaps pl<->L, second swaps pr<->R (mas.py:75-81)
struct LetterMap {
  int pl, L, pr, R;
  __device__ __forceinline__ int operator()(int x) const {
    const int y = x == pl ? L : (x == L ? pl : x);
    return y == pr ? R : (y == R ? pr : y);
  }
};

// Exact score change of applying m to the text whose bigram counts are T, from the row and
// column aggregates R[x][y] = sum_q T[x][q] S[y][q], C[x][y] = sum_q T[q][x] S[q][y].  With
// D = {pl, L, pr, R} (the letters m moves; m(u) = u outside D):
//   delta = sum_{u in D} (R[u][mu] - R[u][u]) + sum_{v in D} (C[v][mv] - C[v][v])
//         + sum_{u,v in D} T[u][v] (S[mu][mv] - S[mu][v] - S[u][mv] + S[u][v]),
// i.e. the terms with u or v in D of sum T[u][v] (S[mu][mv] - S[u][v]), where the row and
// column sums over all v (u) count the D x D block twice and with the wrong S entries, and
// the last line repairs that.  |D| <= 4: ~100 table reads instead of ~600.
template <typename Acc>
__device__ Acc candidate_delta(const int* T, const Acc* S, const Acc* R, const Acc* C,
                               const LetterMap& m) {
  int d[4], md[4];
  int nd = 0;
  const int cand[4] = {m.pl, m.L, m.pr, m.R};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bool dup = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) dup |= j < nd && d[j] == cand[i];
    if (!dup) {
      d[nd] = cand[i];
      md[nd] = m(cand[i]);
      ++nd;
    }
  }
  Acc acc = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= nd) break;
    const int u = d[i], mu = md[i];
    acc += R[u * kAlpha + mu] - R[u * kAlpha + u] + C[u * kAlpha + mu] - C[u * kAlpha + u];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= nd) break;
      const int v = d[j], mv = md[j];
      const int t = T[u * kAlpha + v];
      acc += (Acc)t * (S[mu * kAlpha + mv] - S[mu * kAlpha + v] - S[u * kAlpha + mv] +
                       S[u * kAlpha + v]);
    }
  }
  return acc;
}

// R and C of the current T (all threads of the block; caller syncs)
template <typename Acc>
__device__ __forceinline__ void build_rc(const int* T, const Acc* S, Acc* R, Acc* C) {
  for (int e = threadIdx.x; e < kAlpha * kAlpha; e += blockDim.x) {
    const int x = e / kAlpha, y = e - x * kAlpha;
    Acc r = 0, c = 0;
#pragma unroll 2
    for (int q = 0; q < kAlpha; ++q) {
      r += (Acc)T[x * kAlpha + q] * S[y * kAlpha + q];
      c += (Acc)T[q * kAlpha + x] * S[q * kAlpha + y];
    }
    R[e] = r;
    C[e] = c;
  }
}

// (value, index) first-max over the block; every thread gets the result.
template <typename Acc>
__device__ __forceinline__ void block_first_max(Acc v, int idx, Acc* sv, int* si, Acc& out_v,
                                                int& out_i) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Acc ov = __shfl_down_sync(0xffffffffu, v, o);
    const int oi = __shfl_down_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if (lane == 0) {
    sv[warp] = v;
    si[warp] = idx;
  }
  __syncthreads();
  if (warp == 0) {
    v = lane < kDetThreads / 32 ? sv[lane] : (Acc)(-1);
    idx = lane < kDetThreads / 32 ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const Acc ov = __shfl_down_sync(0xffffffffu, v, o);
      const int oi = __shfl_down_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    if (lane == 0) {
      sv[0] = v;
      si[0] = idx;
    }
  }
  __syncthreads();
  out_v = sv[0];
  out_i = si[0];
  __syncthreads();
}

template <typename Acc>
struct DetShared {
  Acc S[kAlpha * kAlpha];
  Acc R[kAlpha * kAlpha];
  Acc C[kAlpha * kAlpha];
  int T[kAlpha * kAlpha];
  Acc red_v[kDetThreads / 32];
  int red_i[kDetThreads / 32];
  uint8_t map[32];
  int pivot[2];
  uint32_t present;
  uint8_t letters[128];  // PIVOT-stream letters int(u*26) of draws wbase .. wbase+127
};

// T = bigram counts of text[0..n), S = table; returns the score (thread-uniform).
template <typename Acc>
__device__ Acc load_state(DetShared<Acc>& sh, const uint8_t* text, int64_t n, const int64_t* table) {
  for (int i = threadIdx.x; i < kAlpha * kAlpha; i += blockDim.x) {
    sh.S[i] = (Acc)table[i];
    sh.T[i] = 0;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i + 1 < n; i += blockDim.x)
    atomicAdd(&sh.T[text[i] * kAlpha + text[i + 1]], 1);
  __syncthreads();
  build_rc(sh.T, sh.S, sh.R, sh.C);
  Acc part = 0;
  for (int i = threadIdx.x; i < kAlpha * kAlpha; i += blockDim.x) part += (Acc)sh.T[i] * sh.S[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) sh.red_v[threadIdx.x >> 5] = part;
  __syncthreads();
  Acc total = 0;
  for (int w = 0; w < kDetThreads / 32; ++w) total += sh.red_v[w];
  __syncthreads();
  return total;
}

// mas.py:84-120 for a batch of (text, pivot): all 325 candidate scores per text.
template <typename Acc>
__global__ void __launch_bounds__(kDetThreads) det_step_kernel(const uint8_t* texts,
                                                               const int64_t* offsets,
                                                               const int32_t* pivots,
                                                               const int64_t* table,
                                                               int64_t* out) {
  __shared__ DetShared<Acc> sh;
  const int64_t j = blockIdx.x;
  const int64_t off = offsets[j], n = offsets[j + 1] - off;
  const Acc score = load_state(sh, texts + off, n, table);
  const int t = threadIdx.x;
  if (t < kPairs) {
    int L, R;
    pair_of(t, L, R);
    const int pl = pivots[2 * j], pr = pivots[2 * j + 1];
    Acc c = 0;
    if (!(R == pl || L == pr)) c = score + candidate_delta(sh.T, sh.S, sh.R, sh.C, LetterMap{pl, L, pr, R});
    out[j * kPairs + t] = (int64_t)c;
  }
}

// mas.py:140-169 solve_deterministic, one job per CTA.
template <typename Acc>
__global__ void __launch_bounds__(kDetThreads, 5) det_solve_kernel(const MasDetLaunch p) {
  __shared__ DetShared<Acc> sh;
  const int64_t job = blockIdx.x;
  const int32_t cid = p.cipher_of[job];
  const int64_t off = p.offsets[cid], n = p.offsets[cid + 1] - off;
  const uint8_t* text = p.ciphers + off;
  Acc score = load_state(sh, text, n, p.table);
  const int t = threadIdx.x;
  if (t < 32) sh.map[t] = (uint8_t)t;
  if (t == 0) {
    uint32_t pres = 0;
    for (int i = 0; i < kAlpha * kAlpha; ++i)
      if (sh.T[i]) pres |= (1u << (i / kAlpha)) | (1u << (i % kAlpha));
    if (n == 1) pres = 1u << text[0];
    sh.present = pres;
  }
  int L = 0, R = 1;
  if (t < kPairs) pair_of(t, L, R);

  // warp 0 draws the pivots (mas.py:133-137 _draw_present_letter, numpy order) from a
  // 128-letter window of the PIVOT stream that it refills one Philox block per lane, and
  // finds each pivot with a ballot over the next 32 draws instead of one draw at a time
  const uint64_t k0 = p.keys[2 * job], k1 = p.keys[2 * job + 1];
  uint64_t drawn = 0;  // draws consumed
  uint64_t wbase = ~0ull;  // stream index of letters[0] (none yet)
  auto refill = [&](uint64_t pos) {  // warp 0: window starting at pos & ~3
    wbase = pos & ~3ull;
    uint64_t v0, v1, v2, v3;
    philox4x64_10(k0, k1, (wbase >> 2) + 1 + (uint64_t)t, v0, v1, v2, v3);
    sh.letters[4 * t] = (uint8_t)int_below_small(v0, kAlpha);
    sh.letters[4 * t + 1] = (uint8_t)int_below_small(v1, kAlpha);
    sh.letters[4 * t + 2] = (uint8_t)int_below_small(v2, kAlpha);
    sh.letters[4 * t + 3] = (uint8_t)int_below_small(v3, kAlpha);
    __syncwarp();
  };
  // the first draw at or after `drawn` whose letter is present (and != skip); consumes
  // the draws up to and including it
  auto next_present = [&](uint32_t pres, int skip) -> int {
    for (;;) {
      if (wbase == ~0ull || drawn < wbase || drawn + 32 > wbase + 128) refill(drawn);
      const int L0 = sh.letters[drawn - wbase + (uint64_t)t];
      const uint32_t ok = __ballot_sync(0xffffffffu, ((pres >> L0) & 1u) && L0 != skip);
      if (ok) {
        const int j = __ffs(ok) - 1;
        drawn += (uint64_t)j + 1;
        return __shfl_sync(0xffffffffu, L0, j);
      }
      drawn += 32;
    }
  };
  int32_t nh = 0;
  __syncthreads();
  for (int64_t it = 1; it <= p.iterations; ++it) {
    if (t < 32) {
      const uint32_t pres = sh.present;
      const int pl = next_present(pres, -1);
      const int pr = next_present(pres, pl);
      if (t == 0) {
        sh.pivot[0] = pl;
        sh.pivot[1] = pr;
      }
    }
    __syncthreads();
    const int pl = sh.pivot[0], pr = sh.pivot[1];
    Acc c = (Acc)(-1);
    if (t < kPairs) {
      c = 0;
      if (!(R == pl || L == pr)) c = score + candidate_delta(sh.T, sh.S, sh.R, sh.C, LetterMap{pl, L, pr, R});
    }
    Acc best;
    int bi;
    block_first_max(c, t, sh.red_v, sh.red_i, best, bi);
    if (best > score) {  // mas.py:160-164: climb(text, best_index, pivot)
      int bL, bR;
      pair_of(bi, bL, bR);
      const LetterMap m{pl, bL, pr, bR};
      int v0 = 0, v1 = 0;
      const int e0 = t, e1 = t + kDetThreads;
      if (e0 < kAlpha * kAlpha) v0 = sh.T[e0];
      if (e1 < kAlpha * kAlpha) v1 = sh.T[e1];
      uint8_t mp = 0;
      if (t < kAlpha) mp = sh.map[t];
      __syncthreads();
      if (e0 < kAlpha * kAlpha) sh.T[m(e0 / kAlpha) * kAlpha + m(e0 % kAlpha)] = v0;
      if (e1 < kAlpha * kAlpha) sh.T[m(e1 / kAlpha) * kAlpha + m(e1 % kAlpha)] = v1;
      if (t < kAlpha) sh.map[t] = (uint8_t)m(mp);
      if (t == 0) {
        uint32_t np = 0;
        for (int y = 0; y < kAlpha; ++y)
          if ((sh.present >> y) & 1u) np |= 1u << m(y);
        sh.present = np;
        if (p.hist_iter) p.hist_iter[job * p.iterations + nh] = (int32_t)it;
        if (p.hist_score) p.hist_score[job * p.iterations + nh] = (int64_t)best;
      }
      score = best;
      ++nh;
      __syncthreads();
      build_rc(sh.T, sh.S, sh.R, sh.C);
      __syncthreads();
    }
  }
  if (t < kAlpha && p.maps) p.maps[job * kAlpha + t] = sh.map[t];
  if (t == 0) {
    p.scores[job] = (int64_t)score;
    if (p.hist_len) p.hist_len[job] = nh;
    if (p.draws_used) p.draws_used[job] = drawn;
  }
}

}  // namespace

cudaError_t launch_mas_det_step(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                                int64_t n, const int32_t* pivots, const int64_t* table, bool wide,
                                int64_t* out) {
  if (n <= 0) return cudaSuccess;
  if (wide)
    det_step_kernel<long long><<<(unsigned)n, kDetThreads, 0, s>>>(texts, offsets, pivots, table, out);
  else
    det_step_kernel<int><<<(unsigned)n, kDetThreads, 0, s>>>(texts, offsets, pivots, table, out);
  return cudaGetLastError();
}

cudaError_t launch_mas_det_solve(cudaStream_t s, const MasDetLaunch& p, bool wide) {
  if (p.n_jobs <= 0) return cudaSuccess;
  if (wide)
    det_solve_kernel<long long><<<(unsigned)p.n_jobs, kDetThreads, 0, s>>>(p);
  else
    det_solve_kernel<int><<<(unsigned)p.n_jobs, kDetThreads, 0, s>>>(p);
  return cudaGetLastError();
}

// One warp per job copies its history prefix into the packed arrays, so the host reads
// sum(hist_len) entries instead of n_jobs x iterations.
__global__ void compact_history_kernel(const int32_t* __restrict__ hist_iter,
                                       const int64_t* __restrict__ hist_score, int64_t iterations,
                                       const int64_t* __restrict__ offsets, int64_t n_jobs,
                                       int32_t* __restrict__ out_iter, int64_t* __restrict__ out_score) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n_jobs) return;
  const int64_t o = offsets[j], len = offsets[j + 1] - o;
  for (int64_t i = lane; i < len; i += 32) {
    out_iter[o + i] = hist_iter[j * iterations + i];
    out_score[o + i] = hist_score[j * iterations + i];
  }
}

cudaError_t launch_compact_history(cudaStream_t s, const int32_t* hist_iter,
                                   const int64_t* hist_score, int64_t iterations,
                                   const int64_t* offsets, int64_t n_jobs, int32_t* out_iter,
                                   int64_t* out_score) {
  if (n_jobs <= 0) return cudaSuccess;
  const int64_t blocks = (n_jobs + 7) / 8;
  compact_history_kernel<<<(unsigned)blocks, 256, 0, s>>>(hist_iter, hist_score, iterations, offsets,
                                                          n_jobs, out_iter, out_score);
  return cudaGetLastError();
}

}  // namespace ccg
