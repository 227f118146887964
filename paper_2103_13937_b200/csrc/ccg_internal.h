// ccg_internal.h -- shared between the C-ABI layer (ccg_api.cu) and the kernel files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cipherclimb_b200.h"

namespace ccg {

constexpr int kAlpha = 26;
constexpr int kRow = 32;  // padded row stride of the 26x26 smem tables (one row = 32 banks)

// Largest ciphertext the MAS climb handles: bigram counts are packed as 16-bit halves.
constexpr int64_t kMasMaxLen = 65536;
// SCT limits: key length (lane-distributed key, two positions per lane) and the numpy
// pairwise-sum leaf budget (kSctMaxLeaves * <=128 terms).
constexpr int kSctMaxKey = 64;
constexpr int kSctMaxLeaves = 32;
constexpr int64_t kSctMaxLen = 4096;

struct MasLaunch {
  const uint8_t* ciphers;
  const int64_t* offsets;
  const int32_t* cipher_of;
  const uint64_t* keys;
  const uint64_t* skips;
  int64_t n_workers;
  int64_t climbings;
  const int64_t* table;
  int64_t* scores;
  uint8_t* maps;
  uint64_t* draws_used;
  int64_t* last_accept;
  int64_t* tries_done;
  uint32_t flags;
  int64_t* accepts;
  const void* init;  // D-form: per-ciphertext initial states (dform_init_kernel), or NULL
  unsigned long long* tickets;  // worker ticket counter, zero at launch (or NULL: static stride)
};

// MAS climb with an order-G n-gram table (ccg_mas_ngram.cu).
constexpr int64_t kNgramMaxLen = 4096;
struct MasNgramLaunch {
  const uint8_t* ciphers;
  const int64_t* offsets;
  const int32_t* cipher_of;
  const uint64_t* keys;
  const uint64_t* skips;
  int64_t n_workers;
  int64_t climbings;
  int32_t order;
  const uint16_t* table;
  int64_t max_len;
  int64_t* scores;
  uint8_t* maps;
  uint64_t* draws_used;
  int64_t* last_accept;
  int64_t* tries_done;
  uint32_t flags;
  int64_t* computed;
  unsigned long long* tickets;  // worker ticket counter, zero at launch (or NULL)
  int64_t* lookups;             // table reads per worker (or NULL)
};

// Deterministic best-neighbour MAS (ccg_mas_det.cu): one job = one (ciphertext, restart).
struct MasDetLaunch {
  const uint8_t* ciphers;
  const int64_t* offsets;
  const int32_t* cipher_of;
  const uint64_t* keys;  // PIVOT-stream Philox key per job
  int64_t n_jobs;
  int64_t iterations;
  const int64_t* table;
  int64_t* scores;
  uint8_t* maps;
  int32_t* hist_iter;
  int64_t* hist_score;
  int32_t* hist_len;
  uint64_t* draws_used;
};

// numpy pairwise-sum plan for the (n-1) bigram terms of an n-letter text
// (numpy/_core/src/umath/loops_utils.h.src pairwise_sum): leaves in order, and the
// post-order list of leaf merges (dst += src) that reproduces the recursion.
struct SumPlan {
  int32_t n_terms;
  int32_t n_leaves;
  int32_t seq;                      // 1: n_terms < 8, a single sequential leaf
  int32_t leaf_start[kSctMaxLeaves];
  int32_t leaf_len[kSctMaxLeaves];
  int32_t n_merges;
  int8_t merge_dst[kSctMaxLeaves];
  int8_t merge_src[kSctMaxLeaves];
};

struct SctLaunch {
  const uint8_t* ciphers;
  const int64_t* offsets;
  const int32_t* cipher_of;
  const uint64_t* keys;
  const uint64_t* skips;
  int64_t n_workers;
  int32_t n;  // common text length
  int32_t k;
  int64_t climbings;
  int32_t p1, p2, op1_hop, op2_hop;
  int32_t order;  // n-gram order of the log table (2 = the reference's bigrams)
  const int32_t* key_lengths;  // per-worker key length (<= k), or NULL for k
  const double* logs;
  double* scores;
  uint8_t* keys_out;
  uint64_t* draws_used;
  int64_t* last_accept;
  int64_t* tries_done;
  uint32_t flags;
  unsigned long long* tickets;  // worker ticket counter, zero at launch (or NULL)
};

// SCT climb with one worker per lane (ccg_sct_lane.cu).  mode 0 = parity (float64 log table,
// numpy pairwise order, bit-exact with sct.py:158-160); mode 1 = fast (int32-quantised table,
// incremental rescoring of the windows of moved columns; ccg_sct_fast_climb).
constexpr int kSctLaneWarps = 8;
constexpr int kSctLaneMaxHops = 3;  // op1_hop / op2_hop limit of the lane kernels (= the reference default)
struct SctLaneLaunch {
  int32_t mode;
  const uint8_t* ciphers;
  const int64_t* offsets;  // ragged: any mix of text lengths <= max_len
  const int32_t* cipher_of;
  const uint64_t* keys;
  const uint64_t* skips;
  int64_t n_workers;
  int32_t kmax;     // key length (or the largest per-worker key length); keys_out stride
  int32_t max_len;  // longest ciphertext of the launch
  int64_t climbings;
  int32_t p1, p2, op1_hop, op2_hop;
  int32_t order;
  const int32_t* key_lengths;
  const double* logs;     // mode 0: [26^order] float64
  const int32_t* qtable;  // mode 1: [26^order] int32
  double* scores;         // mode 0
  int64_t* iscores;       // mode 1
  uint8_t* keys_out;
  uint64_t* draws_used;
  int64_t* last_accept;
  int64_t* tries_done;
  int64_t* lookups;       // mode 1: table lookups of the incremental rescoring, per worker
  uint32_t flags;
  unsigned long long* tickets;
  const uint8_t* cidx;    // order 3, optional: per-entry index into <= 256 distinct values
  const void* cvals;      // the distinct values (double for mode 0, int32 for mode 1)
  int32_t n_cvals;
  // mode 1, optional: window-sum tables of regular grids (text length a multiple of k):
  // worker i's table at ftab + f_off[i] (f_off[i] < 0: none), see sct_ftab_kernel
  const int32_t* ftab;
  const int64_t* f_off;
};
// One (ciphertext, key length) whose fast-mode window sums are tabulated (regular grid).
struct SctFPair {
  int32_t cipher, k;
  int64_t off;
};
constexpr int64_t kSctFTabMaxEntries = int64_t(1) << 17;  // order * k^order per table
cudaError_t launch_sct_ftab(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                            const SctFPair* pairs, int64_t n_pairs, const int32_t* qtable,
                            int order, int max_len, int32_t* ftab);

#ifdef __CUDACC__
// Worker scheduling for the persistent climb kernels: a warp's first worker is static
// (warp index), later ones are tickets from a global counter zeroed before the launch, so a
// warp that finishes early takes the next worker and the launch's tail is about one worker
// long.  Outputs are per worker, so the assignment does not change any result.  Without a
// counter the warps stride statically.
struct WorkerTickets {
  unsigned long long* ctr;
  int64_t n_warps;  // warps in the grid: the static first workers are 0 .. n_warps-1
  __device__ __forceinline__ int64_t next(int64_t w, int lane) const {
    if (!ctr) return w + n_warps;
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ctr, 1ULL);
    t = __shfl_sync(0xffffffffu, t, 0);
    return n_warps + (int64_t)t;
  }
};

#endif

void build_sum_plan(int64_t n_terms, SumPlan* plan);

// Launchers (return cudaError_t of the launch).  `grid` <= 0 lets the launcher size it.
cudaError_t launch_philox_uniform(cudaStream_t s, uint64_t k0, uint64_t k1, uint64_t skip,
                                  int64_t count, uint32_t bound, double* out_u, int64_t* out_i);
cudaError_t launch_score_text(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                              int64_t n, const int64_t* table, int64_t* out);
cudaError_t launch_log_score_text(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                                  int64_t n, const double* logs, double* out);
cudaError_t launch_mas_delta(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                             int64_t n, const int32_t* ab, const int64_t* table, bool wide,
                             int64_t* out);
cudaError_t launch_mas_delta_counts(cudaStream_t s, const int64_t* counts, int64_t n,
                                    const int32_t* ab, const int64_t* table, bool wide,
                                    int64_t* out);
cudaError_t launch_mas_climb(cudaStream_t s, const MasLaunch& p, bool wide, int sm_count);
// T-form climb (ccg_mas_tform.cu): the fast path whenever mas_tform_ok(max_len, max(S)).
bool mas_tform_ok(int64_t max_len, int64_t table_max);
cudaError_t launch_mas_climb_tform(cudaStream_t s, const MasLaunch& p, int sm_count);
// D-form climb (ccg_mas_dform.cu): maintained table of all 325 exact swap deltas, 32
// proposals per warp instruction; the fast path whenever mas_dform_ok(max_len, max(S)).
bool mas_dform_ok(int64_t max_len, int64_t table_max);
cudaError_t launch_mas_climb_dform(cudaStream_t s, const MasLaunch& p, int sm_count);
size_t dform_init_bytes(int64_t n_ciphers);
cudaError_t launch_dform_init(cudaStream_t s, const MasLaunch& p, int64_t n_ciphers, void* out,
                              int sm_count);
cudaError_t launch_mas_ngram_climb(cudaStream_t s, const MasNgramLaunch& p, int sm_count);
cudaError_t launch_ngram_score(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                               int64_t n, int order, const int64_t* table, int64_t* out);
cudaError_t launch_mas_det_step(cudaStream_t s, const uint8_t* texts, const int64_t* offsets,
                                int64_t n, const int32_t* pivots, const int64_t* table, bool wide,
                                int64_t* out);
cudaError_t launch_mas_det_solve(cudaStream_t s, const MasDetLaunch& p, bool wide);
// pack each job's hist_len[j] history entries (rows of `iterations`) densely at offsets[j]
cudaError_t launch_compact_history(cudaStream_t s, const int32_t* hist_iter,
                                   const int64_t* hist_score, int64_t iterations,
                                   const int64_t* offsets, int64_t n_jobs, int32_t* out_iter,
                                   int64_t* out_score);
cudaError_t launch_group_best_i64(cudaStream_t s, const int64_t* scores, int64_t n_groups,
                                  int32_t group_size, int64_t* out);
cudaError_t launch_group_best_f64(cudaStream_t s, const double* scores, int64_t n_groups,
                                  int32_t group_size, int64_t* out);
cudaError_t launch_sct_score(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                             const int32_t* cipher_of, const uint8_t* keys, int32_t k,
                             int64_t n_keys, int order, const double* logs, double* out,
                             int32_t n_common, const SumPlan& plan);
cudaError_t launch_sct_score_long(cudaStream_t s, const uint8_t* ciphers, const int64_t* offsets,
                                  const int32_t* cipher_of, const uint8_t* keys, int32_t k,
                                  int64_t n_keys, int order, const double* logs, double* out);
cudaError_t launch_sct_climb(cudaStream_t s, const SctLaunch& p, const SumPlan& plan,
                             int sm_count);

cudaError_t launch_sct_lane(cudaStream_t s, const SctLaneLaunch& p, int sm_count);
size_t sct_lane_smem_bytes(int mode, int kmax, int64_t max_len);

cudaError_t launch_encrypt(cudaStream_t s, int kind, const uint8_t* texts, const int64_t* offsets,
                           int64_t n, const uint64_t* keygen, const int32_t* key_lengths,
                           uint8_t* keys, int kmax, uint8_t* out);

cudaError_t bench_smem_bandwidth(cudaStream_t s, int sm_count, double* bytes_per_s);
cudaError_t bench_l2_gather(cudaStream_t s, int sm_count, int64_t entries, double* gathers_per_s);

}  // namespace ccg
