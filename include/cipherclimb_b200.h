/*
 * cipherclimb_b200.h -- C ABI of the B200 hill-climbing attack engine.
 *
 * The reference (`cipherclimb`, pure Python + numpy) has no native FFI; its only
 * execution seam is search.py:49-58 `run_worker_pool(task, args_list, jobs)`, which
 * runs a pure per-worker task over a list of argument tuples and returns the results
 * in submission (worker) order.  Each entry point below replaces one whole batch of
 * such tasks (or one reference primitive used as a fitness oracle) with one call:
 *
 *   ccg_philox_uniform / ccg_philox_int_below   rng.py:58-97   WorkerRng.next_uniform / next_int_below
 *   ccg_score_text_batch                         ngrams.py:134-140 score_text
 *   ccg_log_score_text_batch                     ngrams.py:166-172 log_score_text (numpy pairwise order)
 *   ccg_mas_delta_batch                          mas.py:181-210 swap_delta (via mas.py:315 text_swap_delta)
 *   ccg_mas_delta_counts_batch                   mas.py:181-210 swap_delta on given count matrices
 *   ccg_mas_climb[_dev]                          mas.py:247-250 _stochastic_task -> mas.py:218-244
 *                                                stochastic_worker, for a whole run_worker_pool batch
 *                                                (mas.py:266-272) + search.py:19-25 max_element per group
 *   ccg_ngram_score_batch                        ngrams.py:134-140 score_text generalised to order-n windows
 *   ccg_mas_ngram_climb[_dev]                    mas.py:218-244 stochastic_worker generalised to an order-n
 *                                                (n = 2, 3, 4) integer table (BASELINE configs 4-5)
 *   ccg_mas_det_step_batch                       mas.py:84-120 deterministic_step (all 325 pair-worker scores)
 *   ccg_mas_det_solve[_dev]                      mas.py:140-169 solve_deterministic, a batch of
 *                                                (ciphertext, restart) jobs, whole loop on device
 *   ccg_sct_score_batch                          sct.py:158-160 candidate_score (ciphers.py:71-86,107-113)
 *   ccg_ngram_log_score_batch                    ngrams.py:166-172 generalised to order-n windows
 *   ccg_sct_score_ngram_batch                    sct.py:158-160 with an order-n log table
 *   ccg_encrypt_batch                            ciphers.py:46-49,89-104 mas_encrypt / sct_encrypt with keys
 *                                                rng.py:91-97 permutation(k) on KEYGEN streams (test sets)
 *   ccg_sct_climb[_dev]                          sct.py:173-176 _sct_task -> sct.py:148-170 sct_worker,
 *                                                for a whole batch (sct.py:194-200) + max_element
 *   ccg_sct_fast_climb                           sct.py:148-170 sct_worker with an int32-quantised
 *                                                fitness scored incrementally (opt-in fast mode;
 *                                                not bit-exact with the reference by design)
 *
 * Conventions: plain pointers and sizes only.  Letters are uint8 in [0,26).  Ragged
 * text batches are (concatenated letters, int64 offsets[n+1]).  Philox keys are the
 * (k0, k1) words numpy's Philox actually uses for WorkerRng(seed, stream) -- the Python
 * host layer computes them (rng.py:63-64 plus numpy's key conversion).  `skip` is the
 * number of 64-bit draws already consumed from the stream.
 *
 * Error behaviour: every call returns CCG_OK (0) or a negative CCG_ERR_* code and leaves
 * a message in ccg_last_error() (thread-local).  Nothing throws or exits across the ABI.
 * Input validation mirrors the reference's ValueError preconditions where they apply
 * to the data passed here (mas.py:68-72, sct.py:153-154); the Python layer raises the
 * reference's exact ValueError messages before calling.
 *
 * Entry points without the _dev suffix take HOST pointers and are synchronous (inputs
 * are copied to HBM, outputs back, on the context's stream).  _dev entry points take
 * DEVICE pointers (e.g. from ccg_dev_alloc) and are asynchronous on the context stream.
 */
#ifndef CIPHERCLIMB_B200_H
#define CIPHERCLIMB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CCG_ABI_VERSION 1

enum {
  CCG_OK = 0,
  CCG_ERR_INVALID = -1,     /* bad argument (reference would raise ValueError) */
  CCG_ERR_CUDA = -2,        /* CUDA runtime error */
  CCG_ERR_NO_DEVICE = -3,   /* no sm_100 device visible */
  CCG_ERR_UNSUPPORTED = -4  /* valid for the reference, outside this engine's limits */
};

/* flags for ccg_*_climb_args.flags */
#define CCG_FLAG_EARLY_EXIT 1u /* stop a worker once no proposal can ever be accepted again */
/* MAS kernel selection (results are identical; for tests and benchmarks).  0 = automatic:
 * the D-form kernel (maintained delta table) when its integer gate holds, else the T-form,
 * else the packed / wide count-matrix kernels. */
#define CCG_FLAG_KERNEL_MASK 0x70u
#define CCG_FLAG_KERNEL_DFORM 0x10u  /* deltas computed on demand from the maintained N, T */
#define CCG_FLAG_KERNEL_TFORM 0x20u
#define CCG_FLAG_KERNEL_PACKED 0x30u
#define CCG_FLAG_KERNEL_DTABLE 0x40u /* D-form with the full delta table kept in smem */
/* SCT: with few workers (up to 16 per SM) the climb runs each worker on a CTA of warps that
 * evaluate consecutive proposals speculatively -- up to 74 workers on two SMs each, one
 * parsing the worker's proposal chain ahead (identical results, lower latency); this flag
 * forces the one-warp-per-worker kernel instead. */
#define CCG_FLAG_SCT_NO_SPEC 0x100u
/* SCT kernel selection (identical results; for tests and benchmarks).  Automatic: few workers
 * of one text length -> the speculative CTA-per-worker kernel; mixed text lengths or large
 * bigram batches (>= 32768 workers, where one worker per lane fills the GPU) -> one worker per
 * LANE (ccg_sct_lane.cu); otherwise one warp per worker.  CCG_FLAG_SCT_KERNEL_WARP /
 * CCG_FLAG_SCT_KERNEL_LANE force a family; CCG_FLAG_SCT_TABLE_L2 keeps the lane kernel's
 * trigram table in L2 instead of shared memory. */
#define CCG_FLAG_SCT_KERNEL_WARP 0x200u
#define CCG_FLAG_SCT_TABLE_L2 0x400u
#define CCG_FLAG_SCT_KERNEL_LANE 0x800u
/* SCT latency mode: the speculative kernel whose warps replay their predecessors' draws
 * every round, instead of the chain-parsed kernel (identical results; for tests). */
#define CCG_FLAG_SCT_SPEC_REPLAY 0x1000u
/* SCT fast mode: walk every changed window's column instead of reading the regular-grid
 * window-sum tables (identical results; for tests). */
#define CCG_FLAG_SCT_NO_WINDOW_TABLES 0x2000u

typedef struct ccg_ctx ccg_ctx;

int ccg_abi_version(void);
const char *ccg_last_error(void);
int ccg_device_count(int *out);
int ccg_ctx_create(int device, ccg_ctx **out);
int ccg_ctx_destroy(ccg_ctx *ctx);
int ccg_ctx_synchronize(ccg_ctx *ctx);
int ccg_ctx_stream(ccg_ctx *ctx, void **out_cuda_stream);
int ccg_ctx_device(ccg_ctx *ctx, int *out_device);
/* number of kernels this context has launched so far */
int ccg_ctx_launch_count(ccg_ctx *ctx, int64_t *out);
int ccg_ctx_sm_count(ccg_ctx *ctx, int *out);

int ccg_dev_alloc(ccg_ctx *ctx, size_t bytes, void **out);
int ccg_dev_free(ccg_ctx *ctx, void *ptr);
int ccg_host_alloc(size_t bytes, void **out); /* page-locked */
int ccg_host_free(void *ptr);
int ccg_memcpy_h2d(ccg_ctx *ctx, void *dst_dev, const void *src_host, size_t bytes);
int ccg_memcpy_d2h(ccg_ctx *ctx, void *dst_host, const void *src_dev, size_t bytes);

/* rng.py:68-79: `count` draws of stream key (k0,k1) starting after `skip` draws. */
int ccg_philox_uniform(ccg_ctx *ctx, uint64_t k0, uint64_t k1, uint64_t skip, int64_t count,
                       double *out);
int ccg_philox_int_below(ccg_ctx *ctx, uint64_t k0, uint64_t k1, uint64_t skip, uint32_t bound,
                         int64_t count, int64_t *out);

/* ngrams.py:134-140, one score per text. table: int64[676], entries >= 0. */
int ccg_score_text_batch(ccg_ctx *ctx, const uint8_t *texts, const int64_t *offsets,
                         int64_t n_texts, const int64_t *table, int64_t *out);
/* ngrams.py:166-172, bit-exact numpy pairwise order.  logs: float64[676]. */
int ccg_log_score_text_batch(ccg_ctx *ctx, const uint8_t *texts, const int64_t *offsets,
                             int64_t n_texts, const double *logs, double *out);
/* mas.py:181-210 on the count matrix of each text; ab: int32[2*n_texts] letter pairs. */
int ccg_mas_delta_batch(ccg_ctx *ctx, const uint8_t *texts, const int64_t *offsets,
                        int64_t n_texts, const int32_t *ab, const int64_t *table, int64_t *out);
/* mas.py:181-210 swap_delta(counts, a, b, score_matrix) on explicit count matrices:
 * counts int64[n][676] with entries in 0..65535, score_matrix int64[676] (any sign). */
int ccg_mas_delta_counts_batch(ccg_ctx *ctx, const int64_t *counts, int64_t n, const int32_t *ab,
                               const int64_t *score_matrix, int64_t *out);

typedef struct {
  /* inputs */
  const uint8_t *ciphers;     /* concatenated ciphertexts */
  const int64_t *offsets;     /* [n_ciphers + 1] */
  int64_t n_ciphers;
  const int32_t *cipher_of;   /* [n_workers] cipher index of each worker */
  const uint64_t *keys;       /* [2 * n_workers] Philox key (k0, k1) per worker */
  const uint64_t *skips;      /* [n_workers] draws already consumed, or NULL for 0 */
  int64_t n_workers;
  int64_t climbings;          /* tries per worker (mas.py:234) */
  const int64_t *table;       /* [676] BigramTable.scores */
  /* outputs (NULL = not wanted, except scores) */
  int64_t *scores;            /* [n_workers] final score */
  uint8_t *maps;              /* [26 * n_workers] cipher letter -> plaintext letter */
  uint64_t *draws_used;       /* [n_workers] stream position after the worker */
  int64_t *last_accept;       /* [n_workers] index of the last accepted try, -1 if none */
  int64_t *tries_done;        /* [n_workers] tries executed (== climbings unless early exit) */
  int32_t group_size;         /* >0: consecutive workers form groups (one restart each) */
  int64_t *group_best;        /* [n_workers / group_size] first-max worker index per group */
  /* required by ccg_mas_climb_dev only (computed by the host API otherwise) */
  int64_t max_len;            /* longest ciphertext */
  int64_t table_max;          /* max(table) */
  uint32_t flags;             /* CCG_FLAG_* */
  int64_t *accepts;           /* [n_workers] accepted interchanges, or NULL */
} ccg_mas_climb_args;

int ccg_mas_climb(ccg_ctx *ctx, const ccg_mas_climb_args *args);
int ccg_mas_climb_dev(ccg_ctx *ctx, const ccg_mas_climb_args *args);

/* n-gram extension (the reference has bigrams only).  Window index
 * sum_j 26^(order-1-j) t_{s+j}; a text of n letters has max(0, n-order+1) windows. */
/* ngrams.py:134-140 generalised: table int64[26^order], entries >= 0. */
int ccg_ngram_score_batch(ccg_ctx *ctx, const uint8_t *texts, const int64_t *offsets,
                          int64_t n_texts, int32_t order, const int64_t *table, int64_t *out);

typedef struct {
  const uint8_t *ciphers;     /* concatenated ciphertexts (each <= 4096 letters) */
  const int64_t *offsets;     /* [n_ciphers + 1] */
  int64_t n_ciphers;
  const int32_t *cipher_of;   /* [n_workers] */
  const uint64_t *keys;       /* [2 * n_workers] Philox key (k0, k1) per worker */
  const uint64_t *skips;      /* [n_workers] draws already consumed, or NULL */
  int64_t n_workers;
  int64_t climbings;
  int32_t order;              /* 2, 3 or 4 */
  const uint16_t *table;      /* [26^order] integer n-gram scores (e.g. a quantised log table) */
  int64_t *scores;            /* [n_workers] */
  uint8_t *maps;              /* [26 * n_workers] cipher letter -> plaintext letter, or NULL */
  uint64_t *draws_used;
  int64_t *last_accept;
  int64_t *tries_done;
  int32_t group_size;
  int64_t *group_best;
  int64_t max_len;            /* required by the _dev entry point only */
  uint32_t flags;
  int64_t *computed;          /* [n_workers] deltas computed by a position walk (the other tries
                                 read the delta cache of the unchanged state), or NULL */
  int64_t *lookups;           /* [n_workers] n-gram table reads (walks + accepted refreshes), or
                                 NULL -- the roofline's per-eval traffic for L2-resident tables */
} ccg_mas_ngram_args;

int ccg_mas_ngram_climb(ccg_ctx *ctx, const ccg_mas_ngram_args *args);
int ccg_mas_ngram_climb_dev(ccg_ctx *ctx, const ccg_mas_ngram_args *args);

/* mas.py:84-120 deterministic_step for a batch: text i with pivot (pivots[2i], pivots[2i+1])
 * (distinct letters, both present in the text).  Writes the 325 pair-worker candidate scores of
 * every text (out: int64[325 * n_texts], worker order of pairs.py:27-35; crosswise-excluded
 * workers score 0).  The caller applies max_element (search.py:19-25). */
int ccg_mas_det_step_batch(ccg_ctx *ctx, const uint8_t *texts, const int64_t *offsets,
                           int64_t n_texts, const int32_t *pivots, const int64_t *table,
                           int64_t *out);

typedef struct {
  const uint8_t *ciphers;     /* concatenated ciphertexts (each >= 2 distinct letters) */
  const int64_t *offsets;     /* [n_ciphers + 1] */
  int64_t n_ciphers;
  const int32_t *cipher_of;   /* [n_jobs] cipher index of each job */
  const uint64_t *keys;       /* [2 * n_jobs] Philox key of WorkerRng(seed, pivot_stream_index(r)) */
  int64_t n_jobs;
  int64_t iterations;         /* MasSolverConfig.iterations (mas.py:154) */
  const int64_t *table;       /* [676] BigramTable.scores */
  int64_t *scores;            /* [n_jobs] final score */
  uint8_t *maps;              /* [26 * n_jobs] cipher letter -> plaintext letter, or NULL */
  int32_t *hist_iter;         /* [iterations * n_jobs] accepted iteration numbers, or NULL */
  int64_t *hist_score;        /* [iterations * n_jobs] score after each accept, or NULL */
  int32_t *hist_len;          /* [n_jobs] number of accepts, or NULL */
  uint64_t *draws_used;       /* [n_jobs] pivot draws consumed, or NULL */
  int64_t max_len;            /* required by the _dev entry point only */
  int64_t table_max;          /* required by the _dev entry point only */
  int64_t *hist_offsets;      /* [n_jobs + 1] or NULL (host entry point only): when set, the
                                 histories come back packed -- job j's accepts at
                                 hist_iter/hist_score[hist_offsets[j] .. hist_offsets[j+1]) --
                                 so only their entries are written */
} ccg_mas_det_args;

int ccg_mas_det_solve(ccg_ctx *ctx, const ccg_mas_det_args *args);
int ccg_mas_det_solve_dev(ccg_ctx *ctx, const ccg_mas_det_args *args);

/* sct.py:158-160: score of decrypting ciphers[cipher_of[i]] with keys[i*k:(i+1)*k]. */
int ccg_sct_score_batch(ccg_ctx *ctx, const uint8_t *ciphers, const int64_t *offsets,
                        int64_t n_ciphers, const int32_t *cipher_of, const uint8_t *keys,
                        int32_t key_length, int64_t n_keys, const double *logs, double *out);

typedef struct {
  const uint8_t *ciphers;
  const int64_t *offsets;     /* all ciphertexts of one call must have the same length */
  int64_t n_ciphers;
  const int32_t *cipher_of;
  const uint64_t *keys;       /* [2 * n_workers] */
  const uint64_t *skips;
  int64_t n_workers;
  int32_t key_length;         /* SctSolverConfig.key_length (sct.py:47) */
  int64_t climbings;
  int32_t p1, p2, op1_hop, op2_hop;
  const double *logs;         /* [676] LogBigramTable.logs */
  double *scores;
  uint8_t *keys_out;          /* [key_length * n_workers] */
  uint64_t *draws_used;
  int64_t *last_accept;
  int64_t *tries_done;
  int32_t group_size;
  int64_t *group_best;
  int64_t text_len;           /* required by ccg_sct_climb_dev: the common ciphertext length */
  uint32_t flags;
  int32_t order;              /* n-gram order of `logs` ([26^order]): 0 or 2 = bigram (reference),
                                 3 = trigram, 4 = quadgram (extension) */
  const int32_t *key_lengths; /* [n_workers] per-worker key length in 2..key_length (a ragged
                                 batch in one launch), or NULL: every worker uses key_length.
                                 keys_out keeps the stride key_length. */
} ccg_sct_climb_args;

/* n-gram extension of the two scoring entry points above: logs float64[26^order], windows of
 * `order` letters, numpy pairwise order over the n-order+1 window terms. */
int ccg_ngram_log_score_batch(ccg_ctx *ctx, const uint8_t *texts, const int64_t *offsets,
                              int64_t n_texts, int32_t order, const double *logs, double *out);
int ccg_sct_score_ngram_batch(ccg_ctx *ctx, const uint8_t *ciphers, const int64_t *offsets,
                              int64_t n_ciphers, const int32_t *cipher_of, const uint8_t *keys,
                              int32_t key_length, int64_t n_keys, int32_t order, const double *logs,
                              double *out);

int ccg_sct_climb(ccg_ctx *ctx, const ccg_sct_climb_args *args);
int ccg_sct_climb_dev(ccg_ctx *ctx, const ccg_sct_climb_args *args);

/* Opt-in fast SCT mode (north_star "incremental (delta) ... scoring"): sct.py:148-170
 * sct_worker -- same start key, operators, draws and strict-greater acceptance -- with the
 * fitness replaced by the INTEGER sum of a quantised log table over the order-gram windows of
 * the decryption (table[i] = round(logs[i] * 2^shift), Python ngrams.quantize_sct_table).
 * Integer addition is associative, so a candidate is scored by re-reading only the windows
 * that touch a column whose ciphertext segment moved.  Results are bit-exact with the fast
 * mode's own oracle (oracle/cc_oracle.c cco_sct_fast_worker), not with the reference's
 * float64 climb; the Python layer reports the key agreement with the parity mode.
 * Texts may have any mix of lengths; (n - order + 1) * max|table| must stay below 2^31. */
typedef struct {
  const uint8_t *ciphers;
  const int64_t *offsets;
  int64_t n_ciphers;
  const int32_t *cipher_of;
  const uint64_t *keys;       /* [2 * n_workers] */
  const uint64_t *skips;
  int64_t n_workers;
  int32_t key_length;         /* keys_out stride; every worker's key length if key_lengths NULL */
  int64_t climbings;
  int32_t p1, p2, op1_hop, op2_hop;
  int32_t order;              /* 2, 3 or 4 */
  const int32_t *table;       /* [26^order] quantised log table, entries <= 0 */
  int64_t *scores;            /* quantised fitness of each worker's final key */
  uint8_t *keys_out;          /* [key_length * n_workers] */
  uint64_t *draws_used;
  int64_t *last_accept;
  int64_t *tries_done;
  int32_t group_size;
  int64_t *group_best;
  const int32_t *key_lengths; /* [n_workers] or NULL */
  int64_t *lookups;           /* [n_workers] table lookups of the incremental rescoring, or NULL */
  uint32_t flags;
} ccg_sct_fast_args;

int ccg_sct_fast_climb(ccg_ctx *ctx, const ccg_sct_fast_args *args);

/* Device-side test-set generation for a ragged batch of plaintexts:
 * kind 0 = MAS (ciphers.py:46-49 mas_encrypt), 1 = SCT (ciphers.py:89-104 sct_encrypt,
 * irregular grid).  With keygen (2 * n_texts Philox keys of WorkerRng(seed_i, KEYGEN_STREAM))
 * the key of text i is drawn on the device as permutation(k_i) (rng.py:91-97) and written to
 * keys[i * kmax ...]; with keygen NULL the keys are read from `keys`.  k_i = 26 for MAS,
 * key_lengths[i] in 1..min(kmax, 64) for SCT.  out receives the ciphertexts (same offsets). */
int ccg_encrypt_batch(ccg_ctx *ctx, int32_t kind, const uint8_t *texts, const int64_t *offsets,
                      int64_t n_texts, const uint64_t *keygen, const int32_t *key_lengths,
                      int32_t kmax, uint8_t *keys, uint8_t *out);

/* Roofline denominator: measured shared-memory (LDS) bandwidth of this device, bytes/s. */
int ccg_bench_smem_bandwidth(ccg_ctx *ctx, double *out_bytes_per_s);
/* Roofline denominator of L2-resident tables (the quadgram MAS climb): random 16-bit gathers
 * per second from a table of `table_entries` uint16 (26^4 for quadgrams, 914 KB). */
int ccg_bench_l2_gather(ccg_ctx *ctx, int64_t table_entries, double *out_gathers_per_s);

#ifdef __cplusplus
}
#endif
#endif /* CIPHERCLIMB_B200_H */
