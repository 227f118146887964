/*
 * cc_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the CUDA engine in paper_2103_13937_b200/csrc.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product path never links or calls it.
 *
 * It restates, in plain C, the algorithms of the reference `cipherclimb` package
 * (/root/reference/pkg/src/cipherclimb), following the reference's own data flow
 * (text-form state with a live bigram-count matrix, full decrypt + numpy-order fp64
 * sum per SCT candidate) rather than the engine's pi-form / warp-parallel design,
 * so that the two are independent implementations.
 *
 * Pinning: tests/test_oracle_golden.py checks every function here against golden
 * vectors produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Cited reference lines:
 *   rng.py:58-97      WorkerRng (numpy Philox4x64-10 keyed [seed, stream]; uniform, int_below,
 *                     distinct_pair, permutation).  numpy's Philox: counter incremented before
 *                     each block, double = (x >> 11) * 2^-53.
 *   rng.py:27-33      worker_stream_index
 *   ngrams.py:134-140 score_text;  ngrams.py:166-172 log_score_text (numpy pairwise sum)
 *   mas.py:172-178    bigram_count_matrix;  mas.py:181-210 swap_delta
 *   mas.py:218-244    stochastic_worker
 *   mas.py:84-120     deterministic_step (325 pair-workers, full rescore, crosswise exclusion)
 *   mas.py:133-169    _draw_present_letter / solve_deterministic (PIVOT stream, strict >)
 *   ciphers.py:71-86  transposition_gather_map;  ciphers.py:107-113 sct_decrypt
 *   sct.py:69-135     select_operator / apply_element_swaps / apply_block_swaps / apply_block_shift
 *   sct.py:148-170    sct_worker
 *                     (+ cco_sct_fast_worker: the same climb on a quantised integer fitness,
 *                      the definition of the opt-in fast mode -- not a reference function)
 *   search.py:19-25   max_element (first maximum)
 *
 * n-gram extension (orders 3 and 4; BASELINE.json configs 3-5).  The reference implements
 * bigrams only (ngrams.py:21), so these functions generalise its semantics to
 * windows of `order` letters: index sum_i 26^(order-1-i) t_i, integer score = sum of table
 * entries over the n-order+1 windows (ngrams.py:134-140), log score = numpy pairwise sum of
 * the window log-probabilities (ngrams.py:166-172), MAS worker = stochastic_worker with
 * the exact score change computed by FULL RESCORE of the swapped text, SCT worker =
 * sct_worker with the order-n candidate score.  At order 2 each reduces to the reference
 * function and is pinned by the reference's golden vectors (tests/test_oracle_golden.py);
 * orders 3/4 have no reference outputs ("parity unpinned" beyond that reduction).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ALPHA 26

/* ------------------------------------------------------------------ philox */
typedef struct {
    uint64_t k0, k1;
    uint64_t ctr;        /* blocks generated so far (low 64 bits of the 256-bit counter) */
    uint64_t buf[4];
    int pos;             /* next word in buf; 4 = empty */
} orng;

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
    unsigned __int128 p = (unsigned __int128)a * b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

/* One Philox4x64-10 block for counter value (c0,0,0,0). */
void cco_philox_block(uint64_t k0, uint64_t k1, uint64_t c0, uint64_t out[4]) {
    uint64_t c[4] = {c0, 0, 0, 0};
    for (int r = 0; r < 10; r++) {
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ULL, c[0], &hi0, &lo0);
        mulhilo64(0xCA5A826395121157ULL, c[2], &hi1, &lo1);
        uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
    memcpy(out, c, sizeof c);
}

static void orng_init(orng *g, uint64_t seed, uint64_t stream) {
    g->k0 = seed; g->k1 = stream; g->ctr = 0; g->pos = 4;
}

static inline uint64_t orng_next_u64(orng *g) {
    if (g->pos >= 4) {
        g->ctr++;  /* numpy increments the counter before generating a block */
        cco_philox_block(g->k0, g->k1, g->ctr, g->buf);
        g->pos = 0;
    }
    return g->buf[g->pos++];
}

static inline double orng_uniform(orng *g) {
    return (double)(orng_next_u64(g) >> 11) * (1.0 / 9007199254740992.0);
}

/* rng.py:43-47 -- int(u * bound): an IEEE double multiply then truncation. */
static inline int64_t orng_int_below(orng *g, int64_t bound) {
    return (int64_t)(orng_uniform(g) * (double)bound);
}

static inline void orng_distinct_pair(orng *g, int64_t bound, int64_t *a, int64_t *b) {
    *a = orng_int_below(g, bound);
    *b = orng_int_below(g, bound);
    while (*b == *a) *b = orng_int_below(g, bound);
}

static void orng_permutation(orng *g, int64_t n, int64_t *perm) {
    for (int64_t i = 0; i < n; i++) perm[i] = i;
    for (int64_t i = n - 1; i > 0; i--) {
        int64_t j = orng_int_below(g, i + 1);
        int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
}

/* Exported stream helpers (draw sequences for golden checks). */
void cco_uniform(uint64_t seed, uint64_t stream, int64_t skip, int64_t n, double *out) {
    orng g; orng_init(&g, seed, stream);
    for (int64_t i = 0; i < skip; i++) orng_next_u64(&g);
    for (int64_t i = 0; i < n; i++) out[i] = orng_uniform(&g);
}

void cco_int_below(uint64_t seed, uint64_t stream, int64_t bound, int64_t n, int64_t *out) {
    orng g; orng_init(&g, seed, stream);
    for (int64_t i = 0; i < n; i++) out[i] = orng_int_below(&g, bound);
}

void cco_distinct_pairs(uint64_t seed, uint64_t stream, int64_t bound, int64_t n, int64_t *out) {
    orng g; orng_init(&g, seed, stream);
    for (int64_t i = 0; i < n; i++) orng_distinct_pair(&g, bound, &out[2 * i], &out[2 * i + 1]);
}

void cco_permutation(uint64_t seed, uint64_t stream, int64_t n, int64_t *out) {
    orng g; orng_init(&g, seed, stream);
    orng_permutation(&g, n, out);
}

/* ------------------------------------------------------------------ scoring */
int64_t cco_score_text(const int64_t *t, int64_t n, const int64_t *table) {
    int64_t s = 0;
    for (int64_t i = 0; i + 1 < n; i++) s += table[ALPHA * t[i] + t[i + 1]];
    return s;
}

/* numpy's float64 add.reduce on a contiguous array (pairwise summation,
 * numpy/_core/src/umath/loops_utils.h.src pairwise_sum): the reference's
 * `logs[idx].sum()` at ngrams.py:172 and sct.py:160. */
double cco_pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return cco_pairwise_sum(a, n2) + cco_pairwise_sum(a + n2, n - n2);
    }
}

double cco_log_score_text(const int64_t *t, int64_t n, const double *logs, double *scratch) {
    if (n < 2) return 0.0;
    for (int64_t i = 0; i + 1 < n; i++) scratch[i] = logs[ALPHA * t[i] + t[i + 1]];
    return cco_pairwise_sum(scratch, n - 1);
}

/* ------------------------------------------------------------------ n-gram generalisation */
static inline int64_t ngram_index(const int64_t *t, int order) {
    int64_t idx = 0;
    for (int j = 0; j < order; j++) idx = idx * ALPHA + t[j];
    return idx;
}

int64_t cco_ngram_score_text(const int64_t *t, int64_t n, int order, const int64_t *table) {
    int64_t s = 0;
    for (int64_t i = 0; i + order <= n; i++) s += table[ngram_index(t + i, order)];
    return s;
}

double cco_ngram_log_score_text(const int64_t *t, int64_t n, int order, const double *logs,
                                double *scratch) {
    if (n < order) return 0.0;
    for (int64_t i = 0; i + order <= n; i++) scratch[i] = logs[ngram_index(t + i, order)];
    return cco_pairwise_sum(scratch, n - order + 1);
}

/* stochastic_worker (mas.py:218-244) with an order-n integer table: per try a distinct
 * letter pair, the exact score change of interchanging the two letters in the current text
 * (here: full rescore of the swapped text minus the current score), commit iff > 0. */
int64_t cco_ngram_worker(const int64_t *cipher, int64_t n, int order, const int64_t *S,
                         int64_t climbings, uint64_t seed, uint64_t stream, int64_t skip,
                         int64_t *out_text, int64_t *out_map, int64_t *out_last_accept) {
    orng g; orng_init(&g, seed, stream);
    for (int64_t i = 0; i < skip; i++) orng_next_u64(&g);
    int64_t *text = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t *cand = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    memcpy(text, cipher, sizeof(int64_t) * n);
    int64_t mapping[ALPHA];
    for (int i = 0; i < ALPHA; i++) mapping[i] = i;
    int64_t score = cco_ngram_score_text(text, n, order, S), last = -1;
    for (int64_t t = 0; t < climbings; t++) {
        int64_t a, b;
        orng_distinct_pair(&g, ALPHA, &a, &b);
        for (int64_t i = 0; i < n; i++) cand[i] = text[i] == a ? b : (text[i] == b ? a : text[i]);
        int64_t delta = cco_ngram_score_text(cand, n, order, S) - score;
        if (delta > 0) {
            score += delta;
            memcpy(text, cand, sizeof(int64_t) * n);
            for (int x = 0; x < ALPHA; x++) {
                if (mapping[x] == a) mapping[x] = b;
                else if (mapping[x] == b) mapping[x] = a;
            }
            last = t;
        }
    }
    if (out_text) memcpy(out_text, text, sizeof(int64_t) * n);
    if (out_map) for (int i = 0; i < ALPHA; i++) out_map[i] = mapping[i];
    if (out_last_accept) *out_last_accept = last;
    free(text); free(cand);
    return score;
}

/* ------------------------------------------------------------------ MAS */
/* mas.py:181-210: exact score change of interchanging letters a, b given the
 * current count matrix (row = first letter). */
int64_t cco_swap_delta(const int64_t *counts, int64_t a, int64_t b, const int64_t *S) {
#define C_(x, y) counts[(x) * ALPHA + (y)]
#define S_(x, y) S[(x) * ALPHA + (y)]
    int64_t d = 0;
    for (int y = 0; y < ALPHA; y++) {
        int64_t ys = (y == a) ? b : (y == b) ? a : y;  /* row_a = S[b] with entries a,b swapped */
        d += C_(a, y) * (S_(b, ys) - S_(a, y));        /* counts[a] @ (row_a - S[a]) */
        d += C_(b, y) * (S_(a, ys) - S_(b, y));        /* counts[b] @ (row_b - S[b]) */
        d += C_(y, a) * (S_(ys, b) - S_(y, a));        /* counts[:,a] @ (col_a - S[:,a]) */
        d += C_(y, b) * (S_(ys, a) - S_(y, b));        /* counts[:,b] @ (col_b - S[:,b]) */
    }
    int64_t corner = C_(a, a) * (S_(b, b) - S_(a, a)) + C_(a, b) * (S_(b, a) - S_(a, b)) +
                     C_(b, a) * (S_(a, b) - S_(b, a)) + C_(b, b) * (S_(a, a) - S_(b, b));
    return d - corner;
#undef C_
#undef S_
}

void cco_count_matrix(const int64_t *t, int64_t n, int64_t *counts) {
    memset(counts, 0, sizeof(int64_t) * ALPHA * ALPHA);
    for (int64_t i = 0; i + 1 < n; i++) counts[t[i] * ALPHA + t[i + 1]]++;
}

/* mas.py:218-244.  Starts from the ciphertext itself (identity mapping); per try
 * draws a distinct letter pair, commits the interchange iff delta > 0.
 * Writes the final text into out_text (length n) and the plaintext-letter image
 * of each cipher letter into out_map (26); returns the score.
 * skip = draws already consumed from the stream before the worker started. */
int64_t cco_stochastic_worker(const int64_t *cipher, int64_t n, const int64_t *S, int64_t climbings,
                              uint64_t seed, uint64_t stream, int64_t skip,
                              int64_t *out_text, int64_t *out_map, int64_t *out_last_accept) {
    orng g; orng_init(&g, seed, stream);
    for (int64_t i = 0; i < skip; i++) orng_next_u64(&g);
    int64_t counts[ALPHA * ALPHA];
    cco_count_matrix(cipher, n, counts);
    int64_t mapping[ALPHA];
    for (int i = 0; i < ALPHA; i++) mapping[i] = i;
    int64_t score = 0;
    for (int i = 0; i < ALPHA * ALPHA; i++) score += counts[i] * S[i];
    int64_t last = -1;
    for (int64_t t = 0; t < climbings; t++) {
        int64_t a, b;
        orng_distinct_pair(&g, ALPHA, &a, &b);
        int64_t delta = cco_swap_delta(counts, a, b, S);
        if (delta > 0) {
            score += delta;
            for (int y = 0; y < ALPHA; y++) {  /* swap rows a,b then columns a,b */
                int64_t tmp = counts[a * ALPHA + y];
                counts[a * ALPHA + y] = counts[b * ALPHA + y];
                counts[b * ALPHA + y] = tmp;
            }
            for (int y = 0; y < ALPHA; y++) {
                int64_t tmp = counts[y * ALPHA + a];
                counts[y * ALPHA + a] = counts[y * ALPHA + b];
                counts[y * ALPHA + b] = tmp;
            }
            for (int x = 0; x < ALPHA; x++) {  /* compose: mapping = swap[mapping] */
                if (mapping[x] == a) mapping[x] = b;
                else if (mapping[x] == b) mapping[x] = a;
            }
            last = t;
        }
    }
    if (out_text) for (int64_t i = 0; i < n; i++) out_text[i] = mapping[cipher[i]];
    if (out_map) for (int i = 0; i < ALPHA; i++) out_map[i] = mapping[i];
    if (out_last_accept) *out_last_accept = last;
    return score;
}

/* ------------------------------------------------------------------ MAS deterministic */
/* mas.py:84-120 deterministic_step: worker t = pair (L, R) (pairs.py:27-35, lexicographic)
 * interchanges pivot pl with L, then pr with R (mas.py:75-81 _interchange_maps), and fully
 * rescores the candidate text; crosswise-colliding workers (R == pl or L == pr) score 0.
 * Writes all 325 scores; returns the first-max index (search.py:19-25). */
int64_t cco_det_step(const int64_t *text, int64_t n, int64_t pl, int64_t pr, const int64_t *S,
                     int64_t *scores, int64_t *cand) {
    int64_t t = 0, best = 0;
    for (int64_t L = 0; L < ALPHA; L++)
        for (int64_t R = L + 1; R < ALPHA; R++, t++) {
            if (R == pl || L == pr) { scores[t] = 0; }
            else {
                int64_t first[ALPHA], second[ALPHA], m[ALPHA];
                for (int x = 0; x < ALPHA; x++) first[x] = second[x] = x;
                first[pl] = L; first[L] = pl;
                second[pr] = R; second[R] = pr;
                for (int x = 0; x < ALPHA; x++) m[x] = second[first[x]];
                int64_t s = 0;
                for (int64_t i = 0; i + 1 < n; i++) s += S[ALPHA * m[text[i]] + m[text[i + 1]]];
                scores[t] = s;
            }
            if (scores[t] > scores[best]) best = t;
        }
    if (cand) {
        int64_t L = 0, R = 1, u = 0;
        for (int64_t a = 0; a < ALPHA; a++)
            for (int64_t b = a + 1; b < ALPHA; b++, u++)
                if (u == best) { L = a; R = b; }
        int64_t first[ALPHA], second[ALPHA];
        for (int x = 0; x < ALPHA; x++) first[x] = second[x] = x;
        first[pl] = L; first[L] = pl;
        second[pr] = R; second[R] = pr;
        for (int64_t i = 0; i < n; i++) cand[i] = second[first[text[i]]];
    }
    return best;
}

/* mas.py:133-137 */
static int64_t draw_present(orng *g, const int *present, int64_t exclude) {
    int64_t letter = orng_int_below(g, ALPHA);
    while (!present[letter] || letter == exclude) letter = orng_int_below(g, ALPHA);
    return letter;
}

/* mas.py:140-169 solve_deterministic on the PIVOT stream key (k0, k1).  Writes the final
 * text, the history as (iteration, score) pairs (at most `iterations`), returns the score;
 * *n_hist = number of accepted iterations. */
int64_t cco_solve_deterministic(const int64_t *cipher, int64_t n, const int64_t *S,
                                int64_t iterations, uint64_t k0, uint64_t k1,
                                int64_t *out_text, int64_t *hist, int64_t *n_hist) {
    orng g; orng_init(&g, k0, k1);
    int64_t *text = out_text;
    for (int64_t i = 0; i < n; i++) text[i] = cipher[i];
    int64_t *cand = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t scores[325];
    int64_t score = cco_score_text(text, n, S), nh = 0;
    for (int64_t it = 1; it <= iterations; it++) {
        int present[ALPHA] = {0};
        for (int64_t i = 0; i < n; i++) present[text[i]] = 1;
        int64_t pl = draw_present(&g, present, -1);
        int64_t pr = draw_present(&g, present, pl);
        int64_t best = cco_det_step(text, n, pl, pr, S, scores, cand);
        if (scores[best] > score) {
            memcpy(text, cand, sizeof(int64_t) * n);
            score = scores[best];
            hist[2 * nh] = it; hist[2 * nh + 1] = score; nh++;
        }
    }
    free(cand);
    *n_hist = nh;
    return score;
}

/* ------------------------------------------------------------------ SCT */
/* ciphers.py:71-86: for each ciphertext position, the plaintext position it came from. */
void cco_gather_map(const int64_t *key, int64_t k, int64_t n, int64_t *m) {
    int64_t base = n / k, rem = n % k, pos = 0;
    for (int64_t j = 0; j < k; j++) {
        int64_t col = key[j];
        int64_t len = base + (col < rem ? 1 : 0);
        for (int64_t r = 0; r < len; r++) m[pos++] = col + k * r;
    }
}

void cco_sct_decrypt(const int64_t *cipher, int64_t n, const int64_t *key, int64_t k,
                     int64_t *plain, int64_t *scratch_map) {
    cco_gather_map(key, k, n, scratch_map);
    for (int64_t i = 0; i < n; i++) plain[scratch_map[i]] = cipher[i];
}

typedef struct {
    int64_t k, climbings, p1, p2, op1_hop, op2_hop, order;
} sct_cfg;

/* sct.py:82-89 */
static void op_element_swaps(int64_t *key, int64_t k, orng *g, int64_t max_hops) {
    int64_t hops = 1 + orng_int_below(g, max_hops);
    for (int64_t h = 0; h < hops; h++) {
        int64_t i, j;
        orng_distinct_pair(g, k, &i, &j);
        int64_t t = key[i]; key[i] = key[j]; key[j] = t;
    }
}

/* sct.py:92-112 */
static void op_block_swaps(int64_t *key, int64_t k, orng *g, int64_t max_hops) {
    int64_t hops = 1 + orng_int_below(g, max_hops);
    for (int64_t h = 0; h < hops; h++) {
        int64_t len = 1 + orng_int_below(g, k / 2);
        int64_t p, q;
        orng_distinct_pair(g, k - len + 1, &p, &q);
        while (llabs(p - q) < len) orng_distinct_pair(g, k - len + 1, &p, &q);
        if (p > q) { int64_t t = p; p = q; q = t; }
        for (int64_t i = 0; i < len; i++) {
            int64_t t = key[p + i]; key[p + i] = key[q + i]; key[q + i] = t;
        }
    }
}

/* sct.py:115-135 */
static void op_block_shift(int64_t *key, int64_t k, orng *g) {
    int64_t len = 1 + orng_int_below(g, k - 1);
    int64_t starts = k - len + 1;
    int64_t p = orng_int_below(g, starts);
    int64_t dest = orng_int_below(g, starts);
    while (dest == p) dest = orng_int_below(g, starts);
    int64_t lo = p < dest ? p : dest, hi = (p > dest ? p : dest) + len;
    int64_t w = hi - lo;
    int64_t win[256];
    memcpy(win, key + lo, sizeof(int64_t) * w);
    if (dest > p) {  /* window[len:] + window[:len] */
        for (int64_t i = 0; i < w - len; i++) key[lo + i] = win[len + i];
        for (int64_t i = 0; i < len; i++) key[lo + w - len + i] = win[i];
    } else {         /* window[-len:] + window[:-len] */
        for (int64_t i = 0; i < len; i++) key[lo + i] = win[w - len + i];
        for (int64_t i = 0; i < w - len; i++) key[lo + len + i] = win[i];
    }
}

/* Exported: apply one operator draw sequence to a key (for operator golden checks).
 * op: 1 element swap, 2 block swap, 3 block shift.  Applies `reps` times in
 * sequence on one stream, each time starting from the ORIGINAL key, writing all results. */
void cco_apply_operator(int op, const int64_t *key, int64_t k, int64_t max_hops,
                        uint64_t seed, uint64_t stream, int64_t reps, int64_t *out) {
    orng g; orng_init(&g, seed, stream);
    for (int64_t r = 0; r < reps; r++) {
        int64_t *o = out + r * k;
        memcpy(o, key, sizeof(int64_t) * k);
        if (op == 1) op_element_swaps(o, k, &g, max_hops);
        else if (op == 2) op_block_swaps(o, k, &g, max_hops);
        else op_block_shift(o, k, &g);
    }
}

static double sct_candidate_score(const int64_t *cipher, int64_t n, const int64_t *key, int64_t k,
                                  const double *logs, int order, int64_t *plain, int64_t *map,
                                  double *terms) {
    cco_sct_decrypt(cipher, n, key, k, plain, map);
    return cco_ngram_log_score_text(plain, n, order, logs, terms);
}

/* sct.py:148-170.  Returns the final score; writes the final key. */
double cco_sct_worker(const int64_t *cipher, int64_t n, const double *logs, const int64_t *cfgv,
                      uint64_t seed, uint64_t stream, int64_t skip, int64_t *out_key,
                      int64_t *out_last_accept) {
    sct_cfg cfg = {cfgv[0], cfgv[1], cfgv[2], cfgv[3], cfgv[4], cfgv[5], cfgv[6]};
    int64_t k = cfg.k;
    orng g; orng_init(&g, seed, stream);
    for (int64_t i = 0; i < skip; i++) orng_next_u64(&g);
    int64_t *plain = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *map = (int64_t *)malloc(sizeof(int64_t) * n);
    double *terms = (double *)malloc(sizeof(double) * (n > 1 ? n : 1));
    int64_t key[256], cand[256];
    orng_permutation(&g, k, key);
    double score = sct_candidate_score(cipher, n, key, k, logs, (int)cfg.order, plain, map, terms);
    int64_t last = -1;
    for (int64_t t = 0; t < cfg.climbings; t++) {
        int64_t u = orng_int_below(&g, 100);
        memcpy(cand, key, sizeof(int64_t) * k);
        if (u < cfg.p1) op_element_swaps(cand, k, &g, cfg.op1_hop);
        else if (u < cfg.p2) op_block_swaps(cand, k, &g, cfg.op2_hop);
        else op_block_shift(cand, k, &g);
        double cs = sct_candidate_score(cipher, n, cand, k, logs, (int)cfg.order, plain, map, terms);
        if (cs > score) {
            memcpy(key, cand, sizeof(int64_t) * k);
            score = cs;
            last = t;
        }
    }
    memcpy(out_key, key, sizeof(int64_t) * k);
    if (out_last_accept) *out_last_accept = last;
    free(plain); free(map); free(terms);
    return score;
}

/* The opt-in fast SCT mode (ccg_sct_fast_climb): sct.py:148-170 with the candidate score
 * replaced by the INTEGER sum of a quantised table over the order-gram windows of the full
 * decryption (q[i] = round(logs[i] * 2^shift), ngrams.quantize_sct_table).  Same stream,
 * start key, operators and strict acceptance as cco_sct_worker; the score is recomputed from
 * scratch for every candidate -- the definition the GPU's incremental rescoring must match. */
int64_t cco_sct_fast_worker(const int64_t *cipher, int64_t n, const int64_t *q, const int64_t *cfgv,
                            uint64_t seed, uint64_t stream, int64_t skip, int64_t *out_key,
                            int64_t *out_last_accept) {
    sct_cfg cfg = {cfgv[0], cfgv[1], cfgv[2], cfgv[3], cfgv[4], cfgv[5], cfgv[6]};
    int64_t k = cfg.k;
    int order = (int)cfg.order;
    orng g; orng_init(&g, seed, stream);
    for (int64_t i = 0; i < skip; i++) orng_next_u64(&g);
    int64_t *plain = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *map = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t key[256], cand[256];
    orng_permutation(&g, k, key);
    cco_sct_decrypt(cipher, n, key, k, plain, map);
    int64_t score = cco_ngram_score_text(plain, n, order, q);
    int64_t last = -1;
    for (int64_t t = 0; t < cfg.climbings; t++) {
        int64_t u = orng_int_below(&g, 100);
        memcpy(cand, key, sizeof(int64_t) * k);
        if (u < cfg.p1) op_element_swaps(cand, k, &g, cfg.op1_hop);
        else if (u < cfg.p2) op_block_swaps(cand, k, &g, cfg.op2_hop);
        else op_block_shift(cand, k, &g);
        cco_sct_decrypt(cipher, n, cand, k, plain, map);
        int64_t cs = cco_ngram_score_text(plain, n, order, q);
        if (cs > score) {
            memcpy(key, cand, sizeof(int64_t) * k);
            score = cs;
            last = t;
        }
    }
    memcpy(out_key, key, sizeof(int64_t) * k);
    if (out_last_accept) *out_last_accept = last;
    free(plain); free(map);
    return score;
}

double cco_sct_score(const int64_t *cipher, int64_t n, const double *logs, const int64_t *key,
                     int64_t k, int order) {
    int64_t *plain = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *map = (int64_t *)malloc(sizeof(int64_t) * n);
    double *terms = (double *)malloc(sizeof(double) * (n > 1 ? n : 1));
    double s = sct_candidate_score(cipher, n, key, k, logs, order, plain, map, terms);
    free(plain); free(map); free(terms);
    return s;
}

/* ------------------------------------------------------------------ batched drivers
 * Many independent workers over a ragged cipher batch, spread over host threads
 * (pthreads, dynamic work claiming).  Used as the CPU baseline (bench.py) and for
 * large parity sweeps. */
#include <pthread.h>

typedef struct {
    int kind;  /* 0 = MAS, 1 = SCT, 2 = MAS order-n, 3 = SCT fast (quantised) */
    int order;
    const int64_t *ciphers, *offsets;
    const int32_t *cipher_of;
    const uint64_t *seeds, *streams;
    int64_t n_workers;
    const int64_t *S; const double *logs; const int64_t *cfgv;
    int64_t climbings;
    int64_t *out_iscores; double *out_fscores; int64_t *out_keys;
    int64_t next;
    pthread_mutex_t mu;
} batch_job;

static void *batch_thread(void *arg) {
    batch_job *J = (batch_job *)arg;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= J->n_workers) break;
        int32_t c = J->cipher_of[w];
        const int64_t *txt = J->ciphers + J->offsets[c];
        int64_t n = J->offsets[c + 1] - J->offsets[c];
        if (J->kind == 2) {
            J->out_iscores[w] = cco_ngram_worker(txt, n, J->order, J->S, J->climbings, J->seeds[w],
                                                 J->streams[w], 0, NULL,
                                                 J->out_keys ? J->out_keys + 26 * w : NULL, NULL);
        } else if (J->kind == 0) {
            J->out_iscores[w] = cco_stochastic_worker(txt, n, J->S, J->climbings, J->seeds[w],
                                                      J->streams[w], 0, NULL,
                                                      J->out_keys ? J->out_keys + 26 * w : NULL,
                                                      NULL);
        } else if (J->kind == 3) {
            int64_t k = J->cfgv[0];
            J->out_iscores[w] = cco_sct_fast_worker(txt, n, J->S, J->cfgv, J->seeds[w],
                                                    J->streams[w], 0, J->out_keys + k * w, NULL);
        } else {
            int64_t k = J->cfgv[0];
            J->out_fscores[w] = cco_sct_worker(txt, n, J->logs, J->cfgv, J->seeds[w], J->streams[w],
                                               0, J->out_keys + k * w, NULL);
        }
    }
    return NULL;
}

static void run_batch(batch_job *J, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 512) nthreads = 512;
    pthread_t th[512];
    J->next = 0;
    pthread_mutex_init(&J->mu, NULL);
    for (int i = 0; i < nthreads; i++) pthread_create(&th[i], NULL, batch_thread, J);
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&J->mu);
}

void cco_mas_workers(const int64_t *ciphers, const int64_t *offsets, const int32_t *cipher_of,
                     const uint64_t *seeds, const uint64_t *streams, int64_t n_workers,
                     const int64_t *S, int64_t climbings, int64_t *out_scores, int64_t *out_maps,
                     int nthreads) {
    batch_job J;
    memset(&J, 0, sizeof J);
    J.kind = 0; J.ciphers = ciphers; J.offsets = offsets; J.cipher_of = cipher_of;
    J.seeds = seeds; J.streams = streams; J.n_workers = n_workers; J.S = S;
    J.climbings = climbings; J.out_iscores = out_scores; J.out_keys = out_maps;
    run_batch(&J, nthreads);
}

void cco_sct_workers(const int64_t *ciphers, const int64_t *offsets, const int32_t *cipher_of,
                     const uint64_t *seeds, const uint64_t *streams, int64_t n_workers,
                     const double *logs, const int64_t *cfgv, double *out_scores, int64_t *out_keys,
                     int nthreads) {
    batch_job J;
    memset(&J, 0, sizeof J);
    J.kind = 1; J.ciphers = ciphers; J.offsets = offsets; J.cipher_of = cipher_of;
    J.seeds = seeds; J.streams = streams; J.n_workers = n_workers; J.logs = logs; J.cfgv = cfgv;
    J.out_fscores = out_scores; J.out_keys = out_keys;
    run_batch(&J, nthreads);
}

void cco_ngram_workers(const int64_t *ciphers, const int64_t *offsets, const int32_t *cipher_of,
                       const uint64_t *seeds, const uint64_t *streams, int64_t n_workers, int order,
                       const int64_t *S, int64_t climbings, int64_t *out_scores, int64_t *out_maps,
                       int nthreads) {
    batch_job J;
    memset(&J, 0, sizeof J);
    J.kind = 2; J.order = order; J.ciphers = ciphers; J.offsets = offsets; J.cipher_of = cipher_of;
    J.seeds = seeds; J.streams = streams; J.n_workers = n_workers; J.S = S;
    J.climbings = climbings; J.out_iscores = out_scores; J.out_keys = out_maps;
    run_batch(&J, nthreads);
}

void cco_sct_fast_workers(const int64_t *ciphers, const int64_t *offsets, const int32_t *cipher_of,
                          const uint64_t *seeds, const uint64_t *streams, int64_t n_workers,
                          const int64_t *q, const int64_t *cfgv, int64_t *out_scores,
                          int64_t *out_keys, int nthreads) {
    batch_job J;
    memset(&J, 0, sizeof J);
    J.kind = 3; J.ciphers = ciphers; J.offsets = offsets; J.cipher_of = cipher_of;
    J.seeds = seeds; J.streams = streams; J.n_workers = n_workers; J.S = q; J.cfgv = cfgv;
    J.out_iscores = out_scores; J.out_keys = out_keys;
    run_batch(&J, nthreads);
}
