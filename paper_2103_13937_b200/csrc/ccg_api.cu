// ccg_api.cu -- the C ABI (include/cipherclimb_b200.h): contexts, device memory, argument
// validation and the host<->HBM staging around the kernels in ccg_mas.cu / ccg_sct.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "ccg_internal.h"

using namespace ccg;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(CCG_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CCG_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

}  // namespace

struct ccg_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  // grow-only scratch buffers for the host-pointer entry points, one per slot
  std::vector<std::pair<void*, size_t>> scratch;

  int buf(int slot, size_t bytes, void** out) {
    if ((size_t)slot >= scratch.size()) scratch.resize(slot + 1, {nullptr, 0});
    auto& b = scratch[slot];
    if (b.second < bytes || !b.first) {
      if (b.first) {
        CCG_CUDA(cudaStreamSynchronize(stream));
        CCG_CUDA(cudaFree(b.first));
        b.first = nullptr;
        b.second = 0;
      }
      size_t cap = bytes < 256 ? 256 : bytes;
      cap = (cap + 4095) & ~(size_t)4095;
      CCG_CUDA(cudaMalloc(&b.first, cap));
      b.second = cap;
    }
    *out = b.first;
    return CCG_OK;
  }
  // a zeroed worker ticket counter for the next climb launch (WorkerTickets)
  int tickets(unsigned long long** out) {
    void* t = nullptr;
    int rc = buf(15, sizeof(unsigned long long), &t);
    if (rc) return rc;
    CCG_CUDA(cudaMemsetAsync(t, 0, sizeof(unsigned long long), stream));
    *out = (unsigned long long*)t;
    return CCG_OK;
  }
};

namespace {

int enter(ccg_ctx* ctx) {
  if (!ctx) return fail(CCG_ERR_INVALID, "null context");
  CCG_CUDA(cudaSetDevice(ctx->device));
  return CCG_OK;
}

// upload `bytes` from host into scratch slot; returns device pointer in *dev
int upload(ccg_ctx* ctx, int slot, const void* host, size_t bytes, void** dev) {
  int rc = ctx->buf(slot, bytes, dev);
  if (rc) return rc;
  if (bytes) CCG_CUDA(cudaMemcpyAsync(*dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return CCG_OK;
}

int download(ccg_ctx* ctx, void* host, const void* dev, size_t bytes) {
  if (bytes) CCG_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return CCG_OK;
}

int finish(ccg_ctx* ctx, cudaError_t launch_err, const char* what) {
  if (launch_err != cudaSuccess) return cuda_fail(launch_err, what);
  CCG_CUDA(cudaStreamSynchronize(ctx->stream));
  return CCG_OK;
}

int check_ragged(const uint8_t* texts, const int64_t* offsets, int64_t n, const char* what,
                 int64_t* max_len) {
  if (n < 0) return fail(CCG_ERR_INVALID, "%s: negative count", what);
  if (n > 0 && (!offsets)) return fail(CCG_ERR_INVALID, "%s: null offsets", what);
  if (offsets && offsets[0] != 0) return fail(CCG_ERR_INVALID, "%s: offsets[0] must be 0", what);
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t L = offsets[i + 1] - offsets[i];
    if (L < 0) return fail(CCG_ERR_INVALID, "%s: offsets must be non-decreasing", what);
    m = std::max(m, L);
  }
  const int64_t total = n > 0 ? offsets[n] : 0;
  if (total > 0 && !texts) return fail(CCG_ERR_INVALID, "%s: null texts", what);
  // eight letters per step: a byte is >= 26 iff its top bit is set or (its low 7 bits + 102)
  // reaches 128 (no carry can cross bytes: 127 + 102 < 256); the byte loop only locates it
  bool bad = false;
  int64_t i = 0;
  for (; i + 8 <= total; i += 8) {
    uint64_t x;
    memcpy(&x, texts + i, 8);
    const uint64_t y = x & 0x7f7f7f7f7f7f7f7fULL;
    if (((y + 0x6666666666666666ULL) | x) & 0x8080808080808080ULL) {
      bad = true;
      break;
    }
  }
  if (!bad)
    for (; i < total; ++i) bad |= texts[i] >= kAlpha;
  if (bad)
    for (int64_t j = 0; j < total; ++j)
      if (texts[j] >= kAlpha)
        return fail(CCG_ERR_INVALID, "%s: letter %d at position %lld outside 0..25", what,
                    (int)texts[j], (long long)j);
  if (max_len) *max_len = m;
  return CCG_OK;
}

// min/max over the indices (vectorises), the per-index loop only to report the first bad one
int check_cipher_of(const int32_t* cof, int64_t nw, int64_t n_ciphers) {
  int32_t lo = 0, hi = 0;
  if (nw > 0) lo = hi = cof[0];
  for (int64_t i = 0; i < nw; ++i) {
    lo = std::min(lo, cof[i]);
    hi = std::max(hi, cof[i]);
  }
  if (nw > 0 && (lo < 0 || hi >= n_ciphers))
    for (int64_t i = 0; i < nw; ++i)
      if (cof[i] < 0 || cof[i] >= n_ciphers)
        return fail(CCG_ERR_INVALID, "cipher_of[%lld] out of range", (long long)i);
  return CCG_OK;
}

int check_table(const int64_t* table, int64_t* tmax) {
  if (!table) return fail(CCG_ERR_INVALID, "null table");
  int64_t m = 0;
  for (int i = 0; i < kAlpha * kAlpha; ++i) {
    if (table[i] < 0) return fail(CCG_ERR_INVALID, "bigram scores must be non-negative");
    m = std::max(m, table[i]);
  }
  *tmax = m;
  return CCG_OK;
}

// The packed 16-bit / int32 fast path is exact iff every table entry fits 16 bits and every
// score or partial delta, bounded by (n-1)*max(S), fits int32.
bool mas_needs_wide(int64_t max_len, int64_t table_max) {
  if (table_max > 65535) return true;
  const int64_t n1 = max_len > 0 ? max_len - 1 : 0;
  return table_max > 0 && n1 > (int64_t)2147483647 / table_max;
}

int check_logs(const double* logs) {
  if (!logs) return fail(CCG_ERR_INVALID, "null log table");
  return CCG_OK;
}

}  // namespace

extern "C" {

int ccg_abi_version(void) { return CCG_ABI_VERSION; }

const char* ccg_last_error(void) { return g_err.c_str(); }

int ccg_device_count(int* out) {
  if (!out) return fail(CCG_ERR_INVALID, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    *out = 0;
    cudaGetLastError();
    return CCG_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  *out = n;
  return CCG_OK;
}

int ccg_ctx_create(int device, ccg_ctx** out) {
  if (!out) return fail(CCG_ERR_INVALID, "null out");
  *out = nullptr;
  int n = 0;
  int rc = ccg_device_count(&n);
  if (rc) return rc;
  if (n == 0) return fail(CCG_ERR_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(CCG_ERR_INVALID, "device %d out of range (have %d)", device, n);
  CCG_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  CCG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(CCG_ERR_NO_DEVICE, "device %d is sm_%d%d; this engine is built for sm_100a (B200)",
                device, prop.major, prop.minor);
  ccg_ctx* ctx = new ccg_ctx();
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_fail(e, "cudaStreamCreate");
  }
  *out = ctx;
  return CCG_OK;
}

int ccg_ctx_destroy(ccg_ctx* ctx) {
  if (!ctx) return CCG_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& b : ctx->scratch)
    if (b.first) cudaFree(b.first);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return CCG_OK;
}

int ccg_ctx_synchronize(ccg_ctx* ctx) {
  int rc = enter(ctx);
  if (rc) return rc;
  CCG_CUDA(cudaStreamSynchronize(ctx->stream));
  return CCG_OK;
}

int ccg_ctx_stream(ccg_ctx* ctx, void** out) {
  if (!ctx || !out) return fail(CCG_ERR_INVALID, "null argument");
  *out = (void*)ctx->stream;
  return CCG_OK;
}

int ccg_ctx_device(ccg_ctx* ctx, int* out) {
  if (!ctx || !out) return fail(CCG_ERR_INVALID, "null argument");
  *out = ctx->device;
  return CCG_OK;
}

int ccg_ctx_launch_count(ccg_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return fail(CCG_ERR_INVALID, "null argument");
  *out = ctx->launches;
  return CCG_OK;
}

int ccg_ctx_sm_count(ccg_ctx* ctx, int* out) {
  if (!ctx || !out) return fail(CCG_ERR_INVALID, "null argument");
  *out = ctx->sm_count;
  return CCG_OK;
}

int ccg_dev_alloc(ccg_ctx* ctx, size_t bytes, void** out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!out) return fail(CCG_ERR_INVALID, "null out");
  CCG_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  return CCG_OK;
}

int ccg_dev_free(ccg_ctx* ctx, void* ptr) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (ptr) {
    CCG_CUDA(cudaStreamSynchronize(ctx->stream));
    CCG_CUDA(cudaFree(ptr));
  }
  return CCG_OK;
}

int ccg_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(CCG_ERR_INVALID, "null out");
  CCG_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
  return CCG_OK;
}

int ccg_host_free(void* ptr) {
  if (ptr) CCG_CUDA(cudaFreeHost(ptr));
  return CCG_OK;
}

int ccg_memcpy_h2d(ccg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (bytes) CCG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return CCG_OK;
}

int ccg_memcpy_d2h(ccg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (bytes) CCG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return CCG_OK;
}

// ------------------------------------------------------------------ rng
static int philox_common(ccg_ctx* ctx, uint64_t k0, uint64_t k1, uint64_t skip, uint32_t bound,
                         int64_t count, double* out_u, int64_t* out_i) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (count < 0) return fail(CCG_ERR_INVALID, "count must be non-negative");
  if (count == 0) return CCG_OK;
  if ((out_u == nullptr) == (out_i == nullptr)) return fail(CCG_ERR_INVALID, "null out");
  if (out_i && bound < 1) return fail(CCG_ERR_INVALID, "bound must be at least 1");
  void* d = nullptr;
  rc = ctx->buf(0, (size_t)count * 8, &d);
  if (rc) return rc;
  ctx->launches++;
  cudaError_t e = launch_philox_uniform(ctx->stream, k0, k1, skip, count, bound,
                                        out_u ? (double*)d : nullptr, out_i ? (int64_t*)d : nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "philox kernel");
  rc = download(ctx, out_u ? (void*)out_u : (void*)out_i, d, (size_t)count * 8);
  if (rc) return rc;
  return finish(ctx, cudaSuccess, "philox");
}

int ccg_philox_uniform(ccg_ctx* ctx, uint64_t k0, uint64_t k1, uint64_t skip, int64_t count,
                       double* out) {
  return philox_common(ctx, k0, k1, skip, 1, count, out, nullptr);
}

int ccg_philox_int_below(ccg_ctx* ctx, uint64_t k0, uint64_t k1, uint64_t skip, uint32_t bound,
                         int64_t count, int64_t* out) {
  return philox_common(ctx, k0, k1, skip, bound, count, nullptr, out);
}

// ------------------------------------------------------------------ fitness batches
int ccg_score_text_batch(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                         int64_t n_texts, const int64_t* table, int64_t* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  int64_t max_len = 0, tmax = 0;
  if ((rc = check_ragged(texts, offsets, n_texts, "score_text", &max_len))) return rc;
  if ((rc = check_table(table, &tmax))) return rc;
  if (n_texts == 0) return CCG_OK;
  if (!out) return fail(CCG_ERR_INVALID, "null out");
  void *dt, *doff, *dtab, *dout;
  if ((rc = upload(ctx, 0, texts, (size_t)offsets[n_texts], &dt))) return rc;
  if ((rc = upload(ctx, 1, offsets, (size_t)(n_texts + 1) * 8, &doff))) return rc;
  if ((rc = upload(ctx, 2, table, kAlpha * kAlpha * 8, &dtab))) return rc;
  if ((rc = ctx->buf(3, (size_t)n_texts * 8, &dout))) return rc;
  ctx->launches++;
  cudaError_t e = launch_score_text(ctx->stream, (const uint8_t*)dt, (const int64_t*)doff, n_texts,
                                    (const int64_t*)dtab, (int64_t*)dout);
  if (e != cudaSuccess) return cuda_fail(e, "score_text kernel");
  if ((rc = download(ctx, out, dout, (size_t)n_texts * 8))) return rc;
  return finish(ctx, cudaSuccess, "score_text");
}

// Score (cipher, key) pairs grouped by ciphertext length; keys may be NULL for k=1 identity.
// Score (cipher, key) pairs: texts the warp evaluator's plan covers are grouped by length
// (one plan per length); longer ones take the any-length kernel.  keys may be NULL (k = 1
// identity transposition, i.e. plain log_score_text).
static int sct_score_grouped(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                             int64_t n_texts, const int32_t* cipher_of, const uint8_t* keys,
                             int32_t k, int64_t n_keys, int order, const double* logs,
                             double* out) {
  std::map<int64_t, std::vector<int64_t>> by_len;
  std::vector<int64_t> long_idx;
  for (int64_t i = 0; i < n_keys; ++i) {
    const int32_t c = cipher_of ? cipher_of[i] : (int32_t)i;
    if (c < 0 || c >= n_texts) return fail(CCG_ERR_INVALID, "cipher_of[%lld] out of range", (long long)i);
    const int64_t L = offsets[c + 1] - offsets[c];
    if (L < k) return fail(CCG_ERR_INVALID, "ciphertext shorter than the key");
    if (L < order) {
      out[i] = 0.0;  // ngrams.py:169-170: fewer than two letters (one window) score 0.0
      continue;
    }
    if (L > kSctMaxLen) {
      long_idx.push_back(i);
      continue;
    }
    by_len[L].push_back(i);
  }
  if (by_len.empty() && long_idx.empty()) return CCG_OK;
  int rc;
  void *dt, *doffv, *dlogs;
  if ((rc = upload(ctx, 0, texts, (size_t)offsets[n_texts], &dt))) return rc;
  if ((rc = upload(ctx, 1, offsets, (size_t)(n_texts + 1) * 8, &doffv))) return rc;
  int64_t T = 1;
  for (int q = 0; q < order; ++q) T *= kAlpha;
  if ((rc = upload(ctx, 2, logs, (size_t)T * 8, &dlogs))) return rc;
  const int64_t* doff = (const int64_t*)doffv;
  std::vector<int32_t> cof;
  std::vector<uint8_t> kbuf;
  std::vector<double> res;
  auto run = [&](const std::vector<int64_t>& idx, int64_t L, bool long_path) -> int {
    const int64_t m = (int64_t)idx.size();
    cof.resize(m);
    kbuf.resize((size_t)m * k);
    for (int64_t j = 0; j < m; ++j) {
      const int64_t i = idx[j];
      cof[j] = cipher_of ? cipher_of[i] : (int32_t)i;
      for (int q = 0; q < k; ++q) kbuf[j * k + q] = keys ? keys[i * k + q] : (uint8_t)q;
    }
    void *dcof, *dkeys, *dout;
    int r;
    if ((r = upload(ctx, 3, cof.data(), (size_t)m * 4, &dcof))) return r;
    if ((r = upload(ctx, 4, kbuf.data(), (size_t)m * k, &dkeys))) return r;
    if ((r = ctx->buf(5, (size_t)m * 8, &dout))) return r;
    cudaError_t e;
    SumPlan plan;
    if (!long_path) {
      build_sum_plan(L - order + 1, &plan);
      if (plan.n_leaves > kSctMaxLeaves) long_path = true;
    }
    ctx->launches++;
    if (long_path)
      e = launch_sct_score_long(ctx->stream, (const uint8_t*)dt, doff, (const int32_t*)dcof,
                                (const uint8_t*)dkeys, k, m, order, (const double*)dlogs,
                                (double*)dout);
    else
      e = launch_sct_score(ctx->stream, (const uint8_t*)dt, doff, (const int32_t*)dcof,
                           (const uint8_t*)dkeys, k, m, order, (const double*)dlogs,
                           (double*)dout, (int32_t)L, plan);
    if (e != cudaSuccess) return cuda_fail(e, "sct_score kernel");
    res.resize(m);
    if ((r = download(ctx, res.data(), dout, (size_t)m * 8))) return r;
    CCG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int64_t j = 0; j < m; ++j) out[idx[j]] = res[j];
    return CCG_OK;
  };
  for (auto& kv : by_len)
    if ((rc = run(kv.second, kv.first, false))) return rc;
  if (!long_idx.empty() && (rc = run(long_idx, 0, true))) return rc;
  return CCG_OK;
}

static int log_score_common(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                            int64_t n_texts, int order, const double* logs, double* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (order < 2 || order > 4)
    return fail(CCG_ERR_UNSUPPORTED, "n-gram order %d: the engine supports 2..4", order);
  if ((rc = check_ragged(texts, offsets, n_texts, "log_score_text", nullptr))) return rc;
  if ((rc = check_logs(logs))) return rc;
  if (n_texts == 0) return CCG_OK;
  if (!out) return fail(CCG_ERR_INVALID, "null out");
  // identity transposition (k = 1) decrypts a text to itself
  for (int64_t i = 0; i < n_texts; ++i)
    if (offsets[i + 1] - offsets[i] < 1) out[i] = 0.0;
  std::vector<int32_t> idx;
  for (int64_t i = 0; i < n_texts; ++i)
    if (offsets[i + 1] - offsets[i] >= 1) idx.push_back((int32_t)i);
  std::vector<double> res(idx.size());
  rc = sct_score_grouped(ctx, texts, offsets, n_texts, idx.data(), nullptr, 1,
                         (int64_t)idx.size(), order, logs, res.data());
  if (rc) return rc;
  for (size_t j = 0; j < idx.size(); ++j) out[idx[j]] = res[j];
  return CCG_OK;
}

int ccg_log_score_text_batch(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                             int64_t n_texts, const double* logs, double* out) {
  return log_score_common(ctx, texts, offsets, n_texts, 2, logs, out);
}

int ccg_ngram_log_score_batch(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                              int64_t n_texts, int32_t order, const double* logs, double* out) {
  return log_score_common(ctx, texts, offsets, n_texts, order, logs, out);
}

int ccg_mas_delta_batch(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                        int64_t n_texts, const int32_t* ab, const int64_t* table, int64_t* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  int64_t max_len = 0, tmax = 0;
  if ((rc = check_ragged(texts, offsets, n_texts, "mas_delta", &max_len))) return rc;
  if ((rc = check_table(table, &tmax))) return rc;
  if (n_texts == 0) return CCG_OK;
  if (!ab || !out) return fail(CCG_ERR_INVALID, "null argument");
  if (max_len > kMasMaxLen)
    return fail(CCG_ERR_UNSUPPORTED, "text of %lld letters exceeds the engine limit %lld",
                (long long)max_len, (long long)kMasMaxLen);
  for (int64_t i = 0; i < n_texts; ++i) {
    const int a = ab[2 * i], b = ab[2 * i + 1];
    if (a < 0 || a >= kAlpha || b < 0 || b >= kAlpha || a == b)
      return fail(CCG_ERR_INVALID, "pair %lld: letters must be distinct in 0..25", (long long)i);
  }
  void *dt, *doff, *dab, *dtab, *dout;
  if ((rc = upload(ctx, 0, texts, (size_t)offsets[n_texts], &dt))) return rc;
  if ((rc = upload(ctx, 1, offsets, (size_t)(n_texts + 1) * 8, &doff))) return rc;
  if ((rc = upload(ctx, 2, ab, (size_t)n_texts * 8, &dab))) return rc;
  if ((rc = upload(ctx, 3, table, kAlpha * kAlpha * 8, &dtab))) return rc;
  if ((rc = ctx->buf(4, (size_t)n_texts * 8, &dout))) return rc;
  ctx->launches++;
  cudaError_t e = launch_mas_delta(ctx->stream, (const uint8_t*)dt, (const int64_t*)doff, n_texts,
                                   (const int32_t*)dab, (const int64_t*)dtab,
                                   mas_needs_wide(max_len, tmax), (int64_t*)dout);
  if (e != cudaSuccess) return cuda_fail(e, "mas_delta kernel");
  if ((rc = download(ctx, out, dout, (size_t)n_texts * 8))) return rc;
  return finish(ctx, cudaSuccess, "mas_delta");
}

int ccg_mas_delta_counts_batch(ccg_ctx* ctx, const int64_t* counts, int64_t n, const int32_t* ab,
                               const int64_t* table, int64_t* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (n < 0) return fail(CCG_ERR_INVALID, "negative count");
  if (n == 0) return CCG_OK;
  if (!counts || !ab || !table || !out) return fail(CCG_ERR_INVALID, "null argument");
  int64_t total_max = 0, smax = 0;
  bool neg = false;
  for (int i = 0; i < kAlpha * kAlpha; ++i) {
    neg |= table[i] < 0;
    smax = std::max(smax, table[i] < 0 ? -table[i] : table[i]);
  }
  for (int64_t j = 0; j < n; ++j) {
    int64_t tot = 0;
    for (int i = 0; i < kAlpha * kAlpha; ++i) {
      const int64_t c = counts[j * kAlpha * kAlpha + i];
      if (c < 0 || c > 65535)
        return fail(CCG_ERR_UNSUPPORTED, "count matrix %lld: entries must lie in 0..65535", (long long)j);
      tot += c;
    }
    total_max = std::max(total_max, tot);
    const int a = ab[2 * j], b = ab[2 * j + 1];
    if (a < 0 || a >= kAlpha || b < 0 || b >= kAlpha)
      return fail(CCG_ERR_INVALID, "pair %lld: letters must lie in 0..25", (long long)j);
  }
  const bool wide = neg || mas_needs_wide(total_max + 1, smax);
  void *dc, *dab, *dtab, *dout;
  if ((rc = upload(ctx, 0, counts, (size_t)n * kAlpha * kAlpha * 8, &dc))) return rc;
  if ((rc = upload(ctx, 1, ab, (size_t)n * 8, &dab))) return rc;
  if ((rc = upload(ctx, 2, table, kAlpha * kAlpha * 8, &dtab))) return rc;
  if ((rc = ctx->buf(3, (size_t)n * 8, &dout))) return rc;
  ctx->launches++;
  cudaError_t e = launch_mas_delta_counts(ctx->stream, (const int64_t*)dc, n, (const int32_t*)dab,
                                          (const int64_t*)dtab, wide, (int64_t*)dout);
  if (e != cudaSuccess) return cuda_fail(e, "mas_delta_counts kernel");
  if ((rc = download(ctx, out, dout, (size_t)n * 8))) return rc;
  return finish(ctx, cudaSuccess, "mas_delta_counts");
}

// ------------------------------------------------------------------ MAS climb
static int mas_launch(ccg_ctx* ctx, const ccg_mas_climb_args* a, int64_t max_len, int64_t tmax) {
  if (max_len > kMasMaxLen)
    return fail(CCG_ERR_UNSUPPORTED, "ciphertext of %lld letters exceeds the engine limit %lld",
                (long long)max_len, (long long)kMasMaxLen);
  MasLaunch p;
  p.ciphers = a->ciphers;
  p.offsets = a->offsets;
  p.cipher_of = a->cipher_of;
  p.keys = a->keys;
  p.skips = a->skips;
  p.n_workers = a->n_workers;
  p.climbings = a->climbings;
  p.table = a->table;
  p.scores = a->scores;
  p.maps = a->maps;
  p.draws_used = a->draws_used;
  p.last_accept = a->last_accept;
  p.tries_done = a->tries_done;
  p.flags = a->flags;
  p.accepts = a->accepts;
  if (int rc = ctx->tickets(&p.tickets)) return rc;
  ctx->launches++;
  cudaError_t e;
  const uint32_t kern = a->flags & CCG_FLAG_KERNEL_MASK;
  const bool dform = kern == 0 || kern == CCG_FLAG_KERNEL_DFORM || kern == CCG_FLAG_KERNEL_DTABLE;
  p.init = nullptr;
  if (dform && mas_dform_ok(max_len, tmax)) {
    // workers of a ciphertext share their initial state: compute it once per ciphertext
    if (a->n_ciphers > 0 && a->n_workers >= 4 * a->n_ciphers) {
      void* init = nullptr;
      int rc = ctx->buf(14, dform_init_bytes(a->n_ciphers), &init);
      if (rc) return rc;
      ctx->launches++;
      e = launch_dform_init(ctx->stream, p, a->n_ciphers, init, ctx->sm_count);
      if (e != cudaSuccess) return cuda_fail(e, "dform_init kernel");
      p.init = init;
    }
    e = launch_mas_climb_dform(ctx->stream, p, ctx->sm_count);
  }
  else if ((dform || kern == CCG_FLAG_KERNEL_TFORM) && mas_tform_ok(max_len, tmax))
    e = launch_mas_climb_tform(ctx->stream, p, ctx->sm_count);
  else
    e = launch_mas_climb(ctx->stream, p, mas_needs_wide(max_len, tmax), ctx->sm_count);
  if (e != cudaSuccess) return cuda_fail(e, "mas_climb kernel");
  if (a->group_size > 0 && a->group_best) {
    ctx->launches++;
    e = launch_group_best_i64(ctx->stream, a->scores, a->n_workers / a->group_size, a->group_size,
                              a->group_best);
    if (e != cudaSuccess) return cuda_fail(e, "group_best kernel");
  }
  return CCG_OK;
}

static int check_climb_common(int64_t n_workers, int64_t climbings, int32_t group_size,
                              const void* scores, const void* keys, const void* cipher_of) {
  if (n_workers < 0) return fail(CCG_ERR_INVALID, "n_workers must be non-negative");
  if (climbings < 0) return fail(CCG_ERR_INVALID, "climbings must be non-negative");
  if (climbings > 2147483647LL)
    return fail(CCG_ERR_UNSUPPORTED, "climbings above 2^31-1 per call are not supported");
  if (n_workers > 0 && (!scores || !keys || !cipher_of))
    return fail(CCG_ERR_INVALID, "scores, keys and cipher_of are required");
  if (group_size < 0) return fail(CCG_ERR_INVALID, "group_size must be non-negative");
  if (group_size > 0 && n_workers % group_size)
    return fail(CCG_ERR_INVALID, "n_workers must be a multiple of group_size");
  return CCG_OK;
}

int ccg_mas_climb_dev(ccg_ctx* ctx, const ccg_mas_climb_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if ((rc = check_climb_common(a->n_workers, a->climbings, a->group_size, a->scores, a->keys,
                               a->cipher_of)))
    return rc;
  if (a->table_max < 0) return fail(CCG_ERR_INVALID, "table_max must be set");
  return mas_launch(ctx, a, a->max_len, a->table_max);
}

int ccg_mas_climb(ccg_ctx* ctx, const ccg_mas_climb_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if ((rc = check_climb_common(a->n_workers, a->climbings, a->group_size, a->scores, a->keys,
                               a->cipher_of)))
    return rc;
  int64_t max_len = 0, tmax = 0;
  if ((rc = check_ragged(a->ciphers, a->offsets, a->n_ciphers, "mas_climb", &max_len))) return rc;
  if ((rc = check_table(a->table, &tmax))) return rc;
  const int64_t nw = a->n_workers;
  if (nw == 0) return CCG_OK;
  if ((rc = check_cipher_of(a->cipher_of, nw, a->n_ciphers))) return rc;
  ccg_mas_climb_args d = *a;
  void* p;
  if ((rc = upload(ctx, 0, a->ciphers, (size_t)a->offsets[a->n_ciphers], &p))) return rc;
  d.ciphers = (const uint8_t*)p;
  if ((rc = upload(ctx, 1, a->offsets, (size_t)(a->n_ciphers + 1) * 8, &p))) return rc;
  d.offsets = (const int64_t*)p;
  if ((rc = upload(ctx, 2, a->cipher_of, (size_t)nw * 4, &p))) return rc;
  d.cipher_of = (const int32_t*)p;
  if ((rc = upload(ctx, 3, a->keys, (size_t)nw * 16, &p))) return rc;
  d.keys = (const uint64_t*)p;
  if (a->skips) {
    if ((rc = upload(ctx, 4, a->skips, (size_t)nw * 8, &p))) return rc;
    d.skips = (const uint64_t*)p;
  }
  if ((rc = upload(ctx, 5, a->table, kAlpha * kAlpha * 8, &p))) return rc;
  d.table = (const int64_t*)p;
  if ((rc = ctx->buf(6, (size_t)nw * 8, &p))) return rc;
  d.scores = (int64_t*)p;
  if (a->maps) { if ((rc = ctx->buf(7, (size_t)nw * kAlpha, &p))) return rc; d.maps = (uint8_t*)p; }
  if (a->draws_used) { if ((rc = ctx->buf(8, (size_t)nw * 8, &p))) return rc; d.draws_used = (uint64_t*)p; }
  if (a->last_accept) { if ((rc = ctx->buf(9, (size_t)nw * 8, &p))) return rc; d.last_accept = (int64_t*)p; }
  if (a->tries_done) { if ((rc = ctx->buf(10, (size_t)nw * 8, &p))) return rc; d.tries_done = (int64_t*)p; }
  if (a->accepts) { if ((rc = ctx->buf(12, (size_t)nw * 8, &p))) return rc; d.accepts = (int64_t*)p; }
  const int64_t ng = a->group_size > 0 ? nw / a->group_size : 0;
  if (a->group_best && ng) { if ((rc = ctx->buf(11, (size_t)ng * 8, &p))) return rc; d.group_best = (int64_t*)p; }
  else d.group_best = nullptr;
  if ((rc = mas_launch(ctx, &d, max_len, tmax))) return rc;
  if (a->accepts && (rc = download(ctx, a->accepts, d.accepts, (size_t)nw * 8))) return rc;
  if ((rc = download(ctx, a->scores, d.scores, (size_t)nw * 8))) return rc;
  if (a->maps && (rc = download(ctx, a->maps, d.maps, (size_t)nw * kAlpha))) return rc;
  if (a->draws_used && (rc = download(ctx, a->draws_used, d.draws_used, (size_t)nw * 8))) return rc;
  if (a->last_accept && (rc = download(ctx, a->last_accept, d.last_accept, (size_t)nw * 8))) return rc;
  if (a->tries_done && (rc = download(ctx, a->tries_done, d.tries_done, (size_t)nw * 8))) return rc;
  if (d.group_best && (rc = download(ctx, a->group_best, d.group_best, (size_t)ng * 8))) return rc;
  return finish(ctx, cudaSuccess, "mas_climb");
}

// ------------------------------------------------------------------ n-gram extension
static int check_order(int32_t order) {
  if (order < 2 || order > 4)
    return fail(CCG_ERR_UNSUPPORTED, "n-gram order %d: the engine supports 2..4", order);
  return CCG_OK;
}

static int64_t pow26_i(int order) {
  int64_t v = 1;
  for (int i = 0; i < order; ++i) v *= kAlpha;
  return v;
}

int ccg_ngram_score_batch(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                          int64_t n_texts, int32_t order, const int64_t* table, int64_t* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if ((rc = check_order(order))) return rc;
  if ((rc = check_ragged(texts, offsets, n_texts, "ngram_score", nullptr))) return rc;
  if (!table) return fail(CCG_ERR_INVALID, "null table");
  const int64_t T = pow26_i(order);
  for (int64_t i = 0; i < T; ++i)
    if (table[i] < 0) return fail(CCG_ERR_INVALID, "n-gram scores must be non-negative");
  if (n_texts == 0) return CCG_OK;
  if (!out) return fail(CCG_ERR_INVALID, "null out");
  void *dt, *doff, *dtab, *dout;
  if ((rc = upload(ctx, 0, texts, (size_t)offsets[n_texts], &dt))) return rc;
  if ((rc = upload(ctx, 1, offsets, (size_t)(n_texts + 1) * 8, &doff))) return rc;
  if ((rc = upload(ctx, 2, table, (size_t)T * 8, &dtab))) return rc;
  if ((rc = ctx->buf(3, (size_t)n_texts * 8, &dout))) return rc;
  ctx->launches++;
  cudaError_t e = launch_ngram_score(ctx->stream, (const uint8_t*)dt, (const int64_t*)doff, n_texts,
                                     order, (const int64_t*)dtab, (int64_t*)dout);
  if (e != cudaSuccess) return cuda_fail(e, "ngram_score kernel");
  if ((rc = download(ctx, out, dout, (size_t)n_texts * 8))) return rc;
  return finish(ctx, cudaSuccess, "ngram_score");
}

static int ngram_launch(ccg_ctx* ctx, const ccg_mas_ngram_args* a, int64_t max_len) {
  if (max_len > kNgramMaxLen)
    return fail(CCG_ERR_UNSUPPORTED,
                "ciphertext of %lld letters exceeds the n-gram engine limit %lld",
                (long long)max_len, (long long)kNgramMaxLen);
  MasNgramLaunch p;
  p.ciphers = a->ciphers;
  p.offsets = a->offsets;
  p.cipher_of = a->cipher_of;
  p.keys = a->keys;
  p.skips = a->skips;
  p.n_workers = a->n_workers;
  p.climbings = a->climbings;
  p.order = a->order;
  p.table = a->table;
  p.max_len = max_len < 1 ? 1 : max_len;
  p.scores = a->scores;
  p.maps = a->maps;
  p.draws_used = a->draws_used;
  p.last_accept = a->last_accept;
  p.tries_done = a->tries_done;
  p.computed = a->computed;
  p.lookups = a->lookups;
  p.flags = a->flags;
  if (int rc = ctx->tickets(&p.tickets)) return rc;
  ctx->launches++;
  cudaError_t e = launch_mas_ngram_climb(ctx->stream, p, ctx->sm_count);
  if (e != cudaSuccess) return cuda_fail(e, "mas_ngram kernel");
  if (a->group_size > 0 && a->group_best) {
    ctx->launches++;
    e = launch_group_best_i64(ctx->stream, a->scores, a->n_workers / a->group_size, a->group_size,
                              a->group_best);
    if (e != cudaSuccess) return cuda_fail(e, "group_best kernel");
  }
  return CCG_OK;
}

int ccg_mas_ngram_climb_dev(ccg_ctx* ctx, const ccg_mas_ngram_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if ((rc = check_order(a->order))) return rc;
  if ((rc = check_climb_common(a->n_workers, a->climbings, a->group_size, a->scores, a->keys,
                               a->cipher_of)))
    return rc;
  if (!a->table) return fail(CCG_ERR_INVALID, "null table");
  return ngram_launch(ctx, a, a->max_len);
}

int ccg_mas_ngram_climb(ccg_ctx* ctx, const ccg_mas_ngram_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if ((rc = check_order(a->order))) return rc;
  if ((rc = check_climb_common(a->n_workers, a->climbings, a->group_size, a->scores, a->keys,
                               a->cipher_of)))
    return rc;
  if (!a->table) return fail(CCG_ERR_INVALID, "null table");
  int64_t max_len = 0;
  if ((rc = check_ragged(a->ciphers, a->offsets, a->n_ciphers, "mas_ngram_climb", &max_len)))
    return rc;
  const int64_t nw = a->n_workers;
  if (nw == 0) return CCG_OK;
  for (int64_t i = 0; i < nw; ++i)
    if (a->cipher_of[i] < 0 || a->cipher_of[i] >= a->n_ciphers)
      return fail(CCG_ERR_INVALID, "cipher_of[%lld] out of range", (long long)i);
  const int64_t T = pow26_i(a->order);
  ccg_mas_ngram_args d = *a;
  void* p;
  if ((rc = upload(ctx, 0, a->ciphers, (size_t)a->offsets[a->n_ciphers], &p))) return rc;
  d.ciphers = (const uint8_t*)p;
  if ((rc = upload(ctx, 1, a->offsets, (size_t)(a->n_ciphers + 1) * 8, &p))) return rc;
  d.offsets = (const int64_t*)p;
  if ((rc = upload(ctx, 2, a->cipher_of, (size_t)nw * 4, &p))) return rc;
  d.cipher_of = (const int32_t*)p;
  if ((rc = upload(ctx, 3, a->keys, (size_t)nw * 16, &p))) return rc;
  d.keys = (const uint64_t*)p;
  if (a->skips) {
    if ((rc = upload(ctx, 4, a->skips, (size_t)nw * 8, &p))) return rc;
    d.skips = (const uint64_t*)p;
  }
  if ((rc = upload(ctx, 5, a->table, (size_t)T * 2, &p))) return rc;
  d.table = (const uint16_t*)p;
  if ((rc = ctx->buf(6, (size_t)nw * 8, &p))) return rc;
  d.scores = (int64_t*)p;
  if (a->maps) {
    if ((rc = ctx->buf(7, (size_t)nw * kAlpha, &p))) return rc;
    d.maps = (uint8_t*)p;
  }
  if (a->draws_used) {
    if ((rc = ctx->buf(8, (size_t)nw * 8, &p))) return rc;
    d.draws_used = (uint64_t*)p;
  }
  if (a->last_accept) {
    if ((rc = ctx->buf(9, (size_t)nw * 8, &p))) return rc;
    d.last_accept = (int64_t*)p;
  }
  if (a->tries_done) {
    if ((rc = ctx->buf(10, (size_t)nw * 8, &p))) return rc;
    d.tries_done = (int64_t*)p;
  }
  if (a->computed) {
    if ((rc = ctx->buf(12, (size_t)nw * 8, &p))) return rc;
    d.computed = (int64_t*)p;
  }
  if (a->lookups) {
    if ((rc = ctx->buf(13, (size_t)nw * 8, &p))) return rc;
    d.lookups = (int64_t*)p;
  }
  const int64_t ng = a->group_size > 0 ? nw / a->group_size : 0;
  if (a->group_best && ng) {
    if ((rc = ctx->buf(11, (size_t)ng * 8, &p))) return rc;
    d.group_best = (int64_t*)p;
  } else {
    d.group_best = nullptr;
  }
  if ((rc = ngram_launch(ctx, &d, max_len))) return rc;
  if ((rc = download(ctx, a->scores, d.scores, (size_t)nw * 8))) return rc;
  if (a->maps && (rc = download(ctx, a->maps, d.maps, (size_t)nw * kAlpha))) return rc;
  if (a->draws_used && (rc = download(ctx, a->draws_used, d.draws_used, (size_t)nw * 8))) return rc;
  if (a->last_accept && (rc = download(ctx, a->last_accept, d.last_accept, (size_t)nw * 8)))
    return rc;
  if (a->tries_done && (rc = download(ctx, a->tries_done, d.tries_done, (size_t)nw * 8))) return rc;
  if (a->computed && (rc = download(ctx, a->computed, d.computed, (size_t)nw * 8))) return rc;
  if (a->lookups && (rc = download(ctx, a->lookups, d.lookups, (size_t)nw * 8))) return rc;
  if (ng && a->group_best && (rc = download(ctx, a->group_best, d.group_best, (size_t)ng * 8)))
    return rc;
  return finish(ctx, cudaSuccess, "mas_ngram_climb");
}

// ------------------------------------------------------------------ MAS deterministic
static int check_distinct_letters(const uint8_t* texts, const int64_t* offsets, int64_t i,
                                  const char* what) {
  uint32_t seen = 0;
  for (int64_t q = offsets[i]; q < offsets[i + 1]; ++q) seen |= 1u << texts[q];
  if (offsets[i + 1] - offsets[i] < 2 || __builtin_popcount(seen) < 2)
    return fail(CCG_ERR_INVALID, "%s: ciphertext must contain at least two distinct letters", what);
  return CCG_OK;
}

int ccg_mas_det_step_batch(ccg_ctx* ctx, const uint8_t* texts, const int64_t* offsets,
                           int64_t n_texts, const int32_t* pivots, const int64_t* table,
                           int64_t* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  int64_t max_len = 0, tmax = 0;
  if ((rc = check_ragged(texts, offsets, n_texts, "det_step", &max_len))) return rc;
  if ((rc = check_table(table, &tmax))) return rc;
  if (n_texts == 0) return CCG_OK;
  if (!pivots || !out) return fail(CCG_ERR_INVALID, "null argument");
  for (int64_t i = 0; i < n_texts; ++i) {
    const int pl = pivots[2 * i], pr = pivots[2 * i + 1];
    if (pl < 0 || pl >= kAlpha || pr < 0 || pr >= kAlpha)
      return fail(CCG_ERR_INVALID, "pivot %lld: letters must lie in 0..25", (long long)i);
    if (pl == pr) return fail(CCG_ERR_INVALID, "pivot letters must differ");
    bool hl = false, hr = false;
    for (int64_t q = offsets[i]; q < offsets[i + 1]; ++q) {
      hl |= texts[q] == pl;
      hr |= texts[q] == pr;
    }
    if (!(hl && hr)) return fail(CCG_ERR_INVALID, "both pivot letters must occur in the text");
  }
  void *dt, *doff, *dpiv, *dtab, *dout;
  if ((rc = upload(ctx, 0, texts, (size_t)offsets[n_texts], &dt))) return rc;
  if ((rc = upload(ctx, 1, offsets, (size_t)(n_texts + 1) * 8, &doff))) return rc;
  if ((rc = upload(ctx, 2, pivots, (size_t)n_texts * 8, &dpiv))) return rc;
  if ((rc = upload(ctx, 3, table, kAlpha * kAlpha * 8, &dtab))) return rc;
  if ((rc = ctx->buf(4, (size_t)n_texts * 325 * 8, &dout))) return rc;
  ctx->launches++;
  cudaError_t e = launch_mas_det_step(ctx->stream, (const uint8_t*)dt, (const int64_t*)doff, n_texts,
                                      (const int32_t*)dpiv, (const int64_t*)dtab,
                                      mas_needs_wide(max_len, tmax), (int64_t*)dout);
  if (e != cudaSuccess) return cuda_fail(e, "det_step kernel");
  if ((rc = download(ctx, out, dout, (size_t)n_texts * 325 * 8))) return rc;
  return finish(ctx, cudaSuccess, "det_step");
}

static int det_launch(ccg_ctx* ctx, const ccg_mas_det_args* a, int64_t max_len, int64_t tmax) {
  MasDetLaunch p;
  p.ciphers = a->ciphers;
  p.offsets = a->offsets;
  p.cipher_of = a->cipher_of;
  p.keys = a->keys;
  p.n_jobs = a->n_jobs;
  p.iterations = a->iterations;
  p.table = a->table;
  p.scores = a->scores;
  p.maps = a->maps;
  p.hist_iter = a->hist_iter;
  p.hist_score = a->hist_score;
  p.hist_len = a->hist_len;
  p.draws_used = a->draws_used;
  ctx->launches++;
  cudaError_t e = launch_mas_det_solve(ctx->stream, p, mas_needs_wide(max_len, tmax));
  if (e != cudaSuccess) return cuda_fail(e, "det_solve kernel");
  return CCG_OK;
}

static int check_det_common(const ccg_mas_det_args* a) {
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if (a->n_jobs < 0) return fail(CCG_ERR_INVALID, "n_jobs must be non-negative");
  if (a->iterations < 0) return fail(CCG_ERR_INVALID, "iterations must be non-negative");
  if (a->iterations > 2147483647LL)
    return fail(CCG_ERR_UNSUPPORTED, "iterations above 2^31-1 per call are not supported");
  if (a->n_jobs > 2147483647LL) return fail(CCG_ERR_UNSUPPORTED, "too many jobs in one call");
  if (a->n_jobs > 0 && (!a->scores || !a->keys || !a->cipher_of))
    return fail(CCG_ERR_INVALID, "scores, keys and cipher_of are required");
  if ((a->hist_iter || a->hist_score) && !a->hist_len)
    return fail(CCG_ERR_INVALID, "hist_len is required with a history buffer");
  return CCG_OK;
}

int ccg_mas_det_solve_dev(ccg_ctx* ctx, const ccg_mas_det_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if ((rc = check_det_common(a))) return rc;
  if (a->table_max < 0) return fail(CCG_ERR_INVALID, "table_max must be set");
  return det_launch(ctx, a, a->max_len, a->table_max);
}

int ccg_mas_det_solve(ccg_ctx* ctx, const ccg_mas_det_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if ((rc = check_det_common(a))) return rc;
  int64_t max_len = 0, tmax = 0;
  if ((rc = check_ragged(a->ciphers, a->offsets, a->n_ciphers, "mas_det_solve", &max_len))) return rc;
  if ((rc = check_table(a->table, &tmax))) return rc;
  const int64_t nj = a->n_jobs, it = a->iterations;
  if (nj == 0) return CCG_OK;
  for (int64_t i = 0; i < nj; ++i)
    if (a->cipher_of[i] < 0 || a->cipher_of[i] >= a->n_ciphers)
      return fail(CCG_ERR_INVALID, "cipher_of[%lld] out of range", (long long)i);
  for (int64_t c = 0; c < a->n_ciphers; ++c)
    if ((rc = check_distinct_letters(a->ciphers, a->offsets, c, "mas_det_solve"))) return rc;
  ccg_mas_det_args d = *a;
  void* p;
  if ((rc = upload(ctx, 0, a->ciphers, (size_t)a->offsets[a->n_ciphers], &p))) return rc;
  d.ciphers = (const uint8_t*)p;
  if ((rc = upload(ctx, 1, a->offsets, (size_t)(a->n_ciphers + 1) * 8, &p))) return rc;
  d.offsets = (const int64_t*)p;
  if ((rc = upload(ctx, 2, a->cipher_of, (size_t)nj * 4, &p))) return rc;
  d.cipher_of = (const int32_t*)p;
  if ((rc = upload(ctx, 3, a->keys, (size_t)nj * 16, &p))) return rc;
  d.keys = (const uint64_t*)p;
  if ((rc = upload(ctx, 4, a->table, kAlpha * kAlpha * 8, &p))) return rc;
  d.table = (const int64_t*)p;
  if ((rc = ctx->buf(5, (size_t)nj * 8, &p))) return rc;
  d.scores = (int64_t*)p;
  if (a->maps) { if ((rc = ctx->buf(6, (size_t)nj * kAlpha, &p))) return rc; d.maps = (uint8_t*)p; }
  if (a->hist_iter) { if ((rc = ctx->buf(7, (size_t)nj * it * 4, &p))) return rc; d.hist_iter = (int32_t*)p; }
  if (a->hist_score) { if ((rc = ctx->buf(8, (size_t)nj * it * 8, &p))) return rc; d.hist_score = (int64_t*)p; }
  if (a->hist_len) { if ((rc = ctx->buf(9, (size_t)nj * 4, &p))) return rc; d.hist_len = (int32_t*)p; }
  if (a->draws_used) { if ((rc = ctx->buf(10, (size_t)nj * 8, &p))) return rc; d.draws_used = (uint64_t*)p; }
  if ((rc = det_launch(ctx, &d, max_len, tmax))) return rc;
  if ((rc = download(ctx, a->scores, d.scores, (size_t)nj * 8))) return rc;
  if (a->maps && (rc = download(ctx, a->maps, d.maps, (size_t)nj * kAlpha))) return rc;
  if (a->draws_used && (rc = download(ctx, a->draws_used, d.draws_used, (size_t)nj * 8))) return rc;
  if (a->hist_iter && a->hist_score && a->hist_len) {
    // histories are short (a climb stops at its local optimum): pack them on the device and
    // read back only the entries, then place each job's prefix in its row
    if ((rc = download(ctx, a->hist_len, d.hist_len, (size_t)nj * 4))) return rc;
    CCG_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<int64_t> offs((size_t)nj + 1, 0);
    for (int64_t j = 0; j < nj; ++j) {
      const int32_t l = a->hist_len[j];
      if (l < 0 || l > it) return fail(CCG_ERR_CUDA, "history length out of range");
      offs[j + 1] = offs[j] + l;
    }
    const int64_t total = offs[nj];
    if (total > 0) {
      if ((rc = upload(ctx, 11, offs.data(), offs.size() * 8, &p))) return rc;
      const int64_t* doffs = (const int64_t*)p;
      void *pi, *ps;
      if ((rc = ctx->buf(12, (size_t)total * 4, &pi))) return rc;
      if ((rc = ctx->buf(13, (size_t)total * 8, &ps))) return rc;
      ctx->launches++;
      cudaError_t e = launch_compact_history(ctx->stream, d.hist_iter, d.hist_score, it, doffs, nj,
                                             (int32_t*)pi, (int64_t*)ps);
      if (e != cudaSuccess) return cuda_fail(e, "compact_history kernel");
      std::vector<int32_t> hi;
      std::vector<int64_t> hs;
      int32_t* dst_i = a->hist_iter;  // packed output: straight into the caller's arrays
      int64_t* dst_s = a->hist_score;
      if (!a->hist_offsets) {
        hi.resize((size_t)total);
        hs.resize((size_t)total);
        dst_i = hi.data();
        dst_s = hs.data();
      }
      if ((rc = download(ctx, dst_i, pi, (size_t)total * 4))) return rc;
      if ((rc = download(ctx, dst_s, ps, (size_t)total * 8))) return rc;
      CCG_CUDA(cudaStreamSynchronize(ctx->stream));
      if (!a->hist_offsets)
        for (int64_t j = 0; j < nj; ++j) {
          const int64_t l = offs[j + 1] - offs[j];
          std::memcpy(a->hist_iter + j * it, hi.data() + offs[j], (size_t)l * 4);
          std::memcpy(a->hist_score + j * it, hs.data() + offs[j], (size_t)l * 8);
        }
    }
    if (a->hist_offsets) std::memcpy(a->hist_offsets, offs.data(), offs.size() * 8);
  } else {
    if (a->hist_iter && (rc = download(ctx, a->hist_iter, d.hist_iter, (size_t)nj * it * 4))) return rc;
    if (a->hist_score && (rc = download(ctx, a->hist_score, d.hist_score, (size_t)nj * it * 8))) return rc;
    if (a->hist_len && (rc = download(ctx, a->hist_len, d.hist_len, (size_t)nj * 4))) return rc;
  }
  return finish(ctx, cudaSuccess, "mas_det_solve");
}

// ------------------------------------------------------------------ SCT
static int sct_score_common(ccg_ctx* ctx, const uint8_t* ciphers, const int64_t* offsets,
                            int64_t n_ciphers, const int32_t* cipher_of, const uint8_t* keys,
                            int32_t key_length, int64_t n_keys, int order, const double* logs,
                            double* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (order < 2 || order > 4)
    return fail(CCG_ERR_UNSUPPORTED, "n-gram order %d: the engine supports 2..4", order);
  if ((rc = check_ragged(ciphers, offsets, n_ciphers, "sct_score", nullptr))) return rc;
  if ((rc = check_logs(logs))) return rc;
  if (key_length < 1) return fail(CCG_ERR_INVALID, "key_length must be at least 1");
  if (key_length > kSctMaxKey)
    return fail(CCG_ERR_UNSUPPORTED, "key length %d exceeds the engine limit %d", key_length, kSctMaxKey);
  if (n_keys <= 0) return CCG_OK;
  if (!keys || !cipher_of || !out) return fail(CCG_ERR_INVALID, "null argument");
  for (int64_t i = 0; i < n_keys; ++i) {
    uint64_t seen = 0;
    for (int q = 0; q < key_length; ++q) {
      const int v = keys[i * key_length + q];
      if (v >= key_length || (seen >> v) & 1)
        return fail(CCG_ERR_INVALID, "transposition key must be a permutation of 0..k-1");
      seen |= 1ULL << v;
    }
  }
  return sct_score_grouped(ctx, ciphers, offsets, n_ciphers, cipher_of, keys, key_length, n_keys,
                           order, logs, out);
}

int ccg_sct_score_batch(ccg_ctx* ctx, const uint8_t* ciphers, const int64_t* offsets,
                        int64_t n_ciphers, const int32_t* cipher_of, const uint8_t* keys,
                        int32_t key_length, int64_t n_keys, const double* logs, double* out) {
  return sct_score_common(ctx, ciphers, offsets, n_ciphers, cipher_of, keys, key_length, n_keys, 2,
                          logs, out);
}

int ccg_sct_score_ngram_batch(ccg_ctx* ctx, const uint8_t* ciphers, const int64_t* offsets,
                              int64_t n_ciphers, const int32_t* cipher_of, const uint8_t* keys,
                              int32_t key_length, int64_t n_keys, int32_t order, const double* logs,
                              double* out) {
  return sct_score_common(ctx, ciphers, offsets, n_ciphers, cipher_of, keys, key_length, n_keys,
                          order, logs, out);
}

static int sct_check(const ccg_sct_climb_args* a) {
  int rc;
  if ((rc = check_climb_common(a->n_workers, a->climbings, a->group_size, a->scores, a->keys,
                               a->cipher_of)))
    return rc;
  if (a->key_length < 2) return fail(CCG_ERR_INVALID, "key_length must be at least 2");
  if (a->key_length > kSctMaxKey)
    return fail(CCG_ERR_UNSUPPORTED, "key length %d exceeds the engine limit %d", a->key_length, kSctMaxKey);
  if (!(0 <= a->p1 && a->p1 <= a->p2 && a->p2 <= 100))
    return fail(CCG_ERR_INVALID, "thresholds must satisfy 0 <= p1 <= p2 <= 100");
  if (a->op1_hop < 1 || a->op2_hop < 1) return fail(CCG_ERR_INVALID, "op hops must be at least 1");
  if (a->n_workers > 0 && !a->keys_out) return fail(CCG_ERR_INVALID, "keys_out is required");
  if (!(a->order == 0 || (a->order >= 2 && a->order <= 4)))
    return fail(CCG_ERR_UNSUPPORTED, "n-gram order %d: the engine supports 2..4", a->order);
  return check_logs(a->logs);
}

// The warp-per-worker family (ccg_sct.cu): the speculative latency kernel for few workers,
// else one warp per worker.  Needs one common text length n.
static int sct_launch_warp(ccg_ctx* ctx, const ccg_sct_climb_args* a, int64_t n) {
  if (n < 0)
    return fail(CCG_ERR_INVALID, "the warp SCT kernels need one common ciphertext length per call");
  if (n < a->key_length && !a->key_lengths)
    return fail(CCG_ERR_INVALID, "ciphertext shorter than the key");
  if (n > kSctMaxLen)
    return fail(CCG_ERR_UNSUPPORTED, "ciphertext of %lld letters exceeds the engine limit %lld",
                (long long)n, (long long)kSctMaxLen);
  const int order = a->order == 0 ? 2 : a->order;
  SumPlan plan;
  build_sum_plan(n >= order ? n - order + 1 : 0, &plan);
  if (plan.n_leaves > kSctMaxLeaves)
    return fail(CCG_ERR_UNSUPPORTED, "text length %lld needs %d pairwise leaves (limit %d)",
                (long long)n, plan.n_leaves, kSctMaxLeaves);
  SctLaunch p;
  p.ciphers = a->ciphers;
  p.offsets = a->offsets;
  p.cipher_of = a->cipher_of;
  p.keys = a->keys;
  p.skips = a->skips;
  p.n_workers = a->n_workers;
  p.n = (int32_t)n;
  p.k = a->key_length;
  p.climbings = a->climbings;
  p.p1 = a->p1;
  p.p2 = a->p2;
  p.op1_hop = a->op1_hop;
  p.op2_hop = a->op2_hop;
  p.order = order;
  p.key_lengths = a->key_lengths;
  p.logs = a->logs;
  p.scores = a->scores;
  p.keys_out = a->keys_out;
  p.draws_used = a->draws_used;
  p.last_accept = a->last_accept;
  p.tries_done = a->tries_done;
  p.flags = a->flags;
  if (int rc = ctx->tickets(&p.tickets)) return rc;
  ctx->launches++;
  cudaError_t e = launch_sct_climb(ctx->stream, p, plan, ctx->sm_count);
  if (e != cudaSuccess) return cuda_fail(e, "sct_climb kernel");
  return CCG_OK;
}

extern "C++" {
// A trigram log table has few distinct entries (they are log2 of small counts: 65 for the
// corpus table), so the per-lane kernel can hold it exactly as a byte index per entry plus the
// distinct values (17.6 KB of shared memory instead of 140 KB).  Returns false (no
// compression) beyond 256 distinct bit patterns.  O(n) with a 512-slot open-addressing set.
template <typename V>
static bool compress_table(const V* t, int64_t n, std::vector<uint8_t>& idx, std::vector<V>& vals) {
  static_assert(sizeof(V) <= 8, "");
  uint64_t keys[512];
  int16_t at[512];
  for (int i = 0; i < 512; ++i) at[i] = -1;
  idx.resize((size_t)n);
  vals.clear();
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits = 0;
    memcpy(&bits, &t[i], sizeof(V));
    uint64_t h = bits * 0x9E3779B97F4A7C15ULL;
    int slot = (int)(h >> 55);  // 9 bits
    while (at[slot] >= 0 && keys[slot] != bits) slot = (slot + 1) & 511;
    if (at[slot] < 0) {
      if (vals.size() == 256) return false;
      keys[slot] = bits;
      at[slot] = (int16_t)vals.size();
      vals.push_back(t[i]);
    }
    idx[(size_t)i] = (uint8_t)at[slot];
  }
  return true;
}

// Upload a compressed order-3 table into the launch (scratch slots 16, 17) when it compresses.
template <typename V>
static int attach_compressed(ccg_ctx* ctx, const V* host_table, int order, SctLaneLaunch& p) {
  if (order != 3 || !host_table) return CCG_OK;
  std::vector<uint8_t> idx;
  std::vector<V> vals;
  if (!compress_table(host_table, 17576, idx, vals)) return CCG_OK;
  void* d;
  int rc;
  if ((rc = upload(ctx, 16, idx.data(), idx.size(), &d))) return rc;
  p.cidx = (const uint8_t*)d;
  if ((rc = upload(ctx, 17, vals.data(), vals.size() * sizeof(V), &d))) return rc;
  p.cvals = d;
  p.n_cvals = (int32_t)vals.size();
  return CCG_OK;
}

}  // extern "C++"

// One worker per lane (ccg_sct_lane.cu), parity (mode 0) or fast (mode 1) scoring; texts of
// any mix of lengths up to max_len.
static int sct_launch_lane(ccg_ctx* ctx, SctLaneLaunch& p) {
  if (p.op1_hop > kSctLaneMaxHops || p.op2_hop > kSctLaneMaxHops)
    return fail(CCG_ERR_UNSUPPORTED, "op hops above %d are not supported by the per-lane SCT "
                "kernels (one warp per worker takes any)", kSctLaneMaxHops);
  if (p.mode == 0 && p.max_len > kSctMaxLen)
    return fail(CCG_ERR_UNSUPPORTED, "ciphertext of %lld letters exceeds the engine limit %lld",
                (long long)p.max_len, (long long)kSctMaxLen);
  if (p.mode == 1 && p.max_len > 65535)
    return fail(CCG_ERR_UNSUPPORTED, "ciphertext of %lld letters exceeds the fast-mode limit 65535",
                (long long)p.max_len);
  if (sct_lane_smem_bytes(p.mode, p.kmax, p.max_len) > 200 * 1024)
    return fail(CCG_ERR_UNSUPPORTED, "ciphertext of %lld letters does not fit the per-lane SCT "
                "kernel's shared memory", (long long)p.max_len);
  if (int rc = ctx->tickets(&p.tickets)) return rc;
  ctx->launches++;
  cudaError_t e = launch_sct_lane(ctx->stream, p, ctx->sm_count);
  if (e != cudaSuccess) return cuda_fail(e, "sct_lane kernel");
  return CCG_OK;
}

static bool sct_use_warp_family(ccg_ctx* ctx, uint32_t flags, int64_t n_workers, int64_t n_common,
                                int order, int max_hops) {
  if (flags & CCG_FLAG_SCT_KERNEL_WARP) return true;
  if (max_hops > kSctLaneMaxHops && n_common >= 0) return true;  // lane kernel's event queue
  if ((flags & CCG_FLAG_SCT_KERNEL_LANE) || n_common < 0) return false;
  // latency mode: few workers of one text length -> the speculative CTA-per-worker kernel
  if (!(flags & CCG_FLAG_SCT_NO_SPEC) && n_workers <= 16 * (int64_t)ctx->sm_count) return true;
  // one worker per lane needs ~32k workers to fill 148 SMs; below that, and for the
  // L2-resident quadgram table, one warp per worker is faster (profiles/r2_sct_*: k=10,
  // n=400 -- bigram 1.5e9 vs 1.1e9 and trigram 1.2e9 vs 0.9e9 at 65k workers, bigram 0.5e9
  // vs 1.05e9 at 16k)
  return !(order <= 3 && n_workers >= 32768);
}

// n_common: the common text length (-1: mixed lengths); max_len: the longest text; host_logs:
// the log table on the host (NULL for the _dev entry point), for the compressed trigram table
static int sct_launch(ccg_ctx* ctx, const ccg_sct_climb_args* a, int64_t n_common, int64_t max_len,
                      const double* host_logs = nullptr) {
  int rc;
  if (sct_use_warp_family(ctx, a->flags, a->n_workers, n_common, a->order == 0 ? 2 : a->order,
                          std::max(a->op1_hop, a->op2_hop))) {
    if ((rc = sct_launch_warp(ctx, a, n_common))) return rc;
  } else {
    if (max_len < a->key_length && !a->key_lengths)
      return fail(CCG_ERR_INVALID, "ciphertext shorter than the key");
    SctLaneLaunch p{};
    p.mode = 0;
    p.ciphers = a->ciphers;
    p.offsets = a->offsets;
    p.cipher_of = a->cipher_of;
    p.keys = a->keys;
    p.skips = a->skips;
    p.n_workers = a->n_workers;
    p.kmax = a->key_length;
    p.max_len = (int32_t)max_len;
    p.climbings = a->climbings;
    p.p1 = a->p1;
    p.p2 = a->p2;
    p.op1_hop = a->op1_hop;
    p.op2_hop = a->op2_hop;
    p.order = a->order == 0 ? 2 : a->order;
    p.key_lengths = a->key_lengths;
    p.logs = a->logs;
    p.scores = a->scores;
    p.keys_out = a->keys_out;
    p.draws_used = a->draws_used;
    p.last_accept = a->last_accept;
    p.tries_done = a->tries_done;
    p.flags = a->flags;
    if ((rc = attach_compressed(ctx, host_logs, p.order, p))) return rc;
    if ((rc = sct_launch_lane(ctx, p))) return rc;
  }
  if (a->group_size > 0 && a->group_best) {
    ctx->launches++;
    cudaError_t e = launch_group_best_f64(ctx->stream, a->scores, a->n_workers / a->group_size,
                                          a->group_size, a->group_best);
    if (e != cudaSuccess) return cuda_fail(e, "group_best kernel");
  }
  return CCG_OK;
}

int ccg_sct_climb_dev(ccg_ctx* ctx, const ccg_sct_climb_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if ((rc = sct_check(a))) return rc;
  if (a->n_workers == 0) return CCG_OK;
  return sct_launch(ctx, a, a->text_len, a->text_len);
}

// Host-side checks shared by ccg_sct_climb and ccg_sct_fast_climb: cipher indices, per-worker
// key lengths; returns the common text length (-1 if mixed) and the longest text.
static int sct_scan_workers(const uint8_t* ciphers, const int64_t* offsets, int64_t n_ciphers,
                            const int32_t* cipher_of, const int32_t* key_lengths, int32_t key_length,
                            int64_t nw, int64_t* n_common, int64_t* max_len) {
  int rc;
  if ((rc = check_ragged(ciphers, offsets, n_ciphers, "sct_climb", nullptr))) return rc;
  int64_t n = -2, m = 0;
  for (int64_t i = 0; i < nw; ++i) {
    const int32_t c = cipher_of[i];
    if (c < 0 || c >= n_ciphers) return fail(CCG_ERR_INVALID, "cipher_of[%lld] out of range", (long long)i);
    const int64_t L = offsets[c + 1] - offsets[c];
    if (n == -2) n = L;
    else if (L != n) n = -1;
    m = std::max(m, L);
    const int32_t kw = key_lengths ? key_lengths[i] : key_length;
    if (key_lengths) {
      if (kw < 2) return fail(CCG_ERR_INVALID, "key_length must be at least 2");
      if (kw > key_length)
        return fail(CCG_ERR_INVALID, "key_lengths[%lld] exceeds key_length", (long long)i);
    }
    if (kw > L) return fail(CCG_ERR_INVALID, "ciphertext shorter than the key");
  }
  *n_common = n < 0 ? -1 : n;
  *max_len = m;
  return CCG_OK;
}

int ccg_sct_climb(ccg_ctx* ctx, const ccg_sct_climb_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if ((rc = sct_check(a))) return rc;
  if ((rc = check_ragged(a->ciphers, a->offsets, a->n_ciphers, "sct_climb", nullptr))) return rc;
  const int64_t nw = a->n_workers;
  if (nw == 0) return CCG_OK;
  int64_t n = -1, max_len = 0;
  if ((rc = sct_scan_workers(a->ciphers, a->offsets, a->n_ciphers, a->cipher_of, a->key_lengths,
                             a->key_length, nw, &n, &max_len)))
    return rc;
  if (n < 0 && (a->flags & CCG_FLAG_SCT_KERNEL_WARP))
    return fail(CCG_ERR_INVALID, "all ciphertexts of one sct_climb call must have the same length "
                "for the warp kernel");
  ccg_sct_climb_args d = *a;
  void* p;
  const int k = a->key_length;
  if ((rc = upload(ctx, 0, a->ciphers, (size_t)a->offsets[a->n_ciphers], &p))) return rc;
  d.ciphers = (const uint8_t*)p;
  if ((rc = upload(ctx, 1, a->offsets, (size_t)(a->n_ciphers + 1) * 8, &p))) return rc;
  d.offsets = (const int64_t*)p;
  if ((rc = upload(ctx, 2, a->cipher_of, (size_t)nw * 4, &p))) return rc;
  d.cipher_of = (const int32_t*)p;
  if ((rc = upload(ctx, 3, a->keys, (size_t)nw * 16, &p))) return rc;
  d.keys = (const uint64_t*)p;
  if (a->skips) {
    if ((rc = upload(ctx, 4, a->skips, (size_t)nw * 8, &p))) return rc;
    d.skips = (const uint64_t*)p;
  }
  int64_t T = 1;
  for (int q = 0; q < (a->order == 0 ? 2 : a->order); ++q) T *= kAlpha;
  if ((rc = upload(ctx, 5, a->logs, (size_t)T * 8, &p))) return rc;
  d.logs = (const double*)p;
  if ((rc = ctx->buf(6, (size_t)nw * 8, &p))) return rc;
  d.scores = (double*)p;
  if ((rc = ctx->buf(7, (size_t)nw * k, &p))) return rc;
  d.keys_out = (uint8_t*)p;
  if (a->key_lengths) {
    if ((rc = upload(ctx, 12, a->key_lengths, (size_t)nw * 4, &p))) return rc;
    d.key_lengths = (const int32_t*)p;
  }
  if (a->draws_used) { if ((rc = ctx->buf(8, (size_t)nw * 8, &p))) return rc; d.draws_used = (uint64_t*)p; }
  if (a->last_accept) { if ((rc = ctx->buf(9, (size_t)nw * 8, &p))) return rc; d.last_accept = (int64_t*)p; }
  if (a->tries_done) { if ((rc = ctx->buf(10, (size_t)nw * 8, &p))) return rc; d.tries_done = (int64_t*)p; }
  const int64_t ng = a->group_size > 0 ? nw / a->group_size : 0;
  if (a->group_best && ng) { if ((rc = ctx->buf(11, (size_t)ng * 8, &p))) return rc; d.group_best = (int64_t*)p; }
  else d.group_best = nullptr;
  if ((rc = sct_launch(ctx, &d, n, max_len, a->logs))) return rc;
  if ((rc = download(ctx, a->scores, d.scores, (size_t)nw * 8))) return rc;
  if ((rc = download(ctx, a->keys_out, d.keys_out, (size_t)nw * k))) return rc;
  if (a->draws_used && (rc = download(ctx, a->draws_used, d.draws_used, (size_t)nw * 8))) return rc;
  if (a->last_accept && (rc = download(ctx, a->last_accept, d.last_accept, (size_t)nw * 8))) return rc;
  if (a->tries_done && (rc = download(ctx, a->tries_done, d.tries_done, (size_t)nw * 8))) return rc;
  if (d.group_best && (rc = download(ctx, a->group_best, d.group_best, (size_t)ng * 8))) return rc;
  return finish(ctx, cudaSuccess, "sct_climb");
}

// Fast mode, regular grids (ciphertext length a multiple of the worker's key length, k >= the
// n-gram order): tabulate each (ciphertext, k)'s window sums by column ranks once
// (sct_ftab_kernel), so the climb reads one entry per changed window instead of walking the
// window's column.  The integer sums are the same; other workers keep the column walk.
extern "C++" static int attach_window_tables(ccg_ctx* ctx, const ccg_sct_fast_args* a,
                                             SctLaneLaunch& L) {
  if (a->order > 3 || (a->flags & CCG_FLAG_SCT_NO_WINDOW_TABLES)) return CCG_OK;
  const int64_t nw = a->n_workers;
  std::map<std::pair<int32_t, int32_t>, int64_t> where;
  std::vector<SctFPair> pairs;
  std::vector<int64_t> foff((size_t)nw, -1);
  int64_t total = 0;
  for (int64_t i = 0; i < nw; ++i) {
    const int32_t c = a->cipher_of[i];
    const int32_t kw = a->key_lengths ? a->key_lengths[i] : a->key_length;
    const int64_t n = a->offsets[c + 1] - a->offsets[c];
    // (L = n / k >= 2: the kernel's rank = colstart * ceil(2^32 / L) >> 32 needs L > 1)
    if (kw < a->order || n % kw != 0 || n / kw < 2 || n > 40960) continue;
    int64_t entries = a->order;
    for (int q = 0; q < a->order; ++q) entries *= kw;
    if (entries > kSctFTabMaxEntries) continue;
    auto it = where.find({c, kw});
    if (it == where.end()) {
      if (total + entries > (int64_t(1) << 27)) continue;  // 512 MB of tables at most
      it = where.emplace(std::make_pair(c, kw), total).first;
      pairs.push_back(SctFPair{c, kw, total});
      total += entries;
    }
    foff[(size_t)i] = it->second;
  }
  if (pairs.empty()) return CCG_OK;
  int rc;
  void *pp, *pf, *po;
  if ((rc = upload(ctx, 20, pairs.data(), pairs.size() * sizeof(SctFPair), &pp))) return rc;
  if ((rc = ctx->buf(18, (size_t)total * 4, &pf))) return rc;
  if ((rc = upload(ctx, 19, foff.data(), foff.size() * 8, &po))) return rc;
  ctx->launches++;
  cudaError_t e = launch_sct_ftab(ctx->stream, L.ciphers, L.offsets, (const SctFPair*)pp,
                                  (int64_t)pairs.size(), L.qtable, a->order, L.max_len,
                                  (int32_t*)pf);
  if (e != cudaSuccess) return cuda_fail(e, "sct_ftab kernel");
  L.ftab = (const int32_t*)pf;
  L.f_off = (const int64_t*)po;
  return CCG_OK;
}

int ccg_sct_fast_climb(ccg_ctx* ctx, const ccg_sct_fast_args* a) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!a) return fail(CCG_ERR_INVALID, "null args");
  if ((rc = check_climb_common(a->n_workers, a->climbings, a->group_size, a->scores, a->keys,
                               a->cipher_of)))
    return rc;
  if (a->key_length < 2) return fail(CCG_ERR_INVALID, "key_length must be at least 2");
  if (a->key_length > kSctMaxKey)
    return fail(CCG_ERR_UNSUPPORTED, "key length %d exceeds the engine limit %d", a->key_length, kSctMaxKey);
  if (!(0 <= a->p1 && a->p1 <= a->p2 && a->p2 <= 100))
    return fail(CCG_ERR_INVALID, "thresholds must satisfy 0 <= p1 <= p2 <= 100");
  if (a->op1_hop < 1 || a->op2_hop < 1) return fail(CCG_ERR_INVALID, "op hops must be at least 1");
  if (a->order < 2 || a->order > 4)
    return fail(CCG_ERR_UNSUPPORTED, "n-gram order %d: the engine supports 2..4", a->order);
  if (!a->table) return fail(CCG_ERR_INVALID, "null table");
  const int64_t nw = a->n_workers;
  if (nw == 0) return CCG_OK;
  if (!a->keys_out) return fail(CCG_ERR_INVALID, "keys_out is required");
  int64_t n = -1, max_len = 0;
  if ((rc = sct_scan_workers(a->ciphers, a->offsets, a->n_ciphers, a->cipher_of, a->key_lengths,
                             a->key_length, nw, &n, &max_len)))
    return rc;
  int64_t T = 1;
  for (int q = 0; q < a->order; ++q) T *= kAlpha;
  int64_t amax = 0;
  for (int64_t i = 0; i < T; ++i) amax = std::max(amax, (int64_t)std::abs((int64_t)a->table[i]));
  const int64_t windows = max_len >= a->order ? max_len - a->order + 1 : 0;
  if (amax > 0 && windows > (int64_t)2147483647 / amax)
    return fail(CCG_ERR_UNSUPPORTED, "quantised table too coarse-scaled: %lld windows x max |entry| "
                "%lld overflow the int32 fitness (use a smaller shift)", (long long)windows,
                (long long)amax);
  void* p;
  SctLaneLaunch L{};
  L.mode = 1;
  if ((rc = upload(ctx, 0, a->ciphers, (size_t)a->offsets[a->n_ciphers], &p))) return rc;
  L.ciphers = (const uint8_t*)p;
  if ((rc = upload(ctx, 1, a->offsets, (size_t)(a->n_ciphers + 1) * 8, &p))) return rc;
  L.offsets = (const int64_t*)p;
  if ((rc = upload(ctx, 2, a->cipher_of, (size_t)nw * 4, &p))) return rc;
  L.cipher_of = (const int32_t*)p;
  if ((rc = upload(ctx, 3, a->keys, (size_t)nw * 16, &p))) return rc;
  L.keys = (const uint64_t*)p;
  if (a->skips) {
    if ((rc = upload(ctx, 4, a->skips, (size_t)nw * 8, &p))) return rc;
    L.skips = (const uint64_t*)p;
  }
  if ((rc = upload(ctx, 5, a->table, (size_t)T * 4, &p))) return rc;
  L.qtable = (const int32_t*)p;
  if ((rc = ctx->buf(6, (size_t)nw * 8, &p))) return rc;
  L.iscores = (int64_t*)p;
  const int k = a->key_length;
  if ((rc = ctx->buf(7, (size_t)nw * k, &p))) return rc;
  L.keys_out = (uint8_t*)p;
  if (a->key_lengths) {
    if ((rc = upload(ctx, 12, a->key_lengths, (size_t)nw * 4, &p))) return rc;
    L.key_lengths = (const int32_t*)p;
  }
  if (a->draws_used) { if ((rc = ctx->buf(8, (size_t)nw * 8, &p))) return rc; L.draws_used = (uint64_t*)p; }
  if (a->last_accept) { if ((rc = ctx->buf(9, (size_t)nw * 8, &p))) return rc; L.last_accept = (int64_t*)p; }
  if (a->tries_done) { if ((rc = ctx->buf(10, (size_t)nw * 8, &p))) return rc; L.tries_done = (int64_t*)p; }
  if (a->lookups) { if ((rc = ctx->buf(13, (size_t)nw * 8, &p))) return rc; L.lookups = (int64_t*)p; }
  const int64_t ng = a->group_size > 0 ? nw / a->group_size : 0;
  int64_t* d_best = nullptr;
  if (a->group_best && ng) { if ((rc = ctx->buf(11, (size_t)ng * 8, &p))) return rc; d_best = (int64_t*)p; }
  L.n_workers = nw;
  L.kmax = k;
  L.max_len = (int32_t)max_len;
  L.climbings = a->climbings;
  L.p1 = a->p1;
  L.p2 = a->p2;
  L.op1_hop = a->op1_hop;
  L.op2_hop = a->op2_hop;
  L.order = a->order;
  L.flags = a->flags;
  if ((rc = attach_compressed(ctx, a->table, a->order, L))) return rc;
  if ((rc = attach_window_tables(ctx, a, L))) return rc;
  if ((rc = sct_launch_lane(ctx, L))) return rc;
  if (d_best) {
    ctx->launches++;
    cudaError_t e = launch_group_best_i64(ctx->stream, L.iscores, ng, a->group_size, d_best);
    if (e != cudaSuccess) return cuda_fail(e, "group_best kernel");
  }
  if ((rc = download(ctx, a->scores, L.iscores, (size_t)nw * 8))) return rc;
  if ((rc = download(ctx, a->keys_out, L.keys_out, (size_t)nw * k))) return rc;
  if (a->draws_used && (rc = download(ctx, a->draws_used, L.draws_used, (size_t)nw * 8))) return rc;
  if (a->last_accept && (rc = download(ctx, a->last_accept, L.last_accept, (size_t)nw * 8))) return rc;
  if (a->tries_done && (rc = download(ctx, a->tries_done, L.tries_done, (size_t)nw * 8))) return rc;
  if (a->lookups && (rc = download(ctx, a->lookups, L.lookups, (size_t)nw * 8))) return rc;
  if (d_best && (rc = download(ctx, a->group_best, d_best, (size_t)ng * 8))) return rc;
  return finish(ctx, cudaSuccess, "sct_fast_climb");
}

// ------------------------------------------------------------------ test-set generation
int ccg_encrypt_batch(ccg_ctx* ctx, int32_t kind, const uint8_t* texts, const int64_t* offsets,
                      int64_t n_texts, const uint64_t* keygen, const int32_t* key_lengths,
                      int32_t kmax, uint8_t* keys, uint8_t* out) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (kind != 0 && kind != 1) return fail(CCG_ERR_INVALID, "kind must be 0 (MAS) or 1 (SCT)");
  if ((rc = check_ragged(texts, offsets, n_texts, "encrypt", nullptr))) return rc;
  if (n_texts == 0) return CCG_OK;
  if (!keys || !out) return fail(CCG_ERR_INVALID, "null keys / out");
  if (kind == 0 && kmax < kAlpha) return fail(CCG_ERR_INVALID, "kmax must be >= 26 for MAS");
  if (kind == 1 && !key_lengths) return fail(CCG_ERR_INVALID, "key_lengths required for SCT");
  for (int64_t i = 0; i < n_texts; ++i) {
    const int k = kind == 0 ? kAlpha : key_lengths[i];
    if (k < 1 || k > kmax || k > kSctMaxKey)
      return fail(CCG_ERR_INVALID, "key length %d of text %lld out of range", k, (long long)i);
    if (!keygen) {
      uint64_t seen = 0;
      for (int q = 0; q < k; ++q) {
        const int v = keys[i * kmax + q];
        if (v >= k || (seen >> v) & 1)
          return fail(CCG_ERR_INVALID, kind == 0 ? "substitution key must be a permutation of 0..25"
                                                 : "transposition key must be a permutation of 0..k-1");
        seen |= 1ULL << v;
      }
    }
  }
  const size_t total = (size_t)offsets[n_texts];
  void *dt, *doff, *dkg = nullptr, *dkl = nullptr, *dkeys, *dout;
  if ((rc = upload(ctx, 0, texts, total, &dt))) return rc;
  if ((rc = upload(ctx, 1, offsets, (size_t)(n_texts + 1) * 8, &doff))) return rc;
  if (keygen && (rc = upload(ctx, 2, keygen, (size_t)n_texts * 16, &dkg))) return rc;
  if (key_lengths && (rc = upload(ctx, 3, key_lengths, (size_t)n_texts * 4, &dkl))) return rc;
  if (keygen) {
    if ((rc = ctx->buf(4, (size_t)n_texts * kmax, &dkeys))) return rc;
  } else if ((rc = upload(ctx, 4, keys, (size_t)n_texts * kmax, &dkeys))) {
    return rc;
  }
  if ((rc = ctx->buf(5, total ? total : 1, &dout))) return rc;
  ctx->launches++;
  cudaError_t e = launch_encrypt(ctx->stream, kind, (const uint8_t*)dt, (const int64_t*)doff,
                                 n_texts, (const uint64_t*)dkg, (const int32_t*)dkl,
                                 (uint8_t*)dkeys, kmax, (uint8_t*)dout);
  if (e != cudaSuccess) return cuda_fail(e, "encrypt kernel");
  if (keygen && (rc = download(ctx, keys, dkeys, (size_t)n_texts * kmax))) return rc;
  if ((rc = download(ctx, out, dout, total))) return rc;
  return finish(ctx, cudaSuccess, "encrypt");
}

int ccg_bench_smem_bandwidth(ccg_ctx* ctx, double* out_bytes_per_s) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!out_bytes_per_s) return fail(CCG_ERR_INVALID, "null out");
  ctx->launches += 2;
  cudaError_t e = bench_smem_bandwidth(ctx->stream, ctx->sm_count, out_bytes_per_s);
  if (e != cudaSuccess) return cuda_fail(e, "smem bandwidth kernel");
  return CCG_OK;
}

int ccg_bench_l2_gather(ccg_ctx* ctx, int64_t table_entries, double* out_gathers_per_s) {
  int rc = enter(ctx);
  if (rc) return rc;
  if (!out_gathers_per_s || table_entries < 1 || table_entries > (int64_t)1 << 31)
    return fail(CCG_ERR_INVALID, "bad arguments");
  ctx->launches += 2;
  cudaError_t e = bench_l2_gather(ctx->stream, ctx->sm_count, table_entries, out_gathers_per_s);
  if (e != cudaSuccess) return cuda_fail(e, "L2 gather kernel");
  return CCG_OK;
}

}  // extern "C"
