// ccg_testset.cu -- device-side test-set generation for ragged batches:
// key generation WorkerRng(seed, KEYGEN_STREAM).permutation(k) (rng.py:91-97, the recipe of
// the reference's acceptance tests, tests/test_acceptance.py:152,177) and encryption,
// mas_encrypt (ciphers.py:46-49) or sct_encrypt (ciphers.py:89-104, irregular grid:
// ciphertext segment j is grid column key[j], columns c < n % k hold ceil(n/k) letters).
//
// One warp per text: lane 0 runs the Fisher-Yates draws (k - 1 numpy-exact Philox draws),
// the warp scans the segment lengths and scatters the letters.
#include "ccg_internal.h"
#include "ccg_rng.cuh"

namespace ccg {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;

__global__ void encrypt_kernel(int kind, const uint8_t* __restrict__ texts,
                               const int64_t* __restrict__ offsets, int64_t n_texts,
                               const uint64_t* __restrict__ keygen,
                               const int32_t* __restrict__ key_lengths, uint8_t* keys, int kmax,
                               uint8_t* __restrict__ out) {
  __shared__ int key_s[4][64];
  __shared__ int colstart_s[4][64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= n_texts) return;
  const int k = kind == 0 ? kAlpha : key_lengths[j];
  int* key = key_s[wib];
  if (keygen) {
    if (lane == 0) {  // rng.py:91-97: i = k-1 .. 1, j = int(u * (i + 1)), swap
      for (int i = 0; i < k; ++i) key[i] = i;
      const uint64_t k0 = keygen[2 * j], k1 = keygen[2 * j + 1];
      uint64_t blk[4];
      uint64_t drawn = 0;
      for (int i = k - 1; i > 0; --i) {
        if ((drawn & 3) == 0) philox4x64_10(k0, k1, (drawn >> 2) + 1, blk[0], blk[1], blk[2], blk[3]);
        const int r = (int)int_below_small(blk[drawn & 3], (uint32_t)(i + 1));
        ++drawn;
        const int tmp = key[i];
        key[i] = key[r];
        key[r] = tmp;
      }
    }
    __syncwarp();
    for (int i = lane; i < k; i += 32) keys[j * kmax + i] = (uint8_t)key[i];
  } else {
    for (int i = lane; i < k; i += 32) key[i] = keys[j * kmax + i];
  }
  __syncwarp();
  const int64_t off = offsets[j], n = offsets[j + 1] - off;
  const uint8_t* plain = texts + off;
  uint8_t* cipher = out + off;
  if (kind == 0) {
    for (int64_t i = lane; i < n; i += 32) cipher[i] = (uint8_t)key[plain[i]];
    return;
  }
  // colstart[key[s]] = sum of segment lengths s' < s (key order)
  const int64_t base = n / k, rem = n - base * k;
  if (lane == 0) {
    int64_t acc = 0;
    for (int s = 0; s < k; ++s) {
      const int c = key[s];
      colstart_s[wib][c] = (int)acc;
      acc += base + (c < rem ? 1 : 0);
    }
  }
  __syncwarp();
  // plaintext position t = c + k r goes to ciphertext position colstart[c] + r
  for (int64_t t = lane; t < n; t += 32) {
    const int64_t r = t / k, c = t - r * k;
    cipher[colstart_s[wib][c] + r] = plain[t];
  }
}

}  // namespace

cudaError_t launch_encrypt(cudaStream_t s, int kind, const uint8_t* texts, const int64_t* offsets,
                           int64_t n, const uint64_t* keygen, const int32_t* key_lengths,
                           uint8_t* keys, int kmax, uint8_t* out) {
  if (n <= 0) return cudaSuccess;
  const int64_t threads = n * 32;
  encrypt_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(kind, texts, offsets, n, keygen,
                                                                   key_lengths, keys, kmax, out);
  return cudaGetLastError();
}

}  // namespace ccg
