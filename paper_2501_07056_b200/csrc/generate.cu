// Seeded synthetic inputs on the device (setup only, not the SpGEMM path).
// Bit-identical to paper_2501_07056_b200/generate.py: the same counter-based
// splitmix64 hash of (seed, stream, index) drives both.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/magnus_gen.h"

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t hash3(uint64_t key, uint64_t idx) { return mix64(idx ^ key); }

__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

uint64_t stream_key(uint64_t seed, uint64_t stream) { return mix64(seed ^ (stream << 48)); }

struct LevelKeys {
  uint64_t k[40];
};

__global__ void k_rmat_keys(int scale, int64_t lo, int64_t m, LevelKeys keys, double a, double ab, double abc,
                            uint64_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t e = (uint64_t)(lo + t);
    uint64_t r = 0, c = 0;
    for (int l = 0; l < scale; ++l) {
      const double u = u01(hash3(keys.k[l], e));
      const uint64_t rb = u >= ab;
      const uint64_t cb = (u >= a && u < ab) || (u >= abc);
      r = (r << 1) | rb;
      c = (c << 1) | cb;
    }
    out[t] = (r << scale) | c;
  }
}

__global__ void k_pm1(uint64_t key, int64_t n, double* __restrict__ out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = 2.0 * u01(hash3(key, (uint64_t)p)) - 1.0;
}

// Floyd sampling of d distinct columns per row, sorted (d <= 64).
__global__ void k_uniform_rows(int64_t n_rows, int64_t n_cols, int d, uint64_t key, int32_t* __restrict__ col) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t ch[64];
    for (int s = 0; s < d; ++s) {
      const int64_t j = n_cols - d + s;
      const uint64_t h = hash3(key, (uint64_t)r * (uint64_t)d + (uint64_t)s);
      const int64_t t = (int64_t)(h % (uint64_t)(j + 1));
      bool dup = false;
      for (int q = 0; q < s; ++q) dup |= ch[q] == t;
      ch[s] = dup ? j : t;
    }
    for (int s = 1; s < d; ++s) {  // insertion sort
      const int64_t v = ch[s];
      int q = s - 1;
      while (q >= 0 && ch[q] > v) { ch[q + 1] = ch[q]; --q; }
      ch[q + 1] = v;
    }
    for (int s = 0; s < d; ++s) col[r * d + s] = (int32_t)ch[s];
  }
}

unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (unsigned)(g < 148 * 64 ? (g < 1 ? 1 : g) : 148 * 64);
}

}  // namespace

extern "C" {

int magnus_gen_rmat_keys(int scale, int64_t lo, int64_t m, uint64_t seed, double a, double b, double c, uint64_t* out,
                         void* stream) {
  if (scale < 1 || scale > 31 || m < 0) return 1;
  LevelKeys keys;
  for (int l = 0; l < scale; ++l) keys.k[l] = stream_key(seed, (uint64_t)l);
  const double ab = a + b, abc = a + b + c;
  if (m) k_rmat_keys<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(scale, lo, m, keys, a, ab, abc, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int magnus_gen_uniform_pm1(uint64_t seed, uint64_t stream_id, int64_t n, double* out, void* stream) {
  if (n) k_pm1<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(stream_key(seed, stream_id), n, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

int magnus_gen_uniform_rows(int64_t n_rows, int64_t n_cols, int d, uint64_t seed, int32_t* col, void* stream) {
  if (d < 1 || d > 64 || d > n_cols) return 1;
  if (n_rows)
    k_uniform_rows<<<grid_for(n_rows), 256, 0, (cudaStream_t)stream>>>(n_rows, n_cols, d, stream_key(seed, 0xFE), col);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
