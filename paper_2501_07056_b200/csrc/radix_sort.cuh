// Stable LSD radix sort of (64-bit key, position) pairs on the device: the sort step of the
// sort accumulator's whole-stream microbenchmark (reference bench.py:160-180, np.argsort
// kind="stable") and, optionally, of the ESC baseline.  8-bit digits; per pass: tile
// histograms -> one exclusive scan over (digit, tile) -> stable scatter (warps own contiguous
// pieces of a tile, lanes of a wave are ranked in lane order by match_any).
#pragma once
#include "common.cuh"

namespace mg {

constexpr int kRsT = 256;                 // threads per CTA
constexpr int kRsItems = 8;               // keys per thread
constexpr int kRsTile = kRsT * kRsItems;  // keys per tile
constexpr int kRsW = kRsT / 32;

// hist[d * ntiles + tile] = keys of the tile with digit d
__global__ void __launch_bounds__(kRsT) k_rs_hist(const uint64_t* __restrict__ keys, int64_t n, int shift, int64_t ntiles,
                                                   int64_t* __restrict__ hist) {
  __shared__ uint32_t cnt[256];
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    cnt[threadIdx.x] = 0u;
    __syncthreads();
    const int64_t base = tile * kRsTile;
#pragma unroll
    for (int j = 0; j < kRsItems; ++j) {
      const int64_t q = base + (int64_t)j * kRsT + threadIdx.x;
      if (q < n) atomicAdd(&cnt[(uint32_t)(__ldg(keys + q) >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + tile] = (int64_t)cnt[threadIdx.x];
    __syncthreads();
  }
}

// Stable scatter of one pass.  perm_in == nullptr: the identity (first pass).
__global__ void __launch_bounds__(kRsT) k_rs_scatter(const uint64_t* __restrict__ keys, const int64_t* __restrict__ perm_in,
                                                      int64_t n, int shift, int64_t ntiles, const int64_t* __restrict__ base,
                                                      uint64_t* __restrict__ keys_out, int64_t* __restrict__ perm_out) {
  __shared__ uint32_t wcnt[kRsW][256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int q = threadIdx.x; q < kRsW * 256; q += kRsT) (&wcnt[0][0])[q] = 0u;
    __syncthreads();
    // warp wid owns keys [tile * kRsTile + wid * 256, + 256): kRsItems waves of 32 consecutive keys
    const int64_t w0 = tile * kRsTile + (int64_t)wid * (32 * kRsItems);
    uint64_t k[kRsItems];
    int64_t p[kRsItems];
    uint32_t off[kRsItems];
#pragma unroll
    for (int j = 0; j < kRsItems; ++j) {
      const int64_t q = w0 + j * 32 + lane;
      const bool valid = q < n;
      k[j] = valid ? __ldg(keys + q) : 0ull;
      p[j] = valid ? (perm_in != nullptr ? __ldg(perm_in + q) : q) : 0;
      const uint32_t d = valid ? (uint32_t)(k[j] >> shift) & 255u : 256u + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t rank = __popc(peers & lt);
      uint32_t old = 0;
      if (valid) old = wcnt[wid][d];
      __syncwarp();
      if (valid && rank == 0) wcnt[wid][d] = old + __popc(peers);
      __syncwarp();
      off[j] = old + rank;
    }
    __syncthreads();
    {
      // exclusive prefix over the warps, per digit (thread = digit)
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kRsW; ++w) {
        const uint32_t v = wcnt[w][threadIdx.x];
        wcnt[w][threadIdx.x] = run;
        run += v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRsItems; ++j) {
      const int64_t q = w0 + j * 32 + lane;
      if (q < n) {
        const uint32_t d = (uint32_t)(k[j] >> shift) & 255u;
        const int64_t dst = __ldg(base + (int64_t)d * ntiles + tile) + wcnt[wid][d] + off[j];
        keys_out[dst] = k[j];
        perm_out[dst] = p[j];
      }
    }
    __syncthreads();
  }
}

}  // namespace mg
