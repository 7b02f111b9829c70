// Building-block microbenchmarks on the device (reference bench.py:88-196): the stages of
// single-level locality generation over one synthetic intermediate-product stream
// (u32 index < length, f64 value), each a kernel of its own so it can be timed and
// ncu-profiled in isolation:
//   k_mb_hist        chunk occupancy counts (index >> shift): shared-memory histogram per CTA
//   k_mb_tile_hist   reorder pass 1: per-tile (one warp, kMbTile elements) chunk counts, stored
//                    chunk-major so one exclusive scan (k_scan_*) gives every (chunk, tile) its slot
//   k_mb_scatter     reorder pass 2: stable scatter (ties keep stream order: waves in order,
//                    match_any ranks inside a wave) of (index & (len-1), value) into chunk order
//   k_mb_dense       per-chunk dense accumulation in shared memory, strictly sequential from
//                    +0.0 in slice order (DenseAccumulator), emitted ascending at the slice start
//   k_mb_stream      contiguous 128-bit copy of both arrays (the peak-rate baseline)
// The sort accumulator stage reuses the ESC compress kernels (baselines.cuh) after a stable
// sort of the reordered stream.
#pragma once
#include "common.cuh"

namespace mg {

constexpr int kMbTile = 2048;         // reorder tile: elements per warp
constexpr int kMbWarps = 4;           // warps (tiles) per CTA
constexpr int kMbMaxChunks = 4096;    // reorder: per-warp cursors in shared memory

__global__ void k_mb_hist(const uint32_t* __restrict__ idx, int64_t n, int shift, int nch,
                          unsigned long long* __restrict__ counts) {
  extern __shared__ uint32_t h[];
  for (int c = threadIdx.x; c < nch; c += blockDim.x) h[c] = 0u;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(h + (__ldg(idx + i) >> shift), 1u);
  __syncthreads();
  for (int c = threadIdx.x; c < nch; c += blockDim.x)
    if (h[c]) atomicAdd(counts + c, (unsigned long long)h[c]);
}

__global__ void __launch_bounds__(kMbWarps * 32)
k_mb_tile_hist(const uint32_t* __restrict__ idx, int64_t n, int shift, int nch, int64_t ntiles,
               int64_t* __restrict__ tcount) {
  extern __shared__ uint32_t sh[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t* cnt = sh + (size_t)w * nch;
  const int64_t tile = (int64_t)blockIdx.x * kMbWarps + w;
  for (int c = lane; c < nch; c += 32) cnt[c] = 0u;
  __syncwarp();
  if (tile < ntiles) {
    const int64_t e = min(n, (tile + 1) * kMbTile);
    for (int64_t i = tile * kMbTile + lane; i < e; i += 32) atomicAdd(cnt + (__ldg(idx + i) >> shift), 1u);
    __syncwarp();
    for (int c = lane; c < nch; c += 32) tcount[(int64_t)c * ntiles + tile] = cnt[c];
  }
}

__global__ void __launch_bounds__(kMbWarps * 32)
k_mb_scatter(const uint32_t* __restrict__ idx, const double* __restrict__ val, int64_t n, int shift, int nch,
             int64_t ntiles, const int64_t* __restrict__ toff, uint32_t* __restrict__ ocol,
             double* __restrict__ oval) {
  extern __shared__ uint32_t sh[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t* cur = sh + (size_t)w * nch;
  const int64_t tile = (int64_t)blockIdx.x * kMbWarps + w;
  if (tile >= ntiles) return;
  for (int c = lane; c < nch; c += 32) cur[c] = (uint32_t)toff[(int64_t)c * ntiles + tile];
  __syncwarp();
  const uint32_t mask = (1u << shift) - 1u, lt = (1u << lane) - 1u;
  const int64_t b = tile * kMbTile, e = min(n, b + kMbTile);
  for (int64_t i0 = b; i0 < e; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool v = i < e;
    const uint32_t x = v ? __ldg(idx + i) : 0u;
    const uint32_t c = v ? x >> shift : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, c);
    const uint32_t base = v ? cur[c] : 0u;
    __syncwarp();
    if (v) {
      const uint32_t slot = base + __popc(peers & lt);
      if ((peers >> lane) == 1u) cur[c] = base + __popc(peers);   // highest peer advances the cursor
      ocol[slot] = x & mask;
      oval[slot] = __ldg(val + i);
    }
    __syncwarp();
  }
}

// one warp per chunk; shared memory: chunk_len doubles + chunk_len bits + 32 staged values
__global__ void __launch_bounds__(32)
k_mb_dense(const uint32_t* __restrict__ col, const double* __restrict__ val, const int64_t* __restrict__ off,
           int nch, int chunk_len, uint32_t* __restrict__ ocol, double* __restrict__ oval,
           int64_t* __restrict__ distinct) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* acc = reinterpret_cast<double*>(smem);
  uint32_t* bm = reinterpret_cast<uint32_t*>(acc + chunk_len);
  double* stage = reinterpret_cast<double*>(bm + ((chunk_len + 63) / 64) * 2);
  const int lane = threadIdx.x;
  const int nw = (chunk_len + 31) / 32;
  const int c = blockIdx.x;
  for (int i = lane; i < nw; i += 32) bm[i] = 0u;
  __syncwarp();
  const int64_t s0 = off[c], s1 = off[c + 1];
  for (int64_t i0 = s0; i0 < s1; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool v = i < s1;
    const uint32_t x = v ? col[i] : 0xffffffffu;
    stage[lane] = v ? val[i] : 0.0;
    const uint32_t peers = __match_any_sync(0xffffffffu, x);
    __syncwarp();
    if (v && (peers & ((1u << lane) - 1u)) == 0u) {   // lowest peer applies the run in stream order
      const uint32_t bit = 1u << (x & 31u);
      double s = (bm[x >> 5] & bit) ? acc[x] : 0.0;
      for (uint32_t m = peers; m; m &= m - 1u) s = __dadd_rn(s, stage[__ffs(m) - 1]);
      acc[x] = s;
      atomicOr(bm + (x >> 5), bit);
    }
    __syncwarp();
  }
  // emit ascending at the slice start
  uint32_t run = 0;
  for (int w0 = 0; w0 < nw; w0 += 32) {
    const uint32_t word = w0 + lane < nw ? bm[w0 + lane] : 0u;
    const uint32_t cnt = __popc(word);
    const uint32_t inc = warp_incl_scan(cnt);
    uint32_t pos = run + inc - cnt;
    for (uint32_t m = word; m; m &= m - 1u) {
      const uint32_t x = ((uint32_t)(w0 + lane) << 5) + (__ffs(m) - 1);
      ocol[s0 + pos] = x;
      oval[s0 + pos] = acc[x];
      ++pos;
    }
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) distinct[c] = run;
}

__global__ void k_mb_stream(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    __stcs(dst + i, __ldcs(src + i));
}

}  // namespace mg
