// Setup-phase kernels: row statistics, categorisation / binning, device-wide scan.
#pragma once
#include "common.cuh"

namespace mg {

// row_intermediate_stats (reference gustavson.py:97-134): a group of G lanes per row (G = 32,
// or 8 for matrices with short rows: four rows per warp).  inter[i] = sum of nnz(B_k) over k
// in A_i; [min_col, max_col] spans the first / last column of every referenced non-empty B
// row; empty product -> (0, 0, -1).
template <int G>
__global__ void k_row_stats(DevCsr A, DevCsr B, int64_t* __restrict__ inter, int64_t* __restrict__ mn,
                            int64_t* __restrict__ mx) {
  const int gl = threadIdx.x & (G - 1);
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t iters = (A.n_rows + ngrp - 1) / ngrp;   // every lane runs the same trip count (shuffles)
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = grp + it * ngrp;
    const bool row = i < A.n_rows;
    const int64_t a0 = row ? A.rp(i) : 0, a1 = row ? A.rp(i + 1) : 0;
    int64_t s = 0, lo = INT64_MAX, hi = -1;
    for (int64_t t = a0 + gl; t < a1; t += G) {
      const int64_t k = __ldg(A.col + t);
      const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
      s += b1 - b0;
      if (b1 > b0) {
        const int64_t f = __ldg(B.col + b0), l = __ldg(B.col + b1 - 1);
        lo = f < lo ? f : lo;
        hi = l > hi ? l : hi;
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      int64_t l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
      lo = l2 < lo ? l2 : lo;
      hi = h2 > hi ? h2 : hi;
    }
    if (gl == 0 && row) {
      inter[i] = s;
      mn[i] = s > 0 ? lo : 0;
      mx[i] = s > 0 ? hi : -1;
    }
  }
}

// Input contract of the device path, checked before any kernel indexes through the
// inputs (validate_csr matrix.py:119-150; magnus.py:208-209, 245-246 raise
// ContractViolation for columns outside the planned span).  One warp per row, lanes over
// adjacent pairs (coalesced).  flags: 1 = row_ptr not monotone / row_ptr[0] != 0 /
// row_ptr[n] != nnz, 2 = column >= n_cols, 4 = columns not strictly increasing in a row
// (unsorted or duplicate columns: the device kernels require canonical rows).
template <int G>
__global__ void k_validate(DevCsr M, unsigned long long* __restrict__ flags) {
  const int lane = threadIdx.x & 31, gl = threadIdx.x & (G - 1);
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  const uint64_t ncols = (uint64_t)M.n_cols;
  unsigned f = 0;
  if (grp == 0 && gl == 0) {
    if (M.rp(0) != 0 || M.rp(M.n_rows) != M.nnz) f |= 1u;
  }
  for (int64_t i = grp; i < M.n_rows; i += ngrp) {
    const int64_t a0 = M.rp(i), a1 = M.rp(i + 1);
    if (a1 < a0 || a0 < 0 || a1 > M.nnz) {
      f |= 1u;
      continue;
    }
    for (int64_t t = a0 + gl; t < a1; t += G) {
      const uint32_t c = __ldg(M.col + t);
      if ((uint64_t)c >= ncols) f |= 2u;
      if (t + 1 < a1 && __ldg(M.col + t + 1) <= c) f |= 4u;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (lane == 0 && f) atomicOr(flags, (unsigned long long)f);
}

// Device row classes (execution strategy only; results never depend on them).
constexpr int kClsNone = -1, kClsWarp = 0, kClsBlock = 1, kClsHeavy = 2;
constexpr int64_t kWarpMax = 256;    // <= 256 intermediate elements: one warp, smem bitonic
#ifndef MG_BLOCK_MAX
#define MG_BLOCK_MAX 4096
#endif
constexpr int64_t kBlockMax = MG_BLOCK_MAX;  // <= kBlockMax products: one CTA per row (smem merge)

struct CatParams {
  int64_t crossover;   // sort_dense_crossover
  int64_t l2_bytes;    // SystemParams.l2_bytes
  int64_t val_bytes;   // SystemParams.val_bytes
  int32_t use_coarse;  // symbolic ChunkPlan.use_coarse
};

// stats layout (int64): [0..3] rows per category, [4] sum inter, [5] max nk of heavy rows,
// [6] nW, [7] nB, [8] nH, [9] error flag, [10] n coarse rows
constexpr int kStatCat = 0, kStatInter = 4, kStatMaxNk = 5, kStatNW = 6, kStatNB = 7, kStatNH = 8, kStatErr = 9,
              kStatNCoarse = 10, kStatND = 11, kStatLen = 16;
// dense-category rows handled warp-per-row without sorting (dense_rows.cuh)
constexpr int64_t kDenseRangeMax = 32768, kDenseInterMax = 1024;

// categorize_rows (reference magnus.py:68-94): first matching rule wins.
// Also bins rows into the device execution classes and lists coarse rows.  Counters and
// list appends are warp-aggregated (one atomic per warp and counter: millions of rows).
__device__ __forceinline__ void warp_append(bool flag, int32_t value, int32_t* __restrict__ list,
                                            unsigned long long* __restrict__ count) {
  const uint32_t m = __ballot_sync(0xffffffffu, flag);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  unsigned long long b = 0;
  if (lane == 0) b = atomicAdd(count, (unsigned long long)__popc(m));
  b = __shfl_sync(0xffffffffu, b, 0);
  if (flag) list[b + __popc(m & ((1u << lane) - 1u))] = value;
}

__global__ void k_categorize(int64_t n, DevCsr A, const int64_t* __restrict__ inter, const int64_t* __restrict__ mn,
                             const int64_t* __restrict__ mx, CatParams p, int8_t* __restrict__ cat,
                             int32_t* __restrict__ listW, int32_t* __restrict__ listB, int32_t* __restrict__ listH,
                             int32_t* __restrict__ listCoarse, int32_t* __restrict__ listD,
                             unsigned long long* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long ccount[4] = {0, 0, 0, 0}, isum = 0, maxnk = 0;
  for (int64_t base = w0; base < n; base += stride) {
    const int64_t i = base + lane;
    const bool valid = i < n;
    int64_t s = 0;
    int c = -1;
    if (valid) {
      s = inter[i];
      const int64_t range = mx[i] - mn[i] + 1;
      if (s < p.crossover) c = kCatSort;
      else if (range * (p.val_bytes + 1) <= p.l2_bytes) c = kCatDense;
      else c = p.use_coarse ? kCatCoarse : kCatFine;
      cat[i] = (int8_t)c;
#pragma unroll
      for (int q = 0; q < 4; ++q) ccount[q] += c == q ? 1ull : 0ull;
      isum += (unsigned long long)s;
    }
    warp_append(c == kCatCoarse, (int32_t)i, listCoarse, &stats[kStatNCoarse]);
    const bool any = valid && s > 0;
    const bool isD = any && c == kCatDense && (mx[i] - mn[i] + 1) <= kDenseRangeMax && s <= kDenseInterMax;
    const bool isW = any && !isD && s <= kWarpMax;
    const bool isB = any && !isD && !isW && s <= kBlockMax;
    const bool isH = any && !isD && !isW && !isB;
    warp_append(isD, (int32_t)i, listD, &stats[kStatND]);
    warp_append(isW, (int32_t)i, listW, &stats[kStatNW]);
    warp_append(isB, (int32_t)i, listB, &stats[kStatNB]);
    warp_append(isH, (int32_t)i, listH, &stats[kStatNH]);
    if (isH) maxnk = max(maxnk, (unsigned long long)(A.rp(i + 1) - A.rp(i)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < 4; ++q) ccount[q] += __shfl_xor_sync(0xffffffffu, ccount[q], o);
    isum += __shfl_xor_sync(0xffffffffu, isum, o);
    maxnk = max(maxnk, __shfl_xor_sync(0xffffffffu, maxnk, o));
  }
  if (lane == 0) {
    for (int q = 0; q < 4; ++q)
      if (ccount[q]) atomicAdd(&stats[kStatCat + q], ccount[q]);
    if (isum) atomicAdd(&stats[kStatInter], isum);
    if (maxnk) atomicMax(&stats[kStatMaxNk], maxnk);
  }
}

// heavy rows (> kBlockMax products) in ascending row order: flags for an exclusive scan ...
__global__ void k_heavy_flags(const int64_t* __restrict__ inter, int64_t n, int64_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = inter[i] > kBlockMax ? 1 : 0;
}
// ... and the scatter to the scanned positions
__global__ void k_heavy_scatter(const int64_t* __restrict__ inter, const int64_t* __restrict__ pos, int64_t n,
                                int32_t* __restrict__ listH) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (inter[i] > kBlockMax) listH[pos[i]] = (int32_t)i;
}

// skip list of B: skip[j] = col[32*j]
__global__ void k_build_skip(const uint32_t* __restrict__ col, int64_t nnz, uint32_t* __restrict__ skip) {
  const int64_t n = (nnz + 31) / 32;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    skip[j] = __ldg(col + 32 * j);
}

// ---------------------------------------------------------------- device-wide exclusive scan (int64)
constexpr int kScanT = 512, kScanItems = 16, kScanTile = kScanT * kScanItems;

__global__ void k_scan_reduce(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ tile_sums) {
  __shared__ int64_t sh[kScanT / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t s = 0;
  for (int j = 0; j < kScanItems; ++j) {
    int64_t idx = base + (int64_t)j * kScanT + threadIdx.x;
    if (idx < n) s += in[idx];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kScanT / 32; ++w) t += sh[w];
    tile_sums[blockIdx.x] = t;
  }
}

// exclusive scan of tile sums in place (single block, any count)
__global__ void k_scan_tiles(int64_t* __restrict__ tile_sums, int64_t ntiles) {
  __shared__ int64_t sh[33];
  int64_t carry = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    int64_t idx = base + threadIdx.x;
    int64_t v = idx < ntiles ? tile_sums[idx] : 0;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      int64_t w = lane < (int)(blockDim.x / 32) ? sh[lane] : 0;
      int64_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      if (lane < (int)(blockDim.x / 32)) sh[lane] = wi - w;
      if (lane == 31) sh[32] = wi;
    }
    __syncthreads();
    if (idx < ntiles) tile_sums[idx] = carry + sh[wid] + inc - v;
    carry += sh[32];
    __syncthreads();
  }
}

// out[i] = exclusive prefix of in (out has n+1 entries; out[n] = total)
__global__ void k_scan_apply(const int64_t* __restrict__ in, int64_t n, const int64_t* __restrict__ tile_sums,
                             int64_t* __restrict__ out) {
  __shared__ int64_t sh[33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    int64_t idx = base + j;
    v[j] = idx < n ? in[idx] : 0;
    s += v[j];
  }
  int64_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < kScanT / 32 ? sh[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kScanT / 32) sh[lane] = wi - w;
  }
  __syncthreads();
  int64_t run = tile_sums[blockIdx.x] + sh[wid] + inc - s;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    int64_t idx = base + j;
    if (idx < n) out[idx] = run;
    run += v[j];
    if (idx == n - 1) out[n] = run;
  }
}

// out[j] = v[idx[j]] (the coarse rows' intermediate sizes for build_coarse_batches)
__global__ void k_gather_i64(const int64_t* __restrict__ v, const int32_t* __restrict__ idx, int64_t n,
                             int64_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = v[idx[j]];
}

}  // namespace mg
