// Dense-category rows with a narrow column range (reference categorize_rows rule 2,
// magnus.py:79-81: the row's window fits the cache) -- all of cfg1 and cfg2.
//
// The reference accumulates such a row in a dense window, sequentially in
// ascending k from +0.0 (dense_accumulate, accumulators.py:68-97).  One warp per
// row does exactly that, with no sorting: the row's columns are marked in a
// shared-memory bitmap over its [min_col, max_col] range, compacted to ranks
// (word prefix + popcount), and the B rows are then applied one k at a time:
// inside one B row the columns are distinct, so the 32 lanes update distinct
// rank slots in parallel, and successive k's are ordered by the warp's program
// order.  The sorted output falls out of the bitmap order.
#pragma once
#include "common.cuh"

namespace mg {

constexpr int kDT = 256;                 // threads per CTA (8 warps, one row each)
constexpr int kDRange = 32768;           // max column range (bitmap 4 KB per warp)
constexpr int kDInter = 1024;            // max intermediate elements (>= distinct columns)
constexpr int kDWords = kDRange / 32;
struct DenseRowSmem {
  static constexpr size_t kPerWarp = (size_t)kDWords * 4 + (size_t)kDWords * 2 + (size_t)kDInter * 8;   // 14 KB
  static constexpr size_t kTotal = kPerWarp * (kDT / 32);
};

template <bool Numeric>
__global__ void __launch_bounds__(kDT, 2)
k_rows_dense(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows, const int64_t* __restrict__ mn,
             const int64_t* __restrict__ mx, int64_t* __restrict__ counts, const int64_t* __restrict__ c_rp,
             uint32_t* __restrict__ c_col, double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* base = smem + (size_t)wib * DenseRowSmem::kPerWarp;
  double* acc = reinterpret_cast<double*>(base);
  uint32_t* bm = reinterpret_cast<uint32_t*>(base + (size_t)kDInter * 8);
  uint16_t* pref = reinterpret_cast<uint16_t*>(base + (size_t)kDInter * 8 + (size_t)kDWords * 4);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t w = warp; w < nrows; w += nwarps) {
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    const int64_t lo = mn[i];
    const int nwords = (int)((mx[i] - lo + 32) >> 5);
    for (int wd = lane; wd < nwords; wd += 32) bm[wd] = 0u;
    __syncwarp();
    // mark the row's columns
    for (int64_t t = a0; t < a1; ++t) {
      const int64_t k = __ldg(A.col + t);
      const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
      for (int64_t p = b0 + lane; p < b1; p += 32) {
        const uint32_t c = (uint32_t)((int64_t)__ldg(B.col + p) - lo);
        atomicOr(&bm[c >> 5], 1u << (c & 31));
      }
    }
    __syncwarp();
    // word prefix popcounts -> ranks
    uint32_t carry = 0;
    for (int w0 = 0; w0 < nwords; w0 += 32) {
      const int wd = w0 + lane;
      const uint32_t pc = wd < nwords ? (uint32_t)__popc(bm[wd]) : 0u;
      const uint32_t inc = warp_incl_scan(pc);
      if (wd < nwords) pref[wd] = (uint16_t)(carry + inc - pc);
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    const uint32_t m = carry;
    if (!Numeric) {
      if (lane == 0) counts[i] = m;
      __syncwarp();
      continue;
    }
    const int64_t out0 = c_rp[i], out_n = c_rp[i + 1] - out0;
    if ((int64_t)m != out_n) {
      if (lane == 0) atomicOr(err, 1ull);
      __syncwarp();
      continue;
    }
    for (uint32_t r = lane; r < m; r += 32) acc[r] = 0.0;   // dense accumulator starts at +0.0
    __syncwarp();
    // apply the B rows in ascending k: one k at a time, lanes over its distinct columns
    for (int64_t t = a0; t < a1; ++t) {
      const int64_t k = __ldg(A.col + t);
      const double av = __ldg(A.val + t);
      const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
      for (int64_t p = b0 + lane; p < b1; p += 32) {
        const uint32_t c = (uint32_t)((int64_t)__ldg(B.col + p) - lo);
        const uint32_t wd = c >> 5, bit = 1u << (c & 31);
        const uint32_t r = pref[wd] + __popc(bm[wd] & (bit - 1u));
        acc[r] = __dadd_rn(acc[r], __dmul_rn(av, __ldg(B.val + p)));
      }
      __syncwarp();
    }
    // emit in column order
    for (int wd = lane; wd < nwords; wd += 32) {
      uint32_t bits = bm[wd];
      uint32_t r = pref[wd];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        c_col[out0 + r] = (uint32_t)(lo + wd * 32 + b);
        c_val[out0 + r] = acc[r];
        ++r;
      }
    }
    __syncwarp();
  }
}

}  // namespace mg
