// Rows with a small intermediate product (<= 4096 elements): the whole row's
// product is gathered into shared memory in Gustavson order (ascending k,
// reference gustavson.py:44-59), sorted by (column, position) with a bitonic
// network, and every column segment is reduced with the association the
// reference gives it (see Sem / mode_of).  Warp-per-row up to 256 elements,
// CTA-per-row up to 4096.
#pragma once
#include "common.cuh"

namespace mg {

// --------------------------------------------------------------- bitonic sort in smem
// Sort keys[0..n) ascending (n a power of two), by a group of G threads (G = 32 for a
// warp with __syncwarp, or the block with __syncthreads).
template <int G, bool Warp, class K>
__device__ __forceinline__ void bitonic(K* keys, int n, int t) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < n; i += G) {
        int ixj = i ^ j;
        if (ixj > i) {
          K a = keys[i], b = keys[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) { keys[i] = b; keys[ixj] = a; }
        }
      }
      if (Warp) __syncwarp(); else __syncthreads();
    }
  }
}

__device__ __forceinline__ int pow2_at_least(int n, int lo) {
  int p = lo;
  while (p < n) p <<= 1;
  return p;
}

// lower bound of key in sorted keys[0..n)
template <class K>
__device__ __forceinline__ int lb_smem(const K* keys, int n, K key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Association for a column of row i: true = reference's dense accumulator
// (sequential from +0.0), false = sort accumulator (x0 + pairwise(rest)).
// chunk_count(): number of the row's intermediate elements in the numeric-plan
// fine chunk of this column (only consulted for Fine / Coarse rows).
template <class F>
__device__ __forceinline__ bool seq_mode(int cat, const Sem& sem, const F& chunk_count) {
  if (cat == kCatDense) return true;
  if (cat == kCatSort) return false;
  return chunk_count() >= sem.crossover;
}

// ================================================================ warp per row
constexpr int kWT = 256;  // threads per block (8 warps, one row each)
constexpr int kWSlots = 256;

template <bool Numeric>
__global__ void __launch_bounds__(kWT) k_rows_warp(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows,
                                                   const int8_t* __restrict__ cat, Sem sem, int64_t* __restrict__ counts,
                                                   const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
                                                   double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  // per warp: keys (u64) + vals (f64)
  __shared__ unsigned long long s_keys[kWT / 32][kWSlots];
  __shared__ double s_vals[kWT / 32][kWSlots];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned long long* keys = s_keys[wib];
  double* vals = s_vals[wib];
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t w = warp; w < nrows; w += nwarps) {
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    // gather in Gustavson order; position p = stream index (ascending k)
    int base = 0;
    for (int64_t t0 = a0; t0 < a1; t0 += 32) {
      const int64_t t = t0 + lane;
      int64_t b0 = 0;
      int len = 0;
      double av = 0.0;
      if (t < a1) {
        const int64_t k = __ldg(A.col + t);
        b0 = B.rp(k);
        len = (int)(B.rp(k + 1) - b0);
        av = __ldg(A.val + t);
      }
      const int inc = (int)warp_incl_scan((uint32_t)len);
      const int off = base + inc - len;
      for (int j = 0; j < len; ++j) {
        const uint32_t c = __ldg(B.col + b0 + j);
        const int p = off + j;
        keys[p] = ((unsigned long long)c << 8) | (unsigned long long)p;
        if (Numeric) vals[p] = __dmul_rn(av, __ldg(B.val + b0 + j));
      }
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
    const int n = base;
    const int np2 = pow2_at_least(n, 32);
    for (int p = n + lane; p < np2; p += 32) keys[p] = ~0ull;
    __syncwarp();
    bitonic<32, true>(keys, np2, lane);
    // column heads, ranks
    int rank_base = 0;
    const int ci = Numeric ? (int)cat[i] : 0;
    const int64_t out0 = Numeric ? c_rp[i] : 0;
    const int64_t out_n = Numeric ? c_rp[i + 1] - out0 : 0;
    for (int p0 = 0; p0 < n; p0 += 32) {
      const int p = p0 + lane;
      bool head = false;
      unsigned long long c = 0;
      if (p < n) {
        c = keys[p] >> 8;
        head = (p == 0) || ((keys[p - 1] >> 8) != c);
      }
      const unsigned m = __ballot_sync(0xffffffffu, head);
      if (Numeric && head) {
        const int r = rank_base + __popc(m & ((1u << lane) - 1u));
        int e = p + 1;
        while (e < n && (keys[e] >> 8) == c) ++e;
        auto chunk_count = [&]() -> int64_t {
          const unsigned long long f = c >> sem.shift_num;
          const unsigned long long lo = (f << sem.shift_num) << 8, hi = ((f + 1) << sem.shift_num) << 8;
          return lb_smem(keys, n, hi) - lb_smem(keys, n, lo);
        };
        double s;
        if (seq_mode(ci, sem, chunk_count)) {
          s = 0.0;
          for (int q = p; q < e; ++q) s = __dadd_rn(s, vals[keys[q] & 0xFF]);
        } else {
          auto x = [&](int64_t q) { return vals[keys[q] & 0xFF]; };
          s = vals[keys[p] & 0xFF];
          if (e - p > 1) s = __dadd_rn(s, pairwise(x, p + 1, e - p - 1));
        }
        if (r < out_n) {
          c_col[out0 + r] = (uint32_t)c;
          c_val[out0 + r] = s;
        }
      }
      rank_base += __popc(m);
    }
    if (lane == 0) {
      if (Numeric) {
        if (rank_base != out_n) atomicOr(err, 1ull);
      } else {
        counts[i] = rank_base;
      }
    }
    __syncwarp();
  }
}

// ================================================================ CTA per row
constexpr int kBT = 256;
constexpr int kBSlots = 4096;
constexpr int kBSmem = kBSlots * 16 + (kBT + 4 + kBT + 64) * 4;

template <bool Numeric>
__global__ void __launch_bounds__(kBT) k_rows_block(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows,
                                                    const int8_t* __restrict__ cat, Sem sem, int64_t* __restrict__ counts,
                                                    const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
                                                    double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
  double* vals = reinterpret_cast<double*>(smem + kBSlots * 8);
  uint32_t* koff = reinterpret_cast<uint32_t*>(smem + kBSlots * 16);  // kBT + 1 entries
  uint32_t* kb0 = koff + (kBT + 4);
  uint32_t* scratch = kb0 + kBT;
  __shared__ double s_av[kBT];
  __shared__ uint32_t s_heads[kBT + 1];
  const int tid = threadIdx.x;

  for (int64_t w = blockIdx.x; w < nrows; w += gridDim.x) {
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    uint32_t base = 0;
    // gather in chunks of kBT k's: lengths -> scan -> cooperative copy
    for (int64_t t0 = a0; t0 < a1; t0 += kBT) {
      const int64_t t = t0 + tid;
      uint32_t len = 0;
      if (t < a1) {
        const int64_t k = __ldg(A.col + t);
        const int64_t b0 = B.rp(k);
        len = (uint32_t)(B.rp(k + 1) - b0);
        kb0[tid] = (uint32_t)b0;
        if (Numeric) s_av[tid] = __ldg(A.val + t);
      }
      koff[tid] = len;
      __syncthreads();
      const uint32_t tot = block_excl_scan<kBT>(koff, kBT, scratch);
      if (tid == 0) koff[kBT] = tot;
      __syncthreads();
      // element q of this chunk -> segment via binary search over koff
      for (uint32_t q = tid; q < tot; q += kBT) {
        int lo = 0, hi = kBT;  // find last seg with koff[seg] <= q
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (koff[mid] <= q) lo = mid; else hi = mid;
        }
        const uint32_t j = q - koff[lo];
        const uint32_t src = kb0[lo] + j;
        const uint32_t p = base + q;
        const uint32_t c = __ldg(B.col + src);
        keys[p] = ((unsigned long long)c << 12) | p;
        if (Numeric) vals[p] = __dmul_rn(s_av[lo], __ldg(B.val + src));
      }
      base += tot;
      __syncthreads();
    }
    const int n = (int)base;
    const int np2 = pow2_at_least(n, 64);
    for (int p = n + tid; p < np2; p += kBT) keys[p] = ~0ull;
    __syncthreads();
    bitonic<kBT, false>(keys, np2, tid);
    // heads: each thread owns a contiguous range of sorted positions
    const int per = (n + kBT - 1) / kBT;
    const int pb = tid * per, pe = min(n, pb + per);
    uint32_t nh = 0;
    for (int p = pb; p < pe; ++p)
      if (p == 0 || (keys[p - 1] >> 12) != (keys[p] >> 12)) ++nh;
    s_heads[tid] = nh;
    __syncthreads();
    const uint32_t total = block_excl_scan<kBT>(s_heads, kBT, scratch);
    if (Numeric) {
      const int ci = (int)cat[i];
      const int64_t out0 = c_rp[i];
      const int64_t out_n = c_rp[i + 1] - out0;
      uint32_t r = s_heads[tid];
      for (int p = pb; p < pe; ++p) {
        const unsigned long long c = keys[p] >> 12;
        if (!(p == 0 || (keys[p - 1] >> 12) != c)) continue;
        int e = p + 1;
        while (e < n && (keys[e] >> 12) == c) ++e;
        auto chunk_count = [&]() -> int64_t {
          const unsigned long long f = c >> sem.shift_num;
          const unsigned long long lo = (f << sem.shift_num) << 12, hi = ((f + 1) << sem.shift_num) << 12;
          return lb_smem(keys, n, hi) - lb_smem(keys, n, lo);
        };
        double s;
        if (seq_mode(ci, sem, chunk_count)) {
          s = 0.0;
          for (int q = p; q < e; ++q) s = __dadd_rn(s, vals[keys[q] & 0xFFF]);
        } else {
          auto x = [&](int64_t q) { return vals[keys[q] & 0xFFF]; };
          s = vals[keys[p] & 0xFFF];
          if (e - p > 1) s = __dadd_rn(s, pairwise(x, p + 1, e - p - 1));
        }
        if (r < out_n) {
          c_col[out0 + r] = (uint32_t)c;
          c_val[out0 + r] = s;
        }
        ++r;
      }
      if (tid == 0 && total != out_n) atomicOr(err, 1ull);
    } else if (tid == 0) {
      counts[i] = total;
    }
    __syncthreads();
  }
}

}  // namespace mg
