// Shared device helpers for the B200 MAGNUS kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mg {

constexpr int kCatSort = 0, kCatDense = 1, kCatFine = 2, kCatCoarse = 3;

// CSR view on device.  row_ptr may be int32 or int64 (runtime, warp-uniform).
struct DevCsr {
  int64_t n_rows, n_cols, nnz;
  const int64_t* rp64;
  const int32_t* rp32;
  const uint32_t* col;
  const double* val;
  const uint32_t* skip;   // skip[j] = col[32*j] (built for B by magnus_setup; gallops over long rows)
  __device__ __forceinline__ int64_t rp(int64_t i) const { return rp64 ? __ldg(rp64 + i) : (int64_t)__ldg(rp32 + i); }
};

// Reference-visible semantics of a call: which association each output value gets.
struct Sem {
  int64_t crossover;    // AccumThresholds.sort_dense_crossover (accumulators.py:36)
  int32_t shift_num;    // numeric ChunkPlan.shift_fine (planner.py:106-152, magnus.py:570)
  int32_t mode_words;   // 32-bit words of per-chunk mode bits per heavy row
  int64_t n_chunks_num;  // numeric-plan fine chunks over the whole span (plan_cols >> shift_fine)
};

// ---------------------------------------------------------------- numpy pairwise
// The reference's sort accumulator merges with np.add.reduceat (accumulators.py:129):
// out = x0; out += pairwise_sum(x1..x_{d-1}).  numpy's published pairwise summation,
// restated for an accessor x(j).
template <class F>
__device__ __forceinline__ double pw_leaf(const F& x, int64_t off, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, x(off + i));
    return r;
  }
  double r0 = x(off), r1 = x(off + 1), r2 = x(off + 2), r3 = x(off + 3);
  double r4 = x(off + 4), r5 = x(off + 5), r6 = x(off + 6), r7 = x(off + 7);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, x(off + i)); r1 = __dadd_rn(r1, x(off + i + 1));
    r2 = __dadd_rn(r2, x(off + i + 2)); r3 = __dadd_rn(r3, x(off + i + 3));
    r4 = __dadd_rn(r4, x(off + i + 4)); r5 = __dadd_rn(r5, x(off + i + 5));
    r6 = __dadd_rn(r6, x(off + i + 6)); r7 = __dadd_rn(r7, x(off + i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)), __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, x(off + i));
  return res;
}

template <class F>
__device__ __noinline__ double pairwise(const F& x, int64_t off, int64_t n) {
  if (n <= 128) return pw_leaf(x, off, n);
  // explicit post-order traversal of numpy's recursion (split at n/2 rounded down to a multiple of 8)
  // depth: ceil(log2(n / 128)) + 1 levels (n < 2^32 on the device)
  int64_t so[26], sn[26];
  double sl[26];
  int8_t ss[26];
  int top = 0;
  so[0] = off; sn[0] = n; ss[0] = 0;
  double ret = 0.0;
  while (top >= 0) {
    int64_t o = so[top], m = sn[top];
    if (m <= 128) { ret = pw_leaf(x, o, m); --top; continue; }
    int64_t m2 = m / 2; m2 -= m2 % 8;
    if (ss[top] == 0) { ss[top] = 1; ++top; so[top] = o; sn[top] = m2; ss[top] = 0; }
    else if (ss[top] == 1) { sl[top] = ret; ss[top] = 2; ++top; so[top] = o + m2; sn[top] = m - m2; ss[top] = 0; }
    else { ret = __dadd_rn(sl[top], ret); --top; }
  }
  return ret;
}

// ---------------------------------------------------------------- warp / block scans
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// In-place exclusive scan of a[0..n) (u32) by the whole block; returns the total.
// scratch: >= 33 u32 of shared memory.  Must be called by all threads.
template <int T>
__device__ uint32_t block_excl_scan(uint32_t* a, int n, uint32_t* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + T - 1) / T;
  const int b = tid * per, e = min(n, b + per);
  uint32_t s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  uint32_t inc = warp_incl_scan(s);
  if (lane == 31) scratch[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < T / 32 ? scratch[lane] : 0;
    uint32_t wi = warp_incl_scan(w);
    if (lane < T / 32) scratch[lane] = wi - w;
    if (lane == 31) scratch[32] = wi;
  }
  __syncthreads();
  uint32_t run = scratch[wid] + inc - s;
  for (int i = b; i < e; ++i) { uint32_t v = a[i]; a[i] = run; run += v; }
  uint32_t total = scratch[32];
  __syncthreads();
  return total;
}

template <int T>
__device__ uint32_t block_sum(uint32_t v, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  uint32_t t = 0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < T / 32; ++w) t += scratch[w];
    scratch[32] = t;
  }
  __syncthreads();
  t = scratch[32];
  __syncthreads();
  return t;
}

template <int T>
__device__ int64_t block_min_i64(int64_t v, int64_t* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { int64_t t = __shfl_xor_sync(0xffffffffu, v, o); v = t < v ? t : v; }
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t m = scratch[0];
    for (int w = 1; w < T / 32; ++w) m = scratch[w] < m ? scratch[w] : m;
    scratch[32] = m;
  }
  __syncthreads();
  int64_t r = scratch[32];
  __syncthreads();
  return r;
}

// Conflict-free in-place exclusive scan of a[0..n): each warp owns a contiguous
// slice walked 32 entries at a time (lane-consecutive addresses).
template <int T>
__device__ uint32_t block_scan_striped(uint32_t* a, int n, uint32_t* scratch) {
  constexpr int NW = T / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int per = (((n + NW - 1) / NW) + 31) & ~31;
  const int b = min(n, wid * per), e = min(n, b + per);
  uint32_t s = 0;
  for (int i = b + lane; i < e; i += 32) s += a[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) scratch[wid] = s;
  __syncthreads();
  if (wid == 0) {
    const uint32_t w = lane < NW ? scratch[lane] : 0u;
    const uint32_t wi = warp_incl_scan(w);
    if (lane < NW) scratch[lane] = wi - w;
    if (lane == 31) scratch[32] = wi;
  }
  __syncthreads();
  uint32_t carry = scratch[wid];
  for (int i0 = b; i0 < e; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t v = i < e ? a[i] : 0u;
    const uint32_t inc = warp_incl_scan(v);
    if (i < e) a[i] = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  const uint32_t total = scratch[32];
  __syncthreads();
  return total;
}

// first index in [lo, hi) with col[idx] >= key (B rows are sorted: canonical input)
__device__ __forceinline__ uint32_t lower_bound_col(const uint32_t* __restrict__ col, uint32_t lo, uint32_t hi, uint32_t key) {
  while (lo < hi) {
    uint32_t mid = lo + ((hi - lo) >> 1);
    if (__ldg(col + mid) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace mg
