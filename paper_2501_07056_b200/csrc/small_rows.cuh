// Rows with a small intermediate product (<= 4096 elements): the whole row's
// product is gathered into shared memory in Gustavson order (ascending k,
// reference gustavson.py:44-59), sorted by (column, position) with a bitonic
// network, and every column segment is reduced with the association the
// reference gives it (see Sem / mode_of).  Warp-per-row up to 256 elements,
// CTA-per-row up to 4096.
#pragma once
#include <type_traits>

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

// ---------------------------------------------------------------- register path (<= 64 products)
// Gathers the row's product (<= 32 B rows, <= 64 elements; lane l holds positions l and l+32),
// sorts (column, position) keys with a register bitonic network, and -- when no column
// repeats (the common case: the product of two random sparse rows) -- writes C directly:
// a single contribution is x0 under the sort association and +0.0 + x0 under the dense one.
// Returns 0 when a column repeats: the sorted keys and the values are then left in shared
// memory for the general path.  Mode: 0 count only, 1 values to C, 2 values to the
// row's upper-bound slot of the fused buffer and the count (k_rows_warp).  K: u32 keys
// (column << 8 | position) when columns < 2^24, else u64.
template <int Mode, class K>
__device__ __forceinline__ int reg_row64(const DevCsr& B, int64_t b0, uint32_t inc, uint32_t len, double av, uint32_t nn,
                                         unsigned long long* keys, double* vals, int ci, const Sem& sem,
                                         int64_t* __restrict__ counts, int64_t i, int64_t out0, int64_t out1,
                                         uint32_t* __restrict__ c_col, double* __restrict__ c_val,
                                         unsigned long long* __restrict__ err) {
  constexpr bool Numeric = Mode != 0;
  const int lane = threadIdx.x & 31;
  const uint32_t off = inc - len;
  K k0, k1;
  double v0 = 0.0, v1 = 0.0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint32_t q = (uint32_t)(r * 32 + lane);
    int lo = 0;   // segment of q: last lane with off <= q
#pragma unroll
    for (int st = 16; st > 0; st >>= 1) {
      const uint32_t o = __shfl_sync(0xffffffffu, off, lo + st);
      if (o <= q) lo += st;
    }
    const int64_t bb = __shfl_sync(0xffffffffu, b0, lo);
    const uint32_t oo = __shfl_sync(0xffffffffu, off, lo);
    const double a = __shfl_sync(0xffffffffu, av, lo);
    K key = ~K(0);
    double v = 0.0;
    if (q < nn) {
      const int64_t pp = bb + (q - oo);
      key = ((K)__ldg(B.col + pp) << 8) | (K)q;
      if (Numeric) v = __dmul_rn(a, __ldg(B.val + pp));
    }
    if (r == 0) { k0 = key; v0 = v; } else { k1 = key; v1 = v; }
  }
  // bitonic sort of 64 keys: element e = r * 32 + lane
#pragma unroll
  for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {
        const K lo = k0 < k1 ? k0 : k1, hi = k0 < k1 ? k1 : k0;
        k0 = lo;
        k1 = hi;
      } else {
        const K p0 = __shfl_xor_sync(0xffffffffu, k0, j), p1 = __shfl_xor_sync(0xffffffffu, k1, j);
        const bool lower = (lane & j) == 0;
        const bool up0 = (lane & k) == 0 || k == 64, up1 = ((lane + 32) & k) == 0 || k == 64;
        // take the partner when it belongs here: (lower == up) wants the smaller
        const bool t0 = (lower == up0) ? p0 < k0 : p0 > k0;
        const bool t1 = (lower == up1) ? p1 < k1 : p1 > k1;
        if (t0) k0 = p0;
        if (t1) k1 = p1;
      }
    }
  }
  const K c0 = k0 >> 8, c1 = k1 >> 8;
  const K pc0 = __shfl_up_sync(0xffffffffu, c0, 1), pc1 = __shfl_up_sync(0xffffffffu, c1, 1);
  const K last0 = __shfl_sync(0xffffffffu, c0, 31);
  const bool ok0 = (uint32_t)lane < nn, ok1 = (uint32_t)(lane + 32) < nn;
  const bool h0 = ok0 && (lane == 0 || pc0 != c0);
  const bool h1 = ok1 && (lane == 0 ? last0 != c1 : pc1 != c1);
  const uint32_t m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
  const uint32_t distinct = __popc(m0) + __popc(m1);
  const bool nodup = distinct == nn;
  if (!Numeric) {
    if (lane == 0) counts[i] = distinct;
    return 1;
  }
  if (nodup) {
    // (a Fine / Coarse row would need its chunk counts: only Sort / Dense rows take this path)
    if (ci == kCatSort || ci == kCatDense) {
      const uint32_t q0 = (uint32_t)(k0 & 0xFF), q1 = (uint32_t)(k1 & 0xFF);
      const double a0 = __shfl_sync(0xffffffffu, v0, q0 & 31), a1 = __shfl_sync(0xffffffffu, v1, q0 & 31);
      const double b0v = __shfl_sync(0xffffffffu, v0, q1 & 31), b1v = __shfl_sync(0xffffffffu, v1, q1 & 31);
      double x0 = q0 < 32 ? a0 : a1, x1 = q1 < 32 ? b0v : b1v;
      if (ci == kCatDense) {
        x0 = __dadd_rn(0.0, x0);
        x1 = __dadd_rn(0.0, x1);
      }
      if (out1 - out0 != (int64_t)nn) {
        if (lane == 0) atomicOr(err, 1ull);
        return 1;
      }
      if (ok0) {
        c_col[out0 + lane] = (uint32_t)c0;
        c_val[out0 + lane] = x0;
      }
      if (ok1) {
        c_col[out0 + 32 + lane] = (uint32_t)c1;
        c_val[out0 + 32 + lane] = x1;
      }
      if (Mode == 2 && lane == 0) counts[i] = distinct;
      return 1;
    }
  }
  // general path: sorted keys (as u64 column << 8 | position) and the values (by position)
  keys[lane] = k0 == ~K(0) ? ~0ull : (unsigned long long)k0;
  keys[lane + 32] = k1 == ~K(0) ? ~0ull : (unsigned long long)k1;
  vals[lane] = v0;
  vals[lane + 32] = v1;
  return 0;
}

// ================================================================ warp per row
constexpr int kWT = 256;  // threads per block (8 warps, one row each)
constexpr int kWSlots = 256;

// Mode 0: distinct counts (symbolic); 1: values into C at c_rp (numeric); 2: fused -- values
// into the row's slot of a buffer laid out by the rows' upper bounds (ub: exclusive prefix of
// the listed rows' product counts) and the counts; the numeric pass then only copies
// (k_rows_copy).  Key32: columns < 2^24 (32-bit sort keys).
template <int Mode, bool Key32 = false>
__global__ void __launch_bounds__(kWT) k_rows_warp(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows,
                                                   const int8_t* __restrict__ cat, Sem sem, int64_t* __restrict__ counts,
                                                   const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
                                                   double* __restrict__ c_val, unsigned long long* __restrict__ err,
                                                   const int64_t* __restrict__ ub = nullptr) {
  constexpr bool Numeric = Mode != 0;
  using K = typename std::conditional<Key32, uint32_t, unsigned long long>::type;
  // per warp: keys (u64) + vals (f64)
  __shared__ unsigned long long s_keys[kWT / 32][kWSlots];
  __shared__ double s_vals[kWT / 32][kWSlots];
  __shared__ int s_n[kWT / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned long long* keys = s_keys[wib];
  double* vals = s_vals[wib];
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t w = warp; w < nrows; w += nwarps) {
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    if (a1 - a0 <= 32) {
      // <= 32 k's: row lengths in one wave; a product of <= 64 elements is sorted in registers
      const int64_t t = a0 + lane;
      int64_t b0 = 0;
      uint32_t len = 0;
      double av = 0.0;
      if (t < a1) {
        const int64_t k = __ldg(A.col + t);
        b0 = B.rp(k);
        len = (uint32_t)(B.rp(k + 1) - b0);
        if (Numeric) av = __ldg(A.val + t);
      }
      const uint32_t inc = warp_incl_scan(len);
      const uint32_t nn = __shfl_sync(0xffffffffu, inc, 31);
      if (nn <= 64u) {
        const int64_t o0 = Mode == 1 ? c_rp[i] : (Mode == 2 ? ub[w] : 0);
        const int64_t o1 = Mode == 1 ? c_rp[i + 1] : (Mode == 2 ? ub[w + 1] : 0);
        const int st = reg_row64<Mode, K>(B, b0, inc, len, av, nn, keys, vals, cat[i], sem, counts, i, o0, o1, c_col,
                                          c_val, err);
        if (st) continue;   // done in registers (else: keys / vals sorted in shared memory)
        if (lane == 0) s_n[wib] = (int)nn;
        goto heads;
      }
    }
    {
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
    s_n[wib] = n;
    const int np2 = pow2_at_least(n, 32);
    for (int p = n + lane; p < np2; p += 32) keys[p] = ~0ull;
    __syncwarp();
    bitonic<32, true>(keys, np2, lane);
    }
  heads:
    __syncwarp();
    const int n = s_n[wib];
    // column heads, ranks
    int rank_base = 0;
    const int ci = Numeric ? (int)cat[i] : 0;
    const int64_t out0 = Mode == 1 ? c_rp[i] : (Mode == 2 ? ub[w] : 0);
    const int64_t out_n = Mode == 1 ? c_rp[i + 1] - out0 : (Mode == 2 ? ub[w + 1] - out0 : 0);
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
      if (Mode == 1) {
        if (rank_base != out_n) atomicOr(err, 1ull);
      } else {
        counts[i] = rank_base;
      }
    }
    __syncwarp();
  }
}

// Numeric pass of fused rows: row w of the list moves from its upper-bound slot (ub[w]) of the
// fused buffer to C (one warp per row, <= 256 entries, coalesced).
__global__ void __launch_bounds__(256) k_rows_copy(const int32_t* __restrict__ rows, int64_t nrows,
                                                   const int64_t* __restrict__ ub, const uint32_t* __restrict__ f_col,
                                                   const double* __restrict__ f_val, const int64_t* __restrict__ c_rp,
                                                   uint32_t* __restrict__ c_col, double* __restrict__ c_val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w < nrows; w += nwarps) {
    const int64_t i = rows[w];
    const int64_t d0 = c_rp[i], n = c_rp[i + 1] - d0, s0 = ub[w];
    for (int64_t t = lane; t < n; t += 32) {
      c_col[d0 + t] = __ldg(f_col + s0 + t);
      c_val[d0 + t] = __ldg(f_val + s0 + t);
    }
  }
}

// ub[w] = inter[rows[w]] (then scanned into the fused buffer's row slots)
__global__ void k_gather_inter(const int32_t* __restrict__ rows, int64_t nrows, const int64_t* __restrict__ inter,
                               int64_t* __restrict__ out) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nrows; w += (int64_t)gridDim.x * blockDim.x)
    out[w] = inter[rows[w]];
}

// ================================================================ CTA per row
// Rows with 256 < products <= 4096: the product is gathered in Gustavson order
// (one ascending run per B row), then the runs are merged pairwise (merge path,
// ties from the left run: a stable sort by column that keeps ascending k inside
// every column), then each column is summed by one thread with the association
// the reference gives it.
constexpr int kBT = 256;
constexpr int kBSlots = 4096;
constexpr size_t kBSmem = (size_t)kBSlots * 4 * 2      // keys (ping-pong)
                          + (size_t)kBSlots * 2 * 2    // positions (ping-pong)
                          + (size_t)kBSlots * 8        // values (stream order)
                          + (size_t)(kBSlots + 8) * 2  // run boundaries
                          + (size_t)(kBSlots + 8) * 2  // column starts
                          + (size_t)(kBT + 8) * 4 * 2  // k offsets / starts
                          + 64 * 4;

// merge path: number of elements taken from L when d outputs of merge(L, R) are done
// (stable: on equal keys L goes first)
__device__ __forceinline__ int merge_split(const uint32_t* L, int nl, const uint32_t* R, int nr, int d) {
  int lo = max(0, d - nr), hi = min(d, nl);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (L[mid] <= R[d - 1 - mid]) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <bool Numeric>
__global__ void __launch_bounds__(kBT) k_rows_block(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows,
                                                    const int8_t* __restrict__ cat, Sem sem, int64_t* __restrict__ counts,
                                                    const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
                                                    double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* sp = smem;
  uint32_t* keyA = reinterpret_cast<uint32_t*>(sp); sp += kBSlots * 4;
  uint32_t* keyB = reinterpret_cast<uint32_t*>(sp); sp += kBSlots * 4;
  double* vals = reinterpret_cast<double*>(sp); sp += kBSlots * 8;
  uint16_t* posA = reinterpret_cast<uint16_t*>(sp); sp += kBSlots * 2;
  uint16_t* posB = reinterpret_cast<uint16_t*>(sp); sp += kBSlots * 2;
  uint16_t* runs = reinterpret_cast<uint16_t*>(sp); sp += (kBSlots + 8) * 2;
  uint16_t* cst = reinterpret_cast<uint16_t*>(sp); sp += (kBSlots + 8) * 2;
  uint32_t* koff = reinterpret_cast<uint32_t*>(sp); sp += (kBT + 8) * 4;
  uint32_t* kb0 = reinterpret_cast<uint32_t*>(sp); sp += (kBT + 8) * 4;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sp);
  __shared__ double s_av[kBT];
  __shared__ int s_nr;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  for (int64_t w = blockIdx.x; w < nrows; w += gridDim.x) {
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    uint32_t base = 0;
    if (tid == 0) s_nr = 0;
    // ---- gather in chunks of kBT k's: lengths -> scan -> cooperative copy; runs = non-empty segments
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
      const int nr0 = s_nr;
      const uint32_t ne = __ballot_sync(0xffffffffu, len > 0);
      if (lane == 0) scratch[wid] = __popc(ne);
      const uint32_t tot = block_excl_scan<kBT>(koff, kBT, scratch + 8);
      if (tid == 0) koff[kBT] = tot;
      // run starts of the non-empty segments (in k order)
      uint32_t wb = 0;
      for (int q = 0; q < wid; ++q) wb += scratch[q];
      if (len > 0) runs[nr0 + wb + __popc(ne & ((1u << lane) - 1u))] = (uint16_t)(base + koff[tid]);
      __syncthreads();
      if (tid == 0) {
        uint32_t all = 0;
        for (int q = 0; q < kBT / 32; ++q) all += scratch[q];
        s_nr = nr0 + (int)all;
      }
      for (uint32_t q = tid; q < tot; q += kBT) {
        int lo = 0, hi = kBT;  // last segment with koff[seg] <= q
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (koff[mid] <= q) lo = mid; else hi = mid;
        }
        const uint32_t src = kb0[lo] + (q - koff[lo]);
        const uint32_t p = base + q;
        keyA[p] = __ldg(B.col + src);
        posA[p] = (uint16_t)p;
        if (Numeric) vals[p] = __dmul_rn(s_av[lo], __ldg(B.val + src));
      }
      base += tot;
      __syncthreads();
    }
    const int n = (int)base;
    int nr = s_nr;
    if (tid == 0) runs[nr] = (uint16_t)n;
    __syncthreads();
    // ---- pairwise merge rounds
    uint32_t* kin = keyA;
    uint32_t* kout = keyB;
    uint16_t* pin = posA;
    uint16_t* pout = posB;
    const int per = (n + kBT - 1) / kBT;
    while (nr > 1) {
      const int npair = (nr + 1) >> 1;
      int o = tid * per;
      const int oend = min(n, o + per);
      while (o < oend) {
        // pair j containing output o: last j with runs[2j] <= o
        int lo = 0, hi = npair;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if ((int)runs[2 * mid] <= o) lo = mid; else hi = mid;
        }
        const int ls = runs[2 * lo], ms = runs[min(2 * lo + 1, nr)], re = runs[min(2 * lo + 2, nr)];
        const int nl = ms - ls, nrr = re - ms;
        const int d = o - ls;
        int li = merge_split(kin + ls, nl, kin + ms, nrr, d);
        int ri = d - li;
        const int stop = min(oend, re);
        for (; o < stop; ++o) {
          bool takeL;
          if (li >= nl) takeL = false;
          else if (ri >= nrr) takeL = true;
          else takeL = kin[ls + li] <= kin[ms + ri];
          const int src = takeL ? ls + li : ms + ri;
          kout[o] = kin[src];
          pout[o] = pin[src];
          if (takeL) ++li; else ++ri;
        }
      }
      __syncthreads();
      // run boundaries of the merged runs
      constexpr int kNb = kBSlots / kBT + 1;
      uint16_t nb[kNb];
      const int nnr = npair;
#pragma unroll
      for (int q = 0; q < kNb; ++q) {
        const int j = tid + q * kBT;
        if (j <= nnr) nb[q] = j < nnr ? runs[2 * j] : (uint16_t)n;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kNb; ++q) {
        const int j = tid + q * kBT;
        if (j <= nnr) runs[j] = nb[q];
      }
      __syncthreads();
      nr = nnr;
      uint32_t* tk = kin; kin = kout; kout = tk;
      uint16_t* tp = pin; pin = pout; pout = tp;
    }
    // ---- column heads: warp w scans a contiguous slice of the sorted keys with ballots
    const int sl = ((n + kBT / 32 - 1) / (kBT / 32) + 31) & ~31;
    const int s0 = min(n, wid * sl), s1 = min(n, s0 + sl);
    uint32_t wcount = 0;
    for (int p0 = s0; p0 < s1; p0 += 32) {
      const int p = p0 + lane;
      const bool head = p < s1 && (p == 0 || kin[p - 1] != kin[p]);
      wcount += __popc(__ballot_sync(0xffffffffu, head));
    }
    if (lane == 0) scratch[wid] = wcount;
    __syncthreads();
    uint32_t rb = 0, total = 0;
    for (int q = 0; q < kBT / 32; ++q) {
      const uint32_t v = scratch[q];
      if (q < wid) rb += v;
      total += v;
    }
    for (int p0 = s0; p0 < s1; p0 += 32) {
      const int p = p0 + lane;
      const bool head = p < s1 && (p == 0 || kin[p - 1] != kin[p]);
      const uint32_t m = __ballot_sync(0xffffffffu, head);
      if (head) cst[rb + __popc(m & ((1u << lane) - 1u))] = (uint16_t)p;
      rb += __popc(m);
    }
    if (tid == 0) cst[total] = (uint16_t)n;
    __syncthreads();
    if (Numeric) {
      const int ci = (int)cat[i];
      const int64_t out0 = c_rp[i];
      const int64_t out_n = c_rp[i + 1] - out0;
      for (uint32_t r = tid; r < total; r += kBT) {
        const int p = cst[r], e = cst[r + 1];
        const uint32_t c = kin[p];
        auto chunk_count = [&]() -> int64_t {
          const uint64_t f = (uint64_t)c >> sem.shift_num;
          const uint64_t lo = f << sem.shift_num, hi = (f + 1) << sem.shift_num;
          auto lb = [&](uint64_t key) {
            int a = 0, b = n;
            while (a < b) {
              const int mid = (a + b) >> 1;
              if ((uint64_t)kin[mid] < key) a = mid + 1; else b = mid;
            }
            return a;
          };
          return lb(hi) - lb(lo);
        };
        double sum;
        if (seq_mode(ci, sem, chunk_count)) {
          sum = 0.0;
          for (int q = p; q < e; ++q) sum = __dadd_rn(sum, vals[pin[q]]);
        } else {
          auto x = [&](int64_t q) { return vals[pin[q]]; };
          sum = vals[pin[p]];
          if (e - p > 1) sum = __dadd_rn(sum, pairwise(x, p + 1, e - p - 1));
        }
        if ((int64_t)r < out_n) {
          c_col[out0 + r] = c;
          c_val[out0 + r] = sum;
        }
      }
      if (tid == 0 && total != out_n) atomicOr(err, 1ull);
    } else if (tid == 0) {
      counts[i] = total;
    }
    __syncthreads();
  }
}

}  // namespace mg
