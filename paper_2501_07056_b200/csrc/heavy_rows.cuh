// Rows with a large intermediate product (> 4096 elements): the MAGNUS fine
// level (reference magnus.py:195-262, Alg. 3) retargeted from a core's L2 to an
// SM's shared memory.
//
// The reference reorders a row's whole product into column chunks through a
// memory buffer (histogram, prefix sum, stable scatter).  On the GPU the chunk
// ("window", up to kWin columns) is accumulated in shared memory and its
// elements are fetched straight from B: B rows are sorted (canonical input),
// so the part of B row k inside a window is one contiguous segment whose end is
// found by a binary search from a per-k cursor.  The reorder buffer and its
// write+read traffic disappear; every B element is read once per phase.
//
// Within a window the elements (in ascending-k stream order) are bucketed by
// column with a shared-memory counting sort (histogram -> scan -> scatter);
// each column bucket is then put back into stream order and summed with the
// association the reference gives that column (dense: sequential from +0.0;
// sort: x0 + pairwise).  Windows whose stream exceeds kCap elements are
// processed in stream batches with a per-column carry (sequential association
// only; windows containing pairwise columns are narrowed until they fit).
#pragma once
#include "common.cuh"

namespace mg {

#ifdef MG_PROFILE_PHASES
// debug-build phase timers (thread 0 clocks between the CTA barriers)
__device__ unsigned long long g_phase[32];
#define PH_INIT unsigned long long ph_t0 = clock64(); unsigned long long ph_acc[16] = {0};
#define PH(i) do { if (threadIdx.x == 0) { unsigned long long t1_ = clock64(); ph_acc[i] += t1_ - ph_t0; ph_t0 = t1_; } } while (0)
#define PH_COUNT(i, v) do { if (threadIdx.x == 0) ph_acc[i] += (v); } while (0)
#define PH_FLUSH do { if (threadIdx.x == 0) for (int q_ = 0; q_ < 16; ++q_) atomicAdd(&g_phase[q_], ph_acc[q_]); } while (0)
#else
#define PH_INIT
#define PH(i)
#define PH_COUNT(i, v)
#define PH_FLUSH
#endif

constexpr int kHT = 512;                // symbolic: threads per CTA (1 CTA / SM)
constexpr int kNT = 256;                // numeric: threads per CTA (2 CTAs / SM)
constexpr int kCap = 4096;              // numeric: stream elements per batch
constexpr int kItems = kCap / kNT;      // 16 stream elements per thread per batch
constexpr int kKS = 1024;               // symbolic: k's whose cursors live in shared memory
constexpr int kKSN = 512;               // numeric: k's whose cursors live in shared memory
constexpr int kSymWin = 1 << 20;        // symbolic window width (columns; 128 KB bitmap)
constexpr int kChunkSmem = 8192;        // numeric-plan chunk counters kept in smem (symbolic)

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

// first index in [lo, hi) with col[idx] >= key, galloping from lo (segment ends
// are usually a few elements past the cursor)
__device__ __forceinline__ uint32_t gallop_col(const uint32_t* __restrict__ col, uint32_t lo, uint32_t hi, uint32_t key) {
  if (lo >= hi || __ldg(col + lo) >= key) return lo;
  uint32_t step = 1, prev = lo;   // invariant: col[prev] < key
  while (true) {
    const uint32_t nxt = prev + step;
    if (nxt >= hi) return lower_bound_col(col, prev + 1, hi, key);
    if (__ldg(col + nxt) >= key) return lower_bound_col(col, prev + 1, nxt, key);
    prev = nxt;
    step <<= 1;
  }
}

// Per-row k state: cursor (next B position in this row), segment end in the
// current window, exclusive stream offset, B row end, A value.
struct KState {
  uint32_t* ks;
  uint32_t* ke;
  uint32_t* koff;  // nk + 1
  uint32_t* kend;
  double* kav;
};

template <int T>
__device__ __forceinline__ void kstate_load(const KState& st, const DevCsr& A, const DevCsr& B, int64_t a0, int nk) {
  for (int t = threadIdx.x; t < nk; t += T) {
    const int64_t k = __ldg(A.col + a0 + t);
    st.ks[t] = (uint32_t)B.rp(k);
    st.kend[t] = (uint32_t)B.rp(k + 1);
    st.kav[t] = __ldg(A.val + a0 + t);
  }
}

// Segment ends for window [lo, hi); returns the stream length of the window.
// hi_all: the window reaches past the row's last column (no search needed).
template <int T>
__device__ __forceinline__ uint32_t kstate_segments(const KState& st, const DevCsr& B, int nk, uint32_t hi, bool hi_all,
                                                    uint32_t* scratch) {
  for (int t = threadIdx.x; t < nk; t += T) {
    const uint32_t s = st.ks[t], e0 = st.kend[t];
    const uint32_t e = hi_all ? e0 : gallop_col(B.col, s, e0, hi);
    st.ke[t] = e;
    st.koff[t] = e - s;
  }
  __syncthreads();
  const uint32_t tot = block_scan_striped<T>(st.koff, nk, scratch);
  if (threadIdx.x == 0) st.koff[nk] = tot;
  __syncthreads();
  return tot;
}

// Advance cursors to the segment ends; returns the next column any k still has (or INT64_MAX).
template <int T>
__device__ __forceinline__ int64_t kstate_advance(const KState& st, const DevCsr& B, int nk, int64_t* scratch64) {
  int64_t nxt = INT64_MAX;
  for (int t = threadIdx.x; t < nk; t += T) {
    const uint32_t e = st.ke[t];
    st.ks[t] = e;
    if (e < st.kend[t]) {
      const int64_t c = __ldg(B.col + e);
      nxt = c < nxt ? c : nxt;
    }
  }
  return block_min_i64<T>(nxt, scratch64);
}

// Stream position p -> (segment t, B position): last t with koff[t] <= p.
__device__ __forceinline__ int kstate_find(const KState& st, int nk, uint32_t p) {
  int lo = 0, hi = nk;  // koff[nk] = total > p
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (st.koff[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

// ------------------------------------------------------------------ symbolic
// Exact distinct-column count per row (precise prediction, reference
// magnus.py:420-456) with a shared-memory bitmap per window, plus -- for Fine /
// Coarse rows -- the per-chunk element counts of the numeric plan that decide
// each chunk's accumulator (accumulators.py:132-134), stored as mode bits.
struct HeavySymSmem {
  static constexpr size_t kBitmap = (kSymWin / 32) * 4;                 // 128 KB
  static constexpr size_t kChunk = kChunkSmem * 4;                       // 32 KB
  static constexpr size_t kK = (size_t)kKS * 4 * 4 + (kKS + 4) * 4 + kKS * 8;
  static constexpr size_t kScratch = 64 * 8;
  static constexpr size_t kTotal = kBitmap + kChunk + kK + kScratch;
  static_assert(kBitmap % 16 == 0 && kChunk % 16 == 0 && kK % 16 == 0, "16-byte aligned sections");
};

__global__ void __launch_bounds__(kHT, 1)
k_heavy_symbolic(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows, const int8_t* __restrict__ cat,
                 const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, Sem sem, int64_t* __restrict__ counts,
                 uint32_t* __restrict__ modebits, uint32_t* __restrict__ gk, int64_t gk_stride,
                 uint32_t* __restrict__ gchunk, unsigned long long* __restrict__ work) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem);
  uint32_t* ccnt_s = reinterpret_cast<uint32_t*>(smem + HeavySymSmem::kBitmap);
  unsigned char* kb = smem + HeavySymSmem::kBitmap + HeavySymSmem::kChunk;
  int64_t* scratch64 = reinterpret_cast<int64_t*>(kb + HeavySymSmem::kK);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(scratch64);
  __shared__ int64_t s_row;

  for (int i = threadIdx.x; i < kSymWin / 32; i += kHT) bitmap[i] = 0;
  for (int i = threadIdx.x; i < kChunkSmem; i += kHT) ccnt_s[i] = 0;
  uint32_t* ccnt_g = gchunk + (size_t)blockIdx.x * (size_t)(sem.n_chunks_num);
  const bool chunk_in_smem = sem.n_chunks_num <= kChunkSmem;
  uint32_t* ccnt = chunk_in_smem ? ccnt_s : ccnt_g;
  __syncthreads();

  while (true) {
    if (threadIdx.x == 0) s_row = (int64_t)atomicAdd(work, 1ull);
    __syncthreads();
    const int64_t w = s_row;
    __syncthreads();
    if (w >= nrows) break;
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    const int nk = (int)(a1 - a0);
    KState st;
    if (nk <= kKS) {
      st.ks = reinterpret_cast<uint32_t*>(kb);
      st.ke = st.ks + kKS;
      st.kend = st.ke + kKS;
      st.koff = st.kend + kKS;
      st.kav = reinterpret_cast<double*>(st.koff + kKS + 4);
    } else {
      uint32_t* g = gk + (size_t)blockIdx.x * (size_t)gk_stride * 6;
      st.ks = g;
      st.ke = g + gk_stride;
      st.kend = g + 2 * gk_stride;
      st.koff = g + 3 * gk_stride;
      st.kav = reinterpret_cast<double*>(g + 4 * gk_stride);
    }
    kstate_load<kHT>(st, A, B, a0, nk);
    const int ci = cat[i];
    const bool need_modes = (ci == kCatFine || ci == kCatCoarse);
    const int64_t row_lo = mn[i], row_hi = mx[i];
    int64_t lo = row_lo;
    uint64_t total = 0;
    __syncthreads();
    while (lo <= row_hi) {
      const int64_t hi = lo + kSymWin;
      const bool hi_all = hi > row_hi;
      const uint32_t S = kstate_segments<kHT>(st, B, nk, (uint32_t)(hi_all ? 0 : hi), hi_all, scratch);
      // stream elements: blocked assignment, one search per thread per tile
      for (uint32_t t0 = 0; t0 < S; t0 += kHT * kItems) {
        const uint32_t q0 = t0 + threadIdx.x * kItems;
        if (q0 < S) {
          int t = kstate_find(st, nk, q0);
          for (uint32_t q = q0; q < min(S, q0 + kItems); ++q) {
            while (st.koff[t + 1] <= q) ++t;
            const uint32_t pos = st.ks[t] + (q - st.koff[t]);
            const uint32_t c = __ldg(B.col + pos);
            const uint32_t lc = (uint32_t)(c - lo);
            atomicOr(&bitmap[lc >> 5], 1u << (lc & 31));
            if (need_modes) atomicAdd(&ccnt[c >> sem.shift_num], 1u);
          }
        }
      }
      __syncthreads();
      const int64_t width = (hi_all ? row_hi + 1 : hi) - lo;
      const int words = (int)((width + 31) >> 5);
      uint32_t pc = 0;
      for (int wd = threadIdx.x; wd < words; wd += kHT) {
        pc += __popc(bitmap[wd]);
        bitmap[wd] = 0;
      }
      total += block_sum<kHT>(pc, scratch);
      const int64_t nxt = kstate_advance<kHT>(st, B, nk, scratch64);
      lo = nxt == INT64_MAX ? row_hi + 1 : nxt;
    }
    if (threadIdx.x == 0) counts[i] = (int64_t)total;
    if (need_modes) {
      const int64_t f0 = row_lo >> sem.shift_num, f1 = row_hi >> sem.shift_num;
      uint32_t* mb = modebits + (size_t)w * sem.mode_words;
      for (int64_t wd = (f0 >> 5) + threadIdx.x; wd <= (f1 >> 5); wd += kHT) {
        uint32_t bits = 0;
        for (int b = 0; b < 32; ++b) {
          const int64_t f = wd * 32 + b;
          if (f >= f0 && f <= f1) {
            if (ccnt[f] >= (uint64_t)sem.crossover) bits |= 1u << b;
          }
        }
        mb[wd] = bits;
      }
      __syncthreads();
      for (int64_t f = f0 + threadIdx.x; f <= f1; f += kHT) ccnt[f] = 0;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ numeric
// Window machinery (per CTA, one row at a time):
//  * a window [lo, lo+W) whose stream fits one batch (S <= kCap) is "wide"
//    (W up to 2^18): its columns are compacted through a bitmap (rank = word
//    prefix + popcount), so buckets are indexed by output rank and every phase
//    costs O(S + W/32) -- sparse windows pay nothing per empty column;
//  * a window that cannot fit one batch (dense hub regions) is "dense"
//    (W <= 8192): its stream is processed in batches and every column keeps a
//    carry in shared memory (sequential association only; windows containing
//    pairwise columns are narrowed until they fit one batch).
constexpr uint32_t kSmallBucket = 12;
constexpr int kWinWide = 1 << 17;
constexpr int kWinDense = 4096;
constexpr int kWordsWide = kWinWide / 32;   // 4096
constexpr int kWordsDense = kWinDense / 32; // 128

__device__ __forceinline__ void insertion_sort_u16(uint16_t* bp, uint32_t s0, uint32_t e0) {
  for (uint32_t a = s0 + 1; a < e0; ++a) {
    const uint16_t kp = bp[a];
    uint32_t b = a;
    while (b > s0 && bp[b - 1] > kp) { bp[b] = bp[b - 1]; --b; }
    bp[b] = kp;
  }
}

// Order a big bucket (distinct stream positions) with one warp: mark the
// positions in a per-warp bitmap over the batch, then write them back
// ascending (ballot-free word prefix).  O(d + batch/32).
__device__ __noinline__ void warp_order_bucket(uint16_t* bp, uint32_t s0, uint32_t e0, uint32_t* wbm, int nbw, int lane) {
  for (uint32_t a = s0 + lane; a < e0; a += 32) {
    const uint32_t q = bp[a];
    atomicOr(&wbm[q >> 5], 1u << (q & 31));
  }
  __syncwarp();
  uint32_t base = s0;
  for (int w0 = 0; w0 < nbw; w0 += 32) {
    const int wd = w0 + lane;
    uint32_t bits = wd < nbw ? wbm[wd] : 0u;
    const uint32_t cnt = __popc(bits);
    const uint32_t inc = warp_incl_scan(cnt);
    uint32_t o = base + inc - cnt;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1u;
      bp[o++] = (uint16_t)(wd * 32 + b);
    }
    if (wd < nbw) wbm[wd] = 0;
    base += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncwarp();
}

// true: the reference's dense accumulator (sequential from +0.0); false: its sort accumulator
__device__ __forceinline__ bool column_seq(int ci, int64_t col, const Sem& sem, const uint32_t* __restrict__ mb) {
  if (ci == kCatDense) return true;
  if (ci == kCatSort) return false;
  const int64_t f = col >> sem.shift_num;
  return (__ldg(mb + (f >> 5)) >> (f & 31)) & 1u;
}

__device__ __noinline__ double bucket_pairwise(const double* sv, const uint16_t* bp, uint32_t s0, uint32_t e0) {
  auto x = [&](int64_t q) { return sv[bp[q]]; };
  double s = sv[bp[s0]];
  if (e0 - s0 > 1) s = __dadd_rn(s, pairwise(x, s0 + 1, e0 - s0 - 1));
  return s;
}

// value of one column bucket (positions bp[s0..e0) ascending, values staged in sv[q])
__device__ __forceinline__ double bucket_value(const double* sv, const uint16_t* bp, uint32_t s0, uint32_t e0, bool seq,
                                               double carry) {
  if (seq) {
    double s = carry;
    uint32_t a = s0;
    for (; a + 8 <= e0; a += 8) {   // independent loads first, then the ordered chain
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = sv[bp[a + u]];
#pragma unroll
      for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
    }
    for (; a < e0; ++a) s = __dadd_rn(s, sv[bp[a]]);
    return s;
  }
  return bucket_pairwise(sv, bp, s0, e0);
}

// Visit every set column of the batch bitmap: the m columns are split evenly
// over the warps by rank, and within a warp the set bits of each 32-word chunk
// are dealt to the lanes in rounds of 32 (balanced even when hub regions make a
// few words dense).  fn(c, r) gets the window-local column and its rank.
template <class Fn>
__device__ __forceinline__ void for_each_column(const uint32_t* bm, const uint32_t* wpref, int nwords, uint32_t m,
                                                const Fn& fn) {
  constexpr int NW = kNT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t r_lo = (uint32_t)(((uint64_t)m * wid) / NW), r_hi = (uint32_t)(((uint64_t)m * (wid + 1)) / NW);
  if (r_lo >= r_hi) return;
  int lo = 0, hi = nwords;   // last word with wpref <= r_lo (and a set bit at/after it)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (wpref[mid] <= r_lo) lo = mid; else hi = mid;
  }
  for (int w0 = lo; w0 < nwords; w0 += 32) {
    const int wd = w0 + lane;
    const uint32_t bits = wd < nwords ? bm[wd] : 0u;
    const uint32_t base = wd < nwords ? wpref[wd] : 0xffffffffu;
    if (__shfl_sync(0xffffffffu, base, 0) >= r_hi) break;
    const uint32_t cnt = __popc(bits);
    const uint32_t inc = warp_incl_scan(cnt);
    const uint32_t excl = inc - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    for (uint32_t g0 = 0; g0 < total; g0 += 32) {
      const uint32_t g = g0 + lane;
      int src = 0;   // lane whose word holds the g-th set bit of the chunk
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t e = __shfl_sync(0xffffffffu, excl, src + step);
        if (src + step < 32 && e <= g) src += step;
      }
      const uint32_t sbits = __shfl_sync(0xffffffffu, bits, src);
      const uint32_t sexcl = __shfl_sync(0xffffffffu, excl, src);
      const uint32_t sbase = __shfl_sync(0xffffffffu, base, src);
      if (g < total) {
        const uint32_t nth = g - sexcl;
        const uint32_t bit = __fns(sbits, 0, nth + 1);
        const uint32_t r = sbase + nth;
        if (r >= r_lo && r < r_hi) fn((uint32_t)((w0 + src) * 32 + bit), r);
      }
    }
  }
}

constexpr int kBatchWords = kCap / 32;   // 128

struct HeavyNumSmem {
  static constexpr size_t kRegion = (size_t)kWordsWide * 4 * 2;   // 64 KB: wide bitmap+prefix | dense carry
  static constexpr size_t kSmall = (size_t)kWordsDense * 4 * 3;   // dense: batch bitmap, prefix, touched
  static constexpr size_t kCntl = (size_t)kCap * 4;                // 32 KB bucket counts / offsets
  static constexpr size_t kSv = (size_t)kCap * 8;                  // 64 KB values by stream position
  static constexpr size_t kBp = (size_t)kCap * 2;                  // 16 KB bucket entries (stream positions)
  static constexpr size_t kWbm = (size_t)(kNT / 32) * kBatchWords * 4;  // 16 KB per-warp ordering bitmaps
  static constexpr size_t kK = (size_t)kKSN * 4 * 4 + (kKSN + 4) * 4 + kKSN * 8;
  static constexpr size_t kBig = ((kCap / kSmallBucket + 8) * 4 + 15) / 16 * 16;
  static constexpr size_t kScratch = 64 * 8;
  static constexpr size_t kTotal = kRegion + kSmall + kCntl + kSv + kBp + kWbm + kK + kBig + kScratch;
  static_assert(kRegion % 16 == 0 && kSmall % 16 == 0 && kCntl % 16 == 0 && kSv % 16 == 0 && kBp % 16 == 0 &&
                    kWbm % 16 == 0 && kK % 16 == 0 && kBig % 16 == 0,
                "shared-memory sections must keep 16-byte alignment");
  static_assert(kTotal <= 113 * 1024, "two CTAs per SM (228 KB shared memory per SM)");
};

struct NumCtx {
  uint32_t* bm;     // bitmap of the batch's columns (wide: kWordsWide, dense: kWordsDense)
  uint32_t* wpref;  // word prefix popcounts
  uint32_t* cntl;   // bucket counts -> ends
  double* sv;       // staged values, indexed by stream position in the batch
  uint16_t* bp;     // bucket entries: stream positions
  uint32_t* wbm;    // per-warp ordering bitmaps
  uint32_t* big;
  uint32_t* nbig;
  uint32_t* scratch;
};

// Gather stream positions [B0 + q0, B0 + q0 + kItems) of the window: column into
// registers (window-local), value into sv[q] (q = position in the batch).
struct Items {
  uint32_t c[kItems];   // window-local column, then its rank (bucket)
  int n;
};

__device__ __forceinline__ void gather_items(const KState& st, const DevCsr& B, int nk, uint32_t B0, uint32_t nb,
                                             int64_t lo, Items& it, double* sv) {
  const uint32_t q0 = threadIdx.x * kItems;
  it.n = q0 < nb ? (int)min((uint32_t)kItems, nb - q0) : 0;
  uint32_t pos[kItems];
  int tk[kItems];
  if (it.n > 0) {
    int t = kstate_find(st, nk, B0 + q0);
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      if (j < it.n) {
        const uint32_t p = B0 + q0 + j;
        while (st.koff[t + 1] <= p) ++t;
        pos[j] = st.ks[t] + (p - st.koff[t]);
        tk[j] = t;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (j < it.n) it.c[j] = (uint32_t)((int64_t)__ldg(B.col + pos[j]) - lo);
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (j < it.n) sv[q0 + j] = __dmul_rn(st.kav[tk[j]], __ldg(B.val + pos[j]));
}

// One batch through the bucket pipeline: mark -> rank -> count -> scan -> scatter.
// Returns m = distinct columns of the batch; afterwards bucket r holds the
// stream positions bp[(r ? cntl[r-1] : 0) .. cntl[r]) (unordered) and bm/wpref
// describe the columns.
__device__ __forceinline__ uint32_t bucket_batch(const NumCtx& x, Items& it, int nwords) {
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (j < it.n) atomicOr(&x.bm[it.c[j] >> 5], 1u << (it.c[j] & 31));
  __syncthreads();
  for (int w = threadIdx.x; w < nwords; w += kNT) x.wpref[w] = __popc(x.bm[w]);
  __syncthreads();
  const uint32_t m = block_scan_striped<kNT>(x.wpref, nwords, x.scratch);
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (j < it.n) {
      const uint32_t w = it.c[j] >> 5, bit = 1u << (it.c[j] & 31);
      it.c[j] = x.wpref[w] + __popc(x.bm[w] & (bit - 1u));
      atomicAdd(&x.cntl[it.c[j]], 1u);
    }
  }
  __syncthreads();
  block_scan_striped<kNT>(x.cntl, (int)m, x.scratch);
  const uint32_t q0 = threadIdx.x * kItems;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (j < it.n) {
      const uint32_t slot = atomicAdd(&x.cntl[it.c[j]], 1u);
      x.bp[slot] = (uint16_t)(q0 + j);
    }
  }
  __syncthreads();
  return m;
}

// Big buckets (hub columns): one warp each puts the bucket into stream order,
// then lane 0 runs the ordered sum; finish(c, r, s0, e0) is called by lane 0.
template <class Finish>
__device__ __forceinline__ void big_buckets(const NumCtx& x, uint32_t nb, const Finish& finish) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nbw = (int)((nb + 31) >> 5);
  for (uint32_t b = wid; b < *x.nbig; b += kNT / 32) {
    const uint32_t c = x.big[b] >> 13, r = x.big[b] & 8191u;
    const uint32_t s0 = r ? x.cntl[r - 1] : 0u, e0 = x.cntl[r];
    warp_order_bucket(x.bp, s0, e0, x.wbm + wid * kBatchWords, nbw, lane);
    if (lane == 0) finish(c, r, s0, e0);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kNT, 2)
k_heavy_numeric(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows, const int8_t* __restrict__ cat,
                const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, Sem sem,
                const uint32_t* __restrict__ modebits, const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
                double* __restrict__ c_val, uint32_t* __restrict__ gk, int64_t gk_stride,
                unsigned long long* __restrict__ work, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* sp = smem;
  NumCtx x;
  unsigned char* region = sp; sp += HeavyNumSmem::kRegion;
  uint32_t* small = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kSmall;
  x.cntl = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kCntl;
  x.sv = reinterpret_cast<double*>(sp); sp += HeavyNumSmem::kSv;
  x.bp = reinterpret_cast<uint16_t*>(sp); sp += HeavyNumSmem::kBp;
  x.wbm = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kWbm;
  unsigned char* kb = sp; sp += HeavyNumSmem::kK;
  x.big = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kBig;
  x.scratch = reinterpret_cast<uint32_t*>(sp);
  int64_t* scratch64 = reinterpret_cast<int64_t*>(sp);
  __shared__ int64_t s_row;
  __shared__ uint32_t s_nbig;
  x.nbig = &s_nbig;
  uint32_t* wide_bm = reinterpret_cast<uint32_t*>(region);
  uint32_t* wide_pref = wide_bm + kWordsWide;
  double* dense_acc = reinterpret_cast<double*>(region);
  uint32_t* dense_bm = small;
  uint32_t* dense_pref = small + kWordsDense;
  uint32_t* dense_tb = small + 2 * kWordsDense;

  for (int i = threadIdx.x; i < kWordsWide; i += kNT) wide_bm[i] = 0;
  for (int i = threadIdx.x; i < 3 * kWordsDense; i += kNT) small[i] = 0;
  for (int i = threadIdx.x; i < kCap; i += kNT) x.cntl[i] = 0;
  for (int i = threadIdx.x; i < (kNT / 32) * kBatchWords; i += kNT) x.wbm[i] = 0;
  __syncthreads();
  PH_INIT

  while (true) {
    if (threadIdx.x == 0) s_row = (int64_t)atomicAdd(work, 1ull);
    __syncthreads();
    const int64_t w = s_row;
    __syncthreads();
    if (w >= nrows) break;
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    const int nk = (int)(a1 - a0);
    KState st;
    if (nk <= kKSN) {
      st.ks = reinterpret_cast<uint32_t*>(kb);
      st.ke = st.ks + kKSN;
      st.kend = st.ke + kKSN;
      st.koff = st.kend + kKSN;
      st.kav = reinterpret_cast<double*>(st.koff + kKSN + 4);
    } else {
      uint32_t* g = gk + (size_t)blockIdx.x * (size_t)gk_stride * 6;
      st.ks = g;
      st.ke = g + gk_stride;
      st.kend = g + 2 * gk_stride;
      st.koff = g + 3 * gk_stride;
      st.kav = reinterpret_cast<double*>(g + 4 * gk_stride);
      PH_COUNT(12, 1);
    }
    PH(9);
    kstate_load<kNT>(st, A, B, a0, nk);
    const int ci = cat[i];
    const uint32_t* mb = modebits + (size_t)w * sem.mode_words;
    const int64_t row_hi = mx[i];
    const int64_t out0 = c_rp[i], out_n = c_rp[i + 1] - out0;
    int64_t written = 0;
    int64_t lo = mn[i];
    int64_t wnext = kWinWide;
    __syncthreads();
    while (lo <= row_hi) {
      // ---- choose the window
      int64_t width = wnext;
      uint32_t S;
      bool hi_all;
      while (true) {
        hi_all = lo + width > row_hi;
        S = kstate_segments<kNT>(st, B, nk, (uint32_t)(hi_all ? 0 : lo + width), hi_all, x.scratch);
        PH_COUNT(13, 1);
        if (S <= kCap || width == 1) break;
        if (width > kWinDense) {
          int64_t nw = kWinDense;
          while (nw * 2 <= width / 2 && (double)S * (double)(nw * 2) / (double)width <= 0.75 * kCap) nw *= 2;
          width = nw;
          continue;
        }
        bool pw = false;
        if (ci == kCatSort) {
          pw = true;
        } else if (ci != kCatDense) {
          const int64_t f0 = lo >> sem.shift_num, f1 = (min(lo + width, row_hi + 1) - 1) >> sem.shift_num;
          for (int64_t f = f0 + threadIdx.x; f <= f1; f += kNT)
            if (!((__ldg(mb + (f >> 5)) >> (f & 31)) & 1u)) pw = true;
        }
        if (!__syncthreads_or(pw)) break;
        width >>= 1;
      }
      PH(0);
      PH_COUNT(10, 1);
      PH_COUNT(14, S);
      const int64_t wend = hi_all ? row_hi + 1 : lo + width;
      const int wcols = (int)(wend - lo);
      const int nwords = (wcols + 31) >> 5;
      if (S <= kCap) {
        // ---- wide window: one batch, buckets indexed by output rank
        x.bm = wide_bm;
        x.wpref = wide_pref;
        Items it;
        gather_items(st, B, nk, 0, S, lo, it, x.sv);
        PH(1);
        const uint32_t m = bucket_batch(x, it, nwords);
        PH(2);
        if (threadIdx.x == 0) *x.nbig = 0;
        __syncthreads();
        for_each_column(x.bm, x.wpref, nwords, m, [&](uint32_t c, uint32_t r) {
          const uint32_t s0 = r ? x.cntl[r - 1] : 0u, e0 = x.cntl[r];
          if (e0 - s0 > kSmallBucket) {
            x.big[atomicAdd(x.nbig, 1u)] = (c << 13) | r;
          } else {
            const bool seq = column_seq(ci, lo + c, sem, mb);
            insertion_sort_u16(x.bp, s0, e0);
            const double v = bucket_value(x.sv, x.bp, s0, e0, seq, 0.0);
            const int64_t o = written + r;
            if (o < out_n) {
              c_col[out0 + o] = (uint32_t)(lo + c);
              c_val[out0 + o] = v;
            }
          }
        });
        __syncthreads();
        PH(3);
        big_buckets(x, S, [&](uint32_t c, uint32_t r, uint32_t s0, uint32_t e0) {
          const double v = bucket_value(x.sv, x.bp, s0, e0, column_seq(ci, lo + c, sem, mb), 0.0);
          const int64_t o = written + r;
          if (o < out_n) {
            c_col[out0 + o] = (uint32_t)(lo + c);
            c_val[out0 + o] = v;
          }
        });
        __syncthreads();
        for (int wd = threadIdx.x; wd < nwords; wd += kNT) x.bm[wd] = 0;
        for (uint32_t r = threadIdx.x; r < m; r += kNT) x.cntl[r] = 0;
        written += m;
        PH(15);
      } else {
        // ---- dense window: batches with a per-column carry (sequential association)
        x.bm = dense_bm;
        x.wpref = dense_pref;
        for (uint32_t B0 = 0; B0 < S; B0 += kCap) {
          const uint32_t nb = min((uint32_t)kCap, S - B0);
          PH_COUNT(11, 1);
          Items it;
          gather_items(st, B, nk, B0, nb, lo, it, x.sv);
          PH(4);
          const uint32_t m = bucket_batch(x, it, nwords);
          PH(5);
          if (threadIdx.x == 0) *x.nbig = 0;
          __syncthreads();
          for_each_column(x.bm, x.wpref, nwords, m, [&](uint32_t c, uint32_t r) {
            const uint32_t s0 = r ? x.cntl[r - 1] : 0u, e0 = x.cntl[r];
            if (e0 - s0 > kSmallBucket) {
              x.big[atomicAdd(x.nbig, 1u)] = (c << 13) | r;
            } else {
              const bool had = (dense_tb[c >> 5] >> (c & 31)) & 1u;
              insertion_sort_u16(x.bp, s0, e0);
              dense_acc[c] = bucket_value(x.sv, x.bp, s0, e0, true, had ? dense_acc[c] : 0.0);
            }
          });
          __syncthreads();
          big_buckets(x, nb, [&](uint32_t c, uint32_t r, uint32_t s0, uint32_t e0) {
            const bool had = (dense_tb[c >> 5] >> (c & 31)) & 1u;
            dense_acc[c] = bucket_value(x.sv, x.bp, s0, e0, true, had ? dense_acc[c] : 0.0);
          });
          __syncthreads();
          for (int wd = threadIdx.x; wd < nwords; wd += kNT) {
            dense_tb[wd] |= x.bm[wd];
            x.bm[wd] = 0;
          }
          for (uint32_t r = threadIdx.x; r < m; r += kNT) x.cntl[r] = 0;
          __syncthreads();
          PH(6);
        }
        // emit every column touched by the window, ascending
        for (int wd = threadIdx.x; wd < nwords; wd += kNT) x.wpref[wd] = __popc(dense_tb[wd]);
        __syncthreads();
        const uint32_t nout = block_scan_striped<kNT>(x.wpref, nwords, x.scratch);
        for (int c = threadIdx.x; c < wcols; c += kNT) {
          const uint32_t word = dense_tb[c >> 5], bit = 1u << (c & 31);
          if (word & bit) {
            const int64_t o = written + x.wpref[c >> 5] + __popc(word & (bit - 1u));
            if (o < out_n) {
              c_col[out0 + o] = (uint32_t)(lo + c);
              c_val[out0 + o] = dense_acc[c];
            }
          }
        }
        __syncthreads();
        for (int wd = threadIdx.x; wd < nwords; wd += kNT) dense_tb[wd] = 0;
        for (int q = threadIdx.x; q < kWordsWide * 2; q += kNT) wide_bm[q] = 0;   // region back to a clean bitmap
        written += nout;
        PH(7);
      }
      wnext = width < kWinWide ? width * 2 : kWinWide;
      const int64_t nxt = kstate_advance<kNT>(st, B, nk, scratch64);
      lo = nxt == INT64_MAX ? row_hi + 1 : (nxt > wend ? nxt : wend);
      PH(8);
    }
    if (threadIdx.x == 0 && written != out_n) atomicOr(err, 2ull);
    __syncthreads();
  }
  PH_FLUSH;
}

}  // namespace mg
