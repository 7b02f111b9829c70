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

constexpr int kHT = 512;                // threads per CTA (1 CTA / SM)
constexpr int kWin = 8192;              // numeric window width (columns)
constexpr int kCap = 8192;              // stream elements per batch
constexpr int kItems = kCap / kHT;      // 16 stream elements per thread per batch
constexpr int kKS = 1024;               // k's whose cursors live in shared memory
constexpr int kSymWin = 1 << 20;        // symbolic window width (columns; 128 KB bitmap)
constexpr int kChunkSmem = 8192;        // numeric-plan chunk counters kept in smem (symbolic)

// Per-row k state: cursor (next B position in this row), segment end in the
// current window, exclusive stream offset, B row end, A value.
struct KState {
  uint32_t* ks;
  uint32_t* ke;
  uint32_t* koff;  // nk + 1
  uint32_t* kend;
  double* kav;
};

__device__ __forceinline__ void kstate_load(const KState& st, const DevCsr& A, const DevCsr& B, int64_t a0, int nk) {
  for (int t = threadIdx.x; t < nk; t += kHT) {
    const int64_t k = __ldg(A.col + a0 + t);
    st.ks[t] = (uint32_t)B.rp(k);
    st.kend[t] = (uint32_t)B.rp(k + 1);
    st.kav[t] = __ldg(A.val + a0 + t);
  }
}

// Segment ends for window [lo, hi); returns the stream length of the window.
// hi_all: the window reaches past the row's last column (no search needed).
__device__ __forceinline__ uint32_t kstate_segments(const KState& st, const DevCsr& B, int nk, uint32_t hi, bool hi_all,
                                                    uint32_t* scratch) {
  for (int t = threadIdx.x; t < nk; t += kHT) {
    const uint32_t s = st.ks[t], e0 = st.kend[t];
    const uint32_t e = hi_all ? e0 : lower_bound_col(B.col, s, e0, hi);
    st.ke[t] = e;
    st.koff[t] = e - s;
  }
  __syncthreads();
  const uint32_t tot = block_excl_scan<kHT>(st.koff, nk, scratch);
  if (threadIdx.x == 0) st.koff[nk] = tot;
  __syncthreads();
  return tot;
}

// Advance cursors to the segment ends; returns the next column any k still has (or INT64_MAX).
__device__ __forceinline__ int64_t kstate_advance(const KState& st, const DevCsr& B, int nk, int64_t* scratch64) {
  int64_t nxt = INT64_MAX;
  for (int t = threadIdx.x; t < nk; t += kHT) {
    const uint32_t e = st.ke[t];
    st.ks[t] = e;
    if (e < st.kend[t]) {
      const int64_t c = __ldg(B.col + e);
      nxt = c < nxt ? c : nxt;
    }
  }
  return block_min_i64<kHT>(nxt, scratch64);
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
    kstate_load(st, A, B, a0, nk);
    const int ci = cat[i];
    const bool need_modes = (ci == kCatFine || ci == kCatCoarse);
    const int64_t row_lo = mn[i], row_hi = mx[i];
    int64_t lo = row_lo;
    uint64_t total = 0;
    __syncthreads();
    while (lo <= row_hi) {
      const int64_t hi = lo + kSymWin;
      const bool hi_all = hi > row_hi;
      const uint32_t S = kstate_segments(st, B, nk, (uint32_t)(hi_all ? 0 : hi), hi_all, scratch);
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
      const int64_t nxt = kstate_advance(st, B, nk, scratch64);
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
struct HeavyNumSmem {
  static constexpr size_t kCnt = kWin * 4;            // 32 KB  histogram / offsets / cursors
  static constexpr size_t kAcc = kWin * 8;            // 64 KB  per-column carry
  static constexpr size_t kTouched = (kWin / 32) * 4; // 1 KB
  static constexpr size_t kRank = (kWin / 32) * 4;    // 1 KB
  static constexpr size_t kBp = kCap * 2;             // 16 KB  bucket: stream position in batch
  static constexpr size_t kBv = kCap * 8;             // 64 KB  bucket: value
  static constexpr size_t kK = (size_t)kKS * 4 * 4 + (kKS + 4) * 4 + kKS * 8;
  static constexpr size_t kScratch = 64 * 8;
  static constexpr size_t kTotal = kCnt + kAcc + kTouched + kRank + kBp + kBv + kK + kScratch;
};

__global__ void __launch_bounds__(kHT, 1)
k_heavy_numeric(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows, const int8_t* __restrict__ cat,
                const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, Sem sem,
                const uint32_t* __restrict__ modebits, const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
                double* __restrict__ c_val, uint32_t* __restrict__ gk, int64_t gk_stride,
                unsigned long long* __restrict__ work, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* sp = smem;
  double* acc = reinterpret_cast<double*>(sp); sp += HeavyNumSmem::kAcc;
  double* bv = reinterpret_cast<double*>(sp); sp += HeavyNumSmem::kBv;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kCnt;
  uint32_t* touched = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kTouched;
  uint32_t* rank = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kRank;
  uint16_t* bp = reinterpret_cast<uint16_t*>(sp); sp += HeavyNumSmem::kBp;
  unsigned char* kb = sp; sp += HeavyNumSmem::kK;
  int64_t* scratch64 = reinterpret_cast<int64_t*>(sp);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sp);
  __shared__ int64_t s_row;

  for (int c = threadIdx.x; c < kWin; c += kHT) cnt[c] = 0;
  for (int c = threadIdx.x; c < kWin / 32; c += kHT) touched[c] = 0;
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
    kstate_load(st, A, B, a0, nk);
    const int ci = cat[i];
    const uint32_t* mb = modebits + (size_t)w * sem.mode_words;
    const int64_t row_hi = mx[i];
    const int64_t out0 = c_rp[i], out_n = c_rp[i + 1] - out0;
    int64_t written = 0;
    int64_t lo = mn[i];
    __syncthreads();
    while (lo <= row_hi) {
      int64_t width = kWin;
      uint32_t S;
      bool hi_all;
      while (true) {  // narrow the window until pairwise columns fit one batch
        const int64_t hi = lo + width;
        hi_all = hi > row_hi;
        S = kstate_segments(st, B, nk, (uint32_t)(hi_all ? 0 : hi), hi_all, scratch);
        if (S <= kCap || width == 1) break;
        bool pw = false;
        if (ci == kCatSort) {
          pw = true;
        } else if (ci != kCatDense) {
          const int64_t f0 = lo >> sem.shift_num, f1 = (min(hi, row_hi + 1) - 1) >> sem.shift_num;
          for (int64_t f = f0 + threadIdx.x; f <= f1; f += kHT)
            if (!((mb[f >> 5] >> (f & 31)) & 1u)) pw = true;
        }
        if (!__syncthreads_or(pw)) break;
        width >>= 1;
      }
      const int64_t wend = hi_all ? row_hi + 1 : lo + width;
      const int wcols = (int)(wend - lo);
      const bool single = S <= kCap;
      for (uint32_t B0 = 0; B0 < S; B0 += kCap) {
        const uint32_t nb = min((uint32_t)kCap, S - B0);
        // 1) histogram
        const uint32_t q0 = threadIdx.x * kItems;
        int t0 = 0;
        if (q0 < nb) {
          t0 = kstate_find(st, nk, B0 + q0);
          int t = t0;
          for (uint32_t q = q0; q < min(nb, q0 + kItems); ++q) {
            const uint32_t p = B0 + q;
            while (st.koff[t + 1] <= p) ++t;
            const uint32_t c = __ldg(B.col + st.ks[t] + (p - st.koff[t]));
            atomicAdd(&cnt[c - (uint32_t)lo], 1u);
          }
        }
        __syncthreads();
        block_excl_scan<kHT>(cnt, wcols, scratch);
        // 2) scatter (cnt[c] becomes the end of bucket c)
        if (q0 < nb) {
          int t = t0;
          for (uint32_t q = q0; q < min(nb, q0 + kItems); ++q) {
            const uint32_t p = B0 + q;
            while (st.koff[t + 1] <= p) ++t;
            const uint32_t pos = st.ks[t] + (p - st.koff[t]);
            const uint32_t c = __ldg(B.col + pos);
            const double v = __dmul_rn(st.kav[t], __ldg(B.val + pos));
            const uint32_t slot = atomicAdd(&cnt[c - (uint32_t)lo], 1u);
            bp[slot] = (uint16_t)q;
            bv[slot] = v;
          }
        }
        __syncthreads();
        // 3) per column: restore stream order, accumulate
        for (int c = threadIdx.x; c < wcols; c += kHT) {
          const uint32_t s0 = c ? cnt[c - 1] : 0u, e0 = cnt[c];
          if (s0 == e0) continue;
          for (uint32_t a = s0 + 1; a < e0; ++a) {  // insertion sort by stream position
            const uint16_t kp = bp[a];
            const double kv = bv[a];
            uint32_t b = a;
            while (b > s0 && bp[b - 1] > kp) { bp[b] = bp[b - 1]; bv[b] = bv[b - 1]; --b; }
            bp[b] = kp;
            bv[b] = kv;
          }
          const uint32_t bit = 1u << (c & 31);
          const bool was = (touched[c >> 5] & bit) != 0;
          bool seq = true;
          if (ci == kCatSort) seq = false;
          else if (ci != kCatDense) {
            const int64_t f = (lo + c) >> sem.shift_num;
            seq = (mb[f >> 5] >> (f & 31)) & 1u;
          }
          double s;
          if (seq || !single) {
            s = was ? acc[c] : 0.0;
            for (uint32_t a = s0; a < e0; ++a) s = __dadd_rn(s, bv[a]);
          } else {
            auto x = [&](int64_t q) { return bv[q]; };
            s = bv[s0];
            if (e0 - s0 > 1) s = __dadd_rn(s, pairwise(x, s0 + 1, e0 - s0 - 1));
          }
          acc[c] = s;
          if (!was) atomicOr(&touched[c >> 5], bit);
        }
        __syncthreads();
        for (int c = threadIdx.x; c < wcols; c += kHT) cnt[c] = 0;
        __syncthreads();
      }
      // emit the window's columns in ascending order
      const int words = (wcols + 31) >> 5;
      for (int wd = threadIdx.x; wd < words; wd += kHT) rank[wd] = __popc(touched[wd]);
      __syncthreads();
      const uint32_t nout = block_excl_scan<kHT>(rank, words, scratch);
      for (int c = threadIdx.x; c < wcols; c += kHT) {
        const uint32_t word = touched[c >> 5];
        const uint32_t bit = 1u << (c & 31);
        if (word & bit) {
          const int64_t r = written + rank[c >> 5] + __popc(word & (bit - 1u));
          if (r < out_n) {
            c_col[out0 + r] = (uint32_t)(lo + c);
            c_val[out0 + r] = acc[c];
          }
        }
      }
      __syncthreads();
      for (int wd = threadIdx.x; wd < words; wd += kHT) touched[wd] = 0;
      written += nout;
      const int64_t nxt = kstate_advance(st, B, nk, scratch64);
      lo = nxt == INT64_MAX ? row_hi + 1 : (nxt > wend ? nxt : wend);
    }
    if (threadIdx.x == 0 && written != out_n) atomicOr(err, 2ull);
    __syncthreads();
  }
}

}  // namespace mg
