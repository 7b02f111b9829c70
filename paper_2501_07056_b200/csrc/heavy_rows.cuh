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
#include "binned_rows.cuh"
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
constexpr int kNT = 512;                // numeric: threads per CTA (2 CTAs / SM, 32 warps)
constexpr int kCap = 4096;              // numeric: stream elements per batch
constexpr int kItems = kCap / kNT;      // 16 stream elements per thread per batch
constexpr int kSymItems = 16;           // symbolic: stream elements per thread per tile
#ifndef MG_SYM_KS
#define MG_SYM_KS 512
#endif
#ifndef MG_SYM_WINLOG
#define MG_SYM_WINLOG 19
#endif
#ifndef MG_SYM_CHUNK
#define MG_SYM_CHUNK 2048
#endif
#ifndef MG_SYM_CTAS
#define MG_SYM_CTAS 2
#endif
constexpr int kSymCtas = MG_SYM_CTAS;   // symbolic: CTAs per SM
constexpr int kKS = MG_SYM_KS;          // symbolic: k's whose cursors live in shared memory
constexpr int kKSN = 256;               // numeric: k's whose cursors live in shared memory
constexpr int kSymWin = 1 << MG_SYM_WINLOG;   // symbolic window width (columns; 64 KB bitmap)
constexpr int kChunkSmem = MG_SYM_CHUNK;      // numeric-plan chunk / bin counters kept in smem (symbolic)

// first index in [lo, hi) with col[idx] >= key, galloping from lo (segment ends
// are usually a few elements past the cursor).  Long hops go over the skip list
// (every 32nd column of B) so a hub row costs ~log2(distance/32) probes of a
// dense index plus one 128-byte line, not log2(distance) scattered misses.
__device__ __forceinline__ uint32_t gallop_col(const DevCsr& B, uint32_t lo, uint32_t hi, uint32_t key) {
  const uint32_t* __restrict__ col = B.col;
  if (lo >= hi || __ldg(col + lo) >= key) return lo;
  const uint32_t blk_end = (lo | 31u) + 1u;   // first block head after lo
  if (blk_end >= hi || __ldg(B.skip + (blk_end >> 5)) >= key) return lower_bound_col(col, lo + 1, min(blk_end, hi), key);
  uint32_t jlo = blk_end >> 5;                // col[32*jlo] < key
  const uint32_t jmax = (hi - 1) >> 5;        // last block head inside [lo, hi)
  uint32_t jhi = jmax + 1, step = 1;
  while (true) {
    const uint32_t j = jlo + step;
    if (j > jmax) break;
    if (__ldg(B.skip + j) >= key) { jhi = j; break; }
    jlo = j;
    step <<= 1;
  }
  while (jhi - jlo > 1) {
    const uint32_t mid = (jlo + jhi) >> 1;
    if (__ldg(B.skip + mid) < key) jlo = mid; else jhi = mid;
  }
  return lower_bound_col(col, jlo * 32u + 1u, min(jhi * 32u, hi), key);
}

// Per-row k state: cursor (next B position in this row), segment end in the
// current window, exclusive stream offset, B row end, A value.
struct KState {
  uint32_t* ks;
  uint32_t* ke;
  uint32_t* koff;  // nk + 1
  uint32_t* kend;
  double* kav;
  uint32_t* knext;  // column at the cursor (0xffffffff when the B row is exhausted)
};

template <int T>
__device__ __forceinline__ void kstate_load(const KState& st, const DevCsr& A, const DevCsr& B, int64_t a0, int nk) {
  for (int t = threadIdx.x; t < nk; t += T) {
    const int64_t k = __ldg(A.col + a0 + t);
    const uint32_t b0 = (uint32_t)B.rp(k), b1 = (uint32_t)B.rp(k + 1);
    st.ks[t] = b0;
    st.kend[t] = b1;
    st.kav[t] = __ldg(A.val + a0 + t);
    st.knext[t] = b0 < b1 ? __ldg(B.col + b0) : 0xffffffffu;
  }
}

// Segment ends for window [lo, hi); returns the stream length of the window.
// hi_all: the window reaches past the row's last column (no search needed).
template <int T>
__device__ __forceinline__ uint32_t kstate_segments(const KState& st, const DevCsr& B, int nk, uint32_t hi, bool hi_all,
                                                    uint32_t* scratch) {
  for (int t = threadIdx.x; t < nk; t += T) {
    const uint32_t s = st.ks[t], e0 = st.kend[t];
    // a k whose next column is already past the window contributes nothing: no search
    const uint32_t e = hi_all ? e0 : (st.knext[t] >= hi ? s : gallop_col(B, s, e0, hi));
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
    if (e != st.ks[t]) {
      st.ks[t] = e;
      st.knext[t] = e < st.kend[t] ? __ldg(B.col + e) : 0xffffffffu;
    }
    const uint32_t c = st.knext[t];
    if (c != 0xffffffffu && (int64_t)c < nxt) nxt = c;
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
  static constexpr size_t kChunk = kChunkSmem * 4 * 2;                   // 64 KB: elements + distinct columns per chunk
  static constexpr size_t kK = (size_t)kKS * 4 * 5 + (kKS + 4) * 4 + kKS * 8;
  static constexpr size_t kScratch = 64 * 8;
  static constexpr size_t kTotal = kBitmap + kChunk + kK + kScratch;
  static_assert(kBitmap % 16 == 0 && kChunk % 16 == 0 && kK % 16 == 0, "16-byte aligned sections");
  static_assert(kTotal + 64 <= 232448 / kSymCtas - 1024, "kSymCtas CTAs fit one SM's shared memory");
};

__global__ void __launch_bounds__(kHT, kSymCtas)
k_heavy_symbolic(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows, const int8_t* __restrict__ cat,
                 const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, Sem sem, int64_t* __restrict__ counts,
                 uint32_t* __restrict__ modebits, uint32_t* __restrict__ gk, int64_t gk_stride,
                 uint32_t* __restrict__ gchunk, unsigned long long* __restrict__ work, int binned, int64_t ncnt,
                 const int64_t* __restrict__ choff, uint32_t* __restrict__ ce, uint32_t* __restrict__ cd,
                 uint32_t* __restrict__ cbm_pool, uint32_t* __restrict__ cbm_slot, uint64_t cbm_cap) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(smem);
  uint32_t* ccnt_s = reinterpret_cast<uint32_t*>(smem + HeavySymSmem::kBitmap);
  unsigned char* kb = smem + HeavySymSmem::kBitmap + HeavySymSmem::kChunk;
  int64_t* scratch64 = reinterpret_cast<int64_t*>(kb + HeavySymSmem::kK);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(scratch64);
  __shared__ int64_t s_row;

  for (int i = threadIdx.x; i < kSymWin / 32; i += kHT) bitmap[i] = 0;
  for (int i = threadIdx.x; i < 2 * kChunkSmem; i += kHT) ccnt_s[i] = 0;
  // ncnt counters per array: numeric-plan chunks (mode bits), or column bins (binned numeric path)
  uint32_t* ccnt_g = gchunk + (size_t)blockIdx.x * (size_t)ncnt * 2;
  const bool chunk_in_smem = ncnt <= kChunkSmem;
  uint32_t* ccnt = chunk_in_smem ? ccnt_s : ccnt_g;                      // elements per chunk / bin
  uint32_t* dcnt = chunk_in_smem ? ccnt_s + kChunkSmem : ccnt_g + ncnt;  // distinct columns per bin
  const int shift = binned ? bin_shift_of(sem.shift_num) : sem.shift_num;
  const int wpc = shift >= 5 ? 1 << (shift - 5) : 1;   // bitmap words per bin (binned: windows are bin aligned)
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
      st.knext = reinterpret_cast<uint32_t*>(st.kav + kKS);
    } else {
      uint32_t* g = gk + (size_t)blockIdx.x * (size_t)gk_stride * 7;
      st.ks = g;
      st.ke = g + gk_stride;
      st.kend = g + 2 * gk_stride;
      st.koff = g + 3 * gk_stride;
      st.kav = reinterpret_cast<double*>(g + 4 * gk_stride);
      st.knext = g + 6 * gk_stride;
    }
    kstate_load<kHT>(st, A, B, a0, nk);
    const int ci = cat[i];
    const bool need_modes = !binned && (ci == kCatFine || ci == kCatCoarse);
    const bool need_counts = need_modes || binned;
    const int64_t row_lo = mn[i], row_hi = mx[i];
    const int64_t cmask = binned ? ~(((int64_t)1 << shift) - 1) : ~(int64_t)0;
    int64_t lo = row_lo & cmask;
    uint64_t total = 0;
    __syncthreads();
    while (lo <= row_hi) {
      const int64_t hi = lo + kSymWin;
      const bool hi_all = hi > row_hi;
      const uint32_t S = kstate_segments<kHT>(st, B, nk, (uint32_t)(hi_all ? 0 : hi), hi_all, scratch);
      // stream elements: blocked assignment, one search per thread per tile
      for (uint32_t t0 = 0; t0 < S; t0 += kHT * kSymItems) {
        const uint32_t q0 = t0 + threadIdx.x * kSymItems;
        if (q0 < S) {
          int t = kstate_find(st, nk, q0);
          // consecutive elements mostly share a bitmap word and a chunk: combine in
          // registers, one shared-memory atomic per change
          uint32_t wword = 0xffffffffu, wbits = 0, cchunk = 0xffffffffu, ccount = 0;
          for (uint32_t q = q0; q < min(S, q0 + kSymItems); ++q) {
            while (st.koff[t + 1] <= q) ++t;
            const uint32_t pos = st.ks[t] + (q - st.koff[t]);
            const uint32_t c = __ldg(B.col + pos);
            const uint32_t lc = (uint32_t)(c - lo);
            if ((lc >> 5) != wword) {
              if (wbits) atomicOr(&bitmap[wword], wbits);
              wword = lc >> 5;
              wbits = 0;
            }
            wbits |= 1u << (lc & 31);
            if (need_counts) {
              const uint32_t f = c >> shift;
              if (f != cchunk) {
                if (ccount) atomicAdd(&ccnt[cchunk], ccount);
                cchunk = f;
                ccount = 0;
              }
              ++ccount;
            }
          }
          if (wbits) atomicOr(&bitmap[wword], wbits);
          if (ccount) atomicAdd(&ccnt[cchunk], ccount);
        }
      }
      __syncthreads();
      const int64_t width = (hi_all ? row_hi + 1 : hi) - lo;
      const int words = (int)((width + 31) >> 5);
      uint32_t pc = 0;
      if (binned) {
        // per-chunk distinct counts: one warp per chunk of the window
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (wpc <= 32) {
          // a warp covers 32 consecutive words = 32 / wpc whole bins; segmented lane sums
          for (int w0 = wid * 32; w0 < words; w0 += kHT) {
            const int wd = w0 + lane;
            uint32_t cp = 0;
            if (wd < words) {
              cp = __popc(bitmap[wd]);
              bitmap[wd] = 0;
            }
            for (int o = wpc >> 1; o > 0; o >>= 1) cp += __shfl_xor_sync(0xffffffffu, cp, o);
            if ((lane & (wpc - 1)) == 0 && cp) {
              dcnt[(lo >> shift) + wd / wpc] += cp;
              pc += cp;
            }
          }
        } else {
          const int nchw = (words + wpc - 1) / wpc;
          for (int cj = wid; cj < nchw; cj += kHT / 32) {
            // a chunk too big for the sort reducer: its column bitmap is kept for the
            // dense reducer (k_bin_big), which then needs no marking pass of its own
            const int64_t f = (lo >> shift) + cj;
            const bool big = cbm_pool != nullptr && ccnt[f] > (uint32_t)kBinE;
            uint32_t slot = 0xffffffffu;
            if (big) {
              if (lane == 0) slot = (uint32_t)min((unsigned long long)0xffffffffu, atomicAdd(work + 2, 1ull));
              slot = __shfl_sync(0xffffffffu, slot, 0);
              if (slot >= cbm_cap) slot = 0xffffffffu;
              if (lane == 0) cbm_slot[choff[w] + (f - (row_lo >> shift))] = slot;
            }
            uint32_t* dst = slot != 0xffffffffu ? cbm_pool + (size_t)slot * wpc : nullptr;
            uint32_t cp = 0;
            for (int wd = cj * wpc + lane; wd < min(words, (cj + 1) * wpc); wd += 32) {
              cp += __popc(bitmap[wd]);
              if (dst) dst[wd - cj * wpc] = bitmap[wd];
              bitmap[wd] = 0;
            }
            // a chunk cut by the row's last column: the rest of its words are empty
            if (dst)
              for (int wd = max(words, cj * wpc) + lane; wd < (cj + 1) * wpc; wd += 32) dst[wd - cj * wpc] = 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cp += __shfl_xor_sync(0xffffffffu, cp, o);
            if (lane == 0 && cp) dcnt[(lo >> shift) + cj] += cp;
            pc += lane == 0 ? cp : 0u;
          }
        }
      } else {
        for (int wd = threadIdx.x; wd < words; wd += kHT) {
          pc += __popc(bitmap[wd]);
          bitmap[wd] = 0;
        }
      }
      total += block_sum<kHT>(pc, scratch);
      const int64_t nxt = kstate_advance<kHT>(st, B, nk, scratch64);
      lo = nxt == INT64_MAX ? row_hi + 1 : (nxt & cmask);
    }
    if (threadIdx.x == 0) counts[i] = (int64_t)total;
    const int64_t f0 = row_lo >> shift, f1 = row_hi >> shift;
    if (need_modes) {
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
    }
    __syncthreads();
    if (binned) {
      // chunk tables of this row: exclusive prefixes (buffer offsets / C offsets) + totals
      const int nch = (int)(f1 - f0 + 1);
      const int64_t eo = choff[w];
      const uint32_t te = block_scan_striped<kHT>(ccnt + f0, nch, scratch);
      const uint32_t td = block_scan_striped<kHT>(dcnt + f0, nch, scratch);
      for (int j = threadIdx.x; j < nch; j += kHT) {
        ce[eo + j] = ccnt[f0 + j];
        cd[eo + j] = dcnt[f0 + j];
        ccnt[f0 + j] = 0;
        dcnt[f0 + j] = 0;
      }
      if (threadIdx.x == 0) {
        ce[eo + nch] = te;
        cd[eo + nch] = td;
      }
    } else if (need_modes) {
      for (int64_t f = f0 + threadIdx.x; f <= f1; f += kHT) ccnt[f] = 0;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ numeric
// Per CTA, one row at a time, window by window.  A window's stream (ascending
// k) is staged in shared memory in batches of kCap elements and stably sorted
// by column with a block-wide LSD radix sort (warp ballot ranking, per-warp
// digit histograms): after the sort every column's contributions are one run
// in ascending k, which is exactly the order the reference adds them in.
//  * "wide" window (whole stream fits one batch, up to 2^17 columns): columns
//    are first compacted to ranks through a bitmap (rank = word prefix +
//    popcount), the sort key is the rank (< 8192, 13 bits, 2 passes) and each
//    run is reduced straight to its output slot; pairwise columns allowed.
//  * "dense" window (stream > kCap, <= 4096 columns, sequential association
//    only -- windows holding pairwise columns are narrowed until they fit one
//    batch): key = window-local column (12 bits), runs add into a per-column
//    carry; the touched columns are emitted when the window is done.
constexpr int kWinWide = 1 << 16;
constexpr int kWinDense = 2048;
constexpr int kWordsWide = kWinWide / 32;   // 2048
constexpr int kWordsDense = kWinDense / 32; // 64
constexpr int kRadixBits = 6;
constexpr int kRadix = 1 << kRadixBits;     // 64 digits
constexpr int kNW = kNT / 32;               // 16 warps
constexpr int kWaves = kCap / kNT;          // 16 waves of 32 per warp

// Staging is lane-consecutive (item v of thread t = position v*kNT + t): coalesced
// reads of B and conflict-free shared-memory stores, no padding needed.
__device__ __forceinline__ uint32_t pad_v(uint32_t q) { return q; }
__device__ __forceinline__ uint32_t pad_k(uint32_t q) { return q; }

// true: the reference's dense accumulator (sequential from +0.0); false: its sort accumulator
__device__ __forceinline__ bool column_seq(int ci, int64_t col, const Sem& sem, const uint32_t* __restrict__ mb) {
  if (ci == kCatDense) return true;
  if (ci == kCatSort) return false;
  const int64_t f = col >> sem.shift_num;
  return (__ldg(mb + (f >> 5)) >> (f & 31)) & 1u;
}

// Sequential (ascending-k) sum of a run: values sv[pay[a]] for a in [s0, e0).
__device__ __forceinline__ double run_seq(const double* sv, const uint16_t* pay, uint32_t s0, uint32_t e0, double carry) {
  double s = carry;
  uint32_t a = s0;
  for (; a + 8 <= e0; a += 8) {   // independent loads first, then the ordered chain
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = sv[pad_v(pay[a + u])];
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
  }
  for (; a < e0; ++a) s = __dadd_rn(s, sv[pad_v(pay[a])]);
  return s;
}

__device__ __noinline__ double run_pairwise(const double* sv, const uint16_t* pay, uint32_t s0, uint32_t e0) {
  auto x = [&](int64_t q) { return sv[pad_v(pay[q])]; };
  double s = sv[pad_v(pay[s0])];
  if (e0 - s0 > 1) s = __dadd_rn(s, pairwise(x, s0 + 1, e0 - s0 - 1));
  return s;
}

// One stable LSD pass over n <= kCap (key, payload) pairs on digit (key >> shift) & (2^bits - 1).
// Warp w owns the contiguous positions [w*per, (w+1)*per), per = ceil(n/kNW) rounded to
// 32, walked in waves of 32 (stable: warps in order, waves in order, lanes in order).
template <bool PaddedIn>
__device__ __forceinline__ void radix_pass(const uint16_t* kin, const uint16_t* pin, uint16_t* kout, uint16_t* pout,
                                           uint32_t n, int shift, int bits, uint32_t* hist, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int nd = 1 << bits;
  const uint32_t per = ((n + kNW - 1) / kNW + 31) & ~31u;
  const uint32_t base0 = (uint32_t)wid * per;
  const int nwave = base0 >= n ? 0 : (int)((min(n - base0, per) + 31) / 32);
  for (int i = threadIdx.x; i < nd * kNW; i += kNT) hist[i] = 0;
  __syncthreads();
  uint32_t info[kWaves];   // digit | rank-in-wave << 8 | run count << 16 ; 0xffffffff = empty lane
#pragma unroll
  for (int wv = 0; wv < kWaves; ++wv) {
    info[wv] = 0xffffffffu;
    if (wv < nwave) {
      const uint32_t i = base0 + wv * 32 + lane;
      const bool valid = i < n;
      const uint32_t d = valid ? ((uint32_t)kin[PaddedIn ? pad_k(i) : i] >> shift) & (uint32_t)(nd - 1) : 0u;
      uint32_t peers = __ballot_sync(0xffffffffu, valid);
      for (int b = 0; b < bits; ++b) {
        const uint32_t m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? m : ~m;
      }
      const uint32_t rank = __popc(peers & lt);
      if (valid && rank == 0) hist[d * kNW + wid] += __popc(peers);
      if (valid) info[wv] = d | (rank << 8) | ((uint32_t)__popc(peers) << 16);
      __syncwarp();   // next wave's leaders may update the same counter
    }
  }
  __syncthreads();
  block_scan_striped<kNT>(hist, nd * kNW, scratch);
#pragma unroll
  for (int wv = 0; wv < kWaves; ++wv) {
    if (wv < nwave) {
      const uint32_t f = info[wv];
      const uint32_t i = base0 + wv * 32 + lane;
      uint32_t base = 0;
      if (f != 0xffffffffu) {
        base = hist[(f & 0xffu) * kNW + wid];
        const uint32_t pos = base + ((f >> 8) & 0xffu);
        kout[pos] = kin[PaddedIn ? pad_k(i) : i];
        pout[pos] = pin[PaddedIn ? pad_k(i) : i];
      }
      __syncwarp();
      if (f != 0xffffffffu && ((f >> 8) & 0xffu) == 0u) hist[(f & 0xffu) * kNW + wid] = base + (f >> 16);
      __syncwarp();
    }
  }
  __syncthreads();
}

struct HeavyNumSmem {
  static constexpr size_t kSv = (size_t)kCap * 8;                  // values by stream position
  static constexpr size_t kKeys = (size_t)kCap * 2 * 2;             // sort keys (ping-pong)
  static constexpr size_t kPays = (size_t)kCap * 2 * 2;             // payloads = stream positions
  static constexpr size_t kRegion = (size_t)kWordsWide * 4 * 2;     // 32 KB wide bitmap+prefix | dense carry
  static constexpr size_t kTb = (size_t)kWordsDense * 4 * 2;        // dense touched bitmap + prefix
  static constexpr size_t kPw = (size_t)(kCap / 32) * 4;            // wide: pairwise flag per rank
  static constexpr size_t kHist = (size_t)kRadix * kNW * 4;         // 8 KB
  static constexpr size_t kKcnt = (size_t)kCap * 4;                 // 32 KB elements per sort key -> run starts
  static constexpr size_t kK = (size_t)kKSN * 4 * 5 + (kKSN + 4) * 4 + kKSN * 8;
  static constexpr size_t kScratch = 64 * 8;
  static constexpr size_t kTotal = kSv + kKeys + kPays + kRegion + kTb + kPw + kHist + kKcnt + kK + kScratch;
  static_assert(kSv % 16 == 0 && kKeys % 16 == 0 && kPays % 16 == 0 && kRegion % 16 == 0 && kTb % 16 == 0 &&
                    kPw % 16 == 0 && kHist % 16 == 0 && kK % 16 == 0,
                "shared-memory sections must keep 16-byte alignment");
  static_assert(kTotal <= 113 * 1024, "two CTAs per SM (228 KB shared memory per SM)");
};

// Stage stream positions [B0, B0 + nb) of the window: value into sv[q]; window-local
// column returned in c[v] for q = v*kNT + threadIdx.x (lane-consecutive: a warp reads
// 32 consecutive stream positions, i.e. contiguous pieces of B rows -> coalesced).
__device__ __forceinline__ void stage_items(const KState& st, const DevCsr& B, int nk, uint32_t B0, uint32_t nb, int64_t lo,
                                            double* sv, uint32_t* c) {
  uint32_t pos[kItems];
  int tk[kItems];
#pragma unroll
  for (int v = 0; v < kItems; ++v) {
    const uint32_t q = v * kNT + threadIdx.x;
    if (q < nb) {
      const int t = kstate_find(st, nk, B0 + q);
      pos[v] = st.ks[t] + (B0 + q - st.koff[t]);
      tk[v] = t;
    }
  }
#pragma unroll
  for (int v = 0; v < kItems; ++v) {
    const uint32_t q = v * kNT + threadIdx.x;
    if (q < nb) c[v] = (uint32_t)((int64_t)__ldg(B.col + pos[v]) - lo);
  }
#pragma unroll
  for (int v = 0; v < kItems; ++v) {
    const uint32_t q = v * kNT + threadIdx.x;
    if (q < nb) sv[q] = __dmul_rn(st.kav[tk[v]], __ldg(B.val + pos[v]));
  }
}

// After the sort, key k's run is [kcnt[k-1], kcnt[k]) (kcnt = inclusive prefix of the
// per-key element counts).  fn(k, s0, e0) for every key with a non-empty run; keys are
// dealt to threads round-robin.
template <class Fn>
__device__ __forceinline__ void for_each_key(const uint32_t* kcnt, uint32_t nkeys, const Fn& fn) {
  for (uint32_t k = threadIdx.x; k < nkeys; k += kNT) {
    const uint32_t s0 = k ? kcnt[k - 1] : 0u, e0 = kcnt[k];
    if (e0 > s0) fn(k, s0, e0);
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
  double* sv = reinterpret_cast<double*>(sp); sp += HeavyNumSmem::kSv;
  uint16_t* key0 = reinterpret_cast<uint16_t*>(sp);
  uint16_t* key1 = key0 + kCap; sp += HeavyNumSmem::kKeys;
  uint16_t* pay0 = reinterpret_cast<uint16_t*>(sp);
  uint16_t* pay1 = pay0 + kCap; sp += HeavyNumSmem::kPays;
  unsigned char* region = sp; sp += HeavyNumSmem::kRegion;
  uint32_t* dense_tb = reinterpret_cast<uint32_t*>(sp);
  uint32_t* dense_pref = dense_tb + kWordsDense; sp += HeavyNumSmem::kTb;
  uint32_t* pwbits = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kPw;
  uint32_t* hist = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kHist;
  uint32_t* kcnt = reinterpret_cast<uint32_t*>(sp); sp += HeavyNumSmem::kKcnt;
  unsigned char* kb = sp; sp += HeavyNumSmem::kK;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(sp);
  int64_t* scratch64 = reinterpret_cast<int64_t*>(sp);
  __shared__ int64_t s_row;
  uint32_t* wide_bm = reinterpret_cast<uint32_t*>(region);
  uint32_t* wide_pref = wide_bm + kWordsWide;
  double* dense_acc = reinterpret_cast<double*>(region);

  for (int i = threadIdx.x; i < kWordsWide; i += kNT) wide_bm[i] = 0;
  for (int i = threadIdx.x; i < kWordsDense; i += kNT) dense_tb[i] = 0;
  for (int i = threadIdx.x; i < kCap / 32; i += kNT) pwbits[i] = 0;
  for (int i = threadIdx.x; i < kCap; i += kNT) kcnt[i] = 0;
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
      st.knext = reinterpret_cast<uint32_t*>(st.kav + kKSN);
    } else {
      uint32_t* g = gk + (size_t)blockIdx.x * (size_t)gk_stride * 7;
      st.ks = g;
      st.ke = g + gk_stride;
      st.kend = g + 2 * gk_stride;
      st.koff = g + 3 * gk_stride;
      st.kav = reinterpret_cast<double*>(g + 4 * gk_stride);
      st.knext = g + 6 * gk_stride;
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
        S = kstate_segments<kNT>(st, B, nk, (uint32_t)(hi_all ? 0 : lo + width), hi_all, scratch);
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
        // ---- wide window: one batch; sort key = column rank
        uint32_t c[kItems];
        stage_items(st, B, nk, 0, S, lo, sv, c);
#pragma unroll
        for (int v = 0; v < kItems; ++v)
          if (v * kNT + threadIdx.x < S) atomicOr(&wide_bm[c[v] >> 5], 1u << (c[v] & 31));
        __syncthreads();
        PH(1);
        for (int wd = threadIdx.x; wd < nwords; wd += kNT) wide_pref[wd] = __popc(wide_bm[wd]);
        __syncthreads();
        const uint32_t m = block_scan_striped<kNT>(wide_pref, nwords, scratch);
#pragma unroll
        for (int v = 0; v < kItems; ++v) {
          if (v * kNT + threadIdx.x < S) {
            const uint32_t wd = c[v] >> 5, bit = 1u << (c[v] & 31);
            const uint32_t r = wide_pref[wd] + __popc(wide_bm[wd] & (bit - 1u));
            atomicAdd(&kcnt[r], 1u);
            const int64_t o = written + r;
            if (o < out_n) c_col[out0 + o] = (uint32_t)(lo + c[v]);   // same value from every contributor
            if (!column_seq(ci, lo + c[v], sem, mb)) atomicOr(&pwbits[r >> 5], 1u << (r & 31));
            c[v] = r;   // keep the rank for the election
          }
        }
        __syncthreads();
        PH(2);
        // Stable bucketing by rank without a sort: positions are visited in stream
        // (ascending-k) order in waves of kNT; inside a wave, positions sharing a
        // rank take their bucket slots one election round at a time (lowest
        // position first).  Wide windows rarely repeat a column inside a wave.
        block_scan_striped<kNT>(kcnt, (int)m, scratch);   // exclusive: bucket starts = fill cursors
        uint32_t* tag = wide_bm;                           // per-rank election tag (bitmap no longer needed)
        uint16_t* bucket = pay1;                           // positions, bucket-ordered
        for (uint32_t r = threadIdx.x; r < m; r += kNT) tag[r] = 0xffffffffu;
        __syncthreads();
#pragma unroll
        for (int v = 0; v < kItems; ++v) {
          const uint32_t p0 = v * kNT;
          if (p0 >= S) break;
          const uint32_t p = p0 + threadIdx.x;
          bool pending = p < S;
          const uint32_t r = pending ? c[v] : 0u;
          while (true) {
            if (pending) atomicMin(&tag[r], p);
            __syncthreads();
            const bool win = pending && tag[r] == p;
            if (win) bucket[kcnt[r]++] = (uint16_t)p;
            __syncthreads();
            if (win) {
              tag[r] = 0xffffffffu;
              pending = false;
            }
            if (!__syncthreads_or(pending)) break;
          }
        }
        // kcnt[r] is now the end of bucket r
        PH(3);
        for (uint32_t r = threadIdx.x; r < m; r += kNT) {
          const uint32_t s0 = r ? kcnt[r - 1] : 0u, e0 = kcnt[r];
          const bool pw = (pwbits[r >> 5] >> (r & 31)) & 1u;
          const double v = pw ? run_pairwise(sv, bucket, s0, e0) : run_seq(sv, bucket, s0, e0, 0.0);
          const int64_t o = written + r;
          if (o < out_n) c_val[out0 + o] = v;
        }
        __syncthreads();
        for (uint32_t wd = threadIdx.x; wd < max((uint32_t)nwords, m); wd += kNT) wide_bm[wd] = 0;
        for (uint32_t r = threadIdx.x; r < m; r += kNT) kcnt[r] = 0;
        for (uint32_t r = threadIdx.x; r < (m + 31) / 32; r += kNT) pwbits[r] = 0;
        written += m;
        PH(15);
      } else {
        // ---- dense window: batches sorted by window-local column, per-column carry
        for (uint32_t B0 = 0; B0 < S; B0 += kCap) {
          const uint32_t nb = min((uint32_t)kCap, S - B0);
          PH_COUNT(11, 1);
          uint32_t c[kItems];
          stage_items(st, B, nk, B0, nb, lo, sv, c);
#pragma unroll
          for (int v = 0; v < kItems; ++v) {
            const uint32_t q = v * kNT + threadIdx.x;
            if (q < nb) {
              key0[q] = (uint16_t)c[v];
              pay0[q] = (uint16_t)q;
              atomicAdd(&kcnt[c[v]], 1u);
            }
          }
          __syncthreads();
          PH(4);
          radix_pass<false>(key0, pay0, key1, pay1, nb, 0, 6, hist, scratch);
          radix_pass<false>(key1, pay1, key0, pay0, nb, 6, 5, hist, scratch);
          block_scan_striped<kNT>(kcnt, wcols, scratch);
          PH(5);
          for (int cc = threadIdx.x; cc < wcols; cc += kNT) {
            const uint32_t s0 = kcnt[cc], e0 = cc + 1 < wcols ? kcnt[cc + 1] : nb;
            if (e0 == s0) continue;
            const uint32_t bit = 1u << (cc & 31);
            const bool had = (dense_tb[cc >> 5] & bit) != 0u;
            dense_acc[cc] = run_seq(sv, pay0, s0, e0, had ? dense_acc[cc] : 0.0);
            if (!had) atomicOr(&dense_tb[cc >> 5], bit);
          }
          __syncthreads();
          for (int cc = threadIdx.x; cc < wcols; cc += kNT) kcnt[cc] = 0;
          PH(6);
        }
        // emit every column touched by the window, ascending
        for (int wd = threadIdx.x; wd < nwords; wd += kNT) dense_pref[wd] = __popc(dense_tb[wd]);
        __syncthreads();
        const uint32_t nout = block_scan_striped<kNT>(dense_pref, nwords, scratch);
        for (int cc = threadIdx.x; cc < wcols; cc += kNT) {
          const uint32_t word = dense_tb[cc >> 5], bit = 1u << (cc & 31);
          if (word & bit) {
            const int64_t o = written + dense_pref[cc >> 5] + __popc(word & (bit - 1u));
            if (o < out_n) {
              c_col[out0 + o] = (uint32_t)(lo + cc);
              c_val[out0 + o] = dense_acc[cc];
            }
          }
        }
        __syncthreads();
        // the carry overwrote the wide bitmap: clear the slots it used, then the touched bits
        for (int cc = threadIdx.x; cc < wcols; cc += kNT)
          if ((dense_tb[cc >> 5] >> (cc & 31)) & 1u) dense_acc[cc] = 0.0;
        __syncthreads();
        for (int wd = threadIdx.x; wd < nwords; wd += kNT) dense_tb[wd] = 0;
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
