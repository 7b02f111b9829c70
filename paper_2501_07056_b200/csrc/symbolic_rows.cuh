// Heavy rows (> 4096 products), symbolic phase for the binned / direct numeric paths:
// exact distinct-column count per row (precise prediction, reference
// magnus.py:420-456) plus, per numeric-plan fine chunk of the row, the product
// count n_f (which decides the chunk's accumulator, accumulators.py:132-134) and
// the distinct-column count (the chunk's offset in the C row).
//
// Nothing here depends on the order of the products, so the row's intermediate
// product (the concatenation of its B rows, Gustavson order) is split into equal
// contiguous ranges, one per warp, walked 32 consecutive products per wave with
// coalesced loads; a wave nearly always lies inside one B row (rows of heavy rows
// are long: R-MAT hubs), found without a search.  Columns are marked in a
// shared-memory bitmap of 2^kS2WinLog columns (one window covers the row for
// m_C <= 2^20); the words that went from zero to non-zero are listed, so the
// per-chunk distinct counts cost the touched words, not the row's column range.
// Per-chunk product counts come from run lengths of equal chunks inside a wave.
#pragma once
#include "binned_rows.cuh"
#include "common.cuh"
#include "heavy_rows.cuh"

namespace mg {

#ifndef MG_S2_T
#define MG_S2_T 1024
#endif
#ifndef MG_S2_WIN
#define MG_S2_WIN 20
#endif
#ifndef MG_S2_TOUCH
#define MG_S2_TOUCH 8192
#endif
#ifndef MG_S2_K
#define MG_S2_K 4096
#endif
constexpr int kS2T = MG_S2_T;              // threads per CTA
constexpr int kS2WinLog = MG_S2_WIN;       // bitmap window: 2^20 columns (128 KB)
constexpr int kS2Words = (1 << kS2WinLog) / 32;
constexpr int kS2Touch = MG_S2_TOUCH;             // touched-word list (full scan of the row's words beyond it)
#ifndef MG_S2_TICKET_AHEAD
#define MG_S2_TICKET_AHEAD 1
#endif
#ifndef MG_S2_DENSE4
#define MG_S2_DENSE4 2
#endif
constexpr int kS2Dense4 = MG_S2_DENSE4;  // dense window: 4 x products >= this x spanned words (< 0: never)
constexpr int kS2Chunks = 2048;            // chunk counters per row
constexpr int kS2K = MG_S2_K;                 // k's whose stream offsets live in shared memory
#ifndef MG_S2_U
#define MG_S2_U 4
#endif
constexpr int kS2U = MG_S2_U;              // waves of loads in flight per warp

struct Sym2Smem {
  static constexpr size_t kBitmap = (size_t)kS2Words * 4;
  static constexpr size_t kTouch = (size_t)kS2Touch * 4;
  static constexpr size_t kCnt = (size_t)kS2Chunks * 4 * 2;
  static constexpr size_t kK = (size_t)(kS2K + 32) * 4 * 2;
  static constexpr size_t kScratch = 64 * 8;
  static constexpr size_t kTotal = kBitmap + kTouch + kCnt + kK + kScratch;
  static_assert(kTotal <= 232448 - 1024, "fits one SM");
};

// segment [p0, p1) of B row k inside columns [lo, hi) (hi_all: no upper bound)
__device__ __forceinline__ void seg_in_window(const DevCsr& B, int64_t k, uint32_t& p0, uint32_t& p1, uint32_t lo, uint32_t hi,
                                              bool lo_all, bool hi_all, const int32_t* __restrict__ bslot,
                                              const uint32_t* __restrict__ bidx, int64_t nwin1, int ilog) {
  const int32_t sl = bslot != nullptr ? __ldg(bslot + k) : -1;
  if (sl >= 0) {
    const uint32_t* ix = bidx + (size_t)sl * nwin1;
    if (!lo_all) p0 = __ldg(ix + min((int64_t)(lo >> ilog), nwin1 - 1));
    if (!hi_all) p1 = __ldg(ix + min((int64_t)(hi >> ilog), nwin1 - 1));
  } else {
    if (!lo_all) p0 = lower_bound_col(B.col, p0, p1, lo);
    if (!hi_all) p1 = lower_bound_col(B.col, p0, p1, hi);
  }
}

// Shared-memory atomics on 32-bit shared addresses, predicated (no branch, no compiler
// warp aggregation): this loop is issue-bound.
__device__ __forceinline__ uint32_t sh_atom_or_if(bool p, uint32_t addr, uint32_t v) {
  uint32_t old = 1u;
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q atom.shared.or.b32 %0, [%1], %3;\n}\n"
               : "+r"(old) : "r"(addr), "r"((uint32_t)p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void sh_red_or_if(bool p, uint32_t addr, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q red.shared.or.b32 [%1], %2;\n}\n"
               :: "r"((uint32_t)p), "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sh_red_add_if(bool p, uint32_t addr, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q red.shared.add.u32 [%1], %2;\n}\n"
               :: "r"((uint32_t)p), "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t sh_atom_add(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;\n" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void sh_st_if(bool p, uint32_t addr, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.shared.u32 [%1], %2;\n}\n"
               :: "r"((uint32_t)p), "r"(addr), "r"(v) : "memory");
}

// One warp: stream positions [q_beg, q_end) of the window (koff: exclusive offsets of the
// row's segments, koff[nk] = total; kpos: their B positions).  Marks columns, lists the
// bitmap words that became non-zero, counts products per chunk.  KP: shared or global
// arrays (separate instantiations keep the shared-memory case on LDS).
// Track = false (dense windows): columns are marked without reading the old word back and
// no touched-word list is kept; the caller scans the window's word range instead.
template <class KP, bool Track = true>
__device__ __forceinline__ void sym2_stream(const DevCsr& B, KP koff, KP kpos, int nk, uint32_t q_beg, uint32_t q_end,
                                            uint32_t wlo, int shift, uint32_t f0, uint32_t* bm, uint32_t* touch,
                                            uint32_t* ntouch, uint32_t* ccnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t a_bm = (uint32_t)__cvta_generic_to_shared(bm), a_touch = (uint32_t)__cvta_generic_to_shared(touch),
                 a_nt = (uint32_t)__cvta_generic_to_shared(ntouch), a_cc = (uint32_t)__cvta_generic_to_shared(ccnt);
  const uint32_t lt = lanemask_lt(), le = lanemask_le();
#ifdef MG_S2_WAVE_CURSOR
  // segment of the first position: last j with koff[j] <= q_beg
  int kk = 0;
  {
    int lo = 0, hi = nk;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (koff[mid] <= q_beg) lo = mid; else hi = mid;
    }
    kk = lo;
  }
  uint32_t kend = koff[kk + 1];              // first stream position past segment kk
  uint32_t base = kpos[kk] - koff[kk];       // B position of stream position q is base + q
  for (uint32_t q00 = q_beg; q00 < q_end; q00 += 32 * kS2U) {
    uint32_t cw[kS2U];
#pragma unroll
    for (int u = 0; u < kS2U; ++u) {
      const uint32_t q0 = q00 + 32 * u, q = q0 + lane;
      uint32_t pos = base + q;
      if (q0 + 31 >= kend && q0 < q_end) {
        // the wave crosses segment boundaries: each lane finds its own segment
        int kl = kk;
        while (kl < nk && koff[kl + 1] <= q) ++kl;
        pos = kpos[kl] + (q - koff[kl]);
        kk = __shfl_sync(0xffffffffu, kl, 31);
        kend = koff[kk + 1];
        base = kpos[kk] - koff[kk];
      }
      cw[u] = q < q_end ? __ldg(B.col + pos) : 0xffffffffu;
    }
#else
  // batched segment cursor (E2Cursor::batch) and software pipelining: the column loads of the
  // next kS2U waves are in flight while the current ones update the bitmap
  E2Cursor<KP> cur{koff, kpos, nk, 0, 0, 0};
  cur.init(q_beg);
  uint32_t ncw[kS2U];
  auto fetch = [&](uint32_t q00) {
    uint32_t pos[kS2U];
    int seg[kS2U];
    bool multi[kS2U];
    cur.batch(q00, q_end, pos, seg, multi);
#pragma unroll
    for (int u = 0; u < kS2U; ++u) {
      const uint32_t q = q00 + 32 * u + lane;
      ncw[u] = q < q_end ? __ldg(B.col + pos[u]) : 0xffffffffu;
    }
  };
  fetch(q_beg);
  for (uint32_t q00 = q_beg; q00 < q_end; q00 += 32 * kS2U) {
    uint32_t cw[kS2U];
#pragma unroll
    for (int u = 0; u < kS2U; ++u) cw[u] = ncw[u];
    if (q00 + 32 * kS2U < q_end) fetch(q00 + 32 * kS2U);
#endif
#pragma unroll
    for (int u = 0; u < kS2U; ++u) {
      if (q00 + 32 * u >= q_end) break;
      const uint32_t c = cw[u];
      const bool valid = c != 0xffffffffu;
      const uint32_t lc = c - wlo;
      if (Track) {
        const bool fresh = sh_atom_or_if(valid, a_bm + ((lc >> 5) << 2), 1u << (lc & 31)) == 0u;
        const uint32_t fm = __ballot_sync(0xffffffffu, fresh);
        if (fm) {
          uint32_t b = 0;
          if (lane == 0) b = sh_atom_add(a_nt, (uint32_t)__popc(fm));
          b = __shfl_sync(0xffffffffu, b, 0);
          const uint32_t slot = b + __popc(fm & lt);
          sh_st_if(fresh && slot < (uint32_t)kS2Touch, a_touch + (slot << 2), lc >> 5);
        }
      } else {
        sh_red_or_if(valid, a_bm + ((lc >> 5) << 2), 1u << (lc & 31));
      }
      // products per chunk: runs of equal chunks (invalid lanes end the last run)
      const uint32_t ch = valid ? (c >> shift) - f0 : 0xffffffffu;   // row-relative chunk
      const uint32_t pch = __shfl_up_sync(0xffffffffu, ch, 1);
      const bool head = lane == 0 || ch != pch;
      const uint32_t hm = __ballot_sync(0xffffffffu, head);
      const uint32_t after = hm & ~le;
      const uint32_t nxt = after ? (uint32_t)(__ffs(after) - 1) : 32u;
      sh_red_add_if(valid && head, a_cc + (ch << 2), nxt - (uint32_t)lane);
    }
  }
}

__global__ void __launch_bounds__(kS2T)
k_heavy_sym2(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, int64_t nrows, const int64_t* __restrict__ mn,
             const int64_t* __restrict__ mx, int shift, int64_t* __restrict__ counts, const int64_t* __restrict__ choff,
             uint32_t* __restrict__ ce, uint32_t* __restrict__ cd, uint32_t* __restrict__ cbm_pool,
             uint32_t* __restrict__ cbm_slot, uint64_t cbm_cap, unsigned long long* __restrict__ work,
             const int32_t* __restrict__ bslot, const uint32_t* __restrict__ bidx, int64_t nwin1, int ilog,
             uint32_t* __restrict__ gk, int64_t gk_stride) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem);
  uint32_t* touch = reinterpret_cast<uint32_t*>(smem + Sym2Smem::kBitmap);
  uint32_t* ccnt = reinterpret_cast<uint32_t*>(smem + Sym2Smem::kBitmap + Sym2Smem::kTouch);
  uint32_t* dcnt = ccnt + kS2Chunks;
  uint32_t* ks_off = reinterpret_cast<uint32_t*>(smem + Sym2Smem::kBitmap + Sym2Smem::kTouch + Sym2Smem::kCnt);
  uint32_t* ks_pos = ks_off + kS2K + 32;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + Sym2Smem::kBitmap + Sym2Smem::kTouch + Sym2Smem::kCnt + Sym2Smem::kK);
  __shared__ int64_t s_row;
  __shared__ uint32_t s_ntouch;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = kS2T / 32;
  for (int i = threadIdx.x; i < kS2Words; i += kS2T) bm[i] = 0u;
  for (int i = threadIdx.x; i < 2 * kS2Chunks; i += kS2T) ccnt[i] = 0u;
  const int wpc = shift >= 5 ? 1 << (shift - 5) : 1;   // bitmap words per chunk
  __syncthreads();
#if MG_S2_TICKET_AHEAD
  // the next row is taken while the current one is marked (read after the row's barriers)
  if (threadIdx.x == 0) s_row = (int64_t)atomicAdd(work, 1ull);
  __syncthreads();
#endif
  while (true) {
#if !MG_S2_TICKET_AHEAD
    if (threadIdx.x == 0) s_row = (int64_t)atomicAdd(work, 1ull);
    __syncthreads();
#endif
    const int64_t w = s_row;
    __syncthreads();
    if (w >= nrows) break;
#if MG_S2_TICKET_AHEAD
    if (threadIdx.x == 0) s_row = (int64_t)atomicAdd(work, 1ull);
#endif
    const int64_t i = rows[w];
    const int64_t a0 = A.rp(i);
    const int nk = (int)(A.rp(i + 1) - a0);
    const int64_t row_lo = mn[i], row_hi = mx[i];
    const int64_t f0 = row_lo >> shift, f1 = row_hi >> shift;
    const int nch = (int)(f1 - f0 + 1);
    // per-k stream offsets and B positions: shared memory, or this CTA's global scratch
    uint32_t* koff = nk <= kS2K ? ks_off : gk + (size_t)blockIdx.x * gk_stride * 2;
    uint32_t* kpos = nk <= kS2K ? ks_pos : koff + gk_stride;
    const int64_t wmask = ~(((int64_t)1 << kS2WinLog) - 1);
    for (int64_t wlo = row_lo & wmask; wlo <= row_hi; wlo += (int64_t)1 << kS2WinLog) {
      const int64_t whi = wlo + ((int64_t)1 << kS2WinLog);
      const bool lo_all = wlo <= row_lo, hi_all = whi > row_hi;
      // ---- segments of the window
      for (int j = threadIdx.x; j < nk; j += kS2T) {
        const int64_t k = __ldg(A.col + a0 + j);
        uint32_t p0 = (uint32_t)B.rp(k), p1 = (uint32_t)B.rp(k + 1);
        if (!(lo_all && hi_all))
          seg_in_window(B, k, p0, p1, (uint32_t)wlo, (uint32_t)min(whi, (int64_t)0xffffffff), lo_all, hi_all, bslot, bidx,
                        nwin1, ilog);
        kpos[j] = p0;
        koff[j] = p1 - p0;
      }
      if (threadIdx.x == 0) s_ntouch = 0u;
      __syncthreads();
      const uint32_t T = block_scan_striped<kS2T>(koff, nk, scratch);
      if (threadIdx.x == 0) koff[nk] = T;   // sentinel
      __syncthreads();
      // ---- stream: warp w takes [w L, (w+1) L), L a multiple of 32
      const uint32_t L = ((T + NW - 1) / NW + 31) & ~31u;
      const uint32_t q_beg = min(T, (uint32_t)wid * L), q_end = min(T, q_beg + L);
      // dense window (4 x products >= kS2Dense4 x the bitmap words the row spans in it): no
      // touched-word list, the word range is scanned below
      const int64_t wd_lo = (max(row_lo, wlo) - wlo) >> 5, wd_hi = (min(row_hi, whi - 1) - wlo) >> 5;
      const bool dense = kS2Dense4 >= 0 && 4 * (int64_t)T >= (int64_t)kS2Dense4 * (wd_hi - wd_lo + 1);
      if (q_beg < q_end) {
        if (dense) {
          if (nk <= kS2K) sym2_stream<uint32_t*, false>(B, ks_off, ks_pos, nk, q_beg, q_end, (uint32_t)wlo, shift, (uint32_t)f0, bm, touch, &s_ntouch, ccnt);
          else sym2_stream<uint32_t*, false>(B, koff, kpos, nk, q_beg, q_end, (uint32_t)wlo, shift, (uint32_t)f0, bm, touch, &s_ntouch, ccnt);
        } else {
          if (nk <= kS2K) sym2_stream(B, ks_off, ks_pos, nk, q_beg, q_end, (uint32_t)wlo, shift, (uint32_t)f0, bm, touch, &s_ntouch, ccnt);
          else sym2_stream(B, koff, kpos, nk, q_beg, q_end, (uint32_t)wlo, shift, (uint32_t)f0, bm, touch, &s_ntouch, ccnt);
        }
      }
      __syncthreads();
      // ---- big chunks: keep their column bitmaps for the big-chunk reducer (k_bin_big)
      const int64_t wf0 = max(f0, wlo >> shift), wf1 = min(f1, (min(whi, row_hi + 1) - 1) >> shift);
      if (cbm_pool != nullptr) {
        for (int64_t f = wf0 + wid; f <= wf1; f += NW) {
          const bool big = ccnt[f - f0] > (uint32_t)kBinE;
          if (!big) continue;
          uint32_t slot = 0xffffffffu;
          if (lane == 0) slot = (uint32_t)min((unsigned long long)0xffffffffu, atomicAdd(work + 2, 1ull));
          slot = __shfl_sync(0xffffffffu, slot, 0);
          if (slot >= cbm_cap) slot = 0xffffffffu;
          if (lane == 0) cbm_slot[choff[w] + (f - f0)] = slot;
          if (slot == 0xffffffffu) continue;
          const int64_t wd0 = ((f << shift) - wlo) >> 5;   // chunk-aligned (shift >= 5)
          uint32_t* dst = cbm_pool + (size_t)slot * wpc;
          for (int t = lane; t < wpc; t += 32) dst[t] = bm[wd0 + t];
        }
        __syncthreads();
      }
      // ---- distinct columns per chunk from the touched words (clear them)
      const uint32_t nt = s_ntouch;
      if (!dense && nt <= (uint32_t)kS2Touch) {
        for (uint32_t t = threadIdx.x; t < nt; t += kS2T) {
          const uint32_t wd = touch[t];
          const uint32_t x = bm[wd];
          bm[wd] = 0u;
          if (shift >= 5) {
            atomicAdd(&dcnt[(uint32_t)(((wlo >> 5) + wd) >> (shift - 5)) - (uint32_t)f0], (uint32_t)__popc(x));
          } else {
            for (uint32_t b = 0; b < 32; b += (1u << shift)) {
              const uint32_t part = (x >> b) & ((1u << (1u << shift)) - 1u);
              if (part) atomicAdd(&dcnt[(uint32_t)((((wlo >> 5) + wd) * 32 + b) >> shift) - (uint32_t)f0], (uint32_t)__popc(part));
            }
          }
        }
      } else {
        for (int64_t wd = wd_lo + threadIdx.x; wd <= wd_hi; wd += kS2T) {
          const uint32_t x = bm[wd];
          if (!x) continue;
          bm[wd] = 0u;
          if (shift >= 5) {
            atomicAdd(&dcnt[(uint32_t)(((wlo >> 5) + wd) >> (shift - 5)) - (uint32_t)f0], (uint32_t)__popc(x));
          } else {
            for (uint32_t b = 0; b < 32; b += (1u << shift)) {
              const uint32_t part = (x >> b) & ((1u << (1u << shift)) - 1u);
              if (part) atomicAdd(&dcnt[(uint32_t)((((wlo >> 5) + wd) * 32 + b) >> shift) - (uint32_t)f0], (uint32_t)__popc(part));
            }
          }
        }
      }
      __syncthreads();
    }
    // ---- chunk tables of the row: exclusive prefixes + totals
    const int64_t eo = choff[w];
    const uint32_t te = block_scan_striped<kS2T>(ccnt, nch, scratch);
    const uint32_t td = block_scan_striped<kS2T>(dcnt, nch, scratch);
    for (int j = threadIdx.x; j < nch; j += kS2T) {
      ce[eo + j] = ccnt[j];
      cd[eo + j] = dcnt[j];
      ccnt[j] = 0u;
      dcnt[j] = 0u;
    }
    if (threadIdx.x == 0) {
      ce[eo + nch] = te;
      cd[eo + nch] = td;
      counts[i] = (int64_t)td;
    }
    __syncthreads();
  }
}

}  // namespace mg
