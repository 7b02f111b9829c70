// Big chunks of heavy rows, fused: B -> shared memory -> C, no HBM reorder buffer.
//
// A CTA sweeps a unit -- a range of one heavy row's chunks -- from left to right and reduces
// every big chunk in it; the per-unit lookups (row, A range, chunk tables, short-row cursors)
// are paid once per unit, not per chunk.
//
// The fine level (reference magnus.py:195-262, Alg. 3) histograms a row's intermediate
// columns into chunks, scatters the products stably and accumulates chunk by chunk.  For
// the big chunks (more than kBinE products: always the dense association, sequential from
// +0.0 in ascending k, accumulators.py:68-97) one CTA does all three steps for one
// (row, chunk) without leaving the SM:
//
//   segments   thread per A nonzero k: the piece of B row k inside the chunk, from the B
//              window index (two adjacent loads) or, for rows below the index threshold,
//              from a per-k cursor (position and next column) kept across the sweep.
//              Non-empty segments are compacted in k order into a round of at most kFuR
//              products (rounds keep ascending k, so any chunk size works).
//   gather     the round's stream (segments concatenated, Gustavson order,
//              gustavson.py:44-59) is split into contiguous warp ranges; every lane keeps
//              its kFuU products in registers.
//   scatter    stable counting scatter by column sub-bin (16 per chunk) into a shared-memory
//              slice per sub-bin: per-warp counts, prefix over (bin, warp), ranks inside a
//              wave by run position or match_any -- the reference's stable scatter
//              (magnus.py:236-249) at sub-chunk granularity.
//   apply      one warp per sub-bin slice adds the products in stream order to a
//              column-indexed fp64 accumulator (no ranks: the sub-bins of a chunk own
//              disjoint accumulator ranges); lanes of one wave that hit the same column are
//              applied in lane order.
//   emit       the chunk's column bitmap (kept by the symbolic pass, or marked here) gives
//              every column its place in the C row; columns and sums are written in order.
//
#pragma once
#include "big_direct.cuh"

namespace mg {

#ifndef MG_FU_T
#define MG_FU_T 256
#endif
#ifndef MG_FU_MINB
#define MG_FU_MINB 3
#endif
constexpr int kFuT = MG_FU_T;            // threads per CTA
constexpr int kFuNW = kFuT / 32;
constexpr int kFuU = 8;                  // products per lane per round (two cursor batches of 4 waves)
constexpr int kFuR = kFuT * kFuU;        // products per round
constexpr int kFuS = kFuT * 2;           // non-empty segments per round
constexpr int kFuNB = 16;                // sub-bins per chunk
constexpr int kFuMaxShift = 12;          // accumulator: 2^12 columns
constexpr int kFuKS = 2048;              // A nonzeros whose short-row cursors live in shared memory
#ifndef MG_FU_UNIT
#define MG_FU_UNIT (1 << 15)
#endif
constexpr uint32_t kFuUnit = MG_FU_UNIT; // big-chunk products per unit (a row's big chunks are swept in units)
static_assert(kFuT >= 128 && kFuT <= 1024, "emit: <= 32 columns per thread; one bitmap word per thread");

struct FuSmem {
  static constexpr size_t kAcc = (size_t)(1 << kFuMaxShift) * 8;
  static constexpr size_t kVals = (size_t)kFuR * 8;
  static constexpr size_t kAv = (size_t)kFuS * 8;
  static constexpr size_t kCols = (size_t)kFuR * 2;
  static constexpr size_t kOff = (size_t)(kFuS + 32) * 4;
  static constexpr size_t kPos = (size_t)(kFuS + 32) * 4;
  static constexpr size_t kBm = (size_t)((1 << kFuMaxShift) / 32) * 4;
  static constexpr size_t kPref = kBm;
  static constexpr size_t kCnt = (size_t)kFuNW * kFuNB * 4;
  static constexpr size_t kMisc = 64 * 4;
  static constexpr size_t kStNext = (size_t)kFuKS * 4;
  static constexpr size_t kStRel = (size_t)kFuKS;
  static constexpr size_t kTotal = kAcc + kVals + kAv + kCols + kOff + kPos + kBm + kPref + kCnt + kMisc + kStNext + kStRel;
};

// Per A nonzero p (B row k = A.col[p]): the B window-index slot of row k when it is indexed,
// else -(row length) - 1 (so an empty row is -1); and row k's start in B.
__global__ void k_fu_aprep(DevCsr A, DevCsr B, const int32_t* __restrict__ bslot, int32_t* __restrict__ aslot,
                           uint32_t* __restrict__ abase) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < A.nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = __ldg(A.col + p);
    const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
    const int32_t sl = __ldg(bslot + k);
    aslot[p] = sl >= 0 ? sl : -(int32_t)(b1 - b0) - 1;
    abase[p] = (uint32_t)b0;
  }
}

// inclusive scan of one u32 per thread over the CTA; scratch: >= kFuNW + 1 words
__device__ __forceinline__ uint32_t fu_block_incl_scan(uint32_t v, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t inc = warp_incl_scan(v);
  if (lane == 31) scratch[wid] = inc;
  __syncthreads();
  uint32_t add = 0;
#pragma unroll
  for (int w = 0; w < kFuNW; ++w) add += w < wid ? scratch[w] : 0u;
  __syncthreads();
  return inc + add;
}


// Units of heavy rows [0, nH): chunk ranges holding about kFuUnit big-chunk products, cut
// after a big chunk.  One warp per row.  Large units are listed first (list_slot).
__global__ void k_fu_plan(const int32_t* __restrict__ rows, int64_t nH, const int64_t* __restrict__ mn,
                          const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff,
                          const uint32_t* __restrict__ ce, BinItem* __restrict__ units,
                          unsigned long long* __restrict__ nunit, int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = warp; h < nH; h += nwarps) {
    const int64_t i = rows[h];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[h];
    int ustart = -1;
    uint32_t acc = 0;
    auto emit = [&](int ja, int jb, uint32_t sz) {
      if (lane == 0) {
        const bool front = sz >= kFuUnit / 2;
        const unsigned long long p = atomicAdd(nunit + (front ? 0 : 1), 1ull);
        units[front ? (int64_t)p : cap - 1 - (int64_t)p] = BinItem{(int32_t)h, ja, jb, 0};
      }
    };
    for (int q0 = 0; q0 < rb.nchunk; q0 += 32) {
      const int cj = q0 + lane;
      const uint32_t n = cj < rb.nchunk ? __ldg(e + cj + 1) - __ldg(e + cj) : 0u;
      uint32_t bigm = __ballot_sync(0xffffffffu, n > (uint32_t)kBinE);
      while (bigm) {
        const int b = __ffs(bigm) - 1;
        bigm &= bigm - 1;
        const uint32_t nb = __shfl_sync(0xffffffffu, n, b);
        if (ustart < 0) ustart = q0 + b;
        acc += nb;
        if (acc >= kFuUnit) {
          emit(ustart, q0 + b + 1, acc);
          ustart = -1;
          acc = 0;
        }
      }
    }
    if (ustart >= 0) emit(ustart, rb.nchunk, acc);
  }
}

__global__ void __launch_bounds__(kFuT, MG_FU_MINB)
k_fu_sweep(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, const int64_t* __restrict__ mn,
           const int64_t* __restrict__ mx, Sem sem, const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce,
           const uint32_t* __restrict__ cd, const uint32_t* __restrict__ cbm_slot, const uint32_t* __restrict__ cbm_pool,
           const BinItem* __restrict__ units, const unsigned long long* __restrict__ nunit, int64_t cap_units,
           unsigned long long* __restrict__ ticket, const int32_t* __restrict__ aslot, const uint32_t* __restrict__ abase,
           const uint32_t* __restrict__ bidx, int64_t nwin1, int ilog, uint32_t* __restrict__ gst, int64_t gst_stride,
           const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col, double* __restrict__ c_val,
           unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* acc = reinterpret_cast<double*>(smem);
  double* vals = reinterpret_cast<double*>(smem + FuSmem::kAcc);
  double* s_av = reinterpret_cast<double*>(smem + FuSmem::kAcc + FuSmem::kVals);
  uint16_t* cols = reinterpret_cast<uint16_t*>(smem + FuSmem::kAcc + FuSmem::kVals + FuSmem::kAv);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(smem + FuSmem::kAcc + FuSmem::kVals + FuSmem::kAv + FuSmem::kCols);
  uint32_t* s_pos = s_off + kFuS + 32;
  uint32_t* bm = s_pos + kFuS + 32;
  uint32_t* wpref = bm + (1 << kFuMaxShift) / 32;
  uint32_t* cnt = wpref + (1 << kFuMaxShift) / 32;
  uint32_t* misc = cnt + kFuNW * kFuNB;   // [0..kFuNW]: scan partials, [32..48]: bin starts, [56]: S, [57]: T, [58]: m
  uint32_t* s_next = misc + 64;
  uint8_t* s_rel = reinterpret_cast<uint8_t*>(s_next + kFuKS);
  __shared__ unsigned long long s_t;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int shift = sem.shift_num;
  const uint32_t width = 1u << shift;
  const int nwords = (int)((width + 31) / 32);
  const int bsh = shift > 4 ? shift - 4 : 0;                // sub-bin = local column >> bsh
  const int nbins = (int)(width >> bsh);                    // <= kFuNB
  const uint32_t lt = lanemask_lt(), le = lanemask_le();
  const uint64_t nu_front = nunit[0], nu = nu_front + nunit[1];
  for (uint32_t c = tid; c < width; c += kFuT) acc[c] = 0.0;
  for (int q = tid; q < kFuNW * kFuNB; q += kFuT) cnt[q] = 0u;
  __syncthreads();
  while (true) {
    if (tid == 0) s_t = atomicAdd(ticket, 1ull);
    __syncthreads();
    const unsigned long long tk = s_t;
    __syncthreads();
    if (tk >= nu) break;
    const BinItem it = units[list_slot(tk, nu_front, cap_units)];
    const int64_t i = rows[it.h];
    const int64_t a0 = A.rp(i);
    const int nk = (int)(A.rp(i + 1) - a0);
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[it.h];
    const uint32_t* d = cd + choff[it.h];
    const uint32_t* sl_tab = cbm_slot != nullptr ? cbm_slot + choff[it.h] : nullptr;
    const int64_t crp = c_rp[i];
    uint32_t* st_next = nk <= kFuKS ? s_next : gst + (size_t)blockIdx.x * gst_stride * 2;
    uint8_t* st_rel = nk <= kFuKS ? s_rel : reinterpret_cast<uint8_t*>(st_next + gst_stride);
    // ---- cursors of the rows without a window index: first entry at or after the unit's first column
    {
      const uint32_t c_first = (uint32_t)((rb.c0 + it.ja) << shift);
      for (int j = tid; j < nk; j += kFuT) {
        const int32_t sl = __ldg(aslot + a0 + j);
        if (sl < -1) {
          const uint32_t b0 = __ldg(abase + a0 + j), len = (uint32_t)(-(sl + 1));
          const uint32_t pos = it.ja > 0 ? lower_bound_col(B.col, b0, b0 + len, c_first) : b0;
          st_rel[j] = (uint8_t)(pos - b0);
          st_next[j] = pos < b0 + len ? __ldg(B.col + pos) : 0u;
        }
      }
    }
    __syncthreads();
    for (int cj0 = it.ja; cj0 < it.jb; cj0 += 32) {
      // chunk tables of the next 32 chunks (every warp reads the same words)
      const int cjl = cj0 + lane;
      uint32_t n_l = 0, m_l = 0, d_l = 0, slot_l = 0xffffffffu;
      if (cjl < it.jb) {
        n_l = __ldg(e + cjl + 1) - __ldg(e + cjl);
        d_l = __ldg(d + cjl);
        m_l = __ldg(d + cjl + 1) - d_l;
        if (sl_tab != nullptr && n_l > (uint32_t)kBinE) slot_l = __ldg(sl_tab + cjl);
      }
      uint32_t bigm = __ballot_sync(0xffffffffu, n_l > (uint32_t)kBinE);
      while (bigm) {
        const int bb = __ffs(bigm) - 1;
        bigm &= bigm - 1;
        const int cj = cj0 + bb;
        const uint32_t it_n = __shfl_sync(0xffffffffu, n_l, bb), it_m = __shfl_sync(0xffffffffu, m_l, bb);
        const int64_t out = crp + __shfl_sync(0xffffffffu, d_l, bb);
        const uint32_t bslot = __shfl_sync(0xffffffffu, slot_l, bb);
        const uint32_t c_lo = (uint32_t)((rb.c0 + cj) << shift);
        const uint64_t c_hi = (uint64_t)c_lo + width;
        const uint32_t cidx = c_lo >> ilog;
        const bool marking = bslot == 0xffffffffu;
        for (int wd = tid; wd < nwords; wd += kFuT) bm[wd] = marking ? 0u : __ldg(cbm_pool + (size_t)bslot * nwords + wd);
        // (visible to the apply / emit steps after the barriers of the first round)

        int kp = 0;              // first k of the current piece
        int jdone = kFuT;        // threads of the piece whose segment is consumed (kFuT: fetch a piece)
        uint32_t my_p0 = 0, my_len = 0;
        double my_av = 0.0;
        uint32_t done_products = 0;
        while (true) {
          // ------------------------------------------------ build a round: segments in k order
          uint32_t S = 0, T = 0;
          while (true) {
            if (jdone == kFuT) {
              if (kp >= nk) break;
              const int j = kp + tid;
              my_len = 0;
              if (j < nk) {
                const int32_t sl = __ldg(aslot + a0 + j);
                uint32_t p0 = 0, p1 = 0;
                if (sl >= 0) {
                  const uint32_t* ix = bidx + (size_t)sl * nwin1 + cidx;
                  p0 = __ldg(ix);
                  p1 = __ldg(ix + 1);
                } else if (sl < -1) {
                  const uint32_t len = (uint32_t)(-(sl + 1));
                  uint32_t rel = st_rel[j], nxt = st_next[j];
                  if (rel < len && (uint64_t)nxt < c_hi) {
                    const uint32_t b0 = __ldg(abase + a0 + j), b1 = b0 + len;
                    uint32_t pos = b0 + rel;
                    while (pos < b1 && nxt < c_lo) {
                      ++pos;
                      nxt = pos < b1 ? __ldg(B.col + pos) : 0u;
                    }
                    p0 = pos;
                    while (pos < b1 && (uint64_t)nxt < c_hi) {
                      ++pos;
                      nxt = pos < b1 ? __ldg(B.col + pos) : 0u;
                    }
                    p1 = pos;
                    st_rel[j] = (uint8_t)(pos - b0);
                    st_next[j] = nxt;
                  }
                }
                my_p0 = p0;
                my_len = p1 - p0;
                if (my_len) my_av = __ldg(A.val + a0 + j);
              }
              jdone = 0;
            }
            const bool pend = tid >= jdone;
            const uint32_t len = pend ? my_len : 0u;
            const uint32_t incl = fu_block_incl_scan((len > 0 ? (1u << 22) : 0u) | len, misc);
            const uint32_t sg = incl >> 22, pr = incl & 0x3fffffu;
            const bool fit = pend && S + sg <= (uint32_t)kFuS && T + pr <= (uint32_t)kFuR;
            if (fit && len > 0) {
              const uint32_t ix = S + sg - 1;
              s_off[ix] = T + pr - len;
              s_pos[ix] = my_p0;
              s_av[ix] = my_av;
            }
            const int nfit = __syncthreads_count(fit);
            if (nfit > 0 && tid == jdone + nfit - 1) {
              misc[56] = S + sg;
              misc[57] = T + pr;
            }
            if (nfit == 0 && S == 0 && tid == jdone) {
              // a segment longer than a round: its first kFuR products now, the rest stays pending
              s_off[0] = 0;
              s_pos[0] = my_p0;
              s_av[0] = my_av;
              my_p0 += kFuR;
              my_len -= kFuR;
              misc[56] = 1;
              misc[57] = kFuR;
            }
            __syncthreads();
            if (nfit > 0 || S == 0) {
              S = misc[56];
              T = misc[57];
            }
            jdone += nfit;
            if (jdone == kFuT) {
              kp += kFuT;
              continue;
            }
            break;   // the round is full
          }
          if (T == 0) break;   // no products left
          if (tid == 0) s_off[S] = T;
          __syncthreads();
          done_products += T;

          // ------------------------------------------------ gather: warp ranges of the stream
          const uint32_t L = ((T + kFuNW - 1) / kFuNW + 31) & ~31u;
          const uint32_t q_beg = min(T, (uint32_t)wid * L), q_end = min(T, q_beg + L);
          uint32_t lc[kFuU];
          double pv[kFuU];
          bool multi[kFuU];
          uint32_t* wc = cnt + wid * kFuNB;
          const uint32_t a_wc = (uint32_t)__cvta_generic_to_shared(wc);
#pragma unroll
          for (int u = 0; u < kFuU; ++u) {
            lc[u] = 0xffffffffu;
            pv[u] = 0.0;
            multi[u] = false;
          }
          if (q_beg < q_end) {
            E2Cursor<const uint32_t*> cur{s_off, s_pos, (int)S, 0, 0, 0};
            cur.init(q_beg);
#pragma unroll
            for (int hb = 0; hb < kFuU / 4; ++hb) {
              const uint32_t q00 = q_beg + 128u * hb;
              if (q00 < q_end) {
                uint32_t pos[4];
                int seg[4];
                bool mu[4];
                cur.batch(q00, q_end, pos, seg, mu);
                uint32_t cw[4];
                double vw[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const uint32_t q = q00 + 32 * u + lane;
                  cw[u] = 0xffffffffu;
                  vw[u] = 0.0;
                  if (q < q_end) {
                    cw[u] = __ldg(B.col + pos[u]);
                    vw[u] = __ldg(B.val + pos[u]);
                  }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const uint32_t q = q00 + 32 * u + lane;
                  if (q < q_end) {
                    lc[hb * 4 + u] = cw[u] - c_lo;
                    pv[hb * 4 + u] = __dmul_rn(s_av[seg[u]], vw[u]);
                  }
                  multi[hb * 4 + u] = mu[u];
                }
              }
            }
            // ---- pass 1: this warp's products per sub-bin (runs of equal bins inside a wave)
#pragma unroll
            for (int u = 0; u < kFuU; ++u) {
              if (q_beg + 32 * u >= q_end) break;
              const bool valid = lc[u] != 0xffffffffu;
              const uint32_t b = valid ? lc[u] >> bsh : 0xffffffffu;
              const uint32_t pb = __shfl_up_sync(0xffffffffu, b, 1);
              const bool head = lane == 0 || b != pb;
              const uint32_t hm = __ballot_sync(0xffffffffu, head);
              const uint32_t after = hm & ~le;
              const uint32_t nxt = after ? (uint32_t)(__ffs(after) - 1) : 32u;
              sh_red_add_pred(valid && head, a_wc + (b << 2), nxt - (uint32_t)lane);
            }
          }
          __syncthreads();
          // ---- slice starts: exclusive over (bin, warp)
          if (tid < 32) {
            uint32_t tot = 0;
            if (tid < nbins)
              for (int w = 0; w < kFuNW; ++w) tot += cnt[w * kFuNB + tid];
            const uint32_t inc = warp_incl_scan(tot);
            uint32_t run = inc - tot;
            if (tid < nbins) {
              misc[32 + tid] = run;
              for (int w = 0; w < kFuNW; ++w) {
                const uint32_t v = cnt[w * kFuNB + tid];
                cnt[w * kFuNB + tid] = run;
                run += v;
              }
            }
            if (tid == nbins - 1) misc[32 + nbins] = inc;
          }
          __syncthreads();
          // ---- pass 2: stable scatter into the sub-bin slices
          if (q_beg < q_end) {
#pragma unroll
            for (int u = 0; u < kFuU; ++u) {
              if (q_beg + 32 * u >= q_end) break;
              const bool valid = lc[u] != 0xffffffffu;
              const uint32_t b = valid ? lc[u] >> bsh : 0x40000000u + lane;
              uint32_t rank, lastm;
              if (!multi[u]) {
                const uint32_t pb = __shfl_up_sync(0xffffffffu, b, 1), nb = __shfl_down_sync(0xffffffffu, b, 1);
                const uint32_t hm = __ballot_sync(0xffffffffu, lane == 0 || b != pb);
                rank = (uint32_t)lane - (31u - __clz(hm & le));
                lastm = __ballot_sync(0xffffffffu, lane == 31 || b != nb);
              } else {
                const uint32_t peers = __match_any_sync(0xffffffffu, b);
                rank = __popc(peers & lt);
                lastm = __ballot_sync(0xffffffffu, (peers >> lane) == 1u);
              }
              uint32_t slot = 0;
              if (valid) slot = wc[b] + rank;
              __syncwarp();
              if (valid && ((lastm >> lane) & 1u)) wc[b] = slot + 1;
              if (valid) {
                cols[slot] = (uint16_t)lc[u];
                vals[slot] = pv[u];
              }
              __syncwarp();
            }
          }
          __syncthreads();
          for (int q = tid; q < kFuNW * kFuNB; q += kFuT) cnt[q] = 0u;
          // ------------------------------------------------ apply: one warp per sub-bin slice, stream order
          for (int b = wid; b < nbins; b += kFuNW) {
            const uint32_t s0 = misc[32 + b], e0 = misc[32 + b + 1];
            for (uint32_t q0 = s0; q0 < e0; q0 += 32) {
              const uint32_t q = q0 + lane;
              const bool valid = q < e0;
              const uint32_t c = valid ? (uint32_t)cols[q] : 0x10000u + lane;
              const double v = valid ? vals[q] : 0.0;
              const uint32_t pc = __shfl_up_sync(0xffffffffu, c, 1);
              const uint32_t brk = __ballot_sync(0xffffffffu, valid && lane > 0 && c <= pc);
              if (!brk) {
                if (valid) acc[c] = __dadd_rn(acc[c], v);
              } else {
                const uint32_t peers = __match_any_sync(0xffffffffu, c);
                const int rk = __popc(peers & lt);
                const int mult = __reduce_max_sync(0xffffffffu, valid ? __popc(peers) : 0);
                for (int r = 0; r < mult; ++r) {
                  if (valid && rk == r) acc[c] = __dadd_rn(acc[c], v);
                  __syncwarp();
                }
              }
              if (marking && valid) atomicOr(&bm[c >> 5], 1u << (c & 31));
              __syncwarp();
            }
          }
          __syncthreads();
          if (jdone == kFuT && kp >= nk) break;
        }
        // ------------------------------------------------ emit: columns in order, sums from the accumulator
        {
          const uint32_t pc = tid < nwords ? (uint32_t)__popc(bm[tid]) : 0u;
          uint32_t incl = 0;
          if (nwords <= 32) {
            incl = warp_incl_scan(pc);   // warp 0 holds every word
            __syncthreads();
          } else {
            incl = fu_block_incl_scan(pc, misc);
          }
          if (tid < nwords) wpref[tid] = incl - pc;
          if (tid == nwords - 1) misc[58] = incl;
          __syncthreads();
          const uint32_t m = misc[58];
          const bool ok = m == it_m && done_products == it_n;
          if (!ok && tid == 0) atomicOr(err, 4ull);
          // thread t: columns [t * cpt, (t + 1) * cpt), cpt a power of two <= 32
          const uint32_t cpt = width >= (uint32_t)kFuT ? width / kFuT : 1u;
          for (uint32_t cb = (uint32_t)tid * cpt; cb < width; cb += (uint32_t)kFuT * cpt) {
            const uint32_t wd = cb >> 5, sh = cb & 31;
            const uint32_t word = bm[wd];
            uint32_t bits = (word >> sh) & (cpt >= 32 ? 0xffffffffu : ((1u << cpt) - 1u));
            uint32_t r = wpref[wd] + __popc(word & ((1u << sh) - 1u));
            while (bits) {
              const uint32_t c = cb + (uint32_t)__ffs(bits) - 1u;
              bits &= bits - 1;
              if (ok) {
                __stcs(c_col + out + r, c_lo + c);
                __stcs(c_val + out + r, acc[c]);
              }
              acc[c] = 0.0;
              ++r;
            }
          }
        }
        __syncthreads();
      }
    }
  }
}

}  // namespace mg
