// Big chunks of heavy rows straight from B: no reorder buffer.
//
// The fine level's big chunks (more than kBinE products; always the dense association,
// accumulators.py:68-97, since kBinE >= crossover) carry ~75% of cfg3's heavy products.
// Bucketing them through an HBM reorder buffer (k_bin_expand2 -> k_bin_big) costs 20 B of
// intermediate traffic per product.  Here one warp owns one big chunk (or a column part of
// it) and streams the chunk's products directly from the B rows in ascending k --
// Gustavson order (gustavson.py:44-59), the order the reference's stable fine-level
// scatter leaves inside every chunk (magnus.py:236-249) -- into a rank-indexed dense
// shared-memory accumulator.  Per A nonzero k the chunk's segment of B row k comes from
// the B window index (one load pair; rows >= dir_min_len) or, for short rows, from a
// lane-local scan.  Work items are ordered chunk-major, so the warps of the whole GPU
// work on the same column window of B at any time and B's segments are re-read from L2.
//
// The small chunks keep the binned path (expand -> small-chunk reducers), whose reorder
// buffer then only holds small-chunk products (`cs` tables, k_bd_plan).
#pragma once
#include "binned_rows.cuh"

namespace mg {

struct BdItem {      // a big chunk (or one column part of it) of heavy row h
  int64_t out;       // first C entry of the chunk
  int32_t h;         // heavy row (index into the heavy-row list)
  uint32_t colbase;  // first column of the chunk
  uint32_t n, m;     // products, distinct columns of the chunk
  uint32_t bslot;    // column-bitmap slot in the pool (0xffffffff: none)
  uint32_t kind;     // column part (kind & 0xffff) of (kind >> 16) parts
};

// Per heavy row (one warp): small-chunk element prefix cs (the big chunks' products do not go
// through the reorder buffer) and its total; big-chunk items counted (Phase 0) or written
// into their chunk's bucket (Phase 1; bucket cursors = exclusive prefix of the counts).
template <int Phase>
__global__ void k_bd_plan(const int32_t* __restrict__ rows, int64_t nH, const int64_t* __restrict__ mn,
                          const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff,
                          const uint32_t* __restrict__ ce, const uint32_t* __restrict__ cd,
                          const uint32_t* __restrict__ cbm_slot, const int64_t* __restrict__ c_rp,
                          uint32_t* __restrict__ cs, int64_t* __restrict__ hsmall,
                          unsigned long long* __restrict__ bucket, int64_t n_chunks, BdItem* __restrict__ items,
                          bool chunk_major, bool no_split = false) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = warp; h < nH; h += nwarps) {
    const int64_t i = rows[h];
    const RowBins rb = row_bins(mn[i], mx[i], shift);   // entries == chunks (shift <= kBinMaxShift)
    const uint32_t* e = ce + choff[h];
    const uint32_t* d = cd + choff[h];
    uint32_t carry = 0;
    for (int j0 = 0; j0 < rb.nb; j0 += 32) {
      const int j = j0 + lane;
      const bool valid = j < rb.nb;
      const uint32_t n = valid ? __ldg(e + j + 1) - __ldg(e + j) : 0u;
      const bool big = n > (uint32_t)kBinE;
      const uint32_t s = big ? 0u : n;
      if (Phase == 0) {
        const uint32_t inc = warp_incl_scan(s);
        if (valid) cs[choff[h] + j] = carry + inc - s;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (big) {
        const uint32_t parts = no_split ? 1u : min((uint32_t)kBigMaxParts, (n + kBigSplit - 1) / kBigSplit);
        const int64_t chunk = rb.c0 + j;   // global chunk id
        const uint32_t mm = __ldg(d + j + 1) - __ldg(d + j);
        // two chunk-major lists: <= kBigD distinct columns (1024-rank accumulators) and wider
        unsigned long long* bk = bucket + (mm > (uint32_t)kBigD ? n_chunks : 0) + (chunk_major ? chunk : 0);
        if (Phase == 0) {
          atomicAdd(bk, (unsigned long long)parts);
        } else {
          const unsigned long long p0 = atomicAdd(bk, (unsigned long long)parts);
          BdItem it;
          it.out = c_rp[i] + __ldg(d + j);
          it.h = (int32_t)h;
          it.colbase = (uint32_t)(chunk << shift);
          it.n = n;
          it.m = mm;
          it.bslot = cbm_slot != nullptr ? __ldg(cbm_slot + choff[h] + j) : 0xffffffffu;
          for (uint32_t pp = 0; pp < parts; ++pp) {
            it.kind = (parts << 16) | pp;
            items[p0 + pp] = it;
          }
        }
      }
    }
    if (Phase == 0 && lane == 0) {
      cs[choff[h] + rb.nb] = carry;
      hsmall[h] = carry;
    }
  }
}

// exclusive prefix of n <= 1024 * 64 counters in place (one CTA of 1024 threads); total -> *total
__global__ void k_bd_bucket_scan(unsigned long long* __restrict__ c, int64_t n, unsigned long long* __restrict__ total) {
  __shared__ unsigned long long part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024, lo = t * per, hi = min(n, lo + per);
  unsigned long long s = 0;
  for (int64_t q = lo; q < hi; ++q) s += c[q];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    unsigned long long run = 0;
    for (int q = 0; q < 1024; ++q) {
      const unsigned long long v = part[q];
      part[q] = run;
      run += v;
    }
    *total = run;
  }
  __syncthreads();
  unsigned long long run = part[t];
  for (int64_t q = lo; q < hi; ++q) {
    const unsigned long long v = c[q];
    c[q] = run;
    run += v;
  }
}

// Segment of B row k inside the columns [c_lo, c_hi) -- a superset for one-entry rows, whose
// product is masked by its column when applied: the B window index (entries at the chunk
// boundaries) for indexed rows, a binary search for long rows outside the index budget.
__device__ __forceinline__ void bd_segment(const DevCsr& B, int32_t sl, uint32_t b0, int64_t k,
                                           const uint32_t* __restrict__ bidx, int64_t nwin1, uint32_t cidx,
                                           uint32_t c_lo, uint64_t c_hi, uint32_t& p0, uint32_t& p1) {
  if (sl >= 0) {
    const uint32_t* ix = bidx + (size_t)sl * nwin1 + cidx;
    p0 = __ldg(ix);
    p1 = __ldg(ix + 1);
  } else if (sl == -1) {
    p0 = b0;
    p1 = b0 + 1;
  } else if (sl == -3) {
    p0 = p1 = 0;
  } else {
    const uint32_t b1 = (uint32_t)B.rp(k + 1);
    p0 = lower_bound_col(B.col, b0, b1, c_lo);
    p1 = c_hi >= (uint64_t(1) << 32) ? b1 : lower_bound_col(B.col, p0, b1, (uint32_t)c_hi);
  }
}

#ifndef MG_BD_U
#define MG_BD_U 2
#endif
constexpr int kBdU = MG_BD_U;   // waves of products per group (loads of the next group in flight)
#ifndef MG_BD_W
#define MG_BD_W 4
#endif
constexpr int kBdW = MG_BD_W;   // warps per CTA (independent items)
#ifndef MG_BD_MINB
#define MG_BD_MINB 4
#endif
#ifndef MG_BD_G
#define MG_BD_G 4
#endif
constexpr int kBdG = MG_BD_G;          // lookups per lane and piece
constexpr int kBdPiece = 32 * kBdG;    // k's per piece (segments looked up together)

// Per A nonzero p (B row k = A.col[p]): the B window-index slot of row k, or -1 when row k
// holds one entry, -2 when it is longer but not indexed, -3 when it is empty; and row k's
// start in B.  A segment lookup then needs no load that depends on another one except the
// index entries themselves.
__global__ void k_bd_aprep(DevCsr A, DevCsr B, const int32_t* __restrict__ bslot, int32_t* __restrict__ aslot,
                           uint32_t* __restrict__ abase) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < A.nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = __ldg(A.col + p);
    const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
    const int32_t sl = __ldg(bslot + k);
    aslot[p] = sl >= 0 ? sl : (b1 - b0 == 1 ? -1 : (b1 == b0 ? -3 : -2));
    abase[p] = (uint32_t)b0;
  }
}

// per warp: rank-indexed accumulator, rank -> column, and per bitmap word (bits, rank prefix)
#ifdef MG_BD_STATS
// telemetry build: [list][items, k lookups, pieces, sub-batches, waves, single waves, products, runs, passes]
__device__ unsigned long long g_bd_stats[2][16];
#define BD_STAT(q, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_bd_stats[D > kBigD ? 1 : 0][q], (unsigned long long)(v)); } while (0)
#else
#define BD_STAT(q, v) do { } while (0)
#endif

__host__ __device__ inline size_t bd_warp_smem(int shift, int D) {
  const size_t words = ((size_t(1) << shift) + 31) / 32;
  return (size_t)D * 8 + (((size_t)D * 2 + 15) & ~size_t(15)) + words * 8 + (size_t)kBdPiece * 16;
}

__device__ __forceinline__ uint32_t rank_w(const uint2* wp, uint32_t c) {
  const uint2 w = wp[c >> 5];   // (bits, rank of the word's first column)
  return w.y + __popc(w.x & ((1u << (c & 31)) - 1u));
}

// One warp per item, persistent (tickets over the chunk-major item list).
template <int D>
__global__ void __launch_bounds__(32 * kBdW, MG_BD_MINB)
k_bd_num(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, Sem sem, const BdItem* __restrict__ items,
         uint64_t nit, unsigned long long* __restrict__ ticket,
         const uint32_t* __restrict__ cbm_pool, const int32_t* __restrict__ aslot,
         const uint32_t* __restrict__ abase, const uint32_t* __restrict__ bidx,
         int64_t nwin1, int ilog, uint32_t* __restrict__ c_col, double* __restrict__ c_val,
         unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int shift = sem.shift_num;
  const uint32_t width = 1u << shift;
  const int nwords = (int)((width + 31) / 32);
  unsigned char* sp = smem + (size_t)(threadIdx.x >> 5) * bd_warp_smem(shift, D);
  double* acc = reinterpret_cast<double*>(sp); sp += (size_t)D * 8;
  uint16_t* inv = reinterpret_cast<uint16_t*>(sp); sp += ((size_t)D * 2 + 15) & ~size_t(15);
  uint2* wp = reinterpret_cast<uint2*>(sp); sp += (size_t)nwords * 8;
  double* l_av = reinterpret_cast<double*>(sp); sp += (size_t)kBdPiece * 8;   // a piece's non-empty segments
  uint32_t* l_p0 = reinterpret_cast<uint32_t*>(sp); sp += (size_t)kBdPiece * 4;
  uint32_t* l_incl = reinterpret_cast<uint32_t*>(sp);
  const uint32_t lt = lanemask_lt();
  const int lane = threadIdx.x & 31;
  const uint32_t le = lanemask_le();
  unsigned long long t_next = 0;
  if (lane == 0) t_next = atomicAdd(ticket, 1ull);
  while (true) {
    const uint64_t t = __shfl_sync(0xffffffffu, t_next, 0);
    if (t >= nit) break;
    const BdItem it = items[t];
    if (lane == 0) t_next = atomicAdd(ticket, 1ull);
    const int64_t i = rows[it.h];
    const int64_t a0 = A.rp(i);
    const int nk = (int)(A.rp(i + 1) - a0);
    const uint32_t c_lo = it.colbase;
    const uint64_t c_hi = (uint64_t)c_lo + width;
    const uint32_t cidx = c_lo >> ilog;
    const uint32_t parts = it.kind >> 16, part = it.kind & 0xffffu;
    const uint32_t plo = (uint32_t)(((uint64_t)width * part) / parts), phi = (uint32_t)(((uint64_t)width * (part + 1)) / parts);

    // Walk the chunk's products in ascending k; apply(valid, column - c_lo, product, single)
    // per wave (single: the wave lies inside one B row segment -- distinct columns).  Per 32
    // k's: one segment lookup each (the next 32 looked up while these are streamed), then
    // waves over the concatenated segments in groups of kBdU, the next group's loads issued
    // before the current group is applied.
    auto stream = [&](auto&& apply) {
      // Segment lookups in a three-stage pipeline over pieces of kBdPiece k's (kBdG per lane):
      // stage A loads the A nonzeros' data two pieces ahead, stage B issues the index loads one
      // piece ahead, the current piece's segments are compacted into the shared list.
      int32_t a_sl[kBdG];
      uint32_t a_b0[kBdG];
      double a_av[kBdG];
      uint32_t b_p0[kBdG], b_p1[kBdG];
      double b_av[kBdG];
      auto stageA = [&](int kp) {
#pragma unroll
        for (int g = 0; g < kBdG; ++g) {
          const int j = kp + 32 * g + lane;
          a_sl[g] = -3;
          a_b0[g] = 0;
          a_av[g] = 0.0;
          if (j < nk) {
            a_sl[g] = __ldg(aslot + a0 + j);
            a_b0[g] = __ldg(abase + a0 + j);
            a_av[g] = __ldg(A.val + a0 + j);
          }
        }
      };
      auto stageB = [&](int kp) {
#pragma unroll
        for (int g = 0; g < kBdG; ++g) {
          const int j = kp + 32 * g + lane;
          const int64_t k = (a_sl[g] == -2 && j < nk) ? (int64_t)__ldg(A.col + a0 + j) : 0;
          bd_segment(B, a_sl[g], a_b0[g], k, bidx, nwin1, cidx, c_lo, c_hi, b_p0[g], b_p1[g]);
          b_av[g] = a_av[g];
        }
      };
      stageA(0);
      stageB(0);
      if (kBdPiece < nk) stageA(kBdPiece);
      for (int kp = 0; kp < nk; kp += kBdPiece) {
        // the piece's non-empty segments, in k order, to the list (inclusive product prefix)
        uint32_t cnt = 0, run = 0;
#pragma unroll
        for (int g = 0; g < kBdG; ++g) {
          const uint32_t len = b_p1[g] - b_p0[g];
          const bool ne = len > 0;
          const uint32_t mk = __ballot_sync(0xffffffffu, ne);
          const uint32_t inc = warp_incl_scan(len);
          if (ne) {
            const uint32_t ix = cnt + __popc(mk & lt);
            l_p0[ix] = b_p0[g];
            l_av[ix] = b_av[g];
            l_incl[ix] = run + inc;
          }
          cnt += __popc(mk);
          run += __shfl_sync(0xffffffffu, inc, 31);
        }
        __syncwarp();
        if (kp + kBdPiece < nk) stageB(kp + kBdPiece);
        if (kp + 2 * kBdPiece < nk) stageA(kp + 2 * kBdPiece);
        BD_STAT(2, 1);
        BD_STAT(1, min(nk - kp, kBdPiece));
        for (uint32_t sb = 0; sb < cnt; sb += 32) {
          BD_STAT(3, 1);
          const uint32_t base = sb ? l_incl[sb - 1] : 0u;
          const bool hv = sb + lane < cnt;
          const uint32_t p0 = hv ? l_p0[sb + lane] : 0u;
          const double av = hv ? l_av[sb + lane] : 0.0;
          const uint32_t incl = (hv ? l_incl[sb + lane] : l_incl[cnt - 1]) - base;
          const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
          const uint32_t up = __shfl_up_sync(0xffffffffu, incl, 1);
          const uint32_t exc = lane > 0 ? up : 0u;   // segment start in the sub-batch's product space
          uint32_t gc[kBdU];
          double gv[kBdU];
          int gs[kBdU];
          bool g1[kBdU];
          // loads of the group of waves starting at q00
          auto fetch = [&](uint32_t q00) {
#pragma unroll
            for (int u = 0; u < kBdU; ++u) {
              const uint32_t q0 = q00 + 32 * u, q = q0 + lane;
              gc[u] = 0xffffffffu;
              gv[u] = 0.0;
              gs[u] = 0;
              g1[u] = true;
              if (q0 < tot) {
                // segment of the wave's first position; the wave is single-segment when it ends
                // inside that segment (the common case: long segments)
                const int s0 = __popc(__ballot_sync(0xffffffffu, incl <= q0));
                const uint32_t end0 = __shfl_sync(0xffffffffu, incl, min(s0, 31));
                int sgi = s0;
                if (q0 + 31 >= end0) {
                  g1[u] = false;
                  sgi = 0;
#pragma unroll
                  for (int st = 16; st >= 1; st >>= 1)
                    if (__shfl_sync(0xffffffffu, incl, sgi + st - 1) <= q) sgi += st;
                  sgi = min(sgi, 31);
                }
                const uint32_t pos = __shfl_sync(0xffffffffu, p0, sgi) + (q - __shfl_sync(0xffffffffu, exc, sgi));
                gs[u] = sgi;
                if (q < tot) {   // (raw loads: consumed only when the group is applied)
                  gc[u] = __ldg(B.col + pos);
                  gv[u] = __ldg(B.val + pos);
                }
              }
            }
          };
          fetch(0);
          for (uint32_t q00 = 0; q00 < tot; q00 += 32 * kBdU) {
            uint32_t cc[kBdU];
            double vv[kBdU];
            int sg[kBdU];
            bool one[kBdU];
#pragma unroll
            for (int u = 0; u < kBdU; ++u) {
              cc[u] = gc[u];
              vv[u] = gv[u];
              sg[u] = gs[u];
              one[u] = g1[u];
            }
            if (q00 + 32 * kBdU < tot) fetch(q00 + 32 * kBdU);
#pragma unroll
            for (int u = 0; u < kBdU; ++u) {
              if (q00 + 32 * u >= tot) break;
              const double a = __shfl_sync(0xffffffffu, av, sg[u]);
              const uint32_t c = cc[u] - c_lo;   // outside the chunk: a one-entry row's masked product
              BD_STAT(4, 1);
              BD_STAT(5, one[u] ? 1 : 0);
              apply(q00 + 32 * u + lane < tot && c < width, c, __dmul_rn(a, vv[u]), one[u]);
            }
          }
        }
        __syncwarp();
      }
    };

    // ---- columns of the chunk -> ranks (bitmap kept by the symbolic pass, else marked here)
    uint32_t* bmw = reinterpret_cast<uint32_t*>(acc);   // marking scratch (before the sums)
    if (it.bslot != 0xffffffffu) {
      for (int wd = lane; wd < nwords; wd += 32) bmw[wd] = __ldg(cbm_pool + (size_t)it.bslot * nwords + wd);
      __syncwarp();
    } else {
      for (int wd = lane; wd < nwords; wd += 32) bmw[wd] = 0u;
      __syncwarp();
      stream([&](bool valid, uint32_t c, double, bool) {
        if (valid) atomicOr(&bmw[c >> 5], 1u << (c & 31));
      });
      __syncwarp();
    }
    {
      uint32_t carry = 0;
      for (int w0 = 0; w0 < nwords; w0 += 32) {
        const int wd = w0 + lane;
        const uint32_t bits = wd < nwords ? bmw[wd] : 0u;
        const uint32_t pc = (uint32_t)__popc(bits);
        const uint32_t inc = warp_incl_scan(pc);
        if (wd < nwords) wp[wd] = make_uint2(bits, carry + inc - pc);
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      __syncwarp();
      if (carry != it.m) {
        if (lane == 0) atomicOr(err, 4ull);
        continue;
      }
    }
    const uint32_t m = it.m;
    BD_STAT(0, 1);
    BD_STAT(6, it.n);
    const uint32_t rlo0 = plo < width ? rank_w(wp, plo) : m;
    const uint32_t rhi0 = phi < width ? rank_w(wp, phi) : m;
    for (uint32_t rlo = rlo0; rlo < rhi0; rlo += D) {
      const uint32_t rhi = min(rhi0, rlo + D);
      BD_STAT(8, 1);
      for (uint32_t r = lane; r < rhi - rlo; r += 32) acc[r] = 0.0;
      __syncwarp();
      stream([&](bool valid, uint32_t c, double v, bool single) {
        const uint32_t r = valid ? rank_w(wp, c) : 0u;
        const bool in = valid && r >= rlo && r < rhi;
        const uint32_t key = in ? r - rlo : 0u;
        if (in) inv[key] = (uint16_t)c;   // every contributor of a column writes the same value
        if (single) {
          // one B row segment: distinct columns, no ordering inside the wave
          if (in) acc[key] = __dadd_rn(acc[key], v);
        } else {
          // lanes are in stream order; a repeated rank can only come from a later segment:
          // apply the wave run by run (runs of strictly ascending ranks)
          const uint32_t kk = in ? key : 0x10000u + (uint32_t)lane;
          const uint32_t pk = __shfl_up_sync(0xffffffffu, kk, 1);
          const uint32_t brk = __ballot_sync(0xffffffffu, in && lane > 0 && kk <= pk);
          if (!brk) {
            if (in) acc[key] = __dadd_rn(acc[key], v);
          } else {
            const int run = __popc(brk & le);
            const int nruns = __popc(brk) + 1;
            BD_STAT(7, nruns);
            for (int rr = 0; rr < nruns; ++rr) {
              if (in && run == rr) acc[key] = __dadd_rn(acc[key], v);
              __syncwarp();
            }
          }
        }
        __syncwarp();
      });
      __syncwarp();
      for (uint32_t r = rlo + lane; r < rhi; r += 32) {
        __stcs(c_col + it.out + r, c_lo + (uint32_t)inv[r - rlo]);
        __stcs(c_val + it.out + r, acc[r - rlo]);
      }
      __syncwarp();
    }
  }
}

}  // namespace mg
