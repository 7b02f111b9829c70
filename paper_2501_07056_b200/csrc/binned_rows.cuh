// Rows with a large intermediate product (> 4096 elements): the MAGNUS fine
// level (reference magnus.py:195-262, Alg. 3) as a pipeline through an HBM/L2
// reorder buffer -- the reference's own chunked reorder -- in which every unit
// of work is independent, so all SMs stay busy.
//
// Chunks are the numeric plan's fine chunks (column c in chunk c >> shift_num,
// which decides the association of every output value).  Each chunk is cut
// into sub-bins of at most 512 columns (c >> gs).
//
//   symbolic (heavy_rows.cuh)  per heavy row and sub-bin: element count and
//                              distinct-column count, stored as exclusive
//                              prefixes ce / cd (offsets in the reorder buffer
//                              and in the C row).
//   k_bin_plan                 cuts each row into reduce windows -- runs of
//                              whole "small" chunks (<= kBinE elements, < 2
//                              kBinWinT per window) or one sub-bin of a "big"
//                              chunk -- and into expand units (chunk ranges).
//   k_bin_expand (warp/unit)   walks the row's B rows in ascending k (Gustavson
//                              order, gustavson.py:44-59) and appends each
//                              product to its slice: the whole chunk for a small
//                              chunk, the sub-bin for a big one.  Every slice is
//                              in ascending k: the reference's stable fine-level
//                              scatter order (magnus.py:236-249).
//   k_bin_reduce (warp/window) small chunk: bitmap -> column ranks, stable
//                              counting sort of the slice into shared memory,
//                              then per column the association the reference
//                              gives the chunk (accumulators.py:132-134): dense
//                              = sequential from +0.0 when the chunk holds >=
//                              crossover elements, else sort = x0 +
//                              pairwise(rest).  Big chunk (always dense, since
//                              kBinE >= crossover is a precondition): each
//                              sub-bin is accumulated in stream order into a
//                              dense shared-memory window, as the reference's
//                              dense accumulator does (accumulators.py:68-97).
#pragma once
#include "common.cuh"

namespace mg {

constexpr int kBinT = 128;            // threads per CTA of the expand / reduce kernels (4 warps)
constexpr int kBinE = 512;            // small chunk: <= kBinE elements (sort path); packed windows < kBinE
constexpr int kBinWinT = kBinE / 2;   // window packing quantum
constexpr int kBinMaxShift = 14;      // chunk width <= 16384 columns (u16 chunk-local columns)
constexpr int kSubShift = 14;         // table granularity (sub-bin == chunk while shift_num <= 14)
constexpr int kBinCur = 1024;         // expand: chunk cursors per warp (shared memory)
constexpr int64_t kBinUnitMax = 1 << 18;   // expand: elements per unit (rows above are split by chunk ranges)
constexpr int kBinU = 8;              // waves of loads in flight per lane

__host__ __device__ inline int bin_shift_of(int shift_num) { return shift_num < kSubShift ? shift_num : kSubShift; }

struct BinItem {   // table entries (sub-bins) [ja, jb) of heavy row h
  int32_t h, ja, jb, kind;   // window: 0 = whole small chunks, 1 = one sub-bin of a big chunk; unit: 1 = whole row
};

// shared memory of one reduce warp for chunk width 2^shift
__host__ __device__ inline size_t bin_reduce_warp_smem(int shift) {
  const size_t words = shift >= 5 ? (size_t(1) << (shift - 5)) : 1;
  const size_t w4 = (words * 4 + 15) & ~size_t(15), w2 = (words * 2 + 15) & ~size_t(15);
  return w4 + w2 + (size_t)kBinE * 2 /*u16 counts*/ + (size_t)kBinE * 8 /*values | dense window*/ +
         (size_t)kBinE * 2 /*columns*/;
}

// per heavy row: table entries (sub-bins in [mn >> gs, mx >> gs] plus one total) and its stream size
__global__ void k_bin_prep(const int32_t* __restrict__ rows, int64_t nrows, const int64_t* __restrict__ inter,
                           const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, int gshift,
                           int64_t* __restrict__ nent, int64_t* __restrict__ hinter) {
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nrows; h += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = rows[h];
    nent[h] = (mx[i] >> gshift) - (mn[i] >> gshift) + 2;
    hinter[h] = inter[i];
  }
}

__device__ __forceinline__ uint32_t lanemask_lt() { return (1u << (threadIdx.x & 31)) - 1u; }
__device__ __forceinline__ uint32_t lanemask_le() {
  const int l = threadIdx.x & 31;
  return l == 31 ? 0xffffffffu : ((2u << l) - 1u);
}

// warp-aggregated append of the items whose flag is set
__device__ __forceinline__ void emit_items(bool flag, BinItem it, BinItem* out, unsigned long long* count) {
  const uint32_t m = __ballot_sync(0xffffffffu, flag);
  if (!m) return;
  unsigned long long base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (flag) out[base + __popc(m & lanemask_lt())] = it;
}

// Geometry of one heavy row in table-entry space.
struct RowBins {
  int64_t b0;   // first sub-bin (mn >> gs)
  int64_t c0;   // first chunk (mn >> shift)
  int nb;       // sub-bins (table entries without the total)
  int nchunk;
  int cs;       // log2 sub-bins per chunk
  __device__ __forceinline__ int js(int cj) const { return (int)max((int64_t)0, ((c0 + cj) << cs) - b0); }
  __device__ __forceinline__ int je(int cj) const { return (int)min((int64_t)nb, ((c0 + cj + 1) << cs) - b0); }
};

__device__ __forceinline__ RowBins row_bins(int64_t mn, int64_t mx, int shift) {
  const int gs = bin_shift_of(shift);
  RowBins r;
  r.b0 = mn >> gs;
  r.c0 = mn >> shift;
  r.nb = (int)((mx >> gs) - r.b0 + 1);
  r.nchunk = (int)((mx >> shift) - r.c0 + 1);
  r.cs = shift - gs;
  return r;
}

// Windows and expand units of heavy rows [h0, h1), one warp per row.
__global__ void k_bin_plan(const int32_t* __restrict__ rows, int64_t h0, int64_t h1, const int64_t* __restrict__ mn,
                           const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff,
                           const uint32_t* __restrict__ ce, BinItem* __restrict__ wins, unsigned long long* __restrict__ nwin,
                           BinItem* __restrict__ bigs, unsigned long long* __restrict__ nbig, BinItem* __restrict__ units,
                           unsigned long long* __restrict__ nunit) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = h0 + warp; h < h1; h += nwarps) {
    const int64_t i = rows[h];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[h];
    const int ucj = kBinCur >> rb.cs;                       // chunks per unit (entries <= kBinCur)
    const bool split = (int64_t)__ldg(e + rb.nb) > kBinUnitMax || rb.nchunk > ucj;
    int wstart = 0, ustart = 0;
    for (int q0 = 0; q0 < rb.nchunk; q0 += 32) {
      const int cj = q0 + lane;
      const bool valid = cj < rb.nchunk;
      const int js = valid ? rb.js(cj) : 0, je = valid ? rb.je(cj) : 0;
      const uint32_t pe = valid ? __ldg(e + js) : 0u, pi = valid ? __ldg(e + je) : 0u;
      const uint32_t n = pi - pe;
      const bool big = valid && n > (uint32_t)kBinE;
      const bool next_big = valid && cj + 1 < rb.nchunk && (__ldg(e + rb.je(cj + 1)) - pi) > (uint32_t)kBinE;
      // ---- reduce windows: runs of small chunks; each sub-bin of a big chunk alone
      const bool cut = valid && (cj == rb.nchunk - 1 || big || next_big || pe / kBinWinT != pi / kBinWinT);
      const uint32_t cm = __ballot_sync(0xffffffffu, cut);
      {
        const uint32_t prev = cm & lanemask_lt();
        const int ws = prev ? q0 + 31 - __clz(prev) + 1 : wstart;
        const int wjs = rb.js(ws);
        emit_items(cut && !big && pi > __ldg(e + wjs), BinItem{(int32_t)h, wjs, je, 0}, wins, nwin);
        if (cm) wstart = q0 + 31 - __clz(cm) + 1;
      }
      emit_items(big, BinItem{(int32_t)h, js, je, 1}, bigs, nbig);
      // ---- expand units: chunk ranges (whole chunks, so small-chunk slices stay in one unit)
      const bool ucut = valid && (cj == rb.nchunk - 1 ||
                                  (split && (((cj + 1) % ucj) == 0 ||
                                             (int64_t)pe / kBinUnitMax != (int64_t)pi / kBinUnitMax)));
      const uint32_t um = __ballot_sync(0xffffffffu, ucut);
      {
        const uint32_t prev = um & lanemask_lt();
        const int us = prev ? q0 + 31 - __clz(prev) + 1 : ustart;
        const int ujs = rb.js(us);
        emit_items(ucut && pi > __ldg(e + ujs), BinItem{(int32_t)h, ujs, je, split ? 0 : 1}, units, nunit);
        if (um) ustart = q0 + 31 - __clz(um) + 1;
      }
    }
  }
}

// Expand: one warp per unit; products appended to their slice in ascending k.
__global__ void __launch_bounds__(kBinT)
k_bin_expand(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, const int64_t* __restrict__ mn,
             const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce,
             const int64_t* __restrict__ hbase, int64_t batch_base, const BinItem* __restrict__ units,
             const unsigned long long* __restrict__ nunit, unsigned long long* __restrict__ ticket,
             uint16_t* __restrict__ bcol, double* __restrict__ bval) {
  __shared__ uint32_t s_cur[kBinT / 32][kBinCur];
  __shared__ uint32_t s_big[kBinT / 32][kBinCur / 32];   // big-chunk flags of the unit's chunks
  const int lane = threadIdx.x & 31;
  uint32_t* cur = s_cur[threadIdx.x >> 5];
  uint32_t* bigm = s_big[threadIdx.x >> 5];
  const int gs = bin_shift_of(shift);
  const int64_t nu = (int64_t)*nunit;
  const uint32_t cmask = (1u << shift) - 1u;
  while (true) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(ticket, 1ull);
    u = __shfl_sync(0xffffffffu, u, 0);
    if ((int64_t)u >= nu) break;
    const BinItem it = units[u];
    const int64_t i = rows[it.h];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[it.h];
    const int nent = it.jb - it.ja;
    for (int j = lane; j < nent; j += 32) cur[j] = __ldg(e + it.ja + j);
    // chunks of the unit: [cfirst, clast]
    const int64_t cfirst = (rb.b0 + it.ja) >> rb.cs, clast = (rb.b0 + it.jb - 1) >> rb.cs;
    const int nck = (int)(clast - cfirst + 1);
    for (int w0 = 0; w0 < nck; w0 += 32) {
      const int r = w0 + lane;
      bool big = false;
      if (r < nck) {
        const int cj = (int)(cfirst + r - rb.c0);
        big = __ldg(e + rb.je(cj)) - __ldg(e + rb.js(cj)) > (uint32_t)kBinE;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, big);
      if (lane == 0) bigm[w0 >> 5] = m;
    }
    const int64_t rowbase = hbase[it.h] - batch_base;
    uint16_t* rc = bcol + rowbase;
    double* rv = bval + rowbase;
    const uint32_t clo = (uint32_t)((rb.b0 + it.ja) << gs);
    const int64_t chi64 = (rb.b0 + it.jb) << gs;
    const uint32_t chi = chi64 >= ((int64_t)1 << 32) ? 0xffffffffu : (uint32_t)chi64;
    __syncwarp();
    // groups of 32 k's: the group's segments are flattened into one stream of positions
    // (lane-consecutive), so loads of many short B rows are in flight together
    for (int64_t t0 = a0; t0 < a1; t0 += 32) {
      const int64_t t = t0 + lane;
      uint32_t p0 = 0, p1 = 0;
      double av = 0.0;
      if (t < a1) {
        const int64_t k = __ldg(A.col + t);
        av = __ldg(A.val + t);
        p0 = (uint32_t)B.rp(k);
        p1 = (uint32_t)B.rp(k + 1);
        if (!it.kind) {
          p0 = lower_bound_col(B.col, p0, p1, clo);
          p1 = lower_bound_col(B.col, p0, p1, chi);
        }
      }
      const uint32_t len = p1 - p0;
      const uint32_t inc = warp_incl_scan(len);
      const uint32_t off = inc - len;
      const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
      for (uint32_t q0 = 0; q0 < total; q0 += 32 * kBinU) {
        uint32_t c[kBinU], tk[kBinU];
        double v[kBinU];
#pragma unroll
        for (int w = 0; w < kBinU; ++w) {
          const uint32_t q = q0 + w * 32 + lane;
          // segment of stream position q: last lane with off <= q
          int lo = 0;
#pragma unroll
          for (int st = 16; st > 0; st >>= 1) {
            const uint32_t o = __shfl_sync(0xffffffffu, off, lo + st);
            if (o <= q) lo += st;
          }
          const uint32_t pp = __shfl_sync(0xffffffffu, p0, lo) + (q - __shfl_sync(0xffffffffu, off, lo));
          const double a = __shfl_sync(0xffffffffu, av, lo);
          tk[w] = (uint32_t)lo;
          c[w] = 0xffffffffu;
          v[w] = 0.0;
          if (q < total) {
            c[w] = __ldg(B.col + pp);
            v[w] = __dmul_rn(a, __ldg(B.val + pp));
          }
        }
#pragma unroll
        for (int w = 0; w < kBinU; ++w) {
          if (q0 + w * 32 < total) {
            const bool valid = c[w] != 0xffffffffu;
            uint32_t fl = 0x80000000u | lane;   // unique for invalid lanes
            if (valid) {
              const int64_t ck = c[w] >> shift;
              const int r = (int)(ck - cfirst);
              const bool big = (bigm[r >> 5] >> (r & 31)) & 1u;
              const int64_t ent = big ? (int64_t)(c[w] >> gs) - rb.b0 : max((int64_t)0, (ck << rb.cs) - rb.b0);
              fl = (uint32_t)(ent - it.ja);
            }
            uint32_t rank, last;
            const uint32_t t_first = __shfl_sync(0xffffffffu, tk[w], 0);
            if (__all_sync(0xffffffffu, !valid || tk[w] == t_first)) {
              // one B row: equal slices are contiguous runs
              const uint32_t prevf = __shfl_up_sync(0xffffffffu, fl, 1);
              const uint32_t nextf = __shfl_down_sync(0xffffffffu, fl, 1);
              const uint32_t hm = __ballot_sync(0xffffffffu, lane == 0 || prevf != fl);
              rank = (uint32_t)(lane - (31 - __clz(hm & lanemask_le())));
              last = lane == 31 || nextf != fl;
            } else {
              const uint32_t peers = __match_any_sync(0xffffffffu, fl);
              rank = __popc(peers & lanemask_lt());
              last = (peers >> lane) == 1u;
            }
            uint32_t slot = 0;
            if (valid) slot = cur[fl] + rank;
            __syncwarp();
            if (valid && last) cur[fl] = slot + 1;
            if (valid) {
              rc[slot] = (uint16_t)(c[w] & cmask);
              rv[slot] = v[w];
            }
            __syncwarp();
          }
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- reduce helpers (warp scope)
__device__ __forceinline__ uint32_t u16_get(const uint32_t* a, uint32_t r) { return (a[r >> 1] >> ((r & 1u) * 16)) & 0xffffu; }

__device__ __forceinline__ uint32_t rank_of(const uint32_t* bm, const uint16_t* pref, uint32_t c) {
  const uint32_t wd = c >> 5, bit = 1u << (c & 31);
  return pref[wd] + __popc(bm[wd] & (bit - 1u));
}

// Exclusive word prefix of popcounts over [wlo, whi); returns the total.
__device__ __forceinline__ uint32_t prefix_words(const uint32_t* bm, uint16_t* pref, int wlo, int whi) {
  const int lane = threadIdx.x & 31;
  uint32_t carry = 0;
  for (int w0 = wlo; w0 < whi; w0 += 32) {
    const int wd = w0 + lane;
    const uint32_t pc = wd < whi ? (uint32_t)__popc(bm[wd]) : 0u;
    const uint32_t inc = warp_incl_scan(pc);
    if (wd < whi) pref[wd] = (uint16_t)(carry + inc - pc);
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncwarp();
  return carry;
}

__device__ __forceinline__ double sum_seq_s(const double* sv, uint32_t s0, uint32_t e0) {
  double acc = 0.0;
  for (uint32_t a = s0; a < e0; ++a) acc = __dadd_rn(acc, sv[a]);
  return acc;
}

__device__ __noinline__ double sum_pairwise_s(const double* sv, uint32_t s0, uint32_t e0) {
  auto x = [&](int64_t q) { return sv[q]; };
  double s = sv[s0];
  if (e0 - s0 > 1) s = __dadd_rn(s, pairwise(x, s0 + 1, e0 - s0 - 1));
  return s;
}

struct ReduceSmem {
  uint32_t* bm;
  uint16_t* pref;
  uint32_t* cnt;
  double* sval;
  uint16_t* stc;
};

// Small chunk (n <= kBinE elements): stable counting sort of the slice by column rank
// into shared memory, then one lane per column sums its run with the chunk's association.
__device__ __forceinline__ bool reduce_chunk_sort(const uint16_t* __restrict__ sc, const double* __restrict__ sv_g,
                                                  uint32_t n, uint32_t m, bool seq, uint32_t colbase, const ReduceSmem& S,
                                                  uint32_t* __restrict__ c_col, double* __restrict__ c_val, int64_t out) {
  const int lane = threadIdx.x & 31;
  uint32_t cmin = 0xffffu, cmax = 0u;
  for (uint32_t q = lane; q < n; q += 32) {
    const uint32_t c = __ldg(sc + q);
    S.stc[q] = (uint16_t)c;
    cmin = min(cmin, c);
    cmax = max(cmax, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
    cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  }
  const int wlo = (int)(cmin >> 5), whi = (int)(cmax >> 5) + 1;
  for (int wd = wlo + lane; wd < whi; wd += 32) S.bm[wd] = 0u;
  for (uint32_t r = lane; r < (m + 1) / 2; r += 32) S.cnt[r] = 0u;
  __syncwarp();
  for (uint32_t q = lane; q < n; q += 32) {
    const uint32_t c = S.stc[q];
    atomicOr(&S.bm[c >> 5], 1u << (c & 31));
  }
  __syncwarp();
  if (prefix_words(S.bm, S.pref, wlo, whi) != m) return false;
  for (uint32_t q = lane; q < n; q += 32) {
    const uint32_t r = rank_of(S.bm, S.pref, S.stc[q]);
    S.stc[q] = (uint16_t)r;   // the slice's columns become ranks
    atomicAdd(&S.cnt[r >> 1], 1u << ((r & 1u) * 16));
  }
  __syncwarp();
  {
    uint32_t carry = 0;
    const uint32_t nwc = (m + 1) / 2;
    for (uint32_t w0 = 0; w0 < nwc; w0 += 32) {
      const uint32_t wd = w0 + lane;
      const uint32_t v = wd < nwc ? S.cnt[wd] : 0u;
      const uint32_t lo = v & 0xffffu, hi = v >> 16;
      const uint32_t inc = warp_incl_scan(lo + hi);
      const uint32_t ex = carry + inc - (lo + hi);
      if (wd < nwc) S.cnt[wd] = ex | ((ex + lo) << 16);
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncwarp();
  // scatter values in stream order (ascending k per column): inside one wave, lanes of the
  // same column are ordered by lane (= stream position)
  for (uint32_t q0 = 0; q0 < n; q0 += 32) {
    const uint32_t q = q0 + lane;
    const bool valid = q < n;
    const double v = valid ? __ldg(sv_g + q) : 0.0;
    const uint32_t r = valid ? (uint32_t)S.stc[q] : 0x10000u + lane;
    const uint32_t pr = __shfl_up_sync(0xffffffffu, r, 1);
    const bool brk = valid && lane > 0 && r <= pr;
    if (!__ballot_sync(0xffffffffu, brk)) {
      if (valid) {
        const uint32_t old = atomicAdd(&S.cnt[r >> 1], 1u << ((r & 1u) * 16));
        S.sval[(old >> ((r & 1u) * 16)) & 0xffffu] = v;
      }
    } else {
      const uint32_t peers = __match_any_sync(0xffffffffu, r);
      const uint32_t before = __popc(peers & lanemask_lt());
      uint32_t base = 0;
      if (valid && before == 0) {
        const uint32_t old = atomicAdd(&S.cnt[r >> 1], (uint32_t)__popc(peers) << ((r & 1u) * 16));
        base = (old >> ((r & 1u) * 16)) & 0xffffu;
      }
      base = __shfl_sync(0xffffffffu, base, __ffs(peers) - 1);
      if (valid) S.sval[base + before] = v;
    }
  }
  __syncwarp();
  for (uint32_t r = lane; r < m; r += 32) {
    const uint32_t s0 = r ? u16_get(S.cnt, r - 1) : 0u, e0 = u16_get(S.cnt, r);
    c_val[out + r] = seq ? sum_seq_s(S.sval, s0, e0) : sum_pairwise_s(S.sval, s0, e0);
  }
  for (int wd = wlo + lane; wd < whi; wd += 32) {
    uint32_t bits = S.bm[wd];
    uint32_t r = S.pref[wd];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1u;
      c_col[out + r] = colbase + (uint32_t)(wd * 32 + b);
      ++r;
    }
  }
  __syncwarp();
  return true;
}

// One sub-bin of a big chunk (dense association): stream-order accumulation into a dense
// shared-memory window of the sub-bin's columns.  Inside one wave, lanes of the same
// column are added by the lowest of them, in lane order.
__device__ __forceinline__ bool reduce_bin_dense(const uint16_t* __restrict__ sc, const double* __restrict__ sv_g,
                                                 uint32_t n, uint32_t m, int gs, uint32_t colbase, const ReduceSmem& S,
                                                 uint32_t* __restrict__ c_col, double* __restrict__ c_val, int64_t out) {
  const int lane = threadIdx.x & 31;
  const uint32_t bw = 1u << gs, bmask = bw - 1u;
  const int nwords = (int)((bw + 31) >> 5);
  double* acc = S.sval;
  for (int wd = lane; wd < nwords; wd += 32) S.bm[wd] = 0u;
  for (uint32_t c = lane; c < bw; c += 32) acc[c] = 0.0;
  __syncwarp();
  for (uint32_t q0 = 0; q0 < n; q0 += 32 * kBinU) {
    uint32_t cc[kBinU];
    double vv[kBinU];
#pragma unroll
    for (int w = 0; w < kBinU; ++w) {
      const uint32_t q = q0 + w * 32 + lane;
      cc[w] = 0x10000u + lane;
      vv[w] = 0.0;
      if (q < n) {
        cc[w] = __ldg(sc + q) & bmask;
        vv[w] = __ldg(sv_g + q);
      }
    }
#pragma unroll
    for (int w = 0; w < kBinU; ++w) {
      if (q0 + w * 32 < n) {
        const uint32_t c = cc[w];
        const bool valid = c < 0x10000u;
        const uint32_t pc = __shfl_up_sync(0xffffffffu, c, 1);
        const uint32_t brk = __ballot_sync(0xffffffffu, valid && lane > 0 && c <= pc);
        if (valid) atomicOr(&S.bm[c >> 5], 1u << (c & 31));
        if (!brk) {
          if (valid) acc[c] = __dadd_rn(acc[c], vv[w]);
        } else {
          const uint32_t peers = __match_any_sync(0xffffffffu, c);
          const uint32_t gsz = __popc(peers);
          const uint32_t maxg = __reduce_max_sync(0xffffffffu, valid ? gsz : 0u);
          const bool lead = valid && (peers & lanemask_lt()) == 0u;
          double s = lead ? acc[c] : 0.0;
          uint32_t rem = peers;
          for (uint32_t k = 0; k < maxg; ++k) {
            const int src = rem ? __ffs(rem) - 1 : lane;
            if (rem) rem &= rem - 1u;
            const double x = __shfl_sync(0xffffffffu, vv[w], src);
            if (lead && k < gsz) s = __dadd_rn(s, x);
          }
          if (lead) acc[c] = s;
        }
        __syncwarp();
      }
    }
  }
  if (prefix_words(S.bm, S.pref, 0, nwords) != m) return false;
  for (int wd = lane; wd < nwords; wd += 32) {
    uint32_t bits = S.bm[wd];
    uint32_t r = S.pref[wd];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1u;
      const uint32_t c = (uint32_t)(wd * 32 + b);
      c_col[out + r] = colbase + c;
      c_val[out + r] = acc[c];
      ++r;
    }
  }
  __syncwarp();
  return true;
}

// Reduce: one warp per window.
__global__ void __launch_bounds__(kBinT)
k_bin_reduce(const int32_t* __restrict__ rows, const int8_t* __restrict__ cat, const int64_t* __restrict__ mn,
             const int64_t* __restrict__ mx, Sem sem, const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce,
             const uint32_t* __restrict__ cd, const int64_t* __restrict__ hbase, int64_t batch_base,
             const BinItem* __restrict__ wins, const unsigned long long* __restrict__ nwin,
             unsigned long long* __restrict__ ticket, const uint16_t* __restrict__ bcol,
             const double* __restrict__ bval, const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
             double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int shift = sem.shift_num, gs = bin_shift_of(shift);
  const int words = shift >= 5 ? 1 << (shift - 5) : 1;
  const size_t w4 = ((size_t)words * 4 + 15) & ~size_t(15), w2 = ((size_t)words * 2 + 15) & ~size_t(15);
  unsigned char* base = smem + (size_t)(threadIdx.x >> 5) * bin_reduce_warp_smem(shift);
  ReduceSmem S;
  S.bm = reinterpret_cast<uint32_t*>(base);
  S.pref = reinterpret_cast<uint16_t*>(base + w4);
  S.cnt = reinterpret_cast<uint32_t*>(base + w4 + w2);
  S.sval = reinterpret_cast<double*>(base + w4 + w2 + (size_t)kBinE * 2);
  S.stc = reinterpret_cast<uint16_t*>(base + w4 + w2 + (size_t)kBinE * 10);
  const int64_t nw = (int64_t)*nwin;
  const uint32_t cwmask = ~((1u << shift) - 1u);
  while (true) {
    unsigned long long wi = 0;
    if ((threadIdx.x & 31) == 0) wi = atomicAdd(ticket, 1ull);
    wi = __shfl_sync(0xffffffffu, wi, 0);
    if ((int64_t)wi >= nw) break;
    const BinItem it = wins[wi];
    const int64_t i = rows[it.h];
    const int ci = cat[i];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[it.h];
    const uint32_t* d = cd + choff[it.h];
    const int64_t rowbase = hbase[it.h] - batch_base;
    const int64_t out_row = c_rp[i];
    bool ok = true;
    if (it.kind == 1) {
      const int j = it.ja;
      const uint32_t ej = __ldg(e + j), dj = __ldg(d + j);
      ok = reduce_bin_dense(bcol + rowbase + ej, bval + rowbase + ej, __ldg(e + j + 1) - ej, __ldg(d + j + 1) - dj, gs,
                            (uint32_t)((rb.b0 + j) << gs), S, c_col, c_val, out_row + dj);
    } else {
      int j = it.ja;
      while (j < it.jb) {
        const int je = (int)min((int64_t)it.jb, ((((rb.b0 + j) >> rb.cs) + 1) << rb.cs) - rb.b0);
        const uint32_t ej = __ldg(e + j), n = __ldg(e + je) - ej;
        if (n) {
          const uint32_t dj = __ldg(d + j);
          const bool seq = ci == kCatDense || (int64_t)n >= sem.crossover;
          ok &= reduce_chunk_sort(bcol + rowbase + ej, bval + rowbase + ej, n, __ldg(d + je) - dj, seq,
                                  (uint32_t)((rb.b0 + j) << gs) & cwmask, S, c_col, c_val, out_row + dj);
        }
        j = je;
      }
    }
    if (!ok && (threadIdx.x & 31) == 0) atomicOr(err, 4ull);
  }
}


// Big chunk (> kBinE elements, dense association): one CTA per chunk, a dense
// shared-memory window over the chunk's columns.  Columns are dealt to the 8 warps
// in 16-column granules; the slice is taken in batches of kBigS elements: each warp
// ranks its part of the batch by owner (ballots), a CTA scan turns the counts into
// offsets, the batch is stably partitioned by owner into shared memory, and each
// warp then applies its own elements in stream order -- a column is only ever
// updated by its owner, in ascending k.
constexpr int kBigT = 256;
constexpr int kBigS = 2048;                 // elements per batch
constexpr int kBigWaves = kBigS / kBigT;    // waves of 32 per warp per batch (8)

__host__ __device__ inline size_t bin_big_smem(int shift) {
  const size_t width = size_t(1) << shift, words = (width + 31) / 32;
  return width * 8 + ((words * 4 + 15) & ~size_t(15)) + (size_t)kBigS * 8 + (size_t)kBigS * 2 + 80 * 4;
}

__global__ void __launch_bounds__(kBigT)
k_bin_big(const int32_t* __restrict__ rows, const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, Sem sem,
          const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce, const uint32_t* __restrict__ cd,
          const int64_t* __restrict__ hbase, int64_t batch_base, const BinItem* __restrict__ bigs,
          const unsigned long long* __restrict__ nbig, unsigned long long* __restrict__ ticket,
          const uint16_t* __restrict__ bcol, const double* __restrict__ bval, const int64_t* __restrict__ c_rp,
          uint32_t* __restrict__ c_col, double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NW = kBigT / 32;
  static_assert(NW == 8, "8 owner warps");
  const int shift = sem.shift_num;
  const uint32_t width = 1u << shift;
  const int nwords = (int)((width + 31) / 32);
  double* acc = reinterpret_cast<double*>(smem);
  unsigned char* p = smem + (size_t)width * 8;
  uint32_t* bm = reinterpret_cast<uint32_t*>(p);
  p += ((size_t)nwords * 4 + 15) & ~size_t(15);
  double* stv = reinterpret_cast<double*>(p);
  p += (size_t)kBigS * 8;
  uint16_t* stc = reinterpret_cast<uint16_t*>(p);
  p += (size_t)kBigS * 2;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(p);   // [owner * NW + warp], then [64] = total
  __shared__ unsigned long long s_item;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nbg = (int64_t)*nbig;
  while (true) {
    if (threadIdx.x == 0) s_item = atomicAdd(ticket, 1ull);
    __syncthreads();
    const int64_t bi = (int64_t)s_item;
    if (bi >= nbg) break;
    const BinItem it = bigs[bi];
    const int64_t i = rows[it.h];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[it.h];
    const uint32_t* d = cd + choff[it.h];
    const uint32_t ej = __ldg(e + it.ja), n = __ldg(e + it.jb) - ej;
    const uint32_t dj = __ldg(d + it.ja), m = __ldg(d + it.jb) - dj;
    const int64_t rowbase = hbase[it.h] - batch_base;
    const uint16_t* sc = bcol + rowbase + ej;
    const double* sv = bval + rowbase + ej;
    const int64_t out = c_rp[i] + dj;
    const uint32_t colbase = (uint32_t)(((rb.b0 + it.ja) >> rb.cs) << shift);
    for (uint32_t c = threadIdx.x; c < width; c += kBigT) acc[c] = 0.0;
    for (int wd = threadIdx.x; wd < nwords; wd += kBigT) bm[wd] = 0u;
    __syncthreads();
    for (uint32_t B0 = 0; B0 < n; B0 += kBigS) {
      const uint32_t nb = min((uint32_t)kBigS, n - B0);
      uint32_t cc[kBigWaves], off[kBigWaves];
      double vv[kBigWaves];
#pragma unroll
      for (int v = 0; v < kBigWaves; ++v) {
        const uint32_t q = (uint32_t)wid * (kBigS / NW) + v * 32 + lane;
        cc[v] = 0xffffffffu;
        vv[v] = 0.0;
        if (q < nb) {
          cc[v] = __ldg(sc + B0 + q);
          vv[v] = __ldg(sv + B0 + q);
        }
      }
      uint32_t run_cnt = 0;   // lane l < 8: this warp's elements owned by warp l so far
#pragma unroll
      for (int v = 0; v < kBigWaves; ++v) {
        const bool valid = cc[v] != 0xffffffffu;
        const uint32_t ow = valid ? (cc[v] >> 4) & 7u : 0u;
        const uint32_t vm = __ballot_sync(0xffffffffu, valid);
        const uint32_t x0 = __ballot_sync(0xffffffffu, ow & 1u), x1 = __ballot_sync(0xffffffffu, ow & 2u),
                       x2 = __ballot_sync(0xffffffffu, ow & 4u);
        const uint32_t peers = vm & ((ow & 1u) ? x0 : ~x0) & ((ow & 2u) ? x1 : ~x1) & ((ow & 4u) ? x2 : ~x2);
        const uint32_t mine_l = vm & ((lane & 1) ? x0 : ~x0) & ((lane & 2) ? x1 : ~x1) & ((lane & 4) ? x2 : ~x2);
        off[v] = __shfl_sync(0xffffffffu, run_cnt, ow) + __popc(peers & lanemask_lt());
        if (lane < NW) run_cnt += __popc(mine_l);
      }
      if (lane < NW) cnt[lane * NW + wid] = run_cnt;
      __syncthreads();
      if (wid == 0) {
        const uint32_t a0 = cnt[2 * lane], a1 = cnt[2 * lane + 1];
        const uint32_t inc = warp_incl_scan(a0 + a1);
        const uint32_t ex = inc - a0 - a1;
        cnt[2 * lane] = ex;
        cnt[2 * lane + 1] = ex + a0;
        if (lane == 31) cnt[64] = inc;
      }
      __syncthreads();
#pragma unroll
      for (int v = 0; v < kBigWaves; ++v) {
        if (cc[v] != 0xffffffffu) {
          const uint32_t pos = cnt[((cc[v] >> 4) & 7u) * NW + wid] + off[v];
          stc[pos] = (uint16_t)cc[v];
          stv[pos] = vv[v];
        }
      }
      __syncthreads();
      const uint32_t lo = cnt[wid * NW], hi = wid == NW - 1 ? cnt[64] : cnt[(wid + 1) * NW];
      for (uint32_t p0 = lo; p0 < hi; p0 += 32) {
        const uint32_t q = p0 + lane;
        const bool valid = q < hi;
        const uint32_t c = valid ? (uint32_t)stc[q] : 0x10000u + lane;
        const double v = valid ? stv[q] : 0.0;
        const uint32_t pc = __shfl_up_sync(0xffffffffu, c, 1);
        const uint32_t brk = __ballot_sync(0xffffffffu, valid && lane > 0 && c <= pc);
        if (valid) atomicOr(&bm[c >> 5], 1u << (c & 31));
        if (!brk) {
          if (valid) acc[c] = __dadd_rn(acc[c], v);
        } else {
          // ascending runs one after another (a column repeats only across runs)
          const int run = __popc(brk & lanemask_le());
          const int nruns = __popc(brk) + 1;
          for (int rr = 0; rr < nruns; ++rr) {
            if (valid && run == rr) acc[c] = __dadd_rn(acc[c], v);
            __syncwarp();
          }
        }
        __syncwarp();
      }
      __syncthreads();
    }
    // compact: word prefix over the whole window (block scan), then write the touched columns
    const uint32_t wpt = (nwords + kBigT - 1) / kBigT;   // words per thread (contiguous)
    uint32_t cntw = 0;
    for (uint32_t q = 0; q < wpt; ++q) {
      const uint32_t wd = threadIdx.x * wpt + q;
      if (wd < (uint32_t)nwords) cntw += __popc(bm[wd]);
    }
    const uint32_t inc = warp_incl_scan(cntw);
    if (lane == 31) cnt[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const uint32_t wv = lane < NW ? cnt[lane] : 0u;
      const uint32_t wi = warp_incl_scan(wv);
      if (lane < NW) cnt[lane] = wi - wv;
      if (lane == NW - 1) cnt[64] = wi;
    }
    __syncthreads();
    uint32_t r = cnt[wid] + inc - cntw;
    if (threadIdx.x == 0 && cnt[64] != m) atomicOr(err, 4ull);
    for (uint32_t q = 0; q < wpt; ++q) {
      const uint32_t wd = threadIdx.x * wpt + q;
      if (wd >= (uint32_t)nwords) break;
      uint32_t bits = bm[wd];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        const uint32_t c = wd * 32 + b;
        if (r < m) {
          c_col[out + r] = colbase + c;
          c_val[out + r] = acc[c];
        }
        ++r;
      }
    }
    __syncthreads();
  }
}

}  // namespace mg
