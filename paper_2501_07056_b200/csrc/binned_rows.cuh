// Rows with a large intermediate product (> 4096 elements): the MAGNUS fine
// level (reference magnus.py:195-262, Alg. 3) as a pipeline through an HBM/L2
// reorder buffer -- the reference's own chunked reorder -- in which every unit
// of work is independent, so all SMs stay busy.
//
// Chunks are the numeric plan's fine chunks (column c in chunk c >> shift_num,
// which decides the association of every output value; chunk width <= 2^14).
//
//   symbolic (symbolic_rows.cuh)  per heavy row and chunk: product count and
//                              distinct-column count, stored as exclusive
//                              prefixes ce / cd (offsets in the reorder buffer
//                              and in the C row), and the column bitmaps of
//                              big chunks.
//   k_bin_plan                 cuts each row into reduce windows (runs of
//                              small chunks), big-chunk items and expand units
//                              (chunk ranges).
//   k_bin_expand2 (CTA/unit)   walks the unit's B rows in ascending k (Gustavson
//                              order, gustavson.py:44-59) and appends each
//                              product to its chunk's slice; every slice is in
//                              ascending k: the reference's stable fine-level
//                              scatter order (magnus.py:236-249).
//   k_bin_reduce / _tiny       small chunks (<= kBinE products): stable sort of
//   (warp/window)              the slice by column, then per column the
//                              association the reference gives the chunk
//                              (accumulators.py:132-134): dense = sequential
//                              from +0.0 when the chunk holds >= crossover
//                              elements, else sort = x0 + pairwise(rest).
//   k_bin_big (warp/chunk)     big chunks (always the dense association, since
//                              kBinE >= crossover is a precondition): the slice
//                              is accumulated in stream order into a dense
//                              shared-memory accumulator, as the reference's
//                              dense accumulator does (accumulators.py:68-97).
#pragma once
#include "common.cuh"

namespace mg {

constexpr int kBinT = 128;            // threads per CTA of the expand / reduce kernels (4 warps)
#ifndef MG_BIN_E
#define MG_BIN_E 512
#endif
constexpr int kBinE = MG_BIN_E;       // small chunk: <= kBinE elements (sort path); packed windows < kBinE
constexpr int kBinWinT = kBinE / 2;   // window packing quantum
constexpr int kBinMaxShift = 14;      // chunk width <= 16384 columns (u16 chunk-local columns)
constexpr int kSubShift = 14;         // table granularity (sub-bin == chunk while shift_num <= 14)
#ifndef MG_BIN_CUR
#define MG_BIN_CUR 128
#endif
constexpr int kBinCur = MG_BIN_CUR;   // expand: chunks per unit (cursors / counters in shared memory)
#ifndef MG_UNIT_MAX
#define MG_UNIT_MAX (1 << 17)
#endif
constexpr int64_t kBinUnitMax = MG_UNIT_MAX;   // expand: elements per unit (rows above are split by chunk ranges)
constexpr uint32_t kBigSplit = 1u << 17;   // big chunks above this many elements are split by columns
constexpr uint32_t kBigFront = 1u << 14;   // big chunks scheduled first
constexpr uint32_t kUnitFront = 1u << 15;  // expand units scheduled first
constexpr int kBigMaxParts = 32;
#ifndef MG_BIG_WIDE_PARTS
#define MG_BIG_WIDE_PARTS 1
#endif
#ifndef MG_BIG_WIDE_NARROW
#define MG_BIG_WIDE_NARROW 0
#endif
#ifndef MG_BIG_D
#define MG_BIG_D 1024
#endif
constexpr int kBigD = MG_BIG_D;            // ranks accumulated per pass


__host__ __device__ inline int bin_shift_of(int shift_num) { return shift_num < kSubShift ? shift_num : kSubShift; }

// A big chunk (or one column part of it), resolved by the plan kernel so that the reducer
// needs one load per item: its slice in the reorder buffer, its place in C, its bitmap slot.
struct BigItem {
  int64_t slice;     // first element in the reorder buffer (batch-relative)
  int64_t out;       // first C entry of the chunk
  uint32_t n, m;     // products, distinct columns
  uint32_t colbase;  // first column of the chunk
  uint32_t bslot;    // column-bitmap slot in the pool (0xffffffff: none)
  uint32_t kind;     // column part (kind & 0xffff) of (kind >> 16) parts
  uint32_t pad;
};

struct BinItem {   // table entries (sub-bins) [ja, jb) of heavy row h
  int32_t h, ja, jb, kind;   // unit: 1 = whole row; big chunk: column part (kind & 0xffff) of (kind >> 16) parts
};

// shared memory of one reduce warp for chunk width 2^shift
__host__ __device__ inline size_t bin_reduce_warp_smem(int shift) {
  const size_t words = shift >= 5 ? (size_t(1) << (shift - 5)) : 1;
  const size_t w4 = (words * 4 + 15) & ~size_t(15), w2 = (words * 2 + 15) & ~size_t(15);
  return w4 + w2 + (size_t)kBinE * 2 /*u16 counts*/ + (size_t)kBinE * 8 /*values*/ + (size_t)kBinE * 2 /*columns*/ +
         (size_t)kBinE * 2 /*rank -> column*/;
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

// warp-aggregated append of the items whose flag is set (rev: placed from the end of a
// list of `cap` slots downwards)
__device__ __forceinline__ void emit_items(bool flag, BinItem it, BinItem* out, unsigned long long* count,
                                           int64_t rev_cap = -1) {
  const uint32_t m = __ballot_sync(0xffffffffu, flag);
  if (!m) return;
  unsigned long long base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  const int64_t pos = (int64_t)base + __popc(m & lanemask_lt());
  if (flag) out[rev_cap < 0 ? pos : rev_cap - 1 - pos] = it;
}

// Lists with large items first: items [0, n_front) are the large ones, the others sit at
// [cap - n_back, cap) -- scheduling ticket t maps to the t-th item of that order.
__device__ __forceinline__ int64_t list_slot(uint64_t t, uint64_t n_front, int64_t cap) {
  return t < n_front ? (int64_t)t : cap - 1 - (int64_t)(t - n_front);
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

// Telemetry: products / distinct columns in big (> kBinE products) and other chunks.
__global__ void k_heavy_stats(const int32_t* __restrict__ rows, int64_t nH, const int64_t* __restrict__ mn,
                              const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff,
                              const uint32_t* __restrict__ ce, const uint32_t* __restrict__ cd,
                              unsigned long long* __restrict__ out) {
  unsigned long long pb = 0, db = 0, ps = 0, ds = 0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = warp; h < nH; h += nwarps) {
    const int64_t i = rows[h];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[h];
    const uint32_t* d = cd + choff[h];
    for (int j = threadIdx.x & 31; j < rb.nb; j += 32) {
      const uint32_t n = __ldg(e + j + 1) - __ldg(e + j), m = __ldg(d + j + 1) - __ldg(d + j);
      if (n > (uint32_t)kBinE) { pb += n; db += m; } else { ps += n; ds += m; }
    }
  }
  atomicAdd(out + 0, pb);
  atomicAdd(out + 1, db);
  atomicAdd(out + 2, ps);
  atomicAdd(out + 3, ds);
}

// Windows and expand units of heavy rows [h0, h1), one warp per row.
__global__ void k_bin_plan(const int32_t* __restrict__ rows, int64_t h0, int64_t h1, const int64_t* __restrict__ mn,
                           const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff,
                           const uint32_t* __restrict__ ce, BinItem* __restrict__ wins, unsigned long long* __restrict__ nwin,
                           BinItem* __restrict__ wins_t,
                           BigItem* __restrict__ bigs, unsigned long long* __restrict__ nbig, BinItem* __restrict__ units,
                           unsigned long long* __restrict__ nunit, int64_t cap_units, int64_t cap_bigs,
                           const uint32_t* __restrict__ cd, const int64_t* __restrict__ hbase, int64_t batch_base,
                           const int64_t* __restrict__ c_rp, const uint32_t* __restrict__ cbm_slot) {
  const int lane = threadIdx.x & 31;
  unsigned long long* nunit_back = nwin + 6;
  unsigned long long* nbig_back = nwin + 7;
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
      // chunks above kBinWinT stand alone, so a packed window never holds more than kBinE
      const uint32_t n_next = valid && cj + 1 < rb.nchunk ? __ldg(e + rb.je(cj + 1)) - pi : 0u;
      const bool next_big = n_next > (uint32_t)kBinWinT;
      // chunks of <= 32 products ("tiny") are reduced in registers by a shared-memory-free
      // kernel: windows never mix tiny and other chunks
      const bool tiny = n <= 32u, next_tiny = n_next <= 32u;
      // ---- reduce windows: runs of small chunks; each sub-bin of a big chunk alone
      // (windows also end every kBinWinT chunks: the direct reducer keeps a cursor per chunk)
      const bool cut = valid && (cj == rb.nchunk - 1 || n > (uint32_t)kBinWinT || next_big || pe / kBinWinT != pi / kBinWinT ||
                                 ((cj + 1) % kBinWinT) == 0 || tiny != next_tiny);
      const uint32_t cm = __ballot_sync(0xffffffffu, cut);
      {
        const uint32_t prev = cm & lanemask_lt();
        const int ws = prev ? q0 + 31 - __clz(prev) + 1 : wstart;
        const int wjs = rb.js(ws);
        const bool emit = cut && !big && pi > __ldg(e + wjs);
        emit_items(emit && !tiny, BinItem{(int32_t)h, wjs, je, 0}, wins, nwin);
        emit_items(emit && tiny, BinItem{(int32_t)h, wjs, je, 0}, wins_t, nwin + 8);
        if (cm) wstart = q0 + 31 - __clz(cm) + 1;
      }
      // big chunks: one item, or column parts of ~kBigSplit elements each (every part
      // streams the whole slice but applies only its own columns)
      if (big) {
        int parts = (int)min((uint32_t)kBigMaxParts, (n + kBigSplit - 1) / kBigSplit);
        const bool large = n >= kBigFront;
        // chunks with more distinct columns than one kBigD pass go to the wide-accumulator list
        const uint32_t* dd = cd + choff[h];
        const uint32_t mcols = __ldg(dd + je) - __ldg(dd + js);
        bool wide = mcols > (uint32_t)kBigD;
#if MG_BIG_WIDE_PARTS > 1
        // tuning: wide chunks as column parts (each part streams the slice and applies its columns)
        if (wide) {
          parts = max(parts, MG_BIG_WIDE_PARTS);
          if (MG_BIG_WIDE_NARROW) wide = false;
        }
#endif
        BigItem* bl = wide ? bigs + cap_bigs : bigs;
        unsigned long long* cf = wide ? nwin + 10 : nbig;
        unsigned long long* cb = wide ? nwin + 15 : nbig_back;
        const unsigned long long b0i = atomicAdd(large ? cf : cb, (unsigned long long)parts);
        const uint32_t* d = cd + choff[h];
        BigItem bi;
        bi.slice = hbase[h] - batch_base + pe;
        bi.out = c_rp[i] + __ldg(d + js);
        bi.n = n;
        bi.m = mcols;
        bi.colbase = (uint32_t)(((rb.b0 + js) >> rb.cs) << shift);
        bi.bslot = cbm_slot != nullptr ? __ldg(cbm_slot + choff[h] + js) : 0xffffffffu;
        bi.pad = 0;
        for (int pp = 0; pp < parts; ++pp) {
          bi.kind = ((uint32_t)parts << 16) | (uint32_t)pp;
          bl[large ? (int64_t)(b0i + pp) : cap_bigs - 1 - (int64_t)(b0i + pp)] = bi;
        }
      }
      // ---- expand units: chunk ranges (whole chunks, so small-chunk slices stay in one unit)
      const bool ucut = valid && (cj == rb.nchunk - 1 ||
                                  (split && (((cj + 1) % ucj) == 0 ||
                                             (int64_t)pe / kBinUnitMax != (int64_t)pi / kBinUnitMax)));
      const uint32_t um = __ballot_sync(0xffffffffu, ucut);
      {
        const uint32_t prev = um & lanemask_lt();
        const int us = prev ? q0 + 31 - __clz(prev) + 1 : ustart;
        const int ujs = rb.js(us);
        const uint32_t un = pi - __ldg(e + ujs);
        const bool uemit = ucut && un > 0;
        emit_items(uemit && un >= kUnitFront, BinItem{(int32_t)h, ujs, je, split ? 0 : 1}, units, nunit);
        emit_items(uemit && un < kUnitFront, BinItem{(int32_t)h, ujs, je, split ? 0 : 1}, units, nunit_back, cap_units);
        if (um) ustart = q0 + 31 - __clz(um) + 1;
      }
    }
  }
}

// Direct big-chunk path (MAGNUS_BIG_PATH=direct): windows and expand units of heavy rows
// [h0, h1), one warp per row.  Big chunks (> kBinE
// products) are reduced straight from B by k_bd_num (big_direct.cuh): they get neither a
// window nor a unit, units never span them, and the small chunks' slices are placed by the
// small-chunk element prefix `cs` (k_bd_plan) -- the reorder buffer holds small-chunk
// products only.
__global__ void k_bin_plan_small(const int32_t* __restrict__ rows, int64_t h0, int64_t h1, const int64_t* __restrict__ mn,
                           const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff,
                           const uint32_t* __restrict__ ce, const uint32_t* __restrict__ cs,
                           BinItem* __restrict__ wins, unsigned long long* __restrict__ nwin,
                           BinItem* __restrict__ wins_t, BinItem* __restrict__ units,
                           unsigned long long* __restrict__ nunit, int64_t cap_units) {
  const int lane = threadIdx.x & 31;
  unsigned long long* nunit_back = nwin + 6;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = h0 + warp; h < h1; h += nwarps) {
    const int64_t i = rows[h];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[h];
    const uint32_t* es = cs + choff[h];
    const int ucj = kBinCur >> rb.cs;                       // chunks per unit (entries <= kBinCur)
    bool rowbig = false;
    for (int q0 = 0; q0 < rb.nchunk && !rowbig; q0 += 32) {
      const int cj = q0 + lane;
      const bool big = cj < rb.nchunk && __ldg(e + rb.je(cj)) - __ldg(e + rb.js(cj)) > (uint32_t)kBinE;
      rowbig = __any_sync(0xffffffffu, big);
    }
    const bool split = rowbig || (int64_t)__ldg(es + rb.nb) > kBinUnitMax || rb.nchunk > ucj;
    int wstart = 0, ustart = 0;
    for (int q0 = 0; q0 < rb.nchunk; q0 += 32) {
      const int cj = q0 + lane;
      const bool valid = cj < rb.nchunk;
      const int js = valid ? rb.js(cj) : 0, je = valid ? rb.je(cj) : 0;
      const uint32_t pe = valid ? __ldg(e + js) : 0u, pi = valid ? __ldg(e + je) : 0u;
      const uint32_t spe = valid ? __ldg(es + js) : 0u, spi = valid ? __ldg(es + je) : 0u;
      const uint32_t n = pi - pe;
      const bool big = valid && n > (uint32_t)kBinE;
      // chunks above kBinWinT stand alone, so a packed window never holds more than kBinE
      const uint32_t n_next = valid && cj + 1 < rb.nchunk ? __ldg(e + rb.je(cj + 1)) - pi : 0u;
      const bool next_big = n_next > (uint32_t)kBinWinT;
      const bool next_isbig = n_next > (uint32_t)kBinE;
      // chunks of <= 32 products ("tiny") are reduced in registers by a shared-memory-free
      // kernel: windows never mix tiny and other chunks
      const bool tiny = n <= 32u, next_tiny = n_next <= 32u;
      // ---- reduce windows: runs of small chunks; each sub-bin of a big chunk alone
      // (windows also end every kBinWinT chunks: the direct reducer keeps a cursor per chunk)
      const bool cut = valid && (cj == rb.nchunk - 1 || n > (uint32_t)kBinWinT || next_big || pe / kBinWinT != pi / kBinWinT ||
                                 ((cj + 1) % kBinWinT) == 0 || tiny != next_tiny);
      const uint32_t cm = __ballot_sync(0xffffffffu, cut);
      {
        const uint32_t prev = cm & lanemask_lt();
        const int ws = prev ? q0 + 31 - __clz(prev) + 1 : wstart;
        const int wjs = rb.js(ws);
        const bool emit = cut && !big && pi > __ldg(e + wjs);
        emit_items(emit && !tiny, BinItem{(int32_t)h, wjs, je, 0}, wins, nwin);
        emit_items(emit && tiny, BinItem{(int32_t)h, wjs, je, 0}, wins_t, nwin + 8);
        if (cm) wstart = q0 + 31 - __clz(cm) + 1;
      }
      // ---- expand units: runs of small chunks (whole chunks, so small-chunk slices stay in one
      // unit), cut at big chunks
      const bool ucut = valid && (cj == rb.nchunk - 1 || big || next_isbig ||
                                  (split && (((cj + 1) % ucj) == 0 ||
                                             (int64_t)spe / kBinUnitMax != (int64_t)spi / kBinUnitMax)));
      const uint32_t um = __ballot_sync(0xffffffffu, ucut);
      {
        const uint32_t prev = um & lanemask_lt();
        const int us = prev ? q0 + 31 - __clz(prev) + 1 : ustart;
        const int ujs = rb.js(us);
        const uint32_t un = spi - __ldg(es + ujs);
        const bool uemit = ucut && !big && un > 0;
        emit_items(uemit && un >= kUnitFront, BinItem{(int32_t)h, ujs, je, split ? 0 : 1}, units, nunit);
        emit_items(uemit && un < kUnitFront, BinItem{(int32_t)h, ujs, je, split ? 0 : 1}, units, nunit_back, cap_units);
        if (um) ustart = q0 + 31 - __clz(um) + 1;
      }
    }
  }
}

// Expand, two-pass variant: one CTA per unit.  The unit's stream (its k segments in
// ascending k) is split into kE2W contiguous warp ranges.  Pass 1 counts each warp's
// products per chunk; a prefix over warps gives every warp its starting slot in every
// chunk slice; pass 2 walks the same range again and appends products to the slices
// (stable: warp ranges are in stream order, and inside a wave lanes are in stream order).
// Loads are 32 consecutive B elements per wave, mostly inside one B row (no search).
#ifndef MG_E2_T
#define MG_E2_T 256
#endif
#ifndef MG_E2_K
#define MG_E2_K 256
#endif
constexpr int kE2T = MG_E2_T;              // threads per CTA
constexpr int kE2W = kE2T / 32;            // warp ranges per unit
constexpr int kE2K = MG_E2_K;              // k's whose segments live in shared memory
#ifndef MG_E2_U
#define MG_E2_U 4
#endif
constexpr int kE2U = MG_E2_U;              // waves in flight per warp
#ifndef MG_RED_TICKET_AHEAD
#define MG_RED_TICKET_AHEAD 0
#endif
#ifndef MG_E2_TICKET_AHEAD
#define MG_E2_TICKET_AHEAD 0
#endif
#ifndef MG_E2_P1_SPLIT
#define MG_E2_P1_SPLIT 0
#endif
constexpr bool kE2P1Split = MG_E2_P1_SPLIT != 0;   // pass 1 split across warps independently of ownership
struct Exp2Smem {
  static constexpr size_t kCnt = (size_t)kE2W * kBinCur * 4;            // per warp, per chunk of the unit
  static constexpr size_t kK = (size_t)(kE2K + 32) * (4 + 4 + 8 + 4);   // koff, kpos, kav, kslot
  static constexpr size_t kScratch = 64 * 8;
  static constexpr size_t kTotal = kCnt + kK + kScratch;
};

__device__ __forceinline__ void sh_red_add_pred(bool p, uint32_t addr, uint32_t v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q red.shared.add.u32 [%1], %2;\n}\n"
               :: "r"((uint32_t)p), "r"(addr), "r"(v) : "memory");
}

// position q of the unit's stream -> (segment, B position); the warp keeps the segment of
// its last position (kk, kend = first position past it, base = B position - q)
template <class KP>
struct E2Cursor {
  KP koff, kpos;
  int nk, kk;
  uint32_t kend, base;
  __device__ __forceinline__ void init(uint32_t q_beg) {
    int lo = 0, hi = nk;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (koff[mid] <= q_beg) lo = mid; else hi = mid;
    }
    kk = lo;
    kend = koff[kk + 1];
    base = kpos[kk] - koff[kk];
  }
  // B position of this lane's q in the wave starting at q0 (warp-uniform call); seg: segment
  // of the position; returns true when the wave may span several segments
  __device__ __forceinline__ bool wave(uint32_t q0, uint32_t q, uint32_t q_end, uint32_t& pos, int& seg) {
    pos = base + q;
    seg = kk;
    if (q0 + 31 < kend || q0 >= q_end) return false;
    int kl = kk;
#ifndef MG_E2_SCAN_SEG
    // lane j holds the start of segment kk+1+j; when the wave ends before the 32nd of them, a
    // lane's segment is kk + (starts <= q), found by a 5-step search over the shuffled starts
    const int jb = kk + 1 + (threadIdx.x & 31);
    const uint32_t bnd = jb <= nk ? koff[jb] : 0xffffffffu;
    if (__shfl_sync(0xffffffffu, bnd, 31) > q0 + 31) {
      int cnt = 0;
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1)
        if (__shfl_sync(0xffffffffu, bnd, cnt + st - 1) <= q) cnt += st;
      kl += cnt;
    } else
#endif
      while (kl < nk && koff[kl + 1] <= q) ++kl;
    pos = kpos[kl] + (q - koff[kl]);
    seg = kl;
    kk = __shfl_sync(0xffffffffu, kl, 31);
    kend = koff[kk + 1];
    base = kpos[kk] - koff[kk];
    return true;
  }
  // the kE2U waves from q00 at once (warp-uniform call, q00 < q_end): per wave the lane's B
  // position, its segment and whether the wave may span several segments.  When the batch
  // ends before the 32nd segment start after kk, every wave searches the same shuffled starts
  // (one shared-memory load per batch, no cursor chain from wave to wave).
  template <int U>
  __device__ __forceinline__ void batch(uint32_t q00, uint32_t q_end, uint32_t (&pos)[U], int (&seg)[U], bool (&multi)[U]) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t qlast = q00 + 32 * U - 1;
    if (qlast < kend) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pos[u] = base + q00 + 32 * u + lane;
        seg[u] = kk;
        multi[u] = false;
      }
      return;
    }
    const int jb = kk + 1 + (int)lane;
    const uint32_t bnd = jb <= nk ? koff[jb] : 0xffffffffu;
    const uint32_t qstop = min(qlast, q_end - 1);
    if (__shfl_sync(0xffffffffu, bnd, 31) > qstop) {
      auto starts_le = [&](uint32_t q) {
        int cnt = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1)
          if (__shfl_sync(0xffffffffu, bnd, cnt + st - 1) <= q) cnt += st;
        return cnt;
      };
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q0 = q00 + 32 * u, q = q0 + lane;
        if (q0 + 31 < kend) {
          pos[u] = base + q;
          seg[u] = kk;
          multi[u] = false;
        } else {
          const int kl = kk + starts_le(min(q, qstop));
          pos[u] = kpos[kl] + (q - koff[kl]);
          seg[u] = kl;
          multi[u] = true;
        }
      }
      kk += starts_le(qstop);
      kend = koff[kk + 1];
      base = kpos[kk] - koff[kk];
      return;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) multi[u] = wave(q00 + 32 * u, q00 + 32 * u + lane, q_end, pos[u], seg[u]);
  }
};

template <class KP, class KA, class KS>
__device__ __forceinline__ void exp2_unit(const DevCsr& B, KP koff, KP kpos, KA kav, KS kslot, int nk, uint32_t T, int shift,
                                          uint32_t cb, uint32_t* cnt, const uint32_t* __restrict__ e, int ja, int nent,
                                          uint16_t* __restrict__ rc, double* __restrict__ rv,
                                          const uint32_t* __restrict__ bidx, int64_t nwin1, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t L = ((T + kE2W - 1) / kE2W + 31) & ~31u;
  const uint32_t q_beg = min(T, (uint32_t)wid * L), q_end = min(T, q_beg + L);
  uint32_t* wc = cnt + (size_t)wid * kBinCur;
  const uint32_t a_wc = (uint32_t)__cvta_generic_to_shared(wc);
  const uint32_t lt = lanemask_lt(), le = lanemask_le();
  const uint32_t cmask = (1u << shift) - 1u;
  // ---- pass 1: products per chunk of this warp's range.  A B row segment that lies wholly
  // in the range and holds more elements than the unit has chunks is counted from the B
  // window index (one difference per chunk); the other positions column by column.
  uint32_t a_p1 = a_wc;   // counters pass 1 is adding to (owner of the current range)
  auto count_range = [&](uint32_t qa, uint32_t qb) {
    if (qa >= qb) return;
    E2Cursor<KP> cur{koff, kpos, nk, 0, 0, 0};
    cur.init(qa);
    for (uint32_t q00 = qa; q00 < qb; q00 += 32 * kE2U) {
      uint32_t cw[kE2U], pos[kE2U];
      int seg[kE2U];
      bool multi[kE2U];
#ifdef MG_E2_WAVE_CURSOR
#pragma unroll
      for (int u = 0; u < kE2U; ++u) cur.wave(q00 + 32 * u, q00 + 32 * u + lane, qb, pos[u], seg[u]);
#else
      cur.batch(q00, qb, pos, seg, multi);
#endif
#pragma unroll
      for (int u = 0; u < kE2U; ++u) {
        const uint32_t q = q00 + 32 * u + lane;
        cw[u] = q < qb ? __ldg(B.col + pos[u]) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < kE2U; ++u) {
        if (q00 + 32 * u >= qb) break;
        const bool valid = cw[u] != 0xffffffffu;
        const uint32_t ch = valid ? (cw[u] >> shift) - cb : 0xffffffffu;
        const uint32_t pch = __shfl_up_sync(0xffffffffu, ch, 1);
        const bool head = lane == 0 || ch != pch;
        const uint32_t hm = __ballot_sync(0xffffffffu, head);
        const uint32_t after = hm & ~le;
        const uint32_t nxt = after ? (uint32_t)(__ffs(after) - 1) : 32u;
        sh_red_add_pred(valid && head, a_p1 + (ch << 2), nxt - (uint32_t)lane);
      }
    }
  };
  // pass 1's work split is decoupled from the owner ranges: warp w counts part
  // (w - o) mod kE2W of every owner o's range into o's counters (red.shared: atomic), so a
  // range of short, column-by-column pieces is spread over all warps
  const uint32_t Ls = kE2P1Split ? (((L + kE2W - 1) / kE2W + 31) & ~31u) : L;
  for (int oo = 0; oo < (kE2P1Split ? kE2W : 1); ++oo) {
    const int o = kE2P1Split ? oo : wid;
    const int jp = kE2P1Split ? ((wid - o + kE2W) % kE2W) : 0;
    const uint32_t ob = min(T, (uint32_t)o * L), oe = min(T, ob + L);
    const uint32_t p_beg = min(oe, ob + (uint32_t)jp * Ls), p_end = min(oe, p_beg + Ls);
    a_p1 = (uint32_t)__cvta_generic_to_shared(cnt + (size_t)o * kBinCur);
    if (p_beg < p_end) {
      // segment of p_beg
      int lo = 0, hi = nk;   // koff[lo] <= p_beg < koff[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (koff[mid] <= p_beg) lo = mid; else hi = mid;
      }
      uint32_t q = p_beg;   // positions below q are counted
      // 32 segments at a time: each lane classifies one (its end columns are loaded in
      // parallel), then the eligible ones are counted from the window index in stream order
      for (int j0 = lo; j0 < nk && koff[j0] < p_end; j0 += 32) {
        const int j = j0 + lane;
        bool el = false;
        uint32_t qa = 0, qb = 0, P0 = 0, c0 = 0, c1 = 0;
        int32_t sl = -1;
        if (j < nk && koff[j] < p_end) {
          qa = max(p_beg, (uint32_t)koff[j]);
          qb = min(p_end, (uint32_t)koff[j + 1]);
          sl = (int32_t)kslot[j];
          if (sl >= 0 && qb - qa >= 64u) {
            // the piece [P0, P0 + qb - qa) of B row j inside this range: chunks c0..c1 of the unit
            P0 = kpos[j] + (qa - koff[j]);
            c0 = (__ldg(B.col + P0) >> shift) - cb;
            c1 = (__ldg(B.col + P0 + (qb - qa) - 1) >> shift) - cb;
            el = c1 - c0 + 1 <= qb - qa;   // else sparser than one element per chunk: count columns
          }
        }
        uint32_t m = __ballot_sync(0xffffffffu, el);
        while (m) {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t sqa = __shfl_sync(0xffffffffu, qa, src), sqb = __shfl_sync(0xffffffffu, qb, src);
          const uint32_t sP0 = __shfl_sync(0xffffffffu, P0, src), sP1 = sP0 + (sqb - sqa);
          const uint32_t sc0 = __shfl_sync(0xffffffffu, c0, src), sc1 = __shfl_sync(0xffffffffu, c1, src);
          const int32_t ssl = __shfl_sync(0xffffffffu, sl, src);
          count_range(q, sqa);
          const uint32_t* ix = bidx + (size_t)ssl * nwin1 + cb;
          for (uint32_t cc = sc0; cc <= sc1; cc += 128) {
            uint32_t lo_c[4], hi_c[4];
  #pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t c = cc + 32 * u + lane;
              lo_c[u] = hi_c[u] = 0u;
              if (c <= sc1) {
                lo_c[u] = max(sP0, __ldg(ix + c));
                hi_c[u] = min(sP1, __ldg(ix + c + 1));
              }
            }
  #pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t c = cc + 32 * u + lane;
              sh_red_add_pred(hi_c[u] > lo_c[u], a_p1 + (c << 2), hi_c[u] - lo_c[u]);
            }
          }
          q = sqb;
        }
      }
      count_range(q, p_end);
    }
  }
  __syncthreads();
  // ---- slice starts: chunk start (row-relative, from the symbolic tables) + earlier warps
  for (int c = threadIdx.x; c < nent; c += kE2T) {
    uint32_t run = __ldg(e + ja + c);
#pragma unroll
    for (int w = 0; w < kE2W; ++w) {
      const uint32_t v = cnt[(size_t)w * kBinCur + c];
      cnt[(size_t)w * kBinCur + c] = run;
      run += v;
    }
  }
  __syncthreads();
  // ---- pass 2: append (chunk-local column, product) to the slices.  Software-pipelined: the B
  // loads of the next batch of waves are issued before the current batch is ranked and stored.
  if (q_beg < q_end) {
    E2Cursor<KP> cur{koff, kpos, nk, 0, 0, 0};
    cur.init(q_beg);
    uint32_t ncw[kE2U], pos[kE2U];
    double nvv[kE2U];
    bool nmulti[kE2U];
    int nseg[kE2U];
    auto fetch = [&](uint32_t q00) {
      cur.batch(q00, q_end, pos, nseg, nmulti);
#pragma unroll
      for (int u = 0; u < kE2U; ++u) {
        const uint32_t q = q00 + 32 * u + lane;
        ncw[u] = 0xffffffffu;
        nvv[u] = 0.0;
        if (q < q_end) {
          ncw[u] = __ldg(B.col + pos[u]);
          nvv[u] = __ldg(B.val + pos[u]);
        }
      }
    };
    fetch(q_beg);
    for (uint32_t q00 = q_beg; q00 < q_end; q00 += 32 * kE2U) {
      uint32_t cw[kE2U];
      double vw[kE2U];
      bool multi[kE2U];
      int seg[kE2U];
#pragma unroll
      for (int u = 0; u < kE2U; ++u) {
        cw[u] = ncw[u];
        vw[u] = nvv[u];
        multi[u] = nmulti[u];
        seg[u] = nseg[u];
      }
      if (q00 + 32 * kE2U < q_end) fetch(q00 + 32 * kE2U);
#pragma unroll
      for (int u = 0; u < kE2U; ++u) vw[u] = __dmul_rn(kav[seg[u]], vw[u]);
#pragma unroll
      for (int u = 0; u < kE2U; ++u) {
        if (q00 + 32 * u >= q_end) break;
        const bool valid = cw[u] != 0xffffffffu;
        const uint32_t ch = valid ? (cw[u] >> shift) - cb : 0x40000000u + lane;
        uint32_t rank, lastm;
        if (!multi[u]) {
          // one B row: equal chunks form contiguous runs
          const uint32_t pch = __shfl_up_sync(0xffffffffu, ch, 1), nch = __shfl_down_sync(0xffffffffu, ch, 1);
          const uint32_t hm = __ballot_sync(0xffffffffu, lane == 0 || ch != pch);
          rank = (uint32_t)lane - (31u - __clz(hm & le));
          lastm = __ballot_sync(0xffffffffu, lane == 31 || ch != nch);
        } else {
          const uint32_t peers = __match_any_sync(0xffffffffu, ch);
          rank = __popc(peers & lt);
          lastm = __ballot_sync(0xffffffffu, (peers >> lane) == 1u);
        }
        uint32_t slot = 0;
        if (valid) slot = wc[ch] + rank;
        __syncwarp();
        if (valid && ((lastm >> lane) & 1u)) wc[ch] = slot + 1;
        if (valid) {
          // streaming stores: the reorder buffer must not evict the B rows from L2
          __stcs(rc + slot, (uint16_t)(cw[u] & cmask));
          __stcs(rv + slot, vw[u]);
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  (void)scratch;
}

// 4 CTAs/SM: the pipelined pass 2 fits 61 registers without spills (5 CTAs spill, 208 vs 162 ms on cfg3;
// no minBlocks at all lets ptxas take 64 registers plus a stack)
#ifndef MG_E2_MINB
#define MG_E2_MINB 4
#endif
__global__ void __launch_bounds__(kE2T, MG_E2_MINB)
k_bin_expand2(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, const int64_t* __restrict__ mn,
              const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce,
              const int64_t* __restrict__ hbase, int64_t batch_base, const BinItem* __restrict__ units,
              const unsigned long long* __restrict__ nunit, unsigned long long* __restrict__ ticket, int64_t cap_units,
              uint16_t* __restrict__ bcol, double* __restrict__ bval, const int32_t* __restrict__ bslot,
              const uint32_t* __restrict__ bidx, int64_t nwin1, int ilog, uint32_t* __restrict__ gk, int64_t gk_stride,
              unsigned long long* __restrict__ err, const int8_t* __restrict__ skip_coarse = nullptr) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);
  double* s_kav = reinterpret_cast<double*>(smem + Exp2Smem::kCnt);
  uint32_t* s_koff = reinterpret_cast<uint32_t*>(smem + Exp2Smem::kCnt + (size_t)(kE2K + 32) * 8);
  uint32_t* s_kpos = s_koff + kE2K + 32;
  uint32_t* s_kslot = s_kpos + kE2K + 32;
  uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + Exp2Smem::kCnt + Exp2Smem::kK);
  __shared__ unsigned long long s_u;
  const uint64_t nu_front = nunit[0], nu = nu_front + nunit[5];
#if MG_E2_TICKET_AHEAD
  // the next ticket is taken while the current unit is expanded (its write to s_u is read
  // after the barriers inside the unit)
  if (threadIdx.x == 0) s_u = atomicAdd(ticket, 1ull);
  __syncthreads();
#endif
  while (true) {
#if !MG_E2_TICKET_AHEAD
    if (threadIdx.x == 0) s_u = atomicAdd(ticket, 1ull);
    __syncthreads();
#endif
    const unsigned long long u = s_u;
    __syncthreads();
    if (u >= nu) break;
#if MG_E2_TICKET_AHEAD
    if (threadIdx.x == 0) s_u = atomicAdd(ticket, 1ull);
#endif
    const BinItem it = units[list_slot(u, nu_front, cap_units)];
    const int64_t i = rows[it.h];
    // rows of the Coarse category are expanded by the coarse level (coarse_rows.cuh)
    if (skip_coarse != nullptr && skip_coarse[i] == kCatCoarse) continue;
    const int64_t a0 = A.rp(i);
    const int nk = (int)(A.rp(i + 1) - a0);
    const RowBins rb = row_bins(mn[i], mx[i], shift);   // shift <= kSubShift: entries == chunks
    const uint32_t* e = ce + choff[it.h];
    const int nent = it.jb - it.ja;
    const uint32_t clo = (uint32_t)((rb.b0 + it.ja) << shift);
    const int64_t chi64 = (rb.b0 + it.jb) << shift;
    const uint32_t chi = chi64 >= ((int64_t)1 << 32) ? 0xffffffffu : (uint32_t)chi64;
    const bool big_nk = nk > kE2K;
    uint32_t* koff = big_nk ? gk + (size_t)blockIdx.x * gk_stride * 5 : s_koff;
    uint32_t* kpos = big_nk ? koff + gk_stride : s_kpos;
    double* kav = big_nk ? reinterpret_cast<double*>(koff + 2 * gk_stride) : s_kav;
    uint32_t* kslot = big_nk ? koff + 4 * gk_stride : s_kslot;
    for (int j = threadIdx.x; j < nk; j += kE2T) {
      const int64_t k = __ldg(A.col + a0 + j);
      uint32_t p0 = (uint32_t)B.rp(k), p1 = (uint32_t)B.rp(k + 1);
      const int32_t sl = __ldg(bslot + k);
      kslot[j] = (uint32_t)sl;
      if (!it.kind) {
        if (sl >= 0) {
          const uint32_t* ix = bidx + (size_t)sl * nwin1;
          p0 = __ldg(ix + min((int64_t)(clo >> ilog), nwin1 - 1));
          p1 = __ldg(ix + min(chi64 >> ilog, nwin1 - 1));
        } else {
          p0 = lower_bound_col(B.col, p0, p1, clo);
          p1 = lower_bound_col(B.col, p0, p1, chi);
        }
      }
      koff[j] = p1 - p0;
      kpos[j] = p0;
      kav[j] = __ldg(A.val + a0 + j);
    }
    for (int c = threadIdx.x; c < kE2W * nent; c += kE2T) cnt[(c / nent) * kBinCur + (c % nent)] = 0u;
    __syncthreads();
    const uint32_t T = block_scan_striped<kE2T>(koff, nk, scratch);
    if (threadIdx.x == 0) koff[nk] = T;
    __syncthreads();
    if (T != __ldg(e + it.jb) - __ldg(e + it.ja)) {
      if (threadIdx.x == 0) atomicOr(err, 4ull);
      continue;
    }
    const int64_t rowbase = hbase[it.h] - batch_base;
    if (big_nk)
      exp2_unit(B, (const uint32_t*)koff, (const uint32_t*)kpos, (const double*)kav, (const uint32_t*)kslot, nk, T, shift,
                (uint32_t)(rb.b0 + it.ja), cnt, e, it.ja, nent, bcol + rowbase, bval + rowbase, bidx, nwin1, scratch);
    else
      exp2_unit(B, (const uint32_t*)s_koff, (const uint32_t*)s_kpos, (const double*)s_kav, (const uint32_t*)s_kslot, nk, T,
                shift, (uint32_t)(rb.b0 + it.ja), cnt, e, it.ja, nent, bcol + rowbase, bval + rowbase, bidx, nwin1,
                scratch);
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
  uint16_t* inv;   // rank -> column
};

// Small chunk (n <= kBinE elements): stable counting sort of the slice by column rank
// into shared memory, then one lane per column sums its run with the chunk's association.
// (GlobalIn: the slice is in global memory and read through the read-only path; else it is
// a shared-memory list and must not be: const __restrict__ loads may become ld.global.nc.)
template <bool GlobalIn = true>
__device__ __forceinline__ bool reduce_chunk_sort(const uint16_t* sc, const double* sv_g,
                                                  uint32_t n, uint32_t m, uint64_t seqmask, int mshift, uint32_t colbase,
                                                  const ReduceSmem& S,
                                                  uint32_t* __restrict__ c_col, double* __restrict__ c_val, int64_t out) {
  const int lane = threadIdx.x & 31;
  uint32_t cmin = 0xffffu, cmax = 0u;
  for (uint32_t q = lane; q < n; q += 32) {
    const uint32_t c = GlobalIn ? (uint32_t)__ldg(sc + q) : (uint32_t)sc[q];
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
    const uint32_t c = S.stc[q];
    const uint32_t r = rank_of(S.bm, S.pref, c);
    S.inv[r] = (uint16_t)c;
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
    const double v = valid ? (GlobalIn ? __ldg(sv_g + q) : sv_g[q]) : 0.0;
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
#ifdef MG_DIR_DEBUG
    if (!(s0 <= e0 && e0 <= n)) { printf("sortred r %u s0 %u e0 %u n %u m %u\n", r, s0, e0, n, m); asm volatile("trap;"); }
#endif
    const uint32_t cl = S.inv[r];
    __stcs(c_col + out + r, colbase + cl);
    // association of the column's chunk: bit (cl >> mshift) of seqmask
    __stcs(c_val + out + r,
           ((seqmask >> (cl >> mshift)) & 1ull) ? sum_seq_s(S.sval, s0, e0) : sum_pairwise_s(S.sval, s0, e0));
  }
  __syncwarp();
  return true;
}

// Chunk of at most 32 products (about half of all chunks of heavy rows): one product per
// lane, sorted by (column, stream position) with a register bitonic network, runs of equal
// columns summed with the chunk's association -- sequential from +0.0 (dense) or
// x0 + (((-0.0 + x1) + x2) + ...) (np.add.reduceat, numpy pairwise below 8 terms).
// Returns 1 ok, 0 count mismatch.
// (core: this lane's product already loaded -- cl its chunk-local column, v its value)
__device__ __forceinline__ int reduce_chunk_wave_core(uint32_t cl, double v, uint32_t n, uint32_t m, bool seq,
                                                      uint32_t colbase, uint32_t* __restrict__ c_col,
                                                      double* __restrict__ c_val, int64_t out) {
  const int lane = threadIdx.x & 31;
  const bool valid = (uint32_t)lane < n;
  uint32_t key = valid ? (cl << 5) | (uint32_t)lane : 0xffffffffu;
  if (!valid) v = 0.0;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t pk = __shfl_xor_sync(0xffffffffu, key, j);
      const double pv = __shfl_xor_sync(0xffffffffu, v, j);
      const bool up = (lane & k) == 0 || k == 32;
      const bool lower = (lane & j) == 0;
      const bool take = lower ? (up ? pk < key : pk > key) : (up ? pk > key : pk < key);
      if (take) {
        key = pk;
        v = pv;
      }
    }
  }
  const uint32_t c = key >> 5;
  const uint32_t pc = __shfl_up_sync(0xffffffffu, c, 1);
  const bool head = valid && (lane == 0 || c != pc);
  const uint32_t hm = __ballot_sync(0xffffffffu, head);
  const uint32_t after = hm & ~lanemask_le();
  const uint32_t runlen = head ? (after ? (uint32_t)(__ffs(after) - 1) : n) - (uint32_t)lane : 0u;
  const uint32_t maxd = __reduce_max_sync(0xffffffffu, runlen);
  double acc = seq ? __dadd_rn(0.0, v) : v;
  if (maxd <= 8u) {
    double rest = -0.0;
    for (uint32_t t = 1; t < maxd; ++t) {
      const double x = __shfl_sync(0xffffffffu, v, min(lane + (int)t, 31));
      if (t < runlen) {
        if (seq) acc = __dadd_rn(acc, x);
        else rest = __dadd_rn(rest, x);
      }
    }
    if (!seq && runlen > 1) acc = __dadd_rn(acc, rest);
  } else {
    // a column with 9..32 products: numpy's pairwise of x1..x_{d-1} (8 strided partial sums,
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), the remainder sequentially), streamed over shuffles
    const int nr = (int)runlen - 1;   // rest terms x_1..x_nr
    const int full = nr >= 8 ? nr - nr % 8 : 0;
    double r[8];
    double res = -0.0;
    bool combined = nr < 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = 0.0;
#pragma unroll
    for (int t = 1; t < 32; ++t) {
      const double x = __shfl_sync(0xffffffffu, v, min(lane + t, 31));
      if (t <= nr) {
        if (seq) {
          acc = __dadd_rn(acc, x);
        } else if (t - 1 < full) {
          r[(t - 1) % 8] = t <= 8 ? x : __dadd_rn(r[(t - 1) % 8], x);
        } else {
          if (!combined) {
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            combined = true;
          }
          res = __dadd_rn(res, x);
        }
      }
    }
    if (!seq && nr > 0) {
      if (!combined)
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      acc = __dadd_rn(acc, res);
    }
  }
  const uint32_t rank = __popc(hm & lanemask_lt());
  if (head) {
    __stcs(c_col + out + rank, colbase + c);
    __stcs(c_val + out + rank, acc);
  }
  return __popc(hm) == m ? 1 : 0;
}

__device__ __forceinline__ int reduce_chunk_wave(const uint16_t* __restrict__ sc, const double* __restrict__ sv, uint32_t n,
                                                 uint32_t m, bool seq, uint32_t colbase, uint32_t* __restrict__ c_col,
                                                 double* __restrict__ c_val, int64_t out) {
  const int lane = threadIdx.x & 31;
  const bool valid = (uint32_t)lane < n;
  return reduce_chunk_wave_core(valid ? (uint32_t)__ldg(sc + lane) : 0u, valid ? __ldg(sv + lane) : 0.0, n, m, seq, colbase,
                                c_col, c_val, out);
}

// Prefetch the reorder-buffer range [q0, q1) of a window (columns + values) into L2: the
// window's chunks are then reduced from L2 instead of one DRAM round trip each.
__device__ __forceinline__ void prefetch_slice(const uint16_t* bcol, const double* bval, int64_t q0, int64_t q1) {
  const int lane = threadIdx.x & 31;
  const char* c0 = reinterpret_cast<const char*>(bcol + q0);
  const char* c1 = reinterpret_cast<const char*>(bcol + q1);
  for (const char* p = c0 + lane * 128; p < c1; p += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  const char* v0 = reinterpret_cast<const char*>(bval + q0);
  const char* v1 = reinterpret_cast<const char*>(bval + q1);
  for (const char* p = v0 + lane * 128; p < v1; p += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Reduce, windows of tiny chunks (<= 32 products each): one warp per window, no shared memory.
__global__ void __launch_bounds__(256, 4)
k_bin_reduce_tiny(const int32_t* __restrict__ rows, const int8_t* __restrict__ cat, const int64_t* __restrict__ mn,
                  const int64_t* __restrict__ mx, Sem sem, const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce,
                  const uint32_t* __restrict__ cd, const int64_t* __restrict__ hbase, int64_t batch_base,
                  const BinItem* __restrict__ wins, const unsigned long long* __restrict__ nwin,
                  unsigned long long* __restrict__ ticket, const uint16_t* __restrict__ bcol,
                  const double* __restrict__ bval, const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
                  double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int shift = sem.shift_num, gs = bin_shift_of(shift);
  const int64_t nw = (int64_t)*nwin;
  const uint32_t cwmask = ~((1u << shift) - 1u);
#if MG_RED_TICKET_AHEAD
  // the next window's ticket is taken while the current window is reduced
  unsigned long long wnext = 0;
  if (lane == 0) wnext = atomicAdd(ticket, 1ull);
#endif
  while (true) {
    unsigned long long wi = 0;
#if MG_RED_TICKET_AHEAD
    wi = __shfl_sync(0xffffffffu, wnext, 0);
    if ((int64_t)wi >= nw) break;
    if (lane == 0) wnext = atomicAdd(ticket, 1ull);
#else
    if (lane == 0) wi = atomicAdd(ticket, 1ull);
    wi = __shfl_sync(0xffffffffu, wi, 0);
    if ((int64_t)wi >= nw) break;
#endif
    const BinItem it = wins[wi];
    const int64_t i = rows[it.h];
    const int ci = cat[i];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[it.h];
    const uint32_t* d = cd + choff[it.h];
    const int64_t rowbase = hbase[it.h] - batch_base;
    const int64_t out_row = c_rp[i];
    prefetch_slice(bcol, bval, rowbase + __ldg(e + it.ja), rowbase + __ldg(e + it.jb));
    bool ok = true;
    for (int j0 = it.ja; j0 < it.jb; j0 += 32) {
      // chunk table entries of 32 chunks (tiny windows: sub-bins == chunks)
      const uint32_t e_l = j0 + lane <= it.jb ? __ldg(e + j0 + lane) : 0u;
      const uint32_t d_l = j0 + lane <= it.jb ? __ldg(d + j0 + lane) : 0u;
      const int jn = min(it.jb - j0, 32);
      const uint32_t e_last = __ldg(e + j0 + jn), d_last = __ldg(d + j0 + jn);
      // software-pipelined: the next chunk's product is loaded while this one is sorted and summed
      auto bounds = [&](int t, uint32_t& ej, uint32_t& n) {
        ej = __shfl_sync(0xffffffffu, e_l, min(t, 31));
        const uint32_t en = t + 1 < 32 ? __shfl_sync(0xffffffffu, e_l, min(t + 1, 31)) : e_last;
        n = (t + 1 == jn ? e_last : en) - ej;
      };
      uint32_t ej, n;
      bounds(0, ej, n);
      uint32_t ncl = (uint32_t)lane < n ? (uint32_t)__ldg(bcol + rowbase + ej + lane) : 0u;
      double nv = (uint32_t)lane < n ? __ldg(bval + rowbase + ej + lane) : 0.0;
      for (int t = 0; t < jn; ++t) {
        const uint32_t cl = ncl, cn = n;
        const double v = nv;
        const uint32_t dj = __shfl_sync(0xffffffffu, d_l, t);
        const uint32_t dn = t + 1 < 32 ? __shfl_sync(0xffffffffu, d_l, min(t + 1, 31)) : d_last;
        const uint32_t m = (t + 1 == jn ? d_last : dn) - dj;
        if (t + 1 < jn) {
          bounds(t + 1, ej, n);
          ncl = (uint32_t)lane < n ? (uint32_t)__ldg(bcol + rowbase + ej + lane) : 0u;
          nv = (uint32_t)lane < n ? __ldg(bval + rowbase + ej + lane) : 0.0;
        }
        if (cn == 0) continue;
        const bool seq = ci == kCatDense || (int64_t)cn >= sem.crossover;
        const uint32_t colbase = (uint32_t)((rb.b0 + j0 + t) << gs) & cwmask;
        ok &= reduce_chunk_wave_core(cl, v, cn, m, seq, colbase, c_col, c_val, out_row + dj) == 1;
      }
    }
    if (!ok && lane == 0) atomicOr(err, 4ull);
  }
}

// Reduce: one warp per window.
__global__ void __launch_bounds__(kBinT, 8)
k_bin_reduce(const int32_t* __restrict__ rows, const int8_t* __restrict__ cat, const int64_t* __restrict__ mn,
             const int64_t* __restrict__ mx, Sem sem, const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce,
             const uint32_t* __restrict__ cd, const int64_t* __restrict__ hbase, int64_t batch_base,
             const BinItem* __restrict__ wins, const unsigned long long* __restrict__ nwin,
             unsigned long long* __restrict__ ticket, const uint16_t* __restrict__ bcol,
             const double* __restrict__ bval, const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
             double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
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
  S.inv = reinterpret_cast<uint16_t*>(base + w4 + w2 + (size_t)kBinE * 12);
  const int64_t nw = (int64_t)*nwin;
  const uint32_t cwmask = ~((1u << shift) - 1u);
#if MG_RED_TICKET_AHEAD
  // the next window's ticket is taken while the current window is reduced
  unsigned long long wnext = 0;
  if ((threadIdx.x & 31) == 0) wnext = atomicAdd(ticket, 1ull);
#endif
  while (true) {
    unsigned long long wi = 0;
#if MG_RED_TICKET_AHEAD
    wi = __shfl_sync(0xffffffffu, wnext, 0);
    if ((int64_t)wi >= nw) break;
    if ((threadIdx.x & 31) == 0) wnext = atomicAdd(ticket, 1ull);
#else
    if ((threadIdx.x & 31) == 0) wi = atomicAdd(ticket, 1ull);
    wi = __shfl_sync(0xffffffffu, wi, 0);
    if ((int64_t)wi >= nw) break;
#endif
    const BinItem it = wins[wi];
    const int64_t i = rows[it.h];
    const int ci = cat[i];
    const RowBins rb = row_bins(mn[i], mx[i], shift);
    const uint32_t* e = ce + choff[it.h];
    const uint32_t* d = cd + choff[it.h];
    const int64_t rowbase = hbase[it.h] - batch_base;
    const int64_t out_row = c_rp[i];
    prefetch_slice(bcol, bval, rowbase + __ldg(e + it.ja), rowbase + __ldg(e + it.jb));
    bool ok = true;
    // chunk table entries of the window, 32 chunks per load (lane l: chunk j0 + l)
    int j0 = -1 << 30;
    uint32_t e_l = 0, d_l = 0;
    int j = it.ja;
    while (j < it.jb) {
      const int je = (int)min((int64_t)it.jb, ((((rb.b0 + j) >> rb.cs) + 1) << rb.cs) - rb.b0);
      if (j < j0 || je >= j0 + 32) {
        j0 = j;
        e_l = j0 + lane <= it.jb ? __ldg(e + j0 + lane) : 0u;
        d_l = j0 + lane <= it.jb ? __ldg(d + j0 + lane) : 0u;
      }
      const uint32_t ej = __shfl_sync(0xffffffffu, e_l, j - j0), n = __shfl_sync(0xffffffffu, e_l, je - j0) - ej;
      const uint32_t dj = __shfl_sync(0xffffffffu, d_l, j - j0), dje = __shfl_sync(0xffffffffu, d_l, je - j0);
      if (n) {
        const bool seq = ci == kCatDense || (int64_t)n >= sem.crossover;
        const uint32_t colbase = (uint32_t)((rb.b0 + j) << gs) & cwmask;
        if (n <= 32u)
          ok &= reduce_chunk_wave(bcol + rowbase + ej, bval + rowbase + ej, n, dje - dj, seq, colbase, c_col, c_val,
                                  out_row + dj) == 1;
        else
          ok &= reduce_chunk_sort(bcol + rowbase + ej, bval + rowbase + ej, n, dje - dj, seq ? ~0ull : 0ull, 16,
                                  colbase, S, c_col, c_val, out_row + dj);
      }
      j = je;
    }
#ifdef MG_DIR_DEBUG
    if (!ok && (threadIdx.x & 31) == 0)
      printf("bin_reduce mismatch row %lld h %d ja %d jb %d\n", (long long)i, it.h, it.ja, it.jb);
#endif
    if (!ok && (threadIdx.x & 31) == 0) atomicOr(err, 4ull);
  }
}


// Big chunk (> kBinE elements, always the dense association): one warp per chunk.
// The chunk's columns are marked in a bitmap and ranked (word prefix + popcount);
// the products are then applied in stream order (ascending k) to a dense
// shared-memory accumulator indexed by rank, kBigD ranks per pass (as the
// reference's dense accumulator, accumulators.py:68-97).  Inside one wave the
// lanes of a repeated column are added by the lowest of them, in lane order.
// The slice streams through a ring of kBigNS shared-memory stages filled by
// asynchronous bulk copies (cp.async.bulk, completion on an mbarrier), so many
// bytes per warp are in flight without registers.  Chunks above kBigSplit
// elements are split into column parts handled by different warps.
#ifndef MG_BIG_RS
#define MG_BIG_RS 33
#endif
// waves with fewer run breaks are applied run by run, the others by match_any peer groups; 33 =
// always run by run (match_any costs more than up to 32 predicated passes: 144 -> 124 ms on cfg3)
constexpr int kBigRunSer = MG_BIG_RS;
#ifndef MG_BIG_NS
#define MG_BIG_NS 2
#endif
constexpr int kBigNS = MG_BIG_NS;          // ring stages per warp
#ifndef MG_BIG_SE
#define MG_BIG_SE 128
#endif
constexpr int kBigSE = MG_BIG_SE;          // elements per stage
constexpr int kBigSC = kBigSE * 2 + 16;    // stage bytes: columns (+ alignment slack)
constexpr int kBigSV = kBigSE * 8 + 16;    // stage bytes: values (+ alignment slack)

#ifndef MG_BIG_DW
#define MG_BIG_DW 2048
#endif
constexpr int kBigDWide = MG_BIG_DW;            // ranks per pass for chunks with more than kBigD columns

// The wide variant keeps no rank -> column table: its chunks hold more than kBigD distinct
// columns, so reading the columns back from the bitmap at emission is cheap next to the
// products, and the 2 bytes per rank buy two more warps per SM.
#ifndef MG_BIG_WIDE_INV
#define MG_BIG_WIDE_INV 0
#endif
#ifndef MG_BIG_NARROW_INV
#define MG_BIG_NARROW_INV 1
#endif
__host__ __device__ constexpr bool big_has_inv(int D) { return D <= kBigD ? MG_BIG_NARROW_INV != 0 : MG_BIG_WIDE_INV != 0; }
__host__ __device__ inline size_t bin_big_smem(int shift, int D = kBigD) {
  const size_t width = size_t(1) << shift, words = (width + 31) / 32;
  return (size_t)D * 8 + (big_has_inv(D) ? (size_t)D * 2 : 0) + ((words * 4 + 15) & ~size_t(15)) +
         ((words * 2 + 15) & ~size_t(15)) + (size_t)kBigNS * (kBigSC + kBigSV) + kBigNS * 8;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}

// one thread: expect `bytes` on bar, then issue the two bulk copies that complete them
__device__ __forceinline__ void bulk_load2(uint64_t* bar, void* d0, const void* s0, uint32_t n0, void* d1, const void* s1,
                                           uint32_t n1) {
  asm volatile(
      "{\n .reg .b64 st;\n"
      " mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "r"(n0 + n1)
      : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(d0)),
               "l"(s0), "r"(n0), "r"(smem_u32(bar))
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(d1)),
               "l"(s1), "r"(n1), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct BigStage {
  const uint16_t* c;   // columns of stage elements (offset applied)
  const double* v;
};

template <int D>
__global__ void __launch_bounds__(32)
k_bin_big(Sem sem, const BigItem* __restrict__ bigs, const unsigned long long* __restrict__ nbig,
          unsigned long long* __restrict__ ticket, int64_t cap_bigs,
          const uint32_t* __restrict__ cbm_pool, const uint16_t* __restrict__ bcol, const double* __restrict__ bval,
          uint32_t* __restrict__ c_col, double* __restrict__ c_val, unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int shift = sem.shift_num;
  const uint32_t width = 1u << shift;
  const int nwords = (int)((width + 31) / 32);
  unsigned char* sp = smem;
  double* acc = reinterpret_cast<double*>(sp); sp += (size_t)D * 8;
  unsigned char* stv0 = sp; sp += (size_t)kBigNS * kBigSV;   // 16-byte aligned (kBigD * 8 is)
  unsigned char* stc0 = sp; sp += (size_t)kBigNS * kBigSC;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sp); sp += kBigNS * 8;
  constexpr bool kInv = big_has_inv(D);
  uint16_t* inv = reinterpret_cast<uint16_t*>(sp); sp += kInv ? (size_t)D * 2 : 0;   // rank - rlo -> column
  uint32_t* bm = reinterpret_cast<uint32_t*>(sp); sp += ((size_t)nwords * 4 + 15) & ~size_t(15);
  uint16_t* pref = reinterpret_cast<uint16_t*>(sp);
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int q = 0; q < kBigNS; ++q) mbar_init(bars + q);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  uint32_t uses = 0;   // stage fills issued so far (ring position and parity)
  const uint64_t nb_front = nbig[0], nbg = nb_front + nbig[5];   // nbig[5] = back counter (cnts[7])
  // items by dynamic tickets (large-first list); the next ticket is taken while the current
  // item is reduced
  unsigned long long t_next = 0;
  if (lane == 0) t_next = atomicAdd(ticket, 1ull);
  while (true) {
    const uint64_t t = __shfl_sync(0xffffffffu, t_next, 0);
    if (t >= nbg) break;
    const BigItem it = bigs[list_slot(t, nb_front, cap_bigs)];
    if (lane == 0) t_next = atomicAdd(ticket, 1ull);
    const uint32_t n = it.n, m = it.m;
    const uint16_t* sc = bcol + it.slice;
    const double* sv = bval + it.slice;
    const int64_t out = it.out;
    const uint32_t colbase = it.colbase;
    const uint32_t parts = (uint32_t)it.kind >> 16, part = (uint32_t)it.kind & 0xffffu;
    const uint32_t plo = (uint32_t)(((uint64_t)width * part) / parts), phi = (uint32_t)(((uint64_t)width * (part + 1)) / parts);
    const uint32_t nst = (n + kBigSE - 1) / kBigSE;   // stages of one pass over the slice
    // stage j of the slice -> ring slot; copies of 16-byte aligned supersets
    auto issue = [&](uint32_t j) {
      const uint32_t slot = uses % kBigNS;
      ++uses;
      if (lane == 0) {
        const uint32_t q0 = j * kBigSE, cnt = min((uint32_t)kBigSE, n - q0);
        const uintptr_t ca = reinterpret_cast<uintptr_t>(sc + q0), va = reinterpret_cast<uintptr_t>(sv + q0);
        const uintptr_t ca0 = ca & ~uintptr_t(15), va0 = va & ~uintptr_t(15);
        const uint32_t cb = (uint32_t)(((ca + cnt * 2 - ca0) + 15) & ~uintptr_t(15));
        const uint32_t vb = (uint32_t)(((va + cnt * 8 - va0) + 15) & ~uintptr_t(15));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bulk_load2(bars + slot, stc0 + (size_t)slot * kBigSC, reinterpret_cast<const void*>(ca0), cb,
                   stv0 + (size_t)slot * kBigSV, reinterpret_cast<const void*>(va0), vb);
      }
    };
    // the first stages of the first pass do not depend on the column bitmap: issue them now
    const uint32_t u_first = uses;
    const uint32_t n_first = min(nst, (uint32_t)kBigNS);
    for (uint32_t j = 0; j < n_first; ++j) issue(j);
    auto drain_first = [&]() {   // consume the early stages when no pass runs
      for (uint32_t j = 0; j < n_first; ++j) mbar_wait(bars + (u_first + j) % kBigNS, ((u_first + j) / kBigNS) & 1u);
      __syncwarp();
    };
    // ---- columns of the chunk -> ranks (bitmap kept by the symbolic pass, else marked here)
    const uint32_t bslot = it.bslot;
    if (bslot != 0xffffffffu) {
      for (int wd = lane; wd < nwords; wd += 32) bm[wd] = __ldg(cbm_pool + (size_t)bslot * nwords + wd);
    } else {
      for (int wd = lane; wd < nwords; wd += 32) bm[wd] = 0u;
    }
    __syncwarp();
    for (uint32_t q0 = 0; bslot == 0xffffffffu && q0 < n; q0 += 32 * 8) {
      uint32_t cc[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const uint32_t q = q0 + w * 32 + lane;
        cc[w] = q < n ? (uint32_t)__ldg(sc + q) : 0xffffffffu;
      }
#pragma unroll
      for (int w = 0; w < 8; ++w)
        if (cc[w] != 0xffffffffu) atomicOr(&bm[cc[w] >> 5], 1u << (cc[w] & 31));
    }
    __syncwarp();
    if (prefix_words(bm, pref, 0, nwords) != m) {
#ifdef MG_DIR_DEBUG
      if (lane == 0) printf("bin_big mismatch out %lld n %u m %u bslot %u\n", (long long)out, n, m, bslot);
#endif
      if (lane == 0) atomicOr(err, 4ull);
      drain_first();
      continue;
    }
    const uint32_t rlo0 = plo < width ? rank_of(bm, pref, plo) : m;
    const uint32_t rhi0 = phi < width ? rank_of(bm, pref, phi) : m;
    // ---- sums, D ranks per pass
    if (rlo0 >= rhi0) drain_first();
    for (uint32_t rlo = rlo0; rlo < rhi0; rlo += D) {
      const uint32_t rhi = min(rhi0, rlo + D);
      for (uint32_t r = lane; r < rhi - rlo; r += 32) acc[r] = 0.0;
      uint32_t u0 = u_first;   // ring use index of stage 0 of this pass
      if (rlo != rlo0) {
        u0 = uses;
        for (uint32_t j = 0; j < min(nst, (uint32_t)kBigNS); ++j) issue(j);
      }
      __syncwarp();
      for (uint32_t j = 0; j < nst; ++j) {
        const uint32_t use = u0 + j, slot = use % kBigNS;
        mbar_wait(bars + slot, (use / kBigNS) & 1u);
        const uint32_t q0 = j * kBigSE, cnt = min((uint32_t)kBigSE, n - q0);
        const uint16_t* cs =
            reinterpret_cast<const uint16_t*>(stc0 + (size_t)slot * kBigSC) + ((reinterpret_cast<uintptr_t>(sc + q0) & 15) >> 1);
        const double* vs =
            reinterpret_cast<const double*>(stv0 + (size_t)slot * kBigSV) + ((reinterpret_cast<uintptr_t>(sv + q0) & 15) >> 3);
        uint32_t rr[kBigSE / 32];
#pragma unroll
        for (int w = 0; w < kBigSE / 32; ++w) {
          const uint32_t q = w * 32 + lane;
          rr[w] = q < cnt ? rank_of(bm, pref, cs[q]) : 0xffffffffu;
        }
#pragma unroll
        for (int w = 0; w < kBigSE / 32; ++w) {
          const uint32_t q = w * 32 + lane;
          const uint32_t r = rr[w];
          const bool valid = r >= rlo && r < rhi;
          const double v = valid ? vs[q] : 0.0;
          const uint32_t key = valid ? r - rlo : 0x10000u + lane;
          if (kInv && valid) inv[key] = cs[q];   // every contributor of a column writes the same value
          const uint32_t pk = __shfl_up_sync(0xffffffffu, key, 1);
          const uint32_t brk = __ballot_sync(0xffffffffu, valid && lane > 0 && key <= pk);
          if (!brk) {
            if (valid) acc[key] = __dadd_rn(acc[key], v);
          } else if (__popc(brk) < kBigRunSer) {
            // few ascending runs: apply them one after another
            const int run = __popc(brk & lanemask_le());
            const int nruns = __popc(brk) + 1;
            for (int rr2 = 0; rr2 < nruns; ++rr2) {
              if (valid && run == rr2) acc[key] = __dadd_rn(acc[key], v);
              __syncwarp();
            }
          } else {
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const uint32_t gsz = __popc(peers);
            const uint32_t maxg = __reduce_max_sync(0xffffffffu, valid ? gsz : 0u);
            const bool lead = valid && (peers & lanemask_lt()) == 0u;
            double sacc = lead ? acc[key] : 0.0;
            uint32_t rem = peers;
            for (uint32_t k = 0; k < maxg; ++k) {
              const int src = rem ? __ffs(rem) - 1 : lane;
              if (rem) rem &= rem - 1u;
              const double x = __shfl_sync(0xffffffffu, v, src);
              if (lead && k < gsz) sacc = __dadd_rn(sacc, x);
            }
            if (lead) acc[key] = sacc;
          }
          __syncwarp();
        }
        // the slot is free again: refill it with the stage kBigNS ahead
        if (j + kBigNS < nst) issue(j + kBigNS);
      }
      __syncwarp();
      if (kInv) {
        for (uint32_t r = rlo + lane; r < rhi; r += 32) {
          __stcs(c_col + out + r, colbase + (uint32_t)inv[r - rlo]);
          __stcs(c_val + out + r, acc[r - rlo]);
        }
      } else {
        // values in rank order (coalesced); columns from the bitmap: lane per word, the word's
        // ranks start at pref[word]
        for (uint32_t r = rlo + lane; r < rhi; r += 32) __stcs(c_val + out + r, acc[r - rlo]);
        for (int wd = lane; wd < nwords; wd += 32) {
          uint32_t bits = bm[wd];
          uint32_t r = pref[wd];
          if (r >= rhi || r + (uint32_t)__popc(bits) <= rlo) continue;
          while (bits) {
            const uint32_t b = (uint32_t)__ffs(bits) - 1u;
            bits &= bits - 1u;
            if (r >= rlo && r < rhi) __stcs(c_col + out + r, colbase + ((uint32_t)wd << 5) + b);
            ++r;
          }
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace mg
