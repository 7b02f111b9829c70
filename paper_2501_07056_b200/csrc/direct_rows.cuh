// Rows with a large intermediate product (> 4096 elements), numeric phase,
// "direct" path: the MAGNUS fine level (reference magnus.py:195-262, Alg. 3)
// with the chunk reorder done in shared memory instead of through a memory
// buffer.
//
// One warp owns a work item = a heavy row and a range of its numeric-plan fine
// chunks (column c in chunk c >> shift_fine, which decides the association of
// every output value).  The warp keeps, per A nonzero k of the row, a cursor
// into B row k (next position, the column there, the row end) and walks the
// item's chunks left to right, one dense window (<= 2^kDirLog columns) at a
// time.  For each window it takes the k's 32 at a time; the segment of B row k
// inside the window is [cursor, end) where `end` comes from a per-B-row window
// index (long rows) or a short probe (short rows); the segments of the 32 k's
// are concatenated into one stream -- still in ascending k, the reference's
// stable-scatter order (magnus.py:236-249) -- and loaded 32 products per wave,
// kDirU waves in flight per lane.
//
//  * dense chunk (>= crossover elements, or a Dense-category row): every
//    product is added to a shared-memory dense accumulator indexed by the
//    window-local column, in stream order (lanes of one wave that hit the same
//    column are applied in lane = stream order), i.e. sequentially from +0.0
//    in ascending k: exactly the reference's dense accumulator
//    (accumulators.py:68-97).  The touched columns (bitmap) are emitted in
//    ascending order with coalesced stores and the accumulator is re-zeroed.
//  * sort chunk (< crossover elements): the chunk's stream is gathered into a
//    shared-memory list and reduced by the binned path's sort reducer
//    (x0 + pairwise(rest), accumulators.py:113-129).
//
// Compared with the binned path there is no reorder buffer: a product costs its
// B element (12 B, mostly L2) and one shared-memory update, not 20 B of HBM
// round trip.  Requires chunk width <= 2^kDirMaxShift, crossover <= kDirList and
// fewer than 2^32 columns.
#pragma once
#include "binned_rows.cuh"
#include "common.cuh"

namespace mg {

#ifndef MG_DIR_LOG
#define MG_DIR_LOG 11
#endif
#ifndef MG_DIR_NW
#define MG_DIR_NW 1
#endif
#ifndef MG_DIR_U
#define MG_DIR_U 4
#endif
#ifndef MG_DIR_ITEM
#define MG_DIR_ITEM (1 << 18)
#endif
constexpr int kDirLog = MG_DIR_LOG;          // dense window: at most 2^kDirLog columns
constexpr int kDirW = 1 << kDirLog;
constexpr int kDirWords = kDirW / 32;
constexpr int kDirList = 512;                // list window capacity (crossover <= kDirList)
constexpr int kDirMaxShift = 14;             // chunk width <= 2^14 (u16 chunk-local columns)
constexpr int kDirNW = MG_DIR_NW;            // warps per CTA (independent work items)
constexpr int kDirU = MG_DIR_U;              // waves of loads in flight per lane
#ifndef MG_DIR_G
#define MG_DIR_G 8
#endif
constexpr int kDirG = MG_DIR_G;              // groups of 32 k's whose cursors are loaded together
constexpr int kDirSeg = 32 * kDirG;
constexpr int64_t kDirItem = MG_DIR_ITEM;    // products per work item (rows above are cut by chunks)
constexpr int64_t kDirIdxMinLen = 128;       // shortest B row given a window index
constexpr uint32_t kDirNone = 0xffffffffu;   // cursor: B row exhausted

#ifdef MG_DIR_DEBUG
#define DIR_CHECK(cond, ...)                                  \
  do {                                                       \
    if (!(cond)) {                                           \
      printf("dir check failed line %d: ", __LINE__);        \
      printf(__VA_ARGS__);                                   \
      printf("\n");                                          \
      asm volatile("trap;");                                 \
    }                                                        \
  } while (0)
#else
#define DIR_CHECK(cond, ...) do { } while (0)
#endif

struct DirItem {   // chunks [ja, jb) of heavy row h; whole: the item starts at the row's first chunk
  int32_t h, ja, jb, whole;
};

// shared-memory layout of one warp.  The sort-chunk scratch (gathered list + the sort
// reducer's ReduceSmem) overlays the dense accumulator, which is idle during a sort
// chunk; the touched bytes are re-zeroed afterwards.
struct DirSmem {
  static constexpr size_t kAcc = (size_t)kDirW * 8;
  static constexpr size_t kBm = ((size_t)kDirWords * 4 + 15) & ~size_t(15);
  static constexpr size_t kPref = ((size_t)(kDirWords + 1) * 2 + 15) & ~size_t(15);
  static constexpr size_t kSegOff = (size_t)kDirSeg * 4;   // segment table of one k super-group
  static constexpr size_t kSegPos = (size_t)kDirSeg * 4;
  static constexpr size_t kSegAv = (size_t)kDirSeg * 8;
  static constexpr size_t kWarp = kAcc + kBm + kPref + kSegOff + kSegPos + kSegAv;
  // overlay (byte offsets inside acc)
  static constexpr size_t oLVal = 0, oSVal = oLVal + kDirList * 8, oLCol = oSVal + kDirList * 8,
                          oStc = oLCol + kDirList * 2, oInv = oStc + kDirList * 2, oCnt = oInv + kDirList * 2,
                          oRBm = oCnt + kDirList * 2, oRPref = oRBm + (size_t(1) << (kDirMaxShift - 5)) * 4,
                          oEnd = oRPref + (size_t(1) << (kDirMaxShift - 5)) * 2;
  static_assert(oEnd <= kAcc, "list scratch fits in the dense accumulator (kDirLog >= 11)");
  static_assert(kWarp % 16 == 0, "16-byte aligned warp slices");
};

// ---------------------------------------------------------------- B window index
// Histogram of floor(log2(row length)) over B's rows (chooses the index threshold).
__global__ void k_didx_hist(DevCsr B, unsigned long long* __restrict__ hist) {
  __shared__ unsigned long long sh[40];
  if (threadIdx.x < 40) sh[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < B.n_rows; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = B.rp(k + 1) - B.rp(k);
    if (len > 0) atomicAdd(&sh[63 - __clzll((unsigned long long)len)], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < 40 && sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

// slot[k] = index slot of B row k (rows with >= min_len entries), else -1
__global__ void k_didx_slots(DevCsr B, int64_t min_len, int32_t* __restrict__ slot, unsigned long long* __restrict__ count) {
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x; k0 < B.n_rows; k0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = k0 + threadIdx.x;
    const bool has = k < B.n_rows && B.rp(k + 1) - B.rp(k) >= min_len;
    const uint32_t m = __ballot_sync(0xffffffffu, has);
    unsigned long long b = 0;
    if ((threadIdx.x & 31) == 0 && m) b = atomicAdd(count, (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (k < B.n_rows) slot[k] = has ? (int32_t)(b + __popc(m & lanemask_lt())) : -1;
  }
}

// Window index of an indexed B row: entry g = first position p of the row with
// col[p] >= g << wlog (the row end if none), nwin1 entries per row.  Warp per row.
__global__ void k_didx_fill(DevCsr B, const int32_t* __restrict__ slot, int wlog, int64_t nwin1, uint32_t* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = warp; k < B.n_rows; k += nwarps) {
    const int32_t s = __ldg(slot + k);
    if (s < 0) continue;
    const uint32_t b0 = (uint32_t)B.rp(k), b1 = (uint32_t)B.rp(k + 1);
    uint32_t* out = idx + (size_t)s * nwin1;
    // entries (window of col[p-1], window of col[p]] point at p
    for (uint32_t p = b0 + lane; p < b1; p += 32) {
      const int64_t w = (int64_t)(__ldg(B.col + p) >> wlog);
      const int64_t wp = p == b0 ? -1 : (int64_t)(__ldg(B.col + p - 1) >> wlog);
      for (int64_t g = wp + 1; g <= w; ++g) out[g] = p;
    }
    const int64_t wl = (int64_t)(__ldg(B.col + b1 - 1) >> wlog);
    for (int64_t g = wl + 1 + lane; g < nwin1; g += 32) out[g] = b1;
  }
}

// ---------------------------------------------------------------- plan
// Work items of heavy rows [0, nH): chunk ranges of about kDirItem products (cut where
// the row's product prefix crosses a multiple of `item`).  Large items first.
__global__ void k_dir_plan(const int32_t* __restrict__ rows, int64_t nH, const int64_t* __restrict__ mn,
                           const int64_t* __restrict__ mx, int shift, const int64_t* __restrict__ choff,
                           const uint32_t* __restrict__ ce, int64_t item, DirItem* __restrict__ items,
                           unsigned long long* __restrict__ cnt, int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = warp; h < nH; h += nwarps) {
    const int64_t i = rows[h];
    const RowBins rb = row_bins(mn[i], mx[i], shift);   // shift <= kDirMaxShift: entries == chunks
    const uint32_t* e = ce + choff[h];
    int start = 0;
    for (int q0 = 0; q0 < rb.nb; q0 += 32) {
      const int j = q0 + lane;
      const bool valid = j < rb.nb;
      const uint32_t pe = valid ? __ldg(e + j) : 0u, pi = valid ? __ldg(e + j + 1) : 0u;
      const bool cut = valid && (j == rb.nb - 1 || (int64_t)pe / item != (int64_t)pi / item);
      const uint32_t cm = __ballot_sync(0xffffffffu, cut);
      const uint32_t prev = cm & lanemask_lt();
      const int s = prev ? q0 + 31 - __clz(prev) + 1 : start;
      const uint32_t n = cut ? pi - __ldg(e + s) : 0u;
      const DirItem it{(int32_t)h, s, j + 1, s == 0 ? 1 : 0};
      emit_items(cut && n > 0 && (int64_t)n * 2 >= item, *reinterpret_cast<const BinItem*>(&it),
                 reinterpret_cast<BinItem*>(items), cnt);
      emit_items(cut && n > 0 && (int64_t)n * 2 < item, *reinterpret_cast<const BinItem*>(&it),
                 reinterpret_cast<BinItem*>(items), cnt + 1, cap);
      if (cm) start = q0 + 31 - __clz(cm) + 1;
    }
  }
}

// ---------------------------------------------------------------- numeric
__device__ __forceinline__ uint32_t select_bit(uint32_t x, uint32_t k) {   // position of the k-th set bit
  uint32_t pos = 0, c;
  c = __popc(x & 0xffffu); if (k >= c) { k -= c; x >>= 16; pos += 16; }
  c = __popc(x & 0xffu);   if (k >= c) { k -= c; x >>= 8; pos += 8; }
  c = __popc(x & 0xfu);    if (k >= c) { k -= c; x >>= 4; pos += 4; }
  c = __popc(x & 0x3u);    if (k >= c) { k -= c; x >>= 2; pos += 2; }
  if (k >= (x & 1u)) pos += 1;
  return pos;
}

// first p in (pos, lim] with col[p] >= hi (col[pos] < hi)
__device__ __forceinline__ uint32_t seg_end_probe(const uint32_t* __restrict__ col, uint32_t pos, uint32_t lim, uint32_t hi) {
  uint32_t p = pos + 1;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    if (p >= lim || __ldg(col + p) >= hi) return p;
    ++p;
  }
  return lower_bound_col(col, p, lim, hi);
}

struct DirState {   // per-k cursors of the current item (per-warp global scratch)
  unsigned long long* pn;   // (column at the cursor << 32) | cursor position; column kDirNone: exhausted
  unsigned long long* ls;   // ((uint32)window-index slot << 32) | B row end; slot 0xffffffff: none
};

__device__ __forceinline__ unsigned long long pack_pn(uint32_t pos, uint32_t nxt) {
  return ((unsigned long long)nxt << 32) | pos;
}

// One pass over the columns below hi (window or chunk end; hi_all: no bound) for every k
// of the row, in ascending k.  The k's are taken kDirSeg at a time: their cursors are
// loaded together, the segment ends looked up together, and the segments concatenated
// into one stream loaded kDirU waves at a time, so many loads are in flight per lane.
// Dense: products added to acc/bm (window-local column c & wmask); else appended to the
// list (column c - lbase).  Returns the number of products, advances the
// cursors and sets *nmin = the smallest column any k has left.
template <bool Dense>
__device__ __forceinline__ uint32_t dir_pass(const DevCsr& A, const DevCsr& B, int64_t a0, int nk, const DirState& st,
                                             const uint32_t* __restrict__ bidx, int64_t nwin1, int wlog, uint32_t hi,
                                             bool hi_all, double* acc, uint32_t* bm, uint32_t wmask, uint16_t* lcol,
                                             double* lval, uint32_t lbase, uint32_t* seg_off, uint32_t* seg_pos,
                                             double* seg_av, uint32_t* nmin) {
  const int lane = threadIdx.x & 31;
  uint32_t total = 0, mn_next = kDirNone;
  for (int s0 = 0; s0 < nk; s0 += kDirSeg) {
    unsigned long long pn[kDirG];
    uint32_t actm = 0;
#pragma unroll
    for (int g = 0; g < kDirG; ++g) {
      const int j = s0 + g * 32 + lane;
      pn[g] = j < nk ? st.pn[j] : pack_pn(0, kDirNone);
      const uint32_t nx = (uint32_t)(pn[g] >> 32);
      if (nx != kDirNone && (hi_all || nx < hi)) actm |= 1u << g;
    }
    if (!__any_sync(0xffffffffu, actm != 0)) {
#pragma unroll
      for (int g = 0; g < kDirG; ++g) mn_next = min(mn_next, (uint32_t)(pn[g] >> 32));
      continue;
    }
    unsigned long long ls[kDirG];
    double av[kDirG];
#pragma unroll
    for (int g = 0; g < kDirG; ++g) {
      const int j = s0 + g * 32 + lane;
      ls[g] = 0;
      av[g] = 0.0;
      if ((actm >> g) & 1u) {
        ls[g] = st.ls[j];
        av[g] = __ldg(A.val + a0 + j);
      }
    }
    uint32_t e[kDirG];
#pragma unroll
    for (int g = 0; g < kDirG; ++g) {
      const uint32_t pos = (uint32_t)pn[g];
      e[g] = pos;
      if ((actm >> g) & 1u) {
        const uint32_t lim = (uint32_t)ls[g], sl = (uint32_t)(ls[g] >> 32);
        if (hi_all) e[g] = lim;
        else if (sl != kDirNone) e[g] = __ldg(bidx + (size_t)sl * nwin1 + (hi >> wlog));
        else e[g] = seg_end_probe(B.col, pos, lim, hi);
        DIR_CHECK(e[g] > pos && e[g] <= lim, "seg pos %u e %u lim %u hi %u sl %u", pos, e[g], lim, hi, sl);
      }
    }
    // segment table of the super-group (ascending k)
    uint32_t base = 0;
#pragma unroll
    for (int g = 0; g < kDirG; ++g) {
      const uint32_t pos = (uint32_t)pn[g];
      const uint32_t len = e[g] - pos;
      const uint32_t inc = warp_incl_scan(len);
      seg_off[g * 32 + lane] = base + inc - len;
      seg_pos[g * 32 + lane] = pos;
      seg_av[g * 32 + lane] = av[g];
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
    const uint32_t T = base;
    // next columns of the advanced cursors (independent of the stream)
    uint32_t nnx[kDirG];
#pragma unroll
    for (int g = 0; g < kDirG; ++g) {
      nnx[g] = (uint32_t)(pn[g] >> 32);
      if ((actm >> g) & 1u) nnx[g] = e[g] < (uint32_t)ls[g] ? __ldg(B.col + e[g]) : kDirNone;
    }
    __syncwarp();
    for (uint32_t q0 = 0; q0 < T; q0 += 32 * kDirU) {
      uint32_t c[kDirU];
      double v[kDirU];
#pragma unroll
      for (int w = 0; w < kDirU; ++w) {
        const uint32_t q = q0 + w * 32 + lane;
        c[w] = kDirNone;
        v[w] = 0.0;
        if (q < T) {
          // segment of stream position q: last entry with seg_off <= q (empty segments share
          // their offset with the next entry, so the search lands on a non-empty one)
          int lo = 0;
#pragma unroll
          for (int st2 = kDirSeg / 2; st2 > 0; st2 >>= 1)
            if (seg_off[lo + st2] <= q) lo += st2;
          const uint32_t pp = seg_pos[lo] + (q - seg_off[lo]);
          DIR_CHECK(pp < (uint32_t)B.nnz, "pp %u q %u T %u lo %d", pp, q, T, lo);
          c[w] = __ldg(B.col + pp);
          v[w] = __dmul_rn(seg_av[lo], __ldg(B.val + pp));
        }
      }
#pragma unroll
      for (int w = 0; w < kDirU; ++w) {
        if (q0 + w * 32 >= T) break;
        const bool valid = c[w] != kDirNone;
        DIR_CHECK(!valid || hi_all || c[w] < hi, "col %u hi %u", c[w], hi);
        if (Dense) {
          const uint32_t key = valid ? (c[w] & wmask) : 0x10000u + lane;
          const uint32_t pk = __shfl_up_sync(0xffffffffu, key, 1);
          const uint32_t brk = __ballot_sync(0xffffffffu, valid && lane > 0 && key <= pk);
          if (!brk) {
            if (valid) {
              acc[key] = __dadd_rn(acc[key], v[w]);
              atomicOr(&bm[key >> 5], 1u << (key & 31));
            }
          } else {
            // same column in several lanes: apply in lane (= stream) order
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const uint32_t before = __popc(peers & lanemask_lt());
            const uint32_t rounds = __reduce_max_sync(0xffffffffu, valid ? before : 0u);
            for (uint32_t r = 0; r <= rounds; ++r) {
              if (valid && before == r) acc[key] = __dadd_rn(acc[key], v[w]);
              __syncwarp();
            }
            if (valid && before == 0) atomicOr(&bm[key >> 5], 1u << (key & 31));
          }
        } else {
          const uint32_t q = total + q0 + w * 32 + lane;   // position in the chunk's stream
          if (valid && q < (uint32_t)kDirList) {
            lcol[q] = (uint16_t)(c[w] - lbase);
            lval[q] = v[w];
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int g = 0; g < kDirG; ++g) {
      const int j = s0 + g * 32 + lane;
      if ((actm >> g) & 1u) st.pn[j] = pack_pn(e[g], nnx[g]);
      mn_next = min(mn_next, nnx[g]);
    }
    total += T;
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn_next = min(mn_next, __shfl_xor_sync(0xffffffffu, mn_next, o));
  *nmin = mn_next;
  return total;
}

// Emit the touched columns of a dense window in ascending order (coalesced), re-zero it.
__device__ __forceinline__ uint32_t dir_emit(double* acc, uint32_t* bm, uint16_t* pref, int nwd, uint32_t colbase,
                                             int64_t out, uint32_t* __restrict__ c_col, double* __restrict__ c_val) {
  const int lane = threadIdx.x & 31;
  const int per = (nwd + 31) >> 5;
  const int w0 = min(nwd, lane * per), w1 = min(nwd, w0 + per);
  uint32_t s = 0;
  for (int w = w0; w < w1; ++w) s += __popc(bm[w]);
  const uint32_t inc = warp_incl_scan(s);
  uint32_t run = inc - s;
  for (int w = w0; w < w1; ++w) {
    pref[w] = (uint16_t)run;
    run += __popc(bm[w]);
  }
  const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
  __syncwarp();
  for (uint32_t r = lane; r < total; r += 32) {
    int lo = 0, hi = nwd;   // pref[lo] <= r < pref[hi] (pref[nwd] = total)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((uint32_t)pref[mid] <= r) lo = mid; else hi = mid;
    }
    const uint32_t cl = (uint32_t)lo * 32u + select_bit(bm[lo], r - pref[lo]);
    DIR_CHECK(cl < (uint32_t)nwd * 32u, "emit cl %u nwd %d r %u total %u", cl, nwd, r, total);
    c_col[out + r] = colbase + cl;
    c_val[out + r] = acc[cl];
    acc[cl] = 0.0;
  }
  __syncwarp();
  for (int w = lane; w < nwd; w += 32) bm[w] = 0u;
  __syncwarp();
  return total;
}

// zero bytes [lo, hi) of the accumulator region (rounded out to 8-byte words)
__device__ __forceinline__ void dir_zero(double* acc, size_t lo, size_t hi) {
  for (size_t w = (lo >> 3) + (threadIdx.x & 31); w < ((hi + 7) >> 3); w += 32) acc[w] = 0.0;
}

__global__ void __launch_bounds__(32 * kDirNW)
k_dir_num(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, const int8_t* __restrict__ cat,
          const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, Sem sem, int wlog,
          const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce, const uint32_t* __restrict__ cd,
          const DirItem* __restrict__ items, const unsigned long long* __restrict__ nitems,
          unsigned long long* __restrict__ ticket, int64_t cap_items, const int32_t* __restrict__ bslot,
          const uint32_t* __restrict__ bidx, int64_t nwin1, unsigned long long* __restrict__ kst, int64_t kst_stride,
          const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col, double* __restrict__ c_val,
          unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* sp = smem + (size_t)wib * DirSmem::kWarp;
  unsigned char* accb = sp;
  double* acc = reinterpret_cast<double*>(sp); sp += DirSmem::kAcc;
  uint32_t* bm = reinterpret_cast<uint32_t*>(sp); sp += DirSmem::kBm;
  uint16_t* pref = reinterpret_cast<uint16_t*>(sp); sp += DirSmem::kPref;
  uint32_t* seg_off = reinterpret_cast<uint32_t*>(sp); sp += DirSmem::kSegOff;
  uint32_t* seg_pos = reinterpret_cast<uint32_t*>(sp); sp += DirSmem::kSegPos;
  double* seg_av = reinterpret_cast<double*>(sp);
  // sort-chunk scratch, overlaid on acc
  double* lval = reinterpret_cast<double*>(accb + DirSmem::oLVal);
  uint16_t* lcol = reinterpret_cast<uint16_t*>(accb + DirSmem::oLCol);
  ReduceSmem S;
  S.bm = reinterpret_cast<uint32_t*>(accb + DirSmem::oRBm);
  S.pref = reinterpret_cast<uint16_t*>(accb + DirSmem::oRPref);
  S.cnt = reinterpret_cast<uint32_t*>(accb + DirSmem::oCnt);
  S.sval = reinterpret_cast<double*>(accb + DirSmem::oSVal);
  S.stc = reinterpret_cast<uint16_t*>(accb + DirSmem::oStc);
  S.inv = reinterpret_cast<uint16_t*>(accb + DirSmem::oInv);
  const int shift = sem.shift_num;
  const uint32_t W = 1u << wlog, wmask = W - 1u;
  const int nwd = (int)max(1u, W >> 5);
  for (uint32_t r = lane; r < (uint32_t)kDirW; r += 32) acc[r] = 0.0;
  for (int w = lane; w < nwd; w += 32) bm[w] = 0u;
  __syncwarp();
  DirState st;
  st.pn = kst + ((size_t)blockIdx.x * kDirNW + wib) * (size_t)kst_stride * 2;
  st.ls = st.pn + kst_stride;
  const uint64_t n_front = nitems[0], n_all = n_front + nitems[1];
  const uint64_t ncols = (uint64_t)B.n_cols;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_all) break;
    DIR_CHECK(list_slot(t, n_front, cap_items) >= 0 && list_slot(t, n_front, cap_items) < cap_items, "item slot");
    const DirItem it = items[list_slot(t, n_front, cap_items)];
    const int64_t i = rows[it.h];
    const int64_t a0 = A.rp(i);
    const int nk = (int)(A.rp(i + 1) - a0);
    DIR_CHECK(it.ja >= 0 && it.jb > it.ja && nk <= kst_stride, "item %d %d %d nk %d", it.h, it.ja, it.jb, nk);
    const int64_t rmn = mn[i], rmx = mx[i];
    const RowBins rb = row_bins(rmn, rmx, shift);
    const uint32_t* e = ce + choff[it.h];
    const uint32_t* d = cd + choff[it.h];
    const int ci = cat[i];
    const int64_t cstart = max(rmn, (rb.c0 + it.ja) << shift);
    // cursors at the item's first column
    uint32_t nmin = kDirNone;
    for (int j = lane; j < nk; j += 32) {
      const int64_t k = __ldg(A.col + a0 + j);
      const uint32_t b0 = (uint32_t)B.rp(k), b1 = (uint32_t)B.rp(k + 1);
      const int32_t sl = __ldg(bslot + k);
      uint32_t p = b0;
      if (!it.whole)
        p = sl >= 0 ? __ldg(bidx + (size_t)sl * nwin1 + (cstart >> wlog)) : lower_bound_col(B.col, b0, b1, (uint32_t)cstart);
      DIR_CHECK(p >= b0 && p <= b1, "init p %u b0 %u b1 %u sl %d cstart %lld", p, b0, b1, sl, (long long)cstart);
      const uint32_t nx = p < b1 ? __ldg(B.col + p) : kDirNone;
      st.pn[j] = pack_pn(p, nx);
      st.ls[j] = ((unsigned long long)(uint32_t)sl << 32) | b1;
      nmin = min(nmin, nx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmin = min(nmin, __shfl_xor_sync(0xffffffffu, nmin, o));
    __syncwarp();
    int64_t out = c_rp[i] + __ldg(d + it.ja);
    bool ok = true;
    // chunk table of the item, 32 entries at a time: products n_j and distinct columns m_j
    int b0 = -1 << 30;
    uint32_t n_l = 0, m_l = 0;
    auto load_batch = [&](int j) {
      b0 = j;
      const int jj = j + lane;
      n_l = jj < it.jb ? __ldg(e + jj + 1) - __ldg(e + jj) : 0u;
      m_l = jj < it.jb ? __ldg(d + jj + 1) - __ldg(d + jj) : 0u;
    };
    auto chunk_nm = [&](int j, uint32_t& n, uint32_t& m) {
      if (j < b0 || j >= b0 + 32) load_batch(j);
      n = __shfl_sync(0xffffffffu, n_l, j - b0);
      m = __shfl_sync(0xffffffffu, m_l, j - b0);
    };
    int cj = it.ja;
    while (cj < it.jb) {
      uint32_t n, m;
      chunk_nm(cj, n, m);
      if (n == 0) { ++cj; continue; }
      const int64_t chunk_lo = (rb.c0 + cj) << shift;
      if (n > (uint32_t)kDirList) {
        // big chunk (more than kDirList >= crossover products: the dense association), applied
        // straight into the dense accumulator, W columns at a time
        const int64_t chunk_hi = chunk_lo + ((int64_t)1 << shift);
        uint32_t got = 0, cnt = 0;
        int64_t wlo = max(chunk_lo, (int64_t)(nmin & ~wmask));
        while (wlo < chunk_hi && nmin != kDirNone) {
          const int64_t whi = wlo + W;
          const bool hi_all = (uint64_t)whi >= ncols;
          cnt += dir_pass<true>(A, B, a0, nk, st, bidx, nwin1, wlog, hi_all ? 0u : (uint32_t)whi, hi_all, acc, bm, wmask,
                                lcol, lval, 0u, seg_off, seg_pos, seg_av, &nmin);
          DIR_CHECK(out + got <= c_rp[i + 1], "emit out %lld got %u end %lld", (long long)out, got, (long long)c_rp[i + 1]);
          got += dir_emit(acc, bm, pref, nwd, (uint32_t)wlo, out + got, c_col, c_val);
          wlo = max(whi, (int64_t)(nmin & ~wmask));
        }
#ifdef MG_DIR_DEBUG
        if ((got != m || cnt != n) && lane == 0)
          printf("dense mismatch row %lld cj %d ja %d jb %d n %u cnt %u m %u got %u nmin %u whole %d\n", (long long)i, cj,
                 it.ja, it.jb, n, cnt, m, got, nmin, it.whole);
#endif
        ok &= got == m && cnt == n;
        out += got;
        ++cj;
        continue;
      }
      // list window: a run of small chunks (<= kDirList products in all, <= 2^kDirMaxShift
      // columns, <= 64 chunks) gathered in one pass and reduced by a stable counting sort;
      // each column gets its chunk's association (dense if the chunk holds >= crossover)
      uint64_t seqmask = 0;
      uint32_t ntot = 0, mtot = 0;
      int cj2 = cj;
      while (cj2 < it.jb && cj2 - cj < 64) {
        uint32_t n2, m2;
        chunk_nm(cj2, n2, m2);
        if (n2 > (uint32_t)kDirList || ntot + n2 > (uint32_t)kDirList) break;
        if ((((int64_t)(cj2 + 1 - cj)) << shift) > ((int64_t)1 << kDirMaxShift)) break;
        if (ci == kCatDense || (int64_t)n2 >= sem.crossover) seqmask |= 1ull << (cj2 - cj);
        ntot += n2;
        mtot += m2;
        ++cj2;
      }
      const int64_t whi = (rb.c0 + cj2) << shift;
      const bool hi_all = (uint64_t)whi >= ncols;
      const uint32_t cnt = dir_pass<false>(A, B, a0, nk, st, bidx, nwin1, wlog, hi_all ? 0u : (uint32_t)whi, hi_all, acc,
                                           bm, wmask, lcol, lval, (uint32_t)chunk_lo, seg_off, seg_pos, seg_av, &nmin);
      __syncwarp();
#ifdef MG_DIR_DEBUG
      if (cnt != ntot && lane == 0)
        printf("list mismatch row %lld cj %d..%d n %u cnt %u m %u whole %d\n", (long long)i, cj, cj2, ntot, cnt, mtot,
               it.whole);
#endif
      if (cnt != ntot) {
        ok = false;
      } else {
        ok &= reduce_chunk_sort<false>(lcol, lval, ntot, mtot, seqmask, shift, (uint32_t)chunk_lo, S, c_col, c_val, out);
      }
      // re-zero the overlay bytes the list window touched
      dir_zero(acc, DirSmem::oLVal, DirSmem::oLVal + (size_t)ntot * 8);
      dir_zero(acc, DirSmem::oSVal, DirSmem::oSVal + (size_t)ntot * 8);
      dir_zero(acc, DirSmem::oLCol, DirSmem::oCnt + (size_t)(mtot + 1) / 2 * 4);   // lcol, stc, inv, cnt
      const size_t words = (size_t)((((int64_t)(cj2 - cj)) << shift) + 31) >> 5;
      dir_zero(acc, DirSmem::oRBm, DirSmem::oRBm + words * 4);
      dir_zero(acc, DirSmem::oRPref, DirSmem::oRPref + words * 2);
      __syncwarp();
      out += mtot;
      cj = cj2;
    }
    if (!ok && lane == 0) atomicOr(err, 8ull);
    __syncwarp();
  }
}

}  // namespace mg
