// Coarse level (Alg. 4) on the device, for the rows the planner puts in the Coarse category
// (reference magnus.py:317-406 build_coarse_chunks / coarse_level_batch, matrix.py:153-184
// csr_rows_to_csc).
//
// Per batch of coarse rows the reference builds the CSC view of the batch's rows of A, walks
// the referenced B rows once each (outer product: every B row is multiplied with all the A
// entries of its column), places every product in its (row, coarse chunk) bucket through a
// histogram + row-linked prefix sum + stable scatter, and then runs the fine level on each
// bucket.  Here:
//
//   k_c4_rows      the batch's coarse rows, their A nonzeros numbered, CSC column counts
//   (scan)         CSC column pointers
//   k_c4_fill      CSC entries (row, numbered A nonzero, value) per referenced B row
//   k_c4_koff      per (A nonzero, coarse chunk): products of the same row and chunk that come
//                  from smaller k -- the stable position of the nonzero's segment inside the
//                  bucket (the reference's running `heads`, magnus.py:352-366, in closed form);
//                  the bucket sizes are the symbolic pass's chunk-table differences, and the
//                  row-linked offsets are the reorder-buffer layout itself (bucket (r, c) sits at
//                  rowbase[r] + ce[r][first fine chunk of c])
//   k_c4_scatter   one CTA per (referenced B row, 256 CSC entries of its column): the row is staged tile by tile in shared memory
//                  with bulk async copies (TMA, 16-byte aligned supersets) and reused by every
//                  CSC entry of its column; products go to the coarse buffer (coarse-chunk-local
//                  column, a * b) in bucket order = ascending k (Gustavson order per row)
//   k_c4_fine      fine level per bucket (magnus.py:195-262 via fine_level_chunk): the bucket is
//                  read in order and stably scattered by fine chunk into the reorder buffer the
//                  chunk reducers (k_bin_big / k_bin_reduce) consume
//
// The slices end up exactly as k_bin_expand2 leaves them (same stable order), so the values
// are the reference's bits; tests run both paths.
#pragma once
#include "binned_rows.cuh"
#include "symbolic_rows.cuh"

namespace mg {

constexpr int kC4T = 256;           // threads per CTA of the scatter / fine kernels
constexpr int kC4Tile = 1024;       // B row elements staged per tile
constexpr int kC4MaxCoarse = 1024;  // coarse chunks (boundary table in shared memory)
constexpr int kC4MaxFineLog = 12;   // fine chunks per coarse chunk <= 2^12 (cursor table per warp)

struct C4Geom {
  int sf, sc;     // fine / coarse shifts (sc >= sf)
  int ncc;        // coarse chunks over the planned span
  int64_t h0;     // first heavy row of the batch
};

// The batch's coarse heavy rows: list, first numbered A nonzero of each, CSC column counts.
__global__ void k_c4_rows(DevCsr A, const int32_t* __restrict__ rows, const int8_t* __restrict__ cat, int64_t h0,
                          int64_t h1, int32_t* __restrict__ list, int64_t* __restrict__ apos,
                          unsigned long long* __restrict__ cnt, int64_t* __restrict__ colcnt) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t h = h0 + warp; h < h1; h += nwarps) {
    const int64_t i = rows[h];
    apos[h - h0] = -1;
    if (cat[i] != kCatCoarse) continue;
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    unsigned long long ap = 0;
    if (lane == 0) {
      list[atomicAdd(cnt, 1ull)] = (int32_t)h;
      ap = atomicAdd(cnt + 1, (unsigned long long)(a1 - a0));
      apos[h - h0] = (int64_t)ap;
    }
    for (int64_t p = a0 + lane; p < a1; p += 32)
      atomicAdd(reinterpret_cast<unsigned long long*>(colcnt) + __ldg(A.col + p), 1ull);
  }
}

// csr_rows_to_csc (matrix.py:153-184): entries of column k at [colptr[k], colptr[k+1]).
__global__ void k_c4_fill(DevCsr A, const int32_t* __restrict__ rows, const int32_t* __restrict__ list, int64_t nlist,
                          const int64_t* __restrict__ apos, int64_t h0, const int64_t* __restrict__ colptr,
                          unsigned long long* __restrict__ colcur, int32_t* __restrict__ csc_h,
                          uint32_t* __restrict__ csc_q, double* __restrict__ csc_a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w < nlist; w += nwarps) {
    const int32_t h = list[w];
    const int64_t i = rows[h];
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1), ap = apos[h - h0];
    for (int64_t p = a0 + lane; p < a1; p += 32) {
      const int64_t k = __ldg(A.col + p);
      const int64_t slot = colptr[k] + (int64_t)atomicAdd(colcur + k, 1ull);
      csc_h[slot] = h;
      csc_q[slot] = (uint32_t)(ap + (p - a0));
      csc_a[slot] = __ldg(A.val + p);
    }
  }
}

// Stable position of every A nonzero's segment inside its row's coarse buckets, and the check
// that the buckets have the sizes the symbolic pass counted.  One warp per coarse row: 32 k's at
// a time, every lane walks its B row once from coarse chunk to coarse chunk (window index for
// indexed rows, a cursor for the others); run[] (shared memory, one counter per coarse chunk)
// carries the products of the k's already seen.
__global__ void __launch_bounds__(256)
k_c4_koff(DevCsr A, DevCsr B, const int32_t* __restrict__ rows, const int32_t* __restrict__ list, int64_t nlist,
          const int64_t* __restrict__ apos, C4Geom g, const int64_t* __restrict__ mn, const int64_t* __restrict__ mx,
          const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce, const int32_t* __restrict__ bslot,
          const uint32_t* __restrict__ bidx, int64_t nwin1, int ilog, uint32_t* __restrict__ koff,
          unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  uint32_t* run = reinterpret_cast<uint32_t*>(smem) + (size_t)(threadIdx.x >> 5) * g.ncc;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int csl = g.sc - g.sf;
  for (int64_t w = warp; w < nlist; w += nwarps) {
    const int32_t h = list[w];
    const int64_t i = rows[h];
    const int64_t a0 = A.rp(i), ap = apos[h - g.h0];
    const int nk = (int)(A.rp(i + 1) - a0);
    const RowBins rb = row_bins(mn[i], mx[i], g.sf);
    const uint32_t* e = ce + choff[h];
    const int64_t cc0 = mn[i] >> g.sc, cc1 = mx[i] >> g.sc;
    for (int64_t cc = cc0 + lane; cc <= cc1; cc += 32) run[cc] = 0u;
    __syncwarp();
    for (int j0 = 0; j0 < nk; j0 += 32) {
      const int j = j0 + lane;
      uint32_t pos = 0, b1 = 0;
      const uint32_t* ix = nullptr;
      if (j < nk) {
        const int64_t k = __ldg(A.col + a0 + j);
        pos = (uint32_t)B.rp(k);
        b1 = (uint32_t)B.rp(k + 1);
        const int32_t sl = bslot != nullptr ? __ldg(bslot + k) : -1;
        if (sl >= 0) {
          ix = bidx + (size_t)sl * nwin1;
          pos = __ldg(ix + min((int64_t)((cc0 << g.sc) >> ilog), nwin1 - 1));
        } else {
          pos = lower_bound_col(B.col, pos, b1, (uint32_t)(cc0 << g.sc));
        }
      }
      for (int64_t cc = cc0; cc <= cc1; ++cc) {
        const int64_t hi64 = (cc + 1) << g.sc;
        uint32_t nxt = pos;
        if (j < nk) {
          if (hi64 >= ((int64_t)1 << 32)) {
            nxt = b1;
          } else if (ix != nullptr) {
            nxt = __ldg(ix + min(hi64 >> ilog, nwin1 - 1));
          } else {
            while (nxt < b1 && __ldg(B.col + nxt) < (uint32_t)hi64) ++nxt;
          }
        }
        const uint32_t len = nxt - pos;
        pos = nxt;
        const uint32_t inc = warp_incl_scan(len);
        const uint32_t base = run[cc];
        if (j < nk) koff[(size_t)(ap + j) * g.ncc + cc] = base + inc - len;
        __syncwarp();
        if (lane == 31) run[cc] = base + inc;
        __syncwarp();
      }
    }
    // bucket sizes against the symbolic chunk tables
    for (int64_t cc = cc0 + lane; cc <= cc1; cc += 32) {
      const int64_t jl = max((int64_t)0, (cc << csl) - rb.c0), jh = min((int64_t)rb.nchunk, ((cc + 1) << csl) - rb.c0);
      if (run[cc] != __ldg(e + jh) - __ldg(e + jl)) atomicOr(err, 4ull);
    }
    __syncwarp();
  }
}

struct C4Smem {
  static constexpr size_t kCol = (size_t)(kC4Tile + 8) * 4;
  static constexpr size_t kVal = (size_t)(kC4Tile + 4) * 8;
  static constexpr size_t kBnd = (size_t)(kC4MaxCoarse + 2) * 4;
  static constexpr size_t kTotal = kVal + kCol + kBnd + 16;
};

constexpr int kC4Ent = 256;   // CSC entries of one column per work item

// Work items of the outer-product pass: (referenced B row k, chunk of kC4Ent CSC entries of column k).
__global__ void k_c4_icount(DevCsr B, const int64_t* __restrict__ colptr, int64_t* __restrict__ icnt) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < B.n_rows; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ne = colptr[k + 1] - colptr[k];
    icnt[k] = (ne > 0 && B.rp(k + 1) > B.rp(k)) ? (ne + kC4Ent - 1) / kC4Ent : 0;
  }
}

// Outer-product pass: one CTA per work item (dynamic tickets).  The B row is staged tile by tile
// in shared memory and reused by the item's CSC entries (one warp per entry at a time).
__global__ void __launch_bounds__(kC4T)
k_c4_scatter(DevCsr B, const int32_t* __restrict__ rows, C4Geom g, const int64_t* __restrict__ mn,
             const int64_t* __restrict__ mx, const int64_t* __restrict__ choff, const uint32_t* __restrict__ ce,
             const int64_t* __restrict__ hbase, int64_t batch_base, const int64_t* __restrict__ colptr,
             const int64_t* __restrict__ iptr, const int32_t* __restrict__ csc_h, const uint32_t* __restrict__ csc_q,
             const double* __restrict__ csc_a, const uint32_t* __restrict__ koff, unsigned long long* __restrict__ ticket,
             uint32_t* __restrict__ ccol, double* __restrict__ cval) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_val = reinterpret_cast<double*>(smem);
  uint32_t* s_col = reinterpret_cast<uint32_t*>(smem + C4Smem::kVal);
  uint32_t* s_bnd = reinterpret_cast<uint32_t*>(smem + C4Smem::kVal + C4Smem::kCol);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C4Smem::kVal + C4Smem::kCol + C4Smem::kBnd);
  __shared__ long long s_k, s_e0;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kC4T / 32;
  const int csl = g.sc - g.sf;
  const uint32_t cmask = g.sc >= 32 ? 0xffffffffu : ((1u << g.sc) - 1u);
  const int64_t nitems = iptr[B.n_rows];
  if (tid == 0) {
    mbar_init(bar);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  uint32_t fills = 0;
  while (true) {
    if (tid == 0) {
      const long long t = (long long)atomicAdd(ticket, 1ull);
      long long k = -1, e0 = 0;
      if (t < nitems) {
        int64_t lo = 0, hi = B.n_rows;   // last k with iptr[k] <= t
        while (hi - lo > 1) {
          const int64_t mid = (lo + hi) >> 1;
          if (iptr[mid] <= t) lo = mid; else hi = mid;
        }
        k = lo;
        e0 = colptr[k] + (t - iptr[k]) * kC4Ent;
      }
      s_k = k;
      s_e0 = e0;
    }
    __syncthreads();
    const int64_t k = s_k, e0 = s_e0;
    __syncthreads();
    if (k < 0) break;
    const int64_t e1 = min(colptr[k + 1], e0 + kC4Ent);
    const uint32_t b0 = (uint32_t)B.rp(k), b1 = (uint32_t)B.rp(k + 1);
    for (uint32_t t0 = b0; t0 < b1; t0 += kC4Tile) {
      const uint32_t cnt = min((uint32_t)kC4Tile, b1 - t0);
      // coarse chunks the tile touches: s_bnd[c - c_lo] = first position of the row with column >= c << sc
      const uint32_t c_lo = g.sc >= 32 ? 0u : __ldg(B.col + t0) >> g.sc;
      const uint32_t c_hi = g.sc >= 32 ? 0u : __ldg(B.col + t0 + cnt - 1) >> g.sc;
      // stage the tile: bulk async copies of 16-byte aligned supersets
      const uintptr_t ca = reinterpret_cast<uintptr_t>(B.col + t0), va = reinterpret_cast<uintptr_t>(B.val + t0);
      const uintptr_t ca0 = ca & ~uintptr_t(15), va0 = va & ~uintptr_t(15);
      const uint32_t cskip = (uint32_t)(ca - ca0) / 4, vskip = (uint32_t)(va - va0) / 8;
      __syncthreads();   // the previous tile is consumed
      for (uint32_t c = c_lo + tid; c <= c_hi; c += kC4T)
        s_bnd[c - c_lo] = lower_bound_col(B.col, b0, b1, c << g.sc);
      // (the last elements of B are loaded element by element: an aligned superset would read
      // past the caller's arrays)
      const bool bulk = (int64_t)t0 + cnt + 4 <= B.nnz;
      if (bulk) {
        if (tid == 0) {
          const uint32_t cb = (uint32_t)(((ca + (size_t)cnt * 4 - ca0) + 15) & ~uintptr_t(15));
          const uint32_t vb = (uint32_t)(((va + (size_t)cnt * 8 - va0) + 15) & ~uintptr_t(15));
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          bulk_load2(bar, s_col, reinterpret_cast<const void*>(ca0), cb, s_val, reinterpret_cast<const void*>(va0), vb);
        }
        mbar_wait(bar, fills & 1u);
        ++fills;
      } else {
        for (uint32_t t = tid; t < cnt; t += kC4T) {
          s_col[cskip + t] = __ldg(B.col + t0 + t);
          s_val[vskip + t] = __ldg(B.val + t0 + t);
        }
      }
      __syncthreads();   // boundaries written (and the element-wise tile)
      const uint32_t* tc = s_col + cskip;
      const double* tv = s_val + vskip;
      // every CSC entry of the item reuses the staged tile
      for (int64_t en = e0 + wid; en < e1; en += NW) {
        const int32_t h = __ldg(csc_h + en);
        const uint32_t q = __ldg(csc_q + en);
        const double a = __ldg(csc_a + en);
        const int64_t i = rows[h];
        const int64_t c0 = mn[i] >> g.sf;
        const int64_t rowbase = hbase[h] - batch_base;
        const uint32_t* e = ce + choff[h];
        const uint32_t* ko = koff + (size_t)q * g.ncc;
        for (uint32_t t = lane; t < cnt; t += 32) {
          const uint32_t col = tc[t];
          const uint32_t cc = g.sc >= 32 ? 0u : col >> g.sc;
          const int64_t jl = max((int64_t)0, ((int64_t)cc << csl) - c0);
          const int64_t dst = rowbase + __ldg(e + jl) + __ldg(ko + cc) + ((t0 + t) - s_bnd[cc - c_lo]);
          ccol[dst] = col & cmask;
          cval[dst] = __dmul_rn(a, tv[t]);
        }
      }
    }
  }
}

// Fine level of one (row, coarse chunk) bucket: one CTA reads the bucket in order -- four
// contiguous warp ranges -- and appends every element to its fine chunk's slice.  Pass 1 counts
// each warp's elements per fine chunk, a prefix over the warps gives every warp its first slot
// in every slice, pass 2 scatters (stable: warp ranges are in bucket order, lanes of one wave
// are ranked in lane order).  Buckets by dynamic tickets.
constexpr int kC4FT = 128;
__global__ void __launch_bounds__(kC4FT)
k_c4_fine(const int32_t* __restrict__ rows, const int32_t* __restrict__ list, int64_t nlist, C4Geom g,
          const int64_t* __restrict__ mn, const int64_t* __restrict__ mx, const int64_t* __restrict__ choff,
          const uint32_t* __restrict__ ce, const int64_t* __restrict__ hbase, int64_t batch_base,
          const uint32_t* __restrict__ ccol, const double* __restrict__ cval, unsigned long long* __restrict__ ticket,
          uint16_t* __restrict__ bcol, double* __restrict__ bval) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NW = kC4FT / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int csl = g.sc - g.sf;
  const int nf = 1 << csl;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem);   // [NW][nf]
  uint32_t* cur = cnt + (size_t)wid * nf;
  __shared__ long long s_t;
  const uint32_t fmask = (1u << g.sf) - 1u, lt = lanemask_lt();
  const int64_t nb = nlist * g.ncc;   // (row, coarse chunk) pairs; empty ones cost one ticket
  while (true) {
    if (tid == 0) s_t = (long long)atomicAdd(ticket, 1ull);
    __syncthreads();
    const int64_t t = s_t;
    __syncthreads();
    if (t >= nb) break;
    const int32_t h = list[t / g.ncc];
    const int64_t cc = t % g.ncc;
    const int64_t i = rows[h];
    if (cc < (mn[i] >> g.sc) || cc > (mx[i] >> g.sc)) continue;
    const RowBins rb = row_bins(mn[i], mx[i], g.sf);
    const uint32_t* e = ce + choff[h];
    const int64_t jl = max((int64_t)0, (cc << csl) - rb.c0), jh = min((int64_t)rb.nchunk, ((cc + 1) << csl) - rb.c0);
    const uint32_t s0 = __ldg(e + jl), s1 = __ldg(e + jh);
    if (s0 == s1) continue;
    const int64_t rowbase = hbase[h] - batch_base;
    const int64_t jrel = (cc << csl) - rb.c0;   // row-relative fine chunk of the coarse chunk's first fine chunk
    const uint32_t n = s1 - s0;
    const uint32_t L = ((n + NW - 1) / NW + 31) & ~31u;
    const uint32_t q_beg = s0 + min(n, (uint32_t)wid * L), q_end = s0 + min(n, (uint32_t)(wid + 1) * L);
    for (int f = tid; f < NW * nf; f += kC4FT) cnt[f] = 0u;
    __syncthreads();
    for (uint32_t q = q_beg + lane; q < q_end; q += 32) atomicAdd(&cur[__ldg(ccol + rowbase + q) >> g.sf], 1u);
    __syncthreads();
    for (int f = tid; f < nf; f += kC4FT) {
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t v = cnt[(size_t)w * nf + f];
        cnt[(size_t)w * nf + f] = run;
        run += v;
      }
    }
    __syncthreads();
    for (uint32_t q0 = q_beg; q0 < q_end; q0 += 32) {
      const uint32_t q = q0 + lane;
      const bool valid = q < q_end;
      const uint32_t lc = valid ? __ldg(ccol + rowbase + q) : 0u;
      const double v = valid ? __ldg(cval + rowbase + q) : 0.0;
      const uint32_t f = valid ? lc >> g.sf : 0x40000000u + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, f);
      const uint32_t rank = __popc(peers & lt);
      uint32_t base = 0;
      if (valid) base = cur[f];
      __syncwarp();
      if (valid && rank == 0) cur[f] = base + __popc(peers);
      if (valid) {
        const int64_t dst = rowbase + __ldg(e + (jrel + (int64_t)f)) + base + rank;
        bcol[dst] = (uint16_t)(lc & fmask);
        bval[dst] = v;
      }
      __syncwarp();
    }
  }
}

}  // namespace mg
