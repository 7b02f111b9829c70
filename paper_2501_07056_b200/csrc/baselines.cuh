// Gustavson baselines on the device (reference gustavson.py:155-268): the ablation that
// shows what MAGNUS's locality generation buys on B200, and a second path to check it by.
//
//  * dense (gustavson_dense_symbolic / gustavson_dense_numeric): one CTA per row over a
//    full-width accumulator in global memory (n_cols doubles + an n_cols-bit bitmap per
//    CTA, L2/HBM resident -- no chunking, no locality generation).  Columns are marked
//    with global atomicOr; values are applied one A nonzero (k) at a time in ascending k
//    with a CTA barrier between k's, so every entry is ((+0.0 + x0) + x1) + ... -- the
//    reference's DenseAccumulator (np.bincount / np.add.at, sequential from 0.0).  The row
//    is emitted sorted (canonicalize_csr): a shared-memory bitonic sort of the touched
//    list (<= kGdList columns) or an ordered scan of the row's bitmap range.
//  * esc (gustavson_esc_numeric): per batch of rows, every product is expanded in
//    Gustavson order as key (row << 32 | col) + value, the keys are sorted stably (ties keep
//    Gustavson order, i.e. ascending k), and each run of equal keys is reduced as
//    x0 + pairwise(x1..x_{d-1}) -- the reference's sort_accumulate (np.add.reduceat).
#pragma once
#include "common.cuh"

namespace mg {

constexpr int kGdT = 256;             // threads per CTA
constexpr int kGdW = kGdT / 32;
constexpr int kGdList = 4096;         // touched columns sorted in shared memory

template <bool kNum>
__global__ void __launch_bounds__(kGdT)
k_gd_rows(DevCsr A, DevCsr B, const int64_t* __restrict__ c_rp, uint32_t* __restrict__ c_col,
          double* __restrict__ c_val, int64_t* __restrict__ row_nnz, uint32_t* __restrict__ bm_all,
          double* __restrict__ acc_all, int64_t nwords, unsigned long long* __restrict__ ticket,
          unsigned long long* __restrict__ err) {
  __shared__ uint32_t list[kGdList];
  __shared__ uint32_t s_n, s_wlo, s_whi;
  __shared__ long long s_row;
  __shared__ uint32_t s_wsum[kGdW + 1];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t* bm = bm_all + (size_t)blockIdx.x * nwords;
  double* acc = kNum ? acc_all + (size_t)blockIdx.x * nwords * 32 : nullptr;
  while (true) {
    if (tid == 0) {
      s_row = (long long)atomicAdd(ticket, 1ull);
      s_n = 0u;
      s_wlo = 0xffffffffu;
      s_whi = 0u;
    }
    __syncthreads();
    const int64_t i = s_row;
    if (i >= A.n_rows) break;
    const int64_t a0 = A.rp(i), a1 = A.rp(i + 1);
    // ---- mark the row's columns (any order); first touch zeroes the accumulator entry
    for (int64_t p = a0 + wid; p < a1; p += kGdW) {
      const int64_t k = __ldg(A.col + p);
      const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
      for (int64_t q = b0 + lane; q < b1; q += 32) {
        const uint32_t c = __ldg(B.col + q), bit = 1u << (c & 31u);
        const uint32_t old = atomicOr(bm + (c >> 5), bit);
        if (!(old & bit)) {
          const uint32_t t = atomicAdd(&s_n, 1u);
          if (t < kGdList) list[t] = c;
          atomicMin(&s_wlo, c >> 5);
          atomicMax(&s_whi, c >> 5);
          if (kNum) acc[c] = 0.0;
        }
      }
    }
    __syncthreads();
    const uint32_t n = s_n;
    const uint32_t wlo = s_wlo, whi = s_whi;
    bool ok = true;
    int64_t out = 0;
    if (kNum) {
      out = c_rp[i];
      ok = (int64_t)n == c_rp[i + 1] - out;
      if (!ok && tid == 0) atomicOr(err, 1ull);
      // ---- values: one k at a time, ascending (canonical B rows hold distinct columns)
      if (ok) {
        for (int64_t p = a0; p < a1; ++p) {
          const int64_t k = __ldg(A.col + p);
          const double av = __ldg(A.val + p);
          const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
          for (int64_t q = b0 + tid; q < b1; q += kGdT) {
            const uint32_t c = __ldg(B.col + q);
            acc[c] = __dadd_rn(acc[c], __dmul_rn(__ldg(B.val + q), av));
          }
          __syncthreads();
        }
      }
    } else if (tid == 0) {
      row_nnz[i] = n;
    }
    if (n <= (uint32_t)kGdList) {
      // ---- emit in column order: bitonic sort of the touched list
      if (kNum && ok && n > 1) {
        uint32_t P = 1;
        while (P < n) P <<= 1;
        for (uint32_t t = n + tid; t < P; t += kGdT) list[t] = 0xffffffffu;
        __syncthreads();
        for (uint32_t kk = 2; kk <= P; kk <<= 1) {
          for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
            for (uint32_t t = tid; t < P; t += kGdT) {
              const uint32_t u = t ^ j;
              if (u > t) {
                const uint32_t x = list[t], y = list[u];
                if ((x > y) == ((t & kk) == 0)) { list[t] = y; list[u] = x; }
              }
            }
            __syncthreads();
          }
        }
      }
      for (uint32_t t = tid; t < n; t += kGdT) {
        const uint32_t c = list[t];
        if (kNum && ok) {
          c_col[out + t] = c;
          c_val[out + t] = acc[c];
        }
        bm[c >> 5] = 0u;
      }
    } else if (kNum && ok) {
      // ---- long row: ordered scan of the bitmap words wlo..whi (4 words per thread per round)
      uint32_t carry = 0;
      for (uint32_t w0 = wlo; w0 <= whi; w0 += 4 * kGdT) {
        const uint32_t wb = w0 + 4u * tid;
        uint32_t wv[4], cnt = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          wv[j] = wb + j <= whi ? __ldcg(bm + wb + j) : 0u;   // bits were set by L2 atomics
          cnt += __popc(wv[j]);
        }
        const uint32_t inc = warp_incl_scan(cnt);
        if (lane == 31) s_wsum[wid] = inc;
        __syncthreads();
        if (tid == 0) {
          uint32_t r = 0;
          for (int w = 0; w < kGdW; ++w) { const uint32_t v = s_wsum[w]; s_wsum[w] = r; r += v; }
          s_wsum[kGdW] = r;
        }
        __syncthreads();
        uint32_t pos = carry + s_wsum[wid] + inc - cnt;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t m = wv[j];
          while (m) {
            const uint32_t b = __ffs(m) - 1u;
            m &= m - 1u;
            const uint32_t c = ((wb + j) << 5) + b;
            c_col[out + pos] = c;
            c_val[out + pos] = acc[c];
            ++pos;
          }
          if (wb + j <= whi) bm[wb + j] = 0u;
        }
        carry += s_wsum[kGdW];
        __syncthreads();
      }
    } else {
      for (uint32_t w = wlo + tid; w <= whi; w += kGdT) bm[w] = 0u;
    }
    __syncthreads();
  }
}

// ---- ESC: expand (warp per row; products of row r at ioff[r] - ioff[r0], Gustavson order)
__global__ void __launch_bounds__(256)
k_esc_expand(DevCsr A, DevCsr B, int64_t r0, int64_t r1, const int64_t* __restrict__ ioff,
             uint64_t* __restrict__ keys, double* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = r0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < r1; r += nw) {
    int64_t o = ioff[r] - ioff[r0];
    const uint64_t hi = (uint64_t)(r - r0) << 32;
    const int64_t a1 = A.rp(r + 1);
    for (int64_t p = A.rp(r); p < a1; ++p) {
      const int64_t k = __ldg(A.col + p);
      const double av = __ldg(A.val + p);
      const int64_t b0 = B.rp(k), b1 = B.rp(k + 1);
      for (int64_t q = b0 + lane; q < b1; q += 32) {
        keys[o + (q - b0)] = hi | __ldg(B.col + q);
        vals[o + (q - b0)] = __dmul_rn(__ldg(B.val + q), av);
      }
      o += b1 - b0;
    }
  }
}

// run heads of the sorted keys (1 / 0 as int64, scanned into run indices)
__global__ void k_esc_heads(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ flag) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1 : 0;
}

// one thread per run head: column, and x0 + pairwise(x1..) over the run's values (perm order)
__global__ void k_esc_reduce(const uint64_t* __restrict__ keys, const int64_t* __restrict__ perm,
                             const double* __restrict__ vals, int64_t n, const int64_t* __restrict__ run,
                             int64_t out0, uint32_t* __restrict__ c_col, double* __restrict__ c_val) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[j];
    if (j > 0 && keys[j - 1] == key) continue;
    int64_t e = j + 1;
    while (e < n && keys[e] == key) ++e;
    const int64_t o = out0 + run[j];
    c_col[o] = (uint32_t)(key & 0xffffffffull);
    double s = vals[perm[j]];
    if (e - j > 1) {
      auto x = [&](int64_t q) { return vals[perm[q]]; };
      s = __dadd_rn(s, pairwise(x, j + 1, e - j - 1));
    }
    c_val[o] = s;
  }
}

}  // namespace mg
