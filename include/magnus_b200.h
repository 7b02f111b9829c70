/*
 * magnus_b200 -- C-ABI of the B200-native MAGNUS SpGEMM (C = A.B, CSR in, CSR out).
 *
 * The reference (arxiv/paper_2501_07056, /root/reference/pkg) is a Python
 * package with no FFI; its boundary is the Python function
 *     spgemm_magnus(A, B, sys=None, thresholds=None, threads=1, force_fine_only=False)
 * (magnus.py:545-583) and its two phases magnus_symbolic (magnus.py:420-456)
 * and magnus_numeric (magnus.py:459-542).  This header is what that function
 * binds to (paper_2501_07056_b200/_lib.py, via ctypes): plain pointers and
 * sizes, no torch types.  All array pointers are DEVICE pointers owned by the
 * caller; the library only allocates its own workspace inside a magnus_ctx.
 *
 * Error convention (reference errors.py:4-27): every entry point returns a
 * status code; magnus_last_error() returns the thread-local message.
 */
#ifndef MAGNUS_B200_H
#define MAGNUS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MAGNUS_OK = 0,
  MAGNUS_INPUT = 1,       /* InputError         errors.py:8    */
  MAGNUS_CONTRACT = 2,    /* ContractViolation  errors.py:22   */
  MAGNUS_OVER_BUDGET = 3, /* OverBudgetError    errors.py:26   */
  MAGNUS_CUDA = 4         /* CUDA runtime error (no reference counterpart) */
};

enum { MAGNUS_CAT_SORT = 0, MAGNUS_CAT_DENSE = 1, MAGNUS_CAT_FINE = 2, MAGNUS_CAT_COARSE = 3 };

/* CsrMatrix matrix.py:18-44.  row_ptr is int32 (rp_bytes=4) or int64 (8);
 * col holds the reference's uint32 column indices (util.py:47-49). */
typedef struct {
  int64_t n_rows, n_cols, nnz;
  const void* row_ptr;
  int32_t rp_bytes;
  const uint32_t* col;
  const double* val;
} magnus_csr;

/* SystemParams planner.py:47-68 */
typedef struct {
  int64_t cache_line_bytes, l2_bytes, memory_budget_bytes, histo_type_bytes, prefix_sum_type_bytes, val_bytes;
} magnus_sys;

/* AccumThresholds accumulators.py:34-41 */
typedef struct {
  int64_t sort_dense_crossover, sort_sweet_spot;
} magnus_thresholds;

/* ChunkPlan planner.py:79-92 */
typedef struct {
  int64_t plan_cols, s_dense_accum, s_chunk_fine, n_chunks_fine, chunk_len_fine, shift_fine, m_max_l2, use_coarse,
      n_chunks_coarse, chunk_len_coarse, shift_coarse;
} magnus_chunk_plan;

/* SpgemmResult.counters magnus.py:536-541 */
typedef struct {
  int64_t nnz_c, inter_prod_size, coarse_batches, rows_sort, rows_dense, rows_fine, rows_coarse;
} magnus_counters;

typedef struct magnus_ctx magnus_ctx;

/* compute_chunk_plan planner.py:106-152 (host arithmetic, no device needed). */
int magnus_compute_chunk_plan(const magnus_sys* sys, int64_t m_c, int numeric, int allow_coarse, magnus_chunk_plan* out);

/* Context: owns the device workspace between the phases; bound to the current device. */
int magnus_ctx_create(magnus_ctx** out);
void magnus_ctx_destroy(magnus_ctx* ctx);

/* Setup phase of spgemm_magnus (magnus.py:567-571): row_intermediate_stats
 * (gustavson.py:97-134), both chunk plans, categorize_rows (magnus.py:68-94),
 * build_coarse_batches' budget check (magnus.py:296-300).  A and B must stay
 * alive and unmodified until magnus_numeric returns.  stream = cudaStream_t. */
int magnus_setup(magnus_ctx* ctx, const magnus_csr* A, const magnus_csr* B, const magnus_sys* sys,
                 const magnus_thresholds* thresholds, int force_fine_only, void* stream);

/* magnus_symbolic (magnus.py:420-456): writes C.row_ptr (int64, n_rows+1,
 * device) and the total nnz(C) to *nnz_out (host; the call synchronises). */
int magnus_symbolic(magnus_ctx* ctx, int64_t* c_row_ptr, int64_t* nnz_out, void* stream);

/* magnus_numeric (magnus.py:459-542): fills C.col / C.val (device, nnz(C)
 * entries) canonically; counters (host) as in SpgemmResult.counters. */
int magnus_numeric(magnus_ctx* ctx, const int64_t* c_row_ptr, uint32_t* c_col, double* c_val,
                   magnus_counters* counters, void* stream);

/* row_intermediate_stats gustavson.py:97-134 on device arrays (n_rows each). */
int magnus_row_stats(const magnus_csr* A, const magnus_csr* B, int64_t* inter, int64_t* min_col, int64_t* max_col,
                     void* stream);

/* Per-row categories (int8, MAGNUS_CAT_*) computed by the last magnus_setup; copies n_rows bytes to device dst. */
int magnus_categories(magnus_ctx* ctx, int8_t* dst, void* stream);

/* Caller-owned workspace.  After magnus_symbolic: the device bytes the numeric
 * phase's largest buffer -- the heavy rows' reorder buffer (u16 column + f64 product per heavy-row
 * product) -- takes in one batch (*preferred) and at least (*minimum: the heaviest row); 0 when
 * the call has no heavy rows.  magnus_set_workspace(ctx, ws, bytes): the next magnus_numeric carves
 * that buffer from the caller's device memory (>= *minimum bytes; batches are sized to it) instead
 * of the library pool; (NULL, 0) returns to library-owned workspace. */
int magnus_workspace_bytes(magnus_ctx* ctx, int64_t* preferred, int64_t* minimum);
int magnus_set_workspace(magnus_ctx* ctx, void* ws, int64_t bytes);

/* The library's device workspace (chunk tables, reorder buffers, per-call scratch) comes from a
 * private stream-ordered memory pool of the current device, never from the default pool.  Freed
 * workspace stays reserved there between calls; magnus_release_workspace() synchronises the
 * device and returns it to the driver; magnus_workspace_reserved() = bytes the pool holds. */
int magnus_release_workspace(void);
int64_t magnus_workspace_reserved(void);

/* Number of kernel launches issued by this context since creation (telemetry). */
int64_t magnus_launch_count(magnus_ctx* ctx);

/* Kernel timing telemetry (off by default): when enabled, CUDA events bracket
 * every launch on the launching stream.  magnus_profile_read synchronises and
 * accumulates, per kernel id (MAGNUS_K_*), the total milliseconds and the
 * launch count since the last read (arrays of MAGNUS_K_COUNT entries). */
enum { MAGNUS_K_ROW_STATS = 0, MAGNUS_K_CATEGORIZE, MAGNUS_K_SYM_WARP, MAGNUS_K_SYM_BLOCK, MAGNUS_K_SYM_HEAVY,
       MAGNUS_K_SCAN, MAGNUS_K_NUM_WARP, MAGNUS_K_NUM_BLOCK, MAGNUS_K_NUM_HEAVY, MAGNUS_K_SYM_DENSE,
       MAGNUS_K_NUM_DENSE, MAGNUS_K_BIN_PLAN, MAGNUS_K_BIN_EXPAND, MAGNUS_K_BIN_REDUCE,
       MAGNUS_K_BIN_BIG, MAGNUS_K_DIR_INDEX, MAGNUS_K_DIR_PLAN, MAGNUS_K_DIR_NUM, MAGNUS_K_COUNT };
int magnus_profile_enable(magnus_ctx* ctx, int enable);
int magnus_profile_read(magnus_ctx* ctx, double* ms, int64_t* launches);

/* magnus_numeric, and C (col, val) read back into host memory c_col_host / c_val_host (page-locked
 * for overlap): completed row ranges are copied on a side stream while later heavy-row batches
 * compute.  Returns after the copies have finished.  C stays on the device as well. */
int magnus_numeric_host(magnus_ctx* ctx, const int64_t* c_row_ptr, uint32_t* c_col, double* c_val, uint32_t* c_col_host,
                        double* c_val_host, magnus_counters* counters, void* stream);

/* Heavy-row telemetry after magnus_symbolic (binned / direct paths, else zeros): out[0..3] =
 * products and distinct columns in "big" fine chunks (reduced by the dense big-chunk
 * reducer), products and distinct columns in the other chunks (sort reducer).  Synchronises. */
int magnus_heavy_stats(magnus_ctx* ctx, int64_t* out4);

/* Device coarse level (Alg. 4: build_coarse_chunks / coarse_level_batch magnus.py:317-406) of
 * the last magnus_numeric call: out[0] = Coarse-category rows that went through it, out[1] =
 * device batches, out[2] = CSC entries (A nonzeros of those rows).  Zeros when no row is Coarse,
 * or with MAGNUS_COARSE_PATH=fine (the fine-level expand handles them, same bits). */
int magnus_coarse_level_stats(magnus_ctx* ctx, int64_t* out3);

/* ---- Gustavson baselines (reference gustavson.py:155-268; the ablation without locality generation).
 * Dense: one CTA per row over a full-width accumulator.  scratch (device) must hold at least
 * magnus_gd_scratch_bytes(B->n_cols, 1) bytes; more lets more rows run concurrently (up to 4 per SM).
 * gustavson_dense_symbolic (gustavson.py:155-170): c_row_ptr (n_rows+1, device) = exclusive prefix of the
 * per-row distinct counts.  Synchronises. */
size_t magnus_gd_scratch_bytes(int64_t n_cols, int64_t ctas);
int magnus_gd_symbolic(const magnus_csr* A, const magnus_csr* B, int64_t* c_row_ptr, void* scratch, size_t scratch_bytes,
                       void* stream);
/* gustavson_dense_numeric (gustavson.py:184-220): values sequential from +0.0 in Gustavson order, rows
 * emitted sorted (canonicalize_csr).  MAGNUS_CONTRACT if a row's count differs from c_row_ptr.  Synchronises. */
int magnus_gd_numeric(const magnus_csr* A, const magnus_csr* B, const int64_t* c_row_ptr, uint32_t* c_col, double* c_val,
                      void* scratch, size_t scratch_bytes, void* stream);
/* gustavson_esc_numeric (gustavson.py:223-250), expand step: the products of rows [r0, r1) in Gustavson
 * order; row r's start at inter_off[r] - inter_off[r0] (inter_off = exclusive prefix of the rows' product
 * counts, device int64).  key = (r - r0) << 32 | col, val = B.val * A.val. */
int magnus_esc_expand(const magnus_csr* A, const magnus_csr* B, int64_t r0, int64_t r1, const int64_t* inter_off,
                      uint64_t* keys, double* vals, void* stream);
/* compress step over keys sorted stably (perm: source index of each sorted key into vals): run j of
 * equal keys -> C position out0 + j, column = key's low 32 bits, value = x0 + pairwise(x1..x_{d-1})
 * (sort_accumulate accumulators.py:113-129).  run_scratch: n+1 int64.  *runs_out (host) = number of runs
 * (synchronises before the reduce; with c_col or c_val NULL only the runs are counted). */
int magnus_esc_compress(const uint64_t* keys, const int64_t* perm, const double* vals, int64_t n, int64_t out0,
                        uint32_t* c_col, double* c_val, int64_t* run_scratch, int64_t* runs_out, void* stream);

/* ---- building-block microbenchmarks (reference bench.py:88-196): one synthetic stream of u32
 * indices < length and f64 values, each stage a kernel of its own.  Device pointers; asynchronous.
 * histogram: counts[c] = #{i : idx[i] >> shift == c} (int64, n_chunks <= 16384). */
int magnus_mb_histogram(const uint32_t* idx, int64_t n, int shift, int n_chunks, int64_t* counts, void* stream);
/* reorder: stable scatter of (idx & (2^shift - 1), val) into chunk order (stable_scatter_positions
 * matrix.py:187-204); n_chunks <= 4096; scratch of magnus_mb_reorder_scratch_bytes(n, n_chunks). */
size_t magnus_mb_reorder_scratch_bytes(int64_t n, int n_chunks);
int magnus_mb_reorder(const uint32_t* idx, const double* val, int64_t n, int shift, int n_chunks, void* scratch,
                      size_t scratch_bytes, uint32_t* out_col, double* out_val, void* stream);
/* dense accumulation per chunk (dense_accumulate accumulators.py:68-97; sequential from +0.0 in slice
 * order): chunk c's slice [offsets[c], offsets[c+1]) of chunk-local columns < chunk_len (<= 16384) is
 * replaced at its start by its distinct columns ascending and their sums; distinct[c] = their number. */
int magnus_mb_dense(const uint32_t* col, const double* val, const int64_t* offsets, int n_chunks, int chunk_len,
                    uint32_t* out_col, double* out_val, int64_t* distinct, void* stream);
/* exclusive prefix sum: out[0..n] (out[n] = total) of int64 in[0..n); scratch of magnus_mb_scan_scratch_bytes(n). */
size_t magnus_mb_scan_scratch_bytes(int64_t n);
int magnus_mb_scan(const int64_t* in, int64_t n, int64_t* out, void* scratch, void* stream);
/* stable sort of (key, position) pairs (LSD radix sort, 8-bit digits; one pass per byte of key_mask with a set bit --
 * key_mask covers every bit that can differ between keys): keys_out = the keys ascending, perm_out[j] = position in
 * `keys` of the j-th smallest (np.argsort(kind="stable"), reference bench.py:160-180 / accumulators.py:113-129).
 * scratch (device) of magnus_sort_pairs_scratch_bytes(n) bytes; keys_out / perm_out must not alias keys. */
size_t magnus_sort_pairs_scratch_bytes(int64_t n);
int magnus_sort_pairs(const uint64_t* keys, int64_t n, uint64_t key_mask, uint64_t* keys_out, int64_t* perm_out,
                      void* scratch, void* stream);
/* contiguous copy (the streaming baseline): bytes (multiple of 16, 16-byte aligned). */
int magnus_mb_stream(const void* src, void* dst, int64_t bytes, void* stream);

const char* magnus_last_error(void);
const char* magnus_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MAGNUS_B200_H */
