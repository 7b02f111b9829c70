/* TEST INFRASTRUCTURE ONLY -- CPU oracle restating the reference MAGNUS path.
 * See magnus_oracle.c for the reference citations. */
#pragma once
#include <stdint.h>

enum { ORACLE_OK = 0, ORACLE_INPUT = 1, ORACLE_CONTRACT = 2, ORACLE_OVER_BUDGET = 3 };
enum { ORACLE_CAT_SORT = 0, ORACLE_CAT_DENSE = 1, ORACLE_CAT_FINE = 2, ORACLE_CAT_COARSE = 3 };

typedef struct { int64_t n_rows, n_cols; const int64_t* row_ptr; const uint32_t* col; const double* val; } oracle_csr;
/* SystemParams planner.py:47-68 */
typedef struct { int64_t cache_line_bytes, l2_bytes, memory_budget_bytes, histo_type_bytes, prefix_sum_type_bytes, val_bytes; } oracle_sys;
/* AccumThresholds accumulators.py:34-41 */
typedef struct { int64_t sort_dense_crossover, sort_sweet_spot; } oracle_thresholds;
/* ChunkPlan planner.py:79-92 */
typedef struct { int64_t plan_cols, s_dense_accum, s_chunk_fine, n_chunks_fine, chunk_len_fine, shift_fine,
                 m_max_l2, use_coarse, n_chunks_coarse, chunk_len_coarse, shift_coarse; } oracle_plan;

#ifdef __cplusplus
extern "C" {
#endif
int oracle_compute_chunk_plan(const oracle_sys* sys, int64_t m_c, int numeric, int allow_coarse, oracle_plan* out);
/* info[7] = {nnz_c, inter_prod_size, coarse_batches, rows_sort, rows_dense, rows_fine, rows_coarse} */
int oracle_symbolic(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                    int force_fine_only, int threads, int64_t* row_ptr, int64_t* info);
int oracle_numeric(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                   int force_fine_only, int threads, const int64_t* row_ptr, uint32_t* c_col, double* c_val, int64_t* info);
int oracle_setup(const oracle_csr* A, const oracle_csr* B, const oracle_sys* sys, const oracle_thresholds* th,
                 int force_fine_only, int64_t* inter, int64_t* mn, int64_t* mx, int8_t* cat);
double oracle_pairwise_sum(const double* a, int64_t n);
/* Gustavson baselines (gustavson.py:155-250): phase 0 symbolic -> row_ptr; 1 dense numeric; 2 esc numeric */
int oracle_gustavson(const oracle_csr* A, const oracle_csr* B, int phase, int threads, int64_t* row_ptr, uint32_t* c_col,
                     double* c_val);
const char* oracle_last_error(void);
#ifdef __cplusplus
}
#endif
