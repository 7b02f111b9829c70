/*
 * Device generators for the seeded BASELINE.json inputs (setup plumbing, not
 * the SpGEMM path).  Bit-identical to paper_2501_07056_b200/generate.py.
 * All output pointers are device pointers; stream = cudaStream_t.
 */
#ifndef MAGNUS_GEN_H
#define MAGNUS_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* R-MAT edges lo..lo+m as keys (row << scale) | col (quadrant mapping of the
 * reference's _rmat_edge_batch, generate.py:56-68). */
int magnus_gen_rmat_keys(int scale, int64_t lo, int64_t m, uint64_t seed, double a, double b, double c, uint64_t* out,
                         void* stream);
/* out[p] = U[-1,1) draw of (seed, stream_id, p). */
int magnus_gen_uniform_pm1(uint64_t seed, uint64_t stream_id, int64_t n, double* out, void* stream);
/* exactly d distinct sorted uniform columns per row (Floyd sampling), d <= 64. */
int magnus_gen_uniform_rows(int64_t n_rows, int64_t n_cols, int d, uint64_t seed, int32_t* col, void* stream);
#ifdef __cplusplus
}
#endif
#endif
