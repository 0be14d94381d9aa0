/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the CSR SpMM hot path.
 *
 * This file restates, in plain C, the reference algorithms that pin the
 * results of the B200 kernels.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it; the product package never links
 * or imports anything under oracle/.
 *
 * Parity pin: every function below is checked against fixtures produced by
 * importing the reference package (tests/golden/make_golden.py) -- see
 * tests/test_oracle.py.
 *
 * Reference (paths relative to /root/reference/pkg/src/spmmlab/):
 *   oracle_spmm_*          matrices.py:241-254  dense_spmm_oracle
 *   oracle_search_before   lowering.py:99-116   binary_search_before
 *   oracle_block_starts    lowering.py:119-128  compute_block_starts
 *   oracle_writebacks_*    sim.py:112-165 + lowering.py:459-646 (the
 *                          SimMetrics.atomic_ops counter of sim.run for each
 *                          template family)
 *
 * Build: see oracle/Makefile (-O2 -ffp-contract=off, no fast-math, so every
 * multiply and add rounds separately exactly as numpy does).
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* dense_spmm_oracle (matrices.py:241-254).                                  */
/* For every output row i, out[i,:] starts at 0.0 and accumulates            */
/*   out[i,k] = out[i,k] + (vals[p] * B[col[p],k])                            */
/* for p ascending over the row.  numpy evaluates the product vector first   */
/* (one rounding) and then the add (second rounding); -ffp-contract=off      */
/* keeps the two roundings separate here, which makes the result bitwise     */
/* identical.  Rows are independent, so threading over rows does not change  */
/* any bit of the result.                                                     */
/* ------------------------------------------------------------------------ */

#define ORACLE_SPMM_BODY(IDX_T)                                                  \
    int64_t i;                                                                   \
    _Pragma("omp parallel for schedule(dynamic, 64) num_threads(nthreads)")      \
    for (i = 0; i < num_rows; ++i) {                                             \
        double *out = c + i * n;                                                 \
        for (int64_t k = 0; k < n; ++k) out[k] = 0.0;                            \
        for (int64_t p = (int64_t)row_ptr[i]; p < (int64_t)row_ptr[i + 1]; ++p) { \
            const double a = vals[p];                                            \
            const double *brow = b + (int64_t)col_idx[p] * n;                    \
            for (int64_t k = 0; k < n; ++k) {                                    \
                const double prod = a * brow[k];                                 \
                out[k] = out[k] + prod;                                          \
            }                                                                    \
        }                                                                        \
    }

void oracle_spmm_i64(int64_t num_rows, int64_t n, const int64_t *row_ptr,
                     const int64_t *col_idx, const double *vals, const double *b,
                     double *c, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    ORACLE_SPMM_BODY(int64_t)
}

void oracle_spmm_i32(int64_t num_rows, int64_t n, const int32_t *row_ptr,
                     const int32_t *col_idx, const double *vals, const double *b,
                     double *c, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    ORACLE_SPMM_BODY(int32_t)
}

/* Same order, but the values are float32 widened to double on the fly (the
 * GPU path computes on the float32-rounded inputs; feeding the oracle the same
 * rounded values makes the comparison measure accumulation error only). */
void oracle_spmm_i32_f32in(int64_t num_rows, int64_t n, const int32_t *row_ptr,
                           const int32_t *col_idx, const float *vals,
                           const float *b, double *c, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    int64_t i;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
    for (i = 0; i < num_rows; ++i) {
        double *out = c + i * n;
        for (int64_t k = 0; k < n; ++k) out[k] = 0.0;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const double a = (double)vals[p];
            const float *brow = b + (int64_t)col_idx[p] * n;
            for (int64_t k = 0; k < n; ++k) {
                const double prod = a * (double)brow[k];
                out[k] = out[k] + prod;
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* binary_search_before (lowering.py:99-116): largest p in [lo, hi) with      */
/* array[p] <= target; clamps to lo when none qualifies or the window is      */
/* empty.                                                                     */
/* ------------------------------------------------------------------------ */
int64_t oracle_search_before(const int64_t *array, int64_t lo, int64_t hi,
                             int64_t target) {
    if (hi <= lo) return lo;
    if (array[lo] > target) return lo;
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) / 2;
        if (array[mid] <= target) lo = mid; else hi = mid;
    }
    return lo;
}

/* ------------------------------------------------------------------------ */
/* compute_block_starts (lowering.py:119-128):                                */
/*   starts[b] = searchsorted(row_ptr, b*chunk, side='right') - 1             */
/* i.e. the last index r in [0, num_rows] with row_ptr[r] <= b*chunk, over    */
/* the whole num_rows+1 array (so the value can equal num_rows).              */
/* ------------------------------------------------------------------------ */
void oracle_block_starts(const int64_t *row_ptr, int64_t num_rows,
                         int64_t chunk, int64_t num_blocks, int64_t *starts) {
    for (int64_t b = 0; b <= num_blocks; ++b) {
        const int64_t t = b * chunk;
        /* upper bound over [0, num_rows+1) */
        int64_t lo = 0, hi = num_rows + 1;
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if (row_ptr[mid] <= t) lo = mid + 1; else hi = mid;
        }
        starts[b] = lo - 1;
    }
}

/* Row a lane resolves to in a position-chunked kernel (lowering.py:459-500):
 * the clamped search over the block window, then -- for in-range positions
 * only -- the forward while-advance over rows that end at the position. */
static int64_t lane_row(const int64_t *row_ptr, int64_t num_rows, int64_t nnz,
                        const int64_t *starts, int64_t block, int64_t pos) {
    int64_t hi = starts[block + 1] + 1;
    if (hi > num_rows) hi = num_rows;
    int64_t i = oracle_search_before(row_ptr, starts[block], hi, pos);
    if (pos < nnz) {
        while (pos == row_ptr[i + 1]) ++i;
    }
    return i;
}

/* ------------------------------------------------------------------------ */
/* SimMetrics.atomic_ops restated per family (sim.py:353-393).               */
/* ------------------------------------------------------------------------ */

/* nnz-one, r > 1: SegReduceGroup over aligned groups of r lanes.  Every lane */
/* of the launched grid takes part (out-of-range lanes are zero-extended and   */
/* keep the clamped search row), one writeback per run of equal rows per       */
/* group, for each of the n dense columns (sim.py:139-165,                    */
/* lowering.py:526-537).                                                      */
int64_t oracle_writebacks_nnz_one_segment(const int64_t *row_ptr,
                                          int64_t num_rows, int64_t n,
                                          const int64_t *starts, int64_t grid,
                                          int64_t npb, int64_t r) {
    const int64_t nnz = row_ptr[num_rows];
    int64_t runs = 0;
    for (int64_t b = 0; b < grid; ++b) {
        int64_t prev = -1;
        for (int64_t q = 0; q < npb; ++q) {
            const int64_t pos = b * npb + q;
            const int64_t row = lane_row(row_ptr, num_rows, nnz, starts, b, pos);
            if (q % r == 0 || row != prev) ++runs;
            prev = row;
        }
    }
    return runs * n;
}

/* nnz-multiple: each thread walks g positions of its chunk, flushing an
 * AtomicAdd whenever the walk crosses into a new row, plus one final flush
 * after the walk -- executed even by threads whose chunk starts past nnz
 * (lowering.py:539-571, 639-641).  Every chunk is walked once per dense
 * column. */
int64_t oracle_writebacks_nnz_multiple(const int64_t *row_ptr, int64_t num_rows,
                                       int64_t n, const int64_t *starts,
                                       int64_t grid, int64_t chunk, int64_t g) {
    const int64_t nnz = row_ptr[num_rows];
    const int64_t per_block = chunk / g;
    int64_t flushes = 0;
    for (int64_t b = 0; b < grid; ++b) {
        int64_t hi = starts[b + 1] + 1;
        if (hi > num_rows) hi = num_rows;
        for (int64_t w = 0; w < per_block; ++w) {
            const int64_t base = b * chunk + w * g;
            int64_t i = oracle_search_before(row_ptr, starts[b], hi, base);
            for (int64_t q = 0; q < g; ++q) {
                const int64_t pos = base + q;
                if (pos >= nnz) break;
                if (pos == row_ptr[i + 1]) {
                    ++flushes;
                    while (pos == row_ptr[i + 1]) ++i;
                }
            }
            ++flushes; /* the final flush */
        }
    }
    return flushes * n;
}

/* Size of the per-thread reference workload, used by the bench's CPU leg to
 * report how many threads the oracle can use. */
int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
