/*
 * sgap.h -- C ABI of the B200 (sm_100a) CSR SpMM engine for the Sgap
 * (arXiv 2209.02882) schedule space.  Drop-in for the executor of the
 * reference package `spmmlab` (paths relative to /root/reference/pkg/src/spmmlab).
 *
 * The reference boundary is the Python function
 *     sim.run(kernel: LoweredKernel, a: CsrMatrix, b: DenseMatrix,
 *             c0: DenseMatrix | None = None, *, precision="double")
 *         -> (DenseMatrix, SimMetrics)                       (sim.py:431-487)
 * whose LoweredKernel comes from runner.build_kernel (runner.py:141-156) =
 * templates.algorithm_template (templates.py:220-235) + lowering.lower
 * (lowering.py:649-696).  The entry points below replace:
 *
 *   sgap_legality_rule    space.legality_rule            space.py:177-204
 *   sgap_build_kernel     runner.build_kernel            runner.py:141-156
 *                         (family + divisibility gates   templates.py:82-202,
 *                          + grid/block geometry)         lowering.py:218-243,649-696)
 *   sgap_block_starts     lowering.compute_block_starts  lowering.py:119-128
 *   sgap_plan_workspace_bytes / sgap_plan
 *                         the per-matrix half of         lowering.py:683-696
 *                         runner.build_kernel (block_starts) + the engine's
 *                         side data (row ids, float64 long-row table,
 *                         error-free row list), all built on the device
 *   sgap_validate_csr     CsrMatrix invariants +         matrices.py:58-75,
 *                         SimulationFault on an out-of-  sim.py:279-287
 *                         range index
 *   sgap_run              sim.run                        sim.py:431-487
 *   sgap_run_rbpr_grid    the dgSPARSE RB+PR kernel under one cell of
 *                         space.enumerate_fine_grained   space.py:294-348
 *   sgap_seg_reduce_group sim.exec_seg_reduce_group      sim.py:139-165
 *   sgap_atomic_add_group sim.exec_atomic_add_group      sim.py:112-136
 *
 * Conventions: plain pointers and sizes; every pointer named d_* is device
 * memory, the caller owns all buffers, the library allocates nothing and
 * keeps no mutable global state (reentrant, one call per stream).  All work is
 * stream-ordered on the `stream` argument (a cudaStream_t passed as void*; NULL
 * is the legacy default stream).  Status codes mirror the reference's Python
 * exceptions (see sgap_status_t).
 */
#ifndef SGAP_H_
#define SGAP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGAP_ABI_VERSION 5

typedef enum {
    SGAP_OK = 0,
    SGAP_ERR_ILLEGAL_POINT = 1,   /* templates.IllegalPointError(rule)      */
    SGAP_ERR_NO_TEMPLATE = 2,     /* build_kernel -> None ("no_template")   */
    SGAP_ERR_SHAPE = 3,           /* sim.run ValueError: shape mismatch     */
    SGAP_ERR_PRECISION = 4,       /* sim.run ValueError: unknown precision  */
    SGAP_ERR_CUDA = 5,            /* CUDA runtime / launch failure          */
    SGAP_ERR_ARG = 6,             /* bad argument (null, misaligned, range) */
    SGAP_ERR_FAULT = 7,           /* sim.SimulationFault: group invariant   */
    SGAP_ERR_CONFIG = 8           /* lowering.LoweringError: KernelConfig   */
} sgap_status_t;

/* Template families (templates.py:46-58). */
typedef enum {
    SGAP_NNZ_MULTIPLE = 0,   /* nnz:g,col:c,r:1    EB + serial (TACO)        */
    SGAP_ROW_MULTIPLE = 1,   /* row:g,col:c,r:1    RB + serial               */
    SGAP_ROW_RECIPROCAL = 2, /* row:1/g,col:c,r:g  RB + parallel group       */
    SGAP_NNZ_ONE = 3         /* nnz:1,col:c,r      EB + segment (r>1) / atomic (r=1) */
} sgap_family_t;

typedef enum { SGAP_F32 = 0, SGAP_F64 = 1 } sgap_dtype_t;

/* A schedule point {<data, col>, r} (space.py:55-122). */
typedef enum { SGAP_KIND_NNZ = 0, SGAP_KIND_ROW = 1 } sgap_data_kind_t;
typedef enum { SGAP_AMT_RECIPROCAL = 0, SGAP_AMT_ONE = 1, SGAP_AMT_MULTIPLE = 2 } sgap_amount_kind_t;

typedef struct {
    int32_t data_kind;     /* sgap_data_kind_t                              */
    int32_t data_amount;   /* sgap_amount_kind_t                            */
    int32_t data_param;    /* g (>= 2) for 1/g or g; ignored for ONE         */
    int32_t col_amount;    /* sgap_amount_kind_t                            */
    int32_t col_param;     /* c (>= 2) for 1/c or c; ignored for ONE         */
    int32_t r;             /* group width r >= 1                             */
} sgap_point_t;

/* The lowered kernel: the reference's LoweredKernel integers (grid_size,
 * block_size, family, whether block_starts exist) plus the split factors the
 * device kernels need.  Filled by sgap_build_kernel; a caller that already
 * holds a reference LoweredKernel may fill it directly from its fields. */
typedef struct {
    int32_t family;         /* sgap_family_t                                 */
    int32_t n;              /* KernelConfig.n: dense width N                 */
    int32_t p;              /* KernelConfig.p: parallelism budget            */
    int32_t g;              /* data split factor (1 for ONE)                 */
    int32_t c;              /* column coarsening (1 for ONE)                 */
    int32_t r;              /* group width                                   */
    int64_t chunk;          /* units per logical block: nnz positions
                               (nnz-*), rows (row-multiple), fused (i,k)
                               cells (row-reciprocal)                        */
    int64_t grid_size;      /* == LoweredKernel.grid_size                    */
    int64_t block_size;     /* == LoweredKernel.block_size                   */
    int32_t has_block_starts; /* == (LoweredKernel.block_starts is not None) */
    int32_t hw_block;       /* CTA size override: 0 = auto (256; 128 for the
                               register EB walk), else a warp multiple in
                               [32, 256]                                    */
    int32_t hw_variant;     /* nnz-multiple walk: 0 auto, 1 register-staged
                               (row_ptr tracking when the plan has chunk
                               start rows), 5 register-staged on per-position
                               row ids, 9 = 1 with the plan's cold-column
                               cache hints (SGAP_PLAN_L2_HINTS) and the B
                               rows two batches ahead prefetched into L2
                               (for B far larger than L2), 10 = 1 in
                               column-panel order over the plan's
                               panel-major copy of B (SGAP_PLAN_PANELS: B
                               larger than L2, a panel fits half of it),
                               2 TMA-staged (cp.async.bulk + mbarrier ring),
                               3/4 lane-staged (warp per chunk, 4/8 B-row
                               gathers in flight; needs N/c >= 32).
                               row-multiple: 0/1 logical mapping, 2
                               interleaved rows, 3/4 interleaved + warp per
                               row, lane-staged A (N/c == 32; N/c a larger
                               multiple of 32: one pass per 32c-column
                               panel of B and C in place; N/c == 16 / 8 / 4 /
                               2: 2 / 4 / 8 / 16 rows per warp), 6/7 a
                               warp per 4/8-row block walking the union of
                               its columns (N/c == 32, rows <= 64), 8 a
                               warp per 4-row block: blocks whose rows are
                               shifted copies (row i0+r's columns = row
                               i0's + r, <= 32 each: banded / stencil rows)
                               gather each shared B row once, other blocks
                               take 4's walk; bit-identical to 4 (N/c a
                               multiple of 32, panels as 4; N/c == 16 / 8:
                               two / four 4-row lane groups per warp).
                               nnz-one: 0 the shuffle segment scan, 1 each
                               segment group walked serially by lanes along
                               the columns (same writebacks).
                               Other families: 0.                          */
} sgap_kernel_t;

/* CSR operand on the device (matrices.py:38-86 with int32 indices). */
typedef struct {
    int64_t num_rows;
    int64_t num_cols;
    int64_t nnz;
    const int32_t *d_row_ptr;  /* [num_rows + 1] */
    const int32_t *d_col_idx;  /* [nnz]          */
    const void *d_vals;        /* [nnz] float or double (sgap_dtype_t)      */
} sgap_csr_t;

int sgap_abi_version(void);
const char *sgap_status_string(int status);

/* space.legality_rule: 0 when legal, else the first rule (1..3) that fires. */
int sgap_legality_rule(const sgap_point_t *point);

/* runner.build_kernel without the LLIR: family selection, divisibility
 * gates, launch geometry.  Returns SGAP_OK, SGAP_ERR_ILLEGAL_POINT (rule in
 * *rule_out), SGAP_ERR_NO_TEMPLATE or SGAP_ERR_CONFIG (n < 1, p not a positive
 * warp multiple). */
int sgap_build_kernel(const sgap_point_t *point, int32_t n, int32_t p,
                      int64_t num_rows, int64_t nnz, sgap_kernel_t *out,
                      int32_t *rule_out);

/* lowering.compute_block_starts on the device: d_starts[b] (b = 0..num_blocks)
 * = last r in [0, num_rows] with row_ptr[r] <= b*chunk.  int32 output. */
int sgap_block_starts(const int32_t *d_row_ptr, int64_t num_rows, int64_t chunk,
                      int64_t num_blocks, int32_t *d_starts, void *stream);

/* Per-matrix side data of a kernel (what the reference's LoweredKernel
 * carries beyond its integers, plus the long-row table of this engine).
 * Filled by sgap_plan inside the caller's workspace and read by sgap_run;
 * callers never build it (ABI v4: sgap_run takes a plan, so the float64
 * long-row policy cannot be bypassed).  Field notes:
 *   d_block_starts: [grid_size + 1] from sgap_block_starts
 *     (LoweredKernel.block_starts, lowering.py:683-696); informational: the
 *     kernels use d_rowid instead of per-lane searches in its windows.
 *   d_rowid: [nnz] row owning each position (from sgap_row_ids), bit 31 set
 *     for rows of the long-row table; required for the nnz families.
 *   Long rows (float32 only, nnz families): rows with more than
 *   long_threshold nonzeros receive so many separate atomic flushes that a
 *   float32 running sum in C would exceed the 1e-5 accuracy bound; their
 *   flushes go to a float64 table d_long_acc [long_capacity x n] that
 *   sgap_run folds into C (and clears) after the kernel.  d_long_rows holds
 *   the sorted ids of those rows and d_long_count their number, both filled
 *   by sgap_prepare_long_rows.  long_threshold < 0 disables the table.
 *   long_chunk > 0 (nnz-multiple, = g): rows whose nonzeros straddle a
 *   g-position chunk boundary join the table too, so every split row is
 *   summed in float64 and the overwrite mode needs no zero-fill pre-pass.
 *   d_long_slot: [num_rows] table slot of each table row (other entries
 *   unused), filled by sgap_prepare_long_rows; NULL = search d_long_rows.     */
typedef struct {
    const int32_t *d_block_starts;
    const int32_t *d_rowid;
    int32_t *d_long_rows;
    int32_t *d_long_count;
    double *d_long_acc;
    int64_t long_capacity;
    int64_t long_threshold;
    int32_t has_exact_rows;   /* any row longer than sgap_exact_row_length()?
                                 (0 lets sgap_run skip the error-free pass)  */
    int32_t *d_long_slot;
    int64_t long_chunk;
    const int32_t *d_exact_rows;  /* rows with > max(long_threshold,
                                     sgap_exact_row_length()) nonzeros: the
                                     error-free pass walks exactly these    */
    int32_t exact_count;          /* their number (host-known: sizes the grid) */
    const int32_t *d_chunk_rows;  /* nnz-multiple, g % 4 == 0: [chunks + 1] row
                                     owning each g-chunk's first position
                                     (compute_block_starts at chunk g); the
                                     register walk then tracks rows through
                                     row_ptr instead of reading d_rowid     */
    const int32_t *d_union_off[2];  /* row-multiple, N/c == 32, rows <= 64:
                                        per 4-row [0] / 8-row [1] block, the
                                        offset of its union column stream   */
    const uint32_t *d_union[2];      /* (col | row mask << (32 - R)) entries:
                                        the row-blocked walk (hw variants
                                        6 / 7) gathers each shared B row once */
    const int32_t *d_col_hinted;    /* SGAP_PLAN_L2_HINTS, nnz-multiple: col_idx
                                        with bit 31 set on columns outside
                                        the hot set (the most-gathered
                                        columns whose B rows fill half the
                                        L2); hw variant 9 loads those rows
                                        with the evict-first streaming
                                        operator so the hot rows stay in L2 */
    void *d_panel_b;                /* SGAP_PLAN_PANELS (ABI v5): room for the
                                        panel-major copy of B that hw variant
                                        10 walks one column panel at a time */
    int32_t panel_lanes;            /* its panel width in c-wide column
                                        tiles (0: no panels for this plan)  */
} sgap_aux_t;

/* Per-position row ids (what the reference lowering recovers per lane with
 * binary_search_before over the block window plus a forward advance,
 * lowering.py:459-500), expanded once per matrix; bit 31 marks the rows of
 * the long-row table: longer than long_threshold (pass -1 for none) or, with
 * long_chunk > 0, straddling a long_chunk-position boundary.               */
int sgap_row_ids(const int32_t *d_row_ptr, int64_t num_rows, int64_t nnz,
                 int64_t long_threshold, int64_t long_chunk, int32_t *d_rowid,
                 void *stream);

/* Rows longer than this are accumulated error-free (float64 products of the
 * float32 inputs, summed in float64): float32 product rounding alone would
 * reach ~1e-5 of the reference metric on hub rows of ~2e4+ nonzeros.       */
int64_t sgap_exact_row_length(void);

/* Long-row threshold the planner uses for a kernel (-1: no table: row
 * families keep float64 running sums, float64 values accumulate in
 * float64).  Informational; sgap_plan applies it.                          */
int64_t sgap_long_row_threshold(const sgap_kernel_t *kernel, int32_t dtype);

/* ---- the planner (runner.build_kernel's per-matrix half, on the device) ---
 * A plan binds one kernel to one sparsity structure: block starts, per-
 * position row ids, the float64 long-row table and the error-free row list,
 * all in one caller-owned device workspace.  Values (d_vals), B and C may
 * change between runs; the structure (row_ptr / col_idx buffers and their
 * contents) must not -- sgap_run rejects a CSR whose shape or index buffers
 * differ from the planned ones (SGAP_ERR_SHAPE).
 *
 * sgap_plan runs on `stream` and synchronises it once to read back 24 bytes
 * of row statistics (longest row, number of table rows and of error-free
 * rows), which size the per-run launches.  It allocates nothing.            */
#define SGAP_PLAN_VALIDATE 1u     /* run sgap_validate_csr first            */
#define SGAP_PLAN_L2_HINTS 4u     /* nnz-multiple, g % 4 == 0: build the
                                     cold-column hints of hw variant 9 (a
                                     col_idx copy in the workspace; worth it
                                     when B is far larger than L2: config 5
                                     -4.8%, config 2 slower)                */
#define SGAP_PLAN_PANELS 8u       /* nnz-multiple, g % 4 == 0, B (num_cols x
                                     n) larger than the L2: reserve a copy of
                                     B in column panels of 8-32 c-wide tiles,
                                     the widest whose num_cols rows fit half
                                     the L2 (hw variant 10; config 3 at
                                     N = 256: 64-column panels).  Costs
                                     num_cols x n elements of workspace;
                                     nothing when no panel fits.           */
#define SGAP_PLAN_SPLIT_ROWS 2u   /* nnz-multiple, g >= 128: rows straddling a
                                     g-chunk boundary join the float64 table
                                     (no zero-fill pre-pass; measured slower
                                     on config 2, off by default)           */

typedef struct {
    int32_t abi;            /* SGAP_ABI_VERSION of the planner              */
    int32_t dtype;          /* sgap_dtype_t the plan was built for          */
    sgap_kernel_t kernel;   /* copy; hw_block / hw_variant may be changed
                               between runs, nothing else                  */
    int64_t num_rows, num_cols, nnz;
    const int32_t *d_row_ptr;  /* the planned structure (identity check)    */
    const int32_t *d_col_idx;
    int64_t longest_row;    /* max row length                               */
    int64_t table_rows;     /* rows in the float64 long-row table           */
    sgap_aux_t aux;         /* pointers into the workspace                  */
    void *d_workspace;
    size_t workspace_bytes;
} sgap_plan_t;

/* Workspace bytes sgap_plan needs for (kernel, A's shape, dtype, flags):
 * an upper bound from num_rows / nnz alone (no device access).             */
int sgap_plan_workspace_bytes(const sgap_kernel_t *kernel, const sgap_csr_t *a, int32_t dtype,
                              uint32_t flags, size_t *bytes);

/* Build the plan.  d_workspace: >= sgap_plan_workspace_bytes, 256-byte
 * aligned, owned by the caller and kept alive (unmodified) while the plan is
 * used.  Returns SGAP_ERR_FAULT (with SGAP_PLAN_VALIDATE) for a malformed
 * CSR, SGAP_ERR_ARG / SHAPE / PRECISION / CONFIG / CUDA otherwise.         */
int sgap_plan(const sgap_kernel_t *kernel, const sgap_csr_t *a, int32_t dtype, uint32_t flags,
              void *d_workspace, size_t workspace_bytes, sgap_plan_t *plan, void *stream);

/* The CsrMatrix invariants (matrices.py:58-75: row_ptr[0] == 0, row_ptr
 * non-decreasing, row_ptr[num_rows] == nnz, 0 <= col < num_cols, columns
 * strictly increasing within a row), checked on the device.  Returns SGAP_OK
 * or SGAP_ERR_FAULT; *fault_pos (may be NULL) receives the first offending
 * position: a row_ptr index r as -(r + 1), a col_idx position as itself.
 * d_scratch: 8 bytes of device memory.  Synchronises `stream`.            */
int sgap_validate_csr(const sgap_csr_t *a, void *d_scratch, int64_t *fault_pos, void *stream);

/* sim.run: C (+)= A @ B on the device with a plan from sgap_plan.
 *   a: the planned structure (same shape, row_ptr and col_idx buffers; vals
 *   may differ), values of plan->dtype.
 *   d_b: [a->num_cols x kernel.n] row-major, d_c: [a->num_rows x n] row-major,
 *   aligned to the kernel's column vector (c elements).
 *   accumulate = 1: C += A@B (c0 already in d_c, sim.py:439-441);
 *   accumulate = 0: C = A@B (d_c is overwritten; zero-fill included).
 *   d_writebacks: optional (NULL = off) device counter, incremented by the
 *   number of output writebacks (== SimMetrics.atomic_ops of the reference
 *   simulator for the same kernel; 0 for row-multiple).
 *   Launch-only: no allocation, no host synchronisation.                     */
int sgap_run(const sgap_plan_t *plan, const sgap_csr_t *a, const void *d_b, void *d_c,
             int32_t accumulate, unsigned long long *d_writebacks, void *stream);

/* The dgSPARSE RB+PR+RM kernel under the paper's fine-grained tuning knobs
 * (one cell of space.enumerate_fine_grained,
 * space.py:294-348): groupSz = the plan's g (row:1/g,col:c,r:g, coarsenSz =
 * c), blockSz = block (32..1024), tileSz = tile (a power of two >= g),
 * workerDimR = worker_scale x num_rows row workers.  Same reduction and
 * numerics as sgap_run on the plan (one G-lane group sum per row x column
 * vector, exclusive store); only the thread/block mapping differs.
 * blockDim.x = max(1, min(N, tile)/c) * g, blockDim.y = max(block,
 * 2 blockDim.x) / blockDim.x (<= 1024 threads).  The plan must be of the
 * row-reciprocal family.                                                    */
int sgap_run_rbpr_grid(const sgap_plan_t *plan, const sgap_csr_t *a, const void *d_b, void *d_c,
                       int32_t block, int32_t tile, double worker_scale, int32_t accumulate,
                       unsigned long long *d_writebacks, void *stream);

/* The dense reference product that runner.verify_point checks against
 * (runner.py:193-194 -> matrices.dense_spmm_oracle, matrices.py:241-254),
 * evaluated on the device: C[i,k] in float64, ascending-p accumulation with
 * separately rounded multiply and add, i.e. bit-identical to the reference
 * oracle on the same (widened) inputs.  d_c: [num_rows x n] float64.        */
int sgap_reference_spmm_f64(const sgap_csr_t *a, const void *d_b, int32_t n,
                            int32_t dtype, double *d_c, void *stream);

/* ---- Matrix Market ingest on the device -------------
 * Replaces the entry loop of matrices.loads_matrix_market
 * (matrices.py:144-212) and _coo_to_csr (matrices.py:124-141); the header and
 * any line outside the strict device grammar stay with the host (Python
 * int()/float()), so values, errors and line numbers are the reference's.
 *   sgap_mm_line_flags: d_flag[i] = 1 where a line starts (byte 0 and after
 *     each '\n'); *d_special |= 1 when str.splitlines()/split() would see
 *     separators a '\n' scan does not (lone '\r', control bytes, non-ASCII).
 *   sgap_mm_parse: per line d_status (0 blank/comment, 1 entry, 2 not three
 *     tokens, 3 non-numeric, 4 coordinate out of range, 5 the host checks
 *     the line, 6 entry whose plain-decimal value the host converts) and, for
 *     status 1 and 6, zero-based row/col, the value token's byte offset and
 *     length; for status 1 the value (correctly rounded: Clinger's fast path
 *     or Eisel-Lemire).  rows, cols <= INT32_MAX (SGAP_ERR_SHAPE otherwise:
 *     the sort keys pack row<<32|col).
 *   sgap_mm_expand: COO in the reference's append order at d_pos (exclusive
 *     scan of 1 per entry, 2 for symmetric off-diagonals), key = row<<32|col.
 *   sgap_mm_sum_runs: per run of equal keys in the stably sorted COO, the
 *     np.add.reduceat sum (first + numpy pairwise sum of the rest).
 *   sgap_mm_row_ptr: row_ptr[r] = lower bound of r in the sorted rows.      */
int sgap_mm_line_flags(const uint8_t *d_text, int64_t len, uint8_t *d_flag, int32_t *d_special,
                       void *stream);
int sgap_mm_parse(const uint8_t *d_text, int64_t len, const int64_t *d_starts, int64_t nlines,
                  int64_t rows, int64_t cols, uint8_t *d_status, int64_t *d_r, int64_t *d_c,
                  double *d_v, int64_t *d_tok_off, int32_t *d_tok_len, void *stream);
int sgap_mm_expand(int64_t nlines, const uint8_t *d_status, const int64_t *d_r, const int64_t *d_c,
                   const double *d_v, const int64_t *d_pos, int32_t symmetric, int64_t *d_key,
                   double *d_val, void *stream);
int sgap_mm_sum_runs(int64_t total, const int64_t *d_key, const double *d_val,
                     const int64_t *d_run_start, int64_t nruns, int64_t *d_row, int64_t *d_col,
                     double *d_out, void *stream);
int sgap_mm_row_ptr(const int64_t *d_row, int64_t nnz, int64_t num_rows, int64_t *d_row_ptr,
                    void *stream);

/* Device restatements of the simulator's group macros over lane vectors
 * (lanes = multiple of group_size, group_size in {1,2,4,8,16,32}).  They run
 * the same warp-shuffle code as the SpMM kernels.
 *   d_idx [lanes] int64, d_val [lanes] (dtype), d_active [lanes] uint8 (NULL =
 *   all active), d_out [out_len] (dtype, accumulated into),
 *   d_writebacks: counter (required), d_fault: int64 initialised by the caller
 *   to INT64_MAX; receives the smallest lane that violates the group invariant
 *   (diverging index / decreasing index), if any.                            */
int sgap_seg_reduce_group(const int64_t *d_idx, const void *d_val,
                          const uint8_t *d_active, int64_t lanes,
                          int32_t group_size, void *d_out, int64_t out_len,
                          int32_t dtype, unsigned long long *d_writebacks,
                          long long *d_fault, void *stream);
int sgap_atomic_add_group(const int64_t *d_idx, const void *d_val,
                          const uint8_t *d_active, int64_t lanes,
                          int32_t group_size, void *d_out, int64_t out_len,
                          int32_t dtype, unsigned long long *d_writebacks,
                          long long *d_fault, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SGAP_H_ */
