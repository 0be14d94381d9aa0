// sgap_kernels.cuh -- the four Sgap template families as sm_100a kernels.
//
// Each kernel keeps the reference family's work decomposition -- which
// positions/rows/cells form one reduction, which lanes reduce together, where
// a writeback happens (so SimMetrics.atomic_ops is reproduced exactly) -- and
// chooses its own hardware lane mapping: lanes run along the dense columns in
// c-wide vectors wherever the family allows it, so a B-row gather and a C-row
// writeback are one coalesced request per warp.
//
// Reference (paths relative to /root/reference/pkg/src/spmmlab/):
//   k_row_multiple     row:g,col:c,r:1     templates.py:137-154, lowering.py:416-420,573-585,643-646
//   k_row_reciprocal   row:1/g,col:c,r:g   templates.py:157-177, lowering.py:427-439,587-624
//   k_nnz_one          nnz:1,col:c,r       templates.py:180-202, lowering.py:459-488,526-537,626-642
//   k_nnz_multiple     nnz:g,col:c,r:1     templates.py:114-134, lowering.py:490-500,539-571
#pragma once

#include "sgap_device.cuh"

namespace sgap {

// Warp-uniform grid-stride iteration over warp work items.
#define SGAP_WARP_LOOP(item, items)                                                     \
    for (long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;     \
         item < (items); item += ((long long)gridDim.x * blockDim.x) >> 5)

constexpr int kBatch = 4;     // independent gathers kept in flight per lane
constexpr int kFoldEvery = 8;  // float32 partial sums fold into float64 every 8 terms
#ifndef SGAP_EB_MINB
#define SGAP_EB_MINB 4  // CTAs per SM the register EB walk is compiled for
// (5 / 6: 48 / 40 registers with 450-900 B of spills; config 2 1.03 / 1.36 ms,
// config 3 3.30 / 4.22 ms, against 0.711 / 2.13 ms at 4 and 64 registers;
// 3: 0.827 / 2.53 ms -- fewer warps lose more than the extra registers give)
#endif

// ===========================================================================
// RB + serial reduction: row:g,col:c,r:1 (row-multiple).
// Logical thread (rg, t): rows rg*g .. rg*g+g-1, columns t*c .. t*c+c-1,
// serial dot product over each row, one plain store per (row, tile)
// (cuda_row_multiple.cu:37-43).  Hardware: L = N/c consecutive lanes share a
// row (the logical mapping itself); each lane walks the row with broadcast
// loads -- one 16-byte load each of 4 (col) and 4 (val) once the walk is
// 4-aligned -- keeping 4 B-row gathers in flight, float32 partials folded into
// a float64 running sum every 8 terms; C is written once with st.global.cs
// (no atomics, no zero-fill, deterministic).
// ===========================================================================
template <typename T, int V>
__device__ __forceinline__ void rb_step(Vec<T, V> &acc, const int *__restrict__ ci,
                                        const T *__restrict__ av, int p,
                                        const T *__restrict__ bk, int N) {
    Vec<T, V> b;
    ldg_vec<T, V>(b, row_ptr(bk, __ldg(ci + p), N));
    fma_vec<T, V>(acc, __ldg(av + p), b);
}

// Dot product of one row with one column tile (float64 result).
template <typename T, int V, bool EXACT>
__device__ __forceinline__ Vec<double, V> rb_row_impl(const int *__restrict__ ci,
                                                      const T *__restrict__ av, int p, int end,
                                                      const T *__restrict__ bk, int N,
                                                      bool vec4) {
    Vec<T, V> acc;
    acc.zero();
    Vec<double, V> tot;
    tot.zero();
    int since_fold = 0;
    auto step = [&](T a, const Vec<T, V> &b) {
        if constexpr (EXACT) {  // float64 products of float32 inputs are exact
#pragma unroll
            for (int x = 0; x < V; ++x) tot.v[x] = fma((double)a, (double)b.v[x], tot.v[x]);
        } else {
            fma_vec<T, V>(acc, a, b);
        }
    };
    auto one = [&](int q) {
        Vec<T, V> b;
        ldg_vec<T, V>(b, row_ptr(bk, __ldg(ci + q), N));
        step(__ldg(av + q), b);
    };
    if (vec4) {
        for (; p < end && (p & 3); ++p) one(p);
        for (; p + 4 <= end; p += 4) {
            const int4 c = __ldg(reinterpret_cast<const int4 *>(ci + p));
            Vec<T, 4> v;
            ldg_vec<T, 4>(v, av + p);
            Vec<T, V> b0, b1, b2, b3;
            ldg_vec<T, V>(b0, row_ptr(bk, c.x, N));
            ldg_vec<T, V>(b1, row_ptr(bk, c.y, N));
            ldg_vec<T, V>(b2, row_ptr(bk, c.z, N));
            ldg_vec<T, V>(b3, row_ptr(bk, c.w, N));
            step(v.v[0], b0);
            step(v.v[1], b1);
            step(v.v[2], b2);
            step(v.v[3], b3);
            since_fold += 4;
            if (since_fold >= kFoldEvery) {
                fold<T, V>(tot, acc);
                since_fold = 0;
            }
        }
    } else {
        for (; p + 4 <= end; p += 4) {
            one(p);
            one(p + 1);
            one(p + 2);
            one(p + 3);
            since_fold += 4;
            if (since_fold >= kFoldEvery) {
                fold<T, V>(tot, acc);
                since_fold = 0;
            }
        }
    }
    for (; p < end; ++p) one(p);
    fold<T, V>(tot, acc);
    return tot;
}

template <typename T, int V>
__device__ __forceinline__ Vec<double, V> rb_row(const int *__restrict__ ci,
                                                 const T *__restrict__ av, int p, int end,
                                                 const T *__restrict__ bk, int N, bool vec4) {
    if (sizeof(T) == 4 && end - p > kExactRow)
        return rb_row_impl<T, V, true>(ci, av, p, end, bk, N, vec4);
    return rb_row_impl<T, V, false>(ci, av, p, end, bk, N, vec4);
}

template <typename T, int V>
__global__ void __launch_bounds__(256, 4)
k_row_multiple(const int *__restrict__ rp, const int *__restrict__ ci,
               const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C,
               int M, int N, int g, int vec4, int accumulate) {
    const int L = N / V;
    const Divider byL = Divider::make(L);
    const long long groups = ((long long)M + g - 1) / g;
    const long long total = groups * L;  // logical threads
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < total;
         h += (long long)gridDim.x * blockDim.x) {
        const long long rg = byL.div(h);
        const int t = (int)(h - rg * L);
        const long long kcol = (long long)t * V;
        for (int s = 0; s < g; ++s) {
            const long long i = rg * g + s;
            if (i >= M) break;
            const Vec<double, V> tot = rb_row<T, V>(ci, av, __ldg(rp + i), __ldg(rp + i + 1),
                                                    B + kcol, N, vec4 != 0);
            store_vec<T, V>(C + i * N + kcol, narrow<T, V>(tot), accumulate != 0);
        }
    }
}

// The same logical threads on an interleaved mapping: a CTA owns a tile of
// (rows_per_step x g) consecutive rows and, at each of its g steps, its
// warps work on *adjacent* rows.  Rows i, i+1, ... of banded / mesh matrices
// gather mostly the same B rows, so a step's working set (a few dozen B rows
// per CTA) is served from L1, while tiles still go out in global row order so
// the chip-wide sweep keeps its L2 reuse.  (A persistent band per CTA was
// measured: L1 hit 63% but 592 separate sweep fronts broke L2 reuse, 19.6 GB
// of DRAM reads on config 4.)  Output and numerics are identical to
// k_row_multiple: each row is one serial dot product per column tile.
template <typename T, int V>
__global__ void __launch_bounds__(256, 4)
k_row_interleaved(const int *__restrict__ rp, const int *__restrict__ ci,
                  const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C, int M,
                  int N, int g, int vec4, int accumulate) {
    const int L = N / V;
    const int rows_per_step = blockDim.x / L;
    if ((int)threadIdx.x >= rows_per_step * L) return;
    const int t = (int)(threadIdx.x % L);
    const int slot = (int)(threadIdx.x / L);
    const long long kcol = (long long)t * V;
    const long long tile_rows = (long long)rows_per_step * g;
    const long long tiles = ((long long)M + tile_rows - 1) / tile_rows;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int s = 0; s < g; ++s) {
            const long long i = tile * tile_rows + (long long)s * rows_per_step + slot;
            if (i >= M) break;
            const Vec<double, V> tot = rb_row<T, V>(ci, av, __ldg(rp + i), __ldg(rp + i + 1),
                                                    B + kcol, N, vec4 != 0);
            store_vec<T, V>(C + i * N + kcol, narrow<T, V>(tot), accumulate != 0);
        }
    }
}

// The interleaved mapping with a whole warp per row (hw variant 3, N/c == 32):
// per 32 positions each lane loads one position's (col, val) -- one coalesced
// request per array instead of per-lane broadcast loads with an alignment
// prologue and a tail -- and U B-row gathers go out back to back from
// shuffled columns.  A short tail group re-gathers a valid column and skips
// its FMAs.  Each (row, tile) is still one serial sum in position order: in
// float32 for rows of <= 64 nonzeros (stencil rows: 27), folded into float64
// every 32 positions beyond that, error-free past kExactRow (rb_row).
// ncu on config 4 (27-pt stencil, N=128) for the broadcast walk: 24.5 warp
// instructions per nonzero, 47% warps active, long-scoreboard 62%.
template <typename T, int V, int U>
__device__ __forceinline__ Vec<double, V> rb_row_staged(const int *__restrict__ ci,
                                                        const T *__restrict__ av, int beg,
                                                        int end, const T *__restrict__ bk,
                                                        int N) {
    const unsigned lane = lane_id();
    Vec<T, V> acc;
    acc.zero();
    Vec<double, V> tot;
    tot.zero();
    const bool longrow = end - beg > 64;
    for (int s = beg; s < end; s += 32) {
        const int q = s + (int)lane;
        const int c_l = q < end ? __ldg(ci + q) : __ldg(ci + s);
        const T v_l = q < end ? __ldg(av + q) : T(0);
        const int nv = min(32, end - s);
        for (int j = 0; j < nv; j += U) {
            Vec<T, V> b[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                gather_vec<T, V>(b[u], row_ptr(bk, __shfl_sync(kFull, c_l, (j + u) & 31), N));
            if (j + U <= nv) {
#pragma unroll
                for (int u = 0; u < U; ++u) fma_vec<T, V>(acc, __shfl_sync(kFull, v_l, j + u), b[u]);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const T v = __shfl_sync(kFull, v_l, (j + u) & 31);
                    if (j + u < nv) fma_vec<T, V>(acc, v, b[u]);
                }
            }
        }
        if (longrow) fold<T, V>(tot, acc);
    }
    fold<T, V>(tot, acc);
    return tot;
}

// Rows of <= 64 nonzeros: the float32 walk alone (no float64 state live, so
// the kernel keeps few registers and many warps); longer rows go through a
// call so their float64 state does not set the kernel's register count.
template <typename T, int V, int U>
__device__ __forceinline__ Vec<T, V> rb_short_staged(const int *__restrict__ ci,
                                                     const T *__restrict__ av, int beg, int end,
                                                     const T *__restrict__ bk, int N) {
    const unsigned lane = lane_id();
    Vec<T, V> acc;
    acc.zero();
    for (int s = beg; s < end; s += 32) {
        const int q = s + (int)lane;
        const int c_l = q < end ? __ldg(ci + q) : __ldg(ci + s);
        const T v_l = q < end ? __ldg(av + q) : T(0);
        const int nv = min(32, end - s);
        for (int j = 0; j < nv; j += U) {
            Vec<T, V> b[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                gather_vec<T, V>(b[u], row_ptr(bk, __shfl_sync(kFull, c_l, (j + u) & 31), N));
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const T v = __shfl_sync(kFull, v_l, (j + u) & 31);
                if (j + u < nv) fma_vec<T, V>(acc, v, b[u]);
            }
        }
    }
    return acc;
}

template <typename T, int V, int U>
__device__ __noinline__ void rb_long_staged(const int *__restrict__ ci, const T *__restrict__ av,
                                            int beg, int end, const T *__restrict__ bk, int N,
                                            int vec4, T *__restrict__ out, int accumulate) {
    const Vec<double, V> tot = (sizeof(T) == 4 && end - beg > kExactRow)
                                   ? rb_row<T, V>(ci, av, beg, end, bk, N, vec4 != 0)
                                   : rb_row_staged<T, V, U>(ci, av, beg, end, bk, N);
    store_vec<T, V>(out, narrow<T, V>(tot), accumulate != 0);
}

template <typename T, int V, int U>
__global__ void __launch_bounds__(256, U >= 8 ? 4 : 5)
k_row_staged(const int *__restrict__ rp, const int *__restrict__ ci, const T *__restrict__ av,
             const T *__restrict__ B, T *__restrict__ C, int M, int N, int g, int vec4,
             int accumulate, int min_len) {
    // Measured and not kept on config 4 (N=128, 3.26 ms here):
    // software-pipelining a warp's rows (next row's bounds and (col, val)
    // under this row's gathers): 3.41 ms; a 32-register walk for rows <= 32
    // at 56 warps/SM plus a second launch for longer rows: 3.50 ms; a warp
    // per row PAIR gathering the B rows the two rows share once (1/3 fewer
    // gathers on the stencil, columns matched by shuffle binary search):
    // 3.13 ms, no gain -- the walk is latency-chained, not L1-bound.
    const int warps = (int)(blockDim.x >> 5);
    const int w = (int)(threadIdx.x >> 5);
    const long long kcol = (long long)lane_id() * V;
    const long long tile_rows = (long long)warps * g;
    const long long tiles = ((long long)M + tile_rows - 1) / tile_rows;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int s = 0; s < g; ++s) {
            const long long i = tile * tile_rows + (long long)s * warps + w;
            if (i >= M) break;
            const int beg = __ldg(rp + i), end = __ldg(rp + i + 1);
            if (end - beg <= min_len) continue;  // rows another launch took (min_len < 0: none)
            if (end - beg > 64) {
                rb_long_staged<T, V, U>(ci, av, beg, end, B + kcol, N, vec4, C + i * N + kcol,
                                        accumulate);
            } else {
                store_vec<T, V>(C + i * N + kcol,
                                rb_short_staged<T, V, U>(ci, av, beg, end, B + kcol, N),
                                accumulate != 0);
            }
        }
    }
}

// The warp-per-row walk for N/c = 16 or 8 (hw variants 3/4 at N = 64 / 32
// with c = 4): LPR = N/c lanes per row, 32/LPR adjacent rows per warp, each
// row's (col, val) lane-staged LPR positions at a time and shuffled within
// its LPR-lane segment, U B-row gathers in flight per lane.  The rows of a
// warp share the trip count of the longest one (the shuffles need the whole
// warp converged); shorter rows gather a valid row and skip the FMA.  Rows of
// <= 64 nonzeros sum in float32 (as rb_short_staged); a warp holding a longer
// row walks its rows per lane with rb_row (float64 sums / error-free).
template <typename T, int V, int U, int LPR>
__global__ void __launch_bounds__(256, 5)
k_row_staged_sub(const int *__restrict__ rp, const int *__restrict__ ci,
                 const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C, int M,
                 int N, int g, int vec4, int accumulate) {
    constexpr int RPW = 32 / LPR;  // rows per warp
    const int warps = (int)(blockDim.x >> 5);
    const int w = (int)(threadIdx.x >> 5);
    const unsigned lane = lane_id();
    const int sub = (int)(lane % LPR), slot = (int)(lane / LPR);
    const long long kcol = (long long)sub * V;
    const T *bk = B + kcol;
    const long long tile_rows = (long long)warps * g * RPW;
    const long long tiles = ((long long)M + tile_rows - 1) / tile_rows;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int s = 0; s < g; ++s) {
            const long long i0 = tile * tile_rows + ((long long)s * warps + w) * RPW;
            if (i0 >= M) break;  // warp-uniform
            const long long i = i0 + slot;
            const bool ok = i < M;
            const int beg = ok ? __ldg(rp + i) : 0, end = ok ? __ldg(rp + i + 1) : 0;
            const int len = end - beg;
            const int maxlen = __reduce_max_sync(kFull, len);
            if (maxlen > 64) {  // a long row in this warp's group: per-lane walks
                if (ok)
                    store_vec<T, V>(C + i * N + kcol,
                                    narrow<T, V>(rb_row<T, V>(ci, av, beg, end, bk, N, vec4 != 0)),
                                    accumulate != 0);
                continue;
            }
            Vec<T, V> acc;
            acc.zero();
            for (int s0 = 0; s0 < maxlen; s0 += LPR) {
                const bool in = s0 + sub < len;
                const int c_l = in ? __ldg(ci + beg + s0 + sub) : 0;  // column 0: a valid B row
                const T v_l = in ? __ldg(av + beg + s0 + sub) : T(0);
                const int nv = min(LPR, maxlen - s0);
                for (int j = 0; j < nv; j += U) {
                    Vec<T, V> b[U];
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        gather_vec<T, V>(b[u], row_ptr(bk, __shfl_sync(kFull, c_l, (j + u) & (LPR - 1), LPR), N));
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const T v = __shfl_sync(kFull, v_l, (j + u) & (LPR - 1), LPR);
                        if (j + u < nv && s0 + j + u < len) fma_vec<T, V>(acc, v, b[u]);
                    }
                }
            }
            if (ok) store_vec<T, V>(C + i * N + kcol, acc, accumulate != 0);
        }
    }
}

// ===========================================================================
// Shifted-block RB walk (row-multiple hw variant 8: R = 4 rows per warp,
// N/c == 32, once per 32c-column panel for larger multiples of 32).
// A block of R consecutive rows is "shifted" when every row has the same
// length L <= 32 and row i0+r's column list is row i0's plus r -- the rows of
// a banded / stencil matrix away from the grid edges (27-point stencil: 9
// runs of 3 consecutive columns per row).  Row i0's list is cut into pieces
// of w <= 3 consecutive columns; a piece starting at column cb is needed by
// the block's rows as B rows cb .. cb + R + w - 2, so the warp gathers those
// R + w - 1 rows once and each feeds up to w rows' sums (stencil: 90 B-row
// gathers per 8 rows instead of 216, every FMA useful -- no masks, no zero
// padding).  The values stay in the CSR: lane p holds position p of each of
// the R rows (R coalesced loads) and shuffles it to the FMA.  Each row still
// sums its own nonzeros serially in CSR order in float32, exactly as the
// warp-per-row walk's rb_short_staged does (lowering.py:573-585), so the
// results are bit-identical to hw variant 4 and the writebacks are one per
// (row, tile).  Blocks that are not shifted (grid edges, irregular rows,
// rows > 32) take the warp-per-row walk inline.  The property is checked per
// block from the column stream the walk reads anyway: no plan data.
// Config 4 (N = 128): 2.06 vs 3.07 ms for the warp-per-row walk; ncu: 1.24G
// instructions (from 2.09G), L2->L1 sectors unchanged (764M: the x-neighbour
// reuse moved from L1 to registers), long-scoreboard bound.  Measured and not
// kept (config 4, N = 128/256): R = 8 (124 registers, 2 CTAs/SM) 1.5-1.6x
// slower; two 3-wide pieces gathered back to back (2(R + 2) rows in flight,
// 80 registers) 1.03-1.17x slower; 48 registers for 5 CTAs/SM: spills, 1.5x
// slower; the next piece's B rows prefetched into L1 under this piece's
// gathers: 1.09x slower.
// ===========================================================================
template <typename T, int V, int R, int W, bool SMEM>
__device__ __forceinline__ void shifted_piece(Vec<T, V> (&acc)[R], const T (&v)[R], int p,
                                              const T *__restrict__ bk, int cb, int N,
                                              const T *slab) {
    Vec<T, V> b[R + W - 1];
#pragma unroll
    for (int q = 0; q < R + W - 1; ++q) gather_vec<T, V>(b[q], row_ptr(bk, cb + q, N));
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            if constexpr (SMEM)
                fma_vec<T, V>(acc[r], slab[r * 33 + p + j], b[r + j]);
            else
                fma_vec<T, V>(acc[r], __shfl_sync(kFull, v[r], p + j), b[r + j]);
        }
    }
}

template <typename T, int V, int R, bool SMEM = false>
__global__ void __launch_bounds__(256, 4)
k_row_shifted(const int *__restrict__ rp, const int *__restrict__ ci, const T *__restrict__ av,
              const T *__restrict__ B, T *__restrict__ C, int M, int N, int vec4,
              int accumulate) {
    const int warps = (int)(blockDim.x >> 5);
    const unsigned lane = lane_id();
    const long long kcol = (long long)lane * V;
    const T *bk = B + kcol;
    const long long nblocks = ((long long)M + R - 1) / R;
    extern __shared__ __align__(16) unsigned char shifted_raw[];
    T *slab = reinterpret_cast<T *>(shifted_raw) + (size_t)(threadIdx.x >> 5) * R * 33;
    for (long long blk = (long long)blockIdx.x * warps + (threadIdx.x >> 5); blk < nblocks;
         blk += (long long)gridDim.x * warps) {
        const long long i0 = blk * R;
        // lanes 0..R: the block's row starts (one load)
        const int t = (int)lane <= R ? __ldg(rp + (i0 + lane < M ? i0 + lane : (long long)M)) : 0;
        const int p0 = __shfl_sync(kFull, t, 0);
        const int L = __shfl_sync(kFull, t, 1) - p0;
        const int nxt = __shfl_down_sync(kFull, t, 1);
        bool ok = i0 + R <= M && L >= 1 && L <= 32 &&
                  __all_sync(kFull, (int)lane >= R || nxt - t == L);
        int c0 = 0;
        T v[R];
        if (ok) {
            const bool in = (int)lane < L;
            c0 = in ? __ldg(ci + p0 + lane) : 0;
            bool sh = true;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int q = p0 + r * L + (int)lane;
                v[r] = in ? __ldg(av + q) : T(0);
                if (r > 0 && in) sh = sh && __ldg(ci + q) == c0 + r;
            }
            ok = __all_sync(kFull, sh);
        }
        if (!ok) {  // the warp-per-row walk (hw variant 4) for this block
#pragma unroll 1
            for (int r = 0; r < R; ++r) {
                const long long i = i0 + r;
                if (i >= M) break;
                const int beg = __shfl_sync(kFull, t, r), end = __shfl_sync(kFull, t, r + 1);
                if (end - beg > 64)
                    rb_long_staged<T, V, 4>(ci, av, beg, end, bk, N, vec4, C + i * N + kcol,
                                            accumulate);
                else
                    store_vec<T, V>(C + i * N + kcol,
                                    rb_short_staged<T, V, 4>(ci, av, beg, end, bk, N),
                                    accumulate != 0);
            }
            continue;
        }
        if constexpr (SMEM) {  // the block's values in the warp's shared slab
            __syncwarp();          // (broadcast reads; the previous block's are done)
            if ((int)lane < L) {
#pragma unroll
                for (int r = 0; r < R; ++r) slab[r * 33 + (int)lane] = v[r];
            }
            __syncwarp();
        }
        // bit p: column p of row i0 continues column p - 1 (runs of consecutive columns)
        const int up = __shfl_up_sync(kFull, c0, 1);
        const unsigned long long cont =
            __ballot_sync(kFull, lane > 0 && (int)lane < L && c0 == up + 1);
        Vec<T, V> acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r].zero();
        for (int p = 0; p < L;) {
            const int cb = __shfl_sync(kFull, c0, p);
            const int w = ((cont >> (p + 1)) & 1ull) ? (((cont >> (p + 2)) & 1ull) ? 3 : 2) : 1;
            if (w == 3)
                shifted_piece<T, V, R, 3, SMEM>(acc, v, p, bk, cb, N, slab);
            else if (w == 2)
                shifted_piece<T, V, R, 2, SMEM>(acc, v, p, bk, cb, N, slab);
            else
                shifted_piece<T, V, R, 1, SMEM>(acc, v, p, bk, cb, N, slab);
            p += w;
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            store_vec<T, V>(C + (i0 + r) * (long long)N + kcol, acc[r], accumulate != 0);
    }
}

// Shifted-block walk for N/c = LPR = 16 (hw variant 8 at N = 64 with c = 4):
// G = 32 / LPR lane groups of LPR lanes, each owning 4 consecutive rows of
// an 8-row warp block (config 4 N=64: 1.40 vs 1.61 ms for variant 4; LPR = 8
// was 1.33x / 1.38x slower with R = 4 / 2 rows per group: the slot-indexed
// staged values land in local memory at 64 registers).  When the whole warp block is shifted
// (as k_row_shifted checks it), every group walks the same pieces of row
// i0's column list -- group g's piece starts at column cb + 4g -- gathering
// 3 + w LPR-lane B rows per piece for its 4 rows.  Lane (g, l) keeps
// positions l, l + LPR, ... of its group's rows (32 / LPR slots; the slot of
// a position is warp-uniform) and serves them with LPR-wide shuffles.  Other
// warp blocks run k_row_staged_sub's walk (4 rounds of G rows), so C is
// bit-identical to hw variant 4 at the same N/c.
template <typename T, int V, int LPR, int R, bool SMEM = false>
__global__ void __launch_bounds__(256, 4)
k_row_shifted_sub(const int *__restrict__ rp, const int *__restrict__ ci,
                  const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C, int M,
                  int N, int vec4, int accumulate) {
    constexpr int G = 32 / LPR;  // lane groups per warp
    constexpr int S = 32 / LPR;  // staged slots per lane (L <= 32)
    constexpr int RB = R * G;    // rows per warp block (R rows per lane group)
    constexpr int U = 4;
    const int warps = (int)(blockDim.x >> 5);
    const unsigned lane = lane_id();
    const int sub = (int)(lane % LPR), grp = (int)(lane / LPR);
    const long long kcol = (long long)sub * V;
    const T *bk = B + kcol;
    const long long nblocks = ((long long)M + RB - 1) / RB;
    extern __shared__ __align__(16) unsigned char shifted_raw[];
    T *slab = reinterpret_cast<T *>(shifted_raw) + (size_t)(threadIdx.x >> 5) * RB * 33;
    (void)slab;
    for (long long blk = (long long)blockIdx.x * warps + (threadIdx.x >> 5); blk < nblocks;
         blk += (long long)gridDim.x * warps) {
        const long long i0 = blk * RB;
        const int t = (int)lane <= RB ? __ldg(rp + (i0 + lane < M ? i0 + lane : (long long)M)) : 0;
        const int p0 = __shfl_sync(kFull, t, 0);
        const int L = __shfl_sync(kFull, t, 1) - p0;
        const int nxt = __shfl_down_sync(kFull, t, 1);
        bool ok = i0 + RB <= M && L >= 1 && L <= 32 &&
                  __all_sync(kFull, (int)lane >= RB || nxt - t == L);
        int c0 = 0;
        if (ok) {
            const bool in = (int)lane < L;
            c0 = in ? __ldg(ci + p0 + lane) : 0;
            bool sh = true;
#pragma unroll 4
            for (int r = 1; r < RB; ++r)
                if (in) sh = sh && __ldg(ci + p0 + r * L + (int)lane) == c0 + r;
            ok = __all_sync(kFull, sh);
        }
        if (!ok) {  // k_row_staged_sub's walk: 4 rounds of G adjacent rows (one per
                    // group, paired as that kernel pairs them: a round whose
                    // longest row exceeds 64 walks all its rows in float64)
#pragma unroll 1
            for (int k = 0; k < R; ++k) {
                const long long i = i0 + G * k + grp;
                const bool in = i < M;
                const int beg = in ? __ldg(rp + i) : 0, end = in ? __ldg(rp + i + 1) : 0;
                const int len = end - beg;
                const int maxlen = __reduce_max_sync(kFull, len);
                if (maxlen > 64) {
                    if (in)
                        store_vec<T, V>(C + i * N + kcol,
                                        narrow<T, V>(rb_row<T, V>(ci, av, beg, end, bk, N, vec4 != 0)),
                                        accumulate != 0);
                    continue;
                }
                Vec<T, V> a1;
                a1.zero();
                for (int s0 = 0; s0 < maxlen; s0 += LPR) {
                    const bool q = s0 + sub < len;
                    const int c_l = q ? __ldg(ci + beg + s0 + sub) : 0;
                    const T v_l = q ? __ldg(av + beg + s0 + sub) : T(0);
                    const int nv = min(LPR, maxlen - s0);
                    for (int j = 0; j < nv; j += U) {
                        Vec<T, V> b[U];
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            gather_vec<T, V>(b[u], row_ptr(bk, __shfl_sync(kFull, c_l, (j + u) & (LPR - 1), LPR), N));
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const T v = __shfl_sync(kFull, v_l, (j + u) & (LPR - 1), LPR);
                            if (j + u < nv && s0 + j + u < len) fma_vec<T, V>(a1, v, b[u]);
                        }
                    }
                }
                if (in) store_vec<T, V>(C + i * N + kcol, a1, accumulate != 0);
            }
            continue;
        }
        // group grp's rows i0 + R grp + r: positions sub + LPR s in slot s
        // (SMEM, the launched form: the warp's block in a shared slab of RB
        // rows x 33 values, padded so the groups' rows fall in different
        // banks; the register form measured 0.89-0.95x slower)
        T v[SMEM ? 1 : R][SMEM ? 1 : S];
        if constexpr (SMEM) {
            __syncwarp();  // the previous block's readers are done
            if ((int)lane < L) {
#pragma unroll 4
                for (int rr = 0; rr < RB; ++rr) slab[rr * 33 + (int)lane] = __ldg(av + p0 + rr * L + (int)lane);
            }
            __syncwarp();
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int pos = sub + LPR * s;
                    v[r][s] = pos < L ? __ldg(av + p0 + (R * grp + r) * L + pos) : T(0);
                }
        }
        const int up = __shfl_up_sync(kFull, c0, 1);
        const unsigned long long cont =
            __ballot_sync(kFull, lane > 0 && (int)lane < L && c0 == up + 1);
        Vec<T, V> acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r].zero();
        for (int p = 0; p < L;) {
            const int cb = __shfl_sync(kFull, c0, p) + R * grp;
            const int w = ((cont >> (p + 1)) & 1ull) ? (((cont >> (p + 2)) & 1ull) ? 3 : 2) : 1;
            Vec<T, V> b[R + 2];
#pragma unroll
            for (int q = 0; q < R + 2; ++q)
                if (q < R - 1 + w) gather_vec<T, V>(b[q], row_ptr(bk, cb + q, N));
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    if (j < w) {
                        const int pos = p + j;
                        if constexpr (SMEM) {
                            fma_vec<T, V>(acc[r], slab[(R * grp + r) * 33 + pos], b[r + j]);
                        } else {
                            T x = v[r][0];
#pragma unroll
                            for (int s = 1; s < S; ++s)
                                if (pos / LPR == s) x = v[r][s];
                            fma_vec<T, V>(acc[r], __shfl_sync(kFull, x, pos & (LPR - 1), LPR), b[r + j]);
                        }
                    }
                }
            }
            p += w;
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            store_vec<T, V>(C + (i0 + R * grp + r) * (long long)N + kcol, acc[r], accumulate != 0);
    }
}

// ===========================================================================
// Row-blocked RB walk (row-multiple hw variants 6 / 7, N/c == 32): a warp
// owns R consecutive rows and walks the UNION of their column lists once --
// a plan-time stream of (col | row-mask << (32 - R)) entries per R-row block,
// built by k_union_rows -- so a B row shared by several rows of the block is
// gathered once and feeds every row whose mask bit is set (stencils and
// meshes: adjacent rows share 2/3 of their columns).  Each row still sums its
// own nonzeros in ascending position order (the union is sorted, a row's
// entries appear in its CSR order and its values are read from its own
// position cursor), one serial sum per (row, tile) as the reference's
// row-multiple thread does (lowering.py:573-585); rows are at most 64 long
// (float32 sums, as rb_short_staged), which the plan checks.
// ===========================================================================
template <int R>
struct UnionFmt {
    static constexpr int kShift = 32 - R;
    static constexpr unsigned kColMask = (1u << kShift) - 1u;
};

// Per block of R rows: the number of distinct columns (pass 0) or the
// entries themselves (pass 1) -- an R-way merge of the sorted row lists by
// one thread per block.
template <int R>
__global__ void __launch_bounds__(256)
k_union_rows(const int *__restrict__ rp, const int *__restrict__ ci, int M, long long nblocks,
             const int *__restrict__ off, int *__restrict__ out_count,
             unsigned *__restrict__ out_entries) {
    for (long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks;
         b += (long long)gridDim.x * blockDim.x) {
        const long long i0 = b * R;
        int p[R], e[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool ok = i0 + r < M;
            p[r] = ok ? __ldg(rp + i0 + r) : 0;
            e[r] = ok ? __ldg(rp + i0 + r + 1) : 0;
        }
        long long w = off ? off[b] : 0;
        int count = 0;
        for (;;) {
            int best = INT_MAX;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (p[r] < e[r]) best = min(best, __ldg(ci + p[r]));
            if (best == INT_MAX) break;
            unsigned mask = 0;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (p[r] < e[r] && __ldg(ci + p[r]) == best) {
                    mask |= 1u << r;
                    ++p[r];
                }
            if (out_entries) out_entries[w++] = (unsigned)best | (mask << UnionFmt<R>::kShift);
            ++count;
        }
        if (out_count) out_count[b] = count;
    }
}

// Values: a window of 32 union entries is staged once per warp -- lane e
// holds entry e and fetches, for every row r whose mask bit it carries, that
// row's value at the row's next position (rank of e among the window's
// entries of row r, by ballot + popc; consecutive lanes of one row read
// consecutive positions, so the R loads are coalesced) -- and parks its R
// values in the warp's shared slab.  The walk then reads one R-wide vector
// per entry (a broadcast LDS) instead of one dependent scalar load per
// position, and FMAs only the rows whose mask bit is set (no 0 * inf).
// (Round-2 first cut loaded each value with a per-(entry, row) predicated
// __ldg and measured 1.18x slower than the warp-per-row walk.)
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <typename T, int R>
__device__ __forceinline__ void sv_store(T *p, const T (&v)[R]) {
    if constexpr (sizeof(T) * R % 16 == 0) {
#pragma unroll
        for (int q = 0; q < (int)(sizeof(T) * R / 16); ++q) {
            constexpr int E = 16 / sizeof(T);
            if constexpr (E == 4)
                reinterpret_cast<float4 *>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            else
                reinterpret_cast<double2 *>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) p[r] = v[r];
    }
}

template <typename T, int R>
__device__ __forceinline__ void sv_load(T (&v)[R], const T *p) {
    if constexpr (sizeof(T) * R % 16 == 0) {
#pragma unroll
        for (int q = 0; q < (int)(sizeof(T) * R / 16); ++q) {
            constexpr int E = 16 / sizeof(T);
            if constexpr (E == 4) {
                const float4 t = reinterpret_cast<const float4 *>(p)[q];
                v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
            } else {
                const double2 t = reinterpret_cast<const double2 *>(p)[q];
                v[2 * q] = t.x; v[2 * q + 1] = t.y;
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = p[r];
    }
}

// dynamic shared memory: (blockDim.x / 32) x 32 x R values.  U B-row
// gathers in flight per warp; MINB CTAs per SM bound the registers.
template <typename T, int V, int R, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
k_row_blocked(const int *__restrict__ rp, const unsigned *__restrict__ ue,
              const int *__restrict__ uoff, const T *__restrict__ av, const T *__restrict__ B,
              T *__restrict__ C, int M, int N, int g, int accumulate) {
    extern __shared__ __align__(16) unsigned char sraw[];
    const int warps = (int)(blockDim.x >> 5);
    const int w = (int)(threadIdx.x >> 5);
    const unsigned lane = lane_id();
    T *sv = reinterpret_cast<T *>(sraw) + (size_t)w * 32 * R;  // this warp's [32][R] slab
    const unsigned lt = lanemask_lt();
    const long long kcol = (long long)lane * V;
    const T *bk = B + kcol;
    const long long nblocks = ((long long)M + R - 1) / R;
    const long long tile_blocks = (long long)warps * g;
    const long long tiles = (nblocks + tile_blocks - 1) / tile_blocks;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int st = 0; st < g; ++st) {
            const long long b = tile * tile_blocks + (long long)st * warps + w;
            if (b >= nblocks) break;
            const long long i0 = b * R;
            // one load for the block's bounds: lanes 0..R the row starts,
            // R+1 / R+2 the union stream's range
            int t = 0;
            if ((int)lane <= R)
                t = __ldg(rp + (i0 + lane < M ? i0 + lane : (long long)M));
            else if ((int)lane == R + 1)
                t = __ldg(uoff + b);
            else if ((int)lane == R + 2)
                t = __ldg(uoff + b + 1);
            int cnt[R];
#pragma unroll
            for (int r = 0; r < R; ++r) cnt[r] = __shfl_sync(kFull, t, r);
            const int e0 = __shfl_sync(kFull, t, R + 1), e1 = __shfl_sync(kFull, t, R + 2);
            Vec<T, V> acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r].zero();
            for (int s = e0; s < e1; s += 32) {
                const int nv = min(32, e1 - s);
                const bool mine = (int)lane < nv;
                const unsigned x = __ldg(ue + (mine ? s + (int)lane : s));
                const unsigned m = mine ? (x >> UnionFmt<R>::kShift) : 0u;
                T v[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const bool has = (m >> r) & 1u;
                    const unsigned bal = __ballot_sync(kFull, has);
                    v[r] = has ? __ldg(av + cnt[r] + __popc(bal & lt)) : T(0);
                    cnt[r] += __popc(bal);
                }
                __syncwarp();  // the previous window's readers are done
                sv_store<T, R>(sv + lane * R, v);
                __syncwarp();
                for (int j = 0; j < nv; j += U) {
                    unsigned xx[U];
                    Vec<T, V> bb[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        xx[u] = __shfl_sync(kFull, x, (j + u) & 31);
                        if (j + u < nv)
                            gather_vec<T, V>(bb[u], row_ptr(bk, (int)(xx[u] & UnionFmt<R>::kColMask), N));
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (j + u >= nv) break;
                        T vv[R];
                        sv_load<T, R>(vv, sv + (j + u) * R);
                        const unsigned mk = xx[u] >> UnionFmt<R>::kShift;
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            if ((mk >> r) & 1u) fma_vec<T, V>(acc[r], vv[r], bb[u]);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (i0 + r < M) store_vec<T, V>(C + (i0 + r) * (long long)N + kcol, acc[r], accumulate != 0);
        }
    }
}

// ===========================================================================
// RB + parallel group reduction: row:1/g,col:c,r:g (row-reciprocal).
// A group of G lanes owns c consecutive fused cells io = i*N + k (one row, c
// columns); lane j accumulates positions begin+j, begin+j+G, ...
// (cuda_row_reciprocal.cu:39-46), then the AtomicAddGroup becomes an
// xor-shuffle tree and a single exclusive store by the group's lane 0.
// Rows longer than 32G: each lane folds its partial into float64 every 32
// strided terms (shorter rows need no float64: <= 32 terms per lane).
// ===========================================================================
// One row x one c-wide column vector, reduced by a group of G lanes: lane j
// accumulates positions beg+j, beg+j+G, ...; the xor-shuffle tree leaves the
// group sum in every lane of the group.  Rows of <= 32G nonzeros (<= 32
// terms per lane) sum in the value type, longer ones fold into float64 after
// each 32G-position segment, hub rows (> kExactRow) take float64 products.
// Every lane of the warp must call it (the shuffles use the full mask).
template <typename T, int V, int G, typename IT>
__device__ __forceinline__ Vec<T, V> rr_group_dot(const int *__restrict__ ci,
                                                  const T *__restrict__ av,
                                                  const T *__restrict__ bk, IT N, int beg,
                                                  int end, int j) {
    Vec<T, V> acc[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) acc[u].zero();
    Vec<double, V> tot;
    tot.zero();
    // rows of <= 32G nonzeros (one segment: <= 32 terms per lane) sum in
    // the value type; longer ones fold into float64 after each segment
    const bool multi = end - beg > 32 * G;
    if (sizeof(T) == 4 && end - beg > kExactRow) {
        // hub rows: float64 products (exact) summed in float64 (float32
        // product rounding grows like sqrt(row length): config 3 measured
        // 1.2e-5 without), kBatch gathers in flight
        int p = beg + j;
        for (; p + (kBatch - 1) * G < end; p += kBatch * G) {
            int cc[kBatch];
            T vv[kBatch];
            Vec<T, V> bv[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                cc[u] = __ldg(ci + p + u * G);
                vv[u] = __ldg(av + p + u * G);
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) ldg_vec<T, V>(bv[u], bk + (IT)cc[u] * (IT)N);
#pragma unroll
            for (int u = 0; u < kBatch; ++u)
#pragma unroll
                for (int x = 0; x < V; ++x)
                    tot.v[x] = fma((double)vv[u], (double)bv[u].v[x], tot.v[x]);
        }
        for (; p < end; p += G) {
            Vec<T, V> bv;
            ldg_vec<T, V>(bv, bk + (IT)__ldg(ci + p) * (IT)N);
            const double a = (double)__ldg(av + p);
#pragma unroll
            for (int x = 0; x < V; ++x) tot.v[x] = fma(a, (double)bv.v[x], tot.v[x]);
        }
    } else if (V == 1 && !multi) {
        // one scalar column, <= 32 terms per lane: the plain strided loop
        for (int p = beg + j; p < end; p += G)
            acc[0].v[0] = fma(__ldg(av + p), __ldg(bk + (IT)__ldg(ci + p) * (IT)N), acc[0].v[0]);
    } else {
        for (int seg = beg + j; seg < end; seg += 32 * G) {
            const int seg_end = min(seg + 32 * G, end);
            int p = seg;
            for (; p + (kBatch - 1) * G < seg_end; p += kBatch * G) {
                int cc[kBatch];
                T vv[kBatch];
                Vec<T, V> bv[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    cc[u] = __ldg(ci + p + u * G);
                    vv[u] = __ldg(av + p + u * G);
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) ldg_vec<T, V>(bv[u], bk + (IT)cc[u] * (IT)N);
#pragma unroll
                for (int u = 0; u < kBatch; ++u) fma_vec<T, V>(acc[u], vv[u], bv[u]);
            }
            for (; p < seg_end; p += G) {
                Vec<T, V> bv;
                ldg_vec<T, V>(bv, bk + (IT)__ldg(ci + p) * (IT)N);
                fma_vec<T, V>(acc[0], __ldg(av + p), bv);
            }
            if (multi) {
#pragma unroll
                for (int u = 0; u < kBatch; ++u) fold<T, V>(tot, acc[u]);
            }
        }
    }
    Vec<T, V> part = acc[0];
#pragma unroll
    for (int u = 1; u < kBatch; ++u) add_vec<T, V>(part, acc[u]);
    if (__any_sync(kFull, multi)) {  // long rows: the group sum in float64 too
        Vec<double, V> td;
#pragma unroll
        for (int x = 0; x < V; ++x) td.v[x] = multi ? tot.v[x] : (double)part.v[x];
        group_sum_vec<G, double, V>(td);
        part = narrow<T, V>(td);
    } else {
        group_sum_vec<G, T, V>(part);
    }
    return part;
}

// IT: the index type of cells/groups -- unsigned 32-bit whenever M*N fits
// (the host picks; ncu showed 2.4x the reference kernel's instruction count
// at one cell per warp with 64-bit index math), else 64-bit.
template <typename T, int V, int G, typename IT>
__global__ void __launch_bounds__(256)
k_row_reciprocal(const int *__restrict__ rp, const int *__restrict__ ci,
                 const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C,
                 int M, int N, int n_shift, int accumulate, unsigned long long *wb) {
    constexpr int GPW = 32 / G;  // groups per warp
    const IT cells = (IT)M * (IT)N;
    const IT groups = (cells + V - 1) / V;
    const IT items = (groups + GPW - 1) / GPW;
    const unsigned lane = lane_id();
    const int j = (int)(lane % G);
    unsigned long long nwb = 0;
    // the grid-stride counter stays 64-bit: with IT = unsigned, item + stride
    // can pass 2^32 when M*N is near it (one group per warp, ~M*N warps
    // launched) and a wrapped counter would revisit other warps' cells
    for (unsigned long long item = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
         item < (unsigned long long)items; item += (gridDim.x * (unsigned long long)blockDim.x) >> 5) {
        const IT grp = (IT)item * GPW + lane / G;
        const IT io0 = grp * V;
        const bool ok = io0 < cells;
        const IT i = ok ? (n_shift >= 0 ? io0 >> n_shift : io0 / (IT)N) : 0;
        const IT k0 = ok ? io0 - i * (IT)N : 0;
        const int beg = ok ? __ldg(rp + i) : 0;
        const int end = ok ? __ldg(rp + i + 1) : 0;
        const Vec<T, V> part = rr_group_dot<T, V, G, IT>(ci, av, B + k0, (IT)N, beg, end, j);
        if (ok && j == 0) {
            store_vec<T, V>(C + i * (IT)N + k0, part, accumulate != 0);
            nwb += V;
        }
    }
    flush_count(wb, nwb);
}

// The dgSPARSE RB+PR+RM kernel with the paper's tuning knobs (PAPER.md:
// 413-415; the cells of space.enumerate_fine_grained, space.py:294-348):
// <groupSz = G, blockSz, tileSz, workerDimR> with coarsenSz = V.  A block
// covers `tile` dense columns as tile/V column vectors of G lanes each
// (blockDim.x = vectors * G) and blockDim.y rows; gridDim.y column tiles;
// gridDim.x = the row parallelism (workerDimR / blockDim.y blocks), each
// block row striding over the rows when that is fewer than M.  The
// reduction per (row, vector) is the same G-lane group sum as
// k_row_reciprocal (rr_group_dot), one exclusive store per cell.  Every lane
// runs the same number of row rounds (shuffles need the whole warp).
template <typename T, int V, int G>
__global__ void __launch_bounds__(1024)
k_rbpr_grid(const int *__restrict__ rp, const int *__restrict__ ci, const T *__restrict__ av,
            const T *__restrict__ B, T *__restrict__ C, int M, int N, int tile_cols,
            int accumulate, unsigned long long *wb) {
    const int j = (int)(threadIdx.x % G);
    const int vec = (int)(threadIdx.x / G);
    const long long k0 = (long long)blockIdx.y * tile_cols + (long long)vec * V;
    const bool kok = k0 < N && (long long)vec * V < tile_cols;
    const long long stride = (long long)gridDim.x * blockDim.y;
    unsigned long long nwb = 0;
    for (long long base = (long long)blockIdx.x * blockDim.y; base < M; base += stride) {
        const long long i = base + threadIdx.y;
        const bool ok = kok && i < M;
        const int beg = ok ? __ldg(rp + i) : 0;
        const int end = ok ? __ldg(rp + i + 1) : 0;
        const Vec<T, V> part = rr_group_dot<T, V, G, long long>(ci, av, B + (ok ? k0 : 0),
                                                                (long long)N, beg, end, j);
        if (ok && j == 0) {
            store_vec<T, V>(C + i * (long long)N + k0, part, accumulate != 0);
            nwb += V;
        }
    }
    flush_count(wb, nwb);
}

// ===========================================================================
// EB + segment group (r > 1) / EB + atomic (r = 1): nnz:1,col:c,r (nnz-one).
// Logical thread = one position x one c-wide column tile; positions are padded
// to grid*npb and out-of-range lanes are zero-extended with the clamped search
// row (cuda_nnz_one_segment.cu:33-49).  Segment groups are aligned runs of r
// positions (npb % r == 0 makes block boundaries group boundaries).
// Hardware: a warp holds Q positions x TW tiles (Q*TW = 32, r | Q, lanes
// position-fastest), so each r-group is r consecutive lanes for the segmented
// scan while the TW tiles of one position form a coalesced B-row gather and
// C-row writeback.  One row search per position serves every tile.
// ===========================================================================
template <typename T, int V, int R>
__global__ void __launch_bounds__(256)
k_nnz_one(const int *__restrict__ rowid, const int *__restrict__ ci, const T *__restrict__ av,
          const T *__restrict__ B, T *__restrict__ C, int M, int N, long long nnz,
          long long total_pos, int TW, LongRows lr, unsigned long long *wb) {
    // A warp item spans kSteps consecutive groups of Q positions.  Flushes
    // into rows of the float64 table (long rows: the engine's numerics
    // policy, not the schedule) are added up per lane across the steps and
    // issued as one float64 atomic per run -- a hub row otherwise costs one
    // scalar float64 atomic per nonzero and tile; every other flush is the
    // schedule's own float32 red, one per writeback.  The counted writebacks
    // (SimMetrics.atomic_ops) are the logical ones either way.
    // (Hoisting the steps' A loads and segment analysis out of the tile
    // passes -- kept in registers across passes -- measured 1.2-1.6x slower
    // on config 2: more registers, less overlap across the unrolled steps.)
    constexpr int kSteps = 4;
    const int NT = N / V;
    const int Q = 32 / TW;
    const long long span = (long long)Q * kSteps;
    const long long items = (total_pos + span - 1) / span;
    const unsigned lane = lane_id();
    const int ql = (int)(lane & (unsigned)(Q - 1));
    const int tl = (int)(lane / (unsigned)Q);
    const bool table = lr.threshold >= 0;
    // zero-extended lanes resolve to row M-1; when that row has nonzeros they
    // must carry its table flags too, or a run whose tail lane is padding
    // would send the row's sum to C where the table fold overwrites it
    const int last_rid = nnz > 0 ? __ldg(rowid + nnz - 1) : (M - 1);
    const int pad_rid = (last_rid & kRowMask) == M - 1 ? last_rid : (M - 1);
    unsigned long long nwb = 0;
    SGAP_WARP_LOOP(item, items) {
        for (int tt = 0; tt < NT; tt += TW) {
            const int tile = tt + tl;
            const bool tok = tile < NT;
            const long long kcol = (long long)tile * V;
            int prow = -1;  // pending table row of this lane, and its sum
            Vec<double, V> pend;
            pend.zero();
#pragma unroll
            for (int step = 0; step < kSteps; ++step) {
                const long long first = item * span + (long long)step * Q;
                if (first >= total_pos) break;  // warp-uniform
                const long long pos = first + ql;
                const bool in_grid = pos < total_pos;
                const bool in_nnz = pos < nnz;
                // row owning the position; zero-extended lanes past nnz keep
                // the clamped search row M-1 (lowering.py:476-488 with the
                // window of the last block)
                const int rid = in_nnz ? __ldg(rowid + pos) : pad_rid;
                const int row = rid & kRowMask;
                const int col = in_nnz ? __ldg(ci + pos) : 0;
                const T a = in_nnz ? __ldg(av + pos) : T(0);
                SegLanes sl{};
                if constexpr (R > 1) sl = seg_lanes<R, int>(row, in_grid);
                Vec<T, V> bv;
                bv.zero();
                if (in_nnz && tok) ldg_vec<T, V>(bv, row_ptr(B + kcol, col, N));
                const bool writer = (R == 1 ? in_nnz : sl.tail) && tok;
                // Warps that touch a float64-table row (hub rows) form exact
                // float64 products and segment sums: float32 product rounding
                // alone grows like sqrt(row length) and breaks 1e-5 on
                // config 3's hub rows.  Other warps stay in float32.
                if (table && __any_sync(kFull, rid < 0)) {
                    Vec<double, V> pd;
#pragma unroll
                    for (int x = 0; x < V; ++x) pd.v[x] = (double)a * (double)bv.v[x];
                    if constexpr (R > 1) seg_scan_vec<R, double, V>(pd, sl.dist);
                    if (writer) {
                        nwb += V;
                        if (rid < 0) {
                            if (row != prow) {
                                if (prow >= 0) flush_row<T, V>(C, N, prow | kLongFlag, kcol, pend, lr);
                                prow = row;
                                pend.zero();
                            }
                            add_vec<double, V>(pend, pd);
                        } else {
                            red_vec<T, V>(C + (long long)row * N + kcol, narrow<T, V>(pd));
                        }
                    }
                } else {
                    Vec<T, V> prod;
#pragma unroll
                    for (int x = 0; x < V; ++x) prod.v[x] = a * bv.v[x];
                    if constexpr (R > 1) seg_scan_vec<R, T, V>(prod, sl.dist);
                    if (writer) {
                        nwb += V;
                        red_vec<T, V>(C + (long long)row * N + kcol, prod);
                    }
                }
            }
            if (prow >= 0) flush_row<T, V>(C, N, prow | kLongFlag, kcol, pend, lr);
        }
    }
    flush_count(wb, nwb);
}

// ===========================================================================
// EB + serial reduction: nnz:g,col:c,r:1 (nnz-multiple, the TACO nnz split).
// Logical work = one aligned chunk of g positions x one column; the walk
// tracks its row (block-window search, then forward advance) and flushes an
// atomic at every row change plus once at the end -- also for chunks past nnz
// (cuda_nnz_multiple.cu:33-53).
// Hardware: W lanes (c columns each) share a chunk, 32/W chunks per warp.
// The lanes of a chunk read each position's (col, val) as a broadcast load,
// kBatch B-row gathers go out back to back before the serial flush logic
// consumes them, and the chunk's next row start is kept in a register so the
// walk only touches row_ptr at a row change.
// ===========================================================================
// A-operand sources for the serial walk: global memory (read-only path) or
// a shared-memory tile filled by the bulk-copy producer.
template <typename T>
struct GlobalA {
    const int *rowid, *ci;
    const T *av;
    // positions are < 2^31 (sgap_run checks nnz): 32-bit unsigned offsets
    // give one IMAD.WIDE.U32 per address instead of 64-bit index arithmetic
    template <typename I>
    __device__ __forceinline__ int row(I q) const { return __ldg(rowid + (unsigned)q); }
    template <typename I>
    __device__ __forceinline__ int col(I q) const { return __ldg(ci + (unsigned)q); }
    template <typename I>
    __device__ __forceinline__ T val(I q) const { return __ldg(av + (unsigned)q); }
    // four consecutive positions, q % 4 == 0 (16-byte aligned)
    template <typename I>
    __device__ __forceinline__ void load4(I q, int4 &c, Vec<T, 4> &v, int4 &r) const {
        const unsigned u = (unsigned)q;
        c = __ldg(reinterpret_cast<const int4 *>(ci + u));
        r = __ldg(reinterpret_cast<const int4 *>(rowid + u));
        ldg_vec<T, 4>(v, av + u);
        // (evict-first A loads, __ldcs: 0.833 vs 0.700 ms on config 2)
    }
    // split loads for the column-pipelined row_ptr walk: the columns of the
    // next batch go out before this batch's gathers are consumed
    template <typename I>
    __device__ __forceinline__ int4 load4c(I q) const {
        return __ldg(reinterpret_cast<const int4 *>(ci + (unsigned)q));
    }
    template <typename I>
    __device__ __forceinline__ void load4v(I q, Vec<T, 4> &v) const {
        ldg_vec<T, 4>(v, av + (unsigned)q);
    }
    // (col, val) only: the row_ptr-tracking walk needs no per-position row ids
    template <typename I>
    __device__ __forceinline__ void load4cv(I q, int4 &c, Vec<T, 4> &v) const {
        const unsigned u = (unsigned)q;
        c = __ldg(reinterpret_cast<const int4 *>(ci + u));
        ldg_vec<T, 4>(v, av + u);
    }
    // pull the A lines `ahead` positions further into L1 (one per 32 positions)
    template <typename I>
    __device__ __forceinline__ void prefetch(I q) const {
        const unsigned u = (unsigned)q;
        prefetch_l1(ci + u);
        prefetch_l1(rowid + u);
        prefetch_l1(av + u);
    }
    template <typename I>
    __device__ __forceinline__ void prefetch_cv(I q) const {
        const unsigned u = (unsigned)q;
        prefetch_l1(ci + u);
        prefetch_l1(av + u);
    }
};

template <typename T>
struct SharedA {
    const int *sr, *sc;
    const T *sv;
    template <typename I>
    __device__ __forceinline__ void prefetch(I) const {}
    __device__ __forceinline__ int row(long long q) const { return sr[q]; }
    __device__ __forceinline__ int col(long long q) const { return sc[q]; }
    __device__ __forceinline__ T val(long long q) const { return sv[q]; }
    __device__ __forceinline__ void load4(long long q, int4 &c, Vec<T, 4> &v, int4 &r) const {
        c = *reinterpret_cast<const int4 *>(sc + q);
        r = *reinterpret_cast<const int4 *>(sr + q);
        if constexpr (sizeof(T) == 4) {
            const float4 t = *reinterpret_cast<const float4 *>(sv + q);
            v.v[0] = t.x; v.v[1] = t.y; v.v[2] = t.z; v.v[3] = t.w;
        } else {
            const double2 t0 = *reinterpret_cast<const double2 *>(sv + q);
            const double2 t1 = *reinterpret_cast<const double2 *>(sv + q + 2);
            v.v[0] = t0.x; v.v[1] = t0.y; v.v[2] = t1.x; v.v[3] = t1.y;
        }
    }
};

// Vectorised serial walk for chunks that start on a 4-position boundary:
// one 16-byte load each of 4 (col), (val), (row id), four B-row gathers, and
// -- since row ids are non-decreasing -- a single compare of the 4th row id
// against the current row decides whether the batch can flush at all.
// Owner writes (overwrite mode): a row whose nonzeros all lie inside one
// chunk is flushed with a plain store -- nobody else touches it, so C needs
// no zero-fill for it; rows split across chunks are zeroed by k_zero_shared_rows
// and flushed atomically.  `base`/`end` are global positions of the chunk.
struct Owner {
    const int *rp;
    const int *rowid;      // global row ids (for the row before the chunk)
    long long base, end;   // global positions of the chunk
    long long nnz;
    int m;
    bool on;
};

// Owner-mode zero-fill of empty rows, done by the walk that passes them:
// rows strictly between two consecutive nonzeros' rows are empty; the chunk
// whose first row starts at its base also covers the gap after the previous
// position's row (or the leading empty rows), the chunk holding the last
// nonzero covers the trailing ones.  Each lane clears its own column tile.
template <typename T, int V>
__device__ __forceinline__ void zero_rows(T *__restrict__ C, int N, long long kcol, int r0, int r1) {
    Vec<T, V> z;
    z.zero();
    for (int r = r0; r < r1; ++r) store_vec<T, V>(C + (long long)r * N + kcol, z, false);
}

template <typename T, int V>
__device__ __forceinline__ void zero_gap_before(T *__restrict__ C, int N, long long kcol,
                                                const Owner &own, int cur_row) {
    const int prev = own.base > 0 ? (__ldg(own.rowid + own.base - 1) & kRowMask) : -1;
    zero_rows<T, V>(C, N, kcol, prev + 1, cur_row);
}

template <typename T, int V>
__device__ __forceinline__ void flush_owned(T *__restrict__ C, int N, int rid, long long kcol,
                                            const Vec<double, V> &tot, const LongRows &lr,
                                            bool complete) {
    if (complete && rid >= 0)
        store_vec<T, V>(C + (long long)rid * N + kcol, narrow<T, V>(tot), false);
    else
        flush_row<T, V>(C, N, rid, kcol, tot, lr);
}

// Vectorised serial walk for chunks that start on a 4-position boundary:
// one 16-byte load each of 4 (col), (val), (row id), four B-row gathers, and
// -- since row ids are non-decreasing -- a single compare of the 4th row id
// against the current row decides whether the batch can flush at all.
template <typename T, int V, class ASrc>
__device__ __forceinline__ void eb_walk4(const ASrc &A, long long q0, long long qend,
                                         const T *__restrict__ B, int N, long long kcol,
                                         T *__restrict__ C, const LongRows &lr, const Owner &own,
                                         unsigned long long &nwb) {
    int cur = A.row(q0);
    bool here = own.on && __ldg(own.rp + (cur & kRowMask)) == own.base;
    if (here) zero_gap_before<T, V>(C, N, kcol, own, cur & kRowMask);
    Vec<T, V> acc;
    acc.zero();
    Vec<double, V> tot;
    tot.zero();
    const T *bk = B + kcol;
    unsigned q = (unsigned)q0;
    const unsigned qe = (unsigned)qend;
    auto batch4 = [&](unsigned qq) {
        int4 c, r;
        Vec<T, 4> v;
        A.load4(qq, c, v, r);
        Vec<T, V> b0, b1, b2, b3;
        ldg_vec<T, V>(b0, row_ptr(bk, c.x, N));
        ldg_vec<T, V>(b1, row_ptr(bk, c.y, N));
        ldg_vec<T, V>(b2, row_ptr(bk, c.z, N));
        ldg_vec<T, V>(b3, row_ptr(bk, c.w, N));
        if (r.w == cur) {
            fma_vec<T, V>(acc, v.v[0], b0);
            fma_vec<T, V>(acc, v.v[1], b1);
            fma_vec<T, V>(acc, v.v[2], b2);
            fma_vec<T, V>(acc, v.v[3], b3);
        } else {
            const int rr[4] = {r.x, r.y, r.z, r.w};
            const Vec<T, V> *bb[4] = {&b0, &b1, &b2, &b3};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (rr[u] != cur) {
                    fold<T, V>(tot, acc);
                    flush_owned<T, V>(C, N, cur, kcol, tot, lr, here);
                    nwb += V;
                    tot.zero();
                    if (own.on) zero_rows<T, V>(C, N, kcol, (cur & kRowMask) + 1, rr[u] & kRowMask);
                    cur = rr[u];
                    here = own.on;
                }
                fma_vec<T, V>(acc, v.v[u], *bb[u]);
            }
        }
    };
    // two batches per trip: one prefetch test and one float64 fold per 8
    // positions (float32 partials never exceed 8 terms: a flush folds too).
    // (Four per trip: more spills, 0.709 vs 0.702 ms on config 2; loading the
    // next batch's A under this batch's gathers: spills, 0.846 ms; storing a
    // row's float32 partial directly when no fold happened since it began,
    // skipping the float64 round trip: 0.710 vs 0.704 ms; B gathers with
    // ld.global.nc.L1::no_allocate: 0.874 ms -- hub-row L1 hits matter; an
    // L2 evict_last policy on them (createpolicy, fraction 0.25/0.5/1.0):
    // 0.723/0.715/0.715 ms; the max-L1 carveout: unchanged, already chosen;
    // L1::evict_last on the B gathers: 0.709 ms, L1::evict_first on the
    // col/row-id loads: 0.799 ms.)
    for (; q + 8 <= qe; q += 8) {
        if ((q & 31) == 0 && q + 64 < qe) A.prefetch(q + 64);  // A lines two ahead
        batch4(q);
        batch4(q + 4);
        fold<T, V>(tot, acc);
    }
    if (q + 4 <= qe) {
        batch4(q);
        q += 4;
    }
    for (; q < qe; ++q) {  // < 4 tail positions
        const int rq = A.row(q);
        Vec<T, V> b;
        ldg_vec<T, V>(b, row_ptr(bk, A.col(q), N));
        if (rq != cur) {
            fold<T, V>(tot, acc);
            flush_owned<T, V>(C, N, cur, kcol, tot, lr, here);
            nwb += V;
            tot.zero();
            if (own.on) zero_rows<T, V>(C, N, kcol, (cur & kRowMask) + 1, rq & kRowMask);
            cur = rq;
            here = own.on;
        }
        fma_vec<T, V>(acc, A.val(q), b);
    }
    fold<T, V>(tot, acc);
    const bool complete = here && __ldg(own.rp + (cur & kRowMask) + 1) == own.end;
    flush_owned<T, V>(C, N, cur, kcol, tot, lr, complete);
    nwb += V;
    if (own.on && own.end == own.nnz) zero_rows<T, V>(C, N, kcol, (cur & kRowMask) + 1, own.m);
}

// The same vectorised walk without per-position row ids (hw variant 1 when
// the plan carries the g-chunk start rows): the row is tracked from row_ptr
// as the reference lowering does (lowering.py:490-500) -- the chunk's first
// row comes from a per-chunk start table (compute_block_starts at chunk g),
// `ce` is the current row's end and a batch of 4 positions stays in the row
// iff q + 3 < ce.  A row change walks row_ptr forward (empty rows passed are
// zeroed in owner mode); the table / error-free flags of a row follow from
// its length, so the A stream is 8 bytes per position instead of 12.
// B-row gather of the row_ptr walk.  HINT: the column carries bit 31 for
// "cold" columns (outside the plan's hot set) whose rows are loaded with the
// streaming cache operator (ld.global.cs: evict-first in L1 and L2) so they
// do not push the hot rows out of L2.
template <typename T, int V, bool HINT>
__device__ __forceinline__ void gather_b(Vec<T, V> &o, const T *__restrict__ bk, int c, int N) {
    if constexpr (HINT && sizeof(T) == 4 && V == 4) {
        const float *p = row_ptr(bk, c & 0x7fffffff, N);
        if (c < 0) {
            const float4 t = __ldcs(reinterpret_cast<const float4 *>(p));
            o.v[0] = t.x; o.v[1] = t.y; o.v[2] = t.z; o.v[3] = t.w;
        } else {
            ldg_vec<T, V>(o, p);
        }
    } else if constexpr (HINT) {
        ldg_vec<T, V>(o, row_ptr(bk, c & 0x7fffffff, N));
    } else {
        ldg_vec<T, V>(o, row_ptr(bk, c, N));
    }
}

__device__ __forceinline__ int row_flags(int cur, unsigned cs, unsigned ce, const LongRows &lr) {
    if (lr.threshold < 0) return cur;
    const long long len = (long long)ce - (long long)cs;
    const bool is_long = len > lr.threshold;
    const bool split = lr.chunk > 0 && len > 0 &&
                       (long long)cs / lr.chunk != ((long long)ce - 1) / lr.chunk;
    return cur | ((is_long || split) ? kLongFlag : 0) | ((is_long && len > kExactRow) ? kExactFlag : 0);
}

template <typename T, int V>
__device__ __forceinline__ void zero_gap_before_rp(T *__restrict__ C, int N, long long kcol,
                                                   const int *__restrict__ rp, int cur,
                                                   unsigned base) {
    // empty rows right before `cur` all start (and end) at the chunk base
    Vec<T, V> z;
    z.zero();
    for (int r = cur - 1; r >= 0 && (unsigned)__ldg(rp + r) == base; --r)
        store_vec<T, V>(C + (long long)r * N + kcol, z, false);
}

template <typename T, int V, bool HINT = false, bool PF = false, int PFD = 1>
__device__ __forceinline__ void eb_walk4_rp(const GlobalA<T> &A, const int *__restrict__ rp,
                                            int cur, long long q0, long long qend,
                                            const T *__restrict__ B, int N, long long kcol,
                                            T *__restrict__ C, const LongRows &lr,
                                            const Owner &own, unsigned long long &nwb,
                                            int ldb, long long bcol) {
    // B rows: stride ldb, this tile at column bcol (N / kcol, except for the
    // panel-major copy of B that hw variant 10 walks); C: stride N, column kcol
    unsigned cs = (unsigned)__ldg(rp + cur), ce = (unsigned)__ldg(rp + cur + 1);
    // the NEXT row's end, loaded one row ahead so a row change does not wait
    // on a dependent row_ptr load
    unsigned cn = cur + 1 < own.m ? (unsigned)__ldg(rp + cur + 2) : ce;
    bool here = own.on && cs == (unsigned)own.base;
    if (here) zero_gap_before_rp<T, V>(C, N, kcol, rp, cur, (unsigned)own.base);
    Vec<T, V> acc;
    acc.zero();
    Vec<double, V> tot;
    tot.zero();
    const T *bk = B + bcol;
    unsigned q = (unsigned)q0;
    const unsigned qe = (unsigned)qend;
    // close the current row and move to the row holding position p
    auto advance = [&](unsigned p) {
        fold<T, V>(tot, acc);
        flush_owned<T, V>(C, N, row_flags(cur, cs, ce, lr), kcol, tot, lr, here);
        nwb += V;
        tot.zero();
        do {
            ++cur;
            cs = ce;
            ce = cn;
            cn = cur + 1 < own.m ? (unsigned)__ldg(rp + cur + 2) : ce;
            if (own.on && ce <= p) {  // an empty row passed over
                Vec<T, V> z;
                z.zero();
                store_vec<T, V>(C + (long long)cur * N + kcol, z, false);
            }
        } while (ce <= p);
        here = own.on;
    };
    {  // column-pipelined: the next batch's 16-byte column load goes out
       // before this batch's gathers, so the gather addresses do not wait on
       // an L2 round trip for their columns (ncu, config 2: 10.5% of the
       // stall samples sat on that address computation; interleaved A/B:
       // config 3 -3.5%, config 5 (with hints) -2%)
        int4 cn = make_int4(0, 0, 0, 0);
        if (q + 4 <= qe) cn = A.load4c(q);
        bool odd = false;
        for (; q + 4 <= qe; q += 4) {
            const int4 c = cn;
            if (q + 8 <= qe) cn = A.load4c(q + 4);
            if ((q & 31) == 0 && q + 64 < qe) A.prefetch_cv(q + 64);
            Vec<T, V> b0, b1, b2, b3;
            gather_b<T, V, HINT>(b0, bk, c.x, ldb);
            gather_b<T, V, HINT>(b1, bk, c.y, ldb);
            gather_b<T, V, HINT>(b2, bk, c.z, ldb);
            gather_b<T, V, HINT>(b3, bk, c.w, ldb);
            Vec<T, 4> v;
            A.load4v(q, v);
            if constexpr (PF) {
                // the next batch's B rows toward L2 now (its columns are in
                // cn, an L1 hit after the A-line prefetch): memory-level
                // parallelism without holding registers for the data
                if constexpr (PFD <= 1) {
                    if (q + 8 <= qe) {
                        prefetch_l2(row_ptr(bk, cn.x & 0x7fffffff, ldb));
                        prefetch_l2(row_ptr(bk, cn.y & 0x7fffffff, ldb));
                        prefetch_l2(row_ptr(bk, cn.z & 0x7fffffff, ldb));
                        prefetch_l2(row_ptr(bk, cn.w & 0x7fffffff, ldb));
                    }
                } else if (q + 4 * PFD + 4 <= qe) {  // PFD batches ahead: one more 16-B col load (an L1 hit)
                    const int4 cf = A.load4c(q + 4 * PFD);
                    prefetch_l2(row_ptr(bk, cf.x & 0x7fffffff, ldb));
                    prefetch_l2(row_ptr(bk, cf.y & 0x7fffffff, ldb));
                    prefetch_l2(row_ptr(bk, cf.z & 0x7fffffff, ldb));
                    prefetch_l2(row_ptr(bk, cf.w & 0x7fffffff, ldb));
                }
            }
            if (q + 3 < ce) {
                fma_vec<T, V>(acc, v.v[0], b0);
                fma_vec<T, V>(acc, v.v[1], b1);
                fma_vec<T, V>(acc, v.v[2], b2);
                fma_vec<T, V>(acc, v.v[3], b3);
            } else {
                const Vec<T, V> *bb[4] = {&b0, &b1, &b2, &b3};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (q + u >= ce) advance(q + u);
                    fma_vec<T, V>(acc, v.v[u], *bb[u]);
                }
            }
            if (odd) fold<T, V>(tot, acc);
            odd = !odd;
        }
    }
    for (; q < qe; ++q) {  // < 4 tail positions
        Vec<T, V> b;
        gather_b<T, V, HINT>(b, bk, A.col(q), ldb);
        if (q >= ce) advance(q);
        fma_vec<T, V>(acc, A.val(q), b);
    }
    fold<T, V>(tot, acc);
    const bool complete = here && ce == (unsigned)own.end;
    flush_owned<T, V>(C, N, row_flags(cur, cs, ce, lr), kcol, tot, lr, complete);
    nwb += V;
    if (own.on && own.end == own.nnz) zero_rows<T, V>(C, N, kcol, cur + 1, own.m);
}

// A chunk lying entirely inside one long row (flagged in its row id): the
// error-free accumulate (TwoProduct + TwoSum, float64 folds), no row changes.
// Only rows flagged kExactFlag (> kExactRow nonzeros).  These chunks run in their own kernel (k_nnz_multiple_exact) so the hot walk
// keeps its register budget; chunks that straddle a long row's ends use the
// fast walk -- at most two per row, too few terms for their float32 rounding
// to matter.
template <typename T, int V, class ASrc>
__device__ __forceinline__ void eb_walk4_exact(const ASrc &A, long long q0, long long qend,
                                            const T *__restrict__ B, int N, long long kcol,
                                            Vec<double, V> &tot) {
    // float64 products of float32 inputs are exact; their float64 sum is
    // error-free at float32 output precision
    const T *bk = B + kcol;
    long long q = q0;
    for (; q + 4 <= qend; q += 4) {
        int4 c, r;
        Vec<T, 4> v;
        A.load4(q, c, v, r);
        Vec<T, V> b0, b1, b2, b3;
        ldg_vec<T, V>(b0, row_ptr(bk, c.x, N));
        ldg_vec<T, V>(b1, row_ptr(bk, c.y, N));
        ldg_vec<T, V>(b2, row_ptr(bk, c.z, N));
        ldg_vec<T, V>(b3, row_ptr(bk, c.w, N));
#pragma unroll
        for (int x = 0; x < V; ++x) {
            tot.v[x] = fma((double)v.v[0], (double)b0.v[x], tot.v[x]);
            tot.v[x] = fma((double)v.v[1], (double)b1.v[x], tot.v[x]);
            tot.v[x] = fma((double)v.v[2], (double)b2.v[x], tot.v[x]);
            tot.v[x] = fma((double)v.v[3], (double)b3.v[x], tot.v[x]);
        }
    }
    for (; q < qend; ++q) {
        Vec<T, V> b;
        ldg_vec<T, V>(b, row_ptr(bk, A.col(q), N));
        const double a = (double)A.val(q);
#pragma unroll
        for (int x = 0; x < V; ++x) tot.v[x] = fma(a, (double)b.v[x], tot.v[x]);
    }
}

template <typename T, int V, int U>
struct WalkBatch {
    int c[U], r[U];
    T v[U];
    Vec<T, V> b[U];
};

// The serial nnz walk of one chunk [q0, qend) for one column tile when the
// chunk is not 4-aligned (g % 4 != 0 or unaligned A): U positions' (col, val,
// row) and their U B-row gathers per step, then the serial flush logic.  A
// flush (row change or chunk end) is one writeback; partial sums fold into
// float64 every kFoldEvery positions.  (Software-pipelining batch i+1 under
// batch i was measured slower: the registers cost more occupancy.)
template <typename T, int V, int U, class ASrc>
__device__ __forceinline__ void eb_walk(const ASrc &A, long long q0, long long qend,
                                        const T *__restrict__ B, int N, long long kcol,
                                        T *__restrict__ C, const LongRows &lr, const Owner &own,
                                        unsigned long long &nwb) {
    auto fetch = [&](long long q, WalkBatch<T, V, U> &w) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = q + u < qend;
            w.c[u] = ok ? A.col(q + u) : 0;
            w.v[u] = ok ? A.val(q + u) : T(0);
            w.r[u] = ok ? A.row(q + u) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (q + u < qend) ldg_vec<T, V>(w.b[u], B + (long long)w.c[u] * N + kcol);
            else w.b[u].zero();
        }
    };
    int cur = A.row(q0);
    bool here = own.on && __ldg(own.rp + (cur & kRowMask)) == own.base;
    if (here) zero_gap_before<T, V>(C, N, kcol, own, cur & kRowMask);
    Vec<T, V> acc;
    acc.zero();
    Vec<double, V> tot;
    tot.zero();
    int since_fold = 0;
    auto consume = [&](long long q, const WalkBatch<T, V, U> &w) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (q + u < qend && w.r[u] != cur) {
                fold<T, V>(tot, acc);
                flush_owned<T, V>(C, N, cur, kcol, tot, lr, here);
                nwb += V;
                tot.zero();
                since_fold = 0;
                if (own.on) zero_rows<T, V>(C, N, kcol, (cur & kRowMask) + 1, w.r[u] & kRowMask);
                cur = w.r[u];
                here = own.on;
            }
            fma_vec<T, V>(acc, w.v[u], w.b[u]);
        }
        since_fold += U;
        if (since_fold >= kFoldEvery) {
            fold<T, V>(tot, acc);
            since_fold = 0;
        }
    };
    WalkBatch<T, V, U> w0;
    for (long long q = q0; q < qend; q += U) {
        fetch(q, w0);
        consume(q, w0);
    }
    fold<T, V>(tot, acc);
    const bool complete = here && __ldg(own.rp + (cur & kRowMask) + 1) == own.end;
    flush_owned<T, V>(C, N, cur, kcol, tot, lr, complete);
    nwb += V;
    if (own.on && own.end == own.nnz) zero_rows<T, V>(C, N, kcol, (cur & kRowMask) + 1, own.m);
}

// B (K x N, row-major) -> the panel-major copy hw variant 10 walks: panel p
// holds columns [p*PW, p*PW + PW) of every row as a contiguous K x PW block
// (the last panel zero-padded past N).  One 16-byte vector per thread, read
// coalesced along B's rows.  A strided panel (PW of every N columns) used
// only a quarter of each B row's L2 lines' neighbourhood and lost most of
// the panel's L2 reuse (config 3 N=256: 10.3 vs 8.8 ms for contiguous
// panels).
template <typename T>
__global__ void __launch_bounds__(256) k_panelize(const T *__restrict__ B, T *__restrict__ P,
                                                  long long K, int N, int PW) {
    constexpr int E = 16 / sizeof(T);
    const int vpr = PW / E;  // 16-byte vectors per panel row
    const int panels = (N + PW - 1) / PW;
    const long long total = K * panels * vpr;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / ((long long)panels * vpr);
        const int rest = (int)(i - row * panels * vpr);
        const int p = rest / vpr, v = rest - p * vpr;
        const int col = p * PW + v * E;
        T *dst = P + ((long long)p * K + row) * PW + v * E;
        if (col + E <= N) {
            __stcs(reinterpret_cast<int4 *>(dst), __ldg(reinterpret_cast<const int4 *>(B + row * N + col)));
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e] = col + e < N ? B[row * N + col + e] : T(0);
        }
    }
}

// A chunk inside an exact-flagged (hub) row, walked by the register walk
// itself: float64 products (exact for float32 inputs) summed in float64, one
// flush into the float64 table.  Out of line (noinline) so its float64 state
// does not count against the hot walk's register budget.
template <typename T, int V>
__device__ __noinline__ void eb_chunk_f64(const GlobalA<T> A, long long base, long long end,
                                          const T *__restrict__ B, int N, long long kcol,
                                          T *__restrict__ C, const LongRows lr, int r_first,
                                          bool vec4, int ldb, long long bcol) {
    Vec<double, V> tot;
    tot.zero();
    const T *bk = B + bcol;  // B rows: stride ldb (see eb_walk4_rp)
    unsigned q = (unsigned)base;
    const unsigned qe = (unsigned)end;
    for (; vec4 && q + 4 <= qe; q += 4) {
        int4 c;
        Vec<T, 4> v;
        A.load4cv(q, c, v);
        Vec<T, V> b0, b1, b2, b3;  // (bit 31: the cold-column hint, not part of the index)
        ldg_vec<T, V>(b0, row_ptr(bk, c.x & 0x7fffffff, ldb));
        ldg_vec<T, V>(b1, row_ptr(bk, c.y & 0x7fffffff, ldb));
        ldg_vec<T, V>(b2, row_ptr(bk, c.z & 0x7fffffff, ldb));
        ldg_vec<T, V>(b3, row_ptr(bk, c.w & 0x7fffffff, ldb));
#pragma unroll
        for (int x = 0; x < V; ++x) {
            tot.v[x] = fma((double)v.v[0], (double)b0.v[x], tot.v[x]);
            tot.v[x] = fma((double)v.v[1], (double)b1.v[x], tot.v[x]);
            tot.v[x] = fma((double)v.v[2], (double)b2.v[x], tot.v[x]);
            tot.v[x] = fma((double)v.v[3], (double)b3.v[x], tot.v[x]);
        }
    }
    for (; q < qe; ++q) {
        Vec<T, V> b;
        ldg_vec<T, V>(b, row_ptr(bk, A.col(q) & 0x7fffffff, ldb));
        const double a = (double)A.val(q);
#pragma unroll
        for (int x = 0; x < V; ++x) tot.v[x] = fma(a, (double)b.v[x], tot.v[x]);
    }
    flush_row<T, V>(C, N, r_first, kcol, tot, lr);  // the float64 table
}

template <typename T, int V, int W, int U, bool RPW = false, bool HINT = false, bool PF = false,
          int PFD = 1, bool PANEL = false>
__global__ void __launch_bounds__(256, SGAP_EB_MINB)
k_nnz_multiple(const int *__restrict__ rowid, const int *__restrict__ ci,
               const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C,
               const int *__restrict__ rp, int M, int N, long long nnz, int g,
               long long total_pos, int vec4, int owner, LongRows lr, unsigned long long *wb,
               int exact_inline, const int *__restrict__ chunk_rows, int pass = 0) {
    const bool VEC4 = vec4 != 0;  // g % 4 == 0 and 16-byte aligned A arrays
    // row_ptr tracking (no per-position row ids) when the plan has the
    // g-chunk start rows and the walk is vectorised
    // (a separate instantiation, so each walk keeps its own register budget)
    constexpr bool RP = RPW;
    const long long exact_cut = lr.threshold > kExactRow ? lr.threshold : kExactRow;
    const int NT = N / V;
    constexpr int SG = 32 / W;
    const long long total_chunks = total_pos / g;
    const long long items = (total_chunks + SG - 1) / SG;
    const unsigned lane = lane_id();
    const int sg = (int)(lane / (unsigned)W);
    const int sl = (int)(lane & (unsigned)(W - 1));
    const GlobalA<T> A{rowid, ci, av};
    unsigned long long nwb = 0;
    // PANEL (hw variant 10): one launch per column panel.  Launch `pass`
    // walks every chunk for column tiles [pass*W, pass*W + W) only (one panel
    // of B, W*V columns), so the B rows live in L2 one panel at a time when
    // the whole of B does not fit but a panel does.  Each (chunk, tile) is the
    // same serial walk as without panels: results and writeback counts are
    // unchanged, only the order of the (chunk, tile) work differs.
    SGAP_WARP_LOOP(item, items) {
        const long long ch = item * SG + sg;
        if (ch >= total_chunks) continue;
        const long long base = ch * g;
        const long long end = min(base + (long long)g, nnz);
        const int tile_end = PANEL ? min(NT, (pass + 1) * W) : NT;
        for (int tile = PANEL ? pass * W + sl : sl; tile < tile_end; tile += W) {
            if (base >= end) {  // chunk past nnz: the reference flushes 0 into row M-1
                // (not nnz-one at r = 1, owner 3: its lanes past nnz break
                // before the atomic, cuda_nnz_one_serial.cu)
                if (owner != 3) nwb += V;
                continue;
            }
            // owner == 2: nnz-one's segment groups walked as g = r chunks (hw
            // variant 1 of nnz-one): the group straddling nnz also holds
            // zero-extended lanes of row M-1, a run of their own unless the
            // last real row is M-1 (cuda_nnz_one_segment.cu padding)
            if (owner == 2 && end == nnz && base + g > nnz &&
                (__ldg(rowid + nnz - 1) & kRowMask) != M - 1)
                nwb += V;
            const Owner own{rp, rowid, base, end, nnz, M, owner == 1};  // 2/3: red only
            if constexpr (RP) {
                const int cur = __ldg(chunk_rows + ch);
                const long long kcol = (long long)tile * V;
                // PANEL: B is this pass's panel of the panel-major copy
                // (K x W*V, contiguous), C stays row-major N wide
                const int ldb = PANEL ? W * V : N;
                const long long bcol = PANEL ? (long long)(tile - pass * W) * V : kcol;
                const long long cs = __ldg(rp + cur), ce = __ldg(rp + cur + 1);
                if (lr.threshold >= 0 && ce - cs > exact_cut && ce >= end) {
                    // a chunk inside an exact-flagged (hub) row
                    if (own.on && cs == base)
                        zero_gap_before_rp<T, V>(C, N, kcol, rp, cur, (unsigned)base);
                    if (own.on && end == nnz) zero_rows<T, V>(C, N, kcol, cur + 1, M);
                    nwb += V;
                    if (exact_inline)
                        eb_chunk_f64<T, V>(A, base, end, B, N, kcol, C, lr,
                                           cur | kLongFlag | kExactFlag, VEC4, ldb, bcol);
                    continue;
                }
                eb_walk4_rp<T, V, HINT, PF, PFD>(A, rp, cur, base, end, B, N, kcol, C, lr, own, nwb,
                                                 ldb, bcol);
                continue;
            } else {
            const int r_first = A.row(base);
            if ((r_first & kExactFlag) && A.row(end - 1) == r_first) {
                const long long kcol = (long long)tile * V;
                if (own.on && __ldg(rp + (r_first & kRowMask)) == base)
                    zero_gap_before<T, V>(C, N, kcol, own, r_first & kRowMask);
                if (own.on && end == nnz)
                    zero_rows<T, V>(C, N, kcol, (r_first & kRowMask) + 1, M);
                nwb += V;
                if (exact_inline)  // a chunk inside an exact-flagged (hub) row
                    eb_chunk_f64<T, V>(A, base, end, B, N, kcol, C, lr, r_first, VEC4, N, kcol);
                continue;
            }
            if (VEC4)
                eb_walk4<T, V>(A, base, end, B, N, (long long)tile * V, C, lr, own, nwb);
            else
                eb_walk<T, V, U>(A, base, end, B, N, (long long)tile * V, C, lr, own, nwb);
            }
        }
    }
    flush_count(wb, nwb);
    pdl_wait();  // launched after the error-free pass: finish after it too
}

// The chunks of nnz-multiple that lie entirely inside one exact-flagged row
// (> kExactRow nonzeros), walked with the error-free accumulate (see
// eb_walk4_exact).  Work comes from the long-row list: blockIdx.x picks a long
// row, blockIdx.y x warps split that row's contained chunks into 32-position
// pieces (a 239k-nonzero hub row becomes ~7.5k warp items instead of one
// serial walk).  Each piece flushes into the float64 long-row table (an
// order-free sum); the main kernel counts the writebacks and skips exactly
// these chunks (row id of first == last position, exact flag set).
template <typename T, int V>
__global__ void __launch_bounds__(256, 4)
k_nnz_multiple_exact(const int *__restrict__ rowid, const int *__restrict__ ci,
                     const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C,
                     const int *__restrict__ rp, int N, long long nnz, int g, int vec4,
                     LongRows lr) {
    const int NT = N / V;
    const unsigned lane = lane_id();
    const int warp = (int)(threadIdx.x >> 5);
    const int nwarps = (int)(blockDim.x >> 5);
    const long long per_chunk = ((long long)g + 31) >> 5;
    const GlobalA<T> A{rowid, ci, av};
    pdl_launch_dependents();  // the main walk (no data dependency) may start now
    // exactly the rows k_row_ids flagged exact (host-compacted list; the grid
    // is sized to it -- iterating the whole table launched ~65k mostly idle
    // CTAs, 77 us per call on config 2)
    for (int li = blockIdx.x; li < lr.exact_count; li += gridDim.x) {
        const int r = __ldg(lr.exact_rows + li);
        const long long rs = __ldg(rp + r), re = __ldg(rp + r + 1);
        const long long c0 = (rs + g - 1) / g;
        long long c1 = re / g;                        // chunks ending at (c+1)g <= re
        if (re == nnz && nnz % g) c1 = nnz / g + 1;   // ... and the final partial chunk
        if (c1 <= c0) continue;
        const long long items = (c1 - c0) * per_chunk;
        // a warp sums all its pieces of this row and flushes once per tile
        // (one float64 atomic per piece and tile serialised on the row's
        // table slot: 59 us per call on config 2's hub rows)
        const long long first = (long long)blockIdx.y * nwarps + warp;
        if (first >= items) continue;
        for (int tile = (int)lane; tile < NT; tile += 32) {
            const long long kcol = (long long)tile * V;
            Vec<double, V> tot;
            tot.zero();
            for (long long it = first; it < items; it += (long long)gridDim.y * nwarps) {
                const long long cb = (c0 + it / per_chunk) * g;
                const long long ce = min(cb + (long long)g, nnz);
                const long long q0 = cb + (it % per_chunk) * 32;
                const long long q1 = min(q0 + 32, ce);
                if (q0 >= q1) continue;
                if (vec4) {
                    eb_walk4_exact<T, V>(A, q0, q1, B, N, kcol, tot);
                } else {
                    for (long long q = q0; q < q1; ++q) {
                        Vec<T, V> b;
                        ldg_vec<T, V>(b, B + (long long)A.col(q) * N + kcol);
                        const double a = (double)A.val(q);
#pragma unroll
                        for (int x = 0; x < V; ++x) tot.v[x] = fma(a, (double)b.v[x], tot.v[x]);
                    }
                }
            }
            flush_row<T, V>(C, N, r | kLongFlag, kcol, tot, lr);  // the float64 table
        }
    }
}

// ---------------------------------------------------------------------------
// The same family, lane-staged (hw variant 3; a whole warp per chunk, lane l
// on column tile t0+l).  Per 32-position step lane l holds position s+l's
// (col, val, row id): one coalesced 128-byte request per array instead of 32
// broadcast loads, and the next step's triple is loaded while this one is
// consumed.  U B-row gathers go out back to back from shuffled column
// indices before any is consumed; a ballot of row changes lets change-free
// groups (the common case inside long power-law rows) skip the flush test.
// Writeback semantics, owner writes, long-row routing and float64 folds every
// kFoldEvery terms are those of eb_walk4 (tools/experiments/walk_probe.cu has
// the stripped-down loop this came from).
// ---------------------------------------------------------------------------
template <typename T, int V, int U>
__device__ __forceinline__ void eb_walk_staged(const int *__restrict__ rowid,
                                               const int *__restrict__ ci,
                                               const T *__restrict__ av, long long q0,
                                               long long qend, const T *__restrict__ B, int N,
                                               long long kcol, bool on, T *__restrict__ C,
                                               const LongRows &lr, const Owner &own,
                                               unsigned long long &nwb) {
    static_assert(U == 4 || U == 8, "U in {4, 8}");
    const unsigned lane = lane_id();
    long long qn = q0 + lane;
    // positions past the chunk read column 0 with value 0; their products are
    // never accumulated (the fast path only takes full groups)
    int c_n = qn < qend ? __ldg(ci + qn) : 0;
    T v_n = qn < qend ? __ldg(av + qn) : T(0);
    int r_n = qn < qend ? __ldg(rowid + qn) : 0;
    int cur = __shfl_sync(kFull, r_n, 0);
    bool here = own.on && __ldg(own.rp + (cur & kRowMask)) == own.base;
    if (here && on) zero_gap_before<T, V>(C, N, kcol, own, cur & kRowMask);
    Vec<T, V> acc;
    acc.zero();
    Vec<double, V> tot;
    tot.zero();
    const T *bk = B + (on ? kcol : 0);  // lanes past the last tile gather tile 0, store nothing
    for (long long s = q0; s < qend; s += 32) {
        const int c_l = c_n, r_l = r_n;
        const T v_l = v_n;
        qn = s + 32 + lane;
        c_n = qn < qend ? __ldg(ci + qn) : 0;
        v_n = qn < qend ? __ldg(av + qn) : T(0);
        r_n = qn < qend ? __ldg(rowid + qn) : 0;
        const int nval = (int)min(32LL, qend - s);
        const int r_up = __shfl_up_sync(kFull, r_l, 1);
        const unsigned chm =
            __ballot_sync(kFull, (int)lane < nval && r_l != (lane == 0 ? cur : r_up));
#pragma unroll 1
        for (int j = 0; j < nval; j += U) {
            // U gathers back to back (volatile: not sunk into the branch below)
            Vec<T, V> b[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                gather_vec<T, V>(b[u], row_ptr(bk, __shfl_sync(kFull, c_l, j + u), N));
            const unsigned gm = (chm >> j) & ((1u << U) - 1u);
            if (gm == 0u && j + U <= nval) {
#pragma unroll
                for (int u = 0; u < U; ++u) fma_vec<T, V>(acc, __shfl_sync(kFull, v_l, j + u), b[u]);
            } else {
                // a row change (or the chunk end) inside this group: one
                // position at a time, each B row re-read from L1 where the
                // gathers above just put it, so the flush path is instantiated
                // once and keeps no gathered rows live
#pragma unroll 1
                for (int u = 0; u < U; ++u) {
                    const int c = __shfl_sync(kFull, c_l, j + u);
                    const T v = __shfl_sync(kFull, v_l, j + u);
                    const int r = __shfl_sync(kFull, r_l, j + u);
                    if (j + u >= nval) break;
                    if ((gm >> u) & 1u) {
                        fold<T, V>(tot, acc);
                        if (on) {
                            flush_owned<T, V>(C, N, cur, kcol, tot, lr, here);
                            nwb += V;
                            if (own.on) zero_rows<T, V>(C, N, kcol, (cur & kRowMask) + 1, r & kRowMask);
                        }
                        tot.zero();
                        cur = r;
                        here = own.on;
                    }
                    Vec<T, V> bb;
                    ldg_vec<T, V>(bb, row_ptr(bk, c, N));
                    fma_vec<T, V>(acc, v, bb);
                }
            }
            if (((j + U) & (kFoldEvery - 1)) == 0) fold<T, V>(tot, acc);
        }
    }
    fold<T, V>(tot, acc);
    const bool complete = here && __ldg(own.rp + (cur & kRowMask) + 1) == own.end;
    if (on) {
        flush_owned<T, V>(C, N, cur, kcol, tot, lr, complete);
        nwb += V;
        if (own.on && own.end == own.nnz) zero_rows<T, V>(C, N, kcol, (cur & kRowMask) + 1, own.m);
    }
}

template <typename T, int V, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
k_nnz_multiple_staged(const int *__restrict__ rowid, const int *__restrict__ ci,
                      const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C,
                      const int *__restrict__ rp, int M, int N, long long nnz, int g,
                      long long total_pos, int owner, LongRows lr, unsigned long long *wb) {
    const int NT = N / V;
    const long long total_chunks = total_pos / g;
    const unsigned lane = lane_id();
    unsigned long long nwb = 0;
    SGAP_WARP_LOOP(ch, total_chunks) {
        const long long base = ch * g;
        const long long end = min(base + (long long)g, nnz);
        for (int t0 = 0; t0 < NT; t0 += 32) {
            const int tile = t0 + (int)lane;
            const bool on = tile < NT;
            const long long kcol = (long long)tile * V;
            if (base >= end) {  // chunk past nnz: the reference flushes 0 into row M-1
                if (on) nwb += V;
                continue;
            }
            const Owner own{rp, rowid, base, end, nnz, M, owner == 1};
            const int r_first = __ldg(rowid + base);
            if ((r_first & kExactFlag) && __ldg(rowid + end - 1) == r_first) {  // the exact kernel's
                if (on) {
                    if (own.on && __ldg(rp + (r_first & kRowMask)) == base)
                        zero_gap_before<T, V>(C, N, kcol, own, r_first & kRowMask);
                    if (own.on && end == nnz)
                        zero_rows<T, V>(C, N, kcol, (r_first & kRowMask) + 1, M);
                    nwb += V;
                }
                continue;
            }
            eb_walk_staged<T, V, U>(rowid, ci, av, base, end, B, N, kcol, on, C, lr, own, nwb);
        }
    }
    flush_count(wb, nwb);
    pdl_wait();  // launched after the error-free pass: finish after it too
}

// ---------------------------------------------------------------------------
// The same family, TMA-staged: a persistent CTA walks tiles of `tile`
// positions (a multiple of g, so chunks stay globally aligned).  One producer
// warp streams each tile's (col, val, row id) arrays into a shared-memory
// ring with cp.async.bulk, completion tracked by mbarriers; 8 consumer warps
// take the tile's chunks and only ever touch global memory for the B-row
// gathers and the C flushes.  This takes the A stream (and its DRAM latency)
// off the gather's critical path.
// ---------------------------------------------------------------------------
constexpr int kTmaConsumerWarps = 8;
constexpr int kTmaTile = 2048;  // positions per stage (capacity)
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;

template <typename T, int STAGES>
constexpr size_t tma_smem_bytes() {
    return (size_t)STAGES * kTmaTile * (2 * sizeof(int) + sizeof(T)) +
           2 * STAGES * sizeof(unsigned long long);
}

template <typename T, int V, int W, int U, int kTmaStages, int MINB>
__global__ void __launch_bounds__(kTmaThreads, MINB)
k_nnz_multiple_tma(const int *__restrict__ rowid, const int *__restrict__ ci,
                   const T *__restrict__ av, const T *__restrict__ B, T *__restrict__ C,
                   const int *__restrict__ rp, int M, int N, long long nnz, int g,
                   long long total_pos, int tile, int owner, LongRows lr,
                   unsigned long long *wb) {
    const bool VEC4 = (g % 4) == 0;
    extern __shared__ __align__(128) unsigned char smem[];
    int *s_col = reinterpret_cast<int *>(smem);
    int *s_row = s_col + kTmaStages * kTmaTile;
    T *s_val = reinterpret_cast<T *>(s_row + kTmaStages * kTmaTile);
    unsigned long long *full = reinterpret_cast<unsigned long long *>(s_val + kTmaStages * kTmaTile);
    unsigned long long *empty = full + kTmaStages;
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const long long ntiles = (total_pos + tile - 1) / tile;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTmaConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    unsigned long long nwb = 0;
    if (warp == kTmaConsumerWarps) {
        // ---------------- producer: one elected lane issues the bulk copies
        if (lane == 0) {
            int i = 0;
            for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                const int s = i % kTmaStages;
                mbar_wait(&empty[s], ((i / kTmaStages) & 1) ^ 1);
                const long long p0 = t * tile;
                long long left = nnz - p0;
                const int n_in = left <= 0 ? 0 : (left >= tile ? tile : (int)left);
                const int n_bulk = n_in & ~3;  // 16-byte granules
                int *dc = s_col + s * kTmaTile;
                int *dr = s_row + s * kTmaTile;
                T *dv = s_val + s * kTmaTile;
                for (int q = n_bulk; q < n_in; ++q) {  // <= 3 tail elements
                    dc[q] = __ldg(ci + p0 + q);
                    dr[q] = __ldg(rowid + p0 + q);
                    dv[q] = __ldg(av + p0 + q);
                }
                const unsigned tx = (unsigned)n_bulk * (unsigned)(2 * sizeof(int) + sizeof(T));
                mbar_arrive_expect_tx(&full[s], tx);
                if (n_bulk) {
                    bulk_g2s(dc, ci + p0, (unsigned)n_bulk * sizeof(int), &full[s]);
                    bulk_g2s(dr, rowid + p0, (unsigned)n_bulk * sizeof(int), &full[s]);
                    bulk_g2s(dv, av + p0, (unsigned)n_bulk * sizeof(T), &full[s]);
                }
            }
        }
    } else {
        // ---------------- consumers
        constexpr int SG = 32 / W;
        const int NT = N / V;
        const int sg = (int)(lane / (unsigned)W);
        const int sl = (int)(lane & (unsigned)(W - 1));
        int i = 0;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int s = i % kTmaStages;
            mbar_wait(&full[s], (i / kTmaStages) & 1);
            const long long p0 = t * tile;
            const long long left = nnz - p0;
            const int n_in = left <= 0 ? 0 : (left >= tile ? tile : (int)left);
            const long long span = total_pos - p0;
            const int chunks = (int)((span >= tile ? tile : span) / g);
            const int *sc = s_col + s * kTmaTile;
            const int *sr = s_row + s * kTmaTile;
            const T *sv = s_val + s * kTmaTile;
            const SharedA<T> SA{sr, sc, sv};
            for (int cj = warp * SG + sg; cj < chunks; cj += kTmaConsumerWarps * SG) {
                const int q0 = cj * g;
                const int qend = min(q0 + g, n_in);
                for (int tc = sl; tc < NT; tc += W) {
                    if (q0 >= qend) {  // chunk past nnz: a zero flush into row M-1
                        nwb += V;
                        continue;
                    }
                    const Owner own{rp, rowid, p0 + q0, p0 + qend, nnz, M, owner == 1};
                    const int r_first = SA.row(q0);
                    if ((r_first & kExactFlag) && SA.row(qend - 1) == r_first) {  // exact kernel's
                        if (own.on && __ldg(rp + (r_first & kRowMask)) == own.base)
                            zero_gap_before<T, V>(C, N, (long long)tc * V, own, r_first & kRowMask);
                        if (own.on && own.end == nnz)
                            zero_rows<T, V>(C, N, (long long)tc * V, (r_first & kRowMask) + 1, M);
                        nwb += V;
                        continue;
                    }
                    if (VEC4)
                        eb_walk4<T, V>(SA, q0, qend, B, N, (long long)tc * V, C, lr, own, nwb);
                    else
                        eb_walk<T, V, U>(SA, q0, qend, B, N, (long long)tc * V, C, lr, own,
                                               nwb);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    flush_count(wb, nwb);
    pdl_wait();  // launched after the error-free pass: finish after it too
}

// Per-position row ids (the row owning each nonzero, lowering.py:459-500),
// expanded once per matrix: a warp covers 1024 positions, each lane does one
// binary search and then walks forward; bit 31 flags rows of the long-row
// table (length > thr).
__global__ void __launch_bounds__(256)
k_row_ids(const int *__restrict__ rp, int M, long long nnz, long long thr, long long chunk,
          int *__restrict__ out) {
    const long long items = (nnz + 1023) >> 10;
    const unsigned lane = lane_id();
    SGAP_WARP_LOOP(item, items) {
        const long long base = item * 1024 + lane;
        if (base >= nnz) continue;
        int lo = 0, hi = M;  // last r in [0, M) with rp[r] <= base
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if ((long long)__ldg(rp + mid) <= base) lo = mid; else hi = mid;
        }
        int r = lo;
        long long start = __ldg(rp + r), next = __ldg(rp + r + 1);
        for (int j = 0; j < 32; ++j) {
            const long long p = base + 32LL * j;
            if (p >= nnz) break;
            while (next <= p) {
                ++r;
                start = next;
                next = __ldg(rp + r + 1);
            }
            const bool is_long = thr >= 0 && next - start > thr;
            const bool split = thr >= 0 && chunk > 0 && start / chunk != (next - 1) / chunk;
            const bool exact = is_long && next - start > kExactRow;
            out[p] = r | ((is_long || split) ? kLongFlag : 0) | (exact ? kExactFlag : 0);
        }
    }
}

// Adds the float64 side table of long rows into C (after the SpMM kernel).
template <typename T>
__global__ void __launch_bounds__(256)
k_long_rows_fold(T *__restrict__ C, int N, LongRows lr, int overwrite) {
    const long long total = (long long)(*lr.count) * N;
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < total;
         h += (long long)gridDim.x * blockDim.x) {
        const long long slot = h / N;
        const long long k = h - slot * N;
        const long long off = (long long)__ldg(lr.rows + slot) * N + k;
        const double base = overwrite ? 0.0 : (double)C[off];
        C[off] = (T)(base + lr.acc[h]);
        lr.acc[h] = 0.0;  // leave the table cleared for the next call
    }
}

// Overwrite-mode zero-fill for the owner-write walk: zero only the rows whose
// nonzeros span more than one g-position chunk (they receive atomic flushes),
// except long rows, which the side-table fold overwrites; empty rows are
// zeroed by the walk itself (zero_rows / zero_gap_before).  Lanes test one row each; the warp
// then clears the flagged rows cooperatively with 16-byte stores.
template <typename T>
__global__ void __launch_bounds__(256)
k_zero_shared_rows(const int *__restrict__ rp, int M, int N, long long g, long long thr,
                   T *__restrict__ C) {
    const long long items = ((long long)M + 31) >> 5;
    const unsigned lane = lane_id();
    // positions are < 2^31: 32-bit chunk numbers (a shift when g is a power
    // of two) -- two 64-bit divisions per row made this pass 6% of config 2
    const unsigned ug = (unsigned)g;
    const int shift = (ug & (ug - 1u)) == 0u ? __ffs((int)ug) - 1 : -1;
    SGAP_WARP_LOOP(item, items) {
        const long long r = item * 32 + lane;
        bool need = false;
        if (r < M) {
            const unsigned s = (unsigned)__ldg(rp + r), e = (unsigned)__ldg(rp + r + 1);
            const unsigned len = e - s;
            const bool split = shift >= 0 ? (s >> shift) != ((e - 1u) >> shift)
                                          : s / ug != (e - 1u) / ug;
            need = len > 0u && split && !(thr >= 0 && (long long)len > thr);
        }
        unsigned mask = __ballot_sync(kFull, need);
        while (mask) {
            const int src = __ffs(mask) - 1;
            mask &= mask - 1;
            T *row = C + (item * 32 + src) * (long long)N;
            // 16-byte stores only when every row is 16-byte aligned (row
            // stride a multiple of 16 and C itself aligned: a C-ABI caller
            // may pass a 4- or 8-byte aligned buffer)
            if ((N * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0) {
                float4 *r4 = reinterpret_cast<float4 *>(row);
                const int n4 = (int)(N * sizeof(T) / 16);
                for (int x = lane; x < n4; x += 32) r4[x] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                for (int x = lane; x < N; x += 32) row[x] = T(0);
            }
        }
    }
}

// Marks rows longer than `threshold` (input to the ordered compaction).
struct LongRowPred {
    const int *rp;
    long long threshold;
    long long chunk;  // > 0: rows straddling a chunk boundary join the table
    __host__ __device__ __forceinline__ bool operator()(const int &r) const {
        const long long s = rp[r], e = rp[r + 1];
        if (e - s > threshold) return true;
        return chunk > 0 && e > s && s / chunk != (e - 1) / chunk;
    }
};

// Plan-time row statistics (sgap_plan): out[0] = longest row, out[1] = rows
// the float64 table takes (longer than thr, or straddling a `chunk`
// boundary), out[2] = rows of the error-free pass (longer than exact_cut).
// One warp reduction and three atomics per warp.
__global__ void __launch_bounds__(256)
k_row_stats(const int *__restrict__ rp, int M, long long thr, long long chunk,
            long long exact_cut, unsigned long long *__restrict__ out) {
    const long long items = ((long long)M + 31) >> 5;
    const unsigned lane = lane_id();
    unsigned long long longest = 0, tab = 0, ex = 0;
    SGAP_WARP_LOOP(item, items) {
        const long long r = item * 32 + lane;
        if (r < M) {
            const long long s = __ldg(rp + r), e = __ldg(rp + r + 1);
            const long long len = e - s;
            longest = len > (long long)longest ? (unsigned long long)len : longest;
            const bool split = chunk > 0 && len > 0 && s / chunk != (e - 1) / chunk;
            tab += (thr >= 0 && (len > thr || split)) ? 1 : 0;
            ex += len > exact_cut ? 1 : 0;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long l2 = __shfl_xor_sync(kFull, longest, o);
        longest = l2 > longest ? l2 : longest;
        tab += __shfl_xor_sync(kFull, tab, o);
        ex += __shfl_xor_sync(kFull, ex, o);
    }
    if (lane == 0) {
        atomicMax(out, longest);
        if (tab) atomicAdd(out + 1, tab);
        if (ex) atomicAdd(out + 2, ex);
    }
}

// CsrMatrix invariants (matrices.py:58-75), pass 1: row_ptr.  *fault = the
// smallest row_ptr index r that breaks row_ptr[0] == 0, row_ptr[r] <=
// row_ptr[r+1] or row_ptr[M] == nnz (atomicMin; ULLONG_MAX = none).
__global__ void __launch_bounds__(256)
k_validate_row_ptr(const int *__restrict__ rp, long long M, long long nnz,
                   unsigned long long *__restrict__ fault) {
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r <= M;
         r += (long long)gridDim.x * blockDim.x) {
        const long long v = __ldg(rp + r);
        bool bad = (r == 0 && v != 0) || (r == M && v != nnz) || v < 0 || v > nnz;
        if (r < M && __ldg(rp + r + 1) < v) bad = true;
        if (bad) atomicMin(fault, (unsigned long long)r);
    }
}

// Pass 2 (row_ptr already valid): every column in [0, K) and strictly
// increasing within its row.  *fault = the smallest offending position.
__global__ void __launch_bounds__(256)
k_validate_cols(const int *__restrict__ rp, const int *__restrict__ ci, int M, long long K,
                long long nnz, unsigned long long *__restrict__ fault) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (long long)gridDim.x * blockDim.x) {
        const int c = __ldg(ci + p);
        bool bad = c < 0 || (long long)c >= K;
        if (!bad && p + 1 < nnz) {
            // end of p's row: the first row_ptr entry above p
            int lo = 0, hi = M;
            while (lo < hi) {
                const int mid = (int)(((unsigned)lo + (unsigned)hi) >> 1);
                if ((long long)__ldg(rp + mid + 1) <= p) lo = mid + 1; else hi = mid;
            }
            const long long end = __ldg(rp + lo + 1);
            if (p + 1 < end && __ldg(ci + p + 1) <= c) bad = true;
        }
        if (bad) atomicMin(fault, (unsigned long long)p);
    }
}

// Plan-time cold-column hints (SGAP_PLAN_L2_HINTS): gather counts per
// column, then a copy of col_idx with bit 31 set on columns gathered fewer
// than `thr` times (outside the hot set the L2 can keep).
__global__ void __launch_bounds__(256)
k_col_counts(const int *__restrict__ ci, long long nnz, long long K,
             unsigned *__restrict__ counts) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (long long)gridDim.x * blockDim.x) {
        const int c = __ldg(ci + p);
        // an unvalidated CSR may hold out-of-range columns: never write outside
        if (c >= 0 && (long long)c < K) atomicAdd(counts + c, 1u);
    }
}

__global__ void __launch_bounds__(256)
k_col_hints(const int *__restrict__ ci, long long nnz, long long K,
            const unsigned *__restrict__ counts, const unsigned *__restrict__ thr,
            int *__restrict__ out) {
    const unsigned t = *thr;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
         p += (long long)gridDim.x * blockDim.x) {
        const int c = __ldg(ci + p);
        const bool in = c >= 0 && (long long)c < K;
        out[p] = in && __ldg(counts + c) < t ? (int)((unsigned)c | 0x80000000u) : c;
    }
}

// Row -> slot map of the table (only the table's rows are written).
__global__ void k_long_slots(const int *__restrict__ rows, const int *__restrict__ count,
                             int *__restrict__ slot) {
    const int n = *count;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        slot[rows[i]] = i;
}

// The verification product of runner.verify_point (runner.py:193-194): the
// dense reference C = A@B in float64, per (i,k) ascending-p order with the
// multiply and the add rounded separately (no FMA contraction) -- the same
// arithmetic as matrices.dense_spmm_oracle (matrices.py:241-254), evaluated on
// the device so the check needs no host SpMM.  One lane per (i, k); lanes of a
// warp run along k, so every B-row read is coalesced.
template <typename T>
__global__ void __launch_bounds__(256)
k_reference_f64(const int *__restrict__ rp, const int *__restrict__ ci,
                const T *__restrict__ av, const T *__restrict__ B, double *__restrict__ C,
                int M, int N) {
    const long long cells = (long long)M * N;
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < cells;
         h += (long long)gridDim.x * blockDim.x) {
        const long long i = h / N;
        const long long k = h - i * N;
        double acc = 0.0;
        const int end = __ldg(rp + i + 1);
        for (int p = __ldg(rp + i); p < end; ++p) {
            const double prod = __dmul_rn((double)__ldg(av + p),
                                          (double)__ldg(B + (long long)__ldg(ci + p) * N + k));
            acc = __dadd_rn(acc, prod);
        }
        C[h] = acc;
    }
}

// lowering.compute_block_starts (lowering.py:119-128) on the device.
__global__ void k_block_starts(const int *__restrict__ rp, long long M, long long chunk,
                               long long nb, int *__restrict__ out) {
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    const long long t = b * chunk;
    long long lo = 0, hi = M + 1;
    while (lo < hi) {
        const long long mid = lo + ((hi - lo) >> 1);
        if ((long long)__ldg(rp + mid) <= t) lo = mid + 1; else hi = mid;
    }
    out[b] = (int)(lo - 1);
}

// ===========================================================================
// The simulator's group macros over explicit lane vectors (sim.py:112-165),
// running the same seg_lanes / seg_scan / group_sum code as the kernels.
// ===========================================================================
template <typename T, int R>
__global__ void __launch_bounds__(256)
k_seg_reduce_prim(const long long *__restrict__ idx, const T *__restrict__ val,
                  const unsigned char *__restrict__ active, long long lanes, T *out,
                  long long out_len, unsigned long long *wb, long long *fault) {
    const long long items = (lanes + 31) >> 5;
    unsigned long long nwb = 0;
    SGAP_WARP_LOOP(item, items) {
        const long long L = item * 32 + lane_id();
        const bool act = L < lanes && (active == nullptr || active[L] != 0);
        const long long key = act ? idx[L] : 0;
        const T v = act ? val[L] : T(0);
        const SegLanes s = seg_lanes<R, long long>(key, act);
        if (s.decreasing) atomicMin(fault, L);
        const T sum = seg_scan<R, T>(v, s.dist);
        if (s.tail) {
            if (key < 0 || key >= out_len) atomicMin(fault, L);
            else atomicAdd(out + key, sum);
            ++nwb;
        }
    }
    flush_count(wb, nwb);
}

template <typename T, int R>
__global__ void __launch_bounds__(256)
k_atomic_add_prim(const long long *__restrict__ idx, const T *__restrict__ val,
                  const unsigned char *__restrict__ active, long long lanes, T *out,
                  long long out_len, unsigned long long *wb, long long *fault) {
    const long long items = (lanes + 31) >> 5;
    unsigned long long nwb = 0;
    const unsigned lane = lane_id();
    SGAP_WARP_LOOP(item, items) {
        const long long L = item * 32 + lane;
        const bool act = L < lanes && (active == nullptr || active[L] != 0);
        const long long key = act ? idx[L] : 0;
        T v = act ? val[L] : T(0);
        long long lo = act ? key : LLONG_MAX, hi = act ? key : LLONG_MIN;
#pragma unroll
        for (int off = R / 2; off > 0; off >>= 1) {
            lo = min(lo, __shfl_xor_sync(kFull, lo, off, R));
            hi = max(hi, __shfl_xor_sync(kFull, hi, off, R));
        }
        v = group_sum<R, T>(v);
        const unsigned gbase = lane & ~(unsigned)(R - 1);
        const unsigned gmask = (R >= 32) ? kFull : (((1u << R) - 1u) << gbase);
        const unsigned act_mask = __ballot_sync(kFull, act) & gmask;
        const bool leader = act_mask != 0u && (int)lane == __ffs(act_mask) - 1;
        if (leader) {
            if (lo != hi || key < 0 || key >= out_len) atomicMin(fault, L);
            else atomicAdd(out + key, v);
            ++nwb;
        }
    }
    flush_count(wb, nwb);
}

}  // namespace sgap
