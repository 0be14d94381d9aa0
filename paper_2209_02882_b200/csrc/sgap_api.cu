// sgap_api.cu -- the C ABI (include/sgap.h): host-side planning that mirrors
// the reference's template gates and launch geometry, and stream-ordered
// dispatch of the sm_100a kernels.  No allocation, no global mutable state.
#include <cstdlib>
#include <climits>
#include <cstdint>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>
#include <thrust/iterator/counting_iterator.h>

#include "../../include/sgap.h"
#include "sgap_kernels.cuh"
#include "sgap_ingest.cuh"

using namespace sgap;

namespace {

constexpr int kHwBlock = 256;
// CTA size of the register EB walk (hw variant 1): same 32 warps/SM at 64
// registers, finer blocks balance the long-chunk tail better -- config 2
// 0.693 ms at 128 vs 0.701 at 256 (96: 0.732, 160-192: 0.745); config 3
// 2.037 vs 2.108 ms (64: 2.015).
constexpr int kEbWalkBlock = 128;

inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

inline int pow2_floor(long long x) {
    int p = 1;
    while ((long long)p * 2 <= x && p < 32) p *= 2;
    return p;
}

inline int amount_units(int kind, int param) { return kind == SGAP_AMT_ONE ? 1 : param; }

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int launch_status() {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SGAP_OK : SGAP_ERR_CUDA;
}

inline unsigned grid_for(long long items_per_warp_units, int block) {
    // warps needed, then CTAs; kernels grid-stride past this cap
    long long warps = items_per_warp_units;
    long long ctas = ceil_div(warps, block / 32);
    if (ctas < 1) ctas = 1;
    if (ctas > (1LL << 30)) ctas = 1LL << 30;
    return (unsigned)ctas;
}

bool aligned(const void *p, size_t bytes) {
    return (reinterpret_cast<uintptr_t>(p) % bytes) == 0;
}

// Launch with programmatic stream serialisation when `pdl` (the kernel may
// start while the previous grid on the stream is still running; it calls
// griddepcontrol.wait before it exits).
template <typename... KArgs, typename... Args>
int launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
             bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...) == cudaSuccess
               ? SGAP_OK : SGAP_ERR_CUDA;
}

// ------------------------------------------------------------------ dispatch

// hw_variant for row-multiple: 0/1 the logical mapping (thread (rg, t) owns
// rows rg*g .. rg*g+g-1), 2 the interleaved mapping (a CTA's warps on adjacent
// rows; needs N/c <= CTA size), 3/4 the interleaved mapping with a warp per
// row and lane-staged A (8/4 gathers in flight; N/c == 32, once per
// 32c-column panel when N/c is a larger multiple of 32, and 2 / 4 / 8 / 16
// rows per warp at N/c == 16 / 8 / 4 / 2), 6/7 the row-blocked union walk
// (N/c == 32), 8 the shifted-block walk (4 rows per warp; N/c a multiple
// of 32, panels as 3/4).
template <typename T, int V>
int run_row_multiple(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                     int acc, const LongRows &lr, cudaStream_t st) {
    const int N = k.n, L = N / V;
    const int blk = k.hw_block > 0 ? k.hw_block : kHwBlock;
    const int vec4 = aligned(a.d_col_idx, 16) && aligned(a.d_vals, 16);
    if (k.hw_variant == 6 || k.hw_variant == 7) {  // row-blocked union walk
        const int which = k.hw_variant - 6;
        if (L != 32 || lr.union_e[which] == nullptr) return SGAP_ERR_ARG;
        const int R = which ? 8 : 4;
        const long long nblocks = ceil_div(a.num_rows, R);
        const long long tile_blocks = (long long)(blk / 32) * k.g;
        const long long tiles = ceil_div(nblocks, tile_blocks);
        const unsigned ctas = (unsigned)(tiles < (1LL << 30) ? (tiles > 0 ? tiles : 1) : (1LL << 30));
        const T *Av = static_cast<const T *>(a.d_vals);
        const size_t smem = (size_t)(blk / 32) * 32 * R * sizeof(T);  // per-warp value slabs
        if (blk % 32 || smem > 48 * 1024) return SGAP_ERR_ARG;
        if (which == 0)
            k_row_blocked<T, V, 4, 4, 4><<<ctas, blk, smem, st>>>(a.d_row_ptr, lr.union_e[0],
                                                               lr.union_off[0], Av, B, C,
                                                               (int)a.num_rows, N, k.g, acc);
        else
            k_row_blocked<T, V, 8, 2, 3><<<ctas, blk, smem, st>>>(a.d_row_ptr, lr.union_e[1],
                                                               lr.union_off[1], Av, B, C,
                                                               (int)a.num_rows, N, k.g, acc);
        return launch_status();
    }
    if (k.hw_variant == 8) {  // shifted blocks of 4 rows
        // N/c == 32, or one pass per 32c-column panel (as variant 4); N/c ==
        // 16 / 8: 2 / 4 lane groups of 4 rows per warp.  The block's values sit
        // in a per-warp shared slab (RB rows x 33, padded against bank
        // conflicts) read as broadcasts: config 4 N=128 / 256 / 64 / 32 0.94 /
        // 0.94 / 0.89 / 0.95x of shuffling them from lane registers (which at
        // N/c == 8 spilled to local memory: 1.33x slower than variant 4)
        // 64-thread CTAs by default (config 4 N=128 / 256: 0.98 / 0.89-0.97x of
        // 128 threads, which are 0.91x of 256)
        const int sblk = k.hw_block > 0 ? k.hw_block : 64;
        if (L == 8) {  // 4 lane groups of 4 rows
            const long long nwb = ceil_div(a.num_rows, 16);
            const long long want = ceil_div(nwb, sblk / 32);
            const unsigned ctas = (unsigned)(want < (1LL << 30) ? (want > 0 ? want : 1) : (1LL << 30));
            const size_t smem = (size_t)(sblk / 32) * 16 * 33 * sizeof(T);
            k_row_shifted_sub<T, V, 8, 4, true><<<ctas, sblk, smem, st>>>(
                a.d_row_ptr, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, (int)a.num_rows, N,
                vec4, acc);
            return launch_status();
        }
        if (L == 16) {  // 2 lane groups of 4 rows
            const long long nwb = ceil_div(a.num_rows, 8);
            const long long want = ceil_div(nwb, sblk / 32);
            const unsigned ctas = (unsigned)(want < (1LL << 30) ? (want > 0 ? want : 1) : (1LL << 30));
            const T *Av = static_cast<const T *>(a.d_vals);
            const size_t smem = (size_t)(sblk / 32) * 8 * 33 * sizeof(T);
            k_row_shifted_sub<T, V, 16, 4, true><<<ctas, sblk, smem, st>>>(a.d_row_ptr, a.d_col_idx, Av, B, C,
                                                                           (int)a.num_rows, N, vec4, acc);
            return launch_status();
        }
        if (L % 32) return SGAP_ERR_ARG;
        const long long nblocks = ceil_div(a.num_rows, 4);
        const long long want = ceil_div(nblocks, sblk / 32);
        const unsigned ctas = (unsigned)(want < (1LL << 30) ? (want > 0 ? want : 1) : (1LL << 30));
        const T *Av = static_cast<const T *>(a.d_vals);
        const int M = (int)a.num_rows;
        for (int pan = 0; pan < L / 32; ++pan) {
            const long long off = (long long)pan * 32 * V;
            k_row_shifted<T, V, 4, true><<<ctas, sblk, (size_t)(sblk / 32) * 4 * 33 * sizeof(T), st>>>(
                a.d_row_ptr, a.d_col_idx, Av, B + off, C + off, M, N, vec4, acc);
            const int s0 = launch_status();
            if (s0 != SGAP_OK) return s0;
        }
        return SGAP_OK;
    }
    if (k.hw_variant == 3 || k.hw_variant == 4) {  // lane-staged, a warp per row
        // N/c == 32: one pass.  N/c a multiple of 32 (N >= 256 at c = 4): one
        // pass per 32c-column panel, in place -- B and C keep their N-wide
        // rows (the kernel's N is the row stride), each pass walks every row
        // for its panel only, so the stencil's sliding window of B rows (one
        // z-plane either side) is 32c columns wide instead of N while it is
        // re-read (config 4 N=256/512: separate contiguous 128-column
        // SpMMs 0.82x of the best full-width schedule,
        // tools/experiments/stencil_panel_probe.py)
        if (L == 16 || L == 8 || L == 4 || L == 2) {  // 2 / 4 / 8 / 16 rows per warp
            const long long tile_rows = (long long)(blk / 32) * k.g * (32 / L);
            const long long tiles = ceil_div(a.num_rows, tile_rows);
            const unsigned ctas =
                (unsigned)(tiles < (1LL << 30) ? (tiles > 0 ? tiles : 1) : (1LL << 30));
            const T *Av = static_cast<const T *>(a.d_vals);
            const int M = (int)a.num_rows;
            if (L == 16) {
                if (k.hw_variant == 3)
                    k_row_staged_sub<T, V, 8, 16><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B, C, M, N, k.g, vec4, acc);
                else
                    k_row_staged_sub<T, V, 4, 16><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B, C, M, N, k.g, vec4, acc);
            } else if (L == 8) {
                if (k.hw_variant == 3)
                    k_row_staged_sub<T, V, 8, 8><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B, C, M, N, k.g, vec4, acc);
                else
                    k_row_staged_sub<T, V, 4, 8><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B, C, M, N, k.g, vec4, acc);
            } else if (L == 4) {  // U > LPR would only re-gather the segment
                k_row_staged_sub<T, V, 4, 4><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B, C, M, N, k.g, vec4, acc);
            } else {
                k_row_staged_sub<T, V, 2, 2><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B, C, M, N, k.g, vec4, acc);
            }
            return launch_status();
        }
        if (L % 32) return SGAP_ERR_ARG;
        const long long tile_rows = (long long)(blk / 32) * k.g;
        const long long tiles = ceil_div(a.num_rows, tile_rows);
        const unsigned ctas = (unsigned)(tiles < (1LL << 30) ? (tiles > 0 ? tiles : 1) : (1LL << 30));
        const T *Av = static_cast<const T *>(a.d_vals);
        const int M = (int)a.num_rows;
        for (int pan = 0; pan < L / 32; ++pan) {
            const long long off = (long long)pan * 32 * V;
            if (k.hw_variant == 3)
                k_row_staged<T, V, 8><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B + off,
                                                             C + off, M, N, k.g, vec4, acc, -1);
            else
                k_row_staged<T, V, 4><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx, Av, B + off,
                                                             C + off, M, N, k.g, vec4, acc, -1);
            const int s0 = launch_status();
            if (s0 != SGAP_OK) return s0;
        }
        return SGAP_OK;
    }
    if (k.hw_variant == 2) {
        if (L > blk) return SGAP_ERR_ARG;
        const long long tile_rows = (long long)(blk / L) * k.g;
        const long long tiles = ceil_div(a.num_rows, tile_rows);
        const unsigned ctas = (unsigned)(tiles < (1LL << 30) ? (tiles > 0 ? tiles : 1) : (1LL << 30));
        k_row_interleaved<T, V><<<ctas, blk, 0, st>>>(a.d_row_ptr, a.d_col_idx,
                                                      static_cast<const T *>(a.d_vals), B, C,
                                                      (int)a.num_rows, N, k.g, vec4, acc);
        return launch_status();
    }
    const long long total = ceil_div(a.num_rows, k.g) * (long long)L;
    k_row_multiple<T, V><<<grid_for(ceil_div(total, 32), blk), blk, 0, st>>>(
        a.d_row_ptr, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, (int)a.num_rows, N,
        k.g, vec4, acc);
    return launch_status();
}

template <typename T, int V, int G>
int run_row_reciprocal_g(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                         int acc, unsigned long long *wb, cudaStream_t st) {
    const long long cells = a.num_rows * (long long)k.n;
    const long long total = ceil_div(cells, V) * G;
    const int blk = k.hw_block > 0 ? k.hw_block : kHwBlock;
    const int n_shift = (k.n & (k.n - 1)) == 0 ? __builtin_ctz((unsigned)k.n) : -1;
    const unsigned grid = grid_for(ceil_div(total, 32), blk);
    if (cells + 64 < (1LL << 32) && a.num_cols * (long long)k.n < (1LL << 32))
        k_row_reciprocal<T, V, G, unsigned><<<grid, blk, 0, st>>>(
            a.d_row_ptr, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, (int)a.num_rows,
            k.n, n_shift, acc, wb);
    else
        k_row_reciprocal<T, V, G, long long><<<grid, blk, 0, st>>>(
            a.d_row_ptr, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, (int)a.num_rows,
            k.n, n_shift, acc, wb);
    return launch_status();
}

template <typename T, int V>
int run_row_reciprocal(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C, int acc,
                       unsigned long long *wb, cudaStream_t st) {
    switch (k.g) {
        case 2: return run_row_reciprocal_g<T, V, 2>(k, a, B, C, acc, wb, st);
        case 4: return run_row_reciprocal_g<T, V, 4>(k, a, B, C, acc, wb, st);
        case 8: return run_row_reciprocal_g<T, V, 8>(k, a, B, C, acc, wb, st);
        case 16: return run_row_reciprocal_g<T, V, 16>(k, a, B, C, acc, wb, st);
        case 32: return run_row_reciprocal_g<T, V, 32>(k, a, B, C, acc, wb, st);
        default: return SGAP_ERR_NO_TEMPLATE;
    }
}

template <typename T, int V, int R>
int run_nnz_one_r(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                  const int *rowid, const LongRows &lr, unsigned long long *wb, cudaStream_t st) {
    const int NT = k.n / V;
    const int TW = pow2_floor(NT < 32 / R ? NT : 32 / R);
    const int Q = 32 / TW;
    const long long total_pos = k.grid_size * k.chunk;
    const long long items = ceil_div(total_pos, 4LL * Q);  // kSteps groups of Q per warp item
    const int blk = k.hw_block > 0 ? k.hw_block : kHwBlock;
    k_nnz_one<T, V, R><<<grid_for(items, blk), blk, 0, st>>>(
        rowid, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, (int)a.num_rows, k.n, a.nnz,
        total_pos, TW, lr, wb);
    return launch_status();
}

template <typename T, int V, int W>
int run_nnz_multiple_w(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                       const int *rowid, const LongRows &lr, int owner, bool has_exact,
                       bool zero, unsigned long long *wb, cudaStream_t st);

// nnz-one hw variant 1: each aligned segment group of r positions walked
// serially by N/c lanes along the columns (the register walk with g = r, one
// red per segment -- the same writebacks as the shuffle scan, which gathers
// B rows in (32/r)-tile pieces); the group straddling nnz adds the padded run
// (owner mode 2 in k_nnz_multiple).
template <typename T, int V>
int run_nnz_one_walk(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                     const int *rowid, const LongRows &lr, unsigned long long *wb,
                     cudaStream_t st) {
    sgap_kernel_t km = k;
    km.family = SGAP_NNZ_MULTIPLE;
    km.g = k.r;
    km.hw_variant = 5;  // the row-id walk (the nnz-one plan has row ids, no chunk rows)
    km.hw_block = 0;
    LongRows lw = lr;
    lw.chunk_rows = nullptr;
    // owner mode 2: segment groups (r > 1, padded lanes are a run of row
    // M-1); 3: r = 1 atomics (lanes past nnz do not write)
    const int mode = k.r > 1 ? 2 : 3;
    switch (pow2_floor(k.n / V)) {
        case 1: return run_nnz_multiple_w<T, V, 1>(km, a, B, C, rowid, lw, mode, false, false, wb, st);
        case 2: return run_nnz_multiple_w<T, V, 2>(km, a, B, C, rowid, lw, mode, false, false, wb, st);
        case 4: return run_nnz_multiple_w<T, V, 4>(km, a, B, C, rowid, lw, mode, false, false, wb, st);
        case 8: return run_nnz_multiple_w<T, V, 8>(km, a, B, C, rowid, lw, mode, false, false, wb, st);
        case 16: return run_nnz_multiple_w<T, V, 16>(km, a, B, C, rowid, lw, mode, false, false, wb, st);
        default: return run_nnz_multiple_w<T, V, 32>(km, a, B, C, rowid, lw, mode, false, false, wb, st);
    }
}

template <typename T, int V>
int run_nnz_one(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                const int *rowid, const LongRows &lr, unsigned long long *wb, cudaStream_t st) {
    if (k.hw_variant == 1) return run_nnz_one_walk<T, V>(k, a, B, C, rowid, lr, wb, st);
    if (k.hw_variant != 0) return SGAP_ERR_ARG;
    switch (k.r) {
        case 1: return run_nnz_one_r<T, V, 1>(k, a, B, C, rowid, lr, wb, st);
        case 2: return run_nnz_one_r<T, V, 2>(k, a, B, C, rowid, lr, wb, st);
        case 4: return run_nnz_one_r<T, V, 4>(k, a, B, C, rowid, lr, wb, st);
        case 8: return run_nnz_one_r<T, V, 8>(k, a, B, C, rowid, lr, wb, st);
        case 16: return run_nnz_one_r<T, V, 16>(k, a, B, C, rowid, lr, wb, st);
        case 32: return run_nnz_one_r<T, V, 32>(k, a, B, C, rowid, lr, wb, st);
        default: return SGAP_ERR_NO_TEMPLATE;
    }
}

// TMA tile: the largest multiple of lcm(g, 4) that fits a stage (so tiles
// start on chunk boundaries and on 16-byte boundaries); 0 when none does.
inline int tma_tile_for(int g) {
    long long l = g;
    while (l % 4) l += g;
    if (l > kTmaTile) return 0;
    return (int)((kTmaTile / l) * l);
}

template <typename T, int V, int W, int U, int STAGES = 3, int MINB = 3>
int launch_nnz_multiple(bool tma, int tile, int owner, const sgap_kernel_t &k,
                        const sgap_csr_t &a, const T *B, T *C, const int *rowid,
                        const LongRows &lr, unsigned long long *wb, cudaStream_t st, bool pdl,
                        int exact_inline, const int *chunk_rows, int panel = 0) {
    const long long total_pos = k.grid_size * k.chunk;
    if (tma) {
        const size_t smem = tma_smem_bytes<T, STAGES>();
        auto kern = k_nnz_multiple_tma<T, V, W, U, STAGES, MINB>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return SGAP_ERR_CUDA;
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTmaThreads, smem);
        const long long ntiles = ceil_div(total_pos, tile);
        long long ctas = (long long)sms * (per_sm > 0 ? per_sm : 1);
        if (ctas > ntiles) ctas = ntiles;
        if (ctas < 1) ctas = 1;
        return launch_k(kern, dim3((unsigned)ctas), dim3(kTmaThreads), smem, st, pdl, rowid,
                        a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, a.d_row_ptr,
                        (int)a.num_rows, k.n, a.nnz, k.g, total_pos, tile, owner, lr, wb);
    }
    const long long items = ceil_div(total_pos / k.g, 32 / W);
    const int blk = k.hw_block > 0 ? k.hw_block : kEbWalkBlock;
    const int vec4 = (k.g % 4 == 0) && aligned(rowid, 16) && aligned(a.d_col_idx, 16) &&
                     aligned(a.d_vals, 16);
    if (k.hw_variant == 9) {  // + cold-column cache hints (the plan's flagged col_idx)
        // + the B rows two batches ahead prefetched into L2 (config 5: -3.8%
        // at one batch, another -2.6% at two, none at four, +2% at eight;
        // the L2-resident configs lose 2-6% to it, so only this variant has it)
        if (!vec4 || chunk_rows == nullptr || lr.col_hinted == nullptr) return SGAP_ERR_ARG;
        return launch_k(k_nnz_multiple<T, V, W, U, true, true, true, 2>, dim3(grid_for(items, blk)),
                        dim3(blk), 0, st, pdl, rowid, lr.col_hinted, static_cast<const T *>(a.d_vals),
                        B, C, a.d_row_ptr, (int)a.num_rows, k.n, a.nnz, k.g, total_pos, vec4, owner,
                        lr, wb, exact_inline, chunk_rows, 0);
    }
    if constexpr (W >= 8) {
        if (panel) {  // variant 10: variant 1, one launch per column panel
            if (!vec4 || chunk_rows == nullptr) return SGAP_ERR_ARG;
            // (kernel boundaries keep every warp on one panel: a single
            // launch looping over the panels let warps drift across two
            // panels and was 1.19x slower than variant 1 on config 3 N=256)
            constexpr int PW = W * V;
            const int passes = (int)ceil_div(k.n, PW);
            const long long K = a.num_cols;
            T *P = static_cast<T *>(lr.panel_b);
            const long long vecs = K * passes * (PW * (int)sizeof(T) / 16);
            k_panelize<T><<<grid_for(ceil_div(vecs, 32), kHwBlock), kHwBlock, 0, st>>>(B, P, K, k.n,
                                                                                     PW);
            const int sp = launch_status();
            if (sp != SGAP_OK) return sp;
            auto kern = k_nnz_multiple<T, V, W, U, true, false, false, 1, true>;
            for (int ps = 0; ps < passes; ++ps) {
                const int s0 = launch_k(kern,
                                        dim3(grid_for(items, blk)), dim3(blk), 0, st, pdl && ps == 0,
                                        rowid, a.d_col_idx, static_cast<const T *>(a.d_vals),
                                        static_cast<const T *>(P + (long long)ps * K * PW), C,
                                        a.d_row_ptr, (int)a.num_rows, k.n, a.nnz, k.g, total_pos,
                                        vec4, owner, lr, wb, exact_inline, chunk_rows, ps);
                if (s0 != SGAP_OK) return s0;
            }
            return SGAP_OK;
        }
    }
    if (panel) return SGAP_ERR_ARG;
    if (vec4 && chunk_rows != nullptr)  // row_ptr tracking, no per-position row ids
        return launch_k(k_nnz_multiple<T, V, W, U, true>, dim3(grid_for(items, blk)), dim3(blk), 0,
                        st, pdl, rowid, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C,
                        a.d_row_ptr, (int)a.num_rows, k.n, a.nnz, k.g, total_pos, vec4, owner, lr,
                        wb, exact_inline, chunk_rows, 0);
    return launch_k(k_nnz_multiple<T, V, W, U, false>, dim3(grid_for(items, blk)), dim3(blk), 0, st,
                    pdl, rowid, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, a.d_row_ptr,
                    (int)a.num_rows, k.n, a.nnz, k.g, total_pos, vec4, owner, lr, wb, exact_inline,
                    (const int *)nullptr, 0);
}

// hw_variant: 0 auto; 1 register walk; 2 TMA-staged walk; 3/4 lane-staged walk
// (whole warp per chunk, 4/8 gathers in flight; needs N/c >= 32).  Measured on config
// 2 (profiles/): software pipelining and 8-deep batches were slower (the extra
// registers cost more occupancy than the added in-flight gathers recover), as
// were L2 evict-first hints on the A stream, L1::no_allocate / evict_last on
// the B gathers, and per-lane cp.async (LDGSTS) gathers into a 4-stage shared
// ring (1.21 vs 0.77 ms); the TMA walk needs 3 CTAs/SM (3-stage ring, <= 75
// registers) to beat the register walk.
template <typename T, int V, int W>
int run_nnz_multiple_w(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                       const int *rowid, const LongRows &lr, int owner, bool has_exact,
                       bool zero, unsigned long long *wb, cudaStream_t st) {
    const int tile = tma_tile_for(k.g);
    const bool tma_ok = tile > 0 && aligned(rowid, 16) && aligned(a.d_col_idx, 16) &&
                        aligned(a.d_vals, 16);
    // auto: the TMA-staged walk wins for short chunks with wide lane groups
    // (g <= 128, >= 16 lanes per chunk: config 2, Chung-Lu N=64); the register
    // walk for long chunks (fewer, longer walks amortise the A loads it issues
    // itself) and for narrow N (profiles/r01_selector_regret.json)
    int variant = k.hw_variant == 0 ? ((tma_ok && W >= 16 && k.g <= 128) ? 2 : 1) : k.hw_variant;
    const bool tma = variant == 2;
    // every check that can reject the call runs before the first launch: an
    // error after the exact pass would leave its sums in the float64 table
    // (never folded, so a later call on the same plan would add them to C)
    if (tma && !tma_ok) return SGAP_ERR_ARG;
    if (variant == 9) {  // variant 1 with the plan's cold-column cache hints
        const int vec4 = (k.g % 4 == 0) && aligned(a.d_col_idx, 16) && aligned(a.d_vals, 16);
        if (lr.col_hinted == nullptr || lr.chunk_rows == nullptr || !vec4) return SGAP_ERR_ARG;
        variant = 1;
    }
    const int panel = variant == 10 ? 1 : 0;
    if (panel) {  // variant 1 in column-panel order (W lanes = one panel)
        const int vec4 = (k.g % 4 == 0) && aligned(rowid, 16) && aligned(a.d_col_idx, 16) &&
                         aligned(a.d_vals, 16);
        constexpr int E = 16 / (int)sizeof(T);  // k_panelize moves 16-byte vectors
        if (lr.chunk_rows == nullptr || !vec4 || W < 8 || W >= k.n / V || lr.panel_b == nullptr ||
            W != lr.panel_lanes || k.n % E || (W * V) % E || !aligned(B, 16))
            return SGAP_ERR_ARG;
        variant = 1;
    }
    if (variant < 1 || variant > 5) return SGAP_ERR_ARG;
    const bool staged = variant == 3 || variant == 4;
    if (staged && W != 32) return SGAP_ERR_ARG;  // the staged walk takes a whole warp
    if (staged && k.hw_block > 0 && k.hw_block != kHwBlock) return SGAP_ERR_ARG;
    if (tma) {
        const size_t smem = tma_smem_bytes<T, 3>();
        if (cudaFuncSetAttribute(k_nnz_multiple_tma<T, V, W, 4, 3, 3>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return SGAP_ERR_CUDA;
    }
    if (zero) {
        k_zero_shared_rows<T><<<grid_for(ceil_div(a.num_rows, 32), kHwBlock), kHwBlock, 0, st>>>(
            a.d_row_ptr, (int)a.num_rows, k.n, k.g, lr.threshold, C);
    }
    // chunks inside exact-flagged rows (error-free accumulate) run in their
    // own kernel, launched first; the main walk follows with programmatic
    // dependent launch, so the two overlap (no data dependency: both only add
    // into the float64 table) and the walk's grid exits after the exact pass
    bool pdl = false;
    // the register walk (variant 1) takes exact chunks inline (float64
    // products); the other walks leave them to k_nnz_multiple_exact
    const bool exact_inline = (variant == 1 || variant == 5) && lr.threshold >= 0 && sizeof(T) == 4;
    if (!exact_inline && lr.threshold >= 0 && sizeof(T) == 4 && has_exact && lr.exact_count > 0 &&
        lr.exact_rows != nullptr) {
        const int vec4 = (k.g % 4 == 0) && aligned(rowid, 16) && aligned(a.d_col_idx, 16) &&
                         aligned(a.d_vals, 16);
        const int gx = lr.exact_count < 1024 ? lr.exact_count : 1024;
        int gy = (2 * 148 * 8 + gx - 1) / gx;  // ~2 waves of 8-warp CTAs
        gy = gy < 1 ? 1 : (gy > 64 ? 64 : gy);
        k_nnz_multiple_exact<T, V><<<dim3((unsigned)gx, (unsigned)gy), kHwBlock, 0, st>>>(
            rowid, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, a.d_row_ptr, k.n, a.nnz,
            k.g, vec4, lr);
        const int s0 = launch_status();
        if (s0 != SGAP_OK) return s0;
        pdl = true;
    }
    if (variant == 3 || variant == 4) {
        const long long total_pos = k.grid_size * k.chunk;
        const long long chunks = total_pos / k.g;
        const int blk = kHwBlock;
        const dim3 grid(grid_for(chunks, blk));
        if (variant == 3)
            return launch_k(k_nnz_multiple_staged<T, V, 4, 4>, grid, dim3(blk), 0, st, pdl, rowid,
                            a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, a.d_row_ptr,
                            (int)a.num_rows, k.n, a.nnz, k.g, total_pos, owner, lr, wb);
        return launch_k(k_nnz_multiple_staged<T, V, 8, 3>, grid, dim3(blk), 0, st, pdl, rowid,
                        a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, a.d_row_ptr,
                        (int)a.num_rows, k.n, a.nnz, k.g, total_pos, owner, lr, wb);
    }
    // variant 1 tracks rows through row_ptr when the plan has the chunk start
    // rows; variant 5 is the same walk on per-position row ids
    return launch_nnz_multiple<T, V, W, 4>(tma, tile, owner, k, a, B, C, rowid, lr, wb, st,
                                           pdl, exact_inline ? 1 : 0,
                                           variant == 1 ? lr.chunk_rows : nullptr, panel);
    // (k.hw_variant == 9 selects the cold-hint instantiation inside)
}

// Column-panel width for hw variant 10, in lanes of V columns: the widest
// power-of-two panel (8..32 lanes, at least two panels) whose B rows
// (num_cols x panel columns) fit in half the L2.  0 when none does or when
// the whole of B already fits (config 3 at N = 256: 16 lanes = 64 columns,
// 60 MB of B per panel against 238 MB for all of B; column-panel probe
// profiles/r02_panel_probe_cfg3_n256.log).
int panel_lanes(const sgap_kernel_t &k, const sgap_csr_t &a, int V, size_t esz) {
    int dev = 0, l2 = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess || l2 <= 0) return 0;
    const long long nt = k.n / V;
    if ((long long)a.num_cols * k.n * (long long)esz <= (long long)l2) return 0;
    for (int w = 32; w >= 8; w >>= 1)
        if (w < nt && (long long)a.num_cols * w * V * (long long)esz <= l2 / 2) return w;
    return 0;
}

template <typename T, int V>
int run_nnz_multiple(const sgap_kernel_t &k, const sgap_csr_t &a, const T *B, T *C,
                     const int *rowid, const LongRows &lr, int acc, bool has_exact,
                     unsigned long long *wb, cudaStream_t st) {
    // overwrite mode: zero only rows that will receive atomic flushes (or no
    // flush at all), then let the walk store complete rows outright; with
    // chunk routing every split row is in the float64 table, whose fold
    // overwrites it, so nothing needs zeroing
    const int owner = acc ? 0 : 1;
    const bool routed = lr.threshold >= 0 && lr.chunk == k.g;
    const bool zero = owner && !routed;  // launched by the walk after its checks
    if (k.hw_variant == 10) {  // column panels: W = the panel's lanes
        switch (lr.panel_lanes) {  // chosen by the planner (panel_lanes)
            case 8: return run_nnz_multiple_w<T, V, 8>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
            case 16: return run_nnz_multiple_w<T, V, 16>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
            case 32: return run_nnz_multiple_w<T, V, 32>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
            default: return SGAP_ERR_ARG;  // no panels in the plan (none fits half the L2,
                                           // B already does, or no SGAP_PLAN_PANELS)
        }
    }
    switch (pow2_floor(k.n / V)) {
        case 1: return run_nnz_multiple_w<T, V, 1>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
        case 2: return run_nnz_multiple_w<T, V, 2>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
        case 4: return run_nnz_multiple_w<T, V, 4>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
        case 8: return run_nnz_multiple_w<T, V, 8>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
        case 16: return run_nnz_multiple_w<T, V, 16>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
        default: return run_nnz_multiple_w<T, V, 32>(k, a, B, C, rowid, lr, owner, has_exact, zero, wb, st);
    }
}

template <typename T, int V>
int run_family(const sgap_kernel_t &k, const sgap_csr_t &a, const void *b, void *c, int acc,
               const int *rowid, const LongRows &lr, bool has_exact, unsigned long long *wb,
               cudaStream_t st) {
    const T *B = static_cast<const T *>(b);
    T *C = static_cast<T *>(c);
    switch (k.family) {
        case SGAP_ROW_MULTIPLE: return run_row_multiple<T, V>(k, a, B, C, acc, lr, st);
        case SGAP_ROW_RECIPROCAL: return run_row_reciprocal<T, V>(k, a, B, C, acc, wb, st);
        case SGAP_NNZ_ONE: return run_nnz_one<T, V>(k, a, B, C, rowid, lr, wb, st);
        case SGAP_NNZ_MULTIPLE:
            return run_nnz_multiple<T, V>(k, a, B, C, rowid, lr, acc, has_exact, wb, st);
        default: return SGAP_ERR_ARG;
    }
}

template <typename T>
int run_typed(const sgap_kernel_t &k, const sgap_csr_t &a, const void *b, void *c, int acc,
              const int *rowid, const LongRows &lr, bool has_exact, unsigned long long *wb,
              cudaStream_t st) {
    int status;
    switch (k.c) {
        case 1: status = run_family<T, 1>(k, a, b, c, acc, rowid, lr, has_exact, wb, st); break;
        case 2: status = run_family<T, 2>(k, a, b, c, acc, rowid, lr, has_exact, wb, st); break;
        case 4: status = run_family<T, 4>(k, a, b, c, acc, rowid, lr, has_exact, wb, st); break;
        default: return SGAP_ERR_NO_TEMPLATE;
    }
    if (status != SGAP_OK || lr.threshold < 0) return status;
    // fold the float64 side table of long rows into C (and clear it for the next call)
    long long cap_cells = (long long)k.n * 65536;
    unsigned blocks = (unsigned)ceil_div(cap_cells, kHwBlock);
    if (blocks > 4096) blocks = 4096;
    k_long_rows_fold<T><<<blocks, kHwBlock, 0, st>>>(static_cast<T *>(c), k.n, lr, acc ? 0 : 1);
    return launch_status();
}

template <typename T>
int prim_dispatch(bool seg, const int64_t *idx, const void *val, const uint8_t *active,
                  int64_t lanes, int gs, void *out, int64_t out_len,
                  unsigned long long *wb, long long *fault, cudaStream_t st) {
    const long long items = ceil_div(lanes, 32);
    const unsigned grid = grid_for(items, kHwBlock);
    auto *I = reinterpret_cast<const long long *>(idx);
    auto *Vv = static_cast<const T *>(val);
    auto *O = static_cast<T *>(out);
#define SGAP_PRIM(RR)                                                                    \
    case RR:                                                                              \
        if (seg) k_seg_reduce_prim<T, RR><<<grid, kHwBlock, 0, st>>>(I, Vv, active, lanes, \
                                                                      O, out_len, wb, fault); \
        else k_atomic_add_prim<T, RR><<<grid, kHwBlock, 0, st>>>(I, Vv, active, lanes, O,   \
                                                                  out_len, wb, fault);      \
        break;
    switch (gs) {
        SGAP_PRIM(1)
        SGAP_PRIM(2)
        SGAP_PRIM(4)
        SGAP_PRIM(8)
        SGAP_PRIM(16)
        SGAP_PRIM(32)
        default: return SGAP_ERR_ARG;
    }
#undef SGAP_PRIM
    return launch_status();
}

int prim_entry(bool seg, const int64_t *idx, const void *val, const uint8_t *active,
               int64_t lanes, int32_t gs, void *out, int64_t out_len, int32_t dtype,
               unsigned long long *wb, long long *fault, void *stream) {
    if (lanes < 0 || gs < 1 || gs > 32 || (gs & (gs - 1)) || lanes % gs) return SGAP_ERR_ARG;
    if (wb == nullptr || fault == nullptr) return SGAP_ERR_ARG;
    if (lanes == 0) return SGAP_OK;
    if (idx == nullptr || val == nullptr || out == nullptr) return SGAP_ERR_ARG;
    if (dtype == SGAP_F32)
        return prim_dispatch<float>(seg, idx, val, active, lanes, gs, out, out_len, wb, fault,
                                    as_stream(stream));
    if (dtype == SGAP_F64)
        return prim_dispatch<double>(seg, idx, val, active, lanes, gs, out, out_len, wb, fault,
                                     as_stream(stream));
    return SGAP_ERR_PRECISION;
}

int64_t long_row_chunk(const sgap_kernel_t *k, int32_t dtype) {
    if (k == nullptr || dtype != SGAP_F32 || k->family != SGAP_NNZ_MULTIPLE) return 0;
    // short chunks would put most rows in the table (capacity ~ nnz/g rows x n)
    return k->g >= 128 ? k->g : 0;
}

int64_t long_row_capacity(int64_t nnz, int64_t threshold, int64_t chunk) {
    if (threshold < 0) return 0;
    long long cap = nnz / (threshold + 1) + 1;
    if (chunk > 0) cap += (nnz + chunk - 1) / chunk;  // one straddling row per boundary
    return cap;
}

size_t long_rows_tmp_bytes(int64_t num_rows) {
    size_t bytes = 0;
    LongRowPred pred{nullptr, 0, 0};
    cub::DeviceSelect::If(nullptr, bytes, thrust::counting_iterator<int>(0), (int *)nullptr,
                          (int *)nullptr, (int)(num_rows > 0 ? num_rows : 1), pred);
    return bytes;
}

int prepare_long_rows(const int32_t *d_row_ptr, int64_t num_rows, int32_t n,
                           sgap_aux_t *aux, void *d_tmp, size_t tmp_bytes, void *stream) {
    if (aux == nullptr || d_row_ptr == nullptr || n < 1) return SGAP_ERR_ARG;
    if (aux->long_threshold < 0) return SGAP_OK;
    if (aux->d_long_rows == nullptr || aux->d_long_count == nullptr || aux->d_long_acc == nullptr)
        return SGAP_ERR_ARG;
    if (num_rows > INT_MAX - 1) return SGAP_ERR_SHAPE;
    cudaStream_t st = as_stream(stream);
    if (num_rows == 0) {
        return cudaMemsetAsync(aux->d_long_count, 0, sizeof(int32_t), st) == cudaSuccess
                   ? SGAP_OK : SGAP_ERR_CUDA;
    }
    size_t need = long_rows_tmp_bytes(num_rows);
    if (d_tmp == nullptr || tmp_bytes < need) return SGAP_ERR_ARG;
    LongRowPred pred{d_row_ptr, aux->long_threshold, aux->long_chunk};
    if (cub::DeviceSelect::If(d_tmp, tmp_bytes, thrust::counting_iterator<int>(0),
                              aux->d_long_rows, aux->d_long_count, (int)num_rows, pred, st) !=
        cudaSuccess)
        return SGAP_ERR_CUDA;
    if (aux->d_long_slot != nullptr) {
        long long cap = aux->long_capacity;
        unsigned blocks = (unsigned)ceil_div(cap > 0 ? cap : 1, kHwBlock);
        if (blocks > 4096) blocks = 4096;
        k_long_slots<<<blocks, kHwBlock, 0, st>>>(aux->d_long_rows, aux->d_long_count,
                                                  aux->d_long_slot);
    }
    const size_t acc_bytes = (size_t)aux->long_capacity * (size_t)n * sizeof(double);
    if (acc_bytes && cudaMemsetAsync(aux->d_long_acc, 0, acc_bytes, st) != cudaSuccess)
        return SGAP_ERR_CUDA;
    return launch_status();
}

static int run_impl(const sgap_kernel_t *k, const sgap_csr_t *a, const void *d_b, void *d_c,
                    int32_t dtype, int32_t accumulate, const sgap_aux_t *aux,
                    unsigned long long *d_writebacks, void *stream) {
    if (k == nullptr || a == nullptr) return SGAP_ERR_ARG;
    if (dtype != SGAP_F32 && dtype != SGAP_F64) return SGAP_ERR_PRECISION;
    if (k->n < 1 || k->c < 1 || k->n % k->c) return SGAP_ERR_CONFIG;
    // kernels are compiled with __launch_bounds__(256)
    if (k->hw_block != 0 && (k->hw_block < 32 || k->hw_block > 256 || k->hw_block % 32))
        return SGAP_ERR_ARG;
    if (a->num_rows < 0 || a->num_cols < 0 || a->nnz < 0) return SGAP_ERR_SHAPE;
    if (a->num_rows > INT_MAX - 1 || a->nnz > INT_MAX) return SGAP_ERR_SHAPE;
    const size_t esz = dtype == SGAP_F32 ? 4 : 8;
    const long long out_elems = a->num_rows * (long long)k->n;
    cudaStream_t st = as_stream(stream);
    if (out_elems == 0) return SGAP_OK;
    if (d_c == nullptr || a->d_row_ptr == nullptr) return SGAP_ERR_ARG;
    if (a->nnz > 0 && (d_b == nullptr || a->d_col_idx == nullptr || a->d_vals == nullptr))
        return SGAP_ERR_ARG;
    const size_t vec_bytes = esz * (size_t)(k->c == 4 && esz == 8 ? 2 : k->c);
    if ((d_b && !aligned(d_b, vec_bytes)) || !aligned(d_c, vec_bytes)) return SGAP_ERR_ARG;
    const bool eb = k->family == SGAP_NNZ_ONE || k->family == SGAP_NNZ_MULTIPLE;
    const int32_t *rowid = aux ? aux->d_rowid : nullptr;
    if (eb && k->grid_size > 0 && a->nnz > 0 && rowid == nullptr) return SGAP_ERR_ARG;
    if (k->family == SGAP_NNZ_MULTIPLE && (k->g < 1 || k->chunk % k->g)) return SGAP_ERR_CONFIG;
    LongRows lr{nullptr, nullptr, nullptr, -1, nullptr, 0, nullptr, 0, nullptr, {nullptr, nullptr},
                {nullptr, nullptr}, nullptr};
    const bool has_exact = aux != nullptr && aux->has_exact_rows != 0;
    // exact-flagged chunks are skipped by the main walk: their pass needs the list
    if (has_exact && k->family == SGAP_NNZ_MULTIPLE && dtype == SGAP_F32 &&
        aux->long_threshold >= 0 && (aux->d_exact_rows == nullptr || aux->exact_count <= 0))
        return SGAP_ERR_ARG;
    if (eb && aux && aux->long_threshold >= 0 && dtype == SGAP_F32) {
        if (aux->d_long_rows == nullptr || aux->d_long_count == nullptr || aux->d_long_acc == nullptr)
            return SGAP_ERR_ARG;
        lr = LongRows{aux->d_long_rows, aux->d_long_count, aux->d_long_acc, aux->long_threshold,
                      aux->d_long_slot, aux->long_chunk, aux->d_exact_rows, aux->exact_count,
                      nullptr, {nullptr, nullptr}, {nullptr, nullptr}, nullptr};
    }
    if (k->family == SGAP_NNZ_MULTIPLE && aux != nullptr) {
        lr.chunk_rows = aux->d_chunk_rows;
        lr.col_hinted = aux->d_col_hinted;
        lr.panel_b = aux->d_panel_b;
        lr.panel_lanes = aux->d_panel_b ? aux->panel_lanes : 0;
    }
    if (k->family == SGAP_ROW_MULTIPLE && aux != nullptr) {
        for (int w = 0; w < 2; ++w) {
            lr.union_e[w] = reinterpret_cast<const unsigned *>(aux->d_union[w]);
            lr.union_off[w] = aux->d_union_off[w];
        }
    }
    if (k->family == SGAP_NNZ_ONE && !accumulate) {
        // atomic-writeback families accumulate into C: zero-fill (counts as
        // part of the SpMM); nnz-multiple zero-fills only the
        // rows it cannot store outright (k_zero_shared_rows).
        if (cudaMemsetAsync(d_c, 0, (size_t)out_elems * esz, st) != cudaSuccess)
            return SGAP_ERR_CUDA;
    }
    if (eb && k->grid_size == 0) {
        if (k->family == SGAP_NNZ_MULTIPLE && !accumulate)  // every row is empty
            return cudaMemsetAsync(d_c, 0, (size_t)out_elems * esz, st) == cudaSuccess ? SGAP_OK
                                                                                    : SGAP_ERR_CUDA;
        return SGAP_OK;
    }
    if (dtype == SGAP_F32)
        return run_typed<float>(*k, *a, d_b, d_c, accumulate, rowid, lr, has_exact, d_writebacks,
                                st);
    return run_typed<double>(*k, *a, d_b, d_c, accumulate, rowid, lr, has_exact, d_writebacks, st);
}


// ------------------------------------------------------------------ planner

// Rows longer than `cut` (the error-free pass's list), in ascending order.
struct LongerThan {
    const int *rp;
    long long cut;
    __host__ __device__ __forceinline__ bool operator()(const int &r) const {
        return (long long)rp[r + 1] - rp[r] > cut;
    }
};

// Workspace layout of a plan (every region 256-byte aligned).
struct PlanLayout {
    size_t starts = 0, rowid = 0, slot = 0, rows = 0, count = 0, acc = 0, exact = 0, stats = 0,
           tmp = 0, chunk_rows = 0, union_off[2] = {0, 0}, union_e[2] = {0, 0}, union_tmp = 0,
           hint_counts = 0, hint_sorted = 0, hint_cols = 0, hint_tmp = 0, panel_b = 0, total = 0;
    int panel_lanes = 0;
    size_t hint_tmp_bytes = 0;
    size_t union_tmp_bytes = 0;
    long long thr = -1, chunk = 0, cap = 0, exact_cap = 0, exact_cut = 0;
    size_t tmp_bytes = 0;
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int plan_layout(const sgap_kernel_t &k, const sgap_csr_t &a, int32_t dtype, uint32_t flags,
                PlanLayout &L) {
    const bool eb = k.family == SGAP_NNZ_ONE || k.family == SGAP_NNZ_MULTIPLE;
    const long long M = a.num_rows, nnz = a.nnz;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t at = off;
        off = align256(off + (bytes ? bytes : 1));
        return at;
    };
    L.stats = take(4 * sizeof(unsigned long long));
    if (k.family == SGAP_ROW_MULTIPLE && k.c > 0 && k.n / k.c == 32 && k.n % k.c == 0 && nnz > 0) {
        for (int w = 0; w < 2; ++w) {  // 4-row and 8-row union streams (<= nnz entries each)
            const int R = w ? 8 : 4;
            if (a.num_cols >= (1LL << (32 - R))) continue;
            const long long nb = ceil_div(M, R);
            L.union_off[w] = take((size_t)(nb + 1) * sizeof(int));
            L.union_e[w] = take((size_t)nnz * sizeof(unsigned));
            size_t sb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, sb, (int *)nullptr, (int *)nullptr,
                                          (int)(nb + 1));
            if (sb > L.union_tmp_bytes) L.union_tmp_bytes = sb;
        }
        if (L.union_tmp_bytes) L.union_tmp = take(L.union_tmp_bytes);
    }
    if (eb) {
        L.starts = take((size_t)(k.grid_size + 1) * sizeof(int));
        L.rowid = take((size_t)(nnz > 4 ? nnz : 4) * sizeof(int));
        if (k.family == SGAP_NNZ_MULTIPLE && k.g % 4 == 0 && k.g > 0)
            L.chunk_rows = take((size_t)(k.grid_size * (k.chunk / k.g) + 1) * sizeof(int));
        if (L.chunk_rows && (flags & SGAP_PLAN_L2_HINTS) && nnz > 0 && a.num_cols > 0) {
            const long long K = a.num_cols;
            L.hint_counts = take((size_t)K * sizeof(unsigned));
            L.hint_sorted = take((size_t)K * sizeof(unsigned));
            L.hint_cols = take((size_t)nnz * sizeof(int));
            size_t sb = 0;
            cub::DeviceRadixSort::SortKeysDescending(nullptr, sb, (unsigned *)nullptr,
                                                     (unsigned *)nullptr, (int)K);
            L.hint_tmp_bytes = sb;
            L.hint_tmp = take(sb);
        }
        if (L.chunk_rows && (flags & SGAP_PLAN_PANELS) && nnz > 0) {
            const size_t esz = dtype == SGAP_F32 ? 4 : 8;
            L.panel_lanes = panel_lanes(k, a, k.c, esz);
            if (L.panel_lanes > 0) {
                const long long pw = (long long)L.panel_lanes * k.c;
                const long long passes = ceil_div(k.n, pw);
                L.panel_b = take((size_t)(passes * a.num_cols * pw) * esz);
            }
        }
        L.thr = sgap_long_row_threshold(&k, dtype);
        L.chunk = (L.thr >= 0 && (flags & SGAP_PLAN_SPLIT_ROWS)) ? long_row_chunk(&k, dtype) : 0;
        if (L.thr >= 0) {
            L.cap = long_row_capacity(nnz, L.thr, L.chunk);
            if (L.cap > M) L.cap = M > 0 ? M : 1;
            L.exact_cut = L.thr > kExactRow ? L.thr : kExactRow;
            L.exact_cap = k.family == SGAP_NNZ_MULTIPLE ? nnz / (L.exact_cut + 1) + 1 : 0;
            if (L.exact_cap > M) L.exact_cap = M > 0 ? M : 1;
            L.slot = take((size_t)(M > 0 ? M : 1) * sizeof(int));
            L.rows = take((size_t)L.cap * sizeof(int));
            L.count = take(sizeof(int));
            L.acc = take((size_t)L.cap * (size_t)k.n * sizeof(double));
            L.exact = take((size_t)L.exact_cap * sizeof(int));
            size_t ex_bytes = 0;
            LongerThan pred{nullptr, 0};
            cub::DeviceSelect::If(nullptr, ex_bytes, thrust::counting_iterator<int>(0),
                                  (int *)nullptr, (int *)nullptr, (int)(M > 0 ? M : 1), pred);
            L.tmp_bytes = long_rows_tmp_bytes(M);
            if (ex_bytes > L.tmp_bytes) L.tmp_bytes = ex_bytes;
            L.tmp = take(L.tmp_bytes);
        }
    }
    L.total = off;
    return SGAP_OK;
}

int check_kernel_csr(const sgap_kernel_t *k, const sgap_csr_t *a, int32_t dtype) {
    if (k == nullptr || a == nullptr) return SGAP_ERR_ARG;
    if (dtype != SGAP_F32 && dtype != SGAP_F64) return SGAP_ERR_PRECISION;
    if (k->n < 1 || k->c < 1 || k->n % k->c) return SGAP_ERR_CONFIG;
    if (k->family < SGAP_NNZ_MULTIPLE || k->family > SGAP_NNZ_ONE) return SGAP_ERR_ARG;
    if (a->num_rows < 0 || a->num_cols < 0 || a->nnz < 0) return SGAP_ERR_SHAPE;
    if (a->num_rows > kRowMask - 1 || a->nnz > INT_MAX) return SGAP_ERR_SHAPE;
    if (k->grid_size < 0 || k->chunk < 0) return SGAP_ERR_CONFIG;
    return SGAP_OK;
}

constexpr int32_t kPlanMagicAbi = SGAP_ABI_VERSION;


// ------------------------------------------------------ dgSPARSE RB+PR grid

template <typename T, int V, int G>
int launch_rbpr_grid(const sgap_csr_t &a, const T *B, T *C, int n, int block, int tile,
                     double worker_scale, int acc, unsigned long long *wb, cudaStream_t st) {
    // blockDim.x = min(N, tile)/coarsen * groupSz (>= one vector), blockDim.y =
    // max(blockSz, 2 blockDim.x)/blockDim.x rows, capped at 1024 threads
    const int cols = n < tile ? n : tile;
    int vecs = cols / V;
    if (vecs < 1) vecs = 1;
    const int tile_cols = vecs * V;
    const int bx = vecs * G;
    if (bx > 1024) return SGAP_ERR_CONFIG;
    int threads = block > 2 * bx ? block : 2 * bx;
    if (threads > 1024) threads = 1024;
    int by = threads / bx;
    if (by < 1) by = 1;
    // workerDimR = worker_scale x M row workers -> blocks along the rows
    long long workers = (long long)(worker_scale * (double)a.num_rows + 0.5);
    if (workers < 1) workers = 1;
    long long gx = ceil_div(workers, by);
    if (gx > (1LL << 31) - 1) gx = (1LL << 31) - 1;
    const long long gy = ceil_div(n, tile_cols);
    if (gy > 65535) return SGAP_ERR_CONFIG;
    k_rbpr_grid<T, V, G><<<dim3((unsigned)gx, (unsigned)gy), dim3(bx, by), 0, st>>>(
        a.d_row_ptr, a.d_col_idx, static_cast<const T *>(a.d_vals), B, C, (int)a.num_rows, n,
        tile_cols, acc, wb);
    return launch_status();
}

template <typename T, int V>
int run_rbpr_grid_v(const sgap_csr_t &a, const T *B, T *C, int n, int group, int block, int tile,
                    double ws, int acc, unsigned long long *wb, cudaStream_t st) {
    switch (group) {
        case 2: return launch_rbpr_grid<T, V, 2>(a, B, C, n, block, tile, ws, acc, wb, st);
        case 4: return launch_rbpr_grid<T, V, 4>(a, B, C, n, block, tile, ws, acc, wb, st);
        case 8: return launch_rbpr_grid<T, V, 8>(a, B, C, n, block, tile, ws, acc, wb, st);
        case 16: return launch_rbpr_grid<T, V, 16>(a, B, C, n, block, tile, ws, acc, wb, st);
        case 32: return launch_rbpr_grid<T, V, 32>(a, B, C, n, block, tile, ws, acc, wb, st);
        default: return SGAP_ERR_NO_TEMPLATE;
    }
}

template <typename T>
int run_rbpr_grid(const sgap_csr_t &a, const void *b, void *c, int n, int coarsen, int group,
                  int block, int tile, double ws, int acc, unsigned long long *wb, cudaStream_t st) {
    const T *B = static_cast<const T *>(b);
    T *C = static_cast<T *>(c);
    switch (coarsen) {
        case 1: return run_rbpr_grid_v<T, 1>(a, B, C, n, group, block, tile, ws, acc, wb, st);
        case 2: return run_rbpr_grid_v<T, 2>(a, B, C, n, group, block, tile, ws, acc, wb, st);
        case 4: return run_rbpr_grid_v<T, 4>(a, B, C, n, group, block, tile, ws, acc, wb, st);
        default: return SGAP_ERR_NO_TEMPLATE;
    }
}

}  // namespace

extern "C" {

int sgap_abi_version(void) { return SGAP_ABI_VERSION; }

const char *sgap_status_string(int status) {
    switch (status) {
        case SGAP_OK: return "ok";
        case SGAP_ERR_ILLEGAL_POINT: return "illegal point";
        case SGAP_ERR_NO_TEMPLATE: return "no template covers the point";
        case SGAP_ERR_SHAPE: return "shape mismatch";
        case SGAP_ERR_PRECISION: return "unknown precision";
        case SGAP_ERR_CUDA: return "CUDA error";
        case SGAP_ERR_ARG: return "bad argument";
        case SGAP_ERR_FAULT: return "group invariant violated";
        case SGAP_ERR_CONFIG: return "bad kernel config";
        default: return "unknown status";
    }
}

// space.legality_rule (space.py:177-204).
int sgap_legality_rule(const sgap_point_t *pt) {
    if (pt == nullptr) return -1;
    const bool data_recip = pt->data_amount == SGAP_AMT_RECIPROCAL;
    const bool col_recip = pt->col_amount == SGAP_AMT_RECIPROCAL;
    if (pt->data_kind == SGAP_KIND_NNZ) return (data_recip || col_recip) ? 1 : 0;
    if (data_recip) {
        if (pt->r < pt->data_param) return 2;  // r/g < 1
        if (col_recip) return 3;
    }
    return 0;
}

// runner.build_kernel = templates.template_family + the per-family gates
// (templates.py:82-202) + lowering geometry (lowering.py:218-243, 649-696).
int sgap_build_kernel(const sgap_point_t *pt, int32_t n, int32_t p, int64_t num_rows,
                      int64_t nnz, sgap_kernel_t *out, int32_t *rule_out) {
    if (pt == nullptr || out == nullptr) return SGAP_ERR_ARG;
    if (rule_out) *rule_out = 0;
    if (n < 1 || p < 32 || p % 32 != 0) return SGAP_ERR_CONFIG;
    const int rule = sgap_legality_rule(pt);
    if (rule != 0) {
        if (rule_out) *rule_out = rule;
        return SGAP_ERR_ILLEGAL_POINT;
    }
    if (pt->col_amount == SGAP_AMT_RECIPROCAL) return SGAP_ERR_NO_TEMPLATE;
    std::memset(out, 0, sizeof(*out));
    const long long N = n, P = p;
    const long long c = amount_units(pt->col_amount, pt->col_param);
    const long long g = amount_units(pt->data_amount, pt->data_param);
    const long long r = pt->r;
    out->n = n;
    out->p = p;
    out->c = (int)c;
    out->g = (int)g;
    out->r = (int)r;
    if (pt->data_kind == SGAP_KIND_NNZ) {
        if (pt->data_amount == SGAP_AMT_ONE) {
            if (N % c || (P * c) % N) return SGAP_ERR_NO_TEMPLATE;
            const long long npb = P * c / N;
            if (r > 1 && (32 % r || npb % r || r > npb)) return SGAP_ERR_NO_TEMPLATE;
            out->family = SGAP_NNZ_ONE;
            out->chunk = npb;
            out->grid_size = nnz ? ceil_div(nnz, npb) : 0;
            out->block_size = P;
            out->has_block_starts = 1;
        } else if (pt->data_amount == SGAP_AMT_MULTIPLE && r == 1) {
            if (N % c || (P * c) % N || (P * g * c) % N) return SGAP_ERR_NO_TEMPLATE;
            const long long chunk = P * g * c / N;
            if (((P * c / N) * c) % 32) return SGAP_ERR_NO_TEMPLATE;
            out->family = SGAP_NNZ_MULTIPLE;
            out->chunk = chunk;
            out->grid_size = nnz ? ceil_div(nnz, chunk) : 0;
            out->block_size = (chunk / g) * c;
            out->has_block_starts = 1;
        } else {
            return SGAP_ERR_NO_TEMPLATE;
        }
    } else {
        if (pt->data_amount == SGAP_AMT_RECIPROCAL) {
            if (r != g) return SGAP_ERR_NO_TEMPLATE;
            if (N % c || (c * P) % g || P % g || 32 % g) return SGAP_ERR_NO_TEMPLATE;
            const long long cells = c * P / g;
            out->family = SGAP_ROW_RECIPROCAL;
            out->chunk = cells;
            out->grid_size = ceil_div(num_rows * N, cells);
            out->block_size = P;
        } else {
            if (r != 1) return SGAP_ERR_NO_TEMPLATE;
            if (N % c || (P * g * c) % N || (P * c) % N) return SGAP_ERR_NO_TEMPLATE;
            const long long rows = P * g * c / N;
            out->family = SGAP_ROW_MULTIPLE;
            out->chunk = rows;
            out->grid_size = ceil_div(num_rows, rows);
            out->block_size = P;
        }
    }
    return SGAP_OK;
}

int sgap_block_starts(const int32_t *d_row_ptr, int64_t num_rows, int64_t chunk,
                      int64_t num_blocks, int32_t *d_starts, void *stream) {
    if (chunk < 1 || num_blocks < 0 || num_rows < 0) return SGAP_ERR_ARG;
    if (d_row_ptr == nullptr || d_starts == nullptr) return SGAP_ERR_ARG;
    const long long n = num_blocks + 1;
    k_block_starts<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(
        d_row_ptr, num_rows, chunk, num_blocks, d_starts);
    return launch_status();
}

int64_t sgap_long_row_threshold(const sgap_kernel_t *k, int32_t dtype) {
    if (k == nullptr || dtype != SGAP_F32) return -1;
    // A row split over m chunk flushes accumulates m float32 roundings of
    // partial sums that can be far larger than the row's final value (a
    // power-law row whose column sum cancels).  nnz-multiple: rows longer than
    // clamp(16g, 2048, 32g) (min 128) go to the float64 table -- at g = 512
    // the bound 32g let 32 flushes of 512-term partials reach 1.0e-5 on
    // config 2 (16g: 4.5e-6), at g = 2 the bound 1024 let 512 flushes reach
    // 1.1e-5; 4g cost config 3 6% in float64 atomics for no accuracy gain.
    // nnz-one flushes r-term segment sums: rows past 32r (min 128).
    if (k->family == SGAP_NNZ_MULTIPLE) {
        // <= 32 flushes of short partials (small g), <= 16 of long ones, and
        // never above the error-free length: a row past kExactRow must be in
        // the table to take the exact path (config 3 measured 9.1e-6 with
        // its 4k-8k rows summed in float32 at g = 512)
        long long t = 16LL * k->g;
        if (t < 2048) t = 2048;
        if (t > 32LL * k->g) t = 32LL * k->g;
        if (t > kExactRow) t = kExactRow;
        return t < 128 ? 128 : t;
    }
    if (k->family != SGAP_NNZ_ONE) return -1;  // row families own their rows
    const long long t = 32LL * k->r;
    return t < 128 ? 128 : t;
}

int64_t sgap_exact_row_length(void) { return kExactRow; }

int sgap_row_ids(const int32_t *d_row_ptr, int64_t num_rows, int64_t nnz,
                 int64_t long_threshold, int64_t long_chunk, int32_t *d_rowid, void *stream) {
    if (long_chunk < 0) return SGAP_ERR_ARG;
    if (num_rows < 0 || nnz < 0 || num_rows > INT_MAX - 1 || nnz > INT_MAX) return SGAP_ERR_SHAPE;
    if (nnz == 0) return SGAP_OK;
    if (d_row_ptr == nullptr || d_rowid == nullptr || num_rows == 0) return SGAP_ERR_ARG;
    const long long items = ceil_div(nnz, 1024);
    k_row_ids<<<grid_for(items, kHwBlock), kHwBlock, 0, as_stream(stream)>>>(
        d_row_ptr, (int)num_rows, nnz, long_threshold, long_chunk, d_rowid);
    return launch_status();
}

int sgap_plan_workspace_bytes(const sgap_kernel_t *k, const sgap_csr_t *a, int32_t dtype,
                              uint32_t flags, size_t *bytes) {
    if (bytes == nullptr) return SGAP_ERR_ARG;
    const int st = check_kernel_csr(k, a, dtype);
    if (st != SGAP_OK) return st;
    PlanLayout L;
    plan_layout(*k, *a, dtype, flags, L);
    *bytes = L.total;
    return SGAP_OK;
}

int sgap_validate_csr(const sgap_csr_t *a, void *d_scratch, int64_t *fault_pos, void *stream) {
    if (a == nullptr || d_scratch == nullptr) return SGAP_ERR_ARG;
    if (a->num_rows < 0 || a->num_cols < 0 || a->nnz < 0) return SGAP_ERR_SHAPE;
    if (a->num_rows > INT_MAX - 1 || a->nnz > INT_MAX) return SGAP_ERR_SHAPE;
    if (a->d_row_ptr == nullptr || (a->nnz > 0 && a->d_col_idx == nullptr)) return SGAP_ERR_ARG;
    if (fault_pos) *fault_pos = 0;
    cudaStream_t st = as_stream(stream);
    auto *f = static_cast<unsigned long long *>(d_scratch);
    unsigned long long h = 0;
    auto read = [&]() -> int {
        if (cudaGetLastError() != cudaSuccess) return SGAP_ERR_CUDA;
        if (cudaMemcpyAsync(&h, f, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return SGAP_ERR_CUDA;
        return SGAP_OK;
    };
    if (cudaMemsetAsync(f, 0xff, sizeof(*f), st) != cudaSuccess) return SGAP_ERR_CUDA;
    k_validate_row_ptr<<<(unsigned)ceil_div(a->num_rows + 1 < 1048576 ? a->num_rows + 1 : 1048576, 256),
                         256, 0, st>>>(a->d_row_ptr, a->num_rows, a->nnz, f);
    int s0 = read();
    if (s0 != SGAP_OK) return s0;
    if (h != ~0ULL) {
        if (fault_pos) *fault_pos = -(int64_t)h - 1;
        return SGAP_ERR_FAULT;
    }
    if (a->nnz == 0) return SGAP_OK;
    if (cudaMemsetAsync(f, 0xff, sizeof(*f), st) != cudaSuccess) return SGAP_ERR_CUDA;
    k_validate_cols<<<(unsigned)ceil_div(a->nnz < 4194304 ? a->nnz : 4194304, 256), 256, 0, st>>>(
        a->d_row_ptr, a->d_col_idx, (int)a->num_rows, a->num_cols, a->nnz, f);
    s0 = read();
    if (s0 != SGAP_OK) return s0;
    if (h != ~0ULL) {
        if (fault_pos) *fault_pos = (int64_t)h;
        return SGAP_ERR_FAULT;
    }
    return SGAP_OK;
}

int sgap_plan(const sgap_kernel_t *k, const sgap_csr_t *a, int32_t dtype, uint32_t flags,
              void *d_ws, size_t ws_bytes, sgap_plan_t *plan, void *stream) {
    if (plan == nullptr) return SGAP_ERR_ARG;
    int st0 = check_kernel_csr(k, a, dtype);
    if (st0 != SGAP_OK) return st0;
    if (a->num_rows > 0 && a->d_row_ptr == nullptr) return SGAP_ERR_ARG;
    if (a->nnz > 0 && a->d_col_idx == nullptr) return SGAP_ERR_ARG;
    PlanLayout L;
    plan_layout(*k, *a, dtype, flags, L);
    if (d_ws == nullptr || ws_bytes < L.total || !aligned(d_ws, 256)) return SGAP_ERR_ARG;
    cudaStream_t st = as_stream(stream);
    char *ws = static_cast<char *>(d_ws);
    if (flags & SGAP_PLAN_VALIDATE) {
        int64_t pos = 0;
        const int v = sgap_validate_csr(a, ws + L.stats, &pos, stream);
        if (v != SGAP_OK) return v;
    }
    std::memset(plan, 0, sizeof(*plan));
    plan->abi = kPlanMagicAbi;
    plan->dtype = dtype;
    plan->kernel = *k;
    plan->num_rows = a->num_rows;
    plan->num_cols = a->num_cols;
    plan->nnz = a->nnz;
    plan->d_row_ptr = a->d_row_ptr;
    plan->d_col_idx = a->d_col_idx;
    plan->d_workspace = d_ws;
    plan->workspace_bytes = ws_bytes;
    sgap_aux_t &aux = plan->aux;
    aux.long_threshold = -1;
    const bool eb = k->family == SGAP_NNZ_ONE || k->family == SGAP_NNZ_MULTIPLE;
    const long long M = a->num_rows, nnz = a->nnz;
    // row statistics (one read-back): longest row, table rows, error-free rows
    auto *stats = reinterpret_cast<unsigned long long *>(ws + L.stats);
    unsigned long long h[4] = {0, 0, 0, 0};
    if (cudaMemsetAsync(stats, 0, 4 * sizeof(unsigned long long), st) != cudaSuccess)
        return SGAP_ERR_CUDA;
    if (M > 0) {
        k_row_stats<<<grid_for(ceil_div(M, 32), kHwBlock), kHwBlock, 0, st>>>(
            a->d_row_ptr, (int)M, L.thr, L.chunk, L.thr >= 0 ? L.exact_cut : LLONG_MAX, stats);
        if (cudaGetLastError() != cudaSuccess) return SGAP_ERR_CUDA;
    }
    if (eb && k->grid_size > 0) {
        const int s1 = sgap_block_starts(a->d_row_ptr, M, k->chunk, k->grid_size,
                                         reinterpret_cast<int32_t *>(ws + L.starts), stream);
        if (s1 != SGAP_OK) return s1;
        aux.d_block_starts = reinterpret_cast<const int32_t *>(ws + L.starts);
    }
    if (L.chunk_rows && k->grid_size > 0) {  // the row owning each g-chunk's first position
        const long long chunks = k->grid_size * (k->chunk / k->g);
        const int s4 = sgap_block_starts(a->d_row_ptr, M, k->g, chunks,
                                         reinterpret_cast<int32_t *>(ws + L.chunk_rows), stream);
        if (s4 != SGAP_OK) return s4;
        aux.d_chunk_rows = reinterpret_cast<const int32_t *>(ws + L.chunk_rows);
    }
    if (L.hint_cols) {
        // cold-column hints: per-column gather counts, the count of the
        // H-th most-gathered column (H = half the L2 in B rows) as the hot
        // threshold, then the flagged col_idx copy
        int dev = 0, l2 = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        const size_t esz = dtype == SGAP_F32 ? 4 : 8;
        long long H = (long long)(l2 / 2) / ((long long)k->n * (long long)esz);
        if (H < 1) H = 1;
        if (H > a->num_cols) H = a->num_cols;
        unsigned *counts = reinterpret_cast<unsigned *>(ws + L.hint_counts);
        unsigned *sorted = reinterpret_cast<unsigned *>(ws + L.hint_sorted);
        int *hinted = reinterpret_cast<int *>(ws + L.hint_cols);
        if (cudaMemsetAsync(counts, 0, (size_t)a->num_cols * sizeof(unsigned), st) != cudaSuccess)
            return SGAP_ERR_CUDA;
        const unsigned g1 = (unsigned)ceil_div(nnz < (1LL << 24) ? nnz : (1LL << 24), kHwBlock);
        k_col_counts<<<g1, kHwBlock, 0, st>>>(a->d_col_idx, nnz, a->num_cols, counts);
        size_t tb = L.hint_tmp_bytes;
        if (cub::DeviceRadixSort::SortKeysDescending(ws + L.hint_tmp, tb, counts, sorted,
                                                     (int)a->num_cols, 0, 32, st) != cudaSuccess)
            return SGAP_ERR_CUDA;
        k_col_hints<<<g1, kHwBlock, 0, st>>>(a->d_col_idx, nnz, a->num_cols, counts,
                                             sorted + (H - 1), hinted);
        if (cudaGetLastError() != cudaSuccess) return SGAP_ERR_CUDA;
        aux.d_col_hinted = hinted;
    }
    if (L.panel_b) {
        aux.d_panel_b = ws + L.panel_b;
        aux.panel_lanes = L.panel_lanes;
    }
    if (cudaMemcpyAsync(h, stats, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return SGAP_ERR_CUDA;
    plan->longest_row = (int64_t)h[0];
    if (k->family == SGAP_ROW_MULTIPLE && h[0] <= 64) {
        // union column streams of 4- and 8-row blocks (row-blocked walk):
        // count per block, exclusive scan into offsets, fill
        for (int w = 0; w < 2; ++w) {
            if (!L.union_e[w]) continue;
            const long long nb = ceil_div(M, w ? 8 : 4);
            int *off = reinterpret_cast<int *>(ws + L.union_off[w]);
            unsigned *ent = reinterpret_cast<unsigned *>(ws + L.union_e[w]);
            const unsigned grid = grid_for(ceil_div(nb, 32), kHwBlock);
            if (w == 0)
                k_union_rows<4><<<grid, kHwBlock, 0, st>>>(a->d_row_ptr, a->d_col_idx, (int)M, nb,
                                                           nullptr, off, nullptr);
            else
                k_union_rows<8><<<grid, kHwBlock, 0, st>>>(a->d_row_ptr, a->d_col_idx, (int)M, nb,
                                                           nullptr, off, nullptr);
            if (cudaGetLastError() != cudaSuccess) return SGAP_ERR_CUDA;
            if (cudaMemsetAsync(off + nb, 0, sizeof(int), st) != cudaSuccess) return SGAP_ERR_CUDA;
            size_t tb = L.union_tmp_bytes;
            if (cub::DeviceScan::ExclusiveSum(ws + L.union_tmp, tb, off, off, (int)(nb + 1), st) !=
                cudaSuccess)
                return SGAP_ERR_CUDA;
            if (w == 0)
                k_union_rows<4><<<grid, kHwBlock, 0, st>>>(a->d_row_ptr, a->d_col_idx, (int)M, nb,
                                                           off, nullptr, ent);
            else
                k_union_rows<8><<<grid, kHwBlock, 0, st>>>(a->d_row_ptr, a->d_col_idx, (int)M, nb,
                                                           off, nullptr, ent);
            if (cudaGetLastError() != cudaSuccess) return SGAP_ERR_CUDA;
            aux.d_union_off[w] = off;
            aux.d_union[w] = ent;
        }
    }
    if (!eb) return SGAP_OK;
    long long thr = L.thr;
    if (thr >= 0 && (long long)h[0] <= thr && L.chunk == 0) thr = -1;  // no table needed
    int32_t *rowid = reinterpret_cast<int32_t *>(ws + L.rowid);
    const int s2 = sgap_row_ids(a->d_row_ptr, M, nnz, thr, thr >= 0 ? L.chunk : 0, rowid, stream);
    if (s2 != SGAP_OK) return s2;
    aux.d_rowid = rowid;
    if (thr < 0) return SGAP_OK;
    aux.long_threshold = thr;
    aux.long_chunk = L.chunk;
    aux.long_capacity = L.cap;
    aux.d_long_slot = reinterpret_cast<int32_t *>(ws + L.slot);
    aux.d_long_rows = reinterpret_cast<int32_t *>(ws + L.rows);
    aux.d_long_count = reinterpret_cast<int32_t *>(ws + L.count);
    aux.d_long_acc = reinterpret_cast<double *>(ws + L.acc);
    plan->table_rows = (int64_t)h[1];
    // zero only the rows the table will hold (prepare_long_rows clears cap x n)
    const long long saved_cap = aux.long_capacity;
    aux.long_capacity = (long long)h[1] < saved_cap ? (long long)h[1] : saved_cap;
    const int s3 = prepare_long_rows(a->d_row_ptr, M, k->n, &aux, ws + L.tmp, L.tmp_bytes, stream);
    aux.long_capacity = saved_cap;
    if (s3 != SGAP_OK) return s3;
    if (k->family == SGAP_NNZ_MULTIPLE && h[2] > 0) {
        int32_t *ex = reinterpret_cast<int32_t *>(ws + L.exact);
        LongerThan pred{a->d_row_ptr, L.exact_cut};
        size_t tb = L.tmp_bytes;
        // the count lands in the stats slot 3 (unused by the runs)
        if (cub::DeviceSelect::If(ws + L.tmp, tb, thrust::counting_iterator<int>(0), ex,
                                  reinterpret_cast<int *>(stats + 3), (int)M, pred, st) !=
            cudaSuccess)
            return SGAP_ERR_CUDA;
        aux.d_exact_rows = ex;
        aux.exact_count = (int32_t)h[2];
        aux.has_exact_rows = 1;
    }
    return launch_status();
}

int sgap_run(const sgap_plan_t *plan, const sgap_csr_t *a, const void *d_b, void *d_c,
             int32_t accumulate, unsigned long long *d_writebacks, void *stream) {
    if (plan == nullptr || a == nullptr) return SGAP_ERR_ARG;
    if (plan->abi != kPlanMagicAbi) return SGAP_ERR_ARG;  // not a plan from sgap_plan
    // the plan is bound to one sparsity structure: values may change, the
    // structure may not
    if (a->num_rows != plan->num_rows || a->num_cols != plan->num_cols || a->nnz != plan->nnz ||
        a->d_row_ptr != plan->d_row_ptr || a->d_col_idx != plan->d_col_idx)
        return SGAP_ERR_SHAPE;
    return run_impl(&plan->kernel, a, d_b, d_c, plan->dtype, accumulate, &plan->aux,
                    d_writebacks, stream);
}

int sgap_run_rbpr_grid(const sgap_plan_t *plan, const sgap_csr_t *a, const void *d_b, void *d_c,
                       int32_t block, int32_t tile, double worker_scale, int32_t accumulate,
                       unsigned long long *d_writebacks, void *stream) {
    if (plan == nullptr || a == nullptr) return SGAP_ERR_ARG;
    if (plan->abi != kPlanMagicAbi) return SGAP_ERR_ARG;
    const sgap_kernel_t &k = plan->kernel;
    if (k.family != SGAP_ROW_RECIPROCAL) return SGAP_ERR_ARG;
    if (a->num_rows != plan->num_rows || a->num_cols != plan->num_cols || a->nnz != plan->nnz ||
        a->d_row_ptr != plan->d_row_ptr || a->d_col_idx != plan->d_col_idx)
        return SGAP_ERR_SHAPE;
    if (block < 32 || block > 1024 || block % 32 || tile < k.g || (tile & (tile - 1)) ||
        !(worker_scale > 0.0))
        return SGAP_ERR_CONFIG;
    const long long out_elems = a->num_rows * (long long)k.n;
    if (out_elems == 0) return SGAP_OK;
    const size_t esz = plan->dtype == SGAP_F32 ? 4 : 8;
    const size_t vec_bytes = esz * (size_t)(k.c == 4 && esz == 8 ? 2 : k.c);
    if (d_c == nullptr || (a->nnz > 0 && (d_b == nullptr || a->d_vals == nullptr)))
        return SGAP_ERR_ARG;
    if ((d_b && !aligned(d_b, vec_bytes)) || !aligned(d_c, vec_bytes)) return SGAP_ERR_ARG;
    cudaStream_t st = as_stream(stream);
    if (plan->dtype == SGAP_F32)
        return run_rbpr_grid<float>(*a, d_b, d_c, k.n, k.c, k.g, block, tile, worker_scale,
                                    accumulate, d_writebacks, st);
    return run_rbpr_grid<double>(*a, d_b, d_c, k.n, k.c, k.g, block, tile, worker_scale,
                                 accumulate, d_writebacks, st);
}

int sgap_reference_spmm_f64(const sgap_csr_t *a, const void *d_b, int32_t n, int32_t dtype,
                            double *d_c, void *stream) {
    if (a == nullptr || n < 1) return SGAP_ERR_ARG;
    if (dtype != SGAP_F32 && dtype != SGAP_F64) return SGAP_ERR_PRECISION;
    if (a->num_rows > INT_MAX - 1 || a->nnz > INT_MAX) return SGAP_ERR_SHAPE;
    const long long cells = a->num_rows * (long long)n;
    if (cells == 0) return SGAP_OK;
    if (d_c == nullptr || a->d_row_ptr == nullptr) return SGAP_ERR_ARG;
    if (a->nnz > 0 && (d_b == nullptr || a->d_col_idx == nullptr || a->d_vals == nullptr))
        return SGAP_ERR_ARG;
    long long blocks = ceil_div(cells, kHwBlock);
    if (blocks > (1LL << 30)) blocks = 1LL << 30;
    cudaStream_t st = as_stream(stream);
    if (dtype == SGAP_F32)
        k_reference_f64<float><<<(unsigned)blocks, kHwBlock, 0, st>>>(
            a->d_row_ptr, a->d_col_idx, static_cast<const float *>(a->d_vals),
            static_cast<const float *>(d_b), d_c, (int)a->num_rows, n);
    else
        k_reference_f64<double><<<(unsigned)blocks, kHwBlock, 0, st>>>(
            a->d_row_ptr, a->d_col_idx, static_cast<const double *>(a->d_vals),
            static_cast<const double *>(d_b), d_c, (int)a->num_rows, n);
    return launch_status();
}

// ------------------------------------------------------------ Matrix Market ingest

static unsigned ingest_grid(long long items) {
    long long b = ceil_div(items > 0 ? items : 1, 256);
    return (unsigned)(b < 65536 ? b : 65536);
}

int sgap_mm_line_flags(const uint8_t *d_text, int64_t len, uint8_t *d_flag, int32_t *d_special,
                       void *stream) {
    if (len < 0) return SGAP_ERR_ARG;
    if (len == 0) return SGAP_OK;
    if (d_text == nullptr || d_flag == nullptr || d_special == nullptr) return SGAP_ERR_ARG;
    k_mm_line_flags<<<ingest_grid(len), 256, 0, as_stream(stream)>>>(d_text, len, d_flag,
                                                                      d_special);
    return launch_status();
}

int sgap_mm_parse(const uint8_t *d_text, int64_t len, const int64_t *d_starts, int64_t nlines,
                  int64_t rows, int64_t cols, uint8_t *d_status, int64_t *d_r, int64_t *d_c,
                  double *d_v, int64_t *d_tok_off, int32_t *d_tok_len, void *stream) {
    if (len < 0 || nlines < 0 || rows < 0 || cols < 0) return SGAP_ERR_ARG;
    if (rows > INT_MAX || cols > INT_MAX) return SGAP_ERR_SHAPE;  // (row << 32 | col) sort keys
    if (nlines == 0) return SGAP_OK;
    if (!d_text || !d_starts || !d_status || !d_r || !d_c || !d_v || !d_tok_off || !d_tok_len)
        return SGAP_ERR_ARG;
    k_mm_parse<<<ingest_grid(nlines), 256, 0, as_stream(stream)>>>(
        d_text, len, reinterpret_cast<const long long *>(d_starts), nlines, rows, cols, d_status,
        reinterpret_cast<long long *>(d_r), reinterpret_cast<long long *>(d_c), d_v,
        reinterpret_cast<long long *>(d_tok_off), reinterpret_cast<int *>(d_tok_len));
    return launch_status();
}

int sgap_mm_expand(int64_t nlines, const uint8_t *d_status, const int64_t *d_r, const int64_t *d_c,
                   const double *d_v, const int64_t *d_pos, int32_t symmetric, int64_t *d_key,
                   double *d_val, void *stream) {
    if (nlines < 0) return SGAP_ERR_ARG;
    if (nlines == 0) return SGAP_OK;
    if (!d_status || !d_r || !d_c || !d_v || !d_pos || !d_key || !d_val) return SGAP_ERR_ARG;
    k_mm_expand<<<ingest_grid(nlines), 256, 0, as_stream(stream)>>>(
        nlines, d_status, reinterpret_cast<const long long *>(d_r),
        reinterpret_cast<const long long *>(d_c), d_v, reinterpret_cast<const long long *>(d_pos),
        symmetric, reinterpret_cast<long long *>(d_key), d_val);
    return launch_status();
}

int sgap_mm_sum_runs(int64_t total, const int64_t *d_key, const double *d_val,
                     const int64_t *d_run_start, int64_t nruns, int64_t *d_row, int64_t *d_col,
                     double *d_out, void *stream) {
    if (total < 0 || nruns < 0) return SGAP_ERR_ARG;
    if (nruns == 0) return SGAP_OK;
    if (!d_key || !d_val || !d_run_start || !d_row || !d_col || !d_out) return SGAP_ERR_ARG;
    k_mm_sum_runs<<<ingest_grid(nruns), 256, 0, as_stream(stream)>>>(
        total, reinterpret_cast<const long long *>(d_key), d_val,
        reinterpret_cast<const long long *>(d_run_start), nruns,
        reinterpret_cast<long long *>(d_row), reinterpret_cast<long long *>(d_col), d_out);
    return launch_status();
}

int sgap_mm_row_ptr(const int64_t *d_row, int64_t nnz, int64_t num_rows, int64_t *d_row_ptr,
                    void *stream) {
    if (nnz < 0 || num_rows < 0 || d_row_ptr == nullptr || (nnz > 0 && d_row == nullptr))
        return SGAP_ERR_ARG;
    k_mm_row_ptr<<<ingest_grid(num_rows + 1), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const long long *>(d_row), nnz, num_rows,
        reinterpret_cast<long long *>(d_row_ptr));
    return launch_status();
}

int sgap_seg_reduce_group(const int64_t *d_idx, const void *d_val, const uint8_t *d_active,
                          int64_t lanes, int32_t group_size, void *d_out, int64_t out_len,
                          int32_t dtype, unsigned long long *d_writebacks, long long *d_fault,
                          void *stream) {
    return prim_entry(true, d_idx, d_val, d_active, lanes, group_size, d_out, out_len, dtype,
                      d_writebacks, d_fault, stream);
}

int sgap_atomic_add_group(const int64_t *d_idx, const void *d_val, const uint8_t *d_active,
                          int64_t lanes, int32_t group_size, void *d_out, int64_t out_len,
                          int32_t dtype, unsigned long long *d_writebacks, long long *d_fault,
                          void *stream) {
    return prim_entry(false, d_idx, d_val, d_active, lanes, group_size, d_out, out_len, dtype,
                      d_writebacks, d_fault, stream);
}

}  // extern "C"
