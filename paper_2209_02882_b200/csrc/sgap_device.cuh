// sgap_device.cuh -- device building blocks shared by the SpMM families:
// vector gathers/stores/reductions over B and C rows, the clamped row search,
// and the warp-shuffle group reductions that replace the simulator's macros
// (sim.py:112-165; declared-only in the reference's emitted CUDA, cuda.py:52-56).
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

namespace sgap {

constexpr unsigned kFull = 0xffffffffu;

// The hardware lane (%laneid): equal to threadIdx.x & 31 for 1-D blocks,
// and still right for the 2-D blocks of k_rbpr_grid.
__device__ __forceinline__ unsigned lane_id() {
    unsigned l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

// ---------------------------------------------------------------------------
// c-wide column vectors (c in {1,2,4}); the per-lane unit of a B-row gather and
// of a C writeback.  A column tile of c consecutive floats is one 4/8/16-byte
// access; (32/lanes_per_row) tiles of one B row form one coalesced request.
// ---------------------------------------------------------------------------
template <typename T, int V>
struct Vec {
    T v[V];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int x = 0; x < V; ++x) v[x] = T(0);
    }
};

template <typename T, int V>
__device__ __forceinline__ void ldg_vec(Vec<T, V> &o, const T *p);

template <>
__device__ __forceinline__ void ldg_vec<float, 1>(Vec<float, 1> &o, const float *p) {
    o.v[0] = __ldg(p);
}
template <>
__device__ __forceinline__ void ldg_vec<float, 2>(Vec<float, 2> &o, const float *p) {
    const float2 t = __ldg(reinterpret_cast<const float2 *>(p));
    o.v[0] = t.x; o.v[1] = t.y;
}
template <>
__device__ __forceinline__ void ldg_vec<float, 4>(Vec<float, 4> &o, const float *p) {
    const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
    o.v[0] = t.x; o.v[1] = t.y; o.v[2] = t.z; o.v[3] = t.w;
}
template <>
__device__ __forceinline__ void ldg_vec<double, 1>(Vec<double, 1> &o, const double *p) {
    o.v[0] = __ldg(p);
}
template <>
__device__ __forceinline__ void ldg_vec<double, 2>(Vec<double, 2> &o, const double *p) {
    const double2 t = __ldg(reinterpret_cast<const double2 *>(p));
    o.v[0] = t.x; o.v[1] = t.y;
}
template <>
__device__ __forceinline__ void ldg_vec<double, 4>(Vec<double, 4> &o, const double *p) {
    const double2 t0 = __ldg(reinterpret_cast<const double2 *>(p));
    const double2 t1 = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    o.v[0] = t0.x; o.v[1] = t0.y; o.v[2] = t1.x; o.v[3] = t1.y;
}

// B-row gather as a volatile load: issued where written (the compiler may not
// sink it into the branch that consumes it), so U gathers stay back to back.
template <typename T, int V>
__device__ __forceinline__ void gather_vec(Vec<T, V> &o, const T *p) {
    if constexpr (sizeof(T) == 4 && V == 4) {
        asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(o.v[0]), "=f"(o.v[1]), "=f"(o.v[2]), "=f"(o.v[3])
                     : "l"(p));
    } else if constexpr (sizeof(T) == 4 && V == 2) {
        asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(o.v[0]), "=f"(o.v[1]) : "l"(p));
    } else if constexpr (sizeof(T) == 4 && V == 1) {
        asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(o.v[0]) : "l"(p));
    } else if constexpr (sizeof(T) == 8 && V == 1) {
        asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(o.v[0]) : "l"(p));
    } else if constexpr (sizeof(T) == 8 && V == 2) {
        asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(o.v[0]), "=d"(o.v[1]) : "l"(p));
    } else {
        asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(o.v[0]), "=d"(o.v[1]) : "l"(p));
        asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];"
                     : "=d"(o.v[2]), "=d"(o.v[3])
                     : "l"(p + 2));
    }
}

// Quotient of a non-negative 64-bit index by a runtime divisor that is
// usually a power of two (N, N/c): a shift then, else a 32-bit division when
// both fit, else the 64-bit one (~70 instructions, which dominated the
// per-cell overhead of row-reciprocal at one cell per warp).
struct Divider {
    long long d;
    int shift;  // log2(d), or -1
    __host__ __device__ static Divider make(long long d) {
        Divider v{d, -1};
        if (d > 0 && (d & (d - 1)) == 0) {
            int s = 0;
            while ((1LL << s) < d) ++s;
            v.shift = s;
        }
        return v;
    }
    __device__ __forceinline__ long long div(long long x) const {
        if (shift >= 0) return x >> shift;
        if (x < 0x7fffffffLL && d < 0x7fffffffLL) return (long long)((unsigned)x / (unsigned)d);
        return x / d;
    }
};

// Row `r` (r >= 0) of a row-major matrix with n elements per row: one
// IMAD.WIDE.U32 (32x32 -> 64-bit multiply-add onto the base) where a signed
// 64-bit index costs a sign extension and a 64-bit multiply (~6 SASS
// instructions per B-row gather in the walks' hot loops).
template <typename T>
__device__ __forceinline__ const T *row_ptr(const T *base, int r, int n) {
    return reinterpret_cast<const T *>(reinterpret_cast<const char *>(base) +
                                       (unsigned long long)(unsigned)r *
                                           (unsigned long long)((unsigned)n * (unsigned)sizeof(T)));
}

// Software prefetch of a streamed A line into L1 (non-blocking, no register).
__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void prefetch_l1(const void *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Plain (read-modify-)write of an exclusively owned C tile.  C is written
// exactly once per kernel, so 16-byte tiles are stored evict-first
// (st.global.cs) to keep L2 for the B rows that are re-gathered.
template <typename T, int V>
__device__ __forceinline__ void store_vec(T *p, const Vec<T, V> &a, bool accumulate) {
    Vec<T, V> o = a;
    if (accumulate) {
#pragma unroll
        for (int x = 0; x < V; ++x) o.v[x] += p[x];
    }
    if constexpr (sizeof(T) * V < 16) {
        // narrow tiles: one warp writes a few bytes of a sector, its
        // neighbours the rest -- an evict-first line would leave L2 before
        // they land and cost a DRAM read-modify-write, so plain stores
#pragma unroll
        for (int x = 0; x < V; ++x) p[x] = o.v[x];
        return;
    }
    if constexpr (sizeof(T) * V == 16) {
        if constexpr (sizeof(T) == 4)
            __stcs(reinterpret_cast<float4 *>(p), make_float4(o.v[0], o.v[1], o.v[2], o.v[3]));
        else
            __stcs(reinterpret_cast<double2 *>(p), make_double2(o.v[0], o.v[1]));
    } else if constexpr (sizeof(T) * V == 8 && sizeof(T) == 4) {
        __stcs(reinterpret_cast<float2 *>(p), make_float2(o.v[0], o.v[1]));
    } else if constexpr (V == 4) {  // double x4
        __stcs(reinterpret_cast<double2 *>(p), make_double2(o.v[0], o.v[1]));
        __stcs(reinterpret_cast<double2 *>(p) + 1, make_double2(o.v[2], o.v[3]));
    } else {
#pragma unroll
        for (int x = 0; x < V; ++x) __stcs(p + x, o.v[x]);
    }
}

// Atomic writeback of a C tile that other lanes may also update
// (red.global.add.{f32,v2.f32,v4.f32,f64}; the result is unused so ptxas
// emits REDG).
template <typename T, int V>
__device__ __forceinline__ void red_vec(T *p, const Vec<T, V> &a) {
    if constexpr (sizeof(T) == 4 && V == 4) {
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(a.v[0], a.v[1], a.v[2], a.v[3]));
    } else if constexpr (sizeof(T) == 4 && V == 2) {
        atomicAdd(reinterpret_cast<float2 *>(p), make_float2(a.v[0], a.v[1]));
    } else {
#pragma unroll
        for (int x = 0; x < V; ++x) atomicAdd(p + x, a.v[x]);
    }
}

template <typename T, int V>
__device__ __forceinline__ void fma_vec(Vec<T, V> &acc, T a, const Vec<T, V> &b) {
#pragma unroll
    for (int x = 0; x < V; ++x) acc.v[x] = fma(a, b.v[x], acc.v[x]);
}

template <typename T, int V>
__device__ __forceinline__ void add_vec(Vec<T, V> &acc, const Vec<T, V> &b) {
#pragma unroll
    for (int x = 0; x < V; ++x) acc.v[x] += b.v[x];
}

// ---------------------------------------------------------------------------
// Accumulation numerics.  Products and short partial sums (<= 8 terms) are
// formed in the value type; every running sum that can grow past that is
// carried in float64 ("tot") and rounded to the value type once, at the
// writeback.  (32-term float32 partials of config 2's hub row, whose summed
// duplicate values reach |a| ~ 10, already cost 8.5e-6 of the 1e-5 budget.)  Without this a 40k-nonzero power-law row summed serially in
// float32 misses the 1e-5 bound of the reference metric by 20x.
// ---------------------------------------------------------------------------
template <typename T, int V>
__device__ __forceinline__ void fold(Vec<double, V> &tot, Vec<T, V> &acc) {
#pragma unroll
    for (int x = 0; x < V; ++x) {
        tot.v[x] += (double)acc.v[x];
        acc.v[x] = T(0);
    }
}

// Error-free accumulation of long rows (> kExactRow nonzeros) uses float64
// products of the float32 inputs -- exact, since 24 + 24 bits fit in 53 --
// summed in float64 (DFMA), in every family.

template <typename T, int V>
__device__ __forceinline__ Vec<T, V> narrow(const Vec<double, V> &tot) {
    Vec<T, V> o;
#pragma unroll
    for (int x = 0; x < V; ++x) o.v[x] = (T)tot.v[x];
    return o;
}

// Rows long enough that many separate atomic flushes land on them (hub rows
// of power-law matrices) accumulate those flushes in a float64 side table
// instead of float32 C; a fold pass adds the table into C afterwards.
struct LongRows {
    const int *rows;      // sorted row ids of the table (long or chunk-straddling)
    const int *count;     // number of entries in `rows` (device scalar)
    double *acc;          // [capacity x N] float64 partial sums
    long long threshold;  // < 0: side table disabled (float64 values, RB families)
    const int *slot;      // row -> table slot (nullptr: binary search of `rows`)
    long long chunk;      // > 0: every row straddling a `chunk` boundary is in the table
    const int *exact_rows;  // rows taking the error-free pass (nnz-multiple)
    int exact_count;
    const int *chunk_rows;  // row owning each g-chunk's first position (register
                            // walk without row ids); nullptr: use the row ids
    const unsigned *union_e[2];  // row-blocked RB walk: union column streams of
    const int *union_off[2];     // 4-row [0] and 8-row [1] blocks (k_union_rows)
    const int *col_hinted;       // col_idx with bit 31 on cold columns (variant 9)
    void *panel_b;               // panel-major copy of B (variant 10; host side only)
    int panel_lanes;             // its panel width in c-wide tiles (0: none)
};

// Row ids carry bit 31 when the row belongs to the long-row table and bit 30
// when it is long enough for float32 product rounding to matter (kExactRow).
constexpr int kLongFlag = (int)0x80000000u;
constexpr int kExactFlag = 0x40000000;
constexpr int kRowMask = 0x3fffffff;
// Float32 product rounding alone is a random walk of std ~3.4e-8 *
// sqrt(n) * rms(a*b); over millions of outputs its 5-sigma tail reaches the
// 1e-5 bound (metric max|err|/(|want|+1)) near n ~ 2e4: config 3's
// Chung-Lu hub rows (~20-60k nonzeros) measured 1.33e-5 with plain float32
// products.  Rows beyond this take the error-free accumulate (TwoProduct +
// TwoSum); at 4096 the 5-sigma tail stays under ~4.5e-6.
constexpr int kExactRow = 4096;

// One atomic writeback of a (row, column tile) partial; `rid` is a row id
// (possibly flagged long).
template <typename T, int V>
__device__ __forceinline__ void flush_row(T *__restrict__ C, int N, int rid, long long kcol,
                                          const Vec<double, V> &tot, const LongRows &lr) {
    const int row = rid & kRowMask;
    if (rid < 0 && lr.threshold >= 0) {
        int lo;
        if (lr.slot != nullptr) {
            lo = __ldg(lr.slot + row);
        } else {
            lo = 0;
            int hi = *lr.count;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(lr.rows + mid) < row) lo = mid + 1; else hi = mid;
            }
        }
        double *p = lr.acc + (long long)lo * N + kcol;
#pragma unroll
        for (int x = 0; x < V; ++x) atomicAdd(p + x, tot.v[x]);
    } else {
        red_vec<T, V>(C + (long long)row * N + kcol, narrow<T, V>(tot));
    }
}

// ---------------------------------------------------------------------------
// binary_search_before (lowering.py:99-116; device text cuda.py:37-50):
// largest p in [lo, hi) with a[p] <= target, clamped to lo.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int search_before(const int *__restrict__ a, int lo, int hi,
                                             long long target) {
    if (hi <= lo) return lo;
    if ((long long)__ldg(a + lo) > target) return lo;
    while (hi - lo > 1) {
        const int mid = (int)(((unsigned)lo + (unsigned)hi) >> 1);
        if ((long long)__ldg(a + mid) <= target) lo = mid; else hi = mid;
    }
    return lo;
}

// Row a position-chunked lane resolves to (lowering.py:459-500): clamped
// search in the block window [starts[b], min(starts[b+1]+1, M)), then -- for
// in-range positions -- the forward advance over rows ending at the position.
__device__ __forceinline__ int lane_row(const int *__restrict__ rp,
                                        const int *__restrict__ starts, long long block,
                                        long long pos, long long nnz, int M) {
    int hi = __ldg(starts + block + 1) + 1;
    hi = hi < M ? hi : M;
    int i = search_before(rp, __ldg(starts + block), hi, pos);
    if (pos < nnz) {
        while (pos == (long long)__ldg(rp + i + 1)) ++i;
    }
    return i;
}

// ---------------------------------------------------------------------------
// Segment group (SegReduceGroup, sim.py:139-165): within each aligned group of
// R lanes, runs of equal key among ACTIVE lanes (inactive lanes do not break a
// run) each produce one writeback from the run's last active lane.
// The segment heads come from one ballot; the run sums from a log2(R)-step
// shfl_up scan restricted to the distance to the lane's head.
// ---------------------------------------------------------------------------
struct SegLanes {
    bool head;        // first active lane of a run
    bool tail;        // last active lane of a run: owns the writeback
    bool decreasing;  // key below the previous active key (group invariant broken)
    int dist;         // lanes back to the run head (scan reach)
};

template <int R, typename K>
__device__ __forceinline__ SegLanes seg_lanes(K key, bool active) {
    const unsigned lane = lane_id();
    const unsigned gbase = lane & ~(unsigned)(R - 1);
    const unsigned gmask = (R >= 32) ? kFull : (((1u << R) - 1u) << gbase);
    const unsigned le = kFull >> (31u - lane);
    const unsigned act = __ballot_sync(kFull, active) & gmask;
    const unsigned below = act & (le ^ (1u << lane));
    const int prev = below ? 31 - __clz(below) : (int)lane;
    const K prev_key = __shfl_sync(kFull, key, prev);
    SegLanes s;
    s.head = active && (below == 0u || prev_key != key);
    s.decreasing = active && below != 0u && key < prev_key;
    const unsigned heads = __ballot_sync(kFull, s.head);
    const unsigned above = act & ~le;
    const int next = above ? __ffs(above) - 1 : -1;
    s.tail = active && (next < 0 || ((heads >> next) & 1u));
    const unsigned hb = heads & le & gmask;
    s.dist = hb ? (int)lane - (31 - __clz(hb)) : 0;
    return s;
}

template <int R, typename T>
__device__ __forceinline__ T seg_scan(T v, int dist) {
#pragma unroll
    for (int d = 1; d < R; d <<= 1) {
        const T up = __shfl_up_sync(kFull, v, d, R);
        if (d <= dist) v += up;
    }
    return v;
}

template <int R, typename T, int V>
__device__ __forceinline__ void seg_scan_vec(Vec<T, V> &a, int dist) {
#pragma unroll
    for (int d = 1; d < R; d <<= 1) {
#pragma unroll
        for (int x = 0; x < V; ++x) {
            const T up = __shfl_up_sync(kFull, a.v[x], d, R);
            if (d <= dist) a.v[x] += up;
        }
    }
}

// Parallel group (AtomicAddGroup, sim.py:112-136): xor-tree sum over R lanes;
// every lane ends with the group total.
template <int R, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
    for (int off = R / 2; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off, R);
    return v;
}

template <int R, typename T, int V>
__device__ __forceinline__ void group_sum_vec(Vec<T, V> &a) {
#pragma unroll
    for (int off = R / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int x = 0; x < V; ++x) a.v[x] += __shfl_xor_sync(kFull, a.v[x], off, R);
    }
}

// Programmatic dependent launch (sm_90+): a primary grid lets its dependent
// start early; the dependent waits for the primary's completion (and memory)
// where it needs it.  Both are no-ops for a normally launched grid.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Warp-aggregated writeback counter (SimMetrics.atomic_ops).
__device__ __forceinline__ void flush_count(unsigned long long *counter, unsigned long long mine) {
    if (counter == nullptr) return;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(kFull, mine, off);
    if (lane_id() == 0 && mine) atomicAdd(counter, mine);
}

}  // namespace sgap

namespace sgap {

// ---------------------------------------------------------------------------
// Bulk async copies (TMA engine, cp.async.bulk) + mbarrier pipeline helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D global -> shared bulk copy completing on `bar` (bytes % 16 == 0, both
// addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace sgap
