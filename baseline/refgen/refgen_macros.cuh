// Bodies for the group macros the reference's emitted CUDA declares but never
// defines (cuda.py:52-56 DEVICE_PRELUDE), following the simulator's
// semantics (sim.py:112-165).  Used only to run the reference compiler's own
// kernels on B200 as the fixed-schedule ("naive TACO") baseline; the product
// kernels use paper_2209_02882_b200/csrc/sgap_device.cuh.
//
// Every emitted kernel reaches a macro with whole G-lane groups active (the
// only guards before a macro are per-group `break`s), so the shuffles run on
// __activemask() with full groups.
#pragma once
#include <cuda_runtime.h>

namespace refgen {

__device__ __forceinline__ unsigned laneid() {
    unsigned l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

// AtomicAddGroup (sim.py:112-136): the G lanes of an aligned group share
// `index`; one writeback of the group sum, from the group's first lane.
template <typename T, int G>
__device__ __forceinline__ void atomic_add_group(T *array, int index, T value) {
    const unsigned mask = __activemask();
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) value += __shfl_xor_sync(mask, value, off, G);
    if ((laneid() & (G - 1)) == 0) atomicAdd(array + index, value);
}

// SegReduceGroup (sim.py:139-165): within an aligned G-lane group, each run of
// equal `index` produces one writeback of the run sum (from its last lane).
template <typename T, int G>
__device__ __forceinline__ void seg_reduce_group(T *array, int index, T value) {
    const unsigned mask = __activemask();
    const unsigned lane = laneid();
    const unsigned gl = lane & (G - 1);
    const int prev_idx = __shfl_up_sync(mask, index, 1, G);
    const int next_idx = __shfl_down_sync(mask, index, 1, G);
    const bool head = gl == 0 || prev_idx != index;
    const bool tail = gl == G - 1 || next_idx != index;
    const unsigned heads = __ballot_sync(mask, head);
    const unsigned upto = heads & ((2u << lane) - 1u);  // heads at lanes <= this one
    const int dist = (int)lane - (31 - __clz(upto));
    T v = value;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const T up = __shfl_up_sync(mask, v, d, G);
        if (d <= dist) v += up;
    }
    if (tail) atomicAdd(array + index, v);
}

}  // namespace refgen
