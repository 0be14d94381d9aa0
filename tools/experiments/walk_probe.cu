// Probe: inner-loop structure of the EB (nnz-split) walk at N=128 on a real
// matrix, stripped of the Sgap bookkeeping (all flushes are red.global.add
// into a zeroed C, float32 accumulation).  Compares the gather-only ceiling
// with walks that differ only in how A is staged and how many B-row gathers
// each lane keeps in flight.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o walk_probe walk_probe.cu
//   ./walk_probe <prefix>      (reads <prefix>.rp/.ci/.av/.rid written by dump_csr.py)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

static std::vector<char> slurp(const char *path) {
    FILE *f = fopen(path, "rb");
    if (!f) { printf("cannot open %s\n", path); exit(1); }
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    std::vector<char> v(n);
    if (fread(v.data(), 1, n, f) != (size_t)n) exit(1);
    fclose(f);
    return v;
}

__device__ __forceinline__ void red4(float *p, float4 a) { atomicAdd(reinterpret_cast<float4 *>(p), a); }

// ---- variant 0: gather only (same index stream) --------------------------------
template <int U>
__global__ void __launch_bounds__(256) k_gather(const int *__restrict__ ci, long long nnz,
                                                const float *__restrict__ B, float *__restrict__ C) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    for (long long base = warp * 32; base < nnz; base += nw * 32) {
        const int my = base + lane < nnz ? __ldg(ci + base + lane) : 0;
#pragma unroll 1
        for (int j = 0; j < 32; j += U) {
            float4 t[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = __shfl_sync(~0u, my, j + u);
                t[u] = __ldg(reinterpret_cast<const float4 *>(B + (long long)c * 128) + lane);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) { acc.x += t[u].x; acc.y += t[u].y; acc.z += t[u].z; acc.w += t[u].w; }
        }
    }
    if (acc.x == 1.2345f) C[0] = acc.y + acc.z + acc.w;
}

struct Acc {  // NUM 0: float32; 1: float32 folded into float64 every 8; 2: Kahan float32;
              // 3: float32 partials TwoSum-folded into a (hi, lo) float32 pair every 8
    float4 a, c;
    double4 t;
    float4 h, l;
};
__device__ __forceinline__ void twosum_fold(float &hi, float &lo, float a) {
    const float s = __fadd_rn(hi, a);
    const float bb = __fsub_rn(s, hi);
    const float err = __fadd_rn(__fsub_rn(hi, __fsub_rn(s, bb)), __fsub_rn(a, bb));
    hi = s;
    lo = __fadd_rn(lo, err);
}
template <int NUM> __device__ __forceinline__ void acc_zero(Acc &s) {
    s.a = make_float4(0, 0, 0, 0); s.c = s.a;
    if (NUM == 1) s.t = make_double4(0, 0, 0, 0);
    if (NUM == 3) { s.h = s.a; s.l = s.a; }
}
__device__ __forceinline__ float kadd(float &sum, float &c, float x) {
    const float y = x - c; const float t = sum + y; c = (t - sum) - y; sum = t; return t;
}
template <int NUM> __device__ __forceinline__ void acc_fma(Acc &s, float v, float4 b) {
    if (NUM == 2) {
        kadd(s.a.x, s.c.x, v * b.x); kadd(s.a.y, s.c.y, v * b.y);
        kadd(s.a.z, s.c.z, v * b.z); kadd(s.a.w, s.c.w, v * b.w);
    } else {
        s.a.x = fmaf(v, b.x, s.a.x); s.a.y = fmaf(v, b.y, s.a.y);
        s.a.z = fmaf(v, b.z, s.a.z); s.a.w = fmaf(v, b.w, s.a.w);
    }
}
template <int NUM> __device__ __forceinline__ void acc_fold(Acc &s) {
    if (NUM == 3) {
        twosum_fold(s.h.x, s.l.x, s.a.x); twosum_fold(s.h.y, s.l.y, s.a.y);
        twosum_fold(s.h.z, s.l.z, s.a.z); twosum_fold(s.h.w, s.l.w, s.a.w);
        s.a = make_float4(0, 0, 0, 0);
    }
    if (NUM == 1) {
        s.t.x += s.a.x; s.t.y += s.a.y; s.t.z += s.a.z; s.t.w += s.a.w;
        s.a = make_float4(0, 0, 0, 0);
    }
}
template <int NUM> __device__ __forceinline__ float4 acc_out(Acc &s) {
    acc_fold<NUM>(s);
    if (NUM == 1) return make_float4((float)s.t.x, (float)s.t.y, (float)s.t.z, (float)s.t.w);
    if (NUM == 3) return make_float4(s.h.x + s.l.x, s.h.y + s.l.y, s.h.z + s.l.z, s.h.w + s.l.w);
    return s.a;
}

// ---- variant 1: lane-staged walk --------------------------------------------------
// A warp owns chunks of G positions (G % 32 == 0).  Per 32-position step each
// lane holds one position's (col, val, row); the next step's triple is loaded
// while this one is consumed.  U B rows are gathered back to back, then
// consumed; a ballot of row changes lets change-free groups skip the flush test.
template <int U, int G, int MODE, int MINB, int NUM = 0>
__global__ void __launch_bounds__(256, MINB) k_staged(const int *__restrict__ rid, const int *__restrict__ ci,
                                                const float *__restrict__ av, long long nnz,
                                                const float *__restrict__ B, float *__restrict__ C) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long nchunks = (nnz + G - 1) / G;
    const float4 *B4 = reinterpret_cast<const float4 *>(B) + lane;
    for (long long ch = warp; ch < nchunks; ch += nw) {
        const long long base = ch * G;
        const long long end = min(base + G, nnz);
        long long q = base + lane;
        int c_n = q < end ? __ldg(ci + q) : 0;
        float v_n = q < end ? __ldg(av + q) : 0.f;
        int r_n = q < end ? __ldg(rid + q) : -1;
        int cur = __shfl_sync(~0u, r_n, 0);
        Acc A;
        acc_zero<NUM>(A);
        for (long long s = base; s < end; s += 32) {
            const int c_l = c_n, r_l = r_n;
            const float v_l = v_n;
            q = s + 32 + lane;
            if (s + 32 < end) {
                c_n = q < end ? __ldg(ci + q) : 0;
                v_n = q < end ? __ldg(av + q) : 0.f;
                r_n = q < end ? __ldg(rid + q) : -1;
            }
            const int nval = (int)min(32LL, end - s);
            const int r_prev = __shfl_up_sync(~0u, r_l, 1);
            const unsigned chg = __ballot_sync(~0u, lane < nval && r_l != (lane == 0 ? cur : r_prev));
#pragma unroll 1
            for (int j = 0; j < nval; j += U) {
                float4 t[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = __shfl_sync(~0u, c_l, j + u);
                    t[u] = (j + u < nval) ? __ldg(B4 + (long long)c * 32) : make_float4(0, 0, 0, 0);
                }
                const unsigned gm = (chg >> j) & ((1u << U) - 1u);
                if (gm == 0) {
#pragma unroll
                    for (int u = 0; u < U; ++u) acc_fma<NUM>(A, __shfl_sync(~0u, v_l, j + u), t[u]);
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const float v = __shfl_sync(~0u, v_l, j + u);
                        const int r = __shfl_sync(~0u, r_l, j + u);
                        if ((gm >> u) & 1u) {
                            const float4 acc = acc_out<NUM>(A);
                            if (MODE == 0) red4(C + (long long)cur * 128 + lane * 4, acc);
                            else if (MODE == 1) __stcs(reinterpret_cast<float4 *>(C + (long long)cur * 128) + lane, acc);
                            else if (acc.x == 1.2345f) C[lane] = acc.y;
                            acc_zero<NUM>(A);
                            cur = r;
                        }
                        acc_fma<NUM>(A, v, t[u]);
                    }
                }
                if (((j + U) & 7) == 0) acc_fold<NUM>(A);
            }
        }
        const float4 acc = acc_out<NUM>(A);
        if (MODE == 0) red4(C + (long long)cur * 128 + lane * 4, acc);
        else if (MODE == 1) __stcs(reinterpret_cast<float4 *>(C + (long long)cur * 128) + lane, acc);
        else if (acc.x == 1.2345f) C[lane] = acc.y;
    }
}

// ---- variant 2: B rows gathered by cp.async into a per-warp shared ring ------
// D positions in flight per warp without holding them in registers.
template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) k_ring(const int *__restrict__ rid, const int *__restrict__ ci,
                                                    const float *__restrict__ av, long long nnz,
                                                    const float *__restrict__ B, float *__restrict__ C) {
    constexpr int G = 512;
    extern __shared__ float4 ring[];  // [8 warps][D][32]
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float4 *my = ring + (size_t)wib * D * 32;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(my) + lane * 16;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long nchunks = (nnz + G - 1) / G;
    for (long long ch = warp; ch < nchunks; ch += nw) {
        const long long base = ch * G;
        const long long end = min(base + G, nnz);
        const int n = (int)(end - base);
        auto issue = [&](int p) {  // position p (relative) -> slot p % D
            if (p < n) {
                const int c = __ldg(ci + base + p);
                const float *src = B + (size_t)(unsigned)c * 128 + lane * 4;
                const unsigned dst = sbase + (unsigned)((p % D) * 32 * 16);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
            }
        };
        // prologue: D positions in flight, one commit group per 4
        for (int p = 0; p < D; p += 4) {
            issue(p); issue(p + 1); issue(p + 2); issue(p + 3);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        int cur = __ldg(rid + base);
        float4 acc = make_float4(0, 0, 0, 0);
        for (int p = 0; p < n; p += 4) {
            asm volatile("cp.async.wait_group %0;" ::"n"(D / 4 - 1) : "memory");
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (p + u < n) {
                    const float4 b = my[((p + u) % D) * 32 + lane];
                    const float v = __ldg(av + base + p + u);
                    const int r = __ldg(rid + base + p + u);
                    if (r != cur) {
                        atomicAdd(reinterpret_cast<float4 *>(C + (long long)cur * 128) + lane, acc);
                        acc = make_float4(0, 0, 0, 0);
                        cur = r;
                    }
                    acc.x = fmaf(v, b.x, acc.x); acc.y = fmaf(v, b.y, acc.y);
                    acc.z = fmaf(v, b.z, acc.z); acc.w = fmaf(v, b.w, acc.w);
                }
            }
            __syncwarp();
            issue(p + D); issue(p + D + 1); issue(p + D + 2); issue(p + D + 3);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        atomicAdd(reinterpret_cast<float4 *>(C + (long long)cur * 128) + lane, acc);
        __syncwarp();
    }
}

// ---- reference: one thread per (row, column), float64 ------------------------------
__global__ void k_ref(const int *rp, const int *ci, const float *av, int M, const float *B, double *C) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)M * 128) return;
    const int i = (int)(t / 128), k = (int)(t % 128);
    double s = 0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) s += (double)av[p] * (double)B[(long long)ci[p] * 128 + k];
    C[t] = s;
}

__global__ void k_err(const float *got, const double *want, long long n, float *out) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    float e = 0;
    for (; t < n; t += (long long)gridDim.x * blockDim.x)
        e = fmaxf(e, (float)(fabs((double)got[t] - want[t]) / (fabs(want[t]) + 1.0)));
    for (int o = 16; o; o >>= 1) e = fmaxf(e, __shfl_xor_sync(~0u, e, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int *>(out), __float_as_int(e));
}

template <class F>
static float timeit(F f, int reps = 7) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (r && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return best;
}

int main(int argc, char **argv) {
    const char *pre = argc > 1 ? argv[1] : "/tmp/c2";
    char path[512];
    snprintf(path, sizeof path, "%s.rp", pre); auto hrp = slurp(path);
    snprintf(path, sizeof path, "%s.ci", pre); auto hci = slurp(path);
    snprintf(path, sizeof path, "%s.av", pre); auto hav = slurp(path);
    snprintf(path, sizeof path, "%s.rid", pre); auto hrid = slurp(path);
    const int M = (int)(hrp.size() / 4) - 1;
    const long long nnz = (long long)hci.size() / 4;
    const int K = M, N = 128;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int *rp, *ci, *rid; float *av, *B, *C, *err; double *R;
    CK(cudaMalloc(&rp, hrp.size())); CK(cudaMalloc(&ci, hci.size())); CK(cudaMalloc(&rid, hrid.size()));
    CK(cudaMalloc(&av, hav.size()));
    CK(cudaMalloc(&B, (size_t)K * N * 4)); CK(cudaMalloc(&C, (size_t)M * N * 4));
    CK(cudaMalloc(&R, (size_t)M * N * 8)); CK(cudaMalloc(&err, 4));
    cudaMemcpy(rp, hrp.data(), hrp.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(ci, hci.data(), hci.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(rid, hrid.data(), hrid.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(av, hav.data(), hav.size(), cudaMemcpyHostToDevice);
    {
        std::vector<float> hb((size_t)K * N);
        unsigned s = 1;
        for (auto &x : hb) { s = s * 1664525u + 1013904223u; x = (s >> 8) / 8388608.0f - 1.0f; }
        cudaMemcpy(B, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
    }
    k_ref<<<(unsigned)(((long long)M * N + 255) / 256), 256>>>(rp, ci, av, M, B, R);
    CK(cudaDeviceSynchronize());
    printf("M=%d nnz=%lld N=%d\n", M, nnz, N);
    auto check = [&](const char *name, float ms) {
        cudaMemset(err, 0, 4);
        k_err<<<1184, 256>>>(C, R, (long long)M * N, err);
        float e; cudaMemcpy(&e, err, 4, cudaMemcpyDeviceToHost);
        printf("%-28s %.3f ms  %.0f GFLOP/s  err %.2e\n", name, ms, 2.0 * nnz * N / ms / 1e6, e);
    };
    int occ;
#define GATHER(U)                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather<U>, 256, 0);                  \
    printf("%-28s %.3f ms (occ %d)\n", "gather-only U=" #U,                                    \
           timeit([&] { k_gather<U><<<sms * occ, 256>>>(ci, nnz, B, C); }), occ);
    GATHER(2) GATHER(4) GATHER(8)
#define STAGEDN(U, G, MODE, MINB, NUM)                                                             \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_staged<U, G, MODE, MINB, NUM>, 256, 0);   \
    {                                                                                          \
        cudaMemsetAsync(C, 0, (size_t)M * N * 4);                                              \
        float ms = timeit([&] {                                                                \
            k_staged<U, G, MODE, MINB, NUM><<<sms * occ, 256>>>(rid, ci, av, nnz, B, C);            \
        });                                                                                    \
        char nm[64]; snprintf(nm, 64, "staged U=%d G=%d mode=%d num=%d occ=%d", U, G, MODE, NUM, occ);     \
        if (MODE == 0) {                                                                       \
            cudaMemsetAsync(C, 0, (size_t)M * N * 4);                                          \
            k_staged<U, G, MODE, MINB, NUM><<<sms * occ, 256>>>(rid, ci, av, nnz, B, C);            \
            check(nm, ms);                                                                     \
        } else printf("%-28s %.3f ms\n", nm, ms);                                             \
    }
    STAGEDN(4, 256, 0, 4, 0) STAGEDN(4, 256, 0, 4, 1) STAGEDN(4, 256, 0, 4, 3)
    STAGEDN(8, 256, 0, 3, 0) STAGEDN(8, 256, 0, 3, 1) STAGEDN(8, 256, 0, 3, 3)
    STAGEDN(4, 256, 2, 4, 0) STAGEDN(4, 256, 2, 4, 1) STAGEDN(4, 256, 2, 4, 3)
#define RING(D, MINB)                                                                              \
    {                                                                                              \
        const size_t smem = (size_t)8 * D * 32 * 16;                                               \
        cudaFuncSetAttribute(k_ring<D, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ring<D, MINB>, 256, smem);           \
        cudaMemsetAsync(C, 0, (size_t)M * N * 4);                                                  \
        k_ring<D, MINB><<<sms * occ, 256, smem>>>(rid, ci, av, nnz, B, C);                         \
        CK(cudaDeviceSynchronize());                                                               \
        char nm[64]; snprintf(nm, 64, "ring D=%d occ=%d", D, occ);                                 \
        float ms = timeit([&] { k_ring<D, MINB><<<sms * occ, 256, smem>>>(rid, ci, av, nnz, B, C); }); \
        cudaMemsetAsync(C, 0, (size_t)M * N * 4);                                                  \
        k_ring<D, MINB><<<sms * occ, 256, smem>>>(rid, ci, av, nnz, B, C);                         \
        check(nm, ms);                                                                             \
    }
    RING(8, 4) RING(16, 3) RING(16, 4) RING(24, 2) RING(32, 2)
    float zms = timeit([&] { cudaMemsetAsync(C, 0, (size_t)M * N * 4); });
    printf("%-28s %.3f ms\n", "memset C alone", zms);
    return 0;
}
