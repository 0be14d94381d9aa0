// Probe: column-window staging for banded / mesh SpMM (config 4's shape: a
// 27-point stencil on a 160^3 grid, N = 128, float32).  Compares
//   (a) the warp-per-row gather walk (B rows through L1/L2, like k_row_staged),
//   (b) a window-staged walk: a CTA owns one grid line (160 consecutive rows)
//       and one S-column slice; it stages the 9 neighbouring lines' B slices
//       (the union of every column the line's rows touch: contiguous windows)
//       into shared memory once, then each nonzero reads its B slice from
//       shared memory through a precomputed 16-bit window slot (what a
//       generic plan would store per nonzero).
// Both sum each (row, column) serially in position order, so they agree to
// float32 rounding; the probe reports max |a - b| and the timings.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o window_probe window_probe.cu
//   ./window_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cmath>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int SIDE = 160, N = 128;

// (a) warp per row, 32 lanes x float4 = 128 columns, rows interleaved across the CTA
__global__ void __launch_bounds__(256) k_gather(const int *rp, const int *ci, const float *av,
                                                const float *B, float *C, int M) {
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < M; i += warps) {
        const int beg = rp[i], end = rp[i + 1];
        float4 acc = make_float4(0, 0, 0, 0);
        for (int s = beg; s < end; s += 32) {
            const int q = s + lane;
            const int c_l = q < end ? __ldg(ci + q) : 0;
            const float v_l = q < end ? __ldg(av + q) : 0.f;
            const int nv = min(32, end - s);
            for (int j = 0; j < nv; j += 4) {
                float4 b[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    b[u] = __ldg(reinterpret_cast<const float4 *>(B + (size_t)__shfl_sync(~0u, c_l, (j + u) & 31) * N) + lane);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float v = __shfl_sync(~0u, v_l, (j + u) & 31);
                    if (j + u < nv) {
                        acc.x = fmaf(v, b[u].x, acc.x); acc.y = fmaf(v, b[u].y, acc.y);
                        acc.z = fmaf(v, b[u].z, acc.z); acc.w = fmaf(v, b[u].w, acc.w);
                    }
                }
            }
        }
        reinterpret_cast<float4 *>(C + (size_t)i * N)[lane] = acc;
    }
}

// (b) window-staged: CTA = (line, slice of S columns); smem [9 * SIDE][S]
template <int S>
__global__ void __launch_bounds__(640) k_window(const int *rp, const unsigned short *slot,
                                                         const float *av, const float *B, float *C) {
    extern __shared__ float4 sm[];
    constexpr int LPR = S / 4;  // lanes per row
    const int slices = N / S;
    const int line = blockIdx.x / slices, sl = blockIdx.x % slices;
    const int z = line / SIDE, y = line % SIDE;
    const int col0 = sl * S;
    // stage: window w = (dz+1)*3 + (dy+1) holds line (z+dz, y+dy), x = 0..SIDE-1
    for (int t = threadIdx.x; t < 9 * SIDE * LPR; t += blockDim.x) {
        const int w = t / (SIDE * LPR), rem = t % (SIDE * LPR);
        const int x = rem / LPR, part = rem % LPR;
        const int zz = z + w / 3 - 1, yy = y + w % 3 - 1;
        float4 v = make_float4(0, 0, 0, 0);
        if (zz >= 0 && zz < SIDE && yy >= 0 && yy < SIDE)
            v = __ldg(reinterpret_cast<const float4 *>(B + ((size_t)(zz * SIDE + yy) * SIDE + x) * N + col0) + part);
        sm[(w * SIDE + x) * LPR + part] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < SIDE * LPR; t += blockDim.x) {  // S = 32: two rows per thread
        const int x = t / LPR, part = t % LPR;
        const int i = line * SIDE + x;
        const int beg = __ldg(rp + i), end = __ldg(rp + i + 1);
        float4 acc = make_float4(0, 0, 0, 0);
        for (int p = beg; p < end; ++p) {
            const float v = __ldg(av + p);
            const float4 b = sm[(int)__ldg(slot + p) * LPR + part];
            acc.x = fmaf(v, b.x, acc.x); acc.y = fmaf(v, b.y, acc.y);
            acc.z = fmaf(v, b.z, acc.z); acc.w = fmaf(v, b.w, acc.w);
        }
        reinterpret_cast<float4 *>(C + (size_t)i * N + col0)[part] = acc;
    }
}

int main() {
    const int M = SIDE * SIDE * SIDE;
    std::vector<int> rp(M + 1), ci;
    std::vector<unsigned short> slot;
    std::vector<float> av;
    ci.reserve((size_t)M * 27);
    slot.reserve((size_t)M * 27);
    srand(1);
    for (int z = 0; z < SIDE; ++z)
        for (int y = 0; y < SIDE; ++y)
            for (int x = 0; x < SIDE; ++x) {
                rp[(z * SIDE + y) * SIDE + x] = (int)ci.size();
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int zz = z + dz, yy = y + dy, xx = x + dx;
                            if (zz < 0 || zz >= SIDE || yy < 0 || yy >= SIDE || xx < 0 || xx >= SIDE) continue;
                            ci.push_back((zz * SIDE + yy) * SIDE + xx);
                            slot.push_back((unsigned short)(((dz + 1) * 3 + dy + 1) * SIDE + xx));
                            av.push_back((float)rand() / RAND_MAX * 2.f - 1.f);
                        }
            }
    rp[M] = (int)ci.size();
    const size_t nnz = ci.size();
    std::vector<float> hb((size_t)M * N);
    for (auto &v : hb) v = (float)rand() / RAND_MAX * 2.f - 1.f;
    int *d_rp, *d_ci;
    unsigned short *d_slot;
    float *d_av, *d_b, *d_c1, *d_c2;
    CK(cudaMalloc(&d_rp, (M + 1) * 4));
    CK(cudaMalloc(&d_ci, nnz * 4));
    CK(cudaMalloc(&d_slot, nnz * 2));
    CK(cudaMalloc(&d_av, nnz * 4));
    CK(cudaMalloc(&d_b, (size_t)M * N * 4));
    CK(cudaMalloc(&d_c1, (size_t)M * N * 4));
    CK(cudaMalloc(&d_c2, (size_t)M * N * 4));
    CK(cudaMemcpy(d_rp, rp.data(), (M + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_slot, slot.data(), nnz * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_av, av.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, hb.data(), (size_t)M * N * 4, cudaMemcpyHostToDevice));
    printf("stencil27 side %d: M %d nnz %zu N %d\n", SIDE, M, nnz, N);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int r = 0; r < 7; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = fminf(best, ms);
        }
        printf("%-40s %8.3f ms  %8.1f GF/s\n", name, best, 2.0 * nnz * N / (best * 1e6));
    };
    timeit("(a) warp-per-row gather", [&] { k_gather<<<148 * 8, 256>>>(d_rp, d_ci, d_av, d_b, d_c1, M); });
    std::vector<float> c1((size_t)M * N), c2((size_t)M * N);
    CK(cudaMemcpy(c1.data(), d_c1, c1.size() * 4, cudaMemcpyDeviceToHost));
    auto check = [&](const char *name) {
        CK(cudaMemcpy(c2.data(), d_c2, c2.size() * 4, cudaMemcpyDeviceToHost));
        double err = 0;
        for (size_t k = 0; k < c1.size(); ++k) err = fmax(err, fabs((double)c1[k] - c2[k]) / (fabs((double)c1[k]) + 1));
        printf("   %s max rel diff vs (a): %.3e\n", name, err);
    };
    {
        constexpr int S = 16;
        const int smem = 9 * SIDE * S * 4;
        CK(cudaFuncSetAttribute(k_window<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        timeit("(b) window-staged S=16 (92 KB smem)", [&] {
            k_window<S><<<SIDE * SIDE * (N / S), (SIDE * S / 4 > 640 ? 640 : SIDE * S / 4), smem>>>(d_rp, d_slot, d_av, d_b, d_c2);
        });
        CK(cudaGetLastError());
        check("S=16");
    }
    {
        constexpr int S = 8;
        const int smem = 9 * SIDE * S * 4;
        CK(cudaFuncSetAttribute(k_window<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        timeit("(b) window-staged S=8 (46 KB smem)", [&] {
            k_window<S><<<SIDE * SIDE * (N / S), (SIDE * S / 4 > 640 ? 640 : SIDE * S / 4), smem>>>(d_rp, d_slot, d_av, d_b, d_c2);
        });
        CK(cudaGetLastError());
        check("S=8");
    }
    {
        constexpr int S = 32;
        const int smem = 9 * SIDE * S * 4;
        CK(cudaFuncSetAttribute(k_window<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        timeit("(b) window-staged S=32 (184 KB smem, 640 threads)", [&] {
            k_window<S><<<SIDE * SIDE * (N / S), (SIDE * S / 4 > 640 ? 640 : SIDE * S / 4), smem>>>(d_rp, d_slot, d_av, d_b, d_c2);
        });
        CK(cudaGetLastError());
        check("S=32");
    }
    return 0;
}
