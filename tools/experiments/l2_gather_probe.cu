// Probe: how fast can B200 gather whole B rows (N fp32 = N*4 bytes) by a
// random row index, as the SpMM walks do?  Measures the L2->SM gather
// ceiling that bounds the nnz-multiple / row-multiple kernels on R-MAT.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather_probe l2_gather_probe.cu
//   ./l2_gather_probe            (prints one line per (table rows, N, in-flight) case)
//
// Each warp walks a stream of row indices (one coalesced 4-B index per lane,
// broadcast by shuffle like col_idx in the walks) and gathers U rows at a
// time; lane l owns columns [4l, 4l+4) of every row (N=128) or a slice of
// them.  GB/s = gathered row bytes / kernel time (CUDA events, best of 5).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__global__ void make_idx(int *idx, long long n, uint32_t rows, int skew) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i < n; i += (long long)gridDim.x * blockDim.x) {
        uint32_t h = mix((uint32_t)i * 2654435761U + 12345U);
        if (skew) {
            // power-law-ish: u^4 concentrates on low rows, then scatter by a hash
            float u = (h & 0xffffff) / 16777216.0f;
            uint32_t r = (uint32_t)(u * u * u * u * rows);
            idx[i] = (int)(mix(r + 77U) % rows);
        } else {
            idx[i] = (int)(h % rows);
        }
    }
}

template <int U, int V>  // U rows in flight per lane, V floats per lane per row
__global__ void __launch_bounds__(256) gather(const int *__restrict__ idx, long long n,
                                              const float *__restrict__ B, int N,
                                              float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.f;
    for (long long base = warp * 32; base < n; base += nwarps * 32) {
        const int my = (base + lane < n) ? idx[base + lane] : 0;
#pragma unroll 1
        for (int j = 0; j < 32; j += U) {
            float4 t[U][V / 4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = __shfl_sync(0xffffffffu, my, j + u);
                const float4 *row = reinterpret_cast<const float4 *>(B + (long long)r * N) + lane * (V / 4);
#pragma unroll
                for (int q = 0; q < V / 4; ++q) t[u][q] = __ldg(row + q);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < V / 4; ++q) {
                    acc[4 * q] += t[u][q].x; acc[4 * q + 1] += t[u][q].y;
                    acc[4 * q + 2] += t[u][q].z; acc[4 * q + 3] += t[u][q].w;
                }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) s += acc[v];
    if (s == 123.456f) out[0] = s;  // keep the loads alive
}

template <int U, int V>
static void run(const int *idx, long long n, const float *B, int rows, int N, float *out, int sms,
                const char *tag) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather<U, V>, 256, 0);
    const int grid = sms * occ;
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        gather<U, V><<<grid, 256>>>(idx, n, B, N, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    const double bytes = (double)n * N * 4;
    printf("%-8s table_rows=%-8d table_MB=%-7.1f N=%-3d U=%d occ=%d  %.3f ms  gather %.0f GB/s\n", tag,
           rows, rows * (double)N * 4 / 1e6, N, U, occ, best, bytes / best / 1e6);
}

int main(int argc, char **argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc == 4) {  // <col_idx int32 file> <table rows> <N>: gather-only over a real col_idx
        FILE *f = fopen(argv[1], "rb");
        fseek(f, 0, SEEK_END);
        const long long m = ftell(f) / 4;
        fseek(f, 0, SEEK_SET);
        int *h = (int *)malloc(m * 4);
        if (fread(h, 4, m, f) != (size_t)m) return 1;
        fclose(f);
        const int rows = atoi(argv[2]), N = atoi(argv[3]);
        int *idx; float *B, *out;
        cudaMalloc(&idx, m * 4);
        cudaMalloc(&B, (size_t)rows * N * 4);
        cudaMalloc(&out, 64);
        cudaMemset(B, 0, (size_t)rows * N * 4);
        cudaMemcpy(idx, h, m * 4, cudaMemcpyHostToDevice);
        if (N == 128) {
            run<2, 4>(idx, m, B, rows, N, out, sms, "file");
            run<4, 4>(idx, m, B, rows, N, out, sms, "file");
            run<8, 4>(idx, m, B, rows, N, out, sms, "file");
        }
        printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
        return 0;
    }
    const long long n = 16 * 1024 * 1024;  // positions (config 2 has 16.09M)
    int *idx; float *B, *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&B, 1ull << 31);
    cudaMalloc(&out, 64);
    cudaMemset(B, 0, 1ull << 31);
    for (int skew = 0; skew < 2; ++skew) {
        const char *tag = skew ? "skewed" : "uniform";
        for (int rows : {16384, 131072, 1048576, 4194304}) {
            make_idx<<<1024, 256>>>(idx, n, rows, skew);
            run<2, 4>(idx, n, B, rows, 128, out, sms, tag);
            run<4, 4>(idx, n, B, rows, 128, out, sms, tag);
            run<8, 4>(idx, n, B, rows, 128, out, sms, tag);
        }
        for (int rows : {131072, 1048576}) {
            make_idx<<<1024, 256>>>(idx, n, rows, skew);
            run<4, 8>(idx, n, B, rows, 256, out, sms, tag);
            run<8, 8>(idx, n, B, rows, 256, out, sms, tag);
        }
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
