// Probe: TMA tile::gather4 of 4 B rows (fp32, N columns) into shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -o probe tma_gather4_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap tm, const int *rows, float *out, int n) {
    extern __shared__ __align__(1024) float s[];
    __shared__ unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(s);
    const unsigned bb = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(4 * n * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sb),
            "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(bb)
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W_%=;\n}" ::"r"(bb)
        : "memory");
    for (int i = threadIdx.x; i < 4 * n; i += blockDim.x) out[i] = s[i];
}

int main() {
    const int K = 1000, N = 128;
    std::vector<float> h(K * N);
    for (int i = 0; i < K * N; ++i) h[i] = (float)i;
    float *dB, *dOut;
    int *dRows;
    cudaMalloc(&dB, K * N * 4);
    cudaMalloc(&dOut, 4 * N * 4);
    cudaMalloc(&dRows, 16);
    cudaMemcpy(dB, h.data(), K * N * 4, cudaMemcpyHostToDevice);
    int rows[4] = {7, 999, 0, 512};
    cudaMemcpy(dRows, rows, 16, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no entry point\n"); return 1; }
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)K};
    cuuint64_t gstr[1] = {(cuuint64_t)N * 4};
    cuuint32_t box[2] = {(cuuint32_t)N, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, gdim, gstr, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    k<<<1, 128, 4 * N * 4>>>(tm, dRows, dOut, N);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> o(4 * N);
    cudaMemcpy(o.data(), dOut, 4 * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < 4; ++j)
        for (int c = 0; c < N; ++c)
            if (o[j * N + c] != h[rows[j] * N + c]) ++bad;
    printf("mismatches: %d  sample %f %f %f\n", bad, o[0], o[N], o[3 * N + 5]);
    return 0;
}
