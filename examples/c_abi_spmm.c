/*
 * The drop-in boundary from plain C: build a Sgap kernel for a point, run it
 * through sgap_plan + sgap_run on the device and check against a host double-precision
 * product.  No Python, no torch -- only libsgap.so, sgap.h and the CUDA
 * runtime.  Exit status 0 on success.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_spmm.c \
 *       -L paper_2209_02882_b200 -lsgap -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2209_02882_b200 -o c_abi_spmm && ./c_abi_spmm
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "sgap.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)
#define SG(x) do { int s_ = (x); if (s_ != SGAP_OK) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, sgap_status_string(s_)); return 1; } } while (0)

static unsigned lcg = 12345u;
static float urand(void) { lcg = lcg * 1664525u + 1013904223u; return (lcg >> 8) / 8388608.0f - 1.0f; }

static int run_point(const char *label, sgap_point_t pt, int M, int K, int N, int p) {
    /* a random CSR with a few long rows */
    int *rp = malloc((M + 1) * sizeof(int));
    rp[0] = 0;
    for (int i = 0; i < M; ++i) rp[i + 1] = rp[i] + ((i % 97) == 0 ? 300 : (int)((urand() + 1.0f) * 8.0f));
    const int nnz = rp[M];
    int *ci = malloc(nnz * sizeof(int));
    float *av = malloc(nnz * sizeof(float)), *hb = malloc((size_t)K * N * sizeof(float));
    for (int i = 0; i < M; ++i) {  /* strictly increasing columns per row */
        const int len = rp[i + 1] - rp[i];
        int c = (int)((lcg = lcg * 1664525u + 1013904223u) % (unsigned)(K - len + 1));
        for (int q = rp[i]; q < rp[i + 1]; ++q) { ci[q] = c; c += 1 + (K - c > 2 * (rp[i + 1] - q)); }
        for (int q = rp[i]; q < rp[i + 1]; ++q) av[q] = urand();
    }
    for (size_t x = 0; x < (size_t)K * N; ++x) hb[x] = urand();

    sgap_kernel_t k;
    int32_t rule = 0;
    SG(sgap_build_kernel(&pt, N, p, M, nnz, &k, &rule));
    int *d_rp, *d_ci;
    float *d_av, *d_b, *d_c;
    CK(cudaMalloc((void **)&d_rp, (M + 1) * sizeof(int)));
    CK(cudaMalloc((void **)&d_ci, nnz * sizeof(int)));
    CK(cudaMalloc((void **)&d_av, nnz * sizeof(float)));
    CK(cudaMalloc((void **)&d_b, (size_t)K * N * sizeof(float)));
    CK(cudaMalloc((void **)&d_c, (size_t)M * N * sizeof(float)));
    CK(cudaMemcpy(d_rp, rp, (M + 1) * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci, nnz * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_av, av, nnz * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, hb, (size_t)K * N * sizeof(float), cudaMemcpyHostToDevice));

    /* plan (block starts, row ids, float64 long-row table -- all on the
       device, CSR invariants validated first) + run */
    sgap_csr_t a = {M, K, nnz, d_rp, d_ci, d_av};
    size_t ws_bytes = 0;
    void *d_ws;
    sgap_plan_t plan;
    SG(sgap_plan_workspace_bytes(&k, &a, SGAP_F32, SGAP_PLAN_VALIDATE, &ws_bytes));
    CK(cudaMalloc(&d_ws, ws_bytes));
    SG(sgap_plan(&k, &a, SGAP_F32, SGAP_PLAN_VALIDATE, d_ws, ws_bytes, &plan, NULL));
    unsigned long long *d_wb;
    CK(cudaMalloc((void **)&d_wb, sizeof(unsigned long long)));
    CK(cudaMemset(d_wb, 0, sizeof(unsigned long long)));
    SG(sgap_run(&plan, &a, d_b, d_c, 0, d_wb, NULL));
    CK(cudaDeviceSynchronize());

    float *hc = malloc((size_t)M * N * sizeof(float));
    unsigned long long wb = 0;
    CK(cudaMemcpy(hc, d_c, (size_t)M * N * sizeof(float), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&wb, d_wb, sizeof(wb), cudaMemcpyDeviceToHost));
    double worst = 0.0;  /* runner._max_rel_error: max |got - want| / (|want| + 1) */
    for (int i = 0; i < M; ++i)
        for (int x = 0; x < N; ++x) {
            double want = 0.0;
            for (int q = rp[i]; q < rp[i + 1]; ++q) want += (double)av[q] * (double)hb[(size_t)ci[q] * N + x];
            const double e = fabs((double)hc[(size_t)i * N + x] - want) / (fabs(want) + 1.0);
            if (e > worst) worst = e;
        }
    printf("%-22s family=%d grid=%lld block=%lld nnz=%d writebacks=%llu max_rel_error=%.3e\n", label,
           k.family, (long long)k.grid_size, (long long)k.block_size, nnz, wb, worst);
    cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_av); cudaFree(d_b); cudaFree(d_c); cudaFree(d_wb);
    cudaFree(d_ws);
    free(rp); free(ci); free(av); free(hb); free(hc);
    return worst <= 1e-5 ? 0 : 1;
}

/* SimulationFault (sim.py:279-287) / CsrMatrix invariants (matrices.py:58-75):
   an out-of-range column and a decreasing row_ptr are reported by the
   validating planner, not read out of bounds. */
static int fault_case(void) {
    const int rp_bad_col[4] = {0, 2, 3, 4}, ci_bad_col[4] = {0, 5, 1, 2}; /* K = 4: col 5 */
    const int rp_bad_rp[4] = {0, 3, 2, 4}, ci_ok[4] = {0, 1, 2, 3};
    const float av[4] = {1, 2, 3, 4};
    const sgap_point_t pt = {SGAP_KIND_ROW, SGAP_AMT_ONE, 0, SGAP_AMT_ONE, 0, 1};
    int *d_rp, *d_ci;
    float *d_av;
    void *d_ws;
    CK(cudaMalloc((void **)&d_rp, 4 * sizeof(int)));
    CK(cudaMalloc((void **)&d_ci, 4 * sizeof(int)));
    CK(cudaMalloc((void **)&d_av, 4 * sizeof(float)));
    CK(cudaMemcpy(d_av, av, sizeof(av), cudaMemcpyHostToDevice));
    sgap_kernel_t k;
    SG(sgap_build_kernel(&pt, 32, 256, 3, 4, &k, NULL));
    sgap_csr_t a = {3, 4, 4, d_rp, d_ci, d_av};
    size_t ws = 0;
    SG(sgap_plan_workspace_bytes(&k, &a, SGAP_F32, SGAP_PLAN_VALIDATE, &ws));
    CK(cudaMalloc(&d_ws, ws));
    sgap_plan_t plan;
    int64_t pos = 0;
    CK(cudaMemcpy(d_rp, rp_bad_col, sizeof(rp_bad_col), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci_bad_col, sizeof(ci_bad_col), cudaMemcpyHostToDevice));
    const int s1 = sgap_plan(&k, &a, SGAP_F32, SGAP_PLAN_VALIDATE, d_ws, ws, &plan, NULL);
    const int v1 = sgap_validate_csr(&a, d_ws, &pos, NULL);
    const int64_t pos1 = pos;
    CK(cudaMemcpy(d_rp, rp_bad_rp, sizeof(rp_bad_rp), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci_ok, sizeof(ci_ok), cudaMemcpyHostToDevice));
    const int v2 = sgap_validate_csr(&a, d_ws, &pos, NULL);
    const int64_t pos2 = pos;
    cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_av); cudaFree(d_ws);
    const int ok = s1 == SGAP_ERR_FAULT && v1 == SGAP_ERR_FAULT && pos1 == 1 &&
                   v2 == SGAP_ERR_FAULT && pos2 == -2;
    printf("%-22s plan=%s col fault at %lld, row_ptr fault at %lld\n", "fault detection",
           sgap_status_string(s1), (long long)pos1, (long long)pos2);
    return ok ? 0 : 1;
}

int main(void) {
    if (sgap_abi_version() != SGAP_ABI_VERSION) { fprintf(stderr, "ABI mismatch\n"); return 1; }
    /* nnz:256,col:4,r:1 (EB+SR), nnz:1,col:4,r:8 (EB+segment), row:4,col:4,r:1 (RB+SR),
       row:1/8,col:4,r:8 (RB+PR) -- sgap_point_t = {kind, data amount, g, col amount, c, r} */
    const sgap_point_t pts[4] = {
        {SGAP_KIND_NNZ, SGAP_AMT_MULTIPLE, 256, SGAP_AMT_MULTIPLE, 4, 1},
        {SGAP_KIND_NNZ, SGAP_AMT_ONE, 0, SGAP_AMT_MULTIPLE, 4, 8},
        {SGAP_KIND_ROW, SGAP_AMT_MULTIPLE, 4, SGAP_AMT_MULTIPLE, 4, 1},
        {SGAP_KIND_ROW, SGAP_AMT_RECIPROCAL, 8, SGAP_AMT_MULTIPLE, 4, 8},
    };
    const char *names[4] = {"nnz:256,col:4,r:1", "nnz:1,col:4,r:8", "row:4,col:4,r:1",
                            "row:1/8,col:4,r:8"};
    int bad = 0;
    for (int i = 0; i < 4; ++i) bad |= run_point(names[i], pts[i], 3000, 2000, 64, 256);
    bad |= fault_case();
    printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
