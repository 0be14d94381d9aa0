/*
 * The drop-in boundary from plain C: build a Sgap kernel for a point, run it
 * through sgap_run on the device and check against a host double-precision
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
    int *d_rp, *d_ci, *d_starts = NULL, *d_rowid = NULL, *d_long_rows = NULL, *d_long_count = NULL,
        *d_slot = NULL, *d_exact = NULL;
    float *d_av, *d_b, *d_c;
    double *d_long_acc = NULL;
    CK(cudaMalloc((void **)&d_rp, (M + 1) * sizeof(int)));
    CK(cudaMalloc((void **)&d_ci, nnz * sizeof(int)));
    CK(cudaMalloc((void **)&d_av, nnz * sizeof(float)));
    CK(cudaMalloc((void **)&d_b, (size_t)K * N * sizeof(float)));
    CK(cudaMalloc((void **)&d_c, (size_t)M * N * sizeof(float)));
    CK(cudaMemcpy(d_rp, rp, (M + 1) * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, ci, nnz * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_av, av, nnz * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_b, hb, (size_t)K * N * sizeof(float), cudaMemcpyHostToDevice));

    sgap_aux_t aux = {0};
    const int eb = k.family == SGAP_NNZ_ONE || k.family == SGAP_NNZ_MULTIPLE;
    if (eb) {  /* block starts (LoweredKernel.block_starts), row ids, long-row table */
        CK(cudaMalloc((void **)&d_starts, (k.grid_size + 1) * sizeof(int)));
        SG(sgap_block_starts(d_rp, M, k.chunk, k.grid_size, d_starts, NULL));
        const int64_t thr = sgap_long_row_threshold(&k, SGAP_F32);
        CK(cudaMalloc((void **)&d_rowid, nnz * sizeof(int)));
        SG(sgap_row_ids(d_rp, M, nnz, thr, 0, d_rowid, NULL));
        aux.d_block_starts = d_starts;
        aux.d_rowid = d_rowid;
        aux.long_threshold = thr;
        if (thr >= 0) {
            const int64_t cap = sgap_long_row_capacity(nnz, thr, 0);
            CK(cudaMalloc((void **)&d_long_rows, cap * sizeof(int)));
            CK(cudaMalloc((void **)&d_long_count, sizeof(int)));
            CK(cudaMalloc((void **)&d_long_acc, cap * N * sizeof(double)));
            CK(cudaMalloc((void **)&d_slot, M * sizeof(int)));
            aux.d_long_rows = d_long_rows;
            aux.d_long_count = d_long_count;
            aux.d_long_acc = d_long_acc;
            aux.d_long_slot = d_slot;
            aux.long_capacity = cap;
            /* rows of the error-free pass: longer than max(thr, exact length) */
            const int64_t cut = thr > sgap_exact_row_length() ? thr : sgap_exact_row_length();
            int ne = 0, *ex = malloc(M * sizeof(int));
            for (int i = 0; i < M; ++i) if (rp[i + 1] - rp[i] > cut) ex[ne++] = i;
            if (ne && k.family == SGAP_NNZ_MULTIPLE) {
                CK(cudaMalloc((void **)&d_exact, ne * sizeof(int)));
                CK(cudaMemcpy(d_exact, ex, ne * sizeof(int), cudaMemcpyHostToDevice));
                aux.d_exact_rows = d_exact;
                aux.exact_count = ne;
                aux.has_exact_rows = 1;
            }
            free(ex);
            const size_t tmp_bytes = sgap_long_rows_tmp_bytes(M);
            void *d_tmp;
            CK(cudaMalloc(&d_tmp, tmp_bytes));
            SG(sgap_prepare_long_rows(d_rp, M, N, &aux, d_tmp, tmp_bytes, NULL));
            CK(cudaDeviceSynchronize());
            CK(cudaFree(d_tmp));
        }
    }
    sgap_csr_t a = {M, K, nnz, d_rp, d_ci, d_av};
    unsigned long long *d_wb;
    CK(cudaMalloc((void **)&d_wb, sizeof(unsigned long long)));
    CK(cudaMemset(d_wb, 0, sizeof(unsigned long long)));
    SG(sgap_run(&k, &a, d_b, d_c, SGAP_F32, 0, &aux, d_wb, NULL));
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
    cudaFree(d_starts); cudaFree(d_rowid); cudaFree(d_long_rows); cudaFree(d_long_count);
    cudaFree(d_long_acc); cudaFree(d_slot); cudaFree(d_exact);
    free(rp); free(ci); free(av); free(hb); free(hc);
    return worst <= 1e-5 ? 0 : 1;
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
    printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
