// cuSOLVER dense symmetric eigensolvers at the Rayleigh-Ritz size (3 nb = 48):
// syevd (divide & conquer) vs syevj (Jacobi). nvcc -O3 tools/syev_probe.cu -lcusolver -o tools/bin/syev_probe
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include <cusolverDn.h>
int main() {
    const int n = 48;
    std::vector<double> a(n * n);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> u(-1, 1);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) a[i * n + j] = a[j * n + i] = u(rng) + (i == j ? 10.0 * i : 0.0);
    double *dA, *dW, *dM;
    int* info;
    cudaMalloc(&dA, n * n * 8); cudaMalloc(&dM, n * n * 8); cudaMalloc(&dW, n * 8); cudaMalloc(&info, 4);
    cudaMemcpy(dA, a.data(), n * n * 8, cudaMemcpyHostToDevice);
    cusolverDnHandle_t h; cusolverDnCreate(&h);
    cudaStream_t s; cudaStreamCreate(&s); cusolverDnSetStream(h, s);
    int lw = 0;
    cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dM, n, dW, &lw);
    double* work; cudaMalloc(&work, (lw + 1) * 8);
    syevjInfo_t params; cusolverDnCreateSyevjInfo(&params);
    cusolverDnXsyevjSetTolerance(params, 1e-15); cusolverDnXsyevjSetMaxSweeps(params, 20);
    int lwj = 0;
    cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dM, n, dW, &lwj, params);
    double* workj; cudaMalloc(&workj, (lwj + 1) * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemcpyAsync(dM, dA, n * n * 8, cudaMemcpyDeviceToDevice, s);
            cudaEventRecord(e0, s);
            for (int it = 0; it < 20; ++it) {
                if (mode == 0) cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dM, n, dW, work, lw, info);
                else cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dM, n, dW, workj, lwj, info, params);
            }
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("%s: %.1f us per call\n", mode == 0 ? "syevd" : "syevj", ms * 1000 / 20);
        }
    }
    return 0;
}
