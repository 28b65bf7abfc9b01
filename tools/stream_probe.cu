// Probe: streaming read throughput of a persistent cp.async ring (the panel
// kernels' load path) versus stages / stage size / CTAs per SM, and of plain
// vectorised loads. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/stream_probe.cu -o /tmp/stream_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(void* d, const void* s) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d)), "l"(s) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int S, int WORK = 0>
__global__ void k_ring(const double* __restrict__ x, long n, int R, double* out) {
    extern __shared__ __align__(16) double sb[];
    const int nb = 16, rs = 18;
    long nch_all = (n + R - 1) / R;
    long c0 = nch_all * blockIdx.x / gridDim.x, c1 = nch_all * (blockIdx.x + 1) / gridDim.x;
    int nch = (int)(c1 - c0);
    const int pr = 8, c = threadIdx.x % pr, rstep = blockDim.x / pr;
    auto issue = [&](int k) {
        if (k < nch) {
            long r0 = (c0 + k) * R;
            int rows = (int)min((long)R, n - r0);
            double* t = sb + (k % S) * (R * rs + 2) + 2 * c;
            const double* g = x + r0 * nb + 2 * c;
            for (int r = threadIdx.x / pr; r < rows; r += rstep) cp16(t + r * rs, g + (long)r * nb);
        }
        commit();
    };
    for (int k = 0; k < S - 1; ++k) issue(k);
    double acc = 0;
    for (int k = 0; k < nch; ++k) {
        issue(k + S - 1);
        waitg<S - 1>();
        __syncthreads();
        const double* t = sb + (k % S) * (R * rs + 2);
        if (WORK == 0) {
            for (int e = threadIdx.x; e < R * 8; e += blockDim.x) acc += t[(e / 8) * rs + (e % 8) * 2];
        } else {  // gram-like: thread = (task of 4, row group); 8x4 block per row
            const int task = threadIdx.x % 8, grp = threadIdx.x / 8, G = blockDim.x / 8;
            double a2[32];
            for (int e = 0; e < 32; ++e) a2[e] = 0;
            const int i0 = (task / 4) * 8, j0 = (task % 4) * 4;
            for (int r = grp; r < R; r += G) {
                double a[8], b[4];
                for (int q = 0; q < 4; ++q) { double2 v = *(const double2*)(t + r * rs + i0 + 2 * q); a[2*q] = v.x; a[2*q+1] = v.y; }
                for (int q = 0; q < 2; ++q) { double2 v = *(const double2*)(t + r * rs + j0 + 2 * q); b[2*q] = v.x; b[2*q+1] = v.y; }
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int ii = 0; ii < 8; ++ii) a2[jj * 8 + ii] = fma(a[ii], b[jj], a2[jj * 8 + ii]);
            }
            for (int e = 0; e < 32; ++e) acc += a2[e];
        }
        __syncthreads();
    }
    waitg<0>();
    if (acc == 12345.678) out[0] = acc;
}

__global__ void k_plain(const double2* __restrict__ x, long n2, double* out) {
    double acc = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
        double2 v = __ldg(x + i);
        acc += v.x + v.y;
    }
    if (acc == 12345.678) out[0] = acc;
}

template <int S, int WORK = 0>
void run(const double* x, long n, int R, int ctas_per_sm, double* out, int sms, int tpb = 256) {
    size_t sm = (size_t)S * (R * 18 + 2) * 8;
    cudaFuncSetAttribute(k_ring<S, WORK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int grid = sms * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_ring<S, WORK><<<grid, tpb, sm>>>(x, n, R, out);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) k_ring<S, WORK><<<grid, tpb, sm>>>(x, n, R, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ring<S, WORK>, tpb, sm);
    printf("ring W=%d tpb=%d S=%d R=%d stage=%.1fKB ctas/sm=%d (occ %d): %.0f GB/s  err=%s\n", WORK, tpb, S, R, (R * 18 + 2) * 8 / 1024.0,
           ctas_per_sm, occ, n * 128.0 * 5 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main1() {
    long n = 2900000;
    double *x, *out;
    cudaMalloc(&x, n * 128);
    cudaMalloc(&out, 8);
    cudaMemset(x, 0, n * 128);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int g : {sms * 2, sms * 4, sms * 8, sms * 16}) {
            k_plain<<<g, 256>>>((const double2*)x, n * 8, out);
            cudaEventRecord(a);
            for (int i = 0; i < 5; ++i) k_plain<<<g, 256>>>((const double2*)x, n * 8, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("plain grid=%d: %.0f GB/s\n", g, n * 128.0 * 5 / (ms * 1e-3) / 1e9);
        }
    }
    run<3>(x, n, 256, 1, out, sms);
    run<4, 1>(x, n, 256, 1, out, sms, 256);
    run<4, 1>(x, n, 256, 1, out, sms, 512);
    run<3, 1>(x, n, 256, 2, out, sms, 256);
    run<4, 1>(x, n, 128, 2, out, sms, 256);
    run<4, 1>(x, n, 64, 4, out, sms, 256);
    run<3>(x, n, 256, 2, out, sms);
    run<4>(x, n, 256, 1, out, sms);
    run<4>(x, n, 128, 2, out, sms);
    run<6>(x, n, 128, 1, out, sms);
    run<8>(x, n, 96, 1, out, sms);
    run<8>(x, n, 64, 2, out, sms);
    run<4>(x, n, 64, 4, out, sms);
    run<3>(x, n, 64, 6, out, sms);
    run<12>(x, n, 64, 1, out, sms);
    return 0;
}

// DFMA throughput probe
__global__ void k_dfma(double* out, int iters) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
    const double b = 1.0000001, c = 1e-12;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}
__global__ void k_ffma(float* out, int iters) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9f + i;
    const float b = 1.0000001f, c = 1e-12f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 1.2345f) out[0] = s;
}
int main2() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 4096;
    for (int tpb : {256, 512, 1024}) {
        int grid = sms * (2048 / tpb);
        k_dfma<<<grid, tpb>>>(out, iters);
        cudaEventRecord(a);
        k_dfma<<<grid, tpb>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 16 * iters * (double)grid * tpb;
        printf("dfma tpb=%d: %.1f TFLOP/s fp64\n", tpb, fl / (ms * 1e-3) / 1e12);
        k_ffma<<<grid, tpb>>>((float*)out, iters);
        cudaEventRecord(a);
        k_ffma<<<grid, tpb>>>((float*)out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("ffma tpb=%d: %.1f TFLOP/s fp32\n", tpb, fl / (ms * 1e-3) / 1e12);
    }
    return 0;
}
int main3() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 4096;
    for (int wps : {4, 8, 16, 32, 64}) {  // warps per SM
        int tpb = 128, grid = sms * wps / 4;
        k_dfma<<<grid, tpb>>>(out, iters);
        cudaEventRecord(a);
        k_dfma<<<grid, tpb>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 16 * iters * (double)grid * tpb;
        printf("dfma warps/SM=%d: %.1f TFLOP/s fp64 (16 indep. chains per thread)\n", wps, fl / (ms * 1e-3) / 1e12);
    }
    return 0;
}
__global__ void k_dmma(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2] = {};
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    if (s == 1.2345) out[0] = s;
}
int main4() {
    double* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 4096;
    for (int wps : {4, 8, 16, 32}) {
        int tpb = 128, grid = sms * wps / 4;
        k_dmma<<<grid, tpb>>>(out, iters);
        cudaEventRecord(a);
        k_dmma<<<grid, tpb>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 256 * 8 * iters * (double)grid * (tpb / 32);
        printf("dmma m8n8k4 warps/SM=%d: %.1f TFLOP/s fp64  err=%s\n", wps, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
int main5() {  // cold data: rotate over 4 distinct 371 MB buffers (L2 cannot help)
    long n = 2900000;
    double *x[4], *out;
    for (auto& p : x) { cudaMalloc(&p, n * 128); cudaMemset(p, 1, n * 128); }
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int g : {sms * 4, sms * 8, sms * 16}) {
        k_plain<<<g, 256>>>((const double2*)x[0], n * 8, out);
        cudaEventRecord(a);
        for (int i = 0; i < 8; ++i) k_plain<<<g, 256>>>((const double2*)x[i % 4], n * 8, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cold plain grid=%d: %.0f GB/s\n", g, n * 128.0 * 8 / (ms * 1e-3) / 1e9);
    }
    auto ring = [&](auto kern, int S, int R, int cps, int tpb, const char* name) {
        size_t sm = (size_t)S * (R * 18 + 2) * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int grid = sms * cps;
        kern<<<grid, tpb, sm>>>(x[0], n, R, out);
        cudaEventRecord(a);
        for (int i = 0; i < 8; ++i) kern<<<grid, tpb, sm>>>(x[i % 4], n, R, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cold %s S=%d R=%d ctas/sm=%d tpb=%d: %.0f GB/s %s\n", name, S, R, cps, tpb, n * 128.0 * 8 / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    ring(k_ring<4, 0>, 4, 256, 1, 256, "ring");
    ring(k_ring<6, 0>, 6, 128, 1, 256, "ring");
    ring(k_ring<4, 0>, 4, 128, 2, 256, "ring");
    ring(k_ring<8, 0>, 8, 64, 2, 256, "ring");
    ring(k_ring<4, 0>, 4, 64, 4, 256, "ring");
    ring(k_ring<4, 1>, 4, 256, 1, 256, "ring+gram");
    ring(k_ring<4, 1>, 4, 128, 2, 256, "ring+gram");
    ring(k_ring<4, 1>, 4, 64, 4, 256, "ring+gram");
    ring(k_ring<3, 1>, 3, 64, 6, 256, "ring+gram");
    ring(k_ring<4, 1>, 4, 256, 1, 512, "ring+gram");
    ring(k_ring<4, 1>, 4, 256, 1, 1024, "ring+gram");
    ring(k_ring<4, 1>, 4, 128, 2, 1024, "ring+gram");
    return 0;
}
int main() { main5(); return 0; }
