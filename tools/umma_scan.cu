// Cycles per tcgen05.mma kind::tf32 (SS, M = 128, K = 8, SWIZZLE_128B K-major)
// as a function of N, with the issue loop fully unrolled (descriptors
// precomputed), and the same for kind::f16 (bf16) -- the smem operand-read
// cost of small-N MMAs. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>
__device__ inline uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ inline uint64_t sd(uint32_t a) {
    return ((uint64_t)((a >> 4) & 0x3fff)) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int KIND>
__device__ inline void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, int acc) {
    if (KIND == 0)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
    else
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
template <int KIND, int N, int M, int NACC>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int reps) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int e = threadIdx.x; e < (16384 + 32768) / 4; e += 128) ((float*)sm)[e] = 0.f;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tbase)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tbase;
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint32_t id = (1u << 4) | ((KIND == 0 ? 2u : 1u) << 7) | ((KIND == 0 ? 2u : 1u) << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t a0 = su(sm), b0 = su(sm + 16384);
        uint64_t ad[4], bd[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) { ad[s] = sd(a0 + s * 32); bd[s] = sd(b0 + s * 32); }
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int s = 0; s < 4; ++s) mma<KIND>(tb + (s % NACC) * N, ad[s], bd[s], id, 1);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
        asm volatile("{\n .reg .pred q;\n W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], 0;\n @!q bra W;\n}\n" ::"r"(su(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}
template <int KIND, int N, int M, int NACC = 1>
void run() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 16384 + 32768;
    cudaFuncSetAttribute(k<KIND, N, M, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 2000;
    k<KIND, N, M, NACC><<<148, 128, smem>>>(d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto x : h) mx = x > mx ? x : mx;
    const double cpm = (double)mx / (reps * 4);
    const int kk = KIND == 0 ? 8 : 16;
    printf("%s NACC=%d M=%d N=%3d: %.1f cyc/MMA (%s)  A bytes/cyc %.0f  MAC/cyc %.0f\n", KIND == 0 ? "tf32" : "bf16", NACC, M, N, cpm,
           cudaGetErrorString(e), M * 32 / cpm, (double)M * N * kk / cpm);
    cudaFree(d);
}
int main() {
    run<0, 16, 128, 1>(); run<0, 16, 128, 2>(); run<0, 16, 128, 4>();
    run<0, 32, 128, 1>(); run<0, 32, 128, 2>(); run<0, 32, 128, 4>();
    run<0, 64, 128, 4>(); run<0, 16, 64, 4>();
    run<1, 16, 128, 4>(); run<1, 32, 128, 4>(); run<1, 48, 128, 4>();
}
