// Probe: tcgen05.mma kind::tf32, both operands in shared memory (SS), M = 128,
// small N -- the shape of a densified 128 x 128 CSB sub-tile times a 16-wide
// X panel. Checks the descriptor layouts the SpMM uses (A K-major for
// Y_I += A X_J, the same bytes read MN-major for Y_J += A^T X_I, B MN-major)
// against a CPU product, and times cycles per 128 x 128 tile.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/umma_probe tools/umma_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

constexpr int T = 128;           // tile edge
constexpr int NB = 16;           // panel width
constexpr int SJ = 128;          // A: bytes between 4-column groups
constexpr int SI = 32 * 128;     // A: bytes between 8-row groups
constexpr int BK = 128;          // B (K-major): bytes between 4-row (k) chunks
constexpr int BV = 32 * 128;     // B (K-major): bytes between 8-column (v) groups

#ifdef SW128
// K-major SWIZZLE_128B: atoms of 8 rows x 128 B (32 tf32 along K), 16-byte chunk ^= row % 8;
// row groups at 1 KB (SBO), K atoms at 16 KB
__host__ __device__ inline int a_off(int i, int j) {
    return (j >> 5) * 16384 + (i >> 3) * 1024 + (i & 7) * 128 + ((((j & 31) >> 2) ^ (i & 7)) << 4) + (j & 3) * 4;
}
#else
__host__ __device__ inline int a_off(int i, int j) { return (i >> 3) * SI + (j >> 2) * SJ + (i & 7) * 16 + (j & 3) * 4; }
#endif
// B = X (K = rows k, N = columns v), K-major interleave: core = 8 v x 4 k (128 B)
#ifdef SW128
__host__ __device__ inline int b_off(int k, int v) {
    return (k >> 5) * 4096 + (v >> 3) * 1024 + (v & 7) * 128 + ((((k & 31) >> 2) ^ (v & 7)) << 4) + (k & 3) * 4;
}
#else
__host__ __device__ inline int b_off(int k, int v) { return (v >> 3) * BV + (k >> 2) * BK + (v & 7) * 16 + (k & 3) * 4; }
#endif

__device__ inline std::uint32_t smem_u32(const void* p) { return static_cast<std::uint32_t>(__cvta_generic_to_shared(p)); }

__device__ inline std::uint64_t sdesc(std::uint32_t addr, std::uint32_t lbo, std::uint32_t sbo) {
    std::uint64_t d = 0;
#ifdef SW128
    d |= 2ull << 61;
#endif
    d |= static_cast<std::uint64_t>((addr >> 4) & 0x3fff);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3fff) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3fff) << 32;
    d |= 1ull << 46;  // version (sm100)
    return d;         // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__host__ __device__ constexpr std::uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<std::uint32_t>(a_mn) << 15) |
           (static_cast<std::uint32_t>(b_mn) << 16) | (static_cast<std::uint32_t>(N >> 3) << 17) |
           (static_cast<std::uint32_t>(M >> 4) << 24);
}

__device__ inline void mma_tf32(std::uint32_t dt, std::uint64_t ad, std::uint64_t bd, std::uint32_t id, int acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
        "l"(ad), "l"(bd), "r"(id), "r"(acc));
}

__device__ inline void mbar_init(std::uint64_t* b, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ inline void commit(std::uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ inline void mbar_wait(std::uint64_t* b, int phase) {
    asm volatile(
        "{\n .reg .pred q;\n W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W;\n}\n" ::"r"(
            smem_u32(b)),
        "r"(phase)
        : "memory");
}

template <int N>
__device__ inline void tld(std::uint32_t taddr, float* out) {
    static_assert(N == 16, "x16 only");
    std::uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) out[i] = __uint_as_float(r[i]);
}

// mode 0: pass R (A K-major, N=NR); 1: pass C (A MN-major); 2: both (+ N16 lo product each)
__global__ void __launch_bounds__(128, 1) k_probe(const float* gA, const float* gB, float* gDR, float* gDC, int reps,
                                                  int nr, long long* cyc, int lsu_load) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sA = sm;             // 64 KB
    unsigned char* sB = sm + 65536;     // 16 KB (N = 32, K-major)
    unsigned char* sAT = sm + 65536 + 16384;  // 64 KB: A^T for pass C (MN-major tf32 needs SW128_32B, which K-major cannot share)
    __shared__ std::uint64_t bar;
    __shared__ std::uint32_t tbase;
    const int tid = threadIdx.x;
    for (int e = tid; e < T * T; e += blockDim.x) {
        const int i = e / T, j = e % T;
        *reinterpret_cast<float*>(sA + a_off(i, j)) = gA[e];
        *reinterpret_cast<float*>(sAT + a_off(j, i)) = gA[e];
    }
    for (int e = tid; e < T * 32; e += blockDim.x) {
        const int k = e / 32, v = e % 32;
        *reinterpret_cast<float*>(sB + b_off(k, v)) = gB[e];
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const std::uint32_t tb = tbase;
    const std::uint32_t aA = smem_u32(sA), aB = smem_u32(sB), aAT = smem_u32(sAT);
    long long t0 = clock64();
    float sink = 0.f;
    if (tid == 0) {
        const std::uint32_t idR = idesc_tf32(128, nr, 0, 0), idR16 = idesc_tf32(128, 16, 0, 0);
        const std::uint32_t idC = idR, idC16 = idR16;
        for (int r = 0; r < reps; ++r) {
          for (int in = 0; in < (lsu_load >> 2) + 1; ++in) {
            for (int s = 0; s < 16; ++s) {  // pass R: D_R[i, v] += sum_j A[i, j] B[j, v]
#ifdef SW128
                const std::uint64_t ad = sdesc(aA + (s >> 2) * 16384 + (s & 3) * 32, 16, 1024);
                const std::uint64_t bd = sdesc(aB + (s >> 2) * 4096 + (s & 3) * 32, 16, 1024);
#else
                const std::uint64_t ad = sdesc(aA + s * 2 * SJ, SJ, SI);
                const std::uint64_t bd = sdesc(aB + s * 2 * BK, BK, BV);
#endif
                mma_tf32(tb + 0, ad, bd, idR, (r | s) != 0);
                if (lsu_load & 2) mma_tf32(tb + 0, ad, bd, idR16, 1);
            }
            for (int s = 0; s < 16; ++s) {  // pass C: D_C[j, v] += sum_i A[i, j] B[i, v]
#ifdef SW128
                const std::uint64_t ad = sdesc(aAT + (s >> 2) * 16384 + (s & 3) * 32, 16, 1024);
                const std::uint64_t bd = sdesc(aB + (s >> 2) * 4096 + (s & 3) * 32, 16, 1024);
#else
                const std::uint64_t ad = sdesc(aAT + s * 2 * SJ, SJ, SI);
                const std::uint64_t bd = sdesc(aB + s * 2 * BK, BK, BV);
#endif
                mma_tf32(tb + 32, ad, bd, idC, (r | s) != 0);
                if (lsu_load & 2) mma_tf32(tb + 32, ad, bd, idC16, 1);
            }
          }
            commit(&bar);
            mbar_wait(&bar, r & 1);
        }
    } else if (lsu_load & 1) {  // concurrent LDS traffic from the other warps (crossbar contention)
        for (int r = 0; r < reps * 64; ++r)
            sink += *reinterpret_cast<volatile float*>(sA + ((tid * 16 + r * 128) & 65535));
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // read back: warp w -> lanes 32w..32w+31
    const int w = tid >> 5, l = tid & 31, row = 32 * w + l;
    float v[16];
    for (int c = 0; c < 32; c += 16) {
        tld<16>(tb + ((32 * w) << 16) + c, v);
        for (int i = 0; i < 16; ++i) gDR[(blockIdx.x * T + row) * 32 + c + i] = v[i];
        tld<16>(tb + ((32 * w) << 16) + 32 + c, v);
        for (int i = 0; i < 16; ++i) gDC[(blockIdx.x * T + row) * 32 + c + i] = v[i] + sink * 0.f;
    }
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(128));
}

static float tf32(float x) {
    std::uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    memcpy(&x, &u, 4);
    return x;
}

int main(int argc, char** argv) {
    const int blocks = argc > 1 ? atoi(argv[1]) : 148;
    const int reps = 200;
    std::vector<float> A(T * T), B(T * 32);
    srand(1);
    for (auto& a : A) a = (rand() % 10 == 0) ? (rand() / (float)RAND_MAX * 2 - 1) : 0.f;  // 10% fill
    for (auto& b : B) b = rand() / (float)RAND_MAX * 2 - 1;
    float *dA, *dB, *dR, *dC;
    long long* dc;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dR, blocks * T * 32 * 4));
    CK(cudaMalloc(&dC, blocks * T * 32 * 4));
    CK(cudaMalloc(&dc, blocks * 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const int smem = 65536 + 16384 + 65536;
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int mode : {0, 2, 28, 30, 29})
        for (int nr : {16, 32}) {
            const int rr = 1;
            k_probe<<<blocks, 128, smem>>>(dA, dB, dR, dC, rr, nr, dc, mode);
            CK(cudaDeviceSynchronize());
            // check one rep
            std::vector<float> R(T * 32), Cc(T * 32);
            CK(cudaMemcpy(R.data(), dR, R.size() * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(Cc.data(), dC, Cc.size() * 4, cudaMemcpyDeviceToHost));
            double er = 0, ec = 0, nrm = 0;
            for (int i = 0; i < T; ++i)
                for (int v = 0; v < nr; ++v) {
                    double sr = 0, sc = 0;
                    for (int j = 0; j < T; ++j) {
                        sr += (double)tf32(A[i * T + j]) * tf32(B[j * 32 + v]);
                        sc += (double)tf32(A[j * T + i]) * tf32(B[j * 32 + v]);
                    }
                    if ((mode & 2) && v < 16) {
                        sr *= 2;
                        sc *= 2;
                    }
                    er = fmax(er, fabs(sr - R[i * 32 + v]));
                    ec = fmax(ec, fabs(sc - Cc[i * 32 + v]));
                    nrm = fmax(nrm, fabs(sr));
                }
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_probe<<<blocks, 128, smem>>>(dA, dB, dR, dC, reps, nr, dc, mode);
            cudaEventRecord(e1);
            CK(cudaDeviceSynchronize());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<long long> c(blocks);
            CK(cudaMemcpy(c.data(), dc, blocks * 8, cudaMemcpyDeviceToHost));
            long long mx = 0;
            for (auto x : c) mx = x > mx ? x : mx;
            if (mode == 0 && nr == 16) {
                for (int i = 0; i < 3; ++i) {
                    double sr = 0;
                    for (int j = 0; j < T; ++j) sr += (double)tf32(A[i * T + j]) * tf32(B[j * 32 + 0]);
                    printf("row %d: got R %.5f %.5f C %.5f want R %.5f\n", i, R[i * 32], R[i * 32 + 1], Cc[i * 32], sr);
                }
            }
            printf("mode %d (lsu %d, lo16 %d) N=%d: maxerr R %.3g C %.3g (|D| %.3g); %.1f cyc per tile (both passes), "
                   "kernel %.3f ms for %d tiles/CTA\n",
                   mode, mode & 1, (mode >> 1) & 1, nr, er, ec, nrm, (double)mx / reps / ((mode >> 2) + 1), ms, reps);
        }
    return 0;
}
