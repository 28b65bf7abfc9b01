// Device dense linear algebra for the LOBPCG iteration (see densela.cuh).
// Memory-bound fused panel kernels (Gram, row mixes, trsm, residual norms)
// and single-CTA kernels for the <= 3nb square projected problem; the
// symmetric eigen-decomposition itself is cuSOLVER syevd (no host fallback).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>

#include "densela.cuh"
#include "stream.cuh"

namespace be {
namespace dla {

namespace {

constexpr int kT = 256;

#define BE_CUSOLVER(call)                                                                   \
    do {                                                                                    \
        cusolverStatus_t s_ = (call);                                                       \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                  \
            ::be::fail(BE_ERR_CUSOLVER, std::string(#call) + " failed: " + std::to_string(s_)); \
    } while (0)

// ------------------------------------------------------------------- gram
struct GramDev {
    int npairs, nb, nblk, ncombo, nd;
    const double* panel[24];  // distinct panels
    int ia[12], ib[12];       // panel index of A_p / B_p
};

constexpr int kGramRows = 32;

// partial[blk][combo][16]: 4x4 register block of A_p^T B_p over this CTA's
// rows. cpb combos per CTA slice; the rg = 256 / cpb row groups of a CTA take
// interleaved rows of each staged chunk and are summed in smem at the end.
__global__ void __launch_bounds__(kT) k_gram_partial(GramDev g, std::int64_t n, double* __restrict__ partial, int cpb) {
    extern __shared__ double sp[];  // max(nd x kGramRows x nbp, rg x cpb x 16)
    const int nbp = g.nblk * 4;
    const int rg = kT / cpb;
    const int cl = threadIdx.x % cpb, grp = threadIdx.x / cpb;
    const int combo = blockIdx.y * cpb + cl;
    const bool active = grp < rg && combo < g.ncombo;
    int p = 0, bi = 0, bj = 0;
    if (active) {
        p = combo / (g.nblk * g.nblk);
        const int rem = combo % (g.nblk * g.nblk);
        bi = rem / g.nblk;
        bj = rem % g.nblk;
    }
    double acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0;
    const std::int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const std::int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    for (std::int64_t c0 = r0; c0 < r1; c0 += kGramRows) {
        const int rows = static_cast<int>(r1 - c0 < kGramRows ? r1 - c0 : kGramRows);
        __syncthreads();
        for (int d = 0; d < g.nd; ++d) {
            const double* src = g.panel[d] + c0 * g.nb;
            double* dst = sp + d * kGramRows * nbp;
            if (nbp == g.nb) {  // contiguous rows: straight vector copy
                const int tot = rows * g.nb / 2;
                for (int e = threadIdx.x; e < tot; e += kT)
                    reinterpret_cast<double2*>(dst)[e] = __ldg(reinterpret_cast<const double2*>(src) + e);
            } else {
                for (int e = threadIdx.x; e < kGramRows * nbp; e += kT) {
                    const int r = e / nbp, v = e % nbp;
                    dst[e] = (r < rows && v < g.nb) ? src[r * g.nb + v] : 0.0;
                }
            }
        }
        __syncthreads();
        if (active) {
            const double* A = sp + g.ia[p] * kGramRows * nbp + bi * 4;
            const double* B = sp + g.ib[p] * kGramRows * nbp + bj * 4;
            for (int r = grp; r < rows; r += rg) {
                const double2 a01 = *reinterpret_cast<const double2*>(A + r * nbp);
                const double2 a23 = *reinterpret_cast<const double2*>(A + r * nbp + 2);
                const double2 b01 = *reinterpret_cast<const double2*>(B + r * nbp);
                const double2 b23 = *reinterpret_cast<const double2*>(B + r * nbp + 2);
                const double a0 = a01.x, a1 = a01.y, a2 = a23.x, a3 = a23.y;
                const double b0 = b01.x, b1 = b01.y, b2 = b23.x, b3 = b23.y;
                acc[0] += a0 * b0; acc[1] += a1 * b0; acc[2] += a2 * b0; acc[3] += a3 * b0;
                acc[4] += a0 * b1; acc[5] += a1 * b1; acc[6] += a2 * b1; acc[7] += a3 * b1;
                acc[8] += a0 * b2; acc[9] += a1 * b2; acc[10] += a2 * b2; acc[11] += a3 * b2;
                acc[12] += a0 * b3; acc[13] += a1 * b3; acc[14] += a2 * b3; acc[15] += a3 * b3;
            }
        }
    }
    __syncthreads();
    if (grp < rg)
#pragma unroll
        for (int e = 0; e < 16; ++e) sp[(grp * cpb + cl) * 16 + e] = acc[e];
    __syncthreads();
    for (int e = threadIdx.x; e < cpb * 16; e += kT) {
        const int c = e / 16;
        if (blockIdx.y * cpb + c >= g.ncombo) continue;
        double s = 0.0;
        for (int q = 0; q < rg; ++q) s += sp[(q * cpb + c) * 16 + e % 16];
        partial[(static_cast<std::int64_t>(blockIdx.x) * g.ncombo + blockIdx.y * cpb + c) * 16 + e % 16] = s;
    }
}

struct GramOut {
    double* out[12];
    int sym[12];
};

// ---- streamed Gram (nb % 8 == 0): persistent CTAs, a kGS-stage ring of
// R-row chunks of the distinct panels filled by TMA bulk copies (one per row,
// into rows padded by 16 bytes: conflict-free shared-memory reads). Thread =
// (8 x 8 output block of one pair, row group): per row 64 B of A and 64 B of
// B from shared memory feed 64 FMAs. Row groups are summed in shared memory
// in a fixed order, CTAs by k_gram_reduce8 (deterministic).
constexpr int kGS = 3;  // pipeline stages of trsm (2 CTAs per SM, ~37 KB per stage)
constexpr int kGG = 4;  // pipeline stages of the Gram kernel (1 CTA per SM, ~40 KB per stage)

struct GramS {
    int R;         // rows per chunk
    int rs;        // padded row stride in doubles (nb + 2)
    int ps;        // doubles per panel slot (R * rs + 2: a 16-byte skew between panels)
    int ss;        // doubles per stage (nd * ps)
    int tasks;     // npairs * B
    int groups;    // row groups per CTA
    int bpr;       // 8-row blocks of an nb x nb output (nb / 8)
    int bpc;       // 4-column blocks (nb / 4)
};

// all threads fill one stage with 16-byte cp.async copies: `nsrc` panels x
// `rows` rows into rows padded to `rs` doubles (one commit group per stage)
__device__ __forceinline__ void cp16g(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(stream::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void fill_stage(double* st, const double* const* src, int nsrc, int ps, int rs, int nb,
                                           std::int64_t r0, int rows) {
    const int pr = nb / 2;  // 16-byte pieces per row
    const int c = threadIdx.x % pr, rstep = blockDim.x / pr;
    if (static_cast<int>(threadIdx.x) >= rstep * pr) return;  // pr need not divide the block: no duplicate rows
    for (int d = 0; d < nsrc; ++d) {
        const double* g = src[d] + r0 * nb + 2 * c;
        double* t = st + d * ps + 2 * c;
        for (int r = threadIdx.x / pr; r < rows; r += rstep) cp16g(t + r * rs, g + static_cast<std::int64_t>(r) * nb);
    }
}

// fill_stage for a compile-time row width and block size: the piece index
// and the row step are constants, and the addresses advance by increments
// (no per-chunk integer division, no per-piece 64-bit multiply).
template <int NB, int NT>
__device__ __forceinline__ void fill_stage_c(double* st, const double* const* src, int nsrc, int ps, int rs,
                                             std::int64_t r0, int rows) {
    constexpr int PR = NB / 2, RSTEP = NT / PR;  // (threads past RSTEP * PR idle when PR does not divide NT)
    const int c = threadIdx.x % PR, rf = threadIdx.x / PR;
    if (rf >= RSTEP) return;
    for (int d = 0; d < nsrc; ++d) {
        const double* g = src[d] + (r0 + rf) * NB + 2 * c;
        double* t = st + d * ps + rf * rs + 2 * c;
        for (int r = rf; r < rows; r += RSTEP, g += RSTEP * NB, t += RSTEP * rs) cp16g(t, g);
    }
}

__global__ void __launch_bounds__(512, 1) k_gram_s(GramDev g, GramS q, std::int64_t n, double* __restrict__ partial) {
    extern __shared__ __align__(16) double sbuf[];
    const int tid = threadIdx.x;
    const int nb = g.nb;
    // this CTA's rows: contiguous chunks
    const std::int64_t nchunk_all = (n + q.R - 1) / q.R;
    const std::int64_t c0 = nchunk_all * blockIdx.x / gridDim.x, c1 = nchunk_all * (blockIdx.x + 1) / gridDim.x;
    const int nch = static_cast<int>(c1 - c0);
    auto issue = [&](int c) {  // chunk c of this CTA into stage c % kGG (one commit group, maybe empty)
        if (c < nch) {
            const std::int64_t r0 = (c0 + c) * q.R;
            const int rows = static_cast<int>(min(static_cast<std::int64_t>(q.R), n - r0));
            fill_stage(sbuf + static_cast<std::size_t>(c % kGG) * q.ss, g.panel, g.nd, q.ps, q.rs, nb, r0, rows);
        }
        cp_commit();
    };
    for (int c = 0; c < kGG - 1; ++c) issue(c);

    const int task = tid % q.tasks, grp = tid / q.tasks;
    const bool active = grp < q.groups;
    const int B = q.bpr * q.bpc;
    const int p = task / B, blk = task % B;
    const int i0 = (blk / q.bpc) * 8, j0 = (blk % q.bpc) * 4;
    const int da = g.ia[p], db = g.ib[p];
    double acc[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) acc[e] = 0.0;
    for (int c = 0; c < nch; ++c) {
        issue(c + kGG - 1);  // into the stage consumed at c - 1
        cp_wait<kGG - 1>();
        __syncthreads();     // chunk c landed for every thread
        const std::int64_t r0 = (c0 + c) * q.R;
        const int rows = static_cast<int>(min(static_cast<std::int64_t>(q.R), n - r0));
        const double* st = sbuf + static_cast<std::size_t>(c % kGG) * q.ss;
        if (active) {
            const double* A = st + da * q.ps + i0;
            const double* Bp = st + db * q.ps + j0;
            for (int r = grp; r < rows; r += q.groups) {
                double a[8], b[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double2 x = *reinterpret_cast<const double2*>(A + r * q.rs + 2 * k);
                    a[2 * k] = x.x;
                    a[2 * k + 1] = x.y;
                }
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const double2 y = *reinterpret_cast<const double2*>(Bp + r * q.rs + 2 * k);
                    b[2 * k] = y.x;
                    b[2 * k + 1] = y.y;
                }
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int ii = 0; ii < 8; ++ii) acc[jj * 8 + ii] = fma(a[ii], b[jj], acc[jj * 8 + ii]);
            }
        }
        __syncthreads();  // stage c % kGG is free again
    }
    cp_wait<0>();
    __syncthreads();
    // row groups -> one partial per task (fixed order), reusing the ring
    double* out = partial + static_cast<std::int64_t>(blockIdx.x) * q.tasks * 32;
    if (32 % q.tasks == 0) {
        // lanes of a warp holding the same task: butterfly, then warps in order
        const int nw = blockDim.x / 32, warp = tid >> 5, lane = tid & 31;
        double* red = sbuf;  // nw x tasks x 32
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            double v = active ? acc[e] : 0.0;
            for (int o = q.tasks; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane < q.tasks) red[(warp * q.tasks + lane) * 32 + e] = v;
        }
        __syncthreads();
        for (int e = tid; e < q.tasks * 32; e += blockDim.x) {
            double v = red[e];
            for (int w = 1; w < nw; ++w) v += red[w * q.tasks * 32 + e];
            out[e] = v;
        }
    } else {
        double* red = sbuf;  // tasks x 32, row groups added in order
        for (int k = 0; k < q.groups; ++k) {
            if (active && grp == k)
#pragma unroll
                for (int e = 0; e < 32; ++e) red[task * 32 + e] = k == 0 ? acc[e] : red[task * 32 + e] + acc[e];
            __syncthreads();
        }
        for (int e = tid; e < q.tasks * 32; e += blockDim.x) out[e] = red[e];
    }
}

// ---- Gram on the FP64 tensor cores (nb in {8, 16, 24, 32}): the same
// cp.async row-chunk ring (rows padded to nb + 4 doubles: the m8n8k4 fragment
// reads hit every bank twice, the minimum), then each warp owns a few pairs
// and a row group: per 4 rows it loads the A fragments (8 x 4 of X^T) and B
// fragments (4 x 8 of Y) of its pairs once and issues one DMMA per 8 x 8
// output block (mma.sync m8n8k4 f64: 256 FMAs per instruction, accumulators
// in 2 registers per block). Row groups are summed in shared memory in a
// fixed order, CTAs by k_gram_reduce_m (deterministic).
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct GramM {
    int R;      // rows per chunk (multiple of 4)
    int rs;     // padded row stride (nb + 4)
    int ps;     // doubles per panel slot (R * rs)
    int ss;     // doubles per stage
    int pw;     // pairs per warp
    int ngrp;   // warp groups (pairs split): 8 / rg
    int rg;     // row groups (warps sharing the same pairs)
};

template <int NBB>  // 8-blocks per dimension (nb / 8)
#ifndef BE_GRAM_CTAS
#define BE_GRAM_CTAS 2  // CTAs per SM of the tensor-core Gram kernel (one CTA computes while the other waits on its ring)
#endif
#ifndef BE_GRAM_STAGE_KB
#define BE_GRAM_STAGE_KB 26
#endif
__global__ void __launch_bounds__(256, BE_GRAM_CTAS) k_gram_m(GramDev g, GramM q, std::int64_t n, double* __restrict__ partial) {
    constexpr int MAXPW = 16 / (NBB * NBB) > 0 ? 16 / (NBB * NBB) : 1;  // <= 16 blocks per warp
    extern __shared__ __align__(16) double sbuf[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = g.nb;
    const std::int64_t nchunk_all = (n + q.R - 1) / q.R;
    const std::int64_t c0 = nchunk_all * blockIdx.x / gridDim.x, c1 = nchunk_all * (blockIdx.x + 1) / gridDim.x;
    const int nch = static_cast<int>(c1 - c0);
    auto issue = [&](int c) {
        if (c < nch) {
            const std::int64_t r0 = (c0 + c) * q.R;
            const int rows = static_cast<int>(min(static_cast<std::int64_t>(q.R), n - r0));
            if (nb == 8 * NBB)
                fill_stage_c<8 * NBB, 256>(sbuf + static_cast<std::size_t>(c % kGG) * q.ss, g.panel, g.nd, q.ps, q.rs,
                                           r0, rows);
            else
                fill_stage(sbuf + static_cast<std::size_t>(c % kGG) * q.ss, g.panel, g.nd, q.ps, q.rs, nb, r0, rows);
        }
        cp_commit();
    };
    for (int c = 0; c < kGG - 1; ++c) issue(c);
    const int wg = warp / q.rg, rgi = warp % q.rg;  // pair group, row group
    const int p0 = wg * q.pw;
    const int m = lane >> 2, kq = lane & 3;
    // this warp's pairs: count and panel offsets in a stage, hoisted out of the row loop
    const int npw = max(0, min(q.pw, g.npairs - p0));
    int aoff[MAXPW], boff[MAXPW];
#pragma unroll
    for (int a = 0; a < MAXPW; ++a) {
        aoff[a] = a < npw ? g.ia[p0 + a] * q.ps : 0;
        boff[a] = a < npw ? g.ib[p0 + a] * q.ps : 0;
    }
    double acc[MAXPW][NBB][NBB][2];
#pragma unroll
    for (int a = 0; a < MAXPW; ++a)
#pragma unroll
        for (int i = 0; i < NBB; ++i)
#pragma unroll
            for (int j = 0; j < NBB; ++j) acc[a][i][j][0] = acc[a][i][j][1] = 0.0;
    for (int c = 0; c < nch; ++c) {
        issue(c + kGG - 1);
        cp_wait<kGG - 1>();
        __syncthreads();
        const std::int64_t r0 = (c0 + c) * q.R;
        const int rows = static_cast<int>(min(static_cast<std::int64_t>(q.R), n - r0));
        const double* st = sbuf + static_cast<std::size_t>(c % kGG) * q.ss;
        for (int k0 = 4 * rgi; k0 < rows; k0 += 4 * q.rg) {
            const int r = k0 + kq;
            const bool ok = r < rows;
            const double* sr = st + r * q.rs + m;
#pragma unroll
            for (int a = 0; a < MAXPW; ++a) {
                if (a >= npw) break;
                const double* A = sr + aoff[a];
                const double* B = sr + boff[a];
                double fa[NBB], fb[NBB];
#pragma unroll
                for (int i = 0; i < NBB; ++i) {
                    fa[i] = ok ? A[8 * i] : 0.0;
                    fb[i] = ok ? B[8 * i] : 0.0;
                }
#pragma unroll
                for (int i = 0; i < NBB; ++i)
#pragma unroll
                    for (int j = 0; j < NBB; ++j) dmma884(acc[a][i][j][0], acc[a][i][j][1], fa[i], fb[j]);
            }
        }
        __syncthreads();
    }
    cp_wait<0>();
    __syncthreads();
    // row groups in order -> red[pair][nb][nb] (row-major i, j), then the CTA partial
    double* red = sbuf;
    for (int k = 0; k < q.rg; ++k) {
        if (rgi == k)
#pragma unroll
            for (int a = 0; a < MAXPW; ++a) {
                const int p = p0 + a;
                if (a >= q.pw || p >= g.npairs) break;
#pragma unroll
                for (int i = 0; i < NBB; ++i)
#pragma unroll
                    for (int j = 0; j < NBB; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            double* dst = red + (static_cast<std::size_t>(p) * nb + 8 * i + m) * nb + 8 * j + 2 * kq + h;
                            *dst = k == 0 ? acc[a][i][j][h] : *dst + acc[a][i][j][h];
                        }
            }
        __syncthreads();
    }
    double* out = partial + static_cast<std::int64_t>(blockIdx.x) * g.npairs * nb * nb;
    for (int e = tid; e < g.npairs * nb * nb; e += blockDim.x) out[e] = red[e];
}

// Register-direct Gram (nb = 8 NBB, NBB = 1 or 2; <= 2 pairs over <= 2
// panels): no staging, no CTA barrier in the row loop. The CTA takes a
// contiguous range of 32-row groups, its warps interleave over them; per
// group a lane (g, t) loads, for k-step kk, row 4 kk + t at columns NBB g ..
// NBB g + NBB - 1 of each panel (one 16- or 8-byte load; a warp load is four
// whole rows) -- the m / n index of the m8n8k4 fragments is permuted so that
// fragment element ib of lane g is column NBB g + ib: block (ib, jb) of the
// accumulators holds output entries (NBB g + ib, NBB (2 t + h) + jb). Warps
// are summed in order through shared memory into the CTA partial
// (k_gram_reduce_m sums the CTAs in a fixed order: deterministic).
template <int NBB, int ND, int NPR>
__global__ void __launch_bounds__(512, ND == 2 ? 1 : 2) k_gram_r(GramDev g, std::int64_t n, double* __restrict__ partial) {
    constexpr int NB = 8 * NBB, U = 8;  // 8 k-steps = 32 rows per group
    extern __shared__ __align__(16) double red[];  // [warp][pair][NB][NB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int gq = lane >> 2, t = lane & 3;
    const std::int64_t nq = (n + 31) / 32;
    const std::int64_t q0 = nq * blockIdx.x / gridDim.x, q1 = nq * (blockIdx.x + 1) / gridDim.x;
    int ia[NPR], ib[NPR];
#pragma unroll
    for (int a = 0; a < NPR; ++a) {
        ia[a] = g.ia[a];
        ib[a] = g.ib[a];
    }
    double acc[NPR][NBB][NBB][2];
#pragma unroll
    for (int a = 0; a < NPR; ++a)
#pragma unroll
        for (int i = 0; i < NBB; ++i)
#pragma unroll
            for (int j = 0; j < NBB; ++j) acc[a][i][j][0] = acc[a][i][j][1] = 0.0;
    for (std::int64_t q = q0 + warp; q < q1; q += nw) {
        double x[ND][U][NBB];
#pragma unroll
        for (int d = 0; d < ND; ++d)
#pragma unroll
            for (int kk = 0; kk < U; ++kk) {
                const std::int64_t row = q * 32 + 4 * kk + t;
                const double* p = g.panel[d] + row * NB + NBB * gq;
                if constexpr (NBB == 2) {
                    const double2 v = row < n ? *reinterpret_cast<const double2*>(p) : make_double2(0.0, 0.0);
                    x[d][kk][0] = v.x;
                    x[d][kk][1] = v.y;
                } else {
                    x[d][kk][0] = row < n ? *p : 0.0;
                }
            }
#pragma unroll
        for (int kk = 0; kk < U; ++kk)
#pragma unroll
            for (int a = 0; a < NPR; ++a)
#pragma unroll
                for (int i = 0; i < NBB; ++i)
#pragma unroll
                    for (int j = 0; j < NBB; ++j) {
                        const double fa = ND == 1 || ia[a] == 0 ? x[0][kk][i] : x[ND - 1][kk][i];
                        const double fb = ND == 1 || ib[a] == 0 ? x[0][kk][j] : x[ND - 1][kk][j];
                        dmma884(acc[a][i][j][0], acc[a][i][j][1], fa, fb);
                    }
    }
    // this warp's sums -> red[warp], then the warps in order -> the CTA partial (row-major i, j)
    double* mine = red + static_cast<std::size_t>(warp) * NPR * NB * NB;
#pragma unroll
    for (int a = 0; a < NPR; ++a)
#pragma unroll
        for (int i = 0; i < NBB; ++i)
#pragma unroll
            for (int j = 0; j < NBB; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    mine[(a * NB + NBB * gq + i) * NB + NBB * (2 * t + h) + j] = acc[a][i][j][h];
    __syncthreads();
    for (int e = tid; e < NPR * NB * NB; e += blockDim.x) {
        double s = red[e];
        for (int w = 1; w < nw; ++w) s += red[static_cast<std::size_t>(w) * NPR * NB * NB + e];
        partial[static_cast<std::int64_t>(blockIdx.x) * NPR * NB * NB + e] = s;
    }
}

// out_p(i, j) = sum over CTAs (lane-strided + butterfly, fixed order);
// symmetrised pairs average both halves (gram, densela.hpp:90-97)
__global__ void k_gram_reduce_m(GramDev g, GramOut o, int nparts, const double* __restrict__ partial) {
    const int nb = g.nb;
    const int total = g.npairs * nb * nb;
    const int lane = threadIdx.x & 31;
    for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < total; e += (gridDim.x * blockDim.x) >> 5) {
        const int p = e / (nb * nb), rem = e % (nb * nb);
        const int j = rem / nb, i = rem % nb;  // column-major (i, j)
        if (o.sym[p] && i > j) continue;
        auto sum_at = [&](int ii, int jj) {
            const std::int64_t el = (static_cast<std::int64_t>(p) * nb + ii) * nb + jj;
            double s = 0.0;
            for (int b = lane; b < nparts; b += 32) s += partial[static_cast<std::int64_t>(b) * total + el];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            return s;
        };
        const double sij = sum_at(i, j);
        if (o.sym[p] && i != j) {
            const double s = 0.5 * (sij + sum_at(j, i));
            if (lane == 0) {
                o.out[p][j * nb + i] = s;
                o.out[p][i * nb + j] = s;
            }
        } else if (lane == 0) {
            o.out[p][j * nb + i] = sij;
        }
    }
}

// out_p(i, j) = sum over CTAs (lane-strided + butterfly, fixed order);
// symmetrised pairs average both halves (gram, densela.hpp:90-97)
__global__ void k_gram_reduce8(GramDev g, GramOut o, GramS q, int nparts, const double* __restrict__ partial) {
    const int nb = g.nb;
    const int total = g.npairs * nb * nb;
    const int lane = threadIdx.x & 31;
    const int B = q.bpr * q.bpc;
    for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < total; e += (gridDim.x * blockDim.x) >> 5) {
        const int p = e / (nb * nb), rem = e % (nb * nb);
        const int j = rem / nb, i = rem % nb;  // column-major (i, j)
        if (o.sym[p] && i > j) continue;
        auto sum_at = [&](int ii, int jj) {
            const int task = p * B + (ii / 8) * q.bpc + (jj / 4);
            const int el = (jj % 4) * 8 + (ii % 8);
            double s = 0.0;
            for (int b = lane; b < nparts; b += 32) s += partial[(static_cast<std::int64_t>(b) * q.tasks + task) * 32 + el];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            return s;
        };
        const double sij = sum_at(i, j);
        if (o.sym[p] && i != j) {
            const double s = 0.5 * (sij + sum_at(j, i));
            if (lane == 0) {
                o.out[p][j * nb + i] = s;
                o.out[p][i * nb + j] = s;
            }
        } else if (lane == 0) {
            o.out[p][j * nb + i] = sij;
        }
    }
}

// out_p(i, j) = sum over CTAs (fixed lane-strided order + butterfly, so the
// result is deterministic); symmetrised pairs average both halves. One warp
// per output element.
__global__ void k_gram_reduce(GramDev g, GramOut o, int nparts, const double* __restrict__ partial) {
    const int nb = g.nb;
    const int total = g.npairs * nb * nb;
    const int lane = threadIdx.x & 31;
    for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < total; e += (gridDim.x * blockDim.x) >> 5) {
        const int p = e / (nb * nb), rem = e % (nb * nb);
        const int j = rem / nb, i = rem % nb;  // column-major (i, j)
        if (o.sym[p] && i > j) continue;
        auto sum_at = [&](int ii, int jj) {
            const int combo = p * g.nblk * g.nblk + (ii / 4) * g.nblk + (jj / 4);
            const int el = (jj % 4) * 4 + (ii % 4);
            double s = 0.0;
            for (int b = lane; b < nparts; b += 32) s += partial[(static_cast<std::int64_t>(b) * g.ncombo + combo) * 16 + el];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            return s;
        };
        const double sij = sum_at(i, j);
        if (o.sym[p] && i != j) {
            const double s = 0.5 * (sij + sum_at(j, i));
            if (lane == 0) {
                o.out[p][j * nb + i] = s;
                o.out[p][i * nb + j] = s;
            }
        } else if (lane == 0) {
            o.out[p][j * nb + i] = sij;
        }
    }
}

// --------------------------------------------------------------------- mix
struct MixDev {
    int nb, nout, ncoef;
    const double* coef[12];  // distinct coefficient matrices
    int ld[12];
    struct O {
        double* y;
        int accumulate, nterms, add_from, add_si, acc_si;
        const double* src[3];
        int ci[3];
        int si[3];
        double sign[3];
    } out[4];
};

// CTA tile of RT rows: the distinct source panels' rows are staged in smem
// with 16-byte coalesced loads (row stride nb + 1 doubles: conflict-free
// column reads), then thread = (row, 4-column block) forms every output for
// its row from smem and the transposed coefficients.
#ifndef BE_MIX_ROWS
#define BE_MIX_ROWS 64
#endif
#ifndef BE_MIX_CTAS
#define BE_MIX_CTAS 4  // CTAs per SM in the grid
#endif
constexpr int kMixRows = BE_MIX_ROWS;
struct MixSrc {
    int nsrc;
    const double* src[8];
};
__global__ void __launch_bounds__(kT) k_mix(MixDev m, MixSrc ms, const int* __restrict__ srcidx_dummy, std::int64_t n) {
    extern __shared__ double sh[];
    const int nb = m.nb, nblk = (nb + 3) / 4, nbp = nblk * 4, ld = nb + 1;
    double* ct = sh;                                 // ncoef x nb x nbp
    double* xs = sh + m.ncoef * nb * nbp;            // nsrc x kMixRows x ld
    for (int c = 0; c < m.ncoef; ++c)
        for (int e = threadIdx.x; e < nb * nbp; e += kT) {
            const int i = e / nbp, j = e % nbp;
            ct[c * nb * nbp + e] = j < nb ? m.coef[c][j * m.ld[c] + i] : 0.0;
        }
    const int rpi = kT / nblk;  // rows computed per pass
    for (std::int64_t r0 = static_cast<std::int64_t>(blockIdx.x) * kMixRows; r0 < n;
         r0 += static_cast<std::int64_t>(gridDim.x) * kMixRows) {
        const int rows = static_cast<int>(n - r0 < kMixRows ? n - r0 : kMixRows);
        __syncthreads();
        for (int q = 0; q < ms.nsrc; ++q) {
            const double* src = ms.src[q] + r0 * nb;
            double* dst = xs + q * kMixRows * ld;
            if ((nb & 1) == 0) {
                const int tot = rows * nb / 2;
                for (int e = threadIdx.x; e < tot; e += kT) {
                    const double2 v = __ldg(reinterpret_cast<const double2*>(src) + e);
                    const int r = (2 * e) / nb, c = (2 * e) % nb;
                    dst[r * ld + c] = v.x;
                    dst[r * ld + c + 1] = v.y;
                }
            } else {
                for (int e = threadIdx.x; e < rows * nb; e += kT) dst[(e / nb) * ld + e % nb] = __ldg(src + e);
            }
        }
        __syncthreads();
        for (int rl = threadIdx.x / nblk; rl < rows; rl += rpi) {
            if (threadIdx.x >= rpi * nblk) break;
            const std::int64_t r = r0 + rl;
            const int j0 = (threadIdx.x % nblk) * 4;
            double res[4][4];
            for (int o = 0; o < m.nout; ++o) {
                const auto& O = m.out[o];
                double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                double* y = O.y + r * nb;
                if (O.accumulate) {  // the old value, staged with the sources
                    const double* yo = xs + O.acc_si * kMixRows * ld + rl * ld + j0;
                    a0 = j0 < nb ? yo[0] : 0.0;
                    a1 = j0 + 1 < nb ? yo[1] : 0.0;
                    a2 = j0 + 2 < nb ? yo[2] : 0.0;
                    a3 = j0 + 3 < nb ? yo[3] : 0.0;
                }
                for (int tt = 0; tt < O.nterms; ++tt) {
                    const double* x = xs + O.si[tt] * kMixRows * ld + rl * ld;
                    const double* C = ct + O.ci[tt] * nb * nbp + j0;
                    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
                    for (int i = 0; i < nb; ++i) {
                        const double xi = x[i];
                        const double2 c01 = *reinterpret_cast<const double2*>(C + i * nbp);
                        const double2 c23 = *reinterpret_cast<const double2*>(C + i * nbp + 2);
                        s0 += xi * c01.x;
                        s1 += xi * c01.y;
                        s2 += xi * c23.x;
                        s3 += xi * c23.y;
                    }
                    const double sg = O.sign[tt];
                    a0 += sg * s0;
                    a1 += sg * s1;
                    a2 += sg * s2;
                    a3 += sg * s3;
                }
                if (O.add_from >= 0) {
                    a0 += res[O.add_from][0];
                    a1 += res[O.add_from][1];
                    a2 += res[O.add_from][2];
                    a3 += res[O.add_from][3];
                }
                if (O.add_si >= 0) {
                    const double* x = xs + O.add_si * kMixRows * ld + rl * ld + j0;
                    a0 += x[0];
                    if (j0 + 1 < nb) a1 += x[1];
                    if (j0 + 2 < nb) a2 += x[2];
                    if (j0 + 3 < nb) a3 += x[3];
                }
                res[o][0] = a0;
                res[o][1] = a1;
                res[o][2] = a2;
                res[o][3] = a3;
                if (j0 + 3 < nb && (nb & 1) == 0) {
                    reinterpret_cast<double2*>(y + j0)[0] = make_double2(a0, a1);
                    reinterpret_cast<double2*>(y + j0)[1] = make_double2(a2, a3);
                } else {
                    if (j0 < nb) y[j0] = a0;
                    if (j0 + 1 < nb) y[j0 + 1] = a1;
                    if (j0 + 2 < nb) y[j0 + 2] = a2;
                    if (j0 + 3 < nb) y[j0 + 3] = a3;
                }
            }
        }
    }
}

// Pipelined mix (nb even, nb / 2 divides the block): the CTA walks a
// contiguous range of kMixPRows-row chunks; the distinct source rows of
// chunk c + 1 are in flight (cp.async into the other stage, row stride nb + 2
// doubles: 16-byte aligned and conflict-free column reads) while chunk c is
// formed. Thread = (row, 4-column block) as in k_mix.
#ifndef BE_MIXP_ROWS
#define BE_MIXP_ROWS 64
#endif
#ifndef BE_MIXP_CTAS
#define BE_MIXP_CTAS 2
#endif
constexpr int kMixPRows = BE_MIXP_ROWS;
__global__ void __launch_bounds__(kT, BE_MIXP_CTAS) k_mix_p(MixDev m, MixSrc ms, std::int64_t n) {
    extern __shared__ __align__(16) double sh[];
    const int nb = m.nb, nblk = (nb + 3) / 4, nbp = nblk * 4, ld = nb + 2;
    const int ps = kMixPRows * ld, ss = ms.nsrc * ps;
    double* ct = sh;  // ncoef x nb x nbp (transposed coefficients)
    double* stg = sh + ((m.ncoef * nb * nbp + 1) & ~1);
    const std::int64_t nch_all = (n + kMixPRows - 1) / kMixPRows;
    const std::int64_t c0 = nch_all * blockIdx.x / gridDim.x, c1 = nch_all * (blockIdx.x + 1) / gridDim.x;
    const int nch = static_cast<int>(c1 - c0);
    auto issue = [&](int c) {
        if (c < nch) {
            const std::int64_t r0 = (c0 + c) * kMixPRows;
            const int rows = static_cast<int>(min(static_cast<std::int64_t>(kMixPRows), n - r0));
            fill_stage(stg + (c & 1) * ss, ms.src, ms.nsrc, ps, ld, nb, r0, rows);
        }
        cp_commit();
    };
    issue(0);
    for (int c = 0; c < m.ncoef; ++c)
        for (int e = threadIdx.x; e < nb * nbp; e += kT) {
            const int i = e / nbp, j = e % nbp;
            ct[c * nb * nbp + e] = j < nb ? m.coef[c][j * m.ld[c] + i] : 0.0;
        }
    const int rpi = kT / nblk;  // rows computed per pass
    for (int c = 0; c < nch; ++c) {
        issue(c + 1);
        cp_wait<1>();
        __syncthreads();  // chunk c staged (and the coefficients, first time)
        const double* xs = stg + (c & 1) * ss;
        const std::int64_t r0 = (c0 + c) * kMixPRows;
        const int rows = static_cast<int>(min(static_cast<std::int64_t>(kMixPRows), n - r0));
        if (threadIdx.x < rpi * nblk)
            for (int rl = threadIdx.x / nblk; rl < rows; rl += rpi) {
                const std::int64_t r = r0 + rl;
                const int j0 = (threadIdx.x % nblk) * 4;
                double res[4][4];
                for (int o = 0; o < m.nout; ++o) {
                    const auto& O = m.out[o];
                    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                    if (O.accumulate) {
                        const double* yo = xs + O.acc_si * ps + rl * ld + j0;
                        a0 = j0 < nb ? yo[0] : 0.0;
                        a1 = j0 + 1 < nb ? yo[1] : 0.0;
                        a2 = j0 + 2 < nb ? yo[2] : 0.0;
                        a3 = j0 + 3 < nb ? yo[3] : 0.0;
                    }
                    for (int tt = 0; tt < O.nterms; ++tt) {
                        const double* x = xs + O.si[tt] * ps + rl * ld;
                        const double* C = ct + O.ci[tt] * nb * nbp + j0;
                        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
                        for (int i = 0; i < nb; ++i) {
                            const double xi = x[i];
                            const double2 c01 = *reinterpret_cast<const double2*>(C + i * nbp);
                            const double2 c23 = *reinterpret_cast<const double2*>(C + i * nbp + 2);
                            s0 += xi * c01.x;
                            s1 += xi * c01.y;
                            s2 += xi * c23.x;
                            s3 += xi * c23.y;
                        }
                        const double sg = O.sign[tt];
                        a0 += sg * s0;
                        a1 += sg * s1;
                        a2 += sg * s2;
                        a3 += sg * s3;
                    }
                    if (O.add_from >= 0) {
                        a0 += res[O.add_from][0];
                        a1 += res[O.add_from][1];
                        a2 += res[O.add_from][2];
                        a3 += res[O.add_from][3];
                    }
                    if (O.add_si >= 0) {
                        const double* x = xs + O.add_si * ps + rl * ld + j0;
                        a0 += x[0];
                        if (j0 + 1 < nb) a1 += x[1];
                        if (j0 + 2 < nb) a2 += x[2];
                        if (j0 + 3 < nb) a3 += x[3];
                    }
                    res[o][0] = a0;
                    res[o][1] = a1;
                    res[o][2] = a2;
                    res[o][3] = a3;
                    double* y = O.y + r * nb;
                    if (j0 + 3 < nb) {
                        reinterpret_cast<double2*>(y + j0)[0] = make_double2(a0, a1);
                        reinterpret_cast<double2*>(y + j0)[1] = make_double2(a2, a3);
                    } else {
                        if (j0 < nb) y[j0] = a0;
                        if (j0 + 1 < nb) y[j0 + 1] = a1;
                    }
                }
            }
        __syncthreads();  // stage c & 1 is refilled by the next iteration's issue
    }
    cp_wait<0>();
}

// Tensor-core mix (nb = 8 * NBB, every output a sum of <= 4 terms): the
// chunk pipeline of k_mix_p, then warp w forms rows 8w .. 8w + 7 of every
// output with DMMA (m8n8k4 f64). The coefficient blocks are the B fragments,
// loaded once per CTA into registers (sign folded in); per k-step a lane
// loads one A element (row stride nb + 4 doubles: conflict-free). The
// accumulate / add_src terms are added in the accumulator layout.
struct MixT {
    int nq;           // term slots, output-major
    int qo[4], qs[4]; // output, staged source of each slot
    int last[4];      // slot ends its output
};
// BSM (nb = 24, 32): the B fragments no longer fit the registers and are read
// from shared memory instead, laid out fragment-major so a warp's 32 loads of
// one fragment are one contiguous 256-byte read.
template <int NBB, bool BSM = false>
__global__ void __launch_bounds__(kT, BSM ? 1 : 2) k_mix_t(MixDev m, MixSrc ms, MixT mt, std::int64_t n) {
    constexpr int NB = NBB * 8, KS = NB / 4, LD = NB + 4, MAXT = 4;
    static_assert(kMixPRows == 8 * (kT / 32), "one 8-row block per warp");
    extern __shared__ __align__(16) double sh[];
    const int ps = kMixPRows * LD, ss = ms.nsrc * ps;
    double* stg = sh;
    const std::int64_t nch_all = (n + kMixPRows - 1) / kMixPRows;
    const std::int64_t c0 = nch_all * blockIdx.x / gridDim.x, c1 = nch_all * (blockIdx.x + 1) / gridDim.x;
    const int nch = static_cast<int>(c1 - c0);
    auto issue = [&](int c) {
        if (c < nch) {
            const std::int64_t r0 = (c0 + c) * kMixPRows;
            const int rows = static_cast<int>(min(static_cast<std::int64_t>(kMixPRows), n - r0));
            fill_stage_c<NB, kT>(stg + (c & 1) * ss, ms.src, ms.nsrc, ps, LD, r0, rows);
        }
        cp_commit();
    };
    issue(0);
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, rl = (threadIdx.x >> 5) * 8 + g;
    // B fragments: B[k = t][col = g] of each slot's coefficient block
    double bf[BSM ? 1 : MAXT][BSM ? 1 : KS][BSM ? 1 : NBB];
    double* bsm = sh + 2 * static_cast<std::size_t>(ss);  // (BSM) [slot][k][cb][lane]
    if constexpr (BSM) {
        for (int e = threadIdx.x; e < MAXT * KS * NBB * 32; e += kT) {
            const int ln = e & 31, cb = (e >> 5) % NBB, k = (e >> 5) / NBB % KS, q = (e >> 5) / (NBB * KS);
            const int gg = ln >> 2, tq = ln & 3;
            double v = 0.0;
            if (q < mt.nq) {
                const int o = mt.qo[q];
                int tt = 0;
                for (int p = 0; p < q; ++p) tt += mt.qo[p] == o;
                const double* cf = m.coef[m.out[o].ci[tt]];
                v = m.out[o].sign[tt] * cf[(8 * cb + gg) * m.ld[m.out[o].ci[tt]] + 4 * k + tq];
            }
            bsm[e] = v;
        }  // (visible after the first chunk's barrier below)
    } else {
#pragma unroll
        for (int q = 0; q < MAXT; ++q) {
            const int o = q < mt.nq ? mt.qo[q] : 0;
            int tt = 0;
            for (int p = 0; p < q; ++p) tt += mt.qo[p] == o;
            const double* cf = q < mt.nq ? m.coef[m.out[o].ci[tt]] : nullptr;
            const int ld = q < mt.nq ? m.ld[m.out[o].ci[tt]] : 0;
            const double sg = q < mt.nq ? m.out[o].sign[tt] : 0.0;
#pragma unroll
            for (int k = 0; k < KS; ++k)
#pragma unroll
                for (int cb = 0; cb < NBB; ++cb) bf[q][k][cb] = cf ? sg * cf[(8 * cb + g) * ld + 4 * k + t] : 0.0;
        }
    }
    for (int c = 0; c < nch; ++c) {
        issue(c + 1);
        cp_wait<1>();
        __syncthreads();  // chunk c staged
        const double* xs = stg + (c & 1) * ss;
        const std::int64_t r0 = (c0 + c) * kMixPRows;
        const int rows = static_cast<int>(min(static_cast<std::int64_t>(kMixPRows), n - r0));
        double acc[NBB][2];
#pragma unroll
        for (int cb = 0; cb < NBB; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
#pragma unroll
        for (int q = 0; q < MAXT; ++q) {
            if (q >= mt.nq) break;
            const double* xa = xs + mt.qs[q] * ps + rl * LD + t;
#pragma unroll
            for (int k = 0; k < KS; ++k) {
                const double a = xa[4 * k];
#pragma unroll
                for (int cb = 0; cb < NBB; ++cb) {
                    if constexpr (BSM) dmma884(acc[cb][0], acc[cb][1], a, bsm[((q * KS + k) * NBB + cb) * 32 + lane]);
                    else dmma884(acc[cb][0], acc[cb][1], a, bf[q][k][cb]);
                }
            }
            if (mt.last[q]) {  // output complete: old value / added panel, store, reset
                const auto& O = m.out[mt.qo[q]];
#pragma unroll
                for (int cb = 0; cb < NBB; ++cb) {
                    const int col = 8 * cb + 2 * t;
                    double v0 = acc[cb][0], v1 = acc[cb][1];
                    if (O.accumulate) {
                        const double2 yo = *reinterpret_cast<const double2*>(xs + O.acc_si * ps + rl * LD + col);
                        v0 = yo.x + v0;
                        v1 = yo.y + v1;
                    }
                    if (O.add_si >= 0) {
                        const double2 ad = *reinterpret_cast<const double2*>(xs + O.add_si * ps + rl * LD + col);
                        v0 += ad.x;
                        v1 += ad.y;
                    }
                    if (rl < rows)
                        *reinterpret_cast<double2*>(O.y + (r0 + rl) * NB + col) = make_double2(v0, v1);
                    acc[cb][0] = acc[cb][1] = 0.0;
                }
            }
        }
        __syncthreads();  // stage c & 1 is refilled by the next iteration's issue
    }
    cp_wait<0>();
}

// Register-direct tensor-core mix (nb = 8 or 16, <= 4 term slots, <= 4 panel
// loads): no shared-memory staging and no CTA barrier in the row loop. Warp w
// forms 8-row blocks w, w + W, ... (W = warps of the grid) on its own: lane
// (g, t) loads row g of every panel with 16-byte loads -- term-slot panels
// at columns KS t .. KS t + KS - 1 (KS = nb / 4), the k index of the m8n8k4
// products permuted so that k-step kk uses column KS t + kk (the same
// products, regrouped); accumulated / added panels in the accumulator layout
// (columns 8 cb + 2 t, + 1) -- then forms and stores every output. Four CTAs
// of eight warps per SM keep ~128 KB of loads in flight, like k_residual. The
// B fragments (sign folded) sit in shared memory, fragment-major.
struct MixR {
    int nq;             // term slots (loads 0 .. nq - 1 are their panels)
    const double* src[4];
    int qo[4], last[4];  // output of each slot, slot ends its output
    int accl[4], addl[4];  // per output: load index of the old value / the added panel, or -1
    double* y[4];
    // Gram epilogue (GR): A = output ga, B = output gbo or (gbo < 0) load gbl (accumulator
    // layout); per-CTA partial [a][b] into gpart
    int ga, gbo, gbl;
    int gal;  // ga < 0: A from load gal (accumulator layout)
    double* gpart;
    // residual epilogue (RS): R = HX - X diag(theta) from the term-slot loads rx / rhx, per-CTA
    // column sums of R^2 and X^2 into rpart[blk][2][nb] (k_residual's layout)
    int rx, rhx;
    const double* theta;
    double* rout;
    double* rpart;
};

template <int L, int KS>
__device__ __forceinline__ double pick_load(const double (&x)[L][KS], int l, int i) {
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j)
        if (j == l) v = x[j][i];
    return v;
}

// GR: the Gram A^T B of two of the row blocks the warp holds -- an output and an output or an
// added panel -- formed on the way (the accumulator-layout values moved into DMMA operand
// fragments by shuffles), so the next Gram needs no read of the panels it just wrote.
// RS (with GR): the residual R = HX - X diag(theta) and its column norms from the X / HX term
// loads (lobpcg.hpp:419: residual_block reads only X, HX and theta, which the mix does not change).
template <int NBB, int L, bool GR = false, bool RS = false>
__global__ void __launch_bounds__(256, GR ? (L <= 2 && !RS ? 3 : 2) : 4) k_mix_r(MixDev m, MixR r, std::int64_t n) {
    constexpr int NB = 8 * NBB, KS = NB / 4;
    constexpr int GB = GR ? NBB : 1;
    constexpr int RK = RS ? KS : 1;
    __shared__ __align__(16) double bsm[4 * KS * NBB * 32];  // [slot][kk][cb][lane]
    __shared__ double s_theta[RS ? NB : 1];
    if constexpr (RS)
        if (threadIdx.x < NB) s_theta[threadIdx.x] = r.theta[threadIdx.x];
    double rn[RK], xn[RK];
#pragma unroll
    for (int kk = 0; kk < RK; ++kk) rn[kk] = xn[kk] = 0.0;
    double gacc[GB][GB][2];
#pragma unroll
    for (int i = 0; i < GB; ++i)
#pragma unroll
        for (int j = 0; j < GB; ++j) gacc[i][j][0] = gacc[i][j][1] = 0.0;
    for (int e = threadIdx.x; e < 4 * KS * NBB * 32; e += blockDim.x) {
        const int ln = e & 31, cb = (e >> 5) % NBB, kk = (e >> 5) / NBB % KS, q = (e >> 5) / (NBB * KS);
        double v = 0.0;
        if (q < r.nq) {
            const int o = r.qo[q];
            int tt = 0;
            for (int p = 0; p < q; ++p) tt += r.qo[p] == o;
            const int ci = m.out[o].ci[tt];
            v = m.out[o].sign[tt] * m.coef[ci][(8 * cb + (ln >> 2)) * m.ld[ci] + KS * (ln & 3) + kk];
        }
        bsm[e] = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const std::int64_t nblk = (n + 7) / 8;
    const std::int64_t wstride = static_cast<std::int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (std::int64_t b = static_cast<std::int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nblk;
         b += wstride) {
        const std::int64_t row = b * 8 + g;
        const bool ok = row < n;
        double x[L][KS];
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const bool cl = l >= r.nq;  // accumulator layout
#pragma unroll
            for (int h = 0; h < KS / 2; ++h) {
                const int col = cl ? 8 * h + 2 * t : KS * t + 2 * h;
                double2 v = make_double2(0.0, 0.0);
                if (ok) v = *reinterpret_cast<const double2*>(r.src[l] + row * NB + col);
                x[l][2 * h] = v.x;
                x[l][2 * h + 1] = v.y;
            }
        }
        if constexpr (RS) {  // columns KS t .. KS t + KS - 1 of row `row` (the term-slot layout)
            double rv[KS];
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                const double xv = pick_load(x, r.rx, kk), hv = pick_load(x, r.rhx, kk);
                rv[kk] = hv - xv * s_theta[KS * t + kk];
                rn[kk] += rv[kk] * rv[kk];
                xn[kk] += xv * xv;
            }
            if (ok)
#pragma unroll
                for (int h = 0; h < KS / 2; ++h)
                    *reinterpret_cast<double2*>(r.rout + row * NB + KS * t + 2 * h) = make_double2(rv[2 * h], rv[2 * h + 1]);
        }
        double acc[NBB][2];
#pragma unroll
        for (int cb = 0; cb < NBB; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
        double ka[GB][2], kb[GB][2];  // the Gram operands' row values (accumulator layout)
#pragma unroll
        for (int q = 0; q < L; ++q) {
            if (q >= r.nq) break;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
#pragma unroll
                for (int cb = 0; cb < NBB; ++cb)
                    dmma884(acc[cb][0], acc[cb][1], x[q][kk], bsm[((q * KS + kk) * NBB + cb) * 32 + lane]);
            if (r.last[q]) {  // output complete: old value / added panel, store, reset
                const int o = r.qo[q], al = r.accl[o], dl = r.addl[o];
                double* y = r.y[o] + row * NB + 2 * t;
#pragma unroll
                for (int cb = 0; cb < NBB; ++cb) {
                    double v0 = acc[cb][0], v1 = acc[cb][1];
                    if (al >= 0) {
                        v0 = pick_load(x, al, 2 * cb) + v0;
                        v1 = pick_load(x, al, 2 * cb + 1) + v1;
                    }
                    if (dl >= 0) {
                        v0 += pick_load(x, dl, 2 * cb);
                        v1 += pick_load(x, dl, 2 * cb + 1);
                    }
                    if (ok) *reinterpret_cast<double2*>(y + 8 * cb) = make_double2(v0, v1);
                    if constexpr (GR) {
                        if (o == r.ga) ka[cb][0] = v0, ka[cb][1] = v1;
                        if (o == r.gbo) kb[cb][0] = v0, kb[cb][1] = v1;
                    }
                    acc[cb][0] = acc[cb][1] = 0.0;
                }
            }
        }
        if constexpr (GR) {
            if (r.gbo < 0)
#pragma unroll
                for (int cb = 0; cb < NBB; ++cb) {
                    kb[cb][0] = pick_load(x, r.gbl, 2 * cb);
                    kb[cb][1] = pick_load(x, r.gbl, 2 * cb + 1);
                }
            if (r.ga < 0)
#pragma unroll
                for (int cb = 0; cb < NBB; ++cb) {
                    ka[cb][0] = pick_load(x, r.gal, 2 * cb);
                    ka[cb][1] = pick_load(x, r.gal, 2 * cb + 1);
                }
            // rows past n hold zeros (their loads were zero-filled and nothing was added)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int src = (4 * ks + t) * 4 + (g >> 1);  // lane holding row 4 ks + t, columns 8 cb + g
                double fa[GB], fb[GB];
#pragma unroll
                for (int cb = 0; cb < GB; ++cb) {
                    const double a0 = __shfl_sync(0xffffffffu, ka[cb][0], src), a1 = __shfl_sync(0xffffffffu, ka[cb][1], src);
                    const double b0 = __shfl_sync(0xffffffffu, kb[cb][0], src), b1 = __shfl_sync(0xffffffffu, kb[cb][1], src);
                    fa[cb] = (g & 1) ? a1 : a0;
                    fb[cb] = (g & 1) ? b1 : b0;
                }
#pragma unroll
                for (int i = 0; i < GB; ++i)
#pragma unroll
                    for (int j = 0; j < GB; ++j) dmma884(gacc[i][j][0], gacc[i][j][1], fa[i], fb[j]);
            }
        }
    }
    if constexpr (GR) {  // warps in order -> the CTA partial (row-major a, b)
        __shared__ double red[8][NB * NB];
        const int warp = threadIdx.x >> 5;
#pragma unroll
        for (int i = 0; i < GB; ++i)
#pragma unroll
            for (int j = 0; j < GB; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) red[warp][(8 * i + g) * NB + 8 * j + 2 * t + h] = gacc[i][j][h];
        __syncthreads();
        for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
            double sum = red[0][e];
            for (int w = 1; w < 8; ++w) sum += red[w][e];
            r.gpart[static_cast<std::int64_t>(blockIdx.x) * NB * NB + e] = sum;
        }
    }
    if constexpr (RS) {  // rows of a warp (lanes of equal t) by butterfly, then warps in order
        __shared__ double rred[8][2][NB];
        const int warp = threadIdx.x >> 5;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk)
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                rn[kk] += __shfl_xor_sync(0xffffffffu, rn[kk], o);
                xn[kk] += __shfl_xor_sync(0xffffffffu, xn[kk], o);
            }
        if (g == 0)
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
                rred[warp][0][KS * t + kk] = rn[kk];
                rred[warp][1][KS * t + kk] = xn[kk];
            }
        __syncthreads();
        if (threadIdx.x < 2 * NB) {
            const int wh = threadIdx.x / NB, c = threadIdx.x % NB;
            double sum = rred[0][wh][c];
            for (int w = 1; w < 8; ++w) sum += rred[w][wh][c];
            r.rpart[(static_cast<std::int64_t>(blockIdx.x) * 2 + wh) * NB + c] = sum;
        }
    }
}

// ---- streamed trsm (nb % 2 == 0, nb <= NBP): W <- W R^-1 for one or two
// panels; chunk rows arrive by bulk copy, thread = (panel, row) substitutes
// in registers (rows read / written in a lane-rotated 16-byte order), the
// results go back through the stage and leave by one bulk store per panel.

template <int NBP>
__global__ void __launch_bounds__(256, 2) k_trsm_s(double* __restrict__ w0, double* __restrict__ w1,
                                                  const double* __restrict__ Rg, int nb, std::int64_t n, Status* st,
                                                  int skip_if_rank, int skip_if_notpd, int R, int ps) {
    extern __shared__ __align__(16) double sbuf[];
    __shared__ double Rs[NBP * NBP];
    __shared__ double Rinv[NBP];
    __shared__ int skip;
    const int tid = threadIdx.x;
    const int np = w1 ? 2 : 1;
    const int rs = nb + 2;
    if (tid == 0) {
        int sk = (skip_if_rank && st->rank_deficient) || (skip_if_notpd && st->not_pd);
        if (!sk) {  // trsm_right_inv's conditioning check (densela.hpp:129-136)
            double dmin = INFINITY, dmax = 0.0;
            for (int j = 0; j < nb; ++j) {
                const double d = fabs(Rg[j * nb + j]);
                dmin = fmin(dmin, d);
                dmax = fmax(dmax, d);
            }
            if (!(dmin > 1e-14 * dmax)) {
                sk = 1;
                if (blockIdx.x == 0) st->singular_tri = 1;
            }
        }
        skip = sk;
    }
    for (int e = tid; e < nb * nb; e += 256) Rs[e] = Rg[e];
    if (tid < nb) Rinv[tid] = 1.0 / Rg[tid * nb + tid];
    __syncthreads();
    if (skip) return;
    const std::int64_t nchunk_all = (n + R - 1) / R;
    const std::int64_t c0 = nchunk_all * blockIdx.x / gridDim.x, c1 = nchunk_all * (blockIdx.x + 1) / gridDim.x;
    const int nch = static_cast<int>(c1 - c0);
    const std::size_t ss = static_cast<std::size_t>(np) * ps;
    const double* srcs[2] = {w0, w1};
    auto issue = [&](int c) {
        if (c < nch) {
            const std::int64_t r0 = (c0 + c) * R;
            const int rows = static_cast<int>(min(static_cast<std::int64_t>(R), n - r0));
            if (nb == NBP)
                fill_stage_c<NBP, 256>(sbuf + (c % kGS) * ss, srcs, np, ps, rs, r0, rows);
            else
                fill_stage(sbuf + (c % kGS) * ss, srcs, np, ps, rs, nb, r0, rows);
        }
        cp_commit();
    };
    for (int c = 0; c < kGS - 1; ++c) issue(c);
    const int q = tid / R, rl = tid % R;
    for (int c = 0; c < nch; ++c) {
        issue(c + kGS - 1);
        cp_wait<kGS - 1>();
        __syncthreads();
        const std::int64_t r0 = (c0 + c) * R;
        const int rows = static_cast<int>(min(static_cast<std::int64_t>(R), n - r0));
        double* stg = sbuf + (c % kGS) * ss;
        if (q < np && rl < rows) {
            double* xr = stg + q * ps + rl * rs;
            double x[NBP];
#pragma unroll
            for (int k = 0; k < NBP / 2; ++k)
                if (2 * k < nb) {
                    const double2 v = reinterpret_cast<const double2*>(xr)[k];
                    x[2 * k] = v.x;
                    x[2 * k + 1] = v.y;
                }
#pragma unroll
            for (int j = 0; j < NBP; ++j) {
                if (j < nb) {
                    double s = x[j];
#pragma unroll
                    for (int i = 0; i < j; ++i) s -= x[i] * Rs[j * nb + i];
                    // s / R_jj: reciprocal + one residual correction (the
                    // correctly rounded quotient but for rare last-bit
                    // ties) instead of the ~40-instruction IEEE division
                    const double d = Rs[j * nb + j], ri = Rinv[j];
                    double qj = s * ri;
                    qj = fma(fma(-qj, d, s), ri, qj);
                    x[j] = qj;
                }
            }
#pragma unroll
            for (int k = 0; k < NBP / 2; ++k)
                if (2 * k < nb) reinterpret_cast<double2*>(xr)[k] = make_double2(x[2 * k], x[2 * k + 1]);
        }
        __syncthreads();  // the stage holds the chunk's results: coalesced 16-byte stores
        if (nb == NBP) {  // compile-time piece count: no integer division per store
            constexpr int PR = NBP / 2;
            for (int p = 0; p < np; ++p) {
                double* w = (p == 0 ? w0 : w1) + r0 * NBP;
                const double* sp = stg + p * ps;
                for (int e = tid; e < rows * PR; e += 256) {
                    const int r = e / PR, cc = e % PR;
                    reinterpret_cast<double2*>(w + r * NBP)[cc] = reinterpret_cast<const double2*>(sp + r * rs)[cc];
                }
            }
        } else {
            const int pr = nb / 2, per = rows * pr;
            for (int e = tid; e < per * np; e += 256) {
                const int p = e / per, k = e % per, r = k / pr, cc = k % pr;
                reinterpret_cast<double2*>((p == 0 ? w0 : w1) + (r0 + r) * nb)[cc] =
                    reinterpret_cast<const double2*>(stg + p * ps + r * rs)[cc];
            }
        }
        __syncthreads();  // stage free for the refill at c + 1
    }
    cp_wait<0>();
}

// ---- warp-independent trsm (nb = NB, 8 or 16): W <- W R^-1 for one or two
// panels. A warp takes 32-row blocks w, w + W, ... on its own: 16-byte
// cp.async copies (coalesced, the next block's in flight while this one is
// solved) into a double-buffered warp-private shared-memory tile (rows padded
// to NB + 2 doubles: the row-major copies and the row-per-lane reads are both
// conflict-free), lane l substitutes row l in registers exactly as k_trsm_s,
// the results go back with coalesced 16-byte stores. No CTA barrier after the
// setup. gpart (one panel): the Gram W'^T W' of the result is formed on the
// way -- DMMA over each solved tile in shared memory, warps summed in order
// into the CTA partial [i][j] (k_gram_reduce_m) -- so CholQR's second pass
// needs no separate read of W'.
constexpr int kTrsmWarps = 4;
// shared-memory loads the compiler may not hoist out of the row loop (the
// 120 factor entries would otherwise be kept in registers and spill)
__device__ __forceinline__ double2 lds2_nohoist(const double* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(stream::smem_u32(p)));
    return v;
}
__device__ __forceinline__ double lds_nohoist(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(stream::smem_u32(p)));
    return v;
}
template <int NB>
__global__ void __launch_bounds__(kTrsmWarps * 32) k_trsm_r(double* __restrict__ w0, double* __restrict__ w1,
                                                           const double* __restrict__ Rg, std::int64_t n, Status* st,
                                                           int skip_if_rank, int skip_if_notpd,
                                                           double* __restrict__ gpart) {
    constexpr int NBB = NB / 8;
    constexpr int RS = NB + 2, PR = NB / 2;  // padded row stride (doubles), 16-byte pieces per row
    constexpr int RPI = 32 / PR;             // rows per coalesced warp copy
    constexpr int LPP = NB / 2;              // 16-byte pieces per lane per panel block
    extern __shared__ __align__(16) double sbuf[];
    __shared__ __align__(16) double Rs[NB * NB];
    __shared__ double Rinv[NB];
    __shared__ int skip;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int np = w1 ? 2 : 1;
    if (tid == 0) {
        int sk = (skip_if_rank && st->rank_deficient) || (skip_if_notpd && st->not_pd);
        if (!sk) {  // trsm_right_inv's conditioning check (densela.hpp:129-136)
            double dmin = INFINITY, dmax = 0.0;
            for (int j = 0; j < NB; ++j) {
                const double d = fabs(Rg[j * NB + j]);
                dmin = fmin(dmin, d);
                dmax = fmax(dmax, d);
            }
            if (!(dmin > 1e-14 * dmax)) {
                sk = 1;
                if (blockIdx.x == 0) st->singular_tri = 1;
            }
        }
        skip = sk;
    }
    for (int e = tid; e < NB * NB; e += blockDim.x) Rs[e] = Rg[e];
    if (tid < NB) Rinv[tid] = 1.0 / Rg[tid * NB + tid];
    __syncthreads();
    if (skip) return;
    const int tstride = np * 32 * RS;                                        // one buffer: [panel][row][RS]
    double* tiles = sbuf + static_cast<std::size_t>(warp) * 2 * tstride;  // two buffers per warp
    const std::int64_t nblk = (n + 31) / 32;
    const std::int64_t wstride = static_cast<std::int64_t>(gridDim.x) * kTrsmWarps;
    const int lr = lane / PR, lc = lane % PR;  // coalesced piece: row lr + RPI k, piece lc
    auto issue = [&](std::int64_t b, double* t) {
        if (b < nblk) {
            const std::int64_t r0 = b * 32;
            for (int p = 0; p < np; ++p) {
                const double* w = (p == 0 ? w0 : w1) + r0 * NB;
#pragma unroll
                for (int k = 0; k < LPP; ++k) {
                    const int r = lr + RPI * k;
                    if (r0 + r < n) cp16g(t + p * 32 * RS + r * RS + 2 * lc, w + r * NB + 2 * lc);
                }
            }
        }
        cp_commit();
    };
    std::int64_t b = static_cast<std::int64_t>(blockIdx.x) * kTrsmWarps + warp;
    double gacc[NBB][NBB][2];
#pragma unroll
    for (int i = 0; i < NBB; ++i)
#pragma unroll
        for (int j = 0; j < NBB; ++j) gacc[i][j][0] = gacc[i][j][1] = 0.0;
    issue(b, tiles);
    for (int it = 0; b < nblk; b += wstride, ++it) {
        double* t = tiles + (it & 1) * tstride;
        issue(b + wstride, tiles + ((it + 1) & 1) * tstride);  // next block in flight during the solve
        cp_wait<1>();
        __syncwarp();
        const std::int64_t r0 = b * 32;
        for (int p = 0; p < np; ++p) {
            double* xr = t + p * 32 * RS + lane * RS;
            double x[NB];
#pragma unroll
            for (int k = 0; k < NB / 2; ++k) {
                const double2 v = reinterpret_cast<const double2*>(xr)[k];
                x[2 * k] = v.x;
                x[2 * k + 1] = v.y;
            }
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                double s = x[j];
#pragma unroll
                for (int i = 0; i + 1 < j; i += 2) {  // i ascending, as k_trsm_s
                    const double2 rr = lds2_nohoist(Rs + j * NB + i);
                    s -= x[i] * rr.x;
                    s -= x[i + 1] * rr.y;
                }
                if (j & 1) s -= x[j - 1] * lds_nohoist(Rs + j * NB + j - 1);
                const double d = lds_nohoist(Rs + j * NB + j), ri = lds_nohoist(Rinv + j);
                double qj = s * ri;
                qj = fma(fma(-qj, d, s), ri, qj);
                x[j] = qj;
            }
#pragma unroll
            for (int k = 0; k < NB / 2; ++k) reinterpret_cast<double2*>(xr)[k] = make_double2(x[2 * k], x[2 * k + 1]);
        }
        __syncwarp();
        if (gpart) {  // Gram of the solved tile (rows past n masked: their tile rows were never loaded)
            const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int r = 4 * kk + tq;
                const bool ok = r0 + r < n;
                double f[NBB];
#pragma unroll
                for (int i = 0; i < NBB; ++i) f[i] = ok ? t[r * RS + 8 * i + gq] : 0.0;
#pragma unroll
                for (int i = 0; i < NBB; ++i)
#pragma unroll
                    for (int j = 0; j < NBB; ++j) dmma884(gacc[i][j][0], gacc[i][j][1], f[i], f[j]);
            }
        }
        for (int p = 0; p < np; ++p) {
            double* w = (p == 0 ? w0 : w1) + r0 * NB;
#pragma unroll
            for (int k = 0; k < LPP; ++k) {
                const int r = lr + RPI * k;
                if (r0 + r < n)
                    reinterpret_cast<double2*>(w + r * NB)[lc] =
                        reinterpret_cast<const double2*>(t + p * 32 * RS + r * RS)[lc];
            }
        }
        __syncwarp();  // this buffer is refilled two blocks on
    }
    cp_wait<0>();
    if (gpart) {  // warps in order -> the CTA partial (row-major i, j)
        __syncthreads();
        double* red = sbuf;  // [warp][NB][NB]
        const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
        for (int i = 0; i < NBB; ++i)
#pragma unroll
            for (int j = 0; j < NBB; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) red[(warp * NB + 8 * i + gq) * NB + 8 * j + 2 * tq + h] = gacc[i][j][h];
        __syncthreads();
        for (int e = tid; e < NB * NB; e += blockDim.x) {
            double sum = red[e];
            for (int w = 1; w < kTrsmWarps; ++w) sum += red[w * NB * NB + e];
            gpart[static_cast<std::int64_t>(blockIdx.x) * NB * NB + e] = sum;
        }
    }
}

// -------------------------------------------------------------------- trsm
// 128 rows per CTA pass staged in smem (coalesced), one thread per row does
// the forward substitution of trsm_right_inv (densela.hpp:137-146) from smem.
template <int NBP>
constexpr int trsm_rows() { return NBP <= 16 ? 128 : NBP <= 32 ? 32 : 8; }
template <int NBP>
__global__ void __launch_bounds__(kT) k_trsm(double* __restrict__ w0, double* __restrict__ w1,
                                            const double* __restrict__ Rg, int nb, std::int64_t n, Status* st,
                                            int skip_if_rank, int skip_if_notpd) {
    __shared__ double R[NBP * NBP];
    constexpr int kTrsmRows = trsm_rows<NBP>();
    __shared__ double xs[2][kTrsmRows * (NBP + 1)];
    __shared__ int skip;
    const int ld = nb + 1;
    if (threadIdx.x == 0) {
        int sk = (skip_if_rank && st->rank_deficient) || (skip_if_notpd && st->not_pd);
        if (!sk) {  // trsm_right_inv's conditioning check (densela.hpp:129-136)
            double dmin = INFINITY, dmax = 0.0;
            for (int j = 0; j < nb; ++j) {
                const double d = fabs(Rg[j * nb + j]);
                dmin = fmin(dmin, d);
                dmax = fmax(dmax, d);
            }
            if (!(dmin > 1e-14 * dmax)) {
                sk = 1;
                if (blockIdx.x == 0) st->singular_tri = 1;
            }
        }
        skip = sk;
    }
    for (int e = threadIdx.x; e < nb * nb; e += kT) R[e] = Rg[e];
    __syncthreads();
    if (skip) return;
    const int np = w1 ? 2 : 1;
    for (std::int64_t r0 = static_cast<std::int64_t>(blockIdx.x) * kTrsmRows; r0 < n;
         r0 += static_cast<std::int64_t>(gridDim.x) * kTrsmRows) {
        const int rows = static_cast<int>(n - r0 < kTrsmRows ? n - r0 : kTrsmRows);
        __syncthreads();
        for (int q = 0; q < np; ++q) {
            const double* src = (q == 0 ? w0 : w1) + r0 * nb;
            for (int e = threadIdx.x; e < rows * nb; e += kT) xs[q][(e / nb) * ld + e % nb] = src[e];
        }
        __syncthreads();
        const int q = threadIdx.x / kTrsmRows, rl = threadIdx.x % kTrsmRows;
        if (q < np && rl < rows) {
            double* xr = xs[q] + rl * ld;
            double x[NBP];
#pragma unroll
            for (int j = 0; j < NBP; ++j)
                if (j < nb) x[j] = xr[j];
#pragma unroll
            for (int j = 0; j < NBP; ++j) {
                if (j < nb) {
                    double s = x[j];
#pragma unroll
                    for (int i = 0; i < j; ++i) s -= x[i] * R[j * nb + i];
                    x[j] = s / R[j * nb + j];
                }
            }
#pragma unroll
            for (int j = 0; j < NBP; ++j)
                if (j < nb) xr[j] = x[j];
        }
        __syncthreads();
        for (int qq = 0; qq < np; ++qq) {
            double* dst = (qq == 0 ? w0 : w1) + r0 * nb;
            for (int e = threadIdx.x; e < rows * nb; e += kT) dst[e] = xs[qq][(e / nb) * ld + e % nb];
        }
    }
}

// ------------------------------------------------------- small factorisations
// Block-cooperative floored Cholesky (densela.hpp:103-121 / 155-175): upper R
// with B = R^T R. floored=false reproduces cholesky() (pivot must be > 0).
// Returns the failing pivot index or -1. All threads of the CTA participate.
__device__ int dev_chol_g(const double* B, double* R, int n, double rel_floor, bool floored) {
    __shared__ double s_floor, s_rjj;
    __shared__ int s_fail;
    if (threadIdx.x == 0) {
        double dmax = 0.0;
        for (int i = 0; i < n; ++i) dmax = fmax(dmax, fabs(B[i * n + i]));
        s_floor = floored ? rel_floor * fmax(dmax, 1e-300) : 0.0;
        s_fail = -1;
    }
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) R[e] = 0.0;
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        if (threadIdx.x == 0) {
            double piv = B[j * n + j];
            for (int k = 0; k < j; ++k) piv -= R[j * n + k] * R[j * n + k];
            if (!(piv > s_floor)) {
                s_fail = j;
            } else {
                s_rjj = sqrt(piv);
                R[j * n + j] = s_rjj;
            }
        }
        __syncthreads();
        if (s_fail >= 0) return s_fail;
        const double rjj = s_rjj;
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
            double s = B[i * n + j];  // B(j, i)
            for (int k = 0; k < j; ++k) s -= R[j * n + k] * R[i * n + k];
            R[i * n + j] = s / rjj;  // R(j, i)
        }
        __syncthreads();
    }
    return -1;
}

// The same factorisation on shared-memory copies for n <= kCholS (the
// per-step pivot sums then read shared memory, not L2): identical arithmetic.
constexpr int kCholS = 48;
__device__ int dev_chol(const double* B, double* R, int n, double rel_floor, bool floored) {
    if (n > kCholS) return dev_chol_g(B, R, n, rel_floor, floored);
    __shared__ double sB[kCholS * kCholS], sR[kCholS * kCholS];
    __shared__ double s_floor, s_rjj;
    __shared__ int s_fail;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        sB[e] = B[e];
        sR[e] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double dmax = 0.0;
        for (int i = 0; i < n; ++i) dmax = fmax(dmax, fabs(sB[i * n + i]));
        s_floor = floored ? rel_floor * fmax(dmax, 1e-300) : 0.0;
        s_fail = -1;
    }
    __syncthreads();
    int fail_at = -1;
    for (int j = 0; j < n; ++j) {
        if (threadIdx.x == 0) {
            double piv = sB[j * n + j];
            for (int k = 0; k < j; ++k) piv -= sR[j * n + k] * sR[j * n + k];
            if (!(piv > s_floor)) {
                s_fail = j;
            } else {
                s_rjj = sqrt(piv);
                sR[j * n + j] = s_rjj;
            }
        }
        __syncthreads();
        if (s_fail >= 0) {
            fail_at = s_fail;
            break;
        }
        const double rjj = s_rjj;
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
            double sacc = sB[i * n + j];  // B(j, i)
            for (int k = 0; k < j; ++k) sacc -= sR[j * n + k] * sR[i * n + k];
            sR[i * n + j] = sacc / rjj;  // R(j, i)
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) R[e] = sR[e];
    __syncthreads();
    return fail_at;
}

__global__ void k_qr_chol(double* B, double* R, int nb, Status* st) {
    __shared__ int s_dead;
    if (threadIdx.x == 0) s_dead = st->rank_deficient;
    __syncthreads();
    if (s_dead) return;
    int p = dev_chol(B, R, nb, 1e-14, true);
    if (p < 0) return;
    __shared__ int s_give_up;
    if (threadIdx.x == 0) {  // densela.hpp:425-440
        s_give_up = 0;
        if (++st->qr_failures >= 2) {
            st->rank_deficient = 1;
            s_give_up = 1;
        } else {
            double dmax = 0.0;
            for (int i = 0; i < nb; ++i) dmax = fmax(dmax, B[i * nb + i]);
            const double delta = fmax(dmax, 1.0) * 1e-12 * nb;
            for (int i = 0; i < nb; ++i) B[i * nb + i] += delta;
        }
    }
    __syncthreads();
    if (s_give_up) return;
    p = dev_chol(B, R, nb, 1e-14, true);
    if (p >= 0 && threadIdx.x == 0) st->rank_deficient = 1;
}

__global__ void k_chol(const double* B, double* R, int n, double rel_floor, int floored, Status* st) {
    const int p = dev_chol(B, R, n, rel_floor, floored != 0);
    if (threadIdx.x == 0) st->not_pd = p + 1;
}

// symmetrise M in place (0.5 (M_ij + M_ji)); after a failed Cholesky the
// pencil is meaningless (the host drops it): M = I keeps the eigensolver sane
__global__ void k_sym_or_identity(double* M, int n, const Status* st) {
    const bool bad = st->not_pd != 0;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int j = e / n, i = e % n;
        if (bad) {
            M[e] = i == j ? 1.0 : 0.0;
        } else if (i < j) {
            const double v = 0.5 * (M[j * n + i] + M[i * n + j]);
            M[j * n + i] = v;
            M[i * n + j] = v;
        }
    }
}

// normalize_column_signs (densela.hpp:327-341) of C (n x k) and d = w[:k]
__global__ void k_sign_fix(double* C, const double* w, double* d, int n, int k, const Status* st) {
    if (st->not_pd) return;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        int arg = 0;
        double best = -1.0;
        for (int i = 0; i < n; ++i) {
            const double v = fabs(C[j * n + i]);
            if (v > best) {
                best = v;
                arg = i;
            }
        }
        if (C[j * n + arg] < 0.0)
            for (int i = 0; i < n; ++i) C[j * n + i] = -C[j * n + i];
        d[j] = w[j];
    }
}

// ------------------------------------------------------------- norms etc.
// per-column partial sums of squares over this CTA's rows (2 panels max)
__global__ void __launch_bounds__(kT) k_residual(const double* __restrict__ hx, const double* __restrict__ x,
                                                 const double* __restrict__ theta, double* __restrict__ r, int nb,
                                                 std::int64_t n, double* __restrict__ partial, int mode) {
    // mode 0: r = hx - x*theta, sums of r^2 and x^2; mode 1: sums of x^2 only
    __shared__ double red[2][kT];
    const int tid = threadIdx.x;
    if (nb == 16) {  // 16-byte accesses: thread = (row, column pair)
        constexpr int CP = 8, RPI = kT / CP;
        const int cp = tid % CP, rl = tid / CP;
        double sr0 = 0.0, sr1 = 0.0, sx0 = 0.0, sx1 = 0.0;
        const double th0 = mode == 0 ? theta[2 * cp] : 0.0, th1 = mode == 0 ? theta[2 * cp + 1] : 0.0;
        for (std::int64_t row = blockIdx.x * static_cast<std::int64_t>(RPI) + rl; row < n;
             row += static_cast<std::int64_t>(gridDim.x) * RPI) {
            const double2 xv = reinterpret_cast<const double2*>(x + row * 16)[cp];
            sx0 += xv.x * xv.x;
            sx1 += xv.y * xv.y;
            if (mode == 0) {
                const double2 hv = reinterpret_cast<const double2*>(hx + row * 16)[cp];
                // hx - theta x with two roundings, as written in lobpcg.hpp:208 (no FMA contraction)
                const double r0 = __dsub_rn(hv.x, __dmul_rn(th0, xv.x)), r1 = __dsub_rn(hv.y, __dmul_rn(th1, xv.y));
                reinterpret_cast<double2*>(r + row * 16)[cp] = make_double2(r0, r1);
                sr0 += r0 * r0;
                sr1 += r1 * r1;
            }
        }
        // the 4 row groups of a warp (lanes 8 apart) by butterfly, then red[.][warp * 16 + column]
        for (int o = 8; o < 32; o <<= 1) {
            sr0 += __shfl_xor_sync(0xffffffffu, sr0, o);
            sr1 += __shfl_xor_sync(0xffffffffu, sr1, o);
            sx0 += __shfl_xor_sync(0xffffffffu, sx0, o);
            sx1 += __shfl_xor_sync(0xffffffffu, sx1, o);
        }
        const int lane = tid & 31, warp = tid >> 5;
        if (lane < CP) {
            red[0][warp * 16 + 2 * cp] = sr0;
            red[0][warp * 16 + 2 * cp + 1] = sr1;
            red[1][warp * 16 + 2 * cp] = sx0;
            red[1][warp * 16 + 2 * cp + 1] = sx1;
        }
        __syncthreads();
        if (tid < 16) {
            double a = 0.0, b = 0.0;
            for (int q = 0; q < kT / 32; ++q) {
                a += red[0][q * 16 + tid];
                b += red[1][q * 16 + tid];
            }
            partial[(static_cast<std::int64_t>(blockIdx.x) * 2 + 0) * 16 + tid] = a;
            partial[(static_cast<std::int64_t>(blockIdx.x) * 2 + 1) * 16 + tid] = b;
        }
        return;
    }
    const int rpi = kT / nb;  // rows per iteration
    const int c = tid % nb, rl = tid / nb;
    double s_r = 0.0, s_x = 0.0;
    if (rl < rpi) {
        const double th = mode == 0 ? theta[c] : 0.0;
        for (std::int64_t row = blockIdx.x * static_cast<std::int64_t>(rpi) + rl; row < n;
             row += static_cast<std::int64_t>(gridDim.x) * rpi) {
            const double xv = x[row * nb + c];
            s_x += xv * xv;
            if (mode == 0) {
                const double rv = __dsub_rn(hx[row * nb + c], __dmul_rn(th, xv));  // no FMA (lobpcg.hpp:208)
                r[row * nb + c] = rv;
                s_r += rv * rv;
            }
        }
    }
    red[0][tid] = s_r;
    red[1][tid] = s_x;
    __syncthreads();
    if (tid < nb) {
        double a = 0.0, b = 0.0;
        for (int q = 0; q < rpi; ++q) {
            a += red[0][q * nb + tid];
            b += red[1][q * nb + tid];
        }
        partial[(static_cast<std::int64_t>(blockIdx.x) * 2 + 0) * nb + tid] = a;
        partial[(static_cast<std::int64_t>(blockIdx.x) * 2 + 1) * nb + tid] = b;
    }
}

// column sums of the per-CTA partials: 256 threads = (column, part) with the
// parts summed in a fixed order (deterministic)
__global__ void k_norm_reduce(const double* __restrict__ partial, int nparts, int nb, double* out_r, double* out_x) {
    __shared__ double red[2][256];
    const int tid = threadIdx.x;
    const int P = blockDim.x / nb;  // parts
    const int c = tid % nb, q = tid / nb;
    double a = 0.0, b = 0.0;
    if (q < P)
        for (int p = q; p < nparts; p += P) {
            a += partial[(static_cast<std::int64_t>(p) * 2 + 0) * nb + c];
            b += partial[(static_cast<std::int64_t>(p) * 2 + 1) * nb + c];
        }
    red[0][tid] = a;
    red[1][tid] = b;
    __syncthreads();
    if (tid < nb) {
        double sa = 0.0, sb = 0.0;
        for (int k = 0; k < P; ++k) {
            sa += red[0][k * nb + tid];
            sb += red[1][k * nb + tid];
        }
        if (out_r) out_r[tid] = sa;
        if (out_x) out_x[tid] = sb;
    }
}

__global__ void k_scale_columns(double* a, double* ha, const double* norm2, int nb, std::int64_t n, const Status* st) {
    if (!st->not_pd) return;
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < n * nb;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(e % nb);
        const double an = sqrt(norm2[c]);
        if (an > 1e-300) {
            a[e] *= 1.0 / an;
            ha[e] *= 1.0 / an;
        }
    }
}

__global__ void k_rr_assemble(const double* __restrict__ blocks, int nb, int nblk, double* G, double* O) {
    const int dim = nblk * nb;
    const int ng = nblk * (nblk + 1) / 2;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < dim * dim; e += gridDim.x * blockDim.x) {
        const int j = e / dim, i = e % dim;
        const int li = i >= j ? i : j, lj = i >= j ? j : i;  // lower-triangle source (mirror_lower)
        const int bi = li / nb, bj = lj / nb;
        const int bidx = bi == 0 ? 0 : bi == 1 ? 1 + bj : 3 + bj;  // (0,0) (1,0) (1,1) (2,0) (2,1) (2,2)
        const int oi = li - bi * nb, oj = lj - bj * nb;
        G[j * dim + i] = blocks[static_cast<std::int64_t>(bidx) * nb * nb + oj * nb + oi];
        O[j * dim + i] = blocks[static_cast<std::int64_t>(ng + bidx) * nb * nb + oj * nb + oi];
    }
}

int grid_rows(Ctx* ctx, std::int64_t n, int per) {
    return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * 4, (n + per - 1) / per)));
}

}  // namespace

std::int64_t gram_partials_len(int nb, int npairs, int num_sms) {
    const int nblk = (nb + 3) / 4, nbp8 = (nb + 7) / 8;
    return std::max(static_cast<std::int64_t>(num_sms) * 6 * npairs * nblk * nblk * 16,
                    static_cast<std::int64_t>(4 * num_sms) * npairs * nbp8 * nbp8 * 64);
}

void gram(Ctx* ctx, const GramJob& job, std::int64_t n, double* partials, std::int64_t partials_len, cudaStream_t s) {
    if (job.npairs < 1 || job.npairs > 12 || job.nb < 1 || job.nb > 64) fail(BE_ERR_BAD_PARAMS, "gram: bad job");
    GramDev g{};
    g.npairs = job.npairs;
    g.nb = job.nb;
    g.nblk = (job.nb + 3) / 4;
    g.ncombo = job.npairs * g.nblk * g.nblk;
    g.nd = 0;
    auto idx_of = [&](const double* p) {
        for (int d = 0; d < g.nd; ++d)
            if (g.panel[d] == p) return d;
        g.panel[g.nd] = p;
        return g.nd++;
    };
    GramOut o{};
    for (int p = 0; p < job.npairs; ++p) {
        g.ia[p] = idx_of(job.a[p]);
        g.ib[p] = idx_of(job.b[p]);
        o.out[p] = job.out[p];
        o.sym[p] = job.sym[p];
    }
    static const bool gram_r_on = [] {
        const char* e = std::getenv("BE_GRAM_R");
        return !(e && e[0] == '0');
    }();
    if (gram_r_on && (job.nb == 8 || job.nb == 16) && job.npairs <= 2 && g.nd <= 2 && n > 0) {  // register-direct
        const int grid = static_cast<int>(std::max<std::int64_t>(
            1, std::min<std::int64_t>((g.nd == 2 ? 1 : 2) * ctx->num_sms, (n + 31) / 32)));
        const std::size_t sm = static_cast<std::size_t>(16) * job.npairs * job.nb * job.nb * sizeof(double);
        if (static_cast<std::int64_t>(grid) * job.npairs * job.nb * job.nb <= partials_len) {
#define BE_GRAMR(NBB, ND, NPR)                                                \
    do {                                                                      \
        ensure_dyn_smem(k_gram_r<NBB, ND, NPR>, sm);                          \
        k_gram_r<NBB, ND, NPR><<<grid, 512, sm, s>>>(g, n, partials);         \
    } while (0)
#define BE_GRAMR_NB(NBB)                                                      \
    if (g.nd == 1) {                                                          \
        if (job.npairs == 1) BE_GRAMR(NBB, 1, 1); else BE_GRAMR(NBB, 1, 2);   \
    } else {                                                                  \
        if (job.npairs == 1) BE_GRAMR(NBB, 2, 1); else BE_GRAMR(NBB, 2, 2);   \
    }
            if (job.nb == 8) {
                BE_GRAMR_NB(1)
            } else {
                BE_GRAMR_NB(2)
            }
#undef BE_GRAMR_NB
#undef BE_GRAMR
            const int total = job.npairs * job.nb * job.nb;
            k_gram_reduce_m<<<(total * 32 + 255) / 256, 256, 0, s>>>(g, o, grid, partials);
            BE_CUDA(cudaGetLastError());
            ctx->launches += 2;
            return;
        }
    }
    if (job.nb % 8 == 0 && job.nb <= 32 && n > 0) {  // tensor-core kernel
        GramM q{};
        const int nbb = job.nb / 8, B = nbb * nbb;
        q.pw = std::max(1, std::min(job.npairs, 16 / B));  // <= 16 blocks per warp
        q.ngrp = (job.npairs + q.pw - 1) / q.pw;
        int ngrp = 1;
        while (ngrp < q.ngrp) ngrp *= 2;
        if (ngrp <= 8) {
            q.ngrp = ngrp;
            q.pw = (job.npairs + ngrp - 1) / ngrp;
            q.rg = 8 / ngrp;
            q.rs = job.nb + 4;
            q.R = std::max(16, std::min(256, (BE_GRAM_STAGE_KB * 1024 / (g.nd * q.rs * 8)) & ~3));
            q.ps = q.R * q.rs;
            q.ss = g.nd * q.ps;
            const std::size_t sm = std::max(static_cast<std::size_t>(kGG) * q.ss,
                                            static_cast<std::size_t>(job.npairs) * job.nb * job.nb) * 8;
            const std::int64_t nchunks = (n + q.R - 1) / q.R;
            const int nparts = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(BE_GRAM_CTAS * ctx->num_sms, nchunks)));
            if (static_cast<std::int64_t>(nparts) * job.npairs * job.nb * job.nb <= partials_len) {
#define BE_GRAMM(NBB)                                                     \
    do {                                                                  \
        ensure_dyn_smem(k_gram_m<NBB>, sm);                               \
        k_gram_m<NBB><<<nparts, 256, sm, s>>>(g, q, n, partials);         \
    } while (0)
                switch (nbb) {
                    case 1: BE_GRAMM(1); break;
                    case 2: BE_GRAMM(2); break;
                    case 3: BE_GRAMM(3); break;
                    default: BE_GRAMM(4); break;
                }
#undef BE_GRAMM
                const int total = job.npairs * job.nb * job.nb;
                k_gram_reduce_m<<<(total * 32 + 255) / 256, 256, 0, s>>>(g, o, nparts, partials);
                BE_CUDA(cudaGetLastError());
                ctx->launches += 2;
                return;
            }
        }
    }
    if (job.nb % 8 == 0 && n > 0) {  // streamed kernel (whole 8-column blocks, 16-byte rows)
        GramS q{};
        const int nbp = (job.nb + 7) / 8 * 8;
        q.bpr = nbp / 8;
        q.bpc = nbp / 4;
        q.tasks = job.npairs * q.bpr * q.bpc;
        if (q.tasks <= 512) {
            q.groups = 512 / q.tasks;
            // R rows per chunk: a stage of up to ~40 KB
            q.rs = job.nb + 2;
            q.R = std::max(16, std::min(256, (40 * 1024 / (g.nd * q.rs * 8)) & ~1));
            q.ps = q.R * q.rs + 2;
            q.ss = g.nd * q.ps;
            const std::size_t red = static_cast<std::size_t>(32 % q.tasks == 0 ? 16 : 1) * q.tasks * 32;
            const std::size_t sm = std::max(static_cast<std::size_t>(kGG) * q.ss, red) * 8;
            const std::int64_t nchunks = (n + q.R - 1) / q.R;
            const int nparts = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms, nchunks)));
            if (static_cast<std::int64_t>(nparts) * q.tasks * 32 <= partials_len) {
                ensure_dyn_smem(k_gram_s, sm);
                k_gram_s<<<nparts, 512, sm, s>>>(g, q, n, partials);
                const int total = job.npairs * job.nb * job.nb;
                k_gram_reduce8<<<(total * 32 + 255) / 256, 256, 0, s>>>(g, o, q, nparts, partials);
                BE_CUDA(cudaGetLastError());
                ctx->launches += 2;
                return;
            }
        }
    }
    int nparts = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * 6, (n + 255) / 256)));
    while (nparts > 1 && static_cast<std::int64_t>(nparts) * g.ncombo * 16 > partials_len) nparts /= 2;
    const int cpb = std::min(g.ncombo, kT);
    const int rg = kT / cpb;
    const std::size_t sm = std::max(static_cast<std::size_t>(g.nd) * kGramRows * g.nblk * 4,
                                    static_cast<std::size_t>(rg) * cpb * 16) * sizeof(double);
    ensure_dyn_smem(k_gram_partial, sm);
    dim3 grid(nparts, (g.ncombo + cpb - 1) / cpb);
    k_gram_partial<<<grid, kT, sm, s>>>(g, n, partials, cpb);
    BE_CUDA(cudaGetLastError());
    const int total = job.npairs * job.nb * job.nb;
    k_gram_reduce<<<(total * 32 + 255) / 256, 256, 0, s>>>(g, o, nparts, partials);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 2;
}

bool mix(Ctx* ctx, const MixJob& job, std::int64_t n, cudaStream_t s) {
    if (job.nout < 1 || job.nout > 4 || job.nb < 1 || job.nb > 64) fail(BE_ERR_BAD_PARAMS, "mix: bad job");
    MixDev m{};
    m.nb = job.nb;
    m.nout = job.nout;
    m.ncoef = 0;
    auto cidx = [&](const double* c, int ld) {
        for (int i = 0; i < m.ncoef; ++i)
            if (m.coef[i] == c && m.ld[i] == ld) return i;
        m.coef[m.ncoef] = c;
        m.ld[m.ncoef] = ld;
        return m.ncoef++;
    };
    for (int o = 0; o < job.nout; ++o) {
        const MixOut& J = job.out[o];
        auto& O = m.out[o];
        O.y = J.y;
        O.accumulate = J.accumulate;
        O.nterms = J.nterms;
        O.add_from = J.add_from;
        if (J.add_from >= o) fail(BE_ERR_BAD_PARAMS, "mix: add_from must name an earlier output");
        for (int t = 0; t < J.nterms; ++t) {
            O.src[t] = J.term[t].src;
            O.ci[t] = cidx(J.term[t].coef, J.term[t].ldc > 0 ? J.term[t].ldc : job.nb);
            O.sign[t] = J.term[t].neg ? -1.0 : 1.0;
        }
    }
    MixSrc ms{};
    auto sidx = [&](const double* p) {
        int q = 0;
        while (q < ms.nsrc && ms.src[q] != p) ++q;
        if (q == ms.nsrc) {
            if (ms.nsrc == 6) fail(BE_ERR_BAD_PARAMS, "mix: more than 6 distinct sources");
            ms.src[ms.nsrc++] = p;
        }
        return q;
    };
    for (int o = 0; o < m.nout; ++o) {
        for (int t = 0; t < m.out[o].nterms; ++t) m.out[o].si[t] = sidx(m.out[o].src[t]);
        m.out[o].add_si = job.out[o].add_src ? sidx(job.out[o].add_src) : -1;
        m.out[o].acc_si = job.out[o].accumulate ? sidx(job.out[o].y) : -1;
    }
    const int nblk = (job.nb + 3) / 4;
    {  // tensor-core path: nb in {8, 16}, <= 4 term slots, no add_from, every output has a term
        MixT mt{};
        bool ok = (job.nb == 8 || job.nb == 16 || job.nb == 24 || job.nb == 32);
        for (int o = 0; o < m.nout && ok; ++o) {
            if (m.out[o].add_from >= 0 || m.out[o].nterms < 1 || mt.nq + m.out[o].nterms > 4) {
                ok = false;
                break;
            }
            for (int t = 0; t < m.out[o].nterms; ++t) {
                mt.qo[mt.nq] = o;
                mt.qs[mt.nq] = m.out[o].si[t];
                mt.last[mt.nq] = t + 1 == m.out[o].nterms;
                ++mt.nq;
            }
        }
        static const bool mix_r_on = [] {
            const char* e = std::getenv("BE_MIX_R");
            return !(e && e[0] == '0');
        }();
        if (ok && mix_r_on && (job.nb == 8 || job.nb == 16)) {  // register-direct kernel
            MixR r{};
            r.nq = mt.nq;
            int nl = mt.nq;
            for (int q = 0; q < mt.nq; ++q) {
                r.src[q] = ms.src[mt.qs[q]];
                r.qo[q] = mt.qo[q];
                r.last[q] = mt.last[q];
            }
            bool fits = true;
            for (int o = 0; o < m.nout; ++o) {
                r.y[o] = m.out[o].y;
                r.accl[o] = r.addl[o] = -1;
                if (m.out[o].accumulate) {
                    if (nl == 4) fits = false;
                    else r.src[r.accl[o] = nl++] = m.out[o].y;
                }
                if (m.out[o].add_si >= 0) {
                    if (nl == 4) fits = false;
                    else r.src[r.addl[o] = nl++] = ms.src[m.out[o].add_si];
                }
            }
            static const bool mix_gram_on = [] {
                const char* e = std::getenv("BE_MIX_GRAM");
                return !(e && e[0] == '0');
            }();
            bool gram = false;
            r.gal = -1;
            if (fits && mix_gram_on && job.gram_out && job.gram_a < 0 && job.gram_a_src) {
                if (nl < 4) r.src[r.gal = nl++] = job.gram_a_src;  // else no room: no Gram
            }
            if (fits && mix_gram_on && job.gram_out && ((job.gram_a >= 0 && job.gram_a < m.nout) || r.gal >= 0)) {
                r.ga = job.gram_a;
                r.gbo = job.gram_b;
                r.gbl = -1;
                if (job.gram_b < 0)
                    for (int o = 0; o < m.nout; ++o)
                        if (r.addl[o] >= 0 && r.src[r.addl[o]] == job.gram_b_src) r.gbl = r.addl[o];
                r.gpart = job.gram_partials;
                gram = (r.gbo >= 0 && r.gbo < m.nout) || r.gbl >= 0;
            }
            bool res = false;  // the residual epilogue rides on the Gram kernel
            if (gram && job.res_out) {
                r.rx = r.rhx = -1;
                for (int q = 0; q < r.nq; ++q) {
                    if (r.src[q] == job.res_x) r.rx = q;
                    if (r.src[q] == job.res_hx) r.rhx = q;
                }
                r.theta = job.res_theta;
                r.rout = job.res_out;
                res = r.rx >= 0 && r.rhx >= 0;
                if (!res) gram = false;  // both or neither: the caller then forms them apart
            } else if (job.res_out) {
                gram = false;
            }
            if (fits) {
                const std::int64_t nblk = (n + 7) / 8;
                int grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * 4, (nblk + 7) / 8)));
                if (gram) {
                    const int per_sm = nl <= 2 && !res ? 3 : 2;  // the kernel's resident CTAs (launch bounds)
                    grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * per_sm, (nblk + 7) / 8)));
                    const std::int64_t need = static_cast<std::int64_t>(grid) * job.nb * (job.nb + (res ? 2 : 0));
                    if (need > job.gram_partials_len) gram = false;
                    r.rpart = job.gram_partials + static_cast<std::int64_t>(grid) * job.nb * job.nb;
                }
                if (gram) {
#define BE_MIXG(NBB, RSV)                                                        \
    switch (nl) {                                                               \
        case 1: k_mix_r<NBB, 1, true, RSV><<<grid, 256, 0, s>>>(m, r, n); break; \
        case 2: k_mix_r<NBB, 2, true, RSV><<<grid, 256, 0, s>>>(m, r, n); break; \
        case 3: k_mix_r<NBB, 3, true, RSV><<<grid, 256, 0, s>>>(m, r, n); break; \
        default: k_mix_r<NBB, 4, true, RSV><<<grid, 256, 0, s>>>(m, r, n); break; \
    }
                    if (job.nb == 8) {
                        if (res) { BE_MIXG(1, true) } else { BE_MIXG(1, false) }
                    } else {
                        if (res) { BE_MIXG(2, true) } else { BE_MIXG(2, false) }
                    }
#undef BE_MIXG
                    if (res) {
                        k_norm_reduce<<<1, 256, 0, s>>>(r.rpart, grid, job.nb, job.res_rn2, job.res_xn2);
                        ++ctx->launches;
                    }
                    GramDev gd{};
                    gd.npairs = 1;
                    gd.nb = job.nb;
                    GramOut go{};
                    go.out[0] = job.gram_out;
                    go.sym[0] = job.gram_sym;
                    k_gram_reduce_m<<<(job.nb * job.nb * 32 + 255) / 256, 256, 0, s>>>(gd, go, grid, job.gram_partials);
                    BE_CUDA(cudaGetLastError());
                    ctx->launches += 2;
                    return true;
                }
#define BE_MIXR(NBB, L) k_mix_r<NBB, L><<<grid, 256, 0, s>>>(m, r, n)
#define BE_MIXR_L(NBB)                 \
    switch (nl) {                      \
        case 1: BE_MIXR(NBB, 1); break; \
        case 2: BE_MIXR(NBB, 2); break; \
        case 3: BE_MIXR(NBB, 3); break; \
        default: BE_MIXR(NBB, 4); break; \
    }
                if (job.nb == 8) {
                    BE_MIXR_L(1)
                } else {
                    BE_MIXR_L(2)
                }
#undef BE_MIXR_L
#undef BE_MIXR
                BE_CUDA(cudaGetLastError());
                ++ctx->launches;
                return job.gram_out == nullptr;
            }
        }
        const bool bsm = job.nb > 16;
        const std::size_t smt =2 * static_cast<std::size_t>(ms.nsrc) * kMixPRows * (job.nb + 4) * sizeof(double) +
                                (bsm ? 4 * static_cast<std::size_t>(job.nb / 4) * (job.nb / 8) * 32 * sizeof(double) : 0);
        if (ok && smt <= 200 * 1024) {
            const int grid = static_cast<int>(
                std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * 2, (n + kMixPRows - 1) / kMixPRows)));
            if (job.nb == 8) {
                ensure_dyn_smem(k_mix_t<1>, smt);
                k_mix_t<1><<<grid, kT, smt, s>>>(m, ms, mt, n);
            } else if (job.nb == 16) {
                ensure_dyn_smem(k_mix_t<2>, smt);
                k_mix_t<2><<<grid, kT, smt, s>>>(m, ms, mt, n);
            } else if (job.nb == 24) {
                ensure_dyn_smem(k_mix_t<3, true>, smt);
                k_mix_t<3, true><<<grid, kT, smt, s>>>(m, ms, mt, n);
            } else {
                ensure_dyn_smem(k_mix_t<4, true>, smt);
                k_mix_t<4, true><<<grid, kT, smt, s>>>(m, ms, mt, n);
            }
            BE_CUDA(cudaGetLastError());
            ++ctx->launches;
            return job.gram_out == nullptr;
        }
    }
    const std::size_t smp = (((static_cast<std::size_t>(m.ncoef) * job.nb * nblk * 4 + 1) & ~std::size_t{1}) +
                             2 * static_cast<std::size_t>(ms.nsrc) * kMixPRows * (job.nb + 2)) * sizeof(double);
    if (job.nb % 2 == 0 && kT % (job.nb / 2) == 0 && smp <= 220 * 1024 / BE_MIXP_CTAS) {  // pipelined
        ensure_dyn_smem(k_mix_p, smp);
        const int grid = static_cast<int>(std::max<std::int64_t>(
            1, std::min<std::int64_t>(ctx->num_sms * BE_MIXP_CTAS, (n + kMixPRows - 1) / kMixPRows)));
        k_mix_p<<<grid, kT, smp, s>>>(m, ms, n);
        BE_CUDA(cudaGetLastError());
        ++ctx->launches;
        return job.gram_out == nullptr;
    }
    const std::size_t sm = (static_cast<std::size_t>(m.ncoef) * job.nb * nblk * 4 +
                            static_cast<std::size_t>(ms.nsrc) * kMixRows * (job.nb + 1)) * sizeof(double);
    ensure_dyn_smem(k_mix, sm);
    const int grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * BE_MIX_CTAS, (n + kMixRows - 1) / kMixRows)));
    k_mix<<<grid, kT, sm, s>>>(m, ms, nullptr, n);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
    return job.gram_out == nullptr;
}

void trsm(Ctx* ctx, double* w0, double* w1, const double* R, int nb, std::int64_t n, Status* st, int skip_if_rank,
          int skip_if_notpd, cudaStream_t s) {
    static const bool trsm_r_on = [] {
        const char* e = std::getenv("BE_TRSM_R");
        return !(e && e[0] == '0');
    }();
    if (trsm_r_on && (nb == 8 || nb == 16) && n > 0) {  // warp-independent kernel
        const int np = w1 ? 2 : 1;
        const std::size_t sm = static_cast<std::size_t>(kTrsmWarps) * 2 * np * 32 * (nb + 2) * sizeof(double);
        const int per_sm = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(6, (220u * 1024) / (sm + 2048))));
        const std::int64_t nblk = (n + 31) / 32;
        const int grid = static_cast<int>(std::max<std::int64_t>(
            1, std::min<std::int64_t>(static_cast<std::int64_t>(per_sm) * ctx->num_sms, (nblk + kTrsmWarps - 1) / kTrsmWarps)));
        if (nb == 8) {
            ensure_dyn_smem(k_trsm_r<8>, sm);
            k_trsm_r<8><<<grid, kTrsmWarps * 32, sm, s>>>(w0, w1, R, n, st, skip_if_rank, skip_if_notpd, nullptr);
        } else {
            ensure_dyn_smem(k_trsm_r<16>, sm);
            k_trsm_r<16><<<grid, kTrsmWarps * 32, sm, s>>>(w0, w1, R, n, st, skip_if_rank, skip_if_notpd, nullptr);
        }
        BE_CUDA(cudaGetLastError());
        ++ctx->launches;
        return;
    }
    if (nb % 2 == 0 && nb <= 32 && n > 0) {  // streamed
        const int np = w1 ? 2 : 1;
        const int Rr = 256 / np;
        const int ps = Rr * (nb + 2) + 2;
        const std::size_t sm = static_cast<std::size_t>(kGS) * np * ps * sizeof(double);
        const std::int64_t nchunks = (n + Rr - 1) / Rr;
        const int grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(2 * ctx->num_sms, nchunks)));
#define BE_TRSMS(NBP)                                                                                         \
    do {                                                                                                      \
        ensure_dyn_smem(k_trsm_s<NBP>, sm);                                                                   \
        k_trsm_s<NBP><<<grid, 256, sm, s>>>(w0, w1, R, nb, n, st, skip_if_rank, skip_if_notpd, Rr, ps);       \
    } while (0)
        if (nb <= 8) BE_TRSMS(8);
        else if (nb <= 16) BE_TRSMS(16);
        else BE_TRSMS(32);
#undef BE_TRSMS
        BE_CUDA(cudaGetLastError());
        ++ctx->launches;
        return;
    }
#define BE_TRSM(NBP)                                                                                              \
    k_trsm<NBP><<<static_cast<int>(std::max<std::int64_t>(                                                        \
                      1, std::min<std::int64_t>(ctx->num_sms * 4, (n + trsm_rows<NBP>() - 1) / trsm_rows<NBP>()))), \
                  kT, 0, s>>>(w0, w1, R, nb, n, st, skip_if_rank, skip_if_notpd)
    if (nb <= 8)
        BE_TRSM(8);
    else if (nb <= 16)
        BE_TRSM(16);
    else if (nb <= 32)
        BE_TRSM(32);
    else if (nb <= 64)
        BE_TRSM(64);
    else
        fail(BE_ERR_BAD_PARAMS, "trsm: nb > 64");
#undef BE_TRSM
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

bool trsm_gram(Ctx* ctx, double* w, const double* R, int nb, std::int64_t n, Status* st, double* gram_out,
               double* partials, std::int64_t partials_len, cudaStream_t s) {
    static const bool on = [] {
        const char* e1 = std::getenv("BE_TRSM_R");
        const char* e2 = std::getenv("BE_TRSM_GRAM");
        return !(e1 && e1[0] == '0') && !(e2 && e2[0] == '0');
    }();
    if (!on || !(nb == 8 || nb == 16) || n <= 0) return false;
    const std::size_t sm = static_cast<std::size_t>(kTrsmWarps) * 2 * 32 * (nb + 2) * sizeof(double);
    const int per_sm = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(6, (220u * 1024) / (sm + 2048))));
    const std::int64_t nblk = (n + 31) / 32;
    const int grid = static_cast<int>(std::max<std::int64_t>(
        1, std::min<std::int64_t>(static_cast<std::int64_t>(per_sm) * ctx->num_sms, (nblk + kTrsmWarps - 1) / kTrsmWarps)));
    if (static_cast<std::int64_t>(grid) * nb * nb > partials_len) return false;
    if (nb == 8) {
        ensure_dyn_smem(k_trsm_r<8>, sm);
        k_trsm_r<8><<<grid, kTrsmWarps * 32, sm, s>>>(w, nullptr, R, n, st, 1, 0, partials);
    } else {
        ensure_dyn_smem(k_trsm_r<16>, sm);
        k_trsm_r<16><<<grid, kTrsmWarps * 32, sm, s>>>(w, nullptr, R, n, st, 1, 0, partials);
    }
    GramDev g{};
    g.npairs = 1;
    g.nb = nb;
    GramOut o{};
    o.out[0] = gram_out;
    o.sym[0] = 1;
    k_gram_reduce_m<<<(nb * nb * 32 + 255) / 256, 256, 0, s>>>(g, o, grid, partials);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 2;
    return true;
}

void qr_chol(Ctx* ctx, double* B, double* R, int nb, Status* st, cudaStream_t s) {
    k_qr_chol<<<1, 64, 0, s>>>(B, R, nb, st);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void chol_floored(Ctx* ctx, const double* B, double* R, int n, double rel_floor, Status* st, cudaStream_t s) {
    k_chol<<<1, 128, 0, s>>>(B, R, n, rel_floor, rel_floor > 0.0 ? 1 : 0, st);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void residual(Ctx* ctx, const double* hx, const double* x, const double* theta, double* r, int nb, std::int64_t n,
              double* partials, double* rnorm2, double* xnorm2, cudaStream_t s) {
    if (nb > kT) fail(BE_ERR_BAD_PARAMS, "residual: nb too large");
    const int grid = grid_rows(ctx, n, kT / nb * 64);
    k_residual<<<grid, kT, 0, s>>>(hx, x, theta, r, nb, n, partials, 0);
    k_norm_reduce<<<1, 256, 0, s>>>(partials, grid, nb, rnorm2, xnorm2);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 2;
}

void colnorm2(Ctx* ctx, const double* a, int nb, std::int64_t n, double* partials, double* out, cudaStream_t s) {
    const int grid = grid_rows(ctx, n, kT / nb * 64);
    k_residual<<<grid, kT, 0, s>>>(nullptr, a, nullptr, nullptr, nb, n, partials, 1);
    k_norm_reduce<<<1, 256, 0, s>>>(partials, grid, nb, nullptr, out);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 2;
}

void scale_columns(Ctx* ctx, double* a, double* ha, const double* norm2, int nb, std::int64_t n, const Status* st,
                   cudaStream_t s) {
    const int grid = grid_rows(ctx, n * nb, kT);
    k_scale_columns<<<grid, kT, 0, s>>>(a, ha, norm2, nb, n, st);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void rr_assemble(Ctx* ctx, const double* blocks, int nb, int nblk, double* G, double* O, cudaStream_t s) {
    const int dim = nblk * nb;
    k_rr_assemble<<<(dim * dim + 255) / 256, 256, 0, s>>>(blocks, nb, nblk, G, O);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void Sygv::ensure(Ctx* ctx, int nn) {
    if (!ctx->solver) BE_CUSOLVER(cusolverDnCreate(&ctx->solver));
    if (nn <= n) return;
    n = nn;
    R.reset(static_cast<index_t>(nn) * nn);
    M.reset(static_cast<index_t>(nn) * nn);
    w.reset(nn);
    info.reset(1);
    BE_CUSOLVER(cusolverDnDsyevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, nn, M.get(),
                                            nn, w.get(), &lwork));
    work.reset(std::max(lwork, 1) + static_cast<index_t>(nn) * nn);  // + Y scratch
}

void sygv_lowest(Ctx* ctx, Sygv& ws, double* A, const double* B, int n, int k, double pivot_floor, double* c,
                 double* d, Status* st, cudaStream_t s) {
    if (k < 1 || k > n) fail(BE_ERR_BAD_PARAMS, "sygv_lowest: k out of range");
    if (rr_eig_fits(n)) return sygv_small(ctx, A, B, n, k, pivot_floor, c, d, st, s);
    ws.ensure(ctx, n);
    chol_floored(ctx, B, ws.R.get(), n, pivot_floor, st, s);
    // M = R^-T A R^-1 (densela.hpp:366-390) as two cuBLAS triangular solves,
    // then symmetrised (identity after a failed Cholesky: the host discards it)
    if (!ctx->blas) {
        cublasHandle_t h = nullptr;
        if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) fail(BE_ERR_CUSOLVER, "cublasCreate failed");
        ctx->blas = h;
    }
    BE_CUDA(cudaMemcpyAsync(ws.M.get(), A, static_cast<std::size_t>(n) * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    const double one = 1.0;
    if (cublasSetStream(ctx->blas, s) != CUBLAS_STATUS_SUCCESS ||
        cublasDtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, n, n, &one,
                    ws.R.get(), n, ws.M.get(), n) != CUBLAS_STATUS_SUCCESS ||
        cublasDtrsm(ctx->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n, &one,
                    ws.R.get(), n, ws.M.get(), n) != CUBLAS_STATUS_SUCCESS)
        fail(BE_ERR_CUSOLVER, "cublasDtrsm failed");
    k_sym_or_identity<<<1, 256, 0, s>>>(ws.M.get(), n, st);
    BE_CUDA(cudaGetLastError());
    BE_CUSOLVER(cusolverDnSetStream(ctx->solver, s));
    int lw = 0;
    BE_CUSOLVER(cusolverDnDsyevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                            ws.M.get(), n, ws.w.get(), &lw));
    if (lw > ws.lwork) fail(BE_ERR_CUSOLVER, "syevd workspace grew");
    BE_CUSOLVER(cusolverDnDsyevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, ws.M.get(), n,
                                 ws.w.get(), ws.work.get(), ws.lwork, ws.info.get()));
    // C = R^-1 Q_k (densela.hpp:393-405), then normalize_column_signs
    BE_CUDA(cudaMemcpyAsync(c, ws.M.get(), static_cast<std::size_t>(n) * k * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (cublasDtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, k, &one,
                    ws.R.get(), n, c, n) != CUBLAS_STATUS_SUCCESS)
        fail(BE_ERR_CUSOLVER, "cublasDtrsm failed");
    k_sign_fix<<<1, 64, 0, s>>>(c, ws.w.get(), d, n, k, st);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 3;
}

}  // namespace dla
}  // namespace be
