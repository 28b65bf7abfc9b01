// Fused small generalized eigensolver for the Rayleigh-Ritz step, sm_100a.
//
// Replaces sygv_lowest (densela.hpp:357-407) + the pencil assembly of
// rayleigh_ritz (lobpcg.hpp:113-157) for dim = nblk * nb <= 64 with ONE
// single-CTA launch and no host round trip:
//   1. G, O from the 6 (3) lower Gram blocks, mirrored (place_block /
//      mirror_lower, lobpcg.hpp:89-97, 126-141);
//   2. O = R^T R, floored Cholesky (densela.hpp:155-175, floor 1e-10);
//   3. M = R^-T G R^-1 by forward / right substitution, symmetrised
//      (densela.hpp:366-390: the same per-element operation order);
//   4. eigen-decomposition of M by parallel cyclic Jacobi (round-robin
//      pairing, every 2 x 2 block of J^T M J updated by one thread) -- the
//      reference uses tred2 + tql2 (densela.hpp:180-325); both converge to
//      the eigenpairs to working precision, Jacobi with better relative
//      accuracy and no serial recurrence;
//   5. the k lowest, ascending; C = R^-1 Q_k (densela.hpp:393-405);
//      normalize_column_signs (densela.hpp:327-341).
// rayleigh_ritz's drop-P retry (lobpcg.hpp:380-396) is taken on the device:
// when O fails Cholesky with the P blocks, the 2-block sub-pencil (its
// leading 2nb x 2nb blocks) is solved instead, the P rows of C are zeroed
// (so P+ = W C2 exactly) and Status::rr_dropped = 1; a failure of the
// 2-block pencil sets Status::rr_dropped = 2 (BasisDegenerate, raised by the
// host at the iteration's single synchronisation point).
#include <cuda_runtime.h>

#include <cmath>

#include "densela.cuh"

namespace be {
namespace dla {

namespace {

constexpr int kN = 64;  // largest pencil
constexpr int kLD = kN + 1;  // leading dimension: columns 130 words apart, so a warp walking
                             // across columns hits every bank pair once (no 32-way conflicts)
#ifndef BE_RR_THREADS
#define BE_RR_THREADS 256  // 8 warps: every warp recomputes a round's rotations, so more warps cost issue slots
#endif
constexpr int kRT = BE_RR_THREADS;

struct Smem {
    double M[kN * kLD];  // column-major, leading dimension kLD
    double M2[kN * kLD];  // Jacobi: the other half of the ping-pong pair
    double R[kN * kLD];
    double V[kN * kLD];
    double w[kN];
    int pq[(kN - 1) * (kN / 2)][2];  // Jacobi pair table [round][pair]
    double floor_, red[kRT / 32];
    int fail, sweeps;
};

__device__ __forceinline__ int pair_of(int round, int i, int np, int& p, int& q) {
    // circle method over np (even) indices: index np-1 fixed
    const int m = np - 1;
    if (i == 0) {
        p = round % m;
        q = m;
    } else {
        p = (round + i) % m;
        q = (round - i + m) % m;
    }
    if (p > q) {
        const int t = p;
        p = q;
        q = t;
    }
    return 0;
}

__device__ double block_sum(double v, Smem& S) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += S.red[i];
    __syncthreads();
    return t;
}

// Floored Cholesky of S.R (holds O on entry, upper factor on exit; the
// strict lower part is cleared). Returns the failing pivot or -1.
__device__ int chol_floored_smem(Smem& S, int n, double rel_floor) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        double dmax = 0.0;
        for (int i = 0; i < n; ++i) dmax = fmax(dmax, fabs(S.R[i * kLD + i]));
        S.floor_ = rel_floor * fmax(dmax, 1e-300);
        S.fail = -1;
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        // pivot: O_jj - sum_k R_kj^2 (R_kj already in column j above the diagonal)
        if (tid == 0) {
            double piv = S.R[j * kLD + j];
            for (int k = 0; k < j; ++k) piv -= S.R[j * kLD + k] * S.R[j * kLD + k];
            if (!(piv > S.floor_)) S.fail = j;
            else S.R[j * kLD + j] = sqrt(piv);
        }
        __syncthreads();
        if (S.fail >= 0) return S.fail;
        const double rjj = S.R[j * kLD + j];
        for (int i = j + 1 + tid; i < n; i += blockDim.x) {  // R(j, i) = (O_ji - sum_k R_kj R_ki) / R_jj
            double s = S.R[i * kLD + j];
            for (int k = 0; k < j; ++k) s -= S.R[j * kLD + k] * S.R[i * kLD + k];
            S.R[i * kLD + j] = s / rjj;
        }
        __syncthreads();
    }
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int j = e / n, i = e % n;
        if (i > j) S.R[j * kLD + i] = 0.0;
    }
    __syncthreads();
    return -1;
}

// M <- R^-T M R^-1, symmetrised (densela.hpp:366-390). Column j of M is
// processed by its own threads; the inner sums run over t ascending exactly
// as the reference's loops.
__device__ void reduce_pencil(Smem& S, int n) {
    const int tid = threadIdx.x;
    // Y = R^-T G: for each column j, forward substitution down the rows
    for (int j = tid; j < n; j += blockDim.x)
        for (int i = 0; i < n; ++i) {
            double s = S.M[j * kLD + i];
            for (int t = 0; t < i; ++t) s -= S.R[i * kLD + t] * S.M[j * kLD + t];
            S.M[j * kLD + i] = s / S.R[i * kLD + i];
        }
    __syncthreads();
    // M = Y R^-1: for each row i, M(i, j) = (Y(i, j) - sum_{t<j} M(i, t) R(t, j)) / R(j, j)
    for (int i = tid; i < n; i += blockDim.x)
        for (int j = 0; j < n; ++j) {
            double s = S.M[j * kLD + i];
            for (int t = 0; t < j; ++t) s -= S.M[t * kLD + i] * S.R[j * kLD + t];
            S.M[j * kLD + i] = s / S.R[j * kLD + j];
        }
    __syncthreads();
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int j = e / n, i = e % n;
        if (i < j) {
            const double s = 0.5 * (S.M[j * kLD + i] + S.M[i * kLD + j]);
            S.M[j * kLD + i] = s;
            S.M[i * kLD + j] = s;
        }
    }
    __syncthreads();
}

// f64 reciprocal / reciprocal square root: the hardware approximation (~2^-23)
// refined by Newton steps (each doubles the correct bits), no special-case
// branches -- callers keep the arguments finite, positive and normal.
template <int STEPS>
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
    for (int i = 0; i < STEPS; ++i) y = fma(y, fma(-x, y, 1.0), y);
    return y;
}
template <int STEPS>
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
    for (int i = 0; i < STEPS; ++i) {
        const double hx = 0.5 * x;
        y = fma(y, fma(-hx * y, y, 0.5), y);  // y (3 - x y^2) / 2
    }
    return y;
}

// Parallel cyclic Jacobi on S.M (n x n, symmetric): S.V = eigenvectors,
// S.w = eigenvalues (unsorted). np = n rounded up to even (a zero pad index).
// Round-robin pairing (circle method), P = np / 2 disjoint pairs per round.
// Every warp computes all P rotations of a round itself (lane b: pair b) from
// the current M and writes its share of J^T M J into the other buffer of a
// ping-pong pair (the pairs partition the indices: every entry is written
// once per round), so a round costs one CTA barrier: rotations -> the warp's
// 2 x 2 blocks of J^T M J and rows of V J (operands of other pairs by
// shuffle) -> barrier -> swap. The rotation takes
// one square root, one division and one reciprocal square root:
//   d = a_qq - a_pp, t = sign(d) 2 a_pq / (|d| + sqrt(d^2 + 4 a_pq^2)),
//   c = 1 / sqrt(1 + t^2), s = t c
// (t the smaller root of t^2 + 2 (d / 2 a_pq) t - 1 = 0, as in the classical
// formula th = d / (2 a_pq), t = sign(th) / (|th| + sqrt(1 + th^2))).
__device__ void jacobi(Smem& S, int n) {
    const int tid = threadIdx.x;
    const int np = n + (n & 1);
    const int P = np / 2;
    const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    double* Mc = S.M;
    double* Mn = S.M2;
    for (int e = tid; e < np * np; e += blockDim.x) {
        const int j = e / np, i = e % np;
        S.V[j * kLD + i] = i == j ? 1.0 : 0.0;
        if (i >= n || j >= n) S.M[j * kLD + i] = 0.0;
    }
    for (int e = tid; e < (np - 1) * P; e += blockDim.x) {  // pair table [round][pair]
        const int round = e / P, i = e % P;
        int p, q;
        pair_of(round, i, np, p, q);
        S.pq[e][0] = p;
        S.pq[e][1] = q;
    }
    __syncthreads();
    for (int sweep = 0; sweep < 30; ++sweep) {
        // stop when the off-diagonal mass is at the rounding level (off <= 1e-14 ||M||_F: the
        // eigenvalues are then exact to second order, the vectors to ~1e-14 / gap)
        double off = 0.0, all = 0.0;
        for (int e = tid; e < n * n; e += blockDim.x) {
            const int j = e / n, i = e % n;
            const double v = Mc[j * kLD + i];
            all += v * v;
            if (i != j) off += v * v;
        }
        off = block_sum(off, S);
        all = block_sum(all, S);
        if (tid == 0) S.sweeps = sweep;
        if (off <= 1e-28 * all) break;
        for (int round = 0; round < np - 1; ++round) {
            int pb = 0, qb = 0;
            double cb = 1.0, sb = 0.0;
            if (lane < P) {  // this lane's pair of the round and its rotation (every warp alike)
                pb = S.pq[round * P + lane][0];
                qb = S.pq[round * P + lane][1];
                const double apq = Mc[qb * kLD + pb];
                if (qb < n) {
                    const double app = Mc[pb * kLD + pb], aqq = Mc[qb * kLD + qb];
                    if (apq * apq > 1e-34 * fabs(app * aqq) && fabs(apq) > 1e-300) {
                        const double d = aqq - app, h = 2.0 * apq;
                        // t needs only to annihilate a_pq to first order (the rotation stays exactly
                        // orthogonal through c, s): approximate sqrt / division refined once; c to
                        // full precision. The library routines outside the safe range.
                        const double q2 = d * d + h * h;
                        double t;
                        if (q2 > 1e-280 && q2 < 1e280) {
                            const double r = q2 * rsqrt_nr<1>(q2);
                            t = copysign(1.0, d) * h * rcp_nr<1>(fabs(d) + r);
                        } else {
                            t = fabs(d) > 1e150 ? apq / d : copysign(1.0, d) * h / (fabs(d) + sqrt(q2));
                        }
                        cb = rsqrt_nr<2>(1.0 + t * t);
                        sb = t * cb;
                    }
                }
            }
            // M <- J^T M J: 2 x 2 block (row pair a, column pair lane); V <- V J: rows of the warp,
            // pair lane. All of a warp's loads are issued before its first store (fully unrolled).
            constexpr int AMAX = (kN / 2 + kRT / 32 - 1) / (kRT / 32), IMAX = (kN + kRT / 32 - 1) / (kRT / 32);
            {
                int pa[AMAX], qa[AMAX];
                double ca[AMAX], sa[AMAX], mv[AMAX][4];
#pragma unroll
                for (int j = 0; j < AMAX; ++j) {
                    const int a = warp + j * nw;
                    pa[j] = __shfl_sync(0xffffffffu, pb, a & 31);
                    qa[j] = __shfl_sync(0xffffffffu, qb, a & 31);
                    ca[j] = __shfl_sync(0xffffffffu, cb, a & 31);
                    sa[j] = __shfl_sync(0xffffffffu, sb, a & 31);
                    if (a < P && lane < P) {
                        mv[j][0] = Mc[pb * kLD + pa[j]];
                        mv[j][1] = Mc[qb * kLD + pa[j]];
                        mv[j][2] = Mc[pb * kLD + qa[j]];
                        mv[j][3] = Mc[qb * kLD + qa[j]];
                    }
                }
#pragma unroll
                for (int j = 0; j < AMAX; ++j) {
                    const int a = warp + j * nw;
                    if (a < P && lane < P) {
                        // rows: p' = c p - s q, q' = s p + c q (J = [[c, s], [-s, c]])
                        const double r_pp = ca[j] * mv[j][0] - sa[j] * mv[j][2], r_pq = ca[j] * mv[j][1] - sa[j] * mv[j][3];
                        const double r_qp = sa[j] * mv[j][0] + ca[j] * mv[j][2], r_qq = sa[j] * mv[j][1] + ca[j] * mv[j][3];
                        Mn[pb * kLD + pa[j]] = cb * r_pp - sb * r_pq;  // columns
                        Mn[qb * kLD + pa[j]] = sb * r_pp + cb * r_pq;
                        Mn[pb * kLD + qa[j]] = cb * r_qp - sb * r_qq;
                        Mn[qb * kLD + qa[j]] = sb * r_qp + cb * r_qq;
                    }
                }
            }
            if (lane < P) {
                double vp[IMAX], vq[IMAX];
#pragma unroll
                for (int j = 0; j < IMAX; ++j) {
                    const int i = warp + j * nw;
                    if (i < np) {
                        vp[j] = S.V[pb * kLD + i];
                        vq[j] = S.V[qb * kLD + i];
                    }
                }
#pragma unroll
                for (int j = 0; j < IMAX; ++j) {
                    const int i = warp + j * nw;
                    if (i < np) {
                        S.V[pb * kLD + i] = cb * vp[j] - sb * vq[j];
                        S.V[qb * kLD + i] = sb * vp[j] + cb * vq[j];
                    }
                }
            }
            __syncthreads();
            double* const tmp = Mc;
            Mc = Mn;
            Mn = tmp;
        }
    }
    for (int i = tid; i < n; i += blockDim.x) S.w[i] = Mc[i * kLD + i];
    __syncthreads();
}

// k lowest eigenpairs -> c (n x k, leading dimension ldc, rows n..ldc zeroed),
// d (k); C = R^-1 Q_k, sign-normalised.
__device__ void back_transform(Smem& S, int n, int k, double* c, int ldc, double* d) {
    const int tid = threadIdx.x;
    // ascending order (ties by index): column rank of eigenpair i; Q_k -> S.M columns
    for (int i = tid; i < n; i += blockDim.x) {
        const double wi = S.w[i];
        int r = 0;
        for (int j = 0; j < n; ++j) r += (S.w[j] < wi) || (S.w[j] == wi && j < i);
        if (r < k) {
            for (int t = 0; t < n; ++t) S.M[r * kLD + t] = S.V[i * kLD + t];
            d[r] = wi;
        }
    }
    __syncthreads();
    // back substitution per column (densela.hpp:396-404: t ascending from i + 1)
    for (int j = tid; j < k; j += blockDim.x) {
        double* col = S.M + j * kLD;
        for (int i = n - 1; i >= 0; --i) {
            double s = col[i];
            for (int t = i + 1; t < n; ++t) s -= S.R[t * kLD + i] * col[t];
            col[i] = s / S.R[i * kLD + i];
        }
        // normalize_column_signs: the first largest-magnitude entry made positive
        int arg = 0;
        double best = -1.0;
        for (int i = 0; i < n; ++i) {
            const double v = fabs(col[i]);
            if (v > best) {
                best = v;
                arg = i;
            }
        }
        const double sg = col[arg] < 0.0 ? -1.0 : 1.0;
        for (int i = 0; i < ldc; ++i) c[j * ldc + i] = i < n ? sg * col[i] : 0.0;
    }
    __syncthreads();
}

// The assembled pencil of rayleigh_ritz (nblk blocks of nb) into S.M (G), S.R (O).
__device__ void assemble(Smem& S, const double* __restrict__ blocks, int nb, int nblk, int ng) {
    const int dim = nblk * nb;
    for (int e = threadIdx.x; e < dim * dim; e += blockDim.x) {
        const int j = e / dim, i = e % dim;
        const int li = i >= j ? i : j, lj = i >= j ? j : i;  // mirror_lower: the lower block is the source
        const int bi = li / nb, bj = lj / nb;
        const int bidx = bi == 0 ? 0 : bi == 1 ? 1 + bj : 3 + bj;
        const int oi = li - bi * nb, oj = lj - bj * nb;
        S.M[j * kLD + i] = blocks[static_cast<long long>(bidx) * nb * nb + oj * nb + oi];
        S.R[j * kLD + i] = blocks[static_cast<long long>(ng + bidx) * nb * nb + oj * nb + oi];
    }
    __syncthreads();
}

// blocks: ng G blocks then ng O blocks (ng = nblk (nblk + 1) / 2), nb x nb column-major.
// c: ldc x nb (ldc = nblk * nb), theta: nb, shifts: nb (theta[min(v, k - 1)]).
__global__ void __launch_bounds__(kRT, 1) k_rr_eig(const double* __restrict__ blocks, int nb, int nblk, int k,
                                                   double pivot_floor, double* __restrict__ c,
                                                   double* __restrict__ theta, double* __restrict__ shifts,
                                                   Status* st) {
    extern __shared__ __align__(16) unsigned char raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw);
    const int ng = nblk * (nblk + 1) / 2;
    const int ldc = nblk * nb;
#ifdef BE_RR_PROF
    long long t0 = clock64();
#endif
    int use = nblk;
    for (;;) {
        assemble(S, blocks, nb, use, ng);
        if (chol_floored_smem(S, use * nb, pivot_floor) < 0) break;
        if (use == 3) {  // drop P (lobpcg.hpp:380-396): the leading 2-block sub-pencil
            use = 2;
            continue;
        }
        if (threadIdx.x == 0) st->rr_dropped = 2;  // BasisDegenerate even without P
        return;
    }
    if (threadIdx.x == 0 && use != nblk) st->rr_dropped = 1;
    const int n = use * nb;
#ifdef BE_RR_PROF
    long long t1 = clock64();
#endif
    reduce_pencil(S, n);
#ifdef BE_RR_PROF
    long long t2 = clock64();
#endif
    jacobi(S, n);
#ifdef BE_RR_PROF
    long long t3 = clock64();
#endif
    back_transform(S, n, nb, c, ldc, theta);
#ifdef BE_RR_PROF
    long long t4 = clock64();
    if (threadIdx.x == 0)
        printf("[rr_eig] n %d chol %lld reduce %lld jacobi %lld (sweeps %d) back %lld cycles\n", n, t1 - t0, t2 - t1,
               t3 - t2, S.sweeps, t4 - t3);
#endif
    if (shifts)
        for (int v = threadIdx.x; v < nb; v += blockDim.x) shifts[v] = theta[min(v, k - 1)];
}

// Plain sygv_lowest on n x n column-major A, B (n <= 64): c (n x k), d (k).
__global__ void __launch_bounds__(kRT, 1) k_sygv_small(const double* __restrict__ A, const double* __restrict__ B, int n,
                                                       int k, double pivot_floor, double* __restrict__ c,
                                                       double* __restrict__ d, Status* st) {
    extern __shared__ __align__(16) unsigned char raw[];
    Smem& S = *reinterpret_cast<Smem*>(raw);
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int j = e / n, i = e % n;
        S.M[j * kLD + i] = A[j * n + i];
        S.R[j * kLD + i] = B[j * n + i];
    }
    __syncthreads();
    const int p = chol_floored_smem(S, n, pivot_floor);
    if (p >= 0) {
        if (threadIdx.x == 0) st->not_pd = p + 1;
        return;
    }
    if (threadIdx.x == 0) st->not_pd = 0;
    reduce_pencil(S, n);
    jacobi(S, n);
    __shared__ double dtmp[kN];
    back_transform(S, n, k, c, n, dtmp);
    for (int v = threadIdx.x; v < k; v += blockDim.x) d[v] = dtmp[v];
}

__global__ void k_latch_w_rank(Status* st) {
    if (st->rank_deficient) st->w_rank_first = 1;
}

}  // namespace

void latch_w_rank(Ctx* ctx, Status* st, cudaStream_t s) {
    k_latch_w_rank<<<1, 1, 0, s>>>(st);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

bool rr_eig_fits(int dim) { return dim <= kN; }

void rr_eig(Ctx* ctx, const double* blocks, int nb, int nblk, int k, double pivot_floor, double* c, double* theta,
            double* shifts, Status* st, cudaStream_t s) {
    if (nblk * nb > kN) fail(BE_ERR_BAD_PARAMS, "rr_eig: pencil larger than 64");
    ensure_dyn_smem(k_rr_eig, sizeof(Smem));
    k_rr_eig<<<1, kRT, sizeof(Smem), s>>>(blocks, nb, nblk, k, pivot_floor, c, theta, shifts, st);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void sygv_small(Ctx* ctx, const double* A, const double* B, int n, int k, double pivot_floor, double* c, double* d,
                Status* st, cudaStream_t s) {
    if (n > kN) fail(BE_ERR_BAD_PARAMS, "sygv_small: pencil larger than 64");
    ensure_dyn_smem(k_sygv_small, sizeof(Smem));
    k_sygv_small<<<1, kRT, sizeof(Smem), s>>>(A, B, n, k, pivot_floor, c, d, st);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

}  // namespace dla
}  // namespace be
