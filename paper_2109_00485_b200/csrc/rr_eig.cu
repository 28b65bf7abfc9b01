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
constexpr int kRT = 512;

struct Smem {
    double M[kN * kLD];  // column-major, leading dimension kLD
    double R[kN * kLD];
    double V[kN * kLD];
    double w[kN];
    double cs[kN / 2][2];
    int pq[kN / 2][2];
    double floor_, red[kRT / 32];
    int fail;
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

// Parallel cyclic Jacobi on S.M (n x n, symmetric): S.V = eigenvectors,
// S.w = eigenvalues (unsorted). np = n rounded up to even (a zero pad index).
__device__ void jacobi(Smem& S, int n) {
    const int tid = threadIdx.x;
    const int np = n + (n & 1);
    const int P = np / 2;
    for (int e = tid; e < np * np; e += blockDim.x) {
        const int j = e / np, i = e % np;
        S.V[j * kLD + i] = i == j ? 1.0 : 0.0;
        if (i >= n || j >= n) S.M[j * kLD + i] = 0.0;
    }
    __syncthreads();
    for (int sweep = 0; sweep < 30; ++sweep) {
        // stop when the off-diagonal mass is at the rounding level (off <= 1e-14 ||M||_F: the
        // eigenvalues are then exact to second order, the vectors to ~1e-14 / gap)
        double off = 0.0, all = 0.0;
        for (int e = tid; e < n * n; e += blockDim.x) {
            const int j = e / n, i = e % n;
            const double v = S.M[j * kLD + i];
            all += v * v;
            if (i != j) off += v * v;
        }
        off = block_sum(off, S);
        all = block_sum(all, S);
        if (off <= 1e-28 * all) break;
        for (int round = 0; round < np - 1; ++round) {
            if (tid < P) {  // this round's pairs and rotations
                int p, q;
                pair_of(round, tid, np, p, q);
                const double apq = S.M[q * kLD + p];
                double c = 1.0, s = 0.0;
                if (q < n && fabs(apq) > 1e-300 &&
                    fabs(apq) > 1e-17 * sqrt(fabs(S.M[p * kLD + p]) * fabs(S.M[q * kLD + q]))) {
                    const double app = S.M[p * kLD + p], aqq = S.M[q * kLD + q];
                    const double th = (aqq - app) / (2.0 * apq);
                    // t = tan of the rotation angle, the smaller root; 1 / (2 th) when th^2 would overflow
                    const double t = fabs(th) > 1e150 ? 0.5 / th
                                                      : (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
                    c = 1.0 / sqrt(1.0 + t * t);
                    s = t * c;
                }
                S.cs[tid][0] = c;
                S.cs[tid][1] = s;
                S.pq[tid][0] = p;
                S.pq[tid][1] = q;
            }
            __syncthreads();
            // M <- J^T M J: one 2 x 2 block per (warp row a, lane b); V <- V J: one row per warp step, lane b
            const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
            if (lane < P) {
                const int pb = S.pq[lane][0], qb = S.pq[lane][1];
                const double cb = S.cs[lane][0], sb = S.cs[lane][1];
                for (int a = warp; a < P; a += nw) {
                    const int pa = S.pq[a][0], qa = S.pq[a][1];
                    const double ca = S.cs[a][0], sa = S.cs[a][1];
                    const double m_pp = S.M[pb * kLD + pa], m_pq = S.M[qb * kLD + pa];
                    const double m_qp = S.M[pb * kLD + qa], m_qq = S.M[qb * kLD + qa];
                    // rows: p' = c p - s q, q' = s p + c q (J = [[c, s], [-s, c]])
                    const double r_pp = ca * m_pp - sa * m_qp, r_pq = ca * m_pq - sa * m_qq;
                    const double r_qp = sa * m_pp + ca * m_qp, r_qq = sa * m_pq + ca * m_qq;
                    S.M[pb * kLD + pa] = cb * r_pp - sb * r_pq;  // columns
                    S.M[qb * kLD + pa] = sb * r_pp + cb * r_pq;
                    S.M[pb * kLD + qa] = cb * r_qp - sb * r_qq;
                    S.M[qb * kLD + qa] = sb * r_qp + cb * r_qq;
                }
                for (int i = warp; i < np; i += nw) {
                    const double vp = S.V[pb * kLD + i], vq = S.V[qb * kLD + i];
                    S.V[pb * kLD + i] = cb * vp - sb * vq;
                    S.V[qb * kLD + i] = sb * vp + cb * vq;
                }
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < n; i += blockDim.x) S.w[i] = S.M[i * kLD + i];
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
    reduce_pencil(S, n);
    jacobi(S, n);
    back_transform(S, n, nb, c, ldc, theta);
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
