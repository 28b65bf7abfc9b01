// Device dense linear algebra for the LOBPCG iteration (see densela.cuh).
// Memory-bound fused panel kernels (Gram, row mixes, trsm, residual norms)
// and single-CTA kernels for the <= 3nb square projected problem; the
// symmetric eigen-decomposition itself is cuSOLVER syevd (no host fallback).
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>

#include "densela.cuh"

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

constexpr int kGramRows = 16;

// partial[blk][combo][16]: 4x4 register block of A_p^T B_p over this CTA's rows
__global__ void __launch_bounds__(kT) k_gram_partial(GramDev g, std::int64_t n, double* __restrict__ partial) {
    extern __shared__ double sp[];  // nd x kGramRows x nbp
    const int nbp = g.nblk * 4;
    const int combo = blockIdx.y * kT + threadIdx.x;
    int p = 0, bi = 0, bj = 0;
    if (combo < g.ncombo) {
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
            for (int e = threadIdx.x; e < kGramRows * nbp; e += kT) {
                const int r = e / nbp, v = e % nbp;
                dst[e] = (r < rows && v < g.nb) ? src[r * g.nb + v] : 0.0;
            }
        }
        __syncthreads();
        if (combo < g.ncombo) {
            const double* A = sp + g.ia[p] * kGramRows * nbp + bi * 4;
            const double* B = sp + g.ib[p] * kGramRows * nbp + bj * 4;
            for (int r = 0; r < rows; ++r) {
                const double a0 = A[r * nbp], a1 = A[r * nbp + 1], a2 = A[r * nbp + 2], a3 = A[r * nbp + 3];
                const double b0 = B[r * nbp], b1 = B[r * nbp + 1], b2 = B[r * nbp + 2], b3 = B[r * nbp + 3];
                acc[0] += a0 * b0; acc[1] += a1 * b0; acc[2] += a2 * b0; acc[3] += a3 * b0;
                acc[4] += a0 * b1; acc[5] += a1 * b1; acc[6] += a2 * b1; acc[7] += a3 * b1;
                acc[8] += a0 * b2; acc[9] += a1 * b2; acc[10] += a2 * b2; acc[11] += a3 * b2;
                acc[12] += a0 * b3; acc[13] += a1 * b3; acc[14] += a2 * b3; acc[15] += a3 * b3;
            }
        }
    }
    if (combo < g.ncombo) {
        double* out = partial + (static_cast<std::int64_t>(blockIdx.x) * g.ncombo + combo) * 16;
#pragma unroll
        for (int e = 0; e < 16; ++e) out[e] = acc[e];
    }
}

struct GramOut {
    double* out[12];
    int sym[12];
};

// out_p(i, j) = sum over CTAs in order; symmetrised pairs use both halves
__global__ void k_gram_reduce(GramDev g, GramOut o, int nparts, const double* __restrict__ partial) {
    const int nb = g.nb;
    const int total = g.npairs * nb * nb;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int p = e / (nb * nb), rem = e % (nb * nb);
        const int j = rem / nb, i = rem % nb;  // column-major (i, j)
        auto sum_at = [&](int ii, int jj) {
            const int combo = p * g.nblk * g.nblk + (ii / 4) * g.nblk + (jj / 4);
            const int el = (jj % 4) * 4 + (ii % 4);
            double s = 0.0;
            for (int b = 0; b < nparts; ++b) s += partial[(static_cast<std::int64_t>(b) * g.ncombo + combo) * 16 + el];
            return s;
        };
        if (o.sym[p]) {
            if (i > j) continue;
            if (i == j) {
                o.out[p][j * nb + i] = sum_at(i, j);
            } else {
                const double s = 0.5 * (sum_at(i, j) + sum_at(j, i));
                o.out[p][j * nb + i] = s;
                o.out[p][i * nb + j] = s;
            }
        } else {
            o.out[p][j * nb + i] = sum_at(i, j);
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
        int accumulate, nterms, add_from;
        const double* src[3];
        int ci[3];
        double sign[3];
    } out[4];
};

// thread = (row, 4-column block); coefficients transposed into smem
__global__ void __launch_bounds__(kT) k_mix(MixDev m, std::int64_t n) {
    extern __shared__ double ct[];  // ncoef x nb x nbp (row i, col j) row-major
    const int nb = m.nb, nblk = (nb + 3) / 4, nbp = nblk * 4;
    for (int c = 0; c < m.ncoef; ++c)
        for (int e = threadIdx.x; e < nb * nbp; e += kT) {
            const int i = e / nbp, j = e % nbp;
            ct[c * nb * nbp + e] = j < nb ? m.coef[c][j * m.ld[c] + i] : 0.0;
        }
    __syncthreads();
    const std::int64_t total = n * nblk;
    for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(kT) + threadIdx.x; t < total;
         t += static_cast<std::int64_t>(gridDim.x) * kT) {
        const std::int64_t r = t / nblk;
        const int j0 = static_cast<int>(t % nblk) * 4;
        double res[4][4];  // per output
        for (int o = 0; o < m.nout; ++o) {
            const auto& O = m.out[o];
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            double* y = O.y + r * nb;
            if (O.accumulate) {
                a0 = j0 < nb ? y[j0] : 0.0;
                a1 = j0 + 1 < nb ? y[j0 + 1] : 0.0;
                a2 = j0 + 2 < nb ? y[j0 + 2] : 0.0;
                a3 = j0 + 3 < nb ? y[j0 + 3] : 0.0;
            }
            for (int tt = 0; tt < O.nterms; ++tt) {
                const double* x = O.src[tt] + r * nb;
                const double* C = ct + O.ci[tt] * nb * nbp + j0;
                double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
                for (int i = 0; i < nb; ++i) {
                    const double xi = __ldg(x + i);
                    s0 += xi * C[i * nbp];
                    s1 += xi * C[i * nbp + 1];
                    s2 += xi * C[i * nbp + 2];
                    s3 += xi * C[i * nbp + 3];
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
            res[o][0] = a0;
            res[o][1] = a1;
            res[o][2] = a2;
            res[o][3] = a3;
            if (j0 < nb) y[j0] = a0;
            if (j0 + 1 < nb) y[j0 + 1] = a1;
            if (j0 + 2 < nb) y[j0 + 2] = a2;
            if (j0 + 3 < nb) y[j0 + 3] = a3;
        }
    }
}

// -------------------------------------------------------------------- trsm
template <int NBP>
__global__ void __launch_bounds__(kT) k_trsm(double* __restrict__ w0, double* __restrict__ w1,
                                            const double* __restrict__ Rg, int nb, std::int64_t n, Status* st,
                                            int skip_if_rank, int skip_if_notpd) {
    __shared__ double R[NBP * NBP];
    __shared__ int skip;
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
    for (std::int64_t r = blockIdx.x * static_cast<std::int64_t>(kT) + threadIdx.x; r < n;
         r += static_cast<std::int64_t>(gridDim.x) * kT) {
        for (int which = 0; which < 2; ++which) {
            double* w = which == 0 ? w0 : w1;
            if (!w) continue;
            double x[NBP];
#pragma unroll
            for (int j = 0; j < NBP; ++j)
                if (j < nb) x[j] = w[r * nb + j];
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
                if (j < nb) w[r * nb + j] = x[j];
        }
    }
}

// ------------------------------------------------------- small factorisations
// Block-cooperative floored Cholesky (densela.hpp:103-121 / 155-175): upper R
// with B = R^T R. floored=false reproduces cholesky() (pivot must be > 0).
// Returns the failing pivot index or -1. All threads of the CTA participate.
__device__ int dev_chol(const double* B, double* R, int n, double rel_floor, bool floored) {
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

// M = R^-T A R^-1 (densela.hpp:366-390); skipped after a failed Cholesky
__global__ void k_sygv_form(const double* A, const double* R, double* Y, double* M, int n, const Status* st) {
    if (st->not_pd) return;
    for (int j = threadIdx.x; j < n; j += blockDim.x)  // Y = R^-T A, column j
        for (int i = 0; i < n; ++i) {
            double s = A[j * n + i];
            for (int t = 0; t < i; ++t) s -= R[i * n + t] * Y[j * n + t];
            Y[j * n + i] = s / R[i * n + i];
        }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)  // M R = Y, row i
        for (int j = 0; j < n; ++j) {
            double s = Y[j * n + i];
            for (int t = 0; t < j; ++t) s -= M[t * n + i] * R[j * n + t];
            M[j * n + i] = s / R[j * n + j];
        }
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int j = e / n, i = e % n;
        if (i < j) {
            const double s = 0.5 * (M[j * n + i] + M[i * n + j]);
            M[j * n + i] = s;
            M[i * n + j] = s;
        }
    }
}

// C = R^-1 Q_k, then normalize_column_signs (densela.hpp:327-341, 393-405)
__global__ void k_sygv_back(const double* Q, const double* w, const double* R, double* C, double* d, int n, int k,
                            const Status* st) {
    if (st->not_pd) return;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        for (int i = n - 1; i >= 0; --i) {
            double s = Q[j * n + i];
            for (int t = i + 1; t < n; ++t) s -= R[t * n + i] * C[j * n + t];
            C[j * n + i] = s / R[i * n + i];
        }
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
    const int rpi = kT / nb;  // rows per iteration
    const int tid = threadIdx.x;
    const int c = tid % nb, rl = tid / nb;
    double s_r = 0.0, s_x = 0.0;
    if (rl < rpi) {
        const double th = mode == 0 ? theta[c] : 0.0;
        for (std::int64_t row = blockIdx.x * static_cast<std::int64_t>(rpi) + rl; row < n;
             row += static_cast<std::int64_t>(gridDim.x) * rpi) {
            const double xv = x[row * nb + c];
            s_x += xv * xv;
            if (mode == 0) {
                const double rv = hx[row * nb + c] - th * xv;
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

__global__ void k_norm_reduce(const double* __restrict__ partial, int nparts, int nb, double* out_r, double* out_x) {
    const int c = threadIdx.x;
    if (c >= nb) return;
    double a = 0.0, b = 0.0;
    for (int p = 0; p < nparts; ++p) {
        a += partial[(static_cast<std::int64_t>(p) * 2 + 0) * nb + c];
        b += partial[(static_cast<std::int64_t>(p) * 2 + 1) * nb + c];
    }
    if (out_r) out_r[c] = a;
    if (out_x) out_x[c] = b;
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
    const int nblk = (nb + 3) / 4;
    return static_cast<std::int64_t>(num_sms) * 2 * npairs * nblk * nblk * 16;
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
    int nparts = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * 2, (n + 63) / 64)));
    while (nparts > 1 && static_cast<std::int64_t>(nparts) * g.ncombo * 16 > partials_len) nparts /= 2;
    const std::size_t sm = static_cast<std::size_t>(g.nd) * kGramRows * g.nblk * 4 * sizeof(double);
    if (sm > 48 * 1024) BE_CUDA(cudaFuncSetAttribute(k_gram_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    dim3 grid(nparts, (g.ncombo + kT - 1) / kT);
    k_gram_partial<<<grid, kT, sm, s>>>(g, n, partials);
    BE_CUDA(cudaGetLastError());
    const int total = job.npairs * job.nb * job.nb;
    k_gram_reduce<<<(total + 255) / 256, 256, 0, s>>>(g, o, nparts, partials);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 2;
}

void mix(Ctx* ctx, const MixJob& job, std::int64_t n, cudaStream_t s) {
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
    const int nblk = (job.nb + 3) / 4;
    const std::size_t sm = static_cast<std::size_t>(m.ncoef) * job.nb * nblk * 4 * sizeof(double);
    if (sm > 48 * 1024) BE_CUDA(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    const std::int64_t total = n * nblk;
    const int grid = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(ctx->num_sms * 8, (total + kT - 1) / kT)));
    k_mix<<<grid, kT, sm, s>>>(m, n);
    BE_CUDA(cudaGetLastError());
    ++ctx->launches;
}

void trsm(Ctx* ctx, double* w0, double* w1, const double* R, int nb, std::int64_t n, Status* st, int skip_if_rank,
          int skip_if_notpd, cudaStream_t s) {
    const int grid = grid_rows(ctx, n, kT);
#define BE_TRSM(NBP) k_trsm<NBP><<<grid, kT, 0, s>>>(w0, w1, R, nb, n, st, skip_if_rank, skip_if_notpd)
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
    k_norm_reduce<<<1, 64, 0, s>>>(partials, grid, nb, rnorm2, xnorm2);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 2;
}

void colnorm2(Ctx* ctx, const double* a, int nb, std::int64_t n, double* partials, double* out, cudaStream_t s) {
    const int grid = grid_rows(ctx, n, kT / nb * 64);
    k_residual<<<grid, kT, 0, s>>>(nullptr, a, nullptr, nullptr, nb, n, partials, 1);
    k_norm_reduce<<<1, 64, 0, s>>>(partials, grid, nb, nullptr, out);
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
    ws.ensure(ctx, n);
    chol_floored(ctx, B, ws.R.get(), n, pivot_floor, st, s);
    double* Y = ws.work.get() + std::max(ws.lwork, 1);
    k_sygv_form<<<1, 128, 0, s>>>(A, ws.R.get(), Y, ws.M.get(), n, st);
    BE_CUDA(cudaGetLastError());
    BE_CUSOLVER(cusolverDnSetStream(ctx->solver, s));
    int lw = 0;
    BE_CUSOLVER(cusolverDnDsyevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                            ws.M.get(), n, ws.w.get(), &lw));
    if (lw > ws.lwork) fail(BE_ERR_CUSOLVER, "syevd workspace grew");
    BE_CUSOLVER(cusolverDnDsyevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, ws.M.get(), n,
                                 ws.w.get(), ws.work.get(), ws.lwork, ws.info.get()));
    k_sygv_back<<<1, 64, 0, s>>>(ws.M.get(), ws.w.get(), ws.R.get(), c, d, n, k, st);
    BE_CUDA(cudaGetLastError());
    ctx->launches += 3;
}

}  // namespace dla
}  // namespace be
