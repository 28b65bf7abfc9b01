// Device dense linear algebra of the LOBPCG iteration (densela.hpp, the panel
// parts of lobpcg.hpp). Tall-skinny n x nb panels are row-major fp64 device
// arrays; small matrices (<= 3 nb square) are column-major fp64 device arrays
// exactly like SmallDense (densela.hpp:19-47).
#pragma once

#include <cuda_runtime.h>

#include "device.hpp"

namespace be {
namespace dla {

// Device-side status words of one solve (read by the host at sync points).
struct Status {
    int qr_failures;       // Cholesky failures inside the current qr_of_transpose
    int rank_deficient;    // qr_of_transpose gave up (densela.hpp:426-439)
    int singular_tri;      // trsm_right_inv refused a factor (densela.hpp:135-136)
    int not_pd;            // last floored Cholesky failed (pivot + 1, 0 = ok)
    int ortho_fallback;    // orthonormalize_pair took the column-scaling path
    int rr_dropped;        // rr_eig: 1 dropped P (lobpcg.hpp:380-396), 2 failed without P too
    int w_rank_first;      // the first qr_of_transpose of W gave up (restart with a random W)
    int pad;
};

// Up to 12 Gram products A_p^T B_p (nb x nb, column-major) in one pass over
// the rows. sym[p]: symmetrise (gram(a, a), densela.hpp:90-97).
struct GramJob {
    int npairs;
    int nb;
    const double* a[12];
    const double* b[12];
    int sym[12];
    double* out[12];
};
void gram(Ctx* ctx, const GramJob& job, std::int64_t n, double* partials, std::int64_t partials_len, cudaStream_t s);
std::int64_t gram_partials_len(int nb, int npairs, int num_sms);

// Row-wise linear combinations of panels with small coefficient matrices
// (block_times_small(_add), densela.hpp:448-484). For every output o and row r:
//   y_o[r] = (accumulate ? y_o[r] : 0) + sum_t src_t[r] * (neg_t ? -C_t : C_t)
//            + (add_from >= 0 ? y_{add_from}[r] (already updated) : 0) + (add_src ? add_src[r] : 0)
struct MixTerm {
    const double* src;
    const double* coef;  // nb x nb column-major with leading dimension ldc (0 = nb)
    int neg;
    int ldc;
};
struct MixOut {
    double* y;
    int accumulate;
    int nterms;
    MixTerm term[3];
    int add_from;
    const double* add_src = nullptr;  // + add_src[r] (a panel added as is, after the terms)
};
struct MixJob {
    int nb;
    int nout;
    MixOut out[4];
    // optional Gram epilogue: gram_out = A^T B with A = output gram_a and B = output gram_b, or
    // (gram_b < 0) the panel gram_b_src, which must be one of the job's added panels; symmetrised
    // when gram_sym (gram, densela.hpp:90-97). Formed only by the register-direct kernel.
    double* gram_out = nullptr;
    int gram_a = -1, gram_b = -1, gram_sym = 0;
    const double* gram_a_src = nullptr;  // A = this panel (gram_a < 0), loaded as one more panel
    const double* gram_b_src = nullptr;
    double* gram_partials = nullptr;
    std::int64_t gram_partials_len = 0;
    // optional residual epilogue (with the Gram epilogue only; both or neither are formed):
    // res_out = res_hx - res_x diag(res_theta), column sums of its squares and of res_x's squares
    // into res_rn2 / res_xn2 (residual() below); res_x / res_hx must be term sources of the job
    double* res_out = nullptr;
    const double* res_x = nullptr;
    const double* res_hx = nullptr;
    const double* res_theta = nullptr;
    double* res_rn2 = nullptr;
    double* res_xn2 = nullptr;
};
// returns whether the requested Gram epilogue was formed (false: nothing about it was launched,
// the caller forms it separately; true when none was requested)
bool mix(Ctx* ctx, const MixJob& job, std::int64_t n, cudaStream_t s);

// W <- W R^{-1} for up to two panels (trsm_right_inv, densela.hpp:125-147);
// skipped when st->rank_deficient (skip_if_rank) / st->not_pd (skip_if_notpd).
void trsm(Ctx* ctx, double* w0, double* w1, const double* R, int nb, std::int64_t n, Status* st, int skip_if_rank,
          int skip_if_notpd, cudaStream_t s);
// trsm of one panel (skip_if_rank) that also forms gram_out = W'^T W' of the
// result on the way (CholQR's next pass); false when the fused kernel does
// not apply (nb other than 8 / 16) -- then nothing was launched.
bool trsm_gram(Ctx* ctx, double* w, const double* R, int nb, std::int64_t n, Status* st, double* gram_out,
               double* partials, std::int64_t partials_len, cudaStream_t s);

// Floored Cholesky with the qr_of_transpose retry logic (densela.hpp:412-445):
// B (nb x nb) -> R; updates st->qr_failures / st->rank_deficient.
void qr_chol(Ctx* ctx, double* B, double* R, int nb, Status* st, cudaStream_t s);
// Floored Cholesky (densela.hpp:155-175): st->not_pd = pivot + 1 on failure.
void chol_floored(Ctx* ctx, const double* B, double* R, int n, double rel_floor, Status* st, cudaStream_t s);

// R = HX - X diag(theta); rnorm2 / xnorm2 = per-column sums of squares
// (residual_block + column_norm, lobpcg.hpp:197-233).
void residual(Ctx* ctx, const double* hx, const double* x, const double* theta, double* r, int nb, std::int64_t n,
              double* partials, double* rnorm2, double* xnorm2, cudaStream_t s);
// column sums of squares of one panel
void colnorm2(Ctx* ctx, const double* a, int nb, std::int64_t n, double* partials, double* out, cudaStream_t s);
// orthonormalize_pair fallback (lobpcg.hpp:263-269): scale columns of a, ha
// by 1 / sqrt(norm2) when st->ortho_fallback.
void scale_columns(Ctx* ctx, double* a, double* ha, const double* norm2, int nb, std::int64_t n, const Status* st,
                   cudaStream_t s);

// Rayleigh-Ritz pencil assembly (lobpcg.hpp:126-141): G, O (dim x dim,
// column-major, lower blocks placed then mirrored). blocks: 6 (or 3) G
// blocks then 6 (or 3) O blocks, each nb x nb column-major, in the order
// XtHX, WtHX, WtHW, PtHX, PtHW, PtHP / XtX, WtX, WtW, PtX, PtW, PtP.
// nblk = 1 (initial X-only step: XtHX mirrored, XtX), 2 (no P) or 3.
void rr_assemble(Ctx* ctx, const double* blocks, int nb, int nblk, double* G, double* O, cudaStream_t s);

// sygv_lowest (densela.hpp:357-407) on device: R = chol_floored(B) (failure
// -> st->not_pd), M = R^-T A R^-1 symmetrised, eigen-decomposition with
// cuSOLVER syevd, C = R^-1 Q_k with normalize_column_signs. A, B are n x n
// column-major device matrices (A is overwritten); c (n x k), d (k).
// Fused Rayleigh-Ritz eigensolve (rr_eig.cu) for nblk * nb <= 64: assembly,
// floored Cholesky (pivot_floor), reduction, Jacobi, back-transform, signs and
// the drop-P retry in one single-CTA launch. c: (nblk nb) x nb column-major
// (the P rows zeroed when P was dropped), theta: nb ascending, shifts (may be
// null): theta[min(v, k - 1)] for the next preconditioner apply.
bool rr_eig_fits(int dim);
void rr_eig(Ctx* ctx, const double* blocks, int nb, int nblk, int k, double pivot_floor, double* c, double* theta,
            double* shifts, Status* st, cudaStream_t s);
// sygv_lowest on the same single-CTA solver (n <= 64): c (n x k), d (k)
// st->w_rank_first |= st->rank_deficient (the first W qr's verdict survives the second qr)
void latch_w_rank(Ctx* ctx, Status* st, cudaStream_t s);
void sygv_small(Ctx* ctx, const double* A, const double* B, int n, int k, double pivot_floor, double* c, double* d,
                Status* st, cudaStream_t s);

struct Sygv {
    int n = 0;
    int lwork = 0;
    DBuf<double> work, w, R, M;
    DBuf<int> info;
    void ensure(Ctx* ctx, int n);
};
void sygv_lowest(Ctx* ctx, Sygv& ws, double* A, const double* B, int n, int k, double pivot_floor, double* c,
                 double* d, Status* st, cudaStream_t s);

}  // namespace dla
}  // namespace be
