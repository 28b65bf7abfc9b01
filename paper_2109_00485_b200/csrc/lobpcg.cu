// Device-resident LOBPCG driver (lobpcg_solve, lobpcg.hpp:291-456).
//
// The control flow is the reference's, line for line: CholQR hygiene with
// the seeded random restart (lobpcg.hpp:358-373), one operator application
// per iteration (:376-377), Rayleigh-Ritz over [X W P] with the drop-P retry
// (:380-396), recurrence-updated H-images (:399-406), P hygiene (:412-417),
// residuals and the convergence test (:419-434). Every panel stays in HBM as
// row-major fp64; the host only sees the small status words, the Ritz values
// and the residual norms, read at three synchronisation points per iteration
// (after the first CholQR of W, after the projected eigenproblem, after the
// residual norms). X0 and restart blocks come from the reference's own
// mt19937_64 stream (block_vector.hpp:47-53), generated on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <random>

#include <nvtx3/nvToolsExt.h>

#include "comm.hpp"
#include "densela.cuh"
#include "hostcopy.hpp"
#include "lobpcg.cuh"
#include "precond.cuh"

namespace be {

// random_block (block_vector.hpp:47-53) rows [row_lo, row_lo + n): the
// reference's one mt19937_64 stream over the whole n_global x nb block, of
// which a rank keeps its own rows (multi-GPU X0 / restart blocks match the
// single-GPU ones bit for bit).
std::vector<double> random_block(index_t n, index_t nb, std::uint64_t seed, index_t row_lo) {
    std::vector<double> x(static_cast<std::size_t>(n * nb));
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (index_t i = 0; i < row_lo * nb; ++i) (void)u(rng);
    for (auto& v : x) v = u(rng);
    return x;
}

namespace {


// the small device / pinned buffers a finished solve leaves on its context
struct Keep {
    int nb = 0;
    std::int64_t partials_len = 0;
    DBuf<double> small, partials;
    DBuf<dla::Status> st;
    DBuf<std::int64_t> fallbacks;
    dla::Sygv sygv;
    void* hm = nullptr;  // pinned Solver::Mirror
    ~Keep() {
        if (hm) cudaFreeHost(hm);
    }
};

// NVTX ranges of the iteration phases (the same boundaries as the CUDA events
// of BE_TRACE_SEGMENTS): visible in nsys / Nsight next to the kernels, free
// without an attached tool (NVTX v3 is header-only).
struct NvtxPhases {
    bool open = false;
    void to(const char* name) {
        if (open) nvtxRangePop();
        nvtxRangePushA(name);
        open = true;
    }
    void end() {
        if (open) nvtxRangePop();
        open = false;
    }
};

struct Events {
    cudaEvent_t e[9] = {};
    Events() {
        for (auto& x : e) BE_CUDA(cudaEventCreate(&x));
    }
    ~Events() {
        for (auto& x : e)
            if (x) cudaEventDestroy(x);
    }
    float ms(int a, int b) const {
        float t = 0;
        BE_CUDA(cudaEventElapsedTime(&t, e[a], e[b]));
        return t;
    }
};

struct Solver {
    Ctx* ctx;
    cudaStream_t s;
    index_t n;
    int nb, k;
    Op* op;
    be_host_operator_fn host_op;
    void* host_user;
    Tiles* tiles;
    const be_solver_config& cfg;
    be::Result& res;
    // multi-GPU: panels hold this rank's rows [row_lo, row_lo + n) of n_global;
    // every Gram / norm partial is summed over ranks (distributed_gram_allreduce,
    // dist.hpp:375-391) so all ranks take identical decisions
    Comm* comm = nullptr;
    index_t n_global = 0, row_lo = 0;
    void allreduce(double* p, int count) {
        if (comm) comm->allreduce_f64(p, static_cast<std::size_t>(count), s);
    }

    DBuf<double> X, W, P, HX, HW, HP, R, Xn, HXn, Pn, HPn;
    DBuf<double> small, partials;
    DBuf<dla::Status> st;
    DBuf<std::int64_t> fallbacks;
    dla::Sygv sygv;
    double* blocks = nullptr;  // 12 nb x nb
    double *G = nullptr, *O = nullptr, *C = nullptr, *theta = nullptr;
    double *Bq = nullptr, *Rq = nullptr, *xtp = nullptr, *Bp = nullptr, *Rp = nullptr, *ptw = nullptr;
    double *rn2 = nullptr, *xn2 = nullptr, *shifts = nullptr, *pn2 = nullptr;
    std::int64_t partials_len = 0;
    // pinned host mirror of the small readbacks
    struct Mirror {
        dla::Status st;
        double theta[64];
        double rn2[64];
        double xn2[64];
        double shifts[64];
        std::int64_t fallbacks;
    } * hm = nullptr;
    std::vector<double> host_in, host_out;  // host-operator staging

    Solver(Ctx* c, index_t n_, int nb_, int k_, Op* o, be_host_operator_fn hop, void* hu, Tiles* t,
           const be_solver_config& cf, be::Result& r)
        : ctx(c), s(c->stream), n(n_), nb(nb_), k(k_), op(o), host_op(hop), host_user(hu), tiles(t), cfg(cf), res(r) {
        comm = op ? op->comm : nullptr;
        n_global = n;
        if (comm) {
            n_global = op->cuts.back();
            row_lo = op->row_lo;
        }
        const index_t pn = n * nb;
        for (auto* b : {&X, &W, &P, &HX, &HW, &HP, &R, &Xn, &HXn, &Pn, &HPn})  // pooled on the context
            *b = ctx->panels->take(std::max<index_t>(pn, 1));
        const index_t nb2 = static_cast<index_t>(nb) * nb, dim = 3 * nb;
        partials_len = std::max<std::int64_t>(dla::gram_partials_len(nb, 12, ctx->num_sms),
                                              static_cast<std::int64_t>(ctx->num_sms) * 4 * 2 * nb);
        // the small buffers of the previous solve on this context, when they fit
        auto keep = std::static_pointer_cast<Keep>(ctx->solver_keep);
        ctx->solver_keep.reset();
        if (keep && keep->nb == nb && keep->partials_len == partials_len) {
            small = std::move(keep->small);
            partials = std::move(keep->partials);
            st = std::move(keep->st);
            fallbacks = std::move(keep->fallbacks);
            sygv = std::move(keep->sygv);
            hm = static_cast<Mirror*>(keep->hm);
            keep->hm = nullptr;
        }
        keep.reset();
        if (!small.p) small.reset(12 * nb2 + 2 * dim * dim + dim * nb + 8 * nb2 + 8 * nb);
        double* p = small.get();
        blocks = p; p += 12 * nb2;
        G = p; p += dim * dim;
        O = p; p += dim * dim;
        C = p; p += dim * nb;
        Bq = p; p += nb2;
        Rq = p; p += nb2;
        xtp = p; p += nb2;
        Bp = p; p += nb2;
        Rp = p; p += nb2;
        ptw = p;  // P^T W formed by the X projection's mix
        p += 3 * nb2;
        theta = p; p += nb;
        rn2 = p; p += nb;
        xn2 = p; p += nb;
        shifts = p; p += nb;
        pn2 = p; p += nb;
        if (!partials.p) partials.reset(partials_len);
        if (!st.p) st.reset(1);
        if (!fallbacks.p) fallbacks.reset(1);
        BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(dla::Status), s));
        BE_CUDA(cudaMemsetAsync(fallbacks.get(), 0, sizeof(std::int64_t), s));
        if (!hm) BE_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hm), sizeof(Mirror)));
        sygv.ensure(ctx, dim);
    }
    ~Solver() {
        if (cudaStreamSynchronize(s) != cudaSuccess) {  // queued work may still use the buffers: plain release
            if (hm) cudaFreeHost(hm);
            return;
        }
        for (auto* b : {&X, &W, &P, &HX, &HW, &HP, &R, &Xn, &HXn, &Pn, &HPn}) ctx->panels->give(std::move(*b));
        auto keep = std::make_shared<Keep>();
        keep->nb = nb;
        keep->partials_len = partials_len;
        keep->small = std::move(small);
        keep->partials = std::move(partials);
        keep->st = std::move(st);
        keep->fallbacks = std::move(fallbacks);
        keep->sygv = std::move(sygv);
        keep->hm = hm;
        hm = nullptr;
        ctx->solver_keep = std::move(keep);
    }

    // host wait on the solver stream; with a communicator it watches the group (Comm::sync)
    void wait() {
        if (comm) comm->sync(s);
        else BE_CUDA(cudaStreamSynchronize(s));
    }
    void sync_status() {
        BE_CUDA(cudaMemcpyAsync(&hm->st, st.get(), sizeof(dla::Status), cudaMemcpyDeviceToHost, s));
        wait();
    }
    // qr_failures and rank_deficient only: singular_tri stays set until the iteration's check
    void reset_qr_flags() { BE_CUDA(cudaMemsetAsync(st.get(), 0, 2 * sizeof(int), s)); }

    void apply_op(const double* in, double* out) {
        if (op) {
            op_apply(op, in, out, n, nb, BE_F64, BE_APPLY_SYMMETRIC, s);
        } else {
            host_in.resize(static_cast<std::size_t>(n * nb));
            host_out.assign(static_cast<std::size_t>(n * nb), 0.0);
            BE_CUDA(cudaMemcpyAsync(host_in.data(), in, host_in.size() * 8, cudaMemcpyDeviceToHost, s));
            BE_CUDA(cudaStreamSynchronize(s));
            if (host_op(host_user, host_in.data(), host_out.data(), n, nb) != 0)
                fail(BE_ERR_GENERIC, "lobpcg_solve: host operator callback failed");
            BE_CUDA(cudaMemcpyAsync(out, host_out.data(), host_out.size() * 8, cudaMemcpyHostToDevice, s));
        }
        ++res.operator_calls;
    }

    void gram1(const double* a, const double* b, int sym, double* out) {
        dla::GramJob j{};
        j.npairs = 1;
        j.nb = nb;
        j.a[0] = a;
        j.b[0] = b;
        j.sym[0] = sym;
        j.out[0] = out;
        dla::gram(ctx, j, n, partials.get(), partials_len, s);
        allreduce(out, nb * nb);
    }

    // qr_of_transpose (densela.hpp:412-445); returns false on RankDeficient
    bool qr(double* A, bool check, bool gram_given = false) {
        reset_qr_flags();
        bool have_gram = gram_given;  // Bq already holds A^T A (the producer formed it) / the first
                                      // pass's trsm formed the second pass's Gram
        for (int pass = 0; pass < 2; ++pass) {
            if (!have_gram) gram1(A, A, 1, Bq);
            dla::qr_chol(ctx, Bq, Rq, nb, st.get(), s);
            have_gram = pass == 0 && dla::trsm_gram(ctx, A, Rq, nb, n, st.get(), Bq, partials.get(), partials_len, s);
            if (have_gram) allreduce(Bq, nb * nb);
            else dla::trsm(ctx, A, nullptr, Rq, nb, n, st.get(), 1, 0, s);
        }
        if (!check) return true;
        sync_status();
        if (hm->st.singular_tri) fail(BE_ERR_SINGULAR_TRIANGULAR, "trsm_right_inv: triangular factor is numerically singular");
        return hm->st.rank_deficient == 0;
    }

    void upload_random(double* dst, std::uint64_t seed) {
        const auto h = random_block(n, nb, seed, row_lo);
        BE_CUDA(cudaMemcpyAsync(dst, h.data(), h.size() * 8, cudaMemcpyHostToDevice, s));
        BE_CUDA(cudaStreamSynchronize(s));
    }

    // project_out (lobpcg.hpp:243-246): w -= basis (basis^T w)
    // gram_next: the Gram of the projected w (the next qr_of_transpose's first pass) is formed
    // into Bq on the way; returns whether it was
    // next_basis: instead, the next projection's Gram next_basis^T w' goes into ptw (that basis
    // loaded as one more panel of the mix); basis_gram: xtp already holds basis^T w.
    bool project_out(double* w, const double* basis, bool gram_next = false, const double* next_basis = nullptr,
                     bool basis_gram = false) {
        if (!basis_gram) gram1(basis, w, 0, xtp);
        dla::MixJob m{};
        m.nb = nb;
        m.nout = 1;
        m.out[0] = dla::MixOut{w, 1, 1, {{basis, xtp, 1, 0}}, -1};
        if (gram_next || next_basis) {
            m.gram_out = next_basis ? ptw : Bq;
            m.gram_a = next_basis ? -1 : 0;
            m.gram_a_src = next_basis;
            m.gram_b = 0;
            m.gram_sym = next_basis ? 0 : 1;
            m.gram_partials = partials.get();
            m.gram_partials_len = partials_len;
        }
        const bool g = dla::mix(ctx, m, n, s) && (gram_next || next_basis);
        if (g) allreduce(m.gram_out, nb * nb);
        return g;
    }

    // rayleigh_ritz (lobpcg.hpp:113-157): false on BasisDegenerate
    bool rayleigh_ritz(bool with_p) {
        dla::GramJob j{};
        j.nb = nb;
        const double* gpairs[12][2];
        int sym[12];
        int np = 0;
        auto add = [&](const double* a, const double* b, int sy) {
            gpairs[np][0] = a;
            gpairs[np][1] = b;
            sym[np] = sy;
            ++np;
        };
        add(X.get(), HX.get(), 0);
        add(W.get(), HX.get(), 0);
        add(W.get(), HW.get(), 0);
        if (with_p) {
            add(P.get(), HX.get(), 0);
            add(P.get(), HW.get(), 0);
            add(P.get(), HP.get(), 0);
        }
        add(X.get(), X.get(), 1);
        add(W.get(), X.get(), 0);
        add(W.get(), W.get(), 1);
        if (with_p) {
            add(P.get(), X.get(), 0);
            add(P.get(), W.get(), 0);
            add(P.get(), P.get(), 1);
        }
        j.npairs = np;
        for (int q = 0; q < np; ++q) {
            j.a[q] = gpairs[q][0];
            j.b[q] = gpairs[q][1];
            j.sym[q] = sym[q];
            j.out[q] = blocks + static_cast<index_t>(q) * nb * nb;
        }
        dla::gram(ctx, j, n, partials.get(), partials_len, s);
        allreduce(blocks, np * nb * nb);
        const int nblk = with_p ? 3 : 2;
        if (fused_rr) {  // one launch, no host round trip; verdict read at the iteration's sync
            dla::rr_eig(ctx, blocks, nb, nblk, k, 1e-10, C, theta, shifts, st.get(), s);
            return true;
        }
        dla::rr_assemble(ctx, blocks, nb, nblk, G, O, s);
        dla::sygv_lowest(ctx, sygv, G, O, nblk * nb, nb, 1e-10, C, theta, st.get(), s);
        BE_CUDA(cudaMemcpyAsync(hm->theta, theta, nb * 8, cudaMemcpyDeviceToHost, s));
        sync_status();
        return hm->st.not_pd == 0;
    }

    std::vector<double> th;
    const bool trace_segments = std::getenv("BE_TRACE_SEGMENTS") != nullptr;
    // the fused single-CTA Rayleigh-Ritz eigensolve (rr_eig.cu) when the pencil fits
    const bool fused_rr = dla::rr_eig_fits(3 * nb) && std::getenv("BE_RR_CUSOLVER") == nullptr;
    bool p_active = false, converged = false;
    int iter = 0;
    Events ev;
    NvtxPhases nv;

    void init(const double* x0) {
        if (x0)
            h2d_large(X.get(), x0, static_cast<std::size_t>(n * nb) * 8, s);
        else
            upload_random(X.get(), cfg.seed);
        if (!qr(X.get(), true)) fail(BE_ERR_RANK_DEFICIENT, "qr_of_transpose: Gram Cholesky failed twice");
        apply_op(X.get(), HX.get());
        {  // initial Rayleigh-Ritz on X alone (lobpcg.hpp:320-334)
            dla::GramJob j{};
            j.nb = nb;
            j.npairs = 2;
            j.a[0] = X.get(); j.b[0] = HX.get(); j.sym[0] = 0; j.out[0] = blocks;
            j.a[1] = X.get(); j.b[1] = X.get(); j.sym[1] = 1; j.out[1] = blocks + static_cast<index_t>(nb) * nb;
            dla::gram(ctx, j, n, partials.get(), partials_len, s);
            allreduce(blocks, 2 * nb * nb);
            if (fused_rr) {
                dla::rr_eig(ctx, blocks, nb, 1, k, 1e-10, C, theta, shifts, st.get(), s);
            } else {
                dla::rr_assemble(ctx, blocks, nb, 1, G, O, s);
                dla::sygv_lowest(ctx, sygv, G, O, nb, nb, 1e-10, C, theta, st.get(), s);
            }
            BE_CUDA(cudaMemcpyAsync(hm->theta, theta, nb * 8, cudaMemcpyDeviceToHost, s));
            sync_status();
            if (hm->st.not_pd || hm->st.rr_dropped) fail(BE_ERR_BREAKDOWN_UNRECOVERABLE, "lobpcg_solve: initial block is degenerate");
            dla::MixJob m{};
            m.nb = nb;
            m.nout = 2;
            m.out[0] = dla::MixOut{Xn.get(), 0, 1, {{X.get(), C, 0, nb}}, -1};
            m.out[1] = dla::MixOut{HXn.get(), 0, 1, {{HX.get(), C, 0, nb}}, -1};
            dla::mix(ctx, m, n, s);
            std::swap(X, Xn);
            std::swap(HX, HXn);
        }
        th.assign(hm->theta, hm->theta + nb);
        dla::residual(ctx, HX.get(), X.get(), theta, R.get(), nb, n, partials.get(), rn2, xn2, s);
        allreduce(rn2, 2 * nb);  // rn2, xn2 are adjacent
    }

    // One iteration of lobpcg_solve (lobpcg.hpp:338-441) from the preconditioner
    // on. With the fused Rayleigh-Ritz eigensolve the device takes every
    // decision of the iteration itself (the drop-P retry inside rr_eig, the
    // W restart deferred, see iterate) and the host synchronises once, at the
    // end, to read the status, the Ritz values and the residual norms.
    void iteration_body(bool w_restart) {
        nv.to("precond");
        BE_CUDA(cudaEventRecord(ev.e[0], s));
        if (!w_restart) {
            if (tiles) {  // W = K^{-1} R, shifts theta[min(v, k-1)] (lobpcg.hpp:344-350)
                if (!fused_rr) {  // (the fused eigensolve writes the shifts on the device)
                    for (int v = 0; v < nb; ++v) hm->shifts[v] = th[static_cast<std::size_t>(std::min(v, k - 1))];
                    BE_CUDA(cudaMemcpyAsync(shifts, hm->shifts, nb * 8, cudaMemcpyHostToDevice, s));
                }
                precond_apply(tiles, shifts, R.get(), W.get(), n, nb, cfg.fom_iterations, fallbacks.get(), s);
            } else {
                BE_CUDA(cudaMemcpyAsync(W.get(), R.get(), static_cast<std::size_t>(n * nb) * 8, cudaMemcpyDeviceToDevice, s));
            }
        }
        nv.to("w-hygiene");
        BE_CUDA(cudaEventRecord(ev.e[1], s));
        // W hygiene (lobpcg.hpp:358-373)
        if (w_restart) {  // the first qr_of_transpose of W gave up: a random W (lobpcg.hpp:360-363)
            upload_random(W.get(), cfg.seed + static_cast<std::uint64_t>(iter) * 7919u);
            if (!qr(W.get(), true)) fail(BE_ERR_RANK_DEFICIENT, "qr_of_transpose: Gram Cholesky failed twice");
        } else if (fused_rr && op) {
            // device operator: verdict latched, read at the end of the iteration (a rare redo costs
            // one extra device apply). A host operator is checked now instead: its calls are
            // observable (test_lobpcg.cpp:334-354 counts them), so it is never applied speculatively.
            qr(W.get(), false);
            dla::latch_w_rank(ctx, st.get(), s);
        } else if (!qr(W.get(), true)) {
            upload_random(W.get(), cfg.seed + static_cast<std::uint64_t>(iter) * 7919u);
            if (!qr(W.get(), true)) fail(BE_ERR_RANK_DEFICIENT, "qr_of_transpose: Gram Cholesky failed twice");
        }
        bool wg = project_out(W.get(), X.get(), !p_active, p_active ? P.get() : nullptr);
        if (p_active) {
            if (wg) std::swap(xtp, ptw);  // P^T W' is ready: the second projection's coefficients
            wg = project_out(W.get(), P.get(), true, nullptr, wg);
        }
        qr(W.get(), false, wg);  // RankDeficient swallowed: W keeps the completed passes
        nv.to("spmm");
        BE_CUDA(cudaEventRecord(ev.e[2], s));
        apply_op(W.get(), HW.get());
        nv.to("rayleigh-ritz");
        BE_CUDA(cudaEventRecord(ev.e[3], s));
        // Rayleigh-Ritz with the drop-P retry (lobpcg.hpp:380-396)
        dropped_host = false;
        if (!rayleigh_ritz(p_active)) {  // (host-driven path only: the fused one retries on the device)
            if (!p_active) fail(BE_ERR_BREAKDOWN_UNRECOVERABLE, "lobpcg_solve: 2-block basis failed Cholesky");
            dropped_host = true;
            if (!rayleigh_ritz(false)) fail(BE_ERR_BREAKDOWN_UNRECOVERABLE, "lobpcg_solve: basis repair failed twice");
        }
        nv.to("update");
        BE_CUDA(cudaEventRecord(ev.e[5], s));
        // fused: C keeps the 3-block layout and its P rows are zero after a device-side drop
        const bool with_p = p_active && !dropped_host;
        const int dim = (with_p ? 3 : 2) * nb;
        {  // update_blocks (lobpcg.hpp:168-194): P+ = W C2 + P C3, X+ = X C1 + P+ (and the H-images),
           // as two passes of <= 4 sources each (one 6-source pass runs at a fraction of HBM bandwidth)
            const double* c1 = C;
            const double* c2 = C + nb;
            const double* c3 = C + 2 * nb;
            dla::MixJob m{};
            m.nb = nb;
            m.nout = 2;
            m.out[0] = dla::MixOut{Pn.get(), 0, with_p ? 2 : 1, {{W.get(), c2, 0, dim}, {P.get(), c3, 0, dim}}, -1};
            m.out[1] = dla::MixOut{HPn.get(), 0, with_p ? 2 : 1, {{HW.get(), c2, 0, dim}, {HP.get(), c3, 0, dim}}, -1};
            dla::mix(ctx, m, n, s);
            dla::MixJob m2{};
            m2.nb = nb;
            m2.nout = 2;
            m2.out[0] = dla::MixOut{Xn.get(), 0, 1, {{X.get(), c1, 0, dim}}, -1, Pn.get()};
            m2.out[1] = dla::MixOut{HXn.get(), 0, 1, {{HX.get(), c1, 0, dim}}, -1, HPn.get()};
            // P hygiene's first Gram X+^T P+ formed on the way (both are in the kernel's registers)
            m2.gram_out = xtp;
            m2.gram_a = 0;
            m2.gram_b_src = Pn.get();
            m2.gram_partials = partials.get();
            m2.gram_partials_len = partials_len;
            xtp_ready = dla::mix(ctx, m2, n, s);
            std::swap(X, Xn);
            std::swap(HX, HXn);
            std::swap(P, Pn);
            std::swap(HP, HPn);
        }
        nv.to("p-hygiene");
        BE_CUDA(cudaEventRecord(ev.e[6], s));
        {  // P hygiene (lobpcg.hpp:412-417) + orthonormalize_pair (:254-270)
            if (xtp_ready) allreduce(xtp, nb * nb);
            else gram1(X.get(), P.get(), 0, xtp);
            dla::MixJob m{};
            m.nb = nb;
            m.nout = 2;
            m.out[0] = dla::MixOut{P.get(), 1, 1, {{X.get(), xtp, 1, 0}}, -1};
            m.out[1] = dla::MixOut{HP.get(), 1, 1, {{HX.get(), xtp, 1, 0}}, -1};
            // orthonormalize_pair's Gram of the projected P, formed on the way
            m.gram_out = Bp;
            m.gram_a = 0;
            m.gram_b = 0;
            m.gram_sym = 1;
            m.gram_partials = partials.get();
            m.gram_partials_len = partials_len;
            // residual_block (lobpcg.hpp:419) from the same X / HX loads: it reads only X, HX and
            // theta, which P hygiene leaves alone
            m.res_out = R.get();
            m.res_x = X.get();
            m.res_hx = HX.get();
            m.res_theta = theta;
            m.res_rn2 = rn2;
            m.res_xn2 = xn2;
            res_ready = dla::mix(ctx, m, n, s);
            if (res_ready) allreduce(Bp, nb * nb);
            else gram1(P.get(), P.get(), 1, Bp);
            dla::chol_floored(ctx, Bp, Rp, nb, 1e-8, st.get(), s);
            dla::trsm(ctx, P.get(), HP.get(), Rp, nb, n, st.get(), 0, 1, s);
        }
        nv.to("residual");
        BE_CUDA(cudaEventRecord(ev.e[7], s));
        if (!res_ready) dla::residual(ctx, HX.get(), X.get(), theta, R.get(), nb, n, partials.get(), rn2, xn2, s);
        allreduce(rn2, 2 * nb);
        BE_CUDA(cudaMemcpyAsync(hm->theta, theta, nb * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaMemcpyAsync(hm->rn2, rn2, nb * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaMemcpyAsync(hm->xn2, xn2, nb * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaEventRecord(ev.e[4], s));
        nv.end();
        sync_status();
    }
    bool dropped_host = false;
    bool xtp_ready = false;  // the update's mix formed X+^T P+
    bool res_ready = false;  // P hygiene's mix formed the residual and its norms

    // run up to `count` further iterations (never past maxiter); returns the
    // number executed. Stops at convergence.
    int iterate(int count) {
        int done = 0;
        while (done < count && !converged && iter < cfg.maxiter) {
            ++iter;
            ++done;
            const auto wall0 = std::chrono::steady_clock::now();
            BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(dla::Status), s));
            const bool p_was = p_active;
            iteration_body(false);
            if (hm->st.w_rank_first) {
                // The first qr_of_transpose of W gave up (rare): roll back to the state
                // before the update (the update wrote the other half of every double-buffered
                // panel) and redo the iteration from a random W, as the reference does.
                std::swap(X, Xn);
                std::swap(HX, HXn);
                std::swap(P, Pn);
                std::swap(HP, HPn);
                p_active = p_was;
                --res.operator_calls;
                BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(dla::Status), s));
                iteration_body(true);
            }
            if (hm->st.rr_dropped == 2) fail(BE_ERR_BREAKDOWN_UNRECOVERABLE, "lobpcg_solve: basis repair failed twice");
            if (hm->st.rr_dropped == 1 || dropped_host) ++res.restarts;
            th.assign(hm->theta, hm->theta + nb);
            p_active = true;
            if (hm->st.not_pd) {  // column-scaling fallback of orthonormalize_pair
                dla::colnorm2(ctx, P.get(), nb, n, partials.get(), pn2, s);
                allreduce(pn2, nb);
                dla::scale_columns(ctx, P.get(), HP.get(), pn2, nb, n, st.get(), s);
                BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(dla::Status), s));
            }
            if (hm->st.singular_tri) fail(BE_ERR_SINGULAR_TRIANGULAR, "trsm_right_inv: triangular factor is numerically singular");
            // convergence_check (lobpcg.hpp:216-233)
            IterRecord rec;
            rec.iter = iter;
            rec.theta = th;
            rec.resn.resize(static_cast<std::size_t>(nb));
            int nconv = 0;
            for (int v = 0; v < nb; ++v) {
                const double rn = std::sqrt(hm->rn2[v]), xn = std::sqrt(hm->xn2[v]);
                rec.resn[static_cast<std::size_t>(v)] = rn;
                if (rn <= cfg.tol * std::max(1.0, std::abs(th[static_cast<std::size_t>(v)])) * xn && v < k) ++nconv;
            }
            rec.nconv = nconv;
            rec.t_precond = ev.ms(0, 1) * 1e-3;
            rec.t_spmm = ev.ms(2, 3) * 1e-3;
            rec.t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
            rec.t_dense = std::max(0.0, rec.t_total - rec.t_spmm - rec.t_precond);
            if (trace_segments)  // BE_TRACE_SEGMENTS=1: device time of each phase of the iteration
                std::fprintf(stderr,
                             "[be] iter %d ms: precond %.3f w-hygiene %.3f spmm %.3f rayleigh-ritz %.3f update %.3f "
                             "p-hygiene %.3f residual %.3f wall %.3f\n",
                             iter, ev.ms(0, 1), ev.ms(1, 2), ev.ms(2, 3), ev.ms(3, 5), ev.ms(5, 6), ev.ms(6, 7),
                             ev.ms(7, 4), rec.t_total * 1e3);
            res.records.push_back(rec);
            if (observer) {  // SolverState after the iteration (lobpcg.hpp:52-58, 436)
                std::vector<double> hb;
                const double* ph[6] = {};
                if (cfg.observer_state) {  // X, HX, W, HW, P+, HP+ (the buffers hold exactly these here)
                    const std::size_t pn = static_cast<std::size_t>(n * nb);
                    hb.resize(6 * pn);
                    const double* src[6] = {X.get(), HX.get(), W.get(), HW.get(), P.get(), HP.get()};
                    for (int q = 0; q < 6; ++q) {
                        BE_CUDA(cudaMemcpyAsync(hb.data() + q * pn, src[q], pn * 8, cudaMemcpyDeviceToHost, s));
                        ph[q] = hb.data() + q * pn;
                    }
                    BE_CUDA(cudaStreamSynchronize(s));
                }
                observer(observer_user, iter, n, nb, th.data(), rec.resn.data(), nconv, ph[0], ph[1], ph[2], ph[3],
                         ph[4], ph[5]);
            }
            if (nconv >= k) converged = true;
        }
        return done;
    }

    // The first k columns of X stay on the device (compacted to n x k); the
    // caller's be_result_get copies them straight into its buffer.
    void finish() {
        res.converged = converged;
        res.lambda.assign(th.begin(), th.begin() + k);
        res.device = ctx->device;
        res.pool = ctx->panels;
        res.xdev = ctx->panels->take(std::max<index_t>(n * k, 1));
        if (n > 0)
            BE_CUDA(cudaMemcpy2DAsync(res.xdev.get(), static_cast<std::size_t>(k) * 8, X.get(),
                                      static_cast<std::size_t>(nb) * 8, static_cast<std::size_t>(k) * 8,
                                      static_cast<std::size_t>(n), cudaMemcpyDeviceToDevice, s));
        BE_CUDA(cudaMemcpyAsync(&hm->fallbacks, fallbacks.get(), 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
        res.precond_fallbacks = hm->fallbacks;
    }

    be_observer_fn observer = nullptr;
    void* observer_user = nullptr;
};

}  // namespace

std::unique_ptr<Result> lobpcg_solve(Ctx* ctx, Op* op, be_host_operator_fn host_op, void* host_user, index_t n,
                                     Tiles* tiles, const double* x0, const be_solver_config& cfg,
                                     be_observer_fn observer, void* observer_user) {
    const int nb = cfg.nb > 0 ? cfg.nb : cfg.k + 3;
    // SolverConfig::validate (lobpcg.hpp:38-47) + FomConfig::validate
    if (cfg.k < 1 || cfg.k > nb) fail(BE_ERR_BAD_PARAMS, "SolverConfig: need 1 <= k <= nb");
    const index_t n_all = (op && op->comm) ? op->cuts.back() : n;
    if (static_cast<index_t>(nb) * 3 > n_all) fail(BE_ERR_BAD_PARAMS, "SolverConfig: operator dimension must be at least 3*nb");
    if (!(cfg.tol > 0.0)) fail(BE_ERR_BAD_PARAMS, "SolverConfig: tol must be positive");
    if (cfg.maxiter < 1) fail(BE_ERR_BAD_PARAMS, "SolverConfig: maxiter must be positive");
    if (cfg.fom_iterations < 1) fail(BE_ERR_BAD_PARAMS, "FomConfig: iterations must be >= 1");
    if (nb > 64) fail(BE_ERR_BAD_PARAMS, "lobpcg_solve: block width above 64 is not supported on the device");
    if (!op && !host_op) fail(BE_ERR_BAD_PARAMS, "lobpcg_solve: no operator");
    if (op && (!op->symmetric || op->nrows != n)) fail(BE_ERR_DIMENSION_MISMATCH, "lobpcg_solve: operator dimension mismatch");
    if (tiles && tiles->n != n) fail(BE_ERR_DIMENSION_MISMATCH, "lobpcg_solve: preconditioner dimension mismatch");
    BE_CUDA(cudaSetDevice(ctx->device));
    auto res = std::make_unique<Result>();
    res->n = n;
    res->nb = nb;
    res->k = cfg.k;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    auto sv = std::make_unique<Solver>(ctx, n, nb, cfg.k, op, host_op, host_user, tiles, cfg, *res);
    sv->observer = observer;
    sv->observer_user = observer_user;
    const auto t1 = clk::now();
    sv->init(x0);
    BE_CUDA(cudaStreamSynchronize(sv->s));
    const auto t2 = clk::now();
    sv->iterate(cfg.maxiter);
    const auto t3 = clk::now();
    sv->finish();
    const auto t4 = clk::now();
    const bool trace = sv->trace_segments;
    sv.reset();
    const auto t5 = clk::now();
    if (trace) {
        auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[be] solve ms: setup %.1f init %.1f iterate %.1f finish %.1f teardown %.1f\n", ms(t0, t1),
                     ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5));
    }
    return res;
}

struct Incremental {
    be_solver_config cfg;
    std::unique_ptr<Result> res;
    std::unique_ptr<Solver> sv;
};

void* lobpcg_begin(Ctx* ctx, Op* op, be_host_operator_fn host_op, void* host_user, index_t n, Tiles* tiles,
                   const double* x0, const be_solver_config& cfg) {
    const int nb = cfg.nb > 0 ? cfg.nb : cfg.k + 3;
    if (cfg.k < 1 || cfg.k > nb) fail(BE_ERR_BAD_PARAMS, "SolverConfig: need 1 <= k <= nb");
    const index_t n_all = (op && op->comm) ? op->cuts.back() : n;
    if (static_cast<index_t>(nb) * 3 > n_all) fail(BE_ERR_BAD_PARAMS, "SolverConfig: operator dimension must be at least 3*nb");
    if (!(cfg.tol > 0.0)) fail(BE_ERR_BAD_PARAMS, "SolverConfig: tol must be positive");
    if (cfg.maxiter < 1) fail(BE_ERR_BAD_PARAMS, "SolverConfig: maxiter must be positive");
    if (cfg.fom_iterations < 1) fail(BE_ERR_BAD_PARAMS, "FomConfig: iterations must be >= 1");
    if (nb > 64) fail(BE_ERR_BAD_PARAMS, "lobpcg_solve: block width above 64 is not supported on the device");
    if (!op && !host_op) fail(BE_ERR_BAD_PARAMS, "lobpcg_solve: no operator");
    if (op && (!op->symmetric || op->nrows != n)) fail(BE_ERR_DIMENSION_MISMATCH, "lobpcg_solve: operator dimension mismatch");
    if (tiles && tiles->n != n) fail(BE_ERR_DIMENSION_MISMATCH, "lobpcg_solve: preconditioner dimension mismatch");
    BE_CUDA(cudaSetDevice(ctx->device));
    auto inc = std::make_unique<Incremental>();
    inc->cfg = cfg;
    inc->res = std::make_unique<Result>();
    inc->res->n = n;
    inc->res->nb = nb;
    inc->res->k = cfg.k;
    inc->sv = std::make_unique<Solver>(ctx, n, nb, cfg.k, op, host_op, host_user, tiles, inc->cfg, *inc->res);
    inc->sv->init(x0);
    return inc.release();
}

int lobpcg_step(void* h, int count) { return static_cast<Incremental*>(h)->sv->iterate(count); }

std::unique_ptr<Result> lobpcg_end(void* h) {
    std::unique_ptr<Incremental> inc(static_cast<Incremental*>(h));
    inc->sv->finish();
    inc->sv.reset();
    return std::move(inc->res);
}

void lobpcg_abort(void* h) { delete static_cast<Incremental*>(h); }

}  // namespace be
