// Reference-style test program for the C++ mirror (include/blockeig_b200.hpp):
// the same calls a blockeig user makes (test_kernels.cpp, test_precond.cpp,
// test_lobpcg.cpp patterns), running on the device. Exit code 0 = pass.
// Built by __graft_entry__.build(); run by tests/test_mirror_gpu.py.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <cstdlib>
#include <string>

#include "blockeig_b200.hpp"

using namespace blockeig;

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// dense host product for checking: (L + L^T + D) X
static BlockVector dense_apply(const std::vector<Triple>& lower, const std::vector<double>& d, const BlockVector& x) {
    BlockVector y(x.nrows, x.nvec);
    for (index_t r = 0; r < x.nrows; ++r)
        for (index_t v = 0; v < x.nvec; ++v) y(r, v) = d[static_cast<std::size_t>(r)] * x(r, v);
    for (const Triple& t : lower)
        for (index_t v = 0; v < x.nvec; ++v) {
            y(t.row, v) += t.value * x(t.col, v);
            y(t.col, v) += t.value * x(t.row, v);
        }
    return y;
}

int main() {
    // synthetic Random matrix, CSB, operator (test_kernels.cpp:217-249 style)
    SynthParams p;
    p.n = 3000;
    p.density = 0.01;
    p.block_extent = 700;
    p.seed = 7;
    SynthMatrix s = generate_synthetic(p);
    const auto b = uniform_boundaries(p.n, 700);
    CsbCooMatrix l = build_csb_coo(s.coo.lower, p.n, p.n, b, b);
    CHECK(is_strictly_lower(l));
    {  // Matrix Market (matrix_market.hpp:38-113) through the mirror
        std::stringstream mm;
        SymmetricCoo c;
        c.n = p.n;
        c.lower = s.coo.lower;
        c.diag = s.coo.diag;
        write_matrix_market(mm, c);
        const SymmetricCoo r = ingest_matrix_market(mm);
        CHECK(r.n == c.n && r.lower.size() == c.lower.size() && r.diag == c.diag);
        bool same = true;
        for (std::size_t k = 0; k < r.lower.size(); ++k)
            same = same && r.lower[k].row == c.lower[k].row && r.lower[k].col == c.lower[k].col &&
                   r.lower[k].value == c.lower[k].value;
        CHECK(same);
        std::istringstream bad("%%MatrixMarket matrix coordinate real general\n1 1 0\n");
        CHECK(throws<NotSymmetricHeader>([&] { ingest_matrix_market(bad); }));
    }
    CHECK(l.nnz() == static_cast<index_t>(s.coo.lower.size()));
    {
        auto back = to_triples(l);
        CHECK(back.size() == s.coo.lower.size());
    }
    const BlockVector x = random_block(p.n, 16, 3);
    const BlockVector want = dense_apply(s.coo.lower, s.coo.diag, x);
    for (be_prec prec : {BE_F32, BE_F64}) {
        SymmetricOperator h(l, s.coo.diag, KernelVariant::sm100a(prec));
        BlockVector y(p.n, 16);
        h.apply(x, y);
        const double e = rel_frobenius_distance(y, want);
        CHECK(e < (prec == BE_F32 ? 1e-5 : 1e-12));
        std::printf("apply prec=%d rel_F=%.3e\n", static_cast<int>(prec), e);
    }
    {  // reference variant names still select the device path
        SymmetricOperator h(l, s.coo.diag, variant_from_name("baseline"));
        BlockVector y(p.n, 16);
        h.apply(x, y);
        CHECK(rel_frobenius_distance(y, want) < 1e-5);
    }
    {  // accumulate semantics: U += L W, U += L^T W
        BlockVector u(p.n, 4), w = random_block(p.n, 4, 5);
        for (double& e : u.data) e = 1.0;
        spmm_notrans(l, w, u, KernelVariant::sm100a(BE_F64));
        spmm_trans(l, w, u, KernelVariant::sm100a(BE_F64));
        std::vector<double> zero(static_cast<std::size_t>(p.n), 0.0);
        BlockVector ref = dense_apply(s.coo.lower, zero, w);
        for (double& e : ref.data) e += 1.0;
        CHECK(rel_frobenius_distance(u, ref) < 1e-12);
        CHECK(throws<BadParams>([&] { spmm_notrans(l, u, u); }));
    }
    // constructor / shape errors (kernels.hpp:341-350, 359-360)
    CHECK(throws<DimensionMismatch>([&] { SymmetricOperator(l, std::vector<double>(10, 1.0)); }));
    {
        std::vector<Triple> upper = {{0, 1, 1.0}};
        auto bb = uniform_boundaries(10, 5);
        CsbCooMatrix u = build_csb_coo(upper, 10, 10, bb, bb);
        CHECK(throws<NotStrictlyLower>([&] { SymmetricOperator(u, std::vector<double>(10, 1.0)); }));
        std::vector<Triple> dup = {{3, 1, 1.0}, {3, 1, 2.0}};
        CHECK(throws<DuplicateEntry>([&] { build_csb_coo(dup, 10, 10, bb, bb); }));
        std::vector<Triple> oob = {{30, 1, 1.0}};
        CHECK(throws<IndexOutOfRange>([&] { build_csb_coo(oob, 10, 10, bb, bb); }));
    }
    {
        SymmetricOperator h(l, s.coo.diag);
        BlockVector y(p.n - 1, 16);
        CHECK(throws<DimensionMismatch>([&] { h.apply(x, y); }));
    }

    // preconditioner: Jacobi case m=1 on the diagonal (test_precond.cpp:249-261)
    DiagonalTileSet tiles = extract_tiles(l, s.coo.diag, s.tile_offsets);
    CHECK(tiles.dim() == p.n);
    CHECK(tiles.count() == static_cast<index_t>(s.tile_offsets.size()) - 1);
    CHECK(static_cast<index_t>(tiles.tiles.size()) == tiles.count());
    {
        BlockVector r = random_block(p.n, 3, 9);
        std::vector<double> sh = {0.0, 0.5, -0.25};
        std::int64_t fb = 0;
        BlockVector w = apply_preconditioner(tiles, sh, r, FomConfig{4}, nullptr, &fb);
        // residual of the tile solves is reduced: check || T w - r || < || r || per tile column
        double num = 0.0, den = 0.0;
        for (index_t j = 0; j < tiles.count(); ++j) {
            const SparseTile& t = tiles.tiles[static_cast<std::size_t>(j)];
            const index_t base = s.tile_offsets[static_cast<std::size_t>(j)];
            for (int v = 0; v < 3; ++v) {
                std::vector<double> xv(static_cast<std::size_t>(t.dim)), yv(static_cast<std::size_t>(t.dim));
                for (index_t i = 0; i < t.dim; ++i) xv[static_cast<std::size_t>(i)] = w(base + i, v);
                t.apply(xv, yv);
                for (index_t i = 0; i < t.dim; ++i) {
                    const double res = yv[static_cast<std::size_t>(i)] - sh[static_cast<std::size_t>(v)] * xv[static_cast<std::size_t>(i)] - r(base + i, v);
                    num += res * res;
                    den += r(base + i, v) * r(base + i, v);
                }
            }
        }
        std::printf("precond relative tile residual %.3e fallbacks %lld\n", std::sqrt(num / den), static_cast<long long>(fb));
        CHECK(std::sqrt(num / den) < 0.5);
        CHECK(throws<DimensionMismatch>([&] { apply_preconditioner(tiles, std::vector<double>{0.0}, r, FomConfig{}); }));
        CHECK(throws<BadParams>([&] { apply_preconditioner(tiles, sh, r, FomConfig{0}); }));
    }

    // LOBPCG on diag(1..100) through a generic closure (test_lobpcg.cpp:258-272)
    {
        const index_t n = 100;
        Operator op = [](const BlockVector& in, BlockVector& out) {
            for (index_t r = 0; r < in.nrows; ++r)
                for (index_t v = 0; v < in.nvec; ++v) out(r, v) = static_cast<double>(r + 1) * in(r, v);
        };
        SolverConfig cfg;
        cfg.k = 5;
        int observed = 0;
        cfg.observer = [&](const SolverState& st, int it) {
            ++observed;
            CHECK(st.x.nrows == n && it == observed);
        };
        SolveResult res = lobpcg_solve(op, n, nullptr, nullptr, cfg);
        CHECK(res.converged);
        for (int i = 0; i < 5; ++i) CHECK(std::abs(res.lambda[static_cast<std::size_t>(i)] - (i + 1)) < 1e-8);
        CHECK(res.history.records.size() <= 60);
        CHECK(observed == static_cast<int>(res.history.records.size()));
        CHECK(res.history.operator_calls == static_cast<std::int64_t>(res.history.records.size()) + 1);
        std::printf("diag(1..100): %zu iterations\n", res.history.records.size());
        // an exception thrown by the closure propagates unchanged
        Operator bad = [](const BlockVector&, BlockVector&) { throw SingularProjection("from the closure"); };
        CHECK(throws<SingularProjection>([&] { lobpcg_solve(bad, n, nullptr, nullptr, cfg); }));
        SolverConfig c2;
        c2.k = 40;
        CHECK(throws<BadParams>([&] { lobpcg_solve(op, n, nullptr, nullptr, c2); }));
        // dependent x0 -> RankDeficient (test_lobpcg.cpp:461-475)
        BlockVector x0(n, 8);
        for (index_t r = 0; r < n; ++r)
            for (int v = 0; v < 8; ++v) x0(r, v) = 1.0;
        CHECK(throws<RankDeficient>([&] { lobpcg_solve(op, n, nullptr, &x0, cfg); }));
    }
    // device-resident solve with the preconditioner
    {
        SymmetricOperator h(l, s.coo.diag);
        SolverConfig cfg;
        cfg.k = 4;
        cfg.nb = 8;
        cfg.seed = 1;
        SolveResult res = lobpcg_solve(h, &tiles, nullptr, cfg);
        CHECK(res.converged);
        CHECK(res.x.nrows == p.n && res.x.nvec == 4);
        // residual check of the returned pairs on the host
        BlockVector hx = dense_apply(s.coo.lower, s.coo.diag, res.x);
        for (int v = 0; v < 4; ++v) {
            double rn = 0.0, xn = 0.0;
            for (index_t r = 0; r < p.n; ++r) {
                const double e = hx(r, v) - res.lambda[static_cast<std::size_t>(v)] * res.x(r, v);
                rn += e * e;
                xn += res.x(r, v) * res.x(r, v);
            }
            CHECK(std::sqrt(rn) <= 1e-6 * std::max(1.0, std::abs(res.lambda[static_cast<std::size_t>(v)])) * std::sqrt(xn) * 1.01);
        }
        std::printf("device solve: %zu iterations, lambda0 %.9f\n", res.history.records.size(), res.lambda[0]);
    }
    // CSB1 round trip (test_csb.cpp:107-122)
    {
        const std::string path = "/tmp/blockeig_b200_mirror_test.csb";
        save_csb_file(path, l, s.coo.diag);
        std::vector<double> d2;
        CsbCooMatrix l2 = load_csb_file(path, &d2);
        CHECK(l2.values == l.values && l2.local_rows == l.local_rows && l2.local_cols == l.local_cols);
        CHECK(l2.block_nnz == l.block_nnz && l2.block_nnz_offsets == l.block_nnz_offsets);
        CHECK(d2 == s.coo.diag);
        std::remove(path.c_str());
    }
    if (failures) {
        std::fprintf(stderr, "%d failures\n", failures);
        return 1;
    }
    std::printf("mirror_test: all checks passed\n");
    return 0;
}
