// ORACLE -- test infrastructure only. Not part of the product.
//
// C-ABI shim over the UNMODIFIED reference headers in
// /root/reference/proj/include/blockeig (compiled from where they lie by
// oracle/Makefile into oracle/_ref/libref.so; no reference source is copied
// into this repository). It lets the tests pin the restatement in
// oracle/oracle.cpp and lets bench.py time the reference's own CPU path
// (cpu_baseline kind "reference").
#include <blockeig/densela.hpp>
#include <blockeig/driver.hpp>
#include <blockeig/dist.hpp>
#include <blockeig/kernels.hpp>
#include <blockeig/lobpcg.hpp>
#include <blockeig/matrix_market.hpp>
#include <blockeig/precond.hpp>
#include <blockeig/synth.hpp>

#include <chrono>
#include <fstream>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

using namespace blockeig;

namespace {
thread_local std::string g_msg;

int code_of(const Error& e) {
    if (dynamic_cast<const BlockTooLarge*>(&e)) return 2;
    if (dynamic_cast<const IndexOutOfRange*>(&e)) return 3;
    if (dynamic_cast<const DuplicateEntry*>(&e)) return 4;
    if (dynamic_cast<const DimensionMismatch*>(&e)) return 5;
    if (dynamic_cast<const NotStrictlyLower*>(&e)) return 6;
    if (dynamic_cast<const MisalignedTiles*>(&e)) return 7;
    if (dynamic_cast<const BadParams*>(&e)) return 8;
    if (dynamic_cast<const NotPositiveDefinite*>(&e)) return 9;
    if (dynamic_cast<const SingularTriangular*>(&e)) return 10;
    if (dynamic_cast<const SingularProjection*>(&e)) return 11;
    if (dynamic_cast<const RankDeficient*>(&e)) return 12;
    if (dynamic_cast<const BasisDegenerate*>(&e)) return 13;
    if (dynamic_cast<const BreakdownUnrecoverable*>(&e)) return 14;
    if (dynamic_cast<const NotSymmetricHeader*>(&e)) return 18;
    if (dynamic_cast<const ParseError*>(&e)) return 17;
    return 1;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_msg = e.what();
        return code_of(e);
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 1;
    }
}

struct View {
    index_t nrows, ncols, nrb, ncb, nnz;
    const index_t *ro, *co, *bn, *bo;
    const std::uint16_t *lr, *lc;
    const double* v;
};

CsbCooMatrix to_matrix(const void* p) {
    const View* v = static_cast<const View*>(p);
    CsbCooMatrix m;
    m.nrows = v->nrows;
    m.ncols = v->ncols;
    m.nrowblks = v->nrb;
    m.ncolblks = v->ncb;
    m.row_offsets.assign(v->ro, v->ro + v->nrb + 1);
    m.col_offsets.assign(v->co, v->co + v->ncb + 1);
    m.block_nnz.assign(v->bn, v->bn + v->nrb * v->ncb);
    m.block_nnz_offsets.assign(v->bo, v->bo + v->nrb * v->ncb);
    m.local_rows.assign(v->lr, v->lr + v->nnz);
    m.local_cols.assign(v->lc, v->lc + v->nnz);
    m.values.assign(v->v, v->v + v->nnz);
    return m;
}

std::unique_ptr<ThreadPool> pool_of(int threads) {
    return threads > 1 ? std::make_unique<ThreadPool>(threads) : nullptr;
}

// A prepared problem kept alive across timed calls (bench cpu_baseline).
struct Prepared {
    CsbCooMatrix m;
    std::vector<double> diag;
    std::unique_ptr<ThreadPool> pool;
    std::unique_ptr<SymmetricOperator> op;
    std::optional<DiagonalTileSet> tiles;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

// generate_synthetic (synth.hpp:92): counts first (buffers NULL), then data
int ref_generate_synthetic(int kind, index_t n, double density, index_t bandwidth, index_t block_extent,
                           std::uint64_t seed, index_t* nlower, index_t* rows, index_t* cols, double* vals,
                           double* diag, index_t* ntoff, index_t* toff) {
    return guarded([&] {
        SynthParams p;
        p.kind = kind == 0 ? SynthKind::Banded : kind == 1 ? SynthKind::BlockTile : SynthKind::Random;
        p.n = n;
        p.density = density;
        p.bandwidth = bandwidth;
        p.block_extent = block_extent;
        p.seed = seed;
        const auto s = generate_synthetic(p);
        *nlower = static_cast<index_t>(s.coo.lower.size());
        *ntoff = static_cast<index_t>(s.tile_offsets.size());
        if (rows) {
            for (std::size_t i = 0; i < s.coo.lower.size(); ++i) {
                rows[i] = s.coo.lower[i].row;
                cols[i] = s.coo.lower[i].col;
                vals[i] = s.coo.lower[i].value;
            }
            std::copy(s.coo.diag.begin(), s.coo.diag.end(), diag);
            std::copy(s.tile_offsets.begin(), s.tile_offsets.end(), toff);
        }
    });
}

// build_csb_coo (csb.hpp:100): outputs sized by the caller (nblocks, count)
int ref_build_csb(const index_t* rows, const index_t* cols, const double* vals, index_t count, index_t nrows,
                  index_t ncols, const index_t* rb, index_t nrb, const index_t* cb, index_t ncb, index_t* block_nnz,
                  index_t* block_off, std::uint16_t* lr, std::uint16_t* lc, double* v) {
    return guarded([&] {
        std::vector<Triple> t(static_cast<std::size_t>(count));
        for (index_t i = 0; i < count; ++i) t[i] = {rows[i], cols[i], vals[i]};
        const auto m = build_csb_coo(t, nrows, ncols, std::vector<index_t>(rb, rb + nrb), std::vector<index_t>(cb, cb + ncb));
        std::copy(m.block_nnz.begin(), m.block_nnz.end(), block_nnz);
        std::copy(m.block_nnz_offsets.begin(), m.block_nnz_offsets.end(), block_off);
        std::copy(m.local_rows.begin(), m.local_rows.end(), lr);
        std::copy(m.local_cols.begin(), m.local_cols.end(), lc);
        std::copy(m.values.begin(), m.values.end(), v);
    });
}

// SymmetricOperator::apply / spmm_notrans / spmm_trans with a chosen variant
int ref_spmm(const void* view, const double* diag, const double* X, double* Y, index_t nb, int mode, int variant,
             int threads) {
    return guarded([&] {
        const auto m = to_matrix(view);
        auto pool = pool_of(threads);
        const KernelVariant kv = variant == 0 ? KernelVariant::baseline()
                                 : variant == 1 ? KernelVariant::fused_atomic()
                                                : KernelVariant::cache_blocked();
        const index_t in_rows = mode == 1 ? m.ncols : m.nrows, out_rows = mode == 2 ? m.ncols : m.nrows;
        BlockVector in(in_rows, nb), out(out_rows, nb);
        std::copy(X, X + in_rows * nb, in.data.begin());
        if (mode == 0) {
            SymmetricOperator op(m, std::vector<double>(diag, diag + m.nrows), kv, pool.get());
            op.apply(in, out);
        } else {
            std::copy(Y, Y + out_rows * nb, out.data.begin());
            if (mode == 1)
                spmm_notrans(m, in, out, kv, pool.get());
            else
                spmm_trans(m, in, out, kv, pool.get());
        }
        std::copy(out.data.begin(), out.data.end(), Y);
    });
}

int ref_precond(const void* view, const double* diag, const index_t* off, index_t noff, const double* shifts,
                const double* R, double* W, index_t nb, int m, index_t* fallbacks) {
    return guarded([&] {
        const auto mat = to_matrix(view);
        const auto tiles = extract_tiles(mat, std::span<const double>(diag, mat.nrows), std::vector<index_t>(off, off + noff));
        BlockVector r(mat.nrows, nb);
        std::copy(R, R + mat.nrows * nb, r.data.begin());
        FomConfig cfg;
        cfg.iterations = m;
        std::int64_t fb = 0;
        const auto w = apply_preconditioner(tiles, std::span<const double>(shifts, nb), r, cfg, nullptr, &fb);
        std::copy(w.data.begin(), w.data.end(), W);
        if (fallbacks) *fallbacks = fb;
    });
}

int ref_sygv_lowest(const double* A, const double* B, int n, int k, double floor, double* c, double* d) {
    return guarded([&] {
        SmallDense a(n, n), b(n, n);
        std::copy(A, A + n * n, a.data.begin());
        std::copy(B, B + n * n, b.data.begin());
        const auto r = sygv_lowest(a, b, k, floor);
        std::copy(r.c.data.begin(), r.c.data.end(), c);
        std::copy(r.d.begin(), r.d.end(), d);
    });
}

// lobpcg_solve through the SymmetricOperator overload (lobpcg.hpp:452)
int ref_lobpcg(const void* view, const double* diag, const index_t* off, index_t noff, const double* x0, int k, int nb,
               double tol, int maxiter, int fom_m, std::uint64_t seed, int variant, int threads, double* lambda,
               double* x, double* theta_hist, double* res_hist, int* nconv_hist, double* phase_times,
               index_t* info) {
    return guarded([&] {
        const auto m = to_matrix(view);
        auto pool = pool_of(threads);
        const KernelVariant kv = variant == 0 ? KernelVariant::baseline()
                                 : variant == 1 ? KernelVariant::fused_atomic()
                                                : KernelVariant::cache_blocked();
        SymmetricOperator op(m, std::vector<double>(diag, diag + m.nrows), kv, pool.get());
        std::optional<DiagonalTileSet> tiles;
        if (noff > 0) tiles.emplace(extract_tiles(m, std::span<const double>(diag, m.nrows), std::vector<index_t>(off, off + noff)));
        SolverConfig cfg;
        cfg.k = k;
        cfg.nb = nb;
        cfg.tol = tol;
        cfg.maxiter = maxiter;
        cfg.fom.iterations = fom_m;
        cfg.seed = seed;
        cfg.variant = kv;
        cfg.pool = pool.get();
        std::optional<BlockVector> xb;
        if (x0) {
            xb.emplace(m.nrows, cfg.block_width());
            std::copy(x0, x0 + m.nrows * cfg.block_width(), xb->data.begin());
        }
        const auto res = lobpcg_solve(op, tiles ? &*tiles : nullptr, xb ? &*xb : nullptr, cfg);
        std::copy(res.lambda.begin(), res.lambda.end(), lambda);
        if (x) std::copy(res.x.data.begin(), res.x.data.end(), x);
        const int w = cfg.block_width();
        double ts = 0, tp = 0, td = 0, tt = 0;
        for (std::size_t i = 0; i < res.history.records.size(); ++i) {
            const auto& r = res.history.records[i];
            if (theta_hist) std::copy(r.theta.begin(), r.theta.end(), theta_hist + i * w);
            if (res_hist) std::copy(r.residual_norms.begin(), r.residual_norms.end(), res_hist + i * w);
            if (nconv_hist) nconv_hist[i] = r.n_converged;
            ts += r.t_spmm;
            tp += r.t_precond;
            td += r.t_dense;
            tt += r.t_total;
        }
        if (phase_times) {
            phase_times[0] = ts;
            phase_times[1] = tp;
            phase_times[2] = td;
            phase_times[3] = tt;
        }
        info[0] = res.converged ? 1 : 0;
        info[1] = static_cast<index_t>(res.history.records.size());
        info[2] = res.history.operator_calls;
        info[3] = res.history.precond_fallbacks;
        info[4] = res.history.restarts;
    });
}

// random_block (block_vector.hpp:47-53), the reference's own
int ref_random_block(index_t n, index_t nb, std::uint64_t seed, double* out) {
    return guarded([&] {
        const BlockVector b = random_block(n, nb, seed);
        std::copy(b.data.begin(), b.data.end(), out);
    });
}

// ---- persistent problem for timing loops (bench.py cpu_baseline) ----------
void* ref_prepare(const void* view, const double* diag, const index_t* off, index_t noff, int threads) {
    try {
        auto p = new Prepared;
        p->m = to_matrix(view);
        p->diag.assign(diag, diag + p->m.nrows);
        p->pool = pool_of(threads);
        p->op = std::make_unique<SymmetricOperator>(p->m, p->diag, KernelVariant::baseline(), p->pool.get());
        if (noff > 0)
            p->tiles.emplace(extract_tiles(p->m, p->diag, std::vector<index_t>(off, off + noff)));
        return p;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return nullptr;
    }
}

// The same, from a CSB1 cache file as the reference driver reads it
// (driver.hpp:136-161): load_csb (csb.hpp:264-290), then the u64 length and
// the f64 diagonal section; tile offsets from a plain i64 sidecar (count, then
// offsets), or none (preconditioner off) when tiles_path is NULL.
void* ref_prepare_file(const char* path, const char* tiles_path, int threads) {
    try {
        auto p = new Prepared;
        std::ifstream is(path, std::ios::binary);
        if (!is) throw ParseError(std::string("cannot open cache ") + path);
        p->m = load_csb(is);
        std::uint64_t dlen = 0;
        is.read(reinterpret_cast<char*>(&dlen), sizeof(dlen));
        p->diag.resize(dlen);
        is.read(reinterpret_cast<char*>(p->diag.data()), static_cast<std::streamsize>(dlen * sizeof(double)));
        if (!is) throw ParseError("cache: truncated diagonal section");
        if (static_cast<index_t>(dlen) != p->m.nrows) throw ParseError("cache: dimensions do not match the input matrix");
        p->pool = pool_of(threads);
        p->op = std::make_unique<SymmetricOperator>(p->m, p->diag, KernelVariant::baseline(), p->pool.get());
        if (tiles_path) {
            std::ifstream ts(tiles_path, std::ios::binary);
            std::int64_t cnt = 0;
            ts.read(reinterpret_cast<char*>(&cnt), sizeof(cnt));
            std::vector<index_t> off(static_cast<std::size_t>(cnt));
            ts.read(reinterpret_cast<char*>(off.data()), static_cast<std::streamsize>(cnt * sizeof(index_t)));
            if (!ts) throw ParseError("tile offsets sidecar truncated");
            p->tiles.emplace(extract_tiles(p->m, p->diag, off));
        }
        return p;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return nullptr;
    }
}

index_t ref_prepared_nrows(void* pp) { return static_cast<Prepared*>(pp)->m.nrows; }
index_t ref_prepared_nnz(void* pp) { return static_cast<index_t>(static_cast<Prepared*>(pp)->m.values.size()); }

void ref_release(void* p) { delete static_cast<Prepared*>(p); }

// stored entries of the prepared preconditioner tiles (both triangles + diagonal)
index_t ref_tile_entries(void* pp) {
    auto* p = static_cast<Prepared*>(pp);
    index_t e = 0;
    if (p->tiles)
        for (const auto& t : p->tiles->tiles) e += static_cast<index_t>(t.values.size());
    return e;
}

// time `reps` SymmetricOperator::apply calls; returns seconds per apply (median)
double ref_time_apply(void* pp, index_t nb, std::uint64_t seed, int reps) {
    auto* p = static_cast<Prepared*>(pp);
    const BlockVector w = random_block(p->m.nrows, nb, seed);
    BlockVector u(p->m.nrows, nb);
    std::vector<double> t;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        p->op->apply(w, u);
        t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

// per-iteration wall times (IterationRecord::t_total, lobpcg.hpp:432) of a
// fixed-length run; returns the number of iterations recorded
int ref_lobpcg_iter_times(void* pp, int k, int nb, int iters, std::uint64_t seed, int use_precond, double* times) {
    auto* p = static_cast<Prepared*>(pp);
    SolverConfig cfg;
    cfg.k = k;
    cfg.nb = nb;
    cfg.tol = 1e-300;
    cfg.maxiter = iters;
    cfg.seed = seed;
    cfg.pool = p->pool.get();
    const auto res = lobpcg_solve(*p->op, use_precond && p->tiles ? &*p->tiles : nullptr, nullptr, cfg);
    for (std::size_t i = 0; i < res.history.records.size(); ++i) times[i] = res.history.records[i].t_total;
    return static_cast<int>(res.history.records.size());
}

// run `iters` LOBPCG iterations (tol=1e-300, as test_lobpcg.cpp:341) and
// return wall seconds; phase sums into phase_times[4]
double ref_time_lobpcg(void* pp, int k, int nb, int iters, std::uint64_t seed, int use_precond, double* phase_times) {
    auto* p = static_cast<Prepared*>(pp);
    SolverConfig cfg;
    cfg.k = k;
    cfg.nb = nb;
    cfg.tol = 1e-300;
    cfg.maxiter = iters;
    cfg.seed = seed;
    cfg.pool = p->pool.get();
    const auto t0 = std::chrono::steady_clock::now();
    const auto res = lobpcg_solve(*p->op, use_precond && p->tiles ? &*p->tiles : nullptr, nullptr, cfg);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double ts = 0, tp = 0, td = 0, tt = 0;
    for (const auto& r : res.history.records) {
        ts += r.t_spmm;
        tp += r.t_precond;
        td += r.t_dense;
        tt += r.t_total;
    }
    if (phase_times) {
        phase_times[0] = ts;
        phase_times[1] = tp;
        phase_times[2] = td;
        phase_times[3] = tt;
    }
    return wall;
}

// ---- dist.hpp: the reference's triangular layout and partition (parity
// pinning of the multi-GPU parity variant)
int ref_build_layout(int nd, int* blocks, int* diagonal_ranks) {
    return guarded([&] {
        const auto lt = build_layout(nd);
        for (int r = 0; r < lt.n_ranks; ++r) {
            const auto& b = lt.rank_to_block[static_cast<std::size_t>(r)];
            blocks[3 * r] = b.i;
            blocks[3 * r + 1] = b.j;
            blocks[3 * r + 2] = b.transposed ? 1 : 0;
        }
        for (int g = 0; g < nd; ++g) diagonal_ranks[g] = lt.diagonal_ranks[static_cast<std::size_t>(g)];
    });
}

// partition_matrix of the global strictly-lower triples, then rank r's
// stored entries mapped back to global coordinates (the reassemble rule,
// dist.hpp:203-223) and its segment
int ref_partition_rank(const index_t* rows, const index_t* cols, const double* vals, index_t count,
                       const double* diag, index_t n, int nd, const index_t* sub_bounds, index_t intra_extent,
                       int rank, index_t* out_rows, index_t* out_cols, double* out_vals, index_t* out_count,
                       index_t* seg) {
    return guarded([&] {
        std::vector<Triple> lower(static_cast<std::size_t>(count));
        for (index_t k = 0; k < count; ++k) lower[static_cast<std::size_t>(k)] = {rows[k], cols[k], vals[k]};
        const auto lt = build_layout(nd);
        std::vector<index_t> b(sub_bounds, sub_bounds + nd + 1);
        const auto pb = partition_matrix(lower, std::span<const double>(diag, static_cast<std::size_t>(n)), lt, b,
                                         intra_extent);
        const auto& blk = lt.rank_to_block[static_cast<std::size_t>(rank)];
        const index_t roff = b[static_cast<std::size_t>(blk.i)], coff = b[static_cast<std::size_t>(blk.j)];
        index_t k = 0;
        for (const Triple& t : to_triples(pb.rank_matrix[static_cast<std::size_t>(rank)])) {
            if (k >= *out_count) throw BadParams("ref_partition_rank: buffer too small");
            if (blk.transposed) {
                out_rows[k] = coff + t.col;
                out_cols[k] = roff + t.row;
            } else {
                out_rows[k] = roff + t.row;
                out_cols[k] = coff + t.col;
            }
            out_vals[k] = t.value;
            ++k;
        }
        *out_count = k;
        seg[0] = pb.segment_of_rank[static_cast<std::size_t>(rank)].begin;
        seg[1] = pb.segment_of_rank[static_cast<std::size_t>(rank)].end;
    });
}

// ingest_matrix_market on a text buffer: n, the lower triples (file order) and diag[n]
int ref_mm_parse(const char* text, index_t len, index_t* n, index_t* rows, index_t* cols, double* vals,
                 index_t* count, double* diag, index_t diag_cap) {
    return guarded([&] {
        std::istringstream is(std::string(text, static_cast<std::size_t>(len)));
        const auto m = ingest_matrix_market(is);
        *n = m.n;
        if (rows) {
            if (static_cast<index_t>(m.lower.size()) > *count) throw BadParams("ref_mm_parse: buffer too small");
            for (std::size_t k = 0; k < m.lower.size(); ++k) {
                rows[k] = m.lower[k].row;
                cols[k] = m.lower[k].col;
                vals[k] = m.lower[k].value;
            }
        }
        *count = static_cast<index_t>(m.lower.size());
        if (diag && diag_cap >= m.n) std::memcpy(diag, m.diag.data(), m.diag.size() * sizeof(double));
    });
}

// write_matrix_market into buf (cap bytes); *len = the text length
int ref_mm_write(index_t n, const index_t* rows, const index_t* cols, const double* vals, index_t count,
                 const double* diag, char* buf, index_t cap, index_t* len) {
    return guarded([&] {
        SymmetricCoo m;
        m.n = n;
        for (index_t k = 0; k < count; ++k) m.lower.push_back({rows[k], cols[k], vals[k]});
        m.diag.assign(diag, diag + n);
        std::ostringstream os;
        write_matrix_market(os, m);
        const std::string s = os.str();
        *len = static_cast<index_t>(s.size());
        if (buf && cap > *len) std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

// the reference CLI's `solve` command (driver.hpp:200-290) on a generated
// problem: runs it and keeps its run report ("blockeig/run-report/v1");
// *len receives the report's length, ref_last_report copies it out
static std::string g_last_report;
int ref_cmd_solve(const char* gen, index_t n, double density, index_t block_extent, int k, int nb, double tol,
                  int maxiter, std::uint64_t seed, int no_precond, index_t* len) {
    return guarded([&] {
        DriverArgs a;
        a.gen = gen;
        a.n = n;
        a.density = density;
        a.block_extent = block_extent;
        a.k = k;
        a.nb = nb;
        a.tol = tol;
        a.maxiter = maxiter;
        a.seed = seed;
        a.no_precond = no_precond != 0;
        a.threads = 1;
        std::ostringstream os, es;
        const int rc = cmd_solve(a, os, es);
        if (rc != kExitOk) throw std::runtime_error("cmd_solve exit " + std::to_string(rc) + ": " + es.str());
        g_last_report = os.str();
        *len = static_cast<index_t>(g_last_report.size());
    });
}
int ref_last_report(char* out, index_t cap) {
    return guarded([&] {
        if (cap < static_cast<index_t>(g_last_report.size())) throw std::runtime_error("ref_last_report: buffer too small");
        std::memcpy(out, g_last_report.data(), g_last_report.size());
    });
}

}  // extern "C"
