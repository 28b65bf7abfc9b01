// Device-resident LOBPCG (lobpcg.hpp) result objects.
#pragma once

#include <memory>
#include <vector>

#include "device.hpp"

namespace be {

struct Tiles;

// random_block (block_vector.hpp:47-53): rows [row_lo, row_lo + n) of the reference's
// mt19937_64 U(-1, 1) block (host; X0 and restart blocks are generated here and copied)
std::vector<double> random_block(index_t n, index_t nb, std::uint64_t seed, index_t row_lo = 0);

struct IterRecord {  // IterationRecord, lobpcg.hpp:60-66
    int iter = 0;
    std::vector<double> theta, resn;
    int nconv = 0;
    double t_spmm = 0, t_precond = 0, t_dense = 0, t_total = 0;
};

struct Result {  // SolveResult + ConvergenceHistory, lobpcg.hpp:68-80
    index_t n = 0;
    int nb = 0, k = 0;
    std::vector<double> lambda, x;
    int device = 0;
    DBuf<double> xdev;
    // xdev goes back to the context's pool when the result is freed; a weak reference, so a result
    // outliving its context does not keep the context's pooled panels allocated (xdev is freed then)
    std::weak_ptr<PanelPool> pool;
    Result() = default;
    Result(const Result&) = delete;
    Result& operator=(const Result&) = delete;
    ~Result() {
        if (!xdev.p) return;
        if (auto p = pool.lock()) p->give(std::move(xdev));  // (no CUDA call: the pool keeps it)
    }  // the n x k eigenvector block, kept on the device until read (x stays empty then)
    std::vector<IterRecord> records;
    std::int64_t operator_calls = 0, precond_fallbacks = 0;
    int restarts = 0;
    bool converged = false;
};

std::unique_ptr<Result> lobpcg_solve(Ctx* ctx, Op* op, be_host_operator_fn host_op, void* host_user, index_t n,
                                     Tiles* tiles, const double* x0, const be_solver_config& cfg,
                                     be_observer_fn observer, void* observer_user);

// incremental driver (bench / iteration-level timing)
void* lobpcg_begin(Ctx* ctx, Op* op, be_host_operator_fn host_op, void* host_user, index_t n, Tiles* tiles,
                   const double* x0, const be_solver_config& cfg);
int lobpcg_step(void* h, int count);
std::unique_ptr<Result> lobpcg_end(void* h);
void lobpcg_abort(void* h);

}  // namespace be

struct be_result {
    std::unique_ptr<be::Result> impl;
};
