// C ABI edge of libblockeig_b200.so: every exported function catches the
// library's Failure (and CUDA/std errors) and turns it into a be_status with a
// thread-local message, mirroring the exception taxonomy of errors.hpp.
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <csignal>
#include <cstdlib>
#include <execinfo.h>
#include <unistd.h>
#include <cstring>
#include <sstream>
#include <tuple>
#include <vector>
#include <string>

#include "comm.hpp"
#include "densela.cuh"
#include "hostcopy.hpp"
#include "device.hpp"
#include "lobpcg.cuh"
#include "matrix_market.hpp"
#include "precond.cuh"
#include "tri_layout.hpp"

namespace {
thread_local std::string g_err;
thread_local int g_pivot = -1;

template <class F>
be_status guard(F&& f) {
    try {
        f();
        return BE_OK;
    } catch (const be::Failure& e) {
        g_err = e.what();
        g_pivot = e.pivot;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return BE_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return BE_ERR_GENERIC;
    } catch (...) {
        g_err = "unknown error";
        return BE_ERR_GENERIC;
    }
}
}  // namespace

struct be_csb {
    std::unique_ptr<be::CsbHost> impl;
};
struct be_synth {
    std::unique_ptr<be::Synth> impl;
};

extern "C" {

const char* be_last_error(void) { return g_err.c_str(); }
int be_last_error_pivot(void) { return g_pivot; }
const char* be_version(void) { return "blockeig_b200 0.1 (sm_100a)"; }
void be_free_buffer(void* p) { std::free(p); }

// ---------------------------------------------------------------- host CSB
be_status be_csb_build(const be_triple* triples, int64_t count, int64_t nrows, int64_t ncols,
                       const int64_t* row_bounds, int64_t n_row_bounds, const int64_t* col_bounds,
                       int64_t n_col_bounds, be_csb** out) {
    return guard([&] {
        if (!out || (count > 0 && !triples) || !row_bounds || !col_bounds) be::fail(BE_ERR_BAD_PARAMS, "be_csb_build: null argument");
        auto m = be::build_csb(triples, count, nrows, ncols, row_bounds, n_row_bounds, col_bounds, n_col_bounds);
        *out = new be_csb{std::move(m)};
    });
}

be_status be_uniform_boundaries(int64_t n, int64_t extent, int64_t* out, int64_t* count) {
    return guard([&] {
        auto b = be::uniform_boundaries(n, extent);
        if (count) *count = static_cast<int64_t>(b.size());
        if (out) std::memcpy(out, b.data(), b.size() * sizeof(int64_t));
    });
}

be_status be_random_block(int64_t n, int64_t nb, uint64_t seed, int64_t row_lo, double* out) {
    return guard([&] {
        if (!out || n < 0 || nb < 1 || row_lo < 0) be::fail(BE_ERR_BAD_PARAMS, "be_random_block: bad argument");
        const auto x = be::random_block(n, nb, seed, row_lo);
        std::memcpy(out, x.data(), x.size() * sizeof(double));
    });
}

be_status be_csb_view_get(const be_csb* m, be_csb_view* view) {
    return guard([&] {
        if (!m || !view) be::fail(BE_ERR_BAD_PARAMS, "be_csb_view_get: null argument");
        *view = m->impl->view();
    });
}

be_status be_csb_is_strictly_lower(const be_csb_view* view, int* result) {
    return guard([&] {
        if (!view || !result) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        be::validate_view(*view);
        *result = be::is_strictly_lower(*view) ? 1 : 0;
    });
}

be_status be_csb_to_triples(const be_csb_view* view, be_triple* out) {
    return guard([&] {
        if (!view || (view->nnz > 0 && !out)) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        be::validate_view(*view);
        be::to_triples(*view, out);
    });
}

be_status be_csb_save(const char* path, const be_csb_view* view, const double* diag, int64_t ndiag) {
    return guard([&] {
        if (!path || !view) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        be::validate_view(*view);
        be::save_csb1(path, *view, diag, ndiag);
    });
}

be_status be_csb_load(const char* path, be_csb** out, double** diag, int64_t* ndiag) {
    return guard([&] {
        if (!path || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        std::vector<double> d;
        auto m = be::load_csb1(path, diag ? &d : nullptr);
        if (diag) {
            *diag = nullptr;
            if (!d.empty()) {
                *diag = static_cast<double*>(std::malloc(d.size() * sizeof(double)));
                std::memcpy(*diag, d.data(), d.size() * sizeof(double));
            }
            if (ndiag) *ndiag = static_cast<int64_t>(d.size());
        }
        *out = new be_csb{std::move(m)};
    });
}

be_status be_csb_save_mem(const be_csb_view* view, const double* diag, int64_t ndiag, char** bytes, int64_t* len) {
    return guard([&] {
        if (!view || !bytes || !len) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        be::validate_view(*view);
        std::ostringstream os(std::ios::binary);
        be::save_csb1(os, *view, diag, ndiag);
        const std::string b = os.str();
        *bytes = static_cast<char*>(std::malloc(std::max<std::size_t>(b.size(), 1)));
        if (!*bytes) be::fail(BE_ERR_OUT_OF_MEMORY, "be_csb_save_mem: host allocation failed");
        std::memcpy(*bytes, b.data(), b.size());
        *len = static_cast<int64_t>(b.size());
    });
}

be_status be_csb_load_mem(const char* bytes, int64_t len, be_csb** out, double** diag, int64_t* ndiag) {
    return guard([&] {
        if ((!bytes && len > 0) || len < 0 || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        std::istringstream is(std::string(bytes ? bytes : "", static_cast<std::size_t>(len)), std::ios::binary);
        std::vector<double> d;
        auto m = be::load_csb1(is, diag ? &d : nullptr);
        if (diag) {
            *diag = nullptr;
            if (!d.empty()) {
                *diag = static_cast<double*>(std::malloc(d.size() * sizeof(double)));
                std::memcpy(*diag, d.data(), d.size() * sizeof(double));
            }
            if (ndiag) *ndiag = static_cast<int64_t>(d.size());
        }
        *out = new be_csb{std::move(m)};
    });
}

be_status be_csb_load_rows(const char* path, int64_t brow_begin, int64_t brow_end, be_csb** out, double** diag,
                           int64_t* ndiag) {
    return guard([&] {
        if (!path || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        std::vector<double> d;
        auto m = be::load_csb1_rows(path, brow_begin, brow_end, diag ? &d : nullptr);
        if (diag) {
            *diag = nullptr;
            if (!d.empty()) {
                *diag = static_cast<double*>(std::malloc(d.size() * sizeof(double)));
                std::memcpy(*diag, d.data(), d.size() * sizeof(double));
            }
        }
        if (ndiag) *ndiag = static_cast<int64_t>(d.size());
        *out = new be_csb{std::move(m)};
    });
}

void be_csb_free(be_csb* m) { delete m; }

// ----------------------------------------------------------- Matrix Market
namespace {
void mm_out(be::MmMatrix&& m, int64_t* n, be_triple** lower, int64_t* nlower, double** diag) {
    if (n) *n = m.n;
    if (nlower) *nlower = static_cast<int64_t>(m.lower.size());
    if (lower) {
        *lower = static_cast<be_triple*>(std::malloc(std::max<std::size_t>(m.lower.size(), 1) * sizeof(be_triple)));
        if (!*lower) be::fail(BE_ERR_OUT_OF_MEMORY, "matrix market: host allocation failed");
        if (!m.lower.empty()) std::memcpy(*lower, m.lower.data(), m.lower.size() * sizeof(be_triple));
    }
    if (diag) {
        *diag = static_cast<double*>(std::malloc(std::max<std::size_t>(m.diag.size(), 1) * sizeof(double)));
        if (!*diag) be::fail(BE_ERR_OUT_OF_MEMORY, "matrix market: host allocation failed");
        if (!m.diag.empty()) std::memcpy(*diag, m.diag.data(), m.diag.size() * sizeof(double));
    }
}
}  // namespace

be_status be_mm_parse(const char* text, int64_t len, int64_t* n, be_triple** lower, int64_t* nlower, double** diag) {
    return guard([&] {
        if (!text || len < 0) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        mm_out(be::parse_matrix_market(text, static_cast<std::size_t>(len)), n, lower, nlower, diag);
    });
}

be_status be_mm_read_file(const char* path, int64_t* n, be_triple** lower, int64_t* nlower, double** diag) {
    return guard([&] {
        if (!path) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        mm_out(be::read_matrix_market_file(path), n, lower, nlower, diag);
    });
}

be_status be_mm_write(int64_t n, const be_triple* lower, int64_t nlower, const double* diag, char** text,
                      int64_t* len) {
    return guard([&] {
        if ((!lower && nlower > 0) || (!diag && n > 0) || !text || n < 0 || nlower < 0)
            be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const std::string s = be::write_matrix_market(n, lower, nlower, diag);
        *text = static_cast<char*>(std::malloc(s.size() + 1));
        if (!*text) be::fail(BE_ERR_OUT_OF_MEMORY, "matrix market: host allocation failed");
        std::memcpy(*text, s.c_str(), s.size() + 1);
        if (len) *len = static_cast<int64_t>(s.size());
    });
}

// --------------------------------------------------------------- generators
be_status be_generate_synthetic(const be_synth_params* p, be_synth** out) {
    return guard([&] {
        if (!p || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *out = new be_synth{be::generate_synthetic(*p)};
    });
}

be_status be_synth_get(const be_synth* s, const be_triple** lower, int64_t* nlower, const double** diag,
                       const int64_t** tile_offsets, int64_t* n_tile_offsets) {
    return guard([&] {
        if (!s) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (lower) *lower = s->impl->lower.data();
        if (nlower) *nlower = static_cast<int64_t>(s->impl->lower.size());
        if (diag) *diag = s->impl->diag.data();
        if (tile_offsets) *tile_offsets = s->impl->tile_offsets.data();
        if (n_tile_offsets) *n_tile_offsets = static_cast<int64_t>(s->impl->tile_offsets.size());
    });
}

void be_synth_free(be_synth* s) { delete s; }

be_status be_generate_clustered(const be_cluster_params* p, be_csb** out, double** diag, int64_t** tile_offsets,
                                int64_t* n_tile_offsets) {
    return guard([&] {
        if (!p || !out || !diag || !tile_offsets || !n_tile_offsets) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        std::vector<double> d;
        std::vector<int64_t> t;
        auto m = be::generate_clustered(*p, d, t);
        *diag = static_cast<double*>(std::malloc(d.size() * sizeof(double)));
        std::memcpy(*diag, d.data(), d.size() * sizeof(double));
        *tile_offsets = static_cast<int64_t*>(std::malloc(t.size() * sizeof(int64_t)));
        std::memcpy(*tile_offsets, t.data(), t.size() * sizeof(int64_t));
        *n_tile_offsets = static_cast<int64_t>(t.size());
        *out = new be_csb{std::move(m)};
    });
}

be_status be_generate_clustered_part(const be_cluster_params* p, int64_t brow_begin, int64_t brow_end,
                                     int diag_blocks_only, be_csb** out, double** rowabs,
                                     int64_t** tile_offsets, int64_t* n_tile_offsets) {
    return guard([&] {
        if (!p || !out || !rowabs || !tile_offsets || !n_tile_offsets) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        std::vector<double> r;
        std::vector<int64_t> t;
        auto m = be::generate_clustered_part(*p, brow_begin, brow_end, diag_blocks_only != 0, r, t);
        *rowabs = static_cast<double*>(std::malloc(r.size() * sizeof(double)));
        std::memcpy(*rowabs, r.data(), r.size() * sizeof(double));
        *tile_offsets = static_cast<int64_t*>(std::malloc(t.size() * sizeof(int64_t)));
        std::memcpy(*tile_offsets, t.data(), t.size() * sizeof(int64_t));
        *n_tile_offsets = static_cast<int64_t>(t.size());
        *out = new be_csb{std::move(m)};
    });
}

be_status be_generate_clustered_tile(const be_cluster_params* p, int64_t brow_begin, int64_t brow_end,
                                     int64_t bcol_begin, int64_t bcol_end, be_csb** out, double** rowabs,
                                     int64_t** tile_offsets, int64_t* n_tile_offsets) {
    return guard([&] {
        if (!p || !out || !rowabs || !tile_offsets || !n_tile_offsets) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        std::vector<double> r;
        std::vector<int64_t> t;
        auto m = be::generate_clustered_part(*p, brow_begin, brow_end, false, r, t, bcol_begin, bcol_end);
        *rowabs = static_cast<double*>(std::malloc(r.size() * sizeof(double)));
        std::memcpy(*rowabs, r.data(), r.size() * sizeof(double));
        *tile_offsets = static_cast<int64_t*>(std::malloc(t.size() * sizeof(int64_t)));
        std::memcpy(*tile_offsets, t.data(), t.size() * sizeof(int64_t));
        *n_tile_offsets = static_cast<int64_t>(t.size());
        *out = new be_csb{std::move(m)};
    });
}

be_status be_clustered_block_weights(const be_cluster_params* p, int64_t* weights, int64_t* nblk) {
    return guard([&] {
        if (!p || !nblk) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        int64_t nb = 0;
        const auto w = be::clustered_block_weights(*p, nb);
        *nblk = nb;
        if (weights) std::memcpy(weights, w.data(), w.size() * sizeof(int64_t));
    });
}

be_status be_clustered_diag(const be_cluster_params* p, const double* rowabs, int64_t row_begin, int64_t row_end,
                            double* diag) {
    return guard([&] {
        if (!p || (!rowabs && row_end > row_begin) || (!diag && row_end > row_begin)) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (row_begin < 0 || row_end < row_begin || row_end > p->n) be::fail(BE_ERR_BAD_PARAMS, "be_clustered_diag: bad row range");
        for (int64_t i = row_begin; i < row_end; ++i) diag[i - row_begin] = be::clustered_diag_value(*p, i, rowabs[i - row_begin]);
    });
}

be_status be_clustered_weights(const be_cluster_params* p, int64_t* weights, int64_t* nblk) {
    return guard([&] {
        if (!p || !nblk) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const auto w = be::clustered_block_row_weights(*p);
        *nblk = static_cast<int64_t>(w.size());
        if (weights) std::memcpy(weights, w.data(), w.size() * sizeof(int64_t));
    });
}

// BE_SEGV_TRACE=1: native backtrace on SIGSEGV/SIGABRT (addresses resolve with addr2line -e the .so)
namespace {
void be_segv_handler(int sig) {
    void* frames[64];
    const int n = backtrace(frames, 64);
    const char msg[] = "blockeig_b200: native backtrace\n";
    (void)!write(2, msg, sizeof(msg) - 1);
    backtrace_symbols_fd(frames, n, 2);
    std::signal(sig, SIG_DFL);
    std::raise(sig);
}
struct SegvTrace {
    SegvTrace() {
        if (std::getenv("BE_SEGV_TRACE")) {
            std::signal(SIGSEGV, be_segv_handler);
            std::signal(SIGABRT, be_segv_handler);
        }
    }
} g_segv_trace;
}  // namespace

// ------------------------------------------------------------------ context
be_status be_ctx_create(int device, be_ctx** out) {
    return guard([&] {
        if (!out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            be::fail(BE_ERR_NO_DEVICE, "no CUDA device available");
        }
        if (device < 0 || device >= ndev) be::fail(BE_ERR_NO_DEVICE, "device index out of range");
        auto c = std::make_unique<be::Ctx>();
        c->device = device;
        BE_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        BE_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) be::fail(BE_ERR_NO_DEVICE, "blockeig_b200 needs an sm_100 (B200) device");
        c->num_sms = prop.multiProcessorCount;
        BE_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        be::hostcopy_prepare(device);  // pinned staging for the host-buffer calls, allocated once
        *out = new be_ctx{std::move(c)};
    });
}

be_status be_ctx_destroy(be_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        if (ctx->impl->solver) cusolverDnDestroy(ctx->impl->solver);
        if (ctx->impl->blas) cublasDestroy(ctx->impl->blas);
        if (ctx->impl->stream) cudaStreamDestroy(ctx->impl->stream);
        delete ctx;
    });
}

be_status be_ctx_stream(be_ctx* ctx, void** stream) {
    return guard([&] {
        if (!ctx || !stream) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *stream = ctx->impl->stream;
    });
}

be_status be_ctx_synchronize(be_ctx* ctx) {
    return guard([&] {
        if (!ctx) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        BE_CUDA(cudaSetDevice(ctx->impl->device));
        BE_CUDA(cudaStreamSynchronize(ctx->impl->stream));
    });
}

be_status be_ctx_launches(be_ctx* ctx, int64_t* launches) {
    return guard([&] {
        if (!ctx || !launches) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *launches = ctx->impl->launches;
    });
}

// ------------------------------------------------------------------ operator
be_status be_op_create(be_ctx* ctx, const be_csb_view* L, const double* diag, int values_prec, int flags, be_op** out) {
    return guard([&] {
        if (!ctx || !L || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        BE_CUDA(cudaSetDevice(ctx->impl->device));
        *out = new be_op{be::op_create(ctx->impl.get(), *L, diag, values_prec, flags)};
    });
}

be_status be_op_create_csb1(be_ctx* ctx, const char* path, int values_prec, int flags, int64_t batch_entries,
                           double** diag, int64_t* ndiag, be_op** out) {
    return guard([&] {
        if (!ctx || !path || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        BE_CUDA(cudaSetDevice(ctx->impl->device));
        std::vector<double> d;
        auto op = be::op_create_csb1(ctx->impl.get(), path, values_prec, flags, diag ? &d : nullptr, batch_entries);
        if (diag) {
            *diag = static_cast<double*>(std::malloc(std::max<std::size_t>(d.size(), 1) * sizeof(double)));
            std::memcpy(*diag, d.data(), d.size() * sizeof(double));
        }
        if (ndiag) *ndiag = static_cast<int64_t>(d.size());
        *out = new be_op{std::move(op)};
    });
}

be_status be_op_destroy(be_op* op) {
    return guard([&] { delete op; });
}

be_status be_op_apply(be_op* op, const void* X_dev, void* Y_dev, int64_t nrows, int nb, int panel_prec, int mode,
                      void* stream) {
    return guard([&] {
        if (!op || !X_dev || !Y_dev) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        auto* o = op->impl.get();
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : o->ctx->stream;
        be::op_apply(o, X_dev, Y_dev, nrows, nb, panel_prec, mode, s);
    });
}

be_status be_op_apply_host(be_op* op, const double* X, double* Y, int64_t nrows, int nb, int mode) {
    return guard([&] {
        if (!op || !X || !Y) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        auto* o = op->impl.get();
        if (X == Y) be::fail(BE_ERR_BAD_PARAMS, "spmm: W and U must not alias");
        if (mode == BE_APPLY_SYMMETRIC && !o->symmetric) be::fail(BE_ERR_BAD_PARAMS, "apply: symmetric mode needs a symmetric operator");
        if (mode < 0 || mode > 2) be::fail(BE_ERR_BAD_PARAMS, "apply: unknown mode");
        const int64_t out_rows = mode == BE_APPLY_TRANS_ACC ? o->ncols : o->nrows;
        const int64_t in_rows = mode == BE_APPLY_NOTRANS_ACC ? o->ncols : o->nrows;
        if (nrows != in_rows) be::fail(BE_ERR_DIMENSION_MISMATCH, "apply: shape mismatch");
        if (nb < 1) be::fail(BE_ERR_DIMENSION_MISMATCH, "apply: nb must be positive");
        cudaStream_t s = o->ctx->stream;
        be::DBuf<double> dx(std::max<int64_t>(in_rows * nb, 1)), dy(std::max<int64_t>(out_rows * nb, 1));
        BE_CUDA(cudaMemcpyAsync(dx.get(), X, static_cast<std::size_t>(in_rows * nb) * 8, cudaMemcpyHostToDevice, s));
        if (mode != BE_APPLY_SYMMETRIC)
            BE_CUDA(cudaMemcpyAsync(dy.get(), Y, static_cast<std::size_t>(out_rows * nb) * 8, cudaMemcpyHostToDevice, s));
        be::op_apply(o, dx.get(), dy.get(), nrows, nb, BE_F64, mode, s);
        BE_CUDA(cudaMemcpyAsync(Y, dy.get(), static_cast<std::size_t>(out_rows * nb) * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
    });
}

be_status be_op_get_info(const be_op* op, be_op_info* info) {
    return guard([&] {
        if (!op || !info) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const auto* o = op->impl.get();
        std::memset(info, 0, sizeof(*info));
        info->nrows = o->nrows;
        info->ncols = o->ncols;
        info->nnz = o->nnz;
        info->ntiles = o->ntiles;
        info->device_bytes = static_cast<int64_t>(o->tiles.bytes() + o->runs.bytes() + o->runs_ext.bytes() + o->blobs.bytes() +
                                                  o->det_ptr_n.bytes() + o->det_ptr_t.bytes() + o->det_col.bytes() +
                                                  o->det_val.bytes() + o->rows_val.bytes());
        info->bytes_per_nnz_x1000 = o->nnz ? info->device_bytes * 1000 / o->nnz : 0;
        info->values_prec = o->values_prec;
        info->tile_rows = be::kTile;
        info->tile_cols = be::kTile;
        info->tile_max_nnz = o->max_nnz;
    });
}

be_status be_op_decode(be_op* op, int64_t* rows, int64_t* cols, double* values, int64_t* csb_index) {
    return guard([&] {
        if (!op) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        auto* o = op->impl.get();
        if (o->det || o->rows) be::fail(BE_ERR_BAD_PARAMS, "be_op_decode: operator has no tile format (row-list format)");
        if (o->csb_index.size() != static_cast<std::size_t>(o->padded) || (o->padded == 0 && o->nnz > 0))
            be::fail(BE_ERR_BAD_PARAMS, "be_op_decode: source index not retained for matrices this large");
        std::vector<be::TileHdr> h(static_cast<std::size_t>(o->ntiles));
        std::vector<unsigned char> blob(static_cast<std::size_t>(o->blob_total));
        const std::size_t vsz = o->values_prec == BE_F32 ? 4 : 8;
        if (o->ntiles > 0) {
            BE_CUDA(cudaMemcpy(h.data(), o->tiles.get(), h.size() * sizeof(be::TileHdr), cudaMemcpyDeviceToHost));
            BE_CUDA(cudaMemcpy(blob.data(), o->blobs.get(), blob.size(), cudaMemcpyDeviceToHost));
        }
        auto val = [&](const unsigned char* p) {
            if (vsz == 4) {
                float f;
                std::memcpy(&f, p, 4);
                return static_cast<double>(f);
            }
            double d;
            std::memcpy(&d, p, 8);
            return d;
        };
        // Blob layout (spmm.cu): meta kBlobMeta B = jr u16[136] | jc u16[136] | rank->row u8[128] |
        // rank->col u8[128] | row lengths | column lengths; then values + columns in row-JDS
        // order and values + rows in column-JDS order, npad = nnz rounded up to 16 each.
        // Both orders are validated (ranks by decreasing length, starts = prefix sums of
        // min(len, d), both orders the same entry set); entries come out in row order.
        int64_t p = 0, slot = 0;
        for (const auto& t : h) {
            const int nnz = static_cast<int>(t.packed >> 14), npad = (nnz + 15) & ~15;
            const int nr = static_cast<int>(t.packed & 127u) + 1;
            const int nc = static_cast<int>((t.packed >> 7) & 127u) + 1;
            const unsigned char* b = blob.data() + static_cast<std::size_t>(t.begin16) * 16;
            const std::uint16_t* jd[2] = {reinterpret_cast<const std::uint16_t*>(b), reinterpret_cast<const std::uint16_t*>(b + 272)};
            const unsigned char* perm[2] = {b + 544, b + 672};
            const unsigned char* len[2] = {b + 800, b + 928};
            const unsigned char* sv[2] = {b + be::kBlobMeta, b + be::kBlobMeta + static_cast<std::size_t>(npad) * (vsz + 1)};
            const unsigned char* si[2] = {b + be::kBlobMeta + static_cast<std::size_t>(npad) * vsz,
                                          b + be::kBlobMeta + static_cast<std::size_t>(npad) * (2 * vsz + 1)};
            std::vector<std::tuple<int, int, std::uint64_t>> got[2];
            for (int g = 0; g < 2; ++g) {
                int sum = 0;
                std::vector<char> used(128, 0);
                for (int i = 0; i < 128; ++i) {
                    if (i > 0 && len[g][i] > len[g][i - 1]) be::fail(BE_ERR_GENERIC, "decode: lengths not in rank order");
                    if (used[perm[g][i]]) be::fail(BE_ERR_GENERIC, "decode: rank map is not a permutation");
                    used[perm[g][i]] = 1;
                    sum += len[g][i];
                }
                if (sum != nnz) be::fail(BE_ERR_GENERIC, "decode: lengths do not sum to the tile size");
                for (int d = 0; d <= 128; ++d) {
                    int s = 0;
                    for (int i = 0; i < 128; ++i) s += std::min<int>(len[g][i], d);
                    if (jd[g][d] != s) be::fail(BE_ERR_GENERIC, "decode: JDS starts inconsistent with the lengths");
                }
                for (int r = 0; r < 128; ++r)
                    for (int d = 0; d < len[g][r]; ++d) {
                        const int q = jd[g][d] + r;
                        const int other = si[g][q];
                        const int row = g == 0 ? perm[g][r] : other, col = g == 0 ? other : perm[g][r];
                        if (row >= nr || col >= nc) be::fail(BE_ERR_GENERIC, "decode: local index outside tile");
                        std::uint64_t bits = 0;
                        const double v = val(sv[g] + static_cast<std::size_t>(q) * vsz);
                        std::memcpy(&bits, &v, 8);
                        got[g].emplace_back(row, col, bits);
                        if (g == 0) {
                            if (rows) rows[p] = o->comm ? o->unpad(t.row0 + row) : t.row0 + row;
                            if (cols) cols[p] = o->comm ? o->unpad(t.col0 + col) : t.col0 + col;
                            if (values) values[p] = v;
                            if (csb_index) csb_index[p] = o->csb_index[static_cast<std::size_t>(slot + q)];
                            ++p;
                        }
                    }
            }
            std::sort(got[0].begin(), got[0].end());
            std::sort(got[1].begin(), got[1].end());
            if (got[0] != got[1]) be::fail(BE_ERR_GENERIC, "decode: row and column orders hold different entries");
            slot += npad;
        }
        if (p != o->nnz) be::fail(BE_ERR_GENERIC, "decode: entry count mismatch");
    });
}

be_status be_op_timing(be_op* op, int enable, double* last_kernel_ms, double* last_apply_ms) {
    return guard([&] {
        if (!op) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        auto* o = op->impl.get();
        if (enable >= 0) o->timing = enable != 0;
        if (last_kernel_ms) *last_kernel_ms = o->last_kernel_ms;
        if (last_apply_ms) *last_apply_ms = o->last_apply_ms;
    });
}

// ----------------------------------------------------------- preconditioner
be_status be_tiles_create(be_ctx* ctx, const be_csb_view* L, const double* diag, const int64_t* tile_offsets,
                          int64_t n_tile_offsets, be_tiles** out) {
    return guard([&] {
        if (!ctx || !L || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        BE_CUDA(cudaSetDevice(ctx->impl->device));
        *out = new be_tiles{be::tiles_create(ctx->impl.get(), *L, diag, tile_offsets, n_tile_offsets)};
    });
}

be_status be_tiles_create_range(be_ctx* ctx, const be_csb_view* L, const double* diag_local,
                                const int64_t* tile_offsets, int64_t n_tile_offsets, int64_t row_begin,
                                int64_t row_end, be_tiles** out) {
    return guard([&] {
        if (!ctx || !L || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (row_begin < 0 || row_end < row_begin) be::fail(BE_ERR_BAD_PARAMS, "be_tiles_create_range: bad row range");
        BE_CUDA(cudaSetDevice(ctx->impl->device));
        *out = new be_tiles{be::tiles_create(ctx->impl.get(), *L, diag_local, tile_offsets, n_tile_offsets, row_begin,
                                             row_end)};
    });
}

// ------------------------------------------------------------------ multi-GPU
be_status be_comm_nccl_id(uint8_t id[128]) {
    return guard([&] {
        if (!id) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        be::nccl_unique_id(id);
    });
}

be_status be_comm_create_nccl(be_ctx* ctx, const uint8_t id[128], int rank, int world, be_comm** out) {
    return guard([&] {
        if (!ctx || !id || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *out = new be_comm{be::make_nccl_comm(ctx->impl->device, id, rank, world)};
    });
}

be_status be_comm_group_create(int world, be_comm_group** out) {
    return guard([&] {
        if (!out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *out = new be_comm_group{std::make_unique<be::LocalGroup>(world)};
    });
}

be_status be_comm_group_destroy(be_comm_group* g) {
    return guard([&] { delete g; });
}

be_status be_comm_group_abort(be_comm_group* g) {
    return guard([&] {
        if (!g) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        g->impl->abort();
    });
}

be_status be_comm_create_local(be_ctx* ctx, be_comm_group* g, int rank, be_comm** out) {
    return guard([&] {
        if (!ctx || !g || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *out = new be_comm{be::make_local_comm(ctx->impl->device, g->impl.get(), rank)};
    });
}

be_status be_comm_destroy(be_comm* c) {
    return guard([&] { delete c; });
}

be_status be_comm_info(const be_comm* c, int* rank, int* world, int* backend, int64_t* calls, int64_t* bytes) {
    return guard([&] {
        if (!c) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const auto* k = c->impl.get();
        if (rank) *rank = k->rank;
        if (world) *world = k->world;
        if (backend) *backend = std::strcmp(k->backend(), "nccl") == 0 ? 0 : 1;
        if (calls) *calls = k->calls;
        if (bytes) *bytes = k->bytes_moved;
    });
}

be_status be_comm_allreduce_f64(be_comm* c, double* buf_dev, int64_t count, void* stream) {
    return guard([&] {
        if (!c || (!buf_dev && count > 0)) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (count < 0) be::fail(BE_ERR_BAD_PARAMS, "be_comm_allreduce_f64: negative count");
        BE_CUDA(cudaSetDevice(c->impl->device));
        c->impl->allreduce_f64(buf_dev, static_cast<std::size_t>(count), static_cast<cudaStream_t>(stream));
    });
}

be_status be_dist_rows(const int64_t* bounds, int64_t nbounds, int world, int64_t* cuts) {
    return guard([&] {
        if (!bounds || !cuts || nbounds < 2) be::fail(BE_ERR_BAD_PARAMS, "be_dist_rows: bad arguments");
        for (int64_t i = 1; i < nbounds; ++i)
            if (bounds[i] <= bounds[i - 1]) be::fail(BE_ERR_BAD_PARAMS, "be_dist_rows: boundaries must be strictly increasing");
        const auto c = be::dist_rows(bounds, nbounds, world);
        std::memcpy(cuts, c.data(), c.size() * sizeof(int64_t));
    });
}

be_status be_dist_balance(const int64_t* weights, int64_t nitems, int world, int64_t* cuts) {
    return guard([&] {
        if ((!weights && nitems > 0) || !cuts || nitems < 0) be::fail(BE_ERR_BAD_PARAMS, "be_dist_balance: bad arguments");
        const auto c = be::dist_balance(weights, nitems, world);
        std::memcpy(cuts, c.data(), c.size() * sizeof(int64_t));
    });
}

be_status be_dist_tiles2d(const int64_t* weights, int64_t nblk, const int64_t* bounds, int world, int64_t* rects) {
    return guard([&] {
        if (!weights || !bounds || !rects || nblk < 1) be::fail(BE_ERR_BAD_PARAMS, "be_dist_tiles2d: bad arguments");
        for (int64_t i = 1; i <= nblk; ++i)
            if (bounds[i] <= bounds[i - 1]) be::fail(BE_ERR_BAD_PARAMS, "be_dist_tiles2d: boundaries must be strictly increasing");
        const auto r = be::dist_tiles2d(weights, nblk, bounds, world);
        std::memcpy(rects, r.data(), r.size() * sizeof(int64_t));
    });
}

be_status be_op_create_dist(be_ctx* ctx, be_comm* comm, const be_csb_view* L_slab, const int64_t* cuts,
                            const double* diag_local, int values_prec, be_op** out) {
    return guard([&] {
        if (!ctx || !comm || !L_slab || !cuts || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        BE_CUDA(cudaSetDevice(ctx->impl->device));
        *out = new be_op{be::op_create_dist(ctx->impl.get(), comm->impl.get(), *L_slab, cuts, nullptr, diag_local,
                                            values_prec)};
    });
}

be_status be_op_create_dist_owned(be_ctx* ctx, be_comm* comm, const be_csb_view* L_slab, const int64_t* seg_bounds,
                                  const int* seg_owner, const double* diag_local, int values_prec, be_op** out) {
    return guard([&] {
        if (!ctx || !comm || !L_slab || !seg_bounds || !seg_owner || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        BE_CUDA(cudaSetDevice(ctx->impl->device));
        *out = new be_op{be::op_create_dist(ctx->impl.get(), comm->impl.get(), *L_slab, seg_bounds, seg_owner,
                                            diag_local, values_prec)};
    });
}

// ------------------------------------------------- reference triangular layout
be_status be_tri_layout(int nd, int* blocks, int* diagonal_ranks, int* n_ranks) {
    return guard([&] {
        const auto lt = be::build_tri_layout(nd);
        if (n_ranks) *n_ranks = lt.n_ranks;
        if (blocks)
            for (int r = 0; r < lt.n_ranks; ++r)
                for (int k = 0; k < 3; ++k) blocks[3 * r + k] = lt.blocks[static_cast<std::size_t>(r)][static_cast<std::size_t>(k)];
        if (diagonal_ranks)
            for (int g = 0; g < nd; ++g) diagonal_ranks[g] = lt.diagonal_ranks[static_cast<std::size_t>(g)];
    });
}

be_status be_tri_segments(int nd, const int64_t* sub_bounds, int64_t* seg_begin, int64_t* seg_end) {
    return guard([&] {
        if (!sub_bounds || !seg_begin || !seg_end) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const auto lt = be::build_tri_layout(nd);
        const auto seg = be::tri_segments(lt, sub_bounds);
        for (int r = 0; r < lt.n_ranks; ++r) {
            seg_begin[r] = seg[static_cast<std::size_t>(r)].first;
            seg_end[r] = seg[static_cast<std::size_t>(r)].second;
        }
    });
}

be_status be_tri_rank_triples(const be_csb_view* L, int nd, const int64_t* sub_bounds, int rank, be_triple* out,
                              int64_t* count) {
    return guard([&] {
        if (!L || !sub_bounds || !count) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        be::validate_view(*L);
        const auto lt = be::build_tri_layout(nd);
        const auto t = be::tri_rank_triples(*L, lt, sub_bounds, rank);
        if (out) {
            if (*count < static_cast<int64_t>(t.size())) be::fail(BE_ERR_BAD_PARAMS, "be_tri_rank_triples: buffer too small");
            std::memcpy(out, t.data(), t.size() * sizeof(be_triple));
        }
        *count = static_cast<int64_t>(t.size());
    });
}

be_status be_tiles_destroy(be_tiles* t) {
    return guard([&] { delete t; });
}

be_status be_tiles_count(const be_tiles* t, int64_t* count, int64_t* dim, int64_t* nentries) {
    return guard([&] {
        if (!t) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (count) *count = t->impl->ntiles;
        if (dim) *dim = t->impl->n;
        if (nentries) *nentries = t->impl->nentries;
    });
}

be_status be_tiles_get(const be_tiles* t, int64_t j, int64_t* dim, int64_t* nentries, int32_t* rows, int32_t* cols,
                       double* values, int64_t* diag_pos) {
    return guard([&] {
        if (!t) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (j < 0 || j >= t->impl->ntiles) be::fail(BE_ERR_BAD_PARAMS, "be_tiles_get: tile index out of range");
        const auto& T = t->impl->host[static_cast<std::size_t>(j)];
        if (dim) *dim = T.dim;
        if (nentries) *nentries = static_cast<int64_t>(T.vals.size());
        if (rows) std::memcpy(rows, T.rows.data(), T.rows.size() * 4);
        if (cols) std::memcpy(cols, T.cols.data(), T.cols.size() * 4);
        if (values) std::memcpy(values, T.vals.data(), T.vals.size() * 8);
        if (diag_pos) std::memcpy(diag_pos, T.diag_pos.data(), T.diag_pos.size() * 8);
    });
}

be_status be_precond_apply(be_tiles* t, const double* shifts_dev, const double* R_dev, double* W_dev, int64_t nrows,
                           int nb, int m, int64_t* fallbacks_dev, void* stream) {
    return guard([&] {
        if (!t || !shifts_dev || !R_dev || !W_dev) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->impl->ctx->stream;
        be::precond_apply(t->impl.get(), shifts_dev, R_dev, W_dev, nrows, nb, m, fallbacks_dev, s);
    });
}

be_status be_tiles_create_explicit(be_ctx* ctx, int64_t ntiles, const int64_t* dims, const int64_t* entry_offsets,
                                   const int32_t* rows, const int32_t* cols, const double* values,
                                   const int64_t* diag_pos, be_tiles** out) {
    return guard([&] {
        if (!ctx || !out || ntiles < 0 || (ntiles > 0 && (!dims || !entry_offsets || !diag_pos)))
            be::fail(BE_ERR_BAD_PARAMS, "null argument");
        std::vector<be::HostTile> ts(static_cast<std::size_t>(ntiles));
        int64_t row0 = 0;
        for (int64_t j = 0; j < ntiles; ++j) {
            auto& T = ts[static_cast<std::size_t>(j)];
            T.dim = dims[j];
            const int64_t e0 = entry_offsets[j], e1 = entry_offsets[j + 1];
            if (e1 < e0) be::fail(BE_ERR_BAD_PARAMS, "be_tiles_create_explicit: entry offsets must not decrease");
            if (e1 > e0 && (!rows || !cols || !values)) be::fail(BE_ERR_BAD_PARAMS, "null argument");
            T.rows.assign(rows + e0, rows + e1);
            T.cols.assign(cols + e0, cols + e1);
            T.vals.assign(values + e0, values + e1);
            if (T.dim > 0) T.diag_pos.assign(diag_pos + row0, diag_pos + row0 + T.dim);
            row0 += std::max<int64_t>(T.dim, 0);
        }
        *out = new be_tiles{be::tiles_create_explicit(ctx->impl.get(), ts)};
    });
}

be_status be_precond_apply_host(be_tiles* t, const double* shifts, const double* R, double* W, int64_t nrows, int nb,
                                int m, int64_t* fallbacks) {
    return guard([&] {
        if (!t || !shifts || !R || !W) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (nrows != t->impl->n) be::fail(BE_ERR_DIMENSION_MISMATCH, "apply_preconditioner: residual rows != operator dim");
        cudaStream_t s = t->impl->ctx->stream;
        const std::size_t bytes = static_cast<std::size_t>(nrows * nb) * 8;
        be::DBuf<double> dr(std::max<int64_t>(nrows * nb, 1)), dw(std::max<int64_t>(nrows * nb, 1)), ds(nb);
        be::DBuf<int64_t> df(1);
        BE_CUDA(cudaMemcpyAsync(dr.get(), R, bytes, cudaMemcpyHostToDevice, s));
        BE_CUDA(cudaMemcpyAsync(ds.get(), shifts, static_cast<std::size_t>(nb) * 8, cudaMemcpyHostToDevice, s));
        BE_CUDA(cudaMemsetAsync(df.get(), 0, 8, s));
        be::precond_apply(t->impl.get(), ds.get(), dr.get(), dw.get(), nrows, nb, m, df.get(), s);
        BE_CUDA(cudaMemcpyAsync(W, dw.get(), bytes, cudaMemcpyDeviceToHost, s));
        int64_t f = 0;
        BE_CUDA(cudaMemcpyAsync(&f, df.get(), 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
        if (fallbacks) *fallbacks += f;
    });
}

// ------------------------------------------------------------------- LOBPCG
be_status be_lobpcg_solve(be_ctx* ctx, be_op* op, be_host_operator_fn host_op, void* host_op_user, int64_t n,
                          be_tiles* precond, const double* x0, const be_solver_config* cfg, be_observer_fn observer,
                          void* observer_user, be_result** out) {
    return guard([&] {
        if (!ctx || !cfg || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        auto r = be::lobpcg_solve(ctx->impl.get(), op ? op->impl.get() : nullptr, host_op, host_op_user, n,
                                  precond ? precond->impl.get() : nullptr, x0, *cfg, observer, observer_user);
        *out = new be_result{std::move(r)};
    });
}

be_status be_lobpcg_begin(be_ctx* ctx, be_op* op, be_host_operator_fn host_op, void* host_op_user, int64_t n,
                          be_tiles* precond, const double* x0, const be_solver_config* cfg, be_solver** out) {
    return guard([&] {
        if (!ctx || !cfg || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *out = static_cast<be_solver*>(be::lobpcg_begin(ctx->impl.get(), op ? op->impl.get() : nullptr, host_op,
                                                          host_op_user, n, precond ? precond->impl.get() : nullptr, x0,
                                                          *cfg));
    });
}

be_status be_lobpcg_step(be_solver* s, int count, int* done) {
    be_status st = guard([&] {
        if (!s) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const int d = be::lobpcg_step(s, count);
        if (done) *done = d;
    });
    return st;
}

be_status be_lobpcg_end(be_solver* s, be_result** out) {
    return guard([&] {
        if (!s || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        *out = new be_result{be::lobpcg_end(s)};
    });
}

be_status be_result_get_info(const be_result* r, be_result_info* info) {
    return guard([&] {
        if (!r || !info) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const auto& R = *r->impl;
        info->converged = R.converged ? 1 : 0;
        info->iterations = static_cast<int>(R.records.size());
        info->k = R.k;
        info->nb = R.nb;
        info->n = R.n;
        info->operator_calls = R.operator_calls;
        info->precond_fallbacks = R.precond_fallbacks;
        info->restarts = R.restarts;
    });
}

be_status be_result_get(const be_result* r, double* lambda, double* x) {
    return guard([&] {
        if (!r) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (lambda) std::memcpy(lambda, r->impl->lambda.data(), r->impl->lambda.size() * 8);
        if (x) {
            const auto& R = *r->impl;
            if (R.xdev.p) {
                BE_CUDA(cudaSetDevice(R.device));
                be::d2h_large(x, R.xdev.get(), static_cast<std::size_t>(R.n) * R.k * 8, nullptr);
            } else {
                std::memcpy(x, R.x.data(), R.x.size() * 8);
            }
        }
    });
}

be_status be_result_get_record(const be_result* r, int i, double* theta, double* residual_norms, int* n_converged,
                               double* t_spmm, double* t_precond, double* t_dense, double* t_total) {
    return guard([&] {
        if (!r) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (i < 0 || i >= static_cast<int>(r->impl->records.size())) be::fail(BE_ERR_BAD_PARAMS, "record index out of range");
        const auto& rec = r->impl->records[static_cast<std::size_t>(i)];
        if (theta) std::memcpy(theta, rec.theta.data(), rec.theta.size() * 8);
        if (residual_norms) std::memcpy(residual_norms, rec.resn.data(), rec.resn.size() * 8);
        if (n_converged) *n_converged = rec.nconv;
        if (t_spmm) *t_spmm = rec.t_spmm;
        if (t_precond) *t_precond = rec.t_precond;
        if (t_dense) *t_dense = rec.t_dense;
        if (t_total) *t_total = rec.t_total;
    });
}

void be_result_free(be_result* r) { delete r; }

// ------------------------------------------------------- dense parity hooks
be_status be_gram(be_ctx* ctx, const double* A_dev, int p, const double* B_dev, int q, int64_t n, double* out) {
    return guard([&] {
        if (!ctx || !A_dev || !B_dev || !out) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (p != q) be::fail(BE_ERR_BAD_PARAMS, "be_gram: the device kernel handles square p == q Grams");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        const int64_t plen = be::dla::gram_partials_len(p, 1, c->num_sms);
        be::DBuf<double> part(plen), o(static_cast<int64_t>(p) * q);
        be::dla::GramJob j{};
        j.npairs = 1;
        j.nb = p;
        j.a[0] = A_dev;
        j.b[0] = B_dev;
        j.sym[0] = A_dev == B_dev;
        j.out[0] = o.get();
        be::dla::gram(c, j, n, part.get(), plen, s);
        BE_CUDA(cudaMemcpyAsync(out, o.get(), static_cast<std::size_t>(p) * q * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
    });
}

be_status be_sygv_lowest(be_ctx* ctx, const double* A, const double* B, int n, int k, double pivot_floor, double* c,
                         double* d) {
    return guard([&] {
        if (!ctx || !A || !B || !c || !d) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        if (k < 1 || k > n) be::fail(BE_ERR_BAD_PARAMS, "sygv_lowest: k out of range");
        auto* cx = ctx->impl.get();
        cudaStream_t s = cx->stream;
        const std::size_t nn = static_cast<std::size_t>(n) * n;
        be::DBuf<double> dA(static_cast<int64_t>(nn)), dB(static_cast<int64_t>(nn)), dc(static_cast<int64_t>(n) * k), dd(k);
        be::DBuf<be::dla::Status> st(1);
        BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(be::dla::Status), s));
        BE_CUDA(cudaMemcpyAsync(dA.get(), A, nn * 8, cudaMemcpyHostToDevice, s));
        BE_CUDA(cudaMemcpyAsync(dB.get(), B, nn * 8, cudaMemcpyHostToDevice, s));
        be::dla::Sygv ws;
        be::dla::sygv_lowest(cx, ws, dA.get(), dB.get(), n, k, pivot_floor, dc.get(), dd.get(), st.get(), s);
        be::dla::Status hs{};
        BE_CUDA(cudaMemcpyAsync(&hs, st.get(), sizeof(hs), cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaMemcpyAsync(c, dc.get(), static_cast<std::size_t>(n) * k * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaMemcpyAsync(d, dd.get(), static_cast<std::size_t>(k) * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
        if (hs.not_pd) be::fail(BE_ERR_NOT_POSITIVE_DEFINITE, "cholesky: pivot below floor at index " + std::to_string(hs.not_pd - 1), hs.not_pd - 1);
    });
}

}  // extern "C"

// ------------------------------------------------------ dense, host buffers
// The densela.hpp / lobpcg.hpp panel functions on host buffers (the C++
// mirror's entry points for the reference's own unit suites): panels are
// uploaded, the solver's device kernels run, results come back. Widths that
// differ (p != q) run on zero-padded square panels.
namespace {

struct Staged {  // an n x m device panel holding a host n x w panel in its first w columns
    be::DBuf<double> d;
    int m = 0;
    void up(const double* h, int64_t n, int w, int m_, cudaStream_t s) {
        m = m_;
        d.reset(std::max<int64_t>(n * m, 1));
        if (w != m || !h) BE_CUDA(cudaMemsetAsync(d.get(), 0, d.bytes(), s));
        if (h && n > 0 && w > 0)
            BE_CUDA(cudaMemcpy2DAsync(d.get(), static_cast<std::size_t>(m) * 8, h, static_cast<std::size_t>(w) * 8,
                                      static_cast<std::size_t>(w) * 8, static_cast<std::size_t>(n),
                                      cudaMemcpyHostToDevice, s));
    }
    void down(double* h, int64_t n, int w, cudaStream_t s) const {
        if (n > 0 && w > 0)
            BE_CUDA(cudaMemcpy2DAsync(h, static_cast<std::size_t>(w) * 8, d.get(), static_cast<std::size_t>(m) * 8,
                                      static_cast<std::size_t>(w) * 8, static_cast<std::size_t>(n),
                                      cudaMemcpyDeviceToHost, s));
    }
};

// a small q x q column-major matrix zero-padded into the top-left of an m x m one
be::DBuf<double> small_up(const double* h, int r, int c, int m, cudaStream_t s) {
    std::vector<double> p(static_cast<std::size_t>(m) * m, 0.0);
    for (int j = 0; j < c; ++j)
        for (int i = 0; i < r; ++i) p[static_cast<std::size_t>(j) * m + i] = h[static_cast<std::size_t>(j) * r + i];
    be::DBuf<double> d(static_cast<int64_t>(m) * m);
    BE_CUDA(cudaMemcpyAsync(d.get(), p.data(), p.size() * 8, cudaMemcpyHostToDevice, s));
    BE_CUDA(cudaStreamSynchronize(s));  // p is a temporary
    return d;
}

be::dla::Status read_status(const be::DBuf<be::dla::Status>& st, cudaStream_t s) {
    be::dla::Status h{};
    BE_CUDA(cudaMemcpyAsync(&h, st.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    BE_CUDA(cudaStreamSynchronize(s));
    return h;
}

void gram_dev(be::Ctx* c, const double* a, const double* b, int m, int sym, int64_t n, double* out, cudaStream_t s) {
    const int64_t plen = be::dla::gram_partials_len(m, 1, c->num_sms);
    be::DBuf<double> part(plen);
    be::dla::GramJob j{};
    j.npairs = 1;
    j.nb = m;
    j.a[0] = a;
    j.b[0] = b;
    j.sym[0] = sym;
    j.out[0] = out;
    be::dla::gram(c, j, n, part.get(), plen, s);
    BE_CUDA(cudaStreamSynchronize(s));  // part is released on return
}

}  // namespace

extern "C" {

be_status be_dense_gram(be_ctx* ctx, const double* A, int p, const double* B, int q, int64_t n, int same,
                        double* out) {
    return guard([&] {
        if (!ctx || !out || (n > 0 && (!A || !B)) || p < 1 || q < 1 || n < 0) be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        if (p > 64 || q > 64) be::fail(BE_ERR_BAD_PARAMS, "gram: panel wider than 64 columns");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        const int m = std::max(p, q);
        Staged a, b;
        a.up(A, n, p, m, s);
        if (!same) b.up(B, n, q, m, s);
        be::DBuf<double> o(static_cast<int64_t>(m) * m);
        gram_dev(c, a.d.get(), same ? a.d.get() : b.d.get(), m, same ? 1 : 0, n, o.get(), s);
        std::vector<double> h(static_cast<std::size_t>(m) * m);
        BE_CUDA(cudaMemcpy(h.data(), o.get(), h.size() * 8, cudaMemcpyDeviceToHost));
        for (int j = 0; j < q; ++j)
            for (int i = 0; i < p; ++i) out[static_cast<std::size_t>(j) * p + i] = h[static_cast<std::size_t>(j) * m + i];
    });
}

be_status be_dense_cholesky(be_ctx* ctx, const double* B, int n, double rel_floor, double* R) {
    return guard([&] {
        if (!ctx || !B || !R || n < 1) be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        be::DBuf<double> dB = small_up(B, n, n, n, s), dR(static_cast<int64_t>(n) * n);
        be::DBuf<be::dla::Status> st(1);
        BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(be::dla::Status), s));
        be::dla::chol_floored(c, dB.get(), dR.get(), n, rel_floor, st.get(), s);
        BE_CUDA(cudaMemcpyAsync(R, dR.get(), static_cast<std::size_t>(n) * n * 8, cudaMemcpyDeviceToHost, s));
        const auto h = read_status(st, s);
        if (h.not_pd)
            be::fail(BE_ERR_NOT_POSITIVE_DEFINITE,
                     std::string(rel_floor > 0 ? "cholesky: pivot below floor at index " : "cholesky: non-positive pivot at index ") +
                         std::to_string(h.not_pd - 1),
                     h.not_pd - 1);
    });
}

be_status be_dense_trsm(be_ctx* ctx, double* W, int64_t n, int nb, const double* R) {
    return guard([&] {
        if (!ctx || !R || (n > 0 && !W) || nb < 1 || n < 0) be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        Staged w;
        w.up(W, n, nb, nb, s);
        be::DBuf<double> dR = small_up(R, nb, nb, nb, s);
        be::DBuf<be::dla::Status> st(1);
        BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(be::dla::Status), s));
        be::dla::trsm(c, w.d.get(), nullptr, dR.get(), nb, std::max<int64_t>(n, 0), st.get(), 0, 0, s);
        const auto h = read_status(st, s);
        if (h.singular_tri) be::fail(BE_ERR_SINGULAR_TRIANGULAR, "trsm_right_inv: triangular factor is numerically singular");
        w.down(W, n, nb, s);
        BE_CUDA(cudaStreamSynchronize(s));
    });
}

be_status be_dense_qr(be_ctx* ctx, double* X, int64_t n, int nb, double* R) {
    return guard([&] {
        if (!ctx || !R || (n > 0 && !X) || nb < 1) be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        if (nb > n) be::fail(BE_ERR_DIMENSION_MISMATCH, "qr_of_transpose: more columns than rows");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        Staged x;
        x.up(X, n, nb, nb, s);
        const int64_t nb2 = static_cast<int64_t>(nb) * nb;
        be::DBuf<double> Bq(nb2), Rq(2 * nb2);
        be::DBuf<be::dla::Status> st(1);
        BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(be::dla::Status), s));
        for (int pass = 0; pass < 2; ++pass) {  // densela.hpp:412-445 (rtot = R2 R1)
            gram_dev(c, x.d.get(), x.d.get(), nb, 1, n, Bq.get(), s);
            be::dla::qr_chol(c, Bq.get(), Rq.get() + pass * nb2, nb, st.get(), s);
            be::dla::trsm(c, x.d.get(), nullptr, Rq.get() + pass * nb2, nb, n, st.get(), 1, 0, s);
        }
        const auto h = read_status(st, s);
        if (h.rank_deficient) be::fail(BE_ERR_RANK_DEFICIENT, "qr_of_transpose: Gram matrix is numerically rank deficient");
        if (h.singular_tri) be::fail(BE_ERR_SINGULAR_TRIANGULAR, "trsm_right_inv: triangular factor is numerically singular");
        std::vector<double> r(static_cast<std::size_t>(2 * nb2));
        BE_CUDA(cudaMemcpy(r.data(), Rq.get(), r.size() * 8, cudaMemcpyDeviceToHost));
        x.down(X, n, nb, s);
        BE_CUDA(cudaStreamSynchronize(s));
        // rtot = matmul(R2, R1) (both upper triangular, nb x nb): the small product on the host
        const double* r1 = r.data();
        const double* r2 = r.data() + nb2;
        for (int j = 0; j < nb; ++j)
            for (int i = 0; i < nb; ++i) {
                double acc = 0.0;
                for (int k = 0; k < nb; ++k) {
                    const double b = r1[static_cast<std::size_t>(j) * nb + k];
                    if (b == 0.0) continue;
                    acc += r2[static_cast<std::size_t>(k) * nb + i] * b;
                }
                R[static_cast<std::size_t>(j) * nb + i] = acc;
            }
    });
}

be_status be_dense_mix(be_ctx* ctx, const double* X, int64_t n, int p, const double* C, int q, double* Y,
                       int accumulate) {
    return guard([&] {
        if (!ctx || !C || (n > 0 && (!X || !Y)) || p < 1 || q < 1 || n < 0) be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        if (p > 64 || q > 64) be::fail(BE_ERR_BAD_PARAMS, "block_times_small: panel wider than 64 columns");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        const int m = std::max(p, q);
        Staged x, y;
        x.up(X, n, p, m, s);
        y.up(accumulate ? Y : nullptr, n, q, m, s);
        be::DBuf<double> dC = small_up(C, p, q, m, s);
        be::dla::MixJob job{};
        job.nb = m;
        job.nout = 1;
        job.out[0] = be::dla::MixOut{y.d.get(), accumulate ? 1 : 0, 1, {{x.d.get(), dC.get(), 0, 0}}, -1};
        if (n > 0) be::dla::mix(c, job, n, s);
        y.down(Y, n, q, s);
        BE_CUDA(cudaStreamSynchronize(s));
    });
}

be_status be_dense_residual(be_ctx* ctx, const double* HX, const double* X, const double* theta, int64_t n, int nb,
                            double* R, double* rnorm2, double* xnorm2) {
    return guard([&] {
        if (!ctx || !theta || (n > 0 && (!HX || !X || !R)) || nb < 1 || nb > 64 || n < 0)
            be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        Staged hx, x, r;
        hx.up(HX, n, nb, nb, s);
        x.up(X, n, nb, nb, s);
        r.up(nullptr, n, nb, nb, s);
        be::DBuf<double> th(nb), norms(2 * nb), part(static_cast<int64_t>(c->num_sms) * 64 * 2 * nb);
        BE_CUDA(cudaMemcpyAsync(th.get(), theta, static_cast<std::size_t>(nb) * 8, cudaMemcpyHostToDevice, s));
        BE_CUDA(cudaMemsetAsync(norms.get(), 0, norms.bytes(), s));
        if (n > 0) be::dla::residual(c, hx.d.get(), x.d.get(), th.get(), r.d.get(), nb, n, part.get(), norms.get(), norms.get() + nb, s);
        r.down(R, n, nb, s);
        std::vector<double> h(static_cast<std::size_t>(2 * nb));
        BE_CUDA(cudaMemcpyAsync(h.data(), norms.get(), h.size() * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
        if (rnorm2) std::memcpy(rnorm2, h.data(), static_cast<std::size_t>(nb) * 8);
        if (xnorm2) std::memcpy(xnorm2, h.data() + nb, static_cast<std::size_t>(nb) * 8);
    });
}

be_status be_dense_colnorm2(be_ctx* ctx, const double* A, int64_t n, int nb, double* out) {
    return guard([&] {
        if (!ctx || !out || (n > 0 && !A) || nb < 1 || nb > 64 || n < 0) be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        auto* c = ctx->impl.get();
        cudaStream_t s = c->stream;
        Staged a;
        a.up(A, n, nb, nb, s);
        be::DBuf<double> o(nb), part(static_cast<int64_t>(c->num_sms) * 64 * 2 * nb);
        BE_CUDA(cudaMemsetAsync(o.get(), 0, o.bytes(), s));
        if (n > 0) be::dla::colnorm2(c, a.d.get(), nb, n, part.get(), o.get(), s);
        BE_CUDA(cudaMemcpyAsync(out, o.get(), static_cast<std::size_t>(nb) * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaStreamSynchronize(s));
    });
}

be_status be_rayleigh_ritz(be_ctx* ctx, const double* X, const double* W, const double* P, const double* HX,
                           const double* HW, const double* HP, int64_t n, int nb, int k_keep, double* c,
                           double* theta) {
    return guard([&] {
        if (!ctx || !c || !theta || (n > 0 && (!X || !W || !HX || !HW)) || nb < 1 || nb > 64 || n < 0)
            be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        if ((P == nullptr) != (HP == nullptr))
            be::fail(BE_ERR_DIMENSION_MISMATCH, "rayleigh_ritz: P and HP must be given together");
        const bool with_p = P != nullptr;
        const int nblk = with_p ? 3 : 2, dim = nblk * nb;
        if (k_keep < 1 || k_keep > dim) be::fail(BE_ERR_BAD_PARAMS, "sygv_lowest: k out of range");
        auto* cx = ctx->impl.get();
        cudaStream_t s = cx->stream;
        Staged x, w, p, hx, hw, hp;
        x.up(X, n, nb, nb, s);
        w.up(W, n, nb, nb, s);
        hx.up(HX, n, nb, nb, s);
        hw.up(HW, n, nb, nb, s);
        if (with_p) {
            p.up(P, n, nb, nb, s);
            hp.up(HP, n, nb, nb, s);
        }
        // the 6 (3) lower G blocks then the 6 (3) lower O blocks (lobpcg.hpp:126-141)
        const double* pairs[12][2];
        int sym[12], np = 0;
        auto add = [&](const double* a, const double* b, int sy) {
            pairs[np][0] = a;
            pairs[np][1] = b;
            sym[np++] = sy;
        };
        add(x.d.get(), hx.d.get(), 0);
        add(w.d.get(), hx.d.get(), 0);
        add(w.d.get(), hw.d.get(), 0);
        if (with_p) {
            add(p.d.get(), hx.d.get(), 0);
            add(p.d.get(), hw.d.get(), 0);
            add(p.d.get(), hp.d.get(), 0);
        }
        add(x.d.get(), x.d.get(), 1);
        add(w.d.get(), x.d.get(), 0);
        add(w.d.get(), w.d.get(), 1);
        if (with_p) {
            add(p.d.get(), x.d.get(), 0);
            add(p.d.get(), w.d.get(), 0);
            add(p.d.get(), p.d.get(), 1);
        }
        const int64_t nb2 = static_cast<int64_t>(nb) * nb;
        be::DBuf<double> blocks(12 * nb2), G(static_cast<int64_t>(dim) * dim), O(static_cast<int64_t>(dim) * dim),
            dc(static_cast<int64_t>(dim) * k_keep), dd(k_keep);
        be::dla::GramJob j{};
        j.npairs = np;
        j.nb = nb;
        for (int q = 0; q < np; ++q) {
            j.a[q] = pairs[q][0];
            j.b[q] = pairs[q][1];
            j.sym[q] = sym[q];
            j.out[q] = blocks.get() + q * nb2;
        }
        const int64_t plen = be::dla::gram_partials_len(nb, np, cx->num_sms);
        be::DBuf<double> part(plen);
        be::dla::gram(cx, j, n, part.get(), plen, s);
        be::dla::rr_assemble(cx, blocks.get(), nb, nblk, G.get(), O.get(), s);
        be::DBuf<be::dla::Status> st(1);
        BE_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(be::dla::Status), s));
        be::dla::Sygv ws;
        be::dla::sygv_lowest(cx, ws, G.get(), O.get(), dim, k_keep, 1e-10, dc.get(), dd.get(), st.get(), s);
        BE_CUDA(cudaMemcpyAsync(c, dc.get(), static_cast<std::size_t>(dim) * k_keep * 8, cudaMemcpyDeviceToHost, s));
        BE_CUDA(cudaMemcpyAsync(theta, dd.get(), static_cast<std::size_t>(k_keep) * 8, cudaMemcpyDeviceToHost, s));
        const auto h = read_status(st, s);
        if (h.not_pd)
            be::fail(BE_ERR_BASIS_DEGENERATE, "rayleigh_ritz: overlap matrix failed Cholesky (cholesky: pivot below floor at index " +
                                                  std::to_string(h.not_pd - 1) + ")");
    });
}

be_status be_update_blocks(be_ctx* ctx, const double* X, const double* W, const double* P, const double* HX,
                           const double* HW, const double* HP, int64_t n, int nb, int m, const double* C1,
                           const double* C2, const double* C3, double* Xo, double* HXo, double* Po, double* HPo) {
    return guard([&] {
        if (!ctx || !C1 || !C2 || (n > 0 && (!X || !W || !HX || !HW || !Xo || !HXo || !Po || !HPo)) || nb < 1 ||
            m < 1 || nb > 64 || m > 64 || n < 0)
            be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        if ((P == nullptr) != (HP == nullptr) || (P && !C3))
            be::fail(BE_ERR_DIMENSION_MISMATCH, "update_blocks: P, HP and C3 must be given together");
        auto* cx = ctx->impl.get();
        cudaStream_t s = cx->stream;
        const bool with_p = P != nullptr;
        const int w2 = std::max(nb, m);  // square working width
        Staged x, w, p, hx, hw, hp, xo, hxo, po, hpo;
        x.up(X, n, nb, w2, s);
        w.up(W, n, nb, w2, s);
        hx.up(HX, n, nb, w2, s);
        hw.up(HW, n, nb, w2, s);
        if (with_p) {
            p.up(P, n, nb, w2, s);
            hp.up(HP, n, nb, w2, s);
        }
        for (auto* o : {&xo, &hxo, &po, &hpo}) o->up(nullptr, n, m, w2, s);
        be::DBuf<double> c1 = small_up(C1, nb, m, w2, s), c2 = small_up(C2, nb, m, w2, s);
        be::DBuf<double> c3;
        if (with_p) c3 = small_up(C3, nb, m, w2, s);
        // lobpcg.hpp:168-194: P+ = W C2 + P C3, HP+ likewise; X+ = X C1 + P+, HX+ = HX C1 + HP+
        be::dla::MixJob job{};
        job.nb = w2;
        job.nout = 4;
        job.out[0] = be::dla::MixOut{po.d.get(), 0, with_p ? 2 : 1, {{w.d.get(), c2.get(), 0, 0}, {p.d.get(), c3.get(), 0, 0}}, -1};
        job.out[1] = be::dla::MixOut{hpo.d.get(), 0, with_p ? 2 : 1, {{hw.d.get(), c2.get(), 0, 0}, {hp.d.get(), c3.get(), 0, 0}}, -1};
        job.out[2] = be::dla::MixOut{xo.d.get(), 0, 1, {{x.d.get(), c1.get(), 0, 0}}, 0};
        job.out[3] = be::dla::MixOut{hxo.d.get(), 0, 1, {{hx.d.get(), c1.get(), 0, 0}}, 1};
        if (n > 0) be::dla::mix(cx, job, n, s);
        xo.down(Xo, n, m, s);
        hxo.down(HXo, n, m, s);
        po.down(Po, n, m, s);
        hpo.down(HPo, n, m, s);
        BE_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

extern "C" {

be_status be_dist_touched(const be_csb_view* L, const int64_t* cuts, const int* owner, int world, uint8_t* touched) {
    return guard([&] {
        if (!L || !cuts || !touched || world < 1) be::fail(BE_ERR_BAD_PARAMS, "bad argument");
        be::validate_view(*L);
        auto slot = [&](int64_t row) {
            const int q = static_cast<int>(std::upper_bound(cuts, cuts + world + 1, row) - cuts) - 1;
            if (q < 0 || q >= world) be::fail(BE_ERR_BAD_PARAMS, "be_dist_touched: row outside the cuts");
            return owner ? owner[q] : q;
        };
        std::fill(touched, touched + world, 0);
        for (int64_t bi = 0; bi < L->nrowblks; ++bi)
            for (int64_t bj = 0; bj < L->ncolblks; ++bj)
                if (L->block_nnz[bi * L->ncolblks + bj] > 0) {
                    touched[slot(L->row_offsets[bi])] = 1;
                    touched[slot(L->col_offsets[bj])] = 1;
                }
    });
}

be_status be_op_dist_need(const be_op* op, uint8_t* need) {
    return guard([&] {
        if (!op || !need) be::fail(BE_ERR_BAD_PARAMS, "null argument");
        const auto* o = op->impl.get();
        if (!o->comm) be::fail(BE_ERR_BAD_PARAMS, "be_op_dist_need: not a distributed operator");
        for (std::size_t i = 0; i < o->need.size(); ++i) need[i] = static_cast<uint8_t>(o->need[i]);
    });
}

}  // extern "C"
