// Device-side objects behind the opaque C handles: context, operator (tile
// format of the half-stored matrix), preconditioner tiles.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host_csb.hpp"

struct cusolverDnContext;
struct cublasContext;

namespace be {

struct Comm;

// RAII device buffer
template <class T>
struct DBuf {
    T* p = nullptr;
    index_t n = 0;
    DBuf() = default;
    explicit DBuf(index_t count) { reset(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void reset(index_t count) {
        release();
        n = count;
        if (count > 0) BE_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), static_cast<std::size_t>(count) * sizeof(T)));
    }
    T* get() const { return p; }
    std::size_t bytes() const { return static_cast<std::size_t>(n) * sizeof(T); }
};

// Device panels kept for reuse; shared by a context and the results it
// produced (a result returns its eigenvector block here when freed).
struct PanelPool {
    std::mutex mu;
    std::vector<DBuf<double>> bufs;
    DBuf<double> take(index_t need) {
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = bufs.begin(); it != bufs.end(); ++it)
            if (it->n >= need) {
                DBuf<double> b = std::move(*it);
                bufs.erase(it);
                return b;
            }
        // nothing fits: the smaller pooled panels are dropped
        bufs.erase(std::remove_if(bufs.begin(), bufs.end(), [&](const DBuf<double>& d) { return d.n < need; }),
                   bufs.end());
        return DBuf<double>(need);
    }
    void give(DBuf<double>&& b) {
        if (!b.p) return;
        std::lock_guard<std::mutex> lk(mu);
        bufs.push_back(std::move(b));
    }
};

struct Ctx {
    int device = 0;
    int num_sms = 0;
    int nsmid = 0;  // %nsmid (upper bound of %smid; may exceed num_sms), queried on first use
    cudaStream_t stream = nullptr;
    cusolverDnContext* solver = nullptr;
    cublasContext* blas = nullptr;  // triangular solves of the 3nb x 3nb pencil
    long long launches = 0;  // kernels launched through this context
    // n x nb panels of finished solves (and of freed results), reused by the
    // next solve on this context: no cudaMalloc / cudaFree per call
    std::shared_ptr<PanelPool> panels = std::make_shared<PanelPool>();
    // the small device / pinned buffers of the last finished solve (lobpcg.cu)
    std::shared_ptr<void> solver_keep;
    ~Ctx();
};

// One device work tile: <= kTile rows x <= kTile cols of the lower triangle,
// <= max_nnz entries; its data is one 16-byte aligned blob (spmm.cu). 16 bytes.
struct TileHdr {
    std::uint32_t begin16;  // blob byte offset / 16
    std::int32_t row0;     // first global row of the 128-row tile-row
    std::int32_t col0;     // first global column
    std::uint32_t packed;  // (nr-1) | (nc-1) << 7 | nnz << 14; nr = rows of the tile-row
};

inline constexpr int kTile = 128;
// tile blob metadata (spmm.cu): jr u16[136] | jc u16[136] | rank->row u8[128] | rank->col u8[128] |
// row lengths u8[128] | column lengths u8[128] | work split u16[9] (+ padding) = 1088 bytes
inline constexpr int kBlobMeta = 1088;

// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the
// current device. Monotonic (never lowered), so ranks running as threads of
// one process cannot race one another below a size a launch needs.
void ensure_dyn_smem_raw(const void* kern, std::size_t bytes);
template <class K>
void ensure_dyn_smem(K* kern, std::size_t bytes) {
    ensure_dyn_smem_raw(reinterpret_cast<const void*>(kern), bytes);
}

struct Op {
    Ctx* ctx = nullptr;
    index_t nrows = 0, ncols = 0, nnz = 0, ntiles = 0, padded = 0;
    bool symmetric = false;
    int values_prec = BE_F32;
    int max_nnz = 2048;
    DBuf<TileHdr> tiles;
    DBuf<int2> runs;                 // [tile_begin, tile_end) work items
    index_t nruns = 0;
    DBuf<unsigned char> blobs;       // per tile: JDS meta + row-order and column-order entry streams
    index_t blob_total = 0;          // bytes of all blobs
    int blob_max = 0;                // bytes of the largest possible blob (one stage buffer)
    DBuf<double> diag;               // nrows (symmetric only)
    DBuf<int> counter;               // persistent-kernel tile counter [2]
    DBuf<float> x32, y32;            // f32 staging of f64 panels (f32-values operator)
    std::vector<std::int64_t> csb_index;  // row-order device slot -> CSB index, -1 = padding (small matrices only)
    // deterministic mode (BE_OP_DETERMINISTIC): row lists in the reference's serial summation
    // order instead of the tile format -- L's entries of each output row (det_ptr_n, nrows + 1)
    // and L^T's (det_ptr_t, ncols + 1) over one (column, f64 value) array
    bool det = false;
    DBuf<std::int64_t> det_ptr_n, det_ptr_t;
    DBuf<std::int32_t> det_col;
    DBuf<double> det_val;
    // row-list format for sparse matrices (k_rows_spmm): the same L / L^T row lists with f32 values
    bool rows = false;
    DBuf<float> rows_val;
    int grid = 0;
    // multi-GPU (row e): panel rows are owned in contiguous segments
    // [cuts[q], cuts[q+1]); tile coordinates live in the padded index space
    // q * lmax + (row - cuts[q]) so the f32 X / Y exchange buffers are
    // equal-count NCCL allgather / reduce-scatter operands. `runs` then holds
    // the interior work items (rows and columns both in this rank's segment,
    // computable before the allgather lands) and runs_ext the rest.
    Comm* comm = nullptr;
    int rank = 0, world = 1;
    index_t lmax = 0, row_lo = 0, nlocal = 0;
    std::vector<index_t> cuts;
    DBuf<int2> runs_ext;
    index_t nruns_ext = 0;
    // runs_ext grouped by column segment (segment order): group q = [ext_group[q], ext_group[q+1]).
    // In a lower triangle every tile writing segment q (as column or as row) sits in a group <= q,
    // so segment q's partial Y is final once groups 0..q ran (the overlapped Y exchange).
    std::vector<index_t> ext_group;
    std::vector<cudaEvent_t> ev_grp;
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_x = nullptr, ev_ag = nullptr;
    // segment-wise exchange: need[p * world + r] = rank p's tiles touch the padded slot of rank
    // r (rows or columns); X slots travel only to the ranks that touch them and partial Y
    // slots only to their owners
    std::vector<char> touched, need;
    DBuf<float> ystage;
    std::vector<int> owner, seg_of_rank;  // segment -> rank, rank -> segment
    index_t unpad(index_t p) const {  // padded index -> global row
        const index_t r = p / lmax;
        return cuts[static_cast<std::size_t>(seg_of_rank[static_cast<std::size_t>(r)])] + (p - r * lmax);
    }
    // timing
    bool timing = false;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    double last_kernel_ms = 0, last_apply_ms = 0;
    ~Op();
};

std::unique_ptr<Op> op_create(Ctx* ctx, const be_csb_view& L, const double* diag, int values_prec, int flags);
// the symmetric tile-format operator streamed from a CSB1 file (its diagonal section required)
std::unique_ptr<Op> op_create_csb1(Ctx* ctx, const std::string& path, int values_prec, int flags,
                                   std::vector<double>* diag_out, index_t batch_entries);
// Distributed operator (row e): L holds this rank's slab of the global
// strictly-lower matrix (global coordinates), cuts (world + 1 entries, on L's
// block boundaries) the panel-row ownership, diag_local the diagonal of this
// rank's rows. apply() then maps local f64 panels to local f64 panels.
std::unique_ptr<Op> op_create_dist(Ctx* ctx, Comm* comm, const be_csb_view& L, const index_t* cuts,
                                   const int* owner, const double* diag_local, int values_prec);
// equal-rows ownership on block boundaries / contiguous weight balance
std::vector<index_t> dist_rows(const index_t* bounds, index_t nbounds, int world);
std::vector<index_t> dist_balance(const index_t* weights, index_t nitems, int world);
std::vector<index_t> dist_tiles2d(const index_t* w, index_t nblk, const index_t* bounds, int world);
void op_apply(Op* op, const void* X, void* Y, index_t nrows, int nb, int panel_prec, int mode, cudaStream_t s);

}  // namespace be

struct be_ctx {
    std::unique_ptr<be::Ctx> impl;
};
struct be_op {
    std::unique_ptr<be::Op> impl;
};
