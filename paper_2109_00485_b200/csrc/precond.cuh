// Block-diagonal FOM preconditioner objects (precond.hpp).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "device.hpp"

namespace be {

// SparseTile (precond.hpp:18-30), host copy in the reference layout
struct HostTile {
    index_t dim = 0;
    std::vector<std::int32_t> rows, cols;
    std::vector<double> vals;
    std::vector<index_t> diag_pos;
};

struct Tiles {
    Ctx* ctx = nullptr;
    index_t n = 0, ntiles = 0, nentries = 0, max_dim = 0;
    std::vector<index_t> offsets;
    std::vector<HostTile> host;
    DBuf<unsigned char> tiles;  // TileDev records
    // size classes for the warp-per-(tile, column) kernel: tiles with
    // dim <= class_dim[c] (and > the previous class) listed in class_tiles
    std::vector<int> class_dim;
    std::vector<index_t> class_begin;  // into class_tiles, size = classes + 1
    std::vector<index_t> class_max_ent;  // largest tile (stored entries) per class
    DBuf<std::int32_t> class_tiles;
    index_t big_tiles = 0;             // tiles above the last class (CTA kernel)
    DBuf<std::int32_t> rowptr;
    DBuf<std::uint16_t> cols;
    DBuf<double> vals;
    // per size class: older Krylov vectors of the block kernel (L2-resident
    // scratch slots) and the per-SM mask of the slots resident CTAs hold
    DBuf<double> vscratch[8];
    DBuf<unsigned> slot_mask[8];
    // the size classes run concurrently: side streams joined back by events
    cudaStream_t side[8] = {};
    cudaEvent_t fork = nullptr, join[8] = {};
    ~Tiles() {
        for (auto& x : side)
            if (x) cudaStreamDestroy(x);
        for (auto& x : join)
            if (x) cudaEventDestroy(x);
        if (fork) cudaEventDestroy(fork);
    }
};

// extract_tiles + upload; [row_lo, row_hi) restricts the result to the tiles
// of one rank's rows (multi-GPU; diag then holds those rows only). row_lo < 0:
// the whole matrix.
std::unique_ptr<Tiles> tiles_create(Ctx* ctx, const be_csb_view& L, const double* diag, const index_t* off,
                                    index_t noff, index_t row_lo = -1, index_t row_hi = -1);
// Tiles given explicitly in the reference's SparseTile layout (consecutive row
// ranges in the order given): the fom_solve_tile entry point of the mirror.
std::unique_ptr<Tiles> tiles_create_explicit(Ctx* ctx, const std::vector<HostTile>& tiles);
void precond_apply(Tiles* t, const double* shifts, const double* R, double* W, index_t nrows, int nb, int m,
                   std::int64_t* fallbacks, cudaStream_t s);

}  // namespace be

struct be_tiles {
    std::unique_ptr<be::Tiles> impl;
};
