// Host-side storage types (CsbCooMatrix mirror, generator outputs).
#pragma once

#include <cstdlib>
#include <istream>
#include <ostream>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "common.hpp"

namespace be {

inline constexpr index_t kMaxBlockExtent = 32000;  // csb.hpp:28

// Uninitialised owning buffer: T1-scale arrays (1e9 entries) are filled in
// parallel, so the zero-fill of std::vector would only cost time.
template <class T>
struct Buf {
    T* p = nullptr;
    index_t n = 0;
    Buf() = default;
    explicit Buf(index_t count) { reset(count); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    ~Buf() { std::free(p); }
    void reset(index_t count) {
        std::free(p);
        p = nullptr;
        n = count;
        if (count > 0) {
            p = static_cast<T*>(std::malloc(static_cast<std::size_t>(count) * sizeof(T)));
            if (!p) fail(BE_ERR_OUT_OF_MEMORY, "host allocation failed");
        }
    }
    T* data() { return p; }
    const T* data() const { return p; }
    T& operator[](index_t i) { return p[i]; }
    const T& operator[](index_t i) const { return p[i]; }
};

// CsbCooMatrix (csb.hpp:39-63)
struct CsbHost {
    index_t nrows = 0, ncols = 0, nrowblks = 0, ncolblks = 0, nnz = 0;
    std::vector<index_t> row_offsets, col_offsets, block_nnz, block_nnz_offsets;
    Buf<std::uint16_t> local_rows, local_cols;
    Buf<double> values;
    void allocate(index_t nnz_);
    be_csb_view view() const;
};

struct Synth {
    index_t n = 0;
    std::vector<be_triple> lower;
    std::vector<double> diag;
    std::vector<index_t> tile_offsets;
};

std::vector<index_t> uniform_boundaries(index_t n, index_t extent);
std::unique_ptr<CsbHost> build_csb(const be_triple* t, index_t count, index_t nrows, index_t ncols,
                                   const index_t* rb, index_t nrb, const index_t* cb, index_t ncb);
void validate_view(const be_csb_view& v);
bool is_strictly_lower(const be_csb_view& v);
void to_triples(const be_csb_view& v, be_triple* out);
void save_csb1(const std::string& path, const be_csb_view& v, const double* diag, index_t ndiag);
std::unique_ptr<CsbHost> load_csb1(const std::string& path, std::vector<double>* diag);
void save_csb1(std::ostream& os, const be_csb_view& v, const double* diag, index_t ndiag);
std::unique_ptr<CsbHost> load_csb1(std::istream& is, std::vector<double>* diag);
std::unique_ptr<CsbHost> load_csb1_rows(const std::string& path, index_t b0, index_t b1, std::vector<double>* diag);
std::vector<index_t> csb1_block_row_nnz(const std::string& path, index_t& nrows, index_t& nrowblks);
std::vector<index_t> draw_tile_offsets(index_t n, index_t block_extent, index_t tile_min, index_t tile_max,
                                       std::mt19937_64& rng);
std::unique_ptr<Synth> generate_synthetic(const be_synth_params& p);
std::unique_ptr<CsbHost> generate_clustered(const be_cluster_params& p, std::vector<double>& diag,
                                            std::vector<index_t>& tile_offsets);
// block rows [b0, b1) only (diag_only: their diagonal blocks only); rowabs
// (n) receives this part's contribution to sum |row| of every row
// [c0, c1): block columns kept (default: all; a 2-D tile of the lower triangle)
std::unique_ptr<CsbHost> generate_clustered_part(const be_cluster_params& p, index_t b0, index_t b1, bool diag_only,
                                                 std::vector<double>& rowabs, std::vector<index_t>& tile_offsets,
                                                 index_t c0 = 0, index_t c1 = -1);
double clustered_diag_value(const be_cluster_params& p, index_t i, double rowabs);
std::vector<index_t> clustered_block_row_weights(const be_cluster_params& p);
std::vector<index_t> clustered_block_weights(const be_cluster_params& p, index_t& nblk);

}  // namespace be
