// The reference's own multi-rank layout (dist.hpp:25-198), restated for the
// parity variant of the multi-GPU path: nd sub-matrices, the stored block set
// {(i, j) : (i - j) mod nd <= (nd - 1) / 2} over nd(nd+1)/2 ranks numbered
// column-major, upper-wedge blocks held transposed, and every sub-vector
// split near-evenly over its column group (dist.hpp:184-196). The device
// operator then runs the same exchange as the nnz-balanced partition, with
// segment ownership following this layout instead of rank order.
#include <algorithm>

#include "host_csb.hpp"
#include "tri_layout.hpp"

namespace be {

// build_layout (dist.hpp:49-75)
TriLayout build_tri_layout(int nd) {
    if (nd < 1 || nd % 2 == 0) fail(BE_ERR_EVEN_ND, "build_layout: n_d must be odd and positive");
    TriLayout lt;
    lt.nd = nd;
    lt.n_ranks = nd * (nd + 1) / 2;
    lt.row_groups.assign(static_cast<std::size_t>(nd), {});
    lt.col_groups.assign(static_cast<std::size_t>(nd), {});
    lt.diagonal_ranks.assign(static_cast<std::size_t>(nd), -1);
    const int half = (nd - 1) / 2;
    for (int j = 0; j < nd; ++j)
        for (int i = 0; i < nd; ++i) {
            if ((((i - j) % nd) + nd) % nd > half) continue;
            const int rank = static_cast<int>(lt.blocks.size());
            lt.blocks.push_back({i, j, i < j ? 1 : 0});
            lt.row_groups[static_cast<std::size_t>(i)].push_back(rank);
            lt.col_groups[static_cast<std::size_t>(j)].push_back(rank);
            if (i == j) lt.diagonal_ranks[static_cast<std::size_t>(i)] = rank;
        }
    return lt;
}

// segment table (dist.hpp:184-196): sub-vector g split over its column group
std::vector<std::pair<index_t, index_t>> tri_segments(const TriLayout& lt, const index_t* sub_bounds) {
    std::vector<std::pair<index_t, index_t>> seg(static_cast<std::size_t>(lt.n_ranks));
    const int gsize = (lt.nd + 1) / 2;
    for (int g = 0; g < lt.nd; ++g) {
        const index_t lo = sub_bounds[g], len = sub_bounds[g + 1] - sub_bounds[g];
        for (int m = 0; m < gsize; ++m) {
            const int r = lt.col_groups[static_cast<std::size_t>(g)][static_cast<std::size_t>(m)];
            seg[static_cast<std::size_t>(r)] = {lo + len * m / gsize, lo + len * (m + 1) / gsize};
        }
    }
    return seg;
}

// The stored entries of `rank` (global coordinates, strictly lower), in the
// to_triples order of L: the sub-block (i, j) for a lower stored block, the
// lower sub-block (j, i) for a transposed-stored wedge block
// (partition_matrix's routing, dist.hpp:142-163).
std::vector<be_triple> tri_rank_triples(const be_csb_view& L, const TriLayout& lt, const index_t* sub_bounds,
                                        int rank) {
    if (rank < 0 || rank >= lt.n_ranks) fail(BE_ERR_BAD_PARAMS, "partition: rank out of range");
    if (sub_bounds[0] != 0 || sub_bounds[lt.nd] != L.nrows || L.nrows != L.ncols)
        fail(BE_ERR_BAD_PARAMS, "partition_matrix: boundaries must cover the matrix");
    for (int g = 0; g < lt.nd; ++g)
        if (sub_bounds[g + 1] <= sub_bounds[g]) fail(BE_ERR_BAD_PARAMS, "partition_matrix: boundaries must be strictly increasing");
    const auto& b = lt.blocks[static_cast<std::size_t>(rank)];
    const int bi = b[2] ? b[1] : b[0], bj = b[2] ? b[0] : b[1];  // the lower sub-block it holds
    const index_t r0 = sub_bounds[bi], r1 = sub_bounds[bi + 1], c0 = sub_bounds[bj], c1 = sub_bounds[bj + 1];
    std::vector<be_triple> all(static_cast<std::size_t>(L.nnz));
    to_triples(L, all.data());
    std::vector<be_triple> out;
    for (const auto& t : all)
        if (t.row >= r0 && t.row < r1 && t.col >= c0 && t.col < c1) out.push_back(t);
    return out;
}

}  // namespace be
