// TriangularLayout (dist.hpp:25-47) and partition_matrix's routing, restated.
#pragma once

#include <array>
#include <utility>
#include <vector>

#include "common.hpp"

namespace be {

struct TriLayout {
    int nd = 0, n_ranks = 0;
    std::vector<std::array<int, 3>> blocks;  // per rank: stored (i, j, transposed)
    std::vector<std::vector<int>> row_groups, col_groups;
    std::vector<int> diagonal_ranks;
};

TriLayout build_tri_layout(int nd);
std::vector<std::pair<index_t, index_t>> tri_segments(const TriLayout& lt, const index_t* sub_bounds);
std::vector<be_triple> tri_rank_triples(const be_csb_view& L, const TriLayout& lt, const index_t* sub_bounds, int rank);

}  // namespace be
