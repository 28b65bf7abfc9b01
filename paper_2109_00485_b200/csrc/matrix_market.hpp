// Matrix Market ingest / export (matrix_market.hpp:20-114 of the reference).
#pragma once

#include <string>
#include <vector>

#include "common.hpp"

namespace be {

struct MmMatrix {  // SymmetricCoo (matrix_market.hpp:20-24)
    index_t n = 0;
    std::vector<be_triple> lower;
    std::vector<double> diag;
};

MmMatrix parse_matrix_market(const char* text, std::size_t len);
MmMatrix read_matrix_market_file(const std::string& path);
std::string write_matrix_market(index_t n, const be_triple* lower, index_t nlower, const double* diag);

}  // namespace be
