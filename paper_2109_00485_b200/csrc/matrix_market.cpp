// Matrix Market ingest and export (matrix_market.hpp:38-114), restated:
// coordinate-format real (or integer) symmetric files; entries given in
// either triangle become strictly-lower triples, diagonal entries a dense
// array (zero where absent). Errors follow the reference: a malformed file is
// ParseError, a non-symmetric header NotSymmetricHeader, a repeated diagonal
// entry DuplicateEntry.
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "matrix_market.hpp"

namespace be {
namespace {

std::string folded(const std::string& s) {
    std::string r(s);
    for (auto& c : r) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return r;
}

// whitespace-separated tokens of [p, end)
struct Tokens {
    const char* p;
    const char* end;
    bool next(std::string& tok) {
        while (p < end && std::isspace(static_cast<unsigned char>(*p))) ++p;
        if (p >= end) return false;
        const char* b = p;
        while (p < end && !std::isspace(static_cast<unsigned char>(*p))) ++p;
        tok.assign(b, p);
        return true;
    }
};

bool to_index(const std::string& t, index_t& v) {
    if (t.empty()) return false;
    errno = 0;
    char* e = nullptr;
    const long long x = std::strtoll(t.c_str(), &e, 10);
    if (errno || e != t.c_str() + t.size()) return false;
    v = static_cast<index_t>(x);
    return true;
}

bool to_value(const std::string& t, double& v) {
    if (t.empty()) return false;
    char* e = nullptr;
    v = std::strtod(t.c_str(), &e);
    return e == t.c_str() + t.size();
}

}  // namespace

MmMatrix parse_matrix_market(const char* text, std::size_t len) {
    const char* p = text;
    const char* end = text + len;
    auto getline = [&](std::string& line) {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<std::size_t>(end - p)));
        const char* le = nl ? nl : end;
        line.assign(p, le);
        if (!line.empty() && line.back() == '\r') line.pop_back();
        p = nl ? nl + 1 : end;
        return true;
    };
    std::string line;
    if (!getline(line)) fail(BE_ERR_PARSE, "matrix market: empty input");
    {
        std::istringstream banner(line);
        std::string tag, object, format, field, symmetry;
        banner >> tag >> object >> format >> field >> symmetry;
        if (folded(tag) != "%%matrixmarket" || folded(object) != "matrix")
            fail(BE_ERR_PARSE, "matrix market: bad banner line");
        if (folded(format) != "coordinate") fail(BE_ERR_PARSE, "matrix market: only coordinate format is supported");
        const std::string f = folded(field);
        if (f != "real" && f != "integer")
            fail(BE_ERR_PARSE, "matrix market: only real or integer fields are supported");
        if (folded(symmetry) != "symmetric")
            fail(BE_ERR_NOT_SYMMETRIC_HEADER, "matrix market: header must declare a symmetric matrix");
    }
    // comment (and blank) lines up to the size line
    bool have = false;
    while (getline(line))
        if (!line.empty() && line[0] != '%') {
            have = true;
            break;
        }
    index_t nrows = 0, ncols = 0, count = 0;
    {
        Tokens t{line.data(), line.data() + (have ? line.size() : 0)};
        std::string a, b, c;
        if (!(t.next(a) && t.next(b) && t.next(c) && to_index(a, nrows) && to_index(b, ncols) && to_index(c, count)))
            fail(BE_ERR_PARSE, "matrix market: bad size line");
    }
    if (nrows != ncols) fail(BE_ERR_PARSE, "matrix market: symmetric matrix must be square");
    if (nrows <= 0) fail(BE_ERR_PARSE, "matrix market: empty matrix");
    MmMatrix m;
    m.n = nrows;
    m.diag.assign(static_cast<std::size_t>(nrows), 0.0);
    std::vector<unsigned char> seen(static_cast<std::size_t>(nrows), 0);
    if (count > 0) m.lower.reserve(static_cast<std::size_t>(count));
    Tokens t{p, end};
    std::string ti, tj, tv;
    for (index_t e = 0; e < count; ++e) {
        index_t i = 0, j = 0;
        double v = 0.0;
        if (!(t.next(ti) && t.next(tj) && t.next(tv) && to_index(ti, i) && to_index(tj, j) && to_value(tv, v)))
            fail(BE_ERR_PARSE, "matrix market: truncated entry list");
        if (i < 1 || i > nrows || j < 1 || j > ncols) fail(BE_ERR_PARSE, "matrix market: entry index out of range");
        --i;
        --j;
        if (i == j) {
            if (seen[static_cast<std::size_t>(i)]) fail(BE_ERR_DUPLICATE_ENTRY, "matrix market: repeated diagonal entry");
            seen[static_cast<std::size_t>(i)] = 1;
            m.diag[static_cast<std::size_t>(i)] = v;
        } else {
            m.lower.push_back(i > j ? be_triple{i, j, v} : be_triple{j, i, v});  // upper-given entries mirrored
        }
    }
    return m;
}

MmMatrix read_matrix_market_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) fail(BE_ERR_PARSE, "matrix market: cannot open " + path);
    std::string s((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return parse_matrix_market(s.data(), s.size());
}

// write_matrix_market (matrix_market.hpp:98-113): lower entries, then the
// nonzero diagonal entries, values with 17 significant digits
std::string write_matrix_market(index_t n, const be_triple* lower, index_t nlower, const double* diag) {
    index_t nd = 0;
    for (index_t i = 0; i < n; ++i) nd += diag[i] != 0.0;
    std::string out = "%%MatrixMarket matrix coordinate real symmetric\n";
    char buf[96];
    std::snprintf(buf, sizeof buf, "%lld %lld %lld\n", static_cast<long long>(n), static_cast<long long>(n),
                  static_cast<long long>(nlower + nd));
    out += buf;
    auto entry = [&](index_t r, index_t c, double v) {
        std::snprintf(buf, sizeof buf, "%lld %lld %.17g\n", static_cast<long long>(r + 1), static_cast<long long>(c + 1), v);
        out += buf;
    };
    for (index_t e = 0; e < nlower; ++e) entry(lower[e].row, lower[e].col, lower[e].value);
    for (index_t i = 0; i < n; ++i)
        if (diag[i] != 0.0) entry(i, i, diag[i]);
    return out;
}

}  // namespace be
