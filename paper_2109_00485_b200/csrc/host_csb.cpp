// Host-side CSB_Coo storage and input generators.
//
// build_csb_coo and friends restate csb.hpp:67-202 so that the arrays handed
// to the device are byte-identical to what the reference builds from the same
// triples; the CSB1 cache follows csb.hpp:204-302 (+ the diagonal section the
// driver appends, driver.hpp:136-161). generate_synthetic restates
// synth.hpp:63-158 draw for draw (same std::mt19937_64 stream). The clustered
// generator is new tooling for the Test-1..3 shapes.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>
#include <numeric>
#include <random>

#include "host_csb.hpp"

namespace be {

void parallel_for_dynamic(int nw, index_t njobs, const std::function<void(index_t, int)>& fn) {
    std::atomic<index_t> next{0};
    fan_out(static_cast<int>(std::max<index_t>(1, std::min<index_t>(nw, njobs))), [&](int w) {
        for (;;) {
            const index_t j = next.fetch_add(1, std::memory_order_relaxed);
            if (j >= njobs) return;
            fn(j, w);
        }
    });
}

// ---------------------------------------------------------------------------
// boundaries (csb.hpp:67-96)
// ---------------------------------------------------------------------------

static void check_bounds(const index_t* b, index_t nb, index_t n, const char* what) {
    if (nb < 2 || b[0] != 0 || b[nb - 1] != n)
        fail(BE_ERR_BAD_PARAMS, std::string(what) + " boundaries must start at 0 and end at the dimension");
    for (index_t i = 1; i < nb; ++i) {
        if (b[i] <= b[i - 1]) fail(BE_ERR_BAD_PARAMS, std::string(what) + " boundaries must be strictly increasing");
        if (b[i] - b[i - 1] > kMaxBlockExtent)
            fail(BE_ERR_BLOCK_TOO_LARGE, std::string(what) + " block extent exceeds 32000");
    }
}

std::vector<index_t> uniform_boundaries(index_t n, index_t extent) {
    if (n <= 0) fail(BE_ERR_BAD_PARAMS, "uniform_boundaries: empty dimension");
    if (extent <= 0 || extent > kMaxBlockExtent) fail(BE_ERR_BAD_PARAMS, "uniform_boundaries: bad extent");
    const index_t nblk = (n + extent - 1) / extent;
    std::vector<index_t> b(static_cast<std::size_t>(nblk + 1));
    for (index_t i = 0; i <= nblk; ++i) b[static_cast<std::size_t>(i)] = std::min(n, i * extent);
    return b;
}

static std::vector<std::int32_t> lookup(const index_t* b, index_t nb) {
    std::vector<std::int32_t> lut(static_cast<std::size_t>(b[nb - 1]));
    for (index_t k = 0; k + 1 < nb; ++k)
        for (index_t i = b[k]; i < b[k + 1]; ++i) lut[static_cast<std::size_t>(i)] = static_cast<std::int32_t>(k);
    return lut;
}

// ---------------------------------------------------------------------------
// build_csb_coo (csb.hpp:100-161). Parallel, but the result is identical to
// the serial reference: each worker scans a contiguous slice of the input and
// the per-(worker, block) cursors are laid out in worker order, so entries of
// one block keep their input order.
// ---------------------------------------------------------------------------

void CsbHost::allocate(index_t nnz_) {
    nnz = nnz_;
    local_rows.reset(nnz);
    local_cols.reset(nnz);
    values.reset(nnz);
}

std::unique_ptr<CsbHost> build_csb(const be_triple* t, index_t count, index_t nrows, index_t ncols,
                                   const index_t* rb, index_t nrb, const index_t* cb, index_t ncb) {
    check_bounds(rb, nrb, nrows, "row");
    check_bounds(cb, ncb, ncols, "column");
    auto m = std::make_unique<CsbHost>();
    m->nrows = nrows;
    m->ncols = ncols;
    m->nrowblks = nrb - 1;
    m->ncolblks = ncb - 1;
    m->row_offsets.assign(rb, rb + nrb);
    m->col_offsets.assign(cb, cb + ncb);
    const index_t nblocks = m->nrowblks * m->ncolblks;
    m->block_nnz.assign(static_cast<std::size_t>(nblocks), 0);
    m->block_nnz_offsets.assign(static_cast<std::size_t>(nblocks), 0);

    // range check in input order: the first offending entry is reported,
    // exactly as the counting loop of csb.hpp:125-132 would
    for (index_t i = 0; i < count; ++i) {
        const be_triple& e = t[i];
        if (e.row < 0 || e.row >= nrows || e.col < 0 || e.col >= ncols)
            fail(BE_ERR_INDEX_OUT_OF_RANGE, "build_csb_coo: entry (" + std::to_string(e.row) + ", " +
                                                std::to_string(e.col) + ") outside the matrix");
    }
    const auto rlut = lookup(rb, nrb);
    const auto clut = lookup(cb, ncb);

    const int nw = static_cast<int>(std::max<index_t>(1, std::min<index_t>(hw_threads(), count / 65536 + 1)));
    std::vector<std::vector<index_t>> cnt(static_cast<std::size_t>(nw));
    auto slice = [&](int w, index_t& b, index_t& e) {
        b = count * w / nw;
        e = count * (w + 1) / nw;
    };
    fan_out(nw, [&](int w) {
        auto& c = cnt[static_cast<std::size_t>(w)];
        c.assign(static_cast<std::size_t>(nblocks), 0);
        index_t b, e;
        slice(w, b, e);
        for (index_t i = b; i < e; ++i)
            ++c[static_cast<std::size_t>(rlut[static_cast<std::size_t>(t[i].row)]) * m->ncolblks +
                clut[static_cast<std::size_t>(t[i].col)]];
    });
    for (int w = 0; w < nw; ++w)
        for (index_t b = 0; b < nblocks; ++b) m->block_nnz[static_cast<std::size_t>(b)] += cnt[static_cast<std::size_t>(w)][static_cast<std::size_t>(b)];

    // duplicate detection (csb.hpp:135-144): a repeated coordinate always
    // falls into one block, so sorting keys block by block is equivalent to
    // the reference's single global sort
    {
        std::vector<index_t> off(static_cast<std::size_t>(nblocks + 1), 0);
        for (index_t b = 0; b < nblocks; ++b) off[static_cast<std::size_t>(b + 1)] = off[static_cast<std::size_t>(b)] + m->block_nnz[static_cast<std::size_t>(b)];
        Buf<std::uint64_t> keys(count);
        std::vector<index_t> cur(off.begin(), off.end() - 1);
        for (index_t i = 0; i < count; ++i) {
            const index_t b = static_cast<index_t>(rlut[static_cast<std::size_t>(t[i].row)]) * m->ncolblks + clut[static_cast<std::size_t>(t[i].col)];
            keys[cur[static_cast<std::size_t>(b)]++] =
                static_cast<std::uint64_t>(t[i].row) * static_cast<std::uint64_t>(ncols) + static_cast<std::uint64_t>(t[i].col);
        }
        std::atomic<bool> dup{false};
        parallel_for_dynamic(hw_threads(), nblocks, [&](index_t b, int) {
            std::uint64_t* k0 = keys.data() + off[static_cast<std::size_t>(b)];
            std::uint64_t* k1 = keys.data() + off[static_cast<std::size_t>(b + 1)];
            std::sort(k0, k1);
            if (std::adjacent_find(k0, k1) != k1) dup = true;
        });
        if (dup) fail(BE_ERR_DUPLICATE_ENTRY, "build_csb_coo: duplicate coordinate in input");
    }

    index_t acc = 0;
    for (index_t b = 0; b < nblocks; ++b) {
        m->block_nnz_offsets[static_cast<std::size_t>(b)] = acc;
        acc += m->block_nnz[static_cast<std::size_t>(b)];
    }
    m->allocate(count);
    // per-worker cursors: block offset + counts of all lower-numbered workers
    std::vector<std::vector<index_t>> cursor(static_cast<std::size_t>(nw));
    {
        std::vector<index_t> run(m->block_nnz_offsets);
        for (int w = 0; w < nw; ++w) {
            cursor[static_cast<std::size_t>(w)] = run;
            for (index_t b = 0; b < nblocks; ++b) run[static_cast<std::size_t>(b)] += cnt[static_cast<std::size_t>(w)][static_cast<std::size_t>(b)];
        }
    }
    fan_out(nw, [&](int w) {
        auto& cur = cursor[static_cast<std::size_t>(w)];
        index_t b, e;
        slice(w, b, e);
        for (index_t i = b; i < e; ++i) {
            const index_t bi = rlut[static_cast<std::size_t>(t[i].row)];
            const index_t bj = clut[static_cast<std::size_t>(t[i].col)];
            const index_t k = cur[static_cast<std::size_t>(bi * m->ncolblks + bj)]++;
            m->local_rows[k] = static_cast<std::uint16_t>(t[i].row - rb[bi]);
            m->local_cols[k] = static_cast<std::uint16_t>(t[i].col - cb[bj]);
            m->values[k] = t[i].value;
        }
    });
    return m;
}

be_csb_view CsbHost::view() const {
    be_csb_view v{};
    v.nrows = nrows;
    v.ncols = ncols;
    v.nrowblks = nrowblks;
    v.ncolblks = ncolblks;
    v.nnz = nnz;
    v.row_offsets = row_offsets.data();
    v.col_offsets = col_offsets.data();
    v.block_nnz = block_nnz.data();
    v.block_nnz_offsets = block_nnz_offsets.data();
    v.local_rows = local_rows.data();
    v.local_cols = local_cols.data();
    v.values = values.data();
    return v;
}

void validate_view(const be_csb_view& v) {
    if (v.nrows < 0 || v.ncols < 0 || v.nrowblks < 1 || v.ncolblks < 1)
        fail(BE_ERR_BAD_PARAMS, "csb view: bad shape");
    if (!v.row_offsets || !v.col_offsets || !v.block_nnz || !v.block_nnz_offsets)
        fail(BE_ERR_BAD_PARAMS, "csb view: null table");
    if (v.nnz > 0 && (!v.local_rows || !v.local_cols || !v.values)) fail(BE_ERR_BAD_PARAMS, "csb view: null arrays");
    check_bounds(v.row_offsets, v.nrowblks + 1, v.nrows, "row");
    check_bounds(v.col_offsets, v.ncolblks + 1, v.ncols, "column");
    index_t total = 0;
    for (index_t b = 0; b < v.nrowblks * v.ncolblks; ++b) {
        if (v.block_nnz[b] < 0 || v.block_nnz_offsets[b] < 0 || v.block_nnz_offsets[b] + v.block_nnz[b] > v.nnz)
            fail(BE_ERR_BAD_PARAMS, "csb view: block table out of range");
        total += v.block_nnz[b];
    }
    if (total != v.nnz) fail(BE_ERR_BAD_PARAMS, "csb view: block_nnz does not sum to nnz");
}

// is_strictly_lower (csb.hpp:188-202)
bool is_strictly_lower(const be_csb_view& v) {
    std::atomic<bool> ok{true};
    parallel_for_dynamic(hw_threads(), v.nrowblks, [&](index_t bi, int) {
        if (!ok) return;
        for (index_t bj = 0; bj < v.ncolblks; ++bj) {
            const index_t b = bi * v.ncolblks + bj;
            const index_t k0 = v.block_nnz_offsets[b], k1 = k0 + v.block_nnz[b];
            const index_t rbase = v.row_offsets[bi], cbase = v.col_offsets[bj];
            for (index_t k = k0; k < k1; ++k)
                if (rbase + v.local_rows[k] <= cbase + v.local_cols[k]) {
                    ok = false;
                    return;
                }
        }
    });
    return ok;
}

// to_triples (csb.hpp:165-185)
void to_triples(const be_csb_view& v, be_triple* out) {
    index_t p = 0;
    for (index_t bi = 0; bi < v.nrowblks; ++bi)
        for (index_t bj = 0; bj < v.ncolblks; ++bj) {
            const index_t b = bi * v.ncolblks + bj;
            const index_t k0 = v.block_nnz_offsets[b], k1 = k0 + v.block_nnz[b];
            for (index_t k = k0; k < k1; ++k)
                out[p++] = {v.row_offsets[bi] + v.local_rows[k], v.col_offsets[bj] + v.local_cols[k], v.values[k]};
        }
}

// ---------------------------------------------------------------------------
// CSB1 cache (csb.hpp:204-302), little-endian, + optional diagonal section
// (u64 length, f64 values) as written by driver.hpp:153-160.
// ---------------------------------------------------------------------------

template <class T>
static void put(std::ostream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <class T>
static T get(std::istream& is) {
    T v{};
    is.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!is) fail(BE_ERR_PARSE, "CSB1 cache: truncated file");
    return v;
}

void save_csb1(const std::string& path, const be_csb_view& v, const double* diag, index_t ndiag) {
    std::ofstream os(path, std::ios::binary);
    if (!os) fail(BE_ERR_PARSE, "cannot open " + path + " for writing");
    save_csb1(os, v, diag, ndiag);
    if (!os) fail(BE_ERR_PARSE, "CSB1 cache: write failed for " + path);
}

void save_csb1(std::ostream& os, const be_csb_view& v, const double* diag, index_t ndiag) {
    os.write("CSB1", 4);
    put<std::uint64_t>(os, static_cast<std::uint64_t>(v.nrows));
    put<std::uint64_t>(os, static_cast<std::uint64_t>(v.ncols));
    put<std::uint64_t>(os, static_cast<std::uint64_t>(v.nrowblks));
    put<std::uint64_t>(os, static_cast<std::uint64_t>(v.ncolblks));
    auto put_u64s = [&](const index_t* a, index_t n) {
        for (index_t i = 0; i < n; ++i) put<std::uint64_t>(os, static_cast<std::uint64_t>(a[i]));
    };
    put_u64s(v.row_offsets, v.nrowblks + 1);
    put_u64s(v.col_offsets, v.ncolblks + 1);
    put_u64s(v.block_nnz, v.nrowblks * v.ncolblks);
    put_u64s(v.block_nnz_offsets, v.nrowblks * v.ncolblks);
    // interleaved (row, col) u16 pairs, written in large chunks
    {
        const index_t chunk = 1 << 20;
        std::vector<std::uint16_t> buf(static_cast<std::size_t>(2 * chunk));
        for (index_t k0 = 0; k0 < v.nnz; k0 += chunk) {
            const index_t k1 = std::min(v.nnz, k0 + chunk);
            for (index_t k = k0; k < k1; ++k) {
                buf[static_cast<std::size_t>(2 * (k - k0))] = v.local_rows[k];
                buf[static_cast<std::size_t>(2 * (k - k0) + 1)] = v.local_cols[k];
            }
            os.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(4 * (k1 - k0)));
        }
    }
    os.write(reinterpret_cast<const char*>(v.values), static_cast<std::streamsize>(v.nnz * 8));
    if (diag) {
        put<std::uint64_t>(os, static_cast<std::uint64_t>(ndiag));
        os.write(reinterpret_cast<const char*>(diag), static_cast<std::streamsize>(ndiag * 8));
    }
    if (!os) fail(BE_ERR_PARSE, "CSB1 cache: write failed");
}

// Block rows [b0, b1) of a CSB1 file (global shape and blocks kept, other
// rows empty): the header and block tables are read, then only the slab's
// contiguous ranges of the index and value sections (a multi-GPU rank loads
// its own slab of a Test-3-sized cache without reading the rest). diag, when
// given, receives the cached diagonal of those block rows' rows.
// Header of a CSB1 file only: dimension, block rows and the stored entries per block row.
std::vector<index_t> csb1_block_row_nnz(const std::string& path, index_t& nrows, index_t& nrowblks) {
    std::ifstream is(path, std::ios::binary);
    if (!is) fail(BE_ERR_PARSE, "cannot open " + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "CSB1", 4) != 0) fail(BE_ERR_PARSE, "CSB1 cache: bad magic");
    nrows = static_cast<index_t>(get<std::uint64_t>(is));
    get<std::uint64_t>(is);  // ncols
    nrowblks = static_cast<index_t>(get<std::uint64_t>(is));
    const index_t ncolblks = static_cast<index_t>(get<std::uint64_t>(is));
    if (nrowblks < 1 || ncolblks < 1 || nrowblks > (1 << 24) || ncolblks > (1 << 24))
        fail(BE_ERR_PARSE, "CSB1 cache: implausible block counts");
    for (index_t i = 0; i < nrowblks + 1 + ncolblks + 1; ++i) get<std::uint64_t>(is);
    std::vector<index_t> brn(static_cast<std::size_t>(nrowblks), 0);
    for (index_t b = 0; b < nrowblks * ncolblks; ++b) brn[static_cast<std::size_t>(b / ncolblks)] += static_cast<index_t>(get<std::uint64_t>(is));
    if (!is) fail(BE_ERR_PARSE, "CSB1 cache: truncated header");
    return brn;
}

std::unique_ptr<CsbHost> load_csb1_rows(const std::string& path, index_t b0, index_t b1, std::vector<double>* diag) {
    std::ifstream is(path, std::ios::binary);
    if (!is) fail(BE_ERR_PARSE, "cannot open " + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "CSB1", 4) != 0) fail(BE_ERR_PARSE, "CSB1 cache: bad magic");
    auto m = std::make_unique<CsbHost>();
    m->nrows = static_cast<index_t>(get<std::uint64_t>(is));
    m->ncols = static_cast<index_t>(get<std::uint64_t>(is));
    m->nrowblks = static_cast<index_t>(get<std::uint64_t>(is));
    m->ncolblks = static_cast<index_t>(get<std::uint64_t>(is));
    if (m->nrowblks < 1 || m->ncolblks < 1 || m->nrowblks > (1 << 24) || m->ncolblks > (1 << 24))
        fail(BE_ERR_PARSE, "CSB1 cache: implausible block counts");
    if (b0 < 0 || b1 < b0 || b1 > m->nrowblks) fail(BE_ERR_BAD_PARAMS, "load_csb rows: bad block-row range");
    auto get_u64s = [&](std::vector<index_t>& a, index_t n) {
        a.resize(static_cast<std::size_t>(n));
        for (auto& x : a) x = static_cast<index_t>(get<std::uint64_t>(is));
    };
    get_u64s(m->row_offsets, m->nrowblks + 1);
    get_u64s(m->col_offsets, m->ncolblks + 1);
    std::vector<index_t> bn, bo;
    get_u64s(bn, m->nrowblks * m->ncolblks);
    get_u64s(bo, m->nrowblks * m->ncolblks);
    if (!is) fail(BE_ERR_PARSE, "CSB1 cache: truncated header");
    const std::streamoff data0 = is.tellg();
    const index_t nnz_all = std::accumulate(bn.begin(), bn.end(), index_t{0});
    const index_t nb = m->ncolblks;
    const index_t k0 = b0 < m->nrowblks ? bo[static_cast<std::size_t>(b0 * nb)] : nnz_all;
    const index_t k1 = b1 < m->nrowblks ? bo[static_cast<std::size_t>(b1 * nb)] : nnz_all;
    m->block_nnz.assign(bn.size(), 0);
    m->block_nnz_offsets.assign(bn.size(), 0);
    index_t acc = 0;
    for (std::size_t b = 0; b < bn.size(); ++b) {
        const index_t bi = static_cast<index_t>(b) / nb;
        if (bi >= b0 && bi < b1) m->block_nnz[b] = bn[b];
        m->block_nnz_offsets[b] = acc;
        acc += m->block_nnz[b];
    }
    if (acc != k1 - k0) fail(BE_ERR_PARSE, "CSB1 cache: block tables are not block row-major");
    m->allocate(acc);
    is.seekg(data0 + static_cast<std::streamoff>(4 * k0));
    {
        const index_t chunk = 1 << 20;
        std::vector<std::uint16_t> buf(static_cast<std::size_t>(2 * chunk));
        for (index_t q0 = 0; q0 < acc; q0 += chunk) {
            const index_t q1 = std::min(acc, q0 + chunk);
            is.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(4 * (q1 - q0)));
            if (!is) fail(BE_ERR_PARSE, "CSB1 cache: truncated file");
            for (index_t k = q0; k < q1; ++k) {
                m->local_rows[k] = buf[static_cast<std::size_t>(2 * (k - q0))];
                m->local_cols[k] = buf[static_cast<std::size_t>(2 * (k - q0) + 1)];
            }
        }
    }
    is.seekg(data0 + static_cast<std::streamoff>(4 * nnz_all + 8 * k0));
    is.read(reinterpret_cast<char*>(m->values.data()), static_cast<std::streamsize>(acc * 8));
    if (!is) fail(BE_ERR_PARSE, "CSB1 cache: truncated values");
    if (diag) {
        diag->clear();
        is.seekg(data0 + static_cast<std::streamoff>(12 * nnz_all));
        std::uint64_t dlen = 0;
        is.read(reinterpret_cast<char*>(&dlen), 8);
        if (is && dlen > 0) {
            if (static_cast<index_t>(dlen) != m->nrows) fail(BE_ERR_PARSE, "cache: diagonal length mismatch");
            const index_t r0 = m->row_offsets[static_cast<std::size_t>(b0)], r1 = m->row_offsets[static_cast<std::size_t>(b1)];
            is.seekg(data0 + static_cast<std::streamoff>(12 * nnz_all + 8 + 8 * r0));
            diag->resize(static_cast<std::size_t>(r1 - r0));
            is.read(reinterpret_cast<char*>(diag->data()), static_cast<std::streamsize>((r1 - r0) * 8));
            if (!is) fail(BE_ERR_PARSE, "cache: truncated diagonal section");
        }
    }
    m->nnz = acc;
    return m;
}

std::unique_ptr<CsbHost> load_csb1(const std::string& path, std::vector<double>* diag) {
    std::ifstream is(path, std::ios::binary);
    if (!is) fail(BE_ERR_PARSE, "cannot open " + path);
    return load_csb1(is, diag);
}

std::unique_ptr<CsbHost> load_csb1(std::istream& is, std::vector<double>* diag) {
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "CSB1", 4) != 0) fail(BE_ERR_PARSE, "CSB1 cache: bad magic");
    auto m = std::make_unique<CsbHost>();
    m->nrows = static_cast<index_t>(get<std::uint64_t>(is));
    m->ncols = static_cast<index_t>(get<std::uint64_t>(is));
    m->nrowblks = static_cast<index_t>(get<std::uint64_t>(is));
    m->ncolblks = static_cast<index_t>(get<std::uint64_t>(is));
    if (m->nrowblks < 1 || m->ncolblks < 1 || m->nrowblks > (1 << 24) || m->ncolblks > (1 << 24))
        fail(BE_ERR_PARSE, "CSB1 cache: implausible block counts");
    auto get_u64s = [&](std::vector<index_t>& a, index_t n) {
        a.resize(static_cast<std::size_t>(n));
        for (auto& x : a) x = static_cast<index_t>(get<std::uint64_t>(is));
    };
    get_u64s(m->row_offsets, m->nrowblks + 1);
    get_u64s(m->col_offsets, m->ncolblks + 1);
    get_u64s(m->block_nnz, m->nrowblks * m->ncolblks);
    get_u64s(m->block_nnz_offsets, m->nrowblks * m->ncolblks);
    const index_t nnz = std::accumulate(m->block_nnz.begin(), m->block_nnz.end(), index_t{0});
    m->allocate(nnz);
    {
        const index_t chunk = 1 << 20;
        std::vector<std::uint16_t> buf(static_cast<std::size_t>(2 * chunk));
        for (index_t k0 = 0; k0 < nnz; k0 += chunk) {
            const index_t k1 = std::min(nnz, k0 + chunk);
            is.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(4 * (k1 - k0)));
            if (!is) fail(BE_ERR_PARSE, "CSB1 cache: truncated file");
            for (index_t k = k0; k < k1; ++k) {
                m->local_rows[k] = buf[static_cast<std::size_t>(2 * (k - k0))];
                m->local_cols[k] = buf[static_cast<std::size_t>(2 * (k - k0) + 1)];
            }
        }
    }
    is.read(reinterpret_cast<char*>(m->values.data()), static_cast<std::streamsize>(nnz * 8));
    if (!is) fail(BE_ERR_PARSE, "CSB1 cache: truncated values");
    if (diag) {
        diag->clear();
        std::uint64_t dlen = 0;
        is.read(reinterpret_cast<char*>(&dlen), 8);
        if (is) {
            diag->resize(dlen);
            is.read(reinterpret_cast<char*>(diag->data()), static_cast<std::streamsize>(dlen * 8));
            if (!is) fail(BE_ERR_PARSE, "cache: truncated diagonal section");
        }
    }
    return m;
}

// ---------------------------------------------------------------------------
// generate_synthetic (synth.hpp:63-158), draw for draw.
// ---------------------------------------------------------------------------

std::vector<index_t> draw_tile_offsets(index_t n, index_t block_extent, index_t tile_min, index_t tile_max,
                                       std::mt19937_64& rng) {
    // synth.hpp:67-83
    const index_t lo = std::max<index_t>(1, std::min(tile_min, n));
    const index_t hi = std::max(lo, std::min(tile_max, n));
    std::uniform_real_distribution<double> u(std::log(static_cast<double>(lo)), std::log(static_cast<double>(hi)));
    std::vector<index_t> off = {0};
    while (off.back() < n) {
        const index_t at = off.back();
        index_t size = std::max<index_t>(1, static_cast<index_t>(std::llround(std::exp(u(rng)))));
        const index_t block_end = ((at / block_extent) + 1) * block_extent;
        off.push_back(std::min({at + size, block_end, n}));
    }
    return off;
}

namespace {
// open-addressing set of u64 keys (0 reserved): same accept/reject decisions
// as the reference's std::unordered_set, several times faster
struct KeySet {
    std::vector<std::uint64_t> slot;
    std::uint64_t mask = 0;
    explicit KeySet(index_t expected) {
        std::uint64_t cap = 16;
        while (cap < static_cast<std::uint64_t>(expected) * 2 + 16) cap <<= 1;
        slot.assign(cap, 0);
        mask = cap - 1;
    }
    static std::uint64_t mix(std::uint64_t x) {
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdULL;
        x ^= x >> 33;
        x *= 0xc4ceb9fe1a85ec53ULL;
        x ^= x >> 33;
        return x;
    }
    bool insert(std::uint64_t key) {
        const std::uint64_t k = key + 1;
        for (std::uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
            if (slot[h] == k) return false;
            if (slot[h] == 0) {
                slot[h] = k;
                return true;
            }
        }
    }
};
}  // namespace

std::unique_ptr<Synth> generate_synthetic(const be_synth_params& p) {
    // SynthParams::validate, synth.hpp:45-55
    if (p.n < 10) fail(BE_ERR_BAD_PARAMS, "generate_synthetic: n must be at least 10");
    if (p.kind == BE_SYNTH_RANDOM && (p.density <= 0.0 || p.density > 0.5))
        fail(BE_ERR_BAD_PARAMS, "generate_synthetic: density must lie in (0, 0.5]");
    if (p.bandwidth < 0) fail(BE_ERR_BAD_PARAMS, "generate_synthetic: bandwidth must be non-negative");
    if (p.block_extent < 1 || p.block_extent > kMaxBlockExtent) fail(BE_ERR_BAD_PARAMS, "generate_synthetic: bad block extent");
    if (p.tile_min < 1 || p.tile_max < p.tile_min) fail(BE_ERR_BAD_PARAMS, "generate_synthetic: bad tile size range");
    if (p.dominance < 0.0) fail(BE_ERR_BAD_PARAMS, "generate_synthetic: dominance must be non-negative");
    if (p.kind < 0 || p.kind > 2) fail(BE_ERR_BAD_PARAMS, "unknown generator kind");

    auto s = std::make_unique<Synth>();
    std::mt19937_64 rng(p.seed);
    std::uniform_real_distribution<double> val(-1.0, 1.0);
    s->n = p.n;
    s->tile_offsets = draw_tile_offsets(p.n, p.block_extent, p.tile_min, p.tile_max, rng);
    auto& lower = s->lower;
    switch (p.kind) {
        case BE_SYNTH_BANDED:
            for (index_t i = 0; i < p.n; ++i)
                for (index_t d = 1; d <= p.bandwidth && d <= i; ++d) lower.push_back({i, i - d, val(rng)});
            break;
        case BE_SYNTH_RANDOM: {
            const auto target = static_cast<index_t>(
                std::llround(p.density * static_cast<double>(p.n) * static_cast<double>(p.n - 1) / 2.0));
            KeySet used(target);
            lower.reserve(static_cast<std::size_t>(target));
            std::uniform_int_distribution<index_t> draw(0, p.n - 1);
            index_t have = 0;
            while (have < target) {
                index_t r = draw(rng), c = draw(rng);
                if (r == c) continue;
                if (r < c) std::swap(r, c);
                const std::uint64_t key = static_cast<std::uint64_t>(r) * static_cast<std::uint64_t>(p.n) + static_cast<std::uint64_t>(c);
                if (used.insert(key)) {
                    lower.push_back({r, c, val(rng)});
                    ++have;
                }
            }
            break;
        }
        case BE_SYNTH_BLOCKTILE: {
            std::uniform_real_distribution<double> coin(0.0, 1.0);
            const double tile_fill = 0.3, coupling_fill = 0.01;
            const auto& off = s->tile_offsets;
            for (std::size_t t = 0; t + 1 < off.size(); ++t)
                for (index_t i = off[t]; i < off[t + 1]; ++i)
                    for (index_t j = off[t]; j < i; ++j)
                        if (coin(rng) < tile_fill) lower.push_back({i, j, val(rng)});
            for (std::size_t t = 1; t + 1 < off.size(); ++t) {
                if (off[t - 1] / p.block_extent != (off[t + 1] - 1) / p.block_extent) continue;
                for (index_t i = off[t]; i < off[t + 1]; ++i)
                    for (index_t j = off[t - 1]; j < off[t]; ++j)
                        if (coin(rng) < coupling_fill) lower.push_back({i, j, val(rng)});
            }
            break;
        }
    }
    s->diag.assign(static_cast<std::size_t>(p.n), 0.0);
    std::vector<double> rowabs(static_cast<std::size_t>(p.n), 0.0);
    for (const be_triple& t : lower) {
        rowabs[static_cast<std::size_t>(t.row)] += std::abs(t.value);
        rowabs[static_cast<std::size_t>(t.col)] += std::abs(t.value);
    }
    std::uniform_real_distribution<double> spread(0.0, p.diag_spread);
    for (index_t i = 0; i < p.n; ++i)
        s->diag[static_cast<std::size_t>(i)] = 0.5 + spread(rng) + p.dominance * rowabs[static_cast<std::size_t>(i)];
    return s;
}

// ---------------------------------------------------------------------------
// Clustered generator (new tooling). Counter-based streams keyed
// by (seed, block, tile) -> identical output for any thread count.
// ---------------------------------------------------------------------------

namespace {
inline std::uint64_t splitmix(std::uint64_t& s) {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline std::uint64_t hash4(std::uint64_t a, std::uint64_t b, std::uint64_t c, std::uint64_t d) {
    std::uint64_t s = a ^ 0x5851f42d4c957f2dULL;
    splitmix(s);
    s ^= b * 0x2545f4914f6cdd1dULL;
    splitmix(s);
    s ^= c * 0x9e3779b97f4a7c15ULL;
    splitmix(s);
    s ^= d * 0xda942042e4dd58b5ULL;
    return splitmix(s);
}
inline double unit(std::uint64_t x) { return static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0); }

struct ClusterPlan {
    const be_cluster_params& p;
    std::vector<index_t> bounds;
    index_t nblk;
    double p_tile;
    ClusterPlan(const be_cluster_params& pp) : p(pp) {}
    bool block_on(index_t bi, index_t bj) const {
        if (bi == bj) return true;
        return unit(hash4(p.seed, 0xB10C, static_cast<std::uint64_t>(bi), static_cast<std::uint64_t>(bj))) < p.block_occupancy;
    }
    // occupied sub-tile? diagonal tiles of diagonal blocks always are
    bool tile_on(index_t bi, index_t bj, index_t a, index_t b) const {
        if (bi == bj && a == b) return true;
        const std::uint64_t key = static_cast<std::uint64_t>(bi) * 0x100000000ULL + static_cast<std::uint64_t>(bj);
        return unit(hash4(p.seed, key, static_cast<std::uint64_t>(a), static_cast<std::uint64_t>(b) + 0x7713)) < p_tile;
    }
    // visit the strictly-lower positions of one occupied tile via geometric
    // skipping over its row-major linear index
    template <class F>
    void tile_entries(index_t bi, index_t bj, index_t a, index_t b, index_t br, index_t bc, bool with_values, F&& f) const {
        const index_t r0 = a * p.tile, c0 = b * p.tile;
        const index_t tr = std::min(p.tile, br - r0), tc = std::min(p.tile, bc - c0);
        const bool diag_tile = (bi == bj && a == b);
        const std::uint64_t key = static_cast<std::uint64_t>(bi) * 0x100000000ULL + static_cast<std::uint64_t>(bj);
        std::uint64_t gs = hash4(p.seed ^ 0x6A09E667F3BCC908ULL, key, static_cast<std::uint64_t>(a), static_cast<std::uint64_t>(b));
        std::uint64_t vs = hash4(p.seed ^ 0xBB67AE8584CAA73BULL, key, static_cast<std::uint64_t>(a), static_cast<std::uint64_t>(b));
        const double lq = std::log1p(-p.fill);
        const index_t area = tr * tc;
        index_t pos = -1;
        for (;;) {
            index_t gap = 1;
            if (p.fill < 1.0) {
                const double u = 1.0 - unit(splitmix(gs));  // (0, 1]
                gap = 1 + static_cast<index_t>(std::floor(std::log(u) / lq));
            }
            pos += gap;
            if (pos >= area || pos < 0) break;
            const index_t lr = r0 + pos / tc, lc = c0 + pos % tc;
            if (diag_tile && lr <= lc) continue;
            double v = 0.0;
            if (with_values) v = 2.0 * unit(splitmix(vs)) - 1.0;
            f(lr, lc, v);
        }
    }
};
}  // namespace

// Plan shared by the whole-matrix and the slab generators: the boundaries
// and the occupied-tile rate p_tile that meets target_nnz on average.
static ClusterPlan make_plan(const be_cluster_params& p) {
    if (p.n < 10) fail(BE_ERR_BAD_PARAMS, "generate_clustered: n must be at least 10");
    if (p.block_extent < 1 || p.block_extent > kMaxBlockExtent) fail(BE_ERR_BAD_PARAMS, "generate_clustered: bad block extent");
    if (p.tile < 1 || p.tile > p.block_extent) fail(BE_ERR_BAD_PARAMS, "generate_clustered: bad tile");
    if (!(p.fill > 0.0 && p.fill <= 1.0)) fail(BE_ERR_BAD_PARAMS, "generate_clustered: fill must lie in (0, 1]");
    if (!(p.block_occupancy > 0.0 && p.block_occupancy <= 1.0)) fail(BE_ERR_BAD_PARAMS, "generate_clustered: bad block occupancy");
    if (p.target_nnz < 0) fail(BE_ERR_BAD_PARAMS, "generate_clustered: negative target");
    if (p.tile_min < 1 || p.tile_max < p.tile_min) fail(BE_ERR_BAD_PARAMS, "generate_clustered: bad tile size range");
    ClusterPlan plan(p);
    plan.bounds = uniform_boundaries(p.n, p.block_extent);
    plan.nblk = static_cast<index_t>(plan.bounds.size()) - 1;
    const index_t nblk = plan.nblk;
    const auto& B = plan.bounds;
    auto ntiles_of = [&](index_t len) { return (len + p.tile - 1) / p.tile; };
    // expected area: diagonal tiles of diagonal blocks (strict lower part)
    // always, the other lower tiles of occupied blocks at rate p_tile
    double diag_area = 0.0, other_area = 0.0;
    for (index_t bi = 0; bi < nblk; ++bi) {
        const index_t br = B[bi + 1] - B[bi];
        const index_t nt = ntiles_of(br);
        for (index_t a = 0; a < nt; ++a) {
            const double t = static_cast<double>(std::min(p.tile, br - a * p.tile));
            diag_area += t * (t - 1) / 2;
            for (index_t b = 0; b < a; ++b) other_area += t * static_cast<double>(std::min(p.tile, br - b * p.tile));
        }
        for (index_t bj = 0; bj < bi; ++bj)
            if (plan.block_on(bi, bj)) other_area += static_cast<double>(br) * static_cast<double>(B[bj + 1] - B[bj]);
    }
    const double want_area = static_cast<double>(p.target_nnz) / p.fill;
    plan.p_tile = other_area > 0 ? std::clamp((want_area - diag_area) / other_area, 0.0, 1.0) : 0.0;
    return plan;
}

// Block rows [b0, b1) of the clustered matrix as a CSB of the global shape;
// diag_only keeps only the diagonal blocks (a rank's preconditioner tiles).
// The entries are exactly those of the whole-matrix generator.
static std::unique_ptr<CsbHost> clustered_rows(const ClusterPlan& plan, index_t b0, index_t b1, bool diag_only, int nw,
                                               index_t c0 = 0, index_t c1 = -1) {
    if (c1 < 0) c1 = plan.nblk;
    const auto& p = plan.p;
    const index_t nblk = plan.nblk;
    const auto& B = plan.bounds;
    auto ntiles_of = [&](index_t len) { return (len + p.tile - 1) / p.tile; };
    auto m = std::make_unique<CsbHost>();
    m->nrows = m->ncols = p.n;
    m->nrowblks = m->ncolblks = nblk;
    m->row_offsets = B;
    m->col_offsets = B;
    m->block_nnz.assign(static_cast<std::size_t>(nblk * nblk), 0);
    m->block_nnz_offsets.assign(static_cast<std::size_t>(nblk * nblk), 0);
    auto wanted = [&](index_t bi, index_t bj) {
        return bj >= c0 && bj < c1 && plan.block_on(bi, bj) && (!diag_only || bi == bj);
    };
    // pass 1: counts per block (gap stream only)
    parallel_for_dynamic(nw, b1 - b0, [&](index_t q, int) {
        const index_t bi = b0 + q;
        const index_t br = B[bi + 1] - B[bi];
        for (index_t bj = 0; bj <= bi; ++bj) {
            if (!wanted(bi, bj)) continue;
            const index_t bc = B[bj + 1] - B[bj];
            index_t c = 0;
            for (index_t a = 0; a < ntiles_of(br); ++a)
                for (index_t b = 0; b < (bi == bj ? a + 1 : ntiles_of(bc)); ++b)
                    if (plan.tile_on(bi, bj, a, b))
                        plan.tile_entries(bi, bj, a, b, br, bc, false, [&](index_t, index_t, double) { ++c; });
            m->block_nnz[static_cast<std::size_t>(bi * nblk + bj)] = c;
        }
    });
    index_t acc = 0;
    for (std::size_t b = 0; b < m->block_nnz.size(); ++b) {
        m->block_nnz_offsets[b] = acc;
        acc += m->block_nnz[b];
    }
    m->allocate(acc);
    // pass 2: fill
    parallel_for_dynamic(nw, b1 - b0, [&](index_t q, int) {
        const index_t bi = b0 + q;
        const index_t br = B[bi + 1] - B[bi];
        for (index_t bj = 0; bj <= bi; ++bj) {
            if (!wanted(bi, bj)) continue;
            const index_t bc = B[bj + 1] - B[bj];
            index_t k = m->block_nnz_offsets[static_cast<std::size_t>(bi * nblk + bj)];
            for (index_t a = 0; a < ntiles_of(br); ++a)
                for (index_t b = 0; b < (bi == bj ? a + 1 : ntiles_of(bc)); ++b)
                    if (plan.tile_on(bi, bj, a, b))
                        plan.tile_entries(bi, bj, a, b, br, bc, true, [&](index_t lr, index_t lc, double v) {
                            m->local_rows[k] = static_cast<std::uint16_t>(lr);
                            m->local_cols[k] = static_cast<std::uint16_t>(lc);
                            m->values[k] = v;
                            ++k;
                        });
        }
    });
    return m;
}

// sum |row| of the stored entries of m, row part and column part kept apart
// (each summed in a fixed order so the bytes never depend on the thread count)
static void abs_sums(const CsbHost& m, index_t b0, index_t b1, std::vector<double>& rsum, std::vector<double>& csum,
                     int nw) {
    const index_t nblk = m.nrowblks;
    const auto& B = m.row_offsets;
    rsum.assign(static_cast<std::size_t>(m.nrows), 0.0);
    csum.assign(static_cast<std::size_t>(m.nrows), 0.0);
    parallel_for_dynamic(nw, b1 - b0, [&](index_t q, int) {
        const index_t bi = b0 + q;
        for (index_t bj = 0; bj <= bi; ++bj) {
            const index_t b = bi * nblk + bj;
            const index_t k0 = m.block_nnz_offsets[static_cast<std::size_t>(b)], k1 = k0 + m.block_nnz[static_cast<std::size_t>(b)];
            for (index_t k = k0; k < k1; ++k) rsum[static_cast<std::size_t>(B[bi] + m.local_rows[k])] += std::abs(m.values[k]);
        }
    });
    parallel_for_dynamic(nw, nblk, [&](index_t bj, int) {
        for (index_t bi = std::max(bj, b0); bi < b1; ++bi) {
            const index_t b = bi * nblk + bj;
            const index_t k0 = m.block_nnz_offsets[static_cast<std::size_t>(b)], k1 = k0 + m.block_nnz[static_cast<std::size_t>(b)];
            for (index_t k = k0; k < k1; ++k) csum[static_cast<std::size_t>(B[bj] + m.local_cols[k])] += std::abs(m.values[k]);
        }
    });
}

double clustered_diag_value(const be_cluster_params& p, index_t i, double rowabs) {
    std::uint64_t s = hash4(p.seed, 0xD1A6, static_cast<std::uint64_t>(i), 0);
    return 0.5 + p.diag_spread * unit(splitmix(s)) + p.dominance * rowabs;
}

std::unique_ptr<CsbHost> generate_clustered(const be_cluster_params& p, std::vector<double>& diag,
                                            std::vector<index_t>& tile_offsets) {
    const int nw = p.threads > 0 ? p.threads : hw_threads();
    const ClusterPlan plan = make_plan(p);
    auto m = clustered_rows(plan, 0, plan.nblk, false, nw);
    // diagonal: 0.5 + U(0, spread) + dominance * sum|row| (synth.hpp:147-157 rule)
    std::vector<double> rsum, csum;
    abs_sums(*m, 0, plan.nblk, rsum, csum, nw);
    diag.resize(static_cast<std::size_t>(p.n));
    for (index_t i = 0; i < p.n; ++i)
        diag[static_cast<std::size_t>(i)] = clustered_diag_value(p, i, rsum[static_cast<std::size_t>(i)] + csum[static_cast<std::size_t>(i)]);
    std::mt19937_64 trng(p.seed + 0x7157);
    tile_offsets = draw_tile_offsets(p.n, p.block_extent, p.tile_min, p.tile_max, trng);
    return m;
}

std::unique_ptr<CsbHost> generate_clustered_part(const be_cluster_params& p, index_t b0, index_t b1, bool diag_only,
                                                 std::vector<double>& rowabs, std::vector<index_t>& tile_offsets,
                                                 index_t c0, index_t c1) {
    const int nw = p.threads > 0 ? p.threads : hw_threads();
    const ClusterPlan plan = make_plan(p);
    if (b0 < 0 || b1 < b0 || b1 > plan.nblk) fail(BE_ERR_BAD_PARAMS, "generate_clustered_part: bad block-row range");
    if (c1 < 0) c1 = plan.nblk;
    if (c0 < 0 || c1 < c0 || c1 > plan.nblk) fail(BE_ERR_BAD_PARAMS, "generate_clustered_part: bad block-column range");
    auto m = clustered_rows(plan, b0, b1, diag_only, nw, c0, c1);
    std::vector<double> rsum, csum;
    abs_sums(*m, b0, b1, rsum, csum, nw);
    rowabs.resize(static_cast<std::size_t>(p.n));
    for (std::size_t i = 0; i < rowabs.size(); ++i) rowabs[i] = rsum[i] + csum[i];
    std::mt19937_64 trng(p.seed + 0x7157);
    tile_offsets = draw_tile_offsets(p.n, p.block_extent, p.tile_min, p.tile_max, trng);
    return m;
}

// Expected stored entries of every lower block (bi, bj), row-major nblk x nblk (the 2-D tile
// weights; the block-row weights below are their row sums up to rounding).
std::vector<index_t> clustered_block_weights(const be_cluster_params& p, index_t& nblk_out) {
    const ClusterPlan plan = make_plan(p);
    const auto& B = plan.bounds;
    const index_t nblk = plan.nblk;
    nblk_out = nblk;
    std::vector<index_t> w(static_cast<std::size_t>(nblk * nblk), 0);
    auto ntiles_of = [&](index_t len) { return (len + p.tile - 1) / p.tile; };
    for (index_t bi = 0; bi < nblk; ++bi) {
        const index_t br = B[bi + 1] - B[bi];
        double e = 0.0;  // the diagonal block
        for (index_t a = 0; a < ntiles_of(br); ++a) {
            const double t = static_cast<double>(std::min(p.tile, br - a * p.tile));
            e += t * (t - 1) / 2 * p.fill;
            for (index_t b = 0; b < a; ++b) e += t * static_cast<double>(std::min(p.tile, br - b * p.tile)) * p.fill * plan.p_tile;
        }
        w[static_cast<std::size_t>(bi * nblk + bi)] = static_cast<index_t>(std::llround(e));
        for (index_t bj = 0; bj < bi; ++bj)
            if (plan.block_on(bi, bj))
                w[static_cast<std::size_t>(bi * nblk + bj)] = static_cast<index_t>(
                    std::llround(static_cast<double>(br) * static_cast<double>(B[bj + 1] - B[bj]) * p.fill * plan.p_tile));
    }
    return w;
}

std::vector<index_t> clustered_block_row_weights(const be_cluster_params& p) {
    const ClusterPlan plan = make_plan(p);
    const auto& B = plan.bounds;
    std::vector<index_t> w(static_cast<std::size_t>(plan.nblk));
    auto ntiles_of = [&](index_t len) { return (len + p.tile - 1) / p.tile; };
    for (index_t bi = 0; bi < plan.nblk; ++bi) {  // expected stored entries of block row bi
        const index_t br = B[bi + 1] - B[bi];
        double e = 0.0;
        for (index_t a = 0; a < ntiles_of(br); ++a) {
            const double t = static_cast<double>(std::min(p.tile, br - a * p.tile));
            e += t * (t - 1) / 2 * p.fill;
            for (index_t b = 0; b < a; ++b) e += t * static_cast<double>(std::min(p.tile, br - b * p.tile)) * p.fill * plan.p_tile;
        }
        for (index_t bj = 0; bj < bi; ++bj)
            if (plan.block_on(bi, bj))
                e += static_cast<double>(br) * static_cast<double>(B[bj + 1] - B[bj]) * p.fill * plan.p_tile;
        w[static_cast<std::size_t>(bi)] = static_cast<index_t>(std::llround(e));
    }
    return w;
}

}  // namespace be
