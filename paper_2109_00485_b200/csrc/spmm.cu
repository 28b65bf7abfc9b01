// Symmetric SpMM over the half-stored CSB_Coo Hamiltonian, sm_100a.
//
// Replaces SymmetricOperator::apply (kernels.hpp:357-371) = out.set_zero +
// spmm_notrans (kernels.hpp:290) + spmm_trans (kernels.hpp:302) + the
// diagonal pass (kernels.hpp:363-370). The reference walks the stored
// nonzeros twice (once per pass); this kernel streams every 128 x 128 work
// tile from HBM once and applies each entry twice (A_ij X_j -> Y_i and
// A_ij X_i -> Y_j).
//
// Device format ("work tiles", built on upload from the CSB arrays): every
// CSB block is cut into 128 x 128 sub-tiles aligned to the block origin (a
// sub-tile with more than max_nnz entries is split by rows). Each tile is ONE
// contiguous, 16-byte aligned blob, fetched with a single cp.async.bulk:
//   meta (1088 B): row-JDS starts jr[129] | column-JDS starts jc[129] (u16,
//     padded to 136) | rank -> local row (u8[128]) | rank -> local column |
//     row lengths by rank | column lengths by rank | the 8-warp work split
//     (u16[9], k_sym_spmm_ws)
//   row stream:    values[npad] (f32 or f64) | local column u8[npad]
//   column stream: values[npad]              | local row    u8[npad]
// "JDS" = jagged diagonals: diagonal d holds the d-th entry of every row
// (column) rank whose length exceeds d, ranks sorted by decreasing length, so
// lane r of a warp reads word jr[d] + r -- consecutive words, one shared-
// memory wavefront per 32 entries, in both passes (no indirection). In f32
// that is 10 B per stored entry (the value is stored once per pass order).
//
// Kernel: persistent CTAs of 256 threads (2 per SM) pull work items ("runs":
// up to 32 consecutive tiles of one tile-row inside one L2 column band) from
// an atomic counter, and run the next tile's blob (bulk copy, mbarrier) and
// X_J rows (registers) one tile ahead, across run boundaries, so one
// __syncthreads per tile remains. Per run X_I is staged once and Y_I
// accumulates in shared memory. Warps 0-3 run pass R (Y_I += A X_J: lane =
// row rank, all nb columns in registers), warps 4-7 pass C (Y_J += A^T X_I:
// lane = column rank, flushed with red.global.add.v4.f32). X rows live in
// 128-byte smem lines holding 128 / (nb * 4) replicas; lane L reads its
// 16-byte chunks in the rotated order (i + L) % CH from replica (L / CH) %
// REP, so the 8 lanes of every quarter-warp phase hit 8 distinct bank groups
// whatever rows they gather. Row ranks are assigned so that lanes L and L + 4
// of a quarter-warp own rows of opposite parity where lengths allow, which
// makes the Y_I read-modify-write conflict-free too (64-byte rows at nb = 16).
//
// Runs are ordered by L2 column band (about 64 MB of f32 X_J and Y_J rows per
// band), so the gathered X_J rows and the reduced Y_J rows of one band stay
// L2-resident while every tile-row that touches the band streams past.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <future>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>

#include <nvtx3/nvToolsExt.h>

#include "comm.hpp"
#include "device.hpp"
#include "hostcopy.hpp"
#include "host_csb.hpp"
#include "stream.cuh"

namespace be {

namespace {

constexpr int kThreads = 256;
constexpr index_t kRunMax = 32;  // tiles per work item

// blob layout (bytes)
constexpr int kMetaJr = 0, kMetaJc = 272, kMetaRperm = 544, kMetaCperm = 672, kMetaRlen = 800, kMetaClen = 928;
constexpr int kMetaSeg = 1056;  // u16[9]: the work split of k_sym_spmm_ws (see there)
constexpr int kMetaBytes = kBlobMeta;
static_assert(kMetaSeg + 18 <= kMetaBytes, "blob meta layout");
__host__ __device__ constexpr int pad16(int n) { return (n + 15) & ~15; }
template <typename TV>
__host__ __device__ constexpr std::size_t blob_bytes(int nnz) {
    return kMetaBytes + static_cast<std::size_t>(pad16(nnz)) * (2 * sizeof(TV) + 2);
}

template <typename TC>
struct Vec;
template <>
struct Vec<float> {
    using T = float4;
    static constexpr int N = 4;
};
template <>
struct Vec<double> {
    using T = double2;
    static constexpr int N = 2;
};

__device__ __forceinline__ void vfma(float4& a, float s, const float4& x) {
    a.x = fmaf(s, x.x, a.x);
    a.y = fmaf(s, x.y, a.y);
    a.z = fmaf(s, x.z, a.z);
    a.w = fmaf(s, x.w, a.w);
}
__device__ __forceinline__ void vfma(double2& a, double s, const double2& x) {
    a.x = fma(s, x.x, a.x);
    a.y = fma(s, x.y, a.y);
}
__device__ __forceinline__ void vzero(float4& a) { a = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void vzero(double2& a) { a = make_double2(0.0, 0.0); }
__device__ __forceinline__ void vadd(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}
__device__ __forceinline__ void vadd(double2& a, const double2& b) {
    a.x += b.x;
    a.y += b.y;
}
__device__ __forceinline__ bool vnonzero(const float4& a) { return a.x != 0.f || a.y != 0.f || a.z != 0.f || a.w != 0.f; }
__device__ __forceinline__ bool vnonzero(const double2& a) { return a.x != 0.0 || a.y != 0.0; }

// Fire-and-forget global reductions (REDG, no return value).
__device__ __forceinline__ void red_add(float* p, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_add4(float* p, const float4& v) {  // REDG.E.ADD.F32x4
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// Flush one 16-byte chunk (columns c0 .. c0+VEC-1 of a row) into Y.
template <typename TX>
__device__ __forceinline__ void flush(TX* y, const float4& a, int lim, bool vec_ok) {
    if constexpr (sizeof(TX) == 4) {
        if (lim >= 4 && vec_ok) {
            red_add4(y, a);
        } else {
            if (lim > 0) red_add(y + 0, a.x);
            if (lim > 1) red_add(y + 1, a.y);
            if (lim > 2) red_add(y + 2, a.z);
            if (lim > 3) red_add(y + 3, a.w);
        }
    } else {
        if (lim > 0) red_add(y + 0, static_cast<double>(a.x));
        if (lim > 1) red_add(y + 1, static_cast<double>(a.y));
        if (lim > 2) red_add(y + 2, static_cast<double>(a.z));
        if (lim > 3) red_add(y + 3, static_cast<double>(a.w));
    }
}
template <typename TX>
__device__ __forceinline__ void flush(TX* y, const double2& a, int lim, bool) {
    if (lim > 0) red_add(y + 0, static_cast<TX>(a.x));
    if (lim > 1) red_add(y + 1, static_cast<TX>(a.y));
}

// smem x-panel geometry for NBP padded columns of TC
template <int NBP, typename TC>
struct XGeom {
    static constexpr int VEC = Vec<TC>::N;                          // elements per 16-byte chunk
    static constexpr int CH = NBP / VEC;                            // chunks per row
    static constexpr int RB = NBP * static_cast<int>(sizeof(TC));  // row bytes
    static constexpr int LINEB = RB < 128 ? 128 : RB;               // bytes per smem row line
    static constexpr int REP = LINEB / RB;                          // replicas per line
    static_assert(NBP % VEC == 0 && CH >= 1, "bad NBP");
};

// Stage rows [row0, row0 + nr) of X (TX, row-major, nb columns) into the
// replicated smem lines; all loads of a batch are in flight together.
template <int NBP, typename TC, typename TX>
__device__ __forceinline__ void stage_x(unsigned char* xs, const TX* __restrict__ X, int row0, int nr, int nb, int ld) {
    using G = XGeom<NBP, TC>;
    const TX* src = X + static_cast<std::int64_t>(row0) * ld;
    constexpr int EPC = 16 / sizeof(TX);  // TX elements per 16-byte chunk
    if constexpr ((NBP * sizeof(TX)) % 16 == 0) {
        if (nb == NBP && ld == NBP) {
            constexpr int CPR = NBP / EPC;  // global chunks per row
            const int total = nr * CPR;
            constexpr int PER = 4;
            for (int c0 = threadIdx.x; c0 < total; c0 += PER * kThreads) {
                uint4 buf[PER];
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int c = c0 + i * kThreads;
                    if (c < total) buf[i] = __ldg(reinterpret_cast<const uint4*>(src) + c);
                }
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int c = c0 + i * kThreads;
                    if (c < total) {
                        const int r = c / CPR, v0 = (c % CPR) * EPC;
                        TC* line = reinterpret_cast<TC*>(xs + r * G::LINEB);
                        if constexpr (sizeof(TC) == sizeof(TX)) {  // 16-byte stores (one wavefront per 8 lanes)
                            // replica order rotated by row: neighbouring rows of a phase hit different banks
#pragma unroll
                            for (int q = 0; q < G::REP; ++q)
                                *reinterpret_cast<uint4*>(line + ((q + r) % G::REP) * NBP + v0) = buf[i];
                        } else {
                            const TX* e = reinterpret_cast<const TX*>(&buf[i]);
#pragma unroll
                            for (int q = 0; q < G::REP; ++q)
#pragma unroll
                                for (int j = 0; j < EPC; ++j) line[((q + r) % G::REP) * NBP + v0 + j] = static_cast<TC>(e[j]);
                        }
                    }
                }
            }
            return;
        }
    }
    const int total = nr * NBP;
    for (int e = threadIdx.x; e < total; e += kThreads) {
        const int r = e / NBP, v = e - r * NBP;
        const TC x = v < nb ? static_cast<TC>(__ldg(src + static_cast<std::int64_t>(r) * ld + v)) : TC(0);
        TC* line = reinterpret_cast<TC*>(xs + r * G::LINEB);
#pragma unroll
        for (int q = 0; q < G::REP; ++q) line[q * NBP + v] = x;
    }
}

// X_J rows of the next tile, held in registers while the current tile is
// computed (fast path: TX == TC, nb == NBP, 16-byte aligned X).
template <int NBP, typename TC>
struct XPre {
    static constexpr int CPR = NBP * static_cast<int>(sizeof(TC)) / 16;
    static constexpr int PER = (kTile * CPR + kThreads - 1) / kThreads;
    uint4 v[PER];
    __device__ __forceinline__ void load(const TC* __restrict__ X, int row0, int nr) {
        const uint4* src = reinterpret_cast<const uint4*>(X + static_cast<std::int64_t>(row0) * NBP);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int c = threadIdx.x + i * kThreads;
            if (c < nr * CPR) v[i] = __ldg(src + c);
        }
    }
    __device__ __forceinline__ void store(unsigned char* xs, int nr) const {
        using G = XGeom<NBP, TC>;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int c = threadIdx.x + i * kThreads;
            if (c < nr * CPR) {
                const int r = c / CPR, v0 = (c % CPR) * (16 / static_cast<int>(sizeof(TC)));
                TC* line = reinterpret_cast<TC*>(xs + r * G::LINEB);
#pragma unroll
                for (int q = 0; q < G::REP; ++q) *reinterpret_cast<uint4*>(line + ((q + r) % G::REP) * NBP + v0) = v[i];
            }
        }
    }
};

// One pass of one tile: lane = rank (row rank for pass R, column rank for
// pass C); walks diagonals [d_begin, len) of its jagged row (column) through
// the JDS starts, gathering the matching X line of the other side for every
// entry. Full groups of U entries are branch-free, so the U index / value
// reads and the U x CH gathers of a group are all in flight together.
template <int NBP, typename TC, typename TV>
__device__ __forceinline__ void jds_walk(const std::uint16_t* __restrict__ jd, int d_begin, int len, int rank,
                                         const TV* __restrict__ sv, const unsigned char* __restrict__ sidx,
                                         const unsigned char* __restrict__ xbase, const int* coff,
                                         typename Vec<TC>::T* acc) {
    using G = XGeom<NBP, TC>;
    using V = typename Vec<TC>::T;
    constexpr int U = G::CH <= 4 ? 4 : (G::CH <= 8 ? 2 : 1);
    int d = d_begin;  // a multiple of 4: the starts of a group are one broadcast 8-byte read
    for (; d + U <= len; d += U) {
        int pos[U];
        if constexpr (U == 4) {
            const uint2 q = *reinterpret_cast<const uint2*>(jd + d);
            pos[0] = static_cast<int>(q.x & 0xffffu) + rank;
            pos[1] = static_cast<int>(q.x >> 16) + rank;
            pos[2] = static_cast<int>(q.y & 0xffffu) + rank;
            pos[3] = static_cast<int>(q.y >> 16) + rank;
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) pos[u] = static_cast<int>(jd[d + u]) + rank;
        }
        TC v[U];
        const unsigned char* p[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u] = static_cast<TC>(sv[pos[u]]);
            p[u] = xbase + static_cast<int>(sidx[pos[u]]) * G::LINEB;
        }
        V xv[U][G::CH];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < G::CH; ++i) xv[u][i] = *reinterpret_cast<const V*>(p[u] + coff[i]);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < G::CH; ++i) vfma(acc[i], v[u], xv[u][i]);
    }
    for (; d < len; ++d) {
        const int pos = static_cast<int>(jd[d]) + rank;
        const TC v = static_cast<TC>(sv[pos]);
        const unsigned char* p = xbase + static_cast<int>(sidx[pos]) * G::LINEB;
        V xv[G::CH];
#pragma unroll
        for (int i = 0; i < G::CH; ++i) xv[i] = *reinterpret_cast<const V*>(p + coff[i]);
#pragma unroll
        for (int i = 0; i < G::CH; ++i) vfma(acc[i], v, xv[i]);
    }
}

__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Tail split (load balance inside a pass): ranks are sorted by decreasing
// length, so the first warp of a pass owns the longest rows (columns). Its
// diagonals [D, len) -- D stored at jd[130] -- go to the last warp of the pass,
// which runs them after its own ranks and hands the partial sums over through
// shared memory (named barrier 1 for pass R, 2 for pass C).
constexpr int kSplitSlot = 130;

template <int NBP, typename TC, typename TV, typename TX>
__global__ void __launch_bounds__(kThreads, 2)
    k_sym_spmm(const int2* __restrict__ runs, int nruns, const TileHdr* __restrict__ tiles,
               const unsigned char* __restrict__ blobs, const TX* __restrict__ X, TX* __restrict__ Y, int nb, int ld,
               int do_r, int do_c, int blob_max, int* __restrict__ ctr) {
    using G = XGeom<NBP, TC>;
    using V = typename Vec<TC>::T;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* xi = smem;                              // X_I lines of the current run
    unsigned char* xjb = xi + kTile * G::LINEB;            // X_J lines, two buffers
    V* yi = reinterpret_cast<V*>(xjb + 2 * kTile * G::LINEB);  // kTile x CH chunks: the run's Y_I rows
    V* tail = yi + kTile * G::CH;                          // 2 x 32 x CH: tail-split partial sums
    unsigned char* stg = reinterpret_cast<unsigned char*>(tail + 2 * 32 * G::CH);  // two blob buffers
    __shared__ __align__(8) std::uint64_t bars[2];
    __shared__ TileHdr s_hdr[2][kRunMax];  // headers of the current and the next run
    __shared__ int2 s_rg[2];               // their tile ranges (x >= y: no run)
    __shared__ int s_pend;                 // id of the run after next (its headers are fetched during this run)

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int grp = tid >> 7;  // 0: pass R (row ranks), 1: pass C (column ranks)
    const int rank = tid & 127;
    const int wq = warp & 3;   // warp of the pass
    const bool vec_ok = (nb % G::VEC) == 0 && (ld % G::VEC) == 0 && (reinterpret_cast<std::uintptr_t>(Y) & 15u) == 0;
    const bool fast_x = sizeof(TC) == sizeof(TX) && nb == NBP && ld == NBP && (NBP * sizeof(TX)) % 16 == 0 &&
                        (reinterpret_cast<std::uintptr_t>(X) & 15u) == 0;
    const unsigned char* xrep = ((lane / G::CH) % G::REP) * G::RB + (grp == 0 ? xjb : xi);
    const unsigned char* xrep_c = ((lane / G::CH) % G::REP) * G::RB + xi;
    int coff[G::CH];
#pragma unroll
    for (int i = 0; i < G::CH; ++i) coff[i] = ((i + lane) % G::CH) * 16;
    std::uint64_t policy;  // the blob stream is read once: keep the X / Y bands in L2 instead
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

    // a run's range and headers (warp 0): load into registers, store into the cache later
    auto fetch_run = [&](int id, int2& rg, TileHdr& hd) {
        rg = id < nruns ? runs[id] : make_int2(0, 0);
        if (lane < rg.y - rg.x) hd = tiles[rg.x + lane];
    };
    auto store_run = [&](int slot, const int2& rg, const TileHdr& hd) {
        if (lane == 0) s_rg[slot] = rg;
        if (lane < rg.y - rg.x) s_hdr[slot][lane] = hd;
    };
    if (warp == 0) {
        int id0 = 0, id1 = 0, id2 = 0;
        if (lane == 0) {
            stream::mbar_init(&bars[0], 1);
            stream::mbar_init(&bars[1], 1);
            stream::mbar_init_fence();
            id0 = atomicAdd(ctr, 1);
            id1 = id0 < nruns ? atomicAdd(ctr, 1) : nruns;
            id2 = id1 < nruns ? atomicAdd(ctr, 1) : nruns;
            s_pend = id2;
        }
        id0 = __shfl_sync(0xffffffffu, id0, 0);
        id1 = __shfl_sync(0xffffffffu, id1, 0);
        int2 r0, r1;
        TileHdr h0, h1;
        fetch_run(id0, r0, h0);
        fetch_run(id1, r1, h1);
        store_run(0, r0, h0);
        store_run(1, r1, h1);
    }
    __syncthreads();
    int cur = 0;  // run-cache slot of the current run
    int2 rg = s_rg[0];
    if (rg.x < rg.y) {
        int t = rg.x;
        auto issue = [&](const TileHdr& hh, int slot) {  // one thread: the blob of a tile -> stage slot
            const std::uint32_t bytes = static_cast<std::uint32_t>(blob_bytes<TV>(static_cast<int>(hh.packed >> 14)));
            stream::fence_proxy_async();
            stream::mbar_arrive_expect_tx(&bars[slot], bytes);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                    stream::smem_u32(stg + slot * blob_max)),
                "l"(blobs + static_cast<std::size_t>(hh.begin16) * 16), "r"(bytes), "r"(stream::smem_u32(&bars[slot])),
                "l"(policy)
                : "memory");
        };
        {  // first tile of the first run: synchronous staging
            const TileHdr h0 = s_hdr[0][0];
            if (tid == 0) issue(h0, 0);
            if (do_r) stage_x<NBP, TC, TX>(xjb, X, h0.col0, static_cast<int>((h0.packed >> 7) & 127u) + 1, nb, ld);
            if (do_c) stage_x<NBP, TC, TX>(xi, X, h0.row0, static_cast<int>(h0.packed & 127u) + 1, nb, ld);
            if (do_r)
                for (int e = tid; e < kTile * G::CH; e += kThreads) vzero(yi[e]);
        }
        std::uint32_t phase = 0;  // bit s: parity of stage s's next completion
        int s = 0;
        int2 prg = make_int2(0, 0);  // warp 0: the run after next, fetched during this run
        TileHdr phd{};
        bool run_start = true;
        for (;;) {
            stream::mbar_wait(&bars[s], (phase >> s) & 1u);
            phase ^= 1u << s;
            __syncthreads();  // blob t, X_J(t), X_I, Y_I, run cache visible; stage s^1 and X_J buffer s^1 free
            if (run_start && warp == 0) fetch_run(s_pend, prg, phd);
            run_start = false;
            const TileHdr h = s_hdr[cur][t - rg.x];
            int tn = -1;
            TileHdr hn{};
            if (t + 1 < rg.y) {
                tn = t + 1;
                hn = s_hdr[cur][t + 1 - rg.x];
            } else if (s_rg[cur ^ 1].x < s_rg[cur ^ 1].y) {
                tn = s_rg[cur ^ 1].x;
                hn = s_hdr[cur ^ 1][0];
            }
            XPre<NBP, TC> pre, prei;
            const bool run_end = t == rg.y - 1;
            if (tn >= 0) {
                if (tid == 0) issue(hn, s ^ 1);
                if (do_r && fast_x)
                    pre.load(reinterpret_cast<const TC*>(X), hn.col0, static_cast<int>((hn.packed >> 7) & 127u) + 1);
                if (run_end && do_c && fast_x)  // the next run's X_I, stored after the end-of-run barrier
                    prei.load(reinterpret_cast<const TC*>(X), hn.row0, static_cast<int>(hn.packed & 127u) + 1);
            }
            // ---- compute tile t
            {
                const unsigned char* st = stg + s * blob_max;
                const int npad = pad16(static_cast<int>(h.packed >> 14));
                if (grp == 0 ? do_r : do_c) {
                    const std::uint16_t* jd = reinterpret_cast<const std::uint16_t*>(st + (grp == 0 ? kMetaJr : kMetaJc));
                    const unsigned char* lens = st + (grp == 0 ? kMetaRlen : kMetaClen);
                    const TV* sv = reinterpret_cast<const TV*>(st + kMetaBytes + (grp == 0 ? 0 : npad * (static_cast<int>(sizeof(TV)) + 1)));
                    const unsigned char* sx = st + kMetaBytes + npad * (grp == 0 ? static_cast<int>(sizeof(TV)) : 2 * static_cast<int>(sizeof(TV)) + 1);
                    const unsigned char* xb = grp == 0 ? xrep + s * kTile * G::LINEB : xrep_c;
                    const int split = jd[kSplitSlot];                  // tail of warp 0's ranks: diagonals [split, len)
                    const bool has_tail = split < lens[0];
                    const int len = lens[rank];
                    V acc[G::CH];
#pragma unroll
                    for (int i = 0; i < G::CH; ++i) vzero(acc[i]);
                    jds_walk<NBP, TC, TV>(jd, 0, wq == 0 ? min(len, split) : len, rank, sv, sx, xb, coff, acc);
                    auto out = [&](int rk, V* a) {  // Y_I += A X_J (row rk) / Y_J += A^T X_I (column rk)
                        if (grp == 0) {
                            V* y = yi + static_cast<int>(st[kMetaRperm + rk]) * G::CH;
#pragma unroll
                            for (int i = 0; i < G::CH; ++i) vadd(y[(i + lane) % G::CH], a[i]);
                        } else {
                            TX* y = Y + static_cast<std::int64_t>(h.col0 + st[kMetaCperm + rk]) * ld;
#pragma unroll
                            for (int i = 0; i < G::CH; ++i) {
                                const int c0 = ((i + lane) % G::CH) * G::VEC;
                                if (c0 < nb) flush<TX>(y + c0, a[i], nb - c0, vec_ok);
                            }
                        }
                    };
                    V* tl = tail + (grp * 32 + lane) * G::CH;
                    if (wq == 3) {
                        if (len > 0) out(rank, acc);
                        if (has_tail) {  // the tail of ranks 0..31, handed to warp 0 of the pass
                            const int l0 = lens[lane];
#pragma unroll
                            for (int i = 0; i < G::CH; ++i) vzero(acc[i]);
                            jds_walk<NBP, TC, TV>(jd, split, l0, lane, sv, sx, xb, coff, acc);
#pragma unroll
                            for (int i = 0; i < G::CH; ++i) tl[(i + lane) % G::CH] = acc[i];  // rotated: conflict-free
                            __threadfence_block();
                            named_bar_arrive(1 + grp, 64);
                        }
                    } else {
                        if (wq == 0 && has_tail) {
                            named_bar_sync(1 + grp, 64);
#pragma unroll
                            for (int i = 0; i < G::CH; ++i) vadd(acc[i], tl[(i + lane) % G::CH]);
                        }
                        if (len > 0) out(rank, acc);
                    }
                }
            }
            if (tn >= 0 && do_r) {  // X_J of the next tile into the other buffer
                unsigned char* xn = xjb + (s ^ 1) * kTile * G::LINEB;
                const int ncn = static_cast<int>((hn.packed >> 7) & 127u) + 1;
                if (fast_x) pre.store(xn, ncn);
                else stage_x<NBP, TC, TX>(xn, X, hn.col0, ncn, nb, ld);
            }
            if (run_end) {  // end of the run: flush Y_I, stage the next run's X_I, refill the run cache
                __syncthreads();
                if (do_r) {
                    const int nr = static_cast<int>(h.packed & 127u) + 1;
                    for (int e = tid; e < nr * G::CH; e += kThreads) {
                        const int row = e / G::CH, c0 = (e % G::CH) * G::VEC;
                        if (c0 < nb && vnonzero(yi[e]))
                            flush<TX>(Y + static_cast<std::int64_t>(h.row0 + row) * ld + c0, yi[e], nb - c0, vec_ok);
                        vzero(yi[e]);
                    }
                }
                if (tn >= 0) {
                    if (do_c) {
                        if (fast_x) prei.store(xi, static_cast<int>(hn.packed & 127u) + 1);
                        else stage_x<NBP, TC, TX>(xi, X, hn.row0, static_cast<int>(hn.packed & 127u) + 1, nb, ld);
                    }
                    if (warp == 0) {
                        store_run(cur, prg, phd);  // the run after next replaces the finished one
                        if (lane == 0) s_pend = s_pend < nruns ? atomicAdd(ctr, 1) : nruns;
                    }
                }
                cur ^= 1;
                rg = s_rg[cur];  // (unchanged by the store above: that went to the other slot)
                run_start = true;
            }
            if (tn < 0) break;
            t = tn;
            s ^= 1;
        }
    }
    // last CTA out resets the counter for the next launch
    if (tid == 0) {
        __threadfence();
        const int done = atomicAdd(ctr + 1, 1);
        if (done == static_cast<int>(gridDim.x) - 1) {
            ctr[0] = 0;
            ctr[1] = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// k_sym_spmm_ws: the warp-specialised form of the same tile kernel (f32
// values and panels, nb = 8, 16 or 32, the headline configuration). One CTA
// per SM: a producer warp streams each tile's blob, its X_J rows and its X_I
// rows into a ring of kWsStages shared-memory stages with 1-D bulk copies
// (cp.async.bulk, completion on a per-stage "full" mbarrier); eight consumer
// warps each run one unit of the tile's work -- a pass (R: Y_I += A X_J,
// C: Y_J += A^T X_I) over one group of 32 rank lanes -- warp w taking unit
// (w + tile) mod 8, so over eight tiles every warp runs every unit once; they
// flush each row with red.global.add.v4.f32 and release the stage on a
// per-stage "empty" mbarrier. No CTA-wide barrier: a warp that finishes its
// unit early starts on the next tile (up to kWsStages - 1 tiles ahead), so the
// per-tile imbalance between units (the longest rank group carries ~2x the
// entries of the shortest) averages out instead of idling the shared-memory
// crossbar, and no rank is split between warps (one flush per rank and pass;
// the blob's equal-entry work split, BE_SPMM_WS_ROT=0, costs ~20 % more in
// split-rank flushes). The staged X rows are REP = 128 / (4 nb) plain
// copies, copy q placed at q * 129 rows so that row r of copy q sits in the
// 128-byte bank line slot (q + r) mod REP: lane L reads the copy that puts its
// row in slot (L / CH) mod REP, so a quarter-warp's eight 16-byte reads are
// conflict-free whatever rows it gathers (the replica scheme of k_sym_spmm
// without the per-tile register staging).
// ---------------------------------------------------------------------------
constexpr int kWsThreads = 288;  // 8 consumer warps + 1 producer warp
constexpr std::uint32_t kWsEnd = 0xFFFFFFFFu;

template <int NBP, typename T = float>
struct WsGeom {
    static constexpr int RB = NBP * static_cast<int>(sizeof(T));  // bytes per X row
    static constexpr int REP = RB >= 128 ? 1 : 128 / RB;            // shifted copies per staged panel
    static constexpr int CH = RB / 16;                              // 16-byte chunks per row
    static constexpr int EPC = 16 / static_cast<int>(sizeof(T));    // elements per chunk
    static constexpr int COPY = (kTile + 1) * RB;                   // bytes per copy (one row of shift)
    static constexpr int XREG = REP * COPY;                         // one staged panel
    static_assert(REP >= 1 && (REP & (REP - 1)) == 0 && RB % 16 == 0, "nb must be 8, 16 or 32");
};

__device__ __forceinline__ void red_vec(float* y, const float4& a) { red_add4(y, a); }
__device__ __forceinline__ void red_vec(double* y, const double2& a) {
    red_add(y, a.x);
    red_add(y + 1, a.y);
}

template <int NBP, typename T>
__device__ __forceinline__ void ws_walk(const std::uint16_t* __restrict__ jd, int d, int hi, int rank,
                                        const T* __restrict__ sv, const unsigned char* __restrict__ sidx,
                                        const unsigned char* __restrict__ xreg, int slot, const int* coff,
                                        typename Vec<T>::T* acc) {
    using G = WsGeom<NBP, T>;
    using V = typename Vec<T>::T;
    constexpr int U = G::CH <= 4 ? 4 : 2;
    auto row_ptr = [&](int idx) {  // 16-byte aligned by construction (stage, COPY and RB are multiples of 16)
        return static_cast<const unsigned char*>(
            __builtin_assume_aligned(xreg + ((slot - idx) & (G::REP - 1)) * G::COPY + idx * G::RB, 16));
    };
    for (; d + U <= hi; d += U) {
        int pos[U];
        if constexpr (U == 4) {
            const uint2 q = *reinterpret_cast<const uint2*>(jd + d);
            pos[0] = static_cast<int>(q.x & 0xffffu) + rank;
            pos[1] = static_cast<int>(q.x >> 16) + rank;
            pos[2] = static_cast<int>(q.y & 0xffffu) + rank;
            pos[3] = static_cast<int>(q.y >> 16) + rank;
        } else {
            const std::uint32_t q = *reinterpret_cast<const std::uint32_t*>(jd + d);
            pos[0] = static_cast<int>(q & 0xffffu) + rank;
            pos[1] = static_cast<int>(q >> 16) + rank;
        }
        T v[U];
        const unsigned char* p[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            v[k] = sv[pos[k]];
            p[k] = row_ptr(static_cast<int>(sidx[pos[k]]));
        }
        V xv[U][G::CH];
#pragma unroll
        for (int k = 0; k < U; ++k)
#pragma unroll
            for (int i = 0; i < G::CH; ++i)
                xv[k][i] = *static_cast<const V*>(__builtin_assume_aligned(p[k] + coff[i], 16));
#pragma unroll
        for (int k = 0; k < U; ++k)
#pragma unroll
            for (int i = 0; i < G::CH; ++i) vfma(acc[i], v[k], xv[k][i]);
    }
    for (; d < hi; ++d) {
        const int pos = static_cast<int>(jd[d]) + rank;
        const T v = sv[pos];
        const unsigned char* p = row_ptr(static_cast<int>(sidx[pos]));
        V xv[G::CH];
#pragma unroll
        for (int i = 0; i < G::CH; ++i) xv[i] = *static_cast<const V*>(__builtin_assume_aligned(p + coff[i], 16));
#pragma unroll
        for (int i = 0; i < G::CH; ++i) vfma(acc[i], v, xv[i]);
    }
}

template <int NBP, int kWsStages, typename T = float>
__global__ void __launch_bounds__(kWsThreads, kWsStages <= 2 ? 2 : 1)
    k_sym_spmm_ws(const int2* __restrict__ runs, int nruns, const TileHdr* __restrict__ tiles,
                  const unsigned char* __restrict__ blobs, const T* __restrict__ X, T* __restrict__ Y,
                  int do_r, int do_c, int blob_max, int stage_bytes, int rot, int* __restrict__ ctr) {
    using G = WsGeom<NBP, T>;
    using V = typename Vec<T>::T;
    constexpr int TS = static_cast<int>(sizeof(T));
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) std::uint64_t full[kWsStages], empty[kWsStages], xfull[2], xempty[2];
    __shared__ TileHdr shdr[kWsStages];
    __shared__ int sflag[kWsStages];  // bit 0: first tile of its run, bit 1: last, bit 2: X_I slot
    unsigned char* xis = smem + static_cast<std::size_t>(kWsStages) * stage_bytes;  // two X_I slots (per run)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < kWsStages; ++s) {
            stream::mbar_init(&full[s], 1);
            stream::mbar_init(&empty[s], 8);
        }
        for (int q = 0; q < 2; ++q) {
            stream::mbar_init(&xfull[q], 1);
            stream::mbar_init(&xempty[q], 8);
        }
        stream::mbar_init_fence();
    }
    __syncthreads();
    if (warp == 8) {  // ---------------- producer
        std::uint64_t policy;  // the blob stream is read once: keep the X / Y bands in L2 instead
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
        int s = 0, nrun = 0;
        std::uint32_t eph = (1u << kWsStages) - 1;  // fresh barriers: the "previous" phase counts as complete
        std::uint32_t xeph = 3u;
        for (;;) {
            int id = 0;
            if (lane == 0) id = atomicAdd(ctr, 1);
            id = __shfl_sync(0xffffffffu, id, 0);
            if (id >= nruns) break;
            const int2 rg = runs[id];
            const int cnt = rg.y - rg.x;
            TileHdr hd{};
            if (lane < cnt) hd = tiles[rg.x + lane];
            const int xs = nrun++ & 1;
            if (do_c && lane == 0) {  // the run's X_I rows, once per run
                const std::uint32_t p0 = __shfl_sync(1u, hd.packed, 0);
                const int r0 = __shfl_sync(1u, hd.row0, 0);
                const int nr = static_cast<int>(p0 & 127u) + 1;
                stream::mbar_wait_parked(&xempty[xs], (xeph >> xs) & 1u);
                xeph ^= 1u << xs;
                stream::mbar_arrive_expect_tx(&xfull[xs], static_cast<std::uint32_t>(G::REP * nr * G::RB));
#pragma unroll
                for (int q = 0; q < G::REP; ++q)
                    stream::bulk_g2s(xis + xs * G::XREG + q * G::COPY, X + static_cast<std::int64_t>(r0) * NBP,
                                     static_cast<std::uint32_t>(nr * G::RB), &xfull[xs]);
            }
            for (int i = 0; i < cnt; ++i) {
                TileHdr h;
                h.begin16 = __shfl_sync(0xffffffffu, hd.begin16, i);
                h.row0 = __shfl_sync(0xffffffffu, hd.row0, i);
                h.col0 = __shfl_sync(0xffffffffu, hd.col0, i);
                h.packed = __shfl_sync(0xffffffffu, hd.packed, i);
                if (lane == 0) {
                    stream::mbar_wait_parked(&empty[s], (eph >> s) & 1u);
                    eph ^= 1u << s;
                    shdr[s] = h;
                    sflag[s] = (i == 0 ? 1 : 0) | (i == cnt - 1 ? 2 : 0) | (xs << 2);
                    const int nnz = static_cast<int>(h.packed >> 14);
                    const int nr = static_cast<int>(h.packed & 127u) + 1, nc = static_cast<int>((h.packed >> 7) & 127u) + 1;
                    const std::uint32_t bb = static_cast<std::uint32_t>(blob_bytes<T>(nnz));
                    const std::uint32_t bytes = bb + (do_r ? G::REP * nc * G::RB : 0);
                    unsigned char* st = smem + static_cast<std::size_t>(s) * stage_bytes;
                    stream::mbar_arrive_expect_tx(&full[s], bytes);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                            stream::smem_u32(st)),
                        "l"(blobs + static_cast<std::size_t>(h.begin16) * 16), "r"(bb), "r"(stream::smem_u32(&full[s])),
                        "l"(policy)
                        : "memory");
                    if (do_r)
#pragma unroll
                        for (int q = 0; q < G::REP; ++q)
                            stream::bulk_g2s(st + blob_max + q * G::COPY, X + static_cast<std::int64_t>(h.col0) * NBP,
                                             static_cast<std::uint32_t>(nc * G::RB), &full[s]);
                }
                s = s + 1 == kWsStages ? 0 : s + 1;
            }
        }
        if (lane == 0) {  // end of stream; then the last producer out resets the counter
            stream::mbar_wait_parked(&empty[s], (eph >> s) & 1u);
            shdr[s].packed = kWsEnd;
            stream::mbar_arrive_expect_tx(&full[s], 0);
            __threadfence();
            const int done = atomicAdd(ctr + 1, 1);
            if (done == static_cast<int>(gridDim.x) - 1) {
                ctr[0] = 0;
                ctr[1] = 0;
            }
        }
        return;
    }
    // ---------------- consumers (warps 0..7)
    int coff[G::CH];
#pragma unroll
    for (int i = 0; i < G::CH; ++i) coff[i] = ((i + lane) % G::CH) * 16;
    const int slot = (lane / G::CH) % G::REP;
    int s = 0, tcount = 0;
    std::uint32_t fph = 0, xph = 0;
    for (;;) {
        stream::mbar_wait_parked(&full[s], (fph >> s) & 1u);
        fph ^= 1u << s;
        const TileHdr h = shdr[s];
        if (h.packed == kWsEnd) break;
        const int fl = sflag[s], xs = (fl >> 2) & 1;
        if (do_c && (fl & 1)) {
            stream::mbar_wait_parked(&xfull[xs], (xph >> xs) & 1u);
            xph ^= 1u << xs;
        }
        const unsigned char* st = smem + static_cast<std::size_t>(s) * stage_bytes;
        const int npad = pad16(static_cast<int>(h.packed >> 14));
        const std::uint16_t* seg = reinterpret_cast<const std::uint16_t*>(st + kMetaSeg);
        int b0, b1;
        if (rot) {  // whole units, rotated by tile, no split ranks: warp w runs unit kRotSeq[(w + tile) mod 8]
            // -- the sequence alternates heavy and light rank groups (R0, C3, R1, C2, R2, C1, R3, C0), so
            // a warp never meets two long-row units in a row and its lead / lag stays within the ring
            constexpr unsigned kRotSeq = 0x43526170u;  // nibbles, lowest first: 0 7 1 6 2 5 3 4
            const int un0 = static_cast<int>((kRotSeq >> (4 * ((warp + tcount) & 7))) & 15u);
            b0 = un0 << 8;
            b1 = (un0 + 1) << 8;
        } else {  // the blob's equal-entry pieces
            b0 = seg[warp];
            b1 = seg[warp + 1];
        }
        ++tcount;
        int un = b0 >> 8, d = b0 & 255;
        const int ue = b1 >> 8, de = b1 & 255;
        while (un < ue || (un == ue && d < de)) {
            const int pass = un >> 2, g = un & 3;
            if (pass == 0 ? do_r : do_c) {
                const int dend = un == ue ? de : 255;
                const std::uint16_t* jd = reinterpret_cast<const std::uint16_t*>(st + (pass == 0 ? kMetaJr : kMetaJc));
                const int rank = 32 * g + lane;
                const int len = st[(pass == 0 ? kMetaRlen : kMetaClen) + rank];
                const int hi = min(dend, len);
                if (d < hi) {
                    const T* sv = reinterpret_cast<const T*>(st + kMetaBytes + (pass == 0 ? 0 : npad * (TS + 1)));
                    const unsigned char* sx = st + kMetaBytes + npad * (pass == 0 ? TS : 2 * TS + 1);
                    const unsigned char* xreg = pass == 0 ? st + blob_max : xis + xs * G::XREG;
                    V acc[G::CH];
#pragma unroll
                    for (int i = 0; i < G::CH; ++i) vzero(acc[i]);
                    ws_walk<NBP, T>(jd, d, hi, rank, sv, sx, xreg, slot, coff, acc);
                    const int row = pass == 0 ? h.row0 + st[kMetaRperm + rank] : h.col0 + st[kMetaCperm + rank];
                    T* y = Y + static_cast<std::int64_t>(row) * NBP;
#pragma unroll
                    for (int i = 0; i < G::CH; ++i) red_vec(y + ((i + lane) % G::CH) * G::EPC, acc[i]);
                }
            }
            ++un;
            d = 0;
        }
        // this warp's generic-proxy reads of the stage before the producer's next bulk (async-proxy) writes
        stream::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(stream::smem_u32(&empty[s])) : "memory");
            if (do_c && (fl & 2))
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(stream::smem_u32(&xempty[xs])) : "memory");
        }
        s = s + 1 == kWsStages ? 0 : s + 1;
    }
}

template <int NBP, int S, typename T = float>
bool launch_ws_s(Op* op, const int2* runs, index_t nruns, const T* X, T* Y, int do_r, int do_c, cudaStream_t s) {
    using G = WsGeom<NBP, T>;
    const int stage = ((op->blob_max + G::XREG) + 127) & ~127;
    const std::size_t sm = static_cast<std::size_t>(stage) * S + 2 * G::XREG;
    int dev = 0, optin = 0;
    BE_CUDA(cudaGetDevice(&dev));
    BE_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (sm + 1024 > static_cast<std::size_t>(optin)) return false;
    auto kern = k_sym_spmm_ws<NBP, S, T>;
    ensure_dyn_smem(kern, sm);
    int per_sm = 0;
    BE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWsThreads, sm));
    if (per_sm < 1) return false;
    const int grid = static_cast<int>(std::min<index_t>(static_cast<index_t>(per_sm) * op->ctx->num_sms, nruns));
    op->grid = grid;
    if (grid == 0) return true;
    static const int rot = [] {  // whole units rotated by tile (default) or the blob's equal-entry pieces
        const char* e = std::getenv("BE_SPMM_WS_ROT");
        return e ? std::atoi(e) : 1;
    }();
    kern<<<grid, kWsThreads, sm, s>>>(runs, static_cast<int>(nruns), op->tiles.get(), op->blobs.get(), X, Y, do_r, do_c,
                                      op->blob_max, stage, rot, op->counter.get());
    BE_CUDA(cudaGetLastError());
    ++op->ctx->launches;
    return true;
}

// stages per CTA: 2 (two CTAs per SM: 16 consumer warps, measured fastest) or 3 / 4 (one CTA per
// SM); BE_SPMM_WS_STAGES overrides (experiments)
template <int NBP, typename T = float>
bool launch_ws(Op* op, const int2* runs, index_t nruns, const T* X, T* Y, int do_r, int do_c, cudaStream_t s) {
    static const int stages = [] {
        const char* e = std::getenv("BE_SPMM_WS_STAGES");
        return e ? std::atoi(e) : 2;
    }();
    if (stages == 3) return launch_ws_s<NBP, 3, T>(op, runs, nruns, X, Y, do_r, do_c, s);
    if (stages == 4) return launch_ws_s<NBP, 4, T>(op, runs, nruns, X, Y, do_r, do_c, s);
    return launch_ws_s<NBP, 2, T>(op, runs, nruns, X, Y, do_r, do_c, s);
}

// Deterministic symmetric SpMM (BE_OP_DETERMINISTIC): one warp per output
// row, lane = panel column; the row's entries are summed sequentially in the
// reference's serial order (run_baseline, kernels.hpp:253-276 + the diagonal
// pass :363-370) with separately rounded products and sums (the reference's
// u += v * w compiles without FMA), so the result is bit-reproducible and
// bit-identical to the serial reference on f64 panels.
template <typename TX, typename TV = double>
__global__ void k_det_spmm(const std::int64_t* __restrict__ pa, const std::int64_t* __restrict__ pb,
                           const std::int32_t* __restrict__ col, const TV* __restrict__ val,
                           const double* __restrict__ diag, const TX* __restrict__ X, TX* __restrict__ Y,
                           std::int64_t nout, int nb, int init_zero) {
    const int lane = threadIdx.x & 31;
    const std::int64_t w0 = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const std::int64_t nw = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (std::int64_t r = w0; r < nout; r += nw) {
        for (int v = lane; v < nb; v += 32) {
            double y = init_zero ? 0.0 : static_cast<double>(Y[r * nb + v]);
            for (std::int64_t e = pa[r]; e < pa[r + 1]; ++e)
                y = __dadd_rn(y, __dmul_rn(static_cast<double>(val[e]), static_cast<double>(X[static_cast<std::int64_t>(col[e]) * nb + v])));
            if (pb)
                for (std::int64_t e = pb[r]; e < pb[r + 1]; ++e)
                    y = __dadd_rn(y, __dmul_rn(static_cast<double>(val[e]), static_cast<double>(X[static_cast<std::int64_t>(col[e]) * nb + v])));
            if (diag) y = __dadd_rn(y, __dmul_rn(diag[r], static_cast<double>(X[r * nb + v])));
            Y[r * nb + v] = static_cast<TX>(y);
        }
    }
}

// Row-list SpMM for sparse matrices (the BE_OP_FORMAT_ROWS device format):
// output row r = its L entries, then its L^T entries (the same lists as the
// deterministic mode, f32 values), summed by a group of G = NBP / 4 lanes that
// each own 16 bytes of the row; the X rows are gathered straight from L2 (one
// 64-byte line segment per group and entry at nb = 16) -- no shared-memory
// staging, which a 128 x 128 tile holding a few hundred entries cannot
// amortise. The group's lanes load G entries at once and broadcast them with
// shuffles; every output row is written once, no atomics (deterministic).
// init: 0 = Y <- sum, 1 = Y += sum, 2 = Y <- diag X + sum.
template <int NBP>
__global__ void __launch_bounds__(256) k_rows_spmm(const std::int64_t* __restrict__ pa, const std::int64_t* __restrict__ pb,
                                                   const std::int32_t* __restrict__ col, const float* __restrict__ val,
                                                   const double* __restrict__ diag, const float* __restrict__ X,
                                                   float* __restrict__ Y, std::int64_t nout, int init) {
    constexpr int G = NBP / 4, RPW = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane % G;
    const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane - sub);
    const std::int64_t w0 = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const std::int64_t nw = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (std::int64_t rb = w0 * RPW; rb < nout; rb += nw * RPW) {
        const std::int64_t r = rb + lane / G;
        const bool live = r < nout;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (live && init == 1) acc = reinterpret_cast<const float4*>(Y + r * NBP)[sub];
        if (live && init == 2) {
            const float d = static_cast<float>(diag[r]);
            const float4 x = reinterpret_cast<const float4*>(X + r * NBP)[sub];
            acc = make_float4(d * x.x, d * x.y, d * x.z, d * x.w);
        }
        for (int list = 0; list < (pb ? 2 : 1); ++list) {
            const std::int64_t* ptr = list == 0 ? pa : pb;
            std::int64_t e = live ? ptr[r] : 0;
            const std::int64_t e1 = live ? ptr[r + 1] : 0;
            for (; e < e1; e += G) {  // (lanes of different groups run their own trip counts)
                const bool ok = e + sub < e1;
                const int c = ok ? col[e + sub] : 0;
                const float v = ok ? val[e + sub] : 0.f;
                const int cnt = e1 - e < G ? static_cast<int>(e1 - e) : G;
#pragma unroll 4
                for (int k = 0; k < cnt; ++k) {
                    const int ck = __shfl_sync(gmask, c, k, G);
                    const float vk = __shfl_sync(gmask, v, k, G);
                    const float4 x = __ldg(reinterpret_cast<const float4*>(X + static_cast<std::int64_t>(ck) * NBP) + sub);
                    vfma(acc, vk, x);
                }
            }
        }
        if (live) reinterpret_cast<float4*>(Y + r * NBP)[sub] = acc;
    }
}

// Y = diag(D) X  (the diagonal pass of kernels.hpp:363-370, run first so the
// tile kernel can accumulate straight into Y)
template <typename TX>
__global__ void k_diag_init(const double* __restrict__ d, const TX* __restrict__ X, TX* __restrict__ Y,
                            std::int64_t nrows, int nb) {
    const std::int64_t total = nrows * nb;
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t r = e / nb;
        Y[e] = static_cast<TX>(d[r] * static_cast<double>(X[e]));
    }
}

// f64 panel -> f32 copy for the tile kernel, and a zeroed f32 accumulator
__global__ void k_f64_to_f32(const double* __restrict__ x, float* __restrict__ x32, std::int64_t nin,
                             float* __restrict__ y32, std::int64_t nout) {
    const std::int64_t total = nin > nout ? nin : nout;
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (e < nin) x32[e] = static_cast<float>(x[e]);
        if (e < nout) y32[e] = 0.f;
    }
}

// Y = diag(D) X + Y32 (symmetric) or Y += Y32 (accumulate modes), in f64:
// the diagonal pass of kernels.hpp:363-370 kept in full precision
__global__ void k_finish_f64(const double* __restrict__ d, const double* __restrict__ X,
                             const float* __restrict__ y32, double* __restrict__ Y, std::int64_t nrows, int nb,
                             int symmetric) {
    // two elements per step (nb even: a row never splits a pair); 32-bit row
    // division when the panel allows it
    const std::int64_t total = nrows * nb;
    if (nb % 2 == 0 && total < (std::int64_t{1} << 32)) {
        const std::uint32_t half = static_cast<std::uint32_t>(total / 2), unb = static_cast<std::uint32_t>(nb);
        for (std::uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < half; e += gridDim.x * blockDim.x) {
            const float2 y = reinterpret_cast<const float2*>(y32)[e];
            double2 out;
            if (symmetric) {
                const std::uint32_t row = (unb & (unb - 1)) == 0 ? (2u * e) >> (__ffs(unb) - 1) : (2u * e) / unb;
                const double dr = d[row];
                const double2 x = reinterpret_cast<const double2*>(X)[e];
                out = make_double2(dr * x.x + static_cast<double>(y.x), dr * x.y + static_cast<double>(y.y));
            } else {
                out = reinterpret_cast<const double2*>(Y)[e];
                out.x += static_cast<double>(y.x);
                out.y += static_cast<double>(y.y);
            }
            reinterpret_cast<double2*>(Y)[e] = out;
        }
        return;
    }
    for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        if (symmetric)
            Y[e] = d[e / nb] * X[e] + static_cast<double>(y32[e]);
        else
            Y[e] += static_cast<double>(y32[e]);
    }
}

// out[i] = ((in_0[i] + in_1[i]) + ...) in slot order (the distributed Y sum); out may alias an input
struct SlotPtrs {
    const float* p[16];
};
__global__ void k_sum_slots(SlotPtrs in, int nin, float* out, std::int64_t count) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        float v = in.p[0][i];
        for (int q = 1; q < nin; ++q) v += in.p[q][i];
        out[i] = v;
    }
}

template <int NBP, typename TC, typename TV, typename TX>
std::size_t smem_bytes(int blob_max) {
    using G = XGeom<NBP, TC>;
    return 3 * kTile * G::LINEB + (kTile + 64) * G::CH * 16 + 2 * static_cast<std::size_t>(blob_max);
}

template <int NBP, typename TC, typename TV, typename TX>
void launch_tiles(Op* op, const int2* runs, index_t nruns, const TX* X, TX* Y, int nb, int ld, int do_r, int do_c,
                  cudaStream_t s) {
    auto kern = k_sym_spmm<NBP, TC, TV, TX>;
    const std::size_t sm = smem_bytes<NBP, TC, TV, TX>(op->blob_max);
    ensure_dyn_smem(kern, sm);
    int per_sm = 0;
    BE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, sm));
    if (per_sm < 1) fail(BE_ERR_CUDA, "sym_spmm: kernel does not fit on an SM");
    const int grid = static_cast<int>(std::min<index_t>(static_cast<index_t>(per_sm) * op->ctx->num_sms, nruns));
    op->grid = grid;
    if (grid == 0) return;
    kern<<<grid, kThreads, sm, s>>>(runs, static_cast<int>(nruns), op->tiles.get(), op->blobs.get(), X, Y, nb, ld,
                                    do_r, do_c, op->blob_max, op->counter.get());
    BE_CUDA(cudaGetLastError());
    ++op->ctx->launches;
}

template <typename TC, typename TV, typename TX>
void dispatch_nb(Op* op, const int2* runs, index_t nruns, const TX* X, TX* Y, int nb, int do_r, int do_c,
                 cudaStream_t s) {
    if constexpr (std::is_same_v<TC, double> && std::is_same_v<TV, double> && std::is_same_v<TX, double>) {
        // f64 values and panels (the 12 B/nnz parity mode): the warp-specialised kernel for nb 8 / 16
        static const bool ws64 = [] {
            const char* e = std::getenv("BE_SPMM_WS");
            return !(e && e[0] == '0');
        }();
        const bool aligned = (reinterpret_cast<std::uintptr_t>(X) & 15u) == 0 && (reinterpret_cast<std::uintptr_t>(Y) & 15u) == 0;
        if (ws64 && aligned) {
            if (nb == 16 && launch_ws<16, double>(op, runs, nruns, X, Y, do_r, do_c, s)) return;
            if (nb == 8 && launch_ws<8, double>(op, runs, nruns, X, Y, do_r, do_c, s)) return;
        }
    }
    if constexpr (std::is_same_v<TC, float> && std::is_same_v<TV, float> && std::is_same_v<TX, float>) {
        // the warp-specialised kernel for the widths it covers (T1: nb = 8 4.7 vs 6.3 ms, nb = 16
        // 8.0 vs 9.4 ms, nb = 32 14.9 vs 32.5 ms against the classic kernel); BE_SPMM_WS=0 selects
        // the classic kernel (experiments)
        static const int ws_mode = [] {
            const char* e = std::getenv("BE_SPMM_WS");
            return e && e[0] == '0' ? 0 : 2;
        }();
        const bool aligned = (reinterpret_cast<std::uintptr_t>(X) & 15u) == 0 && (reinterpret_cast<std::uintptr_t>(Y) & 15u) == 0;
        if (ws_mode > 0 && aligned) {
            if (nb == 16 && ws_mode == 2 && launch_ws<16>(op, runs, nruns, X, Y, do_r, do_c, s)) return;
            if (nb == 8 && launch_ws<8>(op, runs, nruns, X, Y, do_r, do_c, s)) return;
            if (nb == 32 && launch_ws<32>(op, runs, nruns, X, Y, do_r, do_c, s)) return;
        }
    }
    constexpr int VEC = Vec<TC>::N;
    // widest panel slice whose X_I / X_J / Y_I lines fit the shared memory of an SM next to the
    // two stage buffers: 64 f32 or 32 f64 columns; wider panels run as column slices (row stride nb)
    constexpr int WMAX = sizeof(TC) == 4 ? 64 : 32;
    for (int c0 = 0; c0 < nb; c0 += WMAX) {
        const int w = std::min(WMAX, nb - c0);
        const TX* x = X + c0;
        TX* y = Y + c0;
        if (w <= VEC) launch_tiles<VEC, TC, TV, TX>(op, runs, nruns, x, y, w, nb, do_r, do_c, s);
        else if (w <= 8) launch_tiles<8, TC, TV, TX>(op, runs, nruns, x, y, w, nb, do_r, do_c, s);
        else if (w <= 16) launch_tiles<16, TC, TV, TX>(op, runs, nruns, x, y, w, nb, do_r, do_c, s);
        else if (w <= 32) launch_tiles<32, TC, TV, TX>(op, runs, nruns, x, y, w, nb, do_r, do_c, s);
        else if constexpr (sizeof(TC) == 4) launch_tiles<64, TC, TV, TX>(op, runs, nruns, x, y, w, nb, do_r, do_c, s);
    }
}

// ---------------------------------------------------------------------------
// Tile-format build (host, parallel over CSB block rows).
// ---------------------------------------------------------------------------

struct RowOut {
    std::vector<TileHdr> hdr;         // begin16 relative to this block row's blob bytes
    std::vector<unsigned char> blob;  // the block row's tile blobs (values as f32 or f64)
    std::vector<std::int64_t> src;    // CSB index per row-order device entry (optional, npad per tile)
    std::vector<unsigned char> cls;   // per tile: 0 interior, 1 exterior (distributed operator)
};

// Padded coordinates of the distributed operator: row r of segment q maps to
// q * lmax + (r - cuts[q]).
struct RowMap {
    const index_t* cuts = nullptr;  // segment q = rows [cuts[q], cuts[q+1]), owned by rank owner[q]
    const int* owner = nullptr;
    int world = 1, rank = 0;
    index_t lmax = 0;
    int seg(index_t r) const {
        int lo = 0, hi = world;  // cuts[lo] <= r < cuts[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (cuts[mid] <= r) lo = mid; else hi = mid;
        }
        return lo;
    }
    int owner_of(index_t r) const { return owner[seg(r)]; }
    index_t pad(index_t r) const {
        const int q = seg(r);
        return static_cast<index_t>(owner[q]) * lmax + (r - cuts[q]);
    }
};

// Rank order of one side (rows or columns) of a tile: decreasing length, ties
// by index. For rows, lanes L and L + 4 of every quarter-warp (ranks 8q + j
// and 8q + j + 4) then get rows of opposite parity where a row of the same
// length allows it: their 64-byte Y_I rows then sit in opposite bank halves
// and the per-tile Y_I read-modify-write is conflict-free (nb = 16, f32).
void rank_order(const int* len, int* order, bool parity) {
    std::iota(order, order + kTile, 0);
    std::stable_sort(order, order + kTile, [&](int a, int b) { return len[a] > len[b]; });
    if (!parity) return;
    for (int p = 0; p < kTile; ++p) {
        if ((p & 7) < 4 || len[order[p]] == 0) continue;
        const int partner = order[p - 4];
        if (((order[p] ^ partner) & 1) != 0) continue;
        for (int q = p + 1; q < kTile && len[order[q]] == len[order[p]]; ++q)
            if (((order[q] ^ partner) & 1) != 0) {
                std::swap(order[p], order[q]);
                break;
            }
    }
}

// Emit one tile piece from `ent` = (local row << 56 | local col << 48 | CSB
// index), sorted by (row, col, index), as a blob (see the format above).
template <typename TV>
void emit_piece(const be_csb_view& L, const std::vector<std::uint64_t>& ent, index_t row0, index_t col0, index_t nr,
                index_t nc, bool keep_src, RowOut& out) {
    const int n = static_cast<int>(ent.size());
    const int npad = pad16(n);
    int rlen[kTile] = {0}, clen[kTile] = {0};
    for (std::uint64_t e : ent) {
        ++rlen[e >> 56];
        ++clen[(e >> 48) & 255u];
    }
    int rorder[kTile], corder[kTile];
    rank_order(rlen, rorder, true);
    rank_order(clen, corder, false);
    // JDS starts: jd[d] = sum over ranks of min(len, d)
    std::uint16_t jr[136] = {0}, jc[136] = {0};
    for (int d = 0; d < kTile; ++d) {
        int cr = 0, cc = 0;
        for (int i = 0; i < kTile; ++i) {
            cr += rlen[i] > d;
            cc += clen[i] > d;
        }
        jr[d + 1] = static_cast<std::uint16_t>(jr[d] + cr);
        jc[d + 1] = static_cast<std::uint16_t>(jc[d] + cc);
    }
    for (int d = kTile + 1; d < 136; ++d) {
        jr[d] = jr[kTile];
        jc[d] = jc[kTile];
    }
    // tail split (see k_sym_spmm): warp 0 of a pass stops at diagonal D, warp 3 takes [D, len)
    auto split_at = [](const int* len, const int* order) -> std::uint16_t {
        const int t0 = len[order[0]], t1 = len[order[32]], t2 = len[order[64]], t3 = len[order[96]];
        const int d = (std::max({t1, t2, (t0 + t3 + 1) / 2}) + 2) & ~3;  // nearest multiple of 4 (aligned starts)
        return static_cast<std::uint16_t>(d >= t0 || d == 0 ? 0xFFFF : d);
    };
    jr[kSplitSlot] = split_at(rlen, rorder);
    jc[kSplitSlot] = split_at(clen, corder);
    // work split of k_sym_spmm_ws: units u = 0..7 (pass R rank groups 0-3, then pass C groups 0-3,
    // 32 ranks each) flattened diagonal by diagonal; 8 contiguous pieces of about equal entry
    // count, cut at multiples of 4 diagonals; boundary w = (unit << 8) | diagonal
    std::uint16_t seg[9];
    {
        const long total = 2L * n;
        long acc = 0;
        int w = 1;
        seg[0] = 0;
        for (int un = 0; un < 8; ++un) {
            const int* len = un < 4 ? rlen : clen;
            const int* ord = un < 4 ? rorder : corder;
            const int g = un & 3;
            const int first = len[ord[32 * g]];
            for (int d0 = 0; d0 < first; d0 += 4) {
                for (int d = d0; d < d0 + 4; ++d)
                    for (int r = 32 * g; r < 32 * g + 32; ++r) acc += len[ord[r]] > d;
                while (w < 8 && acc * 8 >= static_cast<long>(w) * total) {
                    const int nx = d0 + 4;
                    seg[w++] = static_cast<std::uint16_t>(nx >= first ? (un + 1) << 8 : (un << 8) | nx);
                }
            }
        }
        while (w < 9) seg[w++] = static_cast<std::uint16_t>(8 << 8);
    }
    TileHdr hd{};
    hd.begin16 = static_cast<std::uint32_t>(out.blob.size() / 16);
    hd.row0 = static_cast<std::int32_t>(row0);
    hd.col0 = static_cast<std::int32_t>(col0);
    hd.packed = static_cast<std::uint32_t>(nr - 1) | (static_cast<std::uint32_t>(nc - 1) << 7) |
                (static_cast<std::uint32_t>(n) << 14);
    out.hdr.push_back(hd);
    const std::size_t base = out.blob.size();
    out.blob.resize(base + blob_bytes<TV>(n), 0);
    unsigned char* b = out.blob.data() + base;
    std::memcpy(b + kMetaJr, jr, sizeof(jr));
    std::memcpy(b + kMetaJc, jc, sizeof(jc));
    std::memcpy(b + kMetaSeg, seg, sizeof(seg));
    for (int i = 0; i < kTile; ++i) {
        b[kMetaRperm + i] = static_cast<unsigned char>(rorder[i]);
        b[kMetaCperm + i] = static_cast<unsigned char>(corder[i]);
        b[kMetaRlen + i] = static_cast<unsigned char>(rlen[rorder[i]]);
        b[kMetaClen + i] = static_cast<unsigned char>(clen[corder[i]]);
    }
    TV* rv = reinterpret_cast<TV*>(b + kMetaBytes);
    unsigned char* rcol = b + kMetaBytes + static_cast<std::size_t>(npad) * sizeof(TV);
    TV* cv = reinterpret_cast<TV*>(b + kMetaBytes + static_cast<std::size_t>(npad) * (sizeof(TV) + 1));
    unsigned char* crow = b + kMetaBytes + static_cast<std::size_t>(npad) * (2 * sizeof(TV) + 1);
    const std::size_t sbase = out.src.size();
    if (keep_src) out.src.resize(sbase + static_cast<std::size_t>(npad), -1);
    // rows: ent is (row, col)-sorted, so row `row`'s entries are contiguous
    int rstart[kTile + 1];
    rstart[0] = 0;
    for (int i = 0; i < kTile; ++i) rstart[i + 1] = rstart[i] + rlen[i];
    int crank[kTile];
    for (int i = 0; i < kTile; ++i) crank[corder[i]] = i;
    int cnext[kTile] = {0};  // per column: entries placed so far (rows ascend through the row loop)
    for (int r = 0; r < kTile; ++r) {
        const int row = rorder[r];
        for (int j = 0; j < rlen[row]; ++j) {
            const std::uint64_t e = ent[static_cast<std::size_t>(rstart[row] + j)];
            const int col = static_cast<int>((e >> 48) & 255u);
            const index_t k = static_cast<index_t>(e & 0xFFFFFFFFFFFFULL);
            const TV v = static_cast<TV>(L.values[k]);
            const int q = jr[j] + r;
            rv[q] = v;
            rcol[q] = static_cast<unsigned char>(col);
            if (keep_src) out.src[sbase + static_cast<std::size_t>(q)] = k;
        }
    }
    // columns: the j-th entry (by row) of column rank c at jc[j] + c
    for (int row = 0; row < kTile; ++row)
        for (int j = 0; j < rlen[row]; ++j) {
            const std::uint64_t e = ent[static_cast<std::size_t>(rstart[row] + j)];
            const int col = static_cast<int>((e >> 48) & 255u);
            const index_t k = static_cast<index_t>(e & 0xFFFFFFFFFFFFULL);
            const int q = jc[cnext[col]++] + crank[col];
            cv[q] = static_cast<TV>(L.values[k]);
            crow[q] = static_cast<unsigned char>(row);
        }
}

template <typename TV>
void build_block_row(const be_csb_view& L, index_t bi, int max_nnz, bool keep_src, const RowMap* map, RowOut& out) {
    const index_t br = L.row_offsets[bi + 1] - L.row_offsets[bi];
    const index_t ta = (br + kTile - 1) / kTile;
    struct BlockBuckets {  // one CSB block's entries bucketed by (a, b) sub-tile
        index_t bj = 0, tb = 0;
        std::vector<std::int32_t> start;
        std::vector<std::int64_t> idx;
    };
    std::vector<BlockBuckets> blocks;
    for (index_t bj = 0; bj < L.ncolblks; ++bj) {
        const index_t bidx = bi * L.ncolblks + bj;
        const index_t cnt = L.block_nnz[bidx];
        if (cnt == 0) continue;
        const index_t k0 = L.block_nnz_offsets[bidx];
        const index_t bc = L.col_offsets[bj + 1] - L.col_offsets[bj];
        BlockBuckets bb;
        bb.bj = bj;
        bb.tb = (bc + kTile - 1) / kTile;
        bb.start.assign(static_cast<std::size_t>(ta * bb.tb + 1), 0);
        for (index_t k = k0; k < k0 + cnt; ++k)
            ++bb.start[static_cast<std::size_t>((L.local_rows[k] / kTile) * bb.tb + L.local_cols[k] / kTile + 1)];
        for (std::size_t i = 1; i < bb.start.size(); ++i) bb.start[i] += bb.start[i - 1];
        std::vector<std::int32_t> cur(bb.start.begin(), bb.start.end() - 1);
        bb.idx.resize(static_cast<std::size_t>(cnt));
        for (index_t k = k0; k < k0 + cnt; ++k)
            bb.idx[static_cast<std::size_t>(cur[static_cast<std::size_t>((L.local_rows[k] / kTile) * bb.tb + L.local_cols[k] / kTile)]++)] = k;
        blocks.push_back(std::move(bb));
    }
    std::vector<std::uint64_t> keys, piece;
    const int row_own = map ? map->owner_of(L.row_offsets[bi]) : 0;
    for (index_t a = 0; a < ta; ++a) {
      for (int pass = 0; pass < (map ? 2 : 1); ++pass) {  // interior tiles first
        for (const auto& bb : blocks) {
            if (map) {
                const bool interior = row_own == map->rank && map->owner_of(L.col_offsets[bb.bj]) == map->rank;
                if (interior != (pass == 0)) continue;
            }
            for (index_t b = 0; b < bb.tb; ++b) {
                const std::size_t s0 = static_cast<std::size_t>(bb.start[static_cast<std::size_t>(a * bb.tb + b)]);
                const std::size_t s1 = static_cast<std::size_t>(bb.start[static_cast<std::size_t>(a * bb.tb + b + 1)]);
                if (s0 == s1) continue;
                keys.clear();
                for (std::size_t i = s0; i < s1; ++i) {
                    const index_t k = bb.idx[i];
                    const std::uint64_t r = L.local_rows[k] % kTile, c = L.local_cols[k] % kTile;
                    keys.push_back((r << 56) | (c << 48) | static_cast<std::uint64_t>(k));
                }
                std::sort(keys.begin(), keys.end());
                const index_t row0 = L.row_offsets[bi] + a * kTile;
                const index_t col0 = L.col_offsets[bb.bj] + b * kTile;
                const index_t nc = std::min<index_t>(kTile, (L.col_offsets[bb.bj + 1] - L.col_offsets[bb.bj]) - b * kTile);
                const index_t nr = std::min<index_t>(kTile, br - a * kTile);
                std::size_t p0 = 0;
                while (p0 < keys.size()) {  // row pieces of <= max_nnz entries
                    std::size_t p1 = std::min(keys.size(), p0 + static_cast<std::size_t>(max_nnz));
                    if (p1 < keys.size()) {
                        const std::uint64_t rcut = keys[p1] >> 56;
                        while (p1 > p0 && (keys[p1 - 1] >> 56) == rcut) --p1;
                        if (p1 == p0) fail(BE_ERR_BAD_PARAMS, "tile row longer than max_nnz");
                    }
                    piece.assign(keys.begin() + static_cast<std::ptrdiff_t>(p0), keys.begin() + static_cast<std::ptrdiff_t>(p1));
                    emit_piece<TV>(L, piece, map ? map->pad(row0) : row0, map ? map->pad(col0) : col0, nr, nc,
                                   keep_src, out);
                    out.cls.push_back(static_cast<unsigned char>(pass));
                    p0 = p1;
                }
            }
        }
      }
    }
}

}  // namespace

static void op_build(Op* op, const be_csb_view& L, const RowMap* map);
static void op_finish_tiles(Op* op, const std::vector<TileHdr>& all_hdr, const std::vector<unsigned char>& all_cls,
                            const RowMap* map);

Ctx::~Ctx() {}

void ensure_dyn_smem_raw(const void* kern, std::size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, std::size_t> cur;
    int dev = 0;
    BE_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    std::size_t& c = cur[{dev, kern}];
    if (bytes <= c) return;
    BE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    c = bytes;
}

Op::~Op() {
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    if (ev_x) cudaEventDestroy(ev_x);
    if (ev_ag) cudaEventDestroy(ev_ag);
    for (auto& e : ev_grp)
        if (e) cudaEventDestroy(e);
    if (cstream) cudaStreamDestroy(cstream);
}

// Row lists of the deterministic mode (see k_det_spmm): a stable counting sort
// of the CSB storage order (blocks row-major, entries in stored order) by
// global row gives each row's L entries in run_baseline's notrans order (column
// blocks ascending, stored order within a block); by global column, each
// column's entries in its trans order (row blocks ascending).
template <typename TV>
static void op_build_lists(Op* op, const be_csb_view& L, DBuf<TV>& vals_out) {
    const index_t n = L.nrows, m = L.ncols, nnz = L.nnz;
    if (nnz >= (index_t{1} << 40)) fail(BE_ERR_BAD_PARAMS, "row-list operator too large");
    std::vector<std::int64_t> pn(static_cast<std::size_t>(n) + 1, 0), pt(static_cast<std::size_t>(m) + 1, 0);
    auto each = [&](auto&& f) {  // blocks row-major, entries in stored order (the CSB storage order)
        for (index_t bi = 0; bi < L.nrowblks; ++bi)
            for (index_t bj = 0; bj < L.ncolblks; ++bj) {
                const index_t b = bi * L.ncolblks + bj;
                const index_t r0 = L.row_offsets[bi], c0 = L.col_offsets[bj];
                for (index_t k = L.block_nnz_offsets[b]; k < L.block_nnz_offsets[b] + L.block_nnz[b]; ++k)
                    f(k, r0 + L.local_rows[k], c0 + L.local_cols[k]);
            }
    };
    each([&](index_t, index_t r, index_t c) {
        ++pn[static_cast<std::size_t>(r) + 1];
        ++pt[static_cast<std::size_t>(c) + 1];
    });
    for (std::size_t i = 1; i < pn.size(); ++i) pn[i] += pn[i - 1];
    for (std::size_t i = 1; i < pt.size(); ++i) pt[i] += pt[i - 1];
    for (auto& x : pt) x += nnz;  // the L^T lists follow the L lists
    std::vector<std::int32_t> col(static_cast<std::size_t>(2 * nnz));
    std::vector<TV> val(static_cast<std::size_t>(2 * nnz));
    {
        std::vector<std::int64_t> cn(pn.begin(), pn.end() - 1), ct(pt.begin(), pt.end() - 1);
        each([&](index_t k, index_t r, index_t c) {
            const auto qn = cn[static_cast<std::size_t>(r)]++;
            col[static_cast<std::size_t>(qn)] = static_cast<std::int32_t>(c);
            val[static_cast<std::size_t>(qn)] = static_cast<TV>(L.values[k]);
            const auto qt = ct[static_cast<std::size_t>(c)]++;
            col[static_cast<std::size_t>(qt)] = static_cast<std::int32_t>(r);
            val[static_cast<std::size_t>(qt)] = static_cast<TV>(L.values[k]);
        });
    }
    op->det_ptr_n.reset(n + 1);
    op->det_ptr_t.reset(m + 1);
    op->det_col.reset(std::max<index_t>(2 * nnz, 1));
    vals_out.reset(std::max<index_t>(2 * nnz, 1));
    BE_CUDA(cudaMemcpy(op->det_ptr_n.get(), pn.data(), pn.size() * 8, cudaMemcpyHostToDevice));
    BE_CUDA(cudaMemcpy(op->det_ptr_t.get(), pt.data(), pt.size() * 8, cudaMemcpyHostToDevice));
    if (nnz > 0) {
        BE_CUDA(cudaMemcpy(op->det_col.get(), col.data(), col.size() * 4, cudaMemcpyHostToDevice));
        BE_CUDA(cudaMemcpy(vals_out.get(), val.data(), val.size() * sizeof(TV), cudaMemcpyHostToDevice));
    }
}

// Occupied 128 x 128 sub-tiles of L (the tile format's work units), exactly.
static index_t occupied_subtiles(const be_csb_view& L) {
    std::vector<index_t> per(static_cast<std::size_t>(L.nrowblks), 0);
    parallel_for_dynamic(hw_threads(), L.nrowblks, [&](index_t bi, int) {
        std::vector<std::uint64_t> bits;
        index_t c = 0;
        for (index_t bj = 0; bj < L.ncolblks; ++bj) {
            const index_t b = bi * L.ncolblks + bj, cnt = L.block_nnz[b];
            if (cnt == 0) continue;
            const index_t tb = (L.col_offsets[bj + 1] - L.col_offsets[bj] + kTile - 1) / kTile;
            const index_t ta = (L.row_offsets[bi + 1] - L.row_offsets[bi] + kTile - 1) / kTile;
            bits.assign(static_cast<std::size_t>((ta * tb + 63) / 64), 0);
            for (index_t k = L.block_nnz_offsets[b]; k < L.block_nnz_offsets[b] + cnt; ++k) {
                const index_t q = (L.local_rows[k] / kTile) * tb + L.local_cols[k] / kTile;
                bits[static_cast<std::size_t>(q >> 6)] |= std::uint64_t{1} << (q & 63);
            }
            for (auto w : bits) c += __builtin_popcountll(w);
        }
        per[static_cast<std::size_t>(bi)] = c;
    });
    index_t tot = 0;
    for (auto c : per) tot += c;
    return tot;
}

std::unique_ptr<Op> op_create(Ctx* ctx, const be_csb_view& L, const double* diag, int values_prec, int flags) {
    validate_view(L);
    if (values_prec != BE_F32 && values_prec != BE_F64) fail(BE_ERR_BAD_PARAMS, "values_prec must be BE_F32 or BE_F64");
    auto op = std::make_unique<Op>();
    op->ctx = ctx;
    op->nrows = L.nrows;
    op->ncols = L.ncols;
    op->nnz = L.nnz;
    op->values_prec = values_prec;
    op->symmetric = (flags & BE_OP_SYMMETRIC) != 0;
    if (op->symmetric) {  // SymmetricOperator ctor checks, kernels.hpp:341-350
        if (L.nrows != L.ncols) fail(BE_ERR_DIMENSION_MISMATCH, "SymmetricOperator: matrix must be square");
        if (!diag && L.nrows > 0) fail(BE_ERR_DIMENSION_MISMATCH, "SymmetricOperator: diagonal length mismatch");
        if (!is_strictly_lower(L)) fail(BE_ERR_NOT_STRICTLY_LOWER, "SymmetricOperator: stored entry with row <= col");
    }
    if (L.nrows >= (index_t{1} << 31) || L.ncols >= (index_t{1} << 31))
        fail(BE_ERR_BAD_PARAMS, "sym_spmm: dimension exceeds 2^31 rows per device");
    if (flags & BE_OP_DETERMINISTIC) {
        op->values_prec = BE_F64;
        op_build_lists<double>(op.get(), L, op->det_val);
        op->det = true;
    } else {
        bool rows = false;
        if (values_prec == BE_F32 && !(flags & BE_OP_FORMAT_TILES)) {
            if (flags & BE_OP_FORMAT_ROWS) rows = true;
            else if (const char* e = std::getenv("BE_SPMM_FORMAT")) rows = std::strcmp(e, "rows") == 0;  // (experiments)
            else if (L.nnz >= (index_t{1} << 22)) rows = L.nnz < 384 * occupied_subtiles(L);
        }
        if (rows) {
            op_build_lists<float>(op.get(), L, op->rows_val);
            op->rows = true;
        } else {
            op_build(op.get(), L, nullptr);
        }
    }
    if (op->symmetric) {
        op->diag.reset(std::max<index_t>(L.nrows, 1));
        if (L.nrows > 0)
            BE_CUDA(cudaMemcpy(op->diag.get(), diag, static_cast<std::size_t>(L.nrows) * 8, cudaMemcpyHostToDevice));
    }
    return op;
}

#ifndef BE_SPMM_MAXNNZ
#define BE_SPMM_MAXNNZ 2048  // f32 entries per tile piece (two CTAs per SM)
#endif

// Streamed build from a CSB1 file: batches of ~2^26 stored entries (whole block
// rows) are read by a loader thread while the previous batch is cut into tiles on the host
// workers and its blobs go up through the copy pool into a device buffer that grows by 1.5x
// (first sized from the header's entry count). Host memory holds about two batches instead of
// the whole matrix plus its tile format; file reading, tile building and the upload overlap.
// Same tiles, headers and runs as op_build over the whole matrix (tile format; the decode index
// is not kept).
std::unique_ptr<Op> op_create_csb1(Ctx* ctx, const std::string& path, int values_prec, int flags,
                                   std::vector<double>* diag_out, index_t batch_entries) {
    if (values_prec != BE_F32 && values_prec != BE_F64) fail(BE_ERR_BAD_PARAMS, "values_prec must be BE_F32 or BE_F64");
    if (!(flags & BE_OP_SYMMETRIC) || (flags & (BE_OP_DETERMINISTIC | BE_OP_FORMAT_ROWS)))
        fail(BE_ERR_BAD_PARAMS, "be_op_create_csb1: builds the symmetric operator in the tile format");
    index_t n = 0, nblk = 0;
    const std::vector<index_t> brn = csb1_block_row_nnz(path, n, nblk);
    if (n >= (index_t{1} << 31)) fail(BE_ERR_BAD_PARAMS, "sym_spmm: dimension exceeds 2^31 rows per device");
    const index_t nnz = std::accumulate(brn.begin(), brn.end(), index_t{0});
    if (batch_entries <= 0) batch_entries = index_t{1} << 26;
    std::vector<index_t> cut{0};
    for (index_t b = 0, acc = 0; b < nblk; ++b) {
        acc += brn[static_cast<std::size_t>(b)];
        if (acc >= batch_entries || b + 1 == nblk) {
            cut.push_back(b + 1);
            acc = 0;
        }
    }
    auto op = std::make_unique<Op>();
    op->ctx = ctx;
    op->nrows = op->ncols = n;
    op->nnz = nnz;
    op->values_prec = values_prec;
    op->symmetric = true;
    op->max_nnz = values_prec == BE_F32 ? BE_SPMM_MAXNNZ : 1024;
    op->blob_max = static_cast<int>(values_prec == BE_F32 ? blob_bytes<float>(op->max_nnz) : blob_bytes<double>(op->max_nnz));
    op->counter.reset(2);
    BE_CUDA(cudaMemset(op->counter.get(), 0, 2 * sizeof(int)));
    const std::size_t per_entry = values_prec == BE_F32 ? 2 * sizeof(float) + 2 : 2 * sizeof(double) + 2;
    index_t cap = std::max<index_t>(16, static_cast<index_t>(static_cast<double>(nnz) * per_entry * 1.25) + (index_t{1} << 24));
    op->blobs.reset(cap);
    std::vector<double> diag;
    diag.reserve(static_cast<std::size_t>(n));
    std::vector<TileHdr> all_hdr;
    std::vector<unsigned char> all_cls;
    index_t b_off = 0;
    cudaStream_t s = ctx->stream;
    struct Part {
        std::unique_ptr<CsbHost> m;
        std::vector<double> d;
    };
    auto load = [&path, &cut](std::size_t i) {
        Part p;
        p.m = load_csb1_rows(path, cut[i], cut[i + 1], &p.d);
        return p;
    };
    std::future<Part> next = std::async(std::launch::async, load, std::size_t{0});
    for (std::size_t i = 0; i + 1 < cut.size(); ++i) {
        Part part = next.get();
        if (i + 2 < cut.size()) next = std::async(std::launch::async, load, i + 1);
        const be_csb_view L = part.m->view();
        if (!is_strictly_lower(L)) fail(BE_ERR_NOT_STRICTLY_LOWER, "SymmetricOperator: stored entry with row <= col");
        if (part.d.size() != static_cast<std::size_t>(L.row_offsets[cut[i + 1]] - L.row_offsets[cut[i]]))
            fail(BE_ERR_DIMENSION_MISMATCH, "SymmetricOperator: diagonal length mismatch (CSB1 file without its diagonal)");
        diag.insert(diag.end(), part.d.begin(), part.d.end());
        const index_t b0 = cut[i], nb = cut[i + 1] - cut[i];
        std::vector<RowOut> rows(static_cast<std::size_t>(nb));
        parallel_for_dynamic(hw_threads(), nb, [&](index_t q, int) {
            if (values_prec == BE_F32)
                build_block_row<float>(L, b0 + q, op->max_nnz, false, nullptr, rows[static_cast<std::size_t>(q)]);
            else
                build_block_row<double>(L, b0 + q, op->max_nnz, false, nullptr, rows[static_cast<std::size_t>(q)]);
        });
        part.m.reset();
        index_t add = 0;
        for (const auto& r : rows) add += static_cast<index_t>(r.blob.size());
        if (b_off + add > cap) {  // grow by 1.5x, keeping the blobs already up
            const index_t nc = std::max(b_off + add, cap + cap / 2);
            DBuf<unsigned char> nbuf(nc);
            BE_CUDA(cudaStreamSynchronize(s));
            if (b_off) BE_CUDA(cudaMemcpyAsync(nbuf.get(), op->blobs.get(), static_cast<std::size_t>(b_off), cudaMemcpyDeviceToDevice, s));
            BE_CUDA(cudaStreamSynchronize(s));
            op->blobs = std::move(nbuf);
            cap = nc;
        }
        for (auto& r : rows) {
            if (r.hdr.empty()) continue;
            for (auto& h : r.hdr) h.begin16 += static_cast<std::uint32_t>(b_off / 16);
            all_hdr.insert(all_hdr.end(), r.hdr.begin(), r.hdr.end());
            all_cls.insert(all_cls.end(), r.cls.begin(), r.cls.end());
            h2d_large(op->blobs.get() + b_off, r.blob.data(), r.blob.size(), s);
            b_off += static_cast<index_t>(r.blob.size());
            if (b_off / 16 >= (index_t{1} << 32)) fail(BE_ERR_BAD_PARAMS, "sym_spmm: tile blobs exceed 64 GB on one device");
            r = RowOut();
        }
        BE_CUDA(cudaStreamSynchronize(s));  // the batch's pageable sources are released next round
    }
    op->blob_total = b_off;
    op->padded = 0;
    op_finish_tiles(op.get(), all_hdr, all_cls, nullptr);
    op->diag.reset(std::max<index_t>(n, 1));
    if (n > 0) BE_CUDA(cudaMemcpy(op->diag.get(), diag.data(), static_cast<std::size_t>(n) * 8, cudaMemcpyHostToDevice));
    if (diag_out) *diag_out = std::move(diag);
    return op;
}

// Rows of one L2 column band: the f32 X_J and Y_J rows of a band at nb = 16
// (2 x 64 B per row) take about half of the 126 MB L2.
#ifndef BE_SPMM_BAND_ROWS
#define BE_SPMM_BAND_ROWS 500000
#endif

// Tile-format build + upload shared by the single- and multi-GPU operators.
static void op_build(Op* op, const be_csb_view& L, const RowMap* map) {
    const int values_prec = op->values_prec;
#ifndef BE_SPMM_MAXNNZ
#define BE_SPMM_MAXNNZ 2048  // f32 entries per tile piece (two CTAs per SM)
#endif
    op->max_nnz = values_prec == BE_F32 ? BE_SPMM_MAXNNZ : 1024;
    op->blob_max = static_cast<int>(values_prec == BE_F32 ? blob_bytes<float>(op->max_nnz) : blob_bytes<double>(op->max_nnz));
    const bool keep_src = L.nnz <= (index_t{1} << 26);

    std::vector<RowOut> rows(static_cast<std::size_t>(L.nrowblks));
    parallel_for_dynamic(hw_threads(), L.nrowblks, [&](index_t bi, int) {
        if (values_prec == BE_F32)
            build_block_row<float>(L, bi, op->max_nnz, keep_src, map, rows[static_cast<std::size_t>(bi)]);
        else
            build_block_row<double>(L, bi, op->max_nnz, keep_src, map, rows[static_cast<std::size_t>(bi)]);
    });
    index_t ntiles = 0, bytes = 0, padded = 0;
    for (const auto& r : rows) {
        ntiles += static_cast<index_t>(r.hdr.size());
        bytes += static_cast<index_t>(r.blob.size());
        padded += static_cast<index_t>(r.src.size());
    }
    if (bytes / 16 >= (index_t{1} << 32)) fail(BE_ERR_BAD_PARAMS, "sym_spmm: tile blobs exceed 64 GB on one device");
    op->blob_total = bytes;
    op->padded = keep_src ? padded : 0;
    op->blobs.reset(std::max<index_t>(bytes, 16));
    op->counter.reset(2);
    BE_CUDA(cudaMemset(op->counter.get(), 0, 2 * sizeof(int)));
    op->csb_index.clear();
    if (keep_src) op->csb_index.reserve(static_cast<std::size_t>(padded));
    std::vector<TileHdr> all_hdr;
    all_hdr.reserve(static_cast<std::size_t>(ntiles));
    std::vector<unsigned char> all_cls;
    all_cls.reserve(static_cast<std::size_t>(ntiles));
    index_t b_off = 0;
    for (auto& r : rows) {
        if (r.hdr.empty()) continue;
        for (auto& h : r.hdr) h.begin16 += static_cast<std::uint32_t>(b_off / 16);
        all_hdr.insert(all_hdr.end(), r.hdr.begin(), r.hdr.end());
        all_cls.insert(all_cls.end(), r.cls.begin(), r.cls.end());
        // the copy pool (pinned pipelines on 16 host threads) instead of the driver's pageable path
        h2d_large(op->blobs.get() + b_off, r.blob.data(), r.blob.size(), op->ctx->stream);
        if (keep_src) op->csb_index.insert(op->csb_index.end(), r.src.begin(), r.src.end());
        b_off += static_cast<index_t>(r.blob.size());
        r = RowOut();
    }
    BE_CUDA(cudaStreamSynchronize(op->ctx->stream));
    op_finish_tiles(op, all_hdr, all_cls, map);
}

// Tile headers + run lists (shared by the in-memory and the streamed builds).
static void op_finish_tiles(Op* op, const std::vector<TileHdr>& all_hdr, const std::vector<unsigned char>& all_cls,
                            const RowMap* map) {
    const index_t ntiles = static_cast<index_t>(all_hdr.size());
    op->ntiles = ntiles;
    op->tiles.reset(std::max<index_t>(ntiles, 1));
    if (ntiles > 0)
        BE_CUDA(cudaMemcpy(op->tiles.get(), all_hdr.data(), all_hdr.size() * sizeof(TileHdr), cudaMemcpyHostToDevice));
    if (map) {  // padded slots (ranks) whose rows the tiles read or write: tiles never straddle a segment
        op->touched.assign(static_cast<std::size_t>(map->world), 0);
        for (const auto& h : all_hdr) {
            op->touched[static_cast<std::size_t>(h.row0 / map->lmax)] = 1;
            op->touched[static_cast<std::size_t>(h.col0 / map->lmax)] = 1;
        }
    }
    {  // runs: consecutive tiles of one tile-row, class and L2 column band, at most kRunMax tiles each,
       // ordered by (class, band, tile-row)
        struct R {
            int cls;
            index_t band;
            int b, e;
            int seg;
        };
        std::vector<R> all;
        index_t band_rows = BE_SPMM_BAND_ROWS;
        if (const char* e = std::getenv("BE_SPMM_BAND_ROWS")) band_rows = std::atoll(e);  // (experiments)
        band_rows = std::max<index_t>(kTile, band_rows);
        // distributed operator: the column segment of a tile (segment order; the padded slot is its owner)
        auto colseg = [&](const TileHdr& h) -> int {
            if (!map) return 0;
            const int slot = static_cast<int>(h.col0 / map->lmax);
            for (int q = 0; q < map->world; ++q)
                if (map->owner[q] == slot) return q;
            return 0;
        };
        for (index_t t = 0; t < ntiles;) {
            const auto& h0 = all_hdr[static_cast<std::size_t>(t)];
            const unsigned char c0 = all_cls[static_cast<std::size_t>(t)];
            const index_t band = h0.col0 / band_rows;
            const int q0 = colseg(h0);
            index_t e = t + 1;
            while (e < ntiles && e - t < kRunMax && all_hdr[static_cast<std::size_t>(e)].row0 == h0.row0 &&
                   all_cls[static_cast<std::size_t>(e)] == c0 && all_hdr[static_cast<std::size_t>(e)].col0 / band_rows == band &&
                   colseg(all_hdr[static_cast<std::size_t>(e)]) == q0)
                ++e;
            all.push_back(R{c0, band, static_cast<int>(t), static_cast<int>(e), q0});
            t = e;
        }
        std::stable_sort(all.begin(), all.end(), [](const R& a, const R& b) {
            if (a.cls != b.cls) return a.cls < b.cls;
            if (a.seg != b.seg) return a.seg < b.seg;
            return a.band < b.band;
        });
        std::vector<int2> runs[2];
        for (const auto& x : all) runs[x.cls].push_back(make_int2(x.b, x.e));
        if (map) {  // exterior groups by column segment
            op->ext_group.assign(static_cast<std::size_t>(map->world) + 1, 0);
            for (const auto& x : all)
                if (x.cls == 1) ++op->ext_group[static_cast<std::size_t>(x.seg) + 1];
            for (std::size_t q = 1; q < op->ext_group.size(); ++q) op->ext_group[q] += op->ext_group[q - 1];
        }
        op->nruns = static_cast<index_t>(runs[0].size());
        op->runs.reset(std::max<index_t>(op->nruns, 1));
        if (!runs[0].empty())
            BE_CUDA(cudaMemcpy(op->runs.get(), runs[0].data(), runs[0].size() * sizeof(int2), cudaMemcpyHostToDevice));
        op->nruns_ext = static_cast<index_t>(runs[1].size());
        op->runs_ext.reset(std::max<index_t>(op->nruns_ext, 1));
        if (!runs[1].empty())
            BE_CUDA(cudaMemcpy(op->runs_ext.get(), runs[1].data(), runs[1].size() * sizeof(int2),
                               cudaMemcpyHostToDevice));
    }
}

// Distributed apply (row e): Y_local = (L + L^T + D) X over all ranks.
//   1. X_local (f64) -> its f32 segment of the padded exchange panel; the
//      f32 accumulator (world * lmax rows) is zeroed in the same pass.
//   2. allgather of the f32 segments on the communication stream, overlapped
//      with the interior tiles (both coordinates in this rank's segment).
//   3. the remaining tiles once the gather has landed.
//   4. reduce-scatter of the partial Y panels to the row owners, then
//      Y_local = D X_local + y in f64 (the diagonal pass, kernels.hpp:363-370).
// This is distributed_spmm (dist.hpp:256-371) on NCCL collectives.
// Distributed apply, segment-wise exchange. Rank r's panel rows
// live in padded slot r of the f32 exchange buffers. X: rank r sends its slot
// to exactly the ranks whose tiles touch it and receives the slots its own
// tiles touch (NCCL send / recv on the communication stream, overlapped with
// the interior tiles); Y: segment by segment, as soon as the tiles writing a
// segment have run, the ranks that wrote it send their partial to its owner
// (overlapped with the next segments' tiles), and the owner sums the partials
// of its slot in ascending rank order (identical on every run). Only touched
// slots are zeroed; no full-panel collective remains.
static void op_apply_dist(Op* op, const double* X, double* Y, index_t in_rows, int nb, cudaStream_t s) {
    if (in_rows != op->nlocal) fail(BE_ERR_DIMENSION_MISMATCH, "distributed apply: local rows mismatch");
    const int world = op->world, me = op->rank;
    const index_t seg = op->lmax * nb, tot = seg * world;
    if (op->x32.n < tot) {
        op->x32.reset(tot);
        op->y32.reset(tot);
        op->ystage.reset(tot);
    }
    if (!op->cstream) {
        BE_CUDA(cudaStreamCreateWithFlags(&op->cstream, cudaStreamNonBlocking));
        BE_CUDA(cudaEventCreateWithFlags(&op->ev_x, cudaEventDisableTiming));
        BE_CUDA(cudaEventCreateWithFlags(&op->ev_ag, cudaEventDisableTiming));
    }
    if (op->timing) {
        for (auto& e : op->ev)
            if (!e) BE_CUDA(cudaEventCreate(&e));
        BE_CUDA(cudaEventRecord(op->ev[0], s));
    }
    auto need = [&](int p, int r) { return op->need[static_cast<std::size_t>(p) * world + r] != 0; };
    const std::size_t sb = static_cast<std::size_t>(seg) * sizeof(float);
    float* xs = op->x32.get() + static_cast<index_t>(me) * seg;
    const int g = static_cast<int>(std::max<index_t>(1, std::min<index_t>((seg + 255) / 256, op->ctx->num_sms * 8)));
    k_f64_to_f32<<<g, 256, 0, s>>>(X, xs, op->nlocal * nb, nullptr, 0);
    BE_CUDA(cudaGetLastError());
    ++op->ctx->launches;
    for (int r = 0; r < world; ++r)  // the partial Y slots this rank's tiles write
        if (r == me || need(me, r)) BE_CUDA(cudaMemsetAsync(op->y32.get() + static_cast<index_t>(r) * seg, 0, sb, s));
    BE_CUDA(cudaEventRecord(op->ev_x, s));
    BE_CUDA(cudaStreamWaitEvent(op->cstream, op->ev_x, 0));
    {
        std::vector<P2POp> xo;
        for (int p = 0; p < world; ++p) {
            if (p == me) continue;
            if (need(p, me)) xo.push_back(P2POp{p, true, xs, sb});
            if (need(me, p)) xo.push_back(P2POp{p, false, op->x32.get() + static_cast<index_t>(p) * seg, sb});
        }
        nvtxRangePushA("x-exchange");
        op->comm->p2p(xo, op->cstream);
        nvtxRangePop();
    }
    BE_CUDA(cudaEventRecord(op->ev_ag, op->cstream));
    if (op->timing) BE_CUDA(cudaEventRecord(op->ev[1], s));
    if (op->nruns > 0)
        dispatch_nb<float, float, float>(op, op->runs.get(), op->nruns, op->x32.get(), op->y32.get(), nb, 1, 1, s);
    BE_CUDA(cudaStreamWaitEvent(s, op->ev_ag, 0));
    float* ys = op->y32.get() + static_cast<index_t>(me) * seg;
    // Exterior tiles segment by segment; once groups 0..q ran, segment q's partial Y is final and its
    // exchange (call q: every rank that wrote it sends it to the owner, the owner receives) runs on the
    // communication stream while the next groups compute. One call per segment on every rank keeps
    // the calls matched.
    if (op->ev_grp.size() < static_cast<std::size_t>(world)) {
        for (int q = static_cast<int>(op->ev_grp.size()); q < world; ++q) {
            cudaEvent_t e = nullptr;
            BE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            op->ev_grp.push_back(e);
        }
    }
    for (int q = 0; q < world; ++q) {
        const index_t g0 = op->ext_group[static_cast<std::size_t>(q)], g1 = op->ext_group[static_cast<std::size_t>(q) + 1];
        if (g1 > g0)
            dispatch_nb<float, float, float>(op, op->runs_ext.get() + g0, g1 - g0, op->x32.get(), op->y32.get(), nb, 1, 1, s);
        BE_CUDA(cudaEventRecord(op->ev_grp[static_cast<std::size_t>(q)], s));
        BE_CUDA(cudaStreamWaitEvent(op->cstream, op->ev_grp[static_cast<std::size_t>(q)], 0));
        const int o = op->owner[static_cast<std::size_t>(q)];
        std::vector<P2POp> yo;
        if (o != me && need(me, o)) yo.push_back(P2POp{o, true, op->y32.get() + static_cast<index_t>(o) * seg, sb});
        if (o == me)
            for (int p = 0; p < world; ++p)
                if (p != me && need(p, me))
                    yo.push_back(P2POp{p, false, op->ystage.get() + static_cast<index_t>(p) * seg, sb});
        nvtxRangePushA("y-exchange");
        op->comm->p2p(yo, op->cstream);
        nvtxRangePop();
    }
    BE_CUDA(cudaEventRecord(op->ev_ag, op->cstream));
    BE_CUDA(cudaStreamWaitEvent(s, op->ev_ag, 0));
    {
        std::vector<const float*> parts;
        for (int q = 0; q < world; ++q)  // ascending rank order
            if (q == me) parts.push_back(ys);
            else if (need(q, me)) parts.push_back(op->ystage.get() + static_cast<index_t>(q) * seg);
        // ((p0 + p1) + p2) + ... in chunks of 16 pointers; the running sum lands in ys
        for (std::size_t b = 0; b + 1 < parts.size(); b += 15) {
            SlotPtrs in{};
            int nin = 0;
            in.p[nin++] = b == 0 ? parts[0] : ys;
            for (std::size_t q = b + 1; q < parts.size() && nin < 16; ++q) in.p[nin++] = parts[q];
            k_sum_slots<<<g, 256, 0, s>>>(in, nin, ys, seg);
            BE_CUDA(cudaGetLastError());
            ++op->ctx->launches;
        }
    }
    if (op->nlocal > 0) {
        const index_t out = op->nlocal * nb;
        const int g2 = static_cast<int>(std::max<index_t>(1, std::min<index_t>((out + 255) / 256, op->ctx->num_sms * 8)));
        k_finish_f64<<<g2, 256, 0, s>>>(op->diag.get(), X, ys, Y, op->nlocal, nb, 1);
        BE_CUDA(cudaGetLastError());
        ++op->ctx->launches;
    }
    if (op->timing) {
        BE_CUDA(cudaEventRecord(op->ev[2], s));
        BE_CUDA(cudaEventSynchronize(op->ev[2]));
        float a = 0, k = 0;
        BE_CUDA(cudaEventElapsedTime(&a, op->ev[0], op->ev[2]));
        BE_CUDA(cudaEventElapsedTime(&k, op->ev[1], op->ev[2]));
        op->last_apply_ms = a;
        op->last_kernel_ms = k;
    }
}

void op_apply(Op* op, const void* X, void* Y, index_t in_rows, int nb, int panel_prec, int mode, cudaStream_t s) {
    if (nb < 1) fail(BE_ERR_DIMENSION_MISMATCH, "apply: nb must be positive");
    if (panel_prec != BE_F32 && panel_prec != BE_F64) fail(BE_ERR_BAD_PARAMS, "apply: panel_prec must be BE_F32 or BE_F64");
    if (X == Y) fail(BE_ERR_BAD_PARAMS, "spmm: W and U must not alias");
    if (op->comm) {
        if (mode != BE_APPLY_SYMMETRIC || panel_prec != BE_F64)
            fail(BE_ERR_BAD_PARAMS, "distributed apply: symmetric mode on f64 panels only");
        return op_apply_dist(op, static_cast<const double*>(X), static_cast<double*>(Y), in_rows, nb, s);
    }
    int do_r = 0, do_c = 0;
    index_t out_rows = 0;
    switch (mode) {
        case BE_APPLY_SYMMETRIC:
            if (!op->symmetric) fail(BE_ERR_BAD_PARAMS, "apply: symmetric mode needs a symmetric operator");
            if (in_rows != op->nrows) fail(BE_ERR_DIMENSION_MISMATCH, "SymmetricOperator::apply: shape mismatch");
            do_r = do_c = 1;
            out_rows = op->nrows;
            break;
        case BE_APPLY_NOTRANS_ACC:
            if (in_rows != op->ncols) fail(BE_ERR_DIMENSION_MISMATCH, "spmm: operand shapes do not conform to the matrix");
            do_r = 1;
            out_rows = op->nrows;
            break;
        case BE_APPLY_TRANS_ACC:
            if (in_rows != op->nrows) fail(BE_ERR_DIMENSION_MISMATCH, "spmm: operand shapes do not conform to the matrix");
            do_c = 1;
            out_rows = op->ncols;
            break;
        default:
            fail(BE_ERR_BAD_PARAMS, "apply: unknown mode");
    }
    if (op->timing) {
        for (auto& e : op->ev)
            if (!e) BE_CUDA(cudaEventCreate(&e));
        BE_CUDA(cudaEventRecord(op->ev[0], s));
    }
    const index_t in_tot = in_rows * nb, out_tot = out_rows * nb;
    auto grid_for = [&](index_t total) {
        return static_cast<int>(std::max<index_t>(1, std::min<index_t>((total + 255) / 256, op->ctx->num_sms * 8)));
    };
    if (op->rows) {  // row-list format (sparse matrices, f32 values)
        if (op->timing) BE_CUDA(cudaEventRecord(op->ev[1], s));
        const std::int64_t* pa = mode == BE_APPLY_TRANS_ACC ? op->det_ptr_t.get() : op->det_ptr_n.get();
        const std::int64_t* pb = mode == BE_APPLY_SYMMETRIC ? op->det_ptr_t.get() : nullptr;
        const bool f64p = panel_prec == BE_F64;
        const float* xs = static_cast<const float*>(X);
        float* ys = static_cast<float*>(Y);
        if (f64p) {  // f32 copy of X; the f32 sums land in y32 and the finish adds them (and D X) in f64
            const index_t need = std::max(in_tot, out_tot);
            if (op->x32.n < need) {
                op->x32.reset(need);
                op->y32.reset(need);
            }
            k_f64_to_f32<<<grid_for(in_tot), 256, 0, s>>>(static_cast<const double*>(X), op->x32.get(), in_tot, nullptr, 0);
            BE_CUDA(cudaGetLastError());
            ++op->ctx->launches;
            xs = op->x32.get();
            ys = op->y32.get();
        }
        const int init = f64p ? 0 : (mode == BE_APPLY_SYMMETRIC ? 2 : 1);
        const double* dg = init == 2 ? op->diag.get() : nullptr;
        const bool a16 = (reinterpret_cast<std::uintptr_t>(xs) & 15u) == 0 && (reinterpret_cast<std::uintptr_t>(ys) & 15u) == 0;
        if (out_rows > 0) {
            auto launch = [&](auto kern, int rows_per_warp) {
                const index_t warps = (out_rows + rows_per_warp - 1) / rows_per_warp;
                const int g = static_cast<int>(std::max<index_t>(1, std::min<index_t>((warps * 32 + 255) / 256, op->ctx->num_sms * 16)));
                kern<<<g, 256, 0, s>>>(pa, pb, op->det_col.get(), op->rows_val.get(), dg, xs, ys, out_rows, init);
            };
            if (a16 && nb == 16) launch(k_rows_spmm<16>, 8);
            else if (a16 && nb == 8) launch(k_rows_spmm<8>, 16);
            else if (a16 && nb == 32) launch(k_rows_spmm<32>, 4);
            else if (a16 && nb == 4) launch(k_rows_spmm<4>, 32);
            else if (init == 1) {  // other widths: one warp per row, lane = column
                k_det_spmm<float, float><<<grid_for(out_rows * 32), 256, 0, s>>>(pa, pb, op->det_col.get(), op->rows_val.get(),
                                                                              nullptr, xs, ys, out_rows, nb, 0);
            } else {
                if (init == 2) {  // Y = D X first, then the lists accumulate
                    k_diag_init<float><<<grid_for(out_tot), 256, 0, s>>>(op->diag.get(), xs, ys, out_rows, nb);
                    BE_CUDA(cudaGetLastError());
                    ++op->ctx->launches;
                }
                k_det_spmm<float, float><<<grid_for(out_rows * 32), 256, 0, s>>>(pa, pb, op->det_col.get(), op->rows_val.get(),
                                                                              nullptr, xs, ys, out_rows, nb, init == 0 ? 1 : 0);
            }
            BE_CUDA(cudaGetLastError());
            ++op->ctx->launches;
        }
        if (f64p && out_tot > 0) {
            k_finish_f64<<<grid_for(out_tot), 256, 0, s>>>(op->diag.get(), static_cast<const double*>(X), op->y32.get(),
                                                            static_cast<double*>(Y), out_rows, nb,
                                                            mode == BE_APPLY_SYMMETRIC ? 1 : 0);
            BE_CUDA(cudaGetLastError());
            ++op->ctx->launches;
        }
    } else if (op->det) {  // deterministic mode: one pass over the row lists
        if (op->timing) BE_CUDA(cudaEventRecord(op->ev[1], s));
        const std::int64_t* pa = mode == BE_APPLY_TRANS_ACC ? op->det_ptr_t.get() : op->det_ptr_n.get();
        const std::int64_t* pb = mode == BE_APPLY_SYMMETRIC ? op->det_ptr_t.get() : nullptr;
        const double* dg = mode == BE_APPLY_SYMMETRIC ? op->diag.get() : nullptr;
        const int zero = mode == BE_APPLY_SYMMETRIC ? 1 : 0;
        if (out_rows > 0) {
            const int g = grid_for(out_rows * 32);
            if (panel_prec == BE_F64)
                k_det_spmm<double><<<g, 256, 0, s>>>(pa, pb, op->det_col.get(), op->det_val.get(), dg,
                                                     static_cast<const double*>(X), static_cast<double*>(Y), out_rows,
                                                     nb, zero);
            else
                k_det_spmm<float><<<g, 256, 0, s>>>(pa, pb, op->det_col.get(), op->det_val.get(), dg,
                                                    static_cast<const float*>(X), static_cast<float*>(Y), out_rows, nb,
                                                    zero);
            BE_CUDA(cudaGetLastError());
            ++op->ctx->launches;
        }
    } else if (panel_prec == BE_F64 && op->values_prec == BE_F32) {
        // f32 SpMM on f64 panels: X -> f32 copy, tile kernel into a zeroed f32
        // accumulator, then Y = D X + acc in f64 (halves the gathered and
        // reduced vector bytes of the tile kernel)
        const index_t need = std::max(in_tot, out_tot);
        if (op->x32.n < need) {
            op->x32.reset(need);
            op->y32.reset(need);
        }
        k_f64_to_f32<<<grid_for(need), 256, 0, s>>>(static_cast<const double*>(X), op->x32.get(), in_tot,
                                                       op->y32.get(), out_tot);
        BE_CUDA(cudaGetLastError());
        ++op->ctx->launches;
        if (op->timing) BE_CUDA(cudaEventRecord(op->ev[1], s));
        if (op->ntiles > 0) dispatch_nb<float, float, float>(op, op->runs.get(), op->nruns, op->x32.get(), op->y32.get(), nb, do_r, do_c, s);
        if (out_tot > 0) {
            k_finish_f64<<<grid_for(out_tot), 256, 0, s>>>(op->diag.get(), static_cast<const double*>(X), op->y32.get(),
                                                            static_cast<double*>(Y), out_rows, nb,
                                                            mode == BE_APPLY_SYMMETRIC ? 1 : 0);
            BE_CUDA(cudaGetLastError());
            ++op->ctx->launches;
        }
    } else {
        if (mode == BE_APPLY_SYMMETRIC && out_rows > 0) {
            if (panel_prec == BE_F32)
                k_diag_init<float><<<grid_for(out_tot), 256, 0, s>>>(op->diag.get(), static_cast<const float*>(X),
                                                                     static_cast<float*>(Y), out_rows, nb);
            else
                k_diag_init<double><<<grid_for(out_tot), 256, 0, s>>>(op->diag.get(), static_cast<const double*>(X),
                                                                      static_cast<double*>(Y), out_rows, nb);
            BE_CUDA(cudaGetLastError());
            ++op->ctx->launches;
        }
        if (op->timing) BE_CUDA(cudaEventRecord(op->ev[1], s));
        if (op->ntiles > 0) {
            if (op->values_prec == BE_F32) {
                dispatch_nb<float, float, float>(op, op->runs.get(), op->nruns, static_cast<const float*>(X), static_cast<float*>(Y), nb, do_r, do_c, s);
            } else {
                if (panel_prec == BE_F32)
                    dispatch_nb<double, double, float>(op, op->runs.get(), op->nruns, static_cast<const float*>(X), static_cast<float*>(Y), nb, do_r, do_c, s);
                else
                    dispatch_nb<double, double, double>(op, op->runs.get(), op->nruns, static_cast<const double*>(X), static_cast<double*>(Y), nb, do_r, do_c, s);
            }
        }
    }
    if (op->timing) {
        BE_CUDA(cudaEventRecord(op->ev[2], s));
        BE_CUDA(cudaEventSynchronize(op->ev[2]));
        float a = 0, k = 0;
        BE_CUDA(cudaEventElapsedTime(&a, op->ev[0], op->ev[2]));
        BE_CUDA(cudaEventElapsedTime(&k, op->ev[1], op->ev[2]));
        op->last_apply_ms = a;
        op->last_kernel_ms = k;
    }
}

// ---------------------------------------------------------------------------
// Multi-GPU partition (row e). Both rules are integer-exact so every rank (and
// the Python restatement in tests/) derives the same cuts.
// ---------------------------------------------------------------------------

// Equal-rows panel ownership on block boundaries: cut p is the boundary
// closest to n * p / world (the lower one on ties), kept strictly increasing
// so every rank owns at least one block row.
std::vector<index_t> dist_rows(const index_t* b, index_t nbounds, int world) {
    const index_t nblk = nbounds - 1;
    if (world < 1) fail(BE_ERR_BAD_PARAMS, "dist_rows: world must be positive");
    if (nblk < world) fail(BE_ERR_BAD_PARAMS, "dist_rows: fewer block rows than ranks");
    const index_t n = b[nblk];
    std::vector<index_t> k(static_cast<std::size_t>(world) + 1);
    k[0] = 0;
    k[static_cast<std::size_t>(world)] = nblk;
    for (int p = 1; p < world; ++p) {
        const __int128 target = static_cast<__int128>(n) * p;  // compare b * world with n * p
        index_t best = 0;
        __int128 bestd = -1;
        for (index_t j = 0; j <= nblk; ++j) {
            __int128 dd = static_cast<__int128>(b[j]) * world - target;
            if (dd < 0) dd = -dd;
            if (bestd < 0 || dd < bestd) {
                bestd = dd;
                best = j;
            }
        }
        k[static_cast<std::size_t>(p)] = best;
    }
    for (int p = 1; p < world; ++p)  // strictly increasing, room for the ranks after p
        k[static_cast<std::size_t>(p)] = std::min(std::max(k[static_cast<std::size_t>(p)], k[static_cast<std::size_t>(p) - 1] + 1),
                                                  nblk - (world - p));
    std::vector<index_t> cuts(static_cast<std::size_t>(world) + 1);
    for (int p = 0; p <= world; ++p) cuts[static_cast<std::size_t>(p)] = b[k[static_cast<std::size_t>(p)]];
    return cuts;
}

// nnz-balanced 2-D tiles (north_star's partition): recursive coordinate bisection of the lower
// block grid. w[bi * nblk + bj] = stored entries of CSB block (bi, bj) (bi >= bj; the upper part
// is ignored). A rectangle of block rows [r0, r1) x block columns [c0, c1) is first shrunk to the
// bounding box of its non-empty blocks; holding p > 1 ranks it is cut in two -- the first part
// (lower rows or columns) gets p / 2 ranks with the lower rank numbers, the second p - p / 2 --
// across its longer side in matrix rows (rows on ties; a side of one block is never cut) at the
// line k in [1, L - 1] minimising |W(first k lines) * p - W(rect) * (p / 2)| (the smaller k on
// ties). An empty rectangle, or a single block, goes whole to its first rank; the other ranks get
// empty rectangles (0, 0, 0, 0). A rank's tiles touch only the panel segments of its own row and
// column ranges instead of the whole prefix a block-row slab reaches into. out: world x (r0, r1,
// c0, c1).
std::vector<index_t> dist_tiles2d(const index_t* w, index_t nblk, const index_t* bounds, int world) {
    if (world < 1) fail(BE_ERR_BAD_PARAMS, "dist_tiles2d: world must be positive");
    if (nblk < 1) fail(BE_ERR_BAD_PARAMS, "dist_tiles2d: empty block grid");
    for (index_t i = 0; i < nblk * nblk; ++i)
        if (w[i] < 0) fail(BE_ERR_BAD_PARAMS, "dist_tiles2d: negative weight");
    std::vector<index_t> out(static_cast<std::size_t>(world) * 4, 0);
    auto W = [&](index_t bi, index_t bj) { return bj <= bi ? w[bi * nblk + bj] : index_t{0}; };
    std::function<void(index_t, index_t, index_t, index_t, int, int)> rec =
        [&](index_t r0, index_t r1, index_t c0, index_t c1, int p, int rank0) {
            index_t rl = r1, rh = r0, cl = c1, ch = c0;
            for (index_t bi = r0; bi < r1; ++bi)
                for (index_t bj = c0; bj < c1; ++bj)
                    if (W(bi, bj) > 0) {
                        rl = std::min(rl, bi), rh = std::max(rh, bi + 1);
                        cl = std::min(cl, bj), ch = std::max(ch, bj + 1);
                    }
            if (rl >= rh) return;  // empty: every rank of it keeps (0, 0, 0, 0)
            r0 = rl, r1 = rh, c0 = cl, c1 = ch;
            if (p == 1 || (r1 - r0 < 2 && c1 - c0 < 2)) {
                auto* o = out.data() + static_cast<std::size_t>(rank0) * 4;
                o[0] = r0, o[1] = r1, o[2] = c0, o[3] = c1;
                return;
            }
            const bool by_rows = c1 - c0 < 2 || (r1 - r0 >= 2 && bounds[r1] - bounds[r0] >= bounds[c1] - bounds[c0]);
            const index_t L = by_rows ? r1 - r0 : c1 - c0;
            std::vector<__int128> line(static_cast<std::size_t>(L), 0);
            __int128 tot = 0;
            for (index_t bi = r0; bi < r1; ++bi)
                for (index_t bj = c0; bj < c1; ++bj) {
                    const index_t x = W(bi, bj);
                    line[static_cast<std::size_t>(by_rows ? bi - r0 : bj - c0)] += x;
                    tot += x;
                }
            const int pl = p / 2;
            const __int128 target = tot * pl;
            __int128 pre = 0, bestd = -1;
            index_t best = 1;
            for (index_t k = 1; k < L; ++k) {
                pre += line[static_cast<std::size_t>(k - 1)];
                __int128 d = pre * p - target;
                if (d < 0) d = -d;
                if (bestd < 0 || d < bestd) bestd = d, best = k;
            }
            if (by_rows) {
                rec(r0, r0 + best, c0, c1, pl, rank0);
                rec(r0 + best, r1, c0, c1, p - pl, rank0 + pl);
            } else {
                rec(r0, r1, c0, c0 + best, pl, rank0);
                rec(r0, r1, c0 + best, c1, p - pl, rank0 + pl);
            }
        };
    rec(0, nblk, 0, nblk, world, 0);
    return out;
}

// Contiguous weight balance: cut p = first item index whose prefix weight
// reaches total * p / world. Slabs may be empty; the result is item indices.
std::vector<index_t> dist_balance(const index_t* w, index_t nitems, int world) {
    if (world < 1) fail(BE_ERR_BAD_PARAMS, "dist_balance: world must be positive");
    std::vector<index_t> cuts(static_cast<std::size_t>(world) + 1, nitems);
    cuts[0] = 0;
    __int128 total = 0;
    for (index_t i = 0; i < nitems; ++i) {
        if (w[i] < 0) fail(BE_ERR_BAD_PARAMS, "dist_balance: negative weight");
        total += w[i];
    }
    __int128 pre = 0;
    index_t i = 0;
    for (int p = 1; p < world; ++p) {
        const __int128 target = total * p;
        while (i < nitems && pre * world < target) pre += w[i++];
        cuts[static_cast<std::size_t>(p)] = i;
    }
    return cuts;
}

std::unique_ptr<Op> op_create_dist(Ctx* ctx, Comm* comm, const be_csb_view& L, const index_t* cuts,
                                   const int* owner, const double* diag_local, int values_prec) {
    validate_view(L);
    if (!comm) fail(BE_ERR_BAD_PARAMS, "distributed operator: null communicator");
    if (values_prec != BE_F32) fail(BE_ERR_BAD_PARAMS, "distributed operator: f32 values only");
    if (L.nrows != L.ncols) fail(BE_ERR_DIMENSION_MISMATCH, "SymmetricOperator: matrix must be square");
    if (L.nrowblks != L.ncolblks) fail(BE_ERR_DIMENSION_MISMATCH, "distributed operator: row and column blocks differ");
    for (index_t i = 0; i <= L.nrowblks; ++i)
        if (L.row_offsets[i] != L.col_offsets[i])
            fail(BE_ERR_DIMENSION_MISMATCH, "distributed operator: row and column blocks differ");
    if (!is_strictly_lower(L)) fail(BE_ERR_NOT_STRICTLY_LOWER, "SymmetricOperator: stored entry with row <= col");
    const int world = comm->world, rank = comm->rank;
    if (cuts[0] != 0 || cuts[world] != L.nrows) fail(BE_ERR_BAD_PARAMS, "distributed operator: cuts must cover [0, n)");
    for (int p = 0; p < world; ++p) {
        if (cuts[p + 1] < cuts[p]) fail(BE_ERR_BAD_PARAMS, "distributed operator: cuts must be non-decreasing");
        const index_t* e = std::lower_bound(L.row_offsets, L.row_offsets + L.nrowblks + 1, cuts[p]);
        if (e == L.row_offsets + L.nrowblks + 1 || *e != cuts[p])
            fail(BE_ERR_MISALIGNED_TILES, "distributed operator: cut " + std::to_string(cuts[p]) + " is not a block boundary");
    }
    auto op = std::make_unique<Op>();
    op->ctx = ctx;
    op->comm = comm;
    op->rank = rank;
    op->world = world;
    op->cuts.assign(cuts, cuts + world + 1);
    // segment owners: a permutation of the ranks (identity when not given)
    op->owner.resize(static_cast<std::size_t>(world));
    op->seg_of_rank.assign(static_cast<std::size_t>(world), -1);
    for (int q = 0; q < world; ++q) {
        const int o = owner ? owner[q] : q;
        if (o < 0 || o >= world || op->seg_of_rank[static_cast<std::size_t>(o)] >= 0)
            fail(BE_ERR_BAD_PARAMS, "distributed operator: segment owners must be a permutation of the ranks");
        op->owner[static_cast<std::size_t>(q)] = o;
        op->seg_of_rank[static_cast<std::size_t>(o)] = q;
    }
    op->lmax = 1;
    for (int p = 0; p < world; ++p) op->lmax = std::max(op->lmax, cuts[p + 1] - cuts[p]);
    const int mine = op->seg_of_rank[static_cast<std::size_t>(rank)];
    op->row_lo = cuts[mine];
    op->nlocal = cuts[mine + 1] - cuts[mine];
    if (op->lmax * world >= (index_t{1} << 31)) fail(BE_ERR_BAD_PARAMS, "distributed operator: padded dimension exceeds 2^31");
    op->nrows = op->ncols = op->nlocal;
    op->nnz = L.nnz;
    op->values_prec = values_prec;
    op->symmetric = true;
    RowMap map;
    map.cuts = op->cuts.data();
    map.owner = op->owner.data();
    map.world = world;
    map.rank = rank;
    map.lmax = op->lmax;
    op_build(op.get(), L, &map);
    {  // every rank's touched slots (one allreduce at setup)
        const std::size_t w2 = static_cast<std::size_t>(world) * world;
        std::vector<double> h(w2, 0.0);
        for (int r = 0; r < world; ++r) h[static_cast<std::size_t>(rank) * world + r] = op->touched[static_cast<std::size_t>(r)];
        DBuf<double> dv(static_cast<index_t>(w2));
        cudaStream_t cs = ctx->stream;
        BE_CUDA(cudaMemcpyAsync(dv.get(), h.data(), w2 * 8, cudaMemcpyHostToDevice, cs));
        comm->allreduce_f64(dv.get(), w2, cs);
        BE_CUDA(cudaMemcpyAsync(h.data(), dv.get(), w2 * 8, cudaMemcpyDeviceToHost, cs));
        comm->sync(cs);
        op->need.assign(w2, 0);
        for (std::size_t i = 0; i < w2; ++i) op->need[i] = h[i] > 0.5 ? 1 : 0;
    }
    op->diag.reset(std::max<index_t>(op->nlocal, 1));
    if (op->nlocal > 0) {
        if (!diag_local) fail(BE_ERR_DIMENSION_MISMATCH, "SymmetricOperator: diagonal length mismatch");
        BE_CUDA(cudaMemcpy(op->diag.get(), diag_local, static_cast<std::size_t>(op->nlocal) * 8, cudaMemcpyHostToDevice));
    }
    return op;
}

}  // namespace be
