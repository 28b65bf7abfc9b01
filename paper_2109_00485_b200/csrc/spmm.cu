// Symmetric SpMM over the half-stored CSB_Coo Hamiltonian, sm_100a.
//
// Replaces SymmetricOperator::apply (kernels.hpp:357-371) = out.set_zero +
// spmm_notrans (kernels.hpp:290) + spmm_trans (kernels.hpp:302) + the
// diagonal pass (kernels.hpp:363-370). The reference reads every stored
// nonzero twice (once per pass); this kernel reads it once from HBM and
// applies it twice (A_ij X_j -> Y_i and A_ij X_i -> Y_j).
//
// Device format ("work tiles", built on upload from the CSB arrays):
//   every CSB block is cut into 128 x 128 sub-tiles aligned to the block
//   origin (a sub-tile with more than max_nnz entries is split by rows);
//   tiles are ordered by global tile-row. Per entry the HBM stream holds the
//   value (f32 or f64) + rc (u16: local row << 8 | local col) + cperm (u16:
//   column-order permutation): 4 + 2 + 2 = 8 bytes per stored nonzero in f32,
//   the reference's own "f32 value + 2 x u16" budget. Inside
//   a tile the rows are ordered by decreasing length (rank order) and so are
//   the columns of the column order; 256 bytes of per-tile row/column lengths
//   (u8, rank order) complete the format.
//
// Kernel: persistent CTAs of 256 threads pull work items ("runs": up to 32
//   consecutive tiles of one tile-row) from an atomic counter. Per run the
//   CTA stages X_I once (f32, in smem) and accumulates Y_I in smem; per tile
//   it stages X_J and the entry stream (coalesced loads, one round trip).
//   Warps 0-3 then run pass R (Y_I += A X_J: one lane per row rank, all nb
//   columns in registers) while warps 4-7 run pass C (Y_J += A^T X_I: one
//   lane per column rank, flushed with REDG.E.ADD.F32x4). Rank order keeps
//   the 32 lanes of a warp on rows of similar length (little divergence). X
//   rows live in 128-byte smem lines holding 128 / (nb * 4) replicas; lane L
//   reads its 16-byte chunks in the rotated order (i + L) % CH from replica
//   (L / CH) % REP, so the 8 lanes of every quarter-warp phase hit 8 distinct
//   bank groups whatever rows they gather.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>

#include "comm.hpp"
#include "device.hpp"

namespace be {

namespace {

#ifndef BE_SPMM_STAGES
#define BE_SPMM_STAGES 1  // tile staging buffers per CTA (1: copy/compute overlap comes from the other CTAs of the SM)
#endif
constexpr int kThreads = 256;
constexpr index_t kRunMax = 32;  // tiles per work item

template <typename TC>
struct Meta;
template <>
struct __align__(8) Meta<float> {
    float v;
    std::uint32_t off;  // low 16: byte offset of the X_J line, high 16: of the X_I line
};
template <>
struct __align__(16) Meta<double> {
    double v;
    std::uint32_t off;
    std::uint32_t pad;
};

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
#ifdef BE_SPMM_NOREP
    static constexpr int LINEB = RB;                                // one copy per row line
#else
    static constexpr int LINEB = RB < 128 ? 128 : RB;               // bytes per smem row line
#endif
    static constexpr int REP = LINEB / RB;                          // replicas per line
    static_assert(NBP % VEC == 0 && CH >= 1, "bad NBP");
};

// Stage rows [row0, row0 + nr) of X (TX, row-major, nb columns) into the
// replicated smem lines; all loads of a batch are in flight together.
template <int NBP, typename TC, typename TX>
__device__ __forceinline__ void stage_x(unsigned char* xs, const TX* __restrict__ X, int row0, int nr, int nb) {
    using G = XGeom<NBP, TC>;
    const TX* src = X + static_cast<std::int64_t>(row0) * nb;
    constexpr int EPC = 16 / sizeof(TX);  // TX elements per 16-byte chunk
    if constexpr ((NBP * sizeof(TX)) % 16 == 0) {
        if (nb == NBP) {
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
        const TC x = v < nb ? static_cast<TC>(__ldg(src + static_cast<std::int64_t>(r) * nb + v)) : TC(0);
        TC* line = reinterpret_cast<TC*>(xs + r * G::LINEB);
#pragma unroll
        for (int q = 0; q < G::REP; ++q) line[q * NBP + v] = x;
    }
}

// cp.async 16-byte global -> shared copy (LDGSTS), and its group fences
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Raw per-tile staging area (one of two pipeline stages): the entry stream
// in JDS order, the column permutation, the X_J rows and the rank lengths.
template <int NBP, typename TC, typename TV, typename TX>
struct Stage {
    // raw X_J rows (staged asynchronously when small; else loaded directly)
    static constexpr int XRAW = kTile * NBP * static_cast<int>(sizeof(TX));
#ifndef BE_SPMM_XRAW_MAX
#define BE_SPMM_XRAW_MAX 0  // X_J rows staged raw with the tile (cp.async) up to this size (0: loaded into the lines directly, which frees the smem for a third CTA per SM)
#endif
    static constexpr int XB = XRAW <= BE_SPMM_XRAW_MAX ? XRAW : 0;
    __host__ __device__ static std::size_t bytes(int max_nnz) {
        return static_cast<std::size_t>(max_nnz) * (sizeof(TV) + 4) + XB + 256;
    }
};

// Issue the asynchronous copies of one tile into a stage buffer.
template <int NBP, typename TC, typename TV, typename TX>
__device__ __forceinline__ void stage_issue(unsigned char* st, int max_nnz, const TileHdr& h, int t,
                                            const unsigned char* __restrict__ lens, const TV* __restrict__ vals,
                                            const std::uint16_t* __restrict__ rc,
                                            const std::uint16_t* __restrict__ cperm, const TX* __restrict__ X,
                                            int nb, bool do_r, bool do_c, bool xvec) {
    const std::int64_t b = static_cast<std::int64_t>(h.begin8) * 8;
    const int nnz = static_cast<int>(h.packed >> 14);
    const int nc = static_cast<int>((h.packed >> 7) & 127u) + 1;
    const int npad = (nnz + 7) & ~7;
    TV* sv = reinterpret_cast<TV*>(st);
    std::uint16_t* src = reinterpret_cast<std::uint16_t*>(sv + max_nnz);
    std::uint16_t* scp = src + max_nnz;
    unsigned char* sx = reinterpret_cast<unsigned char*>(scp + max_nnz);
    unsigned char* sl = sx + Stage<NBP, TC, TV, TX>::XB;
    const int cv = npad * static_cast<int>(sizeof(TV)) / 16, cr = npad * 2 / 16;
    const int cx = (do_r && xvec) ? nc * nb * static_cast<int>(sizeof(TX)) / 16 : 0;
    const int total = cv + cr + (do_c ? cr : 0) + cx + 16;
    const unsigned char* gx = reinterpret_cast<const unsigned char*>(X + static_cast<std::int64_t>(h.col0) * nb);
    for (int c = threadIdx.x; c < total; c += kThreads) {
        int q = c;
        if (q < cv) { cp16(reinterpret_cast<unsigned char*>(sv) + 16 * q, reinterpret_cast<const unsigned char*>(vals + b) + 16 * q); continue; }
        q -= cv;
        if (q < cr) { cp16(reinterpret_cast<unsigned char*>(src) + 16 * q, reinterpret_cast<const unsigned char*>(rc + b) + 16 * q); continue; }
        q -= cr;
        if (do_c) {
            if (q < cr) { cp16(reinterpret_cast<unsigned char*>(scp) + 16 * q, reinterpret_cast<const unsigned char*>(cperm + b) + 16 * q); continue; }
            q -= cr;
        }
        if (q < cx) { cp16(sx + 16 * q, gx + 16 * q); continue; }
        q -= cx;
        cp16(sl + 16 * q, lens + static_cast<std::int64_t>(t) * 256 + 16 * q);
    }
}

// JDS starts: for the 128 ranks of one group (rows or columns) with lengths
// sorted in decreasing order, jd[j] = sum_r min(len_r, j) for j in [0, 128].
// Threads 0-127 build the row table, 128-255 the column table.
__device__ __forceinline__ void jds_starts(const unsigned char* sl, std::uint16_t* jd_r, std::uint16_t* jd_c,
                                           int* s_tot) {
    // threads 0-255 work (every thread of the CTA passes the barrier)
    const int tid = threadIdx.x, grp = (tid >> 7) & 1, j = tid & 127, lane = tid & 31, warp = tid >> 5;
    const unsigned char* len = sl + grp * 128;
    int cnt = 0, incl = 0;
    if (tid < 256) {
        int lo = 0, hi = 128;  // count_j = #ranks with len > j (lengths are non-increasing)
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (len[mid] > j) lo = mid + 1; else hi = mid;
        }
        cnt = lo;
        incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_tot[warp] = incl;
    }
    __syncthreads();
    if (tid < 256) {
        int start = incl - cnt;
        for (int w = grp * 4; w < warp; ++w) start += s_tot[w];
        std::uint16_t* jd = grp == 0 ? jd_r : jd_c;
        jd[j] = static_cast<std::uint16_t>(start);
        if (j == 127) jd[128] = static_cast<std::uint16_t>(start + cnt);
    }
}

// One work item = a run of consecutive tiles of the same 128-row tile-row.
// Per run the X_I slice is staged once (replicated lines) and Y_I rows
// accumulate in shared memory; per tile, the raw stream of tile t + 1 is
// copied with cp.async while tile t is computed. Pass R (warps 0-3): lane =
// row rank, walks its row through the JDS table; pass C (warps 4-7): lane =
// column rank, walks its column through cperm. Y_J is flushed per tile.
template <int NBP, typename TC, typename TV, typename TX>
#ifndef BE_SPMM_MINB32
#define BE_SPMM_MINB32 3  // CTAs per SM for 17 <= nb <= 64 (f32): 80 registers
#endif
#ifndef BE_SPMM_MINB
#define BE_SPMM_MINB 4  // CTAs per SM (nb <= 16, f32): 64 registers, 55 KB smem
#endif
__global__ void __launch_bounds__(kThreads, sizeof(TC) == 4 ? (NBP <= 16 ? BE_SPMM_MINB : BE_SPMM_MINB32) : 1)
    k_sym_spmm(const int2* __restrict__ runs, int nruns, const TileHdr* __restrict__ tiles,
               const unsigned char* __restrict__ lens, const TV* __restrict__ vals,
               const std::uint16_t* __restrict__ rc, const std::uint16_t* __restrict__ cperm,
               const TX* __restrict__ X, TX* __restrict__ Y, int nb, int do_r, int do_c, int max_nnz,
               int* __restrict__ ctr) {
    using G = XGeom<NBP, TC>;
    using V = typename Vec<TC>::T;
    using S = Stage<NBP, TC, TV, TX>;
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned char* xi = smem;
    unsigned char* xj = xi + kTile * G::LINEB;
    V* yi = reinterpret_cast<V*>(xj + kTile * G::LINEB);  // kTile x CH chunks: the run's Y_I rows
    unsigned char* stg0 = reinterpret_cast<unsigned char*>(yi + kTile * G::CH);
    const std::size_t sbytes = (S::bytes(max_nnz) + 15) & ~static_cast<std::size_t>(15);
    __shared__ __align__(8) std::uint16_t s_jd[2][136];  // read 4 starts at a time
    __shared__ int s_run;
    __shared__ int s_tot[8];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int grp = tid >> 7;  // 0: pass R (row ranks), 1: pass C (column ranks)
    const int rank = tid & 127;
    const bool vec_ok = (nb % G::VEC) == 0;
    const bool xvec = S::XB > 0 && nb == NBP && (NBP * sizeof(TX)) % 16 == 0 &&
                      (reinterpret_cast<std::uintptr_t>(X) & 15u) == 0;
    const unsigned char* xbase = (grp == 0 ? xj : xi) + ((lane / G::CH) % G::REP) * G::RB;
    int coff[G::CH];
#pragma unroll
    for (int i = 0; i < G::CH; ++i) coff[i] = ((i + lane) % G::CH) * 16;

    if (tid == 0) s_run = atomicAdd(ctr, 1);
    __syncthreads();
    int run = s_run;
    while (run < nruns) {
        const int2 rg = runs[run];
        TileHdr h = tiles[rg.x];
        const int row0 = h.row0;
        const int nr = static_cast<int>(h.packed & 127u) + 1;
        stage_issue<NBP, TC, TV, TX>(stg0, max_nnz, h, rg.x, lens, vals, rc, cperm, X, nb, do_r, do_c, xvec);
        cp_commit();
        if (do_c) stage_x<NBP, TC, TX>(xi, X, row0, nr, nb);
        if (do_r)
            for (int e = tid; e < kTile * G::CH; e += kThreads) vzero(yi[e]);
        for (int t = rg.x; t < rg.y; ++t) {
            unsigned char* st = stg0 + (BE_SPMM_STAGES == 2 ? ((t - rg.x) & 1) * sbytes : 0);
            const int nc = static_cast<int>((h.packed >> 7) & 127u) + 1;
            const int col0 = h.col0;
            cp_wait_all();
            __syncthreads();  // stage t complete and visible; stage t+1's buffer is free
            if (BE_SPMM_STAGES == 2 && t + 1 < rg.y) {
                h = tiles[t + 1];
                stage_issue<NBP, TC, TV, TX>(stg0 + ((t + 1 - rg.x) & 1) * sbytes, max_nnz, h, t + 1, lens, vals, rc,
                                             cperm, X, nb, do_r, do_c, xvec);
            }
            cp_commit();
            if (t == rg.y - 1 && tid == 0) s_run = atomicAdd(ctr, 1);  // next run
            const TV* sv = reinterpret_cast<const TV*>(st);
            const std::uint16_t* src = reinterpret_cast<const std::uint16_t*>(sv + max_nnz);
            const std::uint16_t* scp = src + max_nnz;
            const unsigned char* sx = reinterpret_cast<const unsigned char*>(scp + max_nnz);
            const unsigned char* sl = sx + S::XB;
            if (do_r) {  // X_J lines from the raw rows
                if (xvec) {
                    for (int e = tid; e < nc * NBP; e += kThreads) {
                        const int r = e / NBP, v = e % NBP;
                        const TC x = static_cast<TC>(reinterpret_cast<const TX*>(sx)[e]);
                        TC* line = reinterpret_cast<TC*>(xj + r * G::LINEB);
#pragma unroll
                        for (int q = 0; q < G::REP; ++q) line[q * NBP + v] = x;
                    }
                } else {
                    stage_x<NBP, TC, TX>(xj, X, col0, nc, nb);
                }
            }
            jds_starts(sl, s_jd[0], s_jd[1], s_tot);
            __syncthreads();
            const int len = sl[grp * 128 + rank];
            const bool active = len > 0 && (grp == 0 ? do_r : do_c);
            {
                const std::uint16_t* jd = s_jd[grp];
                V acc[G::CH];
#pragma unroll
                for (int i = 0; i < G::CH; ++i) vzero(acc[i]);
                int first = 0;
#ifndef BE_SPMM_UNR
#define BE_SPMM_UNR 4
#endif
                // the pass is warp-uniform: one copy of the walk per pass (no per-entry selects)
                auto walk = [&](auto pass) {
                    constexpr int GP = decltype(pass)::value;
                    for (int j0 = 0; j0 < len; j0 += BE_SPMM_UNR) {
                        int st4[4];  // starts j0 .. j0 + BE_SPMM_UNR - 1 in one shared-memory read
                        if constexpr (BE_SPMM_UNR == 4) {
                            const uint2 q4 = *reinterpret_cast<const uint2*>(jd + j0);
                            st4[0] = q4.x & 0xffffu, st4[1] = q4.x >> 16, st4[2] = q4.y & 0xffffu, st4[3] = q4.y >> 16;
                        } else if constexpr (BE_SPMM_UNR == 2) {
                            const unsigned q2 = *reinterpret_cast<const unsigned*>(jd + j0);
                            st4[0] = q2 & 0xffffu, st4[1] = q2 >> 16;
                        } else {
                            st4[0] = jd[j0];
                        }
#pragma unroll
                        for (int u = 0; u < BE_SPMM_UNR; ++u) {
                            if (j0 + u >= len) break;
                            int pos = st4[u] + rank;
                            if constexpr (GP == 1) pos = scp[pos];
                            const TC v = static_cast<TC>(sv[pos]);
                            const std::uint32_t x = src[pos];
                            if (j0 + u == 0) first = x;
                            const unsigned char* p = xbase + (GP == 0 ? (x & 255u) : (x >> 8)) * G::LINEB;
                            V xv[G::CH];
#pragma unroll
                            for (int i = 0; i < G::CH; ++i) xv[i] = *reinterpret_cast<const V*>(p + coff[i]);
#pragma unroll
                            for (int i = 0; i < G::CH; ++i) vfma(acc[i], v, xv[i]);
                        }
                    }
                };
                if (active) {
                    if (grp == 0) walk(std::integral_constant<int, 0>{});
                    else walk(std::integral_constant<int, 1>{});
                }
                if (active) {
                    if (grp == 0) {  // Y_I += A X_J for this row
                        V* y = yi + (first >> 8) * G::CH;
#pragma unroll
                        for (int i = 0; i < G::CH; ++i) vadd(y[(i + lane) % G::CH], acc[i]);
                    } else {  // Y_J += A^T X_I for this column
                        TX* y = Y + static_cast<std::int64_t>(col0 + (first & 255)) * nb;
#pragma unroll
                        for (int i = 0; i < G::CH; ++i) {
                            const int c0 = ((i + lane) % G::CH) * G::VEC;
                            if (c0 < nb) flush<TX>(y + c0, acc[i], nb - c0, vec_ok);
                        }
                    }
                }
            }
            if (BE_SPMM_STAGES == 1 && t + 1 < rg.y) {  // single buffer: refill after everyone is done with it
                __syncthreads();
                h = tiles[t + 1];
                stage_issue<NBP, TC, TV, TX>(stg0, max_nnz, h, t + 1, lens, vals, rc, cperm, X, nb, do_r, do_c, xvec);
                cp_commit();
            }
        }
        cp_wait_all();
        __syncthreads();
        if (do_r) {  // flush the run's rows (all-zero chunks carry no update)
            for (int e = tid; e < nr * G::CH; e += kThreads) {
                const int row = e / G::CH, c0 = (e % G::CH) * G::VEC;
                if (c0 < nb && vnonzero(yi[e]))
                    flush<TX>(Y + static_cast<std::int64_t>(row0 + row) * nb + c0, yi[e], nb - c0, vec_ok);
            }
        }
        run = s_run;
        __syncthreads();  // yi / xi / s_run are reused by the next run
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

template <int NBP, typename TC, typename TV, typename TX>
std::size_t smem_bytes(int max_nnz) {
    using G = XGeom<NBP, TC>;
    const std::size_t sb = (Stage<NBP, TC, TV, TX>::bytes(max_nnz) + 15) & ~static_cast<std::size_t>(15);
    return 2 * kTile * G::LINEB + kTile * G::CH * 16 + BE_SPMM_STAGES * sb;
}

template <int NBP, typename TC, typename TV, typename TX>
void launch_tiles(Op* op, const int2* runs, index_t nruns, const TX* X, TX* Y, int nb, int do_r, int do_c,
                  cudaStream_t s) {
    auto kern = k_sym_spmm<NBP, TC, TV, TX>;
    const std::size_t sm = smem_bytes<NBP, TC, TV, TX>(op->max_nnz);
    ensure_dyn_smem(kern, sm);
    int per_sm = 0;
    BE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, sm));
    if (per_sm < 1) fail(BE_ERR_CUDA, "sym_spmm: kernel does not fit on an SM");
    const int grid = static_cast<int>(std::min<index_t>(static_cast<index_t>(per_sm) * op->ctx->num_sms, nruns));
    op->grid = grid;
    if (grid == 0) return;
    kern<<<grid, kThreads, sm, s>>>(runs, static_cast<int>(nruns), op->tiles.get(), op->lens.get(),
                                    reinterpret_cast<const TV*>(op->vals.get()), op->rc.get(), op->cperm.get(), X, Y,
                                    nb, do_r, do_c, op->max_nnz, op->counter.get());
    BE_CUDA(cudaGetLastError());
    ++op->ctx->launches;
}

template <typename TC, typename TV, typename TX>
void dispatch_nb(Op* op, const int2* runs, index_t nruns, const TX* X, TX* Y, int nb, int do_r, int do_c,
                 cudaStream_t s) {
    constexpr int VEC = Vec<TC>::N;
    if (nb <= VEC) return launch_tiles<VEC, TC, TV, TX>(op, runs, nruns, X, Y, nb, do_r, do_c, s);
    if (nb <= 8) return launch_tiles<8, TC, TV, TX>(op, runs, nruns, X, Y, nb, do_r, do_c, s);
    if (nb <= 16) return launch_tiles<16, TC, TV, TX>(op, runs, nruns, X, Y, nb, do_r, do_c, s);
    if (nb <= 32) return launch_tiles<32, TC, TV, TX>(op, runs, nruns, X, Y, nb, do_r, do_c, s);
    if (nb <= 64) return launch_tiles<64, TC, TV, TX>(op, runs, nruns, X, Y, nb, do_r, do_c, s);
    fail(BE_ERR_BAD_PARAMS, "sym_spmm: nb > 64 is not supported by the device kernel");
}

// ---------------------------------------------------------------------------
// Tile-format build (host, parallel over CSB block rows).
// ---------------------------------------------------------------------------

struct RowOut {
    std::vector<TileHdr> hdr;         // begin8 relative to this block row
    std::vector<unsigned char> lens;  // 256 per tile: row then column lengths, rank order
    std::vector<double> v;            // values in device order (converted on upload)
    std::vector<std::uint16_t> rc, cp;
    std::vector<std::int64_t> src;    // CSB index per device entry (optional)
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

std::vector<std::uint16_t>& tls_colpos() {
    thread_local std::vector<std::uint16_t> v;
    return v;
}

// Emit one tile piece from `ent` = (local row << 56 | local col << 48 | CSB
// index), sorted by (row, col, index).
void emit_piece(const be_csb_view& L, const std::vector<std::uint64_t>& ent, index_t row0, index_t col0, index_t nr,
                index_t nc, bool keep_src, index_t& pos, RowOut& out) {
    const std::size_t n = ent.size();
    int rlen[kTile] = {0}, clen[kTile] = {0};
    for (std::uint64_t e : ent) {
        ++rlen[e >> 56];
        ++clen[(e >> 48) & 255u];
    }
    // rank order: decreasing length, ties by index
    int rorder[kTile], corder[kTile], rrank[kTile], crank[kTile];
    std::iota(rorder, rorder + kTile, 0);
    std::iota(corder, corder + kTile, 0);
    std::stable_sort(rorder, rorder + kTile, [&](int a, int b) { return rlen[a] > rlen[b]; });
    std::stable_sort(corder, corder + kTile, [&](int a, int b) { return clen[a] > clen[b]; });
    for (int i = 0; i < kTile; ++i) {
        rrank[rorder[i]] = i;
        crank[corder[i]] = i;
    }
    // row-JDS order: diagonal j holds the j-th entry (by column) of every row
    // rank with more than j entries; jd[j] = sum_r min(len_r, j)
    int rstart[kTile + 1], cstart[kTile + 1];  // ent is (row, col)-sorted: rows are contiguous
    rstart[0] = cstart[0] = 0;
    for (int i = 0; i < kTile; ++i) {
        rstart[i + 1] = rstart[i] + rlen[i];
        cstart[i + 1] = cstart[i] + clen[corder[i]];  // by column rank
    }
    const int rmax = rlen[rorder[0]], cmax = clen[corder[0]];
    std::vector<int> jd(static_cast<std::size_t>(rmax) + 1, 0), cjd(static_cast<std::size_t>(cmax) + 1, 0);
    for (int j = 0; j < rmax; ++j) {
        int cnt = 0;
        while (cnt < kTile && rlen[rorder[cnt]] > j) ++cnt;
        jd[static_cast<std::size_t>(j) + 1] = jd[static_cast<std::size_t>(j)] + cnt;
    }
    for (int j = 0; j < cmax; ++j) {
        int cnt = 0;
        while (cnt < kTile && clen[corder[cnt]] > j) ++cnt;
        cjd[static_cast<std::size_t>(j) + 1] = cjd[static_cast<std::size_t>(j)] + cnt;
    }
    TileHdr hd{};
    hd.begin8 = static_cast<std::uint32_t>(pos / 8);
    hd.row0 = static_cast<std::int32_t>(row0);
    hd.col0 = static_cast<std::int32_t>(col0);
    hd.packed = static_cast<std::uint32_t>(nr - 1) | (static_cast<std::uint32_t>(nc - 1) << 7) |
                (static_cast<std::uint32_t>(n) << 14);
    out.hdr.push_back(hd);
    for (int i = 0; i < kTile; ++i) out.lens.push_back(static_cast<unsigned char>(rlen[rorder[i]]));
    for (int i = 0; i < kTile; ++i) out.lens.push_back(static_cast<unsigned char>(clen[corder[i]]));
    const std::size_t base = out.v.size();
    out.v.resize(base + n);
    out.rc.resize(base + n);
    out.cp.resize(base + n);
    if (keep_src) out.src.resize(base + n);
    std::vector<std::uint16_t>& colpos = tls_colpos();
    colpos.resize(n);
    int ccur[kTile];
    std::copy(cstart, cstart + kTile, ccur);
    for (int r = 0; r < kTile; ++r) {
        const int row = rorder[r];
        for (int j = 0; j < rlen[row]; ++j) {
            const std::uint64_t e = ent[static_cast<std::size_t>(rstart[row] + j)];
            const int q = jd[static_cast<std::size_t>(j)] + r;
            const index_t k = static_cast<index_t>(e & 0xFFFFFFFFFFFFULL);
            out.v[base + static_cast<std::size_t>(q)] = L.values[k];
            out.rc[base + static_cast<std::size_t>(q)] = static_cast<std::uint16_t>(((e >> 56) << 8) | ((e >> 48) & 255u));
            if (keep_src) out.src[base + static_cast<std::size_t>(q)] = k;
            // column lists in (column rank, row rank) order
            colpos[static_cast<std::size_t>(ccur[crank[(e >> 48) & 255u]]++)] = static_cast<std::uint16_t>(q);
        }
    }
    // column-JDS order through cperm: cperm[cjd[j] + c] = row-JDS position of
    // the j-th entry of column rank c
    for (int c = 0; c < kTile; ++c)
        for (int j = 0; j < cstart[c + 1] - cstart[c]; ++j)
            out.cp[base + static_cast<std::size_t>(cjd[static_cast<std::size_t>(j)] + c)] =
                colpos[static_cast<std::size_t>(cstart[c] + j)];
    pos += static_cast<index_t>(n);
    while (pos % 8) {  // pad the segment to 8 entries
        out.v.push_back(0.0);
        out.rc.push_back(0);
        out.cp.push_back(0);
        if (keep_src) out.src.push_back(-1);
        ++pos;
    }
}

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
    index_t pos = 0;
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
                    emit_piece(L, piece, map ? map->pad(row0) : row0, map ? map->pad(col0) : col0, nr, nc, keep_src,
                               pos, out);
                    out.cls.push_back(static_cast<unsigned char>(pass));
                    p0 = p1;
                }
            }
        }
      }
    }
}

template <typename TV>
void upload_values(unsigned char* dst, const std::vector<double>& v) {
    if constexpr (sizeof(TV) == 8) {
        BE_CUDA(cudaMemcpy(dst, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(v.size());
        for (std::size_t i = 0; i < v.size(); ++i) f[i] = static_cast<float>(v[i]);
        BE_CUDA(cudaMemcpy(dst, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
    }
}

}  // namespace

static void op_build(Op* op, const be_csb_view& L, const RowMap* map);

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
    if (cstream) cudaStreamDestroy(cstream);
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
    op_build(op.get(), L, nullptr);
    if (op->symmetric) {
        op->diag.reset(std::max<index_t>(L.nrows, 1));
        if (L.nrows > 0)
            BE_CUDA(cudaMemcpy(op->diag.get(), diag, static_cast<std::size_t>(L.nrows) * 8, cudaMemcpyHostToDevice));
    }
    return op;
}

// Tile-format build + upload shared by the single- and multi-GPU operators.
static void op_build(Op* op, const be_csb_view& L, const RowMap* map) {
    const int values_prec = op->values_prec;
#ifndef BE_SPMM_MAXNNZ
#define BE_SPMM_MAXNNZ 1792  // f32 entries per tile piece (keeps four CTAs per SM)
#endif
    op->max_nnz = values_prec == BE_F32 ? BE_SPMM_MAXNNZ : 1024;
    const bool keep_src = L.nnz <= (index_t{1} << 26);

    std::vector<RowOut> rows(static_cast<std::size_t>(L.nrowblks));
    parallel_for_dynamic(hw_threads(), L.nrowblks, [&](index_t bi, int) {
        build_block_row(L, bi, op->max_nnz, keep_src, map, rows[static_cast<std::size_t>(bi)]);
    });
    index_t ntiles = 0, padded = 0;
    for (const auto& r : rows) {
        ntiles += static_cast<index_t>(r.hdr.size());
        padded += static_cast<index_t>(r.v.size());
    }
    if (padded / 8 >= (index_t{1} << 32)) fail(BE_ERR_BAD_PARAMS, "sym_spmm: too many entries for one device");
    op->ntiles = ntiles;
    op->padded = padded;
    const std::size_t vsz = values_prec == BE_F32 ? 4 : 8;
    op->tiles.reset(std::max<index_t>(ntiles, 1));
    op->lens.reset(std::max<index_t>(ntiles, 1) * 256);
    op->vals.reset(std::max<index_t>(padded, 8) * static_cast<index_t>(vsz));
    op->rc.reset(std::max<index_t>(padded, 8));
    op->cperm.reset(std::max<index_t>(padded, 8));
    op->counter.reset(2);
    BE_CUDA(cudaMemset(op->counter.get(), 0, 2 * sizeof(int)));
    if (keep_src) op->csb_index.reserve(static_cast<std::size_t>(padded));
    std::vector<TileHdr> all_hdr;
    all_hdr.reserve(static_cast<std::size_t>(ntiles));
    std::vector<unsigned char> all_cls;
    all_cls.reserve(static_cast<std::size_t>(ntiles));
    index_t t_off = 0, e_off = 0;
    for (auto& r : rows) {
        if (r.hdr.empty()) continue;
        for (auto& h : r.hdr) h.begin8 += static_cast<std::uint32_t>(e_off / 8);
        all_hdr.insert(all_hdr.end(), r.hdr.begin(), r.hdr.end());
        all_cls.insert(all_cls.end(), r.cls.begin(), r.cls.end());
        BE_CUDA(cudaMemcpy(op->lens.get() + t_off * 256, r.lens.data(), r.lens.size(), cudaMemcpyHostToDevice));
        if (values_prec == BE_F32)
            upload_values<float>(op->vals.get() + e_off * 4, r.v);
        else
            upload_values<double>(op->vals.get() + e_off * 8, r.v);
        BE_CUDA(cudaMemcpy(op->rc.get() + e_off, r.rc.data(), r.rc.size() * 2, cudaMemcpyHostToDevice));
        BE_CUDA(cudaMemcpy(op->cperm.get() + e_off, r.cp.data(), r.cp.size() * 2, cudaMemcpyHostToDevice));
        if (keep_src) op->csb_index.insert(op->csb_index.end(), r.src.begin(), r.src.end());
        t_off += static_cast<index_t>(r.hdr.size());
        e_off += static_cast<index_t>(r.v.size());
        r = RowOut();
    }
    if (ntiles > 0)
        BE_CUDA(cudaMemcpy(op->tiles.get(), all_hdr.data(), all_hdr.size() * sizeof(TileHdr), cudaMemcpyHostToDevice));
    {  // runs: consecutive tiles of one tile-row and class, at most kRunMax tiles each
        std::vector<int2> runs[2];
        for (index_t t = 0; t < ntiles;) {
            const auto& h0 = all_hdr[static_cast<std::size_t>(t)];
            const unsigned char c0 = all_cls[static_cast<std::size_t>(t)];
            index_t e = t + 1;
            while (e < ntiles && e - t < kRunMax && all_hdr[static_cast<std::size_t>(e)].row0 == h0.row0 &&
                   all_cls[static_cast<std::size_t>(e)] == c0)
                ++e;
            runs[c0].push_back(make_int2(static_cast<int>(t), static_cast<int>(e)));
            t = e;
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
static void op_apply_dist(Op* op, const double* X, double* Y, index_t in_rows, int nb, cudaStream_t s) {
    if (in_rows != op->nlocal) fail(BE_ERR_DIMENSION_MISMATCH, "distributed apply: local rows mismatch");
    const index_t seg = op->lmax * nb, tot = seg * op->world;
    if (op->x32.n < tot) {
        op->x32.reset(tot);
        op->y32.reset(tot);
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
    float* xs = op->x32.get() + static_cast<index_t>(op->rank) * seg;
    const int g = static_cast<int>(std::max<index_t>(1, std::min<index_t>((tot + 255) / 256, op->ctx->num_sms * 8)));
    k_f64_to_f32<<<g, 256, 0, s>>>(X, xs, op->nlocal * nb, op->y32.get(), tot);
    BE_CUDA(cudaGetLastError());
    ++op->ctx->launches;
    BE_CUDA(cudaEventRecord(op->ev_x, s));
    BE_CUDA(cudaStreamWaitEvent(op->cstream, op->ev_x, 0));
    op->comm->allgather_f32(xs, op->x32.get(), static_cast<std::size_t>(seg), op->cstream);
    BE_CUDA(cudaEventRecord(op->ev_ag, op->cstream));
    if (op->timing) BE_CUDA(cudaEventRecord(op->ev[1], s));
    if (op->nruns > 0)
        dispatch_nb<float, float, float>(op, op->runs.get(), op->nruns, op->x32.get(), op->y32.get(), nb, 1, 1, s);
    BE_CUDA(cudaStreamWaitEvent(s, op->ev_ag, 0));
    if (op->nruns_ext > 0)
        dispatch_nb<float, float, float>(op, op->runs_ext.get(), op->nruns_ext, op->x32.get(), op->y32.get(), nb, 1, 1,
                                         s);
    float* ys = op->y32.get() + static_cast<index_t>(op->rank) * seg;
    op->comm->reduce_scatter_f32(op->y32.get(), ys, static_cast<std::size_t>(seg), s);
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
    if (panel_prec == BE_F64 && op->values_prec == BE_F32) {
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
    op->diag.reset(std::max<index_t>(op->nlocal, 1));
    if (op->nlocal > 0) {
        if (!diag_local) fail(BE_ERR_DIMENSION_MISMATCH, "SymmetricOperator: diagonal length mismatch");
        BE_CUDA(cudaMemcpy(op->diag.get(), diag_local, static_cast<std::size_t>(op->nlocal) * 8, cudaMemcpyHostToDevice));
    }
    return op;
}

}  // namespace be
