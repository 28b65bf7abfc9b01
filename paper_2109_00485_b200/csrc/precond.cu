// Block-diagonal FOM preconditioner (precond.hpp), batched on the device.
//
// extract_tiles (precond.hpp:63-127) runs on the host and keeps the
// reference's SparseTile layout (for bit-exact checks); the upload re-packs
// every tile as CSR with the entries of a row in their original order, so the
// diagonal slot is the last entry of its row (the reference appends the
// diagonal slots after all couplings, precond.hpp:114-125) and the shift is
// folded into it exactly as fom_solve_column does (precond.hpp:154-156).
//
// Kernel: one CTA per (tile, group of gc columns). All gc columns of a tile
// run their m-step Lanczos-FOM (precond.hpp:143-257) in lock-step out of
// shared memory: thread t works on column t % gc over rows t / gc + k P.
// Dot products of all columns are reduced together, so a Lanczos step costs
// a handful of __syncthreads regardless of gc.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "precond.cuh"

namespace be {

namespace {

constexpr int kPT = 128;          // threads per CTA
constexpr int kMaxSteps = 64;     // cap on m (per-column alpha / beta / y arrays)
constexpr std::size_t kSmemBudget = 96 * 1024;

struct TileDev {
    std::int64_t row_off;  // global first row
    std::int32_t dim;
    std::int32_t ptr_off;  // into rowptr (dim + 1 entries)
    std::int64_t ent_off;  // into cols / vals
};

// block-wide sums of one value per column: v[t] for thread t, column t % gc
__device__ __forceinline__ void col_reduce(double v, double* red, double* out, int gc) {
    red[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x < gc) {
        double s = 0.0;
        for (int q = threadIdx.x; q < kPT; q += gc) s += red[q];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kPT) k_fom(const TileDev* __restrict__ tiles, const std::int32_t* __restrict__ rowptr,
                                             const std::uint16_t* __restrict__ cols, const double* __restrict__ vals,
                                             const double* __restrict__ shifts, const double* __restrict__ R,
                                             double* __restrict__ W, int nb, int m, int gc, int ngroups,
                                             std::int64_t* fallbacks, const std::int32_t* __restrict__ list) {
    extern __shared__ double sm[];
    __shared__ double red[kPT];
    __shared__ double s_dot[16], s_beta0[16], s_alpha[16][kMaxSteps], s_beta[16][kMaxSteps], s_y[16][kMaxSteps];
    __shared__ int s_steps[16], s_live[16], s_sing[16];

    const int tile = list ? list[blockIdx.x / ngroups] : static_cast<int>(blockIdx.x / ngroups);
    const int grp = blockIdx.x % ngroups;
    const TileDev td = tiles[tile];
    const int d = td.dim;
    const int cap = min(m, d);
    const int c = threadIdx.x % gc;           // column within the group
    const int part = threadIdx.x / gc, P = kPT / gc;
    const int col = grp * gc + c;             // global column
    const bool colok = col < nb;
    // smem: per column: V[cap][d] then w[d]
    double* V = sm + static_cast<std::size_t>(c) * (cap + 1) * d;
    double* w = V + static_cast<std::size_t>(cap) * d;
    const std::int32_t* rp = rowptr + td.ptr_off;
    const std::uint16_t* cl = cols + td.ent_off;
    const double* vl = vals + td.ent_off;
    const double sigma = colok ? shifts[col] : 0.0;

    // beta0 = ||r||, V0 = r
    double acc = 0.0;
    for (int i = part; i < d; i += P) {
        const double x = colok ? R[(td.row_off + i) * nb + col] : 0.0;
        V[i] = x;
        acc += x * x;
    }
    col_reduce(acc, red, s_dot, gc);
    if (threadIdx.x < gc) {
        s_beta0[threadIdx.x] = sqrt(s_dot[threadIdx.x]);
        s_steps[threadIdx.x] = cap;
        s_live[threadIdx.x] = s_beta0[threadIdx.x] != 0.0;
        s_sing[threadIdx.x] = 0;
    }
    __syncthreads();
    const double beta0 = s_beta0[c];
    if (s_live[c])
        for (int i = part; i < d; i += P) V[i] = V[i] / beta0;
    __syncthreads();

    for (int s = 0; s < cap; ++s) {
        const bool live = s_live[c] != 0;
        const double* vs = V + static_cast<std::size_t>(s) * d;
        // w = (K - sigma I) V_s ; alpha_s = V_s . w
        acc = 0.0;
        if (live)
            for (int i = part; i < d; i += P) {
                double y = 0.0;
                const int e1 = rp[i + 1] - 1;  // the diagonal slot is last
                for (int e = rp[i]; e < e1; ++e) y += vl[e] * vs[cl[e]];
                y += (vl[e1] - sigma) * vs[i];
                w[i] = y;
                acc += vs[i] * y;
            }
        col_reduce(acc, red, s_dot, gc);
        if (threadIdx.x < gc && s_live[threadIdx.x]) s_alpha[threadIdx.x][s] = s_dot[threadIdx.x];
        if (s + 1 == cap) break;
        const double a = s_dot[c];
        if (live) {
            const double bprev = s > 0 ? s_beta[c][s - 1] : 0.0;
            const double* vp = s > 0 ? V + static_cast<std::size_t>(s - 1) * d : vs;
            for (int i = part; i < d; i += P) {
                double x = w[i] - a * vs[i];
                if (s > 0) x -= bprev * vp[i];
                w[i] = x;
            }
        }
        __syncthreads();
        for (int t = 0; t <= s; ++t) {  // one reorthogonalisation pass, in order
            const double* vt = V + static_cast<std::size_t>(t) * d;
            acc = 0.0;
            if (live)
                for (int i = part; i < d; i += P) acc += vt[i] * w[i];
            col_reduce(acc, red, s_dot, gc);
            const double pr = s_dot[c];
            if (live)
                for (int i = part; i < d; i += P) w[i] -= pr * vt[i];
            __syncthreads();
        }
        acc = 0.0;
        if (live)
            for (int i = part; i < d; i += P) acc += w[i] * w[i];
        col_reduce(acc, red, s_dot, gc);
        if (threadIdx.x < gc && s_live[threadIdx.x]) {
            const double nw = sqrt(s_dot[threadIdx.x]);
            if (nw < 1e-14 * s_beta0[threadIdx.x]) {  // Krylov breakdown
                s_steps[threadIdx.x] = s + 1;
                s_live[threadIdx.x] = 0;
            } else {
                s_beta[threadIdx.x][s] = nw;
            }
        }
        __syncthreads();
        if (s_live[c]) {
            const double nw = s_beta[c][s];
            double* vn = V + static_cast<std::size_t>(s + 1) * d;
            for (int i = part; i < d; i += P) vn[i] = w[i] / nw;
        }
        __syncthreads();
    }
    __syncthreads();
    // T y = beta0 e1 by LU with partial pivoting (precond.hpp:208-249); the
    // s x s system of column cc lives in shared memory after the basis
    if (threadIdx.x < gc && s_beta0[threadIdx.x] != 0.0) {
        const int cc = threadIdx.x;
        const int st = s_steps[cc];
        double* Td = sm + static_cast<std::size_t>(gc) * (cap + 1) * d + static_cast<std::size_t>(cc) * cap * cap;
        auto T = [&](int i, int j) -> double& { return Td[j * st + i]; };
        double tmax = 0.0;
        for (int i = 0; i < st * st; ++i) Td[i] = 0.0;
        for (int i = 0; i < st; ++i) {
            T(i, i) = s_alpha[cc][i];
            tmax = fmax(tmax, fabs(T(i, i)));
            if (i + 1 < st) {
                T(i, i + 1) = T(i + 1, i) = s_beta[cc][i];
                tmax = fmax(tmax, fabs(s_beta[cc][i]));
            }
        }
        const double floor = 1e-14 * fmax(1.0, tmax);
        double* y = s_y[cc];
        for (int i = 0; i < st; ++i) y[i] = 0.0;
        y[0] = s_beta0[cc];
        bool sing = false;
        for (int k = 0; k < st; ++k) {
            int piv = k;
            for (int i = k + 1; i < st; ++i)
                if (fabs(T(i, k)) > fabs(T(piv, k))) piv = i;
            if (fabs(T(piv, k)) < floor) {
                sing = true;
                break;
            }
            if (piv != k) {
                for (int j = 0; j < st; ++j) {
                    const double tmp = T(k, j);
                    T(k, j) = T(piv, j);
                    T(piv, j) = tmp;
                }
                const double tmp = y[k];
                y[k] = y[piv];
                y[piv] = tmp;
            }
            for (int i = k + 1; i < st; ++i) {
                const double f = T(i, k) / T(k, k);
                if (f == 0.0) continue;
                for (int j = k; j < st; ++j) T(i, j) -= f * T(k, j);
                y[i] -= f * y[k];
            }
        }
        if (!sing)
            for (int i = st - 1; i >= 0; --i) {
                double a2 = y[i];
                for (int j = i + 1; j < st; ++j) a2 -= T(i, j) * y[j];
                y[i] = a2 / T(i, i);
            }
        s_sing[cc] = sing ? 1 : 0;
        if (sing && col < nb && fallbacks) atomicAdd(reinterpret_cast<unsigned long long*>(fallbacks), 1ull);
    }
    __syncthreads();
    if (!colok) return;
    const double b0 = s_beta0[c];
    const int st = s_steps[c];
    for (int i = part; i < d; i += P) {
        double out = 0.0;
        if (b0 != 0.0) {
            if (s_sing[c]) {
                out = R[(td.row_off + i) * nb + col];  // unpreconditioned fallback column
            } else {
                for (int j = 0; j < st; ++j) out += s_y[c][j] * V[static_cast<std::size_t>(j) * d + i];
            }
        }
        W[(td.row_off + i) * nb + col] = out;
    }
}

// One CTA of NT threads per (tile, group of C columns): the C columns run
// their m-step FOM (precond.hpp:143-257) in lock-step. Thread t owns a chunk
// of CW = 4 adjacent columns (chunk t % (C / 4)) of rows t / (C / 4) + k RL,
// k < RPT, so one fetched tile entry feeds CW FMAs and the gathered basis
// row segment is one 32-byte vector read. The Krylov basis V[s][row][col]
// lives in shared memory (the sparse product gathers arbitrary rows of V_s);
// w and the per-column Lanczos scalars stay in registers, replicated across
// the threads of a column chunk (every thread gets the bitwise-identical
// reduction result, so the tridiagonal solves run redundantly in registers).
// The tile's entries are staged in shared memory when they fit.
constexpr int kCW = 4;

template <int C, int NT>
__device__ __forceinline__ void block_colsum4(double (&v)[kCW], double (*red)[16], int& buf) {
    constexpr int NW = NT / 32, CQ = C / kCW;
    // lanes sharing a column chunk differ in the bits above log2(CQ)
#pragma unroll
    for (int o = CQ; o < 32; o <<= 1)
#pragma unroll
        for (int j = 0; j < kCW; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
    if constexpr (NW > 1) {
        // red rows: [buf][warp] partials, then row 2 * NW + buf: the per-column totals
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int cq = threadIdx.x % CQ;
        if (lane < CQ)
#pragma unroll
            for (int j = 0; j < kCW; ++j) red[buf * NW + warp][cq * kCW + j] = v[j];
        __syncthreads();
        if (threadIdx.x < C) {  // one thread per column sums the warps in order
            double t = red[buf * NW][threadIdx.x];
#pragma unroll
            for (int w = 1; w < NW; ++w) t += red[buf * NW + w][threadIdx.x];
            red[2 * NW + buf][threadIdx.x] = t;
        }
        __syncthreads();
        {
            const double2 p0 = reinterpret_cast<const double2*>(&red[2 * NW + buf][cq * kCW])[0];
            const double2 p1 = reinterpret_cast<const double2*>(&red[2 * NW + buf][cq * kCW])[1];
            v[0] = p0.x, v[1] = p0.y, v[2] = p1.x, v[3] = p1.y;
        }
        buf ^= 1;  // double-buffered: the next reduction cannot overwrite this one before all threads read it
    }
}

template <int NT>
__device__ __forceinline__ void block_sync() {
    if constexpr (NT == 32) __syncwarp(); else __syncthreads();
}

struct V4 {
    double a[kCW];
};
// A row of the C-column basis in shared memory is two halves of H = C / 2
// doubles; the 16-byte piece h of column chunk cq sits at h * H + cq * 2
// doubles. Row lanes of odd parity read (and write) their high piece first
// (hp = H), so the two rows of a quarter-warp phase hit opposite bank halves:
// gathers of arbitrary rows are conflict-free for C = 16 (64-byte halves);
// for C = 8 (32-byte halves) two of the four rows of a phase can share one.
template <int H>
__device__ __forceinline__ V4 ld4(const double* p, int hp) {  // p: row + cq * 2
    const double2 x = *reinterpret_cast<const double2*>(p + hp), y = *reinterpret_cast<const double2*>(p + (H - hp));
    return hp ? V4{{y.x, y.y, x.x, x.y}} : V4{{x.x, x.y, y.x, y.y}};
}
template <int H>
__device__ __forceinline__ void st4(double* p, const double (&v)[kCW], int hp) {
    const double2 lo = make_double2(v[0], v[1]), hi = make_double2(v[2], v[3]);
    *reinterpret_cast<double2*>(p + hp) = hp ? hi : lo;
    *reinterpret_cast<double2*>(p + (H - hp)) = hp ? lo : hi;
}

// x / b, correctly rounded, from r = 1 / b (one reciprocal per column
// instead of one IEEE division per element): q = x r, then one residual
// correction with the exact FMA remainder (Markstein).
__device__ __forceinline__ double div_rcp(double x, double b, double r) {
    const double q = x * r;
    return fma(fma(-q, b, x), r, q);
}

// T y = beta0 e1 for one column's m x m Lanczos tridiagonal: LU with partial
// pivoting and the singular-pivot flag (precond.hpp:208-249). UNR: every
// index unrolled (T and y stay in registers, m <= 4); else rolled loops.
template <int MC, bool UNR, int C>
__device__ __forceinline__ int tri_lu_solve(const double (*sa)[C], const double (*sb)[C], int cc, int st,
                                            double b0, double (&y)[MC]) {
    if constexpr (UNR) {
        double T[MC][MC];
        double tmax = 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i) {
            y[i] = 0.0;
#pragma unroll
            for (int q = 0; q < MC; ++q) T[i][q] = 0.0;
        }
#pragma unroll
        for (int i = 0; i < MC; ++i)
            if (i < st) {
                T[i][i] = sa[i][cc];
                tmax = fmax(tmax, fabs(sa[i][cc]));
                if (i + 1 < MC && i + 1 < st) {
                    T[i][i + 1 < MC ? i + 1 : 0] = sb[i][cc];
                    T[i + 1 < MC ? i + 1 : 0][i] = sb[i][cc];
                    tmax = fmax(tmax, fabs(sb[i][cc]));
                }
            }
        const double floor = 1e-14 * fmax(1.0, tmax);
        y[0] = b0;
        int sg = 0;
        bool go = true;
#pragma unroll
        for (int k = 0; k < MC; ++k) {
            if (!(go && k < st)) continue;
            int piv = k;
            double best = fabs(T[k][k]);
#pragma unroll
            for (int i = k + 1; i < MC; ++i)
                if (i < st && fabs(T[i][k]) > best) {
                    best = fabs(T[i][k]);
                    piv = i;
                }
            if (best < floor) {
                sg = 1;
                go = false;
                continue;
            }
#pragma unroll
            for (int i = k + 1; i < MC; ++i)
                if (i == piv) {
#pragma unroll
                    for (int q = 0; q < MC; ++q) {
                        const double tmp = T[k][q];
                        T[k][q] = T[i][q];
                        T[i][q] = tmp;
                    }
                    const double tmp = y[k];
                    y[k] = y[i];
                    y[i] = tmp;
                }
#pragma unroll
            for (int i = k + 1; i < MC; ++i) {
                if (i >= st) continue;
                const double f = T[i][k] / T[k][k];
                if (f == 0.0) continue;
#pragma unroll
                for (int q = k; q < MC; ++q)
                    if (q < st) T[i][q] -= f * T[k][q];
                y[i] -= f * y[k];
            }
        }
        if (!sg)
#pragma unroll
            for (int i = MC - 1; i >= 0; --i) {
                if (i >= st) continue;
                double a2 = y[i];
#pragma unroll
                for (int q = i + 1; q < MC; ++q)
                    if (q < st) a2 -= T[i][q] * y[q];
                y[i] = a2 / T[i][i];
            }
        return sg;
    } else {
        double T[MC][MC];
        double tmax = 0.0;
#pragma unroll 1
        for (int i = 0; i < MC; ++i) {
            y[i] = 0.0;
#pragma unroll 1
            for (int q = 0; q < MC; ++q) T[i][q] = 0.0;
        }
#pragma unroll 1
        for (int i = 0; i < MC; ++i)
            if (i < st) {
                T[i][i] = sa[i][cc];
                tmax = fmax(tmax, fabs(sa[i][cc]));
                if (i + 1 < MC && i + 1 < st) {
                    T[i][i + 1 < MC ? i + 1 : 0] = sb[i][cc];
                    T[i + 1 < MC ? i + 1 : 0][i] = sb[i][cc];
                    tmax = fmax(tmax, fabs(sb[i][cc]));
                }
            }
        const double floor = 1e-14 * fmax(1.0, tmax);
        y[0] = b0;
        int sg = 0;
        bool go = true;
#pragma unroll 1
        for (int k = 0; k < MC; ++k) {
            if (!(go && k < st)) continue;
            int piv = k;
            double best = fabs(T[k][k]);
#pragma unroll 1
            for (int i = k + 1; i < MC; ++i)
                if (i < st && fabs(T[i][k]) > best) {
                    best = fabs(T[i][k]);
                    piv = i;
                }
            if (best < floor) {
                sg = 1;
                go = false;
                continue;
            }
#pragma unroll 1
            for (int i = k + 1; i < MC; ++i)
                if (i == piv) {
#pragma unroll 1
                    for (int q = 0; q < MC; ++q) {
                        const double tmp = T[k][q];
                        T[k][q] = T[i][q];
                        T[i][q] = tmp;
                    }
                    const double tmp = y[k];
                    y[k] = y[i];
                    y[i] = tmp;
                }
#pragma unroll 1
            for (int i = k + 1; i < MC; ++i) {
                if (i >= st) continue;
                const double f = T[i][k] / T[k][k];
                if (f == 0.0) continue;
#pragma unroll 1
                for (int q = k; q < MC; ++q)
                    if (q < st) T[i][q] -= f * T[k][q];
                y[i] -= f * y[k];
            }
        }
        if (!sg)
#pragma unroll 1
            for (int i = MC - 1; i >= 0; --i) {
                if (i >= st) continue;
                double a2 = y[i];
#pragma unroll 1
                for (int q = i + 1; q < MC; ++q)
                    if (q < st) a2 -= T[i][q] * y[q];
                y[i] = a2 / T[i][i];
            }
        return sg;
    }
}

#ifdef BE_FOM_PROF  // development probe: per-phase clock cycles of thread 0, summed per size class
__device__ unsigned long long g_fom_prof[5][8];
#define BE_FOM_MARK(k)                                                                                     \
    do {                                                                                                   \
        if (threadIdx.x == 0) {                                                                            \
            const long long t_ = clock64();                                                                \
            atomicAdd(&g_fom_prof[NT == 32 ? 0 : NT == 128 ? 1 : (NT == 256 && RPT == 2) ? 2 : (NT == 256 && C == 16) ? 3 : 4][k], \
                      static_cast<unsigned long long>(t_ - prof_t));                                       \
            prof_t = t_;                                                                                   \
        }                                                                                                  \
    } while (0)
#else
#define BE_FOM_MARK(k) do {} while (0)
#endif

template <int MC, int NT, int RPT, bool VSM, int C>
__global__ void __launch_bounds__(NT, NT == 32 ? 8 : (NT >= 512 ? 1 : 2))
    k_fom_blk(const TileDev* __restrict__ tiles, const std::int32_t* __restrict__ list,
              const std::int32_t* __restrict__ rowptr, const std::uint16_t* __restrict__ cols,
              const double* __restrict__ vals, const double* __restrict__ shifts, const double* __restrict__ R,
              double* __restrict__ W, int nb, int m, int ngroups, std::int64_t* fallbacks, int dmax, int stage_cap,
              double* __restrict__ Vg, std::int64_t nrows, unsigned* __restrict__ slot_mask, int kslots) {
    constexpr int CQ = C / kCW;  // column chunks per row
    constexpr int H = C / 2;     // half-row of the basis layout (ld4 / st4)
    constexpr int RL = NT / CQ;  // row lanes
    extern __shared__ __align__(16) double sV[];  // current basis vector [dmax][C], then the staged entries
    __shared__ __align__(16) double red[2 * (NT / 32) + 2][16];
    int rbuf = 0;
#ifdef BE_FOM_PROF
    long long prof_t = clock64();
#endif
    const int tile = list[blockIdx.x / ngroups];
    const int grp = blockIdx.x % ngroups;
    const int col0 = grp * C;
    const TileDev td = tiles[tile];
    const int d = td.dim;
    const int cap = min(m, d);
    const int cq = threadIdx.x % CQ, rl = threadIdx.x / CQ;
    const int c0 = col0 + cq * kCW;  // first global column of the chunk
    const std::int32_t* rp = rowptr + td.ptr_off;
    const std::uint16_t* gcl = cols + td.ent_off;
    const double* gvl = vals + td.ent_off;
    double sigma[kCW];
    bool colok[kCW];
#pragma unroll
    for (int j = 0; j < kCW; ++j) {
        colok[j] = c0 + j < nb;
        sigma[j] = colok[j] ? shifts[c0 + j] : 0.0;
    }
    const double* r = R + td.row_off * nb + c0;
    // VSM: the whole basis V[q][row][C] in shared memory. Otherwise only the
    // current vector is (the gathers need it) and the older ones, read back
    // at this thread's own rows only, live in a per-SM scratch slot that stays
    // in L2 (the launch guarantees one CTA per SM).
    const std::size_t vstride = static_cast<std::size_t>(dmax) * C;
    double* Vcur = sV + cq * 2;  // this chunk's low piece (see ld4)
    const int hp = NT == 32 ? 0 : (rl & 1) * H;  // (the one-warp class is not shared-memory bound)
    double* Vslot = nullptr;
    __shared__ int s_slot;
    unsigned smid = 0;
    if constexpr (!VSM) {  // claim one of the SM's kslots scratch slots (released at exit)
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (threadIdx.x == 0) {
            int k = 0;
            for (;;) {
                const unsigned bit = 1u << k;
                if (!(atomicOr(slot_mask + smid, bit) & bit)) break;
                k = k + 1 == kslots ? 0 : k + 1;
            }
            s_slot = static_cast<int>(smid) * kslots + k;
        }
        __syncthreads();
        Vslot = Vg + static_cast<std::size_t>(s_slot) * MC * vstride + cq * 2;
    }
    auto vg = [&](int q, int i) -> double* {
        if constexpr (VSM) return Vcur + q * vstride + static_cast<std::size_t>(i) * C;
        else return Vslot + q * vstride + static_cast<std::size_t>(i) * C;
    };
    double* Vc = Vcur;  // current vector (advanced per step when VSM)
    // the tile's entries are read cap times: stage them after the basis
    const int nent = __ldg(rp + d);
    double* s_vl = sV + (VSM ? static_cast<std::size_t>(min(m, MC)) : 1) * vstride;
    std::uint16_t* s_cl = reinterpret_cast<std::uint16_t*>(s_vl + stage_cap);
    const bool staged = nent <= stage_cap;
    if (staged)  // eight loads in flight per thread before the stores
        for (int e0 = threadIdx.x; e0 < nent; e0 += 8 * NT) {
            double v[8];
            std::uint16_t c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NT;
                if (e < nent) {
                    v[u] = __ldg(gvl + e);
                    c[u] = __ldg(gcl + e);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NT;
                if (e < nent) {
                    s_vl[e] = v[u];
                    s_cl[e] = c[u];
                }
            }
        }

    int eb[RPT], ee[RPT];  // row i's entries [eb, ee), its diagonal at ee
    double w[RPT][kCW];  // V_s and V_{s-1} are re-read (shared memory / the CTA's slot), not held
    double acc[kCW] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int i = rl + k * RL;
        eb[k] = ee[k] = 0;
#pragma unroll
        for (int j = 0; j < kCW; ++j) w[k][j] = 0.0;
        if (i < d) {
            eb[k] = __ldg(rp + i);
            ee[k] = __ldg(rp + i + 1) - 1;  // the diagonal slot is last
#pragma unroll
            for (int j = 0; j < kCW; ++j) {
                const double x = colok[j] ? r[static_cast<std::int64_t>(i) * nb + j] : 0.0;
                w[k][j] = x;
                acc[j] += x * x;
            }
        }
    }
    block_colsum4<C, NT>(acc, red, rbuf);
    BE_FOM_MARK(0);
    double beta0[kCW], inv[kCW], rinv[kCW];
#pragma unroll
    for (int j = 0; j < kCW; ++j) {
        beta0[j] = sqrt(acc[j]);
        inv[j] = beta0[j] != 0.0 ? beta0[j] : 1.0;
        rinv[j] = 1.0 / inv[j];
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int i = rl + k * RL;
        if (i < d) {
            double v[kCW];
#pragma unroll
            for (int j = 0; j < kCW; ++j) v[j] = div_rcp(w[k][j], inv[j], rinv[j]);
            st4<H>(Vc + static_cast<std::size_t>(i) * C, v, hp);
            if constexpr (!VSM) st4<H>(vg(0, i), v, hp);
        }
    }
    // Lanczos scalars of the CTA's columns (written by row lane 0; every
    // thread holds the same values)
    __shared__ double s_alpha[MC][C], s_beta[MC][C];
    __shared__ int s_steps[C];
    double bprev[kCW] = {0.0, 0.0, 0.0, 0.0};
    int steps[kCW];
    bool live[kCW];
#pragma unroll
    for (int j = 0; j < kCW; ++j) {
        steps[j] = cap;
        live[j] = beta0[j] != 0.0;
    }
    if (rl == 0)
        for (int s2 = 0; s2 < MC; ++s2)
#pragma unroll
            for (int j = 0; j < kCW; ++j) s_alpha[s2][cq * kCW + j] = s_beta[s2][cq * kCW + j] = 0.0;
#pragma unroll 1
    for (int s = 0; s < MC; ++s) {
        if (s >= cap) break;
        block_sync<NT>();  // V_s (and the staged entries) complete
        // w = (K - sigma I) V_s ; alpha_s = V_s . w
#pragma unroll
        for (int j = 0; j < kCW; ++j) acc[j] = 0.0;
        // the entries' address space is fixed per copy (a select between the
        // staged and the global arrays would force generic loads)
        auto matvec = [&](const double* __restrict__ vl, const std::uint16_t* __restrict__ cl) {
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int i = rl + k * RL;
                double y[kCW] = {0.0, 0.0, 0.0, 0.0};
                if (i < d) {
                    int e = eb[k];
                    for (; e + 1 < ee[k]; e += 2) {
                        const double a0 = vl[e], a1 = vl[e + 1];
                        const V4 x0 = ld4<H>(Vc + static_cast<int>(cl[e]) * C, hp);
                        const V4 x1 = ld4<H>(Vc + static_cast<int>(cl[e + 1]) * C, hp);
#pragma unroll
                        for (int j = 0; j < kCW; ++j) y[j] += a0 * x0.a[j];
#pragma unroll
                        for (int j = 0; j < kCW; ++j) y[j] += a1 * x1.a[j];
                    }
                    if (e < ee[k]) {
                        const double a0 = vl[e];
                        const V4 x0 = ld4<H>(Vc + static_cast<int>(cl[e]) * C, hp);
#pragma unroll
                        for (int j = 0; j < kCW; ++j) y[j] += a0 * x0.a[j];
                    }
                    const V4 v = ld4<H>(Vc + static_cast<std::size_t>(i) * C, hp);
                    const double dg = vl[ee[k]];
#pragma unroll
                    for (int j = 0; j < kCW; ++j) {
                        y[j] += (dg - sigma[j]) * v.a[j];
                        acc[j] += v.a[j] * y[j];
                    }
                }
#pragma unroll
                for (int j = 0; j < kCW; ++j) w[k][j] = y[j];
            }
        };
        if (staged) matvec(s_vl, s_cl);
        else matvec(gvl, gcl);
        block_colsum4<C, NT>(acc, red, rbuf);
        BE_FOM_MARK(1);
        double a[kCW];
#pragma unroll
        for (int j = 0; j < kCW; ++j) {
            a[j] = acc[j];
            if (live[j] && rl == 0) s_alpha[s][cq * kCW + j] = a[j];
        }
        if (s + 1 == cap) break;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int i = rl + k * RL;
            if (i >= d) continue;
            const V4 vs = ld4<H>(Vc + static_cast<std::size_t>(i) * C, hp);
            const V4 vp = s > 0 ? ld4<H>(vg(s - 1, i), hp) : V4{{0.0, 0.0, 0.0, 0.0}};
#pragma unroll
            for (int j = 0; j < kCW; ++j) {
                double x = w[k][j] - a[j] * vs.a[j];
                if (s > 0) x -= bprev[j] * vp.a[j];
                w[k][j] = x;
            }
        }
        for (int q = 0; q <= s; ++q) {  // one reorthogonalisation pass, in order
#pragma unroll
            for (int j = 0; j < kCW; ++j) acc[j] = 0.0;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int i = rl + k * RL;
                if (i < d) {
                    const V4 v = (q == s ? ld4<H>(Vc + static_cast<std::size_t>(i) * C, hp) : ld4<H>(vg(q, i), hp));
#pragma unroll
                    for (int j = 0; j < kCW; ++j) acc[j] += v.a[j] * w[k][j];
                }
            }
            block_colsum4<C, NT>(acc, red, rbuf);
#pragma unroll
            for (int k = 0; k < RPT; ++k) {  // V_q re-read (shared memory or this CTA's L1/L2 slot)
                const int i = rl + k * RL;
                if (i < d) {
                    const V4 v = (q == s ? ld4<H>(Vc + static_cast<std::size_t>(i) * C, hp) : ld4<H>(vg(q, i), hp));
#pragma unroll
                    for (int j = 0; j < kCW; ++j) w[k][j] -= acc[j] * v.a[j];
                }
            }
        }
        BE_FOM_MARK(2);
#pragma unroll
        for (int j = 0; j < kCW; ++j) acc[j] = 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
            for (int j = 0; j < kCW; ++j) acc[j] += w[k][j] * w[k][j];
        block_colsum4<C, NT>(acc, red, rbuf);  // its barrier also retires every gather of V_s
#pragma unroll
        for (int j = 0; j < kCW; ++j) {
            const double nw = sqrt(acc[j]);
            inv[j] = 1.0;
            if (live[j]) {
                if (nw < 1e-14 * beta0[j]) {  // Krylov breakdown
                    steps[j] = s + 1;
                    live[j] = false;
                } else {
                    if (rl == 0) s_beta[s][cq * kCW + j] = nw;
                    bprev[j] = nw;
                    inv[j] = nw;
                }
            }
            rinv[j] = 1.0 / inv[j];
        }
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int i = rl + k * RL;
            if (i < d) {
                double v[kCW];
#pragma unroll
                for (int j = 0; j < kCW; ++j) v[j] = div_rcp(w[k][j], inv[j], rinv[j]);
                if constexpr (VSM) {
                    st4<H>(vg(s + 1, i), v, hp);
                } else {
                    st4<H>(Vc + static_cast<std::size_t>(i) * C, v, hp);
                    st4<H>(vg(s + 1, i), v, hp);
                }
            }
        }
        if constexpr (VSM) Vc += vstride;
        BE_FOM_MARK(3);
    }
    // T y = beta0 e1 by LU with partial pivoting (precond.hpp:208-249), one
    // thread per column (register-resident: every index is unrolled); the
    // solutions are broadcast through shared memory
    __shared__ double s_y[C][MC];
    __shared__ double s_b0[C];
    __shared__ int s_sing[C];
    if (rl == 0)
#pragma unroll
        for (int j = 0; j < kCW; ++j) {
            s_steps[cq * kCW + j] = steps[j];
            s_b0[cq * kCW + j] = beta0[j];
        }
    block_sync<NT>();
    if (threadIdx.x < C) {
        const int cc = threadIdx.x;
        const int st = s_steps[cc];
        const double b0 = s_b0[cc];
        double y[MC];
        int sg;
        if constexpr (MC <= 4) sg = tri_lu_solve<MC, true, C>(s_alpha, s_beta, cc, st, b0, y);
        else sg = tri_lu_solve<MC, false, C>(s_alpha, s_beta, cc, st, b0, y);
        if (col0 + cc < nb && b0 != 0.0 && sg && fallbacks)
            atomicAdd(reinterpret_cast<unsigned long long*>(fallbacks), 1ull);
#pragma unroll
        for (int q = 0; q < MC; ++q) s_y[cc][q] = y[q];
        s_sing[cc] = sg;
    }
    block_sync<NT>();
    double* out = W + td.row_off * nb + c0;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int i = rl + k * RL;
        if (i >= d) continue;
        double o[kCW] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < MC; ++q) {  // unrolled: the basis reads are in flight together
            if (q >= cap) break;
            const V4 v = ld4<H>(vg(q, i), hp);
#pragma unroll
            for (int j = 0; j < kCW; ++j)
                if (q < s_steps[cq * kCW + j]) o[j] += s_y[cq * kCW + j][q] * v.a[j];
        }
#pragma unroll
        for (int j = 0; j < kCW; ++j) {
            if (!colok[j]) continue;
            double res = 0.0;
            if (beta0[j] != 0.0)
                res = s_sing[cq * kCW + j] ? r[static_cast<std::int64_t>(i) * nb + j] : o[j];  // fallback: raw column
            out[static_cast<std::int64_t>(i) * nb + j] = res;
        }
    }
    BE_FOM_MARK(4);
#ifdef BE_FOM_PROF
    if (threadIdx.x == 0) atomicAdd(&g_fom_prof[NT == 32 ? 0 : NT == 128 ? 1 : (NT == 256 && RPT == 2) ? 2 : (NT == 256 && C == 16) ? 3 : 4][5], 1ull);
#endif
    if constexpr (!VSM) {  // every thread is done with the slot: release it
        __syncthreads();
        if (threadIdx.x == 0) atomicAnd(slot_mask + smid, ~(1u << (s_slot - static_cast<int>(smid) * kslots)));
    }
}

// size classes of the block kernel: tiles up to kClassDims[c] rows run on
// CTAs of the thread count in precond_apply's launch switch, kClassCols[c] columns per CTA (a tile is
// split over nb / C CTAs), every thread 4 adjacent columns of RPT rows, the
// dynamic shared memory (current vector + staged entries) held to
// kClassBudget[c]. Measured at T1 (profiles/r02_dense_precond_ncu.md): the
// 257..512-row class as two 8-column CTAs of 256 threads per SM (budget
// 104 KB) is 5 % slower than one 16-column CTA of 512 threads -- the same
// threads per SM either way (128 registers each fill the register file), and
// each CTA's Lanczos step costs as long at half the columns.
constexpr int kClassDims[] = {32, 64, 128, 256, 512};
#ifndef BE_FOM_C4_NT
#define BE_FOM_C4_NT 512
#define BE_FOM_C4_RPT 4
#define BE_FOM_C4_C 16
#define BE_FOM_C4_BUDGET_KB 200
#endif
constexpr int kClassCols[] = {16, 16, 16, 16, BE_FOM_C4_C};
constexpr bool kClassVsm[] = {true, true, true, false, false};  // whole basis in shared memory
constexpr std::size_t kStageBudget = 200 * 1024;  // current vector + staged entries per CTA
constexpr std::size_t kClassBudget[] = {kStageBudget, kStageBudget, kStageBudget, kStageBudget,
                                        static_cast<std::size_t>(BE_FOM_C4_BUDGET_KB) * 1024};


__global__ void k_nsmid(int* out) {
    unsigned v;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(v));
    *out = static_cast<int>(v);
}

// Scratch slots are indexed by %smid, which PTX bounds by %nsmid, not by the
// multiprocessor count (floorswept / MIG parts can have holes in the SM ids).
int smid_bound(Ctx* ctx, cudaStream_t cs) {
    if (ctx->nsmid <= 0) {
        DBuf<int> d(1);
        k_nsmid<<<1, 1, 0, cs>>>(d.get());
        int h = 0;
        BE_CUDA(cudaMemcpyAsync(&h, d.get(), sizeof(int), cudaMemcpyDeviceToHost, cs));
        BE_CUDA(cudaStreamSynchronize(cs));
        ctx->nsmid = std::max(h, ctx->num_sms);
    }
    return ctx->nsmid;
}

}  // namespace

// Device CSR of the host tiles (stable by row: a row's diagonal slot, last in
// the host entry order, stays last in its row) and the size-class lists.
static void tiles_upload(Tiles* tp, const index_t* off) {
    Tiles* t = tp;
    const index_t nt = static_cast<index_t>(t->host.size());
    // device CSR (stable by row: a row's diagonal slot stays last)
    std::vector<TileDev> td(static_cast<std::size_t>(nt));
    std::vector<std::int32_t> rowptr;
    std::vector<std::uint16_t> cols;
    std::vector<double> vals;
    t->max_dim = 0;
    for (index_t j = 0; j < nt; ++j) {
        const auto& T = t->host[static_cast<std::size_t>(j)];
        if (T.dim > 65535) fail(BE_ERR_BAD_PARAMS, "preconditioner tile larger than 65535 rows");
        t->max_dim = std::max<index_t>(t->max_dim, T.dim);
        td[static_cast<std::size_t>(j)] = TileDev{off[j], static_cast<std::int32_t>(T.dim),
                                                  static_cast<std::int32_t>(rowptr.size()),
                                                  static_cast<std::int64_t>(vals.size())};
        std::vector<std::int32_t> cnt(static_cast<std::size_t>(T.dim) + 1, 0);
        for (auto r : T.rows) ++cnt[static_cast<std::size_t>(r) + 1];
        for (std::size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
        const std::size_t base = vals.size();
        rowptr.insert(rowptr.end(), cnt.begin(), cnt.end());
        cols.resize(base + T.vals.size());
        vals.resize(base + T.vals.size());
        std::vector<std::int32_t> cur(cnt.begin(), cnt.end() - 1);
        for (std::size_t k = 0; k < T.vals.size(); ++k) {
            const auto p = base + static_cast<std::size_t>(cur[static_cast<std::size_t>(T.rows[k])]++);
            cols[p] = static_cast<std::uint16_t>(T.cols[k]);
            vals[p] = T.vals[k];
        }
    }
    if (rowptr.size() >= (std::size_t{1} << 31)) fail(BE_ERR_BAD_PARAMS, "preconditioner too large");
    t->tiles.reset(std::max<index_t>(nt, 1) * static_cast<index_t>(sizeof(TileDev)));
    t->rowptr.reset(std::max<index_t>(static_cast<index_t>(rowptr.size()), 1));
    t->cols.reset(std::max<index_t>(static_cast<index_t>(cols.size()), 1));
    t->vals.reset(std::max<index_t>(static_cast<index_t>(vals.size()), 1));
    t->ntiles = nt;
    t->nentries = static_cast<index_t>(vals.size());
    if (nt) BE_CUDA(cudaMemcpy(t->tiles.get(), td.data(), td.size() * sizeof(TileDev), cudaMemcpyHostToDevice));
    if (!rowptr.empty()) BE_CUDA(cudaMemcpy(t->rowptr.get(), rowptr.data(), rowptr.size() * 4, cudaMemcpyHostToDevice));
    if (!cols.empty()) BE_CUDA(cudaMemcpy(t->cols.get(), cols.data(), cols.size() * 2, cudaMemcpyHostToDevice));
    if (!vals.empty()) BE_CUDA(cudaMemcpy(t->vals.get(), vals.data(), vals.size() * 8, cudaMemcpyHostToDevice));
    {  // size classes: warp kernel per class, CTA kernel above the last one
        std::vector<std::int32_t> lists;
        t->class_dim.assign(std::begin(kClassDims), std::end(kClassDims));
        t->class_begin.clear();
        int lo = 0;
        for (int c = 0; c <= static_cast<int>(t->class_dim.size()); ++c) {
            t->class_begin.push_back(static_cast<index_t>(lists.size()));
            const int hi = c < static_cast<int>(t->class_dim.size()) ? t->class_dim[static_cast<std::size_t>(c)] : 1 << 30;
            const std::size_t b0 = lists.size();
            for (index_t j = 0; j < nt; ++j) {
                const index_t dd = t->host[static_cast<std::size_t>(j)].dim;
                if (dd > lo && dd <= hi) lists.push_back(static_cast<std::int32_t>(j));
            }
            // largest tiles first (entries + rows): the last wave of CTAs is the short one
            auto work = [&](std::int32_t j) {
                const auto& h = t->host[static_cast<std::size_t>(j)];
                return static_cast<index_t>(h.vals.size()) + 8 * h.dim;
            };
            std::stable_sort(lists.begin() + static_cast<std::ptrdiff_t>(b0), lists.end(),
                             [&](std::int32_t a, std::int32_t b) { return work(a) > work(b); });
            lo = hi;
        }
        t->class_begin.push_back(static_cast<index_t>(lists.size()));
        t->big_tiles = t->class_begin.back() - t->class_begin[t->class_dim.size()];
        t->class_max_ent.assign(t->class_dim.size(), 0);
        for (std::size_t c = 0; c < t->class_dim.size(); ++c)
            for (index_t q = t->class_begin[c]; q < t->class_begin[c + 1]; ++q)
                t->class_max_ent[c] = std::max<index_t>(
                    t->class_max_ent[c], static_cast<index_t>(t->host[static_cast<std::size_t>(lists[static_cast<std::size_t>(q)])].vals.size()));
        t->class_tiles.reset(std::max<index_t>(static_cast<index_t>(lists.size()), 1));
        if (!lists.empty())
            BE_CUDA(cudaMemcpy(t->class_tiles.get(), lists.data(), lists.size() * 4, cudaMemcpyHostToDevice));
    }
}

std::unique_ptr<Tiles> tiles_create(Ctx* ctx, const be_csb_view& L, const double* diag, const index_t* off_all,
                                    index_t noff_all, index_t row_lo, index_t row_hi) {
    validate_view(L);
    // extract_tiles checks (precond.hpp:65-84)
    if (L.nrows != L.ncols) fail(BE_ERR_DIMENSION_MISMATCH, "extract_tiles: matrix must be square");
    if (!off_all || noff_all < 2 || off_all[0] != 0 || off_all[noff_all - 1] != L.nrows)
        fail(BE_ERR_BAD_PARAMS, "extract_tiles: tile offsets must cover [0, n)");
    for (index_t j = 1; j < noff_all; ++j)
        if (off_all[j] <= off_all[j - 1]) fail(BE_ERR_BAD_PARAMS, "extract_tiles: tile offsets must be strictly increasing");
    if (row_lo < 0) row_hi = L.nrows, row_lo = 0;  // whole matrix
    // the rank's row range (multi-GPU) must be a union of whole tiles
    const index_t* lo_it = std::lower_bound(off_all, off_all + noff_all, row_lo);
    const index_t* hi_it = std::lower_bound(off_all, off_all + noff_all, row_hi);
    if (lo_it == off_all + noff_all || *lo_it != row_lo || hi_it == off_all + noff_all || *hi_it != row_hi ||
        row_hi < row_lo)
        fail(BE_ERR_MISALIGNED_TILES, "extract_tiles: row range is not a union of tiles");
    if (!diag && row_hi > row_lo) fail(BE_ERR_DIMENSION_MISMATCH, "extract_tiles: diagonal length mismatch");
    // local tile offsets relative to row_lo; panels of the result have row_hi - row_lo rows
    std::vector<index_t> off_local;
    for (const index_t* q = lo_it; q <= hi_it; ++q) off_local.push_back(*q - row_lo);
    const index_t* off = off_local.data();
    const index_t noff = static_cast<index_t>(off_local.size());
    for (index_t j = 1; j < noff; ++j)
        if (off[j] <= off[j - 1]) fail(BE_ERR_BAD_PARAMS, "extract_tiles: tile offsets must be strictly increasing");
    {
        index_t blk = 0;
        for (index_t j = 0; j + 1 < noff_all; ++j) {
            while (blk + 1 < L.nrowblks + 1 && L.row_offsets[blk + 1] <= off_all[j]) ++blk;
            if (off_all[j + 1] > L.row_offsets[blk + 1])
                fail(BE_ERR_MISALIGNED_TILES, "extract_tiles: tile [" + std::to_string(off_all[j]) + ", " +
                                                  std::to_string(off_all[j + 1]) + ") straddles a block boundary");
        }
    }
    auto t = std::make_unique<Tiles>();
    t->ctx = ctx;
    t->n = row_hi - row_lo;
    t->offsets.assign(off, off + noff);
    const index_t nt = noff - 1;
    t->host.resize(static_cast<std::size_t>(nt));
    std::vector<std::int32_t> owner(static_cast<std::size_t>(t->n));
    for (index_t j = 0; j < nt; ++j) {
        t->host[static_cast<std::size_t>(j)].dim = off[j + 1] - off[j];
        for (index_t i = off[j]; i < off[j + 1]; ++i) owner[static_cast<std::size_t>(i)] = static_cast<std::int32_t>(j);
    }
    // couplings in to_triples order (csb.hpp:165-185), both orientations; only
    // block rows meeting [row_lo, row_hi) can hold them
    for (index_t bi = 0; bi < L.nrowblks; ++bi) {
        if (L.row_offsets[bi + 1] <= row_lo || L.row_offsets[bi] >= row_hi) continue;
        for (index_t bj = 0; bj < L.ncolblks; ++bj) {
            const index_t b = bi * L.ncolblks + bj;
            for (index_t k = L.block_nnz_offsets[b]; k < L.block_nnz_offsets[b] + L.block_nnz[b]; ++k) {
                const index_t r = L.row_offsets[bi] + L.local_rows[k], c = L.col_offsets[bj] + L.local_cols[k];
                if (r <= c) fail(BE_ERR_NOT_STRICTLY_LOWER, "extract_tiles: stored entry with row <= col");
                if (r < row_lo || r >= row_hi || c < row_lo || c >= row_hi) continue;
                const auto j = owner[static_cast<std::size_t>(r - row_lo)];
                if (j != owner[static_cast<std::size_t>(c - row_lo)]) continue;
                auto& T = t->host[static_cast<std::size_t>(j)];
                const auto a = static_cast<std::int32_t>(r - row_lo - off[j]), cc = static_cast<std::int32_t>(c - row_lo - off[j]);
                T.rows.push_back(a);
                T.cols.push_back(cc);
                T.vals.push_back(L.values[k]);
                T.rows.push_back(cc);
                T.cols.push_back(a);
                T.vals.push_back(L.values[k]);
            }
        }
    }
    for (index_t j = 0; j < nt; ++j) {  // diagonal slots last
        auto& T = t->host[static_cast<std::size_t>(j)];
        T.diag_pos.resize(static_cast<std::size_t>(T.dim));
        for (index_t i = 0; i < T.dim; ++i) {
            T.diag_pos[static_cast<std::size_t>(i)] = static_cast<index_t>(T.vals.size());
            T.rows.push_back(static_cast<std::int32_t>(i));
            T.cols.push_back(static_cast<std::int32_t>(i));
            T.vals.push_back(diag[off[j] + i]);
        }
    }
    tiles_upload(t.get(), off);
    return t;
}

std::unique_ptr<Tiles> tiles_create_explicit(Ctx* ctx, const std::vector<HostTile>& tiles) {
    auto t = std::make_unique<Tiles>();
    t->ctx = ctx;
    std::vector<index_t> off(1, 0);
    for (const auto& T : tiles) {
        if (T.dim < 1) fail(BE_ERR_BAD_PARAMS, "SparseTile: dim must be positive");
        if (T.rows.size() != T.vals.size() || T.cols.size() != T.vals.size() ||
            T.diag_pos.size() != static_cast<std::size_t>(T.dim))
            fail(BE_ERR_DIMENSION_MISMATCH, "SparseTile: rows / cols / values / diag_pos sizes disagree");
        // reference layout (precond.hpp:18-30): couplings, then one diagonal slot per row; the
        // device CSR keeps each row's diagonal slot last, so it is moved there if it is not
        std::vector<char> is_diag(T.vals.size(), 0);
        for (index_t i = 0; i < T.dim; ++i) {
            const index_t q = T.diag_pos[static_cast<std::size_t>(i)];
            if (q < 0 || q >= static_cast<index_t>(T.vals.size()) || T.rows[static_cast<std::size_t>(q)] != i ||
                T.cols[static_cast<std::size_t>(q)] != i)
                fail(BE_ERR_BAD_PARAMS, "SparseTile: diag_pos does not point at the diagonal slot of its row");
            is_diag[static_cast<std::size_t>(q)] = 1;
        }
        HostTile h;
        h.dim = T.dim;
        for (std::size_t q = 0; q < T.vals.size(); ++q) {
            if (is_diag[q]) continue;
            if (T.rows[q] < 0 || T.rows[q] >= T.dim || T.cols[q] < 0 || T.cols[q] >= T.dim)
                fail(BE_ERR_INDEX_OUT_OF_RANGE, "SparseTile: entry outside the tile");
            h.rows.push_back(T.rows[q]);
            h.cols.push_back(T.cols[q]);
            h.vals.push_back(T.vals[q]);
        }
        h.diag_pos.resize(static_cast<std::size_t>(T.dim));
        for (index_t i = 0; i < T.dim; ++i) {
            h.diag_pos[static_cast<std::size_t>(i)] = static_cast<index_t>(h.vals.size());
            h.rows.push_back(static_cast<std::int32_t>(i));
            h.cols.push_back(static_cast<std::int32_t>(i));
            h.vals.push_back(T.vals[static_cast<std::size_t>(T.diag_pos[static_cast<std::size_t>(i)])]);
        }
        off.push_back(off.back() + T.dim);
        t->host.push_back(std::move(h));
    }
    t->n = off.back();
    t->offsets = off;
    tiles_upload(t.get(), off.data());
    return t;
}

void precond_apply(Tiles* t, const double* shifts, const double* R, double* W, index_t nrows, int nb, int m,
                   std::int64_t* fallbacks, cudaStream_t s) {
    if (m < 1) fail(BE_ERR_BAD_PARAMS, "FomConfig: iterations must be >= 1");
    if (nrows != t->n) fail(BE_ERR_DIMENSION_MISMATCH, "apply_preconditioner: residual rows != operator dim");
    if (nb < 1) fail(BE_ERR_DIMENSION_MISMATCH, "apply_preconditioner: one shift per column required");
    if (m > kMaxSteps) fail(BE_ERR_BAD_PARAMS, "apply_preconditioner: m above the device kernel's step cap (64)");
    if (t->ntiles == 0) return;
    const auto* tdv = reinterpret_cast<const TileDev*>(t->tiles.get());
    const int ncls = static_cast<int>(t->class_dim.size());
    const bool reg_ok = m <= 8;
    // The classes write disjoint rows of W: the largest class runs on s, launched
    // first, the others on side streams, so small-tile CTAs fill the SMs around
    // the large-tile ones (one 512-thread CTA per SM leaves room).
    static_assert(sizeof(kClassDims) / sizeof(kClassDims[0]) <= 8, "class arrays");
    if (!t->fork) {
        BE_CUDA(cudaEventCreateWithFlags(&t->fork, cudaEventDisableTiming));
        for (int c = 0; c < ncls; ++c) {
            BE_CUDA(cudaStreamCreateWithFlags(&t->side[c], cudaStreamNonBlocking));
            BE_CUDA(cudaEventCreateWithFlags(&t->join[c], cudaEventDisableTiming));
        }
    }
    BE_CUDA(cudaEventRecord(t->fork, s));
    bool joined[8] = {};
    for (int ci = 0; ci < ncls && reg_ok; ++ci) {
        const int c = ncls - 1 - ci;  // largest class first
        const index_t b0 = t->class_begin[static_cast<std::size_t>(c)], b1 = t->class_begin[static_cast<std::size_t>(c) + 1];
        if (b1 == b0) continue;
        cudaStream_t cs = s;
        if (ci > 0) {
            cs = t->side[c];
            BE_CUDA(cudaStreamWaitEvent(cs, t->fork, 0));
            joined[c] = true;
        }
        const int dmax = t->class_dim[static_cast<std::size_t>(c)];
        const int C = kClassCols[c];
        const int ngroups = (nb + C - 1) / C;
        const std::int32_t* list = t->class_tiles.get() + b0;
        const int mc = m <= 4 ? 4 : 8;
        const std::size_t vone = static_cast<std::size_t>(dmax) * C * sizeof(double);
        const bool vsm = kClassVsm[c] && vone * std::min(m, mc) <= 160 * 1024;  // else: scratch slots in L2
        const std::size_t vbytes = vone * (vsm ? std::min(m, mc) : 1);
        // entry staging: up to the class's largest tile, within the smem budget
        const std::size_t budget = kClassBudget[c];
        const std::size_t room = vbytes < budget ? (budget - vbytes) / 10 : 0;
        const int stage_cap = static_cast<int>(std::min<std::size_t>(room, static_cast<std::size_t>(t->class_max_ent[static_cast<std::size_t>(c)]))) & ~7;
        std::size_t sm = vbytes + static_cast<std::size_t>(stage_cap) * 10;
        const unsigned grid = static_cast<unsigned>((b1 - b0) * ngroups);
        int kslots = 1;
        const int nslot_sm = smid_bound(t->ctx, cs);
        auto slots_for = [&](const void* kern, int nt) {  // resident CTAs per SM = scratch slots per SM
            int per = 0;
            BE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, nt, sm));
            kslots = std::max(1, std::min(per, 32));
            const index_t vneed = static_cast<index_t>(mc) * nslot_sm * kslots * dmax * C;
            if (t->vscratch[c].n < vneed) t->vscratch[c].reset(vneed);
            if (t->slot_mask[c].n < nslot_sm) {
                t->slot_mask[c].reset(nslot_sm);
                BE_CUDA(cudaMemsetAsync(t->slot_mask[c].get(), 0, t->slot_mask[c].bytes(), cs));
            }
        };
#define BE_FOMB(MC, NTT, RPT, VS, CC)                                                                              \
    do {                                                                                                               \
        ensure_dyn_smem(k_fom_blk<MC, NTT, RPT, VS, CC>, sm);                                                          \
        if (!(VS)) slots_for(reinterpret_cast<const void*>(k_fom_blk<MC, NTT, RPT, VS, CC>), NTT);                    \
        k_fom_blk<MC, NTT, RPT, VS, CC><<<grid, NTT, sm, cs>>>(tdv, list, t->rowptr.get(), t->cols.get(), t->vals.get(), \
                                                                shifts, R, W, nb, m, ngroups, fallbacks, dmax,         \
                                                                stage_cap, t->vscratch[c].get(), t->n,                 \
                                                                t->slot_mask[c].get(), kslots);                        \
    } while (0)
#define BE_FOMB2(NTT, RPT, CC)                      \
    if (mc == 4) {                                  \
        if (vsm) BE_FOMB(4, NTT, RPT, true, CC);    \
        else BE_FOMB(4, NTT, RPT, false, CC);       \
    } else {                                        \
        if (vsm) BE_FOMB(8, NTT, RPT, true, CC);    \
        else BE_FOMB(8, NTT, RPT, false, CC);       \
    }
        static_assert(BE_FOM_C4_NT / (BE_FOM_C4_C / kCW) * BE_FOM_C4_RPT >= 512, "class 4 rows per CTA");
        switch (c) {
            case 0: BE_FOMB2(32, 4, 16); break;    // 8 rows per pass x 4
            case 1: BE_FOMB2(128, 2, 16); break;   // 32 x 2
            case 2: BE_FOMB2(256, 2, 16); break;   // 64 x 2
            case 3: BE_FOMB2(256, 4, 16); break;   // 64 x 4 (two CTAs per SM)
            default: BE_FOMB2(BE_FOM_C4_NT, BE_FOM_C4_RPT, BE_FOM_C4_C); break;  // 128 x 4, 8 columns
        }
#undef BE_FOMB2
#undef BE_FOMB
        BE_CUDA(cudaGetLastError());
        ++t->ctx->launches;
        if (joined[c]) BE_CUDA(cudaEventRecord(t->join[c], cs));
    }
    for (int c = 0; c < ncls; ++c)
        if (joined[c]) BE_CUDA(cudaStreamWaitEvent(s, t->join[c], 0));
    // everything the register kernel does not cover goes through the CTA kernel
    const index_t big_begin = reg_ok ? t->class_begin[static_cast<std::size_t>(ncls)] : 0;
    const index_t nbig = t->class_begin.back() - big_begin;
    if (nbig == 0) return;
    const index_t cap = std::min<index_t>(m, t->max_dim);
    const std::size_t per_col = (static_cast<std::size_t>(cap + 1) * static_cast<std::size_t>(t->max_dim) +
                                 static_cast<std::size_t>(cap) * cap) * 8;
    int gc = 16;
    while (gc > 1 && (gc > nb * 2 || static_cast<std::size_t>(gc) * per_col > kSmemBudget)) gc /= 2;
    if (per_col > 200 * 1024) fail(BE_ERR_BAD_PARAMS, "apply_preconditioner: tile too large for the device kernel");
    const std::size_t sm = static_cast<std::size_t>(gc) * per_col;
    ensure_dyn_smem(k_fom, sm);
    const int ngroups = (nb + gc - 1) / gc;
    const index_t grid = nbig * ngroups;
    k_fom<<<static_cast<unsigned>(grid), kPT, sm, s>>>(tdv, t->rowptr.get(), t->cols.get(), t->vals.get(), shifts, R, W,
                                                        nb, m, gc, ngroups, fallbacks,
                                                        t->class_tiles.get() + big_begin);
    BE_CUDA(cudaGetLastError());
    ++t->ctx->launches;
}

}  // namespace be

#ifdef BE_FOM_PROF
extern "C" int be_fom_prof_read(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, be::g_fom_prof, sizeof(be::g_fom_prof)) != cudaSuccess) return 1;
    if (reset) {
        static const unsigned long long z[5][8] = {};
        if (cudaMemcpyToSymbol(be::g_fom_prof, z, sizeof(z)) != cudaSuccess) return 1;
    }
    return 0;
}
#endif
