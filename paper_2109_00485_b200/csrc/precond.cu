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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;  // butterfly: every lane holds the bitwise-identical total
}

// One thread group of G threads (a warp, or 4 warps) per (tile, column):
// the m-step FOM of k_fom with the Krylov basis held in registers (each
// thread owns rows tid, tid + G, ... up to RM rows) and only the current
// basis vector in shared memory for the sparse gather. Reductions use warp
// butterflies (+ a named barrier across the 4 warps when G = 128), all in a
// fixed order.
template <int G, int RM, int MC>
__global__ void __launch_bounds__(256) k_fom_reg(const TileDev* __restrict__ tiles, const std::int32_t* __restrict__ list,
                                                 int nlist, const std::int32_t* __restrict__ rowptr,
                                                 const std::uint16_t* __restrict__ cols,
                                                 const double* __restrict__ vals, const double* __restrict__ shifts,
                                                 const double* __restrict__ R, double* __restrict__ W, int nb, int m,
                                                 std::int64_t* fallbacks) {
    constexpr int NG = 256 / G;  // items per CTA
    constexpr int DMAX = G * RM;
    __shared__ double s_vs[NG][DMAX];
    __shared__ double s_red[NG][G / 32];
    __shared__ double s_y[NG][MC];
    __shared__ int s_sing[NG];
    const int g = threadIdx.x / G, t = threadIdx.x % G, lane = threadIdx.x & 31, wg = t >> 5;
    const long item = static_cast<long>(blockIdx.x) * NG + g;
    if (item >= static_cast<long>(nlist) * nb) return;  // whole groups exit together
    auto gsync = [&]() {
        if constexpr (G == 32) {
            __syncwarp();
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(G) : "memory");
        }
    };
    auto gsum = [&](double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if constexpr (G == 32) {
            return v;
        } else {
            if (lane == 0) s_red[g][wg] = v;
            gsync();
            double tot = 0.0;
#pragma unroll
            for (int q = 0; q < G / 32; ++q) tot += s_red[g][q];
            gsync();
            return tot;
        }
    };
    const int col = static_cast<int>(item % nb);
    const TileDev td = tiles[list[item / nb]];
    const int d = td.dim;
    const int cap = min(m, d);
    const std::int32_t* rp = rowptr + td.ptr_off;
    const std::uint16_t* cl = cols + td.ent_off;
    const double* vl = vals + td.ent_off;
    const double sigma = shifts[col];
    const double* r = R + td.row_off * nb + col;
    double* out = W + td.row_off * nb + col;
    double* vs = s_vs[g];

    double V[MC][RM], w[RM];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < RM; ++k) {
        const int i = t + k * G;
        const double x = i < d ? r[static_cast<std::int64_t>(i) * nb] : 0.0;
        V[0][k] = x;
        acc += x * x;
    }
    const double beta0 = sqrt(gsum(acc));
    if (beta0 == 0.0) {
#pragma unroll
        for (int k = 0; k < RM; ++k)
            if (t + k * G < d) out[static_cast<std::int64_t>(t + k * G) * nb] = 0.0;
        return;
    }
#pragma unroll
    for (int k = 0; k < RM; ++k) V[0][k] /= beta0;
    double alpha[MC], beta[MC];
    int steps = cap;
#pragma unroll
    for (int s = 0; s < MC; ++s) {
        if (s >= cap) break;
        // w = (K - sigma I) V_s ; alpha_s = V_s . w
#pragma unroll
        for (int k = 0; k < RM; ++k)
            if (t + k * G < d) vs[t + k * G] = V[s][k];
        gsync();
        acc = 0.0;
#pragma unroll
        for (int k = 0; k < RM; ++k) {
            const int i = t + k * G;
            double yy = 0.0;
            if (i < d) {
                const int e1 = rp[i + 1] - 1;  // the diagonal slot is last
                for (int e = rp[i]; e < e1; ++e) yy += vl[e] * vs[cl[e]];
                yy += (vl[e1] - sigma) * V[s][k];
            }
            w[k] = yy;
            acc += V[s][k] * yy;
        }
        const double a = gsum(acc);
        alpha[s] = a;
        if (s + 1 == cap) break;
#pragma unroll
        for (int k = 0; k < RM; ++k) {
            double x = w[k] - a * V[s][k];
            if (s > 0) x -= beta[s > 0 ? s - 1 : 0] * V[s > 0 ? s - 1 : 0][k];
            w[k] = x;
        }
#pragma unroll
        for (int q = 0; q < MC; ++q) {  // one reorthogonalisation pass, in order
            if (q > s) break;
            acc = 0.0;
#pragma unroll
            for (int k = 0; k < RM; ++k) acc += V[q][k] * w[k];
            const double pr = gsum(acc);
#pragma unroll
            for (int k = 0; k < RM; ++k) w[k] -= pr * V[q][k];
        }
        acc = 0.0;
#pragma unroll
        for (int k = 0; k < RM; ++k) acc += w[k] * w[k];
        const double nw = sqrt(gsum(acc));
        if (nw < 1e-14 * beta0) {  // Krylov breakdown
            steps = s + 1;
            break;
        }
        beta[s] = nw;
        if (s + 1 < MC) {
#pragma unroll
            for (int k = 0; k < RM; ++k) V[s + 1 < MC ? s + 1 : 0][k] = w[k] / nw;
        }
        gsync();  // vs is rewritten by the next step
    }
    if (t == 0) {  // T y = beta0 e1 by LU with partial pivoting (precond.hpp:208-249)
        const int st = steps;
        double T[MC][MC];
        double tmax = 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i)
#pragma unroll
            for (int j = 0; j < MC; ++j) T[i][j] = 0.0;
        double y[MC];
#pragma unroll
        for (int i = 0; i < MC; ++i) {
            y[i] = 0.0;
            if (i < st) {
                T[i][i] = alpha[i];
                tmax = fmax(tmax, fabs(alpha[i]));
                if (i + 1 < st) {
                    T[i][i + 1 < MC ? i + 1 : 0] = beta[i];
                    T[i + 1 < MC ? i + 1 : 0][i] = beta[i];
                    tmax = fmax(tmax, fabs(beta[i]));
                }
            }
        }
        const double floor = 1e-14 * fmax(1.0, tmax);
        y[0] = beta0;
        int sing = 0;
#pragma unroll
        for (int k = 0; k < MC; ++k) {
            if (k >= st || sing) break;
            int piv = k;
#pragma unroll
            for (int i = 0; i < MC; ++i)
                if (i > k && i < st && fabs(T[i][k]) > fabs(T[piv][k])) piv = i;
            if (fabs(T[piv][k]) < floor) {
                sing = 1;
                break;
            }
            if (piv != k) {
#pragma unroll
                for (int j = 0; j < MC; ++j) {
                    const double tmp = T[k][j];
                    T[k][j] = T[piv][j];
                    T[piv][j] = tmp;
                }
                const double tmp = y[k];
                y[k] = y[piv];
                y[piv] = tmp;
            }
#pragma unroll
            for (int i = 0; i < MC; ++i) {
                if (i <= k || i >= st) continue;
                const double f = T[i][k] / T[k][k];
                if (f == 0.0) continue;
#pragma unroll
                for (int j = 0; j < MC; ++j)
                    if (j >= k) T[i][j] -= f * T[k][j];
                y[i] -= f * y[k];
            }
        }
        if (!sing) {
#pragma unroll
            for (int i = MC - 1; i >= 0; --i) {
                if (i >= st) continue;
                double a2 = y[i];
#pragma unroll
                for (int j = 0; j < MC; ++j)
                    if (j > i && j < st) a2 -= T[i][j] * y[j];
                y[i] = a2 / T[i][i];
            }
        }
#pragma unroll
        for (int i = 0; i < MC; ++i) s_y[g][i] = y[i];
        s_sing[g] = sing;
        if (sing && fallbacks) atomicAdd(reinterpret_cast<unsigned long long*>(fallbacks), 1ull);
    }
    gsync();
    const int sing = s_sing[g];
#pragma unroll
    for (int k = 0; k < RM; ++k) {
        const int i = t + k * G;
        if (i >= d) continue;
        double o = 0.0;
        if (sing) {
            o = r[static_cast<std::int64_t>(i) * nb];  // unpreconditioned fallback column
        } else {
#pragma unroll
            for (int j = 0; j < MC; ++j)
                if (j < steps) o += s_y[g][j] * V[j][k];
        }
        out[static_cast<std::int64_t>(i) * nb] = o;
    }
}

constexpr int kClassDims[] = {128, 512};  // warp (4 rows / lane), 4 warps (4 rows / thread)

}  // namespace

std::unique_ptr<Tiles> tiles_create(Ctx* ctx, const be_csb_view& L, const double* diag, const index_t* off,
                                    index_t noff) {
    validate_view(L);
    // extract_tiles checks (precond.hpp:65-84)
    if (L.nrows != L.ncols) fail(BE_ERR_DIMENSION_MISMATCH, "extract_tiles: matrix must be square");
    if (!diag && L.nrows > 0) fail(BE_ERR_DIMENSION_MISMATCH, "extract_tiles: diagonal length mismatch");
    if (!off || noff < 2 || off[0] != 0 || off[noff - 1] != L.nrows)
        fail(BE_ERR_BAD_PARAMS, "extract_tiles: tile offsets must cover [0, n)");
    for (index_t j = 1; j < noff; ++j)
        if (off[j] <= off[j - 1]) fail(BE_ERR_BAD_PARAMS, "extract_tiles: tile offsets must be strictly increasing");
    {
        index_t blk = 0;
        for (index_t j = 0; j + 1 < noff; ++j) {
            while (blk + 1 < L.nrowblks + 1 && L.row_offsets[blk + 1] <= off[j]) ++blk;
            if (off[j + 1] > L.row_offsets[blk + 1])
                fail(BE_ERR_MISALIGNED_TILES, "extract_tiles: tile [" + std::to_string(off[j]) + ", " +
                                                  std::to_string(off[j + 1]) + ") straddles a block boundary");
        }
    }
    auto t = std::make_unique<Tiles>();
    t->ctx = ctx;
    t->n = L.nrows;
    t->offsets.assign(off, off + noff);
    const index_t nt = noff - 1;
    t->host.resize(static_cast<std::size_t>(nt));
    std::vector<std::int32_t> owner(static_cast<std::size_t>(L.nrows));
    for (index_t j = 0; j < nt; ++j) {
        t->host[static_cast<std::size_t>(j)].dim = off[j + 1] - off[j];
        for (index_t i = off[j]; i < off[j + 1]; ++i) owner[static_cast<std::size_t>(i)] = static_cast<std::int32_t>(j);
    }
    // couplings in to_triples order (csb.hpp:165-185), both orientations
    for (index_t bi = 0; bi < L.nrowblks; ++bi)
        for (index_t bj = 0; bj < L.ncolblks; ++bj) {
            const index_t b = bi * L.ncolblks + bj;
            for (index_t k = L.block_nnz_offsets[b]; k < L.block_nnz_offsets[b] + L.block_nnz[b]; ++k) {
                const index_t r = L.row_offsets[bi] + L.local_rows[k], c = L.col_offsets[bj] + L.local_cols[k];
                if (r <= c) fail(BE_ERR_NOT_STRICTLY_LOWER, "extract_tiles: stored entry with row <= col");
                const auto j = owner[static_cast<std::size_t>(r)];
                if (j != owner[static_cast<std::size_t>(c)]) continue;
                auto& T = t->host[static_cast<std::size_t>(j)];
                const auto a = static_cast<std::int32_t>(r - off[j]), cc = static_cast<std::int32_t>(c - off[j]);
                T.rows.push_back(a);
                T.cols.push_back(cc);
                T.vals.push_back(L.values[k]);
                T.rows.push_back(cc);
                T.cols.push_back(a);
                T.vals.push_back(L.values[k]);
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
            for (index_t j = 0; j < nt; ++j) {
                const index_t dd = t->host[static_cast<std::size_t>(j)].dim;
                if (dd > lo && dd <= hi) lists.push_back(static_cast<std::int32_t>(j));
            }
            lo = hi;
        }
        t->class_begin.push_back(static_cast<index_t>(lists.size()));
        t->big_tiles = t->class_begin.back() - t->class_begin[t->class_dim.size()];
        t->class_tiles.reset(std::max<index_t>(static_cast<index_t>(lists.size()), 1));
        if (!lists.empty())
            BE_CUDA(cudaMemcpy(t->class_tiles.get(), lists.data(), lists.size() * 4, cudaMemcpyHostToDevice));
    }
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
    for (int c = 0; c < ncls && reg_ok; ++c) {
        const index_t b0 = t->class_begin[static_cast<std::size_t>(c)], b1 = t->class_begin[static_cast<std::size_t>(c) + 1];
        if (b1 == b0) continue;
        const int dmax = t->class_dim[static_cast<std::size_t>(c)];
        const index_t items = (b1 - b0) * nb;
        const std::int32_t* list = t->class_tiles.get() + b0;
        const int nl = static_cast<int>(b1 - b0);
#define BE_FOMR(G, MC)                                                                                              \
    k_fom_reg<G, 4, MC><<<static_cast<unsigned>((items + 256 / G - 1) / (256 / G)), 256, 0, s>>>(               \
        tdv, list, nl, t->rowptr.get(), t->cols.get(), t->vals.get(), shifts, R, W, nb, m, fallbacks)
        if (dmax <= 128) {
            if (m <= 4) BE_FOMR(32, 4); else BE_FOMR(32, 8);
        } else {
            if (m <= 4) BE_FOMR(128, 4); else BE_FOMR(128, 8);
        }
#undef BE_FOMR
        BE_CUDA(cudaGetLastError());
        ++t->ctx->launches;
    }
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
    BE_CUDA(cudaFuncSetAttribute(k_fom, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));  // static smem counts too
    const int ngroups = (nb + gc - 1) / gc;
    const index_t grid = nbig * ngroups;
    k_fom<<<static_cast<unsigned>(grid), kPT, sm, s>>>(tdv, t->rowptr.get(), t->cols.get(), t->vals.get(), shifts, R, W,
                                                        nb, m, gc, ngroups, fallbacks,
                                                        t->class_tiles.get() + big_begin);
    BE_CUDA(cudaGetLastError());
    ++t->ctx->launches;
}

}  // namespace be
