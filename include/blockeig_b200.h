/*
 * blockeig_b200.h -- C ABI of the B200-native LOBPCG hot path.
 *
 * This is the drop-in boundary for the reference library `blockeig`
 * (/root/reference/proj/include/blockeig/ headers). Every entry point below is
 * plain C: opaque handles, raw pointers and sizes, no C++ or torch types.
 * Each one names the reference interface it replaces (file:line relative to
 * /root/reference/proj/include/blockeig/). The C++ mirror of the reference API
 * (namespace blockeig, include/blockeig_b200.hpp) is a thin header-only layer
 * over these functions and re-throws the reference's typed exceptions from
 * the status codes.
 *
 * Conventions
 *   - Every function returns be_status; BE_OK == 0. On failure the message is
 *     available from be_last_error() (thread-local) and, for
 *     BE_ERR_NOT_POSITIVE_DEFINITE, the pivot index from be_last_error_pivot().
 *   - Multivectors ("panels") are row-major n x nb, element (r, v) at
 *     r * nb + v, exactly the BlockVector layout (block_vector.hpp:16-39).
 *   - "_dev" pointers are CUDA device pointers; "stream" is a cudaStream_t
 *     passed as void* (NULL = the context's own stream).
 *   - Host-buffer variants (suffix _host) copy in/out inside the call; they
 *     are the reference-facing Operator adapter (lobpcg.hpp:20).
 */
#ifndef BLOCKEIG_B200_H
#define BLOCKEIG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One status code per exception class of errors.hpp:11-109. */
typedef enum be_status {
    BE_OK = 0,
    BE_ERR_GENERIC = 1,                 /* blockeig::Error            errors.hpp:11  */
    BE_ERR_BLOCK_TOO_LARGE = 2,         /* BlockTooLarge              errors.hpp:18  */
    BE_ERR_INDEX_OUT_OF_RANGE = 3,      /* IndexOutOfRange            errors.hpp:23  */
    BE_ERR_DUPLICATE_ENTRY = 4,         /* DuplicateEntry             errors.hpp:28  */
    BE_ERR_DIMENSION_MISMATCH = 5,      /* DimensionMismatch          errors.hpp:33  */
    BE_ERR_NOT_STRICTLY_LOWER = 6,      /* NotStrictlyLower           errors.hpp:38  */
    BE_ERR_MISALIGNED_TILES = 7,        /* MisalignedTiles            errors.hpp:43  */
    BE_ERR_BAD_PARAMS = 8,              /* BadParams                  errors.hpp:48  */
    BE_ERR_NOT_POSITIVE_DEFINITE = 9,   /* NotPositiveDefinite{pivot} errors.hpp:55  */
    BE_ERR_SINGULAR_TRIANGULAR = 10,    /* SingularTriangular         errors.hpp:62  */
    BE_ERR_SINGULAR_PROJECTION = 11,    /* SingularProjection         errors.hpp:67  */
    BE_ERR_RANK_DEFICIENT = 12,         /* RankDeficient              errors.hpp:72  */
    BE_ERR_BASIS_DEGENERATE = 13,       /* BasisDegenerate            errors.hpp:77  */
    BE_ERR_BREAKDOWN_UNRECOVERABLE = 14,/* BreakdownUnrecoverable     errors.hpp:82  */
    BE_ERR_EVEN_ND = 15,                /* EvenNd                     errors.hpp:89  */
    BE_ERR_PROTOCOL_DEADLOCK = 16,      /* ProtocolDeadlock           errors.hpp:94  */
    BE_ERR_PARSE = 17,                  /* ParseError                 errors.hpp:101 */
    BE_ERR_NOT_SYMMETRIC_HEADER = 18,   /* NotSymmetricHeader         errors.hpp:106 */
    /* device-side failures with no reference counterpart */
    BE_ERR_CUDA = 32,
    BE_ERR_NO_DEVICE = 33,
    BE_ERR_CUSOLVER = 34,
    BE_ERR_NCCL = 35,
    BE_ERR_OUT_OF_MEMORY = 36
} be_status;

typedef enum be_prec { BE_F32 = 0, BE_F64 = 1 } be_prec;

/* apply modes of the operator (kernels.hpp:290-371) */
typedef enum be_apply_mode {
    BE_APPLY_SYMMETRIC = 0,  /* out  = (L + L^T + diag D) in   SymmetricOperator::apply kernels.hpp:357 */
    BE_APPLY_NOTRANS_ACC = 1,/* out += L in                    spmm_notrans kernels.hpp:290 */
    BE_APPLY_TRANS_ACC = 2   /* out += L^T in                  spmm_trans   kernels.hpp:302 */
} be_apply_mode;

const char* be_last_error(void);
int be_last_error_pivot(void);
const char* be_version(void);

/* ------------------------------------------------------------------------- */
/* Host-side CSB_Coo storage (csb.hpp:39-63).                                 */
/* ------------------------------------------------------------------------- */

/* Triple layout of csb.hpp:20-24 (24 bytes: i64 row, i64 col, f64 value). */
typedef struct be_triple {
    int64_t row;
    int64_t col;
    double value;
} be_triple;

/* Read-only view of a CsbCooMatrix: the same arrays, same meaning. */
typedef struct be_csb_view {
    int64_t nrows, ncols, nrowblks, ncolblks, nnz;
    const int64_t* row_offsets;        /* nrowblks + 1 */
    const int64_t* col_offsets;        /* ncolblks + 1 */
    const int64_t* block_nnz;          /* nrowblks * ncolblks, row-major */
    const int64_t* block_nnz_offsets;  /* same shape, exclusive prefix */
    const uint16_t* local_rows;        /* nnz */
    const uint16_t* local_cols;        /* nnz */
    const double* values;              /* nnz */
} be_csb_view;

typedef struct be_csb be_csb; /* owned host CSB */

/* build_csb_coo (csb.hpp:100-161): block row-major grouping, input order
 * kept inside a block, range check then duplicate check. */
be_status be_csb_build(const be_triple* triples, int64_t count, int64_t nrows, int64_t ncols,
                       const int64_t* row_bounds, int64_t n_row_bounds,
                       const int64_t* col_bounds, int64_t n_col_bounds, be_csb** out);
/* uniform_boundaries (csb.hpp:89-96); *count receives nblk + 1. out may be
 * NULL to query the count. */
be_status be_uniform_boundaries(int64_t n, int64_t extent, int64_t* out, int64_t* count);
/* random_block (block_vector.hpp:47-53): rows [row_lo, row_lo + n) of the
 * reference's mt19937_64(seed) U(-1, 1) n_global x nb block, row-major; the
 * solver's X0 / restart blocks (bit-identical to the reference's). */
be_status be_random_block(int64_t n, int64_t nb, uint64_t seed, int64_t row_lo, double* out);
be_status be_csb_view_get(const be_csb* m, be_csb_view* view);
/* is_strictly_lower (csb.hpp:188-202) on any view; *result = 0/1 */
be_status be_csb_is_strictly_lower(const be_csb_view* view, int* result);
/* to_triples (csb.hpp:165-185); out holds view->nnz triples */
be_status be_csb_to_triples(const be_csb_view* view, be_triple* out);
/* CSB1 binary cache (csb.hpp:204-302) plus the driver's appended diagonal
 * section (driver.hpp:136-161); diag may be NULL/0 for the bare format. */
be_status be_csb_save(const char* path, const be_csb_view* view, const double* diag, int64_t ndiag);
be_status be_csb_load(const char* path, be_csb** out, double** diag, int64_t* ndiag);
/* Block rows [brow_begin, brow_end) of a CSB1 cache (one rank's slab): global
 * shape and blocks, only that slab's index / value ranges read from disk;
 * diag (may be NULL) receives the cached diagonal of those rows. */
be_status be_csb_load_rows(const char* path, int64_t brow_begin, int64_t brow_end, be_csb** out, double** diag,
                           int64_t* ndiag);
/* The same CSB1 bytes in memory (save_csb / load_csb on std::ostream /
 * std::istream, csb.hpp:245-290): *bytes is released with be_free_buffer;
 * a bad magic or a truncated buffer is BE_ERR_PARSE. */
be_status be_csb_save_mem(const be_csb_view* view, const double* diag, int64_t ndiag, char** bytes, int64_t* len);
be_status be_csb_load_mem(const char* bytes, int64_t len, be_csb** out, double** diag, int64_t* ndiag);
void be_free_buffer(void* p);

/* Matrix Market ingest (ingest_matrix_market / _file, matrix_market.hpp:38-94):
 * coordinate real|integer symmetric input; entries of either triangle become
 * strictly-lower triples (file order), diagonal entries a dense diag[n]
 * (0 where absent). BE_ERR_PARSE for a malformed file, BE_ERR_NOT_SYMMETRIC_HEADER
 * for a non-symmetric header, BE_ERR_DUPLICATE_ENTRY for a repeated diagonal
 * entry. *lower and *diag are released with be_free_buffer. */
be_status be_mm_parse(const char* text, int64_t len, int64_t* n, be_triple** lower, int64_t* nlower, double** diag);
be_status be_mm_read_file(const char* path, int64_t* n, be_triple** lower, int64_t* nlower, double** diag);
/* write_matrix_market (matrix_market.hpp:98-113): NUL-terminated text, released with be_free_buffer */
be_status be_mm_write(int64_t n, const be_triple* lower, int64_t nlower, const double* diag, char** text,
                      int64_t* len);
void be_csb_free(be_csb* m);

/* ------------------------------------------------------------------------- */
/* Synthetic inputs (tooling, not the hot path).                              */
/* ------------------------------------------------------------------------- */

typedef enum be_synth_kind { BE_SYNTH_BANDED = 0, BE_SYNTH_BLOCKTILE = 1, BE_SYNTH_RANDOM = 2 } be_synth_kind;

typedef struct be_synth_params { /* SynthParams, synth.hpp:33-56 */
    int kind;
    int64_t n;
    double density;
    int64_t bandwidth;
    int64_t block_extent;
    int64_t tile_min, tile_max;
    double diag_spread;
    double dominance;
    uint64_t seed;
} be_synth_params;

typedef struct be_synth be_synth;
/* generate_synthetic (synth.hpp:92-158): identical triples, diagonal and tile
 * offsets for identical params (same mt19937_64 stream). */
be_status be_generate_synthetic(const be_synth_params* p, be_synth** out);
be_status be_synth_get(const be_synth* s, const be_triple** lower, int64_t* nlower,
                       const double** diag, const int64_t** tile_offsets, int64_t* n_tile_offsets);
void be_synth_free(be_synth* s);

/* Clustered generator for the Test-1..3 shapes (new): CSB blocks
 * of block_extent, occupied tile x tile sub-tiles at fill `fill`, counter-based
 * RNG keyed by (seed, block, tile) so generation is parallel and
 * deterministic. Writes a CSB directly (no triple list) plus the diagonal
 * 0.5 + U(0, diag_spread) + dominance * sum|row| and the log-uniform
 * preconditioner tile offsets of synth.hpp:67-83. */
typedef struct be_cluster_params {
    int64_t n;
    int64_t target_nnz;     /* strictly-lower nonzeros wanted (approximate) */
    int64_t block_extent;   /* CSB block extent (4000) */
    int64_t tile;           /* occupied sub-tile edge (128) */
    double fill;            /* within-tile fill (0.10) */
    double block_occupancy; /* fraction of lower CSB blocks holding tiles (1.0 = all) */
    int64_t tile_min, tile_max;
    double diag_spread, dominance;
    uint64_t seed;
    int threads;            /* 0 = all hardware threads */
} be_cluster_params;
be_status be_generate_clustered(const be_cluster_params* p, be_csb** out, double** diag,
                                int64_t** tile_offsets, int64_t* n_tile_offsets);
/* One rank's part of the same matrix (multi-GPU weak scaling): block rows
 * [brow_begin, brow_end) as a CSB of the global shape (diag_blocks_only: just
 * their diagonal blocks), the part's contribution to sum|row| of all n rows
 * (sum the parts over ranks, then be_clustered_diag), and the tile offsets. */
be_status be_generate_clustered_part(const be_cluster_params* p, int64_t brow_begin, int64_t brow_end,
                                     int diag_blocks_only, be_csb** out, double** rowabs,
                                     int64_t** tile_offsets, int64_t* n_tile_offsets);
/* diag[i - row_begin] = 0.5 + U_i(0, diag_spread) + dominance * rowabs[i - row_begin] */
be_status be_clustered_diag(const be_cluster_params* p, const double* rowabs, int64_t row_begin, int64_t row_end,
                            double* diag);
/* expected stored nonzeros per CSB block row (the slab weights, no generation) */
be_status be_clustered_weights(const be_cluster_params* p, int64_t* weights, int64_t* nblk);
/* Expected stored entries of every lower block (row-major nblk x nblk; weights NULL: nblk only) --
 * the weights of be_dist_tiles2d -- and one 2-D tile of the clustered matrix: block rows
 * [brow_begin, brow_end) x block columns [bcol_begin, bcol_end), exactly the whole-matrix
 * generator's entries there; rowabs / tile offsets as be_generate_clustered_part. */
be_status be_clustered_block_weights(const be_cluster_params* p, int64_t* weights, int64_t* nblk);
be_status be_generate_clustered_tile(const be_cluster_params* p, int64_t brow_begin, int64_t brow_end,
                                     int64_t bcol_begin, int64_t bcol_end, be_csb** out, double** rowabs,
                                     int64_t** tile_offsets, int64_t* n_tile_offsets);

/* ------------------------------------------------------------------------- */
/* Device context and the symmetric operator (SymmetricOperator,             */
/* kernels.hpp:339-378).                                                      */
/* ------------------------------------------------------------------------- */

typedef struct be_ctx be_ctx;
be_status be_ctx_create(int device, be_ctx** out);
be_status be_ctx_destroy(be_ctx* ctx);
be_status be_ctx_stream(be_ctx* ctx, void** stream);
be_status be_ctx_synchronize(be_ctx* ctx);
/* kernel-launch counter of this context (evidence for bench gpu_launches) */
be_status be_ctx_launches(be_ctx* ctx, int64_t* launches);

typedef struct be_op be_op;

enum { BE_OP_SYMMETRIC = 1, BE_OP_DETERMINISTIC = 2, BE_OP_FORMAT_TILES = 4, BE_OP_FORMAT_ROWS = 8 };
/* Upload a CSB to the device and derive the tile format.
 * flags & BE_OP_SYMMETRIC: validates square + strictly lower + diag length
 * like the SymmetricOperator constructor (kernels.hpp:341-350); diag (host,
 * nrows doubles) is copied. Without the flag the matrix may be rectangular
 * and only the NOTRANS/TRANS accumulate modes are valid (diag ignored).
 * flags & BE_OP_DETERMINISTIC: f64 values, every output element summed by one
 * thread in the reference's serial order (run_baseline, kernels.hpp:253-276:
 * L's entries of the row in CSB order, then L^T's, then the diagonal; no FMA
 * contraction) -- bit-reproducible and bit-identical to the serial reference
 * on f64 panels; reads each stored entry twice (the reference's two passes).
 * Device format of the fast path (f32 values): BE_OP_FORMAT_TILES forces the
 * 128 x 128 tile format (dense clustered matrices: each entry read once and
 * applied twice, X rows staged in shared memory), BE_OP_FORMAT_ROWS the
 * row-list format (L and L^T rows, X rows gathered from L2: very sparse
 * matrices, where a 128 x 128 tile holds too few entries to amortise its
 * staging); neither flag: chosen from the matrix (rows when it has >= 2^22
 * entries and fewer than 384 per occupied 128 x 128 sub-tile). */
be_status be_op_create(be_ctx* ctx, const be_csb_view* L, const double* diag, int values_prec,
                       int flags, be_op** out);
/* The symmetric operator streamed from a CSB1 cache file (be_csb_save with its diagonal section;
 * the bytes load_csb, csb.hpp:264-290, and the driver's diagonal section, driver.hpp:136-161,
 * read): batches of about batch_entries stored entries (whole block rows; <= 0: 2^26) are read by
 * a loader thread while the previous batch is cut into tiles and uploaded, so the whole matrix is
 * never resident on the host. flags must hold BE_OP_SYMMETRIC; the tile format is built (the same
 * tiles as be_op_create with BE_OP_FORMAT_TILES). diag (optional, be_free_buffer): the diagonal. */
be_status be_op_create_csb1(be_ctx* ctx, const char* path, int values_prec, int flags, int64_t batch_entries,
                           double** diag, int64_t* ndiag, be_op** out);
be_status be_op_destroy(be_op* op);

/* Y = op(X) on device panels of type panel_prec (BE_F32 / BE_F64),
 * row-major nrows x nb. mode: be_apply_mode. X and Y must not alias
 * (kernels.hpp:284). */
be_status be_op_apply(be_op* op, const void* X_dev, void* Y_dev, int64_t nrows, int nb,
                      int panel_prec, int mode, void* stream);
/* Host-buffer adapter: fp64 host panels in and out (Y read for the
 * accumulate modes), copies inside the call. */
be_status be_op_apply_host(be_op* op, const double* X, double* Y, int64_t nrows, int nb, int mode);

typedef struct be_op_info {
    int64_t nrows, ncols, nnz;
    int64_t ntiles;          /* device work tiles */
    int64_t device_bytes;    /* tile-format bytes resident in HBM */
    int64_t bytes_per_nnz_x1000;
    int values_prec;
    int tile_rows, tile_cols, tile_max_nnz;
} be_op_info;
be_status be_op_get_info(const be_op* op, be_op_info* info);

/* Decode the device tile format back to global coordinates in device order
 * (row, col, value) plus, for each entry, its index in the source CSB arrays.
 * Used by the bit-exact indexing tests. Buffers hold info.nnz entries. */
be_status be_op_decode(be_op* op, int64_t* rows, int64_t* cols, double* values, int64_t* csb_index);

/* Average device time (ms) of the dominant SpMM kernel over the last `n`
 * applies, measured with CUDA events on the launching stream. */
be_status be_op_timing(be_op* op, int enable, double* last_kernel_ms, double* last_apply_ms);

/* ------------------------------------------------------------------------- */
/* Block-diagonal FOM preconditioner (precond.hpp).                           */
/* ------------------------------------------------------------------------- */

typedef struct be_tiles be_tiles;
/* extract_tiles (precond.hpp:63-127) + upload. */
be_status be_tiles_create(be_ctx* ctx, const be_csb_view* L, const double* diag,
                          const int64_t* tile_offsets, int64_t n_tile_offsets, be_tiles** out);
be_status be_tiles_destroy(be_tiles* t);
/* Host copy of tile j in the reference's SparseTile layout (precond.hpp:18-30):
 * query sizes with NULL buffers. */
be_status be_tiles_get(const be_tiles* t, int64_t j, int64_t* dim, int64_t* nentries, int32_t* rows,
                       int32_t* cols, double* values, int64_t* diag_pos);
be_status be_tiles_count(const be_tiles* t, int64_t* count, int64_t* dim, int64_t* nentries);
/* W = K^{-1} R (apply_preconditioner, precond.hpp:287-317). Device fp64
 * panels; shifts_dev: nb doubles on device; fallbacks_dev: one int64 on
 * device incremented by the number of singular columns (may be NULL). */
be_status be_precond_apply(be_tiles* t, const double* shifts_dev, const double* R_dev, double* W_dev,
                           int64_t nrows, int nb, int m, int64_t* fallbacks_dev, void* stream);
/* Tiles given explicitly in the reference's SparseTile layout (precond.hpp:18-30):
 * tile j has dims[j] rows (consecutive row ranges), entries
 * [entry_offsets[j], entry_offsets[j+1]) of rows / cols / values (tile-local
 * indices) and its diagonal slots at diag_pos[sum(dims[<j]) + i] (relative to
 * the tile's first entry). Used by the mirror's fom_solve_tile. */
be_status be_tiles_create_explicit(be_ctx* ctx, int64_t ntiles, const int64_t* dims, const int64_t* entry_offsets,
                                   const int32_t* rows, const int32_t* cols, const double* values,
                                   const int64_t* diag_pos, be_tiles** out);
be_status be_precond_apply_host(be_tiles* t, const double* shifts, const double* R, double* W,
                                int64_t nrows, int nb, int m, int64_t* fallbacks);

/* ------------------------------------------------------------------------- */
/* LOBPCG (lobpcg.hpp:291-456), device-resident.                              */
/* ------------------------------------------------------------------------- */

typedef struct be_solver_config { /* SolverConfig lobpcg.hpp:24-48 */
    int k;
    int nb;                 /* 0 -> k + 3 */
    double tol;
    int maxiter;
    int fom_iterations;     /* FomConfig::iterations precond.hpp:51-57 */
    uint64_t seed;
    int observer_state;     /* 1: copy the SolverState panels to host for the observer */
} be_solver_config;

/* Per-iteration hook (SolverConfig::observer, lobpcg.hpp:33-34, 436) with the
 * SolverState of lobpcg.hpp:52-58: x, hx, w, hw, p, hp are host n x nb copies
 * of X, HX, the iteration's W and HW, and the updated P, HP when
 * observer_state, else NULL (p_active is true after every iteration,
 * lobpcg.hpp:406). */
typedef void (*be_observer_fn)(void* user, int iter, int64_t n, int nb, const double* theta,
                               const double* residual_norms, int n_converged, const double* x,
                               const double* hx, const double* w, const double* hw, const double* p,
                               const double* hp);
/* Generic host operator (lobpcg.hpp:20): out = H in on host panels. */
typedef int (*be_host_operator_fn)(void* user, const double* in, double* out, int64_t n, int nb);

typedef struct be_result be_result;
/* lobpcg_solve: exactly one of op / host_op is used (op wins). precond and
 * x0 (host, n x nb) may be NULL. */
be_status be_lobpcg_solve(be_ctx* ctx, be_op* op, be_host_operator_fn host_op, void* host_op_user,
                          int64_t n, be_tiles* precond, const double* x0, const be_solver_config* cfg,
                          be_observer_fn observer, void* observer_user, be_result** out);

/* Incremental form of the same solve (bench and iteration-level timing):
 * begin = validation + X0 CholQR + first operator call + initial
 * Rayleigh-Ritz (lobpcg.hpp:293-335); step runs up to `count` further
 * iterations (*done receives how many; stops at convergence or maxiter);
 * end returns the SolveResult and releases the solver. */
typedef struct be_solver be_solver;
be_status be_lobpcg_begin(be_ctx* ctx, be_op* op, be_host_operator_fn host_op, void* host_op_user, int64_t n,
                          be_tiles* precond, const double* x0, const be_solver_config* cfg, be_solver** out);
be_status be_lobpcg_step(be_solver* s, int count, int* done);
be_status be_lobpcg_end(be_solver* s, be_result** out);

typedef struct be_result_info {
    int converged;
    int iterations;
    int k;
    int nb;
    int64_t n;
    int64_t operator_calls;
    int64_t precond_fallbacks;
    int restarts;
} be_result_info;
be_status be_result_get_info(const be_result* r, be_result_info* info);
/* lambda: k values; x: n x k row-major. */
be_status be_result_get(const be_result* r, double* lambda, double* x);
/* IterationRecord lobpcg.hpp:60-66 for iteration index i (0-based):
 * theta and residual_norms hold nb values. */
be_status be_result_get_record(const be_result* r, int i, double* theta, double* residual_norms,
                               int* n_converged, double* t_spmm, double* t_precond, double* t_dense,
                               double* t_total);
void be_result_free(be_result* r);

/* ------------------------------------------------------------------------- */
/* Multi-GPU (dist.hpp). One rank per GPU; the reference's simulated          */
/* collectives (SimComm, dist.hpp:85-89; distributed_spmm :256-371;           */
/* distributed_gram_allreduce :375-391) become NCCL allgather /               */
/* reduce-scatter / allreduce over NVLink. A second backend runs the ranks    */
/* as threads of one process (any devices, several ranks per GPU allowed):    */
/* the same code path, exercised on a single GPU.                             */
/* ------------------------------------------------------------------------- */

typedef struct be_comm be_comm;
typedef struct be_comm_group be_comm_group;
/* ncclGetUniqueId: rank 0 creates it and ships the 128 bytes to the others */
be_status be_comm_nccl_id(uint8_t id[128]);
be_status be_comm_create_nccl(be_ctx* ctx, const uint8_t id[128], int rank, int world, be_comm** out);
/* in-process rank group: one be_comm_create_local per rank, each from its own
 * host thread (creation and every collective are group-wide barriers) */
be_status be_comm_group_create(int world, be_comm_group** out);
be_status be_comm_group_destroy(be_comm_group* g);
/* release every rank blocked in (or later entering) a collective of the group
 * with BE_ERR_PROTOCOL_DEADLOCK: called by a rank that failed */
be_status be_comm_group_abort(be_comm_group* g);
be_status be_comm_create_local(be_ctx* ctx, be_comm_group* g, int rank, be_comm** out);
be_status be_comm_destroy(be_comm* c);
/* backend: 0 = NCCL, 1 = local; calls / bytes: collectives issued and bytes
 * received by this rank (the SimComm counters) */
be_status be_comm_info(const be_comm* c, int* rank, int* world, int* backend, int64_t* calls, int64_t* bytes);
/* in-place sum over ranks of count device doubles (distributed_gram_allreduce) */
be_status be_comm_allreduce_f64(be_comm* c, double* buf_dev, int64_t count, void* stream);

/* Partition rules (integer-exact; every rank derives the same cuts).
 * be_dist_rows: panel-row ownership, world + 1 cuts on the block boundaries
 *   `bounds` (nbounds entries), cut p the boundary closest to n p / world.
 * be_dist_balance: contiguous item ranges of near-equal weight (world + 1 item
 *   indices), e.g. CSB block rows weighted by their stored nonzeros: the
 *   nnz-balanced SpMM slabs. Replaces partition_matrix's fixed triangular
 *   layout (dist.hpp:113-198, nd(nd+1)/2 ranks only) for any rank count. */
be_status be_dist_rows(const int64_t* bounds, int64_t nbounds, int world, int64_t* cuts);
/* Segment-wise exchange rule of the distributed operator:
 * touched[r] = 1 when a stored block of this rank's slab L_slab has rows or
 * columns in the panel segment owned by rank r (segment q = [cuts[q],
 * cuts[q+1]), owned by owner[q], identity when owner is NULL). X segment r is
 * sent to exactly the ranks that touch it, partial Y segment r only to rank r.
 * Host only; be_op_dist_need reads a distributed operator's world x world
 * matrix (row p = rank p's touched slots) as built at be_op_create_dist. */
be_status be_dist_touched(const be_csb_view* L_slab, const int64_t* cuts, const int* owner, int world,
                          uint8_t* touched);
be_status be_dist_balance(const int64_t* weights, int64_t nitems, int world, int64_t* cuts);
/* nnz-balanced 2-D tiles (north_star; replaces partition_matrix's fixed triangular layout,
 * dist.hpp:113-198, for any rank count): recursive coordinate bisection of the lower block grid.
 * weights[bi * nblk + bj] = stored entries of block (bi, bj), bi >= bj; bounds the nblk + 1 block
 * boundaries (the cut side is the longer one in matrix rows). rects: world x (r0, r1, c0, c1),
 * rank r owns the stored blocks with r0 <= bi < r1, c0 <= bj < c1 (empty: all zero). The
 * rectangles are disjoint and cover every non-empty block; see DESIGN.md §6 for the rule. */
be_status be_dist_tiles2d(const int64_t* weights, int64_t nblk, const int64_t* bounds, int world, int64_t* rects);

/* Distributed symmetric operator: L_slab is this rank's share of the global
 * strictly-lower CSB (global coordinates and blocks; the ranks' slabs are
 * disjoint and cover L), cuts the panel-row ownership (world + 1 entries on
 * block boundaries), diag_local the diagonal of rows [cuts[rank],
 * cuts[rank+1]). be_op_apply then maps local f64 panels (BE_APPLY_SYMMETRIC)
 * to local f64 panels: distributed_operator (dist.hpp:397-404) without the
 * host scatter / gather. be_lobpcg_* on such an operator run the distributed
 * solver: n = local rows, x0 = local rows of X0, the result holds local rows. */
be_status be_op_create_dist(be_ctx* ctx, be_comm* comm, const be_csb_view* L_slab, const int64_t* cuts,
                            const double* diag_local, int values_prec, be_op** out);
/* The same operator with segment ownership given explicitly: segment q is
 * rows [seg_bounds[q], seg_bounds[q+1]) (world + 1 bounds on block
 * boundaries), owned by rank seg_owner[q] (a permutation of the ranks). The
 * reference triangular layout below uses it (parity variant). */
be_status be_op_create_dist_owned(be_ctx* ctx, be_comm* comm, const be_csb_view* L_slab, const int64_t* seg_bounds,
                                  const int* seg_owner, const double* diag_local, int values_prec, be_op** out);
be_status be_op_dist_need(const be_op* op, uint8_t* need);

/* The reference's own layout (dist.hpp:25-198), restated bit-exactly:
 * build_layout: blocks[3 r .. 3 r + 2] = (i, j, transposed) of rank r over
 * n_ranks = nd (nd + 1) / 2 ranks, diagonal_ranks[g]; BE_ERR_EVEN_ND for an
 * even or non-positive nd (any output may be NULL). */
be_status be_tri_layout(int nd, int* blocks, int* diagonal_ranks, int* n_ranks);
/* segment_of_rank (dist.hpp:184-196): rank r owns rows [seg_begin[r], seg_end[r]) */
be_status be_tri_segments(int nd, const int64_t* sub_bounds, int64_t* seg_begin, int64_t* seg_end);
/* partition_matrix's routing (dist.hpp:142-163): the stored entries of `rank`
 * in global coordinates, in to_triples order (out NULL: *count receives the
 * number; else *count is the capacity on entry). */
be_status be_tri_rank_triples(const be_csb_view* L, int nd, const int64_t* sub_bounds, int rank, be_triple* out,
                              int64_t* count);

/* extract_tiles restricted to the tiles of rows [row_begin, row_end) (a union
 * of whole tiles of tile_offsets, which cover [0, n)); diag_local holds those
 * rows. L must contain the diagonal blocks of those rows. */
be_status be_tiles_create_range(be_ctx* ctx, const be_csb_view* L, const double* diag_local,
                                const int64_t* tile_offsets, int64_t n_tile_offsets, int64_t row_begin,
                                int64_t row_end, be_tiles** out);

/* ------------------------------------------------------------------------- */
/* Device dense kernels exposed for parity tests (densela.hpp).               */
/* ------------------------------------------------------------------------- */

/* out (p x q, column-major like SmallDense densela.hpp:19-47) = A^T B over
 * device fp64 panels A (n x p) and B (n x q); symmetrised when A == B
 * (gram, densela.hpp:70-99). out is a host buffer. */
be_status be_gram(be_ctx* ctx, const double* A_dev, int p, const double* B_dev, int q, int64_t n,
                  double* out);
/* k lowest eigenpairs of (A, B) with the pivot floor (sygv_lowest,
 * densela.hpp:357-407): host n x n column-major inputs, outputs
 * c (n x k column-major) and d (k), computed on the device. */
be_status be_sygv_lowest(be_ctx* ctx, const double* A, const double* B, int n, int k,
                         double pivot_floor, double* c, double* d);

/* The n-row panel functions of densela.hpp / lobpcg.hpp on HOST buffers (the
 * C++ mirror's entry points, used by the reference's own unit suites): the
 * panels are uploaded, the solver's device kernels run, the results come
 * back. Panels are row-major n x w, small matrices column-major. */
/* gram (densela.hpp:70-99): out (p x q) = A^T B; same != 0 symmetrises (gram(a, a)) */
be_status be_dense_gram(be_ctx* ctx, const double* A, int p, const double* B, int q, int64_t n, int same,
                        double* out);
/* cholesky (rel_floor = 0, densela.hpp:103-121) / cholesky_floored (densela.hpp:155-175):
 * R upper, B = R^T R; BE_ERR_NOT_POSITIVE_DEFINITE with the pivot index */
be_status be_dense_cholesky(be_ctx* ctx, const double* B, int n, double rel_floor, double* R);
/* trsm_right_inv (densela.hpp:125-147): W <- W R^{-1}; BE_ERR_SINGULAR_TRIANGULAR */
be_status be_dense_trsm(be_ctx* ctx, double* W, int64_t n, int nb, const double* R);
/* qr_of_transpose (densela.hpp:412-445): X <- Q, R (nb x nb) with X = Q R; BE_ERR_RANK_DEFICIENT */
be_status be_dense_qr(be_ctx* ctx, double* X, int64_t n, int nb, double* R);
/* block_times_small(_add) (densela.hpp:448-484): Y (n x q) (+)= X (n x p) C (p x q) */
be_status be_dense_mix(be_ctx* ctx, const double* X, int64_t n, int p, const double* C, int q, double* Y,
                       int accumulate);
/* residual_block (lobpcg.hpp:197-213) + the column sums of squares of R and X (may be NULL) */
be_status be_dense_residual(be_ctx* ctx, const double* HX, const double* X, const double* theta, int64_t n, int nb,
                            double* R, double* rnorm2, double* xnorm2);
/* per-column sums of squares (column_norm^2, block_vector.hpp:55-62) */
be_status be_dense_colnorm2(be_ctx* ctx, const double* A, int64_t n, int nb, double* out);
/* rayleigh_ritz (lobpcg.hpp:113-157): c ((2 or 3) nb x k_keep, column-major), theta (k_keep);
 * P and HP both NULL for the 2 nb pencil; BE_ERR_BASIS_DEGENERATE on a failed overlap Cholesky */
be_status be_rayleigh_ritz(be_ctx* ctx, const double* X, const double* W, const double* P, const double* HX,
                           const double* HW, const double* HP, int64_t n, int nb, int k_keep, double* c,
                           double* theta);
/* update_blocks (lobpcg.hpp:168-194): C1, C2, C3 are nb x m; outputs n x m (P, HP, C3 NULL without P) */
be_status be_update_blocks(be_ctx* ctx, const double* X, const double* W, const double* P, const double* HX,
                           const double* HW, const double* HP, int64_t n, int nb, int m, const double* C1,
                           const double* C2, const double* C3, double* Xo, double* HXo, double* Po, double* HPo);

#ifdef __cplusplus
}
#endif
#endif /* BLOCKEIG_B200_H */
