/* rsylv-b200: B200-native (sm_100a) robust triangular Sylvester solver — C-ABI boundary.
 *
 * Solves  A*Y + Y*B = alpha*C  for upper quasi-triangular A (m x m) and B (n x n) in real
 * Schur form (1x1 and 2x2 diagonal blocks), with every tile of Y kept below the overflow
 * threshold omega through per-tile power-of-two scale factors (arXiv:1905.10574, Alg. 4).
 *
 * This header is the drop-in boundary for the reference entry point
 *     rsylv::solve_tiled_robust(const QuasiTriangular& a, const QuasiTriangular& b,
 *                               ConstMatrixView c, std::size_t tile_size,
 *                               const OverflowConfig& cfg, ExecutionMode mode,
 *                               const TileProbe& probe)
 *   (/root/reference/proj/include/rsylv/tiled_solve.hpp:36-40, defined in
 *    /root/reference/proj/src/tiled_solve.cpp:183-194).
 * The C++ shim in shim/rsylv_b200_shim.cpp defines that exact symbol on top of this ABI and maps
 * the status codes back to the reference exceptions (errors.hpp:10-37). Plain pointers and sizes
 * only; matrices are column-major with a leading dimension exactly like ConstMatrixView
 * (dense_matrix.hpp:12-30).
 *
 * Diagonal block structure (QuasiTriangular::diag_blocks, partition.hpp:15-42) is passed as one
 * byte per index: blk[i] = 1 -> 1x1 block at i; 2 -> 2x2 block at (i, i+1); 0 -> second index
 * of a 2x2 block. NULL means all 1x1.
 */
#ifndef RSYLV_B200_H
#define RSYLV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. Reference exception each one maps to (errors.hpp, tiled_solve.cpp:187-188,
 * partition.cpp:75-76, tile_grid.cpp:63-72, tiled_solve.cpp:77-79): */
enum {
    RSYLV_OK = 0,
    RSYLV_INVALID_ARGUMENT = 1, /* std::invalid_argument                                      */
    RSYLV_SINGULAR = 2,         /* SingularEquationError(pivot)                               */
    RSYLV_SCALE_UNDERFLOW = 3,  /* ScaleUnderflowError: alpha < DBL_MIN. Y and alpha_exp are  */
                                /* still returned (exponent form).                             */
    RSYLV_CUDA_ERROR = 4,       /* device/runtime failure                                     */
    RSYLV_NO_DEVICE = 5         /* no CUDA device / extension unusable: never a CPU fallback  */
};

/* Why an RSYLV_INVALID_ARGUMENT was raised (the reference's distinct throw sites). */
enum {
    RSYLV_REASON_NONE = 0,
    RSYLV_REASON_NONCONFORMING = 1, /* tiled_solve.cpp:187-188 */
    RSYLV_REASON_TILE_SIZE = 2,     /* partition.cpp:75-76      */
    RSYLV_REASON_A_BOUND = 3,       /* tile_grid.cpp:63-64      */
    RSYLV_REASON_B_BOUND = 4,       /* tile_grid.cpp:71-72      */
    RSYLV_REASON_C_BOUND = 5,       /* tiled_solve.cpp:77-79    */
    RSYLV_REASON_OPTIONS = 6
};

typedef struct {
    double omega;      /* OverflowConfig::omega (overflow.hpp:15); 0 -> DBL_MAX/2           */
    double small_num;  /* OverflowConfig::small_num (overflow.hpp:18); 0 -> DBL_MIN/eps      */
    size_t tile_size;  /* requested tile size (>= 2). The device works on tiles of at most
                          128 (one CTA per tile): a larger request is served by 128-tiles.
                          alpha, scaling_events and the probe's (k, l) indices follow that
                          internal partition (cut moved one index earlier around a 2x2 block);
                          Y/alpha does not depend on it                                     */
    int scheduler;     /* 0: persistent dataflow kernel (default), 1: host-driven wavefront */
    int virtual_ranks; /* >1: emulate that many GPUs on this device (tile columns block-cyclic,
                          solved tiles pushed between per-rank workspaces) -- validates the
                          multi-GPU exchange on one GPU; 0/1 = off                          */
    int host_pipeline; /* rsylv_b200_solve only: stream the inputs in while the solve runs
                          (H2D + pack in shells: tile row of A from its diagonal on, tile
                          column of B, the matching L-shaped piece of C). 0: automatic (from
                          64 tiles), 1: always, -1: never (copy everything first)          */
    int fast_diag;     /* diagonal-tile solves: 0 (default) = the exact exponent-form sub-block
                          path; 1 = a plain-FP64 attempt on the power-of-two normalized tile
                          first (tiles of 1x1 blocks), the exact path only when a pivot /
                          range check fails (Y/alpha agree to rounding either way)          */
} rsylv_b200_options;

/* One TileProbe event (tiled_solve.hpp:24-27): tile (k, l) came to rest with local scale
 * 2^scale_exp and cached inf-norm `norm`. */
typedef struct {
    uint32_t k, l;
    int32_t scale_exp;
    int32_t pad;
    double norm;
} rsylv_b200_probe_event;

typedef struct {
    double alpha;             /* 2^alpha_exp when >= DBL_MIN, else 0                        */
    int32_t alpha_exp;        /* alpha as a power-of-two exponent (always set on OK/UNDERFLOW) */
    int32_t invalid_reason;   /* RSYLV_REASON_*                                            */
    uint64_t scaling_events;  /* guard activations (OverflowConfig::scaling_events)         */
    double pivot;             /* offending pivot for RSYLV_SINGULAR                         */
    double device_ms;         /* device time of the solve (pack .. unpack), CUDA events     */
    double max_tile_norm;     /* max inf-norm over the returned tiles of Y (<= omega)       */
    size_t row_tiles, col_tiles;
    /* optional probe log: caller-owned buffer; probe_count receives the number of events
     * produced (may exceed probe_cap; only the first probe_cap are written) */
    rsylv_b200_probe_event* probe_log;
    size_t probe_cap;
    size_t probe_count;
    /* device-time breakdown (CUDA events on the solve stream) */
    double pack_ms;           /* pack + tile norms (TileGrid + compute_bounds)               */
    double dag_ms;            /* tile DAG: update GEMMs + diagonal solves                    */
    double unpack_ms;         /* consistency scaling + copy-out                              */
    uint64_t dag_launches;    /* kernel launches inside the DAG phase                        */
    uint64_t h2d_bytes;       /* host->device bytes moved by rsylv_b200_solve                */
    uint64_t d2h_bytes;       /* device->host bytes moved by rsylv_b200_solve                */
} rsylv_b200_result;

typedef struct rsylv_b200_ctx rsylv_b200_ctx;

/* Create a context on CUDA device `device` (0-based; -1 = current). */
int rsylv_b200_create(int device, rsylv_b200_ctx** out);
void rsylv_b200_destroy(rsylv_b200_ctx* ctx);
const char* rsylv_b200_status_string(int status);
/* Last CUDA error text of the context (for RSYLV_CUDA_ERROR). */
const char* rsylv_b200_last_error(const rsylv_b200_ctx* ctx);

/* Drop-in solve on HOST buffers (the reference's calling convention). Copies A, B, C to the
 * device, solves, copies Y (m x n, leading dimension ldy) back. Replaces
 * rsylv::solve_tiled_robust (tiled_solve.hpp:36-40). */
int rsylv_b200_solve(rsylv_b200_ctx* ctx, size_t m, size_t n, const double* a, size_t lda,
                     const unsigned char* ablk, const double* b, size_t ldb,
                     const unsigned char* bblk, const double* c, size_t ldc, double* y,
                     size_t ldy, const rsylv_b200_options* opt, rsylv_b200_result* res);

/* Same solve on DEVICE-resident buffers (a, b, c, y are device pointers; ablk/bblk are host
 * arrays). `stream` is a cudaStream_t (NULL = legacy default stream). */
int rsylv_b200_solve_device(rsylv_b200_ctx* ctx, size_t m, size_t n, const double* a,
                            size_t lda, const unsigned char* ablk, const double* b, size_t ldb,
                            const unsigned char* bblk, const double* c, size_t ldc, double* y,
                            size_t ldy, const rsylv_b200_options* opt, void* stream,
                            rsylv_b200_result* res);

/* ---- multi-GPU in one process (the drop-in path for ExecutionMode::workers > 1): R contexts on
 * R distinct GPUs (rsylv_b200_create per device), HOST buffers as rsylv_b200_solve. Tile columns
 * block-cyclic over the GPUs (column j on ctxs[j % R]); each GPU stores the upper tiles of A and B
 * and its own tile columns of C; solved tiles are pushed to the peers over NVLink (peer
 * access), alpha is the MIN over the GPUs. R = 1 is rsylv_b200_solve on ctxs[0]. */
int rsylv_b200_solve_group(rsylv_b200_ctx* const* ctxs, int R, size_t m, size_t n,
                           const double* a, size_t lda, const unsigned char* ablk, const double* b,
                           size_t ldb, const unsigned char* bblk, const double* c, size_t ldc,
                           double* y, size_t ldy, const rsylv_b200_options* opt,
                           rsylv_b200_result* res);
/* 1 when the opt-in fast diagonal-tile path (rsylv_b200_options.fast_diag) is compiled in
 * (make EXTRA=-DRSYLV_FAST_DIAG_BUILD=1); otherwise fast_diag requests run the exact path. */
int rsylv_b200_has_fast_diag(void);
/* Visible CUDA devices (0 when none / the driver is unusable). */
int rsylv_b200_device_count(void);

/* ---- multi-GPU (one process per GPU; tile columns block-cyclic, column j on rank j % nranks).
 * Sequence per solve (the caller provides the collectives, e.g. torch.distributed):
 *   1. rsylv_b200_dist_prepare  : partition, allocate, pack, validate; writes this rank's IPC
 *                                 handles (RSYLV_DIST_HANDLE_BYTES) for the peers
 *   2. all-gather the handles; barrier (every rank packed before anyone pushes)
 *   3. rsylv_b200_dist_run      : persistent kernel on the owned columns; solved tiles are pushed
 *                                 over NVLink into the peers that consume them; returns the local
 *                                 alpha exponent minimum (res->alpha_exp) and the local
 *                                 max_tile_norm relative to it
 *   4. all-reduce MIN / MAX of those two, then
 *   5. rsylv_b200_dist_finish   : consistency scaling to the global alpha + copy-out of the
 *                                 owned columns of Y (other columns are left untouched). */
#define RSYLV_DIST_HANDLE_BYTES 320
int rsylv_b200_dist_prepare(rsylv_b200_ctx* ctx, int nranks, int rank, size_t m, size_t n,
                            const double* a, size_t lda, const unsigned char* ablk,
                            const double* b, size_t ldb, const unsigned char* bblk,
                            const double* c, size_t ldc, const rsylv_b200_options* opt,
                            void* stream, void* handle_out, rsylv_b200_result* res);
int rsylv_b200_dist_run(rsylv_b200_ctx* ctx, const void* all_handles, void* stream,
                        rsylv_b200_result* res);
int rsylv_b200_dist_finish(rsylv_b200_ctx* ctx, int alpha_exp, double* y, size_t ldy,
                           void* stream, rsylv_b200_result* res);

/* One robust augmented-tile update <gamma,C> <- <gamma,C> - <alpha,A><beta,B>
 * (rsylv::robust_update, robust_update.hpp:32-33) on the device, scales as exponents:
 * gamma = 2^c_exp, alpha*beta = 2^ab_exp. C is m x n (ld m), A m x k, B k x n, HOST buffers.
 * On return c holds the updated tile, *c_exp its new exponent and *c_norm its inf-norm. */
int rsylv_b200_robust_update(rsylv_b200_ctx* ctx, size_t m, size_t k, size_t n, double* c,
                             int32_t* c_exp, double* c_norm, const double* a, const double* b,
                             int32_t ab_exp, double omega, uint64_t* events);

/* Development counters: accumulated cycles per tile-task phase over all tasks since the last
 * reset (0 update GEMM, 1 solve setup, 2 sub-block solves, 3 in-tile updates, 4 finalize). */
int rsylv_b200_debug_counters(unsigned long long* out32, int reset);
/* Development: average cycles of one warp-level 16x16 sub-block solve (mode bit 0: 2x2 blocks,
 * bit 1: force the exact solver); out256 (nullable) receives the solution, column-major. */
int rsylv_b200_debug_subsolve(int reps, int mode, long long* cycles, double* out256);

/* Development / test entries for the pieces of the diagonal-tile solver (HOST buffers):
 * rsylv_b200_debug_small_solve: n independent 1x1 / 2x1 / 1x2 / 2x2 block Sylvester solves
 *   a_t z + z b_t = c_t (rs[t], cs[t] in {1, 2}; a, b, c, z 2x2 column-major per case) with the
 *   exact path's complete-pivoting Kronecker solve and division guard (small_solve.cpp:15-106):
 *   on return A z + z B = 2^-dz[t] c, status[t] 0 ok / 2 singular (pivot[t]).
 * rsylv_b200_debug_guards: the exponent-form guards for n inputs -- update guard of
 *   (c + a b) (ProtectUpdate, overflow.cpp:15-40) in the xq integer form (update-phase source
 *   headers) and the xf form (in-tile updates), division guard of bnd / |t| (ProtectDivision,
 *   overflow.cpp:48-64; -1 for t = 0). Each returns d: the scale factor is 2^-d. */
int rsylv_b200_debug_small_solve(size_t n, const int32_t* rs, const int32_t* cs, const double* a,
                                 const double* b, const double* c, double omega,
                                 double small_num, double* z, int32_t* dz, int32_t* status,
                                 double* pivot);
int rsylv_b200_debug_guards(size_t n, const double* c, const double* a, const double* b,
                            const double* bnd, const double* t, double omega, int32_t* d_upd_xq,
                            int32_t* d_upd_xf, int32_t* d_div);

/* ---- FP64 GEMM and residual on the DMMA tensor path (device buffers, column-major) ----
 * C = alpha * op(A) * op(B) + beta * C with op = transpose when ta / tb != 0 (op(A) m x k,
 * op(B) k x n). a_upper: op(A) is upper quasi-triangular (zero below the first subdiagonal),
 * b_upper: op(B) likewise -- the structural zeros are skipped. stream: cudaStream_t (NULL =
 * legacy default stream). Used by the Bartels-Stewart transforms and the residual below. */
int rsylv_b200_dgemm(rsylv_b200_ctx* ctx, int ta, int tb, size_t m, size_t n, size_t k,
                     double alpha, const double* a, size_t lda, const double* b, size_t ldb,
                     double beta, double* c, size_t ldc, int a_upper, int b_upper, void* stream);

/* Relative residual of a solve (src/testgen.cpp:64-79, made overflow-safe):
 *   || A Y + Y B - 2^alpha_exp C ||_F / ((||A||_F + ||B||_F) ||Y||_F + 2^alpha_exp ||C||_F)
 * evaluated on the device in a power-of-two prescaled frame (Y * 2^s with max |Y * 2^s| <=
 * 2^400), so that tiles near omega and alpha far below DBL_MIN stay representable. A (m x m)
 * and B (n x n) are the dense upper quasi-triangular matrices. out[0] = relative residual,
 * out[1..5] = ||R||, ||A||, ||B||, ||Y 2^s||, ||2^(alpha+s) C|| (Frobenius), out[6] = s. */
int rsylv_b200_relative_residual(rsylv_b200_ctx* ctx, size_t m, size_t n, const double* a,
                                 size_t lda, const double* b, size_t ldb, const double* c,
                                 size_t ldc, const double* y, size_t ldy, int32_t alpha_exp,
                                 void* stream, double* out7);

/* ---- benchmark input generation (harness utility; not part of the reference API) ----
 * Fills a device buffer (column-major, ld) with a quasi-triangular matrix whose strict upper
 * triangle is U(up_lo, up_hi), 1x1 diagonal entries U(d_lo, d_hi) and 2x2 blocks
 * [[a, b], [-c, a]] with a ~ U(d_lo, d_hi), b, c ~ U(off_lo, off_hi). Counter-based RNG keyed
 * by (seed, i, j): identical on every device and run. */
int rsylv_b200_generate_quasi_triangular(size_t n, double* dev, size_t ld,
                                         const unsigned char* blk_host, uint64_t seed,
                                         double up_lo, double up_hi, double d_lo, double d_hi,
                                         double off_lo, double off_hi, void* stream);
/* Dense m x n right-hand side: dist 0 = U(lo, hi), 1 = N(0, 1)*hi + lo. Tiles listed in
 * hot_tiles (pairs of nominal tile indices of size hot_tile) are multiplied by hot_factor. */
int rsylv_b200_generate_rhs(size_t m, size_t n, double* dev, size_t ld, uint64_t seed, int dist,
                            double lo, double hi, const int32_t* hot_tiles, size_t n_hot,
                            size_t hot_tile, double hot_factor, void* stream);

#ifdef __cplusplus
}
#endif
#endif
