// Host-side declarations of the kernel launch wrappers defined in kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace rsb {

size_t smem_task();
int has_fast_diag();
int bench_subsolve(int reps, int mode, long long* cycles_host, double* out256);
cudaError_t read_prof(unsigned long long* out);
cudaError_t reset_prof();
cudaError_t configure_kernels();

// normalize = false (the non-robust solve, omega = +inf): off-diagonal tiles stored unscaled
void launch_pack_upper(const double* src, long long ld, const int* cut, int T, int TSP,
                       double* dst, double* norms, int* sexp, cudaStream_t st,
                       bool normalize = true);
void launch_pack_full(const double* src, long long ld, const Problem& P, double* norms,
                      cudaStream_t st);
void launch_tile_diag(const Problem& P, int d, int ntiles, cudaStream_t st);
void launch_update_only(const Problem& P, int i, int j, cudaStream_t st);
void launch_update_bench(const Problem& P, int ctas, cudaStream_t st);
void launch_pack_upper_col(const double* src, long long ld, const int* cut, int T, int TSP,
                           double* dst, double* norms, int* sexp, int k, cudaStream_t st,
                           bool normalize = true);
void launch_pack_upper_row(const double* src, long long ld, const int* cut, int T, int TSP,
                           double* dst, double* norms, int* sexp, int row, cudaStream_t st,
                           bool normalize = true);
void launch_pack_full_col(const double* src, long long ld, const Problem& P, double* norms,
                          int j, int i0, cudaStream_t st);
void launch_pack_full_row(const double* src, long long ld, const Problem& P, double* norms,
                          int i, int jend, cudaStream_t st);
void launch_set_ready(int* ready, int a, int b, int c, cudaStream_t st);
void launch_validate_shell(const Problem& P, int* reason, int rA, int jB, int jC, int i0C, int rC,
                           int jendC, cudaStream_t st);
void launch_persistent(const Problem& P, int grid, cudaStream_t st);
cudaError_t launch_persistent_mr(const Problem* probs_dev, int nranks_here, int grid,
                                 cudaStream_t st);
void launch_unpack(const Problem& P, int alpha_exp, double* y, long long ldy, cudaStream_t st);
size_t smem_gemm();
void launch_debug_small(int n, const int* rs, const int* cs, const double* a, const double* b,
                        const double* c, double omega, double small_num, double* z, int* dz,
                        int* st, double* piv);
void launch_debug_guards(int n, const double* c, const double* a, const double* b,
                         const double* bnd, const double* t, double omega, int* dxq, int* dxf,
                         int* ddiv);
cudaError_t launch_dgemm(int ta, int tb, int m, int n, int k, double alpha, const double* A,
                         long long lda, const double* B, long long ldb, double beta, double* C,
                         long long ldc, int a_upper, int b_upper, cudaStream_t st);
cudaError_t launch_scale_copy(int m, int n, const double* src, long long lds, double* dst,
                              long long ldd, int e, cudaStream_t st);
cudaError_t launch_absmax_sumsq(int m, int n, const double* x, long long ld, int e, int blocks,
                                double* pmax, double* psum, cudaStream_t st);
void launch_gen_qt(int n, double* a, long long ld, const unsigned char* blk,
                   unsigned long long seed, double up_lo, double up_hi, double d_lo, double d_hi,
                   double off_lo, double off_hi, cudaStream_t st);
void launch_gen_rhs(int m, int n, double* c, long long ld, unsigned long long seed, int dist,
                    double lo, double hi, const int* hot, int nhot, int hot_tile,
                    double hot_factor, cudaStream_t st);

}  // namespace rsb
