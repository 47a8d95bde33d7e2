/* TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the rsylv-b200 parity tests.
 *
 * A plain-C restatement of the reference's sequential tiled robust Sylvester solve
 * (/root/reference/proj, arXiv:1905.10574 Alg. 1-4), written to be operation-for-operation
 * identical to the reference so that its outputs are bitwise equal to oracle/_ref (the
 * unmodified reference library) — that equality is what pins this oracle (tests/test_oracle.py).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may call it; the product
 * library never links it.
 *
 * Matrices are column-major with a leading dimension (dense_matrix.hpp:12-52). Diagonal block
 * structure uses the product convention: blk[i] = 1 (1x1 block at i), 2 (2x2 block at i, i+1),
 * 0 (second index of a 2x2 block).
 *
 * Status codes: 0 ok, 1 invalid_argument, 2 SingularEquationError, 3 ScaleUnderflowError.
 */
#ifndef RSYLV_ORACLE_H
#define RSYLV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void (*or_probe_fn)(size_t k, size_t l, double scale, double norm, void* user);

/* overflow.cpp:29-75 */
int or_protect_update(double cnorm, double anorm, double bnorm, double omega, double* zeta);
int or_protect_division(double numer_bound, double divisor, double omega, double* zeta,
                        double* pivot);

/* dense_matrix.cpp:8-31 */
double or_inf_norm(const double* p, size_t rows, size_t cols, size_t ld);

/* small_solve.cpp:15-108,126-141 (guarded flavor, in place on z which holds C on entry) */
int or_small_sylvester(size_t ma, size_t nb, const double* a, const double* b, double* z,
                       double omega, double small_num, double* beta, double* pivot);

/* robust_update.cpp:22-61 — c (m x n, ld m) updated in place */
int or_robust_update(size_t m, size_t k, size_t n, double* c, double* c_scale, double* c_norm,
                     const double* a, double a_scale, double a_norm, const double* b,
                     double b_scale, double b_norm, double omega, uint64_t* events);

/* scalar_solve.cpp:130-149 */
int or_solve_nonrobust(size_t m, size_t n, const double* a, const unsigned char* ablk,
                       const double* b, const unsigned char* bblk, const double* c, double* y,
                       double* pivot);
int or_solve_robust_scalar(size_t m, size_t n, const double* a, const unsigned char* ablk,
                           const double* b, const unsigned char* bblk, const double* c,
                           double omega, double small_num, double* y, double* alpha,
                           uint64_t* events, double* pivot);

/* tiled_solve.cpp:83-96,183-194 — sequential mode of solve_tiled_robust */
int or_solve_tiled(size_t m, size_t n, const double* a, size_t lda, const unsigned char* ablk,
                   const double* b, size_t ldb, const unsigned char* bblk, const double* c,
                   size_t ldc, size_t tile, double omega, double small_num, double* y,
                   size_t ldy, double* alpha, uint64_t* events, double* pivot,
                   or_probe_fn probe, void* probe_user);

/* tests/support/oracles.cpp:56-73 — mn x mn Kronecker solve, partial pivoting */
int or_kron_solve(size_t m, size_t n, const double* a, const double* b, const double* c,
                  double* y);

/* testgen.cpp:64-79 — the reference residual (overflows to NaN/Inf once |Y| >~ 1e154) */
double or_relative_residual(size_t m, size_t n, const double* a, const double* b,
                            const double* c, const double* y, double alpha);

/* Overflow-safe relative residual with alpha given as an exponent (alpha = a_mant * 2^a_exp):
 * ||A Y + Y B - alpha C||_F / ((||A||_F + ||B||_F)||Y||_F + ||alpha C||_F), every operand
 * pre-scaled by powers of two and Frobenius sums accumulated LAPACK-dlassq style.
 * Cost O(m n (m + n)); for small/medium oracle cases only. */
double or_relative_residual_safe(size_t m, size_t n, const double* a, size_t lda,
                                 const double* b, size_t ldb, const double* c, size_t ldc,
                                 const double* y, size_t ldy, double a_mant, int a_exp);

#ifdef __cplusplus
}
#endif
#endif
