/* TEST INFRASTRUCTURE ONLY — CPU oracle for the rsylv-b200 parity tests (see rsylv_oracle.h).
 *
 * Plain-C restatement of the reference's sequential tiled robust solver. Every function cites
 * the reference file:line (relative to /root/reference/proj) it restates. Exceptions of the
 * reference map to longjmp + status codes. Extended-range guard arithmetic uses x87 long double
 * exactly like the reference (overflow.cpp, small_solve.cpp, robust_update.cpp).
 */
#include "rsylv_oracle.h"

#include <float.h>
#include <math.h>
#include <setjmp.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_INVALID = 1, OR_SINGULAR = 2, OR_UNDERFLOW = 3 };

typedef struct {
    jmp_buf jb;
    double omega, small_num;
    uint64_t events;
    double pivot;
} ctx_t;

static void fail(ctx_t* cx, int code) { longjmp(cx->jb, code); }

#define AT(p, ld, i, j) ((p)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

/* ---------------- L0: dense_matrix.cpp ---------------- */

/* dense_matrix.cpp:8-31 — three summation branches, reproduced exactly */
double or_inf_norm(const double* p, size_t rows, size_t cols, size_t ld) {
    if (rows == 0 || cols == 0) return 0.0;
    if (cols == 1) {
        double best = 0.0;
        for (size_t i = 0; i < rows; ++i) {
            double v = fabs(p[i]);
            if (best < v) best = v;
        }
        return best;
    }
    if (rows <= 4 || cols <= 2) {
        double best = 0.0;
        for (size_t i = 0; i < rows; ++i) {
            double s = 0.0;
            for (size_t j = 0; j < cols; ++j) s += fabs(AT(p, ld, i, j));
            if (best < s) best = s;
        }
        return best;
    }
    double* rs = (double*)calloc(rows, sizeof(double));
    for (size_t j = 0; j < cols; ++j) {
        const double* col = p + j * ld;
        for (size_t i = 0; i < rows; ++i) rs[i] += fabs(col[i]);
    }
    double best = rs[0];
    for (size_t i = 1; i < rows; ++i)
        if (best < rs[i]) best = rs[i];
    free(rs);
    return best;
}

static double frob_norm(const double* p, size_t rows, size_t cols, size_t ld) { /* :33-40 */
    double s = 0.0;
    for (size_t j = 0; j < cols; ++j)
        for (size_t i = 0; i < rows; ++i) s += AT(p, ld, i, j) * AT(p, ld, i, j);
    return sqrt(s);
}

/* dense_matrix.cpp:61-82 — C -= A*B, j-outer, k unrolled by 4, i-inner */
static void gemm_update(double* c, size_t ldc, const double* a, size_t lda, const double* b,
                        size_t ldb, size_t m, size_t n, size_t inner) {
    for (size_t j = 0; j < n; ++j) {
        double* cj = c + j * ldc;
        size_t k = 0;
        for (; k + 4 <= inner; k += 4) {
            const double* a0 = a + k * lda;
            const double* a1 = a0 + lda;
            const double* a2 = a1 + lda;
            const double* a3 = a2 + lda;
            const double b0 = AT(b, ldb, k, j), b1 = AT(b, ldb, k + 1, j),
                         b2 = AT(b, ldb, k + 2, j), b3 = AT(b, ldb, k + 3, j);
            for (size_t i = 0; i < m; ++i)
                cj[i] -= a0[i] * b0 + a1[i] * b1 + a2[i] * b2 + a3[i] * b3;
        }
        for (; k < inner; ++k) {
            const double* ak = a + k * lda;
            const double bk = AT(b, ldb, k, j);
            for (size_t i = 0; i < m; ++i) cj[i] -= ak[i] * bk;
        }
    }
}

static void scale(double* p, size_t rows, size_t cols, size_t ld, double f) { /* :84-89 */
    for (size_t j = 0; j < cols; ++j)
        for (size_t i = 0; i < rows; ++i) AT(p, ld, i, j) *= f;
}

/* ---------------- L1: overflow.cpp ---------------- */

static const double kShave = 1.0 - 0x1p-30; /* overflow.cpp:17 */

static void require_bound(ctx_t* cx, double v) { /* overflow.cpp:19-23 */
    if (!(v >= 0.0) || !(v <= cx->omega)) fail(cx, OR_INVALID);
}

/* overflow.cpp:29-40 */
static double update_scale(ctx_t* cx, long double growth) {
    const long double omega = cx->omega;
    if (growth <= omega) return 1.0;
    const long double target = omega * (long double)kShave;
    double zeta = (double)(target / growth);
    while (zeta > 0.0 && (long double)zeta * growth > target) zeta = nextafter(zeta, 0.0);
    if (zeta <= 0.0) fail(cx, OR_UNDERFLOW);
    cx->events++;
    return zeta;
}

/* overflow.cpp:42-46 */
static double accumulate_scale(ctx_t* cx, double acc, double factor) {
    const double next = acc * factor;
    if (next < DBL_MIN) fail(cx, OR_UNDERFLOW);
    return next;
}

/* overflow.cpp:50-57 */
static double protect_update(ctx_t* cx, double cn, double an, double bn) {
    require_bound(cx, cn);
    require_bound(cx, an);
    require_bound(cx, bn);
    const long double growth = (long double)cn + (long double)an * (long double)bn;
    return update_scale(cx, growth);
}

/* overflow.cpp:59-75 */
static double protect_division(ctx_t* cx, double numer_bound, double divisor) {
    require_bound(cx, numer_bound);
    if (divisor == 0.0) {
        cx->pivot = 0.0;
        fail(cx, OR_SINGULAR);
    }
    const double t = fabs(divisor);
    if (t >= 1.0) return 1.0;
    if (numer_bound <= cx->omega * t) return 1.0;
    double zeta = (cx->omega * t) / numer_bound * kShave;
    while (zeta > 0.0 && ((zeta * numer_bound) / t > cx->omega ||
                          (long double)zeta * numer_bound / t > (long double)cx->omega))
        zeta = nextafter(zeta, 0.0);
    if (zeta <= 0.0) fail(cx, OR_UNDERFLOW);
    cx->events++;
    return zeta;
}

/* ---------------- L2: small_solve.cpp ---------------- */

/* small_solve.cpp:15-108 — Kronecker GE with complete pivoting, guarded or plain */
static double small_core(ctx_t* cx, const double* a, size_t lda, size_t ma, const double* b,
                         size_t ldb, size_t nb, double* c, size_t ldc, int guarded) {
    const size_t nk = ma * nb;
    double k[4][4];
    double rhs[4] = {0, 0, 0, 0};
    size_t colp[4] = {0, 1, 2, 3};
    memset(k, 0, sizeof k);
    for (size_t j = 0; j < nb; ++j)
        for (size_t i = 0; i < ma; ++i) {
            const size_t row = j * ma + i;
            rhs[row] = AT(c, ldc, i, j);
            for (size_t p = 0; p < ma; ++p) k[row][j * ma + p] += AT(a, lda, i, p);
            for (size_t l = 0; l < nb; ++l) k[row][l * ma + i] += AT(b, ldb, l, j);
        }
    double beta = 1.0;
#define RESCALE_RHS(z)                                           \
    do {                                                         \
        for (size_t r_ = 0; r_ < nk; ++r_) rhs[r_] *= (z);       \
        beta = accumulate_scale(cx, beta, (z));                  \
    } while (0)

    for (size_t s = 0; s < nk; ++s) {
        size_t pi = s, pj = s;
        double best = -1.0;
        for (size_t j = s; j < nk; ++j)
            for (size_t i = s; i < nk; ++i) {
                const double v = fabs(k[i][j]);
                if (v > best) {
                    best = v;
                    pi = i;
                    pj = j;
                }
            }
        if (!(best >= cx->small_num)) {
            cx->pivot = k[pi][pj];
            fail(cx, OR_SINGULAR);
        }
        if (pi != s) {
            for (size_t j = 0; j < nk; ++j) {
                double t = k[s][j];
                k[s][j] = k[pi][j];
                k[pi][j] = t;
            }
            double t = rhs[s];
            rhs[s] = rhs[pi];
            rhs[pi] = t;
        }
        if (pj != s) {
            for (size_t i = 0; i < nk; ++i) {
                double t = k[i][s];
                k[i][s] = k[i][pj];
                k[i][pj] = t;
            }
            size_t t = colp[s];
            colp[s] = colp[pj];
            colp[pj] = t;
        }
        for (size_t i = s + 1; i < nk; ++i) {
            const double mult = k[i][s] / k[s][s];
            k[i][s] = 0.0;
            for (size_t j = s + 1; j < nk; ++j) k[i][j] -= mult * k[s][j];
            if (guarded) {
                const long double growth =
                    (long double)fabs(rhs[i]) + (long double)fabs(mult) * fabs(rhs[s]);
                const double zeta = update_scale(cx, growth);
                if (zeta != 1.0) RESCALE_RHS(zeta);
            }
            rhs[i] -= mult * rhs[s];
        }
    }
    for (size_t s = nk; s-- > 0;) {
        for (size_t j = s + 1; j < nk; ++j) {
            if (guarded) {
                const long double growth =
                    (long double)fabs(rhs[s]) + (long double)fabs(k[s][j]) * fabs(rhs[j]);
                const double zeta = update_scale(cx, growth);
                if (zeta != 1.0) RESCALE_RHS(zeta);
            }
            rhs[s] -= k[s][j] * rhs[j];
        }
        if (guarded) {
            const double zeta = protect_division(cx, fabs(rhs[s]), k[s][s]);
            if (zeta != 1.0) RESCALE_RHS(zeta);
        }
        rhs[s] /= k[s][s];
    }
#undef RESCALE_RHS
    double z[4];
    for (size_t s = 0; s < nk; ++s) z[colp[s]] = rhs[s];
    for (size_t j = 0; j < nb; ++j)
        for (size_t i = 0; i < ma; ++i) AT(c, ldc, i, j) = z[j * ma + i];
    if (guarded && nb == 2) {
        const double norm = or_inf_norm(c, ma, nb, ldc);
        if (norm > cx->omega) {
            const double zeta = update_scale(cx, (long double)norm);
            scale(c, ma, nb, ldc, zeta);
            beta = accumulate_scale(cx, beta, zeta);
        }
    }
    return beta;
}

/* small_solve.cpp:126-141 */
int or_small_sylvester(size_t ma, size_t nb, const double* a, const double* b, double* z,
                       double omega, double small_num, double* beta, double* pivot) {
    ctx_t cx;
    cx.omega = omega > 0 ? omega : DBL_MAX / 2;
    cx.small_num = small_num > 0 ? small_num : DBL_MIN / DBL_EPSILON;
    cx.events = 0;
    cx.pivot = 0;
    int code = setjmp(cx.jb);
    if (code) {
        if (pivot) *pivot = cx.pivot;
        return code;
    }
    if (ma < 1 || ma > 2 || nb < 1 || nb > 2) return OR_INVALID;
    if (!(or_inf_norm(a, ma, ma, ma) <= cx.omega) || !(or_inf_norm(b, nb, nb, nb) <= cx.omega) ||
        !(or_inf_norm(z, ma, nb, ma) <= cx.omega))
        return OR_INVALID;
    *beta = small_core(&cx, a, ma, ma, b, nb, nb, z, ma, 1);
    return OR_OK;
}

/* ---------------- L2: robust_update.cpp ---------------- */

static void require_scale(ctx_t* cx, double s) { /* robust_update.cpp:10-13 */
    if (!(s >= DBL_MIN) || !(s <= 1.0)) fail(cx, OR_INVALID);
}

/* robust_update.cpp:22-61. `tmp` is caller scratch of >= max(m*k, k*n) doubles. */
static void robust_update(ctx_t* cx, double* c, size_t ldc, double* cscale, double* cnorm,
                          const double* a, size_t lda, double ascale, double anorm,
                          const double* b, size_t ldb, double bscale, double bnorm, size_t m,
                          size_t k, size_t n, double* tmp) {
    require_scale(cx, *cscale);
    require_scale(cx, ascale);
    require_scale(cx, bscale);
    require_bound(cx, *cnorm);
    require_bound(cx, anorm);
    require_bound(cx, bnorm);
    double eta = *cscale;
    if (ascale < eta) eta = ascale;
    if (bscale < eta) eta = bscale;
    const long double growth = (long double)(eta / *cscale) * *cnorm +
                               (long double)eta / ascale / bscale *
                                   ((long double)anorm * (long double)bnorm);
    const double zeta = update_scale(cx, growth);
    const double delta = accumulate_scale(cx, eta, zeta);
    const double cf = delta / *cscale;
    if (cf != 1.0) scale(c, m, n, ldc, cf);
    const double pf = (delta / ascale) / bscale;
    if (pf == 1.0) {
        gemm_update(c, ldc, a, lda, b, ldb, m, n, k);
    } else if (anorm <= bnorm) {
        for (size_t j = 0; j < k; ++j)
            for (size_t i = 0; i < m; ++i) tmp[i + j * m] = AT(a, lda, i, j) * pf;
        gemm_update(c, ldc, tmp, m, b, ldb, m, n, k);
    } else {
        for (size_t j = 0; j < n; ++j)
            for (size_t i = 0; i < k; ++i) tmp[i + j * k] = AT(b, ldb, i, j) * pf;
        gemm_update(c, ldc, a, lda, tmp, k, m, n, k);
    }
    *cscale = delta;
    *cnorm = or_inf_norm(c, m, n, ldc);
}

int or_robust_update(size_t m, size_t k, size_t n, double* c, double* c_scale, double* c_norm,
                     const double* a, double a_scale, double a_norm, const double* b,
                     double b_scale, double b_norm, double omega, uint64_t* events) {
    ctx_t cx;
    cx.omega = omega > 0 ? omega : DBL_MAX / 2;
    cx.small_num = DBL_MIN / DBL_EPSILON;
    cx.events = 0;
    double* tmp = (double*)malloc(sizeof(double) * (m * k + k * n + 1));
    int code = setjmp(cx.jb);
    if (code == 0)
        robust_update(&cx, c, m, c_scale, c_norm, a, m, a_scale, a_norm, b, k, b_scale, b_norm,
                      m, k, n, tmp);
    free(tmp);
    if (events) *events = cx.events;
    return code;
}

/* ---------------- L2: scalar_solve.cpp ---------------- */

typedef struct {
    size_t start, size;
} blk_t;

static size_t blocks_of(const unsigned char* blk, size_t n, blk_t* out) {
    size_t nb = 0;
    for (size_t i = 0; i < n;) {
        size_t s = (blk && blk[i] == 2 && i + 1 < n) ? 2 : 1;
        out[nb].start = i;
        out[nb].size = s;
        ++nb;
        i += s;
    }
    return nb;
}

/* scalar_solve.cpp:13-36 */
static void nonrobust_inplace(ctx_t* cx, const double* a, size_t lda, const blk_t* ab, size_t p,
                              const double* b, size_t ldb, const blk_t* bb, size_t q, double* y,
                              size_t ldy, size_t n) {
    for (size_t lb = 0; lb < q; ++lb) {
        const blk_t bl = bb[lb];
        for (size_t kb = p; kb-- > 0;) {
            const blk_t ak = ab[kb];
            double* ykl = &AT(y, ldy, ak.start, bl.start);
            small_core(cx, &AT(a, lda, ak.start, ak.start), lda, ak.size,
                       &AT(b, ldb, bl.start, bl.start), ldb, bl.size, ykl, ldy, 0);
            if (ak.start > 0)
                gemm_update(&AT(y, ldy, 0, bl.start), ldy, &AT(a, lda, 0, ak.start), lda, ykl,
                            ldy, ak.start, bl.size, ak.size);
            const size_t tail = bl.start + bl.size;
            if (tail < n)
                gemm_update(&AT(y, ldy, ak.start, tail), ldy, ykl, ldy,
                            &AT(b, ldb, bl.start, tail), ldb, ak.size, n - tail, bl.size);
        }
    }
}

/* scalar_solve.cpp:41-51 */
static void scale_except(double* y, size_t ldy, size_t rows, size_t cols, double f, blk_t rowb,
                         blk_t colb) {
    for (size_t j = 0; j < cols; ++j) {
        double* col = y + j * ldy;
        if (j >= colb.start && j < colb.start + colb.size) {
            for (size_t i = 0; i < rowb.start; ++i) col[i] *= f;
            for (size_t i = rowb.start + rowb.size; i < rows; ++i) col[i] *= f;
        } else {
            for (size_t i = 0; i < rows; ++i) col[i] *= f;
        }
    }
}

/* scalar_solve.cpp:53-63 */
static void require_blocks_bounded(ctx_t* cx, const double* m, size_t ld, const blk_t* rows,
                                   size_t nr, const blk_t* cols, size_t nc, int upper_only) {
    for (size_t ib = 0; ib < nr; ++ib)
        for (size_t jb = upper_only ? ib : 0; jb < nc; ++jb) {
            const blk_t r = rows[ib], c = cols[jb];
            if (!(or_inf_norm(&AT(m, ld, r.start, c.start), r.size, c.size, ld) <= cx->omega))
                fail(cx, OR_INVALID);
        }
}

/* scalar_solve.cpp:67-126 — RobustSyl (Alg. 2) with one running alpha */
static double robust_scalar_inplace(ctx_t* cx, const double* a, size_t lda, const blk_t* ab,
                                    size_t p, const double* b, size_t ldb, const blk_t* bb,
                                    size_t q, double* y, size_t ldy, size_t rows, size_t n) {
    require_blocks_bounded(cx, a, lda, ab, p, ab, p, 1);
    require_blocks_bounded(cx, b, ldb, bb, q, bb, q, 1);
    require_blocks_bounded(cx, y, ldy, ab, p, bb, q, 0);
    double alpha = 1.0;
    for (size_t lb = 0; lb < q; ++lb) {
        const blk_t bl = bb[lb];
        for (size_t kb = p; kb-- > 0;) {
            const blk_t ak = ab[kb];
            double* ykl = &AT(y, ldy, ak.start, bl.start);
            const double beta = small_core(cx, &AT(a, lda, ak.start, ak.start), lda, ak.size,
                                           &AT(b, ldb, bl.start, bl.start), ldb, bl.size, ykl,
                                           ldy, 1);
            if (beta != 1.0) {
                alpha = accumulate_scale(cx, alpha, beta);
                scale_except(y, ldy, rows, n, beta, ak, bl);
            }
            if (ak.start > 0) {
                double* ycol = &AT(y, ldy, 0, bl.start);
                const double* acol = &AT(a, lda, 0, ak.start);
                const double g1 = protect_update(cx, or_inf_norm(ycol, ak.start, bl.size, ldy),
                                                 or_inf_norm(acol, ak.start, ak.size, lda),
                                                 or_inf_norm(ykl, ak.size, bl.size, ldy));
                if (g1 != 1.0) {
                    alpha = accumulate_scale(cx, alpha, g1);
                    scale(y, rows, n, ldy, g1);
                }
                gemm_update(ycol, ldy, acol, lda, ykl, ldy, ak.start, bl.size, ak.size);
            }
            const size_t tail = bl.start + bl.size;
            if (tail < n) {
                double cmax = 0.0, bmax = 0.0;
                for (size_t jb = lb + 1; jb < q; ++jb) {
                    const blk_t bj = bb[jb];
                    double v1 = or_inf_norm(&AT(y, ldy, ak.start, bj.start), ak.size, bj.size, ldy);
                    double v2 = or_inf_norm(&AT(b, ldb, bl.start, bj.start), bl.size, bj.size, ldb);
                    if (cmax < v1) cmax = v1;
                    if (bmax < v2) bmax = v2;
                }
                const double g2 =
                    protect_update(cx, cmax, or_inf_norm(ykl, ak.size, bl.size, ldy), bmax);
                if (g2 != 1.0) {
                    alpha = accumulate_scale(cx, alpha, g2);
                    scale(y, rows, n, ldy, g2);
                }
                gemm_update(&AT(y, ldy, ak.start, tail), ldy, ykl, ldy,
                            &AT(b, ldb, bl.start, tail), ldb, ak.size, n - tail, bl.size);
            }
        }
    }
    return alpha;
}

static void init_ctx(ctx_t* cx, double omega, double small_num) {
    cx->omega = omega > 0 ? omega : DBL_MAX / 2;
    cx->small_num = small_num > 0 ? small_num : DBL_MIN / DBL_EPSILON;
    cx->events = 0;
    cx->pivot = 0.0;
}

/* scalar_solve.cpp:130-138 */
int or_solve_nonrobust(size_t m, size_t n, const double* a, const unsigned char* ablk,
                       const double* b, const unsigned char* bblk, const double* c, double* y,
                       double* pivot) {
    ctx_t cx;
    init_ctx(&cx, 0, 0);
    blk_t* ab = (blk_t*)malloc(sizeof(blk_t) * (m + 1));
    blk_t* bb = (blk_t*)malloc(sizeof(blk_t) * (n + 1));
    size_t p = blocks_of(ablk, m, ab), q = blocks_of(bblk, n, bb);
    memcpy(y, c, sizeof(double) * m * n);
    int code = setjmp(cx.jb);
    if (code == 0) nonrobust_inplace(&cx, a, m, ab, p, b, n, bb, q, y, m, n);
    if (code && pivot) *pivot = cx.pivot;
    free(ab);
    free(bb);
    return code;
}

/* scalar_solve.cpp:140-149 */
int or_solve_robust_scalar(size_t m, size_t n, const double* a, const unsigned char* ablk,
                           const double* b, const unsigned char* bblk, const double* c,
                           double omega, double small_num, double* y, double* alpha,
                           uint64_t* events, double* pivot) {
    ctx_t cx;
    init_ctx(&cx, omega, small_num);
    blk_t* ab = (blk_t*)malloc(sizeof(blk_t) * (m + 1));
    blk_t* bb = (blk_t*)malloc(sizeof(blk_t) * (n + 1));
    size_t p = blocks_of(ablk, m, ab), q = blocks_of(bblk, n, bb);
    memcpy(y, c, sizeof(double) * m * n);
    int code = setjmp(cx.jb);
    if (code == 0) *alpha = robust_scalar_inplace(&cx, a, m, ab, p, b, n, bb, q, y, m, m, n);
    if (code && pivot) *pivot = cx.pivot;
    if (events) *events = cx.events;
    free(ab);
    free(bb);
    return code;
}

/* ---------------- L3/L4: partition.cpp, tile_grid.cpp, tiled_solve.cpp ---------------- */

/* partition.cpp:74-91 — cut at pos+ts; a cut that splits a 2x2 block moves one index later */
static size_t partition(const unsigned char* blk, size_t n, size_t ts, size_t* cuts) {
    size_t nc = 0, pos = 0;
    cuts[nc++] = 0;
    while (pos < n) {
        size_t next = pos + ts;
        if (next >= n)
            next = n;
        else if (blk && blk[next - 1] == 2)
            ++next;
        cuts[nc++] = next;
        pos = next;
    }
    return nc - 1;
}

/* tiled_solve.cpp:33-96 + tile_grid.cpp:8-83 (sequential mode) */
int or_solve_tiled(size_t m, size_t n, const double* a, size_t lda, const unsigned char* ablk,
                   const double* b, size_t ldb, const unsigned char* bblk, const double* c,
                   size_t ldc, size_t tile, double omega, double small_num, double* y,
                   size_t ldy, double* alpha_out, uint64_t* events, double* pivot,
                   or_probe_fn probe, void* probe_user) {
    ctx_t cx;
    init_ctx(&cx, omega, small_num);
    if (tile < 2) return OR_INVALID; /* partition.cpp:75-76 */
    size_t* rc = (size_t*)malloc(sizeof(size_t) * (m + 2));
    size_t* cc = (size_t*)malloc(sizeof(size_t) * (n + 2));
    const size_t M = partition(ablk, m, tile, rc), N = partition(bblk, n, tile, cc);
    blk_t* ab = (blk_t*)malloc(sizeof(blk_t) * (m + 1));
    blk_t* bb = (blk_t*)malloc(sizeof(blk_t) * (n + 1));
    size_t* abs_ = (size_t*)malloc(sizeof(size_t) * (M + 1)); /* block index of each row tile */
    size_t* bbs = (size_t*)malloc(sizeof(size_t) * (N + 1));
    const size_t P = blocks_of(ablk, m, ab), Q = blocks_of(bblk, n, bb);
    {
        size_t t = 0;
        for (size_t i = 0; i < P && t <= M; ++i)
            if (ab[i].start == rc[t]) abs_[t++] = i;
        abs_[M] = P;
        t = 0;
        for (size_t i = 0; i < Q && t <= N; ++i)
            if (bb[i].start == cc[t]) bbs[t++] = i;
        bbs[N] = Q;
    }
    double* scl = (double*)malloc(sizeof(double) * M * N + 8);
    double* nrm = (double*)malloc(sizeof(double) * M * N + 8);
    double* abnd = (double*)malloc(sizeof(double) * M * M + 8);
    double* bbnd = (double*)malloc(sizeof(double) * N * N + 8);
    size_t tmax = 0;
    for (size_t t = 0; t < M; ++t)
        if (rc[t + 1] - rc[t] > tmax) tmax = rc[t + 1] - rc[t];
    for (size_t t = 0; t < N; ++t)
        if (cc[t + 1] - cc[t] > tmax) tmax = cc[t + 1] - cc[t];
    double* tmp = (double*)malloc(sizeof(double) * tmax * tmax + 8);
    blk_t* lab = (blk_t*)malloc(sizeof(blk_t) * (tmax + 1));
    blk_t* lbb = (blk_t*)malloc(sizeof(blk_t) * (tmax + 1));

    for (size_t j = 0; j < n; ++j) memcpy(y + j * ldy, c + j * ldc, sizeof(double) * m);
#define TILE(k, l) (&AT(y, ldy, rc[k], cc[l]))
#define TR(k) (rc[(k) + 1] - rc[k])
#define TC(l) (cc[(l) + 1] - cc[l])
    for (size_t k = 0; k < M; ++k)
        for (size_t l = 0; l < N; ++l) {
            scl[k * N + l] = 1.0;
            nrm[k * N + l] = or_inf_norm(TILE(k, l), TR(k), TC(l), ldy);
        }
    int code = setjmp(cx.jb);
    if (code == 0) {
        /* compute_bounds (tile_grid.cpp:54-75) */
        for (size_t i = 0; i < M; ++i)
            for (size_t k = i; k < M; ++k) {
                const double v = or_inf_norm(&AT(a, lda, rc[i], rc[k]), TR(i), TR(k), lda);
                if (!(v <= cx.omega)) fail(&cx, OR_INVALID);
                abnd[i * M + k] = v;
            }
        for (size_t l = 0; l < N; ++l)
            for (size_t j = l; j < N; ++j) {
                const double v = or_inf_norm(&AT(b, ldb, cc[l], cc[j]), TC(l), TC(j), ldb);
                if (!(v <= cx.omega)) fail(&cx, OR_INVALID);
                bbnd[l * N + j] = v;
            }
        /* require_rhs_bounded (tiled_solve.cpp:74-80) */
        for (size_t k = 0; k < M * N; ++k)
            if (!(nrm[k] <= cx.omega)) fail(&cx, OR_INVALID);
        /* run_sequential loop nest (tiled_solve.cpp:87-93) */
        for (size_t k = M; k-- > 0;) {
            for (size_t l = 0; l < N; ++l) {
                /* solve_tile (tiled_solve.cpp:33-50) */
                double* ykl = TILE(k, l);
                size_t p = abs_[k + 1] - abs_[k], q = bbs[l + 1] - bbs[l];
                for (size_t i = 0; i < p; ++i) {
                    lab[i] = ab[abs_[k] + i];
                    lab[i].start -= rc[k];
                }
                for (size_t i = 0; i < q; ++i) {
                    lbb[i] = bb[bbs[l] + i];
                    lbb[i].start -= cc[l];
                }
                double beta = robust_scalar_inplace(&cx, &AT(a, lda, rc[k], rc[k]), lda, lab, p,
                                                    &AT(b, ldb, cc[l], cc[l]), ldb, lbb, q, ykl,
                                                    ldy, TR(k), TC(l));
                double norm = or_inf_norm(ykl, TR(k), TC(l), ldy);
                if (norm > cx.omega) {
                    const double zeta = update_scale(&cx, (long double)norm);
                    scale(ykl, TR(k), TC(l), ldy, zeta);
                    beta = accumulate_scale(&cx, beta, zeta);
                    norm = or_inf_norm(ykl, TR(k), TC(l), ldy);
                }
                scl[k * N + l] = accumulate_scale(&cx, scl[k * N + l], beta);
                nrm[k * N + l] = norm;
                if (probe) probe(k, l, scl[k * N + l], norm, probe_user);
                /* column_update (tiled_solve.cpp:53-61) */
                for (size_t i = k; i-- > 0;) {
                    robust_update(&cx, TILE(i, l), ldy, &scl[i * N + l], &nrm[i * N + l],
                                  &AT(a, lda, rc[i], rc[k]), lda, 1.0, abnd[i * M + k], ykl, ldy,
                                  scl[k * N + l], nrm[k * N + l], TR(i), TR(k), TC(l), tmp);
                    if (probe) probe(i, l, scl[i * N + l], nrm[i * N + l], probe_user);
                }
                /* row_update (tiled_solve.cpp:64-72) */
                for (size_t j = l + 1; j < N; ++j) {
                    robust_update(&cx, TILE(k, j), ldy, &scl[k * N + j], &nrm[k * N + j], ykl,
                                  ldy, scl[k * N + l], nrm[k * N + l], &AT(b, ldb, cc[l], cc[j]),
                                  ldb, 1.0, bbnd[l * N + j], TR(k), TC(l), TC(j), tmp);
                    if (probe) probe(k, j, scl[k * N + j], nrm[k * N + j], probe_user);
                }
            }
        }
        /* reduce_and_scale (tile_grid.cpp:38-52,77-83) */
        double alpha = 1.0;
        for (size_t t = 0; t < M * N; ++t)
            if (scl[t] < alpha) alpha = scl[t];
        for (size_t k = 0; k < M; ++k)
            for (size_t l = 0; l < N; ++l) {
                const double f = alpha / scl[k * N + l];
                if (f != 1.0) scale(TILE(k, l), TR(k), TC(l), ldy, f);
            }
        *alpha_out = alpha;
    }
#undef TILE
#undef TR
#undef TC
    if (code && pivot) *pivot = cx.pivot;
    if (events) *events = cx.events;
    free(rc); free(cc); free(ab); free(bb); free(abs_); free(bbs);
    free(scl); free(nrm); free(abnd); free(bbnd); free(tmp); free(lab); free(lbb);
    return code;
}

/* ---------------- oracles (tests/support/oracles.cpp, testgen.cpp) ---------------- */

/* tests/support/oracles.cpp:56-73 + :34-54 (row-major nested elimination, partial pivoting) */
int or_kron_solve(size_t m, size_t n, const double* a, const double* b, const double* c,
                  double* y) {
    const size_t nk = m * n;
    double* k = (double*)calloc(nk * nk, sizeof(double));
    double* rhs = (double*)malloc(sizeof(double) * nk);
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < m; ++i) {
            const size_t row = j * m + i;
            rhs[row] = AT(c, m, i, j);
            for (size_t p = 0; p < m; ++p) k[row * nk + j * m + p] += AT(a, m, i, p);
            for (size_t l = 0; l < n; ++l) k[row * nk + l * m + i] += AT(b, n, l, j);
        }
    int st = 0;
    for (size_t s = 0; s < nk && !st; ++s) {
        size_t piv = s;
        for (size_t i = s + 1; i < nk; ++i)
            if (fabs(k[i * nk + s]) > fabs(k[piv * nk + s])) piv = i;
        if (k[piv * nk + s] == 0.0) {
            st = OR_SINGULAR;
            break;
        }
        if (piv != s) {
            for (size_t j = 0; j < nk; ++j) {
                double t = k[s * nk + j];
                k[s * nk + j] = k[piv * nk + j];
                k[piv * nk + j] = t;
            }
            double t = rhs[s];
            rhs[s] = rhs[piv];
            rhs[piv] = t;
        }
        for (size_t i = s + 1; i < nk; ++i) {
            const double f = k[i * nk + s] / k[s * nk + s];
            for (size_t j = s; j < nk; ++j) k[i * nk + j] -= f * k[s * nk + j];
            rhs[i] -= f * rhs[s];
        }
    }
    if (!st) {
        for (size_t s = nk; s-- > 0;) {
            for (size_t j = s + 1; j < nk; ++j) rhs[s] -= k[s * nk + j] * rhs[j];
            rhs[s] /= k[s * nk + s];
        }
        for (size_t j = 0; j < n; ++j)
            for (size_t i = 0; i < m; ++i) AT(y, m, i, j) = rhs[j * m + i];
    }
    free(k);
    free(rhs);
    return st;
}

/* testgen.cpp:64-79 */
double or_relative_residual(size_t m, size_t n, const double* a, const double* b,
                            const double* c, const double* y, double alpha) {
    double* r = (double*)malloc(sizeof(double) * m * n);
    for (size_t t = 0; t < m * n; ++t) r[t] = c[t] * alpha;
    const double ac = frob_norm(r, m, n, m);
    gemm_update(r, m, a, m, y, m, m, n, m);
    gemm_update(r, m, y, m, b, n, m, n, n);
    const double den = (frob_norm(a, m, m, m) + frob_norm(b, n, n, n)) * frob_norm(y, m, n, m) + ac;
    const double res = frob_norm(r, m, n, m) / den;
    free(r);
    return res;
}

/* ---- overflow-safe residual (new; replaces testgen.cpp:64-79 for scaled solutions) ---- */

typedef struct {
    double scale, sumsq; /* value = scale * sqrt(sumsq), dlassq convention */
} ssq_t;

static void ssq_add(ssq_t* s, double v) {
    v = fabs(v);
    if (v == 0.0 || v != v) {
        if (v != v) s->sumsq = NAN;
        return;
    }
    if (s->scale < v) {
        s->sumsq = 1.0 + s->sumsq * (s->scale / v) * (s->scale / v);
        s->scale = v;
    } else {
        s->sumsq += (v / s->scale) * (v / s->scale);
    }
}

/* log2 of a Frobenius norm held as scale*sqrt(sumsq)*2^e */
static double ssq_log2(const ssq_t* s, int e) {
    if (s->scale == 0.0) return -INFINITY;
    return log2(s->scale) + 0.5 * log2(s->sumsq) + e;
}

static double log2_add(double x, double y) { /* log2(2^x + 2^y) */
    if (x == -INFINITY) return y;
    if (y == -INFINITY) return x;
    double hi = x > y ? x : y, lo = x > y ? y : x;
    return hi + log2(1.0 + exp2(lo - hi));
}

double or_relative_residual_safe(size_t m, size_t n, const double* a, size_t lda,
                                 const double* b, size_t ldb, const double* c, size_t ldc,
                                 const double* y, size_t ldy, double a_mant, int a_exp) {
    /* pre-scale Y and C by powers of two so max|.| ~ 1; alpha*C = (a_mant*C*2^-ec) * 2^(a_exp+ec) */
    double ymax = 0.0, cmax = 0.0;
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < m; ++i) {
            if (fabs(AT(y, ldy, i, j)) > ymax) ymax = fabs(AT(y, ldy, i, j));
            if (fabs(AT(c, ldc, i, j)) > cmax) cmax = fabs(AT(c, ldc, i, j));
        }
    int ey = 0, ec = 0;
    if (ymax > 0) frexp(ymax, &ey);
    if (cmax > 0) frexp(cmax, &ec);
    /* residual R = A*Ys + Ys*B - alpha*C*2^-ey where Ys = Y*2^-ey; true R = R * 2^ey */
    const int d = a_exp + ec - ey; /* alpha*C*2^-ey = a_mant*(C*2^-ec)*2^d */
    double* ys = (double*)malloc(sizeof(double) * m * n);
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < m; ++i) ys[i + j * m] = ldexp(AT(y, ldy, i, j), -ey);
    ssq_t r = {0.0, 1.0}, fa = {0.0, 1.0}, fb = {0.0, 1.0}, fy = {0.0, 1.0}, fc = {0.0, 1.0};
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < m; ++i) {
            long double acc = 0.0L;
            for (size_t p = i; p < m; ++p) acc += (long double)AT(a, lda, i, p) * ys[p + j * m];
            if (i > 0) acc += (long double)AT(a, lda, i, i - 1) * ys[i - 1 + j * m];
            for (size_t q = 0; q <= j + 1 && q < n; ++q)
                acc += (long double)ys[i + q * m] * AT(b, ldb, q, j);
            const long double cs = (long double)a_mant * ldexp(AT(c, ldc, i, j), -ec);
            acc -= ldexpl(cs, d);
            ssq_add(&r, (double)acc);
            ssq_add(&fy, ys[i + j * m]);
            ssq_add(&fc, a_mant * ldexp(AT(c, ldc, i, j), -ec));
        }
    for (size_t j = 0; j < m; ++j)
        for (size_t i = 0; i < m; ++i) ssq_add(&fa, AT(a, lda, i, j));
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < n; ++i) ssq_add(&fb, AT(b, ldb, i, j));
    free(ys);
    /* everything in log2, relative to the common factor 2^ey */
    const double lr = ssq_log2(&r, 0);
    const double lden = log2_add(ssq_log2(&fy, 0) + log2_add(ssq_log2(&fa, 0), ssq_log2(&fb, 0)),
                                 ssq_log2(&fc, d));
    if (lr == -INFINITY) return 0.0;
    return exp2(lr - lden);
}

/* public guard entry points (overflow.hpp:39,46) */
int or_protect_update(double cnorm, double anorm, double bnorm, double omega, double* zeta) {
    ctx_t cx;
    init_ctx(&cx, omega, 0);
    int code = setjmp(cx.jb);
    if (code == 0) *zeta = protect_update(&cx, cnorm, anorm, bnorm);
    return code;
}

int or_protect_division(double numer_bound, double divisor, double omega, double* zeta,
                        double* pivot) {
    ctx_t cx;
    init_ctx(&cx, omega, 0);
    int code = setjmp(cx.jb);
    if (code == 0) *zeta = protect_division(&cx, numer_bound, divisor);
    if (code && pivot) *pivot = cx.pivot;
    return code;
}
