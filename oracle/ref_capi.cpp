// TEST INFRASTRUCTURE ONLY (oracle). A thin extern "C" wrapper around the UNMODIFIED
// reference library (rsylv, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/). It lets the Python tests and bench.py's reference arm call the reference's
// own public API through ctypes. Nothing in the product path links or loads this file.
//
// Block structure convention shared with the product C-ABI (include/rsylv_b200.h):
//   blk[i] = 1  -> a 1x1 diagonal block starts at i
//   blk[i] = 2  -> a 2x2 diagonal block starts at i (rows/cols i, i+1)
//   blk[i] = 0  -> i is the second index of a 2x2 block
// Status codes: 0 ok, 1 invalid_argument, 2 SingularEquationError, 3 ScaleUnderflowError,
// 4 other exception.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "rsylv/errors.hpp"
#include "rsylv/matrix_io.hpp"
#include "rsylv/overflow.hpp"
#include "rsylv/robust_update.hpp"
#include "rsylv/scalar_solve.hpp"
#include "rsylv/small_solve.hpp"
#include "rsylv/testgen.hpp"
#include "rsylv/tiled_solve.hpp"
#include "rsylv/verify.hpp"

using namespace rsylv;

namespace {

DenseMatrix to_dense(const double* p, std::size_t rows, std::size_t cols, std::size_t ld) {
    DenseMatrix m(rows, cols);
    for (std::size_t j = 0; j < cols; ++j)
        std::memcpy(m.data() + j * rows, p + j * ld, rows * sizeof(double));
    return m;
}

QuasiTriangular to_qt(const double* p, std::size_t n, std::size_t ld, const unsigned char* blk) {
    DenseMatrix m = to_dense(p, n, n, ld);
    if (!blk) return QuasiTriangular(std::move(m));
    std::vector<DiagBlock> blocks;
    for (std::size_t i = 0; i < n; ++i)
        if (blk[i] == 1 || blk[i] == 2) blocks.push_back({i, blk[i]});
    return QuasiTriangular(std::move(m), std::move(blocks));
}

void from_dense(const DenseMatrix& m, double* out, std::size_t ld) {
    for (std::size_t j = 0; j < m.cols(); ++j)
        std::memcpy(out + j * ld, m.data() + j * m.rows(), m.rows() * sizeof(double));
}

template <class F>
int guarded(F&& f, double* pivot) {
    try {
        f();
        return 0;
    } catch (const SingularEquationError& e) {
        if (pivot) *pivot = e.pivot();
        return 2;
    } catch (const ScaleUnderflowError&) {
        return 3;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 4;
    }
}

OverflowConfig make_cfg(double omega, double small_num, std::atomic<std::uint64_t>* ev) {
    OverflowConfig cfg;
    if (omega > 0) cfg.omega = omega;
    if (small_num > 0) cfg.small_num = small_num;
    cfg.scaling_events = ev;
    return cfg;
}

} // namespace

extern "C" {

// rsylv::solve_tiled_robust (tiled_solve.hpp:36-40). workers = 0 -> sequential.
int ref_solve_tiled(std::size_t m, std::size_t n, const double* a, std::size_t lda,
                    const unsigned char* ablk, const double* b, std::size_t ldb,
                    const unsigned char* bblk, const double* c, std::size_t ldc,
                    std::size_t tile, double omega, double small_num, std::size_t workers,
                    double* y, std::size_t ldy, double* alpha, std::uint64_t* events,
                    double* pivot) {
    std::atomic<std::uint64_t> ev{0};
    int st = guarded([&] {
        QuasiTriangular qa = to_qt(a, m, lda, ablk), qb = to_qt(b, n, ldb, bblk);
        OverflowConfig cfg = make_cfg(omega, small_num, &ev);
        SolveResult r = solve_tiled_robust(qa, qb, ConstMatrixView{c, m, n, ldc}, tile, cfg,
                                           ExecutionMode{workers});
        from_dense(r.y, y, ldy);
        *alpha = r.alpha;
    }, pivot);
    if (events) *events = ev.load();
    return st;
}

// rsylv::solve_robust_scalar (scalar_solve.hpp:31-32)
int ref_solve_robust_scalar(std::size_t m, std::size_t n, const double* a, const unsigned char* ablk,
                            const double* b, const unsigned char* bblk, const double* c,
                            double omega, double small_num, double* y, double* alpha,
                            std::uint64_t* events, double* pivot) {
    std::atomic<std::uint64_t> ev{0};
    int st = guarded([&] {
        QuasiTriangular qa = to_qt(a, m, m, ablk), qb = to_qt(b, n, n, bblk);
        SolveResult r = solve_robust_scalar(qa, qb, ConstMatrixView{c, m, n, m},
                                            make_cfg(omega, small_num, &ev));
        from_dense(r.y, y, m);
        *alpha = r.alpha;
    }, pivot);
    if (events) *events = ev.load();
    return st;
}

// rsylv::solve_nonrobust (scalar_solve.hpp:24-25)
int ref_solve_nonrobust(std::size_t m, std::size_t n, const double* a, const unsigned char* ablk,
                        const double* b, const unsigned char* bblk, const double* c, double* y,
                        double* pivot) {
    return guarded([&] {
        QuasiTriangular qa = to_qt(a, m, m, ablk), qb = to_qt(b, n, n, bblk);
        DenseMatrix r = solve_nonrobust(qa, qb, ConstMatrixView{c, m, n, m});
        from_dense(r, y, m);
    }, pivot);
}

// rsylv::robust_update (robust_update.hpp:32-33); c updated in place (ld = m).
int ref_robust_update(std::size_t m, std::size_t k, std::size_t n, double* c, double* c_scale,
                      double* c_norm, const double* a, double a_scale, double a_norm,
                      const double* b, double b_scale, double b_norm, double omega,
                      std::uint64_t* events) {
    std::atomic<std::uint64_t> ev{0};
    int st = guarded([&] {
        Augmented dst{*c_scale, MatrixView{c, m, n, m}, *c_norm};
        robust_update(dst, ConstAugmented{a_scale, ConstMatrixView{a, m, k, m}, a_norm},
                      ConstAugmented{b_scale, ConstMatrixView{b, k, n, k}, b_norm},
                      make_cfg(omega, 0, &ev));
        *c_scale = dst.scale;
        *c_norm = dst.norm;
    }, nullptr);
    if (events) *events = ev.load();
    return st;
}

// rsylv::solve_small_sylvester (small_solve.hpp:21-22)
int ref_small_sylvester(std::size_t ma, std::size_t nb, const double* a, const double* b,
                        const double* c, double omega, double small_num, double* z, double* beta,
                        double* pivot) {
    return guarded([&] {
        ScaledSolve s = solve_small_sylvester(ConstMatrixView{a, ma, ma, ma},
                                              ConstMatrixView{b, nb, nb, nb},
                                              ConstMatrixView{c, ma, nb, ma},
                                              make_cfg(omega, small_num, nullptr));
        from_dense(s.z, z, ma);
        *beta = s.beta;
    }, pivot);
}

// rsylv::protect_update / protect_division (overflow.hpp:39,46)
int ref_protect_update(double cn, double an, double bn, double omega, double* zeta) {
    return guarded([&] { *zeta = protect_update(cn, an, bn, make_cfg(omega, 0, nullptr)); }, nullptr);
}
int ref_protect_division(double nb, double d, double omega, double* zeta, double* pivot) {
    return guarded([&] { *zeta = protect_division(nb, d, make_cfg(omega, 0, nullptr)); }, pivot);
}

// rsylv::relative_residual (testgen.hpp:459-460)
int ref_relative_residual(std::size_t m, std::size_t n, const double* a, const double* b,
                          const double* c, const double* y, double alpha, double* out) {
    return guarded([&] {
        *out = relative_residual(ConstMatrixView{a, m, m, m}, ConstMatrixView{b, n, n, n},
                                 ConstMatrixView{c, m, n, m}, ConstMatrixView{y, m, n, m}, alpha);
    }, nullptr);
}

// Deterministic generators of the reference test suites (testgen.hpp:444-455): pattern
// 0 = mixed (1,2,1,2,...), 1 = ones. Writes an n x n matrix and its block codes.
int ref_generate_quasi_triangular(std::size_t n, double mu, int pattern, double* out,
                                  unsigned char* blk) {
    return guarded([&] {
        QuasiTriangular q = generate_quasi_triangular(
            {n, mu, pattern == 0 ? mixed_pattern(n) : ones_pattern(n)});
        from_dense(q.matrix(), out, n);
        std::memset(blk, 0, n);
        for (const DiagBlock& d : q.diag_blocks()) blk[d.start] = static_cast<unsigned char>(d.size);
    }, nullptr);
}

// verify.hpp:38-41 random_quasi_triangular / random_dense, driven by one mt19937_64 stream in
// the same call order as the reference tests (a, then b, then c).
int ref_random_system(std::uint64_t seed, std::size_t m, std::size_t n, double* a,
                      unsigned char* ablk, double* b, unsigned char* bblk, double* c) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        QuasiTriangular qa = random_quasi_triangular(rng, m);
        QuasiTriangular qb = random_quasi_triangular(rng, n);
        DenseMatrix dc = random_dense(rng, m, n);
        from_dense(qa.matrix(), a, m);
        from_dense(qb.matrix(), b, n);
        from_dense(dc, c, m);
        std::memset(ablk, 0, m);
        std::memset(bblk, 0, n);
        for (const DiagBlock& d : qa.diag_blocks()) ablk[d.start] = static_cast<unsigned char>(d.size);
        for (const DiagBlock& d : qb.diag_blocks()) bblk[d.start] = static_cast<unsigned char>(d.size);
    }, nullptr);
}

// verify.hpp:47-48 dense_kron_solve (mn x mn Gaussian elimination, partial pivoting)
int ref_dense_kron_solve(std::size_t m, std::size_t n, const double* a, const unsigned char* ablk,
                         const double* b, const unsigned char* bblk, const double* c, double* y) {
    return guarded([&] {
        QuasiTriangular qa = to_qt(a, m, m, ablk), qb = to_qt(b, n, n, bblk);
        DenseMatrix r = dense_kron_solve(qa, qb, ConstMatrixView{c, m, n, m});
        from_dense(r, y, m);
    }, nullptr);
}

// matrix_io.hpp format_double (std::to_chars shortest round trip): the CSV / matrix-file number
// format, for pinning paper_1905_10574_b200/records.py. Returns the string length.
int ref_format_double(double v, char* buf, std::size_t cap) {
    const std::string s = format_double(v);
    if (s.size() + 1 > cap) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
}

} // extern "C"
