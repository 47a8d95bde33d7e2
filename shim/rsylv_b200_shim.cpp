// Drop-in definition of the reference entry point on top of the rsylv-b200 C-ABI.
//
// Defines exactly the symbol declared in the reference header
//   /root/reference/proj/include/rsylv/tiled_solve.hpp:36-40
//     rsylv::SolveResult rsylv::solve_tiled_robust(const QuasiTriangular&, const QuasiTriangular&,
//         ConstMatrixView, std::size_t tile_size, const OverflowConfig&, ExecutionMode,
//         const TileProbe&)
// so a maintainer links this translation unit + librsylv_b200.so instead of
// src/tiled_solve.cpp and every existing caller compiles unchanged. Compiled against the
// reference's own headers (layout compatibility of QuasiTriangular / DenseMatrix / SolveResult).
//
// Behaviour mapping:
//  * validation order as the reference: conformance (tiled_solve.cpp:187-188), tile size
//    (partition.cpp:75-76), A/B tile bounds (tile_grid.cpp:63-72), C tile bounds
//    (tiled_solve.cpp:77-79) -> std::invalid_argument;
//  * SingularEquationError(pivot), ScaleUnderflowError as in errors.hpp;
//  * OverflowConfig::scaling_events is bumped by the device's guard-activation count (the
//    granularity differs from the CPU solver: compare trends only);
//  * ExecutionMode::workers is accepted and ignored (one GPU serves every worker count);
//  * TileProbe is replayed after the solve from the device's probe log, tile indices of the
//    B200 partition (tiles <= 128, cut moved earlier around 2x2 blocks).
#include <atomic>
#include <cmath>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "rsylv/errors.hpp"
#include "rsylv/tiled_solve.hpp"
#include "rsylv_b200.h"

namespace {

std::mutex g_mu;
rsylv_b200_ctx* g_ctx = nullptr;

rsylv_b200_ctx* context() {
    if (!g_ctx) {
        const int st = rsylv_b200_create(-1, &g_ctx);
        if (st != RSYLV_OK)
            throw std::runtime_error(std::string("rsylv-b200: no usable CUDA device (") +
                                     rsylv_b200_status_string(st) + ")");
    }
    return g_ctx;
}

std::vector<unsigned char> codes(const rsylv::QuasiTriangular& q) {
    std::vector<unsigned char> c(q.dim(), 0);
    for (const rsylv::DiagBlock& b : q.diag_blocks()) c[b.start] = static_cast<unsigned char>(b.size);
    return c;
}

}  // namespace

namespace rsylv {

SolveResult solve_tiled_robust(const QuasiTriangular& a, const QuasiTriangular& b,
                               ConstMatrixView c, std::size_t tile_size,
                               const OverflowConfig& cfg, ExecutionMode mode,
                               const TileProbe& probe) {
    (void)mode;
    if (c.rows != a.dim() || c.cols != b.dim())
        throw std::invalid_argument("solve_tiled_robust: C does not conform with A and B");
    if (tile_size < 2) throw std::invalid_argument("partition: requested tile size must be >= 2");
    const std::size_t m = c.rows, n = c.cols;
    SolveResult out;
    out.y = DenseMatrix(m, n);
    if (m == 0 || n == 0) return out;

    const std::vector<unsigned char> ac = codes(a), bc = codes(b);
    rsylv_b200_options opt{cfg.omega, cfg.small_num, tile_size, 0, 0};
    rsylv_b200_result res{};
    std::vector<rsylv_b200_probe_event> log;
    if (probe) {
        log.resize(std::size_t(1) << 22);
        res.probe_log = log.data();
        res.probe_cap = log.size();
    }
    int st;
    {
        std::lock_guard<std::mutex> hold(g_mu);
        st = rsylv_b200_solve(context(), m, n, a.matrix().data(), m, ac.data(),
                              b.matrix().data(), n, bc.data(), c.data, c.ld, out.y.data(), m,
                              &opt, &res);
    }
    if (cfg.scaling_events) cfg.scaling_events->fetch_add(res.scaling_events, std::memory_order_relaxed);
    if (probe) {
        const std::size_t ne = std::min(res.probe_count, res.probe_cap);
        for (std::size_t t = 0; t < ne; ++t)
            probe(log[t].k, log[t].l, std::ldexp(1.0, log[t].scale_exp), log[t].norm);
    }
    switch (st) {
        case RSYLV_OK:
            out.alpha = res.alpha;
            return out;
        case RSYLV_INVALID_ARGUMENT:
            switch (res.invalid_reason) {
                case RSYLV_REASON_A_BOUND:
                    throw std::invalid_argument("compute_bounds: a tile norm of A exceeds omega");
                case RSYLV_REASON_B_BOUND:
                    throw std::invalid_argument("compute_bounds: a tile norm of B exceeds omega");
                case RSYLV_REASON_C_BOUND:
                    throw std::invalid_argument("solve_tiled_robust: a tile norm of C exceeds omega");
                default:
                    throw std::invalid_argument("solve_tiled_robust: invalid argument");
            }
        case RSYLV_SINGULAR:
            throw SingularEquationError(res.pivot);
        case RSYLV_SCALE_UNDERFLOW:
            throw ScaleUnderflowError();
        default:
            throw std::runtime_error(std::string("rsylv-b200: ") + rsylv_b200_status_string(st) +
                                     ": " + rsylv_b200_last_error(g_ctx));
    }
}

}  // namespace rsylv
