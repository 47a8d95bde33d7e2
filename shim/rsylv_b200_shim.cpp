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
//  * ExecutionMode::workers (tiled_solve.hpp:16-22) maps to GPUs:
//    workers <= 1 -> one GPU; workers = w >= 2 -> min(w, visible GPUs, 8) GPUs of this process
//    (rsylv_b200_solve_group: tile columns block-cyclic, solved tiles pushed over NVLink). With a
//    single visible GPU and RSYLV_B200_VIRTUAL_RANKS=1 in the environment, min(w, 8) virtual
//    ranks share that GPU instead (the same exchange, used by the tests); a TileProbe request
//    keeps the solve on one GPU (the probe log is per GPU);
//  * TileProbe is replayed after the solve from the device's probe log, tile indices of the
//    B200 partition (tiles <= 128, cut moved earlier around 2x2 blocks).
#include <algorithm>
#include <atomic>
#include <cstdlib>
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
std::vector<rsylv_b200_ctx*> g_group;  // one context per GPU for workers >= 2

rsylv_b200_ctx* context() {
    if (!g_ctx) {
        const int st = rsylv_b200_create(-1, &g_ctx);
        if (st != RSYLV_OK)
            throw std::runtime_error(std::string("rsylv-b200: no usable CUDA device (") +
                                     rsylv_b200_status_string(st) + ")");
    }
    return g_ctx;
}

// contexts of GPUs 0 .. R-1 (context 0 is the single-GPU one when it lives on device 0)
const std::vector<rsylv_b200_ctx*>& group(int R) {
    while ((int)g_group.size() < R) {
        const int d = (int)g_group.size();
        rsylv_b200_ctx* c = nullptr;
        const int st = rsylv_b200_create(d, &c);
        if (st != RSYLV_OK)
            throw std::runtime_error(std::string("rsylv-b200: cannot open GPU ") + std::to_string(d));
        g_group.push_back(c);
    }
    return g_group;
}

bool env_on(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] == '1';
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
        const int w = (int)std::min<std::size_t>(mode.workers, 8);
        const int gpus = w >= 2 && !probe ? rsylv_b200_device_count() : 1;
        if (w >= 2 && !probe && gpus >= 2) {
            const int R = std::min(w, gpus);
            st = rsylv_b200_solve_group(group(R).data(), R, m, n, a.matrix().data(), m, ac.data(),
                                        b.matrix().data(), n, bc.data(), c.data, c.ld,
                                        out.y.data(), m, &opt, &res);
        } else {
            if (w >= 2 && !probe && env_on("RSYLV_B200_VIRTUAL_RANKS")) opt.virtual_ranks = w;
            st = rsylv_b200_solve(context(), m, n, a.matrix().data(), m, ac.data(),
                                  b.matrix().data(), n, bc.data(), c.data, c.ld, out.y.data(), m,
                                  &opt, &res);
        }
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
                                     ": " + rsylv_b200_last_error(g_ctx ? g_ctx : g_group.front()));
    }
}

}  // namespace rsylv
