// Batched tiny-instance solver (kernels_tiny.cu): one CTA per independent
// ALS / GN-CG optimisation, for the likelihood and matmul protocols
// (harness.cpp:488-653).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace cpkit {

constexpr int kTinyMaxOrder = 8;
constexpr int kTinyMaxRank = 64;
constexpr int kTinyThreads = 128;
constexpr std::size_t kTinySmemMax = 200 * 1024;

struct TinyLayout {  // shared-memory offsets (doubles)
    int x, a, root0, root1, t0, t1, grams, gam, l, inv, misc, m, add, g, v, r, z, w, q, at, pairs, pinv, tb, td, bp;
    int total;
};
struct TinyAls {  // AlsConfig (als.hpp:11-22); lambdas[k] = lambda0 / decay^k (host std::pow)
    int max_sweeps;
    double residual_tol, step_tol, lambda0;
    int decay_every;
    const double* lambdas;
};
struct TinyGn {  // GnConfig (gauss_newton.hpp:50-62) with the resolved CG cap
    double grad_tol, residual_tol, step_tol, cg_tol;
    int max_iters, cap;
    int mode;       // 0 constant, 1 varying
    int shape;      // 0 identity, 1 diagonal
    double lambda, mu, lower, upper;
    int direction;  // 0 down, 1 up
    int armijo;
    double c1, shrink;
    int max_backtracks;
    int beta_variant;
};
struct TinyParams {
    int order, rank;
    int dims[kTinyMaxOrder];
    int off[kTinyMaxOrder + 1];  // stacked factor offsets (elements)
    int S, numel, count;
    int optimizer;               // 0 ALS, 1 GN
    int threads;                 // CTA size (32 for the smallest shapes: one warp, cheap barriers)
    TinyAls als;
    TinyGn gn;
    TinyLayout layout;
    const double* x;             // tensors, numel each
    const int* x_index;          // instance -> tensor
    const double* init;          // count x S stacked factors
    double* factors_out;         // optional: count x S final factors
    int* status;                 // TerminalStatus order: 0 residual, 1 step, 2 cap, 3 numerical failure
    int* iterations;
    double* final_residual;
    double* best_residual;
};

// false when the instance shape does not fit one CTA
bool tiny_layout(int order, const std::uint64_t* dims, int rank, TinyLayout& layout, int& numel, int& S);
void launch_tiny(const TinyParams& p, cudaStream_t st);

}  // namespace cpkit
