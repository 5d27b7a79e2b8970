// Dense reference routes on the device for cpkit_run_selftest_oracle (kernels_selftest.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace cpkit {
// H = J^T J (vars x vars, vars = sum_n s_n R; J columns mode-major, column-major per factor)
void launch_explicit_jtj(const std::vector<std::uint64_t>& dims, int rank, const double* A, double* H,
                         cudaStream_t st);
// central differences of 0.5 ||X - [[A]]||^2 w.r.t. every stacked factor entry
void launch_fd_gradient(const std::vector<std::uint64_t>& dims, int rank, const double* A, const double* x,
                        double h, double* out, cudaStream_t st);
// M^(mode) by the dense unfolding route
void launch_dense_mttkrp(const std::vector<std::uint64_t>& dims, int rank, const double* A, const double* x,
                         int mode, double* out, cudaStream_t st);
// ||X - [[A]]|| / ||X||
void launch_dense_residual(const std::vector<std::uint64_t>& dims, int rank, const double* A, const double* x,
                           double* out, cudaStream_t st);
}  // namespace cpkit
