// Dense reference routes for cpkit_run_selftest_oracle (selftest.cpp:15-240),
// evaluated on the device for small instances (prod s <= a few hundred):
// the explicit Gauss-Newton matrix J^T J (gauss_newton.cpp:138-188 column
// order: mode-major, column-major per factor), the dense objective
// 0.5 ||X - reconstruct(A)||^2 and its central finite differences, and the
// dense residual. They check the implicit device operators (matvec, gradient,
// CG, fast residual) the same way the reference's self-test checks its own.
#include <cuda_runtime.h>

#include "common.h"
#include "selftest.h"

namespace cpkit {
namespace {

struct Geo {
    int order, rank;
    int dims[kMaxOrder];
    long long off[kMaxOrder + 1];  // stacked (row-major factor blocks)
    long long colb[kMaxOrder + 1];  // column blocks of J (dims[n] * rank each)
    long long numel;
};

__device__ void index_of(const Geo& g, long long f, int* idx) {
    for (int m = g.order - 1; m >= 0; --m) {
        idx[m] = static_cast<int>(f % g.dims[m]);
        f /= g.dims[m];
    }
}
// J[f][col] for col = colb[n] + r * dims[n] + i: -prod_{m != n} A_m[idx_m, r] when idx_n == i
__device__ double jac(const Geo& g, const double* A, const int* idx, long long col) {
    int n = 0;
    while (col >= g.colb[n + 1]) ++n;
    const long long local = col - g.colb[n];
    const int r = static_cast<int>(local / g.dims[n]), i = static_cast<int>(local % g.dims[n]);
    if (idx[n] != i) return 0.0;
    double p = 1.0;
    for (int m = 0; m < g.order; ++m)
        if (m != n) p *= A[g.off[m] + static_cast<long long>(idx[m]) * g.rank + r];
    return -p;
}

__global__ void explicit_jtj_kernel(Geo g, const double* A, double* H, long long vars) {
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < vars * vars;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long a = e / vars, b = e % vars;
        int idx[kMaxOrder];
        double acc = 0.0;
        for (long long f = 0; f < g.numel; ++f) {
            index_of(g, f, idx);
            const double ja = jac(g, A, idx, a);
            if (ja != 0.0) acc += ja * jac(g, A, idx, b);
        }
        H[e] = acc;
    }
}

__device__ double model_entry(const Geo& g, const double* A, const int* idx) {
    double acc = 0.0;
    for (int r = 0; r < g.rank; ++r) {
        double p = 1.0;
        for (int m = 0; m < g.order; ++m) p *= A[g.off[m] + static_cast<long long>(idx[m]) * g.rank + r];
        acc += p;
    }
    return acc;
}
// objective with one stacked entry perturbed by +-h (or none: var < 0)
__device__ double objective(const Geo& g, const double* A, const double* x, long long var, double delta) {
    int idx[kMaxOrder];
    int vn = 0, vi = 0, vr = 0;
    double orig = 0.0;
    if (var >= 0) {
        while (var >= g.off[vn + 1]) ++vn;
        vi = static_cast<int>((var - g.off[vn]) / g.rank);
        vr = static_cast<int>((var - g.off[vn]) % g.rank);
        orig = A[var];
    }
    double acc = 0.0;
    for (long long f = 0; f < g.numel; ++f) {
        index_of(g, f, idx);
        double m = 0.0;
        for (int r = 0; r < g.rank; ++r) {
            double p = 1.0;
            for (int mm = 0; mm < g.order; ++mm) {
                double a = A[g.off[mm] + static_cast<long long>(idx[mm]) * g.rank + r];
                if (var >= 0 && mm == vn && idx[mm] == vi && r == vr) a = orig + delta;
                p *= a;
            }
            m += p;
        }
        const double d = x[f] - m;
        acc += d * d;
    }
    return 0.5 * acc;
}
__global__ void fd_gradient_kernel(Geo g, const double* A, const double* x, double h, double* out, long long vars) {
    for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < vars;
         v += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double fp = objective(g, A, x, v, h), fm = objective(g, A, x, v, -h);
        out[v] = (fp - fm) / (2.0 * h);
    }
}
__global__ void dense_residual_kernel(Geo g, const double* A, const double* x, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int idx[kMaxOrder];
    double acc = 0.0, xn = 0.0;
    for (long long f = 0; f < g.numel; ++f) {
        index_of(g, f, idx);
        const double d = x[f] - model_entry(g, A, idx);
        acc += d * d;
        xn += x[f] * x[f];
    }
    out[0] = sqrt(acc) / sqrt(xn);
}

// M^(n)[i][r] = sum over entries with idx_n = i of X[f] prod_{m != n} A_m[idx_m][r]
// (matricize(X, n) * Khatri-Rao, selftest.cpp:161-170), one thread per (i, r)
__global__ void dense_mttkrp_kernel(Geo g, const double* A, const double* x, int mode, double* out) {
    const int rows = g.dims[mode];
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * g.rank; e += gridDim.x * blockDim.x) {
        const int i = e / g.rank, r = e % g.rank;
        int idx[kMaxOrder];
        double acc = 0.0;
        for (long long f = 0; f < g.numel; ++f) {
            index_of(g, f, idx);
            if (idx[mode] != i) continue;
            double p = x[f];
            for (int m = 0; m < g.order; ++m)
                if (m != mode) p *= A[g.off[m] + static_cast<long long>(idx[m]) * g.rank + r];
            acc += p;
        }
        out[e] = acc;
    }
}

Geo make_geo(const std::vector<std::uint64_t>& dims, int rank) {
    Geo g{};
    g.order = static_cast<int>(dims.size());
    g.rank = rank;
    g.off[0] = g.colb[0] = 0;
    g.numel = 1;
    for (int n = 0; n < g.order; ++n) {
        g.dims[n] = static_cast<int>(dims[n]);
        g.off[n + 1] = g.off[n] + static_cast<long long>(dims[n]) * rank;
        g.colb[n + 1] = g.off[n + 1];
        g.numel *= static_cast<long long>(dims[n]);
    }
    return g;
}

}  // namespace

void launch_explicit_jtj(const std::vector<std::uint64_t>& dims, int rank, const double* A, double* H,
                         cudaStream_t st) {
    const Geo g = make_geo(dims, rank);
    const long long vars = g.off[g.order];
    explicit_jtj_kernel<<<static_cast<int>((vars * vars + 127) / 128), 128, 0, st>>>(g, A, H, vars);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
void launch_fd_gradient(const std::vector<std::uint64_t>& dims, int rank, const double* A, const double* x,
                        double h, double* out, cudaStream_t st) {
    const Geo g = make_geo(dims, rank);
    const long long vars = g.off[g.order];
    fd_gradient_kernel<<<static_cast<int>((vars + 63) / 64), 64, 0, st>>>(g, A, x, h, out, vars);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
void launch_dense_mttkrp(const std::vector<std::uint64_t>& dims, int rank, const double* A, const double* x,
                         int mode, double* out, cudaStream_t st) {
    const Geo g = make_geo(dims, rank);
    const int n = static_cast<int>(dims[mode]) * rank;
    dense_mttkrp_kernel<<<(n + 63) / 64, 64, 0, st>>>(g, A, x, mode, out);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
void launch_dense_residual(const std::vector<std::uint64_t>& dims, int rank, const double* A, const double* x,
                           double* out, cudaStream_t st) {
    const Geo g = make_geo(dims, rank);
    dense_residual_kernel<<<1, 32, 0, st>>>(g, A, x, out);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

}  // namespace cpkit
