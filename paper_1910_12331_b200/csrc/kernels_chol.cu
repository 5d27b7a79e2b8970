// R x R symmetric positive-definite kernels (fp64, sm_100a).
//
// Reference semantics (matrix_ops.cpp:41-81): Cholesky (LLT) of S + lambda I;
// on failure (a pivot <= 0) retry once with jitter 1e-12 * tr(S) / R added to
// the diagonal, else SingularSystem. spd_solve returns Y with
// Y (S + lambda I) = B, spd_inverse the symmetrised inverse.
//
// Device design: one CTA per matrix factorises a packed lower triangle
// (R(R+1)/2 doubles) held in shared memory when it fits (R <= 240), else in
// the global output buffer; right-looking so each of the R steps is a fully
// parallel rank-1 trailing update. Solves run one warp per right-hand-side
// row with column-oriented substitution (lanes own rhs entries in registers).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace cpkit {

namespace {

__device__ __forceinline__ long long pk(int i, int j) {  // packed lower, i >= j
    return static_cast<long long>(i) * (i + 1) / 2 + j;
}

// mode 0: A = S + lambda I; mode 1: A = S with diag *= (1 + lambda), lambda'=0.
// Jitter trace uses the matrix handed to factor_shifted (gauss_newton.cpp:190-207).
__global__ void chol_kernel(const double* __restrict__ s_all, int R, double lambda, int mode,
                            double* __restrict__ l_all, int* __restrict__ status, int use_smem) {
    extern __shared__ double sh[];
    const int mat = blockIdx.x;
    const double* s = s_all + static_cast<long long>(mat) * R * R;
    const long long np = static_cast<long long>(R) * (R + 1) / 2;
    double* w = use_smem ? sh : l_all + mat * np;
    __shared__ double trace_sh;
    __shared__ int fail_sh;

    if (threadIdx.x == 0) {
        double tr = 0.0;
        for (int i = 0; i < R; ++i) {
            const double d = s[static_cast<long long>(i) * R + i];
            tr += (mode == 1) ? d * (1.0 + lambda) : d;
        }
        trace_sh = tr;
    }
    __syncthreads();
    const double jitter = 1e-12 * trace_sh / static_cast<double>(R);

    int st = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const double add = (mode == 0 ? lambda : 0.0);
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int i = warp; i < R; i += nw) {
            for (int j = lane; j <= i; j += 32) {
                double v = s[static_cast<long long>(i) * R + j];
                if (i == j) {
                    if (mode == 1) v *= (1.0 + lambda);
                    v += add;
                    if (attempt == 1) v += jitter;
                }
                w[pk(i, j)] = v;
            }
        }
        if (threadIdx.x == 0) fail_sh = 0;
        __syncthreads();
        for (int j = 0; j < R; ++j) {
            const double x = w[pk(j, j)];
            if (!(x > 0.0) && !isnan(x)) {  // Eigen LLT: fail iff pivot <= 0
                if (threadIdx.x == 0) fail_sh = 1;
            }
            __syncthreads();
            if (fail_sh) break;
            const double l = sqrt(x);
            // scale column j below the diagonal
            for (int i = j + 1 + threadIdx.x; i < R; i += blockDim.x) w[pk(i, j)] /= l;
            __syncthreads();
            if (threadIdx.x == 0) w[pk(j, j)] = l;
            // trailing update: a_ik -= l_ij l_kj for j < k <= i (warp per row)
            for (int i = j + 1 + warp; i < R; i += nw) {
                const double lij = w[pk(i, j)];
                for (int k = j + 1 + lane; k <= i; k += 32) w[pk(i, k)] -= lij * w[pk(k, j)];
            }
            __syncthreads();
        }
        if (!fail_sh) {
            st = attempt;  // 0 ok, 1 ok after jitter
            break;
        }
        st = 2;
        __syncthreads();
    }
    if (use_smem) {
        double* out = l_all + mat * np;
        for (long long e = threadIdx.x; e < np; e += blockDim.x) out[e] = w[e];
    }
    if (threadIdx.x == 0) status[mat] = st;
}

// One warp per rhs row: solve (L L^T) y = b; L packed lower (R(R+1)/2),
// staged once per CTA in shared memory (every row of a CTA uses the same L).
// Lane q owns entries k = q + 32*c, c < kMaxPer, in registers.
constexpr int kMaxPer = 16;  // R <= 512
constexpr int kSolveWarps = 8;
template <bool kSmem>
__global__ void __launch_bounds__(32 * kSolveWarps)
chol_solve_rows_kernel(const double* __restrict__ l_all, int R, const double* __restrict__ b, long long rows,
                       double* __restrict__ y, long long l_stride, long long rows_per_mat) {
    extern __shared__ double lsh[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long mat = blockIdx.y;
    const double* Lg = l_all + mat * l_stride;
    const long long np = static_cast<long long>(R) * (R + 1) / 2;
    if (kSmem) {
        for (long long e = threadIdx.x; e < np; e += blockDim.x) lsh[e] = Lg[e];
        __syncthreads();
    }
    const double* L = kSmem ? lsh : Lg;
    for (long long local = blockIdx.x * kSolveWarps + warp; local < rows_per_mat;
         local += static_cast<long long>(gridDim.x) * kSolveWarps) {
        const long long row = mat * rows_per_mat + local;
        if (row >= rows) break;
        double v[kMaxPer];
#pragma unroll
        for (int c = 0; c < kMaxPer; ++c) {
            const int k = lane + 32 * c;
            v[c] = (k < R) ? b[row * R + k] : 0.0;
        }
        // forward: z_i = v_i / L_ii ; v_k -= L_ki z_i (k > i)
        for (int i = 0; i < R; ++i) {
            const int owner = i & 31, ci = i >> 5;
            double vi = 0.0;
#pragma unroll
            for (int c = 0; c < kMaxPer; ++c)
                if (c == ci) vi = v[c];
            vi = __shfl_sync(0xffffffffu, vi, owner);
            const double zi = vi / L[pk(i, i)];
#pragma unroll
            for (int c = 0; c < kMaxPer; ++c) {
                const int k = lane + 32 * c;
                if (k == i) v[c] = zi;
                else if (k > i && k < R) v[c] -= L[pk(k, i)] * zi;
            }
        }
        // backward with L^T: y_i = v_i / L_ii ; v_k -= L_ik y_i (k < i)
        for (int i = R - 1; i >= 0; --i) {
            const int owner = i & 31, ci = i >> 5;
            double vi = 0.0;
#pragma unroll
            for (int c = 0; c < kMaxPer; ++c)
                if (c == ci) vi = v[c];
            vi = __shfl_sync(0xffffffffu, vi, owner);
            const double yi = vi / L[pk(i, i)];
#pragma unroll
            for (int c = 0; c < kMaxPer; ++c) {
                const int k = lane + 32 * c;
                if (k == i) v[c] = yi;
                else if (k < i) v[c] -= L[pk(i, k)] * yi;
            }
        }
#pragma unroll
        for (int c = 0; c < kMaxPer; ++c) {
            const int k = lane + 32 * c;
            if (k < R) y[row * R + k] = v[c];
        }
    }
}

void solve_rows(const double* l, int R, const double* b, long long rows, double* y, long long l_stride,
                int nmats, long long rows_per_mat, cudaStream_t st) {
    const std::size_t np = static_cast<std::size_t>(R) * (R + 1) / 2;
    const bool smem = np * 8 <= 200 * 1024;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long per_mat_ctas = std::max<long long>(
        1, std::min<long long>((rows_per_mat + kSolveWarps - 1) / kSolveWarps, std::max(1, 2 * sms / nmats)));
    dim3 grid(static_cast<unsigned>(per_mat_ctas), nmats);
    if (smem) {
        CPK_CUDA(cudaFuncSetAttribute(chol_solve_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(np * 8)));
        chol_solve_rows_kernel<true><<<grid, 32 * kSolveWarps, np * 8, st>>>(l, R, b, rows, y, l_stride, rows_per_mat);
    } else {
        chol_solve_rows_kernel<false><<<grid, 32 * kSolveWarps, 0, st>>>(l, R, b, rows, y, l_stride, rows_per_mat);
    }
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

__global__ void identity_rows_kernel(double* __restrict__ out, int count, int R) {
    const long long total = static_cast<long long>(count) * R * R;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long w = e % (static_cast<long long>(R) * R);
        out[e] = (w / R == w % R) ? 1.0 : 0.0;
    }
}
// inv = 0.5 (Y + Y^T) per matrix (matrix_ops.cpp:78-79)
__global__ void symmetrize_kernel(const double* __restrict__ y, int count, int R,
                                  double* __restrict__ inv) {
    const long long rr = static_cast<long long>(R) * R;
    const long long total = count * rr;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long m = e / rr, w = e % rr;
        const long long i = w / R, j = w % R;
        inv[e] = 0.5 * (y[m * rr + i * R + j] + y[m * rr + j * R + i]);
    }
}

}  // namespace

void launch_chol_batch(const double* s, int count, int R, const double* lambda, int mode,
                       double* l_out, int* status, cudaStream_t st) {
    if (R > 32 * kMaxPer) throw LimitExceeded("rank exceeds the device SPD solver limit (512)");
    const std::size_t np = static_cast<std::size_t>(R) * (R + 1) / 2;
    const bool use_smem = np * 8 <= 220 * 1024;
    const std::size_t smem = use_smem ? np * 8 : 0;
    if (use_smem)
        CPK_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    chol_kernel<<<count, 512, smem, st>>>(s, R, *lambda, mode, l_out, status, use_smem ? 1 : 0); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_chol_solve_rows(const double* l, int R, const double* b, std::int64_t rows, double* y,
                            cudaStream_t st) {
    solve_rows(l, R, b, rows, y, 0, 1, rows, st);
}

void launch_chol_inverse_batch(const double* l, int count, int R, double* inv, double* tmp,
                               cudaStream_t st) {
    const long long rr = static_cast<long long>(R) * R;
    const long long total = count * rr;
    const int g = static_cast<int>(std::min<long long>((total + 255) / 256, 1184));
    identity_rows_kernel<<<g, 256, 0, st>>>(inv, count, R); ::cpkit::count_launch(1);
    const long long rows = static_cast<long long>(count) * R;
    const long long np = static_cast<long long>(R) * (R + 1) / 2;
    solve_rows(l, R, inv, rows, tmp, np, count, R, st);
    symmetrize_kernel<<<g, 256, 0, st>>>(tmp, count, R, inv); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

}  // namespace cpkit
