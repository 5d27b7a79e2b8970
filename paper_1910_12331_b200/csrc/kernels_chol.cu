// R x R symmetric positive-definite kernels (fp64, sm_100a).
//
// Reference semantics (matrix_ops.cpp:41-81): Cholesky (LLT) of S + lambda I;
// on failure (a pivot <= 0) retry once with jitter 1e-12 * tr(S) / R added to
// the diagonal, else SingularSystem. spd_solve returns Y with
// Y (S + lambda I) = B, spd_inverse the symmetrised inverse.
//
// Device design: L is kept as a dense square with odd row stride LD = R + 1
// (row and column walks both conflict-free in shared memory). One CTA per
// matrix factorises right-looking (each of the R steps is a 2-D parallel
// rank-1 trailing update) in shared memory when LD * R fits, else in the
// L2-resident global output. Solves run one warp per right-hand-side row,
// lanes owning rhs entries in registers, L staged once per CTA in shared
// memory, the 32-step blocks unrolled so every register index is static.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace cpkit {

namespace {

constexpr std::size_t kSmemBudget = 200 * 1024;

inline int lda_of(int R) { return R + 1; }
inline bool chol_in_smem(int R) { return static_cast<std::size_t>(R) * lda_of(R) * 8 <= kSmemBudget; }

// mode 0: A = S + lambda I; mode 1: A = S with diag *= (1 + lambda), lambda'=0.
// Jitter trace uses the matrix handed to factor_shifted (gauss_newton.cpp:190-207).
// kSmem selects the working copy's address space at compile time (LDS/STS).
template <bool kSmem>
__global__ void __launch_bounds__(512) chol_kernel(const double* __restrict__ s_all, int R, double lambda, int mode,
                                                   double* __restrict__ l_all, int* __restrict__ status) {
    extern __shared__ double sh[];
    const int LD = R + 1;
    const int mat = blockIdx.x;
    const double* s = s_all + static_cast<long long>(mat) * R * R;
    double* out = l_all + static_cast<long long>(mat) * R * LD;
    double* w = kSmem ? sh : out;
    __shared__ double trace_sh;
    __shared__ int fail_sh;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;

    if (ty == 0) {  // trace, warp-parallel (fixed shuffle order)
        double tr = 0.0;
        for (int i = tx; i < R; i += 32) {
            const double d = s[static_cast<long long>(i) * R + i];
            tr += (mode == 1) ? d * (1.0 + lambda) : d;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tr += __shfl_down_sync(0xffffffffu, tr, o);
        if (tx == 0) trace_sh = tr;
    }
    __syncthreads();
    const double jitter = 1e-12 * trace_sh / static_cast<double>(R);

    int st = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const double add = (mode == 0 ? lambda : 0.0);
        for (int i = ty; i < R; i += ny)
            for (int k = tx; k <= i; k += 32) {
                double v = s[static_cast<long long>(i) * R + k];
                if (i == k) {
                    if (mode == 1) v *= (1.0 + lambda);
                    v += add;
                    if (attempt == 1) v += jitter;
                }
                w[i * LD + k] = v;
            }
        if (threadIdx.x == 0) fail_sh = 0;
        __syncthreads();
        // blocked right-looking: warp 0 factors a kNb-column panel with warp-level
        // syncs only, then all warps apply the rank-kNb trailing update.
        constexpr int kNb = 16;
        for (int j0 = 0; j0 < R && !fail_sh; j0 += kNb) {
            const int j1 = min(R, j0 + kNb);
            if (ty == 0) {
                for (int j = j0; j < j1; ++j) {
                    const double x = w[j * LD + j];
                    if (!(x > 0.0) && !isnan(x)) {  // Eigen LLT: fail iff pivot <= 0
                        if (tx == 0) fail_sh = 1;
                        break;
                    }
                    const double l = sqrt(x);
                    const double inv = 1.0 / l;
                    __syncwarp();
                    for (int i = j + 1 + tx; i < R; i += 32) w[i * LD + j] *= inv;
                    if (tx == 0) {
                        w[j * LD + j] = l;
                        w[j * LD + R] = inv;  // padding column keeps 1 / L_jj for the solves
                    }
                    __syncwarp();
                    for (int i = j + 1 + tx; i < R; i += 32) {
                        const double lij = w[i * LD + j];
                        const int kend = min(j1, i + 1);
                        for (int k = j + 1; k < kend; ++k) w[i * LD + k] -= lij * w[k * LD + j];
                    }
                    __syncwarp();
                }
            }
            __syncthreads();
            if (fail_sh) break;
            // trailing update a_ik -= sum_{j in panel} l_ij l_kj, j1 <= k <= i
            for (int i = j1 + ty; i < R; i += ny)
                for (int k = j1 + tx; k <= i; k += 32) {
                    double acc = w[i * LD + k];
                    for (int j = j0; j < j1; ++j) acc -= w[i * LD + j] * w[k * LD + j];
                    w[i * LD + k] = acc;
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
    if (kSmem)
        for (int i = ty; i < R; i += ny) {
            for (int k = tx; k <= i; k += 32) out[i * LD + k] = w[i * LD + k];
            if (tx == 0) out[i * LD + R] = w[i * LD + R];
        }
    if (threadIdx.x == 0) status[mat] = st;
}

// One warp per rhs row: solve (L L^T) y = b, L lower with row stride LD;
// column R of each row holds 1 / L_ii (written by chol_kernel).
constexpr int kMaxBlk = 16;  // R <= 512
constexpr int kSolveWarps = 8;
template <bool kSmem>
__global__ void __launch_bounds__(32 * kSolveWarps)
chol_solve_rows_kernel(const double* __restrict__ l_all, int R, const double* __restrict__ b, long long rows,
                       double* __restrict__ y, long long l_stride, long long rows_per_mat) {
    extern __shared__ double lsh[];
    const int LD = R + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long mat = blockIdx.y;
    const double* Lg = l_all + mat * l_stride;
    if (kSmem) {
        for (int i = warp; i < R; i += kSolveWarps) {
            for (int k = lane; k <= i; k += 32) lsh[i * LD + k] = Lg[i * LD + k];
            if (lane == 0) lsh[i * LD + R] = Lg[i * LD + R];
        }
        __syncthreads();
    }
    const double* L = kSmem ? lsh : Lg;
    const int nblk = (R + 31) / 32;
    for (long long local = blockIdx.x * kSolveWarps + warp; local < rows_per_mat;
         local += static_cast<long long>(gridDim.x) * kSolveWarps) {
        const long long row = mat * rows_per_mat + local;
        if (row >= rows) break;
        double v[kMaxBlk];
#pragma unroll
        for (int c = 0; c < kMaxBlk; ++c) {
            const int k = lane + 32 * c;
            v[c] = (c < nblk && k < R) ? b[row * R + k] : 0.0;
        }
        // forward: z_i = v_i / L_ii ; v_k -= L_ki z_i (k > i)   [column walk, stride LD]
#pragma unroll
        for (int cb = 0; cb < kMaxBlk; ++cb) {
            if (cb < nblk) {
                const int iend = min(32, R - 32 * cb);
                for (int il = 0; il < iend; ++il) {
                    const int i = 32 * cb + il;
                    const double zi = __shfl_sync(0xffffffffu, v[cb], il) * L[i * LD + R];
                    if (lane == il) v[cb] = zi;
                    if (lane > il && lane + 32 * cb < R) v[cb] -= L[(lane + 32 * cb) * LD + i] * zi;
#pragma unroll
                    for (int c = cb + 1; c < kMaxBlk; ++c) {
                        const int k = lane + 32 * c;
                        if (c < nblk && k < R) v[c] -= L[k * LD + i] * zi;
                    }
                }
            }
        }
        // backward with L^T: y_i = v_i / L_ii ; v_k -= L_ik y_i (k < i)   [row walk]
#pragma unroll
        for (int cb = kMaxBlk - 1; cb >= 0; --cb) {
            if (cb < nblk) {
                const int iend = min(32, R - 32 * cb);
                for (int il = iend - 1; il >= 0; --il) {
                    const int i = 32 * cb + il;
                    const double yi = __shfl_sync(0xffffffffu, v[cb], il) * L[i * LD + R];
                    if (lane == il) v[cb] = yi;
                    if (lane < il) v[cb] -= L[i * LD + lane + 32 * cb] * yi;
#pragma unroll
                    for (int c = 0; c < cb; ++c) v[c] -= L[i * LD + lane + 32 * c] * yi;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < kMaxBlk; ++c) {
            const int k = lane + 32 * c;
            if (c < nblk && k < R) y[row * R + k] = v[c];
        }
    }
}

void solve_rows(const double* l, int R, const double* b, long long rows, double* y, long long l_stride,
                int nmats, long long rows_per_mat, cudaStream_t st) {
    const std::size_t bytes = static_cast<std::size_t>(R) * lda_of(R) * 8;
    const bool smem = bytes <= kSmemBudget;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long per_mat_ctas = std::max<long long>(
        1, std::min<long long>((rows_per_mat + kSolveWarps - 1) / kSolveWarps, std::max(1, 2 * sms / nmats)));
    dim3 grid(static_cast<unsigned>(per_mat_ctas), nmats);
    if (smem) {
        CPK_CUDA(cudaFuncSetAttribute(chol_solve_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(bytes)));
        chol_solve_rows_kernel<true><<<grid, 32 * kSolveWarps, bytes, st>>>(l, R, b, rows, y, l_stride, rows_per_mat);
    } else {
        chol_solve_rows_kernel<false><<<grid, 32 * kSolveWarps, 0, st>>>(l, R, b, rows, y, l_stride, rows_per_mat);
    }
    count_launch(1);
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
__global__ void symmetrize_kernel(const double* __restrict__ y, int count, int R, double* __restrict__ inv) {
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

std::size_t chol_factor_elems(int count, int R) { return static_cast<std::size_t>(count) * R * lda_of(R); }

void launch_chol_batch(const double* s, int count, int R, const double* lambda, int mode, double* l_out, int* status,
                       cudaStream_t st) {
    if (R > 32 * kMaxBlk) throw LimitExceeded("rank exceeds the device SPD solver limit (512)");
    const bool use_smem = chol_in_smem(R);
    const std::size_t smem = use_smem ? static_cast<std::size_t>(R) * lda_of(R) * 8 : 0;
    if (use_smem) {
        CPK_CUDA(cudaFuncSetAttribute(chol_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        chol_kernel<true><<<count, 512, smem, st>>>(s, R, *lambda, mode, l_out, status);
    } else {
        chol_kernel<false><<<count, 512, 0, st>>>(s, R, *lambda, mode, l_out, status);
    }
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_chol_solve_rows(const double* l, int R, const double* b, std::int64_t rows, double* y, cudaStream_t st) {
    solve_rows(l, R, b, rows, y, 0, 1, rows, st);
}

void launch_chol_inverse_batch(const double* l, int count, int R, double* inv, double* tmp, cudaStream_t st) {
    const long long rr = static_cast<long long>(R) * R;
    const long long total = count * rr;
    const int g = static_cast<int>(std::min<long long>((total + 255) / 256, 1184));
    identity_rows_kernel<<<g, 256, 0, st>>>(inv, count, R);
    count_launch(1);
    const long long rows = static_cast<long long>(count) * R;
    solve_rows(l, R, inv, rows, tmp, static_cast<long long>(R) * lda_of(R), count, R, st);
    symmetrize_kernel<<<g, 256, 0, st>>>(tmp, count, R, inv);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

}  // namespace cpkit
