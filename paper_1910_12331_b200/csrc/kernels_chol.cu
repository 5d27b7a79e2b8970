// R x R symmetric positive-definite kernels (fp64, sm_100a).
//
// Reference semantics (matrix_ops.cpp:41-81): Cholesky (LLT) of S + lambda I;
// on failure (a pivot <= 0) retry once with jitter 1e-12 * tr(S) / R added to
// the diagonal, else SingularSystem. spd_solve returns Y with
// Y (S + lambda I) = B, spd_inverse the symmetrised inverse.
//
// Device design. The factor L lives in global memory as a dense square with
// odd row stride LD = R + 1; column R of row i holds 1 / L_ii so the solves
// multiply instead of divide. One CTA factorises one matrix in shared memory
// (square layout up to R ~ 165, packed lower triangle up to R ~ 233, global
// square beyond), right-looking with ONE barrier per column: every thread
// recomputes the pivot from shared memory, the rank-1 trailing update uses the
// unscaled column and 1 / pivot, and the column is scaled one step later (no
// later step reads it). Solves run one warp per right-hand-side row with the
// rhs in registers, L staged in shared memory, and the block count NB a
// template parameter so no predicated-off work is issued.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "common.h"
#include "tile_gemm.cuh"

namespace cpkit {

namespace {

constexpr std::size_t kSmemBudget = 220 * 1024;
#ifndef CPKIT_CHOL_ABLATE
#define CPKIT_CHOL_ABLATE 0  // timing experiments only: 1 skip diag, 2 skip panel, 4 skip update
#endif
constexpr int kCholAblate = CPKIT_CHOL_ABLATE;
#ifndef CPKIT_CHOL_TRACE
#define CPKIT_CHOL_TRACE 0  // timing experiments only: per-phase globaltimer stamps of CTA 0
#endif
__device__ unsigned long long g_chol_trace[64];
__device__ __forceinline__ void chol_stamp(int k) {
    if (CPKIT_CHOL_TRACE && blockIdx.x == 0 && threadIdx.x == 0 && k < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_chol_trace[k] = t;
    }
}

inline int lda_of(int R) { return R + 1; }

// Index maps. Square: row stride LD, inverse pivots in column R.
// Packed: lower triangle row-major, inverse pivots after it.
struct SqIdx {
    int LD, R;
    __device__ __forceinline__ int at(int i, int k) const { return i * LD + k; }
    __device__ __forceinline__ int inv(int i) const { return i * LD + R; }
};
struct PkIdx {
    int LD, R;  // LD unused
    __device__ __forceinline__ int at(int i, int k) const { return ((i * (i + 1)) >> 1) + k; }
    __device__ __forceinline__ int inv(int i) const { return ((R * (R + 1)) >> 1) + i; }
};
inline std::size_t sq_bytes(int R) { return static_cast<std::size_t>(R) * lda_of(R) * 8; }
inline std::size_t pk_bytes(int R) { return (static_cast<std::size_t>(R) * (R + 1) / 2 + R) * 8; }
enum Layout { kSquareSmem = 0, kPackedSmem = 1, kGlobal = 2 };
inline Layout layout_of(int R) {
    if (sq_bytes(R) <= kSmemBudget) return kSquareSmem;
    if (pk_bytes(R) <= kSmemBudget) return kPackedSmem;
    return kGlobal;
}

// mode 0: A = S + lambda I; mode 1: A = S with diag *= (1 + lambda), lambda'=0.
// Jitter trace uses the matrix handed to factor_shifted (gauss_newton.cpp:190-207).
template <class Idx, bool kSmem>
__global__ void __launch_bounds__(512) chol_kernel(const double* __restrict__ s_all, int R, double lambda, int mode,
                                                   double* __restrict__ l_all, int* __restrict__ status,
                                                   long long s_stride) {
    extern __shared__ double sh[];
    const int LD = R + 1;
    const int mat = blockIdx.x;
    const double* s = s_all + static_cast<long long>(mat) * s_stride;
    double* out = l_all + static_cast<long long>(mat) * R * LD;
    double* w = kSmem ? sh : out;
    const Idx ix{LD, R};
    __shared__ double trace_sh, piv_sh[3];
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

    int st = 2;
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
                w[ix.at(i, k)] = v;
            }
        // pivot of column 0 (thread 0); later pivots are produced by thread 0,
        // which owns element (j+1, j+1) of step j's trailing update
        if (threadIdx.x == 0) {
            const double x = w[ix.at(0, 0)];
            piv_sh[0] = x;
            piv_sh[1] = sqrt(x);
            piv_sh[2] = 1.0 / piv_sh[1];
        }
        __syncthreads();
        bool failed = false;
        double inv_prev = 0.0;
        for (int j = 0; j < R; ++j) {
            const double x = piv_sh[0], l = piv_sh[1], inv = piv_sh[2];
            if (!(x > 0.0) && !isnan(x)) {  // Eigen LLT: fail iff pivot <= 0 (uniform branch)
                failed = true;
                break;
            }
            const double inv2 = inv * inv;
            // scale column j-1 (no later step reads it)
            if (j > 0)
                for (int i = j + threadIdx.x; i < R; i += blockDim.x) w[ix.at(i, j - 1)] *= inv_prev;
            // trailing update with the unscaled column j: a_ik -= a_ij a_kj / pivot
            for (int i = j + 1 + ty; i < R; i += ny) {
                const double aij = w[ix.at(i, j)] * inv2;
                for (int k = j + 1 + tx; k <= i; k += 32) w[ix.at(i, k)] -= aij * w[ix.at(k, j)];
            }
            __syncthreads();  // (j+1, j+1) is final; pivot slots are free to overwrite
            if (threadIdx.x == 0) {
                w[ix.at(j, j)] = l;
                w[ix.inv(j)] = inv;
                if (j + 1 < R) {
                    const double xn = w[ix.at(j + 1, j + 1)];
                    piv_sh[0] = xn;
                    piv_sh[1] = sqrt(xn);
                    piv_sh[2] = 1.0 / piv_sh[1];
                }
            }
            __syncthreads();
            inv_prev = inv;
        }
        __syncthreads();
        if (!failed) {
            st = attempt;  // 0 ok, 1 ok after jitter
            break;
        }
    }
    if (kSmem)
        for (int i = ty; i < R; i += ny) {
            for (int k = tx; k <= i; k += 32) out[i * LD + k] = w[ix.at(i, k)];
            if (tx == 0) out[i * LD + R] = w[ix.inv(i)];
        }
    if (threadIdx.x == 0) status[mat] = st;
}

// Blocked right-looking Cholesky for the square shared-memory layout: per
// block of kNB columns, warp 0 factors the diagonal block warp-synchronously
// (lane = row, no CTA barrier per column), then the CTA solves the panel below
// it (one thread per row) and applies the symmetric rank-kNB update to the
// trailing matrix (3 CTA barriers per block instead of 2 per column). Pivot
// test, jitter retry and output layout are those of chol_kernel.
// Warp-synchronous factorisation of the kb x kb diagonal block at (k0, k0)
// (kb <= kNB <= 32): lane i holds row i in registers. No early exit, so the
// row stays in registers. Returns true (all lanes) on a non-positive pivot.
// 1/sqrt(x) for a positive normal x without the libdevice special-case call
// (whose divergent branch forces every later warp shuffle onto the slow
// collective path): MUFU seed, then two cubic Newton steps (>= 60 bits).
__device__ __forceinline__ double rsqrt_pos(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    // the seed is good to 20 bits on sm_100a (tools/probe/rsqrt_prec.cu): one
    // cubic step lands within ~1.2 ulp, the same as two
    const double e = __fma_rn(-x * y, y, 1.0);
    return __fma_rn(y * e, __fma_rn(0.375, e, 0.5), y);
}

template <int kNB, class Idx>
__device__ __noinline__ bool diag_factor(double* w, const Idx ix, int k0, int kb) {
    static_assert(kNB % 2 == 0 && kNB <= 32, "diagonal block: even width, one warp");
    __shared__ __align__(16) double colb[32];  // column j of L, broadcast to the warp
    __syncwarp();
    const int i = threadIdx.x & 31;
    double r[kNB];
#pragma unroll
    for (int m = 0; m < kNB; ++m) r[m] = (i < kb && m <= i) ? w[ix.at(k0 + i, k0 + m)] : 0.0;
    bool failed = false;
    // The pivot of the next column is computed by its own lane from its own row
    // (the same fma as the row update, so bitwise the same value) and shuffled
    // right away, so the column-to-column chain is shuffle -> rsqrt -> scale ->
    // fma -> shuffle with the rank-1 update off it. The update reads column j
    // from shared memory (one warp-wide store, vector loads) and runs
    // unpredicated: entries above the diagonal, rows >= kb and every update
    // after a failed pivot are never stored or read as results.
    double x = __shfl_sync(0xffffffffu, r[0], 0);
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
        if (CPKIT_CHOL_TRACE && k0 == 0 && blockIdx.x == 0 && i == 0) g_chol_trace[24 + j] = clock64();
        if (j < kb && !failed && !(x > 0.0) && !isnan(x)) failed = true;  // Eigen LLT: fail iff pivot <= 0
        const double inv = rsqrt_pos(x > 0.0 ? x : 1.0), l = x * inv;  // L_jj = x / sqrt(x)
        const double lij = i > j ? r[j] * inv : (i == j ? l : r[j]);
        if (j + 1 < kNB) x = __shfl_sync(0xffffffffu, __fma_rn(-lij, lij, r[j + 1]), j + 1);
        if (i == j && j < kb && !failed) w[ix.inv(k0 + j)] = inv;
        r[j] = lij;
        if (j + 1 < kNB) {
            colb[i] = lij;
            __syncwarp();
#pragma unroll
            for (int m = (j + 1) & ~1; m < kNB; m += 2) {
                const double2 c = *reinterpret_cast<const double2*>(colb + m);
                if (m > j) r[m] = __fma_rn(-lij, c.x, r[m]);
                if (m + 1 > j) r[m + 1] = __fma_rn(-lij, c.y, r[m + 1]);
            }
            __syncwarp();
        }
    }
    if (CPKIT_CHOL_TRACE && k0 == 0 && blockIdx.x == 0 && i == 0) g_chol_trace[24 + kNB] = clock64();
#pragma unroll
    for (int m = 0; m < kNB; ++m)
        if (i < kb && m <= i) w[ix.at(k0 + i, k0 + m)] = r[m];
    return failed;
}

// Input of one factorisation: an explicit R x R matrix s, or (grams != null)
// Gamma^(excl) = Ones o S^(m) for ascending m != excl formed on load from the
// Gram matrices, the same products in the same order as gamma_excl_kernel
// (als.cpp:34-37 / kruskal.cpp:42-65), so no separate Gamma pass.
struct CholSrc {
    const double* s;
    const double* grams;
    int order, excl;
    long long s_stride;  // elements between consecutive input matrices
};
__device__ __forceinline__ double chol_src_at(const CholSrc& src, const double* s, long long rr, int e) {
    if (!src.grams) return __ldg(s + e);
    double g = 1.0;
    for (int m = 0; m < src.order; ++m)
        if (m != src.excl) g *= __ldg(src.grams + m * rr + e);
    return g;
}

// Idx = SqIdx: the square R x (R+1) layout in shared memory (R <= ~165), the
// factor leaves in one bulk copy; Idx = PkIdx: the packed lower triangle (R up
// to ~233), rows contiguous, so the panel and DMMA trailing update address it
// the same way; the factor leaves row by row into the square global layout.
template <int kNB, class Idx>
__global__ void __launch_bounds__(256) chol_blocked_kernel(const CholSrc src, int R, double lambda,
                                                           int mode, double* __restrict__ l_all,
                                                           int* __restrict__ status) {
    extern __shared__ __align__(16) double w[];
    const int LD = R + 1;
    const Idx ix{LD, R};
    const int mat = blockIdx.x;
    const long long rr = static_cast<long long>(R) * R;
    const double* s = src.s + static_cast<long long>(mat) * src.s_stride;
    double* out = l_all + static_cast<long long>(mat) * R * LD;
    __shared__ double trace_sh;
    __shared__ int fail_sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

    chol_stamp(0);
    int st = 2;
    for (int attempt = 0; attempt < 2; ++attempt) {
        double jitter = 0.0;
        if (attempt == 1) {  // the trace only matters for the retry (warp-parallel, fixed shuffle order)
            if (warp == 0) {
                double tr = 0.0;
                for (int i = lane; i < R; i += 32) {
                    const double d = chol_src_at(src, s, rr, i * R + i);
                    tr += (mode == 1) ? d * (1.0 + lambda) : d;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tr += __shfl_down_sync(0xffffffffu, tr, o);
                if (lane == 0) trace_sh = tr;
            }
            __syncthreads();
            jitter = 1e-12 * trace_sh / static_cast<double>(R);
        }
        const double add = (mode == 0 ? lambda : 0.0);
        {
            // lower triangle straight into shared memory (async 8-byte copies, all
            // in flight); for Gamma the first Gram factor, the others multiplied in
            // after, in ascending mode order (bitwise gamma_excl's 1 * S_a * S_b ...)
            int first = -1;
            if (src.grams)
                for (int m = 0; m < src.order && first < 0; ++m)
                    if (m != src.excl) first = m;
            const double* s0 = src.grams ? (first >= 0 ? src.grams + first * rr : nullptr) : s;
            if (s0) {
                for (int i = warp; i < R; i += nw)
                    for (int k = lane; k <= i; k += 32) tile::cp_async8(w + ix.at(i, k), s0 + i * R + k);
            } else {  // order 1 (no other mode): Gamma = Ones
                for (int i = warp; i < R; i += nw)
                    for (int k = lane; k <= i; k += 32) w[ix.at(i, k)] = 1.0;
            }
            tile::cp_async_wait_all();
            __syncthreads();
            if (src.grams && first >= 0) {
                for (int m = first + 1; m < src.order; ++m) {
                    if (m == src.excl) continue;
                    const double* sm = src.grams + m * rr;
                    // four rows per warp per round: 16 loads in flight per lane
                    for (int i0 = warp; i0 < R; i0 += 4 * nw) {
                        double f[4][4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int i = i0 + q * nw;
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const int k = lane + 32 * c;
                                f[q][c] = (i < R && k <= i) ? __ldg(sm + i * R + k) : 1.0;
                            }
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int i = i0 + q * nw;
                            if (i >= R) break;
#pragma unroll
                            for (int c = 0; c < 4; ++c)
                                if (lane + 32 * c <= i) w[ix.at(i, lane + 32 * c)] *= f[q][c];
                            for (int k = lane + 128; k <= i; k += 32) w[ix.at(i, k)] *= __ldg(sm + i * R + k);
                        }
                    }
                }
                __syncthreads();
            }
            for (int i = tid; i < R; i += blockDim.x) {  // the diagonal: shape, lambda, jitter
                double x = w[ix.at(i, i)];
                if (mode == 1) x *= (1.0 + lambda);
                x += add;
                if (attempt == 1) x += jitter;
                w[ix.at(i, i)] = x;
            }
        }
        if (tid == 0) fail_sh = 0;
        __syncthreads();
        chol_stamp(1);
        for (int k0 = 0; k0 < R; k0 += kNB) {
            const int kb = min(kNB, R - k0);
            // 1. diagonal block (warp 0): lane i holds row i in registers; per column
            //    the pivot and every L_mj travel by shuffle (no shared-memory round trips)
            if (!(kCholAblate & 1) && warp == 0 && diag_factor<kNB>(w, ix, k0, kb)) fail_sh = 1;
            __syncthreads();
            chol_stamp(2 + 3 * (k0 / kNB));
            if (fail_sh) break;
            // 2. panel: L[i][k0+j] = (A[i][k0+j] - sum_{m<j} L[i][k0+m] L[k0+j][k0+m]) / L_jj,
            //    one thread per row, the row in registers, two partial sums per dot
            for (int i = k0 + kb + tid; i < R && !(kCholAblate & 2); i += blockDim.x) {
                double* row = w + ix.at(i, k0);
                double x[kNB];
#pragma unroll
                for (int m = 0; m < kNB; ++m) x[m] = (m < kb) ? row[m] : 0.0;
#pragma unroll
                for (int j = 0; j < kNB; ++j) {
                    if (j < kb) {
                        const double* lj = w + ix.at(k0 + j, k0);
                        double s0 = 0.0, s1 = 0.0;
#pragma unroll
                        for (int m = 0; m + 1 < j; m += 2) {
                            s0 += x[m] * lj[m];
                            s1 += x[m + 1] * lj[m + 1];
                        }
                        if (j & 1) s0 += x[j - 1] * lj[j - 1];
                        x[j] = (x[j] - (s0 + s1)) * w[ix.inv(k0 + j)];
                    }
                }
#pragma unroll
                for (int m = 0; m < kNB; ++m)
                    if (m < kb) row[m] = x[m];
            }
            __syncthreads();
            chol_stamp(3 + 3 * (k0 / kNB));
            // 3. trailing update: A[i][m] -= sum_j L[i][k0+j] L[m][k0+j], k0+kb <= m <= i.
            //    Full 16-column blocks: one DMMA m16n8k16 per 16x8 tile on or below the
            //    diagonal (rows and columns past R read zero-padded... masked); tail block scalar.
            {
                const int t0 = k0 + kb, n = R - t0;
                if (kCholAblate & 4) {
                } else if (kb == 16 && kNB == 16 && n > 0) {
                    const int g = lane >> 2, t = lane & 3;
                    const int mt = (n + 15) / 16, nt = (n + 7) / 8;
                    for (int tile = warp; tile < mt * nt; tile += nw) {
                        const int bi = tile / nt, bj = tile - bi * nt;
                        const int r0 = t0 + 16 * bi, c0 = t0 + 8 * bj;
                        if (c0 > r0 + 15) continue;  // strictly above the diagonal
                        double a[8], b[4], acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const int row = r0 + g + 8 * (q & 1), col = t + 4 * (q >> 1);
                            a[q] = row < R ? w[ix.at(row, k0 + col)] : 0.0;
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int nn = c0 + g, kk = t + 4 * q;
                            b[q] = nn < R ? w[ix.at(nn, k0 + kk)] : 0.0;
                        }
                        asm volatile(
                            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},"
                            "{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};"
                            : "+d"(acc[0]), "+d"(acc[1]), "+d"(acc[2]), "+d"(acc[3])
                            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                              "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
#pragma unroll
                        for (int h = 0; h < 2; ++h)
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                const int row = r0 + g + 8 * h, col = c0 + 2 * t + c;
                                if (row < R && col <= row) w[ix.at(row, col)] -= acc[2 * h + c];
                            }
                    }
                } else {
                    for (int i = t0 + warp; i < R; i += nw) {
                        const double* li = w + ix.at(i, k0);
                        for (int m = t0 + lane; m <= i; m += 32) {
                            const double* lm = w + ix.at(m, k0);
                            double acc = w[ix.at(i, m)];
                            for (int j = 0; j < kb; ++j) acc -= li[j] * lm[j];
                            w[ix.at(i, m)] = acc;
                        }
                    }
                }
            }
            __syncthreads();
            chol_stamp(4 + 3 * (k0 / kNB));
        }
        if (!fail_sh) {
            st = attempt;  // 0 ok, 1 ok after jitter
            break;
        }
        __syncthreads();
    }
    __syncthreads();
    if (!std::is_same<Idx, SqIdx>::value) {
        // packed: row i's lower triangle and 1 / L_ii into the square layout
        for (int i = warp; i < R; i += nw) {
            for (int k = lane; k <= i; k += 32) out[i * LD + k] = w[ix.at(i, k)];
            if (lane == 0) out[i * LD + R] = w[ix.inv(i)];
        }
        if (tid == 0) status[mat] = st;
        chol_stamp(63);
        return;
    }
    // the factor (same R x (R+1) layout as in shared memory) in one bulk copy
    if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out),
                     "r"(static_cast<unsigned>(__cvta_generic_to_shared(w))),
                     "r"(static_cast<unsigned>(R * LD * sizeof(double)))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        status[mat] = st;
    }
    __syncthreads();
    chol_stamp(63);
}

// One warp per rhs row: solve (L L^T) y = b. L lower, row stride LD (global),
// staged into shared memory with layout Idx; 1 / L_ii at ix.inv(i). NB =
// number of 32-entry blocks of the rhs (R <= 32 NB).
constexpr int kSolveWarps = 8;
template <int NB, class Idx, bool kSmem>
__global__ void __launch_bounds__(32 * kSolveWarps)
chol_solve_rows_kernel(const double* __restrict__ l_all, int R, const double* __restrict__ b, long long rows,
                       double* y, long long l_stride, long long rows_per_mat, const double* old,
                       double* __restrict__ row_sq) {
    extern __shared__ __align__(16) double lsh[];
    const int LD = R + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long mat = blockIdx.y;
    const double* Lg = l_all + mat * l_stride;
    const Idx ix{LD, R};
    if (kSmem && std::is_same<Idx, SqIdx>::value) {
        // square layout = the global layout: one bulk (TMA) copy of the whole factor
        __shared__ __align__(8) unsigned long long bar;
        const unsigned bytes = static_cast<unsigned>(R * LD * sizeof(double));
        const unsigned sbar = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    static_cast<unsigned>(__cvta_generic_to_shared(lsh))),
                "l"(Lg), "r"(bytes), "r"(sbar)
                : "memory");
        }
        __syncthreads();
        for (;;) {
            unsigned ok;
            asm volatile(
                "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                : "=r"(ok)
                : "r"(sbar)
                : "memory");
            if (ok) break;
        }
    } else if (kSmem) {
        // packed: one warp per row, 8-byte async copies of its lower part and 1 / L_ii
        // (no index division; rows of the square global layout start at odd offsets)
        for (int i = warp; i < R; i += kSolveWarps) {
            const double* src = Lg + static_cast<long long>(i) * LD;
            double* dst = lsh + ix.at(i, 0);
            for (int k = lane; k <= i; k += 32) tile::cp_async8(dst + k, src + k);
            if (lane == 0) tile::cp_async8(lsh + ix.inv(i), src + R);
        }
        tile::cp_async_wait_all();
        __syncthreads();
    }
    auto Lat = [&](int i, int k) -> double { return kSmem ? lsh[ix.at(i, k)] : Lg[i * LD + k]; };
    auto Linv = [&](int i) -> double { return kSmem ? lsh[ix.inv(i)] : Lg[i * LD + R]; };
    for (long long local = blockIdx.x * kSolveWarps + warp; local < rows_per_mat;
         local += static_cast<long long>(gridDim.x) * kSolveWarps) {
        const long long row = mat * rows_per_mat + local;
        if (row >= rows) break;
        double v[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) {
            const int k = lane + 32 * c;
            v[c] = (k < R) ? b[row * R + k] : 0.0;
        }
        // forward: z_i = v_i / L_ii ; v_k -= L_ki z_i (k > i)
#pragma unroll
        for (int cb = 0; cb < NB; ++cb) {
            const int iend = min(32, R - 32 * cb);
#pragma unroll 4
            for (int il = 0; il < iend; ++il) {
                const int i = 32 * cb + il;
                const double zi = __shfl_sync(0xffffffffu, v[cb], il) * Linv(i);
                if (lane == il) v[cb] = zi;
                if (lane > il && lane + 32 * cb < R) v[cb] -= Lat(lane + 32 * cb, i) * zi;
#pragma unroll
                for (int c = cb + 1; c < NB; ++c) {
                    const int k = lane + 32 * c;
                    if (k < R) v[c] -= Lat(k, i) * zi;
                }
            }
        }
        // backward with L^T: y_i = v_i / L_ii ; v_k -= L_ik y_i (k < i)
#pragma unroll
        for (int cb = NB - 1; cb >= 0; --cb) {
            const int iend = min(32, R - 32 * cb);
#pragma unroll 4
            for (int il = iend - 1; il >= 0; --il) {
                const int i = 32 * cb + il;
                const double yi = __shfl_sync(0xffffffffu, v[cb], il) * Linv(i);
                if (lane == il) v[cb] = yi;
                if (lane < il) v[cb] -= Lat(i, lane + 32 * cb) * yi;
#pragma unroll
                for (int c = 0; c < cb; ++c) v[c] -= Lat(i, lane + 32 * c) * yi;
            }
        }
        if (old) {  // ALS step norm: this row's ||y - old||^2 (old may alias y: read first)
            double sq = 0.0;
#pragma unroll
            for (int c = 0; c < NB; ++c) {
                const int k = lane + 32 * c;
                if (k < R) {
                    const double d = v[c] - old[row * R + k];
                    sq += d * d;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
            if (lane == 0) row_sq[row] = sq;
            __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < NB; ++c) {
            const int k = lane + 32 * c;
            if (k < R) y[row * R + k] = v[c];
        }
    }
}

template <int NB>
void solve_rows_nb(const double* l, int R, const double* b, long long rows, double* y, long long l_stride, int nmats,
                   long long rows_per_mat, cudaStream_t st, const double* old = nullptr, double* row_sq = nullptr) {
    const int sms = device_sm_count();
    const long long per_mat_ctas = std::max<long long>(
        1, std::min<long long>((rows_per_mat + kSolveWarps - 1) / kSolveWarps, std::max(1, 2 * sms / nmats)));
    const dim3 grid(static_cast<unsigned>(per_mat_ctas), nmats);
    const Layout lay = layout_of(R);
    if (lay == kSquareSmem) {
        auto fn = chol_solve_rows_kernel<NB, SqIdx, true>;
        ensure_dynamic_smem(fn, sq_bytes(R));
        fn<<<grid, 32 * kSolveWarps, sq_bytes(R), st>>>(l, R, b, rows, y, l_stride, rows_per_mat, old, row_sq);
    } else if (lay == kPackedSmem) {
        auto fn = chol_solve_rows_kernel<NB, PkIdx, true>;
        ensure_dynamic_smem(fn, pk_bytes(R));
        fn<<<grid, 32 * kSolveWarps, pk_bytes(R), st>>>(l, R, b, rows, y, l_stride, rows_per_mat, old, row_sq);
    } else {
        chol_solve_rows_kernel<NB, SqIdx, false><<<grid, 32 * kSolveWarps, 0, st>>>(l, R, b, rows, y, l_stride,
                                                                                    rows_per_mat, old, row_sq);
    }
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void solve_rows(const double* l, int R, const double* b, long long rows, double* y, long long l_stride, int nmats,
                long long rows_per_mat, cudaStream_t st, const double* old = nullptr, double* row_sq = nullptr) {
    switch ((R + 31) / 32) {
        case 1: solve_rows_nb<1>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        case 2: solve_rows_nb<2>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        case 3: solve_rows_nb<3>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        case 4: solve_rows_nb<4>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        case 5: solve_rows_nb<5>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        case 6: solve_rows_nb<6>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        case 7: solve_rows_nb<7>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        case 8: solve_rows_nb<8>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
        default: solve_rows_nb<16>(l, R, b, rows, y, l_stride, nmats, rows_per_mat, st, old, row_sq); break;
    }
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

void print_chol_trace() {  // timing experiments only (CPKIT_CHOL_TRACE builds)
    unsigned long long h[64];
    CPK_CUDA(cudaDeviceSynchronize());
    CPK_CUDA(cudaMemcpyFromSymbol(h, g_chol_trace, sizeof h));
    std::fprintf(stderr, "chol: load %.2f us |", (h[1] - h[0]) * 1e-3);
    unsigned long long prev = h[1];
    for (int b = 0; b < 20 && h[4 + 3 * b]; ++b) {
        std::fprintf(stderr, " [%d] diag %.2f panel %.2f trail %.2f", b, (h[2 + 3 * b] - prev) * 1e-3,
                     (h[3 + 3 * b] - h[2 + 3 * b]) * 1e-3, (h[4 + 3 * b] - h[3 + 3 * b]) * 1e-3);
        prev = h[4 + 3 * b];
    }
    std::fprintf(stderr, " | out %.2f | total %.2f us\n", (h[63] - prev) * 1e-3, (h[63] - h[0]) * 1e-3);
    std::fprintf(stderr, "chol diag block 0 cycles per column:");
    for (int j = 0; j < 16; ++j) std::fprintf(stderr, " %llu", h[25 + j] - h[24 + j]);
    std::fprintf(stderr, "\n");
}
void launch_chol_batch(const double* s, int count, int R, const double* lambda, int mode, double* l_out, int* status,
                       cudaStream_t st) {
    launch_chol_batch_src(const_cast<double*>(s), nullptr, 0, -1, count, R, lambda, mode, l_out, status, st);
}
// count matrices read in place s_stride elements apart (e.g. the diagonal
// blocks Gamma(n,n) of the pair array)
void launch_chol_batch_strided(const double* s, long long s_stride, int count, int R, const double* lambda, int mode,
                               double* l_out, int* status, cudaStream_t st) {
    launch_chol_batch_src(const_cast<double*>(s), nullptr, 0, -1, count, R, lambda, mode, l_out, status, st,
                          s_stride);
}
// grams != null: factor Gamma^(excl) formed from the Gram matrices on load when
// the blocked kernel serves R (count 1); otherwise Gamma is formed into `s`
// first (s must then be an R x R workspace).
void launch_chol_batch_src(double* s, const double* grams, int order, int excl, int count, int R,
                           const double* lambda, int mode, double* l_out, int* status, cudaStream_t st,
                           long long s_stride) {
    if (R > 512) throw LimitExceeded("rank exceeds the device SPD solver limit (512)");
    if (s_stride <= 0) s_stride = static_cast<long long>(R) * R;
    const Layout lay = layout_of(R);
    const bool blocked = (lay == kSquareSmem || lay == kPackedSmem) && !std::getenv("CPKIT_CHOL_UNBLOCKED");
    if (grams && !blocked) {
        launch_gamma_excl(grams, order, R, excl, s, st);
        grams = nullptr;
    }
    if (blocked && lay == kSquareSmem) {
        auto fn = chol_blocked_kernel<16, SqIdx>;
        ensure_dynamic_smem(fn, sq_bytes(R));
        fn<<<count, 256, sq_bytes(R), st>>>(CholSrc{s, grams, order, excl, s_stride}, R, *lambda, mode, l_out, status);
    } else if (blocked) {
        auto fn = chol_blocked_kernel<16, PkIdx>;
        ensure_dynamic_smem(fn, pk_bytes(R));
        fn<<<count, 256, pk_bytes(R), st>>>(CholSrc{s, grams, order, excl, s_stride}, R, *lambda, mode, l_out, status);
    } else if (lay == kSquareSmem) {
        auto fn = chol_kernel<SqIdx, true>;
        ensure_dynamic_smem(fn, sq_bytes(R));
        fn<<<count, 512, sq_bytes(R), st>>>(s, R, *lambda, mode, l_out, status, s_stride);
    } else if (lay == kPackedSmem) {
        auto fn = chol_kernel<PkIdx, true>;
        ensure_dynamic_smem(fn, pk_bytes(R));
        fn<<<count, 512, pk_bytes(R), st>>>(s, R, *lambda, mode, l_out, status, s_stride);
    } else {
        chol_kernel<SqIdx, false><<<count, 512, 0, st>>>(s, R, *lambda, mode, l_out, status, s_stride);
    }
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
    if (CPKIT_CHOL_TRACE) print_chol_trace();
}

void launch_chol_solve_rows(const double* l, int R, const double* b, std::int64_t rows, double* y, cudaStream_t st) {
    solve_rows(l, R, b, rows, y, 0, 1, rows, st);
}
void launch_chol_solve_rows_update(const double* l, int R, const double* b, std::int64_t rows, double* a,
                                   double* row_sq, cudaStream_t st) {
    solve_rows(l, R, b, rows, a, 0, 1, rows, st, a, row_sq);
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
