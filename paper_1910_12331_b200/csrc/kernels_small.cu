// Bandwidth/latency-bound kernels of the GN/ALS path (sm_100a, fp64).
// All reductions are two-pass with a fixed grid and a fixed combine order,
// so every result is bitwise reproducible run to run.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.h"
#include "keyed_noise.cuh"
#include "tile_gemm.cuh"

namespace cpkit {

namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocksMax = 592;  // 4 x 148 SMs

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
// Block sum in a fixed order; result valid in thread 0.
__device__ double block_sum(double v) {
    __shared__ double sh[32];
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    double r = 0.0;
    if (w == 0) {
        r = l < nw ? sh[l] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// ---- ||X||^2 (tensor.cpp:61-67), HBM-streaming with 16-byte loads
__global__ void norm2_partial_kernel(const double* __restrict__ x, unsigned long long n,
                                     double* __restrict__ partials) {
    double acc = 0.0;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    const unsigned long long n2 = n / 2;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         i < n2; i += stride) {
        const double2 v = __ldcs(x2 + i);
        acc += v.x * v.x;
        acc += v.y * v.y;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) acc += x[n - 1] * x[n - 1];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void sum_partials_kernel(const double* __restrict__ partials, int n, double* out,
                                    double scale) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) *out = s * scale;
}

// ---- Gram S = A^T A with exact symmetry (matrix_ops.cpp:30-34).
// DMMA 32x32 tiles of the upper triangle, split over row chunks; the
// finalize pass sums the chunks in order and mirrors r <= z, so S is
// bitwise symmetric and deterministic.
constexpr int kGramChunk = 64;
__global__ void __launch_bounds__(tile::kThreads)
gram_tiles_kernel(const double* __restrict__ base, const long long* __restrict__ offs,
                  const long long* __restrict__ rows, int lo, int nmodes, int R, int nsplit,
                  double* __restrict__ partial, const double* __restrict__ sq, int nsq, double* sq_acc,
                  double* __restrict__ direct) {
    __shared__ tile::Smem sm;
    if (sq && blockIdx.x == 0) {  // the ALS step norm: *sq_acc += sqrt(sum of the row partials)
        double v = 0.0;
        for (int i = threadIdx.x; i < nsq; i += blockDim.x) v += sq[i];
        const double s = block_sum(v);
        if (threadIdx.x == 0) *sq_acc += sqrt(s);
    }
    const int tr = (R + tile::kT - 1) / tile::kT;
    const int tri = tr * (tr + 1) / 2;
    const int tasks = nmodes * tri * nsplit;
    for (int task = blockIdx.x; task < tasks; task += gridDim.x) {
        int rem = task;
        const int sp = rem % nsplit; rem /= nsplit;
        int tt = rem % tri; rem /= tri;
        const int n = lo + rem;
        int rt = 0;
        while (tt >= tr - rt) { tt -= tr - rt; ++rt; }
        const int zt = rt + tt;
        const double* a = base + offs[n];
        const long long s = rows[n];
        const long long per = (s + nsplit - 1) / nsplit;
        const long long i0 = sp * per, i1 = min(s, i0 + per);
        const int K = static_cast<int>(max(0LL, i1 - i0));
        const int r0 = rt * tile::kT, z0 = zt * tile::kT;
        auto la = [&](int row, int k) -> double {
            const int r = r0 + row;
            return r < R ? a[(i0 + k) * R + r] : 0.0;
        };
        auto lb = [&](int k, int col) -> double {
            const int z = z0 + col;
            return z < R ? a[(i0 + k) * R + z] : 0.0;
        };
        double acc[4];
        tile::tile_gemm(sm, K, la, lb, acc);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int g = lane >> 2, t = lane & 3;
        if (direct) {  // one split: the final symmetric Gram, mirrored bitwise
            double* out = direct + static_cast<long long>(n) * R * R;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int r = r0 + (warp >> 2) * 16 + g + 8 * h;
                    const int z = z0 + (warp & 3) * 8 + 2 * t + c;
                    if (r < R && z < R && r <= z) {
                        out[r * R + z] = acc[2 * h + c];
                        out[z * R + r] = acc[2 * h + c];
                    }
                }
            continue;
        }
        double* out = partial + (static_cast<long long>(n - lo) * nsplit + sp) * R * R;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int r = r0 + (warp >> 2) * 16 + g + 8 * h;
                const int z = z0 + (warp & 3) * 8 + 2 * t + c;
                if (r < R && z < R && r <= z) out[r * R + z] = acc[2 * h + c];
            }
    }
}
// One thread-block cluster per 32x32 upper-triangle tile of a Gram, one CTA
// per row split: each CTA leaves its partial tile in shared memory and the
// cluster sums the partials through distributed shared memory in split order
// (bitwise the finalize pass's ((0 + p0) + p1) + ...), writing the tile and its
// mirror. No partial workspace round trip and no finalize launch.
__global__ void __launch_bounds__(tile::kThreads)
gram_cluster_kernel(const double* __restrict__ base, const long long* __restrict__ offs,
                    const long long* __restrict__ rows, int lo, int R, int nsplit, double* __restrict__ grams,
                    const double* __restrict__ sq, int nsq, double* sq_acc) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ tile::Smem sm;
    __shared__ double part[tile::kT * tile::kT];
    if (sq && blockIdx.x == 0) {  // the ALS step norm: *sq_acc += sqrt(sum of the row partials)
        double v = 0.0;
        for (int i = threadIdx.x; i < nsq; i += blockDim.x) v += sq[i];
        const double s = block_sum(v);
        if (threadIdx.x == 0) *sq_acc += sqrt(s);
    }
    const int tr = (R + tile::kT - 1) / tile::kT;
    const int tri = tr * (tr + 1) / 2;
    int rem = blockIdx.x;
    const int sp = rem % nsplit; rem /= nsplit;  // == this CTA's rank in its cluster
    int tt = rem % tri; rem /= tri;
    const int n = lo + rem;
    int rt = 0;
    while (tt >= tr - rt) { tt -= tr - rt; ++rt; }
    const int zt = rt + tt;
    const double* a = base + offs[n];
    const long long s = rows[n];
    const long long per = (s + nsplit - 1) / nsplit;
    const long long i0 = sp * per, i1 = min(s, i0 + per);
    const int K = static_cast<int>(max(0LL, i1 - i0));
    const int r0 = rt * tile::kT, z0 = zt * tile::kT;
    auto la = [&](int row, int k) -> double {
        const int r = r0 + row;
        return r < R ? a[(i0 + k) * R + r] : 0.0;
    };
    auto lb = [&](int k, int col) -> double {
        const int z = z0 + col;
        return z < R ? a[(i0 + k) * R + z] : 0.0;
    };
    double acc[4];
    tile::tile_gemm(sm, K, la, lb, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c)
            part[((warp >> 2) * 16 + g + 8 * h) * tile::kT + (warp & 3) * 8 + 2 * t + c] = acc[2 * h + c];
    cluster.sync();
    double* out = grams + static_cast<long long>(n) * R * R;
    const int per_cta = (tile::kT * tile::kT + nsplit - 1) / nsplit;
    for (int e = sp * per_cta + threadIdx.x; e < min(tile::kT * tile::kT, (sp + 1) * per_cta); e += blockDim.x) {
        const int r = r0 + e / tile::kT, z = z0 + e % tile::kT;
        if (r >= R || z >= R || r > z) continue;
        double v = 0.0;
        for (int q = 0; q < nsplit; ++q) v += cluster.map_shared_rank(part, q)[e];
        out[r * R + z] = v;
        out[z * R + r] = v;
    }
    cluster.sync();  // partial tiles stay readable until every CTA of the cluster is done
}
__global__ void gram_finalize_kernel(const double* __restrict__ partial, int lo, int nmodes, int R,
                                     int nsplit, double* __restrict__ grams) {
    const long long RR = static_cast<long long>(R) * R;
    const long long total = nmodes * RR;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long n = e / RR, w = e % RR;
        const int r = static_cast<int>(w / R), z = static_cast<int>(w % R);
        const int a = min(r, z), b = max(r, z);
        double acc = 0.0;
        for (int sp = 0; sp < nsplit; ++sp) acc += partial[(n * nsplit + sp) * RR + a * R + b];
        grams[(lo + n) * RR + w] = acc;
    }
}

// Gamma(n,p) = Ones o S^(m) for ascending m not in {n,p}; computed for p >= n
// and mirrored, so bitwise symmetric (kruskal.cpp:42-65).
__global__ void gamma_pairs_kernel(const double* __restrict__ grams, int order, int R,
                                   double* __restrict__ pair) {
    const int n = blockIdx.y / order, p = blockIdx.y % order;
    if (p < n) return;
    const long long rr = static_cast<long long>(R) * R;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < rr;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        double g = 1.0;
        for (int m = 0; m < order; ++m) {
            if (m == n || m == p) continue;
            g *= grams[m * rr + e];
        }
        pair[(n * order + p) * rr + e] = g;
        if (p != n) pair[(p * order + n) * rr + e] = g;
    }
}
__global__ void gamma_excl_kernel(const double* __restrict__ grams, int order, int R, int n,
                                  double* __restrict__ out) {
    const long long rr = static_cast<long long>(R) * R;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < rr;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        double g = 1.0;
        for (int m = 0; m < order; ++m)
            if (m != n) g *= grams[m * rr + e];
        out[e] = g;
    }
}

// Residual (kruskal.cpp:94-118): partial cross term <M, A> per block plus
// the model norm sum_rz prod_m S^(m)_rz; finalised by one block.
__global__ void residual_partial_kernel(const double* __restrict__ m, const double* __restrict__ a,
                                        long long n, const double* __restrict__ grams, int order,
                                        int R, double* __restrict__ partials) {
    // every block sums a grid-stride slice of the cross term <M, A> AND of the
    // model norm sum_rz prod_m S^(m)_rz; partials[2b] / [2b+1]
    const long long rr = static_cast<long long>(R) * R;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    double cross = 0.0, model = 0.0;
#pragma unroll 4
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
        cross += m[i] * a[i];
#pragma unroll 4
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < rr; e += stride) {
        double g = 1.0;
        for (int q = 0; q < order; ++q) g *= grams[q * rr + e];
        model += g;
    }
    const double c = block_sum(cross);
    const double md = block_sum(model);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = c;
        partials[2 * blockIdx.x + 1] = md;
    }
}
__global__ void residual_final_kernel(const double* __restrict__ partials, int nblocks,
                                      const double* __restrict__ xnorm2, double* __restrict__ out) {
    double c = 0.0, md = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
        c += partials[2 * i];
        md += partials[2 * i + 1];
    }
    const double cross = block_sum(c);
    const double model = block_sum(md);
    if (threadIdx.x == 0) {
        const double x2 = *xnorm2;
        double res2 = x2 - 2.0 * cross + model;
        if (res2 < 0.0) res2 = 0.0;
        const double r = sqrt(res2 / x2);
        out[0] = r;
        out[1] = 1.0 - r;
    }
}

// G = A * Gamma - M   (s x R) (R x R), DMMA tiles with the subtraction in the epilogue
// G = A Gamma(n,n) - M (gauss_newton.cpp:81-94) for one 32x32 output tile: the
// A row panel and the Gamma column slice staged with cp.async (one round trip
// per panel of kPB columns), DMMA tiles
__device__ __forceinline__ void gradient_tile(const double* __restrict__ a, const double* __restrict__ gnn,
                                              const double* __restrict__ m, long long rows, int R,
                                              double* __restrict__ g, long long task, double* gsm) {
    using namespace tile;
    const int tr = (R + kT - 1) / kT;
    double* As = gsm;
    double* Bs = gsm + kT * (kPB + 4);
    const long long i0 = (task / tr) * kT;
    const int c0 = static_cast<int>(task % tr) * kT;
    const int vr = static_cast<int>(min(static_cast<long long>(kT), rows - i0)), vc = min(kT, R - c0);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < R; k0 += kPB) {
        const int kp = min(kPB, R - k0), kpad = pad8(kp);
        stage_rows<32>(As, kPB + 4, kT, kpad, kp,
                       [&](int row) { return row < vr ? a + (i0 + row) * R + k0 : nullptr; });
        stage_rows<16>(Bs, kKS, kpad, kT, vc,
                       [&](int k) { return k < kp ? gnn + static_cast<long long>(k0 + k) * R + c0 : nullptr; });
        cp_async_wait_all();
        __syncthreads();
        mma_panel<false>(As, kPB + 4, Bs, kpad, acc);
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gg = lane >> 2, t = lane & 3;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const long long i = i0 + (warp >> 2) * 16 + gg + 8 * h;
            const int col = c0 + (warp & 3) * 8 + 2 * t + c;
            if (i < rows && col < R) g[i * R + col] = acc[2 * h + c] - m[i * R + col];
        }
}
__global__ void __launch_bounds__(tile::kThreads)
gradient_kernel(const double* __restrict__ a, const double* __restrict__ gnn,
                const double* __restrict__ m, long long rows, int R, double* __restrict__ g) {
    extern __shared__ __align__(16) double gsm[];
    const int tr = (R + tile::kT - 1) / tile::kT;
    const long long tasks = ((rows + tile::kT - 1) / tile::kT) * tr;
    for (long long task = blockIdx.x; task < tasks; task += gridDim.x) gradient_tile(a, gnn, m, rows, R, g, task, gsm);
}
// every mode in one launch: tasks of mode n follow those of mode n-1
struct GradDev {
    int order;
    long long off[kMaxOrder + 1];  // stacked block offsets
    long long rows[kMaxOrder];
};
__global__ void __launch_bounds__(tile::kThreads)
gradient_all_kernel(const GradDev gd, const double* __restrict__ a, const double* __restrict__ pair,
                    const double* __restrict__ m, int R, double* __restrict__ g) {
    extern __shared__ __align__(16) double gsm[];
    const int tr = (R + tile::kT - 1) / tile::kT;
    const long long rr = static_cast<long long>(R) * R;
    long long total = 0;
    for (int n = 0; n < gd.order; ++n) total += ((gd.rows[n] + tile::kT - 1) / tile::kT) * tr;
    for (long long task = blockIdx.x; task < total; task += gridDim.x) {
        long long t = task;
        int n = 0;
        for (; n < gd.order; ++n) {
            const long long tn = ((gd.rows[n] + tile::kT - 1) / tile::kT) * tr;
            if (t < tn) break;
            t -= tn;
        }
        gradient_tile(a + gd.off[n], pair + (n * gd.order + n) * rr, m + gd.off[n], gd.rows[n], R, g + gd.off[n], t,
                      gsm);
    }
}

// Sum over blocks of ||block||_F (gauss_newton.cpp:246-250 norm_sum): partial
// sums of squares per (block, chunk); final kernel does sqrt per block in order.
__global__ void block_sq_partial_kernel(const double* __restrict__ x,
                                        const long long* __restrict__ off, int nblocks, int chunks,
                                        double* __restrict__ partials) {
    const int b = blockIdx.x / chunks, c = blockIdx.x % chunks;
    const long long lo = off[b], hi = off[b + 1];
    double acc = 0.0;
    for (long long i = lo + c * static_cast<long long>(blockDim.x) + threadIdx.x; i < hi;
         i += static_cast<long long>(chunks) * blockDim.x)
        acc += x[i] * x[i];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void block_norm_final_kernel(const double* __restrict__ partials, int nblocks, int chunks,
                                        double* out, double scale) {
    if (threadIdx.x != 0) return;
    double total = 0.0;
    for (int b = 0; b < nblocks; ++b) {
        double sq = 0.0;
        for (int c = 0; c < chunks; ++c) sq += partials[b * chunks + c];
        total += scale * sqrt(sq);
    }
    *out = total;
}

__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, double alpha,
                            unsigned long long n) {
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
        y[i] += alpha * x[i];
}
__global__ void diff_sq_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                       unsigned long long n, double* __restrict__ partials) {
    double acc = 0.0;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void sqrt_add_kernel(const double* __restrict__ partials, int n, double* acc) {
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += partials[i];
    const double s = block_sum(v);
    if (threadIdx.x == 0) *acc += sqrt(s);
}
__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                   unsigned long long n, double* __restrict__ partials) {
    double acc = 0.0;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
        acc += a[i] * b[i];
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void axpby_kernel(double* __restrict__ out, const double* __restrict__ a, double alpha,
                             const double* __restrict__ x, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
        out[i] = a[i] + alpha * x[i];
}
__global__ void all_finite_kernel(const double* __restrict__ x, unsigned long long n, int* flag) {
    bool bad = false;
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 0);
}

// ---- generators (kruskal.cpp:67-92 reconstruct; rng.hpp keyed gaussian)
struct KrpDevS {
    int nmodes;
    long long ext[kMaxOrder];
    const double* fac[kMaxOrder];
};
__global__ void reconstruct_kernel(KrpDevS kd, int R, double* __restrict__ out,
                                   unsigned long long offset, unsigned long long n) {
    for (unsigned long long e = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
         e < n; e += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        unsigned long long f = offset + e;
        long long idx[kMaxOrder];
        for (int m = kd.nmodes - 1; m >= 0; --m) {
            idx[m] = static_cast<long long>(f % kd.ext[m]);
            f /= kd.ext[m];
        }
        double acc = 0.0;
        for (int r = 0; r < R; ++r) {
            double prod = 1.0;
            for (int m = 0; m < kd.nmodes; ++m) prod = __dmul_rn(prod, kd.fac[m][idx[m] * R + r]);
            acc = __dadd_rn(acc, prod);
        }
        out[e] = acc;
    }
}
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ unsigned long long derive(unsigned long long h, unsigned long long v) {
    return mix64(h ^ (v * 0xD6E8FEB86659FD93ull + 0xA0761D6478BD642Full));
}
// ---- keyed noise (keyed_noise.cuh): entry (f', j) of a last-mode slab has the
// keyed index of its GLOBAL flat position f' s_last + slab_lo + j.
// Column-block sums of X^2 and E^2: thread (b, j) sums rows [b blk, (b+1) blk)
// of column j sequentially (adjacent threads read adjacent columns).
__global__ void noise_colsq_part_kernel(const double* __restrict__ x, long long rows, long long slab,
                                        long long blk, unsigned long long base, unsigned long long s_last,
                                        unsigned long long slab_lo, double* __restrict__ part) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<long long>(noise::kNoiseBlocks) * slab) return;
    const long long b = t / slab, j = t % slab;
    const long long r0 = b * blk, r1 = min(rows, r0 + blk);
    double ax = 0.0, ae = 0.0;
    for (long long r = r0; r < r1; ++r) {
        const double v = x[r * slab + j];
        ax = __dadd_rn(ax, __dmul_rn(v, v));
        const double g = noise::keyed_gaussian(base, static_cast<unsigned long long>(r) * s_last + slab_lo +
                                                         static_cast<unsigned long long>(j));
        ae = __dadd_rn(ae, __dmul_rn(g, g));
    }
    part[b * slab + j] = ax;
    part[(noise::kNoiseBlocks + b) * slab + j] = ae;
}
// colsq[j] (X) and colsq[slab + j] (E): the block partials of column j in block order
__global__ void noise_colsq_final_kernel(const double* __restrict__ part, long long slab, double* __restrict__ colsq) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= 2 * slab) return;
    const long long which = t / slab, j = t % slab;
    double a = 0.0;
    for (int b = 0; b < noise::kNoiseBlocks; ++b) a = __dadd_rn(a, part[(which * noise::kNoiseBlocks + b) * slab + j]);
    colsq[t] = a;
}
// scale = rel ||X|| / ||E|| from the gathered per-rank [X cols | E cols] blocks, columns in global order
__global__ void noise_scale_kernel(const double* __restrict__ colsq, int world, long long slab, double rel,
                                   double* __restrict__ out) {
    double nx = 0.0, ne = 0.0;
    for (int g = 0; g < world; ++g)
        for (long long j = 0; j < slab; ++j) {
            nx = __dadd_rn(nx, colsq[g * 2 * slab + j]);
            ne = __dadd_rn(ne, colsq[g * 2 * slab + slab + j]);
        }
    out[0] = __ddiv_rn(__dmul_rn(rel, __dsqrt_rn(nx)), __dsqrt_rn(ne));
    out[1] = nx;
    out[2] = ne;
}
__global__ void noise_add_kernel(double* __restrict__ x, unsigned long long n, unsigned long long slab,
                                 unsigned long long s_last, unsigned long long slab_lo, unsigned long long base,
                                 const double* __restrict__ scale) {
    const double s = scale[0];
    for (unsigned long long e = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        const unsigned long long gidx = (e / slab) * s_last + slab_lo + (e % slab);
        x[e] = __dadd_rn(x[e], __dmul_rn(s, noise::keyed_gaussian(base, gidx)));
    }
}

int grid_for(unsigned long long n, int threads, int cap = kRedBlocksMax) {
    const unsigned long long b = (n + threads - 1) / threads;
    return static_cast<int>(std::max<unsigned long long>(1, std::min<unsigned long long>(b, cap)));
}

}  // namespace

int norm2_parts(std::uint64_t n) { return grid_for(std::max<std::uint64_t>(1, n / 2), kRedThreads); }

void launch_norm2(const double* x, std::uint64_t n, double* partials, int nparts, double* out,
                  cudaStream_t st) {
    if (reinterpret_cast<std::uintptr_t>(x) % 16 != 0) throw DeviceError("norm2: misaligned tensor");
    norm2_partial_kernel<<<nparts, kRedThreads, 0, st>>>(x, n, partials); ::cpkit::count_launch(1);
    sum_partials_kernel<<<1, kRedThreads, 0, st>>>(partials, nparts, out, 1.0); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

int gram_splits(std::int64_t smax) {
    if (const char* e = std::getenv("CPKIT_GRAM_SPLITS")) return std::max(1, std::atoi(e));  // experiments
    return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(32, (smax + kGramChunk - 1) / kGramChunk)));
}
std::size_t gram_workspace_elems(int nmodes, int R, std::int64_t smax) {
    return static_cast<std::size_t>(nmodes) * gram_splits(smax) * R * R;
}
void launch_grams(const double* base, const std::int64_t* offs, const std::int64_t* rows, int lo,
                  int hi, int R, std::int64_t smax, double* ws, double* grams, cudaStream_t st, const double* sq,
                  int nsq, double* sq_acc) {
    const int nsplit = gram_splits(smax);
    const int tr = (R + tile::kT - 1) / tile::kT;
    const int tasks = (hi - lo) * tr * (tr + 1) / 2 * nsplit;
    if (nsplit > 1 && nsplit <= 8 && !std::getenv("CPKIT_GRAM_NO_CLUSTER")) {  // portable cluster sizes
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(tasks));
        cfg.blockDim = dim3(tile::kThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(nsplit);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CPK_CUDA(cudaLaunchKernelEx(&cfg, gram_cluster_kernel, base, reinterpret_cast<const long long*>(offs),
                                    reinterpret_cast<const long long*>(rows), lo, R, nsplit, grams, sq, nsq, sq_acc));
        ::cpkit::count_launch(1);
        return;
    }
    gram_tiles_kernel<<<std::min(tasks, 4 * 148), tile::kThreads, 0, st>>>(
        base, reinterpret_cast<const long long*>(offs), reinterpret_cast<const long long*>(rows), lo, hi - lo, R,
        nsplit, ws, sq, nsq, sq_acc, nsplit == 1 ? grams : nullptr);
    ::cpkit::count_launch(1);
    if (nsplit > 1) {
        const long long total = static_cast<long long>(hi - lo) * R * R;
        gram_finalize_kernel<<<grid_for(total, 256, 592), 256, 0, st>>>(ws, lo, hi - lo, R, nsplit, grams);
        ::cpkit::count_launch(1);
    }
    CPK_CUDA(cudaGetLastError());
}

void launch_gamma_pairs(const double* grams, int order, int R, double* pair, cudaStream_t st) {
    const long long rr = static_cast<long long>(R) * R;
    dim3 grid(static_cast<unsigned>(std::max<long long>(1, std::min<long long>((rr + 255) / 256, 64))),
              order * order);
    gamma_pairs_kernel<<<grid, 256, 0, st>>>(grams, order, R, pair); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_gamma_excl(const double* grams, int order, int R, int n, double* out, cudaStream_t st) {
    const long long rr = static_cast<long long>(R) * R;
    gamma_excl_kernel<<<static_cast<int>(std::max<long long>(1, std::min<long long>((rr + 255) / 256, 64))),
                        256, 0, st>>>(grams, order, R, n, out); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_residual(const double* m_last, const double* a_last, std::int64_t rows, const double* grams,
                     int order, int R, const double* xnorm2, double* partials, double* out2,
                     cudaStream_t st) {
    const long long n = rows * static_cast<long long>(R);
    const int nb = grid_for(std::max<long long>(n, static_cast<long long>(R) * R), kRedThreads, 128);
    residual_partial_kernel<<<nb, kRedThreads, 0, st>>>(m_last, a_last, n, grams, order, R, partials); ::cpkit::count_launch(1);
    residual_final_kernel<<<1, kRedThreads, 0, st>>>(partials, nb, xnorm2, out2); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_gradient_all(const double* a, const double* pair, const double* m, const std::int64_t* off,
                         const std::int64_t* rows, int order, int R, double* g, cudaStream_t st) {
    GradDev gd{};
    gd.order = order;
    long long tasks = 0;
    const int tr = (R + tile::kT - 1) / tile::kT;
    for (int n = 0; n < order; ++n) {
        gd.off[n] = off[n];
        gd.rows[n] = rows[n];
        tasks += ((rows[n] + tile::kT - 1) / tile::kT) * tr;
    }
    gd.off[order] = off[order];
    const std::size_t smem = (tile::kT * (tile::kPB + 4) + tile::kPB * tile::kKS) * sizeof(double);
    ensure_dynamic_smem(gradient_all_kernel, smem);
    gradient_all_kernel<<<static_cast<int>(std::min<long long>(tasks, 2 * 148)), tile::kThreads, smem, st>>>(
        gd, a, pair, m, R, g);
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
void launch_gradient(const double* a, const double* gnn, const double* m, std::int64_t rows, int R,
                     double* g, cudaStream_t st) {
    const long long tasks = ((rows + tile::kT - 1) / tile::kT) * ((R + tile::kT - 1) / tile::kT);
    const std::size_t smem = (tile::kT * (tile::kPB + 4) + tile::kPB * tile::kKS) * sizeof(double);
    ensure_dynamic_smem(gradient_kernel, smem);
    gradient_kernel<<<static_cast<int>(std::min<long long>(tasks, 2 * 148)), tile::kThreads, smem, st>>>(
        a, gnn, m, rows, R, g); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_block_norm_sum(const double* x, const std::int64_t* offsets, int nblocks,
                           double* partials, double* out, double scale, cudaStream_t st) {
    const int chunks = 16;
    block_sq_partial_kernel<<<nblocks * chunks, kRedThreads, 0, st>>>(
        x, reinterpret_cast<const long long*>(offsets), nblocks, chunks, partials); ::cpkit::count_launch(1);
    block_norm_final_kernel<<<1, 32, 0, st>>>(partials, nblocks, chunks, out, scale); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_axpy(double* y, const double* x, double alpha, std::uint64_t n, cudaStream_t st) {
    axpy_kernel<<<grid_for(n, 256, 1184), 256, 0, st>>>(y, x, alpha, n); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_diff_norm_add(const double* a, const double* b, std::uint64_t n, double* partials,
                          double* acc, cudaStream_t st) {
    const int nb = grid_for(n, kRedThreads, 128);
    diff_sq_partial_kernel<<<nb, kRedThreads, 0, st>>>(a, b, n, partials); ::cpkit::count_launch(1);
    sqrt_add_kernel<<<1, kRedThreads, 0, st>>>(partials, nb, acc); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_sqrt_add(const double* partials, int n, double* acc, cudaStream_t st) {
    sqrt_add_kernel<<<1, kRedThreads, 0, st>>>(partials, n, acc); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_dot(const double* a, const double* b, std::uint64_t n, double* partials, double* out,
                cudaStream_t st) {
    const int nb = grid_for(n, kRedThreads, 128);
    dot_partial_kernel<<<nb, kRedThreads, 0, st>>>(a, b, n, partials); ::cpkit::count_launch(1);
    sum_partials_kernel<<<1, kRedThreads, 0, st>>>(partials, nb, out, 1.0); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_axpby(double* out, const double* a, double alpha, const double* x, std::uint64_t n,
                  cudaStream_t st) {
    axpby_kernel<<<grid_for(n, 256, 1184), 256, 0, st>>>(out, a, alpha, x, n); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

namespace {
__global__ void set_flag_scalar_kernel(int* flag, int fv, double* d, double dv) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *flag = fv;
        *d = dv;
    }
}
}  // namespace
namespace {
__global__ void pack_sweep_kernel(const double* __restrict__ scal, int kstep, int kres, const int* __restrict__ flag,
                                  const int* __restrict__ status, int n, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[0] = scal[kstep];
        out[1] = scal[kres];
        out[2] = scal[kres + 1];
        out[3] = static_cast<double>(*flag);
        for (int i = 0; i < n; ++i) out[4 + i] = static_cast<double>(status[i]);
    }
}
}  // namespace
namespace {
__global__ void pack_values_kernel(const double* __restrict__ d, int nd, const int* __restrict__ iv, int ni,
                                   double* out) {
    for (int i = threadIdx.x; i < nd + ni; i += blockDim.x)
        out[i] = i < nd ? d[i] : static_cast<double>(iv[i - nd]);
}
}  // namespace
// out[0..nd) = d[0..nd), out[nd..nd+ni) = iv[0..ni) as doubles, into mapped
// pinned host memory (stream-ordered, no copy engine, no synchronisation).
void launch_pack_values(const double* d, int nd, const int* iv, int ni, double* out_mapped, cudaStream_t st) {
    pack_values_kernel<<<1, 32, 0, st>>>(d, nd, iv, ni, out_mapped);
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
// One sweep's diagnostics (step norm, residual, fitness, finiteness flag,
// per-mode SPD status) written straight into mapped pinned host memory:
// no copy-engine operation and no synchronisation on the solver stream.
void launch_pack_sweep(const double* scal, int kstep, int kres, const int* flag, const int* status, int n,
                       double* out_mapped, cudaStream_t st) {
    pack_sweep_kernel<<<1, 32, 0, st>>>(scal, kstep, kres, flag, status, n, out_mapped);
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
// *flag = fv, *d = dv as a device op (capturable in a CUDA graph, unlike a pageable H2D copy)
void launch_set_flag_scalar(int* flag, int fv, double* d, double dv, cudaStream_t st) {
    set_flag_scalar_kernel<<<1, 32, 0, st>>>(flag, fv, d, dv);
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
namespace {
// The GN update in one launch (gauss_newton.cpp:428-441 and the step norm,
// :435): A += V, per-(mode, chunk) partial sums of ||V||^2 (the same chunks
// and block sums as block_sq_partial_kernel, so the step norm is bitwise
// launch_block_norm_sum's), finiteness of the new A; the last block to finish
// sums the partials in fixed order, stores the step norm and the flag, and
// packs the CG result and both values into the mapped diagnostics.
__global__ void gn_apply_kernel(double* __restrict__ a, const double* __restrict__ v,
                                const long long* __restrict__ off, int nblocks, int chunks,
                                double* __restrict__ partials, int* __restrict__ bad_part,
                                unsigned int* __restrict__ counter, const int* __restrict__ cgres, int ncg,
                                double* out_cg, double* step_out, double* step_slot_zero, int* flag,
                                double* out_step) {
    const int b = blockIdx.x / chunks, c = blockIdx.x % chunks;
    const long long lo = off[b], hi = off[b + 1];
    double acc = 0.0;
    bool bad = false;
    for (long long i = lo + c * static_cast<long long>(blockDim.x) + threadIdx.x; i < hi;
         i += static_cast<long long>(chunks) * blockDim.x) {
        const double x = v[i];
        const double y = a[i] + 1.0 * x;
        a[i] = y;
        acc += x * x;
        bad |= !isfinite(y);
    }
    const double sum = block_sum(acc);
    const int anybad = __syncthreads_or(bad);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = sum;
        bad_part[blockIdx.x] = anybad;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    double total = 0.0;
    int fin = 1;
    for (int q = 0; q < nblocks; ++q) {
        double sq = 0.0;
        for (int k = 0; k < chunks; ++k) sq += __ldcg(partials + q * chunks + k);
        total += 1.0 * sqrt(sq);
    }
    for (int q = 0; q < nblocks * chunks; ++q)
        if (__ldcg(bad_part + q)) fin = 0;
    *step_out = total;
    *step_slot_zero = 0.0;
    *flag = fin;
    for (int i = 0; i < ncg; ++i) out_cg[i] = static_cast<double>(cgres[i]);
    out_step[0] = total;
    out_step[1] = static_cast<double>(fin);
    *counter = 0u;  // ready for the next launch (stream order)
}
}  // namespace
void launch_gn_apply(double* a, const double* v, const std::int64_t* offsets, int nblocks, double* partials,
                     int* bad_part, unsigned int* counter, const int* cgres, int ncg, double* out_cg,
                     double* step_out, double* step_slot_zero, int* flag, double* out_step, cudaStream_t st) {
    const int chunks = 16;
    gn_apply_kernel<<<nblocks * chunks, kRedThreads, 0, st>>>(a, v, reinterpret_cast<const long long*>(offsets),
                                                             nblocks, chunks, partials, bad_part, counter, cgres,
                                                             ncg, out_cg, step_out, step_slot_zero, flag, out_step);
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
void launch_all_finite(const double* x, std::uint64_t n, int* flag, cudaStream_t st) {
    all_finite_kernel<<<grid_for(n, 256, 1184), 256, 0, st>>>(x, n, flag); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

void launch_reconstruct(const KrpDesc& all, int R, double* out, std::uint64_t offset, std::uint64_t n,
                        cudaStream_t st) {
    KrpDevS kd{};
    kd.nmodes = all.nmodes;
    for (int i = 0; i < all.nmodes; ++i) {
        kd.ext[i] = all.ext[i];
        kd.fac[i] = all.fac[i];
    }
    reconstruct_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(kd, R, out, offset, n); ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

std::size_t noise_workspace_elems(std::int64_t slab) {
    return static_cast<std::size_t>(2 * noise::kNoiseBlocks + 2) * static_cast<std::size_t>(slab);
}
void launch_noise_colsq(const double* x, std::int64_t rows, std::int64_t slab, std::uint64_t seed,
                        std::uint64_t s_last, std::uint64_t slab_lo, double* ws, double* colsq, cudaStream_t st) {
    const long long blk = (rows + noise::kNoiseBlocks - 1) / noise::kNoiseBlocks;
    const unsigned long long base = noise::nz_derive(noise::nz_mix64(seed), noise::kNoiseStream);
    const long long threads = static_cast<long long>(noise::kNoiseBlocks) * slab;
    noise_colsq_part_kernel<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, st>>>(x, rows, slab, blk, base,
                                                                                          s_last, slab_lo, ws);
    noise_colsq_final_kernel<<<static_cast<unsigned>((2 * slab + 127) / 128), 128, 0, st>>>(ws, slab, colsq);
    ::cpkit::count_launch(2);
    CPK_CUDA(cudaGetLastError());
}
void launch_noise_scale(const double* colsq_all, int world, std::int64_t slab, double rel, double* out3,
                        cudaStream_t st) {
    noise_scale_kernel<<<1, 1, 0, st>>>(colsq_all, world, slab, rel, out3);
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}
void launch_noise_add(double* x, std::uint64_t n, std::uint64_t slab, std::uint64_t s_last, std::uint64_t slab_lo,
                      std::uint64_t seed, const double* scale, cudaStream_t st) {
    const unsigned long long base = noise::nz_derive(noise::nz_mix64(seed), noise::kNoiseStream);
    noise_add_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(x, n, slab, s_last, slab_lo, base, scale);
    ::cpkit::count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

}  // namespace cpkit
