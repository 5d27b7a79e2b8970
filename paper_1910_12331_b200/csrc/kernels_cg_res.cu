// Tile-resident preconditioned CG: the same recurrence as kernels_cg.cu
// (cp_cg, gauss_newton.cpp:279-349; hessian_matvec :96-136) as ONE persistent
// cooperative kernel with one CTA per SM, where each CTA owns one tm x tn
// tile (mode n, rows i0.., columns c0..) of every CG vector for the whole
// solve and keeps it in registers, laid out exactly as its DMMA accumulator
// fragment. Everything constant across iterations that the tile needs sits in
// shared memory from the first iteration on: the factor rows A_n[i0:i0+tm, :],
// and the column slices Gamma(n,n)[:, c0:c0+tn] and Pinv_n[:, c0:c0+tn].
//
// Per iteration (4 grid barriers; only tile exchanges touch L2):
//   A: W' = Z + beta W (registers; first: W' = Z), publish the W' tile, and
//      the tile's contribution A_n[rows,:]^T W'[rows, cols] to B_n = A_n^T W'_n
//      (R x tn partial; dense partial slabs, summed in fixed order in A2)
//   A2: B_p = sum of the partials; D_n^T = sum_{p != n} Gamma(n,p) o B_p
//      (elementwise, spread over every CTA)
//   B: Q = [W'_n | A_n][rows, :] [Gamma_nn ; D_n^T][:, cols] + lambda Reg(W'):
//      the sibling tiles' W' columns and the D_n^T slice come from L2, A_n
//      rows and Gamma_nn from shared memory; Q stays in registers, published
//   C: alpha = rz / <W, Q>; V += alpha W'; R' = R - alpha Q (registers);
//      Z = R'[rows, :] Pinv_n[:, cols] with the sibling columns of R' rebuilt
//      from R_old and Q with the identical fma; partials of <R', Z>, ||R'_n||^2
// Every scalar decision is recomputed by every CTA from the same partial slots
// in the same order (bitwise identical across CTAs; deterministic run to run).
// Used when every tile fits one CTA (tasks <= #SMs) and the resident set fits
// shared memory; kernels_cg.cu's streaming kernel covers the rest.
// Cluster mode (CLU, the default when R needs 2..8 column tiles): the column
// tiles of one row block form a thread-block cluster; W' and R' reach the
// siblings by DSMEM bulk copies (push_own) instead of global stores + L2
// gathers, bitwise the same arithmetic (tests/test_gpu_cg_cluster.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "grid_sync.cuh"
#include "tile_gemm.cuh"

#ifndef CPKIT_CG_ABLATE
#define CPKIT_CG_ABLATE 0  // timing experiments only: 1 A2 work, 2 gathers, 4 GEMMs, 8 slot sums, 16 phase-A publish
                           // 32: no overlap (A2 loads after the loop-top sums, W' Gamma_nn after the barrier; same bits)
#endif

namespace cpkit {
namespace {
constexpr int kAblate = CPKIT_CG_ABLATE;
#ifdef CPKIT_CG_NO_PF
constexpr int kPrefetchWarps = 1 << 30;
#else
// Measured (us per iteration, prefetch on/off): C2 (12 warps) 21.5 / 22.0; C4 (4 warps) 16.5 / 16.3;
// C3 (3 warps) 15.3 / 15.0 - it pays only where the loop-top block sums are long.
constexpr int kPrefetchWarps = 8;
#endif

using gsync::cta_rank;
using gsync::grid_arrive;
using gsync::grid_barrier;
using gsync::grid_wait;
using tile::cp_async16;
using tile::cp_async8;
using tile::cp_async_wait_all;
using tile::dmma1688;
using tile::dmma16816;

struct RLayout {
    int order, R, tm, tn, nct;
    int rowtiles[kMaxOrder];
    int taskoff[kMaxOrder + 1];
    int tasks;
    int ld;  // row stride (doubles) of A_n rows / row buffers: >= pad16(R), = 4 mod 16
    int ks;  // k-major stride: tn + 4
    int rk;  // pad8(R): GEMM depth over R
    int rm;  // pad16(R): rows of the phase-A GEMM
    int o_gnn, o_pinv, o_row, o_aux, o_ds, smem;  // doubles; A_n rows at 0
    long long bp_off[kMaxOrder];                  // partial slabs of mode p (rowtiles[p] x R x R)
    int a2g, a2lg;                                // A2 lane-group size (pow2 >= order) and its log2
    long long dt_off;                             // D_n^T blocks (order x R x R)
    int bs;                                       // CLU: row stride of a column block of Rb (tn + 4)
};

struct RDev {
    CgParams p;
    RLayout L;
};

__device__ __forceinline__ double* r_slot_wq(const RDev& d) { return d.p.slots; }
__device__ __forceinline__ double* r_slot_rz(const RDev& d) { return d.p.slots + d.L.tasks; }
__device__ __forceinline__ double* r_slot_nrm(const RDev& d) { return d.p.slots + 2 * d.L.tasks; }
__device__ __forceinline__ double* r_slot_fin(const RDev& d) { return d.p.slots + 3 * d.L.tasks; }
__device__ __forceinline__ double* r_bpart(const RDev& d, int p) { return d.p.slots + 4 * d.L.tasks + d.L.bp_off[p]; }
__device__ __forceinline__ double* r_dt(const RDev& d) { return d.p.slots + 4 * d.L.tasks + d.L.dt_off; }
// B_p = A_p^T W_p of the current direction, carried across iterations (order x R x R)
__device__ __forceinline__ double* r_bsum(const RDev& d) {
    return r_dt(d) + static_cast<long long>(d.L.order) * d.L.R * d.L.R;
}

// Fixed-order block sum (WARPS warps), result broadcast to every thread.
template <int WARPS>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < WARPS; ++w) t += red[w];
        red[WARPS] = t;
    }
    __syncthreads();
    const double t = red[WARPS];
    __syncthreads();
    return t;
}

// Three fixed-order block sums with one shared-memory exchange.
template <int WARPS>
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[3 * w] = a;
        red[3 * w + 1] = b;
        red[3 * w + 2] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0, z = 0.0;
        for (int i = 0; i < WARPS; ++i) {
            x += red[3 * i];
            y += red[3 * i + 1];
            z += red[3 * i + 2];
        }
        red[3 * WARPS] = x;
        red[3 * WARPS + 1] = y;
        red[3 * WARPS + 2] = z;
    }
    __syncthreads();
    a = red[3 * WARPS];
    b = red[3 * WARPS + 1];
    c = red[3 * WARPS + 2];
    __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;  // lane 0
}

// Loop-top scalars: rz = sum of the <R, Z> partials, nsum = sum_n sqrt(sum of
// the mode-n ||R||^2 partials) (norm_sum, gauss_newton.cpp:246-250), bad = sum
// of the finiteness flags. Items (mode-n norm sums, rz, bad) go to warps
// round-robin; each is a fixed-order strided warp sum, so every CTA computes
// identical bits.
template <int WARPS>
__device__ void top_sums(const RDev& d, double* red, double& rz, double& nsum, double& bad) {
    const int N = d.L.order, lane = threadIdx.x & 31;
    for (int item = threadIdx.x >> 5; item < N + 2; item += WARPS) {
        const double* src;
        int lo, hi;
        if (item < N) {
            src = r_slot_nrm(d);
            lo = d.L.taskoff[item];
            hi = d.L.taskoff[item + 1];
        } else {
            src = item == N ? r_slot_rz(d) : r_slot_fin(d);
            lo = 0;
            hi = d.L.tasks;
        }
        double v = 0.0;
        for (int i = lo + lane; i < hi; i += 32) v += __ldcg(src + i);
        v = warp_sum(v);
        if (lane == 0) red[item] = v;
    }
    __syncthreads();
    double ns = 0.0;
    for (int q = 0; q < N; ++q) ns += sqrt(red[q]);
    nsum = ns;
    rz = red[N];
    bad = red[N + 1];
    __syncthreads();
}

template <int WARPS>
__device__ double warp0_sum_slots(const double* slots, int n, double* red) {
    if (threadIdx.x < 32) {
        double v = 0.0;
        for (int i = threadIdx.x; i < n; i += 32) v += __ldcg(slots + i);
        v = warp_sum(v);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
}

// cp.async rows r < nrows, columns c < ncols except [skip_lo, skip_hi):
// dst[r * dld + c] = src[r * sld + c]. One warp per row (no index division),
// 16-byte copies when the source rows are 16-byte aligned (sld even, aligned
// base); dld and skip bounds are even.
template <int WARPS>
__device__ __forceinline__ void copy_rows(double* dst, int dld, int nrows, const double* src, long long sld,
                                          int ncols, int skip_lo, int skip_hi) {
    if (nrows <= 0 || ncols <= 0 || (kAblate & 2)) return;
    const int lane = threadIdx.x & 31;
    const bool vec = (sld & 1) == 0 && (reinterpret_cast<std::uintptr_t>(src) & 15) == 0;
    for (int r = threadIdx.x >> 5; r < nrows; r += WARPS) {
        const double* sr = src + r * sld;
        double* dr = dst + r * dld;
        if (vec) {
            for (int c = 2 * lane; c < ncols; c += 64) {
                if (c >= skip_lo && c < skip_hi) continue;
                if (c + 1 < ncols) cp_async16(dr + c, sr + c);
                else cp_async8(dr + c, sr + c);
            }
        } else {
            for (int c = lane; c < ncols; c += 32) {
                if (c >= skip_lo && c < skip_hi) continue;
                cp_async8(dr + c, sr + c);
            }
        }
    }
}

// acc += A[16 rows from am][kpad] * B[kpad][8 cols from bn] (kpad % 8 == 0).
// A row-major (lda) or k-major (kAK: element (row, k) at A[k * lda + row]);
// B k-major (ldb).
template <bool kAK>
__device__ __forceinline__ void warp_mma(const double* A, int lda, int am, const double* B, int ldb, int bn, int kpad,
                                         double acc[4]) {
    if (kAblate & 4) return;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    auto av = [&](int row, int k) { return kAK ? A[k * lda + am + row] : A[(am + row) * lda + k]; };
    int k = 0;
    for (; k + 16 <= kpad; k += 16) {
        double a[8], b[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = av(g + 8 * (i & 1), k + t + 4 * (i >> 1));
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = B[(k + t + 4 * i) * ldb + bn + g];
        dmma16816(acc, a, b);
    }
    if (k < kpad) {
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = av(g + 8 * (i & 1), k + t + 4 * (i >> 1));
#pragma unroll
        for (int i = 0; i < 2; ++i) b[i] = B[(k + t + 4 * i) * ldb + bn + g];
        dmma1688(acc, a, b);
    }
}

__device__ __forceinline__ void r_stamp(const RDev& d, int vb, int it, int k) {
    if (d.p.trace && vb == 0 && threadIdx.x == 0 && it >= 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        d.p.trace[it * 16 + k] = t;
    }
}

// ---- thread-block cluster mode (CLU): the nct column tiles of one row block
// form a cluster, so a row's sibling columns (W' in phase B, R' in phase C)
// arrive by bulk copies into this CTA's shared memory (DSMEM pushes from the
// siblings) instead of being published to global memory and gathered back
// through L2. Measured at C2: 23.9 -> 22.0-22.6 us per CG iteration; pulling
// the columns with ld.shared::cluster instead was slower than the L2 gather
// (28 us), and a cluster-hierarchical grid barrier cost 2.5 us more.
__device__ __forceinline__ void clu_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void clu_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ unsigned clu_map(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

// CLU row buffer: Rb is stored as nct column blocks [block][tm rows][bs],
// so this CTA's own block (its tile of the vector, all tm rows) is one
// contiguous run. push_own sends it to the same place in every sibling's Rb
// with one shared::cta -> shared::cluster bulk copy per sibling, completing
// on the sibling's exchange mbarrier. Every thread fences its own-block
// stores to the async proxy first; thread 0 arms the local barrier with the
// bytes the siblings push here.
__device__ __forceinline__ void push_own(double* Rb, int tm, int bs, int nct, int me, unsigned long long* xbar) {
    tile::fence_async_shared();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned bytes = static_cast<unsigned>(tm * bs * 8);
        const unsigned bar_local = tile::su32(xbar);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_local),
                     "r"(bytes * static_cast<unsigned>(nct - 1))
                     : "memory");
        const unsigned src = tile::su32(Rb + static_cast<long long>(me) * tm * bs);
        for (int k = 0; k < nct; ++k) {
            if (k == me) continue;
            const unsigned dst = clu_map(src, static_cast<unsigned>(k));
            const unsigned bar = clu_map(bar_local, static_cast<unsigned>(k));
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst), "r"(src), "r"(bytes), "r"(bar)
                         : "memory");
        }
    }
}

// acc += Rb[16 rows from am][kpad] * B[kpad][8 cols from bn] with Rb in the
// CLU column-block layout (a k16 step never straddles a block: tn % 16 == 0).
__device__ __forceinline__ void warp_mma_blk(const double* A, int tm, int bs, int tn, int am, const double* B, int ldb,
                                             int bn, int kpad, double acc[4]) {
    if (kAblate & 4) return;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    int k = 0;
    for (; k + 16 <= kpad; k += 16) {
        const int blk = k / tn;
        const double* Ab = A + static_cast<long long>(blk) * tm * bs + (k - blk * tn);
        double a[8], b[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = Ab[(am + g + 8 * (i & 1)) * bs + t + 4 * (i >> 1)];
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = B[(k + t + 4 * i) * ldb + bn + g];
        dmma16816(acc, a, b);
    }
    if (k < kpad) {
        const int blk = k / tn;
        const double* Ab = A + static_cast<long long>(blk) * tm * bs + (k - blk * tn);
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = Ab[(am + g + 8 * (i & 1)) * bs + t + 4 * (i >> 1)];
#pragma unroll
        for (int i = 0; i < 2; ++i) b[i] = B[(k + t + 4 * i) * ldb + bn + g];
        dmma1688(acc, a, b);
    }
}

template <int MT, int NT, bool CLU>
__global__ void __launch_bounds__(MT * NT * 32, 1) cg_res_kernel(const __grid_constant__ RDev d) {
    constexpr int WARPS = MT * NT, THREADS = WARPS * 32;
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[3 * WARPS + 3 + kMaxOrder + 2];
    const CgParams& p = d.p;
    const RLayout& L = d.L;
    const int R = L.R, N = L.order;
    const long long RR = static_cast<long long>(R) * R;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    // CLU: block order = task order (a cluster is the nct column tiles of one row block)
    const int vb = CLU ? static_cast<int>(blockIdx.x) : cta_rank(p.barrier);
    const unsigned nb = gridDim.x;
    auto gbar = [&](unsigned int& rnd) {
        grid_barrier(p.barrier, nb, rnd);
    };
    unsigned int round = 0;

    // ---- this CTA's tile
    const bool has = vb < L.tasks;
    int n = 0, rt = 0, ct = 0;
    if (has) {
        while (vb >= L.taskoff[n + 1]) ++n;
        const int local = vb - L.taskoff[n];
        rt = local / L.nct;
        ct = local % L.nct;
    }
    const long long s = has ? p.rows[n] : 0;
    const long long i0 = static_cast<long long>(rt) * L.tm;
    const int c0 = ct * L.tn;
    const int vr = has ? static_cast<int>(min(static_cast<long long>(L.tm), s - i0)) : 0;  // valid rows
    const int vc = has ? min(L.tn, R - c0) : 0;                                // valid columns
    const long long off = p.off[n];
    const long long rowbase = off + i0 * R;  // element offset of (i0, 0) in a stacked s x R buffer
    double* An = sm;
    double* Gs = sm + L.o_gnn;
    double* Ps = sm + L.o_pinv;
    double* Rb = sm + L.o_row;
    double* Ax = sm + L.o_aux;
    double* Ds = sm + L.o_ds;
    const int ld = L.ld, ks = L.ks;

    // fragment coordinates: thread element k = 2h + c at tile (fi, fc)
    const int wm = (warp / NT) * 16, wn = (warp % NT) * 8;
    int fi[4], fc[4];
    bool fv[4];
    long long fe[4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int k = 2 * h + c;
            fi[k] = wm + g + 8 * h;
            fc[k] = wn + 2 * t + c;
            fv[k] = fi[k] < vr && fc[k] < vc;
            fe[k] = rowbase + static_cast<long long>(fi[k]) * R + c0 + fc[k];
        }

    // ---- resident set: zero everything (pads stay zero), then stage
    for (int e = tid; e < L.smem; e += THREADS) sm[e] = 0.0;
    __syncthreads();
    if (has) {
        copy_rows<WARPS>(An, ld, vr, p.A + rowbase, R, R, 0, 0);
        copy_rows<WARPS>(Gs, ks, R, p.pair + (n * N + n) * RR + c0, R, vc, 0, 0);
        copy_rows<WARPS>(Ps, ks, R, p.pinv + n * RR + c0, R, vc, 0, 0);
    }
    cp_async_wait_all();
    __shared__ unsigned long long xbar;  // CLU: sibling blocks of the row buffer
    unsigned xphase = 0;
    if (CLU) {
        if (tid == 0) {
            tile::bar_init(&xbar);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        clu_arrive();  // every sibling's barrier exists before the first push
        clu_wait();
    }
    __syncthreads();

    // Row buffer Rb[0:vr, 0:R] = own tile (registers) | sibling columns formed
    // from x0 (+ coef * x1 when x1, coef * x0 otherwise).
    auto form_rows = [&](const double* x0, const double* x1, double coef, const double own[4], const double* dext,
                         const double* dsrc) {
        copy_rows<WARPS>(Rb, ld, vr, x0 + rowbase, R, R, c0, c0 + L.tn);
        if (x1) copy_rows<WARPS>(Ax, ld, vr, x1 + rowbase, R, R, c0, c0 + L.tn);
        if (dext) copy_rows<WARPS>(Ds, ks, R, dsrc, R, vc, 0, 0);
        cp_async_wait_all();
        __syncthreads();
        if (x1 || coef != 1.0) {
            for (int r = warp; r < vr; r += WARPS) {
                double* rr = Rb + r * ld;
                const double* ar = Ax + r * ld;
                for (int c = 2 * lane; c < R; c += 64) {  // pairs: R even or the odd tail element
                    if (c >= c0 && c < c0 + L.tn) continue;
                    rr[c] = x1 ? __fma_rn(coef, ar[c], rr[c]) : coef * rr[c];
                    if (c + 1 < R) rr[c + 1] = x1 ? __fma_rn(coef, ar[c + 1], rr[c + 1]) : coef * rr[c + 1];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (fv[k]) Rb[fi[k] * ld + c0 + fc[k]] = own[k];
        __syncthreads();
    };

    // ---- init: R = -G, Z = R Pinv, V = 0 (gauss_newton.cpp:296-303)
    double Rg[4], Vg[4], Wg[4], Zg[4], Qg[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        Rg[k] = fv[k] ? -1.0 * p.G[fe[k]] : 0.0;
        Vg[k] = Wg[k] = Zg[k] = Qg[k] = 0.0;
    }
    int rc = 0;  // Rr[rc] holds the published current residual
    auto phase_c_tail = [&]() {
        // Z = Rb Pinv_n (rows x cols); partials of <R, Z>, ||R||^2, finiteness
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (CLU) warp_mma_blk(Rb, L.tm, L.bs, L.tn, wm, Ps, ks, wn, L.rk, acc);
        else warp_mma<false>(Rb, ld, wm, Ps, ks, wn, L.rk, acc);
        double rz = 0.0, nrm = 0.0, bad = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            Zg[k] = fv[k] ? acc[k] : 0.0;
            if (fv[k]) {
                rz += Rg[k] * Zg[k];
                nrm += Rg[k] * Rg[k];
                if (!isfinite(Vg[k]) || !isfinite(Rg[k])) bad = 1.0;
            }
        }
        block_sum3<WARPS>(rz, nrm, bad, red);
        if (tid == 0) {
            r_slot_rz(d)[vb] = rz;
            r_slot_nrm(d)[vb] = nrm;
            r_slot_fin(d)[vb] = bad;
        }
    };
    // This tile's share A_n[rows,:]^T Z[rows, cols] of A_n^T Z_n (R x tn slab).
    // B_p(W') = A_p^T Z_p + beta B_p(W) then needs no pass of its own: one grid
    // barrier per iteration fewer than forming A_p^T W' after W' exists.
    auto z_partial = [&]() {
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k) Ax[fi[k] * ks + fc[k]] = Zg[k];  // k-major operand [i][z]
        __syncthreads();
        double* bp = r_bpart(d, n) + static_cast<long long>(rt) * RR;
        const int mtiles = L.rm / 16;
        for (int j = warp; j < mtiles * NT; j += WARPS) {
            const int mt = j / NT, nt = j % NT;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            warp_mma<true>(An, ld, mt * 16, Ax, ks, nt * 8, L.tm, acc);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int r = mt * 16 + g + 8 * h, z = nt * 8 + 2 * t + c;
                    if (r < R && z < vc) bp[static_cast<long long>(r) * R + c0 + z] = acc[2 * h + c];
                }
        }
    };
    // CLU: own tile into the own columns of Rb, pushed to the siblings (DSMEM
    // bulk copies); their blocks arrive on xbar
    auto push_rows = [&](const double own[4]) {
        double* blk = Rb + static_cast<long long>(ct) * L.tm * L.bs;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (fv[k]) blk[fi[k] * L.bs + fc[k]] = own[k];
        push_own(Rb, L.tm, L.bs, L.nct, ct, &xbar);
    };
    auto wait_rows = [&]() {
        tile::bar_wait(&xbar, xphase);
        xphase ^= 1u;
    };
    if (has) {
        if (CLU) {
            push_rows(Rg);
            wait_rows();
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (fv[k]) p.Rr[rc][fe[k]] = Rg[k];
            form_rows(p.G, nullptr, -1.0, Rg, nullptr, nullptr);
        }
        phase_c_tail();
        z_partial();
    }
    gbar(round);

    double gnorm, unused0, unused1;
    top_sums<WARPS>(d, red, unused0, gnorm, unused1);  // ||R|| = ||G|| at init
    const double target = p.cg_tol * gnorm;
    int it = 0, hit_cap = 0, breakdown = 0, nonfinite = 0;
    double rz = 0.0, wq = 0.0;
    bool first = true;
    // A2 item of this thread's first pass (element e of mode q's B_q; the G
    // lanes of a group hold the modes of one element)
    const int a2G = L.a2g, a2lg = L.a2lg;
    const int a2items = static_cast<int>(RR) * a2G;
    const int a2stride = static_cast<int>(nb) * WARPS * 32;
    const int a2base0 = (vb * WARPS + warp) * 32;
    constexpr bool kOverlap = !(kAblate & 32);
    constexpr int kPF = 10;  // slab partials held in registers across the loop-top sums
    for (;;) {
        // The slab partials of the first A2
        // pass are requested before the loop-top sums, so both L2 round trips
        // (per-tile slots, slabs) overlap instead of following each other.
        double pf_part[kPF];
        const bool pf_on = WARPS >= kPrefetchWarps && kOverlap && !(kAblate & 1) && a2base0 < a2items;
        if (pf_on) {
            const int w = a2base0 + lane;
            const bool ok = w < a2items;
            const int q = w & (a2G - 1);
            const bool act = ok && q < N;
            const double* src = r_bpart(d, act ? q : 0) + (ok ? (w >> a2lg) : 0);
            const int nt = act ? L.rowtiles[q] : 0;
#pragma unroll
            for (int u = 0; u < kPF; ++u) pf_part[u] = (u < nt) ? __ldcg(src + u * RR) : 0.0;
        }
        double rz_new, nsum, bad;
        if (kAblate & 8) {
            rz_new = 1.0;
            nsum = 1e300;
            bad = 0.0;
        } else {
            top_sums<WARPS>(d, red, rz_new, nsum, bad);
        }
        if (kAblate) bad = 0.0;
        double beta = 0.0;
        if (!first) {
            if (bad != 0.0) {
                nonfinite = 1;
                break;
            }
            beta = (p.beta_variant == 0) ? rz_new / rz : rz_new / wq;
        }
        if (kAblate) {
            beta = 0.5;
            nsum = 1e300;
        }
        rz = rz_new;
        if (!(nsum > target)) break;
        if (it >= p.cap) {
            hit_cap = 1;
            break;
        }
        r_stamp(d, vb, it, 0);
        // ---- A: W' = Z + beta W in registers (first: W' = Z), published for phase B
        if (has) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                Wg[k] = first ? Zg[k] : __fma_rn(beta, Wg[k], Zg[k]);
                if (!CLU && fv[k]) p.W[0][fe[k]] = Wg[k];
            }
            if (CLU) push_rows(Wg);  // waited for in phase B
        }
        r_stamp(d, vb, it, 1);
        r_stamp(d, vb, it, 2);
        // ---- A2: B_p(W') = sum of the A_p^T Z slabs + beta B_p(W);
        // D_n^T[z][r] = sum_{p!=n} Gamma(n,p)[r][z] B_p[r][z].
        // A group of G (pow2 >= N) adjacent lanes per element e: lane q sums mode q's
        // slabs (all loads in flight), the group exchanges the B_p by shuffles and
        // lane q forms D_q.
        if (!(kAblate & 1)) {
            const int G = a2G, lg = a2lg;
            const int items = a2items;
            const int wstride = a2stride;
            for (int base = a2base0; base < items; base += wstride) {
                const int w = base + lane;
                const bool ok = w < items;
                const int e = ok ? (w >> lg) : 0;
                const int q = w & (G - 1);
                const bool act = ok && q < N;
                const bool pre = pf_on && base == a2base0;  // this pass was requested at the loop top
                double pr[kMaxOrder];
#pragma unroll
                for (int m = 0; m < kMaxOrder; ++m)
                    pr[m] = (act && m < N && m != q) ? p.pair[(q * N + m) * RR + e] : 0.0;
                double b = 0.0;
                if (act) {
                    const double* src = r_bpart(d, q) + e;
                    const int nt = L.rowtiles[q];
                    for (int k0 = 0; k0 < nt; k0 += 16) {
                        double part[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            part[u] = (pre && k0 == 0 && u < kPF) ? pf_part[u < kPF ? u : 0] : (k0 + u < nt) ? __ldcg(src + (k0 + u) * RR) : 0.0;
#pragma unroll
                        for (int u = 0; u < 16; ++u)
                            if (k0 + u < nt) b += part[u];
                    }
                }
                if (act) {
                    double* bs = r_bsum(d) + q * RR + e;
                    if (!first) b = __fma_rn(beta, *bs, b);
                    *bs = b;
                }
                const int gl = lane & ~(G - 1);
                double dsum = 0.0;
#pragma unroll
                for (int m = 0; m < kMaxOrder; ++m) {
                    if (m >= G) break;
                    const double bm = __shfl_sync(0xffffffffu, b, gl + m);
                    if (m < N && m != q) dsum += pr[m] * bm;
                }
                if (act) {
                    const int r = e / R, z = e - r * R;
                    r_dt(d)[q * RR + z * R + r] = dsum;
                }
            }
        }
        r_stamp(d, vb, it, 8);
        // CLU: W' Gamma_nn needs no other CTA's global data (the siblings' W'
        // blocks come through DSMEM), so it runs between this barrier's arrive
        // and wait; the accumulation order (Gamma_nn part, then the D part) is
        // the one of the plain sequence.
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const bool early = CLU && kOverlap;
        if (early) {
            grid_arrive(p.barrier, round);
            if (has) {
                wait_rows();  // the siblings' W' blocks (pushed in phase A)
                warp_mma_blk(Rb, L.tm, L.bs, L.tn, wm, Gs, ks, wn, L.rk, acc);
            }
            grid_wait(p.barrier, nb, round);
        } else {
            gbar(round);
        }
        r_stamp(d, vb, it, 3);
        // ---- B: Q = [W' | A_n] [Gamma_nn ; D_n^T] + lambda Reg(W'); <W', Q> partial
        if (has) {
            if (CLU) {
                copy_rows<WARPS>(Ds, ks, R, r_dt(d) + n * RR + c0, R, vc, 0, 0);
                if (!early) wait_rows();
                r_stamp(d, vb, it, 13);
            } else {
                copy_rows<WARPS>(Rb, ld, vr, p.W[0] + rowbase, R, R, c0, c0 + L.tn);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (fv[k]) Rb[fi[k] * ld + c0 + fc[k]] = Wg[k];
                copy_rows<WARPS>(Ds, ks, R, r_dt(d) + n * RR + c0, R, vc, 0, 0);
            }
            cp_async_wait_all();  // sibling W' columns and the D slice
            __syncthreads();
            if (CLU) {
                if (!early) warp_mma_blk(Rb, L.tm, L.bs, L.tn, wm, Gs, ks, wn, L.rk, acc);
            } else {
                warp_mma<false>(Rb, ld, wm, Gs, ks, wn, L.rk, acc);
            }
            warp_mma<false>(An, ld, wm, Ds, ks, wn, L.rk, acc);
            double part = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (fv[k]) {
                    const double w = Wg[k];
                    const double reg = (p.shape == 0) ? p.lambda * w
                                                      : w * (p.lambda * Gs[(c0 + fc[k]) * ks + fc[k]]);
                    Qg[k] = acc[k] + reg;
                    if (!CLU) p.Q[fe[k]] = Qg[k];
                    part += w * Qg[k];
                } else {
                    Qg[k] = 0.0;
                }
            }
            const double tot = block_sum<WARPS>(part, red);
            if (tid == 0) r_slot_wq(d)[vb] = tot;
        }
        r_stamp(d, vb, it, 4);
        gbar(round);
        r_stamp(d, vb, it, 5);
        // ---- C: alpha; V += alpha W'; R' = R - alpha Q; Z = R' Pinv
        wq = (kAblate & 8) ? 1.0 : warp0_sum_slots<WARPS>(r_slot_wq(d), L.tasks, red);
        if (kAblate) wq = 1.0;
        if (!(wq > 0.0)) {
            breakdown = 1;
            break;
        }
        const double alpha = rz / wq;
        r_stamp(d, vb, it, 9);
        if (has) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (fv[k]) {
                    Vg[k] = __fma_rn(alpha, Wg[k], Vg[k]);
                    Rg[k] = __fma_rn(-alpha, Qg[k], Rg[k]);
                    if (!CLU) p.Rr[rc ^ 1][fe[k]] = Rg[k];
                }
            }
            if (CLU) {
                push_rows(Rg);
                wait_rows();
            } else {
                form_rows(p.Rr[rc], p.Q, -alpha, Rg, nullptr, nullptr);
            }
            r_stamp(d, vb, it, 10);
            phase_c_tail();
            r_stamp(d, vb, it, 11);
            z_partial();
            r_stamp(d, vb, it, 12);
        }
        rc ^= 1;
        r_stamp(d, vb, it, 6);
        gbar(round);
        r_stamp(d, vb, it, 7);
        ++it;
        first = false;
    }
    if (has) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (fv[k]) p.V[fe[k]] = Vg[k];
    }
    if (CLU) {  // no CTA leaves while a sibling could still read its shared memory
        clu_arrive();
        clu_wait();
    }
    if (vb == 0 && tid == 0) {
        p.result[0] = it;
        p.result[1] = hit_cap;
        p.result[2] = breakdown;
        p.result[3] = nonfinite;
        p.result[4] = rc;
    }
}

// ---- host: plan + launch
struct Cand {
    int mt, nt;
};
constexpr Cand kCands[] = {{1, 1}, {1, 2}, {1, 3}, {1, 4}, {2, 1}, {2, 2}, {2, 3}, {2, 4}, {3, 1}, {3, 2}, {3, 3}, {3, 4}};

bool make_rlayout(const CgParams& p, int mt, int nt, RLayout& L, bool clu = false) {
    L = RLayout{};
    L.order = p.order;
    L.R = p.R;
    L.tm = 16 * mt;
    L.tn = 8 * nt;
    L.nct = (p.R + L.tn - 1) / L.tn;
    int off = 0;
    long long bp = 0;
    for (int n = 0; n < p.order; ++n) {
        L.rowtiles[n] = static_cast<int>((p.rows[n] + L.tm - 1) / L.tm);
        L.taskoff[n] = off;
        off += L.rowtiles[n] * L.nct;
        L.bp_off[n] = bp;
        bp += static_cast<long long>(L.rowtiles[n]) * p.R * p.R;
    }
    L.a2g = 1;
    L.a2lg = 0;
    while (L.a2g < p.order) {
        L.a2g *= 2;
        ++L.a2lg;
    }
    L.taskoff[p.order] = off;
    L.tasks = off;
    L.dt_off = bp;
    L.rk = (p.R + 7) & ~7;
    L.rm = (p.R + 15) & ~15;
    L.ld = L.rm;
    while (L.ld % 16 != 4) ++L.ld;
    L.ks = L.tn + 4;
    const int rowbuf = L.tm * L.ld;
    const int kslice = L.rk * L.ks;
    L.bs = L.tn + 4;
    while (L.bs % 16 != 4) ++L.bs;
    L.o_gnn = rowbuf;
    L.o_pinv = L.o_gnn + kslice;
    L.o_row = L.o_pinv + kslice;
    if (clu) {  // Rb as nct column blocks; Ax only stages Z for z_partial (no sibling rebuild)
        L.o_aux = L.o_row + L.nct * L.tm * L.bs;
        L.o_ds = L.o_aux + L.tm * L.ks;
    } else {
        L.o_aux = L.o_row + rowbuf;
        L.o_ds = L.o_aux + std::max(rowbuf, L.tm * L.ks);
    }
    L.smem = L.o_ds + kslice;
    return true;
}

template <int MT, int NT>
void launch_res(const RDev& d, int grid, std::size_t smem, cudaStream_t st) {
    auto* fn = cg_res_kernel<MT, NT, false>;
    ensure_dynamic_smem(fn, smem);  // grow-only per device, under the process-wide mutex
    RDev dd = d;
    void* args[] = {&dd};
    launch_cooperative(reinterpret_cast<const void*>(fn), dim3(grid), dim3(MT * NT * 32), args, smem, st);
    count_launch(1);
}
// Cluster mode (clusters of nct column tiles); false when the device cannot
// hold every cluster at once (the caller then launches the plain kernel).
template <int MT>
bool launch_res_clu(const RDev& d, int grid, std::size_t smem, cudaStream_t st) {
    auto* fn = cg_res_kernel<MT, 4, true>;
    ensure_dynamic_smem(fn, smem);
    const unsigned cx = static_cast<unsigned>(d.L.nct);
    if (max_active_clusters(reinterpret_cast<const void*>(fn), dim3(MT * 4 * 32), cx, smem) < grid / d.L.nct)
        return false;
    RDev dd = d;
    void* args[] = {&dd};
    launch_cooperative_cluster(reinterpret_cast<const void*>(fn), dim3(grid), dim3(MT * 4 * 32), cx, args, smem, st);
    count_launch(1);
    return true;
}

}  // namespace

std::size_t cg_res_slots_needed(const CgParams& p) {
    std::size_t need = 0;
    for (const Cand& c : kCands) {
        RLayout L;
        make_rlayout(p, c.mt, c.nt, L);
        need = std::max(need, static_cast<std::size_t>(4 * L.tasks + L.dt_off) +
                                  2 * static_cast<std::size_t>(p.order) * p.R * p.R);
    }
    return need;
}

bool run_cg_resident(const CgParams& p, cudaStream_t st) {
    if (std::getenv("CPKIT_CG_STREAMING")) return false;
    int dev = 0, sms = 0, optin = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    {  // device attributes, cached per device (host path in front of every solve)
        static std::mutex mu;
        static int cache[64][2] = {};
        std::lock_guard<std::mutex> lock(mu);
        if (dev >= 0 && dev < 64 && cache[dev][0] > 0) {
            sms = cache[dev][0];
            optin = cache[dev][1];
        } else {
            CPK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            CPK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            if (dev >= 0 && dev < 64) cache[dev][0] = sms, cache[dev][1] = optin;
        }
    }
    const int budget = optin - 1024;  // static shared memory headroom
    int best = -1, best_cost = 1 << 30;
    RLayout bestL{};
    int force_mt = 0, force_nt = 0;
    if (const char* e = std::getenv("CPKIT_CG_TILE")) std::sscanf(e, "%d,%d", &force_mt, &force_nt);
    for (int i = 0; i < static_cast<int>(sizeof(kCands) / sizeof(kCands[0])); ++i) {
        RLayout L;
        make_rlayout(p, kCands[i].mt, kCands[i].nt, L);
        if (L.tasks > sms || static_cast<long long>(L.smem) * 8 > budget) continue;
        if (force_mt && (kCands[i].mt != force_mt || kCands[i].nt != force_nt)) continue;
        // Columns: one tile across R when R <= 32 (no sibling exchange), else 32-wide
        // tiles (measured best at R = 50..100: wider tiles exchange less, taller
        // ones leave SMs idle). Rows: the shortest tile that fits the machine.
        const int want_nt = std::min(4, (p.R + 7) / 8);
        const int cost = (kCands[i].nt == want_nt ? 0 : 1000) + kCands[i].mt;
        if (cost < best_cost) {
            best_cost = cost;
            best = i;
            bestL = L;
        }
    }
    if (best < 0) return false;
    if (static_cast<std::size_t>(4 * bestL.tasks + bestL.dt_off) + 2 * static_cast<std::size_t>(p.order) * p.R * p.R >
        static_cast<std::size_t>(p.nslots))
        return false;
    RDev d{};
    d.p = p;
    d.L = bestL;
    const int grid = bestL.tasks;
    const std::size_t smem = static_cast<std::size_t>(bestL.smem) * sizeof(double);
    if (!p.barrier_zeroed) CPK_CUDA(cudaMemsetAsync(p.barrier, 0, cg_barrier_words() * sizeof(unsigned int), st));
    // the nct column tiles of a row block as one thread-block cluster (sibling
    // columns through DSMEM); CPKIT_CG_NO_CLUSTER=1 keeps the L2 gathers
    // (R even: every row block is a whole number of 16-byte units, as the bulk copies need)
    if (kCands[best].nt == 4 && bestL.nct >= 2 && bestL.nct <= 8 && !std::getenv("CPKIT_CG_NO_CLUSTER")) {
        RDev dc = d;
        make_rlayout(p, kCands[best].mt, kCands[best].nt, dc.L, true);
        const std::size_t smem_c = static_cast<std::size_t>(dc.L.smem) * sizeof(double);
        bool done = false;
        if (static_cast<long long>(dc.L.smem) * 8 <= budget) {
            switch (kCands[best].mt) {
                case 1: done = launch_res_clu<1>(dc, grid, smem_c, st); break;
                case 2: done = launch_res_clu<2>(dc, grid, smem_c, st); break;
                default: done = launch_res_clu<3>(dc, grid, smem_c, st); break;
            }
        }
        if (done) return true;
    }
    switch (kCands[best].mt * 10 + kCands[best].nt) {
        case 11: launch_res<1, 1>(d, grid, smem, st); break;
        case 12: launch_res<1, 2>(d, grid, smem, st); break;
        case 13: launch_res<1, 3>(d, grid, smem, st); break;
        case 14: launch_res<1, 4>(d, grid, smem, st); break;
        case 21: launch_res<2, 1>(d, grid, smem, st); break;
        case 22: launch_res<2, 2>(d, grid, smem, st); break;
        case 23: launch_res<2, 3>(d, grid, smem, st); break;
        case 24: launch_res<2, 4>(d, grid, smem, st); break;
        case 31: launch_res<3, 1>(d, grid, smem, st); break;
        case 32: launch_res<3, 2>(d, grid, smem, st); break;
        case 33: launch_res<3, 3>(d, grid, smem, st); break;
        default: launch_res<3, 4>(d, grid, smem, st); break;
    }
    return true;
}

}  // namespace cpkit
