// MTTKRP dimension-tree kernels for sm_100a (fp64).
//
// Reference: mttkrp.cpp:160-189 computes M^(n) by contracting the tensor with
// the "back" factors (modes >= h) when n < h, else with the "front" factors,
// caching the root partial, then contracting the remaining kept modes
// (:118-126, :63-75). The reference's root step is a mode-at-a-time Eigen GEMM
// over a full tensor copy (:46-62, :79-87).
//
// B200 design: the root contraction is ONE fused GEMM against the
// Khatri-Rao product of all contracted factors, generated tile-by-tile in
// shared memory and never materialised:
//   back root   P_F[F x R] = X[F x B]   * KRP_B[B x R]   (kernel TRANS=false)
//   front root  P_B[B x R] = X[F x B]^T * KRP_F[F x R]   (kernel TRANS=true, split-K)
// X tiles are staged by TMA (cp.async.bulk.tensor, 128B swizzle) into a
// multi-stage mbarrier pipeline; the math is FP64 DMMA (mma.sync m16n8k16,
// SASS DMMA.8x8x4; tcgen05 has no f64 kind on sm_100a). Each warp owns a
// 16-row strip of the CTA tile and all NT n8-tiles of the rank columns.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "common.h"

namespace cpkit {

namespace {

constexpr int kBK = 32;  // k-depth of one pipeline stage (two 16-double swizzle atoms)

// ---------------------------------------------------------------- TMA plumbing
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw DeviceError("cuTensorMapEncodeTiled entry point unavailable");
    return fn;
}

// 2-D fp64 map over a row-major (outer x inner) matrix with box
// (box_inner x box_outer); swizzled maps use the 128-B atom (box_inner = 16).
CUtensorMap make_map(const double* base, std::uint64_t inner, std::uint64_t outer, std::uint32_t box_inner,
                     std::uint32_t box_outer, bool swizzle) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * sizeof(double)};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(std::uint64_t* bar, unsigned bytes) {  // no arrival
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned phase) {
    // bounded spin: a lost TMA transaction traps instead of hanging the GPU
    for (unsigned long long spin = 0;; ++spin) {
        unsigned ok;
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
        if (ok) return;
        if (spin > (1ull << 26)) __trap();
    }
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, std::uint64_t* bar, void* dst,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void dmma16816(double* d, const double* a, const double* b) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},"
        "{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// Byte offset of element (row, col) inside a 128B-swizzled atom of 16 doubles
// per row (the layout TMA SWIZZLE_128B produces; 1024-B aligned atom base).
__device__ __forceinline__ int swz(int row, int col) {
    return row * 128 + ((((col >> 1) ^ row) & 7) << 4) + ((col & 1) << 3);
}

// Row stride of the B (KRP) tile in shared memory, in doubles, so the
// B-fragment loads are conflict-free: rows are read as t+4i (NN, stride = 8
// mod 16) or as the permuted slots 2t+c+8h (TN, stride = 4 mod 16).
template <bool TRANS>
__host__ __device__ constexpr int krp_stride(int bn) {
    const int want = TRANS ? 4 : 8;
    int s = bn;
    while (s % 16 != want) ++s;
    return s;
}

// k-slot -> physical smem row inside a 16-deep k step (TN only): makes the
// transposed A-fragment reads hit 8 distinct 16B chunks per half-warp.
__device__ __forceinline__ int kperm(int s) { return 2 * (s & 3) + ((s >> 2) & 1) + 8 * (s >> 3); }

struct KrpDev {
    int nmodes;
    long long ext[kMaxOrder];
    const double* fac[kMaxOrder];
};

// KRP[k][r] = prod_j fac_j[i_j(k), r] for k < K, r < R; zero for R <= r < Rs.
// One warp per output row (index decomposition once per row), lanes over r
// with 16-byte stores; streams K x Rs doubles once per contraction.
__global__ void __launch_bounds__(256) krp_fill_kernel(KrpDev kd, long long K, int R, int Rs,
                                                       double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
    const int pairs = Rs / 2;  // Rs is even
    for (long long k = blockIdx.x * static_cast<long long>(blockDim.x >> 5) + (threadIdx.x >> 5); k < K; k += warps) {
        const double* rowp[kMaxOrder];
        long long rem = k;
        for (int j = kd.nmodes - 1; j >= 0; --j) {
            const long long ext = kd.ext[j];
            const long long i = rem % ext;
            rem /= ext;
            rowp[j] = kd.fac[j] + i * R;
        }
        double2* dst = reinterpret_cast<double2*>(out + k * Rs);
        for (int c = lane; c < pairs; c += 32) {
            const int r = 2 * c;
            double v0 = 0.0, v1 = 0.0;
            if (r < R) {
                v0 = __ldg(rowp[0] + r);
                for (int j = 1; j < kd.nmodes; ++j) v0 *= __ldg(rowp[j] + r);
            }
            if (r + 1 < R) {
                v1 = __ldg(rowp[0] + r + 1);
                for (int j = 1; j < kd.nmodes; ++j) v1 *= __ldg(rowp[j] + r + 1);
            }
            dst[c] = make_double2(v0, v1);
        }
    }
}

// Two-mode Khatri-Rao rows (the front root of orders 3-4): KRP[k] = A_0[k / s1] o A_1[k % s1].
// Flat over 16-byte output pairs (fully coalesced stores), 4 pairs in flight per thread.
__global__ void __launch_bounds__(256) krp_fill2_kernel(const double* __restrict__ a0, const double* __restrict__ a1,
                                                        unsigned s1, unsigned K, int R, unsigned P2,
                                                        double2* __restrict__ out) {
    const unsigned total = K * P2;
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < total; q0 += 4 * stride) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned q = q0 + u * stride;
            v[u] = make_double2(0.0, 0.0);
            if (q < total) {
                const unsigned k = q / P2, c = q - k * P2;
                const unsigned i0 = k / s1, i1 = k - i0 * s1;
                const int r = 2 * static_cast<int>(c);
                if (r < R) v[u].x = __ldg(a0 + static_cast<std::size_t>(i0) * R + r) * __ldg(a1 + static_cast<std::size_t>(i1) * R + r);
                if (r + 1 < R)
                    v[u].y = __ldg(a0 + static_cast<std::size_t>(i0) * R + r + 1) * __ldg(a1 + static_cast<std::size_t>(i1) * R + r + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned q = q0 + u * stride;
            if (q < total) out[q] = v[u];
        }
    }
}

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ double lds64(std::uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

// ---------------------------------------------------------------- root GEMM
// TRANS=false: C[m][n] = sum_k X[m][k] KRP[k][n]   (X is M x K, row stride = xmap)
// TRANS=true:  C[m][n] = sum_k X[k][m] KRP[k][n]   (X is K x M)
// Warp-specialised: warps 0..W-1 issue DMMA, warp W is the TMA producer (one
// elected lane) feeding a `stages`-deep ring of (X tile, KRP tile) buffers
// guarded by full/empty mbarriers. The BM x BN CTA tile is a grid of
// (BM/16) x (BN/8) m16n8 cells, dealt to the W DMMA warps as balanced
// contiguous row-major runs of at most MAXC cells (a run spans at most two m16
// rows): the tile need not be a multiple of the warp count, so BM can fit M and
// BN the rank without padding while every SM sub-partition gets equal work.
// Persistent grid over units (n-tile, m-tile, split); block: 32 * (W + 1).
// Block-size bound per run length: long runs (many accumulators) get fewer
// warps and more registers each.
__host__ __device__ constexpr int root_max_threads(int maxc) { return maxc >= 9 ? 32 * 9 : maxc >= 6 ? 32 * 11 : 32 * 13; }
// (The register cap ptxas derives from these bounds is per SM sub-partition:
// 9 warps put 3 on one sub-partition of 16 K registers, so 168 per thread is
// the real limit for the 288-thread variants, not 65536 / 288 = 224 - a
// __maxnreg__(224) build fails to launch.)

// FULL: every warp's run is exactly MAXC cells inside one m16 row (no per-cell
// predicates; the common case of a rank tile that the warps split evenly).
// RS (row split, NN only, 8 warps over 4 m16 rows): an odd number NT8 = 2 MAXC
// - 1 of n8 cells per m16 row is split between the row's two warps as MAXC +
// (MAXC - 1) cells, the longer run alternating so that each SM sub-partition
// (warps w and w + 4) carries exactly NT8 cells: no rank padding and no run
// crossing an m16 row (R = 200: 13 + 12 of 25 cells).
template <int MAXC, bool TRANS, bool GEN, bool FULL, bool RS = false, bool SK = false>
__global__ void __launch_bounds__(root_max_threads(MAXC), 1)
root_gemm_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                 const __grid_constant__ KrpDev kd, long long M, long long K, int R, int BM, int BN, int W,
                 int BNS, int stages, long long k_per_split, int splits, double* __restrict__ out,
                 long long out_split_stride, int brel, double* __restrict__ sk_ws) {
    extern __shared__ __align__(1024) char smem_raw[];
    const std::uint32_t raw = smem_u32(smem_raw);
    const std::uint32_t base = raw + ((1024u - (raw & 1023u)) & 1023u);  // 1024-B aligned (swizzle atom)
    char* const smem = smem_raw + (base - raw);
    const int x_bytes = BM * kBK * 8;
    const int b_bytes = kBK * BNS * 8;
    const int stage_bytes = x_bytes + b_bytes;
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + stages * stage_bytes);
    std::uint64_t* empty = full + stages;
    std::uint64_t* krp_bar = empty + stages;  // GEN: factor rows of the stage landed

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nboxes = TRANS ? BM / 16 : kBK / 16;
    const int box_rows = TRANS ? kBK : BM;
    // persistent work loop: unit u -> (n-tile, m-tile, split), n fastest so the
    // CTAs sharing an X row panel run together (L2 reuse)
    const int ntiles = (R + BN - 1) / BN;
    const long long mtiles = (M + BM - 1) / BM;
    const long long units = static_cast<long long>(ntiles) * mtiles * splits;
    // (32-bit divisions: a 64-bit division by a runtime value is a long
    // subroutine, paid per unit by every warp; the host keeps units < 2^31)
    const unsigned mtiles32 = static_cast<unsigned>(mtiles), ntiles32 = static_cast<unsigned>(ntiles);
    auto unit_geom = [&](long long u, int& n0, long long& m0, long long& kbeg, int& nk, int& split) {
        const unsigned uu = static_cast<unsigned>(u);
        const unsigned rest = ntiles32 == 1 ? uu : uu / ntiles32;
        n0 = ntiles32 == 1 ? 0 : static_cast<int>(uu - rest * ntiles32) * BN;
        const unsigned sp = rest / mtiles32;
        m0 = static_cast<long long>(rest - sp * mtiles32) * BM;
        split = static_cast<int>(sp);
        kbeg = static_cast<long long>(split) * k_per_split;
        const long long kend = min(K, kbeg + k_per_split);
        nk = static_cast<int>((kend - kbeg + kBK - 1) / kBK);
    };

    // Stream-K mode (template SK: a separate instantiation, so the classic
    // kernels carry none of this; one rank tile, no k split): the (row tile, k block)
    // space, tile-major, is cut into gridDim.x equal contiguous ranges, so
    // every CTA does the same number of k blocks whatever the tile count (no
    // partial last wave, no separate tail launch). A CTA's range is a run of
    // segments, one per tile it touches: a segment covering a whole tile goes
    // straight to the output; a tile shared by two or more CTAs leaves partial
    // tiles in sk_ws (slot 2 c for the segment of CTA c that starts inside a
    // tile, 2 c + 1 for the one that starts a tile and ends inside it), summed
    // in CTA (= k) order by streamk_fixup_kernel: deterministic.
    const long long kblocks = (K + kBK - 1) / kBK;
    const long long sk_total = mtiles * kblocks;
    const long long sk_lo = SK ? sk_total * blockIdx.x / gridDim.x : 0;
    const long long sk_hi = SK ? sk_total * (blockIdx.x + 1) / gridDim.x : 0;
    struct Unit {
        int n0, nk;
        long long m0, kbeg, kend;
        double* o;
    };
    auto next_unit = [&](long long& cur, Unit& un) -> bool {
        if (!SK) {
            if (cur >= units) return false;
            int split;
            unit_geom(cur, un.n0, un.m0, un.kbeg, un.nk, split);
            un.kend = min(K, un.kbeg + k_per_split);
            un.o = out + split * out_split_stride;
            cur += gridDim.x;
            return true;
        }
        if (cur >= sk_hi) return false;
        const long long tile = cur / kblocks, kb0 = cur - tile * kblocks;
        const long long len = min(kblocks - kb0, sk_hi - cur);
        un.n0 = 0;
        un.m0 = tile * BM;
        un.kbeg = kb0 * kBK;
        un.kend = min(K, (kb0 + len) * kBK);
        un.nk = static_cast<int>(len);
        un.o = (kb0 == 0 && len == kblocks)
                   ? out
                   : sk_ws + (2 * static_cast<long long>(blockIdx.x) + (kb0 != 0 ? 0 : 1)) * BM * R - un.m0 * R;
        cur += len;
        return true;
    };
    const long long cur0 = SK ? sk_lo : static_cast<long long>(blockIdx.x);

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], W);
            mbar_init(&krp_bar[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == W) {
        // ---------------- producer: one ring across all of this CTA's units.
        // X tiles by TMA (one elected lane). The KRP tile either by TMA from the
        // materialised workspace or (GEN) computed by the whole warp straight
        // into the stage: row k of the stage is prod_j fac_j[i_j(k)], lanes over
        // rank pairs, the mixed-radix index advanced row to row (no division).
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&xmap)) : "memory");
            if (!GEN) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&kmap)) : "memory");
        }
        if (!GEN && lane != 0) return;
        // GEN: KRP row k = A_0[k / s1] o A_1[k % s1]; scale the landed A_1 rows of
        // stage `i` in place by the A_0 row, then release the stage to the consumers
        int pend_n0 = 0;
        long long pend_kk = 0;
        auto gen_finish = [&](long long i, int n0, long long kk) {
            const int s = static_cast<int>(i % stages);
            double* bsm = reinterpret_cast<double*>(smem + s * stage_bytes + x_bytes);
            const long long s1 = kd.ext[1];
            double2 a0v[2][2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const long long k = kk + 16 * h;
                const bool ok = k < K;
                const double* a0 = kd.fac[0] + (k / s1) * R + n0;
#pragma unroll
                for (int pass = 0; pass < 2; ++pass) {
                    const int c = 2 * lane + 64 * pass;
                    const bool c0 = ok && n0 + c < R, c1 = ok && n0 + c + 1 < R;
                    a0v[h][pass] = make_double2(c0 ? __ldg(a0 + c) : 0.0, c1 ? __ldg(a0 + c + 1) : 0.0);
                }
            }
            mbar_wait(&krp_bar[s], static_cast<unsigned>((i / stages) & 1));
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll 4
                for (int q = 16 * h; q < 16 * h + 16; ++q) {
#pragma unroll
                    for (int pass = 0; pass < 2; ++pass) {
                        const int c = 2 * lane + 64 * pass;
                        if (c < BN) {
                            double2* dst = reinterpret_cast<double2*>(bsm + q * BNS + c);
                            const double2 v = *dst;
                            const double2 f = a0v[h][pass];
                            *dst = make_double2(v.x * f.x, v.y * f.y);
                        }
                    }
                }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);  // releases the warp's shared stores
        };
        long long it = 0;  // global stage counter
        // ring slot and lap parity kept incrementally: a runtime `it % stages`
        // is an integer division per stage (I2F/MUFU/IMAD.HI chain; 3 % of the
        // C2 root's stall samples sat on it)
        int ring = -1;
        unsigned lap = 1;  // parity of (it / stages)
        long long cur = cur0;
        Unit un;
        while (next_unit(cur, un)) {
            const int n0 = un.n0, nk = un.nk;
            const long long m0 = un.m0, kbeg = un.kbeg;
            for (int kt = 0; kt < nk; ++kt, ++it) {
                if (++ring == stages) ring = 0;
                if (ring == 0) lap ^= 1u;
                const int s = ring;
                if (it >= stages) mbar_wait(&empty[s], lap ^ 1u);
                const long long kk = kbeg + static_cast<long long>(kt) * kBK;
                char* xs = smem + s * stage_bytes;
                if (lane == 0) {
                    if (GEN) {
                        fence_proxy_async();  // the warp's earlier generic stores to this stage
                        mbar_expect_tx_only(&full[s], static_cast<unsigned>(x_bytes));
                    } else {
                        mbar_expect_tx(&full[s], static_cast<unsigned>(stage_bytes));
                    }
                    for (int b = 0; b < nboxes; ++b) {
                        if (TRANS)
                            tma_load_2d(&xmap, &full[s], xs + b * box_rows * 128, static_cast<int>(m0 + 16 * b),
                                        static_cast<int>(kk));
                        else
                            tma_load_2d(&xmap, &full[s], xs + b * box_rows * 128, static_cast<int>(kk + 16 * b),
                                        static_cast<int>(m0));
                    }
                    if (!GEN) {
                        // brel: batched contraction, the B operand restarts at row 0 in
                        // every split (rows past its extent are TMA zero fill)
                        tma_load_2d(&kmap, &full[s], xs + x_bytes, n0, static_cast<int>(brel ? kk - kbeg : kk));
                    } else {
                        // A_1 rows of the two 16-row halves (s1 % 16 == 0: a half never wraps)
                        mbar_expect_tx(&krp_bar[s], static_cast<unsigned>(b_bytes));
                        const long long s1 = kd.ext[1];
                        for (int h = 0; h < 2; ++h) {
                            const long long k = kk + 16 * h;
                            tma_load_2d(&kmap, &krp_bar[s], xs + x_bytes + h * 16 * BNS * 8, n0,
                                        static_cast<int>(k % s1));
                        }
                    }
                }
                if (GEN) {
                    // finish the previous stage while this one's copies are in flight
                    if (it > 0) gen_finish(it - 1, pend_n0, pend_kk);
                    pend_n0 = n0;
                    pend_kk = kk;
                }
            }
        }
        if (GEN && it > 0) gen_finish(it - 1, pend_n0, pend_kk);
        return;
    }

    // ---------------- DMMA consumers: this warp's run of cells [cs, cs + cnt)
    // of the (BM/16) x NT8 cell grid; the first n1 cells lie in m16 row r0,
    // the rest in row r0 + 1
    const int g = lane >> 2, t = lane & 3;
    const int NT8 = BN / 8;
    const int cells = (BM / 16) * NT8;
    const int cbase = cells / W, cextra = cells % W;
    // RS: warp w takes part w % 2 of m16 row w / 2; the long part (MAXC cells)
    // is the first one when (w / 4) is even, else the second
    const bool rs_long_first = ((warp >> 2) & 1) == 0;
    const int rs_first = rs_long_first ? MAXC : NT8 - MAXC;
    const int cnt = RS ? ((warp & 1) ? NT8 - rs_first : rs_first) : FULL ? MAXC : cbase + (warp < cextra ? 1 : 0);
    const int cs = RS ? (warp >> 1) * NT8 + ((warp & 1) ? rs_first : 0) : warp * cbase + min(warp, cextra);
    const int r0 = cs / NT8, c0 = cs - r0 * NT8;
    const int n1 = (FULL || RS) ? cnt : min(cnt, NT8 - c0);
    // byte offset of cell j's n8 column in a KRP k-row: 64 j + (j < n1 ? ofs_a : ofs_b)
    const std::uint32_t ofs_a = static_cast<std::uint32_t>(c0 * 64), ofs_b = static_cast<std::uint32_t>(-n1 * 64);
    const std::uint32_t rowstep = TRANS ? kBK * 128 : 16 * 128;  // next m16 row of the X tile

    // per-lane constant parts of the fragment addresses
    std::uint32_t aoff[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int mrow = 16 * r0 + g + 8 * (i & 1);
        if (!TRANS) {
            aoff[i] = static_cast<std::uint32_t>(swz(mrow, t + 4 * (i >> 1)));
        } else {
            const int krow = kperm(t + 4 * (i >> 1));
            aoff[i] = static_cast<std::uint32_t>((mrow >> 4) * kBK * 128 + swz(krow, mrow & 15));
        }
    }
    std::uint32_t boff[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int krow = TRANS ? kperm(t + 4 * i) : t + 4 * i;
        boff[i] = static_cast<std::uint32_t>((krow * BNS + g) * 8);
    }
    const bool vec = (R % 2) == 0;

    // The mainloop for a compile-time run length C (warps' counts differ by at
    // most one: C is MAXC or MAXC - 1) and SPAN (the run crosses into row
    // r0 + 1: both rows' A fragments are loaded and selected per cell), so no
    // cell carries a runtime predicate and all loads can be hoisted.
    auto mainloop = [&](auto c_tag, auto span_tag) {
        constexpr int C = decltype(c_tag)::value;
        constexpr bool SPAN = decltype(span_tag)::value;
        int ring = -1;      // ring slot of the current stage and the parity of its lap,
        unsigned lap = 1;   // kept incrementally (no per-stage integer division)
        long long cur = cur0;
        Unit un;
        while (next_unit(cur, un)) {
            const int n0 = un.n0, nk = un.nk;
            const long long m0 = un.m0, kbeg = un.kbeg;
            double acc[C][4];
#pragma unroll
            for (int j = 0; j < C; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0;
            // the unit's last stage holds only 16 valid k (see half_stage below)
            const bool last_half = un.kend - (kbeg + static_cast<long long>(nk - 1) * kBK) <= 16;

            for (int kt = 0; kt < nk; ++kt) {
                if (++ring == stages) ring = 0;
                if (ring == 0) lap ^= 1u;
                const int s = ring;
                mbar_wait(&full[s], lap);
                // plain shared loads (ordered after the full-barrier wait by its
                // memory clobber, otherwise free for the scheduler to hoist)
                const char* xs = smem + s * stage_bytes;
                const char* bs = xs + x_bytes;
                auto ld = [](const char* p, std::uint32_t off) { return *reinterpret_cast<const double*>(p + off); };
                static_assert(kBK == 32, "two k16 steps per stage");
                // a unit's last stage may hold only 16 valid k (its B rows beyond
                // the unit's k range are zero): skip the empty half instead of
                // multiplying zeros
                const bool half_stage = kt == nk - 1 && last_half;
#pragma unroll
                for (int ks = 0; ks < kBK / 16; ++ks) {
                    if (ks == 1 && half_stage) break;
                    double a[8];
                    // NN: box ks holds k in [16ks, 16ks+16). TN: rows 16ks.. of every m-box.
                    const char* abase = TRANS ? xs + ks * 16 * 128 : xs + ks * BM * 128;
#pragma unroll
                    for (int i = 0; i < 8; ++i) a[i] = ld(abase, aoff[i]);
                    const char* bb = bs + ks * 16 * BNS * 8;
#pragma unroll
                    for (int j = 0; j < C; ++j) {
                        const bool first_row = !SPAN || j < n1;
                        const std::uint32_t co = j * 64 + (first_row ? ofs_a : ofs_b);
                        double b[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) b[i] = ld(bb, boff[i] + co);
                        if (SPAN && j == n1) {  // the run continues in row r0 + 1
#pragma unroll
                            for (int i = 0; i < 8; ++i) a[i] = ld(abase + rowstep, aoff[i]);
                        }
                        dmma16816(acc[j], a, b);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }

            // epilogue (overlaps the producer's loads for the next unit):
            // rows m0+16(r0 | r0+1)+g(+8), cols n0+8(cell column)+2t(+1); 16-byte stores when aligned
            double* o = un.o;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                const bool first_row = !SPAN || j < n1;
                const int col = n0 + 8 * (first_row ? c0 + j : j - n1) + 2 * t;
                const int rr = 16 * (r0 + (first_row ? 0 : 1));
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const long long row = m0 + rr + g + 8 * h;
                    if (row < M && col < R) {
                        double* dst = o + row * R + col;
                        if (vec) {
                            *reinterpret_cast<double2*>(dst) = make_double2(acc[j][2 * h], acc[j][2 * h + 1]);
                        } else {
                            dst[0] = acc[j][2 * h];
                            if (col + 1 < R) dst[1] = acc[j][2 * h + 1];
                        }
                    }
                }
            }
        }
    };
    using CFull = std::integral_constant<int, MAXC>;
    using CLess = std::integral_constant<int, (MAXC > 1 ? MAXC - 1 : 1)>;
    using Yes = std::integral_constant<bool, true>;
    using No = std::integral_constant<bool, false>;
    if (FULL) {
        mainloop(CFull{}, No{});
    } else if (RS) {  // runs never cross an m16 row
        if (cnt == MAXC) mainloop(CFull{}, No{});
        else mainloop(CLess{}, No{});
    } else {
        const bool span = n1 < cnt;
        if (cnt == MAXC) {
            if (span) mainloop(CFull{}, Yes{});
            else mainloop(CFull{}, No{});
        } else {
            if (span) mainloop(CLess{}, Yes{});
            else mainloop(CLess{}, No{});
        }
    }
}

// NN root with m8n8k4 DMMA tiles, for ranks that are a multiple of 8 with an
// odd number NC of n8 cells (R = 200: 25 cells). The m16n8k16 kernel above
// needs every warp's run inside one m16 row with the cells split evenly over
// the warps, so it pads 25 cells to 26 (4 % of the DMMA work on zero columns).
// Here the 64-row CTA tile is 8 m8 strips, one per DMMA warp, each strip with
// ALL NC cells: no padding, equal work on the four SM sub-partitions. Per k4
// step a warp loads one A value and NC B values per lane (the B tile is shared
// by the warps) and issues NC DMMA.8x8x4. Same producer, ring, persistent unit
// loop and split-K contract as root_gemm_kernel<.., TRANS=false, GEN=false>.
constexpr int kM8Warps = 8;
template <int NC>
__global__ void __launch_bounds__(32 * (kM8Warps + 1), 1)
root_gemm_m8_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
                    long long M, long long K, int R, int BNS, int stages, long long k_per_split, int splits,
                    double* __restrict__ out, long long out_split_stride) {
    extern __shared__ __align__(1024) char smem_raw[];
    const std::uint32_t raw = smem_u32(smem_raw);
    const std::uint32_t base = raw + ((1024u - (raw & 1023u)) & 1023u);
    char* const smem = smem_raw + (base - raw);
    constexpr int W = kM8Warps, BM = 8 * W;
    const int x_bytes = BM * kBK * 8;
    const int b_bytes = kBK * BNS * 8;
    const int stage_bytes = x_bytes + b_bytes;
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + stages * stage_bytes);
    std::uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long mtiles = (M + BM - 1) / BM;
    const long long units = mtiles * splits;
    auto unit_geom = [&](long long u, long long& m0, long long& kbeg, int& nk) {
        m0 = (u % mtiles) * BM;
        kbeg = (u / mtiles) * k_per_split;
        const long long kend = min(K, kbeg + k_per_split);
        nk = static_cast<int>((kend - kbeg + kBK - 1) / kBK);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], W);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == W) {  // ---------------- producer (one lane)
        if (lane != 0) return;
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&xmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&kmap)) : "memory");
        long long it = 0;
        int ring = -1;
        unsigned lap = 1;
        for (long long u = blockIdx.x; u < units; u += gridDim.x) {
            long long m0, kbeg;
            int nk;
            unit_geom(u, m0, kbeg, nk);
            for (int kt = 0; kt < nk; ++kt, ++it) {
                if (++ring == stages) ring = 0;
                if (ring == 0) lap ^= 1u;
                const int s = ring;
                if (it >= stages) mbar_wait(&empty[s], lap ^ 1u);
                const long long kk = kbeg + static_cast<long long>(kt) * kBK;
                char* xs = smem + s * stage_bytes;
                mbar_expect_tx(&full[s], static_cast<unsigned>(stage_bytes));
                for (int b = 0; b < kBK / 16; ++b)
                    tma_load_2d(&xmap, &full[s], xs + b * BM * 128, static_cast<int>(kk + 16 * b), static_cast<int>(m0));
                tma_load_2d(&kmap, &full[s], xs + x_bytes, 0, static_cast<int>(kk));
            }
        }
        return;
    }
    // ---------------- DMMA consumers: warp w owns rows 8w..8w+7 of the tile, all NC cells
    const int g = lane >> 2, t = lane & 3;
    const int arow = 8 * warp + g;
    int ring = -1;
    unsigned lap = 1;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        long long m0, kbeg;
        int nk;
        unit_geom(u, m0, kbeg, nk);
        double acc[NC][2];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c][0] = acc[c][1] = 0.0;
        const bool last_half = min(K, kbeg + k_per_split) - (kbeg + static_cast<long long>(nk - 1) * kBK) <= 16;
        for (int kt = 0; kt < nk; ++kt) {
            if (++ring == stages) ring = 0;
            if (ring == 0) lap ^= 1u;
            const int s = ring;
            mbar_wait(&full[s], lap);
            const char* xs = smem + s * stage_bytes;
            const double* bs = reinterpret_cast<const double*>(xs + x_bytes);
            const bool half_stage = kt == nk - 1 && last_half;
#pragma unroll
            for (int ks = 0; ks < kBK / 4; ++ks) {
                if (ks == kBK / 8 && half_stage) break;
                const int kr = 4 * ks + t;  // this lane's k inside the stage
                const double a = *reinterpret_cast<const double*>(xs + (kr >> 4) * BM * 128 + swz(arow, kr & 15));
                const double* brow = bs + kr * BNS + g;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double b = brow[8 * c];
                    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                        : "+d"(acc[c][0]), "+d"(acc[c][1])
                        : "d"(a), "d"(b));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        double* o = out + (u / mtiles) * out_split_stride;
        const long long row = m0 + arow;
        if (row < M) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
                *reinterpret_cast<double2*>(o + row * R + 8 * c + 2 * t) = make_double2(acc[c][0], acc[c][1]);
        }
    }
}

__global__ void splitk_reduce_kernel(const double* __restrict__ ws, int splits, long long n,
                                     double* __restrict__ out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < splits; ++k) s += ws[k * n + i];  // fixed order: deterministic
        out[i] = s;
    }
}

// A tile is shared by at most ctas / mtiles + 2 CTAs (plan_streamk checks the bound).
constexpr int kStreamKMaxPieces = 192;
// Stream-K fix-up (root_gemm_kernel, sk mode): block c - 1 looks at the range
// boundary between CTAs c - 1 and c. When it falls inside a row tile and is the
// first boundary inside that tile, the block sums the tile's partial slots in
// CTA (= k) order and writes the tile's output rows.
__global__ void __launch_bounds__(256) streamk_fixup_kernel(const double* __restrict__ ws, double* __restrict__ out,
                                                            long long M, int R, int BM, long long mtiles,
                                                            long long kblocks, int G) {
    const long long T = mtiles * kblocks;
    const int c = static_cast<int>(blockIdx.x) + 1;
    const long long b = T * c / G;
    if (b % kblocks == 0) return;
    const long long t = b / kblocks, t_lo = t * kblocks, t_hi = t_lo + kblocks;
    if (T * (c - 1) / G > t_lo) return;  // an earlier boundary is inside the same tile: that block sums it
    __shared__ int slots[kStreamKMaxPieces];
    __shared__ int nslots;
    if (threadIdx.x == 0) {
        int n = 0;
        for (int j = c - 1; j < G && n < kStreamKMaxPieces; ++j) {
            const long long lo = T * j / G;
            if (lo >= t_hi) break;
            slots[n++] = 2 * j + (lo > t_lo ? 0 : 1);
        }
        nslots = n;
    }
    __syncthreads();
    const long long rows = min(static_cast<long long>(BM), M - t * BM);
    const long long n = rows * R, slab = static_cast<long long>(BM) * R;
    double* o = out + t * BM * R;
    for (long long e = threadIdx.x; e < n; e += blockDim.x) {
        double v = 0.0;
        for (int q = 0; q < nslots; ++q) v += ws[slots[q] * slab + e];
        o[e] = v;
    }
}

KrpDev to_dev(const KrpDesc& d) {
    KrpDev k{};
    k.nmodes = d.nmodes;
    for (int i = 0; i < d.nmodes; ++i) {
        k.ext[i] = d.ext[i];
        k.fac[i] = d.fac[i];
    }
    return k;
}

int num_sms() { return device_sm_count(); }  // per device (runtime.cu)

// ---- tile planning --------------------------------------------------------
// CTA tile = (16 WM rows) x (8 NTW WN rank columns); WM x WN DMMA warps + 1
// TMA producer warp. NTW comes from the instantiated set.
constexpr int kMaxcChoices[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 13, 16};
int round_maxc(int need) {
    for (int c : kMaxcChoices)
        if (c >= need) return c;
    return -1;
}
struct GemmPlan {
    int maxc, nw, wm, nt8, ntiles, bns, stages, mtiles, splits, per_sm;
    long long kps;
    bool m8;  // root_gemm_m8_kernel (wm = 4: 64-row tiles, 8 warps, all nt8 cells per warp)
    bool rs;  // root_gemm_kernel<.., RS>: wm = 4, nw = 8, odd nt8 split per row as maxc + (maxc - 1)
    int BM() const { return 16 * wm; }
    int BN() const { return 8 * nt8; }
};
int bns_for(int bn, bool trans) {
    if (const char* e = std::getenv(trans ? "CPKIT_TN_BNS_MOD" : "CPKIT_NN_BNS_MOD")) {  // experiments only
        int s = bn;
        while (s % 16 != std::atoi(e)) ++s;
        return s;
    }
    return trans ? krp_stride<true>(bn) : krp_stride<false>(bn);
}
std::size_t stage_bytes_of(int BM, int bns) { return static_cast<std::size_t>(BM) * kBK * 8 + kBK * bns * 8; }
std::size_t smem_bytes(const GemmPlan& p) {
    return static_cast<std::size_t>(p.stages) * stage_bytes_of(p.BM(), p.bns) + p.stages * 24 + 1024;
}
// Fraction of the DMMA issue slots doing useful cells when wm x nt8 cells are
// dealt to nw warps as balanced runs (the kernel's rule) and warp w issues on
// SM sub-partition w % 4.
double cell_efficiency(int wm, int nt8, int nw) {
    const int cells = wm * nt8, base = cells / nw, extra = cells % nw;
    int load[4] = {0, 0, 0, 0};
    for (int w = 0; w < nw; ++w) load[w % 4] += base + (w < extra ? 1 : 0);
    const int mx = std::max(std::max(load[0], load[1]), std::max(load[2], load[3]));
    return static_cast<double>(cells) / (4.0 * mx);
}
// A run of maxc cells starting anywhere in a row of nt8 spans at most two rows.
bool runs_fit(int wm, int nt8, int nw) {
    const int cells = wm * nt8, base = cells / nw, extra = cells % nw;
    for (int w = 0; w < nw; ++w) {
        const int cs = w * base + std::min(w, extra), cnt = base + (w < extra ? 1 : 0);
        if (cnt == 0) return false;
        if ((cs % nt8) + cnt > 2 * nt8) return false;
    }
    return true;
}
// Split count with the best wave efficiency (<= 2 waves or the unsplit count),
// keeping >= 8 k-stages per split; ties go to fewer splits.
long long best_splits(long long base, long long slots, long long K, double* eff_out, int min_chunks = 8,
                      int wave_cap = 0) {
    const long long kchunks = (K + kBK - 1) / kBK;
    long long best = 1;
    double best_eff = -1.0;
    // Fewer tiles than one wave (e.g. C4's 79 row tiles): splits may go up to
    // 8 waves, each split's extra output pass (read by the fixed-order reduce,
    // ~24 sp / K of the GEMM's time) charged against its wave efficiency.
    // Otherwise at most 2 waves (the NN root's partial last wave is handled by
    // a separate tail launch, plan_back).
    long long max_waves = base < slots ? 8 : std::max<long long>(2, (base + slots - 1) / slots);
    if (wave_cap > 0) max_waves = std::min<long long>(max_waves, wave_cap);
    double best_score = -1.0;
    for (long long sp = 1; sp <= 64; ++sp) {
        if (sp > 1 && kchunks / sp < min_chunks) break;
        const long long ctas = base * sp;
        const long long waves = (ctas + slots - 1) / slots;
        if (sp > 1 && waves > max_waves) break;
        const double eff = static_cast<double>(ctas) / static_cast<double>(waves * slots);
        const double score = base < slots && sp > 1 ? eff / (1.0 + 24.0 * static_cast<double>(sp) / K) : eff;
        if (score > best_score + 1e-9) {
            best_score = score;
            best_eff = eff;
            best = sp;
        }
    }
    if (eff_out) *eff_out = best_score;  // split candidates carry their reduce cost into the tile score
    (void)best_eff;
    return best;
}
int resident_per_sm(const GemmPlan& p) {
    // ptxas may use up to the launch bound's share of the register file
    const int per_thread = std::min(255, 65536 / root_max_threads(p.maxc)) & ~7;
    const int regs = 32 * (p.nw + 1) * per_thread;
    return std::max(1, std::min<int>(static_cast<int>((228 * 1024) / smem_bytes(p)), 65536 / regs));
}
// Every warp's run is exactly maxc cells in one row (the kernel's FULL case).
bool runs_full(const GemmPlan& p) {
    const int cells = p.wm * p.nt8;
    if (cells % p.nw != 0 || cells / p.nw != p.maxc) return false;
    return p.nt8 % p.maxc == 0;
}

// fixed_kps > 0: batched contraction, split s covers k in [s kps, (s+1) kps)
// and writes its own output slab (no split search, no reduction).
bool rs_enabled() {  // CPKIT_NN_RS=0: no row-split dealing (then the m8 variant, or padding)
    static const int v = [] {
        const char* e = std::getenv("CPKIT_NN_RS");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0;
}
bool m8_enabled() {  // CPKIT_NN_M8=0: always the m16n8k16 kernel
    static const int v = [] {
        const char* e = std::getenv("CPKIT_NN_M8");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0;
}
GemmPlan plan_gemm(long long M, long long K, int R, bool trans, long long fixed_kps = 0, int min_chunks = 8,
                   int wave_cap = 0) {
    GemmPlan p{};
    // rank split: one CTA column covers up to 208 ranks (26 n8 cells)
    p.ntiles = (R + 207) / 208;
    const int per = (R + p.ntiles - 1) / p.ntiles;  // ranks per CTA column
    p.nt8 = (per + 7) / 8;
    // Tile search: BM = 16 wm rows (wm in [4, 10]), nw in {8, 12} DMMA warps,
    // rank tile nt8p >= nt8 n8 cells (padding lets every warp own a full run).
    // Score = useful DMMA slots (cell dealing across sub-partitions, rank
    // padding) x row padding x wave quantisation (split-K counted), with a
    // preference for runs that stay in one row at full length (no second A
    // fragment, no spills). Measured at C2: TN 80 x 104 tiles on 8 warps
    // (two-row runs) 483 us vs 516 us for the former 64 x 112; NN 128 x 104
    // (full runs) 436 us, 64 x 112 (full) 450 us, 64 x 104 (two-row runs) 512 us.
    double best_score = -1.0;
    GemmPlan best = p;
    for (int wm = 4; wm <= 10; ++wm) {
        for (int nw : {4, 8, 12}) {
            for (int nt8p = p.nt8; nt8p <= p.nt8 + 4 && nt8p <= 26; ++nt8p) {
                GemmPlan c = p;
                c.wm = wm;
                c.nw = nw;
                c.nt8 = nt8p;
                c.maxc = round_maxc((wm * nt8p + nw - 1) / nw);
                if (c.maxc < 0 || !runs_fit(wm, nt8p, nw)) continue;
                if (32 * (nw + 1) > root_max_threads(c.maxc)) continue;  // register budget
                const bool full = runs_full(c);
                if (c.maxc >= 10 && !full) continue;  // the long two-row runs spill
                c.bns = bns_for(c.BN(), trans);
                c.stages = 2;
                for (int s = 6; s >= 2; --s) {
                    c.stages = s;
                    if (smem_bytes(c) <= 225 * 1024) break;
                }
                if (smem_bytes(c) > 225 * 1024) continue;
                c.per_sm = resident_per_sm(c);
                const long long mt = (M + c.BM() - 1) / c.BM();
                const double m_eff = static_cast<double>(M) / static_cast<double>(mt * c.BM());
                double w_eff = 1.0;
                if (fixed_kps > 0) {
                    const long long units = static_cast<long long>(c.ntiles) * mt * ((K + fixed_kps - 1) / fixed_kps);
                    const long long slots = static_cast<long long>(num_sms()) * c.per_sm;
                    w_eff = static_cast<double>(units) / static_cast<double>(((units + slots - 1) / slots) * slots);
                } else {
                    best_splits(static_cast<long long>(c.ntiles) * mt, static_cast<long long>(num_sms()) * c.per_sm,
                                K, &w_eff, min_chunks, wave_cap);
                }
                // four DMMA warps = one per SM sub-partition: ~0.93 of the two-per-SMSP
                // issue rate (tools/probe/probe_fp64.cu), only worth it to fill a wave
                const double score = cell_efficiency(wm, nt8p, nw) * (static_cast<double>(p.nt8) / nt8p) * m_eff *
                                     w_eff * (full ? 1.0 : trans ? 0.97 : 0.85) * (1.0 + 0.002 * wm) *
                                     (c.stages >= 3 ? 1.0 : 0.97) * (nw == 4 ? 0.93 : 1.0);
                if (const char* dbg = std::getenv("CPKIT_PLAN_DEBUG"))
                    if (std::atoi(dbg) >= 2)
                        std::fprintf(stderr, "  cand M=%lld wm=%d nw=%d nt8=%d maxc=%d full=%d stages=%d per_sm=%d w_eff=%.3f score=%.4f\n",
                                     M, wm, nw, nt8p, c.maxc, full ? 1 : 0, c.stages, c.per_sm, w_eff, score);
                if (score > best_score + 1e-12) {
                    best_score = score;
                    best = c;
                }
            }
        }
    }
    if (best_score < 0.0) {
        // no candidate (cannot happen for nt8 <= 26): eight warps, one full-length run each
        best.wm = p.nt8 > 16 ? 4 : 8;
        best.nw = 8;
        best.maxc = round_maxc(p.nt8 > 16 ? (p.nt8 + 1) / 2 : p.nt8);
        best.nt8 = p.nt8 > 16 ? 2 * best.maxc : best.maxc;
        best.bns = bns_for(best.BN(), trans);
        best.stages = 2;
        for (int s = 6; s >= 2; --s) {
            best.stages = s;
            if (smem_bytes(best) <= 225 * 1024) break;
        }
    }
    p = best;
    // tuning overrides (experiments only): CPKIT_{NN,TN}_{WM,NW,STAGES}
    auto env = [&](const char* key, int& v) {
        const std::string name = std::string(trans ? "CPKIT_TN_" : "CPKIT_NN_") + key;
        if (const char* e = std::getenv(name.c_str())) v = std::atoi(e);
    };
    const int wm0 = p.wm, nw0 = p.nw, nt0 = p.nt8;
    env("WM", p.wm);
    env("NW", p.nw);
    env("NT8", p.nt8);
    if (p.wm != wm0 || p.nw != nw0 || p.nt8 != nt0) {
        p.ntiles = (R + 8 * p.nt8 - 1) / (8 * p.nt8);  // narrower rank tiles: several CTA columns
        p.maxc = round_maxc((p.wm * p.nt8 + p.nw - 1) / p.nw);
        if (p.maxc < 0 || !runs_fit(p.wm, p.nt8, p.nw) || 32 * (p.nw + 1) > root_max_threads(p.maxc))
            throw DeviceError("CPKIT tile override: bad warp count");
        p.bns = bns_for(p.BN(), trans);
        p.stages = 2;
        for (int s = 6; s >= 2; --s) {
            p.stages = s;
            if (smem_bytes(p) <= 225 * 1024) break;
        }
    }
    env("STAGES", p.stages);
    p.m8 = false;
    p.rs = false;
    // row-split m16 dealing when the plan pads the rank to an even split of an
    // odd cell count (R = 8 NC, NC odd): NC cells per m16 row as MAXC + (MAXC-1)
    {
        const int nc = R / 8, mx = (nc + 1) / 2;
        if (!trans && fixed_kps == 0 && p.ntiles == 1 && R % 8 == 0 && (nc & 1) && nc >= 3 && round_maxc(mx) == mx &&
            8 * p.nt8 > R && rs_enabled()) {
            p.rs = true;
            p.wm = 4;
            p.nw = 8;
            p.nt8 = nc;
            p.maxc = mx;
            p.bns = bns_for(8 * nc, false);
            p.stages = 2;
            for (int st = 6; st >= 2; --st) {
                p.stages = st;
                if (smem_bytes(p) <= 225 * 1024) break;
            }
            env("STAGES", p.stages);
        }
    }
    // m8n8k4 variant (root_gemm_m8_kernel) when the m16n8k16 plan pads the rank:
    // an odd number of n8 cells, no padding (C5s, R = 200: roots 18.90 -> 18.68 ms)
    const int nc = R / 8;
    if (!p.rs && !trans && fixed_kps == 0 && p.ntiles == 1 && R % 8 == 0 && (nc & 1) && nc >= 13 && nc <= 31 &&
        8 * p.nt8 > R && m8_enabled()) {
        p.m8 = true;
        p.nw = kM8Warps;
        p.wm = kM8Warps / 2;  // BM = 8 nw
        p.nt8 = nc;
        p.maxc = nc;
        p.bns = bns_for(8 * nc, false);
        p.stages = 2;
        for (int st = 6; st >= 2; --st) {
            p.stages = st;
            if (smem_bytes(p) <= 225 * 1024) break;
        }
        env("STAGES", p.stages);
    }
    p.per_sm = resident_per_sm(p);
    p.mtiles = static_cast<int>((M + p.BM() - 1) / p.BM());
    const long long base = static_cast<long long>(p.ntiles) * p.mtiles;
    const long long slots = static_cast<long long>(num_sms()) * p.per_sm;
    if (fixed_kps > 0) {
        p.kps = fixed_kps;
    } else {
        const long long sp = best_splits(base, slots, K, nullptr, min_chunks, wave_cap);
        const long long kchunks = (K + kBK - 1) / kBK;
        p.kps = ((kchunks + sp - 1) / sp) * kBK;  // multiple of kBK: splits never share a stage
    }
    p.splits = static_cast<int>((K + p.kps - 1) / p.kps);
    if (std::getenv("CPKIT_PLAN_DEBUG"))
        std::fprintf(stderr, "plan %s M=%lld K=%lld R=%d: wm=%d nw=%d nt8=%d maxc=%d full=%d stages=%d splits=%d\n",
                     trans ? "TN" : "NN", M, K, R, p.wm, p.nw, p.nt8, p.maxc, runs_full(p) ? 1 : 0, p.stages,
                     p.splits);
    return p;
}

template <bool TRANS, bool GEN>
void dispatch(const GemmPlan& p, cudaStream_t st, const CUtensorMap& xmap, const CUtensorMap& kmap, const KrpDev& kd,
              long long M, long long K, int R, double* out, long long oss, int brel = 0, long long max_ctas = 0,
              double* sk_ws = nullptr) {
    const std::size_t smem = smem_bytes(p);
    const long long units = static_cast<long long>(p.ntiles) * p.mtiles * p.splits;
    long long cap = static_cast<long long>(num_sms()) * p.per_sm;
    if (max_ctas > 0) cap = std::min(cap, max_ctas);
    if (units >= (1LL << 31)) throw DeviceError("root GEMM: too many tile units");  // 32-bit unit indices in the kernel
    const int sk = sk_ws != nullptr ? 1 : 0;  // stream-K: exactly max_ctas CTAs share the k blocks
    dim3 grid(static_cast<unsigned>(sk ? cap : std::min<long long>(units, cap)));
    const dim3 block(32 * (p.nw + 1));
    if (!TRANS && !GEN && p.m8) {
#define CPK_M8(NCV)                                                                                     \
    case NCV: {                                                                                         \
        auto fn = root_gemm_m8_kernel<NCV>;                                                             \
        ensure_dynamic_smem(fn, smem);                                                                  \
        fn<<<grid, dim3(32 * (kM8Warps + 1)), smem, st>>>(xmap, kmap, M, K, R, p.bns, p.stages, p.kps,  \
                                                          p.splits, out, oss);                          \
        break;                                                                                          \
    }
        switch (p.nt8) {
            CPK_M8(13) CPK_M8(15) CPK_M8(17) CPK_M8(19) CPK_M8(21) CPK_M8(23) CPK_M8(25) CPK_M8(27) CPK_M8(29)
            CPK_M8(31)
            default: throw DeviceError("unsupported m8 rank tile");
        }
#undef CPK_M8
        count_launch(1);
        CPK_CUDA(cudaGetLastError());
        return;
    }
#define CPK_CASE(NTV)                                                                              \
    case NTV: {                                                                                    \
        auto fn = (!TRANS && !GEN && p.rs) ? root_gemm_kernel<NTV, TRANS, GEN, false, !TRANS && !GEN> \
                  : runs_full(p)           ? root_gemm_kernel<NTV, TRANS, GEN, true>              \
                                           : root_gemm_kernel<NTV, TRANS, GEN, false>;             \
        if (sk) /* stream-K instantiations exist for the NN kernel without RS only (plan_streamk) */ \
            fn = runs_full(p) ? root_gemm_kernel<NTV, TRANS, GEN, true, false, !TRANS && !GEN>     \
                              : root_gemm_kernel<NTV, TRANS, GEN, false, false, !TRANS && !GEN>;   \
        ensure_dynamic_smem(fn, smem);                                                             \
        if (std::getenv("CPKIT_GRID_OCC")) { /* experiments: grid from the real occupancy */        \
            int occ = 1;                                                                           \
            CPK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, static_cast<int>(block.x), smem)); \
            grid.x = static_cast<unsigned>(std::min<long long>(units, static_cast<long long>(num_sms()) * std::max(occ, 1))); \
        }                                                                                          \
        fn<<<grid, block, smem, st>>>(xmap, kmap, kd, M, K, R, p.BM(), p.BN(), p.nw, p.bns, p.stages, p.kps,  \
                                      p.splits, out, oss, brel, sk_ws);                            \
        break;                                                                                     \
    }
    switch (p.maxc) {
        CPK_CASE(1) CPK_CASE(2) CPK_CASE(3) CPK_CASE(4) CPK_CASE(5) CPK_CASE(6) CPK_CASE(7)
        CPK_CASE(8) CPK_CASE(9) CPK_CASE(10) CPK_CASE(12) CPK_CASE(13) CPK_CASE(16)
        default: throw DeviceError("unsupported rank tile");
    }
#undef CPK_CASE
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

// Fill the KRP operand (K x Rs, Rs = R rounded to even) for a contraction.
void fill_krp(const KrpDesc& kd, long long K, int R, double* krp, cudaStream_t st) {
    const int Rs = (R + 1) & ~1;
    if (kd.nmodes == 2 && K * (Rs / 2) < (1LL << 31) && !std::getenv("CPKIT_KRP_FILL_GENERIC")) {
        const unsigned P2 = static_cast<unsigned>(Rs / 2);
        const unsigned long long total = static_cast<unsigned long long>(K) * P2;
        const int blocks = static_cast<int>(std::min<unsigned long long>((total + 1023) / 1024, 8ULL * num_sms()));
        krp_fill2_kernel<<<blocks, 256, 0, st>>>(kd.fac[0], kd.fac[1], static_cast<unsigned>(kd.ext[1]),
                                                 static_cast<unsigned>(K), R, P2, reinterpret_cast<double2*>(krp));
        count_launch(1);
        CPK_CUDA(cudaGetLastError());
        return;
    }
    const int blocks = static_cast<int>(std::min<long long>((K + 7) / 8, 16LL * num_sms()));
    krp_fill_kernel<<<blocks, 256, 0, st>>>(to_dev(kd), K, R, Rs, krp);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

// Wave-quantisation tail of an unsplit NN root: the rows of the full waves
// run as one launch, the last partial wave's rows as a second launch split
// over k (its own plan, >= 3 k-stages per split) and reduced in fixed order.
// The kernel itself is unchanged. rows_main == M: no tail launch.
// reserve_sms: SMs left to a concurrent side-stream kernel (the SPD
// factorisation beside an ALS/GN root) while the full waves run.
struct BackSplit {
    GemmPlan main, tail;
    long long rows_main, main_ctas;
};
BackSplit plan_back(long long M, long long K, int R, int reserve_sms) {
    BackSplit b;
    b.main = plan_gemm(M, K, R, false);
    b.rows_main = M;
    b.main_ctas = 0;
    const GemmPlan& p = b.main;
    if (p.splits != 1 || p.ntiles != 1 || std::getenv("CPKIT_NO_TAIL_LAUNCH")) return b;
    const long long slots = static_cast<long long>(num_sms() - reserve_sms) * p.per_sm;
    const long long all_slots = static_cast<long long>(num_sms()) * p.per_sm;  // the tail runs after: every SM
    const long long units = p.mtiles;
    const long long rem = units % slots;
    if (units <= slots || rem == 0 || 2 * rem > all_slots) return b;
    const long long rows_main = (units - rem) * p.BM();
    GemmPlan tail = plan_gemm(M - rows_main, K, R, false, 0, 3, 1);  // one wave at most
    // the tail must fill (at most) one wave: smaller tiles or a k split
    if (static_cast<long long>(tail.ntiles) * tail.mtiles * tail.splits > all_slots) return b;
    if (tail.splits < 2 && tail.BM() >= p.BM()) return b;  // no smaller tiles and no split: nothing gained
    b.main = plan_gemm(rows_main, K, R, false);
    b.tail = tail;
    b.rows_main = rows_main;
    b.main_ctas = slots;
    return b;
}

// Stream-K plan for an NN root (launch_root_back): the unsplit plan's tile on
// exactly (SMs - reserve) CTAs. Used when the row tiles do not fill one wave
// (the case that otherwise needs a k split into full-size slabs);
// CPKIT_NO_STREAMK=1 keeps that.
struct StreamK {
    bool on = false;
    GemmPlan plan{};
    int ctas = 0;
    std::size_t ws_elems = 0;
};
StreamK plan_streamk(long long M, long long K, int R, int reserve_sms) {
    StreamK sk;
    static const bool off = std::getenv("CPKIT_NO_STREAMK") != nullptr;
    if (off) return sk;
    GemmPlan p = plan_gemm(M, K, R, false);
    if (p.m8 || p.rs || p.ntiles != 1 || p.per_sm != 1) return sk;
    const int ctas = num_sms() - reserve_sms;
    const long long kblocks = (K + kBK - 1) / kBK;
    if (ctas < 2) return sk;
    // Measured: it pays where the unsplit plan has fewer row tiles than CTAs and
    // would otherwise split k into full-size slabs (C4: 79 tiles, ALS sweep
    // 0.860 -> 0.845 ms). With several waves of tiles the tail launch stays: at
    // C5s the root alone gains (18.15 -> 17.97 ms) but inside a sweep, where one
    // SM is left to the side-stream factorisation during the whole launch
    // instead of only during the full waves, the sweep loses (36.53 -> 36.64 ms);
    // short contractions lose outright (C2, 13 k blocks per tile: nearly every
    // CTA ends inside a tile, back root 457 vs 408 us).
    if (p.splits < 2 || kblocks < 128) return sk;
    if (p.mtiles * kblocks < 8LL * ctas) return sk;               // under 8 k blocks per CTA: too little to cut
    if (ctas / p.mtiles + 2 > kStreamKMaxPieces) return sk;        // the fix-up's piece list
    p.splits = 1;
    p.kps = kblocks * kBK;
    sk.on = true;
    sk.plan = p;
    sk.ctas = ctas;
    sk.ws_elems = 2ull * static_cast<std::size_t>(num_sms()) * p.BM() * R;
    if (std::getenv("CPKIT_PLAN_DEBUG"))
        std::fprintf(stderr, "plan stream-K NN M=%lld K=%lld R=%d: %d row tiles x %lld k blocks over %d CTAs\n", M, K, R,
                     p.mtiles, kblocks, ctas);
    return sk;
}

}  // namespace

std::size_t root_back_workspace_elems_classic(std::int64_t F, std::int64_t B, int R);
std::size_t krp_workspace_elems(std::int64_t rows, int R) {
    return static_cast<std::size_t>(rows) * ((R + 1) & ~1);
}

// X is F x Bs row-major (Bs >= B, Bs even: the padded row stride).
void launch_root_back(const double* x, std::int64_t F, std::int64_t B, std::int64_t Bs, int R,
                      const KrpDesc& kb, double* krp, double* pf, double* ws, std::size_t ws_elems,
                      cudaStream_t st, int reserve_sms) {
    {  // stream-K: one launch, every CTA the same number of k blocks
        StreamK sk = plan_streamk(F, B, R, reserve_sms);
        if (sk.on && ws_elems >= sk.ws_elems) {
            const int Rs = (R + 1) & ~1;
            const bool direct = kb.nmodes == 1 && R % 2 == 0;
            if (!direct) fill_krp(kb, B, R, krp, st);
            const CUtensorMap xmap = make_map(x, static_cast<std::uint64_t>(Bs), static_cast<std::uint64_t>(F), 16,
                                              static_cast<std::uint32_t>(sk.plan.BM()), true);
            const CUtensorMap kmap = make_map(direct ? kb.fac[0] : krp, static_cast<std::uint64_t>(Rs),
                                              static_cast<std::uint64_t>(B), static_cast<std::uint32_t>(sk.plan.bns),
                                              kBK, false);
            dispatch<false, false>(sk.plan, st, xmap, kmap, to_dev(kb), F, B, R, pf, 0, 0, sk.ctas, ws);
            streamk_fixup_kernel<<<sk.ctas - 1, 256, 0, st>>>(ws, pf, F, R, sk.plan.BM(), sk.plan.mtiles,
                                                              (B + kBK - 1) / kBK, sk.ctas);
            count_launch(1);
            CPK_CUDA(cudaGetLastError());
            return;
        }
    }
    const BackSplit bs = plan_back(F, B, R, reserve_sms);
    if (bs.rows_main < F &&
        (bs.tail.splits < 2 || ws_elems >= static_cast<std::size_t>(bs.tail.splits) * (F - bs.rows_main) * R)) {
        const int Rs2 = (R + 1) & ~1;
        const bool direct2 = kb.nmodes == 1 && R % 2 == 0;
        if (!direct2) fill_krp(kb, B, R, krp, st);
        const CUtensorMap kmap = make_map(direct2 ? kb.fac[0] : krp, static_cast<std::uint64_t>(Rs2),
                                          static_cast<std::uint64_t>(B), static_cast<std::uint32_t>(bs.main.bns), kBK,
                                          false);
        // full waves: rows [0, rows_main)
        const CUtensorMap xmap = make_map(x, static_cast<std::uint64_t>(Bs), static_cast<std::uint64_t>(bs.rows_main),
                                          16, static_cast<std::uint32_t>(bs.main.BM()), true);
        dispatch<false, false>(bs.main, st, xmap, kmap, to_dev(kb), bs.rows_main, B, R, pf, 0, 0, bs.main_ctas);
        // tail rows, split over k into the workspace, then the fixed-order reduce
        const long long mt = F - bs.rows_main;
        const CUtensorMap xmap_t = make_map(x + bs.rows_main * Bs, static_cast<std::uint64_t>(Bs),
                                            static_cast<std::uint64_t>(mt), 16,
                                            static_cast<std::uint32_t>(bs.tail.BM()), true);
        const CUtensorMap kmap_t = bs.tail.bns == bs.main.bns
                                       ? kmap
                                       : make_map(direct2 ? kb.fac[0] : krp, static_cast<std::uint64_t>(Rs2),
                                                  static_cast<std::uint64_t>(B),
                                                  static_cast<std::uint32_t>(bs.tail.bns), kBK, false);
        if (bs.tail.splits < 2) {  // smaller tiles fill the wave: straight into the output rows
            dispatch<false, false>(bs.tail, st, xmap_t, kmap_t, to_dev(kb), mt, B, R, pf + bs.rows_main * R, 0);
            return;
        }
        dispatch<false, false>(bs.tail, st, xmap_t, kmap_t, to_dev(kb), mt, B, R, ws, mt * R);
        const long long n = mt * static_cast<long long>(R);
        const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 4LL * num_sms()));
        splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, bs.tail.splits, n, pf + bs.rows_main * R);
        count_launch(1);
        CPK_CUDA(cudaGetLastError());
        return;
    }
    const GemmPlan& p = bs.main;
    const int Rs = (R + 1) & ~1;
    // a one-mode Khatri-Rao operand is the factor itself: map it directly (R even:
    // 16-byte row stride), no workspace fill
    const bool direct = kb.nmodes == 1 && R % 2 == 0;
    if (!direct) fill_krp(kb, B, R, krp, st);
    const CUtensorMap xmap = make_map(x, static_cast<std::uint64_t>(Bs), static_cast<std::uint64_t>(F), 16,
                                      static_cast<std::uint32_t>(p.BM()), true);
    const CUtensorMap kmap = make_map(direct ? kb.fac[0] : krp, static_cast<std::uint64_t>(Rs),
                                      static_cast<std::uint64_t>(B), static_cast<std::uint32_t>(p.bns), kBK, false);
    double* out = pf;
    long long oss = 0;
    if (p.splits > 1) {
        if (ws_elems < static_cast<std::size_t>(p.splits) * F * R)
            throw DeviceError("root_back: split-K workspace too small");
        out = ws;
        oss = F * R;
    }
    dispatch<false, false>(p, st, xmap, kmap, to_dev(kb), F, B, R, out, oss);
    if (p.splits > 1) {
        const long long n = F * static_cast<long long>(R);
        const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 4LL * num_sms()));
        splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, p.splits, n, pf);
        count_launch(1);
        CPK_CUDA(cudaGetLastError());
    }
}

std::size_t root_back_workspace_elems(std::int64_t F, std::int64_t B, int R) {
    return std::max(root_back_workspace_elems_classic(F, B, R), plan_streamk(F, B, R, 0).ws_elems);
}
std::size_t root_back_workspace_elems_classic(std::int64_t F, std::int64_t B, int R) {
    std::size_t w = 0;
    for (int reserve = 0; reserve <= 1; ++reserve) {
        const BackSplit bs = plan_back(F, B, R, reserve);
        if (bs.rows_main < F && bs.tail.splits > 1)
            w = std::max<std::size_t>(w, static_cast<std::size_t>(bs.tail.splits) * (F - bs.rows_main) * R);
    }
    if (w) return w;
    const BackSplit bs = plan_back(F, B, R, 0);
    if (bs.rows_main < F) return bs.tail.splits > 1 ? static_cast<std::size_t>(bs.tail.splits) * (F - bs.rows_main) * R : 0;
    const GemmPlan& p = bs.main;
    return p.splits > 1 ? static_cast<std::size_t>(p.splits) * F * R : 0;
}

std::size_t root_front_workspace_elems(std::int64_t F, std::int64_t B, int R) {
    const GemmPlan p = plan_gemm(B, F, R, true);
    return p.splits > 1 ? static_cast<std::size_t>(p.splits) * B * R : 0;
}

void launch_root_front(const double* x, std::int64_t F, std::int64_t B, std::int64_t Bs, int R,
                       const KrpDesc& kf, double* krp, double* pb, double* ws, std::size_t ws_elems,
                       cudaStream_t st) {
    const GemmPlan p = plan_gemm(B, F, R, true);
    const int Rs = (R + 1) & ~1;
    // the Khatri-Rao operand is generated inside the GEMM's producer warp
    // (no K x R workspace round trip) unless the rank tile is too wide for it
    // Optional (CPKIT_KRP_GENERATE=1): form the two-mode Khatri-Rao operand inside
    // the GEMM (A_1 rows by TMA, scaled by the A_0 row in shared memory by the
    // producer warp) instead of materialising it. Measured at C2: 580 us vs
    // 554 us fill + GEMM (the single producer warp starves the DMMA warps, 69%
    // vs 81% pipe activity), so the materialised operand stays the default.
    const bool gen = kf.nmodes == 2 && R % 2 == 0 && kf.ext[1] % 16 == 0 && p.BN() <= 128 &&
                     std::getenv("CPKIT_KRP_GENERATE");
    const bool direct = kf.nmodes == 1 && R % 2 == 0;  // the factor itself (order-2 tensors)
    if (!gen && !direct) fill_krp(kf, F, R, krp, st);
    const CUtensorMap xmap = make_map(x, static_cast<std::uint64_t>(Bs), static_cast<std::uint64_t>(F), 16, kBK,
                                      true);
    const CUtensorMap kmap =
        gen ? make_map(kf.fac[1], static_cast<std::uint64_t>(R), static_cast<std::uint64_t>(kf.ext[1]),
                       static_cast<std::uint32_t>(p.bns), 16, false)
            : make_map(direct ? kf.fac[0] : krp, static_cast<std::uint64_t>(Rs), static_cast<std::uint64_t>(F),
                       static_cast<std::uint32_t>(p.bns), kBK, false);
    double* out = pb;
    long long oss = 0;
    if (p.splits > 1) {
        if (ws_elems < static_cast<std::size_t>(p.splits) * B * R)
            throw DeviceError("root_front: split-K workspace too small");
        out = ws;
        oss = B * R;
    }
    if (gen) dispatch<true, true>(p, st, xmap, kmap, to_dev(kf), B, F, R, out, oss);
    else dispatch<true, false>(p, st, xmap, kmap, to_dev(kf), B, F, R, out, oss);
    if (p.splits > 1) {
        const long long n = B * static_cast<long long>(R);
        const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 4LL * num_sms()));
        splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, p.splits, n, pb);
        count_launch(1);
        CPK_CUDA(cudaGetLastError());
    }
}

// ---------------------------------------------------------------- layout
// Batched 2-D transpose: out[b][c][r] = in[b][r][c] for r < rows, c < cols.
// Builds the mode-permuted tensor copies of the order-3 multi-sweep tree
// (X^(0)[i1][i2][i0], X^(1)[i0][i2][i1]) once per tensor upload, so every
// single-mode root is the same NN GEMM as the back root. 32 x 32 tiles staged
// through shared memory: both the reads and the writes are row-coalesced.
namespace {
__global__ void __launch_bounds__(256) transpose_batched_kernel(const double* __restrict__ in, long long rows,
                                                                long long cols, long long in_ld, long long in_bs,
                                                                double* __restrict__ out, long long out_ld,
                                                                long long out_bs, long long batch) {
    __shared__ double tile[32][33];
    const long long c0 = static_cast<long long>(blockIdx.x) * 32, r0 = static_cast<long long>(blockIdx.y) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (long long b = blockIdx.z; b < batch; b += gridDim.z) {
        const double* src = in + b * in_bs;
        double* dst = out + b * out_bs;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            const long long r = r0 + ty + j, c = c0 + tx;
            tile[ty + j][tx] = (r < rows && c < cols) ? __ldcs(src + r * in_ld + c) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            const long long c = c0 + ty + j, r = r0 + tx;
            if (r < rows && c < cols) dst[c * out_ld + r] = tile[tx][ty + j];
        }
        __syncthreads();
    }
}
}  // namespace

void launch_transpose_batched(const double* in, std::int64_t batch, std::int64_t rows, std::int64_t cols,
                              std::int64_t in_ld, std::int64_t in_bs, double* out, std::int64_t out_ld,
                              std::int64_t out_bs, cudaStream_t st) {
    if (batch <= 0 || rows <= 0 || cols <= 0) return;
    const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32),
                    static_cast<unsigned>(std::min<long long>(batch, 65535)));
    transpose_batched_kernel<<<grid, 256, 0, st>>>(in, rows, cols, in_ld, in_bs, out, out_ld, out_bs, batch);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

// Single-mode roots of the order-3 multi-sweep dimension tree: contract ONE
// mode c < 2 of X [s0][s1][Bs] with its factor as a TN GEMM whose B operand
// is the factor itself (no Khatri-Rao operand, nothing to fill):
//   c = 0: P_0[(i1, i2)][r] = sum_i0 X[i0][(i1, i2)] A_0[i0][r]  (X viewed as s0 x s1 Bs)
//   c = 1: P_1[i0][i2][r]   = sum_i1 X[(i0, i1)][i2] A_1[i1][r]  (s0 batches of s1 rows:
//          split i0 is batch i0, its B rows restart at A_1 row 0 and its
//          output is slab i0; a stage running past s1 meets TMA zero rows of A_1)
// These are the reference's own first contraction steps (contract_mode,
// mttkrp.cpp:46-62) for a mode other than the last.
std::size_t root_single_workspace_elems(std::int64_t s0, std::int64_t s1, std::int64_t Bs, int R) {
    const GemmPlan p = plan_gemm(s1 * Bs, s0, R, true);
    return p.splits > 1 ? static_cast<std::size_t>(p.splits) * s1 * Bs * R : 0;
}

void launch_root_single(const double* x, std::int64_t s0, std::int64_t s1, std::int64_t Bl, std::int64_t Bs, int c,
                        const double* fac, int R, double* out, double* ws, std::size_t ws_elems, cudaStream_t st) {
    if (R % 2 != 0) throw DeviceError("root_single: the factor is the B operand and needs an even rank");
    if (c == 0) {
        const long long M = s1 * Bs, K = s0;
        const GemmPlan p = plan_gemm(M, K, R, true);
        const CUtensorMap xmap = make_map(x, static_cast<std::uint64_t>(M), static_cast<std::uint64_t>(K), 16, kBK, true);
        const CUtensorMap kmap = make_map(fac, static_cast<std::uint64_t>(R), static_cast<std::uint64_t>(s0),
                                          static_cast<std::uint32_t>(p.bns), kBK, false);
        double* o = out;
        long long oss = 0;
        if (p.splits > 1) {
            if (ws_elems < static_cast<std::size_t>(p.splits) * M * R) throw DeviceError("root_single: workspace too small");
            o = ws;
            oss = M * R;
        }
        dispatch<true, false>(p, st, xmap, kmap, KrpDev{}, M, K, R, o, oss);
        if (p.splits > 1) {
            const long long n = M * static_cast<long long>(R);
            const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 4LL * num_sms()));
            splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, p.splits, n, out);
            count_launch(1);
            CPK_CUDA(cudaGetLastError());
        }
    } else if (c == 1) {
        const long long K = s0 * s1;
        const GemmPlan p = plan_gemm(Bl, K, R, true, s1);
        const CUtensorMap xmap = make_map(x, static_cast<std::uint64_t>(Bs), static_cast<std::uint64_t>(K), 16, kBK, true);
        const CUtensorMap kmap = make_map(fac, static_cast<std::uint64_t>(R), static_cast<std::uint64_t>(s1),
                                          static_cast<std::uint32_t>(p.bns), kBK, false);
        dispatch<true, false>(p, st, xmap, kmap, KrpDev{}, Bl, K, R, out, Bl * static_cast<long long>(R), 1);
    } else {
        throw DeviceError("root_single: mode must be 0 or 1");
    }
}

// ---------------------------------------------------------------- second level
// out[i, r] = sum over all other kept indices of P[idx, r] * prod_{l != keep} A_l[idx_l, r]
// (the descending mode-at-a-time contraction of mttkrp.cpp:118-126/:63-75,
// done in one pass). P is [outer][s_keep][inner][R]. HBM-bound: one CTA per
// (i, split), threads over (q-lane, r) with 4 independent loads in flight
// each; q-lanes and splits are combined in a fixed order (deterministic).
namespace {
constexpr int kRedT = 256;
__device__ __forceinline__ double kept_weight(const KrpDev& kd, int keep, long long o, long long in, int r,
                                              int R) {
    double w = 1.0;
    long long rem = in;
    for (int l = kd.nmodes - 1; l > keep; --l) {
        const long long e = kd.ext[l];
        w *= kd.fac[l][(rem % e) * R + r];
        rem /= e;
    }
    rem = o;
    for (int l = keep - 1; l >= 0; --l) {
        const long long e = kd.ext[l];
        w *= kd.fac[l][(rem % e) * R + r];
        rem /= e;
    }
    return w;
}
// Each thread owns VW consecutive rank columns (16-byte loads when R is even)
// and walks its q-lane with 4 independent loads in flight.
template <int VW>
__global__ void __launch_bounds__(kRedT, 3) reduce_kept_kernel(const double* __restrict__ p, KrpDev kd, int keep,
                                                             int R, long long outer, long long sk, long long inner,
                                                             int splits, double* __restrict__ out,
                                                             long long out_split_stride) {
    __shared__ double red[kRedT * VW];
    const long long i = blockIdx.x;
    const int split = blockIdx.y;
    const int cols = (R + VW - 1) / VW;  // threads needed per q-lane
    const int cpad = min(kRedT, ((cols + 31) / 32) * 32);
    const int qlanes = kRedT / cpad;
    const int ql = threadIdx.x / cpad;
    const int cc = threadIdx.x % cpad;
    const long long total = outer * inner;
    const long long per = (total + splits - 1) / splits;
    const long long lo = split * per, hi = min(total, lo + per);
    const bool two = kd.nmodes == 2;
    const double* wfac = two ? kd.fac[keep == 0 ? 1 : 0] : nullptr;
    for (int c0 = 0; c0 < cols; c0 += cpad) {
        const int r = (c0 + cc) * VW;
        double acc[VW];
#pragma unroll
        for (int v = 0; v < VW; ++v) acc[v] = 0.0;
        if (r < R) {
            const long long step_o = qlanes / inner, step_in = qlanes % inner;
            long long q = lo + ql;
            long long o = q / inner, in = q % inner;
            auto load = [&](long long oo, long long ii, double* pv, double* wv) {
                const double* src = p + ((oo * sk + i) * inner + ii) * R + r;
                if (VW == 2) {
                    const double2 t2 = __ldcs(reinterpret_cast<const double2*>(src));
                    pv[0] = t2.x;
                    pv[VW - 1] = t2.y;
                } else {
                    pv[0] = __ldcs(src);
                }
                if (two && VW == 2) {
                    const double2 w2 = __ldg(reinterpret_cast<const double2*>(wfac + (keep == 0 ? ii : oo) * R + r));
                    wv[0] = w2.x;
                    wv[VW - 1] = w2.y;
                } else {
#pragma unroll
                    for (int v = 0; v < VW; ++v)
                        wv[v] = two ? __ldg(wfac + (keep == 0 ? ii : oo) * R + r + v) : kept_weight(kd, keep, oo, ii, r + v, R);
                }
            };
            // four independent loads in flight per thread
            for (; q + 3 * qlanes < hi; q += 4 * qlanes) {
                long long o1 = o, i1 = in;
                i1 += step_in; o1 += step_o; if (i1 >= inner) { i1 -= inner; ++o1; }
                long long o2 = o1, i2 = i1;
                i2 += step_in; o2 += step_o; if (i2 >= inner) { i2 -= inner; ++o2; }
                long long o3 = o2, i3 = i2;
                i3 += step_in; o3 += step_o; if (i3 >= inner) { i3 -= inner; ++o3; }
                double p0[VW], p1[VW], p2[VW], p3[VW], w0[VW], w1[VW], w2[VW], w3[VW];
                load(o, in, p0, w0);
                load(o1, i1, p1, w1);
                load(o2, i2, p2, w2);
                load(o3, i3, p3, w3);
#pragma unroll
                for (int v = 0; v < VW; ++v) acc[v] += p0[v] * w0[v] + p1[v] * w1[v] + p2[v] * w2[v] + p3[v] * w3[v];
                o = o3; in = i3;
                in += step_in; o += step_o; if (in >= inner) { in -= inner; ++o; }
            }
            for (; q < hi; q += qlanes) {
                double p0[VW], w0[VW];
                load(o, in, p0, w0);
#pragma unroll
                for (int v = 0; v < VW; ++v) acc[v] += p0[v] * w0[v];
                in += step_in; o += step_o; if (in >= inner) { in -= inner; ++o; }
            }
        }
#pragma unroll
        for (int v = 0; v < VW; ++v) red[v * kRedT + threadIdx.x] = acc[v];
        __syncthreads();
        if (threadIdx.x < cpad && r < R) {
#pragma unroll
            for (int v = 0; v < VW; ++v) {
                double sum = 0.0;
                for (int l = 0; l < qlanes; ++l) sum += red[v * kRedT + l * cpad + threadIdx.x];
                out[split * out_split_stride + i * R + r + v] = sum;
            }
        }
        __syncthreads();
    }
}
// Two kept modes (order 3 and 4 roots): out[i, r] = sum_q P[base_i + q * stride, r] * W[q, r]
// (keep = 0: rows q of slab i are contiguous; keep = 1: rows are sk apart),
// 16-byte loads, 8 rows in flight per thread, q-lanes combined in fixed order.
__global__ void __launch_bounds__(kRedT, 3) reduce_two_kernel(const double* __restrict__ p,
                                                            const double* __restrict__ w, int R, long long base_step,
                                                            long long stride, long long rows, int splits,
                                                            double* __restrict__ out, long long out_split_stride) {
    __shared__ double2 red[kRedT];
    const long long i = blockIdx.x;
    const int split = blockIdx.y;
    const int pairs = R / 2;
    const int cpad = min(kRedT, ((pairs + 31) / 32) * 32);
    const int qlanes = kRedT / cpad;
    const int ql = threadIdx.x / cpad, cc = threadIdx.x % cpad;
    const long long per = (rows + splits - 1) / splits;
    const long long lo = split * per, hi = min(rows, lo + per);
    const double* src0 = p + i * base_step;
    for (int c0 = 0; c0 < pairs; c0 += cpad) {
        const int c = c0 + cc;
        double2 acc = make_double2(0.0, 0.0);
        if (c < pairs) {
            const double2* ps = reinterpret_cast<const double2*>(src0) + c;
            const double2* ws = reinterpret_cast<const double2*>(w) + c;
            const long long ps_step = stride / 2, ws_step = R / 2;
            long long q = lo + ql;
            for (; q + 7 * qlanes < hi; q += 8 * qlanes) {
                double2 pv[8], wv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const long long qq = q + u * qlanes;
                    pv[u] = __ldcs(ps + qq * ps_step);
                    wv[u] = __ldg(ws + qq * ws_step);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc.x += pv[u].x * wv[u].x;
                    acc.y += pv[u].y * wv[u].y;
                }
            }
            for (; q < hi; q += qlanes) {
                const double2 pv = __ldcs(ps + q * ps_step), wv = __ldg(ws + q * ws_step);
                acc.x += pv.x * wv.x;
                acc.y += pv.y * wv.y;
            }
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < cpad && c < pairs) {
            double2 sum = make_double2(0.0, 0.0);
            for (int l = 0; l < qlanes; ++l) {
                sum.x += red[l * cpad + threadIdx.x].x;
                sum.y += red[l * cpad + threadIdx.x].y;
            }
            *reinterpret_cast<double2*>(out + split * out_split_stride + i * R + 2 * c) = sum;
        }
        __syncthreads();
    }
}

int reduce_splits(const KrpDesc& kept, int keep) {
    const long long sk = kept.ext[keep];
    long long total = 1;
    for (int l = 0; l < kept.nmodes; ++l)
        if (l != keep) total *= kept.ext[l];
    // CTAs = sk * s; prefer an s that fills whole waves of 3 resident CTAs per SM
    const long long wave = 3LL * num_sms();
    if (kept.nmodes == 2 && sk >= num_sms() && !std::getenv("CPKIT_REDUCE_SPLITS")) return 1;  // measured best (C2)
    const long long smax = std::max<long long>(1, total / 32);
    if (const char* e = std::getenv("CPKIT_REDUCE_SPLITS"))
        if (std::atoll(e) > 0) return static_cast<int>(std::min<long long>(smax, std::atoll(e)));
    long long best = 1;
    double best_eff = -1.0;
    for (long long s = 1; s <= std::min<long long>(smax, 64); ++s) {
        const long long ctas = sk * s;
        if (ctas < wave && s < smax && sk * (s + 1) <= 4 * wave) continue;  // at least one full wave when possible
        const long long waves = (ctas + wave - 1) / wave;
        const double eff = static_cast<double>(ctas) / static_cast<double>(waves * wave);
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = s;
        }
        if (ctas >= 4 * wave) break;
    }
    return static_cast<int>(best);
}
}  // namespace

std::size_t reduce_kept_workspace_elems(const KrpDesc& kept, int keep, int R) {
    const int s = reduce_splits(kept, keep);
    return s > 1 ? static_cast<std::size_t>(s) * kept.ext[keep] * R : 0;
}

void launch_reduce_kept(const double* p, const KrpDesc& kept, int keep, int R, double* out, double* ws,
                        std::size_t ws_elems, cudaStream_t st) {
    long long outer = 1, inner = 1;
    for (int l = 0; l < keep; ++l) outer *= kept.ext[l];
    for (int l = keep + 1; l < kept.nmodes; ++l) inner *= kept.ext[l];
    const long long sk = kept.ext[keep];
    const int splits = reduce_splits(kept, keep);
    double* dst = out;
    if (splits > 1) {
        if (ws_elems < static_cast<std::size_t>(splits) * sk * R) throw DeviceError("reduce_kept: workspace too small");
        dst = ws;
    }
    dim3 grid(static_cast<unsigned>(sk), splits);
    if (kept.nmodes == 2 && R % 2 == 0 && !std::getenv("CPKIT_REDUCE_GENERIC")) {
        // keep 0: row (i, j) at (i * inner + j) R, weight A_1[j]; keep 1: row (o, i) at (o * sk + i) R, weight A_0[o]
        const long long base_step = keep == 0 ? inner * R : R;
        const long long stride = keep == 0 ? R : sk * R;
        const long long rows = keep == 0 ? inner : outer;
        reduce_two_kernel<<<grid, kRedT, 0, st>>>(p, kept.fac[keep == 0 ? 1 : 0], R, base_step, stride, rows, splits,
                                                  dst, sk * R);
    } else if (R % 2 == 0)
        reduce_kept_kernel<2><<<grid, kRedT, 0, st>>>(p, to_dev(kept), keep, R, outer, sk, inner, splits, dst, sk * R);
    else
        reduce_kept_kernel<1><<<grid, kRedT, 0, st>>>(p, to_dev(kept), keep, R, outer, sk, inner, splits, dst, sk * R);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
    if (splits > 1) {
        const long long n = sk * R;
        splitk_reduce_kernel<<<static_cast<int>(std::min<long long>((n + 255) / 256, 1024)), 256, 0, st>>>(ws, splits,
                                                                                                           n, out);
        count_launch(1);
        CPK_CUDA(cudaGetLastError());
    }
}

}  // namespace cpkit
