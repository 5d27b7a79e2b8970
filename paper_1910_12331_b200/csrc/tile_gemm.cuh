// DMMA 32x32 tile GEMM building block shared by the CG phases and the small
// dense kernels (Gram, gradient). 256 threads = 8 warps (2 x m16, 4 x n8).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace cpkit {
namespace tile {

constexpr int kT = 32;        // task tile edge
constexpr int kKC = 16;       // k chunk
constexpr int kThreads = 256;  // 8 warps: 2 (m16) x 4 (n8)
constexpr int kAS = kKC + 4;  // A smem row stride (doubles): conflict-free a-fragments
constexpr int kBS = kT + 8;   // B smem row stride

__device__ __forceinline__ void dmma16816(double* d, const double* a, const double* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},"
        "{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

struct RedSmem {
    double red[kThreads / 32 * 4];
    double bcast[8];
};
struct Smem {
    double As[2][kT * kAS];
    double Bs[2][kKC * kBS];
    double red[kThreads / 32 * 4];
    double bcast[8];
};

// C[32x32] tile = sum_{k<K} LA(row, k) * LB(k, col); rows/cols are tile-local.
// Each of the 8 warps owns a 16x8 sub-tile; acc[4] holds (g, 2t..2t+1),
// (g+8, 2t..2t+1). Operands are staged through double-buffered smem with the
// next chunk prefetched into registers while the current one is multiplied.
template <typename LA, typename LB>
__device__ __forceinline__ void tile_gemm(Smem& sm, int K, LA la, LB lb, double acc[4]) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 2) * 16, wn = (warp & 3) * 8;
    acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    const int nch = (K + kKC - 1) / kKC;
    // element assignment: A chunk 32x16 = 512 -> 2 per thread; B chunk 16x32 -> 2
    const int ar0 = tid >> 4, ac0 = tid & 15;            // rows 0..15
    const int ar1 = ar0 + 16;                            // rows 16..31
    const int bk0 = tid >> 5, bc0 = tid & 31;            // k 0..7
    const int bk1 = bk0 + 8;                             // k 8..15
    double pa0, pa1, pb0, pb1;
    auto fetch = [&](int c) {
        const int k0 = c * kKC;
        pa0 = (k0 + ac0 < K) ? la(ar0, k0 + ac0) : 0.0;
        pa1 = (k0 + ac0 < K) ? la(ar1, k0 + ac0) : 0.0;
        pb0 = (k0 + bk0 < K) ? lb(k0 + bk0, bc0) : 0.0;
        pb1 = (k0 + bk1 < K) ? lb(k0 + bk1, bc0) : 0.0;
    };
    auto stash = [&](int buf) {
        sm.As[buf][ar0 * kAS + ac0] = pa0;
        sm.As[buf][ar1 * kAS + ac0] = pa1;
        sm.Bs[buf][bk0 * kBS + bc0] = pb0;
        sm.Bs[buf][bk1 * kBS + bc0] = pb1;
    };
    if (nch > 0) {
        fetch(0);
        stash(0);
    }
    __syncthreads();
    for (int c = 0; c < nch; ++c) {
        const int buf = c & 1;
        if (c + 1 < nch) fetch(c + 1);
        double a[8], b[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = sm.As[buf][(wm + g + 8 * (i & 1)) * kAS + t + 4 * (i >> 1)];
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = sm.Bs[buf][(t + 4 * i) * kBS + wn + g];
        dmma16816(acc, a, b);
        if (c + 1 < nch) stash(buf ^ 1);
        __syncthreads();
    }
}

// Panel variant: the whole A panel [32 x kp] and B panel [kp x 32] are loaded
// into shared memory with every load of the panel in flight at once (deep
// memory-level parallelism for L2-resident operands), then multiplied with no
// further barriers. kp <= kPanel; longer K loops over panels.
constexpr int kPanel = 192;
constexpr int kPAS = kPanel + 4;   // A panel row stride: conflict-free a-fragments
constexpr int kPBS = kT + 8;       // B panel row stride
constexpr std::size_t kPanelSmemBytes = (kT * kPAS + kPanel * kPBS) * sizeof(double);

template <typename LA, typename LB>
__device__ __forceinline__ void tile_gemm_panel(double* psm, int K, LA la, LB lb, double acc[4]) {
    double* As = psm;
    double* Bs = psm + kT * kPAS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 2) * 16, wn = (warp & 3) * 8;
    acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    for (int k0 = 0; k0 < K; k0 += kPanel) {
        const int kp = min(kPanel, K - k0);
        const int kpad = (kp + 15) & ~15;
        // A panel: element e -> (row = e / kpad, k = e % kpad); B panel: (k = e / 32, col = e % 32).
        // Loads are issued in batches of 8 before their shared stores so each
        // thread keeps 8 L2 requests in flight.
        constexpr int kBatch = 8;
        const int na = kT * kpad, nb = kpad * kT;
        for (int e0 = tid; e0 < na; e0 += kBatch * kThreads) {
            double v[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int e = e0 + u * kThreads;
                const int row = e / kpad, k = e - row * kpad;
                v[u] = (e < na && k < kp) ? la(row, k0 + k) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int e = e0 + u * kThreads;
                if (e < na) {
                    const int row = e / kpad, k = e - row * kpad;
                    As[row * kPAS + k] = v[u];
                }
            }
        }
        for (int e0 = tid; e0 < nb; e0 += kBatch * kThreads) {
            double v[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int e = e0 + u * kThreads;
                const int k = e >> 5, col = e & 31;
                v[u] = (e < nb && k < kp) ? lb(k0 + k, col) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int e = e0 + u * kThreads;
                if (e < nb) Bs[(e >> 5) * kPBS + (e & 31)] = v[u];
            }
        }
        __syncthreads();
        for (int c = 0; c < kpad; c += kKC) {
            double a[8], b[4];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = As[(wm + g + 8 * (i & 1)) * kPAS + c + t + 4 * (i >> 1)];
#pragma unroll
            for (int i = 0; i < 4; ++i) b[i] = Bs[(c + t + 4 * i) * kPBS + wn + g];
            dmma16816(acc, a, b);
        }
        __syncthreads();
    }
}

// Fixed-order CTA reduction of one value per thread; returns to all threads.
template <class S>
__device__ __forceinline__ double cta_sum(S& sm, double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sm.red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += sm.red[i];
    __syncthreads();
    return s;
}

}  // namespace tile
}  // namespace cpkit
