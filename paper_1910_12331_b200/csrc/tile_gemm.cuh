// DMMA 32x32 tile GEMM building block shared by the CG phases and the small
// dense kernels (Gram, gradient). 256 threads = 8 warps (2 x m16, 4 x n8).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

#include <cstddef>

namespace cpkit {
namespace tile {

constexpr int kT = 32;        // task tile edge
constexpr int kKC = 16;       // k chunk
constexpr int kThreads = 256;  // 8 warps: 2 (m16) x 4 (n8)
constexpr int kAS = kKC + 4;  // A smem row stride (doubles): conflict-free a-fragments
constexpr int kBS = kT + 4;   // B smem row stride: conflict-free b-fragments (t*4+g)

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
constexpr int kPBS = kT + 4;       // B panel row stride
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

// Asynchronous row-staged panels (CG phases). Operand rows are contiguous
// runs in global memory, moved to shared memory with cp.async (16-byte .cg
// copies where aligned, 8-byte otherwise): no registers are tied up and every
// copy of a panel is in flight at once, so a panel costs one L2 round trip.
// Layouts: A row-major [32][kp + 4] or k-major [k][kKS]; B k-major [k][kKS].
// Panel depths are per phase so each phase fits its operands in one panel at
// R = 100 within a 2-CTA/SM shared-memory budget; k is padded to 8.
constexpr int kKS = kT + 4;  // k-major stride: fragments conflict-free (4 mod 16)
constexpr int kPA = 120;     // phase A (k-major A_p^T, W', aux)
constexpr int kPB = 200;     // phase B ([W'|A_n] row-major, [Gnn; D^T])
constexpr int kPC = 128;     // phase C (R' row-major + aux, Pinv)
constexpr int kSmemA = 3 * kPA * kKS;
constexpr int kSmemB = kT * (kPB + 4) + kPB * kKS;
constexpr int kSmemC = 2 * kT * (kPC + 4) + kPC * kKS;
constexpr int kSmemMax = kSmemA > kSmemB ? (kSmemA > kSmemC ? kSmemA : kSmemC) : (kSmemB > kSmemC ? kSmemB : kSmemC);
constexpr std::size_t kAsyncSmemBytes = kSmemMax * sizeof(double);

__device__ __forceinline__ int pad8(int k) { return (k + 7) & ~7; }

__device__ __forceinline__ void dmma1688(double* d, const double* a, const double* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Rows r < nrows, columns c < width (even): c < valid copied from
// p1(r)[c] (c < split) or p2(r)[c - split] (c >= split); c >= valid zeroed.
// A null p1(r) zeroes the whole row. kLanes threads cooperate on one row.
template <int kLanes, class P1, class P2>
__device__ __forceinline__ void stage_rows(double* dst, int stride, int nrows, int width, int valid, int split,
                                           P1 p1, P2 p2) {
    const int lane = threadIdx.x % kLanes;
    for (int r = threadIdx.x / kLanes; r < nrows; r += kThreads / kLanes) {
        const double* s1 = p1(r);
        const double* s2 = split < valid ? p2(r) - split : s1;
        double* d = dst + r * stride;
        for (int c = 2 * lane; c < width; c += 2 * kLanes) {
            const double* sc = (c < split ? s1 : s2) + c;
            const bool one_src = (c + 1 < split) || (c >= split);
            if (s1 && one_src && c + 1 < valid && (reinterpret_cast<uintptr_t>(sc) & 15) == 0) {
                cp_async16(d + c, sc);
            } else {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (s1 && c + u < valid) cp_async8(d + c + u, (c + u < split ? s1 : s2) + c + u);
                    else d[c + u] = 0.0;
                }
            }
        }
    }
}
template <int kLanes, class P1>
__device__ __forceinline__ void stage_rows(double* dst, int stride, int nrows, int width, int valid, P1 p1) {
    stage_rows<kLanes>(dst, stride, nrows, width, valid, width, p1, p1);
}

// ---- bulk-copy staging (R even: every row run is 16-byte aligned) ----------
// One thread per row issues cp.async.bulk copies of the row's contiguous
// run(s) straight into shared memory, signalling one mbarrier with the byte
// count; padding is zeroed with plain stores (disjoint from the copies).
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void bar_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned parity) {
    for (unsigned long long spin = 0;; ++spin) {
        unsigned ok;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(su32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (spin > (1ull << 26)) __trap();  // a lost transaction traps instead of hanging the GPU
    }
}
__device__ __forceinline__ void bulk_copy(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_async_shared() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Same contract as stage_rows; requires every run start 16-byte aligned and
// split, valid even. Rows are owned by threads r, r + 256, ...
template <class P1, class P2>
__device__ __forceinline__ void stage_rows_bulk(double* dst, int stride, int nrows, int width, int valid, int split,
                                                P1 p1, P2 p2, unsigned long long* bar) {
    unsigned bytes = 0;
    for (int r = threadIdx.x; r < nrows; r += kThreads) {
        const double* s1 = p1(r);
        double* d = dst + r * stride;
        if (!s1) {
            for (int c = 0; c < width; c += 2) *reinterpret_cast<double2*>(d + c) = make_double2(0.0, 0.0);
            continue;
        }
        const int n1 = min(split, valid), n2 = valid - n1;
        const unsigned b = static_cast<unsigned>(n1 + n2) * 8u;
        if (b) bar_expect(bar, b);
        bytes += b;
        if (n1) bulk_copy(d, s1, n1 * 8u, bar);
        if (n2) bulk_copy(d + n1, p2(r), n2 * 8u, bar);
        for (int c = valid; c < width; ++c) d[c] = 0.0;
    }
    (void)bytes;
}
template <class P1>
__device__ __forceinline__ void stage_rows_bulk(double* dst, int stride, int nrows, int width, int valid, P1 p1,
                                                unsigned long long* bar) {
    stage_rows_bulk(dst, stride, nrows, width, valid, width, p1, p1, bar);
}
// All threads: wait for every copy of this panel (call after the staging calls).
__device__ __forceinline__ void bulk_wait(unsigned long long* bar, unsigned& parity) {
    __syncthreads();  // every expect_tx registered
    if (threadIdx.x == 0) bar_arrive(bar);
    bar_wait(bar, parity);
    parity ^= 1u;
}

// v[e] = fma(coef, aux[e], v[e]) (aux == nullptr: v[e] = coef * v[e]) over n entries.
__device__ __forceinline__ void combine(double* v, const double* aux, int n, double coef) {
    for (int e = threadIdx.x; e < n; e += kThreads) v[e] = aux ? __fma_rn(coef, aux[e], v[e]) : coef * v[e];
}

// acc += A[32 x kpad] * B[kpad x 32] for this thread's fragment (kpad % 8 == 0).
// kAKMajor: A stored [k][kKS]; else [row][lda].
template <bool kAKMajor>
__device__ __forceinline__ void mma_panel(const double* As, int lda, const double* Bs, int kpad, double acc[4]) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = (warp >> 2) * 16, wn = (warp & 3) * 8;
    auto aval = [&](int row, int k) { return kAKMajor ? As[k * kKS + row] : As[row * lda + k]; };
    int c = 0;
    for (; c + kKC <= kpad; c += kKC) {
        double a[8], b[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = aval(wm + g + 8 * (i & 1), c + t + 4 * (i >> 1));
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = Bs[(c + t + 4 * i) * kKS + wn + g];
        dmma16816(acc, a, b);
    }
    if (c < kpad) {  // k8 tail
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = aval(wm + g + 8 * (i & 1), c + t + 4 * (i >> 1));
#pragma unroll
        for (int i = 0; i < 2; ++i) b[i] = Bs[(c + t + 4 * i) * kKS + wn + g];
        dmma1688(acc, a, b);
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
