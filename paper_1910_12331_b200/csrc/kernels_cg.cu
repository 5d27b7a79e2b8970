// Preconditioned implicit CG for (J^T J + lambda Reg) vec(V) = -vec(G)
// as ONE persistent cooperative kernel (sm_100a, fp64).
//
// Reference: cp_cg (gauss_newton.cpp:279-349), hessian_matvec (:96-136),
// build_preconditioner (:190-207), norm_sum/dot_sum (:246-258).
//
// The reference calls N^2 small Eigen GEMMs per matvec and recomputes
// A_p^T W_p for every (n, p) pair. Here one CG iteration is three grid-wide
// phases of 32x32 DMMA tile tasks separated by a software grid barrier:
//   A: W' = Z + beta W (ping-pong, written once) and B_p = A_p^T W'_p
//      (split over rows into partial slabs)                     O(R^2 sum s)
//   B: Q_n = [W'_n | A_n] [Gamma(n,n) ; D_n^T] + lambda Reg(W'_n)
//      with D_n = sum_{p!=n} Gamma(n,p) o B_p folded into the operand
//      load, plus per-task partials of <W', Q>                  O(2 R^2 sum s)
//   C: alpha = rz / <W,Q>; V += alpha W'; R' = R - alpha Q (ping-pong);
//      Z = R' Pinv_n; partials of <R', Z> and ||R'_n||^2       O(R^2 sum s)
// Every scalar (alpha, beta, the stop test sum_n ||R_n||_F <= tol sum_n ||G_n||_F,
// the cap, breakdown !(wq > 0), the non-finite check) is recomputed by every
// CTA from the same partial slots in the same order, so all CTAs take the
// same branch with no host round trip. Results are bitwise reproducible.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "common.h"
#include "grid_sync.cuh"
#include "tile_gemm.cuh"

namespace cpkit {

namespace {

using namespace tile;
using gsync::grid_barrier;
using gsync::cta_rank;

// Panel staging: bulk copies (one thread per row, one mbarrier) when every row
// run is 16-byte aligned (R even), cp.async otherwise.
struct Stager {
    unsigned long long* bar;
    unsigned parity;
    bool bulk;
    int vb;  // task-order rank of this CTA (see cta_rank)
    __device__ __forceinline__ void begin() const {
        if (bulk) fence_async_shared();  // prior generic smem accesses before async-proxy writes
    }
    template <int kLanes, class P1, class P2>
    __device__ __forceinline__ void rows(double* dst, int stride, int nrows, int width, int valid, int split, P1 p1,
                                         P2 p2) {
        if (bulk) stage_rows_bulk(dst, stride, nrows, width, valid, split, p1, p2, bar);
        else stage_rows<kLanes>(dst, stride, nrows, width, valid, split, p1, p2);
    }
    template <int kLanes, class P1>
    __device__ __forceinline__ void rows(double* dst, int stride, int nrows, int width, int valid, P1 p1) {
        rows<kLanes>(dst, stride, nrows, width, valid, width, p1, p1);
    }
    __device__ __forceinline__ void wait() {
        if (bulk) {
            bulk_wait(bar, parity);
        } else {
            cp_async_wait_all();
            __syncthreads();
        }
    }
};

struct Layout {
    int order, R, tr;            // tr = tiles along R
    int ksplit;                  // phase A row splits
    int tasksA, tasksBC;
    int rowtiles[kMaxOrder];     // tiles along s_n
    int taskoff[kMaxOrder + 1];  // phase B/C task offsets per mode
};

__device__ __forceinline__ void decode_bc(const Layout& L, int task, int& n, int& rt, int& ct) {
    n = 0;
    while (task >= L.taskoff[n + 1]) ++n;
    const int local = task - L.taskoff[n];
    rt = local / L.tr;
    ct = local % L.tr;
}

struct Dev {
    CgParams p;
    Layout L;
    int mode;  // 0 = full CG, 1 = single matvec (W given in W[0], result in Q)
};
extern __shared__ __align__(16) double cg_panel_smem[];  // staged operand panels

// slot regions (doubles): [0, tasksB) wq partials; then rz, nrm, fin per task C
__device__ __forceinline__ double* slot_wq(const Dev& d) { return d.p.slots; }
__device__ __forceinline__ double* slot_rz(const Dev& d) { return d.p.slots + d.L.tasksBC; }
__device__ __forceinline__ double* slot_nrm(const Dev& d) { return d.p.slots + 2 * d.L.tasksBC; }
__device__ __forceinline__ double* slot_fin(const Dev& d) { return d.p.slots + 3 * d.L.tasksBC; }
__device__ __forceinline__ double* bpart(const Dev& d) { return d.p.slots + 4 * d.L.tasksBC; }
// D_n^T blocks (order x R x R) after the ksplit partial slabs of B_p
__device__ __forceinline__ double* dt_buf(const Dev& d) {
    return bpart(d) + static_cast<long long>(d.L.ksplit) * d.L.order * d.L.R * d.L.R;
}

__device__ __forceinline__ void stamp(const Dev& d, const Stager& st, int it, int k) {
    if (d.p.trace && st.vb == 0 && threadIdx.x == 0 && it >= 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        d.p.trace[it * 16 + k] = t;
    }
}

// ---- phase A2: Bsum_p = sum_ks Bpart; D_n^T[z][r] = sum_{p != n} Gamma(n,p)[r][z] Bsum_p[r][z]
// (gauss_newton.cpp:114-121 d = gamma(n,p) o (A_p^T W_p), folded over p once)
__device__ void phase_a2(const Dev& d) {
    const CgParams& p = d.p;
    const Layout& L = d.L;
    const int R = L.R, N = L.order;
    const long long RR = static_cast<long long>(R) * R;
    const double* bp = bpart(d);
    double* dt = dt_buf(d);
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < RR;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(e / R), z = static_cast<int>(e % R);
        double bs[kMaxOrder];
#pragma unroll
        for (int q = 0; q < kMaxOrder; ++q) bs[q] = 0.0;
        // partial slabs in chunks of 8 independent loads, summed in fixed (ks) order
        for (int q = 0; q < N; ++q) {
            double b = 0.0;
            for (int k0 = 0; k0 < L.ksplit; k0 += 8) {
                double part[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    part[u] = (k0 + u < L.ksplit) ? __ldcg(bp + (static_cast<long long>(k0 + u) * N + q) * RR + e) : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (k0 + u < L.ksplit) b += part[u];
            }
#pragma unroll
            for (int qq = 0; qq < kMaxOrder; ++qq)
                if (qq == q) bs[qq] = b;
        }
        for (int n = 0; n < N; ++n) {
            double dsum = 0.0;
#pragma unroll
            for (int q = 0; q < kMaxOrder; ++q) {
                if (q >= N || q == n) continue;
                dsum += p.pair[(n * N + q) * RR + e] * bs[q];
            }
            dt[n * RR + static_cast<long long>(z) * R + r] = dsum;
        }
    }
}

// ---- phase A: W' = Z + beta W_old (first: W' = Z; matvec: W' = W_in), B_p partials
__device__ void phase_a(const Dev& d, RedSmem& sm, Stager& st, const double* Wold, double* Wnew, double beta,
                        bool first) {
    const CgParams& p = d.p;
    const Layout& L = d.L;
    const int R = L.R;
    for (int task = st.vb; task < L.tasksA; task += gridDim.x) {
        int rem = task;
        const int ks = rem % L.ksplit; rem /= L.ksplit;
        const int zt = rem % L.tr; rem /= L.tr;
        const int rt = rem % L.tr; rem /= L.tr;
        const int pm = rem;
        const long long s = p.rows[pm];
        const long long per = (s + L.ksplit - 1) / L.ksplit;
        const long long k0 = ks * per, k1 = min(s, k0 + per);
        const int K = static_cast<int>(max(0LL, k1 - k0));
        const double* A = p.A + p.off[pm];
        const double* Z = p.Z + p.off[pm];
        const double* Wo = Wold + p.off[pm];
        double* Wn = Wnew + p.off[pm];
        const int r0 = rt * kT, z0 = zt * kT;
        const bool writer = (rt == 0) && d.mode == 0;
        // A_p^T panel (k-major) and W' panel: W_in (matvec), Z (first) or fma(beta, W_old, Z)
        double* As = cg_panel_smem;
        double* Bs = As + kPA * kKS;
        double* Aux = Bs + kPA * kKS;
        const bool comb = d.mode == 0 && !first;
        const double* bsrc = d.mode == 1 ? Wo : Z;
        const int vr = min(kT, R - r0), vz = min(kT, R - z0);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int kk0 = 0; kk0 < K; kk0 += kPA) {
            const int kp = min(kPA, K - kk0), kpad = pad8(kp);
            const long long rb = (k0 + kk0) * R;
            st.begin();
            st.rows<16>(As, kKS, kpad, kT, vr, [&](int k) { return k < kp ? A + rb + k * R + r0 : nullptr; });
            st.rows<16>(Bs, kKS, kpad, kT, vz, [&](int k) { return k < kp ? bsrc + rb + k * R + z0 : nullptr; });
            if (comb) st.rows<16>(Aux, kKS, kpad, kT, vz, [&](int k) { return k < kp ? Wo + rb + k * R + z0 : nullptr; });
            st.wait();
            if (comb) {
                combine(Bs, Aux, kpad * kKS, beta);
                __syncthreads();
            }
            if (writer)
                for (int e = threadIdx.x; e < kp * kT; e += kThreads)
                    if ((e & 31) < vz) Wn[rb + (e >> 5) * R + z0 + (e & 31)] = Bs[(e >> 5) * kKS + (e & 31)];
            mma_panel<true>(As, kKS, Bs, kpad, acc);
            __syncthreads();
        }
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int g = lane >> 2, t = lane & 3;
        double* bout = bpart(d) + (static_cast<long long>(ks) * L.order + pm) * R * R;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int r = r0 + (warp >> 2) * 16 + g + 8 * h;
                const int z = z0 + (warp & 3) * 8 + 2 * t + c;
                if (r < R && z < R) bout[r * R + z] = acc[2 * h + c];
            }
    }
}

// ---- phase B: Q_n = [W'|A_n][Gnn; D^T] + lambda Reg(W'); wq partials
__device__ void phase_b(const Dev& d, RedSmem& sm, Stager& st, const double* Wn_all, double* Qout, int it = -1) {
    const CgParams& p = d.p;
    const Layout& L = d.L;
    const int R = L.R;
    const long long RR = static_cast<long long>(R) * R;
    for (int task = st.vb; task < L.tasksBC; task += gridDim.x) {
        int n, rt, ct;
        decode_bc(L, task, n, rt, ct);
        const long long s = p.rows[n];
        const long long row0 = static_cast<long long>(rt) * kT;
        const int c0 = ct * kT;
        const double* W = Wn_all + p.off[n];
        const double* A = p.A + p.off[n];
        const double* Gnn = p.pair + (n * L.order + n) * RR;
        const double* Dt = dt_buf(d) + n * RR;
        // prefetch this thread's epilogue operands before the panel loads (overlapped)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int g = lane >> 2, t = lane & 3;
        double wpre[4], gdiag[4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const long long i = row0 + (warp >> 2) * 16 + g + 8 * h;
                const int r = c0 + (warp & 3) * 8 + 2 * t + c;
                const bool ok = i < s && r < R;
                wpre[2 * h + c] = ok ? __ldcg(W + i * R + r) : 0.0;
                gdiag[2 * h + c] = ok ? Gnn[r * R + r] : 0.0;
            }
        // [W' | A_n] (row-major) x [Gamma_nn ; D_n^T] (k-major); K = 2R in panels of kPB
        double* As = cg_panel_smem;
        double* Bs = As + kT * (kPB + 4);
        const int vc = min(kT, R - c0);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int kk0 = 0; kk0 < 2 * R; kk0 += kPB) {
            const int kp = min(kPB, 2 * R - kk0), kpad = pad8(kp);
            const int split = max(0, R - kk0);  // panel columns [0, split) from W', the rest from A_n
            st.begin();
            st.rows<32>(
                As, kPB + 4, kT, kpad, kp, split,
                [&](int row) {
                    const long long i = row0 + row;
                    return i < s ? W + i * R + kk0 : nullptr;
                },
                [&](int row) { return A + (row0 + row) * R + max(0, kk0 - R); });
            st.rows<16>(Bs, kKS, kpad, kT, vc, [&](int k) {
                const int kk = kk0 + k;
                if (k >= kp) return static_cast<const double*>(nullptr);
                return kk < R ? Gnn + static_cast<long long>(kk) * R + c0 : Dt + static_cast<long long>(kk - R) * R + c0;
            });
            st.wait();
            if (kk0 == 0) stamp(d, st, it, 9);
            mma_panel<false>(As, kPB + 4, Bs, kpad, acc);
            __syncthreads();
        }
        stamp(d, st, it, 10);
        double part = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const long long i = row0 + (warp >> 2) * 16 + g + 8 * h;
                const int r = c0 + (warp & 3) * 8 + 2 * t + c;
                if (i < s && r < R) {
                    const double w = wpre[2 * h + c];
                    const double reg = (p.shape == 0) ? p.lambda * w : w * (p.lambda * gdiag[2 * h + c]);
                    const double q = acc[2 * h + c] + reg;
                    Qout[p.off[n] + i * R + r] = q;
                    part += w * q;
                }
            }
        const double tot = cta_sum(sm, part);
        stamp(d, st, it, 11);
        if (threadIdx.x == 0 && d.mode == 0) slot_wq(d)[task] = tot;
    }
}

// ---- phase C: V += alpha W'; R' = R - alpha Q (init: R' = -G); Z = R' Pinv
__device__ void phase_c(const Dev& d, RedSmem& sm, Stager& st, const double* Wn_all, const double* Rold_all,
                        double* Rnew_all, double alpha, bool init, int it = -1) {
    const CgParams& p = d.p;
    const Layout& L = d.L;
    const int R = L.R;
    const long long RR = static_cast<long long>(R) * R;
    for (int task = st.vb; task < L.tasksBC; task += gridDim.x) {
        int n, rt, ct;
        decode_bc(L, task, n, rt, ct);
        const long long s = p.rows[n];
        const long long row0 = static_cast<long long>(rt) * kT;
        const int c0 = ct * kT;
        const long long off = p.off[n];
        const double* Pinv = p.pinv + n * RR;
        // R' = fma(-alpha, Q, R_old) (init: -G), formed identically in the operand and the epilogue
        auto rnew = [&](long long e) -> double {
            return init ? -1.0 * p.G[e] : __fma_rn(-alpha, __ldcg(p.Q + e), __ldcg(Rold_all + e));
        };
        // prefetch this thread's epilogue operands (R, Q, V, W') before the panel loads
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int g = lane >> 2, t = lane & 3;
        double rpre[4], vpre[4], wpre[4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const long long i = row0 + (warp >> 2) * 16 + g + 8 * h;
                const int r = c0 + (warp & 3) * 8 + 2 * t + c;
                const bool ok = i < s && r < R;
                const long long e = off + i * R + r;
                rpre[2 * h + c] = ok ? rnew(e) : 0.0;
                vpre[2 * h + c] = (ok && !init) ? __ldcg(p.V + e) : 0.0;
                wpre[2 * h + c] = (ok && !init) ? __ldcg(Wn_all + e) : 0.0;
            }
        stamp(d, st, it, 15);
        // R' (row-major, formed in shared memory) x Pinv (k-major)
        double* As = cg_panel_smem;
        double* Aux = As + kT * (kPC + 4);
        double* Bs = Aux + kT * (kPC + 4);
        const double* Ab = (init ? p.G : Rold_all) + off;
        const int vc = min(kT, R - c0);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int kk0 = 0; kk0 < R; kk0 += kPC) {
            const int kp = min(kPC, R - kk0), kpad = pad8(kp);
            auto rowp = [&](const double* base) {
                return [=](int row) {
                    const long long i = row0 + row;
                    return i < s ? base + i * R + kk0 : nullptr;
                };
            };
            st.begin();
            st.rows<32>(As, kPC + 4, kT, kpad, kp, rowp(Ab));
            if (!init) st.rows<32>(Aux, kPC + 4, kT, kpad, kp, rowp(p.Q + off));
            st.rows<16>(Bs, kKS, kpad, kT, vc,
                        [&](int k) { return k < kp ? Pinv + static_cast<long long>(kk0 + k) * R + c0 : nullptr; });
            st.wait();
            stamp(d, st, it, 12);
            combine(As, init ? nullptr : Aux, kT * (kPC + 4), init ? -1.0 : -alpha);
            __syncthreads();
            mma_panel<false>(As, kPC + 4, Bs, kpad, acc);
            __syncthreads();
        }
        stamp(d, st, it, 13);
        double rz = 0.0, nrm = 0.0, bad = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const long long i = row0 + (warp >> 2) * 16 + g + 8 * h;
                const int r = c0 + (warp & 3) * 8 + 2 * t + c;
                if (i < s && r < R) {
                    const long long e = off + i * R + r;
                    const double rv = rpre[2 * h + c];
                    const double zv = acc[2 * h + c];
                    const double v = init ? 0.0 : vpre[2 * h + c] + alpha * wpre[2 * h + c];
                    p.V[e] = v;
                    Rnew_all[e] = rv;
                    p.Z[e] = zv;
                    rz += rv * zv;
                    nrm += rv * rv;
                    if (!isfinite(v) || !isfinite(rv)) bad = 1.0;
                }
            }
        const double trz = cta_sum(sm, rz);
        const double tnrm = cta_sum(sm, nrm);
        const double tbad = cta_sum(sm, bad);
        stamp(d, st, it, 14);
        if (threadIdx.x == 0) {
            slot_rz(d)[task] = trz;
            slot_nrm(d)[task] = tnrm;
            slot_fin(d)[task] = tbad;
        }
    }
}

// Slot reductions: thread i reads slots i, i + 256, ... (L2 loads, all in
// flight), then a fixed-shape CTA tree; every CTA gets the same bits.
__device__ double sum_slots(RedSmem& sm, const double* slots, int n) {
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += __ldcg(slots + i);
    return cta_sum(sm, v);
}
// sum_n sqrt(sum of the mode-n slots) (norm_sum, gauss_newton.cpp:246-250)
__device__ double norm_sum_slots(const Dev& d, RedSmem& sm) {
    const double* nr = slot_nrm(d);
    double total = 0.0;
    for (int n = 0; n < d.L.order; ++n) {
        double v = 0.0;
        for (int i = d.L.taskoff[n] + threadIdx.x; i < d.L.taskoff[n + 1]; i += blockDim.x) v += __ldcg(nr + i);
        total += sqrt(cta_sum(sm, v));
    }
    return total;
}


__global__ void __launch_bounds__(kThreads, 2) cg_kernel(const __grid_constant__ Dev d) {
    __shared__ RedSmem sm;
    __shared__ unsigned long long stage_bar;
    const CgParams& p = d.p;
    const unsigned nb = gridDim.x;
    unsigned int round = 0;
    if (threadIdx.x == 0) bar_init(&stage_bar);
    Stager st{&stage_bar, 0u, (d.L.R & 1) == 0, cta_rank(p.barrier)};  // (cta_rank syncs the CTA)
    if (p.trace && threadIdx.x == 0 && st.vb < 1024) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[64 * 16 + st.vb] = smid;
    }
    if (d.mode == 1) {
        // U = H W: W in W[0]; B_p from W then Q
        phase_a(d, sm, st, p.W[0], p.W[1], 0.0, false);
        grid_barrier(p.barrier, nb, round);
        phase_a2(d);
        grid_barrier(p.barrier, nb, round);
        phase_b(d, sm, st, p.W[0], p.Q);
        return;
    }
    // init: R = -G, Z = R Pinv, V = 0
    phase_c(d, sm, st, p.W[0], p.Rr[0], p.Rr[1], 0.0, true);
    grid_barrier(p.barrier, nb, round);
    int rc = 1;  // current residual buffer
    int wc = 0;  // current direction buffer (W_old)
    int it = 0;
    double rz = 0.0, wq = 0.0;
    bool first = true;
    const double gnorm = norm_sum_slots(d, sm);  // ||R|| = ||G|| at init
    const double target = p.cg_tol * gnorm;
    int hit_cap = 0, breakdown = 0, nonfinite = 0;
    for (;;) {
        const double rz_new = sum_slots(sm, slot_rz(d), d.L.tasksBC);
        const double nsum = norm_sum_slots(d, sm);
        double beta = 0.0;
        if (!first) {
            const double bad = sum_slots(sm, slot_fin(d), d.L.tasksBC);
            if (bad != 0.0) {
                nonfinite = 1;
                break;
            }
            beta = (p.beta_variant == 0) ? rz_new / rz : rz_new / wq;
        }
        rz = rz_new;
        if (!(nsum > target)) break;
        if (it >= p.cap) {
            hit_cap = 1;
            break;
        }
        stamp(d, st, it, 0);
        phase_a(d, sm, st, p.W[wc], p.W[wc ^ 1], beta, first);
        wc ^= 1;
        stamp(d, st, it, 1);
        grid_barrier(p.barrier, nb, round);
        stamp(d, st, it, 2);
        phase_a2(d);
        grid_barrier(p.barrier, nb, round);
        stamp(d, st, it, 3);
        phase_b(d, sm, st, p.W[wc], p.Q, it);
        stamp(d, st, it, 4);
        grid_barrier(p.barrier, nb, round);
        stamp(d, st, it, 5);
        wq = sum_slots(sm, slot_wq(d), d.L.tasksBC);
        if (!(wq > 0.0)) {
            breakdown = 1;
            break;
        }
        const double alpha = rz / wq;
        stamp(d, st, it, 8);
        phase_c(d, sm, st, p.W[wc], p.Rr[rc], p.Rr[rc ^ 1], alpha, false, it);
        rc ^= 1;
        stamp(d, st, it, 6);
        grid_barrier(p.barrier, nb, round);
        stamp(d, st, it, 7);
        ++it;
        first = false;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.result[0] = it;
        p.result[1] = hit_cap;
        p.result[2] = breakdown;
        p.result[3] = nonfinite;
        p.result[4] = rc;
    }
}

Layout make_layout(const CgParams& p, int grid) {
    Layout L{};
    L.order = p.order;
    L.R = p.R;
    L.tr = (p.R + kT - 1) / kT;
    int off = 0;
    long long smax = 1;
    for (int n = 0; n < p.order; ++n) {
        L.rowtiles[n] = static_cast<int>((p.rows[n] + kT - 1) / kT);
        L.taskoff[n] = off;
        off += L.rowtiles[n] * L.tr;
        smax = std::max<long long>(smax, p.rows[n]);
    }
    L.taskoff[p.order] = off;
    L.tasksBC = off;
    const int base = p.order * L.tr * L.tr;
    int ks = std::max(1, grid / base);  // one round of the grid
    ks = static_cast<int>(std::min<long long>(ks, std::max<long long>(1, smax / 32)));
    L.ksplit = ks;
    L.tasksA = base * ks;
    return L;
}

int occupancy_grid(int device) {
    // per-device result cached: it sits on the host path in front of every solve
    static std::mutex mu;
    static int cached[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (device >= 0 && device < 64 && cached[device] > 0) return cached[device];
    int sms = 0, per = 0;
    CPK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    ensure_dynamic_smem(cg_kernel, kAsyncSmemBytes);
    CPK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cg_kernel, kThreads, kAsyncSmemBytes));
    const int g = sms * std::max(1, per);
    if (device >= 0 && device < 64) cached[device] = g;
    return g;
}

void launch_coop(const Dev& d, int grid, cudaStream_t st) {
    Dev dd = d;
    void* args[] = {&dd};
    launch_cooperative(reinterpret_cast<const void*>(cg_kernel), dim3(grid), dim3(kThreads), args, kAsyncSmemBytes,
                       st);
    count_launch(1);
}

}  // namespace

int cg_max_grid(int device) { return occupancy_grid(device); }

std::size_t cg_slots_needed(const CgParams& p) {
    const Layout L = make_layout(p, 148);
    // generous: ksplit may grow with grid, bound it by the rows/32 cap
    long long smax = 1;
    for (int n = 0; n < p.order; ++n) smax = std::max<long long>(smax, p.rows[n]);
    const long long ksmax = std::max<long long>(1, smax / 32);
    return std::max(static_cast<std::size_t>(4 * L.tasksBC) +
                        static_cast<std::size_t>(ksmax + 1) * p.order * p.R * p.R,
                    cg_res_slots_needed(p));
}

void run_cg(const CgParams& p, int grid, cudaStream_t st) {
    if (run_cg_resident(p, st)) return;  // tile-resident kernel when the tiles fit the machine
    Dev d{};
    d.p = p;
    d.mode = 0;
    // no point in more CTAs than the widest phase has tasks
    const Layout L0 = make_layout(p, grid);
    grid = std::max(1, std::min(grid, std::max(L0.tasksA, L0.tasksBC)));
    d.L = make_layout(p, grid);
    if (!p.barrier_zeroed) CPK_CUDA(cudaMemsetAsync(p.barrier, 0, cg_barrier_words() * sizeof(unsigned int), st));
    launch_coop(d, grid, st);
}

void launch_jtj_matvec(const CgParams& p, const double* w, double* u, cudaStream_t st) {
    int dev = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    Dev d{};
    d.p = p;
    d.p.W[0] = const_cast<double*>(w);
    d.p.Q = u;
    d.mode = 1;
    int grid = cg_max_grid(dev);
    const Layout L0 = make_layout(p, grid);
    grid = std::max(1, std::min(grid, std::max(L0.tasksA, L0.tasksBC)));
    d.L = make_layout(p, grid);
    if (!p.barrier_zeroed) CPK_CUDA(cudaMemsetAsync(p.barrier, 0, cg_barrier_words() * sizeof(unsigned int), st));
    launch_coop(d, grid, st);
}

}  // namespace cpkit
