// Batched tiny-instance CP solver: ONE CTA PER INSTANCE.
//
// The likelihood and matmul protocols (harness.cpp:488-653) run hundreds to
// thousands of independent ALS / GN-CG optimisations on tensors of a few
// dozen entries (e.g. 4x4x4, R <= 9). A per-instance launch sequence on the
// device would be launch-latency bound; the reference runs them on a host
// thread pool. Here each instance is one CTA that keeps its tensor, factors,
// dimension-tree partials and every CG vector in shared memory and runs the
// whole optimiser (als_optimize als.cpp:54-94 / gn_optimize
// gauss_newton.cpp:451-494) without leaving the SM.
//
// Every arithmetic step mirrors the reference's loop order with explicitly
// rounded operations (no FMA contraction): dimension-tree contractions
// (mttkrp.cpp:29-189, contract highest mode first, root partial cached per
// half), gram + exact symmetrisation (matrix_ops.cpp:30-34), left-looking LLT
// with the jitter retry and row solves (matrix_ops.cpp:41-81), the fast
// residual with clamp (kruskal.cpp:94-118), gradient, the per-(n,p) matvec,
// PCG with cap / breakdown / stale-beta (gauss_newton.cpp:81-349), Armijo and
// the regularisation schedule (:47-59, :360-449). Output elements are computed
// in parallel, each with the reference's own sequential accumulation, and
// scalar reductions run on one thread, so the results are bitwise those of
// the reference restatement: same statuses, iteration counts and residuals.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.h"
#include "tiny.h"

namespace cpkit {
namespace {

__device__ __forceinline__ double fadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fdiv(double a, double b) { return __ddiv_rn(a, b); }

// partial descriptor (mttkrp.hpp:15-20): kept modes ascending, their extents,
// rank 0 for the raw tensor
struct PDesc {
    int nk;
    int km[kTinyMaxOrder];
    int kd[kTinyMaxOrder];
    int rank;
};

struct Ctx {
    const TinyParams* P;
    int N, R, S;
    double* X;
    double* A;
    double* root[2];
    bool root_ok[2];
    double* T[2];
    double* grams;
    double* gam;
    double* L;
    double* inv;
    double* misc;  // scalar broadcast slots
    // GN
    double *M, *G, *V, *Rr, *Z, *W, *Q, *At, *pairs, *pinv, *tb, *td, *add, *bp;
};

__device__ __forceinline__ int nthr() { return blockDim.x; }

// ---- dimension tree (mttkrp.cpp:29-77, :118-126, :149-189) ----------------------------
__device__ void contract_mode(const Ctx& c, const double* src, const PDesc& p, int mode, const double* a,
                              double* dst, PDesc& q) {
    const int R = c.R;
    int pos = 0;
    while (p.km[pos] != mode) ++pos;
    int outer = 1, inner = 1;
    for (int i = 0; i < pos; ++i) outer *= p.kd[i];
    for (int i = pos + 1; i < p.nk; ++i) inner *= p.kd[i];
    const int sm = p.kd[pos];
    const int total = outer * inner * R;
    for (int e = threadIdx.x; e < total; e += nthr()) {
        const int r = e % R, oj = e / R;
        const int j = oj % inner, o = oj / inner;
        double acc = 0.0;
        if (p.rank == 0) {
            // :46-62 (inner == 1 is the GEMM, same accumulation order)
            for (int im = 0; im < sm; ++im) acc = fadd(acc, fmul(src[(o * sm + im) * inner + j], a[im * R + r]));
        } else {
            // :63-75 Hadamard-weighted reduction
            for (int im = 0; im < sm; ++im)
                acc = fadd(acc, fmul(src[((o * sm + im) * inner + j) * R + r], a[im * R + r]));
        }
        dst[e] = acc;
    }
    q.nk = p.nk - 1;
    for (int i = 0, k = 0; i < p.nk; ++i)
        if (i != pos) {
            q.km[k] = p.km[i];
            q.kd[k] = p.kd[i];
            ++k;
        }
    q.rank = R;
    __syncthreads();
}

// contract `modes` (any order given; applied highest first) starting from src;
// the result lands in `out` (which may be T[0]/T[1] ping-pong or a root slot)
__device__ void contract_set(const Ctx& c, const double* src, PDesc p, unsigned mask, double* out, PDesc& res) {
    const double* cur = src;
    int ping = 0;
    int left = __popc(mask);
    for (int m = c.N - 1; m >= 0; --m) {
        if (!(mask >> m & 1u)) continue;
        --left;
        double* dst = left == 0 ? out : c.T[ping];
        PDesc q;
        contract_mode(c, cur, p, m, c.A + c.P->off[m], dst, q);
        p = q;
        cur = dst;
        ping ^= 1;
    }
    res = p;
    if (__popc(mask) == 0) {  // nothing to contract: copy
        const int tot = [&] {
            int t = p.rank > 0 ? p.rank : 1;
            for (int i = 0; i < p.nk; ++i) t *= p.kd[i];
            return t;
        }();
        for (int e = threadIdx.x; e < tot; e += nthr()) out[e] = src[e];
        __syncthreads();
    }
}

__device__ PDesc tensor_desc(const Ctx& c) {
    PDesc p;
    p.nk = c.N;
    for (int i = 0; i < c.N; ++i) {
        p.km[i] = i;
        p.kd[i] = c.P->dims[i];
    }
    p.rank = 0;
    return p;
}

// M^(mode) via the dimension tree with the root partial cached per half
// (mttkrp.cpp:160-189); result (s_mode x R) written to out
__device__ void mttkrp_tree(Ctx& c, int mode, double* out) {
    const int N = c.N, h = (N + 1) / 2;
    unsigned contracted = 0, remaining = 0;
    for (int m = 0; m < N; ++m) {
        const bool front = m < h;
        if ((mode < h) != front) contracted |= 1u << m;
        else if (m != mode) remaining |= 1u << m;
    }
    const int slot = mode < h ? 0 : 1;
    PDesc root;
    if (!c.root_ok[slot]) {
        contract_set(c, c.X, tensor_desc(c), contracted, c.root[slot], root);
        c.root_ok[slot] = true;
    }
    // root descriptor (kept = the mode's half, ascending)
    root.nk = 0;
    for (int m = 0; m < N; ++m)
        if (!(contracted >> m & 1u)) {
            root.km[root.nk] = m;
            root.kd[root.nk] = c.P->dims[m];
            ++root.nk;
        }
    root.rank = c.R;
    PDesc r;
    contract_set(c, c.root[slot], root, remaining, out, r);
}
// naive, uncached (mttkrp.cpp:149-158)
__device__ void mttkrp_naive(Ctx& c, int mode, double* out) {
    unsigned mask = 0;
    for (int m = 0; m < c.N; ++m)
        if (m != mode) mask |= 1u << m;
    PDesc r;
    contract_set(c, c.X, tensor_desc(c), mask, out, r);
}
// MttkrpWorkspace::note_factor_update (mttkrp.cpp:136-145): drop partials whose key has the bit
__device__ __forceinline__ void note_update(Ctx& c, int mode) {
    const int h = (c.N + 1) / 2;
    // slot 0 contracted the back half, slot 1 the front half
    if (mode >= h) c.root_ok[0] = false;
    else c.root_ok[1] = false;
}

// ---- small dense ops ------------------------------------------------------------------
// gemm_nn: C[m x n] = A[m x k] B[k x n], ascending k from 0.0 (transposes via strides)
__device__ void gemm(const double* a, int a_rs, int a_cs, const double* b, int b_rs, int b_cs, double* cc, int m,
                     int n, int k) {
    // (i, j) advanced incrementally: one division per call, none per element
    const int T = nthr(), di = T / n, dj = T % n;
    int i = threadIdx.x / n, j = threadIdx.x % n;
    for (; i < m; i += di, j += dj) {
        if (j >= n) {
            j -= n;
            ++i;
            if (i >= m) break;
        }
        const double* ar = a + i * a_rs;
        const double* bc = b + j * b_cs;
        double acc = 0.0;
        for (int kk = 0; kk < k; ++kk) acc = fadd(acc, fmul(ar[kk * a_cs], bc[kk * b_rs]));
        cc[i * n + j] = acc;
    }
    __syncthreads();
}

// gram + exact symmetrisation (matrix_ops.cpp:30-34)
__device__ void gram(const Ctx& c, const double* a, int rows, double* s) {
    const int R = c.R;
    for (int e = threadIdx.x; e < R * R; e += nthr()) {
        const int x = e / R, y = e % R;
        double gxy = 0.0, gyx = 0.0;
        for (int i = 0; i < rows; ++i) {
            gxy = fadd(gxy, fmul(a[i * R + x], a[i * R + y]));
            gyx = fadd(gyx, fmul(a[i * R + y], a[i * R + x]));
        }
        s[e] = fmul(0.5, fadd(gxy, gyx));
    }
    __syncthreads();
}

// serial sum of squares / sums / dots on thread 0, broadcast
__device__ double bcast(const Ctx& c, double v) {
    if (threadIdx.x == 0) c.misc[0] = v;
    __syncthreads();
    const double r = c.misc[0];
    __syncthreads();
    return r;
}
__device__ double norm_of(const Ctx& c, const double* v, int n) {  // Eigen norm: sqrt of plain sum of squares
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < n; ++i) s = fadd(s, fmul(v[i], v[i]));
    return bcast(c, __dsqrt_rn(s));
}
// per-mode sequential sums on threads 0..N-1, combined in ascending mode order
// by thread 0: the same operation sequence as the reference's nested loops
__device__ double norm_sum(const Ctx& c, const double* v) {  // gauss_newton.cpp:246-250
    if (threadIdx.x < c.N) {
        const int n = threadIdx.x;
        double s = 0.0;
        for (int i = c.P->off[n]; i < c.P->off[n + 1]; ++i) s = fadd(s, fmul(v[i], v[i]));
        c.misc[4 + n] = __dsqrt_rn(s);
    }
    __syncthreads();
    double acc = 0.0;
    if (threadIdx.x == 0)
        for (int n = 0; n < c.N; ++n) acc = fadd(acc, c.misc[4 + n]);
    return bcast(c, acc);
}
__device__ double dot_sum(const Ctx& c, const double* a, const double* b) {  // :252-258
    if (threadIdx.x < c.N) {
        const int n = threadIdx.x;
        double s = 0.0;
        for (int i = c.P->off[n]; i < c.P->off[n + 1]; ++i) s = fadd(s, fmul(a[i], b[i]));
        c.misc[4 + n] = s;
    }
    __syncthreads();
    double acc = 0.0;
    if (threadIdx.x == 0)
        for (int n = 0; n < c.N; ++n) acc = fadd(acc, c.misc[4 + n]);
    return bcast(c, acc);
}
__device__ bool all_finite(const Ctx& c, const double* v, int n) {
    if (threadIdx.x == 0) c.misc[1] = 1.0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += nthr())
        if (!isfinite(v[i])) c.misc[1] = 0.0;
    __syncthreads();
    const bool ok = c.misc[1] != 0.0;
    __syncthreads();
    return ok;
}

// left-looking LLT in place on L (R x R) (matrix_ops.cpp:41-56); false on a pivot <= 0
__device__ bool llt(const Ctx& c, double* a) {
    const int R = c.R;
    for (int j = 0; j < R; ++j) {
        if (threadIdx.x == 0) {
            double x = a[j * R + j];
            for (int k = 0; k < j; ++k) x = fsub(x, fmul(a[j * R + k], a[j * R + k]));
            c.misc[2] = x;
            if (!(x <= 0.0)) a[j * R + j] = __dsqrt_rn(x);  // NaN passes, as in Eigen's LLT
        }
        __syncthreads();
        if (c.misc[2] <= 0.0) {
            __syncthreads();
            return false;
        }
        const double l = a[j * R + j];
        for (int i = j + 1 + threadIdx.x; i < R; i += nthr()) {
            double y = a[i * R + j];
            for (int k = 0; k < j; ++k) y = fsub(y, fmul(a[i * R + k], a[j * R + k]));
            a[i * R + j] = fdiv(y, l);
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < R * R; e += nthr())
        if (e % R > e / R) a[e] = 0.0;
    __syncthreads();
    return true;
}
// factor_shifted (matrix_ops.cpp:41-56): L = chol(S + lambda I), one jitter retry
__device__ bool factor_shifted(const Ctx& c, const double* s, double lambda, double* l) {
    const int R = c.R;
    for (int e = threadIdx.x; e < R * R; e += nthr()) l[e] = (e / R == e % R) ? fadd(s[e], lambda) : s[e];
    __syncthreads();
    if (llt(c, l)) return true;
    double tr = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < R; ++i) tr = fadd(tr, s[i * R + i]);
    tr = bcast(c, tr);
    const double jitter = fdiv(fmul(1e-12, tr), static_cast<double>(R));
    for (int e = threadIdx.x; e < R * R; e += nthr())
        l[e] = (e / R == e % R) ? fadd(fadd(s[e], lambda), jitter) : s[e];
    __syncthreads();
    return llt(c, l);
}
// rows of y solved in place with (L L^T) (matrix_ops.cpp:60-71)
__device__ void llt_solve_rows(const Ctx& c, const double* l, double* y, int rows) {
    const int R = c.R;
    for (int row = threadIdx.x; row < rows; row += nthr()) {
        double* v = y + row * R;
        for (int i = 0; i < R; ++i) {
            double s = v[i];
            for (int k = 0; k < i; ++k) s = fsub(s, fmul(l[i * R + k], v[k]));
            v[i] = fdiv(s, l[i * R + i]);
        }
        for (int i = R - 1; i >= 0; --i) {
            double s = v[i];
            for (int k = i + 1; k < R; ++k) s = fsub(s, fmul(l[k * R + i], v[k]));
            v[i] = fdiv(s, l[i * R + i]);
        }
    }
    __syncthreads();
}
// spd_inverse (matrix_ops.cpp:73-81) into out (R x R); false if singular
__device__ bool spd_inverse(const Ctx& c, const double* s, double lambda, double* out) {
    const int R = c.R;
    if (!factor_shifted(c, s, lambda, c.L)) return false;
    for (int e = threadIdx.x; e < R * R; e += nthr()) c.inv[e] = (e / R == e % R) ? 1.0 : 0.0;
    __syncthreads();
    llt_solve_rows(c, c.L, c.inv, R);
    // inv = transpose(inv); o = 0.5 (inv + inv^T): symmetric in the two orders
    for (int e = threadIdx.x; e < R * R; e += nthr()) {
        const int i = e / R, j = e % R;
        out[e] = fmul(0.5, fadd(c.inv[j * R + i], c.inv[i * R + j]));
    }
    __syncthreads();
    return true;
}

// residual_fitness (kruskal.cpp:94-118); last = M^(N-1) or nullptr (naive MTTKRP)
// grams_current: c.grams already holds gram(A_n) of the current factors (same
// values the reference recomputes here)
__device__ double residual(Ctx& c, double xnorm2, const double* last, bool grams_current = false) {
    const int N = c.N, R = c.R;
    if (last == nullptr) {
        mttkrp_naive(c, N - 1, c.add);
        last = c.add;
    }
    const int l = N - 1;
    if (!grams_current)
        for (int n = 0; n < N; ++n) gram(c, c.A + c.P->off[n], c.P->dims[n], c.grams + n * R * R);
    // all = ones o S^(0) o ... elementwise in parallel, then the row-major sum on one thread
    for (int e = threadIdx.x; e < R * R; e += nthr()) {
        double v = 1.0;
        for (int n = 0; n < N; ++n) v = fmul(v, c.grams[n * R * R + e]);
        c.tb[e] = v;
    }
    __syncthreads();
    double res = 0.0;
    if (threadIdx.x == 0) {
        double cross = 0.0;
        const double* al = c.A + c.P->off[l];
        for (int i = 0; i < c.P->dims[l] * R; ++i) cross = fadd(cross, fmul(last[i], al[i]));
        double mn = 0.0;
        for (int e = 0; e < R * R; ++e) mn = fadd(mn, c.tb[e]);
        double res2 = fadd(fsub(xnorm2, fmul(2.0, cross)), mn);
        if (res2 < 0.0) res2 = 0.0;
        res = __dsqrt_rn(fdiv(res2, xnorm2));
    }
    return bcast(c, res);
}

// ---- ALS (als.cpp:22-94) ---------------------------------------------------------------
__device__ int als_run(Ctx& c, const TinyAls& cfg, double xnorm2, int& iters, double& final_r, double& best_r) {
    const int N = c.N, R = c.R;
    iters = 0;
    final_r = 1.0;
    best_r = 1.0;
    for (int sweep = 1; sweep <= cfg.max_sweeps; ++sweep) {
        const double lambda = cfg.decay_every > 0 ? cfg.lambdas[(sweep - 1) / cfg.decay_every] : cfg.lambda0;
        if (!all_finite(c, c.A, c.S)) return -1;  // model.validate()
        for (int n = 0; n < N; ++n) gram(c, c.A + c.P->off[n], c.P->dims[n], c.grams + n * R * R);
        double step = 0.0;
        for (int n = 0; n < N; ++n) {
            for (int e = threadIdx.x; e < R * R; e += nthr()) {
                double g = 1.0;
                for (int m = 0; m < N; ++m)
                    if (m != n) g = fmul(g, c.grams[m * R * R + e]);
                c.gam[e] = g;
            }
            __syncthreads();
            double* mn = c.M + c.P->off[n];
            mttkrp_tree(c, n, mn);
            if (!factor_shifted(c, c.gam, lambda, c.L)) return -1;  // SingularSystem
            const int rows = c.P->dims[n];
            double* an = c.A + c.P->off[n];
            for (int e = threadIdx.x; e < rows * R; e += nthr()) c.add[e] = mn[e];
            __syncthreads();
            llt_solve_rows(c, c.L, c.add, rows);
            double s = 0.0;
            if (threadIdx.x == 0)
                for (int e = 0; e < rows * R; ++e) {
                    const double d = fsub(c.add[e], an[e]);
                    s = fadd(s, fmul(d, d));
                }
            const double dn = bcast(c, __dsqrt_rn(s));
            step = fadd(step, dn);
            for (int e = threadIdx.x; e < rows * R; e += nthr()) an[e] = c.add[e];
            __syncthreads();
            note_update(c, n);
            gram(c, an, rows, c.grams + n * R * R);
        }
        const double res = residual(c, xnorm2, c.M + c.P->off[N - 1], true);
        iters = sweep;
        final_r = res;
        best_r = fmin(best_r, res);
        if (res < cfg.residual_tol) return 0;     // converged_residual
        if (step < cfg.step_tol) return 1;        // converged_step
    }
    return 2;  // cap_hit
}

// ---- GN (gauss_newton.cpp:81-494) -------------------------------------------------------
// stacked element e -> (mode n, row i, column r)
__device__ __forceinline__ void stacked_index(const Ctx& c, int e, int& n, int& i, int& r) {
    n = 0;
    while (e >= c.P->off[n + 1]) ++n;
    const int local = e - c.P->off[n];
    i = local / c.R;
    r = local - i * c.R;
}

// hessian_matvec (gauss_newton.cpp:96-136) in two parallel passes: every
// B_p = A_p^T W_p, then every output element accumulates reg + sum_p add_p in
// ascending p, each add_p with the reference's own k order (same operations
// as the per-(n,p) GEMM sequence, two barriers instead of ~2 N^2).
__device__ void matvec(Ctx& c, const double* w, double lambda, int shape, double* u) {
    const int N = c.N, R = c.R, RR = R * R;
    for (int e = threadIdx.x; e < N * RR; e += nthr()) {
        const int p = e / RR, q = e - p * RR, i = q / R, j = q - i * R;
        const double* ap = c.A + c.P->off[p];
        const double* wp = w + c.P->off[p];
        double acc = 0.0;
        for (int kk = 0; kk < c.P->dims[p]; ++kk) acc = fadd(acc, fmul(ap[kk * R + i], wp[kk * R + j]));
        c.bp[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < c.S; e += nthr()) {
        int n, i, r;
        stacked_index(c, e, n, i, r);
        const double* gnn = c.pairs + (n * N + n) * RR;
        const double* wn = w + c.P->off[n];
        const double* an = c.A + c.P->off[n];
        double un = shape == 0 ? fmul(lambda, wn[i * R + r]) : fmul(wn[i * R + r], fmul(lambda, gnn[r * R + r]));
        for (int p = 0; p < N; ++p) {
            double add = 0.0;
            if (p == n) {
                for (int kk = 0; kk < R; ++kk) add = fadd(add, fmul(wn[i * R + kk], gnn[kk * R + r]));
            } else {
                const double* gnp = c.pairs + (n * N + p) * RR;
                const double* b = c.bp + p * RR;
                for (int kk = 0; kk < R; ++kk)
                    add = fadd(add, fmul(an[i * R + kk], fmul(gnp[r * R + kk], b[r * R + kk])));
            }
            un = fadd(un, add);
        }
        u[e] = un;
    }
    __syncthreads();
}

// Z_n = R_n Pinv_n for every mode in one pass
__device__ void apply_pinv(Ctx& c) {
    const int N = c.N, R = c.R, RR = R * R;
    (void)N;
    for (int e = threadIdx.x; e < c.S; e += nthr()) {
        int n, i, r;
        stacked_index(c, e, n, i, r);
        const double* rn = c.Rr + c.P->off[n];
        const double* pn = c.pinv + n * RR;
        double acc = 0.0;
        for (int kk = 0; kk < R; ++kk) acc = fadd(acc, fmul(rn[i * R + kk], pn[kk * R + r]));
        c.Z[e] = acc;
    }
    __syncthreads();
}

// returns iterations; flags: 1 hit cap, 2 breakdown; -1 non-finite (throws)
__device__ int cp_cg(Ctx& c, const TinyGn& cfg, double lambda, double gnorm, int& flags) {
    const int N = c.N, R = c.R, S = c.S;
    flags = 0;
    for (int e = threadIdx.x; e < S; e += nthr()) c.V[e] = 0.0;
    __syncthreads();
    if (gnorm == 0.0) return 0;
    // preconditioner (gauss_newton.cpp:190-207)
    for (int n = 0; n < N; ++n) {
        const double* gnn = c.pairs + (n * N + n) * R * R;
        bool ok;
        if (cfg.shape == 0) {
            ok = spd_inverse(c, gnn, lambda, c.pinv + n * R * R);
        } else {
            for (int e = threadIdx.x; e < R * R; e += nthr())
                c.tb[e] = (e / R == e % R) ? fmul(gnn[e], fadd(1.0, lambda)) : gnn[e];
            __syncthreads();
            ok = spd_inverse(c, c.tb, 0.0, c.pinv + n * R * R);
        }
        if (!ok) return -1;
    }
    for (int e = threadIdx.x; e < S; e += nthr()) c.Rr[e] = -c.G[e];
    __syncthreads();
    apply_pinv(c);
    for (int e = threadIdx.x; e < S; e += nthr()) c.W[e] = c.Z[e];
    __syncthreads();
    double rz = dot_sum(c, c.Rr, c.Z);
    const double target = fmul(cfg.cg_tol, gnorm);
    int it = 0;
    while (norm_sum(c, c.Rr) > target) {
        if (it >= cfg.cap) {
            flags = 1;
            break;
        }
        matvec(c, c.W, lambda, cfg.shape, c.Q);
        const double wq = dot_sum(c, c.W, c.Q);
        if (!(wq > 0.0)) {
            flags = 2;
            break;
        }
        const double alpha = fdiv(rz, wq);
        for (int e = threadIdx.x; e < S; e += nthr()) {
            c.V[e] = fadd(c.V[e], fmul(alpha, c.W[e]));
            c.Rr[e] = fsub(c.Rr[e], fmul(alpha, c.Q[e]));
        }
        __syncthreads();
        apply_pinv(c);
        const double rz_new = dot_sum(c, c.Rr, c.Z);
        const double beta = cfg.beta_variant == 0 ? fdiv(rz_new, rz) : fdiv(rz_new, wq);
        for (int e = threadIdx.x; e < S; e += nthr()) c.W[e] = fadd(c.Z[e], fmul(beta, c.W[e]));
        __syncthreads();
        rz = rz_new;
        ++it;
        if (!all_finite(c, c.V, S) || !all_finite(c, c.Rr, S)) return -1;
    }
    return it;
}

__device__ int gn_run(Ctx& c, const TinyGn& cfg, double xnorm2, int& iters, double& final_r, double& best_r) {
    const int N = c.N, R = c.R, S = c.S;
    iters = 0;
    final_r = 1.0;
    best_r = 1.0;
    if (!all_finite(c, c.A, S)) return -1;  // model.validate()
    double lambda = cfg.lambda;
    int direction = cfg.direction;
    for (int iter = 1; iter <= cfg.max_iters; ++iter) {
        // gn_step (gauss_newton.cpp:360-449)
        for (int n = 0; n < N; ++n) mttkrp_tree(c, n, c.M + c.P->off[n]);
        for (int n = 0; n < N; ++n) gram(c, c.A + c.P->off[n], c.P->dims[n], c.grams + n * R * R);
        for (int e = threadIdx.x; e < N * N * R * R; e += nthr()) {  // build_gamma_set (kruskal.cpp:42-65)
            const int np = e / (R * R), w = e % (R * R);
            const int n = np / N, p = np % N;
            const int lo = min(n, p), hi = max(n, p);
            double g = 1.0;
            for (int m = 0; m < N; ++m)
                if (m != lo && m != hi) g = fmul(g, c.grams[m * R * R + w]);
            c.pairs[e] = g;
        }
        __syncthreads();
        const double res = residual(c, xnorm2, c.M + c.P->off[N - 1], true);
        if (res < cfg.residual_tol) return 0;  // halt: converged_residual
        for (int e = threadIdx.x; e < S; e += nthr()) {  // gradient (:81-94): A_n Gamma(n,n) - M_n
            int n, i, r;
            stacked_index(c, e, n, i, r);
            const double* an = c.A + c.P->off[n];
            const double* gnn = c.pairs + (n * N + n) * R * R;
            double acc = 0.0;
            for (int kk = 0; kk < R; ++kk) acc = fadd(acc, fmul(an[i * R + kk], gnn[kk * R + r]));
            c.G[e] = fsub(acc, c.M[e]);
        }
        __syncthreads();
        double gnorm = 0.0;
        if (threadIdx.x == 0)
            for (int n = 0; n < N; ++n) {
                double s = 0.0;
                for (int i = c.P->off[n]; i < c.P->off[n + 1]; ++i) s = fadd(s, fmul(c.G[i], c.G[i]));
                gnorm = fadd(gnorm, __dsqrt_rn(s));
            }
        gnorm = bcast(c, gnorm);
        if (gnorm <= cfg.grad_tol) return 1;  // halt: converged_step
        int flags = 0;
        const int cgit = cp_cg(c, cfg, lambda, gnorm, flags);
        if (cgit < 0) return -1;
        double alpha = 1.0, res_after = -1.0;
        if (cfg.armijo) {
            const double f0 = fmul(fmul(fmul(0.5, res), res), xnorm2);
            const double gv = dot_sum(c, c.G, c.V);
            for (int e = threadIdx.x; e < S; e += nthr()) c.At[e] = c.A[e];  // model
            __syncthreads();
            bool accepted = false;
            for (int t = 0; t < cfg.max_backtracks; ++t) {
                for (int e = threadIdx.x; e < S; e += nthr()) c.A[e] = fadd(c.At[e], fmul(alpha, c.V[e]));
                __syncthreads();
                c.root_ok[0] = c.root_ok[1] = false;
                const double r_trial = residual(c, xnorm2, nullptr);
                const double f_trial = fmul(fmul(fmul(0.5, r_trial), r_trial), xnorm2);
                if (f_trial <= fadd(f0, fmul(fmul(cfg.c1, alpha), gv))) {
                    accepted = true;
                    res_after = r_trial;
                    break;
                }
                alpha = fmul(alpha, cfg.shrink);
            }
            if (!accepted) {
                for (int e = threadIdx.x; e < S; e += nthr()) c.A[e] = fadd(c.At[e], fmul(alpha, c.V[e]));
                __syncthreads();
                c.root_ok[0] = c.root_ok[1] = false;
                res_after = residual(c, xnorm2, nullptr);
            }
        } else {
            for (int e = threadIdx.x; e < S; e += nthr()) c.A[e] = fadd(c.A[e], c.V[e]);
            __syncthreads();
        }
        double step = 0.0;
        if (threadIdx.x == 0)
            for (int n = 0; n < N; ++n) {
                double s = 0.0;
                for (int i = c.P->off[n]; i < c.P->off[n + 1]; ++i) s = fadd(s, fmul(c.V[i], c.V[i]));
                step = fadd(step, fmul(alpha, __dsqrt_rn(s)));
            }
        step = bcast(c, step);
        c.root_ok[0] = c.root_ok[1] = false;
        if (!all_finite(c, c.A, S)) return -1;
        if (res_after < 0.0) res_after = residual(c, xnorm2, nullptr);
        // schedule_next (:47-59)
        if (cfg.mode == 1) {
            if (direction == 0) {
                lambda = fdiv(lambda, cfg.mu);
                if (lambda < cfg.lower) direction = 1;
            } else {
                lambda = fmul(lambda, cfg.mu);
                if (lambda > cfg.upper) direction = 0;
            }
        }
        iters = iter;
        final_r = res_after;
        best_r = fmin(best_r, res_after);
        if (res_after < cfg.residual_tol) return 0;
        if (step < cfg.step_tol) return 1;
    }
    return 2;
}

__global__ void __launch_bounds__(kTinyThreads) tiny_kernel(const __grid_constant__ TinyParams P) {
    extern __shared__ double sm[];
    const int inst = blockIdx.x;
    if (inst >= P.count) return;
    Ctx c;
    c.P = &P;
    c.N = P.order;
    c.R = P.rank;
    c.S = P.S;
    const TinyLayout& L = P.layout;
    c.X = sm + L.x;
    c.A = sm + L.a;
    c.root[0] = sm + L.root0;
    c.root[1] = sm + L.root1;
    c.root_ok[0] = c.root_ok[1] = false;
    c.T[0] = sm + L.t0;
    c.T[1] = sm + L.t1;
    c.grams = sm + L.grams;
    c.gam = sm + L.gam;
    c.L = sm + L.l;
    c.inv = sm + L.inv;
    c.misc = sm + L.misc;
    c.M = sm + L.m;
    c.add = sm + L.add;
    c.G = sm + L.g;
    c.V = sm + L.v;
    c.Rr = sm + L.r;
    c.Z = sm + L.z;
    c.W = sm + L.w;
    c.Q = sm + L.q;
    c.At = sm + L.at;
    c.pairs = sm + L.pairs;
    c.pinv = sm + L.pinv;
    c.tb = sm + L.tb;
    c.td = sm + L.td;
    c.bp = sm + L.bp;

    const double* xsrc = P.x + static_cast<long long>(P.x_index[inst]) * P.numel;
    for (int e = threadIdx.x; e < P.numel; e += blockDim.x) c.X[e] = xsrc[e];
    const double* a0 = P.init + static_cast<long long>(inst) * P.S;
    for (int e = threadIdx.x; e < P.S; e += blockDim.x) c.A[e] = a0[e];
    __syncthreads();
    double xn2 = 0.0;  // DenseTensor::norm2 (tensor.cpp:61-67), ascending
    if (threadIdx.x == 0)
        for (int e = 0; e < P.numel; ++e) xn2 = fadd(xn2, fmul(c.X[e], c.X[e]));
    xn2 = bcast(c, xn2);
    int status, iters = 0;
    double final_r = 1.0, best_r = 1.0;
    if (!(xn2 > 0.0)) {
        status = -1;  // InvalidArgument in the optimiser -> numerical_failure
    } else if (P.optimizer == 0) {
        status = als_run(c, P.als, xn2, iters, final_r, best_r);
    } else {
        status = gn_run(c, P.gn, xn2, iters, final_r, best_r);
    }
    if (status < 0) {  // run_instance: any Error -> numerical_failure with a fresh result
        status = 3;
        iters = 0;
        final_r = 1.0;
        best_r = 1.0;
    }
    if (threadIdx.x == 0) {
        P.status[inst] = status;
        P.iterations[inst] = iters;
        P.final_residual[inst] = final_r;
        P.best_residual[inst] = best_r;
    }
    if (P.factors_out)
        for (int e = threadIdx.x; e < P.S; e += blockDim.x) P.factors_out[static_cast<long long>(inst) * P.S + e] = c.A[e];
}

}  // namespace

// ---- host ------------------------------------------------------------------------------
bool tiny_layout(int order, const std::uint64_t* dims, int rank, TinyLayout& L, int& numel, int& S) {
    if (order < 2 || order > kTinyMaxOrder || rank < 1 || rank > kTinyMaxRank) return false;
    long long P = 1, smax = 0, ssum = 0;
    for (int n = 0; n < order; ++n) {
        P *= static_cast<long long>(dims[n]);
        smax = std::max<long long>(smax, dims[n]);
        ssum += static_cast<long long>(dims[n]);
    }
    if (P > (1 << 16)) return false;
    const int h = (order + 1) / 2;
    long long pf = 1, pb = 1, smin = smax;
    for (int n = 0; n < order; ++n) {
        (n < h ? pf : pb) *= static_cast<long long>(dims[n]);
        smin = std::min<long long>(smin, dims[n]);
    }
    const long long R = rank, RR = R * R;
    const long long tmax = std::max<long long>(P / std::max<long long>(1, smin) * R, smax * R);
    long long at = 0;
    auto take = [&](long long n) {
        const long long o = at;
        at += (n + 1) & ~1LL;  // keep 16-byte alignment
        return static_cast<int>(o);
    };
    S = static_cast<int>(ssum * R);
    numel = static_cast<int>(P);
    L.x = take(P);
    L.a = take(S);
    L.root0 = take(pf * R);
    L.root1 = take(pb * R);
    L.t0 = take(tmax);
    L.t1 = take(tmax);
    L.grams = take(order * RR);
    L.gam = take(RR);
    L.l = take(RR);
    L.inv = take(RR);
    L.misc = take(4 + kTinyMaxOrder);
    L.m = take(S);
    L.add = take(std::max<long long>(smax * R, RR));
    L.g = take(S);
    L.v = take(S);
    L.r = take(S);
    L.z = take(S);
    L.w = take(S);
    L.q = take(S);
    L.at = take(S);
    L.pairs = take(static_cast<long long>(order) * order * RR);
    L.pinv = take(order * RR);
    L.tb = take(std::max<long long>(smax * R, RR));
    L.td = take(RR);
    L.bp = take(order * RR);
    L.total = static_cast<int>(at);
    return static_cast<std::size_t>(L.total) * sizeof(double) <= kTinySmemMax;
}

void launch_tiny(const TinyParams& p, cudaStream_t st) {
    const std::size_t smem = static_cast<std::size_t>(p.layout.total) * sizeof(double);
    ensure_dynamic_smem(tiny_kernel, smem);
    tiny_kernel<<<p.count, p.threads > 0 ? p.threads : kTinyThreads, smem, st>>>(p);
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
}

}  // namespace cpkit
