// Internal declarations shared by the host drivers and the sm_100a kernels.
//
// Layout conventions follow the reference exactly (tensor.hpp:14-16,
// matrix_ops.hpp:7-10): every array is fp64, row-major, last index fastest.
// Factors A^(n) are s_n x R row-major; a tensor of order N is viewed as the
// (F x B) row-major matrix with F = prod_{m<h} s_m, B = prod_{m>=h} s_m and
// h = ceil(N/2), the reference's front/back split (mttkrp.cpp:166-178).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace cpkit {

// ---- exception taxonomy (reference errors.hpp:9-49); mapped to cpkit_status
// codes at the C ABI (cpkit.h:30-39).
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class InvalidArgument : public Error { public: using Error::Error; };
class SingularSystem : public Error { public: using Error::Error; };
class NumericalFailure : public Error { public: using Error::Error; };
class LimitExceeded : public Error { public: using Error::Error; };
class IoError : public Error { public: using Error::Error; };
class ParseError : public Error { public: using Error::Error; };
// CUDA / NCCL runtime failures (mapped to CPKIT_ERR_INTERNAL).
class DeviceError : public Error { public: using Error::Error; };

#define CPK_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::cpkit::DeviceError(std::string("CUDA error ") + cudaGetErrorString(e_) + \
                                       " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

// ---- NVTX ranges around the host-side phases (upload, generation, root
// contractions, the CG solve, ALS sweeps, GN steps): the reference's only
// instrumentation is steady_clock around a sweep (als.cpp:67-81); here a
// profiler (ncu --nvtx --nvtx-include "cpkit:root_back/") can select a phase
// by name. Header-only NVTX v3: one pointer test per call with no tool attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- guarded allocation mode (CPKIT_GUARD=1; runtime.cu). compute-sanitizer
// is not available on the GPU pool, so out-of-bounds WRITES are caught here:
// every DevBuf sits between two kGuardBytes red zones filled with kGuardByte,
// and each red zone is checked when the buffer is released (after a device
// synchronisation); a changed byte is reported on stderr and counted
// (cpkit_dev_guard_violations). Out-of-bounds READS return the pattern, which
// the parity tests then see as wrong results.
constexpr std::size_t kGuardBytes = 64 * 1024;
constexpr unsigned char kGuardByte = 0xA5;
bool guard_enabled();
void* guard_alloc(std::size_t bytes);                 // returns the user pointer
void guard_free(void* user, std::size_t bytes);       // checks both red zones, frees
std::uint64_t guard_violations();
// Plain device allocations of DevBuf (runtime.cu). cudaMalloc / cudaFree each
// cost milliseconds on the B200 boxes (a device problem holds ~50 buffers),
// so buffers released inside an OwnerSyncedRelease scope - their owner has
// synchronised every stream that used them - go to a per-device cache keyed
// by size and are handed out again without a driver call; every other release
// is a cudaFree (which orders itself after in-flight work). An allocation that
// fails empties the device's cache and retries. CPKIT_NO_ALLOC_CACHE=1 turns
// the cache off; CPKIT_ALLOC_TRACE=1 reports driver calls slower than 2 ms.
void* dev_alloc(std::size_t bytes);
void dev_free(void* p, std::size_t bytes);
void dev_cache_empty();  // every device: cached blocks back to the driver
std::size_t dev_cache_bytes();  // bytes cached for the current device
// Small pinned host blocks (diagnostic slots, mapped flags) from a process-wide
// free list: cudaFreeHost was measured taking up to 0.7 s on the B200 hosts
// (page unpinning), so the blocks are allocated once (portable, and mapped
// when asked) and recycled, never returned to the driver.
void* pinned_small_alloc(std::size_t bytes, bool mapped);
void pinned_small_free(void* p, std::size_t bytes, bool mapped);
struct OwnerSyncedRelease {  // thread-local scope flag read by dev_free
    OwnerSyncedRelease();
    ~OwnerSyncedRelease();
    OwnerSyncedRelease(const OwnerSyncedRelease&) = delete;
    OwnerSyncedRelease& operator=(const OwnerSyncedRelease&) = delete;
};
bool guard_selftest();  // positive control (CPKIT_GUARD=1 only)
// The red-zone check synchronises the device, which would invalidate another
// thread's CUDA-graph capture: in guard mode captures and checks take this lock.
std::recursive_mutex& guard_capture_mutex();

// ---- owning device buffer
template <typename T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(std::size_t n) { resize(n); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), guarded_(o.guarded_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            guarded_ = o.guarded_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void resize(std::size_t n) {
        if (n == n_) return;
        release();
        if (n) {
            guarded_ = guard_enabled();
            if (guarded_) p_ = static_cast<T*>(guard_alloc(n * sizeof(T)));
            else p_ = static_cast<T*>(dev_alloc(n * sizeof(T)));
        }
        n_ = n;
    }
    void ensure(std::size_t n) { if (n > n_) resize(n); }
    void release() {
        if (p_) {
            if (guarded_) guard_free(p_, n_ * sizeof(T));
            else dev_free(p_, n_ * sizeof(T));
        }
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    std::size_t n_ = 0;
    bool guarded_ = false;
};

// ---- kernel launch accounting (runtime.cu)
void count_launch(int n);
std::uint64_t kernel_launches();

// ---- per-device launch attributes, safe for concurrent solves (runtime.cu)
// SM count of the current device (cached per device).
int device_sm_count();
// Raise fn's dynamic shared-memory limit on the current device to at least
// `bytes`: grow-only per (device, function) under one process-wide mutex, so
// a solve on another thread can never lower it under this one's launch.
void ensure_dynamic_smem(const void* fn, std::size_t bytes);
// Cooperative (grid-barrier) kernels of different streams must not run at the
// same time on one device: two partially resident grids could wait on each
// other's SMs. Every cooperative launch goes through this: the stream waits for
// the device's previous cooperative launch, launches, and becomes the new tail.
void launch_cooperative(const void* fn, dim3 grid, dim3 block, void** args, std::size_t smem, cudaStream_t st);
// Cooperative launch in clusters of cluster_x CTAs (cudaLaunchKernelEx with the
// cooperative and cluster-dimension attributes), serialised like launch_cooperative.
void launch_cooperative_cluster(const void* fn, dim3 grid, dim3 block, unsigned cluster_x, void** args,
                                std::size_t smem, cudaStream_t st);
// Clusters of cluster_x CTAs of fn that can be resident at once (cached per device).
int max_active_clusters(const void* fn, dim3 block, unsigned cluster_x, std::size_t smem);
template <typename F>
inline void ensure_dynamic_smem(F* fn, std::size_t bytes) {
    ensure_dynamic_smem(reinterpret_cast<const void*>(fn), bytes);
}

// ---- device launch helpers (implemented in kernels_*.cu) -------------------

constexpr int kMaxOrder = 16;

// Shape of a KRP operand: the (sub)tensor index k over `nmodes` consecutive
// modes decomposes row-major; value(k, r) = prod_j factor_j[i_j(k), r].
struct KrpDesc {
    int nmodes = 0;
    std::int64_t ext[kMaxOrder] = {};      // extents, slowest first
    const double* fac[kMaxOrder] = {};     // factor pointers (s_j x R row-major)
};

// MTTKRP root contractions (kernels_mttkrp.cu). X is F x B stored with an
// even row stride Bs >= B (TMA needs 16-byte strides); krp is a K x Rs
// workspace (krp_workspace_elems) filled with the Khatri-Rao operand.
//   back root:  P_F[F x R] = X[F x B] * KRP_B        (NN)
//   front root: P_B[B x R] = X[F x B]^T * KRP_F      (TN, split-K)
// reserve_sms: SMs to leave to a concurrent side-stream kernel during the full waves
void launch_root_back(const double* x, std::int64_t F, std::int64_t B, std::int64_t Bs, int R,
                      const KrpDesc& kb, double* krp, double* pf, double* splitk_ws, std::size_t splitk_ws_elems,
                      cudaStream_t st, int reserve_sms = 0);
std::size_t root_back_workspace_elems(std::int64_t F, std::int64_t B, int R);
void launch_root_front(const double* x, std::int64_t F, std::int64_t B, std::int64_t Bs, int R,
                       const KrpDesc& kf, double* krp, double* pb, double* splitk_ws,
                       std::size_t splitk_ws_elems, cudaStream_t st);
std::size_t root_front_workspace_elems(std::int64_t F, std::int64_t B, int R);
// order-3 multi-sweep dimension tree: single-mode root contraction of mode c in {0, 1}
void launch_root_single(const double* x, std::int64_t s0, std::int64_t s1, std::int64_t Bl, std::int64_t Bs, int c,
                        const double* fac, int R, double* out, double* ws, std::size_t ws_elems, cudaStream_t st);
std::size_t root_single_workspace_elems(std::int64_t s0, std::int64_t s1, std::int64_t Bs, int R);
// out[b][c][r] = in[b][r][c] (the multi-sweep tree's mode-permuted tensor copies)
void launch_transpose_batched(const double* in, std::int64_t batch, std::int64_t rows, std::int64_t cols,
                              std::int64_t in_ld, std::int64_t in_bs, double* out, std::int64_t out_ld,
                              std::int64_t out_bs, cudaStream_t st);
std::size_t krp_workspace_elems(std::int64_t rows, int R);

// Second dimension-tree level: P over kept modes (ext[0..k), R) reduced to the
// single kept mode `keep`, weighting by the other kept modes' factor rows.
void launch_reduce_kept(const double* p, const KrpDesc& kept, int keep, int R, double* out,
                        double* ws, std::size_t ws_elems, cudaStream_t st);
std::size_t reduce_kept_workspace_elems(const KrpDesc& kept, int keep, int R);

// Small dense kernels (kernels_small.cu).
void launch_norm2(const double* x, std::uint64_t n, double* partials, int nparts, double* out,
                  cudaStream_t st);
int norm2_parts(std::uint64_t n);
// grams of modes [lo, hi): factor n at base + offs[n] (device arrays), rows[n];
// ws holds gram_workspace_elems(hi - lo, R, max rows) doubles.
std::size_t gram_workspace_elems(int nmodes, int R, std::int64_t smax);
// sq != null: the first CTA also adds sqrt(sum of sq[0..nsq)) to *sq_acc (ALS step norm)
void launch_grams(const double* base, const std::int64_t* offs, const std::int64_t* rows, int lo,
                  int hi, int R, std::int64_t smax, double* ws, double* grams, cudaStream_t st,
                  const double* sq = nullptr, int nsq = 0, double* sq_acc = nullptr);
// pair[(n*order+p)] = Hadamard over grams m not in {n,p} ascending (kruskal.cpp:42-65)
void launch_gamma_pairs(const double* grams, int order, int R, double* pair, cudaStream_t st);
// gamma_one = Hadamard over grams m != n (als.cpp:34-37)
void launch_gamma_excl(const double* grams, int order, int R, int n, double* out, cudaStream_t st);
// scal[0..] <- residual pieces; writes r,f into out2 (kruskal.cpp:94-118)
void launch_residual(const double* m_last, const double* a_last, std::int64_t rows, const double* grams,
                     int order, int R, const double* xnorm2, double* partials, double* out2,
                     cudaStream_t st);
// G_n = A_n * Gamma(n,n) - M_n  (gauss_newton.cpp:81-94)
void launch_gradient(const double* a, const double* gnn, const double* m, std::int64_t rows, int R,
                     double* g, cudaStream_t st);
// G for every mode in one launch (off: N + 1 stacked offsets, rows: N extents)
void launch_gradient_all(const double* a, const double* pair, const double* m, const std::int64_t* off,
                         const std::int64_t* rows, int order, int R, double* g, cudaStream_t st);
// out = sum_n scale*||X_n||_F (per-block Frobenius norms, summed in block order)
void launch_block_norm_sum(const double* x, const std::int64_t* offsets, int nblocks,
                           double* partials, double* out, double scale, cudaStream_t st);
// y += alpha * x ; writes finite flag
void launch_axpy(double* y, const double* x, double alpha, std::uint64_t n, cudaStream_t st);
// out = ||a - b||_F accumulated into *acc (adds); deterministic per call
void launch_diff_norm_add(const double* a, const double* b, std::uint64_t n, double* partials,
                          double* acc, cudaStream_t st);
void launch_dot(const double* a, const double* b, std::uint64_t n, double* partials, double* out,
                cudaStream_t st);
// out = a + alpha * x
void launch_axpby(double* out, const double* a, double alpha, const double* x, std::uint64_t n,
                  cudaStream_t st);
void launch_all_finite(const double* x, std::uint64_t n, int* flag, cudaStream_t st);
void launch_set_flag_scalar(int* flag, int fv, double* d, double dv, cudaStream_t st);
void launch_pack_values(const double* d, int nd, const int* iv, int ni, double* out_mapped, cudaStream_t st);
// GN update A += V with the step norm (sum of per-mode norms), the finiteness
// flag and the packed CG result / step diagnostics, in one launch.
void launch_gn_apply(double* a, const double* v, const std::int64_t* offsets, int nblocks, double* partials,
                     int* bad_part, unsigned int* counter, const int* cgres, int ncg, double* out_cg,
                     double* step_out, double* step_slot_zero, int* flag, double* out_step, cudaStream_t st);
void launch_pack_sweep(const double* scal, int kstep, int kres, const int* flag, const int* status, int n,
                       double* out_mapped, cudaStream_t st);
// Dense evaluation of a Kruskal model + keyed-RNG noise (generators / reconstruct)
void launch_reconstruct(const KrpDesc& all, int R, double* out, std::uint64_t offset, std::uint64_t n,
                        cudaStream_t st);
// Keyed noise (keyed_noise.cuh), bit-identical to the CPU restatement and
// independent of the GPU count. Slab view: rows (all modes but the last) x
// slab columns (this rank's last-mode indices, global offset slab_lo).
std::size_t noise_workspace_elems(std::int64_t slab);
// colsq[0..slab) = per-column sum of X^2, colsq[slab..2 slab) = of E^2 (ws: noise_workspace_elems)
void launch_noise_colsq(const double* x, std::int64_t rows, std::int64_t slab, std::uint64_t seed,
                        std::uint64_t s_last, std::uint64_t slab_lo, double* ws, double* colsq, cudaStream_t st);
// out3 = [rel ||X|| / ||E||, ||X||^2, ||E||^2] from every rank's [X cols | E cols] block (rank-major)
void launch_noise_scale(const double* colsq_all, int world, std::int64_t slab, double rel, double* out3,
                        cudaStream_t st);
// x += scale[0] * E (no fused multiply-add)
void launch_noise_add(double* x, std::uint64_t n, std::uint64_t slab, std::uint64_t s_last, std::uint64_t slab_lo,
                      std::uint64_t seed, const double* scale, cudaStream_t st);

// Cholesky-based SPD kernels (kernels_chol.cu); status: 0 ok, 1 ok after jitter, 2 singular
// chol_factor_elems(count, R) doubles hold the factors (row stride R + 1).
std::size_t chol_factor_elems(int count, int R);
// factor count matrices (contiguous R x R); lambda is a host value; mode 0:
// S + lambda I, mode 1: diag(S) *= (1 + lambda). Lower L per matrix.
void launch_chol_batch(const double* s, int count, int R, const double* lambda, int mode,
                       double* l_out, int* status, cudaStream_t st);
void launch_chol_batch_src(double* s, const double* grams, int order, int excl, int count, int R,
                           const double* lambda, int mode, double* l_out, int* status, cudaStream_t st,
                           long long s_stride = 0);
void launch_chol_batch_strided(const double* s, long long s_stride, int count, int R, const double* lambda, int mode,
                               double* l_out, int* status, cudaStream_t st);
// ALS update: a <- rows solved in place, row_sq[i] = ||a_new_i - a_old_i||^2
void launch_chol_solve_rows_update(const double* l, int R, const double* b, std::int64_t rows, double* a,
                                   double* row_sq, cudaStream_t st);
// *acc += sqrt(sum of n partials)
void launch_sqrt_add(const double* partials, int n, double* acc, cudaStream_t st);
void launch_chol_solve_rows(const double* l, int R, const double* b, std::int64_t rows, double* y,
                            cudaStream_t st);
void launch_chol_inverse_batch(const double* l, int count, int R, double* inv, double* tmp,
                               cudaStream_t st);

// Persistent CG (kernels_cg.cu)
struct CgParams {
    int order = 0;
    int R = 0;
    std::int64_t rows[kMaxOrder] = {};
    std::int64_t off[kMaxOrder + 1] = {};  // block offsets (elements) in stacked s x R buffers
    const double* A = nullptr;     // stacked factors
    const double* pair = nullptr;  // order*order*R*R gamma blocks
    const double* pinv = nullptr;  // order*R*R preconditioner inverses
    const double* G = nullptr;     // gradient
    double* V = nullptr;
    double* Rr[2] = {nullptr, nullptr};
    double* W[2] = {nullptr, nullptr};
    double* Z = nullptr;
    double* Q = nullptr;
    double* Bp = nullptr;          // order*R*R
    double* slots = nullptr;       // per-task partial sums
    int nslots = 0;
    unsigned int* barrier = nullptr;
    double lambda = 0.0;
    int shape = 0;                 // 0 identity, 1 diagonal
    int beta_variant = 0;          // 0 standard, 1 stale denominator
    double cg_tol = 1e-3;
    int cap = 0;
    int* result = nullptr;         // [iters, hit_cap, breakdown, nonfinite, final_buffer]
    unsigned long long* trace = nullptr;  // optional: CTA 0 phase timestamps (ns), 8 per iteration
    bool barrier_zeroed = false;   // the caller guarantees barrier[] is zero (no memset before the launch)
};
void run_cg(const CgParams& p, int grid, cudaStream_t st);
// tile-resident CG (kernels_cg_res.cu); false when the problem does not fit it
bool run_cg_resident(const CgParams& p, cudaStream_t st);
std::size_t cg_res_slots_needed(const CgParams& p);
constexpr int cg_barrier_words() { return 4 + 1024; }  // grid barrier, CTA-order counters, per-SM slots
int cg_max_grid(int device);
std::size_t cg_slots_needed(const CgParams& p);
// U = J^T J W + lambda Reg(W) (same task code as the CG phases)
void launch_jtj_matvec(const CgParams& p, const double* w, double* u, cudaStream_t st);

// FP64 DMMA issue-rate probe (TFLOP/s), used as the measured roofline peak.
double probe_dmma_peak(int device);

}  // namespace cpkit
