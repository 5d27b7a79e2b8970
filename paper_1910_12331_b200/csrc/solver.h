// Host-side mirror of the reference solver API (cpkit::DenseTensor,
// KruskalModel, RegSchedule, GnConfig, AlsConfig, ConvergenceReport and the
// als_optimize / gn_optimize drivers), re-implemented over device-resident
// state. Reference headers: tensor.hpp, kruskal.hpp, gauss_newton.hpp,
// als.hpp, report.hpp, mttkrp.hpp.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "common.h"

namespace cpkit {

// ---------------------------------------------------------------- host types
// Row-major fp64 matrix (matrix_ops.hpp:9-10).
struct Matrix {
    std::int64_t rows = 0, cols = 0;
    std::vector<double> data;
    Matrix() = default;
    Matrix(std::int64_t r, std::int64_t c) : rows(r), cols(c), data(static_cast<std::size_t>(r * c), 0.0) {}
    double norm() const;
    bool all_finite() const;
};

inline constexpr std::uint64_t kDefaultElementCap = 100'000'000ull;  // tensor.hpp:12

std::uint64_t product_of_dims(const std::vector<std::uint64_t>& dims);

// Host storage of a dense tensor: page-locked (cudaHostAlloc) when a CUDA
// device is present, so an upload is one direct DMA at full link bandwidth with
// no driver staging copy; ordinary heap memory otherwise (e.g. CPU-only hosts).
// Not initialised on allocation.
class HostArray {
public:
    HostArray() = default;
    explicit HostArray(std::size_t n);
    ~HostArray();
    HostArray(const HostArray&) = delete;
    HostArray& operator=(const HostArray&) = delete;
    HostArray(HostArray&& o) noexcept : p_(o.p_), n_(o.n_), pinned_(o.pinned_) { o.p_ = nullptr; o.n_ = 0; }
    HostArray& operator=(HostArray&& o) noexcept;
    double* data() { return p_; }
    const double* data() const { return p_; }
    std::size_t size() const { return n_; }
    bool pinned() const { return pinned_; }

private:
    double* p_ = nullptr;
    std::size_t n_ = 0;
    bool pinned_ = false;
};

// tensor.hpp:16-48 (host copy; the device copy lives in DeviceProblem)
class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(std::vector<std::uint64_t> dims);  // zero-filled
    static DenseTensor from_data(std::vector<std::uint64_t> dims, std::vector<double> data);
    // copies n = prod(dims) doubles from src (threaded for large tensors)
    static DenseTensor copy_of(std::vector<std::uint64_t> dims, const double* src);
    static DenseTensor adopt(std::vector<std::uint64_t> dims, HostArray data);
    std::size_t order() const { return dims_.size(); }
    std::uint64_t extent(std::size_t m) const { return dims_[m]; }
    const std::vector<std::uint64_t>& dims() const { return dims_; }
    std::uint64_t size() const { return data_.size(); }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    bool pinned() const { return data_.pinned(); }
    void validate() const;

private:
    std::vector<std::uint64_t> dims_;
    HostArray data_;
};

// kruskal.hpp:15-26
struct KruskalModel {
    std::vector<std::uint64_t> dims;
    std::int64_t rank = 0;
    std::vector<Matrix> factors;
    std::size_t order() const { return dims.size(); }
    void validate() const;
};

// CPKT1 / CPKM1 binary formats (tensor.cpp:197-239, kruskal.cpp:143-203)
void write_tensor(const DenseTensor& t, const std::string& path);
DenseTensor read_tensor(const std::string& path);
// CPKT1 header: extents (and the byte offset of the data)
std::vector<std::uint64_t> read_tensor_header(const std::string& path, std::uint64_t* data_offset);
void write_model(const KruskalModel& m, const std::string& path);
KruskalModel read_model(const std::string& path);

// ---------------------------------------------------------------- configs
enum class RegMode { constant, varying };
enum class RegShape { identity, diagonal };
struct RegSchedule {  // gauss_newton.hpp:19-34
    RegMode mode = RegMode::constant;
    RegShape shape = RegShape::identity;
    double lambda = 1e-3, mu = 2.0, lower = 1e-6, upper = 1e-2;
    enum class Direction { down, up };
    Direction direction = Direction::down;
    static RegSchedule constant(double lambda, RegShape shape = RegShape::identity);
    static RegSchedule varying(double upper = 1e-2, double lower = 1e-6, double mu = 2.0,
                               RegShape shape = RegShape::identity);
    void validate() const;
};
RegSchedule schedule_next(RegSchedule s);  // gauss_newton.cpp:47-59

enum class CgBetaVariant { standard, stale_denominator };
struct ArmijoParams {
    double c1 = 1e-4, shrink = 0.5;
    int max_backtracks = 20;
};
struct GnConfig {  // gauss_newton.hpp:50-62
    double grad_tol = 0.0, residual_tol = 5e-5, step_tol = 1e-7;
    int max_iters = 500;
    double cg_tol = 1e-3;
    int cg_max_iters = 0;
    RegSchedule schedule = RegSchedule::varying();
    std::optional<ArmijoParams> armijo;
    CgBetaVariant cg_beta = CgBetaVariant::standard;
    // residual_after from a third, uncached contraction of the stepped factors
    // (the reference's semantics, gauss_newton.cpp:442-444) instead of the next
    // iteration's tree pass. JSON gn.residual_after = "naive" | "tree" (default),
    // or CPKIT_GN_REF_RESIDUAL=1.
    bool residual_naive = false;
    void validate() const;
};
struct AlsConfig {  // als.hpp:11-22
    int max_sweeps = 10000;
    double residual_tol = 5e-5, step_tol = 1e-7, lambda0 = 0.0, decay_factor = 2.0;
    std::optional<int> decay_every;
    void validate() const;
};

// ---------------------------------------------------------------- reports
enum class TerminalStatus { converged_residual, converged_step, cap_hit, numerical_failure };
const char* to_string(TerminalStatus s);
struct TraceRecord {  // report.hpp:21-28
    int iteration = 0;
    double residual = 0.0, fitness = 0.0, lambda = 0.0;
    int cg_iters = 0;
    double seconds = 0.0;
};
struct ConvergenceReport {
    std::vector<TraceRecord> records;
    TerminalStatus status = TerminalStatus::cap_hit;
    double final_residual() const { return records.empty() ? 1.0 : records.back().residual; }
    double best_residual() const;
};

struct GnStepDiag {  // gauss_newton.hpp:117-131
    enum class Halt { none, residual, gradient };
    Halt halt = Halt::none;
    bool stepped = false;
    double residual_before = 1.0, residual_after = 1.0, grad_norm = 0.0, lambda = 0.0;
    int cg_iters = 0;
    double step_norm = 0.0, alpha = 1.0;
    bool armijo_exhausted = false, cg_hit_cap = false, cg_breakdown = false;
};
struct AlsSweepDiag {  // als.hpp:24-28 (last-mode MTTKRP stays on device)
    double step_norm = 0.0;
    int full_contractions = 0;
};
struct CgResultInfo {
    int iterations = 0;
    bool hit_cap = false, breakdown = false;
};

// ---------------------------------------------------------------- device layer
// Collective hooks for last-mode sharding (NCCL over NVLink when world > 1).
class Comm {
public:
    virtual ~Comm() = default;
    virtual int rank() const = 0;
    virtual int world() const = 0;
    virtual void allreduce_sum(double* dev, std::size_t count, cudaStream_t st) = 0;
    // gather equal-size row blocks from every rank into dev_out (rank-major)
    virtual void allgather(const double* dev_in, double* dev_out, std::size_t count_per_rank,
                           cudaStream_t st) = 0;
};
std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int world);
// Test-only: `world` communicators of one in-process group on one device; each
// rank must be driven by its own host thread (runtime.cu, LoopbackGroup).
std::vector<std::unique_ptr<Comm>> make_loopback_comms(int world);
void nccl_unique_id(void* out128);

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;  // side stream: SPD factorisations overlap the MTTKRP
    cudaStream_t aux2 = nullptr;  // second-level reduces beside the next root GEMM (GN tree pass)
    static constexpr int kEvents = 2 * kMaxOrder + 6;
    static constexpr int kEvAux2A = 2 * kMaxOrder + 2, kEvAux2B = 2 * kMaxOrder + 3,
                         kEvBarrier = 2 * kMaxOrder + 4;  // third-stream hand-offs
    cudaEvent_t ev[kEvents] = {};
    std::unique_ptr<Comm> comm;  // null: single GPU
    explicit Context(int dev);
    ~Context();
    int rank() const { return comm ? comm->rank() : 0; }
    int world() const { return comm ? comm->world() : 1; }
    void sync() const;
    void sync_main() const;  // the solver stream only (side-stream work keeps running)
};

// Slab of the last mode owned by a rank (balanced contiguous split).
void shard_range(std::uint64_t extent, int rank, int world, std::uint64_t* lo, std::uint64_t* hi);

// Device-resident problem: the (local slab of the) tensor, the replicated
// factors, the dimension-tree cache (mttkrp.hpp:35-54) and every GN/ALS buffer.
class DeviceProblem {
public:
    // dims: global extents. local_data: the rank's slab (row-major over
    // dims with the last extent replaced by the slab size); host or device.
    DeviceProblem(Context& ctx, std::vector<std::uint64_t> dims, int rank);
    ~DeviceProblem();
    // H2D copy of the local slab. start (orders >= 4, single GPU): those
    // factors are set first and the back root contraction runs slab by slab
    // while the tensor crosses PCIe; a later set_factors(start) keeps it.
    void upload_tensor(const double* host_local, const KruskalModel* start = nullptr);
    // CPKT1 file -> device, streamed: chunks of whole last-mode rows are read into
    // two pinned staging buffers while the previous chunk crosses to HBM (this
    // rank's slab columns only); finiteness checked on the device (tensor.cpp:71-83)
    void load_tensor_file(const std::string& path);
    void generate_tensor(const KruskalModel& truth, std::uint64_t noise_seed, double noise_rel);
    double* tensor_device() { return x_.get(); }
    void download_tensor(double* host_local);
    std::uint64_t local_elems() const { return local_elems_; }

    int order() const { return static_cast<int>(dims_.size()); }
    int rank() const { return R_; }
    const std::vector<std::uint64_t>& dims() const { return dims_; }
    std::uint64_t slab_lo() const { return slab_lo_; }
    std::uint64_t slab_hi() const { return slab_hi_; }

    void set_factors(const std::vector<const double*>& host);  // host s_n x R blocks
    void get_factors(std::vector<double*>& host);
    void set_factors(const KruskalModel& m);
    void get_factors(KruskalModel& m);
    double* factors_device() { return A_.get(); }
    std::int64_t factor_offset(int n) const { return off_[n]; }

    // ---- reference seams
    double norm2();                                   // ||X||^2 (tensor.cpp:61-67)
    // reps x the second tree level (mttkrp.cpp:63-75) on the cached back-root partial, mode 0:
    // average ms per pass; *bytes = the partial's size (the pass's compulsory HBM traffic)
    double time_second_level(int reps, double* bytes);
    void mttkrp(int mode);                            // tree, into M block (mttkrp.cpp:160-189)
    void mttkrp_naive(int mode);                      // uncached, same kernels
    void note_factor_update(int mode);                // mttkrp.cpp:136-145
    void invalidate_all();
    int full_contractions() const { return contractions_; }
    void reset_contraction_counter() { contractions_ = 0; }
    const double* mttkrp_result(int mode) const { return M_.get() + off_[mode]; }
    void download_mttkrp(int mode, double* host);

    void build_gamma_set();                           // grams + pairwise (kruskal.cpp:42-65)
    void download_gammas(double* grams, double* pair);
    void upload_gammas(const double* grams, const double* pair);
    std::pair<double, double> residual_fitness(double xnorm2, int last_src);  // kruskal.cpp:94-118
    void residual_launch(double xnorm2);  // the same, result left in the scalar slots (no readback)
    void residual_launch_dev();           // the same with ||X||^2 already in its device slot
    void gradient();                                  // G (gauss_newton.cpp:81-94)
    double norm_sum(const double* dev_stacked);       // sum_n ||block_n||_F
    void jtj_matvec(const double* dev_w, double* dev_u, double lambda, RegShape shape);
    // V from G (gauss_newton.cpp:279-349); gnorm = sum_n ||G_n|| when the caller has it (< 0: computed)
    CgResultInfo cp_cg(double lambda, const GnConfig& cfg, double gnorm = -1.0);
    void build_preconditioner(double lambda, RegShape shape);
    // factor the preconditioner blocks on the side stream (joined by cp_cg)
    void launch_preconditioner_factor(double lambda, RegShape shape);
    void spd_solve(const double* dev_s, const double* dev_b, std::int64_t rows, double lambda,
                   double* dev_y);
    void spd_inverse(const double* dev_s, double lambda, double* dev_inv);

    AlsSweepDiag als_sweep(double lambda);            // als.cpp:22-52
    // Pipelined sweeps: launch queues one sweep (optionally followed by the
    // residual of its result, the driver's per-sweep check) and its packed
    // diagnostics without synchronising; finish waits for the oldest queued
    // sweep and decodes them (throws as als_sweep does). At most kSweepSlots
    // sweeps are in flight.
    void als_sweep_launch(double lambda, bool with_residual);
    AlsSweepDiag als_sweep_finish(double* res = nullptr, double* fit = nullptr);
    int als_sweeps_pending() const { return static_cast<int>(pending_.size() + done_.size()); }
    void als_snapshot_factors();   // A -> Atrial (device copy, stream-ordered)
    void als_restore_factors();    // Atrial -> A, caches dropped
    GnStepDiag gn_step(const GnConfig& cfg, RegSchedule& schedule, double xnorm2);  // :360-449
    // the same step with a host decision after every phase (Armijo needs it)
    GnStepDiag gn_step_sync(const GnConfig& cfg, RegSchedule& schedule, double xnorm2);
    static bool ref_residual(const GnConfig& cfg);  // GnConfig::residual_naive or CPKIT_GN_REF_RESIDUAL
    // the default step split for pipelining: queue it (slot 0/1: diagnostics,
    // pre-step snapshot, completion event), then decode it (a step that must not
    // have happened is undone from its slot's snapshot)
    void gn_enqueue(const GnConfig& cfg, const RegSchedule& schedule, double xnorm2, int slot);
    GnStepDiag gn_decode(const GnConfig& cfg, double lambda, int slot);
    void restore_factors_from(const double* dev_src);  // factors <- device copy, caches dropped
    // the last gn_decode threw after its step had been applied (non-finite update)
    bool gn_failed_applied() const { return gn_failed_applied_; }
    const double* gn_snapshot(int slot) const { return slot == 0 ? Atrial_.get() : Asnap1_.get(); }

private:
    // Side-stream chain for a GN step's preconditioner: [Grams + Gamma set,]
    // Cholesky of Gamma(n,n) (+ lambda) and its inverse into pinv_; records
    // ctx_.ev[1]. pinv_ready_ marks a chain launched ahead for (lambda, shape).
    void launch_precond_chain(double lambda, RegShape shape, bool grams_and_gamma);
    bool pinv_ready_ = false;
    bool gn_failed_applied_ = false;
    // the residual slots hold the residual of the current factors for res_xnorm_
    bool res_current_ = false;
    double res_xnorm_ = 0.0;
    // the CG grid barrier was re-zeroed on the solver stream after the last solve
    bool barrier_zero_ = false;
    void cg_barrier_ready() {}
    double pinv_lambda_ = 0.0;
    RegShape pinv_shape_ = RegShape::identity;

public:

    // stacked device buffers (N blocks of s_n x R)
    double* G() { return G_.get(); }
    double* V() { return V_.get(); }
    double* Wbuf() { return W_[0].get(); }
    double* Ubuf() { return Q_.get(); }
    double* grams() { return grams_.get(); }
    double* pairs() { return pair_.get(); }
    double* pinv() { return pinv_.get(); }
    std::int64_t stacked_elems() const { return off_[dims_.size()]; }
    Context& ctx() { return ctx_; }

    // Per-launch CUDA-event timing of the dominant kernels inside a timed region.
    enum ProfKind { kProfBack = 0, kProfFront = 1, kProfCg = 2, kProfKinds = 3 };
    void profile_enable(bool on);
    // total ms and launch count per kind since enable (syncs the stream)
    void profile_read(double* ms, int* count);

private:
    struct ProfEvent {
        cudaEvent_t a, b;
        int kind;
        float ms = -1.0f;  // >= 0: already measured (graph replays)
    };
    // ALS sweep as a CUDA graph: captured once per (lambda, cache state,
    // profiling) and replayed; host bookkeeping restored from the capture.
    struct SweepSig {
        bool pf, pb, mall, prof, grams;
        int pm;
        bool operator==(const SweepSig& o) const {
            return pf == o.pf && pb == o.pb && mall == o.mall && prof == o.prof && grams == o.grams && pm == o.pm;
        }
    };
    // (the multi-sweep tree alternates two cache states, so up to kAlsGraphs
    // captures are kept, keyed by lambda and the state at sweep start)
    struct AlsGraph {
        cudaGraphExec_t exec = nullptr;
        double lambda = 0.0;
        SweepSig pre{}, post{};
        int contr = 0;
        long long kernels = 0;  // kernel launches per replay (counted during capture)
        std::vector<ProfEvent> prof;  // event pairs recorded by the graph
    };
    static constexpr std::size_t kAlsGraphs = 4;
    std::vector<AlsGraph> als_graphs_;
    static constexpr int kSweepSlots = 4, kSlotDoubles = 4 + kMaxOrder;
    struct PendingSweep {
        int slot, contr;
        AlsGraph* graph;  // profiled replay whose event pairs are read at finish (or null)
    };
    std::vector<PendingSweep> pending_;  // FIFO
    struct SweepResult {
        AlsSweepDiag diag;
        double res = 1.0, fit = 0.0;
        int err = 0;  // 1 non-finite factor, 2 singular SPD system
    };
    std::vector<SweepResult> done_;  // completed, not yet handed to the caller (FIFO)
    SweepResult complete_oldest();   // waits for pending_.front() and decodes it
    void drain_pending() {
        while (!pending_.empty()) done_.push_back(complete_oldest());
    }
    int next_slot_ = 0;
    double* hmap_ = nullptr;  // mapped pinned slots (kSweepSlots x kSlotDoubles), then the GN step's area
    static constexpr int kGnMapOff = kSweepSlots * kSlotDoubles, kGnMapDoubles = 16 + 2 * kMaxOrder;
    static constexpr std::size_t kPinBytes = 16 * sizeof(double);
    static constexpr std::size_t kMapBytes = (kGnMapOff + 2 * kGnMapDoubles) * sizeof(double);
    double* dmap_ = nullptr;  // their device alias
    cudaEvent_t slot_ev_[kSweepSlots] = {};
    SweepSig sweep_sig() const { return {pf_valid_, pb_valid_, m_all_valid_, profile_, grams_valid_, pm_mode_}; }
    void drop_als_graph();
    void als_sweep_body(double lambda);
    bool profile_ = false;
    std::vector<ProfEvent> prof_;
    void prof_begin(int kind);
    void prof_end();

    Context& ctx_;
    std::vector<std::uint64_t> dims_;
    int R_ = 0, h_ = 0;
    std::uint64_t slab_lo_ = 0, slab_hi_ = 0, local_elems_ = 0;
    std::int64_t F_ = 0, Bl_ = 0, Bs_ = 0;           // local matrix view F x B_local, row stride Bs
    std::vector<std::int64_t> off_;                  // stacked offsets (elements)
    // armed by the destructor once every stream is idle: the DevBuf members
    // below (destroyed before it) then go back to the allocation cache
    std::optional<OwnerSyncedRelease> release_scope_;
    std::vector<double> preset_;  // factors the upload already contracted (upload_tensor with start)
    bool preset_valid_ = false;
    DevBuf<double> x_;
    DevBuf<double> A_, Atrial_, M_, G_, V_, Z_, Q_, Rr_[2], W_[2];
    DevBuf<double> PF_, PB_, ws_, krp_;
    bool pf_valid_ = false, pb_valid_ = false;
    // Order-3 ALS multi-sweep dimension tree: PM_ caches the single-mode root
    // P_c = X x_c A_c (c = pm_mode_ in {0, 1}; -1 = none). Every root serves
    // the next two mode updates, so a sweep pair needs 3 roots instead of 4.
    bool msdt_ = false;
    int pm_mode_ = -1;
    // a side-stream SPD factorisation is in flight: roots leave it one SM
    bool side_busy_ = false;
    DevBuf<double> PM_;
    // Mode-permuted copies of the local tensor, X^(0)[i1][i2][i0] and
    // X^(1)[i0][i2][i1] (row strides ld0_/ld1_, even for TMA), made once per
    // upload when memory allows: the single-mode roots then run as the same
    // NN GEMM as the back root instead of a TN GEMM with transposed operands.
    bool msdt_copies_ = false;
    std::int64_t ld0_ = 0, ld1_ = 0;
    DevBuf<double> X0_, X1_;
    DevBuf<double> Asnap1_;     // GN pre-step snapshot of slot 1 (slot 0: Atrial_)
    cudaEvent_t gn_ev_[2] = {}; // GN step completion per slot
    // Order >= 4: X^T [B_local][F] (row stride ldT_) when memory allows, so the
    // front root P_B = X^T KRP_F runs as the NN GEMM instead of the TN one.
    bool front_copy_ = false;
    std::int64_t ldT_ = 0;
    DevBuf<double> XT_;
    void build_msdt_copies();  // every layout copy of the tensor (MSDT copies, X^T)
    bool grams_valid_ = false;
    bool defer_coll_ = false;  // compute_all_mttkrp batches the collectives
    double* hpin_ = nullptr;  // pinned host slots for scalar readbacks  // grams_ == gram(A_n) for every n (skips recomputation; same values)
    int contractions_ = 0;
    DevBuf<double> grams_, pair_, gam_, pinv_, chol_, chol_tmp_, anew_, gram_ws_;
    std::int64_t smax_ = 1;
    DevBuf<double> scal_, partials_, slots_;
    double xnorm_dev_ = -1.0;  // the ||X||^2 value the device slot holds (-1: unknown), so an unchanged value is not re-uploaded
    DevBuf<int> status_, cgres_, flag_;
    DevBuf<int> apply_bad_;            // gn_apply: per-block finiteness
    DevBuf<unsigned int> apply_cnt_;   // gn_apply: last-block counter (self-resetting)
    DevBuf<unsigned int> barrier_;
    DevBuf<std::int64_t> offs_dev_, rows_dev_;
    DevBuf<const double*> facptr_dev_;
    double* Mall_gather_ = nullptr;
    bool precond_pending_ = false;
    double precond_lambda_ = 0.0;
    RegShape precond_shape_ = RegShape::identity;
    std::vector<std::int64_t> local_rows_;           // rows of each mode in the LOCAL tensor
    bool m_all_valid_ = false;                       // all M computed for current factors (GN reuse)

    KrpDesc krp(int lo, int hi, const double* base, bool local_last) const;
    void root_back();
    void root_front();
    void second_level_back(int mode, cudaStream_t st = nullptr, double* ws = nullptr, std::size_t ws_elems = 0);
    DevBuf<double> ws_red_;  // reduce workspace of the reduces run beside a root (aux2)
    void second_level_front(int mode);
    void root_single(int c);          // P_c into PM_ (c in {0, 1})
    void second_level_pm(int mode);   // M^(mode) from PM_
    void mttkrp_msdt(int mode);       // ALS: M^(mode) from whichever cached root serves it
    void finish_mode(int mode);  // collectives on M^(mode)
    void compute_all_mttkrp();

public:
    // every M^(n) for the current factors (one tree pass), as gn_step's first call does
    void prepare_gn() {
        if (!m_all_valid_) compute_all_mttkrp();
    }

private:
    void grams_all();
    void check_status(int count, const char* what);
    double read_scalar(int idx);
};

std::pair<KruskalModel, ConvergenceReport> als_optimize(DeviceProblem& p, KruskalModel model,
                                                        const AlsConfig& cfg);
std::pair<KruskalModel, ConvergenceReport> gn_optimize(DeviceProblem& p, KruskalModel model,
                                                       const GnConfig& cfg);

// Generators (generators.cpp:32-117), host side.
KruskalModel random_model_uniform(const std::vector<std::uint64_t>& dims, std::int64_t rank,
                                  std::uint64_t seed, double a, double b);
KruskalModel random_model_gaussian(const std::vector<std::uint64_t>& dims, std::int64_t rank,
                                   std::uint64_t seed);
std::uint64_t problem_seed(std::uint64_t master, int rank, int problem);
std::uint64_t init_seed(std::uint64_t master, int rank, int problem, int init);
double rng_uniform(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, double a, double b);
std::uint64_t rng_mix64(std::uint64_t x);                       // rng.hpp:11-18
std::uint64_t rng_derive(std::uint64_t h, std::uint64_t v);      // rng.hpp:20-23
std::uint64_t rng_keyed(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, std::uint64_t salt);
double rng_gaussian(std::uint64_t seed, std::uint64_t stream, std::uint64_t index);

}  // namespace cpkit
