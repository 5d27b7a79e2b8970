// Host drivers of the GN-CG / ALS hot path over device-resident state.
//
// Mirrors the reference's C++ solver API and semantics:
//   mttkrp + MttkrpWorkspace     mttkrp.cpp:136-189
//   build_gamma_set / residual   kruskal.cpp:42-65, :94-118
//   gradient / cp_cg / gn_step / gn_optimize   gauss_newton.cpp:81-494
//   als_sweep / als_optimize     als.cpp:22-94
// The host only sees per-iteration scalars (one stream sync per ALS sweep /
// GN outer iteration, plus one inside cp_cg); every vector lives in HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <atomic>
#include <thread>

#include "solver.h"

namespace cpkit {

// ================================================================ host types
double Matrix::norm() const {
    double s = 0.0;
    for (double v : data) s += v * v;
    return std::sqrt(s);
}
bool Matrix::all_finite() const {
    for (double v : data)
        if (!std::isfinite(v)) return false;
    return true;
}

std::uint64_t product_of_dims(const std::vector<std::uint64_t>& dims) {  // tensor.cpp:26-37
    std::uint64_t n = 1;
    for (std::uint64_t d : dims) {
        if (d == 0) throw InvalidArgument("tensor extents must be positive");
        if (n > std::numeric_limits<std::uint64_t>::max() / d)
            throw LimitExceeded("tensor element count overflows 64 bits");
        n *= d;
    }
    return n;
}

// ---- host tensor storage
HostArray::HostArray(std::size_t n) : n_(n) {
    if (n == 0) return;
    void* p = nullptr;
    if (cudaHostAlloc(&p, n * sizeof(double), cudaHostAllocPortable) == cudaSuccess) {
        pinned_ = true;
    } else {
        cudaGetLastError();  // no device / pinning refused: ordinary heap memory
        p = std::malloc(n * sizeof(double));
        if (!p) throw std::bad_alloc();
    }
    p_ = static_cast<double*>(p);
}
HostArray::~HostArray() {
    if (!p_) return;
    if (pinned_) cudaFreeHost(p_);
    else std::free(p_);
}
HostArray& HostArray::operator=(HostArray&& o) noexcept {
    if (this != &o) {
        this->~HostArray();
        p_ = o.p_;
        n_ = o.n_;
        pinned_ = o.pinned_;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}

namespace {
// fn(lo, hi) over [0, n) on up to hardware_concurrency threads (large host passes only)
template <typename F>
void host_parallel(std::uint64_t n, F&& fn) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::uint64_t t = n < (1ull << 24) ? 1 : std::min<std::uint64_t>(hw, 16);
    if (t <= 1) {
        fn(std::uint64_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    const std::uint64_t chunk = (n + t - 1) / t;
    for (std::uint64_t i = 0; i < t; ++i) {
        const std::uint64_t lo = i * chunk, hi = std::min(n, lo + chunk);
        if (lo < hi) pool.emplace_back([&, lo, hi] { fn(lo, hi); });
    }
    for (auto& th : pool) th.join();
}
}  // namespace

DenseTensor::DenseTensor(std::vector<std::uint64_t> dims) : dims_(std::move(dims)) {
    if (dims_.empty()) throw InvalidArgument("tensor order must be at least 1");
    data_ = HostArray(product_of_dims(dims_));
    double* d = data_.data();
    host_parallel(data_.size(), [&](std::uint64_t lo, std::uint64_t hi) { std::fill(d + lo, d + hi, 0.0); });
}
DenseTensor DenseTensor::from_data(std::vector<std::uint64_t> dims, std::vector<double> data) {
    if (dims.empty()) throw InvalidArgument("tensor order must be at least 1");
    if (product_of_dims(dims) != data.size()) throw InvalidArgument("tensor data length does not match extents");
    return copy_of(std::move(dims), data.data());
}
DenseTensor DenseTensor::copy_of(std::vector<std::uint64_t> dims, const double* src) {
    if (dims.empty()) throw InvalidArgument("tensor order must be at least 1");
    HostArray a(product_of_dims(dims));
    double* d = a.data();
    host_parallel(a.size(), [&](std::uint64_t lo, std::uint64_t hi) {
        std::memcpy(d + lo, src + lo, (hi - lo) * sizeof(double));
    });
    return adopt(std::move(dims), std::move(a));
}
DenseTensor DenseTensor::adopt(std::vector<std::uint64_t> dims, HostArray data) {
    DenseTensor t;
    t.dims_ = std::move(dims);
    t.data_ = std::move(data);
    if (t.dims_.empty()) throw InvalidArgument("tensor order must be at least 1");
    if (product_of_dims(t.dims_) != t.data_.size()) throw InvalidArgument("tensor data length does not match extents");
    return t;
}
void DenseTensor::validate() const {  // tensor.cpp:71-83
    if (dims_.empty()) throw InvalidArgument("tensor order must be at least 1");
    if (product_of_dims(dims_) != data_.size()) throw InvalidArgument("tensor data length does not match extents");
    std::atomic<bool> bad{false};
    const double* d = data_.data();
    host_parallel(data_.size(), [&](std::uint64_t lo, std::uint64_t hi) {
        for (std::uint64_t i = lo; i < hi; ++i)
            if (!std::isfinite(d[i])) {
                bad = true;
                return;
            }
    });
    if (bad) throw InvalidArgument("tensor contains non-finite entries");
}

void KruskalModel::validate() const {  // kruskal.cpp:27-40
    if (dims.empty() || rank < 1) throw InvalidArgument("model needs order >= 1 and rank >= 1");
    if (factors.size() != dims.size()) throw InvalidArgument("model factor count does not match order");
    for (std::size_t n = 0; n < dims.size(); ++n) {
        if (static_cast<std::uint64_t>(factors[n].rows) != dims[n] || factors[n].cols != rank)
            throw InvalidArgument("model factor shape mismatch");
        if (!factors[n].all_finite()) throw InvalidArgument("model factor contains non-finite entries");
    }
}

namespace {
void put_u64(std::ostream& os, std::uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    os.write(reinterpret_cast<const char*>(b), 8);
}
std::uint64_t get_u64(std::istream& is) {
    unsigned char b[8] = {};
    is.read(reinterpret_cast<char*>(b), 8);
    std::uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
    return v;
}
void put_f64s(std::ostream& os, const double* d, std::size_t n) {
    // little-endian host: bytes of each double in order (tensor.cpp:249-253)
    os.write(reinterpret_cast<const char*>(d), static_cast<std::streamsize>(n * 8));
}
void get_f64s(std::istream& is, double* d, std::size_t n) {
    is.read(reinterpret_cast<char*>(d), static_cast<std::streamsize>(n * 8));
}
}  // namespace

void write_tensor(const DenseTensor& t, const std::string& path) {  // tensor.cpp:264-276
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open for writing: " + path);
    os.write("CPKT1", 5);
    put_u64(os, t.order());
    for (auto d : t.dims()) put_u64(os, d);
    put_f64s(os, t.data(), t.size());
    if (!os) throw IoError("write failed: " + path);
}
std::vector<std::uint64_t> read_tensor_header(const std::string& path, std::uint64_t* data_offset) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw IoError("cannot open for reading: " + path);
    char magic[5];
    is.read(magic, 5);
    if (!is || std::memcmp(magic, "CPKT1", 5) != 0) throw ParseError("bad tensor magic: " + path);
    const std::uint64_t order = get_u64(is);
    if (!is || order == 0 || order > 64) throw ParseError("bad tensor order: " + path);
    std::vector<std::uint64_t> dims(order);
    for (auto& d : dims) d = get_u64(is);
    if (!is) throw ParseError("truncated tensor header: " + path);
    product_of_dims(dims);  // extents > 0, no overflow
    if (data_offset) *data_offset = 5 + 8 * (1 + order);
    return dims;
}
DenseTensor read_tensor(const std::string& path) {  // tensor.cpp:278-306
    std::uint64_t off = 0;
    std::vector<std::uint64_t> dims = read_tensor_header(path, &off);
    std::ifstream is(path, std::ios::binary);
    is.seekg(static_cast<std::streamoff>(off));
    HostArray data(product_of_dims(dims));  // read straight into (pinned) tensor storage
    get_f64s(is, data.data(), data.size());
    if (!is) throw ParseError("truncated tensor data: " + path);
    DenseTensor t = DenseTensor::adopt(std::move(dims), std::move(data));
    t.validate();
    return t;
}
void write_model(const KruskalModel& m, const std::string& path) {  // kruskal.cpp:143-161
    m.validate();
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open for writing: " + path);
    os.write("CPKM1", 5);
    put_u64(os, m.order());
    put_u64(os, static_cast<std::uint64_t>(m.rank));
    for (auto d : m.dims) put_u64(os, d);
    for (const auto& a : m.factors) put_f64s(os, a.data.data(), a.data.size());
    if (!os) throw IoError("write failed: " + path);
}
KruskalModel read_model(const std::string& path) {  // kruskal.cpp:163-203
    std::ifstream is(path, std::ios::binary);
    if (!is) throw IoError("cannot open for reading: " + path);
    char magic[5];
    is.read(magic, 5);
    if (!is || std::memcmp(magic, "CPKM1", 5) != 0) throw ParseError("bad model magic: " + path);
    const std::uint64_t order = get_u64(is);
    const std::uint64_t rank = get_u64(is);
    if (!is || order == 0 || order > 64 || rank == 0) throw ParseError("bad model header: " + path);
    KruskalModel m;
    m.rank = static_cast<std::int64_t>(rank);
    m.dims.resize(order);
    for (auto& d : m.dims) d = get_u64(is);
    if (!is) throw ParseError("truncated model header: " + path);
    for (auto d : m.dims) {
        Matrix a(static_cast<std::int64_t>(d), m.rank);
        get_f64s(is, a.data.data(), a.data.size());
        m.factors.push_back(std::move(a));
    }
    if (!is) throw ParseError("truncated model data: " + path);
    m.validate();
    return m;
}

// ================================================================ configs
RegSchedule RegSchedule::constant(double lambda, RegShape shape) {
    RegSchedule s;
    s.mode = RegMode::constant;
    s.shape = shape;
    s.lambda = lambda;
    s.validate();
    return s;
}
RegSchedule RegSchedule::varying(double upper, double lower, double mu, RegShape shape) {
    RegSchedule s;
    s.mode = RegMode::varying;
    s.shape = shape;
    s.lambda = upper;
    s.mu = mu;
    s.lower = lower;
    s.upper = upper;
    s.direction = Direction::down;
    s.validate();
    return s;
}
void RegSchedule::validate() const {  // gauss_newton.cpp:33-45
    if (lambda < 0) throw InvalidArgument("schedule: lambda must be nonnegative");
    if (mode == RegMode::varying) {
        if (!(mu > 1.0)) throw InvalidArgument("schedule: mu must exceed 1");
        if (!(lower > 0.0) || !(lower < upper)) throw InvalidArgument("schedule: need 0 < lower < upper");
    }
}
RegSchedule schedule_next(RegSchedule s) {  // gauss_newton.cpp:47-59
    if (s.mode == RegMode::constant) return s;
    if (s.direction == RegSchedule::Direction::down) {
        s.lambda /= s.mu;
        if (s.lambda < s.lower) s.direction = RegSchedule::Direction::up;
    } else {
        s.lambda *= s.mu;
        if (s.lambda > s.upper) s.direction = RegSchedule::Direction::down;
    }
    return s;
}
void GnConfig::validate() const {  // gauss_newton.cpp:61-79
    schedule.validate();
    if (grad_tol < 0 || residual_tol < 0 || step_tol < 0) throw InvalidArgument("gn config: negative tolerance");
    if (max_iters < 0 || cg_max_iters < 0) throw InvalidArgument("gn config: negative iteration cap");
    if (!(cg_tol > 0)) throw InvalidArgument("gn config: cg_tol must be positive");
    if (armijo) {
        if (!(armijo->c1 > 0 && armijo->c1 < 1) || !(armijo->shrink > 0 && armijo->shrink < 1) ||
            armijo->max_backtracks < 1)
            throw InvalidArgument("gn config: bad armijo parameters");
    }
}
void AlsConfig::validate() const {  // als.cpp:10-20
    if (max_sweeps < 0 || residual_tol < 0 || step_tol < 0 || lambda0 < 0)
        throw InvalidArgument("als config: negative tolerance, cap or lambda");
    if (decay_factor < 1.0) throw InvalidArgument("als config: decay_factor must be >= 1");
    if (decay_every && *decay_every < 1) throw InvalidArgument("als config: decay_every must be positive");
}

const char* to_string(TerminalStatus s) {
    switch (s) {
        case TerminalStatus::converged_residual: return "converged_residual";
        case TerminalStatus::converged_step: return "converged_step";
        case TerminalStatus::cap_hit: return "cap_hit";
        case TerminalStatus::numerical_failure: return "numerical_failure";
    }
    return "unknown";
}
double ConvergenceReport::best_residual() const {
    double best = 1.0;
    for (const auto& r : records) best = std::min(best, r.residual);
    return best;
}

// ================================================================ rng (rng.hpp:11-46)
namespace {
inline std::uint64_t mix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
inline std::uint64_t derive(std::uint64_t h, std::uint64_t v) {
    return mix64(h ^ (v * 0xD6E8FEB86659FD93ull + 0xA0761D6478BD642Full));
}
inline std::uint64_t keyed(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, std::uint64_t salt) {
    return derive(derive(derive(mix64(seed), stream), index), salt);
}
inline double to_unit(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }
}  // namespace

double rng_uniform(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, double a, double b) {
    return a + (b - a) * to_unit(keyed(seed, stream, index, 0));
}
double rng_gaussian(std::uint64_t seed, std::uint64_t stream, std::uint64_t index) {
    const double u1 = static_cast<double>((keyed(seed, stream, index, 1) >> 11) + 1) * 0x1.0p-53;
    const double u2 = to_unit(keyed(seed, stream, index, 2));
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}
std::uint64_t problem_seed(std::uint64_t master, int rank, int problem) {  // harness.cpp:378-383
    return derive(derive(derive(mix64(master), 0x50524F42ull), static_cast<std::uint64_t>(rank)),
                  static_cast<std::uint64_t>(problem));
}
std::uint64_t init_seed(std::uint64_t master, int rank, int problem, int init) {  // :385-391
    return derive(derive(derive(derive(mix64(master), 0x494E4954ull), static_cast<std::uint64_t>(rank)),
                         static_cast<std::uint64_t>(problem)),
                  static_cast<std::uint64_t>(init));
}
namespace {
template <typename Draw>
KruskalModel fill_model(const std::vector<std::uint64_t>& dims, std::int64_t rank, Draw&& draw) {
    if (rank < 1) throw InvalidArgument("random_model: rank must be positive");
    KruskalModel m;
    m.dims = dims;
    m.rank = rank;
    for (std::size_t n = 0; n < dims.size(); ++n) {
        Matrix a(static_cast<std::int64_t>(dims[n]), rank);
        for (std::int64_t i = 0; i < a.rows; ++i)
            for (std::int64_t r = 0; r < rank; ++r)
                a.data[static_cast<std::size_t>(i * rank + r)] =
                    draw(n, static_cast<std::uint64_t>(i) * static_cast<std::uint64_t>(rank) + static_cast<std::uint64_t>(r));
        m.factors.push_back(std::move(a));
    }
    m.validate();
    return m;
}
}  // namespace
std::uint64_t rng_mix64(std::uint64_t x) { return mix64(x); }
std::uint64_t rng_derive(std::uint64_t h, std::uint64_t v) { return derive(h, v); }
std::uint64_t rng_keyed(std::uint64_t seed, std::uint64_t stream, std::uint64_t index, std::uint64_t salt) {
    return keyed(seed, stream, index, salt);
}
KruskalModel random_model_uniform(const std::vector<std::uint64_t>& dims, std::int64_t rank,
                                  std::uint64_t seed, double a, double b) {  // generators.cpp:59-68
    if (!(a < b)) throw InvalidArgument("random_model: uniform needs a < b");
    return fill_model(dims, rank, [&](std::uint64_t n, std::uint64_t idx) { return rng_uniform(seed, n, idx, a, b); });
}
KruskalModel random_model_gaussian(const std::vector<std::uint64_t>& dims, std::int64_t rank,
                                   std::uint64_t seed) {  // generators.cpp:70-76
    return fill_model(dims, rank, [&](std::uint64_t n, std::uint64_t idx) { return rng_gaussian(seed, n, idx); });
}

// ================================================================ context
Context::Context(int dev) : device(dev) {
    CPK_CUDA(cudaSetDevice(dev));
    CPK_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    // the side stream carries the latency-bound SPD factorisations (one CTA
    // each): top priority, so their CTA is placed before a concurrent
    // bandwidth kernel fills every SM
    int lo = 0, hi = 0;
    CPK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char* pe = std::getenv("CPKIT_AUX_PRIORITY");
    CPK_CUDA(cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, (pe && std::atoi(pe) == 0) ? lo : hi));
    CPK_CUDA(cudaStreamCreateWithFlags(&aux2, cudaStreamNonBlocking));
    for (auto& e : ev) CPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}
Context::~Context() {
    comm.reset();
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    if (aux2) cudaStreamDestroy(aux2);
    if (aux) cudaStreamDestroy(aux);
    if (stream) cudaStreamDestroy(stream);
}
void Context::sync() const {
    CPK_CUDA(cudaStreamSynchronize(aux2));
    CPK_CUDA(cudaStreamSynchronize(aux));
    CPK_CUDA(cudaStreamSynchronize(stream));
}
void Context::sync_main() const { CPK_CUDA(cudaStreamSynchronize(stream)); }

void shard_range(std::uint64_t extent, int rank, int world, std::uint64_t* lo, std::uint64_t* hi) {
    const std::uint64_t base = extent / static_cast<std::uint64_t>(world);
    const std::uint64_t rem = extent % static_cast<std::uint64_t>(world);
    const std::uint64_t r = static_cast<std::uint64_t>(rank);
    *lo = r * base + std::min(r, rem);
    *hi = *lo + base + (r < rem ? 1 : 0);
}

// ================================================================ DeviceProblem
namespace {
// Layout copies of the tensor (order-3 permuted copies, order >= 4 X^T) are
// made when they take at most this share of the HBM still free after X is
// allocated; the rest covers the root partials and workspaces. C5 per GPU:
// P=1 (C5s) and P>=4 copy, P=2 (102 GB slab) runs the TN front root on X.
constexpr double kLayoutCopyShare = 0.7;
enum Scal { kXnorm = 0, kRes = 1, kFit = 2, kStep = 3, kNormSum = 4, kDot = 5, kNScal = 16 };
}

DeviceProblem::DeviceProblem(Context& ctx, std::vector<std::uint64_t> dims, int rank)
    : ctx_(ctx), dims_(std::move(dims)), R_(rank) {
    const int N = order();
    if (N < 2) throw InvalidArgument("mttkrp: tensor order must be at least 2");
    if (N > kMaxOrder) throw LimitExceeded("tensor order exceeds 16");
    if (R_ < 1) throw InvalidArgument("model needs order >= 1 and rank >= 1");
    hpin_ = static_cast<double*>(pinned_small_alloc(kPinBytes, false));
    hmap_ = static_cast<double*>(pinned_small_alloc(kMapBytes, true));
    std::memset(hpin_, 0, kPinBytes);  // recycled blocks: no stale diagnostics
    std::memset(hmap_, 0, kMapBytes);
    for (auto& e : gn_ev_) CPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CPK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dmap_), hmap_, 0));
    als_graphs_.reserve(kAlsGraphs);  // in-flight sweeps hold pointers to their graphs
    for (auto& e : slot_ev_) CPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CPK_CUDA(cudaSetDevice(ctx_.device));
    h_ = (N + 1) / 2;
    shard_range(dims_[N - 1], ctx_.rank(), ctx_.world(), &slab_lo_, &slab_hi_);
    if (ctx_.world() > 1 && dims_[N - 1] % static_cast<std::uint64_t>(ctx_.world()) != 0)
        throw LimitExceeded("sharded runs need the last extent divisible by the GPU count");
    local_rows_.resize(N);
    for (int n = 0; n < N; ++n) local_rows_[n] = static_cast<std::int64_t>(dims_[n]);
    local_rows_[N - 1] = static_cast<std::int64_t>(slab_hi_ - slab_lo_);
    F_ = 1;
    Bl_ = 1;
    for (int n = 0; n < h_; ++n) F_ *= local_rows_[n];
    for (int n = h_; n < N; ++n) Bl_ *= local_rows_[n];
    local_elems_ = static_cast<std::uint64_t>(F_) * static_cast<std::uint64_t>(Bl_);
    Bs_ = (Bl_ % 2 == 0) ? Bl_ : Bl_ + 1;  // TMA needs 16-byte row strides: pad odd rows once

    off_.assign(N + 1, 0);
    for (int n = 0; n < N; ++n) off_[n + 1] = off_[n] + static_cast<std::int64_t>(dims_[n]) * R_;
    const std::size_t S = static_cast<std::size_t>(off_[N]);
    const std::size_t RR = static_cast<std::size_t>(R_) * R_;

    x_.resize(static_cast<std::size_t>(F_) * static_cast<std::size_t>(Bs_));
    if (Bs_ != Bl_) CPK_CUDA(cudaMemset(x_.get(), 0, x_.size() * sizeof(double)));
    krp_.resize(krp_workspace_elems(std::max<std::int64_t>(std::max(F_, Bl_), N == 3 ? std::max(local_rows_[0], local_rows_[1]) : 0), R_));
    A_.resize(S); Atrial_.resize(S); Asnap1_.resize(S); M_.resize(S); G_.resize(S); V_.resize(S); Z_.resize(S); Q_.resize(S);
    for (int i = 0; i < 2; ++i) { Rr_[i].resize(S); W_[i].resize(S); }
    PF_.resize(static_cast<std::size_t>(F_) * R_);
    PB_.resize(static_cast<std::size_t>(Bl_) * R_);
    if (N == 3 && !std::getenv("CPKIT_ALS_TREE")) {
        // the permuted copies need 2 more tensors (X itself is already allocated)
        std::size_t free_b = 0, total_b = 0;
        CPK_CUDA(cudaMemGetInfo(&free_b, &total_b));
        ld0_ = (local_rows_[0] + 1) & ~1LL;
        ld1_ = (local_rows_[1] + 1) & ~1LL;
        const double copy_b = 8.0 * static_cast<double>(Bl_) *
                              static_cast<double>(local_rows_[1] * ld0_ + local_rows_[0] * ld1_);
        const char* ce = std::getenv("CPKIT_MSDT_COPIES");
        msdt_copies_ = ce ? std::atoi(ce) != 0 : copy_b < kLayoutCopyShare * static_cast<double>(free_b);
        // without copies the single-mode roots are TN GEMMs with the factor as the B operand
        msdt_ = msdt_copies_ || (R_ % 2 == 0 && Bs_ == Bl_);
    }
    if (N >= 4) {
        std::size_t free_b = 0, total_b = 0;
        CPK_CUDA(cudaMemGetInfo(&free_b, &total_b));
        free_b += dev_cache_bytes();  // recycled blocks are free for this problem
        ldT_ = (F_ + 1) & ~1LL;
        const double copy_b = 8.0 * static_cast<double>(Bl_) * static_cast<double>(ldT_);
        const char* ce = std::getenv("CPKIT_FRONT_COPY");
        front_copy_ = ce ? std::atoi(ce) != 0 : copy_b < kLayoutCopyShare * static_cast<double>(free_b);
        if (front_copy_) {
            XT_.resize(static_cast<std::size_t>(Bl_ * ldT_));
            if (ldT_ != F_)  // the stride padding column stays zero
                CPK_CUDA(cudaMemset2D(XT_.get() + F_, ldT_ * sizeof(double), 0, sizeof(double), Bl_));
        }
    }
    if (msdt_)
        PM_.resize(static_cast<std::size_t>(std::max(local_rows_[0], local_rows_[1])) * Bl_ * R_);
    if (msdt_copies_) {
        X0_.resize(static_cast<std::size_t>(local_rows_[1] * Bl_ * ld0_));
        X1_.resize(static_cast<std::size_t>(local_rows_[0] * Bl_ * ld1_));
        CPK_CUDA(cudaMemset(X0_.get(), 0, X0_.size() * sizeof(double)));  // stride padding stays zero
        CPK_CUDA(cudaMemset(X1_.get(), 0, X1_.size() * sizeof(double)));
    }
    // split-K and second-level workspaces
    std::size_t ws = std::max(root_front_workspace_elems(F_, Bl_, R_), root_back_workspace_elems(F_, Bl_, R_));
    {
        KrpDesc kf = krp(0, h_, A_.get(), false), kb = krp(h_, N, A_.get(), true);
        for (int n = 0; n < h_; ++n) ws = std::max(ws, reduce_kept_workspace_elems(kf, n, R_));
        for (int n = h_; n < N; ++n) ws = std::max(ws, reduce_kept_workspace_elems(kb, n - h_, R_));
        if (front_copy_) ws = std::max(ws, root_back_workspace_elems(Bl_, F_, R_));
        if (msdt_copies_) {
            ws = std::max(ws, root_back_workspace_elems(local_rows_[1] * Bl_, local_rows_[0], R_));
            ws = std::max(ws, root_back_workspace_elems(local_rows_[0] * Bl_, local_rows_[1], R_));
        }
        if (msdt_) {
            if (!msdt_copies_) ws = std::max(ws, root_single_workspace_elems(local_rows_[0], local_rows_[1], Bs_, R_));
            for (int c = 0; c < 2; ++c) {
                KrpDesc kd{};
                kd.nmodes = 2;
                int j = 0;
                for (int m = 0; m < N; ++m)
                    if (m != c) kd.ext[j++] = local_rows_[m];
                for (int keep = 0; keep < 2; ++keep) ws = std::max(ws, reduce_kept_workspace_elems(kd, keep, R_));
            }
        }
    }
    ws_.resize(std::max<std::size_t>(ws, 1));
    {
        KrpDesc kf = krp(0, h_, A_.get(), false);
        std::size_t wr = 1;
        for (int n = 0; n < h_; ++n) wr = std::max(wr, reduce_kept_workspace_elems(kf, n, R_));
        ws_red_.resize(wr);
    }
    grams_.resize(N * RR);
    pair_.resize(static_cast<std::size_t>(N) * N * RR);
    gam_.resize(N * RR);
    pinv_.resize(N * RR);
    chol_.resize(chol_factor_elems(N, R_));
    chol_tmp_.resize(N * RR);
    std::int64_t smax = 1;
    for (auto d : dims_) smax = std::max<std::int64_t>(smax, static_cast<std::int64_t>(d));
    anew_.resize(static_cast<std::size_t>(smax) * R_);
    smax_ = smax;
    gram_ws_.resize(gram_workspace_elems(N, R_, smax));
    scal_.resize(kNScal);
    partials_.resize(std::max<std::size_t>(std::max(4096, 2 * norm2_parts(static_cast<std::uint64_t>(F_) * Bs_) + 8),
                                           static_cast<std::size_t>(smax)));  // >= one slot per factor row
    status_.resize(std::max(N, 1));
    apply_bad_.resize(static_cast<std::size_t>(N) * 16);
    apply_cnt_.resize(1);
    CPK_CUDA(cudaMemset(apply_cnt_.get(), 0, sizeof(unsigned int)));
    cgres_.resize(8);
    flag_.resize(4);
    barrier_.resize(cg_barrier_words());
    offs_dev_.resize(N + 1);
    rows_dev_.resize(N);
    std::vector<std::int64_t> rows(dims_.begin(), dims_.end());
    CPK_CUDA(cudaMemcpy(offs_dev_.get(), off_.data(), (N + 1) * sizeof(std::int64_t), cudaMemcpyHostToDevice));
    CPK_CUDA(cudaMemcpy(rows_dev_.get(), rows.data(), N * sizeof(std::int64_t), cudaMemcpyHostToDevice));
    CPK_CUDA(cudaMemset(scal_.get(), 0, kNScal * sizeof(double)));
    // CG slots
    CgParams cp{};
    cp.order = N;
    cp.R = R_;
    for (int n = 0; n < N; ++n) cp.rows[n] = static_cast<std::int64_t>(dims_[n]);
    slots_.resize(cg_slots_needed(cp));
}

DeviceProblem::~DeviceProblem() {
    // every stream idle (no throw from a destructor): the buffers can be reused
    const bool idle = cudaStreamSynchronize(ctx_.aux2) == cudaSuccess &&
                      cudaStreamSynchronize(ctx_.aux) == cudaSuccess &&
                      cudaStreamSynchronize(ctx_.stream) == cudaSuccess;
    if (idle) release_scope_.emplace();
    static const bool trace = std::getenv("CPKIT_PHASE_TRACE") != nullptr;  // timing experiments
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!trace) return;
        const auto t1 = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (ms > 1.0) std::fprintf(stderr, "  ~DeviceProblem %s %.1f ms\n", what, ms);
        t0 = t1;
    };
    pending_.clear();
    done_.clear();
    drop_als_graph();
    lap("graphs");
    profile_enable(false);
    pinned_small_free(hpin_, kPinBytes, false);
    pinned_small_free(hmap_, kMapBytes, true);
    lap("pinned");
    for (auto& e : slot_ev_)
        if (e) cudaEventDestroy(e);
    for (auto& e : gn_ev_)
        if (e) cudaEventDestroy(e);
    lap("events");
}

KrpDesc DeviceProblem::krp(int lo, int hi, const double* base, bool local_last) const {
    KrpDesc d{};
    d.nmodes = hi - lo;
    const int N = order();
    for (int m = lo; m < hi; ++m) {
        const bool last = (m == N - 1);
        d.ext[m - lo] = (last && local_last) ? local_rows_[m] : static_cast<std::int64_t>(dims_[m]);
        d.fac[m - lo] = base + off_[m] + ((last && local_last) ? static_cast<std::int64_t>(slab_lo_) * R_ : 0);
    }
    return d;
}

void DeviceProblem::upload_tensor(const double* host_local, const KruskalModel* start) {
    NvtxRange nvtx_range("cpkit:upload_tensor");
    const int N = order();
    if (start && front_copy_ && !ctx_.comm && h_ >= 1 && !std::getenv("CPKIT_UPLOAD_UNCHUNKED") &&
        !std::getenv("CPKIT_UPLOAD_NO_ROOT")) {
        // orders >= 4: H2D by row slabs on the side stream; per slab, the back
        // root's rows on the solver stream and the slab's X^T columns on the
        // third stream, both beside the next slab's copy
        set_factors(*start);
        const std::int64_t chunks = std::max<std::int64_t>(1, std::min<std::int64_t>(8, F_ / 10000));
        const std::int64_t step = (F_ + chunks - 1) / chunks;
        for (std::int64_t a = 0; a < F_; a += step) {
            const std::int64_t rows = std::min(F_, a + step) - a;
            double* xd = x_.get() + a * Bs_;
            if (Bs_ == Bl_)
                CPK_CUDA(cudaMemcpyAsync(xd, host_local + a * Bl_, rows * Bl_ * sizeof(double), cudaMemcpyHostToDevice,
                                         ctx_.aux));
            else
                CPK_CUDA(cudaMemcpy2DAsync(xd, Bs_ * sizeof(double), host_local + a * Bl_, Bl_ * sizeof(double),
                                           Bl_ * sizeof(double), rows, cudaMemcpyHostToDevice, ctx_.aux));
            CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2A], ctx_.aux));
            CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[Context::kEvAux2A], 0));
            CPK_CUDA(cudaStreamWaitEvent(ctx_.aux2, ctx_.ev[Context::kEvAux2A], 0));
            launch_transpose_batched(xd, 1, rows, Bl_, Bs_, 0, XT_.get() + a, ldT_, 0, ctx_.aux2);
            launch_root_back(xd, rows, Bl_, Bs_, R_, krp(h_, N, A_.get(), true), krp_.get(), PF_.get() + a * R_,
                             ws_.get(), ws_.size(), ctx_.stream, 0);
        }
        CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2B], ctx_.aux2));
        CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[Context::kEvAux2B], 0));
        invalidate_all();
        pf_valid_ = true;  // the back root of the start factors
        ++contractions_;
        preset_.clear();
        for (const auto& f : start->factors) preset_.insert(preset_.end(), f.data.begin(), f.data.end());
        preset_valid_ = true;
        return;
    }
    if (msdt_copies_ && !std::getenv("CPKIT_UPLOAD_UNCHUNKED")) {
        // order 3: upload by i0 slabs; each slab's share of both permuted copies is
        // transposed on the third stream while the next slab crosses PCIe
        const std::int64_t s0 = local_rows_[0], s1 = local_rows_[1];
        const std::int64_t chunks = std::min<std::int64_t>(8, s0), step = (s0 + chunks - 1) / chunks;
        for (std::int64_t a = 0; a < s0; a += step) {
            const std::int64_t b = std::min(s0, a + step), rows = (b - a) * s1;
            double* xd = x_.get() + a * s1 * Bs_;
            const double* xh = host_local + a * s1 * Bl_;
            if (Bs_ == Bl_)
                CPK_CUDA(cudaMemcpyAsync(xd, xh, rows * Bl_ * sizeof(double), cudaMemcpyHostToDevice, ctx_.stream));
            else
                CPK_CUDA(cudaMemcpy2DAsync(xd, Bs_ * sizeof(double), xh, Bl_ * sizeof(double), Bl_ * sizeof(double),
                                           rows, cudaMemcpyHostToDevice, ctx_.stream));
            CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2A], ctx_.stream));
            CPK_CUDA(cudaStreamWaitEvent(ctx_.aux2, ctx_.ev[Context::kEvAux2A], 0));
            // X^(0)[i1][i2][i0], columns i0 in [a, b): batch i1, rows i0, cols i2
            launch_transpose_batched(xd, s1, b - a, Bl_, s1 * Bs_, Bs_, X0_.get() + a, ld0_, Bl_ * ld0_, ctx_.aux2);
            // X^(1)[i0][i2][i1] for i0 in [a, b): batch i0, rows i1, cols i2
            launch_transpose_batched(xd, b - a, s1, Bl_, Bs_, s1 * Bs_, X1_.get() + a * Bl_ * ld1_, ld1_,
                                     Bl_ * ld1_, ctx_.aux2);
        }
        CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2B], ctx_.aux2));
        CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[Context::kEvAux2B], 0));
        invalidate_all();
        return;
    }
    if (front_copy_ && !std::getenv("CPKIT_UPLOAD_UNCHUNKED")) {
        // orders >= 4: upload by row slabs; each slab's columns of X^T are
        // transposed on the third stream while the next slab crosses PCIe
        const std::int64_t chunks = std::min<std::int64_t>(8, F_), step = (F_ + chunks - 1) / chunks;
        for (std::int64_t a = 0; a < F_; a += step) {
            const std::int64_t rows = std::min(F_, a + step) - a;
            double* xd = x_.get() + a * Bs_;
            if (Bs_ == Bl_)
                CPK_CUDA(cudaMemcpyAsync(xd, host_local + a * Bl_, rows * Bl_ * sizeof(double), cudaMemcpyHostToDevice,
                                         ctx_.stream));
            else
                CPK_CUDA(cudaMemcpy2DAsync(xd, Bs_ * sizeof(double), host_local + a * Bl_, Bl_ * sizeof(double),
                                           Bl_ * sizeof(double), rows, cudaMemcpyHostToDevice, ctx_.stream));
            CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2A], ctx_.stream));
            CPK_CUDA(cudaStreamWaitEvent(ctx_.aux2, ctx_.ev[Context::kEvAux2A], 0));
            launch_transpose_batched(xd, 1, rows, Bl_, Bs_, 0, XT_.get() + a, ldT_, 0, ctx_.aux2);
        }
        CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2B], ctx_.aux2));
        CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[Context::kEvAux2B], 0));
        invalidate_all();
        return;
    }
    if (Bs_ == Bl_)
        CPK_CUDA(cudaMemcpyAsync(x_.get(), host_local, local_elems_ * sizeof(double), cudaMemcpyHostToDevice,
                                 ctx_.stream));
    else
        CPK_CUDA(cudaMemcpy2DAsync(x_.get(), Bs_ * sizeof(double), host_local, Bl_ * sizeof(double),
                                   Bl_ * sizeof(double), F_, cudaMemcpyHostToDevice, ctx_.stream));
    build_msdt_copies();
    invalidate_all();
}
void DeviceProblem::load_tensor_file(const std::string& path) {
    NvtxRange nvtx_range("cpkit:load_tensor_file");
    std::uint64_t off = 0;
    if (read_tensor_header(path, &off) != dims_) throw InvalidArgument("tensor file extents do not match the problem");
    const int N = order();
    const std::uint64_t sl = dims_[N - 1], slab = slab_hi_ - slab_lo_, rows = local_elems_ / slab;
    std::ifstream is(path, std::ios::binary);
    is.seekg(static_cast<std::streamoff>(off));
    auto read_rows = [&](double* dst, std::uint64_t nr) {
        get_f64s(is, dst, nr * sl);
        if (!is) throw ParseError("truncated tensor data: " + path);
    };
    if (Bs_ != Bl_) {  // padded row stride (odd back extent): gather the slab, then the ordinary upload
        HostArray h(local_elems_), row(sl);
        for (std::uint64_t r = 0; r < rows; ++r) {
            read_rows(row.data(), 1);
            std::memcpy(h.data() + r * slab, row.data() + slab_lo_, slab * sizeof(double));
        }
        upload_tensor(h.data());
    } else {
        // whole last-mode rows per chunk; two pinned staging buffers: chunk k is
        // read while chunk k-1 crosses to HBM (2-D copy of the slab columns if sharded)
        const std::uint64_t per = std::max<std::uint64_t>(1, (64ull << 20) / (sl * sizeof(double)));
        HostArray stage[2] = {HostArray(per * sl), HostArray(per * sl)};
        cudaEvent_t ev[2];
        for (auto& e : ev) CPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        try {
            std::uint64_t k = 0;
            for (std::uint64_t r0 = 0; r0 < rows; r0 += per, ++k) {
                const std::uint64_t nr = std::min(per, rows - r0);
                const int b = static_cast<int>(k & 1);
                if (k >= 2) CPK_CUDA(cudaEventSynchronize(ev[b]));  // its previous copy has landed
                read_rows(stage[b].data(), nr);
                double* dst = x_.get() + r0 * slab;
                if (slab == sl)
                    CPK_CUDA(cudaMemcpyAsync(dst, stage[b].data(), nr * sl * sizeof(double), cudaMemcpyHostToDevice,
                                             ctx_.stream));
                else
                    CPK_CUDA(cudaMemcpy2DAsync(dst, slab * sizeof(double), stage[b].data() + slab_lo_,
                                               sl * sizeof(double), slab * sizeof(double), nr, cudaMemcpyHostToDevice,
                                               ctx_.stream));
                CPK_CUDA(cudaEventRecord(ev[b], ctx_.stream));
            }
            ctx_.sync_main();
        } catch (...) {
            cudaStreamSynchronize(ctx_.stream);
            for (auto& e : ev) cudaEventDestroy(e);
            throw;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        build_msdt_copies();
        invalidate_all();
    }
    // tensor.cpp:71-83 (validate on load), checked on the device
    launch_set_flag_scalar(flag_.get(), 1, scal_.get() + 11, 0.0, ctx_.stream);
    launch_all_finite(x_.get(), static_cast<std::uint64_t>(F_) * static_cast<std::uint64_t>(Bs_), flag_.get(),
                      ctx_.stream);
    int ok = 0;
    CPK_CUDA(cudaMemcpyAsync(&ok, flag_.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync_main();
    if (!ok) throw InvalidArgument("tensor contains non-finite entries");
}
void DeviceProblem::build_msdt_copies() {
    if (front_copy_)  // X^T [B_local][F]
        launch_transpose_batched(x_.get(), 1, F_, Bl_, Bs_, 0, XT_.get(), ldT_, 0, ctx_.stream);
    if (!msdt_copies_) return;
    const std::int64_t s0 = local_rows_[0], s1 = local_rows_[1];
    // X^(0)[i1][i2][i0]: batch i1, rows i0 (stride s1 Bs), cols i2
    launch_transpose_batched(x_.get(), s1, s0, Bl_, s1 * Bs_, Bs_, X0_.get(), ld0_, Bl_ * ld0_, ctx_.stream);
    // X^(1)[i0][i2][i1]: batch i0, rows i1 (stride Bs), cols i2
    launch_transpose_batched(x_.get(), s0, s1, Bl_, Bs_, s1 * Bs_, X1_.get(), ld1_, Bl_ * ld1_, ctx_.stream);
}
void DeviceProblem::download_tensor(double* host_local) {
    if (Bs_ == Bl_)
        CPK_CUDA(cudaMemcpyAsync(host_local, x_.get(), local_elems_ * sizeof(double), cudaMemcpyDeviceToHost,
                                 ctx_.stream));
    else
        CPK_CUDA(cudaMemcpy2DAsync(host_local, Bl_ * sizeof(double), x_.get(), Bs_ * sizeof(double),
                                   Bl_ * sizeof(double), F_, cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
}

// Device-side low-rank (+ noise) generation: the reference's reconstruct
// order per entry (kruskal.cpp:76-90) with non-fused multiply/add, so the
// noiseless tensor is bitwise equal to the CPU generator's; the keyed noise
// (keyed_noise.cuh) is bitwise equal to the CPU restatement's too.
void DeviceProblem::generate_tensor(const KruskalModel& truth, std::uint64_t noise_seed, double noise_rel) {
    NvtxRange nvtx_range("cpkit:generate_tensor");
    set_factors(truth);
    const int N = order();
    KrpDesc all = krp(0, N, A_.get(), true);
    // global flat offset of the local slab is not contiguous when sharded; generate
    // slab-local entries through a local descriptor (last factor already offset).
    DevBuf<double> dense;
    double* xd = x_.get();
    if (Bs_ != Bl_) {
        dense.resize(local_elems_);
        xd = dense.get();
    }
    launch_reconstruct(all, R_, xd, 0, local_elems_, ctx_.stream);
    if (noise_rel > 0.0) {
        // keyed noise E (stream 0x4E01) scaled to noise_rel ||X|| / ||E||, with no
        // tensor-sized buffer: pass 1 sums X^2 and E^2 per last-mode column (E
        // recomputed from its key), the columns are gathered and summed in global
        // order (the same bits for every GPU count), pass 2 adds scale * E
        const std::int64_t slab = local_rows_[N - 1];
        const std::int64_t rows = static_cast<std::int64_t>(local_elems_) / slab;
        const int world = ctx_.world();
        const std::size_t wse = noise_workspace_elems(slab);
        DevBuf<double> nws(wse + 2 * static_cast<std::size_t>(slab) * world);
        double* cs = nws.get() + wse - 2 * slab;  // this rank's [X cols | E cols]
        double* all = nws.get() + wse;
        launch_noise_colsq(xd, rows, slab, noise_seed, dims_[N - 1], slab_lo_, nws.get(), cs, ctx_.stream);
        if (ctx_.comm) ctx_.comm->allgather(cs, all, 2 * static_cast<std::size_t>(slab), ctx_.stream);
        launch_noise_scale(ctx_.comm ? all : cs, world, slab, noise_rel, scal_.get() + 8, ctx_.stream);
        launch_noise_add(xd, local_elems_, static_cast<std::uint64_t>(slab), dims_[N - 1], slab_lo_, noise_seed,
                         scal_.get() + 8, ctx_.stream);
    }
    if (Bs_ != Bl_)
        CPK_CUDA(cudaMemcpy2DAsync(x_.get(), Bs_ * sizeof(double), xd, Bl_ * sizeof(double), Bl_ * sizeof(double),
                                   F_, cudaMemcpyDeviceToDevice, ctx_.stream));
    build_msdt_copies();
    ctx_.sync();
    invalidate_all();
}

void DeviceProblem::set_factors(const std::vector<const double*>& host) {
    preset_valid_ = false;
    for (int n = 0; n < order(); ++n)
        CPK_CUDA(cudaMemcpyAsync(A_.get() + off_[n], host[n], (off_[n + 1] - off_[n]) * sizeof(double),
                                 cudaMemcpyHostToDevice, ctx_.stream));
    invalidate_all();
}
void DeviceProblem::get_factors(std::vector<double*>& host) {
    for (int n = 0; n < order(); ++n)
        CPK_CUDA(cudaMemcpyAsync(host[n], A_.get() + off_[n], (off_[n + 1] - off_[n]) * sizeof(double),
                                 cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
}
void DeviceProblem::set_factors(const KruskalModel& m) {
    if (m.dims != dims_ || m.rank != R_) throw InvalidArgument("model extents/rank do not match the problem");
    if (preset_valid_) {  // the factors the upload contracted: keep them and their back root
        bool same = true;
        std::size_t at = 0;
        for (const auto& a : m.factors) {
            if (at + a.data.size() > preset_.size() ||
                std::memcmp(a.data.data(), preset_.data() + at, a.data.size() * sizeof(double)) != 0) {
                same = false;
                break;
            }
            at += a.data.size();
        }
        preset_valid_ = false;
        if (same && at == preset_.size()) return;
    }
    std::vector<const double*> p;
    for (const auto& a : m.factors) p.push_back(a.data.data());
    set_factors(p);
}
void DeviceProblem::get_factors(KruskalModel& m) {
    m.dims = dims_;
    m.rank = R_;
    m.factors.resize(dims_.size());
    std::vector<double*> p;
    for (std::size_t n = 0; n < dims_.size(); ++n) {
        m.factors[n] = Matrix(static_cast<std::int64_t>(dims_[n]), R_);
        p.push_back(m.factors[n].data.data());
    }
    get_factors(p);
}

// Scalar readback through pinned memory, waiting on the solver stream only, so
// side-stream work (the speculative preconditioner factorisation) keeps running.
double DeviceProblem::read_scalar(int idx) {
    CPK_CUDA(cudaMemcpyAsync(hpin_, scal_.get() + idx, sizeof(double), cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync_main();
    return hpin_[0];
}

double DeviceProblem::norm2() {
    const std::uint64_t stored = static_cast<std::uint64_t>(F_) * static_cast<std::uint64_t>(Bs_);  // pad is zero
    launch_norm2(x_.get(), stored, partials_.get(), norm2_parts(stored), scal_.get() + kXnorm, ctx_.stream);
    if (ctx_.comm) ctx_.comm->allreduce_sum(scal_.get() + kXnorm, 1, ctx_.stream);
    xnorm_dev_ = read_scalar(kXnorm);
    return xnorm_dev_;
}

// ---- launch profiling ----------------------------------------------------------
void DeviceProblem::profile_enable(bool on) {
    for (auto& e : prof_) {
        if (e.a) cudaEventDestroy(e.a);
        if (e.b) cudaEventDestroy(e.b);
    }
    prof_.clear();
    profile_ = on;
}
namespace {
// event record that becomes a graph node when the stream is being captured
void record_event(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CPK_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) CPK_CUDA(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else CPK_CUDA(cudaEventRecord(e, st));
}
}  // namespace
void DeviceProblem::prof_begin(int kind) {
    if (!profile_) return;
    ProfEvent e{};
    e.kind = kind;
    CPK_CUDA(cudaEventCreate(&e.a));
    CPK_CUDA(cudaEventCreate(&e.b));
    record_event(e.a, ctx_.stream);  // a graph node inside a captured ALS sweep
    prof_.push_back(e);
}
void DeviceProblem::prof_end() {
    if (!profile_) return;
    record_event(prof_.back().b, ctx_.stream);
}
void DeviceProblem::profile_read(double* ms, int* count) {
    ctx_.sync();
    for (int k = 0; k < kProfKinds; ++k) {
        ms[k] = 0.0;
        count[k] = 0;
    }
    for (auto& e : prof_) {
        float v = e.ms;
        if (v < 0.0f) CPK_CUDA(cudaEventElapsedTime(&v, e.a, e.b));
        ms[e.kind] += v;
        count[e.kind] += 1;
    }
}

// ---- dimension tree (mttkrp.cpp:160-189) -----------------------------------
void DeviceProblem::root_back() {
    NvtxRange nvtx_range("cpkit:root_back");
    const int N = order();
    prof_begin(kProfBack);
    launch_root_back(x_.get(), F_, Bl_, Bs_, R_, krp(h_, N, A_.get(), true), krp_.get(), PF_.get(), ws_.get(),
                     ws_.size(), ctx_.stream, side_busy_ ? 1 : 0);
    prof_end();
    ++contractions_;
    pf_valid_ = true;
}
void DeviceProblem::root_front() {
    NvtxRange nvtx_range("cpkit:root_front");
    prof_begin(kProfFront);
    if (front_copy_)  // P_B = X^T KRP_F on the transposed copy: the back root's NN GEMM
        launch_root_back(XT_.get(), Bl_, F_, ldT_, R_, krp(0, h_, A_.get(), false), krp_.get(), PB_.get(), ws_.get(),
                         ws_.size(), ctx_.stream, side_busy_ ? 1 : 0);
    else
        launch_root_front(x_.get(), F_, Bl_, Bs_, R_, krp(0, h_, A_.get(), false), krp_.get(), PB_.get(), ws_.get(),
                          ws_.size(), ctx_.stream);
    prof_end();
    ++contractions_;
    pb_valid_ = true;
}
void DeviceProblem::second_level_back(int mode, cudaStream_t st, double* ws, std::size_t ws_elems) {
    if (!st) {
        st = ctx_.stream;
        ws = ws_.get();
        ws_elems = ws_.size();
    }
    double* out = M_.get() + off_[mode];
    if (h_ == 1) {
        CPK_CUDA(cudaMemcpyAsync(out, PF_.get(), static_cast<std::size_t>(F_) * R_ * sizeof(double),
                                 cudaMemcpyDeviceToDevice, st));
    } else {
        launch_reduce_kept(PF_.get(), krp(0, h_, A_.get(), false), mode, R_, out, ws, ws_elems, st);
    }
    if (ctx_.comm && !defer_coll_) ctx_.comm->allreduce_sum(out, static_cast<std::size_t>(dims_[mode]) * R_, st);
}
double DeviceProblem::time_second_level(int reps, double* bytes) {
    if (!pf_valid_) root_back();
    second_level_back(0);  // warm-up
    cudaEvent_t a, b;
    CPK_CUDA(cudaEventCreate(&a));
    CPK_CUDA(cudaEventCreate(&b));
    CPK_CUDA(cudaEventRecord(a, ctx_.stream));
    for (int i = 0; i < reps; ++i) second_level_back(0);
    CPK_CUDA(cudaEventRecord(b, ctx_.stream));
    CPK_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    CPK_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    m_all_valid_ = false;  // M^(0) was rewritten outside the cache bookkeeping
    if (bytes) *bytes = 8.0 * static_cast<double>(F_) * R_;
    return static_cast<double>(ms) / reps;
}
void DeviceProblem::second_level_front(int mode) {
    const int N = order();
    const bool last = (mode == N - 1);
    // rows of the last mode land at their global slab position
    double* out = M_.get() + off_[mode] + (last ? static_cast<std::int64_t>(slab_lo_) * R_ : 0);
    if (N - h_ == 1) {
        CPK_CUDA(cudaMemcpyAsync(out, PB_.get(), static_cast<std::size_t>(Bl_) * R_ * sizeof(double),
                                 cudaMemcpyDeviceToDevice, ctx_.stream));
    } else {
        launch_reduce_kept(PB_.get(), krp(h_, N, A_.get(), true), mode - h_, R_, out, ws_.get(), ws_.size(),
                           ctx_.stream);
    }
    if (ctx_.comm && !defer_coll_) {
        if (last) {
            const std::size_t per = static_cast<std::size_t>(slab_hi_ - slab_lo_) * R_;
            ctx_.comm->allgather(out, M_.get() + off_[mode], per, ctx_.stream);
        } else {
            ctx_.comm->allreduce_sum(out, static_cast<std::size_t>(dims_[mode]) * R_, ctx_.stream);
        }
    }
}

// ---- order-3 ALS: multi-sweep dimension tree --------------------------------
// The ALS update order 0, 1, 2, 0, 1, 2, ... lets one first-level contraction
// serve two consecutive updates: P_c = X x_c A_c with c the mode updated
// neither now nor next stays valid for both (A_c does not change in between),
// and M^(n) is P_c contracted with the other kept factor, the one updated
// just before (the same second-level step as mttkrp.cpp:63-75). The roots
// rotate c = 2, 1, 0 (X A_2 is the tree's back root; X x_1 A_1 and X x_0 A_0
// are single-mode TN contractions), 3 roots per 2 sweeps instead of 4, and no
// Khatri-Rao operand. Each M^(n) is the same sum as the reference tree's, in
// a different association order (roundoff-level differences).
void DeviceProblem::root_single(int c) {
    NvtxRange nvtx_range("cpkit:root_single");
    prof_begin(kProfFront);
    if (msdt_copies_) {
        // P_c = X^(c) A_c: rows (other kept index pairs), the back root's NN GEMM
        KrpDesc kc{};
        kc.nmodes = 1;
        kc.ext[0] = local_rows_[c];
        kc.fac[0] = A_.get() + off_[c];
        const std::int64_t rows = local_rows_[1 - c] * Bl_;
        launch_root_back(c == 0 ? X0_.get() : X1_.get(), rows, local_rows_[c], c == 0 ? ld0_ : ld1_, R_, kc,
                         krp_.get(), PM_.get(), ws_.get(), ws_.size(), ctx_.stream, side_busy_ ? 1 : 0);
    } else {
        launch_root_single(x_.get(), local_rows_[0], local_rows_[1], Bl_, Bs_, c, A_.get() + off_[c], R_, PM_.get(),
                           ws_.get(), ws_.size(), ctx_.stream);
    }
    prof_end();
    ++contractions_;
    pm_mode_ = c;
}
void DeviceProblem::second_level_pm(int mode) {
    const int N = order();
    KrpDesc kd{};
    kd.nmodes = 2;
    int keep = -1;
    for (int m = 0, j = 0; m < N; ++m) {
        if (m == pm_mode_) continue;
        if (m == mode) keep = j;
        const bool last = m == N - 1;
        kd.ext[j] = local_rows_[m];
        kd.fac[j] = A_.get() + off_[m] + (last ? static_cast<std::int64_t>(slab_lo_) * R_ : 0);
        ++j;
    }
    const bool last = mode == N - 1;
    double* out = M_.get() + off_[mode] + (last ? static_cast<std::int64_t>(slab_lo_) * R_ : 0);
    launch_reduce_kept(PM_.get(), kd, keep, R_, out, ws_.get(), ws_.size(), ctx_.stream);
    if (ctx_.comm && !defer_coll_) {
        if (last) {
            const std::size_t per = static_cast<std::size_t>(slab_hi_ - slab_lo_) * R_;
            ctx_.comm->allgather(out, M_.get() + off_[mode], per, ctx_.stream);
        } else {
            ctx_.comm->allreduce_sum(out, static_cast<std::size_t>(dims_[mode]) * R_, ctx_.stream);
        }
    }
}
void DeviceProblem::mttkrp_msdt(int mode) {
    if (pf_valid_ && mode != 2) {  // P_2 = X A_2 serves modes 0 and 1
        second_level_back(mode);
        return;
    }
    if (pm_mode_ >= 0 && pm_mode_ != mode) {
        second_level_pm(mode);
        return;
    }
    const int c = (mode + 2) % 3;  // updated neither now nor next
    if (c == 2) {
        root_back();
        second_level_back(mode);
    } else {
        root_single(c);
        second_level_pm(mode);
    }
}

void DeviceProblem::mttkrp(int mode) {
    if (mode < 0 || mode >= order()) throw InvalidArgument("mttkrp: mode out of range");
    if (mode < h_) {
        if (!pf_valid_) root_back();
        second_level_back(mode);
    } else {
        if (!pb_valid_) root_front();
        second_level_front(mode);
    }
}
void DeviceProblem::mttkrp_naive(int mode) {
    if (mode < 0 || mode >= order()) throw InvalidArgument("mttkrp: mode out of range");
    const int saved = contractions_;
    if (mode < h_) {
        root_back();
        second_level_back(mode);
        pf_valid_ = false;
    } else {
        root_front();
        second_level_front(mode);
        pb_valid_ = false;
    }
    contractions_ = saved;  // the uncached overload does not count (mttkrp.cpp:149-158)
}
void DeviceProblem::note_factor_update(int mode) {
    if (mode >= h_) pf_valid_ = false;  // back-root key holds modes >= h
    else pb_valid_ = false;             // front-root key holds modes < h
    if (mode == pm_mode_) pm_mode_ = -1;
    pinv_ready_ = false;
    res_current_ = false;
    m_all_valid_ = false;
}
void DeviceProblem::invalidate_all() {  // factors changed wholesale
    preset_valid_ = false;
    pinv_ready_ = false;
    res_current_ = false;
    pf_valid_ = pb_valid_ = false;
    pm_mode_ = -1;
    m_all_valid_ = false;
    grams_valid_ = false;
}
void DeviceProblem::download_mttkrp(int mode, double* host) {
    CPK_CUDA(cudaMemcpyAsync(host, M_.get() + off_[mode], (off_[mode + 1] - off_[mode]) * sizeof(double),
                             cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
}
// Every M^(n) of one factor set. Sharded: the N-1 partial s_n x R blocks
// (contiguous in M) are all-reduced in ONE collective and the last mode's
// slab rows all-gathered once (GN).
void DeviceProblem::compute_all_mttkrp() {
    const int N = order();
    defer_coll_ = ctx_.comm != nullptr;
    try {
        if (msdt_copies_) {
            // order 3: M^(0), M^(1) from the back root X A_2; M^(2) from the
            // single-mode root X x_1 A_1 (NN GEMM on the permuted copy, then the
            // i0 contraction) instead of the Khatri-Rao front root. The two
            // HBM-bound reduces of X A_2 run on a third stream beside the
            // DMMA-bound second root (own workspace; collectives deferred).
            if (!pf_valid_) root_back();
            const bool beside = pm_mode_ != 1 && !std::getenv("CPKIT_NO_REDUCE_OVERLAP");
            if (beside) {
                CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2A], ctx_.stream));
                CPK_CUDA(cudaStreamWaitEvent(ctx_.aux2, ctx_.ev[Context::kEvAux2A], 0));
                const bool dc = defer_coll_;
                defer_coll_ = true;  // a sharded run reduces every block after the pass anyway
                second_level_back(0, ctx_.aux2, ws_red_.get(), ws_red_.size());
                second_level_back(1, ctx_.aux2, ws_red_.get(), ws_red_.size());
                defer_coll_ = dc;
                CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2B], ctx_.aux2));
                root_single(1);
                second_level_pm(2);
                CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[Context::kEvAux2B], 0));
            } else {
                mttkrp(0);
                mttkrp(1);
                if (pm_mode_ != 1) root_single(1);
                second_level_pm(2);
            }
        } else {
            for (int n = 0; n < N; ++n) mttkrp(n);
        }
    } catch (...) {
        defer_coll_ = false;
        throw;
    }
    defer_coll_ = false;
    if (ctx_.comm) {
        ctx_.comm->allreduce_sum(M_.get(), static_cast<std::size_t>(off_[N - 1]), ctx_.stream);
        const std::size_t per = static_cast<std::size_t>(slab_hi_ - slab_lo_) * R_;
        ctx_.comm->allgather(M_.get() + off_[N - 1] + static_cast<std::int64_t>(slab_lo_) * R_,
                             M_.get() + off_[N - 1], per, ctx_.stream);
    }
    m_all_valid_ = true;
}

// ---- Gamma set / residual / gradient --------------------------------------
void DeviceProblem::grams_all() {
    if (grams_valid_) return;  // already gram(A_n) for the current factors
    launch_grams(A_.get(), offs_dev_.get(), rows_dev_.get(), 0, order(), R_, smax_, gram_ws_.get(), grams_.get(),
                 ctx_.stream);
    grams_valid_ = true;
}
void DeviceProblem::build_gamma_set() {
    grams_all();
    launch_gamma_pairs(grams_.get(), order(), R_, pair_.get(), ctx_.stream);
}
void DeviceProblem::download_gammas(double* grams, double* pair) {
    const std::size_t RR = static_cast<std::size_t>(R_) * R_;
    const int N = order();
    CPK_CUDA(cudaMemcpyAsync(grams, grams_.get(), N * RR * 8, cudaMemcpyDeviceToHost, ctx_.stream));
    CPK_CUDA(cudaMemcpyAsync(pair, pair_.get(), N * N * RR * 8, cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
}
void DeviceProblem::upload_gammas(const double* grams, const double* pair) {
    const std::size_t RR = static_cast<std::size_t>(R_) * R_;
    const int N = order();
    CPK_CUDA(cudaMemcpyAsync(grams_.get(), grams, N * RR * 8, cudaMemcpyHostToDevice, ctx_.stream));
    CPK_CUDA(cudaMemcpyAsync(pair_.get(), pair, N * N * RR * 8, cudaMemcpyHostToDevice, ctx_.stream));
    grams_valid_ = false;  // caller-provided, not necessarily gram(A)
}
void DeviceProblem::residual_launch(double xnorm2) {
    if (!(xnorm2 > 0.0)) throw InvalidArgument("residual_fitness: tensor norm must be positive");
    const int N = order();
    if (xnorm_dev_ != xnorm2) {  // the slot keeps its value between calls: no copy-engine hop per GN step
        hpin_[8] = xnorm2;       // pinned upload slot (reused only after a later synchronisation)
        CPK_CUDA(cudaMemcpyAsync(scal_.get() + kXnorm, hpin_ + 8, sizeof(double), cudaMemcpyHostToDevice,
                                 ctx_.stream));
        xnorm_dev_ = xnorm2;
    }
    launch_residual(M_.get() + off_[N - 1], A_.get() + off_[N - 1], static_cast<std::int64_t>(dims_[N - 1]),
                    grams_.get(), N, R_, scal_.get() + kXnorm, partials_.get(), scal_.get() + kRes,
                    ctx_.stream);
}
// The residual with ||X||^2 already in its device slot (norm2() leaves it there).
void DeviceProblem::residual_launch_dev() {
    const int N = order();
    launch_residual(M_.get() + off_[N - 1], A_.get() + off_[N - 1], static_cast<std::int64_t>(dims_[N - 1]),
                    grams_.get(), N, R_, scal_.get() + kXnorm, partials_.get(), scal_.get() + kRes,
                    ctx_.stream);
}
std::pair<double, double> DeviceProblem::residual_fitness(double xnorm2, int /*last_src*/) {
    residual_launch(xnorm2);
    CPK_CUDA(cudaMemcpyAsync(hpin_, scal_.get() + kRes, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync_main();
    return {hpin_[0], hpin_[1]};
}
void DeviceProblem::gradient() {
    const int N = order();
    std::vector<std::int64_t> rows(dims_.begin(), dims_.end());
    launch_gradient_all(A_.get(), pair_.get(), M_.get(), off_.data(), rows.data(), N, R_, G_.get(), ctx_.stream);
}
double DeviceProblem::norm_sum(const double* dev_stacked) {
    launch_block_norm_sum(dev_stacked, offs_dev_.get(), order(), partials_.get(), scal_.get() + kNormSum, 1.0,
                          ctx_.stream);
    return read_scalar(kNormSum);
}

// ---- SPD ---------------------------------------------------------------------
void DeviceProblem::check_status(int count, const char* what) {
    std::vector<int> st(count);
    CPK_CUDA(cudaMemcpyAsync(st.data(), status_.get(), count * sizeof(int), cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
    for (int s : st)
        if (s == 2) throw SingularSystem(std::string(what) + ": factorization failed after jitter retry");
}
void DeviceProblem::spd_solve(const double* dev_s, const double* dev_b, std::int64_t rows, double lambda,
                              double* dev_y) {
    launch_chol_batch(dev_s, 1, R_, &lambda, 0, chol_.get(), status_.get(), ctx_.stream);
    check_status(1, "spd_solve");
    launch_chol_solve_rows(chol_.get(), R_, dev_b, rows, dev_y, ctx_.stream);
}
void DeviceProblem::spd_inverse(const double* dev_s, double lambda, double* dev_inv) {
    launch_chol_batch(dev_s, 1, R_, &lambda, 0, chol_.get(), status_.get(), ctx_.stream);
    check_status(1, "spd_solve");
    launch_chol_inverse_batch(chol_.get(), 1, R_, dev_inv, chol_tmp_.get(), ctx_.stream);
}
// gauss_newton.cpp:190-207: per mode (Gamma(n,n) + lambda Reg)^-1. The N
// Cholesky factorisations run on the side stream as soon as the Gamma set
// exists, overlapping the residual / gradient work of gn_step.
void DeviceProblem::launch_preconditioner_factor(double lambda, RegShape shape) {
    if (lambda < 0) throw InvalidArgument("build_preconditioner: lambda must be nonnegative");
    const int N = order();
    const std::size_t RR = static_cast<std::size_t>(R_) * R_;
    CPK_CUDA(cudaEventRecord(ctx_.ev[0], ctx_.stream));  // Gamma set ready
    CPK_CUDA(cudaStreamWaitEvent(ctx_.aux, ctx_.ev[0], 0));
    // Gamma(n,n) read in place from the pair array (diagonal blocks, (N+1) R^2 apart)
    launch_chol_batch_strided(pair_.get(), static_cast<long long>(N + 1) * RR, N, R_, &lambda,
                              shape == RegShape::identity ? 0 : 1, chol_.get(), status_.get(), ctx_.aux);
    CPK_CUDA(cudaEventRecord(ctx_.ev[1], ctx_.aux));
    precond_pending_ = true;
    precond_lambda_ = lambda;
    precond_shape_ = shape;
}
void DeviceProblem::launch_precond_chain(double lambda, RegShape shape, bool grams_and_gamma) {
    if (lambda < 0) throw InvalidArgument("build_preconditioner: lambda must be nonnegative");
    const int N = order();
    const std::size_t RR = static_cast<std::size_t>(R_) * R_;
    CPK_CUDA(cudaEventRecord(ctx_.ev[0], ctx_.stream));  // factors (and, if not recomputed, Gamma set) ready
    CPK_CUDA(cudaStreamWaitEvent(ctx_.aux, ctx_.ev[0], 0));
    if (grams_and_gamma) {
        launch_grams(A_.get(), offs_dev_.get(), rows_dev_.get(), 0, N, R_, smax_, gram_ws_.get(), grams_.get(),
                     ctx_.aux);
        launch_gamma_pairs(grams_.get(), N, R_, pair_.get(), ctx_.aux);
        grams_valid_ = true;
    }
    launch_chol_batch_strided(pair_.get(), static_cast<long long>(N + 1) * RR, N, R_, &lambda,
                              shape == RegShape::identity ? 0 : 1, chol_.get(), status_.get(), ctx_.aux);
    launch_chol_inverse_batch(chol_.get(), N, R_, pinv_.get(), chol_tmp_.get(), ctx_.aux);
    CPK_CUDA(cudaEventRecord(ctx_.ev[1], ctx_.aux));
}
void DeviceProblem::build_preconditioner(double lambda, RegShape shape) {
    NvtxRange nvtx_range("cpkit:build_preconditioner");
    if (lambda < 0) throw InvalidArgument("build_preconditioner: lambda must be nonnegative");
    if (!precond_pending_ || precond_lambda_ != lambda || precond_shape_ != shape)
        launch_preconditioner_factor(lambda, shape);
    precond_pending_ = false;
    CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[1], 0));
    check_status(order(), "spd_solve");
    launch_chol_inverse_batch(chol_.get(), order(), R_, pinv_.get(), chol_tmp_.get(), ctx_.stream);
}

// ---- J^T J v and CG ------------------------------------------------------------
namespace {
CgParams base_params(int N, int R, const std::vector<std::uint64_t>& dims, const std::vector<std::int64_t>& off) {
    CgParams p{};
    p.order = N;
    p.R = R;
    for (int n = 0; n < N; ++n) p.rows[n] = static_cast<std::int64_t>(dims[n]);
    for (int n = 0; n <= N; ++n) p.off[n] = off[n];
    return p;
}
}  // namespace

void DeviceProblem::jtj_matvec(const double* dev_w, double* dev_u, double lambda, RegShape shape) {
    NvtxRange nvtx_range("cpkit:jtj_matvec");
    CgParams p = base_params(order(), R_, dims_, off_);
    p.A = A_.get();
    p.pair = pair_.get();
    p.W[1] = W_[1].get();
    p.slots = slots_.get();
    p.nslots = static_cast<int>(slots_.size());
    p.barrier = barrier_.get();
    p.lambda = lambda;
    p.shape = shape == RegShape::identity ? 0 : 1;
    cg_barrier_ready();
    launch_jtj_matvec(p, dev_w, dev_u, ctx_.stream);
    barrier_zero_ = false;  // used: the next solve zeroes it itself
}

// gauss_newton.cpp:279-349; G must hold the gradient. Result in V.
CgResultInfo DeviceProblem::cp_cg(double lambda, const GnConfig& cfg, double gnorm_in) {
    NvtxRange nvtx_range("cpkit:cp_cg");
    const int N = order();
    const RegShape shape = cfg.schedule.shape;
    int cap = cfg.cg_max_iters;
    if (cap <= 0) {  // default_cg_cap (gauss_newton.cpp:267-275)
        std::uint64_t total = 0;
        for (auto d : dims_) total += d * static_cast<std::uint64_t>(R_);
        cap = static_cast<int>(std::min<std::uint64_t>(total, 10ull * static_cast<std::uint64_t>(R_)));
    }
    CgResultInfo out;
    const double gnorm = gnorm_in >= 0.0 ? gnorm_in : norm_sum(G_.get());
    if (gnorm == 0.0) {
        ctx_.sync();  // drop any speculative preconditioner factorisation
        precond_pending_ = false;
        CPK_CUDA(cudaMemsetAsync(V_.get(), 0, off_[N] * sizeof(double), ctx_.stream));
        return out;
    }
    build_preconditioner(lambda, shape);
    CgParams p = base_params(N, R_, dims_, off_);
    p.A = A_.get();
    p.pair = pair_.get();
    p.pinv = pinv_.get();
    p.G = G_.get();
    p.V = V_.get();
    p.Rr[0] = Rr_[0].get();
    p.Rr[1] = Rr_[1].get();
    p.W[0] = W_[0].get();
    p.W[1] = W_[1].get();
    p.Z = Z_.get();
    p.Q = Q_.get();
    p.slots = slots_.get();
    p.nslots = static_cast<int>(slots_.size());
    p.barrier = barrier_.get();
    p.lambda = lambda;
    p.shape = shape == RegShape::identity ? 0 : 1;
    p.beta_variant = cfg.cg_beta == CgBetaVariant::standard ? 0 : 1;
    p.cg_tol = cfg.cg_tol;
    p.cap = cap;
    p.result = cgres_.get();
    DevBuf<unsigned long long> trace;
    const bool want_trace = std::getenv("CPKIT_CG_TRACE") != nullptr;
    if (want_trace) {
        trace.resize(64 * 16 + 1024);
        CPK_CUDA(cudaMemsetAsync(trace.get(), 0, (64 * 16 + 1024) * 8, ctx_.stream));
        p.trace = trace.get();
    }
    prof_begin(kProfCg);
    cg_barrier_ready();
    run_cg(p, cg_max_grid(ctx_.device), ctx_.stream);
    barrier_zero_ = false;  // used: the next solve zeroes it itself
    prof_end();
    if (want_trace) {
        std::vector<unsigned long long> h(64 * 16 + 1024);
        CPK_CUDA(cudaMemcpyAsync(h.data(), trace.get(), h.size() * 8, cudaMemcpyDeviceToHost, ctx_.stream));
        ctx_.sync();
        std::fprintf(stderr, "cg block->sm:");
        for (int b = 0; b < 16; ++b) std::fprintf(stderr, " %llu", h[64 * 16 + b]);
        std::fprintf(stderr, "\n");
        auto dt = [&](int it, int a, int b) { return (static_cast<double>(h[it * 16 + b]) - static_cast<double>(h[it * 16 + a])) * 1e-3; };
        for (int it = 0; it < 64 && h[it * 16]; ++it) {
            std::fprintf(stderr, "cg it %2d:", it);
            for (int k = 1; k < 8; ++k) std::fprintf(stderr, " %6.2f", dt(it, k - 1, k));
            if (it + 1 < 64 && h[(it + 1) * 16])
                std::fprintf(stderr, " | next %6.2f", (static_cast<double>(h[(it + 1) * 16]) - static_cast<double>(h[it * 16 + 7])) * 1e-3);
            if (h[it * 16 + 12])
                std::fprintf(stderr, " | C wq %5.2f rows %5.2f tail %5.2f zpart %5.2f", dt(it, 5, 9), dt(it, 9, 10),
                             dt(it, 10, 11), dt(it, 11, 12));
            if (h[it * 16 + 8])
                std::fprintf(stderr, " | A2 work %5.2f", dt(it, 2, 8));
            if (h[it * 16 + 13])
                std::fprintf(stderr, " | B pull %5.2f", dt(it, 3, 13));
            std::fprintf(stderr, " us\n");
        }
    }
    int res[5];
    CPK_CUDA(cudaMemcpyAsync(res, cgres_.get(), sizeof res, cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
    if (res[3]) throw NumericalFailure("cp_cg: non-finite iterate");
    out.iterations = res[0];
    out.hit_cap = res[1] != 0;
    out.breakdown = res[2] != 0;
    return out;
}

// ---- ALS sweep (als.cpp:22-52) ----------------------------------------------------
void DeviceProblem::drop_als_graph() {
    for (auto& g : als_graphs_) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        for (auto& e : g.prof) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
    }
    als_graphs_.clear();
}

// The device work of one sweep (no host synchronisation, capturable).
void DeviceProblem::als_sweep_body(double lambda) {
    const int N = order();
    const std::size_t RR = static_cast<std::size_t>(R_) * R_;
    reset_contraction_counter();
    launch_set_flag_scalar(flag_.get(), 1, scal_.get() + kStep, 0.0, ctx_.stream);
    launch_all_finite(A_.get(), off_[N], flag_.get(), ctx_.stream);  // model.validate()
    grams_all();
    const std::size_t LDR = chol_factor_elems(1, R_);
    for (int n = 0; n < N; ++n) {
        // side stream: Gamma^(n) from the current grams, then its Cholesky factor,
        // overlapping the MTTKRP of mode n on the main stream
        CPK_CUDA(cudaEventRecord(ctx_.ev[2 + 2 * n], ctx_.stream));
        CPK_CUDA(cudaStreamWaitEvent(ctx_.aux, ctx_.ev[2 + 2 * n], 0));
        launch_chol_batch_src(gam_.get() + n * RR, grams_.get(), N, n, 1, R_, &lambda, 0, chol_.get() + n * LDR,
                              status_.get() + n, ctx_.aux);
        CPK_CUDA(cudaEventRecord(ctx_.ev[3 + 2 * n], ctx_.aux));
        side_busy_ = true;
        if (msdt_) mttkrp_msdt(n);
        else mttkrp(n);
        side_busy_ = false;
        CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[3 + 2 * n], 0));
        const std::int64_t rows = static_cast<std::int64_t>(dims_[n]);
        // A_n <- M_n (Gamma + lambda I)^-1 in place; the step norm from per-row partials
        launch_chol_solve_rows_update(chol_.get() + n * LDR, R_, M_.get() + off_[n], rows, A_.get() + off_[n],
                                      partials_.get(), ctx_.stream);
        note_factor_update(n);
        // Gram of the new factor; its first CTA also folds in this mode's step norm
        launch_grams(A_.get(), offs_dev_.get(), rows_dev_.get(), n, n + 1, R_, smax_, gram_ws_.get(), grams_.get(),
                     ctx_.stream, partials_.get(), static_cast<int>(rows), scal_.get() + kStep);
    }
    (void)RR;
}

AlsSweepDiag DeviceProblem::als_sweep(double lambda) {
    als_sweep_launch(lambda, false);
    return als_sweep_finish();
}

void DeviceProblem::als_snapshot_factors() {
    CPK_CUDA(cudaMemcpyAsync(Atrial_.get(), A_.get(), off_[order()] * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx_.stream));
}
void DeviceProblem::restore_factors_from(const double* src) {
    CPK_CUDA(cudaMemcpyAsync(A_.get(), src, off_[order()] * sizeof(double), cudaMemcpyDeviceToDevice, ctx_.stream));
    invalidate_all();
}
void DeviceProblem::als_restore_factors() {
    CPK_CUDA(cudaMemcpyAsync(A_.get(), Atrial_.get(), off_[order()] * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx_.stream));
    invalidate_all();
}

void DeviceProblem::als_sweep_launch(double lambda, bool with_residual) {
    NvtxRange nvtx_range("cpkit:als_sweep");
    const int N = order();
    while (static_cast<int>(pending_.size()) >= kSweepSlots - 1) done_.push_back(complete_oldest());
    // CUDA graph: one capture per (lambda, cache state, profiling); replays skip
    // ~30 launch latencies per sweep. Single GPU only (the sharded sweep has
    // NCCL collectives between its kernels).
    const bool graphs = !ctx_.comm && !std::getenv("CPKIT_NO_GRAPH");
    const SweepSig pre = sweep_sig();
    bool replayed = false;
    AlsGraph* hit = nullptr;
    if (graphs)
        for (auto& g : als_graphs_)
            if (g.lambda == lambda && g.pre == pre) hit = &g;
    if (hit && profile_)
        for (const auto& q : pending_)
            if (q.graph == hit) {
                drain_pending();
                break;
            }
    if (hit) {
        CPK_CUDA(cudaGraphLaunch(hit->exec, ctx_.stream));
        count_launch(static_cast<int>(hit->kernels));  // the replay launches the captured kernels again
        pf_valid_ = hit->post.pf;
        pb_valid_ = hit->post.pb;
        m_all_valid_ = hit->post.mall;
        grams_valid_ = hit->post.grams;
        pm_mode_ = hit->post.pm;
        contractions_ = hit->contr;
        replayed = true;
    } else if (graphs) {
        if (als_graphs_.size() >= kAlsGraphs) {
            drain_pending();  // in-flight replays still reference them
            drop_als_graph();
        }
        const std::size_t prof0 = prof_.size();
        const long long k0 = static_cast<long long>(kernel_launches());
        std::unique_lock<std::recursive_mutex> guard_lock(guard_capture_mutex(), std::defer_lock);
        if (guard_enabled()) guard_lock.lock();  // CPKIT_GUARD: red-zone checks synchronise the device
        CPK_CUDA(cudaStreamBeginCapture(ctx_.stream, cudaStreamCaptureModeThreadLocal));
        try {
            als_sweep_body(lambda);
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(ctx_.stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t g = nullptr;
        CPK_CUDA(cudaStreamEndCapture(ctx_.stream, &g));
        AlsGraph ag;
        CPK_CUDA(cudaGraphInstantiate(&ag.exec, g, cudaGraphInstantiateFlagUseNodePriority));
        CPK_CUDA(cudaGraphDestroy(g));
        ag.lambda = lambda;
        ag.pre = pre;
        ag.post = sweep_sig();
        ag.contr = contractions_;
        ag.kernels = static_cast<long long>(kernel_launches()) - k0;  // counted as captured, i.e. as launched by the first replay below
        ag.prof.assign(prof_.begin() + static_cast<std::ptrdiff_t>(prof0), prof_.end());  // owned by the graph now
        prof_.resize(prof0);
        als_graphs_.push_back(std::move(ag));
        hit = &als_graphs_.back();
        CPK_CUDA(cudaGraphLaunch(hit->exec, ctx_.stream));
        replayed = true;
    } else {
        als_sweep_body(lambda);
    }
    if (with_residual) residual_launch_dev();
    const int slot = next_slot_;
    next_slot_ = (next_slot_ + 1) % kSweepSlots;
    launch_pack_sweep(scal_.get(), kStep, kRes, flag_.get(), status_.get(), N, dmap_ + slot * kSlotDoubles,
                      ctx_.stream);
    CPK_CUDA(cudaEventRecord(slot_ev_[slot], ctx_.stream));
    pending_.push_back({slot, contractions_, replayed && profile_ ? hit : nullptr});
}

DeviceProblem::SweepResult DeviceProblem::complete_oldest() {
    const PendingSweep q = pending_.front();
    pending_.erase(pending_.begin());
    CPK_CUDA(cudaEventSynchronize(slot_ev_[q.slot]));
    const double* h = hmap_ + q.slot * kSlotDoubles;
    if (q.graph)  // the graph's event pairs, measured for this replay
        for (const auto& e : q.graph->prof) {
            float v = 0.0f;
            CPK_CUDA(cudaEventElapsedTime(&v, e.a, e.b));
            prof_.push_back({nullptr, nullptr, e.kind, v});
        }
    SweepResult r;
    r.diag.step_norm = h[0];
    r.diag.full_contractions = q.contr;
    r.res = h[1];
    r.fit = h[2];
    if (h[3] == 0.0) r.err = 1;
    for (int n = 0; n < order() && !r.err; ++n)
        if (h[4 + n] == 2.0) r.err = 2;
    return r;
}

AlsSweepDiag DeviceProblem::als_sweep_finish(double* res, double* fit) {
    SweepResult r;
    if (!done_.empty()) {
        r = done_.front();
        done_.erase(done_.begin());
    } else {
        if (pending_.empty()) throw InvalidArgument("als_sweep_finish: no sweep in flight");
        r = complete_oldest();
    }
    if (res) *res = r.res;
    if (fit) *fit = r.fit;
    if (r.err == 1) throw InvalidArgument("model factor contains non-finite entries");
    if (r.err == 2) throw SingularSystem("spd_solve: factorization failed after jitter retry");
    return r.diag;
}

// ---- GN step (gauss_newton.cpp:360-449) -------------------------------------------
// B200 change: the post-step residual reuses the next iteration's tree pass
// (one fused set of two root contractions computes every M^(n) of the new
// factors; M^(N-1) gives residual_after and the rest is cached for the next
// step), instead of a third, naive contraction (:442-444).
// B200 change: the default step (no Armijo search) runs start to finish on
// the device with ONE host synchronisation. The reference's early exits
// (residual / gradient halt, gauss_newton.cpp:370-389), the preconditioner's
// SingularSystem and cp_cg's non-finite check are decided afterwards from
// values packed into mapped pinned memory; a step that must not have happened
// is undone from the device copy of the pre-step factors. Same results as the
// phase-by-phase version (`CPKIT_GN_SYNC=1`, used for Armijo).
bool DeviceProblem::ref_residual(const GnConfig& cfg) {
    static const bool env = std::getenv("CPKIT_GN_REF_RESIDUAL") != nullptr;
    return cfg.residual_naive || env;
}
GnStepDiag DeviceProblem::gn_step(const GnConfig& cfg, RegSchedule& schedule, double xnorm2) {
    if (cfg.armijo || std::getenv("CPKIT_GN_SYNC")) return gn_step_sync(cfg, schedule, xnorm2);
    gn_enqueue(cfg, schedule, xnorm2, 0);
    GnStepDiag diag = gn_decode(cfg, schedule.lambda, 0);
    if (diag.stepped) schedule = schedule_next(schedule);
    return diag;
}

// The whole default step queued on the device. slot selects the diagnostics
// area, the pre-step snapshot and the completion event, so that two steps can
// be in flight (gn_optimize queues step k+1 before reading step k).
void DeviceProblem::gn_enqueue(const GnConfig& cfg, const RegSchedule& schedule, double xnorm2, int slot) {
    NvtxRange nvtx_range("cpkit:gn_step");
    const int N = order();
    const std::uint64_t S = static_cast<std::uint64_t>(off_[N]);
    // [res, fit, (step slot), gnorm | status N | cg 5 | step, fin | res_after, fit_after]
    double* dm = dmap_ + kGnMapOff + slot * kGnMapDoubles;
    double* snap = slot == 0 ? Atrial_.get() : Asnap1_.get();
    static_assert(kRes + 3 == kNormSum, "residual, fitness, step and gradient-norm slots are adjacent");
    const int o_gn = 3, o_st = 4, o_cg = 4 + N, o_step = 9 + N, o_after = 11 + N;
    const RegShape shape = cfg.schedule.shape;
    if (!m_all_valid_) compute_all_mttkrp();
    // ready: launched at the end of the previous step, which waited for it before its residual
    const bool chain_waited = pinv_ready_ && pinv_lambda_ == schedule.lambda && pinv_shape_ == shape;
    if (!chain_waited) {
        build_gamma_set();
        launch_precond_chain(schedule.lambda, shape, false);  // side stream, overlaps residual/gradient
    }
    pinv_ready_ = false;
    precond_pending_ = false;
    if (!(res_current_ && res_xnorm_ == xnorm2)) residual_launch(xnorm2);  // else: the last step's residual_after
    gradient();
    launch_block_norm_sum(G_.get(), offs_dev_.get(), N, partials_.get(), scal_.get() + kNormSum, 1.0, ctx_.stream);
    // pre-step factors (restored when the step must not happen), copied on the
    // third stream while the CG runs; the update waits for it
    CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2A], ctx_.stream));
    CPK_CUDA(cudaStreamWaitEvent(ctx_.aux2, ctx_.ev[Context::kEvAux2A], 0));
    CPK_CUDA(cudaMemcpyAsync(snap, A_.get(), off_[N] * sizeof(double), cudaMemcpyDeviceToDevice, ctx_.aux2));
    CPK_CUDA(cudaEventRecord(ctx_.ev[Context::kEvAux2B], ctx_.aux2));
    // preconditioner inverse ready (its factorisation status is checked at the end)
    if (!chain_waited) CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[1], 0));
    // residual, fitness, gradient norm and the preconditioner status in one launch
    launch_pack_values(scal_.get() + kRes, 4, status_.get(), N, dm, ctx_.stream);
    CgParams p = base_params(N, R_, dims_, off_);
    int cap = cfg.cg_max_iters;
    if (cap <= 0) {  // default_cg_cap (gauss_newton.cpp:267-275)
        std::uint64_t total = 0;
        for (auto d : dims_) total += d * static_cast<std::uint64_t>(R_);
        cap = static_cast<int>(std::min<std::uint64_t>(total, 10ull * static_cast<std::uint64_t>(R_)));
    }
    p.A = A_.get();
    p.pair = pair_.get();
    p.pinv = pinv_.get();
    p.G = G_.get();
    p.V = V_.get();
    p.Rr[0] = Rr_[0].get();
    p.Rr[1] = Rr_[1].get();
    p.W[0] = W_[0].get();
    p.W[1] = W_[1].get();
    p.Z = Z_.get();
    p.Q = Q_.get();
    p.slots = slots_.get();
    p.nslots = static_cast<int>(slots_.size());
    p.barrier = barrier_.get();
    p.lambda = schedule.lambda;
    p.shape = cfg.schedule.shape == RegShape::identity ? 0 : 1;
    p.beta_variant = cfg.cg_beta == CgBetaVariant::standard ? 0 : 1;
    p.cg_tol = cfg.cg_tol;
    p.cap = cap;
    p.result = cgres_.get();
    p.barrier_zeroed = barrier_zero_;  // re-zeroed on the third stream after the previous solve
    cg_barrier_ready();
    prof_begin(kProfCg);
    run_cg(p, cg_max_grid(ctx_.device), ctx_.stream);  // G = 0: 0 iterations, V = 0 (cp_cg's shortcut)
    prof_end();
    // zero the grid barrier for the next solve now (in stream order; cheaper
    // than a cross-stream hand-off in front of the next cooperative launch)
    CPK_CUDA(cudaMemsetAsync(barrier_.get(), 0, cg_barrier_words() * sizeof(unsigned int), ctx_.stream));
    barrier_zero_ = true;
    CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[Context::kEvAux2B], 0));  // pre-step snapshot taken
    // A += V, step norm, finiteness, CG result and step diagnostics: one launch
    launch_gn_apply(A_.get(), V_.get(), offs_dev_.get(), N, partials_.get(), apply_bad_.get(), apply_cnt_.get(),
                    cgres_.get(), 5, dm + o_cg, scal_.get() + kNormSum, scal_.get() + kStep, flag_.get(),
                    dm + o_step, ctx_.stream);
    invalidate_all();
    // the next step's Grams, Gamma set and preconditioner (lambda of the next
    // schedule state) on the side stream, hidden behind the tree pass
    const RegSchedule next = schedule_next(schedule);
    launch_precond_chain(next.lambda, shape, true);
    pinv_ready_ = true;
    pinv_lambda_ = next.lambda;
    pinv_shape_ = shape;
    side_busy_ = true;
    if (ref_residual(cfg)) {
        // reference semantics: an uncached contraction of the stepped factors;
        // the next step recomputes its tree pass and residual_before
        mttkrp_naive(N - 1);
    } else {
        // residual_after from the next iteration's tree pass (cached for the next step)
        compute_all_mttkrp();
    }
    side_busy_ = false;
    CPK_CUDA(cudaStreamWaitEvent(ctx_.stream, ctx_.ev[1], 0));  // Grams
    residual_launch(xnorm2);
    res_current_ = !ref_residual(cfg);
    res_xnorm_ = xnorm2;
    launch_pack_values(scal_.get() + kRes, 2, nullptr, 0, dm + o_after, ctx_.stream);
    CPK_CUDA(cudaEventRecord(gn_ev_[slot], ctx_.stream));
}

// Decode a queued step: waits for its completion event only.
GnStepDiag DeviceProblem::gn_decode(const GnConfig& cfg, double lambda, int slot) {
    const int N = order();
    double* hm = hmap_ + kGnMapOff + slot * kGnMapDoubles;
    const int o_gn = 3, o_st = 4, o_cg = 4 + N, o_step = 9 + N, o_after = 11 + N;
    CPK_CUDA(cudaEventSynchronize(gn_ev_[slot]));
    gn_failed_applied_ = false;
    GnStepDiag diag;
    const double res = hm[0];
    diag.residual_before = res;
    diag.residual_after = res;
    auto undo = [&] {  // the step must not have happened: pre-step factors, caches rebuilt on demand
        restore_factors_from(slot == 0 ? Atrial_.get() : Asnap1_.get());
        ctx_.sync();
    };
    if (res < cfg.residual_tol) {
        undo();
        diag.halt = GnStepDiag::Halt::residual;
        return diag;
    }
    diag.grad_norm = hm[o_gn];
    if (diag.grad_norm <= cfg.grad_tol) {
        undo();
        diag.halt = GnStepDiag::Halt::gradient;
        return diag;
    }
    diag.lambda = lambda;
    if (diag.grad_norm != 0.0) {
        for (int n = 0; n < N; ++n)
            if (hm[o_st + n] == 2.0) {
                undo();
                throw SingularSystem("spd_solve: factorization failed after jitter retry");
            }
        if (hm[o_cg + 3] != 0.0) {
            undo();
            throw NumericalFailure("cp_cg: non-finite iterate");
        }
        diag.cg_iters = static_cast<int>(hm[o_cg]);
        diag.cg_hit_cap = hm[o_cg + 1] != 0.0;
        diag.cg_breakdown = hm[o_cg + 2] != 0.0;
    }
    diag.alpha = 1.0;
    diag.step_norm = hm[o_step];
    if (hm[o_step + 1] == 0.0) {
        gn_failed_applied_ = true;  // the step was applied (the reference throws after its update too)
        throw NumericalFailure("gn_step: non-finite factors after update");
    }
    diag.residual_after = hm[o_after];
    diag.stepped = true;
    return diag;
}


GnStepDiag DeviceProblem::gn_step_sync(const GnConfig& cfg, RegSchedule& schedule, double xnorm2) {
    NvtxRange nvtx_range("cpkit:gn_step_sync");
    const int N = order();
    const std::uint64_t S = static_cast<std::uint64_t>(off_[N]);
    GnStepDiag diag;
    if (!m_all_valid_) compute_all_mttkrp();
    build_gamma_set();
    launch_preconditioner_factor(schedule.lambda, cfg.schedule.shape);  // overlaps residual/gradient
    // residual and gradient norm in one readback (the gradient is computed even
    // when the residual test halts: an unused buffer, no observable difference)
    residual_launch(xnorm2);
    gradient();
    launch_block_norm_sum(G_.get(), offs_dev_.get(), N, partials_.get(), scal_.get() + kNormSum, 1.0, ctx_.stream);
    CPK_CUDA(cudaMemcpyAsync(hpin_, scal_.get() + kRes, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx_.stream));
    CPK_CUDA(cudaMemcpyAsync(hpin_ + 2, scal_.get() + kNormSum, sizeof(double), cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync_main();
    const double res = hpin_[0];
    diag.residual_before = res;
    diag.residual_after = res;
    if (res < cfg.residual_tol) {
        diag.halt = GnStepDiag::Halt::residual;
        ctx_.sync();
        precond_pending_ = false;
        return diag;
    }
    diag.grad_norm = hpin_[2];
    if (diag.grad_norm <= cfg.grad_tol) {
        diag.halt = GnStepDiag::Halt::gradient;
        ctx_.sync();
        precond_pending_ = false;
        return diag;
    }
    diag.lambda = schedule.lambda;
    const CgResultInfo cg = cp_cg(diag.lambda, cfg, diag.grad_norm);
    diag.cg_iters = cg.iterations;
    diag.cg_hit_cap = cg.hit_cap;
    diag.cg_breakdown = cg.breakdown;

    double alpha = 1.0;
    double residual_after = -1.0;
    if (cfg.armijo) {
        const ArmijoParams& ap = *cfg.armijo;
        const double f0 = 0.5 * res * res * xnorm2;
        launch_dot(G_.get(), V_.get(), S, partials_.get(), scal_.get() + kDot, ctx_.stream);
        const double gv = read_scalar(kDot);
        // keep the pre-step factors in Atrial_; A_ holds the trial point
        CPK_CUDA(cudaMemcpyAsync(Atrial_.get(), A_.get(), S * sizeof(double), cudaMemcpyDeviceToDevice, ctx_.stream));
        auto eval_trial = [&](double a) {
            launch_axpby(A_.get(), Atrial_.get(), a, V_.get(), S, ctx_.stream);
            invalidate_all();
            mttkrp_naive(N - 1);
            grams_all();
            return residual_fitness(xnorm2, N - 1).first;
        };
        bool accepted = false;
        for (int t = 0; t < ap.max_backtracks; ++t) {
            const double r_trial = eval_trial(alpha);
            const double f_trial = 0.5 * r_trial * r_trial * xnorm2;
            if (f_trial <= f0 + ap.c1 * alpha * gv) {
                accepted = true;
                residual_after = r_trial;
                break;
            }
            alpha *= ap.shrink;
        }
        if (!accepted) {
            diag.armijo_exhausted = true;
            residual_after = eval_trial(alpha);
        }
    } else {
        launch_axpy(A_.get(), V_.get(), 1.0, S, ctx_.stream);
    }
    diag.alpha = alpha;
    // step norm and the finiteness flag in one readback
    launch_block_norm_sum(V_.get(), offs_dev_.get(), N, partials_.get(), scal_.get() + kNormSum, alpha,
                          ctx_.stream);
    invalidate_all();
    launch_set_flag_scalar(flag_.get(), 1, scal_.get() + kStep, 0.0, ctx_.stream);
    launch_all_finite(A_.get(), S, flag_.get(), ctx_.stream);
    int* fin_pin = reinterpret_cast<int*>(hpin_ + 4);
    CPK_CUDA(cudaMemcpyAsync(hpin_ + 3, scal_.get() + kNormSum, sizeof(double), cudaMemcpyDeviceToHost, ctx_.stream));
    CPK_CUDA(cudaMemcpyAsync(fin_pin, flag_.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx_.stream));
    ctx_.sync();
    diag.step_norm = hpin_[3];
    if (!*fin_pin) throw NumericalFailure("gn_step: non-finite factors after update");
    if (residual_after < 0.0) {
        if (ref_residual(cfg)) mttkrp_naive(N - 1);
        else compute_all_mttkrp();
        grams_all();
        residual_after = residual_fitness(xnorm2, N - 1).first;
    }
    diag.residual_after = residual_after;
    diag.stepped = true;
    schedule = schedule_next(schedule);
    return diag;
}

// ================================================================ drivers
std::pair<KruskalModel, ConvergenceReport> als_optimize(DeviceProblem& p, KruskalModel model,
                                                        const AlsConfig& cfg) {  // als.cpp:54-94
    cfg.validate();
    model.validate();
    p.set_factors(model);
    const double xnorm2 = p.norm2();  // also leaves ||X||^2 in its device slot for the residuals
    if (!(xnorm2 > 0.0)) throw InvalidArgument("als_optimize: tensor norm must be positive");
    ConvergenceReport report;
    report.status = TerminalStatus::cap_hit;
    auto lambda_of = [&](int sweep) {
        double lambda = cfg.lambda0;
        if (cfg.decay_every)
            lambda /= std::pow(cfg.decay_factor, static_cast<double>((sweep - 1) / *cfg.decay_every));
        return lambda;
    };
    // B200 change: sweep k+1 is queued before the host reads sweep k's step
    // norm and residual, so the per-sweep host round trip overlaps device
    // work. When sweep k stops the run, the speculative sweep is drained and
    // the factors restored from the copy taken before it (same result as the
    // reference's sequential loop; the caches are rebuilt on demand).
    const bool pipeline = !std::getenv("CPKIT_ALS_NO_PIPELINE");
    auto drain = [&] {
        while (p.als_sweeps_pending() > 0) {
            try {
                p.als_sweep_finish();
            } catch (...) {  // a discarded speculative sweep's failure is not the run's
            }
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (cfg.max_sweeps >= 1) p.als_sweep_launch(lambda_of(1), true);
    for (int sweep = 1; sweep <= cfg.max_sweeps; ++sweep) {
        const double lambda = lambda_of(sweep);
        const bool spec = pipeline && sweep < cfg.max_sweeps;
        if (spec) {
            p.als_snapshot_factors();
            p.als_sweep_launch(lambda_of(sweep + 1), true);
        }
        double res = 1.0, fit = 0.0;
        AlsSweepDiag diag;
        try {
            diag = p.als_sweep_finish(&res, &fit);
        } catch (...) {
            drain();
            throw;
        }
        const double seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        report.records.push_back({sweep, res, fit, lambda, 0, seconds});
        bool stop = false;
        if (res < cfg.residual_tol) {
            report.status = TerminalStatus::converged_residual;
            stop = true;
        } else if (diag.step_norm < cfg.step_tol) {
            report.status = TerminalStatus::converged_step;
            stop = true;
        }
        if (stop) {
            if (spec) {
                drain();
                p.als_restore_factors();
            }
            break;
        }
        if (!spec && sweep < cfg.max_sweeps) p.als_sweep_launch(lambda_of(sweep + 1), true);
    }
    p.get_factors(model);
    return {std::move(model), std::move(report)};
}

std::pair<KruskalModel, ConvergenceReport> gn_optimize(DeviceProblem& p, KruskalModel model,
                                                       const GnConfig& cfg) {  // gauss_newton.cpp:451-494
    cfg.validate();
    model.validate();
    p.set_factors(model);
    const double xnorm2 = p.norm2();
    if (!(xnorm2 > 0.0)) throw InvalidArgument("gn_optimize: tensor norm must be positive");
    ConvergenceReport report;
    report.status = TerminalStatus::cap_hit;
    RegSchedule schedule = cfg.schedule;
    const auto t0 = std::chrono::steady_clock::now();
    // B200 change (default steps, no Armijo): step k+1 is queued before the host
    // reads step k (the lambda schedule is deterministic), hiding the per-step
    // host round trip. When step k stops the run, the queued step is undone
    // from its own pre-step snapshot (or step k from its snapshot when k itself
    // must not have happened); records and factors are those of the sequential
    // loop (CPKIT_GN_NO_PIPELINE=1 runs it).
    const bool pipeline = !cfg.armijo && !std::getenv("CPKIT_GN_SYNC") && !std::getenv("CPKIT_GN_NO_PIPELINE");
    if (pipeline) {
        int slot = 0;
        p.gn_enqueue(cfg, schedule, xnorm2, slot);
        for (int iter = 1; iter <= cfg.max_iters; ++iter) {
            const RegSchedule next = schedule_next(schedule);
            const bool spec = iter < cfg.max_iters;
            if (spec) p.gn_enqueue(cfg, next, xnorm2, slot ^ 1);
            GnStepDiag diag;
            try {
                diag = p.gn_decode(cfg, schedule.lambda, slot);  // undoes step iter itself when it must
            } catch (...) {
                // step iter applied a non-finite update and step iter+1 ran on top of
                // it: leave the factors the sequential loop leaves (after step iter)
                if (spec && p.gn_failed_applied()) p.restore_factors_from(p.gn_snapshot(slot ^ 1));
                p.ctx().sync();
                throw;
            }
            bool stop = false;
            if (diag.halt == GnStepDiag::Halt::residual) {
                report.status = TerminalStatus::converged_residual;
                stop = true;
            } else if (diag.halt == GnStepDiag::Halt::gradient) {
                report.status = TerminalStatus::converged_step;
                stop = true;
            } else {
                const double seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                report.records.push_back({iter, diag.residual_after, 1.0 - diag.residual_after, diag.lambda,
                                          diag.cg_iters, seconds});
                if (diag.residual_after < cfg.residual_tol) {
                    report.status = TerminalStatus::converged_residual;
                    stop = true;
                } else if (diag.step_norm < cfg.step_tol) {
                    report.status = TerminalStatus::converged_step;
                    stop = true;
                }
                if (stop && spec) p.restore_factors_from(p.gn_snapshot(slot ^ 1));  // drop the queued step
            }
            if (stop) {
                p.ctx().sync();
                break;
            }
            schedule = next;
            slot ^= 1;
        }
        p.get_factors(model);
        return {std::move(model), std::move(report)};
    }
    for (int iter = 1; iter <= cfg.max_iters; ++iter) {
        GnStepDiag diag = p.gn_step(cfg, schedule, xnorm2);
        if (diag.halt == GnStepDiag::Halt::residual) {
            report.status = TerminalStatus::converged_residual;
            break;
        }
        if (diag.halt == GnStepDiag::Halt::gradient) {
            report.status = TerminalStatus::converged_step;
            break;
        }
        const double seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        report.records.push_back({iter, diag.residual_after, 1.0 - diag.residual_after, diag.lambda,
                                  diag.cg_iters, seconds});
        if (diag.residual_after < cfg.residual_tol) {
            report.status = TerminalStatus::converged_residual;
            break;
        }
        if (diag.step_norm < cfg.step_tol) {
            report.status = TerminalStatus::converged_step;
            break;
        }
    }
    p.get_factors(model);
    return {std::move(model), std::move(report)};
}

}  // namespace cpkit
