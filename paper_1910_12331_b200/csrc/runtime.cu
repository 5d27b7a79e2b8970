// Process-level runtime pieces: kernel-launch accounting, the NCCL
// communicator used for last-mode sharding, and the FP64 DMMA peak probe.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <utility>
#include <vector>

#include "solver.h"

namespace cpkit {

// ---------------------------------------------------------------- launch counter
namespace {
std::atomic<std::uint64_t> g_launches{0};
}
// ---- guarded allocation mode (common.h)
namespace {
std::atomic<std::uint64_t> g_guard_violations{0};
bool guard_zone_ok(const unsigned char* dev, const char* which, std::size_t bytes) {
    std::vector<unsigned char> h(kGuardBytes);
    if (cudaMemcpy(h.data(), dev, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return true;  // sticky fault: reported elsewhere
    for (std::size_t i = 0; i < kGuardBytes; ++i)
        if (h[i] != kGuardByte) {
            std::fprintf(stderr, "cpkit guard: %s red zone of a %zu-byte buffer changed at byte %zu\n", which, bytes, i);
            return false;
        }
    return true;
}
}  // namespace
bool guard_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CPKIT_GUARD");
        return e && e[0] && e[0] != '0';
    }();
    return on;
}
void* guard_alloc(std::size_t bytes) {
    const std::size_t body = (bytes + 255) & ~static_cast<std::size_t>(255);  // keep 256-B alignment of the tail zone
    unsigned char* base = nullptr;
    CPK_CUDA(cudaMalloc(&base, body + 2 * kGuardBytes));
    CPK_CUDA(cudaMemset(base, kGuardByte, kGuardBytes));
    CPK_CUDA(cudaMemset(base + kGuardBytes + bytes, kGuardByte, body - bytes + kGuardBytes));
    return base + kGuardBytes;
}
std::recursive_mutex& guard_capture_mutex() {
    static std::recursive_mutex mu;
    return mu;
}
void guard_free(void* user, std::size_t bytes) {
    unsigned char* u = static_cast<unsigned char*>(user);
    unsigned char* base = u - kGuardBytes;
    std::lock_guard<std::recursive_mutex> lock(guard_capture_mutex());  // no graph capture in progress anywhere
    cudaDeviceSynchronize();  // every stream's writes landed
    const bool ok_front = guard_zone_ok(base, "front", bytes);
    const bool ok_back = guard_zone_ok(u + bytes, "back", bytes);
    if (!ok_front || !ok_back) g_guard_violations.fetch_add(1);
    cudaFree(base);
}
std::uint64_t guard_violations() { return g_guard_violations.load(); }
namespace {
bool alloc_trace() {
    static const bool on = std::getenv("CPKIT_ALLOC_TRACE") != nullptr;
    return on;
}
bool alloc_cache_on() {
    static const bool on = std::getenv("CPKIT_NO_ALLOC_CACHE") == nullptr;
    return on;
}
thread_local int t_owner_synced = 0;
std::mutex g_cache_mu;
std::map<int, std::multimap<std::size_t, void*>> g_cache;  // device -> (bytes, block)
void traced(const char* what, std::size_t bytes, std::chrono::steady_clock::time_point t0) {
    if (!alloc_trace()) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 2.0) std::fprintf(stderr, "cpkit %s %zu bytes: %.1f ms\n", what, bytes, ms);
}
void cache_empty_device(int dev) {  // caller holds g_cache_mu
    auto it = g_cache.find(dev);
    if (it == g_cache.end()) return;
    for (auto& kv : it->second) cudaFree(kv.second);
    it->second.clear();
}
}  // namespace
OwnerSyncedRelease::OwnerSyncedRelease() { ++t_owner_synced; }
OwnerSyncedRelease::~OwnerSyncedRelease() { --t_owner_synced; }
void* dev_alloc(std::size_t bytes) {
    int dev = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    if (alloc_cache_on()) {
        std::lock_guard<std::mutex> lock(g_cache_mu);
        auto& c = g_cache[dev];
        auto it = c.find(bytes);
        if (it != c.end()) {
            void* p = it->second;
            c.erase(it);
            return p;
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();  // not sticky: give the cached blocks back and retry once
        {
            std::lock_guard<std::mutex> lock(g_cache_mu);
            cache_empty_device(dev);
        }
        e = cudaMalloc(&p, bytes);
    }
    CPK_CUDA(e);
    traced("alloc", bytes, t0);
    return p;
}
void dev_free(void* p, std::size_t bytes) {
    if (t_owner_synced > 0 && alloc_cache_on()) {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) {
            std::lock_guard<std::mutex> lock(g_cache_mu);
            g_cache[dev].emplace(bytes, p);
            return;
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    cudaFree(p);
    traced("free", bytes, t0);
}
namespace {
std::mutex g_pin_mu;
std::multimap<std::pair<std::size_t, bool>, void*> g_pin_free;
}  // namespace
void* pinned_small_alloc(std::size_t bytes, bool mapped) {
    {
        std::lock_guard<std::mutex> lock(g_pin_mu);
        auto it = g_pin_free.find({bytes, mapped});
        if (it != g_pin_free.end()) {
            void* p = it->second;
            g_pin_free.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    CPK_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable | (mapped ? cudaHostAllocMapped : 0u)));
    return p;
}
void pinned_small_free(void* p, std::size_t bytes, bool mapped) {
    if (!p) return;
    std::lock_guard<std::mutex> lock(g_pin_mu);
    g_pin_free.emplace(std::make_pair(bytes, mapped), p);
}
std::size_t dev_cache_bytes() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lock(g_cache_mu);
    std::size_t b = 0;
    auto it = g_cache.find(dev);
    if (it != g_cache.end())
        for (auto& kv : it->second) b += kv.first;
    return b;
}
void dev_cache_empty() {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : g_cache) {
        cudaSetDevice(kv.first);
        cache_empty_device(kv.first);
    }
    cudaSetDevice(cur);
}
namespace {
__global__ void guard_poke_kernel(double* p, long long i) { p[i] = 1.0; }
}  // namespace
// Positive control: write one element past the end of a guarded buffer and
// one before its start; both must be counted.
bool guard_selftest() {
    if (!guard_enabled()) throw InvalidArgument("guard self-test needs CPKIT_GUARD=1");
    const std::uint64_t before = guard_violations();
    {
        DevBuf<double> b(1000);
        guard_poke_kernel<<<1, 1>>>(b.get(), 1000);
        CPK_CUDA(cudaGetLastError());
        count_launch(1);
    }
    {
        DevBuf<double> b(7);
        guard_poke_kernel<<<1, 1>>>(b.get(), -1);
        CPK_CUDA(cudaGetLastError());
        count_launch(1);
    }
    {
        DevBuf<double> b(1000);  // in bounds: no report
        guard_poke_kernel<<<1, 1>>>(b.get(), 999);
        CPK_CUDA(cudaGetLastError());
        count_launch(1);
    }
    return guard_violations() - before == 2;
}

void count_launch(int n) { g_launches.fetch_add(static_cast<std::uint64_t>(n), std::memory_order_relaxed); }
std::uint64_t kernel_launches() { return g_launches.load(); }

// ---------------------------------------------------------------- launch attributes
namespace {
std::mutex g_attr_mu;
std::map<int, int> g_sms;                                   // device -> SM count
std::map<std::pair<int, const void*>, std::size_t> g_smem;  // (device, kernel) -> limit set
}  // namespace
int device_sm_count() {
    int dev = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_attr_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int sms = 0;
    CPK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    g_sms[dev] = sms;
    return sms;
}
namespace {
std::mutex g_coop_mu;
std::map<int, cudaEvent_t> g_coop_tail;  // device -> completion of its last cooperative launch
}  // namespace
void launch_cooperative(const void* fn, dim3 grid, dim3 block, void** args, std::size_t smem, cudaStream_t st) {
    int dev = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_coop_mu);
    cudaEvent_t& tail = g_coop_tail[dev];
    if (!tail) CPK_CUDA(cudaEventCreateWithFlags(&tail, cudaEventDisableTiming));
    else CPK_CUDA(cudaStreamWaitEvent(st, tail, 0));  // no-op when the last one was on this stream
    CPK_CUDA(cudaLaunchCooperativeKernel(fn, grid, block, args, smem, st));
    CPK_CUDA(cudaEventRecord(tail, st));
}
void launch_cooperative_cluster(const void* fn, dim3 grid, dim3 block, unsigned cluster_x, void** args,
                                std::size_t smem, cudaStream_t st) {
    int dev = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_coop_mu);
    cudaEvent_t& tail = g_coop_tail[dev];
    if (!tail) CPK_CUDA(cudaEventCreateWithFlags(&tail, cudaEventDisableTiming));
    else CPK_CUDA(cudaStreamWaitEvent(st, tail, 0));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_x;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    CPK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    CPK_CUDA(cudaEventRecord(tail, st));
}
int max_active_clusters(const void* fn, dim3 block, unsigned cluster_x, std::size_t smem) {
    int dev = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, unsigned, unsigned, std::size_t>, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(dev, fn, block.x, cluster_x, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cluster_x * 148);
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_x;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[key] = n;
    return n;
}
void ensure_dynamic_smem(const void* fn, std::size_t bytes) {
    int dev = 0;
    CPK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_attr_mu);
    std::size_t& cur = g_smem[{dev, fn}];
    if (cur >= bytes) return;
    CPK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    cur = bytes;
}

// ---------------------------------------------------------------- NCCL (dlopen'd)
// The library links no NCCL at build time; the sharded path resolves the
// handful of symbols it needs from libnccl.so.2 (torch's copy when torch is
// already loaded in the process, else the system one).
namespace {
using ncclComm_t = void*;
struct NcclUniqueId {
    char internal[128];
};
enum NcclDataType { kNcclFloat64 = 8 };
enum NcclRedOp { kNcclSum = 0 };
struct NcclApi {
    int (*GetUniqueId)(NcclUniqueId*) = nullptr;
    int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*AllReduce)(const void*, void*, std::size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*AllGather)(const void*, void*, std::size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.GetUniqueId = reinterpret_cast<int (*)(NcclUniqueId*)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<int (*)(ncclComm_t*, int, NcclUniqueId, int)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<int (*)(ncclComm_t)>(dlsym(h, "ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<int (*)(const void*, void*, std::size_t, int, int, ncclComm_t, cudaStream_t)>(
            dlsym(h, "ncclAllReduce"));
        api.AllGather = reinterpret_cast<int (*)(const void*, void*, std::size_t, int, ncclComm_t, cudaStream_t)>(
            dlsym(h, "ncclAllGather"));
        api.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather)
        throw DeviceError("NCCL (libnccl.so.2) not available for the sharded path");
    return api;
}
void nccl_check(int rc, const char* what) {
    if (rc != 0) {
        const char* msg = nccl().GetErrorString ? nccl().GetErrorString(rc) : "?";
        throw DeviceError(std::string("NCCL ") + what + " failed: " + msg);
    }
}

class NcclComm final : public Comm {
public:
    NcclComm(const void* id, int rank, int world) : rank_(rank), world_(world) {
        NcclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof uid.internal);
        nccl_check(nccl().CommInitRank(&comm_, world, uid, rank), "CommInitRank");
    }
    ~NcclComm() override {
        if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
    }
    int rank() const override { return rank_; }
    int world() const override { return world_; }
    void allreduce_sum(double* dev, std::size_t count, cudaStream_t st) override {
        nccl_check(nccl().AllReduce(dev, dev, count, kNcclFloat64, kNcclSum, comm_, st), "AllReduce");
    }
    void allgather(const double* in, double* out, std::size_t per, cudaStream_t st) override {
        nccl_check(nccl().AllGather(in, out, per, kNcclFloat64, comm_, st), "AllGather");
    }

private:
    ncclComm_t comm_ = nullptr;
    int rank_, world_;
};
}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int world) {
    return std::make_unique<NcclComm>(unique_id, rank, world);
}
void nccl_unique_id(void* out128) {
    NcclUniqueId uid;
    nccl_check(nccl().GetUniqueId(&uid), "GetUniqueId");
    std::memcpy(out128, uid.internal, sizeof uid.internal);
}

// ---------------------------------------------------------------- loopback group
// Test-only collectives for `world` last-mode shards on ONE device, each shard
// driven by its own host thread: the NCCL call sequence of the sharded path
// runs unchanged, with the data movement done as device copies and a
// fixed-order (rank 0, 1, ...) sum. Every rank posts its buffer and an event
// on its stream, meets the others on the host, rank 0's thread enqueues the
// exchange behind all the events, and every stream waits for its completion.
namespace {
constexpr int kLoopMax = 16;
struct RankPtrs {
    const double* p[kLoopMax];
};
__global__ void loopback_sum_kernel(RankPtrs src, int world, double* __restrict__ dst, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        double a = src.p[0][i];
        for (int q = 1; q < world; ++q) a = __dadd_rn(a, src.p[q][i]);
        dst[i] = a;
    }
}

class LoopbackGroup {
public:
    explicit LoopbackGroup(int world) : world_(world), in_(world), out_(world), ready_(world) {
        if (world < 1 || world > kLoopMax) throw InvalidArgument("loopback group: 1..16 shards");
        for (auto& e : ready_) CPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CPK_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    }
    ~LoopbackGroup() {
        for (auto& e : ready_) cudaEventDestroy(e);
        cudaEventDestroy(done_);
    }
    int world() const { return world_; }
    // kind 0: in-place sum of `count` doubles; kind 1: gather `count` doubles per rank
    void collective(int rank, int kind, const double* in, double* out, std::size_t count, cudaStream_t st) {
        CPK_CUDA(cudaEventRecord(ready_[rank], st));
        in_[rank] = in;
        out_[rank] = out;
        meet();  // every rank has posted its buffers and its ready event
        if (rank == 0) {
            for (int q = 0; q < world_; ++q) CPK_CUDA(cudaStreamWaitEvent(st, ready_[q], 0));
            if (kind == 0) {
                tmp_.ensure(count);
                RankPtrs src{};
                for (int q = 0; q < world_; ++q) src.p[q] = in_[q];
                const unsigned blocks = static_cast<unsigned>(std::min<std::size_t>((count + 255) / 256, 1184));
                if (count) {
                    loopback_sum_kernel<<<blocks, 256, 0, st>>>(src, world_, tmp_.get(), count);
                    count_launch(1);
                    CPK_CUDA(cudaGetLastError());
                }
                for (int q = 0; q < world_; ++q)
                    CPK_CUDA(cudaMemcpyAsync(out_[q], tmp_.get(), count * sizeof(double), cudaMemcpyDeviceToDevice, st));
            } else {
                for (int d = 0; d < world_; ++d)
                    for (int q = 0; q < world_; ++q) {
                        double* dst = out_[d] + static_cast<std::size_t>(q) * count;
                        if (dst != in_[q])
                            CPK_CUDA(cudaMemcpyAsync(dst, in_[q], count * sizeof(double), cudaMemcpyDeviceToDevice, st));
                    }
            }
            CPK_CUDA(cudaEventRecord(done_, st));
        }
        meet();  // the exchange is enqueued
        if (rank != 0) CPK_CUDA(cudaStreamWaitEvent(st, done_, 0));
        meet();  // everyone waits on this round's done event before the next round re-records it
    }

private:
    void meet() {
        std::unique_lock<std::mutex> lock(mu_);
        const unsigned gen = gen_;
        if (++arrived_ == world_) {
            arrived_ = 0;
            ++gen_;
            cv_.notify_all();
            return;
        }
        if (!cv_.wait_for(lock, std::chrono::seconds(300), [&] { return gen_ != gen; }))
            throw DeviceError("loopback collective: a shard did not arrive within 300 s");
    }
    int world_;
    std::vector<const double*> in_;
    std::vector<double*> out_;
    std::vector<cudaEvent_t> ready_;
    cudaEvent_t done_ = nullptr;
    DevBuf<double> tmp_;
    std::mutex mu_;
    std::condition_variable cv_;
    int arrived_ = 0;
    unsigned gen_ = 0;
};

class LoopbackComm final : public Comm {
public:
    LoopbackComm(std::shared_ptr<LoopbackGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
    int rank() const override { return rank_; }
    int world() const override { return g_->world(); }
    void allreduce_sum(double* dev, std::size_t count, cudaStream_t st) override {
        g_->collective(rank_, 0, dev, dev, count, st);
    }
    void allgather(const double* in, double* out, std::size_t per, cudaStream_t st) override {
        g_->collective(rank_, 1, in, out, per, st);
    }

private:
    std::shared_ptr<LoopbackGroup> g_;
    int rank_;
};
}  // namespace

std::vector<std::unique_ptr<Comm>> make_loopback_comms(int world) {
    auto g = std::make_shared<LoopbackGroup>(world);
    std::vector<std::unique_ptr<Comm>> out;
    for (int r = 0; r < world; ++r) out.push_back(std::make_unique<LoopbackComm>(g, r));
    return out;
}

// ---------------------------------------------------------------- DMMA peak probe
namespace {
__global__ void dmma_probe_kernel(double* out, int iters) {
    double acc[8][4];
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) b[i] = 1.0 + blockIdx.x * 1e-6;
    for (int c = 0; c < 8; ++c)
        for (int j = 0; j < 4; ++j) acc[c][j] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},"
                "{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};"
                : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                  "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0.0;
    for (int c = 0; c < 8; ++c)
        for (int j = 0; j < 4; ++j) s += acc[c][j];
    if (s == 123.456) out[0] = s;
}
}  // namespace

double probe_dmma_peak(int device) {
    CPK_CUDA(cudaSetDevice(device));
    int sms = 0;
    CPK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DevBuf<double> out(1);
    const int blocks = sms * 2, threads = 256, iters = 4000;
    cudaEvent_t a, b;
    CPK_CUDA(cudaEventCreate(&a));
    CPK_CUDA(cudaEventCreate(&b));
    dmma_probe_kernel<<<blocks, threads>>>(out.get(), iters);  // warm-up
    count_launch(1);
    CPK_CUDA(cudaGetLastError());
    CPK_CUDA(cudaEventRecord(a));
    for (int r = 0; r < 3; ++r) {
        dmma_probe_kernel<<<blocks, threads>>>(out.get(), iters);
        count_launch(1);
    }
    CPK_CUDA(cudaEventRecord(b));
    CPK_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    CPK_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 3.0 * blocks * (threads / 32) * static_cast<double>(iters) * 8 * 2.0 * 16 * 8 * 16;
    return flops / (ms * 1e-3) / 1e12;
}

}  // namespace cpkit
