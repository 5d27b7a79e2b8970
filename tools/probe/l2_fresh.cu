// Probe 3: does reading data that other SMs wrote a moment ago (same kernel,
// after a grid barrier) cost more than reading long-resident L2 data?
// Each CTA writes a 52 KB region; grid barrier; each CTA cp.asyncs the region
// of CTA (b + 37) % grid. Mode 0: region written in this kernel; mode 1: no
// write (data resident from an earlier kernel).
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(dst)), "l"(src) : "memory");
}
__device__ void grid_bar(unsigned* bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned seen;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory"); } while (seen < target);
    }
    __syncthreads();
}
extern __shared__ __align__(16) double sm[];
__global__ void k(double* buf, int n, unsigned* bar, int mode, int reps, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int rep = 0; rep < reps; ++rep) {
        double* mine = buf + (long long)blockIdx.x * n;
        if (mode == 0)
            for (int i = threadIdx.x * 2; i < n; i += blockDim.x * 2)
                *reinterpret_cast<double2*>(mine + i) = make_double2(rep, i);
        grid_bar(bar, (2 * rep + 1) * gridDim.x);
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        const double* src = buf + (long long)((blockIdx.x + 37) % gridDim.x) * n;
        for (int i = threadIdx.x * 2; i < n; i += blockDim.x * 2) cp16(sm + i, src + i);
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        acc += t1 - t0;
        grid_bar(bar, (2 * rep + 2) * gridDim.x);
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc / reps;
}
int main() {
    const int n = 52 * 1024 / 8;
    double* buf; unsigned* bar; unsigned long long* out;
    cudaMalloc(&buf, 148ll * n * 8); cudaMemset(buf, 0, 148ll * n * 8);
    cudaMalloc(&bar, 4); cudaMalloc(&out, 148 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
    std::vector<unsigned long long> h(148);
    for (int threads : {256, 384})
        for (int mode = 0; mode < 2; ++mode) {
            cudaMemset(bar, 0, 4);
            void* args[] = {&buf, (void*)&n, &bar, &mode, nullptr, &out};
            int reps = 50; args[4] = &reps;
            cudaLaunchCooperativeKernel((void*)k, 148, threads, args, 60 * 1024, 0);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            printf("threads=%d %s: 52 KB stage median %.2f us max %.2f us\n", threads, mode ? "resident " : "fresh    ", h[74] / 1e3, h[147] / 1e3);
        }
    return 0;
}
