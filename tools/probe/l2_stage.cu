// Probe: time for one CTA to stage `kb` KB from L2 into shared memory with
// cp.async (16 B), as a function of how many CTAs do it concurrently.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__device__ __forceinline__ void cp16(void* dst, const void* src) {
    unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void ldg_batch(double* dst, const double* src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcg(src + i);
}

extern __shared__ double sm[];
__global__ void stage(const double* src, long long stride_per_cta, int n, int reps, unsigned long long* out, int mode) {
    const double* s = src + blockIdx.x * stride_per_cta;
    unsigned long long t0, t1;
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < reps; ++r) {
        if (mode == 0) {
            for (int i = threadIdx.x * 2; i < n; i += blockDim.x * 2) cp16(sm + i, s + i);
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        } else {
            ldg_batch(sm, s, n);
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    const int maxg = 296;
    const long long per = 1 << 16;  // doubles per CTA region (512 KB)
    double* src;
    unsigned long long* out;
    cudaMalloc(&src, maxg * per * 8);
    cudaMemset(src, 0, maxg * per * 8);
    cudaMalloc(&out, maxg * 8);
    cudaFuncSetAttribute(stage, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    std::vector<unsigned long long> h(maxg);
    for (int mode = 0; mode < 2; ++mode)
        for (int kb : {25, 50, 100}) {
            const int n = kb * 1024 / 8;
            for (int g : {1, 8, 74, 148, 296}) {
                for (int shared = 0; shared < 2; ++shared) {
                    const long long stride = shared ? 0 : per;
                    stage<<<g, 256, 110 * 1024>>>(src, stride, n, 4, out, mode);
                    stage<<<g, 256, 110 * 1024>>>(src, stride, n, 20, out, mode);
                    cudaDeviceSynchronize();
                    cudaMemcpy(h.data(), out, g * 8, cudaMemcpyDeviceToHost);
                    std::sort(h.begin(), h.begin() + g);
                    printf("%s kb=%3d grid=%3d %s  per-stage median %.2f us  max %.2f us  (%.1f GB/s/CTA)\n",
                           mode ? "ldcg " : "cpasy", kb, g, shared ? "same-src" : "own-src ", h[g / 2] / 20e3,
                           h[g - 1] / 20e3, kb * 1024.0 / (h[g / 2] / 20.0));
                }
            }
        }
    return 0;
}
