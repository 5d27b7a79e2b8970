// Probe 2: staging a 32x200 row-major panel + a 200x32 k-major panel (R = 100
// row stride) into shared memory: (a) cp.async 16 B, 2-D thread mapping;
// (b) cp.async.bulk, one copy per row; timed per CTA with globaltimer.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(dst)), "l"(src) : "memory");
}
extern __shared__ __align__(16) double sm[];
__global__ void stage(const double* W, const double* A, const double* G, int R, int reps, int mode,
                      unsigned long long* out, int spread) {
    __shared__ unsigned long long bar;
    const int task = blockIdx.x % spread;
    const double* w = W + (long long)task * 32 * R;
    const double* a = A + (long long)task * 32 * R;
    double* As = sm;
    double* Bs = sm + 32 * 204;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    __syncthreads();
    unsigned parity = 0;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int rep = 0; rep < reps; ++rep) {
        if (mode == 0) {
            // row-major A: row = tid>>3, 8 threads per row, 100 chunks per row (200 doubles)
            const int row = threadIdx.x >> 3;
            for (int ch = threadIdx.x & 7; ch < 100; ch += 8) {
                const int c = 2 * ch;
                const double* src = c < R ? w + row * R + c : a + row * R + (c - R);
                cp16(As + row * 204 + c, src);
            }
            // k-major B: 200 rows x 16 chunks
            for (int k = threadIdx.x >> 4; k < 200; k += 16) {
                const double* src = (k < R ? G + k * R : G + R * R + (k - R) * R) + 2 * (threadIdx.x & 15);
                cp16(Bs + k * 36 + 2 * (threadIdx.x & 15), src);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        } else {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int r = threadIdx.x;
            if (r < 32) {
                asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1600));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(As + r * 204)), "l"(w + r * R), "r"(800), "r"(su(&bar)) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(As + r * 204 + R)), "l"(a + r * R), "r"(800), "r"(su(&bar)) : "memory");
            }
            if (r < 200) {
                const double* src = r < R ? G + r * R : G + R * R + (r - R) * R;
                asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(256));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(Bs + r * 36)), "l"(src), "r"(256), "r"(su(&bar)) : "memory");
            }
            __syncthreads();
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
            for (;;) {
                unsigned ok;
                asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su(&bar)), "r"(parity) : "memory");
                if (ok) break;
            }
            parity ^= 1;
            __syncthreads();
        }
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    const int R = 100, S = 1200;
    double *W, *A, *G;
    unsigned long long* out;
    cudaMalloc(&W, S * R * 8); cudaMalloc(&A, S * R * 8); cudaMalloc(&G, 2 * R * R * 8);
    cudaMemset(W, 0, S * R * 8); cudaMemset(A, 0, S * R * 8); cudaMemset(G, 0, 2 * R * R * 8);
    cudaMalloc(&out, 512 * 8);
    const int smem = (32 * 204 + 200 * 36) * 8;
    cudaFuncSetAttribute(stage, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<unsigned long long> h(512);
    for (int mode = 0; mode < 2; ++mode)
        for (int g : {1, 148, 156, 296}) {
            stage<<<g, 256, smem>>>(W, A, G, R, 4, mode, out, 37);
            stage<<<g, 256, smem>>>(W, A, G, R, 20, mode, out, 37);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(h.data(), out, g * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.begin() + g);
            printf("%s grid=%3d per-stage median %.2f us max %.2f us\n", mode ? "bulk " : "cpasy", g, h[g / 2] / 20e3, h[g - 1] / 20e3);
        }
    return 0;
}
