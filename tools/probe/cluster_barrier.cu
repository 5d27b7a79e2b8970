// Probe: latency of a thread-block-cluster barrier (barrier.cluster arrive.release
// + wait.acquire) for cluster sizes 2..16, and of a DSMEM round trip, on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void cluster_bar(int iters, unsigned long long* out) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}
__global__ void dsmem_rt(int iters, unsigned long long* out) {
    __shared__ double buf[64];
    buf[threadIdx.x & 63] = threadIdx.x;
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    unsigned nr;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nr));
    unsigned local = static_cast<unsigned>(__cvta_generic_to_shared(buf));
    unsigned remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"((rank + 1) % nr));
    double acc = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double v;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote + 8u * (static_cast<unsigned>(acc) & 7u)) : "memory");
        acc += v * 1e-300;
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters + (acc > 1 ? 1 : 0);
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(dsmem_rt, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {2, 4, 8, 16}) {
        for (int threads : {128, 512}) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(threads);
            cudaLaunchAttribute a[1];
            a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = cs;
            a[0].val.clusterDim.y = 1;
            a[0].val.clusterDim.z = 1;
            cfg.attrs = a;
            cfg.numAttrs = 1;
            int iters = 10000;
            cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_bar, iters, d);
            cudaDeviceSynchronize();
            unsigned long long h = 0;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            unsigned long long h2 = 0;
            if (threads == 128) {
                cudaLaunchKernelEx(&cfg, dsmem_rt, 10000, d);
                cudaDeviceSynchronize();
                cudaMemcpy(&h2, d, 8, cudaMemcpyDeviceToHost);
            }
            printf("cluster %2d threads %3d: barrier %llu cycles (%s)  dsmem dependent load %llu cycles\n", cs, threads, h,
                   cudaGetErrorString(e), h2);
        }
    }
    return 0;
}
