// Probe: cycles per column of the warp-synchronous 16x16 diagonal factor.
#include <cstdio>
#include <cuda_runtime.h>
template <int kNB, int kMode>
__device__ __noinline__ bool dfac(double* w, int LD, int R, int k0, int kb) {
    const int i = threadIdx.x & 31;
    double r[kNB];
#pragma unroll
    for (int m = 0; m < kNB; ++m) r[m] = (i < kb && m <= i) ? w[(k0 + i) * LD + k0 + m] : 0.0;
    bool failed = false;
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
        const double x = __shfl_sync(0xffffffffu, r[j], j);
        if (j < kb && !failed && !(x > 0.0) && !isnan(x)) failed = true;
        const bool go = j < kb && !failed;
        double inv, l;
        if (kMode == 0) { inv = rsqrt(x); l = x * inv; }
        else if (kMode == 1) { l = sqrt(x); inv = 1.0 / l; }
        else { inv = __drcp_rn(__dsqrt_rn(x)); l = __dsqrt_rn(x); }
        if (go && i > j) r[j] *= inv;
        if (go && i == j) { r[j] = l; w[(k0 + j) * LD + R] = inv; }
#pragma unroll
        for (int m = j + 1; m < kNB; ++m) {
            const double lmj = __shfl_sync(0xffffffffu, r[j], m);
            if (go && i >= m) r[m] -= r[j] * lmj;
        }
    }
#pragma unroll
    for (int m = 0; m < kNB; ++m)
        if (i < kb && m <= i) w[(k0 + i) * LD + k0 + m] = r[m];
    return failed;
}
template <int kMode>
__global__ void k(double* g, long long* out) {
    __shared__ double w[17 * 17];
    for (int e = threadIdx.x; e < 17 * 17; e += 32) w[e] = g[e];
    __syncwarp();
    long long t0 = clock64();
    bool f = false;
    for (int rep = 0; rep < 10; ++rep) {
        f |= dfac<16, kMode>(w, 17, 16, 0, 16);
        for (int e = threadIdx.x; e < 17 * 17; e += 32) w[e] = g[e];
        __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / 10 + (f ? 1 : 0);
}
int main() {
    double h[17 * 17] = {0};
    for (int i = 0; i < 16; ++i) for (int j = 0; j < 16; ++j) h[i * 17 + j] = (i == j ? 20.0 : 0.5);
    double* g; long long* o; cudaMalloc(&g, sizeof h); cudaMalloc(&o, 8);
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    long long c;
    k<0><<<1, 32>>>(g, o); cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost); printf("rsqrt: %lld cycles per 16-col block (%lld per col)\n", c, c / 16);
    k<1><<<1, 32>>>(g, o); cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost); printf("sqrt+div: %lld cycles per 16-col block (%lld per col)\n", c, c / 16);
    k<2><<<1, 32>>>(g, o); cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost); printf("dsqrt_rn+drcp_rn: %lld cycles per 16-col block (%lld per col)\n", c, c / 16);
    return 0;
}
