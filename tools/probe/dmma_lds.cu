// Probe: DMMA m16n8k16 throughput when fragments come from shared memory each
// k-step (like the root GEMM warp tile 16 x 8*NT, A 8 LDS + B 4*NT LDS per step)
// vs register-resident operands.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double* d, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
template <int NT, bool LDS>
__global__ void k(double* out, int iters) {
    __shared__ double sm[16 * 128 + 16 * 132];
    for (int i = threadIdx.x; i < 16 * 128 + 16 * 132; i += blockDim.x) sm[i] = 1e-3 * i;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
    double acc[NT][4] = {};
    double a[8], b[NT][4];
    for (int i = 0; i < 8; ++i) a[i] = sm[(g + 8 * (i & 1)) * 20 + t + 4 * (i >> 1)];
    for (int j = 0; j < NT; ++j) for (int i = 0; i < 4; ++i) b[j][i] = sm[2048 + (t + 4 * i) * 132 + 8 * j + g];
    for (int it = 0; it < iters; ++it) {
        if (LDS) {
            const int off = (it & 7) * 16;
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = sm[(warp * 16 + g + 8 * (i & 1)) % 128 * 16 + ((off + t + 4 * (i >> 1)) & 15)];
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) b[j][i] = sm[2048 + ((off + t + 4 * i) & 15) * 132 + 8 * j + g];
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[j], a, b[j]);
    }
    double s = 0;
    for (int j = 0; j < NT; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
    if (s == 1.2345) out[0] = s;
}
template <int NT, bool LDS>
void run(int warps) {
    double* o; cudaMalloc(&o, 8);
    int iters = 2000;
    k<NT, LDS><<<148, 32 * warps>>>(o, 10);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<NT, LDS><<<148, 32 * warps>>>(o, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fl = 148.0 * warps * iters * NT * 4096.0;
    printf("NT=%2d LDS=%d warps=%2d: %.2f TFLOP/s\n", NT, LDS, warps, fl / (ms * 1e-3) / 1e12);
}
int main() {
    run<13, false>(8); run<13, true>(8); run<13, true>(16);
    run<7, false>(8); run<7, true>(8); run<7, true>(16);
    return 0;
}
