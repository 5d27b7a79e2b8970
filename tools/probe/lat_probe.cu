// Probe: dependent-issue latency (cycles) of FP64 DFMA, DMUL, the rsqrt.approx.f64
// seed (MUFU.RSQ64H) and a 64-bit warp shuffle on sm_100a (one warp, clock64).
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 1.0; }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31) + 1e-9;
  long long t4 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  const int n = 4096;
  k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize();
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: DFMA %.1f  DMUL %.1f  rsqrt.f64 seed + DADD %.1f  SHFL.64 + DADD %.1f\n",
         h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
  return 0;
}
