// Probe: does FP64 DMMA throughput depend on operand data (power / clock)?
// Three variants of the same m16n8k16 loop, 8 warps x 2 CTAs per SM:
//   const : near-constant register operands (the bench's peak probe)
//   rand  : random [0,1) register operands, fixed across iterations
//   lds   : random [0,1) operands reloaded from shared memory every iteration
//           (the root GEMM's pattern: LDS.64 fragments feeding DMMA)
// Each CTA records clock64 and globaltimer around its loop, so the effective
// SM clock under that load is reported next to the throughput.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);} }while(0)

__device__ __forceinline__ void mma16816(double* d,const double* a,const double* b){
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};" : "+d"(d[0]),"+d"(d[1]),"+d"(d[2]),"+d"(d[3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),"d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
}
__device__ __forceinline__ double urand(uint64_t x){
  x += 0x9E3779B97F4A7C15ull; x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull; x ^= x >> 31;
  return (x >> 11) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ uint64_t gtimer(){ uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

template<int MODE>
__global__ void __launch_bounds__(256) loop(double* out, uint64_t* clk, int iters){
  __shared__ double sm[16 * 12 * 32];   // 16 operand sets x 12 doubles x 32 lanes (48 KB)
  const int lane = threadIdx.x & 31, tid = threadIdx.x;
  double acc[8][4], a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = MODE == 0 ? tid * 1e-3 + i : urand(tid * 131 + i + blockIdx.x * 7919);
  for (int i = 0; i < 4; ++i) b[i] = MODE == 0 ? 1.0 + blockIdx.x * 1e-6 : urand(tid * 977 + i + 55 + blockIdx.x * 104729);
  for (int c = 0; c < 8; ++c) for (int j = 0; j < 4; ++j) acc[c][j] = MODE == 0 ? 0.0 : urand(c * 4 + j + tid * 17);
  if (MODE == 2) {
    for (int i = tid; i < 16 * 12 * 32; i += blockDim.x) sm[i] = urand(i * 3 + blockIdx.x);
    __syncthreads();
  }
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 2) {
      const double* s = sm + (it & 15) * 12 * 32 + lane;
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = s[i * 32];
#pragma unroll
      for (int i = 0; i < 4; ++i) b[i] = s[(8 + i) * 32];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) mma16816(acc[c], a, b);
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
  for (int c = 0; c < 8; ++c) for (int j = 0; j < 4; ++j) s += acc[c][j];
  if (s == 123.456) out[0] = s;
  if (tid == 0) { clk[2 * blockIdx.x] = c1 - c0; clk[2 * blockIdx.x + 1] = t1 - t0; }
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount, blocks = 2 * sms, thr = 256, iters = 40000;
  double* out; uint64_t* clk; CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&clk, 16 * blocks));
  uint64_t* h = (uint64_t*)malloc(16 * blocks);
  const char* names[3] = {"const", "rand", "lds"};
  for (int rep = 0; rep < 2; ++rep)
  for (int m = 0; m < 3; ++m) {
    auto launch = [&]{
      if (m == 0) loop<0><<<blocks, thr>>>(out, clk, iters);
      else if (m == 1) loop<1><<<blocks, thr>>>(out, clk, iters);
      else loop<2><<<blocks, thr>>>(out, clk, iters);
    };
    launch(); CK(cudaDeviceSynchronize());
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    CK(cudaMemcpy(h, clk, 16 * blocks, cudaMemcpyDeviceToHost));
    double mhz = 0; for (int i = 0; i < blocks; ++i) mhz += (double)h[2 * i] / (double)h[2 * i + 1] * 1e3; mhz /= blocks;
    double fl = 2.0 * 16 * 8 * 16 * 8.0 * iters * blocks * (thr / 32);
    printf("%-6s %.2f TF  %.2f ms  SM clock in-kernel %.0f MHz  TF/GHz %.2f\n", names[m], fl / ms / 1e9, ms, mhz, fl / ms / 1e9 / (mhz / 1e3));
  }
  return 0;
}
