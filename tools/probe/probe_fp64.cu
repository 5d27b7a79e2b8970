// Probe: FP64 DMMA vs DFMA throughput on sm_100a, and mma.sync f64 fragment layouts.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);} }while(0)

__device__ __forceinline__ void mma884(double& d0,double& d1,double a,double b){
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(d0),"+d"(d1) : "d"(a),"d"(b));
}
__device__ __forceinline__ void mma1684(double* d,double a0,double a1,double b){
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};" : "+d"(d[0]),"+d"(d[1]),"+d"(d[2]),"+d"(d[3]) : "d"(a0),"d"(a1),"d"(b));
}
__device__ __forceinline__ void mma1688(double* d,const double* a,const double* b){
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};" : "+d"(d[0]),"+d"(d[1]),"+d"(d[2]),"+d"(d[3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(b[0]),"d"(b[1]));
}
__device__ __forceinline__ void mma16816(double* d,const double* a,const double* b){
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};" : "+d"(d[0]),"+d"(d[1]),"+d"(d[2]),"+d"(d[3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),"d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
}

template<int CH>
__global__ void dmma884_loop(double* out,int iters){
  double acc[CH][2]; double a=threadIdx.x*1e-3, b=1.0+blockIdx.x*1e-6;
  for(int c=0;c<CH;c++){acc[c][0]=0;acc[c][1]=0;}
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int c=0;c<CH;c++) mma884(acc[c][0],acc[c][1],a,b);
  }
  double s=0; for(int c=0;c<CH;c++) s+=acc[c][0]+acc[c][1];
  if(s==123.456) out[0]=s;
}
template<int CH>
__global__ void dmma16816_loop(double* out,int iters){
  double acc[CH][4]; double a[8],b[4];
  for(int i=0;i<8;i++) a[i]=threadIdx.x*1e-3+i; for(int i=0;i<4;i++) b[i]=1.0+blockIdx.x*1e-6;
  for(int c=0;c<CH;c++) for(int j=0;j<4;j++) acc[c][j]=0;
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int c=0;c<CH;c++) mma16816(acc[c],a,b);
  }
  double s=0; for(int c=0;c<CH;c++) for(int j=0;j<4;j++) s+=acc[c][j];
  if(s==123.456) out[0]=s;
}
template<int CH>
__global__ void dfma_loop(double* out,int iters){
  double acc[CH]; double a=threadIdx.x*1e-3, b=1.0+blockIdx.x*1e-9;
  for(int c=0;c<CH;c++) acc[c]=c;
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int c=0;c<CH;c++) acc[c]=fma(acc[c],b,a);
  }
  double s=0; for(int c=0;c<CH;c++) s+=acc[c];
  if(s==123.456) out[0]=s;
}

// layout checks: A row-major MxK, B KxN (stored [k][n]), D MxN
__global__ void chk884(const double* A,const double* B,double* D){
  int l=threadIdx.x, g=l>>2, t=l&3; double d0=0,d1=0;
  mma884(d0,d1,A[g*4+t],B[t*8+g]);
  D[g*8+2*t]=d0; D[g*8+2*t+1]=d1;
}
__global__ void chk1684(const double* A,const double* B,double* D){
  int l=threadIdx.x, g=l>>2, t=l&3; double d[4]={0,0,0,0};
  mma1684(d,A[g*4+t],A[(g+8)*4+t],B[t*8+g]);
  D[g*8+2*t]=d[0]; D[g*8+2*t+1]=d[1]; D[(g+8)*8+2*t]=d[2]; D[(g+8)*8+2*t+1]=d[3];
}
__global__ void chk1688(const double* A,const double* B,double* D){
  int l=threadIdx.x, g=l>>2, t=l&3; double d[4]={0,0,0,0}; double a[4],b[2];
  a[0]=A[g*8+t]; a[1]=A[(g+8)*8+t]; a[2]=A[g*8+t+4]; a[3]=A[(g+8)*8+t+4];
  b[0]=B[t*8+g]; b[1]=B[(t+4)*8+g];
  mma1688(d,a,b);
  D[g*8+2*t]=d[0]; D[g*8+2*t+1]=d[1]; D[(g+8)*8+2*t]=d[2]; D[(g+8)*8+2*t+1]=d[3];
}
__global__ void chk16816(const double* A,const double* B,double* D){
  int l=threadIdx.x, g=l>>2, t=l&3; double d[4]={0,0,0,0}; double a[8],b[4];
  for(int i=0;i<8;i++){ int r=g+8*(i&1), c=t+4*(i>>1); a[i]=A[r*16+c]; }
  for(int i=0;i<4;i++) b[i]=B[(t+4*i)*8+g];
  mma16816(d,a,b);
  D[g*8+2*t]=d[0]; D[g*8+2*t+1]=d[1]; D[(g+8)*8+2*t]=d[2]; D[(g+8)*8+2*t+1]=d[3];
}

void check(const char* name,void(*k)(const double*,const double*,double*),int M,int K){
  int N=8; double hA[16*16],hB[16*8],hD[16*8],ref[16*8];
  for(int i=0;i<M*K;i++) hA[i]=(i*7%13)-6+0.5*(i%3);
  for(int i=0;i<K*N;i++) hB[i]=(i*5%11)-5+0.25*(i%2);
  for(int m=0;m<M;m++)for(int n=0;n<N;n++){double s=0;for(int kk=0;kk<K;kk++)s+=hA[m*K+kk]*hB[kk*N+n];ref[m*N+n]=s;}
  double *dA,*dB,*dD; CK(cudaMalloc(&dA,sizeof hA));CK(cudaMalloc(&dB,sizeof hB));CK(cudaMalloc(&dD,sizeof hD));
  CK(cudaMemcpy(dA,hA,sizeof hA,cudaMemcpyHostToDevice));CK(cudaMemcpy(dB,hB,sizeof hB,cudaMemcpyHostToDevice));
  CK(cudaMemset(dD,0,sizeof hD));
  k<<<1,32>>>(dA,dB,dD); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hD,dD,sizeof hD,cudaMemcpyDeviceToHost));
  double err=0; for(int i=0;i<M*N;i++) err=fmax(err,fabs(hD[i]-ref[i]));
  printf("layout %-10s maxerr=%g %s\n",name,err,err==0?"OK":"MISMATCH");
}

template<typename F> float timeit(F f){
  cudaEvent_t a,b; cudaEventCreate(&a);cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a); for(int r=0;r<3;r++) f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms,a,b); return ms/3;
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("%s SMs=%d cc=%d.%d l2=%d MB mem=%.1f GB smem/blk optin=%zu\n",p.name,p.multiProcessorCount,p.major,p.minor,p.l2CacheSize>>20,p.totalGlobalMem/1e9,p.sharedMemPerBlockOptin);
  check("m8n8k4",chk884,8,4); check("m16n8k4",chk1684,16,4); check("m16n8k8",chk1688,16,8); check("m16n8k16",chk16816,16,16);
  double* out; CK(cudaMalloc(&out,8));
  int sms=p.multiProcessorCount; int iters=20000;
  for(int wpb: {4,8,16}){
    for(int bps: {1,2,4}){
      int blocks=sms*bps, thr=32*wpb;
      float ms=timeit([&]{dmma884_loop<8><<<blocks,thr>>>(out,iters);});
      double fl=2.0*8*8*4*8.0*iters*blocks*wpb;
      float ms2=timeit([&]{dmma16816_loop<4><<<blocks,thr>>>(out,iters/4);});
      double fl2=2.0*16*8*16*4.0*(iters/4)*blocks*wpb;
      float ms3=timeit([&]{dfma_loop<16><<<blocks,thr>>>(out,iters);});
      double fl3=2.0*16*iters*(double)blocks*thr;
      printf("warps/blk=%2d blk/SM=%d  DMMA884 %.2f TF  DMMA16816 %.2f TF  DFMA %.2f TF\n",wpb,bps,fl/ms/1e9,fl2/ms2/1e9,fl3/ms3/1e9);
    }
  }
  return 0;
}
