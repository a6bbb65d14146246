// Microbenchmark of the FP32 / MUFU issue rates the interaction kernels rely on (sm_100a).
// Reports per-SM throughput in lane-ops per SM clock (clock64 inside the kernel) so the
// result is independent of the DVFS clock.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0,{%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ u64 fma2(u64 a,u64 b,u64 c){u64 d; asm volatile("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(d):"l"(a),"l"(b),"l"(c)); return d;}
__device__ __forceinline__ float ex2(float a){float r; asm volatile("ex2.approx.ftz.f32 %0,%1;":"=f"(r):"f"(a)); return r;}
constexpr int ITERS = 4096;
__global__ void k_ffma(float *out, float b, float c, long long *cyc) {
  float a[8]; for (int k=0;k<8;++k) a[k]=threadIdx.x*1e-3f+k;
  long long t0=clock64();
  for (int i=0;i<ITERS;++i){
#pragma unroll
    for (int k=0;k<8;++k) a[k]=fmaf(a[k],b,c);
  }
  long long t1=clock64();
  float s=0; for(int k=0;k<8;++k) s+=a[k]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0) atomicMax((unsigned long long*)cyc,(unsigned long long)(t1-t0));
}
__global__ void k_ffma2(float *out, float b, float c, long long *cyc) {
  u64 a[8]; for (int k=0;k<8;++k) a[k]=pk(threadIdx.x*1e-3f+k, k*2.f);
  u64 B=pk(b,b), C=pk(c,c);
  long long t0=clock64();
  for (int i=0;i<ITERS;++i){
#pragma unroll
    for (int k=0;k<8;++k) a[k]=fma2(a[k],B,C);
  }
  long long t1=clock64();
  float s=0; for(int k=0;k<8;++k){float x,y; asm("mov.b64 {%0,%1},%2;":"=f"(x),"=f"(y):"l"(a[k])); s+=x+y;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0) atomicMax((unsigned long long*)cyc,(unsigned long long)(t1-t0));
}
__global__ void k_ex2(float *out, float b, float c, long long *cyc) {
  float a[8]; for (int k=0;k<8;++k) a[k]=-(threadIdx.x*1e-3f+k)*1e-3f;
  long long t0=clock64();
  for (int i=0;i<ITERS;++i){
#pragma unroll
    for (int k=0;k<8;++k) a[k]=ex2(a[k])*b - c;   // MUFU + FFMA
  }
  long long t1=clock64();
  float s=0; for(int k=0;k<8;++k) s+=a[k]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0) atomicMax((unsigned long long*)cyc,(unsigned long long)(t1-t0));
}
__global__ void k_mix(float *out, float b, float c, long long *cyc) {
  // the interaction inner loop's mix per source and target pair: 8 f32x2 FP ops, 2 FSETP, 2 MUFU
  u64 acc[4]; for(int k=0;k<4;++k) acc[k]=pk(0.f,0.f);
  u64 xt=pk(threadIdx.x*1e-3f,1.f), Yt=pk(0.1f,0.2f), Zt=pk(0.3f,0.4f);
  float s0=b, s1=c, s2=b*c, s3=b+c;
  long long t0=clock64();
  for (int i=0;i<ITERS;++i){
    u64 dx; asm volatile("add.rn.f32x2 %0,%1,%2;":"=l"(dx):"l"(xt),"l"(pk(-s0,-s0)));
    u64 v=fma2(dx,dx,pk(s3,s3)); v=fma2(Yt,pk(s1,s1),v); v=fma2(Zt,pk(s2,s2),v);
    float v0,v1; asm("mov.b64 {%0,%1},%2;":"=f"(v0),"=f"(v1):"l"(v));
    float k0 = v0 < 5.f ? ex2(-v0) : 0.f, k1 = v1 < 5.f ? ex2(-v1) : 0.f;
    u64 K=pk(k0,k1);
    acc[0]=fma2(K,pk(s0,s0),acc[0]); acc[1]=fma2(K,pk(s1,s1),acc[1]); acc[2]=fma2(K,pk(s2,s2),acc[2]); acc[3]=fma2(K,pk(s3,s3),acc[3]);
    s0+=1e-7f;
  }
  long long t1=clock64();
  float s=0; for(int k=0;k<4;++k){float x,y; asm("mov.b64 {%0,%1},%2;":"=f"(x),"=f"(y):"l"(acc[k])); s+=x+y;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0) atomicMax((unsigned long long*)cyc,(unsigned long long)(t1-t0));
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out; long long *cyc; cudaMalloc(&out, sizeof(float)*sms*8*256); cudaMalloc(&cyc, 8);
  struct { const char* name; void(*k)(float*,float,float,long long*); double ops; } tests[] = {
    {"FFMA  (lane-FMA/clk/SM)", k_ffma, 8.0*ITERS}, {"FFMA2 (lane-FMA/clk/SM)", k_ffma2, 16.0*ITERS},
    {"MUFU.EX2 (ex2/clk/SM)", k_ex2, 8.0*ITERS}, {"MIX (candidates/clk/SM)", k_mix, 2.0*ITERS}};
  for (auto &t : tests) for (int occ : {8, 16}) {
    int blocks = sms*occ/8*1, threads = 256;  // occ warps per SMSP-ish
    blocks = sms * occ / 2;
    for (int rep=0; rep<2; ++rep){
      cudaMemset(cyc,0,8); cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a); t.k<<<blocks,threads>>>(out,0.999f,1e-4f,cyc); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms,a,b); long long c; cudaMemcpy(&c,cyc,8,cudaMemcpyDeviceToHost);
      double total = t.ops * (double)blocks * threads;
      double per_sm_clk = total / ((double)c * sms) * ((double)blocks / (sms * (double)(occ/2 > 0 ? 1 : 1)));
      // blocks are co-resident when blocks <= sms*8 (256 thr, <=2048 thr/SM): use max cycles of one block
      int resident = blocks / sms; // blocks per SM (all resident)
      double rate = t.ops * threads * resident / (double)c;
      if (rep) printf("%-28s blocks/SM=%2d  %8.2f per clk per SM   (%.3f ms, %lld cyc)\n", t.name, resident, rate, ms, c);
    }
  }
  return 0;
}
