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
  float *out; long long *cyc; cudaMalloc(&out, sizeof(float)*sms*16*256); cudaMalloc(&cyc, 8);
  // ops per thread: FFMA / FFMA2 count lane-FMAs (2 FLOP each), EX2 counts ex2, MIX candidates
  struct { const char* name; const char* key; void(*k)(float*,float,float,long long*); double ops; double flop_per_op; } tests[] = {
    {"FFMA  (lane-FMA/clk/SM)", "ffma", k_ffma, 8.0*ITERS, 2.0}, {"FFMA2 (lane-FMA/clk/SM)", "ffma2", k_ffma2, 16.0*ITERS, 2.0},
    {"MUFU.EX2 (ex2/clk/SM)", "ex2", k_ex2, 8.0*ITERS, 0.0}, {"MIX (candidates/clk/SM)", "mix", k_mix, 2.0*ITERS, 0.0}};
  printf("{\"sms\": %d", sms);
  for (auto &t : tests) {
    double best_clk = 0, best_rate = 0; int best_res = 0;
    for (int resident : {4, 8}) {   // 256-thread blocks per SM, all co-resident
      const int blocks = sms * resident, threads = 256;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(cyc, 0, 8); cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a); t.k<<<blocks, threads>>>(out, 0.999f, 1e-4f, cyc); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double per_clk = t.ops * threads * resident / (double)c;      // per SM per SM clock
        const double per_s = t.ops * (double)threads * blocks / (ms * 1e-3);  // chip, wall clock
        if (rep == 2) fprintf(stderr, "%-28s blocks/SM=%d  %8.2f per clk per SM  %.3e per s  (%.3f ms, %lld cyc, %.0f MHz)\n",
                              t.name, resident, per_clk, per_s, ms, c, c / (ms * 1e3));
        if (rep == 2 && per_s > best_rate) { best_rate = per_s; best_clk = per_clk; best_res = resident; }
      }
    }
    printf(", \"%s_per_clk_per_sm\": %.2f, \"%s_per_s\": %.4e", t.key, best_clk, t.key, best_rate);
    if (t.flop_per_op > 0) printf(", \"%s_tflops\": %.2f", t.key, best_rate * t.flop_per_op / 1e12);
    (void)best_res;
  }
  printf("}\n");
  return 0;
}
