// Staging microbenchmark (development aid): cycles for one warp to move one X-pencil work
// item's worth of small runs (306 runs x ~8 records of 16 B, L2-resident source) into shared
// memory, by (a) one cp.async.bulk (TMA) per run issued from all 32 lanes, (b) 16-B cp.async
// per record, 4 lanes per run.  Several producer warps per SM run concurrently.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2406_16091_b200/csrc/interact_common.cuh"
using namespace pi;

constexpr int RUNS = 306, PER = 8;

template <int MODE>
__global__ void k(const float4 *src, long long nsrc, int iters, long long *cyc, int *sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long *bar = reinterpret_cast<unsigned long long *>(sm) + w;
  float4 *dst = reinterpret_cast<float4 *>(sm + 256) + (size_t)w * RUNS * PER;
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  long long t0 = clock64();
  unsigned phase = 0;
  for (int it = 0; it < iters; ++it) {
    const long long base = ((long long)(blockIdx.x * 4 + w) * 7919 + it * 104729) % (nsrc - RUNS * 40);
    if (MODE == 0) {
      if (lane == 0) mbar_arrive_expect_tx(bar, RUNS * PER * 16);
      __syncwarp();
      for (int r = lane; r < RUNS; r += 32)
        bulk_g2s(dst + r * PER, src + base + (long long)r * 37, PER * 16, bar);
      mbar_wait(bar, phase);
      phase ^= 1;
    } else {
      const int sub = lane >> 2, e0 = lane & 3;
      for (int r = sub; r < RUNS; r += 8)
        for (int e = e0; e < PER; e += 4) cp_async16(dst + r * PER + e, src + base + (long long)r * 37 + e);
      cp_async_wait_all();
      __syncwarp();
    }
    __syncwarp();
    fence_proxy_async();
  }
  long long t1 = clock64();
  if (lane == 0) atomicMax((unsigned long long *)cyc, (unsigned long long)(t1 - t0));
  if (lane == 0 && dst[lane].x == 12345.f) *sink = 1;
}

int main() {
  const long long n = 1 << 21;
  float4 *src;
  cudaMalloc(&src, n * 16);
  cudaMemset(src, 0, n * 16);
  long long *cyc;
  int *sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps = 1; warps <= 4; warps *= 2) {
      const size_t smem = 256 + (size_t)warps * RUNS * PER * 16;
      auto kern = mode == 0 ? k<0> : k<1>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 50;
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(cyc, 0, 8);
        kern<<<sms, warps * 32, smem>>>(src, n, iters, cyc, sink);
        cudaDeviceSynchronize();
      }
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%s warps/SM=%d: %.0f cycles per item (%d runs x %d records)  %s\n",
             mode == 0 ? "TMA bulk per run   " : "cp.async 16B/record", warps, (double)c / iters, RUNS, PER,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
