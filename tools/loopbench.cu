// Inner-loop microbenchmark: the X-pencil core (lane_target) on synthetic shared-memory
// windows, no staging.  Reports candidates per SM clock.  Development aid, not product.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2406_16091_b200/csrc/interact_common.cuh"
using namespace pi;
template <int UNR, int NT>
__global__ void __launch_bounds__(NT) k(float *out, int reps, int wpairs, long long *cyc) {
  extern __shared__ float4 S[];
  const int npairs = 2048;
  for (int i = threadIdx.x; i < 2 * npairs; i += NT) {
    unsigned h = i * 2654435761u;
    float a = (h & 1023) / 1024.f * 0.03f, b = ((h >> 10) & 1023) / 1024.f * 0.03f;
    S[i] = (i & 1) ? make_float4(a, b, 1.f, 1.f) : make_float4(a, b, b, a);
  }
  __syncthreads();
  long long t0 = clock64();
  float acc = 0.f;
  for (int r = 0; r < reps; ++r) {
    const int p0 = ((threadIdx.x >> 3) * 37 * 4 + r * 4 * 101 + (threadIdx.x & 24) / 8) % (npairs - wpairs - 8);
    const float xt = S[2 * p0].x, yt = S[2 * p0].z, zt = S[2 * p0 + 1].x;
    p2 ph = pk(0.f), fx = pk(0.f), fy = pk(0.f), fz = pk(0.f);
    for (int q = p0; q < p0 + wpairs; ++q)
      src_eval<PI_K_GAUSSIAN>(load_pair(S, S + npairs, q), xt, yt, zt, 2.4e-4f, -6.5f / 2.4e-4f, ph, fx, fy, fz);
    acc += lo(ph) + hi(fx) + lo(fy) + hi(fz);
  }
  long long t1 = clock64();
  out[blockIdx.x * NT + threadIdx.x] = acc;
  if (threadIdx.x == 0) atomicMax((unsigned long long *)cyc, (unsigned long long)(t1 - t0));
}
template <int UNR, int NT>
void run(int bps, int sms) {
  float *out; long long *cyc;
  cudaMalloc(&out, 4 << 20); cudaMalloc(&cyc, 8);
  size_t smem = 2 * 2048 * 16;
  cudaFuncSetAttribute(k<UNR, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int reps = 40, wp = 113;
  for (int it = 0; it < 2; ++it) {
    cudaMemset(cyc, 0, 8);
    k<UNR, NT><<<sms * bps, NT, smem>>>(out, reps, wp, cyc);
    cudaDeviceSynchronize();
  }
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<UNR, NT>, NT, smem);
  double cand = 2.0 * wp * reps * NT * bps;  // per SM
  printf("UNR=%d NT=%4d blocks/SM=%d (occ %d) warps/SM=%3d: %.2f candidates/clk/SM  (%.1f%% of 74.45 TF-equiv)\n", UNR, NT, bps, occ,
         NT / 32 * bps, cand / c, cand / c * 9.57 / 256.0 * 100);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 256>(1, sms); run<4, 256>(2, sms); run<4, 256>(3, sms);
  run<2, 256>(1, sms); run<2, 256>(2, sms); run<2, 256>(3, sms);
  run<2, 128>(4, sms); run<2, 128>(6, sms); run<2, 128>(8, sms);
  run<4, 512>(1, sms); run<2, 512>(2, sms);
  return 0;
}
