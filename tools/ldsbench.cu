// Shared-memory wavefronts per LDS.128 for lane address patterns (development aid; run under
// ncu with l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum / smsp__sass_inst_executed_op_shared_ld.sum).
// pattern p: lane -> 16-B word index
#include <cstdio>
__device__ int word_of(int p, int lane) {
  switch (p) {
    case 0: return 0;                         // all lanes one address
    case 1: return lane & 3;                  // 4 consecutive words, 8 lanes each
    case 2: return lane & 7;                  // 8 consecutive
    case 3: return lane & 15;                 // 16 consecutive
    case 4: return lane;                      // 32 consecutive
    case 5: return (lane >> 1);               // 16 consecutive, adjacent lanes share
    case 6: return (lane >> 2);               // 8 consecutive, groups of 4 lanes share
    case 7: return (lane * 7919) % 61;        // 32 pseudo-random words in 61
    case 8: return ((lane >> 1) * 7919) % 37; // 16 pseudo-random (pairs of lanes share)
    case 9: return (lane & 3) * 8;            // 4 words, same bank group
    case 10: return (lane >> 3);              // 4 consecutive, quarter-warps share
    default: return 0;
  }
}
__global__ void k(int p, int iters, float4 *out) {
  __shared__ float4 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_float4(i, i, i, i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int w = word_of(p, lane) + (threadIdx.x >> 5) * 64;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < iters; ++i) {
    float4 v = s[(w + i * 0) & 1023];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    w ^= (i & 1) ? 0 : 0;
    asm volatile("" : "+r"(w));
  }
  if (acc.x == -1.f) out[threadIdx.x] = acc;
}
int main(int argc, char **argv) {
  float4 *o;
  cudaMalloc(&o, 4096 * 16);
  for (int p = 0; p <= 10; ++p) k<<<1, 256>>>(p, 1000, o);
  cudaDeviceSynchronize();
  printf("ok\n");
}
