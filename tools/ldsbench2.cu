// X-pencil walk access pattern: wavefronts per LDS.128, linear vs 128-B XOR-swizzled staging
// (development aid; ncu metrics as tools/ldsbench.cu).  Lane starts simulate 32 consecutive
// sorted targets (X sub-cells with Poisson(2) records, sx = 4): target in sub-cell u starts its
// window at the pair holding the first record of sub-cell u - 4.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
__global__ void k(const int *starts, int nwarps, int swz, int iters, float4 *out) {
  __shared__ float4 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int w = warp; w < nwarps; w += blockDim.x >> 5) {
    const int st = starts[w * 32 + lane];
    for (int i = 0; i < iters; ++i) {
      int p = (st + i) & 2047;
      if (swz) p ^= (p >> 3) & 7;
      const float4 v = s[p];
      acc.x += v.x; acc.y += v.y;
    }
  }
  if (acc.x == -1.f) out[threadIdx.x] = acc;
}
int main() {
  std::mt19937 rng(1);
  std::poisson_distribution<int> pois(2.0);
  const int nw = 4096;
  std::vector<int> st(nw * 32);
  for (int w = 0; w < nw; ++w) {
    int cnt[64], off[65];
    off[0] = 0;
    for (int u = 0; u < 64; ++u) { cnt[u] = pois(rng); off[u + 1] = off[u] + cnt[u]; }
    // targets: the records of sub-cells 4.. in order, 32 of them
    int l = 0;
    for (int u = 4; u < 64 && l < 32; ++u)
      for (int k2 = 0; k2 < cnt[u] && l < 32; ++k2) st[w * 32 + l++] = 256 + off[u - 4] / 2;
    while (l < 32) { st[w * 32 + l] = st[w * 32 + l - 1]; ++l; }
  }
  int *d; float4 *o;
  cudaMalloc(&d, st.size() * 4); cudaMalloc(&o, 4096 * 16);
  cudaMemcpy(d, st.data(), st.size() * 4, cudaMemcpyHostToDevice);
  k<<<1, 256>>>(d, nw, 0, 8, o);
  k<<<1, 256>>>(d, nw, 1, 8, o);
  cudaDeviceSynchronize();
  printf("ok\n");
}
