// a6.3: X-pencil (Alg. 5, §5.2), re-designed for sm_100a.
//
// The paper's block owns an X-pencil of target cells (plus 2 ghost cells), latches one
// target per thread in registers and then stages the <= 8 (Y, Z) +-1 neighbour pencils
// one at a time, with a barrier before and after each (:398-407).  Here a block owns an
// X-segment of one target row (cy, cz) and streams the 9 neighbour rows (dy, dz in
// {-1, 0, 1}) along X through shared memory in rounds:
//
//   * the 9 rows' cells x0-1 .. x0+L are contiguous runs of the cell-sorted array (X-fastest
//     linearisation), located from the global prefix array;
//   * they are staged in a MERGED layout: for every X cell, the particles of its 9 rows are
//     placed side by side (home row first), so the 27-cell candidate set of target cell cx
//     is the single contiguous window [M(cx-1), M(cx+2)) -- no per-row loop, no padding
//     slots, no wasted candidate tests;
//   * per round, as many X cells are staged as the shared-memory capacity holds (the
//     paper fixes the pencil length from M_C at launch, :353; counting the actual
//     occupancy instead needs no M_C read-back and no host synchronisation, and adapts
//     to clustered inputs), a cell whose window alone exceeds the capacity falls back to
//     the global-memory path;
//   * each staged particle is transformed once into the frame-local (A, B) records of
//     interact_common.cuh, and warps compute target cells with the packed-fp32 core.
#include "interact_common.cuh"

namespace pi {
namespace {

struct XpParams {
  long long n;
  const float4 *rec;
  const int32_t *offsets;
  Geom g;
  KParams kp;
  OutDesc out;
  DevCtl *ctl;
  int L;    // target cells per block along X
  int cap;  // staged particles per round
};

// smem carve (all int32 / float4; sizes in elements)
struct XpSmem {
  int *O;      // [9][L+3]  global offsets of cells x0-1 .. x0+L+1 per row (clamped)
  int *Moff;   // [L+3]     merged offsets
  int *D;      // [9][L+2]  dst base per (row, cell): Moff[j] + rowpre(r, j) - O[r][j]
  int *ctl;    // [16]      round control
  float4 *A, *B;
  float *red;  // [nwarps][256]
};

__host__ __device__ inline size_t xp_smem_bytes(int L, int cap, int nthreads) {
  size_t ints = 9 * (L + 3) + (L + 3) + 9 * (L + 2) + 16;
  ints = (ints + 3) & ~size_t(3);
  return ints * 4 + (size_t)cap * 32 + (size_t)(nthreads / 32) * 256 * 4;
}

template <int KERNEL, int NT>
__global__ void __launch_bounds__(NT) k_interact_xpencil(XpParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = p.L;
  XpSmem sm;
  {
    int *ip = reinterpret_cast<int *>(smem_raw);
    sm.O = ip;
    sm.Moff = sm.O + 9 * (L + 3);
    sm.D = sm.Moff + (L + 3);
    sm.ctl = sm.D + 9 * (L + 2);
    size_t ints = 9 * (L + 3) + (L + 3) + 9 * (L + 2) + 16;
    ints = (ints + 3) & ~size_t(3);
    sm.A = reinterpret_cast<float4 *>(smem_raw + ints * 4);
    sm.B = sm.A + p.cap;
    sm.red = reinterpret_cast<float *>(sm.B + p.cap);
  }
  const Geom &g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int x0 = blockIdx.x * L;
  const int cy = blockIdx.y, cz = blockIdx.z;
  const int Lseg = min(L, g.nx - x0);
  unsigned long long cand = 0, fallbacks = 0;

  // ---- tables: global offsets of the 9 neighbour rows over cells x0-1 .. x0+L+1
  for (int k = tid; k < 9 * (L + 3); k += NT) {
    const int r = k / (L + 3), j = k - r * (L + 3);
    const int y = cy + (r % 3) - 1, z = cz + (r / 3) - 1;
    int v = 0;
    if (y >= 0 && y < g.ny && z >= 0 && z < g.nz) {
      const int x = min(max(x0 - 1 + j, 0), g.nx);  // clamped: out-of-grid cells are empty
      v = __ldg(p.offsets + (long long)g.nx * (y + (long long)g.ny * z) + x);
    }
    sm.O[k] = v;
  }
  __syncthreads();
  // merged sizes and offsets (one thread: L <= 64 cells)
  if (tid == 0) {
    int acc = 0;
    for (int j = 0; j < L + 2; ++j) {
      sm.Moff[j] = acc;
      // home row (r = 4) first, then rows 0..3, 5..8
      int pre = acc;
#pragma unroll
      for (int rr = 0; rr < 9; ++rr) {
        const int r = rr == 0 ? 4 : (rr <= 4 ? rr - 1 : rr);
        const int c = sm.O[r * (L + 3) + j + 1] - sm.O[r * (L + 3) + j];
        sm.D[r * (L + 2) + j] = pre - sm.O[r * (L + 3) + j];
        pre += c;
      }
      acc = pre;
    }
    sm.Moff[L + 2] = acc;
  }
  __syncthreads();

  // frame: X from the middle of the segment, Y/Z from the centre of the target row
  const float fxo = fmaf((float)(x0 + L / 2), g.w, g.ox);
  const float fyo = fmaf((float)cy + 0.5f, g.w, g.oy);
  const float fzo = fmaf((float)cz + 0.5f, g.w, g.oz);

  int ja = 1;
  while (ja <= Lseg) {
    // ---- choose the round: targets ja..jb with merged cells ja-1 .. jb+1 <= cap
    if (tid == 0) {
      const int base = sm.Moff[ja - 1];
      int jb = ja - 1;
      while (jb + 1 <= Lseg && sm.Moff[jb + 3] - base <= p.cap) ++jb;
      sm.ctl[0] = jb;
      // per-row staging prefix
      int acc = 0;
      for (int r = 0; r < 9; ++r) {
        sm.ctl[1 + r] = acc;
        if (jb >= ja) acc += sm.O[r * (L + 3) + jb + 2] - sm.O[r * (L + 3) + ja - 1];
      }
      sm.ctl[10] = acc;
    }
    __syncthreads();
    const int jb = sm.ctl[0];
    if (jb < ja) {
      // even one target cell's window does not fit: global-memory fallback for cell ja
      block_fallback_cell<KERNEL>(x0 - 1 + ja, cy, cz, p.rec, p.offsets, g, p.kp, p.out, cand);
      ++fallbacks;
      ++ja;
      __syncthreads();
      continue;
    }
    const int base = sm.Moff[ja - 1];
    const int total = sm.ctl[10];
    int rp[10];
#pragma unroll
    for (int r = 0; r < 10; ++r) rp[r] = sm.ctl[1 + r];
    // ---- stage: flattened over the 9 row runs
    for (int k = tid; k < total; k += NT) {
      int r = 0;
#pragma unroll
      for (int rr = 1; rr < 9; ++rr) r += (k >= rp[rr]) ? 1 : 0;
      const int i = sm.O[r * (L + 3) + ja - 1] + (k - rp[r]);
      const float4 v = __ldg(p.rec + i);
      bool bad = false;
      const int cx = cell_coord(v.x, g.ox, g.inv_w, g.nx, bad);
      const int j = cx - (x0 - 1);
      const int dst = sm.D[r * (L + 2) + j] + i - base;
      stage_record(v, fxo, fyo, fzo, p.kp.s, sm.A[dst], sm.B[dst]);
    }
    __syncthreads();
    // ---- compute: warps take target cells of the round
    for (int j = ja + warp; j <= jb; j += NT / 32) {
      const int nt = sm.O[4 * (L + 3) + j + 1] - sm.O[4 * (L + 3) + j];
      if (nt == 0) continue;
      const int home = sm.Moff[j] - base;
      const int W0 = sm.Moff[j - 1] - base, W1 = sm.Moff[j + 2] - base;
      warp_cell<KERNEL>(sm.A, sm.B, home, nt, W0, W1, sm.O[4 * (L + 3) + j], p.kp.s_inv, p.rec, g, p.kp, p.out,
                        sm.red + warp * 256, cand);
    }
    __syncthreads();
    ja = jb + 1;
  }
  // statistics
  for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
  if ((tid & 31) == 0 && cand) atomicAdd(&p.ctl->candidates, cand);
  if (tid == 0 && fallbacks) atomicAdd(&p.ctl->fallback_cells, fallbacks);
}

template <int KERNEL, int NT>
cudaError_t launch_k(const XpParams &p, cudaStream_t s) {
  const size_t smem = xp_smem_bytes(p.L, p.cap, NT);
  cudaError_t e = cudaFuncSetAttribute(k_interact_xpencil<KERNEL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((p.g.nx + p.L - 1) / p.L, p.g.ny, p.g.nz);
  k_interact_xpencil<KERNEL, NT><<<grid, NT, smem, s>>>(p);
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_nt(const XpParams &p, cudaStream_t s) {
  switch (p.kp.kernel) {
    case PI_K_GAUSSIAN: return launch_k<PI_K_GAUSSIAN, NT>(p, s);
    case PI_K_INDICATOR: return launch_k<PI_K_INDICATOR, NT>(p, s);
    default: return launch_k<PI_K_CANDIDATE, NT>(p, s);
  }
}

}  // namespace

cudaError_t launch_interact_xpencil(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  XpParams p;
  p.n = a.n;
  p.rec = a.rec;
  p.offsets = a.offsets;
  p.g = g;
  p.kp = k;
  p.out = a.out;
  p.ctl = a.ctl;
  p.L = a.tx_len > 0 ? a.tx_len : 16;
  if (p.L > 64) p.L = 64;
  int threads = a.threads == 256 ? 256 : 128;
  if (a.tx_cap > 0) {
    p.cap = a.tx_cap;
  } else {
    // size the staging buffer for the mean occupancy of a round of 9 rows x (L + 2) cells
    double ppc = (double)a.n / (double)g.ncells;
    double want = 9.0 * (p.L + 2) * ppc * 1.3 + 256.0;
    p.cap = (int)want;
  }
  p.cap = (p.cap + 31) & ~31;
  const size_t max_smem = 227 * 1024;
  while (xp_smem_bytes(p.L, p.cap, threads) > max_smem && p.cap > 64) p.cap -= 32;
  if (threads == 256) return launch_nt<256>(p, s);
  return launch_nt<128>(p, s);
}

}  // namespace pi
