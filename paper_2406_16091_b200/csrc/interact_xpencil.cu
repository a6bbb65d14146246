// a6.3: X-pencil (Alg. 5, §5.2), re-designed for sm_100a.
//
// The paper's block owns an X-pencil of target cells (plus 2 ghost cells), latches one
// target per thread in registers and then stages the <= 8 (Y, Z) +-1 neighbour pencils
// one at a time, with a barrier before and after each (:398-407).  Here a block owns an
// X-segment (normally the whole X row) of one target row (cy, cz) and streams the 9
// neighbour rows (dy, dz in {-1, 0, 1}) along X through shared memory in rounds:
//
//   * each (row, cell) of the 9 rows is a contiguous run of the cell-sorted 16-B records
//     (X-fastest linearisation), located from the global prefix array;
//     it is copied by ONE TMA bulk copy (cp.async.bulk, completion on an mbarrier) straight
//     into a MERGED layout: for every X cell the particles of its 9 rows sit side by side
//     (home row first), so the 27-cell candidate set of target cell cx is the single
//     contiguous window [M(cx-1), M(cx+2)) -- no per-row loop and no wasted candidates;
//   * merged cell j starts at an even slot M(j) = 2j (mod 8) (a few inert padding records):
//     windows are whole source PAIRS, and the windows of the ~4 cells of a warp start in
//     distinct 32-B bank groups, so the lanes' window walks do not conflict;
//   * per round, as many X cells are staged as the shared-memory capacity holds (the paper
//     fixes the pencil length from M_C at launch, :353; counting the actual occupancy
//     needs no M_C read-back and no host synchronisation and adapts to clustered inputs);
//     a cell whose window alone exceeds the capacity falls back to the global-memory path;
//   * staged records are interleaved in place into the source-PAIR layout of
//     interact_common.cuh (bitwise copies of the fp32 inputs, no frame, no scaling);
//   * compute: one thread per target ("one thread per particle", :357), like the paper,
//     but each thread walks its cell's whole window two sources per packed-fp32 op.
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
  int cap;  // staged particles (incl. padding) per round
};

// int area: ctl[40] | O[9][L+3] | Dst[9][L+2] | Msz[L+2] | Moff[L+3] | Tpre[L+3]
__host__ __device__ inline int xp_int_words(int L) {
  int ints = 40 + 9 * (L + 3) + 9 * (L + 2) + (L + 2) + (L + 3) + (L + 3);
  return (ints + 3) & ~3;  // keep the mbarrier / float4 area 16-B aligned
}
__host__ __device__ inline size_t xp_smem_bytes(int L, int cap) {
  return (size_t)xp_int_words(L) * 4 + 16 + (size_t)cap * 16;
}

constexpr float DUMMY_X = 1.0e30f;  // inert padding record: (x_s - x_t)^2 = inf, q = 0

template <int KERNEL, int NT>
__global__ void __launch_bounds__(NT) k_interact_xpencil(XpParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = p.L, L3 = L + 3, L2 = L + 2;
  int *ctl = reinterpret_cast<int *>(smem_raw);  // [40] (first: 8-B aligned, reused for u64)
  int *O = ctl + 40;                             // [9][L+3] global offsets, cells x0-1 .. x0+L+1
  int *Dst = O + 9 * L3;                         // [9][L+2] row start inside its merged cell
  int *Msz = Dst + 9 * L2;                       // [L+2]    merged cell sizes
  int *Moff = Msz + L2;                          // [L+3]    padded merged offsets, even, = 2j (mod 8)
  int *Tpre = Moff + L3;                         // [L+3]    target prefix of the round
  unsigned long long *bar = reinterpret_cast<unsigned long long *>(smem_raw + xp_int_words(L) * 4);
  float4 *S = reinterpret_cast<float4 *>(smem_raw + xp_int_words(L) * 4 + 16);

  const Geom &g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int x0 = blockIdx.x * L;
  const int cy = blockIdx.y, cz = blockIdx.z;
  const int Lseg = min(L, g.nx - x0);
  const float thr = p.kp.rc2, mc2 = -p.kp.c2;
  unsigned long long cand = 0, fallbacks = 0;

  if (tid == 0) mbar_init(bar, 1);
  // ---- tables: global offsets of the 9 neighbour rows over cells x0-1 .. x0+L+1
  for (int k = tid; k < 9 * L3; k += NT) {
    const int r = k / L3, j = k - r * L3;
    const int y = cy + (r % 3) - 1, z = cz + (r / 3) - 1;
    int v = 0;
    if (y >= 0 && y < g.ny && z >= 0 && z < g.nz) {
      const int x = min(max(x0 - 1 + j, 0), g.nx);  // clamped: out-of-grid cells are empty
      v = __ldg(p.offsets + (long long)g.nx * (y + (long long)g.ny * z) + x);
    }
    O[k] = v;
  }
  __syncthreads();
  // per merged cell: row starts (home row r = 4 first, then 0..3, 5..8) and size
  for (int j = tid; j < L2; j += NT) {
    int pre = 0;
#pragma unroll
    for (int rr = 0; rr < 9; ++rr) {
      const int r = rr == 0 ? 4 : (rr <= 4 ? rr - 1 : rr);
      Dst[r * L2 + j] = pre;
      pre += O[r * L3 + j + 1] - O[r * L3 + j];
    }
    Msz[j] = pre;
  }
  __syncthreads();
  if (tid == 0) {  // padded offsets: M(j) = 2j (mod 8); sequential, L + 2 <= 66 steps
    int m = 0;
    for (int j = 0; j < L2; ++j) {
      m += (2 * j - m) & 7;
      Moff[j] = m;
      m += Msz[j];
    }
    m += (2 * L2 - m) & 7;
    Moff[L2] = m;
  }
  __syncthreads();

  unsigned phase = 0;
  int ja = 1;
  while (ja <= Lseg) {
    // ---- round: targets ja..jb, staged merged cells ja-1 .. jb+1 (monotone fit test)
    if (warp == 0) {
      const int base = Moff[ja - 1];
      int jb = ja - 1;
      for (int j0 = ja; j0 <= Lseg; j0 += 32) {
        const int j = j0 + lane;
        const bool fit = j <= Lseg && Moff[j + 2] - base <= p.cap;
        const unsigned b = __ballot_sync(0xffffffffu, fit);
        jb += __popc(b);
        if (b != 0xffffffffu) break;
      }
      if (lane == 0) {
        ctl[0] = jb;
        if (jb >= ja) {
          int real = 0;
          for (int j = ja - 1; j <= jb + 1; ++j) real += Msz[j];
          mbar_arrive_expect_tx(bar, (unsigned)real * 16u);
        }
      }
      // target prefix over the round's cells
      if (jb >= ja) {
        int carry = 0;
        for (int j0 = ja; j0 <= jb; j0 += 32) {
          const int j = j0 + lane;
          const int nt = j <= jb ? O[4 * L3 + j + 1] - O[4 * L3 + j] : 0;
          int incl = nt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
          }
          if (j <= jb) Tpre[j] = carry + incl - nt;
          carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
          ctl[1] = carry;  // total targets
          Tpre[jb + 1] = carry;
        }
      }
    }
    __syncthreads();
    const int jb = ctl[0];
    if (jb < ja) {
      // even one target cell's window does not fit: global-memory fallback for cell ja
      block_fallback_cell<KERNEL>(x0 - 1 + ja, cy, cz, p.rec, p.offsets, g, p.kp, p.out, cand);
      ++fallbacks;
      ++ja;
      __syncthreads();
      continue;
    }
    const int base = Moff[ja - 1];
    const int total = Moff[jb + 2] - base;  // even
    const int ntargets = ctl[1];
    // ---- stage: one TMA bulk copy per (row, cell) run into the merged layout
    const int ncell = jb - ja + 3;
    for (int k = tid; k < 9 * ncell; k += NT) {
      const int jj = k / 9, r = k - jj * 9;
      const int j = ja - 1 + jj;
      const int src = O[r * L3 + j];
      const int c = O[r * L3 + j + 1] - src;
      if (c > 0) bulk_g2s(S + (Moff[j] + Dst[r * L2 + j] - base), p.rec + src, (unsigned)c * 16u, bar);
    }
    // padding records (disjoint from the bulk-copy destinations)
    for (int k = tid; k < 8 * ncell; k += NT) {
      const int jj = k >> 3, u = k & 7;
      const int j = ja - 1 + jj;
      const int s = Moff[j] + Msz[j] + u;
      if (s < Moff[j + 1]) S[s - base] = make_float4(DUMMY_X, DUMMY_X, DUMMY_X, 0.f);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    __syncthreads();  // padding written by other threads
    // ---- interleave in place: raw record pairs -> source-pair layout
    for (int k = tid; k < (total >> 1); k += NT) stage_pair(S, k);
    fence_proxy_async();  // our generic writes before the next round's async-proxy writes
    __syncthreads();
    // ---- compute: one thread per target, walking its cell's window
    for (int T = tid; T < ntargets; T += NT) {
      // cell of target T: last j in [ja, jb] with Tpre[j] <= T (binary search)
      int lo_ = ja, hi_ = jb;
      while (lo_ < hi_) {
        const int mid = (lo_ + hi_ + 1) >> 1;
        if (Tpre[mid] <= T) lo_ = mid; else hi_ = mid - 1;
      }
      const int j = lo_;
      const int i = T - Tpre[j];
      const int t = Moff[j] - base + i;                       // staged slot of the target
      const int p0 = (Moff[j - 1] - base) >> 1, p1 = (Moff[j + 2] - base) >> 1;
      const float4 r = lane_target<KERNEL>(S, t >> 1, t & 1, p0, p1, thr, mc2);
      cand += (unsigned long long)(Msz[j - 1] + Msz[j] + Msz[j + 1] - 1);
      const int gs = O[4 * L3 + j] + i;
      float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p.out.upd) me = __ldg(p.rec + gs);
      if (KERNEL == PI_K_GAUSSIAN) {
        const float q = S[2 * (t >> 1) + 1].z * (1 - (t & 1)) + S[2 * (t >> 1) + 1].w * (t & 1);
        const float sc = -q * p.kp.inv_s2;
        write_output(p.out, g, gs, me, r.x, sc * r.y, sc * r.z, sc * r.w);
      } else {
        write_output(p.out, g, gs, me, r.x, 0.f, 0.f, 0.f);
      }
    }
    __syncthreads();
    ja = jb + 1;
  }
  // statistics: one atomic per block, spread over CAND_SLOTS counters
  for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
  __syncthreads();
  unsigned long long *red = reinterpret_cast<unsigned long long *>(ctl);  // ctl area is free now
  if (lane == 0) red[warp] = cand;
  __syncthreads();
  if (tid == 0) {
    unsigned long long tsum = 0;
    for (int w = 0; w < NT / 32; ++w) tsum += red[w];
    if (tsum) atomicAdd(&p.ctl->cand_slots[(blockIdx.x + blockIdx.y * 7 + blockIdx.z * 13) & (CAND_SLOTS - 1)], tsum);
    if (fallbacks) atomicAdd(&p.ctl->fallback_cells, fallbacks);
  }
}

template <int KERNEL, int NT>
cudaError_t launch_k(const XpParams &p, cudaStream_t s) {
  const size_t smem = xp_smem_bytes(p.L, p.cap);
  cudaError_t e =
      cudaFuncSetAttribute(k_interact_xpencil<KERNEL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
  p.L = a.tx_len > 0 ? a.tx_len : 64;
  if (p.L > 64) p.L = 64;
  if (p.L > g.nx) p.L = g.nx;
  const int threads = (a.threads == 64 || a.threads == 128 || a.threads == 256 || a.threads == 1024) ? a.threads : 512;
  if (a.tx_cap > 0) {
    p.cap = a.tx_cap;
  } else {
    // size the staging buffer for the mean occupancy of 9 rows x (L + 2) cells (+ padding)
    const double ppc = (double)a.n / (double)g.ncells;
    p.cap = (int)((9.0 * ppc * 1.1 + 4.0) * (p.L + 2) + 128.0);
  }
  p.cap = (p.cap + 31) & ~31;
  const size_t max_smem = 227 * 1024;
  while (xp_smem_bytes(p.L, p.cap) > max_smem && p.cap > 64) p.cap -= 32;
  if (threads == 64) return launch_nt<64>(p, s);
  if (threads == 128) return launch_nt<128>(p, s);
  if (threads == 256) return launch_nt<256>(p, s);
  if (threads == 1024) return launch_nt<1024>(p, s);
  return launch_nt<512>(p, s);
}

}  // namespace pi
