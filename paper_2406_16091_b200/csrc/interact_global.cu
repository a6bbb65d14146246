// a6.1: Par-Part-NoLoop, the paper's global-memory baseline (Alg. 1, PAPER.md:105-137,
// §4.1): one thread per target particle, "no loop over the particles, and no use of the
// shared memory" (:109); the sources of the 27 neighbour cells are read from global
// memory through L1/L2 (:110); "part_source != part_target" (:127) is an identity test;
// 128 threads per block (:556).
//
// B200 specifics: the cell-sorted state is one 16-B (x, y, z, q) record per particle, so a
// source is one LDG.128; the 3 cells of a neighbour row (dx = -1..1) are contiguous in the
// X-fastest order, so the 27 cells are walked as 9 contiguous runs.
// r^2 is computed directly (dx^2 + dy^2 + dz^2) and the cutoff test is strict (<).
#include "interact_common.cuh"

namespace pi {
namespace {

constexpr int PPNL_THREADS = 128;

template <int KERNEL>
__global__ void __launch_bounds__(PPNL_THREADS) k_interact_global(long long n, const float4 *__restrict__ rec,
                                                                  const int32_t *__restrict__ offsets, Geom g,
                                                                  KParams kp, OutDesc out, DevCtl *ctl,
                                                                  const long long *n_dev) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long cand = 0;
  if (n_dev) n = *n_dev;
  bool owned = false;
  float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
  int cx = 0;
  if (t < n) {
    me = __ldg(rec + t);
    bool bad = false;
    cx = cell_x(g, me.x, bad);
    owned = cx >= g.own_lo && cx < g.own_hi;  // ghost particles are sources only
  }
  if (owned) {
    bool bad = false;
    const int cy = cell_coord(me.y, g.oy, g.inv_w, g.ny, bad);
    const int cz = cell_coord(me.z, g.oz, g.inv_w, g.nz, bad);
    const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.nx - 1);
    float phi = 0.f, fx = 0.f, fy = 0.f, fz = 0.f;
    for (int dz = -1; dz <= 1; ++dz) {
      const int z = cz + dz;
      if (z < 0 || z >= g.nz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= g.ny) continue;
        const long long row = (long long)g.nx * (y + (long long)g.ny * z);
        const int lo = __ldg(offsets + row + xlo);
        const int hi = __ldg(offsets + row + xhi + 1);
        cand += (unsigned long long)(hi - lo);
        for (int s = lo; s < hi; ++s) {
          if (s == t) continue;
          const float4 o = __ldg(rec + s);
          const float dx = me.x - o.x, dy2 = me.y - o.y, dz2 = me.z - o.z;
          const float r2 = fmaf(dz2, dz2, fmaf(dy2, dy2, dx * dx));
          if (KERNEL == PI_K_CANDIDATE) {
            phi += o.w;
          } else if (r2 < kp.rc2) {
            if (KERNEL == PI_K_INDICATOR) {
              phi += o.w;
            } else if (KERNEL == PI_K_LOWFLOP) {
              phi += lf_sum(o.x, o.y, o.z);
              fx += o.x;
              fy += o.y;
              fz += o.z;
            } else {
              float w, wf;
              scalar_term<KERNEL>(kp, r2, o.w, w, wf);
              phi += w;
              fx = fmaf(wf, dx, fx);
              fy = fmaf(wf, dy2, fy);
              fz = fmaf(wf, dz2, fz);
            }
          }
        }
      }
    }
    cand -= 1;  // self
    if (kern_wforce(KERNEL)) {
      const float s = me.w * kp.f_ts;  // summed wf (x_t - x_s)
      phi *= kp.phi_scale;
      fx *= s; fy *= s; fz *= s;
    } else if (KERNEL == PI_K_LOWFLOP) {
    } else {
      fx = fy = fz = 0.f;
    }
    write_output(out, g, (int)t, me, phi, fx, fy, fz);
  }
  // candidates (C) for the statistics
  for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
  if ((threadIdx.x & 31) == 0 && cand) atomicAdd(&ctl->cand_slots[(blockIdx.x * 4 + (threadIdx.x >> 5)) & (CAND_SLOTS - 1)], cand);
}

// P (SURVEY.md §5 statistics): the cutoff pairs of the current sorted state, counted with the
// global baseline's walk and arithmetic (r^2 of the fp32 differences, strict r < r_c).
__global__ void __launch_bounds__(PPNL_THREADS) k_count_pairs(long long n, const float4 *__restrict__ rec,
                                                              const float4 *__restrict__ pairs, long long plane,
                                                              const int32_t *__restrict__ offsets, Geom g, float rc2,
                                                              DevCtl *ctl, const long long *n_dev) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (n_dev) n = *n_dev;
  unsigned long long cnt = 0;
  if (t < n) {
    const float4 me = sorted_rec(rec, pairs, plane, (int)t);
    bool bad = false;
    const int cx = cell_x(g, me.x, bad);
    if (cx >= g.own_lo && cx < g.own_hi) {
      const int cy = cell_coord(me.y, g.oy, g.inv_w, g.ny, bad);
      const int cz = cell_coord(me.z, g.oz, g.inv_w, g.nz, bad);
      const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.nx - 1);
      for (int dz = -1; dz <= 1; ++dz) {
        const int z = cz + dz;
        if (z < 0 || z >= g.nz) continue;
        for (int dy = -1; dy <= 1; ++dy) {
          const int y = cy + dy;
          if (y < 0 || y >= g.ny) continue;
          const long long row = (long long)g.nx * (y + (long long)g.ny * z);
          const int lo = __ldg(offsets + row + xlo), hi = __ldg(offsets + row + xhi + 1);
          for (int s = lo; s < hi; ++s) {
            if (s == t) continue;
            const float4 o = sorted_rec(rec, pairs, plane, s);
            const float dx = me.x - o.x, dy2 = me.y - o.y, dz2 = me.z - o.z;
            cnt += fmaf(dz2, dz2, fmaf(dy2, dy2, dx * dx)) < rc2;
          }
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&ctl->pairs, cnt);
}

}  // namespace

cudaError_t launch_count_pairs(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(&a.ctl->pairs, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess || a.n <= 0) return e;
  const int blocks = (int)((a.n + PPNL_THREADS - 1) / PPNL_THREADS);
  k_count_pairs<<<blocks, PPNL_THREADS, 0, s>>>(a.n, a.rec, a.pairs, a.pair_plane, a.offsets, g, k.rc2, a.ctl,
                                                a.n_dev);
  return cudaGetLastError();
}

cudaError_t launch_interact_global(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  int blocks = (int)((a.n + PPNL_THREADS - 1) / PPNL_THREADS);
  switch (k.kernel) {
    case PI_K_GAUSSIAN:
      k_interact_global<PI_K_GAUSSIAN><<<blocks, PPNL_THREADS, 0, s>>>(a.n, a.rec, a.offsets, g, k, a.out, a.ctl,
                                                                        a.n_dev);
      break;
    case PI_K_INDICATOR:
      k_interact_global<PI_K_INDICATOR><<<blocks, PPNL_THREADS, 0, s>>>(a.n, a.rec, a.offsets, g, k, a.out, a.ctl,
                                                                         a.n_dev);
      break;
    case PI_K_LJ:
      k_interact_global<PI_K_LJ><<<blocks, PPNL_THREADS, 0, s>>>(a.n, a.rec, a.offsets, g, k, a.out, a.ctl, a.n_dev);
      break;
    case PI_K_LOWFLOP:
      k_interact_global<PI_K_LOWFLOP><<<blocks, PPNL_THREADS, 0, s>>>(a.n, a.rec, a.offsets, g, k, a.out, a.ctl,
                                                                       a.n_dev);
      break;
    case PI_K_HIGHFLOP:
      k_interact_global<PI_K_HIGHFLOP><<<blocks, PPNL_THREADS, 0, s>>>(a.n, a.rec, a.offsets, g, k, a.out, a.ctl,
                                                                        a.n_dev);
      break;
    default:
      k_interact_global<PI_K_CANDIDATE><<<blocks, PPNL_THREADS, 0, s>>>(a.n, a.rec, a.offsets, g, k, a.out, a.ctl,
                                                                         a.n_dev);
  }
  return cudaGetLastError();
}

}  // namespace pi
