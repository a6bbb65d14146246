// NEXT #4: the Newton-3rd-law HALF-SHELL, as a selectable strategy
// (PI_A_HALF).  The paper's kernels evaluate every ordered pair twice, once from each side
// (Alg. 1: "for each target, for each source of the 27 cells"); the terms of
// every kernel here are pairwise symmetric or antisymmetric -- phi_i gets q_j K(r_ij), phi_j gets
// q_i K(r_ij); F_i = q_i q_j G(r_ij) (x_i - x_j) = -F_j (§2, Eq. (1) :578-582) --
// so each unordered pair can be evaluated once and credited to both particles.
//
// Walk: one thread per target t in an owned cell (the global baseline's walk, Alg. 1), over the
// UPPER half of its 27-cell neighbourhood only:
//   * the 4 neighbour rows with (dz > 0) or (dz = 0 and dy > 0): their whole 3-cell run;
//   * its own row: the sources after t in the sorted order up to the end of cell cx + 1 -- the
//     rest of its own cell (s > t: each same-cell pair once, no self pair) and cell cx + 1;
//   * the other 4 rows and cell cx - 1 of its own row only where they are GHOST cells of a slab
//     (a8): a ghost is never a target, so a pair with a ghost is evaluated by the owned side.
// Every pair of neighbours with at least one owned particle is then evaluated exactly once.
// The target's sums stay in registers; each source's share (the same kernel value with the
// target's q, the force negated) goes to the source's slot of the sorted-order output with a
// vector reduction (REDG.ADD.F32x4, inside the cutoff only), as does the target's own total at
// the end (it also receives shares from the lower half).  `k_half_finish` then scales the sums
// (q_i f_ts, phi_scale) and writes the outputs / pi_step update like every other strategy.
// Sources in ghost cells get no share (their owner computes them).
//
// The candidates counted for the metric (R4) are the 27-cell ordered candidates of each
// target, as for every strategy.  The summation order differs from the one-sided kernels (the
// tolerance of C10 covers it); the integer kernels (INDICATOR, CANDIDATE with q = 1) stay exact.
#include "interact_common.cuh"

namespace pi {
namespace {

constexpr int HALF_THREADS = 128;

__device__ __forceinline__ void red_add4(float4 *p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// One unordered pair (t, s) at d = x_t - x_s, r2: t's terms added to acc, s's share returned.
// Returns false when the pair contributes nothing (outside the cutoff).
template <int KERNEL>
__device__ __forceinline__ bool pair_terms(const KParams &kp, const float4 &me, const float4 &o, float dx, float dy,
                                           float dz, float r2, float4 &acc, float4 &rs) {
  if (KERNEL != PI_K_CANDIDATE && !(r2 < kp.rc2)) return false;
  if (KERNEL == PI_K_CANDIDATE || KERNEL == PI_K_INDICATOR) {
    acc.x += o.w;
    rs = make_float4(me.w, 0.f, 0.f, 0.f);
  } else if (KERNEL == PI_K_LOWFLOP) {  // c_ij = (x_j + y_j + z_j, x_j, y_j, z_j)
    acc.x += lf_sum(o.x, o.y, o.z);
    acc.y += o.x;
    acc.z += o.y;
    acc.w += o.z;
    rs = make_float4(lf_sum(me.x, me.y, me.z), me.x, me.y, me.z);
  } else {
    float w, wf;  // the kernel values for a unit source value: w (phi), wf (force weight)
    scalar_term<KERNEL>(kp, r2, 1.f, w, wf);
    const float ws = o.w * wf, wt = me.w * wf;
    acc.x = fmaf(o.w, w, acc.x);
    acc.y = fmaf(ws, dx, acc.y);
    acc.z = fmaf(ws, dy, acc.z);
    acc.w = fmaf(ws, dz, acc.w);
    rs = make_float4(me.w * w, -wt * dx, -wt * dy, -wt * dz);  // F_s: (x_s - x_t) = -d
  }
  return true;
}

template <int KERNEL>
__global__ void __launch_bounds__(HALF_THREADS) k_interact_half(long long n, const float4 *__restrict__ rec,
                                                                const int32_t *__restrict__ offsets, Geom g,
                                                                KParams kp, float4 *sums, DevCtl *ctl,
                                                                const long long *n_dev) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
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
    // is cell cx - 1 / cx + 1 a ghost cell (slabs; none on one GPU)?
    const bool ghost_lo = xlo < g.own_lo, ghost_hi = xhi >= g.own_hi;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int dz = -1; dz <= 1; ++dz) {
      const int z = cz + dz;
      if (z < 0 || z >= g.nz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= g.ny) continue;
        const long long row = (long long)g.nx * (y + (long long)g.ny * z);
        const int lo = __ldg(offsets + row + xlo);
        const int hi = __ldg(offsets + row + xhi + 1);
        cand += (unsigned long long)(hi - lo);  // the 27-cell candidates (R4), every row
        const bool upper = dz > 0 || (dz == 0 && dy > 0);
        const bool home = dz == 0 && dy == 0;
        // the runs of this row evaluated from t: [a0, e0) with shares, [a1, e1) ghosts (no share)
        int a0 = 0, e0 = 0, a1 = 0, e1 = 0;
        if (upper) {
          a0 = ghost_lo ? __ldg(offsets + row + xlo + 1) : lo;
          e0 = ghost_hi ? __ldg(offsets + row + xhi) : hi;
        } else if (home) {
          a0 = (int)t + 1;
          e0 = ghost_hi ? __ldg(offsets + row + xhi) : hi;
        }
        // ghost cells at either end of the window: evaluated from t in every row (no share)
        if (ghost_lo) {
          a1 = lo;
          e1 = __ldg(offsets + row + xlo + 1);
        }
        for (int pass = 0; pass < 3; ++pass) {
          int s0, s1;
          if (pass == 0) { s0 = a0; s1 = e0; }
          else if (pass == 1) { s0 = a1; s1 = e1; }
          else if (ghost_hi) { s0 = __ldg(offsets + row + xhi); s1 = hi; }
          else break;
          const bool share = pass == 0;
          for (int s = s0; s < s1; ++s) {
            const float4 o = __ldg(rec + s);
            const float dx = me.x - o.x, dy2 = me.y - o.y, dz2 = me.z - o.z;
            const float r2 = fmaf(dz2, dz2, fmaf(dy2, dy2, dx * dx));
            float4 rs;
            if (pair_terms<KERNEL>(kp, me, o, dx, dy2, dz2, r2, acc, rs) && share)
              red_add4(sums + s, rs.x, rs.y, rs.z, rs.w);
          }
        }
      }
    }
    cand -= 1;  // self
    red_add4(sums + t, acc.x, acc.y, acc.z, acc.w);
  }
  for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
  if ((threadIdx.x & 31) == 0 && cand)
    atomicAdd(&ctl->cand_slots[(blockIdx.x * 4 + (threadIdx.x >> 5)) & (CAND_SLOTS - 1)], cand);
}

// The summed terms of each owned particle -> the outputs (scales as the one-sided kernels).
// `sums` is the sorted-order output array itself (write_output rewrites the slot).
template <int KERNEL, bool UPD>
__global__ void __launch_bounds__(256) k_half_finish(long long n, const float4 *__restrict__ rec, Geom g, KParams kp,
                                                     OutDesc out, const long long *n_dev) {
  if (n_dev) n = *n_dev;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const float4 me = __ldg(rec + t);
    bool bad = false;
    const int cx = cell_x(g, me.x, bad);
    if (cx < g.own_lo || cx >= g.own_hi) continue;
    float4 a = out.sorted[t];
    if (kern_wforce(KERNEL)) {
      const float sc = me.w * kp.f_ts;  // summed wf (x_t - x_s)
      a = make_float4(a.x * kp.phi_scale, a.y * sc, a.z * sc, a.w * sc);
    } else if (KERNEL != PI_K_LOWFLOP) {
      a.y = a.z = a.w = 0.f;
    }
    write_output<UPD>(out, g, (int)t, me, a.x, a.y, a.z, a.w);
  }
}

template <int KERNEL>
cudaError_t launch_k(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  // the sums accumulate in the sorted-order output array: zero its slots first
  cudaError_t e = cudaMemsetAsync(a.out.sorted, 0, sizeof(float4) * (size_t)a.n, s);
  if (e != cudaSuccess) return e;
  const int blocks = (int)((a.n + HALF_THREADS - 1) / HALF_THREADS);
  k_interact_half<KERNEL><<<blocks, HALF_THREADS, 0, s>>>(a.n, a.rec, a.offsets, g, k, a.out.sorted, a.ctl, a.n_dev);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const long long nb = (a.n + 255) / 256;
  const int fb = (int)(nb < 148LL * 16 ? nb : 148LL * 16);
  if (a.out.upd)
    k_half_finish<KERNEL, true><<<fb, 256, 0, s>>>(a.n, a.rec, g, k, a.out, a.n_dev);
  else
    k_half_finish<KERNEL, false><<<fb, 256, 0, s>>>(a.n, a.rec, g, k, a.out, a.n_dev);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_interact_half(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  if (!a.rec) return cudaErrorNotSupported;
  switch (k.kernel) {
    case PI_K_GAUSSIAN: return launch_k<PI_K_GAUSSIAN>(g, k, a, s);
    case PI_K_INDICATOR: return launch_k<PI_K_INDICATOR>(g, k, a, s);
    case PI_K_LJ: return launch_k<PI_K_LJ>(g, k, a, s);
    case PI_K_LOWFLOP: return launch_k<PI_K_LOWFLOP>(g, k, a, s);
    case PI_K_HIGHFLOP: return launch_k<PI_K_HIGHFLOP>(g, k, a, s);
    default: return launch_k<PI_K_CANDIDATE>(g, k, a, s);
  }
}

}  // namespace pi
