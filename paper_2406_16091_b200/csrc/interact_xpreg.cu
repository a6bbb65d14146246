// NEXT #1: X-pencil-reg, "pencil load with register storage" (PAPER.md:421-457,
// §5.3, Fig. "example-x-pencil-reg").
//
// As the paper describes it: the TARGETS of a sub-box of cells (Bx cells along X x By x Bz rows,
// "instead of having target cells organized as a pencil in the X direction, we can target a
// sub-box of cells", :446-447) are first loaded into registers, one thread per target (a few per
// thread here).  Then the (By+2)(Bz+2) source X-pencils around the box (each Bx + 2 cells long:
// the box's X range and its two ghost cells) are loaded into shared memory "one after the other"
// and the interactions computed after each load; the threads whose targets' rows are not adjacent
// to the staged pencil are idle for that pencil (:452-455).  A pencil that runs through the box
// holds the box's own targets: those records are "copied to the shared memory at the right
// iteration" from the registers instead of being read from global memory again (:438-442); only
// its two ghost cells come from global memory.
//
// Every source of the 27 cells of a target is met exactly once (one staged pencil per neighbour
// row, the target's 3-cell window in it), the arithmetic is the global baseline's (one scalar
// r^2, scalar_term), so the results are those of every other strategy.  A pencil longer than the
// staging buffer (dense regions) is staged in chunks; a box with more targets than the threads
// hold is processed in passes.  Not tuned for speed: the paper reports this variant is "not
// faster than the X-pencil approach in practice" (:423-424); it is here as the NEXT row,
// measured beside the others (bench.py "xpreg").
#include "interact_common.cuh"

namespace pi {
namespace {

constexpr int XR_THREADS = 256;
constexpr int XR_TPT = 4;        // targets held per thread (registers) per pass
constexpr int XR_SCAP = 2048;    // staged source records per chunk (32 KB)
constexpr int XR_MAXROWS = 64;   // By * Bz <= 64

struct XrParams {
  const float4 *rec;
  const int32_t *offsets;
  Geom g;
  KParams kp;
  OutDesc out;
  DevCtl *ctl;
  int bx, by, bz;          // box extents (cells)
  int nbx, nby, nbz;       // boxes per axis
};

__device__ __forceinline__ long long lin3(const Geom &g, int x, int y, int z) {
  return (long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z);
}

template <int KERNEL, bool UPD>
__global__ void __launch_bounds__(XR_THREADS) k_interact_xpreg(XrParams p) {
  __shared__ float4 S[XR_SCAP];
  __shared__ int rstart[XR_MAXROWS + 1];  // target prefix over the box's rows
  __shared__ int rslot[XR_MAXROWS];       // sorted slot of each row's first target
  const Geom &g = p.g;
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  const int bxi = b % p.nbx, byi = (b / p.nbx) % p.nby, bzi = b / (p.nbx * p.nby);
  const int x0 = g.own_lo + bxi * p.bx, x1 = min(x0 + p.bx, g.own_hi);  // target cells [x0, x1)
  const int y0 = byi * p.by, y1 = min(y0 + p.by, g.ny);
  const int z0 = bzi * p.bz, z1 = min(z0 + p.bz, g.nz);
  const int nry = y1 - y0, nrows = nry * (z1 - z0);
  if (tid == 0) {
    int acc = 0;
    for (int k = 0; k < nrows; ++k) {
      const int y = y0 + k % nry, z = z0 + k / nry;
      const int a = __ldg(p.offsets + lin3(g, x0, y, z)), e = __ldg(p.offsets + lin3(g, x1 - 1, y, z) + 1);
      rstart[k] = acc;
      rslot[k] = a;
      acc += e - a;
    }
    rstart[nrows] = acc;
  }
  __syncthreads();
  const int nt = rstart[nrows];
  const float thr = p.kp.rc2;
  unsigned long long cand = 0;
  for (int pass = 0; pass < nt; pass += XR_THREADS * XR_TPT) {
    // targets into registers: t = pass + tid + k XR_THREADS
    float4 me[XR_TPT];
    int slot[XR_TPT], ty[XR_TPT], tz[XR_TPT], tcx[XR_TPT];
    float acc[XR_TPT][4];
#pragma unroll
    for (int k = 0; k < XR_TPT; ++k) {
      const int t = pass + tid + k * XR_THREADS;
      slot[k] = -1;
      ty[k] = tz[k] = -9;
      tcx[k] = 0;
      acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.f;
      me[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < nt) {
        int row = 0;
        while (row + 1 < nrows && rstart[row + 1] <= t) ++row;
        slot[k] = rslot[row] + (t - rstart[row]);
        ty[k] = y0 + row % nry;
        tz[k] = z0 + row / nry;
        me[k] = __ldg(p.rec + slot[k]);
        bool bad = false;
        tcx[k] = cell_x(g, me[k].x, bad);
      }
    }
    // the source pencils one after the other (rows y0-1 .. y1, z0-1 .. z1, clamped: open box)
    for (int pz = max(z0 - 1, 0); pz <= min(z1, g.nz - 1); ++pz)
      for (int py = max(y0 - 1, 0); py <= min(y1, g.ny - 1); ++py) {
        const int xs0 = max(x0 - 1, 0), xs1 = min(x1, g.nx - 1);  // cells of the pencil (inclusive)
        const int pa = __ldg(p.offsets + lin3(g, xs0, py, pz)), pb = __ldg(p.offsets + lin3(g, xs1, py, pz) + 1);
        const bool inbox = py >= y0 && py < y1 && pz >= z0 && pz < z1;
        // the box's own records in this pencil: [ia, ib) (held in registers by their threads)
        int ia = pa, ib = pa;
        if (inbox) {
          ia = __ldg(p.offsets + lin3(g, x0, py, pz));
          ib = __ldg(p.offsets + lin3(g, x1 - 1, py, pz) + 1);
        }
        for (int ca = pa; ca < pb; ca += XR_SCAP) {
          const int cb = min(pb, ca + XR_SCAP);
          __syncthreads();  // the previous chunk is consumed
          for (int s = ca + tid; s < cb; s += XR_THREADS)
            if (s < ia || s >= ib) S[s - ca] = __ldg(p.rec + s);  // ghost cells (and out-of-box rows)
          if (inbox) {  // register -> shared memory: the targets of this row in this chunk
#pragma unroll
            for (int k = 0; k < XR_TPT; ++k)
              if (slot[k] >= ca && slot[k] < cb && ty[k] == py && tz[k] == pz) S[slot[k] - ca] = me[k];
            // (a row's targets beyond this pass are not in any register: load them)
            for (int s = max(ca, ia) + tid; s < min(cb, ib); s += XR_THREADS) {
              const int t = rstart[(py - y0) + nry * (pz - z0)] + (s - ia);
              if (t < pass || t >= pass + XR_THREADS * XR_TPT) S[s - ca] = __ldg(p.rec + s);
            }
          }
          __syncthreads();
          // the threads whose targets' rows are adjacent to this pencil compute, the others idle
#pragma unroll
          for (int k = 0; k < XR_TPT; ++k) {
            if (slot[k] < 0 || abs(ty[k] - py) > 1 || abs(tz[k] - pz) > 1) continue;
            const int wa = __ldg(p.offsets + lin3(g, max(tcx[k] - 1, 0), py, pz));
            const int wb = __ldg(p.offsets + lin3(g, min(tcx[k] + 1, g.nx - 1), py, pz) + 1);
            if (ca == pa) cand += (unsigned long long)(wb - wa);
            const int s0 = max(wa, ca), s1 = min(wb, cb);
            for (int s = s0; s < s1; ++s) {
              if (s == slot[k]) continue;  // identity (Alg. 1 :127)
              const float4 o = S[s - ca];
              const float dx = me[k].x - o.x, dy = me[k].y - o.y, dz = me[k].z - o.z;
              const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
              if (KERNEL == PI_K_CANDIDATE) {
                acc[k][0] += o.w;
              } else if (r2 < thr) {
                if (KERNEL == PI_K_INDICATOR) {
                  acc[k][0] += o.w;
                } else if (KERNEL == PI_K_LOWFLOP) {
                  acc[k][0] += lf_sum(o.x, o.y, o.z);
                  acc[k][1] += o.x;
                  acc[k][2] += o.y;
                  acc[k][3] += o.z;
                } else {
                  float w, wf;
                  scalar_term<KERNEL>(p.kp, r2, o.w, w, wf);
                  acc[k][0] += w;
                  acc[k][1] = fmaf(wf, dx, acc[k][1]);
                  acc[k][2] = fmaf(wf, dy, acc[k][2]);
                  acc[k][3] = fmaf(wf, dz, acc[k][3]);
                }
              }
            }
          }
        }
      }
#pragma unroll
    for (int k = 0; k < XR_TPT; ++k) {
      if (slot[k] < 0) continue;
      cand -= 1;  // the self pair is not a candidate
      float phi = acc[k][0], fx = acc[k][1], fy = acc[k][2], fz = acc[k][3];
      if (kern_wforce(KERNEL)) {
        const float s = me[k].w * p.kp.f_ts;  // summed wf (x_t - x_s)
        phi *= p.kp.phi_scale;
        fx *= s;
        fy *= s;
        fz *= s;
      } else if (KERNEL != PI_K_LOWFLOP) {
        fx = fy = fz = 0.f;
      }
      write_output<UPD>(p.out, g, slot[k], me[k], phi, fx, fy, fz);
    }
  }
  for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
  if ((tid & 31) == 0 && cand) atomicAdd(&p.ctl->cand_slots[(blockIdx.x * 8 + (tid >> 5)) & (CAND_SLOTS - 1)], cand);
}

template <bool UPD>
cudaError_t launch_u(const XrParams &p, cudaStream_t s) {
  const int blocks = p.nbx * p.nby * p.nbz;
  switch (p.kp.kernel) {
    case PI_K_GAUSSIAN: k_interact_xpreg<PI_K_GAUSSIAN, UPD><<<blocks, XR_THREADS, 0, s>>>(p); break;
    case PI_K_INDICATOR: k_interact_xpreg<PI_K_INDICATOR, UPD><<<blocks, XR_THREADS, 0, s>>>(p); break;
    case PI_K_LJ: k_interact_xpreg<PI_K_LJ, UPD><<<blocks, XR_THREADS, 0, s>>>(p); break;
    case PI_K_LOWFLOP: k_interact_xpreg<PI_K_LOWFLOP, UPD><<<blocks, XR_THREADS, 0, s>>>(p); break;
    case PI_K_HIGHFLOP: k_interact_xpreg<PI_K_HIGHFLOP, UPD><<<blocks, XR_THREADS, 0, s>>>(p); break;
    default: k_interact_xpreg<PI_K_CANDIDATE, UPD><<<blocks, XR_THREADS, 0, s>>>(p); break;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_interact_xpreg(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  if (!a.rec) return cudaErrorNotSupported;
  XrParams p;
  p.rec = a.rec;
  p.offsets = a.offsets;
  p.g = g;
  p.kp = k;
  p.out = a.out;
  p.ctl = a.ctl;
  // box: 2 x 2 rows, Bx cells along X so that a box holds ~512 targets at the mean density
  // (tuning: xpencil_len = Bx)
  const double ppc = (double)a.n_est / (double)(g.ncells > 0 ? g.ncells : 1);
  p.by = min(2, g.ny);
  p.bz = min(2, g.nz);
  int bx = a.tx_len > 0 ? a.tx_len : (int)(512.0 / (4.0 * (ppc > 0.5 ? ppc : 0.5)));
  bx = max(1, min(bx, 64));
  const int own = g.own_hi - g.own_lo;
  p.bx = min(bx, own);
  p.nbx = (own + p.bx - 1) / p.bx;
  p.nby = (g.ny + p.by - 1) / p.by;
  p.nbz = (g.nz + p.bz - 1) / p.bz;
  if ((long long)p.nbx * p.nby * p.nbz > 0x7fffffffLL) return cudaErrorNotSupported;
  return a.out.upd ? launch_u<true>(p, s) : launch_u<false>(p, s);
}

}  // namespace pi
