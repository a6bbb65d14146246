// a6.2: full load / All-in-SM (Alg. 4, §5.1), re-designed for sm_100a.
//
// As in the paper, one block owns a 3-D sub-box of target cells and stages the sub-box plus
// its one-cell ghost shell into shared memory ONCE; every interior cell is then reused by its
// 3^3 neighbours from shared memory (:236-239).  B200 specifics:
//
//   * the staged region is (Bx+2) x (By+2) x (Bz+2) cells; each of its (By+2)(Bz+2) X-rows is a
//     contiguous run of 16-B records in the cell-sorted array (X-fastest, :322-324), so the
//     whole sub-box arrives with (By+2)(Bz+2) TMA bulk copies (cp.async.bulk, mbarrier
//     completion) instead of one thread per particle (:283-284);
//   * the local offset of a staged row is the "prefix over gaps" of PAPER.md:321-327 (reading
//     R13, pinned by test_local_offsets_gap_reading): the rows are packed back to back, so
//     local(c) = Lst[row] + offsets[c] - offsets[first cell of the row];
//   * the paper sizes the sub-box from M_C (:240-244, :270-276) and needs a device->host
//     read-back; here the box dims are fixed at launch and the capacity from the mean density
//     (x1.25); a block whose staged count does not fit computes its targets from global memory
//     (the Par-Part-NoLoop path) instead -- no M_C, no host synchronisation;
//   * compute: one thread per PAIR of targets of one cell (packed f32x2 registers), the 27
//     candidate cells walked as 9 contiguous 3-cell runs of shared memory, every source a
//     broadcast scalar operand (12 packed-fp32 ops + 2 MUFU.EX2 per source and 2 candidates).
#include "cellsm.cuh"
#include "interact_common.cuh"

namespace pi {
namespace {

struct FlParams {
  long long n;
  const float4 *rec;
  const int32_t *offsets;
  Geom g;
  KParams kp;
  OutDesc out;
  DevCtl *ctl;
  int bx, by, bz;  // interior sub-box dims (cells)
  int cap;         // staged records
  int32_t *dense;  // cells of the boxes that do not fit: listed for the Par-Cell-SM pass
};

// smem: mbarrier (16 B) | ints: Lst[R+1] | O[R][Bx+3] | Ppre[C+1] | ctl[8] | S[cap] (16-B aligned)
//   R = (By+2)(Bz+2) staged rows, C = Bx By Bz interior cells
__host__ __device__ inline int fl_int_words(int bx, int by, int bz) {
  const int R = (by + 2) * (bz + 2), C = bx * by * bz;
  int ints = (R + 1) + R * (bx + 3) + (C + 1) + 8;
  return (ints + 3) & ~3;
}
__host__ __device__ inline size_t fl_smem_bytes(int bx, int by, int bz, int cap) {
  return 16 + (size_t)fl_int_words(bx, by, bz) * 4 + (size_t)cap * 16;
}

template <int KERNEL, int NT>
__global__ void __launch_bounds__(NT) k_interact_fullload(FlParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int bx = p.bx, by = p.by, bz = p.bz;
  const int BX3 = bx + 3;
  const int R = (by + 2) * (bz + 2), C = bx * by * bz;
  unsigned long long *bar = reinterpret_cast<unsigned long long *>(smem_raw);
  int *Lst = reinterpret_cast<int *>(smem_raw + 16);
  int *O = Lst + (R + 1);
  int *Ppre = O + R * BX3;
  int *ctl = Ppre + (C + 1);
  float4 *S = reinterpret_cast<float4 *>(smem_raw + 16 + fl_int_words(bx, by, bz) * 4);

  const Geom &g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int x0 = g.own_lo + blockIdx.x * bx, y0 = blockIdx.y * by, z0 = blockIdx.z * bz;  // owned cells only
  const int ex = min(bx, g.own_hi - x0), ey = min(by, g.ny - y0), ez = min(bz, g.nz - z0);  // interior extent
  const float thr = p.kp.rc2, mc2 = -p.kp.c2;
  unsigned long long cand = 0;

  if (tid == 0) mbar_init(bar, 1);
  // staged rows p = (yy, zz), yy in [y0-1, y0+by], zz in [z0-1, z0+bz]; cells x0-1 .. x0+bx+1
  for (int k = tid; k < R * BX3; k += NT) {
    const int r = k / BX3, j = k - r * BX3;
    const int yy = y0 - 1 + r % (by + 2), zz = z0 - 1 + r / (by + 2);
    int v = 0;
    if (yy >= 0 && yy < g.ny && zz >= 0 && zz < g.nz) {
      const int x = min(max(x0 - 1 + j, 0), g.nx);
      v = __ldg(p.offsets + (long long)g.nx * (yy + (long long)g.ny * zz) + x);
    }
    O[k] = v;
  }
  __syncthreads();
  if (warp == 0) {
    // local row starts: the prefix over the staged rows' lengths (gap reading, :321-327)
    int carry = 0;
    for (int r0 = 0; r0 < R; r0 += 32) {
      const int r = r0 + lane;
      const int len = r < R ? O[r * BX3 + BX3 - 1] - O[r * BX3] : 0;
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (r < R) Lst[r] = carry + incl - len;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) Lst[R] = carry;
  } else if (warp == 1) {
    // target pairs per interior cell (x fastest, then y, z) and their prefix
    int carry = 0;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      int np = 0;
      if (c < C) {
        const int cx = c % bx, cy = (c / bx) % by, cz = c / (bx * by);
        if (cx < ex && cy < ey && cz < ez) {
          const int r = (cy + 1) + (by + 2) * (cz + 1);
          np = (O[r * BX3 + cx + 2] - O[r * BX3 + cx + 1] + 1) >> 1;
        }
      }
      int incl = np;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (c < C) Ppre[c] = carry + incl - np;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) Ppre[C] = carry;
  }
  __syncthreads();
  const int total = Lst[R];
  const int npairs = Ppre[C];
  if (total > p.cap) {
    // the staged sub-box does not fit (dense input): its non-empty cells are listed for the
    // Par-Cell-SM pass that follows this kernel (cellsm.cuh, k_cellsm_list)
    for (int c = tid; c < C; c += NT) {
      const int cx = c % bx, cy = (c / bx) % by, cz = c / (bx * by);
      if (cx >= ex || cy >= ey || cz >= ez) continue;
      const long long home = (long long)g.nx * (y0 + cy + (long long)g.ny * (z0 + cz));
      const int t_lo = __ldg(p.offsets + home + x0 + cx), t_hi = __ldg(p.offsets + home + x0 + cx + 1);
      if (t_hi > t_lo) {
        const unsigned long long k = atomicAdd(&p.ctl->pad[0], 1ull);
        p.dense[k] = (int)(home + x0 + cx);
      }
    }
    if (tid == 0) atomicAdd(&p.ctl->fallback_cells, (unsigned long long)(ex * ey * ez));
  } else {
    // ---- stage: one TMA bulk copy per staged row
    if (tid == 0) mbar_arrive_expect_tx(bar, (unsigned)total * 16u);
    __syncthreads();
    for (int r = tid; r < R; r += NT) {
      const int len = Lst[r + 1] - Lst[r];
      if (len > 0) bulk_g2s(S + Lst[r], p.rec + O[r * BX3], (unsigned)len * 16u, bar);
    }
    mbar_wait(bar, 0);
    // ---- compute: one thread per target pair, 9 runs of 3 cells each
    for (int P = tid; P < npairs; P += NT) {
      int lo_ = 0, hi_ = C - 1;  // last cell with Ppre[c] <= P
      while (lo_ < hi_) {
        const int mid = (lo_ + hi_ + 1) >> 1;
        if (Ppre[mid] <= P) lo_ = mid; else hi_ = mid - 1;
      }
      const int c = lo_;
      const int i = P - Ppre[c];
      const int cx = c % bx, cy = (c / bx) % by, cz = c / (bx * by);
      const int rh = (cy + 1) + (by + 2) * (cz + 1);  // home staged row
      const int hbase = Lst[rh] - O[rh * BX3];
      const int nt = O[rh * BX3 + cx + 2] - O[rh * BX3 + cx + 1];
      const int t0 = hbase + O[rh * BX3 + cx + 1] + 2 * i;
      const int t1 = min(t0 + 1, hbase + O[rh * BX3 + cx + 1] + nt - 1);
      const float4 a0 = S[t0], a1 = S[t1];
      TgtPair tp;
      tp.x = pk(a0.x, a1.x);
      tp.y = pk(a0.y, a1.y);
      tp.z = pk(a0.z, a1.z);
      p2 phi = pk(0.f), fx = pk(0.f), fy = pk(0.f), fz = pk(0.f);
      int ncand = 0;
#pragma unroll 1
      for (int q9 = 0; q9 < 9; ++q9) {
        const int r = rh + (q9 % 3 - 1) + (by + 2) * (q9 / 3 - 1);
        const int base = Lst[r] - O[r * BX3];
        const int s0 = base + O[r * BX3 + cx], s1 = base + O[r * BX3 + cx + 3];  // cells cx-1 .. cx+1
        ncand += s1 - s0;
        int s = s0;
        for (; s + 2 <= s1; s += 2) {
          const float4 u = S[s], v = S[s + 1];
          tp_eval<KERNEL>(tp, u, thr, mc2, phi, fx, fy, fz, p.kp);
          tp_eval<KERNEL>(tp, v, thr, mc2, phi, fx, fy, fz, p.kp);
        }
        if (s < s1) tp_eval<KERNEL>(tp, S[s], thr, mc2, phi, fx, fy, fz, p.kp);
      }
      // identity exclusion (Alg. 1 :127)
      phi = pk(lo(phi) - tp_self<KERNEL>(tp, 0, a0, thr, mc2, p.kp), hi(phi));
      if (t1 != t0) phi = pk(lo(phi), hi(phi) - tp_self<KERNEL>(tp, 1, a1, thr, mc2, p.kp));
      if (KERNEL == PI_K_LOWFLOP) {  // the self pair also added the target's own position
        fx = pk(lo(fx) - a0.x, t1 != t0 ? hi(fx) - a1.x : hi(fx));
        fy = pk(lo(fy) - a0.y, t1 != t0 ? hi(fy) - a1.y : hi(fy));
        fz = pk(lo(fz) - a0.z, t1 != t0 ? hi(fz) - a1.z : hi(fz));
      }
      cand += (unsigned long long)(t1 - t0 + 1) * (unsigned long long)(ncand - 1);
      const int gs0 = O[rh * BX3 + cx + 1] + 2 * i;
      const float4 me0 = p.out.upd ? __ldg(p.rec + gs0) : a0;
      if (kern_wforce(KERNEL)) {
        const float c0 = a0.w * p.kp.f_ts;  // summed wf (x_t - x_s)
        write_output(p.out, g, gs0, me0, lo(phi) * p.kp.phi_scale, c0 * lo(fx), c0 * lo(fy), c0 * lo(fz));
      } else if (KERNEL == PI_K_LOWFLOP) {
        write_output(p.out, g, gs0, me0, lo(phi), lo(fx), lo(fy), lo(fz));
      } else {
        write_output(p.out, g, gs0, me0, lo(phi), 0.f, 0.f, 0.f);
      }
      if (t1 != t0) {
        const float4 me1 = p.out.upd ? __ldg(p.rec + gs0 + 1) : a1;
        if (kern_wforce(KERNEL)) {
          const float c1 = a1.w * p.kp.f_ts;
          write_output(p.out, g, gs0 + 1, me1, hi(phi) * p.kp.phi_scale, c1 * hi(fx), c1 * hi(fy), c1 * hi(fz));
        } else if (KERNEL == PI_K_LOWFLOP) {
          write_output(p.out, g, gs0 + 1, me1, hi(phi), hi(fx), hi(fy), hi(fz));
        } else {
          write_output(p.out, g, gs0 + 1, me1, hi(phi), 0.f, 0.f, 0.f);
        }
      }
    }
  }
  // statistics
  for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
  if (lane == 0 && cand)
    atomicAdd(&p.ctl->cand_slots[(blockIdx.x + 3 * blockIdx.y + 5 * blockIdx.z + warp) & (CAND_SLOTS - 1)], cand);
  (void)ctl;
}

template <int KERNEL, int NT>
cudaError_t launch_k(const FlParams &p, cudaStream_t s) {
  const size_t smem = fl_smem_bytes(p.bx, p.by, p.bz, p.cap);
  cudaError_t e = allow_max_smem(k_interact_fullload<KERNEL, NT>);
  if (e != cudaSuccess) return e;
  const int own = p.g.own_hi - p.g.own_lo;
  dim3 grid((own + p.bx - 1) / p.bx, (p.g.ny + p.by - 1) / p.by, (p.g.nz + p.bz - 1) / p.bz);
  k_interact_fullload<KERNEL, NT><<<grid, NT, smem, s>>>(p);
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_nt(const FlParams &p, cudaStream_t s) {
  switch (p.kp.kernel) {
    case PI_K_GAUSSIAN: return launch_k<PI_K_GAUSSIAN, NT>(p, s);
    case PI_K_INDICATOR: return launch_k<PI_K_INDICATOR, NT>(p, s);
    case PI_K_LJ: return launch_k<PI_K_LJ, NT>(p, s);
    case PI_K_LOWFLOP: return launch_k<PI_K_LOWFLOP, NT>(p, s);
    case PI_K_HIGHFLOP: return launch_k<PI_K_HIGHFLOP, NT>(p, s);
    default: return launch_k<PI_K_CANDIDATE, NT>(p, s);
  }
}

}  // namespace

cudaError_t launch_interact_fullload(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  FlParams p;
  p.n = a.n;
  p.rec = a.rec;
  p.offsets = a.offsets;
  p.g = g;
  p.kp = k;
  p.out = a.out;
  p.ctl = a.ctl;
  p.dense = a.dense;
  const double ppc = (double)a.n_est / (double)g.ncells;
  const size_t max_smem = 227 * 1024;
  if (a.fb[0] > 0 || a.fb[1] > 0 || a.fb[2] > 0) {
    p.bx = a.fb[0] > 0 ? a.fb[0] : 8;
    p.by = a.fb[1] > 0 ? a.fb[1] : 4;
    p.bz = a.fb[2] > 0 ? a.fb[2] : 4;
  } else {
    // the sub-box from the density (the paper sizes it from M_C):
    // the largest of these whose staged cells hold the mean occupancy (+25 %) in shared memory
    static const int boxes[][3] = {{8, 4, 4}, {4, 4, 4}, {4, 4, 2}, {4, 2, 2}, {2, 2, 2}, {2, 2, 1}, {2, 1, 1},
                                   {1, 1, 1}};
    // ... and, as the paper's shrink rule (:270-276), small enough for two blocks per SM
    int k = 0;
    const long long nblk_min = 2LL * 148;
    for (; k < 7; ++k) {
      const double st = (double)(boxes[k][0] + 2) * (boxes[k][1] + 2) * (boxes[k][2] + 2);
      const long long nblk = (long long)((g.own_hi - g.own_lo + boxes[k][0] - 1) / boxes[k][0]) *
                             ((g.ny + boxes[k][1] - 1) / boxes[k][1]) * ((g.nz + boxes[k][2] - 1) / boxes[k][2]);
      if (fl_smem_bytes(boxes[k][0], boxes[k][1], boxes[k][2], (int)(st * ppc * 1.25 + 64.0)) <= max_smem &&
          nblk >= nblk_min)
        break;
    }
    p.bx = boxes[k][0];
    p.by = boxes[k][1];
    p.bz = boxes[k][2];
  }
  p.bx = min(p.bx, g.own_hi - g.own_lo);
  p.by = min(p.by, g.ny);
  p.bz = min(p.bz, g.nz);
  // fewer than 27 staged cells cannot hold one target cell and its ghosts;
  // with the ghost shell always included here the smallest box is 1x1x1 (+ shell = 27 cells)
  const double staged = (double)(p.bx + 2) * (p.by + 2) * (p.bz + 2);
  p.cap = a.fb_cap > 0 ? a.fb_cap : (int)(staged * ppc * 1.25 + 64.0);
  p.cap = (p.cap + 31) & ~31;
  if (fl_smem_bytes(p.bx, p.by, p.bz, 64) > max_smem) return cudaErrorNotSupported;
  while (fl_smem_bytes(p.bx, p.by, p.bz, p.cap) > max_smem && p.cap > 64) p.cap -= 32;
  const int threads = a.threads == 128 ? 128 : (a.threads == 512 ? 512 : 256);
  cudaError_t e = threads == 128 ? launch_nt<128>(p, s) : (threads == 512 ? launch_nt<512>(p, s) : launch_nt<256>(p, s));
  if (e != cudaSuccess) return e;
  // the cells of the boxes that did not fit (usually none: one atomic per block)
  CsParams cp;
  cp.rec = a.rec;
  cp.pairs = a.pairs;
  cp.plane = a.pair_plane;
  cp.offsets = a.offsets;
  cp.from_rec = true;
  cp.list = a.dense;
  cp.g = g;
  cp.kp = k;
  cp.out = a.out;
  cp.ctl = a.ctl;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e2 = allow_max_smem(kern);
    if (e2 != cudaSuccess) return e2;
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, CS_SMEM);
    kern<<<sms * (occ > 0 ? occ : 1), 256, CS_SMEM, s>>>(cp);
    return cudaGetLastError();
  };
  const bool upd = a.out.upd != nullptr;
  switch (k.kernel) {
    case PI_K_GAUSSIAN: return upd ? go(k_cellsm_list<PI_K_GAUSSIAN, true>) : go(k_cellsm_list<PI_K_GAUSSIAN, false>);
    case PI_K_INDICATOR: return upd ? go(k_cellsm_list<PI_K_INDICATOR, true>) : go(k_cellsm_list<PI_K_INDICATOR, false>);
    case PI_K_LJ: return upd ? go(k_cellsm_list<PI_K_LJ, true>) : go(k_cellsm_list<PI_K_LJ, false>);
    case PI_K_LOWFLOP: return upd ? go(k_cellsm_list<PI_K_LOWFLOP, true>) : go(k_cellsm_list<PI_K_LOWFLOP, false>);
    case PI_K_HIGHFLOP: return upd ? go(k_cellsm_list<PI_K_HIGHFLOP, true>) : go(k_cellsm_list<PI_K_HIGHFLOP, false>);
    default: return upd ? go(k_cellsm_list<PI_K_CANDIDATE, true>) : go(k_cellsm_list<PI_K_CANDIDATE, false>);
  }
}

}  // namespace pi
