// a6.3: X-pencil (Alg. 5, §5.2) with SUB-CELL-INTERLEAVED staging (r02,
// tuning xpencil_layout = 1; the default is interact_xpencil.cu's pencil-by-pencil layout, which
// measured faster: DESIGN.md §6).
//
// The paper stages the 9 neighbour pencils of a target pencil and walks, per target, the
// 3-cell window of each (:398-407).  r01 staged the pencils back to back, so a target's
// candidates were 9 separate runs -- 9 loops per target whose trip counts differ from lane to
// lane (25.4 of 32 lanes active) plus per-run bounds and tail code (~25 % of the instructions).
// Here the producer stages the item's records X-SUB-CELL-MAJOR: for every X sub-cell position k
// along the segment (binning order R18), the records of that sub-cell in the 9 pencils, one after
// the other.  A target's candidates -- the sub-cells [klo, khi] within r_c along X in all 9
// pencils (R18) -- are then ONE contiguous range of the staged buffer: one loop per target,
// no run bounds, no out-of-run halves (record granularity), and the lanes' trip counts differ
// only by the Poisson noise of their windows.
//
//   * staging: every (sub-cell, pencil) run of 16-B records is contiguous in the cell-sorted
//     record array (X-fastest); a single producer warp copies them with 16-B cp.async (the runs
//     are ~2 records: TMA bulk copies that small were measured too slow), each lane a chunk of
//     sub-cell positions (prefix over the runs by a warp scan), the staged start of every
//     sub-cell position in a small table; the slot's mbarrier completes when all 32 lanes'
//     copies have landed (cp.async.mbarrier.arrive);
//   * compute: one thread per PAIR of consecutive sorted targets (packed f32x2 over the two
//     targets, the source a broadcast scalar: 12 packed-fp32 ops + 2 MUFU.EX2 per staged record),
//     the union of the two targets' windows (consecutive targets share their X sub-cell or are
//     adjacent); a staged record is read once (LDS.128) for both targets;
//   * everything else as r01: persistent blocks, slots handed over with full/empty mbarriers, no
//     block-wide barrier, slot capacity from shared memory (rounds along X, dense cells listed for
//     the Par-Cell-SM pass), the 27-cell candidates counted by the producer (the unit of the
//     metric, R4), the pi_step update fused into the epilogue.
#include "cellsm.cuh"
#include "interact_common.cuh"

namespace pi {
namespace {

constexpr int MAX_SLOTS2 = 4;
constexpr int META2 = 16;

struct Xp2Params {
  const float4 *rec;        // cell-sorted records (x, y, z, q)
  const int32_t *offsets;   // per cell
  const int32_t *foffsets;  // per fine cell (X sub-cell), the sorted order
  Geom g;
  KParams kp;
  OutDesc out;
  DevCtl *ctl;
  int L, sx, capr, nslot;   // segment length, X sub-cells, staged records per slot, slots
  int32_t *dense;
  int nseg;
  long long nitems;
};

// Slot: R[capr] float4 | meta[16] | SK[KS]  (KS = (L + 2) sx + 1: staged start of each sub-cell
// position k of the item; k = 0 is sub-cell 0 of cell x0 - 1)
// meta: 0 stop, 1 ja, 2 jb, 3 ntargets, 4 x0, 5 cy | cz << 16, 6 batch counter, 7 t0 (global
//       sorted index of the round's first target)
__host__ __device__ inline int lf2(int L, int sx) { return (L + 2) * sx + 1; }
__host__ __device__ inline int slot2_words(int L, int sx) { return (META2 + lf2(L, sx) + 3) & ~3; }
__host__ __device__ inline size_t slot2_bytes(int L, int capr, int sx) {
  return (size_t)capr * 16 + (size_t)slot2_words(L, sx) * 4;
}
// + two producer tables (prefetch stage and current item) of 9 LF ints
__host__ __device__ inline size_t tables2_bytes(int L, int sx) { return (((size_t)18 * lf2(L, sx) * 4) + 15) & ~(size_t)15; }
__host__ __device__ inline size_t xp2_smem_bytes(int L, int capr, int sx, int nslot) {
  return 128 + nslot * slot2_bytes(L, capr, sx) + tables2_bytes(L, sx);
}

struct Slot2 {
  float4 *R;
  int *meta, *SK;
};
__device__ __forceinline__ Slot2 slot2_at(unsigned char *base, int L, int capr, int sx, int s) {
  unsigned char *u = base + (size_t)s * slot2_bytes(L, capr, sx);
  Slot2 sl;
  sl.R = reinterpret_cast<float4 *>(u);
  sl.meta = reinterpret_cast<int *>(u + (size_t)capr * 16);
  sl.SK = sl.meta + META2;
  return sl;
}

__device__ __forceinline__ void mbar_arrive2(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async4_2(int *dst, const int *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}

__device__ __forceinline__ void item_geom2(const Xp2Params &p, long long item, int &x0, int &Lseg, int &cy, int &cz) {
  const int seg = (int)(item % p.nseg);
  const long long row = item / p.nseg;
  cy = (int)(row % p.g.ny);
  cz = (int)(row / p.g.ny);
  x0 = p.g.own_lo + seg * p.L;
  Lseg = min(p.L, p.g.own_hi - x0);
}
// fine offsets of the 9 pencils of `item` at the sub-cell boundaries of cells x0-1 .. x0+L
// (rows outside the grid are empty) -> stage[9][LF], asynchronously (as r01)
__device__ __forceinline__ void prefetch2(const Xp2Params &p, long long item, int *stage) {
  const int lane = threadIdx.x & 31;
  const int LF = lf2(p.L, p.sx), sx = p.sx;
  const Geom &g = p.g;
  int x0, Lseg, cy, cz;
  item_geom2(p, item, x0, Lseg, cy, cz);
  const int nxf = g.nx * sx;
  for (int k = lane; k < LF; k += 32) {
    const int bf = min(max((x0 - 1) * sx + k, 0), nxf);
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const int y = cy + (r % 3) - 1, z = cz + (r / 3) - 1;
      const bool ok = y >= 0 && y < g.ny && z >= 0 && z < g.nz;
      cp_async4_2(stage + r * LF + k, p.foffsets + (ok ? (long long)nxf * (y + (long long)g.ny * z) + bf : 0), ok);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// the largest jb <= Lseg whose 9 pencils (cells ja-1 .. jb+1) fit capr records (jb < ja: cell
// ja's window alone does not fit)
__device__ int choose_round2(const Xp2Params &p, const int *O, int ja, int Lseg) {
  const int lane = threadIdx.x & 31;
  const int LF = lf2(p.L, p.sx), sx = p.sx;
  int jb = ja - 1;
  for (int j0 = ja; j0 <= Lseg; j0 += 32) {
    const int j = j0 + lane;
    int tot = 0;
    if (j <= Lseg) {
#pragma unroll
      for (int r = 0; r < 9; ++r) tot += O[r * LF + (j + 2) * sx] - O[r * LF + (ja - 1) * sx];
    }
    const unsigned b = __ballot_sync(0xffffffffu, j <= Lseg && tot <= p.capr);
    jb += __popc(b);
    if (b != 0xffffffffu) break;
  }
  return jb;
}

// UPD: pi_step (update + carried counts in the epilogue).  Warps 0 .. NC-1 consume; warps NC ..
// NC+NP-1 produce: warp NC runs the item / round logic and the tables, then all NP producer warps
// copy the round's records (a named barrier hands the job over).
constexpr int NP2 = 8;
template <int KERNEL, int NC, bool UPD>
__global__ void __launch_bounds__((NC + NP2) * 32, 1) k_interact_xpencil2(Xp2Params p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int NSLOT = p.nslot;
  unsigned long long *full = reinterpret_cast<unsigned long long *>(smem_raw);
  unsigned long long *empty = full + MAX_SLOTS2;
  unsigned char *slots = smem_raw + 128;
  const int L = p.L, sx = p.sx, LF = lf2(L, sx);
  const Geom &g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long cand = 0, fallbacks = 0;
  int *stage = reinterpret_cast<int *>(slots + (size_t)NSLOT * slot2_bytes(L, p.capr, sx));
  int *O = stage + 9 * LF;  // the current item's table

  if (tid == 0) {
    for (int k = 0; k < NSLOT; ++k) {
      mbar_init(&full[k], 32 * NP2);  // every producer lane (its cp.async copies landed)
      mbar_init(&empty[k], NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp > NC) {
    // ======================== producer helpers: copy the records ========================
    const int pl = (warp - NC) * 32 + lane;  // producer lane 0 .. 32 NP - 1
    for (unsigned use = 0;; ++use) {
      const int s = use % NSLOT;
      const Slot2 sl = slot2_at(slots, L, p.capr, sx, s);
      asm volatile("bar.sync 1, %0;" ::"r"(32 * NP2) : "memory");  // the job of slot s is posted
      if (sl.meta[0]) {
        mbar_arrive2(&full[s]);
        break;
      }
      const int kb = sl.meta[8], ke = sl.meta[9], nk = ke - kb, chunk = (nk + 32 * NP2 - 1) / (32 * NP2);
      for (int k = min(ke, kb + pl * chunk), k1 = min(ke, kb + (pl + 1) * chunk); k < k1; ++k) {
        int base = sl.SK[k];
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          const int a = O[r * LF + k], n = O[r * LF + k + 1] - a;
          for (int o = 0; o < n; ++o) cp_async16(sl.R + base + o, p.rec + a + o);
          base += n;
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      asm volatile("bar.sync 2, %0;" ::"r"(32 * NP2) : "memory");  // done with the item table O
    }
  } else if (warp == NC) {
    // ================================ producer ================================
    long long item = -1, next = 0;
    int x0 = 0, Lseg = 0, cy = 0, cz = 0, ja = 1;
    if (lane == 0) next = (long long)atomicAdd(&p.ctl->xp_items, 1ull);
    next = __shfl_sync(0xffffffffu, next, 0);
    if (next < p.nitems) prefetch2(p, next, stage);
    for (unsigned use = 0;; ++use) {
      const int s = use % NSLOT;
      const Slot2 sl = slot2_at(slots, L, p.capr, sx, s);
      if (use >= NSLOT) mbar_wait_sleep(&empty[s], ((use / NSLOT) - 1) & 1);
      __syncwarp();
      const bool fresh = item < 0 || ja > Lseg;
      if (fresh) {
        item = next;
        if (item >= p.nitems) {  // stop marker (every producer lane arrives, as for a filled slot)
          if (lane == 0) sl.meta[0] = 1;
          asm volatile("bar.sync 1, %0;" ::"r"(32 * NP2) : "memory");
          mbar_arrive2(&full[s]);
          break;
        }
        item_geom2(p, item, x0, Lseg, cy, cz);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        for (int k = lane; k < 9 * LF; k += 32) O[k] = stage[k];
        __syncwarp();
        ja = 1;
      }
      int jb = choose_round2(p, O, ja, Lseg);
      while (jb < ja && ja <= Lseg) {  // a cell whose window alone does not fit: Par-Cell-SM
        if (lane == 0) {
          const unsigned long long k = atomicAdd(&p.ctl->pad[0], 1ull);
          p.dense[k] = (x0 - 1 + ja) + g.nx * (cy + g.ny * cz);
          ++fallbacks;
        }
        ++ja;
        if (ja <= Lseg) jb = choose_round2(p, O, ja, Lseg);
      }
      const bool none = ja > Lseg;
      if (none) jb = ja - 1;
      // the round's 27-cell candidates (the unit of the metric, R4): n_j (c27_j - 1) per cell
      for (int j = ja + lane; j <= jb; j += 32) {
        int c27 = 0;
#pragma unroll
        for (int r = 0; r < 9; ++r) c27 += O[r * LF + (j + 2) * sx] - O[r * LF + (j - 1) * sx];
        const int nj = O[4 * LF + (j + 1) * sx] - O[4 * LF + j * sx];
        cand += (unsigned long long)nj * (unsigned long long)(c27 - 1);
      }
      // interleaved staging of sub-cell positions [kb, ke) (cells ja-1 .. jb+1)
      const int kb = (ja - 1) * sx, ke = none ? kb : (jb + 2) * sx;
      const int nk = ke - kb, chunk = (nk + 31) / 32;
      const int k0 = min(ke, kb + lane * chunk), k1 = min(ke, k0 + chunk);
      int mine = 0;
      for (int k = k0; k < k1; ++k)
#pragma unroll
        for (int r = 0; r < 9; ++r) mine += O[r * LF + k + 1] - O[r * LF + k];
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 0) {
        sl.meta[0] = 0;
        sl.meta[1] = ja;
        sl.meta[2] = jb;
        sl.meta[3] = none ? 0 : O[4 * LF + (jb + 1) * sx] - O[4 * LF + ja * sx];
        sl.meta[4] = x0;
        sl.meta[5] = cy | (cz << 16);
        sl.meta[6] = 0;
        sl.meta[7] = O[4 * LF + ja * sx];
        sl.SK[ke] = total;
      }
      int base = incl - mine;
      for (int k = k0; k < k1; ++k) {
        sl.SK[k] = base;
#pragma unroll
        for (int r = 0; r < 9; ++r) base += O[r * LF + k + 1] - O[r * LF + k];
      }
      if (lane == 0) {
        sl.meta[8] = kb;
        sl.meta[9] = ke;
      }
      // the records, 16 B per cp.async (LDGSTS), by all NP producer warps, each lane a chunk of
      // the sub-cell positions; the slot is full when every producer lane's copies have landed
      // (cp.async.mbarrier.arrive.noinc).  (A TMA bulk copy per (sub-cell, pencil) run was
      // measured first: ~70 cycles per copy for runs of ~2 records.)
      asm volatile("bar.sync 1, %0;" ::"r"(32 * NP2) : "memory");
      {
        const int nkk = ke - kb, chunk = (nkk + 32 * NP2 - 1) / (32 * NP2);
        for (int k = min(ke, kb + lane * chunk), k1 = min(ke, kb + (lane + 1) * chunk); k < k1; ++k) {
          int bs = sl.SK[k];
#pragma unroll
          for (int r = 0; r < 9; ++r) {
            const int a = O[r * LF + k], n = O[r * LF + k + 1] - a;
            for (int o = 0; o < n; ++o) cp_async16(sl.R + bs + o, p.rec + a + o);
            bs += n;
          }
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
      asm volatile("bar.sync 2, %0;" ::"r"(32 * NP2) : "memory");  // the helpers are done with O
      ja = jb + 1;
      if (fresh) {
        if (lane == 0) next = (long long)atomicAdd(&p.ctl->xp_items, 1ull);
        next = __shfl_sync(0xffffffffu, next, 0);
        if (next < p.nitems) prefetch2(p, next, stage);
      }
    }
  } else {
    // ================================ consumers ================================
    const float thr = p.kp.rc2, mc2 = -p.kp.c2, rc = p.kp.rc;
    for (unsigned use = 0;; ++use) {
      const int s = use % NSLOT;
      const Slot2 sl = slot2_at(slots, L, p.capr, sx, s);
      mbar_wait(&full[s], (use / NSLOT) & 1);
      if (sl.meta[0]) break;
      const int ntargets = sl.meta[3], x0 = sl.meta[4], t0 = sl.meta[7];
      const int cy = sl.meta[5] & 0xffff, cz = sl.meta[5] >> 16;
      const int f0 = (x0 - 1 + g.gx_off) * sx;  // global fine index of item position k = 0
      for (;;) {
        int b = 0;
        if (lane == 0) b = atomicAdd(&sl.meta[6], 64);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b >= ntargets) break;
        const int T0 = b + 2 * lane;
        if (T0 < ntargets) {
          const bool two = T0 + 1 < ntargets;
          const float4 a0 = __ldg(p.rec + t0 + T0), a1 = two ? __ldg(p.rec + t0 + T0 + 1) : a0;
          // the targets' cells / X sub-cells (binning contract on the same fp32 values) and their
          // windows of X sub-cells (R18: x_t -/+ r_c rounded outward, clamped to the 3 cells)
          bool bad = false;
          const int fg0 = fine_x_global(g, a0.x, bad), fg1 = fine_x_global(g, a1.x, bad);
          const int j0 = (fg0 >> g.sxs) - g.gx_off - (x0 - 1), j1 = (fg1 >> g.sxs) - g.gx_off - (x0 - 1);
          int wlo, whi;
          if (KERNEL == PI_K_CANDIDATE) {
            wlo = (min(j0, j1) - 1) * sx;
            whi = (max(j0, j1) + 2) * sx - 1;
          } else {
            const int l0 = fine_x_global(g, __fsub_rd(a0.x, rc), bad) - f0;
            const int h0 = fine_x_global(g, __fadd_ru(a0.x, rc), bad) - f0;
            const int l1 = fine_x_global(g, __fsub_rd(a1.x, rc), bad) - f0;
            const int h1 = fine_x_global(g, __fadd_ru(a1.x, rc), bad) - f0;
            wlo = min(max(min(l0, l1), (min(j0, j1) - 1) * sx), (max(j0, j1) + 2) * sx - 1);
            whi = min(max(max(h0, h1), (min(j0, j1) - 1) * sx), (max(j0, j1) + 2) * sx - 1);
          }
          const int ra = sl.SK[wlo], re = sl.SK[whi + 1];
          TgtPair tp;
          tp.x = pk(a0.x, a1.x);
          tp.y = pk(a0.y, a1.y);
          tp.z = pk(a0.z, a1.z);
          p2 phi = pk(0.f), fx = pk(0.f), fy = pk(0.f), fz = pk(0.f);
          p2 phb = pk(0.f), fxb = pk(0.f), fyb = pk(0.f), fzb = pk(0.f);
          const float4 *__restrict__ R = sl.R;
          int q = ra;
          if (KERNEL == PI_K_CANDIDATE) {
            // the test kernel counts every 27-cell candidate (no cutoff): each half takes only the
            // sources of its own target's 3 cells (the two targets' windows may differ)
            for (; q < re; ++q) {
              const float4 u = R[q];
              const int cs = cell_x(g, u.x, bad) - (x0 - 1);
              phi = add2(phi, pk(abs(cs - j0) <= 1 ? u.w : 0.f, abs(cs - j1) <= 1 ? u.w : 0.f));
            }
          } else {
            for (; q + 1 < re; q += 2) {  // two records in flight: two independent chains
              const float4 u = R[q], v = R[q + 1];
              tp_eval<KERNEL>(tp, u, thr, mc2, phi, fx, fy, fz, p.kp);
              tp_eval<KERNEL>(tp, v, thr, mc2, phb, fxb, fyb, fzb, p.kp);
            }
            if (q < re) tp_eval<KERNEL>(tp, R[q], thr, mc2, phi, fx, fy, fz, p.kp);
          }
          phi = add2(phi, phb);
          fx = add2(fx, fxb);
          fy = add2(fy, fyb);
          fz = add2(fz, fzb);
          // identity exclusion (Alg. 1 :127): each target's own record lies in the window
          phi = pk(lo(phi) - tp_self<KERNEL>(tp, 0, a0, thr, mc2, p.kp),
                   two ? hi(phi) - tp_self<KERNEL>(tp, 1, a1, thr, mc2, p.kp) : hi(phi));
          if (KERNEL == PI_K_LOWFLOP) {  // the self pair also added the target's own position
            fx = pk(lo(fx) - a0.x, hi(fx) - a1.x);
            fy = pk(lo(fy) - a0.y, hi(fy) - a1.y);
            fz = pk(lo(fz) - a0.z, hi(fz) - a1.z);
          }
          auto emit = [&](int gs, const float4 &me, int fg, int jj, float ph, float ffx, float ffy, float ffz) {
            int fold = -1;
            if (UPD && p.out.pcounts)
              fold = ((x0 - 1 + jj) * sx + (fg & (sx - 1))) + ((g.nx * (cy + g.ny * cz)) << g.sxs);
            if (kern_wforce(KERNEL)) {
              const float c = me.w * p.kp.f_ts;  // summed wf (x_t - x_s)
              write_output<UPD>(p.out, g, gs, me, ph * p.kp.phi_scale, c * ffx, c * ffy, c * ffz, fold);
            } else if (KERNEL == PI_K_LOWFLOP) {
              write_output<UPD>(p.out, g, gs, me, ph, ffx, ffy, ffz, fold);
            } else {
              write_output<UPD>(p.out, g, gs, me, ph, 0.f, 0.f, 0.f, fold);
            }
          };
          emit(t0 + T0, a0, fg0, j0, lo(phi), lo(fx), lo(fy), lo(fz));
          if (two) emit(t0 + T0 + 1, a1, fg1, j1, hi(phi), hi(fx), hi(fy), hi(fz));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive2(&empty[s]);
    }
  }

  // the dense cells listed so far (Par-Cell-SM, cellsm.cuh), in the staging memory this block
  // no longer uses; the rest is left to k_cellsm_list
  __syncthreads();
  {
    CsParams cp;
    cp.rec = p.rec;
    cp.pairs = nullptr;
    cp.plane = 0;
    cp.offsets = p.offsets;
    cp.list = p.dense;
    cp.g = p.g;
    cp.kp = p.kp;
    cp.out = p.out;
    cp.ctl = p.ctl;
    cp.from_rec = true;
    cellsm_phase<KERNEL, UPD, (NC + NP2) * 32>(cp, slots);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cand += __shfl_xor_sync(0xffffffffu, cand, o);
    fallbacks += __shfl_xor_sync(0xffffffffu, fallbacks, o);
  }
  if (lane == 0) {
    if (cand) atomicAdd(&p.ctl->cand_slots[(blockIdx.x * (NC + NP2) + warp) & (CAND_SLOTS - 1)], cand);
    if (fallbacks) atomicAdd(&p.ctl->fallback_cells, fallbacks);
  }
}

template <int NC>
cudaError_t launch2_nc(const Xp2Params &p, cudaStream_t s) {
  const size_t smem = max(xp2_smem_bytes(p.L, p.capr, p.sx, p.nslot), CS_SMEM + 128);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(kern);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (NC + NP2) * 32, smem);
    if (occ < 1) occ = 1;
    long long blocks = (long long)sms * occ;
    if (blocks > p.nitems) blocks = p.nitems;
    if (blocks < 1) blocks = 1;
    kern<<<(int)blocks, (NC + NP2) * 32, smem, s>>>(p);
    return cudaGetLastError();
  };
  const bool upd = p.out.upd != nullptr;
  switch (p.kp.kernel) {
    case PI_K_GAUSSIAN: return upd ? go(k_interact_xpencil2<PI_K_GAUSSIAN, NC, true>) : go(k_interact_xpencil2<PI_K_GAUSSIAN, NC, false>);
    case PI_K_INDICATOR: return upd ? go(k_interact_xpencil2<PI_K_INDICATOR, NC, true>) : go(k_interact_xpencil2<PI_K_INDICATOR, NC, false>);
    case PI_K_LJ: return upd ? go(k_interact_xpencil2<PI_K_LJ, NC, true>) : go(k_interact_xpencil2<PI_K_LJ, NC, false>);
    case PI_K_LOWFLOP: return upd ? go(k_interact_xpencil2<PI_K_LOWFLOP, NC, true>) : go(k_interact_xpencil2<PI_K_LOWFLOP, NC, false>);
    case PI_K_HIGHFLOP: return upd ? go(k_interact_xpencil2<PI_K_HIGHFLOP, NC, true>) : go(k_interact_xpencil2<PI_K_HIGHFLOP, NC, false>);
    default: return upd ? go(k_interact_xpencil2<PI_K_CANDIDATE, NC, true>) : go(k_interact_xpencil2<PI_K_CANDIDATE, NC, false>);
  }
}

// the cells listed for Par-Cell-SM that no block took before it left (cellsm.cuh)
cudaError_t launch_dense_rest2(const Xp2Params &p, cudaStream_t s) {
  CsParams cp;
  cp.rec = p.rec;
  cp.pairs = nullptr;
  cp.plane = 0;
  cp.offsets = p.offsets;
  cp.list = p.dense;
  cp.g = p.g;
  cp.kp = p.kp;
  cp.out = p.out;
  cp.ctl = p.ctl;
  cp.from_rec = true;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(kern);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, CS_SMEM);
    kern<<<sms * (occ > 0 ? occ : 1), 256, CS_SMEM, s>>>(cp);
    return cudaGetLastError();
  };
  const bool upd = p.out.upd != nullptr;
  switch (p.kp.kernel) {
    case PI_K_GAUSSIAN: return upd ? go(k_cellsm_list<PI_K_GAUSSIAN, true>) : go(k_cellsm_list<PI_K_GAUSSIAN, false>);
    case PI_K_INDICATOR: return upd ? go(k_cellsm_list<PI_K_INDICATOR, true>) : go(k_cellsm_list<PI_K_INDICATOR, false>);
    case PI_K_LJ: return upd ? go(k_cellsm_list<PI_K_LJ, true>) : go(k_cellsm_list<PI_K_LJ, false>);
    case PI_K_LOWFLOP: return upd ? go(k_cellsm_list<PI_K_LOWFLOP, true>) : go(k_cellsm_list<PI_K_LOWFLOP, false>);
    case PI_K_HIGHFLOP: return upd ? go(k_cellsm_list<PI_K_HIGHFLOP, true>) : go(k_cellsm_list<PI_K_HIGHFLOP, false>);
    default: return upd ? go(k_cellsm_list<PI_K_CANDIDATE, true>) : go(k_cellsm_list<PI_K_CANDIDATE, false>);
  }
}

}  // namespace

cudaError_t launch_interact_xpencil2(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  if (!a.rec) return cudaErrorNotSupported;
  Xp2Params p;
  p.rec = a.rec;
  p.offsets = a.offsets;
  p.foffsets = a.foffsets;
  p.g = g;
  p.kp = k;
  p.out = a.out;
  p.ctl = a.ctl;
  p.dense = a.dense;
  p.sx = g.sx;
  const int own = g.own_hi - g.own_lo;
  const double ppc_mean = (double)a.n_est / (double)g.ncells;
  const int l_auto = ppc_mean >= 8.0 ? 64 : (ppc_mean >= 4.0 ? 128 : 256);
  p.L = a.tx_len > 0 ? a.tx_len : l_auto;
  if (p.L > 512) p.L = 512;
  if (p.L > own) p.L = own;
  const int nc_req = a.threads > 0 ? a.threads / 32 : 16;
  const int nc = nc_req <= 8 ? 8 : (nc_req <= 16 ? 16 : 20);
  p.nslot = a.slots >= 2 ? min(a.slots, MAX_SLOTS2) : 2;
  const size_t max_smem = 227 * 1024;
  // the segment must leave room for slots holding a few cells' windows (tables grow with L sx)
  auto fixed_of = [&](int L) { return 128 + tables2_bytes(L, p.sx) + (size_t)p.nslot * slot2_words(L, p.sx) * 4; };
  const size_t min_slot = (size_t)(27 * (ppc_mean + 4.0)) * 16 + 1024;
  while (p.L > 8 && fixed_of(p.L) + (size_t)p.nslot * min_slot > max_smem) p.L = (p.L + 1) / 2;
  p.nseg = (own + p.L - 1) / p.L;
  p.nitems = (long long)p.nseg * g.ny * g.nz;
  int cap = a.tx_cap;
  if (cap <= 0) {
    const size_t fixed = fixed_of(p.L);
    cap = max_smem > fixed ? (int)((max_smem - fixed) / ((size_t)p.nslot * 16)) : 16;
    cap = (int)min((long long)cap, a.n_est + 64);
  }
  p.capr = max(16, cap);
  while (xp2_smem_bytes(p.L, p.capr, p.sx, p.nslot) > max_smem && p.capr > 64) p.capr -= 16;
  if (xp2_smem_bytes(p.L, p.capr, p.sx, p.nslot) > max_smem) return cudaErrorNotSupported;
  cudaError_t e = nc == 8 ? launch2_nc<8>(p, s) : (nc == 16 ? launch2_nc<16>(p, s) : launch2_nc<20>(p, s));
  if (e != cudaSuccess) return e;
  return launch_dense_rest2(p, s);
}

}  // namespace pi
