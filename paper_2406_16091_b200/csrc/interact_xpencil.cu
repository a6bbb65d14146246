// a6.3: X-pencil (Alg. 5, §5.2), re-designed for sm_100a.
//
// The paper's block owns an X-pencil of target cells (plus 2 ghost cells), latches one
// target per thread in registers and then stages the <= 8 (Y, Z) +-1 neighbour pencils
// one at a time, with a barrier before and after each (:398-407).  Here the X-pencil is a
// whole target X-row (cy, cz) (or a segment of it) and the kernel streams rows through
// shared memory with a producer/consumer pipeline:
//
//   * persistent CTAs, NC CONSUMER warps and NSLOT = 2 staging slots, each filled by its own
//     PRODUCER warp and handed over with mbarriers (full / empty) instead of block-wide
//     barriers: while the consumers compute a row from one slot, the other slot is staged;
//   * staging a row (producer warp): the 9 neighbour rows' cells x0-1 .. x0+L are located in
//     the global prefix array; each (row, cell) run of cell-sorted 16-B records (X-fastest
//     linearisation) is copied record by record with 16-B cp.async (LDGSTS)
//     into a MERGED layout: for every X cell the particles of its 9
//     rows sit side by side (home row first), so the 27-cell candidate set of target cell cx
//     is the single contiguous window [M(cx-1), M(cx+2)) -- no per-row loop, no wasted
//     candidates.  Cell starts are padded to slot = 2j (mod 8) with inert records (x = 1e30,
//     q = 0): windows are whole source PAIRS and the ~4 windows of a warp start in distinct
//     bank groups.  The producer then interleaves the records in place into the source-pair
//     layout of interact_common.cuh (bitwise copies of the fp32 inputs);
//   * the slot capacity is fixed at launch from the mean density (the paper sizes the pencil
//     from M_C, :353; counting actual occupancy needs no M_C read-back and no host sync): a
//     row whose windows do not fit is split into rounds, and a cell whose window alone does
//     not fit is handed to the consumers as a global-memory fallback item;
//   * compute (consumer warps): one thread per target ("one thread per particle", :357), each
//     walking its cell's window two sources per packed-fp32 instruction.
#include "interact_common.cuh"

#ifdef XP_PROFILE
#define XP_T(v) long long v = clock64()
#define XP_ADD(i, a, b) if ((threadIdx.x & 31) == 0) atomicAdd(&xp_prof[i], (unsigned long long)((b) - (a)))
__device__ unsigned long long xp_prof[16];
#else
#define XP_T(v)
#define XP_ADD(i, a, b)
#endif

namespace pi {
namespace {

constexpr int NSLOT = 2;

struct XpParams {
  long long n;
  const float4 *rec;
  const int32_t *offsets;
  Geom g;
  KParams kp;
  OutDesc out;
  DevCtl *ctl;
  int L;             // target cells per work item along X (segment length)
  int cap;           // staged records (incl. padding) per slot
  int nseg;          // segments per X row
  long long nitems;  // rows x segments
};

// Per-slot int area: meta[8] | O[9][L+3] | Dst[9][L+2] | Msz[L+2] | Moff[L+3] | Tpre[L+3]
// meta: 0 stop flag (-1), 1 ja, 2 jb, 3 base, 4 ntargets, 5 fallback cell (or -1),
//       6 x0, 7 (cy | cz << 16) -- written by the producer
__host__ __device__ inline int slot_int_words(int L) {
  int ints = 8 + 9 * (L + 3) + 9 * (L + 2) + (L + 2) + (L + 3) + (L + 3);
  return (ints + 3) & ~3;
}
__host__ __device__ inline size_t slot_bytes(int L, int cap) {
  return (size_t)slot_int_words(L) * 4 + (size_t)cap * 16;
}
__host__ __device__ inline size_t xp_smem_bytes(int L, int cap) {
  return 128 /* mbarriers + reduction scratch */ + NSLOT * slot_bytes(L, cap);
}

constexpr float DUMMY_X = 1.0e30f;  // inert padding record: (x_s - x_t)^2 = inf, q = 0

struct Slot {
  int *meta, *O, *Dst, *Msz, *Moff, *Tpre;
  float4 *S;
};
__device__ __forceinline__ Slot slot_at(unsigned char *base, int L, int cap, int s) {
  unsigned char *p = base + (size_t)s * slot_bytes(L, cap);
  Slot sl;
  const int L3 = L + 3, L2 = L + 2;
  sl.meta = reinterpret_cast<int *>(p);
  sl.O = sl.meta + 8;
  sl.Dst = sl.O + 9 * L3;
  sl.Msz = sl.Dst + 9 * L2;
  sl.Moff = sl.Msz + L2;
  sl.Tpre = sl.Moff + L3;
  sl.S = reinterpret_cast<float4 *>(p + slot_int_words(L) * 4);
  return sl;
}

// Named hardware barriers (no spinning): ids 1..NSLOT = "slot full", NSLOT+1..2 NSLOT = "slot
// empty"; each has the producer warp of the slot and the NC consumer warps as participants.
__device__ __forceinline__ void nbar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- producer (one warp)
// Row tables of work item `item` into slot `sl`: offsets of the 9 neighbour rows, row starts
// inside each merged cell (home row first), merged sizes, padded merged offsets.
__device__ void build_tables(const XpParams &p, const Slot &sl, long long item, int &x0, int &cy, int &cz,
                             int &Lseg) {
  const int lane = threadIdx.x & 31;
  const int L = p.L, L3 = L + 3, L2 = L + 2;
  const Geom &g = p.g;
  const int seg = (int)(item % p.nseg);
  const long long row = item / p.nseg;
  cy = (int)(row % g.ny);
  cz = (int)(row / g.ny);
  x0 = g.own_lo + seg * L;  // owned X cells only (ghost layers are staged as sources)
  Lseg = min(L, g.own_hi - x0);
  // offsets of the 9 neighbour rows over cells x0-1 .. x0+L+1: all loads issued first
  constexpr int MAXK = (9 * 67 + 31) / 32;
  int v[MAXK];
#pragma unroll
  for (int u = 0; u < MAXK; ++u) {
    const int k = lane + 32 * u;
    v[u] = 0;
    if (k < 9 * L3) {
      const int r = k / L3, j = k - r * L3;
      const int y = cy + (r % 3) - 1, z = cz + (r / 3) - 1;
      if (y >= 0 && y < g.ny && z >= 0 && z < g.nz) {
        const int x = min(max(x0 - 1 + j, 0), g.nx);  // clamped: out-of-grid cells are empty
        v[u] = __ldg(p.offsets + (long long)g.nx * (y + (long long)g.ny * z) + x);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < MAXK; ++u) {
    const int k = lane + 32 * u;
    if (k < 9 * L3) sl.O[k] = v[u];
  }
  __syncwarp();
  // per merged cell: row starts (home row first) and size; padded size s' = s + ((2 - s) & 7)
  // makes every start M(j) = 2j (mod 8) with the minimal padding, and is a plain prefix sum
  int carry = 0;
  for (int j0 = 0; j0 < L2; j0 += 32) {
    const int j = j0 + lane;
    int pre = 0;
    if (j < L2) {
#pragma unroll
      for (int rr = 0; rr < 9; ++rr) {
        const int r = rr == 0 ? 4 : (rr <= 4 ? rr - 1 : rr);
        sl.Dst[r * L2 + j] = pre;
        pre += sl.O[r * L3 + j + 1] - sl.O[r * L3 + j];
      }
      sl.Msz[j] = pre;
    }
    const int padded = j < L2 ? pre + ((2 - pre) & 7) : 0;
    int incl = padded;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (j < L2) sl.Moff[j] = carry + incl - padded;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) sl.Moff[L2] = carry;
  __syncwarp();
}

// Chooses the round [ja, jb] (warp-cooperative), issues its TMA copies, writes padding and
// the slot meta.  jb < ja means "cell ja needs the fallback".
__device__ int stage_round(const XpParams &p, const Slot &sl, unsigned long long *tma_bar, int ja, int Lseg) {
  const int lane = threadIdx.x & 31;
  const int L = p.L, L3 = L + 3, L2 = L + 2;
  const int base = sl.Moff[ja - 1];
  int jb = ja - 1;
  for (int j0 = ja; j0 <= Lseg; j0 += 32) {
    const int j = j0 + lane;
    const bool fit = j <= Lseg && sl.Moff[j + 2] - base <= p.cap;
    const unsigned b = __ballot_sync(0xffffffffu, fit);
    jb += __popc(b);
    if (b != 0xffffffffu) break;
  }
  if (jb < ja) return jb;
  // target prefix over the round's cells
  int carry = 0;
  for (int j0 = ja; j0 <= jb; j0 += 32) {
    const int j = j0 + lane;
    const int nt = j <= jb ? sl.O[4 * L3 + j + 1] - sl.O[4 * L3 + j] : 0;
    int incl = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (j <= jb) sl.Tpre[j] = carry + incl - nt;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) sl.Tpre[jb + 1] = carry;
  int real = 0;
  for (int j = ja - 1 + lane; j <= jb + 1; j += 32) real += sl.Msz[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) real += __shfl_xor_sync(0xffffffffu, real, o);
  (void)real;
  (void)tma_bar;
  // one (row, cell) run per lane, each record one 16-B cp.async (LDGSTS) into its merged slot
  const int ncell = jb - ja + 3;
  for (int k = lane; k < 9 * ncell; k += 32) {
    const int jj = k / 9, r = k - jj * 9;
    const int j = ja - 1 + jj;
    const int src = sl.O[r * L3 + j];
    const int c = sl.O[r * L3 + j + 1] - src;
    float4 *dst = sl.S + (sl.Moff[j] + sl.Dst[r * L2 + j] - base);
    const float4 *gs = p.rec + src;
    for (int e = 0; e < c; ++e) cp_async16(dst + e, gs + e);
  }
  // padding records (disjoint from the bulk-copy destinations)
  for (int k = lane; k < 8 * ncell; k += 32) {
    const int jj = k >> 3, u = k & 7;
    const int j = ja - 1 + jj;
    const int s = sl.Moff[j] + sl.Msz[j] + u;
    if (s < sl.Moff[j + 1]) sl.S[s - base] = make_float4(DUMMY_X, DUMMY_X, DUMMY_X, 0.f);
  }
  if (lane == 0) {
    sl.meta[1] = ja;
    sl.meta[2] = jb;
    sl.meta[3] = base;
    sl.meta[4] = carry;
    sl.meta[5] = -1;
  }
  return jb;
}

template <int KERNEL, int NC, int UNR>
__global__ void __launch_bounds__((NC + NSLOT) * 32, 2) k_interact_xpencil(XpParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long *full = reinterpret_cast<unsigned long long *>(smem_raw);  // [NSLOT]
  unsigned long long *empty = full + NSLOT;                                      // [NSLOT]
  unsigned long long *tmab = empty + NSLOT;                                      // [NSLOT]
  unsigned long long *red = reinterpret_cast<unsigned long long *>(smem_raw + 64);  // [8]
  unsigned char *slots = smem_raw + 128;
  const int L = p.L, L3 = L + 3;
  const Geom &g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long cand = 0, fallbacks = 0;

  (void)full;
  (void)empty;
  (void)tmab;
  constexpr int NPART = (NC + 1) * 32;  // participants of a slot barrier
  if (tid < 8) red[tid] = 0;
  __syncthreads();

  if (warp >= NC) {
    // ============================ producers (one per slot) ============================
    unsigned used = 0;
    const int slot = warp - NC;
    bool done = false;
    while (!done) {
      long long item = 0;
      if (lane == 0) item = (long long)atomicAdd(&p.ctl->xp_items, 1ull);
      item = __shfl_sync(0xffffffffu, item, 0);
      int x0 = 0, cy = 0, cz = 0, Lseg = 0;
      int ja = 1;
      bool first = true;
      while (first || ja <= Lseg) {
        Slot sl = slot_at(slots, L, p.cap, slot);
        if (used & (1u << slot)) {  // wait until the consumers released this slot
          XP_T(t0);
          nbar_sync(1 + NSLOT + slot, NPART);
          XP_T(t1);
          XP_ADD(0, t0, t1);
        }
        used |= 1u << slot;
        if (item >= p.nitems) {  // stop marker
          if (lane == 0) sl.meta[0] = -1;
          __syncwarp();
          nbar_arrive(1 + slot, NPART);
          done = true;
          break;
        }
        XP_T(t2);
        build_tables(p, sl, item, x0, cy, cz, Lseg);
        XP_T(t3);
        XP_ADD(1, t2, t3);
        first = false;
        const int jb = stage_round(p, sl, &tmab[slot], ja, Lseg);
        XP_T(t4);
        XP_ADD(2, t3, t4);
        if (lane == 0) {
          sl.meta[0] = 0;
          sl.meta[6] = x0;
          sl.meta[7] = cy | (cz << 16);
        }
        if (jb < ja) {  // fallback cell: consumers run the global path for cell ja
          if (lane == 0) {
            sl.meta[1] = ja;
            sl.meta[2] = ja - 1;
            sl.meta[4] = 0;
            sl.meta[5] = ja;
          }
          ++ja;
        } else {
          cp_async_wait_all();
          XP_T(t5);
          XP_ADD(3, t4, t5);
          __syncwarp();
          // interleave in place: raw record pairs -> source-pair layout
          const int total = sl.Moff[jb + 2] - sl.Moff[ja - 1];
          int k = lane;
          for (; k + 96 < (total >> 1); k += 128) {
            stage_pair(sl.S, k);
            stage_pair(sl.S, k + 32);
            stage_pair(sl.S, k + 64);
            stage_pair(sl.S, k + 96);
          }
          for (; k < (total >> 1); k += 32) stage_pair(sl.S, k);
          ja = jb + 1;
        }
        __syncwarp();
        XP_T(t6);
        XP_ADD(4, t4, t6);
        XP_ADD(5, t2, t6);
        nbar_arrive(1 + slot, NPART);  // release: tables, records, meta
      }
    }
  } else {
    // ================================ consumers ================================
    const float thr = p.kp.rc2, mc2 = -p.kp.c2;
    unsigned stopped = 0;  // one bit per slot
    int slot = 0;
    while (stopped != (1u << NSLOT) - 1u) {
      if (stopped & (1u << slot)) {
        slot = (slot + 1) % NSLOT;
        continue;
      }
      XP_T(c0);
      nbar_sync(1 + slot, NPART);
      XP_T(c1);
      XP_ADD(6, c0, c1);
      Slot sl = slot_at(slots, L, p.cap, slot);
      if (sl.meta[0] < 0) {  // this slot's producer ran out of work items
        stopped |= 1u << slot;
        slot = (slot + 1) % NSLOT;
        continue;
      }
      const int ja = sl.meta[1], jb = sl.meta[2], base = sl.meta[3], ntargets = sl.meta[4], fb = sl.meta[5];
      const int x0 = sl.meta[6], cy = sl.meta[7] & 0xffff, cz = sl.meta[7] >> 16;
      if (fb >= 0) {
        // global-memory fallback for one cell, spread over the consumer threads
        const long long home_row = (long long)g.nx * (cy + (long long)g.ny * cz);
        const int cx = x0 - 1 + fb;
        const int t_lo = __ldg(p.offsets + home_row + cx), t_hi = __ldg(p.offsets + home_row + cx + 1);
        for (int t = t_lo + tid; t < t_hi; t += NC * 32)
          fallback_target<KERNEL>(t, cx, cy, cz, p.rec, p.offsets, g, p.kp, p.out, cand);
        if (tid == 0) ++fallbacks;
      } else {
        for (int T = tid; T < ntargets; T += NC * 32) {
          // cell of target T: last j in [ja, jb] with Tpre[j] <= T (binary search)
          int lo_ = ja, hi_ = jb;
          while (lo_ < hi_) {
            const int mid = (lo_ + hi_ + 1) >> 1;
            if (sl.Tpre[mid] <= T) lo_ = mid; else hi_ = mid - 1;
          }
          const int j = lo_;
          const int i = T - sl.Tpre[j];
          const int t = sl.Moff[j] - base + i;  // staged slot of the target
          const int p0 = (sl.Moff[j - 1] - base) >> 1, p1 = (sl.Moff[j + 2] - base) >> 1;
          const float4 r = lane_target<KERNEL, UNR>(sl.S, t >> 1, t & 1, p0, p1, thr, mc2);
          cand += (unsigned long long)(sl.Msz[j - 1] + sl.Msz[j] + sl.Msz[j + 1] - 1);
          const int gs = sl.O[4 * L3 + j] + i;
          float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p.out.upd) me = __ldg(p.rec + gs);
          if (KERNEL == PI_K_GAUSSIAN) {
            const float4 qq = sl.S[2 * (t >> 1) + 1];
            const float q = (t & 1) ? qq.w : qq.z;
            const float sc = -q * p.kp.inv_s2;
            write_output(p.out, g, gs, me, r.x, sc * r.y, sc * r.z, sc * r.w);
          } else {
            write_output(p.out, g, gs, me, r.x, 0.f, 0.f, 0.f);
          }
        }
      }
      __syncwarp();
      XP_T(c2);
      XP_ADD(7, c1, c2);
      XP_ADD(8, 0, 1);
      nbar_arrive(1 + NSLOT + slot, NPART);
      slot = (slot + 1) % NSLOT;
    }
  }
  // statistics: one atomic per block, spread over CAND_SLOTS counters
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
  if (lane == 0 && cand) atomicAdd(&red[warp & 7], cand);
  __syncthreads();
  if (tid == 0) {
    unsigned long long tsum = 0;
    for (int w = 0; w < 8; ++w) tsum += red[w];
    if (tsum) atomicAdd(&p.ctl->cand_slots[blockIdx.x & (CAND_SLOTS - 1)], tsum);
  }
  if (tid < NC * 32 && (tid & 31) == 0 && fallbacks) atomicAdd(&p.ctl->fallback_cells, fallbacks);
}

template <int KERNEL, int NC>
cudaError_t launch_k(const XpParams &p, cudaStream_t s, int blocks_per_sm) {
  constexpr int UNR = NC >= 16 ? 2 : 4;  // registers: 2 blocks x (NC + 2) warps must fit
  const size_t smem = xp_smem_bytes(p.L, p.cap);
  cudaError_t e =
      cudaFuncSetAttribute(k_interact_xpencil<KERNEL, NC, UNR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_interact_xpencil<KERNEL, NC, UNR>, (NC + NSLOT) * 32, smem);
  if (occ < 1) occ = 1;
  long long blocks = (long long)sms * (blocks_per_sm > 0 ? min(occ, blocks_per_sm) : occ);
  if (blocks > p.nitems) blocks = p.nitems;
  if (blocks < 1) blocks = 1;
  k_interact_xpencil<KERNEL, NC, UNR><<<(int)blocks, (NC + NSLOT) * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <int NC>
cudaError_t launch_nc(const XpParams &p, cudaStream_t s, int bps) {
  switch (p.kp.kernel) {
    case PI_K_GAUSSIAN: return launch_k<PI_K_GAUSSIAN, NC>(p, s, bps);
    case PI_K_INDICATOR: return launch_k<PI_K_INDICATOR, NC>(p, s, bps);
    default: return launch_k<PI_K_CANDIDATE, NC>(p, s, bps);
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
  const int own = g.own_hi - g.own_lo;
  p.L = a.tx_len > 0 ? a.tx_len : 32;
  if (p.L > 64) p.L = 64;
  if (p.L > own) p.L = own;
  p.nseg = (own + p.L - 1) / p.L;
  p.nitems = (long long)p.nseg * g.ny * g.nz;
  // consumer warps (threads = 32 * NC target threads + one producer warp)
  const int nc = a.threads == 512 ? 16 : (a.threads == 128 ? 4 : 8);
  if (a.tx_cap > 0) {
    p.cap = a.tx_cap;
  } else {
    // mean occupancy of 9 rows x (L + 2) cells (+ 10 %), plus the padding (< 8 per cell)
    const double ppc = (double)a.n_est / (double)g.ncells;
    p.cap = (int)((9.0 * ppc * 1.1 + 4.0) * (p.L + 2) + 128.0);
  }
  p.cap = (p.cap + 31) & ~31;
  const size_t max_smem = 227 * 1024;
  while (xp_smem_bytes(p.L, p.cap) > max_smem && p.cap > 64) p.cap -= 32;
  const int bps = a.groups;  // blocks-per-SM cap (tuning knob lanes_per_pair reused), 0 = occupancy
  if (nc == 4) return launch_nc<4>(p, s, bps);
  if (nc == 8) return launch_nc<8>(p, s, bps);
  return launch_nc<16>(p, s, bps);
}

}  // namespace pi

#ifdef XP_PROFILE
extern "C" __attribute__((visibility("default"))) void pi_debug_xp_profile(unsigned long long *out) {
  cudaMemcpyFromSymbol(out, xp_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(xp_prof, z, sizeof(z));
}
#endif
