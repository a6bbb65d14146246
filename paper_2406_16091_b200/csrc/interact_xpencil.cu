// a6.3: X-pencil (Alg. 5, §5.2), re-designed for sm_100a.
//
// As in the paper, the work unit is an X-pencil of target cells (a segment of L cells of one
// X row (cy, cz), default the whole row), one thread per target ("one thread per particle",
// :357), and the 9 pencils (cy + dy, cz + dz) around it are staged in shared memory
// (:398-407).  B200 specifics:
//
//   * each of the 9 neighbour pencils is ONE contiguous run of cell-sorted 16-B records
//     (X-fastest linearisation), so a pencil arrives with one TMA bulk copy
//     (cp.async.bulk, completion counted in bytes on the slot's mbarrier): 9 copies per item,
//     issued by a single producer warp -- no per-particle staging work at all;
//   * persistent blocks stream the items through nslot (2..4) slots: while the consumer warps
//     compute one slot the producer refills the other.  Slots are handed over with mbarriers
//     (full: TMA bytes + producer arrival; empty: one arrival per consumer warp), consumer
//     warps take 32-target batches from a per-slot counter and move on to the next slot as
//     soon as the current one is exhausted -- no block-wide barrier anywhere;
//   * a target walks its 27 candidate cells as the 9 contiguous 3-cell runs (one per staged
//     pencil); two consecutive records of a run form an f32x2 source pair
//     (interact_common.cuh, src_eval: 12 packed-fp32 instructions + 2 MUFU.EX2 per 2
//     candidates, differences from the raw fp32 positions);
//   * capacity: the slot is sized from the mean density (+15 %) instead of M_C (:353), so there
//     is no device->host read-back; a row whose 9 pencils do not fit is split into rounds
//     along X, and a cell whose window alone does not fit takes the global-memory path.
#include "cellsm.cuh"
#include "interact_common.cuh"

#ifdef XP_PROFILE  // development counters (tools/build_prof.sh, tools/xp_prof.py)
__device__ unsigned long long xp_prof[16];
#define XP_T(v) long long v = clock64()
#define XP_ADD(i, a, b) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&xp_prof[i], (unsigned long long)((b) - (a)))
extern "C" __attribute__((visibility("default"))) void pi_debug_xp_profile(unsigned long long *out) {
  cudaMemcpyFromSymbol(out, xp_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(xp_prof, z, sizeof(z));
}
#else
#define XP_T(v)
#define XP_ADD(i, a, b)
#endif

namespace pi {
namespace {

constexpr int MAX_SLOTS = 4;
constexpr int META = 16;
constexpr size_t WT_BYTES = 20 * 32 * 4;
constexpr float DUMMY_X = 1.0e30f;  // inert partner of an odd run's last record: K = 0, q = 0

struct XpParams {
  const float4 *rec;
  const float4 *pairs;  // the sorted records as f32x2 source pairs (k_pairify): planes A | B
  long long plane;      // float4 elements per plane
  const int32_t *offsets;
  const int32_t *foffsets;  // fine offsets: sx X sub-cells per cell (the sorted order)
  Geom g;
  KParams kp;
  OutDesc out;
  DevCtl *ctl;
  int L;             // target cells per work item along X (segment length)
  int sx;            // X sub-cells per cell
  bool mask;         // mask the out-of-run halves of a run's end pairs (walk9)
  int capp;          // staged source pairs per slot
  int nslot;         // staging slots (2..MAX_SLOTS)
  int tpl;           // targets per consumer lane (1 or 2)
  int32_t *dense;    // cells whose window alone does not fit a slot: listed for Par-Cell-SM
  int nseg;          // segments per X row (nseg0 of them in the first X range)
  int nseg0;
  int xr[4];         // target X layers (local): [xr0, xr1) then [xr2, xr3) (may be empty)
  long long nitems;  // rows x segments
  int reserve;       // SMs left free (the exchange kernels overlapping this launch)
};

// Shared memory: header (mbarriers, O-table item indices) | nslot slots | NOB = nslot + 1
// offsets tables O[9][LF] | the cell-group consumers' run tables.
// Slot: SA[capp] | SB[capp] float4 (source pairs, planes A and B) | meta[16] | rb[32]
//   rb[r]    first staged pair of pencil r's run in S (rb[9] = total); rb[16 + r] = rb[r] minus
//            the global pair index of the run's first record: staged pair of global pair k
// meta: 0 stop (1), 1 ja, 2 jb (target cells ja..jb of the item in this round; an empty round
//       has ntargets = 0), 3 ntargets, 4 x0, 5 cy | cz << 16, 6 batch counter, 7 O table
// O table (LF = (L+2) sx + 1): O[r][k] = global offset of pencil r (= (dy + 1) + 3 (dz + 1)) at
//   the fine (X sub-cell) boundary k of the cells x0-1 .. x0+L; the cell boundary j is O[r][j sx].
//   Filled by the helper warp one item ahead; the slots of an item's rounds share its table.
constexpr int HDR = 256;
__host__ __device__ inline int lf_of(int L, int sx) { return (L + 2) * sx + 1; }
__host__ __device__ inline int slot_words() { return (META + 32 + 3) & ~3; }
__host__ __device__ inline size_t slot_bytes(int capp) { return (size_t)capp * 32 + (size_t)slot_words() * 4; }
__host__ __device__ inline size_t otab_bytes(int L, int sx) { return ((size_t)9 * lf_of(L, sx) * 4 + 15) & ~size_t(15); }
__host__ __device__ inline size_t xp_smem_bytes(int L, int capp, int sx, int nslot) {
  return HDR + nslot * slot_bytes(capp) + (size_t)(nslot + 1) * otab_bytes(L, sx) + WT_BYTES;
}

struct Slot {
  float4 *S, *SB;  // planes A (x, y) and B (z, q) of the staged source pairs
  int *meta, *O, *rb;
};
__device__ __forceinline__ Slot slot_at(unsigned char *base, int capp, int s) {
  unsigned char *u = base + (size_t)s * slot_bytes(capp);
  Slot sl;
  sl.S = reinterpret_cast<float4 *>(u);
  sl.SB = sl.S + capp;
  sl.meta = reinterpret_cast<int *>(u + (size_t)capp * 32);
  sl.rb = sl.meta + META;
  sl.O = nullptr;
  return sl;
}

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// The cell-sorted records as source pairs A[k] = P[k] = (x_2k, x_2k+1, y_2k, y_2k+1),
// B[k] = P[plane + k] = (z_2k, z_2k+1, q_2k, q_2k+1) (bitwise copies; an odd count gets an inert
// partner), so that a pencil run is staged by TMA already in the layout the f32x2 loop reads.
__global__ void k_pairify(long long n, const long long *n_dev, const float4 *__restrict__ rec, float4 *P,
                          long long plane) {
  if (n_dev) n = *n_dev;
  const long long np = (n + 1) >> 1;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < np; k += (long long)gridDim.x * blockDim.x) {
    const float4 a = rec[2 * k];
    const float4 b = 2 * k + 1 < n ? rec[2 * k + 1] : make_float4(DUMMY_X, DUMMY_X, DUMMY_X, 0.f);
    P[k] = make_float4(a.x, b.x, a.y, b.y);
    P[plane + k] = make_float4(a.z, b.z, a.w, b.w);
  }
}

// ---------------------------------------------------------------- producer (one warp)
// The offsets tables are fetched by a helper warp, one item ahead of the producer, straight into
// the table the slots of that item will use (XP_PROFILE: with the fetch and a copy into the slot
// in the producer's own loop, the producer's ~18K cycles per item set the pace and the consumer
// warps waited ~12 % of their time for a slot).
__device__ __forceinline__ void item_geom(const XpParams &p, long long item, int &x0, int &Lseg, int &cy, int &cz) {
  const int seg = (int)(item % p.nseg);
  const long long row = item / p.nseg;
  cy = (int)(row % p.g.ny);
  cz = (int)(row / p.g.ny);
  const bool first = seg < p.nseg0;
  x0 = first ? p.xr[0] + seg * p.L : p.xr[2] + (seg - p.nseg0) * p.L;
  Lseg = min(p.L, (first ? p.xr[1] : p.xr[3]) - x0);
}
__device__ __forceinline__ void cp_async4(int *dst, const int *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
// Fine offsets of the 9 pencils of `item` at the X sub-cell boundaries of cells x0-1 .. x0+L
// (clamped: rows outside the grid are empty) -> stage[9][LF], asynchronously.
__device__ __forceinline__ void prefetch_offsets(const XpParams &p, long long item, int *stage) {
  const int lane = threadIdx.x & 31;
  const int LF = lf_of(p.L, p.sx), sx = p.sx;
  const Geom &g = p.g;
  int x0, Lseg, cy, cz;
  item_geom(p, item, x0, Lseg, cy, cz);
  const int nxf = g.nx * sx;
  for (int k = lane; k < LF; k += 32) {
    const int bf = min(max((x0 - 1) * sx + k, 0), nxf);
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const int y = cy + (r % 3) - 1, z = cz + (r / 3) - 1;
      const bool ok = y >= 0 && y < g.ny && z >= 0 && z < g.nz;
      cp_async4(stage + r * LF + k, p.foffsets + (ok ? (long long)nxf * (y + (long long)g.ny * z) + bf : 0), ok);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
// Round [ja, jb] of the item: the largest jb <= Lseg whose 9 pencil runs (cells ja-1 .. jb+1,
// whole source pairs) fit the slot (warp-uniform; jb < ja: cell ja alone does not fit).
__device__ int choose_round(const XpParams &p, const Slot &sl, int ja, int Lseg) {
  const int lane = threadIdx.x & 31;
  const int LF = lf_of(p.L, p.sx), sx = p.sx;
  int jb = ja - 1;
  for (int j0 = ja; j0 <= Lseg; j0 += 32) {
    const int j = j0 + lane;
    int tot = 0;
    if (j <= Lseg) {
#pragma unroll
      for (int r = 0; r < 9; ++r)
        tot += ((sl.O[r * LF + (j + 2) * sx] + 1) >> 1) - (sl.O[r * LF + (ja - 1) * sx] >> 1);
    }
    const unsigned b = __ballot_sync(0xffffffffu, j <= Lseg && tot <= p.capp);
    jb += __popc(b);
    if (b != 0xffffffffu) break;
  }
  return jb;
}

// ---------------------------------------------------------------- consumer
// (phi, sum w d) of the target `me` over its 9 runs: fine boundaries klo .. khi+1 of every
// pencil (inside cells j-1 .. j+1: the X sub-cells that can hold a source closer than r_c
// along X).  A run [a, b) of records covers the staged pairs a/2 .. (b-1)/2.  The halves of
// its first and last pair outside the run are the records a-1 and b of the sorted array:
//   MASK = true  (CANDIDATE kernel, or grids under 4 cells along X): they get q = 0;
//   MASK = false (cutoff kernels): they are evaluated as they are -- record a-1 lies in a
//     skipped sub-cell or cell of the same pencil (|dx| >= r_c by construction) or, at a row
//     start, in the last cell of the previous row (|dx| > (nx - 3) w >= r_c), and likewise
//     record b, or b is the inert partner after the last record -- so r^2 >= r_c^2 in fp32 too
//     and they add exactly 0; no peeled iterations.
// The self term (= q_t exactly: d = 0, K(0) = 2^0 = 1) is removed.
template <int KERNEL, bool MASK>
__device__ __forceinline__ float4 walk9(const Slot &sl, int LF, int sx, int ja, int klo, int khi, const float4 me,
                                        const float thr, const float mc2, const KParams &kp) {
  const float4 *__restrict__ S = sl.S;
  const float4 *__restrict__ SB = sl.SB;
  p2 phi = pk(0.f), fx = pk(0.f), fy = pk(0.f), fz = pk(0.f);
  p2 phb = pk(0.f), fxb = pk(0.f), fyb = pk(0.f), fzb = pk(0.f);
#pragma unroll  // the 9 runs unrolled: their bounds loads schedule early (measured: -1 %)
  for (int r = 0; r < 9; ++r) {
    const int a = sl.O[r * LF + klo], b = sl.O[r * LF + khi + 1];
    if (b <= a) continue;
    const int base = sl.rb[16 + r];
    const int p0 = base + (a >> 1), pl = base + ((b - 1) >> 1);  // first and last pair
    if (!MASK) {
      int q = p0;
      for (; q + 1 <= pl; q += 2) {
        const SrcPair s0 = load_pair(S, SB, q), s1 = load_pair(S, SB, q + 1);
        src_eval<KERNEL>(s0, me.x, me.y, me.z, thr, mc2, phi, fx, fy, fz, &kp);
        src_eval<KERNEL>(s1, me.x, me.y, me.z, thr, mc2, phb, fxb, fyb, fzb, &kp);
      }
      if (q <= pl) src_eval<KERNEL>(load_pair(S, SB, q), me.x, me.y, me.z, thr, mc2, phi, fx, fy, fz, &kp);
      continue;
    }
    {
      SrcPair f = load_pair(S, SB, p0);
      f.q = pk((a & 1) ? 0.f : lo(f.q), (p0 == pl && (b & 1)) ? 0.f : hi(f.q));
      src_eval<KERNEL>(f, me.x, me.y, me.z, thr, mc2, phi, fx, fy, fz, &kp);
    }
    if (pl > p0) {
      int q = p0 + 1;
      for (; q + 2 <= pl; q += 2) {
        const SrcPair s0 = load_pair(S, SB, q), s1 = load_pair(S, SB, q + 1);
        src_eval<KERNEL>(s0, me.x, me.y, me.z, thr, mc2, phb, fxb, fyb, fzb, &kp);
        src_eval<KERNEL>(s1, me.x, me.y, me.z, thr, mc2, phi, fx, fy, fz, &kp);
      }
      if (q < pl) src_eval<KERNEL>(load_pair(S, SB, q), me.x, me.y, me.z, thr, mc2, phb, fxb, fyb, fzb, &kp);
      SrcPair l = load_pair(S, SB, pl);
      l.q = pk(lo(l.q), (b & 1) ? 0.f : hi(l.q));
      src_eval<KERNEL>(l, me.x, me.y, me.z, thr, mc2, phb, fxb, fyb, fzb, &kp);
    }
  }
  phi = add2(phi, phb);
  fx = add2(fx, fxb);
  fy = add2(fy, fyb);
  fz = add2(fz, fzb);
  // identity exclusion (Alg. 1 :127): remove the exact term the self pair added (q_t, or the LJ
  // value at d = 0, to phi only; LOWFLOP: the target's own position sums)
  const float4 st = self_terms<KERNEL>(me, kp);
  return make_float4(lo(phi) + hi(phi) - st.x, lo(fx) + hi(fx) - st.y, lo(fy) + hi(fy) - st.z,
                     lo(fz) + hi(fz) - st.w);
}

// Two targets per lane (the register blocking of the paper's X-pencil-reg idea, PAPER.md
// :421-457 §5.3: targets held in registers, every staged source read once for several of them):
// each staged pair is loaded once for both targets, so the lane reads 8 B of shared memory per
// candidate instead of 16 -- shared-memory wavefronts, not the FP32 pipe, bound walk9 (ncu: 81 %
// of the LSU wavefront peak).  The window is the union [klo, khi] of the two targets' windows;
// a source of the union outside a target's own window has |dx| >= r_c (the fine index is
// monotone in x), so, for the cutoff kernels, it adds exactly 0, as do the out-of-run halves of
// the end pairs (walk9, MASK = false).
template <int KERNEL>
__device__ __forceinline__ void walk9x2(const Slot &sl, int LF, int sx, int ja, int klo, int khi, const float4 me0,
                                        const float4 me1, const float thr, const float mc2, const KParams &kp,
                                        float4 &r0, float4 &r1) {
  const float4 *__restrict__ S = sl.S;
  const float4 *__restrict__ SB = sl.SB;
  p2 ph0 = pk(0.f), fx0 = pk(0.f), fy0 = pk(0.f), fz0 = pk(0.f);
  p2 ph1 = pk(0.f), fx1 = pk(0.f), fy1 = pk(0.f), fz1 = pk(0.f);
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    const int a = sl.O[r * LF + klo], b = sl.O[r * LF + khi + 1];
    if (b <= a) continue;
    const int base = sl.rb[16 + r];
    const int p0 = base + (a >> 1), pl = base + ((b - 1) >> 1);  // first and last pair
    int q = p0;
    for (; q + 1 <= pl; q += 2) {
      const SrcPair s0 = load_pair(S, SB, q), s1 = load_pair(S, SB, q + 1);
      src_eval<KERNEL>(s0, me0.x, me0.y, me0.z, thr, mc2, ph0, fx0, fy0, fz0, &kp);
      src_eval<KERNEL>(s0, me1.x, me1.y, me1.z, thr, mc2, ph1, fx1, fy1, fz1, &kp);
      src_eval<KERNEL>(s1, me0.x, me0.y, me0.z, thr, mc2, ph0, fx0, fy0, fz0, &kp);
      src_eval<KERNEL>(s1, me1.x, me1.y, me1.z, thr, mc2, ph1, fx1, fy1, fz1, &kp);
    }
    if (q <= pl) {
      const SrcPair s0 = load_pair(S, SB, q);
      src_eval<KERNEL>(s0, me0.x, me0.y, me0.z, thr, mc2, ph0, fx0, fy0, fz0, &kp);
      src_eval<KERNEL>(s0, me1.x, me1.y, me1.z, thr, mc2, ph1, fx1, fy1, fz1, &kp);
    }
  }
  // identity exclusion (Alg. 1 :127): each target's own self pair was evaluated in the window
  const float4 s0 = self_terms<KERNEL>(me0, kp), s1 = self_terms<KERNEL>(me1, kp);
  r0 = make_float4(lo(ph0) + hi(ph0) - s0.x, lo(fx0) + hi(fx0) - s0.y, lo(fy0) + hi(fy0) - s0.z,
                   lo(fz0) + hi(fz0) - s0.w);
  r1 = make_float4(lo(ph1) + hi(ph1) - s1.x, lo(fx1) + hi(fx1) - s1.y, lo(fy1) + hi(fy1) - s1.z,
                   lo(fz1) + hi(fz1) - s1.w);
}

// Cell-group walk (TPL = 0): the targets of ONE cell share a warp, k = 32 / n_t lanes per
// target, and every target walks the union window of the cell's targets (the fine X window of
// each target, reduced min / max over the warp: a source of the union outside a target's own
// window has |dx| >= r_c, so it adds exactly 0 for the cutoff kernels, as in walk9x2).  The 9
// runs of that window are one flattened sequence of Np staged pairs (wt: cumulative ends
// wt[0..8], staged pair of sequence index g = wt[16 + r] + g), and the k lanes of a target take
// the indices g = jj, jj + k, ...: no per-run tails, and the lanes of all targets read the same
// k staged pairs at a time (k distinct shared-memory addresses per LDS.128 instead of up to 32).
// Returns the lane's partial sums (the self pair is in exactly one lane's share).
template <int KERNEL>
__device__ __forceinline__ float4 walk_flat(const Slot &sl, const int *wt, int Np, int g, int k, const float4 me,
                                            const float thr, const float mc2, const KParams &kp) {
  const float4 *__restrict__ S = sl.S;
  const float4 *__restrict__ SB = sl.SB;
  p2 phi = pk(0.f), fx = pk(0.f), fy = pk(0.f), fz = pk(0.f);
  p2 phb = pk(0.f), fxb = pk(0.f), fyb = pk(0.f), fzb = pk(0.f);
  int r = 0, end = wt[0], off = wt[16];
  for (; g + k < Np; g += 2 * k) {
    while (g >= end) {
      ++r;
      end = wt[r];
      off = wt[16 + r];
    }
    const int pa = off + g;
    const int g2 = g + k;
    while (g2 >= end) {
      ++r;
      end = wt[r];
      off = wt[16 + r];
    }
    const int pb = off + g2;
    const SrcPair s0 = load_pair(S, SB, pa), s1 = load_pair(S, SB, pb);
    src_eval<KERNEL>(s0, me.x, me.y, me.z, thr, mc2, phi, fx, fy, fz, &kp);
    src_eval<KERNEL>(s1, me.x, me.y, me.z, thr, mc2, phb, fxb, fyb, fzb, &kp);
  }
  if (g < Np) {
    while (g >= end) {
      ++r;
      end = wt[r];
      off = wt[16 + r];
    }
    src_eval<KERNEL>(load_pair(S, SB, off + g), me.x, me.y, me.z, thr, mc2, phi, fx, fy, fz, &kp);
  }
  phi = add2(phi, phb);
  fx = add2(fx, fxb);
  fy = add2(fy, fyb);
  fz = add2(fz, fzb);
  return make_float4(lo(phi) + hi(phi), lo(fx) + hi(fx), lo(fy) + hi(fy), lo(fz) + hi(fz));
}

// UPD: pi_step (update + carried counts in the epilogue); TPL: targets per lane (1: walk9,
// 2: walk9x2), 0: cell groups (walk_flat)
template <int KERNEL, int NC, bool UPD, int TPL>
__global__ void __launch_bounds__((NC + 2) * 32, 1) k_interact_xpencil(XpParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int NSLOT = p.nslot, NOB = NSLOT + 1;
  unsigned long long *full = reinterpret_cast<unsigned long long *>(smem_raw);  // [nslot]
  unsigned long long *empty = full + MAX_SLOTS;                                  // [nslot]
  unsigned long long *ofull = empty + MAX_SLOTS;                                 // [nslot + 1]
  unsigned long long *oempty = ofull + MAX_SLOTS + 1;                            // [nslot + 1]
  int *obitem = reinterpret_cast<int *>(oempty + MAX_SLOTS + 1);                 // [nslot + 1]
  int *olast = obitem + MAX_SLOTS + 1;                                           // [nslot + 1]
  unsigned char *slots = smem_raw + HDR;
  const int L = p.L, sx = p.sx, LF = lf_of(L, sx);
  int *obufs = reinterpret_cast<int *>(slots + (size_t)NSLOT * slot_bytes(p.capp));
  const int OBW = (int)(otab_bytes(L, sx) / 4);
  const Geom &g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long cand = 0, fallbacks = 0;

  if (tid == 0) {
    for (int k = 0; k < NSLOT; ++k) {
      mbar_init(&full[k], 1);    // producer lane 0 (arrive.expect_tx) + the TMA bytes
      mbar_init(&empty[k], NC);  // one arrival per consumer warp
    }
    for (int k = 0; k < NOB; ++k) {
      mbar_init(&ofull[k], 1);   // helper lane 0, after its copies landed
      mbar_init(&oempty[k], 1);  // producer lane 0, once the slots using the table are released
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NC + 1) {
    // ================================ helper: offsets tables ================================
    for (int i = 0;; ++i) {
      const int b = i % NOB;
      if (i >= NOB) mbar_wait_sleep(&oempty[b], ((i / NOB) - 1) & 1);
      long long item = 0;
      if (lane == 0) item = (long long)atomicAdd(&p.ctl->xp_items, 1ull);
      item = __shfl_sync(0xffffffffu, item, 0);
      const bool stop = item >= p.nitems;
      if (!stop) {
        prefetch_offsets(p, item, obufs + (size_t)b * OBW);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      if (lane == 0) {
        obitem[b] = stop ? -1 : (int)item;
        mbar_arrive(&ofull[b]);  // release: the table (and the item index)
      }
      if (stop) break;
    }
  } else if (warp == NC) {
    // ================================ producer ================================
    long long item = -1;
    int x0 = 0, Lseg = 0, cy = 0, cz = 0, ja = 1;
    int taken = 0, freed = 0, ob = 0;  // tables received / released; the current item's table
    for (unsigned use = 0;; ++use) {
      const int s = use % NSLOT;
      Slot sl = slot_at(slots, p.capp, s);
      XP_T(tb);
      // The round is prepared (offsets table, round, candidates, runs) before the slot is free:
      // none of it touches the slot, and the consumers waiting for this slot then wait only for
      // the TMA copies (measured: consumers idled ~12 % of their time in slot waits).
      auto wait_slot = [&]() {
        XP_T(t0);
        if (use >= NSLOT) {
          mbar_wait_sleep(&empty[s], ((use / NSLOT) - 1) & 1);  // consumers released it
          // every use up to use - NSLOT is released: free the tables no later use refers to
          while (freed < taken && olast[freed % NOB] <= (int)(use - NSLOT)) {
            if (lane == 0) mbar_arrive(&oempty[freed % NOB]);
            ++freed;
          }
        }
        XP_T(t1);
        XP_ADD(0, t0, t1);
        fence_proxy_async();  // their generic reads of the slot precede the writes below
      };
      const bool fresh = item < 0 || ja > Lseg;
      if (fresh) {
        ob = taken % NOB;
        mbar_wait_sleep(&ofull[ob], (taken / NOB) & 1);
        ++taken;
        item = obitem[ob];
        if (item < 0) {  // stop marker: consumers leave at the first one
          wait_slot();
          if (lane == 0) {
            sl.meta[0] = 1;
            mbar_arrive(&full[s]);
          }
          break;
        }
        item_geom(p, item, x0, Lseg, cy, cz);
        ja = 1;
      }
      // (a next round of the same item reuses its table)
      sl.O = obufs + (size_t)ob * OBW;
      if (lane == 0) olast[ob] = (int)use;
      int jb = choose_round(p, sl, ja, Lseg);
      // a cell whose window alone does not fit the slot is listed for the Par-Cell-SM pass
      // (interact_cellsm.cu) and skipped; an item that ends in such cells leaves an empty round
      while (jb < ja && ja <= Lseg) {
        if (lane == 0) {
          const unsigned long long k = atomicAdd(&p.ctl->pad[0], 1ull);
          p.dense[k] = (x0 - 1 + ja) + g.nx * (cy + g.ny * cz);
          ++fallbacks;
        }
        ++ja;
        if (ja <= Lseg) jb = choose_round(p, sl, ja, Lseg);
      }
      const bool none = ja > Lseg;  // empty round (no targets)
      if (none) jb = ja - 1;
      // the round's 27-cell candidates (the unit of the metric, R4): n_j (c27_j - 1) per target
      // cell j (the fallback round's targets count their own)
      for (int j = ja + lane; j <= jb; j += 32) {
        int c27 = 0;
#pragma unroll
        for (int r = 0; r < 9; ++r) c27 += sl.O[r * LF + (j + 2) * sx] - sl.O[r * LF + (j - 1) * sx];
        const int nj = sl.O[4 * LF + (j + 1) * sx] - sl.O[4 * LF + j * sx];
        cand += (unsigned long long)nj * (unsigned long long)(c27 - 1);
      }
      // run of pencil r: cells ja-1 .. jb+1 (just cell ja's window for a fallback round)
      const int last = jb < ja ? ja : jb;
      int a = 0, len = 0;  // pairs of pencil run `lane`
      if (lane < 9 && !none) {
        a = sl.O[lane * LF + (ja - 1) * sx] >> 1;
        len = ((sl.O[lane * LF + (last + 2) * sx] + 1) >> 1) - a;
      }
      int incl = len;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 8);
      wait_slot();
      if (lane < 9) {
        sl.rb[lane] = incl - len;
        sl.rb[16 + lane] = incl - len - a;
      }
      if (lane == 0) {
        sl.rb[9] = total;
        sl.meta[0] = 0;
        sl.meta[1] = ja;
        sl.meta[2] = jb;
        sl.meta[3] = none ? 0 : sl.O[4 * LF + (last + 1) * sx] - sl.O[4 * LF + ja * sx];
        sl.meta[4] = x0;
        sl.meta[5] = cy | (cz << 16);
        sl.meta[6] = 0;
        sl.meta[7] = ob;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[s], (unsigned)total * 32u);  // release: tables
      __syncwarp();
      if (lane < 9 && len > 0) {
        bulk_g2s(sl.S + (incl - len), p.pairs + a, (unsigned)len * 16u, &full[s]);
        bulk_g2s(sl.SB + (incl - len), p.pairs + p.plane + a, (unsigned)len * 16u, &full[s]);
      }
      ja = last + 1;
      XP_T(t2);
      XP_ADD(1, tb, t2);  // (the whole iteration, the slot wait included)
      XP_ADD(2, 0, 1);
    }
  } else {
    // ================================ consumers ================================
    // in vector registers (a shuffle cannot be rematerialised): read from the constant bank,
    // ptxas reloaded them into uniform registers in every iteration of the walk (3 LDCU + MOV
    // of 47 instructions per 2 source pairs)
    const float thr = __shfl_sync(0xffffffffu, p.kp.rc2, 0), mc2 = __shfl_sync(0xffffffffu, -p.kp.c2, 0);
    for (unsigned use = 0;; ++use) {
      const int s = use % NSLOT;
      Slot sl = slot_at(slots, p.capp, s);
      XP_T(c0);
      mbar_wait(&full[s], (use / NSLOT) & 1);
      XP_T(c1);
      XP_ADD(3, c0, c1);
      if (sl.meta[0]) break;  // out of work items
      sl.O = obufs + (size_t)sl.meta[7] * OBW;
      const int ja = sl.meta[1], jb = sl.meta[2], ntargets = sl.meta[3], x0 = sl.meta[4];
      const int cy = sl.meta[5] & 0xffff, cz = sl.meta[5] >> 16;
      const int *O4 = sl.O + 4 * LF;  // home pencil; cell boundary j at O4[j sx]
      const int t0 = O4[ja * sx];       // global sorted index of the round's first target
      // global fine X index of the item's cell 0 (fine boundaries of the tables start there)
      const int f0 = (x0 - 1 + g.gx_off) * sx;
      const float rc = p.kp.rc;
      // target setup: its cell j (last j in [ja, jb] with O4[j sx] <= gs), its record (from the
      // staged home pencil) and its X sub-cell window [klo, khi] (reading R18: the fine index is
      // monotone in x and x_t -/+ r_c are rounded outward, so every skipped source has
      // |dx| >= r_c exactly; the CANDIDATE test kernel counts every candidate: no pruning)
      auto setup = [&](int gs, int &j, int &sub, float4 &me, int &klo, int &khi) {
        const int tp = sl.rb[16 + 4] + (gs >> 1);  // the target's staged pair
        const float4 ua = sl.S[tp], ub = sl.SB[tp];
        me = (gs & 1) ? make_float4(ua.y, ua.w, ub.y, ub.w) : make_float4(ua.x, ua.z, ub.x, ub.z);
        bool bad = false;
        // its cell and X sub-cell from its position: the binning's own contract (C3) on the
        // same fp32 value, so no search in the offsets table
        const int fg = fine_x_global(g, me.x, bad);
        j = (fg >> g.sxs) - g.gx_off - (x0 - 1);
        sub = fg & (sx - 1);
        const int flo = fine_x_global(g, __fsub_rd(me.x, rc), bad) - f0;
        const int fhi = fine_x_global(g, __fadd_ru(me.x, rc), bad) - f0;
        klo = KERNEL == PI_K_CANDIDATE ? (j - 1) * sx : min(max(flo, (j - 1) * sx), (j + 2) * sx - 1);
        khi = KERNEL == PI_K_CANDIDATE ? (j + 2) * sx - 1 : min(max(fhi, (j - 1) * sx), (j + 2) * sx - 1);
      };
      // epilogue: the target's fine cell (moves of the update are counted against it without
      // recomputing it from the position), the output.  (The 27-cell candidates, the unit of
      // the metric, are counted per cell by the producer.)
      auto finish = [&](int gs, int j, int sub, const float4 &me, const float4 &r) {
        int fold = -1;
        if (UPD && p.out.pcounts) fold = ((x0 - 1 + j) * sx + sub) + ((g.nx * (cy + g.ny * cz)) << g.sxs);
        if (kern_wforce(KERNEL)) {
          const float sc = -me.w * p.kp.f_ts;  // the walk summed wf (x_s - x_t)
          write_output<UPD>(p.out, g, gs, me, r.x * p.kp.phi_scale, sc * r.y, sc * r.z, sc * r.w, fold);
        } else if (KERNEL == PI_K_LOWFLOP) {
          write_output<UPD>(p.out, g, gs, me, r.x, r.y, r.z, r.w, fold);
        } else {
          write_output<UPD>(p.out, g, gs, me, r.x, 0.f, 0.f, 0.f, fold);
        }
      };
      if (TPL == 0) {
        // cell groups: a batch is one target cell j of the round (in chunks of <= 32 targets)
        int *wt = obufs + (size_t)NOB * OBW + warp * 32;
        for (;;) {
          int b = 0;
          if (lane == 0) b = atomicAdd(&sl.meta[6], 1);
          b = __shfl_sync(0xffffffffu, b, 0);
          const int j = ja + b;
          if (j > jb) break;
          const int cs = O4[j * sx], na = O4[(j + 1) * sx] - cs;
          for (int c0 = 0; c0 < na; c0 += 32) {
            const int nt = min(32, na - c0);
            const float rn = __frcp_rn((float)nt);
            const int k = (int)(32.5f * rn);               // floor(32 / nt)
            const int jj = (int)(((float)lane + 0.5f) * rn);  // floor(lane / nt)
            const int t = lane - jj * nt;
            const int gs = cs + c0 + t;
            int jt, sub, klo, khi;
            float4 me;
            setup(gs, jt, sub, me, klo, khi);
            klo = __reduce_min_sync(0xffffffffu, klo);
            khi = __reduce_max_sync(0xffffffffu, khi);
            // the union window's 9 runs as one sequence of staged pairs
            int np = 0, p0 = 0;
            if (lane < 9) {
              const int a = sl.O[lane * LF + klo], e = sl.O[lane * LF + khi + 1];
              if (e > a) {
                p0 = sl.rb[16 + lane] + (a >> 1);
                np = sl.rb[16 + lane] + ((e - 1) >> 1) - p0 + 1;
              }
            }
            int incl = np;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
              const int v = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += v;
            }
            const int Np = __shfl_sync(0xffffffffu, incl, 8);
            if (lane < 9) {
              wt[lane] = incl;
              wt[16 + lane] = p0 - (incl - np);
            }
            __syncwarp();
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (jj < k) r = walk_flat<KERNEL>(sl, wt, Np, jj, k, me, thr, mc2, p.kp);
            // the k partial sums of each target (lanes t, t + nt, ...), tree over jj
            for (int m = 1; m < k; m <<= 1) {
              const float ox = __shfl_down_sync(0xffffffffu, r.x, m * nt);
              const float oy = __shfl_down_sync(0xffffffffu, r.y, m * nt);
              const float oz = __shfl_down_sync(0xffffffffu, r.z, m * nt);
              const float ow = __shfl_down_sync(0xffffffffu, r.w, m * nt);
              if ((jj & (2 * m - 1)) == 0 && jj + m < k) {
                r.x += ox;
                r.y += oy;
                r.z += oz;
                r.w += ow;
              }
            }
            if (jj == 0) {
              const float4 st = self_terms<KERNEL>(me, p.kp);  // the self pair's exact term
              r = make_float4(r.x - st.x, r.y - st.y, r.z - st.z, r.w - st.w);
              finish(gs, jt, sub, me, r);
            }
            __syncwarp();  // wt is rewritten by the next chunk
          }
        }
      } else
      for (;;) {
        int b = 0;
        if (lane == 0) b = atomicAdd(&sl.meta[6], 32 * TPL);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (b >= ntargets) break;
        const int T = b + lane * TPL;  // the lane's first target (TPL consecutive ones)
        if (T < ntargets) {
          const int gs = t0 + T;  // (rounds always have jb >= ja: cells that do not fit are listed)
          if (TPL == 1) {
            int j, sub, klo, khi;
            float4 me;
            setup(gs, j, sub, me, klo, khi);
            const float4 r = p.mask ? walk9<KERNEL, true>(sl, LF, sx, ja, klo, khi, me, thr, mc2, p.kp)
                                    : walk9<KERNEL, false>(sl, LF, sx, ja, klo, khi, me, thr, mc2, p.kp);
            finish(gs, j, sub, me, r);
          } else {
            // two consecutive sorted targets: their fine cells are equal or adjacent (the sorted
            // order is the fine-cell order), so the union of their windows is 5-6 sub-cells
            const bool two = T + 1 < ntargets;
            int j0, s0, klo0, khi0, j1, s1, klo1, khi1;
            float4 me0, me1;
            setup(gs, j0, s0, me0, klo0, khi0);
            setup(two ? gs + 1 : gs, j1, s1, me1, klo1, khi1);
            float4 r0, r1;
            walk9x2<KERNEL>(sl, LF, sx, ja, min(klo0, klo1), max(khi0, khi1), me0, me1, thr, mc2, p.kp, r0, r1);
            finish(gs, j0, s0, me0, r0);
            if (two) finish(gs + 1, j1, s1, me1, r1);
          }
        }
      }
      __syncwarp();
      XP_T(c2);
      XP_ADD(4, c1, c2);
      XP_ADD(5, 0, 1);
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }

  // the dense cells listed so far by the producers of all blocks (Par-Cell-SM, cellsm.cuh), in
  // the staging memory this block no longer uses; the rest is left to k_cellsm_list
  __syncthreads();
  {
    CsParams cp;
    cp.rec = p.rec;
    cp.pairs = p.pairs;
    cp.plane = p.plane;
    cp.offsets = p.offsets;
    cp.list = p.dense;
    cp.g = p.g;
    cp.kp = p.kp;
    cp.out = p.out;
    cp.ctl = p.ctl;
    cp.from_rec = false;
    cellsm_phase<KERNEL, UPD, (NC + 2) * 32>(cp, slots);
  }

  // statistics: warp-level sums, spread over CAND_SLOTS counters
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cand += __shfl_xor_sync(0xffffffffu, cand, o);
    fallbacks += __shfl_xor_sync(0xffffffffu, fallbacks, o);
  }
  if (lane == 0) {
    if (cand) atomicAdd(&p.ctl->cand_slots[(blockIdx.x * (NC + 2) + warp) & (CAND_SLOTS - 1)], cand);
    if (fallbacks) atomicAdd(&p.ctl->fallback_cells, fallbacks);
  }
}

template <int NC>
cudaError_t launch_nc(const XpParams &p, cudaStream_t s) {
  const size_t smem = max(xp_smem_bytes(p.L, p.capp, p.sx, p.nslot), CS_SMEM + HDR);
  constexpr int NT = (NC + 2) * 32;  // consumers, producer, helper
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = allow_max_smem(kern);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (occ < 1) occ = 1;
    long long blocks = (long long)sms * occ - p.reserve;
    if (blocks > p.nitems) blocks = p.nitems;
    if (blocks < 1) blocks = 1;
    kern<<<(int)blocks, NT, smem, s>>>(p);
    return cudaGetLastError();
  };
  const bool upd = p.out.upd != nullptr;
  // two targets per lane for the cutoff kernels (walk9x2 relies on exact exclusion outside a
  // target's own window); the CANDIDATE test kernel and masked grids walk one target per lane
  const bool two = p.tpl == 2 && !p.mask;
  const bool grp = p.tpl == 0 && !p.mask;  // cell groups (walk_flat): the cutoff kernels
  if (grp) {
    switch (p.kp.kernel) {
      case PI_K_GAUSSIAN: return upd ? go(k_interact_xpencil<PI_K_GAUSSIAN, NC, true, 0>) : go(k_interact_xpencil<PI_K_GAUSSIAN, NC, false, 0>);
      case PI_K_INDICATOR: return upd ? go(k_interact_xpencil<PI_K_INDICATOR, NC, true, 0>) : go(k_interact_xpencil<PI_K_INDICATOR, NC, false, 0>);
      case PI_K_LJ: return upd ? go(k_interact_xpencil<PI_K_LJ, NC, true, 0>) : go(k_interact_xpencil<PI_K_LJ, NC, false, 0>);
      case PI_K_LOWFLOP: return upd ? go(k_interact_xpencil<PI_K_LOWFLOP, NC, true, 0>) : go(k_interact_xpencil<PI_K_LOWFLOP, NC, false, 0>);
      case PI_K_HIGHFLOP: return upd ? go(k_interact_xpencil<PI_K_HIGHFLOP, NC, true, 0>) : go(k_interact_xpencil<PI_K_HIGHFLOP, NC, false, 0>);
      default: break;  // CANDIDATE: one target per lane (masked ends)
    }
  }
  switch (p.kp.kernel) {
    case PI_K_GAUSSIAN:
      if (two) return upd ? go(k_interact_xpencil<PI_K_GAUSSIAN, NC, true, 2>) : go(k_interact_xpencil<PI_K_GAUSSIAN, NC, false, 2>);
      return upd ? go(k_interact_xpencil<PI_K_GAUSSIAN, NC, true, 1>) : go(k_interact_xpencil<PI_K_GAUSSIAN, NC, false, 1>);
    case PI_K_INDICATOR:
      if (two) return upd ? go(k_interact_xpencil<PI_K_INDICATOR, NC, true, 2>) : go(k_interact_xpencil<PI_K_INDICATOR, NC, false, 2>);
      return upd ? go(k_interact_xpencil<PI_K_INDICATOR, NC, true, 1>) : go(k_interact_xpencil<PI_K_INDICATOR, NC, false, 1>);
    case PI_K_LJ:
      if (two) return upd ? go(k_interact_xpencil<PI_K_LJ, NC, true, 2>) : go(k_interact_xpencil<PI_K_LJ, NC, false, 2>);
      return upd ? go(k_interact_xpencil<PI_K_LJ, NC, true, 1>) : go(k_interact_xpencil<PI_K_LJ, NC, false, 1>);
    case PI_K_LOWFLOP:
      return upd ? go(k_interact_xpencil<PI_K_LOWFLOP, NC, true, 1>) : go(k_interact_xpencil<PI_K_LOWFLOP, NC, false, 1>);
    case PI_K_HIGHFLOP:
      return upd ? go(k_interact_xpencil<PI_K_HIGHFLOP, NC, true, 1>) : go(k_interact_xpencil<PI_K_HIGHFLOP, NC, false, 1>);
    default:
      return upd ? go(k_interact_xpencil<PI_K_CANDIDATE, NC, true, 1>)
                 : go(k_interact_xpencil<PI_K_CANDIDATE, NC, false, 1>);
  }
}

// the cells listed for Par-Cell-SM that no X-pencil block took before it left (cellsm.cuh)
cudaError_t launch_dense_rest(const XpParams &p, cudaStream_t s) {
  CsParams cp;
  cp.rec = p.rec;
  cp.pairs = p.pairs;
  cp.plane = p.plane;
  cp.offsets = p.offsets;
  cp.list = p.dense;
  cp.g = p.g;
  cp.kp = p.kp;
  cp.out = p.out;
  cp.ctl = p.ctl;
  cp.from_rec = false;
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

cudaError_t launch_interact_xpencil(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  XpParams p;
  p.rec = a.rec;
  p.offsets = a.offsets;
  p.g = g;
  p.kp = k;
  p.out = a.out;
  p.ctl = a.ctl;
  // the target X layers: the owned ones, or the caller's ranges (a8 overlap: the slab's boundary
  // layers first, then the interior while the exchange runs)
  int xr[4] = {g.own_lo, g.own_hi, 0, 0};
  if (a.xr_set)
    for (int k = 0; k < 4; ++k) xr[k] = a.xr[k];
  const int own = max(xr[1] - xr[0], xr[3] - xr[2]);
  if (own <= 0) return cudaSuccess;
  for (int k = 0; k < 4; ++k) p.xr[k] = xr[k];
  p.reserve = a.reserve_sms;
  auto segs = [&]() {
    p.nseg0 = (xr[1] - xr[0] + p.L - 1) / p.L;
    p.nseg = p.nseg0 + (xr[3] - xr[2] + p.L - 1) / p.L;
    p.nitems = (long long)p.nseg * g.ny * g.nz;
  };
  // segment length: ~512 targets per item at the mean density (64 cells at 8 per cell, up to
  // 256 at 2 or fewer), so a slot feeds the consumer warps at low densities too (configs[2]
  // ppc 1: 7.0 -> 3.8 ms with 256 instead of 64; ppc 4: 2.43 -> 1.88 ms with 128)
  const double ppc_mean = (double)a.n_est / (double)g.ncells;
  const int l_auto = ppc_mean >= 8.0 ? 64 : (ppc_mean >= 4.0 ? 128 : 256);
  p.L = a.tx_len > 0 ? a.tx_len : l_auto;
  if (p.L > 512) p.L = 512;
  if (p.L > own) p.L = own;
  segs();
  p.foffsets = a.foffsets;
  p.sx = g.sx;
  p.mask = k.kernel == PI_K_CANDIDATE || g.nx < 4;
  const int nc = a.threads > 0 ? a.threads / 32 : 20;
  p.nslot = a.slots >= 2 ? min(a.slots, MAX_SLOTS) : 2;
  p.dense = a.dense;
  // targets per lane: 1 (one per lane), 2 (two per lane, measured slower), 0 (cell
  // groups, walk_flat; tuning value 3)
  p.tpl = a.tpl == 2 ? 2 : (a.tpl == 3 ? 0 : 1);
  const size_t max_smem = 227 * 1024;
  // the segment must leave room for slots of a useful size: the fixed tables (offsets per X
  // sub-cell boundary of every slot and of the prefetch stage) grow with L * sx (ADVICE r01:
  // L = 256 with sx = 16 did not fit at all).  Halve L until two slots hold the windows of a
  // few cells at the mean density.
  auto fixed_of = [&](int L) {
    return HDR + (size_t)(p.nslot + 1) * otab_bytes(L, p.sx) + (size_t)p.nslot * slot_words() * 4 + WT_BYTES;
  };
  const size_t min_slot = (size_t)(9 * 8 * (ppc_mean + 4.0)) * 16 + 1024;  // ~8 cells' windows
  while (p.L > 8 && fixed_of(p.L) + (size_t)p.nslot * min_slot > max_smem) p.L = (p.L + 1) / 2;
  segs();
  int cap = a.tx_cap;
  if (cap <= 0) {
    // every slot as large as shared memory allows (one block per SM either way): rows through
    // dense regions then need fewer rounds and list fewer cells (clustered configs[3]: -7 %;
    // measured the same as the mean occupancy + 15 % on uniform input), but no more than the
    // particles there are
    const size_t fixed = fixed_of(p.L);
    const long long fit = max_smem > fixed ? (long long)((max_smem - fixed) / ((size_t)p.nslot * 32)) : 16;
    cap = (int)min(2 * fit - 18, a.n_est + 64);
  }
  p.capp = max(16, cap / 2 + 9);  // + one partial pair per run
  while (xp_smem_bytes(p.L, p.capp, p.sx, p.nslot) > max_smem && p.capp > 64) p.capp -= 32;
  if (xp_smem_bytes(p.L, p.capp, p.sx, p.nslot) > max_smem) return cudaErrorNotSupported;
  p.pairs = a.pairs;
  p.plane = a.pair_plane;
  if (!a.pairs_ready) {  // the AoS binning (pi_step) writes the pairs itself
    const long long np = (a.n + 1) / 2;
    int blocks = (int)min((np + 255) / 256, 148LL * 16);
    k_pairify<<<max(blocks, 1), 256, 0, s>>>(a.n, a.n_dev, a.rec, a.pairs, a.pair_plane);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = nc <= 8 ? launch_nc<8>(p, s) : (nc <= 16 ? launch_nc<16>(p, s) : launch_nc<20>(p, s));
  if (e != cudaSuccess) return e;
  return launch_dense_rest(p, s);
}

}  // namespace pi
