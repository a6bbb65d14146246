// Internal declarations of libpi (sm_100a).  Not part of the ABI (see include/pi.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pi.h"

namespace pi {

// ------------------------------------------------------------------------------------
// Geometry and kernel constants, passed by value to every kernel.
// ------------------------------------------------------------------------------------
struct Geom {
  float ox, oy, oz;   // origin of the GLOBAL grid (the cell contract is evaluated globally)
  float w, inv_w;     // cell width and fl32(1/w) (contract C3)
  int nx, ny, nz;     // LOCAL grid dims (nx = owned X layers + 2 ghost layers when nranks > 1)
  long long ncells;   // local cells
  int gnx;            // global dims[0]
  int gx_off;         // global X index of local X cell 0 (-1 + rank * Lx when nranks > 1)
  int own_lo, own_hi; // owned local X cells [own_lo, own_hi): targets of the interaction
  int sx, sxs;        // X sub-cells per cell of the binning order (1, 2, 4, 8, 16), sx = 1 << sxs
  float hx, hy, hz;   // upper faces of the global box (integration walls)
  float lx, ly, lz;   // lower faces
};

struct KParams {
  int kernel;         // pi_kernel
  float rc, rc2;
  float sigma, inv_s2;  // 1/sigma^2
  float c2;             // log2(e) / (2 sigma^2): K = 2^(-c2 r^2)
  float s, s_inv;       // sqrt(c2) and 1/sqrt(c2)
  float lj_inv_r2, lj_e2;  // Lennard-Jones: 1/r^2 and eps^2/r^2, so (d~/r)^2 = d^2 lj_inv_r2 + lj_e2
  // Output scales: phi = phi_scale sum w;  F = q_t f_ts sum wf (x_t - x_s), where a source
  // contributes w = q_s K (Gaussian; K = 2^(-c2 r^2)) or q_s (s^6 - s^3) (LJ), and
  // wf = w (Gaussian) or q_s (12 s^5 - 6 s^2) (LJ):  Gaussian 1, 1/sigma^2;  LJ 4 E0, -4 E0 / r^2
  float phi_scale, f_ts;
};

// Device-resident control / statistics block (in the workspace).
struct DevCtl {
  int scan_tile_ctr;     // dynamic tile ids of the look-back scan
  int scan_done_ctr;     // blocks finished (last one resets)
  unsigned scan_epoch;   // tags the look-back status words of one launch
  int mc_slot[2];        // atomicMax slots for M_C, indexed by epoch parity
  int max_per_cell;      // M_C of the last scan
  int flags;             // sticky error bits
  int pad0;
  // X-slab state (nranks > 1), device resident so no host synchronisation is needed
  long long n_owned, n_total;         // owned particles; owned + ghost particles (binned)
  long long n_stay;                   // stayers after the position update (migration)
  long long migrants_in, migrants_out, ghosts_in;
  long long pad2[2];
  // everything from here on is reset before each interaction
  unsigned long long fallback_cells;
  unsigned long long xp_items;        // X-pencil work-item counter (reset before each launch)
  unsigned long long pad[4];         // X-pencil dense cells: listed [0], Par-Cell-SM ticket [1],
                                      // blocks whose producer finished [2]
  unsigned long long cand_slots[64];  // candidates (C) of the last interaction, spread counters
  unsigned long long pairs;           // cutoff pairs (P) counted by pi_count_pairs
};
constexpr int CAND_SLOTS = 64;

enum : int { FLAG_OUT_OF_BOX = 1, FLAG_CAPACITY = 2, FLAG_INTERNAL = 4, FLAG_DOMAIN = 8 };

// ------------------------------------------------------------------------------------
// a1: cell index, contract C3: c = clamp(floor(fl32(fl32(x - o) * inv_w)), 0, N - 1).
// __fsub_rn / __fmul_rn forbid FMA contraction, so the result is bit-identical to the
// per-operation-rounded definition.  A position outside [o, o + N w] (NaN included) maps to
// the nearest cell and raises FLAG_OUT_OF_BOX (pi.h: positions must lie in the box; the upper
// face itself clamps into the last cell, with a 2^-20 relative slack for its rounding).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ bool outside(float t, int nd) { return !(t >= 0.f && t <= (float)nd * 1.000001f); }
__device__ __forceinline__ int cell_coord(float x, float o, float inv_w, int nd, bool &bad) {
  float t = __fmul_rn(__fsub_rn(x, o), inv_w);
  float f = floorf(t);
  bad |= outside(t, nd);
  int c = (f >= 0.f) ? ((f < (float)nd) ? (int)f : nd - 1) : 0;
  return c;
}

// Local X cell: the global contract, then the slab offset (clamped into the local grid).
__device__ __forceinline__ int cell_x(const Geom &g, float x, bool &bad) {
  const int c = cell_coord(x, g.ox, g.inv_w, g.gnx, bad) - g.gx_off;
  return min(max(c, 0), g.nx - 1);
}

__device__ __forceinline__ int cell_lin(const Geom &g, float x, float y, float z, bool &bad) {
  int cx = cell_x(g, x, bad);
  int cy = cell_coord(y, g.oy, g.inv_w, g.ny, bad);
  int cz = cell_coord(z, g.oz, g.inv_w, g.nz, bad);
  return cx + g.nx * (cy + g.ny * cz);
}

// Fine (sub-cell) X index on the GLOBAL grid: c sx + floor(sx (t - c)), t = fl32(fl32(x - o)
// inv_w) the contract's scaled coordinate and c its cell.  t - c is exact (t in [c, c+1)) and
// sx a power of two, so the index is monotone in x and agrees with the cell contract.
__device__ __forceinline__ int fine_x_global(const Geom &g, float x, bool &bad) {
  const float t = __fmul_rn(__fsub_rn(x, g.ox), g.inv_w);
  const float f = floorf(t);
  bad |= outside(t, g.gnx);
  const int c = (f >= 0.f) ? ((f < (float)g.gnx) ? (int)f : g.gnx - 1) : 0;
  const int sub = min(max((int)((t - (float)c) * (float)g.sx), 0), g.sx - 1);
  return (c << g.sxs) + sub;
}

// Linear FINE cell (the binning order): X sub-cell fastest inside the cell, then the cell
// linearisation; cells outside the local slab clamp into the ghost layers like cell_lin.
__device__ __forceinline__ int fine_lin(const Geom &g, float x, float y, float z, bool &bad) {
  const int fg = fine_x_global(g, x, bad);
  const int cl = (fg >> g.sxs) - g.gx_off;
  const int fx = cl < 0 ? 0 : (cl >= g.nx ? (g.nx << g.sxs) - 1 : (cl << g.sxs) + (fg & (g.sx - 1)));
  const int cy = cell_coord(y, g.oy, g.inv_w, g.ny, bad);
  const int cz = cell_coord(z, g.oz, g.inv_w, g.nz, bad);
  return fx + ((g.nx * (cy + g.ny * cz)) << g.sxs);
}

__device__ __forceinline__ float ex2_approx(float a) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Integration (a7, reading C11): x' = x + dt F, reflect at the walls, clamp into [lo, hi).
__device__ __forceinline__ float integrate1(float x, float f, float dt, float lo, float hi) {
  float y = fmaf(dt, f, x);
  if (y < lo) y = lo + (lo - y);
  if (y >= hi) y = hi - (y - hi);
  const float below = __int_as_float(__float_as_int(hi) - 1);  // largest float < hi (hi > 0)
  y = fminf(fmaxf(y, lo), below);
  return y;
}

// ------------------------------------------------------------------------------------
// Output descriptor of the interaction kernels.
// ------------------------------------------------------------------------------------
// a3 scans fine counts in tiles of 2^SCAN_TILE_SHIFT (binning.cu)
constexpr int SCAN_TILE_SHIFT = 12;

struct OutDesc {
  float4 *sorted;          // [n] (phi, fx, fy, fz) in sorted order (always written)
  const int32_t *perm;     // sorted slot -> caller index (NULL: no caller-order outputs)
  float *phi, *fx, *fy, *fz;  // caller order (each nullable)
  // pi_step: write integrated positions in sorted order
  float4 *upd;             // NULL: no integration
  const int32_t *sid;
  int32_t *uid;
  float dt;
  // persistent per-sub-cell counts of the sorted state (nullable): a particle whose fine cell
  // changes in the update moves one count from its old to its new fine cell
  int32_t *pcounts;
  int32_t *ptsum;          // their per-scan-tile sums (kept current with them)
  int *flags;              // the context's sticky device flags (DevCtl::flags)
};

// UPD = false compiles the pi_step update out (kernels specialised for pi_interact).
// f_old: the target's fine cell if the caller knows it (else -1: computed from rec).
template <bool UPD = true>
__device__ __forceinline__ void write_output(const OutDesc &o, const Geom &g, int t, float4 rec, float phi,
                                             float fx, float fy, float fz, int f_old = -1) {
  o.sorted[t] = make_float4(phi, fx, fy, fz);
  if (o.perm) {
    const int c = o.perm[t];
    if (c >= 0) {  // -1: not a particle of the caller's pi_bin input (ghost)
      if (o.phi) o.phi[c] = phi;
      if (o.fx) o.fx[c] = fx;
      if (o.fy) o.fy[c] = fy;
      if (o.fz) o.fz[c] = fz;
    }
  }
  if (UPD && o.upd) {
    float4 u;
    u.x = integrate1(rec.x, fx, o.dt, g.lx, g.hx);
    u.y = integrate1(rec.y, fy, o.dt, g.ly, g.hy);
    u.z = integrate1(rec.z, fz, o.dt, g.lz, g.hz);
    u.w = rec.w;
    // a non-finite update (NaN / inf force) would be clamped onto the lower wall by integrate1:
    // raise the sticky out-of-box / NaN flag instead of moving it silently
    if (!(isfinite(fmaf(o.dt, fx, rec.x)) && isfinite(fmaf(o.dt, fy, rec.y)) && isfinite(fmaf(o.dt, fz, rec.z))) &&
        o.flags)
      atomicOr(o.flags, FLAG_OUT_OF_BOX);
    o.upd[t] = u;
    o.uid[t] = o.sid[t];
    if (o.pcounts) {
      bool bad = false;
      const int f0 = f_old >= 0 ? f_old : fine_lin(g, rec.x, rec.y, rec.z, bad);
      const int f1 = fine_lin(g, u.x, u.y, u.z, bad);
      if (f1 != f0) {
        atomicSub(o.pcounts + f0, 1);
        atomicAdd(o.pcounts + f1, 1);
        if ((f0 >> SCAN_TILE_SHIFT) != (f1 >> SCAN_TILE_SHIFT)) {
          atomicSub(o.ptsum + (f0 >> SCAN_TILE_SHIFT), 1);
          atomicAdd(o.ptsum + (f1 >> SCAN_TILE_SHIFT), 1);
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// Launchers (host side, in the .cu files).
// ------------------------------------------------------------------------------------
constexpr int PART_NB = 1024;  // max buckets of the partitioned pi_bin (2 per thread in its scan)

// float4 elements per plane of the f32x2 source-pair array of a context of `cap` particles
// (plane A = (x, x, y, y), plane B = (z, z, q, q) of source pairs; 128-B aligned planes)
__host__ __device__ inline long long pair_plane_of(long long cap) {
  if (cap < 1) cap = 1;
  return ((cap / 2 + 1) + 7) & ~7LL;
}

struct BinArgs {
  long long n;                  // particles (upper bound when n_dev is set)
  const long long *n_dev;       // device-resident count (nranks > 1), or NULL
  const float *x, *y, *z, *q;   // SoA input (pi_bin), or NULL when rec_in is used
  const float4 *rec_in;         // AoS input (pi_step re-binning)
  const int32_t *id_in;         // ids (NULL -> index)
  float4 *tmp_rec;              // SoA path scratch [n]: records partitioned into buckets
  int32_t *tmp_idx;             // SoA path scratch [n]: their caller indices
  int32_t *bucket_cur;          // SoA path scratch [PART_NB]: bucket fill cursors
  int32_t *counts;              // [ncells sx] fine counts, zero on entry and again after the binning
  int32_t *offsets;             // [ncells + 1] per cell
  int32_t *foffsets;            // [ncells sx + 1] per fine cell (the sorted order)
  unsigned long long *tile_status;
  int num_tiles_cap;
  float4 *rec_out;              // sorted records (x, y, z, q); NULL: only pairs_out (AoS path)
  int32_t *sid_out;             // sorted ids
  int32_t *perm_out;            // sorted slot -> input index (nullable)
  const int32_t *perm_in;       // AoS path: input index per record (-1 = ghost), or NULL
  float4 *pairs_out;            // AoS input, nullable: also write the sorted records as f32x2 source pairs
                                // (layout of InteractArgs::pairs)
  long long pair_plane;         // float4 elements per plane of the pair array
  int32_t *pcounts;             // [ncells sx] persistent counts of the sorted state (one rank)
  int32_t *ptsum;               // [scan tiles] their per-tile sums (written by the count paths'
                                // scan, kept current by the pi_step update)
  bool delta;                   // AoS re-binning from pcounts (kept current by the pi_step update)
  DevCtl *ctl;
};

cudaError_t launch_bin(const Geom &g, const BinArgs &a, cudaStream_t s);
int scan_tiles(long long nitems);

struct InteractArgs {
  long long n;                  // particles in the sorted state (upper bound if n_dev)
  const long long *n_dev;       // device-resident count (nranks > 1), or NULL
  long long n_est;              // host estimate of the sorted count (sizes staging buffers)
  const float4 *rec;            // sorted records (NULL when only the pair array is current)
  float4 *pairs;                // two planes of pair_plane float4 each: the records as f32x2 source
                                // pairs, A[k] = (x_2k, x_2k+1, y_2k, y_2k+1), B[k] = (z.., z.., q.., q..)
                                // at pairs[k] and pairs[pair_plane + k]
  long long pair_plane;         // >= n / 2 + 1
  bool pairs_ready;             // pairs already hold the current sorted state (AoS binning)
  const int32_t *offsets;       // [ncells + 1]
  const int32_t *foffsets;      // [ncells sx + 1] fine offsets (X sub-cells)
  OutDesc out;
  DevCtl *ctl;
  int tx_len, tx_cap, threads, slots;  // tuning (x-pencil)
  int tpl;                      // tuning (x-pencil): targets per lane (0 = default)
  int32_t *dense;               // [ncells] cells listed by the X-pencil for the Par-Cell-SM pass
  int fb[3], fb_cap;            // tuning (full load)
  bool xr_set;                  // X-pencil: only the target X layers [xr0, xr1) + [xr2, xr3)
  int xr[4];                    //   (local; else every owned layer)
  int reserve_sms;              // X-pencil: SMs left free for kernels overlapping the launch
};

// Lets `func` use the device's whole opt-in shared memory.  The attribute is process-global
// per function, so it is always set to the same (maximum) value: contexts on other host
// threads launching with other sizes never see it lowered under them.
template <typename F>
inline cudaError_t allow_max_smem(F *func) {
  int dev = 0, mx = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  return e;
}

cudaError_t launch_interact_global(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s);
cudaError_t launch_interact_xpencil(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s);
cudaError_t launch_interact_xpencil2(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s);
cudaError_t launch_interact_fullload(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s);
cudaError_t launch_interact_xpreg(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s);
// P: ordered pairs (i, j), j != i, r_ij < r_c, over the owned targets of the sorted state -> ctl->pairs
cudaError_t launch_count_pairs(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s);
cudaError_t launch_interact_half(const Geom &g, const KParams &k, const InteractArgs &a, cudaStream_t s);

}  // namespace pi
