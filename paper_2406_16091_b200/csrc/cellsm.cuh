// Par-Cell-SM (§4.4, Alg. 3) for the DENSE cells of the X-pencil pass.
//
// The X-pencil stages a row segment's 9 neighbour pencils at the mean density; a cell whose
// window alone does not fit one staging slot (clustered input: configs[3] reaches 367
// particles per cell) is listed by the X-pencil producer instead of being computed there, and
// this phase, which every block of the X-pencil kernel runs once its own X-pencil work is
// done, takes the list -- a compacted list of the cells that need it, so no
// block ever visits an empty cell (the paper's "if there are empty cells, they should be
// removed", :95-96).  As in Alg. 3, one block owns one target cell, its threads own the
// targets, and the neighbour cells' particles pass through shared memory "in several steps,
// such that even if there are many particles per cell, this approach remains efficient"
// (:185-187).  B200 specifics:
//   * the 27 neighbour cells are the 9 contiguous 3-cell runs of the X-fastest order, staged
//     as f32x2 source pairs (planes A, B of the sorted state) in chunks of CS_CHUNK pairs with
//     16-B cp.async copies; the out-of-run halves of a run's end pairs are made inert in
//     shared memory (q = 0, x = 1e30), so every kernel, CANDIDATE included, sees exactly the
//     27 cells;
//   * every thread reads the same staged pair at the same time (shared-memory broadcast) and
//     evaluates it for one or two targets (f32x2 over the source pair, src_eval);
//   * the self pair is evaluated (d = 0) and its exact term removed, as in the X-pencil.
#pragma once
#include "interact_common.cuh"

namespace pi {

constexpr int CS_CHUNK = 2048;  // staged source pairs per step (planes A + B: 64 KB)
constexpr size_t CS_SMEM = sizeof(float4) * 2 * CS_CHUNK + sizeof(int) * 48;

struct CsParams {
  const float4 *rec;    // sorted records, or NULL (then from the pair array)
  const float4 *pairs;  // pair planes A | B
  long long plane;
  const int32_t *offsets;
  bool from_rec;           // stage from the records (full load: the pair array may be stale)
  int32_t *list;           // listed cells (local linear ids), -1 when free
  Geom g;
  KParams kp;
  OutDesc out;
  DevCtl *ctl;
};

// staged pairs q0, q0 + G, q0 + 2G, ... of the chunk (G source groups, see cs_targets)
template <int KERNEL, int TPT>
__device__ __forceinline__ void cs_compute(const float4 *__restrict__ A, const float4 *__restrict__ B, int n,
                                           int q0, int G, const float4 *me, const float thr, const float mc2,
                                           const KParams &kp, p2 (*acc)[4]) {
  int q = q0;
  for (; q + G < n; q += 2 * G) {
    const SrcPair s0 = load_pair(A, B, q), s1 = load_pair(A, B, q + G);
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      src_eval<KERNEL>(s0, me[k].x, me[k].y, me[k].z, thr, mc2, acc[k][0], acc[k][1], acc[k][2], acc[k][3], &kp);
      src_eval<KERNEL>(s1, me[k].x, me[k].y, me[k].z, thr, mc2, acc[k][0], acc[k][1], acc[k][2], acc[k][3], &kp);
    }
  }
  if (q < n) {
    const SrcPair s0 = load_pair(A, B, q);
#pragma unroll
    for (int k = 0; k < TPT; ++k)
      src_eval<KERNEL>(s0, me[k].x, me[k].y, me[k].z, thr, mc2, acc[k][0], acc[k][1], acc[k][2], acc[k][3], &kp);
  }
}

// Targets tbase .. of the cell: TPT per thread, or (TPT = 1, a cell of at most NT / 2 targets)
// G source groups of NT / G threads, group g taking every G-th staged pair, so a small cell
// keeps every thread busy; the groups' partial sums meet in shared memory at the end.
template <int KERNEL, bool UPD, int TPT, int NT>
__device__ void cs_targets(const CsParams &p, int t0, int tbase, int nt, int P, const int *rstart, const int *rpa,
                           const int *ra, const int *rb, float4 *A, float4 *B) {
  const int tid = threadIdx.x;
  const float thr = p.kp.rc2, mc2 = -p.kp.c2;
  const int G = TPT == 1 ? max(1, min(4, NT / max(nt - tbase, 1))) : 1, tpg = NT / G;
  const int gi = tid / tpg, ti = tid - gi * tpg;  // source group, target slot in the group
  float4 me[TPT];
  bool ok[TPT];
  p2 acc[TPT][4];
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const int t = tbase + ti + k * NT;
    ok[k] = gi < G && t < nt;
    me[k] = ok[k] ? sorted_rec(p.rec, p.pairs, p.plane, t0 + t) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[k][c] = pk(0.f);
  }
  const bool any = ok[0];  // targets are assigned in thread order: a warp without one skips
  for (int cbase = 0; cbase < P; cbase += CS_CHUNK) {
    const int n = min(CS_CHUNK, P - cbase);
    __syncthreads();  // the previous chunk is consumed
    for (int i = tid; i < n; i += NT) {
      const int ci = cbase + i;
      int r = 0;
      while (r < 8 && rstart[r + 1] <= ci) ++r;
      const long long gp = (long long)rpa[r] + (ci - rstart[r]);
      if (p.from_rec) {  // the pair from two records; halves outside the run are inert
        const float4 inert = make_float4(1.0e30f, 1.0e30f, 1.0e30f, 0.f);
        const long long k0 = 2 * gp, k1 = k0 + 1;
        const float4 u = (k0 >= ra[r] && k0 < rb[r]) ? __ldg(p.rec + k0) : inert;
        const float4 v = (k1 >= ra[r] && k1 < rb[r]) ? __ldg(p.rec + k1) : inert;
        A[i] = make_float4(u.x, v.x, u.y, v.y);
        B[i] = make_float4(u.z, v.z, u.w, v.w);
      } else {
        cp_async16(A + i, p.pairs + gp);
        cp_async16(B + i, p.pairs + p.plane + gp);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    if (tid < 9 && rstart[tid + 1] > rstart[tid]) {  // inert out-of-run halves of run tid's end pairs
      const int r = tid;
      const int f = rstart[r] - cbase, l = rstart[r + 1] - 1 - cbase;
      if ((ra[r] & 1) && f >= 0 && f < n) {
        A[f].x = 1.0e30f; A[f].z = 1.0e30f; B[f].x = 1.0e30f; B[f].z = 0.f;
      }
      if ((rb[r] & 1) && l >= 0 && l < n) {
        A[l].y = 1.0e30f; A[l].w = 1.0e30f; B[l].y = 1.0e30f; B[l].w = 0.f;
      }
    }
    __syncthreads();
    if (any) cs_compute<KERNEL, TPT>(A, B, n, gi, G, me, thr, mc2, p.kp, acc);
  }
  if (G > 1) {  // the groups' partial sums, summed by group 0 (reusing the staging buffer)
    __syncthreads();
    float4 *red = A;
    if (ok[0] && gi > 0)
      red[(gi - 1) * tpg + ti] = make_float4(lo(acc[0][0]) + hi(acc[0][0]), lo(acc[0][1]) + hi(acc[0][1]),
                                             lo(acc[0][2]) + hi(acc[0][2]), lo(acc[0][3]) + hi(acc[0][3]));
    __syncthreads();
    if (ok[0] && gi == 0) {
      for (int h = 1; h < G; ++h) {
        const float4 v = red[(h - 1) * tpg + ti];
        acc[0][0] = add2(acc[0][0], pk(v.x, 0.f));
        acc[0][1] = add2(acc[0][1], pk(v.y, 0.f));
        acc[0][2] = add2(acc[0][2], pk(v.z, 0.f));
        acc[0][3] = add2(acc[0][3], pk(v.w, 0.f));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    if (!ok[k] || gi > 0) continue;
    const float4 st = self_terms<KERNEL>(me[k], p.kp);  // identity exclusion (Alg. 1 :127)
    const float phi = lo(acc[k][0]) + hi(acc[k][0]) - st.x;
    const float sx_ = lo(acc[k][1]) + hi(acc[k][1]) - st.y, sy_ = lo(acc[k][2]) + hi(acc[k][2]) - st.z;
    const float sz_ = lo(acc[k][3]) + hi(acc[k][3]) - st.w;
    const int t = t0 + tbase + ti + k * NT;
    if (kern_wforce(KERNEL)) {
      const float sc = -me[k].w * p.kp.f_ts;  // the walk summed wf (x_s - x_t)
      write_output<UPD>(p.out, p.g, t, me[k], phi * p.kp.phi_scale, sc * sx_, sc * sy_, sc * sz_);
    } else if (KERNEL == PI_K_LOWFLOP) {
      write_output<UPD>(p.out, p.g, t, me[k], phi, sx_, sy_, sz_);
    } else {
      write_output<UPD>(p.out, p.g, t, me[k], phi, 0.f, 0.f, 0.f);
    }
  }
}

// The dense-cell phase: every thread of the block (NT of them) runs it.  A block claims listed
// cells one at a time (compare-and-swap on the ticket counter, so a ticket is only ever taken
// for a cell already counted in the list) and leaves as soon as no listed cell is left: it never
// waits for other blocks, so there is no assumption that the whole grid is resident (ADVICE r01:
// the X-pencil blocks used to wait for every block's producer, which can deadlock when grids of
// concurrent launches share the GPU).  The X-pencil runs the phase opportunistically after its
// own items; the cells listed after a block left are computed by k_cellsm_list, launched after
// the X-pencil kernel (the list is final then).  An entry is published by its value (entries are
// -1 when free: a reader waits for its reserved entry -- the producer that reserved it is running
// and writes it next -- then frees it for the next launch).
template <int KERNEL, bool UPD, int NT>
__device__ void cellsm_phase(const CsParams &p, unsigned char *smem) {
  float4 *A = reinterpret_cast<float4 *>(smem), *B = A + CS_CHUNK;
  int *rstart = reinterpret_cast<int *>(A + 2 * CS_CHUNK);  // [10]
  int *rpa = rstart + 10, *ra = rpa + 9, *rb = ra + 9;      // [9] each
  int *s_sh = rb + 9;                                        // item, n, cell
  const int tid = threadIdx.x;
  const Geom &g = p.g;
  volatile unsigned long long *cnt = &p.ctl->pad[0], *tick = &p.ctl->pad[1];
  volatile int *list = p.list;
  for (;;) {
    __syncthreads();  // the previous cell's shared tables are no longer read
    if (tid == 0) {
      long long t = -1;
      int cell = -1;
      for (;;) {
        const unsigned long long tk = *tick;
        if (tk >= *cnt) break;  // nothing listed left
        if (atomicCAS(&p.ctl->pad[1], tk, tk + 1) == tk) {
          t = (long long)tk;
          while ((cell = list[t]) < 0) __nanosleep(32);
          list[t] = -1;
          break;
        }
      }
      s_sh[2] = cell;
      s_sh[0] = (int)t;
    }
    __syncthreads();
    const int c = s_sh[2], item = s_sh[0];
    if (c < 0) break;
    const int cx = c % g.nx, cy = (c / g.nx) % g.ny, cz = c / (g.nx * g.ny);
    if (tid < 9) {  // run tid: cells cx-1 .. cx+1 of row (cy + dy, cz + dz), clamped (open box)
      const int y = cy + (tid % 3) - 1, z = cz + (tid / 3) - 1;
      int a = 0, b = 0;
      if (y >= 0 && y < g.ny && z >= 0 && z < g.nz) {
        const long long row = (long long)g.nx * (y + (long long)g.ny * z);
        a = __ldg(p.offsets + row + max(cx - 1, 0));
        b = __ldg(p.offsets + row + min(cx + 1, g.nx - 1) + 1);
      }
      ra[tid] = a;
      rb[tid] = b;
      rpa[tid] = a >> 1;
      rstart[tid + 1] = b > a ? ((b - 1) >> 1) - (a >> 1) + 1 : 0;  // pairs of the run
    }
    __syncthreads();
    if (tid == 0) {
      rstart[0] = 0;
      int recs = 0;
      for (int r = 0; r < 9; ++r) {
        rstart[r + 1] += rstart[r];
        recs += rb[r] - ra[r];
      }
      const int t0 = __ldg(p.offsets + c), nt = __ldg(p.offsets + c + 1) - t0;
      s_sh[1] = nt;
      // the 27-cell candidates of the cell's targets (the unit of the metric, R4)
      atomicAdd(&p.ctl->cand_slots[(blockIdx.x + item) & (CAND_SLOTS - 1)],
                (unsigned long long)nt * (unsigned long long)(recs - 1));
    }
    __syncthreads();
    const int nt = s_sh[1], t0 = __ldg(p.offsets + c), P = rstart[9];
    for (int tbase = 0; tbase < nt; tbase += 2 * NT) {
      if (nt - tbase > NT)
        cs_targets<KERNEL, UPD, 2, NT>(p, t0, tbase, nt, P, rstart, rpa, ra, rb, A, B);
      else
        cs_targets<KERNEL, UPD, 1, NT>(p, t0, tbase, nt, P, rstart, rpa, ra, rb, A, B);
    }
  }
}

// The same pass as a kernel of its own, after a non-persistent kernel has listed its cells
// (full load: a block whose sub-box does not fit lists the box's non-empty cells).
template <int KERNEL, bool UPD>
__global__ void __launch_bounds__(256) k_cellsm_list(CsParams p) {
  extern __shared__ __align__(16) unsigned char cs_raw[];
  cellsm_phase<KERNEL, UPD, 256>(p, cs_raw);
}

}  // namespace pi
