// a1-a4: binning of the particles into the cell grid (§2, Fig. 1).
//
//   k_count   a1 + a2: cell index from the position ("without moving the particles",
//             :60) and per-cell counts "by using atomic operations" (:62), at X sub-cell
//             granularity (R18).
//   k_scan    a3: "prefix sum ... where the particles that belong to a given cell should
//             be located" (:63) -- one pass, decoupled look-back over tiles of 4096
//             counts, warp-shuffle scans inside a tile; also M_C, "the maximum number of
//             particles in a cell" retained while computing the prefix sum (:242).
//   k_scatter a4: "move the particles in a secondary array (not in-place)" (:64): slot =
//             offsets[cell] + rank, the rank taken from the kept counts with an atomicSub
//             ("using again atomic operations", :64), which leaves the counts zero for the
//             next binning; one 16-byte (x, y, z, q) record + id per particle, and the same
//             record in the f32x2 source-pair layout the X-pencil stages.
//   AoS input (pi_step re-binning of the nearly sorted updated state, slab input): the count
//             and the scatter aggregate over runs of equal cells among consecutive lanes
//             (shuffle + ballot), one atomic per run.  pi_step with one rank skips the count:
//             the update keeps the persistent counts current (delta re-binning).
//   SoA input (pi_bin, arbitrary order): a direct scatter would write every 16-B record into
//             its own DRAM sector (10x the traffic, measured); k_partition first groups the
//             particles into buckets of consecutive cells with coalesced runs, and the scatter
//             then fills one bucket's region of the sorted order at a time, in L2.
#include <algorithm>

#include "pi_internal.cuh"

namespace pi {

namespace {

constexpr int COUNT_THREADS = 256;
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096 cells per tile
static_assert(SCAN_TILE == (1 << SCAN_TILE_SHIFT), "scan tile");

// a1 + a2 over SoA input (pi_bin, arbitrary order): 4 particles per thread through float4
// loads, warp-aggregated atomics (one per distinct (sub-)cell among the warp's lanes).
// Runs of equal cells among consecutive lanes (the nearly sorted AoS input): one atomic per
// run.  Returns the run's first lane and length for this lane (invalid lanes: runs of one).
__device__ __forceinline__ void lane_run(int lin, bool valid, int &head, int &len) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int key = valid ? lin : -1 - lane;
  const int prev = __shfl_up_sync(full, key, 1);
  const unsigned heads = __ballot_sync(full, lane == 0 || prev != key);
  head = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));  // last head at or below this lane
  const unsigned above = heads & ~(0xffffffffu >> (31 - lane));  // heads above this lane
  const int next = above ? __ffs(above) - 1 : 32;
  len = next - head;
}

// Count pass of the AoS path: one atomicAdd per run of equal cells.
__device__ __forceinline__ void run_count(int32_t *counts, int lin, bool valid) {
  int head, len;
  lane_run(lin, valid, head, len);
  if (valid && (int)(threadIdx.x & 31) == head) atomicAdd(counts + lin, len);
}

__global__ void __launch_bounds__(COUNT_THREADS) k_count_soa(long long n, const float *__restrict__ x,
                                                              const float *__restrict__ y,
                                                              const float *__restrict__ z, Geom g,
                                                              int32_t *__restrict__ counts, DevCtl *ctl) {
  const long long nvec = (n + 3) >> 2;
  const int lane = threadIdx.x & 31;
  bool bad = false;
  // whole warps iterate together (the run aggregation shuffles over all 32 lanes)
  for (long long vb = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); vb < nvec;
       vb += (long long)gridDim.x * blockDim.x) {
    const long long v = vb + lane;
    const long long i0 = v << 2;
    float xs[4] = {0.f, 0.f, 0.f, 0.f}, ys[4] = {0.f, 0.f, 0.f, 0.f}, zs[4] = {0.f, 0.f, 0.f, 0.f};
    if (i0 + 3 < n) {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(x) + v);
      const float4 b = __ldg(reinterpret_cast<const float4 *>(y) + v);
      const float4 c = __ldg(reinterpret_cast<const float4 *>(z) + v);
      xs[0] = a.x; xs[1] = a.y; xs[2] = a.z; xs[3] = a.w;
      ys[0] = b.x; ys[1] = b.y; ys[2] = b.z; ys[3] = b.w;
      zs[0] = c.x; zs[1] = c.y; zs[2] = c.z; zs[3] = c.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool ok = i0 + j < n;
        xs[j] = ok ? x[i0 + j] : 0.f;
        ys[j] = ok ? y[i0 + j] : 0.f;
        zs[j] = ok ? z[i0 + j] : 0.f;
      }
    }
    // warp-aggregated atomics (north star step 2): one atomicAdd per run of equal (sub-)cells
    // among consecutive lanes (particle j of lane l and of lane l + 1 are 4 apart in the input):
    // cell-ordered or clustered input adds whole runs at once, random order costs a shuffle and
    // a ballot per particle
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool valid = i0 + j < n;
      bool b = false;
      const int lin = valid ? fine_lin(g, xs[j], ys[j], zs[j], b) : -1;
      bad |= b;
      run_count(counts, lin, valid);
    }
  }
  if (bad) atomicOr(&ctl->flags, FLAG_OUT_OF_BOX);
}

// Scatter of the AoS path: a distinct rank in [0, count) per particle, taken from the counts
// with one atomicSub per run (which leaves the counts zero).
__device__ __forceinline__ int run_take(int32_t *counts, int lin, bool valid) {
  int head, len;
  lane_run(lin, valid, head, len);
  const int lane = threadIdx.x & 31;
  int top = 0;
  if (valid && lane == head) top = atomicSub(counts + lin, len);
  top = __shfl_sync(0xffffffffu, top, head);
  return top - len + (lane - head);
}

// a1 + a2 over AoS records (pi_step re-binning of the updated sorted state): counts only,
// one atomic per run of equal cells in a warp.
__global__ void __launch_bounds__(COUNT_THREADS) k_count_aos(long long n, const float4 *__restrict__ rec, Geom g,
                                                              int32_t *__restrict__ counts, DevCtl *ctl,
                                                              const long long *n_dev) {
  if (n_dev) n = *n_dev;
  bool bad = false;
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < n; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    const bool ok = i < n;
    const float4 r = ok ? __ldg(rec + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    bool b = false;
    const int lin = fine_lin(g, r.x, r.y, r.z, b);
    bad |= ok && b;
    run_count(counts, lin, ok);
  }
  if (bad) atomicOr(&ctl->flags, FLAG_OUT_OF_BOX);
}

// ---------------------------------------------------------------------------------
// a3: single-pass prefix scan with decoupled look-back.
// Status word per tile: [epoch:30 | flag:2 | value:32]; flag 1 = tile aggregate,
// 2 = inclusive prefix.  The epoch (bumped by the last block of each launch) makes
// stale words of earlier launches invisible, so the status array is never cleared.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// The scan runs over the FINE counts (X sub-cells, sx per cell; sx divides SCAN_ITEMS, so a
// thread's items are whole cells): it writes the fine offsets (the sorted order) and every
// sx-th of them as the per-cell offsets; M_C is the largest per-cell sum.
// KEEP: leave the counts (the scatter consumes them);  copy: nullable, receives the counts read
// (pi_bin: the persistent counts of the new sorted state; delta re-binning: the scatter's copy).
template <bool KEEP>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan(long long ncells, int32_t *__restrict__ counts,
                                                       int32_t *__restrict__ offsets,
                                                       unsigned long long *__restrict__ status, int num_tiles,
                                                       DevCtl *ctl, int sxs, int32_t *__restrict__ cell_offsets,
                                                       int32_t *__restrict__ copy, int32_t *__restrict__ tsum) {
  const int sx = 1 << sxs;
  __shared__ int s_tile;
  __shared__ int s_warp[SCAN_THREADS / 32];
  __shared__ int s_prefix;
  __shared__ unsigned s_epoch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_tile = atomicAdd(&ctl->scan_tile_ctr, 1);
    s_epoch = *((volatile unsigned *)&ctl->scan_epoch);
  }
  __syncthreads();
  const int tile = s_tile;
  const unsigned long long etag = ((unsigned long long)(s_epoch & 0x3fffffffu)) << 34;
  const long long base = (long long)tile * SCAN_TILE + (long long)tid * SCAN_ITEMS;

  int v[SCAN_ITEMS];
  if (base + SCAN_ITEMS <= ncells) {
    int4 *p = reinterpret_cast<int4 *>(counts + base);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS / 4; ++k) {
      int4 a = p[k];
      v[4 * k] = a.x; v[4 * k + 1] = a.y; v[4 * k + 2] = a.z; v[4 * k + 3] = a.w;
      if (!KEEP) p[k] = make_int4(0, 0, 0, 0);  // leave zeroed counts for the next binning
      if (copy) reinterpret_cast<int4 *>(copy + base)[k] = a;
    }
  } else {
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      long long c = base + k;
      v[k] = c < ncells ? counts[c] : 0;
      if (!KEEP && c < ncells) counts[c] = 0;
      if (copy && c < ncells) copy[c] = v[k];
    }
  }
  int mx = 0, sum = 0, grp = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    sum += v[k];
    grp += v[k];
    if (((k + 1) & (sx - 1)) == 0) {  // end of a cell
      mx = max(mx, grp);
      grp = 0;
    }
  }
  // warp inclusive scan of the thread sums
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 31) s_warp[warp] = incl;
  if (lane == 0) atomicMax(&ctl->mc_slot[s_epoch & 1], mx);
  __syncthreads();
  if (warp == 0) {
    int ws = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0;
    int wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - ws;  // exclusive warp offsets
    int tile_total = __shfl_sync(0xffffffffu, wi, SCAN_THREADS / 32 - 1);
    if (tsum && lane == 0) tsum[tile] = tile_total;  // the tile sums of the copy (delta re-binning)
    // publish the aggregate, then look back
    int prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed(status + tile, etag | (2ull << 32) | (unsigned)tile_total);
    } else {
      if (lane == 0) st_relaxed(status + tile, etag | (1ull << 32) | (unsigned)tile_total);
      int look = tile - 1;
      while (true) {
        int t = look - lane;
        unsigned long long w = 0;
        unsigned flag = 0;
        if (t >= 0) {
          do {
            w = ld_relaxed(status + t);
            flag = ((w >> 34) == (etag >> 34)) ? (unsigned)((w >> 32) & 3ull) : 0u;
          } while (flag == 0);
        } else {
          flag = 2;  // below tile 0: nothing
        }
        unsigned incl_mask = __ballot_sync(0xffffffffu, flag == 2);
        int first = incl_mask ? __ffs(incl_mask) - 1 : 32;   // nearest inclusive predecessor
        int val = (t >= 0 && lane <= first) ? (int)(unsigned)(w & 0xffffffffull) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (first < 32) break;
        look -= 32;
      }
      if (lane == 0) st_relaxed(status + tile, etag | (2ull << 32) | (unsigned)(prefix + tile_total));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  int run = s_prefix + s_warp[warp] + incl - sum;
  int outv[SCAN_ITEMS];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) { outv[k] = run; run += v[k]; }
  if (base + SCAN_ITEMS <= ncells) {
    int4 *p = reinterpret_cast<int4 *>(offsets + base);  // offsets is 16-B aligned
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS / 4; ++k)
      p[k] = make_int4(outv[4 * k], outv[4 * k + 1], outv[4 * k + 2], outv[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
      if (base + k < ncells) offsets[base + k] = outv[k];
  }
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k += 1)  // per-cell offsets: every sx-th fine offset
    if ((k & (sx - 1)) == 0 && base + k < ncells) cell_offsets[(base + k) >> sxs] = outv[k];
  if (base <= ncells - 1 && ncells - 1 < base + SCAN_ITEMS) {  // offsets[Nc] = N
    offsets[ncells] = run;
    cell_offsets[ncells >> sxs] = run;
  }
  // last block: publish M_C, reset counters, advance the epoch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    int done = atomicAdd(&ctl->scan_done_ctr, 1);
    if (done == num_tiles - 1) {
      __threadfence();
      unsigned e = s_epoch;
      int m = atomicAdd(&ctl->mc_slot[e & 1], 0);
      ctl->max_per_cell = m;
      ctl->mc_slot[(e + 1) & 1] = 0;
      ctl->scan_tile_ctr = 0;
      ctl->scan_done_ctr = 0;
      __threadfence();
      atomicAdd(&ctl->scan_epoch, 1u);
    }
  }
}

// a3 for the pi_step re-binning: the persistent counts come with their per-tile sums (kept
// current by the update, like the counts), so a tile's prefix is the sum of the tile sums
// before it -- at most a few thousand L2-resident ints per block -- and no tile waits on
// another (the look-back of k_scan was measured as ~30 % of its stall samples, 37 us at 2^24);
// M_C goes straight into ctl->max_per_cell (zeroed before the launch): no last-block step.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_delta(long long ncells, const int32_t *__restrict__ counts,
                                                             const int32_t *__restrict__ tsum,
                                                             int32_t *__restrict__ offsets,
                                                             DevCtl *ctl, int sxs, int32_t *__restrict__ cell_offsets,
                                                             int32_t *__restrict__ copy) {
  const int sx = 1 << sxs;
  __shared__ int s_warp[SCAN_THREADS / 32];
  __shared__ int s_pre[SCAN_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;
  const long long base = (long long)tile * SCAN_TILE + (long long)tid * SCAN_ITEMS;
  int v[SCAN_ITEMS];
  if (base + SCAN_ITEMS <= ncells) {
    const int4 *p = reinterpret_cast<const int4 *>(counts + base);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS / 4; ++k) {
      const int4 a = p[k];
      v[4 * k] = a.x; v[4 * k + 1] = a.y; v[4 * k + 2] = a.z; v[4 * k + 3] = a.w;
      reinterpret_cast<int4 *>(copy + base)[k] = a;
    }
  } else {
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      const long long c = base + k;
      v[k] = c < ncells ? counts[c] : 0;
      if (c < ncells) copy[c] = v[k];
    }
  }
  int pre = 0;  // sum of the tile sums before this tile
  for (int k = tid; k < tile; k += SCAN_THREADS) pre += __ldcg(tsum + k);
  int mx = 0, sum = 0, grp = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    sum += v[k];
    grp += v[k];
    if (((k + 1) & (sx - 1)) == 0) {
      mx = max(mx, grp);
      grp = 0;
    }
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    pre += __shfl_xor_sync(0xffffffffu, pre, o);
  }
  if (lane == 31) s_warp[warp] = incl;
  if (lane == 0) s_pre[warp] = pre;
  __syncthreads();
  if (lane == 0) atomicMax(&ctl->max_per_cell, mx);  // zeroed before the launch (launch_bin)
  int woff = 0, prefix = 0;
#pragma unroll
  for (int w = 0; w < SCAN_THREADS / 32; ++w) {
    woff += w < warp ? s_warp[w] : 0;
    prefix += s_pre[w];
  }
  int run = prefix + woff + incl - sum;
  int outv[SCAN_ITEMS];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) { outv[k] = run; run += v[k]; }
  if (base + SCAN_ITEMS <= ncells) {
    int4 *p = reinterpret_cast<int4 *>(offsets + base);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS / 4; ++k)
      p[k] = make_int4(outv[4 * k], outv[4 * k + 1], outv[4 * k + 2], outv[4 * k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
      if (base + k < ncells) offsets[base + k] = outv[k];
  }
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k += 1)
    if ((k & (sx - 1)) == 0 && base + k < ncells) cell_offsets[(base + k) >> sxs] = outv[k];
  if (base <= ncells - 1 && ncells - 1 < base + SCAN_ITEMS) {  // offsets[Nc] = N
    offsets[ncells] = run;
    cell_offsets[ncells >> sxs] = run;
  }
}

// a4, first pass on arbitrary-order input: partition into coarse buckets (2^bsh consecutive
// cells each; a bucket's region of the sorted order starts at offsets[b << bsh]).  A block
// takes a tile of PART_TILE particles, sorts it by bucket in shared memory and writes each
// bucket's run contiguously (reserved with one atomic per bucket), so the writes are
// coalesced; the second pass then scatters inside one bucket's region at a time, which
// stays in L2 (a direct scatter writes every 16-B record into its own DRAM sector).
constexpr int PART_THREADS = 512;
constexpr int PART_PER = 8;
constexpr int PART_TILE = PART_THREADS * PART_PER;
constexpr size_t PART_SMEM = PART_TILE * (sizeof(float4) + sizeof(int32_t) + sizeof(uint16_t)) +
                             3 * PART_NB * sizeof(int32_t);

__global__ void __launch_bounds__(PART_THREADS) k_partition(long long n, const float *__restrict__ x,
                                                             const float *__restrict__ y,
                                                             const float *__restrict__ z,
                                                             const float *__restrict__ q, Geom g, int bsh, int nb,
                                                             const int32_t *__restrict__ offsets,
                                                             int32_t *__restrict__ bucket_cur,
                                                             float4 *__restrict__ tmp_rec,
                                                             int32_t *__restrict__ tmp_idx) {
  extern __shared__ __align__(16) unsigned char smem[];
  float4 *s_rec = reinterpret_cast<float4 *>(smem);
  int32_t *s_idx = reinterpret_cast<int32_t *>(s_rec + PART_TILE);
  int32_t *hist = s_idx + PART_TILE;
  int32_t *loc = hist + PART_NB;
  int32_t *gb = loc + PART_NB;
  uint16_t *s_b = reinterpret_cast<uint16_t *>(gb + PART_NB);
  __shared__ int s_wsum[PART_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t0 = (long long)blockIdx.x * PART_TILE;
  for (int j = tid; j < nb; j += PART_THREADS) hist[j] = 0;
  __syncthreads();
  float4 r[PART_PER];
  int bk[PART_PER], rk[PART_PER];
#pragma unroll
  for (int k = 0; k < PART_PER; ++k) {
    const long long i = t0 + k * PART_THREADS + tid;
    bk[k] = -1;
    if (i < n) {
      r[k] = make_float4(__ldg(x + i), __ldg(y + i), __ldg(z + i), __ldg(q + i));
      bool bad = false;
      bk[k] = (fine_lin(g, r[k].x, r[k].y, r[k].z, bad) >> g.sxs) >> bsh;
      rk[k] = atomicAdd(hist + bk[k], 1);
    }
  }
  __syncthreads();
  // exclusive scan of the bucket histogram (2 buckets per thread); reserve each bucket's run
  const int j0 = 2 * tid, j1 = 2 * tid + 1;
  const int h0 = j0 < nb ? hist[j0] : 0, h1 = j1 < nb ? hist[j1] : 0;
  int incl = h0 + h1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int ws = lane < PART_THREADS / 32 ? s_wsum[lane] : 0;
    int wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < PART_THREADS / 32) s_wsum[lane] = wi - ws;
  }
  __syncthreads();
  const int ex = s_wsum[warp] + incl - h0 - h1;
  if (j0 < nb) {
    loc[j0] = ex;
    gb[j0] = h0 ? offsets[(long long)j0 << bsh] + atomicAdd(bucket_cur + j0, h0) : 0;
  }
  if (j1 < nb) {
    loc[j1] = ex + h0;
    gb[j1] = h1 ? offsets[(long long)j1 << bsh] + atomicAdd(bucket_cur + j1, h1) : 0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PART_PER; ++k)
    if (bk[k] >= 0) {
      const int pos = loc[bk[k]] + rk[k];
      s_rec[pos] = r[k];
      s_idx[pos] = (int32_t)(t0 + k * PART_THREADS + tid);
      s_b[pos] = (uint16_t)bk[k];
    }
  __syncthreads();
  const int cnt = (int)min((long long)PART_TILE, n - t0);
  for (int pos = tid; pos < cnt; pos += PART_THREADS) {
    const int b = s_b[pos];
    const int dst = gb[b] + pos - loc[b];
    tmp_rec[dst] = s_rec[pos];
    tmp_idx[dst] = s_idx[pos];
  }
}

// a4: out-of-place scatter of AoS records (pi_step re-binning, slab input, or the buckets of
// the partitioned pi_bin), ranks taken from the counts.  GATHER: perm_in maps the record to
// the caller's index, whose id is id_in[perm_in[i]] (partitioned pi_bin).
template <bool GATHER>
__global__ void __launch_bounds__(COUNT_THREADS) k_scatter(long long n, const float4 *__restrict__ rec_in,
                                                            const int32_t *__restrict__ id_in, Geom g,
                                                            int32_t *__restrict__ counts,
                                                            const int32_t *__restrict__ offsets,
                                                            float4 *__restrict__ rec_out,
                                                            int32_t *__restrict__ sid_out,
                                                            int32_t *__restrict__ perm_out,
                                                            const int32_t *__restrict__ perm_in,
                                                            const long long *n_dev,
                                                            float *__restrict__ pairs_out = nullptr,
                                                            long long plane = 0) {
  if (n_dev) n = *n_dev;
  if (!GATHER) {
    // two records per thread and iteration (i, i + blockDim.x): the two dependent chains
    // (record -> cell -> rank atomic -> offset -> stores) overlap
    const long long step = 2LL * gridDim.x * blockDim.x;
    for (long long i0 = 2LL * blockIdx.x * blockDim.x; i0 < n; i0 += step) {
      const long long ia = i0 + threadIdx.x, ib = ia + blockDim.x;
      const bool oka = ia < n, okb = ib < n;
      const float4 ra = oka ? __ldg(rec_in + ia) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 rb = okb ? __ldg(rec_in + ib) : make_float4(0.f, 0.f, 0.f, 0.f);
      const int32_t ida = oka ? (id_in ? __ldg(id_in + ia) : (int32_t)ia) : 0;
      const int32_t idb = okb ? (id_in ? __ldg(id_in + ib) : (int32_t)ib) : 0;
      bool b = false;
      const int lina = fine_lin(g, ra.x, ra.y, ra.z, b), linb = fine_lin(g, rb.x, rb.y, rb.z, b);
      const int rka = run_take(counts, lina, oka);
      const int rkb = run_take(counts, linb, okb);
      const int sa = oka ? __ldg(offsets + lina) + rka : 0, sb = okb ? __ldg(offsets + linb) + rkb : 0;
      auto put = [&](long long i, const float4 &r, int slot, int32_t id) {
        if (rec_out) rec_out[slot] = r;
        if (pairs_out) {
          float *pa = pairs_out + 4 * (long long)(slot >> 1) + (slot & 1);
          float *pb = pa + 4 * plane;
          pa[0] = r.x;
          pa[2] = r.y;
          pb[0] = r.z;
          pb[2] = r.w;
          if (slot == n - 1 && !(slot & 1)) {
            pa[1] = 1.0e30f;
            pa[3] = 1.0e30f;
            pb[1] = 1.0e30f;
            pb[3] = 0.f;
          }
        }
        sid_out[slot] = id;
        if (perm_out) perm_out[slot] = perm_in ? __ldg(perm_in + i) : (int32_t)i;
      };
      if (oka) put(ia, ra, sa, ida);
      if (okb) put(ib, rb, sb, idb);
    }
    return;
  }
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < n; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    const bool ok = i < n;
    const float4 r = ok ? __ldg(rec_in + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    bool b = false;
    const int lin = fine_lin(g, r.x, r.y, r.z, b);
    const int rk = run_take(counts, lin, ok);
    if (!ok) continue;
    int slot = __ldg(offsets + lin) + rk;  // fine offsets
    if (rec_out) rec_out[slot] = r;       // (pi_step with the X-pencil: the pair array only)
    if (pairs_out) {  // f32x2 source pairs: A[k] = (x0, x1, y0, y1), B[k] = (z0, z1, q0, q1), B = A + plane
      float *pa = pairs_out + 4 * (long long)(slot >> 1) + (slot & 1);
      float *pb = pa + 4 * plane;
      pa[0] = r.x;
      pa[2] = r.y;
      pb[0] = r.z;
      pb[2] = r.w;
      if (slot == n - 1 && !(slot & 1)) {  // odd count: an inert partner for the last record
        pa[1] = 1.0e30f;
        pa[3] = 1.0e30f;
        pb[1] = 1.0e30f;
        pb[3] = 0.f;
      }
    }
    if (GATHER) {
      const int32_t orig = __ldg(perm_in + i);
      sid_out[slot] = id_in ? __ldg(id_in + orig) : orig;
      perm_out[slot] = orig;
    } else {
      sid_out[slot] = id_in ? __ldg(id_in + i) : (int32_t)i;
      if (perm_out) perm_out[slot] = perm_in ? __ldg(perm_in + i) : (int32_t)i;
    }
  }
}

int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  long long cap = 148LL * 16;  // persistent-ish cap: 16 blocks per SM
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

int scan_tiles(long long nitems) { return (int)((nitems + SCAN_TILE - 1) / SCAN_TILE); }

cudaError_t launch_bin(const Geom &g, const BinArgs &a, cudaStream_t s) {
  const long long nf = g.ncells * g.sx;  // fine cells
  const int tiles = scan_tiles(nf);
  const int sgrid = grid_for(a.n, COUNT_THREADS);
  float *pairs = reinterpret_cast<float *>(a.pairs_out);
  if (a.delta) {  // pi_step re-binning from the persistent counts: no count pass
    cudaError_t e = cudaMemsetAsync(&a.ctl->max_per_cell, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    k_scan_delta<<<tiles, SCAN_THREADS, 0, s>>>(nf, a.pcounts, a.ptsum, a.foffsets, a.ctl, g.sxs, a.offsets,
                                                a.counts);
    if (a.n > 0)
      k_scatter<false><<<sgrid, COUNT_THREADS, 0, s>>>(a.n, a.rec_in, a.id_in, g, a.counts, a.foffsets, a.rec_out,
                                                       a.sid_out, a.perm_out, a.perm_in, a.n_dev, pairs,
                                                       a.pair_plane);
    return cudaGetLastError();
  }
  if (a.rec_in) {  // AoS: count, scan keeping the counts, scatter taking ranks from them
    if (a.n > 0)
      k_count_aos<<<sgrid, COUNT_THREADS, 0, s>>>(a.n, a.rec_in, g, a.counts, a.ctl, a.n_dev);
    k_scan<true><<<tiles, SCAN_THREADS, 0, s>>>(nf, a.counts, a.foffsets, a.tile_status, tiles, a.ctl, g.sxs,
                                                a.offsets, a.pcounts, a.pcounts ? a.ptsum : nullptr);
    if (a.n > 0)
      k_scatter<false><<<sgrid, COUNT_THREADS, 0, s>>>(a.n, a.rec_in, a.id_in, g, a.counts, a.foffsets, a.rec_out,
                                                       a.sid_out, a.perm_out, a.perm_in, a.n_dev, pairs,
                                                       a.pair_plane);
    return cudaGetLastError();
  }
  // SoA (pi_bin, arbitrary order): count, scan keeping the counts, partition into buckets of
  // ~2^17 particles (their sorted-order regions, records + ids, ~3 MB, stay in L2 while the
  // second pass scatters into them), scatter each bucket taking ranks from the counts.  This
  // pass is bound by L2 requests (~7 per particle); the pair array's four scattered 4-B
  // stores would double them, so pi_bin leaves it to the X-pencil's first launch (k_pairify).
  // 2^24 random-order particles: 2.2 ms as one direct scatter, 0.82 ms this way.
  if (a.n > 0)
    k_count_soa<<<grid_for((a.n + 3) / 4, COUNT_THREADS), COUNT_THREADS, 0, s>>>(a.n, a.x, a.y, a.z, g, a.counts,
                                                                                 a.ctl);
  k_scan<true><<<tiles, SCAN_THREADS, 0, s>>>(nf, a.counts, a.foffsets, a.tile_status, tiles, a.ctl, g.sxs,
                                              a.offsets, a.pcounts, a.pcounts ? a.ptsum : nullptr);
  if (a.n == 0) return cudaGetLastError();
  const long long want = std::min<long long>(PART_NB, std::max<long long>(1, a.n >> 17));
  int bsh = 0;
  while (((g.ncells + (1LL << bsh) - 1) >> bsh) > want) ++bsh;
  const int nb = (int)((g.ncells + (1LL << bsh) - 1) >> bsh);
  cudaError_t e = cudaMemsetAsync(a.bucket_cur, 0, sizeof(int32_t) * nb, s);
  if (e != cudaSuccess) return e;
  // (a constant value, so concurrent contexts on several host threads agree)
  if ((e = cudaFuncSetAttribute(k_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PART_SMEM)) !=
      cudaSuccess)
    return e;
  k_partition<<<(int)((a.n + PART_TILE - 1) / PART_TILE), PART_THREADS, PART_SMEM, s>>>(
      a.n, a.x, a.y, a.z, a.q, g, bsh, nb, a.offsets, a.bucket_cur, a.tmp_rec, a.tmp_idx);
  // one record per thread, blocks in order: the records in flight are a contiguous stretch of
  // buckets (a grid-stride loop with more blocks than fit would spread them over all buckets)
  k_scatter<true><<<(int)((a.n + COUNT_THREADS - 1) / COUNT_THREADS), COUNT_THREADS, 0, s>>>(a.n, a.tmp_rec, a.id_in, g, a.counts, a.foffsets, a.rec_out,
                                                  a.sid_out, a.perm_out, a.tmp_idx, nullptr, nullptr);
  return cudaGetLastError();
}

}  // namespace pi
