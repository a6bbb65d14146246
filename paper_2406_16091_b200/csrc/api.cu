// C ABI of libpi (include/pi.h): context, workspace carving, call sequencing.
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <new>

#include "pi_internal.cuh"
#include "slab.cuh"

using namespace pi;

namespace {

constexpr int RH_SETS = 3;  // pipelined host runs in flight (pi_run_host_submit)

constexpr size_t ALIGN = 256;

size_t align_up(size_t v) { return (v + ALIGN - 1) & ~(ALIGN - 1); }

struct Layout {
  size_t ctl, counts, offsets, foffsets, pcounts, ptsum, dense, tiles, bcur, rec, sid, perm, urec, uid, tidx, outs, io, pairs;
  size_t xrec, xid, xperm, msg[8];  // nranks > 1 (two message sets)
  size_t total;
};

// Decomposition of cfg: local X layers and the fixed message capacity (nranks > 1).
struct SlabGeom {
  int Lx, nx_local, gx_off, own_lo, own_hi;
  long long ncells_local, cap_msg;
};

SlabGeom slab_geom(const pi_config *cfg) {
  SlabGeom s{};
  const int P = cfg->nranks;
  s.Lx = cfg->dims[0] / P;
  if (P > 1) {
    s.nx_local = s.Lx + 2;            // ghost layers at local 0 and Lx + 1
    s.gx_off = cfg->rank * s.Lx - 1;  // global X cell of local cell 0
    s.own_lo = 1;
    s.own_hi = s.Lx + 1;
    // a boundary X layer holds ~capacity / (Lx + 2) particles; 2.5x covers its fluctuation
    // and the migrants of one step (|dx| < w), with a floor for tiny slabs
    const long long cap = cfg->capacity > 0 ? cfg->capacity : 1;
    s.cap_msg = (long long)(2.5 * (double)cap / s.nx_local) + 1024;
  } else {
    s.nx_local = cfg->dims[0];
    s.gx_off = 0;
    s.own_lo = 0;
    s.own_hi = cfg->dims[0];
    s.cap_msg = 0;
  }
  s.ncells_local = (long long)s.nx_local * cfg->dims[1] * cfg->dims[2];
  return s;
}

int x_subcells(const pi_config *cfg) { return cfg->x_subcells > 0 ? cfg->x_subcells : 4; }

Layout make_layout(const pi_config *cfg) {
  const SlabGeom sg = slab_geom(cfg);
  const long long ncells = sg.ncells_local;
  const long long cap = cfg->capacity > 0 ? cfg->capacity : 1;
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes);
    return at;
  };
  const long long nf = ncells * x_subcells(cfg);  // fine (X sub-cell) bins
  L.ctl = take(sizeof(DevCtl));
  L.counts = take(sizeof(int32_t) * (size_t)(nf + 4));
  L.offsets = take(sizeof(int32_t) * (size_t)(ncells + 4));
  L.foffsets = take(sizeof(int32_t) * (size_t)(nf + 4));
  L.pcounts = take(sizeof(int32_t) * (size_t)(nf + 4));
  L.ptsum = take(sizeof(int32_t) * (size_t)(scan_tiles(nf) + 4));
  L.dense = take(sizeof(int32_t) * (size_t)(ncells + 4));
  L.tiles = take(sizeof(unsigned long long) * (size_t)scan_tiles(nf));
  L.bcur = take(sizeof(int32_t) * PART_NB);
  L.rec = take(sizeof(float4) * (size_t)cap);
  L.sid = take(sizeof(int32_t) * (size_t)cap);
  L.perm = take(sizeof(int32_t) * (size_t)cap);
  L.urec = take(sizeof(float4) * (size_t)cap);
  L.uid = take(sizeof(int32_t) * (size_t)cap);
  L.tidx = take(sizeof(int32_t) * (size_t)cap);
  L.outs = take(sizeof(float4) * (size_t)cap);
  L.io = take(sizeof(float) * 8 * RH_SETS * (size_t)cap);  // RH_SETS sets of x,y,z,q in + phi,F out (host paths)
  L.pairs = take(sizeof(float4) * 2 * (size_t)pair_plane_of(cap));  // two planes (A: x, y; B: z, q)
  if (cfg->nranks > 1) {
    L.xrec = take(sizeof(float4) * (size_t)cap);
    L.xid = take(sizeof(int32_t) * (size_t)cap);
    L.xperm = take(sizeof(int32_t) * (size_t)cap);
    for (int k = 0; k < 8; ++k) L.msg[k] = take(msg_bytes(sg.cap_msg));
  }
  L.total = o;
  return L;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---- small utility kernels (introspection / host path) ----
__global__ void k_unpack(long long n, const float4 *__restrict__ rec, const int32_t *__restrict__ ids,
                         const float4 *__restrict__ outs, float *x, float *y, float *z, float *q, int32_t *id,
                         float *phi, float *fx, float *fy, float *fz) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float4 r = rec[i];
    if (x) x[i] = r.x;
    if (y) y[i] = r.y;
    if (z) z[i] = r.z;
    if (q) q[i] = r.w;
    if (id) id[i] = ids[i];
    if (outs) {
      float4 o = outs[i];
      if (phi) phi[i] = o.x;
      if (fx) fx[i] = o.y;
      if (fy) fy[i] = o.z;
      if (fz) fz[i] = o.w;
    }
  }
}

__global__ void k_binning_export(long long n, const long long *n_dev, long long ncells, const float4 *__restrict__ rec,
                                 const int32_t *__restrict__ perm, const int32_t *__restrict__ offsets, Geom g,
                                 int32_t *cell_of, int32_t *counts, int32_t *offs_out, int32_t *perm_out) {
  if (n_dev) n = *n_dev;
  long long stride = (long long)gridDim.x * blockDim.x;
  long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = t0; i < n; i += stride) {
    const int pi_ = perm[i];
    if (cell_of && pi_ >= 0) {
      bool bad = false;
      float4 r = rec[i];
      cell_of[pi_] = cell_lin(g, r.x, r.y, r.z, bad);
    }
    if (perm_out) perm_out[i] = pi_;
  }
  for (long long c = t0; c <= ncells; c += stride) {
    if (offs_out) offs_out[c] = offsets[c];
    if (counts && c < ncells) counts[c] = offsets[c + 1] - offsets[c];
  }
}

int blocks_for(long long n, int t) {
  long long b = (n + t - 1) / t;
  if (b > 148LL * 8) b = 148LL * 8;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

struct pi_ctx_s {
  pi_config cfg;
  pi_tuning tune;
  Geom g;
  KParams kp;
  cudaStream_t stream;
  Layout lay;
  unsigned char *ws;
  DevCtl *ctl;
  int32_t *counts, *offsets, *foffsets, *pcounts, *ptsum, *dense, *sid, *perm, *uid, *tidx, *bcur;
  unsigned long long *tiles;
  float4 *rec, *urec, *outs, *pairs;
  float *io;
  long long n;       // owned particles (exact on the host when nranks == 1; pi_bin's n otherwise)
  int state;         // 0 empty, 1 binned from pi_bin, 2 sorted state from pi_step (update pending)
  bool need_bin;     // pi_step must re-bin (and, nranks > 1, migrate) first
  bool pairs_ready;  // c->pairs hold the sorted records as source pairs (written by the AoS scatter)
  bool pcounts_ok;   // pcounts = per-sub-cell counts of the current sorted state (one rank)
  bool rec_ok;       // rec holds the current sorted records (else only the pair array does)
  bool interacted;
  long long steps;
  SlabState slab;    // nranks > 1
  cudaEvent_t ev[4][2];  // phase timing: 0 bin, 1 interact, 2 exchange, 3 host copies
  bool ev_used[4];
  // pipelined host runs (pi_run_host_submit/_wait): copy streams and per-set events
  cudaStream_t h2d, d2h;
  cudaEvent_t ev_sub, ev_in[RH_SETS], ev_binned[RH_SETS], ev_out[RH_SETS], ev_done[RH_SETS];
  long long rh_issued, rh_done;
  // a8 overlapped step (nranks > 1): exchange stream and its events
  cudaStream_t xs;
  cudaEvent_t ev_bnd, ev_xdone;
  bool ovl_ready;    // the migrant and ghost messages of the pending re-binning have been exchanged
  long long ovl_steps;
  char err[512];
};

static void phase_begin(pi_ctx c, int k) {
  cudaEventRecord(c->ev[k][0], c->stream);
  c->ev_used[k] = true;
}
static void phase_end(pi_ctx c, int k) { cudaEventRecord(c->ev[k][1], c->stream); }

static pi_status fail(pi_ctx c, pi_status s, const char *fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof(c->err), fmt, ap);
    va_end(ap);
  }
  return s;
}

static pi_status cuda_check(pi_ctx c, cudaError_t e, const char *where) {
  if (e == cudaSuccess) return PI_OK;
  return fail(c, PI_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

static bool config_ok(const pi_config *cfg, char *why, size_t n) {
  if (!cfg) { snprintf(why, n, "cfg is NULL"); return false; }
  for (int a = 0; a < 3; ++a)
    if (cfg->dims[a] <= 0) { snprintf(why, n, "dims must be >= 1"); return false; }
  if (!(cfg->cell_width > 0.f)) { snprintf(why, n, "cell_width must be > 0"); return false; }
  if (!(cfg->r_c > 0.f)) { snprintf(why, n, "r_c must be > 0"); return false; }
  if (cfg->r_c > cfg->cell_width) { snprintf(why, n, "cell_width must be >= r_c (PAPER.md:93)"); return false; }
  if (cfg->kernel < 0 || cfg->kernel > 5) { snprintf(why, n, "unknown kernel"); return false; }
  if ((cfg->kernel == PI_K_LJ || cfg->kernel == PI_K_HIGHFLOP) && (cfg->kparam[0] < 0.f || cfg->kparam[1] < 0.f)) {
    snprintf(why, n, "Lennard-Jones r and eps must be >= 0");
    return false;
  }
  if (cfg->capacity < 0 || cfg->capacity > (1LL << 31) - 64) { snprintf(why, n, "capacity out of range"); return false; }
  if (cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks) { snprintf(why, n, "bad rank/nranks"); return false; }
  if (cfg->dims[0] % cfg->nranks) { snprintf(why, n, "dims[0] must be divisible by nranks"); return false; }
  if (cfg->x_subcells < 0 || cfg->x_subcells > 16 || (cfg->x_subcells & (cfg->x_subcells - 1))) {
    snprintf(why, n, "x_subcells must be 0 or a power of two <= 16");
    return false;
  }
  if (cfg->nranks > 1 && !cfg->nccl_unique_id) { snprintf(why, n, "nranks > 1 needs nccl_unique_id"); return false; }
  long long nc = (long long)cfg->dims[0] * cfg->dims[1] * cfg->dims[2];
  if (nc > (1LL << 30)) { snprintf(why, n, "too many cells"); return false; }
  // the fine (X sub-cell) index is 32-bit arithmetic in the kernels; with nranks > 1
  // the local grid has two extra X layers
  const long long lx = cfg->dims[0] / cfg->nranks + (cfg->nranks > 1 ? 2 : 0);
  if (lx * cfg->dims[1] * cfg->dims[2] * x_subcells(cfg) >= (1LL << 31) - 1) {
    snprintf(why, n, "cells x x_subcells must stay below 2^31");
    return false;
  }
  return true;
}

extern "C" {

int32_t pi_abi_version(void) { return PI_ABI_VERSION; }

size_t pi_workspace_bytes(const pi_config *cfg) {
  char why[256];
  if (!config_ok(cfg, why, sizeof(why))) return 0;
  return make_layout(cfg).total;
}

pi_status pi_slab_info(const pi_config *cfg, int64_t out[8]) {
  char why[256];
  if (!out || !config_ok(cfg, why, sizeof(why))) return PI_EINVAL;
  const SlabGeom s = slab_geom(cfg);
  out[0] = s.Lx;
  out[1] = (int64_t)cfg->rank * s.Lx;        // first owned global X cell
  out[2] = (int64_t)(cfg->rank + 1) * s.Lx;  // one past the last
  out[3] = s.nx_local;
  out[4] = s.gx_off;
  out[5] = s.own_lo;
  out[6] = s.own_hi;
  out[7] = s.cap_msg;
  return PI_OK;
}

pi_status pi_nccl_unique_id(void *out128) {
  char why[256];
  if (!out128) return PI_EINVAL;
  return nccl_unique_id(out128, why, sizeof(why)) ? PI_OK : PI_ENCCL;
}

pi_status pi_create(const pi_config *cfg, void *workspace, size_t ws_bytes, pi_ctx *out) {
  char why[256];
  if (!out) return PI_EINVAL;
  *out = nullptr;
  if (!config_ok(cfg, why, sizeof(why))) return PI_EINVAL;
  const SlabGeom sg = slab_geom(cfg);
  Layout lay = make_layout(cfg);
  if (!workspace || ws_bytes < lay.total || (reinterpret_cast<uintptr_t>(workspace) & (ALIGN - 1))) return PI_EINVAL;
  pi_ctx c = new (std::nothrow) pi_ctx_s();
  if (!c) return PI_EINVAL;
  c->cfg = *cfg;
  memset(&c->tune, 0, sizeof(c->tune));
  c->stream = reinterpret_cast<cudaStream_t>(cfg->stream);
  c->lay = lay;
  c->ws = reinterpret_cast<unsigned char *>(workspace);
  c->ctl = reinterpret_cast<DevCtl *>(c->ws + lay.ctl);
  c->counts = reinterpret_cast<int32_t *>(c->ws + lay.counts);
  c->offsets = reinterpret_cast<int32_t *>(c->ws + lay.offsets);
  c->foffsets = reinterpret_cast<int32_t *>(c->ws + lay.foffsets);
  c->pcounts = reinterpret_cast<int32_t *>(c->ws + lay.pcounts);
  c->ptsum = reinterpret_cast<int32_t *>(c->ws + lay.ptsum);
  c->dense = reinterpret_cast<int32_t *>(c->ws + lay.dense);
  c->tiles = reinterpret_cast<unsigned long long *>(c->ws + lay.tiles);
  c->rec = reinterpret_cast<float4 *>(c->ws + lay.rec);
  c->sid = reinterpret_cast<int32_t *>(c->ws + lay.sid);
  c->perm = reinterpret_cast<int32_t *>(c->ws + lay.perm);
  c->urec = reinterpret_cast<float4 *>(c->ws + lay.urec);
  c->uid = reinterpret_cast<int32_t *>(c->ws + lay.uid);
  c->tidx = reinterpret_cast<int32_t *>(c->ws + lay.tidx);
  c->bcur = reinterpret_cast<int32_t *>(c->ws + lay.bcur);
  c->outs = reinterpret_cast<float4 *>(c->ws + lay.outs);
  c->io = reinterpret_cast<float *>(c->ws + lay.io);
  c->pairs = reinterpret_cast<float4 *>(c->ws + lay.pairs);
  // geometry: the cell contract is evaluated on the GLOBAL grid, the local grid is the slab
  Geom &g = c->g;
  g.ox = cfg->origin[0]; g.oy = cfg->origin[1]; g.oz = cfg->origin[2];
  g.w = cfg->cell_width;
  g.inv_w = 1.0f / cfg->cell_width;  // contract C3: fl32(1/w), IEEE division on the host
  g.nx = sg.nx_local; g.ny = cfg->dims[1]; g.nz = cfg->dims[2];
  g.ncells = sg.ncells_local;
  g.gnx = cfg->dims[0];
  g.gx_off = sg.gx_off;
  g.own_lo = sg.own_lo;
  g.own_hi = sg.own_hi;
  g.sx = x_subcells(cfg);
  g.sxs = 0;
  while ((1 << g.sxs) < g.sx) ++g.sxs;
  g.lx = g.ox; g.ly = g.oy; g.lz = g.oz;
  g.hx = g.ox + (float)cfg->dims[0] * g.w;
  g.hy = g.oy + (float)g.ny * g.w;
  g.hz = g.oz + (float)g.nz * g.w;
  KParams &k = c->kp;
  k.kernel = cfg->kernel;
  k.rc = cfg->r_c;
  k.rc2 = cfg->r_c * cfg->r_c;
  float sigma = (cfg->kernel == PI_K_GAUSSIAN && cfg->kparam[0] > 0.f) ? cfg->kparam[0] : cfg->r_c / 3.0f;
  k.sigma = sigma;
  k.inv_s2 = (float)(1.0 / ((double)sigma * (double)sigma));
  k.c2 = (float)(1.4426950408889634 / (2.0 * (double)sigma * (double)sigma));
  k.s = (float)std::sqrt((double)k.c2);
  k.s_inv = (float)(1.0 / std::sqrt((double)k.c2));
  k.phi_scale = 1.0f;
  k.f_ts = k.inv_s2;
  if (cfg->kernel == PI_K_LJ || cfg->kernel == PI_K_HIGHFLOP) {  // Eq. (1), reading R19
    const double r = cfg->kparam[0] > 0.f ? cfg->kparam[0] : cfg->r_c;
    const double eps = cfg->kparam[1];
    const double e0 = cfg->kparam[2] > 0.f ? cfg->kparam[2] : 1.0;
    k.lj_inv_r2 = (float)(1.0 / (r * r));
    k.lj_e2 = (float)(eps * eps / (r * r));
    k.phi_scale = (float)(4.0 * e0);
    k.f_ts = (float)(-4.0 * e0 / (r * r));
  }
  // zero the control block, counts (the scan keeps them zero afterwards) and scan status
  cudaError_t e = cudaMemsetAsync(c->ws, 0, lay.rec, c->stream);
  // the X-pencil's dense-cell list: entries are -1 when free (cellsm.cuh)
  if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + lay.dense, 0xff, lay.tiles - lay.dense, c->stream);
  if (e != cudaSuccess) {
    pi_status s = cuda_check(c, e, "pi_create memset");
    delete c;
    return s;
  }
  for (int kk = 0; kk < 4; ++kk)
    for (int b = 0; b < 2; ++b) {
      e = cudaEventCreate(&c->ev[kk][b]);
      if (e != cudaSuccess) {
        pi_status s = cuda_check(c, e, "pi_create events");
        pi_destroy(c);
        return s;
      }
    }
  if (cfg->nranks > 1) {
    SlabState &S = c->slab;
    S.rank = cfg->rank;
    S.nranks = cfg->nranks;
    S.Lx = sg.Lx;
    S.cap_msg = sg.cap_msg;
    S.sendL = c->ws + lay.msg[0];
    S.sendR = c->ws + lay.msg[1];
    S.recvL = c->ws + lay.msg[2];
    S.recvR = c->ws + lay.msg[3];
    S.g = MsgSet{c->ws + lay.msg[4], c->ws + lay.msg[5], c->ws + lay.msg[6], c->ws + lay.msg[7]};
    S.xrec = reinterpret_cast<float4 *>(c->ws + lay.xrec);
    S.xid = reinterpret_cast<int32_t *>(c->ws + lay.xid);
    S.xperm = reinterpret_cast<int32_t *>(c->ws + lay.xperm);
    if ((e = cudaMemsetAsync(c->ws + lay.msg[0], 0, lay.total - lay.msg[0], c->stream)) != cudaSuccess) {
      pi_status s = cuda_check(c, e, "pi_create memset msgs");
      pi_destroy(c);
      return s;
    }
    S.tr = make_transport(cfg, &S, c->err, sizeof(c->err));
    if (!S.tr) {
      pi_destroy(c);
      return PI_ENCCL;
    }
    // pinned host slot for the exchanged counts (the two-phase exchange reads them back)
    if ((e = cudaHostAlloc(reinterpret_cast<void **>(&S.hcnt), 4 * sizeof(long long), cudaHostAllocDefault)) !=
        cudaSuccess) {
      pi_status s = cuda_check(c, e, "pi_create pinned counts");
      pi_destroy(c);
      return s;
    }
  }
  *out = c;
  return PI_OK;
}

pi_status pi_destroy(pi_ctx c) {
  if (c) {
    for (int k = 0; k < 4; ++k)
      for (int b = 0; b < 2; ++b)
        if (c->ev[k][b]) cudaEventDestroy(c->ev[k][b]);
    if (c->h2d) {
      cudaEventDestroy(c->ev_sub);
      for (int b = 0; b < RH_SETS; ++b) {
        cudaEventDestroy(c->ev_in[b]);
        cudaEventDestroy(c->ev_binned[b]);
        cudaEventDestroy(c->ev_out[b]);
        cudaEventDestroy(c->ev_done[b]);
      }
      cudaStreamDestroy(c->h2d);
      cudaStreamDestroy(c->d2h);
    }
    if (c->xs) {
      cudaEventDestroy(c->ev_bnd);
      cudaEventDestroy(c->ev_xdone);
      cudaStreamDestroy(c->xs);
    }
    delete c->slab.tr;
    if (c->slab.hcnt) cudaFreeHost(c->slab.hcnt);
  }
  delete c;
  return PI_OK;
}

pi_status pi_set_stream(pi_ctx c, void *stream) {
  if (!c) return PI_EINVAL;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  return PI_OK;
}

pi_status pi_set_tuning(pi_ctx c, const pi_tuning *t) {
  if (!c || !t) return PI_EINVAL;
  c->tune = *t;
  c->slab.counted = t->exchange_full == 0;
  return PI_OK;
}

// a1-a4 on SoA input (x != NULL) or on AoS records.
static pi_status do_bin(pi_ctx c, long long n, const float *x, const float *y, const float *z, const float *q,
                        const int32_t *id, const float4 *rec_in, const int32_t *perm_in, const long long *n_dev,
                        bool delta = false, bool pairs_only = false) {
  BinArgs a{};
  const bool one = c->cfg.nranks == 1;
  a.delta = delta;
  // the SoA path's scan records the persistent counts; the delta path re-bins from them
  a.pcounts = one && (delta || !rec_in) ? c->pcounts : nullptr;
  c->pcounts_ok = one && (delta || !rec_in);
  a.ptsum = c->ptsum;
  a.n = n;
  a.n_dev = n_dev;
  a.x = x; a.y = y; a.z = z; a.q = q;
  a.rec_in = rec_in;
  a.id_in = id;
  a.tmp_rec = c->urec;  // free during pi_bin (pi_step's update buffer)
  a.tmp_idx = c->tidx;
  a.bucket_cur = c->bcur;
  a.counts = c->counts;
  a.offsets = c->offsets;
  a.foffsets = c->foffsets;
  a.tile_status = c->tiles;
  a.rec_out = (pairs_only && rec_in) ? nullptr : c->rec;  // pi_step + X-pencil: pairs only
  c->rec_ok = a.rec_out != nullptr;
  a.sid_out = c->sid;
  a.perm_out = (rec_in && !perm_in) ? nullptr : c->perm;
  a.perm_in = perm_in;
  // the f32x2 source-pair array is read only by the X-pencil's pencil-by-pencil layout (the
  // default; the interleaved layout, xpencil_layout = 1, stages records)
  a.pairs_out = (rec_in && c->tune.xpencil_layout != 1) ? c->pairs : nullptr;
  a.pair_plane = pair_plane_of(c->cfg.capacity);
  c->pairs_ready = a.pairs_out != nullptr;
  a.ctl = c->ctl;
  phase_begin(c, 0);
  cudaError_t e = launch_bin(c->g, a, c->stream);
  phase_end(c, 0);
  return cuda_check(c, e, "pi_bin");
}

// a8: exchange the first / last owned X layers as ghosts, append them, bin owned + ghosts.
static pi_status slab_ghosts_and_bin(pi_ctx c) {
  SlabState &S = c->slab;
  const long long cap = c->cfg.capacity;
  cudaError_t e;
  phase_begin(c, 2);
  if ((e = slab_reset(S, c->ctl, c->stream)) != cudaSuccess) return cuda_check(c, e, "slab reset");
  if ((e = slab_select_ghosts(S, c->g, cap, c->ctl, c->stream)) != cudaSuccess) return cuda_check(c, e, "ghosts");
  if ((e = slab_exchange(S, c->stream)) != cudaSuccess) return fail(c, PI_ENCCL, "ghost exchange failed");
  if ((e = slab_append(S, &c->ctl->n_owned, &c->ctl->n_total, &c->ctl->ghosts_in, &c->ctl->pad2[1], cap, c->ctl,
                       c->stream)) !=
      cudaSuccess)
    return cuda_check(c, e, "ghost append");
  phase_end(c, 2);
  return do_bin(c, cap, nullptr, nullptr, nullptr, nullptr, S.xid, S.xrec, S.xperm, &c->ctl->n_total);
}

pi_status pi_bin(pi_ctx c, int64_t n, const float *x, const float *y, const float *z, const float *q,
                 const int32_t *id) {
  if (!c) return PI_EINVAL;
  if (n < 0) return fail(c, PI_EINVAL, "n < 0");
  if (n > c->cfg.capacity) return fail(c, PI_ECAPACITY, "n = %lld exceeds capacity %lld", (long long)n,
                                       (long long)c->cfg.capacity);
  if (n > 0 && (!x || !y || !z || !q)) return fail(c, PI_EINVAL, "NULL position/value pointer");
  if (n > 0 && (!aligned16(x) || !aligned16(y) || !aligned16(z) || !aligned16(q)))
    return fail(c, PI_EINVAL, "x, y, z, q must be 16-byte aligned");
  pi_status s;
  if (c->cfg.nranks > 1) {
    cudaError_t e = slab_from_soa(c->slab, c->g, n, x, y, z, q, id, c->ctl, c->stream);
    if (e != cudaSuccess) return cuda_check(c, e, "pi_bin slab input");
    s = slab_ghosts_and_bin(c);
  } else {
    s = do_bin(c, n, x, y, z, q, id, nullptr, nullptr, nullptr);
  }
  if (s != PI_OK) return s;
  c->n = n;
  c->state = 1;
  c->need_bin = false;
  c->ovl_ready = false;
  c->interacted = false;
  return PI_OK;
}

// PI_A_AUTO: the global-memory kernel below ~3 particles per cell (the paper's crossover: the
// staged kernels pay per-cell overheads with few particles per cell; measured configs[2] ppc 1
// and 2: 1.5 / 1.9 ms against the X-pencil's 3.8 / 2.2), the X-pencil above
static pi_algo resolve_auto(pi_ctx c, pi_algo algo) {
  if (algo != PI_A_AUTO) return algo;
  const double ppc = (double)c->n / (double)(c->g.ncells > 0 ? c->g.ncells : 1);
  return ppc < 3.0 ? PI_A_GLOBAL : PI_A_XPENCIL;
}

// xr (X-pencil only): the target X layers [xr0, xr1) + [xr2, xr3) of this launch (NULL: all
// owned); part: 0 the whole interaction, 1 / 2 its first / second launch (statistics reset by
// the first, phase timing over both), reserve: SMs left to kernels running beside it
static pi_status do_interact(pi_ctx c, pi_algo algo, float *phi, float *fx, float *fy, float *fz, bool integrate,
                             float dt, const int *xr = nullptr, int part = 0, int reserve = 0) {
  algo = resolve_auto(c, algo);
  InteractArgs a{};
  const bool multi = c->cfg.nranks > 1;
  a.n = multi ? c->cfg.capacity : c->n;
  a.n_dev = multi ? &c->ctl->n_total : nullptr;
  a.n_est = multi ? c->n * (long long)(c->slab.Lx + 2) / (c->slab.Lx > 0 ? c->slab.Lx : 1) : c->n;
  const bool r01_layout = (algo == PI_A_XPENCIL || algo == PI_A_AUTO) && c->tune.xpencil_layout != 1;
  if (!c->rec_ok && !r01_layout)
    return fail(c, PI_ESTATE, "internal: sorted records not materialised for this strategy");
  a.rec = c->rec_ok ? c->rec : nullptr;
  a.foffsets = c->foffsets;
  a.pairs = c->pairs;
  a.pair_plane = pair_plane_of(c->cfg.capacity);
  a.pairs_ready = c->pairs_ready;
  a.offsets = c->offsets;
  a.ctl = c->ctl;
  a.out.sorted = c->outs;
  a.out.perm = (phi || fx || fy || fz) ? c->perm : nullptr;
  a.out.phi = phi; a.out.fx = fx; a.out.fy = fy; a.out.fz = fz;
  a.out.upd = integrate ? c->urec : nullptr;
  a.out.sid = c->sid;
  a.out.uid = c->uid;
  a.out.dt = dt;
  a.out.flags = &c->ctl->flags;
  if (integrate && c->pcounts_ok) {  // movers update the persistent counts and their tile sums
    a.out.pcounts = c->pcounts;
    a.out.ptsum = c->ptsum;
  }
  a.tx_len = c->tune.xpencil_len;
  a.tx_cap = c->tune.xpencil_cap;
  a.threads = c->tune.threads;
  a.slots = c->tune.xpencil_slots;
  a.tpl = c->tune.xpencil_targets;
  a.dense = c->dense;
  a.fb[0] = c->tune.fullload_box[0]; a.fb[1] = c->tune.fullload_box[1]; a.fb[2] = c->tune.fullload_box[2];
  a.fb_cap = c->tune.fullload_cap;
  if (xr) {
    a.xr_set = true;
    for (int k = 0; k < 4; ++k) a.xr[k] = xr[k];
  }
  a.reserve_sms = reserve;
  cudaError_t e = part == 2
                      // the second launch: a fresh item counter and dense-cell tickets (the first
                      // launch's listed cells are all computed: every entry is free again)
                      ? cudaMemsetAsync(&c->ctl->xp_items, 0, sizeof(unsigned long long) * 5, c->stream)
                      : cudaMemsetAsync(&c->ctl->fallback_cells, 0,
                                        sizeof(DevCtl) - offsetof(DevCtl, fallback_cells), c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "pi_interact memset");
  if (algo == PI_A_AUTO) algo = PI_A_XPENCIL;
  if (part != 2) phase_begin(c, 1);
  switch (algo) {
    case PI_A_GLOBAL: e = launch_interact_global(c->g, c->kp, a, c->stream); break;
    case PI_A_XPENCIL:
      e = c->tune.xpencil_layout == 1 ? launch_interact_xpencil2(c->g, c->kp, a, c->stream)
                                      : launch_interact_xpencil(c->g, c->kp, a, c->stream);
      break;
    case PI_A_FULLLOAD: e = launch_interact_fullload(c->g, c->kp, a, c->stream); break;
    case PI_A_XPREG: e = launch_interact_xpreg(c->g, c->kp, a, c->stream); break;
    case PI_A_HALF: e = launch_interact_half(c->g, c->kp, a, c->stream); break;
    default: return fail(c, PI_EINVAL, "unknown algo %d", (int)algo);
  }
  if (part != 1) phase_end(c, 1);
  if (e == cudaErrorNotSupported) return fail(c, PI_EINAPPLICABLE, "strategy not applicable to this grid");
  return cuda_check(c, e, "pi_interact");
}

pi_status pi_interact(pi_ctx c, pi_algo algo, float *phi, float *fx, float *fy, float *fz) {
  if (!c) return PI_EINVAL;
  if (c->state == 0) return fail(c, PI_ESTATE, "pi_interact before pi_bin");
  bool caller = phi || fx || fy || fz;
  if (c->state != 1 && caller) return fail(c, PI_ESTATE, "caller-order outputs need a pi_bin binning");
  if (c->need_bin) return fail(c, PI_ESTATE, "sorted state is stale after pi_step (call pi_step or pi_bin)");
  pi_status s = do_interact(c, algo, phi, fx, fy, fz, false, 0.f);
  if (s == PI_OK) c->interacted = true;
  return s;
}

// a8 with the exchange overlapped: the X-pencil first computes (and updates)
// the first and last 2 owned X layers -- every particle that can leave the slab or end up in a
// boundary layer (a ghost of the next step) is there, |dt F| < w (reading C11) -- then the
// interior layers, while a second stream sorts the boundary particles into migrant and ghost
// messages, exchanges the migrants, adds the arrivals to the ghosts and exchanges those.  The
// next pi_step only compacts the stayers and appends what arrived.
static bool overlap_ok(pi_ctx c, pi_algo algo) {
  return c->cfg.nranks > 1 && algo == PI_A_XPENCIL && c->tune.xpencil_layout != 1 && c->tune.exchange_overlap == 0 &&
         c->slab.Lx >= 4;
}

static pi_status step_overlapped(pi_ctx c, float dt) {
  SlabState &S = c->slab;
  const long long cap = c->cfg.capacity;
  cudaError_t e = cudaSuccess;
  if (!c->xs) {
    e = cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_bnd, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_xdone, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_check(c, e, "exchange stream");
  }
  const int lo = c->g.own_lo, hi = c->g.own_hi;
  const int bnd[4] = {lo, lo + 2, hi - 2, hi}, mid[4] = {lo + 2, hi - 2, 0, 0};
  const bool interior = hi - 2 > lo + 2;
  pi_status st = do_interact(c, PI_A_XPENCIL, nullptr, nullptr, nullptr, nullptr, true, dt, bnd, interior ? 1 : 0);
  if (st != PI_OK) return st;
  if ((e = cudaEventRecord(c->ev_bnd, c->stream)) != cudaSuccess) return cuda_check(c, e, "event");
  if ((e = cudaStreamWaitEvent(c->xs, c->ev_bnd, 0)) != cudaSuccess) return cuda_check(c, e, "event wait");
  cudaEventRecord(c->ev[2][0], c->xs);
  c->ev_used[2] = true;
  if ((e = slab_reset(S, c->ctl, c->xs, 0, false)) != cudaSuccess) return cuda_check(c, e, "slab reset");
  if ((e = slab_reset(S, c->ctl, c->xs, 1, false)) != cudaSuccess) return cuda_check(c, e, "slab reset");
  if ((e = slab_migrate_boundary(S, c->g, cap, c->rec, c->urec, c->uid, c->ctl, c->xs)) != cudaSuccess)
    return cuda_check(c, e, "boundary migrate");
  // the interior launch is queued before the exchange blocks this thread on the host; two SMs
  // stay free for the transport's and the exchange kernels
  if (interior) {
    st = do_interact(c, PI_A_XPENCIL, nullptr, nullptr, nullptr, nullptr, true, dt, mid, 2, 2);
    if (st != PI_OK) return st;
  }
  if ((e = slab_exchange(S, c->xs, 0)) != cudaSuccess) return fail(c, PI_ENCCL, "migration exchange failed");
  if ((e = slab_ghost_arrivals(S, c->g, c->ctl, c->xs)) != cudaSuccess) return cuda_check(c, e, "ghost arrivals");
  if ((e = slab_exchange(S, c->xs, 1)) != cudaSuccess) return fail(c, PI_ENCCL, "ghost exchange failed");
  cudaEventRecord(c->ev[2][1], c->xs);
  if ((e = cudaEventRecord(c->ev_xdone, c->xs)) != cudaSuccess) return cuda_check(c, e, "event");
  if ((e = cudaStreamWaitEvent(c->stream, c->ev_xdone, 0)) != cudaSuccess) return cuda_check(c, e, "event wait");
  c->ovl_ready = true;
  c->ovl_steps++;
  return PI_OK;
}

pi_status pi_step(pi_ctx c, pi_algo algo, float dt) {
  if (!c) return PI_EINVAL;
  algo = resolve_auto(c, algo);
  if (c->state == 0) return fail(c, PI_ESTATE, "pi_step before pi_bin");
  if (!std::isfinite(dt)) return fail(c, PI_EINVAL, "dt must be finite");
  if (c->need_bin && c->ovl_ready) {
    // the previous (overlapped) step exchanged the migrants and ghosts already: compact the
    // stayers, append the arrivals (set 0) and the ghosts (set 1), bin
    SlabState &S = c->slab;
    const long long cap = c->cfg.capacity;
    cudaError_t e = cudaMemsetAsync(&c->ctl->n_stay, 0, sizeof(long long), c->stream);
    if (e == cudaSuccess) e = slab_migrate(S, c->g, cap, c->rec, c->urec, c->uid, c->ctl, c->stream, false);
    if (e == cudaSuccess)
      e = slab_append(S, &c->ctl->n_stay, &c->ctl->n_owned, &c->ctl->migrants_in, &c->ctl->migrants_out, cap, c->ctl,
                      c->stream, 0);
    if (e == cudaSuccess)
      e = slab_append(S, &c->ctl->n_owned, &c->ctl->n_total, &c->ctl->ghosts_in, &c->ctl->pad2[1], cap, c->ctl,
                      c->stream, 1);
    if (e != cudaSuccess) return cuda_check(c, e, "overlapped re-binning");
    c->ovl_ready = false;
    pi_status s = do_bin(c, cap, nullptr, nullptr, nullptr, nullptr, S.xid, S.xrec, S.xperm, &c->ctl->n_total);
    if (s != PI_OK) return s;
  } else if (c->need_bin) {
    pi_status s;
    if (c->cfg.nranks > 1) {
      // a8: migration of the particles whose updated cell left the slab, then ghosts + bin
      SlabState &S = c->slab;
      const long long cap = c->cfg.capacity;
      cudaError_t e;
      phase_begin(c, 2);
      if ((e = slab_reset(S, c->ctl, c->stream)) != cudaSuccess) return cuda_check(c, e, "slab reset");
      if ((e = slab_migrate(S, c->g, cap, c->rec, c->urec, c->uid, c->ctl, c->stream)) != cudaSuccess)
        return cuda_check(c, e, "migrate");
      if ((e = slab_exchange(S, c->stream)) != cudaSuccess) return fail(c, PI_ENCCL, "migration exchange failed");
      if ((e = slab_append(S, &c->ctl->n_stay, &c->ctl->n_owned, &c->ctl->migrants_in, &c->ctl->migrants_out, cap,
                           c->ctl, c->stream)) !=
          cudaSuccess)
        return cuda_check(c, e, "migrant append");
      phase_end(c, 2);
      s = slab_ghosts_and_bin(c);
    } else {
      // the X-pencil reads only the pair array: the records need not be written (16 B/particle)
      s = do_bin(c, c->n, nullptr, nullptr, nullptr, nullptr, c->uid, c->urec, nullptr, nullptr, c->pcounts_ok,
                 (algo == PI_A_XPENCIL || algo == PI_A_AUTO) && c->tune.xpencil_layout != 1);
    }
    if (s != PI_OK) return s;
  }
  pi_status s = overlap_ok(c, algo) ? step_overlapped(c, dt)
                                     : do_interact(c, algo, nullptr, nullptr, nullptr, nullptr, true, dt);
  if (s != PI_OK) return s;
  c->state = 2;
  c->need_bin = true;
  c->interacted = true;
  c->steps++;
  return PI_OK;
}

static pi_status rh_wait_all(pi_ctx c);

pi_status pi_run_host(pi_ctx c, pi_algo algo, int64_t n, const float *x, const float *y, const float *z,
                      const float *q, float *phi, float *fx, float *fy, float *fz) {
  if (!c) return PI_EINVAL;
  if (n < 0 || n > c->cfg.capacity) return fail(c, PI_ECAPACITY, "n out of range");
  {  // it uses I/O set 0, which pipelined runs in flight may still read or write
    pi_status s = rh_wait_all(c);
    if (s != PI_OK) return s;
  }
  if (n > 0 && (!x || !y || !z || !q)) return fail(c, PI_EINVAL, "NULL host input");
  size_t cap = (size_t)c->cfg.capacity;
  float *dx = c->io, *dy = c->io + cap, *dz = c->io + 2 * cap, *dq = c->io + 3 * cap;
  float *dphi = c->io + 4 * cap, *dfx = c->io + 5 * cap, *dfy = c->io + 6 * cap, *dfz = c->io + 7 * cap;
  size_t bytes = sizeof(float) * (size_t)n;
  cudaError_t e;
  const float *src[4] = {x, y, z, q};
  float *dst[4] = {dx, dy, dz, dq};
  phase_begin(c, 3);
  for (int k = 0; k < 4; ++k)
    if (n > 0 && (e = cudaMemcpyAsync(dst[k], src[k], bytes, cudaMemcpyHostToDevice, c->stream)) != cudaSuccess)
      return cuda_check(c, e, "pi_run_host H2D");
  pi_status s = pi_bin(c, n, dx, dy, dz, dq, nullptr);
  if (s != PI_OK) return s;
  s = pi_interact(c, algo, phi ? dphi : nullptr, fx ? dfx : nullptr, fy ? dfy : nullptr, fz ? dfz : nullptr);
  if (s != PI_OK) return s;
  float *hout[4] = {phi, fx, fy, fz};
  float *dout[4] = {dphi, dfx, dfy, dfz};
  for (int k = 0; k < 4; ++k)
    if (n > 0 && hout[k] &&
        (e = cudaMemcpyAsync(hout[k], dout[k], bytes, cudaMemcpyDeviceToHost, c->stream)) != cudaSuccess)
      return cuda_check(c, e, "pi_run_host D2H");
  phase_end(c, 3);
  return cuda_check(c, cudaStreamSynchronize(c->stream), "pi_run_host sync");
}

// Pipelined host runs: run k uses I/O set k % RH_SETS of the workspace.  H2D on its own stream,
// bin + interact on the context stream, D2H on a third stream, ordered by events, so the
// copies of run k+1 (host -> device) and run k-1 (device -> host) overlap run k's kernels.
static pi_status rh_wait_one(pi_ctx c) {
  if (c->rh_done >= c->rh_issued) return PI_OK;
  const int k = (int)(c->rh_done % RH_SETS);
  cudaError_t e = cudaEventSynchronize(c->ev_done[k]);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, c->ev_done[k], 0);
  ++c->rh_done;
  return cuda_check(c, e, "pi_run_host_wait");
}

static pi_status rh_wait_all(pi_ctx c) {
  while (c->rh_done < c->rh_issued) {
    pi_status s = rh_wait_one(c);
    if (s != PI_OK) return s;
  }
  return PI_OK;
}

pi_status pi_run_host_submit(pi_ctx c, pi_algo algo, int64_t n, const float *x, const float *y, const float *z,
                             const float *q, float *phi, float *fx, float *fy, float *fz) {
  if (!c) return PI_EINVAL;
  if (c->cfg.nranks > 1) return fail(c, PI_EINVAL, "pi_run_host_submit: one rank only (use pi_run_host)");
  if (n < 0 || n > c->cfg.capacity) return fail(c, PI_ECAPACITY, "n out of range");
  if (n > 0 && (!x || !y || !z || !q)) return fail(c, PI_EINVAL, "NULL host input");
  cudaError_t e = cudaSuccess;
  if (!c->h2d) {  // first use: the copy streams and events
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_sub, cudaEventDisableTiming);
    for (int b = 0; b < RH_SETS && e == cudaSuccess; ++b) {
      e = cudaEventCreateWithFlags(&c->ev_in[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_binned[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_out[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done[b], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_check(c, e, "pi_run_host_submit: streams/events");
  }
  if (c->rh_issued - c->rh_done >= RH_SETS) {  // every I/O set in flight: wait for the oldest run
    pi_status s = rh_wait_one(c);
    if (s != PI_OK) return s;
  }
  const long long run = c->rh_issued;
  const int k = (int)(run % RH_SETS);
  const size_t cap = (size_t)c->cfg.capacity;
  float *in = c->io + (size_t)k * 8 * cap, *out = in + 4 * cap;
  const size_t bytes = sizeof(float) * (size_t)n;
  const float *src[4] = {x, y, z, q};
  float *hout[4] = {phi, fx, fy, fz};
  // host -> device once run-2's binning has consumed this input set; with no run in flight,
  // also after the work already on the context stream (the caller's timing events, say).
  // (Waiting on the context stream while a run is in flight would order this upload after
  // that run's kernels and serialise the pipeline.)
  if (c->rh_issued == c->rh_done) {
    e = cudaEventRecord(c->ev_sub, c->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->h2d, c->ev_sub, 0);
  }
  if (e == cudaSuccess && run >= RH_SETS) e = cudaStreamWaitEvent(c->h2d, c->ev_binned[k], 0);
  for (int a = 0; a < 4 && e == cudaSuccess && n > 0; ++a)
    e = cudaMemcpyAsync(in + a * cap, src[a], bytes, cudaMemcpyHostToDevice, c->h2d);
  if (e == cudaSuccess) e = cudaEventRecord(c->ev_in[k], c->h2d);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, c->ev_in[k], 0);
  if (e != cudaSuccess) return cuda_check(c, e, "pi_run_host_submit H2D");
  pi_status s = pi_bin(c, n, in, in + cap, in + 2 * cap, in + 3 * cap, nullptr);
  if (s != PI_OK) return s;
  e = cudaEventRecord(c->ev_binned[k], c->stream);
  // the output set is free once run-2's results reached the host
  if (e == cudaSuccess && run >= RH_SETS) e = cudaStreamWaitEvent(c->stream, c->ev_done[k], 0);
  if (e != cudaSuccess) return cuda_check(c, e, "pi_run_host_submit");
  s = pi_interact(c, algo, phi ? out : nullptr, fx ? out + cap : nullptr, fy ? out + 2 * cap : nullptr,
                  fz ? out + 3 * cap : nullptr);
  if (s != PI_OK) return s;
  e = cudaEventRecord(c->ev_out[k], c->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->d2h, c->ev_out[k], 0);
  for (int a = 0; a < 4 && e == cudaSuccess && n > 0; ++a)
    if (hout[a]) e = cudaMemcpyAsync(hout[a], out + a * cap, bytes, cudaMemcpyDeviceToHost, c->d2h);
  if (e == cudaSuccess) e = cudaEventRecord(c->ev_done[k], c->d2h);
  if (e != cudaSuccess) return cuda_check(c, e, "pi_run_host_submit D2H");
  ++c->rh_issued;
  return PI_OK;
}

pi_status pi_run_host_wait(pi_ctx c) {
  if (!c) return PI_EINVAL;
  while (c->rh_done < c->rh_issued) {
    pi_status s = rh_wait_one(c);
    if (s != PI_OK) return s;
  }
  return PI_OK;
}

pi_status pi_get_binning(pi_ctx c, int32_t *cell_of, int32_t *counts, int32_t *offsets, int32_t *perm) {
  if (!c) return PI_EINVAL;
  if (c->state == 0) return fail(c, PI_ESTATE, "no binning yet");
  if (c->need_bin && (cell_of || perm)) return fail(c, PI_ESTATE, "binning superseded by pi_step");
  if (c->state != 1 && (cell_of || perm)) return fail(c, PI_ESTATE, "cell_of/perm refer to a pi_bin input");
  const bool multi = c->cfg.nranks > 1;
  long long n = multi ? c->cfg.capacity : c->n;
  long long work = n > c->g.ncells + 1 ? n : c->g.ncells + 1;
  k_binning_export<<<blocks_for(work, 256), 256, 0, c->stream>>>(n, multi ? &c->ctl->n_total : nullptr,
                                                                 c->g.ncells, c->rec, c->perm, c->offsets, c->g,
                                                                 cell_of, counts, offsets, perm);
  return cuda_check(c, cudaGetLastError(), "pi_get_binning");
}

pi_status pi_get_particles(pi_ctx c, float *x, float *y, float *z, float *q, int32_t *id, float *phi, float *fx,
                           float *fy, float *fz) {
  if (!c) return PI_EINVAL;
  if (c->state == 0) return fail(c, PI_ESTATE, "no particles yet");
  const float4 *rec = c->need_bin ? c->urec : c->rec;
  const int32_t *ids = c->need_bin ? c->uid : c->sid;
  if (c->cfg.nranks > 1) {
    // owned particles only (ghost slots are skipped), in an arbitrary order; count in pi_stats
    cudaError_t e = slab_export_owned(c->g, c->cfg.capacity, c->rec, rec, ids, c->interacted ? c->outs : nullptr,
                                      x, y, z, q, id, phi, fx, fy, fz, c->ctl, c->stream);
    return cuda_check(c, e, "pi_get_particles");
  }
  if (c->n > 0)
    k_unpack<<<blocks_for(c->n, 256), 256, 0, c->stream>>>(c->n, rec, ids, c->interacted ? c->outs : nullptr, x, y,
                                                           z, q, id, phi, fx, fy, fz);
  return cuda_check(c, cudaGetLastError(), "pi_get_particles");
}

pi_status pi_get_stats(pi_ctx c, pi_stats *out) {
  if (!c || !out) return PI_EINVAL;
  DevCtl h;
  cudaError_t e = cudaMemcpyAsync(&h, c->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "pi_get_stats");
  memset(out, 0, sizeof(*out));
  if (c->cfg.nranks > 1) {
    out->n_owned = h.n_owned;
    out->n_ghost = h.n_total - h.n_owned;
    out->migrants_in = h.migrants_in;
    out->migrants_out = h.migrants_out;
  } else {
    out->n_owned = c->n;
    out->n_ghost = 0;
  }
  out->max_per_cell = h.max_per_cell;
  out->flags = h.flags;
  unsigned long long cand = 0;
  for (int k = 0; k < CAND_SLOTS; ++k) cand += h.cand_slots[k];
  out->candidates = (int64_t)cand;
  out->fallback_cells = (int64_t)h.fallback_cells;
  out->steps = c->steps;
  out->overlapped_steps = c->ovl_steps;
  out->exchange_bytes = c->slab.bytes_sent;
  for (int k = 0; k < 4; ++k) {
    float ms = 0.f;
    if (c->ev_used[k] && cudaEventElapsedTime(&ms, c->ev[k][0], c->ev[k][1]) == cudaSuccess) out->phase_ms[k] = ms;
  }
  if (h.flags) return fail(c, PI_EDEVICE, "device error flags 0x%x", h.flags);
  return PI_OK;
}

pi_status pi_count_pairs(pi_ctx c, int64_t *pairs) {
  if (!c || !pairs) return PI_EINVAL;
  if (c->state == 0) return fail(c, PI_ESTATE, "pi_count_pairs before pi_bin");
  if (!c->rec_ok && !c->pairs_ready) return fail(c, PI_ESTATE, "pi_count_pairs: no sorted state");
  const bool multi = c->cfg.nranks > 1;
  InteractArgs a{};
  a.n = multi ? c->cfg.capacity : c->n;
  a.n_dev = multi ? &c->ctl->n_total : nullptr;
  a.rec = c->rec_ok ? c->rec : nullptr;
  a.pairs = c->pairs;
  a.pair_plane = pair_plane_of(c->cfg.capacity);
  a.offsets = c->offsets;
  a.ctl = c->ctl;
  cudaError_t e = launch_count_pairs(c->g, c->kp, a, c->stream);
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, &c->ctl->pairs, sizeof(h), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "pi_count_pairs");
  *pairs = (int64_t)h;
  return PI_OK;
}

const char *pi_last_error(pi_ctx c) { return c ? c->err : "NULL context"; }

}  // extern "C"
