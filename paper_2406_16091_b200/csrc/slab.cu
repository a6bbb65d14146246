// X-slab kernels and transports (see slab.cuh).
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <algorithm>

#include "slab.cuh"

namespace pi {
namespace {

constexpr int T = 256;

int blocks_for(long long n) {
  long long b = (n + T - 1) / T;
  if (b > 148LL * 8) b = 148LL * 8;
  return b < 1 ? 1 : (int)b;
}

// Warp-aggregated append: every lane with `want` gets a distinct slot of *counter.
__device__ __forceinline__ long long agg_append(bool want, long long *counter) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  long long base = 0;
  const int lane = threadIdx.x & 31;
  const int leader = m ? __ffs(m) - 1 : 0;
  if (m && lane == leader)
    base = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(counter), (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + __popc(m & lanemask_lt());
}

__device__ __forceinline__ void msg_put(void *msg, long long cap, long long idx, float4 r, int32_t id) {
  if (idx < cap) {
    msg_rec(msg)[idx] = r;
    msg_id(msg, cap)[idx] = id;
  }
}

__global__ void k_reset(void *sL, void *sR, void *rL, void *rR, DevCtl *ctl, bool stay) {
  if (threadIdx.x == 0) {
    if (sL) reinterpret_cast<MsgHeader *>(sL)->count = 0;
    if (sR) reinterpret_cast<MsgHeader *>(sR)->count = 0;
    if (rL) reinterpret_cast<MsgHeader *>(rL)->count = 0;
    if (rR) reinterpret_cast<MsgHeader *>(rR)->count = 0;
    if (stay) ctl->n_stay = 0;
  }
}

// pi_bin input -> xrec; a particle whose global X cell is outside this rank's slab raises
// FLAG_DOMAIN (it would otherwise land in a ghost layer and silently drop out).
__global__ void k_soa_to_x(Geom g, int lo, int hi, long long n, const float *__restrict__ x,
                           const float *__restrict__ y, const float *__restrict__ z, const float *__restrict__ q,
                           const int32_t *__restrict__ id, float4 *xrec, int32_t *xid, int32_t *xperm, DevCtl *ctl) {
  bool bad = false, out = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float px = __ldg(x + i);
    const int cg = cell_coord(px, g.ox, g.inv_w, g.gnx, bad);
    out |= cg < lo || cg >= hi;
    xrec[i] = make_float4(px, __ldg(y + i), __ldg(z + i), __ldg(q + i));
    xid[i] = id ? __ldg(id + i) : (int32_t)i;
    xperm[i] = (int32_t)i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->n_owned = n;
    ctl->n_total = n;
  }
  if (out) atomicOr(&ctl->flags, FLAG_DOMAIN);
}

// Owned sorted slots -> stayers (xrec) or migrants (sendL / sendR) by their NEW global cell.
__global__ void k_migrate(Geom g, long long cap, int rank, int nranks, int Lx, const float4 *__restrict__ rec,
                          const float4 *__restrict__ upd, const int32_t *__restrict__ uid, float4 *xrec,
                          int32_t *xid, int32_t *xperm, void *sL, void *sR, long long cap_msg, DevCtl *ctl,
                          bool send) {
  const long long n = ctl->n_total;
  const int lo = rank * Lx, hi = (rank + 1) * Lx;
  bool bad = false;
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < n; t0 += (long long)gridDim.x * blockDim.x) {
    const long long t = t0 + threadIdx.x;
    bool owned = false;
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    int cls = -1;  // 0 stay, 1 left, 2 right
    int32_t id = 0;
    if (t < n) {
      const int cx = cell_x(g, rec[t].x, bad);
      owned = cx >= g.own_lo && cx < g.own_hi;
      if (owned) {
        u = upd[t];
        id = uid[t];
        const int cg = cell_coord(u.x, g.ox, g.inv_w, g.gnx, bad);
        cls = cg < lo ? 1 : (cg >= hi ? 2 : 0);
        bad |= (cg < lo - Lx) || (cg >= hi + Lx) || (cls == 1 && rank == 0) || (cls == 2 && rank == nranks - 1);
        // overlapped step: a particle now in a boundary layer must come from the 2 layers the
        // boundary launch computed (its ghost copy was taken from there)
        if (!send) bad |= (cg == lo || cg == hi - 1) && cx >= g.own_lo + 2 && cx < g.own_hi - 2;
      }
    }
    const long long is = agg_append(cls == 0, &ctl->n_stay);
    if (!send) {
      if (cls == 0 && is < cap) {
        xrec[is] = u;
        xid[is] = id;
        xperm[is] = -1;
      }
      continue;
    }
    const long long il = agg_append(cls == 1, &reinterpret_cast<MsgHeader *>(sL)->count);
    const long long ir = agg_append(cls == 2, &reinterpret_cast<MsgHeader *>(sR)->count);
    if (cls == 0 && is < cap) {
      xrec[is] = u;
      xid[is] = id;
      xperm[is] = -1;
    }
    if (cls == 1) msg_put(sL, cap_msg, il, u, id);
    if (cls == 2) msg_put(sR, cap_msg, ir, u, id);
  }
  if (bad) atomicOr(&ctl->flags, FLAG_INTERNAL);
}

// Overlapped step, after the boundary launch: the particles of the first / last 2 owned layers
// (old cell) -> leavers into the migrant messages (set 0), stayers whose new cell is the first /
// last owned layer into the ghost messages (set 1) for rank-1 / rank+1.
__global__ void k_migrate_boundary(Geom g, int rank, int nranks, int Lx, const float4 *__restrict__ rec,
                                   const float4 *__restrict__ upd, const int32_t *__restrict__ uid, MsgSet m,
                                   MsgSet gh, long long cap_msg, DevCtl *ctl) {
  const long long n = ctl->n_total;
  const int lo = rank * Lx, hi = (rank + 1) * Lx;
  bool bad = false;
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < n; t0 += (long long)gridDim.x * blockDim.x) {
    const long long t = t0 + threadIdx.x;
    int cls = -1;  // 0 stay (ghost L), 1 left, 2 right, 3 stay (ghost R)
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t id = 0;
    if (t < n) {
      const int cx = cell_x(g, rec[t].x, bad);
      const bool bnd = (cx >= g.own_lo && cx < g.own_lo + 2) || (cx >= g.own_hi - 2 && cx < g.own_hi);
      if (bnd) {
        u = upd[t];
        id = uid[t];
        const int cg = cell_coord(u.x, g.ox, g.inv_w, g.gnx, bad);
        cls = cg < lo ? 1 : (cg >= hi ? 2 : (cg == lo && rank > 0 ? 0 : (cg == hi - 1 && rank < nranks - 1 ? 3 : -1)));
      }
    }
    const long long il = agg_append(cls == 1, &reinterpret_cast<MsgHeader *>(m.sendL)->count);
    const long long ir = agg_append(cls == 2, &reinterpret_cast<MsgHeader *>(m.sendR)->count);
    const long long gl = agg_append(cls == 0, &reinterpret_cast<MsgHeader *>(gh.sendL)->count);
    const long long gr = agg_append(cls == 3, &reinterpret_cast<MsgHeader *>(gh.sendR)->count);
    if (cls == 1) msg_put(m.sendL, cap_msg, il, u, id);
    if (cls == 2) msg_put(m.sendR, cap_msg, ir, u, id);
    if (cls == 0) msg_put(gh.sendL, cap_msg, gl, u, id);
    if (cls == 3) msg_put(gh.sendR, cap_msg, gr, u, id);
  }
  if (bad) atomicOr(&ctl->flags, FLAG_INTERNAL);
}

// ... and the migrants that arrived (they land in the first / last owned layer: |dx| < w) ->
// ghost messages of the same side (an arrival from rank-1 is a ghost for rank-1 again).
__global__ void k_ghost_arrivals(Geom g, int rank, int nranks, int Lx, MsgSet m, MsgSet gh, long long cap_msg,
                                 DevCtl *ctl) {
  const long long cl = m.recvL ? min(reinterpret_cast<const MsgHeader *>(m.recvL)->count, cap_msg) : 0;
  const long long cr = m.recvR ? min(reinterpret_cast<const MsgHeader *>(m.recvR)->count, cap_msg) : 0;
  const int lo = rank * Lx, hi = (rank + 1) * Lx;
  bool bad = false;
  for (long long k0 = (long long)blockIdx.x * blockDim.x; k0 < cl + cr; k0 += (long long)gridDim.x * blockDim.x) {
    const long long k = k0 + threadIdx.x;
    int cls = -1;
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t id = 0;
    if (k < cl + cr) {
      void *msg = k < cl ? m.recvL : m.recvR;
      const long long j = k < cl ? k : k - cl;
      u = msg_rec(msg)[j];
      id = msg_id(msg, cap_msg)[j];
      const int cg = cell_coord(u.x, g.ox, g.inv_w, g.gnx, bad);
      cls = (cg == lo && rank > 0) ? 0 : ((cg == hi - 1 && rank < nranks - 1) ? 3 : -1);
    }
    const long long gl = agg_append(cls == 0, &reinterpret_cast<MsgHeader *>(gh.sendL)->count);
    const long long gr = agg_append(cls == 3, &reinterpret_cast<MsgHeader *>(gh.sendR)->count);
    if (cls == 0) msg_put(gh.sendL, cap_msg, gl, u, id);
    if (cls == 3) msg_put(gh.sendR, cap_msg, gr, u, id);
  }
  (void)bad;
}

// Appends the records of recvL then recvR at *counter; *result = *counter + arrivals.
__global__ void k_append(const void *rL, const void *rR, const void *sL, const void *sR, long long cap_msg,
                         const long long *counter, long long *result, long long *stat, long long *out_stat,
                         long long cap, float4 *xrec, int32_t *xid, int32_t *xperm, DevCtl *ctl) {
  const long long cl_raw = rL ? reinterpret_cast<const MsgHeader *>(rL)->count : 0;
  const long long cr_raw = rR ? reinterpret_cast<const MsgHeader *>(rR)->count : 0;
  const long long cl = min(cl_raw, cap_msg), cr = min(cr_raw, cap_msg);
  const long long base = *counter;
  long long tot = cl + cr;
  const bool overflow = cl_raw > cap_msg || cr_raw > cap_msg || base + tot > cap;
  if (base + tot > cap) tot = max(0LL, cap - base);
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < tot; k += (long long)gridDim.x * blockDim.x) {
    const void *m = k < cl ? rL : rR;
    const long long j = k < cl ? k : k - cl;
    xrec[base + k] = msg_rec(const_cast<void *>(m))[j];
    xid[base + k] = msg_id(const_cast<void *>(m), cap_msg)[j];
    xperm[base + k] = -1;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *result = base + tot;
    *stat = tot;
    *out_stat = (sL ? reinterpret_cast<const MsgHeader *>(sL)->count : 0) +
                (sR ? reinterpret_cast<const MsgHeader *>(sR)->count : 0);
    if (overflow) atomicOr(&ctl->flags, FLAG_CAPACITY);
  }
}

// Owned particles in the first / last owned X layer -> ghosts for rank-1 / rank+1.
__global__ void k_select_ghosts(Geom g, int rank, int nranks, int Lx, const float4 *__restrict__ xrec,
                                const int32_t *__restrict__ xid, void *sL, void *sR, long long cap_msg, DevCtl *ctl) {
  const long long n = ctl->n_owned;
  const int first = rank * Lx, last = (rank + 1) * Lx - 1;
  bool bad = false;
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < n; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    bool wl = false, wr = false;
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t id = 0;
    if (i < n) {
      r = xrec[i];
      id = xid[i];
      const int cg = cell_coord(r.x, g.ox, g.inv_w, g.gnx, bad);
      wl = rank > 0 && cg == first;
      wr = rank < nranks - 1 && cg == last;
    }
    const long long il = agg_append(wl, &reinterpret_cast<MsgHeader *>(sL)->count);
    const long long ir = agg_append(wr, &reinterpret_cast<MsgHeader *>(sR)->count);
    if (wl) msg_put(sL, cap_msg, il, r, id);
    if (wr) msg_put(sR, cap_msg, ir, r, id);
  }
  (void)bad;
}

__global__ void k_export_owned(Geom g, const float4 *__restrict__ rec_old, const float4 *__restrict__ pos,
                               const int32_t *__restrict__ ids, const float4 *__restrict__ outs, float *x, float *y,
                               float *z, float *q, int32_t *id, float *phi, float *fx, float *fy, float *fz,
                               DevCtl *ctl) {
  const long long n = ctl->n_total;
  bool bad = false;
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < n; t0 += (long long)gridDim.x * blockDim.x) {
    const long long t = t0 + threadIdx.x;
    bool owned = false;
    if (t < n) {
      const int cx = cell_x(g, rec_old[t].x, bad);
      owned = cx >= g.own_lo && cx < g.own_hi;
    }
    const long long k = agg_append(owned, &ctl->pad2[0]);
    if (owned) {
      const float4 r = pos[t];
      if (x) x[k] = r.x;
      if (y) y[k] = r.y;
      if (z) z[k] = r.z;
      if (q) q[k] = r.w;
      if (id) id[k] = ids[t];
      if (outs) {
        const float4 o = outs[t];
        if (phi) phi[k] = o.x;
        if (fx) fx[k] = o.y;
        if (fy) fy[k] = o.z;
        if (fz) fz[k] = o.w;
      }
    }
  }
}

// ------------------------------------------------------------------ transports
struct LocalGroup {
  int nranks = 0;
  std::vector<SlabState *> members;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  // false when the other ranks did not arrive within 120 s (a rank failed before its exchange)
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; });
  }
};

std::mutex g_reg_mutex;
std::map<std::string, LocalGroup *> &registry() {
  static std::map<std::string, LocalGroup *> r;
  return r;
}

struct LocalTransport : Transport {
  LocalGroup *grp;
  std::string key;
  int rank;
  LocalTransport(LocalGroup *g, std::string k, int r) : grp(g), key(std::move(k)), rank(r) {}
  ~LocalTransport() override {
    std::lock_guard<std::mutex> lk(g_reg_mutex);
    grp->members[rank] = nullptr;
    bool empty = true;
    for (auto *p : grp->members) empty &= p == nullptr;
    if (empty) {
      registry().erase(key);
      delete grp;
    }
  }
  cudaError_t run(SlabState &S, int set, cudaStream_t s, const Xfer *L, int nL, const Xfer *R, int nR) override {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    if (!grp->barrier()) return cudaErrorTimeout;  // every rank's send buffers are complete
    auto u8 = [](void *p, size_t o) { return static_cast<unsigned char *>(p) + o; };
    const MsgSet me = S.set(set);
    if (S.rank > 0) {
      const MsgSet P = grp->members[S.rank - 1]->set(set);
      for (int k = 0; k < nL && e == cudaSuccess; ++k)
        if (L[k].rbytes)
          e = cudaMemcpyAsync(u8(me.recvL, L[k].off), u8(P.sendR, L[k].off), L[k].rbytes, cudaMemcpyDeviceToDevice, s);
    }
    if (S.rank < S.nranks - 1) {
      const MsgSet P = grp->members[S.rank + 1]->set(set);
      for (int k = 0; k < nR && e == cudaSuccess; ++k)
        if (R[k].rbytes)
          e = cudaMemcpyAsync(u8(me.recvR, R[k].off), u8(P.sendL, R[k].off), R[k].rbytes, cudaMemcpyDeviceToDevice, s);
    }
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(s);
    if (!grp->barrier()) return cudaErrorTimeout;  // nobody overwrites a send buffer still being read
    return e;
  }
  const char *name() const override { return "local"; }
};

// Minimal NCCL declarations (ABI-stable since NCCL 2.0); the library is the one torch loaded.
typedef struct ncclComm *ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
typedef ncclResult_t (*fn_getid)(ncclUniqueId *);
typedef ncclResult_t (*fn_init)(ncclComm_t *, int, ncclUniqueId, int);
typedef ncclResult_t (*fn_destroy)(ncclComm_t);
typedef ncclResult_t (*fn_sendrecv)(void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*fn_group)(void);
typedef const char *(*fn_errstr)(ncclResult_t);

struct NcclApi {
  void *h = nullptr;
  fn_getid getid = nullptr;
  fn_init init = nullptr;
  fn_destroy destroy = nullptr;
  fn_sendrecv send = nullptr, recv = nullptr;
  fn_group gstart = nullptr, gend = nullptr;
  fn_errstr errstr = nullptr;
  bool load(char *why, size_t n) {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(why, n, "dlopen libnccl.so.2 failed: %s", dlerror());
      return false;
    }
    getid = (fn_getid)dlsym(h, "ncclGetUniqueId");
    init = (fn_init)dlsym(h, "ncclCommInitRank");
    destroy = (fn_destroy)dlsym(h, "ncclCommDestroy");
    send = (fn_sendrecv)dlsym(h, "ncclSend");
    recv = (fn_sendrecv)dlsym(h, "ncclRecv");
    gstart = (fn_group)dlsym(h, "ncclGroupStart");
    gend = (fn_group)dlsym(h, "ncclGroupEnd");
    errstr = (fn_errstr)dlsym(h, "ncclGetErrorString");
    if (!getid || !init || !destroy || !send || !recv || !gstart || !gend) {
      snprintf(why, n, "libnccl.so.2 lacks the point-to-point API");
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm) g_nccl.destroy(comm);
  }
  cudaError_t run(SlabState &S, int set, cudaStream_t s, const Xfer *L, int nL, const Xfer *R, int nR) override {
    constexpr int ncclChar = 0;
    auto u8 = [](void *p, size_t o) { return static_cast<unsigned char *>(p) + o; };
    const MsgSet m = S.set(set);
    if (g_nccl.gstart() != 0) return cudaErrorUnknown;
    bool ok = true;
    if (S.rank > 0)
      for (int k = 0; k < nL; ++k) {
        if (L[k].sbytes) ok &= g_nccl.send(u8(m.sendL, L[k].off), L[k].sbytes, ncclChar, S.rank - 1, comm, s) == 0;
        if (L[k].rbytes) ok &= g_nccl.recv(u8(m.recvL, L[k].off), L[k].rbytes, ncclChar, S.rank - 1, comm, s) == 0;
      }
    if (S.rank < S.nranks - 1)
      for (int k = 0; k < nR; ++k) {
        if (R[k].sbytes) ok &= g_nccl.send(u8(m.sendR, R[k].off), R[k].sbytes, ncclChar, S.rank + 1, comm, s) == 0;
        if (R[k].rbytes) ok &= g_nccl.recv(u8(m.recvR, R[k].off), R[k].rbytes, ncclChar, S.rank + 1, comm, s) == 0;
      }
    ok &= g_nccl.gend() == 0;
    return ok ? cudaSuccess : cudaErrorUnknown;
  }
  const char *name() const override { return "nccl"; }
};

}  // namespace

cudaError_t slab_exchange(SlabState &S, cudaStream_t s, int set) {
  const bool hasL = S.rank > 0, hasR = S.rank < S.nranks - 1;
  if (!S.counted || !S.hcnt) {  // the whole fixed-capacity messages, no host synchronisation
    const Xfer x{0, msg_bytes(S.cap_msg), msg_bytes(S.cap_msg)};
    S.bytes_sent += (long long)x.sbytes * (hasL + hasR);
    return S.tr->run(S, set, s, &x, hasL, &x, hasR);
  }
  // phase 1: the headers (counts)
  const Xfer h{0, sizeof(MsgHeader), sizeof(MsgHeader)};
  cudaError_t e = S.tr->run(S, set, s, &h, hasL, &h, hasR);
  const MsgSet m = S.set(set);
  void *hd[4] = {m.sendL, m.sendR, m.recvL, m.recvR};
  for (int k = 0; k < 4 && e == cudaSuccess; ++k)
    e = cudaMemcpyAsync(S.hcnt + k, hd[k], sizeof(long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  auto clampc = [&](long long v) { return (size_t)std::min(std::max(v, 0LL), S.cap_msg); };
  const size_t sl = hasL ? clampc(S.hcnt[0]) : 0, sr = hasR ? clampc(S.hcnt[1]) : 0;
  const size_t rl = hasL ? clampc(S.hcnt[2]) : 0, rr = hasR ? clampc(S.hcnt[3]) : 0;
  // phase 2: rec[0, n) and id[0, n) of each message (k_append reads the counts from the headers)
  const size_t o_rec = sizeof(MsgHeader), o_id = sizeof(MsgHeader) + (size_t)S.cap_msg * 16;
  const Xfer L[2] = {{o_rec, sl * 16, rl * 16}, {o_id, sl * 4, rl * 4}};
  const Xfer R[2] = {{o_rec, sr * 16, rr * 16}, {o_id, sr * 4, rr * 4}};
  S.bytes_sent += (long long)((sl + sr) * 20 + sizeof(MsgHeader) * (hasL + hasR));
  return S.tr->run(S, set, s, L, hasL ? 2 : 0, R, hasR ? 2 : 0);
}

bool nccl_unique_id(void *out128, char *why, size_t n) {
  if (!g_nccl.load(why, n)) return false;
  ncclUniqueId id;
  if (g_nccl.getid(&id) != 0) {
    snprintf(why, n, "ncclGetUniqueId failed");
    return false;
  }
  memcpy(out128, &id, 128);
  return true;
}

Transport *make_transport(const pi_config *cfg, SlabState *S, char *why, size_t n) {
  const char *uid = reinterpret_cast<const char *>(cfg->nccl_unique_id);
  if (!uid) {
    snprintf(why, n, "nranks > 1 needs nccl_unique_id");
    return nullptr;
  }
  if (strncmp(uid, "PILOCAL:", 8) == 0) {
    std::string key(uid + 8, strnlen(uid + 8, 120));
    std::lock_guard<std::mutex> lk(g_reg_mutex);
    LocalGroup *&grp = registry()[key];
    if (!grp) {
      grp = new LocalGroup();
      grp->nranks = cfg->nranks;
      grp->members.assign(cfg->nranks, nullptr);
    }
    if (grp->nranks != cfg->nranks || grp->members[cfg->rank]) {
      snprintf(why, n, "local link '%s': inconsistent nranks or duplicate rank", key.c_str());
      return nullptr;
    }
    grp->members[cfg->rank] = S;
    return new LocalTransport(grp, key, cfg->rank);
  }
  if (!g_nccl.load(why, n)) return nullptr;
  auto *t = new NcclTransport();
  ncclUniqueId id;
  memcpy(&id, uid, 128);
  const ncclResult_t r = g_nccl.init(&t->comm, cfg->nranks, id, cfg->rank);
  if (r != 0) {
    snprintf(why, n, "ncclCommInitRank failed: %s", g_nccl.errstr ? g_nccl.errstr(r) : "?");
    delete t;
    return nullptr;
  }
  return t;
}

cudaError_t slab_reset(SlabState &S, DevCtl *ctl, cudaStream_t s, int set, bool stay) {
  const MsgSet m = S.set(set);
  k_reset<<<1, 32, 0, s>>>(m.sendL, m.sendR, m.recvL, m.recvR, ctl, stay);
  return cudaGetLastError();
}

cudaError_t slab_from_soa(SlabState &S, const Geom &g, long long n, const float *x, const float *y, const float *z,
                          const float *q, const int32_t *id, DevCtl *ctl, cudaStream_t s) {
  k_soa_to_x<<<blocks_for(n), T, 0, s>>>(g, S.rank * S.Lx, (S.rank + 1) * S.Lx, n, x, y, z, q, id, S.xrec, S.xid,
                                         S.xperm, ctl);
  return cudaGetLastError();
}

cudaError_t slab_migrate(SlabState &S, const Geom &g, long long cap, const float4 *rec, const float4 *upd,
                         const int32_t *uid, DevCtl *ctl, cudaStream_t s, bool send) {
  k_migrate<<<blocks_for(cap), T, 0, s>>>(g, cap, S.rank, S.nranks, S.Lx, rec, upd, uid, S.xrec, S.xid, S.xperm,
                                          S.sendL, S.sendR, S.cap_msg, ctl, send);
  return cudaGetLastError();
}

cudaError_t slab_migrate_boundary(SlabState &S, const Geom &g, long long cap, const float4 *rec, const float4 *upd,
                                  const int32_t *uid, DevCtl *ctl, cudaStream_t s) {
  // a few blocks: they run beside the interior launch (on the SMs it leaves free, or in the
  // registers and threads its blocks leave on every SM)
  k_migrate_boundary<<<min(blocks_for(cap), 148 * 2), T, 0, s>>>(g, S.rank, S.nranks, S.Lx, rec, upd, uid, S.set(0),
                                                                 S.set(1), S.cap_msg, ctl);
  return cudaGetLastError();
}

cudaError_t slab_ghost_arrivals(SlabState &S, const Geom &g, DevCtl *ctl, cudaStream_t s) {
  const bool l = S.rank > 0, r = S.rank < S.nranks - 1;
  MsgSet m = S.set(0);
  if (!l) m.recvL = nullptr;
  if (!r) m.recvR = nullptr;
  k_ghost_arrivals<<<blocks_for(2 * S.cap_msg), T, 0, s>>>(g, S.rank, S.nranks, S.Lx, m, S.set(1), S.cap_msg, ctl);
  return cudaGetLastError();
}

cudaError_t slab_append(SlabState &S, long long *counter, long long *result, long long *stat, long long *out_stat,
                        long long cap, DevCtl *ctl, cudaStream_t s, int set) {
  const bool l = S.rank > 0, r = S.rank < S.nranks - 1;
  const MsgSet m = S.set(set);
  k_append<<<blocks_for(2 * S.cap_msg), T, 0, s>>>(l ? m.recvL : nullptr, r ? m.recvR : nullptr, l ? m.sendL : nullptr,
                                                   r ? m.sendR : nullptr, S.cap_msg, counter, result, stat, out_stat,
                                                   cap, S.xrec, S.xid, S.xperm, ctl);
  return cudaGetLastError();
}

cudaError_t slab_select_ghosts(SlabState &S, const Geom &g, long long cap, DevCtl *ctl, cudaStream_t s) {
  k_select_ghosts<<<blocks_for(cap), T, 0, s>>>(g, S.rank, S.nranks, S.Lx, S.xrec, S.xid, S.sendL, S.sendR,
                                                S.cap_msg, ctl);
  return cudaGetLastError();
}

cudaError_t slab_export_owned(const Geom &g, long long cap, const float4 *rec_old, const float4 *pos,
                              const int32_t *ids, const float4 *outs, float *x, float *y, float *z, float *q,
                              int32_t *id, float *phi, float *fx, float *fy, float *fz, DevCtl *ctl,
                              cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(&ctl->pad2[0], 0, sizeof(long long), s);
  if (e != cudaSuccess) return e;
  k_export_owned<<<blocks_for(cap), T, 0, s>>>(g, rec_old, pos, ids, outs, x, y, z, q, id, phi, fx, fy, fz, ctl);
  return cudaGetLastError();
}

}  // namespace pi
