// X-slab decomposition across ranks (north star; the paper itself is single-GPU).
//
// Rank r of P owns the global X cells [r Lx, (r+1) Lx), Lx = dims[0] / P.  Its local grid is
// Lx + 2 X layers: local 0 and Lx+1 are source-only GHOST layers holding the neighbours'
// boundary layers, local 1..Lx are owned (targets).  Boundaries are open, so ranks 0 and P-1
// have one neighbour.  Per step (pi_step): the position update moves particles; the ones
// whose new global cell left the slab MIGRATE to r-1 / r+1 (|dx| < w per step: reading C11);
// then the first / last owned layers are sent as ghosts; owned + ghosts are binned together
// (the ghosts land in the ghost layers) and only owned cells are targets, so no reduction is
// needed.  Messages are fixed-capacity buffers (count header + records).  The exchange runs in
// two phases: the headers (the counts) first, then exactly the counted records
// (rec[0, n) and id[0, n)), so the link carries the real payload, not the capacity; the counts
// reach the host through a pinned buffer (one stream synchronisation per exchange).  With
// counted = false the whole fixed-capacity message is sent and no host synchronisation is needed
// (CUDA-graph capturable with the NCCL transport).
#pragma once
#include "pi_internal.cuh"

namespace pi {

struct MsgHeader {
  long long count;  // records the sender wanted to send (may exceed the capacity: error)
  long long pad;
};
// Message layout: header | float4 rec[cap] | int32 id[cap]
__host__ __device__ inline size_t msg_bytes(long long cap) {
  return (sizeof(MsgHeader) + (size_t)cap * 20 + 255) & ~size_t(255);
}
__host__ __device__ inline float4 *msg_rec(void *m) {
  return reinterpret_cast<float4 *>(reinterpret_cast<unsigned char *>(m) + sizeof(MsgHeader));
}
__host__ __device__ inline int32_t *msg_id(void *m, long long cap) {
  return reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(m) + sizeof(MsgHeader) + (size_t)cap * 16);
}

struct Transport;

// The four message buffers of one exchange.  Set 0 carries migrants and (in the serial step)
// ghosts; set 1 the ghosts of the overlapped step, whose migrant and ghost exchanges are both in
// flight while the interior cells are computed.
struct MsgSet {
  void *sendL, *sendR, *recvL, *recvR;
};

struct SlabState {
  int rank = 0, nranks = 1, Lx = 0;
  long long cap_msg = 0;
  bool counted = true;           // two-phase exchange: headers, then exactly the counted records
  long long *hcnt = nullptr;     // pinned host [4]: send L, send R, recv L, recv R counts
  long long bytes_sent = 0;      // payload bytes this rank put on the links (host bookkeeping)
  void *sendL = nullptr, *sendR = nullptr, *recvL = nullptr, *recvR = nullptr;  // set 0
  MsgSet g{};                                                                     // set 1
  MsgSet set(int k) const { return k ? g : MsgSet{sendL, sendR, recvL, recvR}; }
  float4 *xrec = nullptr;  // owned (+ arrivals, + ghosts) records: input of the binning
  int32_t *xid = nullptr, *xperm = nullptr;
  Transport *tr = nullptr;
};

// One region of the messages moved between neighbours: bytes [off, off + sbytes) of this rank's
// send buffer go to the neighbour, and [off, off + rbytes) of this rank's receive buffer are
// filled from the neighbour's send buffer (the same layout on both sides).
struct Xfer {
  size_t off, sbytes, rbytes;
};

struct Transport {
  virtual ~Transport() {}
  // Grouped point-to-point on message set k: regions L[0..nL) with rank-1 (sendL -> its recvR,
  // its sendR -> recvL) and R[0..nR) with rank+1; stream ordered.  Zero-byte sides are skipped
  // (both ends agree: the sizes come from the same counts).
  virtual cudaError_t run(SlabState &S, int k, cudaStream_t s, const Xfer *L, int nL, const Xfer *R, int nR) = 0;
  virtual const char *name() const = 0;
};
// The a8 exchange of message set k (both phases, see above).
cudaError_t slab_exchange(SlabState &S, cudaStream_t s, int k = 0);

// Creates the transport for cfg: "PILOCAL:<key>" ids link contexts of one process (testing on
// one GPU), otherwise an NCCL communicator over cfg->nccl_unique_id (libnccl.so.2 is loaded
// with dlopen, the same library torch uses).  Returns NULL and fills `why` on failure.
Transport *make_transport(const pi_config *cfg, SlabState *S, char *why, size_t n);
bool nccl_unique_id(void *out128, char *why, size_t n);

// Kernels (slab.cu)
// zeroes the headers of message set k (and n_stay if `stay`)
cudaError_t slab_reset(SlabState &S, DevCtl *ctl, cudaStream_t s, int k = 0, bool stay = true);
cudaError_t slab_from_soa(SlabState &S, const Geom &g, long long n, const float *x, const float *y, const float *z,
                          const float *q, const int32_t *id, DevCtl *ctl, cudaStream_t s);
// send = false: the stayers only (the overlapped step sent the migrants already); the particles
// that reach a boundary layer from outside the layers the first launch computed raise
// FLAG_INTERNAL (the per-step move bound |dt F| < w, reading C11, was broken)
cudaError_t slab_migrate(SlabState &S, const Geom &g, long long cap, const float4 *rec, const float4 *upd,
                         const int32_t *uid, DevCtl *ctl, cudaStream_t s, bool send = true);
// Overlapped step, after the launch over the boundary layers (the first and last 2 owned
// layers): their leavers -> migrant messages (set 0), their stayers now in the first / last
// owned layer -> ghost messages (set 1)
cudaError_t slab_migrate_boundary(SlabState &S, const Geom &g, long long cap, const float4 *rec, const float4 *upd,
                                  const int32_t *uid, DevCtl *ctl, cudaStream_t s);
// ... then, after the migrant exchange, the arrivals (all in a boundary layer) -> ghost messages
cudaError_t slab_ghost_arrivals(SlabState &S, const Geom &g, DevCtl *ctl, cudaStream_t s);
// *stat = records appended from set k, *out_stat = records this rank sent in that exchange
cudaError_t slab_append(SlabState &S, long long *counter, long long *result, long long *stat, long long *out_stat,
                        long long cap, DevCtl *ctl, cudaStream_t s, int k = 0);
cudaError_t slab_select_ghosts(SlabState &S, const Geom &g, long long cap, DevCtl *ctl, cudaStream_t s);
cudaError_t slab_export_owned(const Geom &g, long long cap, const float4 *rec_old, const float4 *pos,
                              const int32_t *ids, const float4 *outs, float *x, float *y, float *z, float *q,
                              int32_t *id, float *phi, float *fx, float *fy, float *fz, DevCtl *ctl,
                              cudaStream_t s);

}  // namespace pi
