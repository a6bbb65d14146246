// X-slab decomposition across ranks (north star; the paper itself is single-GPU).
//
// Rank r of P owns the global X cells [r Lx, (r+1) Lx), Lx = dims[0] / P.  Its local grid is
// Lx + 2 X layers: local 0 and Lx+1 are source-only GHOST layers holding the neighbours'
// boundary layers, local 1..Lx are owned (targets).  Boundaries are open, so ranks 0 and P-1
// have one neighbour.  Per step (pi_step): the position update moves particles; the ones
// whose new global cell left the slab MIGRATE to r-1 / r+1 (|dx| < w per step: reading C11);
// then the first / last owned layers are sent as ghosts; owned + ghosts are binned together
// (the ghosts land in the ghost layers) and only owned cells are targets, so no reduction is
// needed.  Messages are fixed-capacity (count header + records), so the exchange needs no
// host synchronisation and no variable-size handshake.
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

struct SlabState {
  int rank = 0, nranks = 1, Lx = 0;
  long long cap_msg = 0;
  void *sendL = nullptr, *sendR = nullptr, *recvL = nullptr, *recvR = nullptr;
  float4 *xrec = nullptr;  // owned (+ arrivals, + ghosts) records: input of the binning
  int32_t *xid = nullptr, *xperm = nullptr;
  Transport *tr = nullptr;
};

struct Transport {
  virtual ~Transport() {}
  // sendL -> rank-1 (lands in its recvR), sendR -> rank+1 (its recvL); stream ordered.
  virtual cudaError_t exchange(SlabState &S, cudaStream_t s) = 0;
  virtual const char *name() const = 0;
};

// Creates the transport for cfg: "PILOCAL:<key>" ids link contexts of one process (testing on
// one GPU), otherwise an NCCL communicator over cfg->nccl_unique_id (libnccl.so.2 is loaded
// with dlopen, the same library torch uses).  Returns NULL and fills `why` on failure.
Transport *make_transport(const pi_config *cfg, SlabState *S, char *why, size_t n);
bool nccl_unique_id(void *out128, char *why, size_t n);

// Kernels (slab.cu)
cudaError_t slab_reset(SlabState &S, DevCtl *ctl, cudaStream_t s);
cudaError_t slab_from_soa(SlabState &S, const Geom &g, long long n, const float *x, const float *y, const float *z,
                          const float *q, const int32_t *id, DevCtl *ctl, cudaStream_t s);
cudaError_t slab_migrate(SlabState &S, const Geom &g, long long cap, const float4 *rec, const float4 *upd,
                         const int32_t *uid, DevCtl *ctl, cudaStream_t s);
// *stat = records appended, *out_stat = records this rank sent in the same exchange
cudaError_t slab_append(SlabState &S, long long *counter, long long *result, long long *stat, long long *out_stat,
                        long long cap, DevCtl *ctl, cudaStream_t s);
cudaError_t slab_select_ghosts(SlabState &S, const Geom &g, long long cap, DevCtl *ctl, cudaStream_t s);
cudaError_t slab_export_owned(const Geom &g, long long cap, const float4 *rec_old, const float4 *pos,
                              const int32_t *ids, const float4 *outs, float *x, float *y, float *z, float *q,
                              int32_t *id, float *phi, float *fx, float *fy, float *fz, DevCtl *ctl,
                              cudaStream_t s);

}  // namespace pi
