// Shared pieces of the shared-memory interaction kernels (a6.2 full load, a6.3 X-pencil).
//
// Both kernels end up with the same compute core: the candidates of a target cell are ONE
// contiguous window of staged sources in shared memory (the "merged" layout of the staging
// code).  A thread owns one target (as the paper's kernels do) and walks that window two
// sources at a time in packed-fp32 (f32x2) registers: 12 FADD2/FMUL2/FFMA2 and 2 MUFU.EX2
// per 2 candidate pairs:
//
//   d   = x_s - x_t per axis, from the raw fp32 positions (exact when the two are within a
//         factor 2 of each other -- Sterbenz -- so every component is accurate on its own)
//   r2  = |d|^2,  in = r2 < r_c^2              ( r < r_c, strict; PAPER.md:50 )
//   w   = in ? q_s 2^(-c2 r2) : 0              ( = q_s K(r), K = exp(-r^2 / (2 sigma^2)),
//                                                c2 = log2(e) / (2 sigma^2) )
//   phi_t = sum w,   F_t = -(q_t / sigma^2) sum w d
//
// Self-exclusion (Alg. 1 :127, identity): the self pair IS evaluated inside the window (its
// d is exactly 0, so it adds nothing to F); the lane that evaluated it recomputes the
// identical rounded phi term and subtracts it, so an isolated particle comes out exactly 0.
#pragma once
#include "pi_internal.cuh"

namespace pi {

// Packed fp32 (f32x2) helpers on 64-bit registers: ptxas keeps each value in an aligned
// register pair and turns a {s, s} operand into a scalar broadcast (FFMA2 R, R.F32x2, S.F32).
typedef float2 p2;
__device__ __forceinline__ p2 pk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ p2 pk(float a) { return make_float2(a, a); }
__device__ __forceinline__ float lo(p2 v) { return v.x; }
__device__ __forceinline__ float hi(p2 v) { return v.y; }
__device__ __forceinline__ p2 fma2(p2 a, p2 b, p2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ p2 add2(p2 a, p2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ p2 mul2(p2 a, p2 b) { return __fmul2_rn(a, b); }

// ---------------------------------------------------------------- TMA / mbarrier helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// The waiting warp is suspended until the phase completes (suspend-time hint: an upper bound in
// ns, the thread resumes as soon as the barrier completes).  Without the hint a try_wait
// returns at once and the loop spins: measured, X-pencil consumers waiting for a slot issued 17 %
// of the kernel's instructions in that loop, issue slots the computing warps of the same
// scheduler needed.
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
// Wait with backoff, for a warp that has nothing else to do (a producer waiting for its slot
// to be released): without the sleep its try_wait loop takes issue slots from the compute
// warps of its scheduler for the whole wait.
__device__ __forceinline__ bool mbar_try_wait(unsigned long long *bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long *bar, unsigned parity) {
  unsigned ns = 64;
  while (!mbar_try_wait(bar, parity)) {
    __nanosleep(ns);
    ns = ns < 2048 ? 2 * ns : 2048;
  }
}

// 1-D bulk copy global -> shared (TMA, SASS UBLKCP); dst/src 16-B aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 16-B asynchronous global -> shared copy (LDGSTS), bypassing L1.
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Staged sources are stored as PAIRS (sources 2p and 2p+1) in two planes of 16-B elements:
//   A[p] = (x~_2p, x~_2p+1, y~_2p, y~_2p+1)      B[p] = (z~_2p, z~_2p+1, q_2p, q_2p+1)
// so one LDS.128 yields aligned f32x2 operands and the lane's scalar target coordinate is
// the broadcast operand of FADD2 (FADD2 R, R.F32x2, -Rt.F32).  Planes rather than the
// interleaved A[p] B[p] records: the lanes of a quarter-warp read pairs a few apart (targets in
// neighbouring X sub-cells), which conflict when p == p' mod 8 on planes but p == p' mod 4 when
// interleaved (measured: 4.27 wavefronts per LDS.128 interleaved against 3.3 ideal).
struct SrcPair {
  p2 x, y, z, q;
};
__device__ __forceinline__ SrcPair load_pair(const float4 *__restrict__ A, const float4 *__restrict__ B, int p) {
  const float4 a = A[p], b = B[p];
  SrcPair r;
  r.x = pk(a.x, a.y);
  r.y = pk(a.z, a.w);
  r.z = pk(b.x, b.y);
  r.q = pk(b.z, b.w);
  return r;
}

// The kernel-cost sweep's fake kernels (Fig. "diffflops"; reading R22):
//   PI_K_LOWFLOP  "summing the positions": c_ij = (x_j + y_j + z_j, x_j, y_j, z_j) inside r_c;
//   PI_K_HIGHFLOP "the Lennard-Jones kernel with 150 added FLOP": Eq. (1), its potential term
//                 u = s^6 - s^3 run through 75 FMAs t <- t a + b (150 FLOP) before the value
//                 q_j 4 E0 t is summed (the force is the LJ force).  a = 1 - 2^-7, b = 2^-10: the
//                 chain is the affine map A u + B, A = a^75, B = b (1 - A) / (1 - a).
__host__ __device__ constexpr bool kern_lj(int k) { return k == PI_K_LJ || k == PI_K_HIGHFLOP; }
__host__ __device__ constexpr bool kern_wforce(int k) { return k == PI_K_GAUSSIAN || kern_lj(k); }
constexpr int HF_STEPS = 75;
constexpr float HF_A = 0.9921875f;  // 1 - 2^-7
constexpr float HF_B = 0x1p-10f;
__device__ __forceinline__ p2 hf_chain(p2 t) {
#pragma unroll 15
  for (int k = 0; k < HF_STEPS; ++k) t = fma2(t, pk(HF_A), pk(HF_B));
  return t;
}
__device__ __forceinline__ float hf_chain1(float t) {  // the same rounded operations, one value
#pragma unroll 15
  for (int k = 0; k < HF_STEPS; ++k) t = fmaf(t, HF_A, HF_B);
  return t;
}
// LOWFLOP: the sum of a source's position components, in the order every strategy uses
__device__ __forceinline__ float lf_sum(float x, float y, float z) { return __fadd_rn(__fadd_rn(x, y), z); }
__device__ __forceinline__ p2 lf_sum2(p2 x, p2 y, p2 z) { return add2(add2(x, y), z); }

// Lennard-Jones core (Eq. (1), reading R19) on f32x2 values: s = (d~/r)^2 = r2 / r^2 + eps^2 / r^2;
// returns the potential and force weights of the pair halves with q masked to the cutoff
// (qm = r2 < r_c^2 ? q : 0):  w = qm (s^6 - s^3),  wf = qm (12 s^5 - 6 s^2).
template <int KERNEL = PI_K_LJ>
__device__ __forceinline__ void lj_core(p2 r2, p2 q, const float thr, const KParams &kp, p2 &w, p2 &wf) {
  // clamp to r_c^2 before the powers: an inert padding partner (x = 1e30) would give s = inf,
  // inf - inf = NaN and NaN * 0 = NaN; masked halves only need finite values
  const p2 rc = pk(fminf(lo(r2), thr), fminf(hi(r2), thr));
  const p2 s = fma2(rc, pk(kp.lj_inv_r2), pk(kp.lj_e2));
  const p2 s2 = mul2(s, s);
  const p2 s3 = mul2(s2, s);
  const p2 s6 = mul2(s3, s3);
  const p2 s5 = mul2(s3, s2);
  p2 pot = add2(s6, pk(-lo(s3), -hi(s3)));
  if (KERNEL == PI_K_HIGHFLOP) pot = hf_chain(pot);
  const p2 fk = fma2(s5, pk(12.f), mul2(s2, pk(-6.f)));
  const p2 qm = pk((lo(r2) < thr) ? lo(q) : 0.f, (hi(r2) < thr) ? hi(q) : 0.f);
  w = mul2(pot, qm);
  wf = mul2(fk, qm);
}

// One source pair against the thread's target (xt, yt, zt); thr = r_c^2, mc2 = -c2.
// Gaussian: 12 packed-fp32 operations and 2 MUFU.EX2 for 2 candidates.
template <int KERNEL>
__device__ __forceinline__ void src_eval(const SrcPair &s, float xt, float yt, float zt, const float thr,
                                         const float mc2, p2 &phi, p2 &fx, p2 &fy, p2 &fz,
                                         const KParams *kp = nullptr) {
  if (KERNEL == PI_K_CANDIDATE) {
    phi = add2(phi, s.q);
    return;
  }
  // d = x_s - x_t (the target is the broadcast scalar operand)
  const p2 dx = add2(s.x, pk(-xt));
  const p2 dy = add2(s.y, pk(-yt));
  const p2 dz = add2(s.z, pk(-zt));
  p2 r2 = mul2(dx, dx);
  r2 = fma2(dy, dy, r2);
  r2 = fma2(dz, dz, r2);
  if (KERNEL == PI_K_GAUSSIAN) {
    const p2 arg = mul2(r2, pk(mc2));
    const float k0 = (lo(r2) < thr) ? ex2_approx(lo(arg)) : 0.f;
    const float k1 = (hi(r2) < thr) ? ex2_approx(hi(arg)) : 0.f;
    const p2 w = mul2(pk(k0, k1), s.q);
    phi = add2(phi, w);
    fx = fma2(w, dx, fx);
    fy = fma2(w, dy, fy);
    fz = fma2(w, dz, fz);
  } else if (KERNEL == PI_K_LOWFLOP) {  // selects, not products: an inert partner is at 1e30
    const bool i0 = lo(r2) < thr, i1 = hi(r2) < thr;
    const p2 sm = lf_sum2(s.x, s.y, s.z);
    phi = add2(phi, pk(i0 ? lo(sm) : 0.f, i1 ? hi(sm) : 0.f));
    fx = add2(fx, pk(i0 ? lo(s.x) : 0.f, i1 ? hi(s.x) : 0.f));
    fy = add2(fy, pk(i0 ? lo(s.y) : 0.f, i1 ? hi(s.y) : 0.f));
    fz = add2(fz, pk(i0 ? lo(s.z) : 0.f, i1 ? hi(s.z) : 0.f));
  } else if (kern_lj(KERNEL)) {
    p2 w, wf;
    lj_core<KERNEL>(r2, s.q, thr, *kp, w, wf);
    phi = add2(phi, w);
    fx = fma2(wf, dx, fx);
    fy = fma2(wf, dy, fy);
    fz = fma2(wf, dz, fz);
  } else {
    const float k0 = (lo(r2) < thr) ? lo(s.q) : 0.f;
    const float k1 = (hi(r2) < thr) ? hi(s.q) : 0.f;
    phi = add2(phi, pk(k0, k1));
  }
}

// The phi term a walk over the self pair adds for a target of value q (d = 0): q for the
// Gaussian (K(0) = 2^0 = 1), INDICATOR and CANDIDATE kernels; for LJ the same rounded
// operations as lj_core at r2 = 0 (fma(0, ., e2) = e2), so the subtraction is exact.
template <int KERNEL>
__device__ __forceinline__ float self_term(float q, const KParams &kp) {
  if (!kern_lj(KERNEL)) return q;
  const float s = kp.lj_e2;
  const float s2 = __fmul_rn(s, s), s3 = __fmul_rn(s2, s), s6 = __fmul_rn(s3, s3);
  float pot = __fsub_rn(s6, s3);
  if (KERNEL == PI_K_HIGHFLOP) pot = hf_chain1(pot);
  return __fmul_rn(pot, q);
}
// The self pair's full term (phi, F accumulators) for target me: LOWFLOP sums the positions,
// so its self pair adds (x + y + z, x, y, z); every other kernel adds (self_term, 0, 0, 0).
template <int KERNEL>
__device__ __forceinline__ float4 self_terms(const float4 &me, const KParams &kp) {
  if (KERNEL == PI_K_LOWFLOP) return make_float4(lf_sum(me.x, me.y, me.z), me.x, me.y, me.z);
  return make_float4(self_term<KERNEL>(me.w, kp), 0.f, 0.f, 0.f);
}

// Scalar contribution of a source of value qs at squared distance r2 (inside the cutoff):
// w (phi, before phi_scale) and wf (force weight: F += wf (x_t - x_s), before q_t f_ts).
template <int KERNEL>
__device__ __forceinline__ void scalar_term(const KParams &kp, float r2, float qs, float &w, float &wf) {
  if (kern_lj(KERNEL)) {
    const float s = fmaf(r2, kp.lj_inv_r2, kp.lj_e2);
    const float s2 = s * s, s3 = s2 * s, s6 = s3 * s3, s5 = s3 * s2;
    w = (KERNEL == PI_K_HIGHFLOP ? hf_chain1(s6 - s3) : (s6 - s3)) * qs;
    wf = fmaf(s5, 12.f, s2 * -6.f) * qs;
  } else {
    w = qs * ex2_approx(-kp.c2 * r2);
    wf = w;
  }
}

// ---- a PAIR of targets per thread (packed f32x2 over the two targets), sources as broadcast
// scalars (full load; the X-pencil's interleaved staging)
struct TgtPair {
  p2 x, y, z;
};

// One source (scalar broadcast) against the thread's two targets: 12 packed ops, 2 MUFU.
template <int KERNEL>
__device__ __forceinline__ void tp_eval(const TgtPair &t, const float4 a, const float thr, const float mc2, p2 &phi,
                                        p2 &fx, p2 &fy, p2 &fz, const KParams &kp) {
  if (KERNEL == PI_K_CANDIDATE) {
    phi = add2(phi, pk(a.w));
    return;
  }
  const p2 dx = add2(t.x, pk(-a.x));  // d = x_t - x_s
  const p2 dy = add2(t.y, pk(-a.y));
  const p2 dz = add2(t.z, pk(-a.z));
  p2 r2 = mul2(dx, dx);
  r2 = fma2(dy, dy, r2);
  r2 = fma2(dz, dz, r2);
  if (KERNEL == PI_K_GAUSSIAN) {
    const p2 arg = mul2(r2, pk(mc2));
    const float k0 = (lo(r2) < thr) ? ex2_approx(lo(arg)) : 0.f;
    const float k1 = (hi(r2) < thr) ? ex2_approx(hi(arg)) : 0.f;
    const p2 w = mul2(pk(k0, k1), pk(a.w));
    phi = add2(phi, w);
    fx = fma2(w, dx, fx);
    fy = fma2(w, dy, fy);
    fz = fma2(w, dz, fz);
  } else if (kern_lj(KERNEL)) {
    p2 w, wf;
    lj_core<KERNEL>(r2, pk(a.w), thr, kp, w, wf);
    phi = add2(phi, w);
    fx = fma2(wf, dx, fx);
    fy = fma2(wf, dy, fy);
    fz = fma2(wf, dz, fz);
  } else if (KERNEL == PI_K_LOWFLOP) {  // selects (an inert partner is at 1e30)
    const bool i0 = lo(r2) < thr, i1 = hi(r2) < thr;
    const float sm = lf_sum(a.x, a.y, a.z);
    phi = add2(phi, pk(i0 ? sm : 0.f, i1 ? sm : 0.f));
    fx = add2(fx, pk(i0 ? a.x : 0.f, i1 ? a.x : 0.f));
    fy = add2(fy, pk(i0 ? a.y : 0.f, i1 ? a.y : 0.f));
    fz = add2(fz, pk(i0 ? a.z : 0.f, i1 ? a.z : 0.f));
  } else {
    phi = add2(phi, pk((lo(r2) < thr) ? a.w : 0.f, (hi(r2) < thr) ? a.w : 0.f));
  }
}

// The exact phi term added for target half h against itself (d = 0: no force term).
template <int KERNEL>
__device__ __forceinline__ float tp_self(const TgtPair &t, int h, const float4 a, const float thr, const float mc2,
                                         const KParams &kp) {
  if (KERNEL == PI_K_CANDIDATE) return a.w;
  if (KERNEL == PI_K_LOWFLOP) return lf_sum(a.x, a.y, a.z);
  if (kern_lj(KERNEL)) {  // the same lj_core operations as tp_eval, this half
    const p2 dx = add2(t.x, pk(-a.x));
    const p2 dy = add2(t.y, pk(-a.y));
    const p2 dz = add2(t.z, pk(-a.z));
    p2 r2 = mul2(dx, dx);
    r2 = fma2(dy, dy, r2);
    r2 = fma2(dz, dz, r2);
    p2 w, wf;
    lj_core<KERNEL>(r2, pk(a.w), thr, kp, w, wf);
    return h ? hi(w) : lo(w);
  }
  const p2 dx = add2(t.x, pk(-a.x));
  const p2 dy = add2(t.y, pk(-a.y));
  const p2 dz = add2(t.z, pk(-a.z));
  p2 r2 = mul2(dx, dx);
  r2 = fma2(dy, dy, r2);
  r2 = fma2(dz, dz, r2);
  const p2 arg = mul2(r2, pk(mc2));
  const float rr = h ? hi(r2) : lo(r2), ar = h ? hi(arg) : lo(arg);
  if (KERNEL == PI_K_GAUSSIAN) return (rr < thr) ? __fmul_rn(ex2_approx(ar), a.w) : 0.f;
  return (rr < thr) ? a.w : 0.f;
}

// Record s of the sorted state: from the records, or (rec == NULL) from the f32x2 pair array
// A[k] = (x_2k, x_2k+1, y_2k, y_2k+1) = pairs[k], B[k] = (z.., z.., q.., q..) = pairs[plane + k].
__device__ __forceinline__ float4 sorted_rec(const float4 *__restrict__ rec, const float4 *__restrict__ pairs,
                                             long long plane, int s) {
  if (rec) return __ldg(rec + s);
  const float4 a = __ldg(pairs + (s >> 1)), b = __ldg(pairs + plane + (s >> 1));
  return (s & 1) ? make_float4(a.y, a.w, b.y, b.w) : make_float4(a.x, a.z, b.x, b.z);
}

}  // namespace pi
