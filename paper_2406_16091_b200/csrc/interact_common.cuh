// Shared pieces of the shared-memory interaction kernels (a6.2 full load, a6.3 X-pencil).
//
// Both kernels end up with the same compute core: a warp owns one target cell, and the
// candidates of that cell are ONE contiguous window of staged sources in shared memory
// (the "merged pencil" layout below).  Lanes split the (target x source) work as
// (pair of targets) x (source stride group); each lane evaluates 2 candidates per
// source with packed-fp32 (FFMA2/FADD2, f32x2) instructions:
//
//   coordinates are frame-local and scaled by s = sqrt(c2), c2 = log2(e) / (2 sigma^2)
//   source s (staged once per block):  A = (x_s, y_s, z_s, H_s = y_s^2 + z_s^2)
//                                      B = (q_s, q_s x_s, q_s y_s, q_s z_s)
//   target t (registers):  x_t, Y_t = -2 y_t, Z_t = -2 z_t, T_t = y_t^2 + z_t^2
//   v   = (x_t - x_s)^2 + H_s + Y_t y_s + Z_t z_s      ( = c2 r^2 - T_t )
//   in  = v < c2 r_c^2 - T_t                           ( r^2 < r_c^2, strict; PAPER.md:50 )
//   K'  = in ? 2^(-v) : 0                              ( K = 2^(-c2 r^2) = K' 2^(-T_t) )
//   phi' += q_s K';  S_x += (q_s x_s) K';  S_y += (q_s y_s) K';  S_z += (q_s z_s) K'
//   phi_t = 2^(-T_t) phi',  F_t = (q_t / sigma^2) 2^(-T_t) / s (x_t phi' - S_x, ...)
//
// The frame is per block: X relative to the left edge of the first staged cell (x_t - x_s
// is then exact for dyadic widths), Y and Z relative to the centre of the target row, so
// |y|, |z| <= 1.5 w and the rounding of v stays far below the ambiguity band of the oracle
// (DESIGN.md "Arithmetic of the staged kernels").
//
// Self-exclusion (Alg. 1 :127, identity): the self pair IS evaluated inside the window; the
// lane that evaluated it recomputes the identical rounded products and subtracts them, so
// an isolated particle comes out exactly 0 and otherwise the error is ~1 ulp of the sum.
#pragma once
#include "pi_internal.cuh"

namespace pi {

// Packed fp32 (f32x2) helpers on 64-bit registers: ptxas keeps each value in an aligned
// register pair and turns a {s, s} operand into a scalar broadcast (FFMA2 R, R.F32x2, S.F32).
typedef unsigned long long p2;
__device__ __forceinline__ p2 pk(float a, float b) {
  p2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ p2 pk(float a) { return pk(a, a); }
__device__ __forceinline__ float lo(p2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi(p2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ p2 fma2(p2 a, p2 b, p2 c) {
  p2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ p2 add2(p2 a, p2 b) {
  p2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Staged source record, frame-local and scaled by s = sqrt(c2) (c2 = log2(e)/(2 sigma^2)):
//   A = (x~, y~, z~, H~ = y~^2 + z~^2),  B = (q, q x~, q y~, q z~)
// Target constants (per half of the pair):
//   xt = x~_t, Yt = -2 y~_t, Zt = -2 z~_t, thr = c2 r_c^2 - T~_t  with T~_t = y~_t^2 + z~_t^2
// v~ = (x~_t - x~_s)^2 + H~_s + Yt y~_s + Zt z~_s = c2 r^2 - T~_t, inside <=> v~ < thr,
// K = 2^(-c2 r^2) = 2^(-v~) * 2^(-T~_t): the per-target factor E_t = 2^(-T~_t) is applied
// once after the loop, so the inner loop needs no exponent FMA (MUFU.EX2 takes -v~).
struct TargetPair {
  p2 xt, Yt, Zt;
  float thr0, thr1;
};

template <int KERNEL>
__device__ __forceinline__ void pair_eval(const TargetPair &tp, const float4 a, const float4 b, p2 &phi, p2 &sx,
                                          p2 &sy, p2 &sz) {
  p2 dx = add2(tp.xt, pk(-a.x));
  p2 v = fma2(dx, dx, pk(a.w));
  v = fma2(tp.Yt, pk(a.y), v);
  v = fma2(tp.Zt, pk(a.z), v);
  float k0, k1;
  if (KERNEL == PI_K_GAUSSIAN) {
    k0 = (lo(v) < tp.thr0) ? ex2_approx(-lo(v)) : 0.f;
    k1 = (hi(v) < tp.thr1) ? ex2_approx(-hi(v)) : 0.f;
  } else if (KERNEL == PI_K_INDICATOR) {
    k0 = (lo(v) < tp.thr0) ? 1.f : 0.f;
    k1 = (hi(v) < tp.thr1) ? 1.f : 0.f;
  } else {
    k0 = k1 = 1.f;
  }
  const p2 K = pk(k0, k1);
  phi = fma2(K, pk(b.x), phi);
  if (KERNEL == PI_K_GAUSSIAN) {
    sx = fma2(K, pk(b.y), sx);
    sy = fma2(K, pk(b.z), sy);
    sz = fma2(K, pk(b.w), sz);
  }
}

// The exact rounded contribution a lane added for (target half `h`, source (a, b)): the same
// operations as pair_eval, so subtracting them removes the self pair (identity, :127).
template <int KERNEL>
__device__ __forceinline__ void self_terms(const TargetPair &tp, int h, const float4 a, const float4 b, float &p,
                                           float &x, float &y, float &z) {
  p2 dx = add2(tp.xt, pk(-a.x));
  p2 v = fma2(dx, dx, pk(a.w));
  v = fma2(tp.Yt, pk(a.y), v);
  v = fma2(tp.Zt, pk(a.z), v);
  const float vv = h ? hi(v) : lo(v);
  const float thr = h ? tp.thr1 : tp.thr0;
  float K;
  if (KERNEL == PI_K_GAUSSIAN) K = (vv < thr) ? ex2_approx(-vv) : 0.f;
  else if (KERNEL == PI_K_INDICATOR) K = (vv < thr) ? 1.f : 0.f;
  else K = 1.f;
  // fma(K, b, 0) rounds exactly like the product K*b
  p = __fmul_rn(K, b.x);
  x = __fmul_rn(K, b.y);
  y = __fmul_rn(K, b.z);
  z = __fmul_rn(K, b.w);
}

// Staging transform (once per staged particle and block).
__device__ __forceinline__ void stage_record(const float4 v, float fxo, float fyo, float fzo, float s, float4 &A,
                                             float4 &B) {
  const float xl = (v.x - fxo) * s, yl = (v.y - fyo) * s, zl = (v.z - fzo) * s;
  A = make_float4(xl, yl, zl, fmaf(yl, yl, zl * zl));
  B = make_float4(v.w, v.w * xl, v.w * yl, v.w * zl);
}

// Warp computes all targets of one staged cell against its contiguous candidate window
// [W0, W1) of the staged arrays (A, B).  Targets are the `nt` staged particles starting at
// `home` (they are part of the window).  Results go through write_output at global sorted
// slots gslot0 + t.  `red` is a per-warp scratch of 32 * 8 floats.
template <int KERNEL>
__device__ void warp_cell(const float4 *__restrict__ A, const float4 *__restrict__ B, int home, int nt, int W0,
                          int W1, int gslot0, float s_inv, const float4 *__restrict__ rec, const Geom &g,
                          const KParams &kp, const OutDesc &out, float *red, unsigned long long &cand) {
  const int lane = threadIdx.x & 31;
  const float thr_base = kp.c2 * kp.rc2;
  cand += (unsigned long long)nt * (unsigned long long)(W1 - W0 - 1);
  for (int c0 = 0; c0 < nt; c0 += 64) {
    const int ntc = min(64, nt - c0);
    const int S = (ntc + 1) >> 1;
    const int G = 32 / S;
    const int slot = lane % S;
    const int grp = lane / S;
    const bool act = grp < G;
    const int t0 = c0 + 2 * slot;
    const int t1 = min(t0 + 1, c0 + ntc - 1);
    const float4 a0 = A[home + t0], a1 = A[home + t1];
    TargetPair tp;
    // build the packed constants with real f32x2 ops so ptxas gives each an aligned pair
    tp.xt = add2(pk(a0.x, a1.x), pk(0.f));
    tp.Yt = fma2(pk(a0.y, a1.y), pk(-2.f), pk(0.f));
    tp.Zt = fma2(pk(a0.z, a1.z), pk(-2.f), pk(0.f));
    tp.thr0 = thr_base - a0.w;
    tp.thr1 = thr_base - a1.w;
    p2 phi = pk(0.f), sx = pk(0.f), sy = pk(0.f), sz = pk(0.f);
    // each source group takes a contiguous chunk of the window; an odd chunk length puts
    // the G concurrent 16-B loads of a warp in distinct banks (G <= 8)
    int chunk = (W1 - W0 + G - 1) / G;
    chunk |= 1;
    if (act) {
      const int s0 = W0 + grp * chunk;
      const int s1 = min(s0 + chunk, W1);
      const float4 *pa = A + s0;
      const float4 *pb = B + s0;
      const float4 *pe4 = A + s0 + (max(s1 - s0, 0) & ~3);
      const float4 *pe = A + max(s1, s0);
      for (; pa < pe4; pa += 4, pb += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) pair_eval<KERNEL>(tp, pa[u], pb[u], phi, sx, sy, sz);
      }
      for (; pa < pe; ++pa, ++pb) pair_eval<KERNEL>(tp, *pa, *pb, phi, sx, sy, sz);
      // identity exclusion: subtract exactly what this lane added for its own targets
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ts = h ? t1 : t0;
        const int ss = home + ts;
        if ((ss - W0) / chunk == grp && !(h == 1 && t1 == t0)) {
          float p, x, y, z;
          self_terms<KERNEL>(tp, h, A[ss], B[ss], p, x, y, z);
          if (h) {
            phi = pk(lo(phi), hi(phi) - p); sx = pk(lo(sx), hi(sx) - x);
            sy = pk(lo(sy), hi(sy) - y); sz = pk(lo(sz), hi(sz) - z);
          } else {
            phi = pk(lo(phi) - p, hi(phi)); sx = pk(lo(sx) - x, hi(sx));
            sy = pk(lo(sy) - y, hi(sy)); sz = pk(lo(sz) - z, hi(sz));
          }
        }
      }
    }
    // reduce over the G source groups through the warp scratch
    __syncwarp();
    if (act) {
      float *r = red + grp * (8 * S) + slot * 8;
      reinterpret_cast<float4 *>(r)[0] = make_float4(lo(phi), hi(phi), lo(sx), hi(sx));
      reinterpret_cast<float4 *>(r)[1] = make_float4(lo(sy), hi(sy), lo(sz), hi(sz));
    }
    __syncwarp();
    for (int idx = lane; idx < 8 * S; idx += 32) {
      float acc = red[idx];
      for (int gg = 1; gg < G; ++gg) acc += red[gg * 8 * S + idx];
      red[idx] = acc;
    }
    __syncwarp();
    for (int t = lane; t < ntc; t += 32) {
      const int sl = t >> 1, h = t & 1;
      const float *r = red + sl * 8;
      float ph = r[0 + h];
      float fx = 0.f, fy = 0.f, fz = 0.f;
      if (KERNEL == PI_K_GAUSSIAN) {
        const float4 at = A[home + c0 + t];
        const float4 bt = B[home + c0 + t];
        const float E = ex2_approx(-at.w);  // 2^(-T~_t)
        ph *= E;
        const float sc = bt.x * kp.inv_s2 * s_inv * E;
        fx = sc * fmaf(at.x, r[0 + h], -r[2 + h]);
        fy = sc * fmaf(at.y, r[0 + h], -r[4 + h]);
        fz = sc * fmaf(at.z, r[0 + h], -r[6 + h]);
      }
      const int gs = gslot0 + c0 + t;
      float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
      if (out.upd) me = __ldg(rec + gs);
      write_output(out, g, gs, me, ph, fx, fy, fz);
    }
    __syncwarp();
  }
}

// Fallback for a target cell whose candidate window does not fit the staging buffer:
// Par-Part-NoLoop over global memory, one thread per target, the whole block.
template <int KERNEL>
__device__ void block_fallback_cell(int cx, int cy, int cz, const float4 *__restrict__ rec,
                                    const int32_t *__restrict__ offsets, const Geom &g, const KParams &kp,
                                    const OutDesc &out, unsigned long long &cand) {
  const long long home_row = (long long)g.nx * (cy + (long long)g.ny * cz);
  const int t_lo = __ldg(offsets + home_row + cx), t_hi = __ldg(offsets + home_row + cx + 1);
  const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.nx - 1);
  for (int t = t_lo + threadIdx.x; t < t_hi; t += blockDim.x) {
    const float4 me = __ldg(rec + t);
    float phi = 0.f, fx = 0.f, fy = 0.f, fz = 0.f;
    for (int dz = -1; dz <= 1; ++dz) {
      const int z = cz + dz;
      if (z < 0 || z >= g.nz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int y = cy + dy;
        if (y < 0 || y >= g.ny) continue;
        const long long row = (long long)g.nx * (y + (long long)g.ny * z);
        const int lo = __ldg(offsets + row + xlo), hi = __ldg(offsets + row + xhi + 1);
        cand += (unsigned long long)(hi - lo);
        for (int s = lo; s < hi; ++s) {
          if (s == t) continue;
          const float4 o = __ldg(rec + s);
          const float dx = me.x - o.x, dy2 = me.y - o.y, dz2 = me.z - o.z;
          const float r2 = fmaf(dz2, dz2, fmaf(dy2, dy2, dx * dx));
          if (KERNEL == PI_K_CANDIDATE) {
            phi += o.w;
          } else if (r2 < kp.rc2) {
            if (KERNEL == PI_K_INDICATOR) {
              phi += o.w;
            } else {
              const float w = o.w * ex2_approx(-kp.c2 * r2);
              phi += w;
              fx = fmaf(w, dx, fx);
              fy = fmaf(w, dy2, fy);
              fz = fmaf(w, dz2, fz);
            }
          }
        }
      }
    }
    cand -= 1;
    if (KERNEL == PI_K_GAUSSIAN) {
      const float s = me.w * kp.inv_s2;
      fx *= s; fy *= s; fz *= s;
    } else {
      fx = fy = fz = 0.f;
    }
    write_output(out, g, t, me, phi, fx, fy, fz);
  }
}

}  // namespace pi
