/* ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain C fp64 cell-list oracle for the interactions of arXiv 2406.16091.
 * It computes exactly the definition of PAPER.md:49-51 (§2): for every target i,
 * the sum over j != i with r_ij < r_c of the kernel contributions, using the grid
 * only to enumerate the candidates (§2, cell width >= r_c :93 §3,
 * 27 neighbour cells :236 §5.1).  Nothing is blocked, fused or reordered beyond
 * "loop over the 27 clamped neighbour cells, loop over their particles".
 *
 * Cell index: contract C3 of DESIGN.md, fp32 with one rounding per operation
 * (compile without FMA contraction: -ffp-contract=off).
 * Binning: a sequential counting sort (counts, exclusive prefix, placement).
 * Kernels: 0 Gaussian K = exp(-r^2/(2 sigma^2)),
 *            c_ij = (q_j K, q_i q_j K (x_i - x_j)/sigma^2, ...)
 *          1 INDICATOR c_ij = (q_j, 0, 0, 0) inside the cutoff
 *          2 CANDIDATE c_ij = (q_j, 0, 0, 0) for every candidate pair
 *          3 Lennard-Jones, Eq. (1) with softening (reading R19)
 *          4 LOWFLOP  c_ij = (x_j + y_j + z_j, x_j, y_j, z_j) inside the cutoff ("summing the
 *                     positions", reading R22)
 *          5 HIGHFLOP Lennard-Jones whose potential term u goes through 75 steps t <- t a + b,
 *                     a = 1 - 2^-7, b = 2^-10, before q_j 4 E0 t ("150 added FLOP")
 * Outputs per requested target t: out[4] (phi, fx, fy, fz), S[4] = sum |c_ij| over
 * included pairs (Lennard-Jones: per Eq. (1) term, reading R20), A[4] = sum |c_ij| over ambiguous pairs (|r^2 - rc^2| <= band rc^2),
 * C = #candidates, P = #pairs inside the cutoff.  All accumulation in double.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* a1: cell coordinates, contract C3. */
static inline void cell3(float x, float y, float z, const float o[3], float inv_w, const int32_t d[3],
                         int64_t c[3]) {
  float v[3] = {x, y, z};
  for (int a = 0; a < 3; ++a) {
    volatile float t = v[a] - o[a]; /* one rounding */
    volatile float s = t * inv_w;   /* one rounding */
    c[a] = clampi((int64_t)floor((double)s), 0, d[a] - 1);
  }
}

int oracle_cells(int64_t n, const float *x, const float *y, const float *z, const float o[3], float inv_w,
                 const int32_t d[3], int64_t *cell_out) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t c[3];
    cell3(x[i], y[i], z[i], o, inv_w, d, c);
    cell_out[i] = c[0] + (int64_t)d[0] * (c[1] + (int64_t)d[1] * c[2]);
  }
  return 0;
}

/* a2-a4: counts, exclusive prefix (offsets[Nc] = n), out-of-place placement. */
int oracle_bin(int64_t n, const int64_t *cell, int64_t ncells, int64_t *counts, int64_t *offsets, int64_t *order) {
  memset(counts, 0, sizeof(int64_t) * ncells);
  for (int64_t i = 0; i < n; ++i) counts[cell[i]]++;
  offsets[0] = 0;
  for (int64_t c = 0; c < ncells; ++c) offsets[c + 1] = offsets[c] + counts[c];
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (ncells > 0 ? ncells : 1));
  for (int64_t c = 0; c < ncells; ++c) cur[c] = offsets[c];
  for (int64_t i = 0; i < n; ++i) order[cur[cell[i]]++] = i;
  free(cur);
  return 0;
}

int oracle_interact(int64_t n, const float *x, const float *y, const float *z, const float *q, const float o[3],
                    float inv_w, const int32_t d[3], double rc, const double kp[4], int kernel, double band,
                    int64_t nt, const int64_t *targets, double *out, double *S, double *A, int64_t *C,
                    int64_t *P) {
  int64_t ncells = (int64_t)d[0] * d[1] * d[2];
  int64_t *cell = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int64_t *counts = (int64_t *)malloc(sizeof(int64_t) * ncells);
  int64_t *offsets = (int64_t *)malloc(sizeof(int64_t) * (ncells + 1));
  int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  if (!cell || !counts || !offsets || !order) return 1;
  oracle_cells(n, x, y, z, o, inv_w, d, cell);
  oracle_bin(n, cell, ncells, counts, offsets, order);
  /* kp: Gaussian sigma; Lennard-Jones r, eps, E0 (Eq. (1), reading R19) */
  const double sigma = kp[0], ljr = kp[1], ljeps = kp[2], lje0 = kp[3];
  const double rc2 = rc * rc, s2 = sigma * sigma, inv2s2 = 1.0 / (2.0 * sigma * sigma);
  if (nt < 0) nt = n;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t k = 0; k < nt; ++k) {
    int64_t i = targets ? targets[k] : k;
    int64_t ci[3];
    cell3(x[i], y[i], z[i], o, inv_w, d, ci);
    double xi = x[i], yi = y[i], zi = z[i], qi = q[i];
    double acc[4] = {0, 0, 0, 0}, sab[4] = {0, 0, 0, 0}, amb[4] = {0, 0, 0, 0};
    int64_t cc = 0, pp = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int64_t a = ci[0] + dx, b = ci[1] + dy, c = ci[2] + dz;
          if (a < 0 || a >= d[0] || b < 0 || b >= d[1] || c < 0 || c >= d[2]) continue;
          int64_t cl = a + (int64_t)d[0] * (b + (int64_t)d[1] * c);
          for (int64_t s = offsets[cl]; s < offsets[cl + 1]; ++s) {
            int64_t j = order[s];
            if (j == i) continue; /* identity, Alg. 1 */
            ++cc;
            double ddx = xi - (double)x[j], ddy = yi - (double)y[j], ddz = zi - (double)z[j];
            double r2 = ddx * ddx + ddy * ddy + ddz * ddz;
            int inside = r2 < rc2;
            int ambiguous = fabs(r2 - rc2) <= band * rc2;
            double cij[4], mag[4];
            if (kernel == 0) {
              double K = exp(-r2 * inv2s2);
              double w = (double)q[j] * K;
              cij[0] = w;
              cij[1] = qi * w * ddx / s2;
              cij[2] = qi * w * ddy / s2;
              cij[3] = qi * w * ddz / s2;
            } else if (kernel == 4) {
              double px = (double)x[j], py = (double)y[j], pz = (double)z[j];
              cij[0] = px + py + pz;
              cij[1] = px; cij[2] = py; cij[3] = pz;
              mag[0] = fabs(px) + fabs(py) + fabs(pz);
              mag[1] = fabs(px); mag[2] = fabs(py); mag[3] = fabs(pz);
            } else if (kernel == 3 || kernel == 5) {
              /* d~^2 = d^2 + eps^2, s = (d~ / r)^2: K = 4 E0 (s^6 - s^3),
                 force on i = -q_i q_j dK/dd~ (x_i - x_j) / d~ = q_i q_j G (x_i - x_j) */
              double s = (r2 + ljeps * ljeps) / (ljr * ljr);
              double s3 = s * s * s;
              double K = 4.0 * lje0 * (s3 * s3 - s3);
              double chainA = 1.0, chainB = 0.0;  /* kernel 5: the chain's |terms| (A, B) */
              if (kernel == 5) {
                double t = s3 * s3 - s3;
                for (int st = 0; st < 75; ++st) {
                  t = t * (1.0 - 0x1p-7) + 0x1p-10;
                  chainA *= (1.0 - 0x1p-7);
                  chainB = chainB * (1.0 - 0x1p-7) + 0x1p-10;
                }
                K = 4.0 * lje0 * t;
              }
              double G = -(4.0 * lje0 / (ljr * ljr)) * (12.0 * s3 * s * s - 6.0 * s * s);
              double w = (double)q[j];
              cij[0] = w * K;
              cij[1] = qi * w * G * ddx;
              cij[2] = qi * w * G * ddy;
              cij[3] = qi * w * G * ddz;
              /* |c_ij| per Eq. (1) term (reading R20): repulsive and attractive
                 parts counted separately, so the tolerance does not vanish where they cancel */
              double Km = 4.0 * lje0 * (chainA * (s3 * s3 + s3) + chainB);
              double Gm = (4.0 * lje0 / (ljr * ljr)) * (12.0 * s3 * s * s + 6.0 * s * s);
              mag[0] = fabs(w) * Km;
              mag[1] = fabs(qi * w) * Gm * fabs(ddx);
              mag[2] = fabs(qi * w) * Gm * fabs(ddy);
              mag[3] = fabs(qi * w) * Gm * fabs(ddz);
            } else {
              cij[0] = (double)q[j];
              cij[1] = cij[2] = cij[3] = 0.0;
            }
            if (kernel != 3 && kernel != 4 && kernel != 5)
              for (int m = 0; m < 4; ++m) mag[m] = fabs(cij[m]);
            if (kernel == 2) { inside = 1; ambiguous = 0; }
            if (inside) {
              ++pp;
              for (int m = 0; m < 4; ++m) { acc[m] += cij[m]; sab[m] += mag[m]; }
            }
            if (ambiguous)
              for (int m = 0; m < 4; ++m) amb[m] += mag[m];
          }
        }
    for (int m = 0; m < 4; ++m) { out[4 * k + m] = acc[m]; S[4 * k + m] = sab[m]; A[4 * k + m] = amb[m]; }
    C[k] = cc;
    P[k] = (kernel == 2) ? 0 : pp;
  }
  free(cell); free(counts); free(offsets); free(order);
  return 0;
}
