/*
 * wb_oracle.c -- plain-C restatement of the reference hot path (TEST ORACLE).
 *
 * Test infrastructure only (see wb_oracle.h).  Follows
 * /root/reference/pkg/src/wbflow/kernels.py operation by operation; every
 * floating-point expression keeps the reference's association order so that
 * a build with -ffp-contract=off reproduces the Numba results bit for bit.
 * Column loops are OpenMP-parallel (the reference's prange, kernels.py:506,
 * 1031, 1239); every output element is written by exactly one iteration, so
 * results do not depend on the thread count (timestepper.py:27-30).
 */
#include "wb_oracle.h"
#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BC_REFL 1
#define BC_TRANS 2
#define BC_INFLOW 3
#define SONIC_GUARD 1.0e-8

#define AT(i, j, m) ((((size_t)(i)) * ny + (j)) * 5 + (m))
#define AT2(i, j) (((size_t)(i)) * ny + (j))

int wbo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void wbo_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n < 1 ? 1 : n);
#else
  (void)n;
#endif
}

/* kernels.py:13-22 -- the constants are computed exactly as numpy does */
static double GLN[3], GLW[3];
static const double ORW[3] = {4.0 / 3.0, 4.0 / 3.0, -1.0 / 3.0};
static int consts_ready = 0;
static void init_consts(void) {
  if (consts_ready) return;
  double s = sqrt(15.0) / 10.0;
  GLN[0] = 0.5 - s; GLN[1] = 0.5; GLN[2] = 0.5 + s;
  GLW[0] = 5.0 / 18.0; GLW[1] = 8.0 / 18.0; GLW[2] = 5.0 / 18.0;
  consts_ready = 1;
}

/* Python min/max as Numba lowers them (builtins.do_minmax): select(v<acc, v, acc) */
static inline double pmin(double a, double b) { return (b < a) ? b : a; }
static inline double pmax(double a, double b) { return (b > a) ? b : a; }

/* kernels.py:38-43 */
double wbo_tait_p(double rho, double k0, double rho0, double gamma) {
  double ratio = rho / rho0;
  if (gamma == 1.0) return k0 * (ratio - 1.0);
  return k0 * (pow(ratio, gamma) - 1.0);
}
/* kernels.py:46-50 */
double wbo_sound_c2(double rho, double k0, double rho0, double gamma) {
  if (gamma == 1.0) return k0 / rho0;
  return gamma * k0 / rho0 * pow(rho / rho0, gamma - 1.0);
}
/* kernels.py:53-55 */
double wbo_eq_rho(double y, double y0, double k0, double rho0, double g) {
  return rho0 * exp(-(g * rho0 / k0) * (y - y0));
}
/* kernels.py:58-64 */
static inline double sgn(double z) {
  if (z > 0.0) return 1.0;
  if (z < 0.0) return -1.0;
  return 0.0;
}
/* kernels.py:67-71 */
static inline double guarded(double z, double fl) {
  if (fabs(z) < fl) return z >= 0.0 ? fl : -fl;
  return z;
}
/* kernels.py:78-82 (components 3, 4 are 0) */
static inline void flux_x(const double *q, double k0, double rho0, double gamma, double *f) {
  double u = q[1] / q[0];
  double p = wbo_tait_p(q[0] / q[3], k0, rho0, gamma);
  f[0] = q[1];
  f[1] = q[1] * u + q[3] * p;
  f[2] = q[2] * u;
}
/* kernels.py:85-88 */
static inline void flux_y(const double *q, double *f) {
  double v = q[2] / q[0];
  f[0] = q[2];
  f[1] = q[1] * v;
  f[2] = q[2] * v;
}

/* kernels.py:102-119 */
static void abs_a1(double u, double v, double c, double rcp, const double *x, double *y) {
  double c2 = c * c;
  double w1 = 0.5 * (c + u) / c * x[0] - 0.5 / c * x[1] - 0.5 * rcp / c2 * x[3];
  double w2 = -v * x[0] + x[2] + v * rcp / c2 * x[3];
  double w3 = x[3] / c2;
  double w5 = 0.5 * (c - u) / c * x[0] + 0.5 / c * x[1] - 0.5 * rcp / c2 * x[3];
  double au = fabs(u);
  w1 *= fabs(u - c);
  w2 *= au;
  w3 *= au;
  w5 *= fabs(u + c);
  y[0] = w1 + rcp * w3 + w5;
  y[1] = (u - c) * w1 + u * rcp * w3 + (u + c) * w5;
  y[2] = v * w1 + w2 + v * w5;
  y[3] = c2 * w3;
  y[4] = 0.0;
}

/* kernels.py:166-187 */
static void sign_a2(double u, double v, double c, double rcp, double arg, const double *x,
                    double *y) {
  double c2 = c * c;
  double cmv = guarded(c - v, SONIC_GUARD * c);
  double cpv = guarded(c + v, SONIC_GUARD * c);
  double w1 = 0.5 * (c + v) / c * x[0] - 0.5 / c * x[2] - 0.5 * rcp / c2 * x[3] +
              0.5 / c * arg / cmv * x[4];
  double w2 = -u * x[0] + x[1] + u * rcp / c2 * x[3];
  double w3 = x[3] / c2;
  double w5 = 0.5 * (c - v) / c * x[0] + 0.5 / c * x[2] - 0.5 * rcp / c2 * x[3] +
              0.5 / c * arg / cpv * x[4];
  double sv = sgn(v);
  w1 *= sgn(v - c);
  w2 *= sv;
  w3 *= sv;
  w5 *= sgn(v + c);
  y[0] = w1 + rcp * w3 + w5;
  y[1] = u * w1 + w2 + u * w5;
  y[2] = (v - c) * w1 + v * rcp * w3 + (v + c) * w5;
  y[3] = c2 * w3;
  y[4] = 0.0;
}

/* kernels.py:215-271 */
void wbo_osher_x_edge(const double *qm, const double *qp, double k0, double rho0,
                      double gamma, double *o) {
  init_consts();
  if (qm[0] == qp[0] && qm[1] == qp[1] && qm[2] == qp[2] && qm[3] == qp[3] &&
      qm[4] == qp[4]) {
    for (int m = 0; m < 10; m++) o[m] = 0.0;
    return;
  }
  double d[5];
  for (int m = 0; m < 5; m++) d[m] = qp[m] - qm[m];
  double fm[3], fp[3];
  flux_x(qm, k0, rho0, gamma, fm);
  flux_x(qp, k0, rho0, gamma, fp);
  double ubar = 0.0, V[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < 3; k++) {
    double s = GLN[k], w = GLW[k];
    double p0 = qm[0] + s * d[0];
    double p1 = qm[1] + s * d[1];
    double p2 = qm[2] + s * d[2];
    double p3 = qm[3] + s * d[3];
    double rho = p0 / p3;
    double u = p1 / p0;
    double v = p2 / p0;
    double p = wbo_tait_p(rho, k0, rho0, gamma);
    double c2 = wbo_sound_c2(rho, k0, rho0, gamma);
    double c = sqrt(c2);
    double rcp = rho * c2 - p;
    ubar += w * u;
    double t[5];
    abs_a1(u, v, c, rcp, d, t);
    for (int m = 0; m < 5; m++) V[m] += w * t[m];
  }
  double b3 = ubar * d[3];
  double j[5];
  j[0] = fp[0] - fm[0];
  j[1] = fp[1] - fm[1];
  j[2] = fp[2] - fm[2];
  j[3] = 0.0 - 0.0 + b3; /* fp3 - fm3 + b3 with flux components 3 = 0 */
  j[4] = 0.0 - 0.0;
  for (int m = 0; m < 5; m++) {
    o[m] = 0.5 * (j[m] - V[m]);
    o[5 + m] = 0.5 * (j[m] + V[m]);
  }
}

/* kernels.py:278-287 -> d[0..9] = (y, alpha, rho, p, v, rhoE, pE, alpha_f, rho_f, p_f) */
static void decomp_y(double q0, double q2, double q3, double q4, double rE, double aeq,
                     double k0, double rho0, double gamma, double *d) {
  double rho = q0 / q3;
  double p = wbo_tait_p(rho, k0, rho0, gamma);
  double pE = wbo_tait_p(rE, k0, rho0, gamma);
  d[0] = q4; d[1] = q3; d[2] = rho; d[3] = p; d[4] = q2 / q0;
  d[5] = rE; d[6] = pE; d[7] = q3 - aeq; d[8] = rho - rE; d[9] = p - pE;
}
/* kernels.py:290-305 */
static void b_pair_y(const double *da, const double *db, double vmid, double aeq, double g,
                     double *b3, double *b4) {
  *b3 = aeq * (db[9] - da[9]) + (db[7] * db[6] - da[7] * da[6]) +
        (db[7] * db[9] - da[7] * da[9]) +
        (aeq * (0.5 * (da[8] + db[8])) + 0.5 * (da[7] + db[7]) * (0.5 * (da[5] + db[5])) +
         0.5 * (da[7] + db[7]) * (0.5 * (da[8] + db[8]))) *
            g * (db[0] - da[0]);
  *b4 = vmid * (db[1] - da[1]);
}

/* kernels.py:308-425 */
void wbo_or_y_edge(const double *qm, const double *qp, double y0, double aeq, double k0,
                   double rho0, double gamma, double g, double *o) {
  if (qm[0] == qp[0] && qm[1] == qp[1] && qm[2] == qp[2] && qm[3] == qp[3] &&
      qm[4] == qp[4]) {
    for (int m = 0; m < 10; m++) o[m] = 0.0;
    return;
  }
  double ym = qm[4], yp = qp[4];
  int same_h = (yp == ym);
  double rEm = wbo_eq_rho(ym, y0, k0, rho0, g);
  double rEp = same_h ? rEm : wbo_eq_rho(yp, y0, k0, rho0, g);
  double fm0 = qm[0] - aeq * rEm, fm1 = qm[1], fm2 = qm[2], fm3 = qm[3] - aeq;
  double fp0 = qp[0] - aeq * rEp, fp1 = qp[1], fp2 = qp[2], fp3 = qp[3] - aeq;
  double ya = ym + 0.25 * (yp - ym);
  double yh = ym + 0.5 * (yp - ym);
  double yb = ym + 0.75 * (yp - ym);
  double rEa = same_h ? rEm : wbo_eq_rho(ya, y0, k0, rho0, g);
  double rEh = same_h ? rEm : wbo_eq_rho(yh, y0, k0, rho0, g);
  double rEb = same_h ? rEm : wbo_eq_rho(yb, y0, k0, rho0, g);
  (void)ya; (void)yb;

  double xa0 = aeq * rEa + fm0 + 0.25 * (fp0 - fm0);
  double xa1 = fm1 + 0.25 * (fp1 - fm1);
  double xa2 = fm2 + 0.25 * (fp2 - fm2);
  double xa3 = aeq + fm3 + 0.25 * (fp3 - fm3);
  double xh0 = aeq * rEh + fm0 + 0.5 * (fp0 - fm0);
  double xh1 = fm1 + 0.5 * (fp1 - fm1);
  double xh2 = fm2 + 0.5 * (fp2 - fm2);
  double xh3 = aeq + fm3 + 0.5 * (fp3 - fm3);
  double xb0 = aeq * rEb + fm0 + 0.75 * (fp0 - fm0);
  double xb1 = fm1 + 0.75 * (fp1 - fm1);
  double xb2 = fm2 + 0.75 * (fp2 - fm2);
  double xb3 = aeq + fm3 + 0.75 * (fp3 - fm3);

  double d0[10], dh[10], d1[10];
  decomp_y(qm[0], qm[2], qm[3], qm[4], rEm, aeq, k0, rho0, gamma, d0);
  decomp_y(xh0, xh2, xh3, yh, rEh, aeq, k0, rho0, gamma, dh);
  decomp_y(qp[0], qp[2], qp[3], qp[4], rEp, aeq, k0, rho0, gamma, d1);

  double g0[3], gh[3], g1[3];
  double xh[5] = {xh0, xh1, xh2, xh3, yh};
  flux_y(qm, g0);
  flux_y(xh, gh);
  flux_y(qp, g1);

  double b3a, b4a, b3b, b4b, b3f, b4f;
  b_pair_y(d0, dh, xa2 / xa0, aeq, g, &b3a, &b4a);
  b_pair_y(dh, d1, xb2 / xb0, aeq, g, &b3b, &b4b);
  b_pair_y(d0, d1, xh2 / xh0, aeq, g, &b3f, &b4f);

  double R[3][5] = {
      {gh[0] - g0[0], gh[1] - g0[1], gh[2] - g0[2] + b3a, b4a, 0.0},
      {g1[0] - gh[0], g1[1] - gh[1], g1[2] - gh[2] + b3b, b4b, 0.0},
      {g1[0] - g0[0], g1[1] - g0[1], g1[2] - g0[2] + b3f, b4f, 0.0}};
  double P[3][4] = {{xa0, xa1, xa2, xa3}, {xb0, xb1, xb2, xb3}, {xh0, xh1, xh2, xh3}};
  double V[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < 3; k++) {
    double w = ORW[k];
    double rho = P[k][0] / P[k][3];
    double u = P[k][1] / P[k][0];
    double v = P[k][2] / P[k][0];
    double p = wbo_tait_p(rho, k0, rho0, gamma);
    double c2 = wbo_sound_c2(rho, k0, rho0, gamma);
    double c = sqrt(c2);
    double rcp = rho * c2 - p;
    double arg = P[k][3] * rho * g;
    double t[5];
    sign_a2(u, v, c, rcp, arg, R[k], t);
    for (int m = 0; m < 5; m++) V[m] += w * t[m];
  }
  double j[5] = {g1[0] - g0[0], g1[1] - g0[1], g1[2] - g0[2] + b3f, b4f, 0.0};
  for (int m = 0; m < 5; m++) {
    o[m] = 0.5 * (j[m] - V[m]);
    o[5 + m] = 0.5 * (j[m] + V[m]);
  }
}

/* kernels.py:432-453 */
void wbo_detect_columns(const double *q, const uint8_t *mask, int nx, int ny,
                        const double *yfaces, double dy, double *y0s, double *aeqs) {
  for (int i = 0; i < nx; i++) {
    double ssum = 0.0, ylow = yfaces[0], aeq = 1.0;
    int found = 0;
    for (int j = 0; j < ny; j++) {
      if (mask[AT2(i, j)] != 0) {
        if (!found) { ylow = yfaces[j]; aeq = q[AT(i, j, 3)]; found = 1; }
        ssum += q[AT(i, j, 3)];
      }
    }
    y0s[i] = ylow + ssum * dy;
    aeqs[i] = aeq;
  }
}

static inline int admissible(double q0, double q1, double q2, double q3) {
  return q0 > 0.0 && q3 > 0.0 && isfinite(q0) && isfinite(q1) && isfinite(q2) &&
         isfinite(q3);
}

/* kernels.py:497-546 */
void wbo_prepare_step(const wbo_cfg *c, const double *q, const uint8_t *mask,
                      const double *yfaces, const double *ycent, double *y0s,
                      double *aeqs, double *y0s_prev, double *rhoE_c,
                      double *rhoE_fy, double *col_rate, uint8_t *flags) {
  const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nx; i++) {
    double ssum = 0.0, ylow = yfaces[0], aeq = 1.0;
    int found = 0;
    for (int j = 0; j < ny; j++) {
      if (mask[AT2(i, j)] != 0) {
        if (!found) { ylow = yfaces[j]; aeq = q[AT(i, j, 3)]; found = 1; }
        ssum += q[AT(i, j, 3)];
      }
    }
    double y0 = ylow + ssum * c->dy;
    y0s[i] = y0;
    aeqs[i] = aeq;
    if (y0 != y0s_prev[i]) {
      y0s_prev[i] = y0;
      for (int j = 0; j < ny; j++)
        rhoE_c[AT2(i, j)] = wbo_eq_rho(ycent[j], y0, c->k0, c->rho0, c->g);
      for (int j = 0; j < ny + 1; j++)
        rhoE_fy[(size_t)i * (ny + 1) + j] = wbo_eq_rho(yfaces[j], y0, c->k0, c->rho0, c->g);
    }
    double colmax = 0.0;
    for (int j = 0; j < ny; j++) {
      if (mask[AT2(i, j)] == 0) continue;
      double q0 = q[AT(i, j, 0)], q1 = q[AT(i, j, 1)], q2 = q[AT(i, j, 2)],
             q3 = q[AT(i, j, 3)];
      if (!admissible(q0, q1, q2, q3)) { flags[AT2(i, j)] = 1; continue; }
      double u = q1 / q0, v = q2 / q0;
      double cc = sqrt(wbo_sound_c2(q0 / q3, c->k0, c->rho0, c->gamma));
      double r = (fabs(u) + cc) / c->dx + (fabs(v) + cc) / c->dy;
      if (r > colmax) colmax = r;
    }
    col_rate[i] = colmax;
  }
}

/* Barth-Jespersen limiter for one component, kernels.py:694-731 (pattern
 * repeated per component at 733-887). */
static inline double bj_limit(double f, double w, double e, double s, double n, double sx,
                              double sy, double hx, double hy) {
  double lo = pmin(pmin(pmin(pmin(f, w), e), s), n);
  double hi = pmax(pmax(pmax(pmax(f, w), e), s), n);
  double ps = 1.0, r, d;
  d = sx * hx;
  if (d > 0.0) {
    r = (hi - f) / d; if (r < ps) ps = r;
    r = (f - lo) / d; if (r < ps) ps = r;
  } else if (d < 0.0) {
    r = (lo - f) / d; if (r < ps) ps = r;
    r = (f - hi) / d; if (r < ps) ps = r;
  }
  d = sy * hy;
  if (d > 0.0) {
    r = (hi - f) / d; if (r < ps) ps = r;
    r = (f - lo) / d; if (r < ps) ps = r;
  } else if (d < 0.0) {
    r = (lo - f) / d; if (r < ps) ps = r;
    r = (f - hi) / d; if (r < ps) ps = r;
  }
  return ps;
}

/* kernels.py:553-1022 */
static int cell_reconstruct(const wbo_cfg *c, const double *q, const uint8_t *mask, int i,
                            int j, const double *aeqs, const double *rhoE_c,
                            const double *rhoE_fy, const double *ycent,
                            const double *yfaces, double dt_half, double *fW, double *fE,
                            double *fS, double *fN, double *vol, double *psi,
                            uint8_t *quiet) {
  const int nx = c->nx, ny = c->ny;
  const double dx = c->dx, dy = c->dy, k0 = c->k0, rho0 = c->rho0, gamma = c->gamma,
               g = c->g;
  double aeq = aeqs[i];
  double qc[5];
  for (int m = 0; m < 5; m++) qc[m] = q[AT(i, j, m)];
  double f[5] = {qc[0] - aeq * rhoE_c[AT2(i, j)], qc[1], qc[2], qc[3] - aeq,
                 qc[4] - ycent[j]};
  double W[5], E[5], S[5], N[5];
  double alw, ale, als, aln;
  if (i > 0 && mask[AT2(i - 1, j)] != 0) {
    double an = aeqs[i - 1];
    alw = q[AT(i - 1, j, 3)];
    W[0] = q[AT(i - 1, j, 0)] - an * rhoE_c[AT2(i - 1, j)];
    W[1] = q[AT(i - 1, j, 1)]; W[2] = q[AT(i - 1, j, 2)];
    W[3] = alw - an; W[4] = q[AT(i - 1, j, 4)] - ycent[j];
  } else {
    alw = qc[3];
    W[0] = f[0]; W[1] = (i > 0 || c->bcw == BC_REFL) ? -f[1] : f[1];
    W[2] = f[2]; W[3] = f[3]; W[4] = f[4];
  }
  if (i < nx - 1 && mask[AT2(i + 1, j)] != 0) {
    double an = aeqs[i + 1];
    ale = q[AT(i + 1, j, 3)];
    E[0] = q[AT(i + 1, j, 0)] - an * rhoE_c[AT2(i + 1, j)];
    E[1] = q[AT(i + 1, j, 1)]; E[2] = q[AT(i + 1, j, 2)];
    E[3] = ale - an; E[4] = q[AT(i + 1, j, 4)] - ycent[j];
  } else {
    ale = qc[3];
    E[0] = f[0]; E[1] = (i < nx - 1 || c->bce == BC_REFL) ? -f[1] : f[1];
    E[2] = f[2]; E[3] = f[3]; E[4] = f[4];
  }
  if (j > 0 && mask[AT2(i, j - 1)] != 0) {
    als = q[AT(i, j - 1, 3)];
    S[0] = q[AT(i, j - 1, 0)] - aeq * rhoE_c[AT2(i, j - 1)];
    S[1] = q[AT(i, j - 1, 1)]; S[2] = q[AT(i, j - 1, 2)];
    S[3] = als - aeq; S[4] = q[AT(i, j - 1, 4)] - ycent[j - 1];
  } else {
    als = qc[3];
    S[0] = f[0]; S[1] = f[1]; S[2] = (j > 0 || c->bcs == BC_REFL) ? -f[2] : f[2];
    S[3] = f[3]; S[4] = f[4];
  }
  if (j < ny - 1 && mask[AT2(i, j + 1)] != 0) {
    aln = q[AT(i, j + 1, 3)];
    N[0] = q[AT(i, j + 1, 0)] - aeq * rhoE_c[AT2(i, j + 1)];
    N[1] = q[AT(i, j + 1, 1)]; N[2] = q[AT(i, j + 1, 2)];
    N[3] = aln - aeq; N[4] = q[AT(i, j + 1, 4)] - ycent[j + 1];
  } else {
    aln = qc[3];
    N[0] = f[0]; N[1] = f[1]; N[2] = (j < ny - 1 || c->bcn == BC_REFL) ? -f[2] : f[2];
    N[3] = f[3]; N[4] = f[4];
  }
  double athr = 10.0 * c->eps;
  int second = qc[3] > athr && alw > athr && ale > athr && als > athr && aln > athr;
  int is_quiet = 1;
  for (int m = 0; m < 5; m++)
    if (!(f[m] == 0.0 && W[m] == 0.0 && E[m] == 0.0 && S[m] == 0.0 && N[m] == 0.0))
      is_quiet = 0;

  double lx[5] = {0, 0, 0, 0, 0}, ly[5] = {0, 0, 0, 0, 0}, dt[5] = {0, 0, 0, 0, 0};
  double *ps = psi + AT(i, j, 0);
  if (is_quiet) {
    quiet[AT2(i, j)] = 1;
    double v = second ? 1.0 : 0.0;
    for (int m = 0; m < 5; m++) ps[m] = v;
  } else {
    quiet[AT2(i, j)] = 0;
    if (second) {
      double hx = 0.5 * dx, hy = 0.5 * dy;
      double rdx = 1.0 / (2.0 * dx), rdy = 1.0 / (2.0 * dy);
      for (int m = 0; m < 5; m++) {
        double sx = (E[m] - W[m]) * rdx;
        double sy = (N[m] - S[m]) * rdy;
        double p = bj_limit(f[m], W[m], E[m], S[m], N[m], sx, sy, hx, hy);
        ps[m] = p;
        lx[m] = p * sx;
        ly[m] = p * sy;
      }
      /* kernels.py:889-907 with a1_apply/a2_apply (190-208) */
      double rho = qc[0] / qc[3];
      double u = qc[1] / qc[0];
      double v = qc[2] / qc[0];
      double p = wbo_tait_p(rho, k0, rho0, gamma);
      double c2 = wbo_sound_c2(rho, k0, rho0, gamma);
      double e1c = -aeq * (g * rho0 / k0) * rhoE_c[AT2(i, j)];
      double gy0 = ly[0] + e1c;
      double gy4 = ly[4] + 1.0;
      double a1[5], a2[5];
      a1[0] = lx[1];
      a1[1] = (c2 - u * u) * lx[0] + 2.0 * u * lx[1] + (p - rho * c2) * lx[3];
      a1[2] = -u * v * lx[0] + v * lx[1] + u * lx[2];
      a1[3] = u * lx[3];
      a1[4] = 0.0;
      a2[0] = ly[2];
      a2[1] = -u * v * gy0 + v * ly[1] + u * ly[2];
      a2[2] = (c2 - v * v) * gy0 + 2.0 * v * ly[2] + (p - rho * c2) * ly[3] +
              qc[3] * rho * g * gy4;
      a2[3] = v * ly[3];
      a2[4] = 0.0;
      for (int m = 0; m < 5; m++) dt[m] = -(a1[m] + a2[m]);
    } else {
      for (int m = 0; m < 5; m++) ps[m] = 0.0;
    }
  }

  double hx = 0.5 * dx, hy = 0.5 * dy;
  double rES = rhoE_fy[(size_t)i * (ny + 1) + j];
  double rEN = rhoE_fy[(size_t)i * (ny + 1) + j + 1];
  int mode = 0, bad = 0;
  double b[5], fs0, fn0, fs3, fn3;
  double *oW = fW + AT(i, j, 0), *oE = fE + AT(i, j, 0), *oS = fS + AT(i, j, 0),
         *oN = fN + AT(i, j, 0);
  for (;;) {
    if (mode >= 1) {
      for (int m = 0; m < 5; m++) { lx[m] = 0.0; ly[m] = 0.0; dt[m] = 0.0; ps[m] = 0.0; }
    }
    for (int m = 0; m < 5; m++) b[m] = qc[m] + dt[m] * dt_half;
    double fw0 = b[0] - lx[0] * hx, fw3 = b[3] - lx[3] * hx;
    double fe0 = b[0] + lx[0] * hx, fe3 = b[3] + lx[3] * hx;
    oW[0] = fw0; oW[1] = b[1] - lx[1] * hx; oW[2] = b[2] - lx[2] * hx; oW[3] = fw3;
    oW[4] = b[4] - lx[4] * hx;
    oE[0] = fe0; oE[1] = b[1] + lx[1] * hx; oE[2] = b[2] + lx[2] * hx; oE[3] = fe3;
    oE[4] = b[4] + lx[4] * hx;
    if (mode == 2) {
      fs0 = qc[0]; fn0 = qc[0];
    } else {
      fs0 = (aeq * rES + f[0]) - ly[0] * hy + dt[0] * dt_half;
      fn0 = (aeq * rEN + f[0]) + ly[0] * hy + dt[0] * dt_half;
    }
    fs3 = (aeq + f[3]) - ly[3] * hy + dt[3] * dt_half;
    fn3 = (aeq + f[3]) + ly[3] * hy + dt[3] * dt_half;
    oS[0] = fs0; oN[0] = fn0;
    oS[1] = f[1] - ly[1] * hy + dt[1] * dt_half;
    oN[1] = f[1] + ly[1] * hy + dt[1] * dt_half;
    oS[2] = f[2] - ly[2] * hy + dt[2] * dt_half;
    oN[2] = f[2] + ly[2] * hy + dt[2] * dt_half;
    oS[3] = fs3; oN[3] = fn3;
    oS[4] = yfaces[j]; oN[4] = yfaces[j + 1];
    bad = !(fs0 > 0.0 && fs3 > 0.0 && fn0 > 0.0 && fn3 > 0.0 && fw0 > 0.0 && fw3 > 0.0 &&
            fe0 > 0.0 && fe3 > 0.0);
    if (!bad || mode == 2) break;
    mode++;
  }
  /* kernels.py:997-1021 */
  double pES = wbo_tait_p(rES, k0, rho0, gamma);
  double pEN = wbo_tait_p(rEN, k0, rho0, gamma);
  double pS = wbo_tait_p(fs0 / fs3, k0, rho0, gamma);
  double pN = wbo_tait_p(fn0 / fn3, k0, rho0, gamma);
  double afS = fs3 - aeq, afN = fn3 - aeq;
  double pfS = pS - pES, pfN = pN - pEN;
  double rhoc = b[0] / b[3];
  double rfc = rhoc - rhoE_c[AT2(i, j)];
  double afc = b[3] - aeq;
  double uc = b[1] / b[0];
  double vc = b[2] / b[0];
  double *ov = vol + AT(i, j, 0);
  ov[0] = 0.0; ov[1] = 0.0;
  ov[2] = dx * (aeq * (pfN - pfS) + (afN * pEN - afS * pES) + (afN * pfN - afS * pfS)) +
          dx * dy * (aeq * rfc + afc * rhoE_c[AT2(i, j)] + afc * rfc) * g;
  ov[3] = (uc * lx[3] + vc * ly[3]) * dx * dy;
  ov[4] = 0.0;
  return bad;
}

/* kernels.py:1025-1040 */
void wbo_pass_reconstruct(const wbo_cfg *c, const double *q, const uint8_t *mask,
                          const double *aeqs, const double *rhoE_c,
                          const double *rhoE_fy, const double *ycent,
                          const double *yfaces, double dt_half, double *fW,
                          double *fE, double *fS, double *fN, double *vol,
                          double *psi, uint8_t *quiet, uint8_t *flags) {
  const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nx; i++)
    for (int j = 0; j < ny; j++) {
      if (mask[AT2(i, j)] == 0) continue;
      if (cell_reconstruct(c, q, mask, i, j, aeqs, rhoE_c, rhoE_fy, ycent, yfaces, dt_half,
                           fW, fE, fS, fN, vol, psi, quiet))
        flags[AT2(i, j)] = 1;
    }
}

/* grid.py:213-220 */
static int side_mode(int kind, const double *seg, double coord) {
  if (kind == BC_INFLOW) return (seg[0] <= coord && coord <= seg[1]) ? BC_INFLOW : BC_REFL;
  return kind;
}

/* ghost construction for a boundary face, kernels.py:1080-1099 / 1150-1169.
 * `in` is the interior face state, `nrm` the normal-momentum component. */
static void edge_ghost(int code, const double *in, int nrm, double rho0, const double *inflow,
                       double *gh) {
  if (code == BC_REFL) {
    for (int m = 0; m < 5; m++) gh[m] = in[m];
    gh[nrm] = -in[nrm];
  } else if (code == BC_TRANS) {
    double ar = in[3] * rho0;
    gh[0] = ar; gh[1] = ar * (in[1] / in[0]); gh[2] = ar * (in[2] / in[0]);
    gh[3] = in[3]; gh[4] = in[4];
  } else {
    gh[0] = inflow[0]; gh[1] = inflow[1]; gh[2] = inflow[2]; gh[3] = inflow[3];
    gh[4] = in[4];
  }
}

/* x-faces: grid.py:223-246 classification + kernels.py:1047-1116 */
void wbo_sweep_vertical(const wbo_cfg *c, const uint8_t *mask, const double *ycent,
                        const double *fW, const double *fE, double *DW, double *DE,
                        const double *y0s, const double *aeqs, const uint8_t *quiet) {
  const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
  for (int ifc = 0; ifc <= nx; ifc++)
    for (int j = 0; j < ny; j++) {
      int left = ifc >= 1 && mask[AT2(ifc - 1, j)] != 0;
      int right = ifc <= nx - 1 && mask[AT2(ifc, j)] != 0;
      if (!left && !right) continue;
      int bcm;
      if (left && right) bcm = 0;
      else if (right) bcm = -(ifc == 0 ? side_mode(c->kind_l, c->seg_l, ycent[j]) : BC_REFL);
      else bcm = (ifc == nx ? side_mode(c->kind_r, c->seg_r, ycent[j]) : BC_REFL);
      if (bcm == 0 && quiet[AT2(ifc - 1, j)] != 0 && quiet[AT2(ifc, j)] != 0 &&
          y0s[ifc - 1] == y0s[ifc] && aeqs[ifc - 1] == aeqs[ifc]) {
        for (int m = 0; m < 5; m++) { DE[AT(ifc - 1, j, m)] = 0.0; DW[AT(ifc, j, m)] = 0.0; }
        continue;
      }
      double a[5], b[5], o[10];
      if (bcm == 0) {
        memcpy(a, fE + AT(ifc - 1, j, 0), 5 * sizeof(double));
        memcpy(b, fW + AT(ifc, j, 0), 5 * sizeof(double));
      } else if (bcm < 0) {
        memcpy(b, fW + AT(ifc, j, 0), 5 * sizeof(double));
        edge_ghost(-bcm, b, 1, c->rho0, c->in_l, a);
      } else {
        memcpy(a, fE + AT(ifc - 1, j, 0), 5 * sizeof(double));
        edge_ghost(bcm, a, 1, c->rho0, c->in_r, b);
      }
      wbo_osher_x_edge(a, b, c->k0, c->rho0, c->gamma, o);
      if (bcm >= 0) memcpy(DE + AT(ifc - 1, j, 0), o, 5 * sizeof(double));
      if (bcm <= 0) memcpy(DW + AT(ifc, j, 0), o + 5, 5 * sizeof(double));
    }
}

/* y-faces: grid.py:249-272 classification + kernels.py:1119-1186 */
void wbo_sweep_horizontal(const wbo_cfg *c, const uint8_t *mask, const double *xcent,
                          const double *fS, const double *fN, double *DS, double *DN,
                          const double *y0s, const double *aeqs, const uint8_t *quiet) {
  const int nx = c->nx, ny = c->ny;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nx; i++)
    for (int jfc = 0; jfc <= ny; jfc++) {
      int below = jfc >= 1 && mask[AT2(i, jfc - 1)] != 0;
      int above = jfc <= ny - 1 && mask[AT2(i, jfc)] != 0;
      if (!below && !above) continue;
      int bcm;
      if (below && above) bcm = 0;
      else if (above) bcm = -(jfc == 0 ? side_mode(c->kind_b, c->seg_b, xcent[i]) : BC_REFL);
      else bcm = (jfc == ny ? side_mode(c->kind_t, c->seg_t, xcent[i]) : BC_REFL);
      if (bcm == 0 && quiet[AT2(i, jfc - 1)] != 0 && quiet[AT2(i, jfc)] != 0) {
        for (int m = 0; m < 5; m++) { DN[AT(i, jfc - 1, m)] = 0.0; DS[AT(i, jfc, m)] = 0.0; }
        continue;
      }
      double a[5], b[5], o[10];
      if (bcm == 0) {
        memcpy(a, fN + AT(i, jfc - 1, 0), 5 * sizeof(double));
        memcpy(b, fS + AT(i, jfc, 0), 5 * sizeof(double));
      } else if (bcm < 0) {
        memcpy(b, fS + AT(i, jfc, 0), 5 * sizeof(double));
        edge_ghost(-bcm, b, 2, c->rho0, c->in_b, a);
      } else {
        memcpy(a, fN + AT(i, jfc - 1, 0), 5 * sizeof(double));
        edge_ghost(bcm, a, 2, c->rho0, c->in_t, b);
      }
      wbo_or_y_edge(a, b, y0s[i], aeqs[i], c->k0, c->rho0, c->gamma, c->g, o);
      if (bcm >= 0) memcpy(DN + AT(i, jfc - 1, 0), o, 5 * sizeof(double));
      if (bcm <= 0) memcpy(DS + AT(i, jfc, 0), o + 5, 5 * sizeof(double));
    }
}

/* kernels.py:1217-1315 */
void wbo_apply_update(const wbo_cfg *c, const double *q, double *qn,
                      const uint8_t *mask, const double *fW, const double *fE,
                      const double *fS, const double *fN, const double *DW,
                      const double *DE, const double *DS, const double *DN,
                      const double *vol, double rdx, double rdy, double rvol,
                      uint8_t *flags) {
  const int nx = c->nx, ny = c->ny;
  const double rho0 = c->rho0;
  const double rho_lo = 0.5 * rho0, rho_hi = 2.0 * rho0;
  const double vmax = 2.0 * sqrt(wbo_sound_c2(rho0, c->k0, rho0, c->gamma));
  const double athr = 10.0 * c->eps;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nx; i++)
    for (int j = 0; j < ny; j++) {
      size_t b = AT(i, j, 0);
      if (mask[AT2(i, j)] == 0) {
        for (int m = 0; m < 5; m++) qn[b + m] = q[b + m];
        continue;
      }
      double fxw[3], fxe[3], gys[3], gyn[3];
      flux_x(fW + b, c->k0, rho0, c->gamma, fxw);
      flux_x(fE + b, c->k0, rho0, c->gamma, fxe);
      flux_y(fS + b, gys);
      flux_y(fN + b, gyn);
      for (int m = 0; m < 3; m++)
        qn[b + m] = q[b + m] - rdx * (DW[b + m] + DE[b + m] + (fxe[m] - fxw[m])) -
                    rdy * (DS[b + m] + DN[b + m] + (gyn[m] - gys[m])) - rvol * vol[b + m];
      for (int m = 3; m < 5; m++)
        qn[b + m] = q[b + m] - rdx * (DW[b + m] + DE[b + m]) -
                    rdy * (DS[b + m] + DN[b + m]) - rvol * vol[b + m];
      double a_new = qn[b + 3];
      if (a_new > 0.0 && a_new <= athr) {
        double q0n = qn[b + 0], rho, u, v;
        if (q0n > 0.0) {
          rho = q0n / a_new; u = qn[b + 1] / q0n; v = qn[b + 2] / q0n;
        } else {
          rho = rho_lo; u = 0.0; v = 0.0;
        }
        int clamped = 0;
        if (rho < rho_lo) { rho = rho_lo; clamped = 1; }
        else if (rho > rho_hi) { rho = rho_hi; clamped = 1; }
        if (u > vmax) { u = vmax; clamped = 1; }
        else if (u < -vmax) { u = -vmax; clamped = 1; }
        if (v > vmax) { v = vmax; clamped = 1; }
        else if (v < -vmax) { v = -vmax; clamped = 1; }
        if (clamped) {
          double ar = a_new * rho;
          qn[b + 0] = ar; qn[b + 1] = ar * u; qn[b + 2] = ar * v;
        }
      }
      if (!admissible(qn[b + 0], qn[b + 1], qn[b + 2], qn[b + 3])) flags[AT2(i, j)] = 1;
    }
}
