/*
 * sbs_oracle.c -- plain, slow, obviously-correct CPU oracle of one MPC
 * iteration of the Sample-Based Stochastic (SBS) quadruped controller of
 * arxiv 2403.11383 (Alg. 5).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline leg and --impl reference) may load this library.
 * It shares nothing with the CUDA path (paper_2403_11383_b200/csrc).
 *
 * Precision: binary64 throughout, except the normative binary32 noise
 * recipe, which is written here from the recipe using
 * only correctly-rounded binary32 operations (+ - * / sqrtf fmaf).  Build
 * with -ffp-contract=off so that no a*b+c is fused behind our back.
 *
 * Every function cites the passage it follows.  "Ln" readings are listed
 * in DESIGN.md sec. 3.  No blocking, fusion or reordering beyond the
 * definitions: one sample at a time, one step at a time, literal RK4.
 *
 * Pins (tests/test_oracle_*.py): Philox KAT vectors, libm comparisons and
 * moment / KS tests for the noise, closed forms for contact timing, the
 * cone, free fall / hover / single-foot torque, an independent ODE solver
 * for RK4, whole-rollout closed forms (hover, vertical thrust), mirror
 * symmetry, MPPI worked values and limits, CEM == stable sort.
 */
#include "sbs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================
 * O1  Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11; Random123).
 * The paper does not name its RNG (L31); the north star asks for a
 * counter-based Philox sampler.
 * ==================================================================== */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { /* key schedule: Weyl increments between rounds */
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ======================================================================
 * O3-O4  Normative binary32 Box-Muller.  Constants are
 * written here as decimal literals rounded by the compiler to binary32;
 * the CUDA side writes its own.
 * ==================================================================== */
static float f32_from_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t bits_from_f32(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* ln(u1) with u1 = n 2^-24, n = 2 (w >> 9) + 1 (odd, < 2^24). */
float orc_ln_u24(uint32_t w) {
  uint32_t n = 2u * (w >> 9) + 1u;
  float nf = (float)n;                         /* exact: n < 2^24 */
  uint32_t b = bits_from_f32(nf);
  int e = (int)(b >> 23) - 127;
  float m = f32_from_bits((b & 0x007FFFFFu) | 0x3F800000u); /* m in [1,2) */
  if (m > 1.41421353816986083984375f) {        /* binary32 nearest to sqrt 2 */
    m = m * 0.5f;                              /* exact */
    e = e + 1;
  }
  /* ln m = 2 atanh(s), s = (m-1)/(m+1), |s| <= 0.1716 */
  float num = m - 1.0f;                        /* exact (Sterbenz) */
  float den = m + 1.0f;
  float s = num / den;
  float s2 = s * s;
  float p = 1.0f / 9.0f;                       /* series 1/3 + s^2/5 + s^4/7 + s^6/9 */
  p = fmaf(p, s2, 1.0f / 7.0f);
  p = fmaf(p, s2, 1.0f / 5.0f);
  p = fmaf(p, s2, 1.0f / 3.0f);
  float r = s2 * p;
  float two_s = s + s;
  float ln_m = fmaf(two_s, r, two_s);
  float E = (float)(e - 24);
  /* ln 2 split: hi has 12 trailing zero bits */
  return fmaf(E, 0.693145751953125f, fmaf(E, 1.4286068202862268e-06f, ln_m));
}

/* sin, cos of 2 pi u2 with u2 = ((w >> 9) + 1/2) 2^-23, by octant. */
void orc_sincos_2pi_u(uint32_t w, float* s_out, float* c_out) {
  uint32_t oct = w >> 29;                      /* which eighth of the circle */
  uint32_t i = (w >> 9) & 0x000FFFFFu;         /* 20-bit position inside it  */
  if (oct & 1u) i = 0x000FFFFFu - i;           /* odd octant: distance to its end */
  float fr = (float)i + 0.5f;                  /* exact */
  float t = fr * (0.78539816339744830962f * 0x1p-20f); /* binary32(pi/4) 2^-20: t in (0, pi/4) */
  float t2 = t * t;
  /* sin t = t + t^3 (-1/6 + t^2 (1/120 + t^2 (-1/5040 + t^2/362880))) */
  float ps = 1.0f / 362880.0f;
  ps = fmaf(ps, t2, -1.0f / 5040.0f);
  ps = fmaf(ps, t2, 1.0f / 120.0f);
  ps = fmaf(ps, t2, -1.0f / 6.0f);
  float t3 = t2 * t;
  float sn = fmaf(t3, ps, t);
  /* cos t = 1 + t^2 (-1/2 + t^2 (1/24 + t^2 (-1/720 + t^2 (1/40320 - t^2/3628800)))) */
  float pc = -1.0f / 3628800.0f;
  pc = fmaf(pc, t2, 1.0f / 40320.0f);
  pc = fmaf(pc, t2, -1.0f / 720.0f);
  pc = fmaf(pc, t2, 1.0f / 24.0f);
  pc = fmaf(pc, t2, -0.5f);
  float cs = fmaf(t2, pc, 1.0f);
  /* octant o covers [o pi/4, (o+1) pi/4); table of (sin, cos) in terms of (sn, cs) */
  float S, C;
  switch (oct) {
    case 0: S = sn;  C = cs;  break;
    case 1: S = cs;  C = sn;  break;
    case 2: S = cs;  C = -sn; break;
    case 3: S = sn;  C = -cs; break;
    case 4: S = -sn; C = -cs; break;
    case 5: S = -cs; C = -sn; break;
    case 6: S = -cs; C = sn;  break;
    default: S = -sn; C = cs; break;
  }
  *s_out = S;
  *c_out = C;
}

/* Box-Muller on (w0,w1) -> (z0,z1) and (w2,w3) -> (z2,z3). */
void orc_normal4(const uint32_t w[4], float z[4]) {
  for (int pair = 0; pair < 2; ++pair) {
    float ln_u = orc_ln_u24(w[2 * pair]);
    float rad = sqrtf(-2.0f * ln_u);
    float sn, cs;
    orc_sincos_2pi_u(w[2 * pair + 1], &sn, &cs);
    z[2 * pair + 0] = rad * cs;
    z[2 * pair + 1] = rad * sn;
  }
}

/* orc_normal4 over n Philox blocks (tests: exhaustive recipe comparisons). */
void orc_normal4_batch(const uint32_t* w, int64_t n, float* z) {
  for (int64_t i = 0; i < n; ++i) orc_normal4(&w[4 * i], &z[4 * i]);
}

/* ======================================================================
 * a0  Warm start ("initiating each new search from the solution
 * obtained in the previous iteration"; reading L20): the previous mean's
 * spline re-evaluated at knot times shifted by dt, clamped to the horizon
 * end.  In knot units t_p + dt = (p H + (P-1)) / H.
 * ==================================================================== */
static int64_t orc_D(const orc_config* c) { return 12 * (int64_t)c->knots; }

void orc_warm_shift(const orc_config* c, const double* mu, double* mu_shift) {
  const int P = c->knots, H = c->horizon;
  double ch[ORC_MAX_KNOTS];
  for (int leg = 0; leg < 4; ++leg)
    for (int ax = 0; ax < 3; ++ax) {
      for (int p = 0; p < P; ++p) ch[p] = mu[(p * 4 + leg) * 3 + ax];
      for (int p = 0; p < P; ++p) {
        double v;
        orc_spline_eval(P, ch, (int64_t)p * H + (P - 1), H, &v);
        mu_shift[(p * 4 + leg) * 3 + ax] = v;
      }
    }
}

/* ======================================================================
 * O5-O6  One sample (Alg. 5 line "theta_k ~ N(theta, C)", P:236;
 * theta1 uniform over the discretised frequencies).
 * Counter layout: ctr = (q, k, iter, robot), key = (seed_lo, seed_hi).
 * theta2[d] = mu'[d] + sqrt(var[d]) z[d]; sample 0 = mean (L21).
 * ==================================================================== */
void orc_sample(const orc_config* c, const double* mu_shift, const double* var,
                int32_t cur_idx, uint32_t iter, uint32_t robot, int64_t k,
                double* theta, float* z, int32_t* idx) {
  const int64_t D = orc_D(c);
  const uint32_t key[2] = {(uint32_t)(c->seed & 0xFFFFFFFFu), (uint32_t)(c->seed >> 32)};
  if (c->elite_preserve && k == 0) {
    for (int64_t d = 0; d < D; ++d) { z[d] = 0.0f; theta[d] = mu_shift[d]; }
    *idx = cur_idx;
    return;
  }
  for (int64_t q = 0; q < D / 4; ++q) {
    uint32_t ctr[4] = {(uint32_t)q, (uint32_t)k, iter, robot}, w[4];
    orc_philox4x32_10(ctr, key, w);
    orc_normal4(w, &z[4 * q]);
  }
  /* L41: interleaved groups of samples with std scaled by sigma_scale[g] */
  const double sc = c->n_sigma_groups > 1 ? c->sigma_scale[k % c->n_sigma_groups] : 1.0;
  for (int64_t d = 0; d < D; ++d) theta[d] = mu_shift[d] + sc * sqrt(var[d]) * (double)z[d];
  if (c->gait_adapt) {
    uint32_t ctr[4] = {0x80000000u, (uint32_t)k, iter, robot}, w[4];
    orc_philox4x32_10(ctr, key, w);
    *idx = (int32_t)(((uint64_t)w[0] * (uint64_t)c->n_freq) >> 32);
  } else {
    *idx = cur_idx;
  }
}

/* ======================================================================
 * O7  computeContactSequence(theta1) (L22): leg i is in
 * stance at step j iff frac(phi0 + f j dt + offset_i) < D_f, with the
 * phase held as an unsigned Q0.32 fraction of a gait cycle.
 * ==================================================================== */
uint32_t orc_phase_inc(double f_hz, double dt) {
  long long v = llround((f_hz * dt) * 4294967296.0);
  return (uint32_t)(uint64_t)v;
}
uint64_t orc_stance_threshold(double duty_factor) {
  return (uint64_t)llround(duty_factor * 4294967296.0);
}
void orc_contact_sequence(const orc_config* c, uint32_t phase0, double f_hz, int32_t* delta) {
  const uint32_t inc = orc_phase_inc(f_hz, c->dt);
  const uint64_t thr = orc_stance_threshold(c->duty_factor);
  for (int j = 0; j < c->horizon; ++j)
    for (int i = 0; i < 4; ++i) {
      uint32_t off = (uint32_t)(uint64_t)llround(c->phase_offset[i] * 4294967296.0);
      uint32_t ph = phase0 + (uint32_t)j * inc + off; /* mod 2^32 */
      delta[j * 4 + i] = ((uint64_t)ph < thr) ? 1 : 0;
    }
}

/* ======================================================================
 * O8  GRF spline sigma((t_knot, theta2), t) (L7): uniform
 * Catmull-Rom through P knots spanning [0, H dt], phantom end knots by
 * linear extrapolation.  Evaluation point in knot units tau = a_num/a_den.
 * ==================================================================== */
void orc_spline_eval(int32_t P, const double* kn, int64_t a_num, int64_t a_den, double* out) {
  int64_t s = a_num / a_den;
  double u = (double)(a_num % a_den) / (double)a_den;
  if (s >= P - 1) { s = P - 2; u = 1.0; }      /* clamp to the horizon end */
  double km1 = (s - 1 >= 0) ? kn[s - 1] : 2.0 * kn[0] - kn[1];
  double k0 = kn[s];
  double k1 = kn[s + 1];
  double k2 = (s + 2 <= P - 1) ? kn[s + 2] : 2.0 * kn[P - 1] - kn[P - 2];
  double u2 = u * u, u3 = u2 * u;
  double wm1 = (-u3 + 2.0 * u2 - u) / 2.0;
  double w0 = (3.0 * u3 - 5.0 * u2 + 2.0) / 2.0;
  double w1 = (-3.0 * u3 + 4.0 * u2 + u) / 2.0;
  double w2 = (u3 - u2) / 2.0;
  *out = wm1 * km1 + w0 * k0 + w1 * k1 + w2 * k2;
}

/* Gamma_j = sigma(theta2, t_j), t_j = j dt (Alg. 5 policy), for all
 * 12 channels; knot layout d = (p*4 + leg)*3 + axis. */
void orc_spline_step(const orc_config* c, const double* theta, int32_t j, double gamma[12]) {
  const int P = c->knots, H = c->horizon;
  double ch[ORC_MAX_KNOTS];
  for (int leg = 0; leg < 4; ++leg)
    for (int ax = 0; ax < 3; ++ax) {
      for (int p = 0; p < P; ++p) ch[p] = theta[(p * 4 + leg) * 3 + ax];
      orc_spline_eval(P, ch, (int64_t)j * (P - 1), H, &gamma[leg * 3 + ax]);
    }
}

/* ======================================================================
 * O9  Friction cone ("constrained to respect friction cone
 * constraints"; L9): clamp f_z to [fz_min, fz_max], then |f_x|,|f_y| to
 * mu f_z (inner pyramid); pen = squared violation of the raw output.
 * ==================================================================== */
/* written with fmin/fmax (same values as the comparison forms for every non-NaN x) so
 * that the op-counting mode (opcount.cpp) sees a clamped result as sample-dependent */
static double clampd(double x, double lo, double hi) { return fmin(fmax(x, lo), hi); }
static double pos(double x) { return fmax(x, 0.0); }

void orc_cone(const orc_config* c, const double raw[3], double out[3], double* pen) {
  double fz = clampd(raw[2], c->fz_min, c->fz_max);
  double l = c->mu * fz;
  out[0] = clampd(raw[0], -l, l);
  out[1] = clampd(raw[1], -l, l);
  out[2] = fz;
  double vz = pos(c->fz_min - raw[2]) + pos(raw[2] - c->fz_max);
  double vx = pos(fabs(raw[0]) - l), vy = pos(fabs(raw[1]) - l);
  *pen = vz * vz + vx * vx + vy * vy;
}

/* ======================================================================
 * O10  SRBD dynamics, Eq. 1.  State x = (p_c, v_c, Phi, w)
 * with Phi = (roll, pitch, yaw) ZYX (L24) and w in the body frame.
 *   p' = v
 *   v' = (1/m) sum_i delta_i Gamma_i + g
 *   Phi' = E'^-1(Phi) w
 *   w' = I^-1 ( R^T sum_i delta_i (p_f,i - p_c) x Gamma_i  -  w x I w )
 * Gamma and the lever arms are world-frame; R = Rz(yaw) Ry(pitch) Rx(roll).
 * ==================================================================== */
static void mat3_mul(const double A[9], const double B[9], double C[9]) {
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[r * 3 + k] * B[k * 3 + cc];
      C[r * 3 + cc] = s;
    }
}
static void mat3_vec(const double A[9], const double v[3], double o[3]) {
  for (int r = 0; r < 3; ++r) o[r] = A[r * 3 + 0] * v[0] + A[r * 3 + 1] * v[1] + A[r * 3 + 2] * v[2];
}
static void mat3T_vec(const double A[9], const double v[3], double o[3]) {
  for (int r = 0; r < 3; ++r) o[r] = A[0 * 3 + r] * v[0] + A[1 * 3 + r] * v[1] + A[2 * 3 + r] * v[2];
}
static void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
static void mat3_inv(const double A[9], double Ai[9]) { /* adjugate / determinant */
  double a = A[0], b = A[1], cc = A[2], d = A[3], e = A[4], f = A[5], g = A[6], h = A[7], i = A[8];
  double det = a * (e * i - f * h) - b * (d * i - f * g) + cc * (d * h - e * g);
  Ai[0] = (e * i - f * h) / det; Ai[1] = (cc * h - b * i) / det; Ai[2] = (b * f - cc * e) / det;
  Ai[3] = (f * g - d * i) / det; Ai[4] = (a * i - cc * g) / det; Ai[5] = (cc * d - a * f) / det;
  Ai[6] = (d * h - e * g) / det; Ai[7] = (b * g - a * h) / det; Ai[8] = (a * e - b * d) / det;
}

void orc_dynamics(const orc_config* c, const double x[12], const double gamma[12],
                  const int32_t stance[4], const double feet[12], double xd[12]) {
  const double* p = &x[0];
  const double* v = &x[3];
  const double phi = x[6], th = x[7], psi = x[8];
  const double* w = &x[9];
  const double cr = cos(phi), sr = sin(phi), cp = cos(th), sp = sin(th), cy = cos(psi), sy = sin(psi);
  const double Rz[9] = {cy, -sy, 0, sy, cy, 0, 0, 0, 1};
  const double Ry[9] = {cp, 0, sp, 0, 1, 0, -sp, 0, cp};
  const double Rx[9] = {1, 0, 0, 0, cr, -sr, 0, sr, cr};
  double Rzy[9], R[9];
  mat3_mul(Rz, Ry, Rzy);
  mat3_mul(Rzy, Rx, R);

  double F[3] = {0, 0, 0}, tau_w[3] = {0, 0, 0};
  for (int i = 0; i < 4; ++i) {
    if (!stance[i]) continue;
    const double* G = &gamma[3 * i];
    double r[3] = {feet[3 * i] - p[0], feet[3 * i + 1] - p[1], feet[3 * i + 2] - p[2]};
    double rxG[3];
    cross3(r, G, rxG);
    for (int a = 0; a < 3; ++a) { F[a] += G[a]; tau_w[a] += rxG[a]; }
  }
  double Iinv[9], Iw[3], gyro[3], tau_b[3], rhs[3], wd[3];
  mat3_inv(c->inertia, Iinv);
  mat3_vec(c->inertia, w, Iw);
  cross3(w, Iw, gyro);
  mat3T_vec(R, tau_w, tau_b);
  for (int a = 0; a < 3; ++a) rhs[a] = tau_b[a] - gyro[a];
  mat3_vec(Iinv, rhs, wd);

  for (int a = 0; a < 3; ++a) {
    xd[a] = v[a];
    xd[3 + a] = F[a] / c->mass + c->gravity[a];
    xd[9 + a] = wd[a];
  }
  /* E'^-1 for ZYX angles (Rathod2021, cited at P:274) */
  xd[6] = w[0] + tan(th) * (sr * w[1] + cr * w[2]);
  xd[7] = cr * w[1] - sr * w[2];
  xd[8] = (sr * w[1] + cr * w[2]) / cp;
}

/* O11  x_{j+1} = f(x_j, u_j): classic RK4, Gamma and feet held (L8, L25). */
void orc_rk4(const orc_config* c, const double x[12], const double gamma[12],
             const int32_t stance[4], const double feet[12], double h, double xn[12]) {
  double k1[12], k2[12], k3[12], k4[12], t[12];
  orc_dynamics(c, x, gamma, stance, feet, k1);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + 0.5 * h * k1[a];
  orc_dynamics(c, t, gamma, stance, feet, k2);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + 0.5 * h * k2[a];
  orc_dynamics(c, t, gamma, stance, feet, k3);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + h * k3[a];
  orc_dynamics(c, t, gamma, stance, feet, k4);
  for (int a = 0; a < 12; ++a) xn[a] = x[a] + h / 6.0 * (k1[a] + 2.0 * k2[a] + 2.0 * k3[a] + k4[a]);
}

/* ======================================================================
 * O12  Rollout(theta_k, x0), Alg. 2 with the policy pi of
 * Alg. 5 and the cost of P:342-351:
 *   for j = 0..H-1:  u_j = pi(theta, t_j);  J += r(u_j, x_j, x^r_j);
 *                    x_{j+1} = f(x_j, u_j)
 *   J += rho (f_k - f_nominal)^2
 * r = (x-x^r)^T Q (x-x^r) + (u-u^r)^T R (u-u^r) + w_fc pen (L9-L12).
 * Divergence (L26): non-finite, |x_c| > 1e6 or |pitch| >= pi/2 - 1e-3 in
 * any x_{j+1} => J = +inf.
 * ==================================================================== */
static int orc_state_bad(const double x[12]) {
  for (int a = 0; a < 12; ++a)
    if (!isfinite(x[a]) || fabs(x[a]) > 1e6) return 1;
  return fabs(x[7]) >= M_PI / 2.0 - 1e-3;
}

double orc_rollout(const orc_config* c, const double x0[12], uint32_t phase0,
                   const double feet_cur[12], const double feet_next[12],
                   const double* xref, const double* theta, int32_t fidx, double* traj) {
  const int H = c->horizon;
  const double f = c->freq_hz[fidx];
  int32_t* delta = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(H > 0 ? H : 1));
  orc_contact_sequence(c, phase0, f, delta);
  double x[12], xn[12], feet[12];
  memcpy(x, x0, sizeof x);
  memcpy(feet, feet_cur, sizeof feet);
  if (traj) memcpy(traj, x, sizeof x);
  int touched[4] = {0, 0, 0, 0};
  double J = 0.0;
  for (int j = 0; j < H; ++j) {
    const int32_t* st = &delta[4 * j];
    /* lever-arm feet (L23): feet_cur until the leg's first touchdown in the horizon */
    for (int i = 0; i < 4; ++i) {
      if (j > 0 && !touched[i] && delta[4 * (j - 1) + i] == 0 && st[i] == 1) touched[i] = 1;
      for (int a = 0; a < 3; ++a) feet[3 * i + a] = touched[i] ? feet_next[3 * i + a] : feet_cur[3 * i + a];
    }
    /* u_j = [Gamma_j, delta_j]: spline, mask by delta, cone */
    double raw[12], gam[12], pen_sum = 0.0;
    orc_spline_step(c, theta, j, raw);
    int n_st = 0;
    for (int i = 0; i < 4; ++i) n_st += st[i];
    for (int i = 0; i < 4; ++i) {
      if (st[i]) {
        double pen;
        orc_cone(c, &raw[3 * i], &gam[3 * i], &pen);
        pen_sum += pen;
      } else {
        gam[3 * i] = gam[3 * i + 1] = gam[3 * i + 2] = 0.0;
      }
    }
    /* stage cost r(u_j, x_j, x^r_j) */
    const double* xr = &xref[12 * j];
    double stage = 0.0;
    for (int a = 0; a < 12; ++a) {
      double e = x[a] - xr[a];
      if (a == 8) e = remainder(e, 2.0 * M_PI); /* yaw wrapped */
      stage += c->Q[a] * e * e;
    }
    const double ur_z = -c->mass * c->gravity[2] / (double)(n_st > 1 ? n_st : 1); /* L12 */
    for (int i = 0; i < 4; ++i) {
      if (!st[i]) continue;
      for (int a = 0; a < 3; ++a) {
        double ur = (a == 2) ? ur_z : 0.0;
        double e = gam[3 * i + a] - ur;
        stage += c->R[3 * i + a] * e * e;
      }
    }
    stage += c->w_fc * pen_sum;
    J += stage;
    /* x_{j+1} = f(x_j, u_j) */
    orc_rk4(c, x, gam, st, feet, c->dt, xn);
    memcpy(x, xn, sizeof x);
    if (traj) memcpy(&traj[12 * (j + 1)], x, sizeof x);
    if (orc_state_bad(x)) { J = INFINITY; break; }
  }
  free(delta);
  if (isfinite(J)) {
    double df = f - c->f_nominal;
    J += c->rho * df * df;                     /* P:350, once per rollout (L14) */
  }
  if (!isfinite(J)) J = INFINITY;
  return J;
}

/* ======================================================================
 * O13  MPPI UpdateMean (Alg. 4; weights P:165-172, reading L1):
 *   beta = min_k J_k;  w_k = exp(-(J_k - beta)/lambda);  Omega = sum w;
 *   theta_new = sum (w_k / Omega) theta_k.   Covariance unchanged.
 * ==================================================================== */
int orc_mppi(int64_t K, int32_t D, const double* J, const double* theta, double lambda,
             double* mu_new, orc_diag* dg) {
  double beta = INFINITY;
  int64_t argmin = -1, n_fin = 0;
  double sumJ = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    if (J[k] < beta) { beta = J[k]; argmin = k; }
    if (isfinite(J[k])) { ++n_fin; sumJ += J[k]; }
  }
  dg->n_diverged = K - n_fin;
  dg->argmin = argmin;
  dg->j_min = beta;
  dg->j_mean = n_fin ? sumJ / (double)n_fin : INFINITY;
  if (!isfinite(beta)) { dg->omega = 0.0; dg->ess = 0.0; return ORC_WARN_ALL_DIVERGED; }
  double* w = (double*)malloc(sizeof(double) * (size_t)K);
  double Omega = 0.0, W2 = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    w[k] = exp(-(J[k] - beta) / lambda);       /* exp(-inf) = 0 */
    Omega += w[k];
    W2 += w[k] * w[k];
  }
  for (int32_t d = 0; d < D; ++d) {
    double s = 0.0;
    for (int64_t k = 0; k < K; ++k) s += (w[k] / Omega) * theta[k * D + d];
    mu_new[d] = s;
  }
  dg->omega = Omega;
  dg->ess = Omega * Omega / W2;
  free(w);
  return ORC_OK;
}

/* ======================================================================
 * O14  Elite selection (Alg. 1 lines 3-5): the K_e first
 * entries of the samples sorted ascending by cost; ties by sample index
 * (stable), NaN as +inf (L4).  Library qsort on a total order.
 * ==================================================================== */
static const double* g_sort_J;
static int cmp_idx(const void* a, const void* b) {
  int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  double ji = g_sort_J[i], jj = g_sort_J[j];
  if (isnan(ji)) ji = INFINITY;
  if (isnan(jj)) jj = INFINITY;
  if (ji < jj) return -1;
  if (ji > jj) return 1;
  return (i < j) ? -1 : (i > j);               /* stable: by index */
}
int orc_cem_select(int64_t K, const double* J, int64_t K_e, int64_t* elite) {
  if (K_e < 1 || K_e > K) return ORC_ERR_INVALID_ARG;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)K);
  for (int64_t k = 0; k < K; ++k) order[k] = k;
  g_sort_J = J;
  qsort(order, (size_t)K, sizeof(int64_t), cmp_idx); /* total order => result is unique */
  memcpy(elite, order, sizeof(int64_t) * (size_t)K_e);
  free(order);
  return ORC_OK;
}

/* CEM / Naive update (Alg. 1 UpdateMean/UpdateCov; Alg. 3, P:152-153;
 * reading L17/L18): elite mean; diagonal population variance of the elites
 * floored at var_floor (CEM) or unchanged (Naive: K_e = 1). */
int orc_cem_update(int64_t K, int32_t D, const double* J, const double* theta,
                   int64_t K_e, const double* var_floor, int32_t update_var,
                   double* mu_new, double* var_new, int64_t* elite, orc_diag* dg) {
  int64_t n_fin = 0;
  double sumJ = 0.0;
  for (int64_t k = 0; k < K; ++k)
    if (isfinite(J[k])) { ++n_fin; sumJ += J[k]; }
  int rc = orc_cem_select(K, J, K_e, elite);
  if (rc) return rc;
  dg->n_diverged = K - n_fin;
  dg->argmin = elite[0];
  dg->j_min = J[elite[0]];
  dg->j_mean = n_fin ? sumJ / (double)n_fin : INFINITY;
  dg->omega = 0.0;
  dg->ess = 0.0;
  if (n_fin == 0) return ORC_WARN_ALL_DIVERGED;
  int64_t ne = K_e < n_fin ? K_e : n_fin;      /* diverged samples never enter the mean */
  for (int32_t d = 0; d < D; ++d) {
    double s = 0.0;
    for (int64_t e = 0; e < ne; ++e) s += theta[elite[e] * D + d];
    mu_new[d] = s / (double)ne;
  }
  if (update_var) {
    for (int32_t d = 0; d < D; ++d) {
      double s = 0.0;
      for (int64_t e = 0; e < ne; ++e) {
        double dv = theta[elite[e] * D + d] - mu_new[d];
        s += dv * dv;
      }
      double v = s / (double)ne;
      var_new[d] = v > var_floor[d] ? v : var_floor[d];
    }
  }
  dg->omega = (double)ne;
  dg->ess = (double)ne;
  return ORC_OK;
}

/* ======================================================================
 * f3 (L42): CEM with a full covariance C = L L^T (Alg. 1 UpdateCov).
 * Sampling theta2 = mu' + L z (z the same normative noise); the elite
 * covariance (1/n) sum (theta - mu_new)(theta - mu_new)^T plus the diagonal
 * floor diag((sigma_min_frac sigma_axis)^2) (keeps C positive definite for any
 * K_e); L = Cholesky factor (Cholesky-Banachiewicz, textbook order).
 * ==================================================================== */
int orc_cholesky(int32_t D, const double* C, double* L) {
  for (int32_t i = 0; i < D; ++i)
    for (int32_t j = 0; j < D; ++j) L[i * D + j] = 0.0;
  for (int32_t i = 0; i < D; ++i) {
    for (int32_t j = 0; j <= i; ++j) {
      double s = C[i * D + j];
      for (int32_t k = 0; k < j; ++k) s -= L[i * D + k] * L[j * D + k];
      if (i == j) {
        if (!(s > 0.0)) return -1;
        L[i * D + i] = sqrt(s);
      } else {
        L[i * D + j] = s / L[j * D + j];
      }
    }
  }
  return 0;
}

void orc_sample_full(const orc_config* c, const double* mu_shift, const double* L, int32_t cur_idx,
                     uint32_t iter, uint32_t robot, int64_t k, double* theta, float* z, int32_t* idx) {
  const int64_t D = orc_D(c);
  double dummy_var[ORC_MAX_D] = {0};
  orc_sample(c, mu_shift, dummy_var, cur_idx, iter, robot, k, theta, z, idx); /* z, theta1; theta2 = mu' */
  if (c->elite_preserve && k == 0) return;
  for (int64_t i = 0; i < D; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j <= i; ++j) s += L[i * D + j] * (double)z[j];
    theta[i] = mu_shift[i] + s;
  }
}

int orc_cem_update_full(int64_t K, int32_t D, const double* J, const double* theta, int64_t K_e,
                        const double* var_floor, double* mu_new, double* C_new, double* L_new,
                        int64_t* elite, orc_diag* dg) {
  double var_dummy[ORC_MAX_D];
  int rc = orc_cem_update(K, D, J, theta, K_e, var_floor, 0, mu_new, var_dummy, elite, dg);
  if (rc != ORC_OK) return rc;
  int64_t n_fin = K - dg->n_diverged;
  int64_t ne = K_e < n_fin ? K_e : n_fin;
  for (int32_t i = 0; i < D; ++i)
    for (int32_t j = 0; j < D; ++j) {
      double s = 0.0;
      for (int64_t e = 0; e < ne; ++e)
        s += (theta[elite[e] * D + i] - mu_new[i]) * (theta[elite[e] * D + j] - mu_new[j]);
      C_new[i * D + j] = s / (double)ne + (i == j ? var_floor[i] : 0.0);
    }
  return orc_cholesky(D, C_new, L_new) == 0 ? ORC_OK : ORC_ERR_INVALID_ARG;
}

/* ======================================================================
 * Alg. 5: one iteration of the SBS predictive controller.
 *   sample K thetas  ->  J_k = Rollout(theta_k, x0)  ->  update  ->  output
 * Output: u0 = mask(delta_0) proj(mean_new at t = 0).
 * ==================================================================== */
int orc_step(const orc_config* c, uint32_t robot, const double x0[12], uint32_t phase0,
             const double feet_cur[12], const double feet_next[12], const double* xref,
             orc_state* st, orc_output* out, double* J_out, int32_t* fidx_out,
             double* theta_out, float* z_out, int64_t* elite_out) {
  const int64_t K = c->n_samples, D = orc_D(c);
  memset(out, 0, sizeof *out);
  if (K < 1 || c->knots < 2 || c->knots > ORC_MAX_KNOTS || c->horizon < 1) return out->status = ORC_ERR_INVALID_ARG;
  for (int a = 0; a < 12; ++a)
    if (!isfinite(x0[a])) return out->status = ORC_ERR_NONFINITE;
  if (fabs(x0[7]) >= M_PI / 2.0 - 1e-3) return out->status = ORC_ERR_SINGULAR;

  double mu_shift[ORC_MAX_D];
  if (c->warm_shift) orc_warm_shift(c, st->mean, mu_shift);
  else memcpy(mu_shift, st->mean, sizeof(double) * (size_t)D);

  double* theta = (double*)malloc(sizeof(double) * (size_t)(K * D));
  double* J = (double*)malloc(sizeof(double) * (size_t)K);
  int32_t* fidx = (int32_t*)malloc(sizeof(int32_t) * (size_t)K);
  float z[ORC_MAX_D];
  for (int64_t k = 0; k < K; ++k) {
    if (c->full_cov) orc_sample_full(c, mu_shift, st->chol, st->freq_idx, st->iter, robot, k, &theta[k * D], z, &fidx[k]);
    else orc_sample(c, mu_shift, st->var, st->freq_idx, st->iter, robot, k, &theta[k * D], z, &fidx[k]);
    if (z_out) memcpy(&z_out[k * D], z, sizeof(float) * (size_t)D);
    J[k] = orc_rollout(c, x0, phase0, feet_cur, feet_next, xref, &theta[k * D], fidx[k], NULL);
  }

  double mu_new[ORC_MAX_D], var_new[ORC_MAX_D];
  memcpy(var_new, st->var, sizeof(double) * (size_t)D);
  int rc;
  int64_t argmin;
  if (c->mode == ORC_MPPI) {
    rc = orc_mppi(K, (int32_t)D, J, theta, c->lambda, mu_new, &out->diag);
    argmin = out->diag.argmin;
  } else {
    int64_t Ke = (c->mode == ORC_NAIVE) ? 1 : c->n_elite;
    double floor_[ORC_MAX_D];
    for (int64_t d = 0; d < D; ++d) {
      double s = c->sigma_min_frac * c->sigma[d % 3];
      floor_[d] = s * s;
    }
    int64_t* elite = (int64_t*)malloc(sizeof(int64_t) * (size_t)Ke);
    if (c->full_cov && c->mode == ORC_CEM) {
      double* Cn = (double*)malloc(sizeof(double) * (size_t)(D * D));
      double* Ln = (double*)malloc(sizeof(double) * (size_t)(D * D));
      rc = orc_cem_update_full(K, (int32_t)D, J, theta, Ke, floor_, mu_new, Cn, Ln, elite, &out->diag);
      if (rc == ORC_OK) {
        for (int64_t d = 0; d < D; ++d) var_new[d] = Cn[d * D + d];
        memcpy(st->chol, Ln, sizeof(double) * (size_t)(D * D));
      }
      free(Cn);
      free(Ln);
    } else {
      rc = orc_cem_update(K, (int32_t)D, J, theta, Ke, floor_, c->mode == ORC_CEM, mu_new, var_new, elite, &out->diag);
    }
    if (elite_out && rc >= 0) memcpy(elite_out, elite, sizeof(int64_t) * (size_t)Ke);
    argmin = elite[0];
    free(elite);
  }
  if (rc < 0) { free(theta); free(J); free(fidx); return out->status = rc; }
  if (rc == ORC_WARN_ALL_DIVERGED) {               /* L27: keep the distribution */
    memcpy(mu_new, st->mean, sizeof(double) * (size_t)D);
    memcpy(var_new, st->var, sizeof(double) * (size_t)D);
    out->freq_idx = st->freq_idx;
  } else {
    out->freq_idx = fidx[argmin];                  /* L16: theta1 of the best sample */
  }
  out->freq_hz = c->freq_hz[out->freq_idx];

  /* first control: knot 0 of the new mean, masked by delta_0 and projected */
  int32_t d0[4];
  const uint64_t thr = orc_stance_threshold(c->duty_factor);
  for (int i = 0; i < 4; ++i) {
    uint32_t off = (uint32_t)(uint64_t)llround(c->phase_offset[i] * 4294967296.0);
    d0[i] = ((uint64_t)(uint32_t)(phase0 + off) < thr) ? 1 : 0;
    out->contact0[i] = d0[i];
    if (d0[i]) {
      double pen;
      orc_cone(c, &mu_new[3 * i], &out->u0[3 * i], &pen); /* knot 0: d = i*3 + axis */
    } else {
      out->u0[3 * i] = out->u0[3 * i + 1] = out->u0[3 * i + 2] = 0.0;
    }
  }
  if (J_out) memcpy(J_out, J, sizeof(double) * (size_t)K);
  if (fidx_out) memcpy(fidx_out, fidx, sizeof(int32_t) * (size_t)K);
  if (theta_out) memcpy(theta_out, theta, sizeof(double) * (size_t)(K * D));
  memcpy(st->mean, mu_new, sizeof(double) * (size_t)D);
  memcpy(st->var, var_new, sizeof(double) * (size_t)D);
  st->freq_idx = out->freq_idx;
  st->iter += 1;
  free(theta); free(J); free(fidx);
  return out->status = rc;
}

/* ======================================================================
 * the closed loop around one iteration (readings L36-L40).
 * The MPC output drives an SRBD plant for one control period; the gait
 * phase advances at the chosen step frequency; the foothold reference
 * generator (Eq. 3) places the next footholds; the state
 * reference is rebuilt from the command (L13).  Order as in P:212 / P:313:
 * apply u0 -> plant -> leg framework -> next MPC iteration.
 * ==================================================================== */

/* Eq. 3: p_f = p_hip + T_st/2 v_d + sqrt(p_cz / g) (v_c - v_d),
 * horizontal components, z snapped to the flat terrain (L38). */
void orc_foothold(const double p_hip[3], const double v_c[3], const double v_d[3], double p_cz,
                  double t_st, double g, double p_f[3]) {
  const double k = sqrt(fmax(p_cz, 0.0) / g);
  for (int a = 0; a < 2; ++a) p_f[a] = p_hip[a] + 0.5 * t_st * v_d[a] + k * (v_c[a] - v_d[a]);
  p_f[2] = 0.0;
}

/* Eq. 1 with an external wrench at the CoM (L36): force F_e and torque tau_e,
 * both world frame ("wrenches ... applied to the robot CoM"):
 * v_dot += F_e / m,  omega_dot += I^-1 R^T tau_e. */
void orc_plant_dynamics(const orc_config* c, const double x[12], const double gamma[12],
                        const int32_t stance[4], const double feet[12], const double wrench[6],
                        double xd[12]) {
  orc_dynamics(c, x, gamma, stance, feet, xd);
  const double phi = x[6], th = x[7], psi = x[8];
  const double cr = cos(phi), sr = sin(phi), cp = cos(th), sp = sin(th), cy = cos(psi), sy = sin(psi);
  const double Rz[9] = {cy, -sy, 0, sy, cy, 0, 0, 0, 1};
  const double Ry[9] = {cp, 0, sp, 0, 1, 0, -sp, 0, cp};
  const double Rx[9] = {1, 0, 0, 0, cr, -sr, 0, sr, cr};
  double Rzy[9], R[9], tb[3], Iinv[9], wd[3];
  mat3_mul(Rz, Ry, Rzy);
  mat3_mul(Rzy, Rx, R);
  mat3T_vec(R, &wrench[3], tb);
  mat3_inv(c->inertia, Iinv);
  mat3_vec(Iinv, tb, wd);
  for (int a = 0; a < 3; ++a) {
    xd[3 + a] += wrench[a] / c->mass;
    xd[9 + a] += wd[a];
  }
}

/* one control period of the plant: classic RK4, u and wrench held (L36) */
void orc_plant_step(const orc_config* c, const double x[12], const double gamma[12],
                    const int32_t stance[4], const double feet[12], const double wrench[6], double h,
                    double xn[12]) {
  double k1[12], k2[12], k3[12], k4[12], t[12];
  orc_plant_dynamics(c, x, gamma, stance, feet, wrench, k1);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + 0.5 * h * k1[a];
  orc_plant_dynamics(c, t, gamma, stance, feet, wrench, k2);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + 0.5 * h * k2[a];
  orc_plant_dynamics(c, t, gamma, stance, feet, wrench, k3);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + h * k3[a];
  orc_plant_dynamics(c, t, gamma, stance, feet, wrench, k4);
  for (int a = 0; a < 12; ++a) xn[a] = x[a] + h / 6.0 * (k1[a] + 2.0 * k2[a] + 2.0 * k3[a] + k4[a]);
}

/* L13: x^r_j = (p_xy + v_d j dt, h_nom | v_d | 0, 0, psi + yaw_rate j dt | 0, 0, yaw_rate) */
void orc_reference(const orc_config* c, double h_nom, const double x[12], const double v_d[3],
                   double yaw_rate, double* xref) {
  for (int j = 0; j < c->horizon; ++j) {
    double* r = &xref[12 * j];
    const double t = (double)j * c->dt;
    r[0] = x[0] + v_d[0] * t;
    r[1] = x[1] + v_d[1] * t;
    r[2] = h_nom;
    r[3] = v_d[0];
    r[4] = v_d[1];
    r[5] = v_d[2];
    r[6] = 0.0;
    r[7] = 0.0;
    r[8] = x[8] + yaw_rate * t;
    r[9] = 0.0;
    r[10] = 0.0;
    r[11] = yaw_rate;
  }
}

/* the whole advance of one robot (L36-L40); returns the fall flag (L40) */
int orc_advance(const orc_config* c, const orc_loop_config* lc, const double x0[12], uint32_t phase0,
                const double feet_cur[12], const double feet_next[12], const double u0[12],
                const int32_t contact0[4], int32_t freq_idx, const double v_d[3], double yaw_rate,
                const double wrench[6], double x_out[12], uint32_t* phase_out, double feet_cur_out[12],
                double feet_next_out[12], double* xref_out) {
  /* 1. plant: u0 held over dt on the stance legs, lever arms on feet_cur (L36) */
  orc_plant_step(c, x0, u0, contact0, feet_cur, wrench, c->dt, x_out);
  /* 2. fall criterion (L40) */
  int fallen = 0;
  for (int a = 0; a < 12; ++a) fallen |= !isfinite(x_out[a]);
  fallen |= fabs(x_out[6]) > lc->fall_angle || fabs(x_out[7]) > lc->fall_angle || x_out[2] < lc->fall_height;
  /* 3. gait phase at the chosen step frequency (L37) */
  const double f = c->freq_hz[freq_idx];
  *phase_out = phase0 + orc_phase_inc(f, c->dt);
  /* 4. touchdown: a leg that was in swing and is now in stance lands on its planned foothold (L38) */
  const uint64_t thr = orc_stance_threshold(c->duty_factor);
  for (int i = 0; i < 4; ++i) {
    const uint32_t off = (uint32_t)(uint64_t)llround(c->phase_offset[i] * 4294967296.0);
    const int st_new = ((uint64_t)(uint32_t)(*phase_out + off) < thr);
    const int land = !contact0[i] && st_new;
    for (int a = 0; a < 3; ++a) feet_cur_out[3 * i + a] = land ? feet_next[3 * i + a] : feet_cur[3 * i + a];
  }
  /* 5. next footholds, Eq. 3 with T_st = D_f / f_s at the new state */
  const double t_st = c->duty_factor / f;
  const double g = fabs(c->gravity[2]);
  const double cy = cos(x_out[8]), sy = sin(x_out[8]);
  const double v_c[3] = {x_out[3], x_out[4], 0.0};
  for (int i = 0; i < 4; ++i) {
    const double* hp = &lc->hip[3 * i];
    const double p_hip[3] = {x_out[0] + cy * hp[0] - sy * hp[1], x_out[1] + sy * hp[0] + cy * hp[1], 0.0};
    orc_foothold(p_hip, v_c, v_d, x_out[2], t_st, g, &feet_next_out[3 * i]);
  }
  /* 6. reference rebuilt from the command at the new state (L13) */
  if (xref_out) orc_reference(c, lc->h_nom, x_out, v_d, yaw_rate, xref_out);
  return fallen;
}
