/*
 * opcount.cpp -- op-counting mode of the oracle ("freeze the
 * exact number by running the oracle in op-counting mode over the config-2
 * workload").
 *
 * TEST / MEASUREMENT INFRASTRUCTURE ONLY (see sbs_oracle.c).  It compiles the
 * unchanged oracle source sbs_oracle.c a second time, inside namespace cnt, with
 * every `double` replaced by a counting scalar CD, and exports one entry point,
 * orc_count_rollout(), that runs orc_rollout (Alg. 2, with the policy
 * of Alg. 5, and the cost of P:342-351) on one sample and returns
 * the number of arithmetic operations it performed.  Nothing here is on the
 * product path; the CUDA library never sees it.
 *
 * What is counted (the roofline's "algorithmic FLOPs"):
 *   * values are tagged "varying" when they depend on the sample: the sample
 *     theta2 and the rollout state, starting from x0 (the state every rollout
 *     carries).  Config constants, the reference trajectory, the feet, the spline
 *     weights and the contact schedule are not varying; the reference and the
 *     feet are tagged "input data" (never treated as an identity operand);
 *   * every binary64 +, -, *, / with at least one varying operand is one FLOP
 *     (the oracle is built with -ffp-contract=off, so an FMA is two), except
 *     identities with a constant (config or code literal) exact operand: x + 0, x - 0, 0 - x (a
 *     negation), x * 0 (gives a non-varying 0), x * 1, x * -1, x / 1, which no
 *     implementation executes (the zero / one entries of the elementary rotation
 *     matrices, the zero off-diagonal inertia entries, g_x = g_y = 0);
 *   * ops with only non-varying operands are hoistable constants (I^-1, the
 *     Catmull-Rom weights, m g / n, the Q0.32 schedule) and are not counted;
 *   * sin, cos, tan, exp, sqrt, remainder of a varying argument are counted
 *     separately ("transcendental"), comparisons / min / max / abs separately
 *     ("compare"); neither is a FLOP.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>

#include "sbs_oracle.h"  /* the binary64 declarations, for the exported wrapper */

namespace cnt {

struct Counts {
  uint64_t flop, trans, cmp;
};
static Counts g_cnt;

/* binary32 counting scalar for the noise recipe (O3-O4): values converted from the
 * Philox words (integers) depend on the sample; float literals are constants. */
struct CF {
  float v;
  int32_t var;
  CF() : v(0.0f), var(1) {}  /* filled by memcpy from a Philox word (f32_from_bits) */
  CF(float x) : v(x), var(0) {}
  CF(double x) : v((float)x), var(0) {}
  CF(int x) : v((float)x), var(1) {}
  CF(unsigned x) : v((float)x), var(1) {}
  static CF mk(float x, int vr) {
    CF r(x);
    r.var = vr;
    return r;
  }
};
static inline int joinf(const CF& a, const CF& b) { return (a.var == 1 || b.var == 1) ? 1 : (a.var | b.var); }
#define CNT_FOP(op)                                          \
  static inline CF operator op(const CF& a, const CF& b) {   \
    const int vr = joinf(a, b);                              \
    if (vr == 1) ++g_cnt.flop;                               \
    return CF::mk(a.v op b.v, vr);                           \
  }
CNT_FOP(+)
CNT_FOP(-)
CNT_FOP(*)
CNT_FOP(/)
#undef CNT_FOP
static inline CF operator-(const CF& a) { return CF::mk(-a.v, a.var); }
#define CNT_FCMP(op)                                         \
  static inline bool operator op(const CF& a, const CF& b) { \
    if (joinf(a, b) == 1) ++g_cnt.cmp;                       \
    return a.v op b.v;                                       \
  }
CNT_FCMP(<)
CNT_FCMP(>)
#undef CNT_FCMP
static inline CF fmaf(const CF& a, const CF& b, const CF& c) {
  const int vr = (a.var == 1 || b.var == 1 || c.var == 1) ? 1 : (a.var | b.var | c.var);
  if (vr == 1) g_cnt.flop += 2;
  return CF::mk(std::fma(a.v, b.v, c.v), vr);
}
static inline CF sqrtf(const CF& a) {
  if (a.var == 1) ++g_cnt.trans;
  return CF::mk(std::sqrt(a.v), a.var);
}

struct CD {
  double v;
  int32_t var;  /* 0: constant (config, code literal), 1: depends on the sample, 2: input data */
  int32_t pad_;
  CD() = default;
  CD(double x) : v(x), var(0), pad_(0) {}
  CD(const CF& f) : v((double)f.v), var(f.var), pad_(0) {}
  static CD mk(double x, int vr) {
    CD r(x);
    r.var = vr;
    return r;
  }
};
static inline bool is_c(const CD& a, double k) { return a.var == 0 && a.v == k; }
static inline int join(const CD& a, const CD& b) { return (a.var == 1 || b.var == 1) ? 1 : (a.var | b.var); }
static inline bool counted(int vr) { return vr == 1; }

static inline CD operator+(const CD& a, const CD& b) {
  if (is_c(b, 0.0)) return a;
  if (is_c(a, 0.0)) return b;
  const int vr = join(a, b);
  if (counted(vr)) ++g_cnt.flop;
  return CD::mk(a.v + b.v, vr);
}
static inline CD operator-(const CD& a) { return CD::mk(-a.v, a.var); }
static inline CD operator-(const CD& a, const CD& b) {
  if (is_c(b, 0.0)) return a;
  if (is_c(a, 0.0)) return -b;
  const int vr = join(a, b);
  if (counted(vr)) ++g_cnt.flop;
  return CD::mk(a.v - b.v, vr);
}
static inline CD operator*(const CD& a, const CD& b) {
  if (is_c(a, 0.0) || is_c(b, 0.0)) return CD(a.v * b.v);
  if (is_c(a, 1.0)) return b;
  if (is_c(b, 1.0)) return a;
  if (is_c(a, -1.0)) return -b;
  if (is_c(b, -1.0)) return -a;
  const int vr = join(a, b);
  if (counted(vr)) ++g_cnt.flop;
  return CD::mk(a.v * b.v, vr);
}
static inline CD operator/(const CD& a, const CD& b) {
  if (is_c(b, 1.0)) return a;
  if (is_c(a, 0.0)) return CD(a.v / b.v);
  const int vr = join(a, b);
  if (counted(vr)) ++g_cnt.flop;
  return CD::mk(a.v / b.v, vr);
}
static inline CD& operator+=(CD& a, const CD& b) { return a = a + b; }
static inline CD& operator-=(CD& a, const CD& b) { return a = a - b; }
static inline CD& operator*=(CD& a, const CD& b) { return a = a * b; }
static inline CD& operator/=(CD& a, const CD& b) { return a = a / b; }

#define CNT_CMP(op)                                          \
  static inline bool operator op(const CD& a, const CD& b) { \
    if (join(a, b) == 1) ++g_cnt.cmp;                        \
    return a.v op b.v;                                       \
  }
CNT_CMP(<)
CNT_CMP(>)
CNT_CMP(<=)
CNT_CMP(>=)
CNT_CMP(==)
CNT_CMP(!=)
#undef CNT_CMP

#define CNT_T1(fn)                       \
  static inline CD fn(const CD& a) {     \
    if (a.var == 1) ++g_cnt.trans;       \
    return CD::mk(std::fn(a.v), a.var);  \
  }
CNT_T1(sin)
CNT_T1(cos)
CNT_T1(tan)
CNT_T1(exp)
CNT_T1(sqrt)
#undef CNT_T1
static inline CD remainder(const CD& a, const CD& b) {
  if (join(a, b) == 1) ++g_cnt.trans;
  return CD::mk(std::remainder(a.v, b.v), join(a, b));
}
static inline CD fabs(const CD& a) {
  if (a.var == 1) ++g_cnt.cmp;
  return CD::mk(std::fabs(a.v), a.var);
}
static inline CD fmax(const CD& a, const CD& b) {
  if (join(a, b) == 1) ++g_cnt.cmp;
  return CD::mk(std::fmax(a.v, b.v), join(a, b));
}
static inline CD fmin(const CD& a, const CD& b) {
  if (join(a, b) == 1) ++g_cnt.cmp;
  return CD::mk(std::fmin(a.v, b.v), join(a, b));
}
static inline bool isfinite(const CD& a) { return std::isfinite(a.v); }
static inline bool isnan(const CD& a) { return std::isnan(a.v); }
static inline long long llround(const CD& a) { return std::llround(a.v); }

#undef SBS_ORACLE_H
#define double CD
#define float CF
#include "sbs_oracle.c"
#undef float
#undef double

}  // namespace cnt

/* the binary64 config as the counting build's config (field by field) */
static void to_counting(const orc_config* c, cnt::orc_config& k) {
  memset(&k, 0, sizeof k);
  k.mass = c->mass;
  for (int i = 0; i < 9; ++i) k.inertia[i] = c->inertia[i];
  for (int i = 0; i < 3; ++i) k.gravity[i] = c->gravity[i];
  k.mu = c->mu, k.fz_min = c->fz_min, k.fz_max = c->fz_max;
  k.horizon = c->horizon, k.knots = c->knots, k.dt = c->dt;
  k.duty_factor = c->duty_factor;
  for (int i = 0; i < 4; ++i) k.phase_offset[i] = c->phase_offset[i];
  k.n_freq = c->n_freq, k.gait_adapt = c->gait_adapt;
  for (int i = 0; i < ORC_MAX_FREQ; ++i) k.freq_hz[i] = c->freq_hz[i];
  for (int i = 0; i < 12; ++i) k.Q[i] = c->Q[i], k.R[i] = c->R[i];
  k.rho = c->rho, k.f_nominal = c->f_nominal, k.w_fc = c->w_fc;
  k.mode = c->mode, k.elite_preserve = c->elite_preserve;
  k.n_samples = c->n_samples, k.n_elite = c->n_elite, k.lambda = c->lambda;
  for (int i = 0; i < 3; ++i) k.sigma[i] = c->sigma[i];
  k.sigma_min_frac = c->sigma_min_frac;
  k.warm_shift = c->warm_shift, k.seed = c->seed;
  k.n_sigma_groups = c->n_sigma_groups;
  for (int i = 0; i < 8; ++i) k.sigma_scale[i] = c->sigma_scale[i];
  k.full_cov = c->full_cov;
}

/* Run orc_rollout on one sample with counting scalars.  Arguments as orc_rollout
 * (sbs_oracle.h) plus counts[3] = {FLOPs, transcendentals, compares}; returns J. */
extern "C" double orc_count_rollout(const orc_config* c, const double x0[12], uint32_t phase0,
                                    const double feet_cur[12], const double feet_next[12],
                                    const double* xref, const double* theta, int32_t fidx,
                                    uint64_t counts[3]) {
  using cnt::CD;
  cnt::orc_config k;
  to_counting(c, k);
  const int H = c->horizon, D = 12 * c->knots;
  CD X0[12], FC[12], FN[12];
  for (int a = 0; a < 12; ++a) {
    X0[a] = CD::mk(x0[a], 1);  /* the rollout state */
    FC[a] = CD::mk(feet_cur[a], 2);  /* input data: a zero entry is not an identity */
    FN[a] = CD::mk(feet_next[a], 2);
  }
  CD* XR = (CD*)malloc(sizeof(CD) * (size_t)H * 12);
  CD* TH = (CD*)malloc(sizeof(CD) * (size_t)D);
  for (int a = 0; a < H * 12; ++a) XR[a] = CD::mk(xref[a], 2);
  for (int d = 0; d < D; ++d) TH[d] = CD::mk(theta[d], 1);  /* the sample */
  cnt::g_cnt = cnt::Counts{0, 0, 0};
  const CD J = cnt::orc_rollout(&k, X0, phase0, FC, FN, XR, TH, fidx, nullptr);
  counts[0] = cnt::g_cnt.flop;
  counts[1] = cnt::g_cnt.trans;
  counts[2] = cnt::g_cnt.cmp;
  free(XR);
  free(TH);
  return J.v;
}

/* Sampling of one sample (O1-O6: Philox words -> binary32 Box-Muller -> theta2 =
 * mu' + sigma z): counts of the noise recipe's binary32 operations and the theta2
 * formation.  theta[D] receives the sample (equal to orc_sample's). */
extern "C" void orc_count_sample(const orc_config* c, const double* mu_shift, const double* var,
                                 int32_t cur_idx, uint32_t iter, uint32_t robot, int64_t kk,
                                 double* theta, uint64_t counts[3]) {
  using cnt::CD;
  cnt::orc_config k;
  to_counting(c, k);
  const int D = 12 * c->knots;
  CD MU[ORC_MAX_D] = {}, VA[ORC_MAX_D] = {}, TH[ORC_MAX_D] = {};
  cnt::CF Z[ORC_MAX_D];
  for (int d = 0; d < D; ++d) MU[d] = CD::mk(mu_shift[d], 2), VA[d] = CD::mk(var[d], 2);
  int32_t idx;
  cnt::g_cnt = cnt::Counts{0, 0, 0};
  cnt::orc_sample(&k, MU, VA, cur_idx, iter, robot, kk, TH, Z, &idx);
  counts[0] = cnt::g_cnt.flop;
  counts[1] = cnt::g_cnt.trans;
  counts[2] = cnt::g_cnt.cmp;
  for (int d = 0; d < D; ++d) theta[d] = TH[d].v;
}

/* MPPI update over K samples (O13): counts; mu_new[D] receives the new mean. */
extern "C" int orc_count_mppi(int64_t K, int32_t D, const double* J, const double* theta, double lambda,
                              double* mu_new, uint64_t counts[3]) {
  using cnt::CD;
  CD* JJ = (CD*)malloc(sizeof(CD) * (size_t)K);
  CD* TH = (CD*)malloc(sizeof(CD) * (size_t)(K * D));
  CD MU[ORC_MAX_D];
  for (int64_t k = 0; k < K; ++k) JJ[k] = CD::mk(J[k], 1);
  for (int64_t i = 0; i < K * D; ++i) TH[i] = CD::mk(theta[i], 1);
  cnt::orc_diag dg;
  cnt::g_cnt = cnt::Counts{0, 0, 0};
  const int rc = cnt::orc_mppi(K, D, JJ, TH, CD(lambda), MU, &dg);
  counts[0] = cnt::g_cnt.flop;
  counts[1] = cnt::g_cnt.trans;
  counts[2] = cnt::g_cnt.cmp;
  for (int d = 0; d < D; ++d) mu_new[d] = MU[d].v;
  free(JJ);
  free(TH);
  return rc;
}
