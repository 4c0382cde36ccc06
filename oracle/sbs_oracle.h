/*
 * sbs_oracle.h -- CPU oracle for one SBS MPC iteration (arxiv 2403.11383).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path under paper_2403_11383_b200/csrc; neither includes the other.
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * SPEC.md, "Ln" = a reading listed in DESIGN.md section 3 (the paper is
 * silent or garbled there).  Arithmetic is IEEE binary64 except the
 * normative binary32 noise recipe, which both sides
 * implement independently so that the sampled noise is bit-identical.
 */
#ifndef SBS_ORACLE_H
#define SBS_ORACLE_H
#include <stdint.h>

#define ORC_MAX_KNOTS 8
#define ORC_MAX_D (12 * ORC_MAX_KNOTS)
#define ORC_MAX_FREQ 8
#define ORC_NX 12

enum { ORC_MPPI = 0, ORC_CEM = 1, ORC_NAIVE = 2 };
enum {
  ORC_OK = 0,
  ORC_WARN_ALL_DIVERGED = 1,
  ORC_ERR_INVALID_ARG = -1,
  ORC_ERR_SINGULAR = -2,
  ORC_ERR_NONFINITE = -3
};

typedef struct orc_config {
  /* robot model, Eq. 1; values are reading L29 */
  double mass, inertia[9], gravity[3];
  double mu, fz_min, fz_max; /* friction cone */
  /* horizon and GRF spline */
  int32_t horizon, knots;
  double dt;
  /* gait */
  double duty_factor, phase_offset[4];
  int32_t n_freq, gait_adapt;
  double freq_hz[ORC_MAX_FREQ];
  /* cost */
  double Q[12], R[12], rho, f_nominal, w_fc;
  /* optimizer */
  int32_t mode, elite_preserve;
  int64_t n_samples, n_elite;
  double lambda;
  double sigma[3], sigma_min_frac;
  int32_t warm_shift, _pad;
  uint64_t seed;
  /* multiple Gaussians: sample k draws with std sigma_scale[k mod n_sigma_groups] * sigma */
  int32_t n_sigma_groups, _pad2;
  double sigma_scale[8];
  /* full-covariance CEM (Alg. 1 UpdateCov with a full C; L42) */
  int32_t full_cov, _pad3;
} orc_config;

typedef struct orc_diag {
  double j_min, j_mean, omega, ess;
  int64_t n_diverged, argmin;
} orc_diag;

/* ---- O1-O4: noise ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float orc_ln_u24(uint32_t w);                   /* ln(u1), u1 = (2(w>>9)+1) 2^-24  */
void orc_sincos_2pi_u(uint32_t w, float* s, float* c); /* sin/cos(2 pi u2)        */
void orc_normal4(const uint32_t w[4], float z[4]);      /* Box-Muller, 2 pairs     */
void orc_normal4_batch(const uint32_t* w /*[n][4]*/, int64_t n, float* z /*[n][4]*/);

/* ---- O5-O6: one sample theta_k = [theta1, theta2] ---- */
void orc_sample(const orc_config* c, const double* mu_shift, const double* var,
                int32_t cur_idx, uint32_t iter, uint32_t robot, int64_t k,
                double* theta, float* z, int32_t* idx);

/* ---- a0: warm start ---- */
void orc_warm_shift(const orc_config* c, const double* mu, double* mu_shift);

/* ---- O7: contact sequence ---- */
uint32_t orc_phase_inc(double f_hz, double dt);
uint64_t orc_stance_threshold(double duty_factor);
void orc_contact_sequence(const orc_config* c, uint32_t phase0, double f_hz, int32_t* delta /*[H][4]*/);

/* ---- O8: Catmull-Rom GRF spline ---- */
void orc_spline_eval(int32_t P, const double* knots_ch /*[P]*/, int64_t a_num, int64_t a_den, double* out);
void orc_spline_step(const orc_config* c, const double* theta, int32_t j, double gamma[12]);

/* ---- O9: friction cone ---- */
void orc_cone(const orc_config* c, const double raw[3], double out[3], double* pen);

/* ---- O10-O11: SRBD dynamics Eq. 1 and RK4 ---- */
void orc_dynamics(const orc_config* c, const double x[12], const double gamma[12],
                  const int32_t stance[4], const double feet[12], double xdot[12]);
void orc_rk4(const orc_config* c, const double x[12], const double gamma[12],
             const int32_t stance[4], const double feet[12], double h, double xn[12]);

/* ---- O12: rollout and cost, Alg. 2 ---- */
double orc_rollout(const orc_config* c, const double x0[12], uint32_t phase0,
                   const double feet_cur[12], const double feet_next[12],
                   const double* xref /*[H][12]*/, const double* theta, int32_t fidx,
                   double* traj /*[H+1][12] or NULL*/);

/* ---- O13-O14: distribution update, Alg. 3/4 and Alg. 1 ---- */
int orc_mppi(int64_t K, int32_t D, const double* J, const double* theta /*[K][D]*/,
             double lambda, double* mu_new, orc_diag* dg);
int orc_cem_select(int64_t K, const double* J, int64_t K_e, int64_t* elite /*[K_e]*/);
int orc_cem_update(int64_t K, int32_t D, const double* J, const double* theta,
                   int64_t K_e, const double* var_floor, int32_t update_var,
                   double* mu_new, double* var_new, int64_t* elite, orc_diag* dg);

/* ---- full covariance (f3; L42) ---- */
int orc_cholesky(int32_t D, const double* C /*[D][D]*/, double* L /*[D][D], lower*/);
void orc_sample_full(const orc_config* c, const double* mu_shift, const double* L /*[D][D]*/,
                     int32_t cur_idx, uint32_t iter, uint32_t robot, int64_t k,
                     double* theta, float* z, int32_t* idx);
int orc_cem_update_full(int64_t K, int32_t D, const double* J, const double* theta, int64_t K_e,
                        const double* var_floor, double* mu_new, double* C_new /*[D][D]*/,
                        double* L_new /*[D][D]*/, int64_t* elite, orc_diag* dg);

/* ---- whole iteration, Alg. 5 ---- */
typedef struct orc_state {
  double mean[ORC_MAX_D], var[ORC_MAX_D];
  int32_t freq_idx;
  uint32_t iter;
  double chol[ORC_MAX_D * ORC_MAX_D]; /* full_cov: lower Cholesky factor L of C, row-major [D][D]; var = diag(C) */
} orc_state;

typedef struct orc_output {
  double u0[12];
  int32_t contact0[4];
  int32_t freq_idx, status;
  double freq_hz;
  orc_diag diag;
} orc_output;

int orc_step(const orc_config* c, uint32_t robot, const double x0[12], uint32_t phase0,
             const double feet_cur[12], const double feet_next[12], const double* xref,
             orc_state* st, orc_output* out,
             double* J_out /*[K] or NULL*/, int32_t* fidx_out /*[K] or NULL*/,
             double* theta_out /*[K][D] or NULL*/, float* z_out /*[K][D] or NULL*/,
             int64_t* elite_out /*[K_e] or NULL*/);
/* ---- closed loop around the iteration (L36-L40) ---- */
typedef struct orc_loop_config {
  double hip[12];               /* body-frame hip offsets FL, FR, RL, RR (L29); z ignored */
  double h_nom;                 /* nominal CoM height of the rebuilt reference (L13) */
  double fall_angle, fall_height; /* fallen iff |roll| or |pitch| > fall_angle or p_z < fall_height (L40) */
} orc_loop_config;

void orc_foothold(const double p_hip[3], const double v_c[3], const double v_d[3], double p_cz,
                  double t_st, double g, double p_f[3]);                  /* Eq. 3 */
void orc_plant_dynamics(const orc_config* c, const double x[12], const double gamma[12],
                        const int32_t stance[4], const double feet[12], const double wrench[6],
                        double xd[12]);
void orc_plant_step(const orc_config* c, const double x[12], const double gamma[12],
                    const int32_t stance[4], const double feet[12], const double wrench[6], double h,
                    double xn[12]);
void orc_reference(const orc_config* c, double h_nom, const double x[12], const double v_d[3],
                   double yaw_rate, double* xref /*[H][12]*/);
int orc_advance(const orc_config* c, const orc_loop_config* lc, const double x0[12], uint32_t phase0,
                const double feet_cur[12], const double feet_next[12], const double u0[12],
                const int32_t contact0[4], int32_t freq_idx, const double v_d[3], double yaw_rate,
                const double wrench[6], double x_out[12], uint32_t* phase_out, double feet_cur_out[12],
                double feet_next_out[12], double* xref_out /*[H][12] or NULL*/);
#endif
