/*
 * sbs.h -- C ABI of the B200-native (sm_100a) hot path of one MPC iteration
 * of the Sample-Based Stochastic (SBS) quadruped controller, arxiv 2403.11383.
 *
 * Citations: "P:n" = line n of the paper text, "Ln" = reading n in
 * DESIGN.md sec. 3, "S:n" = SPEC.md line n (interface ideas only).
 *
 * The operation (Alg. 5): given the current state estimate x0 and
 * the search distribution N(theta, C), draw K samples theta_k = [theta1,
 * theta2] (gait-frequency index, GRF spline knots), roll each out over the
 * SRBD model (Eq. 1) for H steps while accumulating the cost of
 * P:342-351, and reduce the samples into the next distribution by MPPI
 * (Alg. 4) or by elite selection (CEM = Alg. 1 with K_e elites and
 * a diagonal or, with full_cov, a full covariance refit; Naive = Alg. 3,
 * K_e = 1, C unchanged).  The
 * updated mean is the control: its first knot, masked by the contact
 * flags and projected onto the friction cone, is returned as u0.
 *
 * Conventions
 *  - Every function returns an sbs_status (int) unless stated otherwise.
 *  - Ownership: the context owns all device memory it allocates.  The caller
 *    owns every buffer it passes; the library never retains a caller pointer
 *    after the call returns (device pointers passed to *_device calls must
 *    stay valid until the work enqueued on `stream` has completed).
 *  - Host pointers are plain CPU memory (pinned or pageable).  Device
 *    pointers are CUDA global memory on cfg.device (e.g. torch tensors'
 *    data_ptr()).  `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Errors: on any negative status the distribution state (mean, var,
 *    freq_idx) and the iteration counter are unchanged; sbs_last_error()
 *    returns a message.  A diverged rollout is never an error: its cost is
 *    +inf (L26).
 *  - Threading: a context is used by one host thread at a time.  With
 *    world > 1 every rank calls sbs_step* collectively, in the same order.
 *  - Layouts: states are x = (p_c[3], v_c[3], (roll, pitch, yaw), w_body[3])
 *    (P:277, L24); legs are ordered FL, FR, RL, RR; knot vectors use
 *    d = (p*4 + leg)*3 + axis, D = 12*P (L6).  All reals are IEEE binary32.
 */
#ifndef SBS_H
#define SBS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBS_VERSION 1
#define SBS_MAX_KNOTS 8
#define SBS_MAX_D (12 * SBS_MAX_KNOTS)
#define SBS_MAX_FREQ 8
#define SBS_MAX_HORIZON 64
#define SBS_NX 12

typedef struct sbs_ctx sbs_ctx; /* opaque */

typedef enum {
  SBS_MPPI = 0,  /* Alg. 4: beta = min J, w = exp(-(J-beta)/lambda), weighted mean; C unchanged */
  SBS_CEM = 1,   /* Alg. 1: K_e elites by (J, k); elite mean; diagonal elite variance, floored (L17) */
  SBS_NAIVE = 2  /* Alg. 3: best sample is the new mean; C unchanged (K_e forced to 1)           */
} sbs_mode;

typedef enum {
  SBS_OK = 0,
  SBS_WARN_ALL_DIVERGED = 1, /* every rollout of some robot was +inf: its distribution is kept (L27) */
  SBS_ERR_INVALID_ARG = -1,  /* NULL pointer, bad index/size, or a config invariant violated */
  SBS_ERR_SINGULAR = -2,     /* |pitch(x0)| >= pi/2 - 1e-3 (Euler-rate map singular, L26) */
  SBS_ERR_NONFINITE = -3,    /* non-finite x0 / feet / reference */
  SBS_ERR_STATE = -4,        /* call out of order (e.g. step before every robot has a reference) */
  SBS_ERR_CUDA = -5,         /* CUDA runtime error (message in sbs_last_error) */
  SBS_ERR_NCCL = -6,         /* NCCL error or NCCL unavailable while world > 1 */
  SBS_ERR_OOM = -7           /* device allocation failed */
} sbs_status;

/* Configuration, validated by sbs_create (invariants after each field). */
typedef struct sbs_config {
  /* robot model, Eq. 1; values per L29 */
  float mass;             /* kg, > 0 */
  float inertia[9];       /* body-frame inertia, row-major, symmetric positive definite */
  float gravity[3];       /* world frame, m/s^2; gravity[2] < 0 */
  float mu;               /* friction coefficient, > 0 */
  float fz_min, fz_max;   /* normal-force bounds, 0 <= fz_min < fz_max */
  /* horizon and GRF spline */
  int32_t horizon;        /* H, 1..SBS_MAX_HORIZON */
  int32_t knots;          /* P, 2..SBS_MAX_KNOTS */
  float dt;               /* s, > 0 */
  /* gait (L15, L22) */
  float duty_factor;      /* D_f in (0, 1] */
  float phase_offset[4];  /* per-leg phase offsets in [0, 1) */
  int32_t n_freq;         /* number of step-frequency options, 1..SBS_MAX_FREQ */
  int32_t gait_adapt;     /* 1: theta1 sampled uniformly per sample; 0: current index kept */
  float freq_hz[SBS_MAX_FREQ]; /* strictly increasing, > 0 */
  /* cost (L9-L14) */
  float Q[12];            /* diagonal state weights, >= 0 */
  float R[12];            /* diagonal force weights per leg*3+axis, >= 0 */
  float rho;              /* frequency regularisation weight, >= 0 */
  float f_nominal;        /* theta1 reference f_s^n, Hz */
  float w_fc;             /* friction-cone violation penalty weight, >= 0 */
  /* optimiser */
  int32_t mode;           /* sbs_mode */
  int32_t elite_preserve; /* 1: sample 0 is the (shifted) mean with the current theta1 (L21) */
  int64_t n_samples;      /* K per robot, summed over all ranks, 1..2^24 (finite counts are binary32) */
  int64_t n_elite;        /* K_e for SBS_CEM (1..K); ignored for MPPI; forced to 1 for NAIVE */
  float lambda;           /* MPPI temperature, > 0 */
  float sigma[3];         /* initial std per force axis (x, y, z), > 0 (L19) */
  float sigma_min_frac;   /* CEM variance floor = (sigma_min_frac * sigma[axis])^2, >= 0 */
  int32_t warm_shift;     /* 1: shift the previous mean's spline by dt before sampling (L20) */
  uint64_t seed;          /* Philox key (L31) */
  /* batching and placement */
  int32_t n_robots;       /* R >= 1 independent controllers in one context */
  int32_t robot_offset;   /* global index of robot 0 in the noise counter (robot sharding) */
  int32_t device;         /* CUDA device ordinal */
  int32_t rank, world;    /* sample sharding: rank handles a contiguous slice of the K samples */
  uint8_t nccl_id[128];   /* ncclUniqueId (sbs_nccl_unique_id on rank 0) when world > 1; all zero:
                             the caller exchanges the rank records (sbs_step_records).  CEM with
                             world > 1 needs n_elite <= n_samples / world. */
  /* multiple Gaussians ("we sample from multiple Gaussian distributions"; L41): sample k
     draws theta2 = mu' + sigma_scale[k mod n_sigma_groups] * sigma * z (elite-preserved sample 0
     excepted).  n_sigma_groups 0 or 1: one Gaussian (sigma_scale ignored); at most 8; scales >= 0. */
  int32_t n_sigma_groups;
  float sigma_scale[8];
  /* full-covariance CEM (Alg. 1 UpdateCov with a full C; L42): C = L L^T per
     robot, initially diag(sigma^2); theta2 = mu' + L z; C_new = elite covariance + diag(floor), L_new =
     Cholesky(C_new); var reports diag(C).  CEM only, n_sigma_groups <= 1. */
  int32_t full_cov;
} sbs_config;

/* Per-robot input of one iteration (host for sbs_step, device for sbs_step_device). */
typedef struct sbs_input {
  float x0[12];           /* current state estimate (Alg. 5 "Given x0") */
  uint32_t phase_q32;     /* global gait phase, Q0.32 fraction of a cycle (L22) */
  float feet_cur[12];     /* world-frame stance foot positions, 4 x 3 */
  float feet_next[12];    /* next touchdown positions, 4 x 3 (used after a leg's first touchdown, L23) */
  uint32_t _pad[3];
} sbs_input;

/* Per-robot output of one iteration. */
typedef struct sbs_output {
  float u0[12];           /* first control: delta_0-masked cone projection of knot 0 of the new mean */
  uint8_t contact0[4];    /* delta_0 per leg */
  int32_t freq_idx;       /* chosen theta1 (index into freq_hz) */
  float freq_hz;          /* chosen step frequency */
  int32_t status;         /* SBS_OK or SBS_WARN_ALL_DIVERGED for this robot */
  uint32_t iter;          /* iteration counter used for this step's noise */
  float j_min;            /* best cost (beta) */
  float j_mean;           /* mean of the finite costs */
  float omega;            /* MPPI: sum of weights Omega; CEM/Naive: number of elites used */
  float ess;              /* MPPI effective sample size Omega^2 / sum w^2 */
  int32_t n_diverged;     /* rollouts with J = +inf */
  float device_us;        /* device time of the step, CUDA events (sbs_step with sbs_profile on; 0 otherwise) */
  float mean[SBS_MAX_D];  /* new mean theta2 (first D entries valid) */
  float var[SBS_MAX_D];   /* new diagonal covariance */
} sbs_output;

/* Create a context on cfg->device.  Allocates all device state, derives the
 * constant tables (spline weights, Q0.32 gait increments, inverse inertia),
 * sets every robot's distribution to mean = (0, 0, m*|g_z|/4) per leg and
 * knot, var = sigma^2, freq_idx = 0, iter = 0.  With world > 1 joins the NCCL
 * communicator described by cfg->nccl_id (collective over all ranks).
 * Returns SBS_ERR_INVALID_ARG for any violated invariant. */
int sbs_create(const sbs_config* cfg, sbs_ctx** out);
void sbs_destroy(sbs_ctx* ctx);

/* State reference x^r_j, j = 0..H-1 (Alg. 2 "x^r_i"; L13).
 * _reference: one robot, host [H][12]; copied into pinned staging before the
 * call returns (the caller's buffer is free again) and uploaded in order on the
 * context's stream, ahead of the next sbs_step.  _reference_device: all robots,
 * device [R][H][12], copied on `stream`. */
int sbs_set_reference(sbs_ctx* ctx, int32_t robot, const float* x_ref);
int sbs_set_reference_device(sbs_ctx* ctx, const float* d_x_ref, void* stream);

/* Distribution N(theta, C) of one robot (host [D] arrays; var > 0). */
int sbs_set_distribution(sbs_ctx* ctx, int32_t robot, const float* mean, const float* var, int32_t freq_idx);
int sbs_get_distribution(sbs_ctx* ctx, int32_t robot, float* mean, float* var, int32_t* freq_idx);
uint32_t sbs_get_iter(const sbs_ctx* ctx);
int sbs_set_iter(sbs_ctx* ctx, uint32_t iter);

/* One iteration for all R robots.  in/out: host arrays of R entries.
 * Synchronous: outputs are valid on return.  Validates x0 on the host
 * (SBS_ERR_NONFINITE / SBS_ERR_SINGULAR).  Returns SBS_WARN_ALL_DIVERGED if
 * any robot had every rollout diverge.  iter += 1 on OK or WARN.
 * Transport: with R = 1 (and H <= 16) the inputs, the staged reference and the
 * iteration counter travel inside the kernel parameters (direct launch, no
 * copy); otherwise one pinned block [iter | inputs | references] is copied up
 * by a captured CUDA graph.  The finishing kernel writes the outputs straight
 * into the context's mapped pinned memory; they are copied to `out` on return.
 * Completion (R = 1): the finishing CTA raises a mapped flag after its outputs
 * (system-scope fence) and the calling thread spins on it (checking the stream
 * for errors every 1024 polls) instead of synchronising the stream; later work
 * on the context's stream stays stream-ordered behind the step's kernels. */
int sbs_step(sbs_ctx* ctx, const sbs_input* in, sbs_output* out);

/* Same iteration with device-resident inputs/outputs (R entries each),
 * enqueued on `stream`; outputs valid after the stream is synchronised.
 * x0 is not validated on the host: a singular or non-finite x0 makes every
 * rollout of that robot diverge (status SBS_WARN_ALL_DIVERGED in its output).
 * iter += 1 when the call returns SBS_OK. */
int sbs_step_device(sbs_ctx* ctx, const sbs_input* d_in, sbs_output* d_out, void* stream);

/* Sample sharding with a caller-driven exchange (world > 1 and an
 * all-zero nccl_id): the same iteration as sbs_step_device, split at its one
 * exchange point.  sbs_step_records enqueues this rank's rollouts and writes
 * its record per robot to d_rec (device, R x sbs_record_floats(ctx) floats):
 *   MPPI  [beta_g, k_argmin, theta1, sum w, sum w^2, sum J, n finite, 0 | sum w theta[D]]
 *         (weights relative to this rank's beta_g)
 *   Naive [J_min, k_argmin, theta1, 0, 0, sum J, n finite, 0]
 *   CEM   [same 8-float header | J of the rank's K_e smallest (J, k), index order |
 *          their global k as int32 bits], padded to a multiple of 4 floats
 * The caller gathers every rank's records in rank order ([world][R][record])
 * and passes them to sbs_finish_records, which merges them in rank order
 * (MPPI: rescaled sums; Naive: argmin; CEM: exact K_e-smallest selection over
 * the world x K_e candidates, whose rank-order concatenation is in global
 * index order, then elite moments regenerated from the counter RNG) and
 * finishes the iteration (new distribution, d_out); iter += 1.  Both
 * stream-ordered.  With a nonzero nccl_id, sbs_step / sbs_step_device do the
 * same with one ncclAllGather in between.  Noise, costs, elites and (MPPI
 * aside, whose sums regroup) the new distribution are independent of world. */
int sbs_record_floats(const sbs_ctx* ctx);

/* Peer-memory exchange of the rank records (world > 1, one process per GPU of a
 * node, or several contexts in one process), in place of the NCCL all-gather.
 * Each rank calls sbs_peer_handle (its exchange buffer as a CUDA IPC handle, and
 * its device address for same-process use); the caller exchanges them (e.g. a
 * torch.distributed all_gather_object) and calls sbs_peer_connect with either the
 * addresses (same process; peer access is enabled) or the IPC handles [world][64].
 * From then on every sbs_step / sbs_step_device has the rank's last record-writing
 * CTA store the rank's records straight into every peer's buffer (NVLink stores,
 * system-scope fence, then a per-rank flag = exchange sequence number), and the
 * stream waits in the GPU front-end (cuStreamWaitValue32, no SM held) for the
 * peers' flags before the rank-order merge.  Two buffers alternate, so a fast rank
 * never overwrites records a slower peer is still merging.  Collective: every rank
 * steps in the same order.  world <= 8.  sbs_peer_connect(ctx, NULL, NULL)
 * disconnects (back to the NCCL or caller-driven exchange); the ranks must agree
 * on the exchange in use. */
int sbs_peer_handle(sbs_ctx* ctx, uint8_t handle[64], void** base);
int sbs_peer_connect(sbs_ctx* ctx, void* const* bases, const uint8_t* handles);
int sbs_step_records(sbs_ctx* ctx, const sbs_input* d_in, float* d_rec, void* stream);
int sbs_finish_records(sbs_ctx* ctx, const float* d_recs, const sbs_input* d_in, sbs_output* d_out, void* stream);

/* ---- closed loop around the iteration (DESIGN L36-L40) -------
 * The MPC output drives a plant for one control period and the next
 * iteration's inputs are built on the device, so a whole closed-loop episode
 * (for every robot of the context) runs without host round trips:
 *   plant (L36): x <- one RK4 step (dt) of Eq. 1 with u0 on the
 *     stance legs (contact0, lever arms on feet_cur) plus an external wrench
 *     (world-frame force and torque at the CoM): v_dot += F/m,
 *     omega_dot += I^-1 R^T tau;
 *   fall (L40): |roll| or |pitch| > fall_angle or p_z < fall_height (or a
 *     non-finite state) sets fallen[r]; a fallen robot's inputs are frozen;
 *   gait (L37): phase += Q0.32 increment of the chosen step frequency;
 *     freq_idx <- the chosen theta1 (output freq_idx);
 *   footholds (L38, Eq. 3): a leg that was in swing and is in
 *     stance at the new phase lands on its planned foothold (feet_cur <-
 *     feet_next); every leg's next foothold is Eq. 3 at the new state with
 *     p_hip = p_c + Rz(yaw) hip_i (z = 0) and T_st = D_f / f_s;
 *   reference (L13): the context's x^r is rebuilt from the command at the
 *     new state: p^r_j = p_xy + v_d j dt, h_nom; v^r = v_d;
 *     yaw^r_j = yaw + yaw_rate j dt; omega^r = (0, 0, yaw_rate).
 * A later host-path sbs_step uploads the host-staged reference again (call
 * sbs_set_reference first). */
typedef struct sbs_loop_config {
  float hip[12];          /* body-frame hip offsets FL, FR, RL, RR (z ignored) */
  float h_nom;            /* nominal CoM height of the rebuilt reference (L13) */
  float fall_angle;       /* rad (L40) */
  float fall_height;      /* m (L40) */
  int32_t n_inner;        /* sbs_run_loop: SBS iterations per control step, 1..64 (Alg. 1 "multiple
                             times"; L34): all on the same x0, warm shift on the first only */
} sbs_loop_config;

typedef struct sbs_command {  /* per robot, device */
  float v[3];             /* desired CoM velocity v_c^d, world frame (Eq. 3) */
  float yaw_rate;         /* desired yaw rate (L13) */
} sbs_command;

#define SBS_TRACE_FLOATS 16   /* per robot per iteration: x after the plant step [12], freq_hz,
                                 j_min, fallen, status */

/* One advance of every robot after a step: d_in [R] is updated in place from
 * d_out [R] (the outputs of the step that consumed d_in).  d_cmd [R];
 * d_wrench [R][6] (F, tau) or NULL (no disturbance); d_fallen [R] (in/out,
 * sticky).  Stream-ordered; does not change iter. */
int sbs_advance(sbs_ctx* ctx, sbs_input* d_in, const sbs_output* d_out, const sbs_command* d_cmd,
                const float* d_wrench, int32_t* d_fallen, const sbs_loop_config* lc, void* stream);

/* n_iter closed-loop control steps on the device: each is lc->n_inner x
 * sbs_step_device(d_in, d_out) (the first with the warm shift, the others
 * refining the same distribution at the same x0) then sbs_advance with wrench row i of d_wrench [n_iter][R][6] (or
 * NULL) and, if d_trace [n_iter][R][SBS_TRACE_FLOATS] is not NULL, trace row
 * i.  One iteration is captured once as a CUDA graph (the iteration counter
 * lives in device memory) and replayed n_iter times.  world = 1 only.
 * iter += n_iter * n_inner.  Stream-ordered. */
int sbs_run_loop(sbs_ctx* ctx, int32_t n_iter, sbs_input* d_in, sbs_output* d_out, const sbs_command* d_cmd,
                 const float* d_wrench, int32_t* d_fallen, float* d_trace, const sbs_loop_config* lc,
                 void* stream);

/* Full covariance (full_cov = 1).  sbs_set_covariance: C [D][D] (host, row-major; its symmetric
 * part is factored in binary64; SBS_ERR_INVALID_ARG unless positive definite); var := diag(C).
 * sbs_get_cholesky: the current lower factor L [D][D] (host, row-major, zeros above the
 * diagonal).  sbs_set_distribution on such a context sets C = diag(var). */
int sbs_set_covariance(sbs_ctx* ctx, int32_t robot, const float* C);
int sbs_get_cholesky(sbs_ctx* ctx, int32_t robot, float* L);

/* The context's current reference of one robot (host out [H][12]): the last
 * sbs_set_reference / sbs_set_reference_device, or the rebuild of the last
 * sbs_advance / sbs_run_loop.  Synchronises the context's stream. */
int sbs_get_reference(sbs_ctx* ctx, int32_t robot, float* x_ref);

/* Exact checkpoint of the distribution state (means, vars, freq indices,
 * iteration counter, seed).  nbytes: in = capacity, out = size needed. */
int sbs_get_state(sbs_ctx* ctx, void* buf, uint64_t* nbytes);
int sbs_set_state(sbs_ctx* ctx, const void* buf, uint64_t nbytes);

/* NCCL bootstrap: rank 0 fills id (128 bytes); the caller broadcasts it. */
int sbs_nccl_unique_id(uint8_t id[128]);

/* ---- test / measurement entry points ---------------------------------- */
/* Samples that the NEXT sbs_step would draw for `robot`, global sample
 * indices k0..k0+n-1 (host outputs [n][D] each; any may be NULL). */
int sbs_debug_samples(sbs_ctx* ctx, int32_t robot, int64_t k0, int64_t n, float* z, float* theta,
                      int32_t* fidx);
/* Costs J of the last step: host [R][K_local], K_local = this rank's slice. */
int sbs_debug_costs(sbs_ctx* ctx, float* J);
/* Elite indices (global, ascending) of the last CEM/Naive step: host [K_e]. */
int sbs_debug_elites(sbs_ctx* ctx, int32_t robot, int64_t* idx);
/* Stand-alone elite selection (the K_e smallest of J by (J, k); NaN as +inf)
 * on device `device`; host J[K] in, host idx[K_e] out (ascending). */
int sbs_debug_select(const float* J, int64_t K, int64_t K_e, int64_t* idx, int32_t device);
/* The normative binary32 noise recipe (O3-O4; "theta_k ~ N(theta, C)")
 * applied to given Philox output words on device `device`: host words[n][4] in (one Philox
 * block each: Box-Muller pairs (w0, w1) and (w2, w3)), host z[n][4] out, in the order the
 * sampler uses (z0 = r cos, z1 = r sin of the first pair, then the second pair).  n <= 2^28.
 * Tests only (exhaustive recipe checks); no context needed. */
int sbs_debug_noise(const uint32_t* words, int64_t n, float* z, int32_t device);
/* Philox4x32-10 (O1) on given counters ctr[n][4] and keys key[n][2] on device `device`:
 * ours[n][2][4] = the library's plain and round-key forms, curand_words[n][4] = cuRAND's
 * curand_Philox4x32_10 of the same inputs.  n <= 2^26.  Tests only. */
int sbs_debug_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* ours, uint32_t* curand_words,
                     int32_t device);
/* Slice [k_begin, k_begin + K_local) of the samples owned by this rank. */
int sbs_local_range(const sbs_ctx* ctx, int64_t* k_begin, int64_t* K_local);
/* Per-kernel CUDA-event timing (enable = 1 records events around every launch). */
#define SBS_KERNEL_ROLLOUT 0
#define SBS_KERNEL_REDUCE 1
#define SBS_KERNEL_SELECT 2
#define SBS_KERNEL_ELITE 3
#define SBS_KERNEL_ADVANCE 4
#define SBS_NKERNELS 5
int sbs_profile(sbs_ctx* ctx, int32_t enable);
int sbs_kernel_times(sbs_ctx* ctx, double* total_ms /*[SBS_NKERNELS]*/, int64_t* launches /*[SBS_NKERNELS]*/);
/* Number of kernel launches one sbs_step issues (for the bench's gpu_launches). */
int sbs_launches_per_step(const sbs_ctx* ctx);

const char* sbs_status_str(int status);
const char* sbs_last_error(const sbs_ctx* ctx);
int sbs_version(void);
uint64_t sbs_sizeof_config(void);
uint64_t sbs_sizeof_input(void);
uint64_t sbs_sizeof_output(void);

#ifdef __cplusplus
}
#endif
#endif /* SBS_H */
