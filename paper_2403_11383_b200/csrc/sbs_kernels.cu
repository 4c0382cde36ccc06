// sbs_kernels.cu -- sm_100a kernels of one SBS MPC iteration (arxiv 2403.11383).
//
//   sbs_rollout_kernel   steps a0-a4 (+ a5 / a6 tile epilogue): warm shift, Philox
//                        sampling, contact sequence, GRF spline + cone, SRBD RK4,
//                        cost; one thread per sample, everything in registers;
//                        MPPI: online (min, sum w, sum w theta) record per CTA;
//                        Naive/CEM: (J, k) argmin + finite-cost sums.  FUSED: the
//                        last CTA of each robot merges the records and finishes
//                        the iteration (MPPI a5/a7, Naive a6/a7).  Variants: SPLIT
//                        (latency mode: 4 lanes per sample in the sampler), FC
//                        (full-covariance sampling, L42).
//   sbs_select_kernel    step a6 (CEM): exact radix select of the K_e smallest (J, k);
//                        EMIT / MERGE modes for sample sharding (world > 1).
//   sbs_elite_kernel     step a6/a7 (CEM): regenerate the elites' theta from the
//                        counter RNG, elite mean / variance, output.
//   sbs_cov_kernel       the same with a full covariance (elite covariance, Cholesky).
//   sbs_mppi_finalize, sbs_naive_finalize_kernel
//                        world > 1: rank-order merges of the gathered rank records
//                        (the fused rollout's last CTA emits each rank's record).
//   sbs_debug_samples_kernel   the draws of given sample indices (tests).
// The closed-loop advance kernel is in sbs_loop.cu.
//
// The rollout is FP32 CUDA-core work (not a contraction): it is bound by FP32
// issue and latency, not by HBM (4 bytes written per sample).  See DESIGN.md sec. 7.
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include <type_traits>


#include "sbs_internal.h"
#include "sbs_noise.cuh"
#if defined(SBS_TU_COMMON)
#include <curand_philox4x32_x.h>  // tests only: cuRAND's Philox4x32-10 next to ours
#endif
#include "sbs_robot_model.h"

namespace sbs {
#if defined(SBS_TIMING)  // experiments only: phase timestamps (%globaltimer) of CTA 0 / the last CTA
__device__ unsigned long long g_sbs_ts[32];  // [16, 32): the CEM cluster kernel
#define SBS_TS(i)                                                               \
  do {                                                                          \
    if (threadIdx.x == 0) {                                                     \
      unsigned long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_sbs_ts[i] = t_;                                                         \
    }                                                                           \
  } while (0)
__device__ unsigned long long g_sbs_cta[1024][6];
__device__ unsigned long long g_sbs_bar[4][8];  // integrator warp x chunk: cycles waiting on the chunk barrier (CTA 0)  // per CTA: globaltimer x4, clock64 around the rollout
#define SBS_CTS(i)                                                              \
  do {                                                                          \
    if (threadIdx.x == 0 && blockIdx.x < 1024 && blockIdx.y == 0) {             \
      unsigned long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_sbs_cta[blockIdx.x][i] = (i) >= 4 ? (unsigned long long)clock64() : t_; \
    }                                                                           \
  } while (0)
#define SBS_CTT(i)                                                              \
  do {                                                                          \
    if (threadIdx.x == 0 && blockIdx.x < 1024 && blockIdx.y == 0) {             \
      unsigned long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_sbs_cta[blockIdx.x][i] = t_;                                            \
    }                                                                           \
  } while (0)
#else
#define SBS_CTT(i) \
  do {             \
  } while (0)
#define SBS_TS(i) \
  do {            \
  } while (0)
#define SBS_CTS(i) \
  do {             \
  } while (0)
#endif

#define kInf __int_as_float(0x7f800000)
constexpr long long kSpinLimit = 4000000000LL;  // SM cycles (~2 s) a cross-CTA wait may take before it traps
constexpr float kPitchMax = 1.5697963267948966f;  // pi/2 - 1e-3 (L26)
constexpr float kTwoPi = 6.283185307179586f;
constexpr float kInvTwoPi = 0.15915494309189535f;

// ---------------------------------------------------------------------------
// Per-robot shared inputs: warm-shifted mean, std, x0, feet, reference.
// ---------------------------------------------------------------------------
struct RobotSmem {
  float mu[SBS_MAX_D];
  float sig[SBS_MAX_D];
  float x0[12];
  float4 feet[2][4];  // [0]: feet_cur, [1]: feet_next, per leg (x, y, z, 0): one 16-byte load per stance leg
  float xref[SBS_MAX_HORIZON * 12];  // per step, kernel order (px,py, vx,vy, pz,vz, roll,pitch, yaw,wx, wy,wz)
  uint8_t ctab[SBS_MAX_FREQ][SBS_MAX_HORIZON];  // bits 0-3: stance of leg i at step j; bits 4-7: leg i touched down
  uint32_t phase0;
  uint32_t iter;  // iteration counter of this step (noise counter word 2)
  int cur_idx;
};

// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic-
// serialisation attribute starts while its predecessor drains and waits here until
// the predecessor has completed and its memory is visible (a no-op otherwise).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// robot r's inputs / reference: device buffers, or (host path, R = 1) the kernel parameters themselves
__device__ __forceinline__ const sbs_input* robot_in(const Params& p, int r) { return p.inline_in ? &p.in_inline : p.in + r; }
__device__ __forceinline__ const float* robot_xref(const Params& p, int r) {
  return p.inline_in ? p.xref_inline : p.xref + (size_t)r * p.H * 12;
}

// iteration counter: kernel parameter, or device memory when the step runs as a
// captured CUDA graph (the host writes it with the inputs every step)
__device__ __forceinline__ uint32_t step_iter(const Params& p) { return p.iter_dev ? *p.iter_dev + p.iter_add : p.iter; }

// state-vector index in the kernel's pair order for each index of x = (p, v, Phi, w)
__device__ __forceinline__ int xref_slot(int a) { return a == 2 ? 4 : (a == 3 ? 2 : (a == 4 ? 3 : a)); }

// step a0: mu'[p] = S_mu(min(t_p + dt, T)); std = sqrt(var).
// Also the contact table of every frequency option (O7, L22, L23) from the
// Q0.32 phase: one byte per (theta1, step).
static __device__ void load_robot(const Params& p, int r, RobotSmem& s, bool rollout_inputs = true) {
  const int D = p.D, P = p.P;
  const float* mean = p.mean + (size_t)r * D;
  const float* var = p.var + (size_t)r * D;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const int pk = d / 12, ch = d - 12 * pk;
    float v = 0.0f;
    if (p.warm_shift) {
      for (int q = 0; q < P; ++q) v = fmaf(p.WS[pk][q], mean[q * 12 + ch], v);
    } else {
      v = mean[d];
    }
    s.mu[d] = v;
    s.sig[d] = __fsqrt_rn(var[d]);
  }
  const sbs_input* in = robot_in(p, r);
  SBS_CHECK(r >= 0 && r < p.R);
  if (threadIdx.x == 0) {
    s.cur_idx = p.fidx[r];
    s.iter = step_iter(p);
    SBS_CHECK(s.cur_idx >= 0 && s.cur_idx < p.n_freq);
  }
  if (!rollout_inputs) return;  // sampling only (elite regeneration, debug draws)
  for (int a = threadIdx.x; a < 12; a += blockDim.x) {
    s.x0[a] = in->x0[a];
    reinterpret_cast<float*>(&s.feet[0][a / 3])[a % 3] = in->feet_cur[a];
    reinterpret_cast<float*>(&s.feet[1][a / 3])[a % 3] = in->feet_next[a];
  }
  const float* xr = robot_xref(p, r);
  for (int a = threadIdx.x; a < p.H * 12; a += blockDim.x) {
    const int j = a / 12, c = a - 12 * j;
    s.xref[12 * j + xref_slot(c)] = xr[a];
  }
  const uint32_t ph0 = in->phase_q32;
  for (int f = threadIdx.x; f < p.n_freq; f += blockDim.x) {
    uint32_t ph[4];
    uint32_t prev = 0, td = 0;
    for (int i = 0; i < 4; ++i) ph[i] = ph0 + p.off[i];
    for (int j = 0; j < p.H; ++j) {
      uint32_t st = 0;
      for (int i = 0; i < 4; ++i) {
        if (p.all_stance || ph[i] < p.thr) st |= 1u << i;
        ph[i] += p.inc[f];
      }
      if (j > 0) td |= st & ~prev;  // first swing -> stance transition inside the horizon
      prev = st;
      s.ctab[f][j] = (uint8_t)(st | (td << 4));
    }
  }
  if (threadIdx.x == 0) s.phase0 = ph0;
}

// Latency mode: load_robot split in two so that the L2 round trips of the robot's
// inputs overlap the noise draws.  _issue starts asynchronous global->shared copies
// (cp.async, no register destination) of the raw inputs; _commit waits for them and
// applies the same transforms as load_robot (warm shift, sqrt, contact table).
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(__cvta_generic_to_global(src))
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(__cvta_generic_to_global(src))
               : "memory");
}
static __device__ void load_robot_issue(const Params& p, int r, RobotSmem& s, float* mraw) {
  const int D = p.D;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    cp_async4(&mraw[d], p.mean + (size_t)r * D + d);
    cp_async4(&s.sig[d], p.var + (size_t)r * D + d);  // variance; sqrt in _commit
  }
  if (threadIdx.x == 0) cp_async4(&s.cur_idx, p.fidx + r);
  if (p.inline_in) return;  // parameter-space inputs: copied in _commit
  const sbs_input* in = p.in + r;
  for (int a = threadIdx.x; a < 12; a += blockDim.x) {
    cp_async4(&s.x0[a], &in->x0[a]);
    cp_async4(reinterpret_cast<float*>(&s.feet[0][a / 3]) + a % 3, &in->feet_cur[a]);
    cp_async4(reinterpret_cast<float*>(&s.feet[1][a / 3]) + a % 3, &in->feet_next[a]);
  }
  const float* xr = p.xref + (size_t)r * p.H * 12;
  for (int a = threadIdx.x; a < p.H * 12; a += blockDim.x) {
    const int j = a / 12, c = a - 12 * j;
    cp_async4(&s.xref[12 * j + xref_slot(c)], xr + a);
  }
  if (threadIdx.x == 0) cp_async4(&s.phase0, &in->phase_q32);
}
static __device__ void load_robot_commit(const Params& p, RobotSmem& s, const float* mraw, uint32_t iter) {
  if (p.inline_in) {
    const sbs_input* in = &p.in_inline;
    for (int a = threadIdx.x; a < 12; a += blockDim.x) {
      s.x0[a] = in->x0[a];
      reinterpret_cast<float*>(&s.feet[0][a / 3])[a % 3] = in->feet_cur[a];
      reinterpret_cast<float*>(&s.feet[1][a / 3])[a % 3] = in->feet_next[a];
    }
    for (int a = threadIdx.x; a < p.H * 12; a += blockDim.x) {
      const int j = a / 12, c = a - 12 * j;
      s.xref[12 * j + xref_slot(c)] = p.xref_inline[a];
    }
    if (threadIdx.x == 0) s.phase0 = in->phase_q32;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int D = p.D, P = p.P;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    const int pk = d / 12, ch = d - 12 * pk;
    float v = 0.0f;
    if (p.warm_shift) {
      for (int q = 0; q < P; ++q) v = fmaf(p.WS[pk][q], mraw[q * 12 + ch], v);
    } else {
      v = mraw[d];
    }
    s.mu[d] = v;
    s.sig[d] = __fsqrt_rn(s.sig[d]);
  }
  const uint32_t ph0 = s.phase0;
  for (int f = threadIdx.x; f < p.n_freq; f += blockDim.x) {  // as in load_robot
    uint32_t ph[4];
    uint32_t prev = 0, td = 0;
    for (int i = 0; i < 4; ++i) ph[i] = ph0 + p.off[i];
    for (int j = 0; j < p.H; ++j) {
      uint32_t st = 0;
      for (int i = 0; i < 4; ++i) {
        if (p.all_stance || ph[i] < p.thr) st |= 1u << i;
        ph[i] += p.inc[f];
      }
      if (j > 0) td |= st & ~prev;
      prev = st;
      s.ctab[f][j] = (uint8_t)(st | (td << 4));
    }
  }
  if (threadIdx.x == 0) s.iter = iter;
  __syncthreads();
}

// Latency mode: the normative noise of this lane's Philox blocks q = u, u + 4, ... of
// sample k (before the distribution is known), and the gait draw on lane 0.
template <int P>
struct SplitNoise {
  static constexpr int NB = (3 * P + kSplitLanes - 1) / kSplitLanes;
  float z[NB][4];
  int fi;
};
template <int P>
__device__ __forceinline__ void split_noise(const Params& p, uint32_t robot_g, int64_t k, uint32_t iter, int u,
                                            SplitNoise<P>& n) {
#pragma unroll
  for (int i = 0; i < SplitNoise<P>::NB; ++i) {
    const int q = u + kSplitLanes * i;
    if (q < 3 * P) {
      const U4 w = philox4x32_10_rk((uint32_t)q, (uint32_t)k, iter, robot_g, p.rk);
      box_muller_x2(w, n.z[i]);
    }
  }
  n.fi = -1;
  if (u == 0 && p.gait_adapt) {
    const U4 w = philox4x32_10_rk(0x80000000u, (uint32_t)k, iter, robot_g, p.rk);
    n.fi = (int)__umulhi(w.x, (uint32_t)p.n_freq);
  }
}

// theta2 of one sample in registers, organised per leg: (x, y) knot pairs for
// packed FP32x2 arithmetic and the z knots; element d = (p*4 + leg)*3 + axis.
template <int P>
struct Theta {
  float2 xy[P][4];
  float z[P][4];
  // Gamma_j of one leg (O8): the knots weighted by the step's Catmull-Rom row
  __device__ __forceinline__ void spline(int leg, const float (&Wj)[P], float2& g, float& gz) const {
    g = __fmul2_rn(make_float2(Wj[0], Wj[0]), xy[0][leg]);
    gz = Wj[0] * z[0][leg];
#pragma unroll
    for (int q = 1; q < P; ++q) {
      g = __ffma2_rn(make_float2(Wj[q], Wj[q]), xy[q][leg], g);
      gz = fmaf(Wj[q], z[q][leg], gz);
    }
  }
};


template <int P>
__device__ __forceinline__ void theta_set(Theta<P>& t, int d, float v) {  // d is a compile-time constant here
  const int pk = d / 12, c = d % 12, leg = c / 3, ax = c % 3;
  if (ax == 0) t.xy[pk][leg].x = v;
  else if (ax == 1) t.xy[pk][leg].y = v;
  else t.z[pk][leg] = v;
}
template <int P>
__device__ __forceinline__ float theta_get(const Theta<P>& t, int d) {
  const int pk = d / 12, c = d % 12, leg = c / 3, ax = c % 3;
  return ax == 0 ? t.xy[pk][leg].x : (ax == 1 ? t.xy[pk][leg].y : t.z[pk][leg]);
}

// step a1: theta2 = mu' + sigma z, theta1 index
template <int P, bool WITH_Z>
__device__ __forceinline__ int draw_sample(const Params& p, uint32_t robot_g, int64_t k, const RobotSmem& s,
                                           Theta<P>& th, float* z_out = nullptr) {
  constexpr int D = 12 * P;
  if (p.elite_preserve && k == 0) {  // L21
#pragma unroll
    for (int d = 0; d < D; ++d) theta_set(th, d, s.mu[d]);
    if (WITH_Z)
      for (int d = 0; d < D; ++d) z_out[d] = 0.0f;
    return s.cur_idx;
  }
  const uint32_t kk = (uint32_t)k;
  const bool grp = p.n_sig_groups > 1;  // uniform per launch
  const float sc = grp ? p.sig_scale[(int)(k % p.n_sig_groups)] : 1.0f;
#pragma unroll
  for (int q = 0; q < D / 4; ++q) {
    const U4 w = philox4x32_10_rk((uint32_t)q, kk, s.iter, robot_g, p.rk);
    float z[4];
    box_muller_x2(w, z);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float sg = grp ? __fmul_rn(s.sig[4 * q + i], sc) : s.sig[4 * q + i];
      theta_set(th, 4 * q + i, __fmaf_rn(sg, z[i], s.mu[4 * q + i]));
      if (WITH_Z) z_out[4 * q + i] = z[i];
    }
  }
  int idx = s.cur_idx;
  if (p.gait_adapt) {
    const U4 w = philox4x32_10_rk(0x80000000u, kk, s.iter, robot_g, p.rk);
    idx = (int)__umulhi(w.x, (uint32_t)p.n_freq);  // (w * n) >> 32
  }
  return idx;
}

// One Philox block q (4 coordinates d = 4q..4q+3) of sample k: theta2 values.
// Same recipe and rounding as draw_sample, so results are bitwise identical.
__device__ __forceinline__ void sample_block(const Params& p, uint32_t robot_g, int64_t k, int q,
                                             const RobotSmem& s, float (&th4)[4]) {
  if (p.elite_preserve && k == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) th4[i] = s.mu[4 * q + i];
    return;
  }
  const U4 w = philox4x32_10_rk((uint32_t)q, (uint32_t)k, s.iter, robot_g, p.rk);
  float z[4];
  box_muller_x2(w, z);
  const bool grp = p.n_sig_groups > 1;
  const float sc = grp ? p.sig_scale[(int)(k % p.n_sig_groups)] : 1.0f;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    th4[i] = __fmaf_rn(grp ? __fmul_rn(s.sig[4 * q + i], sc) : s.sig[4 * q + i], z[i], s.mu[4 * q + i]);
}

// f3 (L42): theta2 = mu' + L z with the same normative noise z.  Lt = L^T staged in
// shared memory (Lt[j D + i] = L[i][j]); row i accumulates L_ij z_j for ascending j
// (fmaf from 0), then adds mu'_i.  Broadcast shared-memory reads (all lanes read the
// same L entry).
template <int P, bool WITH_Z>
__device__ __forceinline__ int draw_sample_fc(const Params& p, uint32_t robot_g, int64_t k, const RobotSmem& s,
                                              const float* Lt, Theta<P>& th, float* z_out = nullptr) {
  constexpr int D = 12 * P;
  if (p.elite_preserve && k == 0) {  // L21
#pragma unroll
    for (int d = 0; d < D; ++d) theta_set(th, d, s.mu[d]);
    if (WITH_Z)
      for (int d = 0; d < D; ++d) z_out[d] = 0.0f;
    return s.cur_idx;
  }
  const uint32_t kk = (uint32_t)k;
#pragma unroll
  for (int d = 0; d < D; ++d) theta_set(th, d, 0.0f);
#pragma unroll
  for (int q = 0; q < D / 4; ++q) {
    const U4 w = philox4x32_10_rk((uint32_t)q, kk, s.iter, robot_g, p.rk);
    float z[4];
    box_muller_x2(w, z);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = 4 * q + u;
#pragma unroll
      for (int i = j; i < D; ++i) theta_set(th, i, __fmaf_rn(Lt[j * D + i], z[u], theta_get(th, i)));
      if (WITH_Z) z_out[j] = z[u];
    }
  }
#pragma unroll
  for (int d = 0; d < D; ++d) theta_set(th, d, __fadd_rn(s.mu[d], theta_get(th, d)));
  int idx = s.cur_idx;
  if (p.gait_adapt) {
    const U4 w = philox4x32_10_rk(0x80000000u, kk, s.iter, robot_g, p.rk);
    idx = (int)__umulhi(w.x, (uint32_t)p.n_freq);
  }
  return idx;
}

// L (row-major lower [D][D], global) -> Lt (transposed, shared; upper part of L as zeros)
__device__ __forceinline__ void stage_chol_t(const Params& p, int r, float* Lt) {
  const int D = p.D;
  const float* L = p.Lmat + (size_t)r * D * D;
  for (int idx = threadIdx.x; idx < D * D; idx += blockDim.x) {
    const int i = idx / D, j = idx - i * D;
    Lt[j * D + i] = j <= i ? L[idx] : 0.0f;
  }
}

// noise z of Philox block q of sample k (elite preservation: z = 0)
__device__ __forceinline__ void noise_block(const Params& p, uint32_t robot_g, int64_t k, int q, const RobotSmem& s,
                                            float (&z)[4]) {
  if (p.elite_preserve && k == 0) {
    z[0] = z[1] = z[2] = z[3] = 0.0f;
    return;
  }
  const U4 w = philox4x32_10_rk((uint32_t)q, (uint32_t)k, s.iter, robot_g, p.rk);
  box_muller_x2(w, z);
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }

// Model and cost constants of the rollout.  DynC reads them from the parameter
// block (any robot); ModelC is the compiled-in robot of sbs_robot_model.h, whose
// values the compiler folds into immediate operands (sbs_create selects it only
// when the parameter block holds exactly these values).
struct DynC {
  static constexpr bool kStatic = false;
  __device__ static __forceinline__ float dt(const Params& p) { return p.dt; }
  __device__ static __forceinline__ float inv_mass(const Params& p) { return p.inv_mass; }
  __device__ static __forceinline__ float g(const Params& p, int i) { return p.g[i]; }
  __device__ static __forceinline__ bool diag(const Params& p) { return p.diag_inertia != 0; }
  __device__ static __forceinline__ float I(const Params& p, int i) { return p.I[i]; }
  __device__ static __forceinline__ float Iinv(const Params& p, int i) { return p.Iinv[i]; }
  __device__ static __forceinline__ float gyr(const Params& p, int i) { return p.gyr[i]; }
  __device__ static __forceinline__ float Q(const Params& p, int i) { return p.Q[i]; }
  __device__ static __forceinline__ float Rw(const Params& p, int i) { return p.Rw[i]; }
  __device__ static __forceinline__ float urz(const Params& p, int n) { return p.urz[n]; }
  __device__ static __forceinline__ float mu(const Params& p) { return p.mu; }
  __device__ static __forceinline__ float fz_min(const Params& p) { return p.fz_min; }
  __device__ static __forceinline__ float fz_max(const Params& p) { return p.fz_max; }
  __device__ static __forceinline__ float w_fc(const Params& p) { return p.w_fc; }
};
struct ModelC {
  static constexpr bool kStatic = true;
  __device__ static __forceinline__ constexpr float dt(const Params&) { return model::kDt; }
  __device__ static __forceinline__ constexpr float inv_mass(const Params&) { return model::kInvMass; }
  __device__ static __forceinline__ constexpr float g(const Params&, int i) { return i == 2 ? model::kGz : 0.0f; }
  __device__ static __forceinline__ constexpr bool diag(const Params&) { return true; }
  __device__ static __forceinline__ constexpr float I(const Params&, int i) {
    return i == 0 ? model::kI0 : (i == 4 ? model::kI1 : (i == 8 ? model::kI2 : 0.0f));
  }
  __device__ static __forceinline__ constexpr float Iinv(const Params&, int i) {
    return i == 0 ? model::kIinv0 : (i == 4 ? model::kIinv1 : (i == 8 ? model::kIinv2 : 0.0f));
  }
  __device__ static __forceinline__ constexpr float gyr(const Params&, int i) {
    return i == 0 ? model::kGyr0 : (i == 1 ? model::kGyr1 : model::kGyr2);
  }
  __device__ static __forceinline__ constexpr float Q(const Params&, int i) { return model::Q(i); }
  __device__ static __forceinline__ constexpr float Rw(const Params&, int) { return model::kR; }
  __device__ static __forceinline__ float urz(const Params&, int n) {  // n = stance-leg count 0..4
    return n <= 1 ? model::urz(1) : (n == 2 ? model::urz(2) : (n == 3 ? model::urz(3) : model::urz(4)));
  }
  __device__ static __forceinline__ constexpr float mu(const Params&) { return model::kMu; }
  __device__ static __forceinline__ constexpr float fz_min(const Params&) { return model::kFzMin; }
  __device__ static __forceinline__ constexpr float fz_max(const Params&) { return model::kFzMax; }
  __device__ static __forceinline__ constexpr float w_fc(const Params&) { return model::kWfc; }
};

// 1 / x for the Euler-rate map (|x| = cos(pitch) >= sin(1e-3) on every scored state, L26):
// MUFU reciprocal, flush-to-zero variant (no denormal range fix-up is needed here)
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// NaN-propagating maximum (max.NaN): a NaN component keeps the divergence test failing
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Eq. 1 angular part at one RK4 stage (L24): given the world torque tau,
//   w' = I^-1 (R^T tau - w x I w),  Phi' = E'^-1(Phi) w.
// Angular state in three pairs: A = (roll, pitch), B = (yaw, w_x), C = (w_y, w_z).
template <class KC>
__device__ __forceinline__ void ang_deriv(const Params& p, float2 A, float2 B, float2 C, float tx, float ty, float tz,
                                          float2& dA, float2& dB, float2& dC) {
  float sr, cr, sp, cp, sy, cy;
  __sincosf(A.x, &sr, &cr);
  __sincosf(A.y, &sp, &cp);
  __sincosf(B.x, &sy, &cy);
  const float wx = B.y, wy = C.x, wz = C.y;
  // R^T tau = Rx^T Ry^T Rz^T tau  (R = Rz(yaw) Ry(pitch) Rx(roll))
  const float t1x = fmaf(cy, tx, sy * ty), t1y = fmaf(cy, ty, -sy * tx);
  const float bx = fmaf(cp, t1x, -sp * tz), t2z = fmaf(sp, t1x, cp * tz);
  const float by = fmaf(cr, t1y, sr * t2z), bz = fmaf(cr, t2z, -sr * t1y);
  float dwx;
  float2 dwyz;
  if (KC::diag(p)) {
    // diagonal I: (w x I w)_x = (I_z - I_y) w_y w_z (cyclic), so
    // w'_x = I^-1_x b_x + G_x w_y w_z with G_x = I^-1_x (I_y - I_z) (cyclic; Params::gyr)
    dwx = fmaf(KC::gyr(p, 0), wy * wz, KC::Iinv(p, 0) * bx);
    dwyz = f2(fmaf(KC::gyr(p, 1), wz * wx, KC::Iinv(p, 4) * by), fmaf(KC::gyr(p, 2), wx * wy, KC::Iinv(p, 8) * bz));
  } else {
    const float Lx = fmaf(p.I[0], wx, fmaf(p.I[1], wy, p.I[2] * wz));
    const float Ly = fmaf(p.I[3], wx, fmaf(p.I[4], wy, p.I[5] * wz));
    const float Lz = fmaf(p.I[6], wx, fmaf(p.I[7], wy, p.I[8] * wz));
    const float rx = bx - fmaf(wy, Lz, -wz * Ly);
    const float ry = by - fmaf(wz, Lx, -wx * Lz);
    const float rz = bz - fmaf(wx, Ly, -wy * Lx);
    dwx = fmaf(p.Iinv[0], rx, fmaf(p.Iinv[1], ry, p.Iinv[2] * rz));
    dwyz = f2(fmaf(p.Iinv[3], rx, fmaf(p.Iinv[4], ry, p.Iinv[5] * rz)),
              fmaf(p.Iinv[6], rx, fmaf(p.Iinv[7], ry, p.Iinv[8] * rz)));
  }
  // E'^-1 w: yaw rate (sr wy + cr wz) / cos(pitch); roll rate wx + sin(pitch) * yaw rate
  const float yd = fmaf(sr, wy, cr * wz) * rcp_approx(cp);
  dA = f2(fmaf(sp, yd, wx), fmaf(cr, wy, -sr * wz));
  dB = f2(yd, dwx);
  dC = dwyz;
}

// Stance-leg quantities of one horizon step j (state-independent): the spline forces
// Gamma_j = sigma(theta2, t_j) (O8), their cone projection and penalty (O9), the effort
// (L12) and the net force / moment about the origin.  Per-leg work sits behind the
// stance bit: with a fixed gait every lane of a warp shares the contact schedule, so
// swing legs cost nothing.
struct StepForces {
  float2 F;
  float Fz, Mx, My, Mz;
  float ju;  // control part of the stage cost: (u - u^r)^T R (u - u^r) + w_fc pen
};
constexpr int kStepForceFloats = 7;

// MASK: the stance set as a compile-time constant (0: read from fl).  With a constant set
// no accumulator needs its -0 start value in a register and no leg branches.
template <int P, class KC = DynC, class TH = Theta<P>, uint32_t MASK = 0u>
__device__ __forceinline__ StepForces step_forces(const Params& p, const TH& th, uint32_t fl, const float (&Wj)[P],
                                                  const RobotSmem& s) {
  const float urz = KC::urz(p, MASK ? __popc(MASK) : __popc(fl & 0xFu));
  // accumulators start at -0 (the additive identity), so the first add is not a real op
  StepForces o;
  o.F = f2(-0.f, -0.f);
  o.Fz = -0.f, o.Mx = -0.f, o.My = -0.f, o.Mz = -0.f;
  float2 pen = f2(-0.f, -0.f), eff = f2(-0.f, -0.f);
  float penz = -0.f, effz = -0.f;
#pragma unroll
  for (int leg = 0; leg < 4; ++leg) {
    if ((MASK ? MASK : fl) & (1u << leg)) {
      float2 g;
      float gz;
      th.spline(leg, Wj, g, gz);
      const float fzc = fminf(fmaxf(gz, KC::fz_min(p)), KC::fz_max(p));
      const float l = KC::mu(p) * fzc;
      const float2 c = f2(fminf(fmaxf(g.x, -l), l), fminf(fmaxf(g.y, -l), l));
      // squared violation of the raw output = squared distance to its projection
      // (max(0, |g| - l) = |g - c| and max(0, fz_min - g) + max(0, g - fz_max) = |g - fzc|)
      const float2 dv = fadd2(g, f2(-c.x, -c.y));
      const float dz = gz - fzc;
      pen = ffma2(dv, dv, pen);
      penz = fmaf(dz, dz, penz);
      // effort (u - u^r)^T R (u - u^r), u^r = (0, 0, m|g|/n_stance) (L12)
      const float ez = fzc - urz;
      if constexpr (KC::kStatic) {  // one weight for every component: applied once per step
        eff = ffma2(c, c, eff);
        effz = fmaf(ez, ez, effz);
      } else {
        eff = ffma2(p.pk[14 + leg], fmul2(c, c), eff);  // R (c c), the weight pair uniform
        effz = fmaf(KC::Rw(p, 3 * leg + 2) * ez, ez, effz);
      }
      // net force and moment about the origin; feet switch at touchdown (L23)
      o.F = fadd2(o.F, c);
      o.Fz += fzc;
      const float4 ft = s.feet[(fl >> (4 + leg)) & 1u][leg];  // feet_next after touchdown
      const float fx = ft.x, fy = ft.y, fzz = ft.z;
      o.Mx = fmaf(fy, fzc, fmaf(-fzz, c.y, o.Mx));
      o.My = fmaf(fzz, c.x, fmaf(-fx, fzc, o.My));
      o.Mz = fmaf(fx, c.y, fmaf(-fy, c.x, o.Mz));
    }
  }
  const float pen_s = (pen.x + pen.y) + penz;
  const float eff_s = (eff.x + eff.y) + effz;
  o.ju = fmaf(KC::w_fc(p), pen_s, KC::kStatic ? KC::Rw(p, 0) * eff_s : eff_s);
  return o;
}

// The stance sets of a trot (one diagonal pair, or all four legs in the double-support
// phases of D_f > 0.5) as compile-time sets; any other set at run time.  Every lane of a
// warp shares the set under a fixed gait, so the switch does not diverge there.
template <int P, class KC = DynC, class TH = Theta<P>>
__device__ __forceinline__ StepForces step_forces_any(const Params& p, const TH& th, uint32_t fl, const float (&Wj)[P],
                                                      const RobotSmem& s) {
  switch (fl & 0xFu) {
    case 0x9u: return step_forces<P, KC, TH, 0x9u>(p, th, fl, Wj, s);
    case 0x6u: return step_forces<P, KC, TH, 0x6u>(p, th, fl, Wj, s);
    case 0xFu: return step_forces<P, KC, TH, 0xFu>(p, th, fl, Wj, s);
    default: return step_forces<P, KC, TH, 0u>(p, th, fl, Wj, s);
  }
}

// Latency mode, force-producer side: table [H][kStepForceFloats][kBlock] in shared
// memory, sample column `col` (conflict-free: consecutive lanes, consecutive words).
__device__ __forceinline__ void store_forces(float* tab, int j, int col, const StepForces& f) {
  float* t = tab + (size_t)j * kStepForceFloats * kBlock + col;
  t[0 * kBlock] = f.F.x;
  t[1 * kBlock] = f.F.y;
  t[2 * kBlock] = f.Fz;
  t[3 * kBlock] = f.Mx;
  t[4 * kBlock] = f.My;
  t[5 * kBlock] = f.Mz;
  t[6 * kBlock] = f.ju;
}
__device__ __forceinline__ StepForces load_forces(const float* tab, int j, int col) {
  const float* t = tab + (size_t)j * kStepForceFloats * kBlock + col;
  StepForces f;
  f.F = f2(t[0 * kBlock], t[1 * kBlock]);
  f.Fz = t[2 * kBlock];
  f.Mx = t[3 * kBlock];
  f.My = t[4 * kBlock];
  f.Mz = t[5 * kBlock];
  f.ju = t[6 * kBlock];
  return f;
}

// Latency mode: the horizon is cut into chunks [ab_chunk(c), ab_chunk(c + 1)) of growing
// length (1, 2, 3, ...); the producers arrive on named barrier 1 + c once chunk c is in
// the table, the integrators wait on it before step ab_chunk(c).
__device__ __forceinline__ int ab_chunk(int c) { return c * (c + 1) / 2; }
constexpr int kAbWarpsPerSmsp = 3;  // producer warps per integrator warp (the CTA's other 12 warps)
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// State part of the stage cost r(u_j, x_j, x^r_j): (x - x^r)^T Q (x - x^r),
// yaw error wrapped, packed pairs in the kernel's state order.
__device__ __forceinline__ float state_cost(const Params& p, const float* xr, float2 pxy, float2 vxy, float pz, float vz,
                                            float2 A, float2 Bq, float2 C) {
  const float2 e0 = fadd2(pxy, f2(-xr[0], -xr[1]));
  const float2 e1 = fadd2(vxy, f2(-xr[2], -xr[3]));
  const float2 e2 = fadd2(f2(pz, vz), f2(-xr[4], -xr[5]));
  const float2 e3 = fadd2(A, f2(-xr[6], -xr[7]));
  float2 e4 = fadd2(Bq, f2(-xr[8], -xr[9]));
  e4.x = fmaf(-kTwoPi, rintf(e4.x * kInvTwoPi), e4.x);  // yaw wrapped to [-pi, pi]
  const float2 e5 = fadd2(C, f2(-xr[10], -xr[11]));
  // Q (e e): the weight pair is the uniform operand of each packed multiply-add (Params::pk)
  float2 acc = fmul2(p.pk[8], fmul2(e0, e0));
  acc = ffma2(p.pk[9], fmul2(e1, e1), acc);
  acc = ffma2(p.pk[10], fmul2(e2, e2), acc);
  acc = ffma2(p.pk[11], fmul2(e3, e3), acc);
  acc = ffma2(p.pk[12], fmul2(e4, e4), acc);
  acc = ffma2(p.pk[13], fmul2(e5, e5), acc);
  return acc.x + acc.y;
}

// x_{j+1} = f(x_j, u_j), Eq. 1 with classic RK4.  v' = F/m + g is
// constant over the step, so RK4 on (p, v) is exact and the stage positions q are
// closed-form; each stage's torque about the CoM is tau = M - q x F (M, F about the
// origin, step_forces), and only the 6 angular states run the RK4 recurrence.
template <class KC>
__device__ __forceinline__ void srbd_step(const Params& p, const StepForces& sf, float2& pxy, float2& vxy, float& pz,
                                          float& vz, float2& A, float2& Bq, float2& C) {
  const float dt = KC::dt(p), hdt = 0.5f * dt;
  const float dt2h = 0.5f * dt * dt, dt2q = 0.25f * dt * dt;
  // packed operand pairs from the parameter block (uniform registers; Params::pk)
  const float2 dt_2 = p.pk[0], hdt_2 = p.pk[1], dt6_2 = p.pk[2], two_2 = p.pk[3];
  const float2 dt2h_2 = p.pk[4], dt2q_2 = p.pk[5], im_2 = p.pk[6], gxy = p.pk[7];
  const float2 F = sf.F;
  const float Fz = sf.Fz;
  // tau = M - q x F at the stage position (q, qz)
  auto tq = [&](float2 q, float qz, float& tx, float& ty, float& tz) {
    tx = fmaf(qz, F.y, fmaf(-q.y, Fz, sf.Mx));
    ty = fmaf(q.x, Fz, fmaf(-qz, F.x, sf.My));
    tz = fmaf(q.y, F.x, fmaf(-q.x, F.y, sf.Mz));
  };
  const float2 axy = ffma2(F, im_2, gxy);
  const float az = fmaf(Fz, KC::inv_mass(p), KC::g(p, 2));
  float2 k1A, k1B, k1C, k2A, k2B, k2C, k3A, k3B, k3C, k4A, k4B, k4C;
  float tx, ty, tz;
  tq(pxy, pz, tx, ty, tz);
  ang_deriv<KC>(p, A, Bq, C, tx, ty, tz, k1A, k1B, k1C);
  tq(ffma2(hdt_2, vxy, pxy), fmaf(hdt, vz, pz), tx, ty, tz);
  ang_deriv<KC>(p, ffma2(hdt_2, k1A, A), ffma2(hdt_2, k1B, Bq), ffma2(hdt_2, k1C, C), tx, ty, tz, k2A, k2B, k2C);
  tq(ffma2(dt2q_2, axy, ffma2(hdt_2, vxy, pxy)), fmaf(dt2q, az, fmaf(hdt, vz, pz)), tx, ty, tz);
  ang_deriv<KC>(p, ffma2(hdt_2, k2A, A), ffma2(hdt_2, k2B, Bq), ffma2(hdt_2, k2C, C), tx, ty, tz, k3A, k3B, k3C);
  const float2 n = ffma2(dt2h_2, axy, ffma2(dt_2, vxy, pxy));
  const float nz = fmaf(dt2h, az, fmaf(dt, vz, pz));
  tq(n, nz, tx, ty, tz);
  ang_deriv<KC>(p, ffma2(dt_2, k3A, A), ffma2(dt_2, k3B, Bq), ffma2(dt_2, k3C, C), tx, ty, tz, k4A, k4B, k4C);
  A = ffma2(dt6_2, ffma2(two_2, fadd2(k2A, k3A), fadd2(k1A, k4A)), A);
  Bq = ffma2(dt6_2, ffma2(two_2, fadd2(k2B, k3B), fadd2(k1B, k4B)), Bq);
  C = ffma2(dt6_2, ffma2(two_2, fadd2(k2C, k3C), fadd2(k1C, k4C)), C);
  pxy = n;
  pz = nz;
  vxy = ffma2(dt_2, axy, vxy);
  vz = fmaf(dt, az, vz);
}

// divergence of x_{j+1} (L26): a component beyond 1e6, a NaN (max.NaN keeps it) or
// |pitch| >= pi/2 - 1e-3
__device__ __forceinline__ bool diverged(float2 pxy, float2 vxy, float pz, float vz, float2 A, float2 Bq, float2 C) {
  const float big = fmax_nan(fmax_nan(fmax_nan(fabsf(pxy.x), fabsf(pxy.y)), fmax_nan(fabsf(pz), fabsf(vxy.x))),
                             fmax_nan(fmax_nan(fabsf(vxy.y), fabsf(vz)), fmax_nan(fabsf(A.x), fabsf(Bq.x))));
  const float big2 = fmax_nan(fmax_nan(fabsf(Bq.y), fabsf(C.x)), fabsf(C.y));
  return !(fmax_nan(big, big2) <= 1e6f) || !(fabsf(A.y) < kPitchMax);
}

// steps a2-a4: Rollout(theta_k, x0), Alg. 2 with policy pi:
//   for j: u_j = pi(theta, t_j); J += r(u_j, x_j, x^r_j); x_{j+1} = f(x_j, u_j)
// then J += rho (f - f_n)^2; a diverged rollout costs +inf (L26).
template <int P, class KC = DynC, class TH = Theta<P>>
static __device__ float rollout(const Params& p, const TH& th, int fi, const RobotSmem& s) {
  float2 pxy = f2(s.x0[0], s.x0[1]), vxy = f2(s.x0[3], s.x0[4]);
  float pz = s.x0[2], vz = s.x0[5];
  float2 A = f2(s.x0[6], s.x0[7]), Bq = f2(s.x0[8], s.x0[9]), C = f2(s.x0[10], s.x0[11]);
  SBS_CHECK(fi >= 0 && fi < p.n_freq && p.H <= SBS_MAX_HORIZON);
  const uint8_t* ct = s.ctab[fi];
  float J = 0.0f;
  bool bad = false;
  for (int j = 0; j < p.H; ++j) {
    float Wj[P];
#pragma unroll
    for (int q = 0; q < P; ++q) Wj[q] = p.W[j][q];
    const StepForces sf = step_forces_any<P, KC>(p, th, ct[j], Wj, s);
    J += state_cost(p, &s.xref[12 * j], pxy, vxy, pz, vz, A, Bq, C) + sf.ju;
    srbd_step<KC>(p, sf, pxy, vxy, pz, vz, A, Bq, C);
    bad = bad || diverged(pxy, vxy, pz, vz, A, Bq, C);
  }
  const float df = p.freq_hz[fi] - p.f_nominal;
  J = fmaf(p.rho * df, df, J);  // P:350, once per rollout (L14)
  return (bad || !(J <= FLT_MAX)) ? kInf : J;
}

// Latency mode, integrator warps: rollout() with the stance-leg quantities of every
// step read from the producer warps' table (step_forces: the same arithmetic, the
// same bits), waiting on the chunk barriers.
template <int P, class KC = DynC>
static __device__ float rollout_ab(const Params& p, int fi, const RobotSmem& s, const float* tab, int col) {
  float2 pxy = f2(s.x0[0], s.x0[1]), vxy = f2(s.x0[3], s.x0[4]);
  float pz = s.x0[2], vz = s.x0[5];
  float2 A = f2(s.x0[6], s.x0[7]), Bq = f2(s.x0[8], s.x0[9]), C = f2(s.x0[10], s.x0[11]);
  float J = 0.0f;
  bool bad = false;
  int next_chunk = 0;
  for (int j = 0; j < p.H; ++j) {
#if defined(SBS_TIMING)
    if (j == ab_chunk(next_chunk)) {
      const long long t0 = clock64();
      named_sync(1 + next_chunk, kBlock * (1 + kAbWarpsPerSmsp));
      if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && next_chunk < 8)
        g_sbs_bar[threadIdx.x >> 5][next_chunk] = (unsigned long long)(clock64() - t0);
      ++next_chunk;
    }
#else
    if (j == ab_chunk(next_chunk)) named_sync(1 + next_chunk++, kBlock * (1 + kAbWarpsPerSmsp));
#endif
    const StepForces sf = load_forces(tab, j, col);
    J += state_cost(p, &s.xref[12 * j], pxy, vxy, pz, vz, A, Bq, C) + sf.ju;
    srbd_step<KC>(p, sf, pxy, vxy, pz, vz, A, Bq, C);
    bad = bad || diverged(pxy, vxy, pz, vz, A, Bq, C);
  }
  const float df = p.freq_hz[fi] - p.f_nominal;
  J = fmaf(p.rho * df, df, J);  // P:350, once per rollout (L14)
  return (bad || !(J <= FLT_MAX)) ? kInf : J;
}

// Latency mode, producer warps: the stance-leg table of the integrator warp on the same
// SM sub-partition (warp w: integrator warp w % 4, step class w / 4 - 1), chunk by chunk.
template <int P, class KC = DynC>
__device__ __forceinline__ void produce_forces(const Params& p, const RobotSmem& s, const float* s_th, const int* s_fi,
                                               float* tab) {
  constexpr int D = 12 * P;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = 32 * (warp & 3) + lane, cls = (warp >> 2) - 1;
  Theta<P> th;
#pragma unroll
  for (int d = 0; d < D; ++d) theta_set(th, d, s_th[col * (D + 1) + d]);
  const uint8_t* ct = s.ctab[s_fi[col]];
  for (int c = 0; ab_chunk(c) < p.H; ++c) {
    const int j1 = min(ab_chunk(c + 1), p.H);
    for (int j = ab_chunk(c) + cls; j < j1; j += kAbWarpsPerSmsp) {
      float Wj[P];
#pragma unroll
      for (int q = 0; q < P; ++q) Wj[q] = p.W[j][q];
      store_forces(tab, j, col, step_forces_any<P, KC>(p, th, ct[j], Wj, s));
    }
    named_arrive(1 + c, kBlock * (1 + kAbWarpsPerSmsp));
  }
}

// (J, k) lexicographic order: argmin with lowest-index tie-break (L4, L5)
__device__ __forceinline__ bool jk_less(float ja, int ka, float jb, int kb) {
  return ja < jb || (ja == jb && ka < kb);
}

__device__ __forceinline__ uint32_t cost_key(float J);
__device__ __forceinline__ float key_cost(uint32_t key);
// (J, k) argmin of a warp, the winner's theta1 index: two integer min-reductions
// (REDUX) over the order-preserving cost key and, among the tied lanes, the index.
// Same result as a jk_less butterfly (k is unique per sample; only the sentinel
// lanes (+inf, 0x7fffffff) can tie completely, and then lane 0 wins in both).
__device__ __forceinline__ void warp_argmin(float& m, int& mk, int& mf) {
  const uint32_t key = cost_key(m);
  const uint32_t kmin = __reduce_min_sync(0xffffffffu, key);
  const uint32_t kk = __reduce_min_sync(0xffffffffu, key == kmin ? (uint32_t)mk : 0xffffffffu);
  const uint32_t who = __ballot_sync(0xffffffffu, key == kmin && (uint32_t)mk == kk);
  const int src = __ffs(who) - 1;
  m = __shfl_sync(0xffffffffu, m, src);
  mf = __shfl_sync(0xffffffffu, mf, src);
  mk = (int)kk;
}

// Partial record of (robot r, part c): CTA partials [R][n_cta] (part_c_stride = 1)
// or NCCL-gathered rank partials [world][R] (part_c_stride = R, n_cta = world).
//   [0] min J  [1] k_argmin  [2] theta1 of argmin  [3] S = sum w  [4] S2 = sum w^2
//   [5] sum of finite J  [6] number finite  [7] 0  [8 ..] V = sum w theta2
__device__ __forceinline__ const float* part_rec(const Params& p, int r, int c) {
  SBS_CHECK(r >= 0 && r < p.R && c >= 0 && c < p.n_cta);
  return p.part_c_stride == 1 ? p.part + ((size_t)r * p.n_cta + c) * p.part_stride
                              : p.part + ((size_t)c * p.part_c_stride + r) * p.part_stride;
}

// cooperative copy of n floats (n % 4 == 0, 16-byte aligned) from L2 to shared
// memory, 4 independent 16-byte loads in flight per thread
// records into shared memory by cp.async (L2 -> shared, no register destination: every
// 16-byte piece of the block's share in flight at once, one L2 round trip); stage_wait
// completes the calling thread's copies (a barrier then publishes them to the block)
__device__ __forceinline__ void stage_issue(float* dst, const float* src, int n) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  const int n4 = n >> 2;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) cp_async16(d4 + i, s4 + i);
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// the same through registers, four 16-byte loads in flight per thread (the dynamic-tile
// kernel's node merges, whose headline build it is)
__device__ __forceinline__ void stage_copy(float* dst, const float* src, int n) {
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  const int n4 = n >> 2;
  for (int i0 = threadIdx.x; i0 < n4; i0 += 4 * blockDim.x) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n4) v[u] = __ldcg(s4 + i);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n4) d4[i] = v[u];
    }
  }
}

// ---------------------------------------------------------------------------
// Output (a7): u0 = delta_0-masked cone projection of knot 0.
// ---------------------------------------------------------------------------
// pre: {phase_q32 of the robot's input, iteration counter} already in shared memory, or null (loaded here)
static __device__ void write_output(const Params& p, int r, int status, const float* mean_new, const float* var_new,
                             int fi, float jmin, float jmean, float omega, float ess, int ndiv,
                             const uint32_t* pre = nullptr) {
  SBS_CHECK(r >= 0 && r < p.R);
  sbs_output* o = p.out + r;
  const int D = p.D;
  const uint32_t ph0 = pre ? pre[0] : robot_in(p, r)->phase_q32;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    o->mean[d] = mean_new[d];
    o->var[d] = var_new[d];
  }
  if (threadIdx.x < 4) {
    const int i = threadIdx.x;
    const bool st = p.all_stance || (ph0 + p.off[i] < p.thr);
    o->contact0[i] = st ? 1 : 0;
    const float fx = mean_new[3 * i], fy = mean_new[3 * i + 1], fz = mean_new[3 * i + 2];
    const float fzc = fminf(fmaxf(fz, p.fz_min), p.fz_max);
    const float l = p.mu * fzc;
    o->u0[3 * i] = st ? fminf(fmaxf(fx, -l), l) : 0.0f;
    o->u0[3 * i + 1] = st ? fminf(fmaxf(fy, -l), l) : 0.0f;
    o->u0[3 * i + 2] = st ? fzc : 0.0f;
  }
  if (threadIdx.x == 0) {
    o->freq_idx = fi;
    o->freq_hz = p.freq_hz[fi];
    o->status = status;
    o->iter = pre ? pre[1] : step_iter(p);
    o->j_min = jmin;
    o->j_mean = jmean;
    o->omega = omega;
    o->ess = ess;
    o->n_diverged = ndiv;
    o->device_us = 0.0f;
    p.status[r] = status;
  }
  if (p.done) {  // host path: the outputs are in host memory before the flag (system-scope release)
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.sys.u32 [%0], %1;" ::"l"(p.done), "r"(p.done_value) : "memory");
  }
}

// Block-wide argmin over the partial headers of robot r.
struct Best {
  float m;
  int k, f;
};
static __device__ Best merge_argmin(const Params& p, int r, const float* recs = nullptr, int nrec = 0) {
  __shared__ float s_m[32];
  __shared__ int s_k[32], s_f[32];
  float m = kInf;
  int mk = 0x7fffffff, mf = 0;
  const int nc = recs ? nrec : p.n_cta;
  for (int c0 = threadIdx.x; c0 < nc; c0 += 4 * blockDim.x) {  // four headers' loads in flight per thread
    float mc[4];
    int kc[4], fc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u * blockDim.x;
      mc[u] = kInf;
      kc[u] = 0x7fffffff;
      fc[u] = 0;
      if (c < nc) {
        const float* pc = recs ? recs + (size_t)c * p.part_stride : part_rec(p, r, c);
        mc[u] = __ldcg(pc);
        kc[u] = __float_as_int(__ldcg(pc + 1));
        fc[u] = __float_as_int(__ldcg(pc + 2));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (jk_less(mc[u], kc[u], m, mk)) {
        m = mc[u];
        mk = kc[u];
        mf = fc[u];
      }
  }
  warp_argmin(m, mk, mf);
  if ((threadIdx.x & 31) == 0) {
    s_m[threadIdx.x >> 5] = m;
    s_k[threadIdx.x >> 5] = mk;
    s_f[threadIdx.x >> 5] = mf;
  }
  __syncthreads();
  Best b{s_m[0], s_k[0], s_f[0]};
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
    if (jk_less(s_m[w], s_k[w], b.m, b.k)) b = Best{s_m[w], s_k[w], s_f[w]};
  __syncthreads();
  return b;
}

// ---------------------------------------------------------------------------
// MPPI UpdateMean (Alg. 4) over the partial records of robot r:
// beta = min_c m_c; every record is rescaled by exp(-(m_c - beta)/lambda);
// theta_new = sum V / sum S.  EMIT: write the merged record (rank partial, or
// out_rec) instead of finishing.  The records: the CTA records of robot r
// (part_rec), or recs[0..nrec) (contiguous, stride part_stride).  blockDim.x = 128.
// ---------------------------------------------------------------------------
template <bool EMIT>
static __device__ void mppi_merge_block(const Params& p, int r, float* emit, float* stage, int stage_floats,
                                        const float* recs = nullptr, int nrec = 0, float* out_rec = nullptr) {
  const int tid = threadIdx.x, D = p.D, NR = D + 4, RL = p.part_stride;
  __shared__ float s_row[1][SBS_MAX_D + 4];
  __shared__ float s_sc[128];
  __shared__ float s_mean[SBS_MAX_D], s_var[SBS_MAX_D];
  __shared__ uint32_t s_pre[2];
  __shared__ float s_bm[32];
  __shared__ int s_bk[32], s_bf[32];
  __shared__ float s_part[16 * (SBS_MAX_D + 4)];
  const int nc = recs ? nrec : p.n_cta;
  const bool one_pass = nc <= 128 && nc * RL <= stage_floats;
  Best b;
  float bmin = kInf;
  if (one_pass) {
    // one load round trip: every record, this robot's variance, input phase and iteration counter
    if (recs) {
      stage_issue(stage, recs, nc * RL);
    } else if (p.part_c_stride == 1) {
      stage_issue(stage, part_rec(p, r, 0), nc * RL);  // records of a robot are contiguous
    } else {
      for (int c = 0; c < nc; ++c) stage_issue(stage + c * RL, part_rec(p, r, c), RL);
    }
    if (!EMIT) {
      for (int d = tid; d < D; d += blockDim.x) s_var[d] = p.var[(size_t)r * D + d];
      if (tid == 0) {
        s_pre[0] = robot_in(p, r)->phase_q32;
        s_pre[1] = step_iter(p);
      }
    }
    stage_wait();
    __syncthreads();
    SBS_TS(7);
    // every thread: the smallest record minimum (the scales' reference, no barrier); warp 0
    // also resolves the argmin's (k, theta1) for the outputs
    {  // per warp: lanes over the records, one integer min-reduction of the order-preserving key
      uint32_t kmin = 0xffffffffu;
      for (int c = tid & 31; c < nc; c += 32) kmin = min(kmin, cost_key(stage[c * RL]));
      bmin = key_cost(__reduce_min_sync(0xffffffffu, kmin));
    }
    if (tid < 32) {
      float m = kInf;
      int mk = 0x7fffffff, mf = 0;
      for (int c = tid; c < nc; c += 32) {
        const float* h = stage + c * RL;
        const int kc = __float_as_int(h[1]);
        if (jk_less(h[0], kc, m, mk)) {
          m = h[0];
          mk = kc;
          mf = __float_as_int(h[2]);
        }
      }
      warp_argmin(m, mk, mf);
      if (tid == 0) {
        s_bm[0] = m;
        s_bk[0] = mk;
        s_bf[0] = mf;
      }
    }
  } else {
    b = merge_argmin(p, r, recs, nrec);
  }
  SBS_TS(8);
  const float beta = one_pass ? bmin : b.m;  // (one pass: b is read after the row sums' barrier)
  const int CH = one_pass ? nc : min(128, max(1, stage_floats / RL));
  float acc = 0.f;  // chunked: thread tid < nh NR owns row tid % NR (0..D-1 V, D S, D+1 S2, D+2 sumJ, D+3 nfin), half tid / NR
  const int nh = 2 * NR <= (int)blockDim.x ? 2 : 1;
  for (int c0 = 0; c0 < nc; c0 += CH) {
    const int n = min(CH, nc - c0);
    if (!one_pass) {
      if (recs) {
        stage_issue(stage, recs + (size_t)c0 * RL, n * RL);
      } else if (p.part_c_stride == 1) {
        stage_issue(stage, part_rec(p, r, c0), n * RL);
      } else {
        for (int c = 0; c < n; ++c) stage_issue(stage + c * RL, part_rec(p, r, c0 + c), RL);
      }
      stage_wait();
      __syncthreads();
    }
    if (one_pass) {  // (row, record-chunk) per thread, each computing its records' scales, then chunk sums
      const int nch = max(1, min((int)blockDim.x / NR, 16));  // record chunks
      const int per = (n + nch - 1) / nch;
      float* part = s_part;                                    // [nch][NR]
      if (tid < nch * NR) {
        const int row = tid % NR, ch = tid / NR;
        const int col = row < D ? kPartHdr + row : 3 + (row - D);
        const int kind = row < D + 1 ? 0 : (row == D + 1 ? 1 : 2);
        const int c_end = min(n, (ch + 1) * per);
        float a0 = 0.f, a1 = 0.f;
        int c = ch * per;
        auto scale = [&](int cc) {
          const float mc = stage[cc * RL];
          return (mc < kInf) ? __expf((beta - mc) * p.inv_lambda) : 0.0f;
        };
        for (; c + 1 < c_end; c += 2) {
          float s0 = scale(c), s1 = scale(c + 1);
          if (kind == 1) { s0 *= s0; s1 *= s1; }
          if (kind == 2) { s0 = 1.f; s1 = 1.f; }
          a0 = fmaf(stage[c * RL + col], s0, a0);
          a1 = fmaf(stage[(c + 1) * RL + col], s1, a1);
        }
        if (c < c_end) {
          float s0 = kind == 2 ? 1.f : scale(c);
          if (kind == 1) s0 *= s0;
          a0 = fmaf(stage[c * RL + col], s0, a0);
        }
        part[ch * NR + row] = a0 + a1;
      }
      __syncthreads();
      if (tid < NR) {
        float a = 0.f;
        for (int ch = 0; ch < nch; ++ch) a += part[ch * NR + tid];
        s_row[0][tid] = a;
      }
      break;  // single chunk
    }
    for (int c = tid; c < n; c += blockDim.x) {
      const float mc = stage[c * RL];
      s_sc[c] = (mc < kInf) ? __expf((beta - mc) * p.inv_lambda) : 0.0f;
    }
    __syncthreads();
    if (tid < nh * NR) {  // (row, half of the chunk) per thread
      const int row = tid % NR, h = tid / NR, per = (n + nh - 1) / nh;
      const int col = row < D ? kPartHdr + row : 3 + (row - D);
      const int kind = row < D + 1 ? 0 : (row == D + 1 ? 1 : 2);
      const int c_end = min(n, (h + 1) * per);
      float a0 = 0.f, a1 = 0.f;
      int c = h * per;
#pragma unroll 4
      for (; c + 1 < c_end; c += 2) {
        float s0 = s_sc[c], s1 = s_sc[c + 1];
        if (kind == 1) { s0 *= s0; s1 *= s1; }
        if (kind == 2) { s0 = 1.f; s1 = 1.f; }
        a0 = fmaf(stage[c * RL + col], s0, a0);
        a1 = fmaf(stage[(c + 1) * RL + col], s1, a1);
      }
      if (c < c_end) {
        float s0 = kind == 2 ? 1.f : s_sc[c];
        if (kind == 1) s0 *= s0;
        a0 = fmaf(stage[c * RL + col], s0, a0);
      }
      acc += a0 + a1;
    }
    __syncthreads();
  }
  if (!one_pass) {  // the halves' sums, in order
    if (tid < nh * NR) s_part[tid] = acc;
    __syncthreads();
    if (tid < NR) s_row[0][tid] = nh == 2 ? s_part[tid] + s_part[NR + tid] : s_part[tid];
  }
  __syncthreads();
  if (one_pass) b = Best{s_bm[0], s_bk[0], s_bf[0]};  // (warp 0's argmin, ordered by the barriers above)
  SBS_TS(9);
  if (EMIT) {  // this rank's merged record, relative to its own beta
    float* o = out_rec ? out_rec : emit + (size_t)r * p.part_stride;
    if (tid < D) o[kPartHdr + tid] = s_row[0][tid];
    else if (tid < NR) o[3 + tid - D] = s_row[0][tid];
    if (tid == 0) {
      o[0] = b.m;
      o[1] = __int_as_float(b.k);
      o[2] = __int_as_float(b.f);
      o[7] = 0.0f;
    }
    return;
  }
  const bool all_div = !(b.m < kInf);
  const float S = s_row[0][D], S2 = s_row[0][D + 1], sumJ = s_row[0][D + 2], nfin = s_row[0][D + 3];
  float* mean = p.mean + (size_t)r * D;
  const float* var = p.var + (size_t)r * D;
  for (int d = tid; d < D; d += blockDim.x) {
    s_mean[d] = all_div ? mean[d] : s_row[0][d] / S;
    if (!one_pass) s_var[d] = var[d];
  }
  const int fi = all_div ? p.fidx[r] : b.f;
  __syncthreads();
  for (int d = tid; d < D; d += blockDim.x) mean[d] = s_mean[d];
  if (tid == 0) p.fidx[r] = fi;
  SBS_TS(10);
  write_output(p, r, all_div ? SBS_WARN_ALL_DIVERGED : SBS_OK, s_mean, s_var, fi, b.m,
               nfin > 0.f ? sumJ / nfin : kInf, S, all_div ? 0.f : S * S / S2, (int)((float)p.K_global - nfin),
               one_pass ? s_pre : nullptr);
}

// merges robot r's records (the rollout's CTA records, or the gathered rank
// records) into d: sdiag layout (J_min, k_best, theta1_best, sum J, n finite),
// or, with part_layout, a rank record header [m, k, f, 0, 0, sum J, n finite, 0]
// (hdr: the records' 8-float headers already staged in shared memory, or null: read from L2)
static __device__ void merge_diag(const Params& p, int r, float* d, bool part_layout, const float* hdr = nullptr) {
  if (threadIdx.x >= 32) return;  // one warp, one load round trip; the other warps go on (no block barrier)
  float m = kInf, sj = 0.f, nf = 0.f;
  int mk = 0x7fffffff, mf = 0;
  for (int c = threadIdx.x; c < p.n_cta; c += 32) {
    float mc, sc, nc;
    int kc, fc;
    if (hdr) {
      const float* pc = hdr + 8 * c;
      mc = pc[0], sc = pc[5], nc = pc[6];
      kc = __float_as_int(pc[1]), fc = __float_as_int(pc[2]);
    } else {
      const float* pc = part_rec(p, r, c);
      mc = __ldcg(pc), sc = __ldcg(pc + 5), nc = __ldcg(pc + 6);
      kc = __float_as_int(__ldcg(pc + 1)), fc = __float_as_int(__ldcg(pc + 2));
    }
    if (jk_less(mc, kc, m, mk)) {
      m = mc;
      mk = kc;
      mf = fc;
    }
    sj += sc;
    nf += nc;
  }
  warp_argmin(m, mk, mf);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sj += __shfl_xor_sync(0xffffffffu, sj, o);
    nf += __shfl_xor_sync(0xffffffffu, nf, o);
  }
  if (threadIdx.x == 0) {
    d[0] = m;
    d[1] = __int_as_float(mk);
    d[2] = __int_as_float(mf);
    if (part_layout) {
      d[3] = 0.f;
      d[4] = 0.f;
      d[5] = sj;
      d[6] = nf;
      d[7] = 0.f;
    } else {
      d[3] = sj;
      d[4] = nf;
    }
  }
}

// Naive UpdateMean (Alg. 3): the best sample theta* becomes the mean,
// regenerated from the counter RNG; C unchanged.
template <int P>
static __device__ void naive_finalize_block(const Params& p, int r, const RobotSmem& s) {
  constexpr int D = 12 * P;
  __shared__ float s_mean[D], s_var[D];
  __shared__ float s_sum[2];
  __shared__ uint32_t s_pre[2];
  const int tid = threadIdx.x;
  // issued with the record loads of merge_argmin (one round trip): variance, input phase, iteration
  for (int d = tid; d < D; d += blockDim.x) s_var[d] = p.var[(size_t)r * D + d];
  if (tid == 0) {
    s_pre[0] = robot_in(p, r)->phase_q32;
    s_pre[1] = step_iter(p);
  }
  const Best b = merge_argmin(p, r);
  if (tid < 32) {
    float sj = 0.f, nf = 0.f;
    for (int c = tid; c < p.n_cta; c += 32) {
      const float* pc = part_rec(p, r, c);
      sj += __ldcg(pc + 5);
      nf += __ldcg(pc + 6);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sj += __shfl_xor_sync(0xffffffffu, sj, o);
      nf += __shfl_xor_sync(0xffffffffu, nf, o);
    }
    if (tid == 0) {
      s_sum[0] = sj;
      s_sum[1] = nf;
    }
  }
  const bool all_div = !(b.m < kInf);
  float* mean = p.mean + (size_t)r * D;
  if (!all_div && tid < D / 4) {  // theta* regenerated, one Philox block per thread
    float th4[4];
    sample_block(p, (uint32_t)(p.robot_offset + r), b.k, tid, s, th4);
#pragma unroll
    for (int i = 0; i < 4; ++i) s_mean[4 * tid + i] = th4[i];
  }
  __syncthreads();
  for (int d = tid; d < D; d += blockDim.x)
    if (all_div) s_mean[d] = mean[d];
  const int fi = all_div ? s.cur_idx : b.f;
  __syncthreads();
  for (int d = tid; d < D; d += blockDim.x) mean[d] = s_mean[d];
  if (tid == 0) {
    p.fidx[r] = fi;
    p.elite[r] = (int64_t)b.k;
    p.best[r] = (int64_t)b.k;
  }
  const float nf = s_sum[1];
  write_output(p, r, all_div ? SBS_WARN_ALL_DIVERGED : SBS_OK, s_mean, s_var, fi, b.m,
               nf > 0.f ? s_sum[0] / nf : kInf, all_div ? 0.f : 1.f, all_div ? 0.f : 1.f,
               (int)((float)p.K_global - nf), s_pre);
}

// last CTA of a grid row (robot) to arrive returns true (threadfence pattern)
__device__ __forceinline__ bool arrive_last(int* counter, int n) {
  __shared__ int s_last;
  __syncthreads();  // the CTA's record writes happen-before thread 0's fence (fences are cumulative)
  if (threadIdx.x == 0) {
#if defined(SBS_SC_ARRIVE)
    __threadfence();
    s_last = (atomicAdd(counter, 1) == n - 1);
#else
    // release (the CTA's writes, ordered before by the barrier) and acquire (the other
    // CTAs' records, for this CTA's threads after the next barrier) in one atomic
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
    s_last = (old == n - 1);
#endif
  }
  __syncthreads();
  if (s_last) {
#if defined(SBS_SC_ARRIVE)
    __threadfence();
#endif
    if (threadIdx.x == 0) *counter = 0;  // re-arm for the next launch (stream-ordered)
  }
  return s_last;
}

// Peer-memory exchange of the rank records (world > 1 without NCCL):
// called by every CTA that completed a robot's rank record; the last of them
// copies this rank's records [R][ex_stride] (p.emit = its own gather slot) into
// every peer's gather buffer over NVLink, fences at system scope and raises the
// peer's flag for this rank.  The peers' streams wait on those flags in the
// front-end (cuStreamWaitValue32), not in a kernel.
static __device__ void publish_to_peers(const Params& p) {
  if (p.n_peers == 0 || !arrive_last(p.gcounter, p.R)) return;
  const size_t n = (size_t)p.R * p.ex_stride;
  for (int j = 0; j < p.n_peers; ++j) {
    if (j == p.my_rank) continue;
    float* dst = p.peer_gather[j] + (size_t)p.my_rank * n;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldcg(p.emit + i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int j = 0; j < p.n_peers; ++j)
      if (j != p.my_rank) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.peer_flags[j] + p.my_rank), "r"(p.flag_value) : "memory");
  }
}

// ---------------------------------------------------------------------------
// sbs_rollout_kernel: grid (n_cta, R), block kBlock.  CTA c processes tiles c,
// c + n_cta, ... of its robot's K_local samples and leaves one partial record.
//   EPI_MPPI:   online (min, sum w, sum w^2, sum w theta) over its samples
//   EPI_ARGMIN: (J, k) argmin + finite-cost sum/count (Naive, CEM)
// FUSED: the last CTA of each robot merges the records and finishes the
// iteration (MPPI, Naive): one launch per MPC iteration.
// SPLIT (latency mode, few samples): kSplitLanes x 128 threads per CTA; every
// tile's 128 samples are first drawn kSplitLanes lanes per sample (Philox
// blocks q = u, u + kSplitLanes, ... into shared memory), then the first 128
// threads roll them out while the others wait.  The same draw code and rounding
// as draw_sample, so the samples are bitwise identical; the per-sample dependent
// chain loses (kSplitLanes - 1) / kSplitLanes of the sampler.
// ---------------------------------------------------------------------------
enum { EPI_MPPI = 0, EPI_ARGMIN = 1 };


// Merge of n <= 128 MPPI records (contiguous, stride part_stride) into one record at
// `out`, relative to their smallest minimum -- the tree's inner nodes (and a rank's
// top-level nodes): warp 0 reads the n headers, takes beta = min m_c and the (J, k)
// argmin, and writes every record's scale exp((beta - m_c)/lambda) to shared memory;
// then row thread t sums column t over the records in index order (S2 with squared
// scales, the finite-cost sums unscaled), its loads independent of one another.  The
// same arithmetic for a node whichever GPU count or CTA schedule produced it.
static __device__ void dyn_node_merge(const Params& p, const float* kids, int n, float* out, float* stage,
                                      int stage_floats) {
  const int tid = threadIdx.x, D = p.D, NR = D + 4, RL = p.part_stride;
  __shared__ float s_bm;
  __shared__ int s_bk, s_bf;
  // the records staged in shared memory when they fit (every thread's loads in flight at
  // once), else read from L2 by the row threads
  const bool staged = n * RL + 128 <= stage_floats;
  float* s_sc = staged ? stage + n * RL : stage;
  const float* src = staged ? stage : kids;
  if (staged) {
    stage_copy(stage, kids, n * RL);
    __syncthreads();
  }
  if (tid < 32) {
    float mc[4];
    uint32_t kmin = 0xffffffffu;
    float m = kInf;
    int mk = 0x7fffffff, mf = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // n <= 128: four headers per lane
      const int c = tid + 32 * u;
      mc[u] = kInf;
      if (c < n) {
        const float* h = src + (size_t)c * RL;
        mc[u] = staged ? h[0] : __ldcg(h);
        const int kc = __float_as_int(staged ? h[1] : __ldcg(h + 1));
        const int fc = __float_as_int(staged ? h[2] : __ldcg(h + 2));
        kmin = min(kmin, cost_key(mc[u]));
        if (jk_less(mc[u], kc, m, mk)) {
          m = mc[u];
          mk = kc;
          mf = fc;
        }
      }
    }
    const float beta = key_cost(__reduce_min_sync(0xffffffffu, kmin));
    warp_argmin(m, mk, mf);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = tid + 32 * u;
      if (c < n) s_sc[c] = (mc[u] < kInf) ? __expf((beta - mc[u]) * p.inv_lambda) : 0.0f;
    }
    if (tid == 0) {
      s_bm = m;
      s_bk = mk;
      s_bf = mf;
    }
  }
  __syncthreads();
  if (tid < NR) {
    const int col = tid < D ? kPartHdr + tid : 3 + (tid - D);
    const int kind = tid < D + 1 ? 0 : (tid == D + 1 ? 1 : 2);
    float a0 = 0.f, a1 = 0.f;
    int c = 0;
#pragma unroll 4
    for (; c + 1 < n; c += 2) {
      float s0 = s_sc[c], s1 = s_sc[c + 1];
      if (kind == 1) { s0 *= s0; s1 *= s1; }
      if (kind == 2) { s0 = 1.f; s1 = 1.f; }
      const float v0 = staged ? src[(size_t)c * RL + col] : __ldcg(src + (size_t)c * RL + col);
      const float v1 = staged ? src[(size_t)(c + 1) * RL + col] : __ldcg(src + (size_t)(c + 1) * RL + col);
      a0 = fmaf(v0, s0, a0);
      a1 = fmaf(v1, s1, a1);
    }
    if (c < n) {
      float s0 = kind == 2 ? 1.f : s_sc[c];
      if (kind == 1) s0 *= s0;
      a0 = fmaf(staged ? src[(size_t)c * RL + col] : __ldcg(src + (size_t)c * RL + col), s0, a0);
    }
    if (tid < D) out[kPartHdr + tid] = a0 + a1;
    else out[3 + tid - D] = a0 + a1;
  }
  if (tid == 0) {
    out[0] = s_bm;
    out[1] = __int_as_float(s_bk);
    out[2] = __int_as_float(s_bf);
    out[7] = 0.0f;
  }
}

// The tree's root (world = 1), or the rank-order merge of the ranks' top-level records
// (world > 1, sbs_mppi_finalize): dyn_node_merge into a shared-memory record, then the
// finish of mppi_merge_block (new mean = V / S, outputs).  The finish's own loads
// (variance, input phase, iteration) are issued first and overlap the merge.
// mppi_merge_block's finish from a robot's merged record in shared memory (new mean
// V / S, outputs); s_var, s_pre: the robot's variance and (input phase, iteration)
static __device__ void mppi_finish_record(const Params& p, int r, const float* s_rec, const float* s_var,
                                          const uint32_t* s_pre) {
  const int tid = threadIdx.x, D = p.D;
  __shared__ float s_mean[SBS_MAX_D];
  const float bm = s_rec[0];
  const int bf = __float_as_int(s_rec[2]);
  const bool all_div = !(bm < kInf);
  const float S = s_rec[3], S2 = s_rec[4], sumJ = s_rec[5], nfin = s_rec[6];
  float* mean = p.mean + (size_t)r * D;
  for (int d = tid; d < D; d += blockDim.x) s_mean[d] = all_div ? mean[d] : s_rec[kPartHdr + d] / S;
  const int fi = all_div ? p.fidx[r] : bf;
  __syncthreads();
  for (int d = tid; d < D; d += blockDim.x) mean[d] = s_mean[d];
  if (tid == 0) p.fidx[r] = fi;
  write_output(p, r, all_div ? SBS_WARN_ALL_DIVERGED : SBS_OK, s_mean, s_var, fi, bm,
               nfin > 0.f ? sumJ / nfin : kInf, S, all_div ? 0.f : S * S / S2, (int)((float)p.K_global - nfin), s_pre);
}
// the robot's variance and (input phase, iteration) into shared memory (loads issued, not awaited)
__device__ __forceinline__ void load_finish_inputs(const Params& p, int r, float* s_var, uint32_t* s_pre) {
  for (int d = threadIdx.x; d < p.D; d += blockDim.x) s_var[d] = p.var[(size_t)r * p.D + d];
  if (threadIdx.x == 0) {
    s_pre[0] = robot_in(p, r)->phase_q32;
    s_pre[1] = step_iter(p);
  }
}

static __device__ void dyn_root_finish(const Params& p, int r, const float* kids, int n, float* stage,
                                       int stage_floats) {
  __shared__ __align__(16) float s_rec[kPartHdr + SBS_MAX_D + 4];
  __shared__ float s_var[SBS_MAX_D];
  __shared__ uint32_t s_pre[2];
  load_finish_inputs(p, r, s_var, s_pre);  // (overlap the merge)
  dyn_node_merge(p, kids, n, s_rec, stage, stage_floats);
  __syncthreads();
  mppi_finish_record(p, r, s_rec, s_var, s_pre);
}

// thread 0: the level-1 arrivals of the buffered tiles behind one release fence (one
// fence per kDynBatch tiles instead of per tile: a fence waits for the CTA's writes)
__device__ __forceinline__ void dyn_arrive(const Params& p, const int* pend, int& n_pend) {
  if (n_pend == 0) return;
  __threadfence();
#pragma unroll
  for (int i = 0; i < kDynBatch; ++i)
    if (i < n_pend) atomicAdd(p.dyn_cnt + p.dyn_coff[1] + pend[i] / p.dyn_fan, 1);
  n_pend = 0;
}

// Dynamic tile scheduling (Params::dyn): the tiles' records are reduced by a fixed tree
// of fan-in Params::dyn_fan over the tile index.  Once its tile loop is over (and its
// arrivals flushed), CTA c merges the level-1 nodes c, c + n_cta, ... in index order, each
// as soon as its tiles' arrivals are all in (a CTA takes a tile only while running, so
// every awaited tile is in a running CTA that does not wait itself), then climbs: the CTA
// completing a higher node (one arrival counter per node) merges it likewise.  The top
// level's merge finishes the iteration (world = 1, a single root) or writes this rank's
// top-level node records (world > 1: the rank-order merge after the exchange completes
// the global tree).  The tree and its merge order are fixed by the tile indices alone,
// so the result is the same whichever CTA ran which tile.
static __device__ void dyn_merge_nodes(const Params& p, int r, float* stage, int stage_floats) {
  const int RL = p.part_stride, L = p.dyn_levels;
  for (int node = blockIdx.x; node < p.dyn_n[1]; node += gridDim.x) {
    if (threadIdx.x == 0) {  // wait for the node's tile records (acquire)
      int* c = p.dyn_cnt + p.dyn_coff[1] + node;
      const int nk = min(p.dyn_fan, p.dyn_n[0] - node * p.dyn_fan);
      for (;;) {  // (every awaited arrival comes from a running CTA that does not wait itself)
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        if (v >= nk) break;
        __nanosleep(128);
      }
      *c = 0;  // re-armed (nothing else touches it this launch)
    }
    __syncthreads();
    SBS_CTT(2);  // (timing builds: the node's tiles are in)
    int idx = node;
    for (int l = 1; l <= L; ++l) {
      if (l > 1) {  // arrive at the level-l node; its last arrival merges it
        const int nkids_up = min(p.dyn_fan, p.dyn_n[l - 1] - (idx / p.dyn_fan) * p.dyn_fan);
        if (!arrive_last(p.dyn_cnt + p.dyn_coff[l] + idx / p.dyn_fan, nkids_up)) break;
        idx /= p.dyn_fan;
      }
      const int nkids = min(p.dyn_fan, p.dyn_n[l - 1] - idx * p.dyn_fan);
      SBS_CHECK(l <= kDynMaxLevels && idx >= 0 && idx < p.dyn_n[l] && nkids > 0);
      const float* kids = p.dyn_rec + (size_t)(p.dyn_off[l - 1] + idx * p.dyn_fan) * RL;
      if (l < L) {
        dyn_node_merge(p, kids, nkids, p.dyn_rec + (size_t)(p.dyn_off[l] + idx) * RL, stage, stage_floats);
        SBS_CTT(l == 1 ? 4 : 5);  // (timing builds: level-1 / upper node merged)
      } else if (p.emit) {  // world > 1: this rank's top-level record(s) (the exchange and rank-order merge follow)
        SBS_TS(5);
        dyn_node_merge(p, kids, nkids, p.emit + (size_t)idx * RL, stage, stage_floats);
        if (arrive_last(p.dyn_cnt + p.dyn_ecnt, p.dyn_n[L])) publish_to_peers(p);
        SBS_TS(6);
      } else {
        SBS_TS(5);
        dyn_root_finish(p, r, kids, nkids, stage, stage_floats);
        SBS_TS(6);
      }
    }
    __syncthreads();
  }
}

template <int P, int EPI, bool FUSED, bool FC = false, bool SPLIT = false, bool AB = false, bool MODEL = false,
          bool DYN = false>
__global__ void __launch_bounds__(SPLIT ? kBlock * kSplitLanes : kBlock, SPLIT ? 1 : kRolloutMinBlocks)
    sbs_rollout_kernel(const __grid_constant__ Params p) {
  using KC = typename std::conditional<MODEL, ModelC, DynC>::type;  // compiled-in robot model, or the parameter block
  constexpr int D = 12 * P;
  constexpr int NR = D + 4;  // reduced rows (MPPI): w theta[D], w, w^2, J (finite), 1 (finite)
  constexpr int TS = kBlock;  // samples per tile
  __shared__ RobotSmem s;
  extern __shared__ float s_red[];  // [NR][kRedStride] (MPPI) or L^T [D][D] (FC); SPLIT: + theta [TS][D + 1], fidx [TS]
  float* s_th = s_red + (EPI == EPI_MPPI ? NR * kRedStride : 0);
  int* s_fi = reinterpret_cast<int*>(s_th + TS * (D + 1));
  const bool sampler_thread = !SPLIT || threadIdx.x < kBlock;  // holds a sample in phase 2 / the epilogue
  __shared__ float s_wm[2][kBlock / 32], s_ws[2][kBlock / 32], s_wn[2][kBlock / 32];  // per warp, by tile parity
  __shared__ int s_wk[2][kBlock / 32], s_wf[2][kBlock / 32];
  // the CTA's running record header (MPPI: double-buffered by tile parity, read by the
  // row threads, advanced by thread 0; argmin epilogue: thread 0 only)
  __shared__ float s_rm[2], s_rsj, s_rnf;
  __shared__ int s_rk[2], s_rf[2];
  if (threadIdx.x == 0) {
    s_rm[0] = kInf;
    s_rk[0] = 0x7fffffff;
    s_rf[0] = 0;
    s_rsj = 0.f;
    s_rnf = 0.f;
  }
  int par = 0;  // parity of this CTA's current tile
  // SPLIT (one tile per CTA): the header lives in registers, the same in every thread
  float h_m = kInf, h_sj = 0.f, h_nf = 0.f;
  int h_k = 0x7fffffff, h_f = 0;

  const int r = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  griddep_wait();  // PDL: the previous iteration's distribution / the closed loop's new inputs
  if (blockIdx.x == 0) SBS_TS(0);
  SBS_CTS(0);
  const uint32_t robot_g = (uint32_t)(p.robot_offset + r);
  SplitNoise<P> zn;  // SPLIT: this lane's noise for the CTA's first tile
  if (SPLIT) {       // the inputs' round trips overlap the first tile's Philox / Box-Muller draws
    __shared__ float s_mraw[SBS_MAX_D];
    load_robot_issue(p, r, s, s_mraw);
    const uint32_t it = step_iter(p);
    const int64_t kl1 = (int64_t)blockIdx.x * kBlock + tid / kSplitLanes;
    if (kl1 < p.K_local) split_noise<P>(p, robot_g, p.k_begin + kl1, it, tid % kSplitLanes, zn);
    load_robot_commit(p, s, s_mraw, it);
  } else {
    load_robot(p, r, s);
  }
  if (FC) stage_chol_t(p, r, s_red);
  __syncthreads();
  if (blockIdx.x == 0) SBS_TS(1);
  float run = 0.0f;  // running partial of row `tid` (MPPI)

  // dynamic tile scheduling (throughput MPPI, one robot): the next tile index is fetched
  // at the start of each tile (s_nx[par], read after the tile's last barrier)
  constexpr bool dyn = DYN;  // (its own instantiation: the static kernel's registers are unchanged)
  static_assert(!DYN || (EPI == EPI_MPPI && FUSED && !SPLIT && !FC), "dynamic tiles: throughput MPPI only");
  __shared__ int s_nx[2];
  __shared__ int s_pend[kDynBatch];  // thread 0: tiles whose level-1 arrivals are batched behind one fence
  int n_pend = 0;
  if (dyn) {  // every tile from the counter, the first one too
    if (tid == 0) s_nx[1] = atomicAdd(p.dyn_cnt, 1);
    __syncthreads();
  }
  for (int tile = dyn ? s_nx[1] : (int)blockIdx.x; tile < p.n_tiles; tile = dyn ? s_nx[par ^ 1] : tile + (int)gridDim.x) {
    int nx = 0;  // (the next tile's index is consumed only at the tile's end: no wait here)
    if (dyn && tid == 0) nx = atomicAdd(p.dyn_cnt, 1);
    const int64_t kl = (int64_t)tile * TS + tid;
    const bool valid = sampler_thread && kl < p.K_local;
    const int64_t k = p.k_begin + kl;
    Theta<P> th;
    float J = kInf;
    int fi = 0;
    if (SPLIT) {  // phase 1: kSplitLanes lanes per sample draw its Philox blocks into shared memory
      if (tile != (int)blockIdx.x) __syncthreads();  // (one tile per CTA in this mode; s_th readers done)
      const int sl = tid / kSplitLanes, u = tid % kSplitLanes;
      const int64_t kl1 = (int64_t)tile * TS + sl;
      if (kl1 < p.K_local) {
        const int64_t k1 = p.k_begin + kl1;
        float* dst = s_th + sl * (D + 1);
        if (p.elite_preserve && k1 == 0) {  // L21
          for (int d = u; d < D; d += kSplitLanes) dst[d] = s.mu[d];
          if (u == 0) s_fi[sl] = s.cur_idx;
        } else {
          if (tile != (int)blockIdx.x) split_noise<P>(p, robot_g, k1, s.iter, u, zn);  // (later tiles)
          const bool grp = p.n_sig_groups > 1;
          const float sc = grp ? p.sig_scale[(int)(k1 % p.n_sig_groups)] : 1.0f;
#pragma unroll
          for (int i = 0; i < SplitNoise<P>::NB; ++i) {
            const int q = u + kSplitLanes * i;
            if (q < D / 4) {
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const float sg = grp ? __fmul_rn(s.sig[4 * q + c], sc) : s.sig[4 * q + c];
                dst[4 * q + c] = __fmaf_rn(sg, zn.z[i][c], s.mu[4 * q + c]);
              }
            }
          }
          if (u == 0) s_fi[sl] = zn.fi >= 0 ? zn.fi : s.cur_idx;
        }
      } else {  // past K: a valid contact-table row for the producer warps (results unused)
        if (u == 0) s_fi[sl] = 0;
      }
      __syncthreads();
    }
    if (SPLIT && AB) {  // warps 4..15 tabulate the stance-leg forces, warps 0..3 integrate
      float* tab = reinterpret_cast<float*>(s_fi + TS);
      if (!sampler_thread) {
        produce_forces<P, KC>(p, s, s_th, s_fi, tab);
      } else {
        fi = s_fi[tid];
        if (blockIdx.x == 0) SBS_TS(2);
        SBS_CTS(1);
        SBS_CTS(4);
        const float Ja = rollout_ab<P, KC>(p, fi, s, tab, tid);  // (every integrator lane: barriers)
        SBS_CTS(5);
        SBS_CTS(2);
        if (blockIdx.x == 0) SBS_TS(3);
        if (valid) {
          J = Ja;
          SBS_CHECK(kl >= 0 && kl < p.K_local);
          p.J[(size_t)r * p.K_local + kl] = J;
        }
      }
    } else if (valid) {
      if (SPLIT) {
#pragma unroll
        for (int d = 0; d < D; ++d) theta_set(th, d, s_th[tid * (D + 1) + d]);
        fi = s_fi[tid];
      } else if (FC) {
        fi = draw_sample_fc<P, false>(p, robot_g, k, s, s_red, th);
      } else {
        fi = draw_sample<P, false>(p, robot_g, k, s, th);
      }
      if (blockIdx.x == 0) SBS_TS(2);
      SBS_CTS(1);
      SBS_CTS(4);
      J = rollout<P, KC>(p, th, fi, s);
      SBS_CTS(5);
      SBS_CTS(2);
      if (blockIdx.x == 0) SBS_TS(3);
      SBS_CHECK(kl >= 0 && kl < p.K_local);
      p.J[(size_t)r * p.K_local + kl] = J;
    }
    // ---- per-tile argmin (J, k) ----
    float m = J;
    int mk = valid ? (int)k : 0x7fffffff, mf = fi;
    warp_argmin(m, mk, mf);
    const bool fin = J < kInf;
    if (EPI == EPI_ARGMIN) {
      float sj = fin ? J : 0.f, nf = fin ? 1.f : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sj += __shfl_xor_sync(0xffffffffu, sj, o);
        nf += __shfl_xor_sync(0xffffffffu, nf, o);
      }
      if (lane == 0 && sampler_thread) {
        s_wm[par][warp] = m;
        s_wk[par][warp] = mk;
        s_wf[par][warp] = mf;
        s_ws[par][warp] = sj;
        s_wn[par][warp] = nf;
      }
      __syncthreads();
      if (SPLIT) {
#pragma unroll
        for (int w = 0; w < kBlock / 32; ++w) {
          if (jk_less(s_wm[par][w], s_wk[par][w], h_m, h_k)) {
            h_m = s_wm[par][w];
            h_k = s_wk[par][w];
            h_f = s_wf[par][w];
          }
          h_sj += s_ws[par][w];
          h_nf += s_wn[par][w];
        }
      } else if (tid == 0) {
        for (int w = 0; w < kBlock / 32; ++w) {
          if (jk_less(s_wm[par][w], s_wk[par][w], s_rm[0], s_rk[0])) {
            s_rm[0] = s_wm[par][w];
            s_rk[0] = s_wk[par][w];
            s_rf[0] = s_wf[par][w];
          }
          s_rsj += s_ws[par][w];
          s_rnf += s_wn[par][w];
        }
      }
      par ^= 1;
      continue;
    }
    // ---- step a5 (MPPI), per tile: weights relative to the tile min, then an
    //      online-softmax merge into this CTA's running record ----
    if (lane == 0 && sampler_thread) {
      s_wm[par][warp] = m;
      s_wk[par][warp] = mk;
      s_wf[par][warp] = mf;
    }
    __syncthreads();
    float mt = s_wm[par][0];  // tile argmin, computed by every thread
    int tk = s_wk[par][0], tf = s_wf[par][0];
#pragma unroll
    for (int w = 1; w < kBlock / 32; ++w)
      if (jk_less(s_wm[par][w], s_wk[par][w], mt, tk)) {
        mt = s_wm[par][w];
        tk = s_wk[par][w];
        tf = s_wf[par][w];
      }

    const float w = fin ? __expf((mt - J) * p.inv_lambda) : 0.0f;
    constexpr int kQ = 4;  // SPLIT: sample quarters per reduced row
    if (SPLIT) {           // theta is already in shared memory: rows reduced straight from s_th by 4 x NR threads
      float* s_w = s_red + kQ * NR;  // [4][kBlock]: w, w^2, finite J, finite
      if (sampler_thread) {
        s_w[0 * kBlock + tid] = w;
        s_w[1 * kBlock + tid] = w * w;
        s_w[2 * kBlock + tid] = fin ? J : 0.0f;
        s_w[3 * kBlock + tid] = fin ? 1.0f : 0.0f;
      }
      __syncthreads();
      if (tid < kQ * NR) {
        const int row = tid % NR, q = tid / NR, i0 = q * (kBlock / kQ);
        const int64_t left = p.K_local - ((int64_t)tile * TS + i0);
        const int nv = left <= 0 ? 0 : (left >= kBlock / kQ ? kBlock / kQ : (int)left);
        float a0 = 0.f, a1 = 0.f;
        if (row < D) {
          const float* col = s_th + row;
          int i = 0;
          for (; i + 1 < nv; i += 2) {
            a0 = fmaf(s_w[i0 + i], col[(i0 + i) * (D + 1)], a0);
            a1 = fmaf(s_w[i0 + i + 1], col[(i0 + i + 1) * (D + 1)], a1);
          }
          if (i < nv) a0 = fmaf(s_w[i0 + i], col[(i0 + i) * (D + 1)], a0);
        } else {
          const float* rw = s_w + (row - D) * kBlock + i0;
          for (int i = 0; i < kBlock / kQ; i += 2) {
            a0 += rw[i];
            a1 += rw[i + 1];
          }
        }
        s_red[q * NR + row] = a0 + a1;
      }
      __syncthreads();
    } else {
      if (valid) {
#pragma unroll
        for (int d = 0; d < D; d += 2) {  // w theta, two coordinates per packed multiply
          const float2 v = __fmul2_rn(make_float2(w, w), make_float2(theta_get(th, d), theta_get(th, d + 1)));
          s_red[d * kRedStride + tid] = v.x;
          s_red[(d + 1) * kRedStride + tid] = v.y;
        }
      } else {
#pragma unroll
        for (int d = 0; d < D; ++d) s_red[d * kRedStride + tid] = 0.0f;
      }
      s_red[(D + 0) * kRedStride + tid] = w;
      s_red[(D + 1) * kRedStride + tid] = w * w;
      s_red[(D + 2) * kRedStride + tid] = fin ? J : 0.0f;
      s_red[(D + 3) * kRedStride + tid] = fin ? 1.0f : 0.0f;
      __syncthreads();
    }
    const float mr = SPLIT ? h_m : s_rm[par];
    const float mn = fminf(mr, mt);
    if (tid < NR) {
      float v;
      if (SPLIT) {
        v = (s_red[0 * NR + tid] + s_red[1 * NR + tid]) + (s_red[2 * NR + tid] + s_red[3 * NR + tid]);
      } else {
        // row tid: 16-byte loads (kRedStride keeps rows aligned and 8 consecutive rows on
        // distinct banks), two packed accumulators
        const float4* rowp = reinterpret_cast<const float4*>(&s_red[tid * kRedStride]);
        float2 a01 = f2(0.f, 0.f), a23 = f2(0.f, 0.f);
#pragma unroll 8
        for (int i = 0; i < kBlock / 4; ++i) {
          const float4 q = rowp[i];
          a01 = fadd2(a01, f2(q.x, q.y));
          a23 = fadd2(a23, f2(q.z, q.w));
        }
        v = (a01.x + a01.y) + (a23.x + a23.y);
      }
      if (dyn) {  // this tile's record (relative to its own minimum mt)
        SBS_CHECK(tile >= 0 && tile < p.dyn_n[0]);
        float* o = p.dyn_rec + (size_t)tile * p.part_stride;
        if (tid < D) o[kPartHdr + tid] = v;
        else o[3 + tid - D] = v;
        if (tid == 0) {
          o[0] = mt;
          o[1] = __int_as_float(tk);
          o[2] = __int_as_float(tf);
          o[7] = 0.0f;
        }
      } else {
        const float sa = (mr < kInf) ? __expf((mn - mr) * p.inv_lambda) : 0.0f;
        const float sb = (mt < kInf) ? __expf((mn - mt) * p.inv_lambda) : 0.0f;
        if (tid < D + 1) run = fmaf(run, sa, v * sb);
        else if (tid == D + 1) run = fmaf(run, sa * sa, v * (sb * sb));
        else run += v;
      }
    }
    if (SPLIT) {
      if (jk_less(mt, tk, h_m, h_k)) {
        h_m = mt;
        h_k = tk;
        h_f = tf;
      }
    } else if (tid == 0) {  // next header (the other buffer: this tile's readers may still be reading this one)
      const bool t = jk_less(mt, tk, s_rm[par], s_rk[par]);
      s_rm[par ^ 1] = t ? mt : s_rm[par];
      s_rk[par ^ 1] = t ? tk : s_rk[par];
      s_rf[par ^ 1] = t ? tf : s_rf[par];
    }
    if (dyn && tid == 0) s_nx[par] = nx;
    par ^= 1;
    if (!SPLIT) __syncthreads();  // (measured: throughput mode runs faster with the CTA's warps in step)
    if (dyn && tid == 0) {  // (the tile's record is written: barrier above)
      s_pend[n_pend++] = tile;
      if (n_pend == kDynBatch) dyn_arrive(p, s_pend, n_pend);
    }
  }
  // the next iteration's kernels may be scheduled.  Not for the CEM rollout: a select
  // kernel scheduled early, next to the running rollout, was measured 1.5x slower
  // after an L2 flush (its CTA then starts at grid completion, still PDL-ordered)
  if (FUSED || p.cem_cluster) griddep_launch_dependents();  // (the CEM cluster kernel starts on idle SMs)
  if constexpr (DYN) {
    SBS_CTS(3);
    if (tid == 0) dyn_arrive(p, s_pend, n_pend);
    dyn_merge_nodes(p, r, s_red, NR * kRedStride);
    SBS_CTS(1);  // (DYN: the CTA's node merges done)
    // the last CTA to leave re-arms the tile counter (every CTA has taken its last index)
    if (tid == 0 && atomicAdd(p.dyn_cnt + 1, 1) == (int)gridDim.x - 1) {
      p.dyn_cnt[0] = 0;
      p.dyn_cnt[1] = 0;
    }
  } else {
    if constexpr (EPI == EPI_MPPI && FUSED) {
      if (p.n_cta == 1 && !p.emit) {  // one CTA per robot: its running record is the robot's (merging one
        __shared__ __align__(16) float s_one[kPartHdr + SBS_MAX_D + 4];  // record is the identity): finish here
        __shared__ float s_ovar[SBS_MAX_D];
        __shared__ uint32_t s_opre[2];
        load_finish_inputs(p, r, s_ovar, s_opre);
        if (tid < D) s_one[kPartHdr + tid] = run;
        else if (tid < NR) s_one[3 + tid - D] = run;
        if (tid == 0) {
          s_one[0] = SPLIT ? h_m : s_rm[par];
          s_one[1] = __int_as_float(SPLIT ? h_k : s_rk[par]);
          s_one[2] = __int_as_float(SPLIT ? h_f : s_rf[par]);
        }
        __syncthreads();
        mppi_finish_record(p, r, s_one, s_ovar, s_opre);
        return;
      }
    }
    SBS_CHECK((int)blockIdx.x < p.n_cta && r < p.R);
    float* out = p.part + ((size_t)r * p.n_cta + blockIdx.x) * p.part_stride;
    if (EPI == EPI_MPPI) {
      if (tid < D) out[kPartHdr + tid] = run;
      else if (tid < NR) out[3 + tid - D] = run;
    } else if (tid == 0) {
      out[3] = 0.f;
      out[4] = 0.f;
      out[5] = SPLIT ? h_sj : s_rsj;
      out[6] = SPLIT ? h_nf : s_rnf;
    }
    if (tid == 0) {
      const int hp = EPI == EPI_MPPI ? par : 0;
      out[0] = SPLIT ? h_m : s_rm[hp];
      out[1] = __int_as_float(SPLIT ? h_k : s_rk[hp]);
      out[2] = __int_as_float(SPLIT ? h_f : s_rf[hp]);
      out[7] = 0.0f;
    }
    if (blockIdx.x == 0) SBS_TS(4);
    SBS_CTS(3);
    if (FUSED) {
      if (arrive_last(p.counter + r, gridDim.x)) {
        SBS_TS(5);
        if (p.emit) {  // world > 1: this rank's record per robot (the exchange and rank-order merge follow)
          if (EPI == EPI_MPPI) mppi_merge_block<true>(p, r, p.emit, s_red, NR * kRedStride);
          else merge_diag(p, r, p.emit + (size_t)r * p.ex_stride, true);
          publish_to_peers(p);
        } else {
          if (EPI == EPI_MPPI) mppi_merge_block<false>(p, r, nullptr, s_red, NR * kRedStride);
          else naive_finalize_block<P>(p, r, s);
        }
        SBS_TS(6);
      }
    }
  }
}

// stand-alone merge (world > 1: rank partial before / final merge after the all-gather)
template <bool EMIT>
__global__ void __launch_bounds__(128) sbs_mppi_finalize(const __grid_constant__ Params p, float* emit) {
  __shared__ __align__(16) float stage[4096];
  if (!EMIT && p.dyn && p.R == 1 && p.n_cta <= 128)  // the ranks' tree-node records: the root's merge (GPU-count invariant)
    dyn_root_finish(p, blockIdx.x, part_rec(p, blockIdx.x, 0), p.n_cta, stage, 4096);
  else
    mppi_merge_block<EMIT>(p, blockIdx.x, emit, stage, 4096);
}

// ---------------------------------------------------------------------------
// Elite selection (a6; Alg. 1 lines 3-5, L4): the K_e smallest keys (J, k).
// Radix select on order-preserving 32-bit keys of J (NaN -> +inf, -0 -> +0):
// four 8-bit passes with warp-aggregated shared-memory histograms and a
// parallel digit search, then an index-ordered compaction that takes all
// keys < T and the lowest-index ties == T.  One CTA per robot.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cost_key(float J) {
  if (J != J) J = kInf;
  if (J == 0.0f) J = 0.0f;  // -0 -> +0
  const uint32_t u = __float_as_uint(J);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// inverse of cost_key (for the normalised costs)
__device__ __forceinline__ float key_cost(uint32_t key) {
  return __uint_as_float((key & 0x80000000u) ? (key ^ 0x80000000u) : ~key);
}

constexpr int kSelBlock = 1024;
constexpr int kHistPad = 257;                       // per-warp histogram stride (bank-conflict free)
constexpr int kSelHistWords = (kSelBlock / 32) * kHistPad;
constexpr int kSelSmemBytes = 200 * 1024;           // dynamic shared memory of the select kernels
constexpr int kSelSmemKeys = kSelSmemBytes / 4 - kSelHistWords;

// smem: [kSelHistWords] per-warp histograms, then the keys when K <= kSelSmemKeys
static __device__ void select_block(const float* J, int64_t K, int64_t K_e, int64_t k_begin, int64_t* elite,
                             float* eJ, uint32_t* smem) {
  __shared__ uint32_t s_prefix, s_want;
  __shared__ uint32_t s_wsum[kSelBlock / 32];
  uint32_t* whist = smem;
  uint32_t* keys = smem + kSelHistWords;
  const bool staged = K <= kSelSmemKeys;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  if (tid == 0) {
    s_prefix = 0;
    s_want = (uint32_t)K_e;
  }
  if (staged)
    for (int64_t k = tid; k < K; k += blockDim.x) keys[k] = cost_key(J[k]);
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
    for (int i = tid; i < nw * kHistPad; i += blockDim.x) whist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix, want = s_want;
    uint32_t* my = whist + warp * kHistPad;
    const int64_t K_round = ((K + 31) / 32) * 32;
    for (int64_t k = tid; k < K_round; k += blockDim.x) {
      uint32_t dgt = 0xFFFFFFFFu;
      if (k < K) {
        const uint32_t key = staged ? keys[k] : cost_key(J[k]);
        if ((key & hmask) == prefix) dgt = (key >> shift) & 255u;
      }
      // up to 3 leader rounds absorb the dominant digits with one atomic each (costs
      // cluster in a few bins in the high passes), the rest add directly
      unsigned act = __ballot_sync(0xffffffffu, dgt != 0xFFFFFFFFu);
#pragma unroll
      for (int it = 0; it < 3 && act; ++it) {
        const int leader = __ffs(act) - 1;
        const uint32_t d = __shfl_sync(0xffffffffu, dgt, leader);
        const unsigned m = __ballot_sync(0xffffffffu, dgt == d) & act;
        if (lane == leader) atomicAdd(&my[d], (uint32_t)__popc(m));
        if (m & (1u << lane)) dgt = 0xFFFFFFFFu;
        act &= ~m;
      }
      if (dgt != 0xFFFFFFFFu) atomicAdd(&my[dgt], 1u);
    }
    __syncthreads();
    // sum the warp histograms per bin, inclusive scan over the 256 bins, find the bin of rank `want`
    if (tid < 256) {
      uint32_t h = 0;
      for (int w = 0; w < nw; ++w) h += whist[w * kHistPad + tid];
      uint32_t x = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_wsum[warp] = x;
      whist[tid] = x - h;  // exclusive prefix within the warp (bins of warp 0's histogram are no longer needed)
      whist[256] = 0;
    }
    __syncthreads();
    if (tid < 256) {
      uint32_t off = 0;
      for (int w = 0; w < warp; ++w) off += s_wsum[w];
      const uint32_t excl = whist[tid] + off;
      const uint32_t incl = (tid & 31) == 31 ? s_wsum[warp] + off : whist[tid + 1] + off;
      if (excl < want && want <= incl) {  // exactly one bin
        s_prefix = prefix | ((uint32_t)tid << shift);
        s_want = want - excl;
      }
    }
    __syncthreads();
  }
  const uint32_t T = s_prefix;
  const uint32_t n_eq = s_want;  // ties at T to take, lowest indices first
  uint32_t sel_base = 0, eq_base = 0;
  for (int64_t base = 0; base < K; base += blockDim.x) {
    const int64_t k = base + tid;
    bool lt = false, eq = false;
    if (k < K) {
      const uint32_t key = staged ? keys[k] : cost_key(J[k]);
      lt = key < T;
      eq = key == T;
    }
    const unsigned eqb = __ballot_sync(0xffffffffu, eq);
    const unsigned ltb = __ballot_sync(0xffffffffu, lt);
    if (lane == 0) s_wsum[warp] = __popc(eqb) | ((uint32_t)__popc(ltb) << 16);
    __syncthreads();
    uint32_t eq_before = eq_base + __popc(eqb & ((1u << lane) - 1u));
    uint32_t lt_before = __popc(ltb & ((1u << lane) - 1u));
    uint32_t eq_tot = 0, lt_tot = 0;
    for (int w = 0; w < nw; ++w) {
      const uint32_t c = s_wsum[w];
      if (w < warp) {
        eq_before += c & 0xFFFFu;
        lt_before += c >> 16;
      }
      eq_tot += c & 0xFFFFu;
      lt_tot += c >> 16;
    }
    // selected = lt, or eq within the first n_eq ties; position = number selected before me
    const uint32_t eq_sel_chunk0 = eq_base < n_eq ? eq_base : n_eq;
    const uint32_t eq_sel_before_me = (eq_before < n_eq ? eq_before : n_eq) - eq_sel_chunk0;
    const bool sel = lt || (eq && eq_before < n_eq);
    if (sel) {
      const uint32_t pos = sel_base + lt_before + eq_sel_before_me;
      SBS_CHECK(pos < (uint64_t)K_e);
      elite[pos] = k_begin + k;
      if (eJ) eJ[pos] = J[k];
    }
    const uint32_t eq_end = eq_base + eq_tot;
    sel_base += lt_tot + ((eq_end < n_eq ? eq_end : n_eq) - eq_sel_chunk0);
    eq_base = eq_end;
    __syncthreads();
  }
}

// Fast path for K <= kSelSmallMax: every thread keeps a contiguous run of at most
// 16 keys in registers.  Three passes over 11-, 11- and 10-bit digits (2048 plain
// counters in shared memory; measured 2 us faster per CEM iteration than two passes
// over 16-bit digits with 65536 packed counters, which are kept behind
// SBS_SEL_DIGITS=16) give the exact K_e-th smallest key T and the number of ties at T
// to take; one block scan of per-thread (lt, eq) counts then places the elites in index
// order.
constexpr int kSelSmallMax = 16384;
constexpr int kSelKPT = kSelSmallMax / kSelBlock;
constexpr int kSelSmallSmemBytes = 32768 * 4;
#if defined(SBS_TU_COMMON)
constexpr int kSelTs = 0;  // SBS_TIMING slots of select_block_small: the select kernel's ...
#else
constexpr int kSelTs = 16;  // ... or the CEM cluster kernel's
#endif
constexpr int kSelHdrMax = 256;  // rollout records whose headers the select kernel stages (world = 1)

// exclusive block scan of v over kSelBlock threads; returns the total in *tot
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_w, uint32_t* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = s_w[lane];
    uint32_t wx = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wx, o);
      if (lane >= o) wx += y;
    }
    s_w[lane] = wx - w;       // exclusive warp offsets
    if (lane == 31) s_w[32] = wx;
  }
  __syncthreads();
  const uint32_t r = s_w[warp] + x - v;
  *tot = s_w[32];
  __syncthreads();
  return r;
}

// 16-bit digit pass: count keys with (key & pmask) == pref by digit (key >> sh) & 0xFFFF,
// find digit B with rank `want` inside; returns B and the count strictly below it.
__device__ __forceinline__ void zero_hist16(uint32_t* hist) {  // 32768 words, 16-byte stores
  uint4* h4 = reinterpret_cast<uint4*>(hist);
  for (int i = threadIdx.x; i < 32768 / 4; i += kSelBlock) h4[i] = make_uint4(0u, 0u, 0u, 0u);
}

static __device__ void digit16_pass(const uint32_t (&key)[kSelKPT], int nk, uint32_t pmask, uint32_t pref, int sh,
                             uint32_t want, uint32_t* hist, uint32_t* s_w, uint32_t* s_res, bool zeroed = false) {
  const int tid = threadIdx.x;
  if (!zeroed) zero_hist16(hist);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSelKPT; ++i) {
    if (i >= nk) break;
    if ((key[i] & pmask) == pref) {
      const uint32_t d = (key[i] >> sh) & 0xFFFFu;
      atomicAdd(&hist[d >> 1], 1u << ((d & 1u) << 4));
    }
  }
  __syncthreads();
  // thread t owns digits [64 t, 64 t + 64)
  uint32_t loc = 0;
  for (int w = 0; w < 32; ++w) {
    const uint32_t h = hist[tid * 32 + ((w + tid) & 31)];  // rotated start: no bank conflicts
    loc += (h & 0xFFFFu) + (h >> 16);
  }
  uint32_t tot;
  const uint32_t base = block_excl_scan(loc, s_w, &tot);
  // the warp holding the digit range that contains rank `want` resolves the digit: its
  // lanes take one word (two digits) each of the owner's range, then a warp scan
  const uint32_t owner = __ballot_sync(0xffffffffu, base < want && want <= base + loc);
  if (owner) {
    const int ol = __ffs(owner) - 1, lane = tid & 31;
    const int t = (tid & ~31) + ol;
    const uint32_t obase = __shfl_sync(0xffffffffu, base, ol);
    const uint32_t h = hist[t * 32 + lane];
    const uint32_t c0 = h & 0xFFFFu, c1 = h >> 16;
    uint32_t incl = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t cum = obase + incl - (c0 + c1);  // count below this word's first digit
    const bool hit0 = cum + c0 >= want, hit1 = cum + c0 + c1 >= want;
    const uint32_t first = __ballot_sync(0xffffffffu, hit1);
    if (lane == __ffs(first) - 1) {
      s_res[0] = (uint32_t)(t * 64 + 2 * lane + (hit0 ? 0 : 1));
      s_res[1] = hit0 ? cum : cum + c0;
    }
  }
  __syncthreads();
}

// BITS-bit digit pass (BITS <= 11): 2^BITS plain counters; thread t owns digits
// [t 2^BITS / kSelBlock, ...).  Same contract as digit16_pass.
#ifndef SBS_SEL_DIGITS
#define SBS_SEL_DIGITS 11
#endif
template <int BITS>
static __device__ void digit_pass_narrow(const uint32_t (&key)[kSelKPT], int nk, uint32_t pmask, uint32_t pref,
                                         int sh, uint32_t want, uint32_t* hist, uint32_t* s_w, uint32_t* s_res) {
  constexpr int NB = 1 << BITS, PER = NB / kSelBlock > 0 ? NB / kSelBlock : 1;
  const int tid = threadIdx.x;
  for (int i = tid; i < NB; i += kSelBlock) hist[i] = 0u;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSelKPT; ++i) {
    if (i >= nk) break;
    if ((key[i] & pmask) == pref) atomicAdd(&hist[(key[i] >> sh) & (NB - 1)], 1u);
  }
  __syncthreads();
  uint32_t c[PER], loc = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int dgt = tid * PER + u;
    c[u] = dgt < NB ? hist[dgt] : 0u;
    loc += c[u];
  }
  uint32_t tot;
  const uint32_t base = block_excl_scan(loc, s_w, &tot);
  if (base < want && want <= base + loc) {  // this thread's digits hold rank `want`
    uint32_t cum = base;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      if (cum + c[u] >= want) {
        s_res[0] = (uint32_t)(tid * PER + u);
        s_res[1] = cum;
        break;
      }
      cum += c[u];
    }
  }
  __syncthreads();
}

static __device__ void select_block_small(const float* J, int K, int K_e, int64_t k_begin, int64_t* elite, float* eJ,
                                          uint32_t* hist, bool zeroed = false, bool to_global = true) {
  __shared__ uint32_t s_w[33];
  __shared__ uint32_t s_res[2];
  const int tid = threadIdx.x;
  const int per = (K + kSelBlock - 1) / kSelBlock;
  const int k0 = tid * per;
  const int nk = max(0, min(per, K - k0));
  uint32_t key[kSelKPT];
#pragma unroll
  for (int i = 0; i < kSelKPT; ++i) key[i] = i < nk ? cost_key(J[k0 + i]) : 0xFFFFFFFFu;
  if (blockIdx.x == 0) SBS_TS(kSelTs + 2);
#if SBS_SEL_DIGITS == 11
  // three narrow passes (bits 31..21, 20..10, 9..0): 2048-bin histograms, cheap scans
  (void)zeroed;
  digit_pass_narrow<11>(key, nk, 0u, 0u, 21, (uint32_t)K_e, hist, s_w, s_res);
  const uint32_t dA = s_res[0], bA = s_res[1];
  digit_pass_narrow<11>(key, nk, 0xFFE00000u, dA << 21, 10, (uint32_t)K_e - bA, hist, s_w, s_res);
  if (blockIdx.x == 0) SBS_TS(kSelTs + 3);
  const uint32_t dB = s_res[0], bB = s_res[1];
  digit_pass_narrow<10>(key, nk, 0xFFFFFC00u, (dA << 21) | (dB << 10), 0, (uint32_t)K_e - bA - bB, hist, s_w, s_res);
  if (blockIdx.x == 0) SBS_TS(kSelTs + 4);
  const uint32_t T = (dA << 21) | (dB << 10) | s_res[0];
  const uint32_t n_eq = (uint32_t)K_e - bA - bB - s_res[1];  // ties at T to take, lowest indices first
#else
  digit16_pass(key, nk, 0u, 0u, 16, (uint32_t)K_e, hist, s_w, s_res, zeroed);
  if (blockIdx.x == 0) SBS_TS(kSelTs + 3);
  const uint32_t hi = s_res[0], below_hi = s_res[1];
  digit16_pass(key, nk, 0xFFFF0000u, hi << 16, 0, (uint32_t)K_e - below_hi, hist, s_w, s_res);
  if (blockIdx.x == 0) SBS_TS(kSelTs + 4);
  const uint32_t T = (hi << 16) | s_res[0];
  const uint32_t n_eq = (uint32_t)K_e - below_hi - s_res[1];  // ties at T to take, lowest indices first
#endif
  uint32_t lt = 0, eq = 0;
#pragma unroll
  for (int i = 0; i < kSelKPT; ++i) {
    if (i >= nk) break;
    lt += key[i] < T;
    eq += key[i] == T;
  }
  uint32_t t1;  // one scan of both counts, packed (each total <= K <= 16384 < 2^16)
  const uint32_t both = block_excl_scan(lt | (eq << 16), s_w, &t1);
  const uint32_t lt_before = both & 0xFFFFu;
  uint32_t eq_before = both >> 16;
  uint32_t pos = lt_before + min(eq_before, n_eq);
  if (blockIdx.x == 0) SBS_TS(kSelTs + 5);
  // the compacted list goes through shared memory (the histogram is free now) so that
  // the global writes are coalesced; scattered per-lane writes were measured at ~3 us
  const bool stage = (size_t)K_e * (sizeof(int64_t) + sizeof(float)) <= (size_t)kSelSmallSmemBytes;
  int64_t* s_el = reinterpret_cast<int64_t*>(hist);
  float* s_eJ = reinterpret_cast<float*>(s_el + K_e);
#pragma unroll
  for (int i = 0; i < kSelKPT; ++i) {
    if (i >= nk) break;
    const bool is_eq = key[i] == T;
    const bool take = key[i] < T || (is_eq && eq_before < n_eq);  // ties: lowest indices first
    eq_before += is_eq ? 1u : 0u;
    if (take) {
      SBS_CHECK(pos < (uint32_t)K_e);
      const float Jv = key_cost(key[i]);  // (J itself up to NaN -> +inf, -0 -> +0)
      if (stage) {
        s_eJ[pos] = Jv;
        s_el[pos] = k_begin + k0 + i;
      } else {
        if (eJ) eJ[pos] = Jv;
        elite[pos] = k_begin + k0 + i;
      }
    }
    pos += take ? 1u : 0u;
  }
  if (stage) {  // (to_global false: the list stays staged at the start of `hist`, caller's use)
    __syncthreads();
    for (int e = tid; to_global && e < K_e; e += blockDim.x) {
      elite[e] = s_el[e];
      if (eJ) eJ[e] = s_eJ[e];
    }
  }
  if (blockIdx.x == 0) SBS_TS(kSelTs + 7);
}


// Select kernels, one CTA per robot.
//   SEL_LOCAL (world = 1): rollout records -> p.sdiag; K_e smallest of J -> p.elite, p.elite_J.
//   SEL_EMIT  (world > 1, before the all-gather): this rank's record [8 header | K_e J | K_e k]
//             (the local K_e smallest, index order) -> emit[r].
//   SEL_MERGE (after the all-gather; p.part = [world][R] gathered records): rank-order
//             header merge -> p.sdiag; the K_e smallest of the world*K_e candidates,
//             concatenated in rank order (= global index order, so position order is
//             the (J, k) tie order) -> p.elite (global k, index order), p.elite_J.
enum { SEL_LOCAL = 0, SEL_EMIT = 1, SEL_MERGE = 2 };

#if defined(SBS_TU_COMMON)
template <int MODE, bool SMALL>
__global__ void __launch_bounds__(kSelBlock) sbs_select_kernel(const __grid_constant__ Params p, float* emit) {
  extern __shared__ uint32_t sel_smem[];
  const int r = blockIdx.x, tid = threadIdx.x;
  if (SMALL && SBS_SEL_DIGITS == 16) zero_hist16(sel_smem);  // (independent of the rollout: overlaps its tail under PDL)
  griddep_wait();               // the rollout's J and records
  griddep_launch_dependents();  // the elite kernel may be scheduled now (it waits for us)
  const int64_t Ke = p.n_elite;
  float* hdr = MODE == SEL_EMIT ? emit + (size_t)r * p.ex_stride : p.sdiag + (size_t)r * 8;
  if (blockIdx.x == 0) SBS_TS(0);
  // world = 1: the rollout records' headers arrive by cp.async while the selection runs
  // (their diagnostics are merged at the end, off the selection's critical path)
  __shared__ __align__(16) float s_hdr[kSelHdrMax * 8];
  const bool staged = MODE == SEL_LOCAL && SMALL && p.n_cta <= kSelHdrMax && p.part_c_stride == 1;
  if (staged) {
    for (int c = tid; c < p.n_cta; c += blockDim.x) {
      cp_async16(&s_hdr[8 * c], part_rec(p, r, c));
      cp_async16(&s_hdr[8 * c + 4], part_rec(p, r, c) + 4);
    }
  } else {
    merge_diag(p, r, hdr, MODE == SEL_EMIT);
  }
  if (blockIdx.x == 0) SBS_TS(1);
  const float* J = p.J + (size_t)r * p.K_local;
  int64_t K = p.K_local, kb = p.k_begin;
  if (MODE == SEL_MERGE) {
    float* cand = p.cand + (size_t)r * p.n_cta * Ke;
    for (int64_t i = tid; i < (int64_t)p.n_cta * Ke; i += blockDim.x)
      cand[i] = __ldcg(part_rec(p, r, (int)(i / Ke)) + kPartHdr + i % Ke);
    __syncthreads();
    J = cand;
    K = (int64_t)p.n_cta * Ke;
    kb = 0;
  }
  int64_t* el = p.elite + (size_t)r * Ke;
  float* eJ = p.elite_J + (size_t)r * Ke;
  if (SMALL) select_block_small(J, (int)K, (int)Ke, kb, el, eJ, sel_smem, true);
  else select_block(J, K, Ke, kb, el, eJ, sel_smem);
  if (staged) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (blockIdx.x == 0) SBS_TS(8);
  if (staged) merge_diag(p, r, hdr, false, s_hdr);
  if (blockIdx.x == 0) SBS_TS(6);

  if (MODE == SEL_EMIT) {
    float* o = emit + (size_t)r * p.ex_stride + kPartHdr;
    for (int64_t e = tid; e < Ke; e += blockDim.x) {
      o[e] = eJ[e];
      o[Ke + e] = __int_as_float((int)el[e]);
    }
    publish_to_peers(p);
  }
  if (MODE == SEL_MERGE) {
    for (int64_t e = tid; e < Ke; e += blockDim.x) {
      const int64_t pos = el[e];
      el[e] = (int64_t)__float_as_int(__ldcg(part_rec(p, r, (int)(pos / Ke)) + kPartHdr + Ke + pos % Ke));
    }
  }
}


__global__ void __launch_bounds__(kSelBlock) sbs_select_raw_kernel(const float* J, int64_t K, int64_t K_e,
                                                                   int64_t* idx) {
  extern __shared__ uint32_t sel_smem[];
  select_block(J, K, K_e, 0, idx, nullptr, sel_smem);
}

__global__ void __launch_bounds__(kSelBlock) sbs_select_small_raw_kernel(const float* J, int64_t K, int64_t K_e,
                                                                           int64_t* idx) {
  extern __shared__ uint32_t sel_smem[];
  select_block_small(J, (int)K, (int)K_e, 0, idx, nullptr, sel_smem);
}


// ---- tests only: the normative noise on given Philox words, and the Philox rounds on
//      given counters / keys next to cuRAND's curand_Philox4x32_10 (same definition) ----
__global__ void sbs_debug_noise_kernel(const uint4* w, int64_t n, float4* z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 v = w[i];
  float o[4];
  box_muller_x2(U4{v.x, v.y, v.z, v.w}, o);
  z[i] = make_float4(o[0], o[1], o[2], o[3]);
}
__global__ void sbs_debug_philox_kernel(const uint4* ctr, const uint2* key, int64_t n, uint4* ours, uint4* curand_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 c = ctr[i];
  const uint2 k = key[i];
  const U4 a = philox4x32_10(c.x, c.y, c.z, c.w, k.x, k.y);
  uint32_t rk[10][2];
  for (int r = 0; r < 10; ++r) {
    rk[r][0] = k.x + (uint32_t)r * 0x9E3779B9u;
    rk[r][1] = k.y + (uint32_t)r * 0xBB67AE85u;
  }
  const U4 b = philox4x32_10_rk(c.x, c.y, c.z, c.w, rk);  // the round-key form the rollout uses
  ours[2 * i] = make_uint4(a.x, a.y, a.z, a.w);
  ours[2 * i + 1] = make_uint4(b.x, b.y, b.z, b.w);
  curand_out[i] = curand_Philox4x32_10(c, k);
}
cudaError_t launch_debug_noise(const void* w, int64_t n, void* z, cudaStream_t s) {
  sbs_debug_noise_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(static_cast<const uint4*>(w), n,
                                                                       static_cast<float4*>(z));
  return cudaGetLastError();
}
cudaError_t launch_debug_philox(const void* ctr, const void* key, int64_t n, void* ours, void* curand_out,
                                cudaStream_t s) {
  sbs_debug_philox_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      static_cast<const uint4*>(ctr), static_cast<const uint2*>(key), n, static_cast<uint4*>(ours),
      static_cast<uint4*>(curand_out));
  return cudaGetLastError();
}
#endif  // SBS_TU_COMMON

// ---------------------------------------------------------------------------
// sbs_elite_kernel (CEM, Alg. 1 UpdateMean / UpdateCov, L17): grid (n_eblk, R),
// block 32 x 3P: warp q regenerates Philox block q (coordinates 4q..4q+3) of
// the CTA's 32 elites from the counter RNG (no theta buffer in HBM), then
// reduces shifted moments about mu' over its lanes: S1 = sum (theta - mu'),
// S2 = sum (theta - mu')^2.  The last CTA of a robot merges the records in
// order and finishes: mean = mu' + S1/n, var = max(S2/n - (S1/n)^2, floor).
// ---------------------------------------------------------------------------
// The end of a CEM iteration (Alg. 1 UpdateMean / UpdateCov, L17), one CTA: from the merged
// moments s_tot = [S1[D], n, S2[D]] about mu' and the select kernel's diagnostics s_diag =
// [J_min, k_min, f_min, sum J, n_finite]: mean = mu' + S1/n, var = max(S2/n - (S1/n)^2,
// floor); every sample diverged keeps mean and var.
template <int P>
static __device__ void cem_finish(const Params& p, int r, const RobotSmem& s, const float* s_tot,
                                  const float* s_diag, const uint32_t* s_pre, float* s_mean, float* s_var) {
  constexpr int D = 12 * P;
  const int tid = threadIdx.x;
  const Best b{s_diag[0], __float_as_int(s_diag[1]), __float_as_int(s_diag[2])};
  const float ne = s_tot[D];
  const bool all_div = !(ne > 0.f);
  const float inv = all_div ? 0.f : 1.0f / ne;
  for (int d = tid; d < D; d += blockDim.x) {
    if (all_div) {
      s_mean[d] = p.mean[(size_t)r * D + d];
      s_var[d] = p.var[(size_t)r * D + d];
    } else {
      const float m1 = s_tot[d] * inv;
      s_mean[d] = s.mu[d] + m1;
      s_var[d] = fmaxf(fmaf(-m1, m1, s_tot[D + 1 + d] * inv), p.var_floor[d % 3]);
    }
  }
  __syncthreads();
  const int fi = all_div ? s.cur_idx : b.f;
  for (int d = tid; d < D; d += blockDim.x) {
    p.mean[(size_t)r * D + d] = s_mean[d];
    p.var[(size_t)r * D + d] = s_var[d];
  }
  if (tid == 0) {
    p.fidx[r] = fi;
    p.best[r] = b.k;
  }
  write_output(p, r, all_div ? SBS_WARN_ALL_DIVERGED : SBS_OK, s_mean, s_var, fi, b.m,
               s_diag[4] > 0.f ? s_diag[3] / s_diag[4] : kInf, ne, ne, (int)((float)p.K_global - s_diag[4]), s_pre);
}

constexpr int kEliteGroup = 32;  // elites per CTA

// One warp, Philox block q (coordinates 4q..4q+3) of a group of 32 elites (lane = elite):
// regenerate theta from the counter RNG, then the group's shifted moments about mu',
// S1 = sum (theta - mu') and S2 = sum (theta - mu')^2 for the 4 coordinates, and the
// finite count n.  The 8 lane sums run as a transposing butterfly: at lane bits 4, 3, 2
// each lane keeps half of its values and adds the partner's copy of that half, then two
// plain levels finish; value j = 4 b4 + 2 b3 + b2 (S1 of coordinate 4q + j for j < 4,
// S2 of coordinate 4q + j - 4 after) ends on lanes 4j..4j+3.
struct GroupMoments {
  float t;  // this lane's value total
  int j;    // its value index (lane >> 2)
  float n;  // finite count (every lane)
};
__device__ __forceinline__ GroupMoments elite_group_moments(const Params& p, const RobotSmem& s, uint32_t robot_g,
                                                            bool has_e, int64_t k, float Je, int q) {
  const int lane = threadIdx.x & 31;
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const bool fin = has_e && Je < kInf;  // diverged samples never enter the moments (L17)
  if (fin) {
    float th4[4];
    sample_block(p, robot_g, k, q, s, th4);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = th4[i] - s.mu[4 * q + i];
      v[4 + i] = v[i] * v[i];
    }
  }
  float w4[4], w2[2];
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float keep = b4 ? v[4 + i] : v[i], give = b4 ? v[i] : v[4 + i];
    w4[i] = keep + __shfl_xor_sync(0xffffffffu, give, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float keep = b3 ? w4[2 + i] : w4[i], give = b3 ? w4[i] : w4[2 + i];
    w2[i] = keep + __shfl_xor_sync(0xffffffffu, give, 8);
  }
  GroupMoments m;
  {
    const float keep = b2 ? w2[1] : w2[0], give = b2 ? w2[0] : w2[1];
    m.t = keep + __shfl_xor_sync(0xffffffffu, give, 4);
  }
  m.t += __shfl_xor_sync(0xffffffffu, m.t, 2);
  m.t += __shfl_xor_sync(0xffffffffu, m.t, 1);
  m.j = lane >> 2;
  m.n = (float)__popc(__ballot_sync(0xffffffffu, fin));  // (exact)
  return m;
}
// ... into the record rec = [S1[D], n, S2[D]] (lanes 4j; n by warp q = 0)
template <int P>
__device__ __forceinline__ void elite_group_record(const Params& p, const RobotSmem& s, uint32_t robot_g, bool has_e,
                                                   int64_t k, float Je, int q, float* rec) {
  constexpr int D = 12 * P;
  const GroupMoments m = elite_group_moments(p, s, robot_g, has_e, k, Je, q);
  const int lane = threadIdx.x & 31;
  if ((lane & 3) == 0) rec[m.j < 4 ? 4 * q + m.j : D + 1 + 4 * q + m.j - 4] = m.t;
  if (q == 0 && lane == 0) rec[D] = m.n;
}

template <int P>
__global__ void __launch_bounds__(32 * 3 * P) sbs_elite_kernel(const __grid_constant__ Params p) {
  constexpr int D = 12 * P;
  __shared__ RobotSmem s;
  __shared__ float s_mean[D], s_var[D];
  __shared__ float s_tot[2 * D + 1];
  constexpr int kChunk = 32;  // elite records staged per round trip in the last CTA
  __shared__ __align__(16) float s_stage[kChunk * kEPartStride];
  __shared__ float s_diag[5];
  const int r = blockIdx.y, tid = threadIdx.x, lane = tid & 31, q = tid >> 5;
  const int64_t e = (int64_t)blockIdx.x * kEliteGroup + lane;
  load_robot(p, r, s, false);  // (not written by the select kernel: may overlap it)
  griddep_wait();              // the select kernel's elite list and diagnostics
  if (blockIdx.x == 0) SBS_TS(11);
  const bool has_e = e < p.n_elite;
  SBS_CHECK((int)blockIdx.x < p.n_eblk && r < p.R);
  const int64_t k = has_e ? p.elite[(size_t)r * p.n_elite + e] : 0;
  const float Je = has_e ? p.elite_J[(size_t)r * p.n_elite + e] : kInf;
  SBS_CHECK(k >= 0 && k < p.K_global);
  __syncthreads();
  elite_group_record<P>(p, s, (uint32_t)(p.robot_offset + r), has_e, k, Je, q,
                        p.epart + ((size_t)r * gridDim.x + blockIdx.x) * kEPartStride);
  if (!arrive_last(p.ecounter + r, gridDim.x)) return;
  // ---- last CTA: merge the elite records in order, finish the iteration ----
  __shared__ uint32_t s_pre[2];
  const float* sd = p.sdiag + (size_t)r * 8;
  if (tid == 0) {  // issued with the record loads below
    s_pre[0] = robot_in(p, r)->phase_q32;
    s_pre[1] = step_iter(p);
    for (int i = 0; i < 5; ++i) s_diag[i] = sd[i];  // rank-1 sample and diagnostics (select kernel)
  }
  {
    float a0 = 0.f;  // row tid (2D + 1 <= blockDim = 8D); records summed in block order
    for (int b0 = 0; b0 < (int)gridDim.x; b0 += kChunk) {
      const int nb = min(kChunk, (int)gridDim.x - b0);
      stage_issue(s_stage, p.epart + ((size_t)r * gridDim.x + b0) * kEPartStride, nb * kEPartStride);
      stage_wait();
      __syncthreads();
      if (tid < 2 * D + 1)
        for (int b = 0; b < nb; ++b) a0 += s_stage[b * kEPartStride + tid];
      __syncthreads();
    }
    if (tid < 2 * D + 1) s_tot[tid] = a0;
  }
  __syncthreads();
  cem_finish<P>(p, r, s, s_tot, s_diag, s_pre, s_mean, s_var);
  SBS_TS(12);
}


// ---------------------------------------------------------------------------
// sbs_cem_cluster_kernel (CEM at world = 1, K <= kSelSmallMax, K_e <= 32 kCemMaxGroups,
// diagonal covariance): the select kernel and the elite kernel in one launch, one
// thread-block cluster of C = p.cem_cluster CTAs per robot (grid (C, R)).  The CTAs
// exchange data only by asynchronous stores into each other's shared memory that
// complete on the receiver's transaction barrier (st.async + mbarrier complete_tx):
//   CTA 1, while CTA 0 selects: the robot's sampling distribution (warm-shifted mean,
//     sigma), the rollout records' diagnostics and the output's phase / iteration
//     -> CTA 0 (header barrier);
//   CTA 0: the K_e elites (select_block_small, the select kernel's code) -> each CTA
//     its groups of 32 (group g in CTA g mod C);
//   every CTA: regenerates its groups, one warp per (group, Philox block q)
//     (elite_group_moments, the elite kernel's arithmetic), the group records -> CTA 0
//     (record barrier; CTA 0's own groups by plain stores);
//   CTA 0: sums the records in group order (the elite kernel's last-CTA order) and
//     finishes (cem_finish).
// Same arithmetic in the same order as sbs_select_kernel + sbs_elite_kernel, so the
// results are bitwise the same; what goes is the second launch, the elite list's round
// trip through global memory and the arrival counter.  Every CTA waits only for data
// addressed to it, so a CTA may leave once its last stores are issued.
// ---------------------------------------------------------------------------
constexpr int kCemMaxGroups = 64;  // K_e <= 2048
constexpr int kCemSlots = kCemMaxGroups / 8;  // groups per CTA at the smallest cluster (8)
constexpr int kCemRecStride = 2 * SBS_MAX_D + 4;  // cluster record [S1[D] | S2[D] | n, pad]: 16-byte aligned parts
constexpr int kCemSmemBytes = kSelSmallSmemBytes + kCemMaxGroups * kCemRecStride * 4;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t n;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return n;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared::cluster address of a shared variable's copy in CTA `rank`
__device__ __forceinline__ uint32_t cl_addr(const void* local, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(local)), "r"(rank));
  return a;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {  // phase 0 of a fresh barrier
  uint32_t done = 0;
  const long long t0 = clock64();
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar))
        : "memory");
    if (!done && clock64() - t0 > kSpinLimit) __trap();  // (missing bytes: fail the launch, never hang)
  }
}
__device__ __forceinline__ void st_async(uint32_t addr, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t addr, uint32_t v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr), "r"(v),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t addr, int64_t v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr), "l"(v),
               "r"(bar)
               : "memory");
}

template <int P>
__global__ void __launch_bounds__(kSelBlock) sbs_cem_cluster_kernel(const __grid_constant__ Params p) {
  constexpr int D = 12 * P, NQ = 3 * P, RS = 2 * D + 4;
  // dynamic: [select histogram / staged elite list (CTA 0) | group records [n_eblk][RS] (CTA 0)]
  extern __shared__ __align__(16) uint32_t cem_smem[];
  float* recs = reinterpret_cast<float*>(cem_smem + kSelSmallSmemBytes / 4);
  __shared__ RobotSmem s;
  __shared__ __align__(8) int64_t s_ek[kCemSlots * kEliteGroup];  // this CTA's elites (k, J) (CTAs > 0)
  __shared__ float s_eJ[kCemSlots * kEliteGroup];
  __shared__ float s_mean[D], s_var[D], s_tot[2 * D + 1], s_diag[5];
  __shared__ uint32_t s_pre[2];
  __shared__ __align__(8) uint64_t s_bar[2];  // [0]: elites (CTAs > 0) / records (CTA 0); [1]: header (CTA 0)
  const int r = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank(), C = cluster_size();
  const int Ke = (int)p.n_elite, G = p.n_eblk;
  SBS_CHECK(G <= kCemMaxGroups && (int)C * kCemSlots >= G && C >= 2 && p.K_local <= kSelSmallMax && r < p.R);
  const int mine = (G - (int)rank + (int)C - 1) / (int)C;  // groups rank, rank + C, ...
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (rank == 0) {  // bytes CTA 0 receives: the other CTAs' group records, CTA 1's header
      const int remote = G - (G + (int)C - 1) / (int)C;
      mbar_expect_tx(&s_bar[0], (uint32_t)(remote * (NQ * 32 + 4)));
      mbar_expect_tx(&s_bar[1], (uint32_t)((2 * D + 9) * 4));
    } else {  // this CTA's elites (k, J): 12 bytes each
      int n = 0;
      for (int sl = 0; sl < mine; ++sl) n += max(0, min(kEliteGroup, Ke - ((int)rank + (int)C * sl) * kEliteGroup));
      mbar_expect_tx(&s_bar[0], (uint32_t)(12 * n));
    }
  }
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // barriers initialised (waited before use)
  if (rank != 0) {
    load_robot(p, r, s, false);  // (the distribution: not written by the rollout)
    griddep_wait();
    griddep_launch_dependents();
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (rank == 1) {  // the header CTA 0 needs, while it selects
      merge_diag(p, r, s_diag, false);
      __syncthreads();
      const uint32_t bar = cl_addr(&s_bar[1], 0);
      for (int d = tid; d < D; d += blockDim.x) {
        st_async(cl_addr(&s.mu[d], 0), s.mu[d], bar);
        st_async(cl_addr(&s.sig[d], 0), s.sig[d], bar);
      }
      if (tid < 5) st_async(cl_addr(&s_diag[tid], 0), s_diag[tid], bar);
      if (tid == 32) {
        st_async(cl_addr(&s.cur_idx, 0), (uint32_t)s.cur_idx, bar);
        st_async(cl_addr(&s.iter, 0), s.iter, bar);
        st_async(cl_addr(&s_pre[0], 0), robot_in(p, r)->phase_q32, bar);
        st_async(cl_addr(&s_pre[1], 0), s.iter, bar);
      }
    }
    mbar_wait0(&s_bar[0]);  // this CTA's elites
  } else {
    griddep_wait();  // the rollout's J
    griddep_launch_dependents();
    if (blockIdx.y == 0) SBS_TS(16);
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // (long complete: the others' barriers exist)
    select_block_small(p.J + (size_t)r * p.K_local, (int)p.K_local, Ke, p.k_begin, nullptr, nullptr, cem_smem, true,
                       false);
    if (blockIdx.y == 0) SBS_TS(24);
    const int64_t* el = reinterpret_cast<const int64_t*>(cem_smem);  // select_block_small's staging
    const float* eJ = reinterpret_cast<const float*>(el + Ke);
    const int lc = __ffs((int)C) - 1;  // C = 2^lc
    for (int e = tid; e < Ke; e += blockDim.x) {  // every CTA its groups' elites
      const int g = e >> 5, dst = g & ((int)C - 1), i = ((g >> lc) << 5) + (e & 31);
      if (dst != 0) {
        const uint32_t bar = cl_addr(&s_bar[0], (uint32_t)dst);
        st_async(cl_addr(&s_ek[i], (uint32_t)dst), el[e], bar);
        st_async(cl_addr(&s_eJ[i], (uint32_t)dst), eJ[e], bar);
      } else {
        s_ek[i] = el[e];
        s_eJ[i] = eJ[e];
      }
    }
    for (int e = tid; e < Ke; e += blockDim.x) {  // the list in global memory too (sbs_debug_elites)
      p.elite[(size_t)r * Ke + e] = el[e];
      p.elite_J[(size_t)r * Ke + e] = eJ[e];
    }
    mbar_wait0(&s_bar[1]);  // CTA 1's header: the distribution for this CTA's own groups
    __syncthreads();        // (and its own elites)
  }
  if (rank == 1 && blockIdx.y == 0) SBS_TS(22);
  {
    const uint32_t robot_g = (uint32_t)(p.robot_offset + r);
    const uint32_t bar = cl_addr(&s_bar[0], 0);
    for (int t = warp; t < mine * NQ; t += kSelBlock / 32) {
      const int slot = t / NQ, q = t - slot * NQ;
      const int g = (int)rank + (int)C * slot, i = slot * kEliteGroup + lane;
      const bool has_e = g * kEliteGroup + lane < Ke;
      const int64_t k = has_e ? s_ek[i] : 0;
      const float Je = has_e ? s_eJ[i] : kInf;
      SBS_CHECK(k >= 0 && k < p.K_global);
      const GroupMoments m = elite_group_moments(p, s, robot_g, has_e, k, Je, q);
      float* rec = recs + g * RS;  // [S1[D] | S2[D] | n]
      float* dst = rec + (m.j < 4 ? 4 * q + m.j : D + 4 * q + m.j - 4);
      if (rank == 0) {
        if ((lane & 3) == 0) *dst = m.t;
        if (q == 0 && lane == 0) rec[2 * D] = m.n;
      } else {
        if ((lane & 3) == 0) st_async(cl_addr(dst, 0), m.t, bar);
        if (q == 0 && lane == 0) st_async(cl_addr(rec + 2 * D, 0), m.n, bar);
      }
    }
  }
#if defined(SBS_TIMING)
  __syncthreads();
  if (rank == 0 && blockIdx.y == 0) SBS_TS(26);
  if (rank == 1 && blockIdx.y == 0) SBS_TS(30);
#endif
  if (rank != 0) return;
  mbar_wait0(&s_bar[0]);  // the other CTAs' records
  __syncthreads();        // (and this CTA's own)
  if (blockIdx.y == 0) SBS_TS(29);
  if (tid < 2 * D + 1) {  // row tid of [S1 | n | S2] (the elite kernel's record order)
    const int j = tid < D ? tid : (tid == D ? 2 * D : tid - 1);
    float a0 = 0.f;  // records summed in group order (the elite kernel's order)
#pragma unroll 8
    for (int g = 0; g < G; ++g) a0 += recs[g * RS + j];
    s_tot[tid] = a0;
  }
  __syncthreads();
  if (blockIdx.y == 0) SBS_TS(25);
  cem_finish<P>(p, r, s, s_tot, s_diag, s_pre, s_mean, s_var);
  if (blockIdx.y == 0) SBS_TS(28);
}

// ---------------------------------------------------------------------------
// sbs_cov_kernel (f3, L42: CEM with a full covariance C = L L^T): grid (n_eblk, R),
// block 32 x 3P.  Warp q regenerates noise block q of the CTA's 32 elites, the CTA
// forms their deviations d = L z (= theta - mu') and reduces S1 = sum d and the
// lower triangle of S2 = sum d d^T (elites in order).  The last CTA of a robot
// merges the records in order, forms C = S2/n - m m^T + diag(floor) with
// m = S1/n, factors it (right-looking Cholesky in shared memory) and finishes:
// mean = mu' + m, var = diag(C), L = chol(C).
// dynamic smem: max(Lt [D][D] + Z [32][D+1] + Dv [32][D+1],  tot [fc] + C [D][D])
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int cov_smem_floats(int D) {
  return (D * D + 64 * (D + 1)) > (fc_record_floats(D) + D * D) ? (D * D + 64 * (D + 1))
                                                                  : (fc_record_floats(D) + D * D);
}

template <int P>
__global__ void __launch_bounds__(32 * 3 * P) sbs_cov_kernel(const __grid_constant__ Params p) {
  constexpr int D = 12 * P, NT = 32 * 3 * P, NL = D * (D + 1) / 2, FS = fc_record_floats(D);
  __shared__ RobotSmem s;
  __shared__ float s_mean[D], s_var[D];
  __shared__ float s_diag[2];
  __shared__ int s_fail;
  extern __shared__ float dsm[];
  float* Lt = dsm;                   // [D][D]
  float* Z = dsm + D * D;            // [32][D + 1]
  float* Dv = Z + 32 * (D + 1);      // [32][D + 1]
  const int r = blockIdx.y, tid = threadIdx.x, lane = tid & 31, q = tid >> 5;
  load_robot(p, r, s, false);
  stage_chol_t(p, r, Lt);
  griddep_wait();  // the select kernel's elite list
  __syncthreads();
  const uint32_t robot_g = (uint32_t)(p.robot_offset + r);
  const int64_t e = (int64_t)blockIdx.x * kEliteGroup + lane;
  bool ok = false;
  int64_t k = 0;
  if (e < p.n_elite) {
    k = p.elite[(size_t)r * p.n_elite + e];
    ok = p.elite_J[(size_t)r * p.n_elite + e] < kInf;  // diverged samples never enter the moments (L17)
  }
  {
    float z4[4] = {0.f, 0.f, 0.f, 0.f};
    if (ok) noise_block(p, robot_g, k, q, s, z4);
#pragma unroll
    for (int u = 0; u < 4; ++u) Z[lane * (D + 1) + 4 * q + u] = z4[u];
  }
  const unsigned okb = __ballot_sync(0xffffffffu, ok);
  __syncthreads();
  for (int o = tid; o < 32 * D; o += NT) {  // d = L z, row i in ascending j
    const int ee = o / D, i = o - ee * D;
    const float* zr = Z + ee * (D + 1);
    float a = 0.0f;
    for (int j = 0; j <= i; ++j) a = fmaf(Lt[j * D + i], zr[j], a);
    Dv[ee * (D + 1) + i] = a;
  }
  __syncthreads();
  float* rec = p.epart + ((size_t)r * gridDim.x + blockIdx.x) * FS;
  for (int o = tid; o < D + NL; o += NT) {
    float a = 0.0f;
    if (o < D) {
      for (int ee = 0; ee < 32; ++ee) a += Dv[ee * (D + 1) + o];
      rec[o] = a;
    } else {
      const int t = o - D;
      int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
      while ((i + 1) * (i + 2) / 2 <= t) ++i;
      while (i * (i + 1) / 2 > t) --i;
      const int j = t - i * (i + 1) / 2;
      for (int ee = 0; ee < 32; ++ee) a = fmaf(Dv[ee * (D + 1) + i], Dv[ee * (D + 1) + j], a);
      rec[D + 1 + t] = a;
    }
  }
  if (tid == 0) rec[D] = (float)__popc(okb);
  if (!arrive_last(p.ecounter + r, gridDim.x)) return;
  // ---- last CTA: merge the records in order ----
  float* tot = dsm;            // [FS]
  float* Cm = dsm + FS;        // [D][D] lower
  for (int o = tid; o < D + 1 + NL; o += NT) {
    float a = 0.0f;
    int b = 0;
    for (; b + 4 <= (int)gridDim.x; b += 4) {
      const float* r0 = p.epart + ((size_t)r * gridDim.x + b) * FS + o;
      const float v0 = __ldcg(r0), v1 = __ldcg(r0 + FS), v2 = __ldcg(r0 + 2 * FS), v3 = __ldcg(r0 + 3 * FS);
      a += v0;
      a += v1;
      a += v2;
      a += v3;
    }
    for (; b < (int)gridDim.x; ++b) a += __ldcg(p.epart + ((size_t)r * gridDim.x + b) * FS + o);
    tot[o] = a;
  }
  const float* sd = p.sdiag + (size_t)r * 8;
  const Best best{sd[0], __float_as_int(sd[1]), __float_as_int(sd[2])};
  if (tid == 0) {
    s_diag[0] = sd[3];
    s_diag[1] = sd[4];
    s_fail = 0;
  }
  __syncthreads();
  const float ne = tot[D];
  const bool all_div = !(ne > 0.f);
  const float inv = all_div ? 0.f : 1.0f / ne;
  if (!all_div) {
    for (int t = tid; t < NL; t += NT) {
      int i = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
      while ((i + 1) * (i + 2) / 2 <= t) ++i;
      while (i * (i + 1) / 2 > t) --i;
      const int j = t - i * (i + 1) / 2;
      const float mi = tot[i] * inv, mj = tot[j] * inv;
      float c = fmaf(-mi, mj, tot[D + 1 + t] * inv);
      if (i == j) c += p.var_floor[i % 3];
      Cm[i * D + j] = c;
    }
    __syncthreads();
    for (int d = tid; d < D; d += NT) {
      s_mean[d] = s.mu[d] + tot[d] * inv;
      s_var[d] = Cm[d * D + d];
    }
    // right-looking Cholesky of the lower triangle, in place
    for (int kk = 0; kk < D; ++kk) {
      if (tid == 0) {
        const float c = Cm[kk * D + kk];
        if (!(c > 0.0f)) s_fail = 1;
        Cm[kk * D + kk] = sqrtf(fmaxf(c, 1e-30f));
      }
      __syncthreads();
      const float lkk = Cm[kk * D + kk];
      for (int i = kk + 1 + tid; i < D; i += NT) Cm[i * D + kk] = Cm[i * D + kk] / lkk;
      __syncthreads();
      const int m = D - 1 - kk;  // trailing block (kk, D) x (kk, D), lower triangle: m (m + 1) / 2 entries
      for (int t = tid; t < m * (m + 1) / 2; t += NT) {
        int a = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
        while ((a + 1) * (a + 2) / 2 <= t) ++a;
        while (a * (a + 1) / 2 > t) --a;
        const int b2 = t - a * (a + 1) / 2;
        const int i = kk + 1 + a, j = kk + 1 + b2;
        Cm[i * D + j] = fmaf(-Cm[i * D + kk], Cm[j * D + kk], Cm[i * D + j]);
      }
      __syncthreads();
    }
  }
  const bool keep = all_div || s_fail;  // L27 (or a failed factorisation): keep the distribution
  for (int d = tid; d < D; d += NT) {
    if (keep) {
      s_mean[d] = p.mean[(size_t)r * D + d];
      s_var[d] = p.var[(size_t)r * D + d];
    }
  }
  __syncthreads();
  const int fi = all_div ? s.cur_idx : best.f;
  for (int d = tid; d < D; d += NT) {
    p.mean[(size_t)r * D + d] = s_mean[d];
    p.var[(size_t)r * D + d] = s_var[d];
  }
  if (!keep)
    for (int idx = tid; idx < D * D; idx += NT) {
      const int i = idx / D, j = idx - i * D;
      p.Lmat[(size_t)r * D * D + idx] = j <= i ? Cm[idx] : 0.0f;
    }
  if (tid == 0) {
    p.fidx[r] = fi;
    p.best[r] = best.k;
  }
  write_output(p, r, all_div ? SBS_WARN_ALL_DIVERGED : SBS_OK, s_mean, s_var, fi, best.m,
               s_diag[1] > 0.f ? s_diag[0] / s_diag[1] : kInf, ne, ne, (int)((float)p.K_global - s_diag[1]));
}

// Naive with world > 1, after the all-gather (p.part = [world][R] rank records)
template <int P>
__global__ void __launch_bounds__(128) sbs_naive_finalize_kernel(const __grid_constant__ Params p) {
  __shared__ RobotSmem s;
  load_robot(p, blockIdx.x, s, false);
  __syncthreads();
  naive_finalize_block<P>(p, blockIdx.x, s);
}

// ---------------------------------------------------------------------------
// debug: z, theta, theta1 of samples k0..k0+n-1 of one robot (same draw code)
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(128) sbs_debug_samples_kernel(const __grid_constant__ Params p, int r, int64_t k0,
                                                                int64_t n, float* z, float* theta, int* fidx) {
  constexpr int D = 12 * P;
  __shared__ RobotSmem s;
  extern __shared__ float Lt[];  // full covariance: L^T [D][D]
  load_robot(p, r, s, false);
  if (p.full_cov) stage_chol_t(p, r, Lt);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Theta<P> th;
  float zz[D];
  const int f = p.full_cov ? draw_sample_fc<P, true>(p, (uint32_t)(p.robot_offset + r), k0 + i, s, Lt, th, zz)
                           : draw_sample<P, true>(p, (uint32_t)(p.robot_offset + r), k0 + i, s, th, zz);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    z[i * D + d] = zz[d];
    theta[i * D + d] = theta_get(th, d);
  }
  fidx[i] = f;
}

// ---------------------------------------------------------------------------
// launchers.  The build compiles this file once per knot count P (-DSBS_TU_P=P:
// the rollout / elite / debug kernels for that P) and once with -DSBS_TU_COMMON
// (dispatch, select and merge kernels), in parallel.
// ---------------------------------------------------------------------------
// launch with programmatic stream serialisation (PDL): the kernel may start while the
// previous kernel on the stream drains; it waits in griddep_wait() for its inputs
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, int kind, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
#if defined(SBS_TIMING)  // experiments: SBS_NO_PDL=<mask> launches without the attribute (1 rollout, 2 select, 4 elite)
  {
    static const int mask = getenv("SBS_NO_PDL") ? atoi(getenv("SBS_NO_PDL")) : 0;
    if (mask & kind) attr[0].val.programmaticStreamSerializationAllowed = 0;
  }
#else
  (void)kind;
#endif
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int P>
struct PEntry {
  static cudaError_t rollout(const Params& p, int mode, bool fused, cudaStream_t s);
  static int occupancy(int mode, bool fc, bool split, bool model);
  static cudaError_t elite(const Params& p, cudaStream_t s);
  static cudaError_t cem_cluster(const Params& p, cudaStream_t s);
  static int cem_cluster_size(int want);
  static cudaError_t naive_finalize(const Params& p, cudaStream_t s);
  static cudaError_t debug_samples(const Params& p, int robot, int64_t k0, int64_t n, float* z, float* theta,
                                   int* fidx, cudaStream_t s);
  static cudaError_t prepare();  // function attributes, set once outside any stream capture
};

#if defined(SBS_TU_P)
template <int P, int EPI, bool FC, bool SPLIT>
constexpr size_t rollout_smem() {
  constexpr int D = 12 * P;
  return (EPI == EPI_MPPI ? (size_t)(D + 4) * kRedStride * sizeof(float) : (FC ? (size_t)D * D * sizeof(float) : 0)) +
         (SPLIT ? (size_t)kBlock * (D + 2) * sizeof(float) : 0);
}

// the compiled-in robot model (sbs_robot_model.h) is instantiated for its knot count only
template <int P>
constexpr bool kHasModel = (P == model::kKnots);

template <int P, int EPI, bool FUSED, bool FC, bool SPLIT, bool MODEL>
static cudaError_t launch_rollout_m(const Params& p, cudaStream_t s) {
  dim3 grid(p.n_cta, p.R);
  if constexpr (SPLIT) {  // (separate instantiation: its registers are not sized for the one-thread rollout)
    if (p.ab)
      return launch_pdl(sbs_rollout_kernel<P, EPI, FUSED, FC, SPLIT, true, MODEL>, grid, dim3(kBlock * kSplitLanes),
                        split_smem_bytes(P, EPI == EPI_MPPI, p.H, true), 1, s, p);
  }
  const size_t smem = SPLIT ? split_smem_bytes(P, EPI == EPI_MPPI, p.H, false) : rollout_smem<P, EPI, FC, SPLIT>();
  if constexpr (EPI == EPI_MPPI && FUSED && !SPLIT && !FC) {
    if (p.dyn)
      return launch_pdl(sbs_rollout_kernel<P, EPI, FUSED, FC, SPLIT, false, MODEL, true>, grid, dim3(kBlock), smem, 1,
                        s, p);
  }
  return launch_pdl(sbs_rollout_kernel<P, EPI, FUSED, FC, SPLIT, false, MODEL>, grid,
                    dim3(SPLIT ? kBlock * kSplitLanes : kBlock), smem, 1, s, p);
}

template <int P, int EPI, bool FUSED, bool FC = false, bool SPLIT = false>
static cudaError_t launch_rollout_t(const Params& p, cudaStream_t s) {
  if constexpr (kHasModel<P> && !FC) {
    if (p.model) return launch_rollout_m<P, EPI, FUSED, FC, SPLIT, true>(p, s);
  }
  return launch_rollout_m<P, EPI, FUSED, FC, SPLIT, false>(p, s);
}

template <int P>
cudaError_t PEntry<P>::rollout(const Params& p, int mode, bool fused, cudaStream_t s) {
  if (p.split) {  // latency mode (few samples)
    if (mode == SBS_MPPI)
      return fused ? launch_rollout_t<P, EPI_MPPI, true, false, true>(p, s)
                   : launch_rollout_t<P, EPI_MPPI, false, false, true>(p, s);
    if (mode == SBS_NAIVE && fused) return launch_rollout_t<P, EPI_ARGMIN, true, false, true>(p, s);
    return launch_rollout_t<P, EPI_ARGMIN, false, false, true>(p, s);
  }
  if (mode == SBS_MPPI) return fused ? launch_rollout_t<P, EPI_MPPI, true>(p, s) : launch_rollout_t<P, EPI_MPPI, false>(p, s);
  if (mode == SBS_NAIVE && fused) return launch_rollout_t<P, EPI_ARGMIN, true>(p, s);
  if (p.full_cov) return launch_rollout_t<P, EPI_ARGMIN, false, true>(p, s);  // CEM, full covariance (f3)
  return launch_rollout_t<P, EPI_ARGMIN, false>(p, s);  // CEM, or sharded Naive: records only
}

template <int P>
int PEntry<P>::occupancy(int mode, bool fc, bool split, bool model) {
  size_t smem;
  const void* f;
  constexpr bool M = kHasModel<P>;
  model = model && M && !fc;
  if (mode == SBS_MPPI) {
    smem = split ? rollout_smem<P, EPI_MPPI, false, true>() : rollout_smem<P, EPI_MPPI, false, false>();
    f = split ? (const void*)sbs_rollout_kernel<P, EPI_MPPI, true, false, true>
              : (model ? (const void*)sbs_rollout_kernel<P, EPI_MPPI, true, false, false, false, M>
                       : (const void*)sbs_rollout_kernel<P, EPI_MPPI, true>);
  } else if (fc) {
    smem = rollout_smem<P, EPI_ARGMIN, true, false>();
    f = (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, false, true>;
  } else {
    smem = split ? rollout_smem<P, EPI_ARGMIN, false, true>() : rollout_smem<P, EPI_ARGMIN, false, false>();
    f = split ? (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, false, false, true>
              : (model ? (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, false, false, false, false, M>
                       : (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, false>);
  }
  int n = 0;  // (dynamic shared memory limits: prepare(), which sbs_create runs first)
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, split && !fc ? kBlock * kSplitLanes : kBlock, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

template <int P>
cudaError_t PEntry<P>::elite(const Params& p, cudaStream_t s) {
  dim3 grid(p.n_eblk, p.R);
  if (p.full_cov)
    return launch_pdl(sbs_cov_kernel<P>, grid, dim3(32 * 3 * P), (size_t)cov_smem_floats(12 * P) * sizeof(float), 4, s, p);
  return launch_pdl(sbs_elite_kernel<P>, grid, dim3(32 * 3 * P), 0, 4, s, p);
}

template <int P>
cudaError_t PEntry<P>::cem_cluster(const Params& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.cem_cluster, p.R);
  cfg.blockDim = dim3(kSelBlock);
  cfg.dynamicSmemBytes = kCemSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = p.cem_cluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, sbs_cem_cluster_kernel<P>, p);
}

// the largest cluster (of 16, 8; `want` caps it) that can be resident with the kernel's
// block size and shared memory, 0 if none
template <int P>
int PEntry<P>::cem_cluster_size(int want) {
  for (int c = 16; c >= 8; c /= 2) {
    if (c > want) continue;
    if (c > 8 && cudaFuncSetAttribute(sbs_cem_cluster_kernel<P>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                     cudaSuccess) {
      (void)cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c, 1);
    cfg.blockDim = dim3(kSelBlock);
    cfg.dynamicSmemBytes = kCemSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, sbs_cem_cluster_kernel<P>, &cfg) == cudaSuccess && n > 0) return c;
    (void)cudaGetLastError();
  }
  return 0;
}

template <int P>
cudaError_t PEntry<P>::naive_finalize(const Params& p, cudaStream_t s) {
  sbs_naive_finalize_kernel<P><<<p.R, 128, 0, s>>>(p);
  return cudaGetLastError();
}

template <int P>
cudaError_t PEntry<P>::debug_samples(const Params& p, int robot, int64_t k0, int64_t n, float* z, float* theta,
                                     int* fidx, cudaStream_t s) {
  const int blocks = (int)((n + 127) / 128);
  const size_t smem = p.full_cov ? (size_t)144 * P * P * sizeof(float) : 0;  // L^T [D][D]
  sbs_debug_samples_kernel<P><<<blocks, 128, smem, s>>>(p, robot, k0, n, z, theta, fidx);
  return cudaGetLastError();
}

template <int P>
cudaError_t PEntry<P>::prepare() {
  const int big = 96 * 1024, huge = (int)kSplitSmemMax;
  cudaError_t e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             big);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sbs_cov_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_cem_cluster_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCemSmemBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, true, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, false, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, true, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, false, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, true, false, true, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, false, false, true, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, true, false, true, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, false, false, true, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_debug_samples_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  if constexpr (kHasModel<P>) {  // the compiled-in robot model's instantiations
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, true, false, false, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_MPPI, false, false, false, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, true, false, false, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(sbs_rollout_kernel<P, EPI_ARGMIN, false, false, false, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    for (int ab = 0; ab < 2 && e == cudaSuccess; ++ab) {
      e = cudaFuncSetAttribute(ab ? (const void*)sbs_rollout_kernel<P, EPI_MPPI, true, false, true, true, true>
                                  : (const void*)sbs_rollout_kernel<P, EPI_MPPI, true, false, true, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ab ? (const void*)sbs_rollout_kernel<P, EPI_MPPI, false, false, true, true, true>
                                    : (const void*)sbs_rollout_kernel<P, EPI_MPPI, false, false, true, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ab ? (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, true, false, true, true, true>
                                    : (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, true, false, true, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ab ? (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, false, false, true, true, true>
                                    : (const void*)sbs_rollout_kernel<P, EPI_ARGMIN, false, false, true, false, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, huge);
    }
  }
  // load every remaining kernel of this P now: with CUDA's lazy module loading the first
  // launch of a kernel can wait for the device, which must never happen behind a stream
  // that waits on a peer's flag (peer-memory exchange)
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, sbs_elite_kernel<P>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, sbs_naive_finalize_kernel<P>);
  return e;
}

template struct PEntry<SBS_TU_P>;

#if defined(SBS_TIMING)  // experiments only
#define SBS_CAT2(a, b) a##b
#define SBS_CAT(a, b) SBS_CAT2(a, b)
extern "C" int SBS_CAT(sbs_debug_ts_p, SBS_TU_P)(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_sbs_ts, sizeof(g_sbs_ts));
}
extern "C" int SBS_CAT(sbs_debug_bar_p, SBS_TU_P)(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_sbs_bar, sizeof(g_sbs_bar));
}
extern "C" int SBS_CAT(sbs_debug_cta_p, SBS_TU_P)(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_sbs_cta, sizeof(g_sbs_cta));
}
#endif
#endif  // SBS_TU_P

#if defined(SBS_TU_COMMON)
#if defined(SBS_ONLY_P)  // experiment builds with one knot count (build.py only_p=...)
#define SBS_DISPATCH_P(P_, CALL) \
  if ((P_) == SBS_ONLY_P) return PEntry<SBS_ONLY_P>::CALL;
#else
#define SBS_DISPATCH_P(P_, CALL)                 \
  switch (P_) {                                  \
    case 2: return PEntry<2>::CALL;              \
    case 3: return PEntry<3>::CALL;              \
    case 4: return PEntry<4>::CALL;              \
    case 5: return PEntry<5>::CALL;              \
    case 6: return PEntry<6>::CALL;              \
    case 7: return PEntry<7>::CALL;              \
    case 8: return PEntry<8>::CALL;              \
    default: break;                              \
  }
#endif

cudaError_t launch_rollout(const Params& p, int mode, bool fused, cudaStream_t s) {
  SBS_DISPATCH_P(p.P, rollout(p, mode, fused, s));
  return cudaErrorInvalidValue;
}

int rollout_occupancy(int P, int mode, bool fc, bool split, bool model) {
  SBS_DISPATCH_P(P, occupancy(mode, fc, split, model));
  return 1;
}

cudaError_t launch_elite(const Params& p, cudaStream_t s) {
  SBS_DISPATCH_P(p.P, elite(p, s));
  return cudaErrorInvalidValue;
}

cudaError_t launch_cem_cluster(const Params& p, cudaStream_t s) {
  SBS_DISPATCH_P(p.P, cem_cluster(p, s));
  return cudaErrorInvalidValue;
}

int cem_cluster_size(int P, int want) {
  SBS_DISPATCH_P(P, cem_cluster_size(want));
  return 0;
}

bool cem_cluster_fits(const Params& p) {
  return p.mode == SBS_CEM && !p.full_cov && p.K_local <= kSelSmallMax && p.n_eblk <= kCemMaxGroups &&
         (int64_t)p.n_elite * (sizeof(int64_t) + sizeof(float)) <= (int64_t)kSelSmallSmemBytes;
}

cudaError_t launch_naive_finalize(const Params& p, cudaStream_t s) {
  SBS_DISPATCH_P(p.P, naive_finalize(p, s));
  return cudaErrorInvalidValue;
}

cudaError_t launch_debug_samples(const Params& p, int robot, int64_t k0, int64_t n, float* z, float* theta,
                                 int* fidx, cudaStream_t s) {
  SBS_DISPATCH_P(p.P, debug_samples(p, robot, k0, n, z, theta, fidx, s));
  return cudaErrorInvalidValue;
}

cudaError_t launch_mppi_finalize(const Params& p, cudaStream_t s) {
  sbs_mppi_finalize<false><<<p.R, 128, 0, s>>>(p, nullptr);
  return cudaGetLastError();
}


static size_t select_smem(int64_t K) {
  if (K <= kSelSmallMax) return (size_t)kSelSmallSmemBytes;
  return (size_t)(kSelHistWords + (K <= kSelSmemKeys ? K : 0)) * 4;
}

template <int MODE, bool SMALL>
static cudaError_t set_select_attr() {
  return cudaFuncSetAttribute(sbs_select_kernel<MODE, SMALL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              SMALL ? kSelSmallSmemBytes : kSelSmemBytes);
}

cudaError_t prepare_kernels(int P) {
  cudaError_t e = cudaFuncSetAttribute(sbs_select_raw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSelSmemBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(sbs_select_small_raw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSelSmallSmemBytes);
  if (e == cudaSuccess) e = set_select_attr<SEL_LOCAL, true>();
  if (e == cudaSuccess) e = set_select_attr<SEL_LOCAL, false>();
  if (e == cudaSuccess) e = set_select_attr<SEL_EMIT, true>();
  if (e == cudaSuccess) e = set_select_attr<SEL_EMIT, false>();
  if (e == cudaSuccess) e = set_select_attr<SEL_MERGE, true>();
  if (e == cudaSuccess) e = set_select_attr<SEL_MERGE, false>();
  cudaFuncAttributes fa;  // (lazy loading: see PEntry<P>::prepare)
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, sbs_mppi_finalize<false>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, sbs_mppi_finalize<true>);
  if (e != cudaSuccess || P == 0) return e;
  SBS_DISPATCH_P(P, prepare());
  return cudaErrorInvalidValue;
}

template <int MODE>
static cudaError_t launch_select_t(const Params& p, int64_t K, float* emit, cudaStream_t s) {
  const size_t smem = select_smem(K);
  if (K <= kSelSmallMax) return launch_pdl(sbs_select_kernel<MODE, true>, dim3(p.R), dim3(kSelBlock), smem, 2, s, p, emit);
  return launch_pdl(sbs_select_kernel<MODE, false>, dim3(p.R), dim3(kSelBlock), smem, 2, s, p, emit);
}

cudaError_t launch_select(const Params& p, cudaStream_t s) { return launch_select_t<SEL_LOCAL>(p, p.K_local, nullptr, s); }
cudaError_t launch_select_emit(const Params& p, float* emit, cudaStream_t s) {
  Params q = p;
  q.emit = emit;  // (the peer publisher copies from here)
  return launch_select_t<SEL_EMIT>(q, q.K_local, emit, s);
}
cudaError_t launch_select_merge(const Params& p, cudaStream_t s) {
  return launch_select_t<SEL_MERGE>(p, (int64_t)p.n_cta * p.n_elite, nullptr, s);
}

cudaError_t launch_select_raw(const float* J, int64_t K, int64_t K_e, int64_t* idx, cudaStream_t s) {
  const size_t smem = select_smem(K);
  if (K <= kSelSmallMax) sbs_select_small_raw_kernel<<<1, kSelBlock, smem, s>>>(J, K, K_e, idx);
  else sbs_select_raw_kernel<<<1, kSelBlock, smem, s>>>(J, K, K_e, idx);
  return cudaGetLastError();
}
#if defined(SBS_TIMING)  // experiments only
extern "C" int sbs_debug_ts_common(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_sbs_ts, sizeof(g_sbs_ts));
}
#endif
#endif  // SBS_TU_COMMON

}  // namespace sbs
