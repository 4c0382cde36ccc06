// sbs_kernels.cu -- sm_100a kernels of one SBS MPC iteration (arxiv 2403.11383).
//
//   sbs_rollout_kernel   steps a0-a4 (+ a5 partial for MPPI): warm shift, Philox
//                        sampling, contact sequence, GRF spline + cone, SRBD RK4,
//                        cost; one thread per sample, everything in registers;
//                        MPPI: online (min, sum w, sum w theta) partial per CTA.
//   sbs_mppi_finalize    step a5/a7: merge the CTA partials, new mean, output.
//   sbs_select_kernel    step a6: radix select of the K_e smallest (J, k).
//   sbs_elite_kernel     step a6/a7: regenerate the elites' theta from the counter
//                        RNG, elite mean / variance, output.
//
// The rollout is FP32 CUDA-core work (not a contraction): it is bound by the FMA
// pipe, not by HBM (4 bytes written per sample).  See DESIGN.md sec. 7.
#include <float.h>
#include <math.h>

#include "sbs_internal.h"
#include "sbs_noise.cuh"

namespace sbs {

#define kInf __int_as_float(0x7f800000)
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
  float feet_cur[12];
  float feet_next[12];
  float xref[SBS_MAX_HORIZON * 12];
  uint32_t phase0;
  int cur_idx;
};

// step a0: mu'[p] = S_mu(min(t_p + dt, T)); std = sqrt(var)
__device__ void load_robot(const Params& p, int r, RobotSmem& s) {
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
  const sbs_input* in = p.in + r;
  for (int a = threadIdx.x; a < 12; a += blockDim.x) {
    s.x0[a] = in->x0[a];
    s.feet_cur[a] = in->feet_cur[a];
    s.feet_next[a] = in->feet_next[a];
  }
  const float* xr = p.xref + (size_t)r * p.H * 12;
  for (int a = threadIdx.x; a < p.H * 12; a += blockDim.x) s.xref[a] = xr[a];
  if (threadIdx.x == 0) {
    s.phase0 = in->phase_q32;
    s.cur_idx = p.fidx[r];
  }
}

// step a1: theta2 = mu' + sigma z, theta1 index
template <int P, bool WITH_Z>
__device__ __forceinline__ int draw_sample(const Params& p, uint32_t robot_g, int64_t k, const RobotSmem& s,
                                           float (&th)[12 * P], float* z_out = nullptr) {
  constexpr int D = 12 * P;
  if (p.elite_preserve && k == 0) {  // L21
#pragma unroll
    for (int d = 0; d < D; ++d) th[d] = s.mu[d];
    if (WITH_Z)
      for (int d = 0; d < D; ++d) z_out[d] = 0.0f;
    return s.cur_idx;
  }
  const uint32_t kk = (uint32_t)k;
#pragma unroll
  for (int q = 0; q < D / 4; ++q) {
    const U4 w = philox4x32_10((uint32_t)q, kk, p.iter, robot_g, p.seed_lo, p.seed_hi);
    float z[4];
    box_muller(w.x, w.y, z[0], z[1]);
    box_muller(w.z, w.w, z[2], z[3]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      th[4 * q + i] = __fmaf_rn(s.sig[4 * q + i], z[i], s.mu[4 * q + i]);
      if (WITH_Z) z_out[4 * q + i] = z[i];
    }
  }
  int idx = s.cur_idx;
  if (p.gait_adapt) {
    const U4 w = philox4x32_10(0x80000000u, kk, p.iter, robot_g, p.seed_lo, p.seed_hi);
    idx = (int)__umulhi(w.x, (uint32_t)p.n_freq);  // (w * n) >> 32
  }
  return idx;
}

// Eq. 1 angular part at one RK4 stage (L24): given world torque tau_w,
//   w' = I^-1 (R^T tau_w - w x I w),  Phi' = E'^-1(Phi) w.
__device__ __forceinline__ void ang_deriv(const Params& p, float phi, float th, float psi, float wx, float wy,
                                          float wz, float tx, float ty, float tz, float& dphi, float& dth,
                                          float& dpsi, float& dwx, float& dwy, float& dwz) {
  float sr, cr, sp, cp, sy, cy;
  __sincosf(phi, &sr, &cr);
  __sincosf(th, &sp, &cp);
  __sincosf(psi, &sy, &cy);
  // R^T tau = Rx^T Ry^T Rz^T tau  (R = Rz(yaw) Ry(pitch) Rx(roll))
  const float t1x = fmaf(cy, tx, sy * ty), t1y = fmaf(cy, ty, -sy * tx);
  const float bx = fmaf(cp, t1x, -sp * tz), t2z = fmaf(sp, t1x, cp * tz);
  const float by = fmaf(cr, t1y, sr * t2z), bz = fmaf(cr, t2z, -sr * t1y);
  float Lx, Ly, Lz;
  if (p.diag_inertia) {
    Lx = p.I[0] * wx;
    Ly = p.I[4] * wy;
    Lz = p.I[8] * wz;
  } else {
    Lx = fmaf(p.I[0], wx, fmaf(p.I[1], wy, p.I[2] * wz));
    Ly = fmaf(p.I[3], wx, fmaf(p.I[4], wy, p.I[5] * wz));
    Lz = fmaf(p.I[6], wx, fmaf(p.I[7], wy, p.I[8] * wz));
  }
  const float rx = bx - fmaf(wy, Lz, -wz * Ly);
  const float ry = by - fmaf(wz, Lx, -wx * Lz);
  const float rz = bz - fmaf(wx, Ly, -wy * Lx);
  if (p.diag_inertia) {
    dwx = p.Iinv[0] * rx;
    dwy = p.Iinv[4] * ry;
    dwz = p.Iinv[8] * rz;
  } else {
    dwx = fmaf(p.Iinv[0], rx, fmaf(p.Iinv[1], ry, p.Iinv[2] * rz));
    dwy = fmaf(p.Iinv[3], rx, fmaf(p.Iinv[4], ry, p.Iinv[5] * rz));
    dwz = fmaf(p.Iinv[6], rx, fmaf(p.Iinv[7], ry, p.Iinv[8] * rz));
  }
  const float rc = __fdividef(1.0f, cp);
  const float a = fmaf(sr, wy, cr * wz);
  dphi = fmaf(sp * rc, a, wx);
  dth = fmaf(cr, wy, -sr * wz);
  dpsi = a * rc;
}

// steps a2-a4: Rollout(theta_k, x0), Alg. 2 with policy pi
template <int P>
__device__ float rollout(const Params& p, const float (&th)[12 * P], int fi, const RobotSmem& s) {
  float px = s.x0[0], py = s.x0[1], pz = s.x0[2];
  float vx = s.x0[3], vy = s.x0[4], vz = s.x0[5];
  float an0 = s.x0[6], an1 = s.x0[7], an2 = s.x0[8];
  float wx = s.x0[9], wy = s.x0[10], wz = s.x0[11];
  const float dt = p.dt, hdt = 0.5f * p.dt, dt6 = p.dt * (1.0f / 6.0f);
  const float dt2h = 0.5f * p.dt * p.dt, dt2q = 0.25f * p.dt * p.dt;
  const uint32_t inc = p.inc[fi];
  uint32_t ph[4];
  bool prev[4], td[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ph[i] = s.phase0 + p.off[i];
    prev[i] = false;
    td[i] = false;
  }
  float J = 0.0f;
  bool bad = false;
  for (int j = 0; j < p.H; ++j) {
    // --- contact sequence delta_j (O7, L22) and touchdown (L23) ---
    bool st[4];
    int nst = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      st[i] = p.all_stance || (ph[i] < p.thr);
      td[i] = td[i] || (j > 0 && st[i] && !prev[i]);
      prev[i] = st[i];
      nst += st[i] ? 1 : 0;
      ph[i] += inc;
    }
    // --- Gamma_j = sigma(theta2, t_j), mask, cone, penalty (O8-O9) ---
    float G[12];
    float pen = 0.0f;
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      float v = 0.0f;
#pragma unroll
      for (int q = 0; q < P; ++q) v = fmaf(p.W[j][q], th[q * 12 + c], v);
      G[c] = v;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float fx = G[3 * i], fy = G[3 * i + 1], fz = G[3 * i + 2];
      const float fzc = fminf(fmaxf(fz, p.fz_min), p.fz_max);
      const float l = p.mu * fzc;
      const float vzv = fmaxf(p.fz_min - fz, 0.0f) + fmaxf(fz - p.fz_max, 0.0f);
      const float vxv = fmaxf(fabsf(fx) - l, 0.0f), vyv = fmaxf(fabsf(fy) - l, 0.0f);
      const float pl = fmaf(vzv, vzv, fmaf(vxv, vxv, vyv * vyv));
      pen += st[i] ? pl : 0.0f;
      G[3 * i] = st[i] ? fminf(fmaxf(fx, -l), l) : 0.0f;
      G[3 * i + 1] = st[i] ? fminf(fmaxf(fy, -l), l) : 0.0f;
      G[3 * i + 2] = st[i] ? fzc : 0.0f;
    }
    // --- stage cost r(u_j, x_j, x^r_j) ---
    const float* xr = &s.xref[12 * j];
    float e8 = an2 - xr[8];
    e8 = fmaf(-kTwoPi, rintf(e8 * kInvTwoPi), e8);  // yaw wrapped to [-pi, pi]
    const float e[12] = {px - xr[0], py - xr[1], pz - xr[2], vx - xr[3], vy - xr[4], vz - xr[5],
                         an0 - xr[6], an1 - xr[7], e8,        wx - xr[9], wy - xr[10], wz - xr[11]};
    float stage = 0.0f;
#pragma unroll
    for (int a = 0; a < 12; ++a) stage = fmaf(p.Q[a] * e[a], e[a], stage);
    const float urz = p.urz[nst];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float ez = G[3 * i + 2] - urz;
      float t = fmaf(p.Rw[3 * i] * G[3 * i], G[3 * i], fmaf(p.Rw[3 * i + 1] * G[3 * i + 1], G[3 * i + 1],
                                                              p.Rw[3 * i + 2] * ez * ez));
      stage += st[i] ? t : 0.0f;
    }
    J += fmaf(p.w_fc, pen, stage);
    // --- per-step force and moment about the world origin (Gamma, feet held: L8, L25) ---
    float Fx = 0.f, Fy = 0.f, Fz = 0.f, Mx = 0.f, My = 0.f, Mz = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float fx = td[i] ? s.feet_next[3 * i] : s.feet_cur[3 * i];
      const float fy = td[i] ? s.feet_next[3 * i + 1] : s.feet_cur[3 * i + 1];
      const float fz = td[i] ? s.feet_next[3 * i + 2] : s.feet_cur[3 * i + 2];
      const float gx = G[3 * i], gy = G[3 * i + 1], gz = G[3 * i + 2];
      Fx += gx;
      Fy += gy;
      Fz += gz;
      Mx += fmaf(fy, gz, -fz * gy);
      My += fmaf(fz, gx, -fx * gz);
      Mz += fmaf(fx, gy, -fy * gx);
    }
    // v' = F/m + g is constant over the step: RK4 on (p, v) is exact, so the
    // stage positions are closed-form; the torque is tau = M - p_stage x F.
    const float ax = fmaf(Fx, p.inv_mass, p.g[0]), ay = fmaf(Fy, p.inv_mass, p.g[1]),
                az = fmaf(Fz, p.inv_mass, p.g[2]);
    float k1[6], k2[6], k3[6], k4[6];
    {  // stage 1 at p
      ang_deriv(p, an0, an1, an2, wx, wy, wz, Mx - fmaf(py, Fz, -pz * Fy), My - fmaf(pz, Fx, -px * Fz),
                Mz - fmaf(px, Fy, -py * Fx), k1[0], k1[1], k1[2], k1[3], k1[4], k1[5]);
    }
    {  // stage 2 at p + dt/2 v
      const float qx = fmaf(hdt, vx, px), qy = fmaf(hdt, vy, py), qz = fmaf(hdt, vz, pz);
      ang_deriv(p, fmaf(hdt, k1[0], an0), fmaf(hdt, k1[1], an1), fmaf(hdt, k1[2], an2), fmaf(hdt, k1[3], wx),
                fmaf(hdt, k1[4], wy), fmaf(hdt, k1[5], wz), Mx - fmaf(qy, Fz, -qz * Fy),
                My - fmaf(qz, Fx, -qx * Fz), Mz - fmaf(qx, Fy, -qy * Fx), k2[0], k2[1], k2[2], k2[3], k2[4],
                k2[5]);
    }
    {  // stage 3 at p + dt/2 v + dt^2/4 a
      const float qx = fmaf(dt2q, ax, fmaf(hdt, vx, px)), qy = fmaf(dt2q, ay, fmaf(hdt, vy, py)),
                  qz = fmaf(dt2q, az, fmaf(hdt, vz, pz));
      ang_deriv(p, fmaf(hdt, k2[0], an0), fmaf(hdt, k2[1], an1), fmaf(hdt, k2[2], an2), fmaf(hdt, k2[3], wx),
                fmaf(hdt, k2[4], wy), fmaf(hdt, k2[5], wz), Mx - fmaf(qy, Fz, -qz * Fy),
                My - fmaf(qz, Fx, -qx * Fz), Mz - fmaf(qx, Fy, -qy * Fx), k3[0], k3[1], k3[2], k3[3], k3[4],
                k3[5]);
    }
    // stage 4 at p + dt v + dt^2/2 a  (= p_{j+1})
    const float nx = fmaf(dt2h, ax, fmaf(dt, vx, px)), ny = fmaf(dt2h, ay, fmaf(dt, vy, py)),
                nz = fmaf(dt2h, az, fmaf(dt, vz, pz));
    ang_deriv(p, fmaf(dt, k3[0], an0), fmaf(dt, k3[1], an1), fmaf(dt, k3[2], an2), fmaf(dt, k3[3], wx),
              fmaf(dt, k3[4], wy), fmaf(dt, k3[5], wz), Mx - fmaf(ny, Fz, -nz * Fy), My - fmaf(nz, Fx, -nx * Fz),
              Mz - fmaf(nx, Fy, -ny * Fx), k4[0], k4[1], k4[2], k4[3], k4[4], k4[5]);
    float acc[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) acc[a] = fmaf(2.0f, k2[a] + k3[a], k1[a] + k4[a]);
    an0 = fmaf(dt6, acc[0], an0);
    an1 = fmaf(dt6, acc[1], an1);
    an2 = fmaf(dt6, acc[2], an2);
    wx = fmaf(dt6, acc[3], wx);
    wy = fmaf(dt6, acc[4], wy);
    wz = fmaf(dt6, acc[5], wz);
    px = nx;
    py = ny;
    pz = nz;
    vx = fmaf(dt, ax, vx);
    vy = fmaf(dt, ay, vy);
    vz = fmaf(dt, az, vz);
    // --- divergence of x_{j+1} (L26); NaN fails every <= test ---
    const float big = fmaxf(fmaxf(fmaxf(fabsf(px), fabsf(py)), fmaxf(fabsf(pz), fabsf(vx))),
                            fmaxf(fmaxf(fabsf(vy), fabsf(vz)), fmaxf(fabsf(an0), fabsf(an2))));
    const float big2 = fmaxf(fmaxf(fabsf(wx), fabsf(wy)), fabsf(wz));
    bad = bad || !(big <= 1e6f) || !(big2 <= 1e6f) || !(fabsf(an1) < kPitchMax);
  }
  const float df = p.freq_hz[fi] - p.f_nominal;
  J = fmaf(p.rho * df, df, J);  // P:350, once per rollout (L14)
  return (bad || !(J <= FLT_MAX)) ? kInf : J;
}

// (J, k) lexicographic min helpers for argmin with lowest-index tie-break
__device__ __forceinline__ bool jk_less(float ja, int ka, float jb, int kb) {
  return ja < jb || (ja == jb && ka < kb);
}

// ---------------------------------------------------------------------------
// sbs_rollout_kernel: grid (n_cta, R), block kBlock; CTA c processes tiles
// c, c + n_cta, ... of its robot's K_local samples.
// ---------------------------------------------------------------------------
template <int P, bool MPPI>
__global__ void __launch_bounds__(kBlock) sbs_rollout_kernel(const __grid_constant__ Params p) {
  constexpr int D = 12 * P;
  constexpr int NR = D + 4;  // reduced rows: w theta[D], w, w^2, J (finite), 1 (finite)
  __shared__ RobotSmem s;
  extern __shared__ float s_red[];  // [NR][kBlock + 1]   (MPPI only)
  __shared__ float s_wm[kBlock / 32];
  __shared__ int s_wk[kBlock / 32], s_wf[kBlock / 32];
  __shared__ float s_tile_m, s_run_m;
  __shared__ int s_tile_k, s_tile_f, s_run_k, s_run_f;

  const int r = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  load_robot(p, r, s);
  if (tid == 0) {
    s_run_m = kInf;
    s_run_k = 0x7fffffff;
    s_run_f = 0;
  }
  __syncthreads();
  const uint32_t robot_g = (uint32_t)(p.robot_offset + r);
  float run = 0.0f;  // running partial of row `tid` (MPPI)

  for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const int64_t kl = (int64_t)tile * kBlock + tid;
    const bool valid = kl < p.K_local;
    const int64_t k = p.k_begin + kl;
    float th[D];
    float J = kInf;
    int fi = 0;
    if (valid) {
      fi = draw_sample<P, false>(p, robot_g, k, s, th);
      J = rollout<P>(p, th, fi, s);
      p.J[(size_t)r * p.K_local + kl] = J;
    }
    if (!MPPI) continue;
    // ---- step a5, per tile: min, weights, sums (online softmax merge) ----
    float m = J;
    int mk = valid ? (int)k : 0x7fffffff, mf = fi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const int k2 = __shfl_xor_sync(0xffffffffu, mk, o);
      const int f2 = __shfl_xor_sync(0xffffffffu, mf, o);
      if (jk_less(m2, k2, m, mk)) {
        m = m2;
        mk = k2;
        mf = f2;
      }
    }
    if (lane == 0) {
      s_wm[warp] = m;
      s_wk[warp] = mk;
      s_wf[warp] = mf;
    }
    __syncthreads();
    if (tid == 0) {
      float bm = s_wm[0];
      int bk = s_wk[0], bf = s_wf[0];
      for (int w = 1; w < kBlock / 32; ++w)
        if (jk_less(s_wm[w], s_wk[w], bm, bk)) {
          bm = s_wm[w];
          bk = s_wk[w];
          bf = s_wf[w];
        }
      s_tile_m = bm;
      s_tile_k = bk;
      s_tile_f = bf;
    }
    __syncthreads();
    const float mt = s_tile_m;
    const bool fin = J < kInf;
    const float w = fin ? __expf((mt - J) * p.inv_lambda) : 0.0f;
    if (valid) {
#pragma unroll
      for (int d = 0; d < D; ++d) s_red[d * (kBlock + 1) + tid] = w * th[d];
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) s_red[d * (kBlock + 1) + tid] = 0.0f;
    }
    s_red[(D + 0) * (kBlock + 1) + tid] = w;
    s_red[(D + 1) * (kBlock + 1) + tid] = w * w;
    s_red[(D + 2) * (kBlock + 1) + tid] = fin ? J : 0.0f;
    s_red[(D + 3) * (kBlock + 1) + tid] = fin ? 1.0f : 0.0f;
    __syncthreads();
    const float mr = s_run_m;
    const float mn = fminf(mr, mt);
    if (tid < NR) {
      const float* row = &s_red[tid * (kBlock + 1)];
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 8
      for (int i = 0; i < kBlock; i += 4) {
        a0 += row[i];
        a1 += row[i + 1];
        a2 += row[i + 2];
        a3 += row[i + 3];
      }
      const float v = (a0 + a1) + (a2 + a3);
      const float sa = (mr < kInf) ? __expf((mn - mr) * p.inv_lambda) : 0.0f;
      const float sb = (mt < kInf) ? __expf((mn - mt) * p.inv_lambda) : 0.0f;
      if (tid < D + 1) run = fmaf(run, sa, v * sb);
      else if (tid == D + 1) run = fmaf(run, sa * sa, v * (sb * sb));
      else run += v;
    }
    __syncthreads();
    if (tid == 0 && jk_less(mt, s_tile_k, s_run_m, s_run_k)) {
      s_run_m = mt;
      s_run_k = s_tile_k;
      s_run_f = s_tile_f;
    }
    __syncthreads();
  }
  if (MPPI) {
    float* out = p.part + ((size_t)r * p.n_cta + blockIdx.x) * kPartStride;
    if (tid < D) out[kPartHdr + tid] = run;
    else if (tid == D) out[3] = run;
    else if (tid == D + 1) out[4] = run;
    else if (tid == D + 2) out[5] = run;
    else if (tid == D + 3) out[6] = run;
    if (tid == 0) {
      out[0] = s_run_m;
      out[1] = __int_as_float(s_run_k);
      out[2] = __int_as_float(s_run_f);
      out[7] = 0.0f;
    }
  }
}

// ---------------------------------------------------------------------------
// Output (a7): u0 = delta_0-masked cone projection of knot 0.
// ---------------------------------------------------------------------------
__device__ void write_output(const Params& p, int r, int status, const float* mean_new, const float* var_new,
                             int fi, float jmin, float jmean, float omega, float ess, int ndiv) {
  sbs_output* o = p.out + r;
  const int D = p.D;
  const uint32_t ph0 = p.in[r].phase_q32;
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
    o->iter = p.iter;
    o->j_min = jmin;
    o->j_mean = jmean;
    o->omega = omega;
    o->ess = ess;
    o->n_diverged = ndiv;
    o->device_us = 0.0f;
    p.status[r] = status;
  }
}

// ---------------------------------------------------------------------------
// sbs_mppi_finalize: grid R, block 128.  beta = min over CTA partials; each
// partial rescaled by exp(-(m_c - beta)/lambda) (Alg. 4 UpdateMean).
// ---------------------------------------------------------------------------
// Partial records: CTA partials [R][n_cta] (part_c_stride = 1) or the rank
// partials gathered by NCCL [world][R] (part_c_stride = R, n_cta = world).
__device__ __forceinline__ const float* part_rec(const Params& p, int r, int c) {
  return p.part_c_stride == 1 ? p.part + ((size_t)r * p.n_cta + c) * kPartStride
                              : p.part + ((size_t)c * p.part_c_stride + r) * kPartStride;
}

template <bool EMIT>
__global__ void __launch_bounds__(128) sbs_mppi_finalize(const __grid_constant__ Params p, float* emit) {
  const int r = blockIdx.x, tid = threadIdx.x, D = p.D;
  __shared__ float s_m[4];
  __shared__ int s_k[4], s_f[4];
  __shared__ float s_row[SBS_MAX_D + 4];
  __shared__ float s_mean[SBS_MAX_D], s_var[SBS_MAX_D];
  float m = kInf;
  int mk = 0x7fffffff, mf = 0;
  for (int c = tid; c < p.n_cta; c += blockDim.x) {
    const float* pc = part_rec(p, r, c);
    const float mc = pc[0];
    const int kc = __float_as_int(pc[1]);
    if (jk_less(mc, kc, m, mk)) {
      m = mc;
      mk = kc;
      mf = __float_as_int(pc[2]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const int k2 = __shfl_xor_sync(0xffffffffu, mk, o);
    const int f2 = __shfl_xor_sync(0xffffffffu, mf, o);
    if (jk_less(m2, k2, m, mk)) {
      m = m2;
      mk = k2;
      mf = f2;
    }
  }
  if ((tid & 31) == 0) {
    s_m[tid >> 5] = m;
    s_k[tid >> 5] = mk;
    s_f[tid >> 5] = mf;
  }
  __syncthreads();
  float beta = s_m[0];
  int bk = s_k[0], bf = s_f[0];
  for (int w = 1; w < 4; ++w)
    if (jk_less(s_m[w], s_k[w], beta, bk)) {
      beta = s_m[w];
      bk = s_k[w];
      bf = s_f[w];
    }
  // rows: 0..D-1 -> V, D -> S, D+1 -> S2, D+2 -> sumJ, D+3 -> nfin
  if (tid < D + 4) {
    const int col = tid < D ? kPartHdr + tid : 3 + (tid - D);
    float acc = 0.0f;
    for (int c = 0; c < p.n_cta; ++c) {
      const float* pc = part_rec(p, r, c);
      const float mc = pc[0];
      float sc = (mc < kInf) ? __expf((beta - mc) * p.inv_lambda) : 0.0f;
      if (tid == D + 1) sc = sc * sc;
      if (tid >= D + 2) sc = 1.0f;
      acc = fmaf(pc[col], sc, acc);
    }
    s_row[tid] = acc;
  }
  __syncthreads();
  if (EMIT) {  // this rank's merged partial, relative to its own beta
    float* o = emit + (size_t)r * kPartStride;
    if (tid < D) o[kPartHdr + tid] = s_row[tid];
    else if (tid < D + 4) o[3 + tid - D] = s_row[tid];
    if (tid == 0) {
      o[0] = beta;
      o[1] = __int_as_float(bk);
      o[2] = __int_as_float(bf);
      o[7] = 0.0f;
    }
    return;
  }
  const bool all_div = !(beta < kInf);
  const float S = s_row[D], S2 = s_row[D + 1], sumJ = s_row[D + 2], nfin = s_row[D + 3];
  float* mean = p.mean + (size_t)r * D;
  const float* var = p.var + (size_t)r * D;
  for (int d = tid; d < D; d += blockDim.x) {
    s_mean[d] = all_div ? mean[d] : s_row[d] / S;
    s_var[d] = var[d];
  }
  __syncthreads();
  for (int d = tid; d < D; d += blockDim.x) mean[d] = s_mean[d];
  const int fi = all_div ? p.fidx[r] : bf;
  __syncthreads();
  if (tid == 0) p.fidx[r] = fi;
  const float K = (float)p.K_global;
  write_output(p, r, all_div ? SBS_WARN_ALL_DIVERGED : SBS_OK, s_mean, s_var, fi, beta,
               nfin > 0.f ? sumJ / nfin : kInf, S, all_div ? 0.f : S * S / S2, (int)(K - nfin));
}

// ---------------------------------------------------------------------------
// Elite selection (a6; Alg. 1 lines 3-5, L4): the K_e smallest keys (J, k).
// Radix select on order-preserving 32-bit keys of J (NaN -> +inf, -0 -> +0),
// four 8-bit passes in shared memory, then an index-ordered compaction that
// takes all keys < T and the lowest-index ties == T.  One CTA per robot.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cost_key(float J) {
  if (J != J) J = kInf;
  if (J == 0.0f) J = 0.0f;  // -0 -> +0
  const uint32_t u = __float_as_uint(J);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

constexpr int kSelBlock = 1024;
constexpr int kEliteBlock = 512;  // <= 128 registers per thread: theta[D] and acc[D] stay resident

// returns via smem: elite[0..K_e) ascending global indices, best (rank-1),
// diag[0..2] = (J_min, mean finite J, n diverged)
__device__ void select_block(const float* J, int64_t K, int64_t K_e, int64_t k_begin, int64_t* elite,
                             int64_t* best, float* diag) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_prefix, s_want;
  __shared__ uint32_t s_wsum[kSelBlock / 32];
  __shared__ unsigned long long s_best;
  __shared__ float s_sum[kSelBlock / 32];
  __shared__ int s_nf[kSelBlock / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_prefix = 0;
    s_want = (uint32_t)K_e;
    s_best = ~0ull;
  }
  // diagnostics + best
  unsigned long long b = ~0ull;
  float sj = 0.f;
  int nf = 0;
  for (int64_t k = tid; k < K; k += blockDim.x) {
    const float j = J[k];
    const unsigned long long kk = ((unsigned long long)cost_key(j) << 32) | (unsigned long long)k;
    b = kk < b ? kk : b;
    if (j < kInf) {
      sj += j;
      nf += 1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, b, o);
    b = b2 < b ? b2 : b;
    sj += __shfl_xor_sync(0xffffffffu, sj, o);
    nf += __shfl_xor_sync(0xffffffffu, nf, o);
  }
  if (lane == 0) {
    s_sum[warp] = sj;
    s_nf[warp] = nf;
  }
  __syncthreads();
  if (lane == 0) atomicMin(&s_best, b);
  if (tid == 0) {
    float t = 0.f;
    int n = 0;
    for (int w = 0; w < kSelBlock / 32; ++w) {
      t += s_sum[w];
      n += s_nf[w];
    }
    diag[1] = n > 0 ? t / n : kInf;
    diag[2] = (float)(K - n);
  }
  // four radix passes, most significant digit first
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (int64_t k = tid; k < K; k += blockDim.x) {
      const uint32_t key = cost_key(J[k]);
      if ((key & hmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t want = s_want, cum = 0;
      int dgt = 0;
      for (; dgt < 256; ++dgt) {
        if (cum + hist[dgt] >= want) break;
        cum += hist[dgt];
      }
      s_want = want - cum;
      s_prefix = prefix | ((uint32_t)dgt << shift);
    }
    __syncthreads();
  }
  const uint32_t T = s_prefix;
  const uint32_t n_eq = s_want;  // ties at T to take, lowest indices first
  // index-ordered compaction
  uint32_t sel_base = 0, eq_base = 0;
  for (int64_t base = 0; base < K; base += blockDim.x) {
    const int64_t k = base + tid;
    uint32_t key = 0xFFFFFFFFu;
    bool lt = false, eq = false;
    if (k < K) {
      key = cost_key(J[k]);
      lt = key < T;
      eq = key == T;
    }
    // exclusive scan of eq within the block
    const unsigned eqb = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) s_wsum[warp] = __popc(eqb);
    __syncthreads();
    uint32_t eq_before = eq_base + __popc(eqb & ((1u << lane) - 1u));
    uint32_t eq_tot = 0;
    for (int w = 0; w < kSelBlock / 32; ++w) {
      const uint32_t c = s_wsum[w];
      if (w < warp) eq_before += c;
      eq_tot += c;
    }
    const bool sel = lt || (eq && eq_before < n_eq);
    __syncthreads();
    const unsigned sb = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) s_wsum[warp] = __popc(sb);
    __syncthreads();
    uint32_t pos = sel_base + __popc(sb & ((1u << lane) - 1u));
    uint32_t sel_tot = 0;
    for (int w = 0; w < kSelBlock / 32; ++w) {
      const uint32_t c = s_wsum[w];
      if (w < warp) pos += c;
      sel_tot += c;
    }
    if (sel) elite[pos] = k_begin + k;
    sel_base += sel_tot;
    eq_base += eq_tot;
    __syncthreads();
  }
  if (tid == 0) {
    const unsigned long long bb = s_best;
    *best = k_begin + (int64_t)(bb & 0xFFFFFFFFull);
    const uint32_t key = (uint32_t)(bb >> 32);
    const uint32_t u = (key & 0x80000000u) ? (key & 0x7FFFFFFFu) : ~key;
    diag[0] = __uint_as_float(u);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSelBlock) sbs_select_kernel(const __grid_constant__ Params p) {
  const int r = blockIdx.x;
  select_block(p.J + (size_t)r * p.K_local, p.K_local, p.n_elite, p.k_begin, p.elite + (size_t)r * p.n_elite,
               p.best + r, p.part + (size_t)r * kPartStride);
}

__global__ void __launch_bounds__(kSelBlock) sbs_select_raw_kernel(const float* J, int64_t K, int64_t K_e,
                                                                   int64_t* idx, int64_t* best, float* diag) {
  select_block(J, K, K_e, 0, idx, best, diag);
}

// ---------------------------------------------------------------------------
// sbs_elite_kernel: grid R, block kEliteBlock.  Elite moments from theta
// regenerated with the counter RNG (no theta buffer in HBM).
// ---------------------------------------------------------------------------
template <int P>
__device__ void block_sum_rows(float (&v)[12 * P], float* s_acc /*[32][12P]*/, float* out /*[12P]*/) {
  constexpr int D = 12 * P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    float x = v[d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_acc[warp * D + d] = x;
  }
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float t = 0.f;
    for (int w = 0; w < nw; ++w) t += s_acc[w * D + d];
    out[d] = t;
  }
  __syncthreads();
}

template <int P>
__global__ void __launch_bounds__(kEliteBlock) sbs_elite_kernel(const __grid_constant__ Params p) {
  constexpr int D = 12 * P;
  __shared__ RobotSmem s;
  __shared__ float s_acc[(kEliteBlock / 32) * D];
  __shared__ float s_mean[D], s_var[D], s_sum[D];
  __shared__ int s_n[kEliteBlock / 32];
  __shared__ int s_best_f;
  const int r = blockIdx.x, tid = threadIdx.x;
  load_robot(p, r, s);
  __syncthreads();
  const uint32_t robot_g = (uint32_t)(p.robot_offset + r);
  const int64_t* el = p.elite + (size_t)r * p.n_elite;
  const float* Jr = p.J + (size_t)r * p.K_local;
  const float* diag = p.part + (size_t)r * kPartStride;
  const int64_t kb = p.best[r];
  const bool cem = p.mode == SBS_CEM;
  const bool all_div = !(Jr[kb - p.k_begin] < kInf);
  float th[D];
  float acc[D];
  // pass 1: elite sum and count of finite elites
#pragma unroll
  for (int d = 0; d < D; ++d) acc[d] = 0.f;
  int n = 0;
  for (int64_t e = tid; e < p.n_elite; e += blockDim.x) {
    const int64_t k = el[e];
    if (!(Jr[k - p.k_begin] < kInf)) continue;  // diverged samples never enter the moments (L17)
    draw_sample<P, false>(p, robot_g, k, s, th);
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] += th[d];
    ++n;
  }
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((tid & 31) == 0) s_n[tid >> 5] = n;
  block_sum_rows<P>(acc, s_acc, s_sum);
  int ntot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) ntot += s_n[w];
  for (int d = tid; d < D; d += blockDim.x) s_mean[d] = all_div ? p.mean[(size_t)r * D + d] : s_sum[d] / (float)ntot;
  __syncthreads();
  if (cem && !all_div) {
    // pass 2: diagonal population variance about the elite mean, floored (L17)
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = 0.f;
    for (int64_t e = tid; e < p.n_elite; e += blockDim.x) {
      const int64_t k = el[e];
      if (!(Jr[k - p.k_begin] < kInf)) continue;
      draw_sample<P, false>(p, robot_g, k, s, th);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const float dv = th[d] - s_mean[d];
        acc[d] = fmaf(dv, dv, acc[d]);
      }
    }
    block_sum_rows<P>(acc, s_acc, s_sum);
    for (int d = tid; d < D; d += blockDim.x) s_var[d] = fmaxf(s_sum[d] / (float)ntot, p.var_floor[d % 3]);
  } else {
    for (int d = tid; d < D; d += blockDim.x) s_var[d] = p.var[(size_t)r * D + d];
  }
  if (tid == 0) {
    int f = s.cur_idx;
    if (!all_div) f = draw_sample<P, false>(p, robot_g, kb, s, th);  // theta1 of the rank-1 sample (L16)
    s_best_f = f;
  }
  __syncthreads();
  for (int d = tid; d < D; d += blockDim.x) {
    p.mean[(size_t)r * D + d] = s_mean[d];
    p.var[(size_t)r * D + d] = s_var[d];
  }
  if (tid == 0) p.fidx[r] = s_best_f;
  write_output(p, r, all_div ? SBS_WARN_ALL_DIVERGED : SBS_OK, s_mean, s_var, s_best_f, diag[0], diag[1],
               (float)ntot, (float)ntot, (int)diag[2]);
}

// ---------------------------------------------------------------------------
// debug: z, theta, theta1 of samples k0..k0+n-1 of one robot (same draw code)
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(128) sbs_debug_samples_kernel(const __grid_constant__ Params p, int r, int64_t k0,
                                                                int64_t n, float* z, float* theta, int* fidx) {
  constexpr int D = 12 * P;
  __shared__ RobotSmem s;
  load_robot(p, r, s);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float th[D], zz[D];
  const int f = draw_sample<P, true>(p, (uint32_t)(p.robot_offset + r), k0 + i, s, th, zz);
  for (int d = 0; d < D; ++d) {
    z[i * D + d] = zz[d];
    theta[i * D + d] = th[d];
  }
  fidx[i] = f;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int P, bool MPPI>
static cudaError_t launch_rollout_t(const Params& p, cudaStream_t s) {
  constexpr int D = 12 * P;
  const size_t smem = MPPI ? (size_t)(D + 4) * (kBlock + 1) * sizeof(float) : 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sbs_rollout_kernel<P, MPPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  dim3 grid(p.n_cta, p.R);
  sbs_rollout_kernel<P, MPPI><<<grid, kBlock, smem, s>>>(p);
  return cudaGetLastError();
}

template <int P, bool MPPI>
static int occupancy_t() {
  constexpr int D = 12 * P;
  const size_t smem = MPPI ? (size_t)(D + 4) * (kBlock + 1) * sizeof(float) : 0;
  cudaFuncSetAttribute(sbs_rollout_kernel<P, MPPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sbs_rollout_kernel<P, MPPI>, kBlock, smem) != cudaSuccess)
    return 1;
  return n > 0 ? n : 1;
}

#define SBS_DISPATCH_P(P_, EXPR) \
  switch (P_) {                  \
    case 2: { constexpr int PP = 2; EXPR; } \
    case 3: { constexpr int PP = 3; EXPR; } \
    case 4: { constexpr int PP = 4; EXPR; } \
    case 5: { constexpr int PP = 5; EXPR; } \
    case 6: { constexpr int PP = 6; EXPR; } \
    case 7: { constexpr int PP = 7; EXPR; } \
    case 8: { constexpr int PP = 8; EXPR; } \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_rollout(const Params& p, bool mppi, cudaStream_t s) {
  if (mppi) {
    SBS_DISPATCH_P(p.P, return (launch_rollout_t<PP, true>(p, s)));
  } else {
    SBS_DISPATCH_P(p.P, return (launch_rollout_t<PP, false>(p, s)));
  }
}

int rollout_occupancy(int P, bool mppi) {
  auto f = [&]() -> int {
    if (mppi) {
      switch (P) {
        case 2: return occupancy_t<2, true>();
        case 3: return occupancy_t<3, true>();
        case 4: return occupancy_t<4, true>();
        case 5: return occupancy_t<5, true>();
        case 6: return occupancy_t<6, true>();
        case 7: return occupancy_t<7, true>();
        default: return occupancy_t<8, true>();
      }
    }
    switch (P) {
      case 2: return occupancy_t<2, false>();
      case 3: return occupancy_t<3, false>();
      case 4: return occupancy_t<4, false>();
      case 5: return occupancy_t<5, false>();
      case 6: return occupancy_t<6, false>();
      case 7: return occupancy_t<7, false>();
      default: return occupancy_t<8, false>();
    }
  };
  return f();
}

cudaError_t launch_mppi_finalize(const Params& p, cudaStream_t s) {
  sbs_mppi_finalize<false><<<p.R, 128, 0, s>>>(p, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_mppi_merge(const Params& p, float* dst, cudaStream_t s) {
  sbs_mppi_finalize<true><<<p.R, 128, 0, s>>>(p, dst);
  return cudaGetLastError();
}

cudaError_t launch_select(const Params& p, cudaStream_t s) {
  sbs_select_kernel<<<p.R, kSelBlock, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_elite(const Params& p, cudaStream_t s) {
  SBS_DISPATCH_P(p.P, (sbs_elite_kernel<PP><<<p.R, kEliteBlock, 0, s>>>(p)); return cudaGetLastError());
}

cudaError_t launch_debug_samples(const Params& p, int robot, int64_t k0, int64_t n, float* z, float* theta,
                                 int* fidx, cudaStream_t s) {
  const int blocks = (int)((n + 127) / 128);
  SBS_DISPATCH_P(p.P, (sbs_debug_samples_kernel<PP><<<blocks, 128, 0, s>>>(p, robot, k0, n, z, theta, fidx));
                 return cudaGetLastError());
}

cudaError_t launch_select_raw(const float* J, int64_t K, int64_t K_e, int64_t* idx, int64_t* best,
                              cudaStream_t s) {
  float* diag = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&diag, 4 * sizeof(float), s);
  if (e != cudaSuccess) return e;
  sbs_select_raw_kernel<<<1, kSelBlock, 0, s>>>(J, K, K_e, idx, best, diag);
  e = cudaGetLastError();
  cudaFreeAsync(diag, s);
  return e;
}

}  // namespace sbs
