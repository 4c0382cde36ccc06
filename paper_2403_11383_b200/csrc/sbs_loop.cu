// sbs_loop.cu -- the closed loop around one MPC iteration (
// DESIGN.md readings L36-L40): after a step, one thread per robot advances
// the plant by one control period and builds the next iteration's inputs and
// reference in device memory, so an episode runs without host round trips.
//
//   plant (L36): one RK4 step of Eq. 1 with u0 held on the stance
//                legs and an external CoM wrench, binary32, SFU sin/cos
//                as in the rollout (one thread per robot: the libm versions'
//                slow paths dominated a single robot's control step);
//   fall (L40), gait phase (L37), footholds by Eq. 3,
//   reference (L13).
#include <math.h>

#include "sbs_internal.h"

namespace sbs {

namespace {

// Eq. 1 with the CoM wrench: x = (p, v, (roll, pitch, yaw), omega_body)
__device__ void plant_f(const Params& p, const float x[12], const float u[12], const int st[4], const float feet[12],
                        const float w[6], float xd[12]) {
  float cr, sr, cp, sp, cy, sy;  // SFU sin/cos (abs. error ~4e-7 on the plant's angles), as in the rollout
  __sincosf(x[6], &sr, &cr);
  __sincosf(x[7], &sp, &cp);
  __sincosf(x[8], &sy, &cy);
  // R = Rz(yaw) Ry(pitch) Rx(roll)
  const float R[9] = {cy * cp, cy * sp * sr - sy * cr, cy * sp * cr + sy * sr,
                      sy * cp, sy * sp * sr + cy * cr, sy * sp * cr - cy * sr,
                      -sp,     cp * sr,                cp * cr};
  float F[3] = {w[0], w[1], w[2]};
  float tw[3] = {w[3], w[4], w[5]};
  for (int i = 0; i < 4; ++i) {
    if (!st[i]) continue;
    const float* G = u + 3 * i;
    const float r0 = feet[3 * i] - x[0], r1 = feet[3 * i + 1] - x[1], r2 = feet[3 * i + 2] - x[2];
    F[0] += G[0];
    F[1] += G[1];
    F[2] += G[2];
    tw[0] += r1 * G[2] - r2 * G[1];
    tw[1] += r2 * G[0] - r0 * G[2];
    tw[2] += r0 * G[1] - r1 * G[0];
  }
  const float* wb = x + 9;
  float tb[3], Iw[3];
  for (int a = 0; a < 3; ++a) {
    tb[a] = R[a] * tw[0] + R[3 + a] * tw[1] + R[6 + a] * tw[2];  // R^T tau
    Iw[a] = p.I[3 * a] * wb[0] + p.I[3 * a + 1] * wb[1] + p.I[3 * a + 2] * wb[2];
  }
  const float rhs[3] = {tb[0] - (wb[1] * Iw[2] - wb[2] * Iw[1]), tb[1] - (wb[2] * Iw[0] - wb[0] * Iw[2]),
                        tb[2] - (wb[0] * Iw[1] - wb[1] * Iw[0])};
  for (int a = 0; a < 3; ++a) {
    xd[a] = x[3 + a];
    xd[3 + a] = F[a] * p.inv_mass + p.g[a];
    xd[9 + a] = p.Iinv[3 * a] * rhs[0] + p.Iinv[3 * a + 1] * rhs[1] + p.Iinv[3 * a + 2] * rhs[2];
  }
  const float s = sr * wb[1] + cr * wb[2];
  xd[6] = wb[0] + __fdividef(sp, cp) * s;
  xd[7] = cr * wb[1] - sr * wb[2];
  xd[8] = s / cp;
}

__device__ void plant_rk4(const Params& p, const float x[12], const float u[12], const int st[4], const float feet[12],
                          const float w[6], float h, float xn[12]) {
  float k1[12], k2[12], k3[12], k4[12], t[12];
  plant_f(p, x, u, st, feet, w, k1);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + 0.5f * h * k1[a];
  plant_f(p, t, u, st, feet, w, k2);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + 0.5f * h * k2[a];
  plant_f(p, t, u, st, feet, w, k3);
  for (int a = 0; a < 12; ++a) t[a] = x[a] + h * k3[a];
  plant_f(p, t, u, st, feet, w, k4);
  for (int a = 0; a < 12; ++a) xn[a] = x[a] + h / 6.0f * (k1[a] + 2.0f * k2[a] + 2.0f * k3[a] + k4[a]);
}

__device__ __forceinline__ bool stance_at(const Params& p, uint32_t phase, int leg) {
  return p.all_stance || (phase + p.off[leg] < p.thr);
}

}  // namespace

__global__ void __launch_bounds__(128) sbs_advance_kernel(const __grid_constant__ Params p, const LoopArgs a,
                                                          sbs_input* in, const sbs_output* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the step's outputs
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < p.R) {
    const uint32_t it = a.loop ? (__ldcg(a.loop) - __ldcg(a.loop + 1)) / (uint32_t)a.n_inner : 0u;  // control step
    sbs_input s = in[r];
    const sbs_output& o = out[r];
    const bool was_fallen = a.fallen && a.fallen[r];
    float x[12];
    int fallen = 0;
    if (!was_fallen) {
      float w[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (a.wrench)
        for (int k = 0; k < 6; ++k) w[k] = a.wrench[((size_t)it * p.R + r) * 6 + k];
      int st[4];
      for (int i = 0; i < 4; ++i) st[i] = o.contact0[i];
      // 1. plant (L36)
      plant_rk4(p, s.x0, o.u0, st, s.feet_cur, w, p.dt, x);
      // 2. fall criterion (L40)
      for (int k = 0; k < 12; ++k) fallen |= !isfinite(x[k]);
      fallen |= fabsf(x[6]) > a.fall_angle || fabsf(x[7]) > a.fall_angle || x[2] < a.fall_height;
      // 3. gait phase at the chosen frequency (L37)
      const int fi = o.freq_idx;
      const uint32_t ph = s.phase_q32 + p.inc[fi];
      // 4. touchdown: swing at the old phase (contact0), stance at the new one -> planned foothold (L38)
      for (int i = 0; i < 4; ++i)
        if (!o.contact0[i] && stance_at(p, ph, i))
          for (int k = 0; k < 3; ++k) s.feet_cur[3 * i + k] = s.feet_next[3 * i + k];
      // 5. next footholds: Eq. 3 at the new state, T_st = D_f / f_s
      const sbs_command c = a.cmd ? a.cmd[r] : sbs_command{{0.f, 0.f, 0.f}, 0.f};
      const float t_st = p.duty / p.freq_hz[fi];
      const float kfb = sqrtf(fmaxf(x[2], 0.f) / fabsf(p.g[2]));
      float cy, sy;
      __sincosf(x[8], &sy, &cy);
      for (int i = 0; i < 4; ++i) {
        const float hx = a.hip[3 * i], hy = a.hip[3 * i + 1];
        const float px = x[0] + (cy * hx - sy * hy), py = x[1] + (sy * hx + cy * hy);
        s.feet_next[3 * i] = px + 0.5f * t_st * c.v[0] + kfb * (x[3] - c.v[0]);
        s.feet_next[3 * i + 1] = py + 0.5f * t_st * c.v[1] + kfb * (x[4] - c.v[1]);
        s.feet_next[3 * i + 2] = 0.f;
      }
      // 6. reference (L13) for the next iteration
      float* xr = const_cast<float*>(p.xref) + (size_t)r * p.H * 12;
      for (int j = 0; j < p.H; ++j) {
        const float t = (float)j * p.dt;
        float* q = xr + 12 * j;
        q[0] = x[0] + c.v[0] * t;
        q[1] = x[1] + c.v[1] * t;
        q[2] = a.h_nom;
        q[3] = c.v[0];
        q[4] = c.v[1];
        q[5] = c.v[2];
        q[6] = 0.f;
        q[7] = 0.f;
        q[8] = x[8] + c.yaw_rate * t;
        q[9] = 0.f;
        q[10] = 0.f;
        q[11] = c.yaw_rate;
      }
      for (int k = 0; k < 12; ++k) s.x0[k] = x[k];
      s.phase_q32 = ph;
      in[r] = s;
      if (a.fallen && fallen) a.fallen[r] = 1;
    } else {
      for (int k = 0; k < 12; ++k) x[k] = s.x0[k];
      fallen = 1;
    }
    if (a.trace) {
      float* t = a.trace + ((size_t)it * p.R + r) * SBS_TRACE_FLOATS;
      for (int k = 0; k < 12; ++k) t[k] = x[k];
      t[12] = o.freq_hz;
      t[13] = o.j_min;
      t[14] = (float)(fallen || was_fallen);
      t[15] = (float)o.status;
    }
  }
  if (a.loop) {  // the last CTA to finish moves the device iteration counter (read by the next step)
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(a.counter, 1) == (int)gridDim.x - 1;
      if (s_last) {
        *a.counter = 0;
        a.loop[0] += (uint32_t)a.n_inner;
      }
    }
  }
}

cudaError_t launch_advance(const Params& p, const LoopArgs& a, sbs_input* in, const sbs_output* out, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};  // programmatic dependent launch after the step's last kernel
  cfg.gridDim = dim3((p.R + 127) / 128);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sbs_advance_kernel, p, a, in, out);
}

}  // namespace sbs
