// sbs_robot_model.h -- the robot model compiled into the rollout as immediate
// operands ("compiled-in robot model").
//
// The rollout's model and cost constants (Eq. 1 mass / inertia / gravity,
// P:265-277; the cone of P:294 / L9; the cost weights of P:344-351 / L11; dt of
// P:340) are normally read from the kernel parameter block.  For the robot below
// (Aliengo, reading L29, with the cost of L11 and the cone of L9) a second
// instantiation of the throughput rollout takes them as compile-time constants, so
// the compiler folds them into immediate operands and needs no registers for them.
// sbs_create selects that instantiation only when every value of the context's
// parameter block equals the value computed here, bit for bit (model_matches in
// sbs_api.cpp); any other robot runs the generic instantiation.  Both compute the
// same formulas; the parity tests run both against the oracle.
#pragma once
#include <stdint.h>

namespace sbs {
namespace model {

constexpr int kKnots = 4;                                        // P (the only instantiation)
constexpr float kMass = 21.0f;
constexpr float kI0 = 0.135f, kI1 = 0.54f, kI2 = 0.58f;          // L29, body frame, diagonal
constexpr float kGz = -9.81f;                                    // g = (0, 0, g_z)
constexpr float kDt = 0.02f;
constexpr float kMu = 0.5f, kFzMin = 5.0f, kFzMax = 180.0f;      // L9
constexpr float kQp = 15.0f, kQz = 30.0f, kQv = 2.0f, kQa = 5.0f, kQw = 0.2f;  // L11: (p_xy, p_z | v | Phi | w)
constexpr float kR = 1e-6f;                                      // L11, every force component
constexpr float kWfc = 1e-3f;                                    // L9
__host__ __device__ constexpr float Q(int i) { return i < 2 ? kQp : (i == 2 ? kQz : (i < 6 ? kQv : (i < 9 ? kQa : kQw))); }

// derived exactly as sbs_create derives them (binary64, then rounded once)
constexpr double kDet = (double)kI0 * ((double)kI1 * (double)kI2);
constexpr float kInvMass = (float)(1.0 / (double)kMass);
constexpr float kIinv0 = (float)(((double)kI1 * (double)kI2) / kDet);
constexpr float kIinv1 = (float)(((double)kI0 * (double)kI2) / kDet);
constexpr float kIinv2 = (float)(((double)kI0 * (double)kI1) / kDet);
// gyroscopic coefficients of the diagonal-inertia Euler equations, binary32 as sbs_create
// forms them: G_x = I^-1_x (I_y - I_z), G_y = I^-1_y (I_z - I_x), G_z = I^-1_z (I_x - I_y)
constexpr float kGyr0 = kIinv0 * (kI1 - kI2);
constexpr float kGyr1 = kIinv1 * (kI2 - kI0);
constexpr float kGyr2 = kIinv2 * (kI0 - kI1);
__host__ __device__ constexpr float urz(int n) {  // u^r_z = -m g_z / max(1, n) (L12)
  return (float)(-(double)kMass * (double)kGz / (double)(n > 1 ? n : 1));
}

}  // namespace model
}  // namespace sbs
