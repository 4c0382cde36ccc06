// sbs_internal.h -- shared between the host runtime (sbs_api.cpp) and the
// kernels (sbs_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sbs.h"

// Device-side bounds checks (the SBS_CHECKED build, tests only: compute-sanitizer is not
// available on the GPU pool): every kernel index that addresses a context buffer is
// checked against the bound its allocation was sized with; a violation prints and traps.
#if defined(SBS_CHECKED)
#include <cstdio>
#define SBS_CHECK(cond)                                                                               \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("SBS_CHECK failed: %s (%s:%d) block (%d,%d) thread %d\n", #cond, __FILE__, __LINE__,       \
             (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                                     \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define SBS_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace sbs {

constexpr int kBlock = 128;         // samples per tile = threads per rollout CTA
constexpr int kRedStride = kBlock + 4;  // floats per row of the MPPI tile reduction (16-byte rows)
constexpr int kMaxWorld = 8;               // ranks of one node (peer-memory exchange)
constexpr int kInlineRefFloats = 16 * 12;  // host path, R = 1, H <= 16: inputs and reference ride in the kernel parameters
constexpr int kSplitLanes = 4;      // latency-mode (SPLIT) rollout: lanes per sample in the sampler phase
constexpr int kPartHdr = 8;         // [m, k_argmin, fidx_argmin, S, S2, sumJ, nfin, pad]
constexpr int kEPartStride = 2 * SBS_MAX_D + 4;  // CEM elite-moment record [S1[D], n, S2[D]]
constexpr int kDynMaxLevels = 5;                // dynamic tile scheduling: reduction-tree depth limit
constexpr int kDynBatch = 8;                    // tiles per release fence
// full-covariance CEM elite record [S1[D], n, lower triangle of S2 (D (D + 1) / 2)], 16-byte multiple
__host__ __device__ constexpr int fc_record_floats(int D) { return ((D + 1 + D * (D + 1) / 2) + 3) / 4 * 4; }
// latency-mode shared memory: MPPI reduction rows, theta / theta1 of the tile, and (ab)
// the producer warps' stance-leg table [H][7][kBlock]
constexpr size_t kSplitSmemMax = 200 * 1024;
__host__ __device__ constexpr size_t split_smem_bytes(int P, bool mppi, int H, bool ab) {
  return (mppi ? (size_t)(12 * P + 4) * kRedStride * 4 : 0) + (size_t)kBlock * (12 * P + 2) * 4 +
         (ab ? (size_t)7 * H * kBlock * 4 : 0);
}
#ifndef SBS_ROLLOUT_MIN_BLOCKS
#define SBS_ROLLOUT_MIN_BLOCKS 4
#endif
constexpr int kRolloutMinBlocks = SBS_ROLLOUT_MIN_BLOCKS;  // __launch_bounds__ min CTAs per SM

// Everything a kernel needs, passed by value (__grid_constant__, < 4 KB).
struct Params {
  // --- model (Eq. 1) ---
  float inv_mass;
  float g[3];
  float I[9], Iinv[9];
  int diag_inertia;
  float gyr[3];               // diagonal I: I^-1_x (I_y - I_z), I^-1_y (I_z - I_x), I^-1_z (I_x - I_y) (binary32)
  float mu, fz_min, fz_max;
  float dt;
  float duty;                 // duty factor D_f (closed-loop T_st = D_f / f_s)
  // --- cost ---
  float Q[12], Rw[12];
  float rho, f_nominal, w_fc, inv_lambda;
  float urz[5];               // u^r_z = -m g_z / max(1, n_stance)   (L12)
  // loop-invariant operand pairs of the rollout's packed FP32x2 arithmetic, formed on the
  // host (same binary32 operations as the scalar forms) so that the kernel reads them as
  // uniform-register pairs: dt, dt/2, dt/6, 2, dt^2/2, dt^2/4, (1/m, 1/m), (g_x, g_y),
  // then the cost weights (Q_px, Q_py), (Q_vx, Q_vy), (Q_pz, Q_vz), (Q_roll, Q_pitch),
  // (Q_yaw, Q_wx), (Q_wy, Q_wz), then (R_x, R_y) of legs 0..3
  float2 pk[18];
  // --- gait ---
  uint32_t inc[SBS_MAX_FREQ]; // Q0.32 phase increment per step for each frequency option
  float freq_hz[SBS_MAX_FREQ];
  uint32_t off[4];            // Q0.32 leg offsets
  uint32_t thr;               // stance iff phase < thr ...
  int all_stance;             // ... or always when D_f = 1 (thr = 2^32)
  int n_freq, gait_adapt, elite_preserve, warm_shift;
  // --- spline tables ---
  int H, P, D;
  float W[SBS_MAX_HORIZON][SBS_MAX_KNOTS];   // Gamma_j = sum_p W[j][p] theta[p]  (Catmull-Rom + phantoms)
  float WS[SBS_MAX_KNOTS][SBS_MAX_KNOTS];    // warm shift: mu'[p] = sum_q WS[p][q] mu[q]
  // --- optimiser ---
  int mode;
  int64_t n_elite;
  float var_floor[3];
  int split;                  // latency mode: kSplitTile samples per tile, sampler split over 4 lanes
  int ab;                     // latency mode: 12 producer warps tabulate the stance-leg forces for the 4 integrator warps
  int full_cov;               // f3 (L42): CEM with a full covariance C = L L^T
  int cem_cluster;            // CEM at world = 1: cluster size of the one-launch select + elite path, 0: two kernels
  // throughput-mode MPPI with dynamic tile scheduling (one robot): tiles are taken from a
  // counter and reduced by a fixed tree of fan-in dyn_fan over the tile index, so the result
  // does not depend on which CTA ran which tile
  int dyn;                    // 1: on
  int dyn_levels;             // L: tree levels above the tiles (level L is the root)
  int dyn_fan;                // fan-in: as many records as one merge stages in shared memory (<= 128)
  int dyn_n[kDynMaxLevels + 1];     // nodes per level (dyn_n[0] = n_tiles, dyn_n[L] = 1)
  int dyn_off[kDynMaxLevels + 1];   // record offset of level l in dyn_rec (levels 0..L-1)
  int dyn_coff[kDynMaxLevels + 1];  // arrival counters of level l (1..L) in dyn_cnt
  float* dyn_rec;             // [sum_l dyn_n[l]][part_stride] tile and subtree records
  int* dyn_cnt;               // [0]: next tile, [1]: CTAs done, then the level counters, then dyn_ecnt
  int dyn_ecnt;               // index in dyn_cnt of the emitted top-level records' arrivals (world > 1)
  int model;                  // 1: the constants equal the compiled-in robot model (sbs_robot_model.h)
  float* Lmat;                // [R][D][D] lower Cholesky factor (row-major), full_cov only
  int n_sig_groups;           // multiple Gaussians (L41): sample k uses sig_scale[k mod n_sig_groups]
  float sig_scale[8];
  // --- noise ---
  uint32_t seed_lo, seed_hi;
  uint32_t rk[10][2];         // Philox round keys (seed_lo + r 0x9E3779B9, seed_hi + r 0xBB67AE85)
  uint32_t iter;
  const uint32_t* iter_dev;   // non-null: read the iteration counter from device memory (graph replay) ...
  uint32_t iter_add;          // ... plus this offset (inner iterations of a closed-loop control step)
  int robot_offset;
  // --- sizes / sharding ---
  int R;
  int64_t K_global, k_begin, K_local;
  int n_tiles, n_cta;         // per robot
  int part_stride;             // floats per partial record = kPartHdr + D (tight, 16-byte multiple)
  int part_c_stride;          // 1: CTA partials [R][n_cta]; R: NCCL-gathered rank partials [world][R]
  // --- host path with inline inputs (R = 1): no H2D copy ---
  int inline_in;
  sbs_input in_inline;
  float xref_inline[kInlineRefFloats];
  // --- device buffers ---
  float* mean;                // [R][D]
  float* var;                 // [R][D]
  int* fidx;                  // [R]
  const float* xref;          // [R][H][12]
  const sbs_input* in;        // [R]
  sbs_output* out;            // [R]
  uint32_t* done;             // host path, one robot: mapped flag the finishing CTA sets to done_value after the outputs
  uint32_t done_value;
  float* J;                   // [R][K_local]
  float* part;                // [R][n_cta][part_stride]
  int64_t* elite;             // [R][n_elite]
  int64_t* best;              // [R] global index of rank-1 sample (CEM/Naive)
  int* status;                // [R]
  int* counter;               // [R] CTA arrival counters of the fused rollout tail (re-armed to 0)
  int* ecounter;              // [R] arrival counters of the elite kernel
  float* epart;               // [R][n_eblk][kEPartStride] CEM elite-moment records
  int n_eblk;                 // elite blocks per robot
  float* sdiag;               // [R][8] CEM: J_min, k_best, theta1_best, sum J, n finite (select kernel)
  float* elite_J;             // [R][n_elite] costs of the elites (select kernel)
  float* cand;                // [R][world * n_elite] CEM world > 1: gathered candidate costs
  int ex_stride;              // floats per robot in a rank record (world > 1 exchange)
  float* emit;                // non-null: the fused rollout's last CTA writes the rank record here (MPPI, Naive)
  // --- peer-memory exchange (world > 1 without NCCL): after the last robot's record is
  //     written, the publishing CTA copies [R][ex_stride] into every peer's gather slot
  //     (NVLink stores), fences at system scope and raises the peer's flag [my_rank] ---
  int n_peers;                // 0: no peer publishing
  int my_rank;
  uint32_t flag_value;        // exchange sequence number of this iteration
  int* gcounter;              // arrival counter of the robots' record writers (re-armed to 0)
  float* peer_gather[kMaxWorld];
  uint32_t* peer_flags[kMaxWorld];
};

// closed loop (sbs_loop.cu)
struct LoopArgs {
  float hip[12];
  float h_nom, fall_angle, fall_height;
  const sbs_command* cmd;     // [R] or null (zero command)
  const float* wrench;        // [n_iter][R][6] or null
  int32_t* fallen;            // [R] or null
  float* trace;               // [n_iter][R][SBS_TRACE_FLOATS] or null
  uint32_t* loop;             // null, or device words {iteration counter (Params::iter_dev), counter at call start}
  int n_inner;                // SBS iterations per control step (the advance moves the counter by n_inner)
  int* counter;               // arrival counter (re-armed to 0) of the advance kernel
};
cudaError_t launch_advance(const Params& p, const LoopArgs& a, sbs_input* in, const sbs_output* out, cudaStream_t s);

// launchers (sbs_kernels.cu); return cudaGetLastError()
// mode: SBS_MPPI / SBS_NAIVE (fused: merge + finish in the last CTA; else records only), SBS_CEM (records only)
cudaError_t launch_rollout(const Params& p, int mode, bool fused, cudaStream_t s);
cudaError_t launch_mppi_finalize(const Params& p, cudaStream_t s);
cudaError_t launch_select(const Params& p, cudaStream_t s);
// world > 1 CEM: rank record [8 | K_e J | K_e k] per robot at emit[R][ex_stride]; merge of the gathered records
cudaError_t launch_select_emit(const Params& p, float* emit, cudaStream_t s);
cudaError_t launch_select_merge(const Params& p, cudaStream_t s);
// world > 1 Naive: merge of the gathered rank argmin records + finish
cudaError_t launch_naive_finalize(const Params& p, cudaStream_t s);
cudaError_t launch_elite(const Params& p, cudaStream_t s);
// CEM at world = 1: select + elite moments + finish in one cluster launch (bitwise the
// same results as launch_select + launch_elite) when cem_cluster_fits
cudaError_t launch_cem_cluster(const Params& p, cudaStream_t s);
bool cem_cluster_fits(const Params& p);
int cem_cluster_size(int P, int want);  // the largest resident cluster <= want (16 or 8), 0 if none
cudaError_t launch_debug_samples(const Params& p, int robot, int64_t k0, int64_t n, float* z, float* theta,
                                 int* fidx, cudaStream_t s);
cudaError_t launch_select_raw(const float* J, int64_t K, int64_t K_e, int64_t* idx, cudaStream_t s);
// tests only: the noise recipe on given Philox words [n][4] -> z [n][4]; Philox on given
// counters [n] / keys [n] -> ours [n][2] (plain and round-key forms), cuRAND's [n]
cudaError_t launch_debug_noise(const void* w, int64_t n, void* z, cudaStream_t s);
cudaError_t launch_debug_philox(const void* ctr, const void* key, int64_t n, void* ours, void* curand_out,
                                cudaStream_t s);
int rollout_occupancy(int P, int mode, bool fc = false, bool split = false, bool model = false);
// kernel attributes (dynamic shared memory limits), once per process and P, never inside a capture
cudaError_t prepare_kernels(int P);  // resident CTAs per SM of the rollout kernel

}  // namespace sbs
