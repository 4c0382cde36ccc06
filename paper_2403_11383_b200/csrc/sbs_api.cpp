// sbs_api.cpp -- host runtime behind the C ABI of include/sbs.h.
//
// Owns the device state of one or more SBS controllers (R robots), derives the
// constant tables once at creation (Catmull-Rom weights, warm-shift weights,
// Q0.32 gait increments, inverse inertia), and enqueues one MPC iteration as
// 1 (MPPI, Naive) or 3 (CEM) kernel launches on one stream.  With world > 1 the
// MPPI records of the ranks are exchanged by one NCCL all-gather (or by the
// caller: sbs_step_records / sbs_finish_records).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <string.h>

#include <stdlib.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "sbs_internal.h"
#include "sbs_robot_model.h"

using sbs::Params;

namespace {

// ---- minimal NCCL surface, resolved with dlopen (torch ships libnccl.so.2) ----
typedef struct {
  char internal[128];
} nccl_uid;
typedef void* nccl_comm_t;
typedef int (*PFN_GetUniqueId)(nccl_uid*);
typedef int (*PFN_CommInitRank)(nccl_comm_t*, int, nccl_uid, int);
typedef int (*PFN_AllGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t);
typedef int (*PFN_CommDestroy)(nccl_comm_t);
typedef const char* (*PFN_GetErrorString)(int);
struct Nccl {
  void* h = nullptr;
  PFN_GetUniqueId get_uid = nullptr;
  PFN_CommInitRank init_rank = nullptr;
  PFN_AllGather all_gather = nullptr;
  PFN_CommDestroy destroy = nullptr;
  PFN_GetErrorString err = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    get_uid = (PFN_GetUniqueId)dlsym(h, "ncclGetUniqueId");
    init_rank = (PFN_CommInitRank)dlsym(h, "ncclCommInitRank");
    all_gather = (PFN_AllGather)dlsym(h, "ncclAllGather");
    destroy = (PFN_CommDestroy)dlsym(h, "ncclCommDestroy");
    err = (PFN_GetErrorString)dlsym(h, "ncclGetErrorString");
    return get_uid && init_rank && all_gather && destroy;
  }
};
Nccl g_nccl;
constexpr int kNcclFloat32 = 7;  // ncclFloat32 in nccl.h

thread_local std::string g_create_err;
constexpr int kLoopUnroll = 8;  // control steps per replayed graph of sbs_run_loop

// cuStreamWaitValue32 (driver API, resolved through the runtime): a stream waits in the
// GPU front-end until a 32-bit word reaches a value (GEQ, wrap-around safe)
typedef int (*PFN_WaitValue32)(void* stream, unsigned long long addr, uint32_t value, unsigned int flags);
PFN_WaitValue32 g_wait_fn = nullptr;
int g_wait_value32(cudaStream_t s, const uint32_t* addr, uint32_t value) {
  if (!g_wait_fn) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return -1;
    g_wait_fn = reinterpret_cast<PFN_WaitValue32>(fn);
  }
  return g_wait_fn((void*)s, (unsigned long long)(uintptr_t)addr, value, 0x0 /*CU_STREAM_WAIT_VALUE_GEQ*/);
}

}  // namespace

struct sbs_ctx {
  sbs_config cfg{};
  Params P{};
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  // device-path calls run on the caller's stream: the last one's completion event, so that
  // state getters / setters and the host path order themselves after it
  cudaEvent_t dev_ev = nullptr;
  bool dev_pending = false;
  // device buffers
  float* d_mean = nullptr;
  float* d_var = nullptr;
  int* d_fidx = nullptr;
  float* d_xref = nullptr;
  float* d_J = nullptr;
  float* d_part = nullptr;
  float* d_gather = nullptr;  // [world][R][ex_stride] (world > 1), inside d_xbuf
  char* d_xbuf = nullptr;      // world > 1: exchange buffer [gather 0 | gather 1 | flags[kMaxWorld] uint32]
  size_t xgather_bytes = 0;    // (aligned) bytes of one gather buffer; peers alternate between the two
  size_t xflags_off = 0;
  std::vector<char*> peer_base;  // every rank's exchange buffer, as addressable from this device
  uint32_t* d_xflags = nullptr;  // flags[j] = last exchange sequence number published by rank j
  bool peer = false;             // rank records exchanged over peer memory (sbs_peer_connect)
  uint32_t xseq = 0;             // exchange sequence number (identical on every rank)
  std::vector<void*> ipc_opened; // peer buffers opened with cudaIpcOpenMemHandle
  float* d_eJ = nullptr;      // [R][K_e] elite costs
  float* d_L = nullptr;       // [R][D][D] Cholesky factors (full_cov)
  float* d_cand = nullptr;    // [R][world][K_e] CEM world > 1 candidates
  int64_t* d_elite = nullptr;
  int64_t* d_best = nullptr;
  int* d_status = nullptr;
  int* d_counter = nullptr;
  float* d_epart = nullptr;
  float* d_sdiag = nullptr;
  float* d_dyn_rec = nullptr;  // dynamic tile scheduling: tile and subtree records
  int* d_dyn_cnt = nullptr;    // ... its counters
  int dyn_recs = 0, dyn_cnts = 0;
  sbs_input* d_in = nullptr;
  sbs_output* d_out = nullptr;
  // host path staging: one pinned block [iter | R inputs | R x H x 12 reference], one H2D per step
  char* h_blk = nullptr;
  char* d_blk = nullptr;
  size_t blk_in_off = 0, blk_ref_off = 0, blk_bytes = 0;
  sbs_input* h_in = nullptr;   // = h_blk + blk_in_off
  float* h_xref = nullptr;     // = h_blk + blk_ref_off
  sbs_output* h_out = nullptr; // pinned, mapped: the host path's kernels write the outputs here directly
  sbs_output* h_out_dev = nullptr;  // device address of h_out (null: copied back by a D2H node)
  cudaEvent_t blk_ev = nullptr;  // last H2D of h_blk (the host rewrites it only after this completed)
  bool blk_busy = true;          // blk_ev recorded since the last wait on it
  bool ref_dirty = false;
  uint32_t* h_done = nullptr;    // one-robot host path: mapped completion flag (after h_out), its device address,
  uint32_t* d_done = nullptr;    // and the value of the last step
  uint32_t done_seq = 0;
  cudaGraphExec_t graph = nullptr;
  // closed loop (sbs_run_loop): device words {iteration counter, counter at call start, arrival counter},
  // pinned staging of the start value, and one captured iteration keyed by its arguments
  uint32_t* d_loopw = nullptr;
  uint32_t* h_loopw = nullptr;
  cudaGraphExec_t loop_graph = nullptr;    // one control step
  cudaGraphExec_t loop_graph_u = nullptr;  // kLoopUnroll control steps
  std::vector<char> loop_key;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<char> ref_set;
  uint32_t iter = 0;
  std::string err;
  // profiling
  bool profile = false;
  struct Pending {
    int kernel;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> free_events;
  double kt[SBS_NKERNELS] = {};
  int64_t kl[SBS_NKERNELS] = {};
  // nccl
  nccl_comm_t comm = nullptr;
  bool external = false;  // world > 1 with an all-zero nccl_id: the caller exchanges the records
};

namespace {
// a device-path call enqueued work on the caller's stream s
cudaError_t note_device_work(sbs_ctx* c, cudaStream_t s) {
  c->dev_pending = true;
  return cudaEventRecord(c->dev_ev, s);
}
// the context's own stream and the last device-path work have completed (getters / setters:
// a checkpoint is never torn by a step still running on a caller stream)
cudaError_t sync_ctx(sbs_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && c->dev_pending) {
    e = cudaEventSynchronize(c->dev_ev);
    if (e == cudaSuccess) c->dev_pending = false;
  }
  return e;
}

// the pinned block may be rewritten once its last upload (blk_ev) has completed;
// a host flag skips the driver call when nothing was recorded since the last wait
cudaError_t blk_wait(sbs_ctx* c) {
  if (!c->blk_busy) return cudaSuccess;
  const cudaError_t e = cudaEventSynchronize(c->blk_ev);
  if (e == cudaSuccess) c->blk_busy = false;
  return e;
}
cudaError_t blk_record(sbs_ctx* c, cudaStream_t s) {
  c->blk_busy = true;
  return cudaEventRecord(c->blk_ev, s);
}
}  // namespace


namespace {

int fail(sbs_ctx* c, int st, const std::string& msg) {
  if (c) c->err = msg;
  else g_create_err = msg;
  return st;
}

int cuda_fail(sbs_ctx* c, cudaError_t e, const char* where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  return fail(c, e == cudaErrorMemoryAllocation ? SBS_ERR_OOM : SBS_ERR_CUDA, m);
}

#define CK(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, #call); \
  } while (0)

// the context's model / cost constants equal the compiled-in robot model bit for bit
// (then the rollout may take them as immediate operands: sbs_robot_model.h)
bool same_bits(float a, float b) { return memcmp(&a, &b, sizeof a) == 0; }
bool model_matches(const sbs::Params& P) {
  namespace m = sbs::model;
  if (P.P != m::kKnots || !P.diag_inertia || P.full_cov) return false;
  bool ok = same_bits(P.dt, m::kDt) && same_bits(P.inv_mass, m::kInvMass) && same_bits(P.g[0], 0.0f) &&
            same_bits(P.g[1], 0.0f) && same_bits(P.g[2], m::kGz) && same_bits(P.mu, m::kMu) &&
            same_bits(P.fz_min, m::kFzMin) && same_bits(P.fz_max, m::kFzMax) && same_bits(P.w_fc, m::kWfc);
  ok = ok && same_bits(P.I[0], m::kI0) && same_bits(P.I[4], m::kI1) && same_bits(P.I[8], m::kI2);
  ok = ok && same_bits(P.Iinv[0], m::kIinv0) && same_bits(P.Iinv[4], m::kIinv1) && same_bits(P.Iinv[8], m::kIinv2);
  ok = ok && same_bits(P.gyr[0], m::kGyr0) && same_bits(P.gyr[1], m::kGyr1) && same_bits(P.gyr[2], m::kGyr2);
  for (int i = 0; i < 12; ++i) ok = ok && same_bits(P.Q[i], m::Q(i)) && same_bits(P.Rw[i], m::kR);
  for (int n = 0; n <= 4; ++n) ok = ok && same_bits(P.urz[n], m::urz(n));
  return ok;
}

bool finite_all(const float* v, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// Uniform Catmull-Rom weights on the P real knots for the evaluation point
// tau = num/den (knot units), phantom end knots by linear extrapolation (L7).
void catmull_rom_row(int P, int64_t num, int64_t den, double* w /*[P]*/) {
  for (int q = 0; q < P; ++q) w[q] = 0.0;
  int64_t s = num / den;
  double u = (double)(num % den) / (double)den;
  if (s >= P - 1) {
    s = P - 2;
    u = 1.0;
  }
  const double u2 = u * u, u3 = u2 * u;
  const double c[4] = {0.5 * (-u3 + 2 * u2 - u), 0.5 * (3 * u3 - 5 * u2 + 2), 0.5 * (-3 * u3 + 4 * u2 + u),
                       0.5 * (u3 - u2)};
  for (int t = 0; t < 4; ++t) {
    const int64_t idx = s - 1 + t;
    if (idx < 0) {  // phantom k[-1] = 2 k[0] - k[1]
      w[0] += 2.0 * c[t];
      w[1] -= c[t];
    } else if (idx > P - 1) {  // phantom k[P] = 2 k[P-1] - k[P-2]
      w[P - 1] += 2.0 * c[t];
      w[P - 2] -= c[t];
    } else {
      w[idx] += c[t];
    }
  }
}

uint32_t q32_inc(double f, double dt) { return (uint32_t)(uint64_t)llround((f * dt) * 4294967296.0); }

int validate(const sbs_config* c, std::string& why) {
  auto bad = [&](const char* m) {
    why = m;
    return SBS_ERR_INVALID_ARG;
  };
  if (!(c->mass > 0)) return bad("mass must be > 0");
  const float* I = c->inertia;
  if (!finite_all(I, 9)) return bad("inertia not finite");
  if (I[1] != I[3] || I[2] != I[6] || I[5] != I[7]) return bad("inertia not symmetric");
  const double d1 = I[0], d2 = (double)I[0] * I[4] - (double)I[1] * I[3];
  const double d3 = I[0] * ((double)I[4] * I[8] - (double)I[5] * I[7]) - I[1] * ((double)I[3] * I[8] - (double)I[5] * I[6]) +
                    I[2] * ((double)I[3] * I[7] - (double)I[4] * I[6]);
  if (!(d1 > 0 && d2 > 0 && d3 > 0)) return bad("inertia not positive definite");
  if (!finite_all(c->gravity, 3) || !(c->gravity[2] < 0)) return bad("gravity[2] must be < 0");
  if (!(c->mu > 0)) return bad("mu must be > 0");
  if (!(c->fz_min >= 0 && c->fz_min < c->fz_max)) return bad("need 0 <= fz_min < fz_max");
  if (c->horizon < 1 || c->horizon > SBS_MAX_HORIZON) return bad("horizon out of range");
  if (c->knots < 2 || c->knots > SBS_MAX_KNOTS) return bad("knots out of range");
  if (!(c->dt > 0)) return bad("dt must be > 0");
  if (!(c->duty_factor > 0 && c->duty_factor <= 1)) return bad("duty_factor must be in (0, 1]");
  for (int i = 0; i < 4; ++i)
    if (!(c->phase_offset[i] >= 0 && c->phase_offset[i] < 1)) return bad("phase_offset must be in [0, 1)");
  if (c->n_freq < 1 || c->n_freq > SBS_MAX_FREQ) return bad("n_freq out of range");
  for (int i = 0; i < c->n_freq; ++i) {
    if (!(c->freq_hz[i] > 0)) return bad("freq_hz must be > 0");
    if (i > 0 && !(c->freq_hz[i] > c->freq_hz[i - 1])) return bad("freq_hz must be strictly increasing");
  }
  for (int i = 0; i < 12; ++i)
    if (!(c->Q[i] >= 0) || !(c->R[i] >= 0)) return bad("Q and R must be >= 0");
  if (!(c->rho >= 0) || !(c->w_fc >= 0) || !std::isfinite(c->f_nominal)) return bad("bad rho / w_fc / f_nominal");
  if (c->mode < SBS_MPPI || c->mode > SBS_NAIVE) return bad("bad mode");
  // the finite / diverged counts ride in binary32 record fields (exact below 2^24)
  if (c->n_samples < 1 || c->n_samples > (1LL << 24)) return bad("n_samples out of range (1 .. 2^24)");
  if (c->mode == SBS_CEM && (c->n_elite < 1 || c->n_elite > c->n_samples)) return bad("need 1 <= n_elite <= n_samples");
  if (!(c->lambda > 0)) return bad("lambda must be > 0");
  for (int a = 0; a < 3; ++a)
    if (!(c->sigma[a] > 0)) return bad("sigma must be > 0");
  if (!(c->sigma_min_frac >= 0)) return bad("sigma_min_frac must be >= 0");
  if (c->n_sigma_groups < 0 || c->n_sigma_groups > 8) return bad("n_sigma_groups must be in [0, 8]");
  if (c->full_cov && c->mode != SBS_CEM) return bad("full_cov is a CEM option");
  if (c->full_cov && c->n_sigma_groups > 1) return bad("full_cov does not combine with multiple sigma groups");
  for (int g = 0; g < c->n_sigma_groups; ++g)
    if (!(c->sigma_scale[g] >= 0) || !std::isfinite(c->sigma_scale[g])) return bad("sigma_scale must be finite, >= 0");
  if (c->n_robots < 1) return bad("n_robots must be >= 1");
  if (c->robot_offset < 0) return bad("robot_offset must be >= 0");
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return bad("bad rank / world");
  if (c->world > 1 && c->n_samples < c->world) return bad("n_samples < world");
  if (c->world > 1 && c->mode == SBS_CEM && c->n_samples / c->world < c->n_elite)
    return bad("CEM with world > 1 needs n_elite <= n_samples / world (every rank offers K_e candidates)");
  return SBS_OK;
}

cudaEvent_t take_event(sbs_ctx* c) {
  if (!c->free_events.empty()) {
    cudaEvent_t e = c->free_events.back();
    c->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// launch wrapper with optional per-kernel event timing
template <class F>
cudaError_t timed(sbs_ctx* c, int kernel, cudaStream_t s, F&& launch) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->profile) {
    a = take_event(c);
    b = take_event(c);
    cudaEventRecord(a, s);
  }
  cudaError_t e = launch();
  if (c->profile) {
    cudaEventRecord(b, s);
    c->pending.push_back({kernel, a, b});
  }
  return e;
}

// sample sharding (world > 1), part 1: rollouts of this rank's slice and its
// record per robot at dst[R][ex_stride]:
//   MPPI  [beta_g, k, f, S, S2, sum J, n finite, 0 | V[D]]   (weights relative to beta_g)
//   Naive [J_min, k, f, 0, 0, sum J, n finite, 0]
//   CEM   [J_min, k, f, 0, 0, sum J, n finite, 0 | J[K_e] | k[K_e]]  (local K_e smallest, index order)
int enqueue_records(sbs_ctx* c, cudaStream_t s, float* dst) {
  Params& P = c->P;
  P.iter = c->iter;
  const int mode = c->cfg.mode;
  if (mode == SBS_CEM) {
    CK(timed(c, SBS_KERNEL_ROLLOUT, s, [&] { return sbs::launch_rollout(P, mode, false, s); }));
    CK(timed(c, SBS_KERNEL_SELECT, s, [&] { return sbs::launch_select_emit(P, dst, s); }));
    return SBS_OK;
  }
  // MPPI / Naive: one launch, the last CTA of each robot emits the rank record
  P.emit = dst;
  const cudaError_t e = timed(c, SBS_KERNEL_ROLLOUT, s, [&] { return sbs::launch_rollout(P, mode, true, s); });
  P.emit = nullptr;
  CK(e);
  return SBS_OK;
}

// part 2: merge the `world` ranks' records ([world][R][ex_stride], rank order) and finish
int enqueue_finish(sbs_ctx* c, cudaStream_t s, const float* recs) {
  Params F = c->P;
  F.iter = c->iter;
  F.part = const_cast<float*>(recs);
  F.n_cta = c->cfg.world;
  F.part_c_stride = F.R;
  F.part_stride = F.ex_stride;
  if (c->cfg.mode == SBS_MPPI) {  // every rank's records: the top tree nodes it emitted, in rank order
    F.n_cta = c->cfg.world * (F.ex_stride / c->P.part_stride);
    F.part_stride = c->P.part_stride;
  }
  const int mode = c->cfg.mode;
  if (mode == SBS_MPPI) CK(timed(c, SBS_KERNEL_REDUCE, s, [&] { return sbs::launch_mppi_finalize(F, s); }));
  else if (mode == SBS_NAIVE) CK(timed(c, SBS_KERNEL_REDUCE, s, [&] { return sbs::launch_naive_finalize(F, s); }));
  else {
    CK(timed(c, SBS_KERNEL_SELECT, s, [&] { return sbs::launch_select_merge(F, s); }));
    CK(timed(c, SBS_KERNEL_ELITE, s, [&] { return sbs::launch_elite(F, s); }));
  }
  return SBS_OK;
}

// enqueue one iteration on stream s with inputs c->P.in and outputs c->P.out
int enqueue_step(sbs_ctx* c, cudaStream_t s) {
  Params& P = c->P;
  P.iter = c->iter;
  const int mode = c->cfg.mode;
  if (c->cfg.world > 1) {  // rank record -> exchange -> merge in rank order
    const size_t n = (size_t)P.R * P.ex_stride;
    float* mine = c->d_gather + (size_t)c->cfg.rank * n;
    if (c->peer) {
      // the publishing CTA stores this rank's records into every peer's gather buffer and
      // raises the peer's flag; this stream waits (front-end, no SM) for the peers' flags
      // (two gather buffers alternate with the sequence number: a rank publishing step t + 1
      // cannot overwrite what a slower peer still reads for step t)
      // (the sequence number is committed only once the publishing launch is enqueued: an
      // early return leaves it -- and this rank's state -- unchanged)
      const uint32_t seq = c->xseq + 1;
      const size_t par = (seq & 1u) * c->xgather_bytes;
      float* gat = reinterpret_cast<float*>(c->d_xbuf + par);
      P.n_peers = c->cfg.world;
      P.my_rank = c->cfg.rank;
      P.flag_value = seq;
      for (int j = 0; j < c->cfg.world; ++j) P.peer_gather[j] = reinterpret_cast<float*>(c->peer_base[j] + par);
      int rc = enqueue_records(c, s, gat + (size_t)c->cfg.rank * n);
      P.n_peers = 0;
      if (rc != SBS_OK) return rc;
      c->xseq = seq;
      for (int j = 0; j < c->cfg.world; ++j) {
        if (j == c->cfg.rank) continue;
        const int r2 = g_wait_value32(s, c->d_xflags + j, seq);
        if (r2 != 0) return fail(c, SBS_ERR_CUDA, "cuStreamWaitValue32 failed");
      }
      return enqueue_finish(c, s, gat);
    }
    if (c->external) return fail(c, SBS_ERR_STATE, "external exchange: use sbs_step_records / sbs_finish_records");
    int rc = enqueue_records(c, s, mine);
    if (rc != SBS_OK) return rc;
    rc = g_nccl.all_gather(mine, c->d_gather, n, kNcclFloat32, c->comm, s);
    if (rc != 0) return fail(c, SBS_ERR_NCCL, std::string("ncclAllGather: ") + (g_nccl.err ? g_nccl.err(rc) : "?"));
    return enqueue_finish(c, s, c->d_gather);
  }
  CK(timed(c, SBS_KERNEL_ROLLOUT, s, [&] { return sbs::launch_rollout(P, mode, true, s); }));
  if (mode == SBS_CEM && P.cem_cluster) {
    CK(timed(c, SBS_KERNEL_SELECT, s, [&] { return sbs::launch_cem_cluster(P, s); }));
  } else if (mode == SBS_CEM) {
    CK(timed(c, SBS_KERNEL_SELECT, s, [&] { return sbs::launch_select(P, s); }));
    CK(timed(c, SBS_KERNEL_ELITE, s, [&] { return sbs::launch_elite(P, s); }));
  }
  return SBS_OK;
}

}  // namespace

extern "C" {

int sbs_version(void) { return SBS_VERSION; }
uint64_t sbs_sizeof_config(void) { return sizeof(sbs_config); }
uint64_t sbs_sizeof_input(void) { return sizeof(sbs_input); }
uint64_t sbs_sizeof_output(void) { return sizeof(sbs_output); }

const char* sbs_status_str(int st) {
  switch (st) {
    case SBS_OK: return "SBS_OK";
    case SBS_WARN_ALL_DIVERGED: return "SBS_WARN_ALL_DIVERGED";
    case SBS_ERR_INVALID_ARG: return "SBS_ERR_INVALID_ARG";
    case SBS_ERR_SINGULAR: return "SBS_ERR_SINGULAR";
    case SBS_ERR_NONFINITE: return "SBS_ERR_NONFINITE";
    case SBS_ERR_STATE: return "SBS_ERR_STATE";
    case SBS_ERR_CUDA: return "SBS_ERR_CUDA";
    case SBS_ERR_NCCL: return "SBS_ERR_NCCL";
    case SBS_ERR_OOM: return "SBS_ERR_OOM";
    default: return "SBS_UNKNOWN_STATUS";
  }
}

const char* sbs_last_error(const sbs_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int sbs_nccl_unique_id(uint8_t id[128]) {
  if (!id) return SBS_ERR_INVALID_ARG;
  if (!g_nccl.load()) return fail(nullptr, SBS_ERR_NCCL, "libnccl.so.2 not found");
  nccl_uid u;
  int rc = g_nccl.get_uid(&u);
  if (rc != 0) return fail(nullptr, SBS_ERR_NCCL, "ncclGetUniqueId failed");
  memcpy(id, u.internal, 128);
  return SBS_OK;
}

void sbs_destroy(sbs_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm && g_nccl.destroy) g_nccl.destroy(c->comm);
  for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
  for (void* p : {(void*)c->d_mean, (void*)c->d_var, (void*)c->d_fidx, (void*)c->d_J,
                  (void*)c->d_part, (void*)c->d_xbuf, (void*)c->d_elite, (void*)c->d_best, (void*)c->d_status, (void*)c->d_counter, (void*)c->d_epart, (void*)c->d_sdiag, (void*)c->d_eJ, (void*)c->d_cand, (void*)c->d_L,
                  (void*)c->d_out, (void*)c->d_dyn_rec, (void*)c->d_dyn_cnt})
    if (p) cudaFree(p);
  if (c->h_out) cudaFreeHost(c->h_out);  // (h_in and h_xref point into h_blk)
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->loop_graph) cudaGraphExecDestroy(c->loop_graph);
  if (c->loop_graph_u) cudaGraphExecDestroy(c->loop_graph_u);
  if (c->d_loopw) cudaFree(c->d_loopw);
  if (c->h_loopw) cudaFreeHost(c->h_loopw);
  if (c->h_blk) cudaFreeHost(c->h_blk);
  if (c->d_blk) cudaFree(c->d_blk);
  if (c->blk_ev) cudaEventDestroy(c->blk_ev);
  for (auto& pd : c->pending) {
    cudaEventDestroy(pd.a);
    cudaEventDestroy(pd.b);
  }
  for (auto e : c->free_events) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->dev_ev) cudaEventDestroy(c->dev_ev);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  (void)cudaGetLastError();  // teardown errors (e.g. a context that failed half-way) must not leak into later launches
}

int sbs_create(const sbs_config* cfg, sbs_ctx** out) {
  if (!cfg || !out) return fail(nullptr, SBS_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  std::string why;
  if (validate(cfg, why) != SBS_OK) return fail(nullptr, SBS_ERR_INVALID_ARG, why);
  sbs_ctx* c = new sbs_ctx();
  c->cfg = *cfg;
  auto bail = [&](int st) {
    g_create_err = c->err;
    sbs_destroy(c);
    return st;
  };
  int rc;
#define CKC(call)                                 \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) {                      \
      rc = cuda_fail(c, e_, #call);               \
      return bail(rc);                            \
    }                                             \
  } while (0)
  CKC(cudaSetDevice(cfg->device));
  CKC(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, cfg->device));
  CKC(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CKC(sbs::prepare_kernels(cfg->knots));
  CKC(cudaEventCreateWithFlags(&c->dev_ev, cudaEventDisableTiming));
  CKC(cudaEventCreate(&c->ev0));
  CKC(cudaEventCreate(&c->ev1));

  Params& P = c->P;
  const int H = cfg->horizon, Pk = cfg->knots, D = 12 * Pk, R = cfg->n_robots;
  // ---- model and cost constants ----
  P.inv_mass = (float)(1.0 / (double)cfg->mass);
  for (int a = 0; a < 3; ++a) P.g[a] = cfg->gravity[a];
  {
    const double* dummy = nullptr;
    (void)dummy;
    double A[9];
    for (int i = 0; i < 9; ++i) A[i] = cfg->inertia[i];
    const double det = A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
                       A[2] * (A[3] * A[7] - A[4] * A[6]);
    const double inv[9] = {(A[4] * A[8] - A[5] * A[7]) / det, (A[2] * A[7] - A[1] * A[8]) / det,
                           (A[1] * A[5] - A[2] * A[4]) / det, (A[5] * A[6] - A[3] * A[8]) / det,
                           (A[0] * A[8] - A[2] * A[6]) / det, (A[2] * A[3] - A[0] * A[5]) / det,
                           (A[3] * A[7] - A[4] * A[6]) / det, (A[1] * A[6] - A[0] * A[7]) / det,
                           (A[0] * A[4] - A[1] * A[3]) / det};
    for (int i = 0; i < 9; ++i) {
      P.I[i] = cfg->inertia[i];
      P.Iinv[i] = (float)inv[i];
    }
    P.diag_inertia = (A[1] == 0 && A[2] == 0 && A[5] == 0) ? 1 : 0;
    P.gyr[0] = P.Iinv[0] * (P.I[4] - P.I[8]);
    P.gyr[1] = P.Iinv[4] * (P.I[8] - P.I[0]);
    P.gyr[2] = P.Iinv[8] * (P.I[0] - P.I[4]);
  }
  P.mu = cfg->mu;
  P.fz_min = cfg->fz_min;
  P.fz_max = cfg->fz_max;
  P.dt = cfg->dt;
  P.duty = cfg->duty_factor;
  for (int a = 0; a < 12; ++a) {
    P.Q[a] = cfg->Q[a];
    P.Rw[a] = cfg->R[a];
  }
  P.rho = cfg->rho;
  P.f_nominal = cfg->f_nominal;
  P.w_fc = cfg->w_fc;
  P.inv_lambda = (float)(1.0 / (double)cfg->lambda);
  for (int n = 0; n <= 4; ++n) P.urz[n] = (float)(-(double)cfg->mass * (double)cfg->gravity[2] / (double)std::max(1, n));
  {  // packed operand pairs (Params::pk), binary32 as the kernel would form them
    const float dt = cfg->dt, hdt = 0.5f * dt, dt6 = dt * (1.0f / 6.0f), dt2h = 0.5f * dt * dt,
                dt2q = 0.25f * dt * dt;
    const float v[6] = {dt, hdt, dt6, 2.0f, dt2h, dt2q};
    for (int i = 0; i < 6; ++i) P.pk[i] = make_float2(v[i], v[i]);
    P.pk[6] = make_float2(P.inv_mass, P.inv_mass);
    P.pk[7] = make_float2(cfg->gravity[0], cfg->gravity[1]);
    const int qi[6][2] = {{0, 1}, {3, 4}, {2, 5}, {6, 7}, {8, 9}, {10, 11}};
    for (int i = 0; i < 6; ++i) P.pk[8 + i] = make_float2(cfg->Q[qi[i][0]], cfg->Q[qi[i][1]]);
    for (int i = 0; i < 4; ++i) P.pk[14 + i] = make_float2(cfg->R[3 * i], cfg->R[3 * i + 1]);
  }
  // ---- gait: Q0.32 tables (L22) ----
  for (int f = 0; f < SBS_MAX_FREQ; ++f) {
    P.inc[f] = f < cfg->n_freq ? q32_inc((double)cfg->freq_hz[f], (double)cfg->dt) : 0u;
    P.freq_hz[f] = f < cfg->n_freq ? cfg->freq_hz[f] : 0.f;
  }
  for (int i = 0; i < 4; ++i) P.off[i] = (uint32_t)(uint64_t)llround((double)cfg->phase_offset[i] * 4294967296.0);
  {
    const uint64_t thr = (uint64_t)llround((double)cfg->duty_factor * 4294967296.0);
    P.all_stance = thr >= 4294967296ull ? 1 : 0;
    P.thr = (uint32_t)std::min<uint64_t>(thr, 0xFFFFFFFFull);
  }
  P.n_freq = cfg->n_freq;
  P.gait_adapt = cfg->gait_adapt ? 1 : 0;
  P.elite_preserve = cfg->elite_preserve ? 1 : 0;
  P.warm_shift = cfg->warm_shift ? 1 : 0;
  // ---- spline tables (L7, L20) ----
  P.H = H;
  P.P = Pk;
  P.D = D;
  double w[SBS_MAX_KNOTS];
  for (int j = 0; j < H; ++j) {
    catmull_rom_row(Pk, (int64_t)j * (Pk - 1), H, w);
    for (int q = 0; q < Pk; ++q) P.W[j][q] = (float)w[q];
  }
  for (int p = 0; p < Pk; ++p) {
    catmull_rom_row(Pk, (int64_t)p * H + (Pk - 1), H, w);
    for (int q = 0; q < Pk; ++q) P.WS[p][q] = (float)w[q];
  }
  // ---- optimiser ----
  P.mode = cfg->mode;
  P.n_elite = cfg->mode == SBS_NAIVE ? 1 : (cfg->mode == SBS_CEM ? cfg->n_elite : 0);
  for (int a = 0; a < 3; ++a) {
    const double s = (double)cfg->sigma_min_frac * (double)cfg->sigma[a];
    P.var_floor[a] = (float)(s * s);
  }
  P.n_sig_groups = cfg->n_sigma_groups > 1 ? cfg->n_sigma_groups : 1;
  for (int g = 0; g < 8; ++g) P.sig_scale[g] = g < cfg->n_sigma_groups ? cfg->sigma_scale[g] : 1.0f;
  P.seed_lo = (uint32_t)(cfg->seed & 0xFFFFFFFFull);
  P.seed_hi = (uint32_t)(cfg->seed >> 32);
  for (int r = 0; r < 10; ++r) {
    P.rk[r][0] = P.seed_lo + (uint32_t)r * 0x9E3779B9u;
    P.rk[r][1] = P.seed_hi + (uint32_t)r * 0xBB67AE85u;
  }
  P.robot_offset = cfg->robot_offset;
  // ---- compiled-in robot model (sbs_robot_model.h): every constant bit-identical ----
  P.model = model_matches(P) ? 1 : 0;
  if (const char* e = getenv("SBS_MODEL")) P.model = P.model && atoi(e) != 0;  // experiments / tests: SBS_MODEL=0 disables
  // ---- sharding and launch geometry ----
  P.R = R;
  P.K_global = cfg->n_samples;
  P.k_begin = cfg->n_samples * cfg->rank / cfg->world;
  P.K_local = cfg->n_samples * (cfg->rank + 1) / cfg->world - P.k_begin;
  {
    // latency mode when every 128-sample tile of every robot fits one resident wave of
    // 4 x 128-thread CTAs: the sampler is spread over 4 lanes per sample (shorter
    // per-sample dependent chain; the machine is mostly idle at these sizes anyway)
    P.n_tiles = (int)((P.K_local + sbs::kBlock - 1) / sbs::kBlock);
    const int occ_s = sbs::rollout_occupancy(Pk, cfg->mode, false, true);
    bool split = !cfg->full_cov && (int64_t)R * P.n_tiles <= (int64_t)occ_s * c->sm_count;
    if (const char* e = getenv("SBS_SPLIT")) split = split && atoi(e) != 0;  // experiments: SBS_SPLIT=0 disables
    P.split = split ? 1 : 0;
    // producer / integrator warps (latency mode) when the stance-leg table fits
    bool ab = split && sbs::split_smem_bytes(Pk, cfg->mode == SBS_MPPI, P.H, true) <= sbs::kSplitSmemMax;
    if (const char* e = getenv("SBS_AB")) ab = ab && atoi(e) != 0;  // experiments: SBS_AB=0 disables
    P.ab = ab ? 1 : 0;
    const int occ = sbs::rollout_occupancy(Pk, cfg->mode, cfg->full_cov != 0, split, P.model != 0);
    const int64_t slots = (int64_t)occ * c->sm_count;
    P.n_cta = (int)std::max<int64_t>(1, std::min<int64_t>(P.n_tiles, slots / R));
  }
  P.part_c_stride = 1;
  P.part_stride = sbs::kPartHdr + D;
  // throughput-mode MPPI for one robot with more tiles than CTAs: dynamic tile scheduling
  // (the CTAs sharing an SM do not progress at the same rate, so a static tile split ends
  // with SMs running one or two CTAs; SBS_DYN=0 keeps the static split, for tests / A/B).
  // The tile records are reduced by a tree of fan-in 64 over the tile index.  With world > 1
  // and this rank's tiles made of whole nodes of the level just below the global tree's
  // root, the rank emits those nodes' records instead of merging them, and the rank-order
  // merge after the exchange is the global root's merge: the result does not depend on
  // the number of GPUs.  (One tile per CTA keeps the static split: measured 45.7 vs 53.5 us at
  // K = 2^16; at 1.73 tiles per CTA, K = 2^17, dynamic tiles 59.6 vs 67.7 us.)
  P.dyn = 0;
  if (cfg->mode == SBS_MPPI && R == 1 && !P.split && !cfg->full_cov && P.n_tiles > P.n_cta) {
    const char* e = getenv("SBS_DYN");
    P.dyn = (!e || atoi(e) != 0) ? 1 : 0;
  }
  int emit_nodes = 1;  // MPPI rank records per robot in the world > 1 exchange
  if (P.dyn) {
    // fan-in 64 (measured against 32 and 122, the most one merge stages in the rollout's
    // reduction buffer); SBS_DYN_FAN overrides (experiments)
    P.dyn_fan = 64;
    if (const char* e = getenv("SBS_DYN_FAN")) P.dyn_fan = std::max(2, atoi(e));
    P.dyn_fan = std::min(P.dyn_fan, std::min(128, (D + 4) * (sbs::kBlock + 4) / (int)P.part_stride));
    // the global tree's depth, and the node size (samples) of its level below the root
    int Lg = 0;
    int64_t node = sbs::kBlock;
    for (int64_t n = (cfg->n_samples + sbs::kBlock - 1) / sbs::kBlock; n > 1; n = (n + P.dyn_fan - 1) / P.dyn_fan) {
      ++Lg;
      if (n > P.dyn_fan) node *= P.dyn_fan;
    }
    const bool aligned = cfg->world > 1 && Lg >= 2 && P.k_begin % node == 0 && P.K_local % node == 0;
    int n = P.n_tiles, L = 0, recs = 0, cnts = 2;
    P.dyn_n[0] = n;
    while (n > 1 && !(aligned && L == Lg - 1)) {
      P.dyn_off[L] = recs;
      recs += n;
      n = (n + P.dyn_fan - 1) / P.dyn_fan;
      ++L;
      if (L > sbs::kDynMaxLevels) return bail(SBS_ERR_INVALID_ARG);
      P.dyn_n[L] = n;
      P.dyn_coff[L] = cnts;
      cnts += n;
    }
    P.dyn_levels = L;
    P.dyn_ecnt = cnts++;  // arrivals of the emitted top-level records
    emit_nodes = n;
    c->dyn_recs = recs;
    c->dyn_cnts = cnts;
  }
  // rank record of the world > 1 exchange (16-byte multiple)
  if (cfg->mode == SBS_MPPI) P.ex_stride = emit_nodes * P.part_stride;
  else if (cfg->mode == SBS_NAIVE) P.ex_stride = sbs::kPartHdr;
  else P.ex_stride = (int)((sbs::kPartHdr + 2 * cfg->n_elite + 3) / 4 * 4);
  // ---- device buffers ----
  const size_t RD = (size_t)R * D;
  CKC(cudaMalloc(&c->d_mean, RD * sizeof(float)));
  CKC(cudaMalloc(&c->d_var, RD * sizeof(float)));
  CKC(cudaMalloc(&c->d_fidx, R * sizeof(int)));
  c->blk_in_off = 16;
  c->blk_ref_off = c->blk_in_off + (size_t)R * sizeof(sbs_input);
  c->blk_bytes = c->blk_ref_off + (size_t)R * H * 12 * sizeof(float);
  CKC(cudaMalloc(&c->d_blk, c->blk_bytes));
  CKC(cudaMemset(c->d_blk, 0, c->blk_bytes));
  CKC(cudaMallocHost(&c->h_blk, c->blk_bytes));
  memset(c->h_blk, 0, c->blk_bytes);
  c->h_in = reinterpret_cast<sbs_input*>(c->h_blk + c->blk_in_off);
  c->h_xref = reinterpret_cast<float*>(c->h_blk + c->blk_ref_off);
  c->d_in = reinterpret_cast<sbs_input*>(c->d_blk + c->blk_in_off);
  c->d_xref = reinterpret_cast<float*>(c->d_blk + c->blk_ref_off);
  CKC(cudaEventCreateWithFlags(&c->blk_ev, cudaEventDisableTiming));
  CKC(blk_record(c, c->stream));
  CKC(cudaMalloc(&c->d_J, (size_t)R * P.K_local * sizeof(float)));
  CKC(cudaMalloc(&c->d_part, (size_t)R * P.n_cta * P.part_stride * sizeof(float)));
  if (cfg->world > 1) {
    const size_t gbytes = (size_t)cfg->world * R * P.ex_stride * sizeof(float);
    c->xgather_bytes = (gbytes + 255) / 256 * 256;
    c->xflags_off = 2 * c->xgather_bytes;
    CKC(cudaMalloc(&c->d_xbuf, c->xflags_off + sbs::kMaxWorld * sizeof(uint32_t)));  // (2 gathers + flags)
    CKC(cudaMemset(c->d_xbuf, 0, c->xflags_off + sbs::kMaxWorld * sizeof(uint32_t)));
    c->d_gather = reinterpret_cast<float*>(c->d_xbuf);
    c->d_xflags = reinterpret_cast<uint32_t*>(c->d_xbuf + c->xflags_off);
  }
  if (P.n_elite > 0) {
    CKC(cudaMalloc(&c->d_elite, (size_t)R * P.n_elite * sizeof(int64_t)));
    CKC(cudaMalloc(&c->d_eJ, (size_t)R * P.n_elite * sizeof(float)));
  }
  if (cfg->mode == SBS_CEM && cfg->world > 1)
    CKC(cudaMalloc(&c->d_cand, (size_t)R * cfg->world * P.n_elite * sizeof(float)));
  CKC(cudaMalloc(&c->d_best, R * sizeof(int64_t)));
  CKC(cudaMalloc(&c->d_status, R * sizeof(int)));
  CKC(cudaMalloc(&c->d_counter, (2 * R + 1) * sizeof(int)));  // rollout, elite, peer-publish arrival counters
  CKC(cudaMemset(c->d_counter, 0, (2 * R + 1) * sizeof(int)));
  P.n_eblk = P.n_elite > 0 ? (int)((P.n_elite + 31) / 32) : 1;  // 32 elites per elite-kernel CTA
  P.full_cov = cfg->full_cov ? 1 : 0;
  const int erec = P.full_cov ? std::max(sbs::kEPartStride, sbs::fc_record_floats(D)) : sbs::kEPartStride;
  CKC(cudaMalloc(&c->d_epart, (size_t)R * P.n_eblk * erec * sizeof(float)));
  CKC(cudaMalloc(&c->d_sdiag, (size_t)R * 8 * sizeof(float)));
  CKC(cudaMalloc(&c->d_out, R * sizeof(sbs_output)));
  CKC(cudaHostAlloc(&c->h_out, R * sizeof(sbs_output) + 64, cudaHostAllocMapped));  // + the completion flag
  c->h_done = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c->h_out) + R * sizeof(sbs_output));
  *c->h_done = 0;
  {
    const char* e = getenv("SBS_MAPPED_OUT");  // experiments: SBS_MAPPED_OUT=0 copies the outputs back instead
    if (!e || atoi(e) != 0) {
      CKC(cudaHostGetDevicePointer((void**)&c->h_out_dev, c->h_out, 0));
      const char* f = getenv("SBS_POLL");  // experiments: SBS_POLL=0 waits with cudaStreamSynchronize instead
      if (!f || atoi(f) != 0)
        c->d_done = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(c->h_out_dev) + R * sizeof(sbs_output));
    }
  }
  // initial distribution: mean (0, 0, m|g_z|/4) per leg and knot, var = sigma^2, freq_idx 0
  {
    std::vector<float> m(RD), v(RD);
    const float fz = (float)(-(double)cfg->mass * (double)cfg->gravity[2] / 4.0);
    for (size_t i = 0; i < RD; ++i) {
      const int axis = (int)(i % D) % 3;
      m[i] = axis == 2 ? fz : 0.0f;
      v[i] = (float)((double)cfg->sigma[axis] * (double)cfg->sigma[axis]);
    }
    CKC(cudaMemcpy(c->d_mean, m.data(), RD * sizeof(float), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_var, v.data(), RD * sizeof(float), cudaMemcpyHostToDevice));
    if (cfg->full_cov) {  // C = diag(sigma^2): L = diag(sigma)
      std::vector<float> L((size_t)R * D * D, 0.0f);
      for (int r = 0; r < R; ++r)
        for (int d = 0; d < D; ++d) L[((size_t)r * D + d) * D + d] = cfg->sigma[d % 3];
      CKC(cudaMalloc(&c->d_L, L.size() * sizeof(float)));
      CKC(cudaMemcpy(c->d_L, L.data(), L.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    CKC(cudaMemset(c->d_fidx, 0, R * sizeof(int)));
  }
  P.mean = c->d_mean;
  P.var = c->d_var;
  P.fidx = c->d_fidx;
  P.xref = c->d_xref;
  P.J = c->d_J;
  P.part = c->d_part;
  P.elite = c->d_elite;
  P.best = c->d_best;
  P.status = c->d_status;
  P.counter = c->d_counter;
  P.ecounter = c->d_counter + R;
  P.gcounter = c->d_counter + 2 * R;
  P.epart = c->d_epart;
  P.sdiag = c->d_sdiag;
  P.elite_J = c->d_eJ;
  P.Lmat = c->d_L;
  P.cand = c->d_cand;
  if (P.dyn) {
    CKC(cudaMalloc(&c->d_dyn_rec, (size_t)c->dyn_recs * P.part_stride * sizeof(float)));
    CKC(cudaMalloc(&c->d_dyn_cnt, (size_t)c->dyn_cnts * sizeof(int)));
    CKC(cudaMemset(c->d_dyn_cnt, 0, (size_t)c->dyn_cnts * sizeof(int)));
    P.dyn_rec = c->d_dyn_rec;
    P.dyn_cnt = c->d_dyn_cnt;
  }
  // CEM at world = 1: select + elite moments + finish as one cluster launch (bitwise the
  // two-kernel path's results; SBS_CEM_CLUSTER=0 keeps the two kernels, for tests / A/B)
  // (SBS_CEM_CLUSTER=8 / 16 caps the cluster size).  A latency path: every robot occupies
  // a whole cluster of SMs, so it is taken only while all R clusters fit the GPU at once
  // (many robots keep the two kernels: one select SM per robot).
  P.cem_cluster = 0;
  if (cfg->world == 1 && sbs::cem_cluster_fits(P)) {
    const char* e = getenv("SBS_CEM_CLUSTER");
    int want = e ? atoi(e) : 16;
    while (want >= 8 && (int64_t)R * want > c->sm_count) want /= 2;
    P.cem_cluster = want >= 8 ? sbs::cem_cluster_size(P.P, want) : 0;
  }
  c->ref_set.assign(R, 0);
  // ---- NCCL (sample sharding) ----
  if (cfg->world > 1) {
    bool zero_id = true;
    for (int i = 0; i < 128; ++i) zero_id = zero_id && cfg->nccl_id[i] == 0;
    c->external = zero_id;
  }
  if (cfg->world > 1 && !c->external) {
    if (!g_nccl.load()) {
      c->err = "world > 1 but libnccl.so.2 could not be loaded";
      return bail(SBS_ERR_NCCL);
    }
    nccl_uid u;
    memcpy(u.internal, cfg->nccl_id, 128);
    int r2 = g_nccl.init_rank(&c->comm, cfg->world, u, cfg->rank);
    if (r2 != 0) {
      c->err = std::string("ncclCommInitRank: ") + (g_nccl.err ? g_nccl.err(r2) : "?");
      return bail(SBS_ERR_NCCL);
    }
  }
  CKC(cudaDeviceSynchronize());
  *out = c;
  return SBS_OK;
#undef CKC
}

int sbs_set_reference(sbs_ctx* c, int32_t robot, const float* x_ref) {
  if (!c || !x_ref) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  const int n = c->P.H * 12;
  if (!finite_all(x_ref, n)) return fail(c, SBS_ERR_NONFINITE, "reference not finite");
  CK(cudaSetDevice(c->cfg.device));
  // staged in pinned memory (the caller's buffer is free on return); uploaded with
  // the next step's inputs.  The block is rewritten only after its last upload.
  CK(blk_wait(c));
  memcpy(c->h_xref + (size_t)robot * n, x_ref, n * sizeof(float));
  c->ref_dirty = true;
  c->ref_set[robot] = 1;
  return SBS_OK;
}

int sbs_set_reference_device(sbs_ctx* c, const float* d_x_ref, void* stream) {
  if (!c || !d_x_ref) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  CK(cudaSetDevice(c->cfg.device));
  if (c->ref_dirty) {  // host-staged references of earlier calls are superseded
    CK(blk_wait(c));
    c->ref_dirty = false;
  }
  CK(cudaMemcpyAsync(c->d_xref, d_x_ref, (size_t)c->P.R * c->P.H * 12 * sizeof(float), cudaMemcpyDeviceToDevice,
                     (cudaStream_t)stream));
  // keep the pinned copy in sync for later host-path steps
  CK(cudaMemcpyAsync(c->h_xref, d_x_ref, (size_t)c->P.R * c->P.H * 12 * sizeof(float), cudaMemcpyDeviceToHost,
                     (cudaStream_t)stream));
  CK(blk_record(c, (cudaStream_t)stream));
  CK(note_device_work(c, (cudaStream_t)stream));
  std::fill(c->ref_set.begin(), c->ref_set.end(), 1);
  return SBS_OK;
}

int sbs_set_distribution(sbs_ctx* c, int32_t robot, const float* mean, const float* var, int32_t freq_idx) {
  if (!c || !mean || !var) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  if (freq_idx < 0 || freq_idx >= c->cfg.n_freq) return fail(c, SBS_ERR_INVALID_ARG, "freq_idx out of range");
  const int D = c->P.D;
  if (!finite_all(mean, D) || !finite_all(var, D)) return fail(c, SBS_ERR_NONFINITE, "distribution not finite");
  for (int d = 0; d < D; ++d)
    if (!(var[d] >= 0)) return fail(c, SBS_ERR_INVALID_ARG, "var must be >= 0");
  CK(cudaSetDevice(c->cfg.device));
  CK(sync_ctx(c));  // never under a step still running on a caller stream
  CK(cudaMemcpyAsync(c->d_mean + (size_t)robot * D, mean, D * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->d_var + (size_t)robot * D, var, D * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->d_fidx + robot, &freq_idx, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  if (c->d_L) {  // full covariance: C = diag(var)
    std::vector<float> L((size_t)D * D, 0.0f);
    for (int d = 0; d < D; ++d) L[(size_t)d * D + d] = sqrtf(var[d]);
    CK(cudaMemcpyAsync(c->d_L + (size_t)robot * D * D, L.data(), L.size() * sizeof(float), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return SBS_OK;
  }
  CK(cudaStreamSynchronize(c->stream));
  return SBS_OK;
}

int sbs_set_covariance(sbs_ctx* c, int32_t robot, const float* C) {
  if (!c || !C) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (!c->d_L) return fail(c, SBS_ERR_STATE, "context has no full covariance (full_cov = 0)");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  const int D = c->P.D;
  if (!finite_all(C, D * D)) return fail(c, SBS_ERR_NONFINITE, "covariance not finite");
  // Cholesky-Banachiewicz in binary64 of the symmetric part
  std::vector<double> Ld((size_t)D * D, 0.0);
  for (int i = 0; i < D; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0.5 * ((double)C[i * D + j] + (double)C[j * D + i]);
      for (int k = 0; k < j; ++k) s -= Ld[(size_t)i * D + k] * Ld[(size_t)j * D + k];
      if (i == j) {
        if (!(s > 0.0)) return fail(c, SBS_ERR_INVALID_ARG, "covariance is not positive definite");
        Ld[(size_t)i * D + i] = sqrt(s);
      } else {
        Ld[(size_t)i * D + j] = s / Ld[(size_t)j * D + j];
      }
    }
  std::vector<float> L((size_t)D * D), v(D);
  for (size_t i = 0; i < L.size(); ++i) L[i] = (float)Ld[i];
  for (int d = 0; d < D; ++d) v[d] = C[d * D + d];
  CK(cudaSetDevice(c->cfg.device));
  CK(sync_ctx(c));
  CK(cudaMemcpyAsync(c->d_L + (size_t)robot * D * D, L.data(), L.size() * sizeof(float), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->d_var + (size_t)robot * D, v.data(), D * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return SBS_OK;
}

int sbs_get_cholesky(sbs_ctx* c, int32_t robot, float* L) {
  if (!c || !L) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (!c->d_L) return fail(c, SBS_ERR_STATE, "context has no full covariance (full_cov = 0)");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  const int D = c->P.D;
  CK(cudaSetDevice(c->cfg.device));
  CK(sync_ctx(c));
  CK(cudaMemcpy(L, c->d_L + (size_t)robot * D * D, (size_t)D * D * sizeof(float), cudaMemcpyDeviceToHost));
  return SBS_OK;
}

int sbs_get_distribution(sbs_ctx* c, int32_t robot, float* mean, float* var, int32_t* freq_idx) {
  if (!c) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  const int D = c->P.D;
  CK(cudaSetDevice(c->cfg.device));
  CK(sync_ctx(c));
  if (mean) CK(cudaMemcpy(mean, c->d_mean + (size_t)robot * D, D * sizeof(float), cudaMemcpyDeviceToHost));
  if (var) CK(cudaMemcpy(var, c->d_var + (size_t)robot * D, D * sizeof(float), cudaMemcpyDeviceToHost));
  if (freq_idx) CK(cudaMemcpy(freq_idx, c->d_fidx + robot, sizeof(int), cudaMemcpyDeviceToHost));
  return SBS_OK;
}

uint32_t sbs_get_iter(const sbs_ctx* c) { return c ? c->iter : 0u; }
int sbs_set_iter(sbs_ctx* c, uint32_t iter) {
  if (!c) return SBS_ERR_INVALID_ARG;
  c->iter = iter;
  return SBS_OK;
}

namespace {
// one host-path iteration on c->stream: upload [iter | inputs | reference] in one
// copy, the kernels, the outputs back (captured once into a CUDA graph when possible)
int enqueue_host_step(sbs_ctx* c, cudaStream_t s) {
  // inputs go up with one H2D copy (measured: kernels reading them over PCIe from mapped
  // memory are slower, every CTA pays the PCIe latency); outputs come back written by the
  // finishing CTA straight into mapped pinned memory (no D2H node)
  CK(cudaMemcpyAsync(c->d_blk, c->h_blk, c->blk_bytes, cudaMemcpyHostToDevice, s));
  Params saved = c->P;
  c->P.in = c->d_in;
  c->P.iter_dev = reinterpret_cast<const uint32_t*>(c->d_blk);
  c->P.out = c->h_out_dev ? c->h_out_dev : c->d_out;  // mapped: the finishing CTA writes over PCIe, no D2H node
  int rc = enqueue_step(c, s);
  c->P = saved;
  if (rc != SBS_OK) return rc;
  if (!c->h_out_dev)
    CK(cudaMemcpyAsync(c->h_out, c->d_out, c->P.R * sizeof(sbs_output), cudaMemcpyDeviceToHost, s));
  return SBS_OK;
}
}  // namespace

#if defined(SBS_HOST_TIMING)  // experiments only: host-side phase times of the one-robot sbs_step
#include <time.h>
static double g_ht[8];
static long g_hn;
static inline double ht_now() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}
#define HT(i) (ht[i] = ht_now())
extern "C" int sbs_debug_host_times(double* out) {
  for (int i = 0; i < 8; ++i) out[i] = g_hn ? g_ht[i] / g_hn : 0.0;
  g_hn = 0;
  for (int i = 0; i < 8; ++i) g_ht[i] = 0.0;
  return 0;
}
#else
#define HT(i) ((void)0)
#endif

int sbs_step(sbs_ctx* c, const sbs_input* in, sbs_output* out) {
#if defined(SBS_HOST_TIMING)
  double ht[9];
#endif
  HT(0);
  if (!c || !in || !out) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  const int R = c->P.R;
  for (int r = 0; r < R; ++r) {
    if (!c->ref_set[r]) return fail(c, SBS_ERR_STATE, "sbs_set_reference not called for every robot");
    if (!finite_all(in[r].x0, 12) || !finite_all(in[r].feet_cur, 12) || !finite_all(in[r].feet_next, 12))
      return fail(c, SBS_ERR_NONFINITE, "non-finite x0 / feet");
    if (!(fabsf(in[r].x0[7]) < 1.5697963267948966f)) return fail(c, SBS_ERR_SINGULAR, "|pitch(x0)| >= pi/2 - 1e-3");
  }
  if (c->external && !c->peer)
    return fail(c, SBS_ERR_STATE, "external exchange: use sbs_step_records / sbs_finish_records");
  CK(cudaSetDevice(c->cfg.device));
  cudaStream_t s = c->stream;
  if (c->dev_pending) {  // a device-path step on a caller stream goes first (stream order on the GPU)
    CK(cudaStreamWaitEvent(s, c->dev_ev, 0));
    c->dev_pending = false;  // this step's own completion wait covers it from here on
  }
  if (R == 1 && c->P.H * 12 <= sbs::kInlineRefFloats && c->cfg.world == 1) {
    // inputs, reference and iteration counter ride in the kernel parameters: no copy node,
    // no graph (direct launches); outputs land in mapped pinned memory
    HT(1);
    CK(blk_wait(c));  // a reference staged by sbs_set_reference_device has landed in h_xref
    HT(2);
    Params saved = c->P;
    c->P.inline_in = 1;
    c->P.in_inline = in[0];
    memcpy(c->P.xref_inline, c->h_xref, (size_t)c->P.H * 12 * sizeof(float));
    c->P.iter_dev = nullptr;
    c->P.out = c->h_out_dev ? c->h_out_dev : c->d_out;
    // completion: the finishing CTA raises a mapped flag after the outputs (system-scope
    // fence) and the host polls it -- no event records, no driver synchronisation; with
    // sbs_profile on, CUDA events time the step instead (device_us)
    const bool timed = c->profile != 0;
    const bool poll = c->d_done && !timed;
    if (poll) {
      c->P.done = c->d_done;
      c->P.done_value = ++c->done_seq;
    }
    HT(3);
    if (timed) CK(cudaEventRecord(c->ev0, s));
    HT(4);
    const int rc = enqueue_step(c, s);
    HT(5);
    c->P = saved;
    if (rc != SBS_OK) return rc;
    if (!c->h_out_dev) CK(cudaMemcpyAsync(c->h_out, c->d_out, sizeof(sbs_output), cudaMemcpyDeviceToHost, s));
    if (timed) CK(cudaEventRecord(c->ev1, s));
    HT(6);
    if (poll) {
      // acquire loads: the outputs the finishing CTA wrote before its release store are
      // visible once the flag is (on weakly ordered hosts too)
      uint32_t* flag = c->h_done;
      for (uint32_t n = 1; __atomic_load_n(flag, __ATOMIC_ACQUIRE) != c->done_seq; ++n) {
        if ((n & 1023u) == 0) {  // a failed launch never raises the flag: ask the stream now and then
          const cudaError_t e = cudaStreamQuery(s);
          if (e != cudaErrorNotReady && e != cudaSuccess) CK(e);
          if (e == cudaSuccess && __atomic_load_n(flag, __ATOMIC_ACQUIRE) != c->done_seq)
            return fail(c, SBS_ERR_CUDA, "step completed without its flag");
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
      }
    } else {
      CK(cudaStreamSynchronize(s));
    }
    HT(7);
    float ms = 0.f;
    if (timed) cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    c->h_out[0].device_us = ms * 1000.f;
    memcpy(out, c->h_out, sizeof(sbs_output));
    c->iter += 1;
    HT(8);
#if defined(SBS_HOST_TIMING)
    for (int i = 0; i < 8; ++i) g_ht[i] += ht[i + 1] - ht[i];
    ++g_hn;
#endif
    return c->h_out[0].status == SBS_WARN_ALL_DIVERGED ? SBS_WARN_ALL_DIVERGED : SBS_OK;
  }
  CK(blk_wait(c));
  memcpy(c->h_blk, &c->iter, sizeof(uint32_t));
  memcpy(c->h_in, in, R * sizeof(sbs_input));
  c->ref_dirty = false;  // the whole block (with the reference) goes up with this step
  const bool use_graph = !c->profile && c->cfg.world == 1;
  if (c->profile) CK(cudaEventRecord(c->ev0, s));  // events stay outside the graph (host-synchronisable)
  if (use_graph) {
    if (!c->graph) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      const int rc = enqueue_host_step(c, s);
      const cudaError_t e = cudaStreamEndCapture(s, &g);  // always leave capture mode
      if (rc != SBS_OK) {
        if (e == cudaSuccess) cudaGraphDestroy(g);
        return rc;
      }
      CK(e);
      const cudaError_t ei = cudaGraphInstantiate(&c->graph, g, 0);
      cudaGraphDestroy(g);
      CK(ei);
    }
    CK(cudaGraphLaunch(c->graph, s));
  } else {
    const int rc = enqueue_host_step(c, s);
    if (rc != SBS_OK) return rc;
  }
  if (c->profile) CK(cudaEventRecord(c->ev1, s));
  CK(blk_record(c, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  if (c->profile) cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  int status = SBS_OK;
  for (int r = 0; r < R; ++r) {
    c->h_out[r].device_us = ms * 1000.f;
    if (c->h_out[r].status == SBS_WARN_ALL_DIVERGED) status = SBS_WARN_ALL_DIVERGED;
  }
  memcpy(out, c->h_out, R * sizeof(sbs_output));
  c->iter += 1;
  return status;
}

int sbs_step_device(sbs_ctx* c, const sbs_input* d_in, sbs_output* d_out, void* stream) {
  if (!c || !d_in || !d_out) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  for (int r = 0; r < c->P.R; ++r)
    if (!c->ref_set[r]) return fail(c, SBS_ERR_STATE, "reference not set for every robot");
  CK(cudaSetDevice(c->cfg.device));
  if (c->ref_dirty) {  // references staged by sbs_set_reference go up first, in stream order
    CK(cudaMemcpyAsync(c->d_xref, c->h_xref, (size_t)c->P.R * c->P.H * 12 * sizeof(float),
                       cudaMemcpyHostToDevice, (cudaStream_t)stream));
    CK(blk_record(c, (cudaStream_t)stream));
    c->ref_dirty = false;
  }
  c->P.in = d_in;
  c->P.out = d_out;
  int rc = enqueue_step(c, (cudaStream_t)stream);
  if (rc != SBS_OK) return rc;
  c->iter += 1;
  CK(note_device_work(c, (cudaStream_t)stream));
  return SBS_OK;
}

int sbs_record_floats(const sbs_ctx* c) { return c ? c->P.ex_stride : 0; }

int sbs_peer_handle(sbs_ctx* c, uint8_t handle[64], void** base) {
  if (!c) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (c->cfg.world < 2) return fail(c, SBS_ERR_STATE, "peer exchange needs world > 1");
  if (c->cfg.world > sbs::kMaxWorld) return fail(c, SBS_ERR_INVALID_ARG, "peer exchange supports at most 8 ranks");
  CK(cudaSetDevice(c->cfg.device));
  if (handle) {
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, c->d_xbuf));
    memcpy(handle, &h, 64);
  }
  if (base) *base = c->d_xbuf;
  return SBS_OK;
}

int sbs_peer_connect(sbs_ctx* c, void* const* bases, const uint8_t* handles) {
  if (!c) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (!bases && !handles) {  // disconnect: back to the NCCL / external exchange
    CK(cudaSetDevice(c->cfg.device));
    CK(cudaStreamSynchronize(c->stream));
    for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
    c->ipc_opened.clear();
    c->peer_base.clear();
    c->peer = false;
    return SBS_OK;
  }
  const int W = c->cfg.world, me = c->cfg.rank;
  if (W < 2 || W > sbs::kMaxWorld) return fail(c, SBS_ERR_STATE, "peer exchange needs 2 <= world <= 8");
  CK(cudaSetDevice(c->cfg.device));
  if (g_wait_value32(c->stream, c->d_xflags + me, 0) != 0)  // probes cuStreamWaitValue32 (the own flag is >= 0)
    return fail(c, SBS_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  CK(cudaStreamSynchronize(c->stream));
  c->peer_base.clear();
  for (int j = 0; j < W; ++j) {
    char* b = nullptr;
    if (j == me) {
      b = c->d_xbuf;
    } else if (bases) {
      b = static_cast<char*>(bases[j]);  // same-process contexts (tests, one process driving several GPUs)
      int dev_other = -1;
      cudaPointerAttributes pa;
      if (cudaPointerGetAttributes(&pa, b) == cudaSuccess) dev_other = pa.device;
      if (dev_other >= 0 && dev_other != c->cfg.device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(dev_other, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        (void)cudaGetLastError();
      }
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, handles + 64 * (size_t)j, 64);
      void* q = nullptr;
      CK(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(q);
      b = static_cast<char*>(q);
    }
    c->peer_base.push_back(b);
    c->P.peer_flags[j] = reinterpret_cast<uint32_t*>(b + c->xflags_off);
  }
  c->peer = true;
  return SBS_OK;
}

int sbs_step_records(sbs_ctx* c, const sbs_input* d_in, float* d_rec, void* stream) {
  if (!c || !d_in || !d_rec) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (c->cfg.world < 2) return fail(c, SBS_ERR_STATE, "records exchange needs world > 1");
  for (int r = 0; r < c->P.R; ++r)
    if (!c->ref_set[r]) return fail(c, SBS_ERR_STATE, "reference not set for every robot");
  CK(cudaSetDevice(c->cfg.device));
  if (c->ref_dirty) {
    CK(cudaMemcpyAsync(c->d_xref, c->h_xref, (size_t)c->P.R * c->P.H * 12 * sizeof(float),
                       cudaMemcpyHostToDevice, (cudaStream_t)stream));
    CK(blk_record(c, (cudaStream_t)stream));
    c->ref_dirty = false;
  }
  c->P.in = d_in;
  const int rc = enqueue_records(c, (cudaStream_t)stream, d_rec);
  if (rc != SBS_OK) return rc;
  CK(note_device_work(c, (cudaStream_t)stream));
  return SBS_OK;
}

int sbs_finish_records(sbs_ctx* c, const float* d_recs, const sbs_input* d_in, sbs_output* d_out, void* stream) {
  if (!c || !d_recs || !d_in || !d_out) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (c->cfg.world < 2) return fail(c, SBS_ERR_STATE, "records exchange needs world > 1");
  CK(cudaSetDevice(c->cfg.device));
  c->P.in = d_in;
  c->P.out = d_out;
  const int rc = enqueue_finish(c, (cudaStream_t)stream, d_recs);
  if (rc != SBS_OK) return rc;
  c->iter += 1;
  CK(note_device_work(c, (cudaStream_t)stream));
  return SBS_OK;
}

namespace {
sbs::LoopArgs loop_args(const sbs_loop_config* lc, const sbs_command* d_cmd, const float* d_wrench,
                        int32_t* d_fallen, float* d_trace) {
  sbs::LoopArgs a;
  memset(&a, 0, sizeof a);  // padding too: the struct is part of the loop graph's key
  for (int k = 0; k < 12; ++k) a.hip[k] = lc->hip[k];
  a.h_nom = lc->h_nom;
  a.fall_angle = lc->fall_angle;
  a.fall_height = lc->fall_height;
  a.n_inner = lc->n_inner;
  a.cmd = d_cmd;
  a.wrench = d_wrench;
  a.fallen = d_fallen;
  a.trace = d_trace;
  return a;
}

int check_loop_config(sbs_ctx* c, const sbs_loop_config* lc) {
  if (!lc) return fail(c, SBS_ERR_INVALID_ARG, "NULL loop config");
  if (!finite_all(lc->hip, 12) || !std::isfinite(lc->h_nom) || !(lc->fall_angle > 0) || !std::isfinite(lc->fall_height) ||
      lc->n_inner < 1 || lc->n_inner > 64)
    return fail(c, SBS_ERR_INVALID_ARG, "bad loop config");
  return SBS_OK;
}

int upload_dirty_reference(sbs_ctx* c, cudaStream_t s) {
  if (c->ref_dirty) {  // references staged by sbs_set_reference go up first, in stream order
    CK(cudaMemcpyAsync(c->d_xref, c->h_xref, (size_t)c->P.R * c->P.H * 12 * sizeof(float), cudaMemcpyHostToDevice, s));
    CK(blk_record(c, s));
    c->ref_dirty = false;
  }
  return SBS_OK;
}
}  // namespace

int sbs_advance(sbs_ctx* c, sbs_input* d_in, const sbs_output* d_out, const sbs_command* d_cmd, const float* d_wrench,
                int32_t* d_fallen, const sbs_loop_config* lc, void* stream) {
  if (!c || !d_in || !d_out) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  int rc = check_loop_config(c, lc);
  if (rc != SBS_OK) return rc;
  CK(cudaSetDevice(c->cfg.device));
  cudaStream_t s = (cudaStream_t)stream;
  rc = upload_dirty_reference(c, s);  // keep the stream order of staged references before the rebuild
  if (rc != SBS_OK) return rc;
  const sbs::LoopArgs a = loop_args(lc, d_cmd, d_wrench, d_fallen, nullptr);
  CK(timed(c, SBS_KERNEL_ADVANCE, s, [&] { return sbs::launch_advance(c->P, a, d_in, d_out, s); }));
  CK(note_device_work(c, s));
  std::fill(c->ref_set.begin(), c->ref_set.end(), 1);
  return SBS_OK;
}

int sbs_run_loop(sbs_ctx* c, int32_t n_iter, sbs_input* d_in, sbs_output* d_out, const sbs_command* d_cmd,
                 const float* d_wrench, int32_t* d_fallen, float* d_trace, const sbs_loop_config* lc, void* stream) {
  if (!c || !d_in || !d_out || n_iter < 0) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument or n_iter < 0");
  if (c->cfg.world != 1) return fail(c, SBS_ERR_STATE, "sbs_run_loop needs world = 1 (shard robots across contexts)");
  int rc = check_loop_config(c, lc);
  if (rc != SBS_OK) return rc;
  for (int r = 0; r < c->P.R; ++r)
    if (!c->ref_set[r]) return fail(c, SBS_ERR_STATE, "reference not set for every robot");
  if (n_iter == 0) return SBS_OK;
  CK(cudaSetDevice(c->cfg.device));
  cudaStream_t s = (cudaStream_t)stream;
  rc = upload_dirty_reference(c, s);
  if (rc != SBS_OK) return rc;
  if (!c->d_loopw) {
    CK(cudaMalloc(&c->d_loopw, 4 * sizeof(uint32_t)));
    CK(cudaMemset(c->d_loopw, 0, 4 * sizeof(uint32_t)));
    CK(cudaMallocHost(&c->h_loopw, 2 * sizeof(uint32_t)));
  }
  // device iteration counter := iter (the step kernels read it; the advance kernel moves it)
  CK(blk_wait(c));  // h_loopw's previous upload has completed
  c->h_loopw[0] = c->iter;
  c->h_loopw[1] = c->iter;
  CK(cudaMemcpyAsync(c->d_loopw, c->h_loopw, 2 * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  CK(blk_record(c, s));
  sbs::LoopArgs a = loop_args(lc, d_cmd, d_wrench, d_fallen, d_trace);
  a.loop = c->d_loopw;
  a.counter = reinterpret_cast<int*>(c->d_loopw + 2);
  auto enqueue_iter = [&](cudaStream_t st) -> int {
    for (int k = 0; k < lc->n_inner; ++k) {  // n_inner SBS iterations on the same x0 (warm shift on the first only)
      Params saved = c->P;
      c->P.in = d_in;
      c->P.out = d_out;
      c->P.iter_dev = c->d_loopw;
      c->P.iter_add = (uint32_t)k;
      if (k > 0) c->P.warm_shift = 0;
      int r2 = enqueue_step(c, st);
      c->P = saved;
      if (r2 != SBS_OK) return r2;
    }
    CK(timed(c, SBS_KERNEL_ADVANCE, st, [&] { return sbs::launch_advance(c->P, a, d_in, d_out, st); }));
    return SBS_OK;
  };
  if (c->profile) {  // per-kernel events: no graph
    for (int i = 0; i < n_iter; ++i) {
      rc = enqueue_iter(s);
      if (rc != SBS_OK) return rc;
    }
  } else {
    std::vector<char> key(sizeof(a) + sizeof(d_in) + sizeof(d_out));
    memcpy(key.data(), &a, sizeof(a));
    memcpy(key.data() + sizeof(a), &d_in, sizeof(d_in));
    memcpy(key.data() + sizeof(a) + sizeof(d_in), &d_out, sizeof(d_out));
    if (!c->loop_graph || key != c->loop_key) {
      // two graphs: one control step, and kLoopUnroll control steps (fewer graph launches;
      // consecutive kernels inside a graph keep their programmatic-launch overlap)
      for (cudaGraphExec_t* ge : {&c->loop_graph, &c->loop_graph_u}) {
        if (*ge) {
          CK(cudaGraphExecDestroy(*ge));
          *ge = nullptr;
        }
      }
      for (int which = 0; which < 2; ++which) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int u = 0; u < (which ? kLoopUnroll : 1) && rc == SBS_OK; ++u) rc = enqueue_iter(c->stream);
        const cudaError_t e = cudaStreamEndCapture(c->stream, &g);  // always leave capture mode
        if (rc != SBS_OK) {
          if (e == cudaSuccess) cudaGraphDestroy(g);
          return rc;
        }
        CK(e);
        const cudaError_t ei = cudaGraphInstantiate(which ? &c->loop_graph_u : &c->loop_graph, g, 0);
        cudaGraphDestroy(g);
        CK(ei);
      }
      c->loop_key = key;
    }
    int i = 0;
    for (; i + kLoopUnroll <= n_iter; i += kLoopUnroll) CK(cudaGraphLaunch(c->loop_graph_u, s));
    for (; i < n_iter; ++i) CK(cudaGraphLaunch(c->loop_graph, s));
  }
  c->iter += (uint32_t)n_iter * (uint32_t)lc->n_inner;
  CK(note_device_work(c, s));
  return SBS_OK;
}

int sbs_get_reference(sbs_ctx* c, int32_t robot, float* x_ref) {
  if (!c || !x_ref) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  const int n = c->P.H * 12;
  if (c->ref_dirty) {  // staged on the host, not uploaded yet
    memcpy(x_ref, c->h_xref + (size_t)robot * n, n * sizeof(float));
    return SBS_OK;
  }
  CK(cudaSetDevice(c->cfg.device));
  CK(sync_ctx(c));  // the reference may be rebuilt on any caller stream
  CK(cudaMemcpy(x_ref, c->d_xref + (size_t)robot * n, n * sizeof(float), cudaMemcpyDeviceToHost));
  return SBS_OK;
}

int sbs_get_state(sbs_ctx* c, void* buf, uint64_t* nbytes) {
  if (!c || !nbytes) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  const int R = c->P.R, D = c->P.D;
  const uint64_t LD = c->d_L ? (uint64_t)D * D : 0;  // full covariance: the Cholesky factors follow
  const uint64_t need = 32 + (uint64_t)R * (2 * D * sizeof(float) + sizeof(int32_t)) + (uint64_t)R * LD * sizeof(float);
  if (!buf || *nbytes < need) {
    *nbytes = need;
    return buf ? fail(c, SBS_ERR_INVALID_ARG, "buffer too small") : SBS_OK;
  }
  *nbytes = need;
  char* b = (char*)buf;
  const uint64_t hdr[4] = {0x5342535354415445ull /*"SBSSTATE"*/, (uint64_t)c->iter, c->cfg.seed,
                           ((uint64_t)R << 32) | (uint64_t)D};
  memcpy(b, hdr, 32);
  CK(cudaSetDevice(c->cfg.device));
  CK(sync_ctx(c));
  CK(cudaMemcpy(b + 32, c->d_mean, (size_t)R * D * sizeof(float), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b + 32 + (size_t)R * D * 4, c->d_var, (size_t)R * D * sizeof(float), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b + 32 + (size_t)R * D * 8, c->d_fidx, R * sizeof(int), cudaMemcpyDeviceToHost));
  if (LD)
    CK(cudaMemcpy(b + 32 + (size_t)R * D * 8 + (size_t)R * 4, c->d_L, (size_t)R * LD * sizeof(float),
                  cudaMemcpyDeviceToHost));
  return SBS_OK;
}

int sbs_set_state(sbs_ctx* c, const void* buf, uint64_t nbytes) {
  if (!c || !buf) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  const int R = c->P.R, D = c->P.D;
  const uint64_t LD = c->d_L ? (uint64_t)D * D : 0;  // full covariance: the Cholesky factors follow
  const uint64_t need = 32 + (uint64_t)R * (2 * D * sizeof(float) + sizeof(int32_t)) + (uint64_t)R * LD * sizeof(float);
  if (nbytes != need) return fail(c, SBS_ERR_INVALID_ARG, "state size mismatch");
  const char* b = (const char*)buf;
  uint64_t hdr[4];
  memcpy(hdr, b, 32);
  if (hdr[0] != 0x5342535354415445ull || hdr[2] != c->cfg.seed || hdr[3] != (((uint64_t)R << 32) | (uint64_t)D))
    return fail(c, SBS_ERR_INVALID_ARG, "state does not match this context");
  CK(cudaSetDevice(c->cfg.device));
  CK(sync_ctx(c));
  CK(cudaMemcpy(c->d_mean, b + 32, (size_t)R * D * sizeof(float), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_var, b + 32 + (size_t)R * D * 4, (size_t)R * D * sizeof(float), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_fidx, b + 32 + (size_t)R * D * 8, R * sizeof(int), cudaMemcpyHostToDevice));
  if (LD)
    CK(cudaMemcpy(c->d_L, b + 32 + (size_t)R * D * 8 + (size_t)R * 4, (size_t)R * LD * sizeof(float),
                  cudaMemcpyHostToDevice));
  c->iter = (uint32_t)hdr[1];
  return SBS_OK;
}

int sbs_debug_samples(sbs_ctx* c, int32_t robot, int64_t k0, int64_t n, float* z, float* theta, int32_t* fidx) {
  if (!c || n < 0 || k0 < 0) return fail(c, SBS_ERR_INVALID_ARG, "bad argument");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  if (n == 0) return SBS_OK;
  CK(cudaSetDevice(c->cfg.device));
  const int D = c->P.D;
  float *dz, *dth;
  int* df;
  CK(cudaMalloc(&dz, (size_t)n * D * sizeof(float)));
  CK(cudaMalloc(&dth, (size_t)n * D * sizeof(float)));
  CK(cudaMalloc(&df, (size_t)n * sizeof(int)));
  Params P = c->P;
  P.iter = c->iter;
  // the debug kernel needs an sbs_input for load_robot: use a zero one
  sbs_input* din;
  CK(cudaMalloc(&din, (size_t)c->P.R * sizeof(sbs_input)));
  CK(cudaMemset(din, 0, (size_t)c->P.R * sizeof(sbs_input)));
  P.in = din;
  cudaError_t e = sbs::launch_debug_samples(P, robot, k0, n, dz, dth, df, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && z) e = cudaMemcpy(z, dz, (size_t)n * D * sizeof(float), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && theta) e = cudaMemcpy(theta, dth, (size_t)n * D * sizeof(float), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && fidx) e = cudaMemcpy(fidx, df, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(dz);
  cudaFree(dth);
  cudaFree(df);
  cudaFree(din);
  if (e != cudaSuccess) return cuda_fail(c, e, "sbs_debug_samples");
  return SBS_OK;
}

int sbs_debug_costs(sbs_ctx* c, float* J) {
  if (!c || !J) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(J, c->d_J, (size_t)c->P.R * c->P.K_local * sizeof(float), cudaMemcpyDeviceToHost));
  return SBS_OK;
}

int sbs_debug_elites(sbs_ctx* c, int32_t robot, int64_t* idx) {
  if (!c || !idx) return fail(c, SBS_ERR_INVALID_ARG, "NULL argument");
  if (c->P.n_elite < 1) return fail(c, SBS_ERR_STATE, "no elites in MPPI mode");
  if (robot < 0 || robot >= c->P.R) return fail(c, SBS_ERR_INVALID_ARG, "robot out of range");
  CK(cudaSetDevice(c->cfg.device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(idx, c->d_elite + (size_t)robot * c->P.n_elite, c->P.n_elite * sizeof(int64_t),
                cudaMemcpyDeviceToHost));
  return SBS_OK;
}

int sbs_debug_select(const float* J, int64_t K, int64_t K_e, int64_t* idx, int32_t device) {
  sbs_ctx* c = nullptr;
  if (!J || !idx || K < 1 || K_e < 1 || K_e > K || K > 0x7fffffffLL)
    return fail(nullptr, SBS_ERR_INVALID_ARG, "bad argument");
  CK(cudaSetDevice(device));
  CK(sbs::prepare_kernels(0));
  float* dJ;
  int64_t* di;
  CK(cudaMalloc(&dJ, K * sizeof(float)));
  CK(cudaMalloc(&di, K_e * sizeof(int64_t)));
  cudaError_t e = cudaMemcpy(dJ, J, K * sizeof(float), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = sbs::launch_select_raw(dJ, K, K_e, di, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(idx, di, K_e * sizeof(int64_t), cudaMemcpyDeviceToHost);
  cudaFree(dJ);
  cudaFree(di);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, "sbs_debug_select");
  return SBS_OK;
}

extern "C++" {
namespace {
// host in -> device kernel -> host out, for the stand-alone debug kernels
template <typename F>
int debug_roundtrip(int32_t device, const char* what, const std::vector<std::pair<const void*, size_t>>& ins,
                    const std::vector<std::pair<void*, size_t>>& outs, F launch) {
  sbs_ctx* c = nullptr;
  CK(cudaSetDevice(device));
  std::vector<void*> din(ins.size(), nullptr), dout(outs.size(), nullptr);
  cudaError_t e = cudaSuccess;
  for (size_t i = 0; i < ins.size() && e == cudaSuccess; ++i) {
    e = cudaMalloc(&din[i], ins[i].second);
    if (e == cudaSuccess) e = cudaMemcpy(din[i], ins[i].first, ins[i].second, cudaMemcpyHostToDevice);
  }
  for (size_t i = 0; i < outs.size() && e == cudaSuccess; ++i) e = cudaMalloc(&dout[i], outs[i].second);
  if (e == cudaSuccess) e = launch(din, dout);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  for (size_t i = 0; i < outs.size() && e == cudaSuccess; ++i)
    e = cudaMemcpy(outs[i].first, dout[i], outs[i].second, cudaMemcpyDeviceToHost);
  for (void* p : din) cudaFree(p);
  for (void* p : dout) cudaFree(p);
  if (e != cudaSuccess) return cuda_fail(nullptr, e, what);
  return SBS_OK;
}
}  // namespace
}  // extern "C++"

int sbs_debug_noise(const uint32_t* words, int64_t n, float* z, int32_t device) {
  if (!words || !z || n < 1 || n > (1LL << 28)) return fail(nullptr, SBS_ERR_INVALID_ARG, "bad argument");
  const size_t b = (size_t)n * 16;
  return debug_roundtrip(device, "sbs_debug_noise", {{words, b}}, {{z, b}},
                         [&](std::vector<void*>& i, std::vector<void*>& o) {
                           return sbs::launch_debug_noise(i[0], n, o[0], 0);
                         });
}

int sbs_debug_philox(const uint32_t* ctr, const uint32_t* key, int64_t n, uint32_t* ours, uint32_t* curand_words,
                     int32_t device) {
  if (!ctr || !key || !ours || !curand_words || n < 1 || n > (1LL << 26))
    return fail(nullptr, SBS_ERR_INVALID_ARG, "bad argument");
  return debug_roundtrip(device, "sbs_debug_philox", {{ctr, (size_t)n * 16}, {key, (size_t)n * 8}},
                         {{ours, (size_t)n * 32}, {curand_words, (size_t)n * 16}},
                         [&](std::vector<void*>& i, std::vector<void*>& o) {
                           return sbs::launch_debug_philox(i[0], i[1], n, o[0], o[1], 0);
                         });
}

int sbs_local_range(const sbs_ctx* c, int64_t* k_begin, int64_t* K_local) {
  if (!c || !k_begin || !K_local) return SBS_ERR_INVALID_ARG;
  *k_begin = c->P.k_begin;
  *K_local = c->P.K_local;
  return SBS_OK;
}

int sbs_profile(sbs_ctx* c, int32_t enable) {
  if (!c) return SBS_ERR_INVALID_ARG;
  c->profile = enable != 0;
  return SBS_OK;
}

int sbs_kernel_times(sbs_ctx* c, double* total_ms, int64_t* launches) {
  if (!c) return SBS_ERR_INVALID_ARG;
  CK(cudaSetDevice(c->cfg.device));
  for (auto& pd : c->pending) {
    CK(cudaEventSynchronize(pd.b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, pd.a, pd.b));
    c->kt[pd.kernel] += ms;
    c->kl[pd.kernel] += 1;
    c->free_events.push_back(pd.a);
    c->free_events.push_back(pd.b);
  }
  c->pending.clear();
  for (int k = 0; k < SBS_NKERNELS; ++k) {
    if (total_ms) total_ms[k] = c->kt[k];
    if (launches) launches[k] = c->kl[k];
    c->kt[k] = 0;
    c->kl[k] = 0;
  }
  return SBS_OK;
}

int sbs_launches_per_step(const sbs_ctx* c) {
  if (!c) return 0;
  if (c->cfg.world > 1) return c->cfg.mode == SBS_CEM ? 4 : 2;  // + the exchange (peer stores or ncclAllGather)
  return c->cfg.mode == SBS_CEM ? (c->P.cem_cluster ? 2 : 3) : 1;
}

}  // extern "C"
