// vg.cu — libvg: C ABI (include/vg.h) over the sm_100a kernels in vg_kernels.cuh.
//
// Host side: configuration validation (SURVEY.md §8b conventions), derived fp32 constants,
// scratch ownership, launch sequencing.  No allocation, host synchronization or D2H copy
// happens after vg_world_create except in vg_sync_errors / vg_step_host (documented).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <climits>
#include <new>
#include <vector>

#include <dlfcn.h>
#include <mutex>

#include <nccl.h>          // types only: libnccl is loaded at run time (NcclApi below)
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: no-ops unless a profiler injects itself

#include "vg.h"
#include "vg_kernels.cuh"
#include "vg_policy.cuh"
#include "vg_rl.cuh"

namespace {

thread_local char g_err[512] = "";

vg_status fail(vg_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

#define VG_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(VG_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                           \
  } while (0)

// NCCL, loaded with dlopen on first use (the library itself has no link-time NCCL
// dependency, so it loads on CPU-only machines): $VG_NCCL_LIB, else the libnccl.so.2
// already in the process (torch's), else the system one.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  char err[256] = "";
};

NcclApi& nccl_state() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("VG_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n || !n[0]) continue;
      api.h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
      if (api.h) break;
    }
    if (!api.h) {
      snprintf(api.err, sizeof(api.err), "cannot load libnccl (set VG_NCCL_LIB): %s", dlerror());
      return;
    }
#define VG_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
    VG_NCCL_SYM(GetUniqueId);
    VG_NCCL_SYM(CommInitRank);
    VG_NCCL_SYM(CommDestroy);
    VG_NCCL_SYM(CommGetAsyncError);
    VG_NCCL_SYM(Send);
    VG_NCCL_SYM(Recv);
    VG_NCCL_SYM(GroupStart);
    VG_NCCL_SYM(GroupEnd);
    VG_NCCL_SYM(GetErrorString);
#undef VG_NCCL_SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.CommGetAsyncError ||
        !api.Send || !api.Recv || !api.GroupStart || !api.GroupEnd || !api.GetErrorString) {
      snprintf(api.err, sizeof(api.err), "libnccl lacks a needed symbol (ncclSend/ncclRecv need NCCL >= 2.7)");
      dlclose(api.h);
      api.h = nullptr;
    }
  });
  return api;
}
const NcclApi* nccl_api() { return nccl_state().h ? &nccl_state() : nullptr; }
const char* nccl_err() { return nccl_state().err; }

#define VG_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      return fail(VG_ENCCL, "%s: %s", #call, nccl_api()->GetErrorString(r_));        \
  } while (0)

// NVTX range over one ABI call (host enqueue; a profiler correlates it with the
// kernels it launched): the phases of a step show up by name in nsys / ncu timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

}  // namespace

struct vg_world {
  vg_config cfg;
  vg::Params P;
  int device = -1;
  int n_cells = 0;
  bool binned = false;
  bool fused_bin = false;          // K1-K3 fused per replica (small worlds)
  int staged_bin = 0;              // ... as a persistent shared-memory staged kernel (MODE 1 / 2)
  bool gather_bin = false;         // K2-K3b as one per-cell gather kernel (K3g)
  bool sense_def = false;          // K4 sector pass: the default-constant instance
  size_t scratch_bytes = 0;
  uint32_t* count = nullptr;       // [n_cells]     per-cell histogram (zero between uses)
  uint32_t* tile_sum = nullptr;    // [n_cells / 4096 + 1] multi-CTA scan partials
  uint32_t* cell_start = nullptr;  // [n_cells + 1]
  uint32_t* cell_id = nullptr;     // [R*N]
  uint32_t* slot = nullptr;        // [R*N]         arrival slot within the cell
  uint32_t* tmp_id = nullptr;      // [R*N]         arrival-order agent ids
  uint32_t* perm = nullptr;        // [R*N]         stable order
  float4* tmp_rec = nullptr;       // [R*N]
  float4* sorted = nullptr;        // [R*N]
  float4* xo_rec = nullptr;        // [R*N]         K4 sense order: within a cell by (axis key, id)
  uint32_t* xo_perm = nullptr;     // [R*N]         agent ids in sense order
  float2* xo_xy = nullptr;         // [R*N + 32 H]  positions in sense order (K4 candidate reads)
  uint32_t* sub_tab = nullptr;     // [(n_cells + 1) * kSub] K4 window table (K3b)
  uint2* work = nullptr;           // [work_cap] K4 work items (cell, first query)
  uint32_t* work_cnt = nullptr;    // [1] item count
  long long work_cap = 0;
  float2* ray_dir = nullptr;       // [v] ray vision: sector-centre ray directions (agent frame)
  float2* act_dev = nullptr;       // [R*N]         staging for vg_step_host
  unsigned long long* err_dev = nullptr;  // smallest bad agent index (device word)
  uint32_t* err_flag = nullptr;    // mapped pinned host flag (set by kernels)
  // slab mode (shard = VG_SHARD_SLAB)
  bool slab = false;
  vg::Slab SL{};
  vg::SlabBufs SB{};
  uint32_t* loc_n = nullptr;       // device counter (SB.n_loc)
  uint32_t* slab_ovf = nullptr;    // device overflow flag (SB.overflow)
  unsigned char* msg = nullptr;    // 4 messages: send_l, send_r, recv_l, recv_r
  size_t msg_bytes = 0;
  int left = -1, right = -1;
  int slab_stage = 0;              // 0 binned / 1 begun (vg_slab_begin) / 2 interior done
  ncclComm_t comm = nullptr;       // the world's communicator (cfg.nccl_unique_id)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // phase timing (vg_profile_begin/end): VG_N_PHASES + 1 events per recorded step
  std::vector<cudaEvent_t> prof_ev;
  int prof_max = 0, prof_n = 0;
  // vg_step CUDA graphs, keyed by the (state, actions, outputs) pointers: one graph launch
  // per step instead of five kernel launches (launch-bound small worlds).  Captured on a
  // private stream, launched on the caller's.  Disabled while profiling, inside a caller's
  // capture, or with VG_NO_GRAPH=1.
  struct GraphEntry {
    const void* state;
    const void* actions;
    vg_outputs outs;
    cudaGraphExec_t exec;
    unsigned long long last_use;
  };
  std::vector<GraphEntry> graphs;
  unsigned long long graph_clock = 0;
  cudaStream_t cap_stream = nullptr;
  bool graphs_enabled = true;
  int n_sm = 148;
};

namespace {

// A16: cells per axis G = largest integer with L/G >= d_v (1 + 2^-12), in double.
int auto_grid(double L, double dv) {
  const double need = dv * (1.0 + std::ldexp(1.0, -12));
  int g = (int)std::floor(L / need);
  while (g > 0 && L / g < need) --g;
  return g;
}

vg_status validate(const vg_config& c, int* grid_out) {
  const double PI = 3.14159265358979323846;
  if (c.env != VG_ENV_FLOCK && c.env != VG_ENV_TAG) return fail(VG_EINVAL, "env: must be 0 (flock) or 1 (tag)");
  if (c.vision != VG_VISION_SECTOR && c.vision != VG_VISION_RAY) return fail(VG_EINVAL, "vision: must be 0 (sector) or 1 (ray-disc)");
  if (c.shard != VG_SHARD_REPLICA && c.shard != VG_SHARD_SLAB) return fail(VG_EINVAL, "shard: must be 0 (replica) or 1 (slab)");
  if (c.n_agents <= 0) return fail(VG_EINVAL, "n_agents: must be > 0 (S:241)");
  if (c.n_replicas <= 0) return fail(VG_EINVAL, "n_replicas: must be > 0");
  if ((long long)c.n_agents * c.n_replicas >= (1LL << 31)) return fail(VG_EINVAL, "n_agents*n_replicas: must be < 2^31");
  if (!(c.width > 0.f) || !std::isfinite(c.width)) return fail(VG_EINVAL, "width: must be finite and > 0");
  if (!(c.d_v > 0.f) || !(2.0 * c.d_v < c.width)) return fail(VG_EINVAL, "d_v: must satisfy 0 < d_v < width/2 (A9)");
  if (!(c.d_r > 0.f) || !(2.0 * c.d_r < c.d_v)) return fail(VG_EINVAL, "d_r: must satisfy 0 < 2 d_r < d_v (S:214)");
  if (!(c.fov > 0.f) || !(c.fov <= (float)(2.0 * PI))) return fail(VG_EINVAL, "fov: must satisfy 0 < fov <= 2 pi (S:149)");
  const int ch = (c.env == VG_ENV_FLOCK) ? 1 : 2;
  if (c.v < 1 || ch * c.v > vg::kMaxViewSlots) return fail(VG_EINVAL, "v: must satisfy 1 <= channels*v <= 128");
  if (!(c.theta_max > 0.f) || !(c.theta_max <= (float)PI)) return fail(VG_EINVAL, "theta_max: must satisfy 0 < theta_max <= pi (S:214)");
  if (!(c.s_max > 0.f) || !std::isfinite(c.s_max)) return fail(VG_EINVAL, "s_max: must be finite and > 0");
  if (!(c.s_max < 0.5f * c.width)) return fail(VG_EINVAL, "s_max: must be < width/2");
  if (c.env == VG_ENV_FLOCK) {
    if (!(c.s_min >= 0.f) || !(c.s_min < c.s_max)) return fail(VG_EINVAL, "s_min: must satisfy 0 <= s_min < s_max (S:214)");
    if (!(c.a_max > 0.f) || !std::isfinite(c.a_max)) return fail(VG_EINVAL, "a_max: must be finite and > 0 (S:214)");
  } else {
    if (c.n_chasers < 0 || c.n_chasers > c.n_agents) return fail(VG_EINVAL, "n_chasers: must satisfy 0 <= n_chasers <= n_agents");
    if (!(c.s_max_chaser > 0.f) || !(c.s_max_chaser < 0.5f * c.width)) return fail(VG_EINVAL, "s_max_chaser: must satisfy 0 < s_max_chaser < width/2");
    if (!(c.r_touch >= 0.f) || !std::isfinite(c.r_touch) || c.r_touch > 1e6f) return fail(VG_EINVAL, "r_touch: must be in [0, 1e6]");
    if (!(c.w_prox >= 0.f) || !std::isfinite(c.w_prox)) return fail(VG_EINVAL, "w_prox: must be finite and >= 0");
  }
  if (!(c.c_collide > 0.f) || !std::isfinite(c.c_collide) || c.c_collide > 1e6f) return fail(VG_EINVAL, "c_collide: must be in (0, 1e6]");
  if (!(c.c_near > 0.f) || !std::isfinite(c.c_near) || c.c_near > 1e6f) return fail(VG_EINVAL, "c_near: must be in (0, 1e6]");
  if (!(c.d_peak > 2.f * c.d_r) || !(c.d_peak < c.d_v)) return fail(VG_EINVAL, "d_peak: must satisfy 2 d_r < d_peak < d_v (A5)");
  {
    // The reward is an int64 sum in 2^-32 units (A16b): every row's |reward| <= (N - 1) x
    // the largest per-pair magnitude must stay below 2^31 reward units.
    double mag = std::max((double)c.c_collide, (double)c.c_near);
    if (c.env == VG_ENV_TAG) mag = std::max((double)c.r_touch, (double)c.r_touch + (double)c.w_prox * std::max((double)c.c_collide, (double)c.c_near));
    if (mag * (double)(c.n_agents - 1) >= 2147483647.0)
      return fail(VG_EINVAL, "c_collide/c_near/r_touch/w_prox: (n_agents - 1) x max per-pair reward %g must be < 2^31 (fixed-point reward sum, A16b)", mag);
  }
  int g = c.grid;
  const double need = (double)c.d_v * (1.0 + std::ldexp(1.0, -12));
  if (g == 0) g = auto_grid(c.width, c.d_v);
  if (g < 3) return fail(VG_EINVAL, "grid: G = %d, need G >= 3 (3x3 stencil must not alias)", g);
  if ((double)c.width / g < need) return fail(VG_EINVAL, "grid: cell size L/G = %g must be >= d_v (1 + 2^-12) = %g (A16)", (double)c.width / g, need);
  if (c.vision == VG_VISION_RAY && (double)c.width / g < ((double)c.d_v + c.d_r) * (1.0 + std::ldexp(1.0, -12)))
    return fail(VG_EINVAL, "grid: ray vision needs cell size >= (d_v + d_r)(1 + 2^-12) (S:178)");
  if (c.vision == VG_VISION_RAY && !(2.0 * ((double)c.d_v + c.d_r) < c.width))
    return fail(VG_EINVAL, "d_v: ray vision needs d_v + d_r < width/2");
  if ((long long)g * g * c.n_replicas >= (1LL << 31)) return fail(VG_EINVAL, "grid: n_replicas * G^2 must be < 2^31");
  if (c.shard == VG_SHARD_SLAB) {
    if (c.world_size < 2) return fail(VG_EINVAL, "world_size: slab mode needs world_size >= 2");
    if (c.rank < 0 || c.rank >= c.world_size) return fail(VG_EINVAL, "rank: must satisfy 0 <= rank < world_size");
    if (c.n_replicas != 1) return fail(VG_EINVAL, "n_replicas: slab mode splits one world (n_replicas = 1)");
    if (g % c.world_size != 0) return fail(VG_EINVAL, "grid: slab mode needs world_size | G (G = %d)", g);
    if (g / c.world_size < 2) return fail(VG_EINVAL, "world_size: slab mode needs >= 2 cell columns per rank");
    const double move = (c.env == VG_ENV_TAG) ? std::max((double)c.s_max, (double)c.s_max_chaser) : (double)c.s_max;
    if (!(move < (double)c.width / g)) return fail(VG_EINVAL, "s_max: slab mode needs the largest move < cell size (one column per step)");
    if (c.halo_capacity < 0) return fail(VG_EINVAL, "halo_capacity: must be >= 0 (0 = auto)");
  }
  *grid_out = g;
  return VG_OK;
}

vg::Params derive(const vg_config& c, int g) {
  vg::Params P{};
  P.env = c.env;
  P.N = c.n_agents;
  P.R = c.n_replicas;
  P.G = g;
  P.G2 = g * g;
  P.v = c.v;
  P.channels = (c.env == VG_ENV_FLOCK) ? 1 : 2;
  P.view_slots = P.channels * c.v;
  P.obs_dim = P.view_slots + ((c.env == VG_ENV_FLOCK) ? 1 : 0);
  P.occ_words = (P.view_slots + 31) / 32;
  P.first_chaser = (c.env == VG_ENV_TAG) ? c.n_agents - c.n_chasers : c.n_agents;
  P.total = (long long)c.n_agents * c.n_replicas;
  // fp32 constants (A12): each is one correctly rounded fp32 operation on fp32 inputs.
  volatile float L = c.width;
  P.L = L;
  P.half_L = L * 0.5f;
  P.gs = (float)g / L;                              // RN32(G/L)  (A16)
  P.two_pi = (float)(2.0 * 3.14159265358979323846);  // RN32(2 pi)
  P.s_min = c.s_min;
  P.s_max = c.s_max;
  P.a_max = c.a_max;
  P.theta_max = c.theta_max;
  P.s_max_chaser = c.s_max_chaser;
  P.d_v = c.d_v;
  volatile float dv = c.d_v;
  P.dv2 = dv * dv;
  P.inv_dv = 1.0f / dv;
  P.two_dr = 2.0f * c.d_r;
  volatile float tdr = P.two_dr;
  P.contact2 = tdr * tdr;
  P.half_fov = 0.5f * c.fov;
  P.inv_fov = 1.0f / c.fov;
  P.fv = (float)c.v;
  P.c_collide = c.c_collide;
  P.d_peak = c.d_peak;
  P.k_rise = c.c_near / (c.d_peak - P.two_dr);
  P.k_fall = c.c_near / (c.d_v - c.d_peak);
  P.w_prox = c.w_prox;
  P.d_r = c.d_r;
  {
    volatile float reach = c.d_v + c.d_r;
    P.cand2 = reach * reach;
  }
  P.inv_w = (float)c.v / c.fov;
  P.b_rise = -P.k_rise * P.two_dr;
  P.nk_fall = -P.k_fall;
  P.b_fall = P.k_fall * c.d_v;
  P.fx_k_rise = P.k_rise * 4294967296.0f;
  P.fx_b_rise = P.b_rise * 4294967296.0f;
  P.fx_nk_fall = P.nk_fall * 4294967296.0f;
  P.fx_b_fall = P.b_fall * 4294967296.0f;
  P.fx_mcollide = -P.c_collide * 4294967296.0f;
  P.fx_cnear = c.c_near * 4294967296.0f;
  P.tent_sym = (VG_TENT_SYM && P.k_rise == P.k_fall) ? 1 : 0;
  P.half_v = 0.5f * (float)c.v;
  P.touch_fix = (long long)std::llrint((double)c.r_touch * 4294967296.0);
  P.cell = L / (float)g;
  P.inv_smax = 1.0f / c.s_max;
  P.win_r2 = (c.vision == VG_VISION_RAY) ? P.cand2 : P.dv2;
  // K4 windows only ever widen the candidate set: 1 % of the radius plus 2^-19 L covers the
  // fp32 rounding of the keys, of the pair test and the fuzz of the A16 cell boundaries.
  P.win_margin = 0.01f * std::sqrt(P.win_r2) + L * 1.9073486e-6f;
  return P;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Runs an entry point on the device the object was created on, restoring the caller's.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Record phase boundary `k` of the current profiled step (no-op when not profiling).
inline void prof_mark(vg_world* w, int k, cudaStream_t s) {
  if (w->prof_n < w->prof_max) cudaEventRecord(w->prof_ev[(size_t)w->prof_n * (VG_N_PHASES + 1) + k], s);
}

vg_status check_pending(const vg_world* w) {
  if (*reinterpret_cast<volatile uint32_t*>(w->err_flag))
    return fail(VG_ESTATE, "device-side state error pending; call vg_sync_errors for the agent index");
  return VG_OK;
}

vg_status launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(VG_ECUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return VG_OK;
}

// K4 work items (WorkList, appended by K3b / the fused bin): queries per item, chosen so a world has ~4 items per
// resident CTA when it is small (c1-c3) and whole cells (~54 queries at c5) when it is
// large; dense cells (clusters) are split into many items.
#ifndef VG_SLAB_BCHUNK
#define VG_SLAB_BCHUNK 0   // slab boundary-phase K4 chunk (8 measured 2.1x slower: per-CTA setup)
#endif
int sense_chunk_q(const vg_world* w) {
  const long long queries = w->slab ? (long long)w->P.N / w->cfg.world_size : w->P.total;
#ifndef VG_SENSE_ITEMS_PER_SLOT
#define VG_SENSE_ITEMS_PER_SLOT 4   // slab P = 2/4/8: 2 and 8 measured worse at one of them
#endif
  const long long slots = (long long)w->n_sm * vg::kSenseMinBlocks * VG_SENSE_ITEMS_PER_SLOT;
  long long q = (queries / slots) / 8 * 8;
#ifndef VG_SENSE_CHUNK_MAX
#define VG_SENSE_CHUNK_MAX 128
#endif
#ifndef VG_SENSE_CHUNK_MAX_SINGLE
#define VG_SENSE_CHUNK_MAX_SINGLE 64   // one large world (c5): 64 measured 0.6 % faster; c4 keeps 128
#endif
  const long long cap = (w->P.R == 1 && !w->slab) ? VG_SENSE_CHUNK_MAX_SINGLE : VG_SENSE_CHUNK_MAX;
  return (int)std::max(8LL, std::min(q, cap));
}

vg::WorkList work_list(vg_world* w) {
  vg::WorkList WL{};
  WL.item = w->work;
  WL.n = w->work_cnt;
  WL.chunk_q = sense_chunk_q(w);
  WL.lo = 0;                                              // slab: owned memory columns 0..W-1
  WL.hi = w->slab ? w->SL.W * w->P.G : w->n_cells;
  WL.G = w->P.G;
  WL.nb = w->slab ? w->SL.nb : 0;
  WL.chunk_qb = w->slab ? w->SL.chunk_qb : WL.chunk_q;
  for (int k = 0; k < 4; ++k) WL.bcol[k] = w->SL.bcol[k];
  return WL;
}

template <int ENV, bool INTEGRATE, bool BIN>
vg_status launch_k1(vg_world* w, float4* io, const float4* in, const float2* act, cudaStream_t s) {
  const long long n = w->P.total;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  vg::k_integrate_bin<ENV, INTEGRATE, BIN><<<blocks, 256, 0, s>>>(
      w->P, io, in, act, w->cell_id, w->slot, w->count, w->err_dev, w->err_flag,
      (BIN && w->gather_bin) ? w->work_cnt : nullptr);
  return launch_check("k_integrate_bin");
}

// Exclusive scan of the counts of cells [c0, c1) into cell_start[c0 .. c1] (re-zeroing the
// counts); `cont`: continue from cell_start[c0] (written by an earlier phase) instead of 0.
vg_status scan_cells(vg_world* w, cudaStream_t s, int c0 = 0, int c1 = -1, bool cont = false) {
  if (c1 < 0) c1 = w->n_cells;
  const int n = c1 - c0;
  uint32_t* cnt = w->count + c0;
  uint32_t* start = w->cell_start + c0;
  const uint32_t* base = cont ? start : nullptr;
  if (n <= vg::kScanSmallMax) {                 // (dynamic smem limit set at world creation)
    vg::k_scan_cells<<<1, 1024, (size_t)n * 4, s>>>(cnt, start, n, base);
    return launch_check("k_scan_cells");
  }
  const unsigned tiles = (unsigned)((n + vg::kScanTile - 1) / vg::kScanTile);
  vg::k_scan_tiles<<<tiles, 1024, 0, s>>>(cnt, n, w->tile_sum);
  if (vg_status st = launch_check("k_scan_tiles")) return st;
  vg::k_scan_apply<<<tiles, 1024, 0, s>>>(cnt, start, n, w->tile_sum, base);
  return launch_check("k_scan_apply");
}

template <int ENV, bool INTEGRATE>
vg_status launch_fused_bin(vg_world* w, float4* io, const float4* in, const float2* act,
                           cudaStream_t s) {
  VG_CUDA(cudaMemsetAsync(w->work_cnt, 0, sizeof(uint32_t), s));   // replica CTAs append items
  if (w->staged_bin == 1)       // persistent, shared-memory staged
    vg::k_replica_bin<ENV, INTEGRATE, 1><<<(unsigned)std::min(w->P.R, w->n_sm), vg::kRBThreads,
                                             vg::kRBStagedSmem, s>>>(
        w->P, io, in, act, w->cell_id, w->cell_start, w->sorted, w->perm, w->xo_rec, w->xo_perm,
        w->xo_xy, w->sub_tab, work_list(w), w->err_dev, w->err_flag);
  else if (w->staged_bin == 2)
    vg::k_replica_bin<ENV, INTEGRATE, 2><<<(unsigned)std::min(w->P.R, 2 * w->n_sm), vg::kRB2Threads,
                                             vg::kRBStaged2Smem, s>>>(
        w->P, io, in, act, w->cell_id, w->cell_start, w->sorted, w->perm, w->xo_rec, w->xo_perm,
        w->xo_xy, w->sub_tab, work_list(w), w->err_dev, w->err_flag);
  else
    vg::k_replica_bin<ENV, INTEGRATE, 0><<<w->P.R, vg::kRBThreads, 0, s>>>(
        w->P, io, in, act, w->cell_id, w->cell_start, w->sorted, w->perm, w->xo_rec, w->xo_perm,
        w->xo_xy, w->sub_tab, work_list(w), w->err_dev, w->err_flag);
  if (vg_status st = launch_check("k_replica_bin")) return st;
  w->binned = true;
  return VG_OK;
}

// K3b: one warp per cell, or one CTA per cell when the world has few cells.
#ifndef VG_CTA_SORT_CELLS_PER_SM
#define VG_CTA_SORT_CELLS_PER_SM 8
#endif
// Cells [c0, c1) (default: all), + the sentinel row at c1.
vg_status launch_cell_sort(vg_world* w, cudaStream_t s, int c0 = 0, int c1 = -1) {
  if (c1 < 0) c1 = w->n_cells;
  if (c1 - c0 <= (long long)VG_CTA_SORT_CELLS_PER_SM * w->n_sm) {
    vg::k_cell_sort_cta<<<(unsigned)(c1 - c0 + 1), vg::kCtaSortThreads, 0, s>>>(
        w->P, c1, w->slab ? 1 : 0, w->cell_start, w->tmp_rec, w->tmp_id, w->sorted,
        w->perm, w->xo_rec, w->xo_perm, w->xo_xy, w->sub_tab, work_list(w), w->slot, c0);
    return launch_check("k_cell_sort_cta");
  }
  const long long threads = (long long)(c1 - c0 + 1) * 32;   // + the sentinel row
  vg::k_cell_sort<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
      w->P, c1, w->slab ? 1 : 0, w->cell_start, w->tmp_rec, w->tmp_id, w->sorted,
      w->perm, w->xo_rec, w->xo_perm, w->xo_xy, w->sub_tab, work_list(w), w->slot, c0);
  return launch_check("k_cell_sort");
}

template <int ENV>
vg_status bin_rest(vg_world* w, const float4* state, cudaStream_t s, bool prof = false) {
  const long long n = w->P.total;
  if (w->gather_bin) {                 // K3g: K2 + K3 + K3b in one kernel (small worlds)
    vg::k_cell_gather<ENV><<<(unsigned)(w->n_cells + 1), vg::kGatherThreads, 0, s>>>(
        w->P, w->n_cells, state, w->cell_id, w->cell_start, w->sorted, w->perm, w->xo_rec,
        w->xo_perm, w->xo_xy, w->sub_tab, work_list(w));
    if (vg_status st = launch_check("k_cell_gather")) return st;
    if (prof) for (int k = 2; k <= 4; ++k) prof_mark(w, k, s);
    w->binned = true;
    return VG_OK;
  }
  if (vg_status st = scan_cells(w, s)) return st;
  if (prof) prof_mark(w, 2, s);
  vg::k_scatter<ENV><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      w->P, state, w->cell_id, w->slot, w->cell_start, w->tmp_rec, w->tmp_id, w->work_cnt);
  if (vg_status st = launch_check("k_scatter")) return st;
  if (prof) prof_mark(w, 3, s);
  if (vg_status st = launch_cell_sort(w, s)) return st;
  if (prof) prof_mark(w, 4, s);
  w->binned = true;
  return VG_OK;
}

vg::Outs to_outs(const vg_world* w, const vg_outputs* o) {
  vg::Outs r{};
  if (o) {
    r.obs = o->obs;
    r.reward = o->reward;
    r.n_neigh = o->n_neigh;
    r.n_collide = o->n_collide;
    r.n_touch = o->n_touch;
    r.occ = o->sector_occ;
    r.agent_id = o->agent_id;
  }
  const bool all = r.obs && r.reward && r.n_neigh && r.n_collide && r.occ &&
                   (w->P.env != vg::kTag || r.n_touch) && (!w->slab || r.agent_id);
  const long long rows = w->slab ? (long long)w->P.N : w->P.total;
  r.fast = (all && rows * (w->P.obs_dim + 1) < (1LL << 31)) ? 1 : 0;
  if (r.fast && w->P.occ_words == 4 && (reinterpret_cast<uintptr_t>(r.occ) & 15u) == 0) r.fast = 2;
  return r;
}

// K4's candidate reads hit L1: cap the shared-memory carve-out so the resident CTAs' shared
// memory leaves L1 room.  Set once per kernel instance.
#ifndef VG_SENSE_CARVEOUT
#define VG_SENSE_CARVEOUT 80     // 75-83: same; 86 (8 CTAs/SM, less L1) 1 % slower; 70 11 % slower
#endif
#ifndef VG_SENSE_CARVEOUT_RAY
#define VG_SENSE_CARVEOUT_RAY 86 // the ray instances keep a 1 KB ray table too: 80 gives 7 CTAs
#endif
template <typename K>
void sense_carveout(K* k, int pct) {
  if (pct >= 0) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

template <int ENV, bool VISION, bool SLAB>
void sense_carveouts() {
  sense_carveout(vg::k_sense<ENV, VISION, SLAB, true, false>, VG_SENSE_CARVEOUT_RAY);
  sense_carveout(vg::k_sense<ENV, VISION, SLAB, false, false>, VG_SENSE_CARVEOUT);
  if (VISION) {
    sense_carveout(vg::k_sense<ENV, VISION, SLAB, false, VISION>, VG_SENSE_CARVEOUT);
    if constexpr (VISION && !SLAB) sense_carveout(vg::k_sense<ENV, VISION, SLAB, false, 2>, VG_SENSE_CARVEOUT);
    sense_carveout(vg::k_sense<ENV, VISION, SLAB, true, VISION>, VG_SENSE_CARVEOUT_RAY);
  }
}

// K4's sector pass with the paper's default constants as immediates (vg::sense_defaults):
// only when the world's derived constants are bitwise those (A12: the same fp32 ops).
#ifndef VG_SENSE_DEFAULTS
#define VG_SENSE_DEFAULTS 1
#endif
template <int ENV>
bool sense_defaults_match(const vg::Params& P) {
  const vg::SenseConst a = vg::sense_const(P), b = vg::sense_defaults<ENV>();
  return VG_SENSE_DEFAULTS && std::memcmp(&a, &b, sizeof(a)) == 0;
}

// Function attributes apply to the current device: set them for every world created.
void set_kernel_attributes() {
  cudaFuncSetAttribute(vg::k_scan_cells, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       vg::kScanSmallMax * 4);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kFlock, true, 1>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStagedSmem);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kFlock, false, 1>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStagedSmem);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kTag, true, 1>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStagedSmem);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kTag, false, 1>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStagedSmem);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kFlock, true, 2>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStaged2Smem);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kFlock, false, 2>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStaged2Smem);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kTag, true, 2>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStaged2Smem);
  cudaFuncSetAttribute(vg::k_replica_bin<vg::kTag, false, 2>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kRBStaged2Smem);
  sense_carveouts<vg::kFlock, true, false>();
  sense_carveouts<vg::kFlock, true, true>();
  sense_carveouts<vg::kTag, true, false>();
  sense_carveouts<vg::kTag, true, true>();
  sense_carveouts<vg::kFlock, false, false>();
  sense_carveouts<vg::kTag, false, false>();
  sense_carveouts<vg::kFlock, false, true>();
  sense_carveouts<vg::kTag, false, true>();
}

template <int ENV, bool VISION, bool SLAB>
void sense_kernel(vg_world* w, int cells, const vg::Outs& O, cudaStream_t s) {
  const int cq = sense_chunk_q(w);
  // one CTA per sensed cell + an upper bound on the overflow items (surplus CTAs exit)
  const long long queries = w->slab ? (long long)w->P.N : w->P.total;
  const int cq_min = w->slab ? std::min(cq, w->SL.chunk_qb) : cq;
  const unsigned grid = (unsigned)(cells + std::min<long long>(queries / cq_min + 1, w->work_cap));
  if (w->cfg.vision == VG_VISION_RAY && VISION && w->sense_def)
    vg::k_sense<ENV, VISION, SLAB, true, VISION><<<grid, vg::kSenseWarps * 32, 0, s>>>(
        w->P, w->cell_start, w->xo_rec, w->xo_xy, w->xo_perm, O, w->SL, w->ray_dir, w->sub_tab,
        w->work, w->work_cnt, cq, cells);
  else if (w->cfg.vision == VG_VISION_RAY)
    vg::k_sense<ENV, VISION, SLAB, true, false><<<grid, vg::kSenseWarps * 32, 0, s>>>(
        w->P, w->cell_start, w->xo_rec, w->xo_xy, w->xo_perm, O, w->SL, w->ray_dir, w->sub_tab,
        w->work, w->work_cnt, cq, cells);
  else if (VISION && w->sense_def && !SLAB && w->P.R == 1)      // one large world
    vg::k_sense<ENV, VISION, SLAB, false, (VISION && !SLAB) ? 2 : 0><<<grid, vg::kSenseWarps * 32, 0, s>>>(
        w->P, w->cell_start, w->xo_rec, w->xo_xy, w->xo_perm, O, w->SL, w->ray_dir, w->sub_tab,
        w->work, w->work_cnt, cq, cells);
  else if (VISION && w->sense_def)
    vg::k_sense<ENV, VISION, SLAB, false, VISION><<<grid, vg::kSenseWarps * 32, 0, s>>>(
        w->P, w->cell_start, w->xo_rec, w->xo_xy, w->xo_perm, O, w->SL, w->ray_dir, w->sub_tab,
        w->work, w->work_cnt, cq, cells);
  else
    vg::k_sense<ENV, VISION, SLAB, false, false><<<grid, vg::kSenseWarps * 32, 0, s>>>(
        w->P, w->cell_start, w->xo_rec, w->xo_xy, w->xo_perm, O, w->SL, w->ray_dir, w->sub_tab,
        w->work, w->work_cnt, cq, cells);
}

enum { kSlabInterior = 0, kSlabBoundary = 1, kSlabAll = 2 };   // slab binning / sensing phases

// Slab mode: the owned cells K4 senses in one phase (memory columns, vg::Slab): all
// owned columns [0, W); the inner interior l = 3..W-2 = memory [1, W-3) while the halo is in
// flight; the rest (memory 0, W-3, W-2, W-1; all of [0, W) when W <= 4) after it.
vg::Slab slab_sense_set(const vg_world* w, int phase) {
  vg::Slab SL = w->SL;
  const int W = SL.W;
  SL.snl = 0;
  if (phase == kSlabAll) { SL.sc0 = 0; SL.snc = W; }
  else if (phase == kSlabInterior) { SL.sc0 = 1; SL.snc = std::max(0, W - 4); }
  else if (W <= 4) { SL.sc0 = 0; SL.snc = W; }
  else { SL.snl = 4; SL.scol[0] = 0; SL.scol[1] = W - 3; SL.scol[2] = W - 2; SL.scol[3] = W - 1; }
  return SL;
}

template <bool VISION>
vg_status launch_sense(vg_world* w, const vg_outputs* outs, cudaStream_t s,
                       int slab_phase = kSlabAll) {
  const vg::Outs O = to_outs(w, outs);
  if (w->slab) {                      // owned cells only (this phase's memory columns)
    const vg::Slab saved = w->SL;
    w->SL = slab_sense_set(w, slab_phase);
    const int cells = (w->SL.snl ? w->SL.snl : w->SL.snc) * w->P.G;
    if (cells > 0) {
      if (w->P.env == vg::kFlock) sense_kernel<vg::kFlock, VISION, true>(w, cells, O, s);
      else sense_kernel<vg::kTag, VISION, true>(w, cells, O, s);
    }
    w->SL = saved;
    return launch_check("k_sense(slab)");
  }
  if (w->P.env == vg::kFlock) sense_kernel<vg::kFlock, VISION, false>(w, w->n_cells, O, s);
  else sense_kernel<vg::kTag, VISION, false>(w, w->n_cells, O, s);
  return launch_check("k_sense");
}

unsigned stride_blocks(size_t n) {
  return (unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 148 * 8));   // grid-stride
}

// Bin the slab's local set (owned + ghosts) on the column-major local grid (memory column
// order, vg::Slab), one phase at a time: kSlabInterior = memory columns [0, W-2) (nothing
// there can arrive from a neighbour), kSlabBoundary = [W-2, W+2) after the halo arrived
// (continuing the interior's cell_start and work items), kSlabAll = both at once.
template <int ENV>
vg_status slab_bin(vg_world* w, cudaStream_t s, int phase = kSlabAll) {
  const int nA = (w->SL.W - 2) * w->P.G;
  if (phase == kSlabInterior && nA == 0) {         // W = 2: no interior columns
    VG_CUDA(cudaMemsetAsync(w->work_cnt, 0, sizeof(uint32_t), s));
    VG_CUDA(cudaMemsetAsync(w->cell_start, 0, sizeof(uint32_t), s));
    VG_CUDA(cudaMemsetAsync(w->sub_tab, 0, sizeof(uint32_t), s));
    return VG_OK;
  }
  const unsigned nb = stride_blocks(w->SB.cap_loc);
  if (phase == kSlabAll) {     // (the step phases' keys were computed by begin / unpack)
    vg::k_slab_keys<<<nb, 256, 0, s>>>(w->P, w->SL, w->SB, w->cell_id, w->slot, w->count, phase);
    if (vg_status st = launch_check("k_slab_keys")) return st;
  }
  const int c0 = (phase == kSlabBoundary) ? nA : 0;
  const int c1 = (phase == kSlabInterior) ? nA : w->n_cells;
  if (vg_status st = scan_cells(w, s, c0, c1, phase == kSlabBoundary)) return st;
  vg::k_slab_scatter<ENV><<<nb, 256, 0, s>>>(w->P, w->SB, w->cell_id, w->slot, w->cell_start,
                                              w->tmp_rec, w->tmp_id, w->work_cnt,
                                              phase != kSlabBoundary, (uint32_t)c0, (uint32_t)c1);
  if (vg_status st = launch_check("k_slab_scatter")) return st;
  if (vg_status st = launch_cell_sort(w, s, c0, c1)) return st;
  if (phase != kSlabInterior) w->binned = true;
  return VG_OK;
}

vg_status need_slab(const vg_world* w, bool slab, const char* fn) {
  if (!w) return fail(VG_EINVAL, "%s: world NULL", fn);
  if (w->slab != slab)
    return fail(VG_EINVAL, slab ? "%s: needs a slab-mode world" : "%s: not available in slab mode (use vg_slab_*)", fn);
  return VG_OK;
}

template <typename T>
vg_status dalloc(vg_world* w, T** p, size_t n) {
  const size_t bytes = n * sizeof(T);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes > 0 ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(VG_ENOMEM, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
  }
  w->scratch_bytes += bytes;
  return VG_OK;
}

}  // namespace

extern "C" {

int32_t vg_abi_version(void) { return VG_ABI_VERSION; }

const char* vg_last_error(void) { return g_err; }

#ifndef VG_RB_STAGED_DEFAULT
#define VG_RB_STAGED_DEFAULT 1       // many replicas: the staged fused bin, MODE 1
#endif
#ifndef VG_FUSED_SINGLE_MAX
#define VG_FUSED_SINGLE_MAX 1024     // few replicas: the fused bin only for tiny worlds
#endif
#ifndef VG_GATHER_BIN
#define VG_GATHER_BIN 1
#endif
vg_status vg_world_create(const vg_config* cfg, vg_world** out) {
  g_err[0] = 0;
  if (!out) return fail(VG_EINVAL, "out: NULL");
  *out = nullptr;
  if (!cfg) return fail(VG_EINVAL, "cfg: NULL");
  int g = 0;
  if (vg_status st = validate(*cfg, &g)) return st;
  vg_world* w = new (std::nothrow) vg_world();
  if (!w) return fail(VG_ENOMEM, "host allocation failed");
  w->cfg = *cfg;
  w->P = derive(*cfg, g);
  {
    const char* ng = std::getenv("VG_NO_GRAPH");
    w->graphs_enabled = !(ng && ng[0] && ng[0] != '0');
  }
  w->n_cells = g * g * cfg->n_replicas;
  cudaGetDevice(&w->device);
  cudaDeviceGetAttribute(&w->n_sm, cudaDevAttrMultiProcessorCount, w->device);
  set_kernel_attributes();                         // per device (the current one)
  // Binning path.  K3g (per-cell gather) for worlds with few cells and N <= 16,384 unless
  // they are many replicas, which take the one-CTA-per-replica fused bin; the fused bin
  // also for tiny worlds K3g cannot take; the 4-kernel path otherwise.
  const bool gather_ok = VG_GATHER_BIN && cfg->shard == VG_SHARD_REPLICA &&
                         (long long)g * g * cfg->n_replicas <= 8LL * w->n_sm &&
                         cfg->n_agents <= vg::kGatherMaxN;
  w->fused_bin = cfg->shard == VG_SHARD_REPLICA && g * g <= vg::kRBMaxCells &&
                 cfg->n_agents <= vg::kRBMaxAgents &&
                 (cfg->n_replicas >= 64 ||
                  (cfg->n_agents <= VG_FUSED_SINGLE_MAX && !gather_ok));
  {                                // VG_RB_STAGED=0: the one-CTA-per-replica fused bin (tests)
    const char* sg = std::getenv("VG_RB_STAGED");
    const bool ok = w->fused_bin && cfg->n_agents <= vg::kRBStagedMax && cfg->n_replicas >= w->n_sm;
    w->staged_bin = ok ? ((sg && sg[0] >= '0' && sg[0] <= '2') ? sg[0] - '0' : VG_RB_STAGED_DEFAULT) : 0;
  }
  {                                // VG_SENSE_GENERIC=1: always the generic instance (tests)
    const char* gen = std::getenv("VG_SENSE_GENERIC");
    w->sense_def = !(gen && gen[0] && gen[0] != '0') &&
                   (w->P.env == vg::kFlock ? sense_defaults_match<vg::kFlock>(w->P)
                                           : sense_defaults_match<vg::kTag>(w->P));
  }
  w->gather_bin = gather_ok && !w->fused_bin;
  size_t n = (size_t)w->P.total;
  vg_status st = VG_OK;
  if (cfg->shard == VG_SHARD_SLAB) {
    const int P = cfg->world_size, W = g / P;
    w->slab = true;
    w->SL = vg::Slab{cfg->rank * W, (cfg->rank + 1) * W, W, (W + 2) * g};
    // the boundary phase's columns: memory 0, W-3, W-2, W-1 (W >= 5), with
    // their own K4 chunk size VG_SLAB_BCHUNK (0: the same as every other cell)
    if (W >= 5 && VG_SLAB_BCHUNK > 0) {
      w->SL.nb = 4;
      w->SL.bcol[0] = 0; w->SL.bcol[1] = W - 3; w->SL.bcol[2] = W - 2; w->SL.bcol[3] = W - 1;
    }
    w->SL.chunk_qb = VG_SLAB_BCHUNK > 0 ? VG_SLAB_BCHUNK : sense_chunk_q(w);
    w->n_cells = w->SL.n_lcells;
    w->left = (cfg->rank + P - 1) % P;
    w->right = (cfg->rank + 1) % P;
    const long long col = ((long long)cfg->n_agents + g - 1) / g;
    const uint32_t cap_msg = cfg->halo_capacity > 0 ? (uint32_t)cfg->halo_capacity
                                                    : (uint32_t)std::max(1024LL, 4 * col + 256);
    w->SB.cap_msg = cap_msg;
    w->SB.cap_loc = (uint32_t)(cfg->n_agents + 2ull * cap_msg);
    w->msg_bytes = 16 + 20 * (size_t)cap_msg;
    n = w->SB.cap_loc;
    if (!st) st = dalloc(w, &w->loc_n, 1);
    if (!st) st = dalloc(w, &w->slab_ovf, 1);
    if (!st) st = dalloc(w, &w->SB.loc_rec, n);
    if (!st) st = dalloc(w, &w->SB.loc_id, n);
    if (!st) st = dalloc(w, &w->msg, 4 * w->msg_bytes);
    if (!st) {
      w->SB.n_loc = w->loc_n;
      w->SB.overflow = w->slab_ovf;
      w->SB.send_l = w->msg;
      w->SB.send_r = w->msg + w->msg_bytes;
      w->SB.recv_l = w->msg + 2 * w->msg_bytes;
      w->SB.recv_r = w->msg + 3 * w->msg_bytes;
      cudaError_t e = cudaMemset(w->msg, 0, 4 * w->msg_bytes);
      if (e == cudaSuccess) e = cudaMemset(w->slab_ovf, 0, sizeof(uint32_t));
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&w->comm_stream, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->ev_fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w->ev_join, cudaEventDisableTiming);
      if (e != cudaSuccess) st = fail(VG_ECUDA, "slab init: %s", cudaGetErrorString(e));
    }
    if (!st && cfg->nccl_unique_id) {
      // The world owns its communicator: a collective call, every rank of
      // the slab group creates its world at the same time.
      const NcclApi* nc = nccl_api();
      if (!nc) {
        st = fail(VG_ENCCL, "vg_world_create: %s", nccl_err());
      } else {
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
        ncclResult_t r = nc->CommInitRank(&w->comm, cfg->world_size, id, cfg->rank);
        if (r != ncclSuccess) {
          w->comm = nullptr;
          st = fail(VG_ENCCL, "ncclCommInitRank(%d of %d): %s", cfg->rank, cfg->world_size,
                    nc->GetErrorString(r));
        }
      }
    }
  }
  if (!st) st = dalloc(w, &w->count, w->n_cells);
  if (!st) st = dalloc(w, &w->tile_sum, w->n_cells / vg::kScanTile + 1);
  if (!st) st = dalloc(w, &w->cell_start, w->n_cells + 1);
  if (!st) st = dalloc(w, &w->cell_id, n);
  if (!st) st = dalloc(w, &w->slot, n);
  if (!st && w->slab) {                // k_slab_begin / k_slab_unpack write the binning keys
    w->SB.cell_id = w->cell_id;
    w->SB.slot = w->slot;
    w->SB.count = w->count;
  }
  if (!st) st = dalloc(w, &w->tmp_id, n);
  if (!st) st = dalloc(w, &w->perm, n);
  if (!st) st = dalloc(w, &w->tmp_rec, n);
  if (!st) st = dalloc(w, &w->sorted, n);
  if (!st) st = dalloc(w, &w->xo_rec, n);
  if (!st) st = dalloc(w, &w->xo_perm, n);
  if (!st) st = dalloc(w, &w->xo_xy, n + vg::kSensePad);   // padded: unpredicated K4 loads
  if (!st) st = dalloc(w, &w->sub_tab, ((size_t)w->n_cells + 1) * vg::kSub);
  if (!st) {
    w->work_cap = (long long)w->n_cells + (long long)n / 8 + 1;       // chunk_q >= 8
    st = dalloc(w, &w->work, (size_t)w->work_cap);
  }
  if (!st) st = dalloc(w, &w->work_cnt, 1);
  if (!st) st = dalloc(w, &w->ray_dir, vg::kMaxViewSlots);
  if (!st) {
    // psi_k = -fov/2 + (k + 1/2) fov/v (orientation A3), in double, rounded once
    float2 tab[vg::kMaxViewSlots] = {};
    for (int k = 0; k < cfg->v; ++k) {
      const double psi = -0.5 * (double)cfg->fov + (k + 0.5) * (double)cfg->fov / cfg->v;
      tab[k] = make_float2((float)std::cos(psi), (float)std::sin(psi));
    }
    cudaError_t e = cudaMemcpy(w->ray_dir, tab, sizeof(tab), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) st = fail(VG_ECUDA, "ray table: %s", cudaGetErrorString(e));
  }
  if (!st) st = dalloc(w, &w->act_dev, n);
  if (!st) st = dalloc(w, &w->err_dev, 1);
  if (!st) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&w->err_flag), sizeof(uint32_t),
                                  cudaHostAllocMapped);
    if (e != cudaSuccess) st = fail(VG_ECUDA, "cudaHostAlloc(flag): %s", cudaGetErrorString(e));
  }
  if (!st) {
    *w->err_flag = 0;
    const unsigned long long none = ~0ull;
    cudaError_t e = cudaMemset(w->count, 0, sizeof(uint32_t) * w->n_cells);
    if (e == cudaSuccess) e = cudaMemcpy(w->err_dev, &none, sizeof(none), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) st = fail(VG_ECUDA, "world init: %s", cudaGetErrorString(e));
  }
  if (st) {
    vg_world_destroy(w);
    return st;
  }
  *out = w;
  return VG_OK;
}

void vg_world_destroy(vg_world* w) {
  if (!w) return;
  for (auto& g : w->graphs) cudaGraphExecDestroy(g.exec);
  if (w->cap_stream) cudaStreamDestroy(w->cap_stream);
  for (cudaEvent_t e : w->prof_ev) cudaEventDestroy(e);
  cudaFree(w->count);
  cudaFree(w->tile_sum);
  cudaFree(w->cell_start);
  cudaFree(w->cell_id);
  cudaFree(w->slot);
  cudaFree(w->tmp_id);
  cudaFree(w->perm);
  cudaFree(w->tmp_rec);
  cudaFree(w->sorted);
  cudaFree(w->xo_rec);
  cudaFree(w->xo_perm);
  cudaFree(w->xo_xy);
  cudaFree(w->sub_tab);
  cudaFree(w->work);
  cudaFree(w->work_cnt);
  cudaFree(w->ray_dir);
  cudaFree(w->act_dev);
  cudaFree(w->err_dev);
  cudaFree(w->loc_n);
  cudaFree(w->slab_ovf);
  cudaFree(w->SB.loc_rec);
  cudaFree(w->SB.loc_id);
  cudaFree(w->msg);
  if (w->comm) nccl_api()->CommDestroy(w->comm);
  if (w->comm_stream) cudaStreamDestroy(w->comm_stream);
  if (w->ev_fork) cudaEventDestroy(w->ev_fork);
  if (w->ev_join) cudaEventDestroy(w->ev_join);
  if (w->err_flag) cudaFreeHost(w->err_flag);
  delete w;
}

vg_status vg_world_query(const vg_world* w, vg_world_info* info) {
  if (!w || !info) return fail(VG_EINVAL, "world/info: NULL");
  info->grid = w->P.G;
  info->cell_size = w->cfg.width / (float)w->P.G;
  info->n_cells = w->n_cells;
  info->obs_dim = w->P.obs_dim;
  info->channels = w->P.channels;
  info->occ_words = w->P.occ_words;
  info->total_agents = w->P.total;
  info->scratch_bytes = (int64_t)w->scratch_bytes;
  const int scan_k = (w->n_cells > vg::kScanSmallMax) ? 2 : 1;
  info->sense_defaults = w->sense_def;
  info->kernels_per_step = w->slab ? 6 + scan_k
                                   : (w->fused_bin ? 2 : (w->gather_bin ? 3 : 4 + scan_k));
  return VG_OK;
}

vg_status vg_bin(vg_world* w, const float* state, void* stream) {
  NvtxRange nvtx_("vg_bin");
  if (!w || !state) return fail(VG_EINVAL, "world/state: NULL");
  if (vg_status st = need_slab(w, false, "vg_bin")) return st;
  DeviceGuard dg_(w->device);
  if (vg_status st = check_pending(w)) return st;
  cudaStream_t s = as_stream(stream);
  const float4* in = reinterpret_cast<const float4*>(state);
  if (w->fused_bin)
    return (w->P.env == vg::kFlock) ? launch_fused_bin<vg::kFlock, false>(w, nullptr, in, nullptr, s)
                                    : launch_fused_bin<vg::kTag, false>(w, nullptr, in, nullptr, s);
  if (w->P.env == vg::kFlock) {
    if (vg_status st = launch_k1<vg::kFlock, false, true>(w, nullptr, in, nullptr, s)) return st;
    return bin_rest<vg::kFlock>(w, in, s);
  }
  if (vg_status st = launch_k1<vg::kTag, false, true>(w, nullptr, in, nullptr, s)) return st;
  return bin_rest<vg::kTag>(w, in, s);
}

vg_status vg_sense(vg_world* w, const vg_outputs* outs, void* stream) {
  NvtxRange nvtx_("vg_sense");
  if (!w || !outs) return fail(VG_EINVAL, "world/outs: NULL");
  if (!w->binned) return fail(VG_EINVAL, "vg_sense: no binned state (call vg_bin or vg_step first)");
  DeviceGuard dg_(w->device);
  if (vg_status st = check_pending(w)) return st;
  return launch_sense<true>(w, outs, as_stream(stream));
}

vg_status vg_sense_columns(vg_world* w, const vg_outputs* outs, int32_t col_lo, int32_t col_hi,
                           void* stream) {
  NvtxRange nvtx_("vg_sense_columns");
  if (!w || !outs) return fail(VG_EINVAL, "world/outs: NULL");
  if (vg_status st = need_slab(w, false, "vg_sense_columns")) return st;
  if (w->P.R != 1) return fail(VG_EINVAL, "vg_sense_columns: needs n_replicas = 1");
  if (col_lo < 0 || col_hi > w->P.G || col_lo >= col_hi)
    return fail(VG_EINVAL, "vg_sense_columns: need 0 <= col_lo < col_hi <= G (G = %d)", w->P.G);
  if (!w->binned) return fail(VG_EINVAL, "vg_sense_columns: no binned state (call vg_bin or vg_step first)");
  DeviceGuard dg_(w->device);
  if (vg_status st = check_pending(w)) return st;
  const vg::Slab saved = w->SL;
  w->SL.sc0 = col_lo;
  w->SL.snc = col_hi - col_lo;
  w->SL.snl = 0;
  const vg::Outs O = to_outs(w, outs);
  const int cells = (col_hi - col_lo) * w->P.G;
  if (w->P.env == vg::kFlock) sense_kernel<vg::kFlock, true, false>(w, cells, O, as_stream(stream));
  else sense_kernel<vg::kTag, true, false>(w, cells, O, as_stream(stream));
  w->SL = saved;
  return launch_check("k_sense(columns)");
}

vg_status vg_reward(vg_world* w, const vg_outputs* outs, void* stream) {
  NvtxRange nvtx_("vg_reward");
  if (!w || !outs) return fail(VG_EINVAL, "world/outs: NULL");
  if (!w->binned) return fail(VG_EINVAL, "vg_reward: no binned state (call vg_bin or vg_step first)");
  DeviceGuard dg_(w->device);
  if (vg_status st = check_pending(w)) return st;
  vg_outputs o = *outs;
  o.obs = nullptr;
  o.sector_occ = nullptr;
  return launch_sense<false>(w, &o, as_stream(stream));
}

vg_status vg_integrate(vg_world* w, float* state, const float* actions, void* stream) {
  NvtxRange nvtx_("vg_integrate");
  if (!w || !state || !actions) return fail(VG_EINVAL, "world/state/actions: NULL");
  if (vg_status st = need_slab(w, false, "vg_integrate")) return st;
  DeviceGuard dg_(w->device);
  if (vg_status st = check_pending(w)) return st;
  cudaStream_t s = as_stream(stream);
  float4* io = reinterpret_cast<float4*>(state);
  const float2* a = reinterpret_cast<const float2*>(actions);
  w->binned = false;   // the binned snapshot no longer matches state
  if (w->P.env == vg::kFlock) return launch_k1<vg::kFlock, true, false>(w, io, nullptr, a, s);
  return launch_k1<vg::kTag, true, false>(w, io, nullptr, a, s);
}

namespace {

vg_status launch_step(vg_world* w, float4* io, const float2* a, const vg_outputs* outs,
                      cudaStream_t s) {
  prof_mark(w, 0, s);
  if (w->fused_bin) {
    vg_status st = (w->P.env == vg::kFlock) ? launch_fused_bin<vg::kFlock, true>(w, io, nullptr, a, s)
                                            : launch_fused_bin<vg::kTag, true>(w, io, nullptr, a, s);
    if (st) return st;
    for (int k = 1; k <= 4; ++k) prof_mark(w, k, s);
    st = launch_sense<true>(w, outs, s);
    prof_mark(w, 5, s);
    return st;
  }
  if (w->P.env == vg::kFlock) {
    if (vg_status st = launch_k1<vg::kFlock, true, true>(w, io, nullptr, a, s)) return st;
    prof_mark(w, 1, s);
    if (vg_status st = bin_rest<vg::kFlock>(w, io, s, true)) return st;
  } else {
    if (vg_status st = launch_k1<vg::kTag, true, true>(w, io, nullptr, a, s)) return st;
    prof_mark(w, 1, s);
    if (vg_status st = bin_rest<vg::kTag>(w, io, s, true)) return st;
  }
  vg_status st = launch_sense<true>(w, outs, s);
  prof_mark(w, 5, s);
  return st;
}

bool same_outs(const vg_outputs& a, const vg_outputs& b) {
  return a.obs == b.obs && a.reward == b.reward && a.n_neigh == b.n_neigh &&
         a.n_collide == b.n_collide && a.n_touch == b.n_touch && a.sector_occ == b.sector_occ &&
         a.agent_id == b.agent_id;
}

// Launch the kernel sequence `launch` as a cached CUDA graph keyed by (k1, k2, outs).
extern "C++" template <typename F>
vg_status cached_graph(vg_world* w, const void* k1, const void* k2, const vg_outputs* outs,
                       cudaStream_t s, const char* what, F&& launch) {
  for (auto& g : w->graphs) {
    if (g.state == k1 && g.actions == k2 && same_outs(g.outs, *outs)) {
      g.last_use = ++w->graph_clock;
      VG_CUDA(cudaGraphLaunch(g.exec, s));
      w->binned = true;
      return VG_OK;
    }
  }
  if (!w->cap_stream) VG_CUDA(cudaStreamCreateWithFlags(&w->cap_stream, cudaStreamNonBlocking));
  VG_CUDA(cudaStreamBeginCapture(w->cap_stream, cudaStreamCaptureModeThreadLocal));
  vg_status st = launch(w->cap_stream);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(w->cap_stream, &graph);
  if (st) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return fail(VG_ECUDA, "%s graph capture: %s", what, cudaGetErrorString(e));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(VG_ECUDA, "%s graph instantiate: %s", what, cudaGetErrorString(e));
  if (w->graphs.size() >= 16) {                     // evict the least recently used
    size_t lru = 0;
    for (size_t i = 1; i < w->graphs.size(); ++i)
      if (w->graphs[i].last_use < w->graphs[lru].last_use) lru = i;
    cudaGraphExecDestroy(w->graphs[lru].exec);
    w->graphs.erase(w->graphs.begin() + lru);
  }
  w->graphs.push_back({k1, k2, *outs, exec, ++w->graph_clock});
  VG_CUDA(cudaGraphLaunch(exec, s));
  w->binned = true;
  return VG_OK;
}

vg_status step_graph(vg_world* w, float4* io, const float2* a, const vg_outputs* outs,
                     cudaStream_t s) {
  return cached_graph(w, io, a, outs, s, "vg_step",
                      [&](cudaStream_t cs) { return launch_step(w, io, a, outs, cs); });
}

// Graphs are used when enabled, not profiling, and the caller's stream is not capturing.
bool graph_ok(vg_world* w, cudaStream_t s) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
    cudaGetLastError();
    cap = cudaStreamCaptureStatusActive;            // unknown: stay on the eager path
  }
  return w->graphs_enabled && w->prof_n >= w->prof_max && cap == cudaStreamCaptureStatusNone;
}

}  // namespace

vg_status vg_step(vg_world* w, float* state, const float* actions, const vg_outputs* outs,
                  void* stream) {
  NvtxRange nvtx_("vg_step");
  if (!w || !state || !actions || !outs) return fail(VG_EINVAL, "world/state/actions/outs: NULL");
  if (vg_status st = need_slab(w, false, "vg_step")) return st;
  DeviceGuard dg_(w->device);
  if (vg_status st = check_pending(w)) return st;
  cudaStream_t s = as_stream(stream);
  float4* io = reinterpret_cast<float4*>(state);
  const float2* a = reinterpret_cast<const float2*>(actions);
  if (graph_ok(w, s)) return step_graph(w, io, a, outs, s);
  vg_status st = launch_step(w, io, a, outs, s);
  if (w->prof_n < w->prof_max) ++w->prof_n;
  return st;
}

vg_status vg_step_host(vg_world* w, float* state, const float* actions_host,
                       const vg_outputs* outs, float* reward_host, void* stream) {
  NvtxRange nvtx_("vg_step_host");
  if (!w || !state || !actions_host || !outs) return fail(VG_EINVAL, "world/state/actions_host/outs: NULL");
  DeviceGuard dg_(w->device);
  if (reward_host && !outs->reward) return fail(VG_EINVAL, "reward_host: needs outs->reward");
  cudaStream_t s = as_stream(stream);
  VG_CUDA(cudaMemcpyAsync(w->act_dev, actions_host, sizeof(float2) * (size_t)w->P.total,
                          cudaMemcpyHostToDevice, s));
  if (vg_status st = vg_step(w, state, reinterpret_cast<const float*>(w->act_dev), outs, stream)) return st;
  if (reward_host)
    VG_CUDA(cudaMemcpyAsync(reward_host, outs->reward, sizeof(float) * (size_t)w->P.total,
                            cudaMemcpyDeviceToHost, s));
  return VG_OK;
}

vg_status vg_get_bins(const vg_world* w, const uint32_t** cell_id, const uint32_t** cell_start,
                      const uint32_t** perm, const float** sorted) {
  if (!w) return fail(VG_EINVAL, "world: NULL");
  if (!w->binned) return fail(VG_EINVAL, "vg_get_bins: no binned state");
  if (cell_id) *cell_id = w->cell_id;
  if (cell_start) *cell_start = w->cell_start;
  if (perm) *perm = w->perm;
  if (sorted) *sorted = reinterpret_cast<const float*>(w->sorted);
  return VG_OK;
}

vg_status vg_slab_plan(int32_t grid, int32_t world_size, int32_t rank, int32_t* plan) {
  if (!plan || world_size < 2 || rank < 0 || rank >= world_size || grid % world_size ||
      grid / world_size < 2)
    return fail(VG_EINVAL, "vg_slab_plan: need world_size >= 2, 0 <= rank < world_size, world_size | grid, grid/world_size >= 2");
  const int W = grid / world_size;
  plan[0] = rank * W;
  plan[1] = (rank + 1) * W;
  plan[2] = (rank + world_size - 1) % world_size;
  plan[3] = (rank + 1) % world_size;
  return VG_OK;
}

vg_status vg_slab_load(vg_world* w, const float* state_global, void* stream) {
  NvtxRange nvtx_("vg_slab_load");
  if (vg_status st = need_slab(w, true, "vg_slab_load")) return st;
  DeviceGuard dg_(w->device);
  if (!state_global) return fail(VG_EINVAL, "state_global: NULL");
  if (vg_status st = check_pending(w)) return st;
  cudaStream_t s = as_stream(stream);
  VG_CUDA(cudaMemsetAsync(w->loc_n, 0, sizeof(uint32_t), s));
  const float4* st4 = reinterpret_cast<const float4*>(state_global);
  const unsigned nb = stride_blocks((size_t)w->P.N);
  if (w->P.env == vg::kFlock) {
    vg::k_slab_load<vg::kFlock><<<nb, 256, 0, s>>>(w->P, w->SL, w->SB, st4, w->err_dev, w->err_flag);
    if (vg_status st = launch_check("k_slab_load")) return st;
    return slab_bin<vg::kFlock>(w, s);
  }
  vg::k_slab_load<vg::kTag><<<nb, 256, 0, s>>>(w->P, w->SL, w->SB, st4, w->err_dev, w->err_flag);
  if (vg_status st = launch_check("k_slab_load")) return st;
  return slab_bin<vg::kTag>(w, s);
}

namespace {
vg_status slab_begin_launch(vg_world* w, const float2* a, cudaStream_t s) {
  prof_mark(w, 0, s);
  VG_CUDA(cudaMemsetAsync(w->loc_n, 0, sizeof(uint32_t), s));
  VG_CUDA(cudaMemsetAsync(w->SB.send_l, 0, 16, s));
  VG_CUDA(cudaMemsetAsync(w->SB.send_r, 0, 16, s));
  const unsigned nb = stride_blocks((size_t)w->P.N / w->cfg.world_size + 1);
  if (w->P.env == vg::kFlock)
    vg::k_slab_begin<vg::kFlock><<<nb, 256, 0, s>>>(w->P, w->SL, w->SB, w->cell_start, w->xo_rec,
                                                     w->xo_perm, a, w->err_dev, w->err_flag);
  else
    vg::k_slab_begin<vg::kTag><<<nb, 256, 0, s>>>(w->P, w->SL, w->SB, w->cell_start, w->xo_rec,
                                                   w->xo_perm, a, w->err_dev, w->err_flag);
  vg_status st = launch_check("k_slab_begin");
  prof_mark(w, 1, s);
  return st;
}
}  // namespace

vg_status vg_slab_begin(vg_world* w, const float* actions, void* stream) {
  NvtxRange nvtx_("vg_slab_begin");
  if (vg_status st = need_slab(w, true, "vg_slab_begin")) return st;
  if (!actions) return fail(VG_EINVAL, "actions: NULL");
  if (!w->binned) return fail(VG_EINVAL, "vg_slab_begin: call vg_slab_load first");
  DeviceGuard dg_(w->device);
  if (vg_status st = check_pending(w)) return st;
  cudaStream_t s = as_stream(stream);
  const float2* a = reinterpret_cast<const float2*>(actions);
  static const char kBeginKey = 0;                  // graph key: (actions, &kBeginKey, {})
  vg_status st;
  if (graph_ok(w, s)) {
    const vg_outputs none{};
    st = cached_graph(w, a, &kBeginKey, &none, s, "vg_slab_begin",
                      [&](cudaStream_t cs) { return slab_begin_launch(w, a, cs); });
  } else {
    st = slab_begin_launch(w, a, s);
  }
  if (!st) w->slab_stage = 1;
  return st;
}

vg_status vg_slab_get_io(vg_world* w, vg_slab_io* io) {
  if (vg_status st = need_slab(w, true, "vg_slab_get_io")) return st;
  if (!io) return fail(VG_EINVAL, "io: NULL");
  io->send_left = w->SB.send_l;
  io->send_right = w->SB.send_r;
  io->recv_left = const_cast<unsigned char*>(w->SB.recv_l);
  io->recv_right = const_cast<unsigned char*>(w->SB.recv_r);
  io->message_bytes = (int64_t)w->msg_bytes;
  io->left_rank = w->left;
  io->right_rank = w->right;
  io->lo = w->SL.lo;
  io->hi = w->SL.hi;
  io->capacity_rows = (int64_t)w->P.N;
  return VG_OK;
}

vg_status vg_slab_exchange_loopback(vg_world* const* ws, int32_t n, void* stream) {
  NvtxRange nvtx_("vg_slab_exchange_loopback");
  if (!ws || n < 2) return fail(VG_EINVAL, "vg_slab_exchange_loopback: need >= 2 worlds");
  for (int g = 0; g < n; ++g) {
    if (vg_status st = need_slab(ws[g], true, "vg_slab_exchange_loopback")) return st;
    if (ws[g]->cfg.world_size != n || ws[g]->cfg.rank != g || ws[g]->msg_bytes != ws[0]->msg_bytes)
      return fail(VG_EINVAL, "vg_slab_exchange_loopback: worlds must be ranks 0..n-1 of one slab group");
  }
  cudaStream_t s = as_stream(stream);
  for (int g = 0; g < n; ++g) {
    vg_world* w = ws[g];
    VG_CUDA(cudaMemcpyAsync(const_cast<unsigned char*>(ws[w->left]->SB.recv_r), w->SB.send_l,
                            w->msg_bytes, cudaMemcpyDeviceToDevice, s));
    VG_CUDA(cudaMemcpyAsync(const_cast<unsigned char*>(ws[w->right]->SB.recv_l), w->SB.send_r,
                            w->msg_bytes, cudaMemcpyDeviceToDevice, s));
  }
  return VG_OK;
}

namespace {
// The interior phase: bin memory columns [0, W-2) of the local set and sense their inner
// cells — nothing here waits for the halo.
vg_status slab_interior_launch(vg_world* w, const vg_outputs* outs, cudaStream_t s) {
  vg_status st = (w->P.env == vg::kFlock) ? slab_bin<vg::kFlock>(w, s, kSlabInterior)
                                          : slab_bin<vg::kTag>(w, s, kSlabInterior);
  if (st) return st;
  st = launch_sense<true>(w, outs, s, kSlabInterior);
  prof_mark(w, 2, s);
  return st;
}
// The boundary phase, once the halo arrived: append the received records, bin the boundary
// and ghost columns, sense the owned cells whose stencil reaches them.
vg_status slab_finish_launch(vg_world* w, const vg_outputs* outs, cudaStream_t s) {
  vg::k_slab_unpack<<<stride_blocks(2ull * w->SB.cap_msg), 256, 0, s>>>(w->P, w->SL, w->SB);
  if (vg_status st = launch_check("k_slab_unpack")) return st;
  prof_mark(w, 3, s);
  vg_status st = (w->P.env == vg::kFlock) ? slab_bin<vg::kFlock>(w, s, kSlabBoundary)
                                          : slab_bin<vg::kTag>(w, s, kSlabBoundary);
  if (st) return st;
  prof_mark(w, 4, s);
  st = launch_sense<true>(w, outs, s, kSlabBoundary);
  prof_mark(w, 5, s);
  return st;
}

vg_status slab_interior(vg_world* w, const vg_outputs* outs, cudaStream_t s) {
  static const char kInteriorKey = 0;               // graph key: (nullptr, &kInteriorKey, outs)
  vg_status st;
  if (graph_ok(w, s))
    st = cached_graph(w, nullptr, &kInteriorKey, outs, s, "vg_slab_interior",
                      [&](cudaStream_t cs) { return slab_interior_launch(w, outs, cs); });
  else
    st = slab_interior_launch(w, outs, s);
  w->binned = false;                                // until the boundary phase
  if (!st) w->slab_stage = 2;
  return st;
}

vg_status slab_finish(vg_world* w, const vg_outputs* outs, cudaStream_t s) {
  static const char kFinishKey = 0;                 // graph key: (nullptr, &kFinishKey, outs)
  vg_status st;
  if (graph_ok(w, s)) {
    st = cached_graph(w, nullptr, &kFinishKey, outs, s, "vg_slab_finish",
                      [&](cudaStream_t cs) { return slab_finish_launch(w, outs, cs); });
  } else {
    st = slab_finish_launch(w, outs, s);
    if (w->prof_n < w->prof_max) ++w->prof_n;
  }
  if (!st) {
    w->slab_stage = 0;
    w->binned = true;
  }
  return st;
}
}  // namespace

vg_status vg_slab_interior(vg_world* w, const vg_outputs* outs, void* stream) {
  NvtxRange nvtx_("vg_slab_interior");
  if (vg_status st = need_slab(w, true, "vg_slab_interior")) return st;
  DeviceGuard dg_(w->device);
  if (!outs) return fail(VG_EINVAL, "outs: NULL");
  if (w->slab_stage != 1) return fail(VG_EINVAL, "vg_slab_interior: call vg_slab_begin first (once per step)");
  return slab_interior(w, outs, as_stream(stream));
}

vg_status vg_slab_finish(vg_world* w, const vg_outputs* outs, void* stream) {
  NvtxRange nvtx_("vg_slab_finish");
  if (vg_status st = need_slab(w, true, "vg_slab_finish")) return st;
  DeviceGuard dg_(w->device);
  if (!outs) return fail(VG_EINVAL, "outs: NULL");
  if (w->slab_stage == 0) return fail(VG_EINVAL, "vg_slab_finish: call vg_slab_begin first");
  cudaStream_t s = as_stream(stream);
  if (w->slab_stage == 1)                           // no vg_slab_interior this step
    if (vg_status st = slab_interior(w, outs, s)) return st;
  return slab_finish(w, outs, s);
}

vg_status vg_slab_step(vg_world* w, const float* actions, const vg_outputs* outs, void* stream) {
  NvtxRange nvtx_("vg_slab_step");
  if (vg_status st = need_slab(w, true, "vg_slab_step")) return st;
  if (!actions || !outs) return fail(VG_EINVAL, "actions/outs: NULL");
  if (!w->comm)
    return fail(VG_EINVAL, "vg_slab_step: the world has no communicator (create it with "
                           "cfg.nccl_unique_id), or use vg_slab_begin / exchange / vg_slab_finish");
  DeviceGuard dg_(w->device);
  cudaStream_t s = as_stream(stream);
  if (vg_status st = vg_slab_begin(w, actions, stream)) return st;
  // Halo exchange on the world's comm stream, overlapped with the interior phase on `s`:
  // send_left -> left's recv_right, send_right -> right's recv_left.  Per peer pair NCCL
  // matches sends and receives in issue order, so the same order on every rank pairs them
  // for P = 2 too (both neighbours the same rank).
  const NcclApi* nc = nccl_api();
  VG_CUDA(cudaEventRecord(w->ev_fork, s));
  VG_CUDA(cudaStreamWaitEvent(w->comm_stream, w->ev_fork, 0));
  VG_NCCL(nc->GroupStart());
  VG_NCCL(nc->Send(w->SB.send_l, w->msg_bytes, ncclUint8, w->left, w->comm, w->comm_stream));
  VG_NCCL(nc->Send(w->SB.send_r, w->msg_bytes, ncclUint8, w->right, w->comm, w->comm_stream));
  VG_NCCL(nc->Recv(const_cast<unsigned char*>(w->SB.recv_r), w->msg_bytes, ncclUint8, w->right,
                   w->comm, w->comm_stream));
  VG_NCCL(nc->Recv(const_cast<unsigned char*>(w->SB.recv_l), w->msg_bytes, ncclUint8, w->left,
                   w->comm, w->comm_stream));
  VG_NCCL(nc->GroupEnd());
  VG_CUDA(cudaEventRecord(w->ev_join, w->comm_stream));
  if (vg_status st = slab_interior(w, outs, s)) return st;
  VG_CUDA(cudaStreamWaitEvent(s, w->ev_join, 0));
  return slab_finish(w, outs, s);
}

vg_status vg_nccl_unique_id(void* out, int32_t nbytes) {
  if (!out || nbytes < (int32_t)sizeof(ncclUniqueId))
    return fail(VG_EINVAL, "vg_nccl_unique_id: need a %d-byte buffer", (int)sizeof(ncclUniqueId));
  const NcclApi* nc = nccl_api();
  if (!nc) return fail(VG_ENCCL, "vg_nccl_unique_id: %s", nccl_err());
  ncclUniqueId id;
  VG_NCCL(nc->GetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return VG_OK;
}

vg_status vg_slab_sense(vg_world* w, const vg_outputs* outs, void* stream) {
  NvtxRange nvtx_("vg_slab_sense");
  if (vg_status st = need_slab(w, true, "vg_slab_sense")) return st;
  if (!outs) return fail(VG_EINVAL, "outs: NULL");
  if (!w->binned) return fail(VG_EINVAL, "vg_slab_sense: call vg_slab_load first");
  DeviceGuard dg_(w->device);
  return launch_sense<true>(w, outs, as_stream(stream));
}

vg_status vg_slab_own_count(vg_world* w, void* stream, int64_t* n_own) {
  if (vg_status st = need_slab(w, true, "vg_slab_own_count")) return st;
  DeviceGuard dg_(w->device);
  if (!n_own) return fail(VG_EINVAL, "n_own: NULL");
  VG_CUDA(cudaStreamSynchronize(as_stream(stream)));
  uint32_t b = 0;                                  // owned: memory columns [0, W)
  VG_CUDA(cudaMemcpy(&b, w->cell_start + (size_t)w->SL.W * w->P.G, 4, cudaMemcpyDeviceToHost));
  *n_own = (int64_t)b;
  return VG_OK;
}

// ------------------------------------------------------------------ shared policy (K7)
}  // extern "C"

struct vg_policy {
  vg_policy_config cfg;
  vg::PolicyPacked pk{};
  bool have_weights = false;
  int n_sm = 148;
  int device = -1;
};

extern "C" {

vg_status vg_policy_create(const vg_policy_config* cfg, vg_policy** out) {
  if (!out) return fail(VG_EINVAL, "out: NULL");
  *out = nullptr;
  if (!cfg) return fail(VG_EINVAL, "cfg: NULL");
  if (cfg->obs_dim < 1 || cfg->obs_dim > vg::kPolK1) return fail(VG_EINVAL, "obs_dim: must be in [1, 144]");
  for (int d = 0; d < 2; ++d)
    if (!(cfg->act_lo[d] <= cfg->act_hi[d])) return fail(VG_EINVAL, "act_lo/act_hi: need lo <= hi");
  vg_policy* p = new (std::nothrow) vg_policy();
  if (!p) return fail(VG_ENOMEM, "host allocation failed");
  p->cfg = *cfg;
  int dev = 0;
  cudaGetDevice(&dev);
  p->device = dev;
  cudaDeviceGetAttribute(&p->n_sm, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->pk.B1), vg::kPolN * vg::kPolK1 * 2);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p->pk.B2), vg::kPolN * vg::kPolK2 * 2);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p->pk.B3), vg::kPolN3 * vg::kPolK2 * 2);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p->pk.consts), vg::kConstFloats * 4);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(vg::k_policy, cudaFuncAttributeMaxDynamicSharedMemorySize, vg::kPolSmem);
  if (e != cudaSuccess) {
    vg_policy_destroy(p);
    return fail(VG_ECUDA, "vg_policy_create: %s", cudaGetErrorString(e));
  }
  *out = p;
  return VG_OK;
}

void vg_policy_destroy(vg_policy* p) {
  if (!p) return;
  cudaFree(p->pk.B1);
  cudaFree(p->pk.B2);
  cudaFree(p->pk.B3);
  cudaFree(p->pk.consts);
  delete p;
}

vg_status vg_policy_set_weights(vg_policy* p, const float* const* w, void* stream) {
  if (!p || !w) return fail(VG_EINVAL, "policy/weights: NULL");
  for (int i = 0; i < 13; ++i)
    if (!w[i]) return fail(VG_EINVAL, "weights[%d]: NULL", i);
  DeviceGuard dg_(p->device);
  const int n = vg::kPolN * vg::kPolK1;
  vg::k_policy_pack<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(
      p->cfg.obs_dim, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7], w[8], w[9], w[10], w[11],
      w[12], p->cfg.act_lo[0], p->cfg.act_lo[1], p->cfg.act_hi[0], p->cfg.act_hi[1], p->pk);
  if (vg_status st = launch_check("k_policy_pack")) return st;
  p->have_weights = true;
  return VG_OK;
}

vg_status vg_policy_forward_class(vg_policy* p, const float* obs, int64_t rows,
                                  int64_t period, int64_t split, int32_t cls,
                                  const vg_policy_outputs* outs, uint64_t seed, uint64_t step,
                                  void* stream) {
  NvtxRange nvtx_("vg_policy_forward_class");
  if (!p || !obs || !outs) return fail(VG_EINVAL, "policy/obs/outs: NULL");
  if (!p->have_weights) return fail(VG_EINVAL, "vg_policy_forward: call vg_policy_set_weights first");
  if (rows < 0) return fail(VG_EINVAL, "rows: must be >= 0");
  if (period < 0 || (period > 0 && (split < 0 || split > period || (cls != 0 && cls != 1))))
    return fail(VG_EINVAL, "vg_policy_forward_class: need period >= 0, 0 <= split <= period, cls in {0, 1}");
  if (rows == 0) return VG_OK;
  DeviceGuard dg_(p->device);
  vg::PolicyOut o{outs->mean, outs->value, outs->action, outs->logp};
  const int64_t tiles = (rows + vg::kPolTile - 1) / vg::kPolTile;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, p->n_sm);
  vg::k_policy<<<grid, vg::kPolThreads, vg::kPolSmem, as_stream(stream)>>>(
      obs, rows, p->cfg.obs_dim, p->pk, o, (uint32_t)seed, (uint32_t)(seed >> 32),
      (uint32_t)step, (uint32_t)(step >> 32), period, split, cls);
  return launch_check("k_policy");
}

vg_status vg_policy_forward(vg_policy* p, const float* obs, int64_t rows,
                            const vg_policy_outputs* outs, uint64_t seed, uint64_t step,
                            void* stream) {
  return vg_policy_forward_class(p, obs, rows, 0, 0, 0, outs, seed, step, stream);
}

vg_status vg_gae(const float* reward, const float* value, int64_t n, int32_t t, float gamma,
                 float lambda, float* adv, float* ret, void* stream) {
  NvtxRange nvtx_("vg_gae");
  if (!reward || !value || !adv || !ret) return fail(VG_EINVAL, "vg_gae: NULL pointer");
  if (n < 0 || t < 1) return fail(VG_EINVAL, "vg_gae: need n >= 0 and t >= 1");
  if (!(gamma >= 0.f && gamma <= 1.f) || !(lambda >= 0.f && lambda <= 1.f))
    return fail(VG_EINVAL, "vg_gae: gamma and lambda must be in [0, 1]");
  if (n == 0) return VG_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 1 << 20);
  vg::k_gae<<<blocks, 256, 0, as_stream(stream)>>>(reward, value, n, t, gamma, gamma * lambda,
                                                    adv, ret);
  return launch_check("k_gae");
}

vg_status vg_opinion_step(const int32_t* row_ptr, const int32_t* col, const float* weight,
                          int32_t n, int64_t n_edges, const float* op_in, float* op_out,
                          float threshold, float strength, void* stream) {
  NvtxRange nvtx_("vg_opinion_step");
  if (!row_ptr || !op_in || !op_out) return fail(VG_EINVAL, "vg_opinion_step: NULL pointer");
  if (n < 0) return fail(VG_EINVAL, "vg_opinion_step: n must be >= 0");
  if (n_edges < 0 || n_edges > INT32_MAX) return fail(VG_EINVAL, "vg_opinion_step: n_edges must be in [0, 2^31)");
  if (n_edges > 0 && (!col || !weight)) return fail(VG_EINVAL, "vg_opinion_step: col / weight NULL with n_edges > 0");
  if (op_in == op_out) return fail(VG_EINVAL, "vg_opinion_step: op_in and op_out must differ (simultaneous update)");
  if (!(threshold >= 0.f) || !(strength >= 0.f)) return fail(VG_EINVAL, "vg_opinion_step: threshold, strength must be >= 0");
  if (n == 0) return VG_OK;
  vg::k_opinion<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      row_ptr, col, weight, n, (long long)n_edges, op_in, op_out, threshold, strength);
  return launch_check("k_opinion");
}

vg_status vg_opinion_sync_errors(void* stream, int64_t* bad_node) {
  if (bad_node) *bad_node = -1;
  if (cudaError_t e = cudaStreamSynchronize(as_stream(stream)))
    return fail(VG_ECUDA, "vg_opinion_sync_errors: %s", cudaGetErrorString(e));
  unsigned long long bad = 0, none = ~0ull;
  if (cudaError_t e = cudaMemcpyFromSymbol(&bad, vg::g_opinion_bad, sizeof(bad)))
    return fail(VG_ECUDA, "vg_opinion_sync_errors: %s", cudaGetErrorString(e));
  if (bad == none) return VG_OK;
  cudaMemcpyToSymbol(vg::g_opinion_bad, &none, sizeof(none));
  if (bad_node) *bad_node = (int64_t)bad;
  return fail(VG_ESTATE, "vg_opinion_step: node %llu has an invalid row (row_ptr) or a dangling edge (col outside [0, n))", bad);
}

vg_status vg_rollout(vg_world* w, vg_policy* pol, vg_policy* pol_chaser, float* state,
                     const vg_rollout_buffers* b, int32_t t, uint64_t seed, uint64_t step0,
                     float gamma, float lambda, void* stream) {
  NvtxRange nvtx_("vg_rollout");
  if (!w || !pol || !state || !b) return fail(VG_EINVAL, "vg_rollout: NULL argument");
  if (pol_chaser && w->P.env != vg::kTag) return fail(VG_EINVAL, "vg_rollout: pol_chaser needs a tag world");
  if (pol_chaser && pol_chaser->cfg.obs_dim != w->P.obs_dim)
    return fail(VG_EINVAL, "vg_rollout: chaser policy obs_dim %d != world obs_dim %d", pol_chaser->cfg.obs_dim, w->P.obs_dim);
  if (vg_status st = need_slab(w, false, "vg_rollout")) return st;
  DeviceGuard dg_(w->device);
  if (!b->obs || !b->action || !b->reward || !b->value) return fail(VG_EINVAL, "vg_rollout: obs/action/reward/value buffers required");
  if (t < 1) return fail(VG_EINVAL, "vg_rollout: t must be >= 1");
  if (pol->cfg.obs_dim != w->P.obs_dim) return fail(VG_EINVAL, "vg_rollout: policy obs_dim %d != world obs_dim %d", pol->cfg.obs_dim, w->P.obs_dim);
  if (vg_status st = check_pending(w)) return st;
  cudaStream_t s = as_stream(stream);
  const size_t M = (size_t)w->P.total;
  float4* io = reinterpret_cast<float4*>(state);
  // per-type policies: runners = class 0, chasers = class 1 of period N
  const int64_t per = pol_chaser ? (int64_t)w->P.N : 0;
  const int64_t split = pol_chaser ? (int64_t)(w->P.N - w->cfg.n_chasers) : 0;
  auto forward = [&](const float* obs, const vg_policy_outputs* po, uint64_t step) -> vg_status {
    if (vg_status st = vg_policy_forward_class(pol, obs, (int64_t)M, per, split, 0, po, seed,
                                               step, stream)) return st;
    if (pol_chaser)
      return vg_policy_forward_class(pol_chaser, obs, (int64_t)M, per, split, 1, po, seed,
                                     step, stream);
    return VG_OK;
  };
  for (int k = 0; k < t; ++k) {
    const vg_policy_outputs po{nullptr, b->value + k * M, b->action + k * M * 2,
                               b->logp ? b->logp + k * M : nullptr};
    if (vg_status st = forward(b->obs + k * M * w->P.obs_dim, &po, step0 + (uint64_t)k)) return st;
    vg_outputs o{};
    o.obs = b->obs + (k + 1) * M * w->P.obs_dim;
    o.reward = b->reward + k * M;
    if (vg_status st = launch_step(w, io, reinterpret_cast<const float2*>(b->action + k * M * 2), &o, s)) return st;
  }
  const vg_policy_outputs pv{nullptr, b->value + (size_t)t * M, nullptr, nullptr};
  if (vg_status st = forward(b->obs + (size_t)t * M * w->P.obs_dim, &pv, step0 + (uint64_t)t)) return st;
  if (b->adv && b->ret)
    return vg_gae(b->reward, b->value, (int64_t)M, t, gamma, lambda, b->adv, b->ret, stream);
  return VG_OK;
}

vg_status vg_profile_begin(vg_world* w, int32_t max_steps) {
  if (!w || max_steps < 0 || max_steps > (1 << 20)) return fail(VG_EINVAL, "world/max_steps");
  const size_t need = (size_t)max_steps * (VG_N_PHASES + 1);
  while (w->prof_ev.size() < need) {
    cudaEvent_t e;
    VG_CUDA(cudaEventCreate(&e));
    w->prof_ev.push_back(e);
  }
  w->prof_max = max_steps;
  w->prof_n = 0;
  return VG_OK;
}

vg_status vg_profile_end(vg_world* w, void* stream, double* phase_ms, int32_t* n_steps) {
  if (!w || !phase_ms) return fail(VG_EINVAL, "world/phase_ms: NULL");
  DeviceGuard dg_(w->device);
  VG_CUDA(cudaStreamSynchronize(as_stream(stream)));
  for (int k = 0; k < VG_N_PHASES; ++k) phase_ms[k] = 0.0;
  for (int i = 0; i < w->prof_n; ++i) {
    for (int k = 0; k < VG_N_PHASES; ++k) {
      float ms = 0.f;
      VG_CUDA(cudaEventElapsedTime(&ms, w->prof_ev[(size_t)i * (VG_N_PHASES + 1) + k],
                                   w->prof_ev[(size_t)i * (VG_N_PHASES + 1) + k + 1]));
      phase_ms[k] += ms;
    }
  }
  if (n_steps) *n_steps = w->prof_n;
  w->prof_max = 0;
  w->prof_n = 0;
  return VG_OK;
}

vg_status vg_sync_errors(vg_world* w, void* stream, int64_t* bad_agent) {
  if (!w) return fail(VG_EINVAL, "world: NULL");
  DeviceGuard dg_(w->device);
  VG_CUDA(cudaStreamSynchronize(as_stream(stream)));
  unsigned long long v = 0;
  VG_CUDA(cudaMemcpy(&v, w->err_dev, sizeof(v), cudaMemcpyDeviceToHost));
  if (bad_agent) *bad_agent = (v == ~0ull) ? -1 : (int64_t)v;
  if (w->comm) {
    ncclResult_t ar = ncclSuccess;
    VG_NCCL(nccl_api()->CommGetAsyncError(w->comm, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
      return fail(VG_ENCCL, "slab halo exchange: %s", nccl_api()->GetErrorString(ar));
  }
  if (w->slab) {
    uint32_t ovf = 0;
    VG_CUDA(cudaMemcpy(&ovf, w->slab_ovf, 4, cudaMemcpyDeviceToHost));
    if (ovf) {
      VG_CUDA(cudaMemset(w->slab_ovf, 0, 4));
      return fail(VG_EOVERFLOW, "slab halo/local capacity overflow (raise halo_capacity)");
    }
  }
  if (v != ~0ull) {
    const unsigned long long none = ~0ull;
    VG_CUDA(cudaMemcpy(w->err_dev, &none, sizeof(none), cudaMemcpyHostToDevice));
    *w->err_flag = 0;
    return fail(VG_ESTATE, "invalid state or action at global agent index %llu", v);
  }
  return VG_OK;
}

}  // extern "C"
