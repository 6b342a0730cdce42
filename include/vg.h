/*
 * vg.h — C ABI of libvg: the batched environment step of the Vogue MARL environments
 * (arxiv 2207.03945, "High Performance Simulation for Scalable Multi-Agent Reinforcement
 * Learning"), flock (§4.1) and tag (§4.2), on B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; An = reading of a gap in the
 * paper, listed in DESIGN.md §3.
 *
 * The paper's model: agents embedded in space interact with the agents in their
 * spatial proximity; the model advances in discrete time-steps and every interaction of a
 * step reads the same snapshot ("individual interactions update agents simultaneously").
 * One environment update: "the agents are accelerated and rotated (according to
 * actions sampled from the current policy), after which their local view model and rewards
 * are updated for all pairs of agents in spatial proximity".
 *
 * Data layout (all device memory unless stated; all row-major, contiguous, 4-byte aligned;
 * state/sorted 16-byte aligned):
 *   state    float [R][N][4]  (x, y, theta, s): position on the L x L torus in [0, L),
 *            heading theta in [0, RN32(2 pi)) radians (CCW from +x), flock speed s.
 *            Tag: 4th column is reserved — ignored on input, preserved by integrate; an
 *            agent's type comes from its index: agents [N - n_chasers, N) are chasers (A14).
 *   actions  float [R][N][2]  flock (accelerate, rotate); tag (rotate, move)
 *            (P:194).  Finite out-of-box values are clamped to the box, NaN is an
 *            error.
 *   R = n_replicas independent worlds of N = n_agents agents each (replicas never
 *   interact).
 *
 * Ownership: the caller owns state, actions and every output buffer.  The world owns its
 * scratch (allocated once in vg_world_create).  No call after create allocates, blocks
 * the host, or copies device->host (except vg_sync_errors and vg_step_host, which say so),
 * so vg_bin/vg_sense/vg_reward/vg_integrate/vg_step are CUDA-graph capturable.
 * Concurrency: one stream at a time per world; a world is not thread-safe.
 *
 * Errors: every entry point returns vg_status.  Configuration errors are found
 * synchronously (VG_EINVAL, vg_last_error() names the field).  Device-side state errors
 * (a position outside [0, L), a non-finite or out-of-range heading, a non-finite
 * speed, a NaN action) are recorded in a device error word as the smallest offending
 * global agent index r*N + i; they surface as VG_ESTATE from vg_sync_errors() and from the
 * next call that finds the word set (a non-blocking read of mapped host memory).
 */
#ifndef VG_H
#define VG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VG_ABI_VERSION 3

typedef enum {
  VG_OK = 0,
  VG_EINVAL = 1,     /* invalid argument or configuration (message names the field)     */
  VG_ESTATE = 2,     /* device-side invalid state/action (index in vg_sync_errors)       */
  VG_ECUDA = 3,      /* CUDA runtime error (message has the CUDA error string)           */
  VG_ENCCL = 4,      /* NCCL error (slab mode)                                           */
  VG_EOVERFLOW = 5,  /* fixed-capacity halo buffer overflow (slab mode)                  */
  VG_ENOMEM = 6      /* device allocation failed in vg_world_create                      */
} vg_status;

typedef enum { VG_ENV_FLOCK = 0, VG_ENV_TAG = 1 } vg_env;
/* Vision model (reading A1): SECTOR bins neighbour centres by bearing (hot path); RAY casts
 * one ray per sector centre against neighbour discs of radius d_r (NEXT #2;
 * needs cell size >= (d_v + d_r)(1 + 2^-12)). */
typedef enum { VG_VISION_SECTOR = 0, VG_VISION_RAY = 1 } vg_vision;
typedef enum { VG_SHARD_REPLICA = 0, VG_SHARD_SLAB = 1 } vg_shard;

/* World configuration.  All floats are authoritative fp32 values (A12).  Defaults in
 * brackets are SPEC.md's; the paper fixes only d_v = L/10,
 * fov ~ 250 deg, v = 128 / 2 x 64 and obs_dim 129 / 128. */
typedef struct {
  int32_t env;          /* vg_env                                                          */
  int32_t vision;       /* vg_vision: VG_VISION_SECTOR (default) or VG_VISION_RAY          */
  int32_t shard;        /* vg_shard: VG_SHARD_REPLICA, or VG_SHARD_SLAB (see slab mode)     */
  int32_t n_agents;     /* N > 0, agents per replica                               */
  int32_t n_replicas;   /* R > 0; R*N < 2^31                                               */
  float width;          /* L, square torus side (A9)                           [100]       */
  float d_v;            /* view range = reward radius, 0 < d_v < L/2   [L/10]      */
  float d_r;            /* body radius; contact at d <= 2 d_r, 2 d_r < d_v [0.25]  */
  float fov;            /* field of view, radians, 0 < fov <= 2 pi     [250 deg]   */
  int32_t v;            /* sectors per channel, 1..128 (flock) / 1..64 (tag)   [128 / 64]  */
  int32_t grid;         /* G cells per axis, 0 = auto: largest G with L/G >= d_v(1+2^-12)
                           (A16); must satisfy that bound and G >= 3                      */
  float s_min, s_max;   /* flock speed bounds, 0 <= s_min < s_max      [0.05, 0.5] */
  float a_max;          /* flock acceleration bound > 0                        [0.1]       */
  float theta_max;      /* rotation bound, 0 < theta_max <= pi                 [0.2]       */
  float c_collide;      /* collision penalty > 0 (Fig. 4, A5)                  [1.0]       */
  float c_near;         /* peak closeness bonus > 0 (A5)                       [0.5]       */
  float d_peak;         /* bonus peak, 2 d_r < d_peak < d_v                    [(2d_r+d_v)/2] */
  int32_t n_chasers;    /* tag: 0 <= n_chasers <= N; agents [N - n_chasers, N) are chasers */
  float r_touch;        /* tag touch reward magnitude                          [1.0]       */
  float w_prox;         /* tag runner proximity weight                         [0.1]       */
  float s_max_chaser;   /* tag chaser move bound (runners use s_max)           [0.375]     */
  int32_t rank, world_size, halo_capacity; /* slab mode: this rank, P, records/message   */
  const void* nccl_unique_id;              /* slab mode: NULL, or 128 bytes from vg_nccl_unique_id: the world creates and owns an NCCL communicator (collective over the P ranks) for vg_slab_step */
} vg_config;

/* Caller-owned device output buffers; a NULL pointer means "do not write".  Rows are in
 * agent order r*N + i (not sorted order). */
typedef struct {
  float* obs;           /* [R][N][obs_dim]; obs_dim = 129 flock (128 view + s/s_max, P:171,
                           A24), 128 tag (runner channel 64 | chaser channel 64).
                           View entry = min over visible neighbours in that sector of
                           d/d_v, 1.0 if none (A1-A3)                       */
  float* reward;        /* [R][N] Eq. 1 / Fig. 4 (flock); P:194 rules (tag)               */
  uint32_t* n_neigh;    /* [R][N] #{j != i : d_ij < d_v} (all directions, A4)             */
  uint32_t* n_collide;  /* [R][N] #{j : d_ij <= 2 d_r}; tag: same-type contacts only      */
  uint32_t* n_touch;    /* [R][N] tag only: opposite-type contacts (d <= 2 d_r)           */
  uint32_t* sector_occ; /* [R][N][occ_words] bit (c*v + k) set iff sector k of channel c
                           holds a visible neighbour; occ_words = ceil(channels*v/32)     */
  uint32_t* agent_id;   /* slab mode: [N] global agent id of each output row                */
} vg_outputs;

typedef struct {
  int32_t grid;         /* G                                                               */
  float cell_size;      /* L / G                                                           */
  int32_t n_cells;      /* R * G * G                                                       */
  int32_t obs_dim;      /* 129 flock / 128 tag (for v = 128 / 64)                          */
  int32_t channels;     /* 1 flock / 2 tag                                                 */
  int32_t occ_words;    /* ceil(channels * v / 32)                                         */
  int64_t total_agents; /* R * N                                                           */
  int64_t scratch_bytes;/* device bytes owned by the world                                 */
  int32_t kernels_per_step; /* libvg kernels one vg_step (slab: begin + finish) launches   */
  int32_t sense_defaults;   /* 1: K4's sector pass runs with the paper's default constants
                               compiled in (the world's derived constants are bitwise those);
                               0: constants read from the parameters (same results)         */
} vg_world_info;

typedef struct vg_world vg_world;

/* Validate cfg and allocate all scratch on the current CUDA device.
 * Errors: VG_EINVAL (message names the field), VG_ENOMEM, VG_ECUDA.  *out = NULL on error. */
vg_status vg_world_create(const vg_config* cfg, vg_world** out);
void vg_world_destroy(vg_world* w);
vg_status vg_world_query(const vg_world* w, vg_world_info* info);

/* Spatial binning of `state` (A16): cell_id = cy*G + cx with
 * cx = min(G-1, floor(RN32(x * RN32(G/L)))), a stable counting sort by cell per replica
 * (within a cell, ascending agent id).  Results are owned by the world and read by
 * vg_sense / vg_reward; vg_get_bins exposes them.  Validates the state (error word). */
vg_status vg_bin(vg_world* w, const float* state, void* stream);

/* Sector vision + fused reward for the state last binned (P:158, P:164, P:171-178,
 * P:184): writes every non-NULL buffer of *outs.  All agents read the same
 * snapshot.  Requires a prior vg_bin (or vg_step) on the same stream. */
vg_status vg_sense(vg_world* w, const vg_outputs* outs, void* stream);

/* vg_sense restricted to the cells of grid columns [col_lo, col_hi) of a one-replica world
 * (n_replicas = 1): writes the output rows of exactly the agents binned in those columns
 * (other rows untouched); the same values vg_sense writes for them.  For the replicated-
 * state multi-GPU scheme (every rank holds and bins the whole world and
 * senses its own columns).  Errors: VG_EINVAL (slab world, R > 1, bad range, no binning). */
vg_status vg_sense_columns(vg_world* w, const vg_outputs* outs, int32_t col_lo, int32_t col_hi,
                           void* stream);

/* Reward and neighbour/contact counts only (no bearings, no observation), for the state
 * last binned: flock r_i = sum over j != i with d_ij < d_v of f(d_ij) (Eq. 1, P:174-175;
 * f = the Fig. 4 shape, reading A5: -c_collide for d <= 2 d_r, else rising
 * linearly to c_near at d_peak and falling to 0 at d_v); tag: the P:194 touch rules plus
 * w_prox x the runner-runner f (A15).  n_neigh = #{j: d < d_v}, n_collide (and tag n_touch)
 * = same-type (opposite-type) contacts d <= 2 d_r (A6).  Same values as vg_sense's fused
 * reward (an unfused pass, for tests).  Writes reward, n_neigh, n_collide, n_touch of *outs
 * (others ignored).  Errors: VG_EINVAL (NULL world / outs, or no prior vg_bin / vg_step),
 * VG_ECUDA. */
vg_status vg_reward(vg_world* w, const vg_outputs* outs, void* stream);

/* Integrate actions into state in place (A7, A8, A10): rotate, then
 * (flock) accelerate, then move along the new heading, wrapping on the torus. */
vg_status vg_integrate(vg_world* w, float* state, const float* actions, void* stream);

/* One environment update: integrate, bin, sense + reward — all on device. */
vg_status vg_step(vg_world* w, float* state, const float* actions, const vg_outputs* outs,
                  void* stream);

/* vg_step with HOST buffers for the per-step inputs/results: copies actions_host
 * ([R][N][2], pinned host memory recommended) into a world-owned device buffer, steps,
 * and copies the reward into reward_host ([R][N], may be NULL) — all asynchronously on
 * `stream`; the caller synchronizes the stream before reading reward_host. */
vg_status vg_step_host(vg_world* w, float* state, const float* actions_host,
                       const vg_outputs* outs, float* reward_host, void* stream);

/* Borrowed device pointers to the last binning (valid until the next vg_bin/vg_step):
 * cell_id [R][N] (replica-local cy*G+cx), cell_start [R*G*G + 1] (offsets into the flat
 * [R*N] sorted arrays), perm [R][N] (local agent id of each sorted slot), sorted
 * [R][N][4] (state records in sorted order; tag: 4th column = type 0/1).  Any argument
 * may be NULL. */
vg_status vg_get_bins(const vg_world* w, const uint32_t** cell_id, const uint32_t** cell_start,
                      const uint32_t** perm, const float** sorted);

/* Synchronize `stream`, read and clear the device error word.  *bad_agent = -1 if clean,
 * else the smallest offending global agent index (and VG_ESTATE is returned). */
vg_status vg_sync_errors(vg_world* w, void* stream, int64_t* bad_agent);

/* ---------------------------------------------------------------- slab mode
 * One world (n_replicas = 1, N = n_agents global) split over world_size = P ranks by
 * x-slabs of whole cell columns: rank g owns global columns [g G/P, (g+1) G/P) (P | G,
 * >= 2 columns per rank, and the largest move per step < cell size so an agent crosses
 * at most one column).  All agents are updated simultaneously from one snapshot:
 * the slab decomposition changes nothing but where the work runs.  Each step:
 *   vg_slab_begin     integrate the owned rows and route them: stay, migrate (<= 1 slab),
 *                     or copy as a ghost (boundary column) into two messages (left, right);
 *   exchange          send_left -> left rank's recv_right, send_right -> right rank's
 *                     recv_left (the world's own NCCL communicator in vg_slab_step; or
 *                     the caller: torch.distributed P2P, host staging, or
 *                     vg_slab_exchange_loopback for P worlds in one process);
 *   vg_slab_interior  while the messages are in flight: bin the interior owned columns
 *                     (local 2..W-1, which no neighbour can send records into) and sense
 *                     + reward the owned cells whose 3x3 stencil lies inside them (local
 *                     columns 3..W-2);
 *   vg_slab_finish    after the exchange: append the received records, bin the boundary
 *                     and ghost columns, sense + reward the remaining owned cells (it runs
 *                     vg_slab_interior first if the caller skipped it).
 *   vg_slab_step      all of the above in one call: begin on `stream`, the halo exchange
 *                     (grouped ncclSend/ncclRecv) on the world's comm stream, the interior
 *                     phase on `stream` meanwhile, then the boundary phase after a stream
 *                     wait on the exchange (no host synchronization).  Needs a world
 *                     created with cfg.nccl_unique_id (VG_EINVAL otherwise); NCCL errors
 *                     (synchronous, or asynchronous via vg_sync_errors) are VG_ENCCL.
 * Output rows are the owned agents in (memory cell, y sub-bin, global id) order (K4's
 * sense order, a function of the state alone); outs->agent_id gives each row's global id;
 * the next vg_slab_begin takes actions[row] in that order.  vg_slab_interior and
 * vg_slab_finish of one step must get the same outs.  Every per-agent result is bitwise
 * identical to the single-world (replica) path.
 * Buffers: outputs need capacity N rows.  Messages: {u32 count, 3 x u32}, float4 rec[cap],
 * u32 id[cap], cap = halo_capacity (0 = auto: 4 N/G + 256, >= 1024).  A message or local
 * overflow is reported as VG_EOVERFLOW by vg_sync_errors.  Calls out of order (interior or
 * finish without begin, step without a communicator) are VG_EINVAL. */
typedef struct {
  void* send_left;
  void* send_right;
  void* recv_left;
  void* recv_right;
  int64_t message_bytes;   /* bytes of each of the four message buffers              */
  int32_t left_rank, right_rank;
  int32_t lo, hi;          /* owned global cell columns [lo, hi)                      */
  int64_t capacity_rows;   /* output rows to allocate (= N)                           */
} vg_slab_io;

/* Host-only: plan[0..3] = lo, hi, left rank, right rank of `rank` (no device needed). */
vg_status vg_slab_plan(int32_t grid, int32_t world_size, int32_t rank, int32_t* plan);
/* Select this rank's owned + ghost agents from the full global state [N][4] (device) and
 * bin them (step 0); vg_slab_sense then gives the initial observation. */
vg_status vg_slab_load(vg_world* w, const float* state_global, void* stream);
vg_status vg_slab_sense(vg_world* w, const vg_outputs* outs, void* stream);
vg_status vg_slab_begin(vg_world* w, const float* actions, void* stream);
vg_status vg_slab_get_io(vg_world* w, vg_slab_io* io);
vg_status vg_slab_exchange_loopback(vg_world* const* worlds, int32_t n, void* stream);
vg_status vg_slab_interior(vg_world* w, const vg_outputs* outs, void* stream);
vg_status vg_slab_finish(vg_world* w, const vg_outputs* outs, void* stream);
vg_status vg_slab_step(vg_world* w, const float* actions, const vg_outputs* outs, void* stream);
/* Synchronizes `stream`; *n_own = number of owned agents (valid output rows). */
vg_status vg_slab_own_count(vg_world* w, void* stream, int64_t* n_own);
/* Host-only: a new NCCL unique id (128 bytes into out[nbytes >= 128]) for the slab group's
 * communicator; rank 0 makes it, every rank passes the same bytes in cfg.nccl_unique_id.
 * libnccl is loaded at run time ($VG_NCCL_LIB, else libnccl.so.2): VG_ENCCL if missing. */
vg_status vg_nccl_unique_id(void* out, int32_t nbytes);

/* ------------------------------------------- shared policy forward
 * The actor-critic MLP of P:212 ("two hidden layers with 64 nodes each", tanh)
 * over all agents, on the tcgen05 tensor cores (fp16 operands, fp32 accumulation in TMEM),
 * followed by the Gaussian action sample of P:198 / S:355-372: a = clip(mean +
 * exp(log_std) eps, box) with log_std clamped to [-5, 2], log-prob of the
 * unclipped sample, eps from Philox4x32-10
 * (key = seed, counter = (row, step)) + Box-Muller. */
typedef struct vg_policy vg_policy;
typedef struct {
  int32_t obs_dim;         /* 1..144 (129 flock, 128 tag)                                  */
  float act_lo[2];         /* action box (flock: (-a_max, -theta_max); tag: (-theta_max, 0)) */
  float act_hi[2];
} vg_policy_config;
typedef struct {           /* caller-owned device buffers, NULL = not written              */
  float* mean;             /* [rows][2] actor mean                                          */
  float* value;            /* [rows]    critic value                                        */
  float* action;           /* [rows][2] clipped sample (also needs the sampling to run)     */
  float* logp;             /* [rows]    log-prob of the unclipped sample                    */
} vg_policy_outputs;
vg_status vg_policy_create(const vg_policy_config* cfg, vg_policy** out);
void vg_policy_destroy(vg_policy* p);
/* Upload weights: 13 fp32 device arrays, nn.Linear layout [out][in], in the order
 * W1[64][d] b1[64] W2[64][64] b2[64] W3[2][64] b3[2] log_std[2]
 * V1[64][d] c1[64] V2[64][64] c2[64] V3[1][64] c3[1]  (actor W*, critic V*). */
vg_status vg_policy_set_weights(vg_policy* p, const float* const* weights, void* stream);
/* obs: device [rows][obs_dim] fp32 (e.g. vg_outputs.obs).  Asynchronous on `stream`. */
vg_status vg_policy_forward(vg_policy* p, const float* obs, int64_t rows,
                            const vg_policy_outputs* outs, uint64_t seed, uint64_t step,
                            void* stream);
/* The same, writing only the rows of one class (per-type policies, "the runner and
 * chaser types share independent policies"): row r is of class ((r mod period) >= split),
 * i.e. for a tag world period = N, split = N - n_chasers (chasers are the last indices of
 * every replica, A14); period = 0 means every row (= vg_policy_forward).  Rows of the
 * other class are left untouched; the noise of row r is the same as in vg_policy_forward.
 * Errors: VG_EINVAL for period < 0, split outside [0, period], cls not 0/1. */
vg_status vg_policy_forward_class(vg_policy* p, const float* obs, int64_t rows,
                                  int64_t period, int64_t split, int32_t cls,
                                  const vg_policy_outputs* outs, uint64_t seed, uint64_t step,
                                  void* stream);

/* ------------------------------------------------- GAE over the trajectory buffer (§8f #3)
 * Generalized advantage estimation for n agents x t steps, continuing task
 * (no terminal flags; the value array carries the bootstrap row t).  Time-major device
 * arrays: reward [t][n], value [t+1][n] -> adv [t][n], ret [t][n] (adv + value).
 * A[k] = sum_l (gamma lambda)^l delta[k+l], delta[k] = r[k] + gamma V[k+1] - V[k]. */
vg_status vg_gae(const float* reward, const float* value, int64_t n, int32_t t, float gamma,
                 float lambda, float* adv, float* ret, void* stream);

/* ------------------------------------------ experience collection (Fig. 5)
 * t environment steps of the paper's loop, entirely on the device: for k = 0 .. t-1,
 * the shared policy samples actions from obs[k] (value[k], action[k], logp[k]; noise
 * counter step0 + k), then vg_step integrates them and writes obs[k+1] and reward[k];
 * finally value[t] = V(obs[t]) (bootstrap) and GAE (vg_gae) fills adv / ret.
 * Tag worlds may pass pol_chaser != NULL: runners (agents [0, N - n_chasers) of each
 * replica) then act with `pol` and chasers with `pol_chaser` — the two independent
 * policies of P:198 (vg_policy_forward_class per type); NULL = one shared policy.
 * pol_chaser on a flock world is VG_EINVAL.
 * Time-major device buffers for M = R*N agents: obs [t+1][M][obs_dim] (obs[0] from a prior
 * vg_bin + vg_sense or the previous rollout's obs[t]), action [t][M][2], logp [t][M],
 * reward [t][M], value [t+1][M], adv [t][M], ret [t][M].  Replica mode only.  No host
 * synchronization: the whole call can be captured in one CUDA graph. */
typedef struct {
  float* obs;
  float* action;
  float* logp;
  float* reward;
  float* value;
  float* adv;
  float* ret;
} vg_rollout_buffers;
vg_status vg_rollout(vg_world* w, vg_policy* pol, vg_policy* pol_chaser, float* state,
                     const vg_rollout_buffers* buf, int32_t t, uint64_t seed, uint64_t step0,
                     float gamma, float lambda, void* stream);

/* --------------------------------------- opinion dynamics, Listing 1 (§8f #4)
 * One step of the bounded-confidence graph interaction + self interaction: for each node
 * (me), over its out-edges in CSR order (sorted by (src, dst), row_ptr [n+1], col [E] =
 * dst, weight [E] >= 0): if |op[me] - op[you]| < threshold then w = strength weight,
 * new = (1 - w) new + w op[you]; new starts at op[me]; op_out[me] = new.  op_in and
 * op_out are distinct device arrays [n] (simultaneous update).  n_edges = E (the
 * length of col and weight).
 * Errors: NULL row_ptr/op_in/op_out (or col/weight with E > 0), n < 0, E outside
 * [0, 2^31), op_in == op_out, negative threshold/strength -> VG_EINVAL (synchronous).  A
 * row with row_ptr[i] < 0, row_ptr[i+1] < row_ptr[i] or row_ptr[i+1] > E, or an edge whose
 * col is outside [0, n) (a dangling index) is never read: the node keeps its opinion
 * / skips the edge, and the first such node is recorded for vg_opinion_sync_errors. */
vg_status vg_opinion_step(const int32_t* row_ptr, const int32_t* col, const float* weight,
                          int32_t n, int64_t n_edges, const float* op_in, float* op_out,
                          float threshold, float strength, void* stream);
/* Synchronizes `stream`; if any vg_opinion_step on this device since the last call met an
 * invalid row or dangling edge, writes the lowest such node to *bad_node (else -1), clears
 * the record and returns VG_ESTATE. */
vg_status vg_opinion_sync_errors(void* stream, int64_t* bad_node);

/* Phase timing for measurement.  After vg_profile_begin(w, max_steps), each of the next
 * max_steps vg_step calls records CUDA events on its stream between its phases
 * (VG_N_PHASES: integrate+cell-id+histogram, cell scan, scatter, cell sort, sense+reward).
 * vg_profile_end synchronizes `stream` and writes per-phase total milliseconds over the
 * recorded steps into phase_ms[VG_N_PHASES] and the step count into *n_steps.  Not for
 * use inside CUDA-graph capture.  Errors: VG_EINVAL, VG_ECUDA. */
#define VG_N_PHASES 5
vg_status vg_profile_begin(vg_world* w, int32_t max_steps);
vg_status vg_profile_end(vg_world* w, void* stream, double* phase_ms, int32_t* n_steps);

/* Thread-local message of the last error on this thread ("" if none). */
const char* vg_last_error(void);

/* ABI version (VG_ABI_VERSION). */
int32_t vg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VG_H */
