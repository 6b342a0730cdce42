// vg_kernels.cuh — sm_100a device kernels of the Vogue environment step.
//
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, An = reading in DESIGN.md §3.
// Pipeline of one step:
//   K1 k_integrate_bin  integrate + cell id + per-cell histogram slot   (HBM-bound)
//   K2 k_scan_cells     exclusive scan of the R*G*G cell counts          (latency)
//      (k_scan_tiles + k_scan_apply above 12,288 cells)
//   K3 k_scatter        place each agent at cell_start[cell] + slot      (HBM-bound)
//   K3b k_cell_sort     order each cell by ascending agent id (stable); the K4 sense order
//                       (sub-bins), window table and overflow work items  (HBM/ALU)
//   K1-K3b fused        k_replica_bin: one CTA per small replica world
//   K4 k_sense          3x3-stencil neighbour pass: sector vision + reward (FP32/issue-bound)
//   slab mode           k_slab_begin / load / unpack / keys / scatter
// No library kernels: every step of the path runs here.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace vg {

constexpr int kFlock = 0;
constexpr int kTag = 1;
constexpr uint32_t kOneBits = 0x3f800000u;          // 1.0f: "nothing in this sector" (A2)
constexpr float kBelowOne = 0.99999994f;            // largest float < 1: an occupied sector
constexpr float kFix = 4294967296.0f;               // 2^32: fixed-point reward unit (A16b)
constexpr float kFixInv = 2.3283064365386963e-10f;  // 2^-32
constexpr int kMaxViewSlots = 128;                  // channels * v <= 128
constexpr unsigned kFull = 0xffffffffu;

// Device copy of the configuration + derived fp32 constants (computed once on the host,
// DESIGN.md §4.0).  Passed by value to every kernel.
struct Params {
  int env, N, R, G, G2, v, channels, view_slots, obs_dim, occ_words, first_chaser;
  long long total;             // R * N
  float L, half_L, gs;         // gs = RN32(G / L)   (A16)
  float two_pi;                // RN32(2 pi): heading range [0, two_pi)   (A10)
  float s_min, s_max, a_max, theta_max, s_max_chaser;
  float d_v, dv2, inv_dv, contact2, two_dr;
  float half_fov, inv_fov, fv;  // fov/2, 1/fov, float(v)
  float c_collide, d_peak, k_rise, k_fall, w_prox;
  float b_rise, nk_fall, b_fall;   // f = min(k_rise d + b_rise, nk_fall d + b_fall) (A5)
  // The same line pair and -c_collide times 2^32 (exact scalings): K4 evaluates f directly
  // in fixed-point units, f * 2^32 (A16b), bit-identical to scaling afterwards.
  float fx_k_rise, fx_b_rise, fx_nk_fall, fx_b_fall, fx_mcollide;
  // symmetric tent (k_rise == k_fall, d_peak the midpoint of [2 d_r, d_v]: the defaults):
  // f = c_near - k |d - d_peak|, one add and one FMA (fx_cnear = c_near 2^32)
  int tent_sym;
  float fx_cnear;
  float half_v;                    // v / 2: sector coordinate phi v / fov + v / 2 (A3)
  float d_r, cand2, inv_w;         // ray vision: body radius, RN32((d_v + d_r)^2), v / fov
  float cell;                      // RN32(L / G) (K4 windows only)
  float inv_smax;                  // RN32(1 / s_max): obs[v] = s / s_max to <= 1.5 ulp (A24)
  float win_r2, win_margin;        // K4 window: candidate radius^2, conservative margin
  long long touch_fix;         // r_touch * 2^32
};

struct Outs {
  float* obs;
  float* reward;
  uint32_t* n_neigh;
  uint32_t* n_collide;
  uint32_t* n_touch;
  uint32_t* occ;
  uint32_t* agent_id;   // slab mode: global id of each output row
  int fast;             // every output K4 writes is present and rows x obs_dim < 2^31:
                        // K4 skips the NULL checks and indexes in 32 bits; 2: also the
                        // occupancy rows (4 words) are 16-byte aligned (one vector store)
};

// Slab mode: this rank owns global cell columns [lo, hi), W = hi - lo >= 2.
// The local grid has W + 2 columns l = 0..W+1 (l = 1..W owned, ghost columns 0 and W+1)
// x G rows, column-major, stored in the MEMORY column order m = slab_mcol(l): the interior
// owned columns l = 2..W-1 first (m = 0..W-3), then the owned boundary columns l = 1, W
// (m = W-2, W-1), then the ghosts l = 0, W+1 (m = W, W+1).  Memory cell = m G + cy.  The
// owned agents are the contiguous sorted range [0, cell_start[W G]); the interior columns
// [0, cell_start[(W-2) G]) hold no record a neighbour can send, so they are binned and
// their inner cells (l = 3..W-2) sensed while the halo is in flight (vg_slab_interior),
// and only the boundary columns are binned after it arrives (vg_slab_finish).
struct Slab {
  int lo, hi, W, n_lcells;
  // cells sensed by this K4 launch: memory columns [sc0, sc0 + snc), or, if snl > 0, the
  // memory columns scol[0..snl)
  int sc0, snc, snl, scol[4];
  // the boundary phase's memory columns bcol[0..nb) are cut into K4 work items of chunk_qb
  // queries (WorkList has the same fields for the items' creation)
  int chunk_qb, nb, bcol[4];
};
__host__ __device__ __forceinline__ int slab_mcol(int l, int W) {
  return (l >= 2 && l <= W - 1) ? l - 2 : (l == 1) ? W - 2 : (l == W) ? W - 1 : (l == 0) ? W : W + 1;
}
__host__ __device__ __forceinline__ int slab_lcol(int m, int W) {
  return (m < W - 2) ? m + 2 : (m == W - 2) ? 1 : (m == W - 1) ? W : (m == W) ? 0 : W + 1;
}
// Does this K4 launch sense memory column m?
__host__ __device__ __forceinline__ bool slab_senses(const Slab& SL, int m) {
  if (SL.snl == 0) return m >= SL.sc0 && m < SL.sc0 + SL.snc;
  bool in = false;
  for (int k = 0; k < 4; ++k) in |= (k < SL.snl && SL.scol[k] == m);
  return in;
}

// Record the smallest offending global agent index (S:59 error convention) and raise the
// host-visible flag (mapped pinned memory, plain store).
__device__ __forceinline__ void report_bad(unsigned long long* err, volatile uint32_t* flag,
                                           unsigned long long gi) {
  atomicMin(err, gi);
  *flag = 1u;
}

// Torus wrap of x + dx for x in [0, L), |dx| < L/2 (A10): the subtraction x - L is exact
// (Sterbenz), so a result that wraps to near 0 keeps full relative precision.
__device__ __forceinline__ float wrap_pos(float x, float dx, float L) {
  float t = __fadd_rn(x, dx);
  if (t >= L) {
    t = __fadd_rn(__fsub_rn(x, L), dx);
    if (t < 0.f) t = 0.f;                 // exact sum was just below L: the point is L^- == 0
  } else if (t < 0.f) {
    t = __fadd_rn(t, L);
    if (t >= L) t = 0.f;                  // rounded up to L: the point is 0^-
  }
  return t;
}

// sin / cos of a heading th in [0, two_pi) for the move (every integrate path uses this one
// function, so the paths stay bitwise equal).  VG_FAST_SINCOS: the MUFU on [-pi, pi) (the
// shift is exact by Sterbenz; abs error <= 3.6e-7, i.e. <= 1.8e-7 L of position for any
// admissible speed < L/2, against the 1e-5 L integrate tolerance); else sincosf.
#ifndef VG_FAST_SINCOS
#define VG_FAST_SINCOS 1
#endif
__device__ __forceinline__ void heading_sincos(float th, float two_pi, float* sn, float* cs) {
#if VG_FAST_SINCOS
  __sincosf((th >= 3.14159265f) ? __fsub_rn(th, two_pi) : th, sn, cs);
#else
  (void)two_pi;
  sincosf(th, sn, cs);
#endif
}

// Heading wrap into [0, two_pi) (A10; "heading normalized to [0, 2 pi)").
__device__ __forceinline__ float wrap_heading(float th, float two_pi) {
  if (th < 0.f) {
    th = __fadd_rn(th, two_pi);
    if (th >= two_pi) th = 0.f;
  } else if (th >= two_pi) {
    th = __fsub_rn(th, two_pi);           // exact (Sterbenz)
  }
  return th;
}

// ---------------------------------------------------------------------------------- K1
// One thread per agent.  INTEGRATE: apply the action: rotate, then
// (flock) accelerate with clamp(s + a, s_min, s_max) (A7), then move along the new heading
// (A8), wrapping on the torus.  BIN: cell id cx = min(G-1, floor(RN32(x * gs))) (A16) and
// an atomic per-(replica, cell) histogram whose return value is the agent's arrival slot.
template <int ENV, bool INTEGRATE, bool BIN>
__global__ void __launch_bounds__(256) k_integrate_bin(
    Params P, float4* __restrict__ state_io, const float4* __restrict__ state_in,
    const float2* __restrict__ actions, uint32_t* __restrict__ cell_id,
    uint32_t* __restrict__ slot, uint32_t* __restrict__ count,
    unsigned long long* __restrict__ err, volatile uint32_t* flag,
    uint32_t* __restrict__ gather_work_n) {
  const long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= P.total) return;
  const int r = (int)(gi / P.N);
  const int i = (int)(gi - (long long)r * P.N);
  float4 s = INTEGRATE ? state_io[gi] : state_in[gi];

  // State invariants: position in [0, L), heading in [0, 2 pi), finite speed.
  bool bad = !(s.x >= 0.f && s.x < P.L && s.y >= 0.f && s.y < P.L && s.z >= 0.f &&
               s.z < P.two_pi);
  if (ENV == kFlock) bad |= !isfinite(s.w);

  if (INTEGRATE) {
    const float2 a = actions[gi];
    bad |= isnan(a.x) || isnan(a.y);
    float turn, dist;
    if (ENV == kFlock) {
      const float acc = fminf(fmaxf(a.x, -P.a_max), P.a_max);      // S:257 clamp
      turn = fminf(fmaxf(a.y, -P.theta_max), P.theta_max);
      const float sp = fminf(fmaxf(__fadd_rn(s.w, acc), P.s_min), P.s_max);  // A7
      s.w = sp;
      dist = sp;
    } else {
      turn = fminf(fmaxf(a.x, -P.theta_max), P.theta_max);
      const float smax = (i >= P.first_chaser) ? P.s_max_chaser : P.s_max;
      dist = fminf(fmaxf(a.y, 0.f), smax);
    }
    s.z = wrap_heading(__fadd_rn(s.z, turn), P.two_pi);
    float sn, cs;
    heading_sincos(s.z, P.two_pi, &sn, &cs);
    s.x = wrap_pos(s.x, __fmul_rn(dist, cs), P.L);
    s.y = wrap_pos(s.y, __fmul_rn(dist, sn), P.L);
    state_io[gi] = s;
  }
  if (bad) report_bad(err, flag, (unsigned long long)gi);

  if (BIN) {
    int cx = __float2int_rz(__fmul_rn(s.x, P.gs));
    int cy = __float2int_rz(__fmul_rn(s.y, P.gs));
    cx = min(max(cx, 0), P.G - 1);        // clamps also keep a bad state memory-safe
    cy = min(max(cy, 0), P.G - 1);
    const uint32_t c = (uint32_t)(cy * P.G + cx);
    cell_id[gi] = c;
    if (gather_work_n) {                  // K3g follows: no histogram; zero its item count
      if (gi == 0) *gather_work_n = 0u;
    } else {
      slot[gi] = atomicAdd(&count[(size_t)r * P.G2 + c], 1u);
    }
  }
}

// ---------------------------------------------------------------------------------- K2
// Exclusive scan of n counts into start[0..n] (start[n] = total) and re-zero the counts
// for the next binning.  One CTA of 1024 threads: the counts are staged in shared memory
// with coalesced loads, each thread scans a contiguous chunk there, and the results go
// back out coalesced (n <= kScanSmallMax; larger grids use K2').
#ifndef VG_SCAN_SMALL_MAX
#define VG_SCAN_SMALL_MAX 12288
#endif
constexpr int kScanSmallMax = VG_SCAN_SMALL_MAX;   // 48 KB; above it the 2-kernel K2' is faster (c5: 18,496)
// `base` (nullable): the scan starts from *base instead of 0 (a slab binning phase that
// continues an earlier one: base = start, whose [0] the earlier phase wrote as its total).
__global__ void __launch_bounds__(1024) k_scan_cells(uint32_t* __restrict__ count,
                                                      uint32_t* start, int n,
                                                      const uint32_t* base) {
  extern __shared__ uint32_t s_c[];                     // [n]
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t total_s;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t b0 = base ? *base : 0u;                // read before any thread writes start[]
  __syncthreads();
  for (int k = t; k < n; k += blockDim.x) s_c[k] = count[k];
  __syncthreads();
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b = min(n, t * per), e = min(n, b + per);
  uint32_t sum = 0;
  for (int k = b; k < e; ++k) sum += s_c[k];
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_sums[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t ws = (lane < (int)(blockDim.x >> 5)) ? warp_sums[lane] : 0u;
    uint32_t wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, wi, o);
      if (lane >= o) wi += y;
    }
    warp_sums[lane] = wi - ws;
    if (lane == 31) total_s = wi;
  }
  __syncthreads();
  uint32_t run = b0 + warp_sums[w] + inc - sum;
  for (int k = b; k < e; ++k) {
    const uint32_t c = s_c[k];
    s_c[k] = run;
    run += c;
  }
  __syncthreads();
  for (int k = t; k < n; k += blockDim.x) {
    start[k] = s_c[k];
    count[k] = 0u;
  }
  if (t == 0) start[n] = b0 + total_s;
}

// K2' (multi-CTA): tiles of 4096 counts.  k_scan_tiles sums each tile; k_scan_apply lets
// every CTA add up the sums of the tiles before it (<= a few hundred) and scans its own
// tile, writing start[] and re-zeroing the counts.  Same result as k_scan_cells.
constexpr int kScanTile = 4096;

__global__ void __launch_bounds__(1024) k_scan_tiles(const uint32_t* __restrict__ count, int n,
                                                      uint32_t* __restrict__ tile_sum) {
  __shared__ uint32_t ws[32];
  const int t = threadIdx.x, base = blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int k = base + e * 1024 + t;
    s += (k < n) ? count[k] : 0u;
  }
  s = __reduce_add_sync(kFull, s);
  if ((t & 31) == 0) ws[t >> 5] = s;
  __syncthreads();
  if (t < 32) {
    const uint32_t v = __reduce_add_sync(kFull, ws[t]);
    if (t == 0) tile_sum[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(1024) k_scan_apply(uint32_t* __restrict__ count,
                                                      uint32_t* start, int n,
                                                      const uint32_t* __restrict__ tile_sum,
                                                      const uint32_t* base0) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t s_off;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int base = blockIdx.x * kScanTile;
  if (w == 0) {                                           // offset = sum of earlier tiles
    uint32_t o = base0 ? *base0 : 0u;                     // (+ an earlier phase's total:
    if (lane != 0) o = 0u;                                //  every CTA reads the same value)
    for (int k = lane; k < (int)blockIdx.x; k += 32) o += tile_sum[k];
    o = __reduce_add_sync(kFull, o);
    if (lane == 0) s_off = o;
  }
  // 4 consecutive counts per thread (thread t owns base + 4t .. 4t+3)
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int k = base + 4 * t + e;
    v[e] = (k < n) ? count[k] : 0u;
    sum += v[e];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = ws[lane];
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, xi, o);
      if (lane >= o) xi += y;
    }
    ws[lane] = xi - x;
  }
  __syncthreads();
  uint32_t run = s_off + ws[w] + inc - sum;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int k = base + 4 * t + e;
    if (k < n) {
      start[k] = run;
      count[k] = 0u;
    }
    run += v[e];
  }
  if (blockIdx.x == gridDim.x - 1 && t == 1023) start[n] = run;
}

// ---------------------------------------------------------------------------------- K3
// Place each agent's record at cell_start[cell] + slot (arrival order within a cell).
template <int ENV>
__global__ void __launch_bounds__(256) k_scatter(
    Params P, const float4* __restrict__ state, const uint32_t* __restrict__ cell_id,
    const uint32_t* __restrict__ slot, const uint32_t* __restrict__ cell_start,
    float4* __restrict__ tmp_rec, uint32_t* __restrict__ tmp_id, uint32_t* __restrict__ work_n) {
  const long long gi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi == 0) *work_n = 0u;                          // K3b appends the K4 work items next
  if (gi >= P.total) return;
  const int r = (int)(gi / P.N);
  const int i = (int)(gi - (long long)r * P.N);
  const uint32_t pos = cell_start[(size_t)r * P.G2 + cell_id[gi]] + slot[gi];
  float4 s = state[gi];
  if (ENV == kTag) s.w = (i >= P.first_chaser) ? 1.f : 0.f;   // type in the sorted record
  tmp_rec[pos] = s;
  tmp_id[pos] = (uint32_t)i;
}

// K4 work items: K4 CTA c senses the first chunk_q queries of sensed cell c;
// a denser cell's further chunks are appended here as items (sensed-cell index, first
// query) by the binning kernel that finishes the cell (K3b, or the fused bin), and run by
// the CTAs after the first n_cells — so dense cells are split over many CTAs while the
// bulk keeps the spatial order of the cell grid.
struct WorkList {
  uint2* item;
  uint32_t* n;          // item count (zeroed by the kernel before the appending one)
  int chunk_q;
  int lo, hi;           // local cells [lo, hi) are sensed, as item cell index (cell - lo)
  // slab mode: the cells of memory columns bcol[0..nb) (sensed by the boundary-phase K4,
  // a small launch) are cut into chunks of chunk_qb queries (more, shorter work items)
  int chunk_qb, nb, G, bcol[4];
};

__device__ __forceinline__ uint32_t work_chunk_q(const WorkList& WL, int cell) {
  bool b = false;
  for (int k = 0; k < 4; ++k) b |= (k < WL.nb && WL.bcol[k] == cell / WL.G);
  return (uint32_t)(b ? WL.chunk_qb : WL.chunk_q);
}
// Overflow chunks of a cell (its chunks after the first; K4 CTA c senses the first one).
__device__ __forceinline__ uint32_t work_chunks(const WorkList& WL, int cell, uint32_t m) {
  const uint32_t cq = work_chunk_q(WL, cell);
  return (cell >= WL.lo && cell < WL.hi && m > cq) ? (m - 1u) / cq : 0u;
}

// --------------------------------------------------------------------------------- K3b
// Sub-bins for the K4 candidate windows: cell c, with axis index ca (cx on the
// row-major replica grid, cy on the column-major slab grid), is cut along its axis into kSub
// sub-bins; a record with axis key a lies in sub_bin(ca, a).  The K4 "sense order" (xo_*)
// is, within each cell, ascending (sub-bin, id): along a run of cells of one grid row
// (column) the sub-bins then ascend, and a window [klo, khi] of keys is covered by one
// contiguous range, read from sub_tab[c kSub + s] = first sense-order index of cell c in
// sub-bin >= s (sub_tab[(n_cells) kSub] = total, so sub_tab[c kSub + kSub] = next cell).
// K4 maps klo / khi with the same monotone fp32 formulas, so no key in the window is
// missed.  Outputs never depend on this order (fixed-point sums, min, counts).
// With u = RN32(a G/L) (the A16 product, so ca = min(G-1, floor(u))), the sub-bin is
// floor(kSub u) - kSub ca clamped to [0, kSub) (kSub u is exact): a monotone function of a.
#ifndef VG_SUB_BINS
#define VG_SUB_BINS 32
#endif
constexpr int kSub = VG_SUB_BINS;           // power of 2, 2..32
// VG_BIN_UNI: warp-uniform values (warp index, cell index, member count) of the binning
// kernels pass through a REDUX into uniform registers, so ptxas can prove their warp loops
// convergent (no BRA.DIV / BSSY around every ballot, shuffle and match).
#ifndef VG_BIN_UNI
#define VG_BIN_UNI 1
#endif
__device__ __forceinline__ uint32_t bin_uni(uint32_t v) {
  return VG_BIN_UNI ? __reduce_max_sync(0xffffffffu, v) : v;
}
__device__ __forceinline__ int sub_bin(const Params& P, int ca, float a) {
  const int sb = __float2int_rd(__fmul_rn(a, P.gs) * (float)kSub) - kSub * ca;
  return min(max(sb, 0), kSub - 1);
}

// Lanes of a 32-record batch whose sub-bin is `bin`: from the log2(kSub) bit ballots of the
// lanes' sub-bins (a radix-style multi-split: log2(kSub) ballots instead of kSub).
constexpr int kSubBits = (kSub >= 32) ? 5 : (kSub >= 16) ? 4 : (kSub >= 8) ? 3 : (kSub >= 4) ? 2 : 1;
static_assert((1 << kSubBits) == kSub, "kSub: a power of 2, 2..32");
__device__ __forceinline__ unsigned bin_lanes(const unsigned (&bits)[kSubBits], unsigned valid,
                                              int bin) {
  unsigned m = valid;
#pragma unroll
  for (int k = 0; k < kSubBits; ++k) m &= ((bin >> k) & 1) ? bits[k] : ~bits[k];
  return m;
}

// Sense order of one cell from its stable (id-ordered) records [b, b + m): a stable counting
// sort by sub-bin, one warp.  Writes xo_* and the cell's kSub table entries.
// The cell's records are read from sorted[rb ..] / perm[rb ..] (rb = b, or a shared-memory
// staging copy) and written to xo_*[b ..].  sense_order_place takes the sub-bin counts
// (lane s < kSub: records of the cell in sub-bin s); sense_order_cell counts them first.
template <typename PermT>
__device__ __forceinline__ void sense_order_place(const Params& P, int ca, bool axis_y,
                                                  uint32_t b, int m,
                                                  const float4* sorted, const PermT* perm,
                                                  float4* __restrict__ xo_rec,
                                                  uint32_t* __restrict__ xo_perm,
                                                  float2* __restrict__ xo_xy, uint32_t* tab,
                                                  int lane, unsigned lt, uint32_t rb,
                                                  uint32_t cnt) {
  m = (int)bin_uni((uint32_t)m);
  uint32_t inc = cnt;                                     // exclusive scan over lanes < kSub
#pragma unroll
  for (int o = 1; o < kSub; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  uint32_t run = inc - cnt;                               // lane s: records in sub-bins < s
  if (lane < kSub) tab[lane] = b + run;
  for (int ib = 0; ib < m; ib += 32) {
    const bool valid = ib + lane < m;
    float4 rec = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t id = 0u;
    int sb = 0;
    if (valid) {
      rec = sorted[rb + ib + lane];
      id = perm[rb + ib + lane];
      sb = sub_bin(P, ca, axis_y ? rec.y : rec.x);
    }
    unsigned bits[kSubBits];
#pragma unroll
    for (int k = 0; k < kSubBits; ++k) bits[k] = __ballot_sync(kFull, (sb >> k) & 1);
    const unsigned vmask = __ballot_sync(kFull, valid);
    const uint32_t pos = __shfl_sync(kFull, run, sb) + __popc(bin_lanes(bits, vmask, sb) & lt);
    if (valid) {
      xo_rec[b + pos] = rec;
      xo_perm[b + pos] = id;
      // compact positions for K4; tag: the type rides in the sign bit of x (x >= 0, so a
      // chaser at x = 0 is -0.0)
      xo_xy[b + pos] = make_float2((P.env == kTag && rec.w != 0.f) ? -rec.x : rec.x, rec.y);
    }
    run += __popc(bin_lanes(bits, vmask, lane));          // (lane < kSub used)
  }
}

template <typename PermT>
__device__ __forceinline__ void sense_order_cell(const Params& P, int ca, bool axis_y,
                                                 uint32_t b, int m,
                                                 const float4* sorted, const PermT* perm,
                                                 float4* __restrict__ xo_rec,
                                                 uint32_t* __restrict__ xo_perm,
                                                 float2* __restrict__ xo_xy, uint32_t* tab,
                                                 int lane, unsigned lt, uint32_t rb) {
  m = (int)bin_uni((uint32_t)m);
  uint32_t cnt = 0;                                       // lane s < kSub: records in sub-bin s
  for (int ib = 0; ib < m; ib += 32) {
    const bool valid = ib + lane < m;
    int sb = 0;
    if (valid) {
      const float4 rec = sorted[rb + ib + lane];
      sb = sub_bin(P, ca, axis_y ? rec.y : rec.x);
    }
    unsigned bits[kSubBits];
#pragma unroll
    for (int k = 0; k < kSubBits; ++k) bits[k] = __ballot_sync(kFull, (sb >> k) & 1);
    cnt += __popc(bin_lanes(bits, __ballot_sync(kFull, valid), lane));   // (lane < kSub used)
  }
  sense_order_place(P, ca, axis_y, b, m, sorted, perm, xo_rec, xo_perm, xo_xy, tab, lane, lt,
                    rb, cnt);
}

// Dense cells (m > kRankMax): sort the cell's (id, arrival index) pairs by id with
// 32-element bitonic blocks in registers and merge passes (merge path per output element),
// O(m log m) instead of the O(m^2) rank.  Ping-pong scratch: (keys A, vals A) -> (keys B,
// vals B) -> ...; returns the pair holding the result.  Ids are unique within a world.
constexpr int kRankMax = 128;
__device__ __forceinline__ void cell_merge_sort(uint32_t b, int m, uint32_t* ka, uint32_t* va,
                                                uint32_t* kb, uint32_t* vb, int lane,
                                                uint32_t*& kout, uint32_t*& vout) {
  for (int base = 0; base < m; base += 32) {                // ka holds the arrival ids
    uint32_t k = (base + lane < m) ? ka[b + base + lane] : 0xffffffffu;
    uint32_t v = (uint32_t)(base + lane);
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const uint32_t ok = __shfl_xor_sync(kFull, k, stride), ov = __shfl_xor_sync(kFull, v, stride);
        const bool take_min = ((lane & stride) == 0) == ((lane & size) == 0 || size == 32);
        if (take_min ? (ok < k) : (ok > k)) { k = ok; v = ov; }
      }
    }
    __syncwarp();
    if (base + lane < m) { ka[b + base + lane] = k; va[b + base + lane] = v; }
  }
  __syncwarp();
  uint32_t *sk = ka, *sv = va, *dk = kb, *dv = vb;
  for (int run = 32; run < m; run <<= 1) {
    for (int lo = 0; lo < m; lo += 2 * run) {
      const int mid = min(lo + run, m), hi = min(lo + 2 * run, m);
      const int nl = mid - lo, nr = hi - mid;
      for (int o = lane; o < hi - lo; o += 32) {
        int a = max(0, o - nr), z = min(o, nl);              // left elements among the first o
        while (a < z) {
          const int i = (a + z) >> 1;
          if (sk[b + lo + i] < sk[b + mid + o - i - 1]) a = i + 1; else z = i;
        }
        const int j = o - a;
        const bool left = j >= nr || (a < nl && sk[b + lo + a] < sk[b + mid + j]);
        const uint32_t src = left ? b + lo + a : b + mid + j;
        dk[b + lo + o] = sk[src];
        dv[b + lo + o] = sv[src];
      }
    }
    __syncwarp();
    uint32_t* t = sk; sk = dk; dk = t;
    t = sv; sv = dv; dv = t;
  }
  kout = sk;
  vout = sv;
}

// One warp per cell: rank each member by agent id (ids are unique within a replica) and
// write it to its stable slot ("ascending order (determinism anchor)"); then the
// cell's sense order (above).  Warp n_cells writes the table sentinel.
__global__ void __launch_bounds__(256) k_cell_sort(
    Params P, int n_cells, int axis_y, const uint32_t* __restrict__ cell_start,
    const float4* __restrict__ tmp_rec, const uint32_t* __restrict__ tmp_id,
    float4* __restrict__ sorted, uint32_t* __restrict__ perm, float4* __restrict__ xo_rec,
    uint32_t* __restrict__ xo_perm, float2* __restrict__ xo_xy, uint32_t* __restrict__ sub_tab,
    WorkList WL, uint32_t* __restrict__ scratch, int cell0) {
  // cells [cell0, n_cells) (slab binning phases: a range of memory columns)
  const int cell = (int)bin_uni((uint32_t)(cell0 + (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5)));
  const int lane = threadIdx.x & 31, wib = (int)bin_uni(threadIdx.x >> 5);
  // K4 work items of this block's 8 cells: one atomic per block.
  __shared__ uint32_t s_nch[8], s_base;
  const uint32_t b0 = (cell < n_cells) ? cell_start[cell] : 0u;
  const uint32_t m0 = (cell < n_cells) ? cell_start[cell + 1] - b0 : 0u;
  if (lane == 0) s_nch[wib] = (cell < n_cells) ? work_chunks(WL, cell, m0) : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int k = 0; k < 8; ++k) { const uint32_t c = s_nch[k]; s_nch[k] = t; t += c; }
    s_base = t ? atomicAdd(WL.n, t) : 0u;
  }
  __syncthreads();
  if (cell < n_cells) {
    const uint32_t nch = work_chunks(WL, cell, m0), at = s_base + s_nch[wib];
    for (uint32_t k = lane; k < nch; k += 32)
      WL.item[at + k] = make_uint2((uint32_t)(cell - WL.lo), b0 + (k + 1u) * work_chunk_q(WL, cell));
  }
  if (cell > n_cells) return;
  const uint32_t b = bin_uni(cell_start[cell]);
  if (cell == n_cells) {
    if (lane == 0) sub_tab[(size_t)n_cells * kSub] = b;
    return;
  }
  const int m = (int)bin_uni(cell_start[cell + 1] - b);
  if (m > kRankMax) {                                   // dense cell: merge sort
    uint32_t *ks, *vs;
    cell_merge_sort(b, m, const_cast<uint32_t*>(tmp_id), scratch, perm, xo_perm, lane, ks, vs);
    for (int k = lane; k < m; k += 32) {
      const uint32_t id = ks[b + k], src = vs[b + k];
      sorted[b + k] = tmp_rec[b + src];
      perm[b + k] = id;
    }
  }
  if (m <= kRankMax) {
    // Rank by id against the cell's ids staged in this warp's shared slice (4 per 16-byte
    // broadcast load; padding ids 0xffffffff never count).
    __shared__ __align__(16) uint32_t s_ids[8][kRankMax];
    for (int k = lane; k < ((m + 3) & ~3); k += 32)
      s_ids[wib][k] = (k < m) ? tmp_id[b + k] : 0xffffffffu;
    __syncwarp();
    const uint4* ids4 = reinterpret_cast<const uint4*>(s_ids[wib]);
    for (int base = 0; base < m; base += 32) {
      const int idx = base + lane;
      const bool valid = idx < m;
      const uint32_t id = valid ? s_ids[wib][idx] : 0xffffffffu;
      uint32_t rank = 0;
#pragma unroll 4
      for (int j4 = 0; j4 < (m + 3) >> 2; ++j4) {
        const uint4 o = ids4[j4];
        rank += (o.x < id ? 1u : 0u) + (o.y < id ? 1u : 0u) + (o.z < id ? 1u : 0u) +
                (o.w < id ? 1u : 0u);
      }
      if (valid) {
        sorted[b + rank] = tmp_rec[b + idx];
        perm[b + rank] = id;
      }
    }
  }
  __syncwarp();                                         // this warp's writes are visible
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  sense_order_cell(P, cell % P.G, axis_y != 0, b, m, sorted, perm, xo_rec, xo_perm, xo_xy,
                   sub_tab + (size_t)cell * kSub, lane, lt, b);
}

// K3b, one CTA per cell (worlds with few, populous cells that K3g does not take — N above
// 16,384, or slab mode — where one warp per cell leaves most SMs idle).  The same outputs as k_cell_sort:
// every member's stable slot is its rank by agent id, and its sense-order slot is its rank
// by (sub-bin, id); both ranks are counted by comparison against the cell's keys staged in
// shared memory, all threads of the CTA in parallel.  A cell above kCtaRankMax members
// falls back to warp 0 running k_cell_sort's path.
#ifndef VG_CTA_SORT_SPLIT
#define VG_CTA_SORT_SPLIT 4
#endif
constexpr int kCtaSortSplit = VG_CTA_SORT_SPLIT;       // threads sharing one member's count
constexpr int kCtaSortThreads = 128 * kCtaSortSplit;
constexpr int kCtaRankMax = 1024;
__global__ void __launch_bounds__(kCtaSortThreads) k_cell_sort_cta(
    Params P, int n_cells, int axis_y, const uint32_t* __restrict__ cell_start,
    const float4* __restrict__ tmp_rec, const uint32_t* __restrict__ tmp_id,
    float4* __restrict__ sorted, uint32_t* __restrict__ perm, float4* __restrict__ xo_rec,
    uint32_t* __restrict__ xo_perm, float2* __restrict__ xo_xy, uint32_t* __restrict__ sub_tab,
    WorkList WL, uint32_t* __restrict__ scratch, int cell0) {
  __shared__ uint2 s_key[kCtaRankMax];        // (id, sub-bin) per arrival slot
  __shared__ uint32_t s_rank[kCtaRankMax], s_pos[kCtaRankMax];
  __shared__ uint32_t s_cnt[kSub];
  // cells [cell0, n_cells) (slab binning phases: a range of memory columns)
  const int cell = cell0 + (int)blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const uint32_t b = cell_start[cell];
  if (cell == n_cells) {                                 // sentinel
    if (tid == 0) sub_tab[(size_t)n_cells * kSub] = b;
    return;
  }
  const int m = (int)(cell_start[cell + 1] - b);
  if (tid == 0) {                                        // K4 work items of this cell
    const uint32_t nch = work_chunks(WL, cell, (uint32_t)m);
    const uint32_t at = nch ? atomicAdd(WL.n, nch) : 0u;
    for (uint32_t k = 0; k < nch; ++k)
      WL.item[at + k] = make_uint2((uint32_t)(cell - WL.lo), b + (k + 1u) * work_chunk_q(WL, cell));
  }
  const int ca = cell % P.G;
  if (m > kCtaRankMax) {                                 // rare: the warp path
    if (tid >= 32) return;
    uint32_t *ks, *vs;
    cell_merge_sort(b, m, const_cast<uint32_t*>(tmp_id), scratch, perm, xo_perm, lane, ks, vs);
    for (int k = lane; k < m; k += 32) {
      const uint32_t id = ks[b + k], src = vs[b + k];
      sorted[b + k] = tmp_rec[b + src];
      perm[b + k] = id;
    }
    __syncwarp();
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    sense_order_cell(P, ca, axis_y != 0, b, m, sorted, perm, xo_rec, xo_perm, xo_xy,
                     sub_tab + (size_t)cell * kSub, lane, lt, b);
    return;
  }
  if (tid < kSub) s_cnt[tid] = 0u;
  __syncthreads();
  for (int e = tid; e < m; e += kCtaSortThreads) {
    const float4 rec = tmp_rec[b + e];
    const int sb = sub_bin(P, ca, axis_y ? rec.y : rec.x);
    s_key[e] = make_uint2(tmp_id[b + e], (uint32_t)sb);
    s_rank[e] = 0u;
    s_pos[e] = 0u;
    atomicAdd(&s_cnt[sb], 1u);
  }
  __syncthreads();
  if (tid < kSub) {                                      // sub-bin table: exclusive prefix
    uint32_t before = 0;
    for (int s = 0; s < tid; ++s) before += s_cnt[s];
    sub_tab[(size_t)cell * kSub + tid] = b + before;
  }
  // Member e's ranks by id and by (sub-bin, id), counted over kCtaSortSplit slices of the
  // cell by as many threads (slice = tid / 128) and summed in shared memory.
  {
    const int slice = tid >> 7, per = (m + kCtaSortSplit - 1) / kCtaSortSplit;
    const int j0 = slice * per, j1 = min(m, j0 + per);
    for (int e = tid & 127; e < m; e += 128) {
      const uint2 me = s_key[e];
      uint32_t rank = 0, pos = 0;
#pragma unroll 4
      for (int j = j0; j < j1; ++j) {
        const uint2 o = s_key[j];                        // broadcast
        const bool lt_id = o.x < me.x;
        rank += lt_id ? 1u : 0u;
        pos += (o.y < me.y || (o.y == me.y && lt_id)) ? 1u : 0u;
      }
      if (kCtaSortSplit == 1) {
        s_rank[e] = rank;
        s_pos[e] = pos;
      } else {
        atomicAdd(&s_rank[e], rank);
        atomicAdd(&s_pos[e], pos);
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < m; e += kCtaSortThreads) {
    const uint32_t id = s_key[e].x, rank = s_rank[e], pos = s_pos[e];
    const float4 rec = tmp_rec[b + e];
    sorted[b + rank] = rec;
    perm[b + rank] = id;
    xo_rec[b + pos] = rec;
    xo_perm[b + pos] = id;
    // compact positions for K4; tag: the type rides in the sign bit of x (as in K3b)
    xo_xy[b + pos] = make_float2((P.env == kTag && rec.w != 0.f) ? -rec.x : rec.x, rec.y);
  }
}

// K3g — K2, K3 and K3b in one kernel for small worlds (replica mode, <= 8 cells per SM,
// N <= kGatherMaxN, < 64 replicas: c1, c2, c3).  One CTA per cell c of replica r gathers its members straight
// from the cell ids K1 wrote, in agent-id order (so the stable order needs no rank): thread
// t owns agents [t S, (t+1) S); pass A counts, per thread, agents in cells before c and in
// c; one block scan gives cell_start and each thread's first slot; pass B writes the
// members.  Then the sense order by (sub-bin, id) and the sub-bin table as in K3b'.  Two
// fewer graph nodes than K1 + K2 + K3 + K3b (launch-bound worlds).
constexpr int kGatherThreads = 512;
constexpr int kGatherMaxN = kGatherThreads * 32;
template <int ENV>
__global__ void __launch_bounds__(kGatherThreads) k_cell_gather(
    Params P, int n_cells, const float4* __restrict__ state, const uint32_t* __restrict__ cell_id,
    uint32_t* __restrict__ cell_start, float4* __restrict__ sorted, uint32_t* __restrict__ perm,
    float4* __restrict__ xo_rec, uint32_t* __restrict__ xo_perm, float2* __restrict__ xo_xy,
    uint32_t* __restrict__ sub_tab, WorkList WL) {
  constexpr int T = kGatherThreads, NW = T / 32;
  __shared__ float4 s_rec[kCtaRankMax];
  __shared__ uint32_t s_id[kCtaRankMax];
  __shared__ uint8_t s_sb[kCtaRankMax];
  __shared__ uint32_t s_wa[NW > kSub ? NW : kSub], s_wb[NW], s_cnt[kSub], s_start, s_m;
  const int gc = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (gc == n_cells) {                                   // sentinels
    if (tid == 0) {
      cell_start[n_cells] = (uint32_t)P.total;
      sub_tab[(size_t)n_cells * kSub] = (uint32_t)P.total;
    }
    return;
  }
  const int r = gc / P.G2;
  const uint32_t c = (uint32_t)(gc - r * P.G2);
  const size_t base = (size_t)r * P.N;
  const int S = (P.N + T - 1) / T;
  const int i0 = min(P.N, tid * S), i1 = min(P.N, i0 + S);
  uint32_t before = 0, mine = 0;                         // pass A
#pragma unroll 8
  for (int i = i0; i < i1; ++i) {
    const uint32_t cid = cell_id[base + i];
    before += cid < c ? 1u : 0u;
    mine += cid == c ? 1u : 0u;
  }
  if (tid < kSub) s_cnt[tid] = 0u;
  uint32_t inc = mine;                                   // block exclusive scan of `mine`
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  const uint32_t bsum = __reduce_add_sync(kFull, before);
  if (lane == 31) s_wa[warp] = inc;
  if (lane == 0) s_wb[warp] = bsum;
  __syncthreads();
  if (warp == 0) {
    const uint32_t a = lane < NW ? s_wa[lane] : 0u, bb = lane < NW ? s_wb[lane] : 0u;
    uint32_t ai = a;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, ai, o);
      if (lane >= o) ai += y;
    }
    const uint32_t btot = __reduce_add_sync(kFull, bb);
    if (lane < NW) s_wa[lane] = ai - a;
    if (lane == 31) {
      s_m = ai;
      s_start = (uint32_t)base + btot;
    }
  }
  __syncthreads();
  const uint32_t start = s_start;
  const int m = (int)s_m;
  uint32_t k = s_wa[warp] + inc - mine;                  // pass B: this thread's first slot
  const int ca = (int)(c % (uint32_t)P.G);
#pragma unroll 4
  for (int i = i0; i < i1; ++i) {
    if (cell_id[base + i] != c) continue;
    float4 rec = state[base + i];
    if (ENV == kTag) rec.w = (i >= P.first_chaser) ? 1.f : 0.f;   // type in the record
    sorted[start + k] = rec;
    perm[start + k] = (uint32_t)i;
    if (k < (uint32_t)kCtaRankMax) {
      const int sb = sub_bin(P, ca, rec.x);
      s_rec[k] = rec;
      s_id[k] = (uint32_t)i;
      s_sb[k] = (uint8_t)sb;
      atomicAdd(&s_cnt[sb], 1u);
    }
    ++k;
  }
  if (tid == 0) {
    cell_start[gc] = start;
    const uint32_t nch = work_chunks(WL, gc, (uint32_t)m);   // K4 work items of this cell
    const uint32_t at = nch ? atomicAdd(WL.n, nch) : 0u;
    for (uint32_t q = 0; q < nch; ++q)
      WL.item[at + q] = make_uint2((uint32_t)(gc - WL.lo), start + (q + 1u) * (uint32_t)WL.chunk_q);
  }
  __syncthreads();                                       // sorted / perm / s_* complete
  if (m > kCtaRankMax) {                                 // rare: the warp path reads them back
    if (warp == 0) {
      unsigned lt;
      asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      sense_order_cell(P, ca, false, start, m, sorted, perm, xo_rec, xo_perm, xo_xy,
                       sub_tab + (size_t)gc * kSub, lane, lt, start);
    }
    return;
  }
  if (tid < kSub) {                                      // sub-bin table: exclusive prefix
    uint32_t b4 = 0;
    for (int q = 0; q < tid; ++q) b4 += s_cnt[q];
    sub_tab[(size_t)gc * kSub + tid] = start + b4;
    s_wa[tid] = b4;                                      // (s_wa is free again)
  }
  __syncthreads();
  for (int e = tid; e < m; e += T) {                     // sense order: by (sub-bin, id)
    const int sb = s_sb[e];
    uint32_t pos = s_wa[sb];
    for (int j = 0; j < e; ++j) pos += (s_sb[j] == sb) ? 1u : 0u;
    const float4 rec = s_rec[e];
    xo_rec[start + pos] = rec;
    xo_perm[start + pos] = s_id[e];
    // compact positions for K4; tag: the type rides in the sign bit of x (as in K3b)
    xo_xy[start + pos] = make_float2((ENV == kTag && rec.w != 0.f) ? -rec.x : rec.x, rec.y);
  }
}

// ------------------------------------------------------------------------------ K1-K3 fused
// Small replica worlds (G^2 <= 256 cells, N <= 32768, many replicas): one CTA of 1024
// threads per replica integrates (optional), bins and stably scatters its agents — the same
// results as K1 + K2 + K3 + K3b bit for bit (stable order = ascending agent id).
// Warp w owns the contiguous agent range [w S, (w+1) S) and a private per-cell count row:
//   pass 1  integrate, cell id (A16), warp-private histogram (match_any aggregated);
//   scan    per cell an exclusive scan over the 32 warps (warp shuffles), then over cells;
//   pass 2  each warp walks its range in order: position = cell start + earlier warps +
//           earlier agents of this warp in the cell + lower lanes with the same cell;
//   pass 3  warp per cell: the K4 sense order and window table (sense_order_cell, K3b).
constexpr int kRBMaxCells = 256;
constexpr int kRBMaxAgents = 32768;

#ifndef VG_RB_PREFETCH
#define VG_RB_PREFETCH 1
#endif
#ifndef VG_RB_APRE
#define VG_RB_APRE 1
#endif
#ifndef VG_RB_THREADS
#define VG_RB_THREADS 1024
#endif
constexpr int kRBThreads = VG_RB_THREADS;   // warps per replica CTA x 32; 2048 / it CTAs per SM

// MODE 0: one CTA of kRBThreads per replica (above).  MODE 1 / 2 (many replicas of N <=
// kRBStagedMax agents, e.g. c4): a persistent kernel looping over replicas with the replica
// staged in shared memory: pass 1 keeps the cell ids there; pass 2 scatters
// into a shared-memory copy of the cell-ordered records (no scattered global writes: they
// were L2-transaction bound), written out to sorted / perm as one coalesced block; pass 3
// reads the cells from that copy.
//   MODE 1: one CTA of 1024 threads per SM; the input state arrives by a 1-D TMA bulk
//           copy (issued during the previous replica's write-out and pass 3) and pass 1
//           keeps the integrated state in shared memory for pass 2.
//   MODE 2: two CTAs of 512 threads per SM (two replicas in flight, so one CTA's barriers
//           and load latencies overlap the other's work); 16-bit staging of perm and the
//           per-warp counts; the state is read through L2 (prefetched).
constexpr int kRBStagedMax = 5120;
// MODE 1: state, sorted, perm, cell id, rank + the (cell, sub-bin) histogram (two u16 a word)
constexpr int kRBStagedSmem = kRBStagedMax * (16 + 16 + 4 + 1 + 1) + kRBMaxCells * (kSub / 2) * 4;
constexpr int kRBStaged2Smem = kRBStagedMax * (16 + 2 + 1);       // MODE 2: sorted, perm (u16), cell id
constexpr int kRB2Threads = 512;
template <int MODE> struct RBCfg {
  static constexpr int NT = MODE == 2 ? kRB2Threads : kRBThreads;
  static constexpr int MINB = MODE == 1 ? 1 : MODE == 2 ? 2 : 2048 / kRBThreads;
  using WC = typename std::conditional<MODE != 0, uint16_t, uint32_t>::type;
  using PermT = typename std::conditional<MODE == 2, uint16_t, uint32_t>::type;
};

template <int ENV, bool INTEGRATE, int MODE>
__global__ void __launch_bounds__(RBCfg<MODE>::NT, RBCfg<MODE>::MINB) k_replica_bin(
    Params P, float4* __restrict__ state_io, const float4* __restrict__ state_in,
    const float2* __restrict__ actions, uint32_t* __restrict__ cell_id,
    uint32_t* __restrict__ cell_start, float4* __restrict__ sorted,
    uint32_t* __restrict__ perm, float4* __restrict__ xo_rec, uint32_t* __restrict__ xo_perm,
    float2* __restrict__ xo_xy, uint32_t* __restrict__ sub_tab, WorkList WL,
    unsigned long long* __restrict__ err, volatile uint32_t* flag) {
  constexpr bool STAGED = MODE != 0, TMA = MODE == 1;
  constexpr int NT = RBCfg<MODE>::NT;
  constexpr int NW = NT / 32;
  using PermT = typename RBCfg<MODE>::PermT;
  __shared__ typename RBCfg<MODE>::WC s_wc[NW][kRBMaxCells + 1];   // per-warp counts, then offsets (+1: banks)
  __shared__ uint32_t s_tot[kRBMaxCells];
  __shared__ __align__(8) uint64_t s_bar;                    // STAGED: input-state TMA barrier
  extern __shared__ __align__(128) unsigned char rb_dyn[];   // STAGED: see kRBStagedSmem
  const int tid = threadIdx.x, warp = (int)bin_uni(tid >> 5), lane = tid & 31;
  const int N = P.N, C = P.G2;
  const float4* src = INTEGRATE ? state_io : state_in;
  const int span = (N + NW - 1) / NW;
  const int i0 = min(N, warp * span), i1 = min(N, i0 + span);
  unsigned lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  float4* st = reinterpret_cast<float4*>(rb_dyn);                 // MODE 1: integrated, id order
  float4* s_sorted = st + (TMA ? kRBStagedMax : 0);                // cell order
  PermT* s_perm = reinterpret_cast<PermT*>(s_sorted + kRBStagedMax);
  uint8_t* s_cid = reinterpret_cast<uint8_t*>(s_perm + kRBStagedMax);
  uint8_t* s_rank = s_cid + kRBStagedMax;                          // MODE 1 (span <= 160 < 256)
  uint32_t* s_sbh = reinterpret_cast<uint32_t*>(s_rank + kRBStagedMax);   // MODE 1
  // Ask L2 for a replica's input (state, actions) up front: the warp walks its range one
  // 32-agent round at a time, so later rounds wait on L2, not HBM.  STAGED: the whole CTA
  // prefetches the next replica while processing the current one.
  auto pf = [&](const void* lo, size_t bytes, int t, int nt) {
    const uintptr_t a0 = (uintptr_t)lo & ~(uintptr_t)127, a1 = (uintptr_t)lo + bytes;
    for (uintptr_t a = a0 + 128u * (uintptr_t)t; a < a1; a += 128u * (uintptr_t)nt)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
  };
  const int r_step = STAGED ? (int)gridDim.x : P.R;
  // STAGED: the input state of each replica arrives in `st` by one 1-D TMA bulk copy
  // (cp.async.bulk + mbarrier complete_tx), issued as soon as the previous replica's pass 2
  // has read `st` (it overlaps that replica's write-out and pass 3).
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
  auto tma_state = [&](int rr) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes of st first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)N * 16u) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(st)),
        "l"(src + (size_t)rr * N), "r"((uint32_t)N * 16u), "r"(bar) : "memory");
  };
  if (STAGED && !TMA && VG_RB_PREFETCH && (int)blockIdx.x < P.R) {
    pf(src + (size_t)blockIdx.x * N, (size_t)N * sizeof(float4), tid, NT);
    if (INTEGRATE) pf(actions + (size_t)blockIdx.x * N, (size_t)N * sizeof(float2), tid, NT);
  }
  if (TMA) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;");
      if ((int)blockIdx.x < P.R) tma_state(blockIdx.x);
    }
    if (INTEGRATE && VG_RB_PREFETCH && (int)blockIdx.x < P.R)
      pf(actions + (size_t)blockIdx.x * N, (size_t)N * sizeof(float2), tid, NT);
    __syncthreads();
  }
  if (TMA) {                         // pass 3 re-zeroes each cell's counts after use
    for (int e = tid; e < kRBMaxCells * (kSub / 2); e += NT) s_sbh[e] = 0u;
    __syncthreads();
  }
  uint32_t phase = 0u;
  for (int r = blockIdx.x; r < P.R; r += r_step) {
  const size_t base = (size_t)r * N;
  for (int c = lane; c < C; c += 32) s_wc[warp][c] = 0u;
  if (VG_RB_PREFETCH) {
    if (!STAGED && i1 > i0) {
      pf(src + base + i0, (size_t)(i1 - i0) * sizeof(float4), lane, 32);
      if (INTEGRATE) pf(actions + base + i0, (size_t)(i1 - i0) * sizeof(float2), lane, 32);
    }
    if (STAGED && r + r_step < P.R) {
      const size_t nb = (size_t)(r + r_step) * N;
      if (!TMA) pf(src + nb, (size_t)N * sizeof(float4), tid, NT);
      if (INTEGRATE) pf(actions + nb, (size_t)N * sizeof(float2), tid, NT);
    }
  }
  if (TMA) {                                       // this replica's input state has landed
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "RBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra RBW_%=;\n\t}\n" ::"r"(bar), "r"(phase)
        : "memory");
    phase ^= 1u;
  }
  __syncwarp();
  // MODE 1: every round's actions are requested before the first round is integrated (one
  // L2 latency per replica instead of one per round)
  constexpr int kRounds = TMA ? (kRBStagedMax / NW + 31) / 32 : 1;
  float2 apre[kRounds];
  if (TMA && INTEGRATE && VG_RB_APRE) {
#pragma unroll
    for (int k = 0; k < kRounds; ++k) {
      const int i = i0 + 32 * k + lane;
      apre[k] = (i < i1) ? actions[base + i] : make_float2(0.f, 0.f);
    }
  }
  // ---- pass 1: integrate + cell id + warp-private histogram
#pragma unroll
  for (int kr = 0; !TMA || kr < kRounds; ++kr) {    // MODE 1: a fixed trip count (unrolled)
    const int b = i0 + 32 * kr;
    if (b >= i1) break;
    const int i = b + lane;
    const bool valid = i < i1;
    uint32_t c = 0xFFFFFFFFu;
    if (valid) {
      const size_t gi = base + i;
      float4 s = TMA ? st[i] : src[gi];
      bool bad = !(s.x >= 0.f && s.x < P.L && s.y >= 0.f && s.y < P.L && s.z >= 0.f &&
                   s.z < P.two_pi);
      if (ENV == kFlock) bad |= !isfinite(s.w);
      if (INTEGRATE) {
        const float2 a = (TMA && VG_RB_APRE) ? apre[kr] : actions[gi];
        bad |= isnan(a.x) || isnan(a.y);
        float turn, dist;
        if (ENV == kFlock) {
          const float acc = fminf(fmaxf(a.x, -P.a_max), P.a_max);
          turn = fminf(fmaxf(a.y, -P.theta_max), P.theta_max);
          const float sp = fminf(fmaxf(__fadd_rn(s.w, acc), P.s_min), P.s_max);
          s.w = sp;
          dist = sp;
        } else {
          turn = fminf(fmaxf(a.x, -P.theta_max), P.theta_max);
          const float smax = (i >= P.first_chaser) ? P.s_max_chaser : P.s_max;
          dist = fminf(fmaxf(a.y, 0.f), smax);
        }
        s.z = wrap_heading(__fadd_rn(s.z, turn), P.two_pi);
        float sn, cs;
        heading_sincos(s.z, P.two_pi, &sn, &cs);
        s.x = wrap_pos(s.x, __fmul_rn(dist, cs), P.L);
        s.y = wrap_pos(s.y, __fmul_rn(dist, sn), P.L);
        state_io[gi] = s;
      }
      if (TMA) st[i] = s;                              // pass 2 reads it back from here
      if (bad) report_bad(err, flag, (unsigned long long)gi);
      int cx = __float2int_rz(__fmul_rn(s.x, P.gs));
      int cy = __float2int_rz(__fmul_rn(s.y, P.gs));
      cx = min(max(cx, 0), P.G - 1);
      cy = min(max(cy, 0), P.G - 1);
      c = (uint32_t)(cy * P.G + cx);
      cell_id[gi] = c;
      if (STAGED) s_cid[i] = (uint8_t)c;               // re-read in pass 2 (same warp)
    }
    const unsigned grp = __match_any_sync(kFull, c);
    if (TMA) {
      // MODE 1: each record's rank among its warp's earlier records of its cell, kept for
      // pass 2 (which then has no round-to-round dependency)
      const int leader = __ffs(grp) - 1;
      uint32_t old = 0u;
      if (valid && lane == leader) {
        old = s_wc[warp][c];
        s_wc[warp][c] = old + (uint32_t)__popc(grp);
      }
      old = __shfl_sync(kFull, old, leader);
      if (valid) s_rank[i] = (uint8_t)(old + (uint32_t)__popc(grp & lt));
    } else if (valid && (grp & lt) == 0u) {
      s_wc[warp][c] += __popc(grp);
    }
    __syncwarp();
  }
  __syncthreads();
  // ---- per cell: exclusive scan over the NW warps; totals per cell
  for (int cc = tid; cc < C; cc += NT) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t t = s_wc[w][cc];
      s_wc[w][cc] = run;
      run += t;
    }
    s_tot[cc] = run;
  }
  __syncthreads();
  // ---- exclusive scan over the (<= 256) cells by warp 0: 8 consecutive cells per lane
  if (warp == 0) {
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = lane * 8 + e;
      v[e] = (c < C) ? s_tot[c] : 0u;
      sum += v[e];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = lane * 8 + e;
      if (c < C) {
        s_tot[c] = run;
        cell_start[(size_t)r * C + c] = (uint32_t)base + run;
      }
      run += v[e];
    }
    if (r == P.R - 1 && lane == 0) cell_start[(size_t)P.R * C] = (uint32_t)P.total;
    // K4 work items of this replica's cells: one atomic per replica
    uint32_t nch[8], nsum = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = lane * 8 + e;
      nch[e] = (c < C) ? work_chunks(WL, r * C + c, v[e]) : 0u;
      nsum += nch[e];
    }
    uint32_t ninc = nsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, ninc, o);
      if (lane >= o) ninc += y;
    }
    uint32_t wbase = 0u;
    if (lane == 31 && ninc > 0u) wbase = atomicAdd(WL.n, ninc);
    uint32_t at = __shfl_sync(kFull, wbase, 31) + ninc - nsum;
    uint32_t qs = (uint32_t)base + inc - sum;             // this lane's first cell start
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      for (uint32_t k = 0; k < nch[e]; ++k)
        WL.item[at + k] = make_uint2((uint32_t)(r * C + lane * 8 + e),
                                     qs + (k + 1u) * (uint32_t)WL.chunk_q);
      at += nch[e];
      qs += v[e];
    }
  }
  __syncthreads();
  // ---- pass 2: in-order walk of this warp's range, stable positions, scatter
  if (TMA) {                         // position = cell start + earlier warps + own rank
    for (int i = i0 + lane; i < i1; i += 32) {
      const uint32_t c = s_cid[i];
      const uint32_t pos = s_tot[c] + s_wc[warp][c] + (uint32_t)s_rank[i];
      float4 s = st[i];
      if (ENV == kTag) s.w = (i >= P.first_chaser) ? 1.f : 0.f;
      s_sorted[pos] = s;
      s_perm[pos] = (PermT)i;
      // the (cell, sub-bin) histogram for pass 3's sense order (no count pass there)
      const int sb = sub_bin(P, (int)(c % (uint32_t)P.G), s.x);
      atomicAdd(&s_sbh[c * (kSub / 2) + (sb >> 1)], (sb & 1) ? 65536u : 1u);
    }
  } else
  for (int b = i0; b < i1; b += 32) {
    const int i = b + lane;
    const bool valid = i < i1;
    const uint32_t c = valid ? (STAGED ? (uint32_t)s_cid[i] : cell_id[base + i]) : 0xFFFFFFFFu;
    const unsigned grp = __match_any_sync(kFull, c);
    if (valid) {
      const uint32_t pos = s_tot[c] + s_wc[warp][c] + __popc(grp & lt);
      float4 s = TMA ? st[i] : src[base + i];
      if (ENV == kTag) s.w = (i >= P.first_chaser) ? 1.f : 0.f;
      if (STAGED) {
        s_sorted[pos] = s;
        s_perm[pos] = (PermT)i;
      } else {
        sorted[base + pos] = s;
        perm[base + pos] = (uint32_t)i;
      }
    }
    __syncwarp();
    if (valid && (grp & lt) == 0u) s_wc[warp][c] += __popc(grp);
    __syncwarp();
  }
  __syncthreads();                   // the block's sorted / perm writes are now visible
  if (TMA && tid == 0 && r + r_step < P.R) tma_state(r + r_step);      // st is free again
  if (STAGED)                        // the cell-ordered replica out as one coalesced block
    for (int e = tid; e < N; e += NT) {
      sorted[base + e] = s_sorted[e];
      perm[base + e] = (uint32_t)s_perm[e];
    }
  // ---- pass 3: K4 sense order of each cell (see K3b)
  for (int c = warp; c < C; c += NW) {
    const int m = ((c + 1 < C) ? (int)s_tot[c + 1] : N) - (int)s_tot[c];
    if (TMA) {
      const uint32_t c0 = s_tot[c];
      const uint32_t w2 = (lane < kSub) ? s_sbh[c * (kSub / 2) + (lane >> 1)] : 0u;
      __syncwarp();
      if (lane < kSub / 2) s_sbh[c * (kSub / 2) + lane] = 0u;      // ready for the next replica
      sense_order_place(P, c % P.G, false, (uint32_t)base + c0, m, s_sorted, s_perm, xo_rec,
                        xo_perm, xo_xy, sub_tab + ((size_t)r * C + c) * kSub, lane, lt, c0,
                        (lane & 1) ? (w2 >> 16) : (w2 & 0xffffu));
    } else if (STAGED) {
      const uint32_t c0 = s_tot[c];
      sense_order_cell(P, c % P.G, false, (uint32_t)base + c0, m, s_sorted, s_perm,
                       xo_rec, xo_perm, xo_xy, sub_tab + ((size_t)r * C + c) * kSub, lane, lt,
                       c0);
    } else {
      sense_order_cell(P, c % P.G, false, (uint32_t)base + s_tot[c], m, sorted, perm, xo_rec,
                       xo_perm, xo_xy, sub_tab + ((size_t)r * C + c) * kSub, lane, lt,
                       (uint32_t)base + s_tot[c]);
    }
  }
  if (r == P.R - 1 && tid == 0) sub_tab[(size_t)P.R * C * kSub] = (uint32_t)P.total;
  // MODE 1 needs no barrier here: a warp done with pass 3 goes on to the next replica's
  // pass 1, which touches only its own s_wc row, s_cid / s_rank / st (pass 3 reads none of
  // them) and the new TMA'd state; s_tot and s_sorted are rewritten only after the barrier
  // that ends that pass 1, when every warp has finished this pass 3.
  if (!TMA) __syncthreads();         // s_wc, s_tot, s_cid and this buffer are reused next
  }
}


// ---------------------------------------------------------------------------------- K4
// One CTA per work item (a cell, or a chunk of a dense cell's queries); each warp takes two
// queries at a time.  The queries scan the 3x3 cell stencil — up to 6 contiguous runs of
// the sense-order arrays, each with a uniform torus image shift, each cut to the window the
// two queries can reach — for neighbours within d_v other than themselves
// (P:68); the hits are compacted with ballot/popc into one ring per query (8-byte
// (dx, dy) entries for flock sector vision, 16-byte (dx, dy, d^2, index | type) otherwise),
// and every full batch of 32 pairs takes the contact test, the reward term (fixed point,
// A16b), the bearing, the sector and the per-sector nearest distance by a shared-memory
// min on the float bits (A2, A3).  DESIGN.md §6 (v19-v21) lists each step and its measure.
#ifndef VG_SENSE_NQ
#define VG_SENSE_NQ 2
#endif
#ifndef VG_SENSE_MINB
#define VG_SENSE_MINB 7
#endif
#ifndef VG_SENSE_WARPS
#define VG_SENSE_WARPS 4
#endif
constexpr int kSenseWarps = VG_SENSE_WARPS;
constexpr int kSenseNQ = VG_SENSE_NQ;         // queries sensed together by one warp
constexpr int kSenseMinBlocks = VG_SENSE_MINB;  // launch-bounds minimum; 64 registers give 8 CTAs/SM
// Ring (power of 2): >= 31 carried + one chunk of pushes (32 per half); a second warp sync
// per chunk (after the drain) unless the ring also keeps the next chunk's pushes off the
// slots the drain read (carried + 2 x 32 halves <= ring entries, see the chunk loop).
#ifndef VG_SENSE_PAIRED
#define VG_SENSE_PAIRED 0           // sector pass: both queries' pair batches in packed pairs
#endif
#ifndef VG_SENSE_PACKED_SCAN
#define VG_SENSE_PACKED_SCAN 0      // candidate test of both queries in packed pairs
#endif
#ifndef VG_SENSE_DEF_MINB
#define VG_SENSE_DEF_MINB 8         // the flock default-constant instance: <= 64 registers, 8 CTAs/SM
#endif
#ifndef VG_SENSE_TAG_DEF_MINB
#define VG_SENSE_TAG_DEF_MINB 8     // the tag default-constant instance: <= 64 registers, 8 CTAs/SM
#endif
#ifndef VG_SENSE_HALVES
#define VG_SENSE_HALVES 2          // 32-slot halves per candidate chunk
#endif
constexpr int kSenseHalves = VG_SENSE_HALVES;
#ifndef VG_SENSE_QUEUE
#define VG_SENSE_QUEUE (VG_SENSE_HALVES > 2 ? 256 : 128)
#endif
constexpr int kQueue = VG_SENSE_QUEUE;
// Flock sector vision (E8): 8-byte ring entries (dx, dy) — d^2 is recomputed bitwise in the
// pair pass and the self pair is the entry with dx = dy = +0 (a coincident other agent is
// restored at the emit) — so the same ring bytes hold 2 kQueue entries and a chunk can be
// VG_SENSE_E8_HALVES 32-slot halves.
#ifndef VG_SENSE_E8
#define VG_SENSE_E8 1
#endif
#ifndef VG_SENSE_W2
#define VG_SENSE_W2 32
#endif
#ifndef VG_SENSE_HFORCE
#define VG_SENSE_HFORCE 2
#endif
#ifndef VG_TENT_SYM
#define VG_TENT_SYM 1
#endif
#ifndef VG_OCC_V4
#define VG_OCC_V4 1
#endif
#ifndef VG_SENSE_SCANASM
#define VG_SENSE_SCANASM 1
#endif
#ifndef VG_SENSE_W2_SLAB
#define VG_SENSE_W2_SLAB 0
#endif
// UNI: the item bounds, the stencil-run count and each run's window pass through a REDUX
// (uniform registers), so ptxas can prove the sense loops warp-uniform.
#ifndef VG_SENSE_UNI
#define VG_SENSE_UNI 1
#endif
#ifndef VG_SENSE_DRAIN_UNROLL
#define VG_SENSE_DRAIN_UNROLL 1    // ring drain loop unroll (A/B)
#endif
constexpr int kDrainUnroll = VG_SENSE_DRAIN_UNROLL;
// UCONST: the three constants of the flock pair pass that share an FFMA with another
// constant (the first atan2 coefficient, v / fov, the tent slope) held in uniform registers
// (a REDUX of the value), so ptxas need not re-create them in every 32-pair batch (48 -> 45
// instructions per batch).  Bit 0: the replica instance (DEF = 1; c4 3,603 -> 3,557 us);
// bit 1: the single-world instance (DEF = 2; with two of the three: c5 678 -> 670 us).
#ifndef VG_SENSE_UCONST
#define VG_SENSE_UCONST 3
#endif
// which of the three per instance (1 the atan2 coefficient, 2 the tent slope, 4 v / fov):
// c5 (DEF = 2) measured none 678.4, {c6} 672.8, {slope} 673.3, {v/fov} 671.6, {c6, slope}
// 671.6, {c6, v/fov} 670.6, {slope, v/fov} 670.2, all three 683 us (`gpu_run88.sh`)
#ifndef VG_SENSE_UCMASK1
#define VG_SENSE_UCMASK1 7
#endif
#ifndef VG_SENSE_UCMASK2
#define VG_SENSE_UCMASK2 6
#endif
// XYPTR: the candidate halves of a chunk load from one 64-bit pointer at immediate offsets
// (+0x100 per half) instead of an IMAD.WIDE per half: c5 k_sense 670 -> 663 us, c4 3.556 ->
// 3.445 ms (`tools/runs/gpu_run90.sh`)
// RINGB: a full drain batch addressed as (ring base + lane offset) + (head mod ring size)
// with the head in a uniform register: c5 k_sense 662 -> 652 us, c4 3.445 -> 3.424 ms
// (`tools/runs/gpu_run93.sh`)
#ifndef VG_SENSE_RINGB
#define VG_SENSE_RINGB 1
#endif
#ifndef VG_SENSE_XYPTR
#define VG_SENSE_XYPTR 1
#endif
#ifndef VG_SENSE_KITF
#define VG_SENSE_KITF 1
#endif
#ifndef VG_SENSE_NONAN
#define VG_SENSE_NONAN 1
#endif
#ifndef VG_SENSE_UNSH
#define VG_SENSE_UNSH 1
#endif
#ifndef VG_SENSE_MIXTAIL
#define VG_SENSE_MIXTAIL 1
#endif
#ifndef VG_SENSE_PREDCNT
#define VG_SENSE_PREDCNT 1
#endif
#ifndef VG_SENSE_SCANSELF
#define VG_SENSE_SCANSELF 1
#endif
#ifndef VG_SENSE_LDPRED
#define VG_SENSE_LDPRED 1
#endif
#ifndef VG_SENSE_E8_HALVES
#define VG_SENSE_E8_HALVES 4
#endif
static_assert(31 + 32 * VG_SENSE_E8_HALVES <= 2 * kQueue, "E8 ring: carried + one chunk of pushes");
// candidate slots read past a window's end (xo_xy padding): the longest chunk of any instance
constexpr int kSensePad = 32 * (VG_SENSE_E8_HALVES > kSenseHalves ? VG_SENSE_E8_HALVES : kSenseHalves);
static_assert(kQueue >= 31 + 32 * kSenseHalves, "ring: carried + one chunk of pushes");

// atan2(y, x) in (-pi, pi] with |error| <~ 3.3e-7 rad (the sector band is
// 1e-6 fov = 4.4e-6 rad): octant reduction, t = min/max by the hardware reciprocal, a
// degree-6 minimax polynomial in t^2 for atan(t)/t on [0, 1] (fit error 2.5e-7), then the
// quadrant fix-ups; atan2(+-0, +-0) = +-0.
#ifndef VG_ATAN_DEG
#define VG_ATAN_DEG 6
#endif
__device__ __forceinline__ float vg_atan2(float y, float x, float c6 = 0.006812420208007097f) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  float rc;                                 // <= 1 ulp; mx = 0 (then mn = 0) gives t = 0
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(fmaxf(mx, 1.17549435e-38f)));
  const float t = mn * rc;
  const float s = t * t;
#if VG_ATAN_DEG == 5
  // degree 5 in t^2: fit error 1.7e-6 rad; with the heading (4e-7), fwd/left (2e-7) and
  // sector-coordinate (2.6e-7) errors 2.5e-6 rad, inside the 4.36e-6 rad band (A17)
  float p = -0.011721630f;
  p = fmaf(p, s, 0.052653560f);
  p = fmaf(p, s, -0.11643203f);
  p = fmaf(p, s, 0.19354250f);
  p = fmaf(p, s, -0.33262315f);
  p = fmaf(p, s, 0.99997723f);
#else
  float p = c6;                             // 0.006812420208007097f (a caller may pass it in a uniform register)
  p = fmaf(p, s, -0.03360610455274582f);
  p = fmaf(p, s, 0.07962583005428314f);
  p = fmaf(p, s, -0.13233458995819092f);
  p = fmaf(p, s, 0.198078453540802f);
  p = fmaf(p, s, -0.3331737220287323f);
  p = fmaf(p, s, 0.9999961256980896f);
#endif
  float r = p * t;
  r = (ay > ax) ? (1.5707963705062866f - r) : r;
  r = (x < 0.f) ? (3.1415927410125732f - r) : r;
  return copysignf(r, y);
}

// Packed fp32 pairs (PTX 8.6 .f32x2, sm_100+: FADD2 / FMUL2 / FFMA2, one issue slot for two
// IEEE-rounded lane operations, bitwise equal to the scalar ops).  K4 evaluates the two
// queries of a warp in the two halves of a pair (v19).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo2(f32x2 r) {
  float a;
  asm("{\n\t.reg .f32 t;\n\tmov.b64 {%0, t}, %1;\n\t}" : "=f"(a) : "l"(r));
  return a;
}
__device__ __forceinline__ float hi2(f32x2 r) {
  float b;
  asm("{\n\t.reg .f32 t;\n\tmov.b64 {t, %0}, %1;\n\t}" : "=f"(b) : "l"(r));
  return b;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 bc2(float a) { return pk2(a, a); }

// vg_atan2 on both halves of a pair: the same operations in the same order (the polynomial,
// the products and the pi/2, pi reflections as packed ops), so each half is bitwise
// vg_atan2 of its inputs.
__device__ __forceinline__ f32x2 vg_atan2x2(f32x2 y, f32x2 x) {
  const float x0 = lo2(x), x1 = hi2(x), y0 = lo2(y), y1 = hi2(y);
  const float ax0 = fabsf(x0), ay0 = fabsf(y0), ax1 = fabsf(x1), ay1 = fabsf(y1);
  float rc0, rc1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc0) : "f"(fmaxf(fmaxf(ax0, ay0), 1.17549435e-38f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc1) : "f"(fmaxf(fmaxf(ax1, ay1), 1.17549435e-38f)));
  const f32x2 t = mul2(pk2(fminf(ax0, ay0), fminf(ax1, ay1)), pk2(rc0, rc1));
  const f32x2 s = mul2(t, t);
  f32x2 p = fma2(bc2(0.006812420208007097f), s, bc2(-0.03360610455274582f));
  p = fma2(p, s, bc2(0.07962583005428314f));
  p = fma2(p, s, bc2(-0.13233458995819092f));
  p = fma2(p, s, bc2(0.198078453540802f));
  p = fma2(p, s, bc2(-0.3331737220287323f));
  p = fma2(p, s, bc2(0.9999961256980896f));
  const f32x2 r = mul2(p, t);
  const f32x2 rf = sub2(bc2(1.5707963705062866f), r);
  const float r0 = (ay0 > ax0) ? lo2(rf) : lo2(r), r1 = (ay1 > ax1) ? hi2(rf) : hi2(r);
  const f32x2 rp = sub2(bc2(3.1415927410125732f), pk2(r0, r1));
  return pk2(copysignf((x0 < 0.f) ? lo2(rp) : r0, y0), copysignf((x1 < 0.f) ? hi2(rp) : r1, y1));
}

// K4's outputs (~0.5 KB per agent) are written once and not re-read by the step: with
// VG_SENSE_STREAM_OUT they go out as streaming stores (st.global.cs, evict-first), so the
// output stream does not push the candidate arrays out of L2.
#ifndef VG_SENSE_STREAM_OUT
#define VG_SENSE_STREAM_OUT 1
#endif
__device__ __forceinline__ void vg_st_out(float* p, float v) {
  if (VG_SENSE_STREAM_OUT) __stcs(p, v); else *p = v;
}
__device__ __forceinline__ void vg_st_out(uint32_t* p, uint32_t v) {
  if (VG_SENSE_STREAM_OUT) __stcs(reinterpret_cast<unsigned int*>(p), (unsigned int)v); else *p = v;
}

__device__ __forceinline__ uint32_t sh_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void red_min(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.min.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
// Predicated shared-memory min (no return value): one RED instruction under a predicate,
// no branch around it (the compiler's atomicMin in an `if` costs a BSSY/BRA/BSYNC).
__device__ __forceinline__ void red_min_if(bool p, uint32_t addr, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.min.u32 [%0], %1;\n\t}"
               :: "r"(addr), "r"(v), "r"((uint32_t)p) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

// A run of stencil cells along one grid row (replica) / column (slab): cells with axis
// index a0..a1, linear ids cbase + a0 .. cbase + a1.
struct __align__(16) Seg {
  float csx, csy;    // candidate image shift (0 or -L; exact by Sterbenz, A11)
  float qsx, qsy;    // query image shift (0 or -L)
  float plo, phi;    // the run's extent across its axis (shifted frame, widened by the margin)
  int cbase, a0, a1;
};

// The constants of K4's sector pass.  DEF instances take them as compile-time immediates
// for the paper's default parameters (d_v = 10, d_r = 0.25, fov = 250 deg,
// v = 128 / 64, c_collide = 1, c_near = 0.5, d_peak = 5.25, w = 0.1, s_max = 0.5), computed
// with derive()'s fp32 operations; the host uses them only when every field of the world's
// Params is bitwise equal (sense_defaults_match), so results cannot differ.  Otherwise ptxas
// re-loads these from the parameter bank in every 32-pair batch (~8 of 60 instructions).
struct SenseConst {
  float contact2, fx_mcollide, fx_k_rise, fx_b_rise, fx_nk_fall, fx_b_fall;
  float inv_w, half_v, inv_dv, dv2, w_prox, inv_smax;
  float d_r, cand2, half_fov, two_pi, d_v;         // ray vision
  int v, view_slots, obs_dim, occ_words;
  int tent_sym;
  float d_peak, fx_cnear;
};
__host__ __device__ __forceinline__ SenseConst sense_const(const Params& P) {
  return SenseConst{P.contact2, P.fx_mcollide, P.fx_k_rise, P.fx_b_rise, P.fx_nk_fall,
                    P.fx_b_fall, P.inv_w, P.half_v, P.inv_dv, P.dv2, P.w_prox, P.inv_smax,
                    P.d_r, P.cand2, P.half_fov, P.two_pi, P.d_v,
                    P.v, P.view_slots, P.obs_dim, P.occ_words,
                    P.tent_sym, P.d_peak, P.fx_cnear};
}
template <int ENV>
__host__ __device__ constexpr SenseConst sense_defaults() {
  constexpr float fov = (float)(250.0 * 3.14159265358979323846 / 180.0);
  constexpr float d_v = 10.0f, two_dr = 2.0f * 0.25f, c_near = 0.5f, d_peak = 5.25f;
  constexpr float k_rise = c_near / (d_peak - two_dr), k_fall = c_near / (d_v - d_peak);
  constexpr float fx = 4294967296.0f;
  constexpr int v = (ENV == kFlock) ? 128 : 64, ch = (ENV == kFlock) ? 1 : 2;
  return SenseConst{two_dr * two_dr, -1.0f * fx, k_rise * fx, (-k_rise * two_dr) * fx,
                    (-k_fall) * fx, (k_fall * d_v) * fx, (float)v / fov, 0.5f * (float)v,
                    1.0f / d_v, d_v * d_v, 0.1f, 1.0f / 0.5f,
                    0.25f, (d_v + 0.25f) * (d_v + 0.25f), 0.5f * fov,
                    (float)(2.0 * 3.14159265358979323846), d_v,
                    v, ch * v, ch * v + ((ENV == kFlock) ? 1 : 0), (ch * v + 31) / 32,
                    VG_TENT_SYM ? ((k_rise == k_fall) ? 1 : 0) : 0, d_peak, c_near * fx};
}

// DEF: 0 generic constants; 1 the paper's defaults as immediates (vg::sense_defaults);
// 2 the same for one large world (c5), whose chunks take VG_SENSE_HFORCE_SINGLE halves
// without the window-end skip (measured 681 vs 688 us; replica worlds (c4) 3,605 vs 3,629 us
// with VG_SENSE_HFORCE, and a kernel argument in their place measured slower for both).
#ifndef VG_SENSE_HFORCE_SINGLE
#define VG_SENSE_HFORCE_SINGLE 3
#endif
template <int ENV, bool VISION, bool SLAB, bool RAY, int DEF>
__global__ void __launch_bounds__(kSenseWarps * 32, (DEF && ENV == kTag) ? VG_SENSE_TAG_DEF_MINB : DEF ? VG_SENSE_DEF_MINB : kSenseMinBlocks) k_sense(
    Params P, const uint32_t* __restrict__ cell_start, const float4* __restrict__ sorted,
    const float2* __restrict__ sorted_xy, const uint32_t* __restrict__ perm, Outs O, Slab SL,
    const float2* __restrict__ ray_dir, const uint32_t* __restrict__ sub_tab,
    const uint2* __restrict__ work, const uint32_t* __restrict__ work_n, int chunk_q,
    int n_first) {
  // sorted / sorted_xy / perm are the sense-order arrays (xo_* of K3b): within a cell the
  // records ascend in x (replica grid, runs along rows) or y (slab grid, runs along columns).
  // per (warp, query) sector row + one spare slot (index v <= kMaxViewSlots) that absorbs
  // the minima of invisible flock pairs without a select
  constexpr int kRowW = kMaxViewSlots + 1;
  __shared__ uint32_t s_min[kSenseWarps][kSenseNQ][kRowW];
  __shared__ float2 s_ray[RAY ? kMaxViewSlots : 1];
  // Ring queues, kQueue float4 each, at shared addresses aligned to the ring size (the
  // shared window has a reserved prefix, so the alignment is done on the address).
  __shared__ float4 s_q_raw[(kSenseWarps * kSenseNQ + 1) * kQueue];
  __shared__ Seg s_seg[6];
  __shared__ int s_nseg;

  const int lane = threadIdx.x & 31;
  const int warp = VG_SENSE_UNI ? (int)__reduce_max_sync(kFull, threadIdx.x >> 5) : (int)(threadIdx.x >> 5);
  if (RAY) {
    for (int k = threadIdx.x; k < P.v; k += blockDim.x) s_ray[k] = ray_dir[k];
  }
  unsigned lt_mask;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt_mask));
  // Each warp senses NQ queries of this cell at once: every candidate load, image shift
  // and loop step is shared; each query has its own ballot, queue, sector row and
  // accumulators.  A missing query gets a NaN position (never a neighbour).
  constexpr int NQ = kSenseNQ;
  // Sector vision / reward with two queries per warp: packed candidate tests and the
  // paired pair pass (process2).  Ray vision keeps the per-query pass.
  constexpr bool PAIRED = VG_SENSE_PAIRED && !RAY && NQ == 2;
  constexpr bool PACKED_SCAN = VG_SENSE_PACKED_SCAN && NQ == 2;
  // Ring entry layout: E8 (flock sector vision) 8 bytes (dx, dy), else 16 (dx, dy, d^2, word).
  constexpr bool E8 = VG_SENSE_E8 && ENV == kFlock && !RAY && !PAIRED && !PACKED_SCAN;
  constexpr uint32_t ES = E8 ? 8u : 16u, ES_SH = E8 ? 3u : 4u;
  constexpr uint32_t kRingMask = kQueue * 16u - ES;      // byte offsets within a ring
  constexpr int HV = E8 ? VG_SENSE_E8_HALVES : kSenseHalves;   // 32-slot halves per chunk
  constexpr int HF = (DEF == 2) ? VG_SENSE_HFORCE_SINGLE : VG_SENSE_HFORCE;   // halves without the skip test
  // SS: the self pair never enters the ring — the candidate test also requires slot pj !=
  // the query's own sense-order index (an extra predicate input of the radius test), so
  // the pair pass, the counts and the emit need no self handling at all.
  constexpr bool SS = VG_SENSE_SCANSELF && !PAIRED;
  constexpr bool NONAN = VG_SENSE_NONAN && SS && !PACKED_SCAN;
  constexpr bool SCANASM = VG_SENSE_SCANASM && E8 && SS && NONAN && NQ == 2;
  // Pair-pass constants.  (ptxas sees through this empty asm and re-loads them from the
  // parameter bank per pair batch; forcing them into registers with an opaque add costs 8
  // registers and measured 4 % slower.)
  static_assert(!(DEF && !VISION), "DEF: vision passes only");
  // DEF: compile-time constants; otherwise each use reads the parameter bank (a copy of
  // the whole set held in registers costs the generic instances their occupancy).
  constexpr SenseConst D = sense_defaults<ENV>();
#define VG_SC(f) (DEF ? D.f : P.f)
  float c_contact2 = VG_SC(contact2), c_mcollide = VG_SC(fx_mcollide),
        c_k_rise = VG_SC(fx_k_rise), c_b_rise = VG_SC(fx_b_rise), c_nk_fall = VG_SC(fx_nk_fall),
        c_b_fall = VG_SC(fx_b_fall), c_inv_w = VG_SC(inv_w), c_half_v = VG_SC(half_v),
        c_inv_dv = VG_SC(inv_dv);
  if (!DEF)
    asm volatile("" : "+f"(c_contact2), "+f"(c_mcollide), "+f"(c_k_rise), "+f"(c_b_rise),
                 "+f"(c_nk_fall), "+f"(c_b_fall), "+f"(c_inv_w), "+f"(c_half_v), "+f"(c_inv_dv));
  float u_c6 = 0.006812420208007097f, u_nk_fall = c_nk_fall, u_inv_w = c_inv_w;
  if (DEF && ((VG_SENSE_UCONST >> (DEF > 0 ? DEF - 1 : 0)) & 1)) {
    constexpr int msk = (DEF == 2) ? VG_SENSE_UCMASK2 : VG_SENSE_UCMASK1;   // which of the three
    if (msk & 1) u_c6 = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(u_c6)));
    if (msk & 2) u_nk_fall = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(u_nk_fall)));
    if (msk & 4) u_inv_w = __uint_as_float(__reduce_max_sync(kFull, __float_as_uint(u_inv_w)));
  }
  // CTA c < n_first: the first chunk_q queries of sensed cell c; CTA n_first + k: overflow
  // item k (a later chunk of a dense cell).  The grid bounds the item count; surplus CTAs
  // exit at once.
  {
    uint2 item = make_uint2(blockIdx.x, 0xffffffffu);                 // y: first chunk
    if ((int)blockIdx.x >= n_first) {
      const uint32_t k = blockIdx.x - (uint32_t)n_first;
      if (k >= *work_n) return;
      item = work[k];
      if (SLAB && !slab_senses(SL, (int)item.x / P.G)) return;       // another launch's cell
      if (!SLAB && SL.snc > 0) {                                      // column-restricted launch
        const int cxi = ((int)item.x % P.G2) % P.G;
        if (cxi < SL.sc0 || cxi >= SL.sc0 + SL.snc) return;
      }
    } else if (SLAB) {                                                // this launch's k-th cell
      const int kc = (int)blockIdx.x / P.G;
      item.x = (uint32_t)(((SL.snl ? SL.scol[kc] : SL.sc0 + kc)) * P.G + (int)blockIdx.x % P.G);
    } else if (SL.snc > 0) {          // replica world, one replica: cell columns [sc0, sc0 + snc)
      item.x = (uint32_t)(((int)blockIdx.x / SL.snc) * P.G + SL.sc0 + (int)blockIdx.x % SL.snc);
    }
    const int c = (int)item.x;
  // Replica layout: cell = r G^2 + cy G + cx.  Slab layout: memory cell c = m G + cy of
  // local column lcx = slab_lcol(m).
  const int r = SLAB ? 0 : c / P.G2;
  const int cl = SLAB ? c : c - r * P.G2;
  const int cy = SLAB ? c % P.G : cl / P.G;
  const int cx = SLAB ? slab_lcol(c / P.G, SL.W) : cl - cy * P.G;
  const uint32_t* cs = cell_start + (size_t)r * P.G2;

  if (threadIdx.x == 0 && SLAB) {
    // Stencil columns lcx-1..lcx+1 of the local grid (no x-wrap: ghost columns hold the
    // neighbours).  Ghost column 0 of rank 0 is global column G-1 (candidate shift -L);
    // ghost column W+1 of the last rank is global column 0 (query shift -L) (A11).
    int ns = 0;
    const float mL = -P.L;
    for (int dxc = -1; dxc <= 1; ++dxc) {
      const int col = cx + dxc;
      const float csx = (col == 0 && SL.lo == 0) ? mL : 0.f;
      const float qsx = (col == SL.W + 1 && SL.hi == P.G) ? mL : 0.f;
      const int gcol = (SL.lo + col - 1 + P.G) % P.G;
      const float plo = (float)gcol * P.cell + csx - P.win_margin;
      const float phi = (float)(gcol + 1) * P.cell + csx + P.win_margin;
      const int base = slab_mcol(col, SL.W) * P.G;
      const int g1 = P.G - 1;
      if (cy >= 1 && cy <= P.G - 2) {
        s_seg[ns++] = Seg{csx, 0.f, qsx, 0.f, plo, phi, base, cy - 1, cy + 1};
      } else if (cy == 0) {                          // rows G-1 | 0, 1
        s_seg[ns++] = Seg{csx, mL, qsx, 0.f, plo, phi, base, g1, g1};
        s_seg[ns++] = Seg{csx, 0.f, qsx, 0.f, plo, phi, base, 0, 1};
      } else {                                       // rows G-2, G-1 | 0
        s_seg[ns++] = Seg{csx, 0.f, qsx, 0.f, plo, phi, base, P.G - 2, g1};
        s_seg[ns++] = Seg{csx, 0.f, qsx, mL, plo, phi, base, 0, 0};
      }
    }
    s_nseg = ns;
  }
  if (threadIdx.x == 0 && !SLAB) {
    int ns = 0;
    const float mL = -P.L;
    for (int dy = -1; dy <= 1; ++dy) {
      int yy = cy + dy;
      float csy = 0.f, qsy = 0.f;
      if (yy < 0) { yy += P.G; csy = mL; }           // candidate row G-1 seen from row 0
      if (yy >= P.G) { yy -= P.G; qsy = mL; }        // candidate row 0 seen from row G-1
      const int row = yy * P.G;
      const float plo = (float)yy * P.cell + csy - P.win_margin;
      const float phi = (float)(yy + 1) * P.cell + csy + P.win_margin;
      const int g1 = P.G - 1;
      if (cx >= 1 && cx <= P.G - 2) {
        s_seg[ns++] = Seg{0.f, csy, 0.f, qsy, plo, phi, row, cx - 1, cx + 1};
      } else if (cx == 0) {                          // cells G-1 | 0, 1
        s_seg[ns++] = Seg{mL, csy, 0.f, qsy, plo, phi, row, g1, g1};
        s_seg[ns++] = Seg{0.f, csy, 0.f, qsy, plo, phi, row, 0, 1};
      } else {                                       // cells G-2, G-1 | 0
        s_seg[ns++] = Seg{0.f, csy, 0.f, qsy, plo, phi, row, P.G - 2, g1};
        s_seg[ns++] = Seg{0.f, csy, mL, qsy, plo, phi, row, 0, 0};
      }
    }
    s_nseg = ns;
  }
    __syncthreads();
    const int nseg = VG_SENSE_UNI ? (int)__reduce_max_sync(kFull, (uint32_t)s_nseg) : s_nseg;
    uint32_t cq = (uint32_t)chunk_q;
    if (SLAB)
      for (int k2 = 0; k2 < 4; ++k2)
        if (k2 < SL.nb && SL.bcol[k2] == c / P.G) cq = (uint32_t)SL.chunk_qb;
    uint32_t qb = (item.y == 0xffffffffu) ? cs[cl] : item.y;
    uint32_t qe = min(cs[cl + 1], qb + cq);
    if (VG_SENSE_UNI) {
      qb = __reduce_max_sync(kFull, qb);
      qe = __reduce_max_sync(kFull, qe);
    }
    const uint32_t qstride = NQ * kSenseWarps;
    // W2: the run windows of wn = min(32 / nseg, VG_SENSE_W2) warp-iterations in one pass —
    // lane L computes run L mod nseg of iteration +L / nseg; the next wn - 1 iterations reuse
    // them (an interior cell, 3 runs: 10 iterations, i.e. every window of the warp's queries).
    // (not for slab ranks: their items are short (chunk 24: ~3 iterations per warp), and the
    // batched pass measured 0.186 -> 0.230 ms per rank at P = 8)
    constexpr bool W2 = VG_SENSE_W2 > 1 && (!SLAB || VG_SENSE_W2_SLAB);
    const int wn = W2 ? min(32 / nseg, VG_SENSE_W2) : 1;
    const float inv_nseg = 1.f / (float)nseg;
    uint32_t w2_wb = 0u, w2_we = 0u;
    int w2_left = 0;                       // iterations that still have windows in w2_*
    for (uint32_t q0 = qb + NQ * warp; q0 < qe; q0 += qstride) {
    float4 me[NQ];
    bool live[NQ];
    // Ring queue of query t: kQueue float4 entries at byte address qbase[t] (aligned to the
    // ring size, so slot addresses are qbase | (byte offset & mask)); head/tail in bytes.
    uint32_t tq[NQ], head[NQ], tail[NQ], ncol[NQ], ntouch[NQ], nnb[NQ], qbase[NQ];
    float sn[NQ], csn[NQ];
    long long rs[NQ];
#pragma unroll
    for (int t = 0; t < NQ; ++t) {
      live[t] = q0 + t < qe;
      me[t] = live[t] ? sorted[q0 + t] : make_float4(__int_as_float(0x7fc00000), 0.f, 0.f, 0.f);
      tq[t] = (ENV == kTag) ? (uint32_t)me[t].w : 0u;
      sn[t] = csn[t] = 0.f;
      if (VISION) {
        // heading in [-pi, pi) for the MUFU sin/cos (abs error ~4e-7 rad, inside the band
        // budget of 4.4e-6 rad); the subtraction is exact (Sterbenz).
        const float th = (me[t].z >= 3.14159265f) ? me[t].z - P.two_pi : me[t].z;
        __sincosf(th, &sn[t], &csn[t]);
#pragma unroll
        for (int w = 0; w < kMaxViewSlots / 32; ++w) s_min[warp][t][32 * w + lane] = kOneBits;
      }
      head[t] = tail[t] = ncol[t] = ntouch[t] = nnb[t] = 0u;
      qbase[t] = ((sh_addr(s_q_raw) + (kQueue * 16 - 1)) & ~(uint32_t)(kQueue * 16 - 1)) +
                 (uint32_t)((warp * NQ + t) * kQueue * 16);
      rs[t] = 0;
    }
    __syncwarp();

    const uint32_t srow = sh_addr(&s_min[warp][0][0]);         // this warp's sector rows
    const uint32_t seg_base = sh_addr(&s_seg[0]);
    // Ring entry at byte offset `off` of query t's ring (E8: d^2 recomputed with the scan's
    // own operation, bitwise the value it tested).
    auto ring_entry = [&](const int t, const uint32_t off) {
      if (E8) {
        const float2 v = lds64(qbase[t] | (off & kRingMask));
        return make_float4(v.x, v.y, fmaf(v.x, v.x, v.y * v.y), 0.f);
      }
      return lds128(qbase[t] | (off & kRingMask));
    };
    // FLOCK1: flock sector vision with 8-byte entries, no self pairs in the rings — the pair
    // pass on (dx, dy, d^2) for a query given by its heading (cs_, sn_), sector row offset
    // and accumulators (so the last, partial batches of both queries can share one pass).
    constexpr bool FLOCK1 = ENV == kFlock && E8 && SS && !RAY && VISION && VG_SENSE_PREDCNT;
    auto flock_pair = [&](const float4 e, const float cs_, const float sn_, const uint32_t rowoff,
                          long long& racc, uint32_t& cacc) {
      const float c_nk_fall = u_nk_fall, c_inv_w = u_inv_w;
      const float d2 = e.z;
      float d;
      asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(d2));
      // Eq. 1 / Fig. 4 (A5) in fixed point (A16b); contact (A6, inclusive) test, the term's
      // select and the contact count under one predicate
      const float tent = VG_SC(tent_sym) ? fmaf(c_nk_fall, fabsf(d - VG_SC(d_peak)), VG_SC(fx_cnear))
                                         : fminf(fmaf(c_k_rise, d, c_b_rise), fmaf(c_nk_fall, d, c_b_fall));
      float f;
      asm("{\n\t.reg .pred p;\n\tsetp.le.f32 p, %2, %3;\n\tselp.f32 %0, %4, %5, p;\n\t"
          "@p add.u32 %1, %1, 1;\n\t}"
          : "=f"(f), "+r"(cacc) : "f"(d2), "f"(c_contact2), "f"(c_mcollide), "f"(tent));
      racc += __float2ll_rn(f);
      // bearing (A3) and sector; an invisible pair updates the row's spare slot v
      const float fwd = fmaf(cs_, e.x, sn_ * e.y);
      const float left = fmaf(cs_, e.y, -sn_ * e.x);
      const int k = __float2int_rd(fmaf(vg_atan2(left, fwd, u_c6), c_inv_w, c_half_v));
      const uint32_t idx = min((uint32_t)k, (uint32_t)VG_SC(v));
      red_min(srow + rowoff + idx * 4u, __float_as_uint(fminf(d * c_inv_dv, kBelowOne)));
    };
    // Pair pass over one ring entry (dx, dy, d^2 [, index | type << 31]) of query t.
    auto process = [&](const int t, const float4 e) {
      if (FLOCK1) {
        flock_pair(e, csn[t], sn[t], (uint32_t)(t * kRowW * 4), rs[t], ncol[t]);
        return;
      }
      const uint32_t tagbits = __float_as_uint(e.w);
      // j != i.  The sector pass takes no branch for it: the self pair (always in
      // the queue exactly once, at d = 0: a contact with f = -c_collide) is counted and
      // removed exactly at the emit; it only has to be kept out of the sector minima.
      // E8 has no index: "self" is every entry at dx = dy = +0 (the self pair, and any other
      // agent at exactly the same position, whose sector slot the emit restores; nnb counts
      // them).
      const bool self = SS ? false
                      : E8 ? (__float_as_uint(e.x) | __float_as_uint(e.y)) == 0u
                           : ENV == kFlock ? tagbits == q0 + t : (tagbits & 0x7fffffffu) == q0 + t;
      if (E8 && !SS) nnb[t] += self ? 1u : 0u;
      if ((RAY || PAIRED) && self) return;
      const uint32_t tj = (ENV == kTag) ? tagbits >> 31 : 0u;
      const float d2 = e.z;
      const bool contact = d2 <= c_contact2;                          // A6 (inclusive)
      // d by the MUFU (~1 ulp; sqrt(0) = 0, subnormal d^2 -> 0).  Ray vision also needs
      // 1 / d: MUFU.RSQ without the subnormal rescale, d = d^2 / sqrt(d^2).
      float rsq = 0.f, d;
      if (RAY) {
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rsq) : "f"(d2));
        d = (d2 >= 1.17549435e-38f) ? d2 * rsq : 0.f;
      } else {
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d) : "f"(d2));
      }
      // Eq. 1 / Fig. 4 (A5): contact -> -c_collide, else the tent min(rise, fall); in
      // fixed-point units (x 2^32, A16b).
      const float tent = VG_SC(tent_sym) ? fmaf(c_nk_fall, fabsf(d - VG_SC(d_peak)), VG_SC(fx_cnear))
                                         : fminf(fmaf(c_k_rise, d, c_b_rise), fmaf(c_nk_fall, d, c_b_fall));
      float f = contact ? c_mcollide : tent;
      if (ENV == kFlock && !RAY && VG_SENSE_PREDCNT) {
        // the contact test, the term's select and the contact count under one predicate
        // (ptxas otherwise counts with an add, a predicated move and a copy)
        asm("{\n\t.reg .pred p;\n\tsetp.le.f32 p, %2, %3;\n\tselp.f32 %0, %4, %5, p;\n\t"
            "@p add.u32 %1, %1, 1;\n\t}"
            : "=f"(f), "+r"(ncol[t]) : "f"(d2), "f"(c_contact2), "f"(c_mcollide), "f"(tent));
        rs[t] += __float2ll_rn(f);
      } else if (!RAY || d2 < VG_SC(dv2)) {                                // Eq. 1: d < d_v
        if (RAY) ++nnb[t];
        if (ENV == kFlock) {
          rs[t] += __float2ll_rn(f);
          ncol[t] += contact ? 1u : 0u;
        } else {
          if (contact) {
            if (tj == tq[t]) ++ncol[t]; else ++ntouch[t];
          }
          if (tq[t] == 0u && tj == 0u) rs[t] += __float2ll_rn(VG_SC(w_prox) * f);
        }
      }
      if (VISION && RAY) {
        const float fwd = fmaf(csn[t], e.x, sn[t] * e.y);
        const float left = fmaf(csn[t], e.y, -sn[t] * e.x);
        uint32_t* row = &s_min[warp][t][tj * VG_SC(v)];
        if (d <= VG_SC(d_r)) {                          // origin inside the disc: every ray hits at 0
          for (int k = 0; k < VG_SC(v); ++k) atomicMin(&row[k], 0u);
          return;
        }
        const float phi = vg_atan2(left, fwd);
        // Angular half-width of the disc, asin(d_r / d), bounded from above (the per-ray test
        // below is exact, so the range only has to be conservative): for s = d_r/d <= 1/2,
        // asin(s) <= s (1 + s^2 (1/6 + s^2/10)); nearer discs take asinf.
        const float sr = fminf(VG_SC(d_r) * rsq, 1.f);
        const float alpha = (sr <= 0.5f)
            ? fmaf(sr * sr * sr, fmaf(sr * sr, 0.1f, 0.16666667f), sr) + 1e-6f
            : asinf(sr);
        // Sectors whose centre ray may touch the disc: psi_k in [phi - alpha, phi + alpha]
        // (also shifted by -+2 pi across the blind-spot seam), with a 1e-4-sector margin for
        // the fp32 error of phi and alpha; every ray in the range is then tested exactly.
#pragma unroll 1
        for (int wrap = -1; wrap <= 1; ++wrap) {
          const float lo = phi - alpha + wrap * VG_SC(two_pi), hi = phi + alpha + wrap * VG_SC(two_pi);
          if (hi < -VG_SC(half_fov) - 0.1f || lo > VG_SC(half_fov) + 0.1f) continue;
          const int k0 = max(0, (int)ceilf((lo + VG_SC(half_fov)) * VG_SC(inv_w) - 0.5f - 1e-4f));
          const int k1 = min(VG_SC(v) - 1, (int)floorf((hi + VG_SC(half_fov)) * VG_SC(inv_w) - 0.5f + 1e-4f));
          for (int k = k0; k <= k1; ++k) {
            const float2 ud = s_ray[k];
            const float bb = fmaf(ud.x, fwd, ud.y * left);       // along the ray
            const float pp = fmaf(ud.x, left, -ud.y * fwd);      // perpendicular offset
            const float h = (VG_SC(d_r) - pp) * (VG_SC(d_r) + pp);         // r^2 - p^2, well conditioned
            if (h >= 0.f && bb > 0.f) {
              float sh;                                          // MUFU sqrt (~1 ulp): the
              asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sh) : "f"(h));   // IEEE sqrtf's slow path
              const float tt = fmaxf(bb - sh, 0.f);              // entry distance
              if (tt < VG_SC(d_v))
                atomicMin(&row[k], __float_as_uint(fminf(tt * VG_SC(inv_dv), kBelowOne)));
            }
          }
        }
        return;
      }
      if (VISION) {
        // Bearing in the agent frame (A3): phi = atan2(h x d, h . d), CCW-positive.
        const float fwd = fmaf(csn[t], e.x, sn[t] * e.y);
        const float left = fmaf(csn[t], e.y, -sn[t] * e.x);
        // Sector coordinate (phi + fov/2) v / fov; visible iff 0 <= k < v (A3).
        const int k = __float2int_rd(fmaf(vg_atan2(left, fwd), c_inv_w, c_half_v));
        if (ENV == kFlock && SS) {
          // an invisible pair (k outside [0, v)) updates the spare slot v, never read
          const uint32_t idx = min((uint32_t)k, (uint32_t)VG_SC(v));
          red_min(srow + (uint32_t)(t * kRowW * 4) + idx * 4u,
                  __float_as_uint(fminf(d * c_inv_dv, kBelowOne)));
        } else {
          const bool vis = (unsigned)k < (unsigned)VG_SC(v) && !self;
          // Branch-free update: an invisible pair applies the no-op min(x, ~0) to slot 0.
          const uint32_t val = vis ? __float_as_uint(fminf(d * c_inv_dv, kBelowOne)) : 0xffffffffu;
          red_min(srow + (uint32_t)(t * kRowW * 4) + (uint32_t)(tj * VG_SC(v) + (vis ? k : 0)) * 4u, val);
        }
      }
    };

    // Pair pass over one queue entry of EACH query (sector vision / reward only, NQ = 2):
    // entry e0 of query 0 and e1 of query 1 in the two halves of packed fp32 pairs, so the
    // line pair of f, the bearing, the atan2 polynomial, the sector coordinate and d / d_v
    // take one FFMA2 / FMUL2 / FADD2 for both (v19).  Every half is the
    // same IEEE operation as `process` on that entry, so the outputs are bitwise those of
    // the scalar pass.  v0 / v1: the lane holds an entry of that query.
    auto process2 = [&](const float4 e0, const float4 e1, const bool v0, const bool v1) {
      const uint32_t w0 = __float_as_uint(e0.w), w1 = __float_as_uint(e1.w);
      const uint32_t id0 = (ENV == kTag) ? (w0 & 0x7fffffffu) : w0;
      const uint32_t id1 = (ENV == kTag) ? (w1 & 0x7fffffffu) : w1;
      const bool ok0 = v0 && id0 != q0, ok1 = v1 && id1 != q0 + 1u;          // j != i
      const uint32_t tj0 = (ENV == kTag) ? w0 >> 31 : 0u, tj1 = (ENV == kTag) ? w1 >> 31 : 0u;
      const bool c0 = e0.z <= c_contact2, c1 = e1.z <= c_contact2;            // A6
      float d0, d1;
      asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d0) : "f"(e0.z));
      asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(d1) : "f"(e1.z));
      const f32x2 dd = pk2(d0, d1);
      // Eq. 1 / Fig. 4 (A5) in fixed-point units (A16b): contact -> -c_collide, else the tent.
      const f32x2 rise = fma2(bc2(c_k_rise), dd, bc2(c_b_rise));
      const f32x2 fall = fma2(bc2(c_nk_fall), dd, bc2(c_b_fall));
      const float f0 = c0 ? c_mcollide : fminf(lo2(rise), lo2(fall));
      const float f1 = c1 ? c_mcollide : fminf(hi2(rise), hi2(fall));
      if (ENV == kFlock) {
        if (ok0) { rs[0] += __float2ll_rn(f0); ncol[0] += c0 ? 1u : 0u; }
        if (ok1) { rs[1] += __float2ll_rn(f1); ncol[1] += c1 ? 1u : 0u; }
      } else {
        if (ok0 && c0) { if (tj0 == tq[0]) ++ncol[0]; else ++ntouch[0]; }
        if (ok1 && c1) { if (tj1 == tq[1]) ++ncol[1]; else ++ntouch[1]; }
        const f32x2 wf = mul2(bc2(VG_SC(w_prox)), pk2(f0, f1));
        if (ok0 && tq[0] == 0u && tj0 == 0u) rs[0] += __float2ll_rn(lo2(wf));
        if (ok1 && tq[1] == 0u && tj1 == 0u) rs[1] += __float2ll_rn(hi2(wf));
      }
      if (VISION) {
        // Bearing in the agent frame (A3), CCW-positive; sector k = floor(phi v/fov + v/2).
        const f32x2 dx = pk2(e0.x, e1.x), dy = pk2(e0.y, e1.y);
        const f32x2 fwd = fma2(pk2(csn[0], csn[1]), dx, mul2(pk2(sn[0], sn[1]), dy));
        const f32x2 left = fma2(pk2(csn[0], csn[1]), dy, mul2(pk2(-sn[0], -sn[1]), dx));
        const f32x2 kk = fma2(vg_atan2x2(left, fwd), bc2(c_inv_w), bc2(c_half_v));
        const f32x2 val = mul2(dd, bc2(c_inv_dv));
        const int k0 = __float2int_rd(lo2(kk)), k1 = __float2int_rd(hi2(kk));
        red_min_if(ok0 && (unsigned)k0 < (unsigned)VG_SC(v), srow + (uint32_t)(tj0 * VG_SC(v) + k0) * 4u,
                   __float_as_uint(fminf(lo2(val), kBelowOne)));
        red_min_if(ok1 && (unsigned)k1 < (unsigned)VG_SC(v),
                   srow + (uint32_t)(kRowW * 4) + (uint32_t)(tj1 * VG_SC(v) + k1) * 4u,
                   __float_as_uint(fminf(hi2(val), kBelowOne)));
      }
    };

    // Run windows, lane-parallel: lane i < nseg computes run i's candidate window
    // [wb, we) once per warp-iteration: the queries' distance dperp across the
    // run axis bounds the reach along it to sqrt(r^2 - dperp^2); keys in the candidates' raw
    // frame.  A dead query (NaN) drops out of fminf / fmaxf (dperp -> 0: only ever wider).
    uint32_t my_wb = 0u, my_we = 0u;
    int woff = 0;                          // lane holding run 0's window of this iteration
    if (W2 && w2_left > 0) {
      my_wb = w2_wb;
      my_we = w2_we;
      woff = (wn - w2_left) * nseg;
      --w2_left;
    } else {
      int kit = 0;                           // this lane's iteration offset lane / nseg
      if (VG_SENSE_KITF) {                   // (lane + 1/2) / nseg is >= 1/12 from an integer
        kit = W2 ? __float2int_rz(((float)lane + 0.5f) * inv_nseg) : 0;
      } else {
#pragma unroll
        for (int k = 1; k < 11; ++k) kit += (lane >= k * nseg) ? 1 : 0;   // nseg >= 3: kit <= 10
      }
      const bool nxt = kit > 0;
      if (lane < wn * nseg) {
      const Seg sg = s_seg[lane - kit * nseg];
      float amin = 3.0e38f, amax = -3.0e38f, dperp = 3.0e38f;
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        float px = me[t].x, py = me[t].y;
        if (nxt) {                         // the next iteration's query t (NaN if none)
          const uint32_t qn = q0 + (uint32_t)kit * qstride + (uint32_t)t;
          const float4 rn = (qn < qe) ? sorted[qn] : make_float4(__int_as_float(0x7fc00000), 0.f, 0.f, 0.f);
          px = rn.x;
          py = rn.y;
        }
        const float qxs = px + sg.qsx, qys = py + sg.qsy;             // exact (Sterbenz)
        const float aq = SLAB ? qys : qxs, pq = SLAB ? qxs : qys;
        amin = fminf(amin, aq);
        amax = fmaxf(amax, aq);
        dperp = fminf(dperp, fmaxf(fmaxf(sg.plo - pq, pq - sg.phi), 0.f));
      }
      const float h2 = fmaf(-dperp, dperp, P.win_r2);
      if (h2 > 0.f) {                                                // else out of reach
        float wdt;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(wdt) : "f"(h2));
        wdt += P.win_margin;
        const float csa = SLAB ? sg.csy : sg.csx;
        // Sub-bin lookups (K3b table): from the sub-bin holding klo to the one holding khi,
        // clamped to the run's cells; the same monotone formula as sub_bin().
        const float ulo = __fmul_rn(amin - csa - wdt, P.gs), uhi = __fmul_rn(amax - csa + wdt, P.gs);
        const int ca_lo = min(max(__float2int_rd(ulo), sg.a0), sg.a1);
        const int ca_hi = min(max(__float2int_rd(uhi), sg.a0), sg.a1);
        const int g_lo = kSub * ca_lo + min(max(__float2int_rd(ulo * (float)kSub) - kSub * ca_lo, 0), kSub - 1);
        const int g_hi = kSub * ca_hi + min(max(__float2int_rd(uhi * (float)kSub) - kSub * ca_hi, 0), kSub - 1);
        const uint32_t* tb = sub_tab + (size_t)((SLAB ? 0 : r * P.G2) + sg.cbase) * kSub;
        my_wb = __ldg(&tb[g_lo]);
        my_we = __ldg(&tb[g_hi + 1]);
      }
      }
      if (W2) {
        w2_wb = my_wb;
        w2_we = my_we;
        w2_left = wn - 1;                  // (iterations past qe never run)
      }
    }
    for (int sgi = 0; sgi < nseg; ++sgi) {
      uint32_t wb, we;
      if (VG_SENSE_UNI) {
        const bool src = lane == woff + sgi;
        wb = __reduce_max_sync(kFull, src ? my_wb : 0u);
        we = __reduce_max_sync(kFull, src ? my_we : 0u);
      } else {
        wb = __shfl_sync(kFull, my_wb, woff + sgi);
        we = __shfl_sync(kFull, my_we, woff + sgi);
      }
      if (wb >= we) continue;                                        // warp-uniform
      Seg sg;
      {                                     // the run's image shifts: one broadcast load
        const float4 sh = lds128(seg_base + (uint32_t)(sgi * sizeof(Seg)));
        sg.csx = sh.x;
        sg.csy = sh.y;
        sg.qsx = sh.z;
        sg.qsy = sh.w;
      }
      float qx[NQ], qy[NQ];
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        qx[t] = me[t].x + sg.qsx;                                     // exact (Sterbenz)
        qy[t] = me[t].y + sg.qsy;
      }
      // UNSH: a run without image shifts (every run of an interior cell) reads the candidate
      // positions as they are (x + 0 = x: positions are >= +0); its own instance of the loop.
      auto chunk_loop = [&](auto unsh_c) {
      constexpr bool UNSH = decltype(unsh_c)::value;
      for (uint32_t p0 = wb; p0 < we; p0 += 32 * HV) {
        // Ballot the in-radius candidates of one 32-slot half and append them to each
        // query's ring ((dx, dy), or (dx, dy, d^2, index | type << 31)).
        auto scan = [&](const float cx_, const float cy_, const uint32_t word, const uint32_t pj_) {
          // PAIRED: dx, dy, d^2 of both queries as packed pairs (FADD2 with the candidate
          // broadcast, FMUL2, FFMA2), bitwise the scalar fmaf(dx, dx, dy * dy).
          f32x2 dx2 = 0ull, dy2 = 0ull, dd2 = 0ull;
          if (SCANASM) {
            // E8 + SS + NONAN, two queries: the window test once as a predicate that both
            // queries' tests take as an input; each query's test, ballot, rank and push.
            const float dxa = cx_ - qx[0], dya = cy_ - qy[0], dxb = cx_ - qx[NQ - 1], dyb = cy_ - qy[NQ - 1];
            const float d2a = fmaf(dxa, dxa, dya * dya), d2b = fmaf(dxb, dxb, dyb * dyb);
            asm volatile(
                "{\n\t.reg .pred pw, pa, pb;\n\t.reg .b32 ba, bb, ra, rb;\n\t"
                "setp.lt.u32 pw, %2, %3;\n\t"
                "setp.ne.and.u32 pa, %2, %4, pw;\n\t"
                "setp.ne.and.u32 pb, %2, %5, pw;\n\t"
                "setp.lt.and.f32 pa, %6, %8, pa;\n\t"
                "setp.lt.and.f32 pb, %7, %8, pb;\n\t"
                "vote.sync.ballot.b32 ba, pa, 0xffffffff;\n\t"
                "vote.sync.ballot.b32 bb, pb, 0xffffffff;\n\t"
                "and.b32 ra, ba, %9;\n\tpopc.b32 ra, ra;\n\t"
                "and.b32 rb, bb, %9;\n\tpopc.b32 rb, rb;\n\t"
                "shl.b32 ra, ra, 3;\n\tadd.u32 ra, ra, %0;\n\tand.b32 ra, ra, %12;\n\tor.b32 ra, ra, %10;\n\t"
                "shl.b32 rb, rb, 3;\n\tadd.u32 rb, rb, %1;\n\tand.b32 rb, rb, %12;\n\tor.b32 rb, rb, %11;\n\t"
                "@pa st.shared.v2.f32 [ra], {%13, %14};\n\t"
                "@pb st.shared.v2.f32 [rb], {%15, %16};\n\t"
                "popc.b32 ba, ba;\n\tpopc.b32 bb, bb;\n\t"
                "shl.b32 ba, ba, 3;\n\tshl.b32 bb, bb, 3;\n\t"
                "add.u32 %0, %0, ba;\n\tadd.u32 %1, %1, bb;\n\t}"
                : "+r"(tail[0]), "+r"(tail[NQ - 1])
                : "r"(pj_), "r"(we), "r"(q0), "r"(q0 + 1u), "f"(d2a), "f"(d2b),
                  "f"(VG_SC(dv2)), "r"(lt_mask), "r"(qbase[0]), "r"(qbase[NQ - 1]),
                  "r"(kRingMask), "f"(dxa), "f"(dya), "f"(dxb), "f"(dyb)
                : "memory");
            return;
          }
          if (PACKED_SCAN) {
            dx2 = sub2(bc2(cx_), pk2(qx[0], qx[NQ - 1]));
            dy2 = sub2(bc2(cy_), pk2(qy[0], qy[NQ - 1]));
            dd2 = fma2(dx2, dx2, mul2(dy2, dy2));
          }
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
            float dx, dy, d2;
            if (PACKED_SCAN) {
              dx = t ? hi2(dx2) : lo2(dx2);
              dy = t ? hi2(dy2) : lo2(dy2);
              d2 = t ? hi2(dd2) : lo2(dd2);
            } else {
              dx = cx_ - qx[t];
              dy = cy_ - qy[t];
              d2 = fmaf(dx, dx, dy * dy);
            }
            const bool in = d2 < (RAY ? VG_SC(cand2) : VG_SC(dv2)) &&             // Eq. 1: d < d_v
                            (!SS || pj_ != q0 + (uint32_t)t) &&                      // j != i
                            (!NONAN || pj_ < we);
            const unsigned bal = __ballot_sync(kFull, in);
            if (E8) {
              if (in) sts64(qbase[t] | ((tail[t] + (__popc(bal & lt_mask) << 3)) & kRingMask), dx, dy);
            } else if (in) {
              sts128(qbase[t] | ((tail[t] + (__popc(bal & lt_mask) << 4)) & kRingMask),
                     make_float4(dx, dy, d2, __uint_as_float(word)));
            }
            tail[t] += __popc(bal) << ES_SH;
          }
        };
        // HV 32-slot halves per chunk, 1 candidate per lane each (sorted_xy is padded by
        // kSensePad >= 32 HV: no load predicate); slots past the run end get a NaN
        // position, never within d_v of anyone; halves wholly past it are skipped.
        float cxh[HV], cyh[HV];
        uint32_t wh[HV];
        // XYPTR: one 64-bit address per chunk; the halves load at immediate offsets
        const float2* xyp = sorted_xy + (size_t)(p0 + lane);
#pragma unroll
        for (int h = 0; h < HV; ++h) {
          const uint32_t pj = p0 + 32u * h + lane;
          // VG_SENSE_LDPRED: halves wholly past the window end load nothing (predicated)
          const float2 o = (!VG_SENSE_LDPRED || h < (NONAN ? HF : 1) || p0 + 32u * h < we)
                               ? __ldg(VG_SENSE_XYPTR ? xyp + 32 * h : &sorted_xy[pj]) : make_float2(0.f, 0.f);
          float x = o.x;
          uint32_t tj = 0u;
          if (ENV == kTag) {                 // type in the sign bit of x (K3b)
            tj = __float_as_uint(x) & 0x80000000u;
            x = fabsf(x);
          }
          // slots past the run end: a NaN position (never within d_v), or with NONAN the
          // window test folded into the candidate test's predicate
          cxh[h] = (NONAN || pj < we) ? (UNSH ? x : x + sg.csx) : __int_as_float(0x7fc00000);   // exact (Sterbenz)
          cyh[h] = UNSH ? o.y : o.y + sg.csy;
          wh[h] = E8 ? 0u : pj | tj;
        }
#pragma unroll
        for (int h = 0; h < HV; ++h)
          // the first VG_SENSE_HFORCE halves without the skip test (a window is almost never
          // shorter; past its end the candidate predicate is false anyway)
          if (h < (NONAN ? HF : 1) || p0 + 32u * h < we) scan(cxh[h], cyh[h], wh[h], p0 + 32u * h + lane);
        __syncwarp();                       // ring pushes above are visible to the warp
        if (PAIRED) {
          // Full batches of both queries together (process2); a query's ring is drained
          // alone only when it holds >= 64 entries, so each ring carries <= 63 into the
          // next chunk (63 + 32 kSenseHalves <= kQueue - 1).
          while (tail[0] - head[0] >= 32u * 16u && tail[1] - head[1] >= 32u * 16u) {
            process2(lds128(qbase[0] | ((head[0] + lane * 16u) & (kQueue * 16 - 16))),
                     lds128(qbase[1] | ((head[1] + lane * 16u) & (kQueue * 16 - 16))), true, true);
            head[0] += 32u * 16u;
            head[1] += 32u * 16u;
          }
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
            while (tail[t] - head[t] >= 64u * 16u) {
              process(t, lds128(qbase[t] | ((head[t] + lane * 16u) & (kQueue * 16 - 16))));
              head[t] += 32u * 16u;
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
#if VG_SENSE_DRAIN_UNROLL > 1
#pragma unroll kDrainUnroll
#endif
            while (tail[t] - head[t] >= 32u * ES) {
              // RINGB: head only ever advances by whole batches from 0, so a batch never
              // wraps: lane offset + (head mod ring), a uniform add instead of an add + mask
              if (VG_SENSE_RINGB) {
                const uint32_t a = (qbase[t] + lane * ES) + (head[t] & (kQueue * 16u - 1u));
                if (E8) {
                  const float2 v = lds64(a);
                  process(t, make_float4(v.x, v.y, fmaf(v.x, v.x, v.y * v.y), 0.f));
                } else {
                  process(t, lds128(a));
                }
              } else
              process(t, ring_entry(t, head[t] + lane * ES));
              head[t] += 32u * ES;
            }
          }
        }
        // The drain above read ring entries [h, t + P) with h >= t - carried (P: this chunk's
        // pushes, <= 32 HV); the next chunk writes [t + P, t + P + 32 HV).  Without a warp
        // sync between them a write may land on an entry another lane has not read yet
        // unless carried + 2 x 32 HV <= ring entries (E8 with four halves: 31 + 256 > 256, so
        // it syncs; a warp-uniform test of this chunk's P instead measured slower).
        if ((PAIRED ? 63 : 31) + 64 * HV > (int)(kQueue * 16u / ES)) __syncwarp();
      }
      };
      const bool unsh = VG_SENSE_UNI
          ? __reduce_or_sync(kFull, (sg.csx == 0.f && sg.csy == 0.f) ? 0u : 1u) == 0u
          : (sg.csx == 0.f && sg.csy == 0.f);
      if (VG_SENSE_UNSH && unsh) chunk_loop(std::true_type{});   // warp-uniform
      else chunk_loop(std::false_type{});
    }
    __syncwarp();
    if (PAIRED) {
      // The last (partial) batches of both queries together; lanes past a ring's end hold
      // no entry of that query (v0 / v1 false: nothing is accumulated or stored).
      int n0 = (int)(tail[0] - head[0]) >> 4, n1 = (int)(tail[1] - head[1]) >> 4;
      while (n0 > 0 || n1 > 0) {                                     // warp-uniform
        process2(lds128(qbase[0] | ((head[0] + lane * 16u) & (kQueue * 16 - 16))),
                 lds128(qbase[1] | ((head[1] + lane * 16u) & (kQueue * 16 - 16))),
                 lane < n0, lane < n1);
        head[0] += 32u * 16u;
        head[1] += 32u * 16u;
        n0 -= 32;
        n1 -= 32;
      }
    } else {
      const uint32_t n0 = (tail[0] - head[0]) >> ES_SH, n1 = (tail[NQ - 1] - head[NQ - 1]) >> ES_SH;
      if (FLOCK1 && NQ == 2 && VG_SENSE_MIXTAIL && n0 + n1 <= 32u) {
        // both queries' last entries in one batch: lanes < n0 query 0, the next n1 query 1
        if (lane < n0 + n1) {
          const bool t1 = lane >= n0;
          const uint32_t off = t1 ? head[NQ - 1] + (lane - n0) * ES : head[0] + lane * ES;
          const float2 v = lds64((t1 ? qbase[NQ - 1] : qbase[0]) | (off & kRingMask));
          long long racc = 0;
          uint32_t cacc = 0u;
          flock_pair(make_float4(v.x, v.y, fmaf(v.x, v.x, v.y * v.y), 0.f), t1 ? csn[NQ - 1] : csn[0],
                     t1 ? sn[NQ - 1] : sn[0], t1 ? (uint32_t)(kRowW * 4) : 0u, racc, cacc);
          if (t1) {
            rs[NQ - 1] += racc;
            ncol[NQ - 1] += cacc;
          } else {
            rs[0] += racc;
            ncol[0] += cacc;
          }
        }
      } else {
#pragma unroll
        for (int t = 0; t < NQ; ++t)
          if (lane * ES < tail[t] - head[t]) process(t, ring_entry(t, head[t] + lane * ES));
      }
    }
    __syncwarp();

#pragma unroll
    for (int t = 0; t < NQ; ++t) {
      if (!live[t]) continue;                                        // warp-uniform
      const uint32_t q = q0 + t;
      const uint32_t nn = RAY ? __reduce_add_sync(kFull, nnb[t])
                              : (tail[t] >> ES_SH) - (SS ? 0u : 1u);   // minus the self pair
      if (E8 && !SS && VISION && __reduce_add_sync(kFull, nnb[t]) > 1u) {
        // another agent at exactly this position: its (dx, dy) = (+0, +0) entry was kept out
        // of the sector minima with the self pair's; apply it here as `process` would have
        if (lane == 0) {
          const float z = 0.f;
          const float fwd = fmaf(csn[t], z, sn[t] * z);
          const float left = fmaf(csn[t], z, -sn[t] * z);
          const int k = __float2int_rd(fmaf(vg_atan2(left, fwd), c_inv_w, c_half_v));
          if ((unsigned)k < (unsigned)VG_SC(v))
            red_min(srow + (uint32_t)(t * kRowW * 4) + (uint32_t)k * 4u, 0u);
        }
        __syncwarp();
      }
      // Warp reductions (REDUX): the int64 reward sum as three exact limb partial sums —
      // bits 0-21 and 22-43 unsigned, 44-63 signed: 32 lanes of 22 (20) bits cannot wrap 32
      // bits, so every reward validate() admits (|sum| < 2^63) is reassembled exactly.
      // the self pair's contact and -c_collide term (sector pass, see `process`), removed
      const uint32_t nc = __reduce_add_sync(kFull, ncol[t]) - ((RAY || PAIRED || SS) ? 0u : 1u);
      const uint32_t nt = (ENV == kTag) ? __reduce_add_sync(kFull, ntouch[t]) : 0u;
      const unsigned long long ur = (unsigned long long)rs[t];
      const uint32_t s_lo = __reduce_add_sync(kFull, (uint32_t)(ur & 0x3fffffu));
      const uint32_t s_mid = __reduce_add_sync(kFull, (uint32_t)((ur >> 22) & 0x3fffffu));
      const int s_top = __reduce_add_sync(kFull, (int)((long long)ur >> 44));
      long long rsum = (long long)(((unsigned long long)(long long)s_top << 44) +
                                   ((unsigned long long)s_mid << 22) + (unsigned long long)s_lo);
      if (!RAY && !PAIRED && !SS) {
        if (ENV == kFlock) rsum -= __float2ll_rn(c_mcollide);
        else if (tq[t] == 0u) rsum -= __float2ll_rn(VG_SC(w_prox) * c_mcollide);
      }
      if (ENV == kTag) {
        const long long tt = (long long)nt * P.touch_fix;
        rsum += (tq[t] == 1u) ? tt : -tt;                             // P:194 touch rule
      }
      auto emit = [&](auto fast_c) {
        constexpr bool FAST = decltype(fast_c)::value;
        using idx_t = typename std::conditional<FAST, uint32_t, size_t>::type;
        const idx_t row = SLAB ? (idx_t)q : (idx_t)r * (idx_t)P.N + (idx_t)perm[q];
        if (lane == 0) {
          if (SLAB && (FAST || O.agent_id)) O.agent_id[row] = perm[q];
          if (FAST || O.reward) O.reward[row] = __ll2float_rn(rsum) * kFixInv;
          if (FAST || O.n_neigh) O.n_neigh[row] = nn;
          if (FAST || O.n_collide) O.n_collide[row] = nc;
          if (ENV == kTag && (FAST || O.n_touch)) O.n_touch[row] = nt;
        }
        if (VISION) {
          uint32_t vals[kMaxViewSlots / 32];
#pragma unroll
          for (int w = 0; w < kMaxViewSlots / 32; ++w) {
            const int k = 32 * w + lane;
            vals[w] = (k < VG_SC(view_slots)) ? s_min[warp][t][k] : kOneBits;
          }
          if (FAST || O.obs) {
            float* orow = O.obs + row * (idx_t)VG_SC(obs_dim);
#pragma unroll
            for (int w = 0; w < kMaxViewSlots / 32; ++w)
              if (32 * w + lane < VG_SC(view_slots)) vg_st_out(&orow[32 * w + lane], __uint_as_float(vals[w]));
            if (ENV == kFlock && lane == 0) vg_st_out(&orow[VG_SC(view_slots)], me[t].w * VG_SC(inv_smax));  // A24
          }
          if (FAST || O.occ) {
            uint32_t mine = 0u, bw[kMaxViewSlots / 32];
#pragma unroll
            for (int w = 0; w < kMaxViewSlots / 32; ++w) {
              bw[w] = __ballot_sync(kFull, vals[w] < kOneBits);
              if (lane == w) mine = bw[w];
            }
            if (FAST && VG_OCC_V4 && kMaxViewSlots == 128 && VG_SC(occ_words) == 4 && O.fast == 2) {
              // four occupancy words, 16-byte aligned rows: one vector store by lane 0
              if (lane == 0)
                asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(O.occ + row * (idx_t)4),
                             "r"(bw[0]), "r"(bw[1]), "r"(bw[2]), "r"(bw[3]) : "memory");
            } else if (lane < VG_SC(occ_words)) {
              vg_st_out(&O.occ[row * (idx_t)VG_SC(occ_words) + lane], mine);
            }
          }
        }
      };
      if (O.fast) emit(std::true_type{});
      else emit(std::false_type{});
    }
    __syncwarp();
    }
  }
}


#undef VG_SC

// ------------------------------------------------------------------------- slab mode
// One world split over P ranks by x-slabs of cell columns.
// Message = {u32 count, u32 pad[3]} + float4 rec[cap] + u32 id[cap] (global agent ids).
struct SlabBufs {
  uint32_t* n_loc;         // local set size (owned + ghosts), device counter
  float4* loc_rec;         // [cap_loc]
  uint32_t* loc_id;        // [cap_loc] global agent id
  uint32_t cap_loc;
  unsigned char* send_l;   // message to the left neighbour (global columns lo-1, lo)
  unsigned char* send_r;   // message to the right neighbour (global columns hi-1, hi)
  const unsigned char* recv_l;
  const unsigned char* recv_r;
  uint32_t cap_msg;        // records per message
  uint32_t* overflow;      // device flag (VG_EOVERFLOW)
  // binning keys, computed as records enter the local set (k_slab_begin, k_slab_unpack):
  // cell_id[k] (memory-order local cell) and slot[k] (arrival slot within it, count[cell])
  uint32_t* cell_id;
  uint32_t* slot;
  uint32_t* count;
};

__device__ __forceinline__ uint32_t* msg_count(unsigned char* m) { return reinterpret_cast<uint32_t*>(m); }
__device__ __forceinline__ float4* msg_rec(unsigned char* m) { return reinterpret_cast<float4*>(m + 16); }
__device__ __forceinline__ uint32_t* msg_id(unsigned char* m, uint32_t cap) {
  return reinterpret_cast<uint32_t*>(m + 16 + 16 * (size_t)cap);
}

// Appends are warp-aggregated: one atomic per converged group of lanes (the local set and
// the messages are plain counters, hammered by every agent otherwise).
__device__ __forceinline__ uint32_t warp_reserve(uint32_t* counter) {
  const unsigned m = __activemask();
  const int leader = __ffs(m) - 1;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0u;
  if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(m));
  base = __shfl_sync(m, base, leader);
  return base + (uint32_t)__popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ uint32_t loc_append(const SlabBufs& B, float4 s, uint32_t id) {
  const uint32_t k = warp_reserve(B.n_loc);
  if (k < B.cap_loc) { B.loc_rec[k] = s; B.loc_id[k] = id; }
  else atomicExch(B.overflow, 1u);
  return k;
}

__device__ __forceinline__ void msg_append(unsigned char* m, uint32_t cap, uint32_t* ovf,
                                           float4 s, uint32_t id) {
  const uint32_t k = warp_reserve(msg_count(m));
  if (k < cap) { msg_rec(m)[k] = s; msg_id(m, cap)[k] = id; }
  else atomicExch(ovf, 1u);
}

__device__ __forceinline__ int global_col(const Params& P, float x) {
  return min(max(__float2int_rz(__fmul_rn(x, P.gs)), 0), P.G - 1);   // A16
}

// Binning key of local record k (memory-order local cell, A16 global formula) and its
// arrival slot in the cell's histogram; warp-aggregated (records arrive cell-major).
__device__ __forceinline__ void slab_key(const Params& P, const Slab& SL, const SlabBufs& B,
                                         uint32_t k, float4 s) {
  const int gx = global_col(P, s.x), gy = global_col(P, s.y);
  const int lcx = min((gx - SL.lo + 1 + P.G) % P.G, SL.W + 1);
  const uint32_t c = (uint32_t)(slab_mcol(lcx, SL.W) * P.G + gy);
  const unsigned grp = __match_any_sync(__activemask(), c);
  const int lane = threadIdx.x & 31, leader = __ffs(grp) - 1;
  uint32_t base = 0u;
  if (lane == leader) base = atomicAdd(&B.count[c], (uint32_t)__popc(grp));
  base = __shfl_sync(grp, base, leader);
  if (k < B.cap_loc) {
    B.cell_id[k] = c;
    B.slot[k] = base + (uint32_t)__popc(grp & ((1u << lane) - 1u));
  }
}

// Route one post-integrate agent of this rank: owned columns stay local; columns lo-1 / hi
// (migrants, <= 1 column per step since s_max < cell size) stay local as ghosts and go to
// the neighbour that now owns them; boundary columns lo / hi-1 go to the neighbour as ghosts.
__device__ __forceinline__ void slab_route(const Params& P, const Slab& SL, const SlabBufs& B,
                                           float4 s, uint32_t id, unsigned long long* err,
                                           volatile uint32_t* flag) {
  const int d = (global_col(P, s.x) - SL.lo + P.G) % P.G;   // column offset from lo
  if (d > SL.W && d != P.G - 1) {                            // moved more than one column
    report_bad(err, flag, id);
    return;
  }
  slab_key(P, SL, B, loc_append(B, s, id), s);
  if (d == 0 || d == P.G - 1) msg_append(B.send_l, B.cap_msg, B.overflow, s, id);
  if (d == SL.W - 1 || d == SL.W) msg_append(B.send_r, B.cap_msg, B.overflow, s, id);
}

// Begin a slab step: integrate the owned rows (the previous binning's owned range, in row
// order; actions[row]) exactly as K1 does, then route them.
template <int ENV>
__global__ void __launch_bounds__(256) k_slab_begin(
    Params P, Slab SL, SlabBufs B, const uint32_t* __restrict__ cell_start,
    const float4* __restrict__ sorted, const uint32_t* __restrict__ perm,
    const float2* __restrict__ actions, unsigned long long* err, volatile uint32_t* flag) {
  const uint32_t own_b = 0u;                              // owned: memory columns 0..W-1
  const uint32_t n_own = cell_start[SL.W * P.G];
  for (uint32_t row = blockIdx.x * blockDim.x + threadIdx.x; row < n_own;
       row += gridDim.x * blockDim.x) {
    float4 s = sorted[own_b + row];
    const uint32_t id = perm[own_b + row];
    const float2 a = actions[row];
    bool bad = isnan(a.x) || isnan(a.y);
    float turn, dist;
    if (ENV == kFlock) {
      const float acc = fminf(fmaxf(a.x, -P.a_max), P.a_max);
      turn = fminf(fmaxf(a.y, -P.theta_max), P.theta_max);
      const float sp = fminf(fmaxf(__fadd_rn(s.w, acc), P.s_min), P.s_max);
      s.w = sp;
      dist = sp;
    } else {
      turn = fminf(fmaxf(a.x, -P.theta_max), P.theta_max);
      const float smax = (id >= (uint32_t)P.first_chaser) ? P.s_max_chaser : P.s_max;
      dist = fminf(fmaxf(a.y, 0.f), smax);
    }
    s.z = wrap_heading(__fadd_rn(s.z, turn), P.two_pi);
    float sn, cs;
    heading_sincos(s.z, P.two_pi, &sn, &cs);
    s.x = wrap_pos(s.x, __fmul_rn(dist, cs), P.L);
    s.y = wrap_pos(s.y, __fmul_rn(dist, sn), P.L);
    if (bad) report_bad(err, flag, id);
    slab_route(P, SL, B, s, id, err, flag);
  }
}

// Initial distribution: every rank reads the full global state and keeps what it owns
// plus its two ghost columns (no exchange needed).
template <int ENV>
__global__ void __launch_bounds__(256) k_slab_load(Params P, Slab SL, SlabBufs B,
                                                   const float4* __restrict__ state,
                                                   unsigned long long* err,
                                                   volatile uint32_t* flag) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (uint32_t)P.N;
       i += gridDim.x * blockDim.x) {
    const float4 s = state[i];
    bool bad = !(s.x >= 0.f && s.x < P.L && s.y >= 0.f && s.y < P.L && s.z >= 0.f &&
                 s.z < P.two_pi);
    if (ENV == kFlock) bad |= !isfinite(s.w);
    if (bad) { report_bad(err, flag, i); continue; }
    const int d = (global_col(P, s.x) - SL.lo + P.G) % P.G;
    if (d <= SL.W || d == P.G - 1) loc_append(B, s, i);
  }
}

// Append the records received from both neighbours to the local set.
__global__ void __launch_bounds__(256) k_slab_unpack(Params P, Slab SL, SlabBufs B) {
  const uint32_t nl = min(*reinterpret_cast<const uint32_t*>(B.recv_l), B.cap_msg);
  const uint32_t nr = min(*reinterpret_cast<const uint32_t*>(B.recv_r), B.cap_msg);
  if (*reinterpret_cast<const uint32_t*>(B.recv_l) > B.cap_msg ||
      *reinterpret_cast<const uint32_t*>(B.recv_r) > B.cap_msg) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(B.overflow, 1u);
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl + nr;
       i += gridDim.x * blockDim.x) {
    const unsigned char* m = (i < nl) ? B.recv_l : B.recv_r;
    const uint32_t k = (i < nl) ? i : i - nl;
    const float4 s = reinterpret_cast<const float4*>(m + 16)[k];
    slab_key(P, SL, B, loc_append(B, s, reinterpret_cast<const uint32_t*>(m + 16 + 16 * (size_t)B.cap_msg)[k]), s);
  }
}

// Local cell ids (memory column order, A16 global formula) + histogram slot of the local
// set, for the columns of one binning phase: 0 = interior (memory columns < W-2), 1 =
// boundary + ghosts (>= W-2), 2 = all.  Records of the other phase get kNoCell.
constexpr uint32_t kNoCell = 0xffffffffu;
__global__ void __launch_bounds__(256) k_slab_keys(Params P, Slab SL, SlabBufs B,
                                                   uint32_t* __restrict__ cell_id,
                                                   uint32_t* __restrict__ slot,
                                                   uint32_t* __restrict__ count, int phase) {
  const uint32_t n = min(*B.n_loc, B.cap_loc);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    const float4 s = B.loc_rec[i];
    const int gx = global_col(P, s.x), gy = global_col(P, s.y);
    const int lcx = min((gx - SL.lo + 1 + P.G) % P.G, SL.W + 1);
    const int m = slab_mcol(lcx, SL.W);
    if (phase != 2 && (m < SL.W - 2) != (phase == 0)) {
      cell_id[i] = kNoCell;
      continue;
    }
    const uint32_t c = (uint32_t)(m * P.G + gy);
    cell_id[i] = c;
    // The local set is in the previous sense order (cell-major), so a warp's agents share
    // few cells: one atomic per cell group (match_any), slots by lane rank within it.
    const unsigned grp = __match_any_sync(__activemask(), c);
    const int lane = threadIdx.x & 31, leader = __ffs(grp) - 1;
    uint32_t base = 0u;
    if (lane == leader) base = atomicAdd(&count[c], (uint32_t)__popc(grp));
    base = __shfl_sync(grp, base, leader);
    slot[i] = base + (uint32_t)__popc(grp & ((1u << lane) - 1u));
  }
}

template <int ENV>
__global__ void __launch_bounds__(256) k_slab_scatter(Params P, SlabBufs B,
                                                      const uint32_t* __restrict__ cell_id,
                                                      const uint32_t* __restrict__ slot,
                                                      const uint32_t* __restrict__ cell_start,
                                                      float4* __restrict__ tmp_rec,
                                                      uint32_t* __restrict__ tmp_id,
                                                      uint32_t* __restrict__ work_n,
                                                      int reset_work, uint32_t c_lo,
                                                      uint32_t c_hi) {
  // K3b appends the K4 items next (the boundary phase keeps the interior phase's items)
  if (reset_work && blockIdx.x == 0 && threadIdx.x == 0) *work_n = 0u;
  const uint32_t n = min(*B.n_loc, B.cap_loc);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x) {
    const uint32_t c = cell_id[i];
    if (c < c_lo || c >= c_hi) continue;                     // the other binning phase's
    const uint32_t pos = cell_start[c] + slot[i];
    float4 s = B.loc_rec[i];
    const uint32_t id = B.loc_id[i];
    if (ENV == kTag) s.w = (id >= (uint32_t)P.first_chaser) ? 1.f : 0.f;
    tmp_rec[pos] = s;
    tmp_id[pos] = id;
  }
}

}  // namespace vg
