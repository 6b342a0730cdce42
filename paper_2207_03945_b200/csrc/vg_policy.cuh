// vg_policy.cuh — K7: shared-policy actor-critic forward on the sm_100a tensor cores.
//
// P:212 "The actor and critic PPO networks had two hidden layers with 64 nodes each";
// P:198 shared policy, continuous actions; S:329-333 MLPPolicy (obs -> 64 -> 64 -> out,
// tanh hidden, linear out, state-independent log_std); S:355-372 Gaussian sample, clip to
// the action box, log-prob of the unclipped sample.  SURVEY.md §8f NEXT #1.
//
// Tiles of 128 agents; a persistent CTA (one per SM, 16 warps) runs two tiles at once: warp
// group g (8 warps) owns every other tile of the CTA, its own A operand buffer and its own
// 256 TMEM columns, so one group's MMAs, TMA waits and epilogues overlap the other's.
// Per tile:
//   layer 1  D[128 x 128] = A1[128 x 144] . B1^T   (actor | critic hidden, fp16 in, fp32 acc)
//   layer 2  D[128 x 128] = A2[128 x 128] . B2^T   (B2 block-diagonal: actor | critic)
//   layer 3  D[128 x 16]  = A3[128 x 128] . B3^T   (rows of B3: W3[0], W3[1], V3, zeros)
//   then Philox4x32-10 + Box-Muller noise, clip, log-prob.
// Operands live in shared memory in the canonical K-major no-swizzle layout (8 x 16-byte
// core matrices: SBO = 128 B between 8-row groups, LBO = R x 16 B between 8-column groups),
// tcgen05.mma is issued by one thread, the fp32 accumulator lives in TMEM (128 columns) and
// is read back with tcgen05.ld.32x32b (warp w reads TMEM lanes 32 (w % 4) ..).  One fp32
// staging buffer receives each tile by TMA; the group that owns the tile converts it to its
// fp16 operand and then issues the TMA of the CTA's next tile (the other group's).
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace vg {

constexpr int kPolTile = 128;      // agents per tile (MMA M)
constexpr int kPolHidden = 64;
constexpr int kPolN = 128;         // actor | critic concatenated (MMA N)
constexpr int kPolK1 = 144;        // obs_dim padded to a multiple of 16 (<= 144)
constexpr int kPolK2 = 128;        // hidden actor | critic
constexpr int kPolN3 = 16;         // layer-3 MMA N: mean_0, mean_1, value, 13 zero rows
constexpr int kPolThreads = 512;   // 2 groups x 8 warps: TMEM lane quadrant (w % 4) x column half
constexpr int kPolGroup = 256;     // threads per group

// Shared-memory carve-up (bytes).  Per group one operand buffer A: A1 (layer 1), A2 and A3
// all alias it — each is written only after the MMA reading the previous one has completed.
constexpr int kOffB1 = 0;
constexpr int kOffB2 = kOffB1 + kPolN * kPolK1 * 2;        // 36864
constexpr int kOffB3 = kOffB2 + kPolN * kPolK2 * 2;        // +32768
constexpr int kOffA = kOffB3 + kPolN3 * kPolK2 * 2;        // +4096: A[0], A[1]
constexpr int kABytes = kPolTile * kPolK1 * 2;             // 36864
constexpr int kOffC = kOffA + 2 * kABytes;                 // fp32 constants
// consts: b1[128] b2[128] | b3_0 b3_1 c3 pad | log_std[2] | lo[2] hi[2]
constexpr int kConstFloats = 128 + 128 + 4 + 2 + 4;
// VG_POL_QUARTERS: each tile's obs arrive as four 32-row TMA copies with a barrier each, and
// a quarter of the stage is re-filled with the next tile's rows as soon as it is converted
// (the next tile's transfer overlaps this tile's conversion instead of following it).
#ifndef VG_POL_QUARTERS
#define VG_POL_QUARTERS 0
#endif
constexpr int kPolQ = VG_POL_QUARTERS > 1 ? VG_POL_QUARTERS : VG_POL_QUARTERS ? 4 : 1;   // TMA pieces per tile (1, 2, 4)
constexpr int kOffBar = kOffC + ((kConstFloats * 4 + 15) / 16) * 16;   // mbarriers + tmem slot
constexpr int kBarBytes = 8 * (2 + 2 * kPolQ) + 16;
constexpr int kOffStage = ((kOffBar + kBarBytes + 127) / 128) * 128;     // raw fp32 obs tile (TMA)
constexpr int kStageBytes = kPolTile * kPolK1 * 4;                       // >= 128 rows x obs_dim
constexpr int kPolSmem = kOffStage + kStageBytes;

// Packed weights on the device (written once by k_policy_pack).
struct PolicyPacked {
  __half* B1;        // [kPolN x kPolK1] core-matrix layout
  __half* B2;        // [kPolN x kPolK2] core-matrix layout (block diagonal)
  __half* B3;        // [kPolN3 x kPolK2] core-matrix layout
  float* consts;     // kConstFloats (see above)
};

struct PolicyOut {
  float* mean;       // [M][2]
  float* value;      // [M]
  float* action;     // [M][2] clipped sample (NULL: skip sampling)
  float* logp;       // [M]
};

// Element offset of (r, k) in an R-row K-major core-matrix operand.
__host__ __device__ __forceinline__ int cm_offset(int r, int k, int R) {
  return ((k >> 3) * (R >> 3) + (r >> 3)) * 64 + (r & 7) * 8 + (k & 7);
}

// UMMA shared-memory descriptor: K-major, no swizzle, version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Instruction descriptors, kind::f16: D fp32, A/B fp16, both K-major, M = 128, N = 128 / 16.
constexpr uint32_t kPolIdesc = (1u << 4) | ((uint32_t)(kPolN >> 3) << 17) | ((uint32_t)(kPolTile >> 4) << 24);
constexpr uint32_t kPolIdesc3 = (1u << 4) | ((uint32_t)(kPolN3 >> 3) << 17) | ((uint32_t)(kPolTile >> 4) << 24);

__device__ __forceinline__ uint32_t h2_bits(__half2 h) {
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// tanh(x) = sign(x) (2 / (1 + exp(-2|x|)) - 1), absolute error ~2e-7 (tanh.approx.f32 is
// ~1e-3 absolute, too coarse for the parity budget).
// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier (tx bytes).
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes,
                                            uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

#ifndef VG_TANH_NEWTON
#define VG_TANH_NEWTON 1
#endif
// Hidden-layer tanh: 0 = tanh_fast (fp32, ~2e-7, then rounded to the fp16 operand),
// 1 = tanh.approx.f32 (one MUFU), 2 = tanh.approx.f16x2 on the fp16-rounded pre-activation
// (one MUFU per two units; the result is the fp16 operand itself).
#ifndef VG_TANH_MODE
#define VG_TANH_MODE 1
#endif
__device__ __forceinline__ float tanh_fast(float x) {
#if VG_TANH_NEWTON
  // One MUFU op: e = 2^(-2|x| log2 e) in (0, 1], y = 1 + e in (1, 2], 1/y from a linear
  // start (|rel err| <= 0.09) and three Newton steps on the FMA pipe (9e-8), tanh|x| =
  // 2/y - 1; the SFU (16 lanes/clk) was the K7 limiter with ex2 + rcp.  |error| ~2e-7.
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(x) * -2.8853900817779268f));
  const float y = 1.f + e;
  float r = fmaf(-0.5f, y, 1.4571f);
#pragma unroll
  for (int i = 0; i < 3; ++i) r = fmaf(r, fmaf(-y, r, 1.f), r);
  return copysignf(fmaf(2.f, r, -1.f), x);
#else
  const float e = __expf(2.f * fabsf(x));
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.f));
  return copysignf(fmaf(-2.f, r, 1.f), x);
#endif
}

// 32 consecutive TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  v[0] = __uint_as_float(r0); v[1] = __uint_as_float(r1);
  v[2] = __uint_as_float(r2); v[3] = __uint_as_float(r3);
}

// Philox4x32-10 (Salmon et al. SC'11): the same counter-based generator as oracle/policy.py.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Pack fp32 weights (nn.Linear layout [out][in]) into the resident operand layouts.
__global__ void k_policy_pack(int obs_dim, const float* __restrict__ W1, const float* __restrict__ b1,
                              const float* __restrict__ W2, const float* __restrict__ b2,
                              const float* __restrict__ W3, const float* __restrict__ b3,
                              const float* __restrict__ log_std, const float* __restrict__ V1,
                              const float* __restrict__ c1, const float* __restrict__ V2,
                              const float* __restrict__ c2, const float* __restrict__ V3,
                              const float* __restrict__ c3, float lo0, float lo1, float hi0,
                              float hi1, PolicyPacked pk) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < kPolN * kPolK1) {                                   // B1: rows 0-63 actor, 64-127 critic
    const int n = t / kPolK1, k = t % kPolK1;
    float v = 0.f;
    if (k < obs_dim) v = (n < kPolHidden) ? W1[n * obs_dim + k] : V1[(n - kPolHidden) * obs_dim + k];
    pk.B1[cm_offset(n, k, kPolN)] = __float2half_rn(v);
  }
  if (t < kPolN * kPolK2) {                                   // B2: block diagonal
    const int n = t / kPolK2, k = t % kPolK2;
    float v = 0.f;
    if (n < kPolHidden && k < kPolHidden) v = W2[n * kPolHidden + k];
    if (n >= kPolHidden && k >= kPolHidden) v = V2[(n - kPolHidden) * kPolHidden + (k - kPolHidden)];
    pk.B2[cm_offset(n, k, kPolN)] = __float2half_rn(v);
  }
  if (t < kPolN3 * kPolK2) {                                  // B3: W3[0], W3[1], V3, zeros
    const int n = t / kPolK2, k = t % kPolK2;
    float v = 0.f;
    if (n < 2 && k < kPolHidden) v = W3[n * kPolHidden + k];
    if (n == 2 && k >= kPolHidden) v = V3[k - kPolHidden];
    pk.B3[cm_offset(n, k, kPolN3)] = __float2half_rn(v);
  }
  if (t < kPolN) {
    pk.consts[t] = (t < kPolHidden) ? b1[t] : c1[t - kPolHidden];
    pk.consts[128 + t] = (t < kPolHidden) ? b2[t] : c2[t - kPolHidden];
  }
  if (t == 0) {
    pk.consts[256] = b3[0]; pk.consts[257] = b3[1]; pk.consts[258] = c3[0]; pk.consts[259] = 0.f;
    // log_std clamped to [-5, 2] (both the sample scale and the log-prob use it)
    pk.consts[260] = fminf(fmaxf(log_std[0], -5.f), 2.f);
    pk.consts[261] = fminf(fmaxf(log_std[1], -5.f), 2.f);
    pk.consts[262] = lo0; pk.consts[263] = lo1; pk.consts[264] = hi0; pk.consts[265] = hi1;
  }
}

__device__ __forceinline__ void group_sync(int g) {      // named barrier of one warp group
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kPolGroup) : "memory");
}

// Row classes (per-type policies): with cls_period > 0, row r is of class
// ((r mod cls_period) >= cls_split) and only rows of class `cls` are written (the tiles are
// all computed: a tag world's runner and chaser rows share tiles at every replica edge).
__global__ void __launch_bounds__(kPolThreads, 1) k_policy(
    const float* __restrict__ obs, int64_t M, int obs_dim, PolicyPacked pk, PolicyOut out,
    uint32_t seed_lo, uint32_t seed_hi, uint32_t step_lo, uint32_t step_hi,
    int64_t cls_period, int64_t cls_split, int cls) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __half* sB1 = reinterpret_cast<__half*>(smem + kOffB1);
  __half* sB2 = reinterpret_cast<__half*>(smem + kOffB2);
  __half* sB3 = reinterpret_cast<__half*>(smem + kOffB3);
  float* sC = reinterpret_cast<float*>(smem + kOffC);
  const float* sStage = reinterpret_cast<const float*>(smem + kOffStage);
  // mbarriers: [g] MMA completion of group g; [2 + g kPolQ + q] TMA arrival of piece q of
  // group g's tiles (a barrier per group keeps each one's phases in its own tile order).
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + 8 * (2 + 2 * kPolQ));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp >> 3, gw = warp & 7, gtid = tid & (kPolGroup - 1);
  __half* sA = reinterpret_cast<__half*>(smem + kOffA + g * kABytes);

  // Resident weights: plain 16-byte copies of the packed operands.
  {
    const uint4* g1 = reinterpret_cast<const uint4*>(pk.B1);
    const uint4* g2 = reinterpret_cast<const uint4*>(pk.B2);
    const uint4* g3 = reinterpret_cast<const uint4*>(pk.B3);
    uint4* s1 = reinterpret_cast<uint4*>(sB1);
    uint4* s2 = reinterpret_cast<uint4*>(sB2);
    uint4* s3 = reinterpret_cast<uint4*>(sB3);
    for (int i = tid; i < kPolN * kPolK1 / 8; i += kPolThreads) s1[i] = g1[i];
    for (int i = tid; i < kPolN * kPolK2 / 8; i += kPolThreads) s2[i] = g2[i];
    for (int i = tid; i < kPolN3 * kPolK2 / 8; i += kPolThreads) s3[i] = g3[i];
    for (int i = tid; i < kConstFloats; i += kPolThreads) sC[i] = pk.consts[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 2 + 2 * kPolQ; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot + (uint32_t)(g * 256);   // D: +0..127, D3: +128..143
  const uint32_t bar_mma = smem_u32(&bar[g]), bar_tma = smem_u32(&bar[2 + g * kPolQ]);
  const uint32_t bar_tma_next = smem_u32(&bar[2 + (1 - g) * kPolQ]);   // the other group's
  const uint32_t stage = smem_u32(sStage);
  const uint32_t a = smem_u32(sA);
  const uint32_t b1 = smem_u32(sB1), b2 = smem_u32(sB2), b3 = smem_u32(sB3);
  uint32_t ph_mma = 0;

  // Epilogue mapping: warp gw of the group reads TMEM lanes (rows) 32 (gw % 4) .. (the lane
  // quadrant of its CTA warp id) and columns 64 (gw / 4) ..
  const int erow = 32 * (gw & 3) + lane;
  const int ecol = 64 * (gw >> 2);
  const uint32_t tlane = (uint32_t)(32 * (gw & 3)) << 16;

  const int64_t n_tiles = (M + kPolTile - 1) / kPolTile;
  // A full tile is one contiguous, 16-byte aligned block of 128 x obs_dim floats (m0 is a
  // multiple of 128): one TMA bulk copy.  Only the last tile of the range can be ragged; it
  // is read with plain loads (and, being the last, never precedes a TMA'd tile).
  const uint32_t tile_bytes = (uint32_t)(kPolTile * obs_dim * 4);
  const bool bulk_ok = (tile_bytes % 16u) == 0u &&
                       (reinterpret_cast<uintptr_t>(obs) % 16u) == 0u;
  auto is_full = [&](int64_t t) { return bulk_ok && (t + 1) * kPolTile <= M; };
  const uint32_t piece_bytes = tile_bytes / kPolQ;         // 32 rows x obs_dim x 4 (16 | it)
  if (tid == 0 && blockIdx.x < n_tiles && is_full(blockIdx.x))     // group 0's first tile
    for (int q = 0; q < kPolQ; ++q)
      tma_load_1d(stage + q * piece_bytes,
                  obs + ((int64_t)blockIdx.x * kPolTile + q * (kPolTile / kPolQ)) * obs_dim,
                  piece_bytes, bar_tma + 8u * q);

  // MMA issue (one thread per group): ksteps K-steps of 16 from A (128 rows), B (rb rows).
  auto issue = [&](uint32_t d, uint32_t aa, uint32_t b, int ksteps, int rb, uint32_t idesc) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int k = 0; k < ksteps; ++k)
      mma_f16(d, umma_desc(aa + k * 2 * (kPolTile * 16), kPolTile * 16, 128),
              umma_desc(b + k * 2 * (rb * 16), rb * 16, 128), idesc, k > 0);
    mma_commit(bar_mma);
  };
  auto wait_mma = [&]() {
    mbar_wait(bar_mma, ph_mma);
    ph_mma ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
  };
  // Epilogue of a hidden layer: h = tanh(D + bias) -> fp16 operand of the next layer (A).
  auto hidden_epilogue = [&](const float* bias) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float v[32];
      const int cb = ecol + 32 * half;
      tmem_ld32(tmem + tlane + (uint32_t)cb, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c0 = cb + 8 * q;
        uint4 pkd;
#if VG_TANH_MODE == 2
        // The activation feeds an fp16 operand: z + b rounded to fp16 pairs, then one
        // packed MUFU tanh.approx.f16x2 per two units (test_policy bound).
        uint32_t hz[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t zz = h2_bits(__floats2half2_rn(v[8 * q + 2 * e] + bias[c0 + 2 * e],
                                                        v[8 * q + 2 * e + 1] + bias[c0 + 2 * e + 1]));
          asm("tanh.approx.f16x2 %0, %1;" : "=r"(hz[e]) : "r"(zz));
        }
        pkd.x = hz[0]; pkd.y = hz[1]; pkd.z = hz[2]; pkd.w = hz[3];
#else
        float t[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
#if VG_TANH_MODE == 1
          asm("tanh.approx.f32 %0, %1;" : "=f"(t[e]) : "f"(v[8 * q + e] + bias[c0 + e]));
#else
          t[e] = tanh_fast(v[8 * q + e] + bias[c0 + e]);
#endif
        }
        pkd.x = h2_bits(__floats2half2_rn(t[0], t[1]));
        pkd.y = h2_bits(__floats2half2_rn(t[2], t[3]));
        pkd.z = h2_bits(__floats2half2_rn(t[4], t[5]));
        pkd.w = h2_bits(__floats2half2_rn(t[6], t[7]));
#endif
        *reinterpret_cast<uint4*>(sA + cm_offset(erow, c0, kPolTile)) = pkd;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    group_sync(g);
  };

  uint32_t ph_tma = 0;
  for (int64_t tile = blockIdx.x + (int64_t)g * gridDim.x; tile < n_tiles;
       tile += 2 * (int64_t)gridDim.x) {
    const int64_t m0 = tile * kPolTile;
    const bool full = is_full(tile);
    // ---- A1: obs rows -> fp16 core-matrix layout (zero pad rows >= M, cols >= obs_dim),
    // one TMA piece (kPolTile / kPolQ rows) at a time.
    const int64_t nt = tile + gridDim.x;                 // the CTA's next tile (other group's)
    constexpr int kPR = kPolTile / kPolQ;                // rows per piece
    for (int q = 0; q < kPolQ; ++q) {
    if (full) mbar_wait(bar_tma + 8u * q, ph_tma);       // this piece's TMA has landed
    // Thread -> (row r, 8-column chunk kc); a warp shares kc, so the chunk bounds are uniform.
    for (int it = gtid; it < kPR * (kPolK1 / 8); it += kPolGroup) {
      const int r = q * kPR + it % kPR, kc = it / kPR;
      const int nv = obs_dim - kc * 8;                    // valid columns in this chunk
      const int64_t gr = m0 + r;
      float x[8];
      if (full) {
        const float* src = sStage + r * obs_dim + kc * 8;
        if (nv >= 8) {
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = src[e];
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = (e < nv) ? src[e] : 0.f;
        }
      } else {
        const float* src = obs + gr * obs_dim + kc * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = (gr < M && e < nv) ? __ldg(src + e) : 0.f;
      }
      uint4 pkd;
      pkd.x = h2_bits(__floats2half2_rn(x[0], x[1]));
      pkd.y = h2_bits(__floats2half2_rn(x[2], x[3]));
      pkd.z = h2_bits(__floats2half2_rn(x[4], x[5]));
      pkd.w = h2_bits(__floats2half2_rn(x[6], x[7]));
      *reinterpret_cast<uint4*>(sA + cm_offset(r, kc * 8, kPolTile)) = pkd;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (q == kPolQ - 1) asm volatile("tcgen05.fence::before_thread_sync;");
    group_sync(g);
    // ---- this piece of the stage is free: load the next tile's rows into it
    if (gtid == 0 && nt < n_tiles && is_full(nt))
      tma_load_1d(stage + q * piece_bytes, obs + (nt * kPolTile + q * kPR) * obs_dim,
                  piece_bytes, bar_tma_next + 8u * q);
    }
    if (full) ph_tma ^= 1u;
    // ---- layer 1
    if (gtid == 0) issue(tmem, a, b1, kPolK1 / 16, kPolN, kPolIdesc);
    wait_mma();
    hidden_epilogue(sC);                                 // h1 -> A (A1 consumed)
    // ---- layer 2
    if (gtid == 0) issue(tmem, a, b2, kPolK2 / 16, kPolN, kPolIdesc);
    wait_mma();
    hidden_epilogue(sC + 128);                           // h2 -> A (A2 consumed)
    // ---- layer 3: mean_0, mean_1, value in TMEM columns +128..130
    if (gtid == 0) issue(tmem + 128, a, b3, kPolK2 / 16, kPolN3, kPolIdesc3);
    wait_mma();
    if (gw < 4) {                                        // one thread per row
      float o[4];
      tmem_ld4(tmem + tlane + 128u, o);
      const int64_t gr = m0 + erow;
      const bool mine = cls_period <= 0 || ((gr % cls_period) >= cls_split) == (cls == 1);
      if (gr < M && mine) {
        const float mu0 = o[0] + sC[256], mu1 = o[1] + sC[257];
        if (out.value) out.value[gr] = o[2] + sC[258];
        if (out.mean) { out.mean[2 * gr] = mu0; out.mean[2 * gr + 1] = mu1; }
        if (out.action) {
          uint32_t c[4] = {(uint32_t)gr, step_lo, step_hi, 0u};
          philox4x32_10(c, seed_lo, seed_hi);
          const float u0 = ((float)(c[0] >> 8) + 0.5f) * 5.9604645e-8f;     // (0, 1)
          const float u1 = ((float)(c[1] >> 8) + 0.5f) * 5.9604645e-8f;
          const float rr = sqrtf(-2.f * logf(u0));
          float sn, cs;
          sincospif(2.f * u1, &sn, &cs);
          const float e0 = rr * cs, e1 = rr * sn;
          const float ls0 = sC[260], ls1 = sC[261];
          const float r0 = fmaf(expf(ls0), e0, mu0), r1 = fmaf(expf(ls1), e1, mu1);
          out.action[2 * gr] = fminf(fmaxf(r0, sC[262]), sC[264]);
          out.action[2 * gr + 1] = fminf(fmaxf(r1, sC[263]), sC[265]);
          if (out.logp)
            out.logp[gr] = -0.5f * (e0 * e0 + e1 * e1) - ls0 - ls1 - 1.8378770664093453f;
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    group_sync(g);                                       // TMEM / A free for the next tile
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(512));
}

}  // namespace vg
