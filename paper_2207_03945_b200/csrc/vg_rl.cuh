// vg_rl.cuh — the two NEXT rows that are plain data-parallel passes:
//   K8  k_gae      generalized advantage estimation over the on-device trajectory buffer
//                  (NEXT #3): reverse recursion over t, one thread
//                  per agent, time-major [t][n] layout -> coalesced, HBM-bound.
//   K9  k_opinion  Listing 1 bounded-confidence graph interaction + self
//                  interaction (NEXT #4): one thread per node folds its out-edges
//                  (CSR sorted by (src, dst)) in edge order into new_opinion.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vg {

// A[k] = delta[k] + (gamma lambda) A[k+1], A[t] = 0, delta[k] = r[k] + gamma V[k+1] - V[k];
// R[k] = A[k] + V[k].  (The recursion equals S:376's direct sum; oracle/gae.py.)
__global__ void __launch_bounds__(256) k_gae(const float* __restrict__ r,
                                             const float* __restrict__ v, int64_t n, int t,
                                             float gamma, float gl, float* __restrict__ adv,
                                             float* __restrict__ ret) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float vnext = __ldcs(v + (int64_t)t * n + i);
    float g = 0.f;
    int k = t - 1;
    for (; k >= 7; k -= 8) {                       // 16 independent loads in flight
      float rr[8], vv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        rr[j] = __ldcs(r + (int64_t)(k - j) * n + i);
        vv[j] = __ldcs(v + (int64_t)(k - j) * n + i);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = fmaf(gamma, vnext, rr[j]) - vv[j];
        g = fmaf(gl, g, d);
        __stcs(adv + (int64_t)(k - j) * n + i, g);
        __stcs(ret + (int64_t)(k - j) * n + i, g + vv[j]);
        vnext = vv[j];
      }
    }
    for (; k >= 0; --k) {
      const float rk = __ldcs(r + (int64_t)k * n + i), vk = __ldcs(v + (int64_t)k * n + i);
      const float d = fmaf(gamma, vnext, rk) - vk;
      g = fmaf(gl, g, d);
      __stcs(adv + (int64_t)k * n + i, g);
      __stcs(ret + (int64_t)k * n + i, g + vk);
      vnext = vk;
    }
  }
}

// Listing 1: for each edge (me = src, you = dst, weight) in (src, dst) order:
//   if |me.opinion - you.opinion| < threshold: w = strength weight;
//      me.new_opinion = (1 - w) me.new_opinion + w you.opinion
// with new_opinion starting at the current opinion and every read of `opinion`
// from the previous step (simultaneous update); then opinion <- new_opinion.
// First node whose row or edges are invalid (row_ptr not non-decreasing within [0, E], or
// col outside [0, n)): reported by vg_opinion_sync_errors ("a dangling index is an
// invariant violation").  Invalid edges are never read.
__device__ unsigned long long g_opinion_bad = ~0ull;

__global__ void __launch_bounds__(256) k_opinion(const int32_t* __restrict__ row_ptr,
                                                 const int32_t* __restrict__ col,
                                                 const float* __restrict__ weight, int n,
                                                 long long n_edges,
                                                 const float* __restrict__ op,
                                                 float* __restrict__ op_new, float threshold,
                                                 float strength) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float x = op[i];
    float acc = x;
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    if (e0 < 0 || e1 < e0 || (long long)e1 > n_edges) {
      atomicMin(&g_opinion_bad, (unsigned long long)i);
      op_new[i] = x;
      continue;
    }
    for (int e = e0; e < e1; ++e) {
      const int c = __ldg(col + e);
      if ((unsigned)c >= (unsigned)n) {
        atomicMin(&g_opinion_bad, (unsigned long long)i);
        continue;
      }
      const float y = __ldg(op + c);
      if (fabsf(x - y) < threshold) {
        const float w = strength * __ldg(weight + e);
        acc = fmaf(w, y, (1.f - w) * acc);
      }
    }
    op_new[i] = acc;
  }
}

}  // namespace vg
