// adam_body.cuh — K10 Adam element loop (R19), see k_optim.cu.
#pragma once
#include "internal.h"

namespace spk {

// The body of adam_kernel for CTA `cta` of `ncta` (grid-stride over the elements, bias corrections once
// per CTA, the last CTA to finish stores the step count back and zeroes *reset when given). Shared
// with the fused small-batch critic update (k_critic_mma.cu), so both round identically.
template <bool POL>
__device__ __forceinline__ void adam_body(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                                          float* __restrict__ v, size_t n, long long* counter, float lr, float b1,
                                          float b2, float eps, size_t clo, size_t chi, float cmin,
                                          unsigned int* ticket, const Bf16Views& views, float* amp,
                                          float amp_growth, float amp_backoff, int amp_interval, double lnb1,
                                          double lnb2, float* __restrict__ tp, float tau, const Bf16Views& tviews,
                                          unsigned int cta, unsigned int ncta, unsigned int* reset) {
  // bias corrections once per block, not once per thread
  __shared__ float s_coef[3];
  __shared__ long long s_t;
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    const long long tt = *(volatile long long*)counter + 1;
    s_t = tt;
    adam_coefs(lr, lnb1, lnb2, tt, &s_coef[0], &s_coef[1]);
    // loss scaling: skip the step on a non-finite gradient, else unscale by 1 / scale
    s_skip = amp ? (*(volatile float*)(amp + 2) != 0.0f) : 0;
    s_coef[2] = amp ? __frcp_rn(*(volatile float*)amp) : 1.0f;
  }
  __syncthreads();
  const long long t = s_t;
  const float step_size = s_coef[0];
  const float bc2_sqrt = s_coef[1];
  const float inv_scale = s_coef[2];
  const bool skip = s_skip != 0;
  const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
  const float omt = 1.0f - tau;
  const size_t n4 = n / 4;
  const size_t stride = (size_t)ncta * blockDim.x;
  // two float4 groups per thread and iteration, every load issued before any arithmetic (more
  // bytes in flight per thread: 128 B)
  for (size_t i0 = cta * (size_t)blockDim.x + threadIdx.x; i0 < n4 && !skip; i0 += 2 * stride) {
    float4 pp[2], gg[2], mm[2], vv[2], tt[2];
    const bool two = i0 + stride < n4;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const size_t i = i0 + u * stride;
      if (u == 0 || two) {
        pp[u] = reinterpret_cast<float4*>(p)[i];
        gg[u] = reinterpret_cast<const float4*>(g)[i];
        mm[u] = reinterpret_cast<float4*>(m)[i];
        vv[u] = reinterpret_cast<float4*>(v)[i];
        if constexpr (POL) tt[u] = reinterpret_cast<float4*>(tp)[i];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u == 1 && !two) break;
      const size_t i = i0 + u * stride;
      float* pa = &pp[u].x; float* ga = &gg[u].x; float* ma = &mm[u].x; float* va = &vv[u].x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (amp) ga[j] = __fmul_rn(ga[j], inv_scale);
        pa[j] = adam_elem(pa[j], ga[j], ma[j], va[j], b1, omb1, b2, omb2, bc2_sqrt, eps, step_size);
        const size_t e = 4 * i + j;
        if (e >= clo && e < chi) pa[j] = fmaxf(pa[j], cmin);
        store_views(views, e, pa[j]);
        if constexpr (POL) {
          float* ta = &tt[u].x;
          ta[j] = __fadd_rn(__fmul_rn(tau, pa[j]), __fmul_rn(omt, ta[j]));
          store_views(tviews, e, ta[j]);
        }
      }
      reinterpret_cast<float4*>(p)[i] = pp[u];
      reinterpret_cast<float4*>(m)[i] = mm[u];
      reinterpret_cast<float4*>(v)[i] = vv[u];
      if constexpr (POL) reinterpret_cast<float4*>(tp)[i] = tt[u];
    }
  }
  for (size_t e = 4 * n4 + cta * (size_t)blockDim.x + threadIdx.x; e < n && !skip; e += stride) {
    const float ge = amp ? __fmul_rn(g[e], inv_scale) : g[e];
    float mm = m[e], vv = v[e];
    float pp = adam_elem(p[e], ge, mm, vv, b1, omb1, b2, omb2, bc2_sqrt, eps, step_size);
    if (e >= clo && e < chi) pp = fmaxf(pp, cmin);
    p[e] = pp; m[e] = mm; v[e] = vv;
    store_views(views, e, pp);
    if constexpr (POL) {
      const float x = __fadd_rn(__fmul_rn(tau, pp), __fmul_rn(omt, tp[e]));
      tp[e] = x;
      store_views(tviews, e, x);
    }
  }
  // publish the new step count once every block has read the old one
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(ticket, 1u);
    if (done == ncta - 1) {
      if (!skip) *counter = t;   // a skipped step does not count (PyTorch GradScaler semantics)
      if (amp) {                 // scale update: back off on overflow, grow after amp_interval finite steps
        if (skip) {
          amp[0] = __fmul_rn(amp[0], amp_backoff);
          amp[1] = 0.0f;
        } else {
          amp[1] = __fadd_rn(amp[1], 1.0f);
          if (amp[1] >= (float)amp_interval) { amp[0] = __fmul_rn(amp[0], amp_growth); amp[1] = 0.0f; }
        }
        amp[2] = 0.0f;
      }
      *ticket = 0u;
      if (reset) *reset = 0u;
      __threadfence();
    }
  }
}

}  // namespace spk
