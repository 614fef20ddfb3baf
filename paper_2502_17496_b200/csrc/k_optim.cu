// k_optim.cu — K10 Adam (PyTorch form, R19) with the actor sigma floor
// (R12), K11 Polyak soft update, and the bf16 working-copy
// refresh (master fp32 -> RNE bf16; "master copy of weights in full precision").
// HBM-bound, vectorised elementwise kernels, grid sized in multiples of the 148 SMs.
#include "adam_body.cuh"

namespace spk {

constexpr int kSMs = 148;

static int ew_grid(size_t n, int per_thread) {
  const size_t threads = (n + per_thread - 1) / per_thread;
  const size_t blocks = (threads + 255) / 256;
  const size_t cap = (size_t)kSMs * 8;
  return (int)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

// Streaming kernels (Adam, Polyak): exactly one wave of resident blocks, never more. A grid of
// 8 blocks per SM with 3 resident ran 2.67 waves (ncu r01: Adam at configs[4] size 66% of the
// copy peak, the partial last wave and the ramp of each wave exposed).
template <int KEY, typename K>   // KEY: one occupancy cache per kernel (instantiations share K's type)
static int stream_grid(K kernel, size_t n, int per_thread) {
  static int cache[32] = {};   // per device
  int& per_sm = cache[cur_device()];
  if (!per_sm) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, 256, 0) != cudaSuccess || v < 1) {
      cudaGetLastError();
      v = 2;
    }
    per_sm = v;
  }
  const size_t threads = (n + per_thread - 1) / per_thread;
  const size_t blocks = (threads + 255) / 256;
  const size_t cap = (size_t)num_sms() * per_sm;
  return (int)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

// ------------------------------------------------------------------ bf16 working copies
// Actor: W_l (fp32 [N_l][N_{l-1}]) -> bf16 [P_l][P_{l-1}], zero padded. One thread per padded
// element so the padding is (re)written with zeros every refresh.
__global__ void actor_refresh_kernel(const float* __restrict__ W, int N, int K, int P, int Pk,
                                     __nv_bfloat16* __restrict__ out, int f16) {
  pdl_wait();
  pdl_trigger();
  const size_t total = (size_t)P * Pk;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / Pk), k = (int)(i % Pk);
    const float v = (n < N && k < K) ? W[(size_t)n * K + k] : 0.0f;
    reinterpret_cast<unsigned short*>(out)[i] = op16_bits(v, f16 != 0);
  }
}

int launch_actor_refresh_bf16(const ActorDims& d, const float* params, __nv_bfloat16* out,
                              cudaStream_t st) {
  ProfScope ps_("refresh_bf16", PB_HBM, 0.0, 6.0 * d.boff[3], st);
  for (int l = 1; l <= 3; ++l) {
    const size_t total = (size_t)d.P[l] * d.P[l - 1];
    pdl(actor_refresh_kernel, ew_grid(total, 4), 256, 0, st)(
        params + d.off[SPIKERL_ACTOR_W1 + l - 1], d.N[l], d.N[l - 1], d.P[l], d.P[l - 1],
        out + d.boff[l - 1], d.f16);
    SPK_LAUNCHED();
  }
  return SPIKERL_OK;
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                   size_t n) {
  pdl_wait();
  pdl_trigger();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

int launch_f32_to_bf16(const float* in, __nv_bfloat16* out, size_t n, cudaStream_t st) {
  ProfScope ps_("f32_to_bf16", PB_HBM, 0.0, 6.0 * n, st);
  pdl(f32_to_bf16_kernel, ew_grid(n, 4), 256, 0, st)(in, out, n);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

Bf16Views actor_bf16_views(const ActorDims& d, __nv_bfloat16* out) {
  Bf16Views v{};
  v.kind = out ? 1 : 0;
  v.f16 = d.f16;
  v.out = out;
  for (int l = 1; l <= 3; ++l) {
    v.src[l - 1] = (long long)d.off[SPIKERL_ACTOR_W1 + l - 1];
    v.dst[l - 1] = (long long)d.boff[l - 1];
    v.rows[l - 1] = d.N[l];
    v.cols[l - 1] = d.N[l - 1];
    v.ldd[l - 1] = d.P[l - 1];
    v.colsd[l - 1] = make_fastdiv((uint32_t)d.N[l - 1]);
  }
  return v;
}

// ------------------------------------------------------------------ Adam
// t = *counter + 1 is read by every block; the last block to finish (atomic ticket) stores it
// back, so the call is graph-replayable with an on-device step count.
// POL: the fused Polyak soft update of a target (PolyakFuse) — its own instantiation, so the plain
// Adam keeps its register budget (92 vs 80 registers: one resident block per SM fewer)
template <bool POL>
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                   float* __restrict__ m, float* __restrict__ v,
                                                   size_t n, long long* counter, float lr, float b1,
                                                   float b2, float eps, size_t clo, size_t chi,
                                                   float cmin, unsigned int* ticket,
                                                   const __grid_constant__ Bf16Views views, float* amp,
                                                   float amp_growth, float amp_backoff, int amp_interval,
                                                   double lnb1, double lnb2, float* __restrict__ tp, float tau,
                                                   const __grid_constant__ Bf16Views tviews) {
  pdl_wait();
  pdl_trigger();
  adam_body<POL>(p, g, m, v, n, counter, lr, b1, b2, eps, clo, chi, cmin, ticket, views, amp, amp_growth, amp_backoff,
                 amp_interval, lnb1, lnb2, tp, tau, tviews, blockIdx.x, gridDim.x, nullptr);
}

// found_inf of dynamic loss scaling: any non-finite gradient element sets amp[2]
__global__ void amp_check_kernel(const float* __restrict__ g, size_t n, float* __restrict__ amp) {
  pdl_wait();
  pdl_trigger();
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) amp[2] = 1.0f;
}

int launch_amp_check(const float* g, size_t n, float* amp, cudaStream_t st) {
  ProfScope ps_("amp_check", PB_HBM, 0.0, 4.0 * n, st);
  pdl(amp_check_kernel, ew_grid(n, 4), 256, 0, st)(g, n, amp);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

int launch_adam(float* p, const float* g, float* m, float* v, size_t n, long long* counter,
                float lr, float b1, float b2, float eps, size_t clo, size_t chi, float cmin,
                unsigned int* ticket, const Bf16Views* views, cudaStream_t st, float* amp, float amp_growth,
                float amp_backoff, int amp_interval, const PolyakFuse* polyak) {
  // a skipped (overflowing) loss-scaled step must still move the target: no fusion with the scaler
  if (polyak && amp) { set_error("adam: a fused Polyak update needs amp == NULL"); return SPIKERL_E_ARG; }
  ProfScope ps_(polyak ? "adam_polyak" : "adam", PB_HBM, 0.0, (polyak ? 40.0 : 28.0) * n, st);
  const Bf16Views none{};
  if (((uintptr_t)p | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v | (uintptr_t)(polyak ? polyak->t : nullptr)) & 15) {
    set_error("adam: buffers must be 16-byte aligned");
    return SPIKERL_E_ARG;
  }
  if (polyak)
    pdl(adam_kernel<true>, stream_grid<1>(adam_kernel<true>, n, 8), 256, 0, st)(
        p, g, m, v, n, counter, lr, b1, b2, eps, clo, chi, cmin, ticket, views ? *views : none, amp, amp_growth,
        amp_backoff, amp_interval, log((double)b1), log((double)b2), polyak->t, polyak->tau,
        polyak->views ? *polyak->views : none);
  else
    pdl(adam_kernel<false>, stream_grid<0>(adam_kernel<false>, n, 8), 256, 0, st)(
        p, g, m, v, n, counter, lr, b1, b2, eps, clo, chi, cmin, ticket, views ? *views : none, amp, amp_growth,
        amp_backoff, amp_interval, log((double)b1), log((double)b2), nullptr, 0.f, none);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ------------------------------------------------------------------ Polyak
__global__ void __launch_bounds__(256, 4) polyak_kernel(float* __restrict__ t, const float* __restrict__ s,
                                                      size_t n, float tau, const __grid_constant__ Bf16Views views) {
  pdl_wait();
  pdl_trigger();
  const float omt = 1.0f - tau;
  const size_t n4 = (((uintptr_t)t | (uintptr_t)s) & 15) ? 0 : n / 4;   // float4 body when aligned
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // two float4 groups per thread and iteration, all four loads issued before the arithmetic
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i0 < n4; i0 += 2 * stride) {
    const bool two = i0 + stride < n4;
    float4 sv[2], tv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (u == 0 || two) {
        sv[u] = reinterpret_cast<const float4*>(s)[i0 + u * stride];
        tv[u] = reinterpret_cast<float4*>(t)[i0 + u * stride];
      }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u == 1 && !two) break;
      const size_t i = i0 + u * stride;
      float* ta = &tv[u].x;
      const float* sa = &sv[u].x;
#pragma unroll
      for (int j = 0; j < 4; ++j) ta[j] = __fadd_rn(__fmul_rn(tau, sa[j]), __fmul_rn(omt, ta[j]));
      reinterpret_cast<float4*>(t)[i] = tv[u];
#pragma unroll
      for (int j = 0; j < 4; ++j) store_views(views, 4 * i + j, ta[j]);
    }
  }
  for (size_t i = 4 * n4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float x = __fadd_rn(__fmul_rn(tau, s[i]), __fmul_rn(omt, t[i]));
    t[i] = x;
    store_views(views, i, x);
  }
}

int launch_polyak(float* t, const float* s, size_t n, float tau, const Bf16Views* views, cudaStream_t st) {
  const Bf16Views none{};
  ProfScope ps_("polyak", PB_HBM, 0.0, 12.0 * n, st);
  pdl(polyak_kernel, stream_grid<2>(polyak_kernel, n, 8), 256, 0, st)(t, s, n, tau, views ? *views : none);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

}  // namespace spk
