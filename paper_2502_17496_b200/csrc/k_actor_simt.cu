// k_actor_simt.cu — SIMT (FFMA) kernels of the spiking actor: the fp32 path of configs[0], the
// reference engine the tcgen05 path is cross-checked against, and the elementwise decoder /
// output-scan kernels every engine uses.
//   Forward LIF: north_star c = d_c*c + W*o, v = d_v*v*(1-o_prev) + c, o = [v > V_th]
//   (SPEC.md:141-149). Decoder: PAPER.md:131 / SPEC.md:150-158.
//   Backward: SPEC.md:168-176, R10/R11 (rectangular surrogate, detached reset).
// Layouts: spike and mask planes u32 [T][B][P/32]; gradients G_l
// [T][B][P_l] in fp32 (FP32 precision) or bf16 (BF16 precision, R20 rounding point).
// All reductions run in a fixed order: results are run-to-run bitwise deterministic.
#include "internal.h"

namespace spk {

template <typename WT> __device__ __forceinline__ float ldw(const WT* p);
template <> __device__ __forceinline__ float ldw<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ldw<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// ------------------------------------------------------------------------------ forward layer
template <typename WT>
__global__ void __launch_bounds__(128) lif_fwd_simt_kernel(
    int B, int T, int N, int Win, int Wout, const uint32_t* __restrict__ bits_in,
    const WT* __restrict__ W, int ldw_, LifConst kc, uint32_t* __restrict__ bits_out,
    uint32_t* __restrict__ mask_out, uint8_t* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint32_t s_words[];
  const int b = blockIdx.x;
  const int n = blockIdx.y * 128 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  float c = 0.f, v = 0.f;
  bool o = false;
  int cnt = 0;
  const WT* wrow = W + (size_t)(n < N ? n : 0) * ldw_;
  for (int t = 0; t < T; ++t) {
    const uint32_t* src = bits_in + ((size_t)t * B + b) * Win;
    for (int w = threadIdx.x; w < Win; w += 128) s_words[w] = src[w];
    __syncthreads();
    float I = 0.f;
    if (n < N) {
      for (int w = 0; w < Win; ++w) {
        uint32_t word = s_words[w];
        while (word) {
          const int j = __ffs(word) - 1;
          word &= word - 1;
          I = __fadd_rn(I, ldw<WT>(wrow + 32 * w + j));
        }
      }
    }
    bool h = false;
    if (n < N) {
      lif_step(kc, I, c, v, o, h);
    }
    const uint32_t ob = __ballot_sync(0xffffffffu, o);
    const uint32_t hb = __ballot_sync(0xffffffffu, h);
    if (lane == 0) {
      const size_t wi = ((size_t)t * B + b) * Wout + (n >> 5);
      bits_out[wi] = ob;
      mask_out[wi] = hb;
    }
    cnt += o ? 1 : 0;
    __syncthreads();
  }
  if (counts && n < N) counts[(size_t)b * N + n] = (uint8_t)cnt;
}

int launch_lif_fwd_simt(const ActorDims& d, int l, int B, const uint32_t* bits_in,
                        const float* Wf32, const __nv_bfloat16* Wb16, uint32_t* bits_out,
                        uint32_t* mask_out, uint8_t* counts, cudaStream_t st) {
  ProfScope ps_(l == 1 ? "lif_fwd_simt_L1" : (l == 2 ? "lif_fwd_simt_L2" : "lif_fwd_simt_L3"), PB_ALU,
                2.0 * d.T * B * (double)d.N[l] * d.N[l - 1], 0.0, st);
  LifConst kc{d.dc, d.dv, d.vth, d.win};
  dim3 grid(B, d.P[l] / 128);
  const int Win = d.Wd[l - 1], Wout = d.Wd[l];
  const size_t smem = sizeof(uint32_t) * Win;
  if (d.bf16) {
    pdl((lif_fwd_simt_kernel<__nv_bfloat16>), grid, 128, smem, st)(
        B, d.T, d.N[l], Win, Wout, bits_in, Wb16, d.P[l - 1], kc, bits_out, mask_out, counts);
  } else {
    pdl((lif_fwd_simt_kernel<float>), grid, 128, smem, st)(B, d.T, d.N[l], Win, Wout, bits_in, Wf32,
                                                       d.N[l - 1], kc, bits_out, mask_out, counts);
  }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ------------------------------------------------------------------------------ decoder forward
__global__ void dec_fwd_kernel(int B, int A, int D, int T, const uint8_t* __restrict__ counts,
                               const float* __restrict__ Wd, const float* __restrict__ bd,
                               float* __restrict__ act_out, float* __restrict__ act_tape) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * A) return;
  const int b = i / A, j = i % A;
  const int N3 = A * D;
  const float invT = 1.0f / (float)T;
  float pre = 0.f;
  for (int e = 0; e < D; ++e) {
    const float fr = (float)counts[(size_t)b * N3 + j * D + e] / (float)T;
    pre = __fadd_rn(pre, __fmul_rn(Wd[j * D + e], fr));
  }
  (void)invT;
  pre = __fadd_rn(pre, bd[j]);
  const float a = tanhf(pre);
  act_out[i] = a;
  if (act_tape) act_tape[i] = a;
}

int launch_dec_fwd(const ActorDims& d, int B, const uint8_t* counts, const float* Wd,
                   const float* bd, float* act_out, float* act_tape, cudaStream_t st) {
  ProfScope ps_("dec_fwd", PB_LATENCY, 0.0, (double)B * (d.N3 + 8.0 * d.A), st);
  const int n = B * d.A;
  pdl(dec_fwd_kernel, cdiv(n, 256), 256, 0, st)(B, d.A, d.D, d.T, counts, Wd, bd, act_out, act_tape);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ------------------------------------------------------- decoder backward + output reverse scan
// 32x32 bit-matrix transpose across a warp: lane i holds row i on entry, column i on exit
// (five butterfly stages, each swapping the off-diagonal s x s blocks).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t lo[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0, s = 16; k < 5; ++k, s >>= 1) {
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~lo[k]) | ((y & ~lo[k]) >> s)) : ((x & lo[k]) | ((y & lo[k]) << s));
  }
  return x;
}

// One warp per (b, 32 output neurons), grid-strided over b. For T <= 32 lane t loads the spike
// and mask words of step t and a warp bit transpose hands each neuron its bits over t, so the
// reverse scan waits on no load (ncu r01: per-neuron redundant word loads and 64-bit index math
// made this kernel ~50 instructions per element).
template <typename GTy>
__global__ void __launch_bounds__(128) dec_bwd_outscan_kernel(
    int B, int T, int A, int D, int P3, int W3, float dcc, float dvc, float zh,
    const float* __restrict__ grad_a, const float* __restrict__ act, const float* __restrict__ Wd,
    const uint32_t* __restrict__ bits3, const uint32_t* __restrict__ mask3, GTy* __restrict__ G3,
    float* __restrict__ g_pre_out) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.y * 128 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int N3 = A * D;
  const bool nv = n < N3;
  const int j = nv ? n / D : 0, e = nv ? n % D : 0;
  const float wd = nv ? Wd[j * D + e] : 0.f;
  const size_t ts = (size_t)B * W3;   // bit-plane stride between timesteps
  const size_t gts = (size_t)B * P3;  // G3 stride between timesteps
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    float g = 0.f;
    if (nv) {
      const float a = act[(size_t)b * A + j];
      const float gp = __fmul_rn(grad_a[(size_t)b * A + j], __fsub_rn(1.0f, __fmul_rn(a, a)));
      if (e == 0) g_pre_out[(size_t)b * A + j] = gp;
      g = __fdiv_rn(__fmul_rn(gp, wd), (float)T);  // g_o3 = g_fr / T, constant in t
    }
    float dvn = 0.f, dcn = 0.f;
    GTy* gt = G3 + (size_t)b * P3 + n;
    const uint32_t* po = bits3 + (size_t)b * W3 + (n >> 5);
    const uint32_t* ph = mask3 + (size_t)b * W3 + (n >> 5);
    if (T <= 32) {
      uint32_t wo = 0u, wh = 0u;
      if (lane < T) { wo = __ldg(po + lane * ts); wh = __ldg(ph + lane * ts); }
      const uint32_t om = warp_transpose32(wo, lane), hm = warp_transpose32(wh, lane);
      gt += (size_t)(T - 1) * gts;
      for (int t = T - 1; t >= 0; --t, gt -= gts) {
        const float Gt = lif_back_step(zh, dvc, dcc, g, (om >> t) & 1u, (hm >> t) & 1u, dvn, dcn);
        GT<GTy>::store(gt, nv ? Gt : 0.f);
      }
      continue;
    }
    for (int t = T - 1; t >= 0; --t) {
      float Gt = 0.f;
      if (nv) {
        const uint32_t ow = __ldg(po + t * ts), hw = __ldg(ph + t * ts);
        Gt = lif_back_step(zh, dvc, dcc, g, (ow >> lane) & 1u, (hw >> lane) & 1u, dvn, dcn);
      }
      GT<GTy>::store(gt + (size_t)t * gts, Gt);
    }
  }
}

int launch_dec_bwd_outscan(const ActorDims& d, int B, const float* grad_a, const float* act,
                           const uint8_t* counts, const float* Wd, const uint32_t* bits3,
                           const uint32_t* mask3, void* G3, float* g_pre, cudaStream_t st) {
  ProfScope ps_("dec_bwd_outscan", PB_HBM, 0.0, (double)d.T * B * (d.P[3] * (d.bf16 ? 2.0 : 4.0) + 2.0 * d.Wd[3] * 4), st);
  (void)counts;
  // grid-strided over b: one 128-thread block per (b, 128 neurons) was block-scheduling bound
  const int gy = d.P[3] / 128;
  int gx = (num_sms() * 16 + gy - 1) / gy;
  if (gx > B) gx = B;
  dim3 grid(gx, gy);
  if (d.bf16)
    pdl((dec_bwd_outscan_kernel<__nv_bfloat16>), grid, 128, 0, st)(
        B, d.T, d.A, d.D, d.P[3], d.Wd[3], d.dc, d.dv, d.zh, grad_a, act, Wd, bits3, mask3,
        (__nv_bfloat16*)G3, g_pre);
  else
    pdl((dec_bwd_outscan_kernel<float>), grid, 128, 0, st)(B, d.T, d.A, d.D, d.P[3], d.Wd[3], d.dc,
                                                        d.dv, d.zh, grad_a, act, Wd, bits3, mask3,
                                                        (float*)G3, g_pre);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// dbd[j] = sum_b g_pre[b][j];  dWd[j][e] = sum_b g_pre[b][j] * cnt[b][jD+e] / T.
// One block per (j, e) (e == D row computes dbd); fixed-order block tree reduction.
__global__ void __launch_bounds__(256) dec_param_grads_kernel(int B, int A, int D, int T,
                                                              const float* __restrict__ g_pre,
                                                              const uint8_t* __restrict__ counts,
                                                              float* __restrict__ dWd,
                                                              float* __restrict__ dbd, int accum) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x, e = blockIdx.y;  // e == D -> bias
  const int N3 = A * D;
  float s = 0.f;
  for (int b = threadIdx.x; b < B; b += 256) {
    const float gp = g_pre[(size_t)b * A + j];
    if (e == D) s = __fadd_rn(s, gp);
    else s = __fadd_rn(s, __fmul_rn(gp, (float)counts[(size_t)b * N3 + j * D + e] / (float)T));
  }
  __shared__ float red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = __fadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    float* dst = (e == D) ? (dbd + j) : (dWd + j * D + e);
    *dst = accum ? __fadd_rn(*dst, red[0]) : red[0];
  }
}

int launch_dec_param_grads(const ActorDims& d, int B, const float* g_pre, const uint8_t* counts,
                           float* dWd, float* dbd, int accumulate, cudaStream_t st) {
  ProfScope ps_("dec_param_grads", PB_LATENCY, 0.0, (double)B * (4.0 * d.A + d.N3), st);
  dim3 grid(d.A, d.D + 1);
  pdl(dec_param_grads_kernel, grid, 256, 0, st)(B, d.A, d.D, d.T, g_pre, counts, dWd, dbd, accumulate);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ------------------------------------------------- dX of layer l fused with reverse scan of l-1
// g_o^{l-1}[t][b][k] = sum_n G_l[t][b][n] W_l[n][k]; then the reverse scan of layer l-1 with its
// spike / mask bits gives G_{l-1}; for l == 2 also Gsum1[b][k] = sum_t G_1 (fp32, then rounded).
template <typename GTy, typename WT>
__global__ void __launch_bounds__(128) lif_dx_simt_kernel(
    int B, int T, int Nl, int Pl, int Nprev, int Pprev, int Wprev, float dcc, float dvc, float zh,
    const GTy* __restrict__ Gl, const WT* __restrict__ W, int ldw_, const uint32_t* __restrict__ bits,
    const uint32_t* __restrict__ mask, GTy* __restrict__ Gprev, GTy* __restrict__ Gsum) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_g[];
  const int b = blockIdx.x;
  const int k = blockIdx.y * 128 + threadIdx.x;
  float dvn = 0.f, dcn = 0.f, gs = 0.f;
  for (int t = T - 1; t >= 0; --t) {
    const size_t row = (size_t)t * B + b;
    for (int n = threadIdx.x; n < Nl; n += 128) s_g[n] = GT<GTy>::load(Gl + row * Pl + n);
    __syncthreads();
    float Gt = 0.f;
    if (k < Nprev) {
      float g = 0.f;
      for (int n = 0; n < Nl; ++n) g = __fmaf_rn(s_g[n], ldw<WT>(W + (size_t)n * ldw_ + k), g);
      const uint32_t ow = bits[row * Wprev + (k >> 5)], hw = mask[row * Wprev + (k >> 5)];
      Gt = lif_back_step(zh, dvc, dcc, g, (ow >> (k & 31)) & 1u, (hw >> (k & 31)) & 1u, dvn, dcn);
      gs = __fadd_rn(gs, Gt);
    }
    GT<GTy>::store(Gprev + row * Pprev + k, Gt);
    __syncthreads();
  }
  if (Gsum) GT<GTy>::store(Gsum + (size_t)b * Pprev + k, gs);
}

int launch_lif_dx_simt(const ActorDims& d, int l, int B, const void* Gl, const float* Wf32,
                       const __nv_bfloat16* Wb16, const uint32_t* bits_prev,
                       const uint32_t* mask_prev, void* Gprev, void* Gsum, cudaStream_t st) {
  ProfScope ps_(l == 3 ? "lif_dx_simt_L3" : "lif_dx_simt_L2", PB_ALU, 2.0 * d.T * B * (double)d.N[l] * d.N[l - 1], 0.0, st);
  dim3 grid(B, d.P[l - 1] / 128);
  const size_t smem = sizeof(float) * d.N[l];
  if (d.bf16)
    pdl((lif_dx_simt_kernel<__nv_bfloat16, __nv_bfloat16>), grid, 128, smem, st)(
        B, d.T, d.N[l], d.P[l], d.N[l - 1], d.P[l - 1], d.Wd[l - 1], d.dc, d.dv, d.zh,
        (const __nv_bfloat16*)Gl, Wb16, d.P[l - 1], bits_prev, mask_prev, (__nv_bfloat16*)Gprev,
        (__nv_bfloat16*)Gsum);
  else
    pdl((lif_dx_simt_kernel<float, float>), grid, 128, smem, st)(
        B, d.T, d.N[l], d.P[l], d.N[l - 1], d.P[l - 1], d.Wd[l - 1], d.dc, d.dv, d.zh,
        (const float*)Gl, Wf32, d.N[l - 1], bits_prev, mask_prev, (float*)Gprev, (float*)Gsum);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// -------------------------------------------------------------------------- dW (SIMT reference)
// dW_l[n][k] = sum_{t,b} G_l[t][b][n] * o_{l-1}[t][b][k]; one thread per (n, k), rows staged in
// shared memory in chunks of 256 (t,b) rows.
template <typename GTy>
__global__ void __launch_bounds__(128) lif_dw_simt_kernel(int R, int Nl, int Pl, int K, int Wprev,
                                                          const GTy* __restrict__ Gl,
                                                          const uint32_t* __restrict__ bits,
                                                          float* __restrict__ dW, int accum) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_g[256];
  const int n = blockIdx.y;
  const int k = blockIdx.x * 128 + threadIdx.x;
  float acc = 0.f;
  for (int r0 = 0; r0 < R; r0 += 256) {
    const int rn = min(256, R - r0);
    for (int i = threadIdx.x; i < rn; i += 128) s_g[i] = GT<GTy>::load(Gl + (size_t)(r0 + i) * Pl + n);
    __syncthreads();
    if (k < K) {
      const uint32_t* bp = bits + (size_t)r0 * Wprev + (k >> 5);
      const int sh = k & 31;
      for (int i = 0; i < rn; ++i) {
        if ((bp[(size_t)i * Wprev] >> sh) & 1u) acc = __fadd_rn(acc, s_g[i]);
      }
    }
    __syncthreads();
  }
  if (k < K) {
    float* dst = dW + (size_t)n * K + k;
    *dst = accum ? __fadd_rn(*dst, acc) : acc;
  }
}

int launch_lif_dw_simt(const ActorDims& d, int l, int B, const void* Gl, const uint32_t* bits_prev,
                       float* dW, int accumulate, cudaStream_t st) {
  ProfScope ps_(l == 1 ? "lif_dw_simt_L1" : (l == 2 ? "lif_dw_simt_L2" : "lif_dw_simt_L3"), PB_ALU,
                2.0 * d.T * B * (double)d.N[l] * d.N[l - 1], 0.0, st);
  const int K = d.N[l - 1];
  dim3 grid(cdiv(K, 128), d.N[l]);
  const int R = d.T * B;
  if (d.bf16)
    pdl((lif_dw_simt_kernel<__nv_bfloat16>), grid, 128, 0, st)(
        R, d.N[l], d.P[l], K, d.Wd[l - 1], (const __nv_bfloat16*)Gl, bits_prev, dW, accumulate);
  else
    pdl((lif_dw_simt_kernel<float>), grid, 128, 0, st)(R, d.N[l], d.P[l], K, d.Wd[l - 1],
                                                    (const float*)Gl, bits_prev, dW, accumulate);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ------------------------------------------------------------------------ encoder gradient
// dL/dA[b][k] = sum_n Gsum1[b][n] W1[n][k] (straight-through encoder: do_t/dA = 1, R6);
// dmu[k] = sum_b dL/dA * A * (s - mu)/sigma^2 ; dsigma[k] = sum_b dL/dA * A * (s - mu)^2/sigma^3.
constexpr int kEncChunk = 64;

size_t enc_grad_partial_bytes(const ActorDims& d, int B) {
  return sizeof(float) * 2 * (size_t)cdiv(B, kEncChunk) * d.K0;
}

template <typename GTy, typename WT>
__global__ void __launch_bounds__(128) enc_grad_partial_kernel(
    int B, int S, int E, int K0, int N1, int P1, const GTy* __restrict__ Gsum,
    const WT* __restrict__ W1, int ldw_, const float* __restrict__ A,
    const float* __restrict__ obs, const float* __restrict__ mu, const float* __restrict__ sigma,
    float* __restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float s_g[];
  const int k = blockIdx.x * 128 + threadIdx.x;
  const int chunk = blockIdx.y;
  const int b0 = chunk * kEncChunk, b1 = min(B, b0 + kEncChunk);
  float pm = 0.f, ps = 0.f;
  const float m = k < K0 ? mu[k] : 0.f, sg = k < K0 ? sigma[k] : 1.f;
  const float sg2 = __fmul_rn(sg, sg), sg3 = __fmul_rn(sg2, sg);
  for (int b = b0; b < b1; ++b) {
    for (int n = threadIdx.x; n < N1; n += 128) s_g[n] = GT<GTy>::load(Gsum + (size_t)b * P1 + n);
    __syncthreads();
    if (k < K0) {
      float gA = 0.f;
      for (int n = 0; n < N1; ++n) gA = __fmaf_rn(s_g[n], ldw<WT>(W1 + (size_t)n * ldw_ + k), gA);
      const float a = A[(size_t)b * K0 + k];
      const float dd = __fsub_rn(obs[(size_t)b * S + k / E], m);
      const float ga = __fmul_rn(gA, a);
      pm = __fadd_rn(pm, __fdiv_rn(__fmul_rn(ga, dd), sg2));
      ps = __fadd_rn(ps, __fdiv_rn(__fmul_rn(ga, __fmul_rn(dd, dd)), sg3));
    }
    __syncthreads();
  }
  if (k < K0) {
    partial[((size_t)chunk * K0 + k) * 2 + 0] = pm;
    partial[((size_t)chunk * K0 + k) * 2 + 1] = ps;
  }
}

__global__ void enc_grad_reduce_kernel(int nchunk, int K0, const float* __restrict__ partial,
                                       float* __restrict__ dmu, float* __restrict__ dsg, int accum) {
  pdl_wait();
  pdl_trigger();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K0) return;
  float a = 0.f, s = 0.f;
  for (int c = 0; c < nchunk; ++c) {
    a = __fadd_rn(a, partial[((size_t)c * K0 + k) * 2 + 0]);
    s = __fadd_rn(s, partial[((size_t)c * K0 + k) * 2 + 1]);
  }
  dmu[k] = accum ? __fadd_rn(dmu[k], a) : a;
  dsg[k] = accum ? __fadd_rn(dsg[k], s) : s;
}

int launch_enc_grad_reduce(const ActorDims& d, int nchunk, const float* partial, float* dmu,
                           float* dsigma, int accumulate, cudaStream_t st) {
  pdl(enc_grad_reduce_kernel, cdiv(d.K0, 256), 256, 0, st)(nchunk, d.K0, partial, dmu, dsigma, accumulate);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

int launch_enc_grad_simt(const ActorDims& d, int B, const void* Gsum, const float* W1f32,
                         const __nv_bfloat16* W1b16, const float* A, const float* obs,
                         const float* mu, const float* sigma, float* partial, float* dmu,
                         float* dsigma, int accumulate, cudaStream_t st) {
  ProfScope ps_("enc_grad_simt", PB_ALU, 2.0 * B * (double)d.N1 * d.K0, 0.0, st);
  const int nchunk = cdiv(B, kEncChunk);
  dim3 grid(cdiv(d.K0, 128), nchunk);
  const size_t smem = sizeof(float) * d.N1;
  if (d.bf16)
    pdl((enc_grad_partial_kernel<__nv_bfloat16, __nv_bfloat16>), grid, 128, smem, st)(
        B, d.S, d.E, d.K0, d.N1, d.P[1], (const __nv_bfloat16*)Gsum, W1b16, d.P[0], A, obs, mu,
        sigma, partial);
  else
    pdl((enc_grad_partial_kernel<float, float>), grid, 128, smem, st)(
        B, d.S, d.E, d.K0, d.N1, d.P[1], (const float*)Gsum, W1f32, d.K0, A, obs, mu, sigma,
        partial);
  SPK_LAUNCHED();
  pdl(enc_grad_reduce_kernel, cdiv(d.K0, 256), 256, 0, st)(nchunk, d.K0, partial, dmu, dsigma,
                                                          accumulate);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

}  // namespace spk
