// internal.h — launchers shared between the ABI layer and the kernel files.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace spk {

// ---- encoder (k_encoder.cu)
int launch_enc_fwd(const ActorDims& d, int B, const float* obs, const float* mu, const float* sigma,
                   float* A, uint32_t* bits0, cudaStream_t st);

// ---- SIMT actor kernels (k_actor_simt.cu)
// forward layer l (1..3): bits_in [T][B][W_{l-1}] -> bits_out, mask_out [T][B][W_l] (+counts)
int launch_lif_fwd_simt(const ActorDims& d, int l, int B, const uint32_t* bits_in,
                        const float* Wf32, const __nv_bfloat16* Wb16, uint32_t* bits_out,
                        uint32_t* mask_out, uint8_t* counts, float* v_out, cudaStream_t st);
// TD3 target-policy smoothing fused into the target actor's decoder launch (at != NULL):
// at = clip(a + clip(eps, -c, c), -1, 1) with eps from the update's snapshotted Philox counter (or
// the injected noise); advance: this launch moves *counter past the snapshot
struct TargetSmooth {
  const float* noise;
  float sigma, clip;
  unsigned long long seed;
  int rank;
  unsigned long long* counter;
  const unsigned long long* ctr_snap;
  float* at;
  int advance;
};
int launch_dec_fwd(const ActorDims& d, int B, const uint8_t* counts, const float* Wd,
                   const float* bd, float* act_out, float* act_tape, cudaStream_t st,
                   const TargetSmooth* smooth = nullptr);
// decoder backward + output-layer reverse scan -> G3 [T][B][P3] (fp32 or bf16 per precision)
int launch_dec_bwd_outscan(const ActorDims& d, int B, const float* grad_a, const float* act,
                           const uint8_t* counts, const float* Wd, const uint32_t* bits3,
                           const uint32_t* mask3, const float* v3, void* G3, float* g_pre, cudaStream_t st);
int dec_param_chunks(int B);   // row chunks of the decoder parameter gradient (partials: chunks x (N3 + A))
int launch_dec_param_grads(const ActorDims& d, int B, const float* g_pre, const uint8_t* counts,
                           float* dWd, float* dbd, float* part, int accumulate, cudaStream_t st);
// dX of layer l (3 or 2) fused with the reverse scan of layer l-1 -> G_{l-1} (+Gsum if l==2)
int launch_lif_dx_simt(const ActorDims& d, int l, int B, const void* Gl, const float* Wf32,
                       const __nv_bfloat16* Wb16, const uint32_t* bits_prev,
                       const uint32_t* mask_prev, const float* v_prev, void* Gprev, void* Gsum,
                       cudaStream_t st);
// dW_l = sum_{t,b} G_l^T o_{l-1}  (fp32 [N_l][N_{l-1}] in the master layout)
int launch_lif_dw_simt(const ActorDims& d, int l, int B, const void* Gl, const uint32_t* bits_prev,
                       float* dW, int accumulate, cudaStream_t st);
// encoder gradient from Gsum1 [B][P1]: dmu, dsigma (two-pass deterministic)
int launch_enc_grad_simt(const ActorDims& d, int B, const void* Gsum, const float* W1f32,
                         const __nv_bfloat16* W1b16, const float* A, const float* obs,
                         const float* mu, const float* sigma, float* partial, float* dmu,
                         float* dsigma, int accumulate, cudaStream_t st);
size_t enc_grad_partial_bytes(const ActorDims& d, int B);

// ---- tcgen05 engine (k_tc_gemm.cu)
bool tc_supported(const ActorDims& d);
bool tc_pairs_enabled();   // CTA pairs (cta_group::2) in use (SPIKERL_TC_PAIR=0 turns them off)
int launch_lif_fwd_tc(const ActorDims& d, int l, int B, const uint32_t* bits_in,
                      const __nv_bfloat16* Wb16, uint32_t* bits_out, uint32_t* mask_out,
                      uint8_t* counts, uint8_t* bitsT_out, uint8_t* maskT_out, int row_bytes,
                      float* v_out, cudaStream_t st);
int launch_lif_dx_tc(const ActorDims& d, int l, int B, const void* Gl, const __nv_bfloat16* Wb16,
                     const uint8_t* bitsT_prev, const uint8_t* maskT_prev, int row_bytes,
                     const float* v_prev, void* Gprev, void* Gsum, cudaStream_t st);
int launch_enc_grad_tc(const ActorDims& d, int B, const void* Gsum, const __nv_bfloat16* W1b16,
                       const float* A, const float* obs, const float* mu, const float* sigma,
                       float* partial, float* dmu, float* dsigma, int accumulate, cudaStream_t st);
int launch_lif_dw_tc(const ActorDims& d, int l, int B, const void* Gl, const uint32_t* bits_prev,
                     float* dW, float* part, int accumulate, cudaStream_t st);
size_t tc_enc_partial_bytes(const ActorDims& d, int B);
size_t tc_dw_partial_bytes(const ActorDims& d, int B, int l);
// critic weight gradients on the tcgen05 engine (stacked K-major operands; see k_tc_gemm.cu)
int tc_wgrad_splits(int Bp, int inq);
int launch_critic_wgrad_tc(int Bp, int inq, int xtr, const __nv_bfloat16* dZT, const __nv_bfloat16* XTH,
                           float* part, long long msz, cudaStream_t st);
// twin-critic contractions at large batch on the tcgen05 engine: mode 6 = CF1 (X W1^T -> H1T),
// 7 = CF2 (H1 W2^T -> H2T, q), 8 = CB1 (dZ2 W2 -> dZ1T); see k_tc_gemm.cu
int launch_critic_tc(int mode, int B, int Bp, int nz, const __nv_bfloat16* A, int a_rows, int aoff,
                     const __nv_bfloat16* Bw0, const __nv_bfloat16* Bw1, int bk, int ldb, const float* bias,
                     const __nv_bfloat16* w3, const float* b3, long long ps, __nv_bfloat16* out, long long os,
                     const __nv_bfloat16* mask, float* q, cudaStream_t st);
// 3-D u32 tensor map (dims / box innermost first, strides in bytes), no swizzle, OOB zero fill
int make_u32_map3(CUtensorMap* m, const void* base, const uint64_t* dims, const uint64_t* strides,
                  const uint32_t* box);   // split-K partials of dW_l
int launch_enc_grad_reduce(const ActorDims& d, int nchunk, const float* partial, float* dmu,
                           float* dsigma, int accumulate, cudaStream_t st);

// ---- auxiliary streams (prof.cu): per device, created once outside any graph capture (the
// workspace-size queries create them). Kernels forked onto them are joined back before the
// forking call returns, so a graph capture of the call records a DAG with parallel branches.
// Slots: TD3 step side 0-2, 7 / ev 0-7; actor backward side 3-5 / ev 8-15; critic side 6 / ev 16-19;
// bucketed gradient allreduce of the actor backward: side 8 (the comm stream) / ev 20-27.
struct AuxPool {
  cudaStream_t side[10];
  cudaEvent_t ev[32];
};
int aux_pool(AuxPool** out);
int stream_after(cudaStream_t dst, cudaStream_t src, cudaEvent_t ev);   // dst waits for src's work so far

// ---- optimiser / copies (k_optim.cu)
int launch_actor_refresh_bf16(const ActorDims& d, const float* params, __nv_bfloat16* out,
                              cudaStream_t st);
int launch_f32_to_bf16(const float* in, __nv_bfloat16* out, size_t n, cudaStream_t st);
// bf16 working-copy views of an fp32 master vector: Adam / Polyak write the RNE bf16 value of every
// element they update into each place the refresh kernels would put it (the zero padding, written
// once by a full refresh, is never touched), so the TD3 step needs no separate refresh launches.
// Unsigned 32-bit division by a runtime-invariant divisor without a divide instruction sequence:
// q = (umulhi(x, mul) + x) >> shift with mul = floor(2^32 (2^shift - d) / d) + 1, shift =
// ceil(log2 d) (Granlund-Montgomery; exact for every 32-bit x; the add is done in 64 bits).
struct FastDiv {
  uint32_t d, mul, shift;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0u, 0u};
  while ((1ull << f.shift) < d) ++f.shift;
  f.mul = (uint32_t)(((1ull << 32) * ((1ull << f.shift) - d)) / d + 1);
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  return (uint32_t)(((unsigned long long)__umulhi(x, f.mul) + x) >> f.shift);
}

struct Bf16Views {
  int kind;                  // 0 none, 1 actor W1..W3, 2 critic twin (mma layout), 3 plain copy
  int f16;                   // the 16-bit copy holds fp16 (actor FP16 precision), else bf16
  __nv_bfloat16* out;
  long long src[3], dst[3];  // actor: fp32 offset of W_l, bf16 offset of its padded copy
  int rows[3], cols[3], ldd[3];
  FastDiv colsd[3];
  long long P, tb, oW1, oW2, W1p, W1T, W2T, W2c;   // critic (per-critic block after the [2][P] copy)
  int in, H1, H2, inp;
  // critic: the transposed blocks kept current — W1T rows [w1t_lo, w1t_hi) (dQ1/da reads only the
  // action rows [S, S+A)), W2T when w2t (the data backward's operand; forward-only copies such as the
  // TD3 targets need neither)
  int w1t_lo, w1t_hi, w2t;
  FastDiv Pd, ind, H1d;
};
Bf16Views actor_bf16_views(const ActorDims& d, __nv_bfloat16* out);
Bf16Views critic_bf16_views(const CriticDims& c, __nv_bfloat16* out);
// Adam (PyTorch form; R19) for one element, shared by adam_kernel and the fused
// allreduce + Adam kernel so both round identically: m, v fp32; step = lr / (1 - b1^t) and
// bc2_sqrt = sqrt(1 - b2^t) formed once (fp64, rounded to fp32) by adam_coefs, with b^t = exp(t ln b)
// from ln b computed on the host (a device fp64 pow per launch cost ~5 us of latency in r01's Adam).
__device__ __forceinline__ void adam_coefs(float lr, double lnb1, double lnb2, long long t, float* step_size,
                                           float* bc2_sqrt) {
  *step_size = (float)((double)lr / (1.0 - exp((double)t * lnb1)));
  *bc2_sqrt = (float)sqrt(1.0 - exp((double)t * lnb2));
}
__device__ __forceinline__ float adam_elem(float p, float g, float& m, float& v, float b1, float omb1, float b2,
                                           float omb2, float bc2_sqrt, float eps, float step_size) {
  m = __fadd_rn(__fmul_rn(b1, m), __fmul_rn(omb1, g));
  v = __fadd_rn(__fmul_rn(b2, v), __fmul_rn(__fmul_rn(omb2, g), g));
  const float denom = __fadd_rn(__fdiv_rn(sqrtf(v), bc2_sqrt), eps);
  return __fsub_rn(p, __fmul_rn(step_size, __fdiv_rn(m, denom)));
}
// Writes the RNE bf16 copy of the updated master element e into every working copy that holds
// it. Element indices are < 2^31 (parameter counts), so row / column come from 32-bit
// multiply-high divisions (a 64-bit division per element made Adam ~5x slower than its bytes).
__device__ __forceinline__ void store_views(const Bf16Views& v, size_t e, float x) {
  if (v.kind == 0) return;
  const __nv_bfloat16 h = __ushort_as_bfloat16(op16_bits(x, v.f16 != 0));   // fp16 bits when v.f16
  if (v.kind == 1) {
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const long long r = (long long)e - v.src[l];
      if (r >= 0 && r < (long long)v.rows[l] * v.cols[l]) {
        const uint32_t n = fdiv((uint32_t)r, v.colsd[l]), k = (uint32_t)r - n * (uint32_t)v.cols[l];
        v.out[v.dst[l] + (long long)n * v.ldd[l] + k] = h;
      }
    }
    return;
  }
  v.out[e] = h;   // [2][P] plain copy (kinds 2 and 3)
  if (v.kind != 2) return;
  const uint32_t z = fdiv((uint32_t)e, v.Pd);
  const long long l = (long long)e - (long long)z * v.P;
  __nv_bfloat16* blk = v.out + ((2 * v.P + 7) & ~7LL) + z * v.tb;   // blk_base (k_critic_mma.cu)
  long long r = l - v.oW1;
  if (r >= 0 && r < (long long)v.H1 * v.in) {          // W1[j][i] -> W1p[j][i], W1T[i][j]
    const uint32_t j = fdiv((uint32_t)r, v.ind), i = (uint32_t)r - j * (uint32_t)v.in;
    blk[v.W1p + (long long)j * v.inp + i] = h;
    if ((int)i >= v.w1t_lo && (int)i < v.w1t_hi) blk[v.W1T + (long long)i * v.H1 + j] = h;
    return;
  }
  r = l - v.oW2;
  if (r >= 0 && r < (long long)v.H2 * v.H1) {          // W2[j2][j1] -> W2T[j1][j2], W2c[j2][j1]
    const uint32_t j2 = fdiv((uint32_t)r, v.H1d), j1 = (uint32_t)r - j2 * (uint32_t)v.H1;
    if (v.w2t) blk[v.W2T + (long long)j1 * v.H2 + j2] = h;
    blk[v.W2c + r] = h;
  }
}


// Polyak soft update of a target network fused into the Adam launch of its source (TD3's actor step):
// t <- tau p_new + (1 - tau) t right after p_new is formed, the same arithmetic as polyak_kernel
struct PolyakFuse {
  float* t;
  float tau;
  const Bf16Views* views;
};
int launch_adam(float* p, const float* g, float* m, float* v, size_t n, long long* counter,
                float lr, float b1, float b2, float eps, size_t clo, size_t chi, float cmin,
                unsigned int* done_ticket, const Bf16Views* views, cudaStream_t st, float* amp = nullptr,
                float amp_growth = 2.f, float amp_backoff = 0.5f, int amp_interval = 2000,
                const PolyakFuse* polyak = nullptr);
// fused gradient mean + Adam over symmetric memory (k_fused_dp.cu; spikerl_fused_adam_create)
bool fused_adam_matches(const spikerl_fused_adam* fa, const float* g, const float* p, size_t n);
int fused_adam_launch(spikerl_fused_adam* fa, float* m, float* v, long long* counter, float lr, float b1, float b2,
                      float eps, size_t clo, size_t chi, float cmin, unsigned int* ticket, const Bf16Views* views,
                      cudaStream_t st);
// dynamic loss scaling: amp[2] = 1 when g holds a non-finite element (amp: {scale, count, found, -})
int launch_amp_check(const float* g, size_t n, float* amp, cudaStream_t st);
int launch_polyak(float* t, const float* s, size_t n, float tau, const Bf16Views* views, cudaStream_t st);

// ---- critic (k_critic.cu)
// The TD target of a critic update, read where the loss forms dQ: either given (y),
// or formed there from the target critics' Q'(s', a~) [2][B] (qt), r, done and gamma as
// y = r + gamma (1 - d) min(Q1', Q2') with the operations of the former separate td_target launch,
// so the update is bitwise unchanged and one launch shorter.
struct TdY {
  const float* y;
  const float* r;
  const float* d;
  const float* qt;
  float gamma;
  int B;
  float* out;   // optional: the formed y is stored here (by the reads for critic 0)
  __device__ __forceinline__ float at(int b) const {
    if (y) return y[b];
    return __fadd_rn(r[b], __fmul_rn(__fmul_rn(gamma, __fsub_rn(1.0f, d[b])), fminf(qt[b], qt[B + b])));
  }
  __device__ __forceinline__ float get(int b, int z) const {
    const float v = at(b);
    if (out && z == 0) out[b] = v;
    return v;
  }
};
// The target actor's decoder and TD3 target-policy smoothing formed inside the target critics' forward
// launch (the action columns of its input tile), one launch less on the target path: per (row, action)
// dec_fwd_kernel's arithmetic, then smooth_action; the z = 0 CTAs store a' (act_out, act_tape) and a~
// (ts.at) as the decoder launch would, and advance the counter when ts.advance.
struct CriticDecode {
  const uint8_t* counts;   // [B][A D] output-layer spike counts (NULL: no decoding)
  const float* Wd;
  const float* bd;
  int D, T;
  float* act_out;
  float* act_tape;
  TargetSmooth ts;
};
constexpr int kDecMaxD = 16;
bool critic_decode_ok(const CriticDims& c, int B, int A, int D);   // small-batch tensor-core critic, A <= 32, D <= 16
size_t critic_ws_bytes(const CriticDims& c, int B);
size_t critic_bf16_elems(const CriticDims& c);   // twin pair incl. the mma path's padded/transposed copies
int launch_critic_refresh(const CriticDims& c, const float* params2, __nv_bfloat16* out, cudaStream_t st);
bool critic_mma_ok(const CriticDims& c);
void critic_bf16_layout(const CriticDims& c, long long* out8);   // spikerl_critic_bf16_layout
size_t critic_mma_ws_bytes(const CriticDims& c, int B);
int critic_mma_fwd_bwd(const CriticDims& c, int B, const float* params2, const __nv_bfloat16* pb, const float* obs,
                       int S, const float* act, int A, const TdY* y, float* q, float* loss, float* grad2,
                       float* grad_act, float act_scale, int nz, void* ws, cudaStream_t st,
                       cudaEvent_t wait_before_loss = nullptr, const float* dq_scale = nullptr,
                       const CriticDecode* dec = nullptr);
// Fused small-batch critic launches (bf16 tensor-core critic, B <= 512; SPIKERL_CRITIC_FUSED=0 turns
// them off): the whole critic update of a TD3 step (forward, loss, data backward, weight / bias
// gradients, Adam (+ the targets' Polyak step when polyak != NULL) and the bf16 views) as one launch
// with grid barriers, and the actor objective's critic pass (forward of critic 0, dQ1/da, -mean Q) as
// one launch. Bitwise the results of the separate launches. steps: the critic's {t, ticket} slots of
// spikerl_td3_bufs.adam_steps (the grid barrier uses the high word of steps[1]); ticket (actor pass):
// a zero-at-rest counter word.
bool critic_fused_ok(const CriticDims& c, int B);
bool critic_act_fused_ok(const CriticDims& c, int B);
// the critic's Adam (+ the targets' Polyak) with coalesced stores of the transposed bf16 copy; bitwise
// launch_adam's result (no loss scaling)
bool critic_adam_ok(const CriticDims& c, const Bf16Views* views, const PolyakFuse* polyak);
int launch_critic_adam(const CriticDims& c, float* params2, const float* grad2, float* m, float* v, long long* steps,
                       float lr, float b1, float b2, float eps, const Bf16Views* views, const PolyakFuse* polyak,
                       cudaStream_t st);
int critic_update_fused(const CriticDims& c, int B, float* params2, const __nv_bfloat16* pb, const float* obs, int S,
                        const float* act, int A, const TdY& y, float* q, float* loss, float* grad2, void* ws,
                        float* m, float* v, long long* steps, float lr, float b1, float b2, float eps,
                        const Bf16Views* views, const PolyakFuse* polyak, cudaStream_t st);
int critic_actor_fused(const CriticDims& c, int B, const float* params2, const __nv_bfloat16* pb, const float* obs,
                       int S, const float* act, int A, float* q, float* loss, float* grad_act, float act_scale,
                       void* ws, unsigned int* ticket, cudaStream_t st);
// y: the TD target (critic update) or NULL (forward / actor objective). wait_before_loss (optional):
// the stream waits on this event after the forward and before the loss (the target critics' Q' are
// produced concurrently on another stream).
int critic_fwd_bwd(const CriticDims& c, int B, const float* params2, const __nv_bfloat16* pb16,
                   const float* obs, int S, const float* act, int A, const TdY* y, float* q,
                   float* loss, float* grad2, float* grad_act, float act_scale, int n_critics,
                   void* ws, cudaStream_t st, cudaEvent_t wait_before_loss = nullptr,
                   const float* dq_scale = nullptr,   // dq_scale: device loss scale applied to dQ
                   const CriticDecode* dec = nullptr);   // forward only: actions decoded in the launch

// ---- replay / TD3 glue (k_replay.cu)
// minibatch destinations of one gather launch (1 slot, or the 2 updates of a pair); idx[slot] = NULL:
// indices drawn on the device with the counter value *counter + slot (snapshotted into snap[slot])
struct GatherSlots {
  int n;
  float *s[2], *a[2], *r[2], *s2[2], *d[2];
  unsigned long long* snap[2];
  const long long* idx[2];
};
int launch_replay_gather(int B, int S, int A, const float* rs, const float* ra, const float* rr,
                         const float* rs2, const float* rd, long long N, unsigned long long seed, int rank,
                         const unsigned long long* counter, const GatherSlots& gs, cudaStream_t st);
int launch_scale(float* x, size_t n, float s, cudaStream_t st);

}  // namespace spk
