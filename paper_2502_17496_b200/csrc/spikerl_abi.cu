// spikerl_abi.cu — the extern "C" boundary (include/spikerl.h): argument validation (host-side,
// before anything is enqueued), layouts, and the orchestration of the hot path
//   actor forward  = K1 enc_fwd -> K2 lif_fwd x3 -> K3 dec_fwd
//   actor backward = K4 dec_bwd_outscan -> K7 dW3 -> K5 dX3 -> K7 dW2 -> K5 dX2 -> K7 dW1 -> K6
//   TD3 update     = K9 sample -> target actor -> target critics -> y -> critic fwd/bwd ->
//                    C1 allreduce -> K10 Adam -> [actor fwd, dQ1/da, actor bwd, C1, K10, K11]
//
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <atomic>
#include "internal.h"

namespace spk {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void note_launch(int n) { g_launches += n; }

static thread_local cudaError_t g_launch_err = cudaSuccess;
void note_launch_error(cudaError_t e) { g_launch_err = e; }
cudaError_t take_launch_error() {
  const cudaError_t e = g_launch_err;
  g_launch_err = cudaSuccess;
  return e;
}
int& launch_priority() {
  thread_local int p = 0;
  return p;
}

bool pdl_enabled() {
  static const bool on = [] { const char* e = getenv("SPIKERL_PDL"); return !(e && e[0] == '0'); }();
  return on;
}

static int resolve_engine(const spikerl_actor_cfg* c, ActorDims* d) {
  const bool bf = c->precision == SPIKERL_BF16 || c->precision == SPIKERL_FP16;
  if (c->precision == SPIKERL_FP16) {   // fp16 operands exist on the tcgen05 engine only
    if (c->engine == SPIKERL_ENGINE_SIMT || !tc_supported(*d)) {
      set_error("FP16 precision needs the tcgen05 engine and a shape it supports");
      return SPIKERL_E_UNSUPPORTED;
    }
    d->engine = SPIKERL_ENGINE_TCGEN05;
    return SPIKERL_OK;
  }
  switch (c->engine) {
    case SPIKERL_ENGINE_SIMT: d->engine = SPIKERL_ENGINE_SIMT; return SPIKERL_OK;
    case SPIKERL_ENGINE_TCGEN05:
      if (!bf) { set_error("tcgen05 engine needs BF16 precision"); return SPIKERL_E_UNSUPPORTED; }
      d->engine = SPIKERL_ENGINE_TCGEN05;
      if (!tc_supported(*d)) { set_error("tcgen05 engine does not support this shape"); return SPIKERL_E_UNSUPPORTED; }
      return SPIKERL_OK;
    case SPIKERL_ENGINE_AUTO:
      // fp32 runs on the SIMT engine (the only fp32 engine); bf16 runs on tcgen05, and a shape it
      // cannot tile is an error, not a silent switch of engine (north_star: no multi-backend
      // dispatch). ENGINE_SIMT may still be requested explicitly for bf16.
      if (!bf) { d->engine = SPIKERL_ENGINE_SIMT; return SPIKERL_OK; }
      d->engine = SPIKERL_ENGINE_TCGEN05;
      if (!tc_supported(*d)) {
        set_error("bf16 actor: the tcgen05 engine cannot tile T=%d (needs T <= 16, or even T <= 32); request "
                  "SPIKERL_ENGINE_SIMT explicitly", d->T);
        return SPIKERL_E_UNSUPPORTED;
      }
      return SPIKERL_OK;
    default: set_error("unknown engine %d", c->engine); return SPIKERL_E_ARG;
  }
}

int actor_dims(const spikerl_actor_cfg* c, ActorDims* d) {
  if (!c) { set_error("null actor cfg"); return SPIKERL_E_ARG; }
  if (c->obs_dim < 1 || c->act_dim < 1 || c->pop_enc < 1 || c->pop_dec < 1 || c->hidden1 < 1 ||
      c->hidden2 < 1) {
    set_error("actor dims must be >= 1 (obs %d act %d pop %d/%d hidden %d/%d)", c->obs_dim, c->act_dim,
              c->pop_enc, c->pop_dec, c->hidden1, c->hidden2);
    return SPIKERL_E_DOMAIN;
  }
  if (c->T < 1 || c->T > 255) { set_error("T=%d outside [1,255]", c->T); return SPIKERL_E_DOMAIN; }
  if (!(c->d_c >= 0.f && c->d_c <= 1.f) || !(c->d_v >= 0.f && c->d_v <= 1.f) || !(c->v_th > 0.f) ||
      !(c->surr_window > 0.f) || !(c->sigma_floor >= 0.f)) {
    set_error("LIF constants out of domain (d_c %g d_v %g v_th %g window %g)", c->d_c, c->d_v, c->v_th,
              c->surr_window);
    return SPIKERL_E_DOMAIN;
  }
  if (c->reset_grad != 0 && c->reset_grad != 1) {
    set_error("reset_grad must be 0 (detached) or 1 (through the reset gate), got %d", c->reset_grad);
    return SPIKERL_E_DOMAIN;
  }
  if (c->precision != SPIKERL_FP32 && c->precision != SPIKERL_BF16 && c->precision != SPIKERL_FP16) {
    set_error("unknown precision %d", c->precision);
    return SPIKERL_E_ARG;
  }
  const long long k0 = (long long)c->obs_dim * c->pop_enc, n3 = (long long)c->act_dim * c->pop_dec;
  if (k0 > (1 << 20) || n3 > (1 << 20) || c->hidden1 > (1 << 20) || c->hidden2 > (1 << 20)) {
    set_error("actor too large");
    return SPIKERL_E_UNSUPPORTED;
  }
  d->S = c->obs_dim; d->A = c->act_dim; d->E = c->pop_enc; d->D = c->pop_dec;
  d->K0 = (int)k0; d->N1 = c->hidden1; d->N2 = c->hidden2; d->N3 = (int)n3; d->T = c->T;
  d->N[0] = d->K0; d->N[1] = d->N1; d->N[2] = d->N2; d->N[3] = d->N3;
  for (int l = 0; l < 4; ++l) { d->P[l] = round_up(d->N[l], kPad); d->Wd[l] = d->P[l] / 32; }
  size_t o = 0;
  const size_t sizes[SPIKERL_ACTOR_NPARAM] = {(size_t)d->K0, (size_t)d->K0, (size_t)d->N1 * d->K0,
                                               (size_t)d->N2 * d->N1, (size_t)d->N3 * d->N2,
                                               (size_t)d->A * d->D, (size_t)d->A};
  for (int i = 0; i < SPIKERL_ACTOR_NPARAM; ++i) { d->off[i] = o; o += sizes[i]; }
  d->off[SPIKERL_ACTOR_NPARAM] = o;
  size_t bo = 0;
  for (int l = 1; l <= 3; ++l) { d->boff[l - 1] = bo; bo += (size_t)d->P[l] * d->P[l - 1]; }
  d->boff[3] = bo;
  d->dc = c->d_c; d->dv = c->d_v; d->vth = c->v_th; d->win = c->surr_window; d->zh = c->surr_height;
  d->sigma_floor = c->sigma_floor;
  d->bf16 = c->precision == SPIKERL_BF16 || c->precision == SPIKERL_FP16;
  d->f16 = c->precision == SPIKERL_FP16;
  d->rho = c->reset_grad;
  if (d->rho && d->f16) {
    set_error("reset_grad = 1 is implemented for FP32 and BF16 precision (not FP16)");
    return SPIKERL_E_UNSUPPORTED;
  }
  return resolve_engine(c, d);
}

unsigned long long actor_cfg_hash(const spikerl_actor_cfg* c) {
  unsigned long long h = 1469598103934665603ULL;
  const unsigned char* p = (const unsigned char*)c;
  for (size_t i = 0; i < sizeof(*c); ++i) { h ^= p[i]; h *= 1099511628211ULL; }
  return h;
}

TapeLayout tape_layout(const ActorDims& d, int B) {
  TapeLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += align_up(bytes, 256); return r; };
  L.A = take(sizeof(float) * (size_t)B * d.K0);
  for (int l = 0; l < 4; ++l) L.bits[l] = take(sizeof(uint32_t) * (size_t)d.T * B * d.Wd[l]);
  L.mask[0] = 0;
  for (int l = 1; l < 4; ++l) L.mask[l] = take(sizeof(uint32_t) * (size_t)d.T * B * d.Wd[l]);
  L.counts = take((size_t)B * d.N3);
  L.act = take(sizeof(float) * (size_t)B * d.A);
  L.tpad = round_up(d.T, 16);
  for (int l = 0; l < 4; ++l) { L.bitsT[l] = 0; L.maskT[l] = 0; L.V[l] = 0; }
  if (d.rho)
    for (int l = 1; l <= 3; ++l) L.V[l] = take(sizeof(float) * (size_t)d.T * B * d.P[l]);
  if (d.engine == SPIKERL_ENGINE_TCGEN05) {
    const size_t quads = (size_t)round_up(B, 32) / 4;
    for (int l = 1; l <= 2; ++l) {
      L.bitsT[l] = take(quads * d.P[l] * (L.tpad / 2));
      L.maskT[l] = take(quads * d.P[l] * (L.tpad / 2));
    }
  }
  L.total = o;
  return L;
}

int critic_dims(const spikerl_critic_cfg* c, CriticDims* d) {
  if (!c) { set_error("null critic cfg"); return SPIKERL_E_ARG; }
  if (c->in_dim < 1 || c->hidden1 < 1 || c->hidden2 < 1) {
    set_error("critic dims must be >= 1");
    return SPIKERL_E_DOMAIN;
  }
  if (c->precision != SPIKERL_FP32 && c->precision != SPIKERL_BF16) {
    set_error("unknown precision %d", c->precision);
    return SPIKERL_E_ARG;
  }
  d->in = c->in_dim; d->H1 = c->hidden1; d->H2 = c->hidden2; d->bf16 = c->precision == SPIKERL_BF16;
  const size_t sizes[SPIKERL_CRITIC_NPARAM] = {(size_t)d->H1 * d->in, (size_t)d->H1,
                                                (size_t)d->H2 * d->H1, (size_t)d->H2, (size_t)d->H2, 1};
  size_t o = 0;
  for (int i = 0; i < SPIKERL_CRITIC_NPARAM; ++i) { d->off[i] = o; o += sizes[i]; }
  d->off[SPIKERL_CRITIC_NPARAM] = o;
  return SPIKERL_OK;
}

// compute-time checks of a critic config, made on the host before anything is enqueued
static int critic_supported(const CriticDims& c, bool loss_scaling) {
  if (c.bf16 && !critic_mma_ok(c)) {
    set_error("bf16 critic: the tensor-core critic needs hidden widths 256-256 and in_dim <= 512 (got %d-%d, %d)",
              c.H1, c.H2, c.in);
    return SPIKERL_E_UNSUPPORTED;
  }
  if (loss_scaling && !c.bf16) {
    set_error("dynamic loss scaling needs the bf16 tensor-core critic");
    return SPIKERL_E_UNSUPPORTED;
  }
  return SPIKERL_OK;
}

// ------------------------------------------------------------------ actor workspace layout
struct ActorWs {
  size_t tape;      // inference-only spike planes (TapeLayout at offset 0)
  size_t G[4];      // G1..G3 [T][B][P_l] (fp32 or bf16); G[0] unused
  size_t Gsum;      // [B][P1]
  size_t g_pre;     // [B][A] fp32
  size_t dec_part;  // decoder parameter-gradient chunk partials
  size_t enc_part;  // encoder partials
  size_t dw_part[4];   // tcgen05 split-K dW_l partials (one region per layer: the dW run concurrently)
  size_t total;
};

static ActorWs actor_ws_layout(const ActorDims& d, int B) {
  ActorWs w{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += align_up(bytes, 256); return r; };
  const size_t gsz = d.bf16 ? 2 : 4;
  w.tape = take(tape_layout(d, B).total);
  w.G[0] = 0;
  for (int l = 1; l <= 3; ++l) w.G[l] = take(gsz * (size_t)d.T * B * d.P[l]);
  w.Gsum = take(gsz * (size_t)B * d.P[1]);
  w.g_pre = take(sizeof(float) * (size_t)B * d.A);
  w.dec_part = take(sizeof(float) * (size_t)dec_param_chunks(B) * (d.N3 + d.A));
  const bool tc = d.engine == SPIKERL_ENGINE_TCGEN05;
  const size_t ep = enc_grad_partial_bytes(d, B), ept = tc ? tc_enc_partial_bytes(d, B) : 0;
  w.enc_part = take(ep > ept ? ep : ept);
  w.dw_part[0] = 0;
  for (int l = 1; l <= 3; ++l) w.dw_part[l] = take(tc ? tc_dw_partial_bytes(d, B, l) : 0);
  w.total = o;
  return w;
}

// spikes_only: a forward no backward will read (inference, TD3's target actor): the encoder skips the
// stimulation plane A and computes the exact A only where a spike is possible (enc_fwd_kernel SPK);
// spike planes, counts and actions are bitwise those of the recording forward (tested)
static int actor_forward_impl(const ActorDims& d, int B, const float* params,
                              const __nv_bfloat16* pb16, const float* obs, float* actions,
                              char* tape, cudaStream_t st, const TargetSmooth* smooth = nullptr,
                              bool spikes_only = false, bool skip_decoder = false) {
  const TapeLayout L = tape_layout(d, B);
  float* A = spikes_only ? nullptr : (float*)(tape + L.A);
  uint32_t* bits[4];
  uint32_t* mask[4];
  for (int l = 0; l < 4; ++l) { bits[l] = (uint32_t*)(tape + L.bits[l]); mask[l] = (uint32_t*)(tape + L.mask[l]); }
  uint8_t* counts = (uint8_t*)(tape + L.counts);
  SPK_TRY(launch_enc_fwd(d, B, obs, params + d.off[SPIKERL_ACTOR_MU], params + d.off[SPIKERL_ACTOR_SIGMA],
                         A, bits[0], st));
  for (int l = 1; l <= 3; ++l) {
    const float* Wf = params + d.off[SPIKERL_ACTOR_W1 + l - 1];
    const __nv_bfloat16* Wb = d.bf16 ? pb16 + d.boff[l - 1] : nullptr;
    uint8_t* cnt = (l == 3) ? counts : nullptr;
    float* vout = L.V[l] ? (float*)(tape + L.V[l]) : nullptr;
    if (d.engine == SPIKERL_ENGINE_TCGEN05)
      SPK_TRY(launch_lif_fwd_tc(d, l, B, bits[l - 1], Wb, bits[l], mask[l], cnt,
                                L.bitsT[l] ? (uint8_t*)(tape + L.bitsT[l]) : nullptr,
                                L.maskT[l] ? (uint8_t*)(tape + L.maskT[l]) : nullptr, L.tpad, vout, st));
    else
      SPK_TRY(launch_lif_fwd_simt(d, l, B, bits[l - 1], Wf, Wb, bits[l], mask[l], cnt, vout, st));
  }
  if (skip_decoder) return SPIKERL_OK;   // the caller decodes inside the target critics' launch
  SPK_TRY(launch_dec_fwd(d, B, counts, params + d.off[SPIKERL_ACTOR_WD], params + d.off[SPIKERL_ACTOR_BD],
                         actions, (float*)(tape + L.act), st, smooth));
  return SPIKERL_OK;
}

// the target actor's decoder + smoothing handed to the target critics' forward launch (CriticDecode)
static CriticDecode target_decode(const ActorDims& d, int B, const float* params, char* tape, float* actions,
                                  const TargetSmooth& ts) {
  const TapeLayout L = tape_layout(d, B);
  CriticDecode c{};
  c.counts = (const uint8_t*)(tape + L.counts);
  c.Wd = params + d.off[SPIKERL_ACTOR_WD];
  c.bd = params + d.off[SPIKERL_ACTOR_BD];
  c.D = d.D; c.T = d.T;
  c.act_out = actions;
  c.act_tape = (float*)(tape + L.act);
  c.ts = ts;
  return c;
}

// Gradient buckets of the actor's flat layout mu|sigma|W1|W2|W3|Wd|bd, in the order the backward
// completes them: tail = W3|Wd|bd (dW3 + decoder), W2 (dW2), head = mu|sigma|W1 (dW1 + encoder).
// Bounds: [0, off W2, off W3, total).
static void actor_grad_buckets(const ActorDims& d, size_t out[4]) {
  out[0] = 0;
  out[1] = d.off[SPIKERL_ACTOR_W2];
  out[2] = d.off[SPIKERL_ACTOR_W3];
  out[3] = d.off[SPIKERL_ACTOR_NPARAM];
}

// comm != NULL: the gradient mean over ranks (PAPER.md:135 average_gradients, PAPER.md:144 DDP
// "during backpropagation") runs per bucket on the library's comm stream as soon as the bucket's
// producers finish, overlapping the rest of the backward (the tail and W2 buckets run while dX2,
// dW1 and the encoder gradient compute); the call's stream joins the comm stream at the end.
static int actor_backward_impl(const ActorDims& d, int B, const float* params,
                               const __nv_bfloat16* pb16, const float* obs, const char* tape,
                               const float* grad_a, float* grads, int accum, char* ws,
                               cudaStream_t st, spikerl_comm* comm = nullptr) {
  const TapeLayout L = tape_layout(d, B);
  const ActorWs W = actor_ws_layout(d, B);
  const uint32_t* bits[4];
  const uint32_t* mask[4];
  for (int l = 0; l < 4; ++l) {
    bits[l] = (const uint32_t*)(tape + L.bits[l]);
    mask[l] = (const uint32_t*)(tape + L.mask[l]);
  }
  const uint8_t* counts = (const uint8_t*)(tape + L.counts);
  const float* act = (const float*)(tape + L.act);
  void* G[4] = {nullptr, ws + W.G[1], ws + W.G[2], ws + W.G[3]};
  void* Gsum = ws + W.Gsum;
  float* g_pre = (float*)(ws + W.g_pre);
  const float* V[4] = {nullptr, nullptr, nullptr, nullptr};
  for (int l = 1; l <= 3; ++l) V[l] = L.V[l] ? (const float*)(tape + L.V[l]) : nullptr;
  SPK_TRY(launch_dec_bwd_outscan(d, B, grad_a, act, counts, params + d.off[SPIKERL_ACTOR_WD], bits[3], mask[3],
                                 V[3], G[3], g_pre, st));
  // Small problems (kernels far from filling the GPU): dW_l and the decoder parameter grads run
  // on side streams next to the dX chain, each as soon as its G_l exists; the critical path is
  // then outscan -> dX3 -> dX2 -> max(encoder grad, dW1). Large problems stay on one stream
  // (persistent kernels that each own every SM).
  const bool tc = d.engine == SPIKERL_ENGINE_TCGEN05;
  AuxPool* aux = nullptr;
  SPK_TRY(aux_pool(&aux));
  const bool fork = (long long)d.T * B <= 32768;
  cudaStream_t sw[4] = {st, st, st, st};   // sw[l]: stream of dW_l; sw[0]: decoder params
  if (fork) { sw[0] = aux->side[3]; sw[3] = aux->side[3]; sw[2] = aux->side[4]; sw[1] = aux->side[5]; }
  auto branch = [&](cudaStream_t s, int e) -> int {   // s continues after everything enqueued on st
    if (s == st) return SPIKERL_OK;
    return stream_after(s, st, aux->ev[8 + e]);
  };
  size_t bk[4];
  actor_grad_buckets(d, bk);
  cudaStream_t sc = aux->side[8];
  int nev = 0;
  // bucket [lo, hi) allreduced on the comm stream after the producers' work enqueued so far
  // (np producers: the stream handles themselves may be 0, the legacy default stream)
  auto bucket = [&](size_t lo, size_t hi, cudaStream_t p0, cudaStream_t p1, int np) -> int {
    if (!comm) return SPIKERL_OK;
    const cudaStream_t prod[2] = {p0, p1};
    for (int i = 0; i < np; ++i) {
      SPK_TRY(stream_after(sc, prod[i], aux->ev[20 + nev]));
      ++nev;
    }
    static const char* names[3] = {"allreduce_bucket_head", "allreduce_bucket_W2", "allreduce_bucket_tail"};
    ProfScope ps_(names[lo == bk[0] ? 0 : (lo == bk[1] ? 1 : 2)], PB_LATENCY, 0.0, 8.0 * (hi - lo), sc);
    return spikerl_allreduce_grads(comm, grads + lo, hi - lo, sc);
  };
  SPK_TRY(branch(sw[0], 0));
  SPK_TRY(launch_dec_param_grads(d, B, g_pre, counts, grads + d.off[SPIKERL_ACTOR_WD],
                                 grads + d.off[SPIKERL_ACTOR_BD], (float*)(ws + W.dec_part), accum, sw[0]));
  for (int l = 3; l >= 1; --l) {
    const float* Wf = params + d.off[SPIKERL_ACTOR_W1 + l - 1];
    const __nv_bfloat16* Wb = d.bf16 ? pb16 + d.boff[l - 1] : nullptr;
    float* dW = grads + d.off[SPIKERL_ACTOR_W1 + l - 1];
    if (l != 3) SPK_TRY(branch(sw[l], l));   // G_l was produced on st
    if (tc)
      SPK_TRY(launch_lif_dw_tc(d, l, B, G[l], bits[l - 1], dW, (float*)(ws + W.dw_part[l]), accum, sw[l]));
    else
      SPK_TRY(launch_lif_dw_simt(d, l, B, G[l], bits[l - 1], dW, accum, sw[l]));
    if (l == 3) SPK_TRY(bucket(bk[2], bk[3], sw[3], sw[0], sw[0] != sw[3] ? 2 : 1));
    if (l == 2) SPK_TRY(bucket(bk[1], bk[2], sw[2], sw[2], 1));
    if (l >= 2) {
      if (tc)
        SPK_TRY(launch_lif_dx_tc(d, l, B, G[l], Wb, (const uint8_t*)(tape + L.bitsT[l - 1]),
                                 (const uint8_t*)(tape + L.maskT[l - 1]), L.tpad, V[l - 1], G[l - 1],
                                 l == 2 ? Gsum : nullptr, st));
      else
        SPK_TRY(launch_lif_dx_simt(d, l, B, G[l], Wf, Wb, bits[l - 1], mask[l - 1], V[l - 1], G[l - 1],
                                   l == 2 ? Gsum : nullptr, st));
    }
  }
  const float* A = (const float*)(tape + L.A);
  if (tc)
    SPK_TRY(launch_enc_grad_tc(d, B, Gsum, pb16 + d.boff[0], A, obs, params + d.off[SPIKERL_ACTOR_MU],
                               params + d.off[SPIKERL_ACTOR_SIGMA], (float*)(ws + W.enc_part),
                               grads + d.off[SPIKERL_ACTOR_MU], grads + d.off[SPIKERL_ACTOR_SIGMA], accum, st));
  else
    SPK_TRY(launch_enc_grad_simt(d, B, Gsum, params + d.off[SPIKERL_ACTOR_W1], d.bf16 ? pb16 + d.boff[0] : nullptr,
                                 A, obs, params + d.off[SPIKERL_ACTOR_MU], params + d.off[SPIKERL_ACTOR_SIGMA],
                                 (float*)(ws + W.enc_part), grads + d.off[SPIKERL_ACTOR_MU],
                                 grads + d.off[SPIKERL_ACTOR_SIGMA], accum, st));
  SPK_TRY(bucket(bk[0], bk[1], sw[1], st, sw[1] != st ? 2 : 1));
  if (fork) {   // join every side stream back into st
    for (int i = 3; i <= 5; ++i) {
      SPK_CHECK_CUDA(cudaEventRecord(aux->ev[8 + i], aux->side[i]));
      SPK_CHECK_CUDA(cudaStreamWaitEvent(st, aux->ev[8 + i], 0));
    }
  }
  if (comm) SPK_TRY(stream_after(st, sc, aux->ev[27]));   // join the comm stream
  return SPIKERL_OK;
}

// ------------------------------------------------------------------ TD3 workspace layout
struct Td3Ws {
  size_t s, a, r, s2, d, a2, at, api, qt, q, y, ga, lossa, ctr, tape, actor_ws, critic_ws, critic_ws_t, total;
};

static Td3Ws td3_ws_layout(const ActorDims& ad, const CriticDims& cd, int B) {
  Td3Ws w{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += align_up(bytes, 256); return r; };
  const size_t f = sizeof(float);
  w.s = take(f * B * ad.S); w.a = take(f * B * ad.A); w.r = take(f * B); w.s2 = take(f * B * ad.S);
  w.d = take(f * B); w.a2 = take(f * B * ad.A); w.at = take(f * B * ad.A); w.api = take(f * B * ad.A);
  w.qt = take(f * 2 * B); w.q = take(f * 2 * B); w.y = take(f * B); w.ga = take(f * B * ad.A);
  w.lossa = take(f * 4);
  w.ctr = take(sizeof(unsigned long long));
  w.tape = take(tape_layout(ad, B).total);
  w.actor_ws = take(actor_ws_layout(ad, B).total);
  w.critic_ws = take(critic_ws_bytes(cd, B));
  w.critic_ws_t = take(critic_ws_bytes(cd, B));   // target-critic forward runs concurrently
  w.total = o;
  return w;
}

// The optimiser step of each network after its backward: the gradient mean over ranks + Adam, either
// as the NCCL allreduce (the actor's is already bucketed inside its backward) and the Adam launch, or
// as the one fused allreduce + Adam kernel over symmetric memory when a plan is given (NEXT #1).
// polyak (actor steps): the target soft update t <- tau p + (1 - tau) t of that network, fused into its
// Adam launch (one launch less at the end of the update's critical path); with the fused allreduce
// + Adam kernel or loss scaling it stays a launch of its own right after, same arithmetic.
// bf16 views of a TD3 critic: the online twins keep W1T only for the action rows [S, S+A) (dQ1/da), the
// targets (forward only) neither W1T nor W2T
static Bf16Views td3_critic_views(const CriticDims& cd, const ActorDims& ad, void* buf, bool target) {
  Bf16Views v = critic_bf16_views(cd, ad.bf16 ? (__nv_bfloat16*)buf : nullptr);
  if (v.kind == 2) {
    v.w1t_lo = target ? 0 : ad.S;
    v.w1t_hi = target ? 0 : ad.S + ad.A;
    v.w2t = target ? 0 : 1;
  }
  return v;
}

// the whole critic update as one launch (k_critic_mma.cu critic_update_fused): bf16 small-batch critic,
// one GPU (no gradient allreduce between the gradients and Adam), no loss scaling
static bool critic_update_fusable(const CriticDims& cd, int B, const spikerl_td3_bufs* b, spikerl_comm* comm) {
  return !comm && !b->amp && critic_fused_ok(cd, B);
}

// the target decoder inside the target critics' forward: with the separate critic launches only (A/B r02,
// one box: configs[1] 82.4 -> 80.1, configs[3] B = 100 110.7 -> 109.7 us per update; with the fused
// critic update, configs[2], 109.4 -> 112.9)
static bool target_decode_ok(const CriticDims& cd, const ActorDims& ad, int B, const spikerl_td3_bufs* b,
                             spikerl_comm* comm) {
  return critic_decode_ok(cd, B, ad.A, ad.D) && !critic_update_fusable(cd, B, b, comm);
}

static int critic_optimise(const spikerl_td3_bufs* b, spikerl_comm* comm, const spikerl_td3_cfg* hp, const CriticDims& cd,
                           size_t Pc, const Bf16Views* cv, float* amp_c, cudaStream_t st,
                           const PolyakFuse* polyak = nullptr) {
  if (comm && b->fused_critic) {
    SPK_TRY(fused_adam_launch(b->fused_critic, b->m_critic, b->v_critic, b->adam_steps, hp->lr_critic, hp->beta1,
                              hp->beta2, hp->eps, 0, 0, 0.f, (unsigned int*)(b->adam_steps + 1), cv, st));
    return polyak ? launch_polyak(polyak->t, b->critic, 2 * Pc, polyak->tau, polyak->views, st) : SPIKERL_OK;
  }
  SPK_TRY(spikerl_allreduce_grads(comm, b->grad_critic, 2 * Pc, st));
  if (amp_c) SPK_TRY(launch_amp_check(b->grad_critic, 2 * Pc, amp_c, st));
  // the tensor-core critic: the layout-aware Adam (coalesced W2T stores); SPIKERL_CRITIC_ADAM_TILED=0: the
  // flat adam_kernel (same result)
  static const bool tiled = [] { const char* e = getenv("SPIKERL_CRITIC_ADAM_TILED"); return !(e && e[0] == '0'); }();
  if (tiled && !amp_c && critic_adam_ok(cd, cv, polyak))
    return launch_critic_adam(cd, b->critic, b->grad_critic, b->m_critic, b->v_critic, b->adam_steps, hp->lr_critic,
                              hp->beta1, hp->beta2, hp->eps, cv, polyak, st);
  SPK_TRY(launch_adam(b->critic, b->grad_critic, b->m_critic, b->v_critic, 2 * Pc, b->adam_steps, hp->lr_critic,
                      hp->beta1, hp->beta2, hp->eps, 0, 0, 0.f, (unsigned int*)(b->adam_steps + 1), cv, st, amp_c,
                      hp->amp_growth, hp->amp_backoff, hp->amp_interval, amp_c ? nullptr : polyak));
  return (polyak && amp_c) ? launch_polyak(polyak->t, b->critic, 2 * Pc, polyak->tau, polyak->views, st) : SPIKERL_OK;
}

static int actor_optimise(const spikerl_td3_bufs* b, spikerl_comm* comm, const spikerl_td3_cfg* hp,
                          const ActorDims& ad, size_t Pa, const Bf16Views* av, float* amp_a, cudaStream_t st,
                          const PolyakFuse* polyak = nullptr) {
  if (comm && b->fused_actor) {
    SPK_TRY(fused_adam_launch(b->fused_actor, b->m_actor, b->v_actor, b->adam_steps + 2, hp->lr_actor, hp->beta1,
                              hp->beta2, hp->eps, ad.off[SPIKERL_ACTOR_SIGMA], ad.off[SPIKERL_ACTOR_W1],
                              ad.sigma_floor, (unsigned int*)(b->adam_steps + 3), av, st));
    return polyak ? launch_polyak(polyak->t, b->actor, Pa, polyak->tau, polyak->views, st) : SPIKERL_OK;
  }
  if (amp_a) SPK_TRY(launch_amp_check(b->grad_actor, Pa, amp_a, st));
  SPK_TRY(launch_adam(b->actor, b->grad_actor, b->m_actor, b->v_actor, Pa, b->adam_steps + 2, hp->lr_actor, hp->beta1,
                      hp->beta2, hp->eps, ad.off[SPIKERL_ACTOR_SIGMA], ad.off[SPIKERL_ACTOR_W1], ad.sigma_floor,
                      (unsigned int*)(b->adam_steps + 3), av, st, amp_a, hp->amp_growth, hp->amp_backoff,
                      hp->amp_interval, amp_a ? nullptr : polyak));
  return (polyak && amp_a) ? launch_polyak(polyak->t, b->actor, Pa, polyak->tau, polyak->views, st) : SPIKERL_OK;
}

__global__ void neg_mean_kernel(int B, const float* __restrict__ q, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[256];
  float s = 0.f;
  for (int b = threadIdx.x; b < B; b += 256) s = __fadd_rn(s, q[b]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = __fadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = -__fdiv_rn(red[0], (float)B);
}

}  // namespace spk

using namespace spk;

extern "C" {

const char* spikerl_last_error(void) { return g_err; }
const char* spikerl_version(void) { return "spikerl-b200 0.1 (sm_100a)"; }
long long spikerl_launch_count(int reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}

int spikerl_actor_cfg_check(const spikerl_actor_cfg* cfg) {
  ActorDims d;
  return actor_dims(cfg, &d);
}

int spikerl_actor_param_offsets(const spikerl_actor_cfg* cfg, size_t* offsets) {
  ActorDims d;
  SPK_TRY(actor_dims(cfg, &d));
  if (!offsets) { set_error("null offsets"); return SPIKERL_E_ARG; }
  memcpy(offsets, d.off, sizeof(d.off));
  return SPIKERL_OK;
}

size_t spikerl_actor_param_count(const spikerl_actor_cfg* cfg) {
  ActorDims d;
  return actor_dims(cfg, &d) == SPIKERL_OK ? d.off[SPIKERL_ACTOR_NPARAM] : 0;
}

int spikerl_critic_param_offsets(const spikerl_critic_cfg* cfg, size_t* offsets) {
  CriticDims d;
  SPK_TRY(critic_dims(cfg, &d));
  if (!offsets) { set_error("null offsets"); return SPIKERL_E_ARG; }
  memcpy(offsets, d.off, sizeof(d.off));
  return SPIKERL_OK;
}

size_t spikerl_critic_param_count(const spikerl_critic_cfg* cfg) {
  CriticDims d;
  return critic_dims(cfg, &d) == SPIKERL_OK ? d.off[SPIKERL_CRITIC_NPARAM] : 0;
}

size_t spikerl_actor_bf16_bytes(const spikerl_actor_cfg* cfg) {
  ActorDims d;
  return actor_dims(cfg, &d) == SPIKERL_OK ? d.boff[3] * sizeof(__nv_bfloat16) : 0;
}

size_t spikerl_critic_bf16_bytes(const spikerl_critic_cfg* cfg) {
  CriticDims d;
  return critic_dims(cfg, &d) == SPIKERL_OK ? align_up(critic_bf16_elems(d) * 2, 16) : 0;
}

int spikerl_critic_bf16_layout(const spikerl_critic_cfg* cfg, long long* out8) {
  CriticDims d;
  SPK_TRY(critic_dims(cfg, &d));
  if (!out8) { set_error("spikerl_critic_bf16_layout: null output"); return SPIKERL_E_ARG; }
  if (!critic_mma_ok(d)) { set_error("spikerl_critic_bf16_layout: not the tensor-core critic"); return SPIKERL_E_UNSUPPORTED; }
  critic_bf16_layout(d, out8);
  return SPIKERL_OK;
}

size_t spikerl_actor_tape_bytes(const spikerl_actor_cfg* cfg, int batch) {
  ActorDims d;
  if (actor_dims(cfg, &d) != SPIKERL_OK || batch < 1) return 0;
  return tape_layout(d, batch).total;
}

size_t spikerl_actor_workspace_bytes(const spikerl_actor_cfg* cfg, int batch) {
  ActorDims d;
  if (actor_dims(cfg, &d) != SPIKERL_OK || batch < 1) return 0;
  AuxPool* aux = nullptr;   // create the fork/join streams now, outside any graph capture
  if (aux_pool(&aux) != SPIKERL_OK) cudaGetLastError();   // no device (host-only query): later
  return actor_ws_layout(d, batch).total;
}

size_t spikerl_actor_workspace_tape_offset(const spikerl_actor_cfg* cfg, int batch) {
  ActorDims d;
  if (actor_dims(cfg, &d) != SPIKERL_OK || batch < 1) return 0;
  return actor_ws_layout(d, batch).tape;
}

size_t spikerl_critic_workspace_bytes(const spikerl_critic_cfg* cfg, int batch) {
  CriticDims d;
  if (critic_dims(cfg, &d) != SPIKERL_OK || batch < 1) return 0;
  AuxPool* aux = nullptr;   // create the fork/join streams now, outside any graph capture
  if (aux_pool(&aux) != SPIKERL_OK) cudaGetLastError();   // no device (host-only query): later
  return critic_ws_bytes(d, batch);
}

size_t spikerl_td3_workspace_bytes(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg, int batch) {
  ActorDims ad;
  CriticDims cd;
  if (actor_dims(acfg, &ad) != SPIKERL_OK || critic_dims(ccfg, &cd) != SPIKERL_OK || batch < 1) return 0;
  AuxPool* aux = nullptr;   // create the fork/join streams now, outside any graph capture
  if (aux_pool(&aux) != SPIKERL_OK) cudaGetLastError();   // no device (host-only query): later
  return td3_ws_layout(ad, cd, batch).total;
}

int spikerl_actor_tape_layout(const spikerl_actor_cfg* cfg, int batch, spikerl_tape_layout* out) {
  ActorDims d;
  SPK_TRY(actor_dims(cfg, &d));
  if (!out || batch < 1) { set_error("bad tape layout arguments"); return SPIKERL_E_ARG; }
  const TapeLayout L = tape_layout(d, batch);
  out->A = L.A;
  for (int l = 0; l < 4; ++l) {
    out->bits[l] = L.bits[l]; out->mask[l] = L.mask[l]; out->padded[l] = d.P[l];
    out->bitsT[l] = L.bitsT[l]; out->maskT[l] = L.maskT[l];
  }
  out->tpad = L.tpad;
  for (int l = 0; l < 4; ++l) out->V[l] = L.V[l];
  out->counts = L.counts; out->act = L.act; out->total = L.total;
  return SPIKERL_OK;
}

int spikerl_actor_refresh_bf16(const spikerl_actor_cfg* cfg, const float* params, void* params_bf16,
                               spikerl_stream_t stream) {
  ActorDims d;
  SPK_TRY(actor_dims(cfg, &d));
  if (!params || !params_bf16) { set_error("null params"); return SPIKERL_E_ARG; }
  return launch_actor_refresh_bf16(d, params, (__nv_bfloat16*)params_bf16, (cudaStream_t)stream);
}

int spikerl_critic_refresh_bf16(const spikerl_critic_cfg* cfg, int n_critics, const float* params,
                                void* params_bf16, spikerl_stream_t stream) {
  CriticDims d;
  SPK_TRY(critic_dims(cfg, &d));
  if (!params || !params_bf16 || n_critics != 2) {
    set_error("bad refresh arguments (the bf16 working copy holds a twin pair: n_critics must be 2)");
    return SPIKERL_E_ARG;
  }
  return launch_critic_refresh(d, params, (__nv_bfloat16*)params_bf16, (cudaStream_t)stream);
}

static const unsigned long long kTapeMagic = 0x5350494b45524c31ULL;  // "SPIKERL1"

int spikerl_actor_forward(const spikerl_actor_cfg* cfg, int batch, const float* params,
                          const void* params_bf16, const float* obs, float* actions, spikerl_tape* tape,
                          void* workspace, spikerl_stream_t stream) {
  ActorDims d;
  SPK_TRY(actor_dims(cfg, &d));
  if (batch < 1 || !params || !obs || !actions || (d.bf16 && !params_bf16)) {
    set_error("spikerl_actor_forward: bad arguments (batch %d)", batch);
    return SPIKERL_E_ARG;
  }
  const TapeLayout L = tape_layout(d, batch);
  char* tp;
  if (tape) {
    if (!tape->dev || tape->bytes < L.total) {
      set_error("tape buffer too small (%zu < %zu)", tape->bytes, L.total);
      return SPIKERL_E_ARG;
    }
    tp = (char*)tape->dev;
  } else {
    if (!workspace) { set_error("inference-only forward needs a workspace"); return SPIKERL_E_ARG; }
    tp = (char*)workspace + actor_ws_layout(d, batch).tape;
  }
  SPK_TRY(actor_forward_impl(d, batch, params, (const __nv_bfloat16*)params_bf16, obs, actions, tp,
                             (cudaStream_t)stream, nullptr, tape == nullptr));
  if (tape) {
    tape->magic = kTapeMagic;
    tape->cfg_hash = actor_cfg_hash(cfg);
    tape->batch = batch;
  }
  return SPIKERL_OK;
}

int spikerl_actor_backward(const spikerl_actor_cfg* cfg, int batch, const float* params,
                           const void* params_bf16, const float* obs, const spikerl_tape* tape,
                           const float* grad_actions, float* grad_params, int accumulate, void* workspace,
                           spikerl_stream_t stream) {
  ActorDims d;
  SPK_TRY(actor_dims(cfg, &d));
  if (batch < 1 || !params || !obs || !tape || !grad_actions || !grad_params || !workspace ||
      (d.bf16 && !params_bf16)) {
    set_error("spikerl_actor_backward: bad arguments");
    return SPIKERL_E_ARG;
  }
  if (tape->magic != kTapeMagic || tape->cfg_hash != actor_cfg_hash(cfg) || tape->batch != batch || !tape->dev) {
    set_error("tape does not belong to this (cfg, batch)");
    return SPIKERL_E_STATE;
  }
  return actor_backward_impl(d, batch, params, (const __nv_bfloat16*)params_bf16, obs, (const char*)tape->dev,
                             grad_actions, grad_params, accumulate ? 1 : 0, (char*)workspace,
                             (cudaStream_t)stream);
}

int spikerl_actor_backward_dp(const spikerl_actor_cfg* cfg, int batch, const float* params,
                              const void* params_bf16, const float* obs, const spikerl_tape* tape,
                              const float* grad_actions, float* grad_params, int accumulate, spikerl_comm* comm,
                              void* workspace, spikerl_stream_t stream) {
  ActorDims d;
  SPK_TRY(actor_dims(cfg, &d));
  if (batch < 1 || !params || !obs || !tape || !grad_actions || !grad_params || !workspace ||
      (d.bf16 && !params_bf16)) {
    set_error("spikerl_actor_backward_dp: bad arguments");
    return SPIKERL_E_ARG;
  }
  if (tape->magic != kTapeMagic || tape->cfg_hash != actor_cfg_hash(cfg) || tape->batch != batch || !tape->dev) {
    set_error("tape does not belong to this (cfg, batch)");
    return SPIKERL_E_STATE;
  }
  return actor_backward_impl(d, batch, params, (const __nv_bfloat16*)params_bf16, obs, (const char*)tape->dev,
                             grad_actions, grad_params, accumulate ? 1 : 0, (char*)workspace, (cudaStream_t)stream,
                             comm);
}

int spikerl_actor_grad_buckets(const spikerl_actor_cfg* cfg, size_t* bounds) {
  ActorDims d;
  SPK_TRY(actor_dims(cfg, &d));
  if (!bounds) { set_error("null bounds"); return SPIKERL_E_ARG; }
  actor_grad_buckets(d, bounds);
  return SPIKERL_OK;
}

int spikerl_critic_fwd_bwd(const spikerl_critic_cfg* cfg, int batch, const float* params2,
                           const void* params2_bf16, const float* obs, int obs_dim, const float* act, int act_dim,
                           const float* target_y, float* q, float* loss, float* grad_params2, float* grad_act,
                           float act_grad_scale, void* workspace, spikerl_stream_t stream) {
  CriticDims c;
  SPK_TRY(critic_dims(cfg, &c));
  if (batch < 1 || !params2 || !obs || !act || !q || !workspace || obs_dim < 0 || act_dim < 1 ||
      obs_dim + act_dim != c.in || (c.bf16 && !params2_bf16)) {
    set_error("spikerl_critic_fwd_bwd: bad arguments");
    return SPIKERL_E_ARG;
  }
  SPK_TRY(critic_supported(c, false));
  const TdY ty{target_y, nullptr, nullptr, nullptr, 0.f, batch, nullptr};
  return critic_fwd_bwd(c, batch, params2, (const __nv_bfloat16*)params2_bf16, obs, obs_dim, act, act_dim,
                        target_y ? &ty : nullptr, q, target_y ? loss : nullptr, grad_params2, grad_act, act_grad_scale,
                        2, workspace, (cudaStream_t)stream);
}

int spikerl_adam(float* params, const float* grads, float* m, float* v, size_t n, long long* step_counter,
                 float lr, float beta1, float beta2, float eps, size_t clamp_lo, size_t clamp_hi, float clamp_min,
                 spikerl_stream_t stream) {
  if (!params || !grads || !m || !v || !step_counter || n == 0) {
    set_error("spikerl_adam: bad arguments");
    return SPIKERL_E_ARG;
  }
  return launch_adam(params, grads, m, v, n, step_counter, lr, beta1, beta2, eps, clamp_lo, clamp_hi, clamp_min,
                     (unsigned int*)(step_counter + 1), nullptr, (cudaStream_t)stream);
}

int spikerl_polyak(float* target, const float* source, size_t n, float tau, spikerl_stream_t stream) {
  if (!target || !source || n == 0) { set_error("spikerl_polyak: bad arguments"); return SPIKERL_E_ARG; }
  return launch_polyak(target, source, n, tau, nullptr, (cudaStream_t)stream);
}

// raised launch priority of a TD3 update's critical chain (see spikerl_td3_update_pair)
static int td3_priority(int batch) {
  static const int prio_env = [] { const char* e = getenv("SPIKERL_TD3_PRIO"); return e ? atoi(e) : -1; }();
  if (prio_env >= 0) return -prio_env;
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return batch < 1024 ? hi : 0;
}

int spikerl_td3_update(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg, const spikerl_td3_cfg* hp,
                       const spikerl_td3_bufs* b, long long step, unsigned long long seed, const long long* indices,
                       const float* noise, spikerl_comm* comm, float* losses, void* workspace,
                       spikerl_stream_t stream) {
  ActorDims ad;
  CriticDims cd;
  SPK_TRY(actor_dims(acfg, &ad));
  SPK_TRY(critic_dims(ccfg, &cd));
  if (!hp || !b || !workspace || !losses || step < 1) {
    set_error("spikerl_td3_update: bad arguments");
    return SPIKERL_E_ARG;
  }
  const int B = hp->batch;
  if (B < 1 || cd.in != ad.S + ad.A || hp->policy_delay < 1 || cd.bf16 != ad.bf16) {
    set_error("spikerl_td3_update: inconsistent configs (batch %d, critic in %d vs S+A %d)", B, cd.in, ad.S + ad.A);
    return SPIKERL_E_ARG;
  }
  if (!b->actor || !b->actor_t || !b->critic || !b->critic_t || !b->m_actor || !b->v_actor || !b->m_critic ||
      !b->v_critic || !b->grad_actor || !b->grad_critic || !b->adam_steps || !b->rng_counter || !b->rs ||
      !b->ra || !b->rr || !b->rs2 || !b->rd ||
      (ad.bf16 && (!b->actor_bf16 || !b->actor_t_bf16 || !b->critic_bf16 || !b->critic_t_bf16))) {
    set_error("spikerl_td3_update: null buffer");
    return SPIKERL_E_ARG;
  }
  SPK_TRY(critic_supported(cd, b->amp != nullptr));
  if (comm && (b->fused_critic || b->fused_actor)) {
    if (b->amp) { set_error("fused allreduce + Adam: no dynamic loss scaling"); return SPIKERL_E_UNSUPPORTED; }
    if ((b->fused_critic && !fused_adam_matches(b->fused_critic, b->grad_critic, b->critic, 2 * cd.off[SPIKERL_CRITIC_NPARAM])) ||
        (b->fused_actor && !fused_adam_matches(b->fused_actor, b->grad_actor, b->actor, ad.off[SPIKERL_ACTOR_NPARAM]))) {
      set_error("fused allreduce + Adam plan does not cover this buffer set (grads / params / size)");
      return SPIKERL_E_ARG;
    }
  }
  if (b->replay_size < B) {
    set_error("replay holds %lld < batch %d transitions", b->replay_size, B);
    return SPIKERL_E_NOTREADY;
  }
  LaunchPriority lp_hi(td3_priority(B));   // critical chain raised, branch B at the default
  cudaStream_t st = (cudaStream_t)stream;
  const Td3Ws W = td3_ws_layout(ad, cd, B);
  char* ws = (char*)workspace;
  float* s = (float*)(ws + W.s); float* a = (float*)(ws + W.a); float* r = (float*)(ws + W.r);
  float* s2 = (float*)(ws + W.s2); float* dn = (float*)(ws + W.d); float* a2 = (float*)(ws + W.a2);
  float* at = (float*)(ws + W.at); float* api = (float*)(ws + W.api); float* qt = (float*)(ws + W.qt);
  float* q = (float*)(ws + W.q); float* y = (float*)(ws + W.y); float* ga = (float*)(ws + W.ga);
  char* tape = ws + W.tape;
  char* aws = ws + W.actor_ws;
  void* cws = ws + W.critic_ws;
  const int rank = spikerl_comm_rank(comm);
  const size_t Pa = ad.off[SPIKERL_ACTOR_NPARAM];
  const size_t Pc = cd.off[SPIKERL_CRITIC_NPARAM];
  const __nv_bfloat16* abf = (const __nv_bfloat16*)b->actor_bf16;
  const __nv_bfloat16* atbf = (const __nv_bfloat16*)b->actor_t_bf16;
  const __nv_bfloat16* cbf = (const __nv_bfloat16*)b->critic_bf16;
  const __nv_bfloat16* ctbf = (const __nv_bfloat16*)b->critic_t_bf16;

  AuxPool* aux = nullptr;
  SPK_TRY(aux_pool(&aux));
  cudaStream_t sA = aux->side[0], sB = aux->side[1];
  static const bool serial = [] { const char* e = getenv("SPIKERL_TD3_SERIAL"); return e && e[0] == '1'; }();
  if (serial) sA = sB = st;   // A/B switch: the same work on one stream
  const bool actor_step = (step % hp->policy_delay == 0);
  void* cws_t = ws + W.critic_ws_t;

  // K9: sample (s, a, r, s', d)
  unsigned long long* ctr_snap = (unsigned long long*)(ws + W.ctr);
  {
    GatherSlots gs{};
    gs.n = 1;
    gs.s[0] = s; gs.a[0] = a; gs.r[0] = r; gs.s2[0] = s2; gs.d[0] = dn; gs.snap[0] = ctr_snap; gs.idx[0] = indices;
    SPK_TRY(launch_replay_gather(B, ad.S, ad.A, b->rs, b->ra, b->rr, b->rs2, b->rd, b->replay_size, seed, rank,
                                 b->rng_counter, gs, st));
  }
  // branch A: target path. 1. a~ = clip(pi'(s') + clip(eps), -1, 1) (smoothing in the target actor's decoder
  // launch); 2. Q1', Q2'(s', a~) (y = r + gamma (1 - d) min(Q1', Q2') is formed where the loss reads it)
  SPK_TRY(stream_after(sA, st, aux->ev[0]));
  {
    const TargetSmooth ts{noise, hp->policy_noise, hp->noise_clip, seed, rank, b->rng_counter, ctr_snap, at, 1};
    char* tape_t = aws + actor_ws_layout(ad, B).tape;
    const bool dec_c = target_decode_ok(cd, ad, B, b, comm);   // decoder + smoothing inside the target critics' launch
    SPK_TRY(actor_forward_impl(ad, B, b->actor_t, atbf, s2, a2, tape_t, sA, &ts, true, dec_c));
    const CriticDecode cdec = target_decode(ad, B, b->actor_t, tape_t, a2, ts);
    SPK_TRY(critic_fwd_bwd(cd, B, b->critic_t, ctbf, s2, ad.S, at, ad.A, nullptr, qt, nullptr, nullptr, nullptr, 0.f,
                           2, cws_t, sA, nullptr, nullptr, dec_c ? &cdec : nullptr));
  }
  SPK_CHECK_CUDA(cudaEventRecord(aux->ev[1], sA));
  // branch B (actor steps): the policy's own forward pi(s) depends only on s and the actor
  if (actor_step) {
    SPK_TRY(stream_after(sB, st, aux->ev[2]));
    LaunchPriority lp(0);
    SPK_TRY(actor_forward_impl(ad, B, b->actor, abf, s, api, tape, sB));
    SPK_CHECK_CUDA(cudaEventRecord(aux->ev[3], sB));
  }
  // 3. critic forward Q(s, a) overlaps branch A; the loss waits for Q'; grads, allreduce, Adam
  // (the bf16 working copies are kept current by the optimiser kernels themselves: Bf16Views)
  const Bf16Views cv = td3_critic_views(cd, ad, b->critic_bf16, false);
  const Bf16Views ctv = td3_critic_views(cd, ad, b->critic_t_bf16, true);
  const Bf16Views av = actor_bf16_views(ad, ad.bf16 ? (__nv_bfloat16*)b->actor_bf16 : nullptr);
  const Bf16Views atv = actor_bf16_views(ad, ad.bf16 ? (__nv_bfloat16*)b->actor_t_bf16 : nullptr);
  float* const amp_c = b->amp, * const amp_a = b->amp ? b->amp + 4 : nullptr;   // loss scaling (or none)
  const TdY tdy{nullptr, r, dn, qt, hp->gamma, B, y};   // y = r + gamma (1 - d) min Q' formed inside the loss
  // actor steps: the critic targets' soft update rides on the critic's Adam launch
  const PolyakFuse cpol{b->critic_t, hp->tau, &ctv};
  if (critic_update_fusable(cd, B, b, comm)) {
    SPK_CHECK_CUDA(cudaStreamWaitEvent(st, aux->ev[1], 0));   // Q' from branch A
    SPK_TRY(critic_update_fused(cd, B, b->critic, cbf, s, ad.S, a, ad.A, tdy, q, losses, b->grad_critic, cws,
                                b->m_critic, b->v_critic, b->adam_steps, hp->lr_critic, hp->beta1, hp->beta2, hp->eps,
                                &cv, actor_step ? &cpol : nullptr, st));
  } else {
    SPK_TRY(critic_fwd_bwd(cd, B, b->critic, cbf, s, ad.S, a, ad.A, &tdy, q, losses, b->grad_critic, nullptr, 0.f, 2,
                           cws, st, aux->ev[1], amp_c));
    SPK_TRY(critic_optimise(b, comm, hp, cd, Pc, &cv, amp_c, st, actor_step ? &cpol : nullptr));
  }
  // 4. delayed actor update + targets
  if (actor_step) {
    SPK_CHECK_CUDA(cudaStreamWaitEvent(st, aux->ev[3], 0));   // pi(s) from branch B
    // actor loss -mean Q1(s, pi(s)): formed by the mma critic's data-backward launch itself
    const bool mma = critic_mma_ok(cd);
    if (!amp_a && critic_act_fused_ok(cd, B))
      SPK_TRY(critic_actor_fused(cd, B, b->critic, cbf, s, ad.S, api, ad.A, q, losses + 1, ga, -1.0f / (float)B, cws,
                                 (unsigned int*)(b->adam_steps + 3) + 1, st));
    else
      SPK_TRY(critic_fwd_bwd(cd, B, b->critic, cbf, s, ad.S, api, ad.A, nullptr, q, mma ? losses + 1 : nullptr, nullptr,
                             ga, -1.0f / (float)B, 1, cws, st, nullptr, amp_a));
    if (!mma) {
      pdl(neg_mean_kernel, 1, 256, 0, st)(B, q, losses + 1);
      SPK_LAUNCHED();
    }
    SPK_TRY(actor_backward_impl(ad, B, b->actor, abf, s, tape, ga, b->grad_actor, 0, aws, st,
                                b->fused_actor ? nullptr : comm));
    const PolyakFuse apol{b->actor_t, hp->tau, &atv};
    SPK_TRY(actor_optimise(b, comm, hp, ad, Pa, &av, amp_a, st, &apol));
  }
  return SPIKERL_OK;
}

// Two consecutive updates k (critic only) and k + 1 (critic + actor + targets) with policy_delay 2,
// enqueued as one fork/join DAG. Update k + 1's target path (pi'(s'), smoothing, Q'(s', a~), y) and
// its pi(s) forward read only the targets and the actor, which update k does not change, so they run
// concurrently with update k instead of after it; every kernel and operand is the one the two
// sequential calls use, so the result is bitwise the same (tested). Workspace: two update
// workspaces back to back (spikerl_td3_pair_workspace_bytes).
int spikerl_td3_update_pair(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg, const spikerl_td3_cfg* hp,
                            const spikerl_td3_bufs* b, long long step, unsigned long long seed,
                            const long long* indices, const float* noise, spikerl_comm* comm, float* losses,
                            void* workspace, spikerl_stream_t stream) {
  ActorDims ad;
  CriticDims cd;
  SPK_TRY(actor_dims(acfg, &ad));
  SPK_TRY(critic_dims(ccfg, &cd));
  if (!hp || !b || !workspace || !losses || step < 1) {
    set_error("spikerl_td3_update_pair: bad arguments");
    return SPIKERL_E_ARG;
  }
  if (hp->policy_delay != 2 || step % 2 != 1) {
    set_error("spikerl_td3_update_pair: needs policy_delay 2 and an odd first step (got %d, %lld)", hp->policy_delay,
              step);
    return SPIKERL_E_ARG;
  }
  const int B = hp->batch;
  if (B < 1 || cd.in != ad.S + ad.A || cd.bf16 != ad.bf16) {
    set_error("spikerl_td3_update_pair: inconsistent configs");
    return SPIKERL_E_ARG;
  }
  if (!b->actor || !b->actor_t || !b->critic || !b->critic_t || !b->m_actor || !b->v_actor || !b->m_critic ||
      !b->v_critic || !b->grad_actor || !b->grad_critic || !b->adam_steps || !b->rng_counter || !b->rs ||
      !b->ra || !b->rr || !b->rs2 || !b->rd ||
      (ad.bf16 && (!b->actor_bf16 || !b->actor_t_bf16 || !b->critic_bf16 || !b->critic_t_bf16))) {
    set_error("spikerl_td3_update_pair: null buffer");
    return SPIKERL_E_ARG;
  }
  SPK_TRY(critic_supported(cd, b->amp != nullptr));
  if (comm && (b->fused_critic || b->fused_actor)) {
    if (b->amp) { set_error("fused allreduce + Adam: no dynamic loss scaling"); return SPIKERL_E_UNSUPPORTED; }
    if ((b->fused_critic && !fused_adam_matches(b->fused_critic, b->grad_critic, b->critic, 2 * cd.off[SPIKERL_CRITIC_NPARAM])) ||
        (b->fused_actor && !fused_adam_matches(b->fused_actor, b->grad_actor, b->actor, ad.off[SPIKERL_ACTOR_NPARAM]))) {
      set_error("fused allreduce + Adam plan does not cover this buffer set (grads / params / size)");
      return SPIKERL_E_ARG;
    }
  }
  if (b->replay_size < B) {
    set_error("replay holds %lld < batch %d transitions", b->replay_size, B);
    return SPIKERL_E_NOTREADY;
  }
  // scheduling (latency regime, B < 1024): update k's target path and the critic / actor chain at a
  // raised launch priority, the branches needed later (A1, B) at the default, so their CTAs fill in
  // instead of competing. A/B r02: configs[1] -1 %, configs[2] -2.2 %, but configs[3] B = 4096 +3.5 %
  // (there the late branches are long enough to become critical), hence the batch bound.
  // SPIKERL_TD3_PRIO=<n>: priority -n at any batch (0: off).
  LaunchPriority lp_hi(td3_priority(hp->batch));
  cudaStream_t st = (cudaStream_t)stream;
  const Td3Ws W = td3_ws_layout(ad, cd, B);
  struct Slot {
    float *s, *a, *r, *s2, *dn, *a2, *at, *api, *qt, *q, *y, *ga;
    char *tape, *aws;
    void *cws, *cws_t;
    unsigned long long* snap;
  } sl[2];
  for (int i = 0; i < 2; ++i) {
    char* ws = (char*)workspace + (size_t)i * W.total;
    Slot& x = sl[i];
    x.s = (float*)(ws + W.s); x.a = (float*)(ws + W.a); x.r = (float*)(ws + W.r); x.s2 = (float*)(ws + W.s2);
    x.dn = (float*)(ws + W.d); x.a2 = (float*)(ws + W.a2); x.at = (float*)(ws + W.at); x.api = (float*)(ws + W.api);
    x.qt = (float*)(ws + W.qt); x.q = (float*)(ws + W.q); x.y = (float*)(ws + W.y); x.ga = (float*)(ws + W.ga);
    x.tape = ws + W.tape; x.aws = ws + W.actor_ws; x.cws = ws + W.critic_ws; x.cws_t = ws + W.critic_ws_t;
    x.snap = (unsigned long long*)(ws + W.ctr);
  }
  const int rank = spikerl_comm_rank(comm);
  const size_t Pa = ad.off[SPIKERL_ACTOR_NPARAM];
  const size_t Pc = cd.off[SPIKERL_CRITIC_NPARAM];
  const __nv_bfloat16* abf = (const __nv_bfloat16*)b->actor_bf16;
  const __nv_bfloat16* atbf = (const __nv_bfloat16*)b->actor_t_bf16;
  const __nv_bfloat16* cbf = (const __nv_bfloat16*)b->critic_bf16;
  const __nv_bfloat16* ctbf = (const __nv_bfloat16*)b->critic_t_bf16;
  AuxPool* aux = nullptr;
  SPK_TRY(aux_pool(&aux));
  cudaStream_t sA[2] = {aux->side[0], aux->side[7]}, sB = aux->side[1];
  static const bool serial = [] { const char* e = getenv("SPIKERL_TD3_SERIAL"); return e && e[0] == '1'; }();
  if (serial) sA[0] = sA[1] = sB = st;   // A/B switch: the same work on one stream
  cudaEvent_t evA[2] = {aux->ev[1], aux->ev[7]};
  // sample both minibatches in one launch (update k + 1 draws with the counter value update k
  // advances to)
  {
    GatherSlots gs{};
    gs.n = 2;
    for (int i = 0; i < 2; ++i) {
      gs.s[i] = sl[i].s; gs.a[i] = sl[i].a; gs.r[i] = sl[i].r; gs.s2[i] = sl[i].s2; gs.d[i] = sl[i].dn;
      gs.snap[i] = sl[i].snap; gs.idx[i] = indices ? indices + (size_t)i * B : nullptr;
    }
    SPK_TRY(launch_replay_gather(B, ad.S, ad.A, b->rs, b->ra, b->rr, b->rs2, b->rd, b->replay_size, seed, rank,
                                 b->rng_counter, gs, st));
  }
  // target paths of both updates, concurrently (branches A0, A1); only the second advances the counter
  for (int i = 0; i < 2; ++i) {
    const Slot& x = sl[i];
    LaunchPriority lp(i == 1 ? 0 : launch_priority());   // A1 (needed one critic update later): default
    SPK_TRY(stream_after(sA[i], st, aux->ev[i == 0 ? 0 : 6]));
    const TargetSmooth ts{noise ? noise + (size_t)i * B * ad.A : nullptr, hp->policy_noise, hp->noise_clip, seed,
                          rank, b->rng_counter, x.snap, x.at, i == 1 ? 1 : 0};
    char* tape_t = x.aws + actor_ws_layout(ad, B).tape;
    const bool dec_c = target_decode_ok(cd, ad, B, b, comm);   // decoder + smoothing inside the target critics' launch
    SPK_TRY(actor_forward_impl(ad, B, b->actor_t, atbf, x.s2, x.a2, tape_t, sA[i], &ts, true, dec_c));
    const CriticDecode cdec = target_decode(ad, B, b->actor_t, tape_t, x.a2, ts);
    SPK_TRY(critic_fwd_bwd(cd, B, b->critic_t, ctbf, x.s2, ad.S, x.at, ad.A, nullptr, x.qt, nullptr, nullptr, nullptr,
                           0.f, 2, x.cws_t, sA[i], nullptr, nullptr, dec_c ? &cdec : nullptr));
    SPK_CHECK_CUDA(cudaEventRecord(evA[i], sA[i]));
  }
  // branch B: pi(s) of update k + 1 (the actor is unchanged by update k)
  SPK_TRY(stream_after(sB, st, aux->ev[2]));
  {
    LaunchPriority lp(0);
    SPK_TRY(actor_forward_impl(ad, B, b->actor, abf, sl[1].s, sl[1].api, sl[1].tape, sB));
  }
  SPK_CHECK_CUDA(cudaEventRecord(aux->ev[3], sB));
  const Bf16Views cv = td3_critic_views(cd, ad, b->critic_bf16, false);
  const Bf16Views ctv = td3_critic_views(cd, ad, b->critic_t_bf16, true);
  const Bf16Views av = actor_bf16_views(ad, ad.bf16 ? (__nv_bfloat16*)b->actor_bf16 : nullptr);
  const Bf16Views atv = actor_bf16_views(ad, ad.bf16 ? (__nv_bfloat16*)b->actor_t_bf16 : nullptr);
  float* const amp_c = b->amp, * const amp_a = b->amp ? b->amp + 4 : nullptr;   // loss scaling (or none)
  // the two critic updates, in order
  const PolyakFuse cpol{b->critic_t, hp->tau, &ctv};
  const bool fuse_c = critic_update_fusable(cd, B, b, comm);
  for (int i = 0; i < 2; ++i) {
    const Slot& x = sl[i];
    const TdY tdy{nullptr, x.r, x.dn, x.qt, hp->gamma, B, x.y};
    if (fuse_c) {
      SPK_CHECK_CUDA(cudaStreamWaitEvent(st, evA[i], 0));
      SPK_TRY(critic_update_fused(cd, B, b->critic, cbf, x.s, ad.S, x.a, ad.A, tdy, x.q, losses, b->grad_critic, x.cws,
                                  b->m_critic, b->v_critic, b->adam_steps, hp->lr_critic, hp->beta1, hp->beta2,
                                  hp->eps, &cv, i == 1 ? &cpol : nullptr, st));
      continue;
    }
    SPK_TRY(critic_fwd_bwd(cd, B, b->critic, cbf, x.s, ad.S, x.a, ad.A, &tdy, x.q, losses, b->grad_critic, nullptr,
                           0.f, 2, x.cws, st, evA[i], amp_c));
    SPK_TRY(critic_optimise(b, comm, hp, cd, Pc, &cv, amp_c, st, i == 1 ? &cpol : nullptr));
  }
  // delayed actor update + targets (update k + 1), exactly as spikerl_td3_update's actor step
  const Slot& x = sl[1];
  SPK_CHECK_CUDA(cudaStreamWaitEvent(st, aux->ev[3], 0));
  const bool mma = critic_mma_ok(cd);
  if (!amp_a && critic_act_fused_ok(cd, B))
    SPK_TRY(critic_actor_fused(cd, B, b->critic, cbf, x.s, ad.S, x.api, ad.A, x.q, losses + 1, x.ga, -1.0f / (float)B,
                               x.cws, (unsigned int*)(b->adam_steps + 3) + 1, st));
  else
    SPK_TRY(critic_fwd_bwd(cd, B, b->critic, cbf, x.s, ad.S, x.api, ad.A, nullptr, x.q, mma ? losses + 1 : nullptr,
                           nullptr, x.ga, -1.0f / (float)B, 1, x.cws, st, nullptr, amp_a));
  if (!mma) {
    pdl(neg_mean_kernel, 1, 256, 0, st)(B, x.q, losses + 1);
    SPK_LAUNCHED();
  }
  SPK_TRY(actor_backward_impl(ad, B, b->actor, abf, x.s, x.tape, x.ga, b->grad_actor, 0, x.aws, st,
                              b->fused_actor ? nullptr : comm));
  const PolyakFuse apol{b->actor_t, hp->tau, &atv};
  SPK_TRY(actor_optimise(b, comm, hp, ad, Pa, &av, amp_a, st, &apol));
  return SPIKERL_OK;
}

int spikerl_td3_workspace_layout(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg, int batch,
                                 spikerl_td3_ws_layout* out) {
  ActorDims ad;
  CriticDims cd;
  SPK_TRY(actor_dims(acfg, &ad));
  SPK_TRY(critic_dims(ccfg, &cd));
  if (!out || batch < 1) { set_error("spikerl_td3_workspace_layout: bad arguments"); return SPIKERL_E_ARG; }
  const Td3Ws W = td3_ws_layout(ad, cd, batch);
  out->s = W.s; out->a = W.a; out->r = W.r; out->s2 = W.s2; out->d = W.d; out->a2 = W.a2; out->at = W.at;
  out->api = W.api; out->y = W.y; out->ga = W.ga; out->tape_pi = W.tape;
  out->tape_target = W.actor_ws + actor_ws_layout(ad, batch).tape;
  out->total = W.total;
  return SPIKERL_OK;
}

size_t spikerl_td3_pair_workspace_bytes(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg, int batch) {
  return 2 * spikerl_td3_workspace_bytes(acfg, ccfg, batch);
}

}  // extern "C"
