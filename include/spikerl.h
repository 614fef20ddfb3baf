/*
 * spikerl.h — C ABI of libspikerl.so: the B200-native (sm_100a) data-parallel hot path of
 * SpikeRL (arxiv 2502.17496): the batched forward and surrogate-gradient backward of the
 * population-coded spiking actor inside a TD3 update, the twin-critic MLP, Adam/Polyak and
 * the per-step gradient allreduce.
 *
 * Sources of each operation (PAPER.md line numbers; DESIGN.md "Readings" R1..R30 cover every
 * point the paper leaves open):
 *   encoder   PAPER.md:129-131 (§III-A, "populations use Gaussian distributions to transform
 *             continuous input values into spike trains"), north_star ("deterministic
 *             soft-reset encoder spikes").
 *   LIF       PAPER.md:131 ("integrates presynaptic spikes into a current, which then charges
 *             the membrane voltage ... the neuron fires"); north_star equations
 *             c = d_c*c + W*o, v = d_v*v*(1-o_prev) + c, o = [v > V_th].
 *   decoder   PAPER.md:131 ("aggregates these spikes over time to compute firing rates ...
 *             through a weighted sum").
 *   backward  north_star ("BPTT with a rectangular pseudo-gradient").
 *   critic    PAPER.md:131 ("evaluated by the deep critic network ... TD3"); configs[1].
 *   TD3       PAPER.md:131; SPEC.md:235-259 (target, train_step, soft_update).
 *   comm      PAPER.md:135 (broadcast_weights / average_gradients), PAPER.md:144 (DDP
 *             allreduce over NCCL).
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless marked (host).
 *   - Every call only enqueues work on `stream` (a cudaStream_t) and returns; no call
 *     synchronises the device, so the calls are CUDA-graph capturable (except comm init).
 *   - The caller owns every buffer (params, grads, tape, workspace, replay). The library frees
 *     nothing it did not allocate; it owns only spikerl_comm objects and internal caches.
 *   - Synchronous errors (SPIKERL_E_ARG, _DOMAIN, _STATE, _NOTREADY) are detected on the host
 *     before anything is enqueued, so outputs are untouched. Asynchronous device faults show
 *     up as SPIKERL_E_CUDA at the next call. spikerl_last_error() gives the message.
 *   - Data-dependent preconditions (sigma > 0, finite observations) are documented, not
 *     checked on the device.
 */
#ifndef SPIKERL_H
#define SPIKERL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* spikerl_stream_t; /* a cudaStream_t (NULL = legacy default stream) */

enum spikerl_status {
  SPIKERL_OK = 0,
  SPIKERL_E_ARG = 1,         /* null pointer, batch < 1, size/shape mismatch                  */
  SPIKERL_E_DOMAIN = 2,      /* T<1 or T>255, d_c/d_v outside [0,1], v_th<=0, window<=0, pop<1 */
  SPIKERL_E_STATE = 3,       /* tape header does not match (cfg hash, batch) */
  SPIKERL_E_NOTREADY = 4,    /* replay size < batch: nothing enqueued */
  SPIKERL_E_CUDA = 5,
  SPIKERL_E_NCCL = 6,
  SPIKERL_E_UNSUPPORTED = 7  /* configuration outside what a kernel supports                 */
};

enum spikerl_precision {
  SPIKERL_FP32 = 0,          /* true fp32 (no TF32) SIMT path; configs[0]                      */
  SPIKERL_BF16 = 1,          /* bf16 operands, fp32 accumulate, fp32 master */
  SPIKERL_FP16 = 2           /* actor only, tcgen05 engine: fp16 operands ("FP16 (half
                                precision)" AMP), fp32 accumulate, fp32 master; pair it with dynamic
                                loss scaling (spikerl_td3_bufs.amp). The 16-bit working copy has the
                                bf16 copy's layout and size. */
};

enum spikerl_engine {
  SPIKERL_ENGINE_AUTO = 0,   /* bf16/fp16 -> tcgen05 tensor-core GEMMs; fp32 -> SIMT. Never
                                switches engine silently: a bf16 shape tcgen05 cannot tile (odd
                                T > 16, T > 32) is SPIKERL_E_UNSUPPORTED (north_star: no
                                multi-backend dispatch)                                        */
  SPIKERL_ENGINE_SIMT = 1,   /* plain SIMT kernels (fp32 FFMA), fp32 or bf16 operands; only when
                                asked for                                                       */
  SPIKERL_ENGINE_TCGEN05 = 2 /* tcgen05 (bf16/fp16 only)                                       */
};

/* Opaque NCCL communicator owned by the library (spikerl_comm_init / spikerl_comm_destroy). */
struct spikerl_comm;
typedef struct spikerl_comm spikerl_comm;
/* Opaque fused gradient-mean + Adam plan over symmetric memory (spikerl_fused_adam_create). */
struct spikerl_fused_adam;
typedef struct spikerl_fused_adam spikerl_fused_adam;

/* Actor problem statement (PAPER.md:131 + north_star): obs dim S, action dim A, encoder
 * population E, decoder population D, hidden widths N1, N2, T timesteps, LIF constants. */
typedef struct {
  int obs_dim, act_dim, pop_enc, pop_dec; /* S, A, E, D; K0 = S*E inputs, N3 = A*D outputs    */
  int hidden1, hidden2;                   /* N1, N2                                           */
  int T;                                  /* timesteps, 1..255                                */
  float d_c, d_v, v_th;                   /* LIF constants (0.5, 0.75, 0.5)                   */
  float surr_window, surr_height;         /* h(v) = height*[|v-v_th| < window] (0.5, 1.0)     */
  float sigma_floor;                      /* sigma clamp after the actor Adam step (1e-3)     */
  int precision;                          /* enum spikerl_precision                           */
  int engine;                             /* enum spikerl_engine                              */
  int reset_grad;                         /* rho: 0 = reset gate (1 - o_{t-1}) detached in BPTT
                                             (default); 1 = differentiated through it:
                                             delta_v_t = h_t (g_t - d_v v_t delta_v_{t+1}) +
                                             d_v (1 - o_t) delta_v_{t+1} (needs fp32 v_t in the tape) */
} spikerl_actor_cfg;

/* Twin critic Q_i(s,a) = W3 relu(W2 relu(W1 [s;a] + b1) + b2) + b3 (configs[1]). */
typedef struct {
  int in_dim;                             /* S + A                                            */
  int hidden1, hidden2;                   /* 256, 256                                         */
  int precision;                          /* enum spikerl_precision                           */
} spikerl_critic_cfg;

typedef struct {
  float gamma, tau, policy_noise, noise_clip; /* 0.99, 0.005, 0.2, 0.5                        */
  int policy_delay;                           /* 2                                            */
  float lr_actor, lr_critic, beta1, beta2, eps; /* 1e-4, 1e-3, 0.9, 0.999, 1e-8             */
  int batch;                                  /* per-rank batch B                             */
  /* dynamic loss scaling (PAPER.md:164-167 GradScaler; used when bufs->amp != NULL):
   * scale *= amp_growth after amp_interval consecutive finite steps, *= amp_backoff on overflow */
  float amp_growth, amp_backoff;              /* 2.0, 0.5                                      */
  int amp_interval;                           /* 2000                                          */
} spikerl_td3_cfg;

/* ------------------------------------------------------------------------------------------
 * Sizes and layouts (host-only calls, no device work).
 * Actor flat fp32 parameter layout (also used for grads and Adam m, v), element offsets:
 *   mu[S][E] | sigma[S][E] | W1[N1][K0] | W2[N2][N1] | W3[N3][N2] | Wd[A][D] | bd[A]
 * Critic flat fp32 layout (one critic; twins are [2][P]):
 *   W1[H1][in] | b1[H1] | W2[H2][H1] | b2[H2] | W3[H2] | b3[1]
 * ---------------------------------------------------------------------------------------- */
enum { SPIKERL_ACTOR_MU = 0, SPIKERL_ACTOR_SIGMA, SPIKERL_ACTOR_W1, SPIKERL_ACTOR_W2,
       SPIKERL_ACTOR_W3, SPIKERL_ACTOR_WD, SPIKERL_ACTOR_BD, SPIKERL_ACTOR_NPARAM };
enum { SPIKERL_CRITIC_W1 = 0, SPIKERL_CRITIC_B1, SPIKERL_CRITIC_W2, SPIKERL_CRITIC_B2,
       SPIKERL_CRITIC_W3, SPIKERL_CRITIC_B3, SPIKERL_CRITIC_NPARAM };

/* Validate a cfg (returns a status, no side effects besides spikerl_last_error). */
int spikerl_actor_cfg_check(const spikerl_actor_cfg* cfg);
/* offsets (host, [SPIKERL_ACTOR_NPARAM+1] elements; last = total count). */
int spikerl_actor_param_offsets(const spikerl_actor_cfg* cfg, size_t* offsets /* host */);
size_t spikerl_actor_param_count(const spikerl_actor_cfg* cfg);
int spikerl_critic_param_offsets(const spikerl_critic_cfg* cfg, size_t* offsets /* host */);
size_t spikerl_critic_param_count(const spikerl_critic_cfg* cfg);
/* bf16 working copies (opaque, zero-padded tensor-core layout); produced by *_refresh_bf16. */
size_t spikerl_actor_bf16_bytes(const spikerl_actor_cfg* cfg);
size_t spikerl_critic_bf16_bytes(const spikerl_critic_cfg* cfg); /* twin pair: [2][P] + W1^T, W2^T each */
/* Element offsets of the tensor-core critic's bf16 twin buffer (bf16, hidden 256-256, in_dim <= 512):
 * out[0] first per-critic block (after the [2][P] plain copy), out[1] block stride, then within a
 * block out[2] W1p [H1][inp] (rows zero padded to inp = out[6]), out[3] W1T [inq][H1], out[4] W2T
 * [H1][H2], out[5] W2 [H2][H1], out[6] inp, out[7] inq. TD3 updates keep the whole buffer current
 * except the transposed blocks nothing reads: the targets' W1T / W2T, and the online critics' W1T
 * rows outside the action columns [S, S+A) (spikerl_td3_update). E_UNSUPPORTED for other critics. */
int spikerl_critic_bf16_layout(const spikerl_critic_cfg* cfg, long long* out8);
/* Device buffers the caller allocates for one forward(+backward) at `batch`. */
size_t spikerl_actor_tape_bytes(const spikerl_actor_cfg* cfg, int batch);
size_t spikerl_actor_workspace_bytes(const spikerl_actor_cfg* cfg, int batch);
/* Byte offset inside the actor workspace of the tape an inference-only forward (tape == NULL) writes:
 * its spike / window planes, counts and actions (not the stimulation plane A, which such a forward
 * does not compute; layout as spikerl_actor_tape_layout). For tests and diagnostics. */
size_t spikerl_actor_workspace_tape_offset(const spikerl_actor_cfg* cfg, int batch);
size_t spikerl_critic_workspace_bytes(const spikerl_critic_cfg* cfg, int batch);
size_t spikerl_td3_workspace_bytes(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg,
                                   int batch);

/* Tape layout (byte offsets into the tape device buffer; all 256-byte aligned).
 * Spike / surrogate-mask bit planes are u32 words [T][B][P_l/32]: bit j of word w is neuron
 * 32w+j of layer l at (t, b); P_l = padded width (multiple of 128; pad bits are 0).
 *   A      fp32 [B][K0]        Gaussian stimulation (kept for the encoder gradient)
 *   bits0  u32  [T][B][P0/32]  encoder spikes
 *   bits_l u32  [T][B][Pl/32]  LIF spikes of layer l = 1, 2, 3
 *   mask_l u32  [T][B][Pl/32]  surrogate window bits [|v - v_th| < window], layer l = 1..3
 *   counts u8   [B][N3]        output spike counts
 *   act    fp32 [B][A]         decoded actions (for the decoder backward)
 *   bitsT_l, maskT_l u8 [ceil32(B)/4][P_l][tpad/2]  (tcgen05 engine, l = 1, 2; else offset 0)
 *                              quad-major copies of the hidden planes: one little-endian u64 per
 *                              16 steps, bit 4 (t mod 16) + j of word (q, n, t / 16) is batch row
 *                              4q + j at step t (read by the fused dX epilogue) */
typedef struct {
  size_t A, bits[4], mask[4], counts, act, total;
  int padded[4];           /* P0..P3                                                        */
  size_t bitsT[4], maskT[4];
  int tpad;                /* T rounded up to 16                                            */
  size_t V[4];             /* reset_grad = 1: membrane potentials fp32 [T][B][P_l], l = 1..3 (else 0) */
} spikerl_tape_layout;
int spikerl_actor_tape_layout(const spikerl_actor_cfg* cfg, int batch, spikerl_tape_layout* out);

/* Tape = HOST descriptor + caller-owned DEVICE buffer. forward() stamps magic/cfg_hash/batch
 * on the host so backward() validates without a device->host copy. */
typedef struct {
  unsigned long long magic, cfg_hash;
  int batch;
  void* dev;               /* device buffer of spikerl_actor_tape_bytes(cfg, batch)          */
  size_t bytes;
} spikerl_tape;

/* ------------------------------------------------------------------------------------------
 * Compute entry points
 * ---------------------------------------------------------------------------------------- */

/* Refresh the bf16 working copy from the fp32 master (RNE; PAPER.md:153-174 master weights). */
int spikerl_actor_refresh_bf16(const spikerl_actor_cfg* cfg, const float* params,
                               void* params_bf16, spikerl_stream_t stream);
int spikerl_critic_refresh_bf16(const spikerl_critic_cfg* cfg, int n_critics, const float* params,
                                void* params_bf16, spikerl_stream_t stream);

/* Actor forward: obs [B][S] fp32 -> actions [B][A] fp32 (tanh, bound 1).
 * params: flat fp32 (layout above); params_bf16: working copy (required iff precision=BF16).
 * tape: host descriptor whose .dev/.bytes the caller set (NULL = inference only: the spike
 * planes go to `workspace`, the encoder's stimulation plane A is not formed and the exact A is
 * computed only where a spike is possible; spikes and actions are bitwise those of a recording
 * forward). workspace: spikerl_actor_workspace_bytes(cfg, batch). */
int spikerl_actor_forward(const spikerl_actor_cfg* cfg, int batch, const float* params,
                          const void* params_bf16, const float* obs, float* actions,
                          spikerl_tape* tape, void* workspace, spikerl_stream_t stream);

/* Actor backward (surrogate-gradient BPTT, reset gate detached).
 * grad_actions [B][A] = dL/da. grad_params: flat fp32, overwritten (accumulate=0) or added to
 * (accumulate=1). The tape must come from spikerl_actor_forward with the same cfg and batch
 * (else SPIKERL_E_STATE). */
int spikerl_actor_backward(const spikerl_actor_cfg* cfg, int batch, const float* params,
                           const void* params_bf16, const float* obs, const spikerl_tape* tape,
                           const float* grad_actions, float* grad_params, int accumulate,
                           void* workspace, spikerl_stream_t stream);

/* Actor backward fused with the data-parallel gradient mean (PAPER.md:135 average_gradients,
 * PAPER.md:144 DDP "gradient synchronization ... during backpropagation"): as
 * spikerl_actor_backward, and grad_params ends as the mean over the ranks of comm. The mean runs
 * per bucket (spikerl_actor_grad_buckets, completion order: W3|Wd|bd, W2, mu|sigma|W1) on the
 * library's comm stream as soon as the bucket is computed, overlapping the rest of the backward;
 * `stream` waits for the last bucket before the call's work ends (graph-capturable). comm == NULL:
 * exactly spikerl_actor_backward. Every rank must make the same calls in the same order. */
int spikerl_actor_backward_dp(const spikerl_actor_cfg* cfg, int batch, const float* params,
                              const void* params_bf16, const float* obs, const spikerl_tape* tape,
                              const float* grad_actions, float* grad_params, int accumulate,
                              spikerl_comm* comm, void* workspace, spikerl_stream_t stream);
/* Bucket bounds of the flat actor gradient (host call): bounds[4] = {0, off W2, off W3, total};
 * buckets [bounds[i], bounds[i+1]). */
int spikerl_actor_grad_buckets(const spikerl_actor_cfg* cfg, size_t* bounds);

/* Twin critic forward (+ backward). x = [obs ; act] with obs_dim + act_dim == in_dim.
 * params2 [2][P] fp32 (+ bf16 copy iff precision=BF16). q [2][B] receives Q1, Q2.
 * If target_y [B] != NULL: loss (device scalar, may be NULL) = mean(Q1-y)^2 + mean(Q2-y)^2 and,
 * if grad_params2 != NULL, its gradient w.r.t. both critics (overwritten).
 * If grad_act [B][A] != NULL: grad_act = act_grad_scale * dQ1/da (per sample).
 * BF16 critics run on the tensor-core kernels, which need hidden widths 256-256 and in_dim <= 512
 * (configs[1..3]); other bf16 shapes are SPIKERL_E_UNSUPPORTED (checked before anything is
 * enqueued). FP32 critics run on SIMT GEMMs (any shape). */
int spikerl_critic_fwd_bwd(const spikerl_critic_cfg* cfg, int batch, const float* params2,
                           const void* params2_bf16, const float* obs, int obs_dim,
                           const float* act, int act_dim, const float* target_y, float* q,
                           float* loss, float* grad_params2, float* grad_act,
                           float act_grad_scale, void* workspace, spikerl_stream_t stream);

/* Adam (PyTorch form) over a flat fp32 buffer. step_counter: device int64[2] = {t, scratch};
 * t is read as the previous step count and incremented by the call; scratch must be zero
 * before the first call (the kernel restores it to zero). clamp_lo..clamp_hi (element range, may be empty) is clamped to
 * >= clamp_min after the update (actor sigma floor). */
int spikerl_adam(float* params, const float* grads, float* m, float* v, size_t n,
                 long long* step_counter, float lr, float beta1, float beta2, float eps,
                 size_t clamp_lo, size_t clamp_hi, float clamp_min, spikerl_stream_t stream);
/* Polyak: target <- tau*source + (1-tau)*target over n fp32 elements. */
int spikerl_polyak(float* target, const float* source, size_t n, float tau,
                   spikerl_stream_t stream);

/* Standalone forward LIF scan over precomputed input currents (north_star LIF equations;
 * SPEC.md:141-149; R7): an ablation / diagnostic kernel showing what the
 * fused FWD epilogue saves — the product path never materialises the currents. I [T][B][N] fp32
 * (device); bits / mask [T][B][ceil(N/32)] u32 (device, caller-owned): spike o_t and window
 * h_t = [|v_t - V_th| < window] planes, bit n % 32 of word n / 32. Errors: E_ARG on null / empty. */
int spikerl_lif_scan_forward(const float* I, int T, int B, int N, float d_c, float d_v, float v_th,
                             float window, uint32_t* bits, uint32_t* mask, spikerl_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * TD3 update (one step k). All buffers caller-owned.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  float *actor, *actor_t;          /* [Pa] fp32 master: online, target                        */
  void *actor_bf16, *actor_t_bf16; /* working copies (BF16 precision)                         */
  float *critic, *critic_t;        /* [2][Pc] fp32: online twins, target twins                */
  void *critic_bf16, *critic_t_bf16;
  float *m_actor, *v_actor;        /* Adam state [Pa]                                         */
  float *m_critic, *v_critic;      /* Adam state [2][Pc]                                      */
  float *grad_actor, *grad_critic; /* [Pa], [2][Pc]                                           */
  long long* adam_steps;           /* device [4]: {critic t, 0, actor t, 0} (zero-initialised)  */
  unsigned long long* rng_counter; /* device [1]: Philox counter, advanced every update       */
  const float *rs, *ra, *rr, *rs2, *rd; /* replay shard SoA: s[N][S] a[N][A] r[N] s2[N][S] d[N] */
  long long replay_size;           /* (host) N valid transitions                               */
  /* device [8] or NULL (no scaling): GradScaler state of the critic at [0..3] and of the actor at
   * [4..7] = {loss scale, finite steps since the last scale change, found_inf, unused}. The loss
   * gradient is multiplied by the scale; before each Adam step the gradient is checked for inf /
   * NaN: if any, the optimizer step is skipped (parameters, moments and its step count unchanged)
   * and the scale backs off; otherwise the gradient is unscaled inside the Adam kernel. The caller
   * initialises the scales (e.g. 65536) and zeroes the rest. */
  float* amp;
  /* optional (NULL = the NCCL allreduce + Adam launches): fused gradient mean + Adam plans
   * (spikerl_fused_adam_create over grad_critic / critic and grad_actor / actor, which must then come
   * from spikerl_comm_mem_alloc). Used only with a communicator and without loss scaling. */
  spikerl_fused_adam* fused_critic;
  spikerl_fused_adam* fused_actor;
} spikerl_td3_bufs;


/* One TD3 update. step = 1-based k; the actor and all targets are updated when
 * k % policy_delay == 0. indices [B] (device int64) / noise [B][A] (device fp32 raw eps, before
 * the clip to +-noise_clip) may be NULL: then they are drawn on the device with Philox
 * (seed, rank, *rng_counter). comm == NULL means one GPU (no allreduce). losses: device [2]
 * (critic loss; actor loss or unchanged on critic-only steps).
 * BF16: the four working copies must have been produced once by *_refresh_bf16 (which writes
 * their zero padding); the update then keeps them current itself — Adam and Polyak store the RNE
 * bf16 value of every element they change into each of its places in the copy — so no refresh
 * is needed between updates. */
int spikerl_td3_update(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg,
                       const spikerl_td3_cfg* hp, const spikerl_td3_bufs* bufs, long long step,
                       unsigned long long seed, const long long* indices, const float* noise,
                       spikerl_comm* comm, float* losses, void* workspace,
                       spikerl_stream_t stream);

/* Two consecutive updates k, k + 1 (k odd, policy_delay 2: a critic-only update then a critic +
 * actor + targets update) as one fork/join DAG: update k + 1's target path and its pi(s) forward
 * read only parameters update k leaves unchanged (the actor and the targets), so they overlap
 * update k. Bitwise the same result as spikerl_td3_update(k) followed by spikerl_td3_update(k + 1)
 * (SPEC.md:235-259 order; R15). indices [2][B] / noise [2][B][A] (device) or NULL;
 * workspace: spikerl_td3_pair_workspace_bytes. E_ARG unless policy_delay == 2 and k is odd. */
int spikerl_td3_update_pair(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg,
                            const spikerl_td3_cfg* hp, const spikerl_td3_bufs* bufs, long long step,
                            unsigned long long seed, const long long* indices, const float* noise,
                            spikerl_comm* comm, float* losses, void* workspace,
                            spikerl_stream_t stream);
size_t spikerl_td3_pair_workspace_bytes(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg,
                                        int batch);

/* Byte offsets, inside one update's workspace (the pair workspace holds two such blocks back to
 * back, update k then k + 1), of the intermediates a TD3 update leaves behind (read by the parity
 * tests' teacher-forced protocol; host call, no device work). After spikerl_td3_update(k):
 *   s, a, r, s2, d  fp32 the gathered minibatch ([B][S], [B][A], [B], [B][S], [B])
 *   a2   fp32 [B][A]  target-policy actions pi'(s');   at fp32 [B][A]  smoothed a~
 *   y    fp32 [B]     TD target;                        api fp32 [B][A]  pi(s) (actor steps)
 *   ga   fp32 [B][A]  -(1/B) dQ1/da at (s, pi(s)) (actor steps; times the actor loss scale)
 *   tape_pi, tape_target  tape buffers (spikerl_tape_layout) of the pi(s) / pi'(s') forwards
 * SPEC.md:235-252 (compute_target, train_step). */
typedef struct {
  size_t s, a, r, s2, d, a2, at, api, y, ga, tape_pi, tape_target, total;
} spikerl_td3_ws_layout;
int spikerl_td3_workspace_layout(const spikerl_actor_cfg* acfg, const spikerl_critic_cfg* ccfg, int batch,
                                 spikerl_td3_ws_layout* out);

/* Fill a replay shard on the device: s,s2 ~ N(0,1) clip +-5, a ~ U[-1,1], r ~ N(0,1),
 * done ~ Bernoulli(p_done) (configs[1]); Philox keyed by (seed, rank). */
int spikerl_replay_fill(float* s, float* a, float* r, float* s2, float* d, long long n, int obs_dim,
                        int act_dim, float p_done, unsigned long long seed, int rank,
                        spikerl_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * Data-parallel communication (NCCL 2.28, loaded at spikerl_comm_init). PyTorch supplies only
 * the rendezvous (broadcast of the 128-byte id).
 * ---------------------------------------------------------------------------------------- */
int spikerl_comm_get_unique_id(void* out128 /* host, 128 bytes */);
int spikerl_comm_init(int rank, int world, const void* id128 /* host */, spikerl_comm** out);
int spikerl_comm_destroy(spikerl_comm* comm);
int spikerl_comm_world(const spikerl_comm* comm);
int spikerl_comm_rank(const spikerl_comm* comm);
/* in place: grads <- mean over ranks (ncclAvg, fp32)  — PAPER.md:135 average_gradients.
 * comm == NULL: identity, nothing enqueued. A one-rank communicator still calls NCCL (identity
 * result), so the one-GPU path runs the same NCCL kernels, graph-capturable. */
int spikerl_allreduce_grads(spikerl_comm* comm, float* grads, size_t count,
                            spikerl_stream_t stream);
/* params <- params of `root`  — PAPER.md:135 broadcast_weights */
int spikerl_broadcast_params(spikerl_comm* comm, float* params, size_t count, int root,
                             spikerl_stream_t stream);

/* the gradient mean fused with the optimiser step over NVLink (PAPER.md:135
 * average_gradients + Adam) as one kernel on NCCL 2.28 symmetric memory:
 *   mem_alloc / mem_free: ncclMemAlloc'd device memory (the buffers a plan may use);
 *   fused_adam_create (collective over comm): registers grads and params (n fp32 each, from
 *     mem_alloc) as symmetric windows and creates the device communicator (LSA barriers; NVLS
 *     multimem when use_multimem and the fabric has it, else peer loads / stores);
 *   fused_allreduce_adam: ONE launch per rank: barrier, then for the rank's 1/W shard the mean over
 *     ranks of the peers' gradients (summed in rank order), Adam (PyTorch form, same element
 *     arithmetic as spikerl_adam) on the shard with the clamp, the new values stored into every
 *     rank's params, barrier. params end bitwise identical on all ranks; m and v are kept only for
 *     the rank's shard (ZeRO-1). At world 1 the result equals allreduce + spikerl_adam bitwise.
 * Errors: E_NCCL if the NCCL library has no device API; E_UNSUPPORTED above 8 ranks. */
int spikerl_comm_mem_alloc(spikerl_comm* comm, size_t bytes, void** ptr /* host out */);
int spikerl_comm_mem_free(spikerl_comm* comm, void* ptr);
int spikerl_fused_adam_create(spikerl_comm* comm, float* grads, float* params, size_t n, int use_multimem,
                              spikerl_fused_adam** out);
int spikerl_fused_adam_destroy(spikerl_fused_adam* plan);
int spikerl_fused_allreduce_adam(spikerl_fused_adam* plan, float* m, float* v, long long* step_counter, float lr,
                                 float beta1, float beta2, float eps, size_t clamp_lo, size_t clamp_hi,
                                 float clamp_min, spikerl_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * Diagnostics
 * ---------------------------------------------------------------------------------------- */
const char* spikerl_last_error(void);   /* thread-local message for the last non-OK status  */
const char* spikerl_version(void);
/* Number of kernel launches the library enqueued since the last reset (host counter). */
long long spikerl_launch_count(int reset);

/* Opt-in per-launch timing: while enabled (and the stream is not capturing) every kernel launch
 * is bracketed by CUDA events on its own stream, tagged with the algorithmic work the launcher
 * attributes to it. enable(0/1) clears previous records. summary() synchronises on the recorded
 * events and aggregates per kernel name; returns the number of distinct kernels (or -1). */
typedef struct {
  char name[48];
  int bound;            /* 0 = HBM bytes, 1 = tensor-core flops, 2 = SIMT ALU flops, 3 = latency */
  long long launches;
  double total_ms;
  double flops, bytes;  /* algorithmic work summed over the launches                            */
} spikerl_prof_entry;
void spikerl_prof_enable(int on);
int spikerl_prof_summary(spikerl_prof_entry* out, int max_entries);
/* The profiling pass's launches in enqueue order, each with its start / end (ms) relative to the
 * first recorded launch's start (events on the launch's own stream: concurrent branches show as
 * overlapping intervals). Returns the number of launches (or -1). */
typedef struct {
  char name[48];
  double start_ms, end_ms;
} spikerl_prof_span;
int spikerl_prof_timeline(spikerl_prof_span* out, int max_entries);
/* Live watch of one kernel inside a timed region (bench.py's roofline): every launch named `name`
 * (the names spikerl_prof_summary reports) is bracketed by the next caller-owned event pair
 * (cudaEvent_t created with timing), ev_begin[i] / ev_end[i], i = 0..n-1, recorded on the stream
 * the kernel is launched on; inside a stream capture the records become event nodes of the graph,
 * re-recorded at every replay. name == NULL turns the watch off. watch_count() = pairs used since
 * the last spikerl_prof_watch (re-arming resets it). */
int spikerl_prof_watch(const char* name, void* const* ev_begin, void* const* ev_end, int n);
int spikerl_prof_watch_count(void);
/* name == "*" watches every launch; watch_name(i) = the kernel name of pair i (or ""). */
const char* spikerl_prof_watch_name(int i);

#ifdef __cplusplus
}
#endif
#endif /* SPIKERL_H */
