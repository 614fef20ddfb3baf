// common.cuh — shared internals of libspikerl.so (product path only; no oracle code here).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstddef>
#include "spikerl.h"

namespace spk {

// Current device index (per-device caches below are keyed by it; a process may drive several GPUs).
inline int cur_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 31;
}

// SM count of the current device (cached per device; grids of persistent / grid-strided kernels are
// sized by it)
inline int num_sms() {
  static int n[32] = {};
  const int dev = cur_device();
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

// ----------------------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
void note_launch(int n = 1);
cudaError_t take_launch_error();

#define SPK_CHECK_CUDA(expr)                                                         \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      ::spk::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),       \
                       __FILE__, __LINE__);                                          \
      return SPIKERL_E_CUDA;                                                         \
    }                                                                                \
  } while (0)

#define SPK_LAUNCHED()                                                               \
  do {                                                                               \
    ::spk::note_launch();                                                            \
    cudaError_t e_ = ::spk::take_launch_error();                                     \
    if (e_ == cudaSuccess) e_ = cudaGetLastError();                                  \
    if (e_ != cudaSuccess) {                                                         \
      ::spk::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_),   \
                       __FILE__, __LINE__);                                          \
      return SPIKERL_E_CUDA;                                                         \
    }                                                                                \
  } while (0)

#define SPK_TRY(expr)                                                                \
  do {                                                                               \
    int s_ = (expr);                                                                 \
    if (s_ != SPIKERL_OK) return s_;                                                 \
  } while (0)

// Opt a kernel into > 48 KB of dynamic shared memory once per (call site, device): the attribute
// is per device, so a process driving several GPUs sets it on each before the first launch there.
#define SPK_SMEM_ATTR(kernel, bytes)                                                  \
  do {                                                                               \
    static unsigned done_mask_ = 0u;                                                 \
    const unsigned bit_ = 1u << ::spk::cur_device();                                 \
    if (!(__atomic_load_n(&done_mask_, __ATOMIC_ACQUIRE) & bit_)) {                  \
      SPK_CHECK_CUDA(cudaFuncSetAttribute((kernel),                                  \
                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes)));    \
      __atomic_fetch_or(&done_mask_, bit_, __ATOMIC_ACQ_REL);                        \
    }                                                                                \
  } while (0)

// ----------------------------------------------------------------------------- PDL
// Programmatic dependent launch: every library kernel is launched with programmatic stream
// serialization and begins with pdl_wait() (returns once the preceding kernel in the stream has
// completed and its writes are visible; a no-op without PDL) and pdl_trigger() (the next kernel
// may be scheduled now and run its prologue: launch latency, barrier / TMEM setup, tensor-map
// prefetch overlap this kernel). Because every kernel waits before touching global memory,
// completion stays transitive along the stream. SPIKERL_PDL=0 turns the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
void note_launch_error(cudaError_t e);
// Scheduling priority of the launches enqueued by this host thread (cudaLaunchAttributePriority;
// 0 = the device default, the lowest; negative = higher). Set by LaunchPriority scopes around the
// critical branches of the TD3 update DAG.
int& launch_priority();
struct LaunchPriority {
  int old;
  explicit LaunchPriority(int p) : old(launch_priority()) { launch_priority() = p; }
  ~LaunchPriority() { launch_priority() = old; }
};

template <typename... KArgs>
struct PdlLaunch {
  void (*k)(KArgs...);
  dim3 g, b;
  size_t smem;
  cudaStream_t st;
  template <typename... Args>
  void operator()(Args&&... args) const {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (const int pr = launch_priority()) {
      at[1].id = cudaLaunchAttributePriority;
      at[1].val.priority = pr;
      cfg.numAttrs = 2;
    }
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
    if (e != cudaSuccess) note_launch_error(e);
  }
};
template <typename... KArgs>
inline PdlLaunch<KArgs...> pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st) {
  return PdlLaunch<KArgs...>{k, g, b, smem, st};
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int round_up(int x, int a) { return (x + a - 1) / a * a; }
inline int cdiv(long long x, long long a) { return (int)((x + a - 1) / a); }

// ----------------------------------------------------------------------------- dims
constexpr int kPad = 128;  // neuron padding (MMA M tile; multiple of the 64-wide K tile)

struct ActorDims {
  int S, A, E, D, K0, N1, N2, N3, T;
  int N[4];       // true widths N0=K0, N1, N2, N3
  int P[4];       // padded widths (multiples of kPad)
  int Wd[4];      // u32 words per (t,b) row = P/32
  size_t off[SPIKERL_ACTOR_NPARAM + 1];
  size_t boff[4]; // bf16 copy element offsets of W1, W2, W3 ([P_l][P_{l-1}] each); boff[3] = total
  float dc, dv, vth, win, zh, sigma_floor;
  int bf16;       // 16-bit GEMM operands (precision BF16 or FP16)
  int f16;        // ... and they are fp16 (precision FP16: tcgen05 engine only)
  int engine;     // resolved: SPIKERL_ENGINE_SIMT or SPIKERL_ENGINE_TCGEN05
  int rho;        // reset_grad: BPTT through the reset gate (fp32 v_t kept in the tape)
};
int actor_dims(const spikerl_actor_cfg* cfg, ActorDims* d);
unsigned long long actor_cfg_hash(const spikerl_actor_cfg* cfg);

struct TapeLayout {
  size_t A, bits[4], mask[4], counts, act, total;
  // neuron-major copies of the hidden layers' spike / mask planes (tcgen05 engine only):
  // u8 [ceil32(B)/8][P_l][tpad]: byte (o, n, t) holds batch rows 8o..8o+7 of neuron n at step t;
  // written by the forward epilogue, read by the DX epilogue
  size_t bitsT[4], maskT[4];
  int tpad;   // T rounded up to 16
  size_t V[4];   // rho = 1: fp32 membrane potentials [T][B][P_l], l = 1..3 (else 0)
};
TapeLayout tape_layout(const ActorDims& d, int B);

struct CriticDims {
  int in, H1, H2, bf16;
  size_t off[SPIKERL_CRITIC_NPARAM + 1];
};
int critic_dims(const spikerl_critic_cfg* cfg, CriticDims* d);

// ----------------------------------------------------------------------------- device helpers
// the 16-bit operand bits of x: RNE to fp16 (f16) or to bf16
__device__ __forceinline__ unsigned short op16_bits(float x, bool f16) {
  return f16 ? __half_as_ushort(__float2half_rn(x)) : __bfloat16_as_ushort(__float2bfloat16_rn(x));
}
__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}

template <typename T> struct GT;
template <> struct GT<float> {
  __device__ __forceinline__ static float load(const float* p) { return *p; }
  __device__ __forceinline__ static void store(float* p, float v) { *p = v; }
  __device__ __forceinline__ static float round(float v) { return v; }
};
template <> struct GT<__nv_bfloat16> {
  __device__ __forceinline__ static float load(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
  __device__ __forceinline__ static float round(float v) { return bf16_round(v); }
};

// LIF scan step shared by every forward kernel (north_star equations), so all
// engines agree bit-for-bit on identical currents. c and v each take one fused multiply-add
// (one rounding, closer to the fp64 oracle than a rounded product plus a rounded sum); the
// reset gate is exact: v = c when the neuron fired at t-1.
struct LifConst { float dc, dv, vth, win; };
__device__ __forceinline__ void lif_step(const LifConst& k, float I, float& c, float& v, bool& o,
                                         bool& h) {
  c = __fmaf_rn(k.dc, c, I);
  v = o ? c : __fmaf_rn(k.dv, v, c);   // d_v * v * (1 - o_prev) + c
  o = v > k.vth;
  h = fabsf(__fsub_rn(v, k.vth)) < k.win;
}

// Reverse-scan step (rho = 0; reset gate detached): given g_o(t), o_t, h_t (bits) and the
// carried (dv_next, dc_next), returns G_t = delta_c_t.  SPEC.md:168-176; R11.
//   delta_v_t = h_t z g_t + d_v (1 - o_t) delta_v_{t+1};  delta_c_t = delta_v_t + d_c delta_c_{t+1}
// rho = 1 (reset gate differentiated, SPEC.md:171 variant; R11): the upstream gradient of
// step t becomes g - d_v v_t delta_v_{t+1} before the window factor: delta_v_t = h z (g - d_v v_t
// delta_v_{t+1}) + d_v (1 - o_t) delta_v_{t+1}.
__device__ __forceinline__ float rho_grad(float g, float dvc, float v, float dvn) {
  return __fmaf_rn(-__fmul_rn(dvc, v), dvn, g);
}
__device__ __forceinline__ float lif_back_step(float zh, float dvc, float dcc, float g, bool o,
                                               bool h, float& dvn, float& dcn) {
  const float hg = h ? __fmul_rn(zh, g) : 0.0f;
  const float dvt = o ? hg : __fmaf_rn(dvc, dvn, hg);
  const float dct = __fmaf_rn(dcc, dcn, dvt);
  dvn = dvt;
  dcn = dct;
  return dct;
}

}  // namespace spk

// ----------------------------------------------------------------------------- profiling
// Optional per-launch CUDA-event timing (spikerl_prof_*): bench.py uses it to time the
// dominant kernel on the stream it is launched on and to read the algorithmic work the
// launcher attributes to that launch (flops or bytes), for the roofline fraction.
namespace spk {
enum ProfBound { PB_HBM = 0, PB_TENSOR = 1, PB_ALU = 2, PB_LATENCY = 3 };
bool prof_on();
struct ProfScope {
  int slot = -1;
  int wslot = -1;   // live watch (spikerl_prof_watch): index of the event pair around this launch
  cudaStream_t st;
  ProfScope(const char* name, int bound, double flops, double bytes, cudaStream_t s);
  ~ProfScope();
};
}  // namespace spk
