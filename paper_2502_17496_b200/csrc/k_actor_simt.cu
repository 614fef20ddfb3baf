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
#include "rng.cuh"

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
    uint32_t* __restrict__ mask_out, uint8_t* __restrict__ counts, float* __restrict__ v_out, int P) {
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
    if (v_out) v_out[((size_t)t * B + b) * P + n] = v;   // rho = 1 tape (padding neurons: 0)
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
                        uint32_t* mask_out, uint8_t* counts, float* v_out, cudaStream_t st) {
  ProfScope ps_(l == 1 ? "lif_fwd_simt_L1" : (l == 2 ? "lif_fwd_simt_L2" : "lif_fwd_simt_L3"), PB_ALU,
                2.0 * d.T * B * (double)d.N[l] * d.N[l - 1], 0.0, st);
  LifConst kc{d.dc, d.dv, d.vth, d.win};
  dim3 grid(B, d.P[l] / 128);
  const int Win = d.Wd[l - 1], Wout = d.Wd[l];
  const size_t smem = sizeof(uint32_t) * Win;
  if (d.bf16) {
    pdl((lif_fwd_simt_kernel<__nv_bfloat16>), grid, 128, smem, st)(
        B, d.T, d.N[l], Win, Wout, bits_in, Wb16, d.P[l - 1], kc, bits_out, mask_out, counts, v_out, d.P[l]);
  } else {
    pdl((lif_fwd_simt_kernel<float>), grid, 128, smem, st)(B, d.T, d.N[l], Win, Wout, bits_in, Wf32,
                                                       d.N[l - 1], kc, bits_out, mask_out, counts, v_out, d.P[l]);
  }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ------------------------------------------------------------------------------ decoder forward
__global__ void dec_fwd_kernel(int B, int A, int D, int T, const uint8_t* __restrict__ counts,
                               const float* __restrict__ Wd, const float* __restrict__ bd,
                               float* __restrict__ act_out, float* __restrict__ act_tape, const TargetSmooth ts) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * A) return;
  const int b = i / A, j = i % A;
  const int N3 = A * D;
  const float invT = 1.0f / (float)T;
  float pre = 0.f;
  if (D <= kDecMaxD) {   // every count and weight requested before the (ordered) sum: one round trip
    uint32_t cv[kDecMaxD];
    float wv[kDecMaxD];
#pragma unroll
    for (int e = 0; e < kDecMaxD; ++e) {
      cv[e] = e < D ? counts[(size_t)b * N3 + j * D + e] : 0u;
      wv[e] = e < D ? Wd[j * D + e] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < kDecMaxD; ++e)
      if (e < D) pre = __fadd_rn(pre, __fmul_rn(wv[e], (float)cv[e] / (float)T));
  } else {
    for (int e = 0; e < D; ++e) {
      const float fr = (float)counts[(size_t)b * N3 + j * D + e] / (float)T;
      pre = __fadd_rn(pre, __fmul_rn(Wd[j * D + e], fr));
    }
  }
  (void)invT;
  pre = __fadd_rn(pre, bd[j]);
  const float a = tanhf(pre);
  act_out[i] = a;
  if (act_tape) act_tape[i] = a;
  if (ts.at) {   // target actor of a TD3 update: the smoothed target action (one launch less)
    const unsigned long long ctr = *ts.ctr_snap;
    if (ts.advance && i == 0) *ts.counter = ctr + 1;
    ts.at[i] = smooth_action(a, i, ts.noise, ts.sigma, ts.clip, ts.seed, ts.rank, ctr);
  }
}

int launch_dec_fwd(const ActorDims& d, int B, const uint8_t* counts, const float* Wd,
                   const float* bd, float* act_out, float* act_tape, cudaStream_t st, const TargetSmooth* smooth) {
  ProfScope ps_(smooth ? "dec_fwd_smooth" : "dec_fwd", PB_LATENCY, 0.0, (double)B * (d.N3 + 8.0 * d.A), st);
  const int n = B * d.A;
  const TargetSmooth none{};
  pdl(dec_fwd_kernel, cdiv(n, 256), 256, 0, st)(B, d.A, d.D, d.T, counts, Wd, bd, act_out, act_tape,
                                                 smooth ? *smooth : none);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ------------------------------------------------------- decoder backward + output reverse scan
// Output-layer reverse scan (HBM-bound: writes G3, reads the spike / mask planes). A thread owns
// 8 consecutive neurons of one batch row for all T steps: the 8 scans are independent chains,
// each step's 8 results leave as one 16-byte store (bf16) and the step's spike / mask bits are one
// byte of a word shared by 4 lanes. A warp covers 2 rows x 128 neurons; grid-strided over (row
// pair, group of 4 words). ncu r01: the one-neuron-per-lane version issued ~36 instructions per element and
// reached 31% of HBM bandwidth at configs[4].
template <typename GTy> struct Pack8;
template <> struct Pack8<__nv_bfloat16> {
  __device__ __forceinline__ static void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 u;
    u.x = bf2_bits(v[0], v[1]); u.y = bf2_bits(v[2], v[3]); u.z = bf2_bits(v[4], v[5]); u.w = bf2_bits(v[6], v[7]);
    *reinterpret_cast<uint4*>(p) = u;
  }
  __device__ __forceinline__ static uint32_t bf2_bits(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
};
template <> struct Pack8<__half> {
  __device__ __forceinline__ static void store(__half* p, const float (&v)[8]) {
    uint4 u;
    u.x = h2_bits(v[0], v[1]); u.y = h2_bits(v[2], v[3]); u.z = h2_bits(v[4], v[5]); u.w = h2_bits(v[6], v[7]);
    *reinterpret_cast<uint4*>(p) = u;
  }
  __device__ __forceinline__ static uint32_t h2_bits(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
};
template <> struct Pack8<float> {
  __device__ __forceinline__ static void store(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

template <typename GTy, int TT>
__global__ void __launch_bounds__(256, 4) dec_bwd_outscan_kernel(
    int B, int T, int A, int D, int N3, int W3, float dcc, float dvc, float zh,
    const float* __restrict__ grad_a, const float* __restrict__ act, const float* __restrict__ Wd,
    const uint32_t* __restrict__ bits3, const uint32_t* __restrict__ mask3, const float* __restrict__ v3,
    GTy* __restrict__ G3, float* __restrict__ g_pre_out, int write_pad) {
  pdl_wait();
  pdl_trigger();
  // lane = (row jr of 2, word wq of 4, octet oct of 4): a warp stores 2 rows x 128 neurons, i.e.
  // whole 128-byte lines of G3 (bf16), per step
  const int lane = threadIdx.x & 31, jr = lane >> 4, wq = (lane >> 2) & 3, oct = lane & 3;
  const int WG = W3 / 4;   // groups of 4 words (P3 is a multiple of 128)
  const long long units = (long long)((B + 1) / 2) * WG;
  const int P3 = 32 * W3;
  const size_t ts = (size_t)B * W3;    // bit-plane stride between timesteps
  const size_t gts = (size_t)B * P3;   // G3 stride between timesteps
  for (long long u = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < units;
       u += (long long)gridDim.x * (blockDim.x >> 5)) {
    const int w = (int)(u % WG) * 4 + wq, b = (int)(u / WG) * 2 + jr;
    if (b >= B) continue;   // (no warp-collective operations below)
    const int n0 = 32 * w + 8 * oct;
    // padded neurons (n >= N3) have G = 0: with the tcgen05 engine their columns are never read
    // (TMA zero-fills past N3), so those lanes store nothing
    const bool live = n0 < N3 || write_pad;
    // g_o3 = g_fr / T = g_pre_a Wd[a][d] / T, constant in t; g_pre written once per (b, action)
    float g[8];
    int a = n0 / D, e = n0 - a * D;
    float gp = 0.f;
    if (n0 < N3) {
      const float av = act[(size_t)b * A + a];
      gp = __fmul_rn(grad_a[(size_t)b * A + a], __fsub_rn(1.0f, __fmul_rn(av, av)));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      g[i] = 0.f;
      if (n0 + i < N3) {
        if (e == 0) g_pre_out[(size_t)b * A + a] = gp;
        g[i] = __fmul_rn(zh, __fdiv_rn(__fmul_rn(gp, Wd[a * D + e]), (float)T));   // h z g (h applied below)
      }
      if (++e == D && n0 + i + 1 < N3) {   // next action's population
        e = 0;
        ++a;
        const float av = act[(size_t)b * A + a];
        gp = __fmul_rn(grad_a[(size_t)b * A + a], __fsub_rn(1.0f, __fmul_rn(av, av)));
      }
    }
    float dvn[8], dcn[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { dvn[i] = 0.f; dcn[i] = 0.f; }
    const uint32_t* po = bits3 + (size_t)b * W3 + w;
    const uint32_t* ph = mask3 + (size_t)b * W3 + w;
    GTy* gq = G3 + (size_t)b * P3 + n0 + (size_t)(T - 1) * gts;   // step T-1; walks back by gts
    const float* vq = v3 ? v3 + (size_t)b * P3 + n0 + (size_t)(T - 1) * gts : nullptr;   // rho = 1
    const float zdv = __fmul_rn(zh, dvc);
    auto step = [&](uint32_t ow, uint32_t hw) {
      const uint32_t o8 = (ow >> (8 * oct)) & 0xFFu, h8 = (hw >> (8 * oct)) & 0xFFu;
      float G[8], vv[8];
      if (vq) {
        const float4 a = reinterpret_cast<const float4*>(vq)[0], c = reinterpret_cast<const float4*>(vq)[1];
        vv[0] = a.x; vv[1] = a.y; vv[2] = a.z; vv[3] = a.w; vv[4] = c.x; vv[5] = c.y; vv[6] = c.z; vv[7] = c.w;
        vq -= gts;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // lif_back_step with the window factor z folded into g (z is a constant per layer); rho = 1
        // subtracts z d_v v_t delta_v_{t+1}
        const float gi = vq ? __fmaf_rn(-__fmul_rn(zdv, vv[i]), dvn[i], g[i]) : g[i];
        const float hg = ((h8 >> i) & 1u) ? gi : 0.0f;
        const float dvt = ((o8 >> i) & 1u) ? hg : __fmaf_rn(dvc, dvn[i], hg);
        const float dct = __fmaf_rn(dcc, dcn[i], dvt);
        dvn[i] = dvt;
        dcn[i] = dct;
        G[i] = dct;
      }
      if (live) Pack8<GTy>::store(gq, G);
      gq -= gts;
    };
    if constexpr (TT > 0) {
      // T known: the words of up to 8 steps are requested together before their scan steps (one
      // memory latency per chunk; 8, not 16, keeps 4 blocks per SM resident without spills)
      constexpr int CH = TT > 8 ? 8 : TT;
      static_assert(TT % CH == 0, "T must be a multiple of the chunk");
#pragma unroll
      for (int c0 = TT - CH; c0 >= 0; c0 -= CH) {
        uint32_t ow[CH], hw[CH];
        const uint32_t *qo = po + (size_t)c0 * ts, *qh = ph + (size_t)c0 * ts;
#pragma unroll
        for (int k = 0; k < CH; ++k, qo += ts, qh += ts) { ow[k] = __ldg(qo); hw[k] = __ldg(qh); }
#pragma unroll
        for (int k = CH - 1; k >= 0; --k) step(ow[k], hw[k]);
      }
    } else {
      uint32_t ow = __ldg(po + (size_t)(T - 1) * ts), hw = __ldg(ph + (size_t)(T - 1) * ts);
      for (int t = T - 1; t >= 0; --t) {
        const uint32_t o = ow, h = hw;
        if (t > 0) { ow = __ldg(po + (size_t)(t - 1) * ts); hw = __ldg(ph + (size_t)(t - 1) * ts); }
        step(o, h);
      }
    }
  }
}

// TMA-staged variant (the default whenever its stage fits in shared memory): a block owns R batch
// rows x the live octets of the output layer (no dead lanes: N_3 = 170 uses 22 of a row's 32
// octets), one thread per (row, octet). The spike and mask planes of the block's next R rows and
// all T steps arrive by two 3-D TMA copies ([T][R][W3] boxes, rows past B zero-filled) into the
// other half of a double buffer while the current rows are scanned, so the scan never waits on a
// global load (ncu r01: the direct-load kernel above stalled on long-scoreboard 7.6 cycles per
// issued instruction and reached 29-37% of the copy peak at configs[4]).
namespace osc {
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "OSC_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra OSC_WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3(const CUtensorMap* m, void* dst, uint64_t* b, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(b)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
}  // namespace osc

template <typename GTy, int TT, bool RHO = false>   // RHO: rho = 1 (v3 read), its own instantiation
__global__ void __launch_bounds__(256, 4) dec_bwd_outscan_tma_kernel(
    const __grid_constant__ CUtensorMap map_o, const __grid_constant__ CUtensorMap map_h, int B, int T, int A,
    int D, int N3, int W3, int NO, int R, int planeS, float dcc, float dvc, float zh,
    const float* __restrict__ grad_a, const float* __restrict__ act, const float* __restrict__ Wd,
    const float* __restrict__ v3, GTy* __restrict__ G3, float* __restrict__ g_pre_out, int write_pad) {
  extern __shared__ __align__(128) uint8_t osm[];
  uint32_t* sbuf = reinterpret_cast<uint32_t*>(osm);              // [2 buffers][2 planes][planeS]
  uint64_t* bar = reinterpret_cast<uint64_t*>(osm + (size_t)16 * planeS);
  const int tid = threadIdx.x;
  const int units = (B + R - 1) / R;
  if (tid == 0) {
    osc::bar_init(&bar[0], 1);
    osc::bar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (TT > 0) T = TT;   // compile-time T: the step loop unrolls completely
  const uint32_t txb = 2u * (uint32_t)T * (uint32_t)R * (uint32_t)W3 * 4u;   // whole boxes (OOB rows count)
  auto issue = [&](int unit, int bi) {
    uint32_t* d0 = sbuf + (size_t)(2 * bi) * planeS;
    osc::bar_expect(&bar[bi], txb);
    osc::tma3(&map_o, d0, &bar[bi], 0, unit * R, 0);
    osc::tma3(&map_h, d0 + planeS, &bar[bi], 0, unit * R, 0);
  };
  if (tid == 0 && (int)blockIdx.x < units) issue(blockIdx.x, 0);
  const int o = tid % NO, r = tid / NO;
  const int n0 = 8 * o, w = o >> 2, sh = 8 * (o & 3);
  const int P3 = 32 * W3;
  // every thread's octet is live: NO counts only the octets below N3 (or all of P3 with write_pad)
  const int tstr = R * W3;
  // This thread's octet is fixed: with D >= 8 it spans at most two action populations (a0 for
  // i < split, a0 + 1 after), so its 8 decoder weights are loaded once and each row needs only the
  // pre-activation gradients of two actions, requested one unit ahead (ncu r01: the per-unit loads
  // of act / grad_a and the per-neuron action walk were ~45% of the kernel's stall samples)
  const bool two_max = D >= 8;
  const int a0 = n0 / D, split = D - (n0 - a0 * D);
  const bool has1 = two_max && split < 8 && n0 + split < N3;
  float w8[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w8[i] = (two_max && n0 + i < N3) ? Wd[n0 + i] : 0.f;   // Wd[a][e] at a D + e = n
  const bool pow2T = (T & (T - 1)) == 0;   // g / T is then an exact multiply
  const float invT = 1.0f / (float)T;
  float nav0 = 0.f, nga0 = 0.f, nav1 = 0.f, nga1 = 0.f;   // next unit's act / grad_a of a0, a0 + 1
  auto prefetch = [&](int unit) {
    const int bn = unit * R + r;
    if (two_max && unit < units && bn < B && n0 < N3) {
      nav0 = act[(size_t)bn * A + a0];
      nga0 = grad_a[(size_t)bn * A + a0];
      if (has1) { nav1 = act[(size_t)bn * A + a0 + 1]; nga1 = grad_a[(size_t)bn * A + a0 + 1]; }
    }
  };
  prefetch(blockIdx.x);
  int it = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
    const int bi = it & 1;
    if (tid == 0 && u + (int)gridDim.x < units) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of buffer bi^1
      issue(u + gridDim.x, bi ^ 1);
    }
    const int b = u * R + r;
    // g_o3 = g_fr / T = g_pre_a Wd[a][d] / T (constant in t), window factor z folded in
    float g[8];
    if (b < B && two_max) {
      const float gp0 = __fmul_rn(nga0, __fsub_rn(1.0f, __fmul_rn(nav0, nav0)));
      const float gp1 = __fmul_rn(nga1, __fsub_rn(1.0f, __fmul_rn(nav1, nav1)));
      prefetch(u + gridDim.x);
      if (n0 < N3 && split == D) g_pre_out[(size_t)b * A + a0] = gp0;       // the octet starts action a0
      if (has1) g_pre_out[(size_t)b * A + a0 + 1] = gp1;                    // ... or contains a0 + 1's start
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float x = __fmul_rn(i < split ? gp0 : gp1, w8[i]);
        g[i] = __fmul_rn(zh, pow2T ? __fmul_rn(x, invT) : __fdiv_rn(x, (float)T));
      }
    } else if (b < B) {
      int a = n0 / D, e = n0 - a * D;
      float gp = 0.f;
      if (n0 < N3) {
        const float av = act[(size_t)b * A + a];
        gp = __fmul_rn(grad_a[(size_t)b * A + a], __fsub_rn(1.0f, __fmul_rn(av, av)));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        g[i] = 0.f;
        if (n0 + i < N3) {
          if (e == 0) g_pre_out[(size_t)b * A + a] = gp;
          g[i] = __fmul_rn(zh, __fdiv_rn(__fmul_rn(gp, Wd[a * D + e]), (float)T));
        }
        if (++e == D && n0 + i + 1 < N3) {
          e = 0;
          ++a;
          const float av = act[(size_t)b * A + a];
          gp = __fmul_rn(grad_a[(size_t)b * A + a], __fsub_rn(1.0f, __fmul_rn(av, av)));
        }
      }
    }
    osc::bar_wait(&bar[bi], (uint32_t)(it >> 1) & 1u);
    if (b < B) {
      const uint32_t* so = sbuf + (size_t)(2 * bi) * planeS + r * W3 + w;
      const uint32_t* sm = so + planeS;
      float dvn[8], dcn[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) { dvn[i] = 0.f; dcn[i] = 0.f; }
      // G3 element offsets of this row: 32-bit (T B P3 < 2^32 is checked at launch)
      const uint32_t gts32 = (uint32_t)B * (uint32_t)P3;
      uint32_t go = (uint32_t)b * (uint32_t)P3 + (uint32_t)n0 + (uint32_t)(T - 1) * gts32;
      const float zdv = __fmul_rn(zh, dvc);
#pragma unroll (TT > 0 ? TT : 2)
      for (int t = T - 1; t >= 0; --t) {
        const uint32_t o8 = (so[t * tstr] >> sh) & 0xFFu, h8 = (sm[t * tstr] >> sh) & 0xFFu;
        float G[8], vv[8];
        if constexpr (RHO) {   // rho = 1: v_t of the 8 neurons (same element offsets as G3)
          const float4 a = reinterpret_cast<const float4*>(v3 + go)[0], c = reinterpret_cast<const float4*>(v3 + go)[1];
          vv[0] = a.x; vv[1] = a.y; vv[2] = a.z; vv[3] = a.w; vv[4] = c.x; vv[5] = c.y; vv[6] = c.z; vv[7] = c.w;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float gi = g[i];
          if constexpr (RHO) gi = __fmaf_rn(-__fmul_rn(zdv, vv[i]), dvn[i], g[i]);
          const float hg = ((h8 >> i) & 1u) ? gi : 0.0f;
          const float dvt = ((o8 >> i) & 1u) ? hg : __fmaf_rn(dvc, dvn[i], hg);
          const float dct = __fmaf_rn(dcc, dcn[i], dvt);
          dvn[i] = dvt;
          dcn[i] = dct;
          G[i] = dct;
        }
        Pack8<GTy>::store(G3 + go, G);
        go -= gts32;
      }
    }
    __syncthreads();   // buffer bi is refilled at the top of the next-but-one iteration
  }
}

// shared-memory plan of the staged scan: R rows per unit, the padded plane size in words (128-byte
// aligned TMA destinations); R = 0 when even one row per unit does not fit the budget
static void outscan_plan(const ActorDims& d, int wpad, int* NO, int* R, int* planeS) {
  const int nl = wpad ? d.P[3] : d.N3;
  *NO = (nl + 7) / 8;
  int r = 256 / *NO;
  constexpr size_t kBudget = 96 * 1024;
  while (r > 0 && 16 * (size_t)round_up(d.T * r * d.Wd[3], 32) + 16 > kBudget) --r;
  *R = r;
  *planeS = round_up(d.T * (r > 0 ? r : 1) * d.Wd[3], 32);
}

int launch_dec_bwd_outscan(const ActorDims& d, int B, const float* grad_a, const float* act,
                           const uint8_t* counts, const float* Wd, const uint32_t* bits3,
                           const uint32_t* mask3, const float* v3, void* G3, float* g_pre, cudaStream_t st) {
  // algorithmic bytes: G3 written for the N3 real neurons (tcgen05: padding never written), both
  // bit planes read
  const double gcols = d.engine == SPIKERL_ENGINE_TCGEN05 ? d.N3 : d.P[3];
  ProfScope ps_("dec_bwd_outscan", PB_HBM, 0.0, (double)d.T * B * (gcols * (d.bf16 ? 2.0 : 4.0) + 2.0 * d.Wd[3] * 4), st);
  (void)counts;
  const int wpad = d.engine == SPIKERL_ENGINE_TCGEN05 ? 0 : 1;     // SIMT kernels read P3 columns
  int NO, R, planeS;
  outscan_plan(d, wpad, &NO, &R, &planeS);
  static const bool direct = [] { const char* e = getenv("SPIKERL_OUTSCAN_DIRECT"); return e && e[0] == '1'; }();
  if (R > 0 && !direct && (unsigned long long)d.T * B * d.P[3] < (1ull << 32)) {
    CUtensorMap mo, mh;
    const uint64_t dims[3] = {(uint64_t)d.Wd[3], (uint64_t)B, (uint64_t)d.T};
    const uint64_t strides[2] = {(uint64_t)d.Wd[3] * 4, (uint64_t)B * d.Wd[3] * 4};
    const uint32_t box[3] = {(uint32_t)d.Wd[3], (uint32_t)R, (uint32_t)d.T};
    SPK_TRY(make_u32_map3(&mo, bits3, dims, strides, box));
    SPK_TRY(make_u32_map3(&mh, mask3, dims, strides, box));
    const size_t smem = (size_t)16 * planeS + 16;
    const int threads = NO * R;
    auto launch = [&](auto kern, auto* G) -> int {
      // per launch: the T-specialised kernels share one function-pointer type, so a static "done"
      // flag here would cover only the first of them
      SPK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
      }
      const int units = cdiv(B, R), cap = num_sms() * per_sm;
      const int waves = cdiv(units, cap);
      const int blocks = cdiv(units, waves);   // every block gets `waves` units (the last one fewer)
      pdl(kern, blocks, threads, smem, st)(mo, mh, B, d.T, d.A, d.D, d.N3, d.Wd[3], NO, R, planeS, d.dc, d.dv,
                                            d.zh, grad_a, act, Wd, v3, G, g_pre, wpad);
      SPK_LAUNCHED();
      return SPIKERL_OK;
    };
    if (v3) {   // rho = 1 (bf16 / fp32 operands; fp16 is rejected at configuration)
      if (d.bf16) return launch(dec_bwd_outscan_tma_kernel<__nv_bfloat16, 0, true>, (__nv_bfloat16*)G3);
      return launch(dec_bwd_outscan_tma_kernel<float, 0, true>, (float*)G3);
    }
    if (d.f16) {
      if (d.T == 16) return launch(dec_bwd_outscan_tma_kernel<__half, 16>, (__half*)G3);
      if (d.T == 5) return launch(dec_bwd_outscan_tma_kernel<__half, 5>, (__half*)G3);
      return launch(dec_bwd_outscan_tma_kernel<__half, 0>, (__half*)G3);
    }
    if (d.bf16) {
      if (d.T == 16) return launch(dec_bwd_outscan_tma_kernel<__nv_bfloat16, 16>, (__nv_bfloat16*)G3);
      if (d.T == 5) return launch(dec_bwd_outscan_tma_kernel<__nv_bfloat16, 5>, (__nv_bfloat16*)G3);
      return launch(dec_bwd_outscan_tma_kernel<__nv_bfloat16, 0>, (__nv_bfloat16*)G3);
    }
    return launch(dec_bwd_outscan_tma_kernel<float, 0>, (float*)G3);
  }
  const long long units = (long long)cdiv(B, 2) * (d.Wd[3] / 4);   // warps of work
  long long blocks = cdiv(units, 8);
  if (blocks > (long long)num_sms() * 8) blocks = (long long)num_sms() * 8;
  if (d.f16) {
    pdl((dec_bwd_outscan_kernel<__half, 0>), (int)blocks, 256, 0, st)(
        B, d.T, d.A, d.D, d.N3, d.Wd[3], d.dc, d.dv, d.zh, grad_a, act, Wd, bits3, mask3, v3, (__half*)G3, g_pre, wpad);
  } else if (d.bf16) {
    if (d.T == 16) pdl((dec_bwd_outscan_kernel<__nv_bfloat16, 16>), (int)blocks, 256, 0, st)(
        B, d.T, d.A, d.D, d.N3, d.Wd[3], d.dc, d.dv, d.zh, grad_a, act, Wd, bits3, mask3, v3, (__nv_bfloat16*)G3, g_pre, wpad);
    else if (d.T == 5) pdl((dec_bwd_outscan_kernel<__nv_bfloat16, 5>), (int)blocks, 256, 0, st)(
        B, d.T, d.A, d.D, d.N3, d.Wd[3], d.dc, d.dv, d.zh, grad_a, act, Wd, bits3, mask3, v3, (__nv_bfloat16*)G3, g_pre, wpad);
    else pdl((dec_bwd_outscan_kernel<__nv_bfloat16, 0>), (int)blocks, 256, 0, st)(
        B, d.T, d.A, d.D, d.N3, d.Wd[3], d.dc, d.dv, d.zh, grad_a, act, Wd, bits3, mask3, v3, (__nv_bfloat16*)G3, g_pre, wpad);
  } else {
    pdl((dec_bwd_outscan_kernel<float, 0>), (int)blocks, 256, 0, st)(
        B, d.T, d.A, d.D, d.N3, d.Wd[3], d.dc, d.dv, d.zh, grad_a, act, Wd, bits3, mask3, v3, (float*)G3, g_pre, 1);
  }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// dbd[j] = sum_b g_pre[b][j];  dWd[j][e] = sum_b g_pre[b][j] * cnt[b][jD+e] / T.
// Large B: two fixed-order passes (run-to-run deterministic): a block sums a contiguous chunk of rows for
// every output column (thread = column: the count bytes of a row are read coalesced, g_pre words
// broadcast), then one thread per column adds the chunk partials in chunk order. One chunk writes
// the result directly. (ncu r01: the former one-block-per-(j, e) kernel read the counts with a
// 170-byte stride and ran a 256-long dependent sum per thread: 0.17 ms at configs[4].)
constexpr int kDecRows = 32;   // rows per chunk (at least; chunks are capped at 4 per SM)
int dec_param_chunks(int B) {
  if (B <= 1024) return 1;   // latency regime: one block per column, no second launch
  const int c = cdiv(B, kDecRows), cap = 4 * num_sms();
  return c < cap ? c : cap;
}

__global__ void __launch_bounds__(256) dec_param_partial_kernel(int B, int A, int D, int T, int rows,
                                                                const float* __restrict__ g_pre,
                                                                const uint8_t* __restrict__ counts,
                                                                float* __restrict__ part, float* __restrict__ dWd,
                                                                float* __restrict__ dbd, int accum) {
  pdl_wait();
  pdl_trigger();
  // thread = (column c of a 32-column group, row lane rl of 8): a lane sums every 8th row of the
  // chunk (4 rows' loads in flight), the 8 lanes are added in lane order through shared memory
  __shared__ float red[8][33];
  const int N3 = A * D, NC = N3 + A;
  const int c = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int b0 = blockIdx.x * rows, b1 = min(B, b0 + rows);
  for (int n0 = 0; n0 < NC; n0 += 32) {
    const int n = n0 + c;
    const bool live = n < NC, bias = n >= N3;
    const int j = bias ? n - N3 : n / D;
    float s = 0.f;
    if (live) {
      int b = b0 + rl;
      for (; b + 24 < b1; b += 32) {
        float gp[4], cn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          gp[u] = g_pre[(size_t)(b + 8 * u) * A + j];
          cn[u] = bias ? 1.f : (float)counts[(size_t)(b + 8 * u) * N3 + n];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          s = bias ? __fadd_rn(s, gp[u]) : __fadd_rn(s, __fmul_rn(gp[u], cn[u] / (float)T));
      }
      for (; b < b1; b += 8) {
        const float gp = g_pre[(size_t)b * A + j];
        s = bias ? __fadd_rn(s, gp) : __fadd_rn(s, __fmul_rn(gp, (float)counts[(size_t)b * N3 + n] / (float)T));
      }
    }
    red[rl][c] = s;
    __syncthreads();
    if (rl == 0 && live) {
      float t = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) t = __fadd_rn(t, red[q][c]);
      if (gridDim.x == 1) {
        float* dst = bias ? (dbd + j) : (dWd + n);   // Wd[j][e] sits at j D + e = n
        *dst = accum ? __fadd_rn(*dst, t) : t;
      } else {
        part[(size_t)blockIdx.x * NC + n] = t;
      }
    }
    __syncthreads();
  }
}

// latency regime (B <= 1024): one block per (j, e), e == D the bias; fixed-order tree reduction
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

__global__ void dec_param_reduce_kernel(int A, int D, int chunks, const float* __restrict__ part,
                                        float* __restrict__ dWd, float* __restrict__ dbd, int accum) {
  pdl_wait();
  pdl_trigger();
  const int N3 = A * D, NC = N3 + A;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= NC) return;
  float s = 0.f;
  for (int c = 0; c < chunks; ++c) s = __fadd_rn(s, part[(size_t)c * NC + n]);
  float* dst = n >= N3 ? (dbd + (n - N3)) : (dWd + n);
  *dst = accum ? __fadd_rn(*dst, s) : s;
}

int launch_dec_param_grads(const ActorDims& d, int B, const float* g_pre, const uint8_t* counts,
                           float* dWd, float* dbd, float* part, int accumulate, cudaStream_t st) {
  ProfScope ps_("dec_param_grads", PB_LATENCY, 0.0, (double)B * (4.0 * d.A + d.N3), st);
  const int chunks = dec_param_chunks(B), rows = cdiv(B, chunks), NC = d.N3 + d.A;
  if (chunks == 1) {
    pdl(dec_param_grads_kernel, dim3(d.A, d.D + 1), 256, 0, st)(B, d.A, d.D, d.T, g_pre, counts, dWd, dbd,
                                                               accumulate);
    SPK_LAUNCHED();
    return SPIKERL_OK;
  }
  pdl(dec_param_partial_kernel, chunks, 256, 0, st)(B, d.A, d.D, d.T, rows, g_pre, counts, part, dWd, dbd,
                                                   accumulate);
  SPK_LAUNCHED();
  if (chunks > 1) {
    pdl(dec_param_reduce_kernel, cdiv(NC, 256), 256, 0, st)(d.A, d.D, chunks, part, dWd, dbd, accumulate);
    SPK_LAUNCHED();
  }
  return SPIKERL_OK;
}

// ------------------------------------------------- dX of layer l fused with reverse scan of l-1
// g_o^{l-1}[t][b][k] = sum_n G_l[t][b][n] W_l[n][k]; then the reverse scan of layer l-1 with its
// spike / mask bits gives G_{l-1}; for l == 2 also Gsum1[b][k] = sum_t G_1 (fp32, then rounded).
template <typename GTy, typename WT>
__global__ void __launch_bounds__(128) lif_dx_simt_kernel(
    int B, int T, int Nl, int Pl, int Nprev, int Pprev, int Wprev, float dcc, float dvc, float zh,
    const GTy* __restrict__ Gl, const WT* __restrict__ W, int ldw_, const uint32_t* __restrict__ bits,
    const uint32_t* __restrict__ mask, const float* __restrict__ vprev, GTy* __restrict__ Gprev,
    GTy* __restrict__ Gsum) {
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
      if (vprev) g = rho_grad(g, dvc, vprev[row * Pprev + k], dvn);   // rho = 1
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
                       const uint32_t* mask_prev, const float* v_prev, void* Gprev, void* Gsum,
                       cudaStream_t st) {
  ProfScope ps_(l == 3 ? "lif_dx_simt_L3" : "lif_dx_simt_L2", PB_ALU, 2.0 * d.T * B * (double)d.N[l] * d.N[l - 1], 0.0, st);
  dim3 grid(B, d.P[l - 1] / 128);
  const size_t smem = sizeof(float) * d.N[l];
  if (d.bf16)
    pdl((lif_dx_simt_kernel<__nv_bfloat16, __nv_bfloat16>), grid, 128, smem, st)(
        B, d.T, d.N[l], d.P[l], d.N[l - 1], d.P[l - 1], d.Wd[l - 1], d.dc, d.dv, d.zh,
        (const __nv_bfloat16*)Gl, Wb16, d.P[l - 1], bits_prev, mask_prev, v_prev, (__nv_bfloat16*)Gprev,
        (__nv_bfloat16*)Gsum);
  else
    pdl((lif_dx_simt_kernel<float, float>), grid, 128, smem, st)(
        B, d.T, d.N[l], d.P[l], d.N[l - 1], d.P[l - 1], d.Wd[l - 1], d.dc, d.dv, d.zh,
        (const float*)Gl, Wf32, d.N[l - 1], bits_prev, mask_prev, v_prev, (float*)Gprev, (float*)Gsum);
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
