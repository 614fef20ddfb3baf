// k_critic.cu — K8: twin-critic ReLU MLP forward/backward ("deep critic network";
// SPEC.md:208-211, 279; configs[1] 23->256->256->1). Latency-bound at configs[1..3] batch sizes
// (SURVEY.md §8(d)), so this is a compact tiled SIMT GEMM with fused epilogues, batched over the
// two critics with blockIdx.z. bf16 precision follows DESIGN.md R20: the input x, the weights,
// the hidden activations and the activation-gradients are rounded to bf16 where they enter a
// contraction; accumulation, biases, losses and gradients stay fp32.
#include "internal.h"

namespace spk {

namespace {

enum Epi { EPI_STORE = 0, EPI_BIAS_RELU = 1, EPI_MASK = 2 };

struct GemmArgs {
  int M, N, K;
  const void* A; long long sam, sak, a_bs;   // A(m,k) = A[m*sam + k*sak] (+ z*a_bs)
  const void* Bm; long long sbk, sbn, b_bs;  // B(k,n) = B[k*sbk + n*sbn] (+ z*b_bs)
  float* C; long long ldc, c_bs;             // C[m*ldc + n] (+ z*c_bs)
  float* C2; long long c2_bs;                // EPI_BIAS_RELU: rounded activation out
  const float* bias; long long bias_bs;      // EPI_BIAS_RELU: bias[n]
  const float* mask; long long mask_bs;      // EPI_MASK: pre-activation (mask = z > 0)
  int round_out;                             // round C / C2 to bf16
};

template <typename TA, typename TB> struct Ld;
__device__ __forceinline__ float tof(float x) { return x; }
__device__ __forceinline__ float tof(__nv_bfloat16 x) { return __bfloat162float(x); }

// 32x32 output tiles (latency-bound sizes: maximise the number of blocks), 256 threads with 2x2
// outputs each, K chunks of 32 staged in shared memory with loads coalesced along whichever of
// (m, k) / (k, n) is contiguous in memory; fp32 accumulation in a fixed k order.
constexpr int TM = 32, TN = 32, TK = 32;

template <typename TA, typename TB, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sA[TK][TM + 1];
  __shared__ float sB[TK][TN + 1];
  const int z = blockIdx.z;
  const TA* A = (const TA*)g.A + z * g.a_bs;
  const TB* Bm = (const TB*)g.Bm + z * g.b_bs;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const bool a_kfast = g.sak == 1, b_kfast = g.sbk == 1;
  float acc[2][2] = {};
  // register double buffering: the next K chunk's global loads are in flight while the current
  // chunk is multiplied out of shared memory (loads go through the read-only path, so they are
  // not serialised behind the shared-memory stores)
  constexpr int PER = TK * TM / 256;  // 4 elements of A and of B per thread per chunk
  float ra[PER], rb[PER];
  auto load = [&](int k0) {
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int i = threadIdx.x + r * 256;
      {
        const int kk = a_kfast ? i % TK : i / TM, mm = a_kfast ? i / TK : i % TM;
        const int m = m0 + mm, k = k0 + kk;
        ra[r] = (m < g.M && k < g.K) ? tof(__ldg(A + (long long)m * g.sam + (long long)k * g.sak)) : 0.f;
      }
      {
        const int kk = b_kfast ? i % TK : i / TN, nn = b_kfast ? i / TK : i % TN;
        const int n = n0 + nn, k = k0 + kk;
        rb[r] = (n < g.N && k < g.K) ? tof(__ldg(Bm + (long long)k * g.sbk + (long long)n * g.sbn)) : 0.f;
      }
    }
  };
  load(0);
  for (int k0 = 0; k0 < g.K; k0 += TK) {
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int i = threadIdx.x + r * 256;
      const int ka = a_kfast ? i % TK : i / TM, ma = a_kfast ? i / TK : i % TM;
      const int kb = b_kfast ? i % TK : i / TN, nb = b_kfast ? i / TK : i % TN;
      sA[ka][ma] = ra[r];
      sB[kb][nb] = rb[r];
    }
    __syncthreads();
    if (k0 + TK < g.K) load(k0 + TK);
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      const float a0 = sA[kk][ty * 2], a1 = sA[kk][ty * 2 + 1];
      const float b0 = sB[kk][tx * 2], b1 = sB[kk][tx * 2 + 1];
      acc[0][0] = __fmaf_rn(a0, b0, acc[0][0]);
      acc[0][1] = __fmaf_rn(a0, b1, acc[0][1]);
      acc[1][0] = __fmaf_rn(a1, b0, acc[1][0]);
      acc[1][1] = __fmaf_rn(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
  float* C = g.C + z * g.c_bs;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int m = m0 + ty * 2 + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = n0 + tx * 2 + j;
      if (n >= g.N) continue;
      float val = acc[i][j];
      const long long ci = (long long)m * g.ldc + n;
      if (EPI == EPI_BIAS_RELU) {
        val = __fadd_rn(val, g.bias[z * g.bias_bs + n]);
        C[ci] = val;                                   // pre-activation z (relu mask source)
        float h = fmaxf(val, 0.f);
        if (g.round_out) h = bf16_round(h);
        g.C2[z * g.c2_bs + ci] = h;
      } else if (EPI == EPI_MASK) {
        val = g.mask[z * g.mask_bs + ci] > 0.f ? val : 0.f;
        C[ci] = g.round_out ? bf16_round(val) : val;
      } else {
        C[ci] = val;
      }
    }
  }
}

template <int EPI>
int run_gemm(const GemmArgs& g, int nz, bool a_bf16, bool b_bf16, cudaStream_t st) {
  ProfScope ps_("critic_gemm_simt", PB_ALU, 2.0 * g.M * (double)g.N * g.K * nz, 0.0, st);
  dim3 grid(cdiv(g.N, TN), cdiv(g.M, TM), nz);
  if (a_bf16 && b_bf16) pdl((gemm_simt_kernel<__nv_bfloat16, __nv_bfloat16, EPI>), grid, 256, 0, st)(g);
  else if (a_bf16) pdl((gemm_simt_kernel<__nv_bfloat16, float, EPI>), grid, 256, 0, st)(g);
  else if (b_bf16) pdl((gemm_simt_kernel<float, __nv_bfloat16, EPI>), grid, 256, 0, st)(g);
  else pdl((gemm_simt_kernel<float, float, EPI>), grid, 256, 0, st)(g);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

__global__ void build_x_kernel(int B, int S, int A, const float* __restrict__ obs,
                               const float* __restrict__ act, int round, float* __restrict__ X) {
  pdl_wait();
  pdl_trigger();
  const int in = S + A;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * in; i += gridDim.x * blockDim.x) {
    const int b = i / in, c = i % in;
    float v = c < S ? obs[(size_t)b * S + c] : act[(size_t)b * A + (c - S)];
    X[i] = round ? bf16_round(v) : v;
  }
}

// Q[z][b] = sum_j H2[z][b][j] W3[z][j] + b3[z]: one warp per (z, b), fixed lane-strided order then
// a fixed butterfly.
template <typename TW>
__global__ void critic_out_kernel(int B, int H2, const float* __restrict__ H, long long h_bs,
                                  const TW* __restrict__ W3, long long w_bs,
                                  const float* __restrict__ b3, long long b_bs, float* __restrict__ q) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int z = blockIdx.y;
  if (warp >= B) return;
  const float* h = H + z * h_bs + (size_t)warp * H2;
  const TW* w = W3 + z * w_bs;
  float s = 0.f;
  for (int j = lane; j < H2; j += 32) s = __fmaf_rn(h[j], tof(w[j]), s);
  for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  if (lane == 0) q[(size_t)z * B + warp] = __fadd_rn(s, b3[z * b_bs]);
}

// loss = sum_z mean_b (Q_z - y)^2 ; dQ[z][b] = 2 (Q_z - y)/B. Single block, fixed order.
__global__ void __launch_bounds__(256) critic_loss_kernel(int B, int nz, const float* __restrict__ q,
                                                          const TdY y,
                                                          float* __restrict__ dq,
                                                          float* __restrict__ loss) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[256];
  float tot = 0.f;
  for (int z = 0; z < nz; ++z) {
    float s = 0.f;
    for (int b = threadIdx.x; b < B; b += 256) {
      const float e = __fsub_rn(q[(size_t)z * B + b], y.get(b, z));
      s = __fmaf_rn(e, e, s);
      dq[(size_t)z * B + b] = __fdiv_rn(__fmul_rn(2.0f, e), (float)B);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] = __fadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
      __syncthreads();
    }
    tot = __fadd_rn(tot, __fdiv_rn(red[0], (float)B));
    __syncthreads();
  }
  if (threadIdx.x == 0 && loss) *loss = tot;
}

__global__ void fill_kernel(float* x, int n, float v) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// dZ2[z][b][j] = round(dQ[z][b] * W3[z][j] * [Z2 > 0])
template <typename TW>
__global__ void critic_dz2_kernel(int B, int H2, const float* __restrict__ dq,
                                  const TW* __restrict__ W3, long long w_bs,
                                  const float* __restrict__ Z2, long long zb, int round,
                                  float* __restrict__ dZ2) {
  pdl_wait();
  pdl_trigger();
  const int z = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * H2; i += gridDim.x * blockDim.x) {
    const int b = i / H2, j = i % H2;
    float v = Z2[z * zb + i] > 0.f ? __fmul_rn(dq[(size_t)z * B + b], tof(W3[z * w_bs + j])) : 0.f;
    dZ2[z * zb + i] = round ? bf16_round(v) : v;
  }
}

// column sums: out[z*o_bs + j] = sum_b w_b M[z][b][j]; also dW3 = dQ^T H2. Block = 32 columns x
// 8 row-groups; each row-group sums a strided subset of b, then a fixed-order combine.
__global__ void __launch_bounds__(256) colsum_kernel(int B, int N, const float* __restrict__ M, long long m_bs,
                                                     const float* __restrict__ wgt, long long w_bs,
                                                     float* __restrict__ out, long long o_bs) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][33];
  const int z = blockIdx.y;
  const int jl = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + jl;
  float s = 0.f;
  if (j < N) {
    for (int b = rg; b < B; b += 8) {
      const float m = __ldg(M + z * m_bs + (size_t)b * N + j);
      s = wgt ? __fmaf_rn(__ldg(wgt + z * w_bs + b), m, s) : __fadd_rn(s, m);
    }
  }
  red[rg][jl] = s;
  __syncthreads();
  if (rg == 0 && j < N) {
    float t = red[0][jl];
#pragma unroll
    for (int r = 1; r < 8; ++r) t = __fadd_rn(t, red[r][jl]);
    out[z * o_bs + j] = t;
  }
}

// db3[z] = sum_b dQ[z][b]
__global__ void sum_dq_kernel(int B, const float* __restrict__ dq, float* __restrict__ out,
                              long long o_bs) {
  pdl_wait();
  pdl_trigger();
  const int z = blockIdx.x;
  if (threadIdx.x != 0) return;
  float s = 0.f;
  for (int b = 0; b < B; ++b) s = __fadd_rn(s, dq[(size_t)z * B + b]);
  out[z * o_bs] = s;
}

__global__ void slice_cols_kernel(int B, int in, int S, int A, const float* __restrict__ dX,
                                  float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * A) return;
  const int b = i / A, a = i % A;
  out[i] = dX[(size_t)b * in + S + a];
}

struct CriticWs {
  float *X, *Z1, *H1, *Z2, *H2, *q, *dq, *dZ2, *dZ1, *dX;
};

CriticWs carve(const CriticDims& c, int B, void* base) {
  CriticWs w;
  char* p = (char*)base;
  auto take = [&](size_t n) { float* r = (float*)p; p += align_up(n * sizeof(float), 256); return r; };
  w.X = take((size_t)B * c.in);
  w.Z1 = take(2ull * B * c.H1); w.H1 = take(2ull * B * c.H1);
  w.Z2 = take(2ull * B * c.H2); w.H2 = take(2ull * B * c.H2);
  w.q = take(2ull * B); w.dq = take(2ull * B);
  w.dZ2 = take(2ull * B * c.H2); w.dZ1 = take(2ull * B * c.H1);
  w.dX = take((size_t)B * c.in);
  return w;
}

}  // namespace

size_t critic_ws_bytes(const CriticDims& c, int B) {
  size_t n = 0;
  auto add = [&](size_t e) { n += align_up(e * sizeof(float), 256); };
  add((size_t)B * c.in);
  add(2ull * B * c.H1); add(2ull * B * c.H1); add(2ull * B * c.H2); add(2ull * B * c.H2);
  add(2ull * B); add(2ull * B); add(2ull * B * c.H2); add(2ull * B * c.H1); add((size_t)B * c.in);
  const size_t m = critic_mma_ok(c) ? critic_mma_ws_bytes(c, B) : 0;
  return n > m ? n : m;
}

// SIMT GEMM path: fp32 precision only (bf16 critics run on the tensor-core kernels).
int critic_fwd_bwd(const CriticDims& c, int B, const float* params2, const __nv_bfloat16* pb16,
                   const float* obs, int S, const float* act, int A, const TdY* y, float* q,
                   float* loss, float* grad2, float* grad_act, float act_scale, int nz, void* ws,
                   cudaStream_t st, cudaEvent_t wait_before_loss, const float* dq_scale, const CriticDecode* dec) {
  if (critic_mma_ok(c))
    return critic_mma_fwd_bwd(c, B, params2, pb16, obs, S, act, A, y, q, loss, grad2, grad_act, act_scale, nz, ws, st,
                              wait_before_loss, dq_scale, dec);
  if (dec) { set_error("critic: in-launch decoding needs the small-batch tensor-core critic"); return SPIKERL_E_UNSUPPORTED; }
  if (c.bf16) {   // no silent switch of engine (north_star: no multi-backend dispatch)
    set_error("bf16 critic: the tensor-core critic needs hidden widths 256-256 and in_dim <= 512 (got %d-%d, %d)",
              c.H1, c.H2, c.in);
    return SPIKERL_E_UNSUPPORTED;
  }
  if (dq_scale) { set_error("critic: loss scaling needs the bf16 tensor-core critic"); return SPIKERL_E_UNSUPPORTED; }
  CriticWs w = carve(c, B, ws);
  const bool bf = c.bf16 != 0;
  const long long P = (long long)c.off[SPIKERL_CRITIC_NPARAM];
  auto Wp = [&](int idx) -> const void* {
    return bf ? (const void*)(pb16 + c.off[idx]) : (const void*)(params2 + c.off[idx]);
  };
  const int in = c.in, H1 = c.H1, H2 = c.H2;
  pdl(build_x_kernel, cdiv((long long)B * in, 256) < 1184 ? cdiv((long long)B * in, 256) : 1184, 256, 0, st)(
      B, S, A, obs, act, bf, w.X);
  SPK_LAUNCHED();
  // layer 1: Z1 = X W1^T + b1 ; H1 = round(relu(Z1))
  {
    GemmArgs g{};
    g.M = B; g.N = H1; g.K = in;
    g.A = w.X; g.sam = in; g.sak = 1; g.a_bs = 0;
    g.Bm = Wp(SPIKERL_CRITIC_W1); g.sbk = 1; g.sbn = in; g.b_bs = P;
    g.C = w.Z1; g.ldc = H1; g.c_bs = (long long)B * H1; g.C2 = w.H1; g.c2_bs = g.c_bs;
    g.bias = params2 + c.off[SPIKERL_CRITIC_B1]; g.bias_bs = P; g.round_out = bf;
    SPK_TRY(run_gemm<EPI_BIAS_RELU>(g, nz, false, bf, st));
  }
  // layer 2
  {
    GemmArgs g{};
    g.M = B; g.N = H2; g.K = H1;
    g.A = w.H1; g.sam = H1; g.sak = 1; g.a_bs = (long long)B * H1;
    g.Bm = Wp(SPIKERL_CRITIC_W2); g.sbk = 1; g.sbn = H1; g.b_bs = P;
    g.C = w.Z2; g.ldc = H2; g.c_bs = (long long)B * H2; g.C2 = w.H2; g.c2_bs = g.c_bs;
    g.bias = params2 + c.off[SPIKERL_CRITIC_B2]; g.bias_bs = P; g.round_out = bf;
    SPK_TRY(run_gemm<EPI_BIAS_RELU>(g, nz, false, bf, st));
  }
  // layer 3 -> q
  {
    dim3 grid(cdiv((long long)B * 32, 256), nz);
    if (bf)
      pdl((critic_out_kernel<__nv_bfloat16>), grid, 256, 0, st)(
          B, H2, w.H2, (long long)B * H2, pb16 + c.off[SPIKERL_CRITIC_W3], P,
          params2 + c.off[SPIKERL_CRITIC_B3], P, q);
    else
      pdl((critic_out_kernel<float>), grid, 256, 0, st)(B, H2, w.H2, (long long)B * H2,
                                                     params2 + c.off[SPIKERL_CRITIC_W3], P,
                                                     params2 + c.off[SPIKERL_CRITIC_B3], P, q);
    SPK_LAUNCHED();
  }
  const bool want_params = (y != nullptr && grad2 != nullptr);
  if (wait_before_loss) SPK_CHECK_CUDA(cudaStreamWaitEvent(st, wait_before_loss, 0));
  if (y) {
    pdl(critic_loss_kernel, 1, 256, 0, st)(B, nz, q, *y, w.dq, loss);
    SPK_LAUNCHED();
  }
  if (!want_params && !grad_act) return SPIKERL_OK;
  int nb = nz;
  if (!want_params) {
    // actor step: dQ1 = act_scale for every sample, critic 0 only
    pdl(fill_kernel, cdiv(B, 256), 256, 0, st)(w.dq, B, act_scale);
    SPK_LAUNCHED();
    nb = 1;
  }
  // dZ2 = round(dQ W3 [Z2>0])
  {
    dim3 grid(cdiv((long long)B * H2, 256) < 1184 ? cdiv((long long)B * H2, 256) : 1184, nb);
    if (bf)
      pdl((critic_dz2_kernel<__nv_bfloat16>), grid, 256, 0, st)(B, H2, w.dq, pb16 + c.off[SPIKERL_CRITIC_W3], P,
                                                             w.Z2, (long long)B * H2, bf, w.dZ2);
    else
      pdl((critic_dz2_kernel<float>), grid, 256, 0, st)(B, H2, w.dq, params2 + c.off[SPIKERL_CRITIC_W3], P,
                                                     w.Z2, (long long)B * H2, bf, w.dZ2);
    SPK_LAUNCHED();
  }
  // dZ1 = round((dZ2 W2) [Z1 > 0])
  {
    GemmArgs g{};
    g.M = B; g.N = H1; g.K = H2;
    g.A = w.dZ2; g.sam = H2; g.sak = 1; g.a_bs = (long long)B * H2;
    g.Bm = Wp(SPIKERL_CRITIC_W2); g.sbk = H1; g.sbn = 1; g.b_bs = P;
    g.C = w.dZ1; g.ldc = H1; g.c_bs = (long long)B * H1;
    g.mask = w.Z1; g.mask_bs = (long long)B * H1; g.round_out = bf;
    SPK_TRY(run_gemm<EPI_MASK>(g, nb, false, bf, st));
  }
  if (want_params) {
    // dW3 = dQ^T H2, db3 = sum dQ
    pdl(colsum_kernel, dim3(cdiv(H2, 32), nz), 256, 0, st)(B, H2, w.H2, (long long)B * H2, w.dq, B,
                                                           grad2 + c.off[SPIKERL_CRITIC_W3], P);
    SPK_LAUNCHED();
    pdl(sum_dq_kernel, nz, 32, 0, st)(B, w.dq, grad2 + c.off[SPIKERL_CRITIC_B3], P);
    SPK_LAUNCHED();
    // dW2 = dZ2^T H1 ; db2 = colsum dZ2
    {
      GemmArgs g{};
      g.M = H2; g.N = H1; g.K = B;
      g.A = w.dZ2; g.sam = 1; g.sak = H2; g.a_bs = (long long)B * H2;
      g.Bm = w.H1; g.sbk = H1; g.sbn = 1; g.b_bs = (long long)B * H1;
      g.C = grad2 + c.off[SPIKERL_CRITIC_W2]; g.ldc = H1; g.c_bs = P;
      SPK_TRY(run_gemm<EPI_STORE>(g, nz, false, false, st));
    }
    pdl(colsum_kernel, dim3(cdiv(H2, 32), nz), 256, 0, st)(B, H2, w.dZ2, (long long)B * H2, nullptr, 0,
                                                           grad2 + c.off[SPIKERL_CRITIC_B2], P);
    SPK_LAUNCHED();
    // dW1 = dZ1^T X ; db1 = colsum dZ1
    {
      GemmArgs g{};
      g.M = H1; g.N = in; g.K = B;
      g.A = w.dZ1; g.sam = 1; g.sak = H1; g.a_bs = (long long)B * H1;
      g.Bm = w.X; g.sbk = in; g.sbn = 1; g.b_bs = 0;
      g.C = grad2 + c.off[SPIKERL_CRITIC_W1]; g.ldc = in; g.c_bs = P;
      SPK_TRY(run_gemm<EPI_STORE>(g, nz, false, false, st));
    }
    pdl(colsum_kernel, dim3(cdiv(H1, 32), nz), 256, 0, st)(B, H1, w.dZ1, (long long)B * H1, nullptr, 0,
                                                           grad2 + c.off[SPIKERL_CRITIC_B1], P);
    SPK_LAUNCHED();
  }
  if (grad_act) {
    // dX = dZ1[0] W1[0] ; grad_act = dX[:, S:]
    GemmArgs g{};
    g.M = B; g.N = in; g.K = H1;
    g.A = w.dZ1; g.sam = H1; g.sak = 1; g.a_bs = 0;
    g.Bm = Wp(SPIKERL_CRITIC_W1); g.sbk = in; g.sbn = 1; g.b_bs = 0;
    g.C = w.dX; g.ldc = in; g.c_bs = 0;
    SPK_TRY(run_gemm<EPI_STORE>(g, 1, false, bf, st));
    pdl(slice_cols_kernel, cdiv((long long)B * A, 256), 256, 0, st)(B, in, S, A, w.dX, grad_act);
    SPK_LAUNCHED();
  }
  return SPIKERL_OK;
}

}  // namespace spk
