// k_scan_ablation.cu — a standalone forward LIF scan over precomputed input currents: the ablation
// SURVEY §8(d) D-2 asks for, kept to show what the fused FWD epilogue saves. The product path never
// materialises the currents I_t = W o_{t-1}: the tcgen05 FWD kernel scans them in registers straight
// from TMEM. Unfused, the scan alone must read the fp32 currents from HBM (4 B per neuron-step) and
// write the spike / window bit planes (2 bits), HBM-bound at 4.25 B per neuron-step.
//   Equations (north_star; R7): c_t = d_c c_{t-1} + I_t;
//   v_t = d_v v_{t-1} (1 - o_{t-1}) + c_t; o_t = [v_t > V_th]; h_t = [|v_t - V_th| < window].
// Layout: I [T][B][N] fp32 (N innermost); bits / mask [T][B][W] u32, W = ceil(N / 32), bit n % 32 of
// word n / 32 (the library's batch-major spike planes).
#include "internal.h"

namespace spk {
namespace {

// A block owns one row b and 8 consecutive output words (256 neurons): warp k scans word k (its 32
// lanes = neurons request a 16-step chunk of currents at once — coalesced 128-byte rows — then run
// the fused epilogue's operation sequence, lif_step) and lane 0 parks each step's two ballot words
// in shared memory; per 32-step chunk the block then stores the 8 words of each (step, row)
// together: one full 32-byte sector per plane (a word per store left partial sectors and ran at
// 0.31 of the copy peak; one warp walking its 8 words in turn was latency-bound at 0.25). r02 at the
// configs[4] hidden-layer size (T 16, B 65 536, N 1024: 4.56 GB): 1.30 ms, 0.54 of the copy peak.
constexpr int kScanKW = 8, kScanTC = 32;
__global__ void __launch_bounds__(256) lif_scan_fwd_kernel(const float* __restrict__ I, int T, int B, int N, int W,
                                                           LifConst kc, uint32_t* __restrict__ bits,
                                                           uint32_t* __restrict__ mask) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t sw[2][kScanTC][kScanKW];
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WB = (W + kScanKW - 1) / kScanKW;
  const long long tasks = (long long)B * WB;
  const size_t tstride = (size_t)B * N;
  if (T <= 16) {
    // the common case (configs: T = 5, 16): one chunk per task, the next task's currents requested
    // while this one is scanned (its latency hidden behind the scan and the stores)
    auto load = [&](long long tq, float (&x)[16]) {
      const int b = (int)(tq / WB), wb = (int)(tq - (long long)b * WB);
      const int n = (wb * kScanKW + k) * 32 + lane;
      const float* ip = I + (size_t)b * N + (n < N ? n : 0);
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = (j < T && n < N) ? __ldcs(ip + (size_t)j * tstride) : 0.f;
    };
    float xa[16], xb[16];
    long long tk = blockIdx.x;
    if (tk < tasks) load(tk, xa);
    for (; tk < tasks; tk += gridDim.x) {
      const long long tn = tk + gridDim.x;
      if (tn < tasks) load(tn, xb);
      const int b = (int)(tk / WB), wb = (int)(tk - (long long)b * WB);
      const bool nv = (wb * kScanKW + k) * 32 + lane < N;
      float c = 0.f, v = 0.f;
      bool o = false, h = false;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j >= T) break;
        lif_step(kc, xa[j], c, v, o, h);
        const uint32_t ob = __ballot_sync(0xffffffffu, o && nv);
        const uint32_t hb = __ballot_sync(0xffffffffu, h && nv);
        if (lane == 0) {
          sw[0][j][k] = ob;
          sw[1][j][k] = hb;
        }
      }
      __syncthreads();
      for (int e = threadIdx.x; e < 2 * T * kScanKW; e += blockDim.x) {
        const int pl = e / (T * kScanKW), r = e - pl * T * kScanKW, j = r / kScanKW, kw = r - j * kScanKW;
        const int w = wb * kScanKW + kw;
        if (w < W) (pl ? mask : bits)[((size_t)j * B + b) * W + w] = sw[pl][j][kw];
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) xa[j] = xb[j];
    }
    return;
  }
  for (long long tk = blockIdx.x; tk < tasks; tk += gridDim.x) {
    const int b = (int)(tk / WB), wb = (int)(tk - (long long)b * WB);
    const int n = (wb * kScanKW + k) * 32 + lane;
    const bool nv = n < N;
    const float* ip = I + (size_t)b * N + (nv ? n : 0);
    float c = 0.f, v = 0.f;
    bool o = false, h = false;
    for (int t0 = 0; t0 < T; t0 += kScanTC) {
      const int nt = T - t0 < kScanTC ? T - t0 : kScanTC;
      for (int j0 = 0; j0 < nt; j0 += 16) {
        float x[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = (j0 + j < nt && nv) ? __ldcs(ip + (size_t)(t0 + j0 + j) * tstride) : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j0 + j >= nt) break;
          lif_step(kc, x[j], c, v, o, h);
          const uint32_t ob = __ballot_sync(0xffffffffu, o && nv);
          const uint32_t hb = __ballot_sync(0xffffffffu, h && nv);
          if (lane == 0) {
            sw[0][j0 + j][k] = ob;
            sw[1][j0 + j][k] = hb;
          }
        }
      }
      __syncthreads();
      // thread = (plane, step, word): 8 consecutive threads store one (step, row)'s 8 words
      for (int e = threadIdx.x; e < 2 * nt * kScanKW; e += blockDim.x) {
        const int pl = e / (nt * kScanKW), r = e - pl * nt * kScanKW, j = r / kScanKW, kw = r - j * kScanKW;
        const int w = wb * kScanKW + kw;
        if (w < W) (pl ? mask : bits)[((size_t)(t0 + j) * B + b) * W + w] = sw[pl][j][kw];
      }
      __syncthreads();
    }
  }
}

}  // namespace
}  // namespace spk

using namespace spk;

extern "C" int spikerl_lif_scan_forward(const float* I, int T, int B, int N, float d_c, float d_v, float v_th,
                                        float window, uint32_t* bits, uint32_t* mask, spikerl_stream_t stream) {
  if (!I || !bits || !mask || T < 1 || B < 1 || N < 1) {
    set_error("spikerl_lif_scan_forward: bad arguments");
    return SPIKERL_E_ARG;
  }
  const int W = (N + 31) / 32;
  cudaStream_t st = (cudaStream_t)stream;
  ProfScope ps_("lif_scan_ablation", PB_HBM, 0.0, (double)T * B * (4.0 * N + 8.0 * W), st);
  const long long blocks = (long long)B * ((W + 7) / 8);   // one task (row, 8 words) per block
  const int grid = (int)(blocks < (long long)num_sms() * 8 ? blocks : (long long)num_sms() * 8);
  pdl(lif_scan_fwd_kernel, grid, 256, 0, st)(I, T, B, N, W, LifConst{d_c, d_v, v_th, window}, bits, mask);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}
