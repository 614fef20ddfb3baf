// k_encoder.cu — K1: Gaussian receptive-field stimulation + deterministic soft-reset encoder
// spikes, written straight into the bit-packed spike plane of layer 0.
//   PAPER.md:131 (§III-A "populations use Gaussian distributions to transform continuous input
//   values into spike trains"); north_star ("deterministic soft-reset encoder spikes");
//   SPEC.md:123-140; R4 (fp64 exponent, RNE to fp32, no FTZ) and R5 (acc >= 1).
// A warp owns 32 consecutive encoder neurons k, so one __ballot_sync per timestep yields exactly
// one u32 word of bits0[t][b][:]. Each thread keeps its neuron's constants (obs index, mu, the
// fp64 2 sigma^2) in registers and walks a strided set of batch rows, prefetching the next
// observation, so the grid is a few blocks per SM instead of one block per (b, 128 neurons).
#include "internal.h"

namespace spk {

// TT > 0: T == TT known at compile time (T <= 32), the time loop fully unrolled: per step one
// FADD, FSETP, predicated FADD, VOTE and a lane select (ncu r01: the runtime-T loop cost 14
// instructions per step and 59% of the kernel; a lane-0 shared-memory variant measured slower).
// TT == 0: any T, in chunks of 32 steps.
template <int TT>
__global__ void __launch_bounds__(256) enc_fwd_kernel(int B, int S, int E, int K0, int W0, int T,
                                                      const float* __restrict__ obs,
                                                      const float* __restrict__ mu,
                                                      const float* __restrict__ sigma,
                                                      float* __restrict__ A_out,
                                                      uint32_t* __restrict__ bits0) {
  pdl_wait();
  pdl_trigger();
  const int k = blockIdx.y * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if ((k >> 5) >= W0) return;   // whole warp past the padded width
  const bool kv = k < K0;
  const int i = kv ? k / E : 0;
  const double m = kv ? (double)__ldg(mu + k) : 0.0;
  const double sg = kv ? (double)__ldg(sigma + k) : 1.0;
  const double den = __dmul_rn(2.0, __dmul_rn(sg, sg));
  // q / den as a correctly rounded quotient from the hoisted correctly rounded reciprocal:
  // q0 = RN(q inv) is within one ulp, r = q - den q0 is exact (FMA), RN(q0 + r inv) = RN(q / den)
  // (Markstein). Same value as __ddiv_rn(q, den) (the bit-exact encoder tests pin it against the
  // oracle's IEEE division) at 3 instead of ~12 double operations per element.
  const double inv = __ddiv_rn(1.0, den);
  const size_t tstride = (size_t)B * W0;
  const size_t arow = (size_t)gridDim.x * K0, brow = (size_t)gridDim.x * W0;   // per-iteration strides
  int b = blockIdx.x;
  float* ap = A_out + (size_t)b * K0 + k;
  uint32_t* out = bits0 + (size_t)b * W0 + (k >> 5) + (size_t)lane * tstride;
  float s_next = (kv && b < B) ? __ldg(obs + (size_t)b * S + i) : 0.f;
  for (; b < B; b += gridDim.x, ap += arow, out += brow) {
    const float s = s_next;
    const int bn = b + gridDim.x;
    if (kv && bn < B) s_next = __ldg(obs + (size_t)bn * S + i);
    float A = 0.0f;
    if (kv) {
      const double dd = __dsub_rn((double)s, m);
      const double q = __dmul_rn(dd, dd);
      const double q0 = __dmul_rn(q, inv);
      const double r = __fma_rn(-q0, den, q);
      A = (float)exp(-__fma_rn(r, inv, q0));  // RNE double -> float
      *ap = A;
    }
    float acc = 0.0f;
    if constexpr (TT > 0) {
      // lane t keeps the ballot word of timestep t; one store instruction for all T words
      uint32_t mine = 0;
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        acc = __fadd_rn(acc, A);
        const bool fire = acc >= 1.0f;
        if (fire) acc = __fsub_rn(acc, 1.0f);
        const uint32_t w = __ballot_sync(0xffffffffu, fire);
        mine = (lane == t) ? w : mine;
      }
      if (lane < TT) *out = mine;
    } else {
      for (int t0 = 0; t0 < T; t0 += 32) {
        const int n = T - t0 < 32 ? T - t0 : 32;
        uint32_t mine = 0;
        for (int j = 0; j < n; ++j) {
          acc = __fadd_rn(acc, A);
          const bool fire = acc >= 1.0f;
          if (fire) acc = __fsub_rn(acc, 1.0f);
          const uint32_t w = __ballot_sync(0xffffffffu, fire);
          mine = (lane == j) ? w : mine;
        }
        if (lane < n) out[(size_t)t0 * tstride] = mine;
      }
    }
  }
}

template <int TT>
static void enc_launch(dim3 grid, cudaStream_t st, const ActorDims& d, int B, const float* obs, const float* mu,
                       const float* sigma, float* A, uint32_t* bits0) {
  pdl((enc_fwd_kernel<TT>), grid, 256, 0, st)(B, d.S, d.E, d.K0, d.Wd[0], d.T, obs, mu, sigma, A, bits0);
}

int launch_enc_fwd(const ActorDims& d, int B, const float* obs, const float* mu, const float* sigma,
                   float* A, uint32_t* bits0, cudaStream_t st) {
  ProfScope ps_("enc_fwd", PB_HBM, 0.0, 4.0 * B * (d.S + d.K0 + (double)d.T * d.Wd[0]), st);
  // 256-thread blocks: the 8 warps of a block write 8 consecutive words (one full 32-byte sector)
  // of each bits0[t][b] row, instead of half sectors (ncu r01: 1.89 GB written for 1.49 GB).
  const int ky = (d.P[0] + 255) / 256;
  int bx = (148 * 8 + ky - 1) / ky;  // ~8 resident 256-thread blocks per SM in total
  if (bx > B) bx = B;
  if (bx < 1) bx = 1;
  dim3 grid(bx, ky);
  switch (d.T) {
#define SPK_ENC_T(n) \
  case n: enc_launch<n>(grid, st, d, B, obs, mu, sigma, A, bits0); break;
    SPK_ENC_T(1) SPK_ENC_T(2) SPK_ENC_T(3) SPK_ENC_T(4) SPK_ENC_T(5) SPK_ENC_T(6) SPK_ENC_T(8) SPK_ENC_T(10)
    SPK_ENC_T(12) SPK_ENC_T(16) SPK_ENC_T(20) SPK_ENC_T(24) SPK_ENC_T(32)
#undef SPK_ENC_T
    default: enc_launch<0>(grid, st, d, B, obs, mu, sigma, A, bits0); break;
  }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

}  // namespace spk
