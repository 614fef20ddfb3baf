// k_encoder.cu — K1: Gaussian receptive-field stimulation + deterministic soft-reset encoder
// spikes, written straight into the bit-packed spike plane of layer 0.
//   PAPER.md:131 (§III-A "populations use Gaussian distributions to transform continuous input
//   values into spike trains"); north_star ("deterministic soft-reset encoder spikes");
//   SPEC.md:123-140; R4 (fp64 exponent, RNE to fp32, no FTZ) and R5 (acc >= 1).
//
// Design. A thread owns one encoder neuron k (its constants mu, den = 2 sigma^2 and 1/den stay in
// registers) and a warp 32 consecutive neurons, i.e. one u32 word of every bits0[t][b] row; a
// block of 8 warps owns 256 neurons and walks tiles of R batch rows:
//   1. every element: A = RN32(exp(-(q/den))) in fp64 (Markstein-corrected quotient from the
//      hoisted reciprocal), stored coalesced;
//   2. the accumulate-and-fire loop (R5) runs only for the elements that can fire at all. With the
//      paper's receptive fields (sigma = 0.15 against a mu spacing of 0.667) about 90% of the
//      elements have A < 1/T, yet every warp of 32 consecutive neurons holds a few that do not, so
//      a per-row loop over the warp (one ballot per step) paid the T steps for all 32 lanes. Instead
//      each warp queues its (row, lane, A) candidates in shared memory and then runs the loop with
//      one candidate per lane, OR-ing the spikes into its own words of the tile (shared atomics);
//   3. the tile's words leave with full 32-byte sectors (the 8 warps' words of one (t, row) are
//      adjacent).
// No-fire bound (conservative, so skipping is exact): no spike at any t <= T when
// A < thr = 1 / (T (1 + T 2^-22)): the fp32 accumulator after t steps without a spike is at most
// t A (1 + 2^-24)^t < 1.
#include "internal.h"

namespace spk {

namespace {
constexpr int kEncThreads = 256;   // = neurons per tile (8 warps, 8 words)
constexpr int kEncWarps = kEncThreads / 32;

// dynamic shared memory for R rows and T steps: bit words [T][R][8] + per-warp queues of R*32
// (entry = row << 5 | lane as u16, and the element's A)
// SPK (spikes only): queue entries are the fp64 s - mu (8 B) and the u16 entry; plus per-warp fp64
// den / 1/den of its 32 neurons
inline size_t enc_smem_bytes(int R, int T, bool spk = false) {
  return (size_t)T * R * kEncWarps * 4 + (size_t)kEncWarps * R * 32 * ((spk ? 8 : 4) + 2) +
         (spk ? (size_t)kEncWarps * 32 * 16 : 0);
}
}  // namespace

// exp(-z) in fp64 for 0 <= z <= 110 (within one ulp of libm's exp over the encoder's range, checked
// bit-for-bit after the RNE to fp32 by the encoder parity tests). z = n ln2 - r with n = round(z / ln2)
// (the 1.5 * 2^52 shifter), r from a two-part ln2 (Cody-Waite; ln2_hi has 21 trailing zero bits so
// n ln2_hi is exact), exp(r) by the degree-13 Taylor polynomial in Horner form (|r| <= ln2/2: the
// remainder is below 5e-18), 2^-n added to the exponent (the result stays a normal double). The
// library exp spent ~35 instructions per element on range checks this range never needs. The
// coefficients are read once per thread into registers (ncu r02: taken from the constant bank they
// cost 6 LDCU.128 + 4 UMOV per element, 10 % of the kernel's instructions).
__device__ const double kExpC[12] = {
    1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08, 2.755731922398589e-07,
    2.7557319223985893e-06, 2.48015873015873e-05,  0.0001984126984126984, 0.001388888888888889,
    0.008333333333333333,   0.041666666666666664,  0.16666666666666666,   0.5};
struct ExpCoefs {
  double c[12], ln2_hi, ln2_lo;
  __device__ __forceinline__ void load() {
#pragma unroll
    for (int j = 0; j < 12; ++j) c[j] = __ldg(kExpC + j);
    ln2_hi = -0x1.62e42fee00000p-1;
    ln2_lo = -0x1.a39ef35793c76p-33;
  }
};
__device__ __forceinline__ double exp_neg(double z, const ExpCoefs& k) {
  z = fmin(z, 110.0);                                               // exp(-110) still rounds to fp32 0
  const double t = __fma_rn(-z, 1.4426950408889634, 6755399441055744.0);
  const double nd = __dsub_rn(t, 6755399441055744.0);               // round(-z / ln2), exactly
  double r = __fma_rn(nd, k.ln2_hi, -z);                            // -z - n ln2_hi (exact)
  r = __fma_rn(nd, k.ln2_lo, r);                                    //   - n ln2_lo
  double p = k.c[0];
#pragma unroll
  for (int j = 1; j < 12; ++j) p = __fma_rn(p, r, k.c[j]);
  p = __fma_rn(p, r, 1.0);
  p = __fma_rn(p, r, 1.0);
  return __longlong_as_double(__double_as_longlong(p) + ((long long)__double2loint(t) << 52));
}

// TT > 0: T == TT at compile time (unrolled accumulate-and-fire); TT == 0: runtime T. RR rows per
// tile (compile time: the tile index math is shifts).
// SPK (spikes only; forward passes without a backward, e.g. TD3's target actor): A is not stored, so
// only the elements that can fire need their exact A. An fp32 screen z32 = (s - mu)^2 / (2 sigma^2)
// against zskip (host-derived, conservative: z32 > zskip implies A < thr for the fp64 A, whatever the
// fp32 rounding) drops the rest (~90 % with the paper's receptive fields); the survivors are queued
// per warp with their fp64 s - mu and get the same fp64 A and fire loop as the full kernel, one per
// lane, so the spikes are bitwise those of the full kernel (tested).
template <int TT, int RR, bool SPK = false>
__global__ void __launch_bounds__(kEncThreads) enc_fwd_kernel(int B, int S, int E, int K0, int W0, int T,
                                                              float thr, const float* __restrict__ obs,
                                                              const float* __restrict__ mu,
                                                              const float* __restrict__ sigma,
                                                              float* __restrict__ A_out,
                                                              uint32_t* __restrict__ bits0, float zskip) {
  extern __shared__ __align__(16) unsigned char esm[];
  const int Tn = TT > 0 ? TT : T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = Tn * RR * kEncWarps;                                              // words of a tile
  uint32_t* w_sh = reinterpret_cast<uint32_t*>(esm);                               // [T][RR][8]
  constexpr int QB = SPK ? 8 : 4;                                                  // queue value bytes
  float* qA = reinterpret_cast<float*>(w_sh + nw) + warp * RR * 32;                // per-warp queue (full)
  double* qd = reinterpret_cast<double*>(w_sh + nw) + warp * RR * 32;              // per-warp queue (SPK)
  uint16_t* qe = reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(w_sh + nw) + kEncWarps * RR * 32 * QB) +
                 warp * RR * 32;
  double* nk_sh = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(w_sh + nw) +
                                            kEncWarps * RR * 32 * (QB + 2)) + warp * 64;   // SPK: den, inv of 32 lanes
  const uint32_t lt = (1u << lane) - 1u;
  const int k = blockIdx.y * kEncThreads + tid;
  const bool kv = k < K0;
  const int i = kv ? k / E : 0;
  const int w0 = blockIdx.y * kEncWarps;
  const int tstep = gridDim.x * RR;
  pdl_wait();     // mu / sigma may have just been written by the optimiser
  pdl_trigger();
  // per-neuron constants (fp64, as the oracle's op sequence R4): den = 2 sigma^2 and its reciprocal
  const double m = kv ? (double)__ldg(mu + k) : 0.0;
  const double sg = kv ? (double)__ldg(sigma + k) : 1.0;
  const double den = __dmul_rn(2.0, __dmul_rn(sg, sg));
  const double inv = __ddiv_rn(1.0, den);
  ExpCoefs kx;
  kx.load();
  const float m32 = kv ? __ldg(mu + k) : 0.0f, inv32 = (float)inv;
  if constexpr (SPK) {
    nk_sh[lane] = den;
    nk_sh[32 + lane] = inv;
    __syncwarp();
  }
  // the observation values of a tile are requested one tile ahead (ncu r02: loaded at the tile
  // start, their latency was the kernel's top stall); rows past B read row B - 1 and are not stored
  const float* op = obs + i;
  float sv[RR];
#pragma unroll
  for (int r = 0; r < RR; ++r) sv[r] = __ldg(op + (size_t)min((int)blockIdx.x * RR + r, B - 1) * S);
  for (int b0 = blockIdx.x * RR; b0 < B; b0 += tstep) {
    for (int j = tid; j < nw / 4; j += kEncThreads) reinterpret_cast<uint4*>(w_sh)[j] = make_uint4(0u, 0u, 0u, 0u);
    float svn[RR];
#pragma unroll
    for (int r = 0; r < RR; ++r) svn[r] = __ldg(op + (size_t)min(b0 + tstep + r, B - 1) * S);
    __syncthreads();   // zeroed words; the previous tile's words have been written out
    // ---- 1. stimulation A for every element of the tile, candidates queued per warp. Padding
    // neurons / rows compute on clamped inputs and only their stores are predicated off (no
    // divergent branch around the fp64 chain).
    int cnt = 0;
    if constexpr (SPK) {
      // fp32 screen; survivors queued with their fp64 s - mu
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const float d32 = __fsub_rn(sv[r], m32);
        const bool need = kv && b0 + r < B && !(__fmul_rn(__fmul_rn(d32, d32), inv32) > zskip);
        const uint32_t bal = __ballot_sync(0xffffffffu, need);
        if (need) {
          const int j = cnt + __popc(bal & lt);
          qd[j] = __dsub_rn((double)sv[r], m);
          qe[j] = (uint16_t)((r << 5) | lane);
        }
        cnt += __popc(bal);
      }
      __syncwarp();
      // the exact A of each survivor (its own neuron's constants) and, where A >= thr, the fire loop
      for (int j = lane; j < cnt; j += 32) {
        const int e = qe[j];
        const double dd = qd[j], dn = nk_sh[e & 31], iv = nk_sh[32 + (e & 31)];
        const double q = __dmul_rn(dd, dd);
        const double q0 = __dmul_rn(q, iv);
        const double rr = __fma_rn(-q0, dn, q);
        const float A = (float)exp_neg(__fma_rn(rr, iv, q0), kx);
        if (A >= thr) {
          const uint32_t bit = 1u << (e & 31);
          uint32_t* wp = w_sh + (e >> 5) * kEncWarps + warp;
          float acc = 0.0f;
#pragma unroll
          for (int st = 0; st < (TT > 0 ? TT : Tn); ++st) {
            acc = __fadd_rn(acc, A);
            if (acc >= 1.0f) {
              acc = __fsub_rn(acc, 1.0f);
              atomicOr(wp + st * RR * kEncWarps, bit);
            }
          }
        }
      }
    }
    float* ap = A_out + (size_t)b0 * K0 + k;
#pragma unroll
    for (int r = 0; r < RR && !SPK; ++r, ap += K0) {
      const bool live = kv && b0 + r < B;
      const double dd = __dsub_rn((double)sv[r], m);
      const double q = __dmul_rn(dd, dd);
      // q / den as a correctly rounded quotient from the correctly rounded reciprocal:
      // q0 = RN(q inv) is within one ulp, r = q - den q0 is exact (FMA), RN(q0 + r inv) = RN(q / den)
      // (Markstein); the bit-exact encoder tests pin it against the oracle's IEEE division
      const double q0 = __dmul_rn(q, inv);
      const double rr = __fma_rn(-q0, den, q);
      const float A = (float)exp_neg(__fma_rn(rr, inv, q0), kx);   // RNE double -> float
      if (live) *ap = A;
      const bool cand = live && A >= thr;
      const uint32_t bal = __ballot_sync(0xffffffffu, cand);
      if (cand) {
        const int j = cnt + __popc(bal & lt);
        qA[j] = A;
        qe[j] = (uint16_t)((r << 5) | lane);
      }
      cnt += __popc(bal);
    }
    __syncwarp();
    // ---- 2. accumulate-and-fire (R5: fp32 acc += A; spike iff acc >= 1; acc -= 1), one candidate
    // per lane, each spike OR-ed into its (t, row) word of the warp (shared atomics). ncu r02: a
    // branch-free variant that assembled whole words per lane from T-bit trains was 45 % slower
    // (dependent shared loads)
    for (int j = lane; j < cnt && !SPK; j += 32) {
      const float A = qA[j];
      const int e = qe[j];
      const uint32_t bit = 1u << (e & 31);
      uint32_t* wp = w_sh + (e >> 5) * kEncWarps + warp;   // + step * RR * 8
      float acc = 0.0f;
#pragma unroll
      for (int st = 0; st < (TT > 0 ? TT : Tn); ++st) {
        acc = __fadd_rn(acc, A);
        if (acc >= 1.0f) {
          acc = __fsub_rn(acc, 1.0f);
          atomicOr(wp + st * RR * kEncWarps, bit);
        }
      }
    }
    __syncthreads();
    // ---- 3. the tile's bit words: the 8 words of one (t, row) are one 32-byte sector, written as
    // two 16-byte stores (W0 = P0 / 32 and w0 are multiples of 4 words)
    {
      const int q = tid & 1, r = (tid >> 1) % RR;   // this thread's quarter-sector and row
      const int b = b0 + r;
      if (b < B && w0 + 4 * q < W0) {
        uint4* gp = reinterpret_cast<uint4*>(bits0 + ((size_t)b * W0 + w0 + 4 * q));
        const size_t gstep = (size_t)B * W0 / 4;          // one step t, in uint4
        constexpr int kPer = 2 * RR;                     // threads per step
        for (int st = tid / kPer; st < Tn; st += kEncThreads / kPer)
          gp[(size_t)st * gstep] = reinterpret_cast<const uint4*>(w_sh)[(st * RR + r) * 2 + q];
      }
    }
#pragma unroll
    for (int r = 0; r < RR; ++r) sv[r] = svn[r];
  }
}

template <int TT, int RR, bool SPK>
static int enc_launch(cudaStream_t st, const ActorDims& d, int B, float thr, float zskip, const float* obs,
                      const float* mu, const float* sigma, float* A, uint32_t* bits0) {
  const size_t smem = enc_smem_bytes(RR, d.T, SPK);
  if (smem > 160 * 1024) { set_error("encoder: T = %d too long for the shared tile", d.T); return SPIKERL_E_UNSUPPORTED; }
  SPK_SMEM_ATTR((enc_fwd_kernel<TT, RR, SPK>), 160 * 1024);   // an upper bound; each launch asks for its own size
  // one wave of resident blocks (a second partial wave of row-walking blocks would double the time)
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, enc_fwd_kernel<TT, RR, SPK>, kEncThreads, smem) !=
          cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const int ky = (d.P[0] + kEncThreads - 1) / kEncThreads;
  int bx = num_sms() * per_sm / ky;
  if (bx > cdiv(B, RR)) bx = cdiv(B, RR);
  if (bx < 1) bx = 1;
  pdl((enc_fwd_kernel<TT, RR, SPK>), dim3((unsigned)bx, (unsigned)ky), kEncThreads, smem, st)(
      B, d.S, d.E, d.K0, d.Wd[0], d.T, thr, obs, mu, sigma, A, bits0, zskip);
  return SPIKERL_OK;
}

// A == NULL: spikes only (no stimulation plane; see enc_fwd_kernel's SPK)
int launch_enc_fwd(const ActorDims& d, int B, const float* obs, const float* mu, const float* sigma,
                   float* A, uint32_t* bits0, cudaStream_t st) {
  ProfScope ps_(A ? "enc_fwd" : "enc_fwd_spikes", PB_HBM, 0.0,
                4.0 * B * (d.S + (A ? d.K0 : 0) + (double)d.T * d.Wd[0]), st);
  // no-fire bound (see the file header), rounded down to fp32
  const double thr64 = 1.0 / ((double)d.T * (1.0 + (double)d.T * 0x1p-22));
  float thr = (float)thr64;
  if ((double)thr > thr64) thr = nextafterf(thr, 0.0f);
  // spikes-only screen: z32 > zskip implies A < thr. A = RN32(exp64(-z64)) < thr once the exact z
  // exceeds -ln(thr) + 2^-23; z32 (three fp32 roundings of (s - mu)^2 / (2 sigma^2)) is within
  // 6 * 2^-24 relative of the exact z; both margins are taken ~10x wide, and zskip rounded up
  const double zs64 = (-log((double)thr) + 1e-6) * (1.0 + 1e-6);
  float zskip = (float)zs64;
  if ((double)zskip < zs64) zskip = nextafterf(zskip, INFINITY);
  // 8 rows per tile for the compiled T (a T = 32 tile is ~20 KB: eight resident blocks); 2 rows
  // for any other T (up to 255: 16 KB of words)
  switch (d.T) {
#define SPK_ENC_T(n)                                                                                    \
  case n:                                                                                               \
    if (A) SPK_TRY((enc_launch<n, 8, false>(st, d, B, thr, zskip, obs, mu, sigma, A, bits0)));          \
    else SPK_TRY((enc_launch<n, 8, true>(st, d, B, thr, zskip, obs, mu, sigma, A, bits0)));             \
    break;
    SPK_ENC_T(1) SPK_ENC_T(2) SPK_ENC_T(3) SPK_ENC_T(4) SPK_ENC_T(5) SPK_ENC_T(8) SPK_ENC_T(10) SPK_ENC_T(16)
    SPK_ENC_T(32)
#undef SPK_ENC_T
    default:
      if (A) SPK_TRY((enc_launch<0, 2, false>(st, d, B, thr, zskip, obs, mu, sigma, A, bits0)));
      else SPK_TRY((enc_launch<0, 2, true>(st, d, B, thr, zskip, obs, mu, sigma, A, bits0)));
      break;
  }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

}  // namespace spk
