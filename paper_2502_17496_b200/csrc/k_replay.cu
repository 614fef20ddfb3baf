// k_replay.cu — K9: device-resident replay sampling and the TD3 target arithmetic.
//   Replay: uniform sampling with replacement; synthetic shard recipe of
//   configs[1] (s, s' ~ N(0,1) clipped +-5; a ~ U[-1,1]; r ~ N(0,1); done ~ Bernoulli(0.01)).
//   Target smoothing and target: SPEC.md:235-243 (a~ = clip(pi'(s') + clip(eps,-c,c), -1, 1);
//   y = r + gamma (1 - done) min(Q1', Q2')).
// Random numbers: counter-based Philox4x32-10 keyed by (seed, rank); the counter lives on the
// device so a captured CUDA graph draws fresh numbers on every replay.
#include "internal.h"
#include "rng.cuh"

namespace spk {

// one warp per sampled row: lane 0 draws the index, the warp copies the row's columns
// one warp per sampled row: lane 0 draws the index, the warp copies the row's columns. Up to two
// minibatches (the two updates of a pair) in one launch: warp w < nslots B samples row w % B of
// slot w / B, whose draws use the device counter + slot (the second update of a pair draws with the
// value the first one advances to); block 0 snapshots those values for the target-noise launches.
__global__ void replay_gather_kernel(int B, int S, int A, const float* __restrict__ rs,
                                     const float* __restrict__ ra, const float* __restrict__ rr,
                                     const float* __restrict__ rs2, const float* __restrict__ rd,
                                     long long N, unsigned long long seed, int rank,
                                     const unsigned long long* __restrict__ counter, const GatherSlots gs) {
  pdl_wait();
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x < gs.n) {
    unsigned long long* const sn = threadIdx.x ? gs.snap[1] : gs.snap[0];
    if (sn) *sn = *counter + threadIdx.x;
  }
  if (warp >= gs.n * B) return;
  const int slot = warp / B, row = warp - slot * B;
  // slot pointers by selection (a runtime-indexed kernel-parameter array goes through local memory)
  const bool s1 = slot != 0;
  const long long* const idx = s1 ? gs.idx[1] : gs.idx[0];
  long long i = 0;
  if (lane == 0) {
    if (idx) {
      i = idx[row];
    } else {
      const unsigned long long ctr = *counter + slot;
      const uint4 x = Philox::gen(make_uint4((uint32_t)row, P_INDEX, (uint32_t)ctr, (uint32_t)(ctr >> 32)),
                                  philox_key(seed, rank));
      const unsigned long long u = ((unsigned long long)x.x << 32) | x.y;
      i = (long long)(u % (unsigned long long)N);
    }
  }
  i = __shfl_sync(0xffffffffu, i, 0);
  float* const s = s1 ? gs.s[1] : gs.s[0];
  float* const s2 = s1 ? gs.s2[1] : gs.s2[0];
  float* const a = s1 ? gs.a[1] : gs.a[0];
  const float* const src_s = rs + (size_t)i * S;
  const float* const src_s2 = rs2 + (size_t)i * S;
  float* const dst_s = s + (size_t)row * S;
  float* const dst_s2 = s2 + (size_t)row * S;
  // 16-byte copies when the rows are 16-byte aligned (S % 4 == 0 and aligned bases: configs[3]'s 376)
  if (((S & 3) | (((uintptr_t)rs | (uintptr_t)rs2 | (uintptr_t)s | (uintptr_t)s2) & 15)) == 0) {
    const float4* ps = reinterpret_cast<const float4*>(src_s);
    const float4* ps2 = reinterpret_cast<const float4*>(src_s2);
    float4* qs = reinterpret_cast<float4*>(dst_s);
    float4* qs2 = reinterpret_cast<float4*>(dst_s2);
    for (int c = lane; c < (S >> 2); c += 32) {
      const float4 x = __ldg(ps + c), y = __ldg(ps2 + c);
      qs[c] = x;
      qs2[c] = y;
    }
  } else {
    for (int c = lane; c < S; c += 32) {
      dst_s[c] = src_s[c];
      dst_s2[c] = src_s2[c];
    }
  }
  for (int c = lane; c < A; c += 32) a[(size_t)row * A + c] = ra[(size_t)i * A + c];
  if (lane == 0) {
    (s1 ? gs.r[1] : gs.r[0])[row] = rr[i];
    (s1 ? gs.d[1] : gs.d[0])[row] = rd[i];
  }
}

int launch_replay_gather(int B, int S, int A, const float* rs, const float* ra, const float* rr,
                         const float* rs2, const float* rd, long long N, unsigned long long seed, int rank,
                         const unsigned long long* counter, const GatherSlots& gs, cudaStream_t st) {
  ProfScope ps_("replay_gather", PB_LATENCY, 0.0, 8.0 * gs.n * B * (2.0 * S + A + 2), st);
  pdl(replay_gather_kernel, cdiv((long long)gs.n * B * 32, 256), 256, 0, st)(B, S, A, rs, ra, rr, rs2, rd, N, seed,
                                                                            rank, counter, gs);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

__global__ void scale_kernel(float* x, size_t n, float s) {
  pdl_wait();
  pdl_trigger();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] = __fmul_rn(x[i], s);
}

int launch_scale(float* x, size_t n, float s, cudaStream_t st) {
  pdl(scale_kernel, cdiv((long long)n, 256) < 1184 ? cdiv((long long)n, 256) : 1184, 256, 0, st)(x, n, s);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// synthetic shard fill (configs[1] distributions)
__global__ void replay_fill_kernel(float* s, float* a, float* r, float* s2, float* d, long long n,
                                   int S, int A, float p_done, unsigned long long seed, int rank) {
  pdl_wait();
  pdl_trigger();
  const long long stride = (long long)gridDim.x * blockDim.x;
  const uint2 key = philox_key(seed, rank);
  const long long per = 2LL * S + A + 2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * per; e += stride) {
    const uint4 x = Philox::gen(make_uint4((uint32_t)e, P_FILL, (uint32_t)(e >> 32), 0u), key);
    const long long row = e / per;
    const int c = (int)(e % per);
    const float z = box_muller(x.x, x.y).x;
    if (c < S) s[row * S + c] = fminf(fmaxf(z, -5.f), 5.f);
    else if (c < 2 * S) s2[row * S + (c - S)] = fminf(fmaxf(z, -5.f), 5.f);
    else if (c < 2 * S + A) a[row * A + (c - 2 * S)] = 2.0f * u01(x.z) - 1.0f;
    else if (c == 2 * S + A) r[row] = z;
    else d[row] = u01(x.w) <= p_done ? 1.0f : 0.0f;
  }
}

}  // namespace spk

extern "C" int spikerl_replay_fill(float* s, float* a, float* r, float* s2, float* d, long long n,
                                   int obs_dim, int act_dim, float p_done, unsigned long long seed,
                                   int rank, spikerl_stream_t stream) {
  if (!s || !a || !r || !s2 || !d || n < 1 || obs_dim < 1 || act_dim < 1) {
    spk::set_error("spikerl_replay_fill: bad arguments");
    return SPIKERL_E_ARG;
  }
  spk::pdl(spk::replay_fill_kernel, 148 * 8, 256, 0, (cudaStream_t)stream)(s, a, r, s2, d, n, obs_dim, act_dim,
                                                                      p_done, seed, rank);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}
