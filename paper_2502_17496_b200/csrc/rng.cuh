// rng.cuh — counter-based Philox4x32-10 keyed by (seed, rank), the uniform / normal maps and the
// purposes of the TD3 path's random draws (replay indices, target-policy noise, replay fill). Shared
// by k_replay.cu and the decoder launch that applies the target-policy smoothing.
#pragma once
#include <cstdint>

namespace spk {

struct Philox {
  __device__ static uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  __device__ static uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

__device__ __forceinline__ uint2 philox_key(unsigned long long seed, int rank) {
  return make_uint2((uint32_t)seed, (uint32_t)(seed >> 32) ^ (0x85EBCA6Bu * (uint32_t)(rank + 1)));
}
__device__ __forceinline__ float u01(uint32_t x) {  // (0, 1]
  return ((float)(x >> 8) + 1.0f) * (1.0f / 16777216.0f);
}
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
  const float r = sqrtf(-2.0f * logf(u01(a)));
  float s, c;
  sincospif(2.0f * u01(b), &s, &c);
  return make_float2(r * c, r * s);
}

enum Purpose : uint32_t { P_INDEX = 1, P_NOISE = 2, P_FILL = 3 };

// TD3 target-policy smoothing of element i of the target action:
// a~ = clip(a + clip(eps, -c, c), -1, 1), eps = sigma N(0, 1) from the Philox pair (i / 2) at the
// update's counter value (or the injected noise[i]).
__device__ __forceinline__ float smooth_action(float a, int i, const float* noise, float sigma, float clip,
                                               unsigned long long seed, int rank, unsigned long long ctr) {
  float eps;
  if (noise) {
    eps = noise[i];
  } else {
    const uint4 x = Philox::gen(make_uint4((uint32_t)(i >> 1), P_NOISE, (uint32_t)ctr, (uint32_t)(ctr >> 32)),
                                philox_key(seed, rank));
    const float2 z = box_muller(x.x, x.y);
    eps = sigma * ((i & 1) ? z.y : z.x);
  }
  eps = fminf(fmaxf(eps, -clip), clip);
  return fminf(fmaxf(__fadd_rn(a, eps), -1.0f), 1.0f);
}


}  // namespace spk
