// k_critic_mma.cu — K8, bf16 twin critic on warp-level tensor cores (mma.sync m16n8k16 bf16 ->
// fp32). The critic ("deep critic network"; configs[1] 23->256->256->1) is
// latency-bound at the TD3 batch sizes: the whole forward of both critics is one
// launch (a CTA = 16 batch rows of one critic, hidden activations stay in shared memory), the
// data backward is one launch, the weight gradients are one GEMM launch plus one reduction launch.
// Rounding points follow DESIGN.md R20 exactly as the oracle does: x, h1, h2, dz2, dz1 and the
// weights are bf16 where they enter a contraction; pre-activations, Q, losses and gradients fp32.
// Operand layouts (all k-contiguous so every fragment load is one 32-bit word):
//   forward L1  A = X [16][in_p] (smem)      B = W1p [H1][in_p]   (bf16 copy, rows zero-padded)
//   forward L2  A = h1 [16][H1] (smem)       B = W2  [H2][H1]
//   dH1         A = dz2 [16][H2] (smem)      B = W2T [H1][H2]
//   dQ1/da      A = dz1 [16][H1] (smem)      B = W1T [in_p+32][H1]
//   dW2         A = dZ2T [H2][Bp]            B = H1T [H1][Bp]
//   dW1         A = dZ1T [H1][Bp]            B = XT  [in_q][Bp]
#include "adam_body.cuh"
#include "rng.cuh"

namespace spk {

namespace {

constexpr int RB = 16;       // batch rows per CTA (the MMA M)
constexpr int HW = 256;      // hidden width handled by the MMA path (4 warps x 8 n-tiles x 8)
constexpr int SPAD = 8;      // smem row padding (bf16) -> conflict-free fragment loads

__device__ __forceinline__ uint32_t ld32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// acc[nt] += A[16 x K] * B^T, A rows k-contiguous (lda), B = NT*8 rows (n) k-contiguous (ldb).
// Fragments of the next D k-steps are kept in flight in registers (static rotation), so the
// L2 latency of the weight / activation loads overlaps the MMAs of earlier k-steps.
template <int NT, int D = 4>
__device__ __forceinline__ void warp_mma(float (&acc)[NT][4], const __nv_bfloat16* A, int lda,
                                         const __nv_bfloat16* Bm, long long ldb, int K) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const __nv_bfloat16* a0 = A + g * lda + 2 * t;
  const __nv_bfloat16* a1 = A + (g + 8) * lda + 2 * t;
  const __nv_bfloat16* bp = Bm + g * ldb + 2 * t;
  uint32_t a[D][4], b[D][NT][2];
  auto load = [&](uint32_t (&as)[4], uint32_t (&bs)[NT][2], int k0) {
    if (k0 < K) {
      as[0] = ld32(a0 + k0); as[1] = ld32(a1 + k0); as[2] = ld32(a0 + k0 + 8); as[3] = ld32(a1 + k0 + 8);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        bs[nt][0] = __ldg(reinterpret_cast<const unsigned int*>(bp + nt * 8 * ldb + k0));
        bs[nt][1] = __ldg(reinterpret_cast<const unsigned int*>(bp + nt * 8 * ldb + k0 + 8));
      }
    }
  };
#pragma unroll
  for (int s = 0; s < D; ++s) load(a[s], b[s], s * 16);
  for (int k0 = 0; k0 < K; k0 += 16 * D) {
#pragma unroll
    for (int s = 0; s < D; ++s) {
      if (k0 + s * 16 < K) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mma16816(acc[nt], a[s], b[s][nt][0], b[s][nt][1]);
        load(a[s], b[s], k0 + (s + D) * 16);
      }
    }
  }
}

// Same contraction with B in shared memory too (rows n, k-contiguous, row stride ldb elements).
template <int NT>
__device__ __forceinline__ void warp_mma_ss(float (&acc)[NT][4], const __nv_bfloat16* A, int lda,
                                            const __nv_bfloat16* Bs, int ldb, int K) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const __nv_bfloat16* a0 = A + g * lda + 2 * t;
  const __nv_bfloat16* a1 = A + (g + 8) * lda + 2 * t;
  const __nv_bfloat16* bp = Bs + g * ldb + 2 * t;
#pragma unroll 4
  for (int k0 = 0; k0 < K; k0 += 16) {
    const uint32_t a[4] = {ld32(a0 + k0), ld32(a1 + k0), ld32(a0 + k0 + 8), ld32(a1 + k0 + 8)};
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
      mma16816(acc[nt], a, ld32(bp + nt * 8 * ldb + k0), ld32(bp + nt * 8 * ldb + k0 + 8));
  }
}

// A weight matrix [HW rows][K] bf16 staged into shared memory (row stride K + SPAD) by bulk
// copies (one per row, issued by warp 0 right after the PDL wait), completing on an mbarrier.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void stage_rows(__nv_bfloat16* dst, const __nv_bfloat16* src, int rows, int K, uint64_t* bar) {
  // every thread issues (at most) one row: a single warp issuing all of them stalled on the copy
  // queue and held up the whole CTA at the next barrier (trace r01)
  const uint32_t b = smem_addr(bar);
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"((uint32_t)(rows * K * 2)) : "memory");
  for (int r = threadIdx.x; r < rows; r += blockDim.x)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst + (size_t)r * (K + SPAD))),
                 "l"(src + (size_t)r * K), "r"((uint32_t)(K * 2)), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void stage_wait(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar))
      : "memory");
}
constexpr size_t kW2Smem = (size_t)HW * (HW + SPAD) * 2;   // staged W2 / W2T (135 KB)
constexpr size_t kFusedSmem = kW2Smem + (size_t)RB * (512 + SPAD) * 2;   // + the X tile of the fused kernels

// bf16 twin buffer: [2][P] (fp32 layout; P may be odd), then (from element blk_base(P), a multiple
// of 8 so every row is 16-byte aligned for bulk copies) one block per critic holding every operand
// the MMA path reads: W1p | W1T | W2T | W2
__host__ __device__ inline long long blk_base(long long P) { return (2 * P + 7) & ~7LL; }

struct MmaLayout {
  long long P, W1p, W1T, W2T, W2c, tb;
  int inp, inq;          // in rounded to 16 (K of L1) and to 64 (+32 rows of W1T / XT)
};

MmaLayout mma_layout(const CriticDims& c) {
  MmaLayout L;
  L.P = (long long)c.off[SPIKERL_CRITIC_NPARAM];
  L.inp = round_up(c.in, 16);
  L.inq = round_up(c.in, 64) + 32;
  L.W1p = 0;
  L.W1T = (long long)c.H1 * L.inp;
  L.W2T = L.W1T + (long long)L.inq * c.H1;
  L.W2c = L.W2T + (long long)c.H1 * c.H2;
  L.tb = L.W2c + (long long)c.H2 * c.H1;
  return L;
}

struct MmaWs {
  __nv_bfloat16 *XT, *H1T, *dZ2T, *dZ1T;   // [inq][Bp], [2][H][Bp] x3
  __nv_bfloat16* H2T;                      // [2][H][Bp] (tcgen05 path: h2 for dW3 and the dZ2 mask)
  float *Z1, *Z2, *Hh2, *q, *dq;           // [2][B][H] x3, [2][B] x2
  float* part;                             // [2][Bp/RB] loss partials
  unsigned int* ticket;
  float* wpart;                            // [splits][2][HW*HW + HW*inq] split-K weight-gradient partials
};

// Large batches: the weight-gradient GEMMs (K = batch) run as 64 x 128 tiles split over K (the
// 16 x 256 row tiles re-read the whole B operand per 16 rows: 137 us at configs[3] B = 4096).
inline int wgrad_splits(int B) { return B <= 512 ? 0 : (B >= 2048 ? 4 : 2); }   // 0 = small-batch kernel

MmaWs mma_carve(const CriticDims& c, int B, void* base, size_t* total) {
  const MmaLayout L = mma_layout(c);
  const size_t Bp = round_up(B, RB);
  MmaWs w{};
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = p ? p + off : nullptr; off += align_up(bytes, 256); return r; };
  // (rows up to a multiple of 64: the split weight-gradient kernel's last 64-column warp may read
  // past inq; those rows are never written and only feed columns that are never stored)
  w.XT = (__nv_bfloat16*)take(2 * (size_t)round_up(L.inq, 64) * Bp);
  w.H1T = (__nv_bfloat16*)take(2 * 2 * (size_t)c.H1 * Bp);
  w.dZ2T = (__nv_bfloat16*)take(2 * 2 * (size_t)c.H2 * Bp);
  w.dZ1T = (__nv_bfloat16*)take(2 * 2 * (size_t)c.H1 * Bp);
  w.H2T = (__nv_bfloat16*)take(2 * 2 * (size_t)c.H2 * Bp);
  w.Z1 = (float*)take(4 * 2 * (size_t)B * c.H1);
  w.Z2 = (float*)take(4 * 2 * (size_t)B * c.H2);
  w.Hh2 = (float*)take(4 * 2 * (size_t)B * c.H2);
  w.q = (float*)take(4 * 2 * (size_t)B);
  w.dq = (float*)take(4 * 2 * (size_t)B);
  w.part = (float*)take(4 * 2 * (Bp / RB));
  w.ticket = (unsigned int*)take(4);
  const int ws = wgrad_splits(B);
  const int wt = ws > 0 ? tc_wgrad_splits((int)Bp, L.inq) : 0;   // tcgen05 weight-gradient partials
  const int wmax = ws > wt ? ws : wt;
  w.wpart = (float*)take(wmax > 1 ? sizeof(float) * wmax * 2 * ((size_t)HW * HW + (size_t)HW * L.inq) : 0);
  if (total) *total = off;
  return w;
}

// Loss of the last block to finish (the caller's `last`, block-uniform): per critic z a fixed-order
// sum over the blocks' partials (each thread a strided subset, all its loads in flight, then a
// fixed tree over the 256 threads), then the critics in order: deterministic. (The serial chain of
// one volatile L2 load per partial it replaces cost ~0.3 us per block.) blockDim.x == 256.
__device__ __forceinline__ void final_loss(const float* part, int nb, int nz, int mode, int B, float* loss) {
  __shared__ float red[256];
  float tot = 0.f;
  for (int z = 0; z < nz; ++z) {
    float s = 0.f;
    for (int i = threadIdx.x; i < nb; i += 256) s = __fadd_rn(s, *(volatile const float*)&part[z * nb + i]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] = __fadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
      __syncthreads();
    }
    const float sz = __fdiv_rn(red[0], (float)B);
    tot = mode == 0 ? __fadd_rn(tot, sz) : __fsub_rn(tot, sz);
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = tot;
}

// ------------------------------------------------------------------ forward (both critics)
constexpr int NWARP = 8, NTW = HW / (NWARP * 8);   // 8 warps x 4 n-tiles x 8 columns

__global__ void __launch_bounds__(256) critic_fwd_mma_kernel(
    int B, int Bp, int S, int A, int inp, int inq, const float* __restrict__ obs, const float* __restrict__ act,
    const __nv_bfloat16* __restrict__ pb, long long P, long long tb, long long oW1p, long long oW2,
    long long oW3, const float* __restrict__ params, long long oB1, long long oB2, long long oB3,
    __nv_bfloat16* __restrict__ XT, __nv_bfloat16* __restrict__ H1T, float* __restrict__ Z1,
    float* __restrict__ Z2, float* __restrict__ Hh2, float* __restrict__ q, int store, unsigned int* ticket,
    const __grid_constant__ CriticDecode dec) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __nv_bfloat16* const w2s = (__nv_bfloat16*)dsm;    // this critic's W2 staged: [HW][HW + SPAD]
  __shared__ __align__(8) uint64_t wbar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&wbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  // W2 into shared memory while the input tile and layer 1 run (the K = 256 layer-2 contraction
  // then reads no operand from L2)
  stage_rows(w2s, pb + blk_base(P) + blockIdx.y * tb + oW2, HW, HW, &wbar);
  __shared__ __align__(16) __nv_bfloat16 xs[RB * (512 + SPAD)];
  __shared__ __align__(16) __nv_bfloat16 h1s[RB * (HW + SPAD)];
  __shared__ float red[NWARP][RB];
  const int z = blockIdx.y, tid = threadIdx.x, warp = tid >> 5;
  const int lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int in = S + A, ldx = inp + SPAD, ldh = HW + SPAD;
  if (ticket && blockIdx.x == 0 && z == 0 && tid == 0) *ticket = 0u;   // for the backward launch
  // persistent over 16-row tiles: the staged W2 (135 KB, one CTA per SM) serves every tile of this
  // CTA (large batches: one CTA per 16 rows re-staged W2 512 times per launch at configs[3] B = 4096).
  // The next tile's [s; a] values are requested while the current tile runs (warp = rows warp and
  // warp + 8, lane = every 32nd input column: no index division; ncu r01: the X-tile build waited on
  // its loads for ~54% of the launch's stall samples at B = 4096)
  static_assert(RB == 16 && NWARP == 8, "X tile: two rows per warp");
  const bool decode = dec.counts != nullptr;
  __shared__ float acts[RB][32];   // decode: the tile's smoothed target actions a~ (A <= 32)
  float xv[2][16];
  auto load_x = [&](int rt) {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int b = rt + warp + 8 * rr;
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int i = lane + 32 * cc;
        float v = 0.f;
        if (b < B && i < in) v = i < S ? obs[(size_t)b * S + i] : (decode ? 0.f : act[(size_t)b * A + (i - S)]);
        xv[rr][cc] = v;
      }
    }
  };
  if (blockIdx.x * RB < Bp) load_x(blockIdx.x * RB);
  for (int r0 = blockIdx.x * RB; r0 < Bp; r0 += gridDim.x * RB) {
  if (decode) {
    // a' = tanh(Wd fr + bd) and a~ = smooth(a') per (row, action), in dec_fwd_kernel's operation order
    const int N3 = A * dec.D;
    const unsigned long long ctr = dec.ts.at ? *dec.ts.ctr_snap : 0ull;
    for (int idx = tid; idx < RB * A; idx += 256) {
      const int r = idx / A, j = idx - r * A, b = r0 + r;
      float v = 0.f;
      if (b < B) {
        // every count and weight requested before the (ordered) sum: one round trip, not D
        uint32_t cv[kDecMaxD];
        float wv[kDecMaxD];
#pragma unroll
        for (int e = 0; e < kDecMaxD; ++e) {
          cv[e] = e < dec.D ? dec.counts[(size_t)b * N3 + j * dec.D + e] : 0u;
          wv[e] = e < dec.D ? dec.Wd[j * dec.D + e] : 0.f;
        }
        float pre = 0.f;
#pragma unroll
        for (int e = 0; e < kDecMaxD; ++e) {
          if (e < dec.D) {
            const float fr = (float)cv[e] / (float)dec.T;
            pre = __fadd_rn(pre, __fmul_rn(wv[e], fr));
          }
        }
        pre = __fadd_rn(pre, dec.bd[j]);
        const float a = tanhf(pre);
        const int i = b * A + j;
        v = dec.ts.at ? smooth_action(a, i, dec.ts.noise, dec.ts.sigma, dec.ts.clip, dec.ts.seed, dec.ts.rank, ctr) : a;
        if (z == 0) {
          if (dec.act_out) dec.act_out[i] = a;
          if (dec.act_tape) dec.act_tape[i] = a;
          if (dec.ts.at) dec.ts.at[i] = v;
          if (dec.ts.at && dec.ts.advance && i == 0) *dec.ts.counter = ctr + 1;
        }
      }
      acts[r][j] = v;
    }
    __syncthreads();
  }
  // X tile (bf16-rounded [s; a]); the z == 0 CTAs also write X^T (zeros beyond in / B) for dW1
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      const int i = lane + 32 * cc;
      float v = xv[rr][cc];
      if (decode && i >= S && i < in && r0 + warp + 8 * rr < B) v = acts[warp + 8 * rr][i - S];
      if (i < inp) xs[(warp + 8 * rr) * ldx + i] = __float2bfloat16_rn(v);
    }
  __syncthreads();
  if (r0 + (int)gridDim.x * RB < Bp) load_x(r0 + gridDim.x * RB);
  if (store && z == 0) {
    for (int idx = tid; idx < RB * inq; idx += 256) {
      const int i = idx / RB, r = idx - i * RB;
      XT[(size_t)i * Bp + r0 + r] = i < inp ? xs[r * ldx + i] : __float2bfloat16_rn(0.f);
    }
  }
  const __nv_bfloat16* W1p = pb + blk_base(P) + z * tb + oW1p;
  const float* b1 = params + z * P + oB1;
  const float* b2 = params + z * P + oB2;
  const int n0 = warp * NTW * 8;
  {
    float acc[NTW][4] = {};
    float bias[NTW][2];   // requested before the MMAs (latency hidden behind them)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) { bias[nt][0] = b1[n0 + nt * 8 + 2 * t]; bias[nt][1] = b1[n0 + nt * 8 + 2 * t + 1]; }
    // wide inputs (configs[3]: K = 400): eight k-steps of weight fragments in flight, not four
    if (inp > 128) warp_mma<NTW, 8>(acc, xs, ldx, W1p + (size_t)n0 * inp, inp, inp);
    else warp_mma<NTW>(acc, xs, ldx, W1p + (size_t)n0 * inp, inp, inp);
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1), b = r0 + r;
        const float zz = __fadd_rn(acc[nt][e], bias[nt][e & 1]);
        h1s[r * ldh + col] = b < B ? __float2bfloat16_rn(fmaxf(zz, 0.f)) : __float2bfloat16_rn(0.f);
        if (store && b < B) Z1[((size_t)z * B + b) * HW + col] = zz;
      }
    }
  }
  __syncthreads();
  if (store) {   // h1^T for dW2 (zero rows beyond B), coalesced along the batch
    for (int idx = tid; idx < RB * HW; idx += 256) {
      const int col = idx / RB, r = idx - col * RB;
      H1T[((size_t)z * HW + col) * Bp + r0 + r] = h1s[r * ldh + col];
    }
  }
  const __nv_bfloat16* W3 = pb + z * P + oW3;
  float qp[2] = {0.f, 0.f};
  {
    float acc[NTW][4] = {};
    float bias[NTW][2], w3v[NTW][2];   // requested before the MMAs
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        bias[nt][u] = b2[n0 + nt * 8 + 2 * t + u];
        w3v[nt][u] = __bfloat162float(W3[n0 + nt * 8 + 2 * t + u]);
      }
    stage_wait(&wbar);
    warp_mma_ss<NTW>(acc, h1s, ldh, w2s + (size_t)n0 * (HW + SPAD), HW + SPAD, HW);
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1), b = r0 + r;
        const float zz = __fadd_rn(acc[nt][e], bias[nt][e & 1]);
        const float h = bf16_round(fmaxf(zz, 0.f));
        qp[e >> 1] = __fmaf_rn(h, w3v[nt][e & 1], qp[e >> 1]);
        if (store && b < B) {
          Z2[((size_t)z * B + b) * HW + col] = zz;
          Hh2[((size_t)z * B + b) * HW + col] = h;
        }
      }
    }
  }
  // Q[r] = sum_j h2[r][j] w3[j] + b3: reduce over the quad (t), then warps in a fixed order
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    float s = qp[hh];
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    if (t == 0) red[warp][g + hh * 8] = s;
  }
  __syncthreads();
  if (tid < RB && r0 + tid < B) {
    float s = red[0][tid];
    for (int w = 1; w < NWARP; ++w) s = __fadd_rn(s, red[w][tid]);
    q[(size_t)z * B + r0 + tid] = __fadd_rn(s, params[z * P + oB3]);
  }
  __syncthreads();   // xs / h1s / red are rewritten by the next tile
  }
}

// phase timeline of CTA (0, 0) of the last data-backward launch (diagnostics; spikerl_debug_critic_trace)
__device__ unsigned long long g_ctrace[16];
__device__ __forceinline__ void cstamp(int i) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_ctrace[i] = t;
  }
}

// ------------------------------------------------------------------ data backward
// dZ2 = round(dQ w3 [Z2 > 0]); dZ1 = round((dZ2 W2) [Z1 > 0]); grad_act = (dZ1 W1)[:, S:S+A]
// dQ is formed here (no separate loss launch): mode 0 (critic update) dQ_z[b] = 2 (Q_z - y)/B and
// the loss sum_z mean_b (Q_z - y)^2; mode 1 (actor step, critic 0 only) dQ = act_scale and the
// actor loss -mean_b Q. Each CTA writes dQ for its rows and one partial sum (fixed row order);
// the last CTA to finish (atomic ticket, zeroed by the forward launch) adds the partials in
// a fixed order, so the scalar is deterministic.
__global__ void __launch_bounds__(256) critic_bwd_data_mma_kernel(
    int B, int Bp, int S, int A, int inp, const float* __restrict__ q, const TdY y, int mode,
    float act_scale, float* __restrict__ dq, float* __restrict__ part, unsigned int* __restrict__ ticket,
    float* __restrict__ loss, const __nv_bfloat16* __restrict__ pb,
    long long P, long long tb, long long oW3, long long oW1T, long long oW2T, const float* __restrict__ Z1,
    const float* __restrict__ Z2, __nv_bfloat16* __restrict__ dZ2T, __nv_bfloat16* __restrict__ dZ1T,
    float* __restrict__ grad_act, int store_t, const float* __restrict__ dq_scale) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __nv_bfloat16* const w2s = (__nv_bfloat16*)dsm;    // W2T staged: [HW][HW + SPAD]
  __shared__ __align__(8) uint64_t wbar;
  __shared__ __align__(16) __nv_bfloat16 d2s[RB * (HW + SPAD)];
  __shared__ __align__(16) __nv_bfloat16 d1s[RB * (HW + SPAD)];
  __shared__ float dqs[RB];
  __shared__ bool last;
  const int z = blockIdx.y, r0 = blockIdx.x * RB, tid = threadIdx.x, warp = tid >> 5;
  const int lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int ldh = HW + SPAD;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&wbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cstamp(0);
  pdl_wait();
  pdl_trigger();
  cstamp(1);
  // W2T into shared memory while the dQ / dZ2 phase runs (trace r01: the K = 256 contraction
  // with its B fragments fetched from L2 took 6 us of this launch's 18)
  stage_rows(w2s, pb + blk_base(P) + z * tb + oW2T, HW, HW, &wbar);
  const __nv_bfloat16* W3 = pb + z * P + oW3;
  if (warp == 0) {
    float d = 0.f, c = 0.f;
    const int b = r0 + lane;
    if (lane < RB && b < B) {
      const float qv = q[(size_t)z * B + b];
      if (mode == 0) {
        const float e = __fsub_rn(qv, y.get(b, z));
        d = __fdiv_rn(__fmul_rn(2.0f, e), (float)B);
        c = __fmul_rn(e, e);
      } else {
        d = act_scale;
        c = qv;
      }
      if (dq_scale) d = __fmul_rn(d, *dq_scale);   // dynamic loss scaling (the loss scalar stays unscaled)
      dq[(size_t)z * B + b] = d;
    }
    if (lane < RB) dqs[lane] = d;
    // partial over this CTA's rows in row order (lane 0 sums the 16 values serially)
    float cs[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) cs[r] = __shfl_sync(0xffffffffu, c, r);
    if (lane == 0) {
      float sum = 0.f;
#pragma unroll
      for (int r = 0; r < RB; ++r) sum = __fadd_rn(sum, cs[r]);
      part[z * gridDim.x + blockIdx.x] = sum;
    }
  }
  __syncthreads();
  {   // thread = column j (HW == blockDim): w3_j once, the 16 rows' Z2 loads issued together
    static_assert(HW == 256, "one thread per hidden unit");
    const int j = tid;
    const float w3 = __bfloat162float(W3[j]);
    float zz[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) zz[r] = (r0 + r < B) ? Z2[((size_t)z * B + r0 + r) * HW + j] : 0.f;
#pragma unroll
    for (int r = 0; r < RB; ++r) d2s[r * ldh + j] = __float2bfloat16_rn(zz[r] > 0.f ? __fmul_rn(dqs[r], w3) : 0.f);
  }
  if (tid == 0) {   // publish the partial; the last CTA reduces all of them
    __threadfence();
    const unsigned int n = gridDim.x * gridDim.y;
    last = atomicAdd(ticket, 1u) == n - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    if (loss) final_loss(part, gridDim.x, gridDim.y, mode, B, loss);
    if (tid == 0) *ticket = 0u;
  }
  cstamp(2);
  if (store_t) {
    for (int idx = tid; idx < RB * HW; idx += 256) {
      const int j = idx / RB, r = idx - j * RB;
      dZ2T[((size_t)z * HW + j) * Bp + r0 + r] = d2s[r * ldh + j];
    }
  }
  cstamp(3);
  const int n0 = warp * NTW * 8;
  {
    float acc[NTW][4] = {};
    // the ReLU masks are requested before the MMAs so their latency hides behind them
    float z1v[NTW][4];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1), b = r0 + r;
        z1v[nt][e] = b < B ? Z1[((size_t)z * B + b) * HW + col] : 0.f;
      }
    stage_wait(&wbar);
    warp_mma_ss<NTW>(acc, d2s, ldh, w2s + (size_t)n0 * ldh, ldh, HW);
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1);
        d1s[r * ldh + col] = __float2bfloat16_rn(z1v[nt][e] > 0.f ? acc[nt][e] : 0.f);
      }
    }
  }
  __syncthreads();
  cstamp(4);
  if (store_t) {
    for (int idx = tid; idx < RB * HW; idx += 256) {
      const int j = idx / RB, r = idx - j * RB;
      dZ1T[((size_t)z * HW + j) * Bp + r0 + r] = d1s[r * ldh + j];
    }
  }
  cstamp(5);
  if (grad_act == nullptr || z != 0) return;
  // columns [S, S+A) of dZ1 W1 = dZ1 (W1T)^T in n-tiles of 8 from S rounded down, 32 at a time;
  // each warp takes 32 of the 256 k (2 k-steps) and the partial sums meet in shared memory
  // (trace r01: one warp walking all 16 k-steps made this tail 3 us)
  {
    __shared__ float gpart[NWARP][RB][32];
    const __nv_bfloat16* W1T = pb + blk_base(P) + oW1T;
    const int c0 = S & ~7;
    for (int cb = c0; cb < S + A; cb += 32) {
      float acc[4][4] = {};
      const int kw = warp * (HW / NWARP);
      warp_mma<4, 2>(acc, d1s + kw, ldh, W1T + (size_t)cb * HW + kw, HW, HW / NWARP);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) gpart[warp][g + (e >> 1) * 8][nt * 8 + 2 * t + (e & 1)] = acc[nt][e];
      __syncthreads();
      for (int idx = tid; idx < RB * 32; idx += 256) {
        const int r = idx >> 5, cl = idx & 31, col = cb + cl, b = r0 + r;
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) sum = __fadd_rn(sum, gpart[w][r][cl]);
        if (b < B && col >= S && col < S + A) grad_act[(size_t)b * A + (col - S)] = sum;
      }
      __syncthreads();
    }
  }
  cstamp(6);
}

// ------------------------------------------------------------------ weight gradients
// blockIdx.z = critic; blockIdx.y < HW/16: dW2 row tile; else dW1 row tile. Each CTA: 16 rows x
// 256 columns (4 warps x 64), K = Bp batch rows. Writes the fp32 master layout.
__device__ __forceinline__ void critic_wgrad_mma_body(
    int bx, int by, int z, int Bp, int in, int inq, long long P, long long oW1, long long oW2,
    const __nv_bfloat16* __restrict__ XT, const __nv_bfloat16* __restrict__ H1T, const __nv_bfloat16* __restrict__ dZ2T,
    const __nv_bfloat16* __restrict__ dZ1T, float* __restrict__ grad2) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const int lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int ntile = HW / RB;
  const bool w2 = by < ntile;
  const int m0 = (w2 ? by : by - ntile) * RB;
  const int ncols = w2 ? HW : in;
  const int n0 = bx * 256 + warp * NTW * 8;
  if (n0 >= ncols) return;
  const __nv_bfloat16* Am = (w2 ? dZ2T : dZ1T) + ((size_t)z * HW + m0) * Bp;
  const __nv_bfloat16* Bm = w2 ? H1T + (size_t)z * HW * Bp : XT;
  if (!w2 && n0 + NTW * 8 > inq) return;
  float acc[NTW][4] = {};
  // A is read straight from global (16 rows x Bp); fragments are 32-bit words
  warp_mma<NTW>(acc, Am, Bp, Bm + (size_t)n0 * Bp, Bp, Bp);
  float* out = grad2 + z * P + (w2 ? oW2 : oW1);
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = m0 + g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1);
      if (col < ncols) out[(size_t)r * ncols + col] = acc[nt][e];
    }
  }
}

// Large-batch weight gradients: blockIdx.x = (matrix, 64-row block, 128-column block) flattened,
// blockIdx.y = K split, blockIdx.z = critic. Warp w: rows 16 (w & 3) of the block, 64 columns
// (w >> 2). K split s covers batch rows [s Kc, (s+1) Kc). With one split the tile goes straight to
// the fp32 master layout; otherwise to wpart[s] (reduced in a fixed order by the next kernel).
__global__ void __launch_bounds__(256) critic_wgrad_split_kernel(
    int Bp, int in, int inq, int Kc, long long P, long long oW1, long long oW2, const __nv_bfloat16* __restrict__ XT,
    const __nv_bfloat16* __restrict__ H1T, const __nv_bfloat16* __restrict__ dZ2T,
    const __nv_bfloat16* __restrict__ dZ1T, float* __restrict__ grad2, float* __restrict__ wpart) {
  pdl_wait();
  pdl_trigger();
  const int z = blockIdx.z, ks = blockIdx.y, warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int cb2 = HW / 128, cb1 = (inq + 127) / 128;   // column blocks of dW2, dW1
  int blk = blockIdx.x;
  const bool w2 = blk < (HW / 64) * cb2;
  if (!w2) blk -= (HW / 64) * cb2;
  const int cb = w2 ? cb2 : cb1;
  const int m0 = (blk / cb) * 64 + 16 * (warp & 3), n0 = (blk % cb) * 128 + 64 * (warp >> 2);
  const int ncols = w2 ? HW : in;
  const int k0 = ks * Kc;
  const __nv_bfloat16* Am = (w2 ? dZ2T : dZ1T) + ((size_t)z * HW + m0) * Bp + k0;
  const __nv_bfloat16* Bm = (w2 ? H1T + (size_t)z * HW * Bp : XT) + (size_t)n0 * Bp + k0;
  if (!w2 && n0 >= inq) return;   // (inq is a multiple of 32 >= in; XT rows past in are zero)
  float acc[8][4] = {};
  warp_mma<8, 2>(acc, Am, Bp, Bm, Bp, min(Kc, Bp - k0));   // the last split may be shorter
  const size_t msz = (size_t)HW * HW + (size_t)HW * inq;
  float* dst = gridDim.y == 1 ? grad2 + z * P + (w2 ? oW2 : oW1)
                              : wpart + ((size_t)ks * 2 + z) * msz + (w2 ? 0 : (size_t)HW * HW);
  const int ld = gridDim.y == 1 ? ncols : (w2 ? HW : inq);
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = m0 + g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1);
      if (col < (gridDim.y == 1 ? ncols : ld)) dst[(size_t)r * ld + col] = acc[nt][e];
    }
}

// grad2[z][W] = sum over splits (fixed order) of the partial tiles (true widths only)
__global__ void critic_wgrad_reduce_kernel(int splits, int in, int inq, long long P, long long oW1, long long oW2,
                                           const float* __restrict__ wpart, float* __restrict__ grad2) {
  pdl_wait();
  pdl_trigger();
  const size_t msz = (size_t)HW * HW + (size_t)HW * inq;
  const long long n2 = (long long)HW * HW, n1 = (long long)HW * in, per = n2 + n1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < 2 * per; i += (long long)gridDim.x * blockDim.x) {
    const int z = (int)(i / per);
    const long long e = i - z * per;
    size_t src;
    float* dst;
    if (e < n2) { src = (size_t)e; dst = grad2 + z * P + oW2 + e; }
    else { const long long f = e - n2, r = f / in, c = f - r * in; src = (size_t)n2 + r * inq + c; dst = grad2 + z * P + oW1 + f; }
    float sum = 0.f;
    for (int s = 0; s < splits; ++s) sum = __fadd_rn(sum, wpart[((size_t)s * 2 + z) * msz + src]);
    *dst = sum;
  }
}

// The same sum over the column-major partials of the tcgen05 weight-gradient launch
// (launch_critic_wgrad_tc: part[(s 2 + z) msz + c 256 + r], dW1's columns after dW2's 256): 32 x 32
// tiles through shared memory so the partial reads (along r) and the master-layout writes (along c)
// are both coalesced; one element per thread, 8 loads in flight, splits added in order.
// grid (cdiv(256 + in, 32), 256 / 32, 2), block (32, 32).
__global__ void __launch_bounds__(1024) critic_wgrad_reduce_cm_kernel(int splits, int in, long long msz, long long P,
                                                                      long long oW1, long long oW2,
                                                                      const float* __restrict__ wpart,
                                                                      float* __restrict__ grad2) {
  __shared__ float tile[32][33];
  pdl_wait();
  pdl_trigger();
  const int tx = threadIdx.x, ty = threadIdx.y, z = blockIdx.z;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const bool w2 = c0 < HW;               // 256 is a multiple of 32: a tile is all dW2 or all dW1
  const int cb = w2 ? c0 : c0 - HW;      // first column within its matrix
  const int ncol = w2 ? HW : in;
  {
    const int c = cb + ty, r = r0 + tx;
    if (c < ncol) {
      const float* src = wpart + (size_t)z * msz + (w2 ? 0 : (size_t)HW * HW) + (size_t)c * HW + r;
      const size_t sst = 2 * (size_t)msz;
      float sum = 0.f;
      int s = 0;
      for (; s + 8 <= splits; s += 8) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = src[(size_t)(s + j) * sst];
#pragma unroll
        for (int j = 0; j < 8; ++j) sum = __fadd_rn(sum, v[j]);
      }
      for (; s < splits; ++s) sum = __fadd_rn(sum, src[(size_t)s * sst]);
      tile[ty][tx] = sum;
    }
  }
  __syncthreads();
  const int r = r0 + ty, c = cb + tx;
  if (c < ncol) grad2[z * P + (w2 ? oW2 : oW1) + (size_t)r * ncol + c] = tile[tx][ty];
}

// db1 = rowsum dZ1T, db2 = rowsum dZ2T, dW3 = dQ^T H2, db3 = sum dQ. Small batches: one warp per
// output (blockIdx.x * 8 + warp); large batches (B > 1024): one block per output, each thread a
// strided subset of the rows with four partial sums, then a fixed tree (ncu r02: the warp-per-output
// form took 18-26 us at B = 4096). Both orders are fixed: deterministic.
__device__ __forceinline__ float bias_row_term(int o, int z, int b, int Bp, int B, const __nv_bfloat16* dZ1T,
                                               const __nv_bfloat16* dZ2T, const float* dq, const float* Hh2,
                                               const __nv_bfloat16* H2T) {
  if (o < HW) return __bfloat162float(dZ1T[((size_t)z * HW + o) * Bp + b]);
  if (o < 2 * HW) return __bfloat162float(dZ2T[((size_t)z * HW + o - HW) * Bp + b]);
  if (o < 3 * HW) {
    const int j = o - 2 * HW;
    const float h = H2T ? __bfloat162float(H2T[((size_t)z * HW + j) * Bp + b]) : Hh2[((size_t)z * B + b) * HW + j];
    return __fmul_rn(dq[(size_t)z * B + b], h);
  }
  return dq[(size_t)z * B + b];
}

__global__ void __launch_bounds__(256) critic_bias_grads_kernel(int B, int Bp, long long P, long long oB1,
                                                                long long oB2, long long oW3, long long oB3,
                                                                const __nv_bfloat16* __restrict__ dZ1T,
                                                                const __nv_bfloat16* __restrict__ dZ2T,
                                                                const float* __restrict__ dq,
                                                                const float* __restrict__ Hh2,
                                                                const __nv_bfloat16* __restrict__ H2T,
                                                                float* __restrict__ grad2) {
  pdl_wait();
  pdl_trigger();
  const int z = blockIdx.y;
  const int nout = 3 * HW + 1;
  const bool big = gridDim.x == (unsigned)nout;   // one block per output
  if (big && H2T) {
    // tcgen05 path (rows transposed, Bp a multiple of 16): each thread 8 consecutive rows per
    // 16-byte load, every load of the row issued before the sums; rows past B are zero in dZ1T /
    // dZ2T / H2T, and dq is only read below B
    const int o = blockIdx.x;
    const __nv_bfloat16* row = o < HW ? dZ1T + ((size_t)z * HW + o) * Bp
                             : (o < 2 * HW ? dZ2T + ((size_t)z * HW + o - HW) * Bp
                                           : (o < 3 * HW ? H2T + ((size_t)z * HW + o - 2 * HW) * Bp : nullptr));
    float sacc = 0.f;
    for (int b0 = 8 * threadIdx.x; b0 < Bp; b0 += 4 * 2048) {
      uint4 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        v[i] = (row && b0 + 2048 * i < Bp) ? *reinterpret_cast<const uint4*>(row + b0 + 2048 * i) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int bb = b0 + 2048 * i;
        if (bb >= Bp) break;
        const uint32_t* w = &v[i].x;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float x = __uint_as_float(k & 1 ? (w[k >> 1] & 0xFFFF0000u) : (w[k >> 1] << 16));
          const int b = bb + k;
          if (o < 2 * HW) sacc = __fadd_rn(sacc, x);
          else if (b < B) sacc = o < 3 * HW ? __fmaf_rn(dq[(size_t)z * B + b], x, sacc) : __fadd_rn(sacc, dq[(size_t)z * B + b]);
        }
      }
    }
    for (int off = 16; off > 0; off >>= 1) sacc = __fadd_rn(sacc, __shfl_xor_sync(0xffffffffu, sacc, off));
    __shared__ float red2[8];
    if ((threadIdx.x & 31) == 0) red2[threadIdx.x >> 5] = sacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < 8; ++w) t = __fadd_rn(t, red2[w]);
      float* base = grad2 + z * P;
      if (o < HW) base[oB1 + o] = t;
      else if (o < 2 * HW) base[oB2 + (o - HW)] = t;
      else if (o < 3 * HW) base[oW3 + (o - 2 * HW)] = t;
      else base[oB3] = t;
    }
    return;
  }
  const int o = big ? blockIdx.x : blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = big ? threadIdx.x : threadIdx.x & 31, nl = big ? 256 : 32;
  if (o >= nout) return;
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  int b = lane;
  for (; b + 3 * nl < B; b += 4 * nl) {
#pragma unroll
    for (int k = 0; k < 4; ++k) s4[k] = __fadd_rn(s4[k], bias_row_term(o, z, b + k * nl, Bp, B, dZ1T, dZ2T, dq, Hh2, H2T));
  }
  for (int k = 0; b < B; b += nl, ++k) s4[k & 3] = __fadd_rn(s4[k & 3], bias_row_term(o, z, b, Bp, B, dZ1T, dZ2T, dq, Hh2, H2T));
  float s = __fadd_rn(__fadd_rn(s4[0], s4[1]), __fadd_rn(s4[2], s4[3]));
  for (int off = 16; off > 0; off >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
  if (big) {
    __shared__ float red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      s = 0.f;
      for (int w = 0; w < 8; ++w) s = __fadd_rn(s, red[w]);
    }
  }
  if (lane == 0) {
    float* base = grad2 + z * P;
    if (o < HW) base[oB1 + o] = s;
    else if (o < 2 * HW) base[oB2 + (o - HW)] = s;
    else if (o < 3 * HW) base[oW3 + (o - 2 * HW)] = s;
    else base[oB3] = s;
  }
}

// Small batches (B <= 512): the weight gradients (critic_wgrad_mma_body, grid rows [0, 2 HW / 16)) and
// the bias / w3 gradients (critic_bias_grads_kernel's warp-per-output form, 8 outputs per CTA, the
// grid rows after them) as ONE launch: no side-stream fork / join in front of the critic's Adam (a
// joined branch is a full graph edge, so the Adam launch could not start early; same per-output
// arithmetic, bitwise the two-launch result).
__global__ void __launch_bounds__(256) critic_wgrad_mma_kernel(
    int Bp, int in, int inq, long long P, long long oW1, long long oW2, const __nv_bfloat16* __restrict__ XT,
    const __nv_bfloat16* __restrict__ H1T, const __nv_bfloat16* __restrict__ dZ2T,
    const __nv_bfloat16* __restrict__ dZ1T, float* __restrict__ grad2, int B, long long oB1, long long oB2,
    long long oW3, long long oB3, const float* __restrict__ dq, const float* __restrict__ Hh2) {
  pdl_wait();
  pdl_trigger();
  const int ntile = HW / RB;
  if ((int)blockIdx.y < 2 * ntile) {
    critic_wgrad_mma_body(blockIdx.x, blockIdx.y, blockIdx.z, Bp, in, inq, P, oW1, oW2, XT, H1T, dZ2T, dZ1T, grad2);
    return;
  }
  const int z = blockIdx.z;
  const int bt = (blockIdx.y - 2 * ntile) * gridDim.x + blockIdx.x;   // bias CTA index
  const int o = bt * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int nout = 3 * HW + 1;
  if (o >= nout) return;
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  int b = lane;
  for (; b + 3 * 32 < B; b += 4 * 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) s4[k] = __fadd_rn(s4[k], bias_row_term(o, z, b + k * 32, Bp, B, dZ1T, dZ2T, dq, Hh2, nullptr));
  }
  for (int k = 0; b < B; b += 32, ++k) s4[k & 3] = __fadd_rn(s4[k & 3], bias_row_term(o, z, b, Bp, B, dZ1T, dZ2T, dq, Hh2, nullptr));
  float sum = __fadd_rn(__fadd_rn(s4[0], s4[1]), __fadd_rn(s4[2], s4[3]));
  for (int off = 16; off > 0; off >>= 1) sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, off));
  if (lane == 0) {
    float* base = grad2 + z * P;
    if (o < HW) base[oB1 + o] = sum;
    else if (o < 2 * HW) base[oB2 + (o - HW)] = sum;
    else if (o < 3 * HW) base[oW3 + (o - 2 * HW)] = sum;
    else base[oB3] = sum;
  }
}

// bf16 refresh of the twin pair: [2][P] plain copy, then per critic W1p, W1T, W2T (zero padded)
__global__ void critic_refresh_kernel(const float* __restrict__ params, long long P, int in, int H1, int H2,
                                      int inp, int inq, long long oW1, long long oW2, long long tb,
                                      __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const long long bb = blk_base(P), total = bb + 2 * tb;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    float v;
    if (i < 2 * P) {
      v = params[i];
    } else if (i < bb) {
      v = 0.f;   // alignment gap
    } else {
      const long long f = i - bb;
      const int z = (int)(f / tb);
      long long e = f - z * tb;
      const float* W1 = params + z * P + oW1;
      const float* W2 = params + z * P + oW2;
      const long long n1p = (long long)H1 * inp, n1t = (long long)inq * H1;
      if (e < n1p) {                         // W1p[k][i]
        const int k = (int)(e / inp), ii = (int)(e - (long long)k * inp);
        v = ii < in ? W1[(size_t)k * in + ii] : 0.f;
      } else if ((e -= n1p) < n1t) {         // W1T[i][k]
        const int ii = (int)(e / H1), k = (int)(e - (long long)ii * H1);
        v = ii < in ? W1[(size_t)k * in + ii] : 0.f;
      } else if ((e -= n1t) < (long long)H1 * H2) {   // W2T[k][j] = W2[j][k]
        const int k = (int)(e / H2), j = (int)(e - (long long)k * H2);
        v = W2[(size_t)j * H1 + k];
      } else {                               // W2 (aligned copy)
        v = W2[e - (long long)H1 * H2];
      }
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

// loss = sum_z mean_b (Q_z - y)^2 ; dQ[z][b] = 2 (Q_z - y)/B. Single block, fixed order.
__global__ void __launch_bounds__(256) critic_loss_mma_kernel(int B, int nz, const float* __restrict__ q,
                                                              const TdY y, float* __restrict__ dq,
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

// ------------------------------------------------------------------ large batches (tcgen05 engine)
// X^T = bf16([s; a])^T [inq64][Bp] (zero past in and past B), through a 32 x 32 shared tile (reads
// coalesced along the input, writes along the batch); block (0, 0) also zeroes the loss ticket of
// the data-backward launch.
__global__ void __launch_bounds__(256) critic_xt_kernel(int B, int Bp, int S, int A, int rows,
                                                        const float* __restrict__ obs, const float* __restrict__ act,
                                                        __nv_bfloat16* __restrict__ XT, unsigned int* ticket) {
  pdl_wait();
  pdl_trigger();
  __shared__ float tile[32][33];
  const int b0 = blockIdx.x * 32, i0 = blockIdx.y * 32, tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int in = S + A;
  if (ticket && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *ticket = 0u;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, i = i0 + tx;
    float v = 0.f;
    if (b < B && i < in) v = i < S ? obs[(size_t)b * S + i] : act[(size_t)b * A + (i - S)];
    tile[r][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, b = b0 + tx;
    if (i < rows && b < Bp) XT[(size_t)i * Bp + b] = __float2bfloat16_rn(tile[tx][r]);
  }
}

// dQ (mode 0: 2 (Q_z - y)/B and the MSE; mode 1: act_scale, the actor loss -mean Q), then
// dZ2^T = RN_bf16(dQ w3 [h2 > 0]) [z][H2][Bp]. A block owns 64 batch rows of one critic (thread =
// row (tid & 63), hidden units tid >> 6 + 4 i); its loss partial is summed in row order and the
// last block (ticket) adds the partials in (z, block) order: deterministic.
__global__ void __launch_bounds__(256) critic_dz2_kernel(int B, int Bp, const float* __restrict__ q,
                                                         const TdY y, int mode, float act_scale,
                                                         const float* __restrict__ dq_scale, float* __restrict__ dq,
                                                         float* __restrict__ part, unsigned int* __restrict__ ticket,
                                                         float* __restrict__ loss, const __nv_bfloat16* __restrict__ pb,
                                                         long long P, long long oW3, const __nv_bfloat16* __restrict__ H2T,
                                                         __nv_bfloat16* __restrict__ dZ2T) {
  pdl_wait();
  pdl_trigger();
  __shared__ float dqs[64], cs[64], w3s[HW];
  __shared__ bool last;
  const int z = blockIdx.y, r = threadIdx.x & 63, b = blockIdx.x * 64 + r;
  // w3 in shared memory (ncu r02: read from global inside the store loop, every hidden unit waited
  // on its own L2 round trip: 38 us at B = 4096)
  w3s[threadIdx.x] = __bfloat162float(pb[z * P + oW3 + threadIdx.x]);
  if (threadIdx.x < 64) {
    float d = 0.f, c = 0.f;
    if (b < B) {
      const float qv = q[(size_t)z * B + b];
      if (mode == 0) {
        const float e = __fsub_rn(qv, y.get(b, z));
        d = __fdiv_rn(__fmul_rn(2.0f, e), (float)B);
        c = __fmul_rn(e, e);
      } else {
        d = act_scale;
        c = qv;
      }
      if (dq_scale) d = __fmul_rn(d, *dq_scale);   // dynamic loss scaling (the loss stays unscaled)
      dq[(size_t)z * B + b] = d;
    }
    dqs[r] = d;
    cs[r] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float sum = 0.f;
    for (int k = 0; k < 64; ++k) sum = __fadd_rn(sum, cs[k]);
    part[z * gridDim.x + blockIdx.x] = sum;
    __threadfence();
    const unsigned int n = gridDim.x * gridDim.y;
    last = atomicAdd(ticket, 1u) == n - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    if (loss) final_loss(part, gridDim.x, gridDim.y, mode, B, loss);
    if (threadIdx.x == 0) *ticket = 0u;
  }
  __syncthreads();   // dqs / w3s complete
  // the block's 64 rows x 256 hidden units as 16-byte chunks of 8 rows: 8 chunks per thread, all
  // loads issued before any store (ncu r02: one 2-byte load in flight per thread made this launch
  // 35-38 us at configs[3] B = 4096)
  const int b0 = blockIdx.x * 64;
  uint4 hv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = threadIdx.x + 256 * i, j = c >> 3, bo = (c & 7) * 8;
    hv[i] = b0 + bo < Bp ? *reinterpret_cast<const uint4*>(H2T + ((size_t)z * HW + j) * Bp + b0 + bo)
                         : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = threadIdx.x + 256 * i, j = c >> 3, bo = (c & 7) * 8;
    if (b0 + bo >= Bp) continue;
    const uint32_t* hw = &hv[i].x;
    uint32_t ow[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float h0 = __uint_as_float(hw[k] << 16), h1 = __uint_as_float(hw[k] & 0xFFFF0000u);
      const float v0 = h0 > 0.f ? __fmul_rn(dqs[bo + 2 * k], w3s[j]) : 0.f;
      const float v1 = h1 > 0.f ? __fmul_rn(dqs[bo + 2 * k + 1], w3s[j]) : 0.f;
      ow[k] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v0)) |
              ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v1)) << 16);
    }
    *reinterpret_cast<uint4*>(dZ2T + ((size_t)z * HW + j) * Bp + b0 + bo) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
  }
}

// grad_act[b][a] = sum_j dZ1[b][j] W1[j][S + a] (critic 0). A block owns 32 rows; warp w sums hidden
// units [32 w, 32 w + 32) for every action of its lane's row (the W1T slice staged in shared memory,
// read as warp-wide broadcasts), and the 8 partial sums meet in shared memory in warp order.
constexpr int kGactMaxA = 32;
__global__ void __launch_bounds__(256) critic_gact_kernel(int B, int Bp, int S, int A, const __nv_bfloat16* __restrict__ dZ1T,
                                                          const __nv_bfloat16* __restrict__ W1T, float* __restrict__ grad_act) {
  pdl_wait();
  pdl_trigger();
  // one buffer: first the W1T slice wsl[j][a] = W1[j][S + a], then the partial sums part[w][r][a]
  __shared__ float sbuf[NWARP * 32 * (kGactMaxA + 1)];
  static_assert(HW * kGactMaxA <= NWARP * 32 * (kGactMaxA + 1), "shared buffer");
  float (*wsl)[kGactMaxA] = reinterpret_cast<float (*)[kGactMaxA]>(sbuf);
  float (*part)[32][kGactMaxA + 1] = reinterpret_cast<float (*)[32][kGactMaxA + 1]>(sbuf);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {   // the W1T slice, all loads issued before the shared-memory stores
    float wv[kGactMaxA];
#pragma unroll
    for (int a = 0; a < kGactMaxA; ++a) wv[a] = a < A ? __bfloat162float(W1T[(size_t)(S + a) * HW + threadIdx.x]) : 0.f;
#pragma unroll
    for (int a = 0; a < kGactMaxA; ++a) wsl[threadIdx.x][a] = wv[a];
  }
  __syncthreads();
  const int b = blockIdx.x * 32 + lane;
  float acc[kGactMaxA];
#pragma unroll
  for (int a = 0; a < kGactMaxA; ++a) acc[a] = 0.f;
  float dv[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) dv[u] = b < Bp ? __bfloat162float(dZ1T[(size_t)(32 * warp + u) * Bp + b]) : 0.f;
#pragma unroll
  for (int u = 0; u < 32; ++u) {
    const int j = 32 * warp + u;
#pragma unroll
    for (int a = 0; a < kGactMaxA; ++a)
      if (a < A) acc[a] = __fmaf_rn(dv[u], wsl[j][a], acc[a]);
  }
  __syncthreads();   // every warp is done with wsl
#pragma unroll
  for (int a = 0; a < kGactMaxA; ++a)
    if (a < A) part[warp][lane][a] = acc[a];
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * A; i += 256) {
    const int r = i / A, a = i - r * A, bb = blockIdx.x * 32 + r;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) s = __fadd_rn(s, part[w][r][a]);
    if (bb < B) grad_act[(size_t)bb * A + a] = s;
  }
}

// ------------------------------------------------------------------ fused small-batch critic update
// The latency regime (configs[1..2], configs[3] B = 100): the critic update of a TD3 step as ONE
// launch instead of forward, data backward, weight / bias gradients and Adam (four dependent launches
// of ~5 us each at B = 256, mostly ramp and operand latency). Three phases separated by grid-wide
// barriers (every CTA resident: grid <= SMs, one CTA per SM by its shared memory):
//   F  one 16-row tile of one critic per CTA: forward (W2 staged once), Q, dQ = 2 (Q - y) / B and the
//      loss partial, dZ2, dH1 = dZ2 W2 read from the SAME staged W2 through ldmatrix.trans (no second
//      135 KB staging of W2^T), dZ1; the ReLU masks stay in registers (no Z1 / Z2 planes); the
//      transposed bf16 operands of the weight gradients go to the workspace;
//   W  the weight-gradient tiles and the bias / w3 gradients of both critics, the loss scalar;
//   A  Adam over both critics (+ the targets' Polyak step on actor updates), the bf16 views.
// Every value is formed by the same operations in the same order as the four-launch path (the same
// MMA k order, the same reductions, adam_body), so the result is bitwise that path's (tested).
struct CritFusedArgs {
  int B, Bp, S, A, inp, inq, in, nb;          // nb = Bp / RB row tiles per critic
  const float* obs;
  const float* act;
  const __nv_bfloat16* pb;                    // bf16 twin buffer (mma layout)
  long long P, tb, W1p, W2c, W1T, oW3, oB1, oB2, oB3, oW1, oW2;
  float* params;                              // [2][P] fp32 masters (read: biases; written: Adam)
  TdY y;
  float act_scale;
  float *q, *loss, *grad2, *dq, *part;
  __nv_bfloat16 *XT, *H1T, *H2T, *dZ2T, *dZ1T;
  float* grad_act;
  // Adam
  float *m, *v;
  long long* counter;
  unsigned int *ticket, *gbar;
  float lr, b1, b2, eps;
  double lnb1, lnb2;
  float* tp;
  float tau;
  int dbg;   // SPIKERL_CRITIC_FUSED_DBG ablation bits (wrong results by design): 1 no bf16 views in
             // Adam, 2 no Adam, 4 no bias tasks, 8 no weight-gradient tasks
};

// grid-wide barrier over a counter that is 0 at rest (the last CTA of the launch zeroes it); a
// grid that could not be co-resident traps after ~2 s instead of hanging the device
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int G, unsigned int& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += G;
    __threadfence();
    atomicAdd(ctr, 1u);
    const long long t0 = clock64();
    unsigned int v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if ((int)(v - target) >= 0) break;
      if (clock64() - t0 > (1LL << 32)) __trap();
    }
  }
  __syncthreads();
}

// acc[nt] += A[16 x K] * B with B stored [K][N] row-major in shared memory (n contiguous, row stride
// ldb elements, column offset applied by the caller): the B fragments come from ldmatrix.trans, so
// the values and the k order of every MMA are those of warp_mma_ss over the transposed matrix.
template <int NT>
__device__ __forceinline__ void warp_mma_ss_t(float (&acc)[NT][4], const __nv_bfloat16* A, int lda,
                                              const __nv_bfloat16* Bkn, int ldb, int K) {
  static_assert(NT % 2 == 0, "two n-tiles per ldmatrix.x4");
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const __nv_bfloat16* a0 = A + g * lda + 2 * t;
  const __nv_bfloat16* a1 = A + (g + 8) * lda + 2 * t;
  // matrix j = lane / 8: k rows (j & 1) * 8 .. + 7 of n-tile (j >> 1)
  const uint32_t bb = smem_addr(Bkn + ((lane & 7) + ((lane >> 3) & 1) * 8) * ldb + ((lane >> 4) * 8));
#pragma unroll 4
  for (int k0 = 0; k0 < K; k0 += 16) {
    const uint32_t a[4] = {ld32(a0 + k0), ld32(a1 + k0), ld32(a0 + k0 + 8), ld32(a1 + k0 + 8)};
#pragma unroll
    for (int nt = 0; nt < NT; nt += 2) {
      uint32_t r0, r1, r2, r3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                   : "r"(bb + (uint32_t)((k0 * ldb + nt * 8) * 2)));
      mma16816(acc[nt], a, r0, r1);
      mma16816(acc[nt + 1], a, r2, r3);
    }
  }
}

// 16-byte asynchronous global -> shared copies (LDGSTS: no register staging, any shared destination,
// so padded rows need no per-row bulk copy; 256 per-row bulk copies issued at a launch's start stalled
// the issuing threads for ~2 us, trace r02)
__device__ __forceinline__ void cp16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// rows x (cols bf16, a multiple of 8) from global (row stride gld elements) into shared memory (row
// stride sld elements), every thread of the CTA issuing its share
__device__ __forceinline__ void cp_rows(__nv_bfloat16* sdst, int sld, const __nv_bfloat16* gsrc, long long gld, int rows,
                                        int cols) {
  // thread = (row offset, chunk): one division per call, not one per chunk (the per-chunk division made
  // issuing a 128 KB stage ~700 instructions per thread, trace r02)
  const int cpr = cols >> 3;   // 16-byte chunks per row (<= blockDim.x)
  const int rpp = (int)blockDim.x / cpr, tr = (int)threadIdx.x / cpr, tk = (int)threadIdx.x - tr * cpr;
  if (tr >= rpp) return;
  const __nv_bfloat16* g = gsrc + (size_t)tr * gld + 8 * tk;
  __nv_bfloat16* d = sdst + (size_t)tr * sld + 8 * tk;
#pragma unroll 4
  for (int r = tr; r < rows; r += rpp, g += (size_t)rpp * gld, d += (size_t)rpp * sld) cp16(d, g);
}

// One output row's batch sum from a shared-memory row (bf16 values x[b], b < B), in exactly the order
// of critic_bias_grads_kernel's warp-per-output form (lane-strided, four partial sums, xor tree);
// dqs != NULL: the terms are dq[b] x[b] (dW3); x == NULL: the terms are dq[b] (db3).
__device__ __forceinline__ float warp_row_sum(const __nv_bfloat16* x, const float* dqs, int B) {
  const int lane = threadIdx.x & 31;
  auto term = [&](int b) -> float {
    if (!x) return dqs[b];
    const float v = __bfloat162float(x[b]);
    return dqs ? __fmul_rn(dqs[b], v) : v;
  };
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  int b = lane;
  for (; b + 3 * 32 < B; b += 4 * 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) s4[k] = __fadd_rn(s4[k], term(b + k * 32));
  }
  for (int k = 0; b < B; b += 32, ++k) s4[k & 3] = __fadd_rn(s4[k & 3], term(b));
  float s = __fadd_rn(__fadd_rn(s4[0], s4[1]), __fadd_rn(s4[2], s4[3]));
  for (int off = 16; off > 0; off >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
  return s;
}

// R output rows at once (row r at x + r ld), each summed in warp_row_sum's order: the rows' loads and
// shuffles interleave instead of running R dependent chains one after another (trace r02: 64 rows done
// one at a time took 3.1 us of the weight-gradient phase, 1.9 us this way)
template <int R>
__device__ __forceinline__ void warp_rows_sum(const __nv_bfloat16* x, int ld, const float* dqs, int B, float (&out)[R]) {
  const int lane = threadIdx.x & 31;
  float s4[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r) s4[r][0] = s4[r][1] = s4[r][2] = s4[r][3] = 0.f;
  auto term = [&](int r, int b) -> float {
    const float v = __bfloat162float(x[(size_t)r * ld + b]);
    return dqs ? __fmul_rn(dqs[b], v) : v;
  };
  int b = lane;
  for (; b + 3 * 32 < B; b += 4 * 32) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < 4; ++k) s4[r][k] = __fadd_rn(s4[r][k], term(r, b + k * 32));
  }
  for (int k = 0; b < B; b += 32, ++k) {
#pragma unroll
    for (int r = 0; r < R; ++r) s4[r][k & 3] = __fadd_rn(s4[r][k & 3], term(r, b));
  }
#pragma unroll
  for (int r = 0; r < R; ++r) out[r] = __fadd_rn(__fadd_rn(s4[r][0], s4[r][1]), __fadd_rn(s4[r][2], s4[r][3]));
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int r = 0; r < R; ++r) out[r] = __fadd_rn(out[r], __shfl_xor_sync(0xffffffffu, out[r], off));
  }
}

// Phase W of the fused critic update, one task = one CTA: both operands of a 64 x 64 weight-gradient
// tile staged whole in shared memory (cp.async, one round trip), the tile's MMAs (8 warps x 16 x 32,
// K = Bp in the k order of critic_wgrad_mma_kernel), and the bias sums whose rows the tile holds:
//   kind 0  dW2 tile (rows j2 of dZ2T, cols j1 of H1T); column block 0 also db2 of its rows;
//   kind 1  dW1 tile (rows j of dZ1T, cols i of X^T); column block 0 also db1;
//   kind 2  dW3 of 64 units (rows of H2T, times dQ); unit block 0 also db3.
__device__ __forceinline__ int wtask_count(int in) { return 2 * 16 + 2 * 4 * ((in + 63) / 64) + 2 * 4; }
__device__ __forceinline__ void crit_wtask(const CritFusedArgs& a, int task, __nv_bfloat16* sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int Bp = a.Bp, B = a.B, ld = Bp + SPAD;
  const int nc1 = (a.in + 63) / 64;
  int kind, z, rb, cb;
  if (task < 32) { kind = 0; z = task / 16; rb = (task % 16) / 4; cb = task % 4; }
  else if ((task -= 32) < 8 * nc1) { kind = 1; z = task / (4 * nc1); rb = (task % (4 * nc1)) / nc1; cb = task % nc1; }
  else { task -= 8 * nc1; kind = 2; z = task / 4; rb = task % 4; cb = 0; }
  const int m0 = rb * 64, n0 = cb * 64;
  __nv_bfloat16* As = sm;
  __nv_bfloat16* Bs = sm + (size_t)64 * ld;
  float* dqs = reinterpret_cast<float*>(sm + (size_t)128 * ld);   // [B] (kind 2)
  const __nv_bfloat16* Ag = (kind == 0 ? a.dZ2T : kind == 1 ? a.dZ1T : a.H2T) + ((size_t)z * HW + m0) * Bp;
  cp_rows(As, ld, Ag, Bp, 64, Bp);
  if (kind == 0) cp_rows(Bs, ld, a.H1T + ((size_t)z * HW + n0) * Bp, Bp, 64, Bp);
  if (kind == 1) cp_rows(Bs, ld, a.XT + (size_t)n0 * Bp, Bp, 64, Bp);
  cp_commit();
  if (kind == 2)
    for (int b = threadIdx.x; b < B; b += blockDim.x) dqs[b] = a.dq[(size_t)z * B + b];
  cp_wait_all();
  __syncthreads();
  cstamp(7);
  float* gz = a.grad2 + z * a.P;
  if (kind < 2) {
    const int ncols = kind == 0 ? HW : a.in;
    const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
    float acc[4][4] = {};
    warp_mma_ss<4>(acc, As + (size_t)wm * ld, ld, Bs + (size_t)wn * ld, ld, Bp);
    float* out = gz + (kind == 0 ? a.oW2 : a.oW1);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = m0 + wm + g + (e >> 1) * 8, col = n0 + wn + nt * 8 + 2 * t + (e & 1);
        if (col < ncols) out[(size_t)r * ncols + col] = acc[nt][e];
      }
    cstamp(14);
    if (cb == 0) {   // rows warp 8 .. warp 8 + 7
      float sr[8];
      warp_rows_sum<8>(As + (size_t)warp * 8 * ld, ld, nullptr, B, sr);
      if (lane < 8) {
        float v = sr[0];
#pragma unroll
        for (int r = 1; r < 8; ++r) if (lane == r) v = sr[r];
        gz[(kind == 0 ? a.oB2 : a.oB1) + m0 + warp * 8 + lane] = v;
      }
    }
  } else {
    {
      float sr[8];
      warp_rows_sum<8>(As + (size_t)warp * 8 * ld, ld, dqs, B, sr);
      if (lane < 8) {
        float v = sr[0];
#pragma unroll
        for (int r = 1; r < 8; ++r) if (lane == r) v = sr[r];
        gz[a.oW3 + m0 + warp * 8 + lane] = v;
      }
    }
    if (rb == 0 && warp == 0) {
      const float s = warp_row_sum(nullptr, dqs, B);
      if (lane == 0) gz[a.oB3] = s;
    }
  }
  cstamp(15);
  __syncthreads();   // the shared operands are reused by the CTA's next task
}

// Phase F for one 16-row tile (rows r0.., critic z). MODE 0: critic update (dQ from the TD target,
// transposed operands, h2 and dQ stored for phase W); MODE 1: the actor objective on critic 0 (dQ =
// act_scale, the loss partial sums Q, dQ1/da of the tile's rows).
// the [s; a] values of a tile's rows (warp = rows warp and warp + 8, lane = every 32nd column)
__device__ __forceinline__ void load_xtile(const CritFusedArgs& a, int tile, float (&xv)[2][16]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, in = a.S + a.A;
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int b = tile * RB + warp + 8 * rr;
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      const int i = lane + 32 * cc;
      float v = 0.f;
      if (b < a.B && i < in) v = i < a.S ? a.obs[(size_t)b * a.S + i] : a.act[(size_t)b * a.A + (i - a.S)];
      xv[rr][cc] = v;
    }
  }
}

// xv: the tile's [s; a] (load_xtile), requested by the caller BEFORE its PDL wait — the TD3 callers'
// inputs were written by kernels that completed before this launch's predecessor (the gather, the
// target path / pi(s) branches behind full graph edges), so their round trip overlaps the wait
template <int MODE>
__device__ __forceinline__ void crit_tile(const CritFusedArgs& a, int z, int tile, __nv_bfloat16* w2s, uint64_t* wbar,
                                          __nv_bfloat16* xs, __nv_bfloat16* h1s, __nv_bfloat16* d2s,
                                          __nv_bfloat16* d1s, float (*red)[RB], float* qs, float* dqs,
                                          const float (&xv)[2][16]) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const int lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int B = a.B, r0 = tile * RB;
  const int in = a.S + a.A, ldx = a.inp + SPAD, ldh = HW + SPAD;
  const long long P = a.P;
  // the loss inputs of the tile's rows (TD target or its parts) and b3, requested now: they were on
  // the dQ / Q critical path as two late round trips (trace r02)
  float yv = 0.f, b3v = 0.f;
  if (tid < RB) {
    b3v = a.params[z * P + a.oB3];
    if (MODE == 0 && r0 + tid < B) yv = a.y.at(r0 + tid);
  }
  {
    // W2 into shared memory (per-row bulk copies on the TMA engine, completing on an mbarrier) behind
    // the X-tile loads, while layer 1 runs
    stage_rows(w2s, a.pb + blk_base(P) + z * a.tb + a.W2c, HW, HW, wbar);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int i = lane + 32 * cc;
        if (i < a.inp) xs[(warp + 8 * rr) * ldx + i] = __float2bfloat16_rn(xv[rr][cc]);
      }
  }
  __syncthreads();
  if (MODE == 0) cstamp(8);
  if (MODE == 0 && z == 0) {
    for (int idx = tid; idx < RB * a.inq; idx += 256) {
      const int i = idx / RB, r = idx - i * RB;
      a.XT[(size_t)i * a.Bp + r0 + r] = i < a.inp ? xs[r * ldx + i] : __float2bfloat16_rn(0.f);
    }
  }
  const int n0 = warp * NTW * 8;
  uint32_t m1 = 0u, m2 = 0u;   // ReLU masks of the warp's fragments (bit nt * 4 + e), rows < B only
  {
    const __nv_bfloat16* W1p = a.pb + blk_base(P) + z * a.tb + a.W1p;
    const float* b1 = a.params + z * P + a.oB1;
    float acc[NTW][4] = {};
    float bias[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) { bias[nt][0] = b1[n0 + nt * 8 + 2 * t]; bias[nt][1] = b1[n0 + nt * 8 + 2 * t + 1]; }
    if (a.inp > 128) warp_mma<NTW, 8>(acc, xs, ldx, W1p + (size_t)n0 * a.inp, a.inp, a.inp);
    else warp_mma<NTW>(acc, xs, ldx, W1p + (size_t)n0 * a.inp, a.inp, a.inp);
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1), b = r0 + r;
        const float zz = __fadd_rn(acc[nt][e], bias[nt][e & 1]);
        h1s[r * ldh + col] = b < B ? __float2bfloat16_rn(fmaxf(zz, 0.f)) : __float2bfloat16_rn(0.f);
        if (b < B && zz > 0.f) m1 |= 1u << (nt * 4 + e);
      }
  }
  __syncthreads();
  if (MODE == 0) cstamp(9);
  if (MODE == 0) {
    for (int idx = tid; idx < RB * HW; idx += 256) {
      const int col = idx / RB, r = idx - col * RB;
      a.H1T[((size_t)z * HW + col) * a.Bp + r0 + r] = h1s[r * ldh + col];
    }
  }
  float w3v[NTW][2];
  {
    const float* b2 = a.params + z * P + a.oB2;
    const __nv_bfloat16* W3 = a.pb + z * P + a.oW3;
    float acc[NTW][4] = {};
    float bias[NTW][2];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        bias[nt][u] = b2[n0 + nt * 8 + 2 * t + u];
        w3v[nt][u] = __bfloat162float(W3[n0 + nt * 8 + 2 * t + u]);
      }
    stage_wait(wbar);
    if (MODE == 0) cstamp(10);
    warp_mma_ss<NTW>(acc, h1s, ldh, w2s + (size_t)n0 * ldh, ldh, HW);
    float qp[2] = {0.f, 0.f};
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1), b = r0 + r;
        const float zz = __fadd_rn(acc[nt][e], bias[nt][e & 1]);
        const float h = bf16_round(fmaxf(zz, 0.f));
        qp[e >> 1] = __fmaf_rn(h, w3v[nt][e & 1], qp[e >> 1]);
        if (MODE == 0) d2s[r * ldh + col] = __float2bfloat16_rn(h);   // h2 (bf16-exact), staged for H2T
        if (b < B && zz > 0.f) m2 |= 1u << (nt * 4 + e);
      }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float s = qp[hh];
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
      s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
      if (t == 0) red[warp][g + hh * 8] = s;
    }
  }
  __syncthreads();
  if (MODE == 0) {   // h2^T for dW3 (rows past B are never read)
    for (int idx = tid; idx < RB * HW; idx += 256) {
      const int col = idx / RB, r = idx - col * RB;
      a.H2T[((size_t)z * HW + col) * a.Bp + r0 + r] = d2s[r * ldh + col];
    }
  }
  if (tid < RB) {
    float s = red[0][tid];
    for (int w = 1; w < NWARP; ++w) s = __fadd_rn(s, red[w][tid]);
    const float qv = __fadd_rn(s, b3v);
    qs[tid] = qv;
    if (r0 + tid < B) a.q[(size_t)z * B + r0 + tid] = qv;
  }
  __syncthreads();
  if (MODE == 0) cstamp(11);
  if (warp == 0) {   // dQ and the loss partial, as critic_bwd_data_mma_kernel forms them
    float d = 0.f, c = 0.f;
    const int b = r0 + lane;
    if (lane < RB && b < B) {
      const float qv = qs[lane];
      if (MODE == 0) {
        if (a.y.out && z == 0) a.y.out[b] = yv;   // TdY::get's store, with the value read up front
        const float e = __fsub_rn(qv, yv);
        d = __fdiv_rn(__fmul_rn(2.0f, e), (float)B);
        c = __fmul_rn(e, e);
      } else {
        d = a.act_scale;
        c = qv;
      }
      a.dq[(size_t)z * B + b] = d;
    }
    if (lane < RB) dqs[lane] = d;
    float cs[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) cs[r] = __shfl_sync(0xffffffffu, c, r);
    if (lane == 0) {
      float sum = 0.f;
#pragma unroll
      for (int r = 0; r < RB; ++r) sum = __fadd_rn(sum, cs[r]);
      a.part[z * a.nb + tile] = sum;
    }
  }
  __syncthreads();
  if (MODE == 0) cstamp(12);
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1);
      d2s[r * ldh + col] = __float2bfloat16_rn((m2 >> (nt * 4 + e)) & 1u ? __fmul_rn(dqs[r], w3v[nt][e & 1]) : 0.f);
    }
  __syncthreads();
  if (MODE == 0) {
    for (int idx = tid; idx < RB * HW; idx += 256) {
      const int j = idx / RB, r = idx - j * RB;
      a.dZ2T[((size_t)z * HW + j) * a.Bp + r0 + r] = d2s[r * ldh + j];
    }
  }
  {
    float acc[NTW][4] = {};
    warp_mma_ss_t<NTW>(acc, d2s, ldh, w2s + n0, ldh, HW);
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = g + (e >> 1) * 8, col = n0 + nt * 8 + 2 * t + (e & 1);
        d1s[r * ldh + col] = __float2bfloat16_rn((m1 >> (nt * 4 + e)) & 1u ? acc[nt][e] : 0.f);
      }
  }
  __syncthreads();
  if (MODE == 0) cstamp(13);
  if (MODE == 0) {
    for (int idx = tid; idx < RB * HW; idx += 256) {
      const int j = idx / RB, r = idx - j * RB;
      a.dZ1T[((size_t)z * HW + j) * a.Bp + r0 + r] = d1s[r * ldh + j];
    }
    return;
  }
  // MODE 1: columns [S, S+A) of dZ1 W1 (the tail of critic_bwd_data_mma_kernel)
  {
    __shared__ float gpart[NWARP][RB][32];
    const __nv_bfloat16* W1T = a.pb + blk_base(P) + a.W1T;
    const int c0 = a.S & ~7;
    for (int cb = c0; cb < a.S + a.A; cb += 32) {
      float acc[4][4] = {};
      const int kw = warp * (HW / NWARP);
      warp_mma<4, 2>(acc, d1s + kw, ldh, W1T + (size_t)cb * HW + kw, HW, HW / NWARP);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) gpart[warp][g + (e >> 1) * 8][nt * 8 + 2 * t + (e & 1)] = acc[nt][e];
      __syncthreads();
      for (int idx = tid; idx < RB * 32; idx += 256) {
        const int r = idx >> 5, cl = idx & 31, col = cb + cl, b = r0 + r;
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) sum = __fadd_rn(sum, gpart[w][r][cl]);
        if (b < B && col >= a.S && col < a.S + a.A) a.grad_act[(size_t)b * a.A + (col - a.S)] = sum;
      }
      __syncthreads();
    }
  }
}

// Phase A of the fused critic update: Adam over both critics (adam_elem, the arithmetic of
// adam_kernel) with the layout-aware bf16 stores. W2 goes in 32 x 32 tiles: the master / moment
// accesses and the row-major bf16 copies are coalesced along j1, and the transposed copy W2T (the
// data backward's operand) leaves through a shared-memory transpose as 64-byte row segments instead
// of one scattered 2-byte store per element (ncu/trace r02: the scattered view stores were 60 % of
// the Adam phase). Everything else (W1, biases, w3, b3) is a flat loop through store_views. The last
// CTA stores the step count and zeroes the ticket and the grid-barrier counter.
template <bool POL>
__device__ __forceinline__ void critic_adam_phase(const CritFusedArgs& a, const Bf16Views& views, const Bf16Views& tviews,
                                                  unsigned int cta, unsigned int G) {
  __shared__ float s_coef[2];
  __shared__ long long s_t;
  __shared__ unsigned short tile[32][34];
  if (threadIdx.x == 0) {
    const long long tt = *(volatile long long*)a.counter + 1;
    s_t = tt;
    adam_coefs(a.lr, a.lnb1, a.lnb2, tt, &s_coef[0], &s_coef[1]);
  }
  __syncthreads();
  const float step_size = s_coef[0], bc2_sqrt = s_coef[1];
  const float b1 = a.b1, b2 = a.b2, omb1 = 1.0f - b1, omb2 = 1.0f - b2, eps = a.eps;
  const float tau = a.tau, omt = 1.0f - tau;
  const long long P = a.P, nW2 = (long long)HW * HW, nrest = P - nW2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tiled = views.kind == 2 && (!POL || tviews.kind == 2);
  const int ntile = tiled ? 2 * (HW / 32) * (HW / 32) : 0;
  const long long nflat = tiled ? 2 * nrest : 2 * P;
  const int nft = (int)((nflat + 1023) / 1024);
  for (int task = (int)cta; task < ntile + nft; task += (int)G) {
    if (task < ntile) {
      const int z = task / 64, tr = (task % 64) / 8, tc = task % 8;
      const int j1 = tc * 32 + lane;
      float pp[4], gg[4], mm[4], vv[4], tt[4];
      long long e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j2 = tr * 32 + warp * 4 + k;
        e[k] = z * P + a.oW2 + (long long)j2 * HW + j1;
        pp[k] = a.params[e[k]]; gg[k] = a.grad2[e[k]]; mm[k] = a.m[e[k]]; vv[k] = a.v[e[k]];
        if constexpr (POL) tt[k] = a.tp[e[k]];
      }
      __nv_bfloat16* blk = views.out + blk_base(P) + z * views.tb;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j2 = tr * 32 + warp * 4 + k;
        pp[k] = adam_elem(pp[k], gg[k], mm[k], vv[k], b1, omb1, b2, omb2, bc2_sqrt, eps, step_size);
        a.params[e[k]] = pp[k]; a.m[e[k]] = mm[k]; a.v[e[k]] = vv[k];
        const unsigned short h = op16_bits(pp[k], false);
        reinterpret_cast<unsigned short*>(views.out)[e[k]] = h;
        reinterpret_cast<unsigned short*>(blk)[views.W2c + (long long)j2 * HW + j1] = h;
        tile[warp * 4 + k][lane] = h;
        if constexpr (POL) {
          const float x = __fadd_rn(__fmul_rn(tau, pp[k]), __fmul_rn(omt, tt[k]));
          a.tp[e[k]] = x;
          const unsigned short ht = op16_bits(x, false);
          reinterpret_cast<unsigned short*>(tviews.out)[e[k]] = ht;
          __nv_bfloat16* tblk = tviews.out + blk_base(P) + z * tviews.tb;
          reinterpret_cast<unsigned short*>(tblk)[tviews.W2c + (long long)j2 * HW + j1] = ht;
          if (tviews.w2t) reinterpret_cast<unsigned short*>(tblk)[tviews.W2T + (long long)j1 * HW + j2] = ht;
        }
      }
      if (views.w2t) {
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k) {   // W2T[j1][j2]: row j1 = tc 32 + warp 4 + k, the 32 j2 of the tile along the lanes
          const int j1r = warp * 4 + k;
          reinterpret_cast<unsigned short*>(blk)[views.W2T + (long long)(tc * 32 + j1r) * HW + tr * 32 + lane] =
              tile[lane][j1r];
        }
        __syncthreads();
      }
    } else {
      const long long f0 = (long long)(task - ntile) * 1024 + threadIdx.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long f = f0 + 256 * k;
        if (f >= nflat) break;
        long long ee;
        if (tiled) {
          const int z = f >= nrest ? 1 : 0;
          const long long l = f - z * nrest;
          ee = z * P + (l < a.oW2 ? l : l + nW2);
        } else {
          ee = f;
        }
        float mv = a.m[ee], vv = a.v[ee];
        const float pn = adam_elem(a.params[ee], a.grad2[ee], mv, vv, b1, omb1, b2, omb2, bc2_sqrt, eps, step_size);
        a.params[ee] = pn; a.m[ee] = mv; a.v[ee] = vv;
        store_views(views, (size_t)ee, pn);
        if constexpr (POL) {
          const float x = __fadd_rn(__fmul_rn(tau, pn), __fmul_rn(omt, a.tp[ee]));
          a.tp[ee] = x;
          store_views(tviews, (size_t)ee, x);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(a.ticket, 1u);
    if (done == G - 1) {
      *a.counter = s_t;
      *a.ticket = 0u;
      *a.gbar = 0u;
      __threadfence();
    }
  }
}

// The critic's Adam (+ Polyak) as a launch of its own (the separate-launch path): the tiled,
// layout-aware element loop of the fused update (coalesced W2T stores), same arithmetic as adam_kernel.
template <bool POL>
__global__ void __launch_bounds__(256) critic_adam_kernel(const __grid_constant__ CritFusedArgs a,
                                                          const __grid_constant__ Bf16Views views,
                                                          const __grid_constant__ Bf16Views tviews) {
  pdl_wait();
  pdl_trigger();
  critic_adam_phase<POL>(a, views, tviews, blockIdx.x, gridDim.x);
}

template <bool POL>
__global__ void __launch_bounds__(256, 1) critic_update_fused_kernel(const __grid_constant__ CritFusedArgs a,
                                                                      const __grid_constant__ Bf16Views views,
                                                                      const __grid_constant__ Bf16Views tviews) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __nv_bfloat16* const w2s = (__nv_bfloat16*)dsm;
  __nv_bfloat16* const xs = (__nv_bfloat16*)(dsm + kW2Smem);   // [RB][512 + SPAD]
  __shared__ __align__(8) uint64_t wbar;
  __shared__ __align__(16) __nv_bfloat16 h1s[RB * (HW + SPAD)];
  __shared__ __align__(16) __nv_bfloat16 d2s[RB * (HW + SPAD)];
  __shared__ __align__(16) __nv_bfloat16 d1s[RB * (HW + SPAD)];
  __shared__ float red[NWARP][RB];
  __shared__ float qs[RB], dqs[RB];
  const unsigned int G = gridDim.x, cta = blockIdx.x;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&wbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cstamp(0);
  float xv[2][16];
  if ((int)cta < 2 * a.nb) load_xtile(a, (int)cta % a.nb, xv);   // before the wait (see crit_tile)
  pdl_wait();   // no early trigger: a dependent launched before this grid is resident could take its SMs
  cstamp(1);
  unsigned int target = 0;
  // ---- F
  if ((int)cta < 2 * a.nb)
    crit_tile<0>(a, (int)cta / a.nb, (int)cta % a.nb, w2s, &wbar, xs, h1s, d2s, d1s, red, qs, dqs, xv);
  cstamp(2);
  grid_barrier(a.gbar, G, target);
  cstamp(3);
  // ---- W: weight-gradient tiles with their bias sums (crit_wtask), then the loss
  {
    const int nt = wtask_count(a.in);
    for (int task = (int)cta; task < nt; task += (int)G)
      if (!(a.dbg & 8)) crit_wtask(a, task, w2s);
    if (cta == G - 1 && a.loss) final_loss(a.part, a.nb, 2, 0, a.B, a.loss);
  }
  cstamp(4);
  grid_barrier(a.gbar, G, target);
  cstamp(5);
  pdl_trigger();   // every CTA of this grid is resident by now
  // ---- A: Adam over both critics (+ Polyak of the targets), the bf16 views; the last CTA stores the
  // step count and zeroes the barrier counter
  if (a.dbg & 2) {
    if (cta == 0 && threadIdx.x == 0) *a.gbar = 0u;
  } else if (a.dbg & 1) {
    const Bf16Views none{};
    adam_body<POL>(a.params, a.grad2, a.m, a.v, 2 * (size_t)a.P, a.counter, a.lr, a.b1, a.b2, a.eps, 0, 0, 0.f,
                   a.ticket, none, nullptr, 2.f, 0.5f, 2000, a.lnb1, a.lnb2, a.tp, a.tau, none, cta, G, a.gbar);
  } else {
    critic_adam_phase<POL>(a, views, tviews, cta, G);
  }
  cstamp(6);
}

// The actor objective's critic pass of a TD3 actor step as one launch (forward of critic 0 at
// (s, pi(s)), dQ = act_scale, data backward, dQ1/da, the actor loss -mean Q by the last CTA).
__global__ void __launch_bounds__(256, 1) critic_actor_fused_kernel(const __grid_constant__ CritFusedArgs a) {
  extern __shared__ __align__(128) uint8_t dsm[];
  __nv_bfloat16* const w2s = (__nv_bfloat16*)dsm;
  __nv_bfloat16* const xs = (__nv_bfloat16*)(dsm + kW2Smem);   // [RB][512 + SPAD]
  __shared__ __align__(8) uint64_t wbar;
  __shared__ __align__(16) __nv_bfloat16 h1s[RB * (HW + SPAD)];
  __shared__ __align__(16) __nv_bfloat16 d2s[RB * (HW + SPAD)];
  __shared__ __align__(16) __nv_bfloat16 d1s[RB * (HW + SPAD)];
  __shared__ float red[NWARP][RB];
  __shared__ float qs[RB], dqs[RB];
  __shared__ bool last;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&wbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float xv[2][16];
  load_xtile(a, blockIdx.x, xv);   // before the wait (see crit_tile)
  pdl_wait();
  pdl_trigger();
  crit_tile<1>(a, 0, blockIdx.x, w2s, &wbar, xs, h1s, d2s, d1s, red, qs, dqs, xv);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    if (a.loss) final_loss(a.part, a.nb, 1, 1, a.B, a.loss);
    if (threadIdx.x == 0) *a.ticket = 0u;
  }
}

}  // namespace

bool critic_mma_ok(const CriticDims& c) { return c.bf16 && c.H1 == HW && c.H2 == HW && c.in <= 512; }

size_t critic_bf16_elems(const CriticDims& c) {
  if (!critic_mma_ok(c)) return 2 * c.off[SPIKERL_CRITIC_NPARAM];
  const MmaLayout L = mma_layout(c);
  return blk_base(L.P) + 2 * L.tb;
}

size_t critic_mma_ws_bytes(const CriticDims& c, int B) {
  size_t total = 0;
  mma_carve(c, B, nullptr, &total);
  return total;
}

void critic_bf16_layout(const CriticDims& c, long long* o) {
  const MmaLayout L = mma_layout(c);
  o[0] = blk_base(L.P); o[1] = L.tb; o[2] = L.W1p; o[3] = L.W1T; o[4] = L.W2T; o[5] = L.W2c; o[6] = L.inp; o[7] = L.inq;
}

Bf16Views critic_bf16_views(const CriticDims& c, __nv_bfloat16* out) {
  Bf16Views v{};
  if (!out || !c.bf16) return v;
  v.out = out;
  v.P = (long long)c.off[SPIKERL_CRITIC_NPARAM];
  v.Pd = make_fastdiv((uint32_t)v.P);
  if (!critic_mma_ok(c)) { v.kind = 3; return v; }
  const MmaLayout L = mma_layout(c);
  v.kind = 2;
  v.tb = L.tb;
  v.oW1 = (long long)c.off[SPIKERL_CRITIC_W1];
  v.oW2 = (long long)c.off[SPIKERL_CRITIC_W2];
  v.W1p = L.W1p; v.W1T = L.W1T; v.W2T = L.W2T; v.W2c = L.W2c;
  v.in = c.in; v.H1 = c.H1; v.H2 = c.H2; v.inp = L.inp;
  v.w1t_lo = 0; v.w1t_hi = c.in; v.w2t = 1;   // everything (callers narrow it: TD3's targets, action rows)
  v.Pd = make_fastdiv((uint32_t)v.P); v.ind = make_fastdiv((uint32_t)c.in); v.H1d = make_fastdiv((uint32_t)c.H1);
  return v;
}

int launch_critic_refresh(const CriticDims& c, const float* params2, __nv_bfloat16* out, cudaStream_t st) {
  ProfScope ps_("critic_refresh_bf16", PB_HBM, 0.0, 6.0 * critic_bf16_elems(c), st);
  if (!critic_mma_ok(c)) return launch_f32_to_bf16(params2, out, 2 * c.off[SPIKERL_CRITIC_NPARAM], st);
  const MmaLayout L = mma_layout(c);
  const long long total = blk_base(L.P) + 2 * L.tb;
  pdl(critic_refresh_kernel, (int)(cdiv(total, 256) < 1184 ? cdiv(total, 256) : 1184), 256, 0, st)(
      params2, L.P, c.in, c.H1, c.H2, L.inp, L.inq, (long long)c.off[SPIKERL_CRITIC_W1],
      (long long)c.off[SPIKERL_CRITIC_W2], L.tb, out);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// the tcgen05 weight-gradient launch reads the transposed operands as two stacked maps: dZ1T right
// after dZ2T, H1T right after XT's 64-rounded rows (mma_carve's order); SPIKERL_CRITIC_WG_TC=0 forces
// the mma.sync split kernel
static bool tc_wgrad_ok(const CriticDims& c, const MmaWs& w, int Bp) {
  static const int env = [] { const char* e = getenv("SPIKERL_CRITIC_WG_TC"); return e ? atoi(e) : 1; }();
  const MmaLayout L = mma_layout(c);
  return env != 0 && tc_pairs_enabled() && c.H1 == HW && c.H2 == HW && L.inq <= 3 * 256 &&
         (const char*)w.dZ1T == (const char*)w.dZ2T + (size_t)2 * 2 * HW * Bp &&
         (const char*)w.H1T == (const char*)w.XT + (size_t)2 * round_up(L.inq, 64) * Bp;
}

// Large batches run the critic's contractions on the tcgen05 engine (batch on the MMA's M, the 256
// hidden units on its N). Measured crossover (tools/critic_timing.py, r02): at B = 4096 the update's
// forward + backward takes 65 us against 183 us for the warp-MMA kernels (whose 16-row tiles re-read
// W1 from L2 per tile) and the forward 25 against 39 us; at B = 1024 the warp-MMA kernels are still
// ahead (83 against 102 us per TD3 update: each tcgen05 launch is one unit deep there), so the
// engine switches at B >= 2048. SPIKERL_CRITIC_TC: 0 = never, 2 = from B = 512 on (tests; the
// weight-gradient launch's split-K plan assumes a few 64-row k-blocks, so never below that).
static bool critic_tc_ok(const CriticDims& c, int B) {
  static const int env = [] { const char* e = getenv("SPIKERL_CRITIC_TC"); return e ? atoi(e) : 1; }();
  return env != 0 && c.bf16 && c.H1 == HW && c.H2 == HW && B >= (env == 2 ? 512 : 2048);
}

static int critic_tc_fwd_bwd(const CriticDims& c, int B, const float* params2, const __nv_bfloat16* pb, const float* obs,
                             int S, const float* act, int A, const TdY* y, float* q, float* loss, float* grad2,
                             float* grad_act, float act_scale, int nz, void* ws, cudaStream_t st,
                             cudaEvent_t wait_before_loss, const float* dq_scale) {
  const MmaLayout L = mma_layout(c);
  MmaWs w = mma_carve(c, B, ws, nullptr);
  const int Bp = round_up(B, RB);
  const bool want_params = (y != nullptr && grad2 != nullptr);
  const bool need_bwd = want_params || grad_act != nullptr;
  const long long oW3 = (long long)c.off[SPIKERL_CRITIC_W3];
  const __nv_bfloat16* blk = pb + blk_base(L.P);
  const int xrows = round_up(L.inq, 64);
  const long long os = (long long)HW * Bp;
  {
    ProfScope ps_("critic_fwd_tc", PB_TENSOR, 2.0 * B * nz * ((double)c.in * HW + (double)HW * HW + HW), 0.0, st);
    pdl(critic_xt_kernel, dim3((unsigned)cdiv(Bp, 32), (unsigned)cdiv(xrows, 32)), 256, 0, st)(
        B, Bp, S, A, xrows, obs, act, w.XT, need_bwd ? w.ticket : nullptr);
    SPK_LAUNCHED();
    // layer 1: H1T = RN(relu(X W1^T + b1))^T
    SPK_TRY(launch_critic_tc(6, B, Bp, nz, w.XT, xrows, 0, blk + L.W1p, blk + L.tb + L.W1p, L.inp, L.inp,
                             params2 + c.off[SPIKERL_CRITIC_B1], nullptr, nullptr, L.P, w.H1T, os, nullptr, nullptr,
                             st));
    // layer 2 + output: H2T = RN(relu(H1 W2^T + b2))^T, q = h2 . w3 + b3
    SPK_TRY(launch_critic_tc(7, B, Bp, nz, w.H1T, 2 * HW, HW, blk + L.W2c, blk + L.tb + L.W2c, HW, HW,
                             params2 + c.off[SPIKERL_CRITIC_B2], pb + oW3, params2 + c.off[SPIKERL_CRITIC_B3], L.P,
                             w.H2T, os, nullptr, q, st));
  }
  if (wait_before_loss) SPK_CHECK_CUDA(cudaStreamWaitEvent(st, wait_before_loss, 0));
  if (!need_bwd) {
    if (y) {
      pdl(critic_loss_mma_kernel, 1, 256, 0, st)(B, nz, q, *y, w.dq, loss);
      SPK_LAUNCHED();
    }
    return SPIKERL_OK;
  }
  const int mode = want_params ? 0 : 1;
  const int nb = want_params ? nz : 1;
  {
    ProfScope ps_("critic_bwd_data_tc", PB_TENSOR, 2.0 * B * nb * ((double)HW * HW), 0.0, st);
    pdl(critic_dz2_kernel, dim3((unsigned)cdiv(Bp, 64), (unsigned)nb), 256, 0, st)(
        B, Bp, q, y ? *y : TdY{}, mode, act_scale, dq_scale, w.dq, w.part, w.ticket, (want_params || !y) ? loss : nullptr, pb, L.P,
        oW3, w.H2T, w.dZ2T);
    SPK_LAUNCHED();
    // dZ1T = RN(dZ2 W2 [h1 > 0])^T
    SPK_TRY(launch_critic_tc(8, B, Bp, nb, w.dZ2T, 2 * HW, HW, blk + L.W2T, blk + L.tb + L.W2T, HW, HW, nullptr,
                             nullptr, nullptr, L.P, w.dZ1T, os, w.H1T, nullptr, st));
    if (grad_act) {
      if (A > kGactMaxA) { set_error("critic tc path: action dim %d > %d", A, kGactMaxA); return SPIKERL_E_UNSUPPORTED; }
      pdl(critic_gact_kernel, dim3((unsigned)cdiv(B, 32)), 256, 0, st)(B, Bp, S, A, w.dZ1T, blk + L.W1T, grad_act);
      SPK_LAUNCHED();
    }
  }
  if (want_params) {
    AuxPool* aux = nullptr;
    SPK_TRY(aux_pool(&aux));
    cudaStream_t sb = aux->side[6];
    SPK_TRY(stream_after(sb, st, aux->ev[16]));
    pdl(critic_bias_grads_kernel, dim3(3 * HW + 1, nz), 256, 0, sb)(
        B, Bp, L.P, (long long)c.off[SPIKERL_CRITIC_B1], (long long)c.off[SPIKERL_CRITIC_B2], oW3,
        (long long)c.off[SPIKERL_CRITIC_B3], w.dZ1T, w.dZ2T, w.dq, (const float*)nullptr,
        (const __nv_bfloat16*)w.H2T, grad2);
    SPK_LAUNCHED();
    {
      ProfScope ps_("critic_wgrad_tc", PB_TENSOR, 2.0 * B * nz * ((double)HW * HW + (double)HW * c.in), 0.0, st);
      if (!tc_wgrad_ok(c, w, Bp)) { set_error("critic tc path: weight-gradient operands not adjacent"); return SPIKERL_E_UNSUPPORTED; }
      const long long msz = (long long)HW * HW + (long long)HW * L.inq;
      SPK_TRY(launch_critic_wgrad_tc(Bp, L.inq, round_up(L.inq, 64), w.dZ2T, w.XT, w.wpart, msz, st));
      const int splits = tc_wgrad_splits(Bp, L.inq);
      pdl(critic_wgrad_reduce_cm_kernel, dim3(cdiv(HW + c.in, 32), HW / 32, 2), dim3(32, 32), 0, st)(
          splits, c.in, msz, L.P, (long long)c.off[SPIKERL_CRITIC_W1], (long long)c.off[SPIKERL_CRITIC_W2], w.wpart,
          grad2);
      SPK_LAUNCHED();
    }
    SPK_TRY(stream_after(st, sb, aux->ev[17]));
  }
  return SPIKERL_OK;
}

int critic_mma_fwd_bwd(const CriticDims& c, int B, const float* params2, const __nv_bfloat16* pb, const float* obs,
                       int S, const float* act, int A, const TdY* y, float* q, float* loss, float* grad2,
                       float* grad_act, float act_scale, int nz, void* ws, cudaStream_t st,
                       cudaEvent_t wait_before_loss, const float* dq_scale, const CriticDecode* dec) {
  if (dec && (!critic_decode_ok(c, B, A, dec->D) || y || grad2 || grad_act)) {
    set_error("critic: in-launch decoding is for the small-batch tensor-core critic's forward only");
    return SPIKERL_E_UNSUPPORTED;
  }
  if (critic_tc_ok(c, B))
    return critic_tc_fwd_bwd(c, B, params2, pb, obs, S, act, A, y, q, loss, grad2, grad_act, act_scale, nz, ws, st,
                             wait_before_loss, dq_scale);
  const MmaLayout L = mma_layout(c);
  MmaWs w = mma_carve(c, B, ws, nullptr);
  const int Bp = round_up(B, RB);
  const bool want_params = (y != nullptr && grad2 != nullptr);
  const bool need_bwd = want_params || grad_act != nullptr;
  const long long oW3 = (long long)c.off[SPIKERL_CRITIC_W3];
  {
    ProfScope ps_("critic_fwd_mma", PB_TENSOR, 2.0 * B * nz * ((double)c.in * HW + (double)HW * HW + HW), 0.0, st);
    // one CTA per SM fits (staged W2): at most num_sms / nz CTAs per critic, each looping over tiles
    const int cap = num_sms() / nz > 0 ? num_sms() / nz : 1;
    dim3 grid(Bp / RB < cap ? Bp / RB : cap, nz);
    SPK_SMEM_ATTR(critic_fwd_mma_kernel, kW2Smem);
    pdl(critic_fwd_mma_kernel, grid, 256, kW2Smem, st)(
        B, Bp, S, A, L.inp, L.inq, obs, act, pb, L.P, L.tb, L.W1p, L.W2c, oW3, params2,
        (long long)c.off[SPIKERL_CRITIC_B1], (long long)c.off[SPIKERL_CRITIC_B2], (long long)c.off[SPIKERL_CRITIC_B3],
        w.XT, w.H1T, w.Z1, w.Z2, w.Hh2, q, need_bwd ? 1 : 0, need_bwd ? w.ticket : nullptr,
        dec ? *dec : CriticDecode{});
    SPK_LAUNCHED();
  }
  if (wait_before_loss) SPK_CHECK_CUDA(cudaStreamWaitEvent(st, wait_before_loss, 0));
  // mode 0: critic update (dQ and the MSE from y); mode 1: actor step (dQ = act_scale, critic 0,
  // scalar -mean Q). Both are formed inside the data-backward launch.
  const int mode = want_params ? 0 : 1;
  const bool fused_scalar = need_bwd && (want_params || !y);
  if (y && !fused_scalar) {
    pdl(critic_loss_mma_kernel, 1, 256, 0, st)(B, nz, q, *y, w.dq, loss);
    SPK_LAUNCHED();
  }
  if (!need_bwd) return SPIKERL_OK;
  const int nb = want_params ? nz : 1;
  {
    ProfScope ps_("critic_bwd_data_mma", PB_TENSOR, 2.0 * B * nb * ((double)HW * HW), 0.0, st);
    dim3 grid(Bp / RB, nb);
    SPK_SMEM_ATTR(critic_bwd_data_mma_kernel, kW2Smem);
    pdl(critic_bwd_data_mma_kernel, grid, 256, kW2Smem, st)(
        B, Bp, S, A, L.inp, q, y ? *y : TdY{}, mode, act_scale, w.dq, w.part, w.ticket, fused_scalar ? loss : nullptr, pb, L.P, L.tb,
        oW3, L.W1T, L.W2T, w.Z1, w.Z2, w.dZ2T, w.dZ1T, grad_act, want_params ? 1 : 0, dq_scale);
    SPK_LAUNCHED();
  }
  // merged weight + bias gradient launch (SPIKERL_CRITIC_WG_MERGE=1; default off: A/B r02 against the
  // side-stream bias kernel overlapping the weight-gradient launch, configs[1] 81.7 -> 83.7 us per
  // update, configs[3] B = 100 no different)
  static const bool merge = [] { const char* e = getenv("SPIKERL_CRITIC_WG_MERGE"); return e && e[0] == '1'; }();
  if (want_params && wgrad_splits(B) == 0 && merge) {
    // small batches: weight and bias / w3 gradients as one launch (critic_wgrad_mma_kernel)
    ProfScope ps_("critic_wgrad_mma", PB_TENSOR, 2.0 * B * nz * ((double)HW * HW + (double)HW * c.in), 0.0, st);
    const int nwx = cdiv(L.inq > HW ? L.inq : HW, 256);
    const int nby = cdiv(cdiv(3 * HW + 1, 8), nwx);
    dim3 grid(nwx, 2 * (HW / RB) + nby, nz);
    pdl(critic_wgrad_mma_kernel, grid, 256, 0, st)(Bp, c.in, L.inq, L.P, (long long)c.off[SPIKERL_CRITIC_W1],
                                                  (long long)c.off[SPIKERL_CRITIC_W2], w.XT, w.H1T, w.dZ2T, w.dZ1T,
                                                  grad2, B, (long long)c.off[SPIKERL_CRITIC_B1],
                                                  (long long)c.off[SPIKERL_CRITIC_B2], oW3,
                                                  (long long)c.off[SPIKERL_CRITIC_B3], w.dq, w.Hh2);
    SPK_LAUNCHED();
  } else if (want_params) {
    // the bias / w3 gradients run next to the weight-gradient GEMM
    AuxPool* aux = nullptr;
    SPK_TRY(aux_pool(&aux));
    cudaStream_t sb = aux->side[6];
    SPK_TRY(stream_after(sb, st, aux->ev[16]));
    pdl(critic_bias_grads_kernel, dim3(cdiv(3 * HW + 1, 8), nz), 256, 0, sb)(
        B, Bp, L.P, (long long)c.off[SPIKERL_CRITIC_B1], (long long)c.off[SPIKERL_CRITIC_B2], oW3,
        (long long)c.off[SPIKERL_CRITIC_B3], w.dZ1T, w.dZ2T, w.dq, w.Hh2, (const __nv_bfloat16*)nullptr, grad2);
    SPK_LAUNCHED();
    {
      ProfScope ps_("critic_wgrad_mma", PB_TENSOR, 2.0 * B * nz * ((double)HW * HW + (double)HW * c.in), 0.0, st);
      const int ws = wgrad_splits(B);
      if (ws == 0) {
        dim3 grid(cdiv(L.inq > HW ? L.inq : HW, 256), 2 * (HW / RB), nz);
        pdl(critic_wgrad_mma_kernel, grid, 256, 0, st)(Bp, c.in, L.inq, L.P, (long long)c.off[SPIKERL_CRITIC_W1],
                                                      (long long)c.off[SPIKERL_CRITIC_W2], w.XT, w.H1T, w.dZ2T, w.dZ1T,
                                                      grad2, B, 0, 0, 0, 0, w.dq, w.Hh2);   // (no bias CTAs)
        SPK_LAUNCHED();
      } else if (tc_wgrad_ok(c, w, Bp)) {
        // tcgen05: both weight gradients of both critics as one split-K launch of K-major operand
        // tiles (the mma.sync split kernel below took 104 us at configs[3] B = 4096)
        const long long msz = (long long)HW * HW + (long long)HW * L.inq;
        SPK_TRY(launch_critic_wgrad_tc(Bp, L.inq, round_up(L.inq, 64), w.dZ2T, w.XT, w.wpart, msz, st));
        const int splits = tc_wgrad_splits(Bp, L.inq);
        pdl(critic_wgrad_reduce_cm_kernel, dim3(cdiv(HW + c.in, 32), HW / 32, 2), dim3(32, 32), 0, st)(
            splits, c.in, msz, L.P, (long long)c.off[SPIKERL_CRITIC_W1], (long long)c.off[SPIKERL_CRITIC_W2], w.wpart,
            grad2);
        SPK_LAUNCHED();
      } else {
        // K split in multiples of 16 batch rows (Bp is a multiple of RB = 16)
        const int kc = round_up(cdiv(Bp, ws), 16), splits = cdiv(Bp, kc);
        const int blocks = (HW / 64) * (HW / 128) + (HW / 64) * cdiv(L.inq, 128);
        pdl(critic_wgrad_split_kernel, dim3(blocks, splits, nz), 256, 0, st)(
            Bp, c.in, L.inq, kc, L.P, (long long)c.off[SPIKERL_CRITIC_W1], (long long)c.off[SPIKERL_CRITIC_W2], w.XT,
            w.H1T, w.dZ2T, w.dZ1T, grad2, w.wpart);
        SPK_LAUNCHED();
        if (splits > 1) {
          pdl(critic_wgrad_reduce_kernel, 148 * 4, 256, 0, st)(splits, c.in, L.inq, L.P, (long long)c.off[SPIKERL_CRITIC_W1],
                                                             (long long)c.off[SPIKERL_CRITIC_W2], w.wpart, grad2);
          SPK_LAUNCHED();
        }
      }
    }
    SPK_TRY(stream_after(st, sb, aux->ev[17]));
  }
  return SPIKERL_OK;
}


// ------------------------------------------------------------------ fused small-batch launches
// SPIKERL_CRITIC_FUSED: 1 = every eligible batch (B <= 512), 0 = never; default from B = 384 (r02 A/B,
// one box: configs[2] B = 512 116.6 -> 110.5 us per update; configs[1] B = 256 84.5 -> 86.9 and configs[3]
// B = 100 114.2 -> 135.3 slower: there the separate forward overlaps the target path and the phases'
// dependent round trips outweigh the launches saved)
bool critic_fused_ok(const CriticDims& c, int B) {
  static const int env = [] { const char* e = getenv("SPIKERL_CRITIC_FUSED"); return e ? atoi(e) : -1; }();
  if (env == 0 || (env < 0 && B < 384)) return false;
  return critic_mma_ok(c) && !critic_tc_ok(c, B) && wgrad_splits(B) == 0 && 2 * (round_up(B, RB) / RB) <= num_sms();
}

static CritFusedArgs fused_args(const CriticDims& c, int B, float* params2, const __nv_bfloat16* pb, const float* obs,
                                int S, const float* act, int A, void* ws) {
  const MmaLayout L = mma_layout(c);
  const MmaWs w = mma_carve(c, B, ws, nullptr);
  CritFusedArgs a{};
  a.B = B; a.Bp = round_up(B, RB); a.S = S; a.A = A; a.inp = L.inp; a.inq = L.inq; a.in = c.in; a.nb = a.Bp / RB;
  a.obs = obs; a.act = act; a.pb = pb;
  a.P = L.P; a.tb = L.tb; a.W1p = L.W1p; a.W2c = L.W2c; a.W1T = L.W1T;
  a.oW3 = (long long)c.off[SPIKERL_CRITIC_W3]; a.oB1 = (long long)c.off[SPIKERL_CRITIC_B1];
  a.oB2 = (long long)c.off[SPIKERL_CRITIC_B2]; a.oB3 = (long long)c.off[SPIKERL_CRITIC_B3];
  a.oW1 = (long long)c.off[SPIKERL_CRITIC_W1]; a.oW2 = (long long)c.off[SPIKERL_CRITIC_W2];
  a.params = params2;
  a.dq = w.dq; a.part = w.part; a.H2T = w.H2T;
  a.XT = w.XT; a.H1T = w.H1T; a.dZ2T = w.dZ2T; a.dZ1T = w.dZ1T;
  return a;
}

// grid of the fused update: every row tile of both critics, and 96 CTAs (at least) for the weight-gradient
// and Adam phases (configs[2] per update, late r02, three alternating rounds: 64 CTAs 101.9, 96 100.5,
// 128 102.5, 148 101.7 us) (SPIKERL_CRITIC_FUSED_G overrides; always <= the SM count: the grid barriers need
// the whole grid resident)
static int fused_grid(int tiles) {
  static const int env = [] { const char* e = getenv("SPIKERL_CRITIC_FUSED_G"); return e ? atoi(e) : 96; }();
  int g = tiles > env ? tiles : env;
  return g < num_sms() ? g : num_sms();
}

int critic_update_fused(const CriticDims& c, int B, float* params2, const __nv_bfloat16* pb, const float* obs, int S,
                        const float* act, int A, const TdY& y, float* q, float* loss, float* grad2, void* ws,
                        float* m, float* v, long long* steps, float lr, float b1, float b2, float eps,
                        const Bf16Views* views, const PolyakFuse* polyak, cudaStream_t st) {
  if (!critic_fused_ok(c, B)) { set_error("critic_update_fused: unsupported shape"); return SPIKERL_E_UNSUPPORTED; }
  if (((uintptr_t)params2 | (uintptr_t)grad2 | (uintptr_t)m | (uintptr_t)v | (uintptr_t)(polyak ? polyak->t : nullptr)) & 15) {
    set_error("critic_update_fused: buffers must be 16-byte aligned");
    return SPIKERL_E_ARG;
  }
  CritFusedArgs a = fused_args(c, B, params2, pb, obs, S, act, A, ws);
  a.y = y; a.q = q; a.loss = loss; a.grad2 = grad2;
  a.m = m; a.v = v; a.counter = steps;
  a.ticket = (unsigned int*)(steps + 1);           // Adam's ticket (low word of steps[1])
  a.gbar = (unsigned int*)(steps + 1) + 1;         // the grid barrier (high word; 0 at rest)
  a.lr = lr; a.b1 = b1; a.b2 = b2; a.eps = eps; a.lnb1 = log((double)b1); a.lnb2 = log((double)b2);
  a.tp = polyak ? polyak->t : nullptr; a.tau = polyak ? polyak->tau : 0.f;
  static const int dbg = [] { const char* e = getenv("SPIKERL_CRITIC_FUSED_DBG"); return e ? atoi(e) : 0; }();
  a.dbg = dbg;
  const Bf16Views none{};
  const int G = fused_grid(2 * a.nb);
  const double fl = 2.0 * B * 2 * ((double)c.in * HW + (double)HW * HW + HW) * 3.0;
  ProfScope ps_(polyak ? "critic_update_fused_polyak" : "critic_update_fused", PB_TENSOR, fl, 0.0, st);
  if (polyak) {
    SPK_SMEM_ATTR(critic_update_fused_kernel<true>, kFusedSmem);
    pdl(critic_update_fused_kernel<true>, G, 256, kFusedSmem, st)(a, views ? *views : none,
                                                               polyak->views ? *polyak->views : none);
  } else {
    SPK_SMEM_ATTR(critic_update_fused_kernel<false>, kFusedSmem);
    pdl(critic_update_fused_kernel<false>, G, 256, kFusedSmem, st)(a, views ? *views : none, none);
  }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

bool critic_decode_ok(const CriticDims& c, int B, int A, int D) {
  static const bool env = [] { const char* e = getenv("SPIKERL_CRITIC_DECODE"); return !(e && e[0] == '0'); }();
  return env && critic_mma_ok(c) && !critic_tc_ok(c, B) && A <= 32 && D <= kDecMaxD;
}

bool critic_adam_ok(const CriticDims& c, const Bf16Views* views, const PolyakFuse* polyak) {
  return critic_mma_ok(c) && views && views->kind == 2 && (!polyak || (polyak->views && polyak->views->kind == 2));
}

int launch_critic_adam(const CriticDims& c, float* params2, const float* grad2, float* m, float* v, long long* steps,
                       float lr, float b1, float b2, float eps, const Bf16Views* views, const PolyakFuse* polyak,
                       cudaStream_t st) {
  if (!critic_adam_ok(c, views, polyak)) { set_error("critic adam: needs the tensor-core critic's bf16 views"); return SPIKERL_E_ARG; }
  const MmaLayout L = mma_layout(c);
  CritFusedArgs a{};
  a.P = L.P; a.oW2 = (long long)c.off[SPIKERL_CRITIC_W2];
  a.params = params2; a.grad2 = const_cast<float*>(grad2); a.m = m; a.v = v; a.counter = steps;
  a.ticket = (unsigned int*)(steps + 1); a.gbar = (unsigned int*)(steps + 1) + 1;
  a.lr = lr; a.b1 = b1; a.b2 = b2; a.eps = eps; a.lnb1 = log((double)b1); a.lnb2 = log((double)b2);
  a.tp = polyak ? polyak->t : nullptr; a.tau = polyak ? polyak->tau : 0.f;
  const long long nrest = L.P - (long long)HW * HW;
  const int tasks = 2 * (HW / 32) * (HW / 32) + (int)((2 * nrest + 1023) / 1024);
  const int G = tasks < 2 * num_sms() ? tasks : 2 * num_sms();
  const Bf16Views none{};
  ProfScope ps_(polyak ? "adam_polyak" : "adam", PB_HBM, 0.0, (polyak ? 40.0 : 28.0) * 2 * L.P, st);
  if (polyak)
    pdl(critic_adam_kernel<true>, G, 256, 0, st)(a, *views, *polyak->views);
  else
    pdl(critic_adam_kernel<false>, G, 256, 0, st)(a, *views, none);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// the actor objective's critic pass as one launch: SPIKERL_CRITIC_ACT_FUSED=0 turns it off
bool critic_act_fused_ok(const CriticDims& c, int B) {
  static const int env = [] { const char* e = getenv("SPIKERL_CRITIC_ACT_FUSED"); return e ? atoi(e) : 1; }();
  return env != 0 && critic_mma_ok(c) && !critic_tc_ok(c, B) && wgrad_splits(B) == 0;
}

int critic_actor_fused(const CriticDims& c, int B, const float* params2, const __nv_bfloat16* pb, const float* obs,
                       int S, const float* act, int A, float* q, float* loss, float* grad_act, float act_scale,
                       void* ws, unsigned int* ticket, cudaStream_t st) {
  if (!critic_act_fused_ok(c, B)) { set_error("critic_actor_fused: unsupported shape"); return SPIKERL_E_UNSUPPORTED; }
  CritFusedArgs a = fused_args(c, B, const_cast<float*>(params2), pb, obs, S, act, A, ws);
  a.q = q; a.loss = loss; a.grad_act = grad_act; a.act_scale = act_scale; a.ticket = ticket;
  ProfScope ps_("critic_actor_fused", PB_TENSOR, 2.0 * B * ((double)c.in * HW + 2.0 * HW * HW + HW), 0.0, st);
  SPK_SMEM_ATTR(critic_actor_fused_kernel, kFusedSmem);
  pdl(critic_actor_fused_kernel, a.nb, 256, kFusedSmem, st)(a);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

}  // namespace spk

extern "C" int spikerl_debug_critic_trace(unsigned long long* host8) {
  if (cudaMemcpyFromSymbol(host8, spk::g_ctrace, sizeof(unsigned long long) * 16) != cudaSuccess) return 5;
  return 0;
}
