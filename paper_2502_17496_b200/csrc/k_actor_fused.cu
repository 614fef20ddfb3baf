// k_actor_fused.cu — latency-regime actor forward: the Gaussian encoder,
// the three LIF layers and the decoder of a small batch in ONE launch, instead of five kernels
// whose launch / ramp latencies dominate at TD3 batch sizes (configs[0..1]: 0.1 GFLOP per call).
//   PAPER.md:131 (§III-A population encoder, LIF neurons, firing-rate decoder); north_star
//   (c = d_c c + W o, v = d_v v (1 - o_prev) + c, o = [v > V_th]).
// Work split: a cluster of C = 4 CTAs owns 16 batch rows; CTA c owns 1/C of every layer's
// (padded) neurons. Per layer, each CTA computes its neuron slice for all 16 rows and all T steps
// with warp-level bf16 tensor-core MMAs (mma.sync m16n8k16, fp32 accumulate; the spike operand
// {0,1} is exact) — rows are (t, b) t-major, so m-tile t holds timestep t and every thread owns
// all T steps of its (b, neuron) accumulators: the LIF scan never leaves registers. The slice of
// spikes is then pushed to the 3 peer CTAs with bulk DSMEM copies (cp.async.bulk ... shared::cluster)
// completing on the peers' mbarriers, so the next layer reads the whole spike operand from local
// shared memory. The tape written is exactly the tcgen05 engine's (A, bit / mask planes, quad-major
// copies, counts, actions), so the backward is unchanged.
#include "internal.h"

namespace spk {
namespace fused {

constexpr int C = 4;       // CTAs per cluster (8-CTA clusters: only 15 co-resident on B200 -> 2 waves at B = 256)
constexpr int RB = 16;     // batch rows per cluster
constexpr int NWARP = 8;
constexpr int NTH = 32 * NWARP;
constexpr int SPAD = 8;    // bf16 row padding of an operand slice (conflict-free ldmatrix)
constexpr int WPAD = 8;    // bf16 row padding of a weight slice
constexpr int MAXT = 8;    // m-tiles (timesteps) kept in registers

struct Params {
  int B, S, E, K0, T, A, D, N3;
  int P[4], N[4], Wd[4];
  const float *obs, *mu, *sigma, *Wdec, *bdec;
  const __nv_bfloat16* W[3];
  LifConst kc;
  float* A_tape;
  uint32_t* bits[4];
  uint32_t* mask[4];
  uint8_t* counts;
  float *act_out, *act_tape;
  uint8_t* bitsT[4];
  uint8_t* maskT[4];
  int tpad;
  int buf_bytes;   // one operand buffer: C slices x R rows x (max slice + SPAD) bf16
};

__host__ __device__ inline int slice(const Params& p, int l) { return p.P[l] / C; }
// flags of layer l are replicated to every CTA of the cluster when a 32-neuron word of the bit
// planes spans CTAs, and for the output layer (counts / decoder need all of its neurons)
__host__ __device__ inline bool repl(const Params& p, int l) { return l == 3 || slice(p, l) % 32 != 0; }

struct Smem {   // offsets into dynamic shared memory
  int buf[2], w[3], flags[4], red, bar, total;
};

__host__ __device__ inline Smem smem_layout(const Params& p) {
  Smem s{};
  const int R = RB * p.T;
  int o = 0;
  auto take = [&](int bytes) { const int r = o; o += (bytes + 127) & ~127; return r; };
  for (int i = 0; i < 2; ++i) s.buf[i] = take(p.buf_bytes);
  for (int l = 1; l <= 3; ++l) s.w[l - 1] = take(slice(p, l) * (p.P[l - 1] + WPAD) * 2);
  for (int l = 0; l < 4; ++l) s.flags[l] = take(R * (repl(p, l) ? p.P[l] : slice(p, l)));
  int rw = 0;   // warps that park partial accumulators (k-split layers)
  for (int l = 1; l <= 3; ++l) if (NWARP - slice(p, l) / 8 > rw) rw = NWARP - slice(p, l) / 8;
  s.red = take(max(rw * 32 * p.T * 4 * 4, RB * p.P[3]));   // also the decoder's count scratch
  s.bar = take(64);
  s.total = o;
  return s;
}

// ------------------------------------------------------------------ cluster / async-copy PTX
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// bulk copy shared(this CTA) -> shared(peer), completing `bytes` of transaction on the peer's mbarrier
__device__ __forceinline__ void bulk_to_peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
      "r"(src), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
// bulk copy global -> shared(this CTA)
__device__ __forceinline__ void bulk_from_global(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// all but the most recent committed group have finished reading their source
__device__ __forceinline__ void bulk_wait_read_prev() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// not volatile: the compiler may batch the fragment loads of several m-tiles ahead of their MMAs
// (the "memory" clobber keeps them ordered with the barriers and stores around them)
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void ldsm_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
  asm("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr) : "memory");
}

// phase timeline of CTA 0 of the last launch (diagnostics; spikerl_debug_fused_trace)
__device__ unsigned long long g_ftrace[16];
__device__ __forceinline__ void fstamp(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_ftrace[i] = t;
  }
}

// ------------------------------------------------------------------ one LIF layer (slice of neurons)
// in:   operand buffer with every CTA's spike slice of layer l-1 ([C][R][S_in + SPAD] bf16)
// wsl:  this CTA's rows of W_l ([S_out][P_{l-1} + WPAD] bf16, preloaded)
// out:  this CTA's spike slice of layer l ([R][S_out + SPAD] bf16; null for layer 3)
// flg:  this CTA's flags [R][S_out] u8 (bit 0 spike, bit 1 surrogate window)
// Warp w takes n-tile w % NT and the k-range (w / NT) of KS = NWARP / NT equal parts; partial
// accumulators are added in a fixed order (deterministic) by the k-range-0 warp, which runs the scan.
// not inlined: the three layers share one copy of the code (the kernel runs each phase once per
// launch, so instruction-cache misses on ~3x the code cost more than the call)
template <int TT>
__device__ __noinline__ void lif_layer(const Params& p, int l, int c, const __nv_bfloat16* in,
                                          const __nv_bfloat16* wsl, __nv_bfloat16* out, uint8_t* flg,
                                          float* red, int warp, int lane) {
  constexpr int MT = TT > 0 ? TT : MAXT;   // m-tiles held in registers
  const int T = TT > 0 ? TT : p.T, R = RB * T;
  const int S_in = slice(p, l - 1), S_out = slice(p, l);
  const int ld_in = S_in + SPAD, ld_out = S_out + SPAD, ldw = p.P[l - 1] + WPAD;
  const int NT = S_out / 8, KS = NWARP / NT, Kpart = p.P[l - 1] / KS;
  const int nt = warp % NT, ks = warp / NT;
  const int g = lane >> 2, t4 = lane & 3;
  float acc[MT][4];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
  const uint32_t in_s = smem_u32(in);
  const uint32_t b_addr = smem_u32(wsl) + 2u * (uint32_t)((nt * 8 + (lane & 7)) * ldw + ((lane >> 3) & 1) * 8);
  const uint32_t a_lane = 2u * (uint32_t)((lane & 15) * ld_in + (lane >> 4) * 8);
#pragma unroll 2
  for (int k = ks * Kpart; k < (ks + 1) * Kpart; k += 16) {
    uint32_t b0, b1, a[MT][4];
    ldsm_x2(b0, b1, b_addr + 2u * k);
    const int sl = k / S_in, kk = k - sl * S_in;
    const uint32_t ab = in_s + 2u * (uint32_t)(sl * R * ld_in + kk) + a_lane;
#pragma unroll
    for (int m = 0; m < MT; ++m)
      if (m < T) ldsm_x4(a[m], ab + 2u * (uint32_t)(m * RB * ld_in));
#pragma unroll
    for (int m = 0; m < MT; ++m)
      if (m < T) mma16816(acc[m], a[m], b0, b1);
  }
  float* my = red + ((size_t)(warp - NT) * 32 + lane) * T * 4;   // warps NT.. park partials
  if (ks > 0) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
      if (m < T) reinterpret_cast<float4*>(my)[m] = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
  }
  __syncthreads();
  if (ks > 0) return;
  for (int j2 = 1; j2 < KS; ++j2) {
    const float4* o = reinterpret_cast<const float4*>(red + ((size_t)(warp + j2 * NT - NT) * 32 + lane) * T * 4);
#pragma unroll
    for (int m = 0; m < MT; ++m)
      if (m < T) {
        const float4 v = o[m];
        acc[m][0] = __fadd_rn(acc[m][0], v.x); acc[m][1] = __fadd_rn(acc[m][1], v.y);
        acc[m][2] = __fadd_rn(acc[m][2], v.z); acc[m][3] = __fadd_rn(acc[m][3], v.w);
      }
  }
  // LIF scan over t (the m-tiles) for this thread's 2 batch rows x 2 neurons
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int j = g + 8 * (e >> 1), col = nt * 8 + 2 * t4 + (e & 1), n = c * S_out + col;
    const bool valid = n < p.N[l];
    const LifConst kc{p.kc.dc, p.kc.dv, valid ? p.kc.vth : __int_as_float(0x7f800000), valid ? p.kc.win : -1.f};
    float cc = 0.f, vv = 0.f;
    bool o = false, h = false;
#pragma unroll
    for (int m = 0; m < MT; ++m)
      if (m < T) {
        lif_step(kc, acc[m][e], cc, vv, o, h);
        const int r = m * RB + j;
        if (out) out[r * ld_out + col] = __float2bfloat16_rn(o ? 1.f : 0.f);
        flg[r * S_out + col] = (uint8_t)((o ? 1 : 0) | (h ? 2 : 0));
      }
  }
}

// bit / mask plane words of layer l for this cluster's 16 rows. Replicated flags: words
// w = c, c + C, ... from every CTA's slot; else this CTA's own words from its own flags.
__device__ __forceinline__ void pack_planes(const Params& p, int l, int c, int q, const uint8_t* fl, int warp, int lane) {
  const int T = p.T, R = RB * T, S = slice(p, l);
  const bool rp = repl(p, l);
  const int w0 = rp ? c : c * S / 32, w1 = rp ? p.Wd[l] : (c + 1) * S / 32, ws = rp ? C : 1;
  for (int w = w0; w < w1; w += ws) {
    const int n = 32 * w + lane;
    const uint8_t* base = rp ? fl + (size_t)(n / S) * R * S + (n % S) : fl + (n - c * S);
    for (int r = warp; r < R; r += NWARP) {
      const uint32_t f = base[r * S];
      const uint32_t wo = __ballot_sync(0xffffffffu, f & 1u), wh = __ballot_sync(0xffffffffu, f & 2u);
      const int t = r / RB, b = q * RB + (r - t * RB);
      if (lane == 0 && b < p.B) {
        const size_t wi = ((size_t)t * p.B + b) * p.Wd[l] + w;
        p.bits[l][wi] = wo;
        if (l) p.mask[l][wi] = wh;
      }
    }
  }
}

// quad-major copies of this CTA's neurons (layers 1, 2; read by the tcgen05 DX epilogue): one
// 64-bit word per (batch quad, neuron), nibble t = the quad's bits at step t (T <= 16)
__device__ __forceinline__ void pack_quads(const Params& p, int l, int c, int q, const uint8_t* flags, int tid) {
  const int S = slice(p, l);
  if (tid >= 4 * S) return;
  const int nl = tid % S, qd = tid / S, n = c * S + nl;
  unsigned long long wo = 0ull, wh = 0ull;
  for (int t = 0; t < p.T; ++t) {
    uint32_t bo = 0, bh = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t f = flags[(t * RB + 4 * qd + j) * S + nl];
      bo |= (f & 1u) << j;
      bh |= ((f >> 1) & 1u) << j;
    }
    wo |= (unsigned long long)bo << (4 * t);
    wh |= (unsigned long long)bh << (4 * t);
  }
  const size_t off = ((size_t)(4 * q + qd) * p.P[l] + n) * (p.tpad >> 1);
  *reinterpret_cast<unsigned long long*>(p.bitsT[l] + off) = wo;
  *reinterpret_cast<unsigned long long*>(p.maskT[l] + off) = wh;
}

template <int TT>
__global__ void __launch_bounds__(NTH, 1) actor_fwd_fused_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t sm[];
  const Smem L = smem_layout(p);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = (int)cta_rank(), q = blockIdx.x / C;
  const int T = TT > 0 ? TT : p.T, R = RB * T;
  __nv_bfloat16* const buf0 = (__nv_bfloat16*)(sm + L.buf[0]);
  __nv_bfloat16* const buf1 = (__nv_bfloat16*)(sm + L.buf[1]);
  float* const red = (float*)(sm + L.red);
  const uint32_t bar0 = smem_u32(sm + L.bar), wbar = bar0 + 32;
  auto flags_of = [&](int l, int slot) {   // this CTA's (or slot's) flag block of layer l
    return sm + L.flags[l] + (repl(p, l) ? (size_t)slot * R * slice(p, l) : 0);
  };
  auto xbytes = [&](int l) {   // bytes one CTA pushes to each peer for layer l (bf16 slice + flags)
    return (uint32_t)((l <= 2 ? R * (slice(p, l) + SPAD) * 2 : 0) + (repl(p, l) ? R * slice(p, l) : 0));
  };
  if (tid == 0) {
    for (int l = 0; l < 4; ++l) {
      mbar_init(bar0 + 8 * l, 1);
      // the 7 peers' slices of layer l land here (one phase per launch)
      mbar_expect_tx(bar0 + 8 * l, (uint32_t)(C - 1) * xbytes(l));
    }
    mbar_init(wbar, 1);
    uint32_t wb = 0;
    for (int l = 1; l <= 3; ++l) wb += (uint32_t)(slice(p, l) * p.P[l - 1] * 2);
    mbar_expect_tx(wbar, wb);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fstamp(0);
  cluster_sync();   // every barrier of the cluster exists before any remote complete_tx
  pdl_wait();
  pdl_trigger();
  fstamp(1);
  // this CTA's rows of W1..W3 (bf16 working copies, current after pdl_wait): one bulk copy per row
  if (warp == 0) {
    for (int l = 1; l <= 3; ++l) {
      const int S = slice(p, l), K = p.P[l - 1];
      const uint32_t dst = smem_u32(sm + L.w[l - 1]);
      for (int r = lane; r < S; r += 32)
        bulk_from_global(dst + (uint32_t)(r * (K + WPAD) * 2), p.W[l - 1] + (size_t)(c * S + r) * K, (uint32_t)(K * 2), wbar);
    }
  }

  // ---------------- encoder: this CTA's slice of the K0 population inputs, all 16 rows
  {
    const int S0 = slice(p, 0), ld0 = S0 + SPAD;
    __nv_bfloat16* o0 = buf0 + (size_t)c * R * ld0;
    uint8_t* f0 = flags_of(0, c);
    for (int idx = tid; idx < RB * S0; idx += NTH) {
      const int j = idx / S0, kl = idx - j * S0, k = c * S0 + kl, b = q * RB + j;
      float A = 0.f;
      if (k < p.K0 && b < p.B) {
        // identical operation sequence to enc_fwd_kernel (R4)
        const double m = (double)__ldg(p.mu + k), sg = (double)__ldg(p.sigma + k);
        const double den = __dmul_rn(2.0, __dmul_rn(sg, sg));
        const double dd = __dsub_rn((double)__ldg(p.obs + (size_t)b * p.S + k / p.E), m);
        A = (float)exp(-__ddiv_rn(__dmul_rn(dd, dd), den));
        p.A_tape[(size_t)b * p.K0 + k] = A;
      }
      float acc = 0.f;
      for (int t = 0; t < T; ++t) {
        acc = __fadd_rn(acc, A);
        const bool fire = acc >= 1.0f;
        if (fire) acc = __fsub_rn(acc, 1.0f);
        o0[(t * RB + j) * ld0 + kl] = __float2bfloat16_rn(fire ? 1.f : 0.f);
        f0[(t * RB + j) * S0 + kl] = fire ? 1 : 0;
      }
    }
  }
  fstamp(2);
  // ---------------- layers: exchange layer li's slice (+ flags), then compute layer li + 1
  for (int li = 0; li <= 3; ++li) {
    const int S = slice(p, li), ld = S + SPAD;
    __nv_bfloat16* src_buf = (li & 1) ? buf1 : buf0;
    __syncthreads();                    // this CTA's slice + flags of layer li are complete
    if (tid == 0) {
      fence_proxy_async();              // generic-proxy stores -> visible to the bulk copies
      const uint32_t fsrc = smem_u32(flags_of(li, c)), fbytes = (uint32_t)(R * S);
      const uint32_t src = smem_u32(src_buf + (size_t)c * R * ld), bytes = (uint32_t)(R * ld * 2);
      for (int pr = 1; pr < C; ++pr) {
        const uint32_t peer = (uint32_t)((c + pr) % C), bar = mapa(bar0 + 8 * li, peer);
        if (li <= 2) bulk_to_peer(mapa(src, peer), src, bytes, bar);
        if (repl(p, li)) bulk_to_peer(mapa(fsrc, peer), fsrc, fbytes, bar);
      }
      bulk_commit();
    }
    fstamp(3 + 3 * li);
    const bool own = li <= 2 && !repl(p, li);   // words from this CTA's own flags: pack while copies fly
    if (own) pack_planes(p, li, c, q, sm + L.flags[li], warp, lane);
    if (li == 1 || li == 2) pack_quads(p, li, c, q, flags_of(li, c), tid);
    mbar_wait(bar0 + 8 * li, 0);        // all 7 peer slices of layer li have landed
    fstamp(4 + 3 * li);
    if (li <= 2 && !own) pack_planes(p, li, c, q, sm + L.flags[li], warp, lane);
    if (li == 3) break;
    if (li == 0) mbar_wait(wbar, 0);    // weight slices in shared memory
    // layer li + 1 overwrites the buffer that held layer li - 1's slice: its outgoing copies are done
    if (tid == 0) bulk_wait_read_prev();
    __syncthreads();
    fstamp(5 + 3 * li);
    const int l = li + 1;
    lif_layer<TT>(p, l, c, src_buf, (const __nv_bfloat16*)(sm + L.w[l - 1]),
              l < 3 ? ((l & 1) ? buf1 : buf0) + (size_t)c * R * (slice(p, l) + SPAD) : nullptr,
              flags_of(l, c), red, warp, lane);
  }
  fstamp(13);
  // ---------------- output layer: planes, counts and decoder from the replicated flags
  {
    const int S3 = slice(p, 3), P3 = p.P[3];
    const uint8_t* f3 = sm + L.flags[3];
    uint8_t* cnt = (uint8_t*)red;       // [RB][P3] spike counts (the partial-sum scratch is free now)
    for (int idx = tid; idx < RB * P3; idx += NTH) {
      const int j = idx / P3, n = idx - j * P3;
      const uint8_t* f = f3 + ((size_t)(n / S3) * R + j) * S3 + (n % S3);
      int ct = 0;
      for (int t = 0; t < T; ++t) ct += f[t * RB * S3] & 1;
      cnt[idx] = (uint8_t)ct;
      const int b = q * RB + j;
      if (n < p.N3 && b < p.B && n / S3 == c) p.counts[(size_t)b * p.N3 + n] = (uint8_t)ct;
    }
    pack_planes(p, 3, c, q, f3, warp, lane);
    __syncthreads();
    // a_j = tanh(sum_d Wd[j][d] cnt[jD+d] / T + bd[j]) (dec_fwd_kernel's arithmetic); actions j = c, c+C, ...
    for (int idx = tid; idx < RB * p.A; idx += NTH) {
      const int j = idx / p.A, a = idx - j * p.A, b = q * RB + j;
      if ((a % C) != c || b >= p.B) continue;
      float pre = 0.f;
      for (int e = 0; e < p.D; ++e) {
        const int n = a * p.D + e;
        const float fr = (float)cnt[j * P3 + n] / (float)T;
        pre = __fadd_rn(pre, __fmul_rn(p.Wdec[a * p.D + e], fr));
      }
      pre = __fadd_rn(pre, p.bdec[a]);
      const float av = tanhf(pre);
      p.act_out[(size_t)b * p.A + a] = av;
      if (p.act_tape) p.act_tape[(size_t)b * p.A + a] = av;
    }
  }
  // every incoming copy completed before the waits above; outgoing ones must finish reading
  // this CTA's shared memory before it exits
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  fstamp(14);
}

}  // namespace fused

using namespace fused;

static Params fused_params(const ActorDims& d, int B) {
  Params p{};
  p.B = B; p.S = d.S; p.E = d.E; p.K0 = d.K0; p.T = d.T; p.A = d.A; p.D = d.D; p.N3 = d.N3;
  int mx = 0;
  for (int l = 0; l < 4; ++l) {
    p.P[l] = d.P[l]; p.N[l] = d.N[l]; p.Wd[l] = d.Wd[l];
    if (l < 3 && d.P[l] / C > mx) mx = d.P[l] / C;
  }
  p.buf_bytes = C * RB * d.T * (mx + SPAD) * 2;
  p.tpad = round_up(d.T, 16);
  return p;
}

bool fused_fwd_ok(const ActorDims& d, int B) {
  if (d.f16) return false;   // bf16 operands only
  // opt-in (SPIKERL_FUSED_FWD=1): measured on B200 at configs[1] (B = 256) one launch takes
  // 34.6 us against 28.8 us for the five-kernel chain it replaces (one CTA of 8 warps per SM
  // leaves every phase latency-bound), so the chain stays the default
  static int env = -1;
  if (env < 0) { const char* e = getenv("SPIKERL_FUSED_FWD"); env = (e && e[0] == '1') ? 1 : 0; }
  if (!env || !d.bf16 || d.engine != SPIKERL_ENGINE_TCGEN05) return false;
  if (d.T > MAXT || B > 2048) return false;
  for (int l = 0; l < 4; ++l) {
    if (d.P[l] % (C * 16) != 0 || d.P[l] / C > 64) return false;
    const int nt = d.P[l] / C / 8;   // n-tiles per CTA must divide the 8 warps (k-split)
    if (l && NWARP % nt != 0) return false;
  }
  if (round_up(d.T, 16) != 16) return false;          // quad planes: one u64 per (quad, neuron)
  const Params p = fused_params(d, B);
  return smem_layout(p).total <= 220 * 1024;
}

int launch_actor_fwd_fused(const ActorDims& d, int B, const float* obs, const float* params,
                           const __nv_bfloat16* pb16, const TapeLayout& L, char* tape, float* actions,
                           cudaStream_t st) {
  ProfScope ps_("actor_fwd_fused", PB_TENSOR,
                2.0 * d.T * B * ((double)d.N1 * d.K0 + (double)d.N2 * d.N1 + (double)d.N3 * d.N2), 0.0, st);
  Params p = fused_params(d, B);
  p.obs = obs;
  p.mu = params + d.off[SPIKERL_ACTOR_MU];
  p.sigma = params + d.off[SPIKERL_ACTOR_SIGMA];
  p.Wdec = params + d.off[SPIKERL_ACTOR_WD];
  p.bdec = params + d.off[SPIKERL_ACTOR_BD];
  for (int l = 0; l < 3; ++l) p.W[l] = pb16 + d.boff[l];
  p.kc = LifConst{d.dc, d.dv, d.vth, d.win};
  p.A_tape = (float*)(tape + L.A);
  for (int l = 0; l < 4; ++l) {
    p.bits[l] = (uint32_t*)(tape + L.bits[l]);
    p.mask[l] = l ? (uint32_t*)(tape + L.mask[l]) : nullptr;
    p.bitsT[l] = L.bitsT[l] ? (uint8_t*)(tape + L.bitsT[l]) : nullptr;
    p.maskT[l] = L.maskT[l] ? (uint8_t*)(tape + L.maskT[l]) : nullptr;
  }
  p.counts = (uint8_t*)(tape + L.counts);
  p.act_out = actions;
  p.act_tape = (float*)(tape + L.act);
  const Smem S = smem_layout(p);
  static bool attr = false;
  if (!attr) {
    for (auto k : {actor_fwd_fused_kernel<5>, actor_fwd_fused_kernel<0>}) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      if (e != cudaSuccess) { set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e)); return SPIKERL_E_CUDA; }
    }
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cdiv(B, RB) * C), 1, 1);
  cfg.blockDim = dim3(NTH, 1, 1);
  cfg.dynamicSmemBytes = (size_t)S.total;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  // T = 5 (configs[0..3]) compiled with the time loops unrolled exactly
  cudaError_t e = d.T == 5 ? cudaLaunchKernelEx(&cfg, actor_fwd_fused_kernel<5>, p)
                           : cudaLaunchKernelEx(&cfg, actor_fwd_fused_kernel<0>, p);
  if (e != cudaSuccess) { set_error("cudaLaunchKernelEx (fused actor forward): %s", cudaGetErrorString(e)); return SPIKERL_E_CUDA; }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

}  // namespace spk

extern "C" int spikerl_debug_fused_trace(unsigned long long* host16) {
  if (cudaMemcpyFromSymbol(host16, spk::fused::g_ftrace, sizeof(unsigned long long) * 16) != cudaSuccess) return 5;
  return 0;
}
