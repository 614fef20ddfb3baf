// k_tc_gemm.cu — tcgen05 / TMEM / TMA tensor-core engine for the four contractions of the
// spiking actor, each with its epilogue fused:
//   FWD  I_l = W_l o_{l-1} over all (t,b)  -> LIF forward scan in registers -> spike / mask
//        bit planes (+ output counts)                      north_star
//   DX   g_{l-1} = W_l^T G_l over all (t,b) -> reverse LIF scan of layer l-1 -> G_{l-1} bf16
//        (+ sum_t G_1 for the encoder)                     SPEC.md:168-176; R11
//   ENC  dL/dA = (sum_t G_1) W_1            -> dmu, dsigma partial sums over the tile's rows
//                                                          DESIGN.md R6 (straight-through encoder)
//   DW   dW_l = sum_{t,b} G_l^T o_{l-1}     -> deterministic split-K fp32 partials
// One persistent, warp-specialised kernel (1 CTA/SM, 448 threads; 512 for the long-K pair forward):
//   warp 0      TMA producer (A tiles; B tiles when they are bf16 tensors)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N<=256, K=16 steps)
//   warps 2-5   spike-bit expanders (2-7 for the long-K pair forward): u32 spike words -> bf16 {0,1} tiles
//               in the 128B-swizzled UMMA layout (K-major for FWD, MN-major for DW)
//   next 8      epilogue, 2 groups x 4 warps: tcgen05.ld (32x32b) of the TMEM accumulator, one
//               thread per neuron, each group owning half of the tile's columns (4 groups of 4
//               warps measured no faster: the FWD / DX epilogues are bound by their instruction
//               count, not by latency hiding)
// Pipelines: 4-stage smem ring (full/empty mbarriers), 2-stage TMEM accumulator (2 x 256 cols).
// Neurons sit on TMEM lanes (MMA M) and (t,b) on columns (MMA N) with t-major order, so a
// thread owns every timestep of its neuron: the LIF scans never leave registers, and one
// __ballot_sync per (t,b) yields exactly one u32 word of the next layer's bit plane.
#include <cuda.h>
#include <mutex>
#include <type_traits>
#include "internal.h"

namespace spk {
namespace tc {

// FWD: hidden layers (batch-major spike plane + quad-major spike / mask planes for the DX epilogue);
// FWDO: output layer (batch-major spike and mask planes + spike counts)
// WG: the critic's weight-gradient GEMMs dW = dZ^T X (both operands K-major bf16 by TMA, K = batch),
// split over K, fp32 partial tiles per (job, split)
// CF1 / CF2 / CB1: the twin critic's large-batch contractions (batch on the MMA's M = TMEM lanes,
// the 256 hidden units on its N), A = the batch-contiguous transposed activations (MN-major), B =
// the critic's bf16 weights (K-major, one map per critic: tmB critic 0, tmC critic 1):
//   CF1  Z1 = X W1^T     -> b1, ReLU, bf16: H1T [2][H1][Bp]
//   CF2  Z2 = H1 W2^T    -> b2, ReLU, bf16: H2T [2][H2][Bp], q = h2 . w3 + b3
//   CB1  dH1 = dZ2 W2    -> ReLU mask (h1 > 0), bf16: dZ1T [2][H1][Bp]
enum Mode { FWD = 0, DX = 1, ENC = 2, DW = 3, FWDO = 4, WG = 5, CF1 = 6, CF2 = 7, CB1 = 8 };
__host__ __device__ constexpr bool is_fwd(int m) { return m == FWD || m == FWDO; }
__host__ __device__ constexpr bool is_crit(int m) { return m == CF1 || m == CF2 || m == CB1; }

constexpr int NUM_EPI_WARPS = 8, NUM_EPI_GROUPS = NUM_EPI_WARPS / 4;
constexpr int EXP_WARP0 = 2;
constexpr int BM = 128, BK = 64, STAGES = 4;
// Spike-expander warps per CTA: 4 (at most one warp per ring stage), or 6 in the X6 instantiation of
// the pair forward (6-stage ring), launched for long K loops: ablation r02 (SPIKERL_TC_DBG) put its
// expanders alone at ~80 % of FWD L1's time; A/B with 6: FWD L1 (59 k-blocks per unit) -3.4 %, while
// FWD L2 (16 k-blocks) ran 2.8 % slower. The epilogue warps follow them; DX / ENC / WG / critic modes
// leave the expander warps idle.
__host__ __device__ constexpr int exp_warps(bool x6) { return x6 ? 6 : 4; }
__host__ __device__ constexpr int epi_warp0(bool x6) { return EXP_WARP0 + exp_warps(x6); }
__host__ __device__ constexpr int n_threads(bool x6) { return (epi_warp0(x6) + NUM_EPI_WARPS) * 32; }
constexpr int A_STAGE = BM * BK * 2;             // 16 KB
constexpr int B_STAGE = 256 * BK * 2;            // 32 KB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;   // 48 KB
// batch rows of a (t, b) tile per epilogue group (FWD / DX): a quarter of the tile, at least 4 (one
// quad of the neuron-major planes); groups past BT / epi_hb(BT) idle
__host__ __device__ constexpr int epi_hb(int bt) { return bt / NUM_EPI_GROUPS > 4 ? bt / NUM_EPI_GROUPS : 4; }
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 512;
// DX: each epilogue warp stages its part of G_{l-1} in shared memory, DX_CH steps at a time
// ([t][HB rows][32 neurons] bf16, double-buffered per warp), and its lane 0 stores each chunk with a
// TMA tensor store (rows past B and steps past T are clipped by the tensor map). ncu r01: per-element
// 2-byte global stores with their 64-bit address arithmetic were over half of the DX epilogue's
// instructions.
constexpr int DX_CH = 4;
constexpr int DX_WSTG = 32 * 8 * DX_CH * 2;   // bytes per warp staging buffer (32 neurons x HB <= 8 rows)
constexpr int DX_STG = NUM_EPI_WARPS * DX_WSTG;   // both buffers of all epilogue warps: 2 x DX_STG
constexpr int DW_BN = 256;   // N of one DW MMA
// A DW unit of a CTA pair covers 2 x 256 output columns (two accumulators, sharing every A tile):
// each G_l tile fetched from L2/HBM feeds twice the MMA work, which halves the G_l re-reads over
// the K_{l-1} tiles (ncu r01: dW1 at cfg4 read 6.1 GB from DRAM for a 2.15 GB G_1, and with the
// MMAs disabled its TMA loads alone took 7.3 ms). The epilogue only dumps partial tiles, so the
// accumulator is not double-buffered for these units.
__host__ __device__ constexpr int dw_unit_cols(int cg) { return DW_BN * cg; }

struct Params {
  int T, B, Bt, BN;
  int m_tiles, n_tiles, k_blocks, kps, n_units;   // m_tiles: 128-row tiles per CTA group
  int cg;                                          // 1 = one CTA, 2 = CTA pair (cta_group::2)
  // FWD
  const uint32_t* bits_in; int w_in;
  uint32_t* bits_out; uint32_t* mask_out; int w_out; uint8_t* counts; int n_valid; int n3;
  uint8_t* bitsT_out; uint8_t* maskT_out; int p_out;   // quad-major copies (may be null)
  float* v_out; const float* v_prev;                     // rho = 1: fp32 membrane planes [T][B][P_l]
  LifConst kc; float zh;
  int tpad;                                              // T rounded to 16 (tpad / 2 bytes per (quad, neuron))
  // DX
  const uint8_t* bitsT_prev; const uint8_t* maskT_prev;
  __nv_bfloat16* g_prev; int p_prev; __nv_bfloat16* g_sum;
  // ENC
  const float* A; const float* obs; const float* mu; const float* sigma; float* partial; int K0, S, E;
  // DW
  const uint32_t* bits_dw; int w_dw; float* dw_part; long long split_stride; int ldp; int R; int ldr;
  // WG jobs (critic weight gradients): A / B row bases in the stacked operand maps, partial offset
  // (elements, within one split), row stride and valid columns of the output tile
  int wg_njobs; int wg_arow[8], wg_brow[8], wg_ld[8], wg_ncol[8]; long long wg_off[8];
  // critic modes: per-critic fp32 biases / bf16 w3 (stride cr_ps elements between critics), the
  // transposed bf16 output [2][256][Bp] (critic stride cr_os), CB1's ReLU mask source (H1T), q out,
  // A's K-row offset per critic (H1T / dZ2T hold both critics' rows; XT is shared)
  const float* cr_bias; const __nv_bfloat16* cr_w3; const float* cr_b3; long long cr_ps;
  __nv_bfloat16* cr_out; long long cr_os; int cr_Bp; const __nv_bfloat16* cr_mask; float* cr_q; int cr_aoff;
  int f16;          // 16-bit operands are fp16 (actor FP16 precision), else bf16
  uint32_t one2;    // two 16-bit 1.0 values: 0x3F803F80 (bf16) / 0x3C003C00 (fp16), the expanded spike
  int trace;   // diagnostics: CTA 0 stamps %globaltimer at phase boundaries into g_trace
  int dbg;     // diagnostics only (SPIKERL_TC_DBG, wrong results): 1 = expanders skip their smem
               // stores, 2 = epilogue skips its work, 4 = MMA issuer skips the MMAs, 8 = DW
               // expanders skip their global loads, 16 = TMA producer skips its loads (and the
               // expect_tx, so the stage completes on the expanders' arrivals alone); 32 (results
               // unchanged, A/B) = no weight loads before the PDL wait
};

// Phase timeline of one launch (SPIKERL_TC_TRACE=<n>: the n-th tc launch of the process), read by
// tools/tc_trace.py through spikerl_debug_tc_trace (not part of the public header).
__device__ unsigned long long g_trace[16];
__device__ __forceinline__ void trace_stamp(const Params& p, int i) {
  if (p.trace && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[i] = t;
  }
}

// ------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tma_2d(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// named barrier of the epilogue warps only (barrier 0 is __syncthreads)
__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32) : "memory"); }
__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// UMMA shared-memory descriptor, 128B swizzle (sm_100 "version 1" descriptor).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// instruction descriptor: bf16 x bf16 -> f32, M = 128 (one CTA) or 256 (CTA pair)
__host__ __device__ constexpr uint32_t make_idesc(int N, int a_mn, int b_mn, int M = BM, int f16 = 0) {
  // A / B formats (bits 7-9, 10-12): 1 = bf16, 0 = fp16; accumulator fp32 (bit 4)
  return (1u << 4) | ((f16 ? 0u : 1u) << 7) | ((f16 ? 0u : 1u) << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
template <int N> __device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t (&r)[N]);
template <> __device__ __forceinline__ void tmem_ldn<4>(uint32_t taddr, uint32_t (&r)[4]) { tmem_ld4(taddr, r); }
template <> __device__ __forceinline__ void tmem_ldn<8>(uint32_t taddr, uint32_t (&r)[8]) { tmem_ld8(taddr, r); }
template <> __device__ __forceinline__ void tmem_ldn<16>(uint32_t taddr, uint32_t (&r)[16]) {
  tmem_ld8(taddr, *reinterpret_cast<uint32_t(*)[8]>(&r[0]));
  tmem_ld8(taddr + 8, *reinterpret_cast<uint32_t(*)[8]>(&r[8]));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 8 spike bits -> 8 bf16 values {0, 1.0} (16 bytes). A multiply moves bit i of each nibble to
// the sign bit of byte i (the partial products never overlap, so no carries); prmt with the
// sign-replicate selector bit turns byte pairs into 0x0000 / 0xFFFF halves, masked to 0x3F80 =
// bf16 1.0: 12 instructions per 16 bytes instead of ~20 shift/select pairs (ncu r01: the DW
// expanders were issue-latency bound).
__device__ __forceinline__ uint32_t prmt_sx(uint32_t x, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "r"(sel));
  return r;
}
__device__ __forceinline__ uint4 expand_byte(uint32_t byte, uint32_t one2) {
  const uint32_t zlo = (byte & 0x0Fu) * 0x10204080u;   // bit i     -> bit 8 i + 7
  const uint32_t zhi = (byte & 0xF0u) * 0x01020408u;   // bit 4 + i -> bit 8 i + 7
  uint4 r;
  r.x = prmt_sx(zlo, 0x9988u) & one2;
  r.y = prmt_sx(zlo, 0xBBAAu) & one2;
  r.z = prmt_sx(zhi, 0x9988u) & one2;
  r.w = prmt_sx(zhi, 0xBBAAu) & one2;
  return r;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}


// ---- CTA-pair (cta_group::2) helpers: M = 256 per pair, A split by rows, B split by columns
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same shared-memory offset in CTA rank 0 of the pair. Default
// (.release.cta) semantics: the data this arrival publishes is either shared memory already made
// visible to the async proxy by fence.proxy.async (expanders) or TMEM reads ordered by
// tcgen05.fence::before_thread_sync (epilogue), both consumed by tcgen05 ops the leader issues.
// A .release.cluster arrive costs a MEMBAR.ALL.GPU per arrival (ncu: 1.6x slower FWD).
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;   // shared::cluster address of the pair leader
__device__ __forceinline__ void tma_2d_cg2(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d_cg2(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma_bf16_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// commit to the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

struct Tile { int m, n, kb0, kb1, split; };

// unit u -> this CTA's tile; p.m_tiles counts 128-row tiles per CTA group (pairs when CG = 2)
template <int MODE>
__device__ __forceinline__ Tile decode(const Params& p, int u, int rank, int CG) {
  Tile t;
  t.m = (u % p.m_tiles) * CG + rank;
  int rest = u / p.m_tiles;
  if (MODE == DW || MODE == WG) {
    t.n = rest % p.n_tiles;
    t.split = rest / p.n_tiles;
    t.kb0 = t.split * p.kps;
    t.kb1 = min(p.k_blocks, t.kb0 + p.kps);
  } else {
    t.n = rest;
    t.split = 0;
    t.kb0 = 0;
    t.kb1 = p.k_blocks;
  }
  return t;
}

// ------------------------------------------------------------------------- the kernel

// CG = 1: one CTA computes a 128-row tile. CG = 2: a CTA pair (cluster of 2) computes a 256-row
// tile with tcgen05.mma.cta_group::2 issued by rank 0: each CTA holds its 128 rows of A and half
// of the B columns, every TMA / expander / epilogue completion signals rank 0's barriers, and the
// MMA commits multicast back to both CTAs.
// RHO: the reset-gate-gradient variant (R11, rho = 1): FWD / FWDO write the fp32 membrane
// planes, DX reads the previous layer's; a separate instantiation, so the default path carries no
// extra registers for it
template <int MODE, int BT, int CG, bool F16 = false, bool RHO = false, bool X6 = false>
__global__ void __launch_bounds__(n_threads(X6), 1)
    tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const Params p) {
  // A CTA of a pair holds at most 128 B rows (its half of the MMA's N), so its stages are 32 KB
  // and the same shared memory holds 6 of them instead of 4 (ncu r01: the DW/FWD L1 MMA waited
  // on TMA-filled stages with the ring 4 deep)
  constexpr bool DW2 = (MODE == DW && CG == 2);   // two accumulators per unit, one buffer
  constexpr int SB_ = A_STAGE + (DW2 ? B_STAGE : B_STAGE / CG);
  constexpr int STG_ = MODE == DX ? 2 * DX_STG : 0;   // DX output staging
  constexpr int NST = ((CG == 2 && !DW2) ? 6 : STAGES) - (STG_ + SB_ - 1) / SB_;
  constexpr int NBUF = DW2 ? 1 : 2;               // TMEM accumulator buffers
  static_assert(NST * SB_ + STG_ <= STAGES * STAGE_BYTES, "stage ring exceeds the shared-memory budget");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* stg = smem + NST * SB_;   // DX staging (1024-aligned: SB_ is a multiple of 16 KB)
  uint64_t* full = (uint64_t*)(smem + NST * SB_ + STG_);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  constexpr bool B_EXPAND = (is_fwd(MODE) || MODE == DW);
  constexpr bool A_MN = !is_fwd(MODE) && MODE != WG;
  constexpr bool B_MN = (MODE == DW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int EPI_WARP0 = epi_warp0(X6);
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;   // pair (or CTA) index and count
  if (threadIdx.x == 0) trace_stamp(p, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1 + (B_EXPAND ? CG : 0));   // TMA + one expander warp per CTA
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG * NUM_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CG == 2) tmem_alloc_cg2(tmem_slot, TMEM_COLS);
    else tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();   // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMA loads of one ring stage. what & 1: the stage's expect_tx and its weight operand (A = W for
  // the actor modes, B = the critic's weights for the critic modes); what & 2: the other operand
  const uint32_t bytes_b = (MODE == DX) ? 128u * p.T * p.Bt / CG
                           : ((MODE == ENC || MODE == WG || is_crit(MODE)) ? 128u * p.BN / CG : 0u);
  auto load_stage = [&](const Tile& t, int kb, int stage, int what) {
    uint8_t* sA = smem + stage * SB_;
    uint8_t* sB = sA + A_STAGE;
    uint64_t* bar = &full[stage];
    if (CG == 1) {
      // critic modes: unit column t.n = critic z * (256 / BN) + hidden block; A's K rows of
      // critic z start at z * cr_aoff (H1T / dZ2T stack both critics)
      const int cz = is_crit(MODE) ? t.n / (256 / p.BN) : 0, ch = is_crit(MODE) ? t.n % (256 / p.BN) : 0;
      const int ka = kb * BK + (is_crit(MODE) ? cz * p.cr_aoff : 0);
      auto ld_a = [&]() {
        if (!A_MN) {
          tma_2d(&tmA, sA, bar, kb * BK, t.m * BM);
        } else {
          tma_2d(&tmA, sA, bar, t.m * BM, ka);
          tma_2d(&tmA, sA + 8192, bar, t.m * BM + 64, ka);
        }
      };
      auto ld_b = [&]() {
        if (is_crit(MODE)) tma_2d(cz == 0 ? &tmB : &tmC, sB, bar, kb * BK, ch * p.BN);
        if (MODE == DX) tma_3d(&tmB, sB, bar, kb * BK, t.n * p.Bt, 0);
        if (MODE == ENC) tma_2d(&tmB, sB, bar, kb * BK, t.n * p.BN);
      };
      if (what & 1) {
        mbar_expect_tx(bar, (uint32_t)A_STAGE + bytes_b);
        if (is_crit(MODE)) ld_b(); else ld_a();
      }
      if (what & 2) {
        if (is_crit(MODE)) ld_a(); else ld_b();
      }
    } else if (MODE == WG) {
      if (rank == 0) mbar_expect_tx(bar, 2u * ((uint32_t)A_STAGE + bytes_b));
      tma_2d_cg2(&tmA, sA, bar, kb * BK, p.wg_arow[t.n] + rank * BM);
      tma_2d_cg2(&tmB, sB, bar, kb * BK, p.wg_brow[t.n] + rank * (p.BN / 2));
    } else {
      if (what & 1) {
        if (rank == 0) mbar_expect_tx(bar, 2u * ((uint32_t)A_STAGE + bytes_b));
        if (!A_MN) {
          tma_2d_cg2(&tmA, sA, bar, kb * BK, t.m * BM);
        } else {
          tma_2d_cg2(&tmA, sA, bar, t.m * BM, kb * BK);
          tma_2d_cg2(&tmA, sA + 8192, bar, t.m * BM + 64, kb * BK);
        }
      }
      if (what & 2) {
        if (MODE == DX) tma_3d_cg2(&tmB, sB, bar, kb * BK, t.n * p.Bt, rank * (p.T / 2));
        if (MODE == ENC) tma_2d_cg2(&tmB, sB, bar, kb * BK, t.n * p.BN + rank * (p.BN / 2));
      }
    }
  };
  // The weight operand of the first ring pass is requested BEFORE the PDL wait, so its latency
  // overlaps the previous kernel's tail: the weights are never written by the kernel this one
  // follows in the library's sequences (an actor tcgen05 launch follows the encoder or another
  // forward / backward kernel, a critic one the Xᵀ / dZ2 kernels or another critic mode; only the
  // optimiser and the parameter refresh write weights, and none of them directly precedes a
  // tcgen05 launch). Everything the previous kernel produces is read after the wait.
  constexpr bool PRE_W = is_fwd(MODE) || MODE == DX || MODE == ENC || is_crit(MODE);
  int npre = 0;
  if (PRE_W && warp == 0 && lane == 0 && !(p.dbg & 16) && !(p.dbg & 32) && cid < p.n_units) {
    const Tile t = decode<MODE>(p, cid, rank, CG);
    npre = t.kb1 - t.kb0 < NST ? t.kb1 - t.kb0 : NST;
    for (int j2 = 0; j2 < npre; ++j2) load_stage(t, t.kb0 + j2, j2, 1);   // ring stages start empty
  }
  // the prologue above overlaps the previous kernel (PDL); everything else it may have written only
  // after this point
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) trace_stamp(p, 1);

  if (warp == 0) {
    // ===================== TMA producer (both CTAs load their own halves) =====================
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = cid; u < p.n_units; u += ncl) {
        const Tile t = decode<MODE>(p, u, rank, CG);
        for (int kb = t.kb0; kb < t.kb1; ++kb, ++it) {
          const int stage = it % NST;
          if ((int)it < npre) {   // weights already requested: the other operand only
            load_stage(t, kb, stage, 2);
            continue;
          }
          const uint32_t ph = (it / NST) & 1;
          mbar_wait(&empty[stage], ph ^ 1);
          if (p.dbg & 16) {
            if (CG == 1 || rank == 0) mbar_arrive(&full[stage]);
          } else {
            load_stage(t, kb, stage, 3);
            if (CG == 1 && it == 0) trace_stamp(p, 2);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (rank 0 of a pair) =====================
    if (lane == 0 && rank == 0) {
      uint32_t it = 0, titer = 0;
      const uint32_t idesc = make_idesc(p.BN, A_MN ? 1 : 0, B_MN ? 1 : 0, BM * CG, F16 ? 1 : 0);
      for (int u = cid; u < p.n_units; u += ncl, ++titer) {
        const Tile t = decode<MODE>(p, u, rank, CG);
        const uint32_t a = titer % NBUF, aph = (titer / NBUF) & 1;
        mbar_wait(&tempty[a], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + a * 256;
        // DW2: the second accumulator's columns may lie wholly past the padded K_{l-1} width
        const bool second = DW2 && t.n * dw_unit_cols(CG) + DW_BN < p.ldp;
        for (int kb = t.kb0; kb < t.kb1; ++kb, ++it) {
          const int stage = it % NST;
          const uint32_t ph = (it / NST) & 1;
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          if (it == 0) trace_stamp(p, 3);
          const uint32_t sA = smem_u32(smem + stage * SB_);
          const uint32_t sB = sA + A_STAGE;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? make_desc(sA + kk * 2048, 8192, 1024) : make_desc(sA + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(sB + kk * 2048, 8192, 1024) : make_desc(sB + kk * 32, 16, 1024);
            if (p.dbg & 4) continue;
            if (CG == 2) mma_bf16_cg2(d_tmem, ad, bd, idesc, (kb > t.kb0 || kk > 0) ? 1u : 0u);
            else mma_bf16(d_tmem, ad, bd, idesc, (kb > t.kb0 || kk > 0) ? 1u : 0u);
            if (DW2 && second)
              mma_bf16_cg2(d_tmem + DW_BN, ad, make_desc(sB + 16384 + kk * 2048, 8192, 1024), idesc,
                           (kb > t.kb0 || kk > 0) ? 1u : 0u);
          }
          if (CG == 2) mma_commit_pair(&empty[stage]);
          else mma_commit(&empty[stage]);
        }
        if (CG == 2) mma_commit_pair(&tfull[a]);
        else mma_commit(&tfull[a]);
        if (titer == 0) trace_stamp(p, 4);
      }
    }
  } else if (warp < EPI_WARP0) {
    // ===================== spike-bit expanders =====================
    // Expander warp w fills every stage of ring iterations it = w, w + 4, w + 8, ... on its own:
    // each stage is written, fenced (generic -> async proxy) and published by one warp, so the
    // four warps keep four stages in flight and the fence latency of one overlaps the stores of
    // the others (ncu r01: with all four warps splitting each stage, the stage-serial
    // store -> fence -> arrive chain paced DW/FWD L1 at ~1600 clk per k-block, with the MMAs
    // disabled). The spike words of the warp's next k-block are loaded one iteration ahead into
    // the other half of a statically indexed double buffer.
    // at most one expander warp per ring stage: a warp waits on its stage's empty barrier by phase
    // parity, so two warps must never own items of the same stage at once
    constexpr int NEXP = exp_warps(X6) < NST ? exp_warps(X6) : NST;
    if (B_EXPAND && warp - EXP_WARP0 < NEXP) {
      const int ew = warp - EXP_WARP0;
      uint32_t it = 0;   // ring iterations of all units so far (every warp counts all of them)
      for (int u = cid; u < p.n_units; u += ncl) {
        const Tile t = decode<MODE>(p, u, rank, CG);
        const int nkb = t.kb1 - t.kb0;
        if (is_fwd(MODE)) {
          // K-major: row = (t, j) spike row of the MMA's B columns this CTA holds; one k-block =
          // 2 words per row = 8 chunks of 16 B. Lane l owns rows l + 32 i.
          constexpr int RPL = CG == 2 ? 4 : 8;
          const int rows = p.T * p.Bt / CG;
          const uint32_t* rp[RPL];
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int row = lane + 32 * i;
            const int rg = rank * rows + row;
            const int tt = rg / p.Bt, j = rg - tt * p.Bt;
            const int b = t.n * p.Bt + j;
            rp[i] = (row < rows && b < p.B) ? p.bits_in + ((size_t)tt * p.B + b) * p.w_in : nullptr;
          }
          uint2 q[2][RPL];
          auto ld = [&](uint2 (&dst)[RPL], int kb) {
#pragma unroll
            for (int i = 0; i < RPL; ++i)
              dst[i] = (rp[i] && kb < t.kb1) ? __ldg(reinterpret_cast<const uint2*>(rp[i] + 2 * kb)) : make_uint2(0u, 0u);
          };
          auto body = [&](const uint2 (&cur)[RPL], uint32_t itx) {
            const int stage = itx % NST;
            const uint32_t ph = (itx / NST) & 1;
            mbar_wait(&empty[stage], ph ^ 1);
            const uint32_t sB = smem_u32(smem + stage * SB_ + A_STAGE);
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              const int row = lane + 32 * i;
              if (row < rows) {
                const uint32_t base = sB + row * 128;
                const uint32_t sw = row & 7;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                  const uint32_t w = c < 4 ? cur[i].x : cur[i].y;
                  if (!(p.dbg & 1)) st_shared_v4(base + ((c ^ sw) << 4), expand_byte((w >> (8 * (c & 3))) & 0xFFu, p.one2));
                }
              }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              if (CG == 2) mbar_arrive_leader(&full[stage]);
              else mbar_arrive(&full[stage]);
            }
          };
          // this warp's k-blocks of the unit: local index j = ew, ew + 4, ... (global it + j)
          const int j0 = (int)((ew - it % NEXP + NEXP) % NEXP);
          if (j0 < nkb) ld(q[0], t.kb0 + j0);
          for (int j = j0; j < nkb; j += 2 * NEXP) {
            if (j + NEXP < nkb) ld(q[1], t.kb0 + j + NEXP);
            body(q[0], it + j);
            if (j + NEXP >= nkb) break;
            if (j + 2 * NEXP < nkb) ld(q[0], t.kb0 + j + 2 * NEXP);
            body(q[1], it + j + NEXP);
          }
        } else {
          // MN-major: K row r = one (t,b) row; every CTA expands 256 columns = 8 words = 4 atoms of
          // 64 per k-block: all 256 columns of its MMA (one CTA), or (pair) its 128-column half of
          // each of the unit's two MMAs (atoms 0-1: MMA 0, atoms 2-3: MMA 1). Lane l owns K rows
          // l and l + 32, both halves h (4 words each).
          int wcol[2];
          bool cv[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            wcol[h] = CG == 2 ? t.n * (dw_unit_cols(CG) / 32) + 8 * h + rank * 4 : t.n * (DW_BN / 32) + 4 * h;
            cv[h] = wcol[h] < p.w_dw;
          }
          uint4 q[2][2][2];   // [buffer][row half][h]
          auto ld = [&](uint4 (&dst)[2][2], int kb) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int rg = kb * BK + lane + 32 * i;
              const bool okr = kb < t.kb1 && rg < p.R && !(p.dbg & 8);
#pragma unroll
              for (int h = 0; h < 2; ++h)
                dst[i][h] = (okr && cv[h]) ? __ldg(reinterpret_cast<const uint4*>(p.bits_dw + (size_t)rg * p.w_dw + wcol[h]))
                                           : make_uint4(0u, 0u, 0u, 0u);
            }
          };
          auto body = [&](const uint4 (&cur)[2][2], uint32_t itx) {
            const int stage = itx % NST;
            const uint32_t ph = (itx / NST) & 1;
            mbar_wait(&empty[stage], ph ^ 1);
            const uint32_t sB = smem_u32(smem + stage * SB_ + A_STAGE);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int r = lane + 32 * i;
              const uint32_t sw = r & 7;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint32_t wv[4] = {cur[i][h].x, cur[i][h].y, cur[i][h].z, cur[i][h].w};
#pragma unroll
                for (int wi = 0; wi < 4; ++wi) {
                  const int atom = 2 * h + (wi >> 1), hw = wi & 1;
                  const uint32_t base = sB + atom * 8192 + r * 128;
#pragma unroll
                  for (int c = 0; c < 4; ++c) {
                    const int chunk = hw * 4 + c;
                    if (!(p.dbg & 1)) st_shared_v4(base + ((chunk ^ sw) << 4), expand_byte((wv[wi] >> (8 * c)) & 0xFFu, p.one2));
                  }
                }
              }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              if (CG == 2) mbar_arrive_leader(&full[stage]);
              else mbar_arrive(&full[stage]);
            }
          };
          const int j0 = (int)((ew - it % NEXP + NEXP) % NEXP);
          if (j0 < nkb) ld(q[0], t.kb0 + j0);
          for (int j = j0; j < nkb; j += 2 * NEXP) {
            if (j + NEXP < nkb) ld(q[1], t.kb0 + j + NEXP);
            body(q[0], it + j);
            if (j + NEXP >= nkb) break;
            if (j + 2 * NEXP < nkb) ld(q[0], t.kb0 + j + 2 * NEXP);
            body(q[1], it + j + NEXP);
          }
        }
        it += nkb;
      }
    }
  } else {
    // ===================== epilogue (2 groups x 4 warps) =====================
    // group g handles half of the tile's columns; warp%4 selects the TMEM lane quarter.
    const int q = warp & 3;
    const int g = (warp - EPI_WARP0) >> 2;
    uint32_t titer = 0;
    uint32_t dx_chunk = 0;   // DX staging chunks issued so far (buffer parity)
    (void)dx_chunk;
    constexpr int DX_NQ = MODE == DX ? epi_hb(BT) / 4 : 1;
    unsigned long long nq_o[DX_NQ], nq_h[DX_NQ];
    auto dx_quad_load = [&](const Tile& tn, unsigned long long (&o)[DX_NQ], unsigned long long (&h)[DX_NQ]) {
      const int b0 = tn.n * BT + g * epi_hb(BT);
      const int rw = tn.m * BM + 32 * q + lane;
      const size_t rb = (p.tpad >> 1) / 8;   // u64 words per (quad, neuron) row
      const int ch = (p.T - 1) >> 4;
#pragma unroll
      for (int qi = 0; qi < DX_NQ; ++qi) {
        const size_t w = ((size_t)((b0 >> 2) + qi) * p.p_prev + rw) * rb + ch;
        o[qi] = __ldg(reinterpret_cast<const unsigned long long*>(p.bitsT_prev) + w);
        h[qi] = __ldg(reinterpret_cast<const unsigned long long*>(p.maskT_prev) + w);
      }
    };
    if constexpr (MODE == DX) {
      if (cid < p.n_units) dx_quad_load(decode<MODE>(p, cid, rank, CG), nq_o, nq_h);
    }
    for (int u = cid; u < p.n_units; u += ncl, ++titer) {
      const Tile t = decode<MODE>(p, u, rank, CG);
      const uint32_t a = titer % NBUF, aph = (titer / NBUF) & 1;
      const int row = t.m * BM + 32 * q + lane;  // neuron index (M)
      // DX: this thread's spike / mask bits of the last 16-step chunk (quad-major planes
      // [B/4][P][Tpad/2]) were requested during the previous unit; the next unit's are requested now,
      // so the load latency hides behind a whole unit (ncu r01: loaded at the unit start, they stalled
      // the epilogue on long-scoreboard once per unit)
      unsigned long long dq_o[DX_NQ], dq_h[DX_NQ];
      if constexpr (MODE == DX) {
#pragma unroll
        for (int qi = 0; qi < DX_NQ; ++qi) { dq_o[qi] = nq_o[qi]; dq_h[qi] = nq_h[qi]; }
        if (u + ncl < p.n_units) dx_quad_load(decode<MODE>(p, u + ncl, rank, CG), nq_o, nq_h);
      }
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      if (titer == 0 && warp == EPI_WARP0 && lane == 0) trace_stamp(p, 6);
      const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + a * 256;
      if (p.dbg & 2) {
      } else if constexpr (is_fwd(MODE)) {
        // LIF forward scan of HB batch rows of one neuron, all T steps in registers. Padding
        // neurons (zero weight rows) and padding batch rows (zero spikes) see I = 0 and never fire
        // or enter the window (v = 0 sits on its lower edge), so no validity masking is needed.
        // The reset gate is kept as a factor rv = d_v (1 - o_{t-1}): v = fma(rv, v, c) is exactly
        // c after a spike (ncu r01: the bit-tracked select form cost ~27 instructions per
        // neuron-step with the batch-major mask plane; the hidden layers' mask plane is not written
        // any more, the DX epilogue reads the quad-major copy)
        constexpr int HB = epi_hb(BT);            // batch rows of this group
        constexpr bool OUT = MODE == FWDO;
        if (g < BT / HB) {
          const int jb = g * HB;
          const int b0 = t.n * BT + jb;
          const float dc = p.kc.dc, dv = p.kc.dv, vth = p.kc.vth, win = p.kc.win;
          float c[HB], v[HB], rv[HB];
          int cnt[HB];
#pragma unroll
          for (int j = 0; j < HB; ++j) { c[j] = 0.f; v[j] = 0.f; rv[j] = dv; cnt[j] = 0; }
          // lanes < HB store the step's words of rows b0 + lane: one pointer each, + B W per step
          const bool st_lane = lane < HB && b0 + lane < p.B;
          const size_t wofs = (size_t)(b0 + (lane < HB ? lane : 0)) * p.w_out + ((size_t)(t.m * BM + 32 * q) >> 5);
          const size_t tstride = (size_t)p.B * p.w_out;
          // quad-major copy (DX epilogue input): per batch quad, the nibble of step t enters a
          // 64-bit word (16 steps) written once per 16 steps
          constexpr int NQ = HB / 4;
          unsigned long long qo[NQ], qh[NQ];
#pragma unroll
          for (int qi = 0; qi < NQ; ++qi) { qo[qi] = 0ull; qh[qi] = 0ull; }
          // TMEM loads of CH timesteps are issued together and waited once
          constexpr int CH = HB >= 16 ? 1 : (HB >= 8 ? 4 : 8);
          for (int t0 = 0; t0 < p.T; t0 += CH) {
            uint32_t rr[CH][HB];
#pragma unroll
            for (int ci = 0; ci < CH; ++ci)
              if (t0 + ci < p.T) tmem_ldn<HB>(taddr + (t0 + ci) * BT + jb, rr[ci]);
            tmem_ld_wait();
            if (t0 == 0 && titer == 0 && warp == EPI_WARP0 && lane == 0) trace_stamp(p, 10);
#pragma unroll
            for (int ci = 0; ci < CH; ++ci) {
              const int tt = t0 + ci;
              if (tt >= p.T) break;
              uint32_t ocur = 0, hcur = 0, wo = 0, wh = 0;
#pragma unroll
              for (int j = 0; j < HB; ++j) {
                c[j] = __fmaf_rn(dc, c[j], __uint_as_float(rr[ci][j]));
                v[j] = __fmaf_rn(rv[j], v[j], c[j]);
                const bool o = v[j] > vth;
                const bool h = fabsf(__fsub_rn(v[j], vth)) < win;
                rv[j] = o ? 0.0f : dv;
                if constexpr (RHO) {
                  if (b0 + j < p.B) p.v_out[((size_t)tt * p.B + b0 + j) * p.p_out + row] = v[j];
                }
                if (o) ocur |= 1u << j;
                if (h) hcur |= 1u << j;
                const uint32_t ob = __ballot_sync(0xffffffffu, o);
                if (lane == j) wo = ob;
                if constexpr (OUT) {
                  cnt[j] += o ? 1 : 0;
                  const uint32_t hb = __ballot_sync(0xffffffffu, h);
                  if (lane == j) wh = hb;
                }
              }
              if (st_lane) {
                p.bits_out[wofs + (size_t)tt * tstride] = wo;
                if constexpr (OUT) p.mask_out[wofs + (size_t)tt * tstride] = wh;
              }
              if constexpr (!OUT) {
                const int sh = 4 * (tt & 15);
#pragma unroll
                for (int qi = 0; qi < NQ; ++qi) {
                  qo[qi] |= (unsigned long long)((ocur >> (4 * qi)) & 0xFu) << sh;
                  qh[qi] |= (unsigned long long)((hcur >> (4 * qi)) & 0xFu) << sh;
                }
                if ((tt & 15) == 15 || tt == p.T - 1) {
#pragma unroll
                  for (int qi = 0; qi < NQ; ++qi) {
                    const size_t off = ((size_t)((b0 >> 2) + qi) * p.p_out + row) * (p.tpad >> 1) + ((tt >> 4) << 3);
                    *reinterpret_cast<unsigned long long*>(p.bitsT_out + off) = qo[qi];
                    *reinterpret_cast<unsigned long long*>(p.maskT_out + off) = qh[qi];
                    qo[qi] = 0ull;
                    qh[qi] = 0ull;
                  }
                }
              }
            }
          }
          if (titer == 0 && warp == EPI_WARP0 && lane == 0) trace_stamp(p, 11);
          if constexpr (OUT) {
            if (row < p.n3) {
#pragma unroll
              for (int j = 0; j < HB; ++j) {
                const int b = b0 + j;
                if (b < p.B) p.counts[(size_t)b * p.n3 + row] = (uint8_t)cnt[j];
              }
            }
          }
        }
      } else if constexpr (MODE == DX) {
        // reverse LIF scan of layer l-1 for HB batch rows of one neuron. Padding neurons have
        // g = 0 (zero weight columns) and no spike / window bits, so G = 0 there without masking.
        // G_{l-1} leaves through shared memory: DX_CH steps x HB rows x 32 neurons per warp TMA store.
        // The chunk's spike / window bits are gathered once into one 32-bit word each (quad qi's 16
        // bits = 4 steps x 4 rows at bits 16 qi), so every (step, row) test is one LOP3 against a
        // compile-time mask (ncu r02: 17 instructions per element before, 547 per 4-step chunk)
        constexpr int HB = epi_hb(BT);
        constexpr int NQ = HB / 4;
        static_assert(DX_CH == 4 && NQ <= 2, "one 16-bit field of 4 steps x 4 rows per quad");
        const bool act = g < BT / HB;   // idle groups (BT = 4: HB = 4 rows for group 0 only) skip the scan
        const int jb = act ? g * HB : 0;
        const int b0 = t.n * BT + jb;
        const float zh = p.zh, dvc = p.kc.dv, dcc = p.kc.dc;
        float dvn[HB], dcn[HB], gs[HB];
#pragma unroll
        for (int j = 0; j < HB; ++j) { dvn[j] = 0.f; dcn[j] = 0.f; gs[j] = 0.f; }
        const size_t qstride = (size_t)p.p_prev * (p.tpad >> 1) / 8;   // u64 words between quads
        const unsigned long long* bT = reinterpret_cast<const unsigned long long*>(
            p.bitsT_prev + ((size_t)(b0 >> 2) * p.p_prev + row) * (p.tpad >> 1));
        const unsigned long long* mT = reinterpret_cast<const unsigned long long*>(
            p.maskT_prev + ((size_t)(b0 >> 2) * p.p_prev + row) * (p.tpad >> 1));
        int ch = (p.T - 1) >> 4;
        unsigned long long qo[NQ], qh[NQ];
#pragma unroll
        for (int qi = 0; qi < NQ; ++qi) { qo[qi] = dq_o[qi]; qh[qi] = dq_h[qi]; }
        // each warp stages its own 32 neurons x HB rows x DX_CH steps and stores them with its own
        // TMA store (double-buffered per warp): no barrier between the eight epilogue warps (ncu r02:
        // the two named barriers per chunk were 38 % of DX L3's stall samples)
        uint8_t* const wbuf = stg + (warp - EPI_WARP0) * 2 * DX_WSTG;
        const uint32_t wstg = smem_u32(wbuf);
        const uint32_t soff = (uint32_t)lane * 2u;
        if (act) {
          for (int c = (p.T - 1) / DX_CH; c >= 0; --c, ++dx_chunk) {
            const uint32_t buf = dx_chunk & 1u;
            if (lane == 0) bulk_wait_read1();   // this warp's store from this buffer two chunks ago has read it
            __syncwarp();
            const int tb = c * DX_CH;
            uint32_t rr[DX_CH][HB];
#pragma unroll
            for (int ci = 0; ci < DX_CH; ++ci)
              if (tb + ci < p.T) tmem_ldn<HB>(taddr + (tb + ci) * BT + jb, rr[ci]);
            // rho = 1: the chunk's membrane potentials of this neuron (rows past B read as 0)
            float vv[DX_CH][HB];
            if constexpr (RHO) {
#pragma unroll
              for (int ci = 0; ci < DX_CH; ++ci)
#pragma unroll
                for (int j = 0; j < HB; ++j)
                  vv[ci][j] = (tb + ci < p.T && b0 + j < p.B)
                                  ? __ldg(p.v_prev + ((size_t)(tb + ci) * p.B + b0 + j) * p.p_prev + row) : 0.f;
            }
            if ((tb >> 4) != ch) {
              ch = tb >> 4;
#pragma unroll
              for (int qi = 0; qi < NQ; ++qi) { qo[qi] = __ldg(bT + qi * qstride + ch); qh[qi] = __ldg(mT + qi * qstride + ch); }
            }
            const int sh = 4 * (tb & 15);   // 0, 16, 32 or 48: the chunk's aligned 16-bit field
            uint32_t xo = 0, xh = 0;
#pragma unroll
            for (int qi = 0; qi < NQ; ++qi) {
              xo |= ((uint32_t)(qo[qi] >> sh) & 0xFFFFu) << (16 * qi);
              xh |= ((uint32_t)(qh[qi] >> sh) & 0xFFFFu) << (16 * qi);
            }
            tmem_ld_wait();
            const uint32_t sb = wstg + buf * DX_WSTG + soff;
#pragma unroll
            for (int ci = DX_CH - 1; ci >= 0; --ci) {
              if (tb + ci >= p.T) continue;
#pragma unroll
              for (int j = 0; j < HB; ++j) {
                const uint32_t bm = 1u << (16 * (j >> 2) + 4 * ci + (j & 3));
                float gv = __uint_as_float(rr[ci][j]);
                if constexpr (RHO) gv = rho_grad(gv, dvc, vv[ci][j], dvn[j]);   // rho = 1
                // lif_back_step (common.cuh), same operations: delta_v = h z g + d_v (1 - o) delta_v',
                // delta_c = delta_v + d_c delta_c'
                const float hg = (xh & bm) ? __fmul_rn(zh, gv) : 0.0f;
                const float dvt = (xo & bm) ? hg : __fmaf_rn(dvc, dvn[j], hg);
                const float dct = __fmaf_rn(dcc, dcn[j], dvt);
                dvn[j] = dvt;
                dcn[j] = dct;
                gs[j] = __fadd_rn(gs[j], dct);
                st_shared_u16(sb + (uint32_t)((ci * HB + j) * 64), op16_bits(dct, F16));
              }
            }
            fence_proxy_async();   // generic-proxy smem writes -> the TMA store
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&tmC, wbuf + buf * DX_WSTG, t.m * BM + 32 * q, b0, tb);
              bulk_commit();
            }
          }
          if (p.g_sum) {
#pragma unroll
            for (int j = 0; j < HB; ++j) {
              const int b = b0 + j;
              if (b < p.B) p.g_sum[(size_t)b * p.p_prev + row] = __ushort_as_bfloat16(op16_bits(gs[j], F16));
            }
          }
        }
      } else if (MODE == ENC) {
        // dmu_k = (1/sigma^2) sum_b gA A (s - mu); dsigma_k = (1/sigma^3) sum_b gA A (s - mu)^2
        const bool valid = row < p.K0;
        const int rr = valid ? row : 0;
        const float m = p.mu[rr];
        const int i = rr / p.E;
        constexpr int EJ = NUM_EPI_GROUPS == 2 ? 8 : 4;   // BN is a multiple of 16: qc of EJ
        const int qc = p.BN / NUM_EPI_GROUPS;
        const int c0 = g * qc;
        float pm = 0.f, ps = 0.f;
        // A and s for the columns of chunk c + PD - 1 are requested while chunk c is summed (ncu r01:
        // loaded right before use, one HBM latency per 8-column chunk paced this epilogue at ~15 us
        // per unit); the sum stays in increasing b
        constexpr int PD = 3;
        const int nch = qc / EJ;
        float av[PD][EJ], sv[PD][EJ];
        auto ldc = [&](float (&a)[EJ], float (&sx)[EJ], int ch) {
#pragma unroll
          for (int jj = 0; jj < EJ; ++jj) {
            const int b = t.n * p.BN + c0 + ch * EJ + jj;
            const int bb = b < p.B ? b : 0;
            a[jj] = __ldg(p.A + (size_t)bb * p.K0 + rr);
            sx[jj] = __ldg(p.obs + (size_t)bb * p.S + i);
          }
        };
#pragma unroll
        for (int s2 = 0; s2 < PD - 1; ++s2)
          if (s2 < nch) ldc(av[s2], sv[s2], s2);
        for (int ch0 = 0; ch0 < nch; ch0 += PD) {
#pragma unroll
          for (int s2 = 0; s2 < PD; ++s2) {
            const int ch = ch0 + s2;
            if (ch >= nch) break;
            if (ch + PD - 1 < nch) ldc(av[(s2 + PD - 1) % PD], sv[(s2 + PD - 1) % PD], ch + PD - 1);
            uint32_t r[EJ];
            tmem_ldn<EJ>(taddr + c0 + ch * EJ, r);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < EJ; ++jj) {
              const int b = t.n * p.BN + c0 + ch * EJ + jj;
              if (b < p.B) {
                const float dd = __fsub_rn(sv[s2][jj], m);
                const float gad = __fmul_rn(__fmul_rn(__uint_as_float(r[jj]), av[s2][jj]), dd);
                pm = __fadd_rn(pm, gad);
                ps = __fadd_rn(ps, __fmul_rn(gad, dd));
              }
            }
          }
        }
        if (valid) {
          const float sg = p.sigma[row];
          const float sg2 = __fmul_rn(sg, sg), sg3 = __fmul_rn(sg2, sg);
          p.partial[(((size_t)t.n * NUM_EPI_GROUPS + g) * p.K0 + row) * 2 + 0] = __fdiv_rn(pm, sg2);
          p.partial[(((size_t)t.n * NUM_EPI_GROUPS + g) * p.K0 + row) * 2 + 1] = __fdiv_rn(ps, sg3);
        }
      } else if constexpr (is_crit(MODE)) {
        // thread = batch row b (TMEM lane), group g = hidden units [128 g, 128 g + 128); outputs are
        // transposed [z][n][Bp] (lanes = consecutive rows: 64-byte coalesced stores per column)
        const int nh = 256 / p.BN;                  // hidden blocks per critic (CF1 / CB1: 2, CF2: 1)
        const int z = t.n / nh, hb = t.n % nh;
        const int b = t.m * BM + 32 * q + lane;
        const bool bv = b < p.B, bs = b < p.cr_Bp;
        const int gc = p.BN / NUM_EPI_GROUPS;       // accumulator columns of this group
        const int c0 = g * gc, n0 = hb * p.BN + c0;  // TMEM column, hidden unit of the group's first
        const float* bias = p.cr_bias + (size_t)z * p.cr_ps;
        __nv_bfloat16* out = p.cr_out + (size_t)z * p.cr_os + (bs ? b : 0);
        const __nv_bfloat16* msk = MODE == CB1 ? p.cr_mask + (size_t)z * p.cr_os + (bs ? b : 0) : nullptr;
        const __nv_bfloat16* w3 = MODE == CF2 ? p.cr_w3 + (size_t)z * p.cr_ps : nullptr;
        float qacc = 0.f;
        for (int j1 = 0; j1 < gc; j1 += 32) {
          uint32_t rr[4][8];
#pragma unroll
          for (int ci = 0; ci < 4; ++ci) tmem_ld8(taddr + c0 + j1 + 8 * ci, rr[ci]);
          unsigned short mk[32];
          if constexpr (MODE == CB1) {
#pragma unroll
            for (int e = 0; e < 32; ++e) mk[e] = bs ? __bfloat16_as_ushort(msk[(size_t)(n0 + j1 + e) * p.cr_Bp]) : 0;
          }
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int n = n0 + j1 + e;
            const float v = __uint_as_float(rr[e >> 3][e & 7]);
            __nv_bfloat16 o;
            if constexpr (MODE == CB1) {
              // relu'(z1) from the stored h1 = RN_bf16(relu(z1)) > 0 (R31)
              const bool m = (mk[e] & 0x7FFFu) != 0 && !(mk[e] & 0x8000u);
              o = __float2bfloat16_rn(bv && m ? v : 0.f);
            } else {
              const float zz = __fadd_rn(v, __ldg(bias + n));
              const float h = bv ? fmaxf(zz, 0.f) : 0.f;
              o = __float2bfloat16_rn(h);
              if constexpr (MODE == CF2) qacc = __fmaf_rn(__bfloat162float(o), __bfloat162float(w3[n]), qacc);
            }
            if (bs) out[(size_t)n * p.cr_Bp] = o;
          }
        }
        if constexpr (MODE == CF2) {
          // q = (sum over units 0..127 + sum over 128..255) + b3, the halves meeting in shared memory
          __shared__ float qx[BM];
          if (g == 1) qx[32 * q + lane] = qacc;
          epi_bar_sync();
          if (g == 0 && bv) p.cr_q[(size_t)z * p.B + b] = __fadd_rn(__fadd_rn(qacc, qx[32 * q + lane]), p.cr_b3[(size_t)z * p.cr_ps]);
          epi_bar_sync();
        }
      } else if constexpr (MODE == WG) {
        // dump the fp32 tile of this (job, split) column-major (row stride wg_ld = 256: one warp
        // store = 32 consecutive rows of one column = one 128-byte line, as the DW dump): row =
        // output row within the job's 256, group g covers columns [128 g, 128 g + 128); columns past
        // the job's width are not stored
        constexpr int GC = DW_BN / NUM_EPI_GROUPS;
        const int c0 = g * GC, ld = p.wg_ld[t.n], nc = p.wg_ncol[t.n];
        float* dst = p.dw_part + (size_t)t.split * p.split_stride + p.wg_off[t.n] + (size_t)c0 * ld +
                     (rank * BM + 32 * q + lane);
        for (int j1 = 0; j1 < GC; j1 += 32) {
          if (c0 + j1 < nc) {   // nc is a multiple of 32
            uint32_t rr[4][8];
#pragma unroll
            for (int ci = 0; ci < 4; ++ci) tmem_ld8(taddr + c0 + j1 + 8 * ci, rr[ci]);
            tmem_ld_wait();
#pragma unroll
            for (int ci = 0; ci < 4; ++ci)
#pragma unroll
              for (int e = 0; e < 8; ++e) dst[(size_t)(j1 + 8 * ci + e) * ld] = __uint_as_float(rr[ci][e]);
          }
        }
      } else {  // DW: group g writes columns [GC g, GC g + GC) of the unit (GC = 64, or 128 for DW2)
        // The partial tile is stored column-major (part[split][col][row], rows = this layer's
        // neurons contiguous, stride ldr), so one store instruction of the warp (32 consecutive
        // neurons of one column) is one full 128-byte line; the row-major float4 stores it replaces
        // touched 32 lines per instruction and paced the epilogue (~5 us per unit at configs[1]).
        // dw_reduce_kernel transposes back to the master layout.
        constexpr int GC = (DW2 ? 2 * DW_BN : DW_BN) / NUM_EPI_GROUPS;
        const int c0 = g * GC;
        const int col0 = t.n * dw_unit_cols(CG) + c0;
        float* dst = p.dw_part + (size_t)t.split * p.split_stride + (size_t)col0 * p.ldr + row;
        for (int j1 = 0; j1 < GC; j1 += 32) {   // 4 loads in flight per wait
          if (col0 + j1 < p.ldp) {               // ldp is a multiple of 128
            uint32_t rr[4][8];
#pragma unroll
            for (int ci = 0; ci < 4; ++ci) tmem_ld8(taddr + c0 + j1 + 8 * ci, rr[ci]);
            tmem_ld_wait();
#pragma unroll
            for (int ci = 0; ci < 4; ++ci)
#pragma unroll
              for (int e = 0; e < 8; ++e) dst[(size_t)(j1 + 8 * ci + e) * p.ldr] = __uint_as_float(rr[ci][e]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_leader(&tempty[a]);
        else mbar_arrive(&tempty[a]);
      }
      if (titer == 0 && warp == EPI_WARP0 && lane == 0) trace_stamp(p, 7);
    }
    if (MODE == DX && lane == 0) bulk_wait_all();   // this warp's staged stores done before exit
  }
  tc_fence_before();
  if (threadIdx.x == 0) trace_stamp(p, 8);
  __syncthreads();
  if (CG == 2) cluster_sync_all();   // no CTA of the pair releases smem / TMEM the other still uses
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_cg2(tmem, TMEM_COLS);
    else tmem_dealloc(tmem, TMEM_COLS);
    if (lane == 0) trace_stamp(p, 9);
  }
}

// dW[n][k] (master layout) = sum over splits (fixed order) of the column-major partial tiles
// part[split][k][n] (row stride ldr): one element per thread, 32 x 32 tiles through shared memory,
// so both the partial reads (along n) and the dW writes (along k) are coalesced; the split loop
// issues 8 loads before their (in-order) adds. Block (32, 32).
__global__ void __launch_bounds__(1024) dw_reduce_kernel(const float* __restrict__ part, int splits,
                                                         long long split_stride, int ldr, int N, int K,
                                                         float* __restrict__ dW, int accum) {
  __shared__ float tile[32][33];
  pdl_wait();
  pdl_trigger();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int k0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  {
    const int k = k0 + ty, n = n0 + tx;
    if (k < K && n < N) {
      const float* src = part + (size_t)k * ldr + n;
      float s = 0.f;
      int sp = 0;
      for (; sp + 8 <= splits; sp += 8) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = src[(size_t)(sp + j) * split_stride];
#pragma unroll
        for (int j = 0; j < 8; ++j) s = __fadd_rn(s, v[j]);
      }
      for (; sp < splits; ++sp) s = __fadd_rn(s, src[(size_t)sp * split_stride]);
      tile[ty][tx] = s;
    }
  }
  __syncthreads();
  const int n = n0 + ty, k = k0 + tx;
  if (k < K && n < N) {
    const float s = tile[tx][ty];
    float* o = dW + (size_t)n * K + k;
    *o = accum ? __fadd_rn(*o, s) : s;
  }
}

// ------------------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  });
  return fn;
}

// bf16 tensor map, 128B swizzle, dims/strides listed innermost first (strides in bytes, rank-1 of them)
static int make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                    const uint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, bool f16 = false) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return SPIKERL_E_CUDA; }
  cuuint64_t gd[3], gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) { gd[i] = dims[i]; bx[i] = box[i]; }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides[i];
  CUresult r = fn(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                  const_cast<void*>(base), gd, gs, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return SPIKERL_E_CUDA; }
  return SPIKERL_OK;
}

}  // namespace tc

// u32 tensor map without swizzle (bit planes staged by TMA outside the GEMM engine)
int make_u32_map3(CUtensorMap* m, const void* base, const uint64_t* dims, const uint64_t* strides, const uint32_t* box) {
  tc::EncodeTiledFn fn = tc::encode_fn();
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return SPIKERL_E_CUDA; }
  cuuint64_t gd[3] = {dims[0], dims[1], dims[2]}, gs[2] = {strides[0], strides[1]};
  cuuint32_t bx[3] = {box[0], box[1], box[2]}, es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), gd, gs, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled (u32) failed (%d)", (int)r); return SPIKERL_E_CUDA; }
  return SPIKERL_OK;
}

namespace tc {

// Co-resident CTA pairs: every tc_kernel instance uses one CTA per SM (SMEM_BYTES), so one query
// answers for all; cached so the split-K plan and the launch always agree.
static int pair_slots() {
  static int slots[32] = {};
  const int dev = cur_device();
  if (!slots[dev]) {
    if (cudaFuncSetAttribute(tc_kernel<FWD, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) !=
        cudaSuccess)
      cudaGetLastError();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms() / 2 * 2, 1, 1);
    cfg.blockDim = dim3(n_threads(false), 1, 1);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, tc_kernel<FWD, 8, 2>, &cfg) != cudaSuccess || nc <= 0) {
      cudaGetLastError();
      nc = num_sms() / 2;
    }
    slots[dev] = nc;
  }
  return slots[dev];
}

// CTA pairs (cta_group::2) are used when the tile count allows; SPIKERL_TC_PAIR=0 forces single CTAs.
static bool pairs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPIKERL_TC_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// A/B diagnostics: SPIKERL_TC_CG_LEGACY=<bits> restores the earlier pairing rule per mode (pairs
// whenever the tile count allows): 2 DW, 4 ENC
static int cg_legacy() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SPIKERL_TC_CG_LEGACY");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int MODE, int BT, int CG, bool F16, bool RHO = false, bool X6 = false>
static int launch_cg(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const Params& p, cudaStream_t st) {
  SPK_SMEM_ATTR((tc_kernel<MODE, BT, CG, F16, RHO, X6>), SMEM_BYTES);
  if (CG == 1) {
    const int ncta = num_sms();
    const int grid = p.n_units < ncta ? (int)p.n_units : ncta;
    pdl((tc_kernel<MODE, BT, CG, F16, RHO, X6>), grid, n_threads(X6), SMEM_BYTES, st)(ma, mb, mc, p);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(n_threads(X6), 1, 1);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[3];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (const int pr = launch_priority()) {
      at[2].id = cudaLaunchAttributePriority;
      at[2].val.priority = pr;
      cfg.numAttrs = 3;
    }
    // A persistent grid larger than the number of co-resident pairs would run a second wave of
    // whole pairs; size it to what the GPCs can actually hold (not simply 148 / 2).
    const int slots = pair_slots();
    const long long grid = p.n_units < slots ? p.n_units : slots;
    cfg.gridDim = dim3((unsigned)(grid * CG), 1, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, tc_kernel<MODE, BT, CG, F16, RHO, X6>, ma, mb, mc, p);
    if (e != cudaSuccess) { set_error("cudaLaunchKernelEx (pair): %s", cudaGetErrorString(e)); return SPIKERL_E_CUDA; }
  }
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

static int g_launch_no = 0;
static int trace_launch() {   // 1-based index of the launch to trace (0 = off)
  static int v = -1;
  if (v < 0) { const char* e = getenv("SPIKERL_TC_TRACE"); v = e ? atoi(e) : 0; }
  return v;
}

template <int MODE, int BT>
static int launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const Params& p0, cudaStream_t st) {
  Params p = p0;
  p.trace = (trace_launch() > 0 && ++g_launch_no == trace_launch()) ? 1 : 0;
  static const int dbg = [] { const char* e = getenv("SPIKERL_TC_DBG"); return e ? atoi(e) : 0; }();
  p.dbg = dbg;
  // fp16 operands (actor FP16 precision) are a separate instantiation: the G conversions and the
  // MMA instruction descriptor are then compile-time (a runtime switch cost ~2% at configs[4])
  if constexpr (is_crit(MODE)) {   // bf16, single CTAs only
    return launch_cg<MODE, BT, 1, false>(ma, mb, mc, p, st);
  } else if constexpr (is_fwd(MODE) || MODE == DX) {
    if (p.v_out || p.v_prev) {   // rho = 1 (bf16 operands only; checked by the caller)
      return p.cg == 2 ? launch_cg<MODE, BT, 2, false, true>(ma, mb, mc, p, st)
                       : launch_cg<MODE, BT, 1, false, true>(ma, mb, mc, p, st);
    }
    if (p.f16)
      return p.cg == 2 ? launch_cg<MODE, BT, 2, true>(ma, mb, mc, p, st) : launch_cg<MODE, BT, 1, true>(ma, mb, mc, p, st);
    if constexpr (is_fwd(MODE))   // long K loops: 6 expander warps (see exp_warps)
      if (p.cg == 2 && p.k_blocks >= 32) return launch_cg<MODE, BT, 2, false, false, true>(ma, mb, mc, p, st);
    return p.cg == 2 ? launch_cg<MODE, BT, 2, false>(ma, mb, mc, p, st) : launch_cg<MODE, BT, 1, false>(ma, mb, mc, p, st);
  } else {
    if (MODE != WG && p.f16)
      return p.cg == 2 ? launch_cg<MODE, BT, 2, true>(ma, mb, mc, p, st) : launch_cg<MODE, BT, 1, true>(ma, mb, mc, p, st);
    return p.cg == 2 ? launch_cg<MODE, BT, 2, false>(ma, mb, mc, p, st) : launch_cg<MODE, BT, 1, false>(ma, mb, mc, p, st);
  }
}

template <int MODE>
static int launch_bt(int bt, const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, cudaStream_t st,
                     const CUtensorMap* mc = nullptr) {
  const CUtensorMap& c = mc ? *mc : ma;   // store map (DX only)
  if (MODE == ENC || MODE == DW || MODE == WG || is_crit(MODE)) return launch<MODE, 8>(ma, mb, c, p, st);
  switch (bt) {
    case 8: return launch<MODE, 8>(ma, mb, c, p, st);
    case 16: return launch<MODE, 16>(ma, mb, c, p, st);
    case 32:
      if constexpr (is_fwd(MODE)) return launch<MODE, 32>(ma, mb, c, p, st);
      break;
  }
  set_error("unsupported batch tile %d", bt);
  return SPIKERL_E_UNSUPPORTED;
}

// batch rows per N tile: Bt in {8, 16, 32}, T*Bt % 16 == 0, T*Bt <= 256, Bt <= max_bt (register
// budget: each epilogue group keeps Bt/2 rows of LIF state); prefer the largest Bt that still gives
// >= one wave of tiles, else the smallest valid one.
static int choose_bt(int T, int B, int m_tiles, int max_bt) {
  int best = 0, smallest = 0;
  for (int bt = 8; bt <= max_bt; bt *= 2) {
    if ((T * bt) % 16 != 0 || T * bt > 256) continue;
    if (!smallest) smallest = bt;
    const long long tiles = (long long)m_tiles * ((B + bt - 1) / bt);
    if (tiles >= num_sms()) best = bt;
  }
  return best ? best : smallest;
}

constexpr int FWD_MAX_BT = 32, DX_MAX_BT = 16;

}  // namespace tc

using namespace tc;

bool tc_pairs_enabled() { return pairs_enabled(); }

bool tc_supported(const ActorDims& d) {
  if (!d.bf16) return false;
  for (int bt = 8; bt <= DX_MAX_BT; bt *= 2)
    if ((d.T * bt) % 16 == 0 && d.T * bt <= 256) return true;
  return false;
}

int launch_lif_fwd_tc(const ActorDims& d, int l, int B, const uint32_t* bits_in, const __nv_bfloat16* Wb16,
                      uint32_t* bits_out, uint32_t* mask_out, uint8_t* counts, uint8_t* bitsT_out,
                      uint8_t* maskT_out, int row_bytes, float* v_out, cudaStream_t st) {
  ProfScope ps_(l == 1 ? "lif_fwd_tc_L1" : (l == 2 ? "lif_fwd_tc_L2" : "lif_fwd_tc_L3"), PB_TENSOR,
                2.0 * d.T * B * (double)d.N[l] * d.N[l - 1], 0.0, st);
  Params p{};
  p.f16 = d.f16; p.one2 = d.f16 ? 0x3C003C00u : 0x3F803F80u;
  p.T = d.T; p.B = B;
  const int mt = d.P[l] / BM;
  p.Bt = choose_bt(d.T, B, mt, FWD_MAX_BT);
  p.BN = d.T * p.Bt;
  // (single CTAs below K = 1024 were ~1 us faster per launch alone at configs[1], but slower inside
  // the TD3 update DAG, where three forward passes share the GPU: configs[2] 120.0 -> 128.8 us per
  // update, A/B r02; kept paired)
  p.cg = (pairs_enabled() && mt % 2 == 0) ? 2 : 1;
  p.m_tiles = mt / p.cg;
  p.n_tiles = (B + p.Bt - 1) / p.Bt;
  p.k_blocks = d.P[l - 1] / BK;
  p.n_units = p.m_tiles * p.n_tiles;
  p.bits_in = bits_in; p.w_in = d.Wd[l - 1];
  p.bits_out = bits_out; p.mask_out = mask_out; p.w_out = d.Wd[l];
  p.counts = counts; p.n_valid = d.N[l]; p.n3 = d.N[3];
  p.bitsT_out = bitsT_out; p.maskT_out = maskT_out; p.p_out = d.P[l]; p.tpad = row_bytes;
  p.v_out = v_out;
  p.kc = LifConst{d.dc, d.dv, d.vth, d.win}; p.zh = d.zh;
  CUtensorMap ma, mb;
  const uint64_t dims[2] = {(uint64_t)d.P[l - 1], (uint64_t)d.P[l]};
  const uint64_t strides[1] = {(uint64_t)d.P[l - 1] * 2};
  const uint32_t box[2] = {64, 128};
  SPK_TRY(make_map(&ma, Wb16, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, d.f16));
  mb = ma;
  return l == 3 ? launch_bt<FWDO>(p.Bt, ma, mb, p, st) : launch_bt<FWD>(p.Bt, ma, mb, p, st);
}

// dX of layer l fused with the reverse scan of layer l-1 (G_l bf16 [T][B][P_l])
int launch_lif_dx_tc(const ActorDims& d, int l, int B, const void* Gl, const __nv_bfloat16* Wb16,
                     const uint8_t* bitsT_prev, const uint8_t* maskT_prev, int row_bytes,
                     const float* v_prev, void* Gprev, void* Gsum, cudaStream_t st) {
  ProfScope ps_(l == 3 ? "lif_dx_tc_L3" : "lif_dx_tc_L2", PB_TENSOR, 2.0 * d.T * B * (double)d.N[l] * d.N[l - 1],
                0.0, st);
  Params p{};
  p.f16 = d.f16; p.one2 = d.f16 ? 0x3C003C00u : 0x3F803F80u;
  p.T = d.T; p.B = B;
  const int mt = d.P[l - 1] / BM;
  p.Bt = choose_bt(d.T, B, mt, DX_MAX_BT);
  p.BN = d.T * p.Bt;
  p.cg = (pairs_enabled() && mt % 2 == 0 && d.T % 2 == 0) ? 2 : 1;   // B halves split along t
  p.m_tiles = mt / p.cg;
  p.n_tiles = (B + p.Bt - 1) / p.Bt;
  p.k_blocks = d.P[l] / BK;
  p.n_units = p.m_tiles * p.n_tiles;
  p.bitsT_prev = bitsT_prev; p.maskT_prev = maskT_prev; p.tpad = row_bytes;
  p.g_prev = (__nv_bfloat16*)Gprev; p.p_prev = d.P[l - 1]; p.g_sum = (__nv_bfloat16*)Gsum;
  p.v_prev = v_prev;
  p.n_valid = d.N[l - 1];
  p.kc = LifConst{d.dc, d.dv, d.vth, d.win}; p.zh = d.zh;
  CUtensorMap ma, mb;
  {  // A = W_l^T: W_l [P_l][P_{l-1}], M = P_{l-1} (contiguous) -> MN-major boxes of 64 x 64
    const uint64_t dims[2] = {(uint64_t)d.P[l - 1], (uint64_t)d.P[l]};
    const uint64_t strides[1] = {(uint64_t)d.P[l - 1] * 2};
    const uint32_t box[2] = {64, 64};
    SPK_TRY(make_map(&ma, Wb16, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, d.f16));
  }
  {  // B = G_l [T][B][P_l]: rows (t, b) t-major per tile, K = P_l. The map ends at N_3 for G_3:
     // TMA zero-fills columns past it (the output-layer scan does not write G_3's padding)
    const uint64_t dims[3] = {(uint64_t)(l == 3 ? d.N[3] : d.P[l]), (uint64_t)B, (uint64_t)d.T};
    const uint64_t strides[2] = {(uint64_t)d.P[l] * 2, (uint64_t)d.P[l] * 2 * B};
    const uint32_t box[3] = {64, (uint32_t)p.Bt, (uint32_t)(d.T / p.cg)};
    SPK_TRY(make_map(&mb, Gl, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, d.f16));
  }
  CUtensorMap mc;
  {  // C = G_{l-1} [T][B][P_{l-1}]: one epilogue warp's staged chunk of DX_CH steps x HB rows x 32 neurons
    const uint64_t dims[3] = {(uint64_t)d.P[l - 1], (uint64_t)B, (uint64_t)d.T};
    const uint64_t strides[2] = {(uint64_t)d.P[l - 1] * 2, (uint64_t)d.P[l - 1] * 2 * B};
    const uint32_t box[3] = {32, (uint32_t)epi_hb(p.Bt), (uint32_t)DX_CH};
    SPK_TRY(make_map(&mc, Gprev, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE, d.f16));
  }
  return launch_bt<DX>(p.Bt, ma, mb, p, st, &mc);
}

// CTA pairs for ENC only with a long contraction (K = n_1 >= 512): with n_1 = 256 the unit's four
// k-blocks are short against its epilogue and single CTAs were faster at every batch measured
// (configs[1..3]: 19.1 -> 16.6, 26.8 -> 21.3, 20.7 -> 17.9 us; B = 4096 59.2 -> 53.9 us), while at
// configs[4] (n_1 = 1024) the two are within 2 %
static int enc_cg(const ActorDims& d) {
  return (pairs_enabled() && (d.P[0] / BM) % 2 == 0 && (d.P[1] / BK >= 8 || (cg_legacy() & 4))) ? 2 : 1;
}

// batch columns per ENC unit: 256 when that still gives every SM (pair) a unit; smaller batches
// use narrower units (>= 16) so the per-unit epilogue loop over the batch stays short (cfg1:
// one 256-wide unit = 2 CTAs and an 8 us epilogue; 16-wide units = 16 pairs)
static int enc_bn(const ActorDims& d, int B) {
  const int cg = enc_cg(d);
  const int m_tiles = d.P[0] / BM / cg;
  const int slots = cg == 2 ? pair_slots() : num_sms();
  int bn = 256;
  while (bn > 16 && (long long)m_tiles * cdiv(B, bn) < slots) bn /= 2;
  if (B < bn) bn = round_up(B, 16);
  return bn;
}

size_t tc_enc_partial_bytes(const ActorDims& d, int B) {
  return sizeof(float) * 2 * NUM_EPI_GROUPS * (size_t)cdiv(B, enc_bn(d, B)) * d.K0;   // per epilogue group and N tile
}

int launch_enc_grad_tc(const ActorDims& d, int B, const void* Gsum, const __nv_bfloat16* W1b16, const float* A,
                       const float* obs, const float* mu, const float* sigma, float* partial, float* dmu,
                       float* dsigma, int accumulate, cudaStream_t st) {
  ProfScope ps_("enc_grad_tc", PB_TENSOR, 2.0 * B * (double)d.N1 * d.K0, 0.0, st);
  Params p{};
  p.f16 = d.f16; p.one2 = d.f16 ? 0x3C003C00u : 0x3F803F80u;
  p.T = 1; p.B = B;
  p.BN = enc_bn(d, B);
  p.cg = enc_cg(d);
  p.m_tiles = d.P[0] / BM / p.cg;
  p.n_tiles = cdiv(B, p.BN);
  p.k_blocks = d.P[1] / BK;
  p.n_units = p.m_tiles * p.n_tiles;
  p.A = A; p.obs = obs; p.mu = mu; p.sigma = sigma; p.partial = partial; p.K0 = d.K0; p.S = d.S; p.E = d.E;
  CUtensorMap ma, mb;
  {
    const uint64_t dims[2] = {(uint64_t)d.P[0], (uint64_t)d.P[1]};
    const uint64_t strides[1] = {(uint64_t)d.P[0] * 2};
    const uint32_t box[2] = {64, 64};
    SPK_TRY(make_map(&ma, W1b16, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, d.f16));
  }
  {
    const uint64_t dims[2] = {(uint64_t)d.P[1], (uint64_t)B};
    const uint64_t strides[1] = {(uint64_t)d.P[1] * 2};
    const uint32_t box[2] = {64, (uint32_t)(p.BN / p.cg)};
    SPK_TRY(make_map(&mb, Gsum, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, d.f16));
  }
  SPK_TRY(launch_bt<ENC>(8, ma, mb, p, st));
  return launch_enc_grad_reduce(d, NUM_EPI_GROUPS * p.n_tiles, partial, dmu, dsigma, accumulate, st);
}

// split-K plan for dW_l: pick the CTA grouping cg and split count s minimising a simple cost model
// in units of one single-CTA k-block (a 128 x 256 x 64 MMA step per SM): waves x (k-blocks per unit
// x kKb(cg) + dump(cg)) + the fixed-order reduction of the partial tiles spread over the GPU. A pair
// unit covers a 256 x 512 tile: its k-block does twice a single CTA's MMA work per SM for ~1.28x the
// time (configs[4]: DW L1 4.40 ms paired vs 6.88 ms single), and its epilogue dumps twice the
// fp32 partial columns per CTA (~10 k-blocks, not overlapped: single TMEM buffer) against ~5 for a
// single CTA's 128 x 256 tile. Pairs win when the contraction is long (configs[4]); with few
// k-blocks the dumps dominate and single CTAs win (configs[1] DW L2 28.4 -> 19.8 us, configs[2] DW L1
// 38.1 -> 27.0 us, configs[3] B = 4096 DW L3 41.6 -> 26.4 us). (The wave-efficiency-only rule of r01
// chose 320 one-k-block units for dW3 at configs[3] B = 4096: 278 us.)
struct DwPlan { int cg, splits, kps; };

static DwPlan dw_plan(const ActorDims& d, int l, int B) {
  const int k_blocks = cdiv((long long)d.T * B, BK);
  DwPlan best_p{1, 1, k_blocks};
  double best = 1e300;
  for (int cg = 1; cg <= 2; ++cg) {
    if (cg == 2 && !(pairs_enabled() && (d.P[l] / BM) % 2 == 0)) continue;
    // single CTAs only for short contractions (T B < 8192): at configs[3] B = 4096 the model's
    // single-CTA DW L2 / L3 were faster alone but 1.5 us per update slower inside the TD3 DAG (A/B r02)
    if (cg == 1 && (k_blocks >= 128 || (cg_legacy() & 2)) && pairs_enabled() && (d.P[l] / BM) % 2 == 0) continue;
    const int m_tiles = d.P[l] / BM / cg, n_tiles = cdiv(d.P[l - 1], dw_unit_cols(cg));
    const long long mn = (long long)m_tiles * n_tiles;
    const int slots = cg == 2 ? pair_slots() : num_sms();   // concurrent units (CTA pairs when cg = 2)
    const double kKb = cg == 2 ? 1.28 : 1.0, kDump = cg == 2 ? 10.0 : 5.0;
    const int s_max = k_blocks < 8 * slots ? k_blocks : 8 * slots;
    for (int s = 1; s <= s_max; ++s) {
      const int per = cdiv(k_blocks, s), ss = cdiv(k_blocks, per);
      if (ss != s) continue;   // the same partition as a smaller s
      const long long units = mn * ss;
      const double cost = (double)cdiv(units, slots) * (per * kKb + kDump) + (double)units * kDump / slots;
      if (cost < best - 1e-9) { best = cost; best_p = DwPlan{cg, ss, per}; }
    }
  }
  return best_p;
}

void tc_dw_plan(const ActorDims& d, int l, int B, int* splits, int* kps) {
  const DwPlan pl = dw_plan(d, l, B);
  *kps = pl.kps;
  *splits = pl.splits;
}

size_t tc_dw_partial_bytes(const ActorDims& d, int B, int l) {
  int s, k;
  tc_dw_plan(d, l, B, &s, &k);
  return sizeof(float) * (size_t)s * d.P[l] * d.P[l - 1];
}

int launch_lif_dw_tc(const ActorDims& d, int l, int B, const void* Gl, const uint32_t* bits_prev, float* dW,
                     float* part, int accumulate, cudaStream_t st) {
  Params p{};
  p.f16 = d.f16; p.one2 = d.f16 ? 0x3C003C00u : 0x3F803F80u;
  p.T = d.T; p.B = B; p.BN = DW_BN;
  p.R = d.T * B;
  const DwPlan pl = dw_plan(d, l, B);
  p.cg = pl.cg;
  p.m_tiles = d.P[l] / BM / p.cg;
  p.n_tiles = cdiv(d.P[l - 1], dw_unit_cols(p.cg));
  p.k_blocks = cdiv(p.R, BK);
  const int splits = pl.splits;
  p.kps = pl.kps;
  p.n_units = p.m_tiles * p.n_tiles * splits;
  p.bits_dw = bits_prev; p.w_dw = d.Wd[l - 1];
  p.dw_part = part; p.ldp = d.P[l - 1]; p.ldr = d.P[l]; p.split_stride = (long long)d.P[l] * d.P[l - 1];
  CUtensorMap ma, mb;
  {  // A = G_l viewed [T*B][P_l]: M = P_l contiguous (MN-major), K = rows (ends at N_3 for G_3, as above)
    const uint64_t dims[2] = {(uint64_t)(l == 3 ? d.N[3] : d.P[l]), (uint64_t)p.R};
    const uint64_t strides[1] = {(uint64_t)d.P[l] * 2};
    const uint32_t box[2] = {64, 64};
    SPK_TRY(make_map(&ma, Gl, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, d.f16));
  }
  mb = ma;
  {
    ProfScope ps_(l == 1 ? "lif_dw_tc_L1" : (l == 2 ? "lif_dw_tc_L2" : "lif_dw_tc_L3"), PB_TENSOR,
                  2.0 * d.T * B * (double)d.N[l] * d.N[l - 1], 0.0, st);
    SPK_TRY(launch_bt<DW>(8, ma, mb, p, st));
  }
  // the split-K reduction: reads every partial once, writes (accumulate: reads too) dW
  ProfScope pr_(l == 1 ? "dw_reduce_L1" : (l == 2 ? "dw_reduce_L2" : "dw_reduce_L3"), PB_HBM, 0.0,
                4.0 * (double)d.N[l] * d.N[l - 1] * (splits + (accumulate ? 2 : 1)), st);
  pdl(dw_reduce_kernel, dim3(cdiv(d.N[l - 1], 32), cdiv(d.N[l], 32)), dim3(32, 32), 0, st)(
      part, splits, p.split_stride, p.ldr, d.N[l], d.N[l - 1], dW, accumulate);
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

// ---- critic weight gradients on the tcgen05 engine (large batches)
// Operands (mma critic workspace): A = [dZ2T z0 | dZ2T z1 | dZ1T z0 | dZ1T z1] rows of Bp bf16 (one
// stacked 2-D map), B = [XT (xtr rows) | H1T z0 | H1T z1]. Jobs: per critic z, dW2 (A rows z 256,
// B = H1T z) and dW1 in 256-column tiles (A rows 512 + z 256, B = XT rows n 256). Output: fp32
// partials, column-major (row stride 256), in the layout critic_wgrad_reduce_cm_kernel adds up:
// part[(s 2 + z) msz + c 256 + r] (dW2), part[(s 2 + z) msz + 256^2 + c 256 + r] (dW1).
int tc_wgrad_splits(int Bp, int inq) {
  const int jobs = 2 * (1 + cdiv(inq, 256));
  const int kblocks = cdiv(Bp, BK);
  int s = pairs_enabled() ? pair_slots() / jobs : 1;
  if (s < 1) s = 1;
  if (s > kblocks) s = kblocks;
  const int kps = cdiv(kblocks, s);
  return cdiv(kblocks, kps);
}

int launch_critic_wgrad_tc(int Bp, int inq, int xtr, const __nv_bfloat16* dZT, const __nv_bfloat16* XTH,
                           float* part, long long msz, cudaStream_t st) {
  if (!pairs_enabled()) { set_error("critic wgrad tc: needs CTA pairs"); return SPIKERL_E_UNSUPPORTED; }
  constexpr int HWc = 256;
  Params p{};
  p.one2 = 0x3F803F80u;
  p.BN = 256;
  p.cg = 2;
  p.m_tiles = 1;
  p.k_blocks = cdiv(Bp, BK);
  const int splits = tc_wgrad_splits(Bp, inq);
  p.kps = cdiv(p.k_blocks, splits);
  int nj = 0;
  for (int z = 0; z < 2; ++z) {
    p.wg_arow[nj] = z * HWc; p.wg_brow[nj] = xtr + z * HWc; p.wg_ld[nj] = HWc; p.wg_ncol[nj] = HWc;
    p.wg_off[nj] = (long long)z * msz; ++nj;
    for (int n = 0; n * 256 < inq; ++n) {
      p.wg_arow[nj] = 2 * HWc + z * HWc; p.wg_brow[nj] = n * 256; p.wg_ld[nj] = HWc;
      p.wg_ncol[nj] = inq - n * 256 < 256 ? inq - n * 256 : 256;
      p.wg_off[nj] = (long long)z * msz + (long long)HWc * HWc + (long long)n * 256 * HWc; ++nj;
    }
  }
  if (nj > 8) { set_error("critic wgrad tc: input width too large"); return SPIKERL_E_UNSUPPORTED; }
  p.wg_njobs = nj;
  p.n_tiles = nj;
  p.n_units = nj * cdiv(p.k_blocks, p.kps);
  p.dw_part = part;
  p.split_stride = 2 * msz;
  CUtensorMap ma, mb;
  {
    const uint64_t dims[2] = {(uint64_t)Bp, (uint64_t)(4 * HWc)};
    const uint64_t strides[1] = {(uint64_t)Bp * 2};
    const uint32_t box[2] = {64, 128};
    SPK_TRY(make_map(&ma, dZT, 2, dims, strides, box));
  }
  {
    const uint64_t dims[2] = {(uint64_t)Bp, (uint64_t)(xtr + 2 * HWc)};
    const uint64_t strides[1] = {(uint64_t)Bp * 2};
    const uint32_t box[2] = {64, 128};
    SPK_TRY(make_map(&mb, XTH, 2, dims, strides, box));
  }
  ProfScope ps_("critic_wgrad_tc", PB_TENSOR, 2.0 * 2 * Bp * ((double)HWc * HWc + (double)HWc * inq), 0.0, st);
  return launch_bt<WG>(8, ma, mb, p, st);
}

// ---- twin critic contractions at large batches (modes CF1 / CF2 / CB1; see the Mode enum)
// A: bf16 [a_rows][Bp] (batch contiguous; critic z's K rows start at z * aoff); B: critic z's bf16
// weight rows [256][ldb] (K extent bk), Bw0 / Bw1; outputs transposed [z][256][Bp] (stride os).
int launch_critic_tc(int mode, int B, int Bp, int nz, const __nv_bfloat16* A, int a_rows, int aoff,
                     const __nv_bfloat16* Bw0, const __nv_bfloat16* Bw1, int bk, int ldb, const float* bias,
                     const __nv_bfloat16* w3, const float* b3, long long ps, __nv_bfloat16* out, long long os,
                     const __nv_bfloat16* mask, float* q, cudaStream_t st) {
  Params p{};
  p.one2 = 0x3F803F80u;
  p.B = B;
  // CF1 / CB1 units cover half of the hidden units (N = 128: twice the CTAs, each with half the MMA
  // and epilogue work: a launch is one unit deep at B = 4096, so this halves its latency); CF2 keeps
  // N = 256 so its epilogue forms q = h2 . w3 over every hidden unit
  p.BN = mode == CF2 ? 256 : 128;
  p.cg = 1;
  p.m_tiles = cdiv(Bp, BM);
  p.n_tiles = nz * (256 / p.BN);
  p.k_blocks = cdiv(bk, BK);
  p.n_units = p.m_tiles * p.n_tiles;
  p.cr_bias = bias; p.cr_w3 = w3; p.cr_b3 = b3; p.cr_ps = ps;
  p.cr_out = out; p.cr_os = os; p.cr_Bp = Bp; p.cr_mask = mask; p.cr_q = q; p.cr_aoff = aoff;
  CUtensorMap ma, mb, mc;
  {
    const uint64_t dims[2] = {(uint64_t)Bp, (uint64_t)a_rows};
    const uint64_t strides[1] = {(uint64_t)Bp * 2};
    const uint32_t box[2] = {64, 64};
    SPK_TRY(make_map(&ma, A, 2, dims, strides, box));
  }
  {
    const uint64_t dims[2] = {(uint64_t)bk, 256};
    const uint64_t strides[1] = {(uint64_t)ldb * 2};
    const uint32_t box[2] = {64, (uint32_t)p.BN};
    SPK_TRY(make_map(&mb, Bw0, 2, dims, strides, box));
    SPK_TRY(make_map(&mc, Bw1 ? Bw1 : Bw0, 2, dims, strides, box));
  }
  switch (mode) {
    case CF1: return launch_bt<CF1>(8, ma, mb, p, st, &mc);
    case CF2: return launch_bt<CF2>(8, ma, mb, p, st, &mc);
    case CB1: return launch_bt<CB1>(8, ma, mb, p, st, &mc);
  }
  set_error("launch_critic_tc: bad mode %d", mode);
  return SPIKERL_E_ARG;
}

}  // namespace spk

extern "C" int spikerl_debug_tc_trace(unsigned long long* host16) {
  if (cudaMemcpyFromSymbol(host16, spk::tc::g_trace, sizeof(unsigned long long) * 16) != cudaSuccess) return 5;
  return 0;
}
