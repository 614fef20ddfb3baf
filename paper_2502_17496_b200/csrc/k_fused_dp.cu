// k_fused_dp.cu — SURVEY §8(f) NEXT #1: the data-parallel gradient mean fused with the optimiser
// step, over NCCL 2.28 symmetric memory (PAPER.md:135 average_gradients + PAPER.md:144 DDP; the
// per-step allreduce followed by Adam, as ONE kernel reading and writing peer memory
// over NVLink / NVSwitch).
//
// ZeRO-1 style, per launch, every rank:
//   1. LSA barrier: every rank's gradient is complete;
//   2. for the rank's 1/W shard of the parameters: g = (sum over ranks of their gradient, in rank
//      order, loaded straight from the peers' symmetric buffers; or one multimem.ld_reduce through
//      the NVSwitch when NVLS is on) / W, then Adam on the shard (the same element arithmetic as
//      adam_kernel: adam_elem) and the updated parameter stored into every rank's parameter buffer
//      (peer stores, or one multimem.st);
//   3. LSA barrier: every shard is everywhere; each rank then writes its 16-bit working copies of
//      all parameters and the last block publishes the step count.
// With a peer-load sum the result is bitwise the same on every rank and independent of W's timing;
// at W = 1 it is bitwise adam_kernel's result after a one-rank allreduce (the world-1 GPU test).
// Buffers: gradient and master parameters must come from spikerl_comm_mem_alloc (ncclMemAlloc) and
// be registered once as symmetric windows (spikerl_fused_adam_create, collective); m and v stay
// ordinary replicated buffers (only the shard's slice is read / written).
#include <nccl.h>
#include <nccl_device.h>
#include "internal.h"
#include "comm_internal.h"

struct spikerl_fused_adam {
  spikerl_comm* comm;
  ncclWindow_t gwin, pwin;
  ncclDevComm dev;
  float *g, *p;
  size_t n;
  int blocks, multimem;
};

namespace spk {
namespace {

constexpr int kMaxRanks = 8;   // one NVLink domain of a B200 box

__device__ __forceinline__ float mm_ld_reduce(const float* mp) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(mp) : "memory");
  return r;
}
__device__ __forceinline__ void mm_st(float* mp, float x) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mp), "f"(x) : "memory");
}

__global__ void __launch_bounds__(256) fused_allreduce_adam_kernel(
    ncclDevComm dev, ncclWindow_t gwin, ncclWindow_t pwin, size_t n, float* __restrict__ m, float* __restrict__ v,
    long long* counter, float lr, float b1, float b2, float eps, size_t clo, size_t chi, float cmin,
    unsigned int* ticket, const __grid_constant__ Bf16Views views, int use_mm, double lnb1, double lnb2) {
  pdl_wait();
  pdl_trigger();
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dev, ncclTeamTagLsa(), blockIdx.x);
  // 1. every rank's gradient is complete (release: ours; acquire: the peers')
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  const int W = dev.lsaSize, r = dev.lsaRank;
  __shared__ float s_coef[2];
  __shared__ long long s_t;
  if (threadIdx.x == 0) {
    s_t = *(volatile long long*)counter + 1;
    adam_coefs(lr, lnb1, lnb2, s_t, &s_coef[0], &s_coef[1]);
  }
  __syncthreads();
  const float step_size = s_coef[0], bc2_sqrt = s_coef[1];
  const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
  const float* gq[kMaxRanks];
  float* pq[kMaxRanks];
#pragma unroll
  for (int q = 0; q < kMaxRanks; ++q) {
    gq[q] = q < W ? (const float*)ncclGetLsaPointer(gwin, 0, q) : nullptr;
    pq[q] = q < W ? (float*)ncclGetLsaPointer(pwin, 0, q) : nullptr;
  }
  float* const pmine = (float*)ncclGetLsaPointer(pwin, 0, r);   // (pq[r] with a runtime r would live in local memory)
  const size_t per = (n + W - 1) / W, lo = (size_t)r * per, hi = lo + per < n ? lo + per : n;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // 2. this rank's shard: mean over ranks, Adam, the new value to every rank
  for (size_t e = lo + blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < hi; e += stride) {
    float s;
    if (use_mm) {
      s = mm_ld_reduce((const float*)ncclGetLsaMultimemPointer(gwin, e * sizeof(float), dev));
    } else {
      s = gq[0][e];
#pragma unroll
      for (int q = 1; q < kMaxRanks; ++q)
        if (q < W) s = __fadd_rn(s, gq[q][e]);
    }
    const float g = __fdiv_rn(s, (float)W);
    float mm = m[e], vv = v[e];
    float pp = adam_elem(pmine[e], g, mm, vv, b1, omb1, b2, omb2, bc2_sqrt, eps, step_size);
    if (e >= clo && e < chi) pp = fmaxf(pp, cmin);
    m[e] = mm;
    v[e] = vv;
    if (use_mm) {
      mm_st((float*)ncclGetLsaMultimemPointer(pwin, e * sizeof(float), dev), pp);
    } else {
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q)
        if (q < W) pq[q][e] = pp;
    }
  }
  // 3. every shard is everywhere; the 16-bit working copies of every parameter, the step count
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  if (views.kind != 0)
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += stride) store_views(views, e, pmine[e]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(ticket, 1u);
    if (done == gridDim.x - 1) {
      *counter = s_t;
      *ticket = 0u;
      __threadfence();
    }
  }
}

}  // namespace

int fused_adam_launch(spikerl_fused_adam* fa, float* m, float* v, long long* counter, float lr, float b1, float b2,
                      float eps, size_t clo, size_t chi, float cmin, unsigned int* ticket, const Bf16Views* views,
                      cudaStream_t st) {
  ProfScope ps_("fused_allreduce_adam", PB_HBM, 0.0, 28.0 * fa->n, st);
  Bf16Views none{};
  pdl(fused_allreduce_adam_kernel, fa->blocks, 256, 0, st)(fa->dev, fa->gwin, fa->pwin, fa->n, m, v, counter, lr, b1,
                                                           b2, eps, clo, chi, cmin, ticket, views ? *views : none,
                                                           fa->multimem, log((double)b1), log((double)b2));
  SPK_LAUNCHED();
  return SPIKERL_OK;
}

bool fused_adam_matches(const spikerl_fused_adam* fa, const float* g, const float* p, size_t n) {
  return fa && fa->g == g && fa->p == p && fa->n == n;
}

}  // namespace spk

using namespace spk;

extern "C" {

int spikerl_comm_mem_alloc(spikerl_comm* comm, size_t bytes, void** ptr) {
  if (!comm || !ptr || bytes == 0) { set_error("spikerl_comm_mem_alloc: bad arguments"); return SPIKERL_E_ARG; }
  SPK_TRY(nccl_need_api());
  if (!nccl_api().memAlloc) { set_error("NCCL without ncclMemAlloc (need >= 2.19)"); return SPIKERL_E_NCCL; }
  return nccl_status(nccl_api().memAlloc(ptr, bytes), "ncclMemAlloc");
}

int spikerl_comm_mem_free(spikerl_comm* comm, void* ptr) {
  if (!comm || !ptr) return SPIKERL_OK;
  SPK_TRY(nccl_need_api());
  if (!nccl_api().memFree) { set_error("NCCL without ncclMemFree"); return SPIKERL_E_NCCL; }
  return nccl_status(nccl_api().memFree(ptr), "ncclMemFree");
}

int spikerl_fused_adam_create(spikerl_comm* comm, float* grads, float* params, size_t n, int use_multimem,
                              spikerl_fused_adam** out) {
  if (!comm || !grads || !params || !out || n == 0) {
    set_error("spikerl_fused_adam_create: bad arguments");
    return SPIKERL_E_ARG;
  }
  if (comm_world(comm) > kMaxRanks) {
    set_error("fused allreduce + Adam: at most %d ranks (one NVLink domain)", kMaxRanks);
    return SPIKERL_E_UNSUPPORTED;
  }
  SPK_TRY(nccl_need_api());
  NcclApi& a = nccl_api();
  if (!a.winRegister || !a.devCommCreate) { set_error("NCCL without the device API (need >= 2.28)"); return SPIKERL_E_NCCL; }
  auto* fa = new spikerl_fused_adam{};
  fa->comm = comm;
  fa->g = grads;
  fa->p = params;
  fa->n = n;
  int st = nccl_status(a.winRegister(comm_nccl(comm), grads, n * sizeof(float), &fa->gwin, NCCL_WIN_COLL_SYMMETRIC),
                       "ncclCommWindowRegister(grads)");
  if (st == SPIKERL_OK)
    st = nccl_status(a.winRegister(comm_nccl(comm), params, n * sizeof(float), &fa->pwin, NCCL_WIN_COLL_SYMMETRIC),
                     "ncclCommWindowRegister(params)");
  // one resident wave of 256-thread blocks, one LSA barrier each
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_allreduce_adam_kernel, 256, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  fa->blocks = num_sms() * (per_sm < 4 ? per_sm : 4);
  if (st == SPIKERL_OK) {
    ncclDevCommRequirements req{};
    req.lsaBarrierCount = fa->blocks;
    req.lsaMultimem = use_multimem != 0 && comm_world(comm) > 1;
    st = nccl_status(a.devCommCreate(comm_nccl(comm), &req, &fa->dev), "ncclDevCommCreate");
    fa->multimem = req.lsaMultimem ? 1 : 0;
  }
  if (st != SPIKERL_OK) {
    delete fa;
    return st;
  }
  *out = fa;
  return SPIKERL_OK;
}

int spikerl_fused_adam_destroy(spikerl_fused_adam* fa) {
  if (!fa) return SPIKERL_OK;
  NcclApi& a = nccl_api();
  int st = SPIKERL_OK;
  if (a.devCommDestroy) st = nccl_status(a.devCommDestroy(comm_nccl(fa->comm), &fa->dev), "ncclDevCommDestroy");
  if (a.winDeregister) {
    nccl_status(a.winDeregister(comm_nccl(fa->comm), fa->gwin), "ncclCommWindowDeregister");
    nccl_status(a.winDeregister(comm_nccl(fa->comm), fa->pwin), "ncclCommWindowDeregister");
  }
  delete fa;
  return st;
}

int spikerl_fused_allreduce_adam(spikerl_fused_adam* fa, float* m, float* v, long long* step_counter, float lr,
                                 float beta1, float beta2, float eps, size_t clamp_lo, size_t clamp_hi,
                                 float clamp_min, spikerl_stream_t stream) {
  if (!fa || !m || !v || !step_counter) { set_error("spikerl_fused_allreduce_adam: bad arguments"); return SPIKERL_E_ARG; }
  return fused_adam_launch(fa, m, v, step_counter, lr, beta1, beta2, eps, clamp_lo, clamp_hi, clamp_min,
                           (unsigned int*)(step_counter + 1), nullptr, (cudaStream_t)stream);
}

}  // extern "C"
