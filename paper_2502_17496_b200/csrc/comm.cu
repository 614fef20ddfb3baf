// comm.cu — data-parallel communication: C1 gradient allreduce (PAPER.md:135 average_gradients,
// PAPER.md:144 DDP allreduce over NCCL) and C2 parameter broadcast (PAPER.md:135
// broadcast_weights). NCCL 2.28 (the build torch ships) is loaded with dlopen at
// spikerl_comm_init so libspikerl.so itself has no link-time NCCL dependency; the 128-byte
// unique id is exchanged by the caller (torch.distributed rendezvous).
#include <dlfcn.h>
#include <cstring>
#include <mutex>
#include <string>
#include <nccl.h>
#include "internal.h"

#include "comm_internal.h"

struct spikerl_comm {
  ncclComm_t comm;
  int rank, world;
};

namespace spk {

NcclApi& nccl_api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("SPIKERL_NCCL_LIB");
    const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* c : cands) {
      if (!c) continue;
      a.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) {
      a.why = std::string("dlopen(libnccl.so.2) failed: ") + (dlerror() ? dlerror() : "?");
      return;
    }
#define SPK_SYM(field, name) a.field = (decltype(a.field))dlsym(a.h, name)
    SPK_SYM(getUniqueId, "ncclGetUniqueId");
    SPK_SYM(commInitRank, "ncclCommInitRank");
    SPK_SYM(commDestroy, "ncclCommDestroy");
    SPK_SYM(allReduce, "ncclAllReduce");
    SPK_SYM(broadcast, "ncclBroadcast");
    SPK_SYM(errStr, "ncclGetErrorString");
    SPK_SYM(asyncErr, "ncclCommGetAsyncError");
    SPK_SYM(memAlloc, "ncclMemAlloc");
    SPK_SYM(memFree, "ncclMemFree");
    SPK_SYM(winRegister, "ncclCommWindowRegister");
    SPK_SYM(winDeregister, "ncclCommWindowDeregister");
    SPK_SYM(devCommCreate, "ncclDevCommCreate");
    SPK_SYM(devCommDestroy, "ncclDevCommDestroy");
#undef SPK_SYM
    if (!a.getUniqueId || !a.commInitRank || !a.allReduce || !a.broadcast) a.why = "missing NCCL symbols";
  });
  return a;
}

int nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SPIKERL_OK;
  set_error("%s: %s", what, nccl_api().errStr ? nccl_api().errStr(r) : "nccl error");
  return SPIKERL_E_NCCL;
}

int nccl_need_api() {
  NcclApi& a = nccl_api();
  if (!a.why.empty()) {
    set_error("NCCL unavailable: %s", a.why.c_str());
    return SPIKERL_E_NCCL;
  }
  return SPIKERL_OK;
}

ncclComm_t comm_nccl(const spikerl_comm* c) { return c->comm; }
int comm_world(const spikerl_comm* c) { return c->world; }

}  // namespace spk

extern "C" {

int spikerl_comm_get_unique_id(void* out128) {
  if (!out128) { spk::set_error("null id buffer"); return SPIKERL_E_ARG; }
  SPK_TRY(spk::nccl_need_api());
  ncclUniqueId id;
  SPK_TRY(spk::nccl_status(spk::nccl_api().getUniqueId(&id), "ncclGetUniqueId"));
  memcpy(out128, &id, sizeof(id));
  return SPIKERL_OK;
}

int spikerl_comm_init(int rank, int world, const void* id128, spikerl_comm** out) {
  if (!id128 || !out || world < 1 || rank < 0 || rank >= world) {
    spk::set_error("spikerl_comm_init: bad arguments (rank %d, world %d)", rank, world);
    return SPIKERL_E_ARG;
  }
  SPK_TRY(spk::nccl_need_api());
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  SPK_TRY(spk::nccl_status(spk::nccl_api().commInitRank(&c, world, id, rank), "ncclCommInitRank"));
  *out = new spikerl_comm{c, rank, world};
  return SPIKERL_OK;
}

int spikerl_comm_destroy(spikerl_comm* comm) {
  if (!comm) return SPIKERL_OK;
  int st = spk::nccl_status(spk::nccl_api().commDestroy(comm->comm), "ncclCommDestroy");
  delete comm;
  return st;
}

int spikerl_comm_world(const spikerl_comm* comm) { return comm ? comm->world : 1; }
int spikerl_comm_rank(const spikerl_comm* comm) { return comm ? comm->rank : 0; }

int spikerl_allreduce_grads(spikerl_comm* comm, float* grads, size_t count, spikerl_stream_t stream) {
  if (!comm) return SPIKERL_OK;  // one GPU: identity
  if (!grads && count) { spk::set_error("null grads"); return SPIKERL_E_ARG; }
  if (count == 0) return SPIKERL_OK;
  // world 1 included: NCCL runs one-rank communicators (the mean is the identity), so the one-GPU
  // path exercises the same calls, inside graph captures too
  return spk::nccl_status(spk::nccl_api().allReduce(grads, grads, count, ncclFloat32, ncclAvg, comm->comm,
                                               (cudaStream_t)stream),
                          "ncclAllReduce");
}

int spikerl_broadcast_params(spikerl_comm* comm, float* params, size_t count, int root,
                             spikerl_stream_t stream) {
  if (!comm) return SPIKERL_OK;
  if ((!params && count) || root < 0 || root >= comm->world) {
    spk::set_error("spikerl_broadcast_params: bad arguments");
    return SPIKERL_E_ARG;
  }
  if (count == 0) return SPIKERL_OK;
  return spk::nccl_status(spk::nccl_api().broadcast(params, params, count, ncclFloat32, root, comm->comm,
                                               (cudaStream_t)stream),
                          "ncclBroadcast");
}

}  // extern "C"
