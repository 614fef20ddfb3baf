// comm_internal.h — the NCCL entry points libspikerl.so loads at run time (comm.cu), shared with the
// fused allreduce + Adam (k_fused_dp.cu). Host code only.
#pragma once
#include <string>
#include <nccl.h>
#include <nccl_device.h>

namespace spk {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclCommGetAsyncError) asyncErr = nullptr;
  // symmetric memory + device API (NCCL >= 2.28; optional)
  decltype(&ncclMemAlloc) memAlloc = nullptr;
  decltype(&ncclMemFree) memFree = nullptr;
  decltype(&ncclCommWindowRegister) winRegister = nullptr;
  decltype(&ncclCommWindowDeregister) winDeregister = nullptr;
  decltype(&ncclDevCommCreate) devCommCreate = nullptr;
  decltype(&ncclDevCommDestroy) devCommDestroy = nullptr;
  std::string why;
};

NcclApi& nccl_api();
int nccl_status(ncclResult_t r, const char* what);
int nccl_need_api();
ncclComm_t comm_nccl(const spikerl_comm* c);
int comm_world(const spikerl_comm* c);

}  // namespace spk
