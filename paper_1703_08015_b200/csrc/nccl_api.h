// NCCL entry points resolved at run time (dlopen "libnccl.so.2"): the library joins whichever NCCL
// the process already loaded (torch's bundled copy when torch is imported) instead of linking a
// second one. Used by the native slab halo exchange (engine.cpp).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

namespace splbm_host {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// The resolved API; throws Error(SPLBM_ERR_CUDA) if NCCL cannot be loaded.
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);

}  // namespace splbm_host
