#pragma once
// rbm_nccl.cuh -- the library's NCCL communicator for the partitioned single
// system (SURVEY.md 8(b) rbm_get_nccl_unique_id / rbm_init with an id, 8(e)).
//
// libnccl.so.2 is opened at first use (dlopen), so librbm.so loads without
// NCCL for single-GPU use and shares the NCCL that the process already has
// (torch's, when torch.distributed is in use).  Only the calls the step needs
// are resolved.  The CUDA driver's cuMemGetAddressRange is resolved the same
// way (IPC mapping of the workspace's allocation for the fused exchange).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace rbmhost {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  int (*MemGetAddressRange)(unsigned long long*, size_t*, unsigned long long) = nullptr;  // cuMemGetAddressRange_v2
};

inline NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot open libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather || !api.AllReduce ||
        !api.Send || !api.Recv || !api.GroupStart || !api.GroupEnd || !api.GetErrorString) {
      api.err = "libnccl.so.2 lacks a required symbol";
      return;
    }
    if (void* cu = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL))
      api.MemGetAddressRange = reinterpret_cast<decltype(api.MemGetAddressRange)>(dlsym(cu, "cuMemGetAddressRange_v2"));
    api.ok = true;
  });
  return api;
}

}  // namespace rbmhost
