// NCCL loaded at run time (dlopen) so liboica.so links against whichever libnccl.so.2 the
// process already carries (torch's bundled NCCL) -- only the stable core API is used.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "common.cuh"

namespace oica {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;

  static Nccl& get() {
    static Nccl n;
    if (!n.h) n.load();
    return n;
  }
  void load() {
    const char* names[] = {getenv("OICA_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm) continue;
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) throw Error(OICA_ERR_NCCL, "cannot dlopen libnccl.so.2 (set OICA_NCCL_LIB)");
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p) throw Error(OICA_ERR_NCCL, std::string("missing NCCL symbol ") + s);
      return p;
    };
    GetUniqueId = (decltype(GetUniqueId))sym("ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))sym("ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))sym("ncclCommDestroy");
    AllGather = (decltype(AllGather))sym("ncclAllGather");
    AllReduce = (decltype(AllReduce))sym("ncclAllReduce");
    Broadcast = (decltype(Broadcast))sym("ncclBroadcast");
    GetErrorString = (decltype(GetErrorString))sym("ncclGetErrorString");
    CommGetAsyncError = (decltype(CommGetAsyncError))sym("ncclCommGetAsyncError");
    CommAbort = (decltype(CommAbort))sym("ncclCommAbort");
    Send = (decltype(Send))sym("ncclSend");
    Recv = (decltype(Recv))sym("ncclRecv");
    GroupStart = (decltype(GroupStart))sym("ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))sym("ncclGroupEnd");
  }
};

#define OICA_NCCL(call)                                                                         \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess)                                                                      \
      throw ::oica::Error(OICA_ERR_NCCL, std::string(#call) + ": " +                            \
                                             ::oica::Nccl::get().GetErrorString(r_));           \
  } while (0)

}  // namespace oica
