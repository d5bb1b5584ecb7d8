// nccl_dl.cpp -- NCCL entry points resolved at run time (dlopen), so the
// library has no link-time NCCL dependency and, inside a PyTorch process,
// shares the NCCL that torch already loaded (same soname libnccl.so.2).
#include <dlfcn.h>

#include <mutex>

#include "internal.h"

namespace helrm {

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
    api.broadcast = (decltype(api.broadcast))dlsym(h, "ncclBroadcast");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
    api.commGetAsyncError = (decltype(api.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.broadcast && api.allGather &&
             api.getErrorString && api.commGetAsyncError && api.groupStart && api.groupEnd;
  });
  if (!api.ok) throw Error(HELRM_ERR_NCCL, "libnccl.so.2 not loadable");
  return api;
}

}  // namespace helrm
