// comm.cuh — NCCL for the multi-GPU slab decomposition (SURVEY §8(b) sph_comm_unique_id /
// sph_comm_init, §8(e) halo exchange; the paper's two communication tasks per proxy cell,
// P:1065-1105). NCCL is loaded at run time (dlopen "libnccl.so.2": in a process that already
// holds torch's NCCL this is that library), so libsph has no link-time NCCL dependency and
// every single-GPU entry point works without it.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
#define NCCL_SYM(f)                                                    \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f));      \
  if (!api.f) {                                                        \
    api.why = "libnccl lacks nccl" #f;                                 \
    return;                                                            \
  }
    NCCL_SYM(GetUniqueId)
    NCCL_SYM(CommInitRank)
    NCCL_SYM(CommDestroy)
    NCCL_SYM(Send)
    NCCL_SYM(Recv)
    NCCL_SYM(AllReduce)
    NCCL_SYM(GroupStart)
    NCCL_SYM(GroupEnd)
    NCCL_SYM(GetErrorString)
#undef NCCL_SYM
    api.ok = true;
  });
  return api;
}

#define NCCL_TRY(x)                                                                     \
  do {                                                                                  \
    const ncclResult_t r_ = (x);                                                        \
    if (r_ != ncclSuccess)                                                              \
      throw SphError{SPH_E_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_)};   \
  } while (0)
