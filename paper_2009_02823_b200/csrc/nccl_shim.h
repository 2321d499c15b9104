// Minimal runtime binding of NCCL (dlopen): the engine uses the libnccl.so.2
// already loaded by the process (torch's bundled NCCL) when present, so both
// share one library instance; no link-time dependency.
#pragma once
#include <dlfcn.h>

#include <cstddef>
#include <cuda_runtime.h>
#include <stdexcept>
#include <string>

namespace svgb {

// NCCL failures (status SVG_ENCCL at the C-ABI, RuntimeError in Python)
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct NcclUniqueId {
  char internal[128];
};
typedef struct ncclComm* NcclComm;

enum { kNcclSuccess = 0, kNcclUint8 = 1, kNcclFloat64 = 8 };

struct Nccl {
  using GetUniqueIdFn = int (*)(NcclUniqueId*);
  using CommInitRankFn = int (*)(NcclComm*, int, NcclUniqueId, int);
  using CommDestroyFn = int (*)(NcclComm);
  using CommAbortFn = int (*)(NcclComm);
  using SendFn = int (*)(const void*, size_t, int, int, NcclComm, cudaStream_t);
  using RecvFn = int (*)(void*, size_t, int, int, NcclComm, cudaStream_t);
  using GroupFn = int (*)();
  using AllGatherFn = int (*)(const void*, void*, size_t, int, NcclComm, cudaStream_t);
  using ErrorStringFn = const char* (*)(int);

  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  CommAbortFn comm_abort = nullptr;
  SendFn send = nullptr;
  RecvFn recv = nullptr;
  GroupFn group_start = nullptr;
  GroupFn group_end = nullptr;
  AllGatherFn all_gather = nullptr;
  ErrorStringFn error_string = nullptr;

  static Nccl& get() {
    static Nccl n = load();
    return n;
  }

  void check(int rc, const char* what) const {
    if (rc != kNcclSuccess)
      throw NcclError(std::string(what) + ": " + (error_string ? error_string(rc) : "nccl error"));
  }

 private:
  static Nccl load() {
    Nccl n;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch) first
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw NcclError("libnccl.so.2 not found");
    auto sym = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f) throw NcclError(std::string("NCCL symbol missing: ") + name);
      return f;
    };
    n.get_unique_id = reinterpret_cast<GetUniqueIdFn>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<CommInitRankFn>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<CommDestroyFn>(sym("ncclCommDestroy"));
    n.comm_abort = reinterpret_cast<CommAbortFn>(sym("ncclCommAbort"));
    n.send = reinterpret_cast<SendFn>(sym("ncclSend"));
    n.recv = reinterpret_cast<RecvFn>(sym("ncclRecv"));
    n.group_start = reinterpret_cast<GroupFn>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<GroupFn>(sym("ncclGroupEnd"));
    n.all_gather = reinterpret_cast<AllGatherFn>(sym("ncclAllGather"));
    n.error_string = reinterpret_cast<ErrorStringFn>(sym("ncclGetErrorString"));
    return n;
  }
};

}  // namespace svgb
