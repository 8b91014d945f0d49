// NCCL plumbing for the sharded search. NCCL is resolved at
// run time (dlopen of libnccl.so.2 — the system 2.27 or the one torch already
// loaded) so single-GPU users do not need it.
#include <dlfcn.h>

#include <cstring>

#include "search.hpp"

namespace hpg {

namespace {

struct NcclApi {
  void* lib = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*comm_init_rank)(void**, int, const void*, int) = nullptr;  // id passed by value (128 B)
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*get_error_string)(int) = nullptr;
};

struct UniqueId {
  char internal[128];
};

NcclApi& api() {
  static NcclApi a;
  if (a.lib) return a;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    a.lib = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    if (a.lib) break;
  }
  if (!a.lib) throw InternalError("multi-GPU search needs NCCL (libnccl.so.2 not found)");
  a.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(a.lib, "ncclGetUniqueId"));
  a.all_gather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
      dlsym(a.lib, "ncclAllGather"));
  a.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(a.lib, "ncclCommDestroy"));
  a.get_error_string = reinterpret_cast<const char* (*)(int)>(dlsym(a.lib, "ncclGetErrorString"));
  a.comm_init_rank = reinterpret_cast<int (*)(void**, int, const void*, int)>(
      dlsym(a.lib, "ncclCommInitRank"));
  if (!a.get_unique_id || !a.all_gather || !a.comm_destroy || !a.comm_init_rank)
    throw InternalError("libnccl.so.2 lacks the expected symbols");
  return a;
}

void nccl_check(int rc, const char* what) {
  if (rc != 0) {
    const char* msg = api().get_error_string ? api().get_error_string(rc) : "nccl error";
    throw InternalError(std::string(what) + ": " + msg);
  }
}

// ncclCommInitRank takes the 128-byte ncclUniqueId by value; call through a
// prototype with the struct type so the ABI passes it in memory.
using InitFn = int (*)(void**, int, UniqueId, int);

}  // namespace

void dist_unique_id(uint8_t out[128]) {
  UniqueId id;
  nccl_check(api().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

void dist_init(Dist& d, int rank, int world, const uint8_t idb[128], int device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  UniqueId id;
  std::memcpy(id.internal, idb, 128);
  d.rank = rank;
  d.world = world;
  auto init = reinterpret_cast<InitFn>(reinterpret_cast<void*>(api().comm_init_rank));
  void* comm = nullptr;
  nccl_check(init(&comm, world, id, rank), "ncclCommInitRank");
  d.comm = comm;
}

void dist_allgather(Dist& d, const void* send, void* recv, size_t bytes, cudaStream_t st) {
  // ncclUint8 = 1
  nccl_check(api().all_gather(send, recv, bytes, 1, d.comm, st), "ncclAllGather");
}

void dist_destroy(Dist& d) {
  if (d.comm) api().comm_destroy(d.comm);
  d.comm = nullptr;
}

}  // namespace hpg
