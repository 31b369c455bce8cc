// NCCL binding via dlopen (see comm.h).
#include "executor/comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>

namespace rfx {

namespace {

struct UniqueId {
  char internal[128];
};
using ncclResult_t = int;
using FnGetUniqueId = ncclResult_t (*)(UniqueId*);
using FnCommInitRank = ncclResult_t (*)(void**, int, UniqueId, int);
using FnAllReduce = ncclResult_t (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
using FnBroadcast = ncclResult_t (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
using FnCommDestroy = ncclResult_t (*)(void*);
using FnGetErrorString = const char* (*)(ncclResult_t);

constexpr int kNcclFloat32 = 7;
constexpr int kNcclAvg = 4;

struct Api {
  FnGetUniqueId get_unique_id = nullptr;
  FnCommInitRank comm_init_rank = nullptr;
  FnAllReduce all_reduce = nullptr;
  FnBroadcast broadcast = nullptr;
  FnCommDestroy comm_destroy = nullptr;
  FnGetErrorString error_string = nullptr;
  bool ok = false;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.get_unique_id = reinterpret_cast<FnGetUniqueId>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<FnCommInitRank>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<FnAllReduce>(dlsym(h, "ncclAllReduce"));
    a.broadcast = reinterpret_cast<FnBroadcast>(dlsym(h, "ncclBroadcast"));
    a.comm_destroy = reinterpret_cast<FnCommDestroy>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<FnGetErrorString>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.broadcast && a.comm_destroy;
  });
  return a;
}

bool fail(std::string* err, const std::string& what, int rc) {
  if (err) {
    *err = what;
    if (rc && api().error_string) *err += std::string(": ") + api().error_string(rc);
  }
  return false;
}

}  // namespace

bool NcclComm::get_unique_id(char out[128], std::string* err) {
  if (!api().ok) return fail(err, "NCCL not available (libnccl.so.2 not found)", 0);
  UniqueId id;
  const int rc = api().get_unique_id(&id);
  if (rc != 0) return fail(err, "ncclGetUniqueId", rc);
  std::memcpy(out, id.internal, 128);
  return true;
}

bool NcclComm::init(int nranks, int rank, const char id[128], std::string* err) {
  if (!api().ok) return fail(err, "NCCL not available (libnccl.so.2 not found)", 0);
  UniqueId u;
  std::memcpy(u.internal, id, 128);
  const int rc = api().comm_init_rank(&comm_, nranks, u, rank);
  if (rc != 0) {
    comm_ = nullptr;
    return fail(err, "ncclCommInitRank", rc);
  }
  nranks_ = nranks;
  return true;
}

NcclComm::~NcclComm() {
  if (comm_ && api().ok) api().comm_destroy(comm_);
}

bool NcclComm::allreduce_avg(float* buf, size_t count, cudaStream_t st, std::string* err) {
  const int rc = api().all_reduce(buf, buf, count, kNcclFloat32, kNcclAvg, comm_, st);
  if (rc != 0) return fail(err, "ncclAllReduce", rc);
  return true;
}

bool NcclComm::broadcast(float* buf, size_t count, int root, cudaStream_t st, std::string* err) {
  const int rc = api().broadcast(buf, buf, count, kNcclFloat32, root, comm_, st);
  if (rc != 0) return fail(err, "ncclBroadcast", rc);
  return true;
}

}  // namespace rfx
