// Data-parallel gradient all-reduce over NCCL (NVLink / NVSwitch), loaded at
// run time with dlopen so the library has no link-time NCCL dependency (the
// process normally already holds torch's libnccl.so.2).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace rfx {

class NcclComm {
 public:
  static bool get_unique_id(char out[128], std::string* err);
  bool init(int nranks, int rank, const char id[128], std::string* err);
  ~NcclComm();
  bool ready() const { return comm_ != nullptr; }
  int nranks() const { return nranks_; }
  // in-place average of `count` floats
  bool allreduce_avg(float* buf, size_t count, cudaStream_t st, std::string* err);
  // in-place broadcast of `count` floats from `root`
  bool broadcast(float* buf, size_t count, int root, cudaStream_t st, std::string* err);

 private:
  void* comm_ = nullptr;
  int nranks_ = 1;
};

}  // namespace rfx
