// CUDA layer under the executor: device init, NVRTC compilation for sm_100a
// with an on-disk cubin cache ("compiled once per plan"), module loading.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

namespace stitch::gpu {

[[noreturn]] void throw_cuda(const char* what, const char* detail);

#define STC_RT(x)                                                  \
  do {                                                             \
    cudaError_t r_ = (x);                                          \
    if (r_ != cudaSuccess) ::stitch::gpu::throw_cuda(#x, cudaGetErrorString(r_)); \
  } while (0)

struct DeviceInfo {
  int ordinal = 0;
  int sm_count = 0;
  int l2_bytes = 0;
  int max_smem_optin = 0;
  int cc_major = 0, cc_minor = 0;
};

// selects the device, initialises the primary context, caches attributes
const DeviceInfo& device_init(int ordinal);

// NVRTC for sm_100a; returns the cubin image, using/refreshing the cache.
// `key_out` receives the content hash that names the cache entry.
std::string compile_cubin(const std::string& source, const std::vector<std::string>& options,
                          std::string* key_out = nullptr, bool* cache_hit = nullptr);
std::string cubin_cache_dir();
std::vector<std::string> default_nvrtc_options();

// loaded module (one per plan) with its kernels.  Runtime-API libraries
// (cudaLibraryLoadData), so this library never links libcuda directly and
// loads on hosts without a driver (code generation / NVRTC still work).
class Module {
 public:
  explicit Module(const std::string& cubin);
  ~Module();
  Module(const Module&) = delete;
  Module& operator=(const Module&) = delete;
  cudaKernel_t fn(const std::string& name);
  // device address + size of a __device__ global of the module (nullptr if absent)
  void* global(const std::string& name, size_t* bytes = nullptr);

 private:
  cudaLibrary_t lib_ = nullptr;
  std::map<std::string, cudaKernel_t> fns_;
};

// fixed kernels compiled by nvcc into this library (csrc/kernels/util.cu)
void launch_l2_flush(void* buf, size_t bytes, cudaStream_t s);
// one warp spinning for `ns` nanoseconds of device time (timing prelude)
void launch_spin(unsigned long long ns, cudaStream_t s);

}  // namespace stitch::gpu
