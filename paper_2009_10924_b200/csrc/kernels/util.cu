// Fixed sm_100a kernels compiled by nvcc into libstitch_b200.so (the stitched
// kernels themselves are generated per plan and compiled by NVRTC).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

// Streams a buffer larger than L2 through the cache (write-allocate), evicting
// whatever a timed replay left behind.
__global__ void __launch_bounds__(256) l2_flush_kernel(uint4* __restrict__ buf, size_t n16) {
  const uint4 v = make_uint4(threadIdx.x, blockIdx.x, 0u, 0u);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
    buf[i] = v;
}

}  // namespace

namespace stitch::gpu {

void launch_l2_flush(void* buf, size_t bytes, cudaStream_t s) {
  l2_flush_kernel<<<148 * 8, 256, 0, s>>>(static_cast<uint4*>(buf), bytes / 16);
}

}  // namespace stitch::gpu
