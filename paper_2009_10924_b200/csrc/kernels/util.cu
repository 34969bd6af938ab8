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

// One warp that busy-waits on the global timer: queued ahead of a timed
// launch it keeps the device busy while the host submits the launch and its
// events, so the events bracket the launch's device time and not the host's
// submission latency.
__global__ void __launch_bounds__(32) spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

}  // namespace

namespace stitch::gpu {

void launch_spin(unsigned long long ns, cudaStream_t s) { spin_kernel<<<1, 32, 0, s>>>(ns); }

void launch_l2_flush(void* buf, size_t bytes, cudaStream_t s) {
  l2_flush_kernel<<<148 * 8, 256, 0, s>>>(static_cast<uint4*>(buf), bytes / 16);
}

}  // namespace stitch::gpu
