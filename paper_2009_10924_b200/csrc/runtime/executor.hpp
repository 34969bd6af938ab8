// Plan executor on one B200: the GPU replacement for the reference's
// eval_plan (/root/reference/proj/src/sim.cpp:471-514).
//
// Construction walks the graph in topological order exactly like eval_plan:
// a planned pattern fires at its topologically last member, every uncovered
// fusable op becomes a singleton kernel, every opaque op a placeholder
// kernel.  All kernels of the plan are generated into ONE CUDA source,
// compiled once by NVRTC (cached on disk), and captured into ONE CUDA Graph,
// so a whole-plan execution is a single cudaGraphLaunch.  Only tensors that
// cross a kernel boundary get device buffers.
#pragma once

#include <cuda_runtime.h>

#include <future>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "codegen/cg.hpp"
#include "runtime/cuda_rt.hpp"
#include "stitch/device.hpp"
#include "stitch/graph.hpp"
#include "stitch/planner.hpp"

namespace stitch::gpu {

enum class ExecMode { Stitched = 0, Program = 1, Unfused = 2 };

// All kernels of a plan, generated without touching a device (codegen only).
struct PlanKernels {
  std::vector<KernelSpec> specs;  // launch order
  std::vector<int> params;        // parameter vertices, ascending id
  std::string source;             // prelude + every kernel: one NVRTC module
};
// gemm_opaque (model mode, non-parity): opaque_compute ops shaped like a
// matmul (A[..,M,K] . B[K,N] -> [..,M,N], f32) become cuBLASLt GEMM units
// instead of the reference's mean-of-operands placeholder.
PlanKernels generate_plan_kernels(const CompGraph& g, const FusionPlan& plan,
                                  const std::map<std::string, KernelPlan>& kernels,
                                  const MachineModel& model, ExecMode mode, int sm_count = 148,
                                  bool gemm_opaque = false);
// is opaque vertex v a matmul A[..,M,K] . B[K,N] -> [..,M,N] (all f32)?
bool opaque_is_matmul(const CompGraph& g, int v, int64_t* m = nullptr, int64_t* n = nullptr, int64_t* k = nullptr);

// JSON array of {name, template, pattern, grid, block, smem, cooperative,
// bytes, inputs, outputs} per kernel (stc_exec_describe / stc_codegen)
std::string describe_specs(const std::vector<KernelSpec>& specs);

class Executor {
 public:
  Executor(const CompGraph& g, const FusionPlan& plan,
           const std::map<std::string, KernelPlan>& kernels, const MachineModel& model,
           int device, ExecMode mode, bool use_graph = true, bool gemm_opaque = false,
           bool async_compile = false);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  struct Tensor {
    std::string name;
    int vertex = -1;
    DType dtype = DType::F32;
    int64_t count = 0;
    size_t bytes = 0;
    std::vector<void*> dptr;  // one per buffer set
  };

  const std::vector<KernelSpec>& kernels() const { return specs_; }
  // async construction (paper's asynchronous compilation mode): NVRTC runs on
  // a worker thread; ready() polls, ensure_ready() waits + loads the module.
  // Every execution entry point calls ensure_ready() first.
  bool ready() const;
  void ensure_ready();
  const std::string& source() const { return source_; }
  const std::vector<int>& param_vertices() const { return params_; }
  const std::vector<int>& output_vertices() const { return g_.outputs; }
  const Tensor* tensor(const std::string& name) const;
  cudaStream_t stream() const { return stream_; }

  void upload(const void* const* host_inputs, int set = 0);
  void download(void* const* host_outputs, int set = 0);
  void launch(cudaStream_t s = nullptr, int set = 0);
  void prepare_sets(int sets);  // allocate + replicate set-0 parameters
  // B consecutive replays (rotating sets) captured into ONE graph, so the
  // host/graph launch cost is paid once per B steps; returns #batch graphs
  int prepare_batches(int sets, int batch);
  void launch_batch(cudaStream_t s, int index);
  void sync();
  void run_host(const void* const* in, void* const* out);
  // Host-buffer execution of a batch split into `nchunks` chunks of THIS
  // executor's graph (the chunk graph): chunk k of a chunked input starts at
  // byte k * tensor_bytes of its host buffer, unchunked inputs are shared by
  // every chunk, every output is chunked.  H2D of chunk k+1, the plan on
  // chunk k and D2H of chunk k-1 overlap on three streams (copy engines are
  // per direction), through min(nchunks, 3) device buffer sets.
  void run_host_chunked(const void* const* in, void* const* out, int nchunks, const int* in_chunked);
  // Generalisation: chunk k runs on chunk_exec[k] (shard graphs of one graph,
  // possibly of different batch sizes -- e.g. small first/last chunks to
  // shorten pipeline fill and drain); chunk offsets accumulate each chunk
  // executor's tensor bytes.  Copies on the first executor's streams.
  static void run_host_pipeline(const std::vector<Executor*>& chunk_exec, const void* const* in,
                                void* const* out, const int* in_chunked);
  // Zero-copy host execution: when every parameter and output buffer is
  // pinned host memory mapped into the device address space (cudaHostAlloc /
  // torch pin_memory under UVA), the plan's kernels read their inputs and
  // write their outputs over PCIe directly -- transfer fused with compute,
  // reads and writes overlapping in one pass.  Returns false (nothing done)
  // if some buffer is not device-accessible host memory.
  bool run_host_zero_copy(const void* const* in, void* const* out);

  // CUDA-event timing (see stc_exec_time in include/stitch_b200.h)
  double time(int iters, int warmup, int sets, std::vector<double>* per_kernel_us, int batch = 1);
  // Latency of one call on the device (see stc_exec_time_call): every
  // replay is queued behind a spinning warp so its bracketing events time
  // the replay, not the host's submission of it
  double time_call(int iters, int warmup, int sets, std::vector<double>* per_kernel_us);

  std::string describe_json() const;
  // one replay of set `set` with the in-graph timeline: per kernel (first CTA
  // entry, last CTA exit) in us since the earliest entry (-1 for GEMM units).
  // Needs STITCH_TRACE=1 at construction (adds -DSTITCH_TRACE to NVRTC).
  std::vector<std::pair<double, double>> trace(int set = 0);

 private:
  void plan_launches(const FusionPlan& plan, const std::map<std::string, KernelPlan>& kernels,
                     const MachineModel& model, ExecMode mode, bool gemm_opaque);
  void ensure_sets(int sets);
  // after_kernel: the kernel launched just before this one in the same stream
  // (-1: none) -- decides whether programmatic dependent launch applies
  void launch_kernel(size_t i, int set, cudaStream_t s, int after_kernel = -2,
                     const std::map<std::string, void*>* bind = nullptr);
  void build_graph(int set);
  // Capture one plan replay into `origin` (which must be capturing) as a DAG:
  // kernels whose inputs do not depend on each other go to different streams
  // (fork/join through events), a kernel that follows its producer on the
  // same stream keeps programmatic dependent launch.  `prev` = kernel that
  // ran last on `origin` before this replay (-1: none), for PDL across steps.
  // Returns the kernel left at the tail of `origin`.
  int capture_plan(int set, cudaStream_t origin, int prev);
  void compute_deps();
  void finish_init(const std::string& cubin);  // load module, resolve kernels, GEMM setup

  CompGraph g_;
  const DeviceInfo* dev_ = nullptr;
  bool use_graph_ = true;
  std::vector<KernelSpec> specs_;
  std::string source_;
  std::unique_ptr<Module> module_;
  std::future<std::string> pending_;  // async NVRTC compile
  std::vector<cudaKernel_t> fns_;
  std::vector<int> params_;
  std::map<std::string, Tensor> tensors_;
  std::vector<std::vector<void*>> scratch_;  // [set][kernel]
  int sets_ = 0;
  cudaStream_t stream_ = nullptr;
  std::vector<cudaGraphExec_t> graphs_;  // per set
  std::vector<cudaGraphExec_t> batch_graphs_;
  int batch_ = 0;
  bool coop_in_graph_ = true;
  bool pdl_ = true;  // STITCH_PDL=0 disables programmatic dependent launch
  bool tracing_ = false;
  int trace_ctas_ = 0;  // STITCH_TRACE_CTAS: per-CTA trace slots
  bool dag_ = true;  // STITCH_DAG=0 captures the plan as one linear chain
  bool sources_only_ = false;  // STITCH_DAG=2: fork only producer-less kernels
  std::vector<std::vector<int>> deps_;       // [kernel] -> producer kernels
  std::vector<cudaStream_t> aux_streams_;    // fork targets for independent kernels
  std::vector<cudaEvent_t> kernel_events_;   // [kernel] done-event (capture only)
  cudaEvent_t fork_event_ = nullptr;
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;   // chunked host runs
  struct GemmState;                               // cuBLASLt handle, descriptors, workspace
  std::unique_ptr<GemmState> gemm_;
  void launch_gemm(size_t i, void* a, void* b, void* c, cudaStream_t s);
  std::vector<cudaEvent_t> ev_in_, ev_comp_, ev_out_;
};

}  // namespace stitch::gpu
