#include <thread>
#include <mutex>
#include <atomic>
// extern "C" boundary, device half: code generation, NVRTC, the CUDA-Graph
// executor (include/stitch_b200.h).
#include <cstring>
#include <memory>
#include <sstream>

#include "abi/abi_common.h"
#include "runtime/executor.hpp"

using namespace stitch;
using namespace stc_abi;

struct stc_exec {
  std::unique_ptr<gpu::Executor> ex;
};

namespace {

gpu::ExecMode mode_of(int mode) {
  switch (mode & 7) {
    case STC_EXEC_PROGRAM: return gpu::ExecMode::Program;
    case STC_EXEC_UNFUSED: return gpu::ExecMode::Unfused;
    default: return gpu::ExecMode::Stitched;
  }
}

}  // namespace

extern "C" {

int stc_codegen(const stc_plan* p, int mode, char** cuda_source, char** kernels_json) {
  return guarded([&] {
    auto pk = gpu::generate_plan_kernels(p->graph, p->plan, p->kernels, p->models.machine, mode_of(mode), 148,
                                         (mode & STC_EXEC_GEMM) != 0);
    if (cuda_source) *cuda_source = dup_string(pk.source);
    if (kernels_json) *kernels_json = dup_string(gpu::describe_specs(pk.specs));
  });
}

int stc_exec_create(const stc_plan* p, int device, int mode, stc_exec** out) {
  return guarded([&] {
    auto e = std::make_unique<stc_exec>();
    e->ex = std::make_unique<gpu::Executor>(p->graph, p->plan, p->kernels, p->models.machine, device,
                                            mode_of(mode), (mode & STC_EXEC_NO_GRAPH) == 0,
                                            (mode & STC_EXEC_GEMM) != 0);
    *out = e.release();
  });
}

int stc_exec_create_async(const stc_plan* p, int device, int mode, stc_exec** out) {
  return guarded([&] {
    auto e = std::make_unique<stc_exec>();
    e->ex = std::make_unique<gpu::Executor>(p->graph, p->plan, p->kernels, p->models.machine, device,
                                            mode_of(mode), (mode & STC_EXEC_NO_GRAPH) == 0,
                                            (mode & STC_EXEC_GEMM) != 0, /*async_compile=*/true);
    *out = e.release();
  });
}

int stc_exec_ready(const stc_exec* e) { return e && e->ex->ready() ? 1 : 0; }

int stc_exec_wait(stc_exec* e) {
  return guarded([&] { e->ex->ensure_ready(); });
}

int stc_cache_warm(const stc_plan* const* plans, int n, int mode, int threads, int* compiled, int* cached) {
  return guarded([&] {
    std::vector<std::string> sources;
    for (int i = 0; i < n; ++i)
      sources.push_back(gpu::generate_plan_kernels(plans[i]->graph, plans[i]->plan, plans[i]->kernels,
                                                   plans[i]->models.machine, mode_of(mode), 148,
                                                   (mode & STC_EXEC_GEMM) != 0)
                            .source);
    std::atomic<int> next{0}, comp{0}, hit{0};
    std::string err;
    std::mutex mu;
    auto work = [&] {
      for (int i; (i = next++) < static_cast<int>(sources.size());) {
        try {
          bool h = false;
          gpu::compile_cubin(sources[static_cast<size_t>(i)], gpu::default_nvrtc_options(), nullptr, &h);
          (h ? hit : comp)++;
        } catch (const std::exception& ex) {
          std::lock_guard<std::mutex> lk(mu);
          if (err.empty()) err = ex.what();
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, std::min(threads, n)); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    if (!err.empty()) throw std::runtime_error(err);
    if (compiled) *compiled = comp;
    if (cached) *cached = hit;
  });
}

void stc_exec_destroy(stc_exec* e) { delete e; }

int stc_exec_num_kernels(const stc_exec* e) { return static_cast<int>(e->ex->kernels().size()); }

int stc_exec_describe(const stc_exec* e, char** json) {
  return guarded([&] { *json = dup_string(e->ex->describe_json()); });
}

int stc_exec_source(const stc_exec* e, char** src) {
  return guarded([&] { *src = dup_string(e->ex->source()); });
}

int stc_exec_run_host(stc_exec* e, const void* const* inputs, void* const* outputs) {
  return guarded([&] { e->ex->run_host(inputs, outputs); });
}

int stc_exec_trace(stc_exec* e, double* start_us, double* end_us) {
  return guarded([&] {
    const auto t = e->ex->trace(0);
    for (size_t i = 0; i < t.size(); ++i) {
      if (start_us) start_us[i] = t[i].first;
      if (end_us) end_us[i] = t[i].second;
    }
  });
}

int stc_exec_run_host_zero_copy(stc_exec* e, const void* const* inputs, void* const* outputs) {
  return guarded([&] {
    if (!e->ex->run_host_zero_copy(inputs, outputs))
      throw std::runtime_error("[exec] zero-copy run needs pinned, device-mapped host buffers for every input/output");
  });
}

int stc_exec_run_host_chunked(stc_exec* e, const void* const* inputs, void* const* outputs, int nchunks,
                              const int* input_chunked) {
  return guarded([&] { e->ex->run_host_chunked(inputs, outputs, nchunks, input_chunked); });
}

int stc_exec_run_host_pipeline(stc_exec* const* execs, const int* exec_of_chunk, int nchunks,
                               const void* const* inputs, void* const* outputs, const int* input_chunked) {
  return guarded([&] {
    if (nchunks < 1 || !execs || !exec_of_chunk) throw std::invalid_argument("[abi] bad pipeline arguments");
    std::vector<gpu::Executor*> ex;
    for (int k = 0; k < nchunks; ++k) ex.push_back(execs[exec_of_chunk[k]]->ex.get());
    gpu::Executor::run_host_pipeline(ex, inputs, outputs, input_chunked);
  });
}

int stc_exec_upload(stc_exec* e, const void* const* inputs) {
  return guarded([&] { e->ex->upload(inputs, 0); });
}

int stc_exec_launch(stc_exec* e, void* stream, int set) {
  return guarded([&] { e->ex->launch(static_cast<cudaStream_t>(stream), set); });
}

int stc_exec_prepare_sets(stc_exec* e, int sets) {
  return guarded([&] { e->ex->prepare_sets(sets); });
}

int stc_exec_download(stc_exec* e, void* const* outputs) {
  return guarded([&] { e->ex->download(outputs, 0); });
}

int stc_exec_sync(stc_exec* e) {
  return guarded([&] { e->ex->sync(); });
}

int stc_exec_tensor(const stc_exec* e, const char* name, void** dptr, size_t* bytes) {
  const auto* t = e->ex->tensor(name ? name : "");
  if (!t) {
    g_error = std::string("[abi] no device buffer for tensor ") + (name ? name : "(null)");
    return 4;
  }
  if (dptr) *dptr = t->dptr.empty() ? nullptr : t->dptr[0];
  if (bytes) *bytes = t->bytes;
  return 0;
}

int stc_exec_time(stc_exec* e, int iters, int warmup, int sets, double* us_per_run, double* kernel_us) {
  return guarded([&] {
    std::vector<double> per;
    const double us = e->ex->time(iters, warmup, sets, kernel_us ? &per : nullptr);
    if (us_per_run) *us_per_run = us;
    if (kernel_us)
      for (size_t i = 0; i < per.size(); ++i) kernel_us[i] = per[i];
  });
}

int stc_exec_time_call(stc_exec* e, int iters, int warmup, int sets, double* us_per_call, double* kernel_us) {
  return guarded([&] {
    std::vector<double> per;
    const double us = e->ex->time_call(iters, warmup, sets, kernel_us ? &per : nullptr);
    if (us_per_call) *us_per_call = us;
    if (kernel_us)
      for (size_t i = 0; i < per.size(); ++i) kernel_us[i] = per[i];
  });
}

int stc_exec_prepare_batches(stc_exec* e, int sets, int steps_per_graph, int* n_graphs) {
  return guarded([&] {
    const int n = e->ex->prepare_batches(sets, steps_per_graph);
    if (n_graphs) *n_graphs = n;
  });
}

int stc_exec_launch_batch(stc_exec* e, void* stream, int index) {
  return guarded([&] { e->ex->launch_batch(static_cast<cudaStream_t>(stream), index); });
}

int stc_exec_time_batched(stc_exec* e, int steps, int warmup, int sets, int steps_per_graph,
                          double* us_per_step) {
  return guarded([&] {
    const double us = e->ex->time(steps, warmup, sets, nullptr, steps_per_graph);
    if (us_per_step) *us_per_step = us;
  });
}

int stc_compile(const char* cuda_source, const char* options, char** cubin_key) {
  return guarded([&] {
    std::vector<std::string> opts = gpu::default_nvrtc_options();
    if (options && *options) {
      std::istringstream ss(options);
      for (std::string o; ss >> o;) opts.push_back(o);
    }
    std::string key;
    gpu::compile_cubin(cuda_source, opts, &key);
    if (cubin_key) *cubin_key = dup_string(key);
  });
}

const char* stc_cache_dir(void) {
  static thread_local std::string d;
  d = gpu::cubin_cache_dir();
  return d.c_str();
}

}  // extern "C"
