// Low-level runtime C-ABI (SURVEY.md §8b "C-ABI the CUDA layer must
// export"): device context, NVRTC modules, ctx-owned device buffers,
// explicitly built CUDA Graphs of kernel launches, and an NCCL gather used by
// the multi-GPU verification path only.  The plan executor (abi_exec.cpp) is
// built from the same pieces; this layer lets a host that generates its own
// kernels drive the B200 without C++ types.
//
// NCCL is loaded lazily (dlopen libnccl.so.2) so the library keeps loading on
// hosts without it; the communicator's unique id travels out of band (the
// caller broadcasts the 128 bytes, e.g. over torch.distributed or a file).
// dlopen resolves by soname, so if the host process already loaded an NCCL
// (e.g. torch's bundled build) that one is shared; STITCH_NCCL_LIB overrides.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "abi/abi_common.h"
#include "runtime/cuda_rt.hpp"

using namespace stc_abi;
namespace gpu = stitch::gpu;

struct stc_ctx {
  int device = 0;
  std::set<void*> buffers;
  ~stc_ctx() {
    for (void* p : buffers) cudaFree(p);
  }
};

struct stc_module {
  stc_ctx* ctx = nullptr;
  std::unique_ptr<gpu::Module> mod;
  std::string key;
};

struct stc_cgraph {
  stc_ctx* ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t last = nullptr;
  int nodes = 0;
  ~stc_cgraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};

namespace {

// ---- NCCL through dlopen ----------------------------------------------------
struct NcclApi {
  typedef int (*GetUniqueId)(void* id);
  typedef int (*CommInitRank)(void** comm, int nranks, const void* id_by_value_128, int rank);
  typedef int (*AllGather)(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s);
  typedef int (*CommDestroy)(void* comm);
  typedef const char* (*ErrStr)(int);
  void* h = nullptr;
  GetUniqueId get_id = nullptr;
  void* init_rank = nullptr;  // ncclCommInitRank takes ncclUniqueId BY VALUE (128-byte struct)
  AllGather all_gather = nullptr;
  CommDestroy destroy = nullptr;
  ErrStr err = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  if (const char* p = std::getenv("STITCH_NCCL_LIB"); p && *p) api.h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    if (api.h) break;
    api.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
  }
  if (!api.h) throw std::runtime_error("[nccl] libnccl.so.2 not found");
  api.get_id = reinterpret_cast<NcclApi::GetUniqueId>(dlsym(api.h, "ncclGetUniqueId"));
  api.init_rank = dlsym(api.h, "ncclCommInitRank");
  api.all_gather = reinterpret_cast<NcclApi::AllGather>(dlsym(api.h, "ncclAllGather"));
  api.destroy = reinterpret_cast<NcclApi::CommDestroy>(dlsym(api.h, "ncclCommDestroy"));
  api.err = reinterpret_cast<NcclApi::ErrStr>(dlsym(api.h, "ncclGetErrorString"));
  if (!api.get_id || !api.init_rank || !api.all_gather || !api.destroy)
    throw std::runtime_error("[nccl] missing symbols in libnccl");
  return api;
}

void nccl_check(int r, const char* what) {
  if (r != 0)
    throw std::runtime_error(std::string("[nccl] ") + what + ": " + (nccl().err ? nccl().err(r) : std::to_string(r)));
}

struct UniqueId {
  char bytes[128];
};

}  // namespace

struct stc_comm {
  void* comm = nullptr;
  int nranks = 0, rank = 0;
  ~stc_comm() {
    if (comm) nccl().destroy(comm);
  }
};

extern "C" {

int stc_ctx_create(int device, stc_ctx** out) {
  return guarded([&] {
    gpu::device_init(device);
    auto c = std::make_unique<stc_ctx>();
    c->device = device;
    *out = c.release();
  });
}

void stc_ctx_destroy(stc_ctx* c) { delete c; }

int stc_ctx_compile(stc_ctx* c, const char* cuda_source, const char* const* kernel_names, int n,
                    stc_module** out) {
  return guarded([&] {
    if (!c || !cuda_source) throw std::invalid_argument("null context or source");
    STC_RT(cudaSetDevice(c->device));
    auto m = std::make_unique<stc_module>();
    m->ctx = c;
    m->mod = std::make_unique<gpu::Module>(gpu::compile_cubin(cuda_source, gpu::default_nvrtc_options(), &m->key));
    for (int i = 0; i < n; ++i) m->mod->fn(kernel_names[i]);  // resolve now: fail loudly on a bad name
    *out = m.release();
  });
}

void stc_module_destroy(stc_module* m) { delete m; }

int stc_ctx_alloc(stc_ctx* c, size_t bytes, void** dptr) {
  return guarded([&] {
    STC_RT(cudaSetDevice(c->device));
    void* p = nullptr;
    STC_RT(cudaMalloc(&p, bytes ? bytes : 1));
    c->buffers.insert(p);
    *dptr = p;
  });
}

int stc_ctx_release(stc_ctx* c, void* dptr) {
  return guarded([&] {
    if (!c->buffers.erase(dptr)) throw std::invalid_argument("buffer not owned by this context");
    STC_RT(cudaFree(dptr));
  });
}

int stc_ctx_upload(stc_ctx* c, void* dptr, const void* host, size_t bytes) {
  return guarded([&] {
    STC_RT(cudaSetDevice(c->device));
    STC_RT(cudaMemcpy(dptr, host, bytes, cudaMemcpyHostToDevice));
  });
}

int stc_ctx_download(stc_ctx* c, void* host, const void* dptr, size_t bytes) {
  return guarded([&] {
    STC_RT(cudaSetDevice(c->device));
    STC_RT(cudaMemcpy(host, dptr, bytes, cudaMemcpyDeviceToHost));
  });
}

int stc_cgraph_create(stc_ctx* c, stc_cgraph** out) {
  return guarded([&] {
    auto g = std::make_unique<stc_cgraph>();
    g->ctx = c;
    STC_RT(cudaGraphCreate(&g->graph, 0));
    *out = g.release();
  });
}

int stc_cgraph_add_kernel(stc_cgraph* g, stc_module* m, const char* name, int grid, int block, int smem_bytes,
                          int cooperative, void** args) {
  return guarded([&] {
    if (g->exec) throw std::invalid_argument("graph already instantiated");
    cudaKernel_t k = m->mod->fn(name);
    if (smem_bytes > 48 * 1024)
      STC_RT(cudaFuncSetAttribute(reinterpret_cast<const void*>(k), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_bytes));
    cudaKernelNodeParams p{};
    p.func = reinterpret_cast<void*>(k);
    p.gridDim = dim3(static_cast<unsigned>(grid));
    p.blockDim = dim3(static_cast<unsigned>(block));
    p.sharedMemBytes = static_cast<unsigned>(smem_bytes);
    p.kernelParams = args;
    cudaGraphNode_t node = nullptr;
    // launches run in insertion order, like a stream
    STC_RT(cudaGraphAddKernelNode(&node, g->graph, g->last ? &g->last : nullptr, g->last ? 1 : 0, &p));
    if (cooperative) {
      cudaLaunchAttributeValue v{};
      v.cooperative = 1;
      STC_RT(cudaGraphKernelNodeSetAttribute(node, cudaLaunchAttributeCooperative, &v));
    }
    g->last = node;
    ++g->nodes;
  });
}

int stc_cgraph_instantiate(stc_cgraph* g) {
  return guarded([&] {
    STC_RT(cudaSetDevice(g->ctx->device));
    if (!g->exec) STC_RT(cudaGraphInstantiate(&g->exec, g->graph, 0));
  });
}

int stc_cgraph_launch(stc_cgraph* g, void* cuda_stream) {
  return guarded([&] {
    if (!g->exec) throw std::invalid_argument("graph not instantiated");
    STC_RT(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(cuda_stream)));
  });
}

int stc_cgraph_time(stc_cgraph* g, int iters, size_t flush_bytes, float* us_per_iter) {
  return guarded([&] {
    if (!g->exec) throw std::invalid_argument("graph not instantiated");
    STC_RT(cudaSetDevice(g->ctx->device));
    cudaStream_t s = nullptr;
    STC_RT(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    void* flush = nullptr;
    if (flush_bytes) STC_RT(cudaMalloc(&flush, flush_bytes));
    cudaEvent_t a, b;
    STC_RT(cudaEventCreate(&a));
    STC_RT(cudaEventCreate(&b));
    float total = 0.f;
    STC_RT(cudaGraphLaunch(g->exec, s));  // warm-up
    for (int i = 0; i < iters; ++i) {
      if (flush) gpu::launch_l2_flush(flush, flush_bytes, s);  // L2 cold before every replay
      STC_RT(cudaEventRecord(a, s));
      STC_RT(cudaGraphLaunch(g->exec, s));
      STC_RT(cudaEventRecord(b, s));
      STC_RT(cudaEventSynchronize(b));
      float ms = 0.f;
      STC_RT(cudaEventElapsedTime(&ms, a, b));
      total += ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (flush) cudaFree(flush);
    cudaStreamDestroy(s);
    if (us_per_iter) *us_per_iter = 1000.f * total / static_cast<float>(iters > 0 ? iters : 1);
  });
}

void stc_cgraph_destroy(stc_cgraph* g) { delete g; }

int stc_nccl_unique_id(char* id128) {
  return guarded([&] { nccl_check(nccl().get_id(id128), "ncclGetUniqueId"); });
}

int stc_nccl_comm_init(stc_ctx* c, int nranks, int rank, const char* id128, stc_comm** out) {
  return guarded([&] {
    STC_RT(cudaSetDevice(c->device));
    UniqueId id;
    std::memcpy(id.bytes, id128, sizeof id.bytes);
    auto cm = std::make_unique<stc_comm>();
    cm->nranks = nranks;
    cm->rank = rank;
    auto init = reinterpret_cast<int (*)(void**, int, UniqueId, int)>(nccl().init_rank);
    nccl_check(init(&cm->comm, nranks, id, rank), "ncclCommInitRank");
    *out = cm.release();
  });
}

int stc_nccl_gather(stc_comm* cm, const void* send, void* recv, size_t bytes_per_rank, void* cuda_stream) {
  return guarded([&] {
    nccl_check(nccl().all_gather(send, recv, bytes_per_rank, /*ncclInt8*/ 0, cm->comm,
                                 static_cast<cudaStream_t>(cuda_stream)),
               "ncclAllGather");
  });
}

void stc_nccl_comm_destroy(stc_comm* cm) { delete cm; }

}  // extern "C"
