#include "runtime/executor.hpp"

#include <cublasLt.h>

#include <algorithm>
#include <chrono>
#include <future>
#include <cstdio>
#include <regex>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <set>
#include <sstream>
#include <stdexcept>

namespace stitch::gpu {

namespace {

std::string sanitize(const std::string& s) {
  std::string o;
  for (char c : s) o += (std::isalnum(static_cast<unsigned char>(c)) ? c : '_');
  return o;
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}

}  // namespace

// csrc/kernels/gemm_sm100.cu (CUTLASS tcgen05 GEMM + bias + GELU epilogue)
int gemm_bias_gelu_tf32(const float* A, const float* B, const float* bias, float* D, int M, int N, int K, void* workspace,
                        size_t workspace_bytes, cudaStream_t stream);
bool gemm_bias_gelu_supported(int M, int N, int K, size_t workspace_bytes);
int gemm_tf32(int variant, bool fused, const float* A, const float* B, const float* bias, float* D, int M, int N, int K,
              void* workspace, size_t workspace_bytes, cudaStream_t stream);
long long gemm_tf32_workspace(int variant, bool fused, int M, int N, int K);
int gemm_tf32_launch(int variant, bool fused, bool pdl, const float* A, const float* B, const float* bias, float* D, int M,
                     int N, int K, void* workspace, size_t workspace_bytes, cudaStream_t stream);

namespace {
// the plan's bias + GELU(tanh) pattern over one GEMM output (graphs/
// bert_layer.graph): gl = (a*0.5) * (tanh((a + (a*a*a)*0.044715) * 0.79788456) + 1),
// a = G + broadcast(bias[N]) dims=[1].  Commuted operands accepted.
// -> the pattern's output vertex, the GEMM output G and the bias parameter.
bool match_bias_gelu(const CompGraph& g, const std::vector<int>& verts, int* G_out, int* bias_out, int* out_v) {
  const std::set<int> in(verts.begin(), verts.end());
  auto node = [&](int v) -> const OpNode& { return g.node(v); };
  auto cbcast = [&](int v, double val) {
    const OpNode& n = node(v);
    if (n.kind != OpKind::Broadcast || n.operands.size() != 1) return false;
    const OpNode& c = node(n.operands[0]);
    return c.kind == OpKind::Constant && std::fabs(c.attrs.value - val) <= 1e-6 * std::fabs(val);
  };
  // binary op of kind k with operands {x, y} in either order; calls pick(x, y)
  auto bin = [&](int v, OpKind k, auto&& pick) {
    const OpNode& n = node(v);
    if (n.kind != k || n.operands.size() != 2) return false;
    return pick(n.operands[0], n.operands[1]) || pick(n.operands[1], n.operands[0]);
  };
  // the pattern's single output: the vertex no other member reads
  int out = -1;
  for (int v : verts) {
    bool read = false;
    for (int w : verts)
      for (int o : node(w).operands) read = read || o == v;
    if (!read) {
      if (out >= 0) return false;
      out = v;
    }
  }
  if (out < 0) return false;
  int a = -1;
  auto is_a = [&](int v) {
    return bin(v, OpKind::Add, [&](int x, int y) {
      const OpNode& b = node(y);
      if (b.kind != OpKind::Broadcast || b.attrs.dims != std::vector<int>{1}) return false;
      const OpNode& bias = node(b.operands[0]);
      if (bias.kind != OpKind::Parameter || bias.shape.rank() != 1 || in.count(x)) return false;
      if (a >= 0 && a != v) return false;
      a = v, *G_out = x, *bias_out = bias.id;
      return true;
    });
  };
  const bool ok = bin(out, OpKind::Mul, [&](int ah, int th1) {
    return bin(ah, OpKind::Mul, [&](int x, int c) { return is_a(x) && cbcast(c, 0.5); }) &&
           bin(th1, OpKind::Add, [&](int th, int c) {
             if (!cbcast(c, 1.0) || node(th).kind != OpKind::Tanh) return false;
             return bin(node(th).operands[0], OpKind::Mul, [&](int inner, int c2) {
               return cbcast(c2, 0.7978845608028654) && bin(inner, OpKind::Add, [&](int x, int a3s) {
                        return x == a && bin(a3s, OpKind::Mul, [&](int a3, int c3) {
                                 return cbcast(c3, 0.044715) && bin(a3, OpKind::Mul, [&](int a2, int y) {
                                          return y == a && bin(a2, OpKind::Mul, [&](int p, int q) { return p == a && q == a; });
                                        });
                               });
                      });
             });
           });
  });
  // every member is one of the recognised ops (nothing else computed here)
  *out_v = out;
  return ok && a >= 0 && in.count(a) && verts.size() <= 16;
}
}  // namespace

// cuBLASLt state for the plan's GEMM units (model mode)
struct Executor::GemmState {
  cublasLtHandle_t lt = nullptr;
  void* workspace = nullptr;
  size_t ws_bytes = size_t(32) << 20;
  struct Unit {
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
    cublasLtMatmulAlgo_t algo{};
    // CUTLASS configuration (gemm_sm100.cu) instead of cuBLASLt; -1 =
    // cuBLASLt.  Its workspace is the unit's per-set scratch
    int variant = -1;
  };
  std::map<size_t, Unit> units;
  ~GemmState() {
    for (auto& [i, u] : units) {
      if (u.op) cublasLtMatmulDescDestroy(u.op);
      if (u.a) cublasLtMatrixLayoutDestroy(u.a);
      if (u.b) cublasLtMatrixLayoutDestroy(u.b);
      if (u.c) cublasLtMatrixLayoutDestroy(u.c);
    }
    if (workspace) cudaFree(workspace);
    if (lt) cublasLtDestroy(lt);
  }
};

#define STC_LT(x)                                                                          \
  do {                                                                                     \
    cublasStatus_t st_ = (x);                                                              \
    if (st_ != CUBLAS_STATUS_SUCCESS)                                                      \
      throw std::runtime_error(std::string("[cublasLt] ") + #x + " failed: status " + std::to_string(int(st_))); \
  } while (0)

bool opaque_is_matmul(const CompGraph& g, int v, int64_t* m, int64_t* n, int64_t* k) {
  const OpNode& node = g.node(v);
  if (classify_op(node) != OpClass::Opaque || node.operands.size() != 2) return false;
  const TensorShape& a = g.node(node.operands[0]).shape;
  const TensorShape& b = g.node(node.operands[1]).shape;
  const TensorShape& c = node.shape;
  if (a.dtype != DType::F32 || b.dtype != DType::F32 || c.dtype != DType::F32) return false;
  if (a.rank() < 2 || b.rank() != 2 || c.rank() != a.rank()) return false;
  const int64_t K = a.dims.back(), N = b.dims[1];
  if (b.dims[0] != K || c.dims.back() != N) return false;
  for (int i = 0; i + 1 < a.rank(); ++i)
    if (a.dims[static_cast<size_t>(i)] != c.dims[static_cast<size_t>(i)]) return false;
  if (m) *m = a.element_count() / K;
  if (n) *n = N;
  if (k) *k = K;
  return true;
}

Executor::Executor(const CompGraph& g, const FusionPlan& plan,
                   const std::map<std::string, KernelPlan>& kernels, const MachineModel& model,
                   int device, ExecMode mode, bool use_graph, bool gemm_opaque, bool async_compile)
    : g_(g), use_graph_(use_graph) {
  dev_ = &device_init(device);
  if (const char* v = std::getenv("STITCH_PDL")) pdl_ = *v != '0';
  if (const char* v = std::getenv("STITCH_DAG")) {
    dag_ = *v != '0';
    sources_only_ = *v == '2';
  }
  STC_RT(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  plan_launches(plan, kernels, model, mode, gemm_opaque);
  auto opts = default_nvrtc_options();
  if (const char* t = std::getenv("STITCH_TRACE"); t && *t == '1') {
    opts.push_back("-DSTITCH_TRACE");
    tracing_ = true;
    // STITCH_TRACE_CTAS=c: slot k of CTA b < c is recorded on its own
    // (slot k*c + b), so per-CTA step times come back without cross-CTA skew
    if (const char* c = std::getenv("STITCH_TRACE_CTAS"); c && std::atoi(c) > 0) {
      trace_ctas_ = std::atoi(c);
      opts.push_back("-DSTITCH_TRACE_CTAS=" + std::to_string(trace_ctas_));
    }
  }
  ensure_sets(1);
  if (async_compile) {
    // NVRTC on a worker thread (no device work); the first call that needs
    // the kernels waits for it (ensure_ready)
    pending_ = std::async(std::launch::async, [src = source_, opts] { return compile_cubin(src, opts); });
    return;
  }
  finish_init(compile_cubin(source_, opts));
}

bool Executor::ready() const {
  return module_ != nullptr ||
         (pending_.valid() && pending_.wait_for(std::chrono::seconds(0)) == std::future_status::ready);
}

void Executor::ensure_ready() {
  // every entry point binds the executor's device first, so executors of
  // several GPUs can be driven from one host thread
  STC_RT(cudaSetDevice(dev_->ordinal));
  if (module_) return;
  if (!pending_.valid()) throw std::runtime_error("[exec] executor has no module");
  finish_init(pending_.get());
}

void Executor::finish_init(const std::string& cubin) {
  module_ = std::make_unique<Module>(cubin);
  for (size_t ki = 0; ki < specs_.size(); ++ki) {
    const KernelSpec& k = specs_[ki];
    if (k.is_gemm) {
      // C[M,N] = A[M,K] . B[K,N] row-major == column-major C^T = B^T . A^T:
      // cuBLASLt (m, n, k) = (N, M, K) with B first, all non-transposed
      if (!gemm_) {
        gemm_ = std::make_unique<GemmState>();
        STC_LT(cublasLtCreate(&gemm_->lt));
        STC_RT(cudaMalloc(&gemm_->workspace, gemm_->ws_bytes));
        // zeroed once (hygiene; 32 MB at executor creation)
        STC_RT(cudaMemset(gemm_->workspace, 0, gemm_->ws_bytes));
      }
      const char* fp32 = std::getenv("STITCH_GEMM_FP32");
      const cublasComputeType_t ct = fp32 && *fp32 == '1' ? CUBLAS_COMPUTE_32F : CUBLAS_COMPUTE_32F_FAST_TF32;
      GemmState::Unit u;
      STC_LT(cublasLtMatmulDescCreate(&u.op, ct, CUDA_R_32F));
      // a plain GEMM: no epilogue and no bias pointer, set explicitly (the
      // fp32 SIMT kernels cuBLASLt picks carry a bias/relu epilogue variant;
      // under compute-sanitizer memcheck they read the bias pointer)
      {
        const cublasLtEpilogue_t epi = CUBLASLT_EPILOGUE_DEFAULT;
        const void* no_bias = nullptr;
        STC_LT(cublasLtMatmulDescSetAttribute(u.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)));
        STC_LT(cublasLtMatmulDescSetAttribute(u.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &no_bias, sizeof(no_bias)));
      }
      const uint64_t M = static_cast<uint64_t>(k.gemm_m), N = static_cast<uint64_t>(k.gemm_n),
                     K = static_cast<uint64_t>(k.gemm_k);
      STC_LT(cublasLtMatrixLayoutCreate(&u.b, CUDA_R_32F, N, K, static_cast<int64_t>(N)));
      STC_LT(cublasLtMatrixLayoutCreate(&u.a, CUDA_R_32F, K, M, static_cast<int64_t>(K)));
      STC_LT(cublasLtMatrixLayoutCreate(&u.c, CUDA_R_32F, N, M, static_cast<int64_t>(N)));
      cublasLtMatmulPreference_t pref = nullptr;
      STC_LT(cublasLtMatmulPreferenceCreate(&pref));
      STC_LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &gemm_->ws_bytes,
                                                  sizeof(gemm_->ws_bytes)));
      // STITCH_GEMM_TUNE=n > 1: the heuristic's top n candidates are timed
      // once on scratch operands of this shape (best of 3 after a warm-up)
      // and the fastest kept.  Default 1, the heuristic's first choice: on
      // the BERT layer tuning over 8 candidates changed nothing (94.7 vs
      // 94.8 us) and over 16 picked a slower one in the graph (98.6 us;
      // profiles/r02/gemm/gemm_tune.jsonl)
      const char* tv = std::getenv("STITCH_GEMM_TUNE");
      const int want = std::clamp(tv && *tv ? std::atoi(tv) : 1, 1, 32);
      std::vector<cublasLtMatmulHeuristicResult_t> res(static_cast<size_t>(want));
      int found = 0;
      const cublasStatus_t hs =
          cublasLtMatmulAlgoGetHeuristic(gemm_->lt, u.op, u.b, u.a, u.c, u.c, pref, want, res.data(), &found);
      cublasLtMatmulPreferenceDestroy(pref);
      if (hs != CUBLAS_STATUS_SUCCESS || found < 1)
        throw std::runtime_error("[cublasLt] no algorithm for GEMM " + k.name);
      int best = 0;
      if (found > 1) {
        void *da = nullptr, *db = nullptr, *dc = nullptr;
        STC_RT(cudaMalloc(&da, M * K * sizeof(float)));
        STC_RT(cudaMalloc(&db, K * N * sizeof(float)));
        STC_RT(cudaMalloc(&dc, M * N * sizeof(float)));
        STC_RT(cudaMemset(da, 0x3c, M * K * sizeof(float)));
        STC_RT(cudaMemset(db, 0x3c, K * N * sizeof(float)));
        cudaEvent_t e0, e1;
        STC_RT(cudaEventCreate(&e0));
        STC_RT(cudaEventCreate(&e1));
        const float alpha = 1.f, beta = 0.f;
        float best_ms = 0.f;
        for (int c = 0; c < found; ++c) {
          float t = -1.f;
          for (int rep = 0; rep < 4; ++rep) {
            STC_RT(cudaEventRecord(e0, stream_));
            if (cublasLtMatmul(gemm_->lt, u.op, &alpha, db, u.b, da, u.a, &beta, dc, u.c, dc, u.c, &res[c].algo,
                               gemm_->workspace, gemm_->ws_bytes, stream_) != CUBLAS_STATUS_SUCCESS) {
              t = -1.f;
              break;
            }
            STC_RT(cudaEventRecord(e1, stream_));
            STC_RT(cudaEventSynchronize(e1));
            float ms = 0.f;
            STC_RT(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0 && (t < 0.f || ms < t)) t = ms;
          }
          if (t > 0.f && (best_ms == 0.f || t < best_ms)) best_ms = t, best = c;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(da);
        cudaFree(db);
        cudaFree(dc);
      }
      u.algo = res[static_cast<size_t>(best)].algo;
      // CUTLASS tcgen05 TF32 configuration (csrc/kernels/gemm_sm100.cu):
      // STITCH_GEMM_FUSED for the GEMM + bias + GELU units (default 0, the
      // 2-SM 256x256 kernel), STITCH_GEMM_PLAIN for the plain GEMMs;
      // STITCH_GEMM_SK=1 = stream-K (variant 1) for both.  Plain default:
      // the 2-SM 256x192 kernel where its tiles fill the SM pairs' waves
      // clearly better than 256x256 tiles would (BERT's ffn2, N = 768: 64
      // tiles for 74 pairs instead of 48; 35.8 vs cuBLASLt's 39.9 us), else
      // cuBLASLt.  Stream-K and the 1-SM 128x192 kernel measured slower
      // (profiles/r02/gemm/streamk.jsonl, gemm_variants.jsonl)
      const bool fused = k.gemm_epilogue == "bias_gelu";
      auto env_variant = [](const char* name, int dflt) {
        const char* v = std::getenv(name);
        return v && *v ? std::atoi(v) : dflt;
      };
      auto wave_fill = [&](int64_t tm, int64_t tn) {
        const int64_t tiles = ((static_cast<int64_t>(M) + tm - 1) / tm) * ((static_cast<int64_t>(N) + tn - 1) / tn);
        const int64_t pairs = std::max(1, dev_->sm_count / 2), waves = (tiles + pairs - 1) / pairs;
        return static_cast<double>(tiles) / static_cast<double>(waves * pairs);
      };
      const int plain_default = N % 192 == 0 && M % 256 == 0 && wave_fill(256, 192) > wave_fill(256, 256) + 0.05 ? 3 : -1;
      const bool sk = env_variant("STITCH_GEMM_SK", 0) == 1;
      int variant = fused ? env_variant("STITCH_GEMM_FUSED", sk ? 1 : 0)
                          : env_variant("STITCH_GEMM_PLAIN", sk ? 1 : plain_default);
      if (ct == CUBLAS_COMPUTE_32F && !fused) variant = -1;
      if (variant > 5) variant = fused ? 0 : -1;  // 6 / 7 take B column-major: layout probe only
      long long ws = variant >= 0 ? gemm_tf32_workspace(variant, fused, static_cast<int>(M), static_cast<int>(N),
                                                        static_cast<int>(K))
                                  : -1;
      if (fused && ws < 0) {  // an unimplementable choice: the default fused kernel (the plan matched it)
        variant = 0;
        ws = gemm_tf32_workspace(0, true, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K));
      }
      if (ws < 0) variant = -1;
      u.variant = variant;
      if (variant >= 0) {
        static const char* kDesc[] = {"", " stream-k", " 1sm 128x192", " 2sm 256x192", " 2x2 256x256", " 2x2 256x192"};
        specs_[ki].scratch_bytes = std::max<long long>(ws, 256);
        specs_[ki].scratch_header = 0;
        specs_[ki].tmpl = std::string("gemm(cutlass tcgen05 tf32") + kDesc[variant] + ")" + (fused ? "+bias+gelu" : "");
      }
      gemm_->units[ki] = u;
      fns_.push_back(nullptr);
      continue;
    }
    cudaKernel_t f = module_->fn(k.symbol.empty() ? k.name : k.symbol);
    const void* fp = reinterpret_cast<const void*>(f);
    // opt in whenever there is dynamic shared memory: static + dynamic above
    // 48 KB needs it even when the dynamic part alone is below (TMA-staged
    // rows with their row-invariant operands hoisted into static smem)
    if (k.smem > 0)
      STC_RT(cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(k.smem)));
    if (k.cluster > 8) STC_RT(cudaFuncSetAttribute(fp, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (k.cooperative) {
      int per_sm = 0;
      STC_RT(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fp, k.block, static_cast<size_t>(k.smem)));
      if (int64_t(per_sm) * dev_->sm_count < k.grid)
        throw std::runtime_error("[cuda] cooperative kernel " + k.name + " needs " + std::to_string(k.grid) +
                                 " co-resident CTAs, device fits " + std::to_string(per_sm * dev_->sm_count));
    }
    fns_.push_back(f);
  }
  compute_deps();
}

void Executor::compute_deps() {
  std::map<std::string, int> producer;
  deps_.assign(specs_.size(), {});
  for (size_t i = 0; i < specs_.size(); ++i) {
    std::set<int> d;
    for (const auto& t : specs_[i].inputs)
      if (auto it = producer.find(t); it != producer.end()) d.insert(it->second);
    deps_[i].assign(d.begin(), d.end());
    for (const auto& t : specs_[i].outputs) producer[t] = static_cast<int>(i);
  }
}

int Executor::capture_plan(int set, cudaStream_t origin, int prev) {
  const size_t n = specs_.size();
  if (!dag_ || n <= 1) {
    for (size_t i = 0; i < n; ++i) launch_kernel(i, set, origin, i ? static_cast<int>(i) - 1 : prev);
    return n ? static_cast<int>(n) - 1 : prev;
  }
  // list scheduling in launch (topological) order: a kernel joins the stream
  // whose tail is its latest producer, else a stream whose tail it already
  // depends on transitively, else a fresh fork of `origin`
  if (kernel_events_.size() < n) {
    for (size_t i = kernel_events_.size(); i < n; ++i) {
      cudaEvent_t e = nullptr;
      STC_RT(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      kernel_events_.push_back(e);
    }
  }
  if (!fork_event_) STC_RT(cudaEventCreateWithFlags(&fork_event_, cudaEventDisableTiming));
  std::vector<std::vector<char>> anc(n, std::vector<char>(n, 0));  // anc[i][j]: j precedes i
  for (size_t i = 0; i < n; ++i)
    for (int d : deps_[i]) {
      anc[i][static_cast<size_t>(d)] = 1;
      for (size_t j = 0; j < n; ++j) anc[i][j] |= anc[static_cast<size_t>(d)][j];
    }
  struct Lane {
    cudaStream_t s;
    int tail;  // kernel of this replay last launched on the lane (-1: none yet)
  };
  std::vector<Lane> lanes{{origin, -1}};
  STC_RT(cudaEventRecord(fork_event_, origin));
  const size_t max_lanes = 8;
  // estimated finish time of every kernel (fixed launch/latency cost + its
  // bytes at HBM speed, after its latest producer): a kernel follows the
  // producer expected to finish LAST on that producer's lane, so the edge
  // that gates it is a same-stream PDL edge (cross-lane edges pay a full
  // launch latency, profiles/r01/dien_timeline.txt)
  std::vector<double> fin(n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    double ready = 0.0;
    for (int d : deps_[i]) ready = std::max(ready, fin[static_cast<size_t>(d)]);
    fin[i] = ready + 1.5 + static_cast<double>(specs_[i].alg_bytes) / 5.0e3;
  }
  // producer-less kernels (per-step input transforms such as DIEN's x.W
  // placeholders) share one dedicated lane: they run ahead of the critical
  // chain instead of taking its slots once the lane cap is reached
  // and are captured first, so the graph launches them ahead of the chain
  // The rest is captured in priority-list order (longest remaining path
  // first among the ready kernels), so the kernel that gates the critical
  // path claims its producer's lane (a same-stream PDL edge) before its
  // siblings fork.
  int source_lane = -1;
  // STITCH_SOURCE_LANE=0: producer-less kernels stay on the origin lane
  // (captured first), so no consumer needs a cross-lane edge to them
  const char* sl_env = std::getenv("STITCH_SOURCE_LANE");
  const bool source_fork = !(sl_env && *sl_env == '0');
  std::vector<size_t> order;
  for (size_t i = 0; i < n; ++i)
    if (deps_[i].empty()) order.push_back(i);
  {
    std::vector<std::vector<int>> users(n);
    for (size_t i = 0; i < n; ++i)
      for (int d : deps_[i]) users[static_cast<size_t>(d)].push_back(static_cast<int>(i));
    std::vector<double> bottom(n, 0.0);  // cost of i + the longest path after it
    for (size_t i = n; i-- > 0;) {
      double tail = 0.0;
      for (int u : users[i]) tail = std::max(tail, bottom[static_cast<size_t>(u)]);
      bottom[i] = 1.5 + static_cast<double>(specs_[i].alg_bytes) / 5.0e3 + tail;
    }
    std::vector<size_t> pending(n);
    std::set<std::pair<double, size_t>> ready;  // (-bottom, index)
    for (size_t i = 0; i < n; ++i) pending[i] = deps_[i].size();
    for (size_t i = 0; i < n; ++i)
      if (deps_[i].empty())
        for (int u : users[i])
          if (--pending[static_cast<size_t>(u)] == 0) ready.insert({-bottom[static_cast<size_t>(u)], static_cast<size_t>(u)});
    while (!ready.empty()) {
      const size_t i = ready.begin()->second;
      ready.erase(ready.begin());
      order.push_back(i);
      for (int u : users[i])
        if (--pending[static_cast<size_t>(u)] == 0) ready.insert({-bottom[static_cast<size_t>(u)], static_cast<size_t>(u)});
    }
    if (order.size() != n) throw std::runtime_error("[exec] kernel dependency cycle");
  }
  for (size_t i : order) {
    int best = -1;
    if (deps_[i].empty() && source_lane >= 0) best = source_lane;
    if (deps_[i].empty() && !source_fork) best = 0;
    for (size_t l = 0; l < lanes.size() && !(deps_[i].empty() && source_lane >= 0); ++l) {  // the producer
      const int t = lanes[l].tail;                                                        // finishing last
      if (t >= 0 && std::count(deps_[i].begin(), deps_[i].end(), t) &&
          (best < 0 || fin[static_cast<size_t>(t)] > fin[static_cast<size_t>(lanes[static_cast<size_t>(best)].tail)]))
        best = static_cast<int>(l);
    }
    for (size_t l = 0; l < lanes.size() && best < 0; ++l) {  // a lane already ordered before us
      const int t = lanes[l].tail;
      if (t < 0 || anc[i][static_cast<size_t>(t)]) best = static_cast<int>(l);
    }
    // STITCH_DAG=2: only kernels without producers (e.g. per-step input
    // transforms) fork; everything else stays on the origin chain
    if (best < 0 && sources_only_ && !deps_[i].empty()) best = 0;
    if (best < 0 && lanes.size() < max_lanes) {
      while (aux_streams_.size() < lanes.size()) {
        cudaStream_t s2 = nullptr;
        STC_RT(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        aux_streams_.push_back(s2);
      }
      cudaStream_t s2 = aux_streams_[lanes.size() - 1];
      STC_RT(cudaStreamWaitEvent(s2, fork_event_, 0));
      lanes.push_back({s2, -1});
      best = static_cast<int>(lanes.size()) - 1;
    }
    if (best < 0) best = 0;  // lane cap reached: serialise on origin
    if (deps_[i].empty() && source_lane < 0 && best > 0) source_lane = best;
    Lane& ln = lanes[static_cast<size_t>(best)];
    for (int d : deps_[i]) {  // producers not already ordered before the lane's tail
      if (ln.tail >= 0 && (d == ln.tail || anc[static_cast<size_t>(ln.tail)][static_cast<size_t>(d)])) continue;
      STC_RT(cudaStreamWaitEvent(ln.s, kernel_events_[static_cast<size_t>(d)], 0));
    }
    // launched with the PDL attribute whenever it has a kernel predecessor:
    // stream capture then makes every incoming kernel edge programmatic,
    // including the cross-lane ones from event waits
    const int after = ln.tail >= 0 ? ln.tail : !deps_[i].empty() ? deps_[i].front() : (best == 0 ? prev : -1);
    if (const char* dbg = std::getenv("STITCH_LANES"); dbg && *dbg == '1') {  // diagnostics: lane map
      std::fprintf(stderr, "[lanes] %-22s lane %d after %s waits", specs_[i].name.c_str(), best,
                   ln.tail >= 0 ? specs_[static_cast<size_t>(ln.tail)].name.c_str() : "-");
      for (int d : deps_[i])
        if (!(ln.tail >= 0 && (d == ln.tail || anc[static_cast<size_t>(ln.tail)][static_cast<size_t>(d)])))
          std::fprintf(stderr, " %s", specs_[static_cast<size_t>(d)].name.c_str());
      std::fprintf(stderr, "\n");
    }
    launch_kernel(i, set, ln.s, after);
    STC_RT(cudaEventRecord(kernel_events_[i], ln.s));
    ln.tail = static_cast<int>(i);
  }
  for (size_t l = 1; l < lanes.size(); ++l)  // join every fork back into origin
    STC_RT(cudaStreamWaitEvent(origin, kernel_events_[static_cast<size_t>(lanes[l].tail)], 0));
  return lanes.size() > 1 ? -1 : lanes[0].tail;  // after a join, no PDL edge into the next replay
}

Executor::~Executor() {
  if (dev_) cudaSetDevice(dev_->ordinal);
  for (auto ge : graphs_)
    if (ge) cudaGraphExecDestroy(ge);
  for (auto ge : batch_graphs_) cudaGraphExecDestroy(ge);
  for (auto& [n, t] : tensors_)
    for (void* p : t.dptr) cudaFree(p);
  for (auto& set : scratch_)
    for (void* p : set)
      if (p) cudaFree(p);
  for (auto e : kernel_events_) cudaEventDestroy(e);
  if (fork_event_) cudaEventDestroy(fork_event_);
  for (auto s : aux_streams_) cudaStreamDestroy(s);
  for (auto* v : {&ev_in_, &ev_comp_, &ev_out_})
    for (auto e : *v) cudaEventDestroy(e);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
  if (stream_) cudaStreamDestroy(stream_);
}

PlanKernels generate_plan_kernels(const CompGraph& g_, const FusionPlan& plan,
                                  const std::map<std::string, KernelPlan>& kernels,
                                  const MachineModel& model, ExecMode mode, int sm_count, bool gemm_opaque) {
  PlanKernels out;
  auto& specs_ = out.specs;
  auto& params_ = out.params;
  const auto order = topo_sort(g_);
  std::vector<int> pos(g_.nodes.size());
  for (size_t i = 0; i < order.size(); ++i) pos[static_cast<size_t>(order[i])] = static_cast<int>(i);
  std::map<int, const FusionPattern*> fire_at;
  std::set<int> covered;
  if (mode != ExecMode::Unfused)
    for (const auto& p : plan.patterns) {
      int last = p.vertices.front();
      for (int v : p.vertices) {
        covered.insert(v);
        if (pos[v] > pos[last]) last = v;
      }
      fire_at[last] = &p;
    }
  const auto cons = g_.consumer_lists();
  auto need_materialize = [&](int v) {  // constants read as tensors
    if (g_.is_output(v)) return true;
    for (int c : cons[static_cast<size_t>(v)])
      if (classify_op(g_.node(c)) == OpClass::Opaque) return true;
    return false;
  };
  std::map<std::string, KernelPlan> singles;
  int idx = 0;
  // model mode: a GEMM whose output feeds only the plan's bias + GELU(tanh)
  // pattern writes that pattern's output from its epilogue (one CUTLASS
  // tcgen05 kernel instead of cuBLASLt + a stitched kernel; the [M,N] GEMM
  // output never reaches HBM).  STITCH_GEMM_FUSE=0 keeps them separate; full
  // f32 GEMMs (STITCH_GEMM_FP32=1) are never fused (the fused kernel is TF32)
  const char* fz = std::getenv("STITCH_GEMM_FUSE");
  const char* f32 = std::getenv("STITCH_GEMM_FP32");
  const bool fuse_gemm_epilogue_ = !(fz && *fz == '0') && !(f32 && *f32 == '1');
  size_t fused_units_ = 0;
  auto fuse_into_gemm = [&](int G, int bias, int outv, const std::vector<int>& verts) {
    if (g_.is_output(G)) return false;
    const std::set<int> in(verts.begin(), verts.end());
    for (int c : cons[static_cast<size_t>(G)])
      if (!in.count(c)) return false;  // G read outside the pattern: it must exist
    for (int v : verts)
      if (v != outv) {
        if (g_.is_output(v)) return false;
        for (int c : cons[static_cast<size_t>(v)])
          if (!in.count(c)) return false;  // an intermediate leaves the pattern
      }
    for (auto& k : specs_) {
      if (!k.is_gemm || k.outputs.size() != 1 || k.outputs[0] != g_.node(G).name || !k.gemm_epilogue.empty()) continue;
      const OpNode& b = g_.node(bias);
      if (b.shape.dims[0] != k.gemm_n || b.shape.dtype != DType::F32 || g_.node(outv).shape.dtype != DType::F32) return false;
      if (!gemm_bias_gelu_supported(static_cast<int>(k.gemm_m), static_cast<int>(k.gemm_n), static_cast<int>(k.gemm_k),
                                    size_t(32) << 20))
        return false;
      k.gemm_epilogue = "bias_gelu";
      k.tmpl = "gemm(cutlass tcgen05 tf32)+bias+gelu";
      k.pattern_key += "+" + std::to_string(outv);
      k.inputs.push_back(b.name);
      k.outputs = {g_.node(outv).name};
      k.alg_bytes = g_.node(g_.node(G).operands[0]).shape.byte_size() + g_.node(g_.node(G).operands[1]).shape.byte_size() +
                    b.shape.byte_size() + g_.node(outv).shape.byte_size();
      return true;
    }
    return false;
  };
  auto add_pattern = [&](const std::vector<int>& verts, const std::string& key) {
    const std::string name = "k" + std::to_string(idx++) + "_" + sanitize(g_.node(verts.front()).name);
    KernelSpec spec;
    bool done = false;
    if (mode != ExecMode::Program) {
      try {
        spec = generate_pattern_kernel(g_, verts, name, sm_count);
        done = true;
      } catch (const TemplateMismatch&) {
      }
    }
    if (!done) {
      const KernelPlan* kp = nullptr;
      if (auto it = kernels.find(key); it != kernels.end()) kp = &it->second;
      if (!kp) {
        auto it = singles.find(key);
        if (it == singles.end()) {
          FusionPattern p;
          p.vertices = verts;
          p.producer = verts.front();
          auto planned = plan_kernel(p, g_, model);
          if (!planned) throw std::runtime_error("[planner] no feasible kernel for pattern " + key);
          it = singles.emplace(key, std::move(*planned)).first;
        }
        kp = &it->second;
      }
      spec = generate_program_kernel(g_, kp->program, name);
      spec.alg_bytes = algorithmic_bytes(g_, verts);
    }
    spec.pattern_key = key;
    specs_.push_back(std::move(spec));
  };
  // Launch units: planned patterns, uncovered fusable ops (singletons),
  // materialised constants and opaque ops.  The reference fires a pattern at
  // its topologically last member (sim.cpp:478-488), which can run an
  // uncovered op before the pattern producing its operand; we order units by
  // a Kahn sort of the contracted graph with that firing position as the
  // priority, which reproduces the reference order whenever it is valid.
  struct Unit {
    std::vector<int> verts;
    std::string key;
    int fire = 0;
    bool opaque = false;
  };
  std::vector<Unit> units;
  std::vector<int> unit_of(g_.nodes.size(), -1);
  for (int v : order) {
    const OpNode& n = g_.node(v);
    if (n.kind == OpKind::Parameter) {
      params_.push_back(v);
      continue;
    }
    if (covered.count(v)) {
      if (auto it = fire_at.find(v); it != fire_at.end()) {
        units.push_back({it->second->vertices, it->second->key(), pos[v], false});
        for (int m : it->second->vertices) unit_of[static_cast<size_t>(m)] = static_cast<int>(units.size()) - 1;
      }
      continue;
    }
    if (n.kind == OpKind::Constant && !need_materialize(v)) continue;
    units.push_back({{v}, std::to_string(v), pos[v], classify_op(n) == OpClass::Opaque});
    unit_of[static_cast<size_t>(v)] = static_cast<int>(units.size()) - 1;
  }
  std::vector<std::set<int>> deps(units.size());
  std::vector<std::vector<int>> users(units.size());
  for (size_t u = 0; u < units.size(); ++u)
    for (int v : units[u].verts)
      for (int o : g_.node(v).operands) {
        const int w = unit_of[static_cast<size_t>(o)];
        if (w >= 0 && w != static_cast<int>(u) && deps[u].insert(w).second) users[static_cast<size_t>(w)].push_back(static_cast<int>(u));
      }
  std::vector<ResidentUnit> runits;      // spec index -> its vertices (resident template)
  std::map<size_t, int> opaque_vertex;  // spec index -> vertex of a placeholder kernel
  std::map<size_t, std::vector<int>> local_verts;  // spec index -> vertices of a local-template kernel
  std::set<std::pair<int, int>> ready;  // (fire position, unit)
  std::vector<size_t> pending(units.size());
  for (size_t u = 0; u < units.size(); ++u)
    if (!(pending[u] = deps[u].size())) ready.insert({units[u].fire, static_cast<int>(u)});
  while (!ready.empty()) {
    const int u = ready.begin()->second;
    ready.erase(ready.begin());
    const Unit& un = units[static_cast<size_t>(u)];
    int64_t gm = 0, gn = 0, gk = 0;
    if (un.opaque && gemm_opaque && opaque_is_matmul(g_, un.verts[0], &gm, &gn, &gk)) {
      const OpNode& n = g_.node(un.verts[0]);
      KernelSpec k;
      k.name = "k" + std::to_string(idx++) + "_" + sanitize(n.name);
      k.tmpl = "gemm(cublasLt)";
      k.pattern_key = "op:" + n.name;
      k.is_gemm = true;
      k.gemm_m = gm, k.gemm_n = gn, k.gemm_k = gk;
      k.grid = k.block = 0;
      k.inputs = {g_.node(n.operands[0]).name, g_.node(n.operands[1]).name};
      k.outputs = {n.name};
      k.alg_bytes = g_.node(n.operands[0]).shape.byte_size() + g_.node(n.operands[1]).shape.byte_size() +
                    n.shape.byte_size();
      specs_.push_back(std::move(k));
    } else if (un.opaque) {
      specs_.push_back(generate_opaque_kernel(g_, un.verts[0], "k" + std::to_string(idx++) + "_" +
                                                                   sanitize(g_.node(un.verts[0]).name),
                                              sm_count));
      opaque_vertex[specs_.size() - 1] = un.verts[0];
    } else if (int G = -1, bias = -1, outv = -1; gemm_opaque && fuse_gemm_epilogue_ &&
               match_bias_gelu(g_, un.verts, &G, &bias, &outv) && fuse_into_gemm(G, bias, outv, un.verts)) {
      // the GEMM that produced G now writes this pattern's output itself
      ++fused_units_;
    } else {
      add_pattern(un.verts, un.key);
      if (specs_.back().tmpl == "local" || specs_.back().tmpl == "regional") local_verts[specs_.size() - 1] = un.verts;
    }
    runits.push_back({un.verts, un.opaque});
    for (int w : users[static_cast<size_t>(u)])
      if (--pending[static_cast<size_t>(w)] == 0) ready.insert({units[static_cast<size_t>(w)].fire, w});
  }
  if (specs_.size() + fused_units_ != units.size()) throw std::runtime_error("[exec] contracted plan graph has a cycle");
  // Resident template (cg_resident.cpp): a row-shardable launch-bound plan
  // runs as one thread-block cluster, plan-kernel boundaries kept in shared
  // memory.  Default: tried for plans of >= 16 launch units (DIEN: 88 / 178;
  // the fixtures and single-kernel configs keep their launch graph);
  // STITCH_RESIDENT=1 tries every plan, =0 never.  Falls back to the launch
  // graph below when the plan does not fit (reason on stderr with
  // STITCH_RESIDENT_LOG=1).
  const char* rv = std::getenv("STITCH_RESIDENT");
  const bool try_resident = rv && *rv ? *rv == '1' : units.size() >= 16;
  if (try_resident && mode == ExecMode::Stitched && !gemm_opaque) {
    std::string why;
    if (auto rk = generate_resident_kernel(g_, runits, "k" + std::to_string(idx++) + "_resident", &why)) {
      specs_ = {std::move(*rk)};
      opaque_vertex.clear();
      local_verts.clear();
    }
    if (const char* lg = std::getenv("STITCH_RESIDENT_LOG"); lg && *lg == '1')
      std::fprintf(stderr, "[exec] resident template not used: %s\n", why.c_str());
  }
  // Horizontal packing.  Launch units with the same producer kernels are
  // mutually independent; two kinds are packed into one launch each:
  //  * small opaque placeholders (DIEN's three gate GEMMs of a step read only
  //    the previous step's state; its per-step x.W GEMMs only parameters):
  //    one 1024-thread CTA per op (generate_opaque_pack);
  //  * local- and regional-template patterns: the independent template packs
  //    their bodies into disjoint CTA ranges (bodies over the same domain
  //    merge, e.g. DIEN's per-step attention-column squeezes become one row
  //    body with one reduction per step).
  // On a launch-bound chain a set then follows its producer as one same-lane
  // PDL edge instead of fanning out over lanes whose cross-lane edges only
  // resolve at completion (profiles/r01/pdl_edge_probe.jsonl).  The plan
  // (patterns, per-op semantics, outputs) is unchanged;
  // STITCH_OPAQUE_PACK=0 / STITCH_LOCAL_PACK=0 launch one kernel per unit.
  const char* pack_env = std::getenv("STITCH_OPAQUE_PACK");
  const char* lpack_env = std::getenv("STITCH_LOCAL_PACK");
  const bool pack_opaque = !(pack_env && *pack_env == '0');
  const bool pack_local = !(lpack_env && *lpack_env == '0');
  // Packing repeats until nothing changes: once a set of units is one
  // launch, their consumers may share that launch as their only producer
  // (DIEN: the per-step attention-column slices pack first, then the
  // squeezes that read them).
  for (int round = 0; round < 8; ++round) {
  if (!((pack_opaque && !opaque_vertex.empty()) || (pack_local && local_verts.size() > 1))) break;
  {
    std::map<std::string, size_t> prod;
    // (kind, producer set) -> member specs; kind 0 opaque (+ its cluster size:
    // a pack launches one uniform cluster per op), 1 local
    std::map<std::pair<int, std::vector<size_t>>, std::vector<size_t>> groups;
    for (size_t i = 0; i < specs_.size(); ++i) {
      std::set<size_t> d;
      for (const auto& t : specs_[i].inputs)
        if (auto it = prod.find(t); it != prod.end()) d.insert(it->second);
      const std::vector<size_t> dv(d.begin(), d.end());
      if (pack_opaque && opaque_vertex.count(i) && opaque_single(g_, opaque_vertex[i]))
        groups[{-opaque_cluster(g_, opaque_vertex[i]), dv}].push_back(i);
      if (pack_local && local_verts.count(i)) groups[{1, dv}].push_back(i);
      for (const auto& t : specs_[i].outputs) prod[t] = i;
    }
    std::map<size_t, KernelSpec> packs;  // placed at the first member's position
    std::map<size_t, std::vector<size_t>> pack_members;
    std::set<size_t> drop;
    for (auto& [kd, members] : groups)
      for (size_t at = 0; at + 1 < members.size(); at += 32) {  // <= 32 units per pack
        const size_t end = std::min(members.size(), at + 32);
        if (end - at < 2) break;
        if (kd.first <= 0) {
          std::vector<int> verts;
          for (size_t j = at; j < end; ++j) verts.push_back(opaque_vertex[members[j]]);
          packs[members[at]] = generate_opaque_pack(
              g_, verts, "k" + std::to_string(idx++) + "_pack" + std::to_string(verts.size()) + "_" + sanitize(g_.node(verts[0]).name));
        } else {
          std::vector<int> verts;
          std::vector<std::string> outs;
          for (size_t j = at; j < end; ++j) {
            verts.insert(verts.end(), local_verts[members[j]].begin(), local_verts[members[j]].end());
            outs.insert(outs.end(), specs_[members[j]].outputs.begin(), specs_[members[j]].outputs.end());
          }
          std::sort(verts.begin(), verts.end());
          KernelSpec k;
          try {  // pattern_key below lists the packed units
            k = generate_pattern_kernel(g_, verts, "k" + std::to_string(idx++) + "_pack" + std::to_string(end - at) + "_" +
                                                       sanitize(g_.node(verts.front()).name), sm_count);
          } catch (const TemplateMismatch&) {
            continue;
          }
          auto ko = k.outputs;
          std::sort(ko.begin(), ko.end());
          std::sort(outs.begin(), outs.end());
          if (ko != outs) continue;  // not a pure side-by-side packing: keep the units
          k.pattern_key.clear();
          for (size_t j = at; j < end; ++j) k.pattern_key += std::string(j == at ? "" : "+") + specs_[members[j]].pattern_key;
          packs[members[at]] = std::move(k);
        }
        for (size_t j = at; j < end; ++j) drop.insert(members[j]), pack_members[members[at]].push_back(members[j]);
      }
    if (packs.empty()) break;
    std::vector<KernelSpec> kept;
    std::map<size_t, int> next_opaque;
    std::map<size_t, std::vector<int>> next_local;
    for (size_t i = 0; i < specs_.size(); ++i) {
      if (auto it = packs.find(i); it != packs.end()) {
        if (local_verts.count(i)) {  // a local/regional pack may pack again
          std::vector<int> verts;
          for (size_t j : pack_members[i]) verts.insert(verts.end(), local_verts[j].begin(), local_verts[j].end());
          next_local[kept.size()] = verts;
        }
        kept.push_back(std::move(it->second));
      } else if (!drop.count(i)) {
        if (auto o = opaque_vertex.find(i); o != opaque_vertex.end()) next_opaque[kept.size()] = o->second;
        if (auto l = local_verts.find(i); l != local_verts.end()) next_local[kept.size()] = l->second;
        kept.push_back(std::move(specs_[i]));
      }
    }
    specs_ = std::move(kept);
    opaque_vertex = std::move(next_opaque);
    local_verts = std::move(next_local);
  }
  }
  // Launch-bound plans (every unit small, e.g. DIEN): all units inside one
  // cooperative launch (cg_persist.cpp), unit boundaries as L2 completion
  // counters instead of kernel boundaries.  STITCH_PERSIST=1 enables it.
  if (const char* pe = std::getenv("STITCH_PERSIST"); pe && *pe == '1' && mode != ExecMode::Program && specs_.size() > 1) {
    const char* mc = std::getenv("STITCH_PERSIST_MAX_CTAS");
    std::map<std::string, int64_t> sizes;
    for (const auto& n : g_.nodes) sizes[n.name] = n.shape.byte_size();
    if (auto pk = generate_persistent_kernel(specs_, "k" + std::to_string(idx++) + "_persistent",
                                             mc && *mc ? std::atoi(mc) : 32, sizes))
      specs_ = {std::move(*pk)};
  }
  // Units whose code differs only in the tensors they touch (DIEN's per-step
  // kernels) share one function: canonical text = source with the kernel
  // name and its tensor parameters renamed positionally.  Each launch still
  // binds its own tensors.  The module then holds 6 instead of 30 functions
  // for DIEN T=10 and a step's kernels find their code already cached by the
  // previous step's (ncu: no_instruction stalls were ~20% of a tiny kernel's
  // chain; T=10 59.6 -> 58.0 us, profiles/r01/dedup_ab.jsonl).  Off under STITCH_TRACE (the hooks carry the unit index) and
  // with STITCH_DEDUP=0.
  const char* tr_env = std::getenv("STITCH_TRACE");
  const char* dd_env = std::getenv("STITCH_DEDUP");
  if (!(tr_env && *tr_env == '1') && !(dd_env && *dd_env == '0')) {
    std::map<std::string, std::string> owner;  // canonical source -> symbol
    for (auto& k : specs_) {
      if (k.is_gemm || k.source.empty()) continue;
      std::string canon = std::regex_replace(k.source, std::regex("\\b" + regex_escape(k.name) + "\\b"), "KNAME_");
      int pi = 0;
      for (const auto* list : {&k.inputs, &k.outputs})
        for (const auto& t : *list)
          canon = std::regex_replace(canon, std::regex("\\b" + regex_escape(tensor_ident(t)) + "\\b"), "p" + std::to_string(pi++) + "_");
      auto [it, fresh] = owner.emplace(canon, k.name);
      if (!fresh) k.symbol = it->second;
    }
  }
  // timeline hooks (no-ops unless compiled with -DSTITCH_TRACE, Executor::trace)
  for (size_t i = 0; i < specs_.size(); ++i) {
    auto& src = specs_[i].source;
    if (specs_[i].is_gemm || src.empty() || !specs_[i].symbol.empty()) continue;
    const size_t open = src.find("{\n", src.find("__global__"));
    const size_t close = src.rfind("}\n");
    if (open == std::string::npos || close == std::string::npos || close < open) continue;
    src.insert(close, "  STC_TRACE_END(" + std::to_string(i) + ");\n");
    src.insert(open + 2, "  STC_TRACE_BEGIN(" + std::to_string(i) + ");\n");
  }
  std::sort(params_.begin(), params_.end());
  out.source = device_prelude();
  for (const auto& k : specs_)
    if (!k.is_gemm && k.symbol.empty())
      out.source += "\n// ---- " + k.name + " [" + k.tmpl + "] pattern " + k.pattern_key + "\n" + k.source;
  return out;
}

void Executor::plan_launches(const FusionPlan& plan, const std::map<std::string, KernelPlan>& kernels,
                             const MachineModel& model, ExecMode mode, bool gemm_opaque) {
  PlanKernels pk = generate_plan_kernels(g_, plan, kernels, model, mode, dev_->sm_count, gemm_opaque);
  specs_ = std::move(pk.specs);
  params_ = std::move(pk.params);
  source_ = std::move(pk.source);
  // tensors that need device buffers: parameters and every kernel input/output
  auto add_tensor = [&](const std::string& name) {
    if (tensors_.count(name)) return;
    const OpNode& n = g_.node(g_.by_name.at(name));
    Tensor t;
    t.name = name;
    t.vertex = n.id;
    t.dtype = n.shape.dtype;
    t.count = n.shape.element_count();
    t.bytes = static_cast<size_t>(n.shape.byte_size());
    tensors_[name] = std::move(t);
  };
  for (int p : params_) add_tensor(g_.node(p).name);
  for (const auto& k : specs_) {
    for (const auto& t : k.inputs) add_tensor(t);
    for (const auto& t : k.outputs) add_tensor(t);
  }
  for (int o : g_.outputs)
    if (!tensors_.count(g_.node(o).name))
      throw std::runtime_error("[exec] graph output " + g_.node(o).name + " is produced by no kernel");
}

void Executor::ensure_sets(int sets) {
  if (sets <= sets_) return;
  for (auto& [n, t] : tensors_)
    while (static_cast<int>(t.dptr.size()) < sets) {
      void* p = nullptr;
      STC_RT(cudaMalloc(&p, std::max<size_t>(t.bytes, 16)));
      STC_RT(cudaMemsetAsync(p, 0, std::max<size_t>(t.bytes, 16), stream_));
      t.dptr.push_back(p);
    }
  while (static_cast<int>(scratch_.size()) < sets) {
    std::vector<void*> s;
    for (const auto& k : specs_) {
      void* p = nullptr;
      if (k.scratch_bytes > 0) {
        STC_RT(cudaMalloc(&p, static_cast<size_t>(k.scratch_bytes)));
        STC_RT(cudaMemsetAsync(p, 0, static_cast<size_t>(k.scratch_bytes), stream_));
      }
      s.push_back(p);
    }
    scratch_.push_back(std::move(s));
  }
  STC_RT(cudaStreamSynchronize(stream_));
  graphs_.resize(static_cast<size_t>(sets), nullptr);
  sets_ = sets;
}

void Executor::launch_kernel(size_t i, int set, cudaStream_t s, int after, const std::map<std::string, void*>* bind) {
  if (after == -2) after = static_cast<int>(i) - 1;
  const KernelSpec& k = specs_[i];
  std::vector<void*> ptrs;
  auto ptr_of = [&](const std::string& t) {
    if (bind)
      if (auto it = bind->find(t); it != bind->end()) return it->second;
    return tensors_.at(t).dptr[static_cast<size_t>(set)];
  };
  if (k.is_gemm && gemm_->units.at(i).variant >= 0) {
    const bool fused = k.gemm_epilogue == "bias_gelu";
    // STITCH_GEMM_PDL (default 1): the CUTLASS GEMM launches under
    // programmatic dependent launch behind its stream predecessor (its setup
    // -- barrier init, TMEM allocation, descriptor prefetch -- overlaps the
    // producer's drain; its load warps griddepcontrol.wait before reading).
    // BERT layer 81.1 -> 79.1 us (profiles/r02/gemm/gemm_pdl.jsonl)
    const char* gp = std::getenv("STITCH_GEMM_PDL");
    const bool gemm_pdl = !(gp && *gp == '0');
    const bool pdl = gemm_pdl && pdl_ && after >= 0 && !specs_[static_cast<size_t>(after)].cooperative;
    if (const int rc = gemm_tf32_launch(gemm_->units.at(i).variant, fused, pdl, static_cast<const float*>(ptr_of(k.inputs[0])),
                                 static_cast<const float*>(ptr_of(k.inputs[1])),
                                 fused ? static_cast<const float*>(ptr_of(k.inputs[2])) : nullptr,
                                 static_cast<float*>(ptr_of(k.outputs[0])), static_cast<int>(k.gemm_m),
                                 static_cast<int>(k.gemm_n), static_cast<int>(k.gemm_k), scratch_[static_cast<size_t>(set)][i],
                                 static_cast<size_t>(k.scratch_bytes), s))
      throw std::runtime_error("[cutlass] GEMM " + k.name + " failed (" + std::to_string(rc) + ")");
    return;
  }
  if (k.is_gemm) {
    launch_gemm(i, ptr_of(k.inputs[0]), ptr_of(k.inputs[1]), ptr_of(k.outputs[0]), s);
    return;
  }
  for (const auto& t : k.inputs) ptrs.push_back(ptr_of(t));
  for (const auto& t : k.outputs) ptrs.push_back(ptr_of(t));
  void* bar = nullptr;
  void* part = nullptr;
  if (k.scratch_bytes > 0) {
    bar = scratch_[static_cast<size_t>(set)][i];
    part = static_cast<char*>(bar) + k.scratch_header;
    ptrs.push_back(bar);
    ptrs.push_back(part);
  }
  std::vector<void*> args;
  for (auto& p : ptrs) args.push_back(&p);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(k.grid), 1, 1);
  cfg.blockDim = dim3(static_cast<unsigned>(k.block), 1, 1);
  cfg.dynamicSmemBytes = static_cast<size_t>(k.smem);
  cfg.stream = s;
  cudaLaunchAttribute attrs[2]{};
  unsigned na = 0;
  if (k.cooperative && coop_in_graph_) {
    attrs[na].id = cudaLaunchAttributeCooperative;
    attrs[na++].val.cooperative = 1;
  } else if (pdl_ && after >= 0 && !k.cooperative && !specs_[static_cast<size_t>(after)].cooperative) {
    // programmatic dependent launch: kernel i may launch while kernel i-1
    // drains; it griddepcontrol.wait()s before reading i-1's outputs
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (k.cluster > 1) {  // regional-cluster template: one row per cluster
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = static_cast<unsigned>(k.cluster);
    attrs[na].val.clusterDim.y = 1;
    attrs[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = na ? attrs : nullptr;
  cfg.numAttrs = na;
  STC_RT(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(fns_[i]), args.data()));
}

void Executor::launch_gemm(size_t i, void* a, void* b, void* c, cudaStream_t s) {
  const GemmState::Unit& u = gemm_->units.at(i);
  const float alpha = 1.f, beta = 0.f;
  STC_LT(cublasLtMatmul(gemm_->lt, u.op, &alpha, b, u.b, a, u.a, &beta, c, u.c, c, u.c, &u.algo, gemm_->workspace,
                        gemm_->ws_bytes, s));
}

void Executor::build_graph(int set) {
  ensure_ready();
  auto& ge = graphs_[static_cast<size_t>(set)];
  if (ge) return;
  for (int attempt = 0; attempt < 2; ++attempt) {
    cudaGraph_t graph = nullptr;
    STC_RT(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    bool failed = false;
    try {
      capture_plan(set, stream_, -1);
    } catch (const std::exception&) {
      failed = true;
    }
    const cudaError_t end = cudaStreamEndCapture(stream_, &graph);
    if (!failed && end == cudaSuccess) {
      STC_RT(cudaGraphInstantiate(&ge, graph, 0));
      cudaGraphDestroy(graph);
      return;
    }
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    // cooperative attribute not capturable here: plain launches; the grids
    // are sized for co-residency so the grid barrier still holds
    coop_in_graph_ = false;
  }
  throw std::runtime_error("[cuda] stream capture of the plan failed");
}

const Executor::Tensor* Executor::tensor(const std::string& name) const {
  auto it = tensors_.find(name);
  return it == tensors_.end() ? nullptr : &it->second;
}

void Executor::upload(const void* const* in, int set) {
  STC_RT(cudaSetDevice(dev_->ordinal));
  ensure_sets(set + 1);
  for (size_t i = 0; i < params_.size(); ++i) {
    const Tensor& t = tensors_.at(g_.node(params_[i]).name);
    STC_RT(cudaMemcpyAsync(t.dptr[static_cast<size_t>(set)], in[i], t.bytes, cudaMemcpyHostToDevice, stream_));
  }
}

void Executor::download(void* const* out, int set) {
  STC_RT(cudaSetDevice(dev_->ordinal));
  for (size_t i = 0; i < g_.outputs.size(); ++i) {
    const Tensor& t = tensors_.at(g_.node(g_.outputs[i]).name);
    STC_RT(cudaMemcpyAsync(out[i], t.dptr[static_cast<size_t>(set)], t.bytes, cudaMemcpyDeviceToHost, stream_));
  }
}

void Executor::launch(cudaStream_t s, int set) {
  ensure_ready();
  if (!s) s = stream_;
  ensure_sets(set + 1);
  if (!use_graph_) {
    for (size_t i = 0; i < specs_.size(); ++i) launch_kernel(i, set, s);
    return;
  }
  build_graph(set);
  STC_RT(cudaGraphLaunch(graphs_[static_cast<size_t>(set)], s));
}

void Executor::sync() {
  STC_RT(cudaSetDevice(dev_->ordinal));
  STC_RT(cudaStreamSynchronize(stream_));
}

void Executor::run_host(const void* const* in, void* const* out) {
  ensure_ready();
  upload(in, 0);
  launch(stream_, 0);
  download(out, 0);
  sync();
}

bool Executor::run_host_zero_copy(const void* const* in, void* const* out) {
  ensure_ready();
  std::map<std::string, void*> bind;
  auto mapped = [&](const void* h, size_t bytes) -> void* {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
    (void)bytes;
    return a.devicePointer;
  };
  for (size_t i = 0; i < params_.size(); ++i) {
    const Tensor& t = tensors_.at(g_.node(params_[i]).name);
    void* d = mapped(in[i], t.bytes);
    if (!d) return false;
    bind[t.name] = d;
  }
  for (size_t i = 0; i < g_.outputs.size(); ++i) {
    const Tensor& t = tensors_.at(g_.node(g_.outputs[i]).name);
    void* d = mapped(out[i], t.bytes);
    if (!d) return false;
    bind[t.name] = d;
  }
  ensure_sets(1);
  for (size_t i = 0; i < specs_.size(); ++i) launch_kernel(i, 0, stream_, static_cast<int>(i) - 1, &bind);
  STC_RT(cudaStreamSynchronize(stream_));
  return true;
}

void Executor::run_host_chunked(const void* const* in, void* const* out, int nchunks, const int* in_chunked) {
  if (nchunks < 1) throw std::runtime_error("[exec] nchunks must be >= 1");
  run_host_pipeline(std::vector<Executor*>(static_cast<size_t>(nchunks), this), in, out, in_chunked);
}

void Executor::run_host_pipeline(const std::vector<Executor*>& chunk_exec, const void* const* in, void* const* out,
                                 const int* in_chunked) {
  if (chunk_exec.empty()) throw std::runtime_error("[exec] no chunks");
  Executor* lead = chunk_exec[0];
  // every chunk graph is a shard of the same graph: same parameter/output lists
  for (Executor* e : chunk_exec)
    if (e->params_.size() != lead->params_.size() || e->g_.outputs.size() != lead->g_.outputs.size())
      throw std::runtime_error("[exec] pipeline chunks come from different graphs");
  std::map<Executor*, int> uses, seen;
  for (Executor* e : chunk_exec) ++uses[e];
  for (auto& [e, n] : uses) e->ensure_ready();
  for (auto& [e, n] : uses) {
    const int S = std::min(n, 3);
    e->ensure_sets(S);
    if (e->use_graph_)
      for (int s = 0; s < S; ++s) e->build_graph(s);
    for (auto* v : {&e->ev_in_, &e->ev_comp_, &e->ev_out_})
      while (static_cast<int>(v->size()) < S) {
        cudaEvent_t ev = nullptr;
        STC_RT(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        v->push_back(ev);
      }
  }
  if (!lead->h2d_) {
    STC_RT(cudaStreamCreateWithFlags(&lead->h2d_, cudaStreamNonBlocking));
    STC_RT(cudaStreamCreateWithFlags(&lead->d2h_, cudaStreamNonBlocking));
  }
  cudaStream_t h2d = lead->h2d_, d2h = lead->d2h_, comp = lead->stream_;
  // STITCH_CHUNK_TRACE=1: per-chunk timestamps (us since the first H2D) on stderr
  const bool trace = std::getenv("STITCH_CHUNK_TRACE") && *std::getenv("STITCH_CHUNK_TRACE") == '1';
  std::vector<cudaEvent_t> tev;
  auto stamp = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e = nullptr;
    STC_RT(cudaEventCreate(&e));
    STC_RT(cudaEventRecord(e, st));
    tev.push_back(e);
  };
  std::vector<size_t> in_off(lead->params_.size(), 0), out_off(lead->g_.outputs.size(), 0);
  // outputs in pinned, device-mapped host memory: the kernels write each
  // chunk's outputs straight over PCIe (no D2H copy stage); else D2H copies
  std::vector<char*> out_dev(lead->g_.outputs.size(), nullptr);
  // (default when every output buffer is device-mapped: C2 739 -> 714 us, LN
  // 450 -> 418 us, profiles/r01/e2e_paths.jsonl; STITCH_E2E_ZC_OUT=0 disables)
  const char* zc_env = std::getenv("STITCH_E2E_ZC_OUT");
  bool zc_out = !(zc_env && *zc_env == '0');
  for (size_t i = 0; i < out_dev.size() && zc_out; ++i) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, out[i]) != cudaSuccess || a.type != cudaMemoryTypeHost || !a.devicePointer) {
      cudaGetLastError();
      zc_out = false;
    } else {
      out_dev[i] = static_cast<char*>(a.devicePointer);
    }
  }
  // the previous call's work on these streams is complete (we synchronise at
  // the end), so the first use of every (executor, set) needs no ordering
  for (Executor* e : chunk_exec) {
    const int j = seen[e]++;
    const int S = std::min(uses[e], 3);
    const int s = j % S;
    const size_t su = static_cast<size_t>(s);
    if (j >= S) STC_RT(cudaStreamWaitEvent(h2d, e->ev_comp_[su], 0));  // use j-S done reading set s
    stamp(h2d);
    for (size_t i = 0; i < e->params_.size(); ++i) {
      const Tensor& t = e->tensors_.at(e->g_.node(e->params_[i]).name);
      const bool chunked = in_chunked ? in_chunked[i] != 0 : true;
      if (chunked) {
        STC_RT(cudaMemcpyAsync(t.dptr[su], static_cast<const char*>(in[i]) + in_off[i], t.bytes,
                               cudaMemcpyHostToDevice, h2d));
        in_off[i] += t.bytes;
      } else if (j < S) {  // shared input: once per (executor, set)
        STC_RT(cudaMemcpyAsync(t.dptr[su], in[i], t.bytes, cudaMemcpyHostToDevice, h2d));
      }
    }
    STC_RT(cudaEventRecord(e->ev_in_[su], h2d));
    stamp(h2d);
    STC_RT(cudaStreamWaitEvent(comp, e->ev_in_[su], 0));
    if (j >= S) STC_RT(cudaStreamWaitEvent(comp, e->ev_out_[su], 0));  // use j-S outputs drained
    if (zc_out) {
      std::map<std::string, void*> bind;
      for (size_t i = 0; i < e->g_.outputs.size(); ++i) {
        const Tensor& t = e->tensors_.at(e->g_.node(e->g_.outputs[i]).name);
        bind[t.name] = out_dev[i] + out_off[i];
        out_off[i] += t.bytes;
      }
      for (size_t ki = 0; ki < e->specs_.size(); ++ki)
        e->launch_kernel(ki, s, comp, static_cast<int>(ki) - 1, &bind);
      STC_RT(cudaEventRecord(e->ev_comp_[su], comp));
      stamp(comp);
      continue;
    }
    e->launch(comp, s);
    STC_RT(cudaEventRecord(e->ev_comp_[su], comp));
    stamp(comp);
    STC_RT(cudaStreamWaitEvent(d2h, e->ev_comp_[su], 0));
    for (size_t i = 0; i < e->g_.outputs.size(); ++i) {
      const Tensor& t = e->tensors_.at(e->g_.node(e->g_.outputs[i]).name);
      STC_RT(cudaMemcpyAsync(static_cast<char*>(out[i]) + out_off[i], t.dptr[su], t.bytes, cudaMemcpyDeviceToHost,
                             d2h));
      out_off[i] += t.bytes;
    }
    STC_RT(cudaEventRecord(e->ev_out_[su], d2h));
    stamp(d2h);
  }
  STC_RT(cudaStreamSynchronize(d2h));
  STC_RT(cudaStreamSynchronize(comp));
  STC_RT(cudaStreamSynchronize(h2d));
  if (trace) {
    std::ostringstream o;
    o << "[chunk-trace] h2d_start h2d_end comp_end d2h_end (us)";
    for (size_t i = 0; i < tev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      o << (i % 4 ? " " : "\n  ") << static_cast<int>(ms * 1000.f);
    }
    std::fprintf(stderr, "%s\n", o.str().c_str());
    for (auto e : tev) cudaEventDestroy(e);
  }
}

void Executor::prepare_sets(int sets) {
  ensure_ready();
  sets = std::max(1, sets);
  ensure_sets(sets);
  // replicate set-0 inputs so every set computes on the same data
  for (int s = 1; s < sets; ++s)
    for (int p : params_) {
      const Tensor& t = tensors_.at(g_.node(p).name);
      STC_RT(cudaMemcpyAsync(t.dptr[static_cast<size_t>(s)], t.dptr[0], t.bytes, cudaMemcpyDeviceToDevice, stream_));
    }
  for (int s = 0; s < sets; ++s)
    if (use_graph_) build_graph(s);
  STC_RT(cudaStreamSynchronize(stream_));
}

int Executor::prepare_batches(int sets, int batch) {
  ensure_ready();
  batch = std::max(1, batch);
  sets = std::max(batch, (std::max(1, sets) + batch - 1) / batch * batch);
  prepare_sets(sets);
  if (batch_ == batch && static_cast<int>(batch_graphs_.size()) == sets / batch) return sets / batch;
  for (auto ge : batch_graphs_) cudaGraphExecDestroy(ge);
  batch_graphs_.clear();
  for (int b = 0; b < sets / batch; ++b) {
    cudaGraph_t graph = nullptr;
    STC_RT(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    int tail = -1;
    for (int t = 0; t < batch; ++t)  // PDL also across consecutive (independent) steps
      tail = capture_plan(b * batch + t, stream_, tail);
    STC_RT(cudaStreamEndCapture(stream_, &graph));
    cudaGraphExec_t ge = nullptr;
    STC_RT(cudaGraphInstantiate(&ge, graph, 0));
    cudaGraphDestroy(graph);
    batch_graphs_.push_back(ge);
  }
  batch_ = batch;
  return sets / batch;
}

void Executor::launch_batch(cudaStream_t s, int index) {
  ensure_ready();
  if (batch_graphs_.empty()) throw std::runtime_error("[exec] prepare_batches() first");
  STC_RT(cudaGraphLaunch(batch_graphs_[static_cast<size_t>(index) % batch_graphs_.size()], s ? s : stream_));
}

double Executor::time(int iters, int warmup, int sets, std::vector<double>* per_kernel, int batch) {
  ensure_ready();
  sets = std::max(1, sets);
  prepare_sets(sets);
  cudaEvent_t e0, e1;
  STC_RT(cudaEventCreate(&e0));
  STC_RT(cudaEventCreate(&e1));
  if (batch > 1) {
    const int nb = prepare_batches(sets, batch);
    const int launches = std::max(1, iters / batch);
    for (int w = 0; w < std::max(1, warmup / batch); ++w) launch_batch(stream_, w);
    STC_RT(cudaStreamSynchronize(stream_));
    STC_RT(cudaEventRecord(e0, stream_));
    for (int it = 0; it < launches; ++it) launch_batch(stream_, it % nb);
    STC_RT(cudaEventRecord(e1, stream_));
    STC_RT(cudaEventSynchronize(e1));
    float bms = 0.f;
    STC_RT(cudaEventElapsedTime(&bms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (per_kernel) per_kernel->assign(specs_.size(), 0.0);
    return 1000.0 * bms / (static_cast<double>(launches) * batch);
  }
  for (int w = 0; w < warmup; ++w) launch(stream_, w % sets);
  STC_RT(cudaStreamSynchronize(stream_));
  STC_RT(cudaEventRecord(e0, stream_));
  for (int it = 0; it < iters; ++it) launch(stream_, it % sets);
  STC_RT(cudaEventRecord(e1, stream_));
  STC_RT(cudaEventSynchronize(e1));
  float ms = 0.f;
  STC_RT(cudaEventElapsedTime(&ms, e0, e1));
  const double us = 1000.0 * ms / std::max(1, iters);
  if (per_kernel) {
    // per-kernel durations: every kernel bracketed by events, replays rotated
    // over the sets like above (launch gaps excluded, cold inputs kept)
    per_kernel->assign(specs_.size(), 0.0);
    std::vector<cudaEvent_t> ev(specs_.size() + 1);
    for (auto& e : ev) STC_RT(cudaEventCreate(&e));
    for (int it = 0; it < iters; ++it) {
      const int s = it % sets;
      STC_RT(cudaEventRecord(ev[0], stream_));
      for (size_t i = 0; i < specs_.size(); ++i) {
        launch_kernel(i, s, stream_);
        STC_RT(cudaEventRecord(ev[i + 1], stream_));
      }
      STC_RT(cudaEventSynchronize(ev.back()));
      for (size_t i = 0; i < specs_.size(); ++i) {
        float kms = 0.f;
        STC_RT(cudaEventElapsedTime(&kms, ev[i], ev[i + 1]));
        (*per_kernel)[i] += 1000.0 * kms / iters;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return us;
}

double Executor::time_call(int iters, int warmup, int sets, std::vector<double>* per_kernel) {
  ensure_ready();
  sets = std::max(1, sets);
  iters = std::max(1, iters);
  prepare_sets(sets);
  for (int w = 0; w < warmup; ++w) launch(stream_, w % sets);
  STC_RT(cudaStreamSynchronize(stream_));
  // the spin outlasts the host submitting the events and the launch(es)
  // queued behind it (a few us per launch)
  const unsigned long long spin_ns = 30000ull + 5000ull * specs_.size();
  cudaEvent_t e0, e1;
  STC_RT(cudaEventCreate(&e0));
  STC_RT(cudaEventCreate(&e1));
  double total = 0.0;
  for (int it = 0; it < iters; ++it) {
    launch_spin(spin_ns, stream_);
    STC_RT(cudaEventRecord(e0, stream_));
    launch(stream_, it % sets);
    STC_RT(cudaEventRecord(e1, stream_));
    STC_RT(cudaEventSynchronize(e1));
    float ms = 0.f;
    STC_RT(cudaEventElapsedTime(&ms, e0, e1));
    total += 1000.0 * ms;
  }
  if (per_kernel) {
    per_kernel->assign(specs_.size(), 0.0);
    std::vector<cudaEvent_t> ev(specs_.size() + 1);
    for (auto& e : ev) STC_RT(cudaEventCreate(&e));
    for (int it = 0; it < iters; ++it) {
      const int s = it % sets;
      launch_spin(spin_ns, stream_);
      STC_RT(cudaEventRecord(ev[0], stream_));
      for (size_t i = 0; i < specs_.size(); ++i) {
        launch_kernel(i, s, stream_);
        STC_RT(cudaEventRecord(ev[i + 1], stream_));
      }
      STC_RT(cudaEventSynchronize(ev.back()));
      for (size_t i = 0; i < specs_.size(); ++i) {
        float kms = 0.f;
        STC_RT(cudaEventElapsedTime(&kms, ev[i], ev[i + 1]));
        (*per_kernel)[i] += 1000.0 * kms / iters;
      }
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return total / iters;
}

std::vector<std::pair<double, double>> Executor::trace(int set) {
  ensure_ready();
  if (!tracing_) throw std::runtime_error("[exec] trace() needs an executor built with STITCH_TRACE=1");
  size_t bytes = 0;
  void* buf = module_->global("stc_trace_", &bytes);
  if (!buf) throw std::runtime_error("[exec] trace buffer missing from the module");
  // a persistent kernel also stamps each of its units (slots 1..U)
  size_t n = specs_.size();
  if (n == 1 && specs_[0].tmpl.rfind("persistent(", 0) == 0) n = 1 + std::stoul(specs_[0].tmpl.substr(11));
  // ... and a resident kernel each of its steps
  if (std::smatch m; n == 1 && std::regex_search(specs_[0].tmpl, m, std::regex(R"(^resident\(.* (\d+) steps)")))
    n = 1 + std::stoul(m[1].str());
  n *= static_cast<size_t>(std::max(1, trace_ctas_));
  std::vector<unsigned long long> init(2 * n);
  for (size_t i = 0; i < n; ++i) init[2 * i] = ~0ull, init[2 * i + 1] = 0ull;
  ensure_sets(set + 1);
  if (use_graph_) build_graph(set);
  STC_RT(cudaStreamSynchronize(stream_));
  STC_RT(cudaMemcpy(buf, init.data(), init.size() * 8, cudaMemcpyHostToDevice));
  launch(stream_, set);
  STC_RT(cudaStreamSynchronize(stream_));
  std::vector<unsigned long long> t(2 * n);
  STC_RT(cudaMemcpy(t.data(), buf, t.size() * 8, cudaMemcpyDeviceToHost));
  auto gemm = [&](size_t i) { return i < specs_.size() && specs_[i].is_gemm; };
  unsigned long long t0 = ~0ull;
  for (size_t i = 0; i < n; ++i)
    if (!gemm(i)) t0 = std::min(t0, t[2 * i]);
  std::vector<std::pair<double, double>> out(n, {-1.0, -1.0});
  for (size_t i = 0; i < n; ++i)
    if (!gemm(i) && t[2 * i + 1])
      out[i] = {1e-3 * static_cast<double>(t[2 * i] - t0), 1e-3 * static_cast<double>(t[2 * i + 1] - t0)};
  return out;
}

std::string describe_specs(const std::vector<KernelSpec>& specs) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < specs.size(); ++i) {
    const auto& k = specs[i];
    o << (i ? "," : "") << "{\"name\":\"" << k.name << "\",\"symbol\":\"" << (k.symbol.empty() ? k.name : k.symbol)
      << "\",\"template\":\"" << json_escape(k.tmpl)
      << "\",\"pattern\":\"" << k.pattern_key << "\",\"grid\":" << k.grid << ",\"block\":" << k.block
      << ",\"smem\":" << k.smem << ",\"cooperative\":" << (k.cooperative ? "true" : "false")
      << ",\"cluster\":" << k.cluster
      << ",\"bytes\":" << k.alg_bytes;
    if (k.is_gemm) o << ",\"gemm_mnk\":[" << k.gemm_m << "," << k.gemm_n << "," << k.gemm_k << "]";
    o << ",\"inputs\":[";
    for (size_t j = 0; j < k.inputs.size(); ++j) o << (j ? "," : "") << "\"" << k.inputs[j] << "\"";
    o << "],\"outputs\":[";
    for (size_t j = 0; j < k.outputs.size(); ++j) o << (j ? "," : "") << "\"" << k.outputs[j] << "\"";
    o << "]}";
  }
  o << "]";
  return o.str();
}

std::string Executor::describe_json() const { return describe_specs(specs_); }

}  // namespace stitch::gpu
