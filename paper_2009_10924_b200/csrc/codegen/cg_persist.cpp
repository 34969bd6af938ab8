// Persistent template for launch-bound plans (DIEN-like chains of small
// kernels): the plan's launch units, already generated as dataflow kernels,
// run inside ONE cooperative launch of P co-resident 1024-thread CTAs.
//
// Why: on a chain of tiny kernels every kernel boundary costs a dependent
// launch -- the consumer's griddepcontrol.wait returns ~0.4 us after the
// producer ends, and the consumer then pays its own load round trip --
// ~2.2-2.8 us per DIEN unit (profiles/r01/dien_timeline.txt).  Inside one
// launch a unit waits only for its producer units' completion counters in
// L2 (one acquire poll by one thread), so a boundary costs a fence + an
// atomic + a poll.
//
// Semantics are the units' own: every unit body is the generated kernel's
// code with its CTA/thread indices virtualised (blockIdx.x -> vb_,
// gridDim.x -> vg_, threadIdx.x -> vt_, blockDim.x -> its block size) and
// its loads switched to the coherent L2 path (tensors written earlier in the
// same launch by other CTAs must not be read through the non-coherent
// caches).  A unit whose block B < 1024 runs 1024/B virtual CTAs side by
// side in one physical CTA, so it must be barrier-free (local template);
// 1024-thread units (opaque placeholders) may use __syncthreads.
//
// Completion counters (scratch, zeroed once): word 0 is the launch
// generation g, word 1+u counts the CTAs that finished unit u (only the
// parts[u] CTAs that own one of its virtual CTAs take part in u).  Counters
// only grow: unit u of launch g is complete when its counter reaches
// parts[u]*(g+1).  The last CTA to finish (word 1+U) bumps g.
#include <cstdlib>
#include <map>
#include <optional>
#include <regex>
#include <set>
#include <sstream>

#include "codegen/cg.hpp"

namespace stitch::gpu {

namespace {

bool has_barrier(const std::string& src) {
  return src.find("__syncthreads") != std::string::npos || src.find("bar.sync") != std::string::npos ||
         src.find("__shared__") != std::string::npos || src.find("grid_sync") != std::string::npos ||
         src.find("cluster_") != std::string::npos;
}

// kernel source -> __device__ function FN(params..., vb_, vg_, vt_) with the
// tensor parameters renamed positionally (p0_, p1_, ...): units whose code
// differs only in the tensors they touch (DIEN's per-step kernels) then
// become textually identical and share one function -- code executed once
// per launch per unit would otherwise be fetched cold every time.
std::string as_unit_function(const KernelSpec& k, const std::string& fn) {
  const std::string& src = k.source;
  const size_t at = src.find(k.name + "(");
  if (src.compare(0, 10, "extern \"C\"") != 0 || at == std::string::npos)
    throw std::invalid_argument("persistent: unexpected kernel header in " + k.name);
  std::string body = "__device__ __noinline__ void " + fn + "(" + src.substr(at + k.name.size() + 1);
  int pi = 0;
  for (const auto* list : {&k.inputs, &k.outputs})
    for (const auto& t : *list)
      body = std::regex_replace(body, std::regex("\\b" + regex_escape(tensor_ident(t)) + "\\b"), "p" + std::to_string(pi++) + "_");
  const size_t close = body.find(") {\n");
  if (close == std::string::npos) throw std::invalid_argument("persistent: no signature end in " + k.name);
  body.insert(close, ", const int vb_, const int vg_, const int vt_");
  static const std::vector<std::pair<std::regex, std::string>> rewrites = {
      {std::regex(R"(\bblockIdx\.x\b)"), "vb_"},
      {std::regex(R"(\bgridDim\.x\b)"), "vg_"},
      {std::regex(R"(\bthreadIdx\.x\b)"), "vt_"},
      {std::regex(R"(__restrict__)"), ""},
      {std::regex(R"(\bld4[ckp]?\()"), "ld4_l2("},
      {std::regex(R"(\bld4hk?\()"), "ld4h_l2("},
      {std::regex(R"(\bldv[kp]?\()"), "ldv_l2("},
      {std::regex(R"(\b__ldg\()"), "__ldcg("},
      {std::regex(R"(\bpdl_(wait|launch)\(\);)"), ""},
  };
  for (const auto& [re, to] : rewrites) body = std::regex_replace(body, re, to);
  body = std::regex_replace(body, std::regex(R"(\bblockDim\.x\b)"), std::to_string(k.block));
  return body;
}

}  // namespace

std::optional<KernelSpec> generate_persistent_kernel(const std::vector<KernelSpec>& units, const std::string& name,
                                                     int max_ctas, const std::map<std::string, int64_t>& sizes) {
  auto tensor_bytes = [&](const std::string& t) {
    auto it = sizes.find(t);
    if (it == sizes.end()) throw std::invalid_argument("persistent: no size for tensor " + t);
    return it->second;
  };
  const char* pf = std::getenv("STITCH_PERSIST_PREFETCH");
  const bool prefetch_params = !(pf && *pf == '0');
  if (units.size() < 2) return std::nullopt;
  int P = 1;
  for (const auto& k : units) {
    if (k.is_gemm || k.scratch_bytes > 0 || k.smem > 0 || k.cluster > 1 || k.cooperative || k.block <= 0 ||
        k.block > 1024 || 1024 % k.block != 0)
      return std::nullopt;
    if (k.block < 1024 && has_barrier(k.source)) return std::nullopt;
    const int per = 1024 / k.block;  // virtual CTAs per physical CTA
    P = std::max(P, (k.grid + per - 1) / per);
  }
  if (P > max_ctas) return std::nullopt;
  // unit dependencies through the tensors they exchange
  std::map<std::string, size_t> prod;
  std::vector<std::set<size_t>> deps(units.size());
  std::vector<std::string> reads, writes;
  std::set<std::string> seen_r, written;
  for (size_t u = 0; u < units.size(); ++u) {
    for (const auto& t : units[u].inputs) {
      if (auto it = prod.find(t); it != prod.end()) deps[u].insert(it->second);
      if (!written.count(t) && seen_r.insert(t).second) reads.push_back(t);
    }
    for (const auto& t : units[u].outputs) {
      if (written.insert(t).second) writes.push_back(t);
      prod[t] = u;
    }
  }
  std::vector<std::string> ins;  // tensors only read (graph parameters / tensors of earlier launches)
  for (const auto& t : reads)
    if (!written.count(t)) ins.push_back(t);
  // parameter types come from the unit signatures ("const T* T_name")
  auto type_of = [&](const std::string& t) {
    for (const auto& k : units) {
      const std::string key = "* __restrict__ " + tensor_ident(t);
      for (size_t at = k.source.find(key); at != std::string::npos; at = k.source.find(key, at + 1)) {
        const char c = at + key.size() < k.source.size() ? k.source[at + key.size()] : ',';
        if (c != ',' && c != ')') continue;  // a longer name with this prefix
        size_t b = k.source.rfind(' ', at - 1);
        std::string ty = k.source.substr(b + 1, at - b - 1);
        if (ty == "float" || ty == "f16_t" || ty == "int" || ty == "unsigned char") return ty;
        if (ty == "char") return std::string("unsigned char");
      }
    }
    throw std::invalid_argument("persistent: no type for tensor " + t);
  };
  KernelSpec k;
  k.name = name;
  k.tmpl = "persistent(" + std::to_string(units.size()) + ")";
  k.grid = P;
  k.block = 1024;
  k.cooperative = true;
  k.inputs = ins;
  k.outputs = writes;
  const int U = static_cast<int>(units.size());
  // bar_ words (generation, U unit counters, final counter) fill the header;
  // part_ (unused) follows it
  k.scratch_header = (4 * (U + 2) + 255) / 256 * 256;
  k.scratch_bytes = k.scratch_header + 8;
  std::ostringstream s;
  std::map<std::string, std::string> fn_of_body;  // canonical body -> function
  std::vector<std::string> fn(units.size());
  for (size_t u = 0; u < units.size(); ++u) {
    const std::string canon = as_unit_function(units[u], "FN_");
    auto it = fn_of_body.find(canon);
    if (it == fn_of_body.end()) {
      it = fn_of_body.emplace(canon, "unit" + std::to_string(fn_of_body.size()) + "_").first;
      s << std::regex_replace(canon, std::regex("\\bFN_\\("), it->second + "(") << "\n";
    }
    fn[u] = it->second;
  }
  s << "extern \"C\" __global__ void __launch_bounds__(1024, 1) " << name << "(";
  bool first = true;
  for (const auto& t : ins) {
    s << (first ? "" : ", ") << "const " << type_of(t) << "* " << tensor_ident(t);
    first = false;
  }
  for (const auto& t : writes) {
    s << (first ? "" : ", ") << type_of(t) << "* " << tensor_ident(t);
    first = false;
  }
  // CTA c takes part in unit u iff it owns one of u's virtual CTAs
  // (c < parts[u]); only those wait for u's producers and count u done, so
  // a unit's completion needs parts[u] increments, not P
  std::vector<int> parts(units.size());
  for (size_t u = 0; u < units.size(); ++u) {
    const int per = 1024 / units[u].block;
    parts[u] = std::min(P, (units[u].grid + per - 1) / per);
  }
  s << ", unsigned* __restrict__ bar_, double* __restrict__ part_) {\n"
    << "  (void)part_;\n"
    << "  __shared__ unsigned gen_;\n"
    << "  if (threadIdx.x == 0) gen_ = *(volatile unsigned*)bar_;\n"
    << "  __syncthreads();\n"
    << "  const unsigned g1 = gen_ + 1u;\n";
  // Graph parameters are never written in the launch: pull every one of
  // them toward L2 up front (one prefetch per 128-byte line, spread over all
  // CTAs) so each unit's parameter reads hit L2 -- the per-kernel graph hides
  // that latency by issuing parameter loads before its PDL wait instead
  if (prefetch_params) {
    const char* tw = std::getenv("STITCH_PERSIST_TOUCH");  // diagnostics: 1 = load (not prefetch), 2 = + outputs
    const int touch = tw && *tw ? std::atoi(tw) : 0;
    std::vector<std::string> warm = ins;
    if (touch >= 2) warm.insert(warm.end(), writes.begin(), writes.end());
    for (const auto& t : warm) {
      const int64_t bytes = tensor_bytes(t);
      s << "  for (i64 o_ = ((i64)blockIdx.x * 1024 + threadIdx.x) * 128; o_ < " << bytes
        << "; o_ += (i64)gridDim.x * 1024 * 128) "
        << (touch ? "touch_l2((const char*)" : "prefetch_l2((const char*)") << tensor_ident(t) << " + o_);\n";
    }
  }
  for (int u = 0; u < U; ++u) {
    const KernelSpec& ku = units[static_cast<size_t>(u)];
    const int per = 1024 / ku.block;
    s << "  // unit " << u << ": " << ku.name << " [" << ku.tmpl << "] grid " << ku.grid << " x " << ku.block << " on "
      << parts[static_cast<size_t>(u)] << " CTA(s)\n"
      << "  if (blockIdx.x < " << parts[static_cast<size_t>(u)] << ") {\n";
    if (!deps[static_cast<size_t>(u)].empty()) {
      s << "    if (threadIdx.x == 0) {\n";
      for (size_t d : deps[static_cast<size_t>(u)])
        s << "      while (ld_acquire_u32(bar_ + " << 1 + d << ") < " << parts[d] << "u * g1) {}\n";
      s << "    }\n    __syncthreads();\n";
    }
    s << "    STC_TRACE_BEGIN(" << 1 + u << ");\n";  // diagnostics (STITCH_TRACE): unit u ready
    s << "    for (int v = blockIdx.x" << (per > 1 ? " * " + std::to_string(per) + " + (int)(threadIdx.x / " +
                                                       std::to_string(ku.block) + ")"
                                                 : "")
      << "; v < " << ku.grid << "; v += " << parts[static_cast<size_t>(u)] * per << ") " << fn[static_cast<size_t>(u)] << "(";
    for (const auto& t : ku.inputs) s << tensor_ident(t) << ", ";
    for (const auto& t : ku.outputs) s << tensor_ident(t) << ", ";
    s << "v, " << ku.grid << ", (int)(threadIdx.x" << (per > 1 ? " % " + std::to_string(ku.block) : "") << "));\n";
    s << "    __syncthreads();\n    STC_TRACE_STAMP_END(" << 1 + u << ");\n    if (threadIdx.x == 0) red_release_add_u32(bar_ + "
      << 1 + u << ", 1u);\n  }\n";
  }
  // the last CTA out bumps the generation for the next launch
  s << "  if (threadIdx.x == 0 && atomicAdd(bar_ + " << 1 + U
    << ", 1u) + 1u == g1 * gridDim.x) { __threadfence(); atomicAdd(bar_, 1u); }\n}\n";
  k.source = s.str();
  for (const auto& u : units) k.alg_bytes += u.alg_bytes;
  return k;
}

}  // namespace stitch::gpu
