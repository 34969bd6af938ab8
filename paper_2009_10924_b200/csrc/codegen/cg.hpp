// B200 code generator: fusion pattern (+ its KernelPlan) -> one sm_100a CUDA
// kernel, written as CUDA C++ source for NVRTC.
//
// Templates, chosen per connected component of the pattern:
//   local     no reductions: vectorised (float4) grid-stride elementwise chain,
//             shape ops folded into index math, values kept in registers
//   regional  row reductions over trailing axes: a team of threads owns a row,
//             loads it once into registers, reduces with shuffles (+ smem
//             across warps), and every consumer reads the reduced value from
//             registers — the paper's warp/block composition
//   global    column reductions over leading axes: every CTA folds a row slab
//             of a column strip into f64 partials; the last CTA of the strip
//             to arrive (threadfence + arrival counter) combines all slabs in
//             fixed order and runs the column consumers -- grid-wide
//             stitching without a co-residency requirement or idle waiting
//             (the opaque placeholder keeps a cooperative grid barrier)
//   independent  several components (remote / kernel-packing patterns) in
//             one launch, each on its own CTA range
//   program   anything else: the planner's abstract stitched program
//             translated statement for statement (always applicable)
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "stitch/graph.hpp"
#include "stitch/planner.hpp"
#include "stitch/program.hpp"

namespace stitch::gpu {

struct KernelSpec {
  std::string name;                  // __global__ symbol (unique per launch unit)
  std::string symbol;                // function actually launched when it differs from name:
                                     // units with identical code share one (executor dedup)
  std::string source;                // CUDA C++ (device code only; prelude separate)
  std::string tmpl;                  // local | regional | global | independent | program | opaque
  std::string pattern_key;           // FusionPattern::key() or "op:<name>"
  int grid = 1;
  int block = 256;
  int64_t smem = 0;                  // dynamic shared memory bytes
  bool cooperative = false;          // needs a grid-wide barrier (co-resident launch)
  int cluster = 1;                   // thread-block cluster size (regional-cluster template)
  std::vector<std::string> inputs;   // tensor names bound to the leading pointer params
  std::vector<std::string> outputs;  // then these
  int64_t scratch_bytes = 0;         // trailing (bar_, part_) params when > 0 (zeroed once)
  int64_t scratch_header = 256;      // part_ = scratch + scratch_header
  int64_t alg_bytes = 0;             // algorithmic bytes: unique inputs read once + outputs written once
  // library GEMM launch unit (model mode: an opaque_compute that is a
  // matmul C[M,N] = A[M,K] . B[K,N] runs as cuBLASLt; no generated source)
  bool is_gemm = false;
  int64_t gemm_m = 0, gemm_n = 0, gemm_k = 0;
  // "bias_gelu": the plan's bias + GELU(tanh) pattern on the GEMM output is
  // fused into the GEMM epilogue (model mode, CUTLASS tcgen05 kernel,
  // csrc/kernels/gemm_sm100.cu); inputs = {A, B, bias}, outputs = the
  // pattern's output
  std::string gemm_epilogue;
};

// Thrown when a dataflow template cannot express a component; the caller
// falls back to the program template.
struct TemplateMismatch : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Dataflow templates for a planned pattern. `outputs` = the pattern's
// tensors that leave the kernel (graph outputs or read outside). Throws
// TemplateMismatch if some component fits no template.
KernelSpec generate_pattern_kernel(const CompGraph& g, const std::vector<int>& vertices,
                                   const std::string& name, int sm_count);

// Statement-for-statement translation of an abstract stitched program
// (the reference interpreter's semantics, src/sim.cpp:256-462).  `checked`
// adds the interpreter's fault detection on the GPU: lockstep statement
// execution, (epoch, writer)-tagged shared cells for the happens-before rule,
// global/shared bounds checks; faults land in a trailing `unsigned* fault_`
// scratch word (code, offset) that run_program turns into SimFault.
KernelSpec generate_program_kernel(const CompGraph& g, const StitchedProgram& prog,
                                   const std::string& name, bool checked = false);

// opaque_compute placeholder: mean of all operand elements, broadcast
// (src/sim.cpp:215-226): one CTA for small operands, else a cooperative grid.
KernelSpec generate_opaque_kernel(const CompGraph& g, int vertex, const std::string& name,
                                  int sm_count);

// Several mutually independent small opaque placeholders in one launch, one
// 1024-thread CTA per op (CTA j computes vertices[j]).  Every vertex must be
// small enough for the single-CTA form (opaque_single).
KernelSpec generate_opaque_pack(const CompGraph& g, const std::vector<int>& vertices, const std::string& name);
bool opaque_single(const CompGraph& g, int vertex);
int opaque_cluster(const CompGraph& g, int vertex);  // CTAs (one cluster) per small placeholder

// Persistent template (cg_persist.cpp): the launch units of a launch-bound
// plan inside one cooperative launch of <= max_ctas 1024-thread CTAs, unit
// boundaries as completion counters instead of kernel boundaries.  nullopt
// when some unit does not fit (library GEMM, scratch, dynamic smem,
// clusters, a block size not dividing 1024, barriers in a sub-1024 unit, or
// more than max_ctas CTAs).
std::optional<KernelSpec> generate_persistent_kernel(const std::vector<KernelSpec>& units, const std::string& name,
                                                     int max_ctas, const std::map<std::string, int64_t>& sizes);

// While alive, generate_pattern_kernel emits every pattern for CTAs of
// exactly `block` threads (the resident template's physical CTA): no
// thread-block clusters, no PDL hooks.  TemplateMismatch if a row team needs
// more threads.
struct ForcedBlockScope {
  int old;
  explicit ForcedBlockScope(int block);
  ~ForcedBlockScope();
};

// Resident template (cg_resident.cpp): a launch-bound plan whose tensors
// all share a leading batch axis (every non-opaque op row-local) runs as ONE
// thread-block cluster; CTA r owns batch rows [r*R, (r+1)*R).  Plan kernels
// become phases separated by CTA barriers, their boundary tensors live in
// the CTA's shared memory, and opaque placeholders (means over whole
// operands) combine per-CTA partial sums through distributed shared memory
// behind one cluster barrier.  `units` = the plan's launch units in
// execution order (vertex sets; opaque = a single opaque_compute vertex).
// nullopt when the graph is not row-shardable or does not fit.
struct ResidentUnit {
  std::vector<int> verts;
  bool opaque = false;
};
std::optional<KernelSpec> generate_resident_kernel(const CompGraph& g, const std::vector<ResidentUnit>& units,
                                                   const std::string& name, std::string* why = nullptr);

// device helpers every module includes
const std::string& device_prelude();

// algorithmic bytes of a vertex set
int64_t algorithmic_bytes(const CompGraph& g, const std::vector<int>& vertices);

// Non-parity plan refinement (cg_refine.cpp): greedily
// merge launch units along graph edges while the merge saves HBM bytes or a
// launch and stays plannable + template-expressible.  New patterns' KernelPlans
// are added to `kernels`.
struct RefineStats {
  int merges = 0;
  int64_t bytes_saved = 0;
  int64_t probes = 0;       // feasibility probes (plan_kernel + codegen) spent
  bool budget_hit = false;  // stopped by STITCH_REFINE_MAX_PROBES, not by convergence
};
FusionPlan refine_plan(const CompGraph& g, const FusionPlan& plan, const MachineModel& model,
                       std::map<std::string, KernelPlan>& kernels, RefineStats* stats = nullptr);

// C identifier of a tensor's kernel parameter.  Graph names may contain '.'
// (the reference parser's identifier class, src/parser.cpp:50); names without
// one keep the readable "T_<name>", dotted names become "TX_<escaped>" with
// '_' -> "_U" and '.' -> "_D" -- injective: the prefixes differ, and inside
// the dotted class the escape is reversible.
inline std::string tensor_ident(const std::string& name) {
  if (name.find('.') == std::string::npos) return "T_" + name;
  std::string o = "TX_";
  for (char c : name) o += c == '_' ? std::string("_U") : c == '.' ? std::string("_D") : std::string(1, c);
  return o;
}

// `s` as a literal inside a std::regex (ECMAScript) pattern
inline std::string regex_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (std::string("\\^$.|?*+()[]{}").find(c) != std::string::npos) o += '\\';
    o += c;
  }
  return o;
}

// small formatting helpers shared by the generators
std::string c_float(double v);  // exact float literal of (float)v
const char* c_type(DType d);

}  // namespace stitch::gpu
