// "program" template: the planner's abstract stitched program translated
// statement for statement into CUDA.  The statement semantics are those of
// the reference interpreter (/root/reference/proj/src/sim.cpp:256-462):
//   * registers are f64; fop rounds its result to f32; accum does not round
//   * gload / shared_load under a false guard yield 0; stores are masked
//   * shuffle_from_lane0 reads lane 0's register array at the reader's slot
//   * warp_reduce folds all 32 lanes (here: xor butterfly, f64)
//   * shared memory holds f64 cells at 4-byte offsets; barrier = __syncthreads
// The launch shape is the plan's own (grid/block of the KernelPlan), so this
// path executes exactly the kernel the reference planned — it is the
// always-applicable fallback and the STC_EXEC_PROGRAM mode.
#include <cmath>
#include <cstdio>
#include <map>
#include <memory>
#include <set>
#include <sstream>

#include "codegen/cg.hpp"

namespace stitch::gpu {

namespace {

std::string c_double(double v) {
  if (std::isnan(v)) return "__longlong_as_double(0x7ff8000000000000ll)";
  if (std::isinf(v)) return v > 0 ? "__longlong_as_double(0x7ff0000000000000ll)"
                                  : "__longlong_as_double(0xfff0000000000000ll)";
  char b[64];
  std::snprintf(b, sizeof b, "%.17e", v);
  return b;
}

class ProgramTranslator {
 public:
  ProgramTranslator(const CompGraph& g, const StitchedProgram& p, bool checked)
      : g_(g), p_(p), checked_(checked) {}

  KernelSpec run(const std::string& name) {
    scan();
    KernelSpec k;
    k.name = name;
    k.tmpl = "program";
    k.grid = p_.launch.grid;
    k.block = p_.launch.block;
    const int64_t cells = p_.shmem_bytes / 4;
    k.smem = cells * 8 + (checked_ ? cells * 4 : 0);
    std::ostringstream sig;
    sig << "extern \"C\" __global__ void __launch_bounds__(" << p_.launch.block << ") " << name << "(";
    bool first = true;
    for (const auto& b : p_.inputs) {
      sig << (first ? "" : ", ") << "const " << c_type(b.shape.dtype) << "* __restrict__ " << tname(b.name);
      first = false;
      k.inputs.push_back(b.name);
    }
    for (const auto& b : p_.outputs) {
      sig << (first ? "" : ", ") << c_type(b.shape.dtype) << "* __restrict__ " << tname(b.name);
      first = false;
      k.outputs.push_back(b.name);
    }
    if (checked_) {
      sig << (first ? "" : ", ") << "unsigned* __restrict__ fault_";
      k.scratch_bytes = 256;
    }
    sig << ") {\n";
    std::ostringstream body;
    body << "  extern __shared__ double shm[];\n";
    if (checked_) {
      // lockstep emulation: every statement is followed by a block barrier,
      // shared cells carry (epoch, writer) tags, program barriers bump the
      // epoch -- the interpreter's happens-before rule (sim.cpp:395-419)
      body << "  int* tag_ = reinterpret_cast<int*>(shm + " << cells << ");\n";
      body << "  for (int c_ = threadIdx.x; c_ < " << cells << "; c_ += blockDim.x) tag_[c_] = -1;\n";
      body << "  int epoch_ = 0;\n  __syncthreads();\n";
    }
    body << "  const i64 bid = blockIdx.x, tid = threadIdx.x, lane = threadIdx.x & 31;\n";
    body << "  const i64 wid = (bid * " << p_.launch.block << " + tid) >> 5;\n";
    body << "  (void)bid; (void)lane; (void)wid; (void)shm;\n";
    body << "  pdl_wait();\n";
    for (const auto& r : iregs_) body << "  i64 " << r << " = 0;\n";
    for (const auto& r : fregs_) body << "  double " << r << " = 0.0;\n";
    for (const auto& [a, w] : arrays_) body << "  double " << a << "[" << w << "] = {};\n";
    int depth = 1;
    for (const auto& s : p_.stmts) {
      if (s.kind == Stmt::EndLoop) --depth;
      body << std::string(static_cast<size_t>(2 * depth), ' ') << stmt(s) << "\n";
      if (checked_ && s.kind != Stmt::Comment && s.kind != Stmt::Loop && s.kind != Stmt::EndLoop &&
          s.kind != Stmt::Barrier)
        body << std::string(static_cast<size_t>(2 * depth), ' ') << "__syncthreads();\n";
      if (s.kind == Stmt::Loop) ++depth;
    }
    body << "}\n";
    k.source = sig.str() + body.str();
    return k;
  }

 private:
  static std::string tname(const std::string& n) { return tensor_ident(n); }

  int64_t count_of(const std::string& tensor) const {
    for (const auto& b : p_.inputs)
      if (b.name == tensor) return b.shape.element_count();
    for (const auto& b : p_.outputs)
      if (b.name == tensor) return b.shape.element_count();
    return 0;
  }

  DType dtype_of(const std::string& tensor) const {
    auto it = g_.by_name.find(tensor);
    return it == g_.by_name.end() ? DType::F32 : g_.node(it->second).shape.dtype;
  }

  void scan() {
    std::map<std::string, int64_t> trips;
    for (const auto& s : p_.stmts)
      if (s.kind == Stmt::Loop) trips[s.loop_var] = s.idx->value;
    for (const auto& s : p_.stmts) {
      switch (s.kind) {
        case Stmt::ISet: iregs_.insert(s.dst); break;
        case Stmt::RegSet: {
          int64_t w = 1;
          if (s.dst_slot->kind == Expr::Const) w = s.dst_slot->value + 1;
          if (s.dst_slot->kind == Expr::Var && trips.count(s.dst_slot->name)) w = trips[s.dst_slot->name];
          arrays_[s.dst] = std::max(arrays_[s.dst], w);
          break;
        }
        case Stmt::Loop: case Stmt::EndLoop: case Stmt::GStore: case Stmt::SStore:
        case Stmt::Barrier: case Stmt::Comment: break;
        default:
          if (!s.dst.empty()) fregs_.insert(s.dst);
      }
    }
    for (const auto& s : p_.stmts)
      if ((s.kind == Stmt::RegRead || s.kind == Stmt::Shuffle) && !arrays_.count(s.srcs[0]))
        arrays_[s.srcs[0]] = 1;
    for (const auto& r : iregs_) fregs_.erase(r);
  }

  std::string ex(const ExprP& e) const {
    switch (e->kind) {
      case Expr::Const: return std::to_string(e->value) + "ll";
      case Expr::Var: return e->name;
      case Expr::Reg:
        // interpreter reads registers as llround(value) (sim.cpp:299-302)
        return iregs_.count(e->name) ? e->name : "((i64)llround(" + e->name + "))";
      case Expr::Min: return "min((i64)" + ex(e->a) + ", (i64)" + ex(e->b) + ")";
      default: break;
    }
    static const char* ops[] = {"", "", "", "+", "-", "*", "/", "%", ""};
    return "(" + ex(e->a) + " " + ops[e->kind] + " " + ex(e->b) + ")";
  }

  std::string gd(const BExprP& g) const {
    if (!g) return "true";
    if (g->kind == BExpr::And) return "(" + gd(g->a) + " && " + gd(g->b) + ")";
    static const char* ops[] = {"<", "<=", "==", "!=", ">=", ">"};
    return "(" + ex(g->lhs) + " " + ops[g->op] + " " + ex(g->rhs) + ")";
  }

  std::string slot_read(const std::string& arr, const std::string& slot) const {
    const int64_t w = arrays_.at(arr);
    return "([&]{ const i64 s_ = " + slot + "; return (s_ >= 0 && s_ < " + std::to_string(w) +
           ") ? " + arr + "[s_] : 0.0; }())";
  }

  std::string fop(const Stmt& s) const {
    const auto& a = s.srcs;
    const std::string& k = s.op;
    std::string v;
    if (k == "add") v = a[0] + " + " + a[1];
    else if (k == "sub") v = a[0] + " - " + a[1];
    else if (k == "mul") v = a[0] + " * " + a[1];
    else if (k == "div") v = a[0] + " / " + a[1];
    else if (k == "max") v = "dmax(" + a[0] + ", " + a[1] + ")";
    else if (k == "min") v = "(" + a[1] + " < " + a[0] + " ? " + a[1] + " : " + a[0] + ")";
    else if (k == "power") v = "pow(" + a[0] + ", " + a[1] + ")";
    else if (k == "exp") v = "exp(" + a[0] + ")";
    else if (k == "tanh") v = "tanh(" + a[0] + ")";
    else if (k == "log") v = "log(" + a[0] + ")";
    else if (k == "rsqrt") v = "1.0 / sqrt(" + a[0] + ")";
    else throw std::runtime_error("[codegen] unknown fop kind: " + k);
    return s.dst + " = (double)(float)(" + v + ");";
  }

  std::string stmt(const Stmt& s) const {
    switch (s.kind) {
      case Stmt::Loop:
        return "for (i64 " + s.loop_var + " = 0; " + s.loop_var + " < " + ex(s.idx) + "; ++" +
               s.loop_var + ") {";
      case Stmt::EndLoop: return "}";
      case Stmt::ISet: return s.dst + " = " + ex(s.idx) + ";";
      case Stmt::FConst: return s.dst + " = " + c_double(s.cval) + ";";
      case Stmt::FMove: return s.dst + " = " + s.srcs[0] + ";";
      case Stmt::FOp: return fop(s);
      case Stmt::GLoad:  // coherent loads: the tensor may come from an earlier kernel (prelude, ldvk)
        if (checked_)
          return "if (" + gd(s.guard) + ") { const i64 i_ = " + ex(s.idx) + "; if (i_ < 0 || i_ >= " +
                 std::to_string(count_of(s.tensor)) + "ll) { sim_fault(fault_, 2, i_); " + s.dst +
                 " = 0.0; } else " + s.dst + " = (double)ldvk(" + tname(s.tensor) + ", i_); } else " + s.dst + " = 0.0;";
        return s.dst + " = " + gd(s.guard) + " ? (double)ldvk(" + tname(s.tensor) + ", " + ex(s.idx) +
               ") : 0.0;";
      case Stmt::GStore: {
        if (checked_)
          return "if (" + gd(s.guard) + ") { const i64 i_ = " + ex(s.idx) + "; if (i_ < 0 || i_ >= " +
                 std::to_string(count_of(s.tensor)) + "ll) sim_fault(fault_, 2, i_); else stv(" + tname(s.tensor) +
                 ", i_, (float)" + s.srcs[0] + "); }";
        const DType d = dtype_of(s.tensor);
        std::string v = "(float)" + s.srcs[0];
        return "if (" + gd(s.guard) + ") stv(" + tname(s.tensor) + ", " + ex(s.idx) + ", " + v + ");" +
               (d == DType::F32 ? "" : "");
      }
      case Stmt::SLoad:
        if (checked_)
          return "if (" + gd(s.guard) + ") { const i64 o_ = " + ex(s.idx) + "; if (o_ < 0 || (o_ & 3) || o_ + 4 > " +
                 std::to_string(p_.shmem_bytes) + "ll) { sim_fault(fault_, 3, o_); " + s.dst + " = 0.0; } else { " +
                 "const int tg_ = tag_[o_ >> 2]; if (tg_ >= 0 && (tg_ >> 11) == epoch_ && (tg_ & 2047) != (int)tid) " +
                 "sim_fault(fault_, 1, o_); " + s.dst + " = shm[o_ >> 2]; } } else " + s.dst + " = 0.0;";
        return s.dst + " = " + gd(s.guard) + " ? shm[(" + ex(s.idx) + ") >> 2] : 0.0;";
      case Stmt::SStore:
        if (checked_)
          return "if (" + gd(s.guard) + ") { const i64 o_ = " + ex(s.idx) + "; if (o_ < 0 || (o_ & 3) || o_ + 4 > " +
                 std::to_string(p_.shmem_bytes) + "ll) sim_fault(fault_, 3, o_); else { shm[o_ >> 2] = " + s.srcs[0] +
                 "; tag_[o_ >> 2] = (epoch_ << 11) | (int)tid; } }";
        return "if (" + gd(s.guard) + ") shm[(" + ex(s.idx) + ") >> 2] = " + s.srcs[0] + ";";
      case Stmt::RegSet: {
        const int64_t w = arrays_.at(s.dst);
        return "if (" + gd(s.guard) + ") { const i64 s_ = " + ex(s.dst_slot) + "; if (s_ >= 0 && s_ < " +
               std::to_string(w) + ") " + s.dst + "[s_] = " + s.srcs[0] + "; }";
      }
      case Stmt::RegRead: return s.dst + " = " + slot_read(s.srcs[0], ex(s.src_slot)) + ";";
      case Stmt::Shuffle: {
        const int64_t w = arrays_.at(s.srcs[0]);
        return "{ const i64 s_ = " + ex(s.src_slot) + "; double v_ = 0.0; for (int q_ = 0; q_ < " +
               std::to_string(w) + "; ++q_) { const double x_ = __shfl_sync(FULL_MASK, " + s.srcs[0] +
               "[q_], 0); if (q_ == s_) v_ = x_; } " + s.dst + " = v_; }";
      }
      case Stmt::WarpReduce:
        if (s.op == "sum")
          return s.dst + " = " + s.srcs[0] + "; for (int o_ = 16; o_ > 0; o_ >>= 1) " + s.dst + " += __shfl_xor_sync(FULL_MASK, " + s.dst + ", o_);";
        return s.dst + " = " + s.srcs[0] + "; for (int o_ = 16; o_ > 0; o_ >>= 1) " + s.dst + " = dmax(" + s.dst + ", __shfl_xor_sync(FULL_MASK, " + s.dst + ", o_));";
      case Stmt::Accum:
        return "if (" + gd(s.guard) + ") " + s.dst + " = " +
               (s.op == "sum" ? s.dst + " + " + s.srcs[0] : "dmax(" + s.dst + ", " + s.srcs[0] + ")") + ";";
      case Stmt::Barrier: return checked_ ? "__syncthreads(); ++epoch_;" : "__syncthreads();";
      case Stmt::Comment: return "// " + s.text;
    }
    return "";
  }

  const CompGraph& g_;
  const StitchedProgram& p_;
  bool checked_ = false;
  std::set<std::string> iregs_, fregs_;
  std::map<std::string, int64_t> arrays_;
};

}  // namespace

namespace {
// Register names derived from graph names (buf_<vertex>) may contain '.'
// (src/parser.cpp:50): rename them to C identifiers before translation.
// Names with a '.' get the prefix "R_" (the planner's own register names are
// t<N> / i<N> / acc<N> / buf_<name> / loop variables, none starting "R_")
// and '_' -> "_U", '.' -> "_D", so the renaming is injective.
std::string reg_ident(const std::string& n) {
  if (n.find('.') == std::string::npos) return n;
  std::string o = "R_";
  for (char c : n) o += c == '_' ? std::string("_U") : c == '.' ? std::string("_D") : std::string(1, c);
  return o;
}

ExprP rename_expr(const ExprP& e) {
  if (!e) return e;
  if ((e->kind == Expr::Var || e->kind == Expr::Reg) && e->name.find('.') == std::string::npos && !e->a && !e->b)
    return e;
  auto c = std::make_shared<Expr>(*e);
  if (c->kind == Expr::Var || c->kind == Expr::Reg) c->name = reg_ident(c->name);
  c->a = rename_expr(e->a);
  c->b = rename_expr(e->b);
  return c;
}

BExprP rename_bexpr(const BExprP& e) {
  if (!e) return e;
  auto c = std::make_shared<BExpr>(*e);
  c->lhs = rename_expr(e->lhs);
  c->rhs = rename_expr(e->rhs);
  c->a = rename_bexpr(e->a);
  c->b = rename_bexpr(e->b);
  return c;
}

bool needs_rename(const StitchedProgram& p) {
  for (const auto& s : p.stmts) {
    if (s.dst.find('.') != std::string::npos || s.loop_var.find('.') != std::string::npos) return true;
    for (const auto& x : s.srcs)
      if (x.find('.') != std::string::npos) return true;
  }
  return false;
}
}  // namespace

KernelSpec generate_program_kernel(const CompGraph& g, const StitchedProgram& prog,
                                   const std::string& name, bool checked) {
  if (!needs_rename(prog)) return ProgramTranslator(g, prog, checked).run(name);
  StitchedProgram p = prog;
  for (auto& s : p.stmts) {
    s.dst = reg_ident(s.dst);
    s.loop_var = reg_ident(s.loop_var);
    for (auto& x : s.srcs) x = reg_ident(x);
    s.dst_slot = rename_expr(s.dst_slot);
    s.src_slot = rename_expr(s.src_slot);
    s.idx = rename_expr(s.idx);
    s.guard = rename_bexpr(s.guard);
  }
  return ProgramTranslator(g, p, checked).run(name);
}

}  // namespace stitch::gpu
