// .stitch text form of the abstract stitched program.  Emission is byte
// compatible with /root/reference/proj/src/program.cpp:16-91 (kernel texts are
// compared against the reference in tests/test_plan_parity.py); the reader
// accepts the grammar of docs/formats.md.
#include <sstream>
#include <stdexcept>

#include "stitch/program.hpp"

namespace stitch {

namespace {

std::string guard_suffix(const BExprP& g) { return g ? " if " + to_string(g) : std::string(); }

std::string fconst_text(double v) {
  std::ostringstream s;
  s.precision(17);
  s << v;
  return s.str();
}

std::string stmt_text(const Stmt& s) {
  switch (s.kind) {
    case Stmt::Loop: return "loop " + s.loop_var + " " + to_string(s.idx);
    case Stmt::EndLoop: return "endloop";
    case Stmt::ISet: return "iset " + s.dst + " = " + to_string(s.idx) + guard_suffix(s.guard);
    case Stmt::FConst: return "fconst " + s.dst + " = " + fconst_text(s.cval);
    case Stmt::FMove: return "fmove " + s.dst + " = " + s.srcs[0];
    case Stmt::FOp: {
      std::string t = "fop " + s.op + " " + s.dst + " =";
      for (const auto& a : s.srcs) t += " " + a;
      return t;
    }
    case Stmt::GLoad:
      return "gload " + s.dst + " = " + s.tensor + "[" + to_string(s.idx) + "]" + guard_suffix(s.guard);
    case Stmt::GStore:
      return "gstore " + s.tensor + "[" + to_string(s.idx) + "] = " + s.srcs[0] + guard_suffix(s.guard);
    case Stmt::SLoad:
      return "shared_load " + s.dst + " = shm[" + to_string(s.idx) + "]" + guard_suffix(s.guard);
    case Stmt::SStore:
      return "shared_store shm[" + to_string(s.idx) + "] = " + s.srcs[0] + guard_suffix(s.guard);
    case Stmt::RegSet:
      return "regset " + s.dst + "[" + to_string(s.dst_slot) + "] = " + s.srcs[0] + guard_suffix(s.guard);
    case Stmt::RegRead:
      return "regread " + s.dst + " = " + s.srcs[0] + "[" + to_string(s.src_slot) + "]";
    case Stmt::Shuffle:
      return "shuffle_from_lane0 " + s.dst + " = " + s.srcs[0] + "[" + to_string(s.src_slot) + "]";
    case Stmt::WarpReduce: return "warp_reduce " + s.op + " " + s.dst + " = " + s.srcs[0];
    case Stmt::Accum: return "accum " + s.op + " " + s.dst + " = " + s.srcs[0] + guard_suffix(s.guard);
    case Stmt::Barrier: return "barrier";
    case Stmt::Comment: return "# " + s.text;
  }
  return "";
}

}  // namespace

std::string emit_program_text(const StitchedProgram& p) {
  std::string out = "stitched v1\n";
  out += "launch grid " + std::to_string(p.launch.grid) + " block " + std::to_string(p.launch.block) + "\n";
  out += "shmem " + std::to_string(p.shmem_bytes) + "\n";
  for (const auto& t : p.inputs) out += "in " + t.name + " " + t.shape.str() + "\n";
  for (const auto& t : p.outputs) out += "out " + t.name + " " + t.shape.str() + "\n";
  out += "body\n";
  int depth = 1;
  for (const auto& s : p.stmts) {
    if (s.kind == Stmt::EndLoop) --depth;
    out.append(static_cast<size_t>(2 * depth), ' ');
    out += stmt_text(s);
    out += '\n';
    if (s.kind == Stmt::Loop) ++depth;
  }
  return out;
}

namespace {

struct Toks {
  std::vector<std::string> v;
  int line;
  [[noreturn]] void fail(const std::string& m) const {
    throw std::runtime_error("program line " + std::to_string(line) + ": " + m);
  }
  const std::string& operator[](size_t i) const {
    if (i >= v.size()) fail("missing token");
    return v[i];
  }
  void want(size_t i, const char* t) const {
    if ((*this)[i] != t) fail(std::string("expected '") + t + "', got '" + (*this)[i] + "'");
  }
  BExprP guard_from(size_t i) const {
    if (v.size() <= i) return nullptr;
    if (v[i] != "if") fail("unexpected trailing token: " + v[i]);
    if (v.size() != i + 2) fail("guard must be a single expression token");
    return parse_bexpr(v[i + 1]);
  }
  std::pair<std::string, ExprP> indexed(size_t i) const {
    const std::string& t = (*this)[i];
    const auto lb = t.find('[');
    if (lb == std::string::npos || t.back() != ']') fail("expected name[expr]: " + t);
    return {t.substr(0, lb), parse_expr(t.substr(lb + 1, t.size() - lb - 2))};
  }
};

TensorShape shape_token(const Toks& tk, const std::string& sh) {
  const auto lb = sh.find('[');
  if (lb == std::string::npos) tk.fail("bad shape: " + sh);
  auto dt = dtype_from_name(sh.substr(0, lb));
  if (!dt) tk.fail("bad dtype in shape: " + sh);
  TensorShape s;
  s.dtype = *dt;
  std::stringstream ds(sh.substr(lb + 1, sh.size() - lb - 2));
  for (std::string d; std::getline(ds, d, ',');)
    if (!d.empty()) s.dims.push_back(std::stoll(d));
  return s;
}

}  // namespace

StitchedProgram parse_program_text(const std::string& text) {
  StitchedProgram p;
  std::istringstream in(text);
  std::string line;
  int lineno = 0, depth = 0;
  bool body = false, header = false;
  while (std::getline(in, line)) {
    ++lineno;
    Toks tk{{}, lineno};
    {
      std::istringstream ls(line);
      for (std::string t; ls >> t;) tk.v.push_back(t);
    }
    if (tk.v.empty()) continue;
    const std::string& head = tk.v[0];
    if (head[0] == '#') {
      if (body) {
        Stmt s;
        s.kind = Stmt::Comment;
        const auto hash = line.find('#');
        s.text = line.substr(std::min(line.size(), hash + 2));
        p.stmts.push_back(std::move(s));
      }
      continue;
    }
    if (!body) {
      if (head == "stitched") {
        tk.want(1, "v1");
        header = true;
      } else if (head == "launch") {
        tk.want(1, "grid");
        p.launch.grid = std::stoi(tk[2]);
        tk.want(3, "block");
        p.launch.block = std::stoi(tk[4]);
      } else if (head == "shmem") {
        p.shmem_bytes = std::stoll(tk[1]);
      } else if (head == "in" || head == "out") {
        TensorBinding b{tk[1], shape_token(tk, tk[2])};
        (head == "in" ? p.inputs : p.outputs).push_back(std::move(b));
      } else if (head == "body") {
        body = true;
      } else {
        tk.fail("unexpected header line: " + head);
      }
      continue;
    }
    Stmt s;
    if (head == "loop") {
      s.kind = Stmt::Loop;
      s.loop_var = tk[1];
      s.idx = parse_expr(tk[2]);
      ++depth;
    } else if (head == "endloop") {
      s.kind = Stmt::EndLoop;
      if (--depth < 0) tk.fail("endloop without loop");
    } else if (head == "iset") {
      s.kind = Stmt::ISet;
      s.dst = tk[1];
      tk.want(2, "=");
      s.idx = parse_expr(tk[3]);
      s.guard = tk.guard_from(4);
    } else if (head == "fconst") {
      s.kind = Stmt::FConst;
      s.dst = tk[1];
      tk.want(2, "=");
      s.cval = std::stod(tk[3]);
    } else if (head == "fmove") {
      s.kind = Stmt::FMove;
      s.dst = tk[1];
      tk.want(2, "=");
      s.srcs = {tk[3]};
    } else if (head == "fop") {
      s.kind = Stmt::FOp;
      s.op = tk[1];
      s.dst = tk[2];
      tk.want(3, "=");
      s.srcs.assign(tk.v.begin() + 4, tk.v.end());
      if (s.srcs.empty()) tk.fail("fop needs operands");
    } else if (head == "gload" || head == "shared_load") {
      s.kind = head == "gload" ? Stmt::GLoad : Stmt::SLoad;
      s.dst = tk[1];
      tk.want(2, "=");
      auto [t, e] = tk.indexed(3);
      if (s.kind == Stmt::SLoad && t != "shm") tk.fail("shared_load reads shm[...]");
      s.tensor = s.kind == Stmt::GLoad ? t : "";
      s.idx = e;
      s.guard = tk.guard_from(4);
    } else if (head == "gstore" || head == "shared_store") {
      s.kind = head == "gstore" ? Stmt::GStore : Stmt::SStore;
      auto [t, e] = tk.indexed(1);
      if (s.kind == Stmt::SStore && t != "shm") tk.fail("shared_store writes shm[...]");
      s.tensor = s.kind == Stmt::GStore ? t : "";
      s.idx = e;
      tk.want(2, "=");
      s.srcs = {tk[3]};
      s.guard = tk.guard_from(4);
    } else if (head == "regset") {
      s.kind = Stmt::RegSet;
      auto [r, e] = tk.indexed(1);
      s.dst = r;
      s.dst_slot = e;
      tk.want(2, "=");
      s.srcs = {tk[3]};
      s.guard = tk.guard_from(4);
    } else if (head == "regread" || head == "shuffle_from_lane0") {
      s.kind = head == "regread" ? Stmt::RegRead : Stmt::Shuffle;
      s.dst = tk[1];
      tk.want(2, "=");
      auto [r, e] = tk.indexed(3);
      s.srcs = {r};
      s.src_slot = e;
    } else if (head == "warp_reduce" || head == "accum") {
      s.kind = head == "accum" ? Stmt::Accum : Stmt::WarpReduce;
      s.op = tk[1];
      s.dst = tk[2];
      tk.want(3, "=");
      s.srcs = {tk[4]};
      if (s.kind == Stmt::Accum) s.guard = tk.guard_from(5);
    } else if (head == "barrier") {
      s.kind = Stmt::Barrier;
    } else {
      tk.fail("unknown statement: " + head);
    }
    p.stmts.push_back(std::move(s));
  }
  if (!header) throw std::runtime_error("missing 'stitched v1' header");
  if (depth != 0) throw std::runtime_error("unbalanced loop/endloop");
  return p;
}

}  // namespace stitch
