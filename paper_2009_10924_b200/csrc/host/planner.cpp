// Code-generation planner: for one fusion pattern, enumerate (grouping x
// launch dims x per-root schedule template), emit the abstract stitched
// program for each candidate, cost it with the analytical latency model and
// keep the argmin.
//
// This is a bit-exact restatement of /root/reference/proj/src/planner.cpp:
// the enumeration order, the emitted statements (register/loop naming, memo
// reuse rules, index materialisation), the liveness/histogram accounting and
// the tie-breaks are the same, because the emitted program's histogram and
// register estimate decide which plan wins.  Line references are to that file.
//
// What differs is speed: the ownership check (planner.cpp:216-254), which
// dominates planning time upstream (gprof: Expr eval + std::map lookups),
// evaluates index expressions compiled to a flat slot program instead of
// walking shared_ptr trees against a std::map environment.  It visits the
// same probe points in the same order, so accept/reject decisions are
// identical.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <limits>
#include <set>
#include <stdexcept>
#include <thread>

#include "stitch/planner.hpp"

namespace stitch {

namespace {

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

std::vector<int> positions_of(const CompGraph& g) {
  std::vector<int> pos(g.nodes.size(), 0);
  int i = 0;
  for (int v : topo_sort(g)) pos[static_cast<size_t>(v)] = i++;
  return pos;
}

// members that are graph outputs or read outside the pattern (planner.cpp:24-33)
std::vector<int> pattern_outputs(const FusionPattern& p, const CompGraph& g) {
  std::set<int> out;
  for (int v : p.vertices)
    if (g.is_output(v)) out.insert(v);
  for (const auto& n : g.nodes) {
    if (p.contains(n.id)) continue;
    for (int o : n.operands)
      if (p.contains(o)) out.insert(o);
  }
  return {out.begin(), out.end()};
}

void vars_in(const ExprP& e, std::set<std::string>& vars, bool& reg) {
  if (!e) return;
  if (e->kind == Expr::Var) vars.insert(e->name);
  if (e->kind == Expr::Reg) reg = true;
  vars_in(e->a, vars, reg);
  vars_in(e->b, vars, reg);
}

void vars_in(const BExprP& e, std::set<std::string>& vars, bool& reg) {
  if (!e) return;
  if (e->kind == BExpr::And) {
    vars_in(e->a, vars, reg);
    vars_in(e->b, vars, reg);
  } else {
    vars_in(e->lhs, vars, reg);
    vars_in(e->rhs, vars, reg);
  }
}

struct Infeasible {
  const char* why;
};

// ---- compiled index expressions for the ownership probe -------------------
// Postfix program over integer slots: 0 bid, 1 tid, 2 lane, 3 wid, 4.. loop vars.
struct SlotProgram {
  enum Op : uint8_t { Push, Load, Add, Sub, Mul, Div, Mod, Min, Lt, Le, Eq, Ne, Ge, Gt, And };
  struct Ins {
    Op op;
    int64_t arg;
  };
  std::vector<Ins> code;
  bool empty() const { return code.empty(); }

  int64_t run(const int64_t* slots) const {
    int64_t st[64];
    int sp = 0;
    for (const Ins& in : code) {
      switch (in.op) {
        case Push: st[sp++] = in.arg; break;
        case Load: st[sp++] = slots[in.arg]; break;
        default: {
          const int64_t b = st[--sp], a = st[sp - 1];
          int64_t r = 0;
          switch (in.op) {
            case Add: r = a + b; break;
            case Sub: r = a - b; break;
            case Mul: r = a * b; break;
            case Div:
              if (!b) throw std::runtime_error("division by zero in index expression");
              r = a / b;
              break;
            case Mod:
              if (!b) throw std::runtime_error("mod by zero in index expression");
              r = a % b;
              break;
            case Min: r = std::min(a, b); break;
            case Lt: r = a < b; break;
            case Le: r = a <= b; break;
            case Eq: r = a == b; break;
            case Ne: r = a != b; break;
            case Ge: r = a >= b; break;
            case Gt: r = a > b; break;
            case And: r = a && b; break;
            default: break;
          }
          st[sp - 1] = r;
        }
      }
    }
    return st[0];
  }
};

class SlotCompiler {
 public:
  explicit SlotCompiler(const std::vector<std::string>& loop_vars) : loops_(loop_vars) {}
  SlotProgram expr(const ExprP& e) {
    SlotProgram p;
    emit(e, p);
    return p;
  }
  SlotProgram guard(const BExprP& g) {
    SlotProgram p;
    if (g) emit(g, p);
    return p;
  }

 private:
  int slot_of(const std::string& n) const {
    if (n == "bid") return 0;
    if (n == "tid") return 1;
    if (n == "lane") return 2;
    if (n == "wid") return 3;
    for (size_t i = 0; i < loops_.size(); ++i)
      if (loops_[i] == n) return 4 + static_cast<int>(i);
    throw std::runtime_error("unbound variable: " + n);
  }
  void emit(const ExprP& e, SlotProgram& p) {
    using O = SlotProgram::Op;
    switch (e->kind) {
      case Expr::Const: p.code.push_back({O::Push, e->value}); return;
      case Expr::Var: p.code.push_back({O::Load, slot_of(e->name)}); return;
      case Expr::Reg: throw std::runtime_error("register reference outside thread context");
      default: break;
    }
    emit(e->a, p);
    emit(e->b, p);
    static const O k[] = {O::Push, O::Push, O::Push, O::Add, O::Sub, O::Mul, O::Div, O::Mod, O::Min};
    p.code.push_back({k[e->kind], 0});
  }
  void emit(const BExprP& g, SlotProgram& p) {
    using O = SlotProgram::Op;
    if (g->kind == BExpr::And) {
      emit(g->a, p);
      emit(g->b, p);
      p.code.push_back({O::And, 0});
      return;
    }
    emit(g->lhs, p);
    emit(g->rhs, p);
    static const O k[] = {O::Lt, O::Le, O::Eq, O::Ne, O::Ge, O::Gt};
    p.code.push_back({k[g->op], 0});
  }
  const std::vector<std::string>& loops_;
};

// ---- the abstract-program builder (planner.cpp:64-794) ---------------------
enum class Owner { Thread, Warp, Block };

class ProgramBuilder {
 public:
  ProgramBuilder(const CompGraph& g, const FusionPattern& p, const Grouping& grouping,
                 const std::map<int, std::string>& tpl, LaunchDims ld, const DeviceSpec& dev,
                 const std::vector<int>& pos)
      : g_(g), p_(p), grouping_(grouping), tpl_(tpl), ld_(ld), dev_(dev), pos_(pos) {
    for (int r : grouping.group_roots()) roots_.insert(r);
    prog.launch = ld;
  }

  StitchedProgram prog;
  AllocationMap alloc;
  std::vector<GroupBoundary> boundaries;

  void build() {  // planner.cpp:760-793
    std::map<int, int64_t> requests;
    bool scratch = false;
    for (int r : grouping_.group_roots()) {
      const ScheduleTemplate& t = template_by_id(tpl_.at(r));
      if (t.output_placement != OutputPlacement::SharedMemory) continue;
      if (classify_op(g_.node(r)) == OpClass::Reduction) scratch = true;
      if (feeds_pattern(r)) {
        const int64_t rl = row_len(r);
        requests[r] = cdiv(g_.node(r).shape.element_count() / rl, ld_.grid) * rl * 4;
      }
    }
    alloc = allocate_shared_memory(p_, requests, g_, &grouping_);
    scratch_at_ = scratch ? alloc.total : -1;
    prog.shmem_bytes = alloc.total + (scratch ? int64_t(ld_.block) * 4 : 0);

    std::vector<int> order = grouping_.group_roots();
    std::sort(order.begin(), order.end(), [&](int a, int b) { return pos_[a] < pos_[b]; });
    for (int r : order) {
      current_ = r;
      const ScheduleTemplate& t = template_by_id(tpl_.at(r));
      comment("group " + g_.node(r).name + " " + t.id);
      if (classify_op(g_.node(r)) == OpClass::Reduction)
        reduction_group(r, t);
      else
        elementwise_group(r, t);
      done_roots_.insert(r);
    }
  }

 private:
  struct Memo {
    std::string reg;
    std::string chain;
  };
  struct Frame {
    std::string var;
    int64_t trip;
  };

  int64_t T() const { return ld_.total_threads(); }
  int64_t W() const { return T() / dev_.warp_size; }
  ExprP global_tid() const { return e_add(e_mul(bid_, e_const(ld_.block)), tid_); }
  std::string fresh(const char* prefix) { return prefix + std::to_string(regs_++); }
  void push(Stmt s) { prog.stmts.push_back(std::move(s)); }
  static Stmt make(Stmt::Kind k) {
    Stmt s;
    s.kind = k;
    return s;
  }
  void barrier() { push(make(Stmt::Barrier)); }
  void comment(std::string text) {
    Stmt s = make(Stmt::Comment);
    s.text = std::move(text);
    push(std::move(s));
  }

  // loops with trip <= 1 vanish; their variable becomes 0 (planner.cpp:133-153)
  std::pair<ExprP, bool> open_loop(int64_t trip) {
    if (trip <= 1) return {e_const(0), false};
    const int id = loops_++;
    Stmt s = make(Stmt::Loop);
    s.loop_var = "j" + std::to_string(id);
    s.idx = e_const(trip);
    frames_.push_back({s.loop_var, trip});
    chain_ += "#" + std::to_string(id);
    ExprP var = e_var(s.loop_var);
    push(std::move(s));
    return {var, true};
  }
  void close_loop(bool real) {
    if (!real) return;
    push(make(Stmt::EndLoop));
    frames_.pop_back();
    chain_.resize(chain_.rfind('#'));
  }

  // prefix of the open-loop chain up to the deepest loop the value depends
  // on; a register reference pins it to the whole chain (planner.cpp:157-178)
  std::string chain_of(const ExprP& e, const BExprP& gd) const {
    std::set<std::string> vars;
    bool reg = false;
    vars_in(e, vars, reg);
    vars_in(gd, vars, reg);
    if (reg) return chain_;
    size_t keep = 0, cut = 0;
    for (size_t i = 0; i < frames_.size(); ++i) {
      cut = chain_.find('#', cut + (i ? 1 : 0));
      const size_t end = chain_.find('#', cut + 1);
      if (vars.count(frames_[i].var)) keep = end == std::string::npos ? chain_.size() : end;
    }
    return chain_.substr(0, keep);
  }

  const Memo* reuse(const std::string& key) const {
    auto it = memo_.find(key);
    if (it == memo_.end() || chain_.compare(0, it->second.chain.size(), it->second.chain) != 0)
      return nullptr;
    return &it->second;
  }

  // div/mod index math is computed once into an index register (planner.cpp:195-209)
  ExprP index_reg(const ExprP& idx) {
    if (idx->kind == Expr::Const || idx->kind == Expr::Var) return idx;
    const std::string text = to_string(idx);
    if (text.find_first_of("/%") == std::string::npos) return idx;
    const std::string key = "I|" + text;
    if (const Memo* m = reuse(key)) return e_reg(m->reg);
    Stmt s = make(Stmt::ISet);
    s.dst = fresh("i");
    s.idx = idx;
    const std::string reg = s.dst;
    push(std::move(s));
    memo_[key] = {reg, chain_of(idx, nullptr)};
    return e_reg(reg);
  }

  // every guarded-live probe point must read an element the producer's
  // mapping placed in the reader's own thread / warp / block (planner.cpp:216-254)
  void check_owner(const ExprP& idx, const BExprP& gd, Owner scope, int64_t rl = 1) {
    if (contains_reg(idx)) throw Infeasible{"data-dependent boundary index"};
    std::vector<std::string> loop_vars;
    std::vector<int64_t> radix = {ld_.grid, ld_.block};
    for (const auto& f : frames_) {
      loop_vars.push_back(f.var);
      radix.push_back(f.trip);
    }
    SlotCompiler comp(loop_vars);
    const SlotProgram pe = comp.expr(idx), pg = comp.guard(gd);
    int64_t total = 1;
    for (int64_t r : radix) total *= r;
    const int64_t cap = int64_t(1) << 14;
    const int64_t stride = total <= cap ? 1 : ((total / cap) | 1);
    std::vector<int64_t> slots(4 + frames_.size());
    const int64_t n_t = T(), n_w = W();
    auto probe = [&](int64_t flat) {
      for (size_t i = radix.size(); i-- > 2;) {
        slots[2 + i] = flat % radix[i];
        flat /= radix[i];
      }
      slots[1] = flat % radix[1];
      flat /= radix[1];
      slots[0] = flat % radix[0];
      slots[2] = slots[1] % dev_.warp_size;
      const int64_t gthread = slots[0] * ld_.block + slots[1];
      slots[3] = gthread / dev_.warp_size;
      if (!pg.empty() && !pg.run(slots.data())) return;
      const int64_t e = pe.run(slots.data());
      bool ok = false;
      switch (scope) {
        case Owner::Thread: ok = e % n_t == gthread; break;
        case Owner::Warp: ok = e % n_w == slots[3]; break;
        case Owner::Block: ok = (e / rl) % ld_.grid == slots[0]; break;
      }
      if (!ok) throw Infeasible{"boundary read escapes producer reuse scope"};
    };
    for (int64_t f = 0; f < total; f += stride) probe(f);
    probe(total - 1);
  }

  void bind(int v) {
    if (bound_.insert(v).second) prog.inputs.push_back({g_.node(v).name, g_.node(v).shape});
  }

  static std::string value_key(int v, const ExprP& idx, const BExprP& gd) {
    return "V|" + std::to_string(v) + "|" + to_string(idx) + "|" + to_string(gd);
  }

  // planner.cpp:261-316
  std::string value(int v, const ExprP& idx, const BExprP& gd) {
    const std::string key = value_key(v, idx, gd);
    if (const Memo* m = reuse(key)) return m->reg;
    const OpNode& n = g_.node(v);
    if (!p_.contains(v)) {
      if (n.kind == OpKind::Constant) {
        Stmt s = make(Stmt::FConst);
        s.dst = fresh("t");
        s.cval = n.attrs.value;
        memo_[key] = {s.dst, ""};
        std::string reg = s.dst;
        push(std::move(s));
        return reg;
      }
      bind(v);
      Stmt s = make(Stmt::GLoad);
      s.dst = fresh("t");
      s.tensor = n.name;
      s.idx = index_reg(idx);
      s.guard = gd;
      std::string reg = s.dst;
      push(std::move(s));
      memo_[key] = {reg, chain_of(idx, gd)};
      return reg;
    }
    if (roots_.count(v) && v != current_) return boundary(v, idx, gd, key);
    switch (classify_op(n)) {
      case OpClass::ShapeOp: return shape_op(v, idx, gd, key);
      case OpClass::LightElementwise:
      case OpClass::ExpensiveElementwise: {
        std::string deepest;
        std::vector<std::string> srcs;
        for (int o : n.operands) {
          srcs.push_back(value(o, idx, gd));
          // operands' chains are prefix-comparable; keep the longest
          auto it = memo_.find(value_key(o, idx, gd));
          if (it != memo_.end() && it->second.chain.size() > deepest.size()) deepest = it->second.chain;
        }
        Stmt s = make(Stmt::FOp);
        s.op = kind_name(n.kind);
        s.dst = fresh("t");
        s.srcs = std::move(srcs);
        std::string reg = s.dst;
        push(std::move(s));
        memo_[key] = {reg, deepest};
        return reg;
      }
      default: throw Infeasible{"non-root reduction/opaque inside a group body"};
    }
  }

  // reductions and expensive ops map one element per row; light/shape roots
  // iterate rows x trailing extent (planner.cpp:320-325)
  int64_t row_len(int v) const {
    const OpClass c = classify_op(g_.node(v));
    if (c == OpClass::Reduction || c == OpClass::ExpensiveElementwise) return 1;
    const auto& s = g_.node(v).shape;
    return s.rank() == 0 ? 1 : s.dims.back();
  }

  // planner.cpp:327-369
  std::string boundary(int v, const ExprP& idx, const BExprP& gd, const std::string& key) {
    if (!done_roots_.count(v)) throw Infeasible{"boundary producer not yet emitted"};
    const ScheduleTemplate& pt = template_by_id(tpl_.at(v));
    if (seen_edges_.insert({v, current_}).second)
      boundaries.push_back({v, current_, pt.id, tpl_.at(current_)});
    const std::string reg = fresh("t");
    const std::string buf = "buf_" + g_.node(v).name;
    Stmt s;
    switch (pt.output_placement) {
      case OutputPlacement::ThreadRegister:
        check_owner(idx, gd, Owner::Thread);
        s = make(Stmt::RegRead);
        s.dst = reg;
        s.srcs = {buf};
        s.src_slot = e_div(idx, e_const(T()));
        break;
      case OutputPlacement::WarpLane0Register:
        check_owner(idx, gd, Owner::Warp);
        s = make(Stmt::Shuffle);
        s.dst = reg;
        s.srcs = {buf};
        s.src_slot = e_div(idx, e_const(W()));
        break;
      case OutputPlacement::SharedMemory: {
        const int64_t rl = row_len(v);
        check_owner(idx, gd, Owner::Block, rl);
        s = make(Stmt::SLoad);
        s.dst = reg;
        const int64_t base = alloc.slots.at(v).offset;
        ExprP slot = rl == 1 ? e_div(idx, e_const(ld_.grid))
                             : e_add(e_mul(e_div(e_div(idx, e_const(rl)), e_const(ld_.grid)),
                                           e_const(rl)),
                                     e_mod(idx, e_const(rl)));
        s.idx = index_reg(e_add(e_const(base), e_mul(slot, e_const(4))));
        s.guard = gd;
        break;
      }
      case OutputPlacement::GlobalMemory: throw Infeasible{"global boundary placement unused"};
    }
    push(std::move(s));
    memo_[key] = {reg, chain_of(idx, gd)};
    return reg;
  }

  // broadcast / transpose / slice rewrite the index; gather loads through an
  // index tensor (planner.cpp:371-436)
  std::string shape_op(int v, const ExprP& idx, const BExprP& gd, const std::string& key) {
    const OpNode& n = g_.node(v);
    const TensorShape& out = n.shape;
    const auto ostr = out.strides();
    auto coord = [&](size_t axis) {
      return e_mod(e_div(idx, e_const(ostr[axis])), e_const(out.dims[axis]));
    };
    auto forward = [&](const ExprP& src_idx) {
      const int src = n.operands[0];
      std::string reg = value(src, src_idx, gd);
      memo_[key] = memo_.at(value_key(src, src_idx, gd));
      return reg;
    };
    switch (n.kind) {
      case OpKind::Broadcast: {
        const auto istr = g_.node(n.operands[0]).shape.strides();
        ExprP e = e_const(0);
        for (size_t i = 0; i < istr.size(); ++i)
          e = e_add(e, e_mul(coord(static_cast<size_t>(n.attrs.dims[i])), e_const(istr[i])));
        return forward(e);
      }
      case OpKind::Transpose: {
        const auto istr = g_.node(n.operands[0]).shape.strides();
        ExprP e = e_const(0);
        for (size_t j = 0; j < out.dims.size(); ++j)
          e = e_add(e, e_mul(coord(j), e_const(istr[static_cast<size_t>(n.attrs.perm[j])])));
        return forward(e);
      }
      case OpKind::Slice: {
        const auto istr = g_.node(n.operands[0]).shape.strides();
        ExprP e = e_const(0);
        for (size_t j = 0; j < out.dims.size(); ++j)
          e = e_add(e, e_mul(e_add(coord(j), e_const(n.attrs.starts[j])), e_const(istr[j])));
        return forward(e);
      }
      case OpKind::Gather: {
        const int data = n.operands[0], indices = n.operands[1];
        if (p_.contains(data)) throw Infeasible{"gather data produced inside the pattern"};
        const TensorShape& ds = g_.node(data).shape;
        const int64_t inner = ds.element_count() / ds.dims[0];
        const std::string row_reg = value(indices, e_div(idx, e_const(inner)), gd);
        ExprP e = e_add(e_mul(e_reg(row_reg), e_const(inner)), e_mod(idx, e_const(inner)));
        bind(data);
        Stmt s = make(Stmt::GLoad);
        s.dst = fresh("t");
        s.tensor = g_.node(data).name;
        s.idx = index_reg(e);
        s.guard = gd;
        std::string reg = s.dst;
        push(std::move(s));
        memo_[key] = {reg, chain_};
        return reg;
      }
      default: throw Infeasible{"unexpected shape op in group body"};
    }
  }

  static BExprP below(const ExprP& e, int64_t bound, int64_t reach) {
    return reach > bound ? b_cmp(BExpr::Lt, e, e_const(bound)) : nullptr;
  }

  bool feeds_pattern(int r) const {
    for (const auto& n : g_.nodes)
      if (p_.contains(n.id) && std::find(n.operands.begin(), n.operands.end(), r) != n.operands.end())
        return true;
    return false;
  }
  bool leaves_kernel(int r) const {
    if (g_.is_output(r)) return true;
    for (const auto& n : g_.nodes)
      if (!p_.contains(n.id) && std::find(n.operands.begin(), n.operands.end(), r) != n.operands.end())
        return true;
    return false;
  }

  // regset into the root's buffer and/or gstore to its tensor (planner.cpp:459-482)
  void store(int r, const std::string& val, const ExprP& e, const ExprP& slot, const BExprP& gd,
             bool to_buffer, bool to_global) {
    const std::string& name = g_.node(r).name;
    if (to_buffer) {
      Stmt s = make(Stmt::RegSet);
      s.dst = "buf_" + name;
      s.dst_slot = slot;
      s.srcs = {val};
      s.guard = gd;
      push(std::move(s));
    }
    if (!to_global) return;
    Stmt s = make(Stmt::GStore);
    s.tensor = name;
    s.idx = index_reg(e);
    s.srcs = {val};
    s.guard = gd;
    push(std::move(s));
    bool listed = false;
    for (const auto& b : prog.outputs) listed = listed || b.name == name;
    if (!listed) prog.outputs.push_back({name, g_.node(r).shape});
  }

  void smem_store(const ExprP& byte_off, const std::string& val, const BExprP& gd) {
    Stmt s = make(Stmt::SStore);
    s.idx = index_reg(byte_off);
    s.srcs = {val};
    s.guard = gd;
    push(std::move(s));
  }

  // planner.cpp:484-580
  void elementwise_group(int r, const ScheduleTemplate& t) {
    const int64_t N = g_.node(r).shape.element_count();
    const bool buf = feeds_pattern(r), gst = leaves_kernel(r);
    const bool expensive = t.op_class == OpClass::ExpensiveElementwise;
    const int64_t ws = dev_.warp_size;
    switch (t.scheme) {
      case CompositionScheme::KernelPacking:
      case CompositionScheme::ThreadComposition: {
        const int64_t trip = cdiv(N, T());
        auto [j, real] = open_loop(trip);
        ExprP e = e_add(global_tid(), e_mul(j, e_const(T())));
        BExprP gd = below(e, N, trip * T());
        const std::string v = value(r, e, gd);
        store(r, v, e, j, gd, buf, gst);
        close_loop(real);
        return;
      }
      case CompositionScheme::WarpComposition: {
        if (expensive) {
          const int64_t trip = cdiv(N, W());
          auto [j, real] = open_loop(trip);
          ExprP e = e_add(wid_, e_mul(j, e_const(W())));
          BExprP gd = b_and(below(e, N, trip * W()), b_cmp(BExpr::Eq, lane_, e_const(0)));
          const std::string v = value(r, e, gd);
          store(r, v, e, j, gd, buf, gst);
          close_loop(real);
          return;
        }
        const int64_t rl = row_len(r), rows = N / rl;
        if (buf && rl > 1) throw Infeasible{"lane-strided values unreachable from lane 0"};
        const int64_t rtrip = cdiv(rows, W());
        auto [jr, rreal] = open_loop(rtrip);
        ExprP row = e_add(wid_, e_mul(jr, e_const(W())));
        BExprP rg = below(row, rows, rtrip * W());
        const int64_t ptrip = cdiv(rl, ws);
        auto [jp, preal] = open_loop(ptrip);
        ExprP col = e_add(lane_, e_mul(jp, e_const(ws)));
        BExprP eg = b_and(rg, below(col, rl, ptrip * ws));
        ExprP e = e_add(e_mul(row, e_const(rl)), col);
        const std::string v = value(r, e, eg);
        store(r, v, e, jr, eg, buf, gst);
        close_loop(preal);
        close_loop(rreal);
        return;
      }
      case CompositionScheme::BlockComposition: {
        if (expensive) {
          const int64_t trip = cdiv(N, ld_.grid);
          auto [j, real] = open_loop(trip);
          ExprP e = e_add(bid_, e_mul(j, e_const(ld_.grid)));
          BExprP gd = b_and(below(e, N, trip * ld_.grid), b_cmp(BExpr::Eq, tid_, e_const(0)));
          const std::string v = value(r, e, gd);
          if (buf) smem_store(e_add(e_const(alloc.slots.at(r).offset), e_mul(j, e_const(4))), v, gd);
          store(r, v, e, j, gd, false, gst);
          close_loop(real);
          if (buf) barrier();
          return;
        }
        const int64_t rl = row_len(r), rows = N / rl;
        const int64_t rtrip = cdiv(rows, ld_.grid);
        auto [jr, rreal] = open_loop(rtrip);
        ExprP row = e_add(bid_, e_mul(jr, e_const(ld_.grid)));
        BExprP rg = below(row, rows, rtrip * ld_.grid);
        const int64_t ptrip = cdiv(rl, ld_.block);
        auto [jp, preal] = open_loop(ptrip);
        ExprP col = e_add(tid_, e_mul(jp, e_const(ld_.block)));
        BExprP eg = b_and(rg, below(col, rl, ptrip * ld_.block));
        ExprP e = e_add(e_mul(row, e_const(rl)), col);
        const std::string v = value(r, e, eg);
        if (buf)
          smem_store(e_add(e_const(alloc.slots.at(r).offset),
                           e_mul(e_add(e_mul(jr, e_const(rl)), col), e_const(4))),
                     v, eg);
        store(r, v, e, jr, eg, false, gst);
        close_loop(preal);
        close_loop(rreal);
        if (buf) barrier();
        return;
      }
    }
  }

  // (row, pos) -> operand element via kept/reduced mixed radix (planner.cpp:583-603)
  ExprP reduce_source(const OpNode& n, const ExprP& row, const ExprP& col) const {
    const TensorShape& in = g_.node(n.operands[0]).shape;
    const auto istr = in.strides();
    std::set<int> ax(n.attrs.axes.begin(), n.attrs.axes.end());
    std::vector<size_t> kept, red;
    for (size_t i = 0; i < in.dims.size(); ++i)
      (ax.count(static_cast<int>(i)) ? red : kept).push_back(i);
    ExprP e = e_const(0);
    auto fold = [&](const std::vector<size_t>& axes, const ExprP& linear) {
      int64_t stride = 1;
      for (size_t i = axes.size(); i-- > 0;) {
        const size_t a = axes[i];
        e = e_add(e, e_mul(e_mod(e_div(linear, e_const(stride)), e_const(in.dims[a])),
                           e_const(istr[a])));
        stride *= in.dims[a];
      }
    };
    fold(kept, row);
    fold(red, col);
    return e;
  }

  void fconst(const std::string& reg, double v) {
    Stmt s = make(Stmt::FConst);
    s.dst = reg;
    s.cval = v;
    push(std::move(s));
  }
  void accum(const std::string& op, const std::string& acc, const std::string& v, const BExprP& gd) {
    Stmt s = make(Stmt::Accum);
    s.op = op;
    s.dst = acc;
    s.srcs = {v};
    s.guard = gd;
    push(std::move(s));
  }

  // planner.cpp:624-758
  void reduction_group(int r, const ScheduleTemplate& t) {
    const OpNode& n = g_.node(r);
    const int src = n.operands[0];
    const int64_t R = n.shape.element_count();
    const int64_t L = g_.node(src).shape.element_count() / R;
    const bool buf = feeds_pattern(r), gst = leaves_kernel(r);
    const bool is_sum = n.kind == OpKind::ReduceSum;
    const std::string op = is_sum ? "sum" : "max";
    const double ident = is_sum ? 0.0 : -std::numeric_limits<double>::infinity();
    const int64_t ws = dev_.warp_size;
    switch (t.scheme) {
      case CompositionScheme::KernelPacking:
      case CompositionScheme::ThreadComposition: {
        const int64_t trip = cdiv(R, T());
        auto [jr, rreal] = open_loop(trip);
        ExprP row = e_add(global_tid(), e_mul(jr, e_const(T())));
        BExprP rg = below(row, R, trip * T());
        const std::string acc = fresh("acc");
        fconst(acc, ident);
        auto [jp, preal] = open_loop(L);
        accum(op, acc, value(src, reduce_source(n, row, jp), rg), rg);
        close_loop(preal);
        store(r, acc, row, jr, rg, buf, gst);
        close_loop(rreal);
        return;
      }
      case CompositionScheme::WarpComposition: {
        const int64_t trip = cdiv(R, W());
        auto [jr, rreal] = open_loop(trip);
        ExprP row = e_add(wid_, e_mul(jr, e_const(W())));
        BExprP rg = below(row, R, trip * W());
        const std::string acc = fresh("acc");
        fconst(acc, ident);
        const int64_t ptrip = cdiv(L, ws);
        auto [jp, preal] = open_loop(ptrip);
        ExprP col = e_add(lane_, e_mul(jp, e_const(ws)));
        BExprP eg = b_and(rg, below(col, L, ptrip * ws));
        accum(op, acc, value(src, reduce_source(n, row, col), eg), eg);
        close_loop(preal);
        Stmt wr = make(Stmt::WarpReduce);
        wr.op = op;
        wr.dst = fresh("t");
        wr.srcs = {acc};
        const std::string red = wr.dst;
        push(std::move(wr));
        store(r, red, row, jr, b_and(rg, b_cmp(BExpr::Eq, lane_, e_const(0))), false, gst);
        if (buf) store(r, red, row, jr, rg, true, false);
        close_loop(rreal);
        return;
      }
      case CompositionScheme::BlockComposition: {
        const int64_t trip = cdiv(R, ld_.grid);
        auto [jr, rreal] = open_loop(trip);
        ExprP row = e_add(bid_, e_mul(jr, e_const(ld_.grid)));
        BExprP rg = below(row, R, trip * ld_.grid);
        const std::string acc = fresh("acc");
        fconst(acc, ident);
        const int64_t ptrip = cdiv(L, ld_.block);
        auto [jp, preal] = open_loop(ptrip);
        ExprP col = e_add(tid_, e_mul(jp, e_const(ld_.block)));
        BExprP eg = b_and(rg, below(col, L, ptrip * ld_.block));
        accum(op, acc, value(src, reduce_source(n, row, col), eg), eg);
        close_loop(preal);
        // per-thread partials staged in scratch, then a power-of-two tree
        ExprP mine = e_add(e_const(scratch_at_), e_mul(tid_, e_const(4)));
        smem_store(mine, acc, rg);
        barrier();
        for (int64_t d = ld_.block / 2; d >= 1; d /= 2) {
          BExprP fg = b_and(rg, b_cmp(BExpr::Lt, tid_, e_const(d)));
          const std::string a = fresh("t"), b = fresh("t"), c = fresh("t");
          Stmt la = make(Stmt::SLoad);
          la.dst = a;
          la.idx = index_reg(mine);
          la.guard = fg;
          push(std::move(la));
          Stmt lb = make(Stmt::SLoad);
          lb.dst = b;
          lb.idx = index_reg(e_add(e_const(scratch_at_), e_mul(e_add(tid_, e_const(d)), e_const(4))));
          lb.guard = fg;
          push(std::move(lb));
          Stmt fo = make(Stmt::FOp);
          fo.op = is_sum ? "add" : "max";
          fo.dst = c;
          fo.srcs = {a, b};
          push(std::move(fo));
          smem_store(mine, c, fg);
          barrier();
        }
        BExprP t0 = b_and(rg, b_cmp(BExpr::Eq, tid_, e_const(0)));
        Stmt ld = make(Stmt::SLoad);
        ld.dst = fresh("t");
        ld.idx = e_const(scratch_at_);
        ld.guard = t0;
        const std::string res = ld.dst;
        push(std::move(ld));
        if (buf) smem_store(e_add(e_const(alloc.slots.at(r).offset), e_mul(jr, e_const(4))), res, t0);
        store(r, res, row, jr, t0, false, gst);
        barrier();
        close_loop(rreal);
        return;
      }
    }
  }

  const CompGraph& g_;
  const FusionPattern& p_;
  const Grouping& grouping_;
  const std::map<int, std::string>& tpl_;
  LaunchDims ld_;
  const DeviceSpec& dev_;
  const std::vector<int>& pos_;

  std::set<int> roots_, done_roots_, bound_;
  std::set<std::pair<int, int>> seen_edges_;
  int current_ = -1;
  int64_t scratch_at_ = -1;
  std::map<std::string, Memo> memo_;
  int regs_ = 0, loops_ = 0;
  std::vector<Frame> frames_;
  std::string chain_;
  const ExprP bid_ = e_var("bid"), tid_ = e_var("tid"), lane_ = e_var("lane"), wid_ = e_var("wid");
};

}  // namespace

std::vector<int> Grouping::group_roots() const {
  std::set<int> s(sub_roots.begin(), sub_roots.end());
  s.insert(roots.begin(), roots.end());
  return {s.begin(), s.end()};
}

// planner.cpp:804-852
std::vector<Grouping> enumerate_groupings(const FusionPattern& p, const CompGraph& g, int cap) {
  const std::vector<int> outs = pattern_outputs(p, g);
  const std::set<int> out_set(outs.begin(), outs.end());
  std::vector<int> forced, optional;
  for (int v : p.vertices) {
    const OpClass c = classify_op(g.node(v));
    if (c == OpClass::Reduction)
      forced.push_back(v);
    else if (c == OpClass::ExpensiveElementwise && !out_set.count(v))
      optional.push_back(v);
  }
  std::stable_sort(optional.begin(), optional.end(), [&](int a, int b) {
    return g.node(a).shape.byte_size() > g.node(b).shape.byte_size();
  });
  int bits = 0;
  while ((1 << (bits + 1)) <= cap && bits < static_cast<int>(optional.size())) ++bits;

  const auto pos = positions_of(g);
  const auto cons = g.consumer_lists();
  std::vector<int> rev = p.vertices;
  std::sort(rev.begin(), rev.end(), [&](int a, int b) { return pos[a] > pos[b]; });

  std::vector<Grouping> out;
  for (int mask = 0; mask < (1 << bits); ++mask) {
    Grouping gr;
    gr.sub_roots = forced;
    for (int i = 0; i < bits; ++i)
      if (mask >> i & 1) gr.sub_roots.push_back(optional[static_cast<size_t>(i)]);
    std::sort(gr.sub_roots.begin(), gr.sub_roots.end());
    gr.roots = outs;
    std::set<int> is_root(gr.sub_roots.begin(), gr.sub_roots.end());
    is_root.insert(outs.begin(), outs.end());
    for (int v : rev) {
      if (is_root.count(v)) {
        gr.group_of[v] = v;
        continue;
      }
      int first = -1;  // earliest in-pattern consumer
      for (int c : cons[static_cast<size_t>(v)])
        if (p.contains(c) && (first < 0 || pos[c] < pos[first])) first = c;
      gr.group_of[v] = gr.group_of.at(first);
    }
    out.push_back(std::move(gr));
  }
  return out;
}

std::map<int, std::string> propagate_schedules(const Grouping& grouping,
                                               const std::map<int, std::string>& root_choice,
                                               const CompGraph&) {
  std::map<int, std::string> out;
  for (const auto& [v, root] : grouping.group_of) out[v] = root_choice.at(root);
  return out;
}

// planner.cpp:862-879
std::vector<LaunchDims> enumerate_launch_dims(const FusionPattern& p, const CompGraph& g,
                                              const DeviceSpec& dev) {
  int64_t extent = 1;
  for (int v : p.vertices) {
    extent = std::max(extent, g.node(v).shape.element_count());
    for (int o : g.node(v).operands) extent = std::max(extent, g.node(o).shape.element_count());
  }
  std::vector<LaunchDims> out;
  for (int b : {64, 128, 256, 512, 1024}) {
    if (b > dev.max_threads_per_block) continue;
    const LaunchDims ld{static_cast<int>(std::clamp<int64_t>(cdiv(extent, b), 1, int64_t(8) * dev.sm_count)), b};
    if (std::find(out.begin(), out.end(), ld) == out.end()) out.push_back(ld);
  }
  return out;
}

// lowest-offset first fit over live ranges in topological emission order
// (planner.cpp:881-927)
AllocationMap allocate_shared_memory(const FusionPattern& p, const std::map<int, int64_t>& requests,
                                     const CompGraph& g, const Grouping* grouping) {
  const auto pos = positions_of(g);
  const auto cons = g.consumer_lists();
  auto last_read = [&](int v) {
    int last = pos[v];
    for (int c : cons[static_cast<size_t>(v)]) {
      if (!p.contains(c)) continue;
      last = std::max(last, pos[grouping ? grouping->group_of.at(c) : c]);
    }
    return last;
  };
  std::vector<int> order;
  for (const auto& kv : requests) order.push_back(kv.first);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return pos[a] < pos[b]; });

  AllocationMap out;
  for (int v : order) {
    const int64_t need = requests.at(v);
    std::vector<std::pair<int64_t, int64_t>> live;
    for (const auto& [u, s] : out.slots)
      if (last_read(u) >= pos[v]) live.push_back({s.offset, s.offset + s.size});
    std::sort(live.begin(), live.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    int64_t off = 0;
    for (const auto& [lo, hi] : live) {
      if (off + need <= lo) break;
      off = std::max(off, hi);
    }
    int donor = -1;
    for (const auto& [u, s] : out.slots)
      if (last_read(u) < pos[v] && s.offset < off + need && off < s.offset + s.size &&
          (donor < 0 || pos[u] > pos[donor]))
        donor = u;
    out.slots[v] = {off, need, donor};
    out.total = std::max(out.total, off + need);
  }
  return out;
}

// peak simultaneously-live named values + overhead (planner.cpp:929-986)
int estimate_register_usage(const StitchedProgram& prog, int overhead) {
  std::map<std::string, int64_t> trips;
  for (const auto& s : prog.stmts)
    if (s.kind == Stmt::Loop) trips[s.loop_var] = eval(s.idx, EvalEnv{nullptr, nullptr});
  struct Span {
    int first = -1, last = -1;
    int64_t width = 1;
  };
  std::map<std::string, Span> spans;
  auto touch = [&](const std::string& r, int i) {
    Span& s = spans[r];
    if (s.first < 0) s.first = i;
    s.last = i;
  };
  std::function<void(const ExprP&, int)> touch_e = [&](const ExprP& e, int i) {
    if (!e) return;
    if (e->kind == Expr::Reg) touch(e->name, i);
    touch_e(e->a, i);
    touch_e(e->b, i);
  };
  std::function<void(const BExprP&, int)> touch_b = [&](const BExprP& e, int i) {
    if (!e) return;
    if (e->kind == BExpr::And) {
      touch_b(e->a, i);
      touch_b(e->b, i);
    } else {
      touch_e(e->lhs, i);
      touch_e(e->rhs, i);
    }
  };
  for (int i = 0; i < static_cast<int>(prog.stmts.size()); ++i) {
    const Stmt& s = prog.stmts[static_cast<size_t>(i)];
    if (!s.dst.empty()) touch(s.dst, i);
    for (const auto& r : s.srcs) touch(r, i);
    touch_e(s.idx, i);
    touch_e(s.src_slot, i);
    touch_b(s.guard, i);
    if (s.kind == Stmt::RegSet && s.dst_slot) {
      touch_e(s.dst_slot, i);
      if (s.dst_slot->kind == Expr::Var) {
        auto it = trips.find(s.dst_slot->name);
        if (it != trips.end()) spans[s.dst].width = std::max(spans[s.dst].width, it->second);
      }
    }
  }
  std::map<int, int64_t> delta;
  for (const auto& kv : spans) {
    delta[kv.second.first] += kv.second.width;
    delta[kv.second.last + 1] -= kv.second.width;
  }
  int64_t live = 0, peak = 0;
  for (const auto& kv : delta) peak = std::max(peak, live += kv.second);
  return overhead + static_cast<int>(peak);
}

// per-thread issue histogram with loop trips multiplied through (planner.cpp:988-1015)
std::map<std::string, int64_t> count_instructions(const StitchedProgram& prog) {
  std::map<std::string, int64_t> hist;
  std::vector<int64_t> trips;
  int64_t mult = 1;
  for (const auto& s : prog.stmts) {
    switch (s.kind) {
      case Stmt::Loop:
        trips.push_back(eval(s.idx, EvalEnv{nullptr, nullptr}));
        mult *= trips.back();
        break;
      case Stmt::EndLoop:
        mult /= trips.back();
        trips.pop_back();
        break;
      case Stmt::ISet: hist["index_calc"] += mult; break;
      case Stmt::FOp: hist[s.op] += mult; break;
      case Stmt::SLoad:
      case Stmt::SStore: hist["shared_access"] += mult; break;
      case Stmt::Shuffle: hist["shuffle"] += mult; break;
      case Stmt::WarpReduce: hist["shuffle"] += 5 * mult; break;
      case Stmt::Accum: hist["reduce_step"] += mult; break;
      default: break;
    }
  }
  return hist;
}

std::optional<KernelPlan> plan_kernel(const FusionPattern& p, const CompGraph& g,
                                      const MachineModel& m, const PlanConstraints* cons) {
  if (p.vertices.empty() || static_cast<int>(p.vertices.size()) > m.search.max_pattern_size)
    return std::nullopt;
  for (int v : p.vertices) {
    if (v < 0 || v >= g.num_nodes() || !is_fusable(g.node(v))) return std::nullopt;
    const OpNode& n = g.node(v);
    if (n.kind == OpKind::Gather && p.contains(n.operands[0])) return std::nullopt;
  }
  if (contraction_creates_cycle(g, p)) return std::nullopt;

  const auto pos = positions_of(g);
  std::optional<KernelPlan> best;
  struct Score {
    double cycles;
    int64_t shmem;
    int block;
    std::string key;
  } best_score{0, 0, 0, ""};
  auto better = [](const Score& a, const Score& b) {  // planner.cpp:1025-1030
    if (a.cycles != b.cycles) return a.cycles < b.cycles;
    if (a.shmem != b.shmem) return a.shmem < b.shmem;
    if (a.block != b.block) return a.block < b.block;
    return a.key < b.key;
  };
  const auto launches = enumerate_launch_dims(p, g, m.dev);

  // Enumerate the candidates in the reference's order (grouping x launch x
  // template odometer), stopping where the reference returns at
  // candidate_cap (planner.cpp:1073), then evaluate them -- in parallel for
  // big patterns: each evaluation is independent and the argmin below walks
  // the results in enumeration order with the same strict tie-breaks, so the
  // chosen plan is identical to the sequential search.
  const std::vector<Grouping> groupings = enumerate_groupings(p, g, m.search.grouping_cap);
  struct Cand {
    size_t gi, li;
    std::vector<size_t> odo;
  };
  std::vector<std::vector<std::vector<const ScheduleTemplate*>>> menus(groupings.size());
  std::vector<std::vector<int>> roots_of(groupings.size());
  std::vector<Cand> cands;
  bool capped = false;
  for (size_t gi = 0; gi < groupings.size() && !capped; ++gi) {
    roots_of[gi] = groupings[gi].group_roots();
    auto& menu = menus[gi];
    bool viable = true;
    for (int r : roots_of[gi]) {
      std::vector<const ScheduleTemplate*> opts;
      for (const auto& t : schedules_for(classify_op(g.node(r)))) {
        const bool allowed = !cons || !cons->force_scheme || t.scheme == *cons->force_scheme ||
                             (*cons->force_scheme == CompositionScheme::ThreadComposition &&
                              t.scheme == CompositionScheme::KernelPacking);
        if (allowed) opts.push_back(&t);
      }
      viable = viable && !opts.empty();
      menu.push_back(std::move(opts));
    }
    if (!viable) continue;
    for (size_t li = 0; li < launches.size() && !capped; ++li) {
      std::vector<size_t> odo(roots_of[gi].size(), 0);
      for (;;) {
        if (static_cast<int>(cands.size()) >= m.search.candidate_cap) {
          capped = true;
          break;
        }
        cands.push_back({gi, li, odo});
        size_t i = 0;
        while (i < odo.size() && ++odo[i] == menu[i].size()) odo[i++] = 0;
        if (i == odo.size()) break;
      }
    }
  }
  auto templates_of = [&](const Cand& c, std::string* key) {
    std::map<int, std::string> tpl;
    for (size_t i = 0; i < roots_of[c.gi].size(); ++i) {
      tpl[roots_of[c.gi][i]] = menus[c.gi][i][c.odo[i]]->id;
      if (key) *key += menus[c.gi][i][c.odo[i]]->id + ";";
    }
    return tpl;
  };
  struct Eval {
    bool ok = false;
    Score score{0, 0, 0, ""};
  };
  std::vector<Eval> evals(cands.size());
  auto evaluate = [&](size_t ci) {
    const Cand& c = cands[ci];
    std::string key;
    const auto tpl = templates_of(c, &key);
    const LaunchDims& ld = launches[c.li];
    ProgramBuilder b(g, p, groupings[c.gi], tpl, ld, m.dev, pos);
    try {
      b.build();
    } catch (const Infeasible&) {
      return;
    }
    const int regs = estimate_register_usage(b.prog, m.costs.register_overhead);
    const auto occ = occupancy(ld, regs, b.prog.shmem_bytes, m.dev);
    if (!occ) return;
    double waves = wave_count(double(ld.total_threads()) / m.dev.warp_size, *occ, m.dev);
    if (m.costs.ceil_waves) waves = std::ceil(waves);
    evals[ci].score = Score{waves * warp_latency(count_instructions(b.prog), m.cpi), b.prog.shmem_bytes, ld.block, key};
    evals[ci].ok = true;
  };
  const bool first_feasible = cons && cons->first_feasible;
  unsigned threads = 1;
  if (cands.size() >= 32) {
    const char* t = std::getenv("STITCH_PLAN_THREADS");
    const unsigned want = t && *t ? static_cast<unsigned>(std::atoi(t)) : std::thread::hardware_concurrency();
    threads = std::max(1u, std::min<unsigned>(want, static_cast<unsigned>(cands.size() / 8)));
  }
  size_t chosen = cands.size();
  if (first_feasible && threads > 1) {
    // the explorer's feasibility probe (explorer.cpp:100-131): the FIRST
    // feasible candidate in enumeration order.  Indices are handed out in
    // increasing order and nobody takes one past the lowest feasible index
    // found so far, so every index below it was evaluated and the result is
    // the sequential scan's -- infeasible patterns (the whole cap) no longer
    // take one thread (DIEN T=10 probes: 35 s of its 37 s plan)
    std::atomic<size_t> next{0}, found{cands.size()};
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (size_t ci; (ci = next++) < cands.size() && ci < found.load();) {
          evaluate(ci);
          if (!evals[ci].ok) continue;
          size_t cur = found.load();
          while (ci < cur && !found.compare_exchange_weak(cur, ci)) {
          }
        }
      });
    for (auto& th : pool) th.join();
    if (found.load() < cands.size()) {
      chosen = found.load();
      best_score = evals[chosen].score;
    }
  } else if (threads <= 1) {
    for (size_t ci = 0; ci < cands.size(); ++ci) {
      evaluate(ci);
      if (!evals[ci].ok) continue;
      if (chosen == cands.size() || better(evals[ci].score, best_score)) {
        best_score = evals[ci].score;
        chosen = ci;
      }
      if (first_feasible) break;
    }
  } else {
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (size_t ci; (ci = next++) < cands.size();) evaluate(ci);
      });
    for (auto& th : pool) th.join();
    for (size_t ci = 0; ci < cands.size(); ++ci)
      if (evals[ci].ok && (chosen == cands.size() || better(evals[ci].score, best_score))) {
        best_score = evals[ci].score;
        chosen = ci;
      }
  }
  if (chosen == cands.size()) return best;
  // rebuild the winner's full KernelPlan (deterministic)
  const Cand& c = cands[chosen];
  const auto tpl = templates_of(c, nullptr);
  const LaunchDims& ld = launches[c.li];
  ProgramBuilder b(g, p, groupings[c.gi], tpl, ld, m.dev, pos);
  b.build();
  const int regs = estimate_register_usage(b.prog, m.costs.register_overhead);
  KernelPlan k;
  k.pattern = p;
  k.grouping = groupings[c.gi];
  k.per_op_schedule = propagate_schedules(groupings[c.gi], tpl, g);
  k.launch = ld;
  k.shmem_alloc = b.alloc;
  k.scratch_bytes = b.prog.shmem_bytes - b.alloc.total;
  k.regs_per_thread = regs;
  k.occupancy_value = *occupancy(ld, regs, b.prog.shmem_bytes, m.dev);
  k.estimated_cycles = best_score.cycles;
  k.instr_histogram = count_instructions(b.prog);
  k.boundaries = b.boundaries;
  k.program = std::move(b.prog);
  best = std::move(k);
  return best;
}

std::string emit_kernel_text(const KernelPlan& k) { return emit_program_text(k.program); }

}  // namespace stitch
