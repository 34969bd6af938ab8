// Dataflow stitching templates (local / regional / global / independent).
//
// A pattern is split into connected components; each component is matched to
// a template by the shape of its reductions:
//   no reductions                       -> local   (one body per output shape)
//   all reductions over trailing axes,  -> regional (row-resident teams)
//     same (outer, inner) split
//   all reductions over leading axes,   -> global  (slab partials, last CTA per strip combines)
//     same (reduced, kept) split
// Bodies with the same domain are merged so shared inputs are read once (e.g.
// the two column reductions of colreduce read dy once), and all bodies of a
// pattern run in one launch on disjoint CTA ranges (independent packing).
//
// Values are emitted on demand with common-subexpression elimination keyed by
// (vertex, coordinates): a tensor element requested twice at the same
// coordinates — e.g. x in both LayerNorm reductions and in the normalisation —
// is loaded once and stays in registers.  Coordinates are per-axis C
// expressions; the innermost one may vary across the W (=4) lanes of a
// 128-bit vector, which is how loads become float4 and broadcast sources
// become single scalar loads.
//
// Numerics follow the reference evaluator (src/sim.cpp:111-229): every op's
// result is rounded to its dtype (f32 arithmetic without FMA contraction is
// exactly "compute in f64, round to f32" for + - * /), reductions accumulate
// in f64 and round once, max/min use std::max/min argument order.
#include <algorithm>
#include <cmath>
#include <functional>
#include <map>
#include <set>
#include <sstream>

#include "codegen/cg.hpp"

namespace stitch::gpu {

namespace {

// SMs of the device the kernels are generated for (grid sizing, one-wave
// tests): set per generator call from the executor's device attribute;
// 148 (B200) for device-free code generation
thread_local int tl_sm_count = 148;
struct SmScope {
  int old;
  explicit SmScope(int sm) : old(tl_sm_count) {
    if (sm > 0) tl_sm_count = sm;
  }
  ~SmScope() { tl_sm_count = old; }
};
inline int sm_now() { return tl_sm_count; }

// Resident generation (cg_resident.cpp): every pattern kernel is emitted for
// one 1024-thread CTA that is also the physical CTA -- no clusters, no PDL
thread_local int tl_force_block = 0;

// When a kernel triggers its dependents (griddepcontrol.launch_dependents).
// For large grids (STITCH_PDL_TRIGGER=entry_large, the default; =entry for
// all): first thing in the kernel, before its
// own griddepcontrol.wait.  The hoisted prologue issues every graph-parameter
// load before the wait, so triggering after the wait would hold the next
// kernel back until this one's loads have landed; at entry the dependent
// launches as soon as every CTA of this grid is resident and parks in its own
// wait (softmax 8.33 -> 7.97 us, colreduce 21.27 -> 19.87 us,
// profiles/r01/pdl_trigger_ab.jsonl).  Ordering is unchanged: a dependent's
// wait returns only after its producers complete, and every kernel waits
// before it exits, so completion is transitive along chains.  =wait: trigger
// right after the wait; =entry_small: at entry only for grids of <= 148 CTAs.
// Default =entry_large: at entry for grids of more than 148 CTAs, after the
// wait for smaller ones -- a chain of one-wave kernels (DIEN) does better
// when a dependent is not parked before its own producers have finished
// (T=10 53.8 -> 52.5 us, T=20 108.8 -> 105.3 us; profiles/r01/pdl_trigger_ab.jsonl).
bool entry_trigger(int grid) {
  const char* v = std::getenv("STITCH_PDL_TRIGGER");
  const std::string mode = v && *v ? v : "entry_large";
  if (mode == "entry") return true;
  if (mode == "entry_small") return grid <= sm_now();
  if (mode == "entry_large") return grid > sm_now();
  return false;
}

int64_t pow2ceil(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

struct Coord {
  std::string base;      // C expression (index type)
  bool vary = false;     // lane k adds k
  bool aligned = true;   // base is a multiple of the vector width
};
using Coords = std::vector<Coord>;

struct Val {
  std::vector<std::string> lanes;  // 1 entry = uniform across lanes
  const std::string& at(int k) const { return lanes.size() == 1 ? lanes[0] : lanes[static_cast<size_t>(k)]; }
  bool uniform() const { return lanes.size() == 1; }
};

std::string coords_key(const Coords& c) {
  std::string k;
  for (const auto& x : c) k += x.base + (x.vary ? "~|" : "|");
  return k;
}

// ---- per-kernel emission state ----------------------------------------------
class Emitter {
 public:
  Emitter(const CompGraph& g, const std::set<int>& pattern, bool wide_index)
      : g_(g), pattern_(pattern), ix_(wide_index ? "i64" : "int") {}

  std::ostringstream out;
  std::string ind = "  ";
  int W = 1;
  int block = 256;                         // the kernel's CTA size (every body uses it)
  std::set<int> loaded;                    // external tensors read
  std::map<std::string, Val> reduced;      // (reduction vertex, coords) -> value
  std::set<int> cached_tensors;            // read through L1 (re-read broadcast sources)
  // regional staging: loads at a row body's own (row, chunk) coordinates of a
  // tensor staged in shared memory read the CTA's TMA-filled tile instead
  std::map<std::string, std::string> domain_off;  // coords key -> float offset in a staged tile
  std::map<int, std::string> staged_ptr;          // tensor -> smem base of its tile (current stage)
  std::vector<int> domain_dims;                   // O ++ I of the body being emitted
  std::set<int> staged_hits;                      // tensors seen at domain coordinates
  // register pipeline (regional): coords key -> chunk index, tensors whose
  // current row lives in registers cu_<name>_<chunk> (prefetched a row ahead)
  std::map<std::string, int> domain_chunk;
  std::set<int> reg_staged;
  // row-invariant [L] operands copied once per CTA into shared memory:
  // tensor -> smem array (loads at a chunk offset read it instead of global)
  std::map<int, std::string> smem_bcast;

  const std::string& ix() const { return ix_; }
  std::string fresh(const char* p) { return p + std::to_string(counter_++); }
  void line(const std::string& s) { out << ind << s << "\n"; }
  void open(const std::string& s) {
    line(s + " {");
    ind += "  ";
    scopes_.push_back(memo_);
    wait_scopes_.push_back(waited_);
  }
  void close() {
    ind.resize(ind.size() - 2);
    line("}");
    memo_ = scopes_.back();
    scopes_.pop_back();
    waited_ = wait_scopes_.back();
    wait_scopes_.pop_back();
  }

  // Programmatic dependent launch with a hoisted prologue: graph parameters
  // are never written by a kernel, so their loads may be issued before
  // griddepcontrol.wait -- overlapping the previous kernel's drain.  Every
  // load of a kernel-produced tensor and every global write comes after the
  // wait (emitted lazily, once per control path); the CTA triggers its
  // dependents right after its own wait.
  bool hoist = false;
  void ensure_wait() {
    if (!hoist || waited_) return;
    line("pdl_wait(); pdl_launch();");
    waited_ = true;
  }
  bool is_param(int v) const { return g_.node(v).kind == OpKind::Parameter; }
  void reset_wait() {
    waited_ = false;
    wait_scopes_.clear();
  }
  void clear_memo() { memo_.clear(); }

  static std::string key(int v, const Coords& c) { return std::to_string(v) + "@" + coords_key(c); }

  Val value(int v, const Coords& c) {
    const std::string k = key(v, c);
    if (auto it = memo_.find(k); it != memo_.end()) return it->second;
    Val r = compute(v, c);
    memo_[k] = r;
    return r;
  }

  // linear element index of `c` for lane k (only varying coords shift)
  std::string linear(int v, const Coords& c, int k) const {
    const auto strides = g_.node(v).shape.strides();
    std::string s;
    for (size_t i = 0; i < c.size(); ++i) {
      std::string term = c[i].base;
      if (c[i].vary && k) term = "(" + term + " + " + std::to_string(k) + ")";
      if (term == "0") continue;
      if (strides[i] != 1) term = "(" + ix_ + ")" + term + " * " + std::to_string(strides[i]);
      s += (s.empty() ? "" : " + ") + term;
    }
    return s.empty() ? "0" : s;
  }

 private:
  Val load(int v, const Coords& c) {
    loaded.insert(v);
    if (!is_param(v)) ensure_wait();
    const TensorShape& sh = g_.node(v).shape;
    const std::string ptr = tensor_ident(g_.node(v).name);
    int nvary = 0, last_vary = -1;
    for (size_t i = 0; i < c.size(); ++i)
      if (c[i].vary) ++nvary, last_vary = static_cast<int>(i);
    if (auto sb = smem_bcast.find(v); sb != smem_bcast.end() && W == 4 && c.size() == 1 && c[0].vary) {
      const std::string q = fresh("q");
      line("const float4 " + q + " = lds4(" + sb->second + " + " + c[0].base + ");");
      Val r;
      for (const char* f : {".x", ".y", ".z", ".w"}) r.lanes.push_back(q + f);
      return r;
    }
    if (W == 4 && sh.dtype == DType::F32 && !domain_off.empty()) {
      auto it = domain_off.find(coords_key(c));
      std::vector<int> dd;
      for (auto d : sh.dims) dd.push_back(static_cast<int>(d));
      if (it != domain_off.end() && dd == domain_dims) {
        staged_hits.insert(v);
        if (reg_staged.count(v)) {
          const std::string q = "cu_" + tensor_ident(g_.node(v).name) + "_" + std::to_string(domain_chunk.at(it->first));
          Val r;
          for (const char* f : {".x", ".y", ".z", ".w"}) r.lanes.push_back(q + f);
          return r;
        }
        if (auto sp = staged_ptr.find(v); sp != staged_ptr.end()) {
          const std::string q = fresh("q");
          line("const float4 " + q + " = lds4(" + sp->second + " + " + it->second + ");");
          Val r;
          for (const char* f : {".x", ".y", ".z", ".w"}) r.lanes.push_back(q + f);
          return r;
        }
      }
    }
    // graph parameters: non-coherent loads (immutable for the graph's
    // lifetime); tensors of earlier kernels: coherent (prelude, ld4k)
    const bool param = is_param(v);
    const std::string LV = param ? "ldv(" : "ldvk(";
    if (nvary == 0 || W == 1) {
      const std::string t = fresh("t");
      line("const float " + t + " = " + LV + ptr + ", " + linear(v, c, 0) + ");");
      if (nvary == 0) return {{t}};
      return {{t}};
    }
    const bool contiguous = nvary == 1 && last_vary == static_cast<int>(c.size()) - 1 &&
                            c.back().aligned && sh.dims.back() % W == 0 && W == 4;
    Val r;
    if (contiguous && sh.dtype == DType::F16) {  // 4 halves, one 64-bit load
      const std::string q = fresh("q");
      line("const float4 " + q + " = " + (param ? "ld4h(" : "ld4hk(") + ptr + " + " + linear(v, c, 0) + ");");
      for (const char* f : {".x", ".y", ".z", ".w"}) r.lanes.push_back(q + f);
      return r;
    }
    if (contiguous && sh.dtype == DType::F32) {
      const std::string q = fresh("q");
      const bool cached = cached_tensors.count(v) > 0;
      line("const float4 " + q + " = " + (!param ? "ld4k(" : cached ? "ld4c(" : "ld4(") + ptr + " + " + linear(v, c, 0) + ");");
      for (const char* f : {".x", ".y", ".z", ".w"}) r.lanes.push_back(q + f);
      return r;
    }
    for (int k = 0; k < W; ++k) {
      const std::string t = fresh("t");
      line("const float " + t + " = " + LV + ptr + ", " + linear(v, c, k) + ");");
      r.lanes.push_back(t);
    }
    return r;
  }

  static std::string round_to(DType d, const std::string& e) {
    switch (d) {
      case DType::F32: return e;
      case DType::F16: return "rnd_f16(" + e + ")";
      case DType::I32: return "rnd_i32(" + e + ")";
      case DType::Bool: return "rnd_bool(" + e + ")";
    }
    return e;
  }

  static std::string op_expr(OpKind k, const std::string& a, const std::string& b) {
    switch (k) {
      case OpKind::Add: return a + " + " + b;
      case OpKind::Sub: return a + " - " + b;
      case OpKind::Mul: return a + " * " + b;
      case OpKind::Div: return a + " / " + b;
      case OpKind::Max: return "op_max(" + a + ", " + b + ")";
      case OpKind::Min: return "op_min(" + a + ", " + b + ")";
      case OpKind::Power: return "powf(" + a + ", " + b + ")";
      // MUFU.EX2 form (rel err < 5.5e-6, prelude exp_fast): the softmax chain
      // is close to issue-bound and the accurate expf sequence costs ~8 more
      // instructions per element (C2 8.61 -> 8.29 us, profiles/r01/fast_exp_ab.jsonl)
      case OpKind::Exp: return (env_int("STITCH_FAST_EXP", 1) ? "exp_fast(" : "expf(") + a + ")";
      case OpKind::Tanh: return "tanhf(" + a + ")";
      case OpKind::Log: return "logf(" + a + ")";
      case OpKind::Rsqrt: return "op_rsqrt(" + a + ")";
      default: break;
    }
    throw TemplateMismatch("not an elementwise op");
  }

  // Division by a value shared by all lanes (a row statistic, a constant):
  // one IEEE reciprocal per divisor, then Markstein's correction per element
  // (q = a*r; e = fma(-q, b, a); q + e*r) which is the correctly rounded a/b
  // whenever r is a normal number -- bit-identical to IEEE division, at three
  // FMA-pipe ops instead of the full division sequence.  Divisors outside
  // [2^-125, 2^125] take the IEEE path (uniform branch).
  Val divide_by_uniform(const Val& a, const std::string& b) {
    const std::string rk = "R|" + b;
    std::string r, ok;
    if (auto it = memo_.find(rk); it != memo_.end()) {
      r = it->second.lanes[0];
      ok = it->second.lanes[1];
    } else {
      r = fresh("rcp");
      ok = fresh("rok");
      line("const float " + r + " = 1.0f / " + b + ";");
      line("const bool " + ok + " = fabsf(" + b + ") >= 0x1p-125f && fabsf(" + b + ") <= 0x1p125f;");
      memo_[rk] = Val{{r, ok}};
    }
    Val out;
    std::string decl = "float", fast, slow;
    for (int k = 0; k < W; ++k) {
      const std::string t = fresh("t");
      out.lanes.push_back(t);
      decl += std::string(k ? ", " : " ") + t;
      fast += t + " = div_rcp(" + a.at(k) + ", " + b + ", " + r + "); ";
      slow += t + " = " + a.at(k) + " / " + b + "; ";
    }
    line(decl + ";");
    line("if (" + ok + ") { " + fast + "} else { " + slow + "}");
    return out;
  }

  Val compute(int v, const Coords& c) {
    const OpNode& n = g_.node(v);
    if (!pattern_.count(v) || n.kind == OpKind::Constant) {
      if (n.kind == OpKind::Constant) {
        double val = n.attrs.value;
        if (n.shape.dtype == DType::F16) val = static_cast<double>(static_cast<float>(val));  // approx
        if (n.shape.dtype == DType::I32) val = std::llround(val);
        if (n.shape.dtype == DType::Bool) val = val != 0.0;
        return {{c_float(val)}};
      }
      return load(v, c);
    }
    switch (classify_op(n)) {
      case OpClass::Reduction: {
        auto it = reduced.find(key(v, c));
        if (it == reduced.end())
          throw TemplateMismatch("reduction " + n.name + " read outside the work unit that owns it");
        return it->second;
      }
      case OpClass::LightElementwise:
      case OpClass::ExpensiveElementwise: {
        std::vector<Val> ops;
        bool uni = true;
        for (int o : n.operands) {
          ops.push_back(value(o, c));
          uni = uni && ops.back().uniform();
        }
        Val r;
        const int lanes = uni ? 1 : W;
        if (n.kind == OpKind::Div && !uni && ops[1].uniform() && n.shape.dtype == DType::F32)
          return divide_by_uniform(ops[0], ops[1].at(0));
        for (int k = 0; k < lanes; ++k) {
          const std::string a = ops[0].at(k), b = ops.size() > 1 ? ops[1].at(k) : "";
          const std::string t = fresh("t");
          line("const float " + t + " = " + round_to(n.shape.dtype, op_expr(n.kind, a, b)) + ";");
          r.lanes.push_back(t);
        }
        return r;
      }
      case OpClass::ShapeOp: break;
      case OpClass::Opaque: throw TemplateMismatch("opaque op inside a pattern");
    }
    const int src = n.operands.empty() ? -1 : n.operands[0];
    switch (n.kind) {
      case OpKind::Broadcast: {
        Coords in;
        for (int d : n.attrs.dims) in.push_back(c[static_cast<size_t>(d)]);
        return value(src, in);
      }
      case OpKind::Transpose: {
        Coords in(c.size());
        for (size_t j = 0; j < c.size(); ++j) in[static_cast<size_t>(n.attrs.perm[j])] = c[j];
        return value(src, in);
      }
      case OpKind::Slice: {
        Coords in = c;
        for (size_t j = 0; j < c.size(); ++j) {
          const int s = n.attrs.starts[j];
          if (!s) continue;
          in[j].base = "(" + c[j].base + " + " + std::to_string(s) + ")";
          in[j].aligned = c[j].aligned && s % std::max(W, 1) == 0;
        }
        return value(src, in);
      }
      case OpKind::Gather: {
        const int data = n.operands[0], indices = n.operands[1];
        const int kr = g_.node(indices).shape.rank();
        Coords ic(c.begin(), c.begin() + kr);
        const Val iv = value(indices, ic);
        bool tail_vary = false;
        for (size_t j = static_cast<size_t>(kr); j < c.size(); ++j) tail_vary = tail_vary || c[j].vary;
        const int lanes = (iv.uniform() && !tail_vary) ? 1 : W;
        Val r;
        for (int k = 0; k < lanes; ++k) {
          Coords dc;
          dc.push_back({"(" + ix_ + ")" + iv.at(k), false, false});
          for (size_t j = static_cast<size_t>(kr); j < c.size(); ++j) {
            Coord x = c[j];
            if (x.vary && k) x.base = "(" + x.base + " + " + std::to_string(k) + ")";
            x.vary = false;
            dc.push_back(x);
          }
          if (pattern_.count(data)) throw TemplateMismatch("gather of in-pattern data");
          loaded.insert(data);
          if (!is_param(data)) ensure_wait();
          const std::string t = fresh("t");
          line("const float " + t + " = " + (is_param(data) ? "ldv(" : "ldvk(") + tensor_ident(g_.node(data).name) + ", " +
               linear(data, dc, 0) + ");");
          r.lanes.push_back(t);
        }
        return r;
      }
      default: break;
    }
    throw TemplateMismatch("no dataflow rule for " + n.name);
  }

  const CompGraph& g_;
  const std::set<int>& pattern_;
  std::string ix_;
  int counter_ = 0;
  std::map<std::string, Val> memo_;
  std::vector<std::map<std::string, Val>> scopes_;
  bool waited_ = false;
  std::vector<bool> wait_scopes_;
};

// ---- analysis ---------------------------------------------------------------
struct Component {
  std::vector<int> members;
  std::vector<int> outputs;
  std::vector<int> reductions;
};

enum class Kind { Local, Row, Column };

struct Body {
  Kind kind;
  std::vector<int> dims_a, dims_b;  // local: domain dims; row: outer, inner; column: reduced, kept
  std::vector<int> outputs;         // outputs handled by this body
  std::vector<int> reductions;
  int64_t bytes = 0;
  int blocks = 1;
  // original tensor axis of each position of dims_a ++ dims_b (empty:
  // identity).  Reductions over middle / non-contiguous axes keep the row
  // (last axis reduced) or column (last axis kept) mapping through it.
  std::vector<int> perm;
  // row bodies only: some reductions or outputs live on another trailing
  // domain of the same rows (O ++ J, J != the primary inner dims), e.g. a
  // softmax over a [B,T] score row feeding [B,H] gates of the same sequence;
  // those run as team-strided scalar loops.  tpr > 0 overrides the team size.
  bool multi = false;
  int tpr = 0;
};

// coordinates listed in dims_a ++ dims_b order -> tensor axis order
Coords arrange(const Coords& ab, const std::vector<int>& perm) {
  if (perm.empty()) return ab;
  Coords out(ab.size());
  for (size_t i = 0; i < ab.size(); ++i) out[static_cast<size_t>(perm[i])] = ab[i];
  return out;
}

std::vector<int64_t> to64(const std::vector<int>& v) { return {v.begin(), v.end()}; }

std::vector<int> dims_of(const TensorShape& s) {
  std::vector<int> d;
  for (auto x : s.dims) d.push_back(static_cast<int>(x));
  return d;
}

int64_t prod(const std::vector<int>& d) {
  int64_t p = 1;
  for (int x : d) p *= x;
  return p;
}

// does v (transitively, inside the pattern) depend on a reduction?
bool downstream_of_reduction(const CompGraph& g, const std::set<int>& pat, int v,
                             std::map<int, bool>& memo) {
  if (auto it = memo.find(v); it != memo.end()) return it->second;
  bool r = false;
  if (pat.count(v)) {
    if (classify_op(g.node(v)) == OpClass::Reduction) r = true;
    for (int o : g.node(v).operands) r = r || downstream_of_reduction(g, pat, o, memo);
  }
  memo[v] = r;
  return r;
}

int reduction_level(const CompGraph& g, const std::set<int>& pat, int v, std::map<int, int>& memo) {
  if (!pat.count(v)) return 0;
  if (auto it = memo.find(v); it != memo.end()) return it->second;
  int lvl = 0;
  for (int o : g.node(v).operands) lvl = std::max(lvl, reduction_level(g, pat, o, memo));
  if (classify_op(g.node(v)) == OpClass::Reduction) ++lvl;
  memo[v] = lvl;
  return lvl;
}

std::vector<Component> components_of(const CompGraph& g, const std::vector<int>& verts) {
  std::set<int> in(verts.begin(), verts.end());
  const auto cons = g.consumer_lists();
  std::set<int> seen;
  std::vector<Component> out;
  for (int s : verts) {
    if (seen.count(s)) continue;
    Component c;
    std::vector<int> stack{s};
    seen.insert(s);
    while (!stack.empty()) {
      int v = stack.back();
      stack.pop_back();
      c.members.push_back(v);
      auto visit = [&](int u) {
        if (in.count(u) && seen.insert(u).second) stack.push_back(u);
      };
      for (int o : g.node(v).operands) visit(o);
      for (int x : cons[static_cast<size_t>(v)]) visit(x);
    }
    std::sort(c.members.begin(), c.members.end());
    for (int v : c.members) {
      bool ext = g.is_output(v);
      for (int x : cons[static_cast<size_t>(v)]) ext = ext || !in.count(x);
      if (ext) c.outputs.push_back(v);
      if (classify_op(g.node(v)) == OpClass::Reduction) c.reductions.push_back(v);
    }
    out.push_back(std::move(c));
  }
  return out;
}

// ---- template emitters --------------------------------------------------------
constexpr int kBlock = 256;

// decompose linear index `lin` (expression) over dims into coordinate exprs
std::vector<std::string> decompose(Emitter& em, const std::string& lin, const std::vector<int>& dims,
                                   const std::string& prefix) {
  std::vector<std::string> cs(dims.size());
  int64_t stride = 1;
  for (size_t i = dims.size(); i-- > 0;) {
    const std::string name = em.fresh(prefix.c_str());
    std::string e = lin;
    if (stride != 1) e = "(" + e + ") / " + std::to_string(stride);
    if (i != 0) e = "(" + e + ") % " + std::to_string(dims[i]);
    em.line("const " + em.ix() + " " + name + " = " + e + ";");
    cs[i] = name;
    stride *= dims[i];
  }
  return cs;
}

void store_val(Emitter& em, const CompGraph& g, int v, const Coords& c, const Val& val,
               const std::string& guard) {
  const TensorShape& sh = g.node(v).shape;
  const std::string ptr = tensor_ident(g.node(v).name);
  int nvary = 0;
  for (const auto& x : c) nvary += x.vary;
  const std::string pre = guard.empty() ? "" : "if (" + guard + ") ";
  em.ensure_wait();
  if (em.W == 4 && nvary == 1 && c.back().vary && c.back().aligned &&
      (sh.dtype == DType::F32 || (sh.dtype == DType::F16 && sh.dims.back() % 4 == 0))) {
    em.line(pre + (sh.dtype == DType::F32 ? "st4(" : "st4h(") + ptr + " + " + em.linear(v, c, 0) + ", " + val.at(0) +
            ", " + val.at(1) + ", " + val.at(2) + ", " + val.at(3) + ");");
    return;
  }
  if (nvary == 0) {
    em.line(pre + "stv(" + ptr + ", " + em.linear(v, c, 0) + ", " + val.at(0) + ");");
    return;
  }
  for (int k = 0; k < em.W; ++k)
    em.line(pre + "stv(" + ptr + ", " + em.linear(v, c, k) + ", " + val.at(k) + ");");
}

// 128-bit chunks in flight per thread per grid-stride step: 2, with up to
// 32 CTAs per SM so big domains take ~one pass (B200 sweep,
// profiles/r01/local_sweep.jsonl: bias+GELU 18.4 -> 16.3 us)
int local_unroll(int64_t chunks, int block) {
  (void)chunks, (void)block;
  if (const int u = env_int("STITCH_LOCAL_U", 0); u > 0) return u;
  return 2;
}

// Launch-bound local bodies (domain <= STITCH_LOCAL_SMALL elements, default
// 32768 -- less than one wave at one element per thread; e.g. DIEN's [256,36]
// gates): one element per thread (DIEN T=10 81.5 -> 59.6 us,
// profiles/r01/local_small_ab.jsonl).  Such a kernel is a
// single partial wave whose time is one warp's instruction chain (loads,
// then the dependent math, then stores), so fewer elements per thread -- no
// 128-bit chunks, no unroll -- is shorter (ncu: ra1 at 2 x float4 per thread
// issues 356 instructions per warp at ~20 cycles each).
bool local_small(int64_t elements) { return elements <= env_int("STITCH_LOCAL_SMALL", 32768); }

int local_width(const std::vector<int>& dims) {
  if (dims.empty() || dims.back() % 4 != 0) return 1;
  int64_t n = 1;
  for (int d : dims) n *= d;
  return local_small(n) ? 1 : 4;
}

// local: grid-stride over W-wide chunks of the domain, U chunks per thread
void emit_local(Emitter& em, const CompGraph& g, const Body& b) {
  const std::vector<int>& D = b.dims_a;
  const int64_t N = prod(D);
  em.W = local_width(D);
  const int64_t chunks = N / em.W;
  const int B = em.block;
  const int U = local_small(N) ? 1 : local_unroll(chunks, B);
  em.line("// local body: domain " + std::to_string(N) + " elements, vector " + std::to_string(em.W));
  em.open("for (i64 c0_ = (i64)vbid * " + std::to_string(B * U) + " + threadIdx.x; c0_ < " +
          std::to_string(chunks) + "; c0_ += (i64)vgrid * " + std::to_string(B * U) + ")");
  std::vector<std::tuple<int, Coords, Val, std::string>> stores;
  for (int u = 0; u < U; ++u) {
    const std::string ok = em.fresh("ok"), cc = em.fresh("cc");
    em.line("const bool " + ok + " = c0_ + " + std::to_string(u * B) + " < " + std::to_string(chunks) + ";");
    em.line("const " + em.ix() + " " + cc + " = (" + em.ix() + ")(" + ok + " ? c0_ + " +
            std::to_string(u * B) + " : " + std::to_string(chunks - 1) + ");");
    Coords c;
    if (!D.empty()) {
      const std::string lin = em.W == 1 ? cc : cc + " * " + std::to_string(em.W);
      auto names = decompose(em, lin, D, "d");
      for (size_t i = 0; i < D.size(); ++i) c.push_back({names[i], i + 1 == D.size() && em.W > 1, true});
    }
    for (int o : b.outputs) stores.emplace_back(o, c, em.value(o, c), ok);
  }
  for (auto& [o, c, v, ok] : stores) store_val(em, g, o, c, v, ok);
  em.close();
}

struct RowParams {
  int W, TPR, NJ, RPB, block;
};

// TMA-staged regional pipeline: each persistent CTA owns a contiguous range
// of row tiles (RPB rows) and keeps `stages` tiles of every staged tensor in
// flight in shared memory (cp.async.bulk + mbarrier complete_tx).
struct StageCfg {
  std::vector<int> tensors;  // staged external inputs (dims == O ++ I, f32)
  int stages = 3;
  int64_t tile_floats = 0;   // RPB * L
  int64_t bytes = 0;         // dynamic smem: barriers + stages * tensors * tile
  // STITCH_STAGE=2: per-team rings -- every row team owns `stages` row
  // buffers, each with its own mbarrier; the team's lead thread issues one
  // bulk copy per tensor per row, and a buffer is refilled after a team-only
  // sync (no CTA-wide barrier, no wait on other teams' rows)
  bool team = false;
  int64_t bar_bytes = 128;   // mbarrier region ahead of the buffers
};

// block = 0: the team's natural CTA (max(256, TPR)); else the kernel's CTA
// size, a multiple of TPR
RowParams row_params(const std::vector<int>& inner, int block = 0, int tpr = 0) {
  const int64_t L = prod(inner);
  RowParams p;
  p.W = inner.back() % 4 == 0 ? 4 : (inner.back() % 2 == 0 ? 2 : 1);
  const int64_t nch = L / p.W;
  // chunks per thread: short rows (softmax, 32 float4) want more threads per
  // row and fewer registers (2 chunks); long rows keep ~8 chunks so a team
  // stays within one warp (B200 sweep, profiles/r01/row_chunk_sweep.jsonl)
  const int nj_target = std::max(1, env_int("STITCH_ROW_NJ", nch <= 64 ? 2 : 8));
  p.TPR = tpr > 0 ? tpr : static_cast<int>(std::clamp<int64_t>(pow2ceil((nch + nj_target - 1) / nj_target), 1, 1024));
  p.NJ = static_cast<int>((nch + p.TPR - 1) / p.TPR);
  p.block = block > 0 ? block : std::max(kBlock, p.TPR);
  p.RPB = p.block / p.TPR;
  return p;
}

// regional: a team of TPR threads owns a row; row elements live in registers
// (st != nullptr: the CTA's rows arrive through the TMA pipeline in smem)
// cluster > 1: regional-cluster mapping -- one row per thread-block cluster,
// the row's chunks spread over cluster x block threads, team reductions
// finished across the cluster through distributed shared memory
RowParams cluster_row_params(const std::vector<int>& inner, int cluster, int block) {
  RowParams p;
  const int64_t L = prod(inner);
  p.W = inner.back() % 4 == 0 ? 4 : (inner.back() % 2 == 0 ? 2 : 1);
  p.TPR = cluster * block;
  p.NJ = static_cast<int>((L / p.W + p.TPR - 1) / p.TPR);
  p.block = block;
  p.RPB = 1;
  return p;
}

void emit_row(Emitter& em, const CompGraph& g, const std::set<int>& pat, const Body& b,
              const StageCfg* st = nullptr, const std::vector<int>* pipe = nullptr, int cluster = 1) {
  const std::vector<int>& O = b.dims_a;
  const std::vector<int>& I = b.dims_b;
  const int64_t ROWS = prod(O), L = prod(I);
  const RowParams rp = cluster > 1 ? cluster_row_params(I, cluster, em.block) : row_params(I, em.block, b.tpr);
  em.W = rp.W;
  const int64_t nch = L / rp.W;
  const bool partial = nch % rp.TPR != 0;
  em.line("// regional body: " + std::to_string(ROWS) + " rows x " + std::to_string(L) + ", team " +
          std::to_string(rp.TPR) + " threads x " + std::to_string(rp.NJ) + " chunks x " + std::to_string(rp.W));
  if (cluster > 1)
    em.line("const int crank_ = (int)cluster_ctarank(), tl_ = crank_ * " + std::to_string(rp.block) +
            " + (int)threadIdx.x, team_ = 0;  // cluster of " + std::to_string(cluster) + " CTAs per row");
  else
    em.line("const int tl_ = threadIdx.x % " + std::to_string(rp.TPR) + ", team_ = threadIdx.x / " +
            std::to_string(rp.TPR) + ";");
  std::map<int, int> lvl_memo;
  std::map<int, std::vector<int>> levels;
  for (int r : b.reductions) levels[reduction_level(g, pat, r, lvl_memo)].push_back(r);
  const int cta_team = cluster > 1 ? rp.block : rp.TPR;  // threads of one team inside this CTA
  const int nwarps_team = cta_team > 32 ? cta_team / 32 : 1;
  size_t maxr = 0;
  for (auto& [l, rs] : levels) maxr = std::max(maxr, rs.size());
  if (cta_team > 32)
    em.line("__shared__ double red_smem_[" + std::to_string(maxr) + "][" + std::to_string(rp.block / 32) + "];");
  if (cluster > 1 && maxr) em.line("__shared__ double cl_red_[" + std::to_string(maxr) + "];");
  const std::string sRPB = std::to_string(rp.RPB), sL = std::to_string(L);
  // chunk offsets inside a row depend only on the thread: defined once,
  // outside the row loop
  std::vector<std::string> chunk_p(static_cast<size_t>(rp.NJ)), chunk_ok(static_cast<size_t>(rp.NJ));
  for (int j = 0; j < rp.NJ; ++j) {
    const std::string raw = "(tl_ + " + std::to_string(j * rp.TPR) + ") * " + std::to_string(rp.W);
    chunk_p[j] = em.fresh("p");
    if (partial) {
      chunk_ok[j] = em.fresh("pok");
      em.line("const bool " + chunk_ok[j] + " = " + raw + " < " + std::to_string(L) + ";");
      em.line("const " + em.ix() + " " + chunk_p[j] + " = " + chunk_ok[j] + " ? " + raw + " : " + std::to_string(L - rp.W) + ";");
    } else {
      em.line("const " + em.ix() + " " + chunk_p[j] + " = " + raw + ";");
    }
  }
  // row-invariant operands (a [L] tensor broadcast along the rows, e.g.
  // LayerNorm's gamma/beta): loaded once per thread before the row loop; the
  // memo hands the registers to every row.  Only where a team walks several
  // rows (the register pipeline): with one row per team it just costs
  // registers (residual+LN 7.09 -> 8.11 us; LN 4.69 -> 4.27 us pipelined,
  // profiles/r01/row_hoist_ab.jsonl)
  // With two or more streamed tensors the prefetch registers (2 x streams x
  // NJ float4) plus the hoisted operands exceed the 128-register cap of a
  // 512-thread CTA (residual+LN spilled 160 B/thread): there the operands go
  // to shared memory instead (STITCH_ROW_HOIST_BCAST: 1 registers, 2 shared
  // memory, 0 off; default 2 for >= 2 streams, else 1)
  // The TMA-staged rows (st) hoist them into shared memory as well: re-read
  // per row they were the second-largest stall in the staged LN kernel
  // (ncu source page, profiles/r02/tma/)
  const bool multi_row = (pipe && !pipe->empty() && rp.W == 4) || (st && rp.W == 4);
  const int hoist_mode = env_int("STITCH_ROW_HOIST_BCAST", st || (pipe && pipe->size() >= 2) ? 2 : 1);
  if (I.size() == 1 && multi_row && hoist_mode) {
    std::set<int> srcs;
    for (int v : pat) {
      const OpNode& n = g.node(v);
      if (n.kind != OpKind::Broadcast || pat.count(n.operands[0])) continue;
      const OpNode& src = g.node(n.operands[0]);
      if (src.kind == OpKind::Constant || src.shape.rank() != 1 || src.shape.dims[0] != L) continue;
      if (src.shape.dtype != DType::F32 || L % 4 != 0) continue;
      if (n.attrs.dims.size() != 1 || n.attrs.dims[0] != static_cast<int>(O.size())) continue;
      if (n.shape.rank() != static_cast<int>(O.size() + 1)) continue;
      srcs.insert(src.id);
    }
    for (int sid : srcs) {
      if (hoist_mode == 2) {
        if (!em.is_param(sid)) em.ensure_wait();
        const std::string nm = "sb_" + tensor_ident(g.node(sid).name);
        em.line("__shared__ __align__(16) float " + nm + "[" + sL + "];");
        em.line("for (int i_ = threadIdx.x; i_ < " + std::to_string(L / 4) + "; i_ += " + std::to_string(rp.block) +
                ") reinterpret_cast<float4*>(" + nm + ")[i_] = " + (em.is_param(sid) ? "ld4c(" : "ld4k(") +
                tensor_ident(g.node(sid).name) + " + i_ * 4);");
        em.smem_bcast[sid] = nm;
      } else {
        for (int j = 0; j < rp.NJ; ++j) em.value(sid, Coords{{chunk_p[j], rp.W > 1, true}});
      }
    }
    if (hoist_mode == 2 && !srcs.empty()) em.line("__syncthreads();");
  }
  if (st && st->team) {
    for (int v : st->tensors)
      if (!em.is_param(v)) em.ensure_wait();
    const std::string S = std::to_string(st->stages), sROWS = std::to_string(ROWS);
    const int64_t nt = static_cast<int64_t>(st->tensors.size());
    const std::string ring = std::to_string(int64_t(st->stages) * nt * L);  // floats per team
    em.line("// TMA per-team rings: " + S + " row buffers x " + std::to_string(nt) + " tensor(s) x " +
            std::to_string(L * 4) + " B per team, one mbarrier per buffer");
    em.line("unsigned long long* sbar_ = reinterpret_cast<unsigned long long*>(dsmem_) + team_ * " + S + ";");
    em.line("float* sbuf_ = reinterpret_cast<float*>(dsmem_ + " + std::to_string(st->bar_bytes) + ") + (i64)team_ * " +
            ring + ";");
    em.line("if (tl_ == 0) { for (int s = 0; s < " + S + "; ++s) mbar_init(sbar_ + s, 1); mbar_fence_init(); }");
    em.line("__syncthreads();");
    std::string issue = "auto issue_ = [&](i64 rb, int s) { const i64 r = min(rb + team_, (i64)" +
                        std::to_string(ROWS - 1) + "); mbar_expect_tx(sbar_ + s, " + std::to_string(L * 4 * nt) + "u); ";
    for (int64_t k = 0; k < nt; ++k)
      issue += "bulk_g2s(sbuf_ + (i64)(s * " + std::to_string(nt) + " + " + std::to_string(k) + ") * " + sL + ", " +
               tensor_ident(g.node(st->tensors[static_cast<size_t>(k)]).name) + " + r * " + sL + ", " +
               std::to_string(L * 4) + "u, sbar_ + s); ";
    issue += "};";
    em.line(issue);
    const std::string step = "(i64)vgrid * " + sRPB;
    em.line("if (tl_ == 0) for (int s = 0; s < " + S + "; ++s) { const i64 rb = (i64)vbid * " + sRPB + " + (i64)s * " +
            step + "; if (rb < " + sROWS + ") issue_(rb, s); }");
    em.open("for (i64 rb_ = (i64)vbid * " + sRPB + ", i_ = 0; rb_ < " + sROWS + "; rb_ += " + step + ", ++i_)");
    em.line("const int s_ = (int)(i_ % " + S + ");");
    em.line("mbar_wait(sbar_ + s_, (unsigned)((i_ / " + S + ") & 1));");
    for (int64_t k = 0; k < nt; ++k) {
      const std::string nm = em.fresh("stg");
      em.line("const float* " + nm + " = sbuf_ + (i64)(s_ * " + std::to_string(nt) + " + " + std::to_string(k) + ") * " +
              sL + ";");
      em.staged_ptr[st->tensors[static_cast<size_t>(k)]] = nm;
    }
  } else if (st) {
    // TMA-staged inputs that a kernel produces must wait; graph parameters
    // are streamed before the wait (hoisted prologue)
    for (int v : st->tensors)
      if (!em.is_param(v)) em.ensure_wait();
    const int64_t ntiles = (ROWS + rp.RPB - 1) / rp.RPB;
    const std::string S = std::to_string(st->stages), TF = std::to_string(st->tile_floats);
    const int64_t tile_bytes_full = st->tile_floats * 4;
    em.line("// TMA pipeline: " + std::to_string(ntiles) + " tiles of " + sRPB + " rows, " + S + " stages x " +
            std::to_string(st->tensors.size()) + " staged tensor(s) x " + std::to_string(tile_bytes_full) + " B");
    em.line("const int tb_ = (int)(((i64)vbid * " + std::to_string(ntiles) + ") / vgrid);");
    em.line("const int te_ = (int)(((i64)(vbid + 1) * " + std::to_string(ntiles) + ") / vgrid);");
    em.line("unsigned long long* sbar_ = reinterpret_cast<unsigned long long*>(dsmem_);");
    em.line("float* sbuf_ = reinterpret_cast<float*>(dsmem_ + 128);");
    em.line("if (threadIdx.x == 0) { for (int s = 0; s < " + S + "; ++s) mbar_init(sbar_ + s, 1); mbar_fence_init(); }");
    em.line("__syncthreads();");
    std::string issue = "auto issue_ = [&](int t, int s) { const i64 r0 = (i64)t * " + sRPB +
                        "; const unsigned rows = (unsigned)min((i64)" + sRPB + ", (i64)" + std::to_string(ROWS) +
                        " - r0); const unsigned nb = rows * " + std::to_string(L * 4) + "u; mbar_expect_tx(sbar_ + s, nb * " +
                        std::to_string(st->tensors.size()) + "u); ";
    for (size_t k = 0; k < st->tensors.size(); ++k)
      issue += "bulk_g2s(sbuf_ + (i64)s * " + std::to_string(st->tile_floats * static_cast<int64_t>(st->tensors.size())) +
               " + " + std::to_string(static_cast<int64_t>(k) * st->tile_floats) + ", " + tensor_ident(g.node(st->tensors[k]).name) +
               " + r0 * " + sL + ", nb, sbar_ + s); ";
    issue += "};";
    em.line(issue);
    em.line("if (threadIdx.x == 0) for (int s = 0; s < " + S + " && tb_ + s < te_; ++s) issue_(tb_ + s, s);");
    em.open("for (int t_ = tb_, i_ = 0; t_ < te_; ++t_, ++i_)");
    em.line("const int s_ = i_ % " + S + ";");
    em.line("mbar_wait(sbar_ + s_, (unsigned)((i_ / " + S + ") & 1));");
    em.line("const i64 rb_ = (i64)t_ * " + sRPB + ";");
    for (size_t k = 0; k < st->tensors.size(); ++k) {
      const std::string nm = em.fresh("stg");
      em.line("const float* " + nm + " = sbuf_ + (i64)s_ * " +
              std::to_string(st->tile_floats * static_cast<int64_t>(st->tensors.size())) + " + " +
              std::to_string(static_cast<int64_t>(k) * st->tile_floats) + " + team_ * " + sL + ";");
      em.staged_ptr[st->tensors[k]] = nm;
    }
  } else if (pipe && !pipe->empty() && rp.W == 4) {
    // register pipeline: every team prefetches its NEXT row of the streamed
    // inputs while it reduces and writes the current one
    for (int v : *pipe)
      if (!em.is_param(v)) em.ensure_wait();
    const std::string sROWS = std::to_string(ROWS);
    auto off = [&](int j) {
      const std::string raw = "(tl_ + " + std::to_string(j * rp.TPR) + ") * 4";
      return partial ? "(" + raw + " < " + sL + " ? " + raw + " : " + std::to_string(L - 4) + ")" : raw;
    };
    std::string decl = "float4", first;
    for (int v : *pipe)
      for (int j = 0; j < rp.NJ; ++j) {
        const std::string nm = "pf_" + tensor_ident(g.node(v).name) + "_" + std::to_string(j);
        decl += std::string(decl == "float4" ? " " : ", ") + nm;
        first += nm + " = " + (em.is_param(v) ? "ld4(" : "ld4k(") + tensor_ident(g.node(v).name) + " + r0_ * " + sL + " + " + off(j) + "); ";
      }
    em.line(decl + ";");
    em.line("{ const i64 r0_ = min((i64)vbid * " + sRPB + " + team_, (i64)" + std::to_string(ROWS - 1) + "); " + first + "}");
    em.open("for (i64 rb_ = (i64)vbid * " + sRPB + "; rb_ < " + sROWS + "; rb_ += (i64)vgrid * " + sRPB + ")");
    std::string cur = "float4", next;
    for (int v : *pipe)
      for (int j = 0; j < rp.NJ; ++j) {
        const std::string sfx = tensor_ident(g.node(v).name) + "_" + std::to_string(j);
        cur += std::string(cur == "float4" ? " " : ", ") + "cu_" + sfx + " = pf_" + sfx;
        next += "pf_" + sfx + " = " + (em.is_param(v) ? "ld4(" : "ld4k(") + tensor_ident(g.node(v).name) + " + n_ * " + sL + " + " + off(j) + "); ";
      }
    em.line("const " + cur + ";");
    em.line("{ const i64 n_ = rb_ + (i64)vgrid * " + sRPB + " + team_; if (n_ < " + sROWS + ") { " + next + "} }");
    em.reg_staged.insert(pipe->begin(), pipe->end());
  } else if (cluster > 1) {
    const std::string C = std::to_string(cluster);
    em.open("for (i64 rb_ = (i64)(vbid / " + C + "); rb_ < " + std::to_string(ROWS) + "; rb_ += (i64)(vgrid / " + C + "))");
  } else {
    em.open("for (i64 rb_ = (i64)vbid * " + sRPB + "; rb_ < " + std::to_string(ROWS) +
            "; rb_ += (i64)vgrid * " + sRPB + ")");
  }
  em.line("const bool row_ok = rb_ + team_ < " + std::to_string(ROWS) + ";");
  em.line("const " + em.ix() + " row = (" + em.ix() + ")(row_ok ? rb_ + team_ : " + std::to_string(ROWS - 1) + ");");
  Coords rowc;
  {
    auto names = decompose(em, "row", O, "o");
    for (auto& n : names) rowc.push_back({n, false, true});
  }
  std::vector<Coords> chunk_c(static_cast<size_t>(rp.NJ));
  for (int j = 0; j < rp.NJ; ++j) {
    const std::string& p = chunk_p[j];
    Coords c = rowc;
    if (I.size() == 1) {
      c.push_back({p, rp.W > 1, true});
    } else {
      auto names = decompose(em, p, I, "i");
      for (size_t a = 0; a < I.size(); ++a) c.push_back({names[a], a + 1 == I.size() && rp.W > 1, true});
    }
    c = arrange(c, b.perm);
    chunk_c[j] = c;
    if (b.perm.empty()) {  // contiguous rows only: offsets inside a staged / prefetched row
      em.domain_off[coords_key(c)] = p;
      em.domain_chunk[coords_key(c)] = j;
    }
  }
  em.domain_dims = O;
  em.domain_dims.insert(em.domain_dims.end(), I.begin(), I.end());
  // multi-domain rows: reductions / outputs on another trailing domain J of
  // the same row run as a team-strided scalar loop over J
  auto secondary = [&](const TensorShape& sh) -> std::vector<int> {
    if (!b.multi) return {};
    const auto d = dims_of(sh);
    if (d == em.domain_dims || d.size() <= O.size()) return {};
    return std::vector<int>(d.begin() + static_cast<std::ptrdiff_t>(O.size()), d.end());
  };
  auto open_secondary = [&](const std::vector<int>& J) {
    const std::string q = em.fresh("q");
    em.open("for (int " + q + " = tl_; " + q + " < " + std::to_string(prod(J)) + "; " + q + " += " +
            std::to_string(rp.TPR) + ")");
    Coords c = rowc;
    for (auto& n : decompose(em, q, J, "s")) c.push_back({n, false, true});
    return c;
  };
  for (auto& [lvl, rs] : levels) {
    // sums: compensated f32 partials per thread (kahan_add), folded to f64
    // for the cross-thread tree; max: exact in f32
    std::vector<std::string> acc, ks, kc;
    for (int r : rs) {
      const bool sum = g.node(r).kind == OpKind::ReduceSum;
      acc.push_back(em.fresh("acc"));
      ks.push_back(sum ? em.fresh("ks") : "");
      kc.push_back(sum ? em.fresh("kc") : "");
      if (sum)
        em.line("float " + ks.back() + " = 0.f, " + kc.back() + " = 0.f;");
      else
        em.line("float " + acc.back() + " = __int_as_float(0xff800000);");
    }
    std::map<std::vector<int>, std::vector<size_t>> sec_groups;
    for (size_t i = 0; i < rs.size(); ++i)
      if (auto J = secondary(g.node(g.node(rs[i]).operands[0]).shape); !J.empty()) sec_groups[J].push_back(i);
    auto is_sec = [&](size_t i) {
      for (auto& [J, idx] : sec_groups)
        if (std::count(idx.begin(), idx.end(), i)) return true;
      return false;
    };
    for (int j = 0; j < rp.NJ; ++j) {
      for (size_t i = 0; i < rs.size(); ++i) {
        const int r = rs[i];
        if (is_sec(i)) continue;
        const bool sum = g.node(r).kind == OpKind::ReduceSum;
        const Val v = em.value(g.node(r).operands[0], chunk_c[j]);
        std::string upd;
        if (sum) {  // lanes pairwise, then one compensated add per chunk
          std::string x = v.at(0);
          if (rp.W == 2) x = "(" + v.at(0) + " + " + v.at(1) + ")";
          if (rp.W == 4) x = "((" + v.at(0) + " + " + v.at(1) + ") + (" + v.at(2) + " + " + v.at(3) + "))";
          upd = "kahan_add(" + ks[i] + ", " + kc[i] + ", " + x + "); ";
        } else {
          for (int k = 0; k < rp.W; ++k) upd += acc[i] + " = op_max(" + acc[i] + ", " + v.at(k) + "); ";
        }
        em.line((partial ? "if (" + chunk_ok[j] + ") { " : "{ ") + upd + "}");
      }
    }
    for (auto& [J, idx] : sec_groups) {
      const Coords c = open_secondary(J);
      for (size_t i : idx) {
        const Val v = em.value(g.node(rs[i]).operands[0], c);
        if (g.node(rs[i]).kind == OpKind::ReduceSum)
          em.line("kahan_add(" + ks[i] + ", " + kc[i] + ", " + v.at(0) + ");");
        else
          em.line(acc[i] + " = op_max(" + acc[i] + ", " + v.at(0) + ");");
      }
      em.close();
    }
    for (size_t i = 0; i < rs.size(); ++i)
      if (!ks[i].empty()) em.line("double " + acc[i] + " = (double)" + ks[i] + " - (double)" + kc[i] + ";");
    // team reduction: butterfly inside the warp, smem across the team's warps
    // (and DSMEM across the cluster's CTAs)
    const int w = std::min(cta_team, 32);
    for (size_t i = 0; i < rs.size(); ++i) {
      const bool sum = g.node(rs[i]).kind == OpKind::ReduceSum;
      if (w > 1) em.line(acc[i] + " = " + (sum ? "bfly_sum(" : "bfly_max(") + acc[i] + ", " + std::to_string(w) + ");");
    }
    if (cta_team > 32) {
      em.line("if ((threadIdx.x & 31) == 0) {");
      for (size_t i = 0; i < rs.size(); ++i)
        em.line("  red_smem_[" + std::to_string(i) + "][threadIdx.x >> 5] = " + acc[i] + ";");
      em.line("}");
      em.line("__syncthreads();");
      for (size_t i = 0; i < rs.size(); ++i) {
        const bool sum = g.node(rs[i]).kind == OpKind::ReduceSum;
        em.line("{ const int w0_ = team_ * " + std::to_string(nwarps_team) + "; " + acc[i] +
                " = red_smem_[" + std::to_string(i) + "][w0_]; for (int q_ = 1; q_ < " +
                std::to_string(nwarps_team) + "; ++q_) " + acc[i] + " = " +
                (sum ? acc[i] + " + red_smem_[" + std::to_string(i) + "][w0_ + q_]"
                     : "op_max(" + acc[i] + ", (float)red_smem_[" + std::to_string(i) + "][w0_ + q_])") +
                "; }");
      }
      em.line("__syncthreads();");
    }
    if (cluster > 1) {  // CTA partials -> every thread folds the cluster's in rank order
      em.line("if (threadIdx.x == 0) {");
      for (size_t i = 0; i < rs.size(); ++i) em.line("  cl_red_[" + std::to_string(i) + "] = " + acc[i] + ";");
      em.line("}");
      em.line("cluster_sync_all();");
      for (size_t i = 0; i < rs.size(); ++i) {
        const bool sum = g.node(rs[i]).kind == OpKind::ReduceSum;
        const std::string src = "ld_dsmem_f64(cl_red_ + " + std::to_string(i) + ", q_)";
        em.line("{ " + acc[i] + " = ld_dsmem_f64(cl_red_ + " + std::to_string(i) + ", 0u); for (unsigned q_ = 1; q_ < " +
                std::to_string(cluster) + "u; ++q_) " + acc[i] + " = " +
                (sum ? acc[i] + " + " + src : "op_max(" + acc[i] + ", (float)" + src + ")") + "; }");
      }
      em.line("cluster_sync_all();  // every CTA read the partials before cl_red_ is reused");
    }
    for (size_t i = 0; i < rs.size(); ++i) {
      const std::string t = em.fresh("red");
      std::string e = "(float)" + acc[i];
      const DType d = g.node(rs[i]).shape.dtype;
      if (d == DType::F16) e = "rnd_f16(" + e + ")";
      em.line("const float " + t + " = " + e + ";");
      em.reduced[Emitter::key(rs[i], rowc)] = Val{{t}};
    }
  }
  // outputs
  std::map<std::vector<int>, std::vector<int>> sec_outputs;
  for (int o : b.outputs) {
    const auto& od = g.node(o).shape.dims;
    if (static_cast<int64_t>(od.size()) == static_cast<int64_t>(O.size())) {
      const Val v = em.value(o, rowc);
      em.ensure_wait();
      em.line("if (row_ok && tl_ == 0) stv(" + tensor_ident(g.node(o).name) + ", " + em.linear(o, rowc, 0) + ", " + v.at(0) + ");");
      continue;
    }
    if (auto J = secondary(g.node(o).shape); !J.empty()) {
      sec_outputs[J].push_back(o);
      continue;
    }
    for (int j = 0; j < rp.NJ; ++j) {
      const Val v = em.value(o, chunk_c[j]);
      store_val(em, g, o, chunk_c[j], v, partial ? "row_ok && " + chunk_ok[j] : "row_ok");
    }
  }
  for (auto& [J, outs] : sec_outputs) {
    const Coords c = open_secondary(J);
    for (int o : outs) store_val(em, g, o, c, em.value(o, c), "row_ok");
    em.close();
  }
  if (st && st->team) {  // the team is done with buffer s_: its lead refills it with the team's row S iterations on
    if (rp.TPR > 32)
      em.line("__syncthreads();  // team spans warps (the row loop is CTA-uniform)");
    else if (rp.TPR == 32)
      em.line("__syncwarp();");
    else
      em.line("__syncwarp(((1u << " + std::to_string(rp.TPR) + ") - 1u) << ((threadIdx.x & 31) / " +
              std::to_string(rp.TPR) + " * " + std::to_string(rp.TPR) + "));");
    em.line("if (tl_ == 0) { const i64 nb_ = rb_ + (i64)" + std::to_string(st->stages) + " * vgrid * " + sRPB +
            "; if (nb_ < " + std::to_string(ROWS) + ") { fence_proxy_async(); issue_(nb_, s_); } }");
  } else if (st) {  // every thread is done with stage s_: refill it with tile t_ + stages
    em.line("__syncthreads();");
    em.line("if (threadIdx.x == 0 && t_ + " + std::to_string(st->stages) + " < te_) { fence_proxy_async(); issue_(t_ + " +
            std::to_string(st->stages) + ", s_); }");
  }
  em.close();
  em.domain_off.clear();
  em.domain_chunk.clear();
  em.staged_ptr.clear();
  em.reg_staged.clear();
  em.smem_bcast.clear();
}

bool grid_sync_mode() {
  const char* v = std::getenv("STITCH_COL_SYNC");
  return v && std::string(v) == "grid";
}

struct ColParams {
  int W, CT, RT, NCB, RB, U;
  int64_t NCH, ROWS, COLS;
};

// CT column chunks x RT row lanes per 256-thread CTA; NCB column strips x RB
// row slabs of CTAs, sized for ~3 CTAs per SM (each slab >= RT*U rows).
// Narrow strips (CT 8 = 32 columns) keep the slab count per strip -- and so
// the last CTA's combine -- short (B200 sweep: profiles/r01/colreduce_sweep.jsonl)
ColParams col_params(const std::vector<int>& P, const std::vector<int>& C, int target_blocks, int block) {
  ColParams p;
  p.ROWS = prod(P);
  p.COLS = prod(C);
  p.W = C.back() % 4 == 0 ? 4 : 1;
  p.NCH = p.COLS / p.W;
  p.CT = static_cast<int>(pow2ceil(std::min<int64_t>(std::clamp(env_int("STITCH_COL_CT", 8), 1, 256), p.NCH)));
  p.RT = std::max(1, block / p.CT);
  p.NCB = static_cast<int>((p.NCH + p.CT - 1) / p.CT);
  p.U = std::max(1, env_int("STITCH_COL_U", 8));
  const int64_t max_rb = std::max<int64_t>(1, p.ROWS / (int64_t(p.RT) * p.U));
  p.RB = static_cast<int>(std::clamp<int64_t>(target_blocks / p.NCB, 1, max_rb));
  return p;
}

// global body: each CTA folds its row slab of one column strip into per-column
// f64 partials (compensated f32 per thread, fixed-order smem tree across the
// CTA), writes them to scratch, and the LAST CTA of the strip to arrive
// (threadfence + atomic arrival counter) combines all slabs in slab order and
// runs the column consumers.  Deterministic, no co-residency requirement, no
// CTA ever waits at a barrier.
void emit_column(Emitter& em, const CompGraph& g, const Body& b, const ColParams& cp, int64_t partial_off,
                 int64_t ctr_off, int bar_slot = 0) {
  const std::vector<int>& P = b.dims_a;
  const std::vector<int>& C = b.dims_b;
  em.W = cp.W;
  const std::string sW = std::to_string(cp.W), sCOLS = std::to_string(cp.COLS), sRB = std::to_string(cp.RB);
  em.line("// global body: " + std::to_string(cp.ROWS) + " reduced rows x " + sCOLS + " columns; CTA tile " +
          std::to_string(cp.CT * cp.W) + " cols x " + std::to_string(cp.RT) + " rows, " + sRB + " slabs per strip");
  em.line("const int cx_ = threadIdx.x % " + std::to_string(cp.CT) + ", ry_ = threadIdx.x / " + std::to_string(cp.CT) + ";");
  em.line("const int cb_ = vbid % " + std::to_string(cp.NCB) + ", rbk_ = vbid / " + std::to_string(cp.NCB) + ";");
  em.line("const bool col_ok = cb_ * " + std::to_string(cp.CT) + " + cx_ < " + std::to_string(cp.NCH) + ";");
  em.line("const " + em.ix() + " ch_ = col_ok ? cb_ * " + std::to_string(cp.CT) + " + cx_ : " + std::to_string(cp.NCH - 1) + ";");
  em.line("const i64 rspan_ = (" + std::to_string(cp.ROWS) + " + " + sRB + " - 1) / " + sRB + ";");
  em.line("const i64 r0_ = (i64)rbk_ * rspan_, r1_ = min((i64)" + std::to_string(cp.ROWS) + ", r0_ + rspan_);");
  Coords colc;
  {
    const std::string lin = cp.W == 1 ? "ch_" : "ch_ * " + sW;
    auto names = decompose(em, lin, C, "c");
    for (size_t i = 0; i < C.size(); ++i) colc.push_back({names[i], i + 1 == C.size() && cp.W > 1, true});
  }
  const size_t nr = b.reductions.size();
  std::vector<std::vector<std::string>> acc(nr), kc(nr);
  for (size_t i = 0; i < nr; ++i) {
    const bool sum = g.node(b.reductions[i]).kind == OpKind::ReduceSum;
    for (int k = 0; k < cp.W; ++k) {
      acc[i].push_back(em.fresh("acc"));
      kc[i].push_back(sum ? em.fresh("kc") : "");
      if (sum)
        em.line("float " + acc[i].back() + " = 0.f, " + kc[i].back() + " = 0.f;");
      else
        em.line("float " + acc[i].back() + " = __int_as_float(0xff800000);");
    }
  }
  em.open("for (i64 r_ = r0_ + ry_; r_ < r1_; r_ += " + std::to_string(cp.RT * cp.U) + ")");
  std::vector<std::tuple<int, Coords, Val, std::string>> stores;
  for (int u = 0; u < cp.U; ++u) {
    const std::string ok = em.fresh("ok"), rr = em.fresh("rr");
    em.line("const bool " + ok + " = r_ + " + std::to_string(u * cp.RT) + " < r1_;");
    em.line("const " + em.ix() + " " + rr + " = (" + em.ix() + ")(" + ok + " ? r_ + " + std::to_string(u * cp.RT) + " : r_);");
    Coords c;
    auto names = decompose(em, rr, P, "r");
    for (auto& n : names) c.push_back({n, false, true});
    c.insert(c.end(), colc.begin(), colc.end());
    c = arrange(c, b.perm);
    for (size_t i = 0; i < nr; ++i) {
      const int r = b.reductions[i];
      const bool sum = g.node(r).kind == OpKind::ReduceSum;
      const Val v = em.value(g.node(r).operands[0], c);
      std::string upd;
      for (int k = 0; k < cp.W; ++k)
        upd += sum ? "kahan_add(" + acc[i][k] + ", " + kc[i][k] + ", " + v.at(k) + "); "
                   : acc[i][k] + " = op_max(" + acc[i][k] + ", " + v.at(k) + "); ";
      em.line("if (" + ok + ") { " + upd + "}");
    }
    for (int o : b.outputs)
      if (g.node(o).shape.rank() == static_cast<int>(P.size() + C.size()))
        stores.emplace_back(o, c, em.value(o, c), "col_ok && " + ok);
  }
  for (auto& [o, c, v, ok] : stores) store_val(em, g, o, c, v, ok);
  em.close();
  if (!nr) return;
  em.ensure_wait();  // slab partials / arrival counters are global writes
  // fold the RT row lanes of the tile in smem (fixed order) -> slab partials
  const std::string tile = em.fresh("tile_");
  em.line("__shared__ double " + tile + "[" + std::to_string(cp.RT) + "][" + std::to_string(cp.CT * cp.W) + "];");
  auto part = [&](size_t i, const std::string& slab, const std::string& k) {
    return "part_[" + std::to_string(partial_off + static_cast<int64_t>(i) * cp.RB * cp.COLS) + " + (i64)(" + slab +
           ") * " + sCOLS + " + (i64)ch_ * " + sW + " + " + k + "]";
  };
  for (size_t i = 0; i < nr; ++i) {
    const bool sum = g.node(b.reductions[i]).kind == OpKind::ReduceSum;
    for (int k = 0; k < cp.W; ++k)
      em.line(tile + "[ry_][cx_ * " + sW + " + " + std::to_string(k) + "] = " +
              (sum ? "(double)" + acc[i][k] + " - (double)" + kc[i][k] : acc[i][k]) + ";");
    em.line("__syncthreads();");
    em.open("if (ry_ == 0 && col_ok)");
    for (int k = 0; k < cp.W; ++k) {
      const std::string col = "cx_ * " + sW + " + " + std::to_string(k);
      em.line("{ double s_ = " + tile + "[0][" + col + "]; for (int q_ = 1; q_ < " + std::to_string(cp.RT) +
              "; ++q_) s_ = " + (sum ? "s_ + " + tile + "[q_][" + col + "]" : "dmax(s_, " + tile + "[q_][" + col + "])") +
              "; " + part(i, "rbk_", std::to_string(k)) + " = s_; }");
    }
    em.close();
    em.line("__syncthreads();");
  }
  // last-arriving CTA of this column strip combines the slabs in order
  // (STITCH_COL_SYNC=grid: the north star's cooperative variant -- a
  // grid-wide barrier, then the first slab CTA of each strip combines;
  // measured slower, profiles/r01/colreduce_sync_ab.jsonl)
  const std::string last = em.fresh("last_");
  em.line("__shared__ unsigned " + last + ";");
  if (grid_sync_mode()) {
    // this body's own barrier words (the scratch header's first 64 words)
    // and its own CTA count: in a packed kernel the other bodies' CTAs never
    // arrive here
    em.line("grid_sync(bar_ + " + std::to_string(2 * bar_slot) + ", (unsigned)vgrid);");
    em.line("if (threadIdx.x == 0) " + last + " = rbk_ == 0;");
  } else {
    em.line("__threadfence();");
    em.line("__syncthreads();");
    em.line("if (threadIdx.x == 0) " + last + " = atomicAdd(bar_ + " + std::to_string(ctr_off) + " + cb_, 1u) == " +
            std::to_string(cp.RB - 1) + "u;");
  }
  em.line("__syncthreads();");
  em.open("if (" + last + ")");
  em.line("__threadfence();");
  const int64_t strip_cols = int64_t(cp.CT) * cp.W;
  {
    // every thread of the CTA folds one (reduction, column) pair of the strip
    // over the slabs in slab order (loads independent, adds in fixed order:
    // deterministic, same bits as a serial fold), then the strip's column
    // threads read the folded values back from shared memory
    const std::string cred = em.fresh("cred_");
    em.line("__shared__ float " + cred + "[" + std::to_string(nr) + "][" + std::to_string(strip_cols) + "];");
    em.open("for (int q_ = threadIdx.x; q_ < " + std::to_string(int64_t(nr) * strip_cols) + "; q_ += " +
            std::to_string(em.block) + ")");
    em.line("const int ri_ = q_ / " + std::to_string(strip_cols) + ", cl_ = q_ % " + std::to_string(strip_cols) + ";");
    em.line("const i64 col_ = (i64)cb_ * " + std::to_string(strip_cols) + " + cl_;");
    em.line("if (col_ >= " + sCOLS + ") continue;");
    for (size_t i = 0; i < nr; ++i) {
      const int r = b.reductions[i];
      const bool sum = g.node(r).kind == OpKind::ReduceSum;
      const std::string base = "part_ + " + std::to_string(partial_off + static_cast<int64_t>(i) * cp.RB * cp.COLS) + " + col_";
      std::string e = "(float)s_";
      if (g.node(r).shape.dtype == DType::F16) e = "rnd_f16(" + e + ")";
      em.line(std::string(i ? "else " : "") + "if (ri_ == " + std::to_string(i) + ") { const double* p_ = " + base +
              "; double s_ = __ldcg(p_);\n" + em.ind + "  #pragma unroll 8\n" + em.ind + "  for (int k_ = 1; k_ < " + sRB +
              "; ++k_) s_ = " + (sum ? "s_ + __ldcg(p_ + (i64)k_ * " + sCOLS + ")" : "dmax(s_, __ldcg(p_ + (i64)k_ * " + sCOLS + "))") +
              ";\n" + em.ind + "  " + cred + "[" + std::to_string(i) + "][cl_] = " + e + "; }");
    }
    em.close();
    em.line("__syncthreads();");
    em.open("if (ry_ == 0 && col_ok)");
    for (size_t i = 0; i < nr; ++i) {
      Val v;
      for (int k = 0; k < cp.W; ++k)
        v.lanes.push_back(cred + "[" + std::to_string(i) + "][cx_ * " + sW + " + " + std::to_string(k) + "]");
      em.reduced[Emitter::key(b.reductions[i], colc)] = v;
    }
  }
  for (int o : b.outputs)
    if (g.node(o).shape.dims == to64(C)) store_val(em, g, o, colc, em.value(o, colc), "");
  em.close();
  em.line("if (threadIdx.x == 0) bar_[" + std::to_string(ctr_off) + " + cb_] = 0u;  // re-arm for the next launch");
  em.close();
}

}  // namespace

KernelSpec generate_pattern_kernel(const CompGraph& g, const std::vector<int>& verts,
                                   const std::string& name, int sm_count) {
  const SmScope sm_scope(sm_count);
  const std::set<int> pat(verts.begin(), verts.end());
  std::map<int, bool> dmemo;
  std::vector<Body> bodies;
  auto add_body = [&](Body nb) {
    for (auto& b : bodies)
      if (b.kind == nb.kind && b.dims_a == nb.dims_a && b.dims_b == nb.dims_b && b.perm == nb.perm) {
        b.outputs.insert(b.outputs.end(), nb.outputs.begin(), nb.outputs.end());
        b.reductions.insert(b.reductions.end(), nb.reductions.begin(), nb.reductions.end());
        b.multi = b.multi || nb.multi;
        b.tpr = std::max(b.tpr, nb.tpr);
        std::sort(b.reductions.begin(), b.reductions.end());
        return;
      }
    bodies.push_back(std::move(nb));
  };
  for (const Component& comp : components_of(g, verts)) {
    if (comp.reductions.empty()) {
      for (int o : comp.outputs) add_body({Kind::Local, dims_of(g.node(o).shape), {}, {o}, {}});
      continue;
    }
    // every reduction of the component must reduce the same axes of
    // operands of the same shape; the last axis decides the mapping: reduced
    // -> regional rows (contiguous along the last axis), kept -> global
    // columns.  Suffix / prefix axis sets are the identity layouts.
    std::vector<int> in0, axes0;
    bool multi = false;
    for (size_t i = 0; i < comp.reductions.size(); ++i) {
      const OpNode& r = g.node(comp.reductions[i]);
      const auto in = dims_of(g.node(r.operands[0]).shape);
      std::set<int> ax(r.attrs.axes.begin(), r.attrs.axes.end());
      std::vector<int> axes(ax.begin(), ax.end());
      if (i == 0) {
        in0 = in, axes0 = axes;
      } else if (in != in0 || axes != axes0) {
        multi = true;
      }
    }
    if (multi) {
      // rows of one split, several trailing domains: every reduction must
      // reduce a suffix of its operand's axes with the same kept prefix O;
      // the largest trailing domain is the primary one
      auto suffix_split = [&](int r, std::vector<int>& O, std::vector<int>& I) {
        const OpNode& n = g.node(r);
        const auto in = dims_of(g.node(n.operands[0]).shape);
        std::set<int> ax(n.attrs.axes.begin(), n.attrs.axes.end());
        const int k = static_cast<int>(in.size()) - static_cast<int>(ax.size());
        for (int a = 0; a < static_cast<int>(in.size()); ++a)
          if (ax.count(a) != (a >= k ? 1u : 0u)) return false;
        O.assign(in.begin(), in.begin() + k);
        I.assign(in.begin() + k, in.end());
        return !I.empty();
      };
      std::vector<int> O0, Ibest;
      for (size_t i = 0; i < comp.reductions.size(); ++i) {
        std::vector<int> O, I;
        if (!suffix_split(comp.reductions[i], O, I)) throw TemplateMismatch("reductions of one component disagree on their split");
        if (i == 0) O0 = O;
        if (O != O0) throw TemplateMismatch("reductions of one component disagree on their rows");
        if (Ibest.empty() || prod(I) > prod(Ibest)) Ibest = I;
      }
      in0 = O0;
      in0.insert(in0.end(), Ibest.begin(), Ibest.end());
      axes0.clear();
      for (size_t a = O0.size(); a < in0.size(); ++a) axes0.push_back(static_cast<int>(a));
    }
    const int n = static_cast<int>(in0.size());
    std::vector<int> kept, red;
    for (int a = 0; a < n; ++a) (std::count(axes0.begin(), axes0.end(), a) ? red : kept).push_back(a);
    const bool row_kind = n > 0 && std::count(axes0.begin(), axes0.end(), n - 1);
    Body body;
    body.kind = row_kind ? Kind::Row : Kind::Column;
    body.reductions = comp.reductions;
    const std::vector<int>& first = row_kind ? kept : red;
    const std::vector<int>& second = row_kind ? red : kept;
    for (int a : first) body.dims_a.push_back(in0[static_cast<size_t>(a)]);
    for (int a : second) body.dims_b.push_back(in0[static_cast<size_t>(a)]);
    body.perm = first;
    body.perm.insert(body.perm.end(), second.begin(), second.end());
    bool identity = true;
    for (int a = 0; a < n; ++a) identity = identity && body.perm[static_cast<size_t>(a)] == a;
    if (identity) body.perm.clear();
    if (body.kind == Kind::Column && body.dims_b.empty()) throw TemplateMismatch("column body without kept axes");
    if (multi && !identity) throw TemplateMismatch("multi-domain rows need trailing reductions");
    const std::vector<int>& full = in0;  // operand shape, tensor axis order
    const std::vector<int>& unit = body.kind == Kind::Row ? body.dims_a : body.dims_b;
    // row-aligned: dims = O ++ J for another trailing domain J of the same rows
    auto row_aligned = [&](const std::vector<int>& od) {
      return body.kind == Kind::Row && identity && od.size() > body.dims_a.size() &&
             std::equal(body.dims_a.begin(), body.dims_a.end(), od.begin());
    };
    for (int o : comp.outputs) {
      const auto od = dims_of(g.node(o).shape);
      const bool dep = downstream_of_reduction(g, pat, o, dmemo);
      if (od == full && (body.kind == Kind::Row || !dep)) {
        body.outputs.push_back(o);
      } else if (od == unit && (dep || body.kind == Kind::Row)) {
        body.outputs.push_back(o);
      } else if (!dep) {
        add_body({Kind::Local, od, {}, {o}, {}});
      } else if (row_aligned(od)) {
        body.outputs.push_back(o);
        multi = true;
      } else {
        throw TemplateMismatch("output " + g.node(o).name + " does not fit the reduction domain");
      }
    }
    if (multi) {
      // team size: enough lanes for the widest domain (scalar elements on
      // the secondary ones), within one warp so team reductions stay shuffles
      const int64_t rows = std::max<int64_t>(1, prod(body.dims_a));
      int64_t widest = prod(body.dims_b) / row_params(body.dims_b).W;
      auto widen = [&](const TensorShape& sh) {
        if (dims_of(sh) != full && dims_of(sh) != unit) widest = std::max<int64_t>(widest, sh.element_count() / rows);
      };
      for (int r : body.reductions) widen(g.node(g.node(r).operands[0]).shape);
      for (int o : body.outputs) widen(g.node(o).shape);
      body.multi = true;
      body.tpr = static_cast<int>(std::clamp<int64_t>(pow2ceil(widest), row_params(body.dims_b).TPR, 32));
      if (row_params(body.dims_b).TPR > 32) body.tpr = 0;
    }
    add_body(std::move(body));
  }

  // index width: 32-bit unless some tensor reaches 2^31 elements
  bool wide = false;
  for (int v : verts) {
    wide = wide || g.node(v).shape.element_count() >= (int64_t(1) << 31);
    for (int o : g.node(v).operands) wide = wide || g.node(o).shape.element_count() >= (int64_t(1) << 31);
  }
  Emitter em(g, pat, wide);
  // broadcast sources re-read by many threads go through L1
  for (int v : verts)
    if (g.node(v).kind == OpKind::Broadcast) {
      const int s = g.node(v).operands[0];
      if (!pat.count(s)) em.cached_tensors.insert(s);
    }

  // A row body packed beside a local body (bert_cut: residual+LN next to
  // bias+GELU) spreads each long row over more lanes -- 2 float4 chunks per
  // thread (STITCH_PACKED_ROW_NJ) instead of ~8 -- so the shared CTA holds
  // 32 registers per thread (55 at 6 chunks: the row's values are live
  // across both reductions) and the local body runs at full occupancy:
  // bert_cut 22.55 -> 21.86 us batched (profiles/r02/rows/cut_nj.jsonl)
  {
    bool has_local = false;
    for (const auto& b : bodies) has_local = has_local || b.kind == Kind::Local;
    const int nj = env_int("STITCH_PACKED_ROW_NJ", 2);
    if (has_local && bodies.size() > 1 && nj > 0)
      for (auto& b : bodies)
        if (b.kind == Kind::Row && !b.multi && b.tpr == 0) {
          const RowParams rp0 = row_params(b.dims_b);
          if (rp0.TPR < 32) continue;
          const int64_t nch = prod(b.dims_b) / rp0.W;
          b.tpr = static_cast<int>(std::clamp<int64_t>(pow2ceil((nch + nj - 1) / nj), 32, 1024));
        }
  }
  // one CTA size for every body of the kernel: a multiple of every row team
  int block = kBlock, max_tpr = 1;
  bool has_col = false;
  for (const auto& b : bodies) {
    has_col = has_col || b.kind == Kind::Column;
    if (b.kind == Kind::Row) max_tpr = std::max(max_tpr, row_params(b.dims_b, 0, b.tpr).TPR);
  }
  block = std::max(block, max_tpr);
  // long rows (a warp or more per row) stream through a register pipeline
  // (each team prefetches its next row while it reduces and writes the
  // current one, 2 rows per team) in 256-thread CTAs (B200 sweeps,
  // profiles/r01/row_pipe_sweep.jsonl: LN 5.39 -> 4.88 us, residual+LN
  // 7.36 -> 7.15 us); short rows keep 256-thread CTAs without the pipeline
  // (a kernel that packs other bodies keeps small 2-team CTAs and no
  // pipeline: its register allocation is shared with those bodies -- bias+GELU
  // packed with residual+LN runs 23 us that way vs 36 us pipelined)
  bool any_multi = false;
  for (const auto& b : bodies) any_multi = any_multi || b.multi;
  const bool long_rows = max_tpr >= 32 && !has_col && !any_multi;
  const bool single_row_body = long_rows && bodies.size() == 1;
  if (long_rows) block = std::min(1024, single_row_body ? std::max(256, 2 * max_tpr) : 2 * max_tpr);
  if (single_row_body && max_tpr == 32) {
    // pipelined rows with hoisted broadcasts: the CTA size that balances the
    // prefetch registers against resident CTAs depends on how many tensors
    // stream per row (B200 sweep, profiles/r01/row_hoist_ab.jsonl: LN with
    // one stream 128 threads, residual+LN with two 512)
    em.block = block;
    em.out.str("");
    em.clear_memo();
    em.reduced.clear();
    em.staged_hits.clear();
    em.reset_wait();
    emit_row(em, g, pat, bodies[0]);
    em.reset_wait();
    int streams = 0;
    for (int v : em.staged_hits) streams += !pat.count(v) && g.node(v).shape.dtype == DType::F32;
    // balanced: k CTAs per SM (STITCH_ROW_CTAS_PER_SM, default 2) sized so
    // the grid covers every SM with the same number of row teams (+-1): for
    // 4096 rows, 2 rows per team, 7 teams = 224 threads x 293 CTAs instead
    // of 128 x 512 (3 or 4 CTAs per SM) or 512 x 128 (20 SMs idle).  The
    // prefetch registers cap a CTA at 512 threads (128 registers each).
    // =0: the earlier fixed sizes (one stream 128, two streams 512)
    const int k_sm = env_int("STITCH_ROW_CTAS_PER_SM", 2);
    if (k_sm > 0) {
      const int64_t rows = prod(bodies[0].dims_a);
      const int64_t teams = (rows + 1) / 2;  // the register pipeline's 2 rows per team
      const int64_t per_cta = (teams + int64_t(sm_now()) * k_sm - 1) / (int64_t(sm_now()) * k_sm);
      block = static_cast<int>(std::clamp<int64_t>(per_cta * max_tpr, std::max(64, max_tpr), std::max(512, max_tpr)));
    } else {
      if (streams == 1) block = 128;
      if (streams == 2) block = 512;
    }
  }
  if (const int want = env_int("STITCH_ROW_BLOCK", 0); want > 0) {
    block = std::clamp((std::max(want, max_tpr) + max_tpr - 1) / max_tpr * max_tpr, 32, 1024);
  } else if (want < 0 && bodies.size() == 1 && bodies[0].kind == Kind::Row) {
    // balanced: the fewest CTAs per SM whose row share fits one CTA, so every
    // SM gets the same number of rows (+-1)
    const int64_t rows = prod(bodies[0].dims_a);
    for (int64_t k = 1; k <= 32; ++k) {
      const int64_t rpc = (rows + sm_now() * k - 1) / (sm_now() * k);
      if (rpc * max_tpr <= 1024) {
        block = static_cast<int>(std::max<int64_t>(32, rpc * max_tpr));
        break;
      }
    }
  }
  // regional-cluster: a single row body with too few rows to fill the GPU
  // (fewer row teams than SMs) and long rows spreads each row over a
  // thread-block cluster (<= 16 CTAs, DSMEM team reduction) so ROWS x C CTAs
  // share the row stream
  int cluster = 1;
  if (bodies.size() == 1 && bodies[0].kind == Kind::Row && !bodies[0].multi && env_int("STITCH_ROW_CLUSTER", 1) != 0) {
    const RowParams rp = row_params(bodies[0].dims_b, block, bodies[0].tpr);
    const int64_t rows = prod(bodies[0].dims_a), nch = prod(bodies[0].dims_b) / rp.W;
    const int64_t ntiles = (rows + rp.RPB - 1) / rp.RPB;
    if (ntiles < sm_now() && nch >= 512) {
      int c = 2;
      while (c < 16 && rows * c < 2 * sm_now()) c *= 2;
      const int b2 = static_cast<int>(std::clamp<int64_t>(pow2ceil((nch + int64_t(c) * 4 - 1) / (int64_t(c) * 4)), 128, 1024));
      if ((nch + int64_t(c) * b2 - 1) / (int64_t(c) * b2) <= 16 && int64_t(c) * b2 <= nch) {
        cluster = c;
        block = b2;
      }
    }
  }
  if (tl_force_block > 0) {
    for (const auto& b : bodies)
      if (b.kind == Kind::Row && row_params(b.dims_b, 0, b.tpr).TPR > tl_force_block)
        throw TemplateMismatch("resident: row team wider than the CTA");
    block = tl_force_block;
    cluster = 1;
  }
  em.block = block;
  em.hoist = tl_force_block == 0 && env_int("STITCH_PDL", 1) != 0 && env_int("STITCH_PDL_HOIST", 1) != 0;
  const int per_sm = std::max(1, std::min(env_int("STITCH_COL_CTAS", 3), 2048 / block));

  // local CTAs per SM: 32 by default; packed beside a row body, as many as
  // are resident at once (2048 threads / CTA size: 8 x 256 threads with the
  // 2-chunk rows above, 21.86 vs 22.89 us at 32; 18 for 64-thread CTAs
  // carrying a 6-chunk row body's 55 registers, 22.80 -> 22.56 us), so the
  // local grid-stride CTAs take their passes without a partial second wave
  // (profiles/r02/rows/bert_cut_sweep.jsonl, cut_nj.jsonl)
  bool has_row = false;
  for (const auto& b : bodies) has_row = has_row || b.kind == Kind::Row;
  const int local_ctas = bodies.size() > 1 && has_row ? (block == 64 ? 18 : std::clamp(2048 / block, 1, 32)) : 32;
  // CTA budget per body; scratch = [256 B reserved][strip arrival counters][f64 partials]
  int64_t part_words = 0, ctr_words = 64, dyn_smem = 0;
  std::vector<StageCfg> stage(bodies.size());
  std::vector<std::vector<int>> pipe(bodies.size());
  std::vector<ColParams> cps(bodies.size());
  std::vector<int64_t> part_off(bodies.size(), 0), ctr_off(bodies.size(), 0);
  for (size_t i = 0; i < bodies.size(); ++i) {
    Body& b = bodies[i];
    if (b.kind == Kind::Local) {
      const int64_t N = prod(b.dims_a);
      const int w = local_width(b.dims_a);
      const int64_t chunks = N / w;
      const int U = local_small(N) ? 1 : local_unroll(chunks, block);
      b.blocks = static_cast<int>(std::clamp<int64_t>((chunks + int64_t(block) * U - 1) / (int64_t(block) * U), 1,
                                                      int64_t(sm_now()) * std::max(1, env_int("STITCH_LOCAL_CTAS", local_ctas))));
    } else if (b.kind == Kind::Row && cluster > 1) {
      const int64_t rows = prod(b.dims_a);
      b.blocks = static_cast<int>(std::min<int64_t>(rows, std::max<int64_t>(1, 4 * sm_now() / cluster)) * cluster);
    } else if (b.kind == Kind::Row) {
      const RowParams rp = row_params(b.dims_b, block, b.tpr);
      const int64_t rows = prod(b.dims_a), L = prod(b.dims_b), ntiles = (rows + rp.RPB - 1) / rp.RPB;
      b.blocks = static_cast<int>(std::clamp<int64_t>(ntiles, 1, int64_t(sm_now()) * env_int("STITCH_ROW_CTAS", 16)));
      // dry run: which inputs does the body read at its own (row, chunk)
      // coordinates?  Those can be streamed a row ahead in registers
      // (default, STITCH_ROW_PIPE >= 2 rows per team) or through the opt-in
      // TMA pipeline (STITCH_STAGE=1: measured slower)
      const int pipe_rows = env_int("STITCH_ROW_PIPE", single_row_body ? 2 : 1);
      if ((env_int("STITCH_STAGE", 0) || pipe_rows > 1) && rp.W == 4 && cluster == 1 && !b.multi) {
        em.out.str("");
        em.clear_memo();
        em.reduced.clear();
        em.staged_hits.clear();
        em.reset_wait();
        emit_row(em, g, pat, b);
        em.reset_wait();
        std::vector<int> hits;
        for (int v : em.staged_hits)
          if (!pat.count(v) && g.node(v).shape.dtype == DType::F32) hits.push_back(v);
        // up to two streamed tensors per team row (2 x NJ float4 registers
        // each); beyond that the register pressure costs more than the
        // prefetch hides
        const bool pipe_ok = hits.size() <= 2 || env_int("STITCH_ROW_PIPE", 0) > 1;
        if (!hits.empty() && !env_int("STITCH_STAGE", 0) && pipe_ok) {
          pipe[i] = hits;
          b.blocks = static_cast<int>(std::clamp<int64_t>((ntiles + pipe_rows - 1) / pipe_rows, 1,
                                                          int64_t(sm_now()) * env_int("STITCH_ROW_CTAS", 16)));
        } else if (!hits.empty() && env_int("STITCH_STAGE", 0)) {
          StageCfg& sc = stage[i];
          sc.tensors = hits;
          sc.stages = std::max(2, env_int("STITCH_STAGES", 3));
          sc.tile_floats = int64_t(rp.RPB) * L;
          sc.team = env_int("STITCH_STAGE", 0) == 2;
          auto bar_bytes = [&](int s) { return sc.team ? std::max<int64_t>(128, (int64_t(rp.RPB) * s * 8 + 127) / 128 * 128) : 128; };
          // keep >= 2 CTAs per SM: fewer stages when several tensors are staged
          const int64_t smem_cap = int64_t(env_int("STITCH_STAGE_SMEM_KB", 110)) * 1024;
          while (sc.stages > 2 && bar_bytes(sc.stages) + int64_t(sc.stages) * static_cast<int64_t>(hits.size()) * sc.tile_floats * 4 >
                                      smem_cap)
            --sc.stages;
          sc.bar_bytes = bar_bytes(sc.stages);
          sc.bytes = sc.bar_bytes + int64_t(sc.stages) * static_cast<int64_t>(hits.size()) * sc.tile_floats * 4;
          if (sc.bytes <= 200 * 1024) {
            // (less the row-invariant operands hoisted into static smem, ~2 rows)
            const int64_t fit = std::clamp<int64_t>((int64_t(220 * 1024) - 2 * L * 4) / sc.bytes, 1, 2048 / rp.block);
            b.blocks = static_cast<int>(std::min<int64_t>(ntiles, sm_now() * fit));
            dyn_smem = std::max(dyn_smem, sc.bytes);
          } else {
            sc.tensors.clear();  // a tile set this large would starve occupancy: stay in registers
          }
        }
      }
    } else {
      cps[i] = col_params(b.dims_a, b.dims_b, sm_now() * per_sm, block);
      b.blocks = cps[i].NCB * cps[i].RB;
      ctr_off[i] = ctr_words;
      ctr_words += cps[i].NCB;
      part_off[i] = part_words;
      part_words += static_cast<int64_t>(b.reductions.size()) * cps[i].RB * cps[i].COLS;
    }
  }
  const int64_t header = ((ctr_words * 4 + 255) / 256) * 256;

  std::ostringstream body_src;
  int start = 0, col_slot = 0;
  const bool interleave = bodies.size() > 1 && env_int("STITCH_INTERLEAVE", 0) != 0;
  for (size_t i = 0; i < bodies.size(); ++i) {
    const Body& b = bodies[i];
    em.out.str("");
    em.ind = "    ";
    em.clear_memo();
    em.reduced.clear();
    em.reset_wait();
    if (b.kind == Kind::Local) emit_local(em, g, b);
    else if (b.kind == Kind::Row)
      emit_row(em, g, pat, b, stage[i].tensors.empty() ? nullptr : &stage[i], pipe[i].empty() ? nullptr : &pipe[i],
               cluster);
    else emit_column(em, g, b, cps[i], part_off[i], ctr_off[i], col_slot++);
    em.ensure_wait();  // every path waits before the CTA retires
    if (interleave) {
      body_src << "  " << (i ? "else " : "") << "if (body_ == " << i << ") {\n";
      body_src << "    const int vbid = (int)vb_, vgrid = " << b.blocks << ";\n";
    } else {
      body_src << "  " << (i ? "else " : "") << "if (blockIdx.x < " << start + b.blocks << ") {\n";
      body_src << "    const int vbid = blockIdx.x - " << start << ", vgrid = " << b.blocks << ";\n";
    }
    body_src << "    (void)vbid; (void)vgrid;\n" << em.out.str() << "  }\n";
    start += b.blocks;
  }
  if (interleave) {
    // STITCH_INTERLEAVE=1: packed bodies interleaved in proportion to their
    // CTA counts (body k takes floor((b+1) n_k / N_k) - floor(b n_k / N_k) of
    // the blocks left by bodies < k) so every body progresses at the same
    // rate.  Parity-green but measured slightly slower on bert_cut (24.0 vs
    // 23.6 us, profiles/r01/interleave_ab.jsonl): contiguous ranges are the default
    std::ostringstream pro;
    pro << "  unsigned b_ = blockIdx.x, vb_ = 0;\n  int body_ = " << bodies.size() - 1 << ";\n";
    int64_t remaining = start;
    std::string ind = "  ";
    for (size_t i = 0; i + 1 < bodies.size(); ++i) {
      const int64_t n = bodies[i].blocks;
      pro << ind << "{ const unsigned long long lo_ = (unsigned long long)b_ * " << n << "ull / " << remaining
          << "ull, hi_ = (unsigned long long)(b_ + 1) * " << n << "ull / " << remaining << "ull;\n";
      pro << ind << "  if (hi_ > lo_) { body_ = " << i << "; vb_ = (unsigned)lo_; } else { b_ -= (unsigned)hi_;\n";
      ind += "    ";
      remaining -= n;
    }
    pro << ind << "vb_ = b_;\n";
    for (size_t i = 0; i + 1 < bodies.size(); ++i) {
      ind.resize(ind.size() - 4);
      pro << ind << "} }\n";
    }
    body_src.str(pro.str() + body_src.str());
  }

  KernelSpec k;
  k.name = name;
  k.tmpl = bodies.size() > 1 ? "independent" : bodies[0].kind == Kind::Local ? "local"
                                             : bodies[0].kind == Kind::Row ? "regional" : "global";
  if (bodies.size() > 1) {
    k.tmpl += "(";
    for (size_t i = 0; i < bodies.size(); ++i)
      k.tmpl += std::string(i ? "+" : "") +
                (bodies[i].kind == Kind::Local ? "local" : bodies[i].kind == Kind::Row ? "regional" : "global");
    k.tmpl += ")";
  }
  k.grid = start;
  k.block = block;
  k.cooperative = has_col && grid_sync_mode();
  k.cluster = cluster;
  if (cluster > 1) k.tmpl += "-cluster" + std::to_string(cluster);
  k.smem = dyn_smem;
  k.alg_bytes = algorithmic_bytes(g, verts);
  for (size_t i = 0; i < bodies.size(); ++i)
    if (!stage[i].tensors.empty()) k.tmpl += "+tma";
  std::set<int> outs;
  for (const auto& b : bodies) outs.insert(b.outputs.begin(), b.outputs.end());
  std::ostringstream sig;
  sig << "extern \"C\" __global__ void __launch_bounds__(" << block << (has_col ? ", " + std::to_string(per_sm) : "")
      << ") " << name << "(";
  bool first = true;
  for (int v : em.loaded) {
    sig << (first ? "" : ", ") << "const " << c_type(g.node(v).shape.dtype) << "* __restrict__ " << tensor_ident(g.node(v).name);
    first = false;
    k.inputs.push_back(g.node(v).name);
  }
  for (int v : outs) {
    sig << (first ? "" : ", ") << c_type(g.node(v).shape.dtype) << "* __restrict__ " << tensor_ident(g.node(v).name);
    first = false;
    k.outputs.push_back(g.node(v).name);
  }
  if (has_col) {
    sig << (first ? "" : ", ") << "unsigned* __restrict__ bar_, double* __restrict__ part_";
    k.scratch_header = header;
    k.scratch_bytes = header + part_words * 8;
  }
  sig << ") {\n";
  if (dyn_smem) sig << "  extern __shared__ __align__(128) unsigned char dsmem_[];\n";
  // programmatic dependent launch: hoisted prologue (parameter loads before
  // griddepcontrol.wait, Emitter::ensure_wait) unless STITCH_PDL_HOIST=0,
  // which waits at entry and triggers dependents at exit
  const bool pdl = tl_force_block == 0 && env_int("STITCH_PDL", 1) != 0;
  const bool hoist = pdl && env_int("STITCH_PDL_HOIST", 1) != 0;
  k.source = sig.str() + (pdl && entry_trigger(k.grid) ? "  pdl_launch();\n" : "") +
             (pdl && !hoist ? "  pdl_wait();\n" : "") + body_src.str() + (pdl ? "  pdl_launch();\n" : "") + "}\n";
  return k;
}

// opaque_compute placeholder: mean of every operand element, broadcast
// (src/sim.cpp:215-226).  Phase 1 per-CTA f64 partial sums, grid barrier,
// every CTA folds the partials in the same order, then fills the output.
// Placeholder semantics of one opaque op (mean of every operand element,
// broadcast; src/sim.cpp:215-226): the statements after the PDL wait.  The
// enclosing code defines bid_ / nbid_ (this CTA's index and the CTA count
// of the op) and, for the grid form, bar_ / part_.
int opaque_block();

// 128-bit operand chunks one thread of a single-CTA placeholder holds in
// registers before it folds them (the single path issues every load first)
constexpr int kOpaqueRegChunks = 12;

static int64_t opaque_chunks_per_thread(const CompGraph& g, int vertex, int64_t span) {
  int64_t k = 0;
  for (int o : g.node(vertex).operands) {
    const TensorShape& sh = g.node(o).shape;
    const int64_t cnt = sh.element_count();
    const int64_t units = sh.dtype == DType::F32 && cnt % 4 == 0 ? cnt / 4 : cnt;
    k += (units + span - 1) / span;
  }
  return k;
}

static std::string opaque_body(const CompGraph& g, int vertex, bool single, int grid, int block,
                               const std::string& wait, int csize = 1) {
  const OpNode& n = g.node(vertex);
  int64_t count = 0;
  for (int o : n.operands) count += g.node(o).shape.element_count();
  std::ostringstream s;
  s << "  __shared__ double red_[" << block / 32 << "];\n  double acc = 0.0;\n";
  // an operand listed twice is counted twice, as upstream
  if (single) {
    // one CTA: issue every load of every operand first (128-bit where the
    // tensor allows), then fold -- one memory round trip instead of a chain
    // Graph parameters are never written by a kernel: their loads go before
    // the PDL wait (`wait`), kernel-produced operands after it
    int vi = 0;
    std::vector<std::pair<std::string, int>> regs;  // (array, lanes per element)
    int64_t held = 0;  // chunks in registers not yet folded
    auto fold = [&]() {
      for (const auto& [a, lanes] : regs) {
        s << "  #pragma unroll\n  for (int k = 0; k < (int)(sizeof(" << a << ") / sizeof(" << a << "[0])); ++k) ";
        if (lanes == 4)
          s << "acc += ((double)" << a << "[k].x + (double)" << a << "[k].y) + ((double)" << a << "[k].z + (double)" << a
            << "[k].w);\n";
        else
          s << "acc += (double)" << a << "[k];\n";
      }
      regs.clear();
      held = 0;
    };
    bool hoisted = false;
    for (int pass = 0; pass < 2; ++pass) {
     // ptxas schedules griddepcontrol.wait (ACQBULK) above independent
     // non-coherent loads of the same basic block, which would undo the
     // hoisting; a CTA barrier between them keeps the loads in front
     if (pass == 1 && hoisted && env_int("STITCH_OPAQUE_FENCE", 1) != 0) s << "  __syncthreads();\n";
     if (pass == 1) s << wait;
     for (int o : n.operands) {
      if ((g.node(o).kind == OpKind::Parameter) != (pass == 0)) continue;
      hoisted = hoisted || pass == 0;
      // pre-wait loads are coherent (ld.global, not .nc): ptxas keeps those
      // in front of the barrier below, while it sinks .nc loads past it
      const bool fence = pass == 0 && env_int("STITCH_OPAQUE_FENCE", 1) != 0;
      const std::string L4 = pass == 1 ? "ld4k(" : fence ? "ld4p(" : "ld4(",
                        LV = pass == 1 ? "ldvk(" : fence ? "ldvp(" : "ldv(";
      const TensorShape& sh = g.node(o).shape;
      const int64_t cnt = sh.element_count();
      const bool vec = sh.dtype == DType::F32 && cnt % 4 == 0;
      const int64_t units = vec ? cnt / 4 : cnt;
      const int64_t span = int64_t(block) * csize;  // threads of the op (its cluster)
      const int64_t K = (units + span - 1) / span;
      const std::string a = "v" + std::to_string(vi++) + "_";
      if (K > 8) {  // large operand: vectorised grid-stride loop
        if (vec)
          s << "  for (i64 i = (i64)bid_ * " << block << " + threadIdx.x; i < " << units << "; i += " << span << ") { const float4 q = " << L4
            << tensor_ident(g.node(o).name) << " + 4 * i); acc += ((double)q.x + (double)q.y) + ((double)q.z + (double)q.w); }\n";
        else
          s << "  for (i64 i = (i64)bid_ * " << block << " + threadIdx.x; i < " << units << "; i += " << span << ") acc += (double)" << LV
            << tensor_ident(g.node(o).name) << ", i);\n";
        continue;
      }
      // beyond the register budget: fold what is held before loading more
      if (held > 0 && held + K > kOpaqueRegChunks) fold();
      held += K;
      if (vec) {
        s << "  float4 " << a << "[" << K << "];\n  #pragma unroll\n  for (int k = 0; k < " << K
          << "; ++k) { const i64 i = (i64)bid_ * " << block << " + threadIdx.x + (i64)k * " << span << "; " << a << "[k] = i < " << units
          << " ? " << L4 << tensor_ident(g.node(o).name) << " + 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f); }\n";
        regs.push_back({a, 4});
      } else {
        s << "  float " << a << "[" << K << "];\n  #pragma unroll\n  for (int k = 0; k < " << K
          << "; ++k) { const i64 i = (i64)bid_ * " << block << " + threadIdx.x + (i64)k * " << span << "; " << a << "[k] = i < " << units
          << " ? " << LV << tensor_ident(g.node(o).name) << ", i) : 0.f; }\n";
        regs.push_back({a, 1});
      }
     }
    }
    fold();
  } else if (env_int("STITCH_OPAQUE_GRID_BATCH", 8) <= 0) {
    // grid (the round-1 form): 128-bit grid-stride loads, 4 independent
    // accumulators per thread, everything after the PDL wait
    s << wait;
    s << "  const i64 gt_ = (i64)blockIdx.x * blockDim.x + threadIdx.x, gs_ = (i64)gridDim.x * blockDim.x;\n"
      << "  double a0_ = 0.0, a1_ = 0.0, a2_ = 0.0, a3_ = 0.0;\n";
    for (int o : n.operands) {
      const TensorShape& sh = g.node(o).shape;
      const int64_t cnt = sh.element_count();
      const std::string T = tensor_ident(g.node(o).name);
      const bool param = g.node(o).kind == OpKind::Parameter;
      const std::string L4 = param ? "ld4(" : "ld4k(", LV = param ? "ldv(" : "ldvk(";
      if (sh.dtype == DType::F32 && cnt % 4 == 0) {
        const std::string u = std::to_string(cnt / 4);
        s << "  for (i64 i = gt_; i < " << u << "; i += 4 * gs_) {\n"
          << "    float4 q0 = " << L4 << T << " + 4 * i), q1 = make_float4(0.f, 0.f, 0.f, 0.f), q2 = q1, q3 = q1;\n"
          << "    if (i + gs_ < " << u << ") q1 = " << L4 << T << " + 4 * (i + gs_));\n"
          << "    if (i + 2 * gs_ < " << u << ") q2 = " << L4 << T << " + 4 * (i + 2 * gs_));\n"
          << "    if (i + 3 * gs_ < " << u << ") q3 = " << L4 << T << " + 4 * (i + 3 * gs_));\n"
          << "    a0_ += ((double)q0.x + (double)q0.y) + ((double)q0.z + (double)q0.w);\n"
          << "    a1_ += ((double)q1.x + (double)q1.y) + ((double)q1.z + (double)q1.w);\n"
          << "    a2_ += ((double)q2.x + (double)q2.y) + ((double)q2.z + (double)q2.w);\n"
          << "    a3_ += ((double)q3.x + (double)q3.y) + ((double)q3.z + (double)q3.w);\n  }\n";
      } else {
        s << "  for (i64 i = gt_; i < " << cnt << "; i += gs_) a0_ += (double)" << LV << T << ", i);\n";
      }
    }
    s << "  acc = (a0_ + a1_) + (a2_ + a3_);\n";
  } else {
    // grid: each thread's chunks of every operand are issued as batches of
    // up to STITCH_OPAQUE_GRID_BATCH 128-bit loads into registers before any
    // is folded (one memory round trip per batch instead of one per 4
    // chunks); graph parameters are loaded before the PDL wait (coherent
    // loads + a CTA barrier keep ptxas from sinking them below it), so they
    // stream while the producer drains.  64 registers per thread at
    // 4 CTAs x 256 threads per SM: 8 float4 in flight per thread
    const int B = std::clamp(env_int("STITCH_OPAQUE_GRID_BATCH", 8), 1, 16);
    const int64_t span = int64_t(grid) * block;
    s << "  const i64 gt_ = (i64)blockIdx.x * " << block << " + threadIdx.x;\n";
    int vi = 0;
    int64_t held = 0;
    std::vector<std::pair<std::string, int>> regs;
    auto fold = [&]() {
      for (const auto& [a, lanes] : regs) {
        s << "  #pragma unroll\n  for (int k = 0; k < (int)(sizeof(" << a << ") / sizeof(" << a << "[0])); ++k) ";
        if (lanes == 4)
          s << "acc += ((double)" << a << "[k].x + (double)" << a << "[k].y) + ((double)" << a << "[k].z + (double)" << a
            << "[k].w);\n";
        else
          s << "acc += (double)" << a << "[k];\n";
      }
      regs.clear();
      held = 0;
    };
    bool hoisted = false;
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) {
        fold();
        if (hoisted && env_int("STITCH_OPAQUE_FENCE", 1) != 0) s << "  __syncthreads();\n";
        s << wait;
      }
      for (int o : n.operands) {
        if ((g.node(o).kind == OpKind::Parameter) != (pass == 0)) continue;
        hoisted = hoisted || pass == 0;
        const bool fence = pass == 0 && env_int("STITCH_OPAQUE_FENCE", 1) != 0;
        const std::string L4 = pass == 1 ? "ld4k(" : fence ? "ld4p(" : "ld4(",
                          LV = pass == 1 ? "ldvk(" : fence ? "ldvp(" : "ldv(";
        const TensorShape& sh = g.node(o).shape;
        const int64_t cnt = sh.element_count();
        const bool vec = sh.dtype == DType::F32 && cnt % 4 == 0;
        const int64_t units = vec ? cnt / 4 : cnt;
        const int64_t K = (units + span - 1) / span;
        const std::string T = tensor_ident(g.node(o).name);
        if (K > B) {  // large operand: loop over batches of B chunks, each folded when it lands
          fold();
          const std::string a = "v" + std::to_string(vi++) + "_";
          s << "  for (i64 b_ = gt_; b_ < " << units << "; b_ += " << B * span << ") {\n";
          if (vec)
            s << "    float4 " << a << "[" << B << "];\n    #pragma unroll\n    for (int k = 0; k < " << B
              << "; ++k) { const i64 i = b_ + (i64)k * " << span << "; " << a << "[k] = i < " << units << " ? " << L4
              << T << " + 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f); }\n    #pragma unroll\n    for (int k = 0; k < " << B
              << "; ++k) acc += ((double)" << a << "[k].x + (double)" << a << "[k].y) + ((double)" << a << "[k].z + (double)"
              << a << "[k].w);\n  }\n";
          else
            s << "    float " << a << "[" << B << "];\n    #pragma unroll\n    for (int k = 0; k < " << B
              << "; ++k) { const i64 i = b_ + (i64)k * " << span << "; " << a << "[k] = i < " << units << " ? " << LV << T
              << ", i) : 0.f; }\n    #pragma unroll\n    for (int k = 0; k < " << B << "; ++k) acc += (double)" << a
              << "[k];\n  }\n";
          continue;
        }
        if (held > 0 && held + K > B) fold();
        held += K;
        const std::string a = "v" + std::to_string(vi++) + "_";
        if (vec) {
          s << "  float4 " << a << "[" << K << "];\n  #pragma unroll\n  for (int k = 0; k < " << K
            << "; ++k) { const i64 i = gt_ + (i64)k * " << span << "; " << a << "[k] = i < " << units << " ? " << L4 << T
            << " + 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f); }\n";
          regs.push_back({a, 4});
        } else {
          s << "  float " << a << "[" << K << "];\n  #pragma unroll\n  for (int k = 0; k < " << K
            << "; ++k) { const i64 i = gt_ + (i64)k * " << span << "; " << a << "[k] = i < " << units << " ? " << LV << T
            << ", i) : 0.f; }\n";
          regs.push_back({a, 1});
        }
      }
    }
    fold();
  }
  // warp sums -> warp 0 folds them with one butterfly (fixed order,
  // deterministic) -> broadcast through shared memory
  s << "  acc = bfly_sum(acc, 32);\n  if ((threadIdx.x & 31) == 0) red_[threadIdx.x >> 5] = acc;\n  __syncthreads();\n"
    << "  __shared__ double tot_;\n  if (threadIdx.x < 32) {\n    double w_ = threadIdx.x < " << block / 32
    << " ? red_[threadIdx.x] : 0.0;\n    w_ = bfly_sum(w_, 32);\n    if (threadIdx.x == 0) tot_ = w_;\n  }\n"
    << "  __syncthreads();\n  double tot = tot_;\n";
  if (single && csize > 1)  // the op's CTAs form one cluster: add their partials in rank order (DSMEM)
    s << "  cluster_sync_all();\n  tot = 0.0;\n  #pragma unroll\n  for (unsigned r_ = 0; r_ < " << csize
      << "u; ++r_) tot += ld_dsmem_f64(&tot_, r_);\n  cluster_sync_all();  // peers done reading our tot_\n";
  if (!single)
    s << "  if (threadIdx.x == 0) part_[blockIdx.x] = tot;\n  grid_sync(bar_, gridDim.x);\n"
      << "  __shared__ double all_;\n"
      // every partial load issued before the first add (one L2 round trip,
      // not grid/32 dependent ones), then the same fixed-order fold
      << "  if (threadIdx.x < 32) {\n    double pv_[" << (grid + 31) / 32 << "];\n    #pragma unroll\n    for (int k = 0; k < "
      << (grid + 31) / 32 << "; ++k) { const int b = threadIdx.x + 32 * k; pv_[k] = b < " << grid
      << " ? __ldcg(part_ + b) : 0.0; }\n    double t = 0.0;\n    #pragma unroll\n    for (int k = 0; k < " << (grid + 31) / 32
      << "; ++k) t += pv_[k];\n    t = bfly_sum(t, 32);\n    if (threadIdx.x == 0) all_ = t;\n  }\n"
      << "  __syncthreads();\n  tot = all_;\n";
  s << "  const float fill = (float)(" << (count ? "tot / " + std::to_string(count) + ".0" : "0.0") << ");\n";
  const int64_t nout = n.shape.element_count();
  if (n.shape.dtype == DType::F32 && nout % 4 == 0)  // 128-bit stores
    s << "  for (i64 i = (i64)bid_ * blockDim.x + threadIdx.x; i < " << nout / 4
      << "; i += (i64)nbid_ * blockDim.x) st4(" << tensor_ident(n.name) << " + 4 * i, fill, fill, fill, fill);\n";
  else
    s << "  for (i64 i = (i64)bid_ * blockDim.x + threadIdx.x; i < " << nout
      << "; i += (i64)nbid_ * blockDim.x) stv(" << tensor_ident(n.name) << ", i, fill);\n";
  return s.str();
}

// CTAs (one thread-block cluster) per small placeholder.  Default: the
// fewest CTAs (<= 8) whose threads hold every operand chunk in at most
// kOpaqueRegChunks float4 registers -- 1 for DIEN's per-step gate GEMMs
// (2 x [256,36] operands: 10 chunks per thread), 5 for the attention-score
// GEMM over all T interest states (11 operands: 55 chunks per thread in one
// CTA, which spilled 1.3 KB/thread and ran 20.8 us).  A cluster costs a
// launch + barriers, so small ops stay single-CTA (DIEN T=20 121.8 (1) vs
// 129.2 (3) vs 141.0 us (8) for the gate GEMMs,
// profiles/r01/opaque_cluster_ab.jsonl).  STITCH_OPAQUE_CLUSTER=0 is the
// older auto rule (one 128-bit chunk per thread of the largest tensor),
// =<n> forces n.
int opaque_cluster(const CompGraph& g, int vertex) {
  const int c = env_int("STITCH_OPAQUE_CLUSTER", -1);
  if (c > 0) return std::min(c, 8);
  if (c < 0) {
    for (int k = 1; k <= 8; ++k)
      if (opaque_chunks_per_thread(g, vertex, int64_t(opaque_block()) * k) <= kOpaqueRegChunks) return k;
    return 8;
  }
  const OpNode& n = g.node(vertex);
  int64_t units = n.shape.element_count();
  for (int o : n.operands) units = std::max(units, g.node(o).shape.element_count());
  units = (units + 3) / 4;
  return static_cast<int>(std::clamp<int64_t>((units + 1023) / 1024, 1, 8));
}

// threads of a single-CTA placeholder (STITCH_OPAQUE_BLOCK, 32..1024):
// 512 balances the load/store chain per thread against the depth of the
// block reduction (DIEN T=10 55.3 / 53.8 / 59.6 us at 1024 / 512 / 256,
// profiles/r01/opaque_block_ab.jsonl)
// (1024 under the opt-in persistent template, which runs barrier-using
// units only as whole 1024-thread CTAs)
int opaque_block() {
  if (env_int("STITCH_PERSIST", 0) == 1) return 1024;
  return std::clamp(env_int("STITCH_OPAQUE_BLOCK", 512) / 32 * 32, 32, 1024);
}

bool opaque_single(const CompGraph& g, int vertex) {
  const OpNode& n = g.node(vertex);
  int64_t work = n.shape.element_count();
  for (int o : n.operands) work += g.node(o).shape.element_count();
  return work <= (int64_t(1) << 20);
}

KernelSpec generate_opaque_kernel(const CompGraph& g, int vertex, const std::string& name, int sm_count) {
  const SmScope sm_scope(sm_count);
  const OpNode& n = g.node(vertex);
  std::set<int> ops(n.operands.begin(), n.operands.end());
  // small tensors (e.g. DIEN's [256,36] GEMM outputs): one 1024-thread CTA,
  // no grid-wide barrier; large ones: cooperative grid with a barrier
  const bool single = opaque_single(g, vertex);
  const int csize = single ? opaque_cluster(g, vertex) : 1;
  const int grid = single ? csize : sm_now() * 4;  // cooperative: 4 co-resident 256-thread CTAs per SM
  const int block = single ? opaque_block() : kBlock;
  KernelSpec k;
  k.name = name;
  k.tmpl = single ? "opaque" : "opaque(grid)";
  k.pattern_key = "op:" + n.name;
  k.grid = grid;
  k.block = block;
  k.cooperative = !single;
  k.cluster = csize;
  if (csize > 1) k.tmpl += "-cluster" + std::to_string(csize);
  std::ostringstream s;
  s << "extern \"C\" __global__ void __launch_bounds__(" << block << ", " << (single ? 1 : 4) << ") " << name << "(";
  for (int o : ops) {
    s << "const " << c_type(g.node(o).shape.dtype) << "* __restrict__ " << tensor_ident(g.node(o).name) << ", ";
    k.inputs.push_back(g.node(o).name);
  }
  s << c_type(n.shape.dtype) << "* __restrict__ " << tensor_ident(n.name);
  if (!single) {
    s << ", unsigned* __restrict__ bar_, double* __restrict__ part_";
    k.scratch_bytes = 256 + int64_t(grid) * 8;
  }
  // trigger dependents as soon as our own prerequisites are met: a dependent
  // then launches (and becomes resident) while we run, hiding its launch
  // latency behind our body (STITCH_OPAQUE_EARLY=0: trigger at exit)
  const bool early = env_int("STITCH_OPAQUE_EARLY", 1) != 0;
  s << ") {\n" << (entry_trigger(grid) ? "  pdl_launch();\n" : "");
  k.outputs.push_back(n.name);
  s << "  const int bid_ = blockIdx.x, nbid_ = gridDim.x;\n"
    << opaque_body(g, vertex, single, grid, block, early ? "  pdl_wait();\n  pdl_launch();\n" : "  pdl_wait();\n",
                   csize);
  s << "  pdl_launch();\n}\n";
  k.source = s.str();
  int64_t bytes = n.shape.byte_size();
  for (int o : ops) bytes += g.node(o).shape.byte_size();
  k.alg_bytes = bytes;
  return k;
}

KernelSpec generate_opaque_pack(const CompGraph& g, const std::vector<int>& vertices, const std::string& name) {
  KernelSpec k;
  k.name = name;
  int csize = 1;  // one cluster per op, the largest op's size for all
  for (int v : vertices) csize = std::max(csize, opaque_cluster(g, v));
  k.tmpl = "opaque(pack" + std::to_string(vertices.size()) + (csize > 1 ? "x" + std::to_string(csize) : "") + ")";
  k.grid = static_cast<int>(vertices.size()) * csize;
  const int ob = opaque_block();
  k.block = ob;
  k.cluster = csize;
  const bool early = env_int("STITCH_OPAQUE_EARLY", 1) != 0;
  std::ostringstream sig, body;
  std::set<std::string> seen;
  int64_t bytes = 0;
  sig << "extern \"C\" __global__ void __launch_bounds__(" << ob << ", 1) " << name << "(";
  for (int v : vertices) {
    if (!opaque_single(g, v)) throw std::invalid_argument("opaque pack: " + g.node(v).name + " needs the grid form");
    k.pattern_key += std::string(k.pattern_key.empty() ? "" : "+") + "op:" + g.node(v).name;
    for (int o : g.node(v).operands)
      if (seen.insert(g.node(o).name).second) {
        sig << "const " << c_type(g.node(o).shape.dtype) << "* __restrict__ " << tensor_ident(g.node(o).name) << ", ";
        k.inputs.push_back(g.node(o).name);
        bytes += g.node(o).shape.byte_size();
      }
  }
  for (size_t j = 0; j < vertices.size(); ++j) {
    const OpNode& n = g.node(vertices[j]);
    sig << (j ? ", " : "") << c_type(n.shape.dtype) << "* __restrict__ " << tensor_ident(n.name);
    k.outputs.push_back(n.name);
    bytes += n.shape.byte_size();
    body << "  " << (j ? "} else " : "") << "if (blockIdx.x / " << csize << " == " << j << ") {\n  const int bid_ = blockIdx.x % "
         << csize << ", nbid_ = " << csize << ";\n"
         << opaque_body(g, vertices[j], true, csize, ob, early ? "  pdl_wait();\n  pdl_launch();\n" : "  pdl_wait();\n",
                        csize);
  }
  // dependents are triggered like a single placeholder's (entry_trigger:
  // after the wait for a one-wave pack under the default entry_large)
  k.source = sig.str() + ") {\n" + (entry_trigger(k.grid) ? "  pdl_launch();\n" : "") + body.str() +
             "  }\n  pdl_launch();\n}\n";
  k.alg_bytes = bytes;
  return k;
}

ForcedBlockScope::ForcedBlockScope(int block) : old(tl_force_block) { tl_force_block = block; }
ForcedBlockScope::~ForcedBlockScope() { tl_force_block = old; }

}  // namespace stitch::gpu
