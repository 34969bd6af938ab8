// Resident template: a launch-bound plan as ONE thread-block cluster.
//
// Why.  On DIEN-like graphs (hundreds of [256,36] ops) every plan kernel is a
// few hundred bytes of work per SM, so a CUDA Graph of kernels costs one
// dependent-launch + L2 round trip per kernel boundary (~1.5-2.6 us per DIEN
// unit, profiles/r02/dien_T10_timeline.txt), and the persistent template's
// L2 completion counters cost about the same (profiles/r01/persistent_*).
// The values themselves would fit on chip: a [256,36] f32 tensor is 36 KB.
//
// How.  Every tensor of the graph either carries the batch as its leading
// axis ("sharded") or does not depend on the batch row at all
// ("replicated"), and every non-opaque op is row-local: elementwise ops,
// broadcasts that keep axis 0, reductions / slices / transposes that do not
// touch axis 0.  CTA r of a cluster of C CTAs then owns batch rows
// [r*R, (r+1)*R) of every sharded tensor and computes them alone:
//   * each plan kernel (pattern / singleton / materialised constant) is the
//     dataflow template generated for the SHARD graph (batch R instead of B,
//     same node ids) with one 1024-thread CTA, called as a device function;
//   * tensors that cross plan-kernel boundaries live in the CTA's shared
//     memory (liveness-reused slots), graph parameters and outputs in their
//     global buffers at the CTA's row offset; all accesses are generic
//     loads/stores, ordered by CTA barriers only where a unit reads what an
//     earlier unit since the last barrier wrote;
//   * opaque placeholders (mean of every operand element, broadcast --
//     src/sim.cpp:215-226) are the only cross-row ops: each CTA reduces its
//     rows in f64, pushes the partials of a group of independent placeholders
//     to every peer's shared memory (st.async, completing on the peer's
//     mbarrier of that group; STITCH_RESIDENT_PUSH=0: one cluster barrier
//     per group and DSMEM loads), and every CTA folds the C partials in rank
//     order (identical result everywhere).
// The plan (patterns, per-op f32 rounding, the opaque semantics) is the one
// the graph executor runs; only the kernel boundaries stay on chip.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <optional>
#include <regex>
#include <set>
#include <sstream>

#include "codegen/cg.hpp"

namespace stitch::gpu {

namespace {

int64_t prod_from(const std::vector<int64_t>& d, size_t from) {
  int64_t p = 1;
  for (size_t i = from; i < d.size(); ++i) p *= d[i];
  return p;
}

bool is_elementwise(OpKind k) {
  switch (k) {
    case OpKind::Add: case OpKind::Sub: case OpKind::Mul: case OpKind::Div: case OpKind::Max: case OpKind::Min:
    case OpKind::Exp: case OpKind::Tanh: case OpKind::Log: case OpKind::Rsqrt: case OpKind::Power:
      return true;
    default:
      return false;
  }
}

// batch extent: the leading dimension shared by most rank>=1 parameters
int64_t batch_extent(const CompGraph& g) {
  std::map<int64_t, int> votes;
  for (const auto& n : g.nodes)
    if (n.kind == OpKind::Parameter && n.shape.rank() >= 1) ++votes[n.shape.dims[0]];
  int64_t best = 0;
  int bv = 0;
  for (auto [b, v] : votes)
    if (v > bv || (v == bv && b > best)) best = b, bv = v;
  return best;
}

// sharded[v]: v's leading axis is the batch row.  False + *why when some op
// would mix rows (the graph is not row-shardable).
bool analyse_rows(const CompGraph& g, int64_t B, std::vector<char>& sharded, std::string* why) {
  auto fail = [&](const OpNode& n, const std::string& m) {
    if (why) *why = "op " + n.name + ": " + m;
    return false;
  };
  sharded.assign(g.nodes.size(), 0);
  for (const auto& n : g.nodes) {
    const bool lead_b = n.shape.rank() >= 1 && n.shape.dims[0] == B;
    auto sh = [&](int o) { return sharded[static_cast<size_t>(o)] != 0; };
    char& s = sharded[static_cast<size_t>(n.id)];
    if (n.kind == OpKind::Parameter || n.kind == OpKind::Constant || n.kind == OpKind::OpaqueCompute) {
      s = lead_b;
    } else if (is_elementwise(n.kind)) {
      for (int o : n.operands)
        if (sh(o) != sh(n.operands[0])) return fail(n, "mixes batch-row and replicated operands");
      s = sh(n.operands[0]);
    } else if (n.kind == OpKind::Broadcast) {
      const int x = n.operands[0];
      const auto& d = n.attrs.dims;
      if (sh(x)) {
        if (d.empty() || d[0] != 0 || !lead_b) return fail(n, "broadcast moves the batch axis");
        s = 1;
      } else {
        // replicated data: sharded only when axis 0 is pure replication
        s = lead_b && std::find(d.begin(), d.end(), 0) == d.end();
      }
    } else if (n.kind == OpKind::ReduceSum || n.kind == OpKind::ReduceMax) {
      if (sh(n.operands[0])) {
        if (std::count(n.attrs.axes.begin(), n.attrs.axes.end(), 0)) return fail(n, "reduces over the batch axis");
        s = 1;
      }
    } else if (n.kind == OpKind::Slice) {
      if (sh(n.operands[0])) {
        if (n.attrs.starts.empty() || n.attrs.starts[0] != 0 || n.attrs.limits[0] != B)
          return fail(n, "slices the batch axis");
        s = 1;
      }
    } else if (n.kind == OpKind::Transpose) {
      if (sh(n.operands[0])) {
        if (n.attrs.perm.empty() || n.attrs.perm[0] != 0) return fail(n, "transposes the batch axis");
        s = 1;
      }
    } else {
      for (int o : n.operands)
        if (sh(o)) return fail(n, "gathers across batch rows");
    }
  }
  return true;
}

// the pattern kernel's source as __device__ FN_(tensors..., vb_, vg_):
// tensor params renamed positionally, every global access generic
std::string as_resident_function(const KernelSpec& k) {
  const std::string& src = k.source;
  const size_t at = src.find(k.name + "(");
  if (src.compare(0, 10, "extern \"C\"") != 0 || at == std::string::npos)
    throw std::invalid_argument("resident: unexpected kernel header in " + k.name);
  // every call inlined: the pointers are then known shared-memory slots
  // (LDS/STS).  STITCH_RESIDENT_INLINE=0 keeps one copy of each unit
  // function, so DIEN's per-step calls would reuse code already in the
  // instruction cache (the inlined kernel's top ncu stall is
  // no_instructions, 34% of samples).  Measured slower, because the calls
  // then address generic pointers and lose constant propagation: T=10
  // 20.1 -> 25.9 us, T=20 36.9 -> 49.6 us (profiles/r02/resident/resident_inline.jsonl)
  const char* iv = std::getenv("STITCH_RESIDENT_INLINE");
  const bool inl = !(iv && *iv == '0');
  std::string body = std::string(inl ? "__device__ __forceinline__" : "__device__ __noinline__") + " void FN_(" +
                     src.substr(at + k.name.size() + 1);
  int pi = 0;
  for (const auto* list : {&k.inputs, &k.outputs})
    for (const auto& t : *list)
      body = std::regex_replace(body, std::regex("\\b" + regex_escape(tensor_ident(t)) + "\\b"), "p" + std::to_string(pi++) + "_");
  const size_t close = body.find(") {\n");
  if (close == std::string::npos) throw std::invalid_argument("resident: no signature end in " + k.name);
  body.insert(close, ", const int vb_, const int vg_");
  static const std::vector<std::pair<std::regex, std::string>> rewrites = {
      {std::regex(R"(\bblockIdx\.x\b)"), "vb_"},
      {std::regex(R"(\bgridDim\.x\b)"), "vg_"},
      {std::regex(R"(__restrict__)"), ""},
      {std::regex(R"(\bld4[ckp]?\()"), "ld4_g("},
      {std::regex(R"(\bld4hk?\()"), "ld4h_g("},
      {std::regex(R"(\bldv[kp]?\()"), "ldv_g("},
      {std::regex(R"(\b__ldg\()"), "ldg_g("},
      {std::regex(R"(\bst4\()"), "st4_g("},
      {std::regex(R"(\bst4h\()"), "st4h_g("},
      {std::regex(R"(\bpdl_(wait|launch)\(\);)"), ""},
      {std::regex(R"(\bSTC_TRACE_[A-Z_]+\([^)]*\);)"), ""},
  };
  for (const auto& [re, to] : rewrites) body = std::regex_replace(body, re, to);
  return std::regex_replace(body, std::regex(R"(\bblockDim\.x\b)"), std::to_string(k.block));
}

struct Slot {
  int64_t off = 0, bytes = 0;
};

// Recurrent plans (DIEN) emit the same step block once per time step, equal
// up to integer literals (slot offsets, inbox / mbarrier indices, trace
// slots): ~700 SASS instructions per step, so the straight-line kernel is
// ~8.8k instructions, each fetched cold once per launch (ncu: no_instructions
// is the top stall, 34% of samples).  The longest run of >= 3 consecutive
// blocks (split at placeholder-group markers) that agree outside their
// integer literals becomes ONE loop body; the literals that differ between
// iterations come from a __constant__ table.  A differing literal that
// touches an identifier, a suffix or a float literal aborts the rewrite.
std::string loop_recurrence(const std::string& body, const std::string& tab, std::string* tab_decl, int* iters) {
  static const std::regex marker(R"(\n  \{  // placeholder group: )");
  std::vector<size_t> at;
  for (auto it = std::sregex_iterator(body.begin(), body.end(), marker); it != std::sregex_iterator(); ++it)
    at.push_back(static_cast<size_t>(it->position()));
  if (at.size() < 4) return body;
  static const std::regex digits(R"(\d+)"), comment(R"(//[^\n]*)");
  // blocks without their comments (unit / group labels name the step)
  auto block = [&](size_t i) { return std::regex_replace(body.substr(at[i], at[i + 1] - at[i]), comment, ""); };
  auto shape = [&](size_t i) { return std::regex_replace(block(i), digits, "#"); };
  size_t best_lo = 0, best_n = 0;
  for (size_t lo = 0; lo + 1 < at.size();) {
    const std::string s0 = shape(lo);
    size_t n = 1;
    while (lo + n + 1 < at.size() && shape(lo + n) == s0) ++n;
    if (n > best_n) best_n = n, best_lo = lo;
    lo += n;
  }
  if (best_n < 3) return body;
  struct Tok {
    size_t pos, len;
    std::string val;
  };
  std::vector<std::vector<Tok>> toks(best_n);
  for (size_t b = 0; b < best_n; ++b) {
    const std::string blk = block(best_lo + b);
    for (auto it = std::sregex_iterator(blk.begin(), blk.end(), digits); it != std::sregex_iterator(); ++it)
      toks[b].push_back({static_cast<size_t>(it->position()), static_cast<size_t>(it->length()), it->str()});
  }
  const std::string first = block(best_lo);
  auto ident = [](char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '.'; };
  std::vector<size_t> var;
  std::set<size_t> fn_var;  // the N of a unit call "ruN_(" differs (e.g. DIEN's per-step column slices)
  for (size_t k = 0; k < toks[0].size(); ++k) {
    bool differs = false;
    for (size_t b = 1; b < best_n; ++b) differs = differs || toks[b][k].val != toks[0][k].val;
    if (!differs) continue;
    const Tok& t = toks[0][k];
    const bool unit_fn = t.pos >= 2 && first.compare(t.pos - 2, 2, "ru") == 0 && (t.pos < 3 || !ident(first[t.pos - 3])) &&
                         first.compare(t.pos + t.len, 2, "_(") == 0;
    if (unit_fn) {
      fn_var.insert(var.size());
    } else if ((t.pos > 0 && ident(first[t.pos - 1])) ||
               (t.pos + t.len < first.size() && ident(first[t.pos + t.len]))) {
      return body;  // part of a name, a suffix or a float literal: not a plain integer
    }
    const size_t line = first.rfind('\n', t.pos);
    if (first.find("#pragma", line == std::string::npos ? 0 : line) < t.pos) return body;
    var.push_back(k);
  }
  const std::string V = std::to_string(var.size());
  auto entry = [&](size_t v) { return tab + "[it_ * " + V + " + " + std::to_string(v) + "]"; };
  std::string tmpl;
  size_t cur = 0;
  for (size_t v = 0; v < var.size(); ++v) {
    const Tok& t = toks[0][var[v]];
    tmpl += first.substr(cur, t.pos - cur) + (fn_var.count(v) ? "@F" + std::to_string(v) + "@" : entry(v));
    cur = t.pos + t.len;
  }
  tmpl += first.substr(cur);
  // a unit call whose function differs per step: dispatch on the table entry
  // (one case per distinct function; the arguments are the loop template's)
  for (size_t v : fn_var) {
    const std::string mark = "@F" + std::to_string(v) + "@";
    const size_t m = tmpl.find(mark);
    const size_t ls = tmpl.rfind('\n', m) + 1, le = tmpl.find('\n', m);
    const std::string line = tmpl.substr(ls, le - ls);
    std::set<std::string> names;
    for (size_t b = 0; b < best_n; ++b) names.insert(toks[b][var[v]].val);
    std::string sw = "  switch (" + entry(v) + ") {";
    for (const auto& nm : names) {
      std::string l = line;
      l.replace(l.find(mark), mark.size(), nm);
      sw += "\n  case " + nm + ": " + l.substr(l.find_first_not_of(' ')) + " break;";
    }
    sw += "\n  default: __trap();\n  }";
    tmpl.replace(ls, le - ls, sw);
  }
  if (tmpl.find("@F") != std::string::npos) return body;
  std::ostringstream d;
  d << "__constant__ int " << tab << "[" << std::max<size_t>(1, best_n * var.size()) << "] = {";
  for (size_t b = 0; b < best_n; ++b)
    for (size_t k : var) d << toks[b][k].val << ",";
  d << "};\n";
  *tab_decl = d.str();
  *iters = static_cast<int>(best_n);
  return body.substr(0, at[best_lo]) + "\n  // " + std::to_string(best_n) +
         " recurrent steps as one loop (literals per step in " + tab + ")\n  #pragma unroll 1\n  for (int it_ = 0; it_ < " +
         std::to_string(best_n) + "; ++it_) {" + tmpl + "\n  }" + body.substr(at[best_lo + best_n]);
}

}  // namespace

namespace {
thread_local bool tl_no_handoff = false;  // retry without barrier elision
}

std::optional<KernelSpec> generate_resident_kernel_once(const CompGraph& g, const std::vector<ResidentUnit>& units,
                                                        const std::string& name, std::string* why, bool* smem_bound);

// Eliding barriers delays when freed slots return to the allocator (they are
// reused only after a barrier), so a plan near the shared-memory cap may only
// fit with every barrier kept: retry that way before giving up
std::optional<KernelSpec> generate_resident_kernel(const CompGraph& g, const std::vector<ResidentUnit>& units,
                                                   const std::string& name, std::string* why) {
  bool smem_bound = false;
  auto k = generate_resident_kernel_once(g, units, name, why, &smem_bound);
  if (k || !smem_bound) return k;
  tl_no_handoff = true;
  k = generate_resident_kernel_once(g, units, name, why, &smem_bound);
  tl_no_handoff = false;
  return k;
}

std::optional<KernelSpec> generate_resident_kernel_once(const CompGraph& g, const std::vector<ResidentUnit>& units,
                                                        const std::string& name, std::string* why, bool* smem_bound) {
  auto no = [&](const std::string& m) -> std::optional<KernelSpec> {
    if (why) *why = m;
    return std::nullopt;
  };
  if (units.size() < 2) return no("fewer than two launch units");
  const int64_t B = batch_extent(g);
  if (B < 1) return no("no batch axis");
  std::vector<char> sharded;
  if (!analyse_rows(g, B, sharded, why)) return std::nullopt;
  // cluster size: the most CTAs (<= 16) with a whole number of rows each,
  // a multiple of 4 (16-byte aligned row blocks for 128-bit accesses)
  // (STITCH_RESIDENT_CLUSTER caps it)
  int C = 1;
  const char* cv = std::getenv("STITCH_RESIDENT_CLUSTER");
  const int cmax = cv && *cv ? std::atoi(cv) : 16;
  for (int c : {16, 8, 4, 2})
    if (c <= cmax && B % c == 0 && (B / c) % 4 == 0) {
      C = c;
      break;
    }
  const int64_t R = B / C;
  // folding the C partials: a butterfly over the next power of two lanes;
  // the mean as a product with the correctly rounded reciprocal of the
  // count (a double division is a ~100-cycle subroutine on the step's
  // critical path; the f32 mean it rounds to is the quotient's)
  int fold_w = 1;
  while (fold_w < C) fold_w *= 2;
  fold_w = std::max(fold_w, 2);
  auto inv_count = [](int64_t count) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", 1.0 / static_cast<double>(count));
    return std::string(buf);
  };
  CompGraph gs = g;  // the shard graph: batch R, same node ids
  for (auto& n : gs.nodes) {
    if (!sharded[static_cast<size_t>(n.id)]) continue;
    n.shape.dims[0] = R;
    if (n.kind == OpKind::Slice) n.attrs.limits[0] = static_cast<int>(R);
  }
  auto local_elems = [&](int v) {
    const auto& sh = g.node(v).shape;
    return sharded[static_cast<size_t>(v)] ? R * prod_from(sh.dims, 1) : sh.element_count();
  };
  auto local_bytes = [&](int v) { return local_elems(v) * dtype_bytes(g.node(v).shape.dtype); };

  // per unit: generated code (patterns) or the opaque vertex
  struct U {
    std::vector<int> verts;
    bool opaque = false;
    KernelSpec spec;  // patterns
    std::vector<int> ins, outs;  // tensor vertex ids
    std::set<size_t> deps;
  };
  std::vector<U> us(units.size());
  std::map<int, size_t> producer;  // tensor vertex -> unit
  for (size_t i = 0; i < units.size(); ++i) {
    U& u = us[i];
    u.verts = units[i].verts;
    u.opaque = units[i].opaque;
    if (u.opaque) {
      if (u.verts.size() != 1) return no("opaque unit with several vertices");
      const OpNode& n = g.node(u.verts[0]);
      std::set<int> seen;
      for (int o : n.operands)
        if (seen.insert(o).second) u.ins.push_back(o);
      u.outs = {n.id};
    } else {
      try {
        const ForcedBlockScope fb(1024);
        u.spec = generate_pattern_kernel(gs, u.verts, "RK_", 1);
      } catch (const std::exception& e) {
        return no(std::string("unit ") + g.node(u.verts.front()).name + ": " + e.what());
      }
      if (u.spec.scratch_bytes > 0 || u.spec.cooperative || u.spec.cluster > 1 || u.spec.smem > 0 || u.spec.block != 1024)
        return no("unit " + g.node(u.verts.front()).name + " needs a grid-wide template (" + u.spec.tmpl + ")");
      for (const auto& t : u.spec.inputs) u.ins.push_back(g.by_name.at(t));
      for (const auto& t : u.spec.outputs) u.outs.push_back(g.by_name.at(t));
    }
    for (int t : u.outs) producer[t] = i;
  }
  std::vector<std::vector<size_t>> users(us.size());
  for (size_t i = 0; i < us.size(); ++i)
    for (int t : us[i].ins) {
      if (auto it = producer.find(t); it != producer.end()) {
        if (it->second != i && us[i].deps.insert(it->second).second) users[it->second].push_back(i);
      } else if (g.node(t).kind != OpKind::Parameter) {
        return no("tensor " + g.node(t).name + " is read but produced by no unit");
      }
    }

  // placeholder groups whose partials meet by st.async pushes can be split:
  // phase A (local fold + push) and phase B (wait for the peers' partials,
  // fold, fill), with up to STITCH_RESIDENT_FILL ready CTA-local units that do
  // not depend on the group run in between -- they hide the DSMEM exchange
  // (DIEN: the attention-column units, one triple per recurrent step)
  const char* pv = std::getenv("STITCH_RESIDENT_PUSH");
  const bool push = C > 1 && !(pv && *pv == '0');
  const char* fv = std::getenv("STITCH_RESIDENT_FILL");
  const int fill_units = fv && *fv ? std::max(0, std::atoi(fv)) : 3;
  auto group_partials = [&](const std::vector<size_t>& grp) {
    std::map<int, int> dk;  // operand vertex -> partial index
    for (size_t j : grp)
      for (int o : g.node(us[j].verts[0]).operands) dk.emplace(o, static_cast<int>(dk.size()));
    return dk;
  };
  auto warp_path_of = [&](const std::map<int, int>& dk) {
    bool ok = dk.size() <= 32;
    for (auto [o, k] : dk) ok = ok && local_elems(o) <= 16384;
    return ok;
  };
  auto pushed = [&](const std::vector<size_t>& grp) {
    return push && warp_path_of(group_partials(grp)) && static_cast<int64_t>(grp.size()) * C <= 1024;
  };

  // schedule: CTA-local units as soon as they are ready; ready placeholders
  // wait until nothing else is, then run together as one group -- or, with
  // split groups, as soon as they are ready, with fillers inside the group
  enum Phase { kUnit = 0, kGroupA = 1, kGroupB = 2, kGroup = 3 };
  std::vector<std::vector<size_t>> steps;  // one unit, or a group of placeholders
  std::vector<int> phase;
  {
    std::vector<size_t> pending(us.size());
    std::set<size_t> ready;
    for (size_t i = 0; i < us.size(); ++i)
      if (!(pending[i] = us[i].deps.size())) ready.insert(i);
    size_t done = 0;
    auto finish = [&](size_t i) {
      ++done;
      for (size_t w : users[i])
        if (--pending[w] == 0) ready.insert(w);
    };
    auto next_local = [&]() {
      return std::find_if(ready.begin(), ready.end(), [&](size_t i) { return !us[i].opaque; });
    };
    while (!ready.empty()) {
      std::vector<size_t> ops;
      for (size_t i : ready)
        if (us[i].opaque) ops.push_back(i);
      if (fill_units > 0 && !ops.empty() && pushed(ops)) {
        for (size_t i : ops) ready.erase(i);
        steps.push_back(ops);
        phase.push_back(kGroupA);
        for (int f = 0; f < fill_units; ++f) {
          auto it = next_local();
          if (it == ready.end()) break;
          const size_t i = *it;
          ready.erase(it);
          steps.push_back({i});
          phase.push_back(kUnit);
          finish(i);
        }
        steps.push_back(ops);
        phase.push_back(kGroupB);
        for (size_t i : ops) finish(i);
        continue;
      }
      auto it = next_local();
      if (it != ready.end()) {
        const size_t i = *it;
        ready.erase(it);
        steps.push_back({i});
        phase.push_back(kUnit);
        finish(i);
        continue;
      }
      std::vector<size_t> grp(ready.begin(), ready.end());
      ready.clear();
      steps.push_back(grp);
      phase.push_back(kGroup);
      for (size_t i : grp) finish(i);
    }
    if (done != us.size()) return no("unit dependency cycle");
  }

  // placement: graph parameters / outputs in global memory, everything else
  // crossing a unit boundary in a shared-memory slot (reused after the
  // barrier that follows its last reader)
  std::set<int> graph_out(g.outputs.begin(), g.outputs.end());
  std::map<int, size_t> last_step;
  for (size_t s = 0; s < steps.size(); ++s)
    if (phase[s] != kGroupB)  // phase B only writes the group's outputs
      for (size_t i : steps[s])
        for (int t : us[i].ins) last_step[t] = s;
  std::map<int, Slot> slot;
  std::vector<Slot> free_list, pending_free;
  int64_t smem_top = 0;
  constexpr int64_t kSmemCap = 200 * 1024;
  auto alloc = [&](int64_t bytes) {
    bytes = (bytes + 127) / 128 * 128;
    std::sort(free_list.begin(), free_list.end(), [](const Slot& a, const Slot& b) { return a.off < b.off; });
    for (size_t i = 0; i < free_list.size(); ++i)
      if (free_list[i].bytes >= bytes) {
        Slot s{free_list[i].off, bytes};
        free_list[i].off += bytes;
        free_list[i].bytes -= bytes;
        if (free_list[i].bytes == 0) free_list.erase(free_list.begin() + static_cast<long>(i));
        return s;
      }
    Slot s{smem_top, bytes};
    smem_top += bytes;
    return s;
  };

  std::ostringstream fns, body;
  std::map<std::string, std::string> fn_of;  // canonical unit source -> function name
  auto ptr = [&](int t) -> std::string {
    const OpNode& n = g.node(t);
    const std::string ty = c_type(n.shape.dtype);
    if (auto it = slot.find(t); it != slot.end())
      return "reinterpret_cast<" + ty + "*>(rs_smem_ + " + std::to_string(it->second.off) + ")";
    const std::string off = sharded[static_cast<size_t>(t)] ? " + (i64)rk_ * " + std::to_string(local_elems(t)) : "";
    return "(" + tensor_ident(n.name) + off + ")";
  };
  std::set<size_t> since_barrier;  // units executed after the last CTA barrier
  std::set<int> params_used, outs_written;
  int opaque_slots = 0, max_group = 1, n_barriers = 0, n_cluster = 0;
  auto barrier = [&]() {
    body << "  __syncthreads();\n";
    ++n_barriers;
    since_barrier.clear();
    free_list.insert(free_list.end(), pending_free.begin(), pending_free.end());
    pending_free.clear();
  };
  auto place_outputs = [&](size_t i) {
    for (int t : us[i].outs) {
      if (graph_out.count(t)) {
        outs_written.insert(t);
        continue;
      }
      if (slot.count(t)) continue;
      slot[t] = alloc(local_bytes(t));
    }
  };
  std::set<int> retired;  // a tensor read by several members of a group is freed once
  auto retire_inputs = [&](size_t s) {
    for (size_t i : steps[s])
      for (int t : us[i].ins)
        if (last_step[t] == s && slot.count(t) && !graph_out.count(t) && retired.insert(t).second)
          pending_free.push_back(slot[t]);
  };
  // graph parameters: staged whole into shared memory at kernel entry by
  // the TMA engine (one cp.async.bulk per parameter slice -- a sharded
  // slice is R contiguous rows -- completing on one mbarrier), so every unit
  // reads them on chip; slots are reused after their last reader like any
  // other.  STITCH_RESIDENT_STAGE=0 reads them from global memory instead.
  std::vector<int> staged;
  int64_t staged_bytes = 0;
  {
    const char* st = std::getenv("STITCH_RESIDENT_STAGE");
    const bool stage = !(st && *st == '0');
    std::set<int> ps;
    for (const auto& u : us)
      for (int t : u.ins)
        if (g.node(t).kind == OpKind::Parameter) ps.insert(t);
    for (int t : ps)
      if (stage && local_bytes(t) % 16 == 0 && local_bytes(t) > 0) {
        slot[t] = alloc(local_bytes(t));
        staged.push_back(t);
        staged_bytes += local_bytes(t);
      }
  }
  const std::set<int> staged_set(staged.begin(), staged.end());
  // every CTA writes its rows of each placeholder output with the folded mean
  auto emit_fills = [&](const std::vector<size_t>& grp) {
    for (size_t i : grp) place_outputs(i);
    for (size_t j = 0; j < grp.size(); ++j) {
      const OpNode& n = g.node(us[grp[j]].verts[0]);
      const int64_t nout = local_elems(n.id);
      const bool rep_out = !sharded[static_cast<size_t>(n.id)] && graph_out.count(n.id);
      const std::string guard = rep_out ? "if (rk_ == 0) " : "";
      body << "    { const float fill = rs_fill_[" << j << "];\n";
      if (n.shape.dtype == DType::F32 && nout % 4 == 0)
        body << "      " << guard << "for (int i = threadIdx.x; i < " << nout / 4 << "; i += 1024) st4_g(" << ptr(n.id)
             << " + 4 * i, fill, fill, fill, fill); }\n";
      else
        body << "      " << guard << "for (int i = threadIdx.x; i < " << nout << "; i += 1024) stv(" << ptr(n.id)
             << ", i, fill); }\n";
    }
  };
  // STITCH_RESIDENT_PUSH=0: placeholder partials meet behind a cluster
  // barrier (DSMEM pull) instead of st.async pushes + per-group mbarriers
  int n_push = 0;
  std::map<size_t, std::pair<int, int>> split_of;  // group's first unit -> (mbarrier, inbox slot base)
  bool staged_ready = staged.empty();
  // A local unit consuming another local unit's output needs no barrier
  // when every element reaches it through the thread that wrote it: both
  // are single local bodies over the same domain and vector width, with the
  // same virtual grid (same element-to-thread map: c = v * 1024 + tid,
  // grid-stride), and in the consumer the handed-over tensors (shape = the
  // domain) feed only elementwise ops of that shape (identity coordinates).
  // DIEN: each step's reset-gate unit -> update unit.
  // STITCH_RESIDENT_HANDOFF=0 keeps every barrier.
  const char* hv = std::getenv("STITCH_RESIDENT_HANDOFF");
  const bool handoff = !(hv && *hv == '0') && !tl_no_handoff;
  static const std::regex local_sig(R"(// local body: domain (\d+) elements, vector (\d+))");
  // placeholder members filled "one element per thread" (direct fold below)
  // hand over like a local unit with vector 1 and grid 1
  std::map<size_t, std::string> fill_sig;
  auto local_domain = [&](size_t i) -> std::string {
    if (us[i].opaque) {
      auto it = fill_sig.find(i);
      return it == fill_sig.end() ? "" : it->second;
    }
    if (us[i].spec.tmpl != "local") return "";
    const std::string& src = us[i].spec.source;
    auto it = std::sregex_iterator(src.begin(), src.end(), local_sig);
    if (it == std::sregex_iterator()) return "";
    const std::string sig = it->str(1) + "x" + it->str(2) + "g" + std::to_string(us[i].spec.grid);
    return ++it == std::sregex_iterator() ? sig : "";  // exactly one local body
  };
  auto same_thread_handoff = [&](size_t i, size_t d) {
    if (!handoff) return false;
    const std::string di = local_domain(i), dd = local_domain(d);
    if (di.empty() || di != dd) return false;
    const int64_t n = std::stoll(di.substr(0, di.find('x')));
    bool any = false;
    for (int t : us[d].outs) {
      if (std::find(us[i].ins.begin(), us[i].ins.end(), t) == us[i].ins.end()) continue;
      any = true;
      const TensorShape& ts = gs.node(t).shape;
      if (ts.element_count() != n) return false;
      for (int v : us[i].verts) {
        const OpNode& c = gs.node(v);
        if (std::find(c.operands.begin(), c.operands.end(), t) == c.operands.end()) continue;
        if (!is_elementwise(c.kind) || c.shape.dims != ts.dims) return false;
      }
    }
    return any;
  };
  for (size_t s = 0; s < steps.size(); ++s) {
    if (phase[s] == kGroupB) {
      // the peers' partials: wait, fold in rank order, fill (the barrier
      // inside orders the fillers run since phase A as well)
      const auto& grp = steps[s];
      const auto [bar, base] = split_of.at(grp[0]);
      body << "  STC_TRACE_STAMP_END(" << s << ");\n  STC_TRACE_BEGIN(" << 1 + s << ");\n";
      body << "  {  // placeholder group (wait):";
      for (size_t i : grp) body << " " << g.node(us[i].verts[0]).name;
      // small groups (DIEN's three gates per step): every filling thread
      // folds the C partials itself, in rank order, and writes its share of
      // the fills -- no butterfly, no rs_fill_ round trip, no barrier here
      // (the next reader of the fills barriers as usual).  The group's
      // output slots come only from barrier-protected free slots: the
      // fillers since phase A may still be reading theirs
      // (STITCH_RESIDENT_DIRECT_FOLD=0: butterfly fold + barrier + fill)
      const char* dfv = std::getenv("STITCH_RESIDENT_DIRECT_FOLD");
      if (!(dfv && *dfv == '0') && grp.size() <= 4) {
        for (size_t i : grp) place_outputs(i);
        int64_t most = 1;
        for (size_t i : grp) {
          const OpNode& n = g.node(us[i].verts[0]);
          const int64_t nout = local_elems(n.id);
          most = std::max<int64_t>(most, n.shape.dtype == DType::F32 && nout % 4 == 0 ? nout / 4 : nout);
        }
        // STITCH_RESIDENT_SCALAR_FILL=1 (every member a sharded [<= 1024
        // elements] f32 tensor inside the kernel): thread t folds and writes
        // element t of each -- the map a vector-1 local unit reads with, so
        // that consumer needs no barrier.  Measured slower (576 threads each
        // folding the peers' partials: T=10 19.4 -> 21.8 us,
        // profiles/r02/resident/resident_scalar_fill.jsonl)
        const char* sfv = std::getenv("STITCH_RESIDENT_SCALAR_FILL");
        bool scalar_map = handoff && sfv && *sfv == '1';
        int64_t most_el = 1;
        for (size_t i : grp) {
          const OpNode& n = g.node(us[i].verts[0]);
          most_el = std::max<int64_t>(most_el, local_elems(n.id));
          scalar_map = scalar_map && sharded[static_cast<size_t>(n.id)] && !graph_out.count(n.id) &&
                       n.shape.dtype == DType::F32 && local_elems(n.id) <= 1024;
        }
        if (scalar_map) most = most_el;
        const int T = static_cast<int>(std::min<int64_t>(1024, (most + 31) / 32 * 32));
        body << "\n    if (threadIdx.x < " << T << ") {\n      mbar_wait_cluster(&rs_gbar_[" << bar << "], 0u);\n";
        for (size_t j = 0; j < grp.size(); ++j) body << "      double t" << j << "_ = 0.0;\n";
        body << "      #pragma unroll\n      for (int r_ = 0; r_ < " << C << "; ++r_) {";
        for (size_t j = 0; j < grp.size(); ++j)
          body << " t" << j << "_ += rs_inbox_[(" << base + static_cast<int>(j) << ") * " << C << " + r_];";
        body << " }\n";
        for (size_t j = 0; j < grp.size(); ++j) {
          const OpNode& n = g.node(us[grp[j]].verts[0]);
          int64_t count = 0;
          for (int o : n.operands) count += g.node(o).shape.element_count();
          const int64_t nout = local_elems(n.id);
          const bool rep_out = !sharded[static_cast<size_t>(n.id)] && graph_out.count(n.id);
          const std::string guard = rep_out ? "if (rk_ == 0) " : "";
          body << "      { const float fill = (float)(" << (count ? "t" + std::to_string(j) + "_ * " + inv_count(count) : "0.0")
               << ");\n";
          if (scalar_map) {
            body << "        if (threadIdx.x < " << nout << ") " << ptr(n.id) << "[threadIdx.x] = fill; }\n";
            fill_sig[grp[j]] = std::to_string(nout) + "x1g1";
          } else if (n.shape.dtype == DType::F32 && nout % 4 == 0)
            body << "        " << guard << "for (int i = threadIdx.x; i < " << nout / 4 << "; i += " << T << ") st4_g("
                 << ptr(n.id) << " + 4 * i, fill, fill, fill, fill); }\n";
          else
            body << "        " << guard << "for (int i = threadIdx.x; i < " << nout << "; i += " << T << ") stv(" << ptr(n.id)
                 << ", i, fill); }\n";
        }
        body << "    }\n  }\n";
        for (size_t i : grp) since_barrier.insert(i);
        continue;
      }
      // only the folding warps read the inbox: they alone wait on it (a
      // cluster-scope acquire per thread); the barrier below holds the rest
      body << "\n    if (threadIdx.x < " << 32 * std::min<size_t>(grp.size(), 32)
           << ") mbar_wait_cluster(&rs_gbar_[" << bar << "], 0u);\n";
      body << "    {\n      const int w_ = threadIdx.x >> 5, l_ = threadIdx.x & 31;\n";
      for (size_t j = 0; j < grp.size(); ++j) {
        const OpNode& n = g.node(us[grp[j]].verts[0]);
        int64_t count = 0;
        for (int o : n.operands) count += g.node(o).shape.element_count();
        body << "      if (w_ == " << j % 32 << ") { double t_ = l_ < " << C << " ? rs_inbox_[(" << base + static_cast<int>(j)
             << ") * " << C << " + l_] : 0.0; t_ = bfly_sum(t_, " << fold_w << "); if (l_ == 0) rs_fill_[" << j << "] = (float)("
             << (count ? "t_ * " + inv_count(count) : "0.0") << "); }\n";
      }
      body << "    }\n    __syncthreads();\n";
      ++n_barriers;
      since_barrier.clear();
      free_list.insert(free_list.end(), pending_free.begin(), pending_free.end());
      pending_free.clear();
      emit_fills(grp);
      body << "  }\n";
      for (size_t i : grp) since_barrier.insert(i);
      continue;
    }
    if (!staged_ready) {
      bool reads = false;
      for (size_t i : steps[s])
        for (int t : us[i].ins) reads = reads || staged_set.count(t);
      if (reads) {
        body << "  mbar_wait(&rs_mbar_, 0u);  // staged parameters have landed\n";
        staged_ready = true;
      }
    }
    bool need = false;
    for (size_t i : steps[s])
      for (size_t d : us[i].deps) need = need || (since_barrier.count(d) && !same_thread_handoff(i, d));
    if (need) barrier();
    // diagnostics (STITCH_TRACE builds): slot 1+s = [first CTA entering step
    // s, last CTA leaving it]
    if (s) body << "  STC_TRACE_STAMP_END(" << s << ");\n";
    body << "  STC_TRACE_BEGIN(" << 1 + s << ");\n";
    for (size_t i : steps[s])
      for (int t : us[i].ins)
        if (g.node(t).kind == OpKind::Parameter) params_used.insert(t);
    if (!us[steps[s][0]].opaque) {
      const size_t i = steps[s][0];
      place_outputs(i);
      const std::string canon = as_resident_function(us[i].spec);
      auto it = fn_of.find(canon);
      if (it == fn_of.end()) {
        it = fn_of.emplace(canon, "ru" + std::to_string(fn_of.size()) + "_").first;
        fns << std::regex_replace(canon, std::regex("\\bFN_\\("), it->second + "(") << "\n";
      }
      body << "  // unit " << i << ": " << us[i].spec.tmpl << " {" << g.node(us[i].verts.front()).name
           << (us[i].verts.size() > 1 ? ", ..." : "") << "} grid " << us[i].spec.grid << "\n";
      body << "  for (int v_ = 0; v_ < " << us[i].spec.grid << "; ++v_) " << it->second << "(";
      for (const auto& tn : us[i].spec.inputs) body << ptr(g.by_name.at(tn)) << ", ";
      for (const auto& tn : us[i].spec.outputs) body << ptr(g.by_name.at(tn)) << ", ";
      body << "v_, " << us[i].spec.grid << ");\n";
      since_barrier.insert(i);
      retire_inputs(s);
      // a unit with its own shared scratch (cross-warp team reductions):
      // the next call of the same function must not overwrite it early
      if (canon.find("__shared__") != std::string::npos) barrier();
      continue;
    }
    // a group of opaque placeholders: f64 partials of this CTA's rows,
    // block fold, one cluster barrier, rank-ordered fold of the C partials
    const auto& grp = steps[s];
    max_group = std::max<int>(max_group, static_cast<int>(grp.size()));
    body << "  {  // placeholder group:";
    for (size_t i : grp) body << " " << g.node(us[i].verts[0]).name;
    body << "\n";
    // one f64 partial per DISTINCT operand slice (the group's placeholders
    // share operands: x_t and h_t), then each member adds the partials of
    // its operand list -- an operand listed twice counts twice (opaque_body)
    std::map<int, int> dk;  // operand vertex -> partial index
    for (size_t j : grp)
      for (int o : g.node(us[j].verts[0]).operands) dk.emplace(o, static_cast<int>(dk.size()));
    // small slices (every DIEN operand: 144 float4 per CTA): warp k folds
    // operand k on its own (strided 128-bit loads + one butterfly), all
    // operands in parallel, then thread j adds member j's operand partials;
    // larger ones: block-wide per-thread partials + two-level fold
    bool warp_path = dk.size() <= 32;
    for (auto [o, k] : dk) warp_path = warp_path && local_elems(o) <= 16384;
    // W warps per operand (32 / operands, at most one chunk per lane each):
    // warp k*W + j folds chunks j*32 + lane, step W*32, of operand k; the
    // operand's partial is then the W warp sums added in j order
    // (STITCH_RESIDENT_WARPS caps W; 1 = one warp per operand, the round-2
    // first form: 0.65 us per DIEN step fold, profiles/r02/resident/)
    int W = 1;
    if (warp_path) {
      int64_t most = 1;
      for (auto [o, k] : dk) {
        const int64_t cnt = local_elems(o);
        most = std::max<int64_t>(most, g.node(o).shape.dtype == DType::F32 && cnt % 4 == 0 ? cnt / 4 : cnt);
      }
      const char* wv = std::getenv("STITCH_RESIDENT_WARPS");
      const int wcap = wv && *wv ? std::max(1, std::atoi(wv)) : 32;
      W = static_cast<int>(std::clamp<int64_t>((most + 31) / 32, 1, std::min<int64_t>(wcap, 32 / std::max<size_t>(1, dk.size()))));
    }
    auto operand_partial = [&](int k) {
      std::string e = "rs_red_[" + std::to_string(k * W) + "]";
      for (int j = 1; j < W; ++j) e = "(" + e + " + rs_red_[" + std::to_string(k * W + j) + "])";
      return e;
    };
    if (warp_path) {
      body << "    {\n      const int w_ = threadIdx.x >> 5, l_ = threadIdx.x & 31;\n";
      for (auto [o, k] : dk) {
        const TensorShape& sh = g.node(o).shape;
        const int64_t cnt = local_elems(o);
        const std::string guard = !sharded[static_cast<size_t>(o)] ? " && rk_ == 0" : "";
        body << "      if (w_ >= " << k * W << " && w_ < " << (k + 1) * W << ") { const int j_ = w_ - " << k * W
             << "; double d_ = 0.0;\n        if (true" << guard << ") ";
        if (sh.dtype == DType::F32 && cnt % 4 == 0)
          body << "for (int i = j_ * 32 + l_; i < " << cnt / 4 << "; i += " << 32 * W << ") { const float4 q = ld4_g(" << ptr(o)
               << " + 4 * i); d_ += ((double)q.x + (double)q.y) + ((double)q.z + (double)q.w); }\n";
        else
          body << "for (int i = j_ * 32 + l_; i < " << cnt << "; i += " << 32 * W << ") d_ += (double)ldv_g(" << ptr(o)
               << ", i);\n";
        body << "        d_ = bfly_sum(d_, 32); if (l_ == 0) rs_red_[" << k * W << " + j_] = d_; }\n";
      }
      body << "    }\n    __syncthreads();\n";
      if (pushed(grp)) {
        // push: thread (j, r) sends member j's partial to rank r's inbox
        // (st.async, completing on rank r's mbarrier of this group); every
        // CTA waits only for the C x G partials addressed to it
        body << "    if (threadIdx.x < " << grp.size() * C << ") {\n      const int j_ = threadIdx.x / " << C
             << ", r_ = threadIdx.x % " << C << ";\n      double v_ = 0.0;\n";
        for (size_t j = 0; j < grp.size(); ++j) {
          body << "      " << (j ? "else " : "") << "if (j_ == " << j << ") v_ = 0.0";
          for (int o : g.node(us[grp[j]].verts[0]).operands) body << " + " << operand_partial(dk[o]);
          body << ";\n";
        }
        body << "      st_async_f64(&rs_inbox_[(" << opaque_slots << " + j_) * " << C << " + rk_], v_, &rs_gbar_["
             << n_push << "], (unsigned)r_);\n    }\n"
             << "    if (threadIdx.x == 0) mbar_expect_tx(&rs_gbar_[" << n_push << "], " << grp.size() * C * 8 << "u);\n";
        if (phase[s] == kGroupA) {  // phase B waits, after the fillers
          split_of[grp[0]] = {n_push, opaque_slots};
          ++n_push;
          opaque_slots += static_cast<int>(grp.size());
          body << "  }\n";
          // the barrier after the local fold ordered everything before it
          since_barrier.clear();
          free_list.insert(free_list.end(), pending_free.begin(), pending_free.end());
          pending_free.clear();
          retire_inputs(s);
          continue;
        }
        body << "    if (threadIdx.x < " << 32 * std::min<size_t>(grp.size(), 32) << ") mbar_wait_cluster(&rs_gbar_["
             << n_push << "], 0u);\n";
        ++n_push;
        body << "    {\n      const int w_ = threadIdx.x >> 5, l_ = threadIdx.x & 31;\n";
        for (size_t j = 0; j < grp.size(); ++j) {
          const OpNode& n = g.node(us[grp[j]].verts[0]);
          int64_t count = 0;
          for (int o : n.operands) count += g.node(o).shape.element_count();
          body << "      if (w_ == " << j % 32 << ") { double t_ = l_ < " << C << " ? rs_inbox_[("
               << opaque_slots + static_cast<int>(j) << ") * " << C << " + l_] : 0.0; t_ = bfly_sum(t_, " << fold_w << "); if (l_ == 0) rs_fill_["
               << j << "] = (float)(" << (count ? "t_ * " + inv_count(count) : "0.0") << "); }\n";
        }
        body << "    }\n    __syncthreads();\n";
        emit_fills(grp);
        opaque_slots += static_cast<int>(grp.size());
        body << "  }\n";
        since_barrier.clear();
        free_list.insert(free_list.end(), pending_free.begin(), pending_free.end());
        pending_free.clear();
        for (size_t i : grp) since_barrier.insert(i);
        retire_inputs(s);
        continue;
      }
      for (size_t j = 0; j < grp.size(); ++j) {
        body << "    if (threadIdx.x == " << j << ") rs_part_[" << opaque_slots + static_cast<int>(j) << "] = 0.0";
        for (int o : g.node(us[grp[j]].verts[0]).operands) body << " + " << operand_partial(dk[o]);
        body << ";\n";
      }
      body << "    {\n";
    } else {
      for (auto [o, k] : dk) {
        const TensorShape& sh = g.node(o).shape;
        const int64_t cnt = local_elems(o);
        const std::string guard = !sharded[static_cast<size_t>(o)] ? "if (rk_ == 0) " : "";
        body << "    double d" << k << "_ = 0.0;\n";
        if (sh.dtype == DType::F32 && cnt % 4 == 0)
          body << "    " << guard << "for (int i = threadIdx.x; i < " << cnt / 4 << "; i += 1024) { const float4 q = ld4_g("
               << ptr(o) << " + 4 * i); d" << k << "_ += ((double)q.x + (double)q.y) + ((double)q.z + (double)q.w); }\n";
        else
          body << "    " << guard << "for (int i = threadIdx.x; i < " << cnt << "; i += 1024) d" << k << "_ += (double)ldv_g("
               << ptr(o) << ", i);\n";
      }
      for (size_t j = 0; j < grp.size(); ++j) {
        body << "    { double a_ = 0.0";
        for (int o : g.node(us[grp[j]].verts[0]).operands) body << " + d" << dk[o] << "_";
        body << ";\n      a_ = bfly_sum(a_, 32);\n      if ((threadIdx.x & 31) == 0) rs_red_[" << j * 32
             << " + (threadIdx.x >> 5)] = a_; }\n";
      }
      // warp j folds member j's 32 warp sums into this CTA's partial
      body << "    __syncthreads();\n    {\n      const int w_ = threadIdx.x >> 5, l_ = threadIdx.x & 31;\n";
      for (size_t j = 0; j < grp.size(); ++j)
        body << "      if (w_ == " << j % 32 << ") { const double v_ = bfly_sum(rs_red_[" << j * 32
             << " + l_], 32); if (l_ == 0) rs_part_[" << opaque_slots + static_cast<int>(j) << "] = v_; }\n";
    }
    body << "    }\n    cluster_sync_all();\n";
    ++n_cluster;
    // warp j: lane r reads rank r's partial of member j (DSMEM, all in
    // flight at once); a butterfly folds them in the same order in every CTA
    body << "    {\n      const int w_ = threadIdx.x >> 5, l_ = threadIdx.x & 31;\n";
    for (size_t j = 0; j < grp.size(); ++j) {
      const OpNode& n = g.node(us[grp[j]].verts[0]);
      int64_t count = 0;
      for (int o : n.operands) count += g.node(o).shape.element_count();
      body << "      if (w_ == " << j % 32 << ") { double t_ = l_ < " << C << " ? ld_dsmem_f64(&rs_part_["
           << opaque_slots + static_cast<int>(j) << "], (unsigned)l_) : 0.0; t_ = bfly_sum(t_, " << fold_w << "); if (l_ == 0) rs_fill_["
           << j << "] = (float)(" << (count ? "t_ * " + inv_count(count) : "0.0") << "); }\n";
    }
    body << "    }\n    __syncthreads();\n";
    emit_fills(grp);
    body << "  }\n";
    opaque_slots += static_cast<int>(grp.size());
    // the cluster barrier ordered everything before it
    since_barrier.clear();
    free_list.insert(free_list.end(), pending_free.begin(), pending_free.end());
    pending_free.clear();
    for (size_t i : grp) since_barrier.insert(i);
    retire_inputs(s);
  }
  body << "  STC_TRACE_STAMP_END(" << steps.size() << ");\n";
  if (smem_top > kSmemCap) {
    *smem_bound = true;
    return no("boundary tensors need " + std::to_string(smem_top) + " B of shared memory per CTA");
  }

  KernelSpec k;
  k.name = name;
  k.tmpl = "resident(" + std::to_string(us.size()) + " units, " + std::to_string(steps.size()) + " steps, cluster " +
           std::to_string(C) + ")";
  k.grid = C;
  k.block = 1024;
  k.cluster = C;
  k.smem = std::max<int64_t>(smem_top, 16);
  // STITCH_RESIDENT_LOOP=1 rolls the recurrent steps into one loop.  Off by
  // default: it removes most instruction-fetch stalls of a cold launch (ncu:
  // no_instructions 67 -> 17 samples, 28.7 -> 26.3 us) but back-to-back
  // launches find the straight-line code warm in L2, and the loop's table
  // loads and switch add 15% instructions: T=10 20.1 -> 22.7 us, T=20
  // 36.8 -> 42.8 us (profiles/r02/resident/resident_loop.jsonl)
  std::string body_src = body.str(), tab_decl;
  int loop_iters = 0;
  if (const char* lv = std::getenv("STITCH_RESIDENT_LOOP"); lv && *lv == '1')
    body_src = loop_recurrence(body_src, "rs_tab_" + name, &tab_decl, &loop_iters);
  if (loop_iters) k.tmpl += ", loop " + std::to_string(loop_iters);
  std::ostringstream s;
  s << fns.str() << tab_decl;
  s << "extern \"C\" __global__ void __launch_bounds__(1024, 1) " << name << "(";
  bool first = true;
  for (int t : params_used) {
    s << (first ? "" : ", ") << "const " << c_type(g.node(t).shape.dtype) << "* " << tensor_ident(g.node(t).name);
    k.inputs.push_back(g.node(t).name);
    first = false;
  }
  for (int t : outs_written) {
    s << (first ? "" : ", ") << c_type(g.node(t).shape.dtype) << "* " << tensor_ident(g.node(t).name);
    k.outputs.push_back(g.node(t).name);
    first = false;
  }
  s << ") {\n"
    << "  // " << B << " batch rows, " << R << " per CTA; " << us.size() << " plan units in " << steps.size()
    << " steps, " << n_barriers << " CTA barriers, " << n_cluster << " cluster barriers; " << smem_top
    << " B of boundary tensors per CTA\n"
    << "  extern __shared__ __align__(128) unsigned char rs_smem_[];\n"
    << "  __shared__ double rs_red_[" << 32 * max_group << "];\n"
    << "  __shared__ double rs_part_[" << std::max(1, opaque_slots) << "];\n"
    << "  __shared__ float rs_fill_[" << max_group << "];\n"
    << (n_push ? "  __shared__ double rs_inbox_[" + std::to_string(opaque_slots * C) + "];\n"
                 "  __shared__ __align__(8) unsigned long long rs_gbar_[" + std::to_string(n_push) + "];\n" : std::string())
    << "  const int rk_ = (int)cluster_ctarank();\n  (void)rk_;\n";
  // the parameter staging is issued first: its HBM round trip then overlaps
  // the cluster barrier that publishes the inbox mbarriers below
  if (!staged.empty()) {
    s << "  __shared__ __align__(8) unsigned long long rs_mbar_;\n"
      << "  if (threadIdx.x == 0) {\n    mbar_init(&rs_mbar_, 1);\n    mbar_fence_init();\n"
      << "    mbar_expect_tx(&rs_mbar_, " << staged_bytes << "u);\n";
    for (int t : staged) {
      const std::string off = sharded[static_cast<size_t>(t)] ? " + (i64)rk_ * " + std::to_string(local_elems(t)) : "";
      s << "    bulk_g2s(rs_smem_ + " << slot[t].off << ", " << tensor_ident(g.node(t).name) << off << ", "
        << local_bytes(t) << "u, &rs_mbar_);\n";
    }
    s << "  }\n";
    if (!n_push) s << "  __syncthreads();  // the mbarrier is initialised before anyone waits on it\n";
  }
  if (n_push) {  // peers push into our inbox only after every mbarrier of the cluster is initialised
    s << "  if (threadIdx.x < " << n_push << ") mbar_init(&rs_gbar_[threadIdx.x], 1);\n"
      << "  if (threadIdx.x == 0) mbar_fence_init();\n  cluster_sync_all();  // also orders rs_mbar_'s init before any wait\n";
  }
  s << body_src
    << "  cluster_sync_all();  // peers may still read rs_part_ through DSMEM\n}\n";
  k.source = s.str();
  for (const auto& u : us) k.alg_bytes += u.opaque ? 0 : u.spec.alg_bytes;
  for (const auto& u : us)
    if (u.opaque) {
      const OpNode& n = g.node(u.verts[0]);
      k.alg_bytes += n.shape.byte_size();
      for (int o : u.ins) k.alg_bytes += g.node(o).shape.byte_size();
    }
  return k;
}

}  // namespace stitch::gpu
