// Non-parity plan refinement: the extended cost terms of SURVEY.md §8f item 1
// (HBM bytes and launch count), applied after the reference's explorer.
//
// The reference explorer scores candidate patterns with the latency model and
// keeps a top-k / beam search (src/explorer.cpp:151-406); on graphs such as
// the full BERT layer it leaves LayerNorm's affine tail, the broadcast of
// beta and tiny constant broadcasts as separate kernels whose tensors make a
// full round trip through HBM.  refine_plan() starts from that plan and
// greedily merges a launch unit into a unit that consumes it whenever
//   * the merged vertex set is a valid pattern: no opaque op, no cycle in the
//     contracted graph (contraction_creates_cycle), feasible for the
//     reference's own plan_kernel (so a KernelPlan / .stitch program exists),
//     and expressible by a dataflow stitching template;
//   * it saves HBM bytes (algorithmic bytes of the two kernels minus those of
//     the merged one) or at least a launch.
// Best gain first, until no merge applies.  Parity mode never calls this.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <map>
#include <set>

#include "codegen/cg.hpp"
#include "stitch/baseline.hpp"

namespace stitch::gpu {

namespace {

struct Unit {
  std::vector<int> verts;  // ascending
  bool opaque = false;
  bool alive = true;
};

std::vector<int> merged(const std::vector<int>& a, const std::vector<int>& b) {
  std::vector<int> m;
  std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(m));
  return m;
}

}  // namespace

FusionPlan refine_plan(const CompGraph& g, const FusionPlan& plan, const MachineModel& model,
                       std::map<std::string, KernelPlan>& kernels, RefineStats* stats) {
  // launch units exactly as the executor forms them: patterns, uncovered
  // fusable vertices (singletons), opaque ops
  std::vector<Unit> units;
  std::vector<int> unit_of(g.nodes.size(), -1);
  for (const auto& p : plan.patterns) {
    units.push_back({p.vertices, false, true});
    for (int v : p.vertices) unit_of[static_cast<size_t>(v)] = static_cast<int>(units.size()) - 1;
  }
  for (const auto& n : g.nodes) {
    if (unit_of[static_cast<size_t>(n.id)] >= 0) continue;
    const bool opaque = classify_op(n) == OpClass::Opaque;
    if (!opaque && (!is_fusable(n) || n.kind == OpKind::Constant)) continue;
    units.push_back({{n.id}, opaque, true});
    unit_of[static_cast<size_t>(n.id)] = static_cast<int>(units.size()) - 1;
  }
  const auto cons = g.consumer_lists();
  std::map<std::vector<int>, bool> feasible_memo;
  // plan_kernel is the expensive part (the reference emitter on the merged
  // pattern): bound the merged size and the number of feasibility probes --
  // a count, not a clock, so the refined plan never depends on host speed
  const char* bs = std::getenv("STITCH_REFINE_MAX_PROBES");
  const int64_t max_probes = bs && *bs ? std::atoll(bs) : 2000;
  const char* ms = std::getenv("STITCH_REFINE_MAX_VERTS");
  const int max_verts = std::min(model.search.max_pattern_size, ms && *ms ? std::atoi(ms) : 64);
  RefineStats st;
  auto out_of_time = [&] { return st.probes >= max_probes; };
  auto feasible = [&](const std::vector<int>& verts) {
    if (auto it = feasible_memo.find(verts); it != feasible_memo.end()) return it->second;
    ++st.probes;
    bool ok = static_cast<int>(verts.size()) <= max_verts;
    FusionPattern p;
    p.vertices = verts;
    p.producer = verts.front();
    ok = ok && !contraction_creates_cycle(g, p);
    if (ok) {
      try {
        generate_pattern_kernel(g, verts, "refine_probe", 148);
      } catch (const TemplateMismatch&) {
        ok = false;
      }
    }
    if (ok) {
      auto kp = plan_kernel(p, g, model);
      ok = kp.has_value();
      if (ok) kernels[p.key()] = std::move(*kp);
    }
    feasible_memo[verts] = ok;
    return ok;
  };
  while (!out_of_time()) {
    // candidate merges: (producer unit, consumer unit) pairs along graph edges
    struct Cand {
      int64_t gain;
      int a, b;
    };
    std::vector<Cand> cands;
    std::set<std::pair<int, int>> seen;
    for (size_t ua = 0; ua < units.size(); ++ua) {
      const Unit& A = units[ua];
      if (!A.alive || A.opaque) continue;
      for (int v : A.verts)
        for (int c : cons[static_cast<size_t>(v)]) {
          const int ub = unit_of[static_cast<size_t>(c)];
          if (ub < 0 || ub == static_cast<int>(ua) || units[static_cast<size_t>(ub)].opaque) continue;
          if (!seen.insert({static_cast<int>(ua), ub}).second) continue;
          const auto m = merged(A.verts, units[static_cast<size_t>(ub)].verts);
          const int64_t saved = algorithmic_bytes(g, A.verts) + algorithmic_bytes(g, units[static_cast<size_t>(ub)].verts) -
                                algorithmic_bytes(g, m);
          if (saved < 0) continue;
          cands.push_back({saved, static_cast<int>(ua), ub});
        }
    }
    std::sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) {
      return x.gain != y.gain ? x.gain > y.gain : std::make_pair(x.a, x.b) < std::make_pair(y.a, y.b);
    });
    bool done = false;
    for (const Cand& c : cands) {
      if (out_of_time()) break;
      Unit& A = units[static_cast<size_t>(c.a)];
      Unit& B = units[static_cast<size_t>(c.b)];
      const auto m = merged(A.verts, B.verts);
      if (!feasible(m)) continue;
      A.verts = m;
      B.alive = false;
      for (int v : m) unit_of[static_cast<size_t>(v)] = c.a;
      ++st.merges;
      st.bytes_saved += c.gain;
      done = true;
      break;
    }
    if (!done) break;
  }
  FusionPlan out;
  for (const Unit& u : units) {
    if (!u.alive || u.opaque) continue;
    if (u.verts.size() == 1 && !kernels.count(std::to_string(u.verts[0]))) {
      // an unmerged singleton stays uncovered (the executor launches it as
      // before) unless it was a pattern of the original plan
      bool was_pattern = false;
      for (const auto& p : plan.patterns) was_pattern = was_pattern || p.vertices == u.verts;
      if (!was_pattern) continue;
    }
    FusionPattern p;
    p.vertices = u.verts;
    p.producer = u.verts.front();
    for (const auto& q : plan.patterns)  // keep the reference's producer/remote flag when unchanged
      if (q.vertices == u.verts) p = q;
    out.patterns.push_back(p);
  }
  std::sort(out.patterns.begin(), out.patterns.end(),
            [](const FusionPattern& x, const FusionPattern& y) { return x.vertices.front() < y.vertices.front(); });
  st.budget_hit = out_of_time();
  if (stats) *stats = st;
  return out;
}

}  // namespace stitch::gpu
