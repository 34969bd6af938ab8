// plan.json (the plan-parity artifact) and the DOT rendering.
// Field order and value formatting follow /root/reference/proj/src/pipeline.cpp:45-108;
// doubles are printed by the same third-party serializer (nlohmann/json
// 3.11.3 ordered_json, dump(2)) so the bytes match.
#include <cstdio>
#include <set>
#include <sstream>

#include <json.hpp>

#include "stitch/pipeline.hpp"

namespace stitch {

std::string plan_to_json(const CompGraph& g, const FusionPlan& plan,
                         const std::map<std::string, KernelPlan>& kernels, int stitched_kernels,
                         int baseline_kernels, uint64_t seed) {
  using nlohmann::ordered_json;
  ordered_json doc;
  doc["total_score"] = plan.total_score;
  doc["stitched_kernels"] = stitched_kernels;
  doc["baseline_kernels"] = baseline_kernels;
  doc["seed"] = seed;
  ordered_json pats = ordered_json::array();
  for (const auto& p : plan.patterns) {
    ordered_json jp;
    jp["key"] = p.key();
    jp["producer"] = g.node(p.producer).name;
    jp["remote"] = p.remote;
    jp["score"] = p.score;
    ordered_json names = ordered_json::array();
    for (int v : p.vertices) names.push_back(g.node(v).name);
    jp["vertices"] = std::move(names);
    if (auto it = kernels.find(p.key()); it != kernels.end()) {
      const KernelPlan& k = it->second;
      jp["launch"] = {{"grid", k.launch.grid}, {"block", k.launch.block}};
      jp["shmem_bytes"] = k.shmem_total();
      jp["regs_per_thread"] = k.regs_per_thread;
      jp["occupancy"] = k.occupancy_value;
      jp["estimated_cycles"] = k.estimated_cycles;
      ordered_json sched;
      for (const auto& [v, t] : k.per_op_schedule) sched[g.node(v).name] = t;
      jp["schedule"] = std::move(sched);
    }
    pats.push_back(std::move(jp));
  }
  doc["patterns"] = std::move(pats);
  return doc.dump(2) + "\n";
}

namespace {
std::string g6(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.6g", v);
  return b;
}
}  // namespace

std::string graph_to_dot(const CompGraph& g, const FusionPlan& plan) {
  std::ostringstream o;
  o << "digraph stitched {\n  rankdir=TB;\n  node [shape=box, fontname=\"monospace\"];\n";
  std::set<int> covered;
  auto label = [&](const OpNode& n) {
    return "\"" + n.name + "\" [label=\"" + n.name + "\\n" + kind_name(n.kind) + " " + n.shape.str() + "\"";
  };
  for (size_t i = 0; i < plan.patterns.size(); ++i) {
    const auto& p = plan.patterns[i];
    o << "  subgraph cluster_" << i << " {\n    label=\"pattern " << i << "  f=" << g6(p.score)
      << "\";\n    style=rounded;\n";
    for (int v : p.vertices) {
      covered.insert(v);
      o << "    " << label(g.node(v)) << "];\n";
    }
    o << "  }\n";
  }
  for (const auto& n : g.nodes) {
    if (covered.count(n.id)) continue;
    o << "  " << label(n);
    if (!is_fusable(n) && classify_op(n) != OpClass::Opaque) o << ", style=dashed";
    o << "];\n";
  }
  for (const auto& n : g.nodes)
    for (int src : n.operands) o << "  \"" << g.node(src).name << "\" -> \"" << n.name << "\";\n";
  o << "}\n";
  return o.str();
}

}  // namespace stitch
