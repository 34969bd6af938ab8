// extern "C" boundary, host half: graph IR and planning (include/stitch_b200.h).
#include <cstdlib>
#include <cstring>
#include <memory>

#include "abi/abi_common.h"
#include "codegen/cg.hpp"
#include "stitch/baseline.hpp"
#include "stitch/parser.hpp"
#include "stitch/pipeline.hpp"

using namespace stitch;

namespace stc_abi {

thread_local std::string g_error;

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  return p;
}

MachineModel model_for(const char* cfg_path) {
  if (cfg_path && *cfg_path) return load_machine_model(cfg_path);
  return machine_model_from_env();
}

}  // namespace stc_abi

using namespace stc_abi;

extern "C" {

const char* stc_last_error(void) { return g_error.c_str(); }
void stc_free(void* p) { std::free(p); }
const char* stc_version(void) { return "stitch-b200 0.1 (sm_100a)"; }

int stc_graph_parse(const char* text, stc_graph** out) {
  return guarded([&] {
    auto g = std::make_unique<stc_graph>();
    g->g = parse_graph(text ? text : "");
    *out = g.release();
  });
}

void stc_graph_destroy(stc_graph* g) { delete g; }

int stc_graph_serialize(const stc_graph* g, char** out) {
  return guarded([&] { *out = dup_string(serialize_graph(g->g)); });
}

int stc_graph_num_nodes(const stc_graph* g) { return g ? g->g.num_nodes() : -1; }

int stc_graph_io(const stc_graph* g, int which, int i, const char** name, int* dtype, int* rank,
                 int64_t* dims) {
  std::vector<int> ids;
  if (which == 0) {
    for (const auto& n : g->g.nodes)
      if (n.kind == OpKind::Parameter) ids.push_back(n.id);
  } else {
    ids = g->g.outputs;
  }
  if (i < 0) return static_cast<int>(ids.size());
  if (i >= static_cast<int>(ids.size())) {
    g_error = "stc_graph_io: index out of range";
    return -1;
  }
  const OpNode& n = g->g.node(ids[static_cast<size_t>(i)]);
  if (name) *name = n.name.c_str();
  if (dtype) *dtype = static_cast<int>(n.shape.dtype);
  if (rank) *rank = n.shape.rank();
  if (dims)
    for (int a = 0; a < n.shape.rank() && a < 8; ++a) dims[a] = n.shape.dims[static_cast<size_t>(a)];
  return static_cast<int>(ids.size());
}

int stc_plan_create(const stc_graph* g, const char* cfg_path, int k, int beam, stc_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<stc_plan>();
    p->graph = g->g;
    p->models.machine = model_for(cfg_path);
    if (k > 0) p->models.machine.search.k = k;
    if (beam > 0) p->models.machine.search.beam_width = beam;
    std::vector<std::string> warnings;
    p->plan = explore_fusion_plan(p->graph, p->models, &warnings);
    for (const auto& pat : p->plan.patterns) {
      const KernelPlan* kp = p->models.plan_for(pat, p->graph);
      if (!kp) throw std::runtime_error("[planner] no feasible kernel for pattern " + pat.key());
      p->kernels[pat.key()] = *kp;
    }
    p->stitched = kernel_count(p->graph, p->plan);
    p->baseline = kernel_count(p->graph, run_baseline(p->graph));
    *out = p.release();
  });
}

int stc_plan_from_patterns(const stc_graph* g, const char* cfg_path, const int* verts,
                           const int* offs, int n_patterns, stc_plan** out) {
  return guarded([&] {
    auto p = std::make_unique<stc_plan>();
    p->graph = g->g;
    p->models.machine = model_for(cfg_path);
    for (int i = 0; i < n_patterns; ++i) {
      FusionPattern pat;
      pat.vertices.assign(verts + offs[i], verts + offs[i + 1]);
      std::sort(pat.vertices.begin(), pat.vertices.end());
      pat.producer = pat.vertices.front();
      pat.score = delta_evaluate(pat, p->graph, p->models).f;
      const KernelPlan* kp = p->models.plan_for(pat, p->graph);
      if (!kp) throw std::runtime_error("[planner] no feasible kernel for pattern " + pat.key());
      p->kernels[pat.key()] = *kp;
      p->plan.patterns.push_back(pat);
      p->plan.total_score += pat.score;
    }
    p->stitched = kernel_count(p->graph, p->plan);
    p->baseline = kernel_count(p->graph, run_baseline(p->graph));
    *out = p.release();
  });
}

void stc_plan_destroy(stc_plan* p) { delete p; }

int stc_plan_json(const stc_plan* p, uint64_t seed, char** out) {
  return guarded([&] {
    *out = dup_string(plan_to_json(p->graph, p->plan, p->kernels, p->stitched, p->baseline, seed));
  });
}

int stc_plan_num_patterns(const stc_plan* p) { return static_cast<int>(p->plan.patterns.size()); }

int stc_plan_pattern(const stc_plan* p, int i, int* verts, int cap) {
  const auto& vs = p->plan.patterns.at(static_cast<size_t>(i)).vertices;
  for (int j = 0; j < cap && j < static_cast<int>(vs.size()); ++j) verts[j] = vs[static_cast<size_t>(j)];
  return static_cast<int>(vs.size());
}

int stc_plan_kernel_text(const stc_plan* p, int i, char** out) {
  return guarded([&] {
    const auto& pat = p->plan.patterns.at(static_cast<size_t>(i));
    *out = dup_string(emit_kernel_text(p->kernels.at(pat.key())));
  });
}

int stc_plan_refine(stc_plan* p, int* merges, int64_t* bytes_saved) {
  return guarded([&] {
    stitch::gpu::RefineStats st;
    p->plan = stitch::gpu::refine_plan(p->graph, p->plan, p->models.machine, p->kernels, &st);
    p->stitched = kernel_count(p->graph, p->plan);
    if (merges) *merges = st.merges;
    if (bytes_saved) *bytes_saved = st.bytes_saved;
    p->refine_probes = st.probes;
    p->refine_budget_hit = st.budget_hit ? 1 : 0;
  });
}

int stc_plan_refine_info(const stc_plan* p, int64_t* probes, int* budget_hit) {
  if (probes) *probes = p->refine_probes;
  if (budget_hit) *budget_hit = p->refine_budget_hit;
  return 0;
}

int stc_plan_stats(const stc_plan* p, int* stitched, int* baseline, int64_t* calls) {
  if (stitched) *stitched = p->stitched;
  if (baseline) *baseline = p->baseline;
  if (calls) *calls = p->models.delta_evaluate_calls;
  return 0;
}

int stc_plan_kernel(const stc_graph* g, const char* cfg_path, const int* verts, int n,
                    char** program_text) {
  bool feasible = true;
  int rc = guarded([&] {
    FusionPattern pat;
    pat.vertices.assign(verts, verts + n);
    std::sort(pat.vertices.begin(), pat.vertices.end());
    pat.producer = pat.vertices.front();
    auto kp = plan_kernel(pat, g->g, model_for(cfg_path));
    if (!kp) {
      feasible = false;
      return;
    }
    *program_text = dup_string(emit_kernel_text(*kp));
  });
  if (rc == 0 && !feasible) {
    g_error = "[planner] pattern is infeasible";
    return 1;
  }
  return rc;
}

}  // extern "C"
