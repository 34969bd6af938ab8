// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver around the UNMODIFIED reference library, which
// oracle/Makefile compiles from /root/reference/proj/src/*.cpp into
// oracle/_ref/libstitch_ref.so.  Nothing in the product links or loads this;
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs do, as the checker and the CPU baseline.
//
// Entry points mirror the reference's public API:
//   ref_plan        parse_graph -> explore_fusion_plan -> plan_for ->
//                   run_baseline/kernel_count -> plan_to_json
//                   (/root/reference/proj/src/pipeline.cpp:110-150)
//   ref_serialize   serialize_graph (src/parser.cpp:259-285)
//   ref_random      random_inputs   (src/sim.cpp:630-659)
//   ref_eval        eval_reference  (src/sim.cpp:231-250)
//   ref_eval_plan   eval_plan       (src/sim.cpp:471-514)  (SIMT interpreter)
//   ref_run_pipeline run_pipeline (src/pipeline.cpp:110-224): plan.json,
//                   kernels/*.stitch, report.txt, graph.dot artifacts
//   ref_time_eval   best-of-N wall time of eval_reference over K shard graphs
//                   run concurrently on K host threads
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "stitch/baseline.hpp"
#include "stitch/explorer.hpp"
#include "stitch/parser.hpp"
#include "stitch/pipeline.hpp"
#include "stitch/planner.hpp"
#include "stitch/sim.hpp"

using namespace stitch;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  return p;
}

MachineModel model_for(const char* cfg_path) {
  if (cfg_path && *cfg_path) return load_machine_model(cfg_path);
  return default_machine_model();
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    g_err = "[parser] " + e.code + ": " + e.what();
    return 1;
  } catch (const SimFault& e) {
    g_err = std::string("[sim] ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("[ref] ") + e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_run_pipeline(const char* graph_path, const char* cfg_path, int k, int beam, const char* out_dir,
                     int emit_dot, int run_sim, int run_baseline, uint64_t seed) {
  RunConfig c;
  c.graph_path = graph_path;
  c.device_config_path = cfg_path ? cfg_path : "";
  c.k = k;
  c.beam_width = beam;
  c.output_dir = out_dir;
  c.emit_dot = emit_dot != 0;
  c.run_sim = run_sim != 0;
  c.run_baseline = run_baseline != 0;
  c.seed = seed;
  return run_pipeline(c);
}
void ref_free(void* p) { std::free(p); }

// plan.json exactly as run_pipeline writes it, plus every kernel's program
// text ("=== <key>\n<text>" blocks) and a small summary line.
int ref_plan(const char* graph_text, const char* cfg_path, int k, int beam, uint64_t seed,
             char** plan_json, char** kernels_text, char** summary) {
  return guarded([&] {
    CompGraph g = parse_graph(graph_text);
    CostModels models;
    models.machine = model_for(cfg_path);
    if (k > 0) models.machine.search.k = k;
    if (beam > 0) models.machine.search.beam_width = beam;
    std::vector<std::string> warnings;
    FusionPlan plan = explore_fusion_plan(g, models, &warnings);
    std::map<std::string, KernelPlan> kernels;
    std::string ktext;
    for (const auto& p : plan.patterns) {
      const KernelPlan* kp = models.plan_for(p, g);
      if (!kp) throw std::runtime_error("no feasible kernel for pattern " + p.key());
      kernels[p.key()] = *kp;
      ktext += "=== " + p.key() + "\n" + emit_kernel_text(*kp);
    }
    FusionPlan base = run_baseline(g);
    int stitched = kernel_count(g, plan);
    int baseline = kernel_count(g, base);
    *plan_json = dup(plan_to_json(g, plan, kernels, stitched, baseline, seed));
    *kernels_text = dup(ktext);
    *summary = dup("stitched " + std::to_string(stitched) + " baseline " +
                   std::to_string(baseline) + " delta_calls " +
                   std::to_string(models.delta_evaluate_calls));
  });
}

// plan_kernel for an explicit vertex set (ids), program text out; rc 3 = infeasible
int ref_plan_kernel(const char* graph_text, const char* cfg_path, const int* verts, int n,
                    char** program_text) {
  int feasible = 1;
  int rc = guarded([&] {
    CompGraph g = parse_graph(graph_text);
    MachineModel m = model_for(cfg_path);
    FusionPattern p;
    p.vertices.assign(verts, verts + n);
    p.producer = p.vertices.front();
    auto kp = plan_kernel(p, g, m);
    if (!kp) {
      feasible = 0;
      return;
    }
    *program_text = dup(emit_kernel_text(*kp));
  });
  if (rc == 0 && !feasible) return 3;
  return rc;
}

int ref_serialize(const char* graph_text, char** out) {
  return guarded([&] { *out = dup(serialize_graph(parse_graph(graph_text))); });
}

// random_inputs: fills the parameters in declaration order into caller
// buffers (doubles; values already rounded to the parameter dtype)
int ref_random(const char* graph_text, uint64_t seed, double** bufs, int n) {
  return guarded([&] {
    CompGraph g = parse_graph(graph_text);
    TensorMap in = random_inputs(g, seed);
    int i = 0;
    for (const auto& node : g.nodes) {
      if (node.kind != OpKind::Parameter) continue;
      if (i >= n) throw std::runtime_error("too few buffers");
      const auto& d = in.at(node.name).data;
      std::memcpy(bufs[i++], d.data(), d.size() * sizeof(double));
    }
  });
}

namespace {
TensorMap pack_inputs(const CompGraph& g, const double* const* ins, int n_in) {
  TensorMap in;
  int i = 0;
  for (const auto& node : g.nodes) {
    if (node.kind != OpKind::Parameter) continue;
    if (i >= n_in) throw std::runtime_error("too few inputs");
    TensorValue t = TensorValue::zeros(node.shape);
    std::memcpy(t.data.data(), ins[i++], t.data.size() * sizeof(double));
    in[node.name] = std::move(t);
  }
  return in;
}
void unpack_outputs(const CompGraph& g, const TensorMap& out, double** outs, int n_out) {
  int i = 0;
  for (int o : g.outputs) {
    if (i >= n_out) throw std::runtime_error("too few output buffers");
    const auto& d = out.at(g.node(o).name).data;
    std::memcpy(outs[i++], d.data(), d.size() * sizeof(double));
  }
}
}  // namespace

// eval_reference: parameters in declaration order, outputs in g.outputs order
int ref_eval(const char* graph_text, const double* const* ins, int n_in, double** outs,
             int n_out) {
  return guarded([&] {
    CompGraph g = parse_graph(graph_text);
    unpack_outputs(g, eval_reference(g, pack_inputs(g, ins, n_in)), outs, n_out);
  });
}

// eval_plan with the reference's own plan (explore + plan_for under cfg)
int ref_eval_plan(const char* graph_text, const char* cfg_path, const double* const* ins,
                  int n_in, double** outs, int n_out) {
  return guarded([&] {
    CompGraph g = parse_graph(graph_text);
    CostModels models;
    models.machine = model_for(cfg_path);
    FusionPlan plan = explore_fusion_plan(g, models);
    std::map<std::string, KernelPlan> kernels;
    for (const auto& p : plan.patterns) kernels[p.key()] = *models.plan_for(p, g);
    unpack_outputs(g, eval_plan(g, plan, kernels, pack_inputs(g, ins, n_in)), outs, n_out);
  });
}

// Best-of-`reps` wall seconds of eval_reference, one host thread per shard
// graph, all shards concurrently; inputs are random_inputs(shard, seed).
int ref_time_eval(const char* const* shard_texts, int n_shards, uint64_t seed, int reps,
                  double* best_seconds) {
  return guarded([&] {
    std::vector<CompGraph> gs;
    std::vector<TensorMap> ins;
    for (int i = 0; i < n_shards; ++i) {
      gs.push_back(parse_graph(shard_texts[i]));
      ins.push_back(random_inputs(gs.back(), seed));
    }
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int i = 0; i < n_shards; ++i)
        th.emplace_back([&, i] { volatile auto n = eval_reference(gs[i], ins[i]).size(); (void)n; });
      for (auto& t : th) t.join();
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (s < best) best = s;
    }
    *best_seconds = best;
  });
}

}  // extern "C"
