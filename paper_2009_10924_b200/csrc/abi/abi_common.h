// Shared state behind the extern "C" handles (include/stitch_b200.h).
#pragma once

#include <map>
#include <memory>
#include <stdexcept>
#include <string>

#include "stitch/explorer.hpp"
#include "stitch/graph.hpp"
#include "stitch/parser.hpp"
#include "stitch/planner.hpp"
#include "stitch_b200.h"

namespace stitch::gpu {
class Executor;
class CudaError;
}

struct stc_graph {
  stitch::CompGraph g;
};

struct stc_plan {
  stitch::CompGraph graph;
  stitch::CostModels models;
  stitch::FusionPlan plan;
  std::map<std::string, stitch::KernelPlan> kernels;
  int stitched = 0, baseline = 0;
  int64_t refine_probes = 0;   // last stc_plan_refine: feasibility probes spent
  int refine_budget_hit = 0;   // ... and whether STITCH_REFINE_MAX_PROBES stopped it
};

namespace stc_abi {

extern thread_local std::string g_error;
char* dup_string(const std::string& s);
stitch::MachineModel model_for(const char* cfg_path);

// Runs f, mapping exceptions onto the ABI's status codes (no exception
// crosses the boundary).
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const stitch::ParseError& e) {
    g_error = "[parser] " + e.code + ": " + e.what() +
              (e.line ? " (line " + std::to_string(e.line) + ")" : std::string());
    return 1;
  } catch (const std::invalid_argument& e) {
    g_error = std::string("[abi] ") + e.what();
    return 4;
  } catch (const std::exception& e) {
    g_error = e.what();
    const std::string& m = g_error;
    if (m.rfind("[cuda]", 0) == 0 || m.rfind("[nvrtc]", 0) == 0) return 3;
    if (m.rfind("[sim]", 0) == 0) return 2;
    return 1;
  }
}

}  // namespace stc_abi
