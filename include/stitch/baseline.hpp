// stitch-b200: rule-based XLA-like fuser used only to report "baseline
// kernels" beside the stitched plan (drop-in for include/stitch/baseline.hpp).
#pragma once

#include "stitch/graph.hpp"

namespace stitch {

FusionPlan run_baseline(const CompGraph& g);
int kernel_count(const CompGraph& g, const FusionPlan& plan);

}  // namespace stitch
