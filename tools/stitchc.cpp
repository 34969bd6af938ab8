// stitchc — drop-in for the reference's CLI (proj/tools/stitchc.cpp:8-18):
// same flags, same RunConfig, same exit codes; --run-sim executes the plan on
// the B200.  CLI11 is not available here, so flags are parsed by hand
// (`--name value` or `--name=value`).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "stitch/pipeline.hpp"

namespace {

void usage() {
  std::fprintf(stderr,
               "usage: stitchc --graph FILE [--device-config FILE] [--k N] [--beam-width N] [--out DIR]\n"
               "               [--emit-dot] [--run-sim] [--run-baseline] [--seed N]\n");
}

bool positive(const std::string& v, int* out) {
  char* end = nullptr;
  const long x = std::strtol(v.c_str(), &end, 10);
  if (!end || *end || x <= 0) return false;
  *out = static_cast<int>(x);
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  stitch::RunConfig cfg;
  bool have_graph = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i], v;
    const auto eq = a.find('=');
    if (eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    auto value = [&]() -> std::string {
      if (eq != std::string::npos) return v;
      if (i + 1 >= argc) {
        std::fprintf(stderr, "%s: missing value\n", a.c_str());
        std::exit(106);
      }
      return argv[++i];
    };
    if (a == "--graph") {
      cfg.graph_path = value();
      have_graph = true;
    } else if (a == "--device-config") {
      cfg.device_config_path = value();
    } else if (a == "--k" || a == "--beam-width") {
      int x = 0;
      if (!positive(value(), &x)) {
        std::fprintf(stderr, "%s: value must be a positive number\n", a.c_str());
        return 105;
      }
      (a == "--k" ? cfg.k : cfg.beam_width) = x;
    } else if (a == "--out") {
      cfg.output_dir = value();
    } else if (a == "--emit-dot") {
      cfg.emit_dot = true;
    } else if (a == "--run-sim") {
      cfg.run_sim = true;
    } else if (a == "--run-baseline") {
      cfg.run_baseline = true;
    } else if (a == "--seed") {
      cfg.seed = std::strtoull(value().c_str(), nullptr, 10);
    } else if (a == "-h" || a == "--help") {
      usage();
      return 0;
    } else {
      std::fprintf(stderr, "unknown option: %s\n", a.c_str());
      usage();
      return 109;
    }
  }
  if (!have_graph) {
    std::fprintf(stderr, "--graph is required\n");
    usage();
    return 106;
  }
  return stitch::run_pipeline(cfg);
}
