// stitch-b200: abstract stitched-kernel program (drop-in for the reference's
// include/stitch/program.hpp; text format of src/program.cpp).
//
// On B200 this program is the *semantic specification* of a planned kernel:
// the planner emits it exactly as the reference does (its instruction
// histogram and register liveness drive plan selection), and the code
// generator (paper_2009_10924_b200/csrc/codegen) produces an sm_100a kernel
// that computes the same outputs — either through a dataflow template
// (local / regional / global / independent) or, for anything else, by
// translating the statements one for one (run_program).
#pragma once

#include <string>
#include <vector>

#include "stitch/device.hpp"
#include "stitch/expr.hpp"
#include "stitch/graph.hpp"

namespace stitch {

struct Stmt {
  enum Kind {
    Loop, EndLoop, ISet, FConst, FMove, FOp, GLoad, GStore, SLoad, SStore,
    RegSet, RegRead, Shuffle, WarpReduce, Accum, Barrier, Comment,
  };
  Kind kind;
  std::string dst;
  ExprP dst_slot;
  std::vector<std::string> srcs;
  ExprP src_slot;
  std::string op;
  ExprP idx;
  BExprP guard;
  std::string tensor;
  double cval = 0.0;
  std::string loop_var;
  std::string text;
};

struct TensorBinding {
  std::string name;
  TensorShape shape;
};

struct StitchedProgram {
  LaunchDims launch;
  int64_t shmem_bytes = 0;
  std::vector<TensorBinding> inputs;
  std::vector<TensorBinding> outputs;
  std::vector<Stmt> stmts;
};

std::string emit_program_text(const StitchedProgram& p);
StitchedProgram parse_program_text(const std::string& text);

}  // namespace stitch
