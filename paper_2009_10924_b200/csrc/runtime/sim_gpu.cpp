// stitch::eval_plan / run_program / eval_reference on the B200, plus the
// host-side tensor utilities of sim.hpp (random_inputs, compare, STT1 I/O)
// with the reference's semantics (/root/reference/proj/src/sim.cpp:13-75,
// 516-659).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>

#include "runtime/executor.hpp"
#include "stitch/explorer.hpp"
#include "stitch/sim.hpp"

namespace stitch {

namespace {

int device_from_env() {
  const char* d = std::getenv("STITCH_DEVICE");
  return d && *d ? std::atoi(d) : 0;
}

// f32 -> f16 bits, round-nearest-even (the reference's conversion, sim.cpp:14-37)
uint16_t half_bits(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = x & 0x80000000u;
  const int32_t e = static_cast<int32_t>((x >> 23) & 0xff) - 127;
  const uint32_t m = x & 0x7fffffu;
  if (e > 15) return static_cast<uint16_t>((sign >> 16) | 0x7c00);
  if (e < -24) return static_cast<uint16_t>(sign >> 16);
  if (e < -14) {
    const int sh = -14 - e;
    uint32_t q = (m | 0x800000u) >> (13 + sh);
    const uint32_t rest = (m | 0x800000u) & ((1u << (13 + sh)) - 1);
    if (rest > (1u << (12 + sh)) || (rest == (1u << (12 + sh)) && (q & 1))) ++q;
    return static_cast<uint16_t>((sign >> 16) | q);
  }
  uint32_t q = m >> 13;
  const uint32_t rest = m & 0x1fffu;
  if (rest > 0x1000u || (rest == 0x1000u && (q & 1))) ++q;
  return static_cast<uint16_t>((sign >> 16) | ((static_cast<uint32_t>(e + 15) << 10) + q));
}

// f16 bits -> f32 (exact widening)
float half_value(uint16_t h) {
  const uint32_t hs = (h & 0x8000u) << 16, he = (h >> 10) & 0x1f, hm = h & 0x3ffu;
  uint32_t out;
  if (he == 0x1f) {
    out = hs | 0x7f800000u | (hm << 13);
  } else if (he == 0) {
    if (!hm) {
      out = hs;
    } else {
      int k = -1;
      uint32_t mm = hm;
      while (!(mm & 0x400u)) {
        mm <<= 1;
        ++k;
      }
      out = hs | (static_cast<uint32_t>(127 - 15 - k) << 23) | ((mm & 0x3ffu) << 13);
    }
  } else {
    out = hs | ((he + 127 - 15) << 23) | (hm << 13);
  }
  float f;
  std::memcpy(&f, &out, 4);
  return f;
}

float via_half(float f) { return half_value(half_bits(f)); }

// TensorValue (f64) <-> device-layout bytes
std::vector<uint8_t> pack(const TensorValue& t) {
  const size_t n = t.data.size();
  std::vector<uint8_t> b(n * static_cast<size_t>(dtype_bytes(t.shape.dtype)));
  for (size_t i = 0; i < n; ++i) {
    const double v = t.data[i];
    switch (t.shape.dtype) {
      case DType::F32: {
        const float f = static_cast<float>(v);
        std::memcpy(&b[i * 4], &f, 4);
        break;
      }
      case DType::F16: {
        const uint16_t h = half_bits(static_cast<float>(v));
        std::memcpy(&b[i * 2], &h, 2);
        break;
      }
      case DType::I32: {
        const int32_t x = static_cast<int32_t>(v);
        std::memcpy(&b[i * 4], &x, 4);
        break;
      }
      case DType::Bool: b[i] = v != 0.0; break;
    }
  }
  return b;
}

TensorValue unpack(const TensorShape& s, const std::vector<uint8_t>& b) {
  TensorValue t = TensorValue::zeros(s);
  for (size_t i = 0; i < t.data.size(); ++i) {
    switch (s.dtype) {
      case DType::F32: {
        float f;
        std::memcpy(&f, &b[i * 4], 4);
        t.data[i] = f;
        break;
      }
      case DType::F16: {
        uint16_t h;
        std::memcpy(&h, &b[i * 2], 2);
        t.data[i] = half_value(h);
        break;
      }
      case DType::I32: {
        int32_t x;
        std::memcpy(&x, &b[i * 4], 4);
        t.data[i] = x;
        break;
      }
      case DType::Bool: t.data[i] = b[i] ? 1.0 : 0.0; break;
    }
  }
  return t;
}

TensorMap run_on_gpu(const CompGraph& g, const FusionPlan& plan,
                     const std::map<std::string, KernelPlan>& kernels, const TensorMap& inputs,
                     gpu::ExecMode mode) {
  gpu::Executor ex(g, plan, kernels, machine_model_from_env(), device_from_env(), mode);
  std::vector<std::vector<uint8_t>> in_bytes;
  std::vector<const void*> in_ptrs;
  for (int p : ex.param_vertices()) {
    const OpNode& n = g.node(p);
    auto it = inputs.find(n.name);
    if (it == inputs.end()) throw SimFault("missing input: " + n.name);
    if (it->second.shape.dims != n.shape.dims) throw SimFault("input shape mismatch: " + n.name);
    TensorValue tv = it->second;
    tv.shape.dtype = n.shape.dtype;
    in_bytes.push_back(pack(tv));
    in_ptrs.push_back(in_bytes.back().data());
  }
  std::vector<std::vector<uint8_t>> out_bytes;
  std::vector<void*> out_ptrs;
  for (int o : g.outputs) {
    out_bytes.emplace_back(static_cast<size_t>(g.node(o).shape.byte_size()));
    out_ptrs.push_back(out_bytes.back().data());
  }
  ex.run_host(in_ptrs.data(), out_ptrs.data());
  TensorMap out;
  for (size_t i = 0; i < g.outputs.size(); ++i)
    out[g.node(g.outputs[i]).name] = unpack(g.node(g.outputs[i]).shape, out_bytes[i]);
  return out;
}

}  // namespace

double round_to_dtype(double v, DType d) {
  switch (d) {
    case DType::F32: return static_cast<double>(static_cast<float>(v));
    case DType::F16: return static_cast<double>(via_half(static_cast<float>(v)));
    case DType::I32: return static_cast<double>(static_cast<int32_t>(std::llround(v)));
    case DType::Bool: return v != 0.0 ? 1.0 : 0.0;
  }
  return v;
}

TensorValue TensorValue::zeros(const TensorShape& s) {
  TensorValue t;
  t.shape = s;
  t.data.assign(static_cast<size_t>(s.element_count()), 0.0);
  return t;
}

// one op as a one-kernel graph: operands become parameters (sim.cpp:111-229 semantics)
TensorValue eval_node(const OpNode& n, const std::vector<const TensorValue*>& operands) {
  CompGraph g;
  TensorMap inputs;
  std::vector<int> ids;
  for (size_t i = 0; i < operands.size(); ++i) {
    OpNode p;
    p.id = g.num_nodes();
    p.name = "in" + std::to_string(i);
    p.kind = OpKind::Parameter;
    p.shape = operands[i]->shape;
    g.by_name[p.name] = p.id;
    g.nodes.push_back(p);
    inputs[p.name] = *operands[i];
    ids.push_back(p.id);
  }
  OpNode op = n;
  op.id = g.num_nodes();
  op.name = "out";
  op.operands = ids;
  g.by_name[op.name] = op.id;
  g.nodes.push_back(op);
  g.outputs = {op.id};
  return run_on_gpu(g, FusionPlan{}, {}, inputs, gpu::ExecMode::Unfused).at("out");
}

TensorMap eval_plan(const CompGraph& g, const FusionPlan& plan,
                    const std::map<std::string, KernelPlan>& kernel_plans, const TensorMap& inputs) {
  return run_on_gpu(g, plan, kernel_plans, inputs, gpu::ExecMode::Stitched);
}

TensorMap eval_reference(const CompGraph& g, const TensorMap& inputs) {
  return run_on_gpu(g, FusionPlan{}, {}, inputs, gpu::ExecMode::Unfused);
}

void run_program(const StitchedProgram& prog, TensorMap& tensors) {
  // a one-kernel graph whose parameters are the program's bindings
  CompGraph g;
  auto add = [&](const TensorBinding& b) {
    if (g.by_name.count(b.name)) return;
    OpNode n;
    n.id = g.num_nodes();
    n.name = b.name;
    n.kind = OpKind::Parameter;
    n.shape = b.shape;
    g.by_name[b.name] = n.id;
    g.nodes.push_back(n);
  };
  for (const auto& b : prog.inputs) add(b);
  for (const auto& b : prog.outputs) add(b);
  const auto& dev = gpu::device_init(device_from_env());
  (void)dev;
  auto spec = gpu::generate_program_kernel(g, prog, "stitched_program", /*checked=*/true);
  gpu::Module mod(gpu::compile_cubin(gpu::device_prelude() + spec.source, gpu::default_nvrtc_options()));
  const void* f = reinterpret_cast<const void*>(mod.fn(spec.name));
  if (spec.smem > 48 * 1024)
    STC_RT(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(spec.smem)));
  std::vector<void*> bufs;
  for (const auto& b : prog.inputs) {
    auto it = tensors.find(b.name);
    if (it == tensors.end()) throw SimFault("unbound tensor: " + b.name);
    if (it->second.shape.dims != b.shape.dims) throw SimFault("kernel input shape mismatch: " + b.name);
    TensorValue tv = it->second;
    tv.shape.dtype = b.shape.dtype;
    auto bytes = pack(tv);
    void* p = nullptr;
    STC_RT(cudaMalloc(&p, std::max<size_t>(bytes.size(), 16)));
    STC_RT(cudaMemcpy(p, bytes.data(), bytes.size(), cudaMemcpyHostToDevice));
    bufs.push_back(p);
  }
  for (const auto& b : prog.outputs) {
    TensorValue tv = tensors.count(b.name) ? tensors[b.name] : TensorValue::zeros(b.shape);
    tv.shape.dtype = b.shape.dtype;
    auto bytes = pack(tv);
    void* p = nullptr;
    STC_RT(cudaMalloc(&p, std::max<size_t>(bytes.size(), 16)));
    STC_RT(cudaMemcpy(p, bytes.data(), bytes.size(), cudaMemcpyHostToDevice));
    bufs.push_back(p);
  }
  void* fault = nullptr;
  STC_RT(cudaMalloc(&fault, 256));
  STC_RT(cudaMemset(fault, 0, 256));
  std::vector<void*> args;
  for (auto& p : bufs) args.push_back(&p);
  args.push_back(&fault);
  STC_RT(cudaLaunchKernel(f, dim3(static_cast<unsigned>(spec.grid)), dim3(static_cast<unsigned>(spec.block)),
                          args.data(), static_cast<size_t>(spec.smem), nullptr));
  STC_RT(cudaDeviceSynchronize());
  unsigned fw[4] = {0, 0, 0, 0};
  STC_RT(cudaMemcpy(fw, fault, sizeof fw, cudaMemcpyDeviceToHost));
  cudaFree(fault);
  if (fw[0]) {
    for (void* p : bufs) cudaFree(p);
    const std::string where = " (thread " + std::to_string(fw[2]) + ", block " + std::to_string(fw[3]) + ")";
    if (fw[0] == 1) throw SimFault("shared read of un-barriered write at offset " + std::to_string(fw[1]) + where);
    if (fw[0] == 2) throw SimFault("global access out of bounds at element " + std::to_string(fw[1]) + where);
    throw SimFault("shared access out of bounds at offset " + std::to_string(fw[1]) + where);
  }
  for (size_t i = 0; i < prog.outputs.size(); ++i) {
    const auto& b = prog.outputs[i];
    std::vector<uint8_t> bytes(static_cast<size_t>(b.shape.byte_size()));
    STC_RT(cudaMemcpy(bytes.data(), bufs[prog.inputs.size() + i], bytes.size(), cudaMemcpyDeviceToHost));
    tensors[b.name] = unpack(b.shape, bytes);
  }
  for (void* p : bufs) cudaFree(p);
}

// pass iff abs <= abs_tol OR rel <= rel_tol; integral dtypes exact (sim.cpp:516-547)
CompareReport compare(const TensorMap& got, const TensorMap& want, double rel_tol, double abs_tol) {
  CompareReport r;
  for (const auto& [name, w] : want) {
    auto it = got.find(name);
    if (it == got.end()) {
      r.pass = false;
      r.message = "missing output: " + name;
      return r;
    }
    if (it->second.shape.dims != w.shape.dims) {
      r.pass = false;
      r.message = "shape mismatch on " + name;
      return r;
    }
    const bool integral = w.shape.dtype == DType::I32 || w.shape.dtype == DType::Bool;
    for (size_t i = 0; i < w.data.size(); ++i) {
      const double a = it->second.data[i], b = w.data[i];
      const double ad = std::abs(a - b);
      const double rd = ad / std::max({std::abs(a), std::abs(b), 1e-30});
      r.max_abs = std::max(r.max_abs, ad);
      if (ad > 0) r.max_rel = std::max(r.max_rel, rd);
      const bool ok = integral ? a == b : (ad <= abs_tol || rd <= rel_tol);
      if (!ok && r.pass) {
        r.pass = false;
        r.message = "mismatch on " + name + "[" + std::to_string(i) + "]: got " + std::to_string(a) +
                    ", want " + std::to_string(b);
      }
    }
  }
  return r;
}

// STT1: magic, u8 dtype, u8 rank, u64 dims, row-major payload (f16 widened to f32)
void write_tensor(const std::string& path, const TensorValue& t) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw SimFault("cannot write " + path);
  f.write("STT1", 4);
  f.put(static_cast<char>(static_cast<uint8_t>(t.shape.dtype)));
  f.put(static_cast<char>(static_cast<uint8_t>(t.shape.rank())));
  for (int64_t d : t.shape.dims) {
    const uint64_t u = static_cast<uint64_t>(d);
    f.write(reinterpret_cast<const char*>(&u), 8);
  }
  for (double v : t.data) {
    if (t.shape.dtype == DType::Bool) {
      const uint8_t x = v != 0.0;
      f.write(reinterpret_cast<const char*>(&x), 1);
    } else if (t.shape.dtype == DType::I32) {
      const int32_t x = static_cast<int32_t>(v);
      f.write(reinterpret_cast<const char*>(&x), 4);
    } else {
      const float x = static_cast<float>(v);
      f.write(reinterpret_cast<const char*>(&x), 4);
    }
  }
}

TensorValue read_tensor(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  char magic[4];
  if (!f.read(magic, 4) || std::string(magic, 4) != "STT1") throw SimFault("bad tensor container: " + path);
  TensorValue t;
  t.shape.dtype = static_cast<DType>(f.get());
  const int rank = f.get();
  for (int i = 0; i < rank; ++i) {
    uint64_t d = 0;
    f.read(reinterpret_cast<char*>(&d), 8);
    t.shape.dims.push_back(static_cast<int64_t>(d));
  }
  t.data.resize(static_cast<size_t>(t.shape.element_count()));
  for (auto& v : t.data) {
    if (t.shape.dtype == DType::Bool) {
      char x = 0;
      f.read(&x, 1);
      v = x ? 1.0 : 0.0;
    } else if (t.shape.dtype == DType::I32) {
      int32_t x = 0;
      f.read(reinterpret_cast<char*>(&x), 4);
      v = x;
    } else {
      float x = 0;
      f.read(reinterpret_cast<char*>(&x), 4);
      v = x;
    }
  }
  if (!f) throw SimFault("truncated tensor container: " + path);
  return t;
}

// splitmix64 from seed + phi; f32/f16 uniform(-1,1) rounded; i32 bounded by
// the smallest gather extent (default 10); bool = low bit (sim.cpp:630-659)
TensorMap random_inputs(const CompGraph& g, uint64_t seed) {
  uint64_t state = seed + 0x9e3779b97f4a7c15ull;
  auto next = [&]() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  TensorMap out;
  for (const auto& n : g.nodes) {
    if (n.kind != OpKind::Parameter) continue;
    TensorValue t = TensorValue::zeros(n.shape);
    if (n.shape.dtype == DType::I32) {
      int64_t bound = 10;
      for (const auto& c : g.nodes)
        if (c.kind == OpKind::Gather && c.operands.size() == 2 && c.operands[1] == n.id)
          bound = std::min(bound, g.node(c.operands[0]).shape.dims[0]);
      for (auto& v : t.data) v = static_cast<double>(next() % static_cast<uint64_t>(bound));
    } else if (n.shape.dtype == DType::Bool) {
      for (auto& v : t.data) v = static_cast<double>(next() & 1);
    } else {
      for (auto& v : t.data)
        v = round_to_dtype(static_cast<double>(next() >> 11) * 0x1p-53 * 2.0 - 1.0, n.shape.dtype);
    }
    out[n.name] = std::move(t);
  }
  return out;
}

}  // namespace stitch
