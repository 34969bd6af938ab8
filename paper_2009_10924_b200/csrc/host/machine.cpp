// Machine model: built-in V100-like defaults, INI loader layered over them,
// and the analytical-latency building blocks (Eq.1 of the paper).
// Formulas follow /root/reference/proj/src/device.cpp:25-72 exactly (parity
// mode); the loader follows src/config.cpp:10-138 (unknown keys rejected, so
// any .cfg we ship also loads in the reference).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>

#include "stitch/device.hpp"

namespace stitch {

double CpiTable::cpi(const std::string& kind) const {
  auto it = cycles.find(kind);
  if (it == cycles.end()) throw std::runtime_error("no CPI configured for instruction kind: " + kind);
  return it->second;
}

const char* transition_name(MemTransition t) {
  switch (t) {
    case MemTransition::GlobalToRegister: return "global_to_register";
    case MemTransition::GlobalToShared: return "global_to_shared";
    case MemTransition::SharedToRegister: return "shared_to_register";
  }
  return "?";
}

// blocks/SM = min(block cap, smem cap, register cap, warp-slot cap);
// occupancy = resident warps / max warps, clamped to [1/max_warps, 1].
std::optional<double> occupancy(const LaunchDims& ld, int regs, int64_t smem,
                                const DeviceSpec& dev) {
  if (smem > dev.shared_mem_per_block_limit) return std::nullopt;
  const int64_t block = ld.block;
  const int64_t r = std::max(regs, 1);
  const int64_t lim_smem = dev.shared_mem_per_sm / std::max<int64_t>(smem, 1);
  const int64_t lim_regs = dev.registers_per_sm / (r * block);
  const int64_t lim_warps = int64_t(dev.max_warps_per_sm) * dev.warp_size / block;
  const int64_t blocks =
      std::min(std::min<int64_t>(dev.max_blocks_per_sm, lim_smem), std::min(lim_regs, lim_warps));
  const int64_t warps = blocks * ((block + dev.warp_size - 1) / dev.warp_size);
  const double occ = static_cast<double>(warps) / dev.max_warps_per_sm;
  return std::clamp(occ, 1.0 / dev.max_warps_per_sm, 1.0);
}

double wave_count(double n_warps, double occ, const DeviceSpec& dev) {
  return n_warps / (occ * dev.sm_count * dev.max_warps_per_sm);
}

double warp_latency(const std::map<std::string, int64_t>& hist, const CpiTable& cpi) {
  double cycles = 0.0;
  for (const auto& [kind, n] : hist) cycles += static_cast<double>(n) * cpi.cpi(kind);
  return cycles;
}

// piecewise-linear through (0,0) and the breakpoints; last slope extrapolated
double mem_transfer_saving(int64_t bytes, MemTransition t, const MemLatencyModel& m) {
  auto it = m.curves.find(t);
  if (it == m.curves.end() || it->second.empty())
    throw std::runtime_error(std::string("unsupported memory transition: ") + transition_name(t));
  const auto& pts = it->second;
  if (bytes <= 0) return 0.0;
  double x0 = 0.0, y0 = 0.0;
  for (const auto& p : pts) {
    if (bytes <= p.bytes)
      return y0 + static_cast<double>(bytes - x0) / (static_cast<double>(p.bytes) - x0) * (p.cycles - y0);
    x0 = static_cast<double>(p.bytes);
    y0 = p.cycles;
  }
  const size_t n = pts.size();
  const double xa = n > 1 ? static_cast<double>(pts[n - 2].bytes) : 0.0;
  const double ya = n > 1 ? pts[n - 2].cycles : 0.0;
  const double slope = (pts[n - 1].cycles - ya) / (static_cast<double>(pts[n - 1].bytes) - xa);
  return pts[n - 1].cycles + slope * (static_cast<double>(bytes) - static_cast<double>(pts[n - 1].bytes));
}

MachineModel default_machine_model() {
  MachineModel m;
  for (const char* k : {"add", "sub", "mul", "div", "max", "min"}) m.cpi.cycles[k] = 4.0;
  for (const char* k : {"exp", "tanh", "log", "rsqrt", "power"}) m.cpi.cycles[k] = 32.0;
  m.cpi.cycles["reduce_step"] = 8.0;
  m.cpi.cycles["shared_access"] = 30.0;
  m.cpi.cycles["shuffle"] = 5.0;
  m.cpi.cycles["index_calc"] = 4.0;
  m.memlat.curves[MemTransition::GlobalToRegister] = {{4096, 2200}, {1 << 20, 560000}};
  m.memlat.curves[MemTransition::GlobalToShared] = {{4096, 2000}, {1 << 20, 500000}};
  m.memlat.curves[MemTransition::SharedToRegister] = {{4096, 250}, {1 << 20, 64000}};
  return m;
}

namespace {

std::string strip(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}

std::vector<MemLatencyModel::Point> curve_of(const std::string& v, const std::string& key) {
  std::vector<MemLatencyModel::Point> pts;
  std::stringstream ss(v);
  for (std::string item; std::getline(ss, item, ',');) {
    item = strip(item);
    if (item.empty()) continue;
    const auto colon = item.find(':');
    if (colon == std::string::npos)
      throw std::runtime_error("bad memlat point '" + item + "' for " + key);
    MemLatencyModel::Point p{std::stoll(item.substr(0, colon)), std::stod(item.substr(colon + 1))};
    if (p.bytes == 0) continue;
    if (!pts.empty() && p.bytes <= pts.back().bytes)
      throw std::runtime_error("memlat breakpoints must be strictly increasing: " + key);
    if (!pts.empty() && p.cycles < pts.back().cycles)
      throw std::runtime_error("memlat curve must be monotone non-decreasing: " + key);
    pts.push_back(p);
  }
  if (pts.empty()) throw std::runtime_error("empty memlat curve: " + key);
  return pts;
}

bool truthy(const std::string& v) { return v == "true" || v == "1"; }

using Setter = std::function<void(MachineModel&, const std::string&)>;

const std::map<std::string, std::map<std::string, Setter>>& key_table() {
  static const std::map<std::string, std::map<std::string, Setter>> t = {
      {"device",
       {{"sm_count", [](MachineModel& m, const std::string& v) { m.dev.sm_count = std::stoi(v); }},
        {"max_warps_per_sm", [](MachineModel& m, const std::string& v) { m.dev.max_warps_per_sm = std::stoi(v); }},
        {"max_threads_per_block", [](MachineModel& m, const std::string& v) { m.dev.max_threads_per_block = std::stoi(v); }},
        {"warp_size", [](MachineModel& m, const std::string& v) { m.dev.warp_size = std::stoi(v); }},
        {"shared_mem_per_sm", [](MachineModel& m, const std::string& v) { m.dev.shared_mem_per_sm = std::stoll(v); }},
        {"shared_mem_per_block_limit", [](MachineModel& m, const std::string& v) { m.dev.shared_mem_per_block_limit = std::stoll(v); }},
        {"registers_per_sm", [](MachineModel& m, const std::string& v) { m.dev.registers_per_sm = std::stoll(v); }},
        {"max_blocks_per_sm", [](MachineModel& m, const std::string& v) { m.dev.max_blocks_per_sm = std::stoi(v); }},
        {"global_mem_bandwidth", [](MachineModel& m, const std::string& v) { m.dev.global_mem_bandwidth = std::stoll(v); }}}},
      {"costs",
       {{"context_switch_cycles", [](MachineModel& m, const std::string& v) { m.costs.context_switch_cycles = std::stod(v); }},
        {"register_overhead", [](MachineModel& m, const std::string& v) { m.costs.register_overhead = std::stoi(v); }},
        {"delta_fixed_registers", [](MachineModel& m, const std::string& v) { m.costs.delta_fixed_registers = std::stoi(v); }},
        {"opaque_kernel_cycles", [](MachineModel& m, const std::string& v) { m.costs.opaque_kernel_cycles = std::stod(v); }},
        {"ceil_waves", [](MachineModel& m, const std::string& v) { m.costs.ceil_waves = truthy(v); }}}},
      {"search",
       {{"k", [](MachineModel& m, const std::string& v) { m.search.k = std::stoi(v); }},
        {"beam_width", [](MachineModel& m, const std::string& v) { m.search.beam_width = std::stoi(v); }},
        {"max_pattern_size", [](MachineModel& m, const std::string& v) { m.search.max_pattern_size = std::stoi(v); }},
        {"grouping_cap", [](MachineModel& m, const std::string& v) { m.search.grouping_cap = std::stoi(v); }},
        {"candidate_cap", [](MachineModel& m, const std::string& v) { m.search.candidate_cap = std::stoi(v); }},
        {"reverse_beam_order", [](MachineModel& m, const std::string& v) { m.search.reverse_beam_order = truthy(v); }}}},
  };
  return t;
}

}  // namespace

MachineModel load_machine_model(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open device config: " + path);
  MachineModel m = default_machine_model();
  std::string section;
  int lineno = 0;
  for (std::string raw; std::getline(in, raw);) {
    ++lineno;
    std::string line = strip(raw.substr(0, raw.find('#')));
    if (line.empty()) continue;
    if (line.front() == '[' && line.back() == ']') {
      section = strip(line.substr(1, line.size() - 2));
      continue;
    }
    const auto eq = line.find('=');
    if (eq == std::string::npos)
      throw std::runtime_error(path + ":" + std::to_string(lineno) + ": expected key = value");
    const std::string key = strip(line.substr(0, eq)), val = strip(line.substr(eq + 1));
    try {
      if (section == "cpi") {
        const double v = std::stod(val);
        if (v <= 0) throw std::runtime_error("CPI must be > 0: " + key);
        m.cpi.cycles[key] = v;
      } else if (section == "memlat") {
        static const std::map<std::string, MemTransition> names = {
            {"global_to_register", MemTransition::GlobalToRegister},
            {"global_to_shared", MemTransition::GlobalToShared},
            {"shared_to_register", MemTransition::SharedToRegister}};
        auto it = names.find(key);
        if (it == names.end()) throw std::runtime_error("unknown memlat key: " + key);
        m.memlat.curves[it->second] = curve_of(val, key);
      } else {
        auto sec = key_table().find(section);
        if (sec == key_table().end()) throw std::runtime_error("unknown section: [" + section + "]");
        auto k = sec->second.find(key);
        if (k == sec->second.end()) throw std::runtime_error("unknown " + section + " key: " + key);
        k->second(m, val);
      }
    } catch (const std::invalid_argument&) {
      throw std::runtime_error(path + ":" + std::to_string(lineno) + ": bad value for " + key);
    }
  }
  return m;
}

MachineModel machine_model_from_env() {
  const char* p = std::getenv("STITCH_DEVICE_CONFIG");
  return (p && *p) ? load_machine_model(p) : default_machine_model();
}

}  // namespace stitch
