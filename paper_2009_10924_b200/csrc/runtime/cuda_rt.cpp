// Device init, NVRTC (sm_100a) compilation with a content-addressed cubin
// cache, and module loading.
#include "runtime/cuda_rt.hpp"

#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <thread>
#include <fstream>
#include <mutex>
#include <sstream>
#include <stdexcept>

namespace stitch::gpu {

void throw_cuda(const char* what, const char* detail) {
  throw std::runtime_error(std::string("[cuda] ") + what + ": " + detail);
}

const DeviceInfo& device_init(int ordinal) {
  static std::mutex mu;
  static std::map<int, DeviceInfo> infos;
  std::lock_guard<std::mutex> lock(mu);
  STC_RT(cudaSetDevice(ordinal));
  auto it = infos.find(ordinal);
  if (it != infos.end()) return it->second;
  STC_RT(cudaFree(nullptr));  // creates the primary context and makes it current
  DeviceInfo d;
  d.ordinal = ordinal;
  STC_RT(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, ordinal));
  STC_RT(cudaDeviceGetAttribute(&d.l2_bytes, cudaDevAttrL2CacheSize, ordinal));
  STC_RT(cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ordinal));
  STC_RT(cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, ordinal));
  STC_RT(cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, ordinal));
  if (d.cc_major != 10)
    throw std::runtime_error("[cuda] stitch-b200 kernels are sm_100a only; device reports sm_" +
                             std::to_string(d.cc_major) + std::to_string(d.cc_minor));
  return infos[ordinal] = d;
}

namespace {

uint64_t fnv1a(const std::string& s, uint64_t h) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

std::string lib_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&lib_dir), &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const auto slash = p.rfind('/');
    if (slash != std::string::npos) return p.substr(0, slash);
  }
  return ".";
}

void mkdirs(const std::string& path) {
  std::string cur;
  std::stringstream ss(path);
  for (std::string part; std::getline(ss, part, '/');) {
    cur += part + "/";
    if (!part.empty()) mkdir(cur.c_str(), 0755);
  }
}

#define STC_NVRTC(x)                                                        \
  do {                                                                      \
    nvrtcResult r_ = (x);                                                   \
    if (r_ != NVRTC_SUCCESS)                                                \
      throw std::runtime_error(std::string("[nvrtc] ") + #x + ": " + nvrtcGetErrorString(r_)); \
  } while (0)

}  // namespace

std::string cubin_cache_dir() {
  const char* e = std::getenv("STITCH_CACHE_DIR");
  return (e && *e) ? std::string(e) : lib_dir() + "/cubin_cache";
}

std::vector<std::string> default_nvrtc_options() {
  // -fmad=false: no FMA contraction, so f32 + - * / match the reference's
  // "compute in f64, round to f32" bit for bit; IEEE div/sqrt are NVRTC's
  // defaults (no fast-math).
  std::vector<std::string> o{"-arch=sm_100a", "--std=c++17", "-fmad=false", "-lineinfo", "-default-device"};
  // experiment knobs: STITCH_NVRTC_DEFINES="STITCH_L2_256B STITCH_ST_CS"
  if (const char* d = std::getenv("STITCH_NVRTC_DEFINES")) {
    std::string s(d), w;
    for (size_t i = 0; i <= s.size(); ++i) {
      if (i == s.size() || s[i] == ' ' || s[i] == ',' || s[i] == ':') {
        if (!w.empty()) o.push_back("-D" + w);
        w.clear();
      } else {
        w += s[i];
      }
    }
  }
  return o;
}

std::string compile_cubin(const std::string& source, const std::vector<std::string>& options,
                          std::string* key_out, bool* cache_hit) {
  if (cache_hit) *cache_hit = false;
  int maj = 0, min = 0;
  STC_NVRTC(nvrtcVersion(&maj, &min));
  std::string salt = std::to_string(maj) + "." + std::to_string(min);
  for (const auto& o : options) salt += "\x1f" + o;
  char key[40];
  std::snprintf(key, sizeof key, "%016llx%016llx",
                static_cast<unsigned long long>(fnv1a(source, fnv1a(salt, 0xcbf29ce484222325ull))),
                static_cast<unsigned long long>(fnv1a(salt + source, 0x84222325cbf29ce4ull)));
  if (key_out) *key_out = key;
  const std::string dir = cubin_cache_dir();
  const std::string path = dir + "/" + key + ".cubin";
  {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      std::ostringstream ss;
      ss << in.rdbuf();
      if (!ss.str().empty()) {
        if (cache_hit) *cache_hit = true;
        return ss.str();
      }
    }
  }
  nvrtcProgram prog;
  STC_NVRTC(nvrtcCreateProgram(&prog, source.c_str(), "stitched.cu", 0, nullptr, nullptr));
  std::vector<const char*> opts;
  for (const auto& o : options) opts.push_back(o.c_str());
  const nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data());
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, log.data());
    nvrtcDestroyProgram(&prog);
    throw std::runtime_error("[nvrtc] compile failed: " + log.substr(0, 4000));
  }
  if (const char* v = std::getenv("STITCH_NVRTC_LOG"); v && *v == '1') {
    size_t ln = 0;
    nvrtcGetProgramLogSize(prog, &ln);
    std::string log(ln, '\0');
    nvrtcGetProgramLog(prog, log.data());
    std::fprintf(stderr, "[nvrtc] %s\n", log.c_str());
  }
  size_t n = 0;
  STC_NVRTC(nvrtcGetCUBINSize(prog, &n));
  std::string cubin(n, '\0');
  STC_NVRTC(nvrtcGetCUBIN(prog, cubin.data()));
  nvrtcDestroyProgram(&prog);
  mkdirs(dir);
  // unique per process AND thread (cache warm-up compiles concurrently)
  const std::string tmp = path + ".tmp" + std::to_string(getpid()) + "_" +
                          std::to_string(std::hash<std::thread::id>{}(std::this_thread::get_id()));
  {
    std::ofstream out(tmp, std::ios::binary);
    out.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
  }
  std::rename(tmp.c_str(), path.c_str());
  return cubin;
}

Module::Module(const std::string& cubin) {
  STC_RT(cudaLibraryLoadData(&lib_, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
}

Module::~Module() {
  if (lib_) cudaLibraryUnload(lib_);
}

void* Module::global(const std::string& name, size_t* bytes) {
  void* p = nullptr;
  size_t n = 0;
  if (cudaLibraryGetGlobal(&p, &n, lib_, name.c_str()) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (bytes) *bytes = n;
  return p;
}

cudaKernel_t Module::fn(const std::string& name) {
  auto it = fns_.find(name);
  if (it != fns_.end()) return it->second;
  cudaKernel_t k;
  STC_RT(cudaLibraryGetKernel(&k, lib_, name.c_str()));
  return fns_[name] = k;
}

}  // namespace stitch::gpu
