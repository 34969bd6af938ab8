"""Recalibrate the planner's latency cost model from B200 measurements
(north star: "the latency cost model and
resource-constraint checks, recalibrated from B200 measurements").

    python tools/calibrate_b200.py [--out paper_2009_10924_b200/configs/b200.cfg]
                                   [--json profiles/r01/calibration_b200.json]

Every value of the reference's cost model (configs/default.cfg, V100) is
re-measured on the B200 in SM cycles at clocks.max.sm (1965 MHz):

[cpi]     one warp, a dependent chain of the op exactly as our code generator
          emits it (-fmad=false, IEEE div/sqrt, accurate expf/tanhf/logf/powf;
          rsqrt = 1/sqrtf), cycles per op (the reference's CPI is the op
          latency a stitched thread pays: src/device.cpp:53-58).
          reduce_step = f64 add (the interpreter's Accum), shuffle =
          shfl from lane 0, shared_access = dependent shared-memory load,
          index_calc = dependent integer multiply-add.
[memlat]  global_to_register(b): cycles a kernel boundary costs for an
          intermediate of b bytes = one write + one read of b bytes, i.e. a
          b-byte copy kernel in a CUDA graph minus an empty node
          (src/device.cpp:60-72 interpolates these points).
          global_to_shared: the same copy staged through shared memory.
          shared_to_register(b): b bytes spread over all 148 SMs read from
          shared memory, minus an empty node.
[costs]   context_switch_cycles: per-kernel cost of a chain of dependent tiny
          kernels replayed from one CUDA graph with programmatic dependent
          launch (how the executor runs plans).  opaque_kernel_cycles: the
          opaque placeholder for a [256,36] operand in the same setting.
          register_overhead / delta_fixed_registers: kept (the planner's
          register estimate is for its abstract program, not our templates;
          the measured template registers are recorded beside it).
[device]  B200 resource limits (cudaGetDeviceProperties), as b200_device.cfg.

The file keeps the reference loader's keys only, so the UNMODIFIED reference
planner (oracle/_ref) reads it too and plan parity stays checkable under the
calibrated model.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from cuda.bindings import driver as cu  # noqa: E402
from cuda.bindings import nvrtc  # noqa: E402

SRC = r'''
#define BAR_F(x) asm volatile("" : "+f"(x))
#define BAR_D(x) asm volatile("" : "+d"(x))
#define BAR_I(x) asm volatile("" : "+r"(x))
#define CHAIN(NAME, T, BAR, STEP)                                                   \
extern "C" __global__ void lat_##NAME(const T* in, T* out, long long* cyc, int n) {  \
  T x = in[threadIdx.x]; const T y = in[32 + threadIdx.x];                          \
  (void)y;                                                                          \
  __syncwarp();                                                                     \
  const long long t0 = clock64();                                                   \
  for (int i = 0; i < n; ++i) {                                                     \
    _Pragma("unroll") for (int u = 0; u < 16; ++u) { STEP; BAR(x); }                \
  }                                                                                 \
  const long long t1 = clock64();                                                   \
  out[threadIdx.x] = x;                                                             \
  if (threadIdx.x == 0) cyc[0] = t1 - t0;                                           \
}
CHAIN(add, float, BAR_F, x = x + y)
CHAIN(sub, float, BAR_F, x = x - y)
CHAIN(mul, float, BAR_F, x = x * y)
CHAIN(div, float, BAR_F, x = x / y)
CHAIN(max, float, BAR_F, x = x < y ? y : x)
CHAIN(min, float, BAR_F, x = y < x ? y : x)
CHAIN(exp, float, BAR_F, x = expf(x))
CHAIN(tanh, float, BAR_F, x = tanhf(x))
CHAIN(log, float, BAR_F, x = logf(x))
CHAIN(rsqrt, float, BAR_F, x = 1.0f / sqrtf(x))
CHAIN(power, float, BAR_F, x = powf(x, y))
CHAIN(reduce_step, double, BAR_D, x = x + y)
CHAIN(shuffle, float, BAR_F, asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 0x1f, 0xffffffff;" : "+f"(x)))
CHAIN(index_calc, int, BAR_I, x = x * y + 3)

extern "C" __global__ void lat_shared_access(const int* in, int* out, long long* cyc, int n) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i * 97 + 31) & 1023;
  __syncwarp();
  int x = in[threadIdx.x] & 1023;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = s[x];
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

extern "C" __global__ void empty_k() {}

// b-byte copy, float4, grid-stride (a kernel boundary's write + read)
extern "C" __global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, long long n4) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    b[i] = __ldg(a + i);
  asm volatile("griddepcontrol.launch_dependents;");
}

// the same copy staged through shared memory
extern "C" __global__ void copy_smem_k(const float4* __restrict__ a, float4* __restrict__ b, long long n4) {
  __shared__ float4 t[256];
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < n4; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    if (i < n4) t[threadIdx.x] = __ldg(a + i);
    __syncthreads();
    if (i < n4) b[i] = t[threadIdx.x ^ 1];
    __syncthreads();
  }
}

// every CTA reads `per` bytes of its own shared memory (float4, 256 threads)
extern "C" __global__ void smem_read_k(float* out, int per4) {
  extern __shared__ float4 sm[];
  const int n = per4 < 12288 ? per4 : 12288;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < per4; i += blockDim.x) {
    const float4 v = sm[i % n];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x == -1.f) out[blockIdx.x] = acc.y + acc.z + acc.w;
}
'''

MHZ = 1965.0  # clocks.max.sm (B200_PROFILING.md); clock64() counts SM cycles


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(str(err))
    if isinstance(r, tuple):
        return r[1] if len(r) == 2 else r[1:]
    return None


class Dev:
    def __init__(self):
        ck(cu.cuInit(0))
        self.dev = ck(cu.cuDeviceGet(0))
        ctx = ck(cu.cuDevicePrimaryCtxRetain(self.dev))
        ck(cu.cuCtxSetCurrent(ctx))
        prog = ck(nvrtc.nvrtcCreateProgram(SRC.encode(), b"calib.cu", 0, [], []))
        opts = [b"-arch=sm_100a", b"--std=c++17", b"-fmad=false", b"-default-device"]
        r = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
        if int(r[0]) != 0:
            n = ck(nvrtc.nvrtcGetProgramLogSize(prog))
            log = b" " * n
            nvrtc.nvrtcGetProgramLog(prog, log)
            raise RuntimeError(log.decode())
        n = ck(nvrtc.nvrtcGetCUBINSize(prog))
        cubin = b" " * n
        ck(nvrtc.nvrtcGetCUBIN(prog, cubin))
        self.mod = ck(cu.cuModuleLoadData(cubin))
        self.stream = ck(cu.cuStreamCreate(1))
        self.e0, self.e1 = ck(cu.cuEventCreate(0)), ck(cu.cuEventCreate(0))
        self.keep = []

    def fn(self, name):
        return ck(cu.cuModuleGetFunction(self.mod, name.encode()))

    def attr(self, a):
        return ck(cu.cuDeviceGetAttribute(a, self.dev))

    def launch(self, f, grid, block, args, smem=0, pdl=False):
        vals = [ctypes.c_void_p(int(a)) if isinstance(a, cu.CUdeviceptr) else a for a in args]
        ptrs = (ctypes.c_void_p * max(1, len(vals)))(*[ctypes.addressof(v) for v in vals])
        self.keep.append((vals, ptrs))
        cfg = cu.CUlaunchConfig()
        cfg.gridDimX, cfg.gridDimY, cfg.gridDimZ = grid, 1, 1
        cfg.blockDimX, cfg.blockDimY, cfg.blockDimZ = block, 1, 1
        cfg.sharedMemBytes = smem
        cfg.hStream = self.stream
        if pdl:
            at = cu.CUlaunchAttribute()
            at.id = cu.CUlaunchAttributeID.CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION
            at.value.programmaticStreamSerializationAllowed = 1
            cfg.attrs = [at]
            cfg.numAttrs = 1
        else:
            cfg.numAttrs = 0
        ck(cu.cuLaunchKernelEx(cfg, f, ctypes.addressof(ptrs) if args else 0, 0))

    def graph(self, n, make):
        ck(cu.cuStreamBeginCapture(self.stream, cu.CUstreamCaptureMode.CU_STREAM_CAPTURE_MODE_THREAD_LOCAL))
        for i in range(n):
            make(i)
        g = ck(cu.cuStreamEndCapture(self.stream))
        return ck(cu.cuGraphInstantiate(g, 0))

    def graph_us(self, gexec, n, reps=20):
        ck(cu.cuGraphLaunch(gexec, self.stream))
        ck(cu.cuStreamSynchronize(self.stream))
        ck(cu.cuEventRecord(self.e0, self.stream))
        for _ in range(reps):
            ck(cu.cuGraphLaunch(gexec, self.stream))
        ck(cu.cuEventRecord(self.e1, self.stream))
        ck(cu.cuEventSynchronize(self.e1))
        return ck(cu.cuEventElapsedTime(self.e0, self.e1)) * 1000.0 / (reps * n)


def measure(d):
    res = {"mhz": MHZ, "cpi": {}, "memlat": {}, "costs": {}, "raw": {}}
    buf = ck(cu.cuMemAlloc(1 << 20))
    out = ck(cu.cuMemAlloc(1 << 20))
    cyc = ck(cu.cuMemAlloc(64))
    init = (ctypes.c_float * 64)(*([1.0001] * 64))
    ck(cu.cuMemcpyHtoD(buf, init, 256))
    n_iter = 512
    ops = ["add", "sub", "mul", "div", "max", "min", "exp", "tanh", "log", "rsqrt", "power", "reduce_step",
           "shuffle", "index_calc", "shared_access"]
    for op in ops:
        f = d.fn("lat_" + op)
        if op == "reduce_step":
            ck(cu.cuMemcpyHtoD(buf, (ctypes.c_double * 64)(*([1.0001] * 64)), 512))
        elif op in ("index_calc", "shared_access"):
            ck(cu.cuMemcpyHtoD(buf, (ctypes.c_int * 64)(*([3] * 64)), 256))
        else:
            ck(cu.cuMemcpyHtoD(buf, init, 256))
        samples = []
        for _ in range(5):
            d.launch(f, 1, 32, [buf, out, cyc, ctypes.c_int(n_iter)])
            ck(cu.cuStreamSynchronize(d.stream))
            c = (ctypes.c_longlong * 1)()
            ck(cu.cuMemcpyDtoH(c, cyc, 8))
            samples.append(c[0] / (n_iter * 16.0))
        res["cpi"][op] = round(min(samples), 2)

    empty = d.fn("empty_k")
    ge = d.graph(100, lambda i: d.launch(empty, 148, 256, []))
    empty_us = d.graph_us(ge, 100)
    res["raw"]["graph_empty_node_us"] = empty_us

    copy, copy_s, smem = d.fn("copy_k"), d.fn("copy_smem_k"), d.fn("smem_read_k")
    sizes = [4096, 65536, 1 << 20, 16 << 20, 64 << 20, 256 << 20]
    g2r, g2s = [], []
    for b in sizes:
        n = max(4, min(64, (1 << 30) // (2 * b)))
        bufs = [(ck(cu.cuMemAlloc(b)), ck(cu.cuMemAlloc(b))) for _ in range(n)]
        n4 = b // 16
        grid = int(min(148 * 8, max(1, (n4 + 255) // 256)))
        row = {"bytes": b}
        for key, f in (("g2r", copy), ("g2s", copy_s)):
            ge = d.graph(n, lambda i: d.launch(f, grid, 256, [bufs[i][0], bufs[i][1], ctypes.c_longlong(n4)]))
            us = d.graph_us(ge, n)
            row[key + "_us"] = us
            (g2r if key == "g2r" else g2s).append((b, max(1.0, (us - empty_us) * MHZ)))
        res["raw"].setdefault("copy", []).append(row)
        for a, c in bufs:
            cu.cuMemFree(a)
            cu.cuMemFree(c)
    res["memlat"]["global_to_register"] = [(b, round(c, 1)) for b, c in g2r]
    res["memlat"]["global_to_shared"] = [(b, round(c, 1)) for b, c in g2s]
    big = res["raw"]["copy"][-1]
    res["raw"]["hbm_copy_GBps"] = 2 * big["bytes"] / big["g2r_us"] / 1e3

    ck(cu.cuFuncSetAttribute(smem, cu.CUfunction_attribute.CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                             12288 * 16))
    s2r = []
    for b in (4096, 1 << 20, 16 << 20, 64 << 20):
        per4 = max(1, b // 148 // 16)
        ge = d.graph(20, lambda i: d.launch(smem, 148, 256, [out, ctypes.c_int(per4)], smem=min(per4, 12288) * 16))
        us = d.graph_us(ge, 20)
        s2r.append((b, round(max(1.0, (us - empty_us) * MHZ), 1)))
        res["raw"].setdefault("smem_read_us", []).append({"bytes": b, "us": us})
    res["memlat"]["shared_to_register"] = s2r

    # context switch: chain of dependent 4 KB copies (b_i = copy(b_{i-1})), PDL
    chain = [ck(cu.cuMemAlloc(4096)) for _ in range(65)]
    for pdl in (True, False):
        ge = d.graph(64, lambda i: d.launch(copy, 1, 256, [chain[i], chain[i + 1], ctypes.c_longlong(256)], pdl=pdl))
        res["raw"]["dependent_4KB_node_us_pdl" if pdl else "dependent_4KB_node_us"] = d.graph_us(ge, 64)
    res["costs"]["context_switch_cycles"] = round(res["raw"]["dependent_4KB_node_us_pdl"] * MHZ, 1)
    return res


def opaque_cycles():
    from paper_2009_10924_b200 import stitch
    g = stitch.Graph("x = parameter : f32[256,36]\ny = opaque_compute(x) : f32[256,36]\noutput y\n")
    ex = stitch.Executor(stitch.Plan(g, "b200"))
    ex.upload(stitch.random_inputs(g, 1))
    us = ex.time_batched(steps=256, warmup=32, sets=16, steps_per_graph=16)
    return us


def write_cfg(res, path, device):
    c = res["cpi"]

    def mono(pts):  # the loader requires non-decreasing cycles
        out, hi = [], 0.0
        for b, v in pts:
            hi = max(hi, v)
            out.append((b, hi))
        return out

    curve = lambda pts: ", ".join("%d:%s" % (b, ("%.1f" % v).rstrip("0").rstrip(".")) for b, v in pts)
    lines = [
        "# B200 (sm_100a) cost model, RECALIBRATED from measurements on a B200",
        "# (tools/calibrate_b200.py; raw numbers in profiles/r01/calibration_b200.json).",
        "# Cycles are SM cycles at %.0f MHz.  Only keys the reference loader accepts," % MHZ,
        "# so the unmodified reference planner reads this file too (plan parity).",
        "[device]",
    ]
    for k, v in device.items():
        lines.append("%s = %s" % (k, v))
    lines += ["", "# dependent-chain latency of each op as emitted by the code generator (1 warp)", "[cpi]"]
    for k in ["add", "sub", "mul", "div", "max", "min", "exp", "tanh", "log", "rsqrt", "power", "reduce_step",
              "shared_access", "shuffle", "index_calc"]:
        lines.append("%s = %s" % (k, ("%.2f" % c[k]).rstrip("0").rstrip(".")))
    lines += ["", "# kernel-boundary cost of an intermediate: write + read of b bytes (graph node, minus launch floor)",
              "[memlat]",
              "global_to_register = " + curve(mono(res["memlat"]["global_to_register"])),
              "global_to_shared = " + curve(mono(res["memlat"]["global_to_shared"])),
              "shared_to_register = " + curve(mono(res["memlat"]["shared_to_register"])),
              "", "[costs]",
              "# per-kernel cost of a dependent launch inside one CUDA graph with PDL",
              "context_switch_cycles = %s" % res["costs"]["context_switch_cycles"],
              "register_overhead = 8",
              "delta_fixed_registers = 16",
              "# opaque placeholder kernel ([256,36] operand) in the same setting",
              "opaque_kernel_cycles = %s" % res["costs"]["opaque_kernel_cycles"],
              "ceil_waves = false",
              "", "[search]", "k = 3", "beam_width = 3", "max_pattern_size = 128", "grouping_cap = 64",
              "candidate_cap = 20000", ""]
    with open(path, "w") as f:
        f.write("\n".join(lines))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2009_10924_b200", "configs", "b200.cfg"))
    ap.add_argument("--json", default=os.path.join(ROOT, "profiles", "r01", "calibration_b200.json"))
    a = ap.parse_args()
    d = Dev()
    A = cu.CUdevice_attribute
    device = {
        "sm_count": d.attr(A.CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT),
        "max_warps_per_sm": d.attr(A.CU_DEVICE_ATTRIBUTE_MAX_THREADS_PER_MULTIPROCESSOR) // 32,
        "max_threads_per_block": d.attr(A.CU_DEVICE_ATTRIBUTE_MAX_THREADS_PER_BLOCK),
        "warp_size": d.attr(A.CU_DEVICE_ATTRIBUTE_WARP_SIZE),
        "shared_mem_per_sm": d.attr(A.CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_MULTIPROCESSOR),
        "shared_mem_per_block_limit": d.attr(A.CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN),
        "registers_per_sm": d.attr(A.CU_DEVICE_ATTRIBUTE_MAX_REGISTERS_PER_MULTIPROCESSOR),
        "max_blocks_per_sm": d.attr(A.CU_DEVICE_ATTRIBUTE_MAX_BLOCKS_PER_MULTIPROCESSOR),
    }
    res = measure(d)
    device["global_mem_bandwidth"] = int(round(res["raw"]["hbm_copy_GBps"]))
    us = opaque_cycles()
    res["raw"]["opaque_256x36_us"] = us
    res["costs"]["opaque_kernel_cycles"] = round(us * MHZ, 1)
    res["device"] = device
    os.makedirs(os.path.dirname(a.json), exist_ok=True)
    with open(a.json, "w") as f:
        json.dump(res, f, indent=1)
    write_cfg(res, a.out, device)
    print(json.dumps(res))
    print(open(a.out).read())


if __name__ == "__main__":
    main()
