"""B200 calibration microbenchmarks (diagnostics, not the product): fixed
kernel overhead and one-shot copy bandwidth at the sizes our subgraphs move,
so a stitched kernel's time can be compared with the floor for its bytes.

    python tools/calib.py            # prints one JSON line per probe
"""
import ctypes
import json

import numpy as np
from cuda.bindings import driver as cu
from cuda.bindings import nvrtc

SRC = r'''
extern "C" __global__ void empty_k() {}
// one-shot: every thread moves `per` float4 (like a row-resident regional kernel)
extern "C" __global__ void copy_shot(const float4* __restrict__ a, float4* __restrict__ b, int per, long n4) {
  long base = ((long)blockIdx.x * blockDim.x + threadIdx.x);
  long stride = (long)gridDim.x * blockDim.x;
  float4 v[8];
  #pragma unroll
  for (int j = 0; j < 8; ++j) if (j < per && base + j * stride < n4) v[j] = __ldg(a + base + j * stride);
  #pragma unroll
  for (int j = 0; j < 8; ++j) if (j < per && base + j * stride < n4) b[base + j * stride] = v[j];
}
// grid-stride streaming copy, 4 float4 in flight per thread
extern "C" __global__ void copy_gs(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
  long i = (long)blockIdx.x * blockDim.x * 4 + threadIdx.x;
  long step = (long)gridDim.x * blockDim.x * 4;
  for (; i < n4; i += step) {
    float4 v0, v1, v2, v3;
    v0 = __ldg(a + i);
    if (i + blockDim.x < n4) v1 = __ldg(a + i + blockDim.x);
    if (i + 2 * blockDim.x < n4) v2 = __ldg(a + i + 2 * blockDim.x);
    if (i + 3 * blockDim.x < n4) v3 = __ldg(a + i + 3 * blockDim.x);
    b[i] = v0;
    if (i + blockDim.x < n4) b[i + blockDim.x] = v1;
    if (i + 2 * blockDim.x < n4) b[i + 2 * blockDim.x] = v2;
    if (i + 3 * blockDim.x < n4) b[i + 3 * blockDim.x] = v3;
  }
}
'''


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) == 2 else (r[1:] if isinstance(r, tuple) else None)


def main():
    ck(cu.cuInit(0))
    dev = ck(cu.cuDeviceGet(0))
    ctx = ck(cu.cuDevicePrimaryCtxRetain(dev))
    ck(cu.cuCtxSetCurrent(ctx))
    prog = ck(nvrtc.nvrtcCreateProgram(SRC.encode(), b"calib.cu", 0, [], []))
    opts = [b"-arch=sm_100a"]
    r = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
    if int(r[0]) != 0:
        n = ck(nvrtc.nvrtcGetProgramLogSize(prog))
        log = b" " * n
        nvrtc.nvrtcGetProgramLog(prog, log)
        raise RuntimeError(log.decode())
    n = ck(nvrtc.nvrtcGetCUBINSize(prog))
    cubin = b" " * n
    ck(nvrtc.nvrtcGetCUBIN(prog, cubin))
    mod = ck(cu.cuModuleLoadData(cubin))
    fn = {k: ck(cu.cuModuleGetFunction(mod, k.encode())) for k in ("empty_k", "copy_shot", "copy_gs")}
    stream = ck(cu.cuStreamCreate(0))
    e0, e1 = ck(cu.cuEventCreate(0)), ck(cu.cuEventCreate(0))

    def alloc(nbytes):
        return ck(cu.cuMemAlloc(nbytes))

    def launch(f, grid, block, args):
        if args:
            vals = [ctypes.c_void_p(int(a)) if isinstance(a, cu.CUdeviceptr) else a for a in args]
            ptrs = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
            ck(cu.cuLaunchKernel(f, grid, 1, 1, block, 1, 1, 0, stream, ctypes.addressof(ptrs), 0))
            return vals, ptrs
        ck(cu.cuLaunchKernel(f, grid, 1, 1, block, 1, 1, 0, stream, 0, 0))

    def timed(run, iters=200):
        for _ in range(10):
            run(0)
        ck(cu.cuEventRecord(e0, stream))
        for i in range(iters):
            run(i)
        ck(cu.cuEventRecord(e1, stream))
        ck(cu.cuEventSynchronize(e1))
        return ck(cu.cuEventElapsedTime(e0, e1)) * 1000.0 / iters

    out = []
    out.append({"probe": "empty_kernel_512x256", "us": timed(lambda i: launch(fn["empty_k"], 512, 256, None))})

    # GPU-side per-kernel cost inside ONE CUDA graph (no host launch overhead):
    # N nodes per graph, graph replayed, time / (replays * N)
    def graph_of(n, make):
        ck(cu.cuStreamBeginCapture(stream, cu.CUstreamCaptureMode.CU_STREAM_CAPTURE_MODE_THREAD_LOCAL))
        keep = [make(i) for i in range(n)]
        graph = ck(cu.cuStreamEndCapture(stream))
        gexec = ck(cu.cuGraphInstantiate(graph, 0))
        return gexec, keep

    def graph_us(gexec, n, reps=20):
        ck(cu.cuGraphLaunch(gexec, stream))
        ck(cu.cuStreamSynchronize(stream))
        ck(cu.cuEventRecord(e0, stream))
        for _ in range(reps):
            ck(cu.cuGraphLaunch(gexec, stream))
        ck(cu.cuEventRecord(e1, stream))
        ck(cu.cuEventSynchronize(e1))
        return ck(cu.cuEventElapsedTime(e0, e1)) * 1000.0 / (reps * n)

    for grid in (148, 512, 2048):
        gexec, _ = graph_of(100, lambda i: launch(fn["empty_k"], grid, 256, None))
        out.append({"probe": "graph_empty_node_grid%d" % grid, "us_per_node": graph_us(gexec, 100)})
    for mb in (12.6, 25.2, 50.3):
        nbytes = int(mb * 1e6) // 16 * 16
        n = max(8, int(1.2e9 // (2 * nbytes)))
        bufs = [(alloc(nbytes), alloc(nbytes)) for _ in range(n)]
        n4 = nbytes // 16
        grid = int((n4 + 256 * 6 - 1) // (256 * 6))
        gexec, keep = graph_of(n, lambda i: launch(fn["copy_shot"], grid, 256,
                                                   [bufs[i][0], bufs[i][1], ctypes.c_int(6), ctypes.c_long(n4)]))
        us = graph_us(gexec, n)
        out.append({"probe": "graph_copy_shot_%gMB" % mb, "us_per_node": us, "GBps_rw": 2 * nbytes / us / 1e3,
                    "nodes": n})
        for a, b in bufs:
            cu.cuMemFree(a)
            cu.cuMemFree(b)
    for mb in (12.6, 25.2, 50.3):
        nbytes = int(mb * 1e6) // 16 * 16
        sets = max(4, int(1.2e9 // (2 * nbytes)))
        bufs = [(alloc(nbytes), alloc(nbytes)) for _ in range(sets)]
        n4 = nbytes // 16
        for per in (4, 6, 8):
            grid = int((n4 + 256 * per - 1) // (256 * per))
            us = timed(lambda i: launch(fn["copy_shot"], grid, 256,
                                        [bufs[i % sets][0], bufs[i % sets][1], ctypes.c_int(per), ctypes.c_long(n4)]))
            out.append({"probe": "copy_shot_%gMB_per%d" % (mb, per), "us": us, "GBps_rw": 2 * nbytes / us / 1e3,
                        "grid": grid})
        for grid in (148 * 4, 148 * 8, 148 * 16):
            us = timed(lambda i: launch(fn["copy_gs"], grid, 256,
                                        [bufs[i % sets][0], bufs[i % sets][1], ctypes.c_long(n4)]))
            out.append({"probe": "copy_gs_%gMB_grid%d" % (mb, grid), "us": us, "GBps_rw": 2 * nbytes / us / 1e3})
        for a, b in bufs:
            cu.cuMemFree(a)
            cu.cuMemFree(b)
    for o in out:
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in o.items()}), flush=True)


if __name__ == "__main__":
    main()
