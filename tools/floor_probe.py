"""Same-byte floors for the isolated (one launch, cold L2) latency of a config
kernel: an empty kernel and a plain 128-bit streaming kernel that reads R and
writes W bytes -- R and W equal to the config kernel's algorithmic bytes --
built with the same runtime (NVRTC sm_100a, CUDA Graph, one launch per replay,
L2 flushed before each replay), so that

    python tools/floor_probe.py                 # event times, JSON lines
    ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_elapsed.max \\
        python tools/floor_probe.py --ncu       # the same launches, cold, under ncu

puts each config kernel next to the fastest kernel that moves its bytes.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch  # noqa: E402

# (config, read bytes, write bytes) -- algorithmic bytes of the one planned kernel
SHAPES = [("ln_4096x768", 12589056, 12582912), ("bert_resln", 25174016, 12582912),
          ("attn_softmax", 25182208, 25165824), ("bert_gelu", 50343936, 50331648),
          ("colreduce", 134217728, 8192), ("bert_cut", 75518976, 62914560)]

SRC = r"""
extern "C" __global__ void empty_k() {}
// every output chunk j = sum of the input chunks j, j + nw, j + 2 nw, ... (< nr):
// reads all R bytes once, writes all W bytes once, 8 chunks per thread
extern "C" __global__ void __launch_bounds__(256) stream_k(const float4* __restrict__ in, float4* __restrict__ out,
                                                           long long nr, long long nw) {
  const long long base = (long long)blockIdx.x * 256 * 8 + threadIdx.x;
  float4 v[8];
  #pragma unroll
  for (int k = 0; k < 8; ++k) {
    const long long j = base + 256LL * k;
    v[k] = j < nw ? __ldcs(in + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  #pragma unroll
  for (int k = 0; k < 8; ++k) {
    const long long j = base + 256LL * k;
    if (j >= nw) continue;
    for (long long i = j + nw; i < nr; i += nw) {
      const float4 q = __ldcs(in + i);
      v[k].x += q.x; v[k].y += q.y; v[k].z += q.z; v[k].w += q.w;
    }
    __stcs(out + j, v[k]);
  }
}
// columns: W is tiny (8 KB), so chunks stride over R instead (reduce-like read stream)
extern "C" __global__ void __launch_bounds__(256) read_k(const float4* __restrict__ in, float4* __restrict__ out,
                                                         long long nr, long long nw) {
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < nr; i += (long long)gridDim.x * 256) {
    const float4 q = __ldcs(in + i);
    a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
  }
  if (a.x == 12345.f) out[threadIdx.x % nw] = a;
}
"""


def main():
    ncu = "--ncu" in sys.argv
    ctx = stitch.Context(0)
    mod = ctx.compile(SRC, ["empty_k", "stream_k", "read_k"])
    iters = 3 if ncu else 200
    flush = 0 if ncu else 256 << 20
    g = ctx.graph()
    g.add_kernel(mod, "empty_k", 148, 256, [])
    g.instantiate()
    print(json.dumps({"probe": "empty_kernel_graph_one_launch", "us": round(g.time(iters, flush), 3)}), flush=True)
    for name, r, w in SHAPES:
        inp, out = ctx.alloc(r), ctx.alloc(max(w, 4096))
        nr, nw = r // 16, max(1, w // 16)
        args = [ctypes.c_void_p(inp), ctypes.c_void_p(out), ctypes.c_int64(nr), ctypes.c_int64(nw)]
        g = ctx.graph()
        if w >= r // 8:
            grid = (nw + 2047) // 2048
            g.add_kernel(mod, "stream_k", grid, 256, args)
        else:
            grid = 148 * 8
            g.add_kernel(mod, "read_k", grid, 256, args)
        g.instantiate()
        us = g.time(iters, flush)
        print(json.dumps({"probe": "stream_floor", "config": name, "read_bytes": r, "write_bytes": w, "grid": grid,
                          "us_one_launch_flushed": round(us, 3),
                          "GBps": round((r + w) / us / 1e3, 1)}), flush=True)
        if not ncu:  # the config kernel itself, the same way
            gr = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
            ex = stitch.Executor(stitch.Plan(gr, "b200"))
            ex.upload(stitch.random_inputs(gr, 1))
            us1, kus = ex.time(iters=200, warmup=20, sets=max(2, (8 * 126 << 20) // (r + w) + 1), per_kernel=True)
            print(json.dumps({"probe": "config_kernel", "config": name, "us_one_launch_per_step": round(us1, 3),
                              "kernel_event_us": [round(x, 3) for x in kus]}), flush=True)


if __name__ == "__main__":
    main()
