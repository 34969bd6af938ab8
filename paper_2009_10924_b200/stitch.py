"""Python host API over the C-ABI (include/stitch_b200.h), mirroring the
reference's ``stitch::`` entry points for the stitched execution path:

    reference (C++, /root/reference/proj)         here
    ---------------------------------------       ---------------------------------
    parse_graph / serialize_graph  parser.hpp     Graph(text), Graph.serialize()
    explore_fusion_plan + plan_for explorer.hpp   Plan(graph, cfg)
    plan_to_json                   pipeline.hpp   Plan.json()
    emit_kernel_text               planner.hpp    Plan.kernel_text(i)
    plan_kernel                    planner.hpp    plan_kernel(graph, vertices, cfg)
    eval_plan                      sim.hpp        Executor(plan).run(inputs)      [B200]
    run_program                    sim.hpp        Executor(plan, mode="program")  [B200]
    eval_reference                 sim.hpp        Executor(plan, mode="unfused")  [B200]
    random_inputs / compare        sim.hpp        random_inputs(), compare()
    run_pipeline                   pipeline.hpp   run_pipeline(...)

Every compute call runs on the GPU through libstitch_b200.so; there is no
CPU execution path, and a missing library raises instead of falling back.
Errors from the library raise ``StitchError`` carrying its status code
(1 parse/config/planner, 2 execution fault, 3 CUDA/NVRTC, 4 bad argument).
"""
from __future__ import annotations

import ctypes
import json
import re
import warnings
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libstitch_b200.so")
CONFIGS = os.path.join(PKG, "configs")
GRAPHS = os.path.join(PKG, "graphs")

DTYPES = {0: ("f32", np.float32), 1: ("f16", np.float16), 2: ("i32", np.int32), 3: ("bool", np.uint8)}
MODES = {"stitched": 0, "program": 1, "unfused": 2}
NO_GRAPH = 8
GEMM = 16  # model mode: matmul-shaped opaque_compute ops as cuBLASLt GEMMs


class StitchError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


_lib = None


def lib():
    """Load libstitch_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        # a fresh checkout: build the native library in-tree (g++/nvcc/NVRTC;
        # no GPU needed) -- there is no non-native fallback
        try:
            from paper_2009_10924_b200 import build as _build
            _build.build()
        except Exception as e:
            raise StitchError(4, "libstitch_b200.so is not built and the in-tree build failed: %s" % e)
        if not os.path.exists(LIB_PATH):
            raise StitchError(4, "libstitch_b200.so is not built (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    vp, cp, ip, i64 = ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int64
    P = ctypes.POINTER
    sig = {
        "stc_last_error": (cp, []), "stc_free": (None, [vp]), "stc_version": (cp, []),
        "stc_graph_parse": (ip, [cp, P(vp)]), "stc_graph_destroy": (None, [vp]),
        "stc_graph_serialize": (ip, [vp, P(vp)]), "stc_graph_num_nodes": (ip, [vp]),
        "stc_graph_io": (ip, [vp, ip, ip, P(cp), P(ip), P(ip), P(i64)]),
        "stc_plan_create": (ip, [vp, cp, ip, ip, P(vp)]),
        "stc_plan_from_patterns": (ip, [vp, cp, P(ip), P(ip), ip, P(vp)]),
        "stc_plan_destroy": (None, [vp]), "stc_plan_json": (ip, [vp, ctypes.c_uint64, P(vp)]),
        "stc_plan_num_patterns": (ip, [vp]), "stc_plan_pattern": (ip, [vp, ip, P(ip), ip]),
        "stc_plan_kernel_text": (ip, [vp, ip, P(vp)]),
        "stc_plan_stats": (ip, [vp, P(ip), P(ip), P(i64)]),
        "stc_plan_refine": (ip, [vp, P(ip), P(i64)]), "stc_plan_refine_info": (ip, [vp, P(i64), P(ip)]),
        "stc_plan_kernel": (ip, [vp, cp, P(ip), ip, P(vp)]),
        "stc_codegen": (ip, [vp, ip, P(vp), P(vp)]),
        "stc_exec_create": (ip, [vp, ip, ip, P(vp)]), "stc_exec_destroy": (None, [vp]),
        "stc_exec_create_async": (ip, [vp, ip, ip, P(vp)]), "stc_exec_ready": (ip, [vp]),
        "stc_exec_wait": (ip, [vp]), "stc_cache_warm": (ip, [P(vp), ip, ip, ip, P(ip), P(ip)]),
        "stc_exec_num_kernels": (ip, [vp]), "stc_exec_describe": (ip, [vp, P(vp)]),
        "stc_exec_source": (ip, [vp, P(vp)]),
        "stc_exec_run_host": (ip, [vp, P(vp), P(vp)]), "stc_exec_upload": (ip, [vp, P(vp)]),
        "stc_exec_run_host_chunked": (ip, [vp, P(vp), P(vp), ip, P(ip)]),
        "stc_exec_run_host_zero_copy": (ip, [vp, P(vp), P(vp)]),
        "stc_exec_run_host_pipeline": (ip, [P(vp), P(ip), ip, P(vp), P(vp), P(ip)]),
        "stc_exec_trace": (ip, [vp, P(ctypes.c_double), P(ctypes.c_double)]),
        "stc_exec_launch": (ip, [vp, vp, ip]), "stc_exec_prepare_sets": (ip, [vp, ip]),
        "stc_exec_download": (ip, [vp, P(vp)]),
        "stc_exec_sync": (ip, [vp]),
        "stc_exec_tensor": (ip, [vp, cp, P(vp), P(ctypes.c_size_t)]),
        "stc_exec_time": (ip, [vp, ip, ip, ip, P(ctypes.c_double), P(ctypes.c_double)]),
        "stc_exec_time_call": (ip, [vp, ip, ip, ip, P(ctypes.c_double), P(ctypes.c_double)]),
        "stc_exec_prepare_batches": (ip, [vp, ip, ip, P(ip)]),
        "stc_exec_launch_batch": (ip, [vp, vp, ip]),
        "stc_exec_time_batched": (ip, [vp, ip, ip, ip, ip, P(ctypes.c_double)]),
        "stc_compile": (ip, [cp, cp, P(vp)]), "stc_cache_dir": (cp, []),
        "stc_ctx_create": (ip, [ip, P(vp)]), "stc_ctx_destroy": (None, [vp]),
        "stc_ctx_compile": (ip, [vp, cp, P(cp), ip, P(vp)]), "stc_module_destroy": (None, [vp]),
        "stc_ctx_alloc": (ip, [vp, ctypes.c_size_t, P(vp)]), "stc_ctx_release": (ip, [vp, vp]),
        "stc_ctx_upload": (ip, [vp, vp, vp, ctypes.c_size_t]), "stc_ctx_download": (ip, [vp, vp, vp, ctypes.c_size_t]),
        "stc_cgraph_create": (ip, [vp, P(vp)]),
        "stc_cgraph_add_kernel": (ip, [vp, vp, cp, ip, ip, ip, ip, P(vp)]),
        "stc_cgraph_instantiate": (ip, [vp]), "stc_cgraph_launch": (ip, [vp, vp]),
        "stc_cgraph_time": (ip, [vp, ip, ctypes.c_size_t, P(ctypes.c_float)]), "stc_cgraph_destroy": (None, [vp]),
        "stc_nccl_unique_id": (ip, [ctypes.c_char_p]), "stc_nccl_comm_init": (ip, [vp, ip, ip, ctypes.c_char_p, P(vp)]),
        "stc_nccl_gather": (ip, [vp, vp, vp, ctypes.c_size_t, vp]), "stc_nccl_comm_destroy": (None, [vp]),
        "stc_run_pipeline": (ip, [cp, cp, ip, ip, cp, ip, ip, ip, ctypes.c_uint64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise StitchError(rc, lib().stc_last_error().decode())


def _take(p: ctypes.c_void_p) -> str:
    s = ctypes.string_at(p.value).decode()
    lib().stc_free(p)
    return s


def cfg_path(name: Optional[str]) -> str:
    """'v100' / 'b200' (B200 device shape) / 'b200cal' (+ recalibrated costs) / a path / None (-> $STITCH_DEVICE_CONFIG or built-in defaults)."""
    if not name:
        return ""
    if name in ("v100", "default"):
        return os.path.join(CONFIGS, "v100_default.cfg")
    if name == "b200":
        return os.path.join(CONFIGS, "b200_device.cfg")
    if name == "b200cal":  # cost model recalibrated from B200 measurements
        return os.path.join(CONFIGS, "b200.cfg")
    return name


class TensorInfo:
    def __init__(self, name, dtype, dims):
        self.name, self.dtype, self.dims = name, dtype, tuple(dims)

    @property
    def np_dtype(self):
        return {"f32": np.float32, "f16": np.float16, "i32": np.int32, "bool": np.uint8}[self.dtype]

    @property
    def count(self):
        return int(np.prod(self.dims)) if self.dims else 1

    @property
    def nbytes(self):
        return self.count * np.dtype(self.np_dtype).itemsize

    def __repr__(self):
        return "%s:%s%s" % (self.name, self.dtype, list(self.dims))


class Graph:
    """stitch::CompGraph (parse_graph, src/parser.cpp:162-257)."""

    def __init__(self, text: str):
        self.text = text
        self._h = ctypes.c_void_p()
        _check(lib().stc_graph_parse(text.encode(), ctypes.byref(self._h)))
        self.params = self._io(0)
        self.outputs = self._io(1)

    @classmethod
    def from_file(cls, path: str) -> "Graph":
        with open(path) as f:
            return cls(f.read())

    def _io(self, which) -> List[TensorInfo]:
        L = lib()
        n = L.stc_graph_io(self._h, which, -1, None, None, None, None)
        out = []
        for i in range(n):
            name, dt, rank = ctypes.c_char_p(), ctypes.c_int(), ctypes.c_int()
            dims = (ctypes.c_int64 * 8)()
            L.stc_graph_io(self._h, which, i, ctypes.byref(name), ctypes.byref(dt), ctypes.byref(rank), dims)
            out.append(TensorInfo(name.value.decode(), DTYPES[dt.value][0], list(dims[: rank.value])))
        return out

    @property
    def num_nodes(self) -> int:
        return lib().stc_graph_num_nodes(self._h)

    def serialize(self) -> str:
        p = ctypes.c_void_p()
        _check(lib().stc_graph_serialize(self._h, ctypes.byref(p)))
        return _take(p)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stc_graph_destroy(self._h)
            self._h = None


class Plan:
    """explore_fusion_plan + per-pattern plan_kernel under a machine model."""

    def __init__(self, graph: Graph, cfg: Optional[str] = None, k: int = 0, beam: int = 0,
                 patterns: Optional[Sequence[Sequence[int]]] = None):
        self.graph = graph
        self.cfg = cfg_path(cfg)
        self._h = ctypes.c_void_p()
        if patterns is None:
            _check(lib().stc_plan_create(graph._h, self.cfg.encode(), k, beam, ctypes.byref(self._h)))
        else:
            verts = [v for p in patterns for v in p]
            offs = [0]
            for p in patterns:
                offs.append(offs[-1] + len(p))
            va = (ctypes.c_int * max(1, len(verts)))(*verts)
            oa = (ctypes.c_int * len(offs))(*offs)
            _check(lib().stc_plan_from_patterns(graph._h, self.cfg.encode(), va, oa, len(patterns),
                                                ctypes.byref(self._h)))

    def refine(self):
        """NON-PARITY: merge launch units while it saves HBM bytes or launches
        (stc_plan_refine) -> (merges, bytes_saved)"""
        m, b = ctypes.c_int(), ctypes.c_int64()
        _check(lib().stc_plan_refine(self._h, ctypes.byref(m), ctypes.byref(b)))
        pr, hit = ctypes.c_int64(), ctypes.c_int()
        lib().stc_plan_refine_info(self._h, ctypes.byref(pr), ctypes.byref(hit))
        self.refine_info = {"merges": m.value, "bytes_saved": b.value, "probes": pr.value,
                            "budget_hit": bool(hit.value)}
        if hit.value:
            warnings.warn("plan refinement stopped by STITCH_REFINE_MAX_PROBES after %d probes" % pr.value)
        return m.value, b.value

    def json(self, seed: int = 0) -> str:
        p = ctypes.c_void_p()
        _check(lib().stc_plan_json(self._h, seed, ctypes.byref(p)))
        return _take(p)

    @property
    def num_patterns(self) -> int:
        return lib().stc_plan_num_patterns(self._h)

    def patterns(self) -> List[List[int]]:
        out = []
        for i in range(self.num_patterns):
            buf = (ctypes.c_int * 4096)()
            n = lib().stc_plan_pattern(self._h, i, buf, 4096)
            out.append(list(buf[:n]))
        return out

    def kernel_text(self, i: int) -> str:
        p = ctypes.c_void_p()
        _check(lib().stc_plan_kernel_text(self._h, i, ctypes.byref(p)))
        return _take(p)

    def stats(self):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        lib().stc_plan_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        return {"stitched_kernels": a.value, "baseline_kernels": b.value, "delta_evaluate_calls": c.value}

    def codegen(self, mode: str = "stitched", gemm: bool = False):
        """(cuda_source, [kernel descriptions]) without touching a device"""
        s, j = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().stc_codegen(self._h, MODES[mode] | (GEMM if gemm else 0), ctypes.byref(s), ctypes.byref(j)))
        return _take(s), json.loads(_take(j))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stc_plan_destroy(self._h)
            self._h = None


class Context:
    """Low-level runtime (stc_ctx_* / stc_cgraph_* / stc_nccl_*): a device
    context owning buffers, NVRTC modules, explicit CUDA Graphs of launches."""

    def __init__(self, device: int = 0):
        self._h = ctypes.c_void_p()
        _check(lib().stc_ctx_create(device, ctypes.byref(self._h)))
        self._keep = []

    def compile(self, source: str, kernels: Sequence[str]):
        m = ctypes.c_void_p()
        names = (ctypes.c_char_p * len(kernels))(*[k.encode() for k in kernels])
        _check(lib().stc_ctx_compile(self._h, source.encode(), names, len(kernels), ctypes.byref(m)))
        self._keep.append(m)
        return m

    def alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _check(lib().stc_ctx_alloc(self._h, nbytes, ctypes.byref(p)))
        return p.value

    def upload(self, dptr: int, a: np.ndarray):
        a = np.ascontiguousarray(a)
        _check(lib().stc_ctx_upload(self._h, ctypes.c_void_p(dptr), a.ctypes.data, a.nbytes))

    def download(self, dptr: int, out: np.ndarray) -> np.ndarray:
        _check(lib().stc_ctx_download(self._h, out.ctypes.data, ctypes.c_void_p(dptr), out.nbytes))
        return out

    def graph(self):
        return CudaGraph(self)

    def nccl_comm(self, nranks: int, rank: int, unique_id: bytes):
        c = ctypes.c_void_p()
        _check(lib().stc_nccl_comm_init(self._h, nranks, rank, unique_id, ctypes.byref(c)))
        return c

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            for m in self._keep:
                _lib.stc_module_destroy(m)
            _lib.stc_ctx_destroy(self._h)
            self._h = None


class CudaGraph:
    def __init__(self, ctx: Context):
        self.ctx = ctx
        self._h = ctypes.c_void_p()
        _check(lib().stc_cgraph_create(ctx._h, ctypes.byref(self._h)))

    def add_kernel(self, module, name: str, grid: int, block: int, args, smem: int = 0, cooperative: bool = False):
        """args: ctypes values (c_void_p for device pointers, c_int, c_float, ...)"""
        ptrs = (ctypes.c_void_p * max(1, len(args)))(*[ctypes.addressof(a) for a in args])
        _check(lib().stc_cgraph_add_kernel(self._h, module, name.encode(), grid, block, smem, int(cooperative), ptrs))

    def instantiate(self):
        _check(lib().stc_cgraph_instantiate(self._h))

    def launch(self, stream: int = 0):
        _check(lib().stc_cgraph_launch(self._h, ctypes.c_void_p(stream or None)))

    def time(self, iters: int = 20, flush_bytes: int = 0) -> float:
        us = ctypes.c_float()
        _check(lib().stc_cgraph_time(self._h, iters, flush_bytes, ctypes.byref(us)))
        return us.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stc_cgraph_destroy(self._h)
            self._h = None


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().stc_nccl_unique_id(buf))
    return buf.raw


def nccl_gather(comm, send_dptr: int, recv_dptr: int, bytes_per_rank: int, stream: int = 0):
    _check(lib().stc_nccl_gather(comm, ctypes.c_void_p(send_dptr), ctypes.c_void_p(recv_dptr), bytes_per_rank,
                                 ctypes.c_void_p(stream or None)))


def warm_cache(plans: Sequence["Plan"], mode: str = "stitched", threads: int = 8, gemm: bool = False):
    """NVRTC-compile the modules of `plans` into the persistent cubin cache
    (no GPU needed) -> (compiled_now, already_cached)"""
    arr = (ctypes.c_void_p * max(1, len(plans)))(*[p._h.value for p in plans])
    c, h = ctypes.c_int(), ctypes.c_int()
    _check(lib().stc_cache_warm(arr, len(plans), MODES[mode] | (GEMM if gemm else 0), threads, ctypes.byref(c),
                                ctypes.byref(h)))
    return c.value, h.value


def plan_kernel(graph: Graph, vertices: Sequence[int], cfg: Optional[str] = None) -> Optional[str]:
    """stitch::plan_kernel for one vertex set -> program text, None if infeasible."""
    arr = (ctypes.c_int * len(vertices))(*vertices)
    p = ctypes.c_void_p()
    rc = lib().stc_plan_kernel(graph._h, cfg_path(cfg).encode(), arr, len(vertices), ctypes.byref(p))
    if rc == 1 and "infeasible" in lib().stc_last_error().decode():
        return None
    _check(rc)
    return _take(p)


def compile_cuda(source: str, options: str = "") -> str:
    """NVRTC sm_100a compile through the cubin cache; returns the cache key."""
    p = ctypes.c_void_p()
    _check(lib().stc_compile(source.encode(), options.encode(), ctypes.byref(p)))
    return _take(p)


class Executor:
    """A plan compiled for one B200 and replayed as one CUDA Graph
    (eval_plan / run_program / eval_reference, src/sim.cpp:231-514)."""

    def __init__(self, plan: Plan, device: int = 0, mode: str = "stitched", graph: bool = True, gemm: bool = False,
                 async_compile: bool = False):
        self.plan = plan
        self.g = plan.graph
        self._h = ctypes.c_void_p()
        flags = MODES[mode] | (0 if graph else NO_GRAPH) | (GEMM if gemm else 0)
        create = lib().stc_exec_create_async if async_compile else lib().stc_exec_create
        _check(create(plan._h, device, flags, ctypes.byref(self._h)))

    @property
    def ready(self) -> bool:
        """module compiled (always True for synchronous construction)"""
        return bool(lib().stc_exec_ready(self._h))

    def wait(self):
        _check(lib().stc_exec_wait(self._h))

    @property
    def num_kernels(self) -> int:
        return lib().stc_exec_num_kernels(self._h)

    def describe(self):
        p = ctypes.c_void_p()
        _check(lib().stc_exec_describe(self._h, ctypes.byref(p)))
        return json.loads(_take(p))

    def source(self) -> str:
        p = ctypes.c_void_p()
        _check(lib().stc_exec_source(self._h, ctypes.byref(p)))
        return _take(p)

    def _in_ptrs(self, inputs: Dict[str, np.ndarray]):
        arrs = []
        for t in self.g.params:
            a = np.ascontiguousarray(inputs[t.name], dtype=t.np_dtype)
            if a.size != t.count:
                raise StitchError(4, "input %s has %d elements, expected %d" % (t.name, a.size, t.count))
            arrs.append(a)
        return arrs, (ctypes.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])

    def _out_ptrs(self):
        outs = [np.empty(t.dims, dtype=t.np_dtype) for t in self.g.outputs]
        return outs, (ctypes.c_void_p * max(1, len(outs)))(*[o.ctypes.data for o in outs])

    def run(self, inputs: Dict[str, np.ndarray], out: Optional[Dict[str, np.ndarray]] = None):
        """host inputs -> H2D -> one graph launch -> D2H -> host outputs
        (`out`: preallocated, e.g. pinned, output arrays to fill)"""
        keep, ip = self._in_ptrs(inputs)
        if out is None:
            outs, op = self._out_ptrs()
        else:
            outs = [out[t.name] for t in self.g.outputs]
            for o, t in zip(outs, self.g.outputs):
                if not (o.flags.c_contiguous and o.dtype == t.np_dtype and o.size == t.count):
                    raise StitchError(4, "bad output buffer for " + t.name)
            op = (ctypes.c_void_p * max(1, len(outs)))(*[o.ctypes.data for o in outs])
        _check(lib().stc_exec_run_host(self._h, ip, op))
        return {t.name: o for t, o in zip(self.g.outputs, outs)}

    def run_zero_copy(self, inputs: Dict[str, np.ndarray], out: Dict[str, np.ndarray]):
        """pinned host inputs/outputs read and written by the kernels directly
        over PCIe (stc_exec_run_host_zero_copy); every buffer must be pinned"""
        keep, ip = self._in_ptrs(inputs)
        outs = [out[t.name] for t in self.g.outputs]
        for o, t in zip(outs, self.g.outputs):
            if not (o.flags.c_contiguous and o.dtype == t.np_dtype and o.size == t.count):
                raise StitchError(4, "bad output buffer for " + t.name)
        op = (ctypes.c_void_p * max(1, len(outs)))(*[o.ctypes.data for o in outs])
        _check(lib().stc_exec_run_host_zero_copy(self._h, ip, op))
        return {t.name: o for t, o in zip(self.g.outputs, outs)}

    def trace(self):
        """[(start_us, end_us)] per kernel of one replay (needs STITCH_TRACE=1
        in the environment when the executor was created)"""
        n = self.num_kernels
        d = self.describe()
        if n == 1 and d[0]["template"].startswith("persistent("):  # + one entry per unit
            n = 1 + int(d[0]["template"][11:-1])
        if n == 1 and d[0]["template"].startswith("resident("):  # + one entry per step
            n = 1 + int(re.search(r" (\d+) steps", d[0]["template"]).group(1))
        n *= max(1, int(os.environ.get("STITCH_TRACE_CTAS", "0") or 0))  # per-CTA slots: k * CTAS + CTA
        a, b = (ctypes.c_double * max(1, n))(), (ctypes.c_double * max(1, n))()
        _check(lib().stc_exec_trace(self._h, a, b))
        return list(zip(a[:n], b[:n]))

    def upload(self, inputs: Dict[str, np.ndarray]):
        keep, ip = self._in_ptrs(inputs)
        _check(lib().stc_exec_upload(self._h, ip))
        _check(lib().stc_exec_sync(self._h))

    def launch(self, stream: int = 0, set: int = 0):
        """async replay of the plan's CUDA Graph on `stream` (a cudaStream_t as int)"""
        _check(lib().stc_exec_launch(self._h, ctypes.c_void_p(stream or None), set))

    def prepare_sets(self, sets: int):
        _check(lib().stc_exec_prepare_sets(self._h, sets))

    def sync(self):
        _check(lib().stc_exec_sync(self._h))

    def download(self) -> Dict[str, np.ndarray]:
        outs, op = self._out_ptrs()
        _check(lib().stc_exec_download(self._h, op))
        _check(lib().stc_exec_sync(self._h))
        return {t.name: o for t, o in zip(self.g.outputs, outs)}

    def tensor_ptr(self, name: str):
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().stc_exec_tensor(self._h, name.encode(), ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def time(self, iters: int = 100, warmup: int = 10, sets: int = 1, per_kernel: bool = False):
        """(us per graph replay, [us per kernel] or None)"""
        us = ctypes.c_double()
        kus = (ctypes.c_double * max(1, self.num_kernels))() if per_kernel else None
        _check(lib().stc_exec_time(self._h, iters, warmup, sets, ctypes.byref(us), kus))
        return us.value, (list(kus[: self.num_kernels]) if per_kernel else None)

    def time_call(self, iters: int = 100, warmup: int = 10, sets: int = 1, per_kernel: bool = False):
        """(us per call, [us per kernel] or None): each replay queued behind a
        spinning warp so the events time the device, not the host submission"""
        us = ctypes.c_double()
        kus = (ctypes.c_double * max(1, self.num_kernels))() if per_kernel else None
        _check(lib().stc_exec_time_call(self._h, iters, warmup, sets, ctypes.byref(us), kus))
        return us.value, (list(kus[: self.num_kernels]) if per_kernel else None)

    def prepare_batches(self, sets: int, steps_per_graph: int) -> int:
        n = ctypes.c_int()
        _check(lib().stc_exec_prepare_batches(self._h, sets, steps_per_graph, ctypes.byref(n)))
        return n.value

    def launch_batch(self, stream: int, index: int):
        _check(lib().stc_exec_launch_batch(self._h, ctypes.c_void_p(stream or None), index))

    def time_batched(self, steps: int = 512, warmup: int = 32, sets: int = 8, steps_per_graph: int = 16):
        us = ctypes.c_double()
        _check(lib().stc_exec_time_batched(self._h, steps, warmup, sets, steps_per_graph, ctypes.byref(us)))
        return us.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stc_exec_destroy(self._h)
            self._h = None


class ChunkedExecutor:
    """Host-buffer execution of a batch-sharded graph as pipelined chunks:
    each chunk graph (re-planned by the bit-exact planner for its own shape)
    runs on device while the next chunk's H2D and the previous chunk's D2H are
    in flight.  `chunks` = number of equal chunks, or a list of chunk extents
    along the sharded axis (e.g. [1, 3, 4, 4, 4, 4, 4, 4, 3, 1]: small first /
    last chunks shorten the pipeline's fill and drain) -> one executor per
    distinct extent, stc_exec_run_host_pipeline.  `rule` is a
    shard.ShardRule whose sharded axis is 0 for every chunked tensor."""

    def __init__(self, text: str, rule, chunks, cfg: str = "b200", device: int = 0):
        if isinstance(chunks, int):
            chunks = [rule.shard_size(chunks)] * chunks
        if sum(chunks) != rule.full:
            raise StitchError(4, "chunk extents %s do not sum to %d" % (chunks, rule.full))
        self.rule, self.chunks = rule, list(chunks)
        self.nchunks = len(chunks)
        self.full = Graph(text)
        self.execs = {}
        for b in sorted(set(chunks)):
            self.execs[b] = Executor(Plan(Graph(rule.extent_text(text, b)), cfg), device=device)
        self.ex = self.execs[chunks[0]]
        sizes = sorted(self.execs)
        self._handles = (ctypes.c_void_p * len(sizes))(*[self.execs[b]._h.value for b in sizes])
        self._of_chunk = (ctypes.c_int * len(chunks))(*[sizes.index(b) for b in chunks])
        for t in self.full.params:
            if rule.axis_of.get(t.name) not in (None, 0):
                raise StitchError(4, "input %s is not sharded along axis 0" % t.name)
        for t in self.full.outputs:
            if rule.axis_of.get(t.name) != 0:
                raise StitchError(4, "output %s is not sharded along axis 0" % t.name)
        self._flags = (ctypes.c_int * max(1, len(self.full.params)))(
            *[1 if t.name in rule.axis_of else 0 for t in self.full.params])

    def run(self, inputs: Dict[str, np.ndarray], out: Optional[Dict[str, np.ndarray]] = None):
        keep = [np.ascontiguousarray(inputs[t.name], dtype=t.np_dtype) for t in self.full.params]
        for a, t in zip(keep, self.full.params):
            if a.size != t.count:
                raise StitchError(4, "input %s has %d elements, expected %d" % (t.name, a.size, t.count))
        ip = (ctypes.c_void_p * max(1, len(keep)))(*[a.ctypes.data for a in keep])
        outs = [out[t.name] if out is not None else np.empty(t.dims, dtype=t.np_dtype) for t in self.full.outputs]
        for o, t in zip(outs, self.full.outputs):
            if not (o.flags.c_contiguous and o.dtype == t.np_dtype and o.size == t.count):
                raise StitchError(4, "bad output buffer for " + t.name)
        op = (ctypes.c_void_p * max(1, len(outs)))(*[o.ctypes.data for o in outs])
        _check(lib().stc_exec_run_host_pipeline(self._handles, self._of_chunk, self.nchunks, ip, op, self._flags))
        return {t.name: o for t, o in zip(self.full.outputs, outs)}


def run_pipeline(graph_path: str, device_config: Optional[str] = None, k: int = 3, beam_width: int = 3,
                 output_dir: str = "out", emit_dot: bool = False, run_sim: bool = False,
                 run_baseline: bool = False, seed: int = 0) -> int:
    """stitch::run_pipeline: 0 ok, 1 parse/config/planner error, 2 sim mismatch."""
    return lib().stc_run_pipeline(graph_path.encode(), cfg_path(device_config).encode(), k, beam_width,
                                  output_dir.encode(), int(emit_dot), int(run_sim), int(run_baseline),
                                  seed)


# ---- host-side utilities (sim.hpp) ----------------------------------------
_PHI = np.uint64(0x9E3779B97F4A7C15)


def random_inputs(graph: Graph, seed: int, gather_bounds: Optional[Dict[str, int]] = None):
    """splitmix64 uniform(-1,1) draws rounded to dtype, parameters in
    declaration order (src/sim.cpp:630-659).  Vectorised counter form: draw k
    uses state seed + phi*(k+2)."""
    out, drawn = {}, 0
    with np.errstate(over="ignore"):
        for t in graph.params:
            k = np.arange(drawn, drawn + t.count, dtype=np.uint64)
            drawn += t.count
            z = np.uint64(seed) + _PHI * (k + np.uint64(2))
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            if t.dtype == "i32":
                bound = (gather_bounds or {}).get(t.name, 10)
                v = (z % np.uint64(bound)).astype(np.int32)
            elif t.dtype == "bool":
                v = (z & np.uint64(1)).astype(np.uint8)
            else:
                u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0
                v = u.astype(np.float32).astype(t.np_dtype)
            out[t.name] = v.reshape(t.dims)
    return out


def compare(got: Dict[str, np.ndarray], want: Dict[str, np.ndarray], rel_tol: float, abs_tol: float):
    """per element: pass iff abs <= abs_tol OR rel <= rel_tol (src/sim.cpp:516-547)"""
    res = {"pass": True, "max_abs": 0.0, "max_rel": 0.0, "message": ""}
    for name, w in want.items():
        a = np.asarray(got[name], dtype=np.float64).reshape(-1)
        b = np.asarray(w, dtype=np.float64).reshape(-1)
        ad = np.abs(a - b)
        rd = ad / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-30)
        if ad.size:
            res["max_abs"] = max(res["max_abs"], float(np.max(ad)))
            if (ad > 0).any():
                res["max_rel"] = max(res["max_rel"], float(rd[ad > 0].max()))
        ok = (ad <= abs_tol) | (rd <= rel_tol)
        if not ok.all() and res["pass"]:
            i = int(np.argmin(ok))
            res["pass"] = False
            res["message"] = "mismatch on %s[%d]: got %.9g, want %.9g" % (name, i, a[i], b[i])
    return res
