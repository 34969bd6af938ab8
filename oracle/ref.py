"""ctypes binding of oracle/_ref/libstitch_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the unmodified reference (/root/reference/proj/src, built by
oracle/Makefile) plus oracle/ref_shim.cpp.  Used by tests/, smoke() and
bench.py's CPU-baseline leg; never by the product path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libstitch_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError("oracle/_ref/libstitch_ref.so not built (make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        c, P = ctypes.c_char_p, ctypes.POINTER
        L.ref_last_error.restype = c
        L.ref_plan.argtypes = [c, c, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                               P(ctypes.c_void_p), P(ctypes.c_void_p), P(ctypes.c_void_p)]
        L.ref_plan_kernel.argtypes = [c, c, P(ctypes.c_int), ctypes.c_int, P(ctypes.c_void_p)]
        L.ref_serialize.argtypes = [c, P(ctypes.c_void_p)]
        L.ref_random.argtypes = [c, ctypes.c_uint64, P(ctypes.c_void_p), ctypes.c_int]
        L.ref_eval.argtypes = [c, P(ctypes.c_void_p), ctypes.c_int, P(ctypes.c_void_p),
                               ctypes.c_int]
        L.ref_eval_plan.argtypes = [c, c, P(ctypes.c_void_p), ctypes.c_int,
                                    P(ctypes.c_void_p), ctypes.c_int]
        L.ref_time_eval.argtypes = [P(c), ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                    P(ctypes.c_double)]
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_run_pipeline.argtypes = [c, c, ctypes.c_int, ctypes.c_int, c, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_uint64]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise RuntimeError("reference rc=%d: %s" % (rc, lib().ref_last_error().decode()))


def _take(p):
    s = ctypes.string_at(p.value).decode()
    lib().ref_free(p)
    return s


def plan(graph_text: str, cfg_path: str = "", k: int = 0, beam: int = 0, seed: int = 0):
    """-> (plan_json_text, {pattern_key: program_text}, summary_text)"""
    a, b, c = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _check(lib().ref_plan(graph_text.encode(), cfg_path.encode(), k, beam, seed,
                          ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    pj, kt, summ = _take(a), _take(b), _take(c)
    progs = {}
    for block in kt.split("=== ")[1:]:
        key, body = block.split("\n", 1)
        progs[key] = body
    return pj, progs, summ


def plan_kernel(graph_text: str, verts, cfg_path: str = ""):
    arr = (ctypes.c_int * len(verts))(*verts)
    out = ctypes.c_void_p()
    rc = lib().ref_plan_kernel(graph_text.encode(), cfg_path.encode(), arr, len(verts),
                               ctypes.byref(out))
    if rc == 3:
        return None
    _check(rc)
    return _take(out)


def serialize(graph_text: str) -> str:
    out = ctypes.c_void_p()
    _check(lib().ref_serialize(graph_text.encode(), ctypes.byref(out)))
    return _take(out)


def _ptrs(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def random_inputs(graph_text: str, param_shapes, seed: int):
    """param_shapes: list of (name, dims) in declaration order -> {name: f64 array}"""
    bufs = [np.zeros(int(np.prod(d)) if d else 1, dtype=np.float64) for _, d in param_shapes]
    _check(lib().ref_random(graph_text.encode(), seed, _ptrs(bufs), len(bufs)))
    return {n: b.reshape(d) for (n, d), b in zip(param_shapes, bufs)}


def eval_reference(graph_text: str, inputs_in_order, output_shapes):
    ins = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in inputs_in_order]
    outs = [np.zeros(int(np.prod(d)) if d else 1, dtype=np.float64) for d in output_shapes]
    _check(lib().ref_eval(graph_text.encode(), _ptrs(ins), len(ins), _ptrs(outs), len(outs)))
    return [o.reshape(d) for o, d in zip(outs, output_shapes)]


def eval_plan(graph_text: str, cfg_path: str, inputs_in_order, output_shapes):
    ins = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in inputs_in_order]
    outs = [np.zeros(int(np.prod(d)) if d else 1, dtype=np.float64) for d in output_shapes]
    _check(lib().ref_eval_plan(graph_text.encode(), cfg_path.encode(), _ptrs(ins), len(ins),
                               _ptrs(outs), len(outs)))
    return [o.reshape(d) for o, d in zip(outs, output_shapes)]


def time_eval(shard_texts, seed: int = 1, reps: int = 3) -> float:
    """best-of-reps wall seconds of eval_reference, one thread per shard graph"""
    arr = (ctypes.c_char_p * len(shard_texts))(*[t.encode() for t in shard_texts])
    best = ctypes.c_double()
    _check(lib().ref_time_eval(arr, len(shard_texts), seed, reps, ctypes.byref(best)))
    return best.value


def run_pipeline(graph_path: str, cfg_path: str, out_dir: str, k: int = 3, beam: int = 3, emit_dot: bool = False,
                 run_sim: bool = False, run_baseline: bool = False, seed: int = 0) -> int:
    """the reference's run_pipeline (src/pipeline.cpp:110-224) -> return code"""
    return lib().ref_run_pipeline(graph_path.encode(), (cfg_path or "").encode(), k, beam, out_dir.encode(),
                                  int(emit_dot), int(run_sim), int(run_baseline), seed)
