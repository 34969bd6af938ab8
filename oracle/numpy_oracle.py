"""CPU ORACLE — test infrastructure only, never imported by the product path.

A numpy restatement of the reference's numeric semantics for the stitched
execution path, used by tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg as the checker.  Each function cites the reference code it
restates (paths relative to /root/reference/proj):

* ``parse_graph``    — src/parser.cpp:17-257 (statement split, attrs, output /
                       alias roots, implicit sink outputs) + src/graph.cpp:155-245
                       (shape rules).  Validation is reduced to what shape
                       inference needs; the product parser is checked against the
                       reference's own serializer instead.
* ``round_to_dtype`` — src/sim.cpp:67-75 (f32 via float cast; f16 via f32->f16
                       round-nearest-even; i32 llround; bool != 0).
* ``eval_node`` / ``eval_reference`` — src/sim.cpp:111-250: f64 compute on
                       dtype-rounded operands, result rounded per op; reductions
                       accumulate in f64 (numpy's pairwise order instead of the
                       reference's input order — differences are O(1e-16)
                       relative, below f32 resolution); ``opaque_compute`` is
                       the mean of all operand elements broadcast (sim.cpp:215-226).
* ``random_inputs``  — src/sim.cpp:630-659: splitmix64 from seed+phi, one draw
                       per element, parameters in node order; f32 = uniform(-1,1)
                       rounded; i32 = next % bound (bound = min gather extent,
                       default 10); bool = next & 1.  Vectorised: draw k uses
                       state seed + phi*(k+2).
* ``compare``        — src/sim.cpp:516-547: pass iff abs <= abs_tol OR
                       rel <= rel_tol per element, integral dtypes exact.

Parity of this restatement is PINNED against the reference itself: the
committed vectors in tests/golden/ were produced by the unmodified reference
(oracle/_ref, built by oracle/Makefile) with tests/golden/make_golden.py, and
tests/test_oracle.py checks this module against them bit for bit.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

LIGHT = ("add", "sub", "mul", "div", "max", "min")
EXPENSIVE = ("exp", "tanh", "log", "rsqrt", "power")
REDUCE = ("reduce_sum", "reduce_max")
SHAPE = ("broadcast", "transpose", "slice", "gather", "constant", "parameter")
ARITY = {**{k: 2 for k in LIGHT}, "exp": 1, "tanh": 1, "log": 1, "rsqrt": 1, "power": 2,
         "reduce_sum": 1, "reduce_max": 1, "broadcast": 1, "transpose": 1, "slice": 1,
         "gather": 2, "constant": 0, "parameter": 0, "opaque_compute": -1}
DTYPE_BYTES = {"f32": 4, "f16": 2, "i32": 4, "bool": 1}
PHI = np.uint64(0x9E3779B97F4A7C15)


@dataclass
class Node:
    id: int
    name: str
    kind: str
    operands: list
    dtype: str
    dims: tuple
    attrs: dict = field(default_factory=dict)


@dataclass
class Graph:
    nodes: list
    outputs: list
    by_name: dict

    def params(self):
        return [n for n in self.nodes if n.kind == "parameter"]


def _split_statements(text):
    out, cur, line, cur_line, in_comment = [], [], 1, 1, False
    for c in text:
        if c == "\n":
            s = "".join(cur).strip(" \t\r")
            if s:
                out.append((s, cur_line))
            cur, in_comment = [], False
            line += 1
            cur_line = line
        elif c == "#":
            in_comment = True
        elif c == ";" and not in_comment:
            s = "".join(cur).strip(" \t\r")
            if s:
                out.append((s, cur_line))
            cur, cur_line = [], line
        elif not in_comment:
            cur.append(c)
    s = "".join(cur).strip(" \t\r")
    if s:
        out.append((s, cur_line))
    return out


def _int_list(v):
    v = v.strip()
    if v.startswith("["):
        v = v[1:-1]
    return [int(x) for x in v.split(",") if x.strip()]


_SHAPE_RE = re.compile(r"^(f32|f16|i32|bool)\[([0-9,\s]*)\]$")


def _infer(kind, ops, attrs, declared):
    if kind in ("parameter", "constant", "opaque_compute"):
        return declared
    if kind == "broadcast":
        return (ops[0][0], declared[1])
    if kind == "transpose":
        return (ops[0][0], tuple(ops[0][1][p] for p in attrs["perm"]))
    if kind == "slice":
        return (ops[0][0], tuple(l - s for s, l in zip(attrs["starts"], attrs["limits"])))
    if kind == "gather":
        return (ops[0][0], tuple(ops[1][1]) + tuple(ops[0][1][1:]))
    if kind in REDUCE:
        ax = set(attrs["axes"])
        return (ops[0][0], tuple(d for i, d in enumerate(ops[0][1]) if i not in ax))
    return ops[0]


def parse_graph(text: str) -> Graph:
    nodes, by_name, outputs = [], {}, []
    for stmt, _line in _split_statements(text):
        m = re.match(r"^output(?![A-Za-z0-9_.])\s*([A-Za-z0-9_.]+)$", stmt)
        if m:
            nid = by_name[m.group(1)]
            if nid not in outputs:
                outputs.append(nid)
            continue
        lhs, rhs = [s.strip() for s in stmt.split("=", 1)]
        m = re.match(r"^([A-Za-z0-9_.]+)\s*(.*)$", rhs)
        head, rest = m.group(1), m.group(2)
        if head not in ARITY:
            if head in by_name and not rest.strip():
                if by_name[head] not in outputs:
                    outputs.append(by_name[head])
                continue
            raise ValueError("unknown op kind: " + head)
        operands, attrs, declared = [], {}, None

        def apply(k, v):
            if k in ("axes", "axis"):
                attrs["axes"] = _int_list(v)
            elif k in ("dims", "perm", "starts", "limits"):
                attrs[k] = _int_list(v)
            elif k == "value":
                attrs["value"] = float(v)
            else:
                raise ValueError("unknown attribute " + k)

        rest = rest.strip()
        if rest.startswith("("):
            depth, j = 0, 0
            for j, c in enumerate(rest):
                depth += c == "("
                depth -= c == ")"
                if depth == 0:
                    break
            inner, rest = rest[1:j], rest[j + 1:]
            items, cur, d = [], "", 0
            for c in inner:
                d += c == "["
                d -= c == "]"
                if c == "," and d == 0:
                    items.append(cur)
                    cur = ""
                else:
                    cur += c
            if cur.strip():
                items.append(cur)
            for it in items:
                it = it.strip()
                if "=" in it:
                    k, v = it.split("=", 1)
                    apply(k.strip(), v.strip())
                else:
                    operands.append(by_name[it])
        toks, cur, d = [], "", 0
        for c in rest:
            d += c == "["
            d -= c == "]"
            if d == 0 and c in " \t:":
                if cur:
                    toks.append(cur)
                cur = ""
            else:
                cur += c
        if cur:
            toks.append(cur)
        for t in toks:
            sm = _SHAPE_RE.match(t)
            if sm:
                dims = tuple(int(x) for x in sm.group(2).split(",") if x.strip())
                declared = (sm.group(1), dims)
            elif "=" in t:
                k, v = t.split("=", 1)
                apply(k, v)
            else:
                raise ValueError("unexpected token " + t)
        ops = [(nodes[o].dtype, nodes[o].dims) for o in operands]
        dtype, dims = _infer(head, ops, attrs, declared)
        n = Node(len(nodes), lhs, head, operands, dtype, tuple(dims), attrs)
        by_name[lhs] = n.id
        nodes.append(n)
    if not outputs:
        consumed = {o for n in nodes for o in n.operands}
        outputs = [n.id for n in nodes if n.id not in consumed]
    return Graph(nodes, outputs, by_name)


def round_to_dtype(a, dtype):
    a = np.asarray(a, dtype=np.float64)
    if dtype == "f32":
        return a.astype(np.float32).astype(np.float64)
    if dtype == "f16":
        return a.astype(np.float32).astype(np.float16).astype(np.float64)
    if dtype == "i32":
        r = np.where(a >= 0, np.floor(a + 0.5), np.ceil(a - 0.5))  # llround
        return r.astype(np.int64).astype(np.int32).astype(np.float64)
    if dtype == "bool":
        return (a != 0).astype(np.float64)
    raise ValueError(dtype)


def _broadcast(x, in_dims, out_dims, dims):
    # dims[i] = output axis of input axis i (src/sim.cpp:166-179)
    order = np.argsort(dims, kind="stable")
    xt = np.transpose(x.reshape(in_dims), order) if len(in_dims) else x.reshape(())
    shape = [1] * len(out_dims)
    for i in order:
        shape[dims[i]] = in_dims[i]
    return np.broadcast_to(xt.reshape(shape), out_dims)


def eval_node(n: Node, ops, g: Graph):
    k, shp = n.kind, n.dims
    if k == "constant":
        return np.full(shp, round_to_dtype(n.attrs.get("value", 0.0), n.dtype))
    if k in LIGHT or k == "power":
        a, b = ops
        with np.errstate(all="ignore"):
            r = {"add": lambda: a + b, "sub": lambda: a - b, "mul": lambda: a * b,
                 "div": lambda: a / b, "max": lambda: np.where(a < b, b, a),
                 "min": lambda: np.where(b < a, b, a), "power": lambda: np.power(a, b)}[k]()
        return round_to_dtype(r, n.dtype)
    if k in ("exp", "tanh", "log", "rsqrt"):
        (a,) = ops
        with np.errstate(all="ignore"):
            r = {"exp": np.exp, "tanh": np.tanh, "log": np.log,
                 "rsqrt": lambda v: 1.0 / np.sqrt(v)}[k](a)
        return round_to_dtype(r, n.dtype)
    if k in REDUCE:
        ax = tuple(sorted(set(n.attrs["axes"])))
        r = ops[0].sum(axis=ax) if k == "reduce_sum" else ops[0].max(axis=ax)
        return round_to_dtype(np.asarray(r).reshape(shp), n.dtype)
    if k == "broadcast":
        src = g.nodes[n.operands[0]]
        return np.ascontiguousarray(_broadcast(ops[0], src.dims, shp, n.attrs.get("dims", [])))
    if k == "transpose":
        return np.ascontiguousarray(np.transpose(ops[0], n.attrs["perm"]))
    if k == "slice":
        sl = tuple(slice(s, l) for s, l in zip(n.attrs["starts"], n.attrs["limits"]))
        return np.ascontiguousarray(ops[0][sl])
    if k == "gather":
        data, idx = ops
        return np.ascontiguousarray(data[idx.astype(np.int64)])
    if k == "opaque_compute":
        tot = sum(float(o.sum()) for o in ops)
        cnt = sum(o.size for o in ops)
        return np.full(shp, round_to_dtype(tot / cnt if cnt else 0.0, n.dtype))
    raise ValueError("no evaluation rule for " + k)


def eval_reference(g: Graph, inputs: dict, opaque=None) -> dict:
    """inputs: name -> float64 array (dtype-rounded).  Returns outputs by name.
    `opaque(node, operand_values)` may replace the placeholder semantics of
    opaque_compute (model-mode checks; None -> the reference's mean)."""
    vals = {}
    for n in g.nodes:  # parsed graphs are topologically ordered by id
        if n.kind == "parameter":
            vals[n.id] = np.asarray(inputs[n.name], dtype=np.float64).reshape(n.dims)
            continue
        ops = [vals[o] for o in n.operands]
        r = opaque(n, ops) if (opaque is not None and n.kind == "opaque_compute") else None
        vals[n.id] = r if r is not None else eval_node(n, ops, g)
    return {g.nodes[o].name: vals[o] for o in g.outputs}


def matmul_opaque(n: Node, ops):
    """model-mode semantics of a matmul-shaped opaque_compute (A[..,M,K] .
    B[K,N] -> [..,M,N]): the f64 product rounded to the node dtype; None for
    any other opaque op (keeps the placeholder)"""
    if len(ops) != 2 or ops[1].ndim != 2 or ops[0].ndim < 2 or ops[0].shape[-1] != ops[1].shape[0]:
        return None
    return round_to_dtype(ops[0] @ ops[1], n.dtype)


def _splitmix(seed, start, count):
    k = np.arange(start, start + count, dtype=np.uint64)
    z = np.uint64(seed) + PHI * (k + np.uint64(2))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def random_inputs(g: Graph, seed: int) -> dict:
    out, drawn = {}, 0
    for n in g.params():
        cnt = int(np.prod(n.dims)) if n.dims else 1
        z = _splitmix(seed, drawn, cnt)
        drawn += cnt
        if n.dtype == "i32":
            bound = 10
            for c in g.nodes:
                if c.kind == "gather" and len(c.operands) == 2 and c.operands[1] == n.id:
                    bound = min(bound, g.nodes[c.operands[0]].dims[0])
            v = (z % np.uint64(bound)).astype(np.float64)
        elif n.dtype == "bool":
            v = (z & np.uint64(1)).astype(np.float64)
        else:
            u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0
            v = round_to_dtype(u, n.dtype)
        out[n.name] = v.reshape(n.dims)
    return out


@dataclass
class CompareReport:
    passed: bool
    max_abs: float
    max_rel: float
    message: str = ""


def compare(got: dict, want: dict, rel_tol: float, abs_tol: float, dtypes=None) -> CompareReport:
    ok, max_abs, max_rel, msg = True, 0.0, 0.0, ""
    for name, w in want.items():
        if name not in got:
            return CompareReport(False, max_abs, max_rel, "missing output: " + name)
        a = np.asarray(got[name], dtype=np.float64).reshape(-1)
        b = np.asarray(w, dtype=np.float64).reshape(-1)
        if a.shape != b.shape:
            return CompareReport(False, max_abs, max_rel, "shape mismatch on " + name)
        ad = np.abs(a - b)
        den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-30)
        rd = ad / den
        if ad.size:
            max_abs = max(max_abs, float(np.nanmax(ad)) if not np.isnan(ad).all() else np.inf)
            pos = ad > 0
            if pos.any():
                max_rel = max(max_rel, float(rd[pos].max()))
        integral = dtypes is not None and dtypes.get(name) in ("i32", "bool")
        good = (a == b) if integral else ((ad <= abs_tol) | (rd <= rel_tol))
        if not good.all() and ok:
            i = int(np.argmin(good))
            ok = False
            msg = "mismatch on %s[%d]: got %.9g, want %.9g" % (name, i, a[i], b[i])
    return CompareReport(ok, max_abs, max_rel, msg)


def algorithmic_bytes(g: Graph, patterns) -> int:
    """per kernel, unique external (non-constant) inputs read
    once + tensors leaving the kernel written once; summed over kernels."""
    cons = {n.id: [] for n in g.nodes}
    for n in g.nodes:
        for o in set(n.operands):
            cons[o].append(n.id)
    total = 0
    for verts in patterns:
        vs = set(verts)
        ins = {o for v in vs for o in g.nodes[v].operands
               if o not in vs and g.nodes[o].kind != "constant"}
        outs = {v for v in vs if v in g.outputs or any(c not in vs for c in cons[v])}
        for t in ins | outs:
            n = g.nodes[t]
            total += int(np.prod(n.dims) if n.dims else 1) * DTYPE_BYTES[n.dtype]
    return total
