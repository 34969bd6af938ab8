"""Parity plan vs NON-PARITY refined plan (stc_plan_refine, SURVEY §8f item
1): kernels, bytes, us per subgraph, and refined outputs vs the oracle."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2009_10924_b200 import stitch
from oracle import numpy_oracle as no

cases = [("bert_layer", "b200"), ("bert_layer", "v100"), ("bert_cut", "v100"), ("bert_gelu", "v100"),
         ("dien_T10", "b200"), ("dien_T20", "b200")]
for name, cfg in cases:
    text = open(os.path.join(stitch.GRAPHS, name + ".graph")).read()
    g = stitch.Graph(text)
    inputs = stitch.random_inputs(g, 1)
    rec = {"graph": name, "cfg": cfg}
    for mode in ("parity", "refined"):
        plan = stitch.Plan(g, cfg)
        if mode == "refined":
            t0 = time.perf_counter()
            rec["merges"], saved = plan.refine()
            rec["refine_s"] = round(time.perf_counter() - t0, 2)
        ex = stitch.Executor(plan)
        d = ex.describe()
        got = ex.run(inputs)
        per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
        sets = min(64, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
        us = ex.time_batched(steps=64, warmup=8, sets=sets, steps_per_graph=8)
        rec[mode] = {"kernels": len(d), "bytes": sum(k["bytes"] for k in d), "us": round(us, 2)}
        if mode == "refined":
            og = no.parse_graph(text)
            want = no.eval_reference(og, {k: v.astype(np.float64) for k, v in inputs.items()})
            rep = stitch.compare(got, want, 1e-4, 1e-5)
            rec["refined_vs_oracle"] = {"pass": rep["pass"], "max_rel": rep["max_rel"]}
    print(json.dumps(rec), flush=True)
