"""Plans under the parity B200 profile (b200_device.cfg: device shape only)
vs the recalibrated cost model (b200.cfg): planning time, kernels, bytes,
measured us per subgraph (batched graph replays, inputs rotated past L2).

    python tools/compare_cfgs.py [cfg_a] [cfg_b] [graph ...]
"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

GRAPHS = ["ln_4096x768", "ln2pass_4096x768", "attn_softmax", "colreduce", "bert_gelu", "bert_resln", "bert_cut",
          "bert_layer", "dien_T10", "dien_cut_T10"]
args = sys.argv[1:]
cfgs = [a for a in args if a.startswith("b200") or a.endswith(".cfg") or a == "v100"][:2] or ["b200", "b200cal"]
graphs = [a for a in args if a not in cfgs] or GRAPHS
gpu = os.environ.get("NO_GPU", "0") != "1"
for name in graphs:
    for cfg in cfgs:
        g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
        t0 = time.perf_counter()
        plan = stitch.Plan(g, cfg)
        plan_s = time.perf_counter() - t0
        j = json.loads(plan.json())
        rec = {"graph": name, "cfg": cfg, "plan_s": round(plan_s, 2), "stitched_kernels": j["stitched_kernels"],
               "baseline_kernels": j["baseline_kernels"],
               "patterns": [len(p["vertices"]) for p in j["patterns"]]}
        if gpu:
            ex = stitch.Executor(plan)
            ex.upload(stitch.random_inputs(g, 1))
            d = ex.describe()
            per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
            sets = min(128, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
            rec["launched"] = len(d)
            rec["bytes"] = sum(k["bytes"] for k in d)
            rec["us"] = round(ex.time_batched(steps=128, warmup=16, sets=sets, steps_per_graph=8), 2)
        print(json.dumps(rec), flush=True)
