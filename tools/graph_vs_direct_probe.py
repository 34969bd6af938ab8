"""One-call latency through a CUDA Graph replay vs direct kernel launches
(Executor(graph=False)) for single- and multi-kernel plans (JSON lines).

    python tools/graph_vs_direct_probe.py [graph ...]
"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch  # noqa: E402

TINY = "x = parameter : f32[4]\ny = parameter : f32[4]\nz = add(x, y)\noutput z\n"
names = sys.argv[1:] or ["tiny_4", "ln_4096x768", "bert_cut", "bert_layer", "dien_T10"]
for name in names:
    text = TINY if name == "tiny_4" else open(os.path.join(stitch.GRAPHS, name + ".graph")).read()
    g = stitch.Graph(text)
    plan = stitch.Plan(g, "b200")
    per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
    sets = min(128, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
    rec = {"graph": name}
    for graph in (True, False):
        ex = stitch.Executor(plan, graph=graph)
        ex.upload(stitch.random_inputs(g, 1))
        tag = "graph" if graph else "direct"
        rec["launches_" + tag] = ex.num_kernels
        rec["us_one_call_" + tag] = round(ex.time_call(iters=200, warmup=20, sets=sets)[0], 3)
        rec["us_one_launch_" + tag] = round(ex.time(iters=200, warmup=20, sets=sets)[0], 3)
        del ex
    print(json.dumps(rec), flush=True)
