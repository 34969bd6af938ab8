"""In-graph kernel timeline (diagnostics): one replay of a plan's CUDA Graph
with %globaltimer stamps at first-CTA entry / last-CTA exit of every kernel.

    python tools/trace_timeline.py dien_T10 [--linear]
"""
import json, os, sys
os.environ["STITCH_TRACE"] = "1"
if "--linear" in sys.argv:
    os.environ["STITCH_DAG"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

name = [a for a in sys.argv[1:] if not a.startswith("--")][0]
g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
ex = stitch.Executor(stitch.Plan(g, "b200"))
ex.upload(stitch.random_inputs(g, 1))
for _ in range(3):
    t = ex.trace()
d = ex.describe()
span = max(e for _, e in t)
busy = sum(e - s for s, e in t)
print(json.dumps({"graph": name, "kernels": len(d), "span_us": round(span, 2), "sum_kernel_us": round(busy, 2)}))
prod = {}
for i, k in enumerate(d):
    for o in k["outputs"]:
        prod[o] = i
for i, (k, (s, e)) in sorted(enumerate(zip(d, t)), key=lambda x: x[1][1][0]):
    deps = sorted({prod[x] for x in k["inputs"] if x in prod})
    ready = max([t[j][1] for j in deps], default=0.0)
    print("%-12s %-10s grid %5d  start %8.2f  end %8.2f  dur %6.2f  deps-ready %8.2f  gap %6.2f  deps %s"
          % (k["name"], k["template"][:10], k["grid"], s, e, e - s, ready, s - ready, [d[j]["name"] for j in deps]))
