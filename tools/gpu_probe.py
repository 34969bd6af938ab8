"""GPU diagnostics (not the bench): for each config graph, step time with one
graph launch per step vs B steps per graph, over >= 8x L2 of rotating sets."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch  # noqa: E402

L2 = 126 * 1024 * 1024
names = sys.argv[1:] or ["ln_4096x768", "ln2pass_4096x768", "attn_softmax", "colreduce", "bert_gelu",
                         "bert_resln", "dien_T10", "bert_layer"]
for name in names:
    t0 = time.time()
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    plan = stitch.Plan(g, "b200")
    t1 = time.time()
    try:
        ex = stitch.Executor(plan)
        t2 = time.time()
        ex.upload(stitch.random_inputs(g, 1))
        desc = ex.describe()
        alg = sum(k["bytes"] for k in desc)
        per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
        sets = min(256, max(2, math.ceil(8 * L2 / per_set)))
        us1, kus = ex.time(iters=200, warmup=20, sets=sets, per_kernel=True)
        rec = {"graph": name, "kernels": len(desc), "bytes": alg, "sets": sets, "us_step": round(us1, 3),
               "GBps": round(alg / us1 / 1e3, 1), "plan_s": round(t1 - t0, 2), "compile_s": round(t2 - t1, 2)}
        for b in (4, 16):
            usb = ex.time_batched(steps=max(256, 8 * b), warmup=2 * b, sets=sets, steps_per_graph=b)
            rec["us_step_B%d" % b] = round(usb, 3)
            rec["GBps_B%d" % b] = round(alg / usb / 1e3, 1)
        top = sorted(zip(kus, desc), key=lambda x: -x[0])[:2]
        rec["top_event_us"] = [(round(u, 2), d["name"], d["template"], d["grid"], d["block"]) for u, d in top]
        print(json.dumps(rec), flush=True)
    except Exception as e:
        print(json.dumps({"graph": name, "error": str(e)[:2000]}), flush=True)
