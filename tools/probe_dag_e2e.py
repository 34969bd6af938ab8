"""Probe (diagnostics): plan-graph DAG capture vs linear chain on the
launch-bound configs, and pipelined host execution vs chunk count."""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2009_10924_b200 import stitch, shard

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2009_10924_b200", "graphs")
txt = lambda n: open(os.path.join(G, n + ".graph")).read()

for name in sys.argv[1:] or ["dien_T10", "dien_T20", "dien_cut_T10", "bert_layer", "bert_cut"]:
    for dag in ("1", "0"):
        os.environ["STITCH_DAG"] = dag
        g = stitch.Graph(txt(name))
        ex = stitch.Executor(stitch.Plan(g, "b200"))
        ex.upload(stitch.random_inputs(g, 1))
        per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
        sets = min(64, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
        us1, _ = ex.time(iters=100, warmup=10, sets=sets)
        usb = ex.time_batched(steps=64, warmup=8, sets=sets, steps_per_graph=8)
        print(json.dumps({"graph": name, "dag": dag, "kernels": ex.num_kernels, "us_one_launch": round(us1, 2),
                          "us_batched8": round(usb, 2)}), flush=True)
os.environ["STITCH_DAG"] = "1"

text = txt("attn_softmax")
g = stitch.Graph(text)
inputs = stitch.random_inputs(g, 1)
pin_in = {t.name: torch.from_numpy(inputs[t.name]).pin_memory().numpy() for t in g.params}
pin_out = {t.name: torch.empty(t.dims, dtype=torch.float32).pin_memory().numpy() for t in g.outputs}
nbytes = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
ex = stitch.Executor(stitch.Plan(g, "b200"))
ex.run(pin_in, out=pin_out)
t0 = time.perf_counter()
for _ in range(20):
    ex.run(pin_in, out=pin_out)
s = (time.perf_counter() - t0) / 20
print(json.dumps({"e2e": "plain", "us": round(s * 1e6, 1), "GBps": round(nbytes / s / 1e9, 2)}), flush=True)
for n in (2, 4, 8, 16, 32):
    cx = stitch.ChunkedExecutor(text, shard.RULES["attn_softmax"], n)
    cx.run(pin_in, out=pin_out)
    t0 = time.perf_counter()
    for _ in range(20):
        cx.run(pin_in, out=pin_out)
    s = (time.perf_counter() - t0) / 20
    print(json.dumps({"e2e": "chunked", "nchunks": n, "us": round(s * 1e6, 1), "GBps": round(nbytes / s / 1e9, 2)}),
          flush=True)
