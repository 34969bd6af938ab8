"""e2e chunk-shape sweep (diagnostics): attn_softmax from pinned host memory
through ChunkedExecutor with several batch splits; bitwise check vs the
device-resident run."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2009_10924_b200 import stitch, shard

name = "attn_softmax"
text = open(os.path.join(stitch.GRAPHS, name + ".graph")).read()
g = stitch.Graph(text)
inputs = stitch.random_inputs(g, 1)
pin_in = {t.name: torch.from_numpy(inputs[t.name]).pin_memory().numpy() for t in g.params}
pin_out = {t.name: torch.empty(t.dims, dtype=torch.float32).pin_memory().numpy() for t in g.outputs}
nbytes = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
ref = {k: v.copy() for k, v in stitch.Executor(stitch.Plan(g, "b200")).run(inputs).items()}
for chunks in (4, [11, 11, 10], [7, 7, 6, 6, 6], [6, 6, 5, 5, 5, 5], [4, 8, 8, 8, 4], [8, 8, 8, 6, 2], [3, 9, 10, 10]):
    ce = stitch.ChunkedExecutor(text, shard.RULES[name], chunks)
    ce.run(pin_in, out=pin_out)
    reps = 30
    t0 = time.perf_counter()
    for _ in range(reps):
        ce.run(pin_in, out=pin_out)
    us = (time.perf_counter() - t0) / reps * 1e6
    ok = all(np.array_equal(pin_out[k], ref[k]) for k in ref)
    print(json.dumps({"graph": name, "chunks": chunks, "us": round(us, 1), "GBps": round(nbytes / us / 1e3, 2), "bitwise_equal": ok}), flush=True)
