"""e2e of the C3 headline graph (bert_cut) through stc_exec_run_host_chunked
for 2..16 chunks, with the per-chunk copy/compute timeline of one call
(STITCH_CHUNK_TRACE=1 on stderr) -- where a host-buffer call's time goes.

    python tools/e2e_cut_probe.py [graph]
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2009_10924_b200 import shard, stitch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bert_cut"
text = open(os.path.join(stitch.GRAPHS, name + ".graph")).read()
g = stitch.Graph(text)
inputs = stitch.random_inputs(g, 1)
pin_in = {t.name: torch.from_numpy(inputs[t.name]).pin_memory().numpy() for t in g.params}
pin_out = {t.name: torch.empty(t.dims, dtype=torch.float32).pin_memory().numpy() for t in g.outputs}
nbytes = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
for n in (2, 4, 8, 16):
    cx = stitch.ChunkedExecutor(text, shard.RULES[name], n)
    for _ in range(3):
        cx.run(pin_in, out=pin_out)
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        cx.run(pin_in, out=pin_out)
    s = (time.perf_counter() - t0) / reps
    print(json.dumps({"graph": name, "chunks": n, "us": round(s * 1e6, 1), "GBps": round(nbytes / s / 1e9, 2)}), flush=True)
    os.environ["STITCH_CHUNK_TRACE"] = "1"
    cx.run(pin_in, out=pin_out)
    os.environ["STITCH_CHUNK_TRACE"] = "0"
