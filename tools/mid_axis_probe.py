import sys, math, json; sys.path.insert(0,'.')
from paper_2009_10924_b200 import stitch
cases = {
 "mid_axis_sum [64,512,256] axes=1": "x = parameter : f32[64,512,256]\ne = exp(x)\ns = reduce_sum(e) axes=1\ny = mul(s, s)\noutput y\n",
 "outer_inner_max [64,512,256] axes=[0,2]": "x = parameter : f32[64,512,256]\nm = reduce_max(x) axes=[0,2]\ny = mul(m, m)\noutput y\n",
}
for n, txt in cases.items():
    g = stitch.Graph(txt)
    for mode in ("stitched", "program"):
        ex = stitch.Executor(stitch.Plan(g, "b200"), mode=mode)
        ex.upload(stitch.random_inputs(g, 1))
        d = ex.describe()
        per = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
        us = ex.time_batched(steps=64, warmup=8, sets=min(64, max(2, math.ceil(8*126*2**20/per))), steps_per_graph=8)
        print(json.dumps({"graph": n, "mode": mode, "templates": [k["template"] for k in d], "us": round(us, 2),
                          "GBps": round(sum(k["bytes"] for k in d) / us / 1e3, 1)}))
