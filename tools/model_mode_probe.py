"""Model mode: the BERT FFN layer (A.4) with its two
GEMMs as cuBLASLt between the stitched memory-intensive kernels, one CUDA
Graph.  Prints us per layer and the per-kernel split (GEMM vs stitched)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

name = sys.argv[1] if len(sys.argv) > 1 else "bert_layer"
for prec in os.environ.get("PROBE_PRECS", "tf32,fp32").split(","):
    os.environ["STITCH_GEMM_FP32"] = "1" if prec == "fp32" else "0"
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    ex = stitch.Executor(stitch.Plan(g, "b200"), gemm=True)
    ex.upload(stitch.random_inputs(g, 1))
    d = ex.describe()
    per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
    sets = min(64, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
    us_b = ex.time_batched(steps=64, warmup=8, sets=sets, steps_per_graph=8)
    us1, kus = ex.time(iters=50, warmup=5, sets=sets, per_kernel=True)
    gemm_us = sum(u for k, u in zip(d, kus) if k["template"].startswith("gemm"))
    flops = sum(0 for _ in d)
    env = {k: v for k, v in os.environ.items() if k.startswith("STITCH_GEMM_")}
    print(json.dumps({"graph": name, "gemm": prec, "env": env, "kernels": len(d), "us_per_layer_batched": round(us_b, 2),
                      "us_per_layer_one_launch": round(us1, 2), "gemm_us_events": round(gemm_us, 2),
                      "stitched_us_events": round(sum(kus) - gemm_us, 2),
                      "per_kernel": [[k["name"], k["template"], round(u, 2)] for k, u in zip(d, kus)]}), flush=True)
