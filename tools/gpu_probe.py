"""GPU diagnostics: plan + compile + time every config graph (not the bench)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

names = sys.argv[1:] or ["ln_4096x768", "ln2pass_4096x768", "attn_softmax", "colreduce", "bert_gelu",
                         "bert_resln", "dien_T10", "dien_cut_T10", "bert_layer"]
for name in names:
    t0 = time.time()
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    plan = stitch.Plan(g, "b200")
    t1 = time.time()
    for mode in ("stitched", "program", "unfused"):
        try:
            ex = stitch.Executor(plan, mode=mode)
            t2 = time.time()
            ex.upload(stitch.random_inputs(g, 1))
            desc = ex.describe()
            total_bytes = sum(k["bytes"] for k in desc)
            per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
            sets = max(1, int(3 * 126e6 / max(per_set, 1)) + 1)
            sets = min(sets, 64)
            us, kus = ex.time(iters=50, warmup=5, sets=sets, per_kernel=True)
            top = sorted(zip(kus, desc), key=lambda x: -x[0])[:3]
            print(json.dumps({"graph": name, "mode": mode, "kernels": len(desc), "us": round(us, 2),
                              "GBps": round(total_bytes / us / 1e3, 1), "bytes": total_bytes, "sets": sets,
                              "plan_s": round(t1 - t0, 2), "compile_s": round(t2 - t1, 2),
                              "top": [(round(u, 2), d["name"], d["template"], d["grid"], d["block"],
                                       round(d["bytes"] / max(u, 1e-9) / 1e3, 1)) for u, d in top]}), flush=True)
        except Exception as e:
            print(json.dumps({"graph": name, "mode": mode, "error": str(e)[:3000]}), flush=True)
