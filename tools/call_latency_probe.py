"""Where a single subgraph call's time goes, per config (JSON lines):

  us_batched      64 steps per graph launch, PDL between steps (bench `us`)
  us_serial       64 steps per graph launch, STITCH_PDL=0: every step's
                  kernels start after the previous step completed -- the
                  kernel's own fill / stream / drain, no launch latency
  us_one_launch   one graph launch per step, back to back (host rate bound)
  us_one_call     one graph launch queued behind a spinning warp, events
                  around it: launch-to-completion on an idle device

plus the same four for a 4-element graph (the fixed cost of a call).

    python tools/call_latency_probe.py [graph ...]
"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch  # noqa: E402

TINY = "x = parameter : f32[4]\ny = parameter : f32[4]\nz = add(x, y)\noutput z\n"


def measure(text, label):
    g = stitch.Graph(text)
    plan = stitch.Plan(g, "b200")
    per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
    sets = min(128, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
    rec = {"graph": label, "bytes": per_set}
    for pdl in ("1", "0"):
        os.environ["STITCH_PDL"] = pdl
        ex = stitch.Executor(plan)
        ex.upload(stitch.random_inputs(g, 1))
        us = ex.time_batched(steps=512, warmup=64, sets=sets, steps_per_graph=64)
        if pdl == "1":
            rec["us_batched"] = round(us, 3)
            rec["us_one_launch"] = round(ex.time(iters=200, warmup=20, sets=sets)[0], 3)
            rec["us_one_call"] = round(ex.time_call(iters=200, warmup=20, sets=sets)[0], 3)
        else:
            rec["us_serial"] = round(us, 3)
            rec["us_one_call_nopdl"] = round(ex.time_call(iters=200, warmup=20, sets=sets)[0], 3)
        del ex
    os.environ.pop("STITCH_PDL", None)
    print(json.dumps(rec), flush=True)


measure(TINY, "tiny_4")
for name in sys.argv[1:] or ["ln_4096x768", "bert_resln", "attn_softmax", "bert_gelu", "colreduce", "bert_cut"]:
    measure(open(os.path.join(stitch.GRAPHS, name + ".graph")).read(), name)
