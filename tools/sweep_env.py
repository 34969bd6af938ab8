"""Sweep codegen knobs (env vars) for one graph: us per subgraph (batched
graph replays, inputs rotated past L2), us_serial (the same with STITCH_PDL=0:
no cross-step overlap), us with one graph launch per step
(host submission rate included), us of one call on the device
(replay queued behind a spinning warp; plus per-kernel event times), grid, block.

    python tools/sweep_env.py <graph> 'VAR=a,b VAR2=c,d' ...
"""
import itertools, json, math, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("SWEEP_CHILD"):
    from paper_2009_10924_b200 import stitch
    name = sys.argv[1]
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    ex = stitch.Executor(stitch.Plan(g, os.environ.get("SWEEP_CFG", "b200")))
    ex.upload(stitch.random_inputs(g, 1))
    d = ex.describe()
    per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
    sets = min(128, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
    us = ex.time_batched(steps=256, warmup=32, sets=sets, steps_per_graph=16)
    us1, _ = ex.time(iters=200, warmup=20, sets=sets)
    usc, kus = ex.time_call(iters=200, warmup=20, sets=sets, per_kernel=True)
    del ex
    # serial: the same batched replay with STITCH_PDL=0 -- each step starts
    # after the previous completed (fill + stream + drain, no launch latency)
    os.environ["STITCH_PDL"] = "0"
    exs = stitch.Executor(stitch.Plan(g, os.environ.get("SWEEP_CFG", "b200")))
    exs.upload(stitch.random_inputs(g, 1))
    uss = exs.time_batched(steps=256, warmup=32, sets=sets, steps_per_graph=16)
    print(json.dumps({"us": round(us, 3), "GBps": round(sum(k["bytes"] for k in d) / us / 1e3, 1),
                      "us_serial": round(uss, 3), "us_one_launch": round(us1, 3), "us_one_call": round(usc, 3),
                      "kernel_us_one_call": [round(x, 3) for x in kus],
                      "grid": [k["grid"] for k in d], "block": [k["block"] for k in d]}))
    sys.exit(0)
name = sys.argv[1]
axes = []
for spec in sys.argv[2:]:
    for part in spec.split():
        k, vals = part.split("=")
        axes.append([(k, v) for v in vals.split(",")])
for combo in itertools.product(*axes) if axes else [()]:
    env = dict(os.environ, SWEEP_CHILD="1", **dict(combo))
    r = subprocess.run([sys.executable, __file__, name], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-300:]
    print(json.dumps({"graph": name, "env": dict(combo)}), line, flush=True)
