"""Persistent template A/B (diagnostics): launch-bound plans run as one
cooperative launch (STITCH_PERSIST=1) vs the per-unit CUDA Graph; outputs
compared bitwise, then timed (batched replays, inputs rotated past L2).

    python tools/persist_probe.py dien_T10 dien_T20
"""
import json, math, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("PERSIST_TRACE"):  # unit timeline of one persistent replay
    os.environ["STITCH_TRACE"] = "1"
    os.environ["STITCH_PERSIST"] = "1"
    from paper_2009_10924_b200 import stitch
    name = sys.argv[1]
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    src, units = stitch.Plan(g, "b200").codegen()  # unit names come from the source comments
    names = [l.split(": ", 1)[1] for l in src.splitlines() if l.startswith("  // unit ")]
    ex = stitch.Executor(stitch.Plan(g, "b200"))
    ex.upload(stitch.random_inputs(g, 1))
    for _ in range(3):
        t = ex.trace()
    print("kernel %.2f .. %.2f us" % t[0])
    for u, (a, b) in enumerate(t[1:]):
        prev = t[u][1] if u else t[0][0]
        print("%-60s ready %7.2f  done %7.2f  dur %5.2f" % (names[u][:60], a, b, b - a))
    sys.exit(0)
if os.environ.get("PERSIST_CHILD"):
    import numpy as np
    from paper_2009_10924_b200 import stitch
    name = sys.argv[1]
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    ex = stitch.Executor(stitch.Plan(g, "b200"))
    inputs = stitch.random_inputs(g, 1)
    out = ex.run(inputs)
    np.savez("/tmp/persist_%s_%s.npz" % (name, os.environ.get("STITCH_PERSIST", "0")), **out)
    per_set = sum(t.nbytes for t in g.params) + sum(t.nbytes for t in g.outputs)
    sets = min(128, max(2, math.ceil(8 * 126 * 2**20 / per_set)))
    if os.environ.get("PERSIST_SETS"):  # diagnostics: warm (few, L2-resident) buffer sets
        sets = int(os.environ["PERSIST_SETS"])
    us = ex.time_batched(steps=256, warmup=32, sets=sets, steps_per_graph=16)
    us1 = ex.time(iters=100, warmup=10, sets=sets)[0]
    d = ex.describe()
    print(json.dumps({"us": round(us, 3), "us_one_launch": round(us1, 3), "launches": len(d),
                      "templates": sorted({k["template"] for k in d})}))
    sys.exit(0)
import numpy as np
for name in sys.argv[1:]:
    res = {}
    for mode in ("0", "1"):
        env = dict(os.environ, PERSIST_CHILD="1", STITCH_PERSIST=mode)
        r = subprocess.run(["timeout", "120", sys.executable, __file__, name], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-400:]
        res[mode] = line
        print(json.dumps({"graph": name, "STITCH_PERSIST": mode}), line, flush=True)
    try:
        a = np.load("/tmp/persist_%s_0.npz" % name)
        b = np.load("/tmp/persist_%s_1.npz" % name)
        print(json.dumps({"graph": name, "bitwise_equal": all(np.array_equal(a[k], b[k]) for k in a.files)}), flush=True)
    except Exception as e:
        print(json.dumps({"graph": name, "compare_error": str(e)[:200]}), flush=True)
