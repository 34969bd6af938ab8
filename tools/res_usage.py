"""Registers / spill / shared memory of every kernel a plan generates (no GPU
needed): NVRTC-compiles the plan's module through the cubin cache and reads
`cuobjdump -res-usage`.

    python tools/res_usage.py <graph> [<graph> ...]    (env knobs apply)
"""
import json, os, re, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

for name in sys.argv[1:]:
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    src, desc = stitch.Plan(g, os.environ.get("RES_CFG", "b200")).codegen()
    key = stitch.compile_cuda(src)
    path = os.path.join(stitch.lib().stc_cache_dir().decode(), key + ".cubin")
    out = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
    res = {}
    for fn, body in re.findall(r"Function (\w+):\s*\n\s*(REG:.*)", out):
        res[fn] = dict((k, int(v)) for k, v in re.findall(r"(\w+):(\d+)", body))
    for k in desc:
        r = res.get(k["symbol"], {})
        print(json.dumps({"graph": name, "kernel": k["name"], "template": k["template"], "grid": k["grid"],
                          "block": k["block"], "REG": r.get("REG"), "STACK": r.get("STACK"),
                          "LOCAL": r.get("LOCAL"), "SHARED": r.get("SHARED")}))
