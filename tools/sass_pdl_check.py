"""PDL ordering check on the SASS of a plan's module (no GPU needed).

Under programmatic dependent launch every kernel must not write global memory
before griddepcontrol.wait (SASS ACQBULK) -- the previous kernel may still be
reading what it overwrites -- and must not read a kernel-produced tensor
before it.  The second is enforced at the source level (kernel-produced
tensors are read with coherent loads, which ptxas keeps below the wait;
tests/test_abi.py); this tool checks the first, and reports how many
non-coherent (parameter) loads each kernel issues ahead of its wait.

    python tools/sass_pdl_check.py dien_T10 bert_layer ...
"""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def check(name, cfg="b200", plan=None):
    from paper_2009_10924_b200 import stitch
    if plan is None:
        plan = stitch.Plan(stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph")), cfg)
    src, _ = plan.codegen()
    key = stitch.compile_cuda(src)
    cache = os.environ.get("STITCH_CACHE_DIR", os.path.join(os.path.dirname(stitch.__file__), "lib", "cubin_cache"))
    sass = subprocess.run(["cuobjdump", "-sass", os.path.join(cache, key + ".cubin")], capture_output=True,
                          text=True, check=True).stdout
    out = {}
    fn = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            out[fn] = {"writes_before_wait": 0, "param_loads_before_wait": 0, "coherent_loads_before_wait": 0,
                       "waited": False}
            continue
        if fn is None:
            continue
        r = out[fn]
        if "ACQBULK" in line:
            r["waited"] = True
        elif not r["waited"]:
            if re.search(r"\b(STG|RED|ATOM)\b", line):
                r["writes_before_wait"] += 1
            elif "LDG" in line:
                r["param_loads_before_wait" if "CONSTANT" in line else "coherent_loads_before_wait"] += 1
    return out


if __name__ == "__main__":
    import json
    for n in sys.argv[1:]:
        for fn, r in check(n).items():
            print(json.dumps({"graph": n, "kernel": fn, **r}))
