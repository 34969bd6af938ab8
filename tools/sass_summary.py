"""SASS evidence per stitching template (no GPU needed): compiles each plan's
module through the NVRTC cache and counts the instructions that show what
the kernel does on sm_100a -- 128-bit global loads/stores (LDG.E.128 /
STG.E.128, .EF = evict-first streaming), MUFU.EX2 (exp), SHFL (warp
reductions), DADD (f64 folds), cluster barriers / DSMEM (UCGABAR, mapa'd
LDS), bulk copies (UBLKCP, TMA path), PDL (ACQBULK / griddepcontrol).

    python tools/sass_summary.py > profiles/r01/sass_summary.json
"""
import collections, json, os, re, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch
from tests.test_gpu_exec import _softmax_text  # noqa: E402

CASES = {name: open(os.path.join(stitch.GRAPHS, name + ".graph")).read()
         for name in ["ln_4096x768", "attn_softmax", "bert_gelu", "bert_resln", "colreduce", "bert_cut", "dien_T10"]}
CASES["softmax_8x65536 (regional-cluster)"] = _softmax_text(8, 65536)
out = {}
for name, text in CASES.items():
    plan = stitch.Plan(stitch.Graph(text), "b200")
    src, desc = plan.codegen()
    key = stitch.compile_cuda(src)
    path = os.path.join(stitch.lib().stc_cache_dir().decode(), key + ".cubin")
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    ops = collections.Counter()
    for line in sass.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            ops[m.group(1)] += 1
    rec = {"kernels": [(k["name"], k["template"]) for k in desc][:6], "instructions": sum(ops.values())}
    cats = {
        "LDG 128-bit": lambda k: k.startswith("LDG") and ".128" in k,
        "LDG 64-bit": lambda k: k.startswith("LDG") and ".64" in k,
        "STG 128-bit": lambda k: k.startswith("STG") and ".128" in k,
        "STG evict-first (.EF)": lambda k: k.startswith("STG") and ".EF" in k,
        "MUFU.EX2": lambda k: k.startswith("MUFU.EX2"),
        "MUFU.RCP": lambda k: k.startswith("MUFU.RCP"),
        "SHFL": lambda k: k.startswith("SHFL"),
        "DADD": lambda k: k.startswith("DADD"),
        "BAR.SYNC": lambda k: k.startswith("BAR.SYNC"),
        "cluster barrier (UCGABAR)": lambda k: k.startswith("UCGABAR"),
        "DSMEM load (LD via mapa)": lambda k: k.startswith("LD.E"),
        "bulk copy (UBLKCP)": lambda k: k.startswith("UBLKCP"),
        "PDL wait (ACQBULK)": lambda k: k.startswith("ACQBULK"),
        "atomics (ATOMG/RED)": lambda k: k.startswith("ATOMG") or k.startswith("RED"),
    }
    for label, pred in cats.items():
        n = sum(v for k, v in ops.items() if pred(k))
        if n:
            rec[label] = n
    out[name] = rec
print(json.dumps(out, indent=1))
