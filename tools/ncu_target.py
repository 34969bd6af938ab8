"""Small driver for ncu captures: plan each named config graph, upload
inputs, replay the plan a few times (kernel names k<i>_<producer>)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

names = sys.argv[1:] or ["bert_cut", "ln_4096x768", "attn_softmax", "colreduce", "bert_gelu", "bert_resln", "ln2pass_4096x768"]
for name in names:
    g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
    ex = stitch.Executor(stitch.Plan(g, "b200"), graph=False)
    ex.upload(stitch.random_inputs(g, 1))
    for _ in range(int(os.environ.get("REPS", "3"))):
        ex.launch()
    ex.sync()
    print(name, [k["name"] for k in ex.describe()], flush=True)
