"""Step timeline of one resident-kernel replay (diagnostics, STITCH_TRACE):
first CTA entering / last CTA leaving each step of the cluster kernel.

    python tools/resident_timeline.py dien_T10
"""
import os, sys
os.environ["STITCH_TRACE"] = "1"
os.environ["STITCH_RESIDENT"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch

name = sys.argv[1]
g = stitch.Graph.from_file(os.path.join(stitch.GRAPHS, name + ".graph"))
plan = stitch.Plan(g, "b200")
# step labels from the straight-line source (the recurrent-step loop drops
# them; its steps keep their trace slot numbers)
_loop = os.environ.get("STITCH_RESIDENT_LOOP")
os.environ["STITCH_RESIDENT_LOOP"] = "0"
src, _ = plan.codegen()
if _loop is None:
    os.environ.pop("STITCH_RESIDENT_LOOP")
else:
    os.environ["STITCH_RESIDENT_LOOP"] = _loop
labels = [l.strip() for l in src.splitlines() if l.startswith("  // unit ") or l.startswith("  {  // placeholder group")]
ex = stitch.Executor(plan)
ex.upload(stitch.random_inputs(g, 1))
for _ in range(3):
    t = ex.trace()
print("kernel %.2f .. %.2f us, %s" % (t[0][0], t[0][1], ex.describe()[0]["template"]))
for s, (a, b) in enumerate(t[1:]):
    print("step %3d  begin %7.2f  end %7.2f  dur %5.2f  %s" % (s, a, b, b - a, labels[s][:90] if s < len(labels) else ""))
