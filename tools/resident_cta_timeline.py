"""Per-CTA step timeline of one resident-kernel replay (STITCH_TRACE=1 +
STITCH_TRACE_CTAS=16): for every step, each CTA's own duration (end - begin,
min / median / max over the cluster) and the spread of the CTAs' begin times.

    python tools/resident_cta_timeline.py dien_T10
"""
import os, statistics, sys
os.environ["STITCH_TRACE"] = "1"
os.environ["STITCH_RESIDENT"] = "1"
os.environ.setdefault("STITCH_TRACE_CTAS", "16")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_10924_b200 import stitch  # noqa: E402

C = int(os.environ["STITCH_TRACE_CTAS"])
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
slots = len(t) // C
print("kernel: CTA 0 %.2f .. %.2f us, %s" % (t[0][0], t[0][1], ex.describe()[0]["template"]))
print("step   begin-spread  dur min / med / max (us)   label")
tot_med = 0.0
for k in range(1, slots):
    rows = [t[k * C + c] for c in range(C) if t[k * C + c][1] >= 0]
    if not rows:
        continue
    durs = sorted(b - a for a, b in rows)
    begins = [a for a, _ in rows]
    tot_med += statistics.median(durs)
    print("%4d   %6.2f        %5.2f / %5.2f / %5.2f       %s" % (k - 1, max(begins) - min(begins), durs[0],
                                                            statistics.median(durs), durs[-1],
                                                            labels[k - 1][:70] if k - 1 < len(labels) else ""))
print("sum of median step durations: %.2f us" % tot_med)
