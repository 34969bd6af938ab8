"""Bit-exact plan parity with the reference planner (SURVEY.md §8a A1-A15,
A21): same graph + same cfg -> byte-identical plan.json (nlohmann 3.11.3
dump(2)), identical .stitch program text for every kernel (the emitter's
histogram and liveness decide plan choice), identical serialize_graph text.
Goldens were produced by the unmodified reference (tests/golden/make_golden.py)."""
import hashlib
import json
import os

import pytest

from tests.conftest import GOLD, cached_plan, golden_plan, graph_text

PLAN_FILES = sorted(f[:-5] for f in os.listdir(os.path.join(GOLD, "plans")) if f.endswith(".json"))
SLOW = {"bert_cut", "dien_T20"}  # reference planner: 172 s / 14 s


def _stitch():
    from paper_2009_10924_b200 import stitch
    return stitch


@pytest.mark.parametrize("case", [c for c in PLAN_FILES if c.split("__")[0].split("@")[0] not in SLOW])
def test_plan_bytes(case):
    stitch = _stitch()
    name, cfg = case.split("__")
    rec = golden_plan(name, cfg)
    # per-shard plans carry their shard graph text
    plan = cached_plan(rec["graph_text"] if "graph_text" in rec else graph_text(name), cfg)
    assert plan.graph.serialize() == rec["serialized"]
    pj = plan.json()
    assert pj == rec["plan_json"]
    keys = [p["key"] for p in json.loads(pj)["patterns"]]
    for i, k in enumerate(keys):
        assert plan.kernel_text(i) == rec["programs"][k], (case, k)
    summary = rec["summary"].split()
    st = plan.stats()
    assert st["stitched_kernels"] == int(summary[1]) and st["baseline_kernels"] == int(summary[3])
    assert st["delta_evaluate_calls"] == int(summary[5])


@pytest.mark.slow
@pytest.mark.parametrize("case", [c for c in PLAN_FILES if c.split("__")[0].split("@")[0] in SLOW])
def test_plan_bytes_slow(case):
    test_plan_bytes(case)


def test_random_graphs():
    """100 random graphs x 2 cfgs; planned on host threads (ctypes releases
    the GIL and every Plan owns its CostModels, as in the reference)"""
    from concurrent.futures import ThreadPoolExecutor
    stitch = _stitch()
    with open(os.path.join(GOLD, "random_plans.json")) as f:
        rnd = json.load(f)
    assert len(rnd) == 100

    def check(item):
        seed, entry, cfg = item
        g = stitch.Graph(entry["graph"])
        plan = stitch.Plan(g, cfg)
        pj = plan.json()
        assert pj == entry[cfg]["plan_json"], (seed, cfg)
        keys = [p["key"] for p in json.loads(pj)["patterns"]]
        for i, k in enumerate(keys):
            h = hashlib.sha256(plan.kernel_text(i).encode()).hexdigest()
            assert h == entry[cfg]["programs_sha"][k], (seed, cfg, k)

    work = [(seed, entry, cfg) for seed, entry in rnd.items() for cfg in ("v100", "b200")]
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
        list(pool.map(check, work))


def test_plan_kernel_infeasible_and_explicit_patterns():
    stitch = _stitch()
    g = stitch.Graph(graph_text("layernorm"))
    # parameters are not fusable -> plan_kernel infeasible (planner.cpp:1040-1041)
    assert stitch.plan_kernel(g, [0, 7]) is None
    txt = stitch.plan_kernel(g, [7])  # s1 alone
    assert txt.startswith("stitched v1\n") and "reduce_" in txt
    plan = stitch.Plan(g, "v100", patterns=[[7, 8]])
    assert plan.num_patterns == 1 and plan.patterns() == [[7, 8]]


def test_calibrated_cfg_parity_with_reference():
    """the recalibrated B200 cost model (configs/b200.cfg, measured by
    tools/calibrate_b200.py) uses only keys the reference loader accepts, so
    the unmodified reference planner (oracle/_ref) plans with it too: plans
    must stay byte-identical under the calibrated model"""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    stitch = _stitch()
    cfg = stitch.cfg_path("b200cal")
    from tests.conftest import fixture_graphs
    cases = dict(fixture_graphs())
    for name in ("colreduce", "bert_gelu"):
        cases[name] = graph_text(name)
    with open(os.path.join(GOLD, "random_plans.json")) as f:
        rnd = json.load(f)
    for seed in sorted(rnd, key=int)[:15]:
        cases["random%s" % seed] = rnd[seed]["graph"]
    for name, text in cases.items():
        want, progs, _ = ref.plan(text, cfg)
        plan = stitch.Plan(stitch.Graph(text), "b200cal")
        assert plan.json() == want, name
        keys = [p["key"] for p in json.loads(want)["patterns"]]
        for i, k in enumerate(keys):
            assert plan.kernel_text(i) == progs[k], (name, k)


def test_refined_plans_merge_units():
    """NON-PARITY refinement (stc_plan_refine): starting
    from the reference plan, merges along graph edges that save HBM bytes or
    launches; every merged pattern stays plannable by the reference planner"""
    stitch = _stitch()
    for name, cfg, before, after in (("bert_layer", "b200", 8, 4), ("bert_gelu", "v100", 3, 1),
                                     ("attn_softmax", "b200", 1, 1)):
        p = stitch.Plan(stitch.Graph(graph_text(name)), cfg)
        assert p.stats()["stitched_kernels"] == before
        p.refine()
        assert p.stats()["stitched_kernels"] == after, name
        for i in range(p.num_patterns):
            assert p.kernel_text(i).startswith("stitched v1")
