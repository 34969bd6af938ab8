"""Regenerate the committed golden vectors from the UNMODIFIED reference.

Runs only in the build container (needs /root/reference and the oracle
library built by ``make -C oracle``):

    python tests/golden/make_golden.py [--skip-slow]

Writes, under tests/golden/:
  fixtures.json        the reference's 9 fixture graphs (proj/fixtures/*.graph),
                       as data, so tests run where /root/reference is absent
  plans/<g>__<cfg>.json   per (graph, cfg): the reference's plan.json bytes
                       (pipeline.cpp:45-78), every kernel's .stitch program text
                       (program.cpp:16-91), kernel counts, serialize_graph text
  random_plans.json    100 random_graph(seed, 10) graphs (test_util.hpp:46-116,
                       restated in tests/golden/random_graph.py) x 2 cfgs:
                       plan.json bytes + sha256 of each program text
  numeric.json         sha256 of the reference's eval_reference outputs (f32
                       bytes) for fixtures x seeds 1..10 and config graphs x
                       seeds 1..3, plus the inputs' sha256 (random_inputs)
  numeric_small.npz    full eval_reference outputs, fixtures x seed 1
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import numpy_oracle as no  # noqa: E402
from oracle import ref  # noqa: E402
from tests.golden.random_graph import random_graph_text  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
GRAPHS = os.path.join(ROOT, "paper_2009_10924_b200", "graphs")
CFGS = {"v100": os.path.join(ROOT, "paper_2009_10924_b200", "configs", "v100_default.cfg"),
        "b200": os.path.join(ROOT, "paper_2009_10924_b200", "configs", "b200_device.cfg")}
REF_FIXTURES = "/root/reference/proj/fixtures"
FIXTURES = ["layernorm", "softmax", "attention_softmax", "variance", "remote", "light_chain",
            "expensive_chain", "bias_reduce", "scale_reduce_scale"]
CONFIG_GRAPHS = ["ln_4096x768", "ln2pass_4096x768", "attn_softmax", "colreduce", "bert_gelu",
                 "bert_resln", "bert_layer", "dien_T10", "dien_cut_T10", "dien_T20", "bert_cut"]
SLOW = {"bert_cut", "dien_T20"}


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def f32sha(a) -> str:
    return sha(np.ascontiguousarray(a, dtype=np.float64).astype(np.float32).tobytes())


def plan_record(text, cfg):
    t0 = time.time()
    pj, progs, summ = ref.plan(text, CFGS[cfg])
    return {"plan_json": pj, "programs": progs, "summary": summ,
            "planner_seconds": round(time.time() - t0, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-slow", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--numeric-only", action="store_true",
                    help="only numeric.json / numeric_small.npz (fixtures x seeds 1..10, configs x seeds 1..3)")
    ap.add_argument("--shards", action="store_true",
                    help="per-shard plans (SURVEY §8e): <graph>@<n>__b200.json for n in 2,4,8")
    args = ap.parse_args()
    if args.shards:
        from paper_2009_10924_b200.shard import RULES
        os.makedirs(os.path.join(GOLD, "plans"), exist_ok=True)
        for name in ("attn_softmax", "ln_4096x768", "ln2pass_4096x768", "colreduce", "bert_gelu", "bert_resln"):
            full = open(os.path.join(GRAPHS, name + ".graph")).read()
            for n in (2, 4, 8):
                text = RULES[name].graph_text(full, n)
                rec = plan_record(text, "b200")
                rec["serialized"] = ref.serialize(text)
                rec["graph_text"] = text
                with open(os.path.join(GOLD, "plans", "%s@%d__b200.json" % (name, n)), "w") as fh:
                    json.dump(rec, fh, indent=1, sort_keys=True)
                print("shard plan", name, n, rec["summary"], flush=True)
        return
    os.makedirs(os.path.join(GOLD, "plans"), exist_ok=True)

    fixtures = {f: open(os.path.join(REF_FIXTURES, f + ".graph")).read() for f in FIXTURES}
    with open(os.path.join(GOLD, "fixtures.json"), "w") as fh:
        json.dump(fixtures, fh, indent=1, sort_keys=True)

    graphs = {f: fixtures[f] for f in FIXTURES}
    for c in CONFIG_GRAPHS:
        if args.skip_slow and c in SLOW:
            continue
        graphs[c] = open(os.path.join(GRAPHS, c + ".graph")).read()
    if args.only:
        graphs = {k: v for k, v in graphs.items() if k in args.only.split(",")}

    for name, text in ({} if args.numeric_only else graphs).items():
        for cfg in CFGS:
            path = os.path.join(GOLD, "plans", "%s__%s.json" % (name, cfg))
            rec = plan_record(text, cfg)
            rec["serialized"] = ref.serialize(text)
            with open(path, "w") as fh:
                json.dump(rec, fh, indent=1, sort_keys=True)
            print("plan", name, cfg, rec["summary"], rec["planner_seconds"], "s", flush=True)
    if args.only:
        return

    rnd = {}
    seed = 0
    while len(rnd) < 100 and not args.numeric_only:
        seed += 1
        text = random_graph_text(seed, 10)
        if text is None:
            continue
        entry = {"graph": text}
        for cfg in CFGS:
            pj, progs, summ = ref.plan(text, CFGS[cfg])
            entry[cfg] = {"plan_json": pj, "summary": summ,
                          "programs_sha": {k: sha(v.encode()) for k, v in progs.items()}}
        rnd[str(seed)] = entry
    if not args.numeric_only:
        with open(os.path.join(GOLD, "random_plans.json"), "w") as fh:
            json.dump(rnd, fh, indent=1, sort_keys=True)
        print("random plans done", flush=True)

    numeric, small = {}, {}
    for name, text in graphs.items():
        g = no.parse_graph(text)
        ps = [(p.name, p.dims) for p in g.params()]
        outs = [g.nodes[o].dims for o in g.outputs]
        seeds = range(1, 11) if name in fixtures else range(1, 4)
        rec = {}
        for seed in seeds:
            ins = ref.random_inputs(text, ps, seed)
            got = ref.eval_reference(text, [ins[p] for p, _ in ps], outs)
            rec[str(seed)] = {
                "inputs": {p: f32sha(ins[p]) for p, _ in ps},
                "outputs": {g.nodes[o].name: f32sha(a) for o, a in zip(g.outputs, got)}}
            if name in fixtures and seed == 1:
                for o, a in zip(g.outputs, got):
                    small["%s/%s" % (name, g.nodes[o].name)] = a.astype(np.float32)
        numeric[name] = rec
        print("numeric", name, flush=True)
    with open(os.path.join(GOLD, "numeric.json"), "w") as fh:
        json.dump(numeric, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(GOLD, "numeric_small.npz"), **small)


if __name__ == "__main__":
    main()
