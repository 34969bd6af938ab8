import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLD = os.path.join(ROOT, "tests", "golden")
GRAPHS = os.path.join(ROOT, "paper_2009_10924_b200", "graphs")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running (full-size planning)")


def fixture_graphs():
    with open(os.path.join(GOLD, "fixtures.json")) as f:
        return json.load(f)


def config_graph(name):
    with open(os.path.join(GRAPHS, name + ".graph")) as f:
        return f.read()


def graph_text(name):
    fx = fixture_graphs()
    return fx[name] if name in fx else config_graph(name)


def golden_plan(name, cfg):
    path = os.path.join(GOLD, "plans", "%s__%s.json" % (name, cfg))
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


def dotted(text, prefix="layer."):
    """the same graph with every node renamed to a dotted identifier (the
    reference parser accepts '.' in names, src/parser.cpp:50), plus an
    underscore so the escape of both characters is exercised"""
    import re
    names = [l.split("=")[0].strip() for l in text.splitlines() if "=" in l and not l.strip().startswith("#")]
    for n in sorted(names, key=len, reverse=True):
        text = re.sub(r"(?<![A-Za-z0-9_.])%s(?![A-Za-z0-9_.])" % re.escape(n), prefix + n + "_q", text)
    return text


_PLANS = {}


def cached_plan(text, cfg):
    """one stitch.Plan per (graph text, cfg) per test session: plans are
    immutable after construction and planning DIEN takes ~40 s on this host
    (the reference: ~100 s).  Tests about planning itself construct fresh ones
    where they check the search (test_plan_parity.test_random_graphs)."""
    from paper_2009_10924_b200 import stitch
    key = (text, cfg)
    if key not in _PLANS:
        _PLANS[key] = stitch.Plan(stitch.Graph(text), cfg)
    return _PLANS[key]
