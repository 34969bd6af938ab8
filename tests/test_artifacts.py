"""Artifact parity (src/pipeline.cpp:45-224):
run_pipeline / stitchc write plan.json, kernels/kNNN_<producer>.stitch,
report.txt and graph.dot byte-identical to the UNMODIFIED reference's
run_pipeline (oracle/_ref) on every fixture under both device profiles."""
import os
import subprocess

import pytest

from tests.conftest import ROOT, fixture_graphs


def _tree(d):
    out = {}
    for base, _, files in os.walk(d):
        for f in files:
            p = os.path.join(base, f)
            with open(p, "rb") as fh:
                out[os.path.relpath(p, d)] = fh.read()
    return out


@pytest.mark.parametrize("cfg", ["v100", "b200"])
def test_pipeline_artifacts_byte_identical(tmp_path, cfg):
    from oracle import ref
    from paper_2009_10924_b200 import stitch
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    for name, text in sorted(fixture_graphs().items()):
        g = tmp_path / (name + ".graph")
        g.write_text(text)
        mine, theirs = tmp_path / ("ours_" + name), tmp_path / ("ref_" + name)
        rc = stitch.run_pipeline(str(g), cfg, output_dir=str(mine), emit_dot=True, run_baseline=True, seed=7)
        rc_ref = ref.run_pipeline(str(g), stitch.cfg_path(cfg), str(theirs), emit_dot=True, run_baseline=True,
                                  seed=7)
        assert rc == rc_ref == 0, name
        a, b = _tree(str(mine)), _tree(str(theirs))
        assert sorted(a) == sorted(b), (name, sorted(a), sorted(b))
        for f in a:
            assert a[f] == b[f], (name, f)


def test_stitchc_cli_matches_reference_pipeline(tmp_path):
    """tools/stitchc (the drop-in for the reference's CLI) -> same artifacts"""
    from oracle import ref
    from paper_2009_10924_b200 import stitch
    tool = os.path.join(ROOT, "tools", "stitchc")
    if not (ref.available() and os.path.exists(tool)):
        pytest.skip("stitchc / oracle not built")
    g = tmp_path / "layernorm.graph"
    g.write_text(fixture_graphs()["layernorm"])
    r = subprocess.run([tool, "--graph", str(g), "--device-config", stitch.cfg_path("b200"), "--out", str(tmp_path / "a"),
                        "--emit-dot"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert ref.run_pipeline(str(g), stitch.cfg_path("b200"), str(tmp_path / "b"), emit_dot=True) == 0
    a, b = _tree(str(tmp_path / "a")), _tree(str(tmp_path / "b"))
    assert a == b
