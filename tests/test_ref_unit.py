"""The reference's OWN test suite against this framework: its 94 doctest unit
tests (/root/reference/proj/tests/test_*.cpp) and its 8-criterion acceptance
gate (tests/acceptance.cpp) compiled UNCHANGED against the drop-in headers
(include/stitch) and linked with libstitch_b200.so (tests/ref_unit/Makefile;
doctest shim tests/ref_unit/doctest.h).  Execution entry points
(run_program / eval_plan / eval_reference / run_pipeline --run-sim) run on the
B200, so those cases are GPU tests; everything else runs here.

The binaries are built where /root/reference exists (this container, by
build() or on first use) and travel with the repo snapshot to the GPU box."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REF_UNIT = os.path.join(HERE, "ref_unit")
BUILD = os.path.join(REF_UNIT, "_build")
# cases that execute a plan (need a GPU with this framework's library)
EXEC_CASES = [
    "pipeline writes the full artifact set", "sim comparison passes on every shipped fixture",
    "reduce_sum of ones over axis 1", "full-range slice is a bitwise identity",
    "layer-norm reference output has zero-mean", "fused light chain matches the reference bitwise",
    "warp-composition row reduction", "recompute and reuse plans", "removing a barrier trips",
]


def _binaries():
    ut, acc = os.path.join(BUILD, "unit_tests"), os.path.join(BUILD, "acceptance")
    if not (os.path.exists(ut) and os.path.exists(acc)):
        if not os.path.isdir("/root/reference/proj/tests") or not shutil.which("make"):
            pytest.skip("reference tests not built and /root/reference absent")
        subprocess.run(["python", os.path.join(REF_UNIT, "prepare_data.py")], check=True, capture_output=True)
        subprocess.run(["make", "-C", REF_UNIT, "-j8"], check=True, capture_output=True)
    if not os.path.isdir(os.path.join(REF_UNIT, "_data")):
        subprocess.run(["python", os.path.join(REF_UNIT, "prepare_data.py")], check=True, capture_output=True)
    return ut, acc


def _run(cmd, timeout):
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=REF_UNIT)
    return r.returncode, r.stdout + r.stderr


def test_reference_unit_tests_host_side():
    """parser, graph, device model, schedule catalog, planner, explorer,
    baseline, expr/program: the reference's own checks, our library"""
    ut, _ = _binaries()
    rc, out = _run([ut, "--exclude=" + ",".join(EXEC_CASES)], 600)
    assert rc == 0, out[-3000:]
    assert "0 failed" in out, out[-2000:]


@pytest.mark.gpu
def test_reference_unit_tests_all_on_gpu():
    ut, _ = _binaries()
    rc, out = _run([ut], 900)
    assert rc == 0, out[-3000:]
    assert ", 0 failed" in out.split("test cases:")[-1], out[-2000:]


@pytest.mark.gpu
def test_reference_acceptance_gate_on_gpu():
    """criteria 1-8 of tests/acceptance.cpp (criterion 4 executes every
    fixture's plan on the B200 and compares with eval_reference)"""
    _, acc = _binaries()
    rc, out = _run([acc], 1500)
    assert rc == 0, out[-3000:]
    assert "FAIL" not in out, out[-3000:]
