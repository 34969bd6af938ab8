"""Resident template, device-free half: which plans it takes, what it emits
(cg_resident.cpp).  The GPU parity tests are in test_gpu_exec.py."""
import re

import pytest

from tests.conftest import cached_plan, config_graph


def _codegen(name, monkeypatch, resident=True):
    from paper_2009_10924_b200 import stitch
    monkeypatch.setenv("STITCH_RESIDENT", "1" if resident else "0")
    return cached_plan(config_graph(name), "b200").codegen()


@pytest.mark.parametrize("name,rows", [("dien_T10", 16), ("dien_T20", 16)])
def test_dien_plan_becomes_one_cluster_kernel(name, rows, monkeypatch):
    src, kernels = _codegen(name, monkeypatch)
    assert len(kernels) == 1
    k = kernels[0]
    assert k["template"].startswith("resident(") and k["cluster"] == k["grid"] == 16 and k["block"] == 1024
    assert 0 < k["smem"] <= 200 * 1024
    assert "256 batch rows, %d per CTA" % rows in src
    # one cluster barrier per placeholder group: T=10 -> prologue + one per step
    m = re.search(r"(\d+) cluster barriers", src)
    assert m and int(m.group(1)) <= 21
    # every unit's global accesses are generic in the resident kernel
    body = src[src.index("// ---- " + k["name"]):]
    for raw in ("ld.global", "ld4(", "ld4k(", "ld4c(", "st4(", "griddepcontrol"):
        assert raw not in body, raw


@pytest.mark.parametrize("name", ["colreduce", "ln_4096x768", "bert_cut"])
def test_non_row_local_or_large_plans_fall_back(name, monkeypatch):
    """column reductions reduce over the batch axis; the BERT/LN configs'
    boundary tensors exceed the shared-memory budget: the launch graph runs"""
    _, kernels = _codegen(name, monkeypatch)
    assert not any(k["template"].startswith("resident(") for k in kernels)


def test_resident_source_compiles_for_sm100a(monkeypatch):
    from paper_2009_10924_b200 import stitch
    src, _ = _codegen("dien_T10", monkeypatch)
    assert stitch.compile_cuda(src)


@pytest.mark.parametrize("name", ["dien_T10", "dien_T20"])
def test_shared_memory_slots_never_alias_live_tensors(name, monkeypatch):
    """every unit call binds distinct tensors to distinct shared-memory slots
    (a slot read by several placeholders of one group is freed once)"""
    src, _ = _codegen(name, monkeypatch)
    calls = re.findall(r"\bru\d+_\((.*), v_, \d+\);", src)
    assert calls
    for args in calls:
        # a unit binds each of its (distinct) tensors once: distinct slots
        offs = re.findall(r"rs_smem_ \+ (\d+)\)", args)
        assert len(set(offs)) == len(offs), args


@pytest.mark.parametrize("name", ["dien_T10", "dien_T20"])
def test_split_groups_fill_no_slot_a_filler_binds(name, monkeypatch):
    """split placeholder groups (phase A push, fillers, phase B fold + fill):
    the fillers run without a barrier before phase B's fills, so no fill may
    land in a shared-memory slot any filler between the two phases binds,
    and every filler is independent of its group (it reads none of the
    group's outputs)"""
    src, _ = _codegen(name, monkeypatch)
    body = src[src.index("// ---- "):]
    parts = re.split(r"\n  \{  // placeholder group", body)
    splits = 0
    for i, part in enumerate(parts[1:], 1):
        if not part.startswith(" (wait):"):
            continue
        splits += 1
        fills = set(re.findall(r"st4_g\(reinterpret_cast<float\*>\(rs_smem_ \+ (\d+)\)", part.split("\n  }\n")[0]))
        assert fills, part[:200]
        fillers = parts[i - 1].split("\n  }\n", 1)[1] if "\n  }\n" in parts[i - 1] else ""
        bound = set()
        for args in re.findall(r"\bru\d+_\((.*), v_, \d+\);", fillers):
            bound |= set(re.findall(r"rs_smem_ \+ (\d+)\)", args))
        assert not (fills & bound), (sorted(fills & bound), part[:120])
    assert splits >= (9 if name == "dien_T10" else 19)
