"""The C-ABI library (include/stitch_b200.h) loads without a GPU, exports
every declared symbol, and maps errors onto its status codes; code generation
and NVRTC sm_100a compilation work without a device."""
import ctypes
import os
import re
import shutil

import pytest

from tests.conftest import ROOT, cached_plan, config_graph, fixture_graphs

HEADER = os.path.join(ROOT, "include", "stitch_b200.h")


def _stitch():
    from paper_2009_10924_b200 import stitch
    return stitch


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(stc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_stitch().LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_has_no_hard_driver_dependency():
    # loads on a host without libcuda (this container); CUDA runtime resolves lazily
    deps = os.popen("ldd %s" % _stitch().LIB_PATH).read()
    assert "libcuda.so" not in deps
    assert "libnvrtc" in deps and "libcudart" in deps


def test_error_codes():
    stitch = _stitch()
    with pytest.raises(stitch.StitchError) as e:
        stitch.Graph("p = parameter : f32[4]\np = parameter : f32[4]\n")
    assert e.value.code == 1 and "duplicate-id" in str(e.value) and "line 2" in str(e.value)
    with pytest.raises(stitch.StitchError) as e:
        stitch.Graph("p = warble() : f32[4]\n")
    assert "unknown-op" in str(e.value)
    g = stitch.Graph(fixture_graphs()["softmax"])
    with pytest.raises(stitch.StitchError) as e:
        stitch.Plan(g, "/nonexistent.cfg")
    assert e.value.code == 1 and "cannot open device config" in str(e.value)


def test_graph_io_introspection():
    stitch = _stitch()
    g = stitch.Graph(fixture_graphs()["layernorm"])
    assert [p.name for p in g.params] == ["x", "gamma", "beta"]
    assert g.params[0].dims == (64, 256) and g.params[0].dtype == "f32"
    assert [o.name for o in g.outputs] == ["y"]
    assert g.num_nodes == 24


@pytest.mark.parametrize("mode", ["stitched", "program", "unfused"])
def test_codegen_and_nvrtc_compile_all_fixtures(mode):
    stitch = _stitch()
    for name, text in sorted(fixture_graphs().items()):
        plan = stitch.Plan(stitch.Graph(text), "v100")
        src, kernels = plan.codegen(mode)
        assert len(kernels) == plan.stats()["stitched_kernels"] or mode == "unfused"
        assert "extern \"C\" __global__" in src
        key = stitch.compile_cuda(src)
        assert re.fullmatch(r"[0-9a-f]{32}", key)


@pytest.mark.parametrize("persist", ["0", "1"])
def test_dotted_tensor_names_compile(monkeypatch, persist):
    """graph names with '.' (valid in the reference's parser) become C
    identifiers through one injective escape in every generator (dataflow,
    program, unfused, packed, deduplicated, persistent)"""
    from tests.conftest import config_graph, dotted
    monkeypatch.setenv("STITCH_PERSIST", persist)
    stitch = _stitch()
    texts = [dotted(t) for t in fixture_graphs().values()] + [dotted(config_graph("dien_T10"), "a.b_")]
    for text in texts:
        plan = cached_plan(text, "b200")
        for mode in ("stitched", "program", "unfused"):
            src, kernels = plan.codegen(mode)
            assert "TX_" in src
            assert not re.search(r"\bT_[A-Za-z0-9_]*\.", src)
            assert re.fullmatch(r"[0-9a-f]{32}", stitch.compile_cuda(src))
    # injective: 'a.b' and 'a_b' side by side stay distinct parameters
    text = "a.b = parameter : f32[64]\na_b = parameter : f32[64]\ny = add(a.b, a_b)\noutput y\n"
    src, kernels = stitch.Plan(stitch.Graph(text), "b200").codegen()
    assert "TX_a_Db" in src and "T_a_b" in src
    stitch.compile_cuda(src)


def test_dataflow_templates_chosen_for_fixtures():
    stitch = _stitch()
    want = {"layernorm": "regional", "softmax": "regional", "variance": "regional",
            "light_chain": "local", "expensive_chain": "local", "remote": "local",
            "bias_reduce": "regional", "scale_reduce_scale": "regional"}
    for name, tmpl in want.items():
        _, kernels = stitch.Plan(stitch.Graph(fixture_graphs()[name]), "v100").codegen()
        assert [k["template"].split("+")[0] for k in kernels] == [tmpl], name


def test_launch_units_packed_per_producer_set(monkeypatch):
    """launch units with the same producer kernels share one launch
    (executor-level; the plan is unchanged): small opaque placeholders a CTA
    per op, local-template patterns side by side.  DIEN T=10: the 13
    parameter-only placeholders form one pack, each step's three gate
    placeholders another; packing repeats over the packs, so the nine
    attention-column slices, then their squeezes (regional), then the
    attention broadcasts each become one launch -> 88 plan kernels in 34
    launches (the attention-score placeholder over all T states is a
    5-CTA cluster of its own).  Launch graph only: STITCH_RESIDENT=0"""
    monkeypatch.setenv("STITCH_RESIDENT", "0")
    stitch = _stitch()
    from tests.conftest import config_graph
    plan = cached_plan(config_graph("dien_T10"), "b200")
    _, packed = plan.codegen()
    monkeypatch.setenv("STITCH_LOCAL_PACK", "0")
    _, opaque_only = plan.codegen()
    monkeypatch.setenv("STITCH_OPAQUE_PACK", "0")
    _, single = plan.codegen()
    assert len(single) == plan.stats()["stitched_kernels"] == 88
    assert len(opaque_only) == 58
    assert len(packed) == 34
    units = lambda ks: sorted(p for k in ks for p in k["pattern"].split("+"))
    assert units(packed) == units(opaque_only) == units(single)  # every unit exactly once
    packs = [k for k in opaque_only if k["template"].startswith("opaque(pack")]
    assert sorted(k["grid"] for k in packs) == [3] * 9 + [13]
    assert all(k["grid"] == len(k["pattern"].split("+")) for k in packs)
    outs = lambda ks: sorted(o for k in ks for o in k["outputs"])
    assert outs(packed) == outs(single)
    # launches with identical code (modulo their tensors) share one function
    assert len({k["symbol"] for k in packed}) == 10
    monkeypatch.setenv("STITCH_DEDUP", "0")
    _, nodedup = plan.codegen()
    assert len({k["symbol"] for k in nodedup}) == 88


@pytest.mark.parametrize("mode", ["1", "2"])
def test_tma_staged_rows_codegen(monkeypatch, mode):
    """TMA-staged regional rows compile for sm_100a without a device: mode 1
    (one ring of row tiles per CTA, the whole tile on one mbarrier), mode 2
    (per-team rings: one bulk copy per row and tensor, one mbarrier per row
    buffer, a team-only sync before the refill -- __syncwarp for teams of at
    most one warp, the CTA barrier for wider teams)"""
    stitch = _stitch()
    monkeypatch.setenv("STITCH_STAGE", mode)
    for name in ("ln_4096x768", "bert_resln", "attn_softmax"):
        src, kernels = stitch.Plan(stitch.Graph(config_graph(name)), "b200").codegen()
        assert all(k["template"].endswith("+tma") for k in kernels), (name, kernels)
        assert "bulk_g2s(" in src and "mbar_wait(" in src
        if mode == "2":
            assert "TMA per-team rings" in src and "__syncwarp" in src, name
        else:
            assert "TMA pipeline" in src, name
        assert re.fullmatch(r"[0-9a-f]{32}", stitch.compile_cuda(src))


def test_persistent_template_codegen(monkeypatch):
    """opt-in persistent template: a launch-bound plan becomes one cooperative
    kernel whose unit bodies are shared between textually identical units
    (DIEN's per-step kernels); plans with large kernels are left alone"""
    stitch = _stitch()
    from tests.conftest import config_graph
    monkeypatch.setenv("STITCH_PERSIST", "1")
    monkeypatch.setenv("STITCH_RESIDENT", "0")
    monkeypatch.setenv("STITCH_OPAQUE_CLUSTER", "1")  # the persistent template takes no clusters
    src, kernels = cached_plan(config_graph("dien_T10"), "b200").codegen()
    assert [k["template"] for k in kernels] == ["persistent(33)"]
    assert len(set(re.findall(r"\bunit\d+_\(", src))) == 9  # 33 units, 9 distinct bodies
    assert re.fullmatch(r"[0-9a-f]{32}", stitch.compile_cuda(src))
    _, big = cached_plan(config_graph("bert_layer"), "b200").codegen()
    assert len(big) > 1 and not any(k["template"].startswith("persistent") for k in big)


def test_kernel_produced_tensors_never_read_non_coherently(monkeypatch):
    """under programmatic dependent launch a tensor written by an earlier
    kernel is not read-only for the consumer's lifetime: only graph
    parameters may go through the ld.global.nc helpers (ld4 / ld4c / ld4h /
    ldv); everything else must use the coherent ones (ld4k / ldvk / ld4hk),
    which ptxas keeps below griddepcontrol.wait"""
    monkeypatch.setenv("STITCH_RESIDENT", "0")  # the launch graph's kernels (resident units read generically)
    stitch = _stitch()
    from tests.conftest import config_graph, fixture_graphs
    texts = [config_graph(n) for n in ("dien_T10", "bert_layer", "bert_cut")] + list(fixture_graphs().values())
    for text in texts:
        plan = cached_plan(text, "b200")
        params = {t.name for t in plan.graph.params}
        for mode in ("stitched", "unfused"):
            src, _ = plan.codegen(mode)
            for fn, t in re.findall(r"\b(ld4c?|ld4h|ldv)\(T_(\w+)", src):
                assert t in params, (fn, t)


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not on PATH")
def test_sass_no_global_write_before_pdl_wait(monkeypatch):
    """SASS of the generated kernels (tools/sass_pdl_check.py): no global
    store / reduction / atomic ahead of griddepcontrol.wait (ACQBULK) in any
    kernel, and every kernel waits"""
    monkeypatch.setenv("STITCH_RESIDENT", "0")  # launch-graph kernels (the resident kernel has no PDL)
    from tools.sass_pdl_check import check
    for name in ("dien_T10", "bert_layer", "attn_softmax", "colreduce", "bert_resln"):
        for fn, r in check(name, plan=cached_plan(config_graph(name), "b200")).items():
            assert r["waited"] and r["writes_before_wait"] == 0, (name, fn, r)


def test_cubin_cache_warm_up(tmp_path, monkeypatch):
    """stc_cache_warm: NVRTC-compiles plan modules into
    the persistent cache on host threads without a GPU; a second warm-up is
    all cache hits"""
    monkeypatch.setenv("STITCH_CACHE_DIR", str(tmp_path))
    stitch = _stitch()
    from tests.conftest import fixture_graphs
    plans = [stitch.Plan(stitch.Graph(t), "b200") for _, t in sorted(fixture_graphs().items())[:4]]
    assert stitch.warm_cache(plans, threads=4) == (4, 0)
    assert stitch.warm_cache(plans, threads=4) == (0, 4)
    assert len([f for f in os.listdir(tmp_path) if f.endswith(".cubin")]) == 4
