"""Tuned-plan selection (runner.load_plans) and the committed tuned tables."""

import json
import os

import pytest
import torch

from paper_2012_15667_b200 import runner
from paper_2012_15667_b200.dataflow import TileConfig


def _write(tmp_path, layers):
    d = tmp_path / "tuned"
    d.mkdir()
    (d / "b200_toy.json").write_text(json.dumps({"n_tune": 8, "layers": layers}))
    return str(d)


def test_load_plans_picks_fastest_allowed_candidate(tmp_path, monkeypatch):
    t_dir = TileConfig(8, 4, 16, 8192, 2, 2, 4).to_dict()
    t_w = TileConfig(8, 8, 16, 32768, 4, 4, 4, e=2).to_dict()
    t_tc = TileConfig(28, 4, 64, 32768, 1, 1, 1, layout="HWC").to_dict()
    layers = {"L": {"algorithm": "direct", "tile": t_dir, "candidates": {
        "direct": {"tuner": {"best": t_dir, "seconds": 3e-3}},
        "winograd2": {"tuner": {"best": t_w, "seconds": 2e-3}},
        "igemm_3xtf32": {"tuner": {"best": t_tc, "seconds": 1e-3}},
        "igemm_tf32": {"tuner": {"best": t_tc, "seconds": 0.5e-3}},
        "winograd4": {"error": "no tile"},
    }}}
    monkeypatch.setattr(runner, "TUNED_DIR", _write(tmp_path, layers))
    fp32 = runner.load_plans("toy")
    assert fp32["L"]["algorithm"] == "igemm_3xtf32"            # fastest FP32-accurate
    cuda = runner.load_plans("toy", runner.CUDA_CORE_ALGORITHMS)
    assert cuda["L"]["algorithm"] == "winograd" and cuda["L"]["e"] == 2
    tf32 = runner.load_plans("toy", ("igemm_tf32",))
    assert tf32["L"]["tile"].layout == "HWC"


def test_missing_table_means_untuned(tmp_path, monkeypatch):
    monkeypatch.setattr(runner, "TUNED_DIR", str(tmp_path))
    assert runner.load_plans("nothing") == {}


@pytest.mark.parametrize("workload", ["resnet50", "vgg16"])
def test_committed_tables_name_real_layers_and_legal_tiles(workload):
    path = os.path.join(runner.TUNED_DIR, f"b200_{workload}.json")
    if not os.path.exists(path):
        pytest.skip("not tuned yet")
    plans = runner.load_plans(workload)
    names = {s.name for s in runner.WORKLOADS[workload]}
    assert set(plans) <= names and plans
    for name, plan in plans.items():
        assert plan["algorithm"] in runner.FP32_ALGORITHMS
        assert isinstance(plan["tile"], TileConfig)


@pytest.mark.parametrize("key,alg,e", [
    ("direct", "direct", None), ("direct_nhwc", "direct", None), ("winograd2", "winograd", 2),
    ("winograd4", "winograd", 4), ("igemm_3xtf32", "igemm_3xtf32", None),
    ("igemm_bf16", "igemm_bf16", None), ("winograd_tc_3xtf32_e4", "winograd_tc_3xtf32", 4),
    ("winograd_tc_bf16_e2", "winograd_tc_bf16", 2),
])
def test_candidate_keys_map_to_algorithms(key, alg, e):
    assert runner.candidate_algorithm(key) == (alg, e)


def test_tensor_core_winograd_and_bf16_plans(tmp_path, monkeypatch):
    t_wtc = TileConfig(4, 4, 256, 16384, 1, 1, 2, layout="HWC", e=4).to_dict()
    t_ig = TileConfig(2, 2, 256, 32768, 1, 1, 2, layout="HWC").to_dict()
    t_nhwc = TileConfig(2, 2, 128, 32768, 1, 1, 1, layout="HWC").to_dict()
    layers = {"L": {"candidates": {
        "winograd_tc_3xtf32_e4": {"tuner": {"best": t_wtc, "seconds": 1e-3}},
        "igemm_3xtf32": {"tuner": {"best": t_ig, "seconds": 2e-3}},
        "igemm_bf16": {"tuner": {"best": t_ig, "seconds": 0.2e-3}},
        "winograd_tc_bf16_e4": {"tuner": {"best": t_wtc, "seconds": 0.1e-3}},
        "direct_nhwc": {"tuner": {"best": t_nhwc, "seconds": 5e-3}},
    }}}
    monkeypatch.setattr(runner, "TUNED_DIR", _write(tmp_path, layers))
    fp32 = runner.load_plans("toy")["L"]
    assert fp32["algorithm"] == "winograd_tc_3xtf32" and fp32["e"] == 4   # bf16 is never FP32
    bf16 = runner.load_plans("toy", ("igemm_bf16", "winograd_tc_bf16"))["L"]
    assert bf16["algorithm"] == "winograd_tc_bf16"
    cuda = runner.load_plans("toy", runner.CUDA_CORE_ALGORITHMS)["L"]
    assert cuda["algorithm"] == "direct" and cuda["tile"].layout == "HWC"
    spec = runner.LayerSpec("L", 64, 14, 256)
    layer = runner.ConvLayer(spec, None, fp32)
    assert layer.precision == "3xtf32" and layer.layout == "HWC" and layer.e == 4
    assert layer.filter_elems() == 36 * 64 * 256


def test_per_batch_table_preferred_for_the_local_batch(tmp_path, monkeypatch):
    d = tmp_path / "tuned"
    d.mkdir()
    t1 = TileConfig(2, 2, 256, 32768, 1, 1, 2, layout="HWC").to_dict()
    t2 = TileConfig(1, 1, 128, 32768, 1, 1, 1, layout="HWC").to_dict()
    (d / "b200_toy.json").write_text(json.dumps({"n_tune": 256, "layers": {"L": {"candidates": {
        "igemm_3xtf32": {"tuner": {"best": t1, "seconds": 1e-3}}}}}}))
    (d / "b200_toy_n32.json").write_text(json.dumps({"n_tune": 32, "layers": {"L": {"candidates": {
        "igemm_3xtf32": {"tuner": {"best": t2, "seconds": 1e-4}}}}}}))
    monkeypatch.setattr(runner, "TUNED_DIR", str(d))
    assert runner.load_plans("toy")["L"]["tile"].z == 256
    assert runner.load_plans("toy", n=32)["L"]["tile"].z == 128
    assert runner.load_plans("toy", n=64)["L"]["tile"].z == 128   # no n64 table: the nearest batch's (32)
    assert runner.load_plans("toy", n=200)["L"]["tile"].z == 256  # nearer the full-batch table
    assert runner.tuned_table("toy", 8).endswith("b200_toy_n32.json")


@pytest.mark.parametrize("n", [256, 32])
def test_group_layers_stacks_repeated_3xf16_layers(n):
    """bench.py's timed step runs the repeated same-plan ResNet-50 3x3 layers as grouped
    launches: the groups are exactly the runs of identical specs on one 3xF16 pair plan,
    and each layer's filter workspace is its slice of the group's packed buffer."""
    specs = runner.expand(runner.WORKLOADS["resnet50"])
    plans = runner.load_plans("resnet50", n=n)
    layers = [runner.ConvLayer(s, torch.zeros(s.k, s.c, s.r, s.r), plans.get(s.name)) for s in specs]
    units = runner.group_layers(layers, n, "cpu")
    assert sorted(i for _, _, idx in units for i in idx) == list(range(len(layers)))
    for kind, unit, idx in units:
        if kind != "group":
            continue
        assert len(idx) >= 2 and idx == list(range(idx[0], idx[-1] + 1))
        assert {layers[i].spec for i in idx} == {unit.spec} and unit.tile.n_zt >= 2
        assert all(layers[i].algorithm == "igemm_3xf16" for i in idx)
        s = unit.spec
        assert unit.x.shape == (len(idx) * n, s.c, s.hw, s.hw) and unit.x.stride()[1] == 1
        for g, i in enumerate(idx):
            ws = layers[i]._ws
            assert ws.data_ptr() == unit.wbuf.data_ptr() + g * unit.slice_bytes
            assert ws.numel() * 4 <= unit.slice_bytes
            assert unit.x_of(g).data_ptr() == unit.x.data_ptr() + g * n * s.c * s.hw * s.hw * 4
    grouped = [idx for kind, _, idx in units if kind == "group"]
    assert grouped, "the tuned ResNet-50 tables put the repeated layers on 3xF16 pair tiles"
    # bench.py's plans: the group table's overrides move repeated Winograd layers onto a
    # grouped 3xF16 launch; every overridden layer then sits in a group with its tile
    over = runner.load_group_overrides("resnet50", n)
    plans.update(over)
    layers = [runner.ConvLayer(s, torch.zeros(s.k, s.c, s.r, s.r), plans.get(s.name)) for s in specs]
    gp = runner.load_group_plans("resnet50", n)
    units = runner.group_layers(layers, n, "cpu", gp)
    for name, plan in over.items():
        idx = [i for i, s in enumerate(specs) if s.name == name]
        unit = next(u for kind, u, ix in units if kind == "group" and ix == idx)
        assert unit.tile == plan["tile"] == gp[name]


@pytest.mark.parametrize("workload", ["resnet50", "vgg16"])
def test_group_plans_table_gives_feasible_tiles(workload):
    """The committed grouped-launch table (scripts/tune_groups.py): every per-batch group
    entry names a real repeated layer, its best tile is one of its measured candidates,
    and the tile's CTA-pair image stack divides the per-layer batch."""
    path = runner.group_table(workload)
    if not os.path.exists(path):
        pytest.skip("no grouped-launch table")
    tab = json.load(open(path))
    names = {s.name: s for s in runner.WORKLOADS[workload]}
    for n, groups in tab["groups"].items():
        plans = runner.load_group_plans(workload, int(n))
        assert set(plans) == set(groups)
        overrides = runner.load_group_overrides(workload, int(n))
        for name, ent in groups.items():
            assert names[name].count == ent["layers"] >= 2
            if ent.get("replaces"):   # a repeated non-3xF16 layer moved onto a grouped 3xF16 launch
                assert ent["us_with_prep"] < 0.97 * ent["own_us_with_prep"] and name in overrides
                assert all(r["use_group"] for r in ent.get("runs", [ent]))
                assert overrides[name]["algorithm"] == "igemm_3xf16" and overrides[name]["tile"] == plans[name]
                continue
            assert name not in overrides
            measured = [c for c in ent["candidates"] if "us" in c]
            if "runs" not in ent:   # one tuning run: its fastest candidate
                assert ent["us"] == min(c["us"] for c in measured)
            assert ent["tile"] in [c["tile"] for c in measured]
            t = plans[name]
            if not ent.get("use_group", True):
                assert t is None and ent["singles_us"] <= ent["us"]
                continue
            assert t.n_zt >= 2 and t.layout == "HWC"


@pytest.mark.parametrize("shape,alg", [((192, 17, 192, 1), "igemm_3xf16"), ((512, 7, 512, 1), "igemm_3xf16"),
                                       ((256, 28, 512, 2), "igemm_3xf16"), ((96, 35, 96, 1), "direct"),
                                       ((3, 64, 32, 1), "direct")])
def test_default_plan_for_untuned_shapes(shape, alg):
    """A layer no tuned table covers gets the FP32-accurate tensor-core plan the planner
    accepts at its batch (FFMA direct only when no tcgen05 tile applies); plan_for keeps a
    tuned plan that fits the batch and replaces one that does not."""
    c, hw, k, stride = shape
    spec = runner.LayerSpec("untuned", c, hw, k, stride=stride)
    for n in (1, 5, 64):
        plan = runner.default_plan(spec, n)
        assert plan["algorithm"] == alg
        assert runner.plan_feasible(spec, n, plan)
    tuned = runner.load_plans("resnet50", n=256)
    res4 = next(s for s in runner.WORKLOADS["resnet50"] if s.name == "res4_3x3")
    assert runner.plan_for(res4, 256, tuned) is tuned["res4_3x3"]
    big_stack = {"res4_3x3": {"algorithm": "igemm_3xf16", "e": None,
                              "tile": TileConfig(1, 1, 256, 32768, 1, 1, 2, layout="HWC")}}
    assert runner.plan_feasible(res4, 256, big_stack["res4_3x3"])


def test_group_layers_skips_stacks_that_straddle_layers():
    """At a batch no table was tuned for, a group whose tile stacks more images per CTA
    pair than divide the per-layer batch runs as single launches instead of failing."""
    t64 = TileConfig(1, 2, 256, 32768, 1, 1, 2, layout="HWC")      # 64 images per stack
    assert runner.group_stack_ok(t64, 128, 5) and not runner.group_stack_ok(t64, 96, 5)
    assert runner.group_stack_ok(TileConfig(30, 4, 64, 32768, 2, 1, 4, layout="HWC"), 7, 3)   # halo: 1 image
    t32 = TileConfig(2, 2, 256, 32768, 1, 1, 2, layout="HWC")     # min(32, 5 x n) images per stack
    assert runner.group_stack_ok(t32, 32, 5) and not runner.group_stack_ok(t32, 1, 5)
    spec = next(s for s in runner.WORKLOADS["resnet50"] if s.name == "res4_3x3")
    plan = {"algorithm": "igemm_3xf16", "tile": t64, "e": None}
    layers = [runner.ConvLayer(spec, torch.zeros(spec.k, spec.c, 3, 3), plan) for _ in range(5)]
    assert [k for k, _, _ in runner.group_layers(layers, 96, "cpu")] == ["single"] * 5
    assert [k for k, _, _ in runner.group_layers(layers, 128, "cpu")] == ["group"]
