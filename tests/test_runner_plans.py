"""Tuned-plan selection (runner.load_plans) and the committed tuned tables."""

import json
import os

import pytest

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
