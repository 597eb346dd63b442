"""Measurement backends of the tuner: the device backend is swapped for a
deterministic cost table here (the reference's own mock strategy,
pkg/tests/test_autotune.py:129-143), so the tuner loop, the exhaustive oracle
and random search run their device code paths without a GPU."""

import math

import pytest

from paper_2012_15667_b200 import autotune as A
from paper_2012_15667_b200.autotune import build_space, tune, exhaustive_oracle, random_search
from paper_2012_15667_b200.device import b200_hw_model, shape_of, B200_S_SM
from paper_2012_15667_b200.model import ConvShape, HwModel


def _table_cost(cfg, shape, hw, algorithm, winograd):
    # a smooth synthetic "device time": prefers 8x8x16 blocks of 128 threads
    if cfg.threads > 512:
        return math.inf
    return (abs(cfg.x - 8) + abs(cfg.y - 8) + abs(cfg.z - 16) / 2 + abs(cfg.threads - 128) / 32
            + cfg.s_b / 65536 + 1.0)


A.register_measure_backend("table", _table_cost)


def test_unknown_backend_raises():
    with pytest.raises(ValueError):
        A.measure(None, None, None, "direct", backend="nope")


def test_tune_with_table_backend_reaches_exhaustive_optimum_region():
    shape = ConvShape.from_output(16, 16, 32, 16, 3, 3)
    hw = HwModel(s=16384, s_sm=8192, n_p=2)
    space = build_space(shape, hw, "direct")
    ex_cfg, ex_cost = exhaustive_oracle(space, backend="table")
    sess = tune(shape, hw, "direct", budget=96, seed=3, n_s=8, space=space, backend="table")
    assert math.isfinite(sess.best_cost)
    assert sess.best_cost <= ex_cost * 1.5
    rs_cfg, rs_cost = random_search(space, 96, 3, backend="table")
    assert ex_cost <= rs_cost and ex_cost <= sess.best_cost
    assert all(m.cost == _table_cost(m.config, shape, hw, "direct", None) for m in sess.measurements)


def test_measure_backend_context_routes_default_calls():
    shape = ConvShape.from_output(4, 4, 4, 4, 3, 3)
    hw = HwModel(s=4096)
    cfg = build_space(shape, hw, "direct").members[0]
    model_cost = A.measure(cfg, shape, hw, "direct").cost
    with A.measure_backend("table"):
        assert A.measure(cfg, shape, hw, "direct").cost == _table_cost(cfg, shape, hw, "direct", None)
    assert A.measure(cfg, shape, hw, "direct").cost == model_cost


def test_b200_machine_model():
    hw = b200_hw_model()
    assert hw.s_sm == B200_S_SM == 65536 + 58368
    assert hw.n_p == 296 and hw.s == 296 * (B200_S_SM // 2)
    assert A.default_sb_values(hw)[-1] == 32768


def test_legal_projection_without_gpu():
    dt = pytest.importorskip("paper_2012_15667_b200.device_tuner")
    dt.set_padding(1)
    try:
        shape = shape_of(4, 64, 56, 56, 64, 3, 1, 1)
        full = build_space(shape, b200_hw_model(), "direct", thread_axes=False, layouts=("CHW",))
        legal = dt.legal_projection(full)
        assert 0 < legal.size <= full.size
        assert all(c in set(full.members) for c in legal.members)
        assert list(legal.members) == sorted(legal.members, key=A._member_key)
    finally:
        dt.set_padding(0)
