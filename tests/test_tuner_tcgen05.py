"""Host logic of the tensor-core engines in the tuner (CPU): the tcgen05 searching
domain and its I/O-model pruning (device_tuner.tcgen05_space / tcgen05_io_words),
the engine switch, and the per-layer bound report bench.py prints next to the
measured SM <-> L2 bytes (reference pkg/src/convio/bounds.py:230-271,
dataflow.py:377-407)."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2012_15667_b200 import device_tuner as DT  # noqa: E402
from paper_2012_15667_b200.bounds import lower_bound_dc  # noqa: E402
from paper_2012_15667_b200.dataflow import TileConfig, dc_io_at_optimum  # noqa: E402
from paper_2012_15667_b200.device import shape_of  # noqa: E402
from paper_2012_15667_b200.model import WinogradParams  # noqa: E402


def test_tcgen05_machine_model():
    hw = DT.tcgen05_hw_model()
    assert hw.s_sm == 228 * 1024 // 4 + 256 * 1024 // 4 and hw.n_p == 148
    assert hw.s == 148 * (hw.s_sm // 2)


@pytest.mark.parametrize("args,committed", [
    ((256, 256, 14, 14, 256, 3, 1, 1), TileConfig(2, 2, 256, 32768, 1, 1, 2, layout="HWC")),
    ((256, 64, 56, 56, 64, 3, 1, 1), TileConfig(30, 4, 64, 32768, 2, 1, 2, layout="HWC")),
    ((256, 512, 14, 14, 512, 3, 2, 1), TileConfig(1, 1, 256, 32768, 1, 1, 2, layout="HWC")),
])
def test_domain_contains_plans_and_pruning_keeps_them(args, committed):
    shape = shape_of(*args)
    hw = DT.tcgen05_hw_model()
    full = DT.tcgen05_space(shape, hw, "igemm_3xf16", check_legal=False, prune=None)
    pruned = DT.tcgen05_space(shape, hw, "igemm_3xf16", check_legal=False)
    assert committed in full and committed in pruned
    assert pruned.size <= full.size < full.unconstrained_size
    assert set(pruned.members) <= set(full.members)
    assert all(m.layout == "HWC" and m.n_zt in (2, 4, 8) for m in full.members)   # 3xF16: pair tiles
    # members stay in the reference's sorted order (autotune.py:154-155)
    keys = [(m.s_b, m.x, m.y, m.z, m.n_xt, m.n_yt, m.n_zt) for m in full.members]
    assert keys == sorted(keys)


def test_io_model_ranks_activation_rereads():
    shape = shape_of(256, 256, 14, 14, 256, 3, 1, 1)
    wide = TileConfig(2, 2, 256, 32768, 1, 1, 2, layout="HWC")
    narrow = TileConfig(2, 2, 64, 32768, 1, 1, 2, layout="HWC")
    # z = 64 re-reads the activations K / z = 4 times
    assert DT.tcgen05_io_words(shape, narrow) > 2 * DT.tcgen05_io_words(shape, wide)
    halo = TileConfig(14, 8, 256, 32768, 2, 1, 2, layout="HWC")
    assert DT.tcgen05_io_words(shape, halo) < DT.tcgen05_io_words(shape, wide)


def test_winograd_domain():
    shape = shape_of(256, 256, 14, 14, 256, 3, 1, 1)
    hw = DT.tcgen05_hw_model()
    sp = DT.tcgen05_space(shape, hw, "winograd_tc_3xf16", WinogradParams(4, 3), check_legal=False)
    assert sp.algorithm == "winograd" and sp.size == 12
    assert all(m.x == m.y == m.e == 4 and m.n_zt == 2 for m in sp.members)
    fp = DT.tcgen05_space(shape, hw, "winograd_tc_fp32", WinogradParams(4, 3), check_legal=False)
    assert all(m.n_zt == 1 and m.z <= 128 for m in fp.members)


def test_engine_switch():
    assert DT._engine_for("direct") == "ffma"
    with DT.use_engine("igemm_3xf16"):
        assert DT._engine_for("direct") == "igemm_3xf16"
        assert DT._engine_for("winograd") == "ffma"
        with DT.use_engine("winograd_tc_3xtf32"):
            assert DT._engine_for("winograd") == "winograd_tc_3xtf32"
        assert DT._engine_for("direct") == "igemm_3xf16"
    assert DT._engine_for("direct") == "ffma"
    with pytest.raises(ValueError):
        DT.set_engine("cudnn")


def test_bench_bound_report_matches_the_reference_formulas():
    import bench
    from paper_2012_15667_b200.runner import WORKLOADS
    from paper_2012_15667_b200.device import b200_hw_model
    hw = b200_hw_model()
    spec = WORKLOADS["resnet50"][0]
    b = bench.layer_io_bounds(spec, 256, "igemm_3xf16", None, hw)
    shape = shape_of(256, spec.c, spec.hw, spec.hw, spec.k, 3, 1, 1)
    assert b["omega_bytes"] == int(4 * 256 * lower_bound_dc(shape, hw.s_sm).omega)
    assert b["io_at_optimum_bytes"] == int(4 * dc_io_at_optimum(shape, hw))
    assert b["dataflow"] == "DC"
    w = bench.layer_io_bounds(WORKLOADS["resnet50"][2], 256, "winograd_tc_3xf16", 4, hw)
    assert w["dataflow"] == "WA" and w["omega_bytes"] > 0


def test_network_sequence_is_vgg16():
    from paper_2012_15667_b200.network import VGG16_SEQUENCE, _SHAPE_OF
    convs = [n for n in VGG16_SEQUENCE if n != "M"]
    assert len(convs) == 13 and VGG16_SEQUENCE.count("M") == 5
    assert all(v in convs for v in _SHAPE_OF)
