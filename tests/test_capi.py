"""The C-ABI library on a CPU-only machine: it loads, exports every symbol the
header declares, and its host-side planning (legality of a TileConfig's
device projection, transform matrices) answers without a GPU.  No kernel is
launched here."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import winograd_mats as wm
from paper_2012_15667_b200 import _native as N
from paper_2012_15667_b200 import TileConfig
from paper_2012_15667_b200.conv import query

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "convio_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(convio_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    names = _declared()
    assert "convio_conv_direct_f32" in names and "convio_query" in names
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTED)
    assert lib.convio_version() >= 100


def test_struct_layouts_match_header():
    assert ctypes.sizeof(N.ConvDesc) == 10 * 4
    assert ctypes.sizeof(N.Tile) == 9 * 4
    assert N.LaunchInfo.flops.offset % 8 == 0


def test_query_legal_and_illegal_projections():
    ok = query((1, 64, 56, 56), (64, 64, 3, 3), 1, 1, "CHW", TileConfig(56, 4, 64, 32768, 7, 4, 8))
    assert ok["rc"] == 0 and ok["legal"] == 1
    assert (ok["grid_x"], ok["grid_y"], ok["grid_z"]) == (1, 14, 1)
    assert ok["block_threads"] == 224 and ok["p"] == ok["q"] == 56
    assert ok["flops"] == 231211008
    assert "tma" in ok["reason"]          # NCHW with 16-byte strides: TMA ring
    assert 1 <= ok["stages"] <= 4 and ok["channel_chunk"] >= 1
    # resident set above s_b -> ScheduleError class (rc 3)
    bad = query((1, 64, 56, 56), (64, 64, 3, 3), 1, 1, "CHW", TileConfig(56, 4, 64, 2000, 7, 4, 8))
    assert bad["rc"] == 3 and "resident" in bad["reason"]
    # ragged tile refused like the model refuses it
    rag = query((1, 64, 56, 56), (64, 64, 3, 3), 1, 1, "CHW", TileConfig(5, 4, 64, 32768, 5, 4, 8))
    assert rag["rc"] == 3 and "divide" in rag["reason"]
    # 14x14 maps: 56-byte rows cannot be a TMA box -> cp.async ring
    small = query((1, 256, 14, 14), (256, 256, 3, 3), 1, 1, "CHW",
                  TileConfig(14, 14, 32, 16384, 2, 7, 16))
    assert small["rc"] == 0 and "cp.async" in small["reason"]


def test_winograd_projection():
    ok = query((1, 64, 56, 56), (64, 64, 3, 3), 1, 1, "CHW",
               TileConfig(8, 8, 32, 32768, 8, 8, 4, e=2), "winograd")
    assert ok["rc"] == 0 and ok["block_threads"] == 256
    assert ok["flops"] == 2 * 16 * 28 * 28 * 64 * 64
    stride2 = query((1, 64, 56, 56), (64, 64, 3, 3), 2, 1, "CHW",
                    TileConfig(4, 4, 32, 32768, 2, 2, 4, e=2), "winograd")
    assert stride2["rc"] == 3 and "stride" in stride2["reason"]


def test_default_tiles_are_legal():
    lib = N.lib()
    for n, c, h, k, st in [(8, 64, 56, 64, 1), (4, 256, 14, 256, 1), (2, 128, 28, 128, 2)]:
        d = N.make_desc(n, c, h, h, k, 3, 3, st, 1, 0)
        t = N.Tile()
        assert lib.convio_default_tile(ctypes.byref(d), 0, 0, ctypes.byref(t)) == 0
        rc, info = N.query(d, t, N.ALG_DIRECT)
        assert rc == 0 and info["legal"] == 1


@pytest.mark.parametrize("e", [2, 4])
def test_kernel_transform_matrices_match_oracle(e):
    m = e + 2
    at = np.zeros(e * m, np.float32)
    g = np.zeros(m * 3, np.float32)
    bt = np.zeros(m * m, np.float32)
    rc = N.lib().convio_winograd_matrices(e, 3, at.ctypes.data, g.ctypes.data, bt.ctypes.data)
    assert rc == 0
    mats = wm.matrices_float(e, 3)
    assert np.array_equal(at.reshape(e, m), mats["AT"].astype(np.float32))
    assert np.allclose(g.reshape(m, 3), mats["G"], rtol=0, atol=1e-7)
    assert np.array_equal(bt.reshape(m, m), mats["BT"].astype(np.float32))


def test_error_codes_map_to_reference_exceptions():
    from paper_2012_15667_b200.dataflow import ScheduleError, InfeasibleTileError
    lib = N.lib()
    d = N.make_desc(1, 4, 8, 8, 4, 3, 3, 1, 1, 0)
    info = N.LaunchInfo()
    rc = lib.convio_query(ctypes.byref(d), ctypes.byref(N.make_tile(TileConfig(3, 8, 4, 4096))),
                          0, ctypes.byref(info))
    with pytest.raises(ScheduleError):
        N.check(rc)
    rc = lib.convio_query(ctypes.byref(d), ctypes.byref(N.make_tile(TileConfig(8, 8, 4, 8192, 1, 1, 4))),
                          0, ctypes.byref(info))
    with pytest.raises(InfeasibleTileError):
        N.check(rc)
    bad = N.make_desc(0, 4, 8, 8, 4, 3, 3, 1, 1, 0)
    rc = lib.convio_query(ctypes.byref(bad), ctypes.byref(N.make_tile(TileConfig(8, 8, 4, 8192))),
                          0, ctypes.byref(info))
    with pytest.raises(ValueError):
        N.check(rc)


def test_no_cpu_fallback_for_conv():
    torch = pytest.importorskip("torch")
    from paper_2012_15667_b200 import conv as C
    x = torch.zeros(1, 2, 4, 4)
    w = torch.zeros(2, 2, 3, 3)
    with pytest.raises(ValueError, match="CUDA"):
        C.conv_direct(x, w, padding=1)
    with pytest.raises(ValueError, match="CUDA"):
        C.conv_winograd(x, w, e=2, padding=1)


def test_tensor_core_projections_plan_pairs_split_k_and_chunks():
    """Host-side planning of the tcgen05 kernels (no launch): the CTA-pair tile
    kinds, the pair split-K decision (148 SMs without a device) and the
    tensor-core Winograd chunking."""
    hwc = "HWC"
    # ResNet-50 res5 stride 2 at batch 256: 98 pair items on 74 pairs -> split K
    s2 = query((256, 512, 14, 14), (512, 512, 3, 3), 2, 1, hwc,
               TileConfig(1, 1, 256, 32768, 1, 1, 2, layout=hwc), "igemm_3xtf32")
    assert s2["rc"] == 0 and "CTA pair" in s2["reason"] and "split-K" in s2["reason"]
    # res4 stride 2: 196 items = 2.65 rounds -> the last 48 tile items split 3 ways
    # (2 x 36 + 2 x 12 k-blocks per pair instead of 3 x 36)
    s4 = query((256, 256, 28, 28), (256, 256, 3, 3), 2, 1, hwc,
               TileConfig(1, 2, 256, 32768, 1, 1, 2, layout=hwc), "igemm_3xtf32")
    assert s4["rc"] == 0 and "split-K" in s4["reason"]
    # res3 A-in-TMEM at batch 256: 784 items = 10.6 rounds of 18 k-blocks; a split tail
    # saves < 5 % -> whole tiles
    s3 = query((256, 128, 28, 28), (128, 128, 3, 3), 1, 1, hwc,
               TileConfig(1, 4, 128, 32768, 1, 1, 4, layout=hwc), "igemm_3xf16")
    assert s3["rc"] == 0 and "split-K" not in s3["reason"]
    # halo + fold tiles never split
    fold = query((4, 64, 56, 56), (64, 64, 3, 3), 1, 1, hwc,
                 TileConfig(30, 4, 64, 32768, 2, 1, 2, layout=hwc), "igemm_3xtf32")
    assert fold["rc"] == 0 and "3 taps per MMA" in fold["reason"] and "split-K" not in fold["reason"]
    tsa = query((64, 128, 28, 28), (128, 128, 3, 3), 1, 1, hwc,
                TileConfig(4, 1, 128, 32768, 1, 1, 4, layout=hwc), "igemm_3xtf32")
    assert tsa["rc"] == 0 and "A in TMEM" in tsa["reason"]
    bad = query((64, 128, 28, 28), (256, 128, 3, 3), 1, 1, hwc,
                TileConfig(4, 1, 256, 32768, 1, 1, 4, layout=hwc), "igemm_3xtf32")
    assert bad["rc"] == 3
    # Winograd chunk budget 16 KB x s_b: 9 images of 56x56x64 F(4,3) at s_b 2048,
    # the whole batch at s_b 32768
    w2 = query((24, 64, 56, 56), (64, 64, 3, 3), 1, 1, hwc,
               TileConfig(4, 4, 64, 2048, 1, 1, 2, layout=hwc, e=4), "winograd_tc_3xtf32")
    assert w2["rc"] == 0 and "chunk 9 img" in w2["reason"]
    w32 = query((24, 64, 56, 56), (64, 64, 3, 3), 1, 1, hwc,
                TileConfig(4, 4, 64, 32768, 1, 1, 4, layout=hwc, e=4), "winograd_tc_3xtf32")
    assert w32["rc"] == 0 and "chunk 24 img" in w32["reason"]
    # A in TMEM needs 3xTF32 and z <= 128
    wbad = query((24, 64, 56, 56), (256, 64, 3, 3), 1, 1, hwc,
                 TileConfig(4, 4, 256, 32768, 1, 1, 4, layout=hwc, e=4), "winograd_tc_3xtf32")
    assert wbad["rc"] == 3


def test_winograd_3xf16_projection():
    hwc = "HWC"
    ok = query((8, 128, 28, 28), (128, 128, 3, 3), 1, 1, hwc,
               TileConfig(4, 4, 128, 32768, 1, 1, 2, layout=hwc, e=4), "winograd_tc_3xf16")
    assert ok["rc"] == 0
    single = query((8, 128, 28, 28), (128, 128, 3, 3), 1, 1, hwc,
                   TileConfig(4, 4, 128, 32768, 1, 1, 1, layout=hwc, e=4), "winograd_tc_3xf16")
    assert single["rc"] == 3 and "pair" in single["reason"]
    odd = query((8, 96, 28, 28), (128, 96, 3, 3), 1, 1, hwc,
                TileConfig(4, 4, 128, 32768, 1, 1, 2, layout=hwc, e=4), "winograd_tc_3xf16")
    assert odd["rc"] == 3
