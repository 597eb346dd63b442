"""3xF16 tcgen05 implicit GEMM (CONVIO_PREC_3XF16 through convio_conv_igemm): the
activations are TMA-staged as fp32 and split on chip into power-of-two-scaled fp16
hi / lo planes (one scale per tensor), the filter into fp16 planes with one scale
per output channel; 3 kind::f16 MMAs per k-step.  Parity against the float64
oracle (restating reference pkg/src/convio/dag.py:247-285) at the 3xTF32 bound."""

import numpy as np
import pytest
import torch

from oracle import conv_oracle as co
from paper_2012_15667_b200 import TileConfig, InfeasibleTileError
from paper_2012_15667_b200 import conv as C

import os
import sys
sys.path.insert(0, os.path.dirname(__file__))
from tolerances import tol_3xtf32  # noqa: E402

pytestmark = pytest.mark.gpu


def _inputs(n, c, h, w, k, r=3, seed=0):
    g = np.random.default_rng(seed)
    x = g.uniform(-1, 1, (n, c, h, w)).astype(np.float32)
    wt = (np.random.default_rng(seed + 1).uniform(-1, 1, (k, c, r, r)) / np.sqrt(c * r * r)).astype(np.float32)
    return x, wt


def _hwc(a):
    return C.to_layout(torch.from_numpy(a).cuda(), "HWC")


CASES = [
    # (n, c, h, k, stride, tile, what)
    (2, 64, 56, 64, 1, TileConfig(28, 4, 64, 32768, 1, 1, 2, layout="HWC"), "pair z=64"),
    (3, 128, 14, 256, 1, TileConfig(14, 7, 256, 32768, 1, 1, 2, layout="HWC"), "pair z=256"),
    (3, 64, 28, 128, 2, TileConfig(14, 7, 128, 32768, 1, 1, 2, layout="HWC"), "stride 2"),
    (5, 64, 7, 64, 1, TileConfig(7, 7, 64, 32768, 1, 1, 2, layout="HWC"), "odd block count"),
    (4, 128, 28, 256, 2, TileConfig(14, 7, 256, 32768, 1, 1, 2, layout="HWC"), "stride 2 z=256"),
    (2, 64, 56, 128, 1, TileConfig(14, 8, 128, 32768, 2, 1, 2, layout="HWC"), "halo"),
    (3, 128, 28, 256, 1, TileConfig(14, 8, 256, 32768, 2, 1, 2, layout="HWC"), "halo ragged"),
    (2, 128, 14, 128, 1, TileConfig(14, 8, 128, 32768, 2, 1, 2, layout="HWC"), "halo ragged y"),
    (2, 64, 56, 64, 1, TileConfig(14, 8, 64, 32768, 2, 1, 2, layout="HWC"), "fold (3 taps per MMA)"),
    (3, 64, 28, 64, 1, TileConfig(30, 4, 64, 32768, 2, 1, 2, layout="HWC"), "fold 30x4"),
    (16, 512, 14, 256, 2, TileConfig(1, 1, 256, 32768, 1, 1, 2, layout="HWC"), "split-K"),
    # n_zt = 4: the split activations in tensor memory (tcgen05.mma A operand from TMEM)
    (3, 128, 28, 128, 1, TileConfig(1, 1, 128, 32768, 1, 1, 4, layout="HWC"), "tsa z=128"),
    (2, 64, 56, 64, 1, TileConfig(28, 4, 64, 32768, 1, 1, 4, layout="HWC"), "tsa z=64"),
    (3, 256, 14, 256, 1, TileConfig(1, 1, 256, 32768, 1, 1, 4, layout="HWC"), "tsa z=256 (one accumulator)"),
    (3, 128, 28, 128, 2, TileConfig(2, 1, 128, 32768, 1, 1, 4, layout="HWC"), "tsa stride 2"),
    (16, 512, 14, 256, 2, TileConfig(1, 1, 256, 32768, 1, 1, 4, layout="HWC"), "tsa split-K"),
    # (2, 1, 4): halo footprint, the converters shift each tap's rows into TMEM
    (2, 64, 56, 128, 1, TileConfig(14, 8, 128, 32768, 2, 1, 4, layout="HWC"), "halo tsa z=128"),
    (3, 128, 28, 128, 1, TileConfig(30, 4, 128, 32768, 2, 1, 4, layout="HWC"), "halo tsa 30x4 ragged x"),
    (3, 128, 28, 256, 1, TileConfig(14, 8, 256, 32768, 2, 1, 4, layout="HWC"), "halo tsa z=256 ragged y"),
    (2, 128, 14, 64, 1, TileConfig(14, 8, 64, 32768, 2, 1, 4, layout="HWC"), "halo tsa z=64"),
    (2, 64, 56, 64, 1, TileConfig(14, 8, 64, 32768, 2, 1, 4, layout="HWC"), "fold tsa resident filter"),
    (3, 128, 28, 64, 1, TileConfig(30, 4, 64, 32768, 2, 1, 4, layout="HWC"), "fold tsa 30x4 2 channel blocks"),
    # (1, 1, 8): exact x * y * imgs blocks, the footprint gathered into TMEM tap by tap
    (10, 128, 28, 128, 1, TileConfig(4, 4, 128, 32768, 1, 1, 8, layout="HWC"), "gather 4x4 x 8 img, ragged image group"),
    (2, 64, 56, 128, 1, TileConfig(8, 8, 128, 32768, 1, 1, 8, layout="HWC"), "gather 8x8 x 2 img"),
    (4, 256, 14, 256, 1, TileConfig(2, 2, 256, 32768, 1, 1, 8, layout="HWC"), "gather 2x2 x 32 img z=256"),
    (4, 64, 28, 128, 2, TileConfig(2, 2, 128, 32768, 1, 1, 8, layout="HWC"), "gather stride 2"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[-1] for c in CASES])
def test_igemm_3xf16_matches_oracle(case):
    n, c, h, k, stride, tile, what = case
    x, wt = _inputs(n, c, h, h, k)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    info = C.query(x.shape, wt.shape, stride, 1, "HWC", tile, "igemm_3xf16")
    assert info["rc"] == 0, info
    if what.startswith("fold"):
        assert "3 taps per MMA" in info["reason"], info
    if what.endswith("split-K"):
        assert "split-K" in info["reason"], info
    if what.startswith("tsa"):
        assert "A in TMEM" in info["reason"], info
    if "halo tsa" in what or "fold tsa" in what:
        assert "shifted into TMEM" in info["reason"], info
    if what.startswith("gather"):
        assert "gathered into TMEM" in info["reason"], info
    if "resident" in what:
        assert "resident filter" in info["reason"], info
    y = C.conv_igemm(_hwc(x), torch.from_numpy(wt).cuda(), padding=1, stride=stride, tile=tile,
                     precision="3xf16", bias=torch.from_numpy(b).cuda())
    ref = co.direct_conv(x, wt, stride, 1) + b[None, :, None, None]
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= tol_3xtf32(c), err
    assert err > 0.0


def test_igemm_3xf16_packed_filter_and_relu_match():
    x, wt = _inputs(2, 128, 28, 28, 128)
    tile = TileConfig(14, 8, 128, 32768, 2, 1, 2, layout="HWC")
    w = torch.from_numpy(wt).cuda()
    wp = C.pack_filter_igemm_f16x3(w)
    y1 = C.conv_igemm(_hwc(x), w, padding=1, tile=tile, precision="3xf16", relu=True)
    y2 = C.conv_igemm(_hwc(x), w, padding=1, tile=tile, precision="3xf16", relu=True, w_packed=wp)
    assert torch.equal(y1, y2)
    ref = np.maximum(co.direct_conv(x, wt, 1, 1), 0)
    assert co.rel_err(y1.contiguous().cpu().numpy(), ref) <= tol_3xtf32(128)


@pytest.mark.parametrize("sx,sw", [(-60, -60), (-70, -50), (60, 60), (-70, 60), (20, 0)],
                         ids=["x2^-60,w2^-60", "x2^-70,w2^-50", "x2^60,w2^60", "x2^-70,w2^60", "x2^20"])
def test_igemm_3xf16_extreme_operand_scales(sx, sw):
    """Tensor / channel exponents whose sum passes pow2f's range: unscaled with two
    exact multiplies, so only the split's relative error remains."""
    x, wt = _inputs(2, 64, 28, 28, 128)
    x = x * np.float32(2.0 ** sx)
    wt = wt * np.float32(2.0 ** sw)
    for tile in (TileConfig(14, 7, 128, 32768, 1, 1, 2, layout="HWC"),
                 TileConfig(14, 8, 128, 32768, 2, 1, 2, layout="HWC"),
                 TileConfig(14, 8, 128, 32768, 2, 1, 4, layout="HWC")):
        y = C.conv_igemm(_hwc(x), torch.from_numpy(wt).cuda(), padding=1, tile=tile, precision="3xf16")
        err = co.rel_err(y.contiguous().cpu().numpy(), co.direct_conv(x, wt, 1, 1))
        assert np.isfinite(err) and err <= tol_3xtf32(64), (tile, err)


def test_igemm_3xf16_rejects_single_cta_and_c_not_multiple_of_64():
    x, wt = _inputs(1, 64, 14, 14, 64)
    with pytest.raises(InfeasibleTileError):
        C.conv_igemm(_hwc(x), torch.from_numpy(wt).cuda(), padding=1, precision="3xf16",
                     tile=TileConfig(14, 7, 64, 32768, 1, 1, 1, layout="HWC"))
    x, wt = _inputs(1, 32, 14, 14, 64)
    with pytest.raises(InfeasibleTileError):
        C.conv_igemm(_hwc(x), torch.from_numpy(wt).cuda(), padding=1, precision="3xf16",
                     tile=TileConfig(14, 7, 64, 32768, 1, 1, 2, layout="HWC"))


@pytest.mark.parametrize("tile", [TileConfig(14, 7, 128, 32768, 1, 1, 2, layout="HWC"),
                                  TileConfig(2, 1, 128, 32768, 1, 1, 4, layout="HWC"),
                                  TileConfig(14, 8, 128, 32768, 2, 1, 4, layout="HWC")],
                         ids=["pair", "tsa", "halo tsa"])
def test_igemm_3xf16_speculative_scale(tile):
    """The activation scale is speculated from the previous call on the same workspace
    (state in its first bytes) and checked on the device against this call's max |x|:
    the same data reuses it; a 2^20 jump (fp16 overflow) or a 2^-20 drop (lost bits)
    makes the checking launch redo the conv with the exact scale.  Every call must match
    the oracle, and the state must end up holding the last call's max |x|."""
    x, wt = _inputs(2, 64, 28, 28, 128)
    w = torch.from_numpy(wt).cuda()
    info = C.query(x.shape, wt.shape, 1, 1, "HWC", tile, "igemm_3xf16")
    assert info["rc"] == 0, info
    ws = torch.full((info["workspace_bytes"],), 0x7f, dtype=torch.uint8, device="cuda")   # foreign bytes
    ref = co.direct_conv(x, wt, 1, 1)
    for scale in (1.0, 1.0, 2.0 ** 20, 2.0 ** 20, 2.0 ** -20, 1.0, 3.0):
        xs = (x * np.float32(scale)).astype(np.float32)
        y = C.conv_igemm(_hwc(xs), w, padding=1, tile=tile, precision="3xf16", workspace=ws)
        err = co.rel_err(y.contiguous().cpu().numpy(), ref * scale)
        assert np.isfinite(err) and err <= tol_3xtf32(64), (scale, err)
        state = ws[:8].view(torch.int32).cpu().numpy()
        assert state[0] == np.float32(np.abs(xs).max()).view(np.int32), (scale, state)
        assert state[1] == state[0] ^ 0x5CA1AB1E


def test_batched_filter_packing_matches_per_filter_packing():
    """convio_pack_filters_igemm_f16x3_batched (a step's 3xF16 filter prep in one launch)
    writes exactly what the per-filter packing writes, and the runner uses it."""
    from paper_2012_15667_b200 import runner as R
    g = torch.Generator(device="cuda").manual_seed(5)
    shapes = [(64, 64, 3), (128, 64, 3), (256, 128, 3), (512, 256, 1), (64, 128, 3), (64, 34, 3)]
    ws = [torch.rand((k, c, r, r), device="cuda", generator=g) - 0.5 for k, c, r in shapes]
    singles = [C.pack_filter_igemm_f16x3(w) for w in ws]
    import ctypes
    from paper_2012_15667_b200 import _native as N
    outs = [torch.empty_like(s) for s in singles]
    descs = (N.ConvDesc * len(ws))(*[N.make_desc(1, w.shape[1], 8, 8, w.shape[0], w.shape[2], w.shape[3], 1, 0, 2)
                                     for w in ws])
    rc = N.lib().convio_pack_filters_igemm_f16x3_batched(
        len(ws), descs, (ctypes.c_void_p * len(ws))(*[w.data_ptr() for w in ws]),
        (ctypes.c_void_p * len(ws))(*[o.data_ptr() for o in outs]), None)
    assert rc == 0, N.last_error()
    torch.cuda.synchronize()
    for s1, o in zip(singles, outs):
        assert torch.equal(s1, o)
    # a filter row over the shared-memory staging limit (C*R*S > 12288): the unstaged form
    big = [torch.rand((32, 2048, 3, 3), device="cuda", generator=g) - 0.5]
    ref, out = C.pack_filter_igemm_f16x3(big[0]), None
    out = torch.empty_like(ref)
    rc = N.lib().convio_pack_filters_igemm_f16x3_batched(
        1, (N.ConvDesc * 1)(N.make_desc(1, 2048, 8, 8, 32, 3, 3, 1, 0, 2)),
        (ctypes.c_void_p * 1)(big[0].data_ptr()), (ctypes.c_void_p * 1)(out.data_ptr()), None)
    assert rc == 0, N.last_error()
    used = 4 * 32 * 2048 * 9 + 4 * 32   # hi / lo planes, then the 32 column exponents (no tail padding)
    assert torch.equal(ref[:used], out[:used])
    # the runner's step prep: 3xF16 layers batched, the others one by one
    specs = [s for s in R.WORKLOADS["resnet50"]][:4]
    layers = [R.ConvLayer(s, R.make_weights(s, torch.device("cuda"), i),
                          {"algorithm": "igemm_3xf16", "tile": TileConfig(2, 2, s.k if s.k <= 256 else 256, 32768,
                                                                          1, 1, 2, layout="HWC"), "e": None})
              for i, s in enumerate(specs)]
    assert R.prepare_layers(layers, torch.device("cuda")) == 1
    for l in layers:
        ref = C.pack_filter_igemm_f16x3(l.weight)
        assert torch.equal(l._ws.view(torch.uint8)[:ref.numel()], ref)


@pytest.mark.parametrize("e", [2, 4])
@pytest.mark.parametrize("prec", ["3xf16", "3xtf32"])
def test_batched_winograd_filter_transform_matches_per_filter(prec, e):
    """convio_winograd_filter_transform_tc_batched == the per-filter transform, bit for bit.
    For 3xF16 the batched form is one fused launch (transform + split, no fp32 U): the
    hi / lo planes and exponents the GEMM reads must equal the two-kernel per-filter
    path's; the fp32 U region ahead of them is scratch the fused kernel never writes."""
    g = torch.Generator(device="cuda").manual_seed(9)
    shapes = [(256, 128), (512, 512), (128, 64)]
    ws = [torch.rand((k, c, 3, 3), device="cuda", generator=g) - 0.5 for k, c in shapes]
    ws[1][:7] *= 2.0 ** -30   # rows whose exponents differ widely from the rest
    singles = [C.winograd_filter_transform_tc(w, e, prec) for w in ws]
    import ctypes
    from paper_2012_15667_b200 import _native as N
    outs = [torch.zeros_like(s) for s in singles]
    descs = (N.ConvDesc * len(ws))(*[N.make_desc(1, w.shape[1], 8, 8, w.shape[0], 3, 3, 1, 0, 2) for w in ws])
    rc = N.lib().convio_winograd_filter_transform_tc_batched(
        len(ws), descs, e, N.PRECISIONS[prec], (ctypes.c_void_p * len(ws))(*[w.data_ptr() for w in ws]),
        (ctypes.c_void_p * len(ws))(*[o.data_ptr() for o in outs]), None)
    assert rc == 0, N.last_error()
    assert C.last_launch_count() == 1
    torch.cuda.synchronize()
    m = e + 2
    for (k, c), s1, o in zip(shapes, singles, outs):
        n = s1.numel() * s1.element_size()
        skip = m * m * k * c * 4 if prec == "3xf16" else 0   # the fp32 U scratch
        assert torch.equal(s1.view(torch.uint8).flatten()[skip:n], o.view(torch.uint8).flatten()[skip:n])


@pytest.mark.parametrize("case", [
    (3, 16, 128, 28, 128, 1, TileConfig(4, 2, 128, 32768, 1, 1, 4, layout="HWC")),  # A in TMEM
    (2, 4, 64, 56, 64, 1, TileConfig(30, 4, 64, 32768, 2, 1, 4, layout="HWC")),     # halo fold
    (4, 32, 256, 14, 256, 1, TileConfig(2, 2, 256, 32768, 1, 1, 2, layout="HWC")),  # pair (+ tail split)
    (2, 32, 128, 28, 128, 2, TileConfig(2, 2, 128, 32768, 1, 1, 4, layout="HWC")),  # stride 2
    (2, 8, 128, 28, 128, 1, TileConfig(4, 4, 128, 32768, 1, 1, 8, layout="HWC")),   # gathered footprint
    (3, 4, 64, 56, 64, 1, TileConfig(30, 4, 64, 32768, 2, 1, 2, layout="HWC")),     # fold, smem A, 3 layers
], ids=["tsa", "fold", "pair", "stride2", "gather", "fold-smem-3"])
def test_grouped_3xf16_conv_matches_per_layer_and_oracle(case):
    """convio_conv_igemm_grouped: G independent layers (own filters and biases) of one
    shape in one launch == G single-layer launches, and the oracle."""
    layers, n, c, hw, k, stride, tile = case
    g = np.random.default_rng(11)
    xs = [g.uniform(-1, 1, (n, c, hw, hw)).astype(np.float32) for _ in range(layers)]
    wts = [(g.uniform(-1, 1, (k, c, 3, 3)) / np.sqrt(c * 9)).astype(np.float32) for _ in range(layers)]
    bs = [g.uniform(-0.2, 0.2, k).astype(np.float32) for _ in range(layers)]
    sb = C.f16x3_slice_bytes(k, c, 3, 3)
    packed = torch.zeros(layers * sb, dtype=torch.uint8, device="cuda")
    for l, wt in enumerate(wts):
        p1 = C.pack_filter_igemm_f16x3(torch.from_numpy(wt).cuda())
        packed[l * sb:l * sb + p1.numel()] = p1
    xg = _hwc(np.concatenate(xs))
    bias = torch.from_numpy(np.concatenate(bs)).cuda()
    yg = C.conv_igemm_grouped(xg, (k, c, 3, 3), packed, layers, sb, padding=1, stride=stride, tile=tile,
                              bias=bias)
    yg = yg.contiguous().cpu().numpy()
    for l in range(layers):
        y1 = C.conv_igemm(_hwc(xs[l]), torch.from_numpy(wts[l]).cuda(), padding=1, stride=stride, tile=tile,
                          precision="3xf16", bias=torch.from_numpy(bs[l]).cuda())
        ref = co.direct_conv(xs[l], wts[l], stride, 1) + bs[l][None, :, None, None]
        got = yg[l * n:(l + 1) * n]
        assert co.rel_err(got, ref) <= tol_3xtf32(c), l
        assert np.abs(got - y1.contiguous().cpu().numpy()).max() <= 1e-5 * np.abs(ref).max(), l
