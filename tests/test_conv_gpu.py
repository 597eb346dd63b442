"""GPU parity: the sm_100a kernels vs the float64 CPU oracle (``oracle/``).

Tolerances (norm-wise max error ``||y - y_ref||_inf / ||y_ref||_inf``):
tests/tolerances.py, each within ~10x of the error measured on a B200.
Every call goes through the C-ABI.
"""

import numpy as np
import pytest
import torch

from oracle import conv_oracle as co
from paper_2012_15667_b200 import TileConfig, ScheduleError, InfeasibleTileError
from paper_2012_15667_b200 import conv as C

pytestmark = pytest.mark.gpu

from tolerances import (TOL_DIRECT, TOL_TF32, TOL_BF16, TOL_WTC, tol_fp32,  # noqa: E402
                        tol_3xtf32, tol_wino)


def _inputs(n, c, h, w, k, r, s, seed=0):
    g = np.random.default_rng(seed)
    x = g.uniform(-1, 1, (n, c, h, w)).astype(np.float32)
    g1 = np.random.default_rng(seed + 1)
    wt = (g1.uniform(-1, 1, (k, c, r, s)) / np.sqrt(c * r * s)).astype(np.float32)
    return x, wt


def _dev(a, layout="CHW"):
    t = torch.from_numpy(a).cuda()
    return C.to_layout(t, layout) if t.dim() == 4 and layout != "CHW" else t


DIRECT_CASES = [
    # (n, c, h, w, k, r, stride, pad, tile)
    (1, 64, 56, 56, 64, 3, 1, 1, TileConfig(56, 4, 64, 32768, 7, 4, 8)),
    (1, 64, 56, 56, 64, 3, 1, 1, TileConfig(8, 8, 32, 16384, 1, 8, 4)),
    (2, 16, 14, 14, 32, 3, 1, 1, TileConfig(14, 2, 32, 8192, 2, 2, 4)),
    (1, 3, 32, 32, 16, 3, 1, 1, TileConfig(32, 4, 16, 8192, 4, 4, 2)),
    (2, 32, 28, 28, 64, 3, 2, 1, TileConfig(14, 2, 16, 8192, 2, 2, 4)),
    (1, 8, 7, 7, 16, 3, 1, 1, TileConfig(7, 7, 16, 4096, 1, 7, 4)),
    (2, 32, 16, 16, 64, 1, 1, 0, TileConfig(16, 4, 64, 16384, 2, 4, 8)),
    (1, 5, 9, 11, 6, 3, 1, 0, None),    # ragged: library default tile / generic path
    (1, 3, 23, 23, 8, 5, 2, 2, None),   # 5x5 stride 2: generic kernel
]


@pytest.mark.parametrize("case", DIRECT_CASES, ids=[str(i) for i in range(len(DIRECT_CASES))])
def test_direct_matches_oracle(case):
    n, c, h, w, k, r, stride, pad, tile = case
    x, wt = _inputs(n, c, h, w, k, r, r)
    y = C.conv_direct(_dev(x), _dev(wt), stride=stride, padding=pad, tile=tile)
    torch.cuda.synchronize()
    ref = co.direct_conv(x, wt, stride, pad)
    assert y.shape == ref.shape
    assert co.rel_err(y.cpu().numpy(), ref) <= TOL_DIRECT


@pytest.mark.parametrize("layout", ["HWC", "CWH"])
def test_direct_layouts(layout):
    x, wt = _inputs(2, 16, 28, 28, 32, 3, 3)
    tile = TileConfig(28, 4, 32, 16384, 7, 4, 4, layout=layout)
    y = C.conv_direct(_dev(x, layout), _dev(wt), stride=1, padding=1, tile=tile)
    assert C.infer_layout(y) == layout
    ref = co.direct_conv(x, wt, 1, 1)
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= TOL_DIRECT


def test_direct_bias_relu_and_packed_filter():
    x, wt = _inputs(1, 32, 14, 14, 16, 3, 3)
    b = np.linspace(-0.5, 0.5, 16).astype(np.float32)
    wp = C.pack_filter_direct(_dev(wt))
    y = C.conv_direct(_dev(x), _dev(wt), padding=1, bias=_dev(b), relu=True, w_packed=wp,
                      tile=TileConfig(14, 2, 16, 8192, 2, 2, 2))
    ref = np.maximum(co.direct_conv(x, wt, 1, 1) + b[None, :, None, None], 0)
    assert co.rel_err(y.cpu().numpy(), ref) <= TOL_DIRECT


def test_direct_illegal_tiles_raise_reference_errors():
    x, wt = _inputs(1, 8, 8, 8, 8, 3, 3)
    with pytest.raises(ScheduleError):      # does not divide the output
        C.conv_direct(_dev(x), _dev(wt), padding=1, tile=TileConfig(3, 8, 8, 4096))
    with pytest.raises(ScheduleError):      # resident set > s_b
        C.conv_direct(_dev(x), _dev(wt), padding=1, tile=TileConfig(8, 8, 8, 64))
    with pytest.raises(InfeasibleTileError):  # micro-tile 8x8x1 is not compiled
        C.conv_direct(_dev(x), _dev(wt), padding=1, tile=TileConfig(8, 8, 8, 8192, 1, 1, 8))


WINO_CASES = [
    (1, 64, 56, 56, 64, 2, TileConfig(8, 8, 32, 32768, 8, 8, 4, e=2)),
    (1, 64, 56, 56, 64, 4, TileConfig(8, 8, 32, 32768, 4, 8, 4, e=4)),
    (2, 16, 14, 14, 32, 2, TileConfig(14, 14, 8, 32768, 7, 7, 8, e=2)),
    (2, 16, 16, 16, 16, 4, TileConfig(16, 8, 16, 32768, 4, 8, 4, e=4)),
    (1, 3, 12, 12, 8, 2, None),
    (1, 32, 28, 28, 32, 4, None),
]


@pytest.mark.parametrize("case", WINO_CASES, ids=[str(i) for i in range(len(WINO_CASES))])
def test_winograd_matches_oracle(case):
    n, c, h, w, k, e, tile = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    y = C.conv_winograd(_dev(x), _dev(wt), e=e, padding=1, tile=tile)
    ref = co.direct_conv(x, wt, 1, 1)
    assert co.rel_err(y.cpu().numpy(), ref) <= tol_wino(e, c)
    # and against the Winograd oracle itself (same transform matrices)
    assert co.rel_err(y.cpu().numpy(), co.winograd_conv(x, wt, e, 1)) <= tol_wino(e, c)


def test_winograd_filter_transform_matches_oracle():
    from oracle import winograd_mats as wm
    _, wt = _inputs(1, 8, 4, 4, 16, 3, 3)
    for e in (2, 4):
        u = C.winograd_filter_transform(_dev(wt), e).cpu().numpy()
        g = wm.matrices_float(e, 3)["G"]
        ref = np.einsum("ij,kcjl,ml->imkc", g, wt.astype(np.float64), g)
        m = e + 2
        ref = ref.reshape(m * m, 16, 8).transpose(0, 2, 1)
        assert np.max(np.abs(u - ref)) <= 1e-6 * max(1.0, np.max(np.abs(ref)))


IGEMM_CASES = [
    (2, 64, 56, 56, 64, TileConfig(28, 4, 64, 32768, 1, 1, 1, layout="HWC")),
    (2, 64, 56, 56, 128, TileConfig(14, 8, 128, 32768, 1, 1, 1, layout="HWC")),
    (3, 128, 14, 14, 256, TileConfig(14, 7, 256, 32768, 1, 1, 1, layout="HWC")),
    (5, 32, 7, 7, 64, TileConfig(7, 7, 64, 32768, 1, 1, 1, layout="HWC")),   # 2 images / tile
]


@pytest.mark.parametrize("case", IGEMM_CASES, ids=[str(i) for i in range(len(IGEMM_CASES))])
def test_igemm_tcgen05_tf32_matches_oracle(case):
    n, c, h, w, k, tile = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    y = C.conv_igemm_tf32(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, bias=_dev(b))
    ref = co.direct_conv(x, wt, 1, 1) + b[None, :, None, None]
    assert C.infer_layout(y) == "HWC"
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= TOL_TF32


def test_igemm_tcgen05_tf32_stride2():
    x, wt = _inputs(2, 64, 28, 28, 128, 3, 3)
    tile = TileConfig(14, 7, 128, 32768, 1, 1, 1, layout="HWC")
    y = C.conv_igemm_tf32(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, stride=2)
    ref = co.direct_conv(x, wt, 2, 1)
    assert y.shape == ref.shape
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= TOL_TF32


SPLIT_CASES = [
    (2, 64, 56, 56, 64, 1, TileConfig(28, 4, 64, 32768, 1, 1, 1, layout="HWC")),
    (2, 128, 14, 14, 256, 1, TileConfig(14, 7, 256, 32768, 1, 1, 1, layout="HWC")),
    (2, 256, 14, 14, 128, 1, TileConfig(14, 7, 128, 32768, 1, 1, 1, layout="HWC")),
    (3, 64, 7, 7, 64, 1, TileConfig(7, 7, 64, 32768, 1, 1, 1, layout="HWC")),
    (2, 128, 28, 28, 128, 2, TileConfig(14, 7, 128, 32768, 1, 1, 1, layout="HWC")),
]


@pytest.mark.parametrize("case", SPLIT_CASES, ids=[str(i) for i in range(len(SPLIT_CASES))])
def test_igemm_tcgen05_3xtf32_meets_fp32_tolerance(case):
    n, c, h, w, k, stride, tile = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    y = C.conv_igemm_tf32(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, stride=stride, split=True)
    ref = co.direct_conv(x, wt, stride, 1)
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= tol_fp32(c)
    # the FFMA direct path on the same layer for comparison: same tolerance class
    yd = C.conv_direct(_dev(x), _dev(wt), stride=stride, padding=1)
    assert co.rel_err(yd.cpu().numpy(), ref) <= tol_fp32(c)


@pytest.mark.parametrize("c", [256, 512])
def test_direct_fp32_error_at_long_reductions(c):
    x, wt = _inputs(1, c, 14, 14, 64, 3, 3)
    y = C.conv_direct(_dev(x), _dev(wt), padding=1, tile=TileConfig(14, 14, 32, 16384, 2, 7, 4))
    assert co.rel_err(y.cpu().numpy(), co.direct_conv(x, wt, 1, 1)) <= tol_fp32(c)


# ---- BF16 tcgen05 implicit GEMM (kind::f16) -------------------------------------

BF16_CASES = [
    (2, 64, 56, 56, 64, 1, TileConfig(28, 4, 64, 32768, 1, 1, 1, layout="HWC")),
    (2, 128, 28, 28, 256, 2, TileConfig(14, 7, 256, 32768, 1, 1, 1, layout="HWC")),
    (5, 128, 7, 7, 128, 1, TileConfig(7, 7, 128, 16384, 1, 1, 1, layout="HWC")),
]


@pytest.mark.parametrize("case", BF16_CASES, ids=[str(i) for i in range(len(BF16_CASES))])
def test_igemm_tcgen05_bf16_matches_oracle(case):
    n, c, h, w, k, stride, tile = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    y = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, stride=stride, tile=tile,
                     precision="bf16", bias=_dev(b), relu=True)
    ref = np.maximum(co.direct_conv(x, wt, stride, 1) + b[None, :, None, None], 0)
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= TOL_BF16
    assert err > 1e-6   # really computed at bf16 (not a silent fp32 path)
    # pre-packed bf16 filter gives the same result
    wp = C.pack_filter_igemm_bf16(_dev(wt))
    assert wp.dtype == torch.bfloat16
    y2 = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, stride=stride, tile=tile,
                      precision="bf16", bias=_dev(b), relu=True, w_packed=wp)
    assert torch.equal(y, y2)


PAIR_CASES = [
    # (n, c, h, w, k, stride, precision, tile) -- n_zt = 2: persistent CTA pair
    (2, 64, 56, 56, 64, 1, "3xtf32", TileConfig(28, 4, 64, 32768, 1, 1, 2, layout="HWC")),
    (3, 128, 14, 14, 256, 1, "3xtf32", TileConfig(14, 7, 256, 32768, 1, 1, 2, layout="HWC")),
    (3, 64, 28, 28, 128, 2, "3xtf32", TileConfig(14, 7, 128, 32768, 1, 1, 2, layout="HWC")),
    (5, 32, 7, 7, 64, 1, "tf32", TileConfig(7, 7, 64, 32768, 1, 1, 2, layout="HWC")),  # odd block count
    (3, 128, 14, 14, 256, 1, "tf32", TileConfig(14, 7, 256, 32768, 1, 1, 2, layout="HWC")),
    (4, 128, 28, 28, 256, 2, "bf16", TileConfig(14, 7, 256, 32768, 1, 1, 2, layout="HWC")),
    (1, 64, 14, 14, 128, 1, "bf16", TileConfig(14, 2, 128, 32768, 1, 1, 2, layout="HWC")),  # 7 blocks
    # n_zt = 4: 3xTF32 pair with the A operand (hi / lo) in tensor memory
    (2, 64, 56, 56, 64, 1, "3xtf32", TileConfig(8, 1, 64, 32768, 1, 1, 4, layout="HWC")),
    (3, 128, 28, 28, 128, 1, "3xtf32", TileConfig(4, 1, 128, 32768, 1, 1, 4, layout="HWC")),
    (3, 256, 7, 7, 128, 1, "3xtf32", TileConfig(1, 1, 128, 32768, 1, 1, 4, layout="HWC")),
    (2, 64, 28, 28, 128, 2, "3xtf32", TileConfig(14, 7, 128, 32768, 1, 1, 4, layout="HWC")),
]
TOL_PREC = {"tf32": TOL_TF32, "bf16": TOL_BF16}


@pytest.mark.parametrize("case", PAIR_CASES, ids=[str(i) for i in range(len(PAIR_CASES))])
def test_igemm_cta_pair_matches_oracle_and_single_cta(case):
    n, c, h, w, k, stride, prec, tile = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    y = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, stride=stride, tile=tile, precision=prec,
                     bias=_dev(b))
    ref = co.direct_conv(x, wt, stride, 1) + b[None, :, None, None]
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= TOL_PREC.get(prec, tol_3xtf32(c)), err
    single = TileConfig(tile.x, tile.y, tile.z, tile.s_b, 1, 1, 1, layout="HWC")
    if tile.n_zt == 4:
        assert "A in TMEM" in C.query(x.shape, wt.shape, stride, 1, "HWC", tile,
                                      f"igemm_{prec}")["reason"]
    y1 = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, stride=stride, tile=single,
                      precision=prec, bias=_dev(b))
    # same products; the summation order differs by MMA-internal order and, on small
    # grids, by the single-CTA kernel's split-K partial sums
    assert co.rel_err(y.contiguous().cpu().numpy(), y1.contiguous().cpu().numpy()) <= 2 * tol_3xtf32(c)


HALO_CASES = [
    # (n, c, h, w, k, precision, tile) -- n_xt = 2: footprint staged once per channel
    # block, taps = row offsets into it (stride 1, pair kernel)
    (2, 64, 56, 56, 64, "3xtf32", TileConfig(14, 8, 64, 32768, 2, 1, 2, layout="HWC")),
    (2, 64, 56, 56, 128, "tf32", TileConfig(6, 16, 128, 32768, 2, 1, 2, layout="HWC")),
    (3, 128, 28, 28, 256, "3xtf32", TileConfig(14, 8, 256, 32768, 2, 1, 2, layout="HWC")),  # ragged
    (2, 128, 14, 14, 128, "bf16", TileConfig(14, 8, 128, 32768, 2, 1, 2, layout="HWC")),   # ragged y
    (2, 32, 20, 20, 64, "tf32", TileConfig(6, 16, 64, 32768, 2, 1, 2, layout="HWC")),      # ragged x, y
    # z = K = 64: the 3 horizontal taps folded into one MMA of N = 192
    (2, 64, 56, 56, 64, "bf16", TileConfig(14, 8, 64, 32768, 2, 1, 2, layout="HWC")),
    (3, 64, 28, 28, 64, "tf32", TileConfig(30, 4, 64, 32768, 2, 1, 2, layout="HWC")),
]


@pytest.mark.parametrize("case", HALO_CASES, ids=[str(i) for i in range(len(HALO_CASES))])
def test_igemm_halo_staging_matches_oracle(case):
    n, c, h, w, k, prec, tile = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    info = C.query(x.shape, wt.shape, 1, 1, "HWC", tile, f"igemm_{prec}")
    assert info["rc"] == 0 and "halo" in info["reason"], info
    assert ("3 taps per MMA" in info["reason"]) == (tile.z == k == 64), info
    y = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, precision=prec, bias=_dev(b))
    ref = co.direct_conv(x, wt, 1, 1) + b[None, :, None, None]
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= TOL_PREC.get(prec, tol_3xtf32(c)), err


def test_igemm_generic_entry_matches_split_entry():
    x, wt = _inputs(2, 64, 28, 28, 64, 3, 3)
    tile = TileConfig(14, 4, 64, 16384, 1, 1, 1, layout="HWC")
    # relu: keeps the small grid unsplit (split-K partial sums add in atomic order)
    y1 = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, precision="3xtf32", relu=True)
    y2 = C.conv_igemm_tf32(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, split=True, relu=True)
    assert torch.equal(y1, y2)


def test_igemm_bf16_rejects_c_not_multiple_of_64():
    x, wt = _inputs(1, 32, 14, 14, 64, 3, 3)
    with pytest.raises(InfeasibleTileError):
        C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, precision="bf16",
                     tile=TileConfig(14, 7, 64, 16384, 1, 1, 1, layout="HWC"))


# ---- Winograd with the element-wise GEMMs on tcgen05 ------------------------------
WTC_CASES = [
    # (n, c, h, w, k, e, precision, z)
    (2, 64, 56, 56, 64, 4, "3xtf32", 64),
    (2, 64, 56, 56, 64, 2, "3xtf32", 64),
    (3, 128, 14, 14, 256, 4, "3xtf32", 128),
    (4, 256, 7, 7, 128, 2, "3xtf32", 128),    # ragged: 7 = 3*2 + 1
    (4, 256, 7, 7, 128, 4, "3xtf32", 128),    # ragged: 7 = 4 + 3
    (2, 64, 28, 28, 128, 4, "tf32", 128),
    (2, 64, 28, 28, 128, 2, "tf32", 128),
    (2, 128, 28, 28, 256, 4, "bf16", 256),
    (3, 64, 13, 13, 64, 2, "bf16", 64),
    (2, 128, 14, 14, 256, 4, "3xtf32", 256),
    # precision "fp32": the element-wise GEMMs on the CUDA cores (FFMA, batched)
    (2, 64, 56, 56, 64, 4, "fp32", 64),
    (2, 64, 28, 28, 128, 2, "fp32", 128),
    (4, 256, 7, 7, 128, 4, "fp32", 128),       # ragged, several T blocks per xi
    (10, 64, 56, 56, 64, 2, "fp32", 64),       # two chunks at s_b = 2048 (32 MB)
]
# Reduced-precision Winograd: the operand rounding error is amplified by the
# transforms (F(4,3)'s B^T / G entries up to 5 and 1/6..1/24), so the stated
# tolerances are looser than the direct conv's at the same precision:
#   tf32: F(2,3) 5e-3, F(4,3) 2e-2;  bf16: F(2,3) 5e-2, F(4,3) 1.5e-1.


@pytest.mark.parametrize("case", WTC_CASES, ids=[str(i) for i in range(len(WTC_CASES))])
def test_winograd_tc_matches_oracle(case):
    n, c, h, w, k, e, prec, z = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    nzt = 1 if prec == "fp32" else (2 if n % 2 else 1)
    tile = TileConfig(e, e, z, 2048 if n >= 10 else 16384, 1, 1, nzt, layout="HWC", e=e)
    y = C.conv_winograd_tc(_dev(x, "HWC"), _dev(wt), e=e, padding=1, tile=tile, precision=prec,
                           bias=_dev(b))
    ref = co.direct_conv(x, wt, 1, 1) + b[None, :, None, None]
    assert C.infer_layout(y) == "HWC"
    tol = TOL_WTC.get((prec, e), tol_wino(e, c))
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= tol, (err, tol)


@pytest.mark.parametrize("case", [(3, 128, 28, 28, 128, 4, 128), (2, 64, 56, 56, 64, 2, 64),
                                  (4, 256, 7, 7, 128, 4, 128), (5, 64, 14, 14, 192, 4, 64)])
def test_winograd_tc_a_operand_in_tmem(case):
    """n_zt = 4: the 3xTF32 batched GEMMs on the CTA pair with A (the V tiles) in TMEM."""
    n, c, h, w, k, e, z = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    tile = TileConfig(e, e, z, 16384, 1, 1, 4, layout="HWC", e=e)
    y = C.conv_winograd_tc(_dev(x, "HWC"), _dev(wt), e=e, padding=1, tile=tile, precision="3xtf32",
                           bias=_dev(b), relu=True)
    ref = np.maximum(co.direct_conv(x, wt, 1, 1) + b[None, :, None, None], 0)
    tol = tol_wino(e, c)
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= tol, (err, tol)


def test_winograd_tc_pretransformed_filter_and_relu():
    x, wt = _inputs(2, 64, 28, 28, 64, 3, 3)
    u = C.winograd_filter_transform_tc(_dev(wt), 4, "3xtf32")
    assert tuple(u.shape) == (36, 64, 64)
    y1 = C.conv_winograd_tc(_dev(x, "HWC"), _dev(wt), e=4, relu=True)
    y2 = C.conv_winograd_tc(_dev(x, "HWC"), _dev(wt), e=4, relu=True, u=u)
    assert torch.equal(y1, y2)
    ref = np.maximum(co.direct_conv(x, wt, 1, 1), 0)
    assert co.rel_err(y1.contiguous().cpu().numpy(), ref) <= tol_wino(4, 64)


def test_winograd_tc_filter_transform_matches_oracle():
    from oracle import winograd_mats as wm
    _, wt = _inputs(1, 32, 4, 4, 64, 3, 3)
    for e in (2, 4):
        u = C.winograd_filter_transform_tc(_dev(wt), e, "3xtf32").cpu().numpy()
        g = wm.matrices_float(e, 3)["G"]
        m = e + 2
        ref = np.einsum("ij,kcjl,ml->imkc", g, wt.astype(np.float64), g).reshape(m * m, 64, 32)
        assert np.max(np.abs(u - ref)) <= 1e-6 * max(1.0, np.max(np.abs(ref)))


def test_winograd_tc_chunks_the_batch():
    # s_b = 2048: chunks of V + M <= 32 MB (9 images here): three chunks, same answer
    x, wt = _inputs(24, 64, 56, 56, 64, 3, 3)
    tile = TileConfig(4, 4, 64, 2048, 1, 1, 2, layout="HWC", e=4)
    info = C.query(x.shape, wt.shape, 1, 1, "HWC", tile, algorithm="winograd_tc_3xtf32")
    assert info["rc"] == 0 and "chunk 9 img" in info["reason"], info["reason"]
    y = C.conv_winograd_tc(_dev(x, "HWC"), _dev(wt), e=4, precision="3xtf32", tile=tile)
    assert C.last_launch_count() > 4   # filter + 3 launches per chunk, > 1 chunk
    ref = co.direct_conv(x[:2], wt, 1, 1)
    assert co.rel_err(y[:2].contiguous().cpu().numpy(), ref) <= tol_wino(4, 64)
    ref_last = co.direct_conv(x[-2:], wt, 1, 1)
    assert co.rel_err(y[-2:].contiguous().cpu().numpy(), ref_last) <= tol_wino(4, 64)


# ---- channels-last FP32 direct kernel (stacked pixels, TMA ring) -----------------
NHWC_CASES = [
    # (n, c, h, w, k, stride, tile) -- n_xt*n_yt = 16, n_zt = 16, z in {64, 128}
    (2, 64, 56, 56, 64, 1, TileConfig(28, 4, 64, 32768, 4, 4, 16, layout="HWC")),
    (2, 64, 56, 56, 128, 1, TileConfig(56, 2, 128, 32768, 8, 2, 16, layout="HWC")),
    (3, 128, 14, 14, 128, 1, TileConfig(14, 7, 128, 32768, 1, 1, 1, layout="HWC")),
    (5, 64, 7, 7, 64, 1, TileConfig(7, 7, 64, 16384, 1, 1, 1, layout="HWC")),   # 2 images / block
    (2, 128, 28, 28, 128, 2, TileConfig(14, 7, 128, 32768, 1, 1, 1, layout="HWC")),
    (2, 32, 16, 16, 64, 1, TileConfig(16, 8, 64, 16384, 4, 4, 16, layout="HWC")),
    (3, 256, 7, 7, 128, 1, TileConfig(7, 7, 128, 32768, 1, 1, 1, layout="HWC")),   # library threads
    (3, 64, 14, 14, 64, 2, TileConfig(7, 7, 64, 32768, 1, 1, 1, layout="HWC")),
]


@pytest.mark.parametrize("case", NHWC_CASES, ids=[str(i) for i in range(len(NHWC_CASES))])
def test_direct_nhwc_matches_oracle(case):
    n, c, h, w, k, stride, tile = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.5, 0.5, k).astype(np.float32)
    info = C.query(x.shape, wt.shape, stride, 1, "HWC", tile)
    assert info["rc"] == 0 and "channels-last" in info["reason"], info
    y = C.conv_direct(_dev(x, "HWC"), _dev(wt), stride=stride, padding=1, tile=tile, bias=_dev(b),
                      relu=True)
    assert C.infer_layout(y) == "HWC"
    ref = np.maximum(co.direct_conv(x, wt, stride, 1) + b[None, :, None, None], 0)
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= tol_fp32(c)


def test_direct_nhwc_illegal_tiles():
    x, wt = _inputs(1, 48, 14, 14, 64, 3, 3)   # C not a multiple of 32
    with pytest.raises(InfeasibleTileError):
        C.conv_direct(_dev(x, "HWC"), _dev(wt), padding=1,
                      tile=TileConfig(14, 7, 64, 32768, 1, 1, 1, layout="HWC"))


@pytest.mark.parametrize("prec", ["3xtf32", "tf32"])
def test_igemm_split_k_on_small_grids(prec):
    # 2 images of a 7x7x512 layer: 4 output tiles -> the library splits K over CTAs
    x, wt = _inputs(2, 512, 7, 7, 512, 3, 3)
    b = np.linspace(-0.25, 0.25, 512).astype(np.float32)
    tile = TileConfig(7, 7, 128, 32768, 1, 1, 1, layout="HWC")
    info = C.query(x.shape, wt.shape, 1, 1, "HWC", tile, f"igemm_{prec}")
    assert info["rc"] == 0 and "split-K" in info["reason"] and info["grid_z"] > 1, info
    ref = co.direct_conv(x, wt, 1, 1) + b[None, :, None, None]
    tol = TOL_PREC.get(prec, tol_3xtf32(512))
    y = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, precision=prec, bias=_dev(b))
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= tol
    # ReLU does not commute with the split sum: the library runs it unsplit
    yr = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, tile=tile, precision=prec, bias=_dev(b),
                      relu=True)
    assert co.rel_err(yr.contiguous().cpu().numpy(), np.maximum(ref, 0)) <= tol


@pytest.mark.parametrize("case", [
    # (n, c, h, k, stride, tile, precision): CTA-pair tiles whose work items leave the
    # last round of pairs idle -> the library splits each item's K loop
    (16, 512, 14, 256, 2, TileConfig(1, 1, 256, 32768, 1, 1, 2, layout="HWC"), "3xtf32"),
    (16, 256, 28, 256, 2, TileConfig(1, 2, 256, 32768, 1, 1, 2, layout="HWC"), "tf32"),
    (8, 512, 7, 128, 1, TileConfig(7, 7, 128, 32768, 1, 1, 4, layout="HWC"), "3xtf32"),
    (4, 512, 7, 256, 1, TileConfig(7, 7, 256, 32768, 1, 1, 2, layout="HWC"), "bf16"),
])
def test_igemm_pair_split_k(case):
    n, c, h, k, stride, tile, prec = case
    x, wt = _inputs(n, c, h, h, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    info = C.query(x.shape, wt.shape, stride, 1, "HWC", tile, f"igemm_{prec}")
    assert info["rc"] == 0 and "split-K" in info["reason"], info["reason"]
    ref = co.direct_conv(x, wt, stride, 1) + b[None, :, None, None]
    tol = TOL_PREC.get(prec, tol_3xtf32(c))
    y = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, stride=stride, tile=tile, precision=prec,
                     bias=_dev(b))
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= tol
    yr = C.conv_igemm(_dev(x, "HWC"), _dev(wt), padding=1, stride=stride, tile=tile, precision=prec,
                      bias=_dev(b), relu=True)   # unsplit: ReLU does not commute with the split sum
    assert co.rel_err(yr.contiguous().cpu().numpy(), np.maximum(ref, 0)) <= tol


@pytest.mark.parametrize("case", [
    # (n, c, h, w, k, stride): K8, the channels-last small-C kernel (C <= 4)
    (2, 3, 224, 224, 64, 1),    # VGG-16 conv1_1 shape (2 images)
    (3, 3, 30, 30, 64, 1),      # ragged 16 x 16 blocks
    (2, 2, 20, 17, 32, 1),
    (2, 4, 33, 30, 96, 2),
    (1, 3, 18, 18, 256, 1),   # 8 output-channel chunks per block
    (1, 2, 16, 16, 32, 2),
])
def test_direct_small_c_matches_oracle(case):
    n, c, h, w, k, stride = case
    x, wt = _inputs(n, c, h, w, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    tile = TileConfig(16, 16, 32, 32768, 1, 1, 1, layout="HWC")
    info = C.query(x.shape, wt.shape, stride, 1, "HWC", tile, "direct")
    assert info["rc"] == 0 and "small-C" in info["reason"], info["reason"]
    y = C.conv_direct(_dev(x, "HWC"), _dev(wt), stride=stride, padding=1, tile=tile, bias=_dev(b),
                      relu=True)
    assert C.infer_layout(y) == "HWC"
    ref = np.maximum(co.direct_conv(x, wt, stride, 1) + b[None, :, None, None], 0)
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= 1e-5
    wp = C.pack_filter_direct(_dev(wt))
    y2 = C.conv_direct(_dev(x, "HWC"), _dev(wt), stride=stride, padding=1, tile=tile, bias=_dev(b),
                       relu=True, w_packed=wp)
    assert torch.equal(y, y2)


@pytest.mark.parametrize("case", [
    # (n, c, h, k, e, z): scaled-fp16 3-product Winograd GEMMs (CONVIO_PREC_3XF16)
    (2, 64, 28, 64, 4, 64), (3, 128, 14, 256, 4, 256), (2, 256, 7, 128, 2, 128),
    (2, 512, 7, 512, 4, 256), (4, 128, 28, 128, 4, 128),
])
def test_winograd_tc_3xf16_matches_oracle(case):
    n, c, h, k, e, z = case
    x, wt = _inputs(n, c, h, h, k, 3, 3)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    tile = TileConfig(e, e, z, 32768, 1, 1, 2, layout="HWC", e=e)
    y = C.conv_winograd_tc(_dev(x, "HWC"), _dev(wt), e=e, padding=1, tile=tile, precision="3xf16",
                           bias=_dev(b))
    ref = co.direct_conv(x, wt, 1, 1) + b[None, :, None, None]
    tol = tol_wino(e, c)   # the FP32 Winograd tolerance
    assert co.rel_err(y.contiguous().cpu().numpy(), ref) <= tol
    # rows of very different magnitude: the per-row power-of-two scales keep them exact
    xs = x * np.float32(2.0 ** 20)
    ys = C.conv_winograd_tc(_dev(xs, "HWC"), _dev(wt), e=e, padding=1, tile=tile, precision="3xf16")
    refs = co.direct_conv(xs, wt, 1, 1)
    assert co.rel_err(ys.contiguous().cpu().numpy(), refs) <= tol


@pytest.mark.parametrize("sx,sw", [(-60, -60), (-70, -50), (60, 60), (-70, 60)],
                         ids=["x2^-60,w2^-60", "x2^-70,w2^-50", "x2^60,w2^60", "x2^-70,w2^60"])
@pytest.mark.parametrize("e", [4, 2])
def test_winograd_tc_3xf16_extreme_operand_scales(sx, sw, e):
    """Row (input tile) and column (filter) scale exponents whose sum passes pow2f's
    range: the epilogue unscales with two exact multiplies, so only the relative
    error of the split remains (outputs near 2^-120 .. 2^120 are normal floats)."""
    x, wt = _inputs(2, 64, 14, 14, 128, 3, 3)
    x = x * np.float32(2.0 ** sx)
    wt = wt * np.float32(2.0 ** sw)
    tile = TileConfig(e, e, 128, 32768, 1, 1, 2, layout="HWC", e=e)
    y = C.conv_winograd_tc(_dev(x, "HWC"), _dev(wt), e=e, padding=1, tile=tile, precision="3xf16")
    ref = co.direct_conv(x, wt, 1, 1)
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert np.isfinite(err) and err <= tol_wino(e, 64), err
