"""Device convolution entry points: the schedules of :mod:`.dataflow` run as
sm_100a CUDA kernels through the C-ABI (``libconvio_b200.so``).

* :func:`conv_direct`   -- output-stationary direct dataflow
  (reference schedule ``pkg/src/convio/dataflow.py:219-250``)
* :func:`conv_winograd` -- fused Winograd F(e x e, 3 x 3) dataflow with the
  shared kernel transform (``dataflow.py:253-310``, ``shared_kernel_transform``)
* :func:`winograd_filter_transform` -- ``U = G g G^T`` once per filter

Tensors are PyTorch CUDA fp32 tensors with logical shape NCHW / KCRS; the
physical activation layout (``CHW`` = NCHW, ``HWC`` = NHWC/channels_last,
``CWH`` = N C W H) is read from the strides and is the reference's
``LAYOUTS`` axis.  PyTorch is used for memory and streams only -- every
output value is produced by this package's kernels; there is no CPU path.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N
from .dataflow import LAYOUTS, TileConfig

__all__ = ["conv_direct", "conv_winograd", "conv_igemm_tf32", "conv_igemm", "conv_winograd_tc",
           "winograd_filter_transform", "winograd_filter_transform_tc",
           "pack_filter_direct", "pack_filter_igemm", "pack_filter_igemm_bf16", "pack_filter_igemm_f16x3",
           "conv_igemm_grouped", "f16x3_slice_bytes",
           "infer_layout", "to_layout", "maxpool2x2", "empty_act", "query", "last_launch_count"]


def _strides_for(layout: str, n: int, c: int, h: int, w: int) -> tuple[int, int, int, int]:
    if layout == "HWC":
        return (h * w * c, 1, w * c, c)
    if layout == "CWH":
        return (c * h * w, h * w, 1, h)
    return (c * h * w, h * w, w, 1)


def infer_layout(x: torch.Tensor) -> str:
    """Physical layout of a logical-NCHW tensor; raises for anything else."""
    n, c, h, w = x.shape
    st = tuple(x.stride())
    for lay in LAYOUTS:   # CHW first: wins when sizes make layouts coincide
        want = _strides_for(lay, n, c, h, w)
        if all(sz == 1 or a == b for sz, a, b in zip(x.shape, st, want)):
            return lay
    raise ValueError(f"tensor strides {st} match none of the layouts {LAYOUTS}")


def empty_act(n: int, c: int, h: int, w: int, layout: str = "CHW",
              device=None, dtype=torch.float32) -> torch.Tensor:
    """Uninitialised activation tensor, logical NCHW, physical ``layout``."""
    return torch.empty_strided((n, c, h, w), _strides_for(layout, n, c, h, w),
                               device=device, dtype=dtype)


def to_layout(x: torch.Tensor, layout: str, stream=None) -> torch.Tensor:
    """Copy ``x`` into ``layout`` (a separate, explicitly requested staging step).

    CUDA fp32 NCHW <-> NHWC goes through the library's transpose kernels
    (``convio_nchw_to_nhwc`` / ``convio_nhwc_to_nchw``: a counted launch, one read
    and one write of every element); other cases (the CWH axis, host tensors) are
    a framework copy."""
    src = infer_layout(x)
    if src == layout:
        return x
    y = empty_act(*x.shape, layout=layout, device=x.device, dtype=x.dtype)
    if x.is_cuda and x.dtype == torch.float32 and {src, layout} == {"CHW", "HWC"} and x.numel():
        n, c, h, w = x.shape
        fn = N.lib().convio_nchw_to_nhwc if layout == "HWC" else N.lib().convio_nhwc_to_nchw
        N.check(fn(_ptr(x), _ptr(y), n, c, h, w, _stream_ptr(stream)), "to_layout")
        return y
    y.copy_(x)
    return y


def maxpool2x2(x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """2x2 / stride-2 max pooling of a channels-last (HWC) activation."""
    _check_tensor(x, "x")
    if infer_layout(x) != "HWC":
        raise ValueError("maxpool2x2 needs a channels-last (HWC) input")
    n, c, h, w = x.shape
    if out is None:
        out = empty_act(n, c, h // 2, w // 2, "HWC", device=x.device)
    N.check(N.lib().convio_maxpool2x2_nhwc(_ptr(x), _ptr(out), n, h, w, c, _stream_ptr(stream)), "maxpool2x2")
    return out


def _check_tensor(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32, got {t.dtype}")


def _stream_ptr(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p | None:
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _desc(x: torch.Tensor, w: torch.Tensor, stride: int, padding: int, layout: str) -> N.ConvDesc:
    n, c, h, wd = x.shape
    k, c2, r, s = w.shape
    if c2 != c:
        raise ValueError(f"filter has {c2} input channels, input has {c}")
    return N.make_desc(n, c, h, wd, k, r, s, stride, padding, LAYOUTS.index(layout))


def _out_hw(h, w, r, s, stride, padding):
    return (h + 2 * padding - r) // stride + 1, (w + 2 * padding - s) // stride + 1


ALGORITHMS = {"direct": N.ALG_DIRECT, "winograd": N.ALG_WINOGRAD,
              "igemm_tf32": N.ALG_IGEMM_TF32, "igemm_3xtf32": N.ALG_IGEMM_3XTF32,
              "igemm_bf16": N.ALG_IGEMM_BF16, "igemm_3xf16": N.ALG_IGEMM_3XF16,
              "winograd_tc_tf32": N.ALG_WINOGRAD_TC_TF32,
              "winograd_tc_3xtf32": N.ALG_WINOGRAD_TC_3XTF32,
              "winograd_tc_bf16": N.ALG_WINOGRAD_TC_BF16, "winograd_nhwc": N.ALG_WINOGRAD_NHWC,
              "winograd_tc_fp32": N.ALG_WINOGRAD_NHWC, "winograd_tc_3xf16": N.ALG_WINOGRAD_TC_3XF16}


def query(x_shape, w_shape, stride: int = 1, padding: int = 0, layout: str = "CHW",
          tile: TileConfig | None = None, algorithm: str = "direct") -> dict:
    """Device projection of ``tile`` for this layer (legality + launch shape)."""
    n, c, h, w = x_shape
    k, _, r, s = w_shape
    desc = N.make_desc(n, c, h, w, k, r, s, stride, padding, LAYOUTS.index(layout))
    alg = ALGORITHMS[algorithm]
    rc, info = N.query(desc, N.make_tile(tile), alg)
    info["rc"] = rc
    return info


def pack_filter_direct(w: torch.Tensor, stream=None) -> torch.Tensor:
    """KCRS -> C R S K repack consumed by the direct kernel (cacheable per layer)."""
    _check_tensor(w, "w")
    w = w.contiguous()
    k, c, r, s = w.shape
    out = torch.empty((c, r, s, k), device=w.device, dtype=torch.float32)
    desc = N.make_desc(1, c, r, s, k, r, s, 1, 0, 0)
    N.check(N.lib().convio_pack_filter_direct(ctypes.byref(desc), _ptr(w), _ptr(out),
                                              _stream_ptr(stream)), "pack_filter_direct")
    return out


def conv_direct(x: torch.Tensor, w: torch.Tensor, stride: int = 1, padding: int = 0,
                tile: TileConfig | None = None, bias: torch.Tensor | None = None,
                relu: bool = False, out: torch.Tensor | None = None, stream=None,
                w_packed: torch.Tensor | None = None,
                workspace: torch.Tensor | None = None) -> torch.Tensor:
    """``y = conv2d(x, w)`` (+bias, +ReLU) by the direct dataflow kernel.

    ``tile`` is a :class:`TileConfig`; ``None`` lets the library pick its
    default device tile.  ``w_packed`` (from :func:`pack_filter_direct`)
    skips the per-call filter repack.  Illegal tiles raise the reference's
    ``ScheduleError`` / ``InfeasibleTileError``.
    """
    _check_tensor(x, "x")
    _check_tensor(w, "w")
    layout = infer_layout(x)
    if tile is not None and tile.layout != layout:
        raise ValueError(f"tile layout {tile.layout} but input is {layout}")
    desc = _desc(x, w, stride, padding, layout)
    p, q = _out_hw(desc.h, desc.w, desc.r, desc.s, stride, padding)
    if out is None:
        out = empty_act(desc.n, desc.k, p, q, layout, device=x.device)
    else:
        _check_tensor(out, "out")
        if tuple(out.shape) != (desc.n, desc.k, p, q) or infer_layout(out) != layout:
            raise ValueError("out has the wrong shape or layout")
    if bias is not None:
        _check_tensor(bias, "bias")
    if w_packed is not None:
        wsrc, is_packed, ws, ws_bytes = w_packed, 1, None, 0
    else:
        need = desc.k * desc.c * desc.r * desc.s
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, device=x.device, dtype=torch.float32)
        wsrc, is_packed, ws, ws_bytes = w.contiguous(), 0, workspace, 4 * need
    rc = N.lib().convio_conv_direct_f32(
        ctypes.byref(desc), ctypes.byref(N.make_tile(tile)) if tile is not None else None,
        _ptr(x), _ptr(wsrc), is_packed, _ptr(bias), int(bool(relu)), _ptr(out),
        _ptr(ws), ws_bytes, _stream_ptr(stream))
    N.check(rc, "conv_direct")
    return out


def winograd_filter_transform(w: torch.Tensor, e: int, stream=None) -> torch.Tensor:
    """``U[xi][c][k] = (G g G^T)[xi]`` for F(e x e, 3 x 3) -- the shared J_k."""
    _check_tensor(w, "w")
    w = w.contiguous()
    k, c, r, s = w.shape
    m = e + r - 1
    u = torch.empty((m * m, c, k), device=w.device, dtype=torch.float32)
    desc = N.make_desc(1, c, max(r, 3), max(s, 3), k, r, s, 1, 0, 0)
    N.check(N.lib().convio_winograd_filter_transform(ctypes.byref(desc), e, _ptr(w), _ptr(u),
                                                     _stream_ptr(stream)),
            "winograd_filter_transform")
    return u


def conv_winograd(x: torch.Tensor, w: torch.Tensor, e: int = 2, padding: int = 0,
                  tile: TileConfig | None = None, bias: torch.Tensor | None = None,
                  relu: bool = False, out: torch.Tensor | None = None, stream=None,
                  u: torch.Tensor | None = None,
                  workspace: torch.Tensor | None = None) -> torch.Tensor:
    """``y = conv2d(x, w)`` (3x3, stride 1) by the fused Winograd F(e, 3) kernel.

    ``u`` (from :func:`winograd_filter_transform`) skips the per-call filter
    transform.  Outputs not divisible by the tile are refused like the model
    refuses ragged tiles.
    """
    _check_tensor(x, "x")
    _check_tensor(w, "w")
    layout = infer_layout(x)
    if tile is not None and tile.layout != layout:
        raise ValueError(f"tile layout {tile.layout} but input is {layout}")
    desc = _desc(x, w, 1, padding, layout)
    p, q = _out_hw(desc.h, desc.w, desc.r, desc.s, 1, padding)
    if out is None:
        out = empty_act(desc.n, desc.k, p, q, layout, device=x.device)
    else:
        _check_tensor(out, "out")
        if tuple(out.shape) != (desc.n, desc.k, p, q) or infer_layout(out) != layout:
            raise ValueError("out has the wrong shape or layout")
    if bias is not None:
        _check_tensor(bias, "bias")
    m = e + desc.r - 1
    if u is not None:
        wsrc, is_t, ws, ws_bytes = u, 1, None, 0
    else:
        need = m * m * desc.c * desc.k
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, device=x.device, dtype=torch.float32)
        wsrc, is_t, ws, ws_bytes = w.contiguous(), 0, workspace, 4 * need
    rc = N.lib().convio_conv_winograd_f32(
        ctypes.byref(desc), ctypes.byref(N.make_tile(tile)) if tile is not None else None, e,
        _ptr(x), _ptr(wsrc), is_t, _ptr(bias), int(bool(relu)), _ptr(out), _ptr(ws), ws_bytes,
        _stream_ptr(stream))
    N.check(rc, "conv_winograd")
    return out


def pack_filter_igemm(w: torch.Tensor, stream=None) -> torch.Tensor:
    """KCRS -> [R*S][K][C] for the tcgen05 implicit GEMM (K-major B operand)."""
    _check_tensor(w, "w")
    w = w.contiguous()
    k, c, r, s = w.shape
    out = torch.empty((r * s, k, c), device=w.device, dtype=torch.float32)
    desc = N.make_desc(1, c, r, s, k, r, s, 1, 0, 2)
    N.check(N.lib().convio_pack_filter_igemm(ctypes.byref(desc), _ptr(w), _ptr(out),
                                             _stream_ptr(stream)), "pack_filter_igemm")
    return out


def conv_igemm_tf32(x: torch.Tensor, w: torch.Tensor, padding: int = 0,
                    tile: TileConfig | None = None, bias: torch.Tensor | None = None,
                    relu: bool = False, out: torch.Tensor | None = None, stream=None,
                    w_packed: torch.Tensor | None = None,
                    workspace: torch.Tensor | None = None, stride: int = 1,
                    split: bool = False) -> torch.Tensor:
    """Direct conv as a tcgen05 implicit GEMM, FP32 accumulation in TMEM.

    ``x`` must be channels-last (layout ``HWC``), ``C % 32 == 0``, stride 1/2,
    ``tile.x * tile.y <= 128``.  ``split=False``: TF32 inputs, ``tile.z in
    {64,128,256}``, tolerance 5e-3.  ``split=True``: 3xTF32
    (hi/lo operand split, 3 MMAs per k-step) -- FP32-level accuracy,
    ``tile.z in {64,128}``.
    """
    _check_tensor(x, "x")
    _check_tensor(w, "w")
    layout = infer_layout(x)
    if layout != "HWC":
        raise ValueError("conv_igemm_tf32 needs a channels-last (HWC) input")
    if tile is None:
        raise ValueError("conv_igemm_tf32 needs an explicit tile")
    desc = _desc(x, w, stride, padding, layout)
    p, q = _out_hw(desc.h, desc.w, desc.r, desc.s, stride, padding)
    if out is None:
        out = empty_act(desc.n, desc.k, p, q, layout, device=x.device)
    if w_packed is not None:
        wsrc, is_packed, ws, ws_bytes = w_packed, 1, None, 0
    else:
        need = desc.k * desc.c * desc.r * desc.s
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, device=x.device, dtype=torch.float32)
        wsrc, is_packed, ws, ws_bytes = w.contiguous(), 0, workspace, 4 * need
    fn = N.lib().convio_conv_igemm_3xtf32 if split else N.lib().convio_conv_igemm_tf32
    rc = fn(ctypes.byref(desc), ctypes.byref(N.make_tile(tile, 2)), _ptr(x), _ptr(wsrc), is_packed,
            _ptr(bias), int(bool(relu)), _ptr(out), _ptr(ws), ws_bytes, _stream_ptr(stream))
    N.check(rc, "conv_igemm_3xtf32" if split else "conv_igemm_tf32")
    return out


def pack_filter_igemm_bf16(w: torch.Tensor, stream=None) -> torch.Tensor:
    """KCRS fp32 -> [R*S][K][C] bf16 for the BF16 tcgen05 implicit GEMM."""
    _check_tensor(w, "w")
    w = w.contiguous()
    k, c, r, s = w.shape
    out = torch.empty((r * s, k, c), device=w.device, dtype=torch.bfloat16)
    desc = N.make_desc(1, c, r, s, k, r, s, 1, 0, 2)
    N.check(N.lib().convio_pack_filter_igemm_bf16(ctypes.byref(desc), _ptr(w), _ptr(out),
                                                  _stream_ptr(stream)), "pack_filter_igemm_bf16")
    return out


def pack_filter_igemm_f16x3(w: torch.Tensor, stream=None) -> torch.Tensor:
    """KCRS fp32 filter -> the 3xF16 implicit-GEMM operand (uint8 buffer: fp16
    hi / lo planes ``[2][R*S][K][C]`` scaled by ``2^e[k]`` per output channel,
    then ``e[K]``), for ``conv_igemm(..., precision="3xf16", w_packed=...)``."""
    _check_tensor(w, "w")
    k, c, r, s_ = w.shape
    desc = N.make_desc(1, c, r, s_, k, r, s_, 1, 0, 2)
    nbytes = int(N.lib().convio_pack_filter_igemm_f16x3_bytes(ctypes.byref(desc)))
    out = torch.empty(nbytes, device=w.device, dtype=torch.uint8)
    N.check(N.lib().convio_pack_filter_igemm_f16x3(ctypes.byref(desc), _ptr(w.contiguous()), _ptr(out),
                                                   _stream_ptr(stream)), "pack_filter_igemm_f16x3")
    return out


def f16x3_slice_bytes(k: int, c: int, r: int, s: int) -> int:
    """Bytes of one packed 3xF16 filter (``pack_filter_igemm_f16x3``), rounded to 256."""
    desc = N.make_desc(1, c, max(8, r), max(8, s), k, r, s, 1, 0, 2)
    return 256 * ((int(N.lib().convio_pack_filter_igemm_f16x3_bytes(ctypes.byref(desc))) + 255) // 256)


def conv_igemm_grouped(x: torch.Tensor, w_shape, w_packed: torch.Tensor, layers: int, slice_bytes: int,
                       padding: int = 0, stride: int = 1, tile: TileConfig | None = None,
                       bias: torch.Tensor | None = None, relu: bool = False,
                       out: torch.Tensor | None = None, stream=None,
                       workspace: torch.Tensor | None = None) -> torch.Tensor:
    """``layers`` independent 3xF16 convolutions of one shape and tile in ONE launch
    (``convio_conv_igemm_grouped``): ``x`` channels-last with the layers' batches
    stacked along N, ``w_packed`` the layers' :func:`pack_filter_igemm_f16x3` outputs
    as ``slice_bytes``-apart slices, ``bias`` ``layers x K``; returns the stacked
    outputs.  Layer l's images are ``[l * N / layers, (l + 1) * N / layers)``."""
    _check_tensor(x, "x")
    if infer_layout(x) != "HWC":
        raise ValueError("conv_igemm_grouped needs a channels-last (HWC) input")
    if tile is None:
        raise ValueError("conv_igemm_grouped needs an explicit tile")
    n_all = x.shape[0]
    if layers < 1 or n_all % layers:
        raise ValueError(f"{n_all} stacked images do not split into {layers} layers")
    k, c, r, s_ = w_shape
    desc = N.make_desc(n_all // layers, x.shape[1], x.shape[2], x.shape[3], k, r, s_, stride, padding, 2)
    p, q = _out_hw(desc.h, desc.w, r, s_, stride, padding)
    if out is None:
        out = empty_act(n_all, k, p, q, "HWC", device=x.device)
    need = 256 * ((4 * 296 + 255) // 256)
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.zeros(need, device=x.device, dtype=torch.uint8)
    rc = N.lib().convio_conv_igemm_grouped(
        ctypes.byref(desc), ctypes.byref(N.make_tile(tile, 2)), N.PREC_3XF16, layers, _ptr(x), _ptr(w_packed),
        slice_bytes, _ptr(bias), int(bool(relu)), _ptr(out), _ptr(workspace), need, _stream_ptr(stream))
    N.check(rc, "conv_igemm_grouped[3xf16]")
    return out


# conv_igemm precisions -> the C-ABI algorithm ids (workspace size / query)
_IGEMM_ALG = {"tf32": N.ALG_IGEMM_TF32, "3xtf32": N.ALG_IGEMM_3XTF32, "bf16": N.ALG_IGEMM_BF16,
              "3xf16": N.ALG_IGEMM_3XF16}


def _precision(precision: str) -> int:
    try:
        return N.PRECISIONS[precision]
    except KeyError:
        raise ValueError(f"precision must be one of {sorted(N.PRECISIONS)}, got {precision!r}")


def conv_igemm(x: torch.Tensor, w: torch.Tensor, padding: int = 0, stride: int = 1,
               tile: TileConfig | None = None, precision: str = "3xtf32",
               bias: torch.Tensor | None = None, relu: bool = False,
               out: torch.Tensor | None = None, stream=None,
               w_packed: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Direct conv as a tcgen05 implicit GEMM at ``precision`` ("tf32",
    "3xtf32", "3xf16" or "bf16"; FP32 accumulation in TMEM).  Channels-last
    input, ``C % 32 == 0`` (``% 64`` for bf16 / 3xf16).  For bf16 the
    activations are converted to bf16 in the workspace by the library; 3xf16
    (CTA-pair tiles) splits them on chip into power-of-two-scaled fp16 hi / lo
    planes (FP32-level accuracy at the f16 tensor rate).  ``w_packed`` must come
    from :func:`pack_filter_igemm_bf16` (bf16), :func:`pack_filter_igemm_f16x3`
    (3xf16) or :func:`pack_filter_igemm`.
    Tolerances (tests/tolerances.py): 3xtf32 / 3xf16 FP32-level, tf32 5e-3, bf16 2e-2.
    ``tile.n_zt`` selects the kernel: 1 = one 128-pixel tile per CTA, 2 = the
    persistent CTA pair (``tcgen05.mma.cta_group::2``, M = 256, z/2 filter
    rows staged per CTA, double-buffered TMEM accumulators).
    """
    _check_tensor(x, "x")
    _check_tensor(w, "w")
    prec = _precision(precision)
    layout = infer_layout(x)
    if layout != "HWC":
        raise ValueError("conv_igemm needs a channels-last (HWC) input")
    if tile is None:
        raise ValueError("conv_igemm needs an explicit tile")
    desc = _desc(x, w, stride, padding, layout)
    p, q = _out_hw(desc.h, desc.w, desc.r, desc.s, stride, padding)
    if out is None:
        out = empty_act(desc.n, desc.k, p, q, layout, device=x.device)
    need = int(N.lib().convio_workspace_bytes(ctypes.byref(desc), None, _IGEMM_ALG[precision]))
    wsrc, is_packed = (w_packed, 1) if w_packed is not None else (w.contiguous(), 0)
    if w_packed is not None and prec == N.PREC_3XF16:
        need = 256 * ((4 * 296 + 255) // 256)   # the activation-scale state only
    elif w_packed is not None and prec != N.PREC_BF16:
        need = 0
    if need and (workspace is None or workspace.numel() * workspace.element_size() < need):
        workspace = torch.empty(need, device=x.device, dtype=torch.uint8)
    rc = N.lib().convio_conv_igemm(
        ctypes.byref(desc), ctypes.byref(N.make_tile(tile, 2)), prec, _ptr(x), _ptr(wsrc),
        is_packed, _ptr(bias), int(bool(relu)), _ptr(out), _ptr(workspace) if need else None,
        need, _stream_ptr(stream))
    N.check(rc, f"conv_igemm[{precision}]")
    return out


def winograd_filter_transform_tc(w: torch.Tensor, e: int, precision: str = "3xtf32",
                                 stream=None) -> torch.Tensor:
    """``U[xi][k][c] = (G g G^T)[xi]`` (K-major B operand of the tensor-core
    Winograd GEMMs; bf16 for ``precision="bf16"``); ``precision="fp32"`` (the
    FFMA GEMM) gives ``U[xi][c][k]``."""
    _check_tensor(w, "w")
    prec = _precision(precision)
    w = w.contiguous()
    k, c, r, s = w.shape
    m = e + r - 1
    shape = (m * m, c, k) if prec == N.PREC_FP32 else (m * m, k, c)
    if prec == N.PREC_3XF16:   # packed: fp32 U, fp16 hi / lo planes, per-row exponents
        shape = (m * m, k, 2 * c + 1)
    u = torch.empty(shape, device=w.device,
                    dtype=torch.bfloat16 if prec == N.PREC_BF16 else torch.float32)
    desc = N.make_desc(1, c, 8, 8, k, r, s, 1, 1, 2)
    N.check(N.lib().convio_winograd_filter_transform_tc(ctypes.byref(desc), e, prec, _ptr(w),
                                                        _ptr(u), _stream_ptr(stream)),
            "winograd_filter_transform_tc")
    return u


def conv_winograd_tc(x: torch.Tensor, w: torch.Tensor, e: int = 4, padding: int = 1,
                     tile: TileConfig | None = None, precision: str = "3xtf32",
                     bias: torch.Tensor | None = None, relu: bool = False,
                     out: torch.Tensor | None = None, stream=None,
                     u: torch.Tensor | None = None,
                     workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Winograd F(e x e, 3 x 3) with the element-wise batched GEMM on tcgen05
    (``convio_winograd_bgemm``).  Channels-last input, stride 1.  ``u`` from
    :func:`winograd_filter_transform_tc` (same precision) skips the filter
    transform.  Ragged outputs (P, Q not multiples of e) are handled by
    zero-padded tiles.  ``precision="fp32"`` runs the element-wise GEMMs on
    the CUDA cores (FP32 FFMA, the paper-faithful arithmetic) instead.  Tolerances: 3xtf32 as the FP32 Winograd (F(2,3) 1e-4,
    F(4,3) 1e-3), tf32 5e-3, bf16 3e-2.
    """
    _check_tensor(x, "x")
    _check_tensor(w, "w")
    prec = _precision(precision)
    layout = infer_layout(x)
    if layout != "HWC":
        raise ValueError("conv_winograd_tc needs a channels-last (HWC) input")
    desc = _desc(x, w, 1, padding, layout)
    p, q = _out_hw(desc.h, desc.w, desc.r, desc.s, 1, padding)
    if out is None:
        out = empty_act(desc.n, desc.k, p, q, layout, device=x.device)
    if tile is not None:
        ct = N.make_tile(tile, 2)
    elif prec == N.PREC_FP32:   # library default for the FFMA GEMM
        ct = N.Tile(e, e, 128 if desc.k % 128 == 0 else 64, 8192, 1, 1, 1, 2, e)
    else:   # library default: widest N tile dividing K, CTA-pair kernel
        z = 256 if desc.k % 256 == 0 else (128 if desc.k % 128 == 0 else 64)
        ct = N.Tile(e, e, z, 8192, 1, 1, 2, 2, e)
    alg = N.ALG_WINOGRAD_TC_3XF16 if prec == N.PREC_3XF16 else N.ALG_WINOGRAD_TC_TF32 + prec
    need = int(N.lib().convio_workspace_bytes(ctypes.byref(desc), ctypes.byref(ct), alg))
    if need < 0:
        rc, _ = N.query(desc, ct, alg)
        N.check(rc if rc else 3, "conv_winograd_tc")
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(max(need, 1), device=x.device, dtype=torch.uint8)
    wsrc, is_t = (u, 1) if u is not None else (w.contiguous(), 0)
    rc = N.lib().convio_winograd_bgemm(
        ctypes.byref(desc), ctypes.byref(ct), e, prec, _ptr(x), _ptr(wsrc), is_t,
        _ptr(bias), int(bool(relu)), _ptr(out), _ptr(workspace), need, _stream_ptr(stream))
    N.check(rc, f"conv_winograd_tc[{precision}]")
    return out


def last_launch_count() -> int:
    """Kernel launches issued by the last conv call on this thread."""
    return int(N.lib().convio_last_launch_count())
