"""ctypes binding of ``libconvio_b200.so`` (the C-ABI in ``include/convio_b200.h``).

The library is built in-tree (``paper_2012_15667_b200/lib``) by
``__graft_entry__.build()`` / ``make -C paper_2012_15667_b200/csrc``.  There
is no fallback: if the library is missing every device entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .dataflow import LAYOUTS, InfeasibleTileError, ScheduleError
from .model import GeometryError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
# CONVIO_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("CONVIO_LIB") or os.path.join(LIB_DIR, "libconvio_b200.so")

ALG_DIRECT, ALG_WINOGRAD, ALG_IGEMM_TF32, ALG_IGEMM_3XTF32 = 0, 1, 2, 3
ALG_IGEMM_BF16 = 4
ALG_WINOGRAD_TC_TF32, ALG_WINOGRAD_TC_3XTF32, ALG_WINOGRAD_TC_BF16 = 5, 6, 7
ALG_WINOGRAD_NHWC = 8
ALG_WINOGRAD_TC_3XF16 = 9
ALG_IGEMM_3XF16 = 10
PREC_TF32, PREC_3XTF32, PREC_BF16, PREC_FP32, PREC_3XF16 = 0, 1, 2, 3, 4
PRECISIONS = {"tf32": PREC_TF32, "3xtf32": PREC_3XTF32, "bf16": PREC_BF16, "fp32": PREC_FP32,
              "3xf16": PREC_3XF16}


class ConvDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in
                ("n", "c", "h", "w", "k", "r", "s", "stride", "pad", "layout")]


class Tile(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in
                ("x", "y", "z", "s_b", "n_xt", "n_yt", "n_zt", "layout", "e")]


class LaunchInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in
                ("legal", "grid_x", "grid_y", "grid_z", "block_threads", "smem_bytes",
                 "regs_per_thread", "channel_chunk", "stages", "smem_pitch", "p", "q")] + [
        ("flops", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
        ("reason", ctypes.c_char * 160)]

    def to_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "reason"}
        d["reason"] = self.reason.decode(errors="replace")
        return d


class DeviceError(RuntimeError):
    """CUDA / internal failure inside libconvio_b200 (return code 4)."""


_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing -- build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` or `make -C paper_2012_15667_b200/csrc`; there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        D, T, LI = ctypes.POINTER(ConvDesc), ctypes.POINTER(Tile), ctypes.POINTER(LaunchInfo)
        sigs = {
            "convio_version": ([], ctypes.c_int),
            "convio_last_error": ([], ctypes.c_char_p),
            "convio_last_error_kind": ([], ctypes.c_int),
            "convio_last_launch_count": ([], ctypes.c_int),
            "convio_query": ([D, T, I32, LI], ctypes.c_int),
            "convio_workspace_bytes": ([D, T, I32], I64),
            "convio_pack_filter_direct": ([D, P, P, P], ctypes.c_int),
            "convio_conv_direct_f32": ([D, T, P, P, I32, P, I32, P, P, SZ, P], ctypes.c_int),
            "convio_winograd_filter_transform": ([D, I32, P, P, P], ctypes.c_int),
            "convio_conv_winograd_f32": ([D, T, I32, P, P, I32, P, I32, P, P, SZ, P], ctypes.c_int),
            "convio_winograd_matrices": ([I32, I32, P, P, P], ctypes.c_int),
            "convio_ffma_peak": ([P, I32, I32, ctypes.POINTER(I64), P], ctypes.c_int),
            "convio_default_tile": ([D, I32, I32, T], ctypes.c_int),
            "convio_pack_filter_igemm": ([D, P, P, P], ctypes.c_int),
            "convio_conv_igemm_tf32": ([D, T, P, P, I32, P, I32, P, P, SZ, P], ctypes.c_int),
            "convio_conv_igemm_3xtf32": ([D, T, P, P, I32, P, I32, P, P, SZ, P], ctypes.c_int),
            "convio_conv_igemm": ([D, T, I32, P, P, I32, P, I32, P, P, SZ, P], ctypes.c_int),
            "convio_pack_filter_igemm_bf16": ([D, P, P, P], ctypes.c_int),
            "convio_convert_bf16": ([P, P, I64, P], ctypes.c_int),
            "convio_winograd_filter_transform_tc": ([D, I32, I32, P, P, P], ctypes.c_int),
            "convio_winograd_bgemm": ([D, T, I32, I32, P, P, I32, P, I32, P, P, SZ, P],
                                      ctypes.c_int),
            "convio_pack_filter_igemm_f16x3": ([D, P, P, P], ctypes.c_int),
            "convio_pack_filter_igemm_f16x3_bytes": ([D], I64),
            "convio_pack_filters_igemm_f16x3_batched": ([I32, D, P, P, P], ctypes.c_int),
            "convio_conv_igemm_grouped": ([D, T, I32, I32, P, P, SZ, P, I32, P, P, SZ, P], ctypes.c_int),
            "convio_winograd_filter_transform_tc_batched": ([I32, D, I32, I32, P, P, P], ctypes.c_int),
            "convio_nchw_to_nhwc": ([P, P, I32, I32, I32, I32, P], ctypes.c_int),
            "convio_nhwc_to_nchw": ([P, P, I32, I32, I32, I32, P], ctypes.c_int),
            "convio_maxpool2x2_nhwc": ([P, P, I32, I32, I32, I32, P], ctypes.c_int),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


EXPORTED = (
    "convio_version", "convio_last_error", "convio_last_error_kind", "convio_last_launch_count", "convio_query",
    "convio_workspace_bytes", "convio_pack_filter_direct", "convio_conv_direct_f32",
    "convio_winograd_filter_transform", "convio_conv_winograd_f32", "convio_winograd_matrices",
    "convio_ffma_peak", "convio_default_tile", "convio_pack_filter_igemm", "convio_conv_igemm_tf32",
    "convio_conv_igemm_3xtf32", "convio_conv_igemm", "convio_pack_filter_igemm_bf16",
    "convio_convert_bf16", "convio_winograd_filter_transform_tc", "convio_winograd_bgemm",
    "convio_pack_filter_igemm_f16x3", "convio_pack_filter_igemm_f16x3_bytes",
    "convio_pack_filters_igemm_f16x3_batched", "convio_winograd_filter_transform_tc_batched",
    "convio_conv_igemm_grouped",
    "convio_nchw_to_nhwc", "convio_nhwc_to_nchw", "convio_maxpool2x2_nhwc",
)


def last_error() -> str:
    msg = lib().convio_last_error()
    return msg.decode(errors="replace") if msg else ""


EKIND_NONE, EKIND_SCHEDULE, EKIND_INFEASIBLE, EKIND_GEOMETRY = 0, 1, 2, 3
_KIND_CLASS = {EKIND_SCHEDULE: ScheduleError, EKIND_GEOMETRY: GeometryError}


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI return code onto the reference's exception classes.

    rc 3 carries its class explicitly (``convio_last_error_kind``): the
    reference's ``ScheduleError`` / ``GeometryError``, else
    ``InfeasibleTileError`` -- so ``measure()``'s
    ``except (ScheduleError, InfeasibleTileError)`` keeps its meaning
    whatever the message text says.
    """
    if rc == 0:
        return
    msg = last_error() or what
    if rc == 2:
        raise ValueError(msg)
    if rc == 3:
        raise _KIND_CLASS.get(lib().convio_last_error_kind(), InfeasibleTileError)(msg)
    raise DeviceError(f"{what}: {msg} (rc={rc})")


def make_tile(tile, layout: int | None = None) -> Tile | None:
    if tile is None:
        return None
    t = Tile()
    for f in ("x", "y", "z", "s_b", "n_xt", "n_yt", "n_zt"):
        setattr(t, f, int(getattr(tile, f)))
    t.layout = LAYOUTS.index(tile.layout) if layout is None else layout
    t.e = int(tile.e or 0)
    return t


def make_desc(n, c, h, w, k, r, s, stride, pad, layout: int) -> ConvDesc:
    return ConvDesc(n, c, h, w, k, r, s, stride, pad, layout)


def query(desc: ConvDesc, tile: Tile | None, algorithm: int) -> tuple[int, dict]:
    info = LaunchInfo()
    rc = lib().convio_query(ctypes.byref(desc), ctypes.byref(tile) if tile else None,
                            algorithm, ctypes.byref(info))
    d = info.to_dict()
    d["kind"] = lib().convio_last_error_kind() if rc != 0 else EKIND_NONE
    if rc != 0 and not d["reason"]:
        d["reason"] = last_error()
    return rc, d
