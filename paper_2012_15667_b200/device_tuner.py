"""Device-timed measurement for the lower-bound auto-tuner.

Registers the ``"device"`` backend of :func:`.autotune.measure`: the cost of a
``TileConfig`` is the median CUDA-event time (seconds) of its device
projection on synthetic tensors of the layer's shape -- the reference's
"artifact substitution for GPU timing" (``SPEC.md:513``) replaced by the real
thing.  Infeasible configurations (schedule errors, or no legal device
projection: threads, registers, shared memory, compiled micro-tiles) cost
``inf`` and never raise, as in the reference (``autotune.py:182-190``).

:func:`legal_projection` filters a :class:`ConfigSpace` down to the members
the device can launch (SURVEY.md §7 hard part 1); the tuner and the
exhaustive oracle then search that projection.
"""

from __future__ import annotations

import math
import threading
from dataclasses import replace

import torch

from . import _native as N
from . import conv as C
from .autotune import ConfigSpace, register_measure_backend, build_space
from .dataflow import LAYOUTS, TileConfig, ScheduleError, InfeasibleTileError
from .model import ConvShape, WinogradParams, HwModel, GeometryError

_lock = threading.Lock()
_cache: dict = {}
TIMING = {"target_ms": 2.0, "batches": 3, "max_reps": 200}
# zero padding the measured layer uses: the reference's ConvShape is valid-padding
# geometry (model.py:65-70); a padded layer is the same output on an input
# smaller by 2*pad, which is what the bench and the runner launch
_PADDING = [0]


def set_padding(pad: int) -> None:
    """Measure layers as ``pad``-padded convolutions (same outputs, same work)."""
    _PADDING[0] = int(pad)


def _physical(shape: ConvShape) -> tuple[int, int, int]:
    pad = _PADDING[0]
    return shape.h_in - 2 * pad, shape.w_in - 2 * pad, pad


def _tensors(shape: ConvShape, layout: str, algorithm: str, e: int | None):
    """Device tensors for ``shape`` (valid padding: input is w_in x h_in, pad 0)."""
    key = (shape, layout, algorithm, e, _PADDING[0])
    with _lock:
        hit = _cache.get(key)
        if hit is not None:
            return hit
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(1234)
    h, wd, _ = _physical(shape)
    x = C.empty_act(shape.n, shape.c_in, h, wd, layout, device=dev)
    x.uniform_(-1.0, 1.0, generator=g)
    w = (torch.rand((shape.c_out, shape.c_in, shape.h_ker, shape.w_ker), device=dev, generator=g)
         * 2 - 1) / math.sqrt(shape.c_in * shape.h_ker * shape.w_ker)
    y = C.empty_act(shape.n, shape.c_out, shape.h_out, shape.w_out, layout, device=dev)
    prep = C.winograd_filter_transform(w, e) if algorithm == "winograd" else C.pack_filter_direct(w)
    val = (x, w, y, prep)
    with _lock:
        _cache[key] = val
    return val


def clear_cache() -> None:
    with _lock:
        _cache.clear()


def _launcher(cfg: TileConfig, shape: ConvShape, algorithm: str, winograd):
    e = winograd.e if winograd is not None else None
    x, w, y, prep = _tensors(shape, cfg.layout, algorithm, e)
    pad = _PADDING[0]
    if algorithm == "direct":
        return lambda: C.conv_direct(x, w, stride=shape.stride, padding=pad, tile=cfg, out=y,
                                     w_packed=prep)
    return lambda: C.conv_winograd(x, w, e=e, padding=pad, tile=cfg, out=y, u=prep)


def is_legal(cfg: TileConfig, shape: ConvShape, algorithm: str,
             winograd: WinogradParams | None = None) -> bool:
    """Does ``cfg`` have a device projection for this layer (``convio_query``)?"""
    if algorithm == "winograd" and winograd is not None and cfg.e != winograd.e:
        cfg = replace(cfg, e=winograd.e)
    h, wd, pad = _physical(shape)
    desc = N.make_desc(shape.n, shape.c_in, h, wd, shape.c_out, shape.h_ker,
                       shape.w_ker, shape.stride, pad, LAYOUTS.index(cfg.layout))
    rc, _ = N.query(desc, N.make_tile(cfg), N.ALG_DIRECT if algorithm == "direct" else N.ALG_WINOGRAD)
    return rc == 0


def device_time(fn) -> float:
    """Median seconds per launch over a few back-to-back batches (CUDA events)."""
    stream = torch.cuda.current_stream()
    fn()
    stream.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn()
    b.record(stream)
    b.synchronize()
    one = max(a.elapsed_time(b), 1e-3)
    reps = int(min(TIMING["max_reps"], max(1, TIMING["target_ms"] / one)))
    times = []
    for _ in range(TIMING["batches"]):
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b) / 1e3 / reps)
    times.sort()
    return times[len(times) // 2]


def measure_device(cfg: TileConfig, shape: ConvShape, hw: HwModel, algorithm: str,
                   winograd: WinogradParams | None = None) -> float:
    """Seconds per launch of ``cfg``'s device projection; ``inf`` if infeasible."""
    try:
        if algorithm == "winograd":
            if winograd is None:
                return math.inf
            winograd.check_shape(shape)
            if cfg.e != winograd.e:
                cfg = replace(cfg, e=winograd.e)
        if not is_legal(cfg, shape, algorithm, winograd):
            return math.inf
        return device_time(_launcher(cfg, shape, algorithm, winograd))
    except (ScheduleError, InfeasibleTileError, GeometryError, ValueError):
        return math.inf


register_measure_backend("device", measure_device)


def legal_projection(space: ConfigSpace) -> ConfigSpace:
    """The members of ``space`` with a device projection (order preserved)."""
    keep = tuple(c for c in space.members
                 if is_legal(c, space.shape, space.algorithm, space.winograd))
    if not keep:
        raise InfeasibleTileError("no member of the searching domain has a device projection")
    return ConfigSpace(space.shape, space.hw, space.algorithm, space.winograd, space.r_factor,
                       keep, space.unconstrained_size)


def device_space(shape: ConvShape, hw: HwModel, algorithm: str,
                 winograd: WinogradParams | None = None, layouts=("CHW",),
                 thread_axes: bool = True) -> ConfigSpace:
    """Table-1 domain (reference ``build_space``) restricted to its legal projection."""
    return legal_projection(build_space(shape, hw, algorithm, winograd, thread_axes=thread_axes,
                                        layouts=tuple(layouts)))
