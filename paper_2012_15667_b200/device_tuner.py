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

**Engines.**  The reference API knows two algorithms, ``"direct"`` and
``"winograd"``; which device kernel family realises a configuration is the
*engine* (:func:`set_engine` / :func:`use_engine`): ``"ffma"`` (default: the
FP32 CUDA-core dataflows K1 / K6 / K2) or a tcgen05 family -- ``igemm_<prec>``
for ``"direct"`` and ``winograd_tc_<prec>`` for ``"winograd"``, ``prec`` in
tf32 / 3xtf32 / 3xf16 / bf16.  So ``tune(shape, hw, "direct", budget, seed,
backend="device", space=tcgen05_space(...))`` under ``use_engine("igemm_3xf16")``
searches the shipped tensor-core kernels through the reference's own tuner.
:func:`tcgen05_space` is their searching domain, pruned by the tensor-memory
machine model (:func:`tcgen05_hw_model`); :func:`tune_layer` is the per-layer
search the tuned plan tables come from.
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
# the device kernel family that realises "direct" / "winograd" configurations
_ENGINE = ["ffma"]
ENGINES = ("ffma", "igemm_tf32", "igemm_3xtf32", "igemm_3xf16", "igemm_bf16",
           "winograd_tc_tf32", "winograd_tc_3xtf32", "winograd_tc_3xf16", "winograd_tc_bf16",
           "winograd_tc_fp32")   # winograd_tc_fp32: the same pipeline, FFMA element-wise GEMMs


def set_engine(engine: str) -> None:
    """Select the kernel family measured for "direct" / "winograd" configs."""
    if engine not in ENGINES:
        raise ValueError(f"engine must be one of {ENGINES}, got {engine!r}")
    _ENGINE[0] = engine


class use_engine:
    """``with use_engine("igemm_3xf16"): tune(..., backend="device")``"""

    def __init__(self, engine: str):
        self.engine, self.prev = engine, None

    def __enter__(self):
        self.prev = _ENGINE[0]
        set_engine(self.engine)
        return self

    def __exit__(self, *exc):
        _ENGINE[0] = self.prev
        return False


def _engine_for(algorithm: str) -> str:
    """The engine that realises ``algorithm`` now ("ffma" when the engine's kind
    does not match: igemm engines realise "direct", winograd_tc engines "winograd")."""
    eng = _ENGINE[0]
    if eng.startswith("igemm_") and algorithm == "direct":
        return eng
    if eng.startswith("winograd_tc_") and algorithm == "winograd":
        return eng
    return "ffma"


def set_padding(pad: int) -> None:
    """Measure layers as ``pad``-padded convolutions (same outputs, same work)."""
    _PADDING[0] = int(pad)


def _physical(shape: ConvShape) -> tuple[int, int, int]:
    pad = _PADDING[0]
    return shape.h_in - 2 * pad, shape.w_in - 2 * pad, pad


def _tensors(shape: ConvShape, layout: str, algorithm: str, e: int | None):
    """Device tensors for ``shape`` (valid padding: input is w_in x h_in, pad 0)."""
    engine = _engine_for(algorithm)
    key = (shape, layout, algorithm, e, _PADDING[0], engine)
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
    if engine == "ffma":
        prep = C.winograd_filter_transform(w, e) if algorithm == "winograd" else C.pack_filter_direct(w)
    elif engine.startswith("igemm_"):
        prec = engine[len("igemm_"):]
        prep = (C.pack_filter_igemm_bf16(w) if prec == "bf16" else
                C.pack_filter_igemm_f16x3(w) if prec == "3xf16" else C.pack_filter_igemm(w))
    else:
        prep = C.winograd_filter_transform_tc(w, e, engine[len("winograd_tc_"):])
    val = (x, w, y, prep)
    with _lock:
        _cache[key] = val
    return val


def clear_cache() -> None:
    with _lock:
        _cache.clear()


_WS: dict = {}


def _workspace(nbytes: int):
    dev = torch.cuda.current_device()
    buf = _WS.get(dev)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), device=torch.device("cuda", dev), dtype=torch.uint8)
        _WS[dev] = buf
    return buf


def _launcher(cfg: TileConfig, shape: ConvShape, algorithm: str, winograd):
    e = winograd.e if winograd is not None else None
    x, w, y, prep = _tensors(shape, cfg.layout, algorithm, e)
    pad = _PADDING[0]
    engine = _engine_for(algorithm)
    if engine.startswith("igemm_"):
        prec = engine[len("igemm_"):]
        ws = _workspace(2 * x.numel() + (1 << 20))
        return lambda: C.conv_igemm(x, w, padding=pad, stride=shape.stride, tile=cfg, precision=prec,
                                    out=y, w_packed=prep, workspace=ws)
    if engine.startswith("winograd_tc_"):
        prec = engine[len("winograd_tc_"):]
        info = C.query(tuple(x.shape), tuple(w.shape), 1, pad, cfg.layout, cfg, engine)
        ws = _workspace(int(info["workspace_bytes"]))
        return lambda: C.conv_winograd_tc(x, w, e=e, padding=pad, tile=cfg, precision=prec, u=prep,
                                          out=y, workspace=ws)
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
    engine = _engine_for(algorithm)
    alg = (C.ALGORITHMS[engine] if engine != "ffma" else
           (N.ALG_DIRECT if algorithm == "direct" else N.ALG_WINOGRAD))
    rc, _ = N.query(desc, N.make_tile(cfg), alg)
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


# ---------------------------------------------------------------------------
# the tcgen05 kernels' searching domain and the per-layer search
# ---------------------------------------------------------------------------

def tcgen05_hw_model(sms: int = 148) -> HwModel:
    """The reference machine model (model.py:123-156) for the tcgen05 kernels: the
    fast memory of a CTA is its shared memory (the TMA ring, 228 KiB) plus its
    tensor memory (the accumulators, 256 KiB): ``s_sm = 58368 + 65536 = 123904``
    words; one persistent CTA per SM, so ``n_p = 148`` blocks and ``s_b`` up to
    ``s_sm / 2`` words of ring (the model's ``2 s_b <= s_sm`` rule)."""
    s_sm = 228 * 1024 // 4 + 256 * 1024 // 4
    return HwModel(s=sms * (s_sm // 2), s_sm=s_sm, n_p=sms)


def _block_ok(bx: int, by: int, n: int) -> bool:
    """Pixel blocks of the stacked-pixel kernels: x*y <= 128 MMA rows, and either
    >= 32 pixels per image or a divisor of 128 (then 128/(x*y) images fill every
    row: 2x2 blocks x 32 images on 14x14 maps, 1x1 x 128 on 7x7)."""
    px = bx * by
    return px <= 128 and (px >= 32 or (128 % px == 0 and n * px >= 128))


def tcgen05_io_words(shape: ConvShape, tile: TileConfig) -> float:
    """SM <-> L2 words of one implicit-GEMM call with ``tile`` -- the tcgen05
    dataflow's counterpart of the reference's exact reading count (Eq. 17,
    ``analytic_dc_io``'s ``reading_exact``, dataflow.py:388-402): per M tile
    (``rows`` output pixels of ``imgs`` stacked images, or a halo footprint) and
    per N block of ``z`` output channels, the A operand (R*S tap-shifted row
    blocks, or the footprint once per channel block) plus the B operand (z filter
    rows, shared by the two CTAs of a pair), then the outputs once."""
    n, q, p, c, k = shape.n, shape.w_out, shape.h_out, shape.c_in, shape.c_out
    rs = shape.w_ker * shape.h_ker
    if tile.n_zt == 8:   # gather: [imgs][fh][fw] footprint per exact block
        imgs = max(1, min(128 // (tile.x * tile.y), n))
        fw = (tile.x - 1) * shape.stride + shape.w_ker
        fh = (tile.y - 1) * shape.stride + shape.h_ker
        rows_valid = tile.x * tile.y * imgs
        a = fw * fh * imgs * c
    elif tile.n_xt == 2:   # halo: footprint rows (y + R - 1) * fpr, x valid columns per row
        fpr = tile.x + shape.w_ker - 1
        rows_valid = tile.x * tile.y
        a = (tile.y + shape.h_ker - 1) * fpr * c
    else:
        px = tile.x * tile.y
        imgs = max(1, min(128 // px, n))
        rows_valid = px * imgs
        a = px * imgs * c * rs
    tiles_m = -(-(n * p * q) // rows_valid)
    nblocks = max(1, k // tile.z)
    b = tile.z * c * rs / (2 if tile.n_zt >= 2 else 1)
    return tiles_m * nblocks * (a + b) + n * p * q * k


def tcgen05_space(shape: ConvShape, hw: HwModel, engine: str,
                  winograd: WinogradParams | None = None, check_legal: bool = True,
                  prune: float | None = 2.5) -> ConfigSpace:
    """The searching domain of a tcgen05 engine as a reference ``ConfigSpace``.

    The Table-1 rules of ``build_space`` (autotune.py:40-156) are derived for the
    FFMA block whose outputs live in registers (``z^2 R <= s_b``); the tcgen05
    block keeps its outputs in tensor memory and stacks images into the M = 128
    rows, so its domain is enumerated with the machine model's own capacity
    rules (:func:`tcgen05_hw_model`): ``2 s_b <= s_sm`` (the ring fits),
    the accumulator ``128 x z`` fits TMEM twice (``z <= 256``), ``x | Q``,
    ``y | P``, x*y <= 128 rows (pixel blocks per ``_block_ok``), z | K with
    z in {64, 128, 256}; threads select the kernel -- (1,1,1) one CTA,
    (1,1,2) CTA pair, (1,1,4) pair with the split A operand in TMEM, (2,1,2)
    halo-staged footprint (stride 1; ``(x + S - 1) * y = 128``, x not
    necessarily dividing Q), (2,1,4) (3xF16) the halo footprint with the
    converters shifting each tap's rows into TMEM, (1,1,8) (3xF16) exact blocks
    whose [imgs][fh][fw] footprint the converters gather tap by tap into TMEM; Winograd engines: x = y = e, z over the GEMM's N
    tiles, n_zt in {1, 2, 4}.  ``unconstrained_size`` counts the raw product of
    the axes; ``check_legal`` keeps only members with a device projection.
    ``prune`` (implicit GEMM): the I/O-model cut -- members whose modelled SM <-> L2
    traffic (:func:`tcgen05_io_words`) exceeds ``prune`` x the best member's are
    dropped before any device time is spent, the role Table 1 plays for the FFMA
    domain (e.g. z = 64 tiles that re-read the activations K / 64 times)."""
    prec = engine.split("_")[-1]
    q, p, k = shape.w_out, shape.h_out, shape.c_out
    zs = [z for z in (64, 128, 256) if k % z == 0]
    s_bs = [sb for sb in (16384, 32768) if 2 * sb <= hw.s_sm]
    members, raw = [], 0
    if engine.startswith("igemm_"):
        threads = [(1, 1, 1), (1, 1, 2)] + ([(1, 1, 4)] if prec in ("3xtf32", "3xf16") else [])
        if prec == "3xf16":
            threads = [(1, 1, 2), (1, 1, 4)]
        for bx in range(1, q + 1):
            for by in range(1, p + 1):
                for z in zs:
                    for sb in s_bs:
                        for t in threads:
                            raw += 1
                            if q % bx or p % by or not _block_ok(bx, by, shape.n):
                                continue
                            if t[2] >= 2 and sb != 32768:   # persistent pair: the whole smem is the ring
                                continue
                            members.append(TileConfig(bx, by, z, sb, *t, layout="HWC"))
        if prec == "3xf16":   # (1,1,8): exact blocks, footprint gathered into TMEM
            for bx in range(1, q + 1):
                for by in range(1, p + 1):
                    for z in zs:
                        raw += 1
                        if q % bx or p % by or not _block_ok(bx, by, shape.n) or bx * by > 64:
                            continue
                        members.append(TileConfig(bx, by, z, 32768, 1, 1, 8, layout="HWC"))
        if shape.stride == 1:
            for fpr in (8, 16, 32, 64, 128):
                x_, y_ = fpr - shape.w_ker + 1, 128 // fpr
                nzts = (2, 4) if prec == "3xf16" else (2,)   # 4: footprint rows shifted into TMEM
                raw += len(zs) * len(nzts)
                if 1 <= x_ <= q + shape.w_ker - 1 and y_ <= p + shape.h_ker - 1 and x_ % 2 == 0:
                    members += [TileConfig(x_, y_, z, 32768, 2, 1, nz, layout="HWC") for z in zs for nz in nzts]
        if prune and members:
            io = {m: tcgen05_io_words(shape, m) for m in members}
            floor = min(io.values())
            members = [m for m in members if io[m] <= prune * floor]
        algorithm = "direct"
    else:
        # the GEMM's M tile is fixed (128 Winograd tiles per CTA); z = its N tile, s_b
        # sizes the batch chunk (V + M <= 16 KB x s_b), n_zt the GEMM kernel
        e = winograd.e if winograd is not None else 4
        for z in (zs if prec != "fp32" else [z for z in zs if z <= 128]):
            ns = ([(1, 1, 1)] if prec == "fp32" else [(1, 1, 2)] if prec == "3xf16" else
                  [(1, 1, 1), (1, 1, 2)] + ([(1, 1, 4)] if prec == "3xtf32" and z <= 128 else []))
            for sb in (2048, 8192, 16384, 32768):
                for t in ns:
                    raw += 1
                    if 2 * sb <= hw.s_sm:
                        members.append(TileConfig(e, e, z, sb, *t, layout="HWC", e=e))
        algorithm = "winograd"
    members = sorted(set(members), key=lambda c: (LAYOUTS.index(c.layout), c.s_b, c.x, c.y, c.z,
                                                   c.n_xt, c.n_yt, c.n_zt))
    from fractions import Fraction
    space = ConfigSpace(shape, hw, algorithm, winograd,
                        Fraction(shape.w_ker * shape.h_ker, shape.stride ** 2) if algorithm == "direct"
                        else Fraction(winograd.r ** 2 if winograd else 9, 1),
                        tuple(members), raw)
    if check_legal:
        with use_engine(engine):
            space = legal_projection(space)
    return space


def tune_layer(spec, n: int, engines, budget: int = 64, seed: int = 0, log=print) -> dict:
    """The per-layer device search behind the tuned plan tables: for each engine,
    the reference tuner (``tune``: GBR cost model + random walks, backend="device")
    over that engine's searching domain -- the Table-1 projection for "ffma", the
    tcgen05 domain otherwise -- with a budget covering the whole domain when it is
    small (then the result is the exhaustive optimum).  Returns
    ``{engine: {"tuner": {"best", "seconds", "measurements"}, "space": size}}``."""
    from .autotune import tune
    from .device import shape_of
    set_padding(spec.pad)
    shape = shape_of(n, spec.c, spec.hw, spec.hw, spec.k, spec.r, spec.stride, spec.pad)
    out = {}
    for engine in engines:
        wino = engine.startswith("winograd")
        e = int(engine.rsplit("_e", 1)[1]) if "_e" in engine else None
        eng = engine.rsplit("_e", 1)[0] if "_e" in engine else engine
        if wino and (spec.stride != 1 or spec.r != 3):
            continue
        wp = WinogradParams(e, 3) if wino else None
        try:
            with use_engine(eng):
                hw = tcgen05_hw_model()
                space = tcgen05_space(shape, hw, eng, wp)
                sess = tune(shape, hw, "winograd" if wino else "direct", min(budget, space.size), seed,
                            winograd=wp, n_s=min(16, max(2, space.size // 4)), space=space,
                            backend="device")
        except InfeasibleTileError as exc:
            out[engine] = {"error": str(exc)}
            continue
        best = sess.best
        out[engine] = {"tuner": {"best": best.config.to_dict() if best else None,
                                 "seconds": best.cost if best else None,
                                 "measurements": len(sess.measurements)},
                       "space": space.size, "unconstrained": space.unconstrained_size}
        log(f"    {engine}: {space.size} configs, best {best.config if best else None} "
            f"{best.cost if best else None}")
    return out
