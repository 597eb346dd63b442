"""Per-layer runner: named CNN 3x3 conv layer sets, tuned plans, batch sharding.

This is the "step after the path" of SURVEY.md §8(f) item 3: a layer list
(ResNet-50 / VGG-16 3x3 convolutions, the BASELINE.json configs 3-4) whose
per-layer algorithm and tile come from the lower-bound auto-tuner's device
results (``tuned/*.json``), executed through the public conv API.

Batch sharding (BASELINE config 4): rank ``g`` of ``G``
takes images ``[g N/G, (g+1) N/G)``; filters are replicated (same seed on
every rank); outputs stay sharded unless :func:`gather_outputs` is asked to
collect them with an NCCL all-gather.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import torch

from .dataflow import TileConfig
from . import conv as C
from .device import direct_flops

TUNED_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tuned")


@dataclass(frozen=True)
class LayerSpec:
    name: str
    c: int
    hw: int          # input height = width
    k: int
    stride: int = 1
    r: int = 3
    pad: int = 1
    count: int = 1   # identical layers in the network

    @property
    def out_hw(self) -> int:
        return (self.hw + 2 * self.pad - self.r) // self.stride + 1

    def flops(self, n: int) -> int:
        """Direct-convolution algorithmic flops for a batch of ``n`` (one instance)."""
        o = self.out_hw
        return direct_flops(n, self.c, self.k, o, o, self.r, self.r)


# ResNet-50 v1.5 bottleneck 3x3 convolutions (stride on the 3x3), 16 layers
RESNET50_3X3 = [
    LayerSpec("res2_3x3", 64, 56, 64, 1, count=3),
    LayerSpec("res3_3x3_s2", 128, 56, 128, 2),
    LayerSpec("res3_3x3", 128, 28, 128, 1, count=3),
    LayerSpec("res4_3x3_s2", 256, 28, 256, 2),
    LayerSpec("res4_3x3", 256, 14, 256, 1, count=5),
    LayerSpec("res5_3x3_s2", 512, 14, 512, 2),
    LayerSpec("res5_3x3", 512, 7, 512, 1, count=2),
]

# VGG-16: all 13 3x3 convolutions
VGG16_3X3 = [
    LayerSpec("conv1_1", 3, 224, 64), LayerSpec("conv1_2", 64, 224, 64),
    LayerSpec("conv2_1", 64, 112, 128), LayerSpec("conv2_2", 128, 112, 128),
    LayerSpec("conv3_1", 128, 56, 256), LayerSpec("conv3_2", 256, 56, 256, count=2),
    LayerSpec("conv4_1", 256, 28, 512), LayerSpec("conv4_2", 512, 28, 512, count=2),
    LayerSpec("conv5_1", 512, 14, 512, count=3),
]

# BASELINE config 1/2: the single ResNet 3x3 layer at N=1
SINGLE_RESNET = [LayerSpec("res2_3x3", 64, 56, 64, 1)]

WORKLOADS = {"resnet50": RESNET50_3X3, "vgg16": VGG16_3X3, "single": SINGLE_RESNET}
# BASELINE.json batch of each workload (config 4: 256, config 3: 32, configs 1-2: 1)
DEFAULT_BATCH = {"resnet50": 256, "vgg16": 32, "single": 1}


def expand(layers: list[LayerSpec]) -> list[LayerSpec]:
    """One entry per layer instance (``count`` copies)."""
    return [spec for spec in layers for _ in range(spec.count)]


# Algorithms whose results meet the FP32 tolerance (1e-5 normwise vs the float64
# oracle; Winograd F(e,3) is looser by construction, 1e-4 / 1e-3) -- the
# headline plan picks among these; "igemm_tf32" is the reduced-precision variant.
FP32_ALGORITHMS = ("direct", "winograd", "igemm_3xtf32", "winograd_tc_3xtf32", "winograd_nhwc",
                   "winograd_tc_3xf16", "igemm_3xf16")
CUDA_CORE_ALGORITHMS = ("direct", "winograd", "winograd_nhwc")


def candidate_algorithm(key: str) -> tuple[str, int | None]:
    """Tuned-candidate key -> (algorithm, e): ``direct`` / ``direct_nhwc`` (FFMA
    direct, NCHW register micro-tiles / channels-last stacked pixels), ``winograd2|4`` (FFMA
    Winograd), ``winograd_tc_<prec>_e2|4`` (tensor-core Winograd), ``igemm_<prec>``."""
    if key.startswith("winograd_tc_"):
        prec, _, e = key[len("winograd_tc_"):].partition("_e")
        return f"winograd_tc_{prec}", int(e)
    if key.startswith("winograd_nhwc_e"):   # FP32 FFMA element-wise GEMMs, channels-last
        return "winograd_nhwc", int(key[len("winograd_nhwc_e"):])
    if key.startswith("winograd"):
        return "winograd", int(key[len("winograd"):])
    if key == "direct_nhwc":   # the channels-last FFMA direct kernel (an HWC "direct" tile)
        return "direct", None
    return key, None


def tuned_table(workload: str, n: int | None = None) -> str:
    """Path of the tuned table for ``workload``: the per-batch table
    ``b200_<workload>_n<n>.json`` tuned at the local batch of a sharded run
    (strong scaling gives each rank N/G images) when one exists; for a batch no table
    was tuned at, the table tuned at the nearest batch (log scale: its tiles' image
    stacks and grid shapes were chosen for a similar work size); else the table tuned
    at the workload's full batch."""
    default = os.path.join(TUNED_DIR, f"b200_{workload}.json")
    if n is None:
        return default
    path = os.path.join(TUNED_DIR, f"b200_{workload}_n{n}.json")
    if os.path.exists(path):
        return path
    import glob
    import math
    cands = []
    if os.path.exists(default):
        try:
            with open(default) as fh:
                n_tune = json.load(fh).get("n_tune")
        except (OSError, ValueError):
            n_tune = None
        if n_tune:
            cands.append((int(n_tune), default))
    for p in glob.glob(os.path.join(TUNED_DIR, f"b200_{workload}_n*.json")):
        tail = os.path.basename(p)[len(f"b200_{workload}_n"):-len(".json")]
        if tail.isdigit():
            cands.append((int(tail), p))
    if not cands or n < 1:
        return default
    return min(cands, key=lambda c: (abs(math.log(n / c[0])), -c[0]))[1]


def load_plans(workload: str, allowed=FP32_ALGORITHMS, n: int | None = None) -> dict:
    """Tuned per-layer plans ``{name: {"algorithm", "tile", "e"}}`` (empty if untuned).

    Each layer takes the fastest tuned candidate whose algorithm is in ``allowed``;
    ``n`` (local batch) selects a per-batch table when one was tuned.
    """
    path = tuned_table(workload, n)
    if not os.path.exists(path):
        return {}
    with open(path) as fh:
        raw = json.load(fh)
    plans = {}
    for name, entry in raw.get("layers", {}).items():
        best, best_t = None, float("inf")
        for key, cand in entry.get("candidates", {}).items():
            alg, e = candidate_algorithm(key)
            tuned = cand.get("tuner") or {}
            t = tuned.get("seconds")
            if alg not in allowed or t is None or not tuned.get("best"):
                continue
            if t < best_t:
                best, best_t = {"algorithm": alg, "tile": TileConfig(**tuned["best"]), "e": e}, t
        if best is None and entry.get("algorithm") in allowed and entry.get("tile"):
            best = {"algorithm": entry["algorithm"], "tile": TileConfig(**entry["tile"]),
                    "e": entry.get("e")}
        if best is not None:
            plans[name] = best
    return plans


# untuned shapes: CTA-pair tiles tried in order (x, y) -- small pixel blocks of many
# stacked images first (deep layers), larger blocks for wide feature maps
_DEFAULT_XY = [(2, 2), (1, 2), (2, 1), (1, 1), (4, 2), (2, 4), (4, 4), (7, 7), (8, 8), (14, 8), (16, 8)]


def plan_feasible(spec: "LayerSpec", n: int, plan: dict | None) -> bool:
    """Whether ``plan`` runs ``spec`` at batch ``n`` (the library's planner, host only;
    FFMA kernels take any batch)."""
    if not plan or plan.get("tile") is None or plan.get("algorithm") in ("direct", "winograd", "winograd_nhwc"):
        return True
    t = plan["tile"]
    alg = plan["algorithm"]
    try:
        info = C.query((n, spec.c, spec.hw, spec.hw), (spec.k, spec.c, spec.r, spec.r), spec.stride, spec.pad,
                       t.layout, t, alg)
    except Exception:  # noqa: BLE001 -- an unknown algorithm name is infeasible here
        return False
    return info.get("rc", 1) == 0


def default_plan(spec: "LayerSpec", n: int) -> dict:
    """The plan of a layer no tuned table covers (or whose tuned tile does not fit
    batch ``n``): the FP32-accurate 3xF16 implicit GEMM (C % 64 == 0) or 3xTF32 (C % 32
    == 0) on the first CTA-pair tile the planner accepts, else the FFMA direct kernel
    with its default tile -- instead of always falling back to FFMA."""
    for alg, cmod in (("igemm_3xf16", 64), ("igemm_3xtf32", 32)):
        if spec.c % cmod:
            continue
        for z in (256, 128, 64):
            if spec.k % z:
                continue
            for nzt in (2, 4):
                for x, y in _DEFAULT_XY:
                    plan = {"algorithm": alg, "tile": TileConfig(x, y, z, 32768, 1, 1, nzt, layout="HWC"), "e": None}
                    if plan_feasible(spec, n, plan):
                        return plan
    return {"algorithm": "direct", "tile": None, "e": None}


def plan_for(spec: "LayerSpec", n: int, plans: dict) -> dict:
    """``plans[spec.name]`` when it runs at batch ``n``, else :func:`default_plan`."""
    plan = plans.get(spec.name)
    return plan if plan is not None and plan_feasible(spec, n, plan) else default_plan(spec, n)


# 3xF16 implicit GEMM: the speculative activation-scale state (tagged max |x| of the
# previous call + one observed max per CTA) at the start of the layer's workspace; it
# persists across calls, which is what lets the second and later calls skip the redo
F16X3_PARTIALS_BYTES = 256 * ((4 * 296 + 255) // 256)


def _f16x3_filter_bytes(s: "LayerSpec") -> int:
    from . import _native as N
    import ctypes
    desc = N.make_desc(1, s.c, s.r, s.r, s.k, s.r, s.r, 1, 0, 2)
    return int(N.lib().convio_pack_filter_igemm_f16x3_bytes(ctypes.byref(desc)))


def _on(t: torch.Tensor, device) -> bool:
    """``t`` lives on ``device`` ("cuda" meaning the current CUDA device)."""
    d = torch.device(device)
    if d.type == "cuda" and d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return t.device == d


class LayerGroup:
    """``G`` independent layers of one shape and one 3xF16 implicit-GEMM plan run as ONE
    persistent launch (``conv.conv_igemm_grouped``, like a grouped GEMM): their inputs and
    outputs are slices of stacked buffers, their packed filters slices of one buffer (the
    layers' own filter workspaces point into it, so :func:`prepare_layers` fills it).
    Saves the per-layer launch, ramp, drain, last-round imbalance and checking launch."""

    def __init__(self, layers, n: int, device):
        s = layers[0].spec
        self.layers, self.n, self.spec = layers, n, s
        self.tile = layers[0].tile
        g = len(layers)
        self.slice_bytes = C.f16x3_slice_bytes(s.k, s.c, s.r, s.r)
        self.wbuf = torch.zeros(g * self.slice_bytes, dtype=torch.uint8, device=device)
        for i, l in enumerate(layers):
            off = i * self.slice_bytes
            l._ws = self.wbuf[off:off + 4 * l.filter_elems()].view(torch.float32)
        self.x = C.empty_act(g * n, s.c, s.hw, s.hw, "HWC", device=device)
        self.y = C.empty_act(g * n, s.k, s.out_hw, s.out_hw, "HWC", device=device)
        biases = [l.bias for l in layers]
        self.bias = torch.cat(biases) if all(b is not None for b in biases) else None
        if self.bias is None and any(b is not None for b in biases):
            raise ValueError("a group's layers must all have a bias or none")
        self.relu = layers[0].relu
        self.ws = torch.zeros(4096, dtype=torch.uint8, device=device)   # activation-scale state
        self.launches = 0

    def x_of(self, i: int) -> torch.Tensor:
        return self.x[i * self.n:(i + 1) * self.n]

    def y_of(self, i: int) -> torch.Tensor:
        return self.y[i * self.n:(i + 1) * self.n]

    def run(self, stream=None) -> torch.Tensor:
        s = self.spec
        C.conv_igemm_grouped(self.x, (s.k, s.c, s.r, s.r), self.wbuf, len(self.layers), self.slice_bytes,
                             padding=s.pad, stride=s.stride, tile=self.tile, bias=self.bias, relu=self.relu,
                             out=self.y, stream=stream, workspace=self.ws)
        self.launches = C.last_launch_count()
        return self.y


def group_table(workload: str) -> str:
    """Path of the grouped-launch table (``scripts/tune_groups.py``)."""
    return os.path.join(TUNED_DIR, f"b200_{workload}_groups.json")


def load_group_plans(workload: str, n: int) -> dict:
    """``{layer name: TileConfig | None}`` for the grouped launches at per-layer batch
    ``n``: the fastest measured tile for the G-layer launch (a G*n-image GEMM prefers
    the tiles tuned at larger batches), None where G single launches measured faster,
    ``{}`` when untuned."""
    try:
        with open(group_table(workload)) as fh:
            tab = json.load(fh)
    except (OSError, ValueError):
        return {}
    out = {}
    for name, ent in tab.get("groups", {}).get(str(n), {}).items():
        if not ent.get("use_group", True):
            out[name] = None
        elif ent.get("tile"):
            out[name] = TileConfig(**ent["tile"])
    return out


def load_group_overrides(workload: str, n: int) -> dict:
    """Plans ``{layer name: {"algorithm": "igemm_3xf16", "tile", "e"}}`` that replace a
    repeated layer's own plan (e.g. res5's Winograd) because its grouped 3xF16 launch,
    filter prep included, measured faster (``scripts/tune_groups.py``)."""
    try:
        with open(group_table(workload)) as fh:
            tab = json.load(fh)
    except (OSError, ValueError):
        return {}
    return {name: {"algorithm": ent["algorithm"], "tile": TileConfig(**ent["tile"]), "e": None}
            for name, ent in tab.get("groups", {}).get(str(n), {}).items()
            if ent.get("replaces") and ent.get("use_group", True)}


def group_stack_ok(tile: TileConfig, n: int, layers: int) -> bool:
    """Whether a grouped launch of ``layers`` x ``n`` images can use ``tile``: its CTA-pair
    blocks stack ``min(128 / (x y), layers * n)`` images (1 for halo tiles), and a stack
    must not straddle two layers (convio_conv_igemm_grouped)."""
    if tile.n_zt < 2:
        return False
    imgs = 1 if tile.n_xt == 2 else max(1, min(128 // (tile.x * tile.y), layers * n))
    return n % imgs == 0


def group_layers(layers, n: int, device, group_plans: dict | None = None) -> list:
    """Runs of consecutive layers with the same shape and the same 3xF16 implicit-GEMM
    plan (CTA-pair tiles whose image stack divides ``n``) as :class:`LayerGroup`; other
    layers stay single.  ``group_plans`` (:func:`load_group_plans`) may give a group
    its own tile.  Returns units ``(kind, obj, [layer indices])``."""
    units, i = [], 0
    while i < len(layers):
        l = layers[i]
        j = i + 1
        if l.algorithm == "igemm_3xf16" and l.tile is not None and l.tile.n_zt >= 2:
            while (j < len(layers) and layers[j].algorithm == "igemm_3xf16" and layers[j].spec == l.spec
                   and layers[j].tile == l.tile and (layers[j].bias is None) == (l.bias is None)):
                j += 1
        if j - i >= 2 and group_plans and l.spec.name in group_plans and group_plans[l.spec.name] is None:
            j = i + 1   # measured: single launches win for this group
        tile = group_plans.get(l.spec.name) if group_plans else None
        tile = tile or l.tile
        if j - i >= 2 and not group_stack_ok(tile, n, j - i):
            j = i + 1   # e.g. an untabled batch whose image stacks would straddle layers
        if j - i >= 2:
            try:
                grp = LayerGroup(layers[i:j], n, device)
                grp.tile = tile
                units.append(("group", grp, list(range(i, j))))
            except ValueError:
                units += [("single", layers[k], [k]) for k in range(i, j)]
        else:
            units += [("single", layers[k], [k]) for k in range(i, j)]
        i = j
    return units


def prepare_layers(layers, device, stream=None) -> int:
    """Filter prep of a whole step: the 3xF16 implicit-GEMM layers' fp16 splits in ONE
    launch (``convio_pack_filters_igemm_f16x3_batched``), the tensor-core Winograd
    transforms one launch per (e, precision) group, every other layer its own prep.
    Returns the number of launches."""
    import ctypes
    from . import _native as N
    f16 = [l for l in layers if l.algorithm == "igemm_3xf16"]
    launches = 0
    for i in range(0, len(f16), 32):
        chunk = f16[i:i + 32]
        jobs = [l._f16x3_pack_job(device) for l in chunk]
        descs = (N.ConvDesc * len(jobs))(*[j[0] for j in jobs])
        ws = (ctypes.c_void_p * len(jobs))(*[j[1].data_ptr() for j in jobs])
        outs = (ctypes.c_void_p * len(jobs))(*[j[2].data_ptr() for j in jobs])
        N.check(N.lib().convio_pack_filters_igemm_f16x3_batched(len(jobs), descs, ws, outs,
                                                                 C._stream_ptr(stream)),
                "pack_filters_igemm_f16x3_batched")
        launches += 1
    # tensor-core Winograd filter transforms with an fp32 U, grouped by (e, precision)
    groups = {}
    for l in layers:
        if l.algorithm.startswith("winograd_tc") and l.precision in ("tf32", "3xtf32", "3xf16"):
            groups.setdefault((l.e, l.precision), []).append(l)
    batched = {id(l) for g in groups.values() for l in g}
    for (e, prec), g in groups.items():
        for i in range(0, len(g), 32):
            chunk = g[i:i + 32]
            descs, ws, us = [], [], []
            for l in chunk:
                s = l.spec
                if l._ws is None or not _on(l._ws, device) or l._ws.dtype != torch.float32:
                    l._ws = torch.empty(l.filter_elems(), device=device, dtype=torch.float32)
                descs.append(N.make_desc(1, s.c, max(s.hw, s.r), max(s.hw, s.r), s.k, s.r, s.r, 1, 0, 2))
                ws.append(l.weight.data_ptr())
                us.append(l._ws.data_ptr())
            N.check(N.lib().convio_winograd_filter_transform_tc_batched(
                len(chunk), (N.ConvDesc * len(chunk))(*descs), e, N.PRECISIONS[prec],
                (ctypes.c_void_p * len(chunk))(*ws), (ctypes.c_void_p * len(chunk))(*us),
                C._stream_ptr(stream)), "winograd_filter_transform_tc_batched")
            launches += C.last_launch_count()
    for l in layers:
        if l.algorithm != "igemm_3xf16" and id(l) not in batched:
            l.prepare(device, stream)
            launches += 1
    return launches


class ConvLayer:
    """One conv layer: filters on the device plus its tuned plan."""

    def __init__(self, spec: LayerSpec, weight: torch.Tensor, plan: dict | None = None):
        self.spec = spec
        self.weight = weight
        plan = plan or {}
        self.algorithm = plan.get("algorithm", "direct")
        self.tile = plan.get("tile")
        self.e = plan.get("e") or (self.tile.e if self.tile is not None and self.tile.e else 2)
        if self.algorithm.startswith("winograd") and (spec.stride != 1 or spec.r != 3):
            self.algorithm = "direct"
            self.tile = None
        self._ws = None
        self._run_ws = None
        self.launches = 0
        # fused epilogue of a network layer (network.py): bias per output channel, ReLU
        self.bias: torch.Tensor | None = None
        self.relu = False

    @property
    def precision(self) -> str | None:
        """Operand precision of a tensor-core plan (tf32 / 3xtf32 / bf16), else None."""
        if self.algorithm == "winograd_nhwc":
            return "fp32"
        for prefix in ("igemm_", "winograd_tc_"):
            if self.algorithm.startswith(prefix):
                return self.algorithm[len(prefix):]
        return None

    @property
    def layout(self) -> str:
        """Activation layout this layer's plan runs in (HWC for the tensor-core GEMM)."""
        return self.tile.layout if self.tile is not None else "CHW"

    def filter_elems(self) -> int:
        s = self.spec
        if self.algorithm.startswith("winograd"):
            m = self.e + s.r - 1
            if self.algorithm == "winograd_tc_3xf16":   # fp32 U + fp16 hi / lo planes + exponents
                return m * m * s.k * (2 * s.c + 1)
            return m * m * s.c * s.k
        if self.algorithm == "igemm_3xf16":   # fp16 hi / lo planes + per-channel exponents
            return -(-_f16x3_filter_bytes(s) // 4)
        return s.k * s.c * s.r * s.r

    def prepare(self, device, stream=None) -> None:
        """Filter prep into the layer's workspace: KCRS repack (direct) or U = G g G^T."""
        import ctypes
        from . import _native as N
        s = self.spec
        prec = self.precision
        dtype = torch.bfloat16 if prec == "bf16" else torch.float32
        if self._ws is None or not _on(self._ws, device) or self._ws.dtype != dtype:
            self._ws = torch.empty(self.filter_elems(), device=device, dtype=dtype)
        w = self.weight
        desc = N.make_desc(1, s.c, max(s.hw, s.r), max(s.hw, s.r), s.k, s.r, s.r, 1, 0,
                           2 if prec else 0)
        sp = C._stream_ptr(stream)
        if self.algorithm.startswith("winograd_tc") or self.algorithm == "winograd_nhwc":
            rc = N.lib().convio_winograd_filter_transform_tc(ctypes.byref(desc), self.e,
                                                             N.PRECISIONS[prec], C._ptr(w),
                                                             C._ptr(self._ws), sp)
        elif self.algorithm == "igemm_bf16":
            rc = N.lib().convio_pack_filter_igemm_bf16(ctypes.byref(desc), C._ptr(w),
                                                       C._ptr(self._ws), sp)
        elif self.algorithm == "igemm_3xf16":
            rc = N.lib().convio_pack_filter_igemm_f16x3(ctypes.byref(desc), C._ptr(w),
                                                        C._ptr(self._ws), sp)
        elif self.algorithm == "winograd":
            rc = N.lib().convio_winograd_filter_transform(ctypes.byref(desc), self.e,
                                                          C._ptr(w), C._ptr(self._ws), sp)
        elif self.algorithm.startswith("igemm"):
            rc = N.lib().convio_pack_filter_igemm(ctypes.byref(desc), C._ptr(w),
                                                  C._ptr(self._ws), sp)
        else:
            rc = N.lib().convio_pack_filter_direct(ctypes.byref(desc), C._ptr(w),
                                                   C._ptr(self._ws), sp)
        N.check(rc, "filter prep")

    def _f16x3_pack_job(self, device):
        """(descriptor, filter, packed buffer) of this layer's 3xF16 filter prep."""
        from . import _native as N
        s = self.spec
        if self._ws is None or not _on(self._ws, device) or self._ws.dtype != torch.float32:
            self._ws = torch.empty(self.filter_elems(), device=device, dtype=torch.float32)
        desc = N.make_desc(1, s.c, max(s.hw, s.r), max(s.hw, s.r), s.k, s.r, s.r, 1, 0, 2)
        return desc, self.weight, self._ws

    def run(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """The conv kernel alone, on the prepared filter."""
        s = self.spec
        if self.algorithm.startswith("winograd_tc") or self.algorithm == "winograd_nhwc":
            if self._run_ws is None or self._run_ws.device != x.device:
                info = C.query(tuple(x.shape), tuple(self.weight.shape), 1, s.pad, "HWC",
                               self.tile, self.algorithm)
                self._run_ws = torch.empty(max(1, info["workspace_bytes"]), device=x.device,
                                           dtype=torch.uint8)
            y = C.conv_winograd_tc(x, self.weight, e=self.e, padding=s.pad, tile=self.tile,
                                   precision=self.precision, out=out, stream=stream,
                                   u=self._ws, workspace=self._run_ws, bias=self.bias, relu=self.relu)
        elif self.algorithm == "igemm_bf16":
            if self._run_ws is None or self._run_ws.device != x.device:
                self._run_ws = torch.empty(2 * x.numel() + (1 << 20), device=x.device,
                                           dtype=torch.uint8)
            y = C.conv_igemm(x, self.weight, padding=s.pad, stride=s.stride, tile=self.tile,
                             precision="bf16", out=out, stream=stream, w_packed=self._ws,
                             workspace=self._run_ws, bias=self.bias, relu=self.relu)
        elif self.algorithm == "igemm_3xf16":
            if self._run_ws is None or self._run_ws.device != x.device:
                self._run_ws = torch.empty(F16X3_PARTIALS_BYTES, device=x.device, dtype=torch.uint8)
            y = C.conv_igemm(x, self.weight, padding=s.pad, stride=s.stride, tile=self.tile,
                             precision="3xf16", out=out, stream=stream, w_packed=self._ws,
                             workspace=self._run_ws, bias=self.bias, relu=self.relu)
        elif self.algorithm == "winograd":
            u = self._ws.view(-1)
            y = C.conv_winograd(x, self.weight, e=self.e, padding=s.pad, tile=self.tile, out=out,
                                stream=stream, u=u, bias=self.bias, relu=self.relu)
        elif self.algorithm.startswith("igemm"):
            y = C.conv_igemm_tf32(x, self.weight, padding=s.pad, tile=self.tile, out=out,
                                  stream=stream, w_packed=self._ws, stride=s.stride,
                                  split=self.algorithm == "igemm_3xtf32", bias=self.bias, relu=self.relu)
        else:
            wp = self._ws.view(s.c, s.r, s.r, s.k)
            y = C.conv_direct(x, self.weight, stride=s.stride, padding=s.pad, tile=self.tile,
                              out=out, stream=stream, w_packed=wp, bias=self.bias, relu=self.relu)
        self.launches = C.last_launch_count()
        return y

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Filter prep + conv (two kernel launches)."""
        self.prepare(x.device, stream)
        y = self.run(x, out, stream)
        self.launches += 1
        return y


def make_weights(spec: LayerSpec, device, seed: int) -> torch.Tensor:
    """``w ~ U(-1, 1) / sqrt(C R S)``, same on every rank."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    w = (torch.rand((spec.k, spec.c, spec.r, spec.r), generator=g) * 2 - 1)
    return (w / (spec.c * spec.r * spec.r) ** 0.5).to(device)


def make_input(spec: LayerSpec, n: int, device, seed: int, layout: str = "CHW") -> torch.Tensor:
    """``x ~ U(-1, 1)`` generated on the device (seeded per layer and rank)."""
    g = torch.Generator(device=device).manual_seed(seed)
    x = C.empty_act(n, spec.c, spec.hw, spec.hw, layout, device=device)
    x.uniform_(-1.0, 1.0, generator=g)
    return x


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous image range of ``rank`` (SURVEY.md §8(e) partitioning)."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_outputs(y_local: torch.Tensor, world: int) -> torch.Tensor:
    """All-gather of equal batch shards into the full output (only when collecting).

    NCCL (NVLink / NVSwitch) on GPUs via ``all_gather_into_tensor``; the list
    form on backends without it (gloo, used by the CPU tests).
    """
    import torch.distributed as dist
    y_local = y_local.contiguous()
    if dist.get_backend() == "nccl":
        out = torch.empty((world * y_local.shape[0],) + tuple(y_local.shape[1:]),
                          device=y_local.device, dtype=y_local.dtype)
        dist.all_gather_into_tensor(out, y_local)
        return out
    parts = [torch.empty_like(y_local) for _ in range(world)]
    dist.all_gather(parts, y_local)
    return torch.cat(parts, 0)
