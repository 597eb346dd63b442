"""Chained network forward: VGG-16's convolutional feature extractor end to end
(SURVEY.md §8(f) item 3 -- the step after the path; the paper's end-to-end
claims, are whole-network runs).

The 13 3x3 convolutions run the plans the device tuner picked for their shapes
(``tuned/b200_vgg16.json``, the same table the per-layer bench uses), each with
its bias and ReLU fused into the conv kernel's epilogue; the 2x2 max pools and
the NCHW -> NHWC staging of the input are library kernels too
(``convio_maxpool2x2_nhwc``, ``convio_nchw_to_nhwc``), so every launch of a
forward is ours and counted.  Activations stay channels-last on the device
between layers; the input arrives as NCHW (a host tensor or a device tensor)
and the features can be returned NCHW (``convio_nhwc_to_nchw``).

Filter preparation (repacking / Winograd transforms / fp16 splits) happens once
in :meth:`Vgg16Features.prepare`, as a deployed network would cache it; a
forward is then ``1 + 13 + 5`` kernel launches (+ the 3xF16 layers' checking
launches, which exit at once when the speculated activation scale held),
capturable as one CUDA graph.
"""

from __future__ import annotations

import torch

from . import conv as C
from .dataflow import TileConfig
from .runner import VGG16_3X3, ConvLayer, load_plans, make_weights, plan_for

# the 13 convolutions in order, "M" = 2x2 max pool; names map to the tuned table's
# layer shapes (conv3_3 has conv3_2's shape, conv4_3 conv4_2's, conv5_x conv5_1's)
VGG16_SEQUENCE = ("conv1_1", "conv1_2", "M", "conv2_1", "conv2_2", "M", "conv3_1", "conv3_2",
                  "conv3_3", "M", "conv4_1", "conv4_2", "conv4_3", "M", "conv5_1", "conv5_2",
                  "conv5_3", "M")
_SHAPE_OF = {"conv3_3": "conv3_2", "conv4_3": "conv4_2", "conv5_2": "conv5_1", "conv5_3": "conv5_1"}

# conv1_1 (C = 3) in the channels-last chain: the small-C direct kernel K8 on the
# NHWC input (the NCHW register micro-tile K1 would need the 64-channel output
# transposed instead of the 3-channel input)
CONV1_1_HWC = TileConfig(16, 16, 32, 32768, 1, 1, 1, layout="HWC")


class Vgg16Features:
    """VGG-16 conv features for ``n`` 224 x 224 RGB images on one GPU."""

    def __init__(self, n: int, device, seed: int = 0, plans: dict | None = None):
        self.n = n
        self.device = torch.device(device)
        specs = {s.name: s for s in VGG16_3X3}
        plans = load_plans("vgg16", n=n) if plans is None else plans
        self.layers: list[ConvLayer | None] = []
        g = torch.Generator(device=self.device).manual_seed(seed + 77)
        for i, name in enumerate(VGG16_SEQUENCE):
            if name == "M":
                self.layers.append(None)
                continue
            spec = specs[_SHAPE_OF.get(name, name)]
            # (a table tuned at another batch may hold tiles this batch cannot take)
            plan = dict(plan_for(spec, n, plans))
            if name == "conv1_1" or (plan.get("tile") is not None and plan["tile"].layout != "HWC"):
                plan = {"algorithm": "direct", "tile": CONV1_1_HWC if spec.c <= 4 else None, "e": None}
            layer = ConvLayer(spec, make_weights(spec, self.device, seed + i), plan)
            layer.name = name
            layer.bias = (torch.rand(spec.k, device=self.device, generator=g) - 0.5) * 0.1
            layer.relu = True
            self.layers.append(layer)
        self._acts = None
        self._prepared = False

    @property
    def conv_layers(self) -> list[ConvLayer]:
        return [l for l in self.layers if l is not None]

    def flops(self) -> int:
        return sum(l.spec.flops(self.n) for l in self.conv_layers)

    def prepare(self, stream=None) -> None:
        """Filter preparation of every layer, once."""
        for layer in self.conv_layers:
            layer.prepare(self.device, stream)
        self._prepared = True

    def _buffers(self):
        """Channels-last activation buffers for every step of the chain."""
        if self._acts is None:
            acts, c, hw = [C.empty_act(self.n, 3, 224, 224, "HWC", device=self.device)], 3, 224
            for layer in self.layers:
                if layer is None:
                    hw //= 2
                else:
                    c = layer.spec.k
                acts.append(C.empty_act(self.n, c, hw, hw, "HWC", device=self.device))
            self._acts = acts
        return self._acts

    def forward(self, x: torch.Tensor, stream=None, nchw_out: bool = False) -> torch.Tensor:
        """Features (n, 512, 7, 7) of the NCHW batch ``x`` (device tensor), channels-last
        unless ``nchw_out``; every launch is a library kernel."""
        if not self._prepared:
            self.prepare(stream)
        if tuple(x.shape) != (self.n, 3, 224, 224):
            raise ValueError(f"expected a ({self.n}, 3, 224, 224) input, got {tuple(x.shape)}")
        acts = self._buffers()
        n = self.n
        N = C.N
        C.N.check(N.lib().convio_nchw_to_nhwc(C._ptr(x.contiguous()), C._ptr(acts[0]), n, 3, 224, 224,
                                               C._stream_ptr(stream)), "nchw_to_nhwc")
        h = acts[0]
        for i, layer in enumerate(self.layers):
            out = acts[i + 1]
            if layer is None:
                C.maxpool2x2(h, out=out, stream=stream)
            else:
                layer.run(h, out=out, stream=stream)
            h = out
        if nchw_out:
            return C.to_layout(h, "CHW", stream=stream)
        return h

    def launches_per_forward(self) -> int:
        """Kernel launches of one forward after :meth:`prepare` (layout kernel,
        convs with their auxiliary launches, pools)."""
        return 1 + sum(1 if l is None else max(1, l.launches) for l in self.layers)
