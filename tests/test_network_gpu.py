"""The steps either side of the conv path and the chained network forward
(SURVEY.md §8(f) items 2-3): NCHW <-> NHWC staging and 2x2 max pooling kernels
(bit-exact: pure data movement / max), and VGG-16's 13 convolutions + 5 pools
chained through the tuned plans with fused bias + ReLU, against a float64
reference of the same network (the per-layer conv oracle is
oracle/conv_oracle.py, restating reference pkg/src/convio/dag.py:247-285; the
composition is checked against float64 torch convolutions on the device)."""

import numpy as np
import pytest
import torch

from paper_2012_15667_b200 import conv as C
from paper_2012_15667_b200.network import Vgg16Features, VGG16_SEQUENCE

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(2, 3, 224, 224), (3, 64, 28, 28), (1, 37, 5, 9), (2, 256, 14, 14)])
def test_layout_kernels_are_exact_transposes(shape):
    x = torch.randn(shape, device="cuda")
    y = C.to_layout(x, "HWC")
    assert C.infer_layout(y) == "HWC" and torch.equal(y, x)
    z = C.to_layout(y, "CHW")
    assert C.infer_layout(z) == "CHW" and torch.equal(z, x)
    assert C.last_launch_count() == 1   # one library kernel, not a framework copy


@pytest.mark.parametrize("shape", [(2, 64, 224, 224), (3, 512, 14, 14), (1, 8, 7, 9)])
def test_maxpool_matches_torch(shape):
    x = C.to_layout(torch.randn(shape, device="cuda"), "HWC")
    y = C.maxpool2x2(x)
    assert torch.equal(y, torch.nn.functional.max_pool2d(x, 2))


def _reference(net, x):
    h = x.double()
    for layer in net.layers:
        if layer is None:
            h = torch.nn.functional.max_pool2d(h, 2)
        else:
            h = torch.nn.functional.conv2d(h, layer.weight.double(), layer.bias.double(), padding=1)
            h = torch.relu(h)
    return h


def test_vgg16_chained_forward_matches_float64():
    torch.backends.cudnn.allow_tf32 = False
    net = Vgg16Features(2, "cuda", seed=3)
    x = torch.rand((2, 3, 224, 224), device="cuda") * 2 - 1
    y = net.forward(x, nchw_out=True)
    torch.cuda.synchronize()
    ref = _reference(net, x)
    assert y.shape == (2, 512, 7, 7)
    err = float((y.double() - ref).abs().max() / ref.abs().max())
    # 13 FP32-level layers (3xF16 / 3xTF32 / FFMA, Winograd F(4,3) on the deep ones):
    # the per-layer bounds (tests/tolerances.py) compound to ~1e-4
    assert err <= 1e-4, err
    assert err > 0.0
    algs = [l.algorithm for l in net.conv_layers]
    assert algs[0] == "direct" and any(a.startswith("igemm") for a in algs), algs


def test_vgg16_forward_replays_in_a_cuda_graph():
    net = Vgg16Features(2, "cuda", seed=5)
    x = torch.rand((2, 3, 224, 224), device="cuda") * 2 - 1
    net.prepare()
    eager = net.forward(x).clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        net.forward(x, stream=side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        out = net.forward(x, stream=side)
    out.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    assert len(VGG16_SEQUENCE) == 18
