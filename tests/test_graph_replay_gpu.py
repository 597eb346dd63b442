"""The bench's timing path: every tuned ResNet-50 plan (3xTF32 fold / pair /
A-in-TMEM / split-K implicit GEMM, unchunked tensor-core Winograd, all launched
with programmatic dependent launch) captured into one CUDA graph and replayed;
each layer's replayed output must match its eager output and the float64 oracle
(on a 2-image slice), so the graph-timed headline computes what the tests check."""

import numpy as np
import pytest
import torch

from oracle import conv_oracle as co
from paper_2012_15667_b200 import conv as C
from paper_2012_15667_b200 import runner as R

pytestmark = pytest.mark.gpu

from tolerances import tol_for  # noqa: E402


def test_tuned_resnet50_plans_replay_in_a_cuda_graph():
    dev = torch.device("cuda:0")
    n = 8
    plans = R.load_plans("resnet50", n=256)
    assert plans, "tuned table missing"
    layers, xs, ys = [], [], []
    for i, spec in enumerate(R.WORKLOADS["resnet50"]):
        layer = R.ConvLayer(spec, R.make_weights(spec, dev, seed=i), plans.get(spec.name))
        x = C.to_layout(R.make_input(spec, n, dev, seed=100 + i), layer.layout)
        layer.prepare(dev)
        layers.append(layer)
        xs.append(x)
        ys.append(layer.run(x))
        # a second eager call: the steady state the graph replays (3xF16 implicit GEMMs
        # speculate their activation scale from the previous call on the same workspace;
        # the first call on a fresh one takes the exact-scale fallback with whole-K tiles)
        layer.run(x, out=ys[-1])
    torch.cuda.synchronize()
    eager = [y.clone() for y in ys]
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for layer, x, y in zip(layers, xs, ys):
            layer.prepare(dev, stream=side)
            layer.run(x, out=y, stream=side)
    for y in ys:
        y.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    for layer, x, y, ye in zip(layers, xs, ys, eager):
        s = layer.spec
        assert torch.isfinite(y).all(), s.name
        assert torch.allclose(y, ye, rtol=0, atol=1e-5 * float(ye.abs().max())), s.name
        xc = x[:2].contiguous().cpu().numpy()   # logical NCHW whatever the physical layout
        ref = co.direct_conv(xc, layer.weight.cpu().numpy(), s.stride, s.pad)
        err = co.rel_err(y[:2].contiguous().cpu().numpy(), ref)
        tol = tol_for(layer.algorithm, s.c, layer.e)
        assert err <= tol, (s.name, layer.algorithm, err, tol)
