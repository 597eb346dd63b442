"""Every committed plan table, replayed at the batch it was tuned for (and the
bench measures), against the C oracle on the first and last two images of each
layer: the persistent CTA-pair work lists, split-K decisions, Winograd chunking
and grid shapes all depend on the batch, so the benchmarked configuration itself
is what is checked here (tables: ResNet-50 n=256 and its n=128/64/32 shard
tables, VGG-16 n=32, the single layer n=1).  Through the C-ABI, via the runner
the bench uses (filter prep + conv)."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import conv_oracle as co
from paper_2012_15667_b200 import runner as R

from tolerances import tol_for

pytestmark = pytest.mark.gpu

TABLES = [("resnet50", 256), ("resnet50", 128), ("resnet50", 64), ("resnet50", 32),
          ("vgg16", 32), ("single", 1)]
# the plan sets the bench times: the FP32-accurate headline and its variants
PLAN_SETS = {
    "fp32": R.FP32_ALGORITHMS,
    "cuda_cores": R.CUDA_CORE_ALGORITHMS,
    "tf32": ("igemm_tf32", "winograd_tc_tf32"),
    "bf16": ("igemm_bf16", "winograd_tc_bf16"),
}
CASES = [(w, n, "fp32") for w, n in TABLES] + [("resnet50", 256, v) for v in ("cuda_cores", "tf32", "bf16")]


def _edge_images(n):
    return sorted({0, min(1, n - 1), max(0, n - 2), n - 1})


@pytest.mark.parametrize("workload,n,plan_set", CASES, ids=[f"{w}-n{n}-{p}" for w, n, p in CASES])
def test_plan_table_at_its_batch_matches_oracle(workload, n, plan_set):
    path = R.tuned_table(workload, n)
    with open(path) as fh:
        tuned_n = json.load(fh).get("n_tune")
    assert tuned_n in (None, n), f"{os.path.basename(path)} was tuned at n={tuned_n}"
    plans = R.load_plans(workload, PLAN_SETS[plan_set], n=n)
    assert plans, f"no {plan_set} plans in {os.path.basename(path)}"
    dev = torch.device("cuda:0")
    imgs = _edge_images(n)
    for i, spec in enumerate(R.expand(R.WORKLOADS[workload])):
        plan = plans.get(spec.name)
        if plan is None:
            continue
        layer = R.ConvLayer(spec, R.make_weights(spec, dev, seed=1000 + i), plan)
        x = R.make_input(spec, n, dev, seed=7919 * (i + 1), layout=layer.layout)
        y = layer.forward(x)
        torch.cuda.synchronize()
        xs = x[imgs].contiguous().cpu().numpy()    # logical NCHW whatever the physical layout
        ref = co.c_direct_conv(xs, layer.weight.cpu().numpy(), spec.stride, spec.pad)
        err = co.rel_err(y[imgs].contiguous().cpu().numpy(), ref)
        tol = tol_for(layer.algorithm, spec.c, layer.e)
        assert err <= tol, (spec.name, layer.algorithm, layer.tile, err, tol)
        del x, y


@pytest.mark.parametrize("workload,n", [("resnet50", 256), ("resnet50", 128), ("resnet50", 64), ("resnet50", 32),
                                        ("vgg16", 32)])
def test_grouped_units_at_bench_batch_match_oracle(workload, n):
    """The timed step as bench.py runs it: the group table's plan overrides and tiles,
    each group of repeated layers in ONE grouped launch over the stacked batch, after
    the step's batched filter prep -- every layer of every group against the C oracle
    on its first and last two images."""
    plans = R.load_plans(workload, n=n)
    plans.update(R.load_group_overrides(workload, n))
    dev = torch.device("cuda:0")
    specs = R.expand(R.WORKLOADS[workload])
    layers = [R.ConvLayer(s, R.make_weights(s, dev, seed=1000 + i), plans.get(s.name)) for i, s in enumerate(specs)]
    units = R.group_layers(layers, n, dev, R.load_group_plans(workload, n))
    groups = [(u, idx) for kind, u, idx in units if kind == "group"]
    assert groups, "the bench step has grouped launches at this batch"
    for u, idx in groups:
        for g, i in enumerate(idx):
            u.x_of(g).copy_(R.make_input(specs[i], n, dev, seed=7919 * (i + 1), layout="HWC"))
    R.prepare_layers(layers, dev)
    imgs = _edge_images(n)
    for u, idx in groups:
        u.run()
        torch.cuda.synchronize()
        for g, i in enumerate(idx):
            spec, layer = specs[i], layers[i]
            xs = u.x_of(g)[imgs].contiguous().cpu().numpy()
            ref = co.c_direct_conv(xs, layer.weight.cpu().numpy(), spec.stride, spec.pad)
            err = co.rel_err(u.y_of(g)[imgs].contiguous().cpu().numpy(), ref)
            tol = tol_for("igemm_3xf16", spec.c, None)
            assert err <= tol, (spec.name, g, u.tile, err, tol)
    del units, groups, layers
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shape", [(192, 17, 192, 1), (512, 7, 512, 1), (256, 28, 512, 2), (96, 35, 96, 1)])
def test_default_plan_matches_oracle(shape):
    """runner.default_plan (untuned shapes) through the runner, against the C oracle."""
    c, hw, k, stride = shape
    spec = R.LayerSpec("untuned", c, hw, k, stride=stride)
    n = 3
    dev = torch.device("cuda:0")
    plan = R.default_plan(spec, n)
    layer = R.ConvLayer(spec, R.make_weights(spec, dev, seed=5), plan)
    x = R.make_input(spec, n, dev, seed=11, layout=layer.layout)
    y = layer.forward(x)
    torch.cuda.synchronize()
    ref = co.c_direct_conv(x.contiguous().cpu().numpy(), layer.weight.cpu().numpy(), spec.stride, spec.pad)
    err = co.rel_err(y.contiguous().cpu().numpy(), ref)
    assert err <= tol_for(layer.algorithm, spec.c, layer.e), (plan, err)
