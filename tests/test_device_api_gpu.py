"""The public device entry points of the reference-facing API on the GPU:
``dataflow.execute`` (a reference ``Schedule`` run by the kernels),
``autotune.measure(..., backend="device")``, ``autotune.tune(...,
backend="device")`` over the legal device projection, and the CLI's
``simulate / tune / report --device`` modes (reference ``cli.py:271-390``)."""

import json
import math

import numpy as np
import pytest
import torch

from oracle import conv_oracle as co
from paper_2012_15667_b200 import (ConvShape, WinogradParams, TileConfig, plan_direct_dataflow,
                                   plan_winograd_dataflow, measure, tune)
from paper_2012_15667_b200 import device_tuner as DT
from paper_2012_15667_b200.cli import main as cli_main
from paper_2012_15667_b200.dataflow import execute
from paper_2012_15667_b200.device import b200_hw_model

from tolerances import tol_fp32, tol_wino

pytestmark = pytest.mark.gpu


def _xw(shape, seed=0):
    g = np.random.default_rng(seed)
    x = g.uniform(-1, 1, (shape.n, shape.c_in, shape.h_in, shape.w_in)).astype(np.float32)
    w = (np.random.default_rng(seed + 1).uniform(-1, 1, (shape.c_out, shape.c_in, shape.h_ker, shape.w_ker))
         / np.sqrt(shape.window_size)).astype(np.float32)
    return x, w


def test_execute_direct_schedule_matches_oracle():
    shape = ConvShape.from_output(28, 28, 32, 16, 3, 3)     # valid padding, input 30x30
    hw = b200_hw_model()
    sched = plan_direct_dataflow(shape, hw, TileConfig(28, 4, 32, 16384, 7, 4, 4))
    x, w = _xw(shape)
    y = execute(sched, shape, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), hw=hw)
    err = co.rel_err(y.cpu().numpy(), co.direct_conv(x, w, 1, 0))
    assert err <= tol_fp32(16)


def test_execute_winograd_schedule_matches_oracle():
    shape = ConvShape.from_output(28, 28, 32, 16, 3, 3)
    p = WinogradParams(2, 3)
    hw = b200_hw_model()
    tile = TileConfig(28, 4, 32, 32768, 7, 4, 4, e=2)     # a compiled micro-tile (smoke's)
    sched = plan_winograd_dataflow(shape, p, hw, tile, shared_kernel_transform=True)
    x, w = _xw(shape, 3)
    y = execute(sched, shape, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), hw=hw, winograd=p)
    assert co.rel_err(y.cpu().numpy(), co.direct_conv(x, w, 1, 0)) <= tol_wino(2, 16)


def test_measure_device_backend_times_legal_and_rejects_illegal():
    shape = ConvShape.from_output(56, 56, 64, 64, 3, 3)
    hw = b200_hw_model()
    ok = measure(TileConfig(56, 4, 64, 32768, 7, 4, 8), shape, hw, "direct", backend="device")
    assert math.isfinite(ok.cost) and 0 < ok.cost < 1e-2
    # resident set above s_b (ScheduleError) and an uncompiled micro-tile: inf, never raises
    assert measure(TileConfig(8, 8, 8, 64), shape, hw, "direct", backend="device").cost == math.inf
    assert measure(TileConfig(8, 8, 8, 8192, 1, 1, 8), shape, hw, "direct",
                   backend="device").cost == math.inf


def test_tune_device_backend_over_legal_projection():
    shape = ConvShape.from_output(14, 14, 32, 32, 3, 3)
    hw = b200_hw_model()
    space = DT.device_space(shape, hw, "direct")
    assert 0 < space.size <= space.unconstrained_size
    sess = tune(shape, hw, "direct", budget=24, seed=0, n_s=8, space=space, backend="device")
    best = sess.best
    assert best is not None and math.isfinite(best.cost)
    assert best.config in space
    # the tuned tile computes the convolution
    x, w = _xw(shape, 5)
    y = execute(plan_direct_dataflow(shape, hw, best.config), shape, torch.from_numpy(x).cuda(),
                torch.from_numpy(w).cuda(), hw=hw)
    assert co.rel_err(y.cpu().numpy(), co.direct_conv(x, w, 1, 0)) <= tol_fp32(32)


def test_cli_simulate_tune_report_device_modes(capsys, tmp_path):
    # the B200 machine model (device.b200_hw_model): s words over n_p = 296 blocks
    hw = b200_hw_model()
    base = ["--alg", "direct", "--cin", "32", "--out", "28x28x32", "--ker", "3x3", "--pad", "1",
            "--s", str(hw.s), "--ssm", str(hw.s_sm), "--np", str(hw.n_p)]
    # a compiled K1 micro-tile (4 x 1 x 8 outputs per thread), as in smoke()
    assert cli_main(["simulate", *base, "--tile", "28x4x32", "--threads", "7x4x4", "--sb", "16384",
                     "--device"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["device"]["legal"] and out["device"]["seconds"] > 0 and out["device"]["gflops"] > 0
    ds = tmp_path / "ds.json"
    assert cli_main(["tune", *base, "--budget", "16", "--ns", "8", "--device", "--save-dataset", str(ds)]) == 0
    best = json.loads(capsys.readouterr().out)
    assert best["best_cost"] > 0 and math.isfinite(best["best_cost"])
    assert best["best_config"] is not None and best["measurements"] == 16
    saved = json.loads(ds.read_text())
    assert len(saved) == 16 and all(float(r["cost"]) > 0 for r in saved)
    assert cli_main(["report", *base, "--device"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert "device_projection" in rep


def test_reference_tune_over_tcgen05_domain_reproduces_the_plan_table():
    """The shipped tensor-core kernels through the reference tuner API: tune(shape, hw,
    "direct", ..., backend="device") under the igemm_3xf16 engine, over the I/O-pruned
    tcgen05 domain, lands on the committed res4 plan or within 5 % of its time."""
    from paper_2012_15667_b200 import device_tuner as DT
    from paper_2012_15667_b200.autotune import tune
    from paper_2012_15667_b200.device import shape_of
    from paper_2012_15667_b200.runner import WORKLOADS, load_plans
    spec = next(s for s in WORKLOADS["resnet50"] if s.name == "res4_3x3")
    plan = load_plans("resnet50", allowed=("igemm_3xf16",), n=256)[spec.name]
    DT.set_padding(spec.pad)
    try:
        shape = shape_of(256, spec.c, spec.hw, spec.hw, spec.k, spec.r, spec.stride, spec.pad)
        with DT.use_engine("igemm_3xf16"):
            hw = DT.tcgen05_hw_model()
            space = DT.tcgen05_space(shape, hw, "igemm_3xf16")
            assert plan["tile"] in space, (plan["tile"], space.size)
            assert space.size < space.unconstrained_size
            sess = tune(shape, hw, "direct", space.size, 0, n_s=8, space=space, backend="device")
            t_plan = DT.measure_device(plan["tile"], shape, hw, "direct")
        assert sess.best is not None and math.isfinite(sess.best.cost)
        assert sess.best.config == plan["tile"] or sess.best.cost <= 1.05 * t_plan, (sess.best, t_plan)
    finally:
        DT.set_padding(0)
