"""Benchmark: per-layer conv GFLOP/s on B200 (BASELINE.json metric), JSON line out.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload resnet50|vgg16|single]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the CPU path (oracle port, all host threads)
    python bench.py --gpus 2 --dry-run    # CPU/gloo rehearsal of the rank / shard / max-over-ranks logic

``--gpus N`` without a torchrun environment (no WORLD_SIZE) re-executes itself
under ``torch.distributed.run --nproc-per-node N`` (127.0.0.1), and every arm
checks that the launched world size equals ``--gpus``.

Workload (default): BASELINE config 4 -- the 16 ResNet-50 3x3 convolutions at
global batch 256, batch-sharded over the ranks (strong scaling: 256/N images
per GPU), each layer with the algorithm + tile the lower-bound auto-tuner
picked on the device (``paper_2012_15667_b200/tuned/b200_resnet50.json``).
A step = filter prep + conv of all 16 layers over the local batch.  ``value``
is the whole-job direct-equivalent conv GFLOP/s (sum over ranks of
2*N*K*C*R*S*P*Q / the max-over-ranks step time).  Inputs are synthetic
(``x ~ U(-1,1)``, ``w ~ U(-1,1)/sqrt(CRS)``), fp32, resident in HBM; the
per-step working set is far larger than the 126 MB L2, so no flush is needed
(``--workload single`` flushes L2 between steps instead).

``e2e`` repeats the step through the public API with pinned-host inputs:
H2D copy of every layer's input, conv, D2H copy of every output, all inside
the timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv GFLOP/s per layer & DRAM bytes vs I/O lower bound, 1/2/4/8 B200 vs CPU ref"
L2_BYTES = 126 * 1024 * 1024
DEFAULT_BATCH = {"resnet50": 256, "vgg16": 32, "single": 1}
WORKLOAD_NAME = {
    "resnet50": "ResNet-50 3x3 conv layers (16), batch-sharded (BASELINE config 4)",
    "vgg16": "VGG-16 3x3 conv layers (13) (BASELINE config 3)",
    "single": "single 3x3 conv N=1 C=64 56x56 K=64 s1 p1 (BASELINE config 1)",
}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (C, OpenMP) on a bounded sample
# ---------------------------------------------------------------------------
def cpu_oracle_gflops(layers, images: int = 1, threads: int = 0):
    """Time the C oracle (fp32 in, fp64 accumulate) over ``layers`` x ``images``.

    Input generation is excluded; returns (GFLOP/s, seconds of conv work).
    """
    import numpy as np
    from oracle import conv_oracle
    rng = np.random.default_rng(0)
    flops, busy = 0, 0.0
    for spec in layers:
        x = rng.uniform(-1, 1, (images, spec.c, spec.hw, spec.hw)).astype(np.float32)
        w = (rng.uniform(-1, 1, (spec.k, spec.c, spec.r, spec.r))
             / np.sqrt(spec.c * spec.r * spec.r)).astype(np.float32)
        t1 = time.perf_counter()
        conv_oracle.c_direct_conv(x, w, spec.stride, spec.pad, threads=threads)
        busy += time.perf_counter() - t1
        flops += spec.flops(images)
    return flops / busy / 1e9, busy


def onednn_gflops(specs, threads: int, images: int = 1, reps: int = 3):
    """Numeric CPU conv baseline: torch.nn.functional.conv2d fp32 on the
    host (oneDNN), all `threads`, `images` per layer; median of `reps` after a warm-up.
    Returns (GFLOP/s, seconds of conv work per pass)."""
    import torch
    torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(0)
    total = 0.0
    flops = 0
    for spec in specs:
        x = torch.rand((images, spec.c, spec.hw, spec.hw), generator=g) * 2 - 1
        w = (torch.rand((spec.k, spec.c, spec.r, spec.r), generator=g) * 2 - 1) / (spec.c * spec.r * spec.r) ** 0.5
        torch.nn.functional.conv2d(x, w, stride=spec.stride, padding=spec.pad)
        ts = []
        for _ in range(reps):
            t1 = time.perf_counter()
            torch.nn.functional.conv2d(x, w, stride=spec.stride, padding=spec.pad)
            ts.append(time.perf_counter() - t1)
        total += statistics.median(ts)
        flops += spec.flops(images)
    return flops / total / 1e9, total


def model_cpu_timings() -> dict:
    """The reference's own CPU path (its model: SURVEY §8(a) a6-a21),
    timed through this package's bit-exact restatement (the reference itself is not on
    the GPU box): lower bound, analytic tile, schedule + simulate, Table-1 space and a
    budget-32 GBR tune, on BASELINE config 1 and on ResNet-50 res4 at batch 256.
    Single process, single thread, as the reference runs."""
    from paper_2012_15667_b200.autotune import build_space, tune
    from paper_2012_15667_b200.bounds import lower_bound_dc
    from paper_2012_15667_b200.dataflow import optimal_tile_dc, plan_direct_dataflow, simulate
    from paper_2012_15667_b200.device import b200_hw_model, shape_of
    hw = b200_hw_model()
    out = {}
    for name, shape in (("config1", shape_of(1, 64, 56, 56, 64, 3, 1, 1)),
                        ("res4_3x3_n256", shape_of(256, 256, 14, 14, 256, 3, 1, 1))):
        def med(fn, reps):
            ts = []
            for _ in range(reps):
                t1 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t1)
            return statistics.median(ts)
        tile = optimal_tile_dc(shape, hw)
        row = {
            "lower_bound_dc_us": round(1e6 * med(lambda: lower_bound_dc(shape, hw.s_sm), 200), 2),
            "optimal_tile_dc_us": round(1e6 * med(lambda: optimal_tile_dc(shape, hw), 20), 1),
            "plan_and_simulate_ms": round(1e3 * med(lambda: simulate(plan_direct_dataflow(shape, hw, tile), hw), 5), 3),
        }
        t1 = time.perf_counter()
        space = build_space(shape, hw, "direct", thread_axes=False)
        row["build_space_s"] = round(time.perf_counter() - t1, 3)
        row["space_size"] = space.size
        t1 = time.perf_counter()
        tune(shape, hw, "direct", 32, 0, space=space)
        row["tune_budget32_s"] = round(time.perf_counter() - t1, 3)
        out[name] = row
    return out


def layer_io_bounds(spec, n: int, algorithm: str, e, hw) -> dict:
    """The paper's I/O bounds for one layer call in bytes (fp32 words x 4): the
    red-blue-pebble lower bound Omega(S) and q_exact(S) per image x n
    (reference pkg/src/convio/bounds.py:230-271) at S = one SM's fast memory of the
    B200 machine model (registers + shared memory, device.py), and the Eq. 18/19
    I/O of the model's optimal tile (dataflow.py:377-378, 403-407).  These bound the
    traffic between the SMs and the next level -- L2 -- not DRAM."""
    from paper_2012_15667_b200.bounds import lower_bound_dc, lower_bound_wa
    from paper_2012_15667_b200.dataflow import dc_io_at_optimum, wa_io_at_optimum
    from paper_2012_15667_b200.device import shape_of
    from paper_2012_15667_b200.model import WinogradParams
    shape = shape_of(n, spec.c, spec.hw, spec.hw, spec.k, spec.r, spec.stride, spec.pad)
    s = hw.s_sm
    wino = algorithm.startswith("winograd") and bool(e)
    if wino:
        p = WinogradParams(e, spec.r)
        rep_, opt = lower_bound_wa(shape, p, s), wa_io_at_optimum(shape, p, hw)
    else:
        rep_, opt = lower_bound_dc(shape, s), dc_io_at_optimum(shape, hw)
    return {"dataflow": "WA" if wino else "DC", "s_words": s,
            "omega_bytes": int(4 * n * rep_.omega), "q_exact_bytes": int(4 * n * rep_.q_exact),
            "io_at_optimum_bytes": int(4 * opt)}


def cudnn_layers(torch, specs, n: int, dev, reps: int = 10) -> dict:
    """The GPU comparison point (north star): cuDNN through
    torch.nn.functional.conv2d, cudnn.benchmark on, FP32 (TF32 off) and TF32, the
    faster of NCHW / channels_last per layer; CUDA events over `reps` back-to-back
    calls after warm-up.  {layer name: {"fp32": ms, "tf32": ms}}."""
    F = torch.nn.functional
    saved = (torch.backends.cudnn.benchmark, torch.backends.cudnn.allow_tf32)
    torch.backends.cudnn.benchmark = True
    out = {}
    try:
        for spec in {s.name: s for s in specs}.values():
            g = torch.Generator(device=dev).manual_seed(0)
            x = torch.rand((n, spec.c, spec.hw, spec.hw), device=dev, generator=g) * 2 - 1
            w = (torch.rand((spec.k, spec.c, spec.r, spec.r), device=dev, generator=g) * 2 - 1) / (
                spec.c * spec.r * spec.r) ** 0.5
            row = {}
            for prec in ("fp32", "tf32"):
                torch.backends.cudnn.allow_tf32 = prec == "tf32"
                best = float("inf")
                for fmt in (torch.contiguous_format, torch.channels_last):
                    xx, ww = x.contiguous(memory_format=fmt), w.contiguous(memory_format=fmt)
                    for _ in range(3):
                        F.conv2d(xx, ww, stride=spec.stride, padding=spec.pad)
                    torch.cuda.synchronize(dev)
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(reps):
                        F.conv2d(xx, ww, stride=spec.stride, padding=spec.pad)
                    b.record()
                    b.synchronize()
                    best = min(best, a.elapsed_time(b) / reps)
                    del xx, ww
                row[prec] = round(best, 4)
            out[spec.name] = row
            del x, w
    finally:
        torch.backends.cudnn.benchmark, torch.backends.cudnn.allow_tf32 = saved
        torch.cuda.empty_cache()
    return out


def network_bench(torch, dev, steps: int, warmup: int, n: int = 32) -> dict:
    """The chained network forward: VGG-16's 13 convs +
    5 max pools + the NCHW -> NHWC staging, batch ``n`` (BASELINE config 3), all our
    kernels, replayed as one CUDA graph; beside it the same network through
    torch/cuDNN (fp32 and TF32, channels_last, cudnn.benchmark), and end to end
    from a pinned NCHW host batch to host features."""
    from paper_2012_15667_b200.network import Vgg16Features
    F = torch.nn.functional
    net = Vgg16Features(n, dev, seed=11)
    x = torch.rand((n, 3, 224, 224), device=dev) * 2 - 1
    net.prepare()
    stream = torch.cuda.current_stream(dev)

    def graph_of(fn):
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                fn(side)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            fn(side)
        torch.cuda.synchronize(dev)
        return g

    def timed(g):
        g.replay()
        torch.cuda.synchronize(dev)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            g.replay()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / steps

    ours = timed(graph_of(lambda st: net.forward(x, stream=st)))
    flops = net.flops()
    out = {"model": f"VGG-16 conv features (13 conv + bias + ReLU, 5 max pools), batch {n}, 224x224, "
                    "NCHW input staged to NHWC on the device",
           "ms_per_forward": round(ours, 4), "images_per_s": round(n / (ours / 1e3), 1),
           "gflops_direct_equiv": round(flops / (ours / 1e3) / 1e9, 1),
           "launches_per_forward": net.launches_per_forward(),
           "plans": {l.name: l.algorithm for l in net.conv_layers}}
    # cuDNN through torch, same weights, channels_last
    saved = (torch.backends.cudnn.benchmark, torch.backends.cudnn.allow_tf32)
    torch.backends.cudnn.benchmark = True
    ws = [(l.weight.contiguous(memory_format=torch.channels_last), l.bias) for l in net.conv_layers]
    xl = x.contiguous(memory_format=torch.channels_last)

    def torch_forward(st):
        with torch.cuda.stream(st):
            h, j = xl, 0
            for layer in net.layers:
                if layer is None:
                    h = F.max_pool2d(h, 2)
                else:
                    h = torch.relu(F.conv2d(h, ws[j][0], ws[j][1], padding=1))
                    j += 1
            return h
    try:
        for prec in ("fp32", "tf32"):
            torch.backends.cudnn.allow_tf32 = prec == "tf32"
            t = timed(graph_of(torch_forward))
            out[f"cudnn_{prec}_ms_per_forward"] = round(t, 4)
            out[f"ours_speedup_vs_cudnn_{prec}"] = round(t / ours, 3)
    finally:
        torch.backends.cudnn.benchmark, torch.backends.cudnn.allow_tf32 = saved
    # end to end: pinned NCHW host batch -> device -> features -> pinned host
    hx = torch.empty((n, 3, 224, 224), pin_memory=True).copy_(x)
    hy = torch.empty((n, 512, 7, 7), pin_memory=True)
    dx = torch.empty_like(x)

    def e2e(st):
        with torch.cuda.stream(st):
            dx.copy_(hx, non_blocking=True)
            y = net.forward(dx, stream=st, nchw_out=True)
            hy.copy_(y, non_blocking=True)
    for _ in range(2):
        e2e(stream)
    torch.cuda.synchronize(dev)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        e2e(stream)
    b.record(stream)
    b.synchronize()
    te = a.elapsed_time(b) / steps
    out["e2e"] = {"ms_per_forward": round(te, 4), "images_per_s": round(n / (te / 1e3), 1),
                  "h2d_bytes": hx.numel() * 4, "d2h_bytes": hy.numel() * 4}
    del net
    torch.cuda.empty_cache()
    return out


def run_reference(args, rank: int, world: int) -> None:
    """``--impl reference``: the CPU implementation of the path on host cores."""
    if rank != 0:
        return
    from paper_2012_15667_b200.runner import WORKLOADS, expand
    layers = expand(WORKLOADS[args.workload])
    cores = os.cpu_count() or 1
    images = 1
    # warm-up: W passes over a small sample
    for _ in range(args.warmup):
        cpu_oracle_gflops(layers[:1], images, cores)
    times, flops = [], sum(s.flops(images) for s in layers)
    for _ in range(args.steps):
        _, el = cpu_oracle_gflops(layers, images, cores)
        times.append(el)
    total = sum(times)
    value = flops * args.steps / total / 1e9
    sample = f"{images} image per layer instance x {len(layers)} layers per step (C oracle, fp64 accumulate)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAME[args.workload], "global_batch": DEFAULT_BATCH[args.workload],
                   "sample_batch": images},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# the GPU arm
# ---------------------------------------------------------------------------
def ffma_peak_tflops(torch, stream) -> float:
    import ctypes
    from paper_2012_15667_b200 import _native as N
    sink = torch.zeros(148 * 64, device="cuda")
    flops = ctypes.c_int64()
    blocks, iters = 148 * 8, 1500
    sp = ctypes.c_void_p(stream.cuda_stream)
    best = 0.0
    for _ in range(4):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        N.check(N.lib().convio_ffma_peak(ctypes.c_void_p(sink.data_ptr()), blocks, iters,
                                         ctypes.byref(flops), sp))
        b.record(stream)
        b.synchronize()
        best = max(best, flops.value / (a.elapsed_time(b) / 1e3) / 1e12)
    return best


PROFILE_ROUND = "r2"   # the committed evidence of the current round: profiles/r2/


def load_profile_traffic() -> dict:
    """DRAM / L2 bytes per layer call from the committed ncu summaries
    (profiles/<round>/*_traffic.json, written by scripts/run_layer.py --parse)."""
    out = {}
    pdir = os.path.join(ROOT, "profiles", PROFILE_ROUND)
    if not os.path.isdir(pdir):
        return out
    for fn in sorted(os.listdir(pdir)):
        if fn.endswith("_traffic.json"):
            try:
                with open(os.path.join(pdir, fn)) as fh:
                    out.update(json.load(fh))
            except (OSError, ValueError):
                pass
    return out


def _l2_measured(tab: dict, workload: str, layer: str, algorithm: str, n: int):
    """ncu L2->SM read bytes per layer call (lts__t_sectors_srcunit_tex_op_read x 32 B,
    summed over the call's kernels) from the committed capture, or None."""
    t = tab.get(f"{workload}:{layer}:{algorithm}")
    if not isinstance(t, dict) or t.get("n") not in (None, n) or t.get("l2_sm_read_bytes_per_call") is None:
        return None
    return t


def _traffic(tab: dict, workload: str, fam: dict, dom: str, n: int | None = None):
    """DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, one capture
    per layer call, committed under profiles/<round>/*_traffic.json) of the dominant family's
    layers: {layer: bytes}; None if no capture is committed."""
    alg = dom.split()[0]
    out = {}
    for layer in sorted(fam["layers"]):
        t = tab.get(f"{workload}:{layer}:{alg}")
        if isinstance(t, dict):
            if n is not None and t.get("n") not in (None, n):
                continue   # captured at another batch
            out[layer] = t.get("dram_bytes_per_call")
        elif t is not None:
            out[layer] = t
    return out or None


def _traffic_mean(by_layer: dict | None, fam: dict):
    """One figure for `roofline.traffic`: DRAM bytes per launch averaged over the
    dominant family's launches (each layer weighted by its launch count)."""
    if not by_layer:
        return None
    cnt = fam.get("layer_launches", {})
    num = sum(v * cnt.get(k, 1) for k, v in by_layer.items() if v is not None)
    den = sum(cnt.get(k, 1) for k, v in by_layer.items() if v is not None)
    return int(num / den) if den else None


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def reexec_under_torchrun(n: int) -> None:
    """``--gpus N`` outside torchrun: one rank per GPU via torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def run_dry(args, rank: int, world: int) -> None:
    """``--dry-run``: the multi-rank host logic of the GPU arm on CPU (gloo).

    Same shard ranges, replicated-by-seed filters, barrier + max-over-ranks
    timing and whole-job value as the GPU arm; the per-rank "step" is the C
    oracle over the rank's images (test infrastructure standing in for the
    kernels, which need a B200).  Prints one JSON line on rank 0.
    """
    import numpy as np
    import torch
    import torch.distributed as dist
    from oracle import conv_oracle
    from paper_2012_15667_b200.runner import WORKLOADS, expand, shard_range
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    distributed = dist.is_available() and dist.is_initialized()
    n_total = args.batch or world
    lo, hi = shard_range(n_total, rank, world)
    specs = expand(WORKLOADS[args.workload])[:2]
    rng = np.random.default_rng(1000)
    ws = [(rng.uniform(-1, 1, (s.k, s.c, s.r, s.r)) / np.sqrt(s.c * s.r * s.r)).astype(np.float32)
          for s in specs]
    xs = [np.random.default_rng(7919 * (i + 1)).uniform(-1, 1, (n_total, s.c, s.hw, s.hw))
          .astype(np.float32)[lo:hi] for i, s in enumerate(specs)]
    threads = max(1, (os.cpu_count() or 1) // world)

    def step():
        for s, x, w in zip(specs, xs, ws):
            if len(x):
                conv_oracle.c_direct_conv(x, w, s.stride, s.pad, threads=threads)

    def reduce(v: float, op) -> float:
        if not distributed:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    if distributed:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    if distributed:
        dist.barrier()
    t_max = reduce(el, dist.ReduceOp.MAX if distributed else None)
    flops_all = reduce(float(sum(s.flops(hi - lo) for s in specs)), dist.ReduceOp.SUM if distributed else None)
    images = reduce(float(hi - lo), dist.ReduceOp.SUM if distributed else None)
    if rank == 0:
        print(json.dumps({
            "impl": "dry-run", "metric": METRIC, "value": round(flops_all * args.steps / t_max / 1e9, 3),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * t_max / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME[args.workload] + " (first 2 layers, CPU oracle)",
                       "global_batch": n_total, "images_over_ranks": int(images),
                       "parallelism": f"batch-sharded x{world} (gloo, no data-path collective)"},
        }), flush=True)
    if distributed:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=["resnet50", "vgg16", "single"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--gather", action="store_true", help="all-gather outputs to every rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cudnn", action="store_true", help="skip the cuDNN comparison point")
    ap.add_argument("--no-network", action="store_true", help="skip the chained VGG-16 forward")
    ap.add_argument("--no-group", action="store_true",
                    help="one launch per layer in the timed step (no grouped same-plan launches)")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU (gloo) rehearsal of the multi-rank logic; no GPU needed")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        reexec_under_torchrun(args.gpus)   # does not return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s) "
                         "(WORLD_SIZE); run `python bench.py --gpus N` or torchrun --nproc-per-node N")
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2012_15667_b200 import conv as C
    from paper_2012_15667_b200.runner import (
        WORKLOADS, ConvLayer, expand, group_layers, group_table, load_group_overrides, load_group_plans,
        load_plans,
        make_input, make_weights,
        prepare_layers,
        shard_range,
        tuned_table,
        gather_outputs, CUDA_CORE_ALGORITHMS)
    from paper_2012_15667_b200.device import winograd_gemm_flops

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # under torchrun (MASTER_ADDR set) the process group is created even for one
    # rank, so the max-over-ranks / barrier path is the same code at N=1 and N=8
    if world > 1 or "MASTER_ADDR" in os.environ:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL prints its version banner on stdout when the communicator is created;
        # the contract is one JSON line there, so communicator setup writes to stderr
        if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
            os.environ["NCCL_DEBUG"] = "WARN"
        sys.stdout.flush()
        saved_fd = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved_fd, 1)
            os.close(saved_fd)
    distributed = dist.is_available() and dist.is_initialized()

    def barrier():
        if distributed:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if not distributed:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if not distributed:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    stream = torch.cuda.current_stream(dev)
    n_total = args.batch or DEFAULT_BATCH[args.workload]
    lo, hi = shard_range(n_total, rank, world)
    n_local = hi - lo
    specs = expand(WORKLOADS[args.workload])
    weights = [make_weights(s, dev, 1000 + i) for i, s in enumerate(specs)]
    flops_local = sum(s.flops(n_local) for s in specs)
    flops_all = sum_over_ranks(float(flops_local))

    class Arm:
        """One plan set: per-layer ConvLayers, inputs in each plan's layout, outputs."""

        def __init__(self, plans):
            self.plans = plans
            self.layers = [ConvLayer(s, weights[i], plans.get(s.name)) for i, s in enumerate(specs)]
            self.xs = [make_input(s, n_local, dev, seed=7919 * (i + 1) + lo, layout=lay.layout)
                       for i, (s, lay) in enumerate(zip(specs, self.layers))]
            self.ys = [C.empty_act(n_local, s.k, s.out_hw, s.out_hw, lay.layout, device=dev)
                       for s, lay in zip(specs, self.layers)]
            # same-shape, same-plan 3xF16 layers (res2 x3, res3 x3, res4 x5) run as grouped
            # launches in the timed step; their inputs / outputs are slices of the stacked buffers
            self.units = group_layers(self.layers, n_local, dev, load_group_plans(args.workload, n_local)) \
                if not args.no_group else \
                [("single", l, [i]) for i, l in enumerate(self.layers)]
            for kind, unit, idx in self.units:
                if kind == "group":
                    for g_i, li in enumerate(idx):
                        unit.x_of(g_i).copy_(self.xs[li])
                        self.xs[li], self.ys[li] = unit.x_of(g_i), unit.y_of(g_i)
            self.work_bytes = sum(x.numel() * 4 for x in self.xs) + sum(y.numel() * 4 for y in self.ys)

        def step(self, events=None, st=None, per_layer=False):
            st = st or stream
            # the step's filter prep (all 3xF16 splits in one launch), then the convs:
            # grouped launches for same-plan layers; the per-layer breakdown (events)
            # runs every layer on its own so each gets its own timing
            launches = prepare_layers(self.layers, dev, st)
            if events is None and not per_layer:
                for kind, unit, idx in self.units:
                    if kind == "group":
                        unit.run(st)
                    else:
                        unit.run(self.xs[idx[0]], out=self.ys[idx[0]], stream=st)
                    launches += unit.launches
                return launches
            for i, layer in enumerate(self.layers):
                if events is not None:
                    events[i][0].record(st)
                layer.run(self.xs[i], out=self.ys[i], stream=st)
                if events is not None:
                    events[i][1].record(st)
                launches += layer.launches
            return launches

        def capture(self):
            """One step (filter prep + all convs) captured as a CUDA graph: the
            launches are replayed by the driver, no per-call host work."""
            side = torch.cuda.Stream(dev)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                self.step(st=side)
            torch.cuda.synchronize(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self.graph_launches = self.step(st=side)
            torch.cuda.synchronize(dev)
            return g

        def timed_graph(self, steps, graph, flush_buf=None):
            """K device-timed graph replays (barrier + sync both sides)."""
            barrier()
            torch.cuda.synchronize(dev)
            total = 0.0
            if flush_buf is not None:
                for k in range(steps):
                    flush_buf.fill_(float(k))
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    graph.replay()
                    b.record(stream)
                    b.synchronize()
                    total += a.elapsed_time(b)
            else:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(steps):
                    graph.replay()
                b.record(stream)
                torch.cuda.synchronize(dev)
                total = a.elapsed_time(b)
            barrier()
            torch.cuda.synchronize(dev)
            return total

        def timed(self, steps, flush_buf=None):
            """K device-timed steps (barrier + sync both sides); per-layer events."""
            ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in self.layers]
                  for _ in range(steps)]
            launches = 0
            barrier()
            torch.cuda.synchronize(dev)
            if flush_buf is not None:
                total = 0.0
                for k in range(steps):
                    flush_buf.fill_(float(k))
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    launches += self.step(ev[k])
                    b.record(stream)
                    b.synchronize()
                    total += a.elapsed_time(b)
            else:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for k in range(steps):
                    launches += self.step(ev[k])
                b.record(stream)
                torch.cuda.synchronize(dev)
                total = a.elapsed_time(b)
            barrier()
            torch.cuda.synchronize(dev)
            return total, ev, launches

        def breakdown(self, ev, steps):
            rows, fam = [], {}
            for i, (s, layer) in enumerate(zip(specs, self.layers)):
                ts = [ev[k][i][0].elapsed_time(ev[k][i][1]) for k in range(steps)]
                t_med = statistics.median(ts)
                f_dir = s.flops(n_local)
                if layer.algorithm == "winograd":
                    f_alg = winograd_gemm_flops(n_local, s.c, s.k, s.out_hw, s.out_hw, layer.e)
                    name = f"winograd F({layer.e},3)"
                elif layer.algorithm.startswith("winograd_tc") or layer.algorithm == "winograd_nhwc":
                    f_alg = winograd_gemm_flops(n_local, s.c, s.k, s.out_hw, s.out_hw, layer.e)
                    name = f"{layer.algorithm} F({layer.e},3)"
                else:
                    f_alg = f_dir
                    name = layer.algorithm
                agg = fam.setdefault(name, {"ms": 0.0, "flops": 0.0, "launches": 0, "layers": set(),
                                            "layer_launches": {}})
                agg["layer_launches"][s.name] = agg["layer_launches"].get(s.name, 0) + steps
                agg["ms"] += sum(ts)
                agg["flops"] += f_alg * steps
                agg["launches"] += steps
                agg["layers"].add(s.name)
                comp = 4 * (n_local * s.c * s.hw * s.hw + s.k * s.c * s.r * s.r
                            + n_local * s.k * s.out_hw * s.out_hw)
                t = layer.tile
                rows.append({
                    "layer": s.name, "algorithm": name, "_alg": layer.algorithm, "_e": layer.e,
                    "tile": None if t is None else [t.x, t.y, t.z, t.s_b, t.n_xt, t.n_yt, t.n_zt, t.layout],
                    "ms": round(t_med, 4), "gflops": round(f_dir / (t_med / 1e3) / 1e9, 1),
                    "q_dram_bytes": comp,
                })
            return rows, fam

        def unit_families(self, reps, flush_buf=None):
            """Kernel families of the TIMED step: each unit (a grouped launch or a single
            layer, filter prep excluded) captured as its own CUDA graph and replayed
            ``reps`` times with CUDA events around each replay on the launching stream (L2
            flushed between replays when the step is flushed): device time without the
            host gaps an eager per-layer pass has at small batches."""
            fam = {}
            for kind, unit, idx in self.units:
                if kind == "group":
                    def fn(st, unit=unit):
                        unit.run(st)
                else:
                    def fn(st, unit=unit, i=idx[0]):
                        unit.run(self.xs[i], out=self.ys[i], stream=st)
                side = torch.cuda.Stream(dev)
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    fn(side)
                    fn(side)
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    fn(side)
                torch.cuda.synchronize(dev)
                ts = []
                for _ in range(reps):
                    if flush_buf is not None:
                        flush_buf.fill_(1.0)
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    g.replay()
                    b.record(stream)
                    b.synchronize()
                    ts.append(a.elapsed_time(b))
                del g
                layer = self.layers[idx[0]]
                s = specs[idx[0]]
                if layer.algorithm.startswith("winograd"):
                    f_alg = winograd_gemm_flops(n_local, s.c, s.k, s.out_hw, s.out_hw, layer.e)
                    name = (f"winograd F({layer.e},3)" if layer.algorithm == "winograd"
                            else f"{layer.algorithm} F({layer.e},3)")
                else:
                    f_alg = s.flops(n_local)
                    name = layer.algorithm
                agg = fam.setdefault(name, {"ms": 0.0, "flops": 0.0, "launches": 0, "layers": set(),
                                            "layer_launches": {}, "units": []})
                agg["ms"] += sum(ts)
                agg["flops"] += f_alg * len(idx) * reps
                agg["launches"] += reps
                agg["layers"].add(s.name)
                agg["layer_launches"][s.name] = agg["layer_launches"].get(s.name, 0) + len(idx) * reps
                agg["units"].append({"unit": s.name + (f" x{len(idx)}" if kind == "group" else ""),
                                     "ms": round(statistics.median(ts), 4)})
            return fam

    plans = load_plans(args.workload, n=n_local)
    if not args.no_group:   # repeated layers whose grouped 3xF16 launch beat their own plan
        plans.update(load_group_overrides(args.workload, n_local))
    arm = Arm(plans)
    flush = arm.work_bytes < 4 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, device=dev) if flush else None
    for _ in range(args.warmup):
        arm.step()
        # the eager per-layer pass below launches every layer on its own: warm its
        # per-layer state too (each launch's speculative activation scale)
        arm.step(per_layer=True)
    torch.cuda.synchronize(dev)

    # ---- device-timed region: exactly K steps --------------------------------
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    # eager pass: per-layer CUDA events (the roofline / per_layer breakdown)
    eager_ms, ev, launches = arm.timed(args.steps, scratch)
    total_ms = eager_ms
    graph_used = False
    if not args.no_graph:
        # the timed value: the same step replayed as a CUDA graph (no host work per call)
        g = arm.capture()
        g.replay()
        torch.cuda.synchronize(dev)
        total_ms = arm.timed_graph(args.steps, g, scratch)
        launches = arm.graph_launches * args.steps   # the replayed step (grouped launches)
        graph_used = True
    clk = clocks.stop()
    t_max_ms = max_over_ranks(total_ms)
    value = flops_all * args.steps / (t_max_ms / 1e3) / 1e9
    per_layer, _ = arm.breakdown(ev, args.steps)
    # the roofline's kernel families from the timed step's own launches (grouped units)
    fam = arm.unit_families(max(args.steps, 5), scratch)

    # ---- roofline of the dominant kernel (largest share of the step) ------------
    dom = max(fam, key=lambda k: fam[k]["ms"])
    d = fam[dom]
    achieved = d["flops"] / (d["ms"] / 1e3) / 1e12 if d["ms"] else 0.0
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except (OSError, ValueError):
        pass
    traffic_tab = load_profile_traffic()
    if dom.startswith("igemm") or dom.startswith("winograd_tc"):
        # tensor pipe: dense TF32 = 1/2 of the measured bf16 rate; 3xTF32 issues 3 MMAs per
        # algorithmic flop; BF16 runs at the bf16 rate
        prec = dom.split()[0].rsplit("_", 1)[-1]
        # 3xTF32 / 3xF16 issue 3 MMAs per algorithmic flop; f16 and bf16 run at the
        # bf16 rate, TF32 at half of it
        mma_per_flop = 3 if prec in ("3xtf32", "3xf16") else 1
        bf16 = peaks.get("bf16_tflops") or 1590.0
        peak = bf16 if prec in ("bf16", "3xf16") else bf16 / 2
        kind = {"bf16": "kind::f16 (bf16)", "3xf16": "kind::f16 (scaled fp16 hi/lo)"}.get(prec, "kind::tf32")
        what = ("implicit GEMM" if dom.startswith("igemm") else
                "Winograd pipeline: input transform + batched GEMM + output transform, "
                "flops = element-wise GEMM flops")
        roofline = {
            "bound": "tensor", "kernel": f"{dom} (tcgen05.mma {kind}; {what})",
            "achieved": round(achieved * mma_per_flop, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
            "frac": round(achieved * mma_per_flop / peak, 4),
            "achieved_algorithmic": round(achieved, 3), "mma_flops_per_algorithmic_flop": mma_per_flop,
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops" + ("" if prec in ("bf16", "3xf16") else " / 2 (dense TF32 rate)")
                            if peaks.get("bf16_tflops") else "fallback 1.59 PFLOP/s bf16"),
            "traffic": _traffic_mean(_traffic(traffic_tab, args.workload, d, dom, n_local), d),
            "traffic_by_layer": _traffic(traffic_tab, args.workload, d, dom, n_local),
        }
    else:
        peak = ffma_peak_tflops(torch, stream)
        roofline = {
            "bound": "fp32", "kernel": f"{dom} conv (FFMA)",
            "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4) if peak else None,
            "peak_source": "live FFMA probe (convio_ffma_peak); MEASURED_PEAKS.json has no FP32 entry",
            "traffic": _traffic_mean(_traffic(traffic_tab, args.workload, d, dom, n_local), d),
            "traffic_by_layer": _traffic(traffic_tab, args.workload, d, dom, n_local),
        }
    roofline["layers"] = sorted(d["layers"])
    roofline["share_of_step"] = round(d["ms"] / sum(f["ms"] for f in fam.values()), 3)
    roofline["units"] = d["units"]
    roofline["timing"] = ("per unit of the timed step (grouped launch or single layer, with its checking "
                          "launch) as its own CUDA graph, CUDA events around each replay"
                          + (", L2 flushed between replays" if flush else "")
                          + "; traffic = ncu DRAM bytes per single-layer call")
    # the same family against HBM: the committed ncu DRAM bytes of its layer calls
    # over their device time (the unfused Winograd pipeline moves V and M through
    # HBM, so bandwidth, not the tensor pipe, is its ceiling)
    by_layer = roofline.get("traffic_by_layer") or {}
    cnt = d.get("layer_launches", {})
    if by_layer and d["ms"] and all(by_layer.get(k) for k in d["layers"]):
        moved = sum(by_layer[k] * cnt.get(k, 1) for k in d["layers"])   # over all timed steps
        gbs = moved / (d["ms"] / 1e3) / 1e9
        hbm = peaks.get("hbm_gbs")
        roofline["hbm_view"] = {"achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                                "frac": round(gbs / hbm, 4) if hbm else None,
                                "bytes_per_step": int(moved / max(1, args.steps)),
                                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy read+write)"}

    # ---- variants: paper-faithful FP32 CUDA cores only, and reduced-precision TF32 ----
    variants = {}
    if not args.no_variants:
        for vname, allowed in (("fp32_cuda_cores", CUDA_CORE_ALGORITHMS),
                               # the direct (DC) dataflows only: every layer within the
                               # 1.5 x Q_DRAM gate (Winograd's V / M planes exceed it)
                               ("fp32_direct_only", ("direct", "igemm_3xtf32", "igemm_3xf16")),
                               ("tf32_tcgen05", ("igemm_tf32", "winograd_tc_tf32")),
                               ("bf16_tcgen05", ("igemm_bf16", "winograd_tc_bf16"))):
            vplans = load_plans(args.workload, allowed, n=n_local)
            if not vplans:
                continue
            varm = Arm(vplans)
            for _ in range(2):
                varm.step()
                varm.step(per_layer=True)
            vt, vev, _ = varm.timed(args.steps, scratch)
            if not args.no_graph:   # same timing basis as the headline: graph replay
                vg = varm.capture()
                vg.replay()
                torch.cuda.synchronize(dev)
                vt = varm.timed_graph(args.steps, vg, scratch)
                del vg
            vt = max_over_ranks(vt)
            rows, _ = varm.breakdown(vev, args.steps)
            variants[vname] = {
                "value": round(flops_all * args.steps / (vt / 1e3) / 1e9, 3), "unit": "GFLOP/s",
                "ms_per_step": round(vt / args.steps, 4),
                "tolerance": {"tf32_tcgen05": "5e-3 direct, 5e-3..2e-2 Winograd (TF32 operands)",
                              "bf16_tcgen05": "3e-2 direct, 5e-2..1.5e-1 Winograd (BF16 operands)"}.get(
                                  vname, "1e-5" if vname == "fp32_direct_only"
                                  else "1e-5 direct / 1e-4..1e-3 Winograd"),
                "per_layer": [{k: r[k] for k in ("layer", "algorithm", "ms", "gflops")} for r in rows],
            }
            del varm
    layers, xs, ys = arm.layers, arm.xs, arm.ys
    work_bytes = arm.work_bytes

    # ---- end-to-end through the public API with host buffers -------------------
    e2e = None
    if not args.no_e2e:
        hx = [torch.empty_strided(x.shape, x.stride(), dtype=torch.float32, pin_memory=True).copy_(x)
              for x in xs]
        hy = [torch.empty_strided(y.shape, y.stride(), dtype=torch.float32, pin_memory=True)
              for y in ys]
        dx = [torch.empty_like(x) for x in xs]
        h2d = sum(h.numel() * 4 for h in hx)
        d2h = sum(h.numel() * 4 for h in hy)

        # copies overlap compute: H2D of every layer's input on one stream, the convs on
        # the compute stream (each waits for its input), D2H of each output on a third
        # stream as soon as it is produced -- PCIe runs both directions at once.
        # WAR hazards across steps (dx / ys reuse) are ordered by events.
        s_h2d = torch.cuda.Stream(dev)
        s_d2h = torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in layers]
        ev_done = [torch.cuda.Event() for _ in layers]
        ev_out = [torch.cuda.Event() for _ in layers]
        ev_drained = [torch.cuda.Event() for _ in layers]
        first = [True]

        def e2e_step():
            for i in range(len(layers)):
                if not first[0]:
                    s_h2d.wait_event(ev_done[i])        # previous conv i has read dx[i]
                with torch.cuda.stream(s_h2d):
                    dx[i].copy_(hx[i], non_blocking=True)
                ev_in[i].record(s_h2d)
            for i, layer in enumerate(layers):
                stream.wait_event(ev_in[i])
                if not first[0]:
                    stream.wait_event(ev_drained[i])    # previous D2H of ys[i] finished
                y = layer.forward(dx[i], out=ys[i], stream=stream)
                ev_done[i].record(stream)
                s_d2h.wait_event(ev_done[i])
                with torch.cuda.stream(s_d2h):
                    hy[i].copy_(y, non_blocking=True)
                ev_drained[i].record(s_d2h)
            first[0] = False
        e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s_h2d.wait_stream(stream)
        for _ in range(args.steps):
            e2e_step()
        stream.wait_stream(s_d2h)
        stream.wait_stream(s_h2d)
        b.record(stream)
        b.synchronize()
        barrier()
        e_ms = max_over_ranks(a.elapsed_time(b))
        e2e = {"value": round(flops_all * args.steps / (e_ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(sum_over_ranks(float(h2d))),
               "d2h_bytes_per_step": int(sum_over_ranks(float(d2h))),
               "ms_per_step": round(e_ms / args.steps, 3)}

    gathered = None
    if args.gather and distributed:
        torch.cuda.synchronize(dev)
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for y in ys:
            gather_outputs(y, world)
        b.record(stream)
        b.synchronize()
        gathered = {"allgather_ms_per_step": round(max_over_ranks(a.elapsed_time(b)), 3)}

    # ---- comparison points: cuDNN on the same GPU, per layer and per step -------------
    cudnn = None
    if rank == 0 and world == 1 and not args.no_cudnn:
        per = cudnn_layers(torch, specs, n_local, dev)
        cudnn = {"method": "torch.nn.functional.conv2d, cudnn.benchmark, faster of NCHW / "
                           "channels_last per layer, CUDA events over 10 eager calls"}
        for prec in ("fp32", "tf32"):
            ms = sum(per[s.name][prec] for s in specs)
            cudnn[prec] = {"value": round(flops_local / (ms / 1e3) / 1e9, 3), "unit": "GFLOP/s",
                           "ms_per_step": round(ms, 4),
                           "ours_speedup": round(ms / (t_max_ms / args.steps), 3)}
        for row in per_layer:
            row["cudnn_fp32_ms"] = per[row["layer"]]["fp32"]
            row["cudnn_tf32_ms"] = per[row["layer"]]["tf32"]

    # ---- the paper's bound against the SM<->L2 traffic (per layer) --------------------
    from paper_2012_15667_b200.device import b200_hw_model
    hw_b200 = b200_hw_model()
    bounds_cache = {}
    for row, s in zip(per_layer, specs):
        key = (s.name, row["_alg"], row["_e"])
        if key not in bounds_cache:
            b = layer_io_bounds(s, n_local, row["_alg"], row["_e"], hw_b200)
            m = _l2_measured(traffic_tab, args.workload, s.name, row["_alg"], n_local)
            if m is not None:
                b["measured_l2_sm_read_bytes"] = m["l2_sm_read_bytes_per_call"]
                b["measured_dram_bytes"] = m.get("dram_bytes_per_call")
                b["measured_over_omega"] = round(m["l2_sm_read_bytes_per_call"] / b["omega_bytes"], 3)
                b["measured_over_io_at_optimum"] = round(
                    m["l2_sm_read_bytes_per_call"] / b["io_at_optimum_bytes"], 3)
                b["source"] = m.get("source", f"committed ncu capture (profiles/{PROFILE_ROUND}/*_traffic.json)")
            else:
                b["measured_l2_sm_read_bytes"] = None
            bounds_cache[key] = b
        row["l2_sm_bytes_vs_bound"] = bounds_cache[key]
    for row in per_layer:
        row.pop("_alg", None)
        row.pop("_e", None)

    network = None
    if rank == 0 and world == 1 and not args.no_network:
        try:
            network = network_bench(torch, dev, args.steps, args.warmup)
        except Exception as exc:  # noqa: BLE001
            network = {"unavailable": str(exc)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        try:
            sample_layers = specs
            gf, el = cpu_oracle_gflops(sample_layers, 1, cores)
            cpu = {"value": round(gf, 3), "unit": "GFLOP/s", "cores": cores, "kind": "port",
                   "sample": f"1 image x {len(sample_layers)} layers, C oracle (oracle/conv_oracle.c, "
                             f"fp64 accumulate, OpenMP), {el:.2f} s"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "GFLOP/s", "cores": cores, "kind": "port",
                   "sample": f"unavailable: {exc}"}
        try:
            gf, el = onednn_gflops(specs, cores, images=4)
            cpu["onednn"] = {"value": round(gf, 3), "unit": "GFLOP/s", "cores": cores,
                             "sample": f"4 images x {len(specs)} layers, torch.nn.functional.conv2d fp32 "
                                       f"on the host (oneDNN), median of 3, {el:.2f} s per pass"}
        except Exception as exc:  # noqa: BLE001
            cpu["onednn"] = {"value": None, "sample": f"unavailable: {exc}"}
        try:
            cpu["model"] = model_cpu_timings()
            cpu["model"]["what"] = ("the reference's CPU path (lower bound, analytic tile, schedule + "
                                    "simulate, Table-1 space, GBR tune) via this package's bit-exact "
                                    "restatement, 1 thread")
        except Exception as exc:  # noqa: BLE001
            cpu["model"] = {"unavailable": str(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": WORKLOAD_NAME[args.workload], "global_batch": n_total,
                "parallelism": f"batch-sharded x{world} (no data-path collective)",
                "l2": ("flushed between steps" if flush else
                       f"per-step working set {work_bytes / 2**30:.2f} GiB per GPU > 126 MB L2"),
                "tuned_plans": bool(plans),
                "step": ("filter prep + all convs replayed as one CUDA graph, repeated same-plan 3xF16 "
                         "layers as grouped launches (" + ", ".join(
                             f"{arm.layers[idx[0]].spec.name} x{len(idx)}" for kind, _, idx in arm.units
                             if kind == "group") + "); per_layer / roofline from an eager pass with one "
                         f"launch per layer and per-layer events ({eager_ms / args.steps:.4f} ms/step)"
                         if graph_used else "eager launches, one per layer"),
                "tuned_table": os.path.basename(tuned_table(args.workload, n_local)),
                "group_table": (os.path.basename(group_table(args.workload))
                                if not args.no_group and os.path.exists(group_table(args.workload)) else None),
                "plans": "per layer the fastest device-tuned FP32-accurate algorithm: direct / Winograd "
                         "(FFMA), 3xTF32 tcgen05 implicit GEMM or 3xTF32 tcgen05 Winograd "
                         "(FP32-level GEMM accuracy)",
            },
            "e2e": e2e,
            "roofline": roofline,
            "variants": variants,
            "cpu_baseline": cpu,
            "cudnn": cudnn,
            "network": network,
            "clocks": clk,
            "gpu_launches": launches,
            "per_layer": per_layer,
        }
        if gathered:
            line["gather"] = gathered
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
