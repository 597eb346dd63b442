"""Batch sharding across ranks with world_size 2 on gloo/CPU.

The GPU path shards images with no data-path collective and all-gathers the
outputs over NCCL only when asked; the host logic (partitioning, replicated
filters, gather order, max-over-ranks timing) is exercised here on CPU with
the oracle standing in for the per-rank conv.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_15667_b200.runner import (RESNET50_3X3, shard_range, make_weights,
                                          gather_outputs, LayerSpec)


def test_shard_ranges_partition_the_batch():
    for n in (1, 7, 32, 256, 255):
        for world in (1, 2, 4, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_resnet_layer_list_matches_baseline_config():
    from paper_2012_15667_b200.runner import expand
    layers = expand(RESNET50_3X3)
    assert len(layers) == 16
    total = sum(s.flops(256) for s in layers)
    assert total == 16 * 59190018048      # 59.19 GFLOP each at N=256


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import conv_oracle
        spec = LayerSpec("t", 3, 8, 4)
        w = make_weights(spec, "cpu", 1000)          # replicated by seed on every rank
        g = torch.Generator().manual_seed(5)
        x_full = torch.rand((n_total, spec.c, spec.hw, spec.hw), generator=g) * 2 - 1
        lo, hi = shard_range(n_total, rank, world)
        y_local = torch.from_numpy(conv_oracle.direct_conv(x_full[lo:hi].numpy(), w.numpy(), 1, 1)).float()
        y = gather_outputs(y_local, world)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wsum = torch.tensor([float(w.sum())], dtype=torch.float64)
        dist.all_reduce(wsum)
        if rank == 0:
            ref = conv_oracle.direct_conv(x_full.numpy(), w.numpy(), 1, 1)
            q.put((float(np.max(np.abs(y.numpy() - ref))), float(t.item()),
                   float(wsum.item()), float(w.sum()) * world))
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_conv_gather_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 6, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    err, tmax, wsum, wsum_expect = q.get(timeout=10)
    assert err < 1e-6                      # gathered shards == full-batch conv
    assert tmax == 2.0                     # max over ranks
    assert wsum == pytest.approx(wsum_expect)   # identical replicated filters


def _bench(*argv, env=None):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *argv], capture_output=True,
                       text=True, timeout=300, env=e, cwd=root)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r.returncode, (json.loads(lines[-1]) if lines else None), r.stderr


def test_bench_gpus_2_relaunches_two_ranks():
    """``bench.py --gpus 2`` re-executes under torchrun: two gloo ranks shard the
    batch, time with barrier + max over ranks, and rank 0 reports n_gpus 2."""
    rc, line, err = _bench("--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "3", "--batch", "3")
    assert rc == 0, err[-2000:]
    assert line["n_gpus"] == 2
    assert line["config"]["images_over_ranks"] == 3       # 2 + 1 images: the whole batch
    assert line["value"] > 0 and line["ms_per_step"] > 0


def test_bench_rejects_world_size_mismatch():
    rc, line, err = _bench("--gpus", "2", "--dry-run", env={"WORLD_SIZE": "1"})
    assert rc != 0 and line is None
    assert "--gpus 2" in err
