"""BASELINE config 5: lower-bound-pruned search vs exhaustive, on the device.

    python scripts/tuner_sweep.py [--n 8] [--budget 64] [--cap 6000] [--out FILE]
    python scripts/tuner_sweep.py --engine igemm_3xf16 --n 32 --budget 16
        (the shipped tensor-core kernels: I/O-pruned tcgen05 domain vs its
         unpruned legal domain, device_tuner.tcgen05_space)

For 10 MobileNet-v1 / SqueezeNet-1.1 / ResNet-50 layers:
  * unconstrained domain = divisor constraints and xyz <= s_b only
    (the reference's ``unconstrained_size``, autotune.py:92-156), and the
    Table-1 pruned domain (``build_space``), both restricted to their legal
    device projection;
  * exhaustive device search of each (capped at --cap members, uniformly
    subsampled above that and marked so);
  * the reference tuner (GBR + random walks, ``tune(..., backend="device")``)
    on the pruned projection with --budget measurements, and random search.
Reports sizes, reduction ratio, best device time of each, and measurements
the tuner needed to reach its best.
"""

import argparse
import json
import math
import os
import sys
import time
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_15667_b200 import autotune as A  # noqa: E402
from paper_2012_15667_b200 import device_tuner as DT  # noqa: E402
from paper_2012_15667_b200.dataflow import TileConfig, divisors, LAYOUTS  # noqa: E402
from paper_2012_15667_b200.device import b200_hw_model, shape_of  # noqa: E402
from paper_2012_15667_b200.autotune import ConfigSpace  # noqa: E402

# name, C_in, input H=W, K, kernel, stride, pad
LAYERS = [
    ("mobilenet_conv1", 3, 224, 32, 3, 2, 1),
    ("mobilenet_pw2", 32, 112, 64, 1, 1, 0),
    ("mobilenet_pw_256", 256, 28, 256, 1, 1, 0),
    ("mobilenet_pw_512", 512, 14, 512, 1, 1, 0),
    ("squeezenet_conv1", 3, 224, 64, 3, 2, 0),
    ("squeezenet_fire2_squeeze", 64, 55, 16, 1, 1, 0),
    ("squeezenet_fire2_expand3", 16, 55, 64, 3, 1, 1),
    ("squeezenet_fire9_expand3", 64, 13, 256, 3, 1, 1),
    ("resnet50_res2_3x3", 64, 56, 64, 3, 1, 1),
    ("resnet50_res5_3x3", 512, 7, 512, 3, 1, 1),
]


def unconstrained_space(shape, hw, thread_axes=True):
    """Divisor constraints + xyz <= s_b only (no Table-1 prune), CHW layout."""
    r = A.reuse_factor(shape)
    dx, dy, dz = divisors(shape.w_out), divisors(shape.h_out), divisors(shape.c_out)
    members = []
    for s_b in A.default_sb_values(hw):
        for x in dx:
            for y in dy:
                for z in dz:
                    if x * y * z > s_b:
                        continue
                    thr = ([(a, b, c) for a in divisors(x) for b in divisors(y) for c in divisors(z)]
                           if thread_axes else [(1, 1, 1)])
                    members.extend(TileConfig(x, y, z, s_b, a, b, c, "CHW") for a, b, c in thr)
    members.sort(key=A._member_key)
    return ConfigSpace(shape, hw, "direct", None, r, tuple(members), len(members))


def exhaustive(space, cap, seed=0):
    members = list(space.members)
    sampled = len(members) > cap
    if sampled:
        idx = np.random.default_rng(seed).choice(len(members), size=cap, replace=False)
        members = [members[i] for i in sorted(int(i) for i in idx)]
    best, best_t = None, math.inf
    t0 = time.time()
    for cfg in members:
        t = A.measure(cfg, space.shape, space.hw, "direct", backend="device").cost
        if t < best_t:
            best, best_t = cfg, t
    return {"best": best.to_dict() if best else None, "seconds": None if math.isinf(best_t) else best_t,
            "measured": len(members), "sampled": sampled, "wall_s": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--budget", type=int, default=64)
    ap.add_argument("--cap", type=int, default=6000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--engine", default="ffma", choices=DT.ENGINES)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    args.out = args.out or os.path.join(ROOT, "gpurun_out", f"tuner_sweep_{args.engine}.json")
    warnings.simplefilter("ignore")
    DT.TIMING.update(target_ms=0.5, batches=3)
    DT.set_engine(args.engine)
    tc = args.engine != "ffma"
    hw = DT.tcgen05_hw_model() if tc else b200_hw_model()
    rows = []
    for name, c, hw_in, k, r, stride, pad in LAYERS:
        DT.set_padding(pad)
        shape = shape_of(args.n, c, hw_in, hw_in, k, r, stride, pad)
        try:
            if tc:
                pruned = DT.tcgen05_space(shape, hw, args.engine)
                unc = DT.tcgen05_space(shape, hw, args.engine, prune=None)
            else:
                pruned = DT.legal_projection(A.build_space(shape, hw, "direct", layouts=("CHW",)))
                unc = DT.legal_projection(unconstrained_space(shape, hw))
        except A.InfeasibleTileError as exc:
            row = {"layer": name, "shape": str(shape), "error": str(exc)}
            print(json.dumps(row), flush=True)
            rows.append(row)
            continue
        row = {"layer": name, "shape": str(shape),
               "unconstrained_legal": unc.size, "pruned_legal": pruned.size,
               "reduction_ratio": round(pruned.size / unc.size, 4),
               "model_reduction_ratio": (round(unc.unconstrained_size and pruned.size / unc.unconstrained_size, 4)
                                         if tc else
                                         round(A.build_space(shape, hw, "direct", layouts=("CHW",))
                                               .reduction_ratio, 4))}
        row["exhaustive_unconstrained"] = exhaustive(unc, args.cap, args.seed)
        row["exhaustive_pruned"] = exhaustive(pruned, args.cap, args.seed)
        t0 = time.time()
        sess = A.tune(shape, hw, "direct", min(args.budget, pruned.size), args.seed,
                      n_s=min(16, max(2, min(args.budget, pruned.size) // 4)), space=pruned,
                      backend="device")
        row["tuner_pruned"] = {"best": sess.best.config.to_dict() if sess.best else None,
                               "seconds": sess.best.cost if sess.best else None,
                               "measurements": len(sess.measurements),
                               "measurements_to_best": sess.best.index + 1 if sess.best else None,
                               "wall_s": round(time.time() - t0, 1)}
        cfg, cost = A.random_search(pruned, min(args.budget, pruned.size), args.seed, backend="device")
        row["random_pruned"] = {"seconds": None if math.isinf(cost) else cost}
        ex = row["exhaustive_unconstrained"]["seconds"]
        tb = row["tuner_pruned"]["seconds"]
        row["tuner_vs_exhaustive_unconstrained"] = round(tb / ex, 4) if ex and tb else None
        print(json.dumps(row), flush=True)
        rows.append(row)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump({"n": args.n, "budget": args.budget, "cap": args.cap, "engine": args.engine,
                   "layers": rows}, fh, indent=1)
    print(f"wrote {args.out}")


if __name__ == "__main__":
    main()
