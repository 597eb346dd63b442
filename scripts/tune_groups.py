"""Tune the grouped launches of a workload's repeated same-shape 3xF16 layers
(``runner.group_layers``): for each per-layer batch n and each group of G layers, time
the grouped launch with every igemm_3xf16 tile the per-batch tables hold for that layer
(a G*n-image GEMM often prefers a tile tuned at a larger batch), keep the fastest, and
record whether it beats G single launches on the layers' own plans.

    python scripts/tune_groups.py --workload resnet50 [--batches 32,64,128,256]

Writes paper_2012_15667_b200/tuned/b200_<workload>_groups.json (read by
runner.load_group_plans; bench.py's timed step uses it).
"""

import argparse
import glob
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import conv as C  # noqa: E402
from paper_2012_15667_b200.dataflow import TileConfig  # noqa: E402
from paper_2012_15667_b200.runner import (TUNED_DIR, WORKLOADS, ConvLayer, expand, group_layers,  # noqa: E402
                                           group_table, load_plans, make_input, make_weights, prepare_layers)


def candidate_tiles(workload, name):
    """Every igemm_3xf16 tile of layer ``name`` across the workload's tuned tables."""
    tiles = []
    for path in sorted(glob.glob(os.path.join(TUNED_DIR, f"b200_{workload}*.json"))):
        if path.endswith("_groups.json"):
            continue
        ent = json.load(open(path)).get("layers", {}).get(name, {})
        best = (ent.get("candidates", {}).get("igemm_3xf16", {}).get("tuner") or {}).get("best")
        if best:
            t = TileConfig(**best)
            if t not in tiles:
                tiles.append(t)
    return tiles


def time_us(fn, reps, rounds=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(rounds):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / reps * 1e3)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--batches", default="32,64,128,256")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda")
    specs = expand(WORKLOADS[args.workload])
    out = {"workload": args.workload, "device": torch.cuda.get_device_name(),
           "method": "grouped launch timed with CUDA events (median of 5 x reps back-to-back), "
                     "candidates = the layer's igemm_3xf16 tiles from every per-batch table",
           "groups": {}}
    for n in [int(b) for b in args.batches.split(",")]:
        plans = load_plans(args.workload, n=n)
        layers = [ConvLayer(s, make_weights(s, dev, 1000 + i), plans.get(s.name)) for i, s in enumerate(specs)]
        units = group_layers(layers, n, dev)
        prepare_layers(layers, dev)
        res = {}
        for kind, grp, idx in units:
            if kind != "group":
                continue
            name = specs[idx[0]].name
            for g, i in enumerate(idx):
                grp.x_of(g).copy_(make_input(specs[i], n, dev, seed=7919 * (i + 1), layout="HWC"))
            own = grp.tile
            cands = []
            for t in [own] + [t for t in candidate_tiles(args.workload, name) if t != own]:
                grp.tile = t
                try:
                    us = time_us(lambda: grp.run(), args.reps)
                except Exception as exc:  # noqa: BLE001 -- infeasible for this batch: recorded
                    cands.append({"tile": t.to_dict(), "error": str(exc).splitlines()[0][:160]})
                    continue
                cands.append({"tile": t.to_dict(), "us": round(us, 2)})
            ok = [c for c in cands if "us" in c]
            best = min(ok, key=lambda c: c["us"])
            # the alternative: G single launches, each layer on its own tuned plan
            ys = [C.empty_act(n, specs[i].k, specs[i].out_hw, specs[i].out_hw, "HWC", device=dev) for i in idx]

            def singles():
                for j, i in enumerate(idx):
                    layers[i].run(grp.x_of(j), out=ys[j])
            singles_us = time_us(singles, args.reps)
            res[name] = {"layers": len(idx), "n": n, "tile": best["tile"], "us": best["us"],
                         "own_plan_us": ok[0]["us"] if cands and "us" in cands[0] else None,
                         "singles_us": round(singles_us, 2), "use_group": best["us"] < singles_us,
                         "candidates": cands}
            grp.tile = own
            print(f"n={n:4d} {name:12s} x{len(idx)} best {best['us']:8.2f} us (own plan {res[name]['own_plan_us']}, "
                  f"singles {singles_us:.2f}) {TileConfig(**best['tile'])}", flush=True)
        out["groups"][str(n)] = res
        del layers, units
        torch.cuda.empty_cache()
    path = group_table(args.workload)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
