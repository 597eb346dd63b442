"""Tune the grouped launches of a workload's repeated same-shape 3xF16 layers
(``runner.group_layers``): for each per-layer batch n and each group of G layers, time
the grouped launch with every igemm_3xf16 tile the per-batch tables hold for that layer
(a G*n-image GEMM often prefers a tile tuned at a larger batch), keep the fastest, and
record whether it beats G single launches on the layers' own plans.  Repeated layers
on another plan (Winograd) are offered the same grouped 3xF16 launch, compared with
each side's filter prep included; a win replaces their plan (runner.load_group_overrides).

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


def domain_tiles(spec, n_stacked, cap):
    """The 3xF16 tcgen05 searching domain of the STACKED problem (device_tuner.tcgen05_space
    at batch G*n, I/O-model pruned), the ``cap`` members with the least modelled traffic."""
    from paper_2012_15667_b200.device import shape_of
    from paper_2012_15667_b200.device_tuner import set_padding, tcgen05_hw_model, tcgen05_io_words, tcgen05_space
    set_padding(spec.pad)
    shape = shape_of(n_stacked, spec.c, spec.hw, spec.hw, spec.k, spec.r, spec.stride, spec.pad)
    space = tcgen05_space(shape, tcgen05_hw_model(), "igemm_3xf16", check_legal=False)
    return sorted(space.members, key=lambda t: tcgen05_io_words(shape, t))[:cap]


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


def time_graph_us(fn, reps, rounds=5):
    """``fn(stream)`` captured as one CUDA graph and replayed (no host time between its
    launches: a fair race between a 1-launch and a 4-launch alternative)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn(side)
        fn(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        fn(side)
    torch.cuda.synchronize()
    return time_us(g.replay, reps, rounds)


def merge(paths, out_path):
    """Combine group tables tuned on different boxes (box-to-box spread is ~10 %): per
    group, the tile with the least geometric-mean time over the runs that measured it in
    all of them; a replacement only when it won in every run."""
    import math
    tabs = [json.load(open(p)) for p in paths]
    out = dict(tabs[0])
    out["method"] = tabs[0]["method"] + f"; merged over {len(tabs)} runs on different boxes (geometric mean)"
    out["groups"] = {}
    for n in tabs[0]["groups"]:
        res = {}
        for name, ent in tabs[0]["groups"][n].items():
            ents = [t["groups"].get(n, {}).get(name) for t in tabs]
            if any(e is None for e in ents):
                continue
            key = "us_with_prep" if ent.get("replaces") else "us"
            times = {}
            for e in ents:
                for c in e["candidates"]:
                    if key in c:
                        times.setdefault(json.dumps(c["tile"], sort_keys=True), []).append(c[key])
            full = {k: math.exp(sum(map(math.log, v)) / len(v)) for k, v in times.items() if len(v) == len(tabs)}
            if not full:
                continue
            best = min(full, key=full.get)
            merged = dict(ent)
            merged["tile"] = json.loads(best)
            merged[key] = round(full[best], 2)
            merged["runs"] = [{k: e.get(k) for k in ("tile", key, "own_plan_us", "singles_us", "own_us_with_prep",
                                                     "use_group")} for e in ents]
            if ent.get("replaces"):
                own = math.exp(sum(math.log(e["own_us_with_prep"]) for e in ents) / len(ents))
                merged["own_us_with_prep"] = round(own, 2)
                if not (all(e.get("use_group") for e in ents) and full[best] < 0.97 * own):
                    continue   # not a clear win on every box: keep the layer's own plan
            else:
                singles = math.exp(sum(math.log(e["singles_us"]) for e in ents) / len(ents))
                merged["singles_us"] = round(singles, 2)
                merged["use_group"] = full[best] < singles
            res[name] = merged
        out["groups"][n] = res
    with open(out_path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", out_path)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--merge":   # --merge OUT A.json B.json ...
        merge(sys.argv[3:], sys.argv[2])
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--batches", default="32,64,128,256")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--domain", type=int, default=0,
                    help="also race this many members of the stacked problem's tcgen05 domain")
    args = ap.parse_args()
    dev = torch.device("cuda")
    specs = expand(WORKLOADS[args.workload])
    out = {"workload": args.workload, "device": torch.cuda.get_device_name(),
           "method": "grouped launch timed with CUDA events (median of 5 x reps back-to-back), "
                     "candidates = the layer's igemm_3xf16 tiles from every per-batch table"
                     + (f" + {args.domain} members of the stacked problem's tcgen05 domain (least modelled "
                        "SM<->L2 traffic first)" if args.domain else ""),
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
            tiles = [own] + [t for t in candidate_tiles(args.workload, name) if t != own]
            if args.domain:
                tiles += [t for t in domain_tiles(specs[idx[0]], n * len(idx), args.domain) if t not in tiles]
            for t in tiles:
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
        # repeated layers on another plan (res5's Winograd): one grouped 3xF16 launch instead,
        # compared WITH each side's filter prep (a Winograd U is 4x the filter, a 3xF16 pack 1x)
        i = 0
        while i < len(specs):
            j = i
            while j < len(specs) and specs[j] == specs[i]:
                j += 1
            idx, i = list(range(i, j)), j
            name = specs[idx[0]].name
            own_alg = layers[idx[0]].algorithm
            if len(idx) < 2 or own_alg == "igemm_3xf16" or name in res:
                continue
            ig_plan = load_plans(args.workload, allowed=("igemm_3xf16",), n=n).get(name)
            if not ig_plan:
                continue
            xs = [make_input(specs[k], n, dev, seed=7919 * (k + 1), layout="HWC") for k in idx]
            ys = [C.empty_act(n, specs[k].k, specs[k].out_hw, specs[k].out_hw, "HWC", device=dev) for k in idx]
            own_layers = [layers[k] for k in idx]

            def own_step(st):
                prepare_layers(own_layers, dev, st)
                for q, l in enumerate(own_layers):
                    l.run(xs[q], out=ys[q], stream=st)
            own_us = time_graph_us(own_step, args.reps)
            ig_layers = [ConvLayer(specs[k], layers[k].weight, ig_plan) for k in idx]
            ug = group_layers(ig_layers, n, dev)
            if not ug or ug[0][0] != "group":
                continue
            grp = ug[0][1]
            for q in range(len(idx)):
                grp.x_of(q).copy_(xs[q])
            cands = []
            tiles = [ig_plan["tile"]] + [t for t in candidate_tiles(args.workload, name) if t != ig_plan["tile"]]
            if args.domain:
                tiles += [t for t in domain_tiles(specs[idx[0]], n * len(idx), args.domain) if t not in tiles]
            for t in tiles:
                grp.tile = t

                def ig_step(st):
                    prepare_layers(ig_layers, dev, st)
                    grp.run(st)
                try:
                    us = time_graph_us(ig_step, args.reps)
                except Exception as exc:  # noqa: BLE001 -- infeasible for this batch: recorded
                    cands.append({"tile": t.to_dict(), "error": str(exc).splitlines()[0][:160]})
                    continue
                cands.append({"tile": t.to_dict(), "us_with_prep": round(us, 2)})
            ok = [c for c in cands if "us_with_prep" in c]
            if not ok:
                continue
            best = min(ok, key=lambda c: c["us_with_prep"])
            if best["us_with_prep"] < 0.97 * own_us:   # a clear win only (box-to-box noise ~3 %)
                res[name] = {"layers": len(idx), "n": n, "algorithm": "igemm_3xf16", "replaces": own_alg,
                             "tile": best["tile"], "us_with_prep": best["us_with_prep"],
                             "own_us_with_prep": round(own_us, 2), "use_group": True, "candidates": cands}
            print(f"n={n:4d} {name:12s} x{len(idx)} grouped 3xF16 + pack {best['us_with_prep']:8.2f} us vs "
                  f"{own_alg} + its prep {own_us:8.2f} us -> {'replace' if name in res else 'keep'}", flush=True)
            del ig_layers, ug, grp
        out["groups"][str(n)] = res
        del layers, units
        torch.cuda.empty_cache()
    path = group_table(args.workload)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
