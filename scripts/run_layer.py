"""Run one tuned layer of a workload (its bench plan) a few times: the ncu target
for the per-launch DRAM traffic that bench.py reports as ``roofline.traffic``.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/traffic_res4.csv \
        python scripts/run_layer.py --workload resnet50 --layer res4_3x3
    python scripts/run_layer.py --parse gpurun_out/traffic_*.csv --out profiles/r2/r2_resnet50_traffic.json
"""

import argparse
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(args):
    import torch
    from paper_2012_15667_b200 import conv as C
    from paper_2012_15667_b200.runner import (WORKLOADS, DEFAULT_BATCH, ConvLayer, load_plans,
                                               make_input, make_weights)
    spec = next(s for s in WORKLOADS[args.workload] if s.name == args.layer)
    n = args.batch or DEFAULT_BATCH[args.workload]
    plan = load_plans(args.workload).get(spec.name)
    dev = torch.device("cuda")
    if args.group:   # the bench's grouped launch of the layer's `count` repeats
        from paper_2012_15667_b200.runner import group_layers, load_group_plans, prepare_layers
        layers = [ConvLayer(spec, make_weights(spec, dev, 1000 + i), plan) for i in range(spec.count)]
        units = group_layers(layers, n, dev, load_group_plans(args.workload, n))
        kind, grp, _ = units[0]
        if kind != "group":
            raise SystemExit(f"{spec.name}: no grouped launch at n={n}")
        for g in range(spec.count):
            grp.x_of(g).copy_(make_input(spec, n, dev, seed=7919 + g, layout="HWC"))
        prepare_layers(layers, dev)
        for _ in range(args.reps):
            grp.run()
        torch.cuda.synchronize()
        meta = {"layer": spec.name, "algorithm": layers[0].algorithm, "group": spec.count, "reps": args.reps,
                "tile": grp.tile.to_dict(), "n": n}
        if args.meta:
            with open(args.meta, "w") as fh:
                json.dump(meta, fh)
        print(json.dumps(meta))
        return
    layer = ConvLayer(spec, make_weights(spec, dev, 1000), plan)
    x = make_input(spec, n, dev, seed=7919, layout=layer.layout)
    y = C.empty_act(n, spec.k, spec.out_hw, spec.out_hw, layer.layout, device=dev)
    layer.prepare(dev)
    for _ in range(args.reps):
        layer.run(x, out=y)
    torch.cuda.synchronize()
    meta = {"layer": spec.name, "algorithm": layer.algorithm, "e": layer.e, "reps": args.reps,
            "tile": None if layer.tile is None else layer.tile.to_dict(), "n": n}
    if args.meta:
        with open(args.meta, "w") as fh:
            json.dump(meta, fh)
    print(json.dumps(meta))


def parse(paths, workload, out):
    """Per (layer, algorithm): DRAM bytes per call, summed over the call's kernels
    (filter prep excluded), from the last complete call in each ncu CSV."""
    table = {}
    for path in paths:
        meta_path = path[:-4] + ".json"
        if not os.path.exists(meta_path):
            continue
        meta = json.load(open(meta_path))
        rows = list(csv.reader(open(path)))
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]
        ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
        per = {}
        names = {}
        # ncu prints byte metrics with units (e.g. "Mbyte") unless --print-units base
        for r in rows[hdr + 1:]:
            if len(r) < len(h) or "pack_filter" in r[ki] or "filter_tc" in r[ki] or "filter_transform" in r[ki] or "u_split" in r[ki]:
                continue
            per.setdefault(int(r[ii]), {})[r[ni]] = float(r[vi].replace(",", ""))
            names[int(r[ii])] = r[ki].split("(")[0]
        ids = sorted(per)
        calls = meta.get("reps", 2)
        last = ids[-(len(ids) // calls):] if calls and len(ids) >= calls else ids
        l2 = sum(per[i].get("lts__t_sectors_srcunit_tex_op_read.sum", 0) for i in last) * 32
        xbar = sum(per[i].get("l1tex__m_xbar2l1tex_read_bytes.sum", 0) for i in last)
        rd = sum(per[i].get("dram__bytes_read.sum", 0) for i in last)
        wr = sum(per[i].get("dram__bytes_write.sum", 0) for i in last)
        ns = sum(per[i].get("gpu__time_duration.sum", 0) for i in last)
        key = f"{workload}:{meta['layer']}:{meta['algorithm']}"
        table[key] = {"dram_bytes_per_call": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                      "kernels_per_call": len(last), "ncu_ns_per_call": ns,
                      "kernels": sorted({names[i] for i in last}), "n": meta.get("n"),
                      "tile": meta.get("tile")}
        if l2:
            table[key]["l2_sm_read_bytes_per_call"] = int(l2)
            table[key]["l1tex_xbar_read_bytes_per_call"] = int(xbar)
            table[key]["source"] = ("ncu --cache-control none, last of 3 calls: lts__t_sectors_srcunit_tex_op_read"
                                    ".sum x 32 B (SM -> L2 reads incl. TMA), dram__bytes_read/write.sum")
    with open(out, "w") as fh:
        json.dump(table, fh, indent=1, sort_keys=True)
    print(json.dumps(table, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--layer", default="res4_3x3")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--meta", default="", help="write the run's plan as JSON here")
    ap.add_argument("--group", action="store_true",
                    help="run the layer's repeats as the bench's grouped launch (runner.LayerGroup)")
    ap.add_argument("--parse", nargs="*")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if args.parse is not None:
        paths = [p for pat in args.parse for p in glob.glob(pat)]
        parse(paths, args.workload, args.out)
    else:
        run(args)


if __name__ == "__main__":
    main()
