"""Where a bench step's time goes at a given batch: each unit of the timed step (the
filter prep, each grouped launch, each single layer) captured as its own CUDA graph
and replayed back to back, against the whole step as one graph.

    python scripts/dev/step_breakdown.py --batch 32 [--no-group]
    CONVIO_DEV_SKIP_CHECK=1 python scripts/dev/step_breakdown.py --batch 32   (no checking launch)

Development tool; the contract numbers come from bench.py.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import conv as C  # noqa: E402
from paper_2012_15667_b200.runner import (WORKLOADS, ConvLayer, expand, group_layers,  # noqa: E402
                                           load_group_overrides, load_group_plans, load_plans, make_input, make_weights,
                                           prepare_layers)


def graph_of(fn, stream):
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        fn(side)
        fn(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        fn(side)
    torch.cuda.synchronize()
    return g


def time_graph(g, reps):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3   # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--no-group", action="store_true")
    ap.add_argument("--allowed", default="", help="comma list: restrict the plans to these algorithms")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = args.batch
    specs = expand(WORKLOADS[args.workload])
    plans = (load_plans(args.workload, allowed=tuple(args.allowed.split(",")), n=n) if args.allowed
             else load_plans(args.workload, n=n))
    if not args.no_group and not args.allowed:
        plans.update(load_group_overrides(args.workload, n))
    layers = [ConvLayer(s, make_weights(s, dev, 1000 + i), plans.get(s.name)) for i, s in enumerate(specs)]
    xs = [make_input(s, n, dev, seed=7919 * (i + 1), layout=l.layout) for i, (s, l) in enumerate(zip(specs, layers))]
    ys = [C.empty_act(n, s.k, s.out_hw, s.out_hw, l.layout, device=dev) for s, l in zip(specs, layers)]
    units = ([("single", l, [i]) for i, l in enumerate(layers)] if args.no_group else
             group_layers(layers, n, dev, load_group_plans(args.workload, n)))
    for kind, u, idx in units:
        if kind == "group":
            for g, i in enumerate(idx):
                u.x_of(g).copy_(xs[i])
                xs[i], ys[i] = u.x_of(g), u.y_of(g)
    stream = torch.cuda.current_stream()

    def run_unit(unit, st):
        kind, u, idx = unit
        if kind == "group":
            u.run(st)
        else:
            u.run(xs[idx[0]], out=ys[idx[0]], stream=st)

    def step(st):
        prepare_layers(layers, dev, st)
        for unit in units:
            run_unit(unit, st)

    rows = []
    t_step = time_graph(graph_of(step, stream), args.reps)
    t_prep = time_graph(graph_of(lambda st: prepare_layers(layers, dev, st), stream), args.reps)
    rows.append({"unit": "prep", "us": round(t_prep, 2)})
    total = t_prep
    for unit in units:
        t = time_graph(graph_of(lambda st, unit=unit: run_unit(unit, st), stream), args.reps)
        kind, u, idx = unit
        f = sum(specs[i].flops(n) for i in idx)
        name = specs[idx[0]].name + (f" x{len(idx)}" if kind == "group" else "")
        alg = layers[idx[0]].algorithm
        rows.append({"unit": name, "alg": alg, "us": round(t, 2), "tflops": round(f / t / 1e6, 1),
                     "launches": u.launches})
        total += t
    out = {"batch": n, "grouped": not args.no_group, "skip_check": bool(os.environ.get("CONVIO_DEV_SKIP_CHECK")),
           "step_us": round(t_step, 2), "sum_of_units_us": round(total, 2),
           "step_tflops": round(sum(s.flops(n) for s in specs) / t_step / 1e6, 1), "units": rows}
    print(json.dumps(out))
    for r in rows:
        print(f"  {r['unit']:18s} {r.get('alg', ''):20s} {r['us']:8.2f} us  {r.get('tflops', '')}")


if __name__ == "__main__":
    main()
