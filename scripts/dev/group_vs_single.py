"""Grouped launch of G same-shape layers vs one layer over the stacked batch (same
tile) vs G single launches.  Development tool.

    python scripts/dev/group_vs_single.py --layer res2_3x3 --n 128 --g 3
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import conv as C  # noqa: E402
from paper_2012_15667_b200.dataflow import TileConfig  # noqa: E402
from paper_2012_15667_b200.runner import WORKLOADS, load_plans, make_weights  # noqa: E402


def t_us(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="res2_3x3")
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--g", type=int, default=3)
    ap.add_argument("--plan-n", type=int, default=0)
    ap.add_argument("--tile", default="", help="x,y,z,s_b,n_xt,n_yt,n_zt (HWC) instead of the table's")
    args = ap.parse_args()
    s = next(x for x in WORKLOADS["resnet50"] if x.name == args.layer)
    tile = (TileConfig(*[int(v) for v in args.tile.split(",")], layout="HWC") if args.tile
            else load_plans("resnet50", n=args.plan_n or args.n)[s.name]["tile"])
    n, g = args.n, args.g
    dev = torch.device("cuda")
    w = make_weights(s, dev, 1)
    wp = C.pack_filter_igemm_f16x3(w)
    sb = C.f16x3_slice_bytes(s.k, s.c, 3, 3)
    wg = torch.zeros(g * sb, dtype=torch.uint8, device=dev)
    for i in range(g):
        wg[i * sb:i * sb + wp.numel()] = wp
    x = C.to_layout(torch.rand(n * g, s.c, s.hw, s.hw, device=dev) - 0.5, "HWC")
    y = C.empty_act(n * g, s.k, s.out_hw, s.out_hw, "HWC", device=dev)
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    f = s.flops(n * g)

    def single_big():
        C.conv_igemm(x, w, padding=s.pad, stride=s.stride, tile=tile, precision="3xf16", w_packed=wp, out=y,
                     workspace=ws)

    xs = [x[i * n:(i + 1) * n] for i in range(g)]
    ys = [y[i * n:(i + 1) * n] for i in range(g)]

    def singles():
        for i in range(g):
            C.conv_igemm(xs[i], w, padding=s.pad, stride=s.stride, tile=tile, precision="3xf16", w_packed=wp,
                         out=ys[i], workspace=ws)

    def grouped():
        C.conv_igemm_grouped(x, (s.k, s.c, 3, 3), wg, g, sb, padding=s.pad, stride=s.stride, tile=tile, out=y,
                             workspace=ws)

    print(s.name, "n", n, "g", g, tile)
    for name, fn in (("one launch, stacked batch", single_big), ("g single launches", singles),
                     ("grouped", grouped)):
        t = t_us(fn)
        print(f"  {name:28s} {t:8.2f} us  {f / t / 1e6:7.1f} TF/s  launches {C.last_launch_count()}")
    q = C.query((n * g, s.c, s.hw, s.hw), (s.k, s.c, 3, 3), s.stride, s.pad, "HWC", tile, "igemm_3xf16")
    print("  plan:", q.get("reason") or q)


if __name__ == "__main__":
    main()
