"""Run one conv configuration a few times (target for ncu captures).

    python scripts/run_one.py --alg direct --n 32 --c 64 --hw 56 --k 64 \
        --tile 56,4,64,32768,7,4,8 [--e 2] [--reps 3]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import TileConfig  # noqa: E402
from paper_2012_15667_b200 import conv as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alg", default="direct")
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--c", type=int, default=64)
    ap.add_argument("--hw", type=int, default=56)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--e", type=int, default=2)
    ap.add_argument("--tile", default="")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    x = torch.randn(args.n, args.c, args.hw, args.hw, device="cuda")
    w = torch.randn(args.k, args.c, 3, 3, device="cuda") / (args.c * 9) ** 0.5
    tile = None
    if args.tile:
        v = [int(t) for t in args.tile.split(",")]
        tile = TileConfig(*v[:7], e=args.e if args.alg == "winograd" else None)
    if args.alg == "direct":
        wp = C.pack_filter_direct(w)
        for _ in range(args.reps):
            C.conv_direct(x, w, stride=args.stride, padding=1, tile=tile, w_packed=wp)
        print(C.query(x.shape, w.shape, args.stride, 1, "CHW", tile) if tile else "default tile")
    else:
        u = C.winograd_filter_transform(w, args.e)
        for _ in range(args.reps):
            C.conv_winograd(x, w, e=args.e, padding=1, tile=tile, u=u)
        print(C.query(x.shape, w.shape, 1, 1, "CHW", tile, "winograd") if tile else "default tile")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
