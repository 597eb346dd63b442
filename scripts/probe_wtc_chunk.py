"""Tensor-core Winograd: time vs chunk budget (tile s_b; chunk V + M = 16 KB x s_b).

    python scripts/probe_wtc_chunk.py --workload resnet50 --layer res5_3x3 --n 256
    python scripts/probe_wtc_chunk.py ... --one 4096      (one s_b, 3 calls: the ncu target)
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import TileConfig  # noqa: E402
from paper_2012_15667_b200 import conv as C  # noqa: E402
from paper_2012_15667_b200 import runner as R  # noqa: E402
from scripts.probe_tc import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--layer", default="res5_3x3")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--z", type=int, default=256)
    ap.add_argument("--nzt", type=int, default=2)
    ap.add_argument("--e", type=int, default=4)
    ap.add_argument("--one", type=int, default=0)
    ap.add_argument("--sweep", default="512,1024,2048,4096,8192,16384")
    args = ap.parse_args()
    spec = next(s for s in R.WORKLOADS[args.workload] if s.name == args.layer)
    x = C.to_layout(torch.rand(args.n, spec.c, spec.hw, spec.hw, device="cuda") * 2 - 1, "HWC")
    w = (torch.rand(spec.k, spec.c, 3, 3, device="cuda") * 2 - 1) / (spec.c * 9) ** 0.5
    u = C.winograd_filter_transform_tc(w, args.e, "3xtf32")
    out = C.empty_act(args.n, spec.k, spec.out_hw, spec.out_hw, "HWC", device="cuda")
    for sb in ([args.one] if args.one else [int(v) for v in args.sweep.split(",")]):
        tile = TileConfig(args.e, args.e, args.z, sb, 1, 1, args.nzt, layout="HWC", e=args.e)
        info = C.query(tuple(x.shape), tuple(w.shape), 1, 1, "HWC", tile, "winograd_tc_3xtf32")
        ws = torch.empty(info["workspace_bytes"], dtype=torch.uint8, device="cuda")

        def fn():
            return C.conv_winograd_tc(x, w, e=args.e, padding=1, tile=tile, precision="3xtf32",
                                      u=u, out=out, workspace=ws)
        if args.one:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            return
        t = timeit(fn, reps=10)
        print(f"{args.layer} s_b={sb:6d} chunk={16 * sb // 1024:5d} MB  {t * 1e3:.3f} ms  "
              f"{info['reason'][-60:]}", flush=True)


if __name__ == "__main__":
    main()
