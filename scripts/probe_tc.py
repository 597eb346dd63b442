"""Probe the tensor-core paths per ResNet-50 / VGG-16 3x3 layer: tcgen05 implicit
GEMM (tf32 / 3xtf32 / bf16) and tcgen05 Winograd F(2,3)/F(4,3) against cuDNN.

    python scripts/probe_tc.py [--workload resnet50] [--n 256] [--layers res2_3x3,...]
    python scripts/probe_tc.py --one winograd_tc_3xtf32:4:128 --layers res4_3x3 --reps 3
        (one configuration, a few reps: the ncu capture target)

CUDA-event timing of back-to-back launches (filters pre-transformed), plus the
normwise error against the 3xTF32 implicit GEMM (FP32-level) on the same inputs.
Development tool; the contract numbers come from bench.py.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import TileConfig  # noqa: E402
from paper_2012_15667_b200 import conv as C  # noqa: E402
from paper_2012_15667_b200 import runner as R  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def igemm_tile(spec, z, nzt=1):
    o = spec.out_hw
    # largest x*y <= 128 block with x | Q, y | P, preferring full rows
    best = None
    for x in range(1, o + 1):
        if o % x:
            continue
        for y in range(1, o + 1):
            if o % y or x * y > 128:
                continue
            rows = (128 // (x * y)) * x * y      # images stacked to fill the 128-row tile
            key = (rows, x * y, x)
            if best is None or key > best[0]:
                best = (key, x, y)
    _, x, y = best
    return TileConfig(x, y, z, 32768, 1, 1, nzt, layout="HWC")


TILE_OVERRIDE = None   # --tile x,y,z,s_b,n_xt,n_yt,n_zt for the igemm kinds


def build(spec, kind, n, x, w, wcache):
    """Return a zero-argument launcher for (algorithm kind string)."""
    alg, *rest = kind.split(":")
    if alg.startswith("igemm_"):
        prec = alg[len("igemm_"):]
        z = int(rest[0]) if rest else 128
        nzt = int(rest[1]) if len(rest) > 1 else 2
        if spec.k % z:
            return None
        tile = igemm_tile(spec, z, nzt)
        if len(rest) > 2 and rest[2].startswith("h"):   # halo-staged footprint, fpr = h<N>
            if spec.stride != 1:
                return None
            fpr = int(rest[2][1:])
            tile = TileConfig(fpr - 2, 128 // fpr, z, 32768, 2, 1, nzt, layout="HWC")   # nzt 4: rows into TMEM
        if TILE_OVERRIDE:
            tile = TileConfig(*TILE_OVERRIDE, layout="HWC")
        key = ("ig", "bf16" if prec == "bf16" else ("f16x3" if prec == "3xf16" else "f32"))
        if key not in wcache:
            wcache[key] = (C.pack_filter_igemm_bf16(w) if prec == "bf16" else
                           C.pack_filter_igemm_f16x3(w) if prec == "3xf16" else C.pack_filter_igemm(w))
        wp = wcache[key]
        out = C.empty_act(n, spec.k, spec.out_hw, spec.out_hw, "HWC", device="cuda")
        ws = torch.empty(max(1, n * spec.c * spec.hw * spec.hw * 2 + (1 << 20)), dtype=torch.uint8,
                         device="cuda")
        return lambda: C.conv_igemm(x, w, padding=1, stride=spec.stride, tile=tile, precision=prec,
                                    w_packed=wp, out=out, workspace=ws)
    if alg.startswith("winograd_tc_"):
        if spec.stride != 1:
            return None
        prec = alg[len("winograd_tc_"):]
        e = int(rest[0]) if rest else 4
        z = int(rest[1]) if len(rest) > 1 else 128
        nzt = int(rest[2]) if len(rest) > 2 else 2
        if spec.k % z:
            return None
        key = ("wtc", prec, e)
        if key not in wcache:
            wcache[key] = C.winograd_filter_transform_tc(w, e, prec)
        u = wcache[key]
        tile = TileConfig(e, e, z, 16384, 1, 1, nzt, layout="HWC", e=e)
        out = C.empty_act(n, spec.k, spec.out_hw, spec.out_hw, "HWC", device="cuda")
        info = C.query(x.shape, w.shape, 1, 1, "HWC", tile, "winograd_tc_" + prec)
        if info["rc"]:
            print("  illegal", kind, info["reason"])
            return None
        ws = torch.empty(info["workspace_bytes"], dtype=torch.uint8, device="cuda")
        return lambda: C.conv_winograd_tc(x, w, e=e, padding=1, tile=tile, precision=prec, u=u,
                                          out=out, workspace=ws)
    if alg == "direct_nhwc":
        z = int(rest[0]) if rest else 128
        if spec.k % z or spec.c % 32:
            return None
        t = igemm_tile(spec, z)
        tile = TileConfig(t.x, t.y, z, 32768, 1, 1, 1, layout="HWC")
        if "dwp" not in wcache:
            wcache["dwp"] = C.pack_filter_direct(w)
        out = C.empty_act(n, spec.k, spec.out_hw, spec.out_hw, "HWC", device="cuda")
        return lambda: C.conv_direct(x, w, stride=spec.stride, padding=1, tile=tile,
                                     w_packed=wcache["dwp"], out=out)
    if alg.startswith("cudnn"):
        tf32 = alg == "cudnn_tf32"
        xc = x.contiguous(memory_format=torch.channels_last)
        wc = w.contiguous(memory_format=torch.channels_last)

        def run():
            torch.backends.cudnn.allow_tf32 = tf32
            return torch.nn.functional.conv2d(xc, wc, stride=spec.stride, padding=1)
        return run
    raise ValueError(kind)


KINDS = ["igemm_3xtf32:128", "igemm_3xtf32:64", "igemm_3xtf32:256", "igemm_tf32:128", "igemm_tf32:256",
         "igemm_bf16:128", "igemm_bf16:256",
         "winograd_tc_3xtf32:2:128", "winograd_tc_3xtf32:4:128", "winograd_tc_3xtf32:4:64",
         "winograd_tc_3xtf32:4:256", "winograd_tc_tf32:4:128", "winograd_tc_bf16:4:128",
         "winograd_tc_bf16:4:256", "cudnn_fp32", "cudnn_tf32"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--layers", default="")
    ap.add_argument("--kinds", default=",".join(KINDS))
    ap.add_argument("--one", default="", help="run one kind a few times (ncu target)")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="")
    ap.add_argument("--tile", default="", help="x,y,z,s_b,n_xt,n_yt,n_zt for igemm kinds")
    args = ap.parse_args()
    global TILE_OVERRIDE
    if args.tile:
        TILE_OVERRIDE = [int(v) for v in args.tile.split(",")]
    torch.backends.cudnn.benchmark = True
    specs = R.WORKLOADS[args.workload]
    if args.layers:
        specs = [s for s in specs if s.name in args.layers.split(",")]
    results = []
    for spec in specs:
        if spec.c % 32:
            continue
        g = torch.Generator(device="cuda").manual_seed(0)
        x = (torch.rand(args.n, spec.c, spec.hw, spec.hw, device="cuda", generator=g) * 2 - 1)
        x = C.to_layout(x, "HWC")
        w = (torch.rand(spec.k, spec.c, 3, 3, device="cuda", generator=g) * 2 - 1) / (spec.c * 9) ** 0.5
        wcache = {}
        if args.one:
            fn = build(spec, args.one, args.n, x, w, wcache)
            if fn is None:
                print("skip", args.one, spec.name)
                continue
            for _ in range(args.reps):
                fn()
            torch.cuda.synchronize()
            print("ran", args.one, spec.name)
            continue
        saved, TILE_OVERRIDE = TILE_OVERRIDE, None   # the reference keeps its own tile
        ref = build(spec, "igemm_3xtf32:128:1" if spec.k % 128 == 0 else "igemm_3xtf32:64:1",
                    args.n, x, w, wcache)().clone()
        TILE_OVERRIDE = saved
        flops = spec.flops(args.n)
        for kind in args.kinds.split(","):
            try:
                fn = build(spec, kind, args.n, x, w, wcache)
            except Exception as exc:  # noqa: BLE001 -- probe: report and continue
                print(f"{spec.name:12s} {kind:26s} ERROR {exc}")
                continue
            if fn is None:
                continue
            try:
                y = fn()
                err = float(((y.float() - ref).abs().max() / ref.abs().max()).item())
                t = timeit(fn, reps=args.reps)
            except Exception as exc:  # noqa: BLE001
                print(f"{spec.name:12s} {kind:26s} ERROR {exc}")
                continue
            row = {"layer": spec.name, "kind": kind, "ms": t * 1e3,
                   "tflops_direct_equiv": flops / t / 1e12, "err_vs_3xtf32": err}
            results.append(row)
            print(f"{spec.name:12s} {kind:26s} {t * 1e3:8.3f} ms {flops / t / 1e12:8.1f} TF/s "
                  f"err {err:.2e}", flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(results, fh, indent=1)


if __name__ == "__main__":
    main()
