"""Lower-bound auto-tuning of every layer of a workload on the device.

    python scripts/tune_layers.py --workload resnet50 --n 64 --budget 128 \
        [--exhaustive-cap 0] [--out paper_2012_15667_b200/tuned/b200_resnet50.json]

Per distinct layer and per algorithm (direct, Winograd F(2,3), F(4,3)):
  1. the Table-1 searching domain of the B200 machine model (reference
     ``build_space``) restricted to its legal device projection;
  2. the model's analytic tile (``optimal_tile_dc/wa``) and its device time
     if it has a projection;
  3. the reference tuner (``tune``: GBR cost model + random walks) with
     ``backend="device"``;
  4. optionally the exhaustive oracle over the legal projection
     (``--exhaustive-cap``), for the pruned-vs-exhaustive comparison.
The fastest (algorithm, tile) per layer is written as the layer's plan.
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

import torch  # noqa: E402

from paper_2012_15667_b200 import device_tuner as DT  # noqa: E402
from paper_2012_15667_b200.autotune import tune, exhaustive_oracle, random_search  # noqa: E402
from paper_2012_15667_b200.dataflow import optimal_tile_dc, optimal_tile_wa, InfeasibleTileError  # noqa: E402
from paper_2012_15667_b200.device import b200_hw_model, shape_of  # noqa: E402
from paper_2012_15667_b200.model import WinogradParams  # noqa: E402
from paper_2012_15667_b200.runner import (WORKLOADS, TUNED_DIR, FP32_ALGORITHMS,  # noqa: E402
                                           candidate_algorithm)


def tune_one(shape, hw, alg, wp, budget, seed, exhaustive_cap, log):
    t0 = time.time()
    try:
        space = DT.device_space(shape, hw, alg, wp)
    except InfeasibleTileError as exc:
        return {"error": str(exc)}
    out = {"legal_space": space.size, "unconstrained": space.unconstrained_size}
    # the model's analytic pick
    try:
        mt = optimal_tile_dc(shape, hw) if alg == "direct" else optimal_tile_wa(shape, wp, hw)
        mcost = DT.measure_device(mt, shape, hw, alg, wp)
        out["model_tile"] = {"tile": mt.to_dict(), "seconds": None if math.isinf(mcost) else mcost}
    except InfeasibleTileError as exc:
        out["model_tile"] = {"error": str(exc)}
    n_s = min(16, max(2, budget // 4))
    sess = tune(shape, hw, alg, min(budget, space.size), seed, winograd=wp, n_s=min(n_s, space.size),
                space=space, backend="device")
    best = sess.best
    out["tuner"] = {"best": best.config.to_dict() if best else None,
                    "seconds": best.cost if best else None,
                    "measurements": len(sess.measurements), "iterations": sess.iterations,
                    "stopped_by": sess.stopped_by,
                    "measurements_to_best": (best.index + 1) if best else None,
                    "wall_s": round(time.time() - t0, 1)}
    rs_cfg, rs_cost = random_search(space, min(budget, space.size), seed, backend="device")
    out["random_search"] = {"best": rs_cfg.to_dict() if rs_cfg else None,
                            "seconds": None if math.isinf(rs_cost) else rs_cost}
    if exhaustive_cap and space.size <= exhaustive_cap:
        t1 = time.time()
        ex_cfg, ex_cost = exhaustive_oracle(space, cap=exhaustive_cap, backend="device")
        out["exhaustive"] = {"best": ex_cfg.to_dict() if ex_cfg else None,
                             "seconds": None if math.isinf(ex_cost) else ex_cost,
                             "wall_s": round(time.time() - t1, 1)}
    log(f"    {alg}{'' if wp is None else wp.e}: legal {space.size}, tuner best "
        f"{out['tuner']['seconds']} in {out['tuner']['measurements']} meas "
        f"({out['tuner']['wall_s']} s), random {out['random_search']['seconds']}"
        + (f", exhaustive {out['exhaustive']['seconds']}" if "exhaustive" in out else ""))
    return out


def tune_direct_nhwc(shape, spec, log):
    """Channels-last FFMA direct kernel (stacked pixels): exhaustive device
    search over its own space (x | Q, y | P, 32 <= x*y <= 128, z in {64, 128},
    s_b in {16384, 32768}), threads = library layout (1, 1, 1).  Like the
    tensor-core kernels it lies outside Table 1 (z^2 R <= s_b assumes the
    paper's x*y ~ R*z block shape; this block is 128 stacked pixels x z)."""
    import math as _m
    from paper_2012_15667_b200.dataflow import TileConfig
    from paper_2012_15667_b200 import conv as C
    small_c = spec.c <= 4 and spec.r == 3 and spec.k % 32 == 0   # K8 (direct_smallc.cu)
    if (spec.c % 32 and not small_c) or spec.stride > 2:
        return {"error": "needs C % 32 == 0 (or C <= 4) and stride <= 2"}
    q, p = shape.w_out, shape.h_out
    x = torch.empty((shape.n, spec.c, spec.hw, spec.hw), device="cuda").uniform_(-1, 1)
    xh = C.to_layout(x, "HWC")
    w = torch.empty((spec.k, spec.c, spec.r, spec.r), device="cuda").uniform_(-1, 1) / (spec.c * 9) ** 0.5
    wp = C.pack_filter_direct(w)
    out = C.empty_act(shape.n, spec.k, p, q, "HWC", device="cuda")
    best, best_t, tried = None, _m.inf, 0
    if small_c:   # one tile shape: 16 x 16 pixels x 32 channels, the whole C staged
        tile = TileConfig(16, 16, 32, 32768, 1, 1, 1, layout="HWC")
        try:
            best_t = DT.device_time(lambda: C.conv_direct(xh, w, stride=spec.stride, padding=spec.pad,
                                                           tile=tile, w_packed=wp, out=out))
            best, tried = tile, 1
        except Exception:  # noqa: BLE001 -- illegal projection
            pass
    for bx in [d for d in range(1, q + 1) if q % d == 0 and not small_c]:
        for by in [d for d in range(1, p + 1) if p % d == 0]:
            if not DT._block_ok(bx, by, shape.n):
                continue
            for z in [z for z in (64, 128) if spec.k % z == 0]:
                for sb in (16384, 32768):
                    tile = TileConfig(bx, by, z, sb, 1, 1, 1, layout="HWC")
                    try:
                        t = DT.device_time(lambda: C.conv_direct(xh, w, stride=spec.stride,
                                                                  padding=spec.pad, tile=tile,
                                                                  w_packed=wp, out=out))
                    except Exception:  # noqa: BLE001 -- illegal projection
                        continue
                    tried += 1
                    if t < best_t:
                        best, best_t = tile, t
    log(f"    direct_nhwc: {tried} tiles, best {best} {best_t}")
    return {"tuner": {"best": best.to_dict() if best else None,
                      "seconds": best_t if best else None, "measurements": tried},
            "space": "exhaustive channels-last FFMA projection"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--budget", type=int, default=128)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--exhaustive-cap", type=int, default=0)
    ap.add_argument("--algs", default="direct,direct_nhwc,winograd2,winograd4,igemm_3xtf32,igemm_tf32,"
                    "igemm_bf16,igemm_3xf16,winograd_tc_3xtf32_e2,winograd_tc_3xtf32_e4,"
                    "winograd_tc_tf32_e4,winograd_tc_bf16_e4,winograd_nhwc_e2,winograd_nhwc_e4,"
                    "winograd_tc_3xf16_e4")
    ap.add_argument("--layers", default="")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    warnings.simplefilter("ignore")
    torch.cuda.init()
    hw = b200_hw_model()
    full_batch = {"resnet50": 256, "vgg16": 32, "single": 1}.get(args.workload)
    out_path = args.out or os.path.join(
        TUNED_DIR, f"b200_{args.workload}.json" if args.n == full_batch
        else f"b200_{args.workload}_n{args.n}.json")
    result = {"workload": args.workload, "n_tune": args.n, "budget": args.budget,
              "hw_model": {"s": hw.s, "s_sm": hw.s_sm, "n_p": hw.n_p},
              "device": torch.cuda.get_device_name(), "layers": {}}
    if os.path.exists(out_path):
        with open(out_path) as fh:
            prev = json.load(fh)
        if prev.get("n_tune") == args.n:
            result["layers"].update(prev.get("layers", {}))

    def log(msg):
        print(msg, flush=True)

    wanted = set(args.layers.split(",")) if args.layers else None
    for spec in WORKLOADS[args.workload]:
        if wanted and spec.name not in wanted:
            continue
        DT.set_padding(spec.pad)
        shape = shape_of(args.n, spec.c, spec.hw, spec.hw, spec.k, spec.r, spec.stride, spec.pad)
        log(f"{spec.name}: {shape}")
        cands = dict(result["layers"].get(spec.name, {}).get("candidates", {}))
        for alg in args.algs.split(","):
            if alg == "direct":
                cands["direct"] = tune_one(shape, hw, "direct", None, args.budget, args.seed,
                                           args.exhaustive_cap, log)
            elif alg == "direct_nhwc":
                cands[alg] = tune_direct_nhwc(shape, spec, log)
            elif alg.startswith("igemm") or alg.startswith("winograd_tc_"):
                # the tensor-core engines: the reference tuner over the I/O-pruned tcgen05
                # domain (device_tuner.tune_layer; budget >= domain size = its optimum)
                if alg.startswith("igemm") or (spec.stride == 1 and spec.r == 3):
                    cands.update(DT.tune_layer(spec, args.n, [alg], budget=args.budget, seed=args.seed,
                                               log=log))
            elif alg.startswith("winograd_nhwc_e"):
                if spec.stride == 1 and spec.r == 3:
                    got = DT.tune_layer(spec, args.n, [f"winograd_tc_fp32_e{alg[-1]}"], budget=args.budget,
                                        seed=args.seed, log=log)
                    if got:
                        cands[alg] = next(iter(got.values()))
            elif alg.startswith("winograd") and spec.stride == 1 and spec.r == 3:
                e = int(alg[len("winograd"):])
                cands[alg] = tune_one(shape, hw, "winograd", WinogradParams(e, 3), args.budget,
                                      args.seed, args.exhaustive_cap, log)
        best_key, best_t = None, math.inf
        for key, c in cands.items():
            t = (c.get("tuner") or {}).get("seconds")
            alg_k, _ = candidate_algorithm(key)
            if alg_k not in FP32_ALGORITHMS:   # reduced precision: never the layer's FP32 plan
                continue
            if t is not None and t < best_t:
                best_key, best_t = key, t
        if best_key is None:
            log(f"  no legal plan for {spec.name}")
            continue
        tile = cands[best_key]["tuner"]["best"]
        flops = spec.flops(args.n)
        best_alg, best_e = candidate_algorithm(best_key)
        result["layers"][spec.name] = {
            "algorithm": best_alg, "e": best_e,
            "tile": tile, "seconds": best_t, "gflops_direct_equiv": round(flops / best_t / 1e9, 1),
            "candidates": cands,
        }
        log(f"  -> {best_key} {tile} {best_t * 1e3:.3f} ms {flops / best_t / 1e12:.2f} TFLOP/s")
        os.makedirs(os.path.dirname(out_path), exist_ok=True)
        with open(out_path, "w") as fh:
            json.dump(result, fh, indent=1, sort_keys=True)
    print(f"wrote {out_path}")


if __name__ == "__main__":
    main()
