"""Quick device probe: FFMA peak, a few direct / Winograd tiles vs cuDNN.

    python scripts/probe.py [--n 32]

Prints one line per configuration (CUDA-event timing, median of 20 after 5
warm-ups).  Development tool; the contract numbers come from bench.py.
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import TileConfig  # noqa: E402
from paper_2012_15667_b200 import conv as C  # noqa: E402
from paper_2012_15667_b200 import _native as N  # noqa: E402


def timeit(fn, reps=20, warm=5):
    """Mean device time of back-to-back launches (host overhead overlapped)."""
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


def ffma_peak():
    import ctypes
    sink = torch.zeros(148 * 64, device="cuda")
    flops = ctypes.c_int64()
    blocks = 148 * 8
    iters = 2000

    def run():
        N.check(N.lib().convio_ffma_peak(ctypes.c_void_p(sink.data_ptr()), blocks, iters,
                                         ctypes.byref(flops),
                                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    t = timeit(run, reps=10, warm=3)
    return flops.value / t / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--only-tc", action="store_true", help="skip the FFMA / Winograd searches")
    args = ap.parse_args()
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    print(f"ffma peak probe: {ffma_peak():.1f} TFLOP/s", flush=True)
    layers = [
        ("c2", 64, 56, 64, 1),
        ("c3", 128, 28, 128, 1),
        ("c4", 256, 14, 256, 1),
        ("c5", 512, 7, 512, 1),
    ]
    n = args.n
    for name, c, hw, k, st in layers:
        if args.only_tc and c % 32:
            continue
        x = torch.randn(n, c, hw, hw, device="cuda")
        w = torch.randn(k, c, 3, 3, device="cuda") / (c * 9) ** 0.5
        flops = 2.0 * n * k * c * 9 * hw * hw
        t = timeit(lambda: torch.nn.functional.conv2d(x, w, padding=1))
        print(f"{name} cudnn fp32: {t*1e3:.3f} ms {flops/t/1e12:.2f} TFLOP/s", flush=True)
        wp = C.pack_filter_direct(w)
        cands = []
        if args.only_tc:
            cands = None
        for TX in (8, 7, 4):
            for TZ in (8, 16, 4):
                for TY in ((1, 2) if not args.only_tc else ()):
                    for nzt in (4, 8, 16):
                        z = TZ * nzt
                        if k % z:
                            continue
                        for nxt in (1, 2, 4, 7, 8, 14):
                            x_ = TX * nxt
                            if hw % x_:
                                continue
                            for nyt in (1, 2, 4, 7, 8):
                                y_ = TY * nyt
                                if hw % y_:
                                    continue
                                thr = nxt * nyt * nzt
                                if thr < 64 or thr > 512:
                                    continue
                                for sb in (16384, 32768):
                                    cands.append(TileConfig(x_, y_, z, sb, nxt, nyt, nzt))
        best = None
        t0 = time.time()
        for tile in (cands or []):
            info = C.query(x.shape, w.shape, 1, 1, "CHW", tile)
            if info["rc"] != 0:
                continue
            try:
                t = timeit(lambda: C.conv_direct(x, w, padding=1, tile=tile, w_packed=wp), reps=5, warm=2)
            except Exception as exc:  # noqa: BLE001
                print("  fail", tile, exc)
                continue
            if best is None or t < best[0]:
                best = (t, tile, info)
            if time.time() - t0 > 60:
                break
        if best is None:
            best = (float("nan"), None, {"regs_per_thread": 0, "smem_bytes": 0, "channel_chunk": 0})
        t, tile, info = best
        print(f"{name} direct best: {t*1e3:.3f} ms {flops/t/1e12:.2f} TFLOP/s  {tile} "
              f"regs={info['regs_per_thread']} smem={info['smem_bytes']} ck={info['channel_chunk']}",
              flush=True)
        if c % 32 == 0:
            xh = C.to_layout(x, "HWC")
            wq = C.pack_filter_igemm(w)
            for bx, by in ((28, 4), (14, 8), (hw, min(hw, 128 // hw)), (7, 7)):
                for bn in (64, 128, 256):
                    if k % bn or hw % bx or hw % by or bx * by > 128:
                        continue
                    for sb in (16384, 32768):
                        for split in (False, True):
                            tile = TileConfig(bx, by, bn, sb, 1, 1, 1, layout="HWC")
                            try:
                                t = timeit(lambda: C.conv_igemm_tf32(xh, w, padding=1, tile=tile,
                                                                      w_packed=wq, split=split))
                                info = C.query(xh.shape, w.shape, 1, 1, "HWC", tile,
                                               "igemm_3xtf32" if split else "igemm_tf32")
                                print(f"{name} tcgen05 {'3xtf32' if split else 'tf32'} {bx}x{by}x{bn} "
                                      f"sb={sb}: {t*1e3:.3f} ms {flops/t/1e12:.2f} TFLOP/s "
                                      f"[{info['reason']}]", flush=True)
                            except Exception as exc:  # noqa: BLE001
                                print(f"{name} tcgen05 {bx}x{by}x{bn}: {exc}", flush=True)
        for e in ((2, 4) if not args.only_tc else ()):
            try:
                u = C.winograd_filter_transform(w, e)
                t = timeit(lambda: C.conv_winograd(x, w, e=e, padding=1, u=u))
                print(f"{name} winograd F({e},3) default: {t*1e3:.3f} ms eff {flops/t/1e12:.2f} TFLOP/s",
                      flush=True)
            except Exception as exc:  # noqa: BLE001
                print(f"{name} winograd F({e},3): {exc}")


if __name__ == "__main__":
    main()
