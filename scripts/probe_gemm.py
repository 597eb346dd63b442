"""Raw GEMM efficiency of the tcgen05 kernels: a 1x1 convolution over a
128-wide image row is a plain GEMM whose A box is one contiguous 16 KB block,
so comparing it with the 3x3 layers separates kernel (MMA / pipeline)
efficiency from the implicit-GEMM tap-shifted loads; cuBLAS (torch.matmul)
on the same GEMM is the library reference point.

    python scripts/probe_gemm.py [--m 16384] [--n 1024] [--k 1024]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import TileConfig  # noqa: E402
from paper_2012_15667_b200 import conv as C  # noqa: E402
from scripts.probe_tc import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--k", type=int, default=1024)
    ap.add_argument("--one", default="", help="prec:z:nzt -- run one config twice (ncu target)")
    args = ap.parse_args()
    m, n, k = args.m, args.n, args.k
    h = m // 128
    x = C.to_layout(torch.rand(1, k, h, 128, device="cuda") * 2 - 1, "HWC")
    w = (torch.rand(n, k, 1, 1, device="cuda") * 2 - 1) / k ** 0.5
    flops = 2.0 * m * n * k
    out = C.empty_act(1, n, h, 128, "HWC", device="cuda")
    ws = torch.empty(2 * x.numel() + (1 << 20), dtype=torch.uint8, device="cuda")
    if args.one:
        prec, z, nzt = args.one.split(":")
        wp = C.pack_filter_igemm_bf16(w) if prec == "bf16" else C.pack_filter_igemm(w)
        tile = TileConfig(128, 1, int(z), 65536, 1, 1, int(nzt), layout="HWC")
        for _ in range(2):
            C.conv_igemm(x, w, padding=0, tile=tile, precision=prec, w_packed=wp, out=out, workspace=ws)
        torch.cuda.synchronize()
        return
    for prec in ("tf32", "bf16", "3xtf32", "3xf16"):
        wp = (C.pack_filter_igemm_bf16(w) if prec == "bf16" else C.pack_filter_igemm_f16x3(w) if prec == "3xf16"
              else C.pack_filter_igemm(w))
        for z, nzt in ((256, 2), (128, 2), (128, 1), (256, 1), (128, 4)):
            tile = TileConfig(128, 1, z, 65536, 1, 1, nzt, layout="HWC")
            try:
                t = timeit(lambda: C.conv_igemm(x, w, padding=0, tile=tile, precision=prec,
                                                w_packed=wp, out=out, workspace=ws), reps=20)
            except Exception as exc:  # noqa: BLE001
                print(f"{prec:7s} z={z} n_zt={nzt}: {exc}")
                continue
            mult = 3 if prec in ("3xtf32", "3xf16") else 1
            print(f"{prec:7s} z={z:3d} n_zt={nzt}: {t * 1e3:7.3f} ms {flops / t / 1e12:7.1f} TF/s "
                  f"(MMA rate {mult * flops / t / 1e12:7.1f})", flush=True)
    a = torch.rand(m, k, device="cuda")
    b = torch.rand(k, n, device="cuda")
    for name, dt, tf32 in (("cublas tf32", torch.float32, True), ("cublas bf16", torch.bfloat16, False),
                           ("cublas fp32", torch.float32, False)):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        aa, bb = a.to(dt), b.to(dt)
        t = timeit(lambda: aa @ bb, reps=20)
        print(f"{name}: {t * 1e3:7.3f} ms {flops / t / 1e12:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
