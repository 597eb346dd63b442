"""Pipeline trace of the CTA-pair implicit GEMM (dev tool; needs a -DCONVIO_TRACE
build: scripts/build_variant.sh trace -DCONVIO_TRACE).

    CONVIO_LIB=paper_2012_15667_b200/lib/variants/trace/libconvio_b200.so \
        python scripts/dev/pair_trace.py --layer res4_3x3 --tile 2,2,256,32768,1,1,2 --prec 3xf16

Stamps (clock64, leader CTA of cluster 0): producer may issue k-block i (P),
converter saw / finished it (C1 / C2), MMA issuer saw it converted / issued its
MMAs (M3 / M4), epilogue saw / drained accumulator t (E5 / E6)."""

import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2012_15667_b200 import TileConfig, _native as N, conv as C  # noqa: E402
from paper_2012_15667_b200.runner import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--layer", default="res4_3x3")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--tile", default="2,2,256,32768,1,1,2")
    ap.add_argument("--prec", default="3xf16")
    ap.add_argument("--show", type=int, default=24)
    args = ap.parse_args()
    spec = next(s for s in WORKLOADS[args.workload] if s.name == args.layer)
    t = [int(v) for v in args.tile.split(",")]
    tile = TileConfig(*t, layout="HWC")
    x = C.to_layout(torch.rand((args.n, spec.c, spec.hw, spec.hw), device="cuda") * 2 - 1, "HWC")
    w = (torch.rand((spec.k, spec.c, 3, 3), device="cuda") * 2 - 1) / (spec.c * 9) ** 0.5
    for _ in range(3):
        C.conv_igemm(x, w, padding=1, stride=spec.stride, tile=tile, precision=args.prec)
    torch.cuda.synchronize()
    C.conv_igemm(x, w, padding=1, stride=spec.stride, tile=tile, precision=args.prec)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (24 * 1024))()
    lib = N.lib()
    assert lib.convio_dev_trace(buf) == 0, "not a CONVIO_TRACE build"
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(24, 1024).astype(np.int64)
    fine = tr[18:24]
    st, en = tr[16], tr[17]
    ok = (st > 0) & (en > 0)
    if ok.any():
        t0g = st[ok].min()
        dur = (en[ok] - t0g) / 1e3
        print(f"per-CTA end (us after first start): min {dur.min():.1f} med {np.median(dur):.1f} max {dur.max():.1f}; "
              f"start spread {(st[ok].max() - t0g) / 1e3:.1f} us; CTAs {int(ok.sum())}")
    peer = tr[8:16]
    tr = tr[0:8]
    nz = [int((tr[r] > 0).sum()) for r in range(8)]
    print("stamps per row:", nz, "info:", C.query(tuple(x.shape), tuple(w.shape), spec.stride, 1, "HWC",
                                                   tile, f"igemm_{args.prec}")["reason"])
    t0 = min(tr[r][tr[r] > 0].min() for r in range(7) if nz[r])
    P, C1, C2, M3, M4, E5, E6, M7 = (tr[r] - t0 for r in range(8))
    pP, pC1, pC2 = (peer[r] - t0 for r in range(3))   # the peer CTA (clock64 of another SM: offset unknown)
    k = min(nz[0] or nz[3], nz[3], nz[4])   # (resident-filter tiles stamp no producer k-blocks)
    k1 = min(k, nz[1], nz[2]) if nz[1] else 0

    def med(a):
        return statistics.median(a) if len(a) else float("nan")
    if k1:
        print(f"converter: data-wait after issue (C1-P) med {med(C1[:k1] - P[:k1]):.0f} cyc, "
              f"convert (C2-C1) med {med(C2[:k1] - C1[:k1]):.0f}")
    f21, f22 = fine[3] - t0, fine[4] - t0   # converter warp 8, CTA 0: A data seen / tconv signalled
    if k1 and (fine[3] > 0).sum() and (fine[4] > 0).sum():
        kk = min(k1, int((fine[3] > 0).sum()), int((fine[4] > 0).sum()))
        print(f"converter fine (ARING): C2 -> signalled med {med(f22[:kk] - C2[:kk]):.0f}, "
              f"signalled -> next A data med {med(f21[1:kk] - f22[:kk - 1]):.0f}, "
              f"A data -> C1 (TMEM slot free) med {med(C1[1:kk] - f21[1:kk]):.0f}")
    gaps = [M3[i] - M4[i - 1] for i in range(1, k)]
    per = [M4[i] - M4[i - 1] for i in range(1, k)]
    print(f"MMA issuer: k-block period med {med(per):.0f} cyc, idle waiting for data med {med(gaps):.0f} "
          f"(sum {sum(gaps)} of {M4[k - 1] - M4[0]})")
    ns = next((i for i in range(1, k) if P[i] > M4[0]), None)
    print(f"ring: producer stalls (P[i] after M4[i-NS]) from k-block {ns}")
    ne = min(nz[5], nz[6])
    if ne and (fine[0] > 0).sum():
        f18, f19, f20 = (fine[i][:ne] - t0 for i in range(3))
        print(f"epilogue fine: tfull -> origin {med(f18 - E5[:ne]):.0f}, -> TMEM loads waited {med(f19 - f18):.0f}, "
              f"-> fold adds {med(f20 - f19):.0f}, -> unscaled {med(M7[:ne] - f20):.0f}")
    if ne and nz[7]:
        print(f"epilogue: tfull -> chunk 0 in registers med {med(M7[:ne] - E5[:ne]):.0f}, "
              f"-> staged (resident-filter builds) med {med(P[:ne] - E5[:ne]) if not nz[0] or nz[0] == ne else float('nan'):.0f}, "
              f"-> accumulator released med {med(E6[:ne] - E5[:ne]):.0f}")
    if ne:
        print(f"epilogue: drain (E6-E5) med {med(E6[:ne] - E5[:ne]):.0f} cyc, items {ne}, "
              f"item period med {med(np.diff(E5[:ne])):.0f}")
    print(" i      P     C1     C2     M3  M7(1st MMA)  M4 | peer P  C1  C2 (own clock)")
    for i in range(min(args.show, k)):
        print(f"{i:3d} {P[i]:7d} {C1[i] if k1 else 0:7d} {C2[i] if k1 else 0:7d} {M3[i]:7d} {M7[i]:7d} {M4[i]:7d} | "
              f"{pP[i]:7d} {pC1[i]:7d} {pC2[i]:7d}")


if __name__ == "__main__":
    main()
