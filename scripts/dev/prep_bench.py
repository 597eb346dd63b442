"""Time a step's filter prep pieces: the batched 3xF16 pack of the implicit-GEMM
layers and the batched Winograd U transforms (3xTF32 / 3xF16), with their
algorithmic bytes.  Development tool; the contract numbers come from bench.py.

    python scripts/dev/prep_bench.py [--workload resnet50]
"""

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2012_15667_b200 import _native as N  # noqa: E402
from paper_2012_15667_b200 import conv as C  # noqa: E402
from paper_2012_15667_b200.runner import WORKLOADS, expand, make_weights  # noqa: E402


def t_us(fn, reps=50):
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
    wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "resnet50"
    dev = torch.device("cuda")
    specs = expand(WORKLOADS[wl])
    ws = [make_weights(s, dev, i) for i, s in enumerate(specs)]
    res = {}
    # every layer through the batched 3xF16 pack
    outs = [torch.empty(C.f16x3_slice_bytes(s.k, s.c, s.r, s.r), dtype=torch.uint8, device=dev) for s in specs]
    descs = (N.ConvDesc * len(specs))(*[N.make_desc(1, s.c, 8, 8, s.k, s.r, s.r, 1, 0, 2) for s in specs])
    wp = (ctypes.c_void_p * len(specs))(*[w.data_ptr() for w in ws])
    op = (ctypes.c_void_p * len(specs))(*[o.data_ptr() for o in outs])
    t = t_us(lambda: N.lib().convio_pack_filters_igemm_f16x3_batched(len(specs), descs, wp, op, None))
    nbytes = sum(w.numel() * 4 * 2 for w in ws)   # fp32 read + fp16 hi / lo written
    res["pack_f16x3_all_layers"] = {"us": round(t, 2), "GB/s": round(nbytes / t / 1e3, 1), "bytes": nbytes}
    # the stride-1 3x3 layers through the batched Winograd transform
    wsp = [(s, w) for s, w in zip(specs, ws) if s.stride == 1 and s.r == 3]
    for e in (2, 4):
        for prec in ("3xtf32", "3xf16"):
            us = [C.winograd_filter_transform_tc(w, e, prec) for _, w in wsp]
            d = (N.ConvDesc * len(wsp))(*[N.make_desc(1, s.c, 8, 8, s.k, 3, 3, 1, 0, 2) for s, _ in wsp])
            wq = (ctypes.c_void_p * len(wsp))(*[w.data_ptr() for _, w in wsp])
            uq = (ctypes.c_void_p * len(wsp))(*[u.data_ptr() for u in us])
            t = t_us(lambda: N.lib().convio_winograd_filter_transform_tc_batched(
                len(wsp), d, e, N.PRECISIONS[prec], wq, uq, None))
            m = e + 2
            nbytes = sum(w.numel() * 4 + s.k * s.c * m * m * 4 for s, w in wsp)
            res[f"winograd_u_e{e}_{prec}"] = {"us": round(t, 2), "GB/s": round(nbytes / t / 1e3, 1),
                                             "bytes": nbytes, "launches": C.last_launch_count()}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
