"""3xF16 Winograd parity + timing check (development probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import conv_oracle as co
from paper_2012_15667_b200 import TileConfig
from paper_2012_15667_b200 import conv as C
from scripts.probe_tc import timeit

for (n, c, h, k, e, z) in [(2, 64, 28, 64, 4, 64), (3, 128, 14, 256, 4, 256), (2, 256, 7, 128, 2, 128),
                           (2, 512, 7, 512, 4, 256), (4, 128, 28, 128, 4, 128)]:
    g = np.random.default_rng(0)
    x = g.uniform(-1, 1, (n, c, h, h)).astype(np.float32)
    w = (g.uniform(-1, 1, (k, c, 3, 3)) / np.sqrt(c * 9)).astype(np.float32)
    b = np.linspace(-0.25, 0.25, k).astype(np.float32)
    xd = C.to_layout(torch.from_numpy(x).cuda(), "HWC")
    ref = co.direct_conv(x, w, 1, 1) + b[None, :, None, None]
    for prec in ("3xtf32", "3xf16"):
        t = TileConfig(e, e, z, 32768, 1, 1, 2, layout="HWC", e=e)
        try:
            y = C.conv_winograd_tc(xd, torch.from_numpy(w).cuda(), e=e, padding=1, tile=t, precision=prec,
                                   bias=torch.from_numpy(b).cuda())
            err = co.rel_err(y.contiguous().cpu().numpy(), ref)
            print(n, c, h, k, e, z, prec, f"err {err:.3e}", flush=True)
        except Exception as ex:  # noqa: BLE001
            print(n, c, h, k, e, z, prec, "ERROR", str(ex)[:200], flush=True)

from paper_2012_15667_b200 import runner as R
for name, z in (("res3_3x3", 128), ("res4_3x3", 256), ("res5_3x3", 256), ("res2_3x3", 64)):
    spec = next(s for s in R.WORKLOADS["resnet50"] if s.name == name)
    x = C.to_layout(torch.rand(256, spec.c, spec.hw, spec.hw, device="cuda") * 2 - 1, "HWC")
    w = (torch.rand(spec.k, spec.c, 3, 3, device="cuda") * 2 - 1) / (spec.c * 9) ** 0.5
    out = C.empty_act(256, spec.k, spec.out_hw, spec.out_hw, "HWC", device="cuda")
    for prec, nzt in (("3xtf32", 2), ("3xf16", 2)):
        t = TileConfig(4, 4, z, 32768, 1, 1, nzt, layout="HWC", e=4)
        u = C.winograd_filter_transform_tc(w, 4, prec)
        info = C.query(tuple(x.shape), tuple(w.shape), 1, 1, "HWC", t, f"winograd_tc_{prec}")
        ws = torch.empty(info["workspace_bytes"], dtype=torch.uint8, device="cuda")
        tt = timeit(lambda: C.conv_winograd_tc(x, w, e=4, padding=1, tile=t, precision=prec, u=u, out=out,
                                               workspace=ws), reps=10)
        print(name, prec, f"{tt * 1e3:.3f} ms", flush=True)
