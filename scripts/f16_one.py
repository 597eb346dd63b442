import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2012_15667_b200 import TileConfig
from paper_2012_15667_b200 import conv as C
from paper_2012_15667_b200 import runner as R
name, z, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
spec = next(s for s in R.WORKLOADS["resnet50"] if s.name == name)
x = C.to_layout(torch.rand(256, spec.c, spec.hw, spec.hw, device="cuda") * 2 - 1, "HWC")
w = (torch.rand(spec.k, spec.c, 3, 3, device="cuda") * 2 - 1) / (spec.c * 9) ** 0.5
t = TileConfig(4, 4, z, 32768, 1, 1, 2, layout="HWC", e=4)
u = C.winograd_filter_transform_tc(w, 4, prec)
for _ in range(3):
    C.conv_winograd_tc(x, w, e=4, padding=1, tile=t, precision=prec, u=u)
torch.cuda.synchronize()
