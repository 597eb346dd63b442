"""The FP32 direct-convolution kernels against conv values computed by the
REFERENCE's own DAG (``tests/golden/dag_golden.npz``, see test_dag_parity.py):
the library's default (generic) path and, for every golden case, NCHW and
channels-last layouts, through the C-ABI."""

import os

import numpy as np
import pytest
import torch

from oracle import conv_oracle as co
from paper_2012_15667_b200 import conv as C

from tolerances import tol_fp32

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "dag_golden.npz"))
CASES = sorted({k.split("_")[0] for k in G.files if k.startswith("direct")}, key=lambda s: int(s[6:]))


@pytest.mark.parametrize("layout", ["CHW", "HWC"])
@pytest.mark.parametrize("case", CASES)
def test_direct_kernel_matches_reference_dag_values(case, layout):
    x, w, y = G[f"{case}_x"], G[f"{case}_w"], G[f"{case}_y"]
    st = int(G[f"{case}_stride"])
    xt = torch.from_numpy(x).cuda()
    if layout != "CHW":
        xt = C.to_layout(xt, layout)
    out = C.conv_direct(xt, torch.from_numpy(w).cuda(), stride=st, padding=0)
    assert tuple(out.shape) == y.shape
    err = co.rel_err(out.contiguous().cpu().numpy(), y)
    assert err <= tol_fp32(w.shape[1], w.shape[2], w.shape[3]) / 10, err
