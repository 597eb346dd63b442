"""The CPU oracle itself: transforms exact, numpy == C == float64 torch.

Conv values have no reference golden vector (the reference never computes a
convolution), so the oracle is pinned by independent cross-checks here.
"""

import random
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import conv_oracle as co
from oracle import winograd_mats as wm


@pytest.mark.parametrize("e,r", [(2, 3), (4, 3), (3, 3), (6, 3), (2, 5), (2, 2), (1, 3), (3, 2)])
def test_transforms_compute_the_correlation_exactly(e, r):
    rnd = random.Random(e * 10 + r)
    for _ in range(6):
        d = [Fraction(rnd.randint(-9, 9), rnd.randint(1, 4)) for _ in range(e + r - 1)]
        g = [Fraction(rnd.randint(-9, 9)) for _ in range(r)]
        want = [sum(d[i + k] * g[k] for k in range(r)) for i in range(e)]
        assert wm.correlate_1d_exact(d, g, e, r) == want


def test_lavin_matrices_and_toom_cook_agree_functionally():
    for e in (2, 4):
        tc = wm.toom_cook(e, 3)
        lv = wm.matrices(e, 3)
        assert len(tc["BT"]) == len(lv["BT"]) == e + 2
        d = [Fraction(v) for v in range(1, e + 3)]
        g = [Fraction(3), Fraction(-1), Fraction(2)]
        # both define the same linear map d, g -> y
        y_tc = [sum(a * b for a, b in zip(row, [x * y for x, y in zip(
            [sum(p * q for p, q in zip(gr, g)) for gr in tc["G"]],
            [sum(p * q for p, q in zip(br, d)) for br in tc["BT"]])])) for row in tc["AT"]]
        assert y_tc == wm.correlate_1d_exact(d, g, e, 3)


def _rand(n, c, h, w, k, r, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32)
    wt = (rng.uniform(-1, 1, (k, c, r, r)) / np.sqrt(c * r * r)).astype(np.float32)
    return x, wt


@pytest.mark.parametrize("stride,pad,r", [(1, 1, 3), (2, 1, 3), (1, 0, 3), (2, 2, 5), (1, 0, 1), (4, 0, 11)])
def test_direct_oracle_matches_torch_float64(stride, pad, r):
    x, wt = _rand(2, 4, 23, 19, 5, r)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(wt).double(),
                                     stride=stride, padding=pad).numpy()
    y = co.direct_conv(x, wt, stride, pad)
    assert y.shape == ref.shape
    assert co.rel_err(y, ref) < 1e-13


@pytest.mark.parametrize("e", [2, 4, 3, 6])
def test_winograd_oracle_matches_direct(e):
    x, wt = _rand(2, 6, 13, 17, 4, 3, seed=e)   # ragged outputs: padded domain + crop
    ref = co.direct_conv(x, wt, 1, 1)
    assert co.rel_err(co.winograd_conv(x, wt, e, 1), ref) < 1e-12


def test_c_oracle_matches_numpy_oracle():
    co.load_c_oracle()
    for stride, pad in ((1, 1), (2, 1), (1, 0)):
        x, wt = _rand(2, 5, 12, 14, 6, 3, seed=stride + pad)
        assert co.rel_err(co.c_direct_conv(x, wt, stride, pad), co.direct_conv(x, wt, stride, pad)) == 0.0
    x, wt = _rand(1, 3, 10, 10, 4, 3)
    for e in (2, 4):
        assert co.rel_err(co.c_winograd_conv(x, wt, e, 1), co.direct_conv(x, wt, 1, 1)) < 1e-12


def test_c_oracle_bounded_sample_and_threads_do_not_change_values():
    x, wt = _rand(3, 4, 9, 9, 5, 3)
    full = co.c_direct_conv(x, wt, 1, 1, threads=1)
    many = co.c_direct_conv(x, wt, 1, 1, threads=4)
    assert np.array_equal(full, many)
    part = co.c_direct_conv(x, wt, 1, 1, images=1)
    assert np.array_equal(part[0], full[0]) and not part[1:].any()


def test_empty_channel_and_single_pixel_edges():
    x, wt = _rand(1, 1, 1, 1, 1, 1)
    assert co.direct_conv(x, wt).shape == (1, 1, 1, 1)
    assert co.direct_conv(x, wt)[0, 0, 0, 0] == pytest.approx(float(x[0, 0, 0, 0]) * float(wt[0, 0, 0, 0]))
    x, wt = _rand(1, 2, 3, 3, 2, 3)
    y = co.direct_conv(x, wt, 1, 0)
    assert y.shape == (1, 2, 1, 1)
