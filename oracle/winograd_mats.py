"""Exact-rational Winograd F(e, r) transform matrices (TEST INFRASTRUCTURE).

This module is part of ``oracle/``: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline leg may import it, as the checker.  The
product (``paper_2012_15667_b200``) never does.

The reference leaves the transform matrices unspecified: they are edge
coefficients of the Winograd DAG, not vertices (``pkg/src/convio/dag.py:6-8``;
``SPEC.md:153``).  We therefore fix them here:

* F(2,3) and F(4,3) are Lavin & Gray's published matrices ("Fast Algorithms
  for Convolutional Neural Networks", 2016) -- the same ones the CUDA kernels
  hard-code (cross-checked through ``convio_winograd_matrices`` in the C-ABI).
* Any other F(e, r) comes from the Toom-Cook construction below with the
  interpolation points ``0, 1, -1, 2, -2, 1/2, -1/2, 3, -3, ...`` and infinity.

Toom-Cook by transposition: the linear convolution ``s = g * h`` of an
``r``-tap ``g`` and ``e``-tap ``h`` is ``s = C[(V_g g) . (V_h h)]`` with ``V_*``
evaluation matrices at ``m = e + r - 1`` points and ``C`` the interpolation
matrix.  The correlation ``y_i = sum_k d_{i+k} g_k`` (what the DAG computes,
``dag.py:358-401``) is the transpose of ``h -> g * h``, hence
``y = V_h^T [(V_g g) . (C^T d)]``: ``A^T = V_h^T``, ``G = V_g``, ``B^T = C^T``,
with each row of ``B^T`` rescaled to coprime integers (scale moved into ``G``).
"""

from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from math import gcd

F = Fraction

LAVIN = {
    (2, 3): {
        "AT": [[1, 1, 1, 0], [0, 1, -1, -1]],
        "G": [[1, 0, 0], [F(1, 2), F(1, 2), F(1, 2)], [F(1, 2), F(-1, 2), F(1, 2)], [0, 0, 1]],
        "BT": [[1, 0, -1, 0], [0, 1, 1, 0], [0, -1, 1, 0], [0, 1, 0, -1]],
    },
    (4, 3): {
        "AT": [[1, 1, 1, 1, 1, 0], [0, 1, -1, 2, -2, 0], [0, 1, 1, 4, 4, 0],
               [0, 1, -1, 8, -8, 1]],
        "G": [[F(1, 4), 0, 0], [F(-1, 6), F(-1, 6), F(-1, 6)], [F(-1, 6), F(1, 6), F(-1, 6)],
              [F(1, 24), F(1, 12), F(1, 6)], [F(1, 24), F(-1, 12), F(1, 6)], [0, 0, 1]],
        "BT": [[4, 0, -5, 0, 1, 0], [0, -4, -4, 1, 1, 0], [0, 4, -4, -1, 1, 0],
               [0, -2, -1, 2, 1, 0], [0, 2, -1, -2, 1, 0], [0, 4, 0, -5, 0, 1]],
    },
}


def _points(count: int) -> list[Fraction]:
    pts = [F(0)]
    k = 1
    while len(pts) < count:
        for cand in (F(k), F(-k), F(1, k + 1), F(-1, k + 1)):
            if cand not in pts and len(pts) < count:
                pts.append(cand)
        k += 1
    return pts[:count]


def _eval_matrix(points: list[Fraction], ncoef: int, with_inf: bool) -> list[list[Fraction]]:
    rows = [[p ** j for j in range(ncoef)] for p in points]
    if with_inf:
        rows.append([F(0)] * (ncoef - 1) + [F(1)])
    return rows


def _inverse(mat: list[list[Fraction]]) -> list[list[Fraction]]:
    n = len(mat)
    aug = [list(map(F, row)) + [F(int(i == j)) for j in range(n)] for i, row in enumerate(mat)]
    for col in range(n):
        piv = next(r for r in range(col, n) if aug[r][col] != 0)
        aug[col], aug[piv] = aug[piv], aug[col]
        pv = aug[col][col]
        aug[col] = [v / pv for v in aug[col]]
        for r in range(n):
            if r != col and aug[r][col] != 0:
                f = aug[r][col]
                aug[r] = [a - f * b for a, b in zip(aug[r], aug[col])]
    return [row[n:] for row in aug]


def _transpose(mat):
    return [list(col) for col in zip(*mat)]


def _lcm(a: int, b: int) -> int:
    return a * b // gcd(a, b)


@lru_cache(maxsize=None)
def toom_cook(e: int, r: int) -> dict:
    """General F(e, r) matrices from the construction in the module docstring."""
    m = e + r - 1
    pts = _points(m - 1)
    vs = _eval_matrix(pts, m, True)          # m x m
    vg = _eval_matrix(pts, r, True)          # m x r
    vh = _eval_matrix(pts, e, True)          # m x e
    bt = _transpose(_inverse(vs))            # C^T
    g = [list(row) for row in vg]
    for i, row in enumerate(bt):             # integer-normalise B^T rows
        den = 1
        for v in row:
            den = _lcm(den, v.denominator)
        ints = [int(v * den) for v in row]
        div = 0
        for v in ints:
            div = gcd(div, abs(v))
        scale = F(den, div or 1)
        bt[i] = [v * scale for v in row]
        g[i] = [v / scale for v in g[i]]
    return {"AT": _transpose(vh), "G": g, "BT": bt}


def matrices(e: int, r: int) -> dict:
    """``{"AT": e x m, "G": m x r, "BT": m x m}`` as exact Fractions."""
    src = LAVIN.get((e, r)) or toom_cook(e, r)
    return {k: [[F(v) for v in row] for row in mat] for k, mat in src.items()}


def matrices_float(e: int, r: int) -> dict:
    import numpy as np
    return {k: np.array([[float(v) for v in row] for row in mat], dtype=np.float64)
            for k, mat in matrices(e, r).items()}


def correlate_1d_exact(d, g, e: int, r: int) -> list[Fraction]:
    """``A^T [(G g) . (B^T d)]`` in exact arithmetic (for self-checks)."""
    mats = matrices(e, r)
    gg = [sum(F(a) * F(b) for a, b in zip(row, g)) for row in mats["G"]]
    dd = [sum(F(a) * F(b) for a, b in zip(row, d)) for row in mats["BT"]]
    prod = [a * b for a, b in zip(gg, dd)]
    return [sum(a * b for a, b in zip(row, prod)) for row in mats["AT"]]
