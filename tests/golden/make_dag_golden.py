"""Generate ``dag_golden.npz``: convolution VALUES computed by the REFERENCE's
own DAGs (test infrastructure; build container only -- ``/root/reference``
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_dag_golden.py

The reference never computes a convolution, but its direct-convolution DAG
(``pkg/src/convio/dag.py:247-285``) fixes every arithmetic step: INPUT
vertices in ``img[b,c,y,x]`` then ``wt[oc,c,ky,kx]`` order, one 2-input
product vertex per window term, one left-deep 2-input sum per output in
``(c, ky, kx)`` order, OUTPUT vertices in ``(b, oc, oy, ox)`` order.  This
script evaluates that DAG vertex by vertex in float64 on seeded inputs
(fp32-representable, so every product is exact) and stores inputs + outputs.

For Winograd the reference DAG carries no transform coefficients
(``dag.py:6-8``), so its values are undefined; what it does fix is which
input pixels form each tile's patch (``dag.py:358-363``).  The script records,
for every step-1 input-transform tree, the ``(b, c, y, x)`` of its leaves, so
the oracle's tiling can be checked against it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from convio.dag import INPUT, OUTPUT, build_direct_conv_dag, build_winograd_dag  # noqa: E402
from convio.model import ConvShape, WinogradParams  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dag_golden.npz")

# (w_out, h_out, c_out, c_in, w_ker, h_ker, stride, n): strides 1/2/3, 1x1 / 3x3 / 5x5 /
# non-square kernels, batch > 1, ragged maps
DIRECT_SHAPES = [
    (4, 4, 3, 2, 3, 3, 1, 1),
    (5, 3, 2, 3, 3, 3, 1, 2),
    (3, 3, 4, 2, 3, 3, 2, 1),
    (4, 4, 2, 5, 1, 1, 1, 1),
    (3, 2, 3, 3, 1, 1, 2, 2),
    (2, 2, 2, 2, 5, 5, 1, 1),
    (2, 3, 2, 2, 5, 5, 2, 1),
    (3, 3, 2, 2, 3, 2, 1, 1),
    (6, 6, 2, 1, 3, 3, 1, 1),
    (2, 2, 3, 4, 3, 3, 3, 1),
    (7, 7, 2, 2, 3, 3, 1, 1),
]
# (w_out, h_out, c_out, c_in, e, r, n)
WINOGRAD_SHAPES = [
    (4, 4, 1, 2, 2, 3, 1),
    (4, 2, 2, 1, 2, 3, 2),
    (4, 4, 1, 1, 4, 3, 1),
]


def eval_direct(shape, seed):
    dag = build_direct_conv_dag(shape)
    g = np.random.default_rng(seed)
    n_img = shape.n * shape.c_in * shape.h_in * shape.w_in
    n_wt = shape.c_out * shape.c_in * shape.h_ker * shape.w_ker
    inputs = dag.input_vertices()
    assert inputs == list(range(n_img + n_wt))
    vals = np.zeros(dag.n_vertices, dtype=np.float64)
    x = g.uniform(-1, 1, n_img).astype(np.float32)
    w = g.uniform(-1, 1, n_wt).astype(np.float32)
    vals[:n_img] = x
    vals[n_img:n_img + n_wt] = w
    preds = dag.predecessors()
    for v in range(n_img + n_wt, dag.n_vertices):     # construction order is topological
        a, b = preds[v]
        vals[v] = vals[a] * vals[b] if dag.steps[v] == 1 else vals[a] + vals[b]
    y = vals[dag.output_vertices()]
    return (x.reshape(shape.n, shape.c_in, shape.h_in, shape.w_in),
            w.reshape(shape.c_out, shape.c_in, shape.h_ker, shape.w_ker),
            y.reshape(shape.n, shape.c_out, shape.h_out, shape.w_out))


def winograd_patches(shape, p):
    """(b, c, y, x) of the leaves of every step-1 input-transform tree, in tree order."""
    dag = build_winograd_dag(shape, p)
    n_img = shape.n * shape.c_in * shape.h_in * shape.w_in
    coords = np.array(np.unravel_index(np.arange(n_img), (shape.n, shape.c_in, shape.h_in, shape.w_in))).T
    preds = dag.predecessors()
    m2 = p.m * p.m
    trees = []
    for v in range(dag.n_vertices):
        # the scaling vertices of an input-transform tree read an image INPUT vertex
        if dag.steps[v] == 1 and len(preds[v]) == 1 and preds[v][0] < n_img:
            trees.append(preds[v][0])
    leaves = np.array(trees).reshape(-1, m2)          # consecutive m^2 leaves per tree
    return coords[leaves]                             # [trees, m^2, 4]


def main() -> None:
    out = {}
    for i, (wo, ho, co, ci, wk, hk, st, n) in enumerate(DIRECT_SHAPES):
        shape = ConvShape.from_output(wo, ho, co, ci, wk, hk, stride=st, n=n)
        x, w, y = eval_direct(shape, 100 + i)
        out[f"direct{i}_x"], out[f"direct{i}_w"], out[f"direct{i}_y"] = x, w, y
        out[f"direct{i}_stride"] = np.array(st)
    for i, (wo, ho, co, ci, e, r, n) in enumerate(WINOGRAD_SHAPES):
        shape = ConvShape.from_output(wo, ho, co, ci, r, r, n=n)
        out[f"wino{i}_patches"] = winograd_patches(shape, WinogradParams(e, r))
        out[f"wino{i}_shape"] = np.array([wo, ho, co, ci, e, r, n])
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(DIRECT_SHAPES)} direct DAG evaluations, "
          f"{len(WINOGRAD_SHAPES)} Winograd patch maps")


if __name__ == "__main__":
    main()
