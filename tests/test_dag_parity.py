"""Conv-value parity pinned to the REFERENCE's own code (not to torch).

``tests/golden/dag_golden.npz`` holds outputs computed by evaluating the
reference's ``build_direct_conv_dag`` (``pkg/src/convio/dag.py:247-285``)
vertex by vertex (``tests/golden/make_dag_golden.py``).  The float64 oracle
(numpy and C) must reproduce them bit for bit -- same products, same
left-deep ``(c, ky, kx)`` sums -- and the oracle's Winograd tiling must read
exactly the patch leaves of the reference's ``build_winograd_dag``
(``dag.py:358-363``).  This package's own DAG builders must produce the
reference's graphs (same vertex numbering) and the same values.  The GPU
kernels are held to the same golden values in ``test_dag_parity_gpu``.
"""

import os

import numpy as np
import pytest

from oracle import conv_oracle as co
from paper_2012_15667_b200.dag import build_direct_conv_dag, build_winograd_dag
from paper_2012_15667_b200.model import ConvShape, WinogradParams

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "dag_golden.npz")
G = np.load(GOLDEN)
DIRECT = sorted({k.split("_")[0] for k in G.files if k.startswith("direct")}, key=lambda s: int(s[6:]))
WINO = sorted({k.split("_")[0] for k in G.files if k.startswith("wino")}, key=lambda s: int(s[4:]))


@pytest.mark.parametrize("case", DIRECT)
def test_numpy_oracle_reproduces_reference_dag_bit_for_bit(case):
    x, w, y = G[f"{case}_x"], G[f"{case}_w"], G[f"{case}_y"]
    out = co.direct_conv(x, w, int(G[f"{case}_stride"]), 0)
    assert out.shape == y.shape
    assert np.array_equal(out, y)


@pytest.mark.parametrize("case", DIRECT)
def test_c_oracle_reproduces_reference_dag_bit_for_bit(case):
    x, w, y = G[f"{case}_x"], G[f"{case}_w"], G[f"{case}_y"]
    out = co.c_direct_conv(x, w, int(G[f"{case}_stride"]), 0)
    assert np.array_equal(out, y)


@pytest.mark.parametrize("case", DIRECT)
def test_package_dag_evaluates_to_the_reference_values(case):
    """This package's build_direct_conv_dag, evaluated the same way, gives the same
    values: the graphs have the same vertices, edges and order."""
    x, w, y = G[f"{case}_x"], G[f"{case}_w"], G[f"{case}_y"]
    n, c, hi, wi = x.shape
    k, _, kh, kw = w.shape
    st = int(G[f"{case}_stride"])
    shape = ConvShape.from_output(y.shape[3], y.shape[2], k, c, kw, kh, stride=st, n=n)
    assert (shape.h_in, shape.w_in) == (hi, wi)
    dag = build_direct_conv_dag(shape)
    vals = np.zeros(dag.n_vertices)
    vals[:x.size] = x.ravel()
    vals[x.size:x.size + w.size] = w.ravel()
    pred = dag.predecessors()
    for v in range(x.size + w.size, dag.n_vertices):
        a, b = pred[v]
        vals[v] = vals[a] * vals[b] if dag.steps[v] == 1 else vals[a] + vals[b]
    assert np.array_equal(vals[dag.output_vertices()].reshape(y.shape), y)


@pytest.mark.parametrize("case", WINO)
def test_oracle_winograd_tiling_is_the_reference_patch_map(case):
    wo, ho, co_, ci, e, r, n = (int(v) for v in G[f"{case}_shape"])
    leaves = G[f"{case}_patches"]                    # [trees, m^2, (b, c, y, x)]
    shape = ConvShape.from_output(wo, ho, co_, ci, r, r, n=n)
    m = e + r - 1
    # an index image: the oracle's patches then carry each pixel's coordinates
    ids = np.arange(n * ci * shape.h_in * shape.w_in, dtype=np.float64).reshape(
        n, ci, shape.h_in, shape.w_in)
    patches = co.tile_patches(ids, e, m, ho // e, wo // e)   # [n, c, ty, tx, m, m]
    coords = np.array(np.unravel_index(patches.astype(np.int64), ids.shape))  # [4, n, c, ty, tx, m, m]
    # the reference emits m^2 input trees per (b, oc, ty, tx, c), all over the same patch
    ref = leaves.reshape(n, co_, ho // e, wo // e, ci, m * m, m * m, 4)
    for xi in range(m * m):
        got = ref[:, :, :, :, :, xi]                            # [n, oc, ty, tx, c, m^2, 4]
        want = coords.transpose(1, 3, 4, 2, 5, 6, 0).reshape(n, 1, ho // e, wo // e, ci, m * m, 4)
        assert np.array_equal(got, np.broadcast_to(want, got.shape))


@pytest.mark.parametrize("case", WINO)
def test_package_winograd_dag_has_the_reference_patch_map(case):
    wo, ho, co_, ci, e, r, n = (int(v) for v in G[f"{case}_shape"])
    shape = ConvShape.from_output(wo, ho, co_, ci, r, r, n=n)
    dag = build_winograd_dag(shape, WinogradParams(e, r))
    n_img = n * ci * shape.h_in * shape.w_in
    pred = dag.predecessors()
    leaves = [pred[v][0] for v in range(dag.n_vertices)
              if dag.steps[v] == 1 and len(pred[v]) == 1 and pred[v][0] < n_img]
    coords = np.array(np.unravel_index(np.array(leaves), (n, ci, shape.h_in, shape.w_in))).T
    assert np.array_equal(coords.reshape(G[f"{case}_patches"].shape), G[f"{case}_patches"])
