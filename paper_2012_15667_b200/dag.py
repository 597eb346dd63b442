"""Closed-form vertex counts of the convolution DAGs.

Only the parts of reference ``pkg/src/convio/dag.py`` that the hot path
consumes live here: the lemma counts ``|V|`` used by the composite lower
bounds (``dag.py:184-204``, consumed at ``bounds.py:234,256``) and the
Winograd output padding (``dag.py:291-299``).  Graph materialisation,
adjacency I/O and multi-step-partition validation are theory tooling on
<=1e7-vertex graphs and are out of scope.

The DAG *semantics* -- left-deep sums over ``(c, ky, kx)`` for direct
convolution (``dag.py:274-284``) and the four Winograd steps
(``dag.py:358-401``) -- are what the CUDA kernels compute and what the
CPU oracle in ``oracle/`` restates.
"""

from __future__ import annotations

from .model import ConvShape, WinogradParams

# vertex kinds, same integer codes as the reference (dag.py:16)
INPUT, INTERNAL, OUTPUT = 0, 1, 2


def dc_internal_output_count(shape: ConvShape) -> int:
    """Internal + output vertices of the direct DAG: ``(2k - 1) * outputs * n``.

    Every output is one window of ``k`` products summed by a left-deep tree
    of ``k - 1`` adds.
    """
    per_output = 2 * shape.window_size - 1
    return per_output * shape.outputs_per_image * shape.n


def wa_per_tile_count(p: WinogradParams, c_in: int) -> int:
    """Vertices added by one (tile position, output channel) pair.

    Terms, in DAG step order: input-transform linear combinations, kernel
    transform linear combinations, element-wise products, channel sums,
    output transform (reference ``dag.py:190-199``).
    """
    m2 = p.m ** 2
    step1_input = m2 * (2 * m2 - 1) * c_in
    step1_kernel = m2 * (2 * p.r * p.r - 1) * c_in
    step2 = m2 * c_in
    step3 = m2 * (c_in - 1)
    step4 = p.e * p.e * (2 * m2 - 1)
    return step1_input + step1_kernel + step2 + step3 + step4


def wa_internal_output_count(shape: ConvShape, p: WinogradParams) -> int:
    pairs = (shape.w_out // p.e) * (shape.h_out // p.e) * shape.c_out
    return pairs * wa_per_tile_count(p, shape.c_in) * shape.n


def pad_shape_for_winograd(shape: ConvShape, p: WinogradParams) -> ConvShape:
    """Round the output up to a multiple of ``e``; the input grows to match."""
    def round_up(v: int) -> int:
        return ((v + p.e - 1) // p.e) * p.e

    return ConvShape.from_output(
        round_up(shape.w_out), round_up(shape.h_out), shape.c_out,
        shape.c_in, shape.w_ker, shape.h_ker, shape.stride, shape.n,
    )
