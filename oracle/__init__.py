"""CPU oracle for the convolution hot path -- TEST INFRASTRUCTURE ONLY.

Imported exclusively by ``tests/``, ``__graft_entry__.smoke()`` and the CPU
baseline / ``--impl reference`` leg of ``bench.py``, always as the checker or
the reported CPU baseline.  The product package ``paper_2012_15667_b200``
never imports, links or executes anything under ``oracle/``.

* ``winograd_mats``: exact-rational F(e, r) transforms (Lavin-Gray for
  F(2,3)/F(4,3), Toom-Cook otherwise).
* ``conv_oracle``: float64 direct and Winograd convolution following the
  reference DAG semantics (``pkg/src/convio/dag.py:247-403``), in numpy and
  as a multi-threaded C restatement (``conv_oracle.c``).

Parity status for conv VALUES: the reference pins none (it never computes a
convolution), so this oracle is pinned by independent cross-checks instead
(``tests/test_oracle.py``): direct vs float64 ``torch.nn.functional.conv2d``,
Winograd vs direct, C vs numpy.  Model-layer parity (bounds, tiles, traffic,
tuner) is pinned against the reference itself (``tests/golden/``).
"""
