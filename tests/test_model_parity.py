"""Bit-exact parity of the model layer with the reference ``convio``.

The golden file was produced by running the reference itself
(``tests/golden/make_model_golden.py``); every float is compared with ``==``.
Cases: BASELINE.json layers under the B200 machine model plus the
reference tests' own small shapes (``tests/golden/cases.py``).
"""

import json
import math
import os
import warnings
from fractions import Fraction

import pytest

from paper_2012_15667_b200 import bounds, dataflow, autotune
from paper_2012_15667_b200.model import ConvShape, WinogradParams, HwModel

from cases import B200_HW  # noqa: F401  (tests/golden on sys.path via conftest)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "model_golden.json")

with open(GOLDEN) as fh:
    G = json.load(fh)


def _shape(d):
    return ConvShape.from_output(*d["out"], d["cin"], *d["ker"], stride=d.get("stride", 1),
                                 n=d.get("n", 1))


def _fl(v):
    return float(v) if isinstance(v, str) else v


def _wp(case):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return WinogradParams(case["e"], case["r"])


def _ids(rows):
    return [f"{i}" for i in range(len(rows))]


@pytest.mark.parametrize("row", G["bounds"], ids=_ids(G["bounds"]))
def test_lower_bounds_bit_exact(row):
    case = row["case"]
    shape = _shape(case)
    if case["alg"] == "direct":
        rep = bounds.lower_bound_dc(shape, case["s"])
    else:
        rep = bounds.lower_bound_wa(shape, _wp(case), case["s"])
    assert rep.to_dict() == row["report"]
    assert rep.to_json() == row["json"]


@pytest.mark.parametrize("row", G["t_upper"], ids=_ids(G["t_upper"]))
def test_t_upper_bit_exact(row):
    case = row["case"]
    if case["alg"] == "direct":
        prof = bounds.dc_profile(Fraction(case["R"]))
        closed = bounds.t_upper_dc(case["s"], Fraction(case["R"]))
    else:
        prof = bounds.wa_profile(case["e"], case["r"], case.get("variant", False))
        closed = bounds.t_upper_wa(case["s"], case["e"], case["r"])
    val, ks = bounds.t_upper_generic_argmax(prof, case["s"])
    assert val == row["value"]
    assert list(ks) == row["argmax"]
    assert closed == row["closed"]


def test_tile_selection_bit_exact():
    for row in G["tiles"]:
        case = row["case"]
        shape = _shape(case)
        hw = HwModel(**case["hw"])
        try:
            if case["alg"] == "direct":
                t = dataflow.optimal_tile_dc(shape, hw)
            else:
                t = dataflow.optimal_tile_wa(shape, _wp(case), hw)
        except dataflow.InfeasibleTileError as exc:
            assert row.get("error") == str(exc), case
            continue
        assert t.to_dict() == row["tile"], case


def test_schedules_and_simulation_bit_exact():
    for row in G["sims"]:
        case = row["case"]
        shape = _shape(case)
        hw = HwModel(**case["hw"])
        tile = dataflow.TileConfig(**case["tile"])
        try:
            if case["alg"] == "direct":
                sch = dataflow.plan_direct_dataflow(shape, hw, tile)
                est = dataflow.analytic_dc_io(shape, hw, tile)
                opt = dataflow.dc_io_at_optimum(shape, hw)
            else:
                p = _wp(case)
                shared = case.get("shared", False)
                sch = dataflow.plan_winograd_dataflow(shape, p, hw, tile, shared)
                est = dataflow.analytic_wa_io(shape, p, hw, tile, shared)
                opt = dataflow.wa_io_at_optimum(shape, p, hw)
            rep = dataflow.simulate(sch, hw)
        except (dataflow.ScheduleError, dataflow.InfeasibleTileError) as exc:
            assert row.get("error") == type(exc).__name__ + ": " + str(exc), case
            continue
        assert sch.summary() == row["summary"]
        assert rep.to_dict() == row["sim"]
        assert est.to_dict() == row["est"]
        assert opt == row["optimum"]
        trace = dataflow.stage_trace_rows(sch)
        assert trace[:2] == row["trace_head"] and trace[-1:] == row["trace_tail"]


def _digest(space):
    import hashlib
    h = hashlib.sha256()
    for c in space.members:
        h.update(repr(tuple(c.to_dict().values())).encode())
    return h.hexdigest()


@pytest.mark.parametrize("row", G["spaces"], ids=_ids(G["spaces"]))
def test_search_space_identical(row):
    case = row["case"]
    shape = _shape(case)
    hw = HwModel(**case["hw"])
    p = _wp(case) if case["alg"] == "winograd" else None
    sp = autotune.build_space(shape, hw, case["alg"], p, thread_axes=case["threads"])
    assert (sp.size, sp.unconstrained_size) == (row["size"], row["unconstrained"])
    assert sp.reduction_ratio == row["ratio"]
    assert str(sp.r_factor) == row["r_factor"]
    assert _digest(sp) == row["digest"]
    step = max(1, sp.size // 7)
    assert [sp.members[i].to_dict() for i in range(0, sp.size, step)] == row["sample"]
    step = max(1, sp.size // 11)
    costs = [autotune.measure(sp.members[i], shape, hw, case["alg"], p).cost
             for i in range(0, sp.size, step)]
    assert costs == [_fl(c) for c in row["costs"]]


@pytest.mark.parametrize("row", G["tunes"], ids=_ids(G["tunes"]))
def test_seeded_tuner_history_identical(row):
    case = row["case"]
    shape = _shape(case)
    hw = HwModel(**case["hw"])
    p = _wp(case) if case["alg"] == "winograd" else None
    sess = autotune.tune(shape, hw, case["alg"], case["budget"], case["seed"], winograd=p,
                         n_s=case["n_s"], patience=case.get("patience", 50))
    assert sess.history == row["history"]
    assert sess.to_best_json() == row["best_json"]


@pytest.mark.parametrize("row", G["oracles"], ids=_ids(G["oracles"]))
def test_exhaustive_and_random_search_identical(row):
    case = row["case"]
    shape = _shape(case)
    hw = HwModel(**case["hw"])
    p = _wp(case) if case["alg"] == "winograd" else None
    sp = autotune.build_space(shape, hw, case["alg"], p, thread_axes=case["threads"])
    cfg, cost = autotune.exhaustive_oracle(sp)
    assert [cfg.to_dict(), cost] == [row["exhaustive"][0], _fl(row["exhaustive"][1])]
    cfg, cost = autotune.random_search(sp, case["budget"], case["seed"])
    assert [cfg.to_dict(), cost] == [row["random"][0], _fl(row["random"][1])]


def test_reference_cli_golden_tune():
    """The reference's own golden run (pkg/tests/golden/tune_best.json, copied)."""
    shape = ConvShape.from_output(2, 2, 2, 2, 3, 3)
    hw = HwModel(s=256, s_sm=128)
    sess = autotune.tune(shape, hw, "direct", 12, 7, n_s=4)
    with open(os.path.join(os.path.dirname(__file__), "golden", "tune_best.json")) as fh:
        assert json.loads(sess.to_best_json()) == json.load(fh)
    assert sess.best_cost == 340.0 and math.isfinite(sess.best_cost)
