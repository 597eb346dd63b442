"""Generate ``model_golden.json`` by running the REFERENCE ``convio`` package.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_model_golden.py

The fixture pins the hot-path model functions -- lower bounds, T(S),
tile selection, schedules/simulation, analytic volumes, the Table-1 space and
seeded tuner runs -- to the reference's own outputs; ``tests/test_model_parity.py``
diffs this package against it with ``==`` on every float.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import warnings

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import convio  # noqa: E402  (the reference)
from convio.model import ConvShape, WinogradParams, HwModel  # noqa: E402
from convio import bounds, dataflow, autotune  # noqa: E402

from cases import (  # noqa: E402
    B200_HW, BOUND_CASES, T_CASES, TILE_CASES, SIM_CASES, SPACE_CASES,
    TUNE_CASES, ORACLE_CASES,
)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "model_golden.json")


def _shape(d):
    return ConvShape.from_output(*d["out"], d["cin"], *d["ker"], stride=d.get("stride", 1),
                                 n=d.get("n", 1))


def _hw(d):
    return HwModel(**d)


def _fl(v):
    """JSON-safe float that round-trips exactly (inf/nan as strings)."""
    if v is None:
        return None
    v = float(v)
    if math.isfinite(v):
        return v
    return repr(v)


def space_digest(space):
    h = hashlib.sha256()
    for c in space.members:
        h.update(repr(tuple(c.to_dict().values())).encode())
    return h.hexdigest()


def main():
    warnings.simplefilter("ignore")
    out = {"reference": "convio " + convio.__version__, "b200_hw": B200_HW}

    rows = []
    for case in BOUND_CASES:
        shape = _shape(case)
        if case["alg"] == "direct":
            rep = bounds.lower_bound_dc(shape, case["s"])
        else:
            rep = bounds.lower_bound_wa(shape, WinogradParams(case["e"], case["r"]), case["s"])
        d = rep.to_dict()
        rows.append({"case": case, "report": d, "json": rep.to_json()})
    out["bounds"] = rows

    rows = []
    for case in T_CASES:
        if case["alg"] == "direct":
            prof = bounds.dc_profile(case["R"])
        else:
            prof = bounds.wa_profile(case["e"], case["r"], case.get("variant", False))
        val, ks = bounds.t_upper_generic_argmax(prof, case["s"])
        closed = (bounds.t_upper_dc(case["s"], case["R"]) if case["alg"] == "direct"
                  else bounds.t_upper_wa(case["s"], case["e"], case["r"]))
        rows.append({"case": case, "value": val, "argmax": list(ks), "closed": closed})
    out["t_upper"] = rows

    rows = []
    for case in TILE_CASES:
        shape = _shape(case)
        hw = _hw(case["hw"])
        try:
            if case["alg"] == "direct":
                t = dataflow.optimal_tile_dc(shape, hw)
            else:
                t = dataflow.optimal_tile_wa(shape, WinogradParams(case["e"], case["r"]), hw)
            rows.append({"case": case, "tile": t.to_dict()})
        except dataflow.InfeasibleTileError as exc:
            rows.append({"case": case, "error": str(exc)})
    out["tiles"] = rows

    rows = []
    for case in SIM_CASES:
        shape = _shape(case)
        hw = _hw(case["hw"])
        tile = dataflow.TileConfig(**case["tile"])
        try:
            if case["alg"] == "direct":
                sch = dataflow.plan_direct_dataflow(shape, hw, tile)
                est = dataflow.analytic_dc_io(shape, hw, tile)
                opt = dataflow.dc_io_at_optimum(shape, hw)
            else:
                p = WinogradParams(case["e"], case["r"])
                shared = case.get("shared", False)
                sch = dataflow.plan_winograd_dataflow(shape, p, hw, tile, shared)
                est = dataflow.analytic_wa_io(shape, p, hw, tile, shared)
                opt = dataflow.wa_io_at_optimum(shape, p, hw)
            rep = dataflow.simulate(sch, hw)
            rows.append({
                "case": case, "summary": sch.summary(), "sim": rep.to_dict(),
                "est": est.to_dict(), "optimum": opt,
                "trace_head": dataflow.stage_trace_rows(sch)[:2],
                "trace_tail": dataflow.stage_trace_rows(sch)[-1:],
            })
        except (dataflow.ScheduleError, dataflow.InfeasibleTileError) as exc:
            rows.append({"case": case, "error": type(exc).__name__ + ": " + str(exc)})
    out["sims"] = rows

    rows = []
    for case in SPACE_CASES:
        shape = _shape(case)
        hw = _hw(case["hw"])
        p = WinogradParams(case["e"], case["r"]) if case["alg"] == "winograd" else None
        sp = autotune.build_space(shape, hw, case["alg"], p, thread_axes=case["threads"])
        sample = [sp.members[i].to_dict() for i in range(0, sp.size, max(1, sp.size // 7))]
        costs = [_fl(autotune.measure(sp.members[i], shape, hw, case["alg"], p).cost)
                 for i in range(0, sp.size, max(1, sp.size // 11))]
        rows.append({"case": case, "size": sp.size, "unconstrained": sp.unconstrained_size,
                     "ratio": sp.reduction_ratio, "digest": space_digest(sp),
                     "sample": sample, "costs": costs, "r_factor": str(sp.r_factor)})
    out["spaces"] = rows

    rows = []
    for case in TUNE_CASES:
        shape = _shape(case)
        hw = _hw(case["hw"])
        p = WinogradParams(case["e"], case["r"]) if case["alg"] == "winograd" else None
        sess = autotune.tune(shape, hw, case["alg"], case["budget"], case["seed"], winograd=p,
                             n_s=case["n_s"], patience=case.get("patience", 50))
        rows.append({"case": case, "best_json": sess.to_best_json(), "history": sess.history})
    out["tunes"] = rows

    rows = []
    for case in ORACLE_CASES:
        shape = _shape(case)
        hw = _hw(case["hw"])
        p = WinogradParams(case["e"], case["r"]) if case["alg"] == "winograd" else None
        sp = autotune.build_space(shape, hw, case["alg"], p, thread_axes=case["threads"])
        ex_cfg, ex_cost = autotune.exhaustive_oracle(sp)
        rs_cfg, rs_cost = autotune.random_search(sp, case["budget"], case["seed"])
        rows.append({"case": case, "exhaustive": [ex_cfg.to_dict(), _fl(ex_cost)],
                     "random": [rs_cfg.to_dict(), _fl(rs_cost)]})
    out["oracles"] = rows

    with open(OUT, "w") as fh:
        json.dump(out, fh, sort_keys=True, indent=1)
        fh.write("\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
