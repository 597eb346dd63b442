"""CLI drop-in: same payloads, exit codes and byte-identical JSON as the
reference CLI on the hot-path subcommands (golden: tests/golden/tune_best.json;
live reference comparison when /root/reference is mounted)."""

import json
import os
import sys

import pytest

from paper_2012_15667_b200.cli import main, RunConfig

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
REF_SRC = "/root/reference/pkg/src"


def run(capsys, *argv):
    code = main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


def test_lower_bound_values(capsys):
    code, out, _ = run(capsys, "lower-bound", "--alg", "direct", "--cin", "256", "--out",
                       "13x13x384", "--ker", "3x3", "--stride", "1", "--s", "1024")
    assert code == 0 and json.loads(out)["omega"] == pytest.approx(275328, rel=1e-4)
    code, out, _ = run(capsys, "lower-bound", "--alg", "winograd", "--e", "2", "--cin", "256",
                       "--out", "13x13x384", "--ker", "3x3", "--s", "1024")
    assert code == 0 and json.loads(out)["omega"] == pytest.approx(3115008, rel=1e-3)


def test_usage_and_infeasible_exit_codes(capsys):
    code, _, err = run(capsys, "lower-bound", "--alg", "direct", "--cin", "4", "--out", "4x4x4",
                       "--ker", "3x3")
    assert code == 2 and "required" in err
    code, _, err = run(capsys, "simulate", "--alg", "direct", "--out", "6x6x4", "--ker", "3x3",
                       "--cin", "2", "--s", "144", "--tile", "6x6x4", "--sb", "100")
    assert code == 3 and "resident" in err
    code, _, err = run(capsys, "tune", "--alg", "direct", "--out", "4x4x4", "--ker", "3x3",
                       "--cin", "8", "--s", "512", "--ssm", "256", "--ns", "8", "--budget", "4")
    assert code == 2 and "budget" in err
    code, _, err = run(capsys, "pebble", "--fixture", "nope", "--s", "3")
    assert code == 2 and "available" in err
    code, _, err = run(capsys, "dag-stats", "--alg", "direct", "--out", "64x64x64", "--ker", "3x3",
                       "--cin", "64", "--cap", "1000")
    assert code == 3 and "vertices" in err


def test_dag_stats_and_pebble(capsys, tmp_path):
    export = tmp_path / "dc.dag"
    code, out, _ = run(capsys, "dag-stats", "--alg", "direct", "--out", "2x2x1", "--ker", "3x3",
                       "--cin", "2", "--export", str(export))
    payload = json.loads(out)
    assert code == 0 and payload["match"] == "yes" and payload["internal_plus_output"] == 140
    assert payload["steps"] == [1, 2] and export.exists()
    code, out, _ = run(capsys, "dag-stats", "--alg", "winograd", "--e", "2", "--out", "2x2x1",
                       "--ker", "3x3", "--cin", "1")
    assert code == 0 and json.loads(out)["match"] == "yes"
    code, out, _ = run(capsys, "pebble", "--fixture", "product2", "--s", "3")
    payload = json.loads(out)
    assert code == 0 and payload["q_min"] == 3 and payload["holds"] is True
    code, out, _ = run(capsys, "pebble", "--dag", str(export), "--s", "3")
    assert code == 3        # 2x2x1 output of a 2-channel 3x3 conv: too big for the exact oracle


def test_simulate_and_trace(capsys, tmp_path):
    trace = tmp_path / "t.csv"
    code, out, _ = run(capsys, "simulate", "--alg", "direct", "--out", "6x6x4", "--ker", "3x3",
                       "--cin", "2", "--s", "144", "--trace", str(trace))
    payload = json.loads(out)
    assert code == 0 and payload["simulated"]["q_total"] == payload["analytic"]["total_exact"] == 344
    assert trace.read_text().startswith("stage,")


def test_tune_golden_and_resume(capsys, tmp_path):
    with open(os.path.join(GOLDEN, "tune_best.json")) as fh:
        golden = json.load(fh)
    code, out, _ = run(capsys, "tune", "--alg", "direct", "--out", "2x2x2", "--ker", "3x3",
                       "--cin", "2", "--s", "256", "--ssm", "128", "--ns", "4", "--budget", "12",
                       "--seed", "7")
    assert code == 0 and json.loads(out) == golden
    ds = tmp_path / "ds.json"
    code, out1, _ = run(capsys, "tune", "--alg", "direct", "--out", "4x4x4", "--ker", "3x3",
                        "--cin", "8", "--s", "512", "--ssm", "256", "--ns", "8", "--budget", "40",
                        "--seed", "1", "--save-dataset", str(ds), "--csv", str(tmp_path / "h.csv"))
    code2, out2, _ = run(capsys, "tune", "--alg", "direct", "--out", "4x4x4", "--ker", "3x3",
                         "--cin", "8", "--s", "512", "--ssm", "256", "--ns", "8", "--budget", "16",
                         "--seed", "2", "--resume", str(ds))
    assert code == code2 == 0
    assert json.loads(out2)["best_cost"] <= json.loads(out1)["best_cost"]


def test_config_file_precedence_and_round_trip(capsys, tmp_path):
    text = "[shape]\nout = 6x6x4\nker=3x3\ncin = 2\n\n[hardware]\ns = 144\n"
    rc = RunConfig.from_text(text)
    assert RunConfig.from_text(rc.to_text()) == rc
    cfg = tmp_path / "run.cfg"
    cfg.write_text(text)
    code, out, _ = run(capsys, "simulate", "--config", str(cfg), "--alg", "direct")
    assert code == 0 and json.loads(out)["simulated"]["q_total"] == 344
    code, out, _ = run(capsys, "simulate", "--config", str(cfg), "--cin", "4", "--alg", "direct")
    assert json.loads(out)["simulated"]["q_total"] == 544


CASES = [
    ["lower-bound", "--alg", "direct", "--cin", "64", "--out", "56x56x64", "--ker", "3x3", "--s", "29184"],
    ["lower-bound", "--alg", "winograd", "--e", "4", "--cin", "64", "--out", "56x56x64", "--ker", "3x3",
     "--s", "29184"],
    ["simulate", "--alg", "direct", "--out", "56x56x64", "--ker", "3x3", "--cin", "64", "--s",
     "8638464", "--ssm", "58368", "--np", "296"],
    ["simulate", "--alg", "winograd", "--e", "2", "--out", "8x8x16", "--ker", "3x3", "--cin", "5",
     "--s", "8192", "--shared-j"],
    ["report", "--alg", "direct", "--out", "8x8x16", "--ker", "3x3", "--cin", "32", "--stride", "3",
     "--s", "256"],
    ["tune", "--alg", "direct", "--out", "8x8x16", "--ker", "3x3", "--cin", "32", "--s", "4096",
     "--ssm", "2048", "--ns", "8", "--budget", "24", "--seed", "3"],
]


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted")
@pytest.mark.parametrize("argv", CASES, ids=[c[0] + str(i) for i, c in enumerate(CASES)])
def test_byte_identical_to_reference_cli(argv, capsys):
    sys.path.insert(0, REF_SRC)
    try:
        import importlib
        ref_cli = importlib.import_module("convio.cli")
    finally:
        sys.path.remove(REF_SRC)
    ref_code = ref_cli.main(list(argv))
    ref_out = capsys.readouterr().out
    code, out, _ = run(capsys, *argv)
    assert (code, out) == (ref_code, ref_out)
