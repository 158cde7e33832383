"""Harness / CLI: report shapes, table round trips, exit codes (reference tests/test_harness.py).
The host-only pieces run on CPU; anything that solves is marked gpu."""

import csv
import io
import json
import os

import numpy as np
import pytest

from paper_2604_23175_b200 import harness as H
from paper_2604_23175_b200.cli import build_parser, main

CASES = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2604_23175_b200", "cases")
CASE14 = os.path.join(CASES, "ieee14.m")
CASE118 = os.path.join(CASES, "ieee118.m")


def spec_for(path=CASE14, **kw):
    base = dict(case_path=path, repeats=2, seed=0, method="centralized")
    base.update(kw)
    return H.ExperimentSpec(**base)


# ---- CPU: host logic ---------------------------------------------------------------------------------
def test_parser_has_the_reference_subcommands_and_flags():
    ap = build_parser()
    for cmd in ("run", "sweep-k", "mask", "gen-measurements", "partition", "compare"):
        args = ap.parse_args([cmd, "--case", "x.m"])
        assert args.repeats == 11 and args.tol == 1e-6 and args.max_iters == 10 and args.inner_steps == 1
        assert args.method == "multiarea" and args.deterministic is True and args.output_format == "json"
        assert args.sigma_vm == 0.01 and args.sigma_power == 0.02 and args.reuse_plan is False


def test_write_rows_csv_and_json_round_trip(tmp_path):
    rows = [{"k": 2, "feasible": True, "boundary_dim": 10, "error": ""}, {"k": 99, "feasible": False, "error": "boom"}]
    text = H.write_rows(rows, H.SWEEP_COLUMNS, None, "csv")
    back = list(csv.DictReader(io.StringIO(text)))
    assert [r["k"] for r in back] == ["2", "99"] and back[1]["error"] == "boom" and list(back[0]) == list(H.SWEEP_COLUMNS)
    out = tmp_path / "t.json"
    H.write_rows(rows, H.SWEEP_COLUMNS, str(out), "json")
    assert json.loads(out.read_text())["rows"][0]["boundary_dim"] == 10
    with pytest.raises(ValueError, match="output format"):
        H.write_rows(rows, H.SWEEP_COLUMNS, None, "xml")


def test_columns_match_the_reference_tables():
    assert H.RUN_COLUMNS == ("run", "iterations", "converged", "objective", "weighted_residual_norm", "total_time_s",
                             "assembly_s", "local_condense_s", "boundary_assemble_s", "boundary_solve_s", "recovery_s")
    assert H.MASK_COLUMNS == ("family", "removed_rows", "iterations", "converged", "mean_time_s", "objective", "error")


def test_file_commands_and_error_exit_codes(tmp_path, capsys):
    out = tmp_path / "m.json"
    assert main(["gen-measurements", "--case", CASE14, "--out", str(out)]) == 0
    assert "wrote 122 rows" in capsys.readouterr().out
    pout = tmp_path / "p.json"
    assert main(["partition", "--case", CASE14, "--k", "3", "--out", str(pout)]) == 0
    summary = json.loads(capsys.readouterr().out)
    assert summary["k"] == 3 and summary["boundary_dim"] > 0 and json.loads(pout.read_text())
    assert main(["run", "--case", str(tmp_path / "missing.m")]) == 2          # reference cli.py:192-194
    assert "error:" in capsys.readouterr().err
    with pytest.raises(ValueError, match="repeats"):
        H.run_experiment(spec_for(repeats=0))


def test_load_inputs_uses_files_when_given(tmp_path):
    main(["gen-measurements", "--case", CASE14, "--out", str(tmp_path / "m.csv"), "--seed", "3"])
    main(["partition", "--case", CASE14, "--k", "2", "--out", str(tmp_path / "p.json")])
    net, ms, part = H.load_inputs(H.ExperimentSpec(case_path=CASE14, measurements_path=str(tmp_path / "m.csv"),
                                                   partition_path=str(tmp_path / "p.json")))
    assert net.n_bus == 14 and ms.m == 122 and part.k == 2


# ---- GPU: the studies ----------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("reuse", [False, True])
def test_run_report_shape(reuse):
    doc = H.run_experiment(spec_for(repeats=3, reuse_plan=reuse))
    assert doc["n_bus"] == 14 and doc["n_branch"] == 20 and doc["n_measurements"] == 122 and len(doc["runs"]) == 3
    mean = doc["mean_excluding_first"]
    assert mean["total_time_s"] == pytest.approx(np.mean([r["total_time_s"] for r in doc["runs"][1:]]))
    assert doc["all_converged"] is True and len({r["objective"] for r in doc["runs"]}) == 1
    assert doc["runs"][0]["objective"] == pytest.approx(92.88760446747206, rel=1e-10)      # SURVEY.md 6.2 (centralized)
    for r in doc["runs"]:
        assert sum(r[c] for c in H.RUN_COLUMNS[6:]) <= r["total_time_s"]


@pytest.mark.gpu
def test_sweep_k_rows_and_infeasible_k():
    rows = H.sweep_k(spec_for(CASE118, method="multiarea", repeats=2, reuse_plan=True), [2, 3, 6, 500])
    assert [r["k"] for r in rows] == [2, 3, 6, 500]
    assert all(r["feasible"] and r["converged"] for r in rows[:3])
    assert rows[2]["boundary_dim"] == 79 and rows[2]["iterations"] == 4
    assert all(0.0 <= r["coordinator_share"] <= 1.0 for r in rows[:3])
    assert rows[3]["feasible"] is False and rows[3]["error"]


@pytest.mark.gpu
def test_mask_experiment_rows():
    rows = H.mask_experiment(spec_for(CASE14, method="multiarea", k=2, repeats=2))
    assert [r["family"] for r in rows] == ["none", "pf", "pt", "qf", "qt"]
    assert rows[0]["removed_rows"] == 0 and all(r["removed_rows"] == 20 for r in rows[1:])
    assert all(r["converged"] is True for r in rows)
    assert rows[0]["objective"] == pytest.approx(92.8876044674714, rel=1e-10) and rows[1]["objective"] < rows[0]["objective"]


@pytest.mark.gpu
def test_compare_and_cli_exit_codes(tmp_path, capsys):
    doc = H.compare_methods(spec_for(CASE118, k=6))
    assert doc["k"] == 6 and doc["max_state_diff"] < 1e-9 and doc["objectives_agree_1e6"] and doc["all_converged"]
    assert main(["run", "--case", CASE14, "--k", "2", "--repeats", "2", "--output-format", "csv"]) == 0
    table = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    assert table[-1]["run"] == "mean_excl_first" and len(table) == 3
    assert main(["run", "--case", CASE14, "--k", "2", "--repeats", "1", "--max-iters", "1"]) == 1     # not converged
    capsys.readouterr()
    assert main(["compare", "--case", CASE14, "--out", str(tmp_path / "c.json")]) == 0
    assert json.loads((tmp_path / "c.json").read_text())["k"] == 2
