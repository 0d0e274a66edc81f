"""CLI solves on the GPU: summary line, summary JSON schema, history CSV,
exit codes and sweeps, as the reference's pkg/tests/test_cli.py pins them
(counts from tests/golden/runs.json, produced by the unmodified reference)."""

import json
import os

import pytest

from paper_2105_07544_b200 import cli

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "runs.json")))


def run_main(capsys, *args):
    rc = cli.main(list(args))
    out, err = capsys.readouterr()
    return rc, out, err


def test_solve_reports_one_summary_line(capsys):
    rc, so, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16")
    assert rc == 0
    g = GOLD["gmres_l2d16_m50"]
    line = so.strip()
    assert line.startswith("gmres double n=256 iters=%d restarts=%d relres=" % (g["iters"], g["restarts"]))
    assert line.endswith("converged")


def test_summary_json_has_the_full_schema(tmp_path, capsys):
    p = tmp_path / "s.json"
    rc, _, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--summary", str(p))
    assert rc == 0
    s = json.loads(p.read_text())
    assert list(s) == ["solver", "precision", "n", "nnz", "m", "rtol", "converged", "total_iters", "restarts",
                       "final_relres", "loss_of_accuracy", "wall_seconds"]
    assert (s["solver"], s["precision"], s["n"], s["nnz"], s["m"], s["rtol"]) == ("gmres", "double", 256, 1216,
                                                                                  50, 1e-10)
    assert s["converged"] is True and s["total_iters"] == 31 and s["restarts"] == 1
    assert 0 < s["final_relres"] <= 1e-10 and s["loss_of_accuracy"] is False and s["wall_seconds"] > 0


def test_history_csv_rows_follow_the_header(tmp_path, capsys):
    p = tmp_path / "h.csv"
    rc, _, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--history", str(p))
    assert rc == 0
    lines = p.read_text().splitlines()
    assert lines[0] == "iter,phase,implicit_relres,explicit_relres"
    assert lines[1] == "0,double,,1.0000000000e+00"
    assert len(lines) == 33
    last = lines[-1].split(",")
    assert last[:2] == ["31", "double"] and float(last[2]) <= 1e-10 and float(last[3]) <= 1e-10
    assert lines[5].split(",")[3] == ""
    # the implicit estimates agree with the reference's history to rounding
    ref = GOLD["gmres_l2d16_m50"]["history"]
    for row, r in zip(lines[2:], ref[1:]):
        v = float(row.split(",")[2])
        assert abs(v - r[2]) <= 1e-6 * r[2] + 1e-15


def test_refinement_and_switch_solvers(capsys):
    rc, so, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--solver", "gmres-ir")
    assert rc == 0 and so.startswith("gmres-ir double n=256 iters=")
    assert abs(int(so.split("iters=")[1].split()[0]) - GOLD["ir_l2d16_m50"]["iters"]) <= 50
    rc, so, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--solver", "gmres-fd",
                         "--switch-iter", "50")
    assert rc == 0 and so.startswith("gmres-fd double n=256") and "converged" in so


def test_single_precision_and_preconditioners(capsys):
    rc, so, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--precision", "single",
                         "--tol", "1e-5")
    assert rc == 0 and so.startswith("gmres single n=256")
    rc, so, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--precond", "jacobi:4")
    assert rc == 0 and "converged" in so
    rc, plain, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "32", "--tol", "1e-8")
    rc2, poly, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "32", "--tol", "1e-8",
                            "--precond", "poly:10", "--rhs", "random", "--seed", "7")
    assert rc == 0 and rc2 == 0
    it = lambda s: int(s.split("iters=")[1].split()[0])  # noqa: E731
    assert it(poly) < it(plain)


def test_exhausted_budget_exits_with_code_two(capsys):
    rc, so, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--max-iters", "5")
    assert rc == 2 and "not converged" in so


def test_rcm_and_repeat(tmp_path, capsys):
    p = tmp_path / "s.json"
    rc, _, _ = run_main(capsys, "solve", "--preset", "Laplace2D", "--nx", "16", "--rcm", "--repeat", "3",
                        "--summary", str(p))
    s = json.loads(p.read_text())
    assert rc == 0 and s["converged"] and s["final_relres"] <= 1e-10


def test_sweeps_write_the_expected_csv(tmp_path, capsys):
    out = tmp_path / "sw.csv"
    rc, _, _ = run_main(capsys, "sweep-switch", "--preset", "Laplace2D", "--nx", "32", "--switch-points",
                        "0,50,100", "--output", str(out))
    lines = out.read_text().splitlines()
    assert rc == 0 and lines[0] == "switch_iter,total_iters,iters_single,iters_double,converged"
    assert [ln.split(",")[0] for ln in lines[1:]] == ["0", "50", "100"]
    assert all(ln.endswith(",true") for ln in lines[1:])
    for ln in lines[1:]:
        s, t, lo, hi, _ = ln.split(",")
        assert int(t) == int(lo) + int(hi)
        gk = "fd_l2d32_s%s" % s
        if gk in GOLD:
            assert abs(int(t) - GOLD[gk]["iters"]) <= 50
    out2 = tmp_path / "rs.csv"
    rc, _, _ = run_main(capsys, "sweep-restart", "--preset", "Laplace2D", "--nx", "32", "--sizes", "25,50",
                        "--output", str(out2))
    lines = out2.read_text().splitlines()
    assert rc == 0 and lines[0] == "m,iters_double,iters_ir" and len(lines) == 3
    for ln in lines[1:]:
        m, itd, iti = ln.split(",")
        assert abs(int(itd) - GOLD["gmres_l2d32_m%s" % m]["iters"]) <= 1
        assert abs(int(iti) - GOLD["ir_l2d32_m%s" % m]["iters"]) <= int(m)
