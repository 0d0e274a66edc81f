"""CLI plumbing on CPU (no solve): generate, dry runs, usage and data errors.
Mirrors the reference's pkg/tests/test_cli.py cases that do not solve."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2105_07544_b200 as mk
from paper_2105_07544_b200 import cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_main(capsys, *args):
    rc = cli.main(list(args))
    out, err = capsys.readouterr()
    return rc, out, err


def test_generate_writes_a_readable_matrix(tmp_path, capsys):
    out = tmp_path / "lap8.mtx"
    rc, so, _ = run_main(capsys, "generate", "--preset", "Laplace2D", "--nx", "8", "--out", str(out))
    assert rc == 0 and so.strip() == "N=64 NNZ=288 -> %s" % out
    A = mk.read_matrix_market(str(out))
    B = mk.generate_stencil(mk.ProblemSpec("Laplace2D", 8))
    assert (A.n, A.nnz) == (B.n, B.nnz)
    assert np.array_equal(A.values, B.values) and np.array_equal(A.col_idx, B.col_idx)


def test_dry_runs_print_dimensions(capsys):
    rc, so, _ = run_main(capsys, "generate", "--preset", "BentPipe2D", "--nx", "1500", "--dry-run")
    assert rc == 0 and so.strip() == "N=2250000 NNZ=11244000"
    rc, so, _ = run_main(capsys, "solve", "--preset", "Laplace3D", "--nx", "200", "--dry-run")
    assert rc == 0 and so.strip() == "N=8000000 NNZ=55760000"


def test_solve_dry_run_from_matrix_file(tmp_path, capsys):
    out = tmp_path / "l.mtx"
    assert run_main(capsys, "generate", "--preset", "Laplace2D", "--nx", "8", "--out", str(out))[0] == 0
    rc, so, _ = run_main(capsys, "solve", "--matrix", str(out), "--dry-run")
    assert rc == 0 and so.strip() == "N=64 NNZ=288"


def test_generate_requires_an_output_path(capsys):
    rc, _, err = run_main(capsys, "generate", "--preset", "Laplace2D", "--nx", "8")
    assert rc == 1 and err.startswith("error:")


@pytest.mark.parametrize("args", [
    ("solve", "--preset", "NoSuchPreset"),
    ("solve",),
    ("solve", "--preset", "Laplace2D", "--matrix", "x.mtx"),
    ("solve", "--preset", "Laplace2D", "--tol", "2.0"),
    ("solve", "--preset", "Laplace2D", "--precond", "lu:3"),
    ("solve", "--preset", "Laplace2D", "--restart", "0"),
    ("solve", "--preset", "Laplace2D", "--solver", "gmres-ir", "--precision", "single"),
    ("solve", "--preset", "Laplace2D", "--solver", "gmres-fd"),
    ("solve", "--preset", "Laplace2D", "--solver", "gmres-fd", "--switch-iter", "7"),
    ("solve", "--matrix", "/nonexistent/file.mtx"),
    ("sweep-switch", "--preset", "Laplace2D", "--switch-points", "", "--output", "/tmp/x.csv"),
    ("sweep-restart", "--preset", "Laplace2D", "--sizes", "a,b", "--output", "/tmp/x.csv"),
])
def test_usage_and_data_errors_exit_with_code_one(args, capsys):
    rc, _, err = run_main(capsys, *args)
    assert rc == 1 and err.startswith("error:")


def test_module_entry_point():
    proc = subprocess.run([sys.executable, "-m", "paper_2105_07544_b200", "generate", "--preset", "Laplace3D",
                           "--nx", "40", "--dry-run"], capture_output=True, text=True, cwd=ROOT)
    assert proc.returncode == 0 and proc.stdout.strip() == "N=64000 NNZ=438400"
