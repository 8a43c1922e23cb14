"""`flz-speig`, the speig-compatible command line (csrc/tools/speig_cli.cpp): the checks of the
reference's own CLI suite (proj/tests/cli_test.cpp) — report schema and accounting identities,
exit codes 0/1/2/3, --plain, --vectors, filter-info, info, bench.  filter-info and the usage
errors are host-only and run without a GPU; everything that solves is marked gpu."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2409_15053_b200 import _lib, matrices as M

CLI = os.path.join(_lib.PKG_DIR, "flz-speig")

DIAG5 = ("%%MatrixMarket matrix coordinate real symmetric\n5 5 5\n"
         "1 1 1.0\n2 2 2.0\n3 3 3.0\n4 4 4.0\n5 5 5.0\n")


def run(*args, timeout=300):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)


def write_laplacian(path, grid):
    """Matrix Market file (symmetric, lower triangle) of the reference's laplacian2d."""
    n, rp, ci, va = M.laplacian2d(grid)
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = ci <= rows
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        f.write(f"{n} {n} {int(keep.sum())}\n")
        for r, c, v in zip(rows[keep], ci[keep], va[keep]):
            f.write(f"{r + 1} {c + 1} {v:.17g}\n")


@pytest.fixture()
def diag5(tmp_path):
    p = tmp_path / "diag5.mtx"
    p.write_text(DIAG5)
    return p


# ------------------------------------------------------------------ host only (no GPU)
def test_cli_is_built():
    assert os.access(CLI, os.X_OK)
    r = run("--help")
    assert r.returncode == 0 and all(s in r.stdout for s in ("solve", "filter-info", "info", "bench"))
    assert run().returncode == 1 and run("frobnicate").returncode == 1


def test_filter_info_emits_coefficients_and_samples():      # cli_test.cpp:143-183
    r = run("filter-info", "--lo", 0.1, "--hi", 0.3, "--degree", 80)
    assert r.returncode == 0
    lines = r.stdout.splitlines()
    assert "# degree,80" in lines
    assert sum(l.startswith("coef,") for l in lines) == 81
    assert sum(l.startswith("sample,") for l in lines) == 2001
    # known answer (filter_test.cpp:27-47): b_0([0.1, 0.3]) on [-1, 1]
    assert float(next(l for l in lines if l.startswith("coef,0,")).split(",")[2]) == 0.06510240359141833
    # auto degree on [-1, -0.5] is 10 (filter_test.cpp:96-99)
    assert "# degree,10" in run("filter-info", "--lo", -1, "--hi", -0.5).stdout
    # the full interval is the constant 1
    r = run("filter-info", "--lo", -1, "--hi", 1, "--degree", 5, "--samples", 11)
    vals = [float(l.rsplit(",", 1)[1]) for l in r.stdout.splitlines() if l.startswith("sample,")]
    assert len(vals) == 11 and max(abs(v - 1.0) for v in vals) <= 1e-14
    assert run("filter-info", "--lo", 0.5, "--hi", 0.1).returncode == 2     # invalid interval
    j = json.loads(run("filter-info", "--lo", 0.1, "--hi", 0.3, "--degree", 12, "--json").stdout)
    assert j["degree"] == 12 and len(j["coefficients"]) == 13 and j["clamped"] is False
    # --bounds as "lo,hi" and as two values; = syntax
    a = run("filter-info", "--lo", 1, "--hi", 2, "--bounds", "0,8", "--degree=20").stdout
    b = run("filter-info", "--lo", 1, "--hi", 2, "--bounds", 0, 8, "--degree", 20).stdout
    assert a == b and "# bounds,0,8" in a


def test_usage_errors_are_exit_1(tmp_path):                   # cli_test.cpp:93-101
    assert run("solve", "--lo", 0, "--hi", 1).returncode == 1                     # --matrix missing
    assert run("solve", "--matrix", tmp_path / "nope.mtx", "--lo", 0, "--hi", 1).returncode == 1
    assert run("solve", "--matrix", "x", "--lo", "abc", "--hi", 1).returncode == 1
    assert run("solve", "--matrix", "x", "--lo", 0, "--hi", 1, "--frob").returncode == 1
    assert run("info", "--matrix", tmp_path / "gone.mtx").returncode == 1
    assert run("solve", "--help").returncode == 0
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n")
    r = run("info", "--matrix", bad)
    assert r.returncode == 1 and "error:" in r.stderr


# ------------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_solve_writes_a_correct_report(tmp_path, diag5):      # cli_test.cpp:37-73
    rep = tmp_path / "report.json"
    r = run("solve", "--matrix", diag5, "--lo", 1.5, "--hi", 3.5, "--block", 1, "--out", rep)
    assert r.returncode == 0, r.stderr
    j = json.loads(rep.read_text())
    assert j["eigs"] == 2 and j["converged"] is True and len(j["eigenvalues"]) == 2
    assert abs(j["eigenvalues"][0] - 2.0) < 1e-9 and abs(j["eigenvalues"][1] - 3.0) < 1e-9
    assert j["interval"] == [1.5, 3.5] and j["max_residual"] <= 1e-10
    assert j["mv"] == j["config"]["block"] * j["degree"] * j["iters"]      # accounting identity
    shares = [j["preproc_pct"], j["orth_pct"], j["mv_pct"]]
    assert all(0.0 <= p <= 100.0 for p in shares) and sum(shares) <= 100.0 + 1e-9
    assert "eigenvalues" in r.stdout and "degree" in r.stdout
    assert list(j) == sorted(j)                       # key order of the reference's JSON library
    assert set(j["config"]) == {"block", "tol", "max_dim", "seed", "check_every", "epsilon",
                                "degree", "plain"}
    assert j["config"]["degree"] == "auto" and j["mv_total"] == j["mv"] + j["mv_bounds"]


@pytest.mark.gpu
def test_exit_codes(tmp_path, diag5):                        # cli_test.cpp:84-117
    assert run("solve", "--matrix", diag5, "--lo", 3.5, "--hi", 1.5).returncode == 2
    assert run("solve", "--matrix", diag5, "--lo", 10, "--hi", 20).returncode == 2
    lap = tmp_path / "lap100.mtx"
    write_laplacian(lap, 10)
    rep = tmp_path / "partial.json"
    r = run("solve", "--matrix", lap, "--lo", 3.5, "--hi", 4.5, "--max-dim", 12, "--out", rep)
    assert r.returncode == 3 and "not converged" in r.stderr
    assert json.loads(rep.read_text())["converged"] is False


@pytest.mark.gpu
def test_plain_mode_and_vectors(tmp_path, diag5):             # cli_test.cpp:119-141
    rep = tmp_path / "plain.json"
    assert run("solve", "--matrix", diag5, "--lo", 4.5, "--hi", 5.5, "--block", 1, "--plain",
               "--out", rep).returncode == 0
    j = json.loads(rep.read_text())
    assert j["eigs"] == 1 and j["degree"] == 0 and abs(j["eigenvalues"][0] - 5.0) < 1e-9
    vecs = tmp_path / "vecs.mtx"
    assert run("solve", "--matrix", diag5, "--lo", 1.5, "--hi", 3.5, "--block", 1, "--vectors",
               vecs).returncode == 0
    lines = vecs.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix array real general" and lines[1] == "5 2"
    V = np.array([float(x) for x in lines[2:]]).reshape(2, 5).T
    assert np.abs(np.abs(V[[1, 2], [0, 1]]) - 1.0).max() < 1e-9              # unit vectors e_2, e_3


@pytest.mark.gpu
def test_info_prints_the_summary(diag5):                      # cli_test.cpp:185-196
    r = run("info", "--matrix", diag5)
    assert r.returncode == 0
    for s in ("n         5", "nnz       5", "nnz/n     1.0", "spectral interval"):
        assert s in r.stdout


@pytest.mark.gpu
def test_bench_runs_one_row_per_degree(tmp_path):             # cli_test.cpp:198-239
    lap = tmp_path / "lap100.mtx"
    write_laplacian(lap, 10)
    csv, js = tmp_path / "bench.csv", tmp_path / "bench.json"
    r = run("bench", "--matrix", lap, "--lo", 3.0, "--hi", 3.8, "--degrees", "30,60,auto", "--csv",
            csv, "--out", js)
    assert r.returncode == 0, r.stderr
    rows = json.loads(js.read_text())
    assert len(rows) == 3
    for row in rows:
        assert row["converged"] is True and row["mv"] == 3 * row["degree"] * row["iters"]
    assert rows[2]["config"]["degree"] == "auto" and rows[0]["config"]["degree"] == 30
    assert "matrix,lo,hi,eigs,degree" in csv.read_text()
    js2 = tmp_path / "bench2.json"
    assert run("bench", "--matrix", lap, "--lo", 3.0, "--hi", 3.8, "--degrees", "30,60,auto",
               "--out", js2).returncode == 0
    again = json.loads(js2.read_text())
    assert all(again[i]["eigenvalues"] == rows[i]["eigenvalues"] for i in range(3))   # deterministic
    assert run("bench", "--matrix", lap, "--lo", 3.0, "--hi", 3.8, "--degrees", "0").returncode == 1
