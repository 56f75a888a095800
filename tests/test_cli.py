"""Command line (reference cli.py, tests/test_cli.py behaviour): generation
and argument handling on CPU; solves on the GPU."""

import json
import os

import numpy as np
import pytest

from paper_1602_05033_b200 import mmio, problems as P
from paper_1602_05033_b200.cli import main


def test_gen_writes_problem_files(tmp_path):
    assert main(["gen", "--problem", "laplacian2d", "--n", "6", "--s", "2",
                 "--out", str(tmp_path)]) == 0
    a = mmio.read_coordinate(str(tmp_path / "A.mtx"))
    c = mmio.read_array(str(tmp_path / "C1.mtx"))
    assert (a != P.gen_fd2d("laplacian2d", 6)).nnz == 0     # exact round trip
    assert np.array_equal(c, P.gen_rhs(36, 2, 0))


def test_gen_pair_writes_both_sides(tmp_path):
    assert main(["gen", "--problem", "fd3d-split", "--n", "5", "--out", str(tmp_path)]) == 0
    for f in ("A.mtx", "B.mtx", "C1.mtx", "C2.mtx"):
        assert (tmp_path / f).exists()
    b = mmio.read_coordinate(str(tmp_path / "B.mtx"))
    assert (b != P.gen_fd3d_split(5)[1]).nnz == 0


def test_missing_n_is_an_error(tmp_path, capsys):
    assert main(["gen", "--problem", "laplacian2d", "--out", str(tmp_path)]) == 1
    assert "needs" in capsys.readouterr().err


def test_problem_and_files_are_exclusive(tmp_path, capsys):
    assert main(["solve-lyap", "--out", str(tmp_path)]) == 1
    assert "either --problem or explicit matrix files" in capsys.readouterr().err


def test_unknown_problem_kind_rejected(tmp_path):
    with pytest.raises(SystemExit):
        main(["gen", "--problem", "nope", "--n", "4", "--out", str(tmp_path)])


def test_bad_config_line(tmp_path, capsys):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("problem laplacian2d\n")
    assert main(["gen", "--config", str(cfg), "--out", str(tmp_path)]) == 1
    assert "key = value" in capsys.readouterr().err


def test_matrix_market_round_trip(tmp_path):
    a = P.gen_fd2d("fd2d-trig", 7)
    mmio.write_coordinate(str(tmp_path / "a.mtx"), a, symmetric=False)
    assert (mmio.read_coordinate(str(tmp_path / "a.mtx")) != a).nnz == 0
    m = np.random.default_rng(0).standard_normal((5, 3))
    mmio.write_array(str(tmp_path / "m.mtx"), m)
    assert np.array_equal(mmio.read_array(str(tmp_path / "m.mtx")), m)
    (tmp_path / "bad.mtx").write_text("not a matrix market file\n")
    with pytest.raises(mmio.MatrixMarketError):
        mmio.read_array(str(tmp_path / "bad.mtx"))


# ------------------------------------------------------------------ GPU solves
@pytest.mark.gpu
def test_solve_lyap_generated_to_convergence(tmp_path):
    out = tmp_path / "run"
    assert main(["solve-lyap", "--problem", "laplacian2d", "--n", "20", "--s", "2",
                 "--tol", "1e-8", "--out", str(out)]) == 0
    summary = json.loads((out / "summary.json").read_text())
    assert summary["converged"] and summary["final_relative_residual"] <= 1e-8
    hist = (out / "history.csv").read_text().splitlines()
    assert hist[0] == "m,space_dim,relative_residual,cum_basis_secs,cum_residual_secs"
    z = mmio.read_array(str(out / "Z.mtx"))
    assert z.shape == (400, summary["rank"])


@pytest.mark.gpu
def test_solve_lyap_config_file_with_flag_precedence(tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("problem = laplacian2d\nn = 12\ntol = 1e-3   # overridden\nstorage = windowed\n")
    out = tmp_path / "run"
    assert main(["solve-lyap", "--config", str(cfg), "--tol", "1e-9", "--out", str(out)]) == 0
    s = json.loads((out / "summary.json").read_text())
    assert s["tol"] == 1e-9 and s["storage"] == "windowed" and s["peak_basis_vectors"] == 3


@pytest.mark.gpu
def test_solve_lyap_asymmetric_file_rejected(tmp_path, capsys):
    (tmp_path / "A.mtx").write_text("%%MatrixMarket matrix coordinate real general\n"
                                    "2 2 3\n1 1 -2.0\n1 2 1.0\n2 2 -2.0\n")
    assert main(["solve-lyap", "--A", str(tmp_path / "A.mtx"), "--out", str(tmp_path)]) == 1
    err = capsys.readouterr().err
    assert "not symmetric" in err and "(0, 1)" in err


@pytest.mark.gpu
def test_solve_sylv_one_and_two_sided(tmp_path):
    for args, one in ((["--problem", "fd3d-split", "--n", "12"], True),
                      (["--problem", "fd2d-pair", "--n", "10", "--max-m", "300"], False)):
        out = tmp_path / ("one" if one else "two")
        assert main(["solve-sylv", *args, "--tol", "1e-8", "--out", str(out)]) == 0
        s = json.loads((out / "summary.json").read_text())
        assert s["one_sided"] is one and s["final_relative_residual"] <= 1e-8
        z1, z2 = mmio.read_array(str(out / "Z1.mtx")), mmio.read_array(str(out / "Z2.mtx"))
        assert z1.shape[1] == z2.shape[1] == s["rank"]


@pytest.mark.gpu
def test_nonconvergence_exit_code_and_history(tmp_path, capsys):
    out = tmp_path / "run"
    assert main(["solve-lyap", "--problem", "laplacian2d", "--n", "30", "--tol", "1e-14",
                 "--max-m", "5", "--out", str(out)]) == 1
    assert "no convergence" in capsys.readouterr().err
    assert len((out / "history.csv").read_text().splitlines()) == 6


@pytest.mark.gpu
def test_bench_residual(tmp_path):
    out = tmp_path / "run"
    assert main(["bench-residual", "--problem", "laplacian2d", "--n", "15", "--tol", "1e-6",
                 "--out", str(out)]) == 0
    rows = (out / "bench.csv").read_text().splitlines()
    assert rows[0].startswith("m,space_dim,res_fast,res_naive")
    for r in rows[1:]:
        f = [float(x) for x in r.split(",")]
        assert abs(f[2] - f[3]) <= 1e-12 * max(f[3], 1e-300) + 1e-15
