"""bench_cli (the reference's bench CLI/CSV, tools/bench.cpp, experiments.cpp) and
.dmat I/O (io.cpp:44-72)."""
import csv
import os

import numpy as np
import pytest

from oracle import oracle as o
from paper_2111_11148_b200 import bench_cli, dmat


def test_grid_syntax():  # grids.cpp:28-47, test_bench.cpp
    assert bench_cli.parse_grid("1e3:1e6") == [1e3, 1e4, 1e5, 1e6]
    assert bench_cli.parse_grid("1:8:1") == [1, 2, 3, 4, 5, 6, 7, 8]
    assert bench_cli.parse_grid("5") == [5.0]
    for bad in ("a", "9:1", "1:2:0", "1:2:3:4"):
        with pytest.raises(bench_cli.UsageError):
            bench_cli.parse_grid(bad)
    assert bench_cli.parse_methods("rqr,rlu") == [5, 4]
    with pytest.raises(bench_cli.UsageError):
        bench_cli.parse_methods("nope")
    assert bench_cli.parse_shift("fixed:1e-15").value == 1e-15


def test_usage_errors_exit_2(tmp_path):  # tools/bench.cpp exit codes
    assert bench_cli.main([]) == 2
    assert bench_cli.main(["accuracy"]) == 2  # --out missing
    assert bench_cli.main(["accuracy", "--methods", "bogus", "--out", str(tmp_path / "x.csv")]) == 2
    assert bench_cli.main(["scaling", "--mode", "sideways", "--out", str(tmp_path / "x.csv")]) == 2


def test_header_matches_reference_schema():  # experiments.cpp:45-55
    assert bench_cli.HEADER[:11] == ["method", "m", "n", "l", "p", "kappa", "seed", "status", "orth_err", "res_err",
                                     "cond_x"]
    assert bench_cli.HEADER[11:18] == ["t_sketch_ms", "t_precondition_ms", "t_gram_ms", "t_cholesky_ms",
                                       "t_trisolve_ms", "t_recover_ms", "t_householder_ms"]
    assert bench_cli.HEADER[-3:] == ["t_total_ms", "comm_rounds", "comm_volume"]
    assert bench_cli.derive(1, 0x5E7C) == o.derive(1, 0x5E7C)


def test_dmat_round_trip(tmp_path):  # test_matgen.cpp:107-127
    a = o.gaussian_matrix(37, 5, 3)
    p = str(tmp_path / "a.dmat")
    dmat.save_dmat(p, a)
    assert os.path.getsize(p) == 16 + 37 * 5 * 8
    assert np.array_equal(dmat.load_dmat(p), a)
    with open(p, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(ValueError):
        dmat.load_dmat(p)


@pytest.mark.gpu
def test_accuracy_csv_on_device(tmp_path):  # acceptance.cpp:97-122 (C2, small)
    out = str(tmp_path / "acc.csv")
    rc = bench_cli.main(["accuracy", "--m", "20000", "--n", "20", "--kappa", "1e4:1e12",
                         "--methods", "cholqr,cholqr2,rqr,rlu,rqr-gaussian,scholqr3", "--seeds", "1", "--out", out])
    assert rc == 0
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 9 * 6
    st = {(r["method"], float(r["kappa"])): r for r in rows}
    assert st[("cholqr", 1e4)]["status"] == "ok" and st[("cholqr", 1e12)]["status"] == "breakdown"
    assert st[("cholqr2", 1e12)]["status"] == "breakdown"
    for meth in ("rqr", "rlu", "rqr-gaussian", "scholqr3"):
        r = st[(meth, 1e12)]
        assert r["status"] == "ok" and float(r["orth_err"]) <= 1e-11 and float(r["res_err"]) <= 1e-12
        assert float(r["t_total_ms"]) > 0
    assert st[("rqr", 1e12)]["l"] == "40"


@pytest.mark.gpu
def test_synthesize_dev_spectrum():  # test_matgen.cpp:34-44
    from paper_2111_11148_b200 import cholqr as cq

    a = cq.synthesize_dev(5000, 20, 1e5, 11).cpu().numpy()
    sv = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(sv, 1e5 ** (-np.arange(20) / 19.0), rtol=1e-8)
    b = cq.synthesize_dev(5000, 20, 1e5, 11).cpu().numpy()
    assert np.array_equal(a, b)
    # two-segment spectrum (BASELINE c4): geometric then flat
    sig = np.concatenate([10.0 ** (-8 * np.arange(10) / 9), np.full(10, 1e-8)])
    c = cq.synthesize_dev(4000, 20, sigma=sig, seed=3).cpu().numpy()
    assert np.allclose(np.linalg.svd(c, compute_uv=False), np.sort(sig)[::-1], rtol=1e-7)
