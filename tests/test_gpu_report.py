"""``kltune report matrix|histogram --backend cuda`` on live B200 sessions.

Reference: cli.py:294-351 (report commands), report.py:63-215 (fraction of
optimum, cross matrix, PPM, histogram).  The reference can only re-evaluate
simulated sessions; here two short live tuning sessions of diff_uvw fp32 at
two shapes are re-measured on the GPU by the CLI's cuda evaluator.

Checks: the efficiency matrix diagonal is 1 up to timing noise (a scenario's
own optimum re-measured on its own problem), every entry is a positive
fraction, ``report ppm --matrix`` equals ``report.ppm`` of the rows, and the
histogram counts every successful evaluation once with the Table-2 default
marked as a fraction of the optimum.
"""

import csv

import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128, 128), (192, 96, 160)]


@pytest.fixture(scope="module")
def sessions(gpu_ctx, tmp_path_factory):
    from paper_2303_12374_b200.autotune import tune_problem
    from paper_2303_12374_b200.tuner import Budget

    out = tmp_path_factory.mktemp("sessions")
    paths = []
    for grid in SHAPES:
        session, _ = tune_problem("diff_uvw", "fp32", grid, gpu_ctx, strategy="random", budget=Budget(8, 300.0),
                                  seed=5, wisdom_dir=None, session_dir=out, repetitions=5, warmup=2,
                                  family="TMA", log=lambda *a: None)
        assert session.best is not None
        paths.append(next(out.glob(f"diff_uvw_fp32_{'x'.join(map(str, grid))}.*.klsession")))
    return paths


def _read(path):
    with open(path, newline="") as fh:
        return list(csv.reader(fh))


def test_report_matrix_and_ppm_on_the_gpu(sessions, tmp_path):
    from paper_2303_12374_b200 import cli
    from paper_2303_12374_b200.report import ppm

    mat = tmp_path / "matrix.csv"
    assert cli.main(["report", "matrix", *map(str, sessions), "--backend", "cuda", "--out", str(mat)]) == 0
    rows = _read(mat)
    assert rows[0][0] == "scenario" and len(rows) == 3 and all(len(r) == 3 for r in rows)
    entries = [[float(c) for c in r[1:]] for r in rows[1:]]
    for i, row in enumerate(entries):
        assert 0.8 <= row[i] <= 1.25, entries  # own optimum, re-measured
        assert all(0.0 < e <= 1.5 for e in row), entries
    out = tmp_path / "ppm.csv"
    assert cli.main(["report", "ppm", "--matrix", str(mat), "--out", str(out)]) == 0
    got = _read(out)
    assert got[0] == ["label", "best", "worst", "ppm"]
    for (label, *vals), row, src in zip(got[1:], entries, rows[1:]):
        want = ppm(row)
        assert label == src[0]
        assert [float(v) for v in vals] == pytest.approx([want.best, want.worst, want.ppm], abs=2e-6)


def test_report_histogram_on_the_gpu(sessions, tmp_path):
    from paper_2303_12374_b200 import cli
    from paper_2303_12374_b200.tuner import load_session

    out = tmp_path / "hist.csv"
    assert cli.main(["report", "histogram", str(sessions[0]), "--bins", "5", "--backend", "cuda",
                     "--out", str(out)]) == 0
    rows = _read(out)
    assert rows[0] == ["bin_low", "bin_high", "count"]
    counts = [int(r[2]) for r in rows[1:6]]
    assert sum(counts) == len(load_session(sessions[0]).ok_evaluations())
    markers = {r[1]: float(r[2]) for r in rows[6:] if r[0] == "marker"}
    assert 0.0 < markers["default"] <= 1.25  # the Table-2 default as a fraction of the tuned optimum
