"""CSV interop with the reference's `nbodybench report`."""
import os
import sys

import pytest

import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import report

REF_SRC = "/root/reference/pkg/src"
REPO_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _fake_result(gpus=1, prec=nb.Precision.SINGLE, n=131072):
    cfg = report.GpuBenchConfig(n_bodies=n, steps=10, precision=prec, gpus=gpus, seed=0)
    r = report.GpuBenchResult(config=cfg, times_s=[0.08, 0.09], best_time_s=0.08, mean_time_s=0.085,
                              gflops_best=report.gflops(n, 10, 0.08), gflops_mean=report.gflops(n, 10, 0.085),
                              checksum=54.053778966743266, host_label="box/x86_64/16c/NVIDIA B200",
                              timestamp_utc="2026-10-20T00:00:00Z")
    return r


def test_header_is_the_reference_schema(golden_constants):
    assert report.CSV_HEADER == golden_constants["csv_header"]
    assert len(report.CSV_HEADER) == 18


def test_gflops_convention():
    assert report.gflops(1000, 100, 2.0) == 1.0          # pkg/tests/test_harness.py:15-16
    assert abs(report.gflops(524288, 100, 360.7) - 1524) < 1  # paper's FP32 peak inversion
    with pytest.raises(ValueError):
        report.gflops(0, 1, 1.0)


def test_row_format(tmp_path):
    r = _fake_result()
    row = report.result_row(r)
    assert len(row) == 18 and row[0] == "b200-f32-p1" and row[15] == "ok"
    assert row[14] == "54.053778966743266"
    path = tmp_path / "gpu.csv"
    report.emit_csv([r], str(path))
    report.emit_csv([_fake_result(prec=nb.Precision.DOUBLE)], str(path), append=True)
    lines = path.read_text().strip().splitlines()
    assert lines[0].split(",") == report.CSV_HEADER and len(lines) == 3


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present (GPU box)")
def test_reference_report_renders_gpu_rows(tmp_path):
    """The reference's own reader and markdown report accept the rows."""
    sys.path.insert(0, REF_SRC)
    try:
        from nbodybench.cli import read_rows, render_report
    finally:
        sys.path.remove(REF_SRC)
    path = tmp_path / "gpu.csv"
    report.emit_csv([_fake_result(1), _fake_result(1, nb.Precision.DOUBLE), _fake_result(2)], str(path))
    rows = read_rows(str(path))
    assert [r["variant"] for r in rows] == ["b200-f32-p1", "b200-f64-p1", "b200-f32-p2"]
    md = render_report(str(path))
    assert "b200-f32-p1" in md and "GFLOPS" in md


def test_defaults_are_the_reference_harness_defaults():
    """GpuBenchConfig defaults = harness.BenchConfig's (harness.py:55-71); a row of
    other physics says so in its label, since the schema has no dt/eps2 column."""
    c = report.GpuBenchConfig(n_bodies=256, steps=10)
    assert (c.precision, c.seed, c.repetitions, c.warmup_runs, c.dt, c.softening_sq,
            c.gravitational_constant) == (nb.Precision.DOUBLE, 42, 5, 1, 0.01, 1e-9, 1.0)
    assert report.GpuBenchResult(config=c).variant_label == "b200-f64-p1"
    odd = report.GpuBenchConfig(n_bodies=256, steps=10, precision=nb.Precision.SINGLE, dt=1e-3, softening_sq=1e-3)
    assert report.GpuBenchResult(config=odd).variant_label == "b200-f32-p1-dt0.001-eps2_0.001"


@pytest.mark.gpu
def test_measure_on_gpu(tmp_path):
    r = report.measure(report.GpuBenchConfig(n_bodies=4096, steps=5, repetitions=2))
    assert r.status == "ok" and r.gflops_best > 0 and len(r.times_s) == 2
    report.emit_csv([r], str(tmp_path / "m.csv"))


@pytest.mark.gpu
def test_measure_golden_rows_through_reference_report(tmp_path):
    """Real GPU rows through the CSV path: report.measure with the reference
    harness defaults reproduces GOLDEN_SIM_CHECKSUM (N=256, 10 steps, seed 42;
    pkg/tests/conftest.py:25-29) to 1e-12, the BASELINE C1 run reproduces the C1
    known answer 9.5618706445328652 to 1e-12 -- in the CSV
    text, i.e. after the 17-digit checksum formatting -- and the installed
    reference's own read_rows/render_report (cli.py:435-545) accept the rows."""
    import paper_2203_08263_b200 as nbb
    golden = report.measure(report.GpuBenchConfig(n_bodies=256, steps=10, repetitions=2))
    c1 = nbb.BASELINE_CONFIGS["C1"]
    c1_cfg = report.GpuBenchConfig(n_bodies=c1.n, steps=c1.steps, seed=0, dt=c1.dt, softening_sq=c1.softening_sq,
                                   repetitions=2)
    c1_row = report.measure(c1_cfg, init_fn=lambda n, seed, prec: c1.system())
    f32 = report.measure(report.GpuBenchConfig(n_bodies=256, steps=10, repetitions=2,
                                               precision=nb.Precision.SINGLE))
    path = tmp_path / "gpu.csv"
    report.emit_csv([golden, c1_row, f32], str(path))
    import csv as _csv
    rows = list(_csv.DictReader(open(path)))
    assert abs(float(rows[0]["checksum"]) - 387.73663935192604) <= 1e-12 * 387.73663935192604
    assert abs(float(rows[1]["checksum"]) - 9.5618706445328652) <= 1e-12 * 9.5618706445328652
    assert abs(float(rows[2]["checksum"]) - 387.73663935192604) <= 5e-4 * 387.73663935192604
    assert [r["status"] for r in rows] == ["ok"] * 3
    assert [r["variant"] for r in rows] == ["b200-f64-p1", "b200-f64-p1-eps2_0.01", "b200-f32-p1"]
    ref = os.path.join(REPO_ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "nbodybench")):
        pytest.skip("installed reference (baseline/_ref) missing: run __graft_entry__.build()")
    sys.path.insert(0, ref)
    try:
        from nbodybench.cli import read_rows, render_report
    finally:
        sys.path.remove(ref)
    parsed = read_rows(str(path))
    assert [r["variant"] for r in parsed] == [r["variant"] for r in rows]
    md = render_report(str(path))
    assert "b200-f64-p1" in md
