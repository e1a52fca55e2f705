"""CSV interop with the reference's `nbodybench report`."""
import os
import sys

import pytest

import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import report

REF_SRC = "/root/reference/pkg/src"


def _fake_result(gpus=1, prec=nb.Precision.SINGLE, n=131072):
    cfg = report.GpuBenchConfig(n_bodies=n, steps=10, precision=prec, gpus=gpus)
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


@pytest.mark.gpu
def test_measure_on_gpu(tmp_path):
    r = report.measure(report.GpuBenchConfig(n_bodies=4096, steps=5, repetitions=2))
    assert r.status == "ok" and r.gflops_best > 0 and len(r.times_s) == 2
    report.emit_csv([r], str(tmp_path / "m.csv"))
