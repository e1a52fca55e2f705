"""Benchmark rows in the reference's CSV schema.

`nbodybench report` renders GFLOPS tables from a CSV with a fixed 18-column
header (/root/reference/pkg/src/nbodybench/cli.py:40-45, rows at :394-432,
parsed at :435-467).  ``measure`` times the GPU ``simulate`` with the
reference's own protocol -- initialisation outside the clock, warm-up runs,
best of R repetitions on a monotonic clock, checksum of the last final state
(harness.py:120-162) -- and ``emit_csv`` writes rows that the reference's
``report`` subcommand accepts unchanged, so GPU rows sit beside CPU rows.

The ``variant`` label is ``b200-<precision>-p<gpus>``; ``threads`` carries the
GPU count (the reference's parallelism axis); GFLOPS use the reference
convention 20*N^2*steps/t (harness.py:39-47).  Defaults are the reference
harness's own (BenchConfig, harness.py:55-71: double precision, seed 42,
dt 0.01, eps2 1e-9, G 1, 5 repetitions, 1 warm-up; initial state from
init_system, core.py:200-227), so a GPU row sits beside CPU rows of the same
physics.  The 18-column schema has no dt/eps2 columns: when either differs from
those defaults the variant label says so (``b200-f32-p1-dt0.001-eps2_0.001``).
"""

from __future__ import annotations

import csv
import math
import os
import platform
import time
from dataclasses import dataclass, field
from datetime import datetime, timezone
from typing import Callable, List, Optional, Sequence

from .core import Precision, SimParams, checksum, format_checksum, init_system
from .kernels import simulate

__all__ = ["CSV_HEADER", "GpuBenchConfig", "GpuBenchResult", "gflops", "measure", "result_row",
           "emit_csv"]

#: The reference's fixed schema, cli.py:40-45 (pinned by tests/test_report.py).
CSV_HEADER = [
    "variant", "layout", "math_form", "block_size", "threads", "precision",
    "n_bodies", "steps", "seed", "repetitions", "best_time_s", "mean_time_s",
    "gflops_best", "gflops_mean", "checksum", "status", "host_label",
    "timestamp_utc",
]

FLOPS_PER_INTERACTION = 20


def gflops(n: int, steps: int, seconds: float) -> float:
    """20 * n^2 * steps / (seconds * 1e9), with harness.py:39-47's argument checks."""
    if n < 1:
        raise ValueError("n must be positive")
    if steps < 1:
        raise ValueError("steps must be positive")
    if not seconds > 0:
        raise ValueError(f"seconds must be positive, got {seconds!r}")
    return FLOPS_PER_INTERACTION * float(n) * float(n) * float(steps) / (seconds * 1e9)


#: harness.BenchConfig's defaults (harness.py:55-71).
REFERENCE_DT = 0.01
REFERENCE_EPS2 = 1e-9


@dataclass(frozen=True)
class GpuBenchConfig:
    n_bodies: int
    steps: int
    precision: Precision = Precision.DOUBLE
    seed: int = 42
    repetitions: int = 5
    warmup_runs: int = 1
    gravitational_constant: float = 1.0
    dt: float = REFERENCE_DT
    softening_sq: float = REFERENCE_EPS2
    gpus: int = 1

    def sim_params(self) -> SimParams:
        return SimParams(self.gravitational_constant, self.dt, self.softening_sq, self.steps)


@dataclass
class GpuBenchResult:
    config: GpuBenchConfig
    times_s: List[float] = field(default_factory=list)
    best_time_s: Optional[float] = None
    mean_time_s: Optional[float] = None
    gflops_best: Optional[float] = None
    gflops_mean: Optional[float] = None
    checksum: Optional[float] = None
    status: str = "ok"
    host_label: str = ""
    timestamp_utc: str = ""

    @property
    def variant_label(self) -> str:
        c = self.config
        p = "f32" if c.precision is Precision.SINGLE else "f64"
        label = f"b200-{p}-p{c.gpus}"
        if c.dt != REFERENCE_DT:
            label += f"-dt{c.dt:g}"
        if c.softening_sq != REFERENCE_EPS2:
            label += f"-eps2_{c.softening_sq:g}"
        if c.gravitational_constant != 1.0:
            label += f"-G{c.gravitational_constant:g}"
        return label


def _host_label() -> str:
    try:
        import torch
        dev = torch.cuda.get_device_name(0) if torch.cuda.is_available() else "nogpu"
    except Exception:  # pragma: no cover
        dev = "nogpu"
    return f"{platform.node() or 'unknown'}/{platform.machine()}/{os.cpu_count()}c/{dev}"


def measure(config: GpuBenchConfig, *, init_fn: Callable = init_system,
            clock: Callable[[], float] = time.perf_counter,
            simulate_fn: Optional[Callable] = None) -> GpuBenchResult:
    """harness.measure's protocol (harness.py:120-162) around the GPU simulate."""
    sim = simulate_fn or simulate
    params = config.sim_params()
    sys0 = init_fn(config.n_bodies, config.seed, config.precision)
    for _ in range(config.warmup_runs):
        sim(sys0, params)
    times, final = [], None
    for _ in range(config.repetitions):
        t0 = clock()
        final = sim(sys0, params)
        times.append(clock() - t0)
    cs = checksum(final)
    best, mean = min(times), sum(times) / len(times)
    return GpuBenchResult(
        config=config, times_s=times, best_time_s=best, mean_time_s=mean,
        gflops_best=gflops(config.n_bodies, config.steps, best),
        gflops_mean=gflops(config.n_bodies, config.steps, mean), checksum=cs,
        status="ok" if math.isfinite(cs) else "error:non-finite checksum",
        host_label=_host_label(),
        timestamp_utc=datetime.now(timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ"))


def _fmt(v: Optional[float]) -> str:
    return "" if v is None else repr(float(v))


def result_row(r: GpuBenchResult) -> List[str]:
    """One CSV row in the order of CSV_HEADER (cli.py:394-416 field formats)."""
    c = r.config
    return [r.variant_label, "soa", "recip", "", str(c.gpus), c.precision.value, str(c.n_bodies),
            str(c.steps), str(c.seed), str(c.repetitions), _fmt(r.best_time_s), _fmt(r.mean_time_s),
            _fmt(r.gflops_best), _fmt(r.gflops_mean),
            "" if r.checksum is None else format_checksum(r.checksum), r.status,
            r.host_label.replace(",", ";"), r.timestamp_utc]


def emit_csv(results: Sequence[GpuBenchResult], path: str, append: bool = False) -> None:
    """Header + rows (cli.py:419-432 semantics; append keeps an existing header)."""
    need_header = not (append and os.path.exists(path) and os.path.getsize(path) > 0)
    with open(path, "a" if append else "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        if need_header:
            w.writerow(CSV_HEADER)
        for r in results:
            w.writerow(result_row(r))
