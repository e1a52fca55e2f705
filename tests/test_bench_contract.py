"""bench.py's JSON contract on the GPU box (small config, seconds)."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_contract():
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--config", "C2", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(line) == 1
    d = json.loads(line[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 1e11
    assert d["config"]["workload"] == "C2"
    rf = d["roofline"]
    assert 0.3 < rf["frac"] < 1.0 and rf["unit"] == "TFLOP/s" and rf["achieved"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3 * 101
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["value"] > 0


def test_reference_arm_contract():
    """--impl reference runs on the host only (no GPU needed)."""
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "interactions/s"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_multi_rank_bench_driver():
    """bench.py under torchrun with 2 ranks: the multi-rank driver logic (shards,
    in-place gather, barrier + max-over-ranks timing, rank-0 JSON, sharded e2e
    through the public API).  On a 1-GPU box the ranks share the device and
    exchange through gloo on the host (the NB_BENCH_BACKEND test hook) -- no
    rank's kernel waits on another's; the numbers are not a measurement."""
    env = dict(os.environ, NB_BENCH_BACKEND="gloo", OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(REPO, "bench.py"),
                        "--gpus", "2", "--config", "C1", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert "cpu_baseline" not in d  # rank 0 of N=1 only
