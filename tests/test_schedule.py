"""The stream-K schedule's invariants on the CPU (tests/native/sched_check.cu,
built with nvcc against the kernels' own header): exact cover, no empty CTA,
cost balance, cta_of/start consistency, equal split when nothing is skipped.
A CTA owning no units while a split i-block's fixup waited on its slot would
deadlock the in-kernel fixup, so this is checked exhaustively here."""
import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not os.path.exists(NVCC) and shutil.which("nvcc") is None, reason="nvcc not available")
def test_stream_k_schedule_invariants(tmp_path):
    exe = tmp_path / "sched_check"
    subprocess.run([NVCC, "-std=c++17", "-O1", "-I", os.path.join(REPO, "paper_2203_08263_b200", "csrc"),
                    os.path.join(REPO, "tests", "native", "sched_check.cu"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
