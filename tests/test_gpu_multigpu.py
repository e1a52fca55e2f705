"""Multi-GPU i-sharding on real GPUs, against the ORACLE.

One NCCL process per GPU (torch.distributed.run of tests/_mgpu_worker.py),
2 / 4 / 8 ranks as the box allows, for every exchange transport:

* ``nccl`` -- in-place all-gather on torch.distributed's NCCL, overlapped with
  the local-source pass (sharded.run_sharded);
* ``capi`` -- the same exchange through the library's own nb_comm_* C ABI;
* ``p2p``  -- the fused peer-store epilogue into symmetric memory;
* ``api``  -- the public ``simulate()``, which shards itself over the group.

Cases (tests/_mgpu_worker.py): a C4-shaped FP64 cube (N = 65536, 5 steps), a
C5-shaped FP32 Plummer sphere (N = 262144, 3 steps) and a ragged FP32 case
(N = 30001, eps2 = 0: padding + the self mask).  Tolerances:
``_position_dev`` <= 1e-12 (FP64) and <= 10x the reference's own FP32-vs-FP64
deviation (FP32), every rank holding the same final state bit for bit.

These need >= 2 GPUs and skip on the 1-GPU box; there, the same worker and
checks run with 2 ranks sharing the GPU over gloo (host-staged exchange, no
rank's kernel waits on another's) so the driver logic is exercised anyway.
Also: ``bench.py --gpus 2`` launches its own ranks.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(REPO, "tests", "_mgpu_worker.py")
sys.path.insert(0, os.path.join(REPO, "tests"))

pytestmark = pytest.mark.gpu


def _ngpu() -> int:
    import torch
    return torch.cuda.device_count()


def _port() -> int:
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _launch(world, case, transport, out, backend="nccl", timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), WORKER, "--case", case,
           "--transport", transport, "--out", str(out), "--backend", backend]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
    d = np.load(out)
    assert int(d["world"]) == world and int(d["ranks_agree"]) == 1
    return d["pos"], d["vel"]


_ORACLE = {}


def _oracle_case(case, oracle):
    """(FP64 oracle positions, tolerance) for a case, computed once per session."""
    if case not in _ORACLE:
        from _mgpu_worker import case_system
        s, c = case_system(case)
        th = oracle.host_threads()
        pos, vel, m = s.position_matrix(), np.stack(s.velocities, 1), s.masses
        ref64, _ = oracle.simulate(pos, vel.astype(np.float64), m.astype(np.float64), 1.0, c["dt"], c["eps2"],
                                   c["steps"], threads=th)
        if c["prec"] == "double":
            tol = 1e-12
        else:
            ref32, _ = oracle.simulate(np.stack(s.positions, 1), vel, m, 1.0, c["dt"], c["eps2"], c["steps"],
                                       threads=th)
            tol = 10 * oracle.position_dev(ref32, ref64)
        _ORACLE[case] = (ref64, tol)
    return _ORACLE[case]


RUNS = [(2, t, c) for c in ("c4s", "c5s") for t in ("nccl", "capi", "p2p", "api")] + \
       [(2, "nccl", "ragged"), (4, "nccl", "c4s"), (4, "p2p", "c5s"), (4, "capi", "ragged"),
        (8, "nccl", "c5s"), (8, "p2p", "c4s")]


@pytest.mark.parametrize("world,transport,case", RUNS)
def test_sharded_simulate_vs_oracle(world, transport, case, oracle, tmp_path):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs (one process per GPU), found {_ngpu()}")
    pos, _ = _launch(world, case, transport, tmp_path / "out.npz")
    ref, tol = _oracle_case(case, oracle)
    dev = oracle.position_dev(pos, ref)
    print(case, transport, f"P={world}", "position_dev", dev, "tol", tol)
    assert dev <= tol


@pytest.mark.parametrize("case", ["c4s", "ragged"])
def test_sharded_driver_two_ranks_one_gpu_gloo(case, oracle, tmp_path):
    """The worker and the oracle comparison with 2 ranks on one GPU over gloo:
    the multi-rank driver (shards, padding, host-staged all-gather, final
    velocity gather, rank agreement) on the 1-GPU box."""
    pos, _ = _launch(2, case, "nccl", tmp_path / "out.npz", backend="gloo")
    ref, tol = _oracle_case(case, oracle)
    dev = oracle.position_dev(pos, ref)
    print(case, "gloo x2 on one GPU", "position_dev", dev, "tol", tol)
    assert dev <= tol


def test_bench_launches_its_own_ranks():
    """python bench.py --gpus 2 without torchrun: spawns its ranks (one per GPU)
    and prints one JSON line with n_gpus 2."""
    if _ngpu() < 2:
        pytest.skip(f"needs 2 GPUs, found {_ngpu()}")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "2",
                        "--warmup", "3", "--config", "C2", "--no-traffic"],
                       capture_output=True, text=True, timeout=900, cwd=REPO)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
