"""The GPU optimisation ladder held to the reference's
ladder parity: the reference pins every rung of its CPU ladder to the
reference-variant checksum within 1e-9 (double) / 5e-4 (single)
(pkg/tests/test_kernels.py:178-201, validation.py:33).  Here every GPU rung
(tools/variants.py LADDER: pow form, recip form, MUFU rsqrt, unrolling,
register blocking, packed FFMA2, the LG2/EX2 weights -- each built as its own
library) computes FP32 accelerations within 1e-5 of the long-double oracle
(``_accel_dev``) and a 5-step trajectory whose checksum is within 5e-4 of the
FP64 oracle's; the shipped library equals the top rung bit for bit."""
import os
import shutil
import sys

import numpy as np
import pytest

import paper_2203_08263_b200 as nb

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "tools"))

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                                 reason="nvcc needed to build the ladder rungs")]


@pytest.fixture(scope="module")
def rungs():
    import variants
    return variants.ladder_libs()


def test_ladder_rungs_match_oracle(rungs, oracle):
    import variants
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    n, eps2, dt, steps = 8192, 1e-3, 1e-3, 5
    s = nb.uniform_cube(n, 0, nb.Precision.SINGLE)
    dtype = np.dtype(np.float32)
    st = DeviceState(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, dtype)
    mask = kernel_flags(s.masses, eps2, dtype)
    rows = np.unique(np.concatenate([[0, n - 1], np.random.default_rng(4).integers(0, n, 190)]))
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k].astype(dtype)) for k in range(3)), s.masses,
                                rows, 1.0, eps2)
    ref64, _ = oracle.simulate(pos, np.stack(s.velocities, 1).astype(np.float64), s.masses.astype(np.float64),
                               1.0, dt, eps2, steps, threads=oracle.host_threads())
    cs64 = oracle.checksum(ref64)
    shipped = nb.simulate(s, nb.SimParams(1.0, dt, eps2, steps)).position_matrix()
    report = []
    for i, path in sorted(rungs.items()):
        a = variants.variant_accel(path, st, n, eps2, mask, dtype)
        dev = oracle.accel_dev(a[rows], want)
        fin = variants.variant_simulate(path, s, 1.0, dt, eps2, steps, mask, dtype)
        cs = oracle.checksum(fin)
        rel = abs(cs - cs64) / abs(cs64)
        report.append((variants.LADDER[i][0], dev, rel))
        print(f"{variants.LADDER[i][0]:60s} accel_dev {dev:.2e} checksum rel {rel:.2e}")
        assert dev <= 1e-5, (i, dev)
        assert rel <= 5e-4, (i, rel)
        if variants.LADDER[i][1] == {}:  # the shipped configuration
            np.testing.assert_array_equal(fin, shipped)
    assert len(report) == len(variants.LADDER)
