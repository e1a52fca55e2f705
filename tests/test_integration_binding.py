"""The Cython binding of INTEGRATION.md §3 (integration/_accel_b200.pyx): the
reference's backend protocol over the C ABI, built with typed memoryviews the
way the reference's own compiled backend is."""
import glob
import importlib.util
import os

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binding():
    paths = glob.glob(os.path.join(REPO, "integration", "_accel_b200*.so"))
    if not paths:
        import subprocess, sys
        subprocess.run([sys.executable, os.path.join(REPO, "integration", "build.py")], check=True)
        paths = glob.glob(os.path.join(REPO, "integration", "_accel_b200*.so"))
    spec = importlib.util.spec_from_file_location("_accel_b200", paths[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_binding_exposes_the_backend_protocol(binding):
    assert binding.NAME == "b200"
    for fn in ("accel_soa", "accel_aos", "step_soa", "step_aos"):
        assert callable(getattr(binding, fn))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_binding_matches_python_backend(binding, dtype):
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200 import backend
    prec = nb.Precision.SINGLE if dtype == np.float32 else nb.Precision.DOUBLE
    s = nb.uniform_cube(2000, 9, prec)
    px, py, pz = (c.copy() for c in s.positions)
    a1 = [np.zeros(2000, dtype) for _ in range(3)]
    a2 = [np.zeros(2000, dtype) for _ in range(3)]
    binding.accel_soa(px, py, pz, s.masses, 1.0, 1e-3, True, 0, 4, *a1)
    backend.accel_soa(px, py, pz, s.masses, 1.0, 1e-3, True, 0, 4, *a2)
    for u, v in zip(a1, a2):
        np.testing.assert_array_equal(u, v)
    pos = np.ascontiguousarray(np.stack([px, py, pz], 1))
    vel = np.ascontiguousarray(np.stack(s.velocities, 1))
    p1, v1 = pos.copy(), vel.copy()
    binding.step_aos(p1, v1, *a1, 1e-3)
    p2, v2 = pos.copy(), vel.copy()
    backend.step_aos(p2, v2, *a2, 1e-3)
    np.testing.assert_array_equal(p1, p2)
    np.testing.assert_array_equal(v1, v2)
    # registered as one more entry of the reference's backend table
    backends = {"b200": binding}
    assert backends["b200"].NAME == "b200"
