"""CPU: the host-side mirror of the reference interface (data model, variant
rules, argument checks) and the sharding arithmetic -- no GPU calls."""
import numpy as np
import pytest

import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import kernels
from paper_2203_08263_b200.device import needs_self_mask
from paper_2203_08263_b200.sharded import pad_system, padded_count, shard_range


def test_simparams_checks_mirror_reference():
    for bad in (dict(gravitational_constant=0.0), dict(dt=0.0), dict(softening_sq=-1.0), dict(steps=0)):
        with pytest.raises(ValueError):
            nb.SimParams(**bad)
    p = nb.SimParams()
    assert (p.gravitational_constant, p.dt, p.softening_sq, p.steps) == (1.0, 0.01, 1e-9, 100)


def test_kernel_variant_rules_mirror_reference():
    with pytest.raises(ValueError):
        nb.KernelVariant(nb.Layout.AOS, threads=4)
    with pytest.raises(ValueError):
        nb.KernelVariant(nb.Layout.AOS, math_form=nb.MathForm.RECIPROCAL_MULTIPLY)
    with pytest.raises(ValueError):
        nb.KernelVariant(nb.Layout.AOS, block=8)
    with pytest.raises(ValueError):
        nb.KernelVariant(threads=0)
    with pytest.raises(ValueError):
        nb.KernelVariant(block=0)
    assert nb.KernelVariant(nb.Layout.AOS).name == "aos"
    assert nb.reference_variant().name == "soa"
    assert nb.KernelVariant(nb.Layout.SOA, nb.MathForm.RECIPROCAL_MULTIPLY, 8, 4).name == "soa-recip-b8"
    assert len(nb.ladder()) == 1 + 2 * 4 * 3


def test_check_rejects_like_reference():
    s = nb.system_from_arrays([[0.0, 0, 0], [1.0, 0, 0]], np.zeros((2, 3)), [1.0, 1.0])
    with pytest.raises(ValueError):
        kernels._check(s, nb.KernelVariant(nb.Layout.AOS), None)
    with pytest.raises(ValueError):
        kernels._check(s, nb.KernelVariant(block=8), None)
    with pytest.raises(ValueError):
        kernels._check(s, None, nb.AccelerationBuffer.allocate(3, nb.Precision.DOUBLE))
    with pytest.raises(ValueError):
        kernels._check(s, None, nb.AccelerationBuffer.allocate(2, nb.Precision.SINGLE))
    kernels._check(s, nb.reference_variant(), nb.AccelerationBuffer.allocate(2, nb.Precision.DOUBLE))


def test_system_validation():
    with pytest.raises(ValueError):
        nb.system_from_arrays([[0.0, 0, 0]], [[0.0, 0, 0]], [0.0])
    with pytest.raises(ValueError):
        nb.system_from_arrays([[np.nan, 0, 0]], [[0.0, 0, 0]], [1.0])
    with pytest.raises(ValueError):
        nb.init_system(0, nb.Seed(1))
    with pytest.raises(ValueError):
        nb.Seed(-1)


def test_layout_roundtrip_and_checksum_invariance():
    s = nb.uniform_cube(100, 5, nb.Precision.SINGLE)
    a = nb.convert_layout(s, nb.Layout.AOS)
    b = nb.convert_layout(a, nb.Layout.SOA)
    for u, v in zip(s.positions, b.positions):
        np.testing.assert_array_equal(u, v)
    assert nb.checksum(s) == nb.checksum(a)
    two = nb.system_from_arrays([[1.0, 2, 3], [4.0, 5, 6]], np.zeros((2, 3)), [1.0, 1.0])
    assert nb.checksum(two) == 21.0


def test_single_precision_is_rounded_double():
    d = nb.uniform_cube(64, 9, nb.Precision.DOUBLE)
    s = nb.uniform_cube(64, 9, nb.Precision.SINGLE)
    for u, v in zip(d.positions, s.positions):
        np.testing.assert_array_equal(u.astype(np.float32), v)


def test_plummer_generator_shape():
    s = nb.plummer_sphere(4096, 0, nb.Precision.SINGLE)
    r = np.linalg.norm(s.position_matrix(), axis=1)
    assert np.all(np.isfinite(r)) and np.all(s.masses == np.float32(1 / 4096))
    # half-mass radius of a Plummer sphere of scale 1 is ~1.305
    assert 1.15 < np.median(r) < 1.45
    assert np.all(np.stack(s.velocities, 1) == 0)


def test_baseline_configs_match_baseline_json():
    c = nb.BASELINE_CONFIGS
    assert (c["C1"].n, c["C1"].precision, c["C1"].softening_sq, c["C1"].dt, c["C1"].steps) == \
        (1024, nb.Precision.DOUBLE, 1e-2, 1e-2, 10)
    assert (c["C2"].n, c["C2"].precision, c["C2"].steps) == (16384, nb.Precision.SINGLE, 100)
    assert (c["C3-f32"].n, c["C3-f64"].precision, c["C3-f32"].softening_sq) == (131072, nb.Precision.DOUBLE, 1e-3)
    assert (c["C4"].n, c["C4"].steps, c["C4"].gpus) == (524288, 5, (1, 2, 4, 8))
    assert (c["C5"].n, c["C5"].softening_sq, c["C5"].generator) == (4194304, 1e-4, nb.plummer_sphere)
    assert c["C3-f32"].interactions == 131072 ** 2 * 11


def test_self_mask_rule():
    m = np.ones(4)
    assert needs_self_mask(m, 0.0, np.float64)
    assert not needs_self_mask(m, 1e-9, np.float64)
    assert needs_self_mask(m, 1e-46, np.float32)       # rounds to 0 in FP32
    assert needs_self_mask(m, 1e-27, np.float32)       # m*eps2^-1.5 overflows FP32
    assert not needs_self_mask(m, 1e-4, np.float32)
    # uniform-mass kernels form eps2^-1.5 without m: a small uniform mass must
    # not hide an overflowing self term
    assert needs_self_mask(np.full(4, 1e-10), 1e-26, np.float32)
    assert needs_self_mask(np.full(4, 1e-10, np.float32), 1e-26, np.float32)


def test_shard_arithmetic():
    assert padded_count(10, 4) == 12 and padded_count(12, 4) == 12
    assert [shard_range(12, r, 4) for r in range(4)] == [(0, 3), (3, 3), (6, 3), (9, 3)]
    pos = np.random.default_rng(0).random((10, 3))
    p, v, m = pad_system(pos, np.zeros((10, 3)), np.ones(10), 4)
    assert p.shape == (12, 3) and np.all(m[10:] == 0) and np.all(np.abs(p[10:]) > 1e17)
    p2, _, _ = pad_system(pos, np.zeros((10, 3)), np.ones(10), 5)
    assert p2 is pos


def test_empty_and_mismatched_inputs_rejected_before_device_work():
    """Empty and ragged inputs raise ValueError like the reference's validation
    (core.py:157-180) -- no device is touched."""
    with pytest.raises(ValueError):
        nb.simulate_arrays(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0), 1e-3, 1e-3, 1)
    with pytest.raises(ValueError):
        nb.simulate_arrays(np.zeros((4, 3)), np.zeros((3, 3)), np.ones(4), 1e-3, 1e-3, 1)
    with pytest.raises(ValueError):
        nb.simulate_arrays(np.zeros((4, 3)), np.zeros((4, 3)), np.ones(4), 1e-3, 1e-3, 0)
    with pytest.raises(ValueError):
        nb.simulate_arrays(np.zeros((4, 3)), np.zeros((4, 3)), np.ones(4), -1.0, 1e-3, 1)
    with pytest.raises(ValueError):
        nb.system_from_arrays(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0))


def test_precision_mismatch_rejected_before_device_work():
    """A system whose arrays are not in its declared precision raises ValueError
    before any device work, as the reference's typed buffers do at the FFI call
    (_accel_cy.pyx:114); nothing is silently cast."""
    pos = tuple(np.zeros(4) for _ in range(3))
    vel = tuple(np.zeros(4) for _ in range(3))
    bad = nb.ParticleSystem(nb.Layout.SOA, nb.Precision.SINGLE, pos, vel, np.ones(4))
    with pytest.raises(ValueError, match="dtype mismatch"):
        nb.simulate(bad, nb.SimParams(1.0, 1e-3, 1e-3, 1))
    with pytest.raises(ValueError, match="dtype mismatch"):
        nb.compute_accelerations(bad, nb.SimParams(1.0, 1e-3, 1e-3, 1))
    mixed = nb.ParticleSystem(nb.Layout.AOS, nb.Precision.DOUBLE, np.zeros((4, 3)),
                              np.zeros((4, 3), np.float32), np.ones(4))
    with pytest.raises(ValueError, match="dtype mismatch"):
        nb.simulate(mixed, nb.SimParams(1.0, 1e-3, 1e-3, 1))
