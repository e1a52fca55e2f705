"""GPU parity tests: the sm_100a path (through the package API and the C ABI)
against the CPU oracle and the reference's golden values.  Run on a B200:
``python -m pytest tests -m gpu``.

Tolerances (BASELINE.json north_star):
  * per-step accelerations, the `_accel_dev` metric of validation.py:212-225:
    <= 1e-5 (FP32) / <= 1e-12 (FP64) against an FP64-or-better oracle on the
    same rounded inputs;
  * trajectories, the `_position_dev` metric of validation.py:204-209: FP64
    <= 1e-12; FP32 <= 10x the reference's own FP32-vs-FP64 deviation;
  * the update arithmetic is bit-exact (same rounding sequence as step_soa/_kick).
"""
import numpy as np
import pytest

import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import _native
from paper_2203_08263_b200.core import uniform_cube

pytestmark = pytest.mark.gpu

import os
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

F64_ACC_TOL = 1e-12
F32_ACC_TOL = 1e-5
F64_POS_TOL = 1e-12

EPS0 = nb.SimParams(1.0, 0.1, 0.0, 1)


def accel_of(sys_, params, variant=None):
    out = nb.AccelerationBuffer.allocate(sys_.count, sys_.precision)
    nb.compute_accelerations(sys_, params, variant, out)
    return out


def as_mat(buf):
    return np.stack([buf.x, buf.y, buf.z], axis=1)


def two_body(precision=nb.Precision.DOUBLE, layout=nb.Layout.SOA):
    return nb.system_from_arrays([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]], np.zeros((2, 3)), [1.0, 1.0],
                                 layout=layout, precision=precision)


def cube(n, seed, prec):
    return uniform_cube(n, seed, nb.Precision(prec))


# --------------------------------------------------------------------------- known answers
# pkg/tests/test_kernels.py:22-55 restated for the GPU.

@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("eps2", [0.0, 1e-3])
def test_single_body_zero_acceleration(prec, eps2):
    s = nb.system_from_arrays([[0.3, 0.4, 0.5]], np.zeros((1, 3)), [2.5], precision=prec)
    a = accel_of(s, nb.SimParams(1.0, 0.1, eps2, 1))
    assert a.x[0] == 0.0 and a.y[0] == 0.0 and a.z[0] == 0.0


@pytest.mark.parametrize("prec", ["double", "single"])
def test_two_body_unit_case(prec):
    a = accel_of(two_body(nb.Precision(prec)), EPS0)
    tol = 2.3e-16 if prec == "double" else 1.2e-7
    np.testing.assert_allclose([a.x[0], a.x[1]], [1.0, -1.0], rtol=tol, atol=0)
    assert np.all(a.y == 0.0) and np.all(a.z == 0.0)


def test_unit_square_corner():
    s = nb.system_from_arrays([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.0]],
                              np.zeros((4, 3)), np.ones(4))
    a = accel_of(s, EPS0)
    expect = 1.0 + 2.0 ** -1.5
    np.testing.assert_allclose(a.x[0], expect, rtol=1e-15)
    np.testing.assert_allclose(a.y[0], expect, rtol=1e-15)
    assert a.z[0] == 0.0


@pytest.mark.parametrize("prec", ["double", "single"])
def test_coincident_bodies_without_softening_are_non_finite(prec):
    s = nb.system_from_arrays([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5]], np.zeros((2, 3)), [1.0, 1.0],
                              precision=prec)
    a = accel_of(s, EPS0)
    assert not np.all(np.isfinite(a.x))


def test_buffer_checks_match_reference():
    s = two_body()
    with pytest.raises(ValueError):
        nb.compute_accelerations(s, EPS0, nb.reference_variant(), nb.AccelerationBuffer.allocate(3, "double"))
    with pytest.raises(ValueError):
        nb.compute_accelerations(s, EPS0, nb.reference_variant(), nb.AccelerationBuffer.allocate(2, "single"))


# --------------------------------------------------------------------------- golden cases

def test_golden_case_accelerations(golden_cases, golden_arrays):
    worst = {}
    for c in golden_cases:
        s = cube(c["n"], c["seed"], c["precision"])
        a = as_mat(accel_of(s, nb.SimParams(1.0, c["dt"], c["eps2"], c["steps"])))
        want = golden_arrays[c["key"] + "_acc_oracle"]
        dev = 0.0 if c["n"] == 1 else nb_accel_dev(a, want)
        tol = F64_ACC_TOL if c["precision"] == "double" else F32_ACC_TOL
        worst[c["key"]] = dev
        assert dev <= tol, (c["key"], dev)
        if c["n"] == 1:
            assert np.all(a == 0.0)
    print("accel_dev per golden case:", worst)


def test_golden_case_trajectories(golden_cases, golden_arrays, oracle):
    for c in golden_cases:
        s = cube(c["n"], c["seed"], c["precision"])
        p = nb.SimParams(1.0, c["dt"], c["eps2"], c["steps"])
        fin = nb.simulate(s, p)
        pos = fin.position_matrix()
        opos = golden_arrays[c["key"] + "_pos_oracle"]
        if c["n"] == 1:
            np.testing.assert_array_equal(pos, golden_arrays[c["key"] + "_pos_ref"])
            continue
        dev = oracle.position_dev(pos, opos)
        if c["precision"] == "double":
            assert dev <= F64_POS_TOL, (c["key"], dev)
        else:
            ref_dev = oracle.position_dev(golden_arrays[c["key"] + "_pos_ref"], opos)
            assert dev <= max(10 * ref_dev, 1e-7), (c["key"], dev, ref_dev)


def nb_accel_dev(got, want):
    from oracle.oracle import accel_dev
    return accel_dev(got, want)


def test_c1_known_answer(golden_constants, golden_arrays, oracle):
    """BASELINE.json configs[0]: checksum 9.5618706445328652 (compiled reference)."""
    cfg = nb.BASELINE_CONFIGS["C1"]
    s = cfg.system()
    np.testing.assert_array_equal(s.position_matrix(), golden_arrays["c1_pos0"])
    a = as_mat(accel_of(s, cfg.params()))
    assert nb_accel_dev(a, golden_arrays["c1_acc_oracle"]) <= F64_ACC_TOL
    fin = nb.simulate(s, cfg.params())
    cs = nb.checksum(fin)
    want = golden_constants["c1_checksum"]
    assert abs(cs - want) / abs(want) <= 1e-12, (cs, want)
    assert oracle.position_dev(fin.position_matrix(), golden_arrays["c1_pos_oracle"]) <= F64_POS_TOL
    assert oracle.position_dev(fin.position_matrix(), golden_arrays["c1_pos_final"]) <= F64_POS_TOL


def test_c1_single_precision_trajectory(golden_arrays, oracle):
    cfg = nb.BASELINE_CONFIGS["C1"]
    s = uniform_cube(1024, 0, nb.Precision.SINGLE)
    fin = nb.simulate(s, cfg.params())
    opos = golden_arrays["c1_f32_pos_oracle"]
    ref_dev = oracle.position_dev(golden_arrays["c1_f32_pos_final"], opos)
    dev = oracle.position_dev(fin.position_matrix(), opos)
    assert dev <= 10 * ref_dev, (dev, ref_dev)


def test_reference_golden_sim_checksum(golden_constants):
    """GOLDEN_SIM_CHECKSUM (pkg/tests/conftest.py:25-29): N=256, steps=10, seed 42,
    G=1, dt=0.01, eps2=1e-9, double, within 1e-12."""
    s = nb.init_system(256, nb.Seed(42))
    fin = nb.simulate(s, nb.SimParams(1.0, 0.01, 1e-9, 10))
    want = golden_constants["sim_checksum_n256_seed42_steps10"]
    assert want == 387.73663935192604
    assert abs(nb.checksum(fin) - want) / want <= 1e-12


# --------------------------------------------------------------------------- update: bit-exact

@pytest.mark.parametrize("prec", ["double", "single"])
def test_integrate_step_bitwise(prec, oracle):
    s = cube(1000, 3, prec)
    acc = accel_of(s, nb.SimParams(1.0, 1e-3, 1e-3, 1))
    gpu = s.copy()
    nb.integrate_step(gpu, acc, nb.SimParams(1.0, 1e-3, 1e-3, 1))
    ref = s.copy()
    oracle.step_soa(*ref.positions, *ref.velocities, acc.x, acc.y, acc.z, 1e-3)
    for u, v in zip(gpu.positions + gpu.velocities, ref.positions + ref.velocities):
        np.testing.assert_array_equal(u, v)


def test_integrate_force_free_drift():
    s = nb.system_from_arrays([[0.0, 0.0, 0.0]], [[0.25, -1.0, 2.0]], [1.0])
    acc = nb.AccelerationBuffer.allocate(1, nb.Precision.DOUBLE)
    nb.integrate_step(s, acc, nb.SimParams(dt=0.5, steps=1))
    assert s.positions[0][0] == 0.125 and s.positions[1][0] == -0.5 and s.positions[2][0] == 1.0
    assert s.velocities[0][0] == 0.25


@pytest.mark.parametrize("prec", ["double", "single"])
def test_kick_kernel_bitwise(prec, oracle):
    import torch
    dtype = np.dtype(np.float32 if prec == "single" else np.float64)
    rng = np.random.default_rng(5)
    n = 777
    v, a1, a0 = (rng.standard_normal((n, 3)).astype(dtype) for _ in range(3))
    dev = torch.device("cuda")
    T = {np.float32: torch.float32, np.float64: torch.float64}[dtype.type]
    def pk(x):
        t = torch.zeros((n, 4), dtype=T)
        t[:, :3] = torch.from_numpy(x)
        return t.to(dev)
    tv, t1, t0 = pk(v), pk(a1), pk(a0)
    sfx = "_f32" if prec == "single" else "_f64"
    _native.call("nb_dev_kick" + sfx, tv.data_ptr(), t1.data_ptr(), t0.data_ptr(), n, 0.5 * 1e-3, 0)
    got = tv[:, :3].cpu().numpy()
    vx, vy, vz = (np.ascontiguousarray(v[:, k]) for k in range(3))
    oracle.kick(vx, vy, vz, [np.ascontiguousarray(a1[:, k]) for k in range(3)],
                [np.ascontiguousarray(a0[:, k]) for k in range(3)], 0.5 * 1e-3)
    np.testing.assert_array_equal(got, np.stack([vx, vy, vz], 1))


@pytest.mark.parametrize("prec", ["double", "single"])
def test_fused_step_matches_manual_pass_bitwise(prec, monkeypatch):
    """pkg/tests/test_kernels.py:153-166: one-step positions equal a manual
    compute_accelerations + integrate_step pass, bit for bit (the fused
    epilogue runs the same rounding sequence as the stand-alone update).  The
    small-N kernel sums the forces in another order, so it is off here."""
    monkeypatch.setenv("NB_SMALL_MAX_N", "0")
    s = cube(2000, 4, prec)
    p = nb.SimParams(1.0, 1e-3, 1e-3, 1)
    manual = s.copy()
    acc = accel_of(manual, p)
    nb.integrate_step(manual, acc, p)
    fin = nb.simulate(s, p)
    for u, v in zip(fin.positions, manual.positions):
        np.testing.assert_array_equal(u, v)


# --------------------------------------------------------------------------- simulate contract

def test_simulate_leaves_input_untouched():
    s = nb.init_system(16, nb.Seed(1))
    before = [c.copy() for c in s.positions]
    nb.simulate(s, nb.SimParams(1.0, 0.01, 1e-9, 10), nb.reference_variant())
    for u, v in zip(before, s.positions):
        assert np.array_equal(u, v)


def test_simulate_aos_equals_soa():
    s = cube(300, 9, "double")
    p = nb.SimParams(1.0, 1e-3, 1e-3, 4)
    a = nb.simulate(s, p)
    b = nb.simulate(nb.convert_layout(s, nb.Layout.AOS), p, nb.KernelVariant(nb.Layout.AOS))
    assert b.layout is nb.Layout.AOS
    np.testing.assert_array_equal(a.position_matrix(), b.position_matrix())


def test_variant_layout_mismatch_rejected():
    with pytest.raises(ValueError):
        nb.simulate(two_body(layout=nb.Layout.AOS), EPS0, nb.reference_variant())
    with pytest.raises(ValueError):
        nb.simulate(two_body(), EPS0, nb.KernelVariant(nb.Layout.SOA, block=8))


def test_two_body_mirror_symmetry():
    fin = nb.simulate(two_body(), nb.SimParams(1.0, 0.01, 1e-9, 50), nb.reference_variant())
    x, y, z = fin.positions
    np.testing.assert_allclose(x[0] + x[1], 1.0, atol=1e-14)
    np.testing.assert_allclose(y[0] + y[1], 0.0, atol=1e-14)
    np.testing.assert_allclose(z[0] + z[1], 0.0, atol=1e-14)


def test_momentum_conserved_from_rest():
    s = nb.init_system(256, nb.Seed(42))
    fin = nb.simulate(s, nb.SimParams(1.0, 0.01, 1e-9, 100))
    m = fin.masses
    v = np.stack(fin.velocities, axis=1)
    assert np.linalg.norm(m @ v) <= 1e-9 * float(np.sum(m * np.linalg.norm(v, axis=1)))


def test_integrate_direct_substitution():
    """pkg/tests/test_kernels.py:118-124: dv = a*dt, dp = (v_old + dv/2)*dt, exact."""
    s = nb.system_from_arrays([[0.0, 0.0, 0.0]], np.zeros((1, 3)), [1.0])
    acc = nb.AccelerationBuffer.allocate(1, nb.Precision.DOUBLE)
    acc.x[0] = 1.0
    nb.integrate_step(s, acc, nb.SimParams(1.0, 1.0, 1e-9, 1), nb.reference_variant())
    assert s.velocities[0][0] == 1.0
    assert s.positions[0][0] == 0.5


def test_integrate_two_body_first_step():
    """pkg/tests/test_kernels.py:127-140: the first kick-drift of the unit
    two-body system, expected values as the update rule evaluates them."""
    s = two_body()
    params = nb.SimParams(1.0, 0.1, 0.0, 1)
    acc = accel_of(s, params)
    nb.integrate_step(s, acc, params, nb.reference_variant())
    assert s.velocities[0][0] == 0.1 and s.velocities[0][1] == -0.1
    assert s.positions[0][0] == (0.0 + 0.5 * 0.1) * 0.1
    assert s.positions[0][1] == 1.0 + (0.0 + 0.5 * -0.1) * 0.1


LADDER_SUBSET = [
    nb.KernelVariant(nb.Layout.SOA, nb.MathForm.RECIPROCAL_MULTIPLY),
    nb.KernelVariant(nb.Layout.SOA, block=8),
    nb.KernelVariant(nb.Layout.SOA, block=64),
    nb.KernelVariant(nb.Layout.SOA, block=128),
    nb.KernelVariant(nb.Layout.SOA, nb.MathForm.RECIPROCAL_MULTIPLY, 32, 2),
    nb.KernelVariant(nb.Layout.SOA, threads=4),
    nb.KernelVariant(nb.Layout.AOS),
]


@pytest.mark.parametrize("variant", LADDER_SUBSET, ids=lambda v: f"{v.name}-T{v.threads}")
def test_variant_equivalence_small(variant, oracle):
    """pkg/tests/test_kernels.py:190-201 and :212-217 on the GPU path: every
    ladder rung reproduces the FP64 reference checksum (the oracle's simulate of
    the same state) within 1e-9 in FP64 and 5e-4 in FP32."""
    params = nb.SimParams(1.0, 0.01, 1e-9, 10)
    s64 = nb.init_system(192, nb.Seed(42))
    fin, _ = oracle.simulate(s64.position_matrix(), np.stack(s64.velocities, 1), s64.masses, 1.0, 0.01, 1e-9, 10,
                             recip=False)
    ref = oracle.checksum(fin)
    got = nb.checksum(nb.simulate(nb.init_system(192, nb.Seed(42), nb.Precision.DOUBLE, variant.layout),
                                  params, variant))
    assert abs(got - ref) / abs(ref) <= 1e-9
    got32 = nb.checksum(nb.simulate(nb.init_system(192, nb.Seed(42), nb.Precision.SINGLE, variant.layout),
                                    params, variant))
    assert abs(got32 - ref) / abs(ref) <= 5e-4


def test_two_body_energy_drift():
    """pkg/tests/test_acceptance.py:80-86 on the GPU path: unit two-body system,
    dt = 1e-3, 100 steps, |E1 - E0| / |E0| <= 1e-4, energies from the GPU
    diagnostics pass."""
    params = nb.SimParams(1.0, 1e-3, 1e-9, 100)
    e0 = nb.diagnostics_gpu(two_body(), params)["total"]
    e1 = nb.diagnostics_gpu(nb.simulate(two_body(), params, nb.reference_variant()), params)["total"]
    assert abs(e1 - e0) / abs(e0) <= 1e-4


def test_second_order_convergence(oracle):
    """pkg/tests/test_acceptance.py:88-100 on the GPU path: halving dt shrinks the
    position error against a dt/2048 FP64 run (the oracle's simulate) by a factor
    in [3, 5] -- velocity Verlet is second order."""
    eps2, total = 0.25, 1.0
    s = two_body()
    fine, _ = oracle.simulate(s.position_matrix(), np.stack(s.velocities, 1), s.masses, 1.0, total / 2048, eps2,
                              2048)
    err = [float(np.max(np.abs(nb.simulate(two_body(), nb.SimParams(1.0, total / k, eps2, k),
                                           nb.reference_variant()).position_matrix() - fine)))
           for k in (128, 256)]
    assert 3.0 <= err[0] / err[1] <= 5.0, err


@pytest.mark.parametrize("prec,n", [("double", 20000), ("single", 20000), ("single", 70000)])
def test_runs_are_bitwise_reproducible(prec, n):
    """Also covers the TMA-staged FP32 path (N >= 65536)."""
    s = cube(n, 8, prec)
    p = nb.SimParams(1.0, 1e-3, 1e-3, 3)
    a = nb.simulate(s, p).position_matrix()
    b = nb.simulate(s, p).position_matrix()
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("n,eps2", [(1000, 1e-3), (5000, 1e-3), (3000, 0.0), (8000, 1e-3)])
def test_persistent_simulate_matches_per_launch(prec, n, eps2, monkeypatch):
    """Small N runs the whole loop in one cooperative launch (simulate_kernel);
    nb_dev_simulate_timed always launches per step.  Same decomposition and
    partial-sum order: bitwise identical results.  (The small-N kernel, which
    sums in another order, is switched off here and tested below.)"""
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    monkeypatch.setenv("NB_SMALL_MAX_N", "0")
    s = cube(n, 12, prec)
    dt_ = s.precision.dtype
    a = DeviceState(s.position_matrix().astype(dt_), np.stack(s.velocities, 1), s.masses, dt_)
    b = DeviceState(s.position_matrix().astype(dt_), np.stack(s.velocities, 1), s.masses, dt_)
    f = kernel_flags(s.masses, eps2, dt_)
    a.simulate(1.0, 1e-3, eps2, 5, f)
    ms = b.simulate_timed(1.0, 1e-3, eps2, 5, f)
    assert len(ms) == 6 and all(t > 0 for t in ms)
    np.testing.assert_array_equal(a.positions_host(), b.positions_host())
    np.testing.assert_array_equal(a.velocities_host(), b.velocities_host())


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("n,eps2,uniform", [(1, 1e-3, False), (17, 1e-3, False), (1024, 1e-2, False),
                                            (1000, 0.0, False), (2048, 1e-3, True), (2048, 1e-3, False),
                                            (4096, 1e-3, False), (3001, 0.0, True)])
def test_small_simulate_kernel(prec, n, eps2, uniform, oracle, monkeypatch):
    """The small-N cooperative kernel (source split inside the CTA, no global
    partials): against the stream-K per-launch path (another summation order:
    tolerance, not bits), against the FP64 oracle, and bitwise run to run."""
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    s = cube(n, 21, prec)
    dt_ = s.precision.dtype
    masses = np.full(n, 0.75, dtype=dt_) if uniform else s.masses
    pos, vel = s.position_matrix().astype(dt_), np.stack(s.velocities, 1)
    f = kernel_flags(masses, eps2, dt_)
    if eps2 == 0.0:
        assert f & 1
    if uniform:
        assert f & 2

    def run(small):
        monkeypatch.setenv("NB_SMALL_MAX_N", "1000000000" if small else "0")
        st = DeviceState(pos, vel, masses, dt_)
        st.simulate(1.0, 1e-3, eps2, 4, f)
        return st.positions_host(), st.velocities_host()

    p1, v1 = run(True)
    p2, v2 = run(True)
    np.testing.assert_array_equal(p1, p2)
    np.testing.assert_array_equal(v1, v2)
    p3, v3 = run(False)
    ref_pos, _ = oracle.simulate(pos.astype(np.float64), vel.astype(np.float64), masses.astype(np.float64), 1.0, 1e-3,
                                 eps2, 4, threads=oracle.host_threads())
    d_path, d_small, d_sk = (oracle.position_dev(p1, p3), oracle.position_dev(p1, ref_pos),
                             oracle.position_dev(p3, ref_pos))
    print(f"{prec} n={n} eps2={eps2} small-vs-streamK {d_path:.2e} small-vs-oracle {d_small:.2e} "
          f"streamK-vs-oracle {d_sk:.2e}")
    if prec == "double":
        assert d_path <= F64_POS_TOL and d_small <= F64_POS_TOL
    else:  # FP32: no further from the FP64 oracle than the stream-K path (or within 2e-5)
        assert d_small <= max(2e-5, 2 * d_sk)
        assert d_path <= max(2e-5, 2 * d_sk)


def test_exchange_c_abi_single_gpu():
    """nb_comm_* (the NCCL position exchange behind the C ABI) on the one GPU
    this run has: unique id -> a 1-rank communicator -> in-place all-gather of
    packed rows (nothing to receive: the buffer is unchanged) -> destroy; and
    the single-process set-up (ncclCommInitAll) with its grouped all-gather."""
    import ctypes
    import torch
    t = torch.arange(64 * 4, dtype=torch.float32, device="cuda").reshape(64, 4)
    want = t.clone()
    stream = torch.cuda.current_stream().cuda_stream
    comm = _native.comm_init_rank(1, 0, _native.comm_unique_id())
    _native.comm_allgather(t.data_ptr(), t.numel() * 4, comm, stream)
    torch.cuda.synchronize()
    assert torch.equal(t, want)
    _native.comm_destroy(comm)
    comms = (ctypes.c_void_p * 1)()
    devs = (ctypes.c_int * 1)(torch.cuda.current_device())
    _native.call("nb_comm_init_all", 1, devs, comms)
    bufs = (ctypes.c_void_p * 1)(t.data_ptr())
    streams = (ctypes.c_void_p * 1)(stream)
    _native.call("nb_comm_allgather_all", bufs, t.numel() * 4, comms, streams, 1)
    torch.cuda.synchronize()
    assert torch.equal(t, want)
    _native.comm_destroy(comms[0])


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("n", [2560, 2561, 4096, 4097, 8192, 8193])
def test_simulate_path_boundaries(prec, n, oracle):
    """simulate() switches kernels with N (small-N cooperative kernel up to
    3584 FP32 / 2560 FP64, cluster kernels or the stream-K persistent kernel up to 8192, per-step
    launches beyond): trajectories on both sides of each switch agree with the
    FP64 oracle."""
    s = cube(n, 11, prec)
    fin = nb.simulate(s, nb.SimParams(1.0, 1e-3, 1e-3, 3))
    ref, _ = oracle.simulate(s.position_matrix().astype(np.float64), np.stack(s.velocities, 1).astype(np.float64),
                             s.masses.astype(np.float64), 1.0, 1e-3, 1e-3, 3, threads=oracle.host_threads())
    dev = oracle.position_dev(fin.position_matrix(), ref)
    assert dev <= (F64_POS_TOL if prec == "double" else 2e-5), dev


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("eps2", [1e-3, 0.0])
def test_separate_force_and_update_match_fused(prec, eps2, monkeypatch):
    """SURVEY 8(b)'s proposed pair: nb_force then nb_update each step (two acc
    buffers, the host schedules the modes) equals the fused per-step path of
    nb_dev_simulate bit for bit -- same force decomposition, same rounding
    sequence in the update."""
    import torch
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    from paper_2203_08263_b200._native import NB_STEP_FIRST, NB_STEP_KICK_DRIFT, NB_STEP_FINAL_KICK
    monkeypatch.setenv("NB_SMALL_MAX_N", "0")
    monkeypatch.setenv("NB_PERSISTENT_MAX_N", "0")
    n, steps, dt = 3000, 4, 1e-3
    s = cube(n, 17, prec)
    dtype = s.precision.dtype
    pos, vel = s.position_matrix().astype(dtype), np.stack(s.velocities, 1)
    fused = DeviceState(pos, vel, s.masses, dtype)
    fused.simulate(1.0, dt, eps2, steps, kernel_flags(s.masses, eps2, dtype))
    st = DeviceState(pos, vel, s.masses, dtype)
    sfx = st.sfx
    stream = torch.cuda.current_stream().cuda_stream
    acc = [torch.zeros_like(st.acc), torch.zeros_like(st.acc)]
    cur, nxt = st.pos_a, st.pos_b
    for k in range(steps + 1):
        mode = NB_STEP_FIRST if k == 0 else (NB_STEP_KICK_DRIFT if k < steps else NB_STEP_FINAL_KICK)
        a_new, a_old = acc[k % 2], acc[(k + 1) % 2]
        _native.call("nb_force" + sfx, cur.data_ptr(), n, 0, n, eps2, 1.0, a_new.data_ptr(), st.ws.data_ptr(),
                     st.ws_bytes, stream)
        _native.call("nb_update" + sfx, nxt.data_ptr(), cur.data_ptr(), st.vel.data_ptr(), a_new.data_ptr(),
                     a_old.data_ptr(), n, dt, mode, stream)
        if mode != NB_STEP_FINAL_KICK:
            cur, nxt = nxt, cur
    torch.cuda.synchronize()
    # the final kick writes pos_next = pos_cur: compare the state the fused path reports
    np.testing.assert_array_equal(cur[:, :3].cpu().numpy(), fused.positions_host())
    np.testing.assert_array_equal(st.vel[:, :3].cpu().numpy(), fused.velocities_host())
    np.testing.assert_array_equal(acc[steps % 2][:, :3].cpu().numpy(), fused.acc[:, :3].cpu().numpy())


def test_native_kernels_launched():
    before = _native.launch_count()
    nb.simulate(cube(64, 1, "single"), nb.SimParams(1.0, 1e-3, 1e-3, 2))
    assert _native.launch_count() - before >= 1  # small N: one persistent launch


# --------------------------------------------------------------------------- sizes & edges

RAGGED = [1, 2, 3, 5, 31, 127, 128, 129, 255, 256, 257, 1023, 1024, 1025, 3001, 5000]


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("n", RAGGED)
def test_ragged_sizes(prec, n, oracle):
    s = cube(n, 100 + n, prec)
    eps2 = 1e-3
    a = as_mat(accel_of(s, nb.SimParams(1.0, 1e-3, eps2, 1)))
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)),
                                s.masses.astype(np.float64), np.arange(n), 1.0, eps2)
    if n == 1:
        assert np.all(a == 0)
        return
    tol = F64_ACC_TOL if prec == "double" else F32_ACC_TOL
    assert nb_accel_dev(a, want) <= tol


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("g", [2.5, 6.674e-11])
@pytest.mark.parametrize("n", [700, 5000])
def test_gravitational_constant(prec, g, n, oracle):
    """G != 1 (SimParams.gravitational_constant; accel_soa scales by G,
    _accel_cy.pyx:149-152): accelerations against the oracle with the same G,
    and a short trajectory (small-N kernel at n=700, stream-K at n=5000)."""
    s = cube(n, 3 * n, prec)
    eps2 = 1e-3
    a = as_mat(accel_of(s, nb.SimParams(g, 1e-3, eps2, 1)))
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)),
                                s.masses.astype(np.float64), np.arange(n), g, eps2)
    assert nb_accel_dev(a, want) <= (F64_ACC_TOL if prec == "double" else F32_ACC_TOL)
    # dt chosen so G*dt^2 moves bodies by a comparable amount for both G
    dt = 1e-3 / np.sqrt(g)
    fin = nb.simulate(s, nb.SimParams(g, dt, eps2, 3))
    ref, _ = oracle.simulate(pos.astype(np.float64), np.stack(s.velocities, 1).astype(np.float64),
                             s.masses.astype(np.float64), g, dt, eps2, 3, threads=oracle.host_threads())
    dev = oracle.position_dev(fin.position_matrix(), ref)
    assert dev <= (F64_POS_TOL if prec == "double" else 2e-5), dev


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("n", [2, 130, 1025, 4099])
def test_zero_softening_excludes_self(prec, n, oracle):
    s = cube(n, 7 * n, prec)
    a = as_mat(accel_of(s, nb.SimParams(1.0, 1e-3, 0.0, 1)))
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)),
                                s.masses.astype(np.float64), np.arange(n), 1.0, 0.0)
    assert np.all(np.isfinite(a))
    tol = 1e-11 if prec == "double" else 1e-4  # unsoftened: condition number is unbounded
    assert nb_accel_dev(a, want) <= tol


@pytest.mark.parametrize("cfg_name", ["C2", "C3-f32", "C3-f64", "C4", "C5"])
def test_full_size_accelerations_row_sampled(cfg_name, oracle):
    """BASELINE sizes (up to C5's 4,194,304 bodies, the maximum size): 192 rows
    (first, last, random; 48 at C5) of the initial accelerations against the
    long-double oracle."""
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    s = cfg.system()
    a = as_mat(accel_of(s, cfg.params()))
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([[0, 1, cfg.n - 1], rng.integers(0, cfg.n, 45 if cfg_name == "C5" else 189)]))
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)),
                                s.masses.astype(np.float64), rows, 1.0, cfg.softening_sq)
    tol = F64_ACC_TOL if cfg.precision is nb.Precision.DOUBLE else F32_ACC_TOL
    dev = nb_accel_dev(a[rows], want)
    print(cfg_name, "accel_dev", dev)
    assert dev <= tol


def _wrapping_split_accelerations(n=70001):
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    n = 70001
    s = cube(n, 44, "single")
    st = DeviceState(s.position_matrix().astype(np.float32), np.stack(s.velocities, 1), s.masses, np.float32)
    f = kernel_flags(s.masses, 1e-3, np.float32)
    out = __import__("torch").zeros((n, 4), dtype=__import__("torch").float32, device="cuda")
    split = 12345  # phase 1: sources [12345, 12345+65537) mod n wraps; phase 2: the rest
    st.step(1.0, 1e-3, 0.0, 0, f, j_begin=split, j_count=65537, carry_mode=1, acc_out=out)
    st.step(1.0, 1e-3, 0.0, 0, f, j_begin=(split + 65537) % n, j_count=n - 65537, carry_mode=2, acc_out=out)
    return s, out[:, :3].cpu().numpy()


def test_split_wrapping_source_ranges(oracle):
    """A circular source range that wraps past N (the multi-GPU second phase),
    split at an odd offset into two carry phases, against the oracle."""
    s, got = _wrapping_split_accelerations()
    rows = np.arange(0, s.count, 701)
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)), s.masses, rows, 1.0, 1e-3)
    assert nb_accel_dev(got[rows], want) <= F32_ACC_TOL


def test_tma_staging_option(tmp_path):
    """NB_TMA=1: source tiles staged by cp.async.bulk on mbarriers (two copies
    per tile when the source range wraps); same accuracy, deterministic."""
    import subprocess, sys, textwrap
    script = textwrap.dedent(f"""
        import os, sys, numpy as np
        sys.path.insert(0, {REPO!r}); sys.path.insert(0, {os.path.join(REPO, "tests")!r})
        import test_gpu_parity as T
        from oracle import oracle as O
        s, a = T._wrapping_split_accelerations()
        _, b = T._wrapping_split_accelerations()
        assert np.array_equal(a, b)
        rows = np.arange(0, s.count, 701)
        pos = s.position_matrix()
        want = O.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)), s.masses, rows, 1.0, 1e-3)
        dev = O.accel_dev(a[rows], want)
        print("DEV", dev)
        assert dev <= 1e-5, dev
    """)
    env = dict(os.environ, NB_TMA="1")
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("cfg_name", ["C2", "C3-f32", "C3-f64"])
def test_full_size_trajectory_vs_oracle(cfg_name, oracle):
    """SURVEY.md 8(c) trajectory tolerances at full BASELINE size: the whole
    simulate against the FP64 oracle port (all host cores) on the same rounded
    inputs -- FP64 within 1e-12; FP32 within 10x the reference's own FP32-vs-FP64
    deviation (the reference's recip-form FP32 run, reproduced bit for bit by the
    port)."""
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    s = cfg.system()
    p = cfg.params()
    fin = nb.simulate(s, p).position_matrix()
    pos64 = s.position_matrix()
    vel64 = np.stack(s.velocities, 1).astype(np.float64)
    th = oracle.host_threads()
    ref64, _ = oracle.simulate(pos64, vel64, s.masses.astype(np.float64), 1.0, p.dt, p.softening_sq, p.steps,
                               threads=th)
    dev = oracle.position_dev(fin, ref64)
    if cfg.precision is nb.Precision.DOUBLE:
        assert dev <= F64_POS_TOL, dev
    else:
        ref32, _ = oracle.simulate(np.stack(s.positions, 1), np.stack(s.velocities, 1), s.masses, 1.0, p.dt,
                                   p.softening_sq, p.steps, threads=th)
        ref_dev = oracle.position_dev(ref32, ref64)
        print(cfg_name, "gpu", dev, "reference fp32", ref_dev)
        assert dev <= 10 * ref_dev, (dev, ref_dev)


def test_plummer_row_sampled(oracle):
    """C5's distribution (Plummer, equal masses) at 1/16 of its N."""
    s = nb.plummer_sphere(262144, 0, nb.Precision.SINGLE)
    a = as_mat(accel_of(s, nb.SimParams(1.0, 1e-4, 1e-4, 1)))
    rows = np.random.default_rng(2).integers(0, 262144, 64)
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)),
                                s.masses.astype(np.float64), rows, 1.0, 1e-4)
    assert nb_accel_dev(a[rows], want) <= F32_ACC_TOL


def test_full_size_trajectory_properties():
    """C3-f32 at full size: finite, deterministic, and momentum stays at the
    rounding level of its initial value (a size-independent property)."""
    cfg = nb.BASELINE_CONFIGS["C3-f32"]
    s = cfg.system()
    fin = nb.simulate(s, cfg.params())
    v = np.stack(fin.velocities, 1).astype(np.float64)
    v0 = np.stack(s.velocities, 1).astype(np.float64)
    m = fin.masses.astype(np.float64)
    assert np.all(np.isfinite(v)) and np.all(np.isfinite(fin.position_matrix()))
    p0, p1 = m @ v0, m @ v
    scale = float(np.sum(m * np.linalg.norm(v, axis=1)))
    assert np.linalg.norm(p1 - p0) <= 1e-5 * scale


@pytest.mark.parametrize("config", ["C3-f32", "C4"])
def test_full_size_energy_conservation(config):
    """BASELINE sizes (C3-f32 N=131072, C4 N=524288 FP64): total energy from the
    FP64 diagnostics pass drifts by at most 1e-4 relative (the reference's
    acceptance bound, pkg/tests/test_acceptance.py:80-86, here at full size where
    the reference's O(N^2) Python diagnostics cannot run).  The BASELINE dt
    (1e-3) does not resolve these systems' collapse -- |a| ~ N/R^2 ~ 1e5, the
    dynamical time ~3e-3 -- so energy is not conserved at that dt on any
    implementation; the check runs the same states with dt = 1e-6."""
    cfg = nb.BASELINE_CONFIGS[config]
    s = cfg.system()
    p = nb.SimParams(1.0, 1e-6, cfg.softening_sq, 10)
    e0 = nb.diagnostics_gpu(s, p)
    fin = nb.simulate(s, p)
    e1 = nb.diagnostics_gpu(fin, p)
    drift = abs(e1["total"] - e0["total"]) / abs(e0["total"])
    print(f"{config}: E0 {e0['total']:.12e} E1 {e1['total']:.12e} drift {drift:.3e}")
    # measured 2.5e-10 (C3-f32) and 1.6e-12 (C4): assert 100x inside the reference bound
    assert np.isfinite(e1["total"]) and drift <= 1e-6


# --------------------------------------------------------------------------- sharding on one GPU

@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_driver_on_one_gpu(prec, world):
    """The multi-GPU step loop with P emulated ranks on one device, run in lock
    step (no rank waits on another's kernel): every rank owns an i-shard, sums
    its local sources into the FP64 carry, then the rest; positions are
    exchanged by copying rows (the all-gather)."""
    from paper_2203_08263_b200.device import DeviceState, needs_self_mask
    from paper_2203_08263_b200.sharded import pad_system, shard_range
    from paper_2203_08263_b200._native import NB_STEP_FIRST, NB_STEP_KICK_DRIFT, NB_STEP_FINAL_KICK
    s = cube(3000, 21, prec)
    p = nb.SimParams(1.0, 1e-3, 1e-3, 4)
    ref = nb.simulate(s, p)
    dtype = s.precision.dtype
    pos, vel, m = pad_system(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, world)
    npad = pos.shape[0]
    ranks = []
    for r in range(world):
        i0, ni = shard_range(npad, r, world)
        ranks.append(DeviceState(pos, vel, m, dtype, i_begin=i0, n_i=ni))
    mask = needs_self_mask(m[: s.count], p.softening_sq, dtype)
    for step in range(p.steps + 1):
        mode = NB_STEP_FIRST if step == 0 else (NB_STEP_KICK_DRIFT if step < p.steps else NB_STEP_FINAL_KICK)
        for st in ranks:
            st.step(1.0, p.softening_sq, p.dt, mode, mask, j_begin=st.i_begin, j_count=st.n_i, carry_mode=1)
            st.step(1.0, p.softening_sq, p.dt, mode, mask, j_begin=(st.i_begin + st.n_i) % npad,
                    j_count=npad - st.n_i, carry_mode=2)
        if mode != NB_STEP_FINAL_KICK:
            for st in ranks:
                st.swap()
            for st in ranks:
                for src in ranks:
                    sl = slice(src.i_begin, src.i_begin + src.n_i)
                    st.pos_cur[sl] = src.pos_cur[sl]
    got = ranks[0].pos_cur[: s.count, :3].cpu().numpy().astype(np.float64)
    tol = 1e-13 if prec == "double" else 1e-6
    from oracle.oracle import position_dev
    assert position_dev(got, ref.position_matrix()) <= tol


@pytest.mark.parametrize("prec", ["double", "single"])
def test_uniform_mass_path_matches_general_path(prec, oracle):
    """NB_FLAG_UNIFORM_MASS (m applied once per body, used automatically for
    equal-mass systems such as C5's Plummer sphere) agrees with the general
    per-pair-mass kernel and with the oracle."""
    from paper_2203_08263_b200.device import DeviceState
    from paper_2203_08263_b200._native import NB_FLAG_UNIFORM_MASS
    s = nb.plummer_sphere(20000, 3, nb.Precision(prec))
    dtype = s.precision.dtype
    st = DeviceState(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, dtype)
    a_gen = st.accelerations(1.0, 1e-4, 0)[:, :3].cpu().numpy().astype(np.float64)
    a_uni = st.accelerations(1.0, 1e-4, NB_FLAG_UNIFORM_MASS)[:, :3].cpu().numpy().astype(np.float64)
    rows = np.arange(0, 20000, 97)
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)), s.masses, rows, 1.0, 1e-4)
    tol = F64_ACC_TOL if prec == "double" else F32_ACC_TOL
    assert nb_accel_dev(a_uni[rows], want) <= tol
    assert nb_accel_dev(a_gen[rows], want) <= tol
    assert nb_accel_dev(a_uni, a_gen) <= (1e-14 if prec == "double" else 2e-6)


@pytest.mark.parametrize("prec", ["double", "single"])
def test_device_generators_match_host(prec):
    """nb_dev_init: the uniform cube is bit-identical to core.uniform_cube; the
    Plummer sphere (libm pow/sincos on the device) agrees to <= 2 ulp."""
    from paper_2203_08263_b200.device import DeviceState
    n = 100003
    dtype = np.dtype(np.float32 if prec == "single" else np.float64)
    st = DeviceState.from_generator("uniform_cube", n, 7, dtype)
    host = nb.uniform_cube(n, 7, nb.Precision(prec))
    np.testing.assert_array_equal(st.positions_host(), host.position_matrix().astype(dtype))
    np.testing.assert_array_equal(st.velocities_host(), np.stack(host.velocities, 1))
    np.testing.assert_array_equal(st.masses_host(), host.masses)
    pl = DeviceState.from_generator("plummer_sphere", n, 7, dtype)
    hp = nb.plummer_sphere(n, 7, nb.Precision(prec))
    got, want = pl.positions_host().astype(np.float64), hp.position_matrix()
    # component errors measured in ulps of the body's radius (a component near 0
    # inherits the absolute error of cos/sin, not a relative one)
    # r = (u^(-2/3) - 1)^(-1/2) is ill-conditioned as u -> 1 (r -> infinity), so a
    # 1-ulp pow difference can grow there: bound all bodies loosely, the bulk tightly.
    # condition number of r in w = u^(-2/3): |d ln r / d ln w| = w / (2 (w - 1)).
    from paper_2203_08263_b200.core import unit_stream
    u = np.maximum(unit_stream(7, 3 * n).reshape(n, 3)[:, 0], 2.0 ** -53)
    w = u ** (-2.0 / 3.0)
    cond = 1.0 + w / (2.0 * (w - 1.0))
    norm = np.linalg.norm(want, axis=1)
    eps = float(np.finfo(dtype).eps)
    rel = np.max(np.abs(got - want), axis=1) / norm
    assert np.all(rel <= 8 * eps * cond), float(np.max(rel / (eps * cond)))
    np.testing.assert_array_equal(pl.masses_host(), hp.masses)


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("world", [2, 4])
def test_peer_store_epilogue_on_one_gpu(prec, world):
    """nb_dev_step_p2p: P emulated ranks on one device in lock step; each rank's
    remote-source pass stores its drifted rows straight into every other rank's
    next-position buffer (the fused exchange; no all-gather).  Sequential launches
    on one stream stand in for the cross-GPU barrier."""
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    from paper_2203_08263_b200.sharded import pad_system, shard_range
    from paper_2203_08263_b200._native import NB_STEP_FIRST, NB_STEP_KICK_DRIFT, NB_STEP_FINAL_KICK
    from oracle.oracle import position_dev
    s = cube(2500, 33, prec)
    p = nb.SimParams(1.0, 1e-3, 1e-3, 4)
    ref = nb.simulate(s, p)
    dtype = s.precision.dtype
    pos, vel, m = pad_system(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, world)
    npad = pos.shape[0]
    ranks = [DeviceState(pos, vel, m, dtype, i_begin=shard_range(npad, r, world)[0],
                         n_i=shard_range(npad, r, world)[1]) for r in range(world)]
    flags = kernel_flags(m, p.softening_sq, dtype)
    for step in range(p.steps + 1):
        mode = NB_STEP_FIRST if step == 0 else (NB_STEP_KICK_DRIFT if step < p.steps else NB_STEP_FINAL_KICK)
        for st in ranks:
            st.step(1.0, p.softening_sq, p.dt, mode, flags, j_begin=st.i_begin, j_count=st.n_i, carry_mode=1)
        for st in ranks:
            peers = None if mode == NB_STEP_FINAL_KICK else [q.pos_next.data_ptr() for q in ranks if q is not st]
            st.step(1.0, p.softening_sq, p.dt, mode, flags, j_begin=(st.i_begin + st.n_i) % npad,
                    j_count=npad - st.n_i, carry_mode=2, peers=peers)
        if mode != NB_STEP_FINAL_KICK:
            for st in ranks:
                st.swap()
    tol = 1e-13 if prec == "double" else 1e-6
    for st in ranks:  # every rank holds every row
        got = st.pos_cur[: s.count, :3].cpu().numpy().astype(np.float64)
        assert position_dev(got, ref.position_matrix()) <= tol


def test_symmetric_memory_p2p_path_single_rank(tmp_path):
    """The symmetric-memory plumbing of transport="p2p" (allocation, rendezvous,
    device barrier) on a 1-rank NCCL group, in a subprocess."""
    import subprocess, sys, textwrap, socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    script = textwrap.dedent(f"""
        import os, sys, numpy as np, torch, torch.distributed as dist
        sys.path.insert(0, {REPO!r})
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="{port}", RANK="0", WORLD_SIZE="1")
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
        import paper_2203_08263_b200 as nb
        from paper_2203_08263_b200.sharded import simulate_sharded
        s = nb.uniform_cube(3000, 5, nb.Precision.SINGLE)
        pos, vel = simulate_sharded(s.position_matrix().astype(np.float32), np.stack(s.velocities, 1),
                                    s.masses, np.float32, 1.0, 1e-3, 1e-3, 3, transport="p2p")
        ref = nb.simulate(s, nb.SimParams(1.0, 1e-3, 1e-3, 3)).position_matrix()
        err = float(np.max(np.abs(pos - ref)))
        dist.destroy_process_group()
        print("ERR", err)
        assert err <= 1e-6, err
    """)
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


# --------------------------------------------------------------------------- plugin + diagnostics

@pytest.mark.parametrize("prec", ["double", "single"])
def test_backend_plugin_protocol(prec, oracle):
    from paper_2203_08263_b200 import backend
    s = cube(513, 17, prec)
    px, py, pz = (c.copy() for c in s.positions)
    ax, ay, az = (np.zeros(513, s.precision.dtype) for _ in range(3))
    backend.accel_soa(px, py, pz, s.masses, 1.0, 1e-3, True, 0, 1, ax, ay, az)
    want = oracle.accel_rows_ld(px, py, pz, s.masses.astype(np.float64), np.arange(513), 1.0, 1e-3)
    tol = F64_ACC_TOL if prec == "double" else F32_ACC_TOL
    assert nb_accel_dev(np.stack([ax, ay, az], 1), want) <= tol
    pos = np.ascontiguousarray(np.stack([px, py, pz], 1))
    bx, by, bz = (np.zeros_like(ax) for _ in range(3))
    backend.accel_aos(pos, s.masses, 1.0, 1e-3, bx, by, bz)
    np.testing.assert_array_equal(np.stack([ax, ay, az], 1), np.stack([bx, by, bz], 1))
    vx, vy, vz = (c.copy() for c in s.velocities)
    rpx, rpy, rpz, rvx, rvy, rvz = (c.copy() for c in (px, py, pz, vx, vy, vz))
    backend.step_soa(px, py, pz, vx, vy, vz, ax, ay, az, 1e-3, 4)
    oracle.step_soa(rpx, rpy, rpz, rvx, rvy, rvz, ax, ay, az, 1e-3)
    for u, v in zip((px, py, pz, vx, vy, vz), (rpx, rpy, rpz, rvx, rvy, rvz)):
        np.testing.assert_array_equal(u, v)


def test_backend_simulate_matches_package():
    from paper_2203_08263_b200 import backend
    s = cube(700, 5, "double")
    p = nb.SimParams(1.0, 1e-3, 1e-3, 3)
    cols = [c.copy() for c in s.positions + s.velocities]
    backend.simulate_soa(*cols, s.masses, 1.0, 1e-3, 1e-3, 3)
    np.testing.assert_array_equal(np.stack(cols[:3], 1), nb.simulate(s, p).position_matrix())


@pytest.mark.parametrize("n,prec,eps2", [(2048, "double", 1e-3), (1, "double", 1e-3), (2, "double", 0.0),
                                         (777, "single", 1e-2), (40000, "double", 1e-3), (65537, "single", 1e-4)])
def test_energy_diagnostics(oracle, n, prec, eps2):
    """nb_dev_energy (FP64 potential pass with source ranges + fixed-order
    reduction) against the oracle's long-double diagnostics, ragged sizes, one
    body, eps2 = 0 (self pair masked), FP32 systems upcast."""
    s = cube(n, 31, prec)
    p = nb.SimParams(1.0, 1e-3, eps2, 1)
    d = nb.diagnostics_gpu(s, p)
    want = oracle.diagnostics(s.position_matrix(), np.stack(s.velocities, 1), s.masses, 1.0, eps2)
    assert abs(d["kinetic"] - want["kinetic"]) <= 1e-12 * abs(want["kinetic"])
    assert abs(d["potential"] - want["potential"]) <= 1e-12 * max(abs(want["potential"]), 1e-300)
    if n == 1:
        assert d["potential"] == 0.0
    np.testing.assert_allclose(d["momentum"], want["momentum"], rtol=1e-12, atol=1e-13 * n)


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("shard", [False, True])
def test_column_staging_roundtrip(prec, shard):
    """DeviceState.load (column staging, nb_dev_load_cols) and columns_host
    (nb_dev_store_cols): packed rows equal the input bit for bit from either input
    form, and the columns come back unchanged -- for a sharded state only the
    owned velocity rows."""
    from paper_2203_08263_b200.device import DeviceState
    dtype = np.dtype(np.float32 if prec == "single" else np.float64)
    s = nb.uniform_cube(4099, 3, nb.Precision(prec))
    pos, vel = s.position_matrix().astype(dtype), np.stack(s.velocities, 1)
    lo, ni = (1000, 1500) if shard else (0, None)
    a = DeviceState(pos, vel, s.masses, dtype, i_begin=lo, n_i=ni)
    b = DeviceState(tuple(s.positions), tuple(s.velocities), s.masses, dtype, i_begin=lo, n_i=ni)
    hi = lo + a.n_i
    for st in (a, b):
        rows = st.pos_cur.cpu().numpy()
        np.testing.assert_array_equal(rows[:, :3], pos)
        np.testing.assert_array_equal(rows[:, 3], s.masses)
        v = st.vel.cpu().numpy()[: st.n_i]
        np.testing.assert_array_equal(v[:, :3], vel[lo:hi])
        assert not v[:, 3].any()
        pc, vc = st.columns_host()
        for k in range(3):
            assert pc[k].flags.c_contiguous and vc[k].flags.c_contiguous
            np.testing.assert_array_equal(pc[k], pos[:, k])
            np.testing.assert_array_equal(vc[k], vel[lo:hi, k])
    # reload reuses the staging
    a.load(tuple(s.velocities), tuple(s.positions), s.masses)
    np.testing.assert_array_equal(a.pos_cur.cpu().numpy()[:, :3], vel)
