"""The cluster split-source kernel (pair_kernel: 2-CTA clusters, one i-block of
224 targets per cluster, 16 warp slices of the sources reduced through
distributed shared memory; nbody_force.cu) against the long-double oracle.

It is chosen automatically for FP32 launches whose i-blocks fill one wave of
clusters (C2: N = 16384, and the per-rank size of C3 at 8 GPUs); NB_PAIR=1
forces it wherever the i-blocks fit one wave, so ragged, tiny, self-masked,
uniform-mass and carry (sharded) launches are covered here too.  Tolerance:
the north star's 1e-5 relative per-step acceleration bound
(_accel_dev, validation.py:212-225)."""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

TOL_F32 = 1e-5

SCRIPT = textwrap.dedent(f"""
    import sys, numpy as np
    sys.path.insert(0, {REPO!r})
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    from paper_2203_08263_b200._native import NB_MODE_ACCEL
    out = {{}}
    cases = [("n1", 1, nb.uniform_cube, 1e-3), ("n33", 33, nb.uniform_cube, 1e-3),
             ("n4097", 4097, nb.uniform_cube, 1e-3), ("ragged_self", 12345, nb.uniform_cube, 0.0),
             ("uni", 15000, nb.plummer_sphere, 1e-4), ("c2", 16384, nb.uniform_cube, 1e-2),
             ("full_wave", 16576, nb.uniform_cube, 1e-3),
             # the K family (2..7 targets per lane: 4736 ... 16576 target slots)
             ("k2_full", 4736, nb.uniform_cube, 1e-3), ("k3", 7000, nb.uniform_cube, 1e-3),
             ("k4_self_full", 9472, nb.uniform_cube, 0.0), ("k5", 11111, nb.uniform_cube, 1e-3),
             ("k5_uni", 11000, nb.plummer_sphere, 1e-4), ("k6", 14000, nb.uniform_cube, 1e-2)]
    for name, n, gen, eps2 in cases:
        s = gen(n, 3, nb.Precision.SINGLE)
        pos = s.position_matrix().astype(np.float32)
        st = DeviceState(pos, np.stack(s.velocities, 1), s.masses, np.float32)
        f = kernel_flags(s.masses, eps2, np.float32)
        a = st.accelerations(1.0, eps2, f)[:, :3].cpu().numpy().astype(np.float64)
        a2 = st.accelerations(1.0, eps2, f)[:, :3].cpu().numpy().astype(np.float64)
        out[name] = a
        out[name + "_again"] = a2
        out[name + "_pos"] = np.concatenate([pos, s.masses[:, None].astype(np.float32)], 1)
        out[name + "_eps2"] = np.array([eps2])
    # one rank of a 3-way shard (rows [5000, 10000) of 15000): its own sources
    # into the FP64 carry, then the circular remainder (run_sharded's two phases)
    s = nb.uniform_cube(15000, 4, nb.Precision.SINGLE)
    pos = s.position_matrix().astype(np.float32)
    st = DeviceState(pos, np.stack(s.velocities, 1), s.masses, np.float32, i_begin=5000, n_i=5000)
    f = kernel_flags(s.masses, 1e-3, np.float32)
    st.step(1.0, 1e-3, 0.0, NB_MODE_ACCEL, f, j_begin=5000, j_count=5000, carry_mode=1)
    st.step(1.0, 1e-3, 0.0, NB_MODE_ACCEL, f, j_begin=10000, j_count=10000, carry_mode=2)
    out["shard"] = st.acc[:5000, :3].cpu().numpy().astype(np.float64)
    out["shard_pos"] = np.concatenate([pos, s.masses[:, None].astype(np.float32)], 1)
    out["shard_eps2"] = np.array([1e-3])
    # a 3-step trajectory at C2's size through the public API
    s = nb.uniform_cube(16384, 0, nb.Precision.SINGLE)
    fin = nb.simulate(s, nb.SimParams(1.0, 1e-2, 1e-2, 3))
    out["traj"] = fin.position_matrix().astype(np.float64)
    np.savez(sys.argv[1], **out)
""")

_cache = {}


def _run(tmp_path, pair):
    if pair in _cache:
        return _cache[pair]
    path = tmp_path / f"pair{pair}.npz"
    env = dict(os.environ, NB_PAIR=str(pair))
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(path)], capture_output=True, text=True, timeout=900,
                       env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    _cache[pair] = dict(np.load(path))
    return _cache[pair]


def _rows(n, k=96, seed=5):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, k)]))


@pytest.fixture(scope="module")
def oracle():
    from oracle import oracle as O
    return O


@pytest.mark.parametrize("name", ["n1", "n33", "n4097", "ragged_self", "uni", "c2", "full_wave",
                                  "k2_full", "k3", "k4_self_full", "k5", "k5_uni", "k6"])
def test_forced_pair_kernel_vs_oracle(name, oracle, tmp_path):
    d = _run(tmp_path, 1)
    pos, eps2 = d[name + "_pos"], float(d[name + "_eps2"][0])
    n = pos.shape[0]
    rows = _rows(n)
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(4)), rows, 1.0, eps2)
    got = d[name][rows]
    assert np.all(np.isfinite(d[name]))
    if n == 1:  # a lone body feels nothing
        assert np.all(got == 0.0)
        return
    dev = oracle.accel_dev(got, want)
    print(name, "accel_dev", dev)
    assert dev <= TOL_F32
    np.testing.assert_array_equal(d[name], d[name + "_again"])  # bitwise reproducible


def test_pair_kernel_sharded_carry_vs_oracle(oracle, tmp_path):
    d = _run(tmp_path, 1)
    pos = d["shard_pos"]
    local = _rows(5000)
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(4)), 5000 + local, 1.0, 1e-3)
    dev = oracle.accel_dev(d["shard"][local], want)
    print("shard accel_dev", dev)
    assert dev <= TOL_F32


def test_pair_is_the_default_at_c2_and_stream_k_agrees(oracle, tmp_path):
    """At C2's size the default path IS the pair kernel (its sums differ in the
    last bits from stream-K's, NB_PAIR=0), and both match the oracle; the
    3-step trajectories agree to FP32 rounding."""
    auto = _run(tmp_path, -1)
    pair = _run(tmp_path, 1)
    sk = _run(tmp_path, 0)
    np.testing.assert_array_equal(auto["c2"], pair["c2"])
    assert not np.array_equal(sk["c2"], pair["c2"])
    rows = _rows(16384)
    pos = sk["c2_pos"]
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(4)), rows, 1.0, 1e-2)
    assert oracle.accel_dev(sk["c2"][rows], want) <= TOL_F32
    assert oracle.accel_dev(pair["c2"][rows], want) <= TOL_F32
    np.testing.assert_array_equal(auto["traj"], pair["traj"])
    assert oracle.position_dev(pair["traj"], sk["traj"]) <= 1e-5


def test_k_family_selection():
    """Which force kernel a launch shape takes (nb_dev_step_kernel): the cluster
    kernel with the smallest K that holds the targets, where its slots are filled
    to the measured break-even (DESIGN 3.4); stream-K elsewhere."""
    from paper_2203_08263_b200 import _native
    name = lambda n, j=None: _native.step_kernel_name(4, n, n if j is None else j)
    for n in (3600, 4096, 4097, 4736, 5000, 7104, 8192, 9472, 10600, 11840, 12900, 14208, 15400, 16384, 16576):
        assert name(n) == "pair_kernel", n
    for n in (1000, 3500, 9600, 10000, 12000, 12700, 14500, 15300, 16577, 20000, 131072):
        assert name(n) == "step_kernel", n
    assert name(16384, 131072) == "pair_kernel"   # a rank's shard of C3 at 8 GPUs
    assert name(8192, 1024) == "step_kernel"      # too few sources for 16 slices of one tile
    # FP64 (pair_kernel_f64, K = 2 / 4): above the small-N kernel's range up to 4736, and 8146 ... 9472
    name64 = lambda n, j=None: _native.step_kernel_name(8, n, n if j is None else j)
    for n in (2561, 3072, 4096, 4736, 8192, 9000, 9472):
        assert name64(n) == "pair_kernel", n
    for n in (1024, 2557, 4737, 6144, 8000, 9473, 16384, 131072):
        assert name64(n) == "step_kernel", n
    assert name64(4096, 524288) == "pair_kernel" and name64(4096, 2047) == "step_kernel"


@pytest.mark.parametrize("n,eps2,gen", [(2561, 1e-3, "uniform_cube"), (4096, 1e-3, "uniform_cube"),
                                        (4736, 0.0, "uniform_cube"), (3000, 1e-4, "plummer_sphere"),
                                        (8192, 1e-2, "uniform_cube"), (9472, 0.0, "uniform_cube")])
def test_fp64_cluster_kernel_vs_oracle(n, eps2, gen, oracle):
    """pair_kernel_f64 (the default at these sizes): accelerations against the
    long-double oracle at the north star's FP64 bound, bitwise run to run, and a
    4-step trajectory through simulate() (per-step launches of the cluster kernel)."""
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200 import _native
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    assert _native.step_kernel_name(8, n, n) == "pair_kernel"
    s = getattr(nb, gen)(n, 3, nb.Precision.DOUBLE)
    pos = s.position_matrix()
    st = DeviceState(pos, np.stack(s.velocities, 1), s.masses, np.float64)
    f = kernel_flags(s.masses, eps2, np.float64)
    a = st.accelerations(1.0, eps2, f)[:, :3].cpu().numpy()
    b = st.accelerations(1.0, eps2, f)[:, :3].cpu().numpy()
    np.testing.assert_array_equal(a, b)
    rows = _rows(n)
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)), s.masses, rows, 1.0, eps2)
    dev = oracle.accel_dev(a[rows], want)
    print(n, "accel_dev", dev)
    assert dev <= 1e-12
    p = nb.SimParams(1.0, 1e-4, eps2, 4)
    fin = nb.simulate(s, p).position_matrix()
    ref, _ = oracle.simulate(pos, np.stack(s.velocities, 1), s.masses, 1.0, p.dt, eps2, 4,
                             threads=oracle.host_threads())
    assert oracle.position_dev(fin, ref) <= 1e-12


def test_fp64_cluster_kernel_sharded_carry_vs_oracle(oracle):
    """One rank of a 3-way FP64 shard (rows [3000, 6000) of 9000) through
    pair_kernel_f64: its own sources into the FP64 carry, then the circular
    remainder (run_sharded's two phases), against the long-double oracle."""
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200 import _native
    from paper_2203_08263_b200._native import NB_MODE_ACCEL
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    n, i0, ni = 9000, 3000, 3000
    assert _native.step_kernel_name(8, ni, ni) == "pair_kernel" and _native.step_kernel_name(8, ni, n - ni) == "pair_kernel"
    s = nb.uniform_cube(n, 4, nb.Precision.DOUBLE)
    pos = s.position_matrix()
    st = DeviceState(pos, np.stack(s.velocities, 1), s.masses, np.float64, i_begin=i0, n_i=ni)
    f = kernel_flags(s.masses, 1e-3, np.float64)
    st.step(1.0, 1e-3, 0.0, NB_MODE_ACCEL, f, j_begin=i0, j_count=ni, carry_mode=1)
    st.step(1.0, 1e-3, 0.0, NB_MODE_ACCEL, f, j_begin=i0 + ni, j_count=n - ni, carry_mode=2)
    got = st.acc[:ni, :3].cpu().numpy()
    local = _rows(ni)
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)), s.masses, i0 + local, 1.0, 1e-3)
    dev = oracle.accel_dev(got[local], want)
    print("fp64 shard accel_dev", dev)
    assert dev <= 1e-12
