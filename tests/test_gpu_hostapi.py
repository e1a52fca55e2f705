"""simulate()'s single native call (nb_dev_simulate_cols) against the packed
device-state path (DeviceState.load + simulate + readback) on the same inputs:
bitwise equal -- the small-N kernel reading and writing the host column block
itself, and NB_FLAG_AUTO deriving the kernel flags from the staged masses in C
(exclude-self for eps2 = 0 and for an overflowing self term with a small
uniform mass, uniform-mass for equal masses), at sizes on every simulate path
(small-N kernel, persistent stream-K kernel, per-step launches)."""
import numpy as np
import pytest

import paper_2203_08263_b200 as nb

pytestmark = pytest.mark.gpu


def _packed_path(s, p):
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    dtype = s.precision.dtype
    st = DeviceState(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, dtype)
    st.simulate(p.gravitational_constant, p.dt, p.softening_sq, p.steps, kernel_flags(s.masses, p.softening_sq, dtype))
    return st.positions_host(), st.velocities_host()


CASES = [
    ("cube", 1024, "double", 1e-2), ("cube", 2000, "double", 0.0), ("cube", 3000, "single", 1e-3),
    ("plummer", 3000, "single", 1e-4), ("plummer", 4000, "double", 1e-4), ("cube", 6000, "single", 1e-3),
    ("plummer", 20000, "single", 1e-4), ("cube", 9000, "double", 0.0),
]


@pytest.mark.parametrize("kind,n,prec,eps2", CASES)
def test_columns_call_equals_packed_path(kind, n, prec, eps2):
    gen = nb.uniform_cube if kind == "cube" else nb.plummer_sphere
    s = gen(n, 3, nb.Precision(prec))
    p = nb.SimParams(1.0, 1e-3, eps2, 4)
    fin = nb.simulate(s, p)
    pos, vel = _packed_path(s, p)
    assert np.all(np.isfinite(fin.position_matrix()))
    np.testing.assert_array_equal(fin.position_matrix(), pos.astype(np.float64))
    np.testing.assert_array_equal(np.stack(fin.velocities, 1), vel)


def test_auto_flags_mask_small_uniform_mass():
    """Equal masses of 1e-10 with eps2 = 1e-26 in FP32: the uniform-mass kernel's
    self term eps2^-1.5 = 1e39 overflows, so the self pair must be masked (else
    0 * inf = NaN everywhere) -- the C flag derivation does what the Python one
    does."""
    pos = np.random.default_rng(0).uniform(-1, 1, (512, 3))
    s = nb.system_from_arrays(pos, np.zeros((512, 3)), np.full(512, 1e-10), precision="single")
    fin = nb.simulate(s, nb.SimParams(1.0, 1e-3, 1e-26, 2))
    assert np.all(np.isfinite(fin.position_matrix())) and np.all(np.isfinite(np.stack(fin.velocities, 1)))


@pytest.mark.parametrize("eps2", [1e-28, 1e-40])
def test_nb_force_masks_overflowing_self_term(eps2, oracle):
    """nb_force_f32 with a tiny positive eps2 (1e-28: m*eps2^-1.5 = 1e42 overflows
    FP32; 1e-40: subnormal, flushed by the FTZ rsqrt): the masses are on the
    device, so the self pair is always masked -- finite accelerations matching
    the oracle (they were NaN)."""
    import torch
    from paper_2203_08263_b200 import _native
    from paper_2203_08263_b200.device import DeviceState
    s = nb.uniform_cube(2000, 9, nb.Precision.SINGLE)
    st = DeviceState(s.position_matrix().astype(np.float32), np.stack(s.velocities, 1), s.masses, np.float32)
    out = torch.zeros((2000, 4), dtype=torch.float32, device="cuda")
    _native.call("nb_force_f32", st.pos_cur.data_ptr(), 2000, 0, 2000, eps2, 1.0, out.data_ptr(), st.ws.data_ptr(),
                 st.ws_bytes, st.stream_ptr())
    a = out[:, :3].cpu().numpy()
    assert np.all(np.isfinite(a))
    rows = np.arange(0, 2000, 37)
    pos = s.position_matrix()
    want = oracle.accel_rows_ld(*(np.ascontiguousarray(pos[:, k].astype(np.float32)) for k in range(3)), s.masses,
                                rows, 1.0, float(np.float32(eps2)))
    assert oracle.accel_dev(a[rows], want) <= 1e-4  # unsoftened: condition number is unbounded
