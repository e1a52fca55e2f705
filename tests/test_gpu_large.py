"""Parity at the sharded BASELINE sizes on one GPU (C4: 524288 bodies FP64,
C5: 4194304 bodies FP32 Plummer), SURVEY.md 8(c) tolerances against the oracle:

* per-step accelerations (``_accel_dev``, validation.py:212-225) of the GPU's
  OWN state after steps 0, 1 and 2 -- not just the initial state -- against the
  long-double oracle on that state, row-sampled (<= 1e-12 FP64, <= 1e-5 FP32);
* the same through an i-shard of the multi-GPU decomposition (P = 4 / 8 ranks'
  two-phase carry: local sources, then the circular remote range), run for one
  rank on this GPU -- a rank's kernels never wait on another rank's;
* the one-step state of sampled rows: p1 and v1 depend only on that row's a0,
  so the reference's update rule (_accel_cy.pyx:218-226) applied to the
  oracle's a0 must reproduce the GPU's within what the acceleration tolerance
  allows;
* C4's whole 5-step trajectory against the FP64 oracle port on every host core
  (``_position_dev`` <= 1e-12; ~5 min of CPU, marked slow).
"""
import numpy as np
import pytest

import paper_2203_08263_b200 as nb
from paper_2203_08263_b200._native import (NB_FLAG_EXCLUDE_SELF, NB_MODE_ACCEL, NB_STEP_FINAL_KICK,
                                           NB_STEP_FIRST, NB_STEP_KICK_DRIFT)

pytestmark = pytest.mark.gpu

F64_ACC_TOL = 1e-12
F32_ACC_TOL = 1e-5


def _tol(cfg):
    return F64_ACC_TOL if cfg.precision is nb.Precision.DOUBLE else F32_ACC_TOL


def _rows(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, 1, n - 1], rng.integers(0, n, k)]))


def _state(cfg):
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    s = cfg.system()
    dtype = cfg.precision.dtype
    st = DeviceState(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, dtype)
    return s, st, kernel_flags(s.masses, cfg.softening_sq, dtype)


def _oracle_rows(oracle, pos4, rows, eps2):
    cols = [np.ascontiguousarray(pos4[:, k]) for k in range(3)]
    return oracle.accel_rows_ld(*cols, np.ascontiguousarray(pos4[:, 3]), rows, 1.0, eps2)


@pytest.mark.parametrize("cfg_name", ["C4", "C5"])
def test_accelerations_of_gpu_state_after_steps(cfg_name, oracle):
    """a_k of the GPU's own positions p_k for k = 0, 1, 2 (the fused launches of
    simulate: FIRST, then KICK_DRIFT), row-sampled against the oracle on p_k."""
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    s, st, flags = _state(cfg)
    p = cfg.params()
    rows = _rows(cfg.n, 45 if cfg_name == "C5" else 93, 11)
    for k, mode in enumerate((NB_STEP_FIRST, NB_STEP_KICK_DRIFT, NB_STEP_KICK_DRIFT)):
        pk = st.pos_cur.cpu().numpy()  # (N, 4): x, y, z, m
        st.step(1.0, p.softening_sq, p.dt, mode, flags)
        a = st.acc[:, :3].cpu().numpy()
        want = _oracle_rows(oracle, pk, rows, p.softening_sq)
        dev = oracle.accel_dev(a[rows], want)
        print(cfg_name, "step", k, "accel_dev", dev)
        assert dev <= _tol(cfg), (k, dev)
        if k > 0:  # the state really moved
            assert not np.array_equal(pk[:, :3], prev[:, :3])
        prev = pk
        st.swap()


@pytest.mark.parametrize("cfg_name,world,rank", [("C4", 4, 1), ("C5", 8, 3)])
def test_sharded_rank_accelerations_full_size(cfg_name, world, rank, oracle):
    """One rank of the P-way i-shard at full size: its N/P targets summed over
    its own rows (carry_mode 1) and then the circular remote range (carry_mode
    2), as run_sharded issues them, against the oracle."""
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    from paper_2203_08263_b200.sharded import pad_system, shard_range
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    s = cfg.system()
    dtype = cfg.precision.dtype
    pos, vel, m = pad_system(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, world)
    npad = pos.shape[0]
    i0, ni = shard_range(npad, rank, world)
    st = DeviceState(pos, vel, m, dtype, i_begin=i0, n_i=ni)
    flags = kernel_flags(m, cfg.softening_sq, dtype)
    eps2 = cfg.softening_sq
    st.step(1.0, eps2, 0.0, NB_MODE_ACCEL, flags, j_begin=i0, j_count=ni, carry_mode=1)
    st.step(1.0, eps2, 0.0, NB_MODE_ACCEL, flags, j_begin=(i0 + ni) % npad, j_count=npad - ni, carry_mode=2)
    a = st.acc[:ni, :3].cpu().numpy()
    local = _rows(ni, 45, 5)
    want = _oracle_rows(oracle, np.concatenate([pos, m[:, None]], 1), i0 + local, eps2)
    dev = oracle.accel_dev(a[local], want)
    print(cfg_name, f"rank {rank}/{world}", "accel_dev", dev)
    assert dev <= _tol(cfg)


@pytest.mark.parametrize("cfg_name", ["C4", "C5"])
def test_one_step_state_of_sampled_rows(cfg_name, oracle):
    """The first step of simulate at full size, row by row: the reference's
    update (_accel_cy.pyx:218-226: dv = a*dt; p += (v + half*dv)*dt; v += dv, in
    the system precision) applied to the ORACLE's a0 of each sampled row must
    reproduce the GPU's p1 and v1 to within what the acceleration tolerance
    allows (|da| <= tol*|a0| moves p by half*dt^2*|da| and v by dt*|da|) plus
    2 ulp of rounding -- and the state must actually have moved (C5's FP32
    positions do not move by an ulp in one step of dt = 1e-4 from rest; its
    velocities do)."""
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    s, st, flags = _state(cfg)
    p = cfg.params()
    dtype = cfg.precision.dtype
    p0 = st.pos_cur.cpu().numpy()
    v0 = st.vel[:, :3].cpu().numpy()
    st.step(1.0, p.softening_sq, p.dt, NB_STEP_FIRST, flags)
    st.swap()
    p1 = st.pos_cur[:, :3].cpu().numpy()
    v1 = st.vel[:, :3].cpu().numpy()
    rows = _rows(cfg.n, 93, 17)
    a64 = _oracle_rows(oracle, p0, rows, p.softening_sq)
    a0 = a64.astype(dtype)
    dt, half = dtype.type(p.dt), dtype.type(0.5)
    dv = a0 * dt
    want_p = p0[rows, :3] + (v0[rows] + half * dv) * dt
    want_v = v0[rows] + dv
    amag = np.linalg.norm(a64, axis=1)[:, None]
    tol = _tol(cfg)
    ulp_p = np.spacing(np.abs(want_p).astype(dtype)).astype(np.float64)
    ulp_v = np.spacing(np.abs(want_v).astype(dtype)).astype(np.float64)
    err_p = np.abs(p1[rows] - want_p.astype(np.float64))
    err_v = np.abs(v1[rows] - want_v.astype(np.float64))
    bound_p = 0.5 * p.dt ** 2 * tol * amag + 2 * ulp_p
    bound_v = p.dt * tol * amag + 2 * ulp_v
    print(cfg_name, "p1 err/bound", float(np.max(err_p / bound_p)), "v1 err/bound", float(np.max(err_v / bound_v)))
    assert np.all(err_p <= bound_p)
    assert np.all(err_v <= bound_v)
    assert not (np.array_equal(p1[rows], p0[rows, :3]) and np.array_equal(v1[rows], v0[rows]))


@pytest.mark.slow
def test_c4_full_trajectory_vs_oracle(oracle):
    """C4 at full size (524288 bodies, FP64, 5 steps): the GPU simulate against
    the FP64 oracle port on all host cores, _position_dev <= 1e-12."""
    cfg = nb.BASELINE_CONFIGS["C4"]
    s = cfg.system()
    p = cfg.params()
    fin = nb.simulate(s, p).position_matrix()
    ref, _ = oracle.simulate(s.position_matrix(), np.stack(s.velocities, 1).astype(np.float64),
                             s.masses.astype(np.float64), 1.0, p.dt, p.softening_sq, p.steps,
                             threads=oracle.host_threads())
    dev = oracle.position_dev(fin, ref)
    print("C4 position_dev", dev)
    assert dev <= 1e-12
