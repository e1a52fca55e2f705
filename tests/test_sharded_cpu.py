"""CPU, world_size 2 and 3 over gloo: the multi-GPU host logic of
paper_2203_08263_b200.sharded.run_sharded (i-shards, local-sources-first split
with an FP64 carry, in-place all-gather of positions) driving an
oracle-backed stand-in for the device state.  The stand-in implements the
nb_dev_step contract (carry modes, update modes) in NumPy float64; the test
checks the sharded trajectory against the single-process oracle simulate."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_08263_b200._native import NB_MODE_ACCEL, NB_STEP_FINAL_KICK, NB_STEP_FIRST
from paper_2203_08263_b200.sharded import pad_system, run_sharded, shard_range


class OracleShardState:
    """NumPy float64 implementation of the DeviceState.step contract."""

    def __init__(self, pos, vel, m, i0, ni):
        n = pos.shape[0]
        self.n, self.i_begin, self.n_i = n, i0, ni
        self.pos_a = torch.zeros((n, 4), dtype=torch.float64)
        self.pos_a[:, :3] = torch.from_numpy(pos)
        self.pos_a[:, 3] = torch.from_numpy(m)
        self.pos_b = self.pos_a.clone()
        self.vel = torch.zeros((ni, 4), dtype=torch.float64)
        self.vel[:, :3] = torch.from_numpy(vel[i0:i0 + ni])
        self.acc = torch.zeros((ni, 4), dtype=torch.float64)
        self.carry = np.zeros((ni, 3))
        self.cur_is_a = True

    @property
    def pos_cur(self):
        return self.pos_a if self.cur_is_a else self.pos_b

    @property
    def pos_next(self):
        return self.pos_b if self.cur_is_a else self.pos_a

    def swap(self):
        self.cur_is_a = not self.cur_is_a

    def step(self, g, eps2, dt, mode, exclude_self, j_begin=None, j_count=None, carry_mode=0):
        P = self.pos_cur.numpy()
        j_begin = self.i_begin if j_begin is None else j_begin
        j_count = self.n if j_count is None else j_count
        rows = np.arange(self.i_begin, self.i_begin + self.n_i)
        js = (j_begin + np.arange(j_count)) % self.n
        d = P[js, :3][None, :, :] - P[rows, :3][:, None, :]
        d2 = np.sum(d * d, axis=2) + eps2
        with np.errstate(divide="ignore", invalid="ignore"):
            w = P[js, 3][None, :] / (d2 * np.sqrt(d2))
        w[rows[:, None] == js[None, :]] = 0.0
        s = np.sum(d * w[:, :, None], axis=1)
        if carry_mode == 2:
            s = self.carry + s
        if carry_mode == 1:
            self.carry = s
            return
        a = s * g
        if mode != NB_MODE_ACCEL:
            v = self.vel.numpy()[:, :3]
            if mode != NB_STEP_FIRST:
                v += (a - self.acc.numpy()[:, :3]) * (0.5 * dt)
            if mode != NB_STEP_FINAL_KICK:
                dv = a * dt
                nxt = self.pos_next.numpy()
                nxt[rows, :3] = P[rows, :3] + (v + 0.5 * dv) * dt
                nxt[rows, 3] = P[rows, 3]
                v += dv
        self.acc.numpy()[:, :3] = a


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, steps, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_08263_b200.core import Precision, uniform_cube
    s = uniform_cube(n, 77, Precision.DOUBLE)
    pos0, vel0 = s.position_matrix(), np.stack(s.velocities, 1)
    pos, vel, m = pad_system(pos0, vel0, s.masses, world)
    i0, ni = shard_range(pos.shape[0], rank, world)
    st = OracleShardState(pos, vel, m, i0, ni)

    def gather(full, local):
        return dist.all_gather_into_tensor(full, local.clone(), async_op=True)

    run_sharded(st, 1.0, 1e-3, 1e-3, steps, False, gather, world)
    vel_full = torch.zeros((pos.shape[0], 4), dtype=torch.float64)
    dist.all_gather_into_tensor(vel_full, st.vel.contiguous())
    if rank == 0:
        np.savez(out_path, pos=st.pos_cur[:n, :3].numpy(), vel=vel_full[:n, :3].numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 64), (3, 50)])
def test_sharded_loop_matches_single_process_oracle(world, n, tmp_path, oracle):
    out = str(tmp_path / "res.npz")
    steps = 4
    mp.spawn(_worker, args=(world, _free_port(), n, steps, out), nprocs=world, join=True)
    res = np.load(out)
    from paper_2203_08263_b200.core import Precision, uniform_cube
    s = uniform_cube(n, 77, Precision.DOUBLE)
    ref_pos, ref_vel = oracle.simulate(s.position_matrix(), np.stack(s.velocities, 1), s.masses,
                                       1.0, 1e-3, 1e-3, steps, threads=1)
    assert oracle.position_dev(res["pos"], ref_pos) <= 1e-13
    np.testing.assert_allclose(res["vel"], ref_vel, rtol=1e-11, atol=1e-13)
