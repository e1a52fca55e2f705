"""Device-resident state and the GPU driver for one device.

PyTorch is used only for what it is good at here: device allocation, pinned
host staging and the CUDA stream handle.  All arithmetic runs in the sm_100a
kernels behind libnbody_b200.so (``_native``).

HBM layout (one GPU, or one i-shard of a multi-GPU run):

* ``pos_a``, ``pos_b`` -- (N, 4) packed (x, y, z, m), ping-ponged between steps
  (the force pass reads all N while the fused epilogue writes the next
  positions of its own rows, so the two must not alias);
* ``vel``, ``acc`` -- (n_i, 4) for the target rows only; ``acc`` holds the
  previous step's accelerations for the trapezoidal kick;
* ``carry`` -- (3, n_i) FP64 partial sums for a split source range;
* ``ws`` -- the stream-K workspace (FP64 partial slots of split i-blocks; every
  slot is written before it is read within a launch, so it needs no init).
"""

from __future__ import annotations

import ctypes
import math
from typing import Optional, Tuple

import numpy as np
import torch

from . import _native
from ._native import (NB_FLAG_EXCLUDE_SELF, NB_FLAG_UNIFORM_MASS, NB_MODE_ACCEL, NB_STEP_FINAL_KICK,
                      NB_STEP_FIRST, NB_STEP_KICK_DRIFT)

__all__ = ["DeviceState", "needs_self_mask", "kernel_flags", "pack_bodies", "TORCH_DTYPE"]

TORCH_DTYPE = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


def _self_mask(mmax: float, eps2: float, dtype: np.dtype) -> bool:
    e = float(dtype.type(eps2))
    if not e > 0.0:
        return True
    big = 1e30 if dtype == np.float32 else 1e300
    # max(mmax, 1): uniform-mass kernels form eps2^-1.5 without m, so a small
    # uniform mass must not hide an overflowing self term (host_flags does the same).
    return not (max(mmax, 1.0) * (1.0 / e) / math.sqrt(e) < big)


def needs_self_mask(masses: np.ndarray, eps2: float, dtype) -> bool:
    """True when the self pair must be excluded explicitly: (real)eps2 == 0
    (0*inf at j == i, the case pinned by pkg/tests/test_kernels.py:51-55), or a
    self term m*eps2^-1.5 that would overflow the system precision."""
    m = np.asarray(masses)
    return _self_mask(float(m.max()) if m.size else 0.0, eps2, np.dtype(dtype))


def kernel_flags(masses: np.ndarray, eps2: float, dtype, allow_uniform: bool = True) -> int:
    """nb_dev_step flags for a system: NB_FLAG_EXCLUDE_SELF when the self pair
    must be masked, NB_FLAG_UNIFORM_MASS when every mass is identical (m is then
    applied once per body; C5's Plummer sphere has m = 1/N for all bodies).
    (Masses are finite and positive -- validated at the boundary -- so
    max == min is "all equal".)"""
    m = np.asarray(masses)
    if not m.size:
        return NB_FLAG_EXCLUDE_SELF if _self_mask(0.0, eps2, np.dtype(dtype)) else 0
    mmax, mmin = float(m.max()), float(m.min())
    flags = NB_FLAG_EXCLUDE_SELF if _self_mask(mmax, eps2, np.dtype(dtype)) else 0
    if allow_uniform and mmax == mmin:
        flags |= NB_FLAG_UNIFORM_MASS
    return flags


def pack_bodies(pos: np.ndarray, w: Optional[np.ndarray], dtype, pin: bool) -> torch.Tensor:
    """(N,3) coordinates (+ optional 4th column) -> (N,4) host tensor, pinned if asked."""
    n = pos.shape[0]
    t = torch.empty((n, 4), dtype=TORCH_DTYPE[np.dtype(dtype)], pin_memory=pin)
    a = t.numpy()
    a[:, :3] = pos
    a[:, 3] = 0 if w is None else w
    return t


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class DeviceState:
    """Packed device buffers for the target rows [i_begin, i_begin+n_i) of an
    N-body system (all N positions are resident: every target needs every source)."""

    def __init__(self, positions: np.ndarray, velocities: np.ndarray, masses: np.ndarray, dtype,
                 device: Optional[torch.device] = None, i_begin: int = 0, n_i: Optional[int] = None,
                 pos_buffer: Optional[torch.Tensor] = None):
        self.dtype = np.dtype(dtype)
        if self.dtype not in TORCH_DTYPE:
            raise ValueError(f"unsupported precision {self.dtype}")
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise RuntimeError("DeviceState needs a CUDA device; there is no CPU fallback")
        self.n = int(np.asarray(masses).shape[0])
        self.i_begin = int(i_begin)
        self.n_i = self.n - self.i_begin if n_i is None else int(n_i)
        self.sfx = "_f32" if self.dtype == np.float32 else "_f64"
        self.pbytes = self.dtype.itemsize
        tdt = TORCH_DTYPE[self.dtype]
        self._alloc_staging()
        if pos_buffer is not None:
            # caller-provided (2, N, 4) storage, e.g. symmetric memory peers can write into
            if tuple(pos_buffer.shape) != (2, self.n, 4) or pos_buffer.dtype != tdt:
                raise ValueError("pos_buffer must be a (2, N, 4) tensor of the system precision")
            self.pos_a, self.pos_b = pos_buffer[0], pos_buffer[1]
        else:
            self.pos_a = torch.empty((self.n, 4), dtype=tdt, device=self.device)
            self.pos_b = torch.empty_like(self.pos_a)
        self.vel = torch.empty((max(self.n_i, 1), 4), dtype=tdt, device=self.device)
        # acc, carry and the stream-K slots are always written before they are read
        self.acc = torch.empty((max(self.n_i, 1), 4), dtype=tdt, device=self.device)
        self.carry = torch.empty((3, max(self.n_i, 1)), dtype=torch.float64, device=self.device)
        self.ws_bytes = _native.workspace_bytes(self.pbytes, max(self.n_i, 1))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.load(positions, velocities, masses)

    def _alloc_staging(self) -> None:
        """Column staging reused by every load()/readback: 7 columns (x, y, z, m of
        all N bodies; vx, vy, vz of the n_i owned ones) in pinned host memory and on
        the device, so each transfer is ONE contiguous copy and the (de)interleave
        to the packed rows runs on the GPU (nb_dev_load_cols / nb_dev_store_cols)."""
        tdt = TORCH_DTYPE[self.dtype]
        ncol = 4 * self.n + 3 * max(self.n_i, 1)
        self._h_cols = torch.empty(ncol, dtype=tdt, pin_memory=True)
        self._d_cols = torch.empty(ncol, dtype=tdt, device=self.device)
        # fixed for the life of the state: the numpy view and the raw pointers
        self._h_np = self._h_cols.numpy()
        self._cols_ptrs = (self._h_cols.data_ptr(), self._d_cols.data_ptr())
        self._h_out = torch.empty((self.n, 4), dtype=tdt, pin_memory=True)
        self._h2d_done = None
        self._h2d_pending = False

    def _fill_staging(self, positions, velocities, masses) -> None:
        """Write the column block (x, y, z, m of all N; vx, vy, vz of the owned
        rows) into the pinned staging."""
        if self._h2d_pending:
            self._h2d_done.synchronize()  # staging still feeding the previous copy
        self.masses = np.ascontiguousarray(masses, dtype=self.dtype)
        n, ni = self.n, self.n_i
        h = self._h_np
        lo, hi = self.i_begin, self.i_begin + ni
        if not isinstance(positions, (tuple, list)):
            positions = tuple(np.asarray(positions)[:, k] for k in range(3))
            velocities = tuple(np.asarray(velocities)[:, k] for k in range(3))
        for k in range(3):
            h[k * n:(k + 1) * n] = positions[k]
            h[4 * n + k * max(ni, 1): 4 * n + k * max(ni, 1) + ni] = velocities[k][lo:hi]
        h[3 * n:4 * n] = self.masses

    def _staged_columns(self):
        """Fresh host columns from the staging: ONE copy of the block, returned
        as six contiguous 1-D views of it (positions x, y, z; owned velocities)."""
        n, ni = self.n, self.n_i
        h = np.array(self._h_np)
        pos = tuple(h[k * n:(k + 1) * n] for k in range(3))
        vel = tuple(h[4 * n + k * max(ni, 1): 4 * n + k * max(ni, 1) + ni] for k in range(3))
        return pos, vel

    def simulate_columns(self, positions, velocities, masses, g: float, dt: float, eps2: float, steps: int,
                         flags: int):
        """load + simulate + readback of an unsharded system in ONE native call
        (nb_dev_simulate_cols): returns the final (x, y, z) and (vx, vy, vz)
        columns as fresh host arrays."""
        if self.i_begin != 0 or self.n_i != self.n:
            raise ValueError("DeviceState.simulate_columns runs an unsharded system")
        self._fill_staging(positions, velocities, masses)
        hp, dp = self._cols_ptrs
        final_in_b = ctypes.c_int(0)
        _native.call("nb_dev_simulate_cols" + self.sfx, hp, dp, self.pos_a.data_ptr(), self.pos_b.data_ptr(),
                     self.vel.data_ptr(), self.acc.data_ptr(), self.n, g, dt, eps2, steps, int(flags),
                     self.ws.data_ptr(), self.ws_bytes, self.stream_ptr(), ctypes.byref(final_in_b))
        self._h2d_pending = False  # the call synchronized the stream
        self.cur_is_a = not final_in_b.value
        return self._staged_columns()

    def load(self, positions, velocities, masses: np.ndarray) -> None:
        """(Re)initialise the resident state from host data -- (N,3) arrays or
        (x, y, z) column tuples: contiguous column writes into the pinned staging,
        one asynchronous H2D and two pack launches on the current stream."""
        self._fill_staging(positions, velocities, masses)
        n, ni = self.n, self.n_i
        # one native call: H2D of the column block + the two pack launches
        hp, dp = self._cols_ptrs
        _native.call("nb_dev_load_cols" + self.sfx, hp, dp, n, ni, self.pos_a.data_ptr(), self.vel.data_ptr(),
                     self.stream_ptr())
        if self._h2d_done is None:
            self._h2d_done = torch.cuda.Event()
        self._h2d_done.record()
        self._h2d_pending = True
        self.cur_is_a = True

    def columns_host(self):
        """Current positions (x, y, z of all N) and velocities (of the n_i owned
        rows) as six fresh contiguous host arrays: one native call (two unpack
        launches, the D2H into the pinned staging, a stream sync), six memcpys."""
        n, ni = self.n, self.n_i
        # (a pending H2D from the staging is earlier on the same stream: no wait needed)
        self._h2d_pending = False
        # one native call: the two unpack launches + D2H of the block + stream sync
        hp, dp = self._cols_ptrs
        _native.call("nb_dev_store_cols" + self.sfx, self.pos_cur.data_ptr(), self.vel.data_ptr(), n, ni, dp, hp,
                     self.stream_ptr())
        return self._staged_columns()

    @classmethod
    def from_generator(cls, kind: str, n: int, seed: int, dtype,
                       device: Optional[torch.device] = None) -> "DeviceState":
        """A resident system generated on the device (nb_dev_init): ``kind`` is
        "uniform_cube" or "plummer_sphere", the BASELINE.json generators of
        ``core`` -- no host generation and no H2D copy of the state."""
        codes = {"uniform_cube": _native.NB_INIT_UNIFORM_CUBE, "plummer_sphere": _native.NB_INIT_PLUMMER}
        if kind not in codes:
            raise ValueError(f"unknown generator {kind!r}")
        dtype = np.dtype(dtype)
        self = cls.__new__(cls)
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n, self.i_begin, self.n_i = int(n), 0, int(n)
        self.sfx = "_f32" if dtype == np.float32 else "_f64"
        self.pbytes = dtype.itemsize
        tdt = TORCH_DTYPE[dtype]
        self.pos_a = torch.empty((self.n, 4), dtype=tdt, device=self.device)
        self.pos_b = torch.empty_like(self.pos_a)
        self.vel = torch.empty((self.n, 4), dtype=tdt, device=self.device)
        _native.call("nb_dev_init" + self.sfx, codes[kind], int(seed), self.n, self.pos_a.data_ptr(),
                     self.vel.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
        self.masses = None  # device-resident only; see masses_host()
        self._alloc_staging()
        self.acc = torch.empty((self.n, 4), dtype=tdt, device=self.device)
        self.carry = torch.empty((3, self.n), dtype=torch.float64, device=self.device)
        self.ws_bytes = _native.workspace_bytes(self.pbytes, self.n)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.cur_is_a = True
        return self

    def masses_host(self) -> np.ndarray:
        return self.pos_cur[:, 3].cpu().numpy()

    # -------------------------------------------------------------- buffers
    @property
    def pos_cur(self) -> torch.Tensor:
        return self.pos_a if self.cur_is_a else self.pos_b

    @property
    def pos_next(self) -> torch.Tensor:
        return self.pos_b if self.cur_is_a else self.pos_a

    def swap(self) -> None:
        self.cur_is_a = not self.cur_is_a

    def stream_ptr(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    # -------------------------------------------------------------- kernels
    def step(self, g: float, eps2: float, dt: float, mode: int, flags: int,
             j_begin: Optional[int] = None, j_count: Optional[int] = None, carry_mode: int = 0,
             acc_out: Optional[torch.Tensor] = None, peers: Optional[list] = None) -> None:
        """One fused force(+update) launch on the current positions (nb_dev_step).
        ``peers``: device pointers of other GPUs' next-position buffers; the drifted
        rows are then also stored there by the kernel (nb_dev_step_p2p)."""
        j_begin = self.i_begin if j_begin is None else j_begin
        j_count = self.n if j_count is None else j_count
        acc = self.acc if acc_out is None else acc_out
        drift = mode in (NB_STEP_FIRST, NB_STEP_KICK_DRIFT)
        args = [self.pos_cur.data_ptr(), self.n, self.i_begin, self.n_i, j_begin % self.n, j_count, g, eps2,
                dt, mode, int(flags), self.carry.data_ptr() if carry_mode else None, carry_mode,
                acc.data_ptr(), self.vel.data_ptr() if mode != NB_MODE_ACCEL else None,
                self.pos_next.data_ptr() if drift else None]
        if peers:
            arr = (ctypes.c_void_p * len(peers))(*peers)
            _native.call("nb_dev_step_p2p" + self.sfx, *args, arr, len(peers), self.ws.data_ptr(),
                         self.ws_bytes, self.stream_ptr())
        else:
            _native.call("nb_dev_step" + self.sfx, *args, self.ws.data_ptr(), self.ws_bytes, self.stream_ptr())

    def simulate(self, g: float, dt: float, eps2: float, steps: int, flags: int) -> None:
        """Whole single-device velocity-Verlet run (nb_dev_simulate): steps+1 launches."""
        if self.i_begin != 0 or self.n_i != self.n:
            raise ValueError("DeviceState.simulate runs an unsharded system; use sharded.simulate")
        final_in_b = ctypes.c_int(0)
        _native.call("nb_dev_simulate" + self.sfx, self.pos_cur.data_ptr(), self.pos_next.data_ptr(),
                     self.vel.data_ptr(), self.acc.data_ptr(), self.n, g, dt, eps2, steps,
                     int(flags), self.ws.data_ptr(), self.ws_bytes, self.stream_ptr(),
                     ctypes.byref(final_in_b))
        if steps % 2 == 1:
            self.swap()

    def simulate_timed(self, g: float, dt: float, eps2: float, steps: int, flags: int) -> list:
        """``simulate`` that also returns the CUDA-event time (ms) of each of the
        steps+1 force evaluations, measured on this stream (synchronizes)."""
        if self.i_begin != 0 or self.n_i != self.n:
            raise ValueError("DeviceState.simulate_timed runs an unsharded system")
        final_in_b = ctypes.c_int(0)
        ms = (ctypes.c_float * (steps + 1))()
        _native.call("nb_dev_simulate_timed" + self.sfx, self.pos_cur.data_ptr(), self.pos_next.data_ptr(),
                     self.vel.data_ptr(), self.acc.data_ptr(), self.n, g, dt, eps2, steps,
                     int(flags), self.ws.data_ptr(), self.ws_bytes, self.stream_ptr(),
                     ctypes.byref(final_in_b), ms)
        if steps % 2 == 1:
            self.swap()
        return list(ms)

    def accelerations(self, g: float, eps2: float, flags: int) -> torch.Tensor:
        """(n_i, 4) device accelerations of the current positions (mode ACCEL)."""
        out = torch.empty((max(self.n_i, 1), 4), dtype=self.acc.dtype, device=self.device)
        self.step(g, eps2, 0.0, NB_MODE_ACCEL, flags, j_begin=0, j_count=self.n, acc_out=out)
        return out[: self.n_i]

    def energy(self, g: float, eps2: float) -> Tuple[float, float, Tuple[float, float, float]]:
        """(kinetic, potential, momentum) in FP64 (unsharded state only)."""
        if self.n_i != self.n:
            raise ValueError("energy diagnostics need the whole system on one device")
        out = torch.zeros(6, dtype=torch.float64, device=self.device)
        ws = torch.empty(_native.energy_workspace_bytes(self.pbytes, self.n), dtype=torch.uint8, device=self.device)
        _native.call("nb_dev_energy" + self.sfx, self.pos_cur.data_ptr(), self.vel.data_ptr(), self.n,
                     g, eps2, out.data_ptr(), ws.data_ptr(), ws.numel(), self.stream_ptr())
        v = out.cpu().numpy()
        return float(v[0]), float(v[1]), (float(v[2]), float(v[3]), float(v[4]))

    # -------------------------------------------------------------- host views
    def positions_packed(self) -> np.ndarray:
        """(N, 4) pinned view of the current positions (x, y, z, m); valid until
        the next readback of this state."""
        self._h_out.copy_(self.pos_cur)
        return self._h_out.numpy()

    def velocities_packed(self) -> np.ndarray:
        """(n_i, 4) pinned view of the owned velocities; valid until the next readback."""
        self._h_out[: self.vel.shape[0]].copy_(self.vel)
        return self._h_out.numpy()[: self.n_i]

    def positions_host(self) -> np.ndarray:
        """Current positions (N, 3): one D2H of the packed rows into pinned memory."""
        self._h_out.copy_(self.pos_cur)
        return np.array(self._h_out.numpy()[:, :3])

    def velocities_host(self) -> np.ndarray:
        self._h_out[: self.vel.shape[0]].copy_(self.vel)
        return np.array(self._h_out.numpy()[: self.n_i, :3])
