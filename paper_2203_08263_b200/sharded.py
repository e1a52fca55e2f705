"""i-body sharding across GPUs: one process per GPU, NCCL all-gather of positions.

The reference parallelises only over target bodies i (OpenMP static schedule,
/root/reference/pkg/src/nbodybench/kernels/_accel_cy.pyx:132-136), each worker
writing its own slice.  Across GPUs the same axis shards: rank r
owns the contiguous rows [r*N/P, (r+1)*N/P), keeps all N positions resident,
and after every drift the ranks exchange their new position rows with one
in-place all-gather (the only data-path collective; masses ride in .w).

Overlap: the force pass of step k+1 first sums over the rank's OWN rows as
sources (already valid locally) into an FP64 carry, while the all-gather of
step k's positions is in flight on NCCL's stream; the compute stream then waits
for the gather and sums the remaining N - N/P sources (one circular range
starting after the local slice) before the fused update.

The driver is written against a small state interface (``DeviceState``) and an
``allgather(full, local)`` callable, so its host logic is exercised on CPU with
gloo and an oracle-backed state in tests/test_sharded_cpu.py.
"""

from __future__ import annotations

from typing import Callable, Optional, Tuple

import numpy as np

from ._native import NB_STEP_FINAL_KICK, NB_STEP_FIRST, NB_STEP_KICK_DRIFT

__all__ = ["shard_range", "padded_count", "run_sharded", "simulate_sharded"]


def padded_count(n: int, world: int) -> int:
    """Bodies after padding N up to a multiple of the world size (equal shards
    are what an in-place all-gather needs)."""
    return ((n + world - 1) // world) * world


def shard_range(n_padded: int, rank: int, world: int) -> Tuple[int, int]:
    per = n_padded // world
    return rank * per, per


def pad_system(pos: np.ndarray, vel: np.ndarray, m: np.ndarray, world: int):
    """Pad to equal shards with massless bodies far from everything: they add
    exactly 0 to every real body (w = 0 * r^3 with finite r) and their own rows
    are discarded."""
    n = pos.shape[0]
    npad = padded_count(n, world)
    if npad == n:
        return pos, vel, m
    extra = npad - n
    far = np.float64(1e18) if pos.dtype == np.float64 else np.float32(1e17)
    pad_pos = np.full((extra, 3), far, dtype=pos.dtype) * (1 + np.arange(extra, dtype=pos.dtype))[:, None]
    return (np.concatenate([pos, pad_pos]), np.concatenate([vel, np.zeros((extra, 3), vel.dtype)]),
            np.concatenate([m, np.zeros(extra, m.dtype)]))


def run_sharded(state, g: float, dt: float, eps2: float, steps: int, flags: int,
                allgather: Callable, world: int) -> None:
    """Velocity-Verlet loop of kernels.simulate (kernels/__init__.py:240-252) on
    one shard.  ``state`` holds all positions and this rank's rows; ``allgather``
    starts an in-place gather of ``pos[i0:i0+ni]`` into ``pos`` on every rank and
    returns an object with ``wait()``."""
    n, i0, ni = state.n, state.i_begin, state.n_i
    if world == 1:
        for s in range(steps):
            state.step(g, eps2, dt, NB_STEP_FIRST if s == 0 else NB_STEP_KICK_DRIFT, flags)
            state.swap()
        state.step(g, eps2, dt, NB_STEP_FINAL_KICK, flags)
        return
    pending = None
    for s in range(steps + 1):
        mode = NB_STEP_FIRST if s == 0 else (NB_STEP_KICK_DRIFT if s < steps else NB_STEP_FINAL_KICK)
        # local sources first: rows [i0, i0+ni) of the current positions are ours
        state.step(g, eps2, dt, mode, flags, j_begin=i0, j_count=ni, carry_mode=1)
        if pending is not None:
            pending.wait()
        # then every other source, as one circular range after the local slice
        state.step(g, eps2, dt, mode, flags, j_begin=(i0 + ni) % n, j_count=n - ni, carry_mode=2)
        if mode != NB_STEP_FINAL_KICK:
            state.swap()
            pending = allgather(state.pos_cur, state.pos_cur[i0:i0 + ni])
    if pending is not None:
        pending.wait()


def run_sharded_p2p(state, g: float, dt: float, eps2: float, steps: int, flags: int,
                    peer_next: Callable, barrier: Callable) -> None:
    """The same loop with the exchange fused into the force kernel: the epilogue
    of the remote-source pass stores each drifted row into every peer GPU's
    next-position buffer over NVLink (nb_dev_step_p2p); no all-gather.

    ``peer_next(cur_is_a)`` returns the peers' next-buffer pointers for the current
    ping-pong parity; ``barrier()`` is a stream-ordered barrier over all ranks.
    Ordering: step s sums its local sources, then barrier(s) -- every rank has
    finished step s-1, so (RAW) all rows of p_s have landed and (WAR) nobody still
    reads the p_{s-1} buffer the step-s epilogue now overwrites -- then the remote
    sources and the peer-store epilogue."""
    n, i0, ni = state.n, state.i_begin, state.n_i
    barrier()  # every rank's buffers exist (after rendezvous / upload)
    for s in range(steps + 1):
        mode = NB_STEP_FIRST if s == 0 else (NB_STEP_KICK_DRIFT if s < steps else NB_STEP_FINAL_KICK)
        state.step(g, eps2, dt, mode, flags, j_begin=i0, j_count=ni, carry_mode=1)
        if s > 0:
            barrier()
        peers = peer_next(state.cur_is_a) if mode != NB_STEP_FINAL_KICK else None
        state.step(g, eps2, dt, mode, flags, j_begin=(i0 + ni) % n, j_count=n - ni, carry_mode=2,
                   peers=peers)
        if mode != NB_STEP_FINAL_KICK:
            state.swap()
    barrier()


class _Done:
    """Handle of an exchange that already completed (host-staged path)."""

    def wait(self) -> None:
        return None


def gather_into(full, local, group=None, async_op: bool = False):
    """In-place all-gather of this rank's rows ``local`` (a slice of ``full``)
    into ``full`` on every rank.  NCCL: one in-place ncclAllGather on the device
    buffers.  Any other backend (gloo, for CPU-side tests of the multi-rank
    driver) is staged through host memory."""
    import torch.distributed as dist

    if full.device.type != "cuda" or dist.get_backend(group) == "nccl":
        return dist.all_gather_into_tensor(full, local, group=group, async_op=async_op)
    host = full.cpu()
    dist.all_gather_into_tensor(host, local.cpu(), group=group)
    full.copy_(host)
    return _Done() if async_op else None


def _torch_allgather(group):
    def gather(full, local):
        return gather_into(full, local, group, async_op=True)
    return gather


_COMM_CACHE: dict = {}


class _StreamWait:
    """Handle of an exchange running on a side stream: wait() orders the current
    (compute) stream after it."""

    def __init__(self, event):
        self.event = event

    def wait(self) -> None:
        import torch
        torch.cuda.current_stream().wait_event(self.event)


def _capi_allgather(group):
    """The exchange through the library's own C ABI (nb_comm_*), as a host that
    is not Python would drive it: rank 0's NCCL unique id is shared over the
    process group, every rank opens its communicator with nb_comm_init_rank
    (cached per group), and each gather is nb_comm_allgather in place on a side
    stream that starts after the drift step and is waited on before the remote-
    source pass -- the same overlap as the torch.distributed transport."""
    import torch
    import torch.distributed as dist

    from . import _native
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    key = (id(group), world, rank, torch.cuda.current_device())
    entry = _COMM_CACHE.get(key)
    if entry is None:
        box = [_native.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        entry = _COMM_CACHE[key] = (_native.comm_init_rank(world, rank, box[0]), torch.cuda.Stream())
    comm, side = entry

    def gather(full, local):
        ready = torch.cuda.Event()
        ready.record()
        side.wait_event(ready)
        _native.comm_allgather(full.data_ptr(), local.numel() * local.element_size(), comm, side.cuda_stream)
        done = torch.cuda.Event()
        done.record(side)
        return _StreamWait(done)
    return gather


def _p2p_setup(pos, vel, m, dtype, i0, ni, group):
    """Positions in symmetric memory (CUDA IPC-mapped on every peer) and the
    symmetric-memory device barrier."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    from .device import TORCH_DTYPE, DeviceState
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world - 1 > 8:
        raise ValueError("the peer-store epilogue supports up to 9 GPUs")
    if group is None:
        group = dist.group.WORLD
    try:
        symm_mem.enable_symm_mem_for_group(group.group_name)
    except (AttributeError, RuntimeError):
        pass
    n = pos.shape[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    buf = symm_mem.empty((2, n, 4), dtype=TORCH_DTYPE[np.dtype(dtype)], device=dev)
    hdl = symm_mem.rendezvous(buf, group.group_name)
    state = DeviceState(pos, vel, m, dtype, i_begin=i0, n_i=ni, pos_buffer=buf)
    half = n * 4 * np.dtype(dtype).itemsize
    peers = [q for q in range(world) if q != rank]
    ptrs = list(hdl.buffer_ptrs)

    def peer_next(cur_is_a: bool):
        return [ptrs[q] + (half if cur_is_a else 0) for q in peers]

    def barrier():
        hdl.barrier(channel=0)
    return state, peer_next, barrier


_SHARD_CACHE: dict = {}


def _shard_state(pos, vel, m, dtype, i0: int, ni: int):
    """The rank's DeviceState, reused across simulate_sharded calls with the same
    shape (device buffers and pinned staging are allocated once; load() refills)."""
    import torch

    from .device import DeviceState
    key = (pos.shape[0], np.dtype(dtype).str, i0, ni, torch.cuda.current_device())
    st = _SHARD_CACHE.get(key)
    if st is None:
        if len(_SHARD_CACHE) >= 4:
            _SHARD_CACHE.clear()
        st = _SHARD_CACHE[key] = DeviceState(pos, vel, m, dtype, i_begin=i0, n_i=ni)
    else:
        st.load(pos, vel, m)
    return st


def simulate_sharded(positions: np.ndarray, velocities: np.ndarray, masses: np.ndarray, dtype,
                     g: float, dt: float, eps2: float, steps: int, group=None,
                     flags: Optional[int] = None, transport: str = "nccl") -> Tuple[np.ndarray, np.ndarray]:
    """Multi-GPU simulate: every rank passes the full initial state and gets the
    full final (positions, velocities) back.  Uses the default process group
    (NCCL, one process per GPU) unless ``group`` is given.  ``transport``:
    "nccl" (in-place all-gather overlapped with the local-source pass), "capi"
    (the same exchange through the library's nb_comm_* C ABI) or "p2p"
    (peer-store epilogue into symmetric-memory buffers; see run_sharded_p2p)."""
    import torch
    import torch.distributed as dist

    from ._native import NB_FLAG_EXCLUDE_SELF
    from .device import DeviceState, kernel_flags, needs_self_mask

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = positions.shape[0]
    dtype = np.dtype(dtype)
    pos, vel, m = pad_system(np.asarray(positions, dtype), np.asarray(velocities, dtype),
                             np.asarray(masses, dtype), world)
    npad = pos.shape[0]
    i0, ni = shard_range(npad, rank, world)
    if flags is None:
        # uniform masses only if no massless padding was added
        flags = kernel_flags(m, eps2, dtype) & ~NB_FLAG_EXCLUDE_SELF
        flags |= NB_FLAG_EXCLUDE_SELF if needs_self_mask(m[:n], eps2, dtype) else 0
    if transport == "p2p":
        state, peer_next, barrier = _p2p_setup(pos, vel, m, dtype, i0, ni, group)
        run_sharded_p2p(state, g, dt, eps2, steps, flags, peer_next, barrier)
    elif transport in ("nccl", "capi"):
        state = _shard_state(pos, vel, m, dtype, i0, ni)
        gather = _torch_allgather(group) if transport == "nccl" else _capi_allgather(group)
        run_sharded(state, g, dt, eps2, steps, flags, gather, world)
    else:
        raise ValueError(f"unknown transport {transport!r} (expected 'nccl', 'capi' or 'p2p')")
    vel_full = torch.empty((npad, 4), dtype=state.vel.dtype, device=state.device)
    gather_into(vel_full, state.vel[:ni].contiguous(), group)
    out_pos = state.pos_cur[:n, :3].cpu().numpy()
    out_vel = vel_full[:n, :3].cpu().numpy()
    return out_pos, out_vel
