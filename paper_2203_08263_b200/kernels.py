"""The N-body entry points, drop-in for ``nbodybench.kernels``.

Same names, argument objects, return types and ``ValueError`` checks as the
reference's kernel API (/root/reference/pkg/src/nbodybench/kernels/__init__.py):

* ``simulate(sys_, params, variant)`` -- kernels/__init__.py:230-253: returns a
  NEW system after ``params.steps`` velocity-Verlet steps (steps+1 force
  evaluations); the input is left untouched.
* ``compute_accelerations(sys_, params, variant, out)`` -- :183-202.
* ``integrate_step(sys_, acc, params, variant)`` -- :205-217.
* ``KernelVariant`` / ``MathForm`` / ``reference_variant`` / ``AccelerationBuffer``
  -- :82-168, with the same validation.

Every call runs on the GPU through libnbody_b200.so; there is no CPU path.
Objects are read by duck typing (``layout.value``, ``precision.value``,
``positions``, ``velocities``, ``masses``), so systems built by the reference
package itself are accepted and a system of the caller's own class is returned.

The variant's ladder axes (layout aside) do not change the GPU arithmetic:
``block``/``threads`` are CPU tiling knobs and the math form is always
m*d*rsqrt(d2)^3, which the reference pins as equivalent to both forms
(pkg/tests/test_kernels.py:220-227).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, replace
from enum import Enum
from typing import Optional, Tuple

import numpy as np

from .core import Layout, Precision

__all__ = [
    "MathForm", "KernelVariant", "AccelerationBuffer", "reference_variant", "ladder",
    "compute_accelerations", "integrate_step", "simulate", "simulate_arrays",
    "diagnostics_gpu",
]

NAME = "b200"


class MathForm(Enum):
    POW_THEN_DIVIDE = "pow"
    RECIPROCAL_MULTIPLY = "recip"

    @classmethod
    def parse(cls, token: str) -> "MathForm":
        try:
            return cls(token)
        except ValueError:
            raise ValueError(f"unknown math form {token!r} (expected 'pow' or 'recip')")


def _value(x) -> str:
    return getattr(x, "value", x)


@dataclass(frozen=True)
class KernelVariant:
    """One rung of the reference's optimisation ladder (kernels/__init__.py:94-135)."""
    layout: Layout = Layout.SOA
    math_form: MathForm = MathForm.POW_THEN_DIVIDE
    block: Optional[int] = None
    threads: int = 1

    def __post_init__(self):
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.block is not None and self.block < 1:
            raise ValueError("block size must be >= 1 when given")
        if _value(self.layout) == "aos":
            if _value(self.math_form) != "pow":
                raise ValueError("aos layout supports only the pow math form")
            if self.block is not None:
                raise ValueError("aos layout does not support blocking")
            if self.threads != 1:
                raise ValueError("aos layout is sequential (threads must be 1)")

    def validate_for(self, n: int) -> None:
        if self.block is not None and self.block > n:
            raise ValueError(f"block size {self.block} exceeds body count {n}")

    def with_threads(self, threads: int) -> "KernelVariant":
        return replace(self, threads=threads)

    @property
    def name(self) -> str:
        parts = [_value(self.layout)]
        if _value(self.math_form) == "recip":
            parts.append("recip")
        if self.block is not None:
            parts.append(f"b{self.block}")
        return "-".join(parts)


def reference_variant() -> KernelVariant:
    return KernelVariant(Layout.SOA, MathForm.POW_THEN_DIVIDE, None, 1)


def ladder(blocks=(8, 64, 256), thread_counts=(1, 2, 4)) -> list:
    variants = [KernelVariant(Layout.AOS)]
    for math_form in MathForm:
        for block in (None, *blocks):
            for threads in thread_counts:
                variants.append(KernelVariant(Layout.SOA, math_form, block, threads))
    return variants


@dataclass
class AccelerationBuffer:
    """Per-axis accelerations in the system precision (kernels/__init__.py:153-168)."""
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray

    @classmethod
    def allocate(cls, n: int, precision) -> "AccelerationBuffer":
        dtype = Precision(_value(precision)).dtype
        return cls(np.zeros(n, dtype), np.zeros(n, dtype), np.zeros(n, dtype))

    @property
    def count(self) -> int:
        return int(self.x.shape[0])


# --------------------------------------------------------------------------- boundary helpers

_PRECISION_DTYPE = {"single": np.dtype(np.float32), "double": np.dtype(np.float64)}


def _dtype(sys_) -> np.dtype:
    p = _value(sys_.precision)
    dt = _PRECISION_DTYPE.get(p) if isinstance(p, str) else None
    return dt if dt is not None else Precision(p).dtype


def _count(sys_) -> int:
    return int(sys_.masses.shape[0])


def _matrix(sys_, field: str) -> np.ndarray:
    """(N,3) view/copy of positions or velocities in the system precision."""
    data = getattr(sys_, field)
    if _value(sys_.layout) == "soa":
        return np.stack(data, axis=1)
    return np.asarray(data)


def _columns(sys_, field: str):
    """(x, y, z) 1-D views of positions or velocities (no copy), either layout."""
    data = getattr(sys_, field)
    if _value(sys_.layout) == "soa":
        return tuple(data)
    return data[:, 0], data[:, 1], data[:, 2]


def _store(state, field: str, values: np.ndarray) -> None:
    """Write (N,3) results into a system's own buffers, preserving its layout."""
    data = getattr(state, field)
    if _value(state.layout) == "soa":
        for k in range(3):
            data[k][...] = values[:, k]
    else:
        data[...] = values


_CTYPE = {np.dtype(np.float32): "float", np.dtype(np.float64): "double"}


def _check_buffers(sys_) -> None:
    """Every state array must already be in the system precision, as the
    reference's typed buffers demand: its compiled backend raises the buffer
    dtype ValueError at the FFI call (_accel_cy.pyx:114, fused type ``real``);
    this raises the same before any device work instead of casting."""
    want = _dtype(sys_)
    if _value(sys_.layout) == "soa":
        arrays = (*sys_.positions, *sys_.velocities, sys_.masses)
    else:
        arrays = (sys_.positions, sys_.velocities, sys_.masses)
    for a in arrays:
        got = a.dtype if isinstance(a, np.ndarray) else np.asarray(a).dtype
        if got != want:
            raise ValueError(f"Buffer dtype mismatch, expected '{_CTYPE.get(want, want)}' but got "
                             f"'{_CTYPE.get(got, got)}' (system precision is {_value(sys_.precision)})")


def _check(sys_, variant, out) -> None:
    """Mirror of kernels/__init__.py:171-180."""
    if variant is not None:
        if _value(sys_.layout) != _value(variant.layout):
            raise ValueError(f"system layout {_value(sys_.layout)} does not match variant layout "
                             f"{_value(variant.layout)}")
        variant.validate_for(_count(sys_))
    if out is not None:
        if out.count != _count(sys_):
            raise ValueError("acceleration buffer length must equal the body count")
        if out.x.dtype != _dtype(sys_):
            raise ValueError("acceleration buffer precision must match the system")


def _distributed_world(group) -> int:
    import sys
    dist = sys.modules.get("torch.distributed")
    if dist is None:  # never imported: no process group can exist
        return 1
    if not dist.is_available() or not dist.is_initialized():
        return 1
    return dist.get_world_size(group)


# --------------------------------------------------------------------------- entry points

def compute_accelerations(sys_, params, variant: Optional[KernelVariant] = None,
                          out: Optional[AccelerationBuffer] = None) -> AccelerationBuffer:
    """Softened all-pairs accelerations of the current state, written into
    ``out`` (allocated if None) in the system precision; returns ``out``."""
    from .device import kernel_flags
    dtype = _dtype(sys_)
    if out is None:
        out = AccelerationBuffer.allocate(_count(sys_), _value(sys_.precision))
    _check(sys_, variant, out)
    _check_buffers(sys_)
    pos = _matrix(sys_, "positions")
    m = np.asarray(sys_.masses, dtype)
    eps2 = params.softening_sq
    z = np.zeros(pos.shape[0], dtype)
    with _STATE_LOCK:
        st = _resident_state((pos[:, 0], pos[:, 1], pos[:, 2]), (z, z, z), m, dtype)
        a = st.accelerations(params.gravitational_constant, eps2, kernel_flags(m, eps2, dtype))
        host = a[:, :3].cpu().numpy()
    out.x[...] = host[:, 0]
    out.y[...] = host[:, 1]
    out.z[...] = host[:, 2]
    return out


def integrate_step(sys_, acc: AccelerationBuffer, params, variant: Optional[KernelVariant] = None) -> None:
    """In-place kick-drift update (_accel_cy.pyx:205-237) on the GPU."""
    import torch

    from . import _native
    from .device import pack_bodies
    _check(sys_, variant, acc)
    _check_buffers(sys_)
    dtype = _dtype(sys_)
    n = _count(sys_)
    dev = torch.device("cuda", torch.cuda.current_device())
    p = pack_bodies(_matrix(sys_, "positions"), np.asarray(sys_.masses, dtype), dtype, pin=False).to(dev)
    v = pack_bodies(_matrix(sys_, "velocities"), None, dtype, pin=False).to(dev)
    a = pack_bodies(np.stack([acc.x, acc.y, acc.z], axis=1), None, dtype, pin=False).to(dev)
    sfx = "_f32" if dtype == np.float32 else "_f64"
    _native.call("nb_dev_drift" + sfx, p.data_ptr(), v.data_ptr(), a.data_ptr(), n, params.dt,
                 torch.cuda.current_stream(dev).cuda_stream)
    _store(sys_, "positions", p[:, :3].cpu().numpy())
    _store(sys_, "velocities", v[:, :3].cpu().numpy())


def simulate_arrays(positions, velocities, masses, softening_sq: float, dt: float, steps: int,
                    G: float = 1.0, precision=None, group=None) -> Tuple[np.ndarray, np.ndarray]:
    """Array form of ``simulate``: (N,3) positions and velocities and N masses in,
    final (N,3) positions and velocities out, in the input precision (float32 or
    float64; ``precision`` overrides).  Runs sharded over the process group when
    torch.distributed is initialised with more than one rank."""
    from .device import kernel_flags
    pos = np.asarray(positions)
    if precision is not None:
        dtype = Precision(_value(precision)).dtype
    else:
        dtype = pos.dtype if pos.dtype in (np.float32, np.float64) else np.dtype(np.float64)
    pos = np.ascontiguousarray(pos, dtype=dtype).reshape(-1, 3)
    vel = np.ascontiguousarray(velocities, dtype=dtype).reshape(-1, 3)
    m = np.ascontiguousarray(masses, dtype=dtype).reshape(-1)
    if not (pos.shape[0] == vel.shape[0] == m.shape[0] and pos.shape[0] >= 1):
        raise ValueError("positions, velocities and masses must describe the same N >= 1 bodies")
    if steps < 1:
        raise ValueError("steps must be >= 1")
    if not dt > 0:
        raise ValueError("dt must be positive")
    if softening_sq < 0:
        raise ValueError("softening_sq must be non-negative")
    if _distributed_world(group) > 1:
        from .sharded import simulate_sharded
        return simulate_sharded(pos, vel, m, dtype, G, dt, softening_sq, steps, group=group)
    with _STATE_LOCK:
        st = _resident_state((pos[:, 0], pos[:, 1], pos[:, 2]), (vel[:, 0], vel[:, 1], vel[:, 2]), m, dtype)
        st.simulate(G, dt, softening_sq, steps, kernel_flags(m, softening_sq, dtype))
        pc, vc = st.columns_host()
    return np.stack(pc, 1), np.stack(vc, 1)


_STATE_CACHE: dict = {}
# Calls share cached device states: one caller at a time (the reference's
# harness is single-threaded too, harness.py:5-6).
_STATE_LOCK = threading.RLock()


def _resident_state(pos, vel, m, dtype, load: bool = True):
    """A DeviceState for (N, precision, device), reused across calls so repeated
    simulate() calls pay only the H2D/D2H of their own data, not allocation
    (``load=False``: the caller uploads itself)."""
    import torch

    from .device import DeviceState
    key = (m.shape[0], np.dtype(dtype).str, torch.cuda.current_device())
    st = _STATE_CACHE.get(key)
    if st is None:
        if len(_STATE_CACHE) >= 4:
            _STATE_CACHE.clear()
        st = _STATE_CACHE[key] = DeviceState(pos, vel, m, dtype)
    elif load:
        st.load(pos, vel, m)
    return st


def simulate(sys_, params, variant: Optional[KernelVariant] = None, group=None):
    """Run ``params.steps`` velocity-Verlet steps on the GPU and return a new
    system (same class, layout and precision); ``sys_`` is not modified."""
    if variant is not None:
        _check(sys_, variant, None)
    n, dtype = _count(sys_), _dtype(sys_)
    fast = n >= 1 and params.steps >= 1 and _distributed_world(group) <= 1
    if not fast:
        _check_buffers(sys_)
        if params.steps < 1:
            raise ValueError("steps must be >= 1")
        state = sys_.copy()
        pos, vel = simulate_arrays(_matrix(sys_, "positions"), _matrix(sys_, "velocities"), sys_.masses,
                                   params.softening_sq, params.dt, params.steps,
                                   params.gravitational_constant, precision=_value(sys_.precision),
                                   group=group)
        _store(state, "positions", pos)
        _store(state, "velocities", vel)
        return state
    # Single GPU: ONE native call through the CPython binding (_hostpath, the
    # buffer protocol -- no per-array ctypes pointer extraction) into
    # nb_host_simulate: the columns are staged into the library's pinned block,
    # uploaded once, simulated (at small N the simulate kernel reads the device
    # columns and stores the final state straight into the pinned block) and
    # copied into one fresh 6*N result block; the kernel flags come from the
    # masses inside the call.
    try:
        hp, device = _host_binding()
    except (RuntimeError, ImportError, AssertionError):
        _check_buffers(sys_)  # a dtype mismatch is still the reference's ValueError, not a device error
        raise
    soa = _value(sys_.layout) == "soa"
    if soa:
        (px, py, pz), (vx, vy, vz) = sys_.positions, sys_.velocities
    else:  # (N, 3) blocks: contiguous column copies
        px, py, pz, vx, vy, vz = (np.ascontiguousarray(c) for c in
                                  (*_columns(sys_, "positions"), *_columns(sys_, "velocities")))
    out = np.empty((6, n), dtype)
    try:  # (the binding checks every buffer's item type against the precision)
        rc = hp.simulate(px, py, pz, sys_.masses, vx, vy, vz, out, params.gravitational_constant, params.dt,
                         params.softening_sq, params.steps, device(), dtype.itemsize)
    except TypeError:
        _check_buffers(sys_)  # the reference's dtype ValueError (_accel_cy.pyx:114)
        raise
    if rc:
        from . import _native
        _native.check("nb_host_simulate", rc)
    x, y, z, ux, uy, uz = out
    if soa:
        return type(sys_)(sys_.layout, sys_.precision, (x, y, z), (ux, uy, uz), sys_.masses.copy())
    return type(sys_)(sys_.layout, sys_.precision, np.stack((x, y, z), 1), np.stack((ux, uy, uz), 1),
                      sys_.masses.copy())


_HOST = None


def _host_binding():
    """(the bound _hostpath module, the current-CUDA-device function), resolved
    once: simulate()'s per-call host cost is on C1's critical path."""
    global _HOST
    if _HOST is None:
        import torch

        from . import _native
        torch.cuda.init()
        _HOST = (_native.hostpath(), torch._C._cuda_getDevice)
    return _HOST


def diagnostics_gpu(sys_, params) -> dict:
    """Kinetic and softened potential energy and momentum of a state, FP64 on
    the GPU (validation.diagnostics, validation.py:134-145, is an O(N^2) Python
    loop that is infeasible at N >= 131072)."""
    from .device import DeviceState
    dtype = _dtype(sys_)
    st = DeviceState(_matrix(sys_, "positions"), _matrix(sys_, "velocities"),
                     np.asarray(sys_.masses, dtype), dtype)
    ke, pe, mom = st.energy(params.gravitational_constant, params.softening_sq)
    return {"kinetic": ke, "potential": pe, "total": ke + pe, "momentum": mom}
