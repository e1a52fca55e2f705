"""The reference's backend plugin protocol, served by the GPU.

``nbodybench.kernels`` selects a backend module with ``NAME``, ``accel_soa``,
``accel_aos``, ``step_soa`` and ``step_aos`` (kernels/__init__.py:38-79; the
signatures are those of _accel_cy.pyx:114,155,205,240).  This module provides
exactly that protocol on top of the host-pointer C ABI (``nb_host_*``), so a
maintainer can register it as one more entry of the reference's ``_BACKENDS``
(INTEGRATION.md).  Every call copies its arrays to the device and back; the
device-resident path is ``paper_2203_08263_b200.simulate``.
"""

from __future__ import annotations

import numpy as np

from . import _native

NAME = "b200"


def _sfx(a: np.ndarray) -> str:
    if a.dtype == np.float32:
        return "_f32"
    if a.dtype == np.float64:
        return "_f64"
    raise ValueError(f"Buffer dtype mismatch: unsupported dtype {a.dtype}")


def _same(dtype, *arrays) -> None:
    for a in arrays:
        if a.dtype != dtype:
            raise ValueError(f"Buffer dtype mismatch, expected '{dtype}' but got '{a.dtype}'")
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("ndarray is not C-contiguous")


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def accel_soa(px, py, pz, m, g, eps2, recip, block, threads, ax, ay, az) -> None:
    _same(px.dtype, py, pz, m, ax, ay, az)
    n = px.shape[0]
    _native.call("nb_host_accel_soa" + _sfx(px), _p(px), _p(py), _p(pz), _p(m), n, float(g),
                 float(eps2), int(bool(recip)), int(block), int(threads), _p(ax), _p(ay), _p(az))


def accel_aos(pos, m, g, eps2, ax, ay, az) -> None:
    _same(pos.dtype, m, ax, ay, az)
    n = pos.shape[0]
    _native.call("nb_host_accel_aos" + _sfx(pos), _p(pos), _p(m), n, float(g), float(eps2),
                 _p(ax), _p(ay), _p(az))


def step_soa(px, py, pz, vx, vy, vz, ax, ay, az, dt, threads) -> None:
    _same(px.dtype, py, pz, vx, vy, vz, ax, ay, az)
    n = px.shape[0]
    _native.call("nb_host_step_soa" + _sfx(px), _p(px), _p(py), _p(pz), _p(vx), _p(vy), _p(vz),
                 _p(ax), _p(ay), _p(az), n, float(dt), int(threads))


def step_aos(pos, vel, ax, ay, az, dt) -> None:
    _same(pos.dtype, vel, ax, ay, az)
    n = pos.shape[0]
    _native.call("nb_host_step_aos" + _sfx(pos), _p(pos), _p(vel), _p(ax), _p(ay), _p(az), n,
                 float(dt))


def simulate_soa(px, py, pz, vx, vy, vz, m, g, dt, eps2, steps) -> None:
    """Whole kernels.simulate loop on the device, in place on SoA host arrays."""
    _same(px.dtype, py, pz, vx, vy, vz, m)
    n = px.shape[0]
    _native.call("nb_host_simulate_soa" + _sfx(px), _p(px), _p(py), _p(pz), _p(vx), _p(vy), _p(vz),
                 _p(m), n, float(g), float(dt), float(eps2), int(steps))
