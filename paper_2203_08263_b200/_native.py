"""ctypes binding of libnbody_b200.so (the C ABI in include/nbody_b200.h).

There is no fallback: if the shared library is missing or fails to load, every
entry point raises.  Build it with ``python -m paper_2203_08263_b200._build``
(or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
import re
from typing import Optional

_PKG = os.path.dirname(os.path.abspath(__file__))
# NB_LIB_PATH selects another build of the same ABI (e.g. the bounds-checked one
# from tools/check_build.sh); the default is the in-tree release library.
LIB_PATH = os.environ.get("NB_LIB_PATH") or os.path.join(_PKG, "libnbody_b200.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "nbody_b200.h")

NB_MODE_ACCEL = 0
NB_STEP_FIRST = 1
NB_STEP_KICK_DRIFT = 2
NB_STEP_FINAL_KICK = 3
NB_FLAG_EXCLUDE_SELF = 1
NB_FLAG_UNIFORM_MASS = 2
NB_FLAG_AUTO = 256  # nb_dev_simulate_cols_*: flags derived from the staged masses in C
NB_INIT_UNIFORM_CUBE = 0
NB_INIT_PLUMMER = 1

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
_i = ctypes.c_int

_ARGTYPES = {
    "nb_host_accel_soa": [_p] * 4 + [_i64, _d, _d, _i, _i64, _i] + [_p] * 3,
    "nb_host_accel_aos": [_p, _p, _i64, _d, _d] + [_p] * 3,
    "nb_host_step_soa": [_p] * 9 + [_i64, _d, _i],
    "nb_host_step_aos": [_p] * 5 + [_i64, _d],
    "nb_host_simulate_soa": [_p] * 7 + [_i64, _d, _d, _d, _i64],
    "nb_host_simulate": [_p] * 7 + [_i64, _d, _d, _d, _i64, _p, _i],
    "nb_dev_step": [_p, _i64, _i64, _i64, _i64, _i64, _d, _d, _d, _i, _i, _p, _i, _p, _p, _p, _p, _i64, _p],
    "nb_dev_step_p2p": [_p, _i64, _i64, _i64, _i64, _i64, _d, _d, _d, _i, _i, _p, _i, _p, _p, _p, _p, _i, _p,
                        _i64, _p],
    "nb_dev_simulate": [_p, _p, _p, _p, _i64, _d, _d, _d, _i64, _i, _p, _i64, _p, ctypes.POINTER(_i)],
    "nb_dev_simulate_timed": [_p, _p, _p, _p, _i64, _d, _d, _d, _i64, _i, _p, _i64, _p, ctypes.POINTER(_i),
                              ctypes.POINTER(ctypes.c_float)],
    "nb_dev_pack": [_p, _p, _p, _p, _i64, _p, _p],
    "nb_dev_unpack": [_p, _i64, _p, _p, _p, _p],
    "nb_force": [_p, _i64, _i64, _i64, _d, _d, _p, _p, _i64, _p],
    "nb_update": [_p, _p, _p, _p, _p, _i64, _d, _i, _p],
    "nb_dev_simulate_cols": [_p, _p, _p, _p, _p, _p, _i64, _d, _d, _d, _i64, _i, _p, _i64, _p, ctypes.POINTER(_i)],
    "nb_dev_load_cols": [_p, _p, _i64, _i64, _p, _p, _p],
    "nb_dev_store_cols": [_p, _p, _i64, _i64, _p, _p, _p],
    "nb_dev_drift": [_p, _p, _p, _i64, _d, _p],
    "nb_dev_kick": [_p, _p, _p, _i64, _d, _p],
    "nb_dev_energy": [_p, _p, _i64, _d, _d, _p, _p, _i64, _p],
    "nb_dev_init": [_i, ctypes.c_uint64, _i64, _p, _p, _p],
}

_lib: Optional[ctypes.CDLL] = None


class NativeError(RuntimeError):
    """A nonzero return code from libnbody_b200 (message from nb_last_error)."""

    def __init__(self, func: str, code: int, message: str):
        super().__init__(f"{func} failed with code {code}: {message}")
        self.code = code


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA extension has not been built "
                "(run `python -m paper_2203_08263_b200._build`); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for base, args in _ARGTYPES.items():
            for sfx in ("_f32", "_f64"):
                fn = getattr(L, base + sfx)
                fn.argtypes = args
                fn.restype = _i
        L.nb_dev_workspace_bytes.argtypes = [_i, _i64]
        L.nb_dev_workspace_bytes.restype = _i64
        L.nb_dev_step_kernel.argtypes = [_i, _i64, _i64]
        L.nb_dev_step_kernel.restype = ctypes.c_char_p
        L.nb_energy_workspace_bytes.argtypes = [_i, _i64]
        L.nb_energy_workspace_bytes.restype = _i64
        L.nb_comm_unique_id.argtypes = [_p]
        L.nb_comm_init_rank.argtypes = [_i, _i, _p, ctypes.POINTER(_p)]
        L.nb_comm_init_all.argtypes = [_i, ctypes.POINTER(_i), ctypes.POINTER(_p)]
        L.nb_comm_allgather.argtypes = [_p, ctypes.c_size_t, _p, _p]
        L.nb_comm_allgather_all.argtypes = [ctypes.POINTER(_p), ctypes.c_size_t, ctypes.POINTER(_p),
                                            ctypes.POINTER(_p), _i]
        L.nb_comm_destroy.argtypes = [_p]
        for f in ("nb_comm_unique_id", "nb_comm_init_rank", "nb_comm_init_all", "nb_comm_allgather",
                  "nb_comm_allgather_all", "nb_comm_destroy"):
            getattr(L, f).restype = _i
        L.nb_last_error.restype = ctypes.c_char_p
        L.nb_version.restype = ctypes.c_char_p
        L.nb_launch_count.restype = _i64
        _check_digest(L)
        _lib = L
    return _lib


_hostpath = None


def hostpath():
    """The CPython binding of nb_host_simulate_f32/f64 (csrc/hostpath.c), bound
    to this process's loaded library.  ImportError if it was not built: the
    product path has no fallback."""
    global _hostpath
    if _hostpath is None:
        L = lib()
        from . import _hostpath as H  # built next to the library by _build.build()
        H.bind(ctypes.cast(L.nb_host_simulate_f32, ctypes.c_void_p).value,
               ctypes.cast(L.nb_host_simulate_f64, ctypes.c_void_p).value)
        _hostpath = H
    return _hostpath


def check(name: str, rc: int) -> None:
    """Raise NativeError for a nonzero C ABI status returned by ``name``."""
    if rc != 0:
        msg = lib().nb_last_error()
        raise NativeError(name, rc, msg.decode() if msg else "")


def call(name: str, *args) -> None:
    """Call an int-returning entry point and raise NativeError on failure."""
    L = lib()
    rc = getattr(L, name)(*args)
    if rc != 0:
        msg = L.nb_last_error()
        raise NativeError(name, rc, msg.decode() if msg else "")


COMM_ID_BYTES = 128


def comm_unique_id() -> bytes:
    """NB_COMM_ID_BYTES of NCCL unique id (rank 0 makes it, the host shares it)."""
    buf = ctypes.create_string_buffer(COMM_ID_BYTES)
    call("nb_comm_unique_id", buf)
    return buf.raw


def comm_init_rank(nranks: int, rank: int, uid: bytes) -> int:
    """Opaque NCCL communicator handle for one rank (nb_comm_init_rank)."""
    if len(uid) != COMM_ID_BYTES:
        raise ValueError(f"unique id must be {COMM_ID_BYTES} bytes")
    out = ctypes.c_void_p()
    call("nb_comm_init_rank", nranks, rank, ctypes.create_string_buffer(uid, COMM_ID_BYTES), ctypes.byref(out))
    return int(out.value)


def comm_allgather(buf_ptr: int, bytes_per_rank: int, comm: int, stream: int) -> None:
    call("nb_comm_allgather", buf_ptr, bytes_per_rank, comm, stream)


def comm_destroy(comm: int) -> None:
    call("nb_comm_destroy", comm)


def energy_workspace_bytes(precision_bytes: int, n: int) -> int:
    return int(lib().nb_energy_workspace_bytes(precision_bytes, n))


def workspace_bytes(precision_bytes: int, n_i: int) -> int:
    return int(lib().nb_dev_workspace_bytes(precision_bytes, n_i))


def step_kernel_name(precision_bytes: int, n_i: int, j_count: int) -> str:
    """The force kernel nb_dev_step runs for this launch shape (current device)."""
    return lib().nb_dev_step_kernel(precision_bytes, n_i, j_count).decode()


def launch_count() -> int:
    return int(lib().nb_launch_count())


def version() -> str:
    return lib().nb_version().decode()


def _check_digest(L) -> None:
    from ._build import source_digest
    want = source_digest()
    got = L.nb_version().decode().rsplit("src:", 1)[-1]
    if got != want:
        raise ImportError(f"{LIB_PATH} was built from sources {got}, but the tree holds {want}: "
                          "rebuild with `python -m paper_2203_08263_b200._build` (no stale prebuilt library "
                          "stands in for the current sources)")


def verify_build() -> str:
    """Raise if the loaded library was not compiled from the sources in this
    tree (nb_version()'s src: digest vs _build.source_digest()); returns the digest."""
    _check_digest(lib())
    return version().rsplit("src:", 1)[-1]


def declared_symbols(header: str = HEADER) -> list:
    """Function names declared in include/nbody_b200.h."""
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nb_[a-z0-9_]+)\s*\(", text)))
