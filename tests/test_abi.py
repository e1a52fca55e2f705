"""CPU: the C-ABI library loads, exports every symbol include/nbody_b200.h
declares, and rejects bad arguments before touching a device."""
import ctypes
import os

import pytest

from paper_2203_08263_b200 import _native


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_native.LIB_PATH):
        from paper_2203_08263_b200 import _build
        _build.build()
    return _native.lib()


def test_exports_every_declared_symbol(lib):
    declared = _native.declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(lib, s)]
    assert missing == []


def test_only_declared_symbols_exported():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if " T " in ln})
    assert exported == _native.declared_symbols()


def test_version(lib):
    assert "sm_100a" in _native.version()


def test_library_built_from_these_sources(lib):
    """nb_version() carries the digest of the sources the library was compiled
    from; loading a library built from other sources raises (no stale .so)."""
    from paper_2203_08263_b200._build import source_digest
    assert _native.version().endswith("src:" + source_digest())
    assert _native.verify_build() == source_digest()


def test_argument_errors_without_device(lib):
    with pytest.raises(_native.NativeError) as e:
        _native.call("nb_dev_step_f32", None, 0, 0, 0, 0, 0, 1.0, 0.0, 0.0, 0, 0, None, 0,
                     None, None, None, None, 0, None)
    assert e.value.code == 1 and "target range" in str(e.value)
    with pytest.raises(_native.NativeError) as e:
        _native.call("nb_dev_step_f64", None, 10, 0, 10, 0, 10, 1.0, 1e-3, 0.0, 7, 0, None, 0,
                     None, None, None, None, 0, None)
    assert "mode" in str(e.value)
    with pytest.raises(_native.NativeError) as e:
        _native.call("nb_dev_step_f64", None, 10, 0, 10, 0, 10, 1.0, -1.0, 0.0, 0, 0, None, 0,
                     None, None, None, None, 0, None)
    assert "eps2" in str(e.value)
    with pytest.raises(_native.NativeError):
        _native.call("nb_host_simulate_soa_f32", None, None, None, None, None, None, None, 0, 1.0,
                     0.01, 0.0, 1)
    # n_i == 0 is a no-op, not an error
    _native.call("nb_dev_step_f32", None, 10, 0, 0, 0, 10, 1.0, 0.0, 0.0, 0, 0, None, 0,
                 None, None, None, None, 0, None)
    # the exchange ABI validates before it loads NCCL
    with pytest.raises(_native.NativeError) as e:
        _native.comm_init_rank(0, 0, bytes(_native.COMM_ID_BYTES))
    assert e.value.code == 1 and "rank" in str(e.value)
    with pytest.raises(_native.NativeError) as e:
        _native.comm_allgather(0, 64, 0, 0)
    assert e.value.code == 1
    with pytest.raises(ValueError):
        _native.comm_init_rank(2, 0, b"short")
    _native.comm_destroy(0)  # null communicator: no-op


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(ImportError):
        _native.lib()


def test_product_does_not_import_oracle():
    import pathlib
    import re
    pkg = pathlib.Path(_native.__file__).parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), f
        assert "liboracle" not in text and "orc_" not in text, f
