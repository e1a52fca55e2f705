"""pytest plugin for the drop-in test (tests/test_gpu_dropin.py): run the
reference's OWN test suite -- baseline/_ref/_tests, copied by
``__graft_entry__.build()`` from /root/reference/pkg/tests next to the installed
reference package -- with this repo's GPU backend registered in the installed
reference's backend table and made the active default.

That is the maintainer-side integration INTEGRATION.md describes: one more entry
in ``nbodybench.kernels._BACKENDS`` (the plugin protocol of
/root/reference/pkg/src/nbodybench/kernels/__init__.py:38-79) and
``set_backend``.  The conftest's ``backend`` fixture is parametrised over
``available_backends()`` when it is imported, after this plugin, so every
backend-parametrised reference test also runs on "b200"; every test that uses
the active default backend (harness.measure, the acceptance gates) runs on it.

NB_REF_BINDING selects the module registered: "python" (paper_2203_08263_b200.
backend, ctypes over the C ABI) or "cython" (integration/_accel_b200, the typed
memoryview binding of INTEGRATION.md section 3).
"""
import glob
import importlib.util
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
sys.path.insert(1, REPO)

import nbodybench  # noqa: E402  (the installed, unmodified reference)
from nbodybench import kernels as _K  # noqa: E402


def _binding():
    which = os.environ.get("NB_REF_BINDING", "python")
    if which == "cython":
        path = glob.glob(os.path.join(REPO, "integration", "_accel_b200*.so"))[0]
        spec = importlib.util.spec_from_file_location("_accel_b200", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod
    from paper_2203_08263_b200 import backend
    return backend


_mod = _binding()
assert _mod.NAME == "b200"
_K._BACKENDS["b200"] = _mod
nbodybench.set_backend("b200")


def pytest_report_header(config):
    return [f"reference package: {nbodybench.__file__}",
            f"registered backend b200 = {_mod.__name__} ({getattr(_mod, '__file__', '?')}); active: "
            f"{nbodybench.get_backend()}"]
