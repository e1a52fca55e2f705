"""B200-native all-pairs N-body hot path behind the reference's N-body entry point.

Drop-in for the force/integrate path of ``nbodybench`` (arXiv 2203.08263
artifact): ``simulate``, ``compute_accelerations`` and ``integrate_step`` take
the reference's own argument objects and return the same types, computed by
hand-written sm_100a CUDA kernels in ``libnbody_b200.so`` (C ABI in
``include/nbody_b200.h``).  There is no CPU fallback.
"""

from .core import (BASELINE_CONFIGS, BaselineConfig, Layout, ParticleSystem, Precision, Seed,
                   SimParams, checksum, convert_layout, format_checksum, init_system,
                   plummer_sphere, splitmix64_stream, system_from_arrays, uniform_cube)
from .kernels import (AccelerationBuffer, KernelVariant, MathForm, compute_accelerations,
                      diagnostics_gpu, integrate_step, ladder, reference_variant, simulate,
                      simulate_arrays)

__version__ = "0.1.0"

__all__ = [
    "Layout", "ParticleSystem", "Precision", "Seed", "SimParams", "checksum",
    "convert_layout", "format_checksum", "init_system", "system_from_arrays",
    "splitmix64_stream", "uniform_cube", "plummer_sphere", "BaselineConfig",
    "BASELINE_CONFIGS", "AccelerationBuffer", "KernelVariant", "MathForm",
    "compute_accelerations", "integrate_step", "simulate", "simulate_arrays",
    "reference_variant", "ladder", "diagnostics_gpu", "__version__",
]
