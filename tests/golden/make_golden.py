"""Generate the golden fixtures under tests/golden/ by importing the Python
reference (`nbodybench`, /root/reference/pkg) in THIS container.

The reference cannot travel to the GPU box, so its outputs are frozen here as
small fixtures.  The reference package is imported from a scratch copy under
/tmp with its compiled kernel (built from its own .pyx by oracle/Makefile)
dropped in, so `nbodybench.kernels` selects its "cext" backend exactly as an
installed reference would.  Nothing is copied into this repository except the
numbers the reference produced.

Run:  python tests/golden/make_golden.py
"""
import glob
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/nbodybench"
SCRATCH = "/tmp/nbodybench_ref_import"


def import_reference():
    if os.path.isdir(SCRATCH):
        shutil.rmtree(SCRATCH)
    shutil.copytree(REF_SRC, os.path.join(SCRATCH, "nbodybench"))
    so = glob.glob(os.path.join(REPO, "oracle", "_ref", "_accel_cy*.so"))
    if not so:
        raise SystemExit("build oracle/_ref first: make -f oracle/Makefile")
    shutil.copy(so[0], os.path.join(SCRATCH, "nbodybench", "kernels", os.path.basename(so[0])))
    sys.path.insert(0, SCRATCH)
    import nbodybench as nb  # noqa: E402
    assert nb.kernels.get_backend() == "cext", nb.kernels.available_backends()
    return nb


def survey_cube(nb, n, seed, precision):
    """BASELINE uniform cube on top of the reference's own
    splitmix64 unit stream (core.py:110-113)."""
    from nbodybench.core import _units
    u = _units(seed, 7 * n).reshape(n, 7)
    pos = np.stack([-1.0 + 2.0 * u[:, k] for k in range(3)], axis=1)
    vel = np.stack([-0.1 + 0.2 * u[:, 3 + k] for k in range(3)], axis=1)
    m = 0.5 + u[:, 6]
    return nb.system_from_arrays(pos, vel, m, nb.Layout.SOA, precision)


def acc_arrays(buf):
    return np.stack([buf.x, buf.y, buf.z], axis=1)


def main():
    nb = import_reference()
    from nbodybench.validation import reference_accelerations, reference_simulate
    consts = {}
    consts["splitmix64_seed42_first16"] = [int(v) for v in nb.core.splitmix64_stream(42, 16)]
    consts["unit_doubles_seed42_first4"] = [float(v) for v in nb.core._units(42, 4)]
    consts["init_checksum_n256_seed42"] = nb.checksum(nb.init_system(256, nb.Seed(42)))
    params = nb.SimParams(1.0, 0.01, 1e-9, 10)
    final = nb.simulate(nb.init_system(256, nb.Seed(42)), params, nb.reference_variant())
    consts["sim_checksum_n256_seed42_steps10"] = nb.checksum(final)

    # C1 known answer (BASELINE.json configs[0]) with the reference's own kernels.
    c1 = survey_cube(nb, 1024, 0, nb.Precision.DOUBLE)
    c1p = nb.SimParams(1.0, 1e-2, 1e-2, 10)
    c1_final = nb.simulate(c1, c1p, nb.reference_variant())
    consts["c1_body0"] = {"pos": [float(c[0]) for c in c1.positions],
                          "vel": [float(c[0]) for c in c1.velocities],
                          "mass": float(c1.masses[0])}
    consts["c1_checksum"] = nb.checksum(c1_final)
    c1_acc = acc_arrays(reference_accelerations(c1, c1p))
    consts["c1_oracle_acc0"] = [float(v) for v in c1_acc[0]]
    from nbodybench.cli import CSV_HEADER
    consts["csv_header"] = list(CSV_HEADER)
    with open(os.path.join(HERE, "reference_constants.json"), "w") as f:
        json.dump(consts, f, indent=1)

    arrays = {}
    # C1 in full: initial state, oracle accelerations, compiled-reference final state,
    # oracle trajectory, and the reference's own FP32 run (its FP32-vs-FP64 deviation
    # calibrates the FP32 trajectory tolerance).
    arrays["c1_pos0"] = c1.position_matrix()
    arrays["c1_vel0"] = np.stack(c1.velocities, axis=1)
    arrays["c1_m"] = c1.masses.copy()
    arrays["c1_acc_oracle"] = c1_acc
    arrays["c1_pos_final"] = c1_final.position_matrix()
    arrays["c1_vel_final"] = np.stack(c1_final.velocities, axis=1)
    ref_pos, ref_vel = reference_simulate(c1, c1p)
    arrays["c1_pos_oracle"] = ref_pos
    arrays["c1_vel_oracle"] = ref_vel
    c1_32 = survey_cube(nb, 1024, 0, nb.Precision.SINGLE)
    f32 = nb.simulate(c1_32, c1p, nb.KernelVariant(nb.Layout.SOA, nb.MathForm.RECIPROCAL_MULTIPLY))
    arrays["c1_f32_pos_final"] = np.stack(f32.positions, axis=1)
    r32_pos, _ = reference_simulate(c1_32, c1p)
    arrays["c1_f32_pos_oracle"] = r32_pos

    # Ragged sizes (not multiples of any tile), both precisions, several softenings:
    # oracle accelerations on the system's own rounded inputs + the compiled
    # reference's recip-form accelerations in system precision.
    cases = []
    for n, seed, prec, eps2 in [(1, 3, "double", 0.0), (2, 5, "double", 1e-3), (3, 5, "single", 1e-3),
                                (37, 7, "double", 1e-2), (37, 7, "single", 1e-2),
                                (129, 11, "double", 1e-9), (300, 13, "single", 1e-4),
                                (513, 17, "double", 0.0), (1000, 19, "single", 1e-2)]:
        p = nb.Precision(prec)
        s = survey_cube(nb, n, seed, p)
        sp = nb.SimParams(1.0, 1e-3, eps2, 3)
        key = f"n{n}_s{seed}_{prec}_e{eps2:g}"
        cases.append({"key": key, "n": n, "seed": seed, "precision": prec, "eps2": eps2,
                      "dt": 1e-3, "steps": 3})
        arrays[key + "_acc_oracle"] = acc_arrays(reference_accelerations(s, sp))
        out = nb.AccelerationBuffer.allocate(n, p)
        nb.compute_accelerations(s, sp, nb.KernelVariant(nb.Layout.SOA, nb.MathForm.RECIPROCAL_MULTIPLY), out)
        arrays[key + "_acc_ref"] = acc_arrays(out)
        fin = nb.simulate(s, sp, nb.KernelVariant(nb.Layout.SOA, nb.MathForm.RECIPROCAL_MULTIPLY))
        arrays[key + "_pos_ref"] = np.stack(fin.positions, axis=1)
        arrays[key + "_vel_ref"] = np.stack(fin.velocities, axis=1)
        opos, ovel = reference_simulate(s, sp)
        arrays[key + "_pos_oracle"] = opos
        arrays[key + "_vel_oracle"] = ovel
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
