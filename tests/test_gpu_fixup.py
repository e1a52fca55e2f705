"""The split-i-block fixup inside the step kernel (ready flags per partial slot,
each contributor finishing its share; NB_FIXUP_KERNEL=0 -- an opt-in variant,
measured slower) against the separate fixup_kernel launch (the shipped
default, NB_FIXUP_KERNEL=1): the same partial sums in the same
ascending CTA order, so the trajectories must be bitwise identical -- at the
C2 size (11 i-blocks over 148 CTAs: every i-block split), FP64, a ragged N, a
sharded two-phase (carry) step and the uniform-mass path."""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

SCRIPT = textwrap.dedent(f"""
    import sys, numpy as np
    sys.path.insert(0, {REPO!r})
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    out = {{}}
    for name, n, prec, gen, eps2 in [("c2", 16384, "single", nb.uniform_cube, 1e-2),
                                     ("f64", 20000, "double", nb.uniform_cube, 1e-3),
                                     ("ragged", 12345, "single", nb.uniform_cube, 0.0),
                                     ("uni", 30000, "single", nb.plummer_sphere, 1e-4)]:
        s = gen(n, 1, nb.Precision(prec))
        fin = nb.simulate(s, nb.SimParams(1.0, 1e-3, eps2, 3))
        out[name] = np.concatenate([fin.position_matrix(), np.stack(fin.velocities, 1).astype(np.float64)], 1)
    # one rank of a 3-way shard: local sources into the carry, then the circular remainder
    s = nb.uniform_cube(24001, 2, nb.Precision.SINGLE)
    st = DeviceState(s.position_matrix().astype(np.float32), np.stack(s.velocities, 1), s.masses, np.float32,
                     i_begin=8000, n_i=8000)
    f = kernel_flags(s.masses, 1e-3, np.float32)
    st.step(1.0, 1e-3, 1e-3, 1, f, j_begin=8000, j_count=8000, carry_mode=1)
    st.step(1.0, 1e-3, 1e-3, 1, f, j_begin=16000, j_count=24001 - 8000, carry_mode=2)
    st.swap()
    out["shard"] = st.pos_cur.cpu().numpy().astype(np.float64)
    np.savez(sys.argv[1], **out)
""")


def _run(path, fixup_kernel):
    # NB_PAIR=0: the stream-K path (C2-sized FP32 launches would take pair_kernel)
    env = dict(os.environ, NB_FIXUP_KERNEL="1" if fixup_kernel else "0", NB_PAIR="0")
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(path)], capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return dict(np.load(path))


def test_in_kernel_fixup_bitwise_equals_fixup_kernel(tmp_path):
    a = _run(tmp_path / "infix.npz", False)
    b = _run(tmp_path / "fixk.npz", True)
    assert sorted(a) == sorted(b)
    for k in a:
        assert np.all(np.isfinite(a[k][:, :3])), k
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
