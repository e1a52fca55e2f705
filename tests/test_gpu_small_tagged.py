"""The small-N kernel's tagged position exchange (small_simulate_kernel,
nbody_force.cu): between the first and the last drift of a launch the bodies are
published as single coherent records whose fourth word is the step tag, and the
next step's staging polls for that tag instead of crossing a grid barrier.

* NB_SMALL_TAGGED=1 (default) and =0 (a grid barrier per step) give bitwise the
  same final state -- the exchange only changes when data becomes visible;
* repeated launches on the same resident buffers (stale tags of earlier launches
  in the scratch buffer) reproduce the first result bit for bit;
* the trajectory matches the oracle (FP64 1e-12, FP32 <= 10x the
  reference's own FP32 deviation, here a fixed 2e-5 at these sizes);
* the packed device state keeps real masses in the current buffer afterwards
  (other kernels read them there).
Covers FP64/FP32, 8- and 16-target CTAs, uniform masses (m applied once from
shared memory), eps2 = 0 (self mask), steps 1..3 (no tagged step) and odd/even
step counts (which buffer ends up current)."""
import hashlib
import json
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import paper_2203_08263_b200 as nb

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

# (name, n, precision, generator, eps2, dt, steps)
CASES = [
    ("c1", 1024, "double", "uniform_cube", 1e-2, 1e-2, 10),
    ("f64_odd_steps", 1000, "double", "uniform_cube", 1e-3, 1e-3, 7),
    ("f64_16_targets", 2304, "double", "uniform_cube", 1e-2, 1e-3, 6),
    ("f64_self_mask", 777, "double", "uniform_cube", 0.0, 1e-4, 5),
    ("f32", 2000, "single", "uniform_cube", 1e-2, 1e-2, 9),
    ("f32_uniform_mass", 3000, "single", "plummer_sphere", 1e-4, 1e-4, 8),
    ("f32_16_targets", 4096, "single", "uniform_cube", 1e-2, 1e-3, 4),
    ("f64_three_steps", 512, "double", "uniform_cube", 1e-2, 1e-2, 3),
    ("f64_two_steps", 512, "double", "uniform_cube", 1e-2, 1e-2, 2),
    ("f64_one_step", 512, "double", "uniform_cube", 1e-2, 1e-2, 1),
]

SCRIPT = textwrap.dedent(f"""
    import hashlib, json, sys, numpy as np
    sys.path.insert(0, {REPO!r})
    import paper_2203_08263_b200 as nb
    out = {{}}
    for name, n, prec, gen, eps2, dt, steps in json.loads(sys.argv[1]):
        s = getattr(nb, gen)(n, 5, nb.Precision(prec))
        fin = nb.simulate(s, nb.SimParams(1.0, dt, eps2, steps))
        h = hashlib.sha256()
        for a in list(fin.positions) + list(fin.velocities):
            h.update(np.ascontiguousarray(a).tobytes())
        out[name] = h.hexdigest()
    print(json.dumps(out))
""")


def _digest(sys_out):
    h = hashlib.sha256()
    for a in list(sys_out.positions) + list(sys_out.velocities):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _run(tagged):
    env = dict(os.environ, NB_SMALL_TAGGED=str(tagged))
    r = subprocess.run([sys.executable, "-c", SCRIPT, json.dumps(CASES)], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_tagged_exchange_bitwise_equals_grid_barrier():
    on, off = _run(1), _run(0)
    assert set(on) == {c[0] for c in CASES}
    for name in on:
        assert on[name] == off[name], name
    # and the in-process default (tagged) agrees with both
    name, n, prec, gen, eps2, dt, steps = CASES[0]
    s = getattr(nb, gen)(n, 5, nb.Precision(prec))
    assert _digest(nb.simulate(s, nb.SimParams(1.0, dt, eps2, steps))) == on[name]


@pytest.mark.parametrize("case", CASES[:7], ids=[c[0] for c in CASES[:7]])
def test_tagged_exchange_vs_oracle(case, oracle):
    name, n, prec, gen, eps2, dt, steps = case
    s = getattr(nb, gen)(n, 5, nb.Precision(prec))
    p = nb.SimParams(1.0, dt, eps2, steps)
    fin = nb.simulate(s, p).position_matrix().astype(np.float64)
    pos = s.position_matrix().astype(np.float64)
    ref, _ = oracle.simulate(pos, np.stack(s.velocities, 1).astype(np.float64), s.masses.astype(np.float64),
                             1.0, dt, eps2, steps, threads=oracle.host_threads())
    dev = oracle.position_dev(fin, ref)
    print(name, "position_dev", dev)
    assert dev <= (1e-12 if prec == "double" else 2e-5)


@pytest.mark.parametrize("prec,n,steps", [("double", 1024, 10), ("double", 900, 7), ("single", 2000, 6)])
def test_repeated_launches_on_resident_buffers(prec, n, steps):
    """Device-resident path: the same DeviceState simulated again from a restored
    initial state (its scratch buffer now holds the first launch's tags) gives the
    same bits, and the current buffer holds the real masses afterwards."""
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    s = nb.uniform_cube(n, 9, nb.Precision(prec))
    dtype = s.precision.dtype
    pos = s.position_matrix().astype(dtype)
    vel = np.stack(s.velocities, 1)
    flags = kernel_flags(s.masses, 1e-2, dtype)
    st = DeviceState(pos, vel, s.masses, dtype)
    first = None
    for rep in range(3):
        st.load(pos, vel, s.masses)
        st.simulate(1.0, 1e-2, 1e-2, steps, flags)
        cur = st.pos_cur.cpu().numpy()
        assert np.array_equal(cur[:, 3], s.masses.astype(dtype)), "current buffer must hold the masses"
        got = (cur[:, :3].copy(), st.vel.cpu().numpy()[:, :3].copy())
        if first is None:
            first = got
        else:
            assert np.array_equal(first[0], got[0]) and np.array_equal(first[1], got[1]), rep
    # the accelerations of the final state through the per-launch kernels read that buffer
    a = st.accelerations(1.0, 1e-2, flags)[:, :3].cpu().numpy()
    assert np.all(np.isfinite(a))
