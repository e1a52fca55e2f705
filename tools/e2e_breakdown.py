"""Where the end-to-end simulate() time goes beyond the device loop (C3-f32).
usage: python tools/e2e_breakdown.py [CONFIG]"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import kernels as K
from paper_2203_08263_b200.device import kernel_flags

cfg = nb.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3-f32"]
s, p = cfg.system(), cfg.params()
dt = cfg.precision.dtype
for _ in range(2):
    nb.simulate(s, p)
torch.cuda.synchronize()
T = {}
def tick(name, t0):
    torch.cuda.synchronize()
    T[name] = T.get(name, 0.0) + time.perf_counter() - t0
    return time.perf_counter()
R = 5
for _ in range(R):
    t = time.perf_counter()
    m = np.asarray(s.masses, dt)
    fl = kernel_flags(m, p.softening_sq, dt)
    t = tick("flags", t)
    st = K._resident_state(K._columns(s, "positions"), K._columns(s, "velocities"), m, dt)
    t = tick("load (pack + H2D)", t)
    st.simulate(p.gravitational_constant, p.dt, p.softening_sq, p.steps, fl)
    t = tick("device simulate", t)
    pos, vel = st.columns_host()
    t = tick("unpack + D2H + split", t)
    type(s)(s.layout, s.precision, pos, vel, s.masses.copy())
    t = tick("result object", t)
t0 = time.perf_counter()
for _ in range(R):
    nb.simulate(s, p)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / R
for k, v in T.items():
    print(f"{k:22s} {1e3 * v / R:8.3f} ms")
print(f"{'simulate() total':22s} {1e3 * tot:8.3f} ms")
