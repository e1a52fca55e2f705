"""Host-side cost of the pieces of simulate() at small N (C1), each timed alone
over many repetitions (perf_counter; the GPU pieces with a synchronize).
usage: python tools/host_overhead.py [CONFIG]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import _native, kernels as K
from paper_2203_08263_b200.device import kernel_flags

cfg = nb.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
s, p = cfg.system(), cfg.params()
dt = cfg.precision.dtype
m = np.asarray(s.masses, dt)
for _ in range(3):
    nb.simulate(s, p)
torch.cuda.synchronize()
st = K._resident_state(K._columns(s, "positions"), K._columns(s, "velocities"), m, dt)
REP = 200


def t(name, f, sync=False):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(REP):
        f()
        if sync:
            torch.cuda.synchronize()
    dt_ = (time.perf_counter() - t0) / REP
    print(f"{name:44s} {dt_ * 1e6:8.1f} us", flush=True)


t("torch.cuda.synchronize (idle)", lambda: torch.cuda.synchronize())
t("kernel_flags", lambda: kernel_flags(m, p.softening_sq, dt))
t("ctypes no-op call (nb_launch_count)", lambda: _native.launch_count())
t("st.load (host part, async)", lambda: st.load(K._columns(s, "positions"), K._columns(s, "velocities"), m))
t("st.load + sync", lambda: st.load(K._columns(s, "positions"), K._columns(s, "velocities"), m), sync=True)
f = kernel_flags(m, p.softening_sq, dt)
t("st.simulate (host part, async)", lambda: st.simulate(1.0, p.dt, p.softening_sq, p.steps, f))
t("st.simulate + sync", lambda: st.simulate(1.0, p.dt, p.softening_sq, p.steps, f), sync=True)
t("st.columns_host (syncs)", lambda: st.columns_host())
t("d_cols.copy_(h_cols) H2D + sync", lambda: st._d_cols.copy_(st._h_cols, non_blocking=True), sync=True)
t("h_cols.copy_(d_cols) D2H (syncs)", lambda: st._h_cols.copy_(st._d_cols))
t("nb.simulate end to end", lambda: nb.simulate(s, p))
pc, vc = K._columns(s, "positions"), K._columns(s, "velocities")
t("st._fill_staging (python)", lambda: st._fill_staging(pc, vc, m))
t("st._staged_columns (python)", lambda: st._staged_columns())
t("st.simulate_columns (one native call, syncs)",
  lambda: st.simulate_columns(pc, vc, m, 1.0, p.dt, p.softening_sq, p.steps, _native.NB_FLAG_AUTO))
t("nb.simulate end to end (again)", lambda: nb.simulate(s, p))
