"""One nb_dev_simulate of a BASELINE config (for ncu: at small N this is the
single small-N cooperative launch).  usage: python tools/profile_simulate.py CONFIG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags

cfg = nb.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
s = cfg.system()
dt = cfg.precision.dtype
st = DeviceState(s.position_matrix().astype(dt), np.stack(s.velocities, 1), s.masses, dt)
st.simulate(1.0, cfg.dt, cfg.softening_sq, cfg.steps, kernel_flags(s.masses, cfg.softening_sq, dt))
torch.cuda.synchronize()
print("ok", cfg.name)
