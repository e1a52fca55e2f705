"""Launch a few fused step kernels on a BASELINE config (for ncu).
usage: python tools/profile_step.py CONFIG LAUNCHES"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags
from paper_2203_08263_b200._native import NB_STEP_FIRST, NB_STEP_KICK_DRIFT

name = sys.argv[1] if len(sys.argv) > 1 else "C3-f32"
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = nb.BASELINE_CONFIGS[name]
s = cfg.system()
dt = cfg.precision.dtype
st = DeviceState(s.position_matrix().astype(dt), np.stack(s.velocities, 1), s.masses, dt)
mask = kernel_flags(s.masses, cfg.softening_sq, dt)
for k in range(launches):
    st.step(1.0, cfg.softening_sq, cfg.dt, NB_STEP_FIRST if k == 0 else NB_STEP_KICK_DRIFT, mask)
    st.swap()
torch.cuda.synchronize()
print("ok", name, launches)
