cd $GRAFT_REPO_ROOT
python tools/profile_step.py C2 20 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_elapsed.avg --clock-control none --csv --log-file gpurun_out/launches_C2.csv python tools/profile_step.py C2 20 > gpurun_out/ncu_launch.log 2>&1
python - > gpurun_out/c2_timing.log 2>&1 <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags
cfg = nb.BASELINE_CONFIGS["C2"]; s = cfg.system(); dt = cfg.precision.dtype
st = DeviceState(s.position_matrix().astype(dt), np.stack(s.velocities, 1), s.masses, dt)
f = kernel_flags(s.masses, cfg.softening_sq, dt)
for _ in range(3): st.simulate(1.0, cfg.dt, cfg.softening_sq, cfg.steps, f)
ms = st.simulate_timed(1.0, cfg.dt, cfg.softening_sq, cfg.steps, f)
print("per-launch ms (events between launches):", np.mean(ms), np.min(ms), np.max(ms))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); st.simulate(1.0, cfg.dt, cfg.softening_sq, cfg.steps, f); e1.record(); torch.cuda.synchronize()
print("simulate ms", e0.elapsed_time(e1), "per step", e0.elapsed_time(e1) / (cfg.steps + 1))
PY
