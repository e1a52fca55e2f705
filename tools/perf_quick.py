"""Quick device-resident timing of the fused step kernels for the BASELINE configs."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags

PEAK32 = 148 * 128 * 2 * 1.965e9
PEAK64 = PEAK32 / 2
names = sys.argv[1:] or ["C2", "C3-f32", "C3-f64"]
for name in names:
    cfg = nb.BASELINE_CONFIGS[name]
    s = cfg.system()
    pos = s.position_matrix().astype(cfg.precision.dtype); vel = np.stack(s.velocities, 1)
    st = DeviceState(pos, vel, s.masses, cfg.precision.dtype)
    mask = kernel_flags(s.masses, cfg.softening_sq, cfg.precision.dtype)
    p = cfg.params()
    for _ in range(2):
        st.simulate(1.0, p.dt, p.softening_sq, p.steps, mask)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(5):
        e0.record(); st.simulate(1.0, p.dt, p.softening_sq, p.steps, mask); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = min(times)
    inter = cfg.interactions / t
    peak = PEAK32 if cfg.precision is nb.Precision.SINGLE else PEAK64
    print(json.dumps({"cfg": name, "t_s": t, "inter_per_s": inter, "gflops20": 20 * inter / 1e9,
                      "frac_nominal": 20 * inter / peak}), flush=True)
