"""Rate of the FP32 step kernel with random masses vs equal masses (the
uniform-mass variant skips one FMUL2 per interaction pair) on the same state.
usage: python tools/uni_probe.py [CONFIG ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags

for name in sys.argv[1:] or ["C3-f32", "C2"]:
    cfg = nb.BASELINE_CONFIGS[name]
    s = cfg.system()
    dt_ = cfg.precision.dtype
    for label, m in (("random masses", s.masses), ("equal masses", np.ones(cfg.n, dtype=dt_))):
        st = DeviceState(s.position_matrix().astype(dt_), np.stack(s.velocities, 1), m, dt_)
        f = kernel_flags(m, cfg.softening_sq, dt_)
        st.simulate(1.0, cfg.dt, cfg.softening_sq, cfg.steps, f)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); st.simulate(1.0, cfg.dt, cfg.softening_sq, cfg.steps, f); e1.record()
            torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 1e3)
        rate = cfg.interactions / best
        print(f"{name:8s} {label:14s} flags={f} rate={rate:.4e} frac={20 * rate / 74.44992e12:.4f}", flush=True)
