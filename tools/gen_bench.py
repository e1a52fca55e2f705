"""Measure on-device input generation: nb_dev_init at the
BASELINE sizes, bodies/s and written bytes/s against the measured HBM copy
bandwidth (MEASURED_PEAKS.json).  CUDA events, best of 5 after a warm-up.
usage: python tools/gen_bench.py > profiles/generators_r01.md"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2203_08263_b200 import _native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    HBM = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
except (OSError, KeyError, ValueError):
    HBM = 7700.0
print("# On-device BASELINE generators (nb_dev_init), one B200\n")
print(f"Writes (x,y,z,m) and (vx,vy,vz,0) per body; HBM peak {HBM:.0f} GB/s (MEASURED_PEAKS.json copy).\n")
print("| generator | precision | N | t (ms) | bodies/s | written GB/s | frac of HBM |")
print("|---|---|---|---|---|---|---|")
for kind, code in (("uniform_cube", _native.NB_INIT_UNIFORM_CUBE), ("plummer_sphere", _native.NB_INIT_PLUMMER)):
    for dt, sfx in ((torch.float32, "_f32"), (torch.float64, "_f64")):
        n = 4194304
        pos = torch.empty((n, 4), dtype=dt, device="cuda")
        vel = torch.empty_like(pos)
        s = torch.cuda.current_stream().cuda_stream
        run = lambda: _native.call("nb_dev_init" + sfx, code, 0, n, pos.data_ptr(), vel.data_ptr(), s)
        run()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); run(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        nbytes = 2 * pos.numel() * pos.element_size()
        gbs = nbytes / (best / 1e3) / 1e9
        print(f"| {kind} | {sfx[1:]} | {n} | {best:.3f} | {n / (best / 1e3):.3e} | {gbs:.0f} | {gbs / HBM:.3f} |",
              flush=True)
