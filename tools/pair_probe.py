"""Per-launch time of the FP32 force pass (mode ACCEL, back-to-back launches on
one stream, PDL intact) at arbitrary N, for the cluster split-source kernel vs
stream-K (run once with NB_PAIR=1 and once with NB_PAIR=0).
usage: NB_PAIR=0|1 python tools/pair_probe.py N [N ...] [--j J,J,...]
(--j: also time each N's targets against only the first J sources: the slope
over J is the source loop's rate, the intercept the per-launch fixed cost)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags
from paper_2203_08263_b200._native import NB_MODE_ACCEL

CLK = 1.965e9
PREC = nb.Precision(os.environ.get("NB_PROBE_PREC", "single"))  # NB_PROBE_PREC=double: the FP64 kernels
DT = PREC.dtype
LANES = 256 if PREC is nb.Precision.SINGLE else 128
js = []
if "--j" in sys.argv:
    k = sys.argv.index("--j")
    js = [int(v) for v in sys.argv[k + 1].split(",")]
    del sys.argv[k:k + 2]
for n in [int(a) for a in sys.argv[1:]]:
    s = nb.uniform_cube(n, 0, PREC)
    st = DeviceState(s.position_matrix().astype(DT), np.stack(s.velocities, 1), s.masses, DT)
    flags = kernel_flags(s.masses, 1e-3, DT)
    reps = max(10, int(2e11 / (n * n)))
    for _ in range(3):
        st.step(1.0, 1e-3, 0.0, NB_MODE_ACCEL, flags)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(reps):
            st.step(1.0, 1e-3, 0.0, NB_MODE_ACCEL, flags)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3 / reps)
    inter = float(n) * n
    print(json.dumps({"n": n, "pair": os.environ.get("NB_PAIR", "auto"), "us": best * 1e6,
                      "frac_nominal": 20 * inter / best / (148 * LANES * CLK),
                      "int_per_clk_sm": inter / best / CLK / 148}), flush=True)
    for j in js:
        def run():
            st.step(1.0, 1e-3, 0.0, NB_MODE_ACCEL, flags, j_begin=0, j_count=j)
        run()
        torch.cuda.synchronize()
        t = 1e9
        for _ in range(3):
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            t = min(t, e0.elapsed_time(e1) / 1e3 / reps)
        print(json.dumps({"n": n, "j": j, "pair": os.environ.get("NB_PAIR", "auto"), "us": t * 1e6}), flush=True)
