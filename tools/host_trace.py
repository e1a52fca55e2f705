"""Host-side phases of simulate()'s single native call at C1 (trace build):
python-side time around the call, and inside nb_host_simulate: arena, staging
memcpy, H2D + mapping, the cooperative launch, the stream sync, the copy out.  usage (GPU): NB_LIB_PATH=tools/variants/lib_trace.so python tools/host_trace.py [CONFIG] [REPS]"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = nb.BASELINE_CONFIGS[name]
s = cfg.system()
p = cfg.params()
L = _native.lib()
L.nb_host_trace.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
buf = (ctypes.c_double * 16)()
names = ["arena + checks", "staging memcpy", "H2D + map", "launch (dev_simulate)", "D2H enqueue", "stream sync", "memcpy out"]
acc = {k: [] for k in names}
tot, outer = [], []
sub = ([], [], [], [], [])
for r in range(reps + 20):
    t0 = time.perf_counter_ns()
    nb.simulate(s, p)
    t1 = time.perf_counter_ns()
    k = L.nb_host_trace(buf, 16)
    t = [buf[i] for i in range(k)]
    if r >= 20 and k >= 8:
        for i, nm in enumerate(names):
            acc[nm].append((t[i + 1] - t[i]) / 1e3)
        tot.append((t[7] - t[0]) / 1e3)
        if k >= 10:
            sub[0].append((t[8] - t[3]) / 1e3)
            sub[1].append((t[9] - t[8]) / 1e3)
        if k >= 14:
            sub[2].append((t[11] - t[10]) / 1e3)
            sub[3].append((t[12] - t[11]) / 1e3)
            sub[4].append((t[13] - t[12]) / 1e3)
        outer.append((t1 - t0) / 1e3)
print(f"# {name}: nb.simulate host phases, median of {reps} calls (us)")
for nm in names:
    print(f"{nm:28s} {np.median(acc[nm]):8.2f}")
print(f"{'native call total':28s} {np.median(tot):8.2f}")
print(f"{'  of launch: make_step_args':28s} {np.median(sub[0]):8.2f}")
print(f"{'  of launch: small launch':28s} {np.median(sub[1]):8.2f}")
print(f"{'    prep (caches, ppw)':28s} {np.median(sub[2]):8.2f}")
print(f"{'    args':28s} {np.median(sub[3]):8.2f}")
print(f"{'    cudaLaunchCooperativeKernel':28s} {np.median(sub[4]):8.2f}")
print(f"{'nb.simulate end to end':28s} {np.median(outer):8.2f}")
print(f"{'python outside the call':28s} {np.median(np.array(outer) - np.array(tot)):8.2f}")
