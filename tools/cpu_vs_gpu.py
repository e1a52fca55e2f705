"""the reference's CPU path timed on the GPU box's own host cores
beside the GPU, for every BASELINE config.  The CPU side is the reference's own
compiled kernel (oracle/_ref, soa-recip -- its fastest rung -- on all host
threads): a full simulate where it finishes in seconds (C1, C2), one force
evaluation of the config's state otherwise (C3-f32, C3-f64, C4), and for C5 the
rate of a C5-distribution evaluation at N=524288, extrapolated (labelled).
The GPU side is paper_2203_08263_b200.simulate() end to end (host arrays in/out).
usage: python tools/cpu_vs_gpu.py > profiles/cpu_vs_gpu_r01.md"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_08263_b200 as nb
from oracle import oracle as O

R = O.ref_module()
T = O.host_threads()
rows = []
for name in ["C1", "C2", "C3-f32", "C3-f64", "C4", "C5"]:
    cfg = nb.BASELINE_CONFIGS[name]
    dtype = cfg.precision.dtype
    if name == "C5":  # a C5-distribution state at N=524288 for the CPU rate
        s_cpu = nb.plummer_sphere(524288, 0, cfg.precision)
    else:
        s_cpu = cfg.system()
    n_cpu = s_cpu.count
    cols = [np.ascontiguousarray(c) for c in s_cpu.positions]
    m = np.ascontiguousarray(s_cpu.masses)
    if name in ("C1", "C2"):
        t0 = time.perf_counter()
        O.ref_simulate(s_cpu.position_matrix().astype(dtype), np.stack(s_cpu.velocities, 1), m, 1.0, cfg.dt,
                       cfg.softening_sq, cfg.steps, recip=True, threads=T)
        t = time.perf_counter() - t0
        cpu_rate = float(n_cpu) ** 2 * (cfg.steps + 1) / t
        how = f"full simulate ({cfg.steps} steps), {t:.2f} s"
    else:
        out = [np.empty(n_cpu, dtype) for _ in range(3)]
        t0 = time.perf_counter()
        R.accel_soa(cols[0], cols[1], cols[2], m, 1.0, cfg.softening_sq, True, 0, T, *out)
        t = time.perf_counter() - t0
        cpu_rate = float(n_cpu) ** 2 / t
        how = f"one force evaluation at N={n_cpu}, {t:.1f} s" + (" (extrapolated to N=4M)" if name == "C5" else "")
    # GPU, end to end through the public API (host arrays), best of 2 after a warm-up
    s = cfg.system()
    p = cfg.params()
    reps = 1 if name == "C5" else 2
    nb.simulate(s, p) if name != "C5" else None
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        nb.simulate(s, p)
        best = min(best, time.perf_counter() - t0)
    gpu_rate = float(cfg.n) ** 2 * (cfg.steps + 1) / best
    rows.append((name, cfg.n, dtype.name, cpu_rate, how, gpu_rate, gpu_rate / cpu_rate))
    print(json.dumps(rows[-1][:4] + rows[-1][5:]), file=sys.stderr, flush=True)

print("# Reference CPU path vs B200, every BASELINE config (same box)\n")
print(f"CPU: the reference's compiled kernel (oracle/_ref, soa-recip) on {T} host threads "
      f"({os.cpu_count()} logical CPUs). GPU: `simulate()` end to end from host arrays, 1 B200.\n")
print("| config | N | dtype | CPU interactions/s | CPU sample | GPU e2e interactions/s | GPU / CPU |")
print("|---|---|---|---|---|---|---|")
for name, n, dt, c, how, g, r in rows:
    print(f"| {name} | {n} | {dt} | {c:.3e} | {how} | {g:.3e} | {r:.0f}x |")
