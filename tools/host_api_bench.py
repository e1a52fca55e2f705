"""Latency of the synchronous host entry points (the backend-plugin path:
nb_host_accel_soa per force evaluation) for a library, N = 1024 ... 16384.
usage: python tools/host_api_bench.py [LIB ...]"""
import ctypes, os, sys, time
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = sys.argv[1:] or [os.path.join(REPO, "paper_2203_08263_b200", "libnbody_b200.so")]
p, i64, d, i = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
for path in libs:
    L = ctypes.CDLL(path)
    f = L.nb_host_accel_soa_f64
    f.argtypes = [p] * 4 + [i64, d, d, i, i64, i] + [p] * 3
    for n in (1024, 4096, 16384):
        rng = np.random.default_rng(0)
        px, py, pz = (rng.uniform(-1, 1, n) for _ in range(3))
        m = rng.uniform(0.5, 1.5, n)
        ax, ay, az = (np.empty(n) for _ in range(3))
        args = [a.ctypes.data for a in (px, py, pz, m)] + [n, 1.0, 1e-3, 1, 0, 1] + [a.ctypes.data for a in (ax, ay, az)]
        assert f(*args) == 0
        reps = 50
        t0 = time.perf_counter()
        for _ in range(reps):
            f(*args)
        dt = (time.perf_counter() - t0) / reps
        print(f"{os.path.basename(path):28s} N={n:6d} {dt * 1e6:9.1f} us per nb_host_accel_soa_f64", flush=True)

# the whole simulate through the host entry point vs the Python API (C1: N=1024, FP64, 10 steps)
if os.environ.get("NB_HOST_SIM", "1") == "1":
    sys.path.insert(0, REPO)
    import paper_2203_08263_b200 as nb
    cfg = nb.BASELINE_CONFIGS["C1"]
    s, prm = cfg.system(), cfg.params()
    L = ctypes.CDLL(libs[-1])
    f = L.nb_host_simulate_soa_f64
    f.argtypes = [p] * 7 + [i64, d, d, d, i64]
    cols = [c.copy() for c in s.positions + s.velocities]
    m = s.masses.copy()

    def host_call():
        for k in range(6):
            cols[k][...] = (s.positions + s.velocities)[k]
        assert f(*[c.ctypes.data for c in cols], m.ctypes.data, s.count, 1.0, prm.dt, prm.softening_sq, prm.steps) == 0
    for name, fn in (("nb_host_simulate_soa_f64", host_call), ("paper_2203_08263_b200.simulate", lambda: nb.simulate(s, prm))):
        fn(); fn()
        t0 = time.perf_counter()
        for _ in range(50):
            fn()
        print(f"C1 simulate via {name:32s} {(time.perf_counter() - t0) / 50 * 1e6:9.1f} us", flush=True)
    print("checksums", nb.checksum(nb.simulate(s, prm)), np.sum((cols[0] + cols[1]) + cols[2]))
