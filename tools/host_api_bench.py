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
