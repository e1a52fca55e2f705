"""cProfile of the Python side of nb.simulate at a BASELINE config (GPU box):
where the host time outside the native call goes.
usage: python tools/py_profile.py [CONFIG] [CALLS]"""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08263_b200 as nb

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
cfg = nb.BASELINE_CONFIGS[name]
s = cfg.system()
p = cfg.params()
for _ in range(50):
    nb.simulate(s, p)
t0 = time.perf_counter()
for _ in range(calls):
    nb.simulate(s, p)
print(f"plain: {(time.perf_counter() - t0) / calls * 1e6:.1f} us per nb.simulate")
pr = cProfile.Profile()
pr.enable()
for _ in range(calls):
    nb.simulate(s, p)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
