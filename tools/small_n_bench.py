"""Small-N simulate paths on one GPU: the small-N cooperative kernel (source split
inside the CTA), the stream-K persistent cooperative kernel and per-step
launches, timed on the same device state (nb_dev_simulate, CUDA events, best of
5 after a warm-up).  Sets the NB_SMALL_MAX_N / NB_PERSISTENT_MAX_N crossovers.
usage: python tools/small_n_bench.py [STEPS] > profiles/small_n_r01.md"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
NS = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [256, 512, 1024, 1536, 2048, 2368, 3072, 4096, 6144, 8192, 16384, 32768]
PATHS = {"small": ("1000000000", "0", ""), "small/8": ("1000000000", "0", "4"), "small/16": ("1000000000", "0", "8"),
         "persistent": ("0", "1000000000", ""), "per-launch": ("0", "0", "")}


def best_ms(st, eps2, flags, small, pers, ppw):
    os.environ["NB_SMALL_MAX_N"], os.environ["NB_PERSISTENT_MAX_N"] = small, pers
    if ppw:
        os.environ["NB_SMALL_PPW"] = ppw
    else:
        os.environ.pop("NB_SMALL_PPW", None)
    st.simulate(1.0, 1e-3, eps2, steps, flags)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.simulate(1.0, 1e-3, eps2, steps, flags)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


print(f"# Small-N simulate paths, one B200: {steps} steps ({steps + 1} force evaluations), uniform cube, eps2 = 1e-3\n")
print("µs per force evaluation (the whole simulate / (steps+1)); interactions/s of the fastest path.\n")
print("`small` = the small-N kernel with its default CTA size, `small/8`, `small/16` = forced 8 / 16 targets "
      "per CTA (NB_SMALL_PPW); a small-N column equal to per-launch means the kernel did not fit and fell back.\n")
print("| precision | N | small (µs) | small/8 | small/16 | persistent (µs) | per-launch (µs) | best | interactions/s (best) |")
print("|---|---|---|---|---|---|---|---|---|")
for prec in ("double", "single"):
    for n in NS:
        s = nb.uniform_cube(n, 0, nb.Precision(prec))
        dt_ = s.precision.dtype
        st = DeviceState(s.position_matrix().astype(dt_), np.stack(s.velocities, 1), s.masses, dt_)
        f = kernel_flags(s.masses, 1e-3, dt_)
        row = {}
        for name, (sm, pe, ppw) in PATHS.items():
            try:
                row[name] = best_ms(st, 1e-3, f, sm, pe, ppw) * 1e3 / (steps + 1)
            except Exception as e:  # the small kernel may not fit (cooperative grid / smem)
                row[name] = float("nan")
        best = min((v, k) for k, v in row.items() if v == v)
        rate = float(n) * n / (best[0] * 1e-6)
        print(f"| {prec} | {n} | {row['small']:.2f} | {row['small/8']:.2f} | {row['small/16']:.2f} | "
              f"{row['persistent']:.2f} | {row['per-launch']:.2f} | "
              f"{best[1]} | {rate:.3e} |", flush=True)
