"""Per-CTA timeline of the per-launch simulate path (trace build), to see where a
step's time goes beyond the force math: launch ramp, tail, fixup, gaps.
  python tools/variants.py build   (with "trace": {"NB_TRACE": 1} in VARIANTS)
  python tools/trace_launches.py [CONFIG] [STEPS]   (on the GPU)
Records (thread 0 of every CTA, %globaltimer ns): kernel tag (1 step, 2 fixup),
CTA, SM, entry, after griddepcontrol.wait, end."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags

HERE = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.environ.get("NB_TRACE_LIB", os.path.join(HERE, "variants", "lib_trace.so")))
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = nb.BASELINE_CONFIGS[name]
s = cfg.system()
dt = cfg.precision.dtype
sfx = "_f32" if dt == np.float32 else "_f64"
st = DeviceState(s.position_matrix().astype(dt), np.stack(s.velocities, 1), s.masses, dt)
flags = kernel_flags(s.masses, cfg.softening_sq, dt)
L.nb_dev_workspace_bytes.restype = ctypes.c_int64
L.nb_dev_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int64]
wsb = L.nb_dev_workspace_bytes(dt.itemsize, cfg.n)
ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
fn = getattr(L, "nb_dev_simulate" + sfx)
fn.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
flag = ctypes.c_int(0)
cap = 1 << 20
buf = torch.zeros(8 * cap, dtype=torch.int64, device="cuda")
L.nb_trace_setup.argtypes = [ctypes.c_void_p, ctypes.c_int64]
L.nb_trace_count.restype = ctypes.c_int64


def sim():
    assert fn(st.pos_a.data_ptr(), st.pos_b.data_ptr(), st.vel.data_ptr(), st.acc.data_ptr(), cfg.n, 1.0, cfg.dt,
              cfg.softening_sq, steps, int(flags), ws.data_ptr(), wsb, None, ctypes.byref(flag)) == 0


sim()
torch.cuda.synchronize()
assert L.nb_trace_setup(buf.data_ptr(), cap) == 0
sim()
torch.cuda.synchronize()
n = L.nb_trace_count()
r = buf[: 8 * min(n, cap)].view(-1, 8).cpu().numpy()
if (r[:, 0] == 6).any():  # small-N kernel: per CTA per step (start, staged, computed, reduced+stored, synced)
    p = r[r[:, 0] == 6]
    step = p[:, 1] >> 32
    print(f"# {name}: small-N kernel, {len(p)} (CTA, step) records; per step, us (median over CTAs; "
          "compute = thread 0's source loop)\n")
    print("| step | stage | compute | reduce + epilogue | grid sync | step total |")
    print("|---|---|---|---|---|---|")
    for k in np.unique(step):
        q = p[step == k]
        t0, t1, t2, t3, t4 = (q[:, 3 + i].astype(np.float64) for i in range(5))
        tot = (np.median(t4 - t0)) / 1e3
        print(f"| {k} | {np.median(t1 - t0) / 1e3:.2f} | {np.median(t2 - t1) / 1e3:.2f} | "
              f"{np.median(t3 - t2) / 1e3:.2f} | {np.median(t4 - t3) / 1e3:.2f} | {tot:.2f} |")
    starts = [p[step == k][:, 3].min() for k in np.unique(step)]
    print(f"\nstep period (first CTA start to next): {np.median(np.diff(starts)) / 1e3:.2f} us")
    sys.exit(0)
if (r[:, 0] == 3).any():  # persistent simulate_kernel: per CTA per step (start, pass, sync1, fixup, sync2)
    p = r[r[:, 0] == 3]
    step = p[:, 1] >> 32
    base = p[:, 3].min()
    print(f"# {name}: persistent kernel, {len(p)} (CTA, step) records; per step, us (median over CTAs)\n")
    print("| step | pass | wait at sync 1 | fixup | wait at sync 2 | step total |")
    print("|---|---|---|---|---|---|")
    for k in np.unique(step):
        q = p[step == k]
        t0, t1, t2, t3, t4 = (q[:, 3 + i].astype(np.float64) for i in range(5))
        print(f"| {k} | {np.median(t1 - t0) / 1e3:.2f} | {np.median(t2 - t1) / 1e3:.2f} | {np.median(t3 - t2) / 1e3:.2f} | "
              f"{np.median(t4 - t3) / 1e3:.2f} | {np.median(t4 - t0) / 1e3:.2f} |")
    print(f"\nmax pass {np.max(p[:, 4] - p[:, 3]) / 1e3:.2f} us, max fixup {np.max(p[:, 6] - p[:, 5]) / 1e3:.2f} us")
    sys.exit(0)
seg = r[r[:, 0] == 4]
if len(seg):  # per stream-K segment: start, first tile staged, tiles done, epilogue done, #sources
    setup = (seg[:, 4] - seg[:, 3]) / 1e3
    loop = (seg[:, 5] - seg[:, 4]) / 1e3
    epi = (seg[:, 6] - seg[:, 5]) / 1e3
    nsrc = seg[:, 7]
    per_src = loop / np.maximum(nsrc, 1) * 1e3
    print(f"# segments: {len(seg)}; median setup (targets + first tile) {np.median(setup):.2f} us, "
          f"loop {np.median(loop):.2f} us for {np.median(nsrc):.0f} sources ({np.median(per_src):.2f} ns/source), "
          f"epilogue {np.median(epi):.2f} us; per CTA per launch: segments {len(seg) / max(1, len(np.unique(seg[:, 1] & 0xffffffff))):.2f}\n")
r = r[r[:, 0] != 4]
r = r[:, :6]
t0 = r[:, 3].min()
r[:, 3:] -= t0
# launches: consecutive groups in time order of (tag, wait time)
order = np.argsort(r[:, 4], kind="stable")
r = r[order]
groups, cur = [], [r[0]]
for row in r[1:]:
    if row[0] != cur[-1][0] or row[4] - cur[-1][4] > 2000:  # new kernel when the tag changes or waits are >2 us apart
        groups.append(np.array(cur)); cur = [row]
    else:
        cur.append(row)
groups.append(np.array(cur))
print(f"# {name}: {len(groups)} kernel launches traced (steps={steps}), times in us from the first CTA entry\n")
print("| # | kernel | CTAs | first entry | wait released (min..max) | first end | last end | median CTA busy |")
print("|---|---|---|---|---|---|---|---|")
prev_end = None
for k, g in enumerate(groups):
    kind = "step" if g[0, 0] == 1 else "fixup"
    busy = np.median(g[:, 5] - g[:, 4]) / 1e3
    print(f"| {k} | {kind} | {len(g)} | {g[:, 3].min() / 1e3:.1f} | {g[:, 4].min() / 1e3:.1f}..{g[:, 4].max() / 1e3:.1f} | "
          f"{g[:, 5].min() / 1e3:.1f} | {g[:, 5].max() / 1e3:.1f} | {busy:.1f} |")
steps_g = [g for g in groups if g[0, 0] == 1]
if len(steps_g) > 2:
    per = np.diff([g[:, 4].min() for g in steps_g]) / 1e3
    work = [np.median(g[:, 5] - g[:, 4]) / 1e3 for g in steps_g]
    tails = [(g[:, 5].max() - g[:, 5].min()) / 1e3 for g in steps_g]
    ramps = [(g[:, 4].max() - g[:, 4].min()) / 1e3 for g in steps_g]
    print(f"\nstep period {np.median(per):.2f} us; median CTA busy {np.median(work):.2f} us; "
          f"end spread (tail) {np.median(tails):.2f} us; wait-release spread {np.median(ramps):.2f} us")
