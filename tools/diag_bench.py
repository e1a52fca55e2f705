"""Measure the GPU diagnostics pass: nb_dev_energy on the
BASELINE states -- FP64 softened potential over all N^2 pairs + the fixed-order
energy/momentum reduction -- against its FP64-pipe roofline (13 DP lane-ops per
pair: 3 DADD, 3 DFMA for d2, 6 for the refined m/r, 1 DADD accumulate; ceiling
= 148 SM x 64 lanes x 1.965 GHz / 13).  CUDA events, best of 3 after a warm-up.
usage: python tools/diag_bench.py [CONFIG ...] > profiles/diagnostics_r01.md
NB_DIAG_LEGACY_LIB=<older libnbody_b200.so> times that library's nb_dev_energy
(its own workspace size; 8*n for the first version) on the same device states, for a before/after comparison."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200 import _native
from paper_2203_08263_b200.device import DeviceState

OPS = 13
CEIL = 148 * 64 * 1.965e9 / OPS
names = sys.argv[1:] or ["C2", "C3-f32", "C3-f64", "C4", "C5"]
legacy = os.environ.get("NB_DIAG_LEGACY_LIB")
if legacy:
    LL = ctypes.CDLL(legacy)
    for sfx in ("_f32", "_f64"):
        getattr(LL, "nb_dev_energy" + sfx).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                                      ctypes.c_int64, ctypes.c_void_p]


def energy(st, eps2):
    if not legacy:
        return st.energy(1.0, eps2)
    out = torch.zeros(6, dtype=torch.float64, device=st.device)
    if hasattr(LL, "nb_energy_workspace_bytes"):
        LL.nb_energy_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int64]
        LL.nb_energy_workspace_bytes.restype = ctypes.c_int64
        nbytes = LL.nb_energy_workspace_bytes(st.pbytes, st.n)
    else:
        nbytes = 8 * st.n
    ws = torch.empty(nbytes, dtype=torch.uint8, device=st.device)
    rc = getattr(LL, "nb_dev_energy" + st.sfx)(st.pos_cur.data_ptr(), st.vel.data_ptr(), st.n, 1.0, eps2,
                                               out.data_ptr(), ws.data_ptr(), ws.numel(),
                                               torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc
    v = out.cpu().numpy()
    return float(v[0]), float(v[1]), tuple(v[2:5])


print("# GPU diagnostics pass (energy + momentum), one B200\n")
print(f"`nb_dev_energy` on each BASELINE state (device generators), library `{os.path.basename(legacy or _native.LIB_PATH)}`; "
      f"pairs/s = N^2 / t; ceiling {CEIL:.3e} pairs/s = FP64 pipe at {OPS} DP ops per pair.\n")
print("| config | N | t (ms) | pairs/s | frac of FP64-pipe ceiling | PE |")
print("|---|---|---|---|---|---|")
for name in names:
    cfg = nb.BASELINE_CONFIGS[name]
    kind = "plummer_sphere" if cfg.generator is nb.plummer_sphere else "uniform_cube"
    st = DeviceState.from_generator(kind, cfg.n, 0, cfg.precision.dtype)
    energy(st, cfg.softening_sq)
    torch.cuda.synchronize()
    best, pe = 1e30, None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ke, pe, mom = energy(st, cfg.softening_sq)  # synchronizes (D2H of the 6 results)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    rate = float(cfg.n) ** 2 / (best / 1e3)
    print(f"| {name} | {cfg.n} | {best:.3f} | {rate:.3e} | {rate / CEIL:.3f} | {pe:.12e} |", flush=True)
