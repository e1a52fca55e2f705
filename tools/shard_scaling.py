"""Per-rank compute of the i-sharded multi-GPU step, measured on ONE B200.

Each rank of a P-GPU run computes the forces of its N/P target rows against all
N sources, in two launches (its own rows as sources, then the other N - N/P as
one circular range, joined through the FP64 carry) -- exactly run_sharded's
sequence.  No rank waits on another's kernel, so one rank's launches can be
timed alone on one GPU.  Efficiency of the compute part of strong scaling:
E_compute(P) = (N^2 / t_1) / (P * (N^2/P) / t_P) = t_1 / (P * t_P).  The position
exchange adds (P-1)/P * N * bytes_per_body per step over NVLink (estimated at
the 770 GB/s measured peer bandwidth, B200_PROFILING.md) and overlaps the
local-source launch.
usage: python tools/shard_scaling.py [C4 C5] > profiles/shard_scaling_r01.md"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags
from paper_2203_08263_b200._native import NB_STEP_KICK_DRIFT

NVLINK_GBS = 770.0
names = sys.argv[1:] or ["C4", "C5"]
print("# Per-rank compute of the sharded step, timed on one B200\n")
print("One force evaluation + fused update of rank r's N/P targets against all N sources "
      "(local-source launch + remote-source launch with the FP64 carry), CUDA events, best of 3.\n")
print("| config | P | rank | targets | t_eval (ms) | rank rate (int/s) | E_compute(P) | exchange/step (MB) | exchange at 770 GB/s (ms) |")
print("|---|---|---|---|---|---|---|---|---|")
for name in names:
    cfg = nb.BASELINE_CONFIGS[name]
    dt = cfg.precision.dtype
    kind = "plummer_sphere" if cfg.generator is nb.plummer_sphere else "uniform_cube"
    full = DeviceState.from_generator(kind, cfg.n, 0, dt)
    masses = full.masses_host()
    flags = kernel_flags(masses, cfg.softening_sq, dt)
    pos_host = full.positions_host()
    vel_host = full.velocities_host()
    t1 = None
    for P in (1, 2, 4, 8):
        per = cfg.n // P
        for r in sorted({0, P - 1}):
            st = DeviceState(pos_host, vel_host, masses, dt, i_begin=r * per, n_i=per)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e30
            for _ in range(3):
                torch.cuda.synchronize()
                e0.record()
                if P == 1:
                    st.step(1.0, cfg.softening_sq, cfg.dt, NB_STEP_KICK_DRIFT, flags)
                else:
                    st.step(1.0, cfg.softening_sq, cfg.dt, NB_STEP_KICK_DRIFT, flags, j_begin=r * per,
                            j_count=per, carry_mode=1)
                    st.step(1.0, cfg.softening_sq, cfg.dt, NB_STEP_KICK_DRIFT, flags,
                            j_begin=(r * per + per) % cfg.n, j_count=cfg.n - per, carry_mode=2)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            if P == 1:
                t1 = best
            rate = float(per) * cfg.n / (best / 1e3)
            eff = t1 / (P * best)
            mb = (P - 1) / P * cfg.n * 4 * dt.itemsize / 1e6
            print(f"| {name} | {P} | {r} | {per} | {best:.2f} | {rate:.3e} | {eff:.3f} | {mb:.1f} | "
                  f"{mb / 1e3 / NVLINK_GBS * 1e3:.3f} |", flush=True)
            del st
    del full
    torch.cuda.empty_cache()
