"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel variant (f32/f64, exclude-self, uniform mass), split i-blocks
(stream-K fixup), the two-phase carry, the peer-store epilogue, updates, init,
energy.  usage: compute-sanitizer --tool <tool> python tools/sanitize_case.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags
from paper_2203_08263_b200._native import NB_STEP_FIRST, NB_STEP_KICK_DRIFT, NB_STEP_FINAL_KICK

for prec in (nb.Precision.SINGLE, nb.Precision.DOUBLE):
    for n, eps2 in ((3001, 1e-3), (700, 0.0)):
        s = nb.uniform_cube(n, 3, prec)
        nb.simulate(s, nb.SimParams(1.0, 1e-3, eps2, 2))
        nb.compute_accelerations(s, nb.SimParams(1.0, 1e-3, eps2, 1))
    pl = nb.plummer_sphere(2048, 1, prec)
    nb.simulate(pl, nb.SimParams(1.0, 1e-4, 1e-4, 2))
    nb.diagnostics_gpu(pl, nb.SimParams(1.0, 1e-4, 1e-4, 1))
    dt_ = prec.dtype
    g = DeviceState.from_generator("uniform_cube", 1000, 2, dt_)
    g.simulate(1.0, 1e-3, 1e-3, 2, 0)
    # two emulated ranks: carry split + peer-store epilogue
    s = nb.uniform_cube(1200, 4, prec)
    pos, vel, m = s.position_matrix().astype(dt_), np.stack(s.velocities, 1), s.masses
    ranks = [DeviceState(pos, vel, m, dt_, i_begin=r * 600, n_i=600) for r in range(2)]
    f = kernel_flags(m, 1e-3, dt_)
    for step, mode in enumerate((NB_STEP_FIRST, NB_STEP_KICK_DRIFT, NB_STEP_FINAL_KICK)):
        for st in ranks:
            st.step(1.0, 1e-3, 1e-3, mode, f, j_begin=st.i_begin, j_count=600, carry_mode=1)
        for st in ranks:
            peers = None if mode == NB_STEP_FINAL_KICK else [q.pos_next.data_ptr() for q in ranks if q is not st]
            st.step(1.0, 1e-3, 1e-3, mode, f, j_begin=(st.i_begin + 600) % 1200, j_count=600, carry_mode=2,
                    peers=peers)
        if mode != NB_STEP_FINAL_KICK:
            for st in ranks:
                st.swap()
    from paper_2203_08263_b200 import backend
    px, py, pz = (c.copy() for c in s.positions)
    ax, ay, az = (np.zeros(1200, dt_) for _ in range(3))
    backend.accel_soa(px, py, pz, s.masses, 1.0, 1e-3, True, 0, 1, ax, ay, az)
    vx, vy, vz = (c.copy() for c in s.velocities)
    backend.step_soa(px, py, pz, vx, vy, vz, ax, ay, az, 1e-3, 1)
torch.cuda.synchronize()
print("sanitize case ok")
