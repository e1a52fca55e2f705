#!/bin/bash
# FP64 cluster split-source kernel (pair_kernel_f64, K = 2 / 4) forced on (NB_PAIR=1) vs off:
# per-launch force pass at mid-size N, plus parity of the forced kernel against the oracle.
cd "$(dirname "$0")/.."
O=gpurun_out/pair_f64; mkdir -p $O
NS="2561 3072 3500 4096 4400 4736 6144 7104 7600 8192 9000 9472"
NB_PROBE_PREC=double NB_PAIR=0 timeout 300 python tools/pair_probe.py $NS > $O/off.log 2>&1
NB_PROBE_PREC=double NB_PAIR=1 timeout 300 python tools/pair_probe.py $NS > $O/on.log 2>&1
NB_PAIR=1 timeout 300 python - > $O/parity.log 2>&1 <<'P'
import numpy as np, paper_2203_08263_b200 as nb
from paper_2203_08263_b200.device import DeviceState, kernel_flags
from paper_2203_08263_b200 import _native
from oracle import oracle as O
O.lib()
for n, eps2, gen in [(1, 1e-3, nb.uniform_cube), (33, 1e-3, nb.uniform_cube), (4096, 1e-3, nb.uniform_cube), (4736, 0.0, nb.uniform_cube),
                     (3000, 1e-4, nb.plummer_sphere), (8192, 1e-2, nb.uniform_cube), (9472, 1e-3, nb.uniform_cube), (7001, 0.0, nb.uniform_cube)]:
    s = gen(n, 3, nb.Precision.DOUBLE)
    pos = s.position_matrix()
    st = DeviceState(pos, np.stack(s.velocities, 1), s.masses, np.float64)
    f = kernel_flags(s.masses, eps2, np.float64)
    a = st.accelerations(1.0, eps2, f)[:, :3].cpu().numpy()
    a2 = st.accelerations(1.0, eps2, f)[:, :3].cpu().numpy()
    rows = np.unique(np.concatenate([[0, n - 1], np.random.default_rng(1).integers(0, n, 64)]))
    want = O.accel_rows_ld(*(np.ascontiguousarray(pos[:, k]) for k in range(3)), s.masses, rows, 1.0, eps2)
    dev = O.accel_dev(a[rows], want) if n > 1 else float(np.abs(a).max())
    print(n, eps2, gen.__name__, _native.step_kernel_name(8, n, n), "accel_dev", dev, "repro", bool(np.array_equal(a, a2)), flush=True)
    assert dev <= 1e-12 and np.array_equal(a, a2)
# trajectory through the per-step path
s = nb.uniform_cube(4096, 5, nb.Precision.DOUBLE)
fin = nb.simulate(s, nb.SimParams(1.0, 1e-3, 1e-3, 4)).position_matrix()
ref, _ = O.simulate(s.position_matrix(), np.stack(s.velocities, 1), s.masses, 1.0, 1e-3, 1e-3, 4, threads=O.host_threads())
print("traj 4096 position_dev", O.position_dev(fin, ref))
assert O.position_dev(fin, ref) <= 1e-12
print("parity ok")
P
echo "parity rc=$?" >> $O/parity.log
cat $O/parity.log | tail -n 14
paste <(grep '"n"' $O/off.log) <(grep '"n"' $O/on.log) | python -c "
import sys, json
for l in sys.stdin:
    a, b = l.strip().split('\t')
    a, b = json.loads(a), json.loads(b)
    print(a['n'], 'off', round(a['us'], 1), 'on', round(b['us'], 1), 'ratio', round(a['us'] / b['us'], 3))"
