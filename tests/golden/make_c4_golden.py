"""Generate tests/golden/c4_final_sample.npz: the FP64 oracle's final state of
BASELINE config C4 (524288 bodies, FP64, 5 steps) on a fixed sample of rows.

The full oracle run is ~5 min on 16 host cores, more than the rest of the GPU
suite together, so the default GPU test compares the GPU trajectory with this
frozen sample (every sampled body's final position depends on all N bodies
through all 6 force evaluations); the live full-size comparison stays in
tests/test_gpu_large.py behind NB_FULL_ORACLE=1.

The numbers come from oracle/nbody_oracle.c (the restatement of the reference's
accel_soa / step_soa / _kick, bitwise equal to the reference's compiled kernel:
tests/test_oracle.py) -- reproducible anywhere with
    python tests/golden/make_c4_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

SAMPLE_ROWS = 2048
SAMPLE_SEED = 20260421


def sample_rows(n: int) -> np.ndarray:
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.unique(np.concatenate([[0, 1, n - 1], rng.integers(0, n, SAMPLE_ROWS)]))


def main():
    import paper_2203_08263_b200 as nb
    from oracle import oracle as O
    O.lib()
    cfg = nb.BASELINE_CONFIGS["C4"]
    s = cfg.system()
    p = cfg.params()
    pos, vel = O.simulate(s.position_matrix(), np.stack(s.velocities, 1).astype(np.float64),
                          s.masses.astype(np.float64), 1.0, p.dt, p.softening_sq, p.steps,
                          threads=O.host_threads())
    rows = sample_rows(cfg.n)
    np.savez_compressed(os.path.join(HERE, "c4_final_sample.npz"), rows=rows, pos=pos[rows], vel=vel[rows],
                        max_norm=np.array(float(np.max(np.linalg.norm(pos, axis=1)))),
                        checksum=np.array(O.checksum(pos)),
                        n=np.array(cfg.n), steps=np.array(p.steps), dt=np.array(p.dt), eps2=np.array(p.softening_sq))
    print("rows", rows.size, "max_norm", float(np.max(np.linalg.norm(pos, axis=1))), "checksum", repr(O.checksum(pos)))


if __name__ == "__main__":
    main()
