"""Soak of the small-N kernel's tagged exchange: many launches per case, each
compared bit for bit (on the device) with the grid-barrier form's result
(NB_SMALL_TAGGED=0, computed once in a child process).
usage: python tools/soak_tagged.py [LAUNCHES_PER_CASE]"""
import json, os, subprocess, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

CASES = [("double", 256, 10), ("double", 1024, 10), ("double", 1184, 25), ("double", 2304, 12),
         ("single", 512, 16), ("single", 2000, 10), ("single", 3072, 9), ("single", 4096, 6)]


def final_state(prec, n, steps, reps=1, want=None):
    import torch
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    s = nb.uniform_cube(n, 1, nb.Precision(prec))
    dtype = s.precision.dtype
    pos, vel = s.position_matrix().astype(dtype), np.stack(s.velocities, 1)
    flags = kernel_flags(s.masses, 1e-2, dtype)
    st = DeviceState(pos, vel, s.masses, dtype)
    p0, v0 = None, None
    bad = 0
    for r in range(reps):
        st.load(pos, vel, s.masses)
        st.simulate(1.0, 1e-2, 1e-2, steps, flags)
        if want is not None:
            if p0 is None:
                p0 = torch.from_numpy(want[0]).to(st.pos_cur.device)
                v0 = torch.from_numpy(want[1]).to(st.pos_cur.device)
            if not (torch.equal(st.pos_cur, p0) and torch.equal(st.vel, v0)):
                bad += 1
    return st.pos_cur.cpu().numpy(), st.vel.cpu().numpy(), bad


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--ref":
        out = {}
        for prec, n, steps in CASES:
            p, v, _ = final_state(prec, n, steps)
            out[f"{prec}_{n}_p"], out[f"{prec}_{n}_v"] = p, v
        np.savez(sys.argv[2], **out)
        sys.exit(0)
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    with tempfile.TemporaryDirectory() as d:
        ref = os.path.join(d, "ref.npz")
        subprocess.run([sys.executable, os.path.abspath(__file__), "--ref", ref], check=True,
                       env=dict(os.environ, NB_SMALL_TAGGED="0"))
        want = dict(np.load(ref))
    total_bad = 0
    for prec, n, steps in CASES:
        _, _, bad = final_state(prec, n, steps, reps, (want[f"{prec}_{n}_p"], want[f"{prec}_{n}_v"]))
        total_bad += bad
        print(json.dumps({"precision": prec, "n": n, "steps": steps, "launches": reps, "mismatches": bad}), flush=True)
    sys.exit(1 if total_bad else 0)
