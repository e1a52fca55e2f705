"""Worker of tests/test_gpu_multigpu.py, launched one process per GPU by
torch.distributed.run: runs the multi-GPU simulate (sharded.simulate_sharded,
NCCL process group) on a named case with one transport and has rank 0 write
the final positions and velocities to --out (npz)."""
import argparse
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

CASES = {
    # C4-shaped: FP64 uniform cube, eps2 1e-3, dt 1e-3, 5 steps (N reduced to 65536)
    "c4s": dict(n=65536, kind="cube", prec="double", eps2=1e-3, dt=1e-3, steps=5),
    # C5-shaped: FP32 Plummer, equal masses 1/N, eps2 1e-4, dt 1e-4, 3 steps (N reduced to 262144)
    "c5s": dict(n=262144, kind="plummer", prec="single", eps2=1e-4, dt=1e-4, steps=3),
    # ragged: N not divisible by the world size (massless padding), FP32, eps2 = 0 (self mask)
    "ragged": dict(n=30001, kind="cube", prec="single", eps2=0.0, dt=1e-4, steps=2),
}


def case_system(name):
    import paper_2203_08263_b200 as nb
    c = CASES[name]
    gen = nb.uniform_cube if c["kind"] == "cube" else nb.plummer_sphere
    return gen(c["n"], 0, nb.Precision(c["prec"])), c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True, choices=sorted(CASES))
    ap.add_argument("--transport", required=True, choices=["nccl", "capi", "p2p", "api"])
    ap.add_argument("--out", required=True)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: ranks share GPU 0 and exchange through host memory (driver-logic check on a "
                         "1-GPU box; no rank's kernel waits on another's)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    local = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200.sharded import simulate_sharded
    s, c = case_system(args.case)
    dtype = s.precision.dtype
    if args.transport == "api":
        # the public entry point: simulate() shards itself over the process group
        fin = nb.simulate(s, nb.SimParams(1.0, c["dt"], c["eps2"], c["steps"]))
        pos, vel = fin.position_matrix(), np.stack(fin.velocities, 1)
    else:
        pos, vel = simulate_sharded(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses,
                                    dtype, 1.0, c["dt"], c["eps2"], c["steps"], transport=args.transport)
    # every rank holds the full result: check they agree bit for bit
    where = "cuda" if args.backend == "nccl" else "cpu"
    got = torch.tensor(np.ascontiguousarray(pos, np.float64), device=where)
    ref = got.clone()
    dist.broadcast(ref, 0)
    same = torch.tensor([int(torch.equal(got, ref))], device=where)
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    if dist.get_rank() == 0:
        np.savez(args.out, pos=np.asarray(pos, np.float64), vel=np.asarray(vel, np.float64),
                 ranks_agree=int(same.item()), world=dist.get_world_size())
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
