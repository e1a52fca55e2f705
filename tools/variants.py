"""Build and time kernel tuning variants (-D overrides of nbody_force.cu knobs).

  python tools/variants.py build            # here: compile every variant .so
  python tools/variants.py run [CONFIG...]  # on the GPU: time each variant

Each variant is a full copy of libnbody_b200.so under tools/variants/."""
import ctypes, json, os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
OUT = os.path.join(HERE, "variants")

VARIANTS = {
    "base": {},
    "trace": {"NB_TRACE": 1},  # per-CTA timelines for tools/trace_launches.py
    "old": None,  # a prebuilt library copied to tools/variants/lib_old.so (A/B against an earlier commit)
    # e^2 term of the FP64 rsqrt corrections on the FP32/INT pipes (sq_term_f32)
    "f64_mixed": {"NB_F64_MIXED": 1, "NB_DIAG_MIXED": 1},
    # 12 / 16 warps per SM (3 / 4 per scheduler) with fewer targets per thread, same 1536-body
    # i-block for T=384 x K=4; FP64 sums in registers to fit the 48 KB static shared memory
    "t384_k4": {"NB_F32_T": 384, "NB_F32_K": 4, "NB_F32_TJ": 384, "NB_F32_SUMS_IN_REGS": 1,
                "NB_F32_EXP2_MASK": 33, "NB_F32_EXP2_PHASES": 4},
    "t384_k4_q": {"NB_F32_T": 384, "NB_F32_K": 4, "NB_F32_TJ": 384, "NB_F32_SUMS_IN_REGS": 1,
                  "NB_F32_EXP2_MASK": 1, "NB_F32_EXP2_PHASES": 2},
    # 8 targets per thread (more independent chains per warp) in 128-thread CTAs, 2 per SM
    "t128_k8_b2": {"NB_F32_T": 128, "NB_F32_K": 8, "NB_F32_MINB": 2, "NB_F32_EXP2_MASK": 37},
    "t128_k8_b2_q": {"NB_F32_T": 128, "NB_F32_K": 8, "NB_F32_MINB": 2, "NB_F32_EXP2_MASK": 33},
    "t128_k8_b1": {"NB_F32_T": 128, "NB_F32_K": 8, "NB_F32_MINB": 1, "NB_F32_EXP2_MASK": 37},
    # FP64 geometry: more / fewer targets per thread
    "f64_k8_t128": {"NB_F64_K": 8, "NB_F64_T": 128, "NB_F64_MINB": 2},
    "t512_k2": {"NB_F32_T": 512, "NB_F32_K": 2, "NB_F32_TJ": 512, "NB_F32_SUMS_IN_REGS": 1,
                "NB_F32_EXP2_MASK": 1, "NB_F32_EXP2_PHASES": 4},
    "t512_k2_p3": {"NB_F32_T": 512, "NB_F32_K": 2, "NB_F32_TJ": 512, "NB_F32_SUMS_IN_REGS": 1,
                   "NB_F32_EXP2_MASK": 1, "NB_F32_EXP2_PHASES": 3, "NB_F32_UNROLL": 12},
    "t512_k2_u8": {"NB_F32_T": 512, "NB_F32_K": 2, "NB_F32_TJ": 512, "NB_F32_SUMS_IN_REGS": 1,
                   "NB_F32_EXP2_MASK": 1, "NB_F32_EXP2_PHASES": 4, "NB_F32_UNROLL": 8},
    "t512_k2_smem": {"NB_F32_T": 512, "NB_F32_K": 2, "NB_F32_TJ": 512,
                     "NB_F32_EXP2_MASK": 1, "NB_F32_EXP2_PHASES": 4},
    # i-block geometry vs N: K=4 (IB=1024: C2 = 16 whole blocks)
    # with 1/3 of the weights on LG2/EX2 over 3 source phases (K=8 exceeds 48 KB static smem;
    # 3 phases do not divide the x16 unroll: the phase test becomes a runtime branch),
    # and with 3/8 or 1/4 over 4 phases
    "k4_p3": {"NB_F32_K": 4, "NB_F32_EXP2_MASK": 9, "NB_F32_EXP2_PHASES": 3},
    "k4_p4_3of8": {"NB_F32_K": 4, "NB_F32_EXP2_MASK": 25, "NB_F32_EXP2_PHASES": 4},
    "k4_p4_2of8": {"NB_F32_K": 4, "NB_F32_EXP2_MASK": 33, "NB_F32_EXP2_PHASES": 4},
    # round 2: split-i-block fixup in the step kernel (INFIX) and the partial last
    # i-block's dead-group skipping with the cost-balanced schedule (PG), each on/off
    "pg0_fixk": {"NB_PARTIAL_GROUPS": 0, "NB_INFIX_DEFAULT": 0},
    "pg0_infix": {"NB_PARTIAL_GROUPS": 0, "NB_INFIX_DEFAULT": 1},
    "pg1_fixk": {"NB_PARTIAL_GROUPS": 1, "NB_INFIX_DEFAULT": 0},
    "pg1_infix": {"NB_PARTIAL_GROUPS": 1, "NB_INFIX_DEFAULT": 1},
    # round 2: the cluster split-source kernel with 6 targets per thread (no odd target)
    "pair_k6": {"NB_PAIR_K": 6},
    "pair_k5": {"NB_PAIR_K": 5},
    "pair_k4": {"NB_PAIR_K": 4},
    "pair_k3": {"NB_PAIR_K": 3},
    "pair_k2": {"NB_PAIR_K": 2},
    "pair_u8": {"NB_PAIR_UNROLL": 8},
    "pair_u12": {"NB_PAIR_UNROLL": 12},
    "pair_u32": {"NB_PAIR_UNROLL": 32},
    "pair_oddfirst": {"NB_PAIR_ODD_FIRST": 1},
    "pair_shfl0": {"NB_PAIR_SHFL": 0},
    "pair_shfl1": {"NB_PAIR_SHFL": 1},
    "pair_oddexp2_2": {"NB_PAIR_ODD_EXP2": 2},
    "pair_oddexp2_4": {"NB_PAIR_ODD_EXP2": 4},
    "pair_oddexp2_8": {"NB_PAIR_ODD_EXP2": 8},
    "pair_oddexp2_16": {"NB_PAIR_ODD_EXP2": 16},
    "pair_stagewise": {"NB_F32_STAGEWISE": 1},
    "pair_tj128": {"NB_PAIR_TJ": 128},
    # small-N cooperative kernel with 12 / 16 warps per CTA (more latency hiding per SM)
    "small_t384": {"NB_SMALL_T": 384},
    "small_t512": {"NB_SMALL_T": 512},
    # round 2: accumulating FFMA2s of a group of G sources behind a loop boundary
    # (triples adjacent: w from the operand reuse cache), NB_F32_SPLIT_ACC = G
    "split2": {"NB_F32_SPLIT_ACC": 2, "NB_F32_SPLIT_KIND": 2},
    "split4": {"NB_F32_SPLIT_ACC": 4, "NB_F32_SPLIT_KIND": 2},
    "split8": {"NB_F32_SPLIT_ACC": 8, "NB_F32_SPLIT_KIND": 2},
    "split4_u8": {"NB_F32_SPLIT_ACC": 4, "NB_F32_SPLIT_KIND": 2, "NB_F32_UNROLL": 8},
    "split4_u4": {"NB_F32_SPLIT_ACC": 4, "NB_F32_SPLIT_KIND": 2, "NB_F32_UNROLL": 4},
    "f64_split1": {"NB_F64_SPLIT_ACC": 1},
    "f64_split2": {"NB_F64_SPLIT_ACC": 2},
    "f64_split4": {"NB_F64_SPLIT_ACC": 4},
    # extra nvcc flags per variant: {"_flags": ["-Xptxas", "..."]}
}

# GPU optimisation ladder: the reference's ladder axes --
# math form (pow / recip), blocking, SIMD-friendly layout, precision -- mapped
# onto GPU knobs, each rung adding one change to the previous one (FP32, C3).
LADDER = [
    ("L0 pow form, scalar FP32, K=2, no unroll, per-pair order",
     {"NB_F32_MATH": 2, "NB_F32_PACKED": 0, "NB_F32_K": 2, "NB_F32_UNROLL": 1, "NB_F32_STAGEWISE": 0,
      "NB_F32_EXP2_MASK": 0}),
    ("L1 + recip form (reference's fastest CPU rung)",
     {"NB_F32_MATH": 1, "NB_F32_PACKED": 0, "NB_F32_K": 2, "NB_F32_UNROLL": 1, "NB_F32_STAGEWISE": 0,
      "NB_F32_EXP2_MASK": 0}),
    ("L2 + MUFU rsqrt form",
     {"NB_F32_MATH": 0, "NB_F32_PACKED": 0, "NB_F32_K": 2, "NB_F32_UNROLL": 1, "NB_F32_STAGEWISE": 0,
      "NB_F32_EXP2_MASK": 0}),
    ("L3 + unrolled source loop (x16)",
     {"NB_F32_PACKED": 0, "NB_F32_K": 2, "NB_F32_STAGEWISE": 0, "NB_F32_EXP2_MASK": 0}),
    ("L4 + register blocking, 6 targets/thread",
     {"NB_F32_PACKED": 0, "NB_F32_STAGEWISE": 0, "NB_F32_EXP2_MASK": 0}),
    ("L5 + packed FFMA2/FADD2/FMUL2", {"NB_F32_EXP2_MASK": 0}),
    ("L6 + 1/3 of the weights via MUFU.LG2/EX2 (shipped)", {}),
    ("L6' (alternative) stage-wise source order across the pairs", {"NB_F32_STAGEWISE": 1}),
]
if os.environ.get("NB_LADDER"):  # NB_LADDER=1 python tools/variants.py build|run C3-f32
    VARIANTS.update({f"ladder{i}": d for i, (_, d) in enumerate(LADDER)})


def build_one(name, defs):
    from paper_2203_08263_b200 import _build as B
    objdir = os.path.join(OUT, name)
    os.makedirs(objdir, exist_ok=True)
    defs = dict(defs)
    extra = defs.pop("_flags", [])  # extra nvcc flags for this variant
    dflags = [f"-D{k}={v}" for k, v in defs.items()] + list(extra) + [f'-DNB_SRC_DIGEST="{B.source_digest()}"']
    objs = []
    for src in B.SOURCES:
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *dflags, "-Xptxas", "-v", "-c", os.path.join(B.CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            return name, "FAILED " + r.stderr[-2000:]
        if src == "nbody_force.cu":
            log = r.stderr
        objs.append(o)
    lib = os.path.join(OUT, f"lib_{name}.so")
    r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs], capture_output=True, text=True)
    if r.returncode:
        return name, "LINK FAILED " + r.stderr
    regs = []
    lines = log.splitlines()
    for i, ln in enumerate(lines):
        if "Function properties for" in ln and "step_kernel" in ln:
            tag = "f32" if "CoreF32" in ln else "f64"
            mask = "M" if "ILb1E" in ln else "-"
            spill = lines[i + 1].strip()
            used = lines[i + 2].split("Used")[1].split(",")[0].strip() if i + 2 < len(lines) and "Used" in lines[i + 2] else "?"
            regs.append(f"{tag}{mask}:{used}|{spill.split(',')[1].strip()}")
    return name, " ".join(regs)


def build(only=None):
    todo = [kv for kv in VARIANTS.items() if kv[1] is not None and (not only or kv[0] in only)]
    with ThreadPoolExecutor(8) as ex:
        for name, info in ex.map(lambda kv: build_one(*kv), todo):
            print(f"{name:16s} {info}")


def ladder_libs(rungs=None) -> dict:
    """{rung index: path} of the ladder-rung libraries, building missing ones
    (one nvcc run per rung, in parallel)."""
    rungs = range(len(LADDER)) if rungs is None else rungs
    missing = {f"ladder{i}": LADDER[i][1] for i in rungs if not os.path.exists(os.path.join(OUT, f"lib_ladder{i}.so"))}
    if missing:
        with ThreadPoolExecutor(8) as ex:
            for name, info in ex.map(lambda kv: build_one(*kv), missing.items()):
                if "FAILED" in info:
                    raise RuntimeError(f"{name}: {info}")
    return {i: os.path.join(OUT, f"lib_ladder{i}.so") for i in rungs}


def variant_accel(path, st, n, eps2, mask, dtype):
    """Accelerations of the state through one variant library's nb_dev_step (mode ACCEL)."""
    import numpy as np
    import torch
    sfx = "_f32" if dtype == np.float32 else "_f64"
    L = ctypes.CDLL(path)
    wsb = L.nb_dev_workspace_bytes
    wsb.restype = ctypes.c_int64
    wsb.argtypes = [ctypes.c_int, ctypes.c_int64]
    nbytes = wsb(np.dtype(dtype).itemsize, n)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    step = getattr(L, "nb_dev_step" + sfx)
    step.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                     ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                     ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    acc = torch.zeros((n, 4), dtype=st.acc.dtype, device="cuda")
    rc = step(st.pos_a.data_ptr(), n, 0, n, 0, n, 1.0, eps2, 0.0, 0, int(mask), None, 0, acc.data_ptr(), None,
              None, ws.data_ptr(), nbytes, 0)
    torch.cuda.synchronize()
    assert rc == 0, rc
    return acc[:, :3].cpu().numpy().astype(np.float64)


def variant_simulate(path, sys0, g, dt, eps2, steps, mask, dtype):
    """Final positions (N, 3) of one variant library's nb_dev_simulate."""
    import numpy as np
    import torch
    from paper_2203_08263_b200.device import DeviceState
    sfx = "_f32" if dtype == np.float32 else "_f64"
    L = ctypes.CDLL(path)
    fn = getattr(L, "nb_dev_simulate" + sfx)
    fn.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
    wsb = L.nb_dev_workspace_bytes
    wsb.restype = ctypes.c_int64
    wsb.argtypes = [ctypes.c_int, ctypes.c_int64]
    n = sys0.count
    nbytes = wsb(np.dtype(dtype).itemsize, n)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    st = DeviceState(sys0.position_matrix().astype(dtype), np.stack(sys0.velocities, 1), sys0.masses, dtype)
    flag = ctypes.c_int(0)
    rc = fn(st.pos_a.data_ptr(), st.pos_b.data_ptr(), st.vel.data_ptr(), st.acc.data_ptr(), n, g, dt, eps2, steps,
            int(mask), ws.data_ptr(), nbytes, 0, ctypes.byref(flag))
    torch.cuda.synchronize()
    assert rc == 0, rc
    return (st.pos_b if flag.value else st.pos_a)[:, :3].cpu().numpy().astype(np.float64)


def run(configs):
    import numpy as np
    import torch
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    from paper_2203_08263_b200 import _native
    results = {}
    for cfgname in configs:
        cfg = nb.BASELINE_CONFIGS[cfgname]
        s = cfg.system()
        dt = cfg.precision.dtype
        sfx = "_f32" if dt == np.float32 else "_f64"
        if sfx == "_f64" and cfgname != "C3-f64":
            pass
        ref_state = DeviceState(s.position_matrix().astype(dt), np.stack(s.velocities, 1), s.masses, dt)
        mask = kernel_flags(s.masses, cfg.softening_sq, dt)
        ref_acc = ref_state.accelerations(1.0, cfg.softening_sq, mask).cpu().numpy().astype(np.float64)
        # the oracle (long-double rows on the same rounded inputs) for every variant's accuracy
        from oracle import oracle as O
        rows = np.unique(np.concatenate([[0, cfg.n - 1], np.random.default_rng(3).integers(0, cfg.n, 126)]))
        pos = s.position_matrix()
        want = O.accel_rows_ld(*(np.ascontiguousarray(pos[:, k].astype(dt)) for k in range(3)),
                               s.masses, rows, 1.0, cfg.softening_sq)
        only = [v for v in os.environ.get("NB_VARIANTS", "").split(",") if v]
        for name in VARIANTS:
            if only and name not in only:
                continue
            path = os.path.join(OUT, f"lib_{name}.so")
            if not os.path.exists(path):
                continue
            if sfx == "_f32" and name.startswith("f64"):
                continue
            if sfx == "_f64" and not (name.startswith("f64") or name == "base"):
                continue
            L = ctypes.CDLL(path)
            fn = getattr(L, "nb_dev_simulate" + sfx)
            fn.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                                   ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                                   ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
            wsb = L.nb_dev_workspace_bytes
            wsb.restype = ctypes.c_int64
            wsb.argtypes = [ctypes.c_int, ctypes.c_int64]
            nbytes = wsb(dt.itemsize, cfg.n)
            st = DeviceState(s.position_matrix().astype(dt), np.stack(s.velocities, 1), s.masses, dt)
            ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
            flag = ctypes.c_int(0)
            step = getattr(L, "nb_dev_step" + sfx)
            step.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                             ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
            acc = torch.zeros((cfg.n, 4), dtype=st.acc.dtype, device="cuda")
            rc = step(st.pos_a.data_ptr(), cfg.n, 0, cfg.n, 0, cfg.n, 1.0, cfg.softening_sq, 0.0, 0, int(mask),
                      None, 0, acc.data_ptr(), None, None, ws.data_ptr(), nbytes, 0)
            torch.cuda.synchronize()
            a = acc[:, :3].cpu().numpy().astype(np.float64)
            dev = float(np.max(np.abs(a - ref_acc[:, :3]) / np.maximum(np.linalg.norm(ref_acc[:, :3], axis=1), 1e-300)[:, None]))
            odev = O.accel_dev(a[rows], want)

            def sim():
                r = fn(st.pos_a.data_ptr(), st.pos_b.data_ptr(), st.vel.data_ptr(), st.acc.data_ptr(), cfg.n, 1.0,
                       cfg.dt, cfg.softening_sq, cfg.steps, int(mask), ws.data_ptr(), nbytes, 0, ctypes.byref(flag))
                assert r == 0, r
            sim(); sim()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(3):
                e0.record(); sim(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 1e3)
            t = min(ts)
            rate = cfg.interactions / t
            peak = 148 * (128 if dt == np.float32 else 64) * 2 * 1.965e9
            results[f"{cfgname}/{name}"] = {"rate": rate, "frac": 20 * rate / peak, "rc": rc, "dev_vs_base": dev,
                                            "accel_dev_vs_oracle": odev, "oracle_rows": int(rows.size)}
            print(f"{cfgname:8s} {name:16s} rate={rate:.4e} frac={20 * rate / peak:.4f} dev={dev:.2e} "
                  f"oracle_dev={odev:.2e}", flush=True)
    with open(os.path.join(REPO, "gpurun_out", "variants.json"), "w") as f:
        json.dump(results, f, indent=1)


def ladder_report(path):
    res = json.load(open(os.path.join(REPO, "gpurun_out", "variants.json")))
    lines = ["# GPU optimisation ladder (FP32, C3: N=131072, 10 steps, 1 B200)", "",
             "Each rung adds one change to the previous rung; rates from `tools/variants.py run`",
             "(`nb_dev_simulate`, best of 3). Fraction = 20 flop/interaction / nominal FP32 peak.", "",
             "Accuracy: `_accel_dev` (validation.py:212-225) of the rung's accelerations of the C3 initial",
             "state against the long-double oracle on 128 sampled rows (bound 1e-5, SURVEY.md 8(c)).", "",
             "| rung | interactions/s | frac of nominal FP32 | speed-up vs L0 | vs previous | accel_dev vs oracle |",
             "|---|---|---|---|---|---|"]
    base = prev = None
    for i, (name, _) in enumerate(LADDER):
        r = res.get(f"C3-f32/ladder{i}")
        if r is None:
            continue
        base = base or r["rate"]
        od = r.get("accel_dev_vs_oracle")
        lines.append(f"| {name} | {r['rate']:.3e} | {r['frac']:.3f} | {r['rate'] / base:.2f}x | "
                     f"{(r['rate'] / prev if prev else 1.0):.2f}x | {'—' if od is None else f'{od:.1e}'} |")
        prev = r["rate"]
    open(path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:] or None)
    elif sys.argv[1] == "ladder-report":
        ladder_report(sys.argv[2])
    else:
        run(sys.argv[2:] or ["C3-f32", "C2", "C3-f64"])
