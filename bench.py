#!/usr/bin/env python
"""Benchmark of the B200 all-pairs N-body hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3-f32] [--impl ours|reference]

One bench *step* = one ``simulate`` of the configuration (``steps`` velocity-
Verlet steps = steps+1 force evaluations of N^2 interactions each, the loop of
kernels/__init__.py:240-252) on the device-resident initial state.  Rank 0
prints ONE JSON line.

* ``value``  -- interactions/s over the whole job (all ranks), inputs resident
  in HBM, CUDA events around each step on the launching stream, max over ranks;
  L2 is flushed (256 MB write) between timed steps, outside the events.
* ``e2e``    -- the same metric through the public API ``simulate(system, params)``
  from host NumPy arrays (pinned staging, H2D, kernels, D2H) every step.
* ``roofline`` -- the fused force+update kernel: 20 flop/interaction x N^2 per
  launch / mean launch time, against the nominal FP32 (FP64) CUDA-core peak
  148 SM x 128 (64) lanes x 2 x 1.965 GHz (MEASURED_PEAKS.json carries no
  CUDA-core figure; the microbenchmarked FFMA peak is reported beside it).
* ``cpu_baseline`` -- the reference's own compiled kernel (oracle/_ref, built
  from /root/reference by oracle/Makefile) on all host cores, rank 0 at N=1.

``--impl reference`` times only the reference's CPU implementation of the path
(same config, metric and unit) and prints its own line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "body-body interactions/s (GFLOP/s at 20 flop/int) vs FP32/FP64 CUDA-core peak"
UNIT = "interactions/s"
FLOP_PER_INTERACTION = 20
NOMINAL_CLOCK_HZ = 1.965e9
SMS = 148
# Measured on this pool's B200 with tools/pipe_peaks.cu (profiles/pipe_peaks_r01.txt):
# FFMA 121.3 and DFMA 60.2 lane-ops/SM/clk at 1965 MHz.
MEASURED_FFMA_TFLOPS = 70.6
MEASURED_DFMA_TFLOPS = 35.0
PUBLISHED_CPU_GFLOPS_FP32 = 1524.0  # PAPER.md:445, Numba FP32 best, reference convention
L2_FLUSH_BYTES = 256 << 20


def nominal_peak_tflops(precision_bytes: int) -> float:
    lanes = 128 if precision_bytes == 4 else 64
    return SMS * lanes * 2 * NOMINAL_CLOCK_HZ / 1e12


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML in-process every 5 ms plus one sample right at start and stop
    (so even a sub-millisecond region, C1's, has samples); nvidia-smi as the
    fallback when NVML is unavailable."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, power_w, reason names)
        self._stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _nvml_sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except AttributeError:  # pragma: no cover
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        names = [n for n, attr in self.REASONS if bits & getattr(nv, attr, 0)]
        self.samples.append((float(sm), float(mx), pw, names))

    def _nvml_loop(self):
        while not self._stop.wait(0.005):
            try:
                self._nvml_sample()
            except Exception:  # pragma: no cover
                break

    def start(self):
        try:
            self.nvml = self._nvml_handle()
            self._nvml_sample()
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def _summary(self, source: str) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": source}
        sm = [x[0] for x in self.samples]
        loaded = [x[0] for x in self.samples if x[2] > 300] or sm
        reasons = sorted({n for x in self.samples for n in x[3]})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": reasons, "samples": len(self.samples),
                "power_w_max": max(x[2] for x in self.samples), "source": source}

    def stop(self) -> dict:
        if self.nvml is not None:
            self._stop.set()
            self.thread.join(timeout=2)
            try:
                self._nvml_sample()
            except Exception:  # pragma: no cover
                pass
            return self._summary("nvml (5 ms + start/stop samples)")
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:  # pragma: no cover
            self.proc.kill()
        self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                rec = (float(parts[0]), float(parts[1]), float(parts[2]))
            except ValueError:
                continue
            self.samples.append((*rec, [n for n, flag in zip(names, parts[4:8]) if flag.lower() == "active"]))
        return self._summary("nvidia-smi -lms 100")


# --------------------------------------------------------------------------- CPU baseline

def cpu_reference_rate(cfg, sys0, fixed_n: int = 0, reps: int = 2, warm: bool = True):
    """Reference CPU path on this host: the reference's compiled accel_soa
    (oracle/_ref) over all host threads, soa-recip (its fastest rung), on the
    config's state.  Returns (interactions/s, description dict)."""
    from oracle import oracle as O
    threads = O.host_threads()
    dtype = cfg.precision.dtype
    n = fixed_n or cfg.n
    cols = [np.ascontiguousarray(c[:n], dtype=dtype) for c in sys0.positions]
    m = np.ascontiguousarray(sys0.masses[:n], dtype=dtype)
    out = [np.empty(n, dtype) for _ in range(3)]
    if O.ref_available():
        R = O.ref_module()
        kind = "reference"

        def run():
            R.accel_soa(cols[0], cols[1], cols[2], m, 1.0, cfg.softening_sq, True, 0, threads, *out)
    else:  # the restated port (oracle/nbody_oracle.c), same arithmetic
        kind = "port"

        def run():
            O.accel_soa(cols[0], cols[1], cols[2], m, 1.0, cfg.softening_sq, True, 0, threads)
    if warm:
        run()  # warm-up: OpenMP team, page faults, clock ramp
    t0 = time.perf_counter()
    for _ in range(reps):
        run()
    t = (time.perf_counter() - t0) / reps
    return float(n) * n / t, {"kind": kind, "cores": threads, "seconds": t, "n": n, "reps": reps}


def cpu_rate_isolated(cfg_name: str, fixed_n: int = 0):
    """cpu_reference_rate in a child process, so that a host whose ISA differs
    from the build host of oracle/_ref (-march=native) cannot take the GPU arm
    down with it: the compiled reference first, then the C port; None if both fail."""
    for kind in ("reference", "port"):
        cmd = [sys.executable, os.path.abspath(__file__), "--cpu-child", cfg_name, str(fixed_n), kind]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        except subprocess.TimeoutExpired:
            continue
        if r.returncode == 0 and r.stdout.strip():
            try:
                rate, desc = json.loads(r.stdout.strip().splitlines()[-1])
                return rate, desc
            except ValueError:
                pass
        print(f"cpu baseline ({kind}) failed: rc={r.returncode} {r.stderr[-300:]}", file=sys.stderr)
    return None


def _cpu_child(cfg_name: str, fixed_n: int, kind: str) -> None:
    import paper_2203_08263_b200 as nb
    from oracle import oracle as O
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    if kind == "port":
        O._ref_mod = None
        O.ref_available = lambda: False
    rate, desc = cpu_reference_rate(cfg, cfg.system(), fixed_n=fixed_n)
    print(json.dumps([rate, desc]))


def host_cpu_topology() -> dict:
    """Logical CPUs usable by this process and the physical cores behind them
    (lscpu: distinct (socket, core) pairs), plus the CPU model."""
    info = {"logical_cpus_in_affinity": len(os.sched_getaffinity(0)), "physical_cores": None, "model": None}
    try:
        out = subprocess.run(["lscpu", "-p=CPU,CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        allowed = os.sched_getaffinity(0)
        cores = {(ln.split(",")[2], ln.split(",")[1]) for ln in out.splitlines()
                 if ln and not ln.startswith("#") and int(ln.split(",")[0]) in allowed}
        info["physical_cores"] = len(cores) or None
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name:"):
                info["model"] = ln.split(":", 1)[1].strip()
    except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
        pass
    return info


# --------------------------------------------------------------------------- GPU arm

def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


NCU = "/usr/local/cuda/bin/ncu"


def measure_traffic(args, single_launch: bool) -> dict:
    """roofline.traffic measured in this run: one ncu pass (DRAM read + write
    bytes, --clock-control none) over one launch of the same kernel on the same
    config, in a child process after the timed region (ncu serialises and
    replays the kernel, so nothing it prints is a timing).  Falls back to the
    committed ncu summary (profiles/ncu_summary.json) when ncu is unavailable."""
    if args.no_traffic or not os.path.exists(NCU):
        return {"traffic": load_traffic(args.config), "traffic_source": "profiles/ncu_summary.json (committed capture)"}
    kname = "regex:small_simulate_kernel|simulate_kernel" if single_launch else "regex:step_kernel|pair_kernel"
    cmd = [NCU, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
           "-k", kname, "--launch-skip", "1", "-c", "1", "--csv", "--print-units", "base",
           sys.executable, os.path.abspath(__file__), "--traffic-child", args.config]
    try:
        import csv
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        total = 0.0
        seen = 0
        hdr = None
        for row in csv.reader(ln for ln in r.stdout.splitlines() if ln.startswith('"')):
            if hdr is None:
                hdr = row
                continue
            rec = dict(zip(hdr, row))
            if rec.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(rec.get("Metric Unit"), 1)
                total += float(rec["Metric Value"].replace(",", "")) * scale
                seen += 1
        if seen == 2:
            return {"traffic": total, "traffic_unit": "bytes per launch (dram read + write)",
                    "traffic_source": "ncu in this run: " + " ".join(cmd[1:12]) + " ... (one launch, cold L2)"}
        why = f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-200:]}"
    except (OSError, subprocess.TimeoutExpired, ValueError) as e:
        why = f"ncu failed: {e}"
    return {"traffic": load_traffic(args.config),
            "traffic_source": "profiles/ncu_summary.json (committed capture; in-run ncu unavailable: %s)" % why}


def _traffic_child(cfg_name: str) -> None:
    """Two launches of the config's kernel for the in-run ncu pass (the first is
    skipped): the same state, flags and code path as the timed simulate."""
    import torch
    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200.device import DeviceState, kernel_flags
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    s = cfg.system()
    dtype = cfg.precision.dtype
    st = DeviceState(s.position_matrix().astype(dtype), np.stack(s.velocities, 1), s.masses, dtype)
    p = cfg.params()
    flags = kernel_flags(s.masses, p.softening_sq, dtype)
    for _ in range(2):
        st.simulate(p.gravitational_constant, p.dt, p.softening_sq, p.steps, flags)
    torch.cuda.synchronize()


def load_traffic(config_name: str):
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            data = json.load(f)
        entry = data.get(config_name) or {}
        return entry.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def run_ours(args) -> dict:
    import torch
    import torch.distributed as dist

    import paper_2203_08263_b200 as nb
    from paper_2203_08263_b200 import _native
    from paper_2203_08263_b200._native import NB_STEP_FINAL_KICK, NB_STEP_FIRST, NB_STEP_KICK_DRIFT
    from paper_2203_08263_b200.device import DeviceState, kernel_flags, needs_self_mask
    from paper_2203_08263_b200.sharded import gather_into, pad_system, run_sharded, shard_range

    world, rank, local = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # One process per GPU.  Test hook (never the measured configuration):
    # NB_BENCH_BACKEND=gloo with more ranks than GPUs runs the multi-rank driver
    # logic with ranks sharing a device and a host-side exchange.
    backend = os.environ.get("NB_BENCH_BACKEND", "nccl")
    if backend == "nccl" and world > torch.cuda.device_count():
        raise SystemExit(f"--gpus {world} needs {world} visible GPUs (one process per GPU); "
                         f"found {torch.cuda.device_count()}")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            # NCCL's communicator log (stderr) shows every rank joining
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = nb.BASELINE_CONFIGS[args.config]
    params = cfg.params()
    sys0 = cfg.system()
    dtype = cfg.precision.dtype
    pbytes = dtype.itemsize
    pos0 = sys0.position_matrix().astype(dtype)
    vel0 = np.stack(sys0.velocities, axis=1)
    m0 = sys0.masses
    pos, vel, m = pad_system(pos0, vel0, m0, world)
    npad = pos.shape[0]
    i0, ni = shard_range(npad, rank, world)
    mask = kernel_flags(m, cfg.softening_sq, dtype) & ~1
    mask |= 1 if needs_self_mask(m0, cfg.softening_sq, dtype) else 0
    p2p = world > 1 and args.transport == "p2p"
    if p2p:
        from paper_2203_08263_b200.sharded import _p2p_setup, run_sharded_p2p
        state, peer_next, p2p_barrier = _p2p_setup(pos, vel, m, dtype, i0, ni, None)
    else:
        state = DeviceState(pos, vel, m, dtype, device=dev, i_begin=i0, n_i=ni)
    capi_gather = None
    if world > 1 and args.transport == "capi":  # the exchange through the library's nb_comm_* C ABI
        from paper_2203_08263_b200.sharded import _capi_allgather
        capi_gather = _capi_allgather(None)
    pristine_pos = state.pos_a.clone()
    pristine_vel = state.vel.clone()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    g, dt, eps2, steps = params.gravitational_constant, params.dt, params.softening_sq, params.steps

    def reset():
        state.pos_a.copy_(pristine_pos)
        state.vel.copy_(pristine_vel)
        state.acc.zero_()
        state.cur_is_a = True

    launch_ms_all = []

    def one_step(record_launches: bool):
        """One simulate of the config on the resident state (steps+1 launches).
        N=1: the product's own C loop (nb_dev_simulate[_timed]); the timed
        variant records a CUDA event between consecutive launches on the launch
        stream and returns each launch's device time.  N>1: the sharded driver."""
        if world == 1:
            if record_launches:
                ms = state.simulate_timed(g, dt, eps2, steps, mask)
                launch_ms_all.append(ms)
                return sum(ms)
            state.simulate(g, dt, eps2, steps, mask)
            return None

        if p2p:
            run_sharded_p2p(state, g, dt, eps2, steps, mask, peer_next, p2p_barrier)
            return None

        if capi_gather is not None:
            run_sharded(state, g, dt, eps2, steps, mask, capi_gather, world)
            return None

        def gather(full, local_rows):
            return gather_into(full, local_rows, async_op=True)
        run_sharded(state, g, dt, eps2, steps, mask, gather, world)
        return None

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local_dev])
            else:
                dist.barrier()

    # ---------------------------------------------------------------- warm-up
    for _ in range(args.warmup):
        reset()
        one_step(False)
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed region
    clocks = ClockSampler(local_dev)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches_before = _native.launch_count()
    barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        reset()
        flush.zero_()  # L2 flush between timed steps (outside the events)
        starts[k].record()
        one_step(record_launches=False)
        ends[k].record()
    torch.cuda.synchronize()
    barrier()
    launches = _native.launch_count() - launches_before
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    # Per-launch kernel time for the roofline: the same simulate once more with an
    # event between consecutive launches (kept out of the timed steps because an
    # event between launches breaks the programmatic-dependent-launch overlap).
    if world == 1:
        reset()
        flush.zero_()
        one_step(record_launches=True)
        torch.cuda.synchronize()
    clk = clocks.stop()
    total_s = sum(step_ms) / 1e3
    if world > 1:
        t = torch.tensor([total_s], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = float(t.item())
    interactions = float(cfg.n) * cfg.n * (steps + 1) * args.steps
    value = interactions / total_s

    # per-launch kernel durations (N=1): the dominant (only) kernel of the step
    kernel_ms = [x for ms in launch_ms_all for x in ms]
    peak = nominal_peak_tflops(pbytes)
    launches_per_sim = launches / max(1, args.steps)
    kernel_name = "nb::step_kernel (fused force + velocity-Verlet epilogue) + nb::fixup_kernel"
    if world == 1 and _native.step_kernel_name(pbytes, cfg.n, cfg.n) == "pair_kernel":
        kernel_name = ("nb::pair_kernel (2-CTA cluster split-source force + velocity-Verlet epilogue; "
                       "no fixup launch)")
    launch_timing = ("CUDA events between consecutive launches on the launch stream "
                     "(nb_dev_simulate_timed), one simulate right after the timed steps")
    single_launch = world == 1 and launches_per_sim == 1
    if single_launch:
        # Small N: the whole simulate is ONE cooperative launch (small_simulate_kernel
        # or simulate_kernel), so the events around each timed step bracket exactly
        # that kernel; its steps+1 force evaluations are the algorithmic work.
        mean_launch_s = statistics.mean(step_ms) / 1e3
        achieved = FLOP_PER_INTERACTION * float(cfg.n) * cfg.n * (steps + 1) / mean_launch_s / 1e12
        kernel_name = ("nb::small_simulate_kernel" if cfg.n <= (3584 if pbytes == 4 else 2560)
                       else "nb::simulate_kernel") + " (the whole simulate in one cooperative launch)"
        launch_timing = "CUDA events around each timed step = around its single launch"
    elif world == 1:
        # Each timed step is one simulate = steps+1 step launches back to back on
        # the launch stream (each followed by its split-i-block fixup launch, PDL
        # overlap intact): the events around the step over steps+1 are the step
        # kernel's mean launch duration with its fixup included.  The events-
        # between-launches pass (kernel_ms) serialises each launch pair and is
        # reported beside it.
        mean_launch_s = statistics.mean(step_ms) / 1e3 / (steps + 1)
        achieved = FLOP_PER_INTERACTION * float(cfg.n) * cfg.n / mean_launch_s / 1e12
        launch_timing = ("CUDA events around each timed simulate on its launch stream / its steps+1 step "
                         "launches (with their fixup launches where stream-K splits i-blocks; PDL overlap intact)")
    else:
        mean_launch_s = total_s / (args.steps * (steps + 1))
        achieved = FLOP_PER_INTERACTION * interactions / total_s / 1e12 / world
    roofline = {
        "bound": "fp32_cuda_core" if pbytes == 4 else "fp64_cuda_core",
        "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
        "peak_source": "nominal 148 SM x %d lanes x 2 x 1.965 GHz (no CUDA-core figure in MEASURED_PEAKS.json)"
                       % (128 if pbytes == 4 else 64),
        "peak_measured_microbench": MEASURED_FFMA_TFLOPS if pbytes == 4 else MEASURED_DFMA_TFLOPS,
        "frac_of_measured_microbench": achieved / (MEASURED_FFMA_TFLOPS if pbytes == 4 else MEASURED_DFMA_TFLOPS),
        "kernel": kernel_name,
        "mean_launch_ms": mean_launch_s * 1e3,
        "launch_timing": launch_timing,
        "mean_launch_ms_serialised": statistics.mean(kernel_ms) if kernel_ms else None,
        "algorithmic_flop_per_launch": FLOP_PER_INTERACTION * float(cfg.n) * cfg.n * ((steps + 1) if single_launch else 1),
    }
    roofline.update(measure_traffic(args, single_launch) if world == 1 else
                    {"traffic": None, "traffic_source": "not measured for N > 1 (ncu profiles one GPU)"})

    # ---------------------------------------------------------------- e2e through the public API
    e2e = None
    if not args.no_e2e:
        sys_host = cfg.system()
        for _ in range(args.warmup):
            nb.simulate(sys_host, params)
        torch.cuda.synchronize()
        # Sub-millisecond simulates (C1: ~75 us) are timed over ~0.2 s of calls
        # (after as many more warm-up calls) so the rate is not a handful of
        # calls' jitter; every call is a full simulate with its own uploads and
        # readback.
        tw = time.perf_counter()
        nb.simulate(sys_host, params)
        per_call = time.perf_counter() - tw
        calls = max(args.steps, min(5000, int(0.2 / max(per_call, 1e-6)) + 1))
        if world > 1:
            # every rank runs the same number of calls -- agreed BEFORE the extra
            # warm-up calls: a sharded simulate is a collective, so ranks whose own
            # timings gave different counts would otherwise leave it mismatched
            t = torch.tensor([calls], dtype=torch.int64, device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            calls = int(t.item())
        for _ in range(calls if calls > args.steps else 0):
            nb.simulate(sys_host, params)
        barrier()
        t0 = time.perf_counter()
        final = None
        for _ in range(calls):
            final = nb.simulate(sys_host, params)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) * args.steps / calls
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        # Bytes each simulate() moves (whole job): N=1 uploads the column block
        # x, y, z, m, vx, vy, vz (7 N) and reads the same block back (one copy:
        # the result columns plus the unchanged masses); a sharded rank uploads
        # x, y, z, m of all padded bodies plus its own velocity rows and reads
        # back all N positions and velocities.
        if world == 1:
            h2d, d2h = 7 * cfg.n * pbytes, 7 * cfg.n * pbytes
        else:
            h2d = world * (4 * npad + 3 * ni) * pbytes
            d2h = world * 6 * cfg.n * pbytes
        e2e = {"value": interactions / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "api": "paper_2203_08263_b200.simulate(ParticleSystem, SimParams) from host NumPy arrays"
                      + (f" on each of {world} ranks (i-sharded; bytes summed over ranks)" if world > 1 else ""),
               "checksum": nb.checksum(final),
               "calls_timed": calls}

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_s * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": (FLOP_PER_INTERACTION * float(cfg.n) * cfg.n * steps * args.steps / total_s / 1e9)
                       / PUBLISHED_CPU_GFLOPS_FP32 if pbytes == 4 else None,
        "dtype": "f32" if pbytes == 4 else "f64", "data": "synthetic (BASELINE.json generator, seed 0)",
        "config": {"workload": cfg.name, "n_bodies": cfg.n, "integrator_steps": steps,
                   "force_evaluations_per_step": steps + 1, "softening_sq": cfg.softening_sq,
                   "dt": cfg.dt, "distribution": cfg.generator.__name__,
                   "parallelism": f"i-shard x{world} ({args.transport})" if world > 1 else "1 GPU",
                   "l2": "flushed (256 MB write) between timed steps"},
        "gflops_20": FLOP_PER_INTERACTION * value / 1e9,
        "gflops_reference_convention": FLOP_PER_INTERACTION * float(cfg.n) * cfg.n * steps * args.steps
                                       / total_s / 1e9,
        "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        got = cpu_rate_isolated(args.config)
        if got is None:
            result["cpu_baseline"] = {"value": None, "unit": UNIT, "unavailable": "CPU reference failed on this host"}
        else:
            rate, desc = got
            what = "the reference's compiled accel_soa" if desc["kind"] == "reference" else "the oracle C port"
            result["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": desc["cores"], "kind": desc["kind"],
                "host_cpu": host_cpu_topology(),
                "sample": f"mean of {desc['reps']} force evaluations (N^2 = {desc['n'] ** 2:.3e} "
                          f"interactions each, after one warm-up evaluation) of the {cfg.name} initial "
                          f"state through {what} (soa-recip, {desc['cores']} threads), "
                          f"{desc['seconds']:.2f} s each"}
    if world > 1:
        dist.destroy_process_group()
    return result if rank == 0 else None


BASELINE_REF = os.path.join(REPO, "baseline", "_ref")


def _ref_child(cfg_name: str, n_s: int, reps: int, warm: int) -> None:
    """The UNMODIFIED reference (baseline/_ref, pip-installed from /root/reference)
    through its own public API: nbodybench.harness.measure on the config (its
    first n_s bodies), variant soa-recip on every host thread -- the
    reference's fastest rung -- so kernels.simulate runs its stock path
    (compiled accel_soa + step_soa + NumPy _kick).  Prints one JSON list."""
    sys.path.insert(0, BASELINE_REF)
    import nbodybench as R
    from nbodybench import harness
    import paper_2203_08263_b200 as nb
    from oracle import oracle as O
    cfg = nb.BASELINE_CONFIGS[cfg_name]
    assert "cext" in R.kernels.available_backends(), "reference compiled extension missing"
    R.set_backend("cext")
    threads = O.host_threads()
    full = cfg.system()
    prec = R.Precision(cfg.precision.value)

    def init_fn(n, seed, precision, layout):  # the BASELINE generator, as a reference ParticleSystem
        pos = tuple(np.ascontiguousarray(c[:n]) for c in full.positions)
        vel = tuple(np.ascontiguousarray(c[:n]) for c in full.velocities)
        return R.ParticleSystem(R.Layout.SOA, precision, pos, vel, np.ascontiguousarray(full.masses[:n]))

    bc = harness.BenchConfig(n_bodies=n_s, steps=cfg.steps,
                             variant=R.KernelVariant(R.Layout.SOA, R.MathForm.RECIPROCAL_MULTIPLY, None, threads),
                             precision=prec, repetitions=reps, warmup_runs=warm,
                             gravitational_constant=1.0, dt=cfg.dt, softening_sq=cfg.softening_sq)
    res = harness.measure(bc, init_fn=init_fn)
    print(json.dumps([res.times_s, res.checksum, res.gflops_mean, res.status, res.backend, threads,
                      R.__file__]))


def run_reference(args) -> dict:
    """The reference's own CPU implementation of the path on the host cores;
    same config, metric and unit.  Rank 0 only.  Primary: the installed
    reference package's harness.measure -> kernels.simulate (stock code path)
    on a bounded sample of the config's bodies; fallback (package missing or
    unusable on this host): its compiled accel_soa (oracle/_ref), one force
    evaluation per step."""
    import paper_2203_08263_b200 as nb
    world, rank, _ = _dist_env()
    if rank != 0:
        return None
    cfg = nb.BASELINE_CONFIGS[args.config]
    sys0 = cfg.system()
    probe = cpu_rate_isolated(args.config)  # also proves the compiled kernel runs on this host
    if probe is None:
        return {"impl": "reference", "unavailable": "the reference's compiled CPU kernel and its C port "
                                                    "both failed on this host"}
    rate, desc = probe
    # size the sample so the whole run (warm-up + timed simulates) stays within ~3 minutes
    budget = 150.0
    evals = cfg.steps + 1
    per_sim_full = desc["seconds"] * evals
    n_s = cfg.n
    if per_sim_full * (args.steps + args.warmup) > budget:
        n_s = int(cfg.n * (budget / (per_sim_full * (args.steps + args.warmup))) ** 0.5) // 1024 * 1024
        n_s = max(min(n_s, cfg.n), 1024)
    base = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if cfg.precision.dtype.itemsize == 4 else "f64",
            "data": "synthetic (BASELINE.json generator, seed 0)"}
    cmd = [sys.executable, os.path.abspath(__file__), "--ref-child", args.config, str(n_s), str(args.steps),
           str(args.warmup)]
    got = None
    if os.path.isdir(os.path.join(BASELINE_REF, "nbodybench")):
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
            if r.returncode == 0 and r.stdout.strip():
                got = json.loads(r.stdout.strip().splitlines()[-1])
            else:
                print(f"reference package run failed: rc={r.returncode} {r.stderr[-400:]}", file=sys.stderr)
        except (subprocess.TimeoutExpired, ValueError) as e:
            print(f"reference package run failed: {e}", file=sys.stderr)
    if got is not None:
        times, checksum, gflops_mean, status, backend, threads, where = got
        total = float(sum(times))
        value = float(n_s) * n_s * evals * len(times) / total
        sample = (f"nbodybench.harness.measure (the installed reference, {os.path.relpath(where, REPO)}) on the "
                  f"first {n_s} bodies of the {cfg.name} state, {cfg.steps} steps = {evals} force evaluations "
                  f"per simulate, variant soa-recip on {threads} threads, backend {backend}; "
                  f"{args.warmup} untimed warm-up + {len(times)} timed simulates (harness clock)")
        return {**base, "value": value, "ms_per_step": total * 1e3 / len(times),
                "config": {"workload": cfg.name, "n_bodies": cfg.n, "sample_bodies": n_s,
                           "integrator_steps": cfg.steps, "force_evaluations_per_step": evals,
                           "softening_sq": cfg.softening_sq, "dt": cfg.dt,
                           "path": "nbodybench.kernels.simulate via harness.measure (stock)"},
                "gflops_20": FLOP_PER_INTERACTION * value / 1e9,
                "gflops_reference_convention": gflops_mean, "checksum": checksum, "status": status,
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                                 "host_cpu": host_cpu_topology(), "sample": sample},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}

    # fallback: one force evaluation per step through the compiled accel_soa
    from oracle import oracle as O
    if desc["kind"] != "reference":
        O.ref_available = lambda: False
    n_f = max(min(cfg.n, int(n_s * evals ** 0.5) // 1024 * 1024), 1024)
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, sys0, fixed_n=n_f, reps=1, warm=False)
    total, inter = 0.0, 0.0
    for _ in range(args.steps):
        r, d = cpu_reference_rate(cfg, sys0, fixed_n=n_f, reps=1, warm=False)
        total += d["seconds"]
        inter += float(n_f) * n_f
    value = inter / total
    sample = (f"per step one force evaluation of the first {n_f} bodies of the {cfg.name} state "
              f"({float(n_f) ** 2:.3e} interactions) through the reference's compiled accel_soa "
              f"(soa-recip, {desc['cores']} threads); simulate() is steps+1 such evaluations "
              f"(installed reference package unavailable)")
    return {**base, "value": value, "ms_per_step": total * 1e3 / args.steps,
            "config": {"workload": cfg.name, "n_bodies": cfg.n, "sample_bodies": n_f,
                       "path": "compiled accel_soa only (fallback)"},
            "gflops_20": FLOP_PER_INTERACTION * value / 1e9,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": desc["cores"], "kind": desc["kind"],
                             "host_cpu": host_cpu_topology(), "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def spawn_ranks(args, argv) -> int:
    """``--gpus N > 1`` without a torchrun environment: re-run this script under
    ``torch.distributed.run`` with one process per GPU (the driver's own launch
    form), forwarding the ranks' output; rank 0 prints the one JSON line.
    NCCL's communicator log stays on (NCCL_DEBUG=INFO, stderr) so the rank count
    is visible in the log."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3-f32",
                    choices=["C1", "C2", "C3-f32", "C3-f64", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--transport", default="nccl", choices=["nccl", "capi", "p2p"],
                    help="N>1 position exchange: NCCL all-gather through torch.distributed (default), the same through the library's nb_comm_* C ABI, or the fused peer-store epilogue")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-traffic", action="store_true", help="skip the in-run ncu DRAM-traffic pass")
    ap.add_argument("--traffic-child", metavar="CONFIG", help=argparse.SUPPRESS)
    ap.add_argument("--ref-child", nargs=4, metavar=("CONFIG", "N", "REPS", "WARM"), help=argparse.SUPPRESS)
    ap.add_argument("--cpu-child", nargs=3, metavar=("CONFIG", "N", "KIND"), help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.cpu_child:
        _cpu_child(args.cpu_child[0], int(args.cpu_child[1]), args.cpu_child[2])
        return
    if args.traffic_child:
        _traffic_child(args.traffic_child)
        return
    if args.ref_child:
        c, n, reps, warm = args.ref_child
        _ref_child(c, int(n), int(reps), int(warm))
        return
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args, sys.argv[1:] if argv is None else list(argv)))
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
