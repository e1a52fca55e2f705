"""Summarise an ncu --set full report (and optional launch-list CSV) into profiles/.
usage: python tools/ncu_summarize.py REPORT.ncu-rep CONFIG [LAUNCHES.csv]"""
import csv, io, json, os, subprocess, sys
rep, config = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else None
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_elapsed.avg",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]
out = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    ent = {}
    for k in KEYS:
        if k in hdr:
            v = r[hdr.index(k)]
            try:
                ent[k] = float(v.replace(",", ""))
                ent[k + ".unit"] = units[hdr.index(k)]
            except ValueError:
                ent[k] = v
    out.setdefault(name, ent)
def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return v * scale
summ_path = os.path.join(REPO, "profiles", "ncu_summary.json")
summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
# excess shared-memory wavefronts (bank conflicts that cost time) from the source page
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
excess = None
if len(srows) > 2 and "L1 Wavefronts Shared Excessive" in srows[1]:
    sh = srows[1]
    iw, iws = sh.index("L1 Wavefronts Shared Excessive"), sh.index("L1 Wavefronts Shared")
    num = lambda v: float(v.replace(",", "")) if v not in ("", "-") else 0.0
    excess = {"shared_wavefronts": sum(num(r[iws]) for r in srows[2:]),
              "shared_wavefronts_excessive": sum(num(r[iw]) for r in srows[2:])}
for name, ent in out.items():
    if excess:
        ent.update(excess)
    if "step_kernel" in name or "pair_kernel" in name or "simulate_kernel" in name:
        dr = to_bytes(ent.get("dram__bytes_read.sum", 0), ent.get("dram__bytes_read.sum.unit", "byte"))
        dw = to_bytes(ent.get("dram__bytes_write.sum", 0), ent.get("dram__bytes_write.sum.unit", "byte"))
        summ[config] = {"kernel": name, "dram_bytes_per_launch": dr + dw, "metrics": ent,
                        "report": os.path.basename(rep)}
if launches:
    lrows = [r for r in csv.reader(open(launches)) if len(r) > 5]
    h = lrows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in lrows[1:]:
        try:
            agg.setdefault(r[ki].split("(")[0][:80], []).append(float(r[vi].replace(",", "")))
        except (ValueError, IndexError):
            pass
    tot = sum(sum(v) for v in agg.values())
    summ.setdefault(config, {})["launch_list"] = {k: {"count": len(v), "total_ns": sum(v), "share": sum(v) / tot}
                                                  for k, v in agg.items()}
json.dump(summ, open(summ_path, "w"), indent=1)
print(json.dumps(summ[config], indent=1)[:3000])
