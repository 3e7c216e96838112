"""Write a markdown summary of a gpu_round.sh output directory into profiles/.

Usage: python tools/profile_summary.py gpurun_out/<tag> profiles/<tag>
Produces <prefix>_ncu_summary.md (per-kernel ncu --set full metrics), <prefix>_launches.txt
(aggregated launch list) and copies the bench lines.
"""
import csv
import json
import os
import subprocess
import sys

src, prefix = sys.argv[1], sys.argv[2]
WANT = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Executed Instructions", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"
traffic = {}
out = ["# ncu --set full summaries (" + os.path.basename(src.rstrip('/')) + ")", "",
       "One capture per kernel of `bench.py --workload W --steps 1 --warmup 3`, "
       "`--clock-control none`. Times under ncu are serialised and cold-cache; compare shares, "
       "not absolutes.", ""]
for f in sorted(os.listdir(src)):
    if not f.endswith(".ncu-rep"):
        continue
    rep = os.path.join(src, f)
    d = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(d.splitlines()))
    if not rows:
        continue
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    kname = rows[1][ki] if len(rows) > 1 else f
    got = {}
    for r in rows[1:]:
        if r[mi] in WANT and r[mi] not in got:
            got[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rawv, stalls, units = {}, {}, {}
    if len(rr) >= 3:
        for k, u, v in zip(rr[0], rr[1], rr[2]):
            if k in RAW:
                rawv[k] = v
                units[k] = u
            if k.startswith(STALLS) and not k.endswith("not_issued"):
                try:
                    stalls[k[len(STALLS):]] = float(v)
                except ValueError:
                    pass
    try:
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        nbytes = sum(float(rawv[k]) * scale[units[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        short = kname.split("::")[-1].split("(")[0].split("<")[0].strip()
        wl = f.split("_")[1] if f.startswith("full_") else ""  # full_<workload>_<kernel>
        traffic[f"{wl}:{short}" if wl else short] = {
            "dram_bytes_per_launch": nbytes, "kernel": kname, "workload": wl,
            "source": os.path.basename(prefix) + "_ncu_summary.md"}
    except (ValueError, KeyError):
        pass
    out.append(f"## `{kname[:110]}`" + (f" — {f.split('_')[1]}" if f.startswith("full_") else ""))
    out.append("")
    out.append("| metric | value |")
    out.append("|---|---|")
    for k in WANT:
        if k in got:
            out.append(f"| {k} | {got[k]} |")
    for k in RAW:
        if k in rawv:
            out.append(f"| {k} | {rawv[k]} {units.get(k, '')} |")
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda x: -x[1])[:6]
    out.append("| top stall reasons (pc samples) | " +
               ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top) + " |")
    out.append("")
with open(prefix + "_ncu_summary.md", "w") as fh:
    fh.write("\n".join(out) + "\n")
for lname in sorted(os.listdir(src)):
    if not (lname.startswith("launches") and lname.endswith(".csv")):
        continue
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "launch_table.py"),
                        os.path.join(src, lname), "5"], capture_output=True, text=True).stdout
    with open(prefix + "_" + lname[:-4] + ".txt", "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none, "
                 "bench.py --steps 2 --warmup 3 (5 device builds + 5 public builds)\n" + r)
for name in ("bench.json", "bench_ref.json", "bench_sharded1.json"):
    p = os.path.join(src, name)
    if os.path.exists(p):
        lines = [ln for ln in open(p).read().splitlines() if ln.strip().startswith("{")]
        if lines:
            with open(prefix + "_" + name, "w") as fh:
                fh.write(lines[-1] + "\n")
with open(os.path.join(os.path.dirname(prefix) or ".", "roofline_traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)
print("wrote", prefix + "_*")
