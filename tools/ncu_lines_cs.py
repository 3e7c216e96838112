"""Per-CUDA-line instruction and stall share from an ncu report (cuda,sass source view).

Usage: python tools/ncu_lines_cs.py REPORT.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, fname = [], None
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    ie = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        agg.append((int(r[ie] or 0), int(r[st] or 0), f"{fname}:{r[0]}", r[1][:90]))
    except ValueError:
        pass
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"total instructions {ti}, stall samples {ts}")
for a in sorted(agg, key=lambda x: -x[0])[:top]:
    print(f"{100 * a[0] / ti:5.1f}% inst {100 * a[1] / ts:5.1f}% stall  {a[2]:>14}  {a[3]}")
