"""Summarise an ncu report: key SOL/occupancy/scheduler metrics + SASS hot spots."""
import csv, subprocess, sys
rep = sys.argv[1]
want = ('Duration','DRAM Throughput','L1/TEX Cache Throughput','L2 Cache Throughput','Compute (SM) Throughput',
        'Executed Ipc Active','Issue Slots Busy','Achieved Occupancy','Theoretical Occupancy','Registers Per Thread',
        'Executed Instructions','Warp Cycles Per Issued Instruction','Avg. Active Threads Per Warp',
        'Dynamic Shared Memory Per Block','Block Limit Shared Mem','Grid Size','Block Size','Eligible Warps Per Scheduler','No Eligible')
out = subprocess.run(['ncu','-i',rep,'--page','details','--csv'],capture_output=True,text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
seen=set()
for x in r[1:]:
    if x[mi] in want and (x[ki],x[mi]) not in seen:
        seen.add((x[ki],x[mi])); print(f"{x[ki][:50]:50s} {x[mi]:40s} {x[vi]} {x[ui]}")
if len(sys.argv) > 2:
    out = subprocess.run(['ncu','-i',rep,'--page','source','--csv'],capture_output=True,text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[1]; rows = r[2:]
    ie=h.index('Instructions Executed'); st=h.index('Warp Stall Sampling (All Samples)'); src=h.index('Source')
    tot=sum(int(x[ie] or 0) for x in rows); stt=sum(int(x[st] or 0) for x in rows)
    thr=float(sys.argv[2])
    for k,x in enumerate(rows):
        v=int(x[ie] or 0); s=int(x[st] or 0)
        if v>tot*thr or s>stt*thr:
            print(f"{k:5d} {v/1e6:8.2f}M {100*s/stt:5.1f}% {x[src].strip()[:90]}")
