"""Instruction/stall breakdown of an ncu report's SASS by runs of equal execution count."""
import csv, subprocess, sys
rep = sys.argv[1]; rows_per = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(['ncu','-i',rep,'--page','source','--csv'],capture_output=True,text=True).stdout
r = list(csv.reader(out.splitlines())); h = r[1]; rows = r[2:]
ie=h.index('Instructions Executed'); st=h.index('Warp Stall Sampling (All Samples)'); src=h.index('Source')
tot=sum(int(x[ie] or 0) for x in rows); stt=sum(int(x[st] or 0) for x in rows)
print(f"total instr {tot/1e6:.0f}M = {tot/rows_per:.0f} per unit")
prev=None; start=0; accv=0; accs=0; segs=[]
for k,x in enumerate(rows+[['0']*len(h)]):
    v=int(x[ie] or 0) if k < len(rows) else -1; s=int(x[st] or 0) if k < len(rows) else 0
    key=round(v/(tot/2000+1))
    if prev is None or key!=prev:
        if prev is not None and accv>0: segs.append((start,k-1,accv,accs,rows[start][src].strip()[:60]))
        prev=key; start=k; accv=0; accs=0
    accv+=max(v,0); accs+=s
for a,b,v,s,t in segs:
    if v>tot*0.01 or s>stt*0.01:
        cnt=int(rows[a][ie] or 0)
        print(f"{a:5d}-{b:5d} x{cnt/rows_per:7.1f}/unit  {b-a+1:4d} ins  instr={100*v/tot:5.1f}% stall={100*s/stt:5.1f}%  {t}")
