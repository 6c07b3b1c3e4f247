#!/usr/bin/env python
"""Split the SASS page of one kernel of an .ncu-rep into segments of equal execution count (basic blocks,
loop bodies) and print each segment's share of the warp instructions, mean active lanes and opcode mix:
    ncu -i rep.ncu-rep --page source --csv --print-source sass -k regex:k_solve_group > sass.csv
    python scripts/ncu_segments.py sass.csv [min_share]
(development tooling; needs -lineinfo and --import-source on at capture time)"""
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=[r for r in rows[2:] if len(r)==len(hdr) and r[0].startswith("0x")]
ia=hdr.index("Address"); isrc=hdr.index("Source"); ie=hdr.index("Instructions Executed"); it=hdr.index("Avg. Threads Executed"); isamp=hdr.index("# Samples")
tot=sum(int(r[ie]) for r in data)
prev=None; seg=[]
out=[]
for k,r in enumerate(data):
    e=int(r[ie]); 
    if prev is None or abs(e-prev)>0.02*max(e,prev,1):
        if seg: out.append(seg)
        seg=[]
    seg.append((k,r[isrc].strip(),e,float(r[it]),int(r[isamp])))
    prev=e
out.append(seg)
print("total",tot, "segments",len(out), "sass",len(data))
thr=float(sys.argv[2]) if len(sys.argv)>2 else 0.004
for seg in out:
    e=sum(s[2] for s in seg); 
    if e/tot<thr: continue
    ops={}
    for s in seg:
        w=s[1].split()
        op=w[0] if not w[0].startswith('@') else w[1]
        op=op.split('.')[0]
        ops[op]=ops.get(op,0)+1
    top=sorted(ops.items(), key=lambda x:-x[1])[:7]
    print(f"[{seg[0][0]:5d}-{seg[-1][0]:5d}] n={len(seg):4d} exec/inst={seg[0][2]:9d} share={e/tot:6.2%} thr={sum(s[3] for s in seg)/len(seg):5.1f} samp={sum(s[4] for s in seg):6d} {top}")
