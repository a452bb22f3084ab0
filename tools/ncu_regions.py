"""Region-level instruction and stall shares of one kernel from an `ncu --page source --csv --print-source sass` dump (gz): python tools/ncu_regions.py dump.csv.gz "kernel name substring" [nth]."""
import csv,gzip,sys
csv.field_size_limit(10**9)
rows=list(csv.reader(gzip.open(sys.argv[1],'rt')))
want=sys.argv[2]; nth=int(sys.argv[3]) if len(sys.argv)>3 else 0
starts=[i+1 for i,r in enumerate(rows) if r[0]=='Kernel Name' and want in r[1]]
start=starts[nth]
def kern(start):
    hdr=rows[start]; ix=hdr.index('Instructions Executed'); st=hdr.index('Warp Stall Sampling (All Samples)')
    th=hdr.index('Avg. Threads Executed') if 'Avg. Threads Executed' in hdr else None
    out=[]
    for r in rows[start+1:]:
        if r[0]=='Kernel Name': break
        out.append((int(r[0],16), r[1].strip(), int(r[ix]), int(r[st]), float(r[th]) if th else 0))
    return out
k=kern(start)
base=k[0][0]
tot=sum(x[2] for x in k); stot=sum(x[3] for x in k)
print(rows[start-1][1][:80]); print('total',tot,'samples',stot)
blk=[];acc=0;sacc=0;s0=0
for i,(a,s,n,stl,th) in enumerate(k):
    acc+=n;sacc+=stl
    if 'BRA' in s or 'BAR' in s or 'EXIT' in s or 'BSYNC' in s:
        blk.append((s0,i,acc,sacc)); s0=i+1;acc=0;sacc=0
for (s,e,acc,sacc) in blk:
    if acc>tot*0.004 or sacc>stot*0.01:
        print(f"{k[s][0]-base:5x}-{k[e][0]-base:5x} n={e-s+1:4d} exec {acc/tot*100:5.2f}%  stall {sacc/stot*100:5.2f}%  per-line {acc/(e-s+1):.3g}  thr {sum(x[4]*x[2] for x in k[s:e+1])/max(acc,1):.1f} {k[e][1][:40]}")
