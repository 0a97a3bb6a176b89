"""Dev tool: per-kernel totals of an ncu --csv gpu__time_duration launch list.
usage: python tools/launch_summary.py launches.csv"""
import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r))
    if d.get('Metric Name')!='gpu__time_duration.sum': continue
    v=float(d['Metric Value'].replace(',','')); u=d['Metric Unit']
    v = v/1e6 if u in ('nsecond','ns') else v/1e3 if u in ('usecond','us') else v
    k=d['Kernel Name'][:90]; agg[k][0]+=1; agg[k][1]+=v
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{v[1]:10.3f} ms {v[0]:5d} {100*v[1]/tot:5.1f}%  {k}")
print(f"total {tot:.3f} ms")
