"""Aggregate an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel name."""
import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; k={}
for r in rows:
    if r and r[0]=="ID": hdr={h:i for i,h in enumerate(r)}; continue
    if hdr is None or len(r)!=len(hdr): continue
    key=(int(r[hdr["ID"]]), r[hdr["Kernel Name"]])
    k.setdefault(key,{})[r[hdr["Metric Name"]]]=float(r[hdr["Metric Value"]].replace(",",""))
agg=defaultdict(lambda:[0,0.0,0.0])
for (i,n),m in k.items():
    name=n.split("(")[0][:60]
    a=agg[name]; a[0]+=1; a[1]+=m.get("gpu__time_duration.sum",0)/1e3; a[2]+=(m.get("dram__bytes_read.sum",0)+m.get("dram__bytes_write.sum",0))/1e6
tot=sum(a[1] for a in agg.values())
for n,a in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{n:60s} n={a[0]:4d} {a[1]:9.1f} us ({100*a[1]/tot:4.1f}%) {a[2]/a[1] if a[1] else 0:7.2f} TB/s")
print("total", tot)
