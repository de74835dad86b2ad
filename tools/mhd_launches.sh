# per-kernel time / DRAM bytes of one MHD step (128^3 O3 Orszag-Tang) -> stdout table
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/mhd_launch.csv python tools/mhd_profile_run.py ${1:-128} ${2:-3} > /dev/null 2>&1
python - <<PY
import csv
from collections import defaultdict
rows=list(csv.reader(open("gpurun_out/mhd_launch.csv")))
hi=next(i for i,r in enumerate(rows) if "Kernel Name" in r); h=rows[hi]
k=h.index("Kernel Name"); m=h.index("Metric Name"); v=h.index("Metric Value")
d=defaultdict(lambda: defaultdict(float)); c=defaultdict(int)
for r in rows[hi+1:]:
    d[r[k][:40]][r[m]]+=float(r[v].replace(",",""))
    if r[m]=="gpu__time_duration.sum": c[r[k][:40]]+=1
tot=sum(x["gpu__time_duration.sum"] for x in d.values())
for name,x in d.items():
    n=c[name]; t=x["gpu__time_duration.sum"]/n
    print(f"{name:42s} {t/1e3:9.1f} us  {100*x['gpu__time_duration.sum']/tot:5.1f}%  {(x['dram__bytes_read.sum']+x['dram__bytes_write.sum'])/n/1e6:9.1f} MB")
PY
