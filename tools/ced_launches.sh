# per-kernel time / DRAM bytes of CED steps (128^3 O3 plane wave) -> stdout table
cat > /tmp/cedrun.py <<PY
import sys; sys.path.insert(0, '.')
from paper_2211_13295_b200 import ced
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = ced.make_geometry(n, n, n, 3, (0, 0, 0), (1, 1, 1))
st = ced.CedStepper(g, ced.make_params(3)); st.upload(ced.plane_wave(g), 1.0)
st.set_time(0.0, st.cfl_dt(0.4)); st.step(1); st.step(1); st.sync()
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/ced_launch.csv python /tmp/cedrun.py ${1:-128} > /dev/null 2>&1
python - <<PY
import csv
from collections import defaultdict
rows=list(csv.reader(open("gpurun_out/ced_launch.csv")))
hi=next(i for i,r in enumerate(rows) if "Kernel Name" in r); h=rows[hi]
k=h.index("Kernel Name"); m=h.index("Metric Name"); v=h.index("Metric Value")
d=defaultdict(lambda: defaultdict(list))
for r in rows[hi+1:]:
    d[r[k][:40]][r[m]].append(float(r[v].replace(",","")))
for name,x in d.items():
    n=len(x["gpu__time_duration.sum"]); t=sum(x["gpu__time_duration.sum"])/n
    b=(sum(x["dram__bytes_read.sum"])+sum(x["dram__bytes_write.sum"]))/n
    print(f"{name:42s} {t/1e3:9.1f} us {b/1e6:9.1f} MB regs {x['launch__registers_per_thread'][0]:.0f}")
PY
