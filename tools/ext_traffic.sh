# DRAM traffic per zone-update of the MHD and CED extension steps (all kernels of 2 steps,
# 128^3 O3, ncu launch lists) -> profiles/r2_ext_traffic.json. Run on the GPU box.
set -e
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ext_mhd.csv \
    python tools/mhd_profile_run.py 128 3 > /dev/null 2>&1
cat > /tmp/cedrun.py <<PY
import sys; sys.path.insert(0, '.')
from paper_2211_13295_b200 import ced
g = ced.make_geometry(128, 128, 128, 3, (0, 0, 0), (1, 1, 1))
st = ced.CedStepper(g, ced.make_params(3)); st.upload(ced.plane_wave(g), 1.0)
st.set_time(0.0, st.cfl_dt(0.4)); st.step(1); st.step(1); st.sync()
PY
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ext_ced.csv \
    python /tmp/cedrun.py > /dev/null 2>&1
python - <<PY
import csv, json
from collections import defaultdict
out = {"how": "ncu --metrics $M over every kernel of 2 steps at 128^3 O3 (tools/ext_traffic.sh); "
              "bytes and time per step, per zone-update"}
for name, f in (("mhd", "gpurun_out/ext_mhd.csv"), ("ced", "gpurun_out/ext_ced.csv")):
    rows = list(csv.reader(open(f)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r); h = rows[hi]
    k, m, v = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = defaultdict(float); per = defaultdict(lambda: defaultdict(float))
    for r in rows[hi + 1:]:
        x = float(r[v].replace(",", ""))
        tot[r[m]] += x
        per[r[k][:48]][r[m]] += x
    zones = 128 ** 3 * 2
    out[name] = {"dram_bytes_per_zone": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / zones,
                 "kernel_ns_per_zone": tot["gpu__time_duration.sum"] / zones,
                 "kernels": {kk: {"dram_bytes_per_zone": (vv["dram__bytes_read.sum"] + vv["dram__bytes_write.sum"]) / zones,
                                  "share": vv["gpu__time_duration.sum"] / tot["gpu__time_duration.sum"]}
                             for kk, vv in per.items()}}
    print(name, round(out[name]["dram_bytes_per_zone"], 1), "B/zone")
json.dump(out, open("gpurun_out/r2_ext_traffic.json", "w"), indent=1)
PY
