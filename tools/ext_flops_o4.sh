# Executed FP64 flops (DADD + DMUL + 2 DFMA, ncu) of one order-4 MHD / CED step at 64^3: the
# whole-process totals of 2 steps minus 1 step (setup kernels cancel) -> gpurun_out/ext_o4_flops.json
set -e
mkdir -p gpurun_out
cat > /tmp/ext_one.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2211_13295_b200 import mhd, ced
w, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if w == "mhd":
    g = mhd.make_geometry(n, n, n, 4, (-5, -5, -5), (5, 5, 5))
    st = mhd.MhdStepper(g, mhd.make_params(4)); st.upload(mhd.mhd_vortex(g, 4))
    st.set_time(0.0, st.cfl_dt(0.4), 0.4)
else:
    g = ced.make_geometry(n, n, n, 4, (0, 0, 0), (1, 1, 1))
    st = ced.CedStepper(g, ced.make_params(4)); st.upload(ced.plane_wave(g), 1.0)
    st.set_time(0.0, st.cfl_dt(0.4))
st.step(steps); st.sync()
PY
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
for w in mhd ced; do for s in 1 2; do
  ncu --metrics $M --clock-control none --csv python /tmp/ext_one.py $w 64 $s > gpurun_out/ext_${w}_$s.csv 2>/dev/null
done; done
python - <<'PY'
import csv, io, json
def total(path):
    lines = [l for l in open(path).read().splitlines() if l.startswith('"ID"') or (l.startswith('"') and l[1:2].isdigit())]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]; iM = h.index("Metric Name"); iV = h.index("Metric Value")
    return sum((2 if 'dfma' in r[iM] else 1) * float(r[iV].replace(',', '')) for r in rows[1:])
out = {"how": "ncu executed FP64 flops (DADD + DMUL + 2 DFMA) of the whole process, 2 steps minus 1 step, 64^3, order 4 (tools/ext_flops_o4.sh)"}
for w in ("mhd", "ced"):
    out[w + "_o4"] = (total(f"gpurun_out/ext_{w}_2.csv") - total(f"gpurun_out/ext_{w}_1.csv")) / 64 ** 3
print(json.dumps(out)); json.dump(out, open("gpurun_out/ext_o4_flops.json", "w"), indent=1)
PY
