# ncu --set full captures of the extension kernels (MHD predictor / EMF / flux, CED predictor /
# edge) at 128^3 O3 -> gpurun_out/prof_{mhd,ced}.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:"k_mhd_(predict|emf|flux|update)" -s 12 -c 6 -o gpurun_out/prof_mhd python tools/mhd_profile_run.py 128 3 > gpurun_out/pm.log 2>&1
cat > /tmp/cedrun.py <<PY
import sys; sys.path.insert(0, '.')
from paper_2211_13295_b200 import ced
n = 128
g = ced.make_geometry(n, n, n, 3, (0, 0, 0), (1, 1, 1))
st = ced.CedStepper(g, ced.make_params(3)); st.upload(ced.plane_wave(g), 0.0)
st.set_time(0.0, st.cfl_dt(0.4)); st.step(3); st.sync()
PY
ncu --set full --clock-control none --import-source on -k regex:"k_ced_(predict|edge|update)" -s 5 -c 5 -o gpurun_out/prof_ced python /tmp/cedrun.py > gpurun_out/pc.log 2>&1
ls -la gpurun_out/*.ncu-rep
