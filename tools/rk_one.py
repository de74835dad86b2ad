"""One RK step of the fused stepper at n^3 (ncu flop-count target):
python tools/rk_one.py n order integrator(2|3) [exact]"""
import os
import sys
sys.path.insert(0, os.getcwd())
from paper_2211_13295_b200 import hydro  # noqa: E402

n, order, integ = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
exact = len(sys.argv) > 4 and sys.argv[4] == "exact"
api = hydro.HostApi()
g = hydro.make_geometry(n, n, n, order)
s0 = api.init_isentropic_vortex(g, order)
st = hydro.Stepper(g, hydro.make_params(order), exact=exact, integrator=integ)
st.upload(s0)
st.set_time(0.0, api.initial_dt(g, s0, 0.4), 0.4)
st.step(1)
st.sync()
print(st.kernel_info())
st.close()
