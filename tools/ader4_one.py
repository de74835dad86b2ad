"""One order-4 ADER step at n^3 (ncu target): python tools/ader4_one.py [n]"""
import os
import sys
sys.path.insert(0, os.getcwd())
from paper_2211_13295_b200 import hydro  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
api = hydro.HostApi()
g = hydro.make_geometry(n, n, n, 3)
s0 = api.init_isentropic_vortex(g, 3)
st = hydro.Ader4Stepper(g, hydro.make_params(3))
st.upload(s0)
st.set_time(0.0, api.initial_dt(g, s0, 0.4), 0.4)
st.step(1)
st.sync()
st.close()
