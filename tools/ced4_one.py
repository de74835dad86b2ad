"""One CED order-4 step at n^3 (ncu target): python tools/ced4_one.py [n]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import ced  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
g = ced.make_geometry(n, n, n, 4, (0, 0, 0), (1, 1, 1))
st = ced.CedStepper(g, ced.make_params(4))
st.upload(ced.plane_wave(g), 1.0)
st.set_time(0.0, st.cfl_dt(0.4))
st.step(1)
st.sync()
st.close()
