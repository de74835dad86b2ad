import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2211_13295_b200 import mhd, hydro
for order in (2, 3):
    n = 128
    g = mhd.make_geometry(n, n, 4, order, (0,0,0), (1,1,4.0/n))
    s = mhd.rotor(g, order)
    st = mhd.MhdStepper(g, mhd.make_params(order, gamma=1.4))
    st.upload(s)
    try:
        t, dt, done = st.run(0.4, t_final=0.15)
        out = st.download()
        print("order", order, "ok t", t, "steps", done, "rho range", out[0].min(), out[0].max(), "divb", st.max_divb(), "floored", st.floored)
    except Exception as e:
        print("order", order, "FAILED", str(e)[:200])
