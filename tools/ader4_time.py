import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2211_13295_b200 import hydro
api = hydro.HostApi()
for n in (128, 256):
    g = hydro.make_geometry(n, n, n, 3)
    s0 = api.init_isentropic_vortex(g, 3)
    st = hydro.Ader4Stepper(g, hydro.make_params(3))
    st.upload(s0); st.set_time(0.0, api.initial_dt(g, s0, 0.4), 0.4)
    st.step(2); st.sync()
    t0 = time.perf_counter(); st.step(5); st.sync(); dt = (time.perf_counter() - t0) / 5
    print(n, "ms/step", dt * 1e3, "Mzone/s", n**3 / dt / 1e6)
    st.close()
