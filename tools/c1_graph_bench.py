"""configs[0] (128 x 128 x 4, O3, periodic): steps/s with the CUDA-graph replay vs plain
launches (HC_NO_GRAPH=1 in the environment)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import hydro  # noqa: E402

api = hydro.HostApi()
g = hydro.make_geometry(128, 128, 4, 3)
s0 = api.init_isentropic_vortex(g, 3)
st = hydro.Stepper(g, hydro.make_params(3), exact=False)
st.upload(s0)
st.set_time(0.0, api.initial_dt(g, s0, 0.4), 0.4)
st.step(50)
st.sync()
t0 = time.perf_counter()
st.step(2000)
st.sync()
dt = time.perf_counter() - t0
print(f"graph={'off' if os.environ.get('HC_NO_GRAPH') else 'on'} "
      f"us/step={dt / 2000 * 1e6:.1f} Mzone-updates/s={128 * 128 * 4 * 2000 / dt / 1e6:.0f}")
