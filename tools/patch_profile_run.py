"""One hc_ader_step (per-kernel path, reference layouts, host buffers) at n^3 O3 -- for the
ncu capture of the per-kernel kernels (tools/ext_profile.sh style)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import hydro  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
api = hydro.HostApi()
g = hydro.make_geometry(n, n, n, 3)
s = api.init_isentropic_vortex(g, 3)
api.apply_boundary_skinny(g, hydro.PERIODIC, s)
m = hydro.zeros_modal(g, 3)
fx, fy, fz = hydro.zeros_faces(g)
r = hydro.zeros_rate(g)
dt = api.initial_dt(g, s, 0.4)
for _ in range(2):
    api.ader_step(g, hydro.make_params(3), m, s, fx, fy, fz, r, dt, 0.4)
