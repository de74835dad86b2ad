"""Convergence of the CED orders 2 / 3 / 4 on the oblique plane wave (tests' _wave_error setup:
16^3 -> 32^3 -> 64^3 to t = 0.25, L1 error of the face fields vs the exact face averages),
and the uniform-field relaxation exp(-sigma t / eps) at sigma dt = 5 for order 4 (the
implicit Radau IIA predictor). One JSON line."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2211_13295_b200 import ced  # noqa: E402


def active(s, g):
    gh = g.ghost
    return s[:, gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]


def wave(n, order, tf=0.25):
    g = ced.make_geometry(n, n, n, order, (0, 0, 0), (1, 1, 1))
    st = ced.CedStepper(g, ced.make_params(order))
    st.upload(ced.plane_wave(g), 0.0)
    t, steps = st.run(0.4, tf)
    err = float(np.abs(active(st.download(), g) - active(ced.plane_wave(g, t=t), g)).mean())
    divb, divd = st.max_div()
    st.close()
    return err, divb, divd


res = {}
for order in (2, 3, 4):
    e = [wave(n, order) for n in (16, 32, 64)]
    res[f"o{order}"] = {"l1": [x[0] for x in e], "div": [max(x[1], x[2]) for x in e],
                        "order": [math.log2(e[i][0] / e[i + 1][0]) for i in range(2)]}
g = ced.make_geometry(8, 8, 8, 4, (0, 0, 0), (1, 1, 1))
st = ced.CedStepper(g, ced.make_params(4))
d0 = (1.0, -0.5, 0.25)
dt = st.cfl_dt(0.4)
sig = 5.0 / dt
st.upload(ced.uniform_field(g, d0), sig)
st.set_time(0.0, dt)
st.step(10)
t, _, _ = st.sync()
s = active(st.download(), g)
res["relax_o4"] = {"sigma_dt": 5.0, "D_over_exact": float(s[0].mean() / (d0[0] * math.exp(-sig * t)))}
st.close()
print(json.dumps(res))
