"""Convergence of the fourth-order ADER step (csrc/ader4.cu) on the isentropic vortex (2D,
z-invariant, nz = 4) against the exact solution's cell averages, beside the fused stepper's O3
(the reference's scheme) and WENO-AO O4 (reference ADER structure). Prints one JSON line:
per mesh the L1 density error and the observed orders. Usage: python tools/ader4_order.py
[t_final] [meshes...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2211_13295_b200 import hydro  # noqa: E402

t_final = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
meshes = [int(v) for v in sys.argv[2:]] or [32, 64, 128]
api = hydro.HostApi()


def err(n, scheme, cfl):
    order = 3 if scheme in ("o3", "ader4") else 4
    g = hydro.make_geometry(n, n, 4, order, lo=(-5, -5, -5 * 4 / n), hi=(5, 5, 5 * 4 / n))
    s0 = api.init_isentropic_vortex(g, order)
    dt0 = api.initial_dt(g, s0, cfl)
    if scheme == "ader4":
        st = hydro.Ader4Stepper(g, hydro.make_params(3))
    else:
        st = hydro.Stepper(g, hydro.make_params(order), exact=False)
    st.upload(s0)
    st.set_time(0.0, dt0, cfl, t_final)
    done = 0
    while True:
        st.step(64)
        t, _, n_done = st.sync()
        if n_done == done or t >= t_final * (1 - 1e-12):
            break
        done = n_done
    out = st.download()
    ex = api.init_isentropic_vortex(g, order, t=t)
    gh = g.ghost
    st.close()
    return float(np.abs(out[gh:-gh, gh:-gh, gh:-gh, 0] - ex[gh:-gh, gh:-gh, gh:-gh, 0]).mean()), t


res = {"t_final": t_final, "meshes": meshes}
for scheme, cfl in (("ader4", 0.4), ("o3", 0.4), ("o4_weno_ao", 0.4)):
    e = [err(n, scheme, cfl) for n in meshes]
    res[scheme] = {"l1_rho": [x[0] for x in e], "t": [x[1] for x in e],
                   "order": [float(np.log2(e[i][0] / e[i + 1][0])) for i in range(len(e) - 1)]}
print(json.dumps(res))
