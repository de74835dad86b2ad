"""FMA build vs bit-exact build at full size: per-variable relative L1 / Linf difference of the
256^3 O3 HLL vortex after K steps (the north star's bar is 1e-10 relative L1; the bit-exact build
is the reference's bits). Run: python tools/fma_drift.py [n] [steps] > profiles/r1_fma_drift.json"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import hydro  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    g = hydro.make_geometry(n, n, n, 3)
    api = hydro.HostApi()
    s0 = api.init_isentropic_vortex(g, 3)
    dt0 = api.initial_dt(g, s0, 0.4)
    out = {}
    for exact in (True, False):
        st = hydro.Stepper(g, hydro.make_params(3), exact=exact)
        st.upload(s0)
        st.set_time(0.0, dt0, 0.4)
        st.step(steps)
        t, dt, done = st.sync()
        out[exact] = (st.download(), t)
        st.close()
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    a, b = out[False][0][act].reshape(-1, 5), out[True][0][act].reshape(-1, 5)
    res = {"n": n, "order": 3, "solver": "hll", "steps": steps,
           "t_fma": out[False][1], "t_exact": out[True][1], "rel_l1": [], "rel_linf": []}
    for q in range(5):
        den = max(np.abs(b[:, q]).mean(), 1e-300)
        res["rel_l1"].append(float(np.abs(a[:, q] - b[:, q]).mean() / den))
        res["rel_linf"].append(float(np.abs(a[:, q] - b[:, q]).max() / max(np.abs(b[:, q]).max(), 1e-300)))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
