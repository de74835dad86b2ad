"""CPU checks of the CED restatement (oracle/ced_oracle.py), the checker of the CED kernels
(parity unpinned, no reference CED): discrete divergence of D and B preserved, a uniform
field in a uniform conductor decays exactly, and the exact plane wave is approached."""
import math

import numpy as np

from oracle import ced_oracle as co
from oracle.mhd_oracle import Geom
from paper_2211_13295_b200 import ced


def test_plane_wave_divergence_and_accuracy():
    for order in (2, 3):
        n = (8, 8, 8)
        g = ced.make_geometry(*n, order, (0, 0, 0), (1, 1, 1))
        G = Geom(*n, order, (0, 0, 0), (1, 1, 1))
        s = ced.plane_wave(g)
        sig = np.zeros(G.shape)
        par = co.Params(order)
        co.fill_ghosts(s, sig, G, par.bc)
        assert max(co.max_div(s, G)) < 1e-14
        e0 = co.energy(s, G, par)
        t, k = co.run_steps(s, sig, G, par, co.cfl_dt(G, par, 0.4), 6)
        assert max(co.max_div(s, G)) < 1e-13
        assert co.energy(s, G, par) <= e0 * (1 + 1e-12)  # upwind: energy never grows


def test_uniform_field_exact_decay():
    n, order = (6, 6, 6), 2
    g = ced.make_geometry(*n, order, (0, 0, 0), (1, 1, 1))
    G = Geom(*n, order, (0, 0, 0), (1, 1, 1))
    s = ced.uniform_field(g)
    par = co.Params(order)
    dt = co.cfl_dt(G, par, 0.4)
    sig = np.full(G.shape, 3.0 / dt)
    t, k = co.run_steps(s, sig, G, par, dt, 5)
    gh = G.gh
    assert np.allclose(s[0][gh:-gh - 1, gh:-gh - 1, gh:-gh - 1], math.exp(-3.0 * 5), rtol=1e-12)
