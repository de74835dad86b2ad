"""CPU checks of the MHD restatement (oracle/mhd_oracle.py) -- the checker the GPU kernels
are compared against bit for bit (tests/test_mhd_gpu.py). The reference has no MHD (parity
unpinned), so the restatement itself is held to the scheme's defining properties: the
discrete divergence of the face fields is preserved to round-off by the CT update,
fluid variables are conserved to round-off, the ADER predictor + CT converge on the smooth
MHD vortex, and the initial data are divergence-free."""
import numpy as np
import pytest

from oracle import mhd_oracle as mo
from paper_2211_13295_b200 import mhd


def active(s, G):
    gh = G.gh
    return s[:, gh:gh + G.n[2], gh:gh + G.n[1], gh:gh + G.n[0]]


@pytest.mark.parametrize("order,bc", [(2, (0, 0, 0)), (3, (0, 0, 0)), (3, (1, 0, 1))])
def test_divb_and_conservation(order, bc):
    n = (8, 9, 10)
    g = mhd.make_geometry(*n, order, (0, 0, 0), (1, 1, 1))
    s = mhd.random_field(g, order)
    G = mo.Geom(*n, order, (0, 0, 0), (1, 1, 1))
    par = mo.Params(order, bc=bc)
    mo.fill_ghosts(s, G, bc)
    bmax = np.abs(active(s, G)[5:]).max()
    assert mo.max_divb(s, G) < 1e-14 * bmax
    tot0 = active(s, G)[:5].sum(axis=(1, 2, 3))
    dt0 = mo.cfl_dt(s, G, par, 0.4)
    mo.run_steps(s, G, par, 0.4, 4, dt0)
    assert mo.max_divb(s, G) < 1e-13 * bmax
    if bc == (0, 0, 0):  # periodic: every conserved total is invariant
        tot1 = active(s, G)[:5].sum(axis=(1, 2, 3))
        assert np.allclose(tot0, tot1, rtol=0, atol=1e-12 * np.abs(tot0).max())


def test_constant_state_is_fixed_point():
    n, order = (6, 6, 6), 3
    G = mo.Geom(*n, order)
    s = np.zeros((8,) + G.shape)
    s[0], s[1], s[2], s[3] = 1.3, 0.2, -0.1, 0.05
    s[5], s[6], s[7] = 0.3, -0.2, 0.1
    s[4] = 2.0 / (5.0 / 3.0 - 1.0) + 0.5 * (0.2 ** 2 + 0.1 ** 2 + 0.05 ** 2) / 1.3 + \
        0.5 * (0.3 ** 2 + 0.2 ** 2 + 0.1 ** 2)
    s0 = s.copy()
    par = mo.Params(order)
    dt0 = mo.cfl_dt(s, G, par, 0.4)
    mo.run_steps(s, G, par, 0.4, 2, dt0)
    assert np.allclose(active(s, G), active(s0, G), rtol=1e-14, atol=1e-15)


def test_vortex_convergence_o2():
    errs = []
    for n in (16, 32):
        g = mhd.make_geometry(n, n, 4, 2, (-5, -5, -5), (5, 5, 5))
        s = mhd.mhd_vortex(g, 2)
        G = mo.Geom(n, n, 4, 2, (-5, -5, -5), (5, 5, 5))
        par = mo.Params(2)
        dt0 = mo.cfl_dt(s, G, par, 0.4)
        dts, dt, t = mo.run_steps(s, G, par, 0.4, 10000, min(dt0, 0.5), t_final=0.5)
        ex = mhd.mhd_vortex(g, 2, t=t)
        errs.append(np.abs(active(s, G)[5] - active(ex, G)[5]).mean())
    assert np.log2(errs[0] / errs[1]) > 1.5, errs


def test_initial_data_divergence_free():
    for order in (2, 3):
        g = mhd.make_geometry(16, 12, 4, order, (0, 0, 0), (1, 1, 1))
        s = mhd.orszag_tang(g, order)
        G = mo.Geom(16, 12, 4, order, (0, 0, 0), (1, 1, 1))
        assert mo.max_divb(s, G) < 1e-15
