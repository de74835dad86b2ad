"""Ideal MHD at order 4 (csrc/mhd.cu k_mhd4_*; EXTENSION, parity unpinned): the local space-
time predictor and Gauss-point quadrature in time and along faces / edges, constrained
transport unchanged. On the smooth Balsara (2004) MHD vortex its convergence order (PAPER.md
:1562-1580 reports O4 runs of the authors' MHD code) against the O3 path (the reference's ADER
structure), div B at round-off, conservation."""
import numpy as np
import pytest

from paper_2211_13295_b200 import mhd

pytestmark = pytest.mark.gpu


def active(s, g):
    gh = g.ghost
    return s[:, gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]


def _vortex(n, order, t_final=1.0, solver=mhd.HLL):
    g = mhd.make_geometry(n, n, 4, order, (-5, -5, -5 * 4 / n), (5, 5, 5 * 4 / n))
    s0 = mhd.mhd_vortex(g, order)
    st = mhd.MhdStepper(g, mhd.make_params(order, face_solver=solver))
    st.upload(s0)
    t, dt, done = st.run(0.4, t_final=t_final)
    s = st.download()
    divb = st.max_divb()
    st.close()
    ex = mhd.mhd_vortex(g, order, t=t)
    a, b = active(s, g), active(ex, g)
    return (np.abs(a[0] - b[0]).mean(), np.abs(a[5] - b[5]).mean(), t, divb, s0, s, g)


@pytest.mark.parametrize("solver", [mhd.HLL, mhd.HLLD])
def test_mhd4_vortex_fourth_order(solver):
    res = [_vortex(n, 4, solver=solver) for n in (32, 64, 128)]
    rho = [r[0] for r in res]
    bx = [r[1] for r in res]
    for r in res:
        assert abs(r[2] - 1.0) < 1e-12 and r[3] < 1e-12
    o_rho = [np.log2(rho[i] / rho[i + 1]) for i in range(2)]
    o_b = [np.log2(bx[i] / bx[i + 1]) for i in range(2)]
    assert min(o_rho[1], o_b[1]) >= 3.5, (rho, bx, o_rho, o_b)
    r3 = _vortex(128, 3)
    assert rho[2] < r3[0] / 5.0 and bx[2] < r3[1] / 5.0, (rho[2], r3[0], bx[2], r3[1])


def test_mhd4_conserves():
    e_rho, e_b, t, divb, s0, s, g = _vortex(32, 4, t_final=0.5)
    a = active(s, g)[:5].reshape(5, -1).sum(1)
    b = active(s0, g)[:5].reshape(5, -1).sum(1)
    scale = np.abs(active(s0, g)[:5]).reshape(5, -1).sum(1)
    scale = np.maximum(scale, 1e-3 * scale.max())
    assert (np.abs(a - b) <= 1e-12 * scale).all(), (a - b) / scale
    assert divb < 1e-12
