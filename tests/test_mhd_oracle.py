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


# ------------------------------------------------------------------- HLLD face solver

def _cons(rho, v, p, b, gamma=5.0 / 3.0):
    """conserved 8-vectors of arrays from primitives (rho, v[3], p, B[3])"""
    rho = np.asarray(rho, float)
    v = [np.broadcast_to(np.asarray(x, float), rho.shape) for x in v]
    b = [np.broadcast_to(np.asarray(x, float), rho.shape) for x in b]
    p = np.broadcast_to(np.asarray(p, float), rho.shape)
    e = p / (gamma - 1.0) + 0.5 * rho * (v[0] ** 2 + v[1] ** 2 + v[2] ** 2) + \
        0.5 * (b[0] ** 2 + b[1] ** 2 + b[2] ** 2)
    return [rho, rho * v[0], rho * v[1], rho * v[2], e, b[0], b[1], b[2]]


def _hlld(ul, ur, A, gamma=5.0 / 3.0):
    ql, qr = mo.prim(ul, gamma), mo.prim(ur, gamma)
    cl, cr = mo.fast_speed(ul, ql, gamma, A), mo.fast_speed(ur, qr, gamma, A)
    return mo.hlld(ul, ur, ql, qr, cl, cr, A)


def _random_states(rng, n, A):
    rho = rng.uniform(0.2, 3.0, n)
    v = [rng.uniform(-2, 2, n) for _ in range(3)]
    p = rng.uniform(0.1, 3.0, n)
    b = [rng.uniform(-2, 2, n) for _ in range(3)]
    return rho, v, p, b


@pytest.mark.parametrize("A", [0, 1, 2])
def test_hlld_consistency(A):
    """F(U, U) = F(U): every wave speed collapses onto the state, U* = U** = U"""
    rng = np.random.default_rng(11 + A)
    u = _cons(*_random_states(rng, 400, A))
    f = _hlld(u, u, A)
    fx = mo.mhd_flux(u, mo.prim(u, 5.0 / 3.0), A)
    for q in range(5):
        assert np.allclose(f[q], fx[q], rtol=1e-12, atol=1e-12), q


@pytest.mark.parametrize("A", [0, 1, 2])
def test_hlld_resolves_stationary_contact_and_tangential(A):
    """isolated stationary contact (density jump, B_n != 0) and tangential discontinuity
    (B_n = 0; density, tangential v and B jump at constant total pressure): HLLD's flux is
    the exact one -- no mass or energy flux, momentum flux = total pressure - B_n B -- where
    HLL diffuses the jump"""
    rng = np.random.default_rng(3 + A)
    n = 200
    T1, T2 = (A + 1) % 3, (A + 2) % 3
    # contact
    v = [np.zeros(n)] * 3
    vt = [np.zeros(n), np.zeros(n), np.zeros(n)]
    vt[T1] = rng.uniform(-1, 1, n)
    vt[T2] = rng.uniform(-1, 1, n)
    b = [rng.uniform(-1, 1, n) for _ in range(3)]
    p = rng.uniform(0.2, 2.0, n)
    ul = _cons(rng.uniform(0.2, 3.0, n), vt, p, b)
    ur = _cons(rng.uniform(0.2, 3.0, n), vt, p, b)
    f = _hlld(ul, ur, A)
    assert np.abs(f[0]).max() < 1e-13
    assert np.abs(f[4] - (-b[A] * (vt[T1] * b[T1] + vt[T2] * b[T2]))).max() < 1e-12
    pt = p + 0.5 * (b[0] ** 2 + b[1] ** 2 + b[2] ** 2)
    assert np.abs(f[1 + A] - (pt - b[A] * b[A])).max() < 1e-12
    # HLL smears the same contact
    ql, qr = mo.prim(ul, 5.0 / 3.0), mo.prim(ur, 5.0 / 3.0)
    cl, cr = mo.fast_speed(ul, ql, 5.0 / 3.0, A), mo.fast_speed(ur, qr, 5.0 / 3.0, A)
    sl, sr = np.minimum(-cl, -cr), np.maximum(cl, cr)
    hll_mass = sl * sr * (ur[0] - ul[0]) / (sr - sl)
    assert np.abs(hll_mass).max() > 0.1
    # tangential discontinuity
    b = [rng.uniform(-1, 1, n) for _ in range(3)]
    b[A] = np.zeros(n)
    br = [rng.uniform(-1, 1, n) for _ in range(3)]
    br[A] = np.zeros(n)
    vr = [rng.uniform(-1, 1, n) for _ in range(3)]
    vr[A] = np.zeros(n)
    pl = rng.uniform(1.0, 2.0, n)
    ptl = pl + 0.5 * (b[0] ** 2 + b[1] ** 2 + b[2] ** 2)
    pr_ = ptl - 0.5 * (br[0] ** 2 + br[1] ** 2 + br[2] ** 2)
    keep = pr_ > 0.05
    ul = _cons(rng.uniform(0.2, 3.0, n), vt, pl, b)
    ur = _cons(rng.uniform(0.2, 3.0, n), vr, pr_, br)
    ul = [x[keep] for x in ul]
    ur = [x[keep] for x in ur]
    f = _hlld(ul, ur, A)
    assert np.abs(f[0]).max() < 1e-13 and np.abs(f[4]).max() < 1e-12
    assert np.abs(f[1 + A] - ptl[keep]).max() < 1e-12
    for T in (T1, T2):
        assert np.abs(f[1 + T]).max() < 1e-13


def test_hlld_mirror_symmetry():
    """x -> -x (u_x, B_x change sign, left and right swap): F_rho, F_my, F_mz, F_E change
    sign and F_mx is unchanged"""
    rng = np.random.default_rng(5)
    n = 400
    rl, vl, pl, bl = _random_states(rng, n, 0)
    rr, vr, pr_, br = _random_states(rng, n, 0)
    br[0] = bl[0]  # single-valued normal field
    ul, ur = _cons(rl, vl, pl, bl), _cons(rr, vr, pr_, br)

    def mirror(rho, v, p, b):
        return _cons(rho, [-v[0], v[1], v[2]], p, [-b[0], b[1], b[2]])
    f = _hlld(ul, ur, 0)
    g = _hlld(mirror(rr, vr, pr_, br), mirror(rl, vl, pl, bl), 0)
    sign = [-1, 1, -1, -1, -1]
    for q in range(5):
        assert np.allclose(g[q], sign[q] * f[q], rtol=1e-10, atol=1e-12), q
