"""GPU tests of the CED extension (include/hydro_ced.h): Maxwell in a conducting medium with
CT, the 2D upwind edge solver and the exponential (L-stable) conduction step. PARITY
UNPINNED (no reference CED): (1) the sm_100a kernels against the builder-authored
numpy restatement oracle/ced_oracle.py -- bitwise where sigma = 0, within 1e-13 relative
where the conduction decay (exp/expm1, CUDA vs libm) enters; (2) self-consistency: exact
plane waves converge, div B and (uniform sigma) div D stay at round-off, a uniform field
decays exactly as exp(-sigma t/eps) for any sigma dt (no stiffness limit on dt), and a wave
entering a good conductor is absorbed without instability."""
import math

import numpy as np
import pytest

from oracle import ced_oracle as co
from oracle.mhd_oracle import Geom
from paper_2211_13295_b200 import ced

pytestmark = pytest.mark.gpu


def active(s, g):
    gh = g.ghost
    return s[:, gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("n,order,bc,sig", [
    ((10, 9, 8), 2, (0, 0, 0), 0.0),
    ((10, 9, 8), 3, (0, 0, 0), 0.0),
    ((9, 8, 10), 3, (1, 0, 1), 0.0),
    ((8, 10, 9), 3, (0, 0, 0), "random"),
    ((10, 8, 6), 2, (1, 1, 0), "random"),
])
def test_ced_vs_restatement(n, order, bc, sig):
    g = ced.make_geometry(*n, order, (0, 0, 0), (1, 1, 1))
    G = Geom(*n, order, (0, 0, 0), (1, 1, 1))
    s0 = ced.plane_wave(g)
    if sig == "random":
        sigma = np.random.default_rng(5).uniform(0.0, 50.0, G.shape)
    else:
        sigma = np.full(G.shape, sig)
    par = co.Params(order, bc=bc)
    st = ced.CedStepper(g, ced.make_params(order, bc=bc))
    st.upload(s0, sigma)
    dt = st.cfl_dt(0.4)
    assert dt == co.cfl_dt(G, par, 0.4)
    s_ref = s0.copy()
    sg = sigma.copy()
    co.fill_ghosts(s_ref, sg, G, bc)
    co.run_steps(s_ref, sg, G, par, dt, 4)
    st.set_time(0.0, dt)
    st.step(4)
    t, _, k = st.sync()
    out = st.download()
    a, b = active(out, g), active(s_ref, g)
    if sig == 0.0:
        assert (bits(a) == bits(b)).all(), np.abs(a - b).max()
    else:
        assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
    assert k == 4
    st.close()


def _wave_error(n, order, tf=0.25):
    g = ced.make_geometry(n, n, n, order, (0, 0, 0), (1, 1, 1))
    st = ced.CedStepper(g, ced.make_params(order))
    st.upload(ced.plane_wave(g), 0.0)
    t, steps = st.run(0.4, tf)
    err = np.abs(active(st.download(), g) - active(ced.plane_wave(g, t=t), g)).mean()
    divb, divd = st.max_div()
    st.close()
    return err, divb, divd, t


@pytest.mark.parametrize("order", [2, 3])
def test_ced_plane_wave_convergence_and_divergence(order):
    res = [_wave_error(n, order) for n in (16, 32, 64)]
    e = [r[0] for r in res]
    for err, divb, divd, t in res:
        assert abs(t - 0.25) < 1e-12
        assert divb < 1e-12 and divd < 1e-12
    assert np.log2(e[1] / e[2]) > 1.8, e


def test_ced_uniform_field_decays_exactly_for_any_sigma_dt():
    n, order = (8, 8, 8), 3
    g = ced.make_geometry(*n, order, (0, 0, 0), (1, 1, 1))
    st = ced.CedStepper(g, ced.make_params(order))
    d0 = (1.0, -0.5, 0.25)
    dt = st.cfl_dt(0.4)
    sigma = 5.0 / dt  # sigma dt = 5: an explicit source update would be unstable
    st.upload(ced.uniform_field(g, d0), sigma)
    st.set_time(0.0, dt)
    st.step(10)
    t, _, _ = st.sync()
    s = active(st.download(), g)
    for q in range(3):
        assert np.allclose(s[q], d0[q] * math.exp(-sigma * t), rtol=1e-12, atol=0)
    assert np.abs(s[3:]).max() == 0.0


def test_ced_wave_absorbed_by_conductor():
    """a plane wave along x meets a slab with sigma dt = 1e4: stable, energy never grows, the
    field inside the conductor is screened"""
    n, order = (64, 4, 4), 3
    g = ced.make_geometry(*n, order, (0, 0, 0), (1, 1.0 / 16, 1.0 / 16))
    st = ced.CedStepper(g, ced.make_params(order))
    s0 = ced.plane_wave(g, n=(1, 0, 0), pol=(0, 1, 0), L=(1, 1.0 / 16, 1.0 / 16))
    dt = st.cfl_dt(0.4)
    x = g.origin[0] + (np.arange(g.mx + 1) - g.ghost + 0.5) * g.dx
    sigma = np.zeros((g.mz + 1, g.my + 1, g.mx + 1))
    sigma[:, :, (x > 0.6) & (x < 0.8)] = 1e4 / dt
    st.upload(s0, sigma)
    st.set_time(0.0, dt)
    e0 = (active(s0, g) ** 2).sum()
    energies = []
    for _ in range(8):
        st.step(50)
        energies.append((active(st.download(), g) ** 2).sum())
    s = st.download()
    assert np.isfinite(s).all()
    assert all(b <= a * (1 + 1e-12) for a, b in zip([e0] + energies, energies))
    # inside a good conductor E (= D/eps) is screened; the wave is reflected at its surface
    xa = x[g.ghost:g.ghost + g.nx]
    inner = (xa > 0.65) & (xa < 0.75)
    d_in = np.abs(active(s, g)[:3][..., inner]).max()
    assert d_in < 1e-2 * np.abs(active(s0, g)[:3]).max(), d_in
    divb, _ = st.max_div()
    assert divb < 1e-12
    st.close()


@pytest.mark.parametrize("sigma", [1e3, 5e3, 1e5])
def test_ced_magnetic_diffusion_limit(sigma):
    """B_z = sin(2 pi x) in a good conductor (sigma dt = 2 .. 200): after the fast transient
    the slow mode decays at lambda = (-s + sqrt(s^2 - 4 c^2 k^2)) / 2 (~ -k^2 / (mu sigma)).
    The asymptotic-preserving edge dissipation keeps the rate within 1 % for any sigma h."""
    n = 64
    L = (1.0, 4.0 / n, 4.0 / n)
    g = ced.make_geometry(n, 4, 4, 2, (0, 0, 0), L)
    st = ced.CedStepper(g, ced.make_params(2))
    st.upload(ced.diffusion_mode(g), sigma)
    gh = g.ghost
    x = (np.arange(n) + 0.5) / n

    def amp():
        bz = st.download()[5][gh:gh + 4, gh:gh + 4, gh:gh + n].mean(axis=(0, 1))
        return 2 * (bz * np.sin(2 * math.pi * x)).mean()
    k = 2 * math.pi
    lam_th = (-sigma + math.sqrt(sigma * sigma - 4 * k * k)) / 2
    t1 = 0.2
    t2 = min(2.0, 0.5 / abs(lam_th))  # decay of at least ~40 %
    st.run(0.4, t1)
    a1 = amp()
    dt = st.cfl_dt(0.4)
    st.set_time(t1, dt, t2)
    while st.sync()[0] < t2 * (1 - 1e-12):
        st.step(256)
    a2 = amp()
    lam = math.log(a2 / a1) / (t2 - t1)
    assert abs(lam / lam_th - 1) < 0.01, (sigma, lam, lam_th)
    st.close()
