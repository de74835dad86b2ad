"""HLLC and HLLI (extensions; the reference has neither, SPEC.md:339 -- parity unpinned). The oracle's
restatement (oracle/hydro_oracle.c or_hllc_flux) is checked here against the properties that
define HLLC (Toro 2009, sec. 10.4), so the GPU kernels' bitwise match to it (test_gpu_parity)
means something: consistency, exact resolution of isolated contacts and shear waves (which
HLL smears), upwinding of supersonic states, mirror symmetry."""
import numpy as np
import pytest

from oracle import pyoracle as po


@pytest.fixture(scope="module")
def orc():
    return po.Oracle()


def cons(rho, u, v, w, p, gamma=1.4):
    return np.array([rho, rho * u, rho * v, rho * w, p / (gamma - 1) + 0.5 * rho * (u * u + v * v + w * w)])


def states(seed, n):
    r = np.random.default_rng(seed)
    return [cons(r.uniform(0.1, 4), *r.uniform(-2, 2, 3), r.uniform(0.1, 4)) for _ in range(n)]


def test_consistency(orc):
    for u in states(5, 200):
        for axis in range(3):
            f = orc.hllc_flux(u, u, axis)
            fe = orc.hll_flux(u, u, axis)  # = the physical flux for equal states
            assert np.allclose(f, fe, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_stationary_contact_exact(orc, axis):
    # density jump, zero normal velocity, equal pressure: only the pressure term survives
    vel = [0.0, 0.0, 0.0]
    vel[(axis + 1) % 3] = 0.7  # shear: a tangential velocity jump is held too
    ul = cons(1.0, *vel, 1.0)
    vel[(axis + 1) % 3] = -0.3
    ur = cons(0.125, *vel, 1.0)
    f = orc.hllc_flux(ul, ur, axis)
    expect = np.zeros(5)
    expect[1 + axis] = 1.0
    assert np.array_equal(f, expect) or np.allclose(f, expect, rtol=0, atol=1e-15)
    h = orc.hll_flux(ul, ur, axis)
    assert abs(h[0]) > 1e-3  # HLL diffuses the contact


def test_moving_contact_upwind(orc):
    ul = cons(1.0, 0.5, 0.2, -0.1, 1.0)
    ur = cons(0.3, 0.5, -0.4, 0.3, 1.0)
    f = orc.hllc_flux(ul, ur, 0)
    fl = orc.hll_flux(ul, ul, 0)  # exact flux of the upwind (left) state
    assert np.allclose(f, fl, rtol=1e-13, atol=1e-14)


def test_supersonic_upwind(orc):
    ul = cons(1.0, 4.0, 0.1, 0.0, 1.0)
    ur = cons(0.5, 3.5, 0.0, 0.2, 0.8)
    assert np.array_equal(orc.hllc_flux(ul, ur, 0), orc.hll_flux(ul, ul, 0))
    ul = cons(1.0, -4.0, 0.1, 0.0, 1.0)
    ur = cons(0.5, -3.5, 0.0, 0.2, 0.8)
    assert np.array_equal(orc.hllc_flux(ul, ur, 0), orc.hll_flux(ur, ur, 0))


def test_mirror_symmetry(orc):
    s = states(7, 100)
    for a in range(0, 100, 2):
        ul, ur = s[a], s[a + 1]
        f = orc.hllc_flux(ul, ur, 0)
        m = np.array([1, -1, 1, 1, 1.0])
        g = orc.hllc_flux(ur * m, ul * m, 0)
        assert np.allclose(f * -m, g, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------------------ HLLI

def test_hlli_consistency_and_upwinding(orc):
    for u in states(9, 100):
        for axis in range(3):
            assert np.allclose(orc.hlli_flux(u, u, axis), orc.hll_flux(u, u, axis), rtol=1e-13,
                               atol=1e-13)
    ul = cons(1.0, 4.0, 0.1, 0.0, 1.0)
    ur = cons(0.5, 3.5, 0.0, 0.2, 0.8)
    assert np.array_equal(orc.hlli_flux(ul, ur, 0), orc.hll_flux(ul, ul, 0))


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_hlli_stationary_contact_and_shear_exact(orc, axis):
    """a stationary contact (density jump at rest) and a stationary shear layer (tangential
    velocity jump at constant density) are each a single linearly degenerate wave at the
    average state, so HLLI removes all of HLL's dissipation on them"""
    expect = np.zeros(5)
    expect[1 + axis] = 1.0
    f = orc.hlli_flux(cons(1.0, 0, 0, 0, 1.0), cons(0.125, 0, 0, 0, 1.0), axis)
    assert np.allclose(f, expect, rtol=0, atol=1e-14), f
    vl, vr = [0.0] * 3, [0.0] * 3
    vl[(axis + 1) % 3], vr[(axis + 1) % 3] = 0.7, -0.3
    vl[(axis + 2) % 3], vr[(axis + 2) % 3] = -0.2, 0.4
    f = orc.hlli_flux(cons(0.8, *vl, 1.0), cons(0.8, *vr, 1.0), axis)
    assert np.allclose(f, expect, rtol=0, atol=1e-14), f
    assert abs(orc.hll_flux(cons(0.8, *vl, 1.0), cons(0.8, *vr, 1.0), axis)[1 + (axis + 1) % 3]) > 1e-3


def test_hlli_moving_contact_upwind(orc):
    ul = cons(1.0, 0.5, 0.2, -0.1, 1.0)
    ur = cons(0.3, 0.5, 0.2, -0.1, 1.0)  # pure entropy wave moving right
    assert np.allclose(orc.hlli_flux(ul, ur, 0), orc.hll_flux(ul, ul, 0), rtol=1e-13, atol=1e-14)


def test_hlli_mirror_symmetry(orc):
    s = states(17, 100)
    m = np.array([1, -1, 1, 1, 1.0])
    for a in range(0, 100, 2):
        f = orc.hlli_flux(s[a], s[a + 1], 0)
        g = orc.hlli_flux(s[a + 1] * m, s[a] * m, 0)
        assert np.allclose(f * -m, g, rtol=1e-12, atol=1e-12)
