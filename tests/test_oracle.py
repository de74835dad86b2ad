"""The C restatement (oracle/) pinned against the reference library built from its own
sources (oracle/_ref) -- bit for bit -- and against the committed golden vectors.
CPU only."""
import numpy as np
import pytest

from oracle import pyoracle as po

ref_required = pytest.mark.skipif(not po.have_reference(),
                                  reason="oracle/_ref not built (no /root/reference here)")


@pytest.fixture(scope="module")
def orc():
    return po.Oracle()


@pytest.fixture(scope="module")
def ref():
    r = po.Reference()
    r.set_threads(4)
    return r


def rng_states(seed, n):
    """test_support.hpp:12-18 random_cons distribution (numpy RNG, not mt19937)."""
    r = np.random.default_rng(seed)
    rho = r.uniform(0.1, 5.0, n)
    v = r.uniform(-2, 2, (n, 3))
    p = r.uniform(0.05, 5.0, n)
    u = np.empty((n, 5))
    u[:, 0] = rho
    u[:, 1:4] = rho[:, None] * v
    u[:, 4] = p / 0.4 + 0.5 * rho * (v * v).sum(1)
    return u


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@ref_required
def test_pointwise_bitwise(orc, ref):
    u = rng_states(97, 600)
    for a in range(0, 600, 2):
        for axis in range(3):
            for fn in ("hll_flux", "rusanov_flux"):
                x = getattr(orc, fn)(u[a], u[a + 1], axis)
                y = getattr(ref, fn)(u[a], u[a + 1], axis)
                assert (bits(x) == bits(y)).all()
        d1 = orc.eval_tstep_ptwise(u[a], 0.6, 0.1, 0.2, 0.3)
        d2 = ref.eval_tstep_ptwise(u[a], 0.6, 0.1, 0.2, 0.3)
        assert d1 == d2
    r = np.random.default_rng(11)
    for _ in range(2000):
        a, b, c = r.uniform(-3, 3), r.uniform(-3, 3), r.choice([1.0, 1.5, 2.0])
        assert bits(np.array(orc.mc_limiter(a, b, c))) == bits(np.array(ref.mc_limiter(a, b, c)))
        s = r.uniform(0, 2, 5)
        assert orc.weno3_point(s) == ref.weno3_point(s)
    for modes in (5, 11):
        for _ in range(200):
            z = np.zeros(5 * modes)
            base = rng_states(int(r.integers(1 << 30)), 1)[0]
            for q in range(5):
                z[q * modes] = base[q]
                for m in range(1, modes - 1):
                    z[q * modes + m] = r.uniform(-0.05, 0.05) * abs(base[q])
            res = []
            for lib in (orc, ref):
                try:
                    res.append(lib.predictor_ptwise(z, modes, 0.01, 0.1, 0.2, 0.15))
                except po.UnphysicalError as e:
                    res.append(str(e))
            if isinstance(res[0], str):
                assert res[0] == res[1]
            else:
                assert (bits(res[0]) == bits(res[1])).all()


@ref_required
@pytest.mark.parametrize("order", [2, 3])
def test_patch_kernels_bitwise(orc, ref, order):
    """test_parallel_serial.cpp:37-88, restatement vs reference, every kernel."""
    g = po.make_geometry(10, 9, 8, order)
    M = po.modes_for_order(order)
    s = orc.init_isentropic_vortex(g, order)
    s2 = ref.init_isentropic_vortex(g, order)
    assert (bits(s) == bits(s2)).all()
    orc.apply_boundary_skinny(g, po.PERIODIC, s)
    ref.apply_boundary_skinny(g, po.PERIODIC, s2)
    assert (bits(s) == bits(s2)).all()
    m1, m2 = po.zeros_modal(g, order), po.zeros_modal(g, order)
    orc.skinny_to_modal(g, M, s, m1)
    ref.skinny_to_modal(g, M, s2, m2)
    assert (bits(m1) == bits(m2)).all()
    if order == 2:
        orc.limit_patch_o2(g, m1)
        ref.limit_patch_o2(g, m2)
    else:
        orc.reconstruct_patch_o3(g, m1)
        ref.reconstruct_patch_o3(g, m2)
    assert (bits(m1) == bits(m2)).all()
    orc.predict_patch(g, M, m1, 0.004)
    ref.predict_patch(g, M, m2, 0.004)
    assert (bits(m1) == bits(m2)).all()
    for solver in (po.RUSANOV, po.HLL):
        f1, f2 = po.zeros_faces(g), po.zeros_faces(g)
        for ax in range(3):
            orc.make_flux_axis(g, M, m1, ax, solver, f1[ax])
            ref.make_flux_axis(g, M, m2, ax, solver, f2[ax])
            assert (bits(f1[ax]) == bits(f2[ax])).all()
    r1, r2 = po.zeros_rate(g), po.zeros_rate(g)
    orc.make_du_dt(g, *f1, 0.004, r1)
    ref.make_du_dt(g, *f2, 0.004, r2)
    assert (bits(r1) == bits(r2)).all()
    d1 = orc.update_u_timestep(g, M, m1, s, r1, 0.5)
    d2 = ref.update_u_timestep(g, M, m2, s2, r2, 0.5)
    assert (bits(m1) == bits(m2)).all() and (bits(s) == bits(s2)).all() and d1 == d2
    assert orc.compute_dt_next(g, M, m1, 0.5) == ref.compute_dt_next(g, M, m2, 0.5)


@ref_required
@pytest.mark.parametrize("order,solver,bc", [(2, po.HLL, po.PERIODIC), (3, po.HLL, po.PERIODIC),
                                             (2, po.RUSANOV, po.OUTFLOW),
                                             (3, po.RUSANOV, po.PERIODIC)])
def test_ader_steps_bitwise(orc, ref, order, solver, bc):
    g = po.make_geometry(8, 8, 8, order)
    par = po.make_params(order, solver)
    M = po.modes_for_order(order)
    s1 = orc.init_isentropic_vortex(g, order)
    s2 = s1.copy()
    cfl = 0.6 if order == 2 else 0.4
    dt1 = dt2 = orc.initial_dt(g, s1, cfl)
    a = (po.zeros_modal(g, order), *po.zeros_faces(g), po.zeros_rate(g))
    b = (po.zeros_modal(g, order), *po.zeros_faces(g), po.zeros_rate(g))
    for _ in range(4):
        orc.apply_boundary_skinny(g, bc, s1)
        ref.apply_boundary_skinny(g, bc, s2)
        dt1 = orc.ader_step(g, par, a[0], s1, a[1], a[2], a[3], a[4], dt1, cfl)
        dt2 = ref.ader_step(g, par, b[0], s2, b[1], b[2], b[3], b[4], dt2, cfl)
        for x, y in zip(a, b):
            assert (bits(x) == bits(y)).all()
        assert (bits(s1) == bits(s2)).all() and dt1 == dt2
    assert M in (5, 11)


@ref_required
@pytest.mark.parametrize("order,nst", [(2, 2), (3, 3)])
def test_rk_step_bitwise(orc, ref, order, nst):
    g = po.make_geometry(8, 6, 7, order)
    par = po.make_params(order)
    s1 = orc.init_isentropic_vortex(g, order)
    s2 = s1.copy()
    a = [po.zeros_modal(g, order), *po.zeros_faces(g), po.zeros_rate(g), po.zeros_skinny(g)]
    b = [x.copy() for x in a]
    d1 = orc.rk_step(g, par, nst, *a[:1], s1, *a[1:], po.PERIODIC, 0.01, 0.5)
    d2 = ref.rk_step(g, par, nst, *b[:1], s2, *b[1:], po.PERIODIC, 0.01, 0.5)
    assert d1 == d2 and (bits(s1) == bits(s2)).all()
    for x, y in zip(a, b):
        assert (bits(x) == bits(y)).all()


@ref_required
def test_error_messages_match(orc, ref):
    """test_corrector.cpp:217-232: the zone id in the update error text."""
    g = po.make_geometry(4, 4, 4, 2, (0, 0, 0), (1, 1, 1))
    for lib in (orc, ref):
        m = po.zeros_modal(g, 2)
        m[..., 0, 0] = 1.0
        m[..., 4, 0] = 2.5
        s = po.zeros_skinny(g)
        r = po.zeros_rate(g)
        r[1, 2, 3, 0] = -5.0
        with pytest.raises(po.UnphysicalError) as ei:
            lib.update_u_timestep(g, 5, m, s, r, 0.6)
        assert "(3,2,1)" in str(ei.value)
    assert orc.error() == ref.error()


def test_golden_vectors(orc):
    """The restatement against the reference-produced fixtures (tests/golden/)."""
    from tests.golden import golden
    cases = golden.load_all()
    assert cases, "no golden fixtures committed"
    for name, case in cases.items():
        out = golden.run_case(orc, case["meta"])
        for key, want in case["digests"].items():
            assert golden.digest(out[key]) == want, (name, key)
        for key, want in case["arrays"].items():
            got = out[key]
            assert got.shape == want.shape, (name, key)
            assert (bits(got) == bits(want)).all(), (name, key)
