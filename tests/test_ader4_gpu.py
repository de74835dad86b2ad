"""The formally fourth-order ADER step (csrc/ader4.cu, hc_ader4_*; EXTENSION -- parity
unpinned, there is no fourth-order reference code): its convergence order on the smooth
isentropic vortex against the exact solution (PAPER.md:1514-1525 reports 4.04-4.22 for the
authors' O4 CFD code), beside the reference's own ADER structure at O3 and with the WENO-AO
reconstruction, which both stay near second order asymptotically; conservation to round-off;
a uniform state as an exact fixed point; a shock tube with outflow boundaries."""
import numpy as np
import pytest

from paper_2211_13295_b200 import hydro

pytestmark = pytest.mark.gpu


def _run(scheme, n, t_final=1.0, cfl=0.4, solver=hydro.HLL):
    api = hydro.HostApi()
    order = 4 if scheme == "weno_ao" else 3
    g = hydro.make_geometry(n, n, 4, order, lo=(-5, -5, -5 * 4 / n), hi=(5, 5, 5 * 4 / n))
    s0 = api.init_isentropic_vortex(g, order)
    dt0 = api.initial_dt(g, s0, cfl)
    if scheme == "ader4":
        st = hydro.Ader4Stepper(g, hydro.make_params(3, solver))
    else:
        st = hydro.Stepper(g, hydro.make_params(order, solver), exact=False)
    st.upload(s0)
    st.set_time(0.0, dt0, cfl, t_final)
    done = -1
    while True:
        st.step(64)
        t, _, n_done = st.sync()
        if n_done == done:
            break
        done = n_done
    out = st.download()
    st.close()
    ex = api.init_isentropic_vortex(g, order, t=t)
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    return out, ex, g, t, np.abs(out[act][..., 0] - ex[act][..., 0]).mean()


def test_ader4_converges_at_fourth_order():
    e = [_run("ader4", n)[4] for n in (32, 64, 128)]
    orders = [np.log2(e[i] / e[i + 1]) for i in range(2)]
    assert all(o >= 3.7 for o in orders), (e, orders)  # measured 4.31, 4.48
    # the reference's ADER structure at O3 and with WENO-AO: no better than ~2.5 at 64 -> 128
    for scheme in ("o3", "weno_ao"):
        f = [_run(scheme, n)[4] for n in (64, 128)]
        assert np.log2(f[0] / f[1]) < 2.6, (scheme, f)
        assert e[2] < f[1] / 10.0


@pytest.mark.parametrize("solver", [hydro.RUSANOV, hydro.HLL])
def test_ader4_conserves_and_reaches_t_final(solver):
    api = hydro.HostApi()
    out, ex, g, t, _ = _run("ader4", 32, t_final=0.5, solver=solver)
    assert t == pytest.approx(0.5, rel=1e-12)
    gh = g.ghost
    s0 = api.init_isentropic_vortex(g, 3)
    a = out[gh:-gh, gh:-gh, gh:-gh].reshape(-1, 5).sum(0)
    b = s0[gh:-gh, gh:-gh, gh:-gh].reshape(-1, 5).sum(0)
    scale = np.abs(s0[gh:-gh, gh:-gh, gh:-gh]).reshape(-1, 5).sum(0)
    scale = np.maximum(scale, 1e-3 * scale.max())  # (w-momentum is identically zero)
    assert (np.abs(a - b) <= 1e-12 * scale).all(), (a - b) / scale


def test_ader4_uniform_state_is_a_fixed_point():
    api = hydro.HostApi()
    g = hydro.make_geometry(16, 12, 8, 3)
    s0 = api.init_constant(g)
    st = hydro.Ader4Stepper(g, hydro.make_params(3))
    st.upload(s0)
    st.set_time(0.0, api.initial_dt(g, s0, 0.4), 0.4)
    st.step(5)
    st.sync()
    out = st.download()
    st.close()
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    np.testing.assert_allclose(out[act], s0[act], rtol=1e-13, atol=1e-13)


def test_ader4_shock_tube_outflow_stays_physical():
    """Sod with outflow boundaries: the unlimited cross terms and the high-order predictor stay
    physical on the 1D shock tube (the mixed terms vanish for x-only data)."""
    api = hydro.HostApi()
    g = hydro.make_geometry(64, 4, 4, 3, lo=(0, 0, 0), hi=(1, 1.0 / 16, 1.0 / 16))
    s0 = api.init_sod(g)
    st = hydro.Ader4Stepper(g, hydro.make_params(3, hydro.HLL), boundary=hydro.OUTFLOW)
    st.upload(s0)
    st.set_time(0.0, api.initial_dt(g, s0, 0.4), 0.4, 0.1)
    st.step(400)
    t, _, n = st.sync()
    out = st.download()
    st.close()
    gh = g.ghost
    rho = out[gh:-gh, gh:-gh, gh:-gh, 0]
    assert t == pytest.approx(0.1) and n > 10
    assert (rho > 0.1).all() and (rho < 1.01).all()
