"""GPU parity: the sm_100a kernels against the C restatement (oracle/) and the golden vectors
the reference produced. Bit-exact for the exact build; the FMA build within a stated
tolerance. Mirrors proj/tests/test_parallel_serial.cpp and test_corrector.cpp."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2211_13295_b200 import hydro
from tests.golden import golden

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def same(a, b):
    return a.shape == b.shape and bool((bits(a) == bits(b)).all())


@pytest.fixture(scope="module")
def api():
    assert hydro.device_count() > 0, "GPU tests need a CUDA device"
    return hydro.HostApi()


@pytest.fixture(scope="module")
def orc():
    return po.Oracle()


def geoms(n, order, lo=(-5, -5, -5), hi=(5, 5, 5)):
    return hydro.make_geometry(*n, order, lo, hi), po.make_geometry(*n, order, lo, hi)


@pytest.mark.parametrize("order", [2, 3])
def test_every_kernel_bitwise(api, orc, order):
    """test_parallel_serial.cpp:37-88 with the GPU kernels in place of the OpenMP ones."""
    g, go = geoms((10, 9, 8), order)
    M = hydro.modes_for_order(order)
    s = orc.init_isentropic_vortex(go, order)
    orc.apply_boundary_skinny(go, po.PERIODIC, s)
    s_gpu = s.copy()
    api.apply_boundary_skinny(g, hydro.PERIODIC, s_gpu)
    assert same(s, s_gpu)
    mg, mo = hydro.zeros_modal(g, order), po.zeros_modal(go, order)
    api.skinny_to_modal(g, M, s_gpu, mg)
    orc.skinny_to_modal(go, M, s, mo)
    assert same(mg, mo)
    if order == 2:
        api.limit_patch_o2(g, mg)
        orc.limit_patch_o2(go, mo)
    else:
        api.reconstruct_patch_o3(g, mg)
        orc.reconstruct_patch_o3(go, mo)
    assert same(mg, mo)
    api.predict_patch(g, M, mg, 0.004)
    orc.predict_patch(go, M, mo, 0.004)
    assert same(mg, mo)
    for solver in (hydro.RUSANOV, hydro.HLL, hydro.HLLC, hydro.HLLI):
        fg, fo = hydro.zeros_faces(g), po.zeros_faces(go)
        for ax in range(3):
            api.make_flux_axis(g, M, mg, ax, solver, fg[ax])
            orc.make_flux_axis(go, M, mo, ax, solver, fo[ax])
            assert same(fg[ax], fo[ax]), (solver, ax)
    rg, ro = hydro.zeros_rate(g), po.zeros_rate(go)
    api.make_du_dt(g, *fg, 0.004, rg)
    orc.make_du_dt(go, *fo, 0.004, ro)
    assert same(rg, ro)
    d1 = api.update_u_timestep(g, M, mg, s_gpu, rg, 0.5)
    d2 = orc.update_u_timestep(go, M, mo, s, ro, 0.5)
    assert same(mg, mo) and same(s_gpu, s) and d1 == d2
    assert api.compute_dt_next(g, M, mg, 0.5) == orc.compute_dt_next(go, M, mo, 0.5)
    # boundary fill of mode 0 in the modal state, zero_temporal_mode, modal_to_skinny
    api.apply_boundary_modal(g, M, hydro.OUTFLOW, mg)
    orc.apply_boundary_modal(go, M, po.OUTFLOW, mo)
    assert same(mg, mo)
    api.zero_temporal_mode(g, M, mg)
    orc.zero_temporal_mode(go, M, mo)
    assert same(mg, mo)
    s2, s3 = np.zeros_like(s), np.zeros_like(s)
    api.modal_to_skinny(g, M, mg, s2)
    orc.modal_to_skinny(go, M, mo, s3)
    assert same(s2, s3)


@pytest.mark.parametrize("name", sorted(golden.CASES))
def test_golden_cases_host_api(api, name):
    """Whole ADER / RK steps through the host-buffer C ABI vs the reference's digests."""
    cases = golden.load_all()
    case = cases[name]
    out = golden.run_case(api, case["meta"])
    for key, want in case["digests"].items():
        assert golden.digest(out[key]) == want, (name, key)


def test_unphysical_errors_carry_the_reference_text(api, orc):
    """test_corrector.cpp:217-232 and test_predictor.cpp:281-293."""
    g, go = geoms((4, 4, 4), 2, (0, 0, 0), (1, 1, 1))
    m = hydro.zeros_modal(g, 2)
    m[..., 0, 0] = 1.0
    m[..., 4, 0] = 2.5
    s = hydro.zeros_skinny(g)
    r = hydro.zeros_rate(g)
    r[1, 2, 3, 0] = -5.0
    with pytest.raises(hydro.UnphysicalError) as e1:
        api.update_u_timestep(g, 5, m.copy(), s.copy(), r, 0.6)
    with pytest.raises(po.UnphysicalError) as e2:
        orc.update_u_timestep(go, 5, m.copy(), s.copy(), r, 0.6)
    assert str(e1.value) == str(e2.value)
    assert "update: zone (3,2,1): non-positive density" in str(e1.value)
    # a zone whose face extrapolation has negative pressure fails in the predictor
    m2 = m.copy()
    gh = g.ghost
    m2[gh + 1, gh + 2, gh + 3, 4, 0] = 0.05
    m2[gh + 1, gh + 2, gh + 3, 4, 1] = 1.0  # energy slope
    with pytest.raises(hydro.UnphysicalError) as e3:
        api.predict_patch(g, 5, m2.copy(), 0.01)
    with pytest.raises(po.UnphysicalError) as e4:
        orc.predict_patch(go, 5, m2.copy(), 0.01)
    assert str(e3.value) == str(e4.value)
    assert str(e3.value).startswith("predictor: zone (3,2,1): non-positive pressure")


# ------------------------------------------------------------------ fused stepper

STEPPER_CASES = [
    # order, solver, bc, n, problem, steps
    (2, hydro.HLL, hydro.PERIODIC, (24, 24, 24), "vortex", 6),
    (3, hydro.HLL, hydro.PERIODIC, (20, 18, 16), "vortex", 4),
    (2, hydro.RUSANOV, hydro.OUTFLOW, (40, 12, 9), "sod", 8),
    (3, hydro.RUSANOV, hydro.PERIODIC, (33, 17, 5), "vortex", 3),
    (2, hydro.HLL, hydro.PERIODIC, (17, 9, 70), "vortex", 3),
    (3, hydro.HLL, hydro.OUTFLOW, (16, 8, 4), "vortex", 3),
    # HLLC: extension without a reference counterpart, pinned to the C restatement
    (3, hydro.HLLC, hydro.PERIODIC, (20, 18, 16), "vortex", 4),
    (2, hydro.HLLC, hydro.OUTFLOW, (40, 12, 9), "sod", 8),
    (3, hydro.HLLI, hydro.PERIODIC, (20, 18, 16), "vortex", 4),
    (2, hydro.HLLI, hydro.OUTFLOW, (40, 12, 9), "sod", 8),
]


def _ic(api, g, problem, order):
    if problem == "sod":
        return api.init_sod(g)
    return api.init_isentropic_vortex(g, order)


def _run_oracle(orc, go, order, solver, bc, s, steps, cfl):
    par = po.make_params(order, solver)
    dt0 = orc.initial_dt(go, s, cfl)
    dts = orc.run_steps(go, par, bc, cfl, steps, s, dt0)
    return dts


@pytest.mark.parametrize("order,solver,bc,n,problem,steps", STEPPER_CASES)
def test_fused_stepper_bitwise(api, orc, order, solver, bc, n, problem, steps):
    lo, hi = ((0, 0, 0), (1, 1, 1)) if problem == "sod" else ((-5, -5, -5), (5, 5, 5))
    g, go = geoms(n, order, lo, hi)
    cfl = 0.6 if order == 2 else 0.4
    s0 = _ic(api, g, problem, order)
    s_ref = s0.copy()
    dts = _run_oracle(orc, go, order, solver, bc, s_ref, steps, cfl)
    st = hydro.Stepper(g, hydro.make_params(order, solver), bc=(bc, bc, bc), exact=True)
    st.upload(s0)
    st.set_time(0.0, dts[0], cfl)
    st.step(steps)
    t, dt_next, ndone = st.sync()
    out = st.download()
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    assert ndone == steps
    assert same(out[act], s_ref[act])
    assert dt_next == dts[-1]
    tt = 0.0
    for d in dts[:-1]:
        tt = tt + d
    assert t == tt
    assert st.launches >= 3 * steps  # ghost fill (1-3 launches) + fused + advance per step


@pytest.mark.parametrize("order,nst,bc,n", [(2, 2, hydro.PERIODIC, (18, 14, 11)),
                                            (3, 3, hydro.PERIODIC, (16, 12, 9)),
                                            (3, 2, hydro.OUTFLOW, (17, 9, 8)),
                                            (2, 3, hydro.PERIODIC, (24, 24, 24))])
def test_fused_rk_stepper_bitwise(api, orc, order, nst, bc, n):
    """Heun / SSP-RK3 on the fused stepper (one launch per stage, temporal mode zero) vs
    the oracle's rk_step (stepper.cpp:145-157), several steps."""
    g, go = geoms(n, order)
    cfl = 0.6 if order == 2 else 0.4
    s0 = api.init_isentropic_vortex(g, order)
    s = s0.copy()
    par = po.make_params(order)
    dt = orc.initial_dt(go, s, cfl)
    dts = [dt]
    bufs = [po.zeros_modal(go, order), *po.zeros_faces(go), po.zeros_rate(go),
            po.zeros_skinny(go)]
    for _ in range(3):
        dt = orc.rk_step(go, par, nst, bufs[0], s, *bufs[1:], bc, dt, cfl)
        dts.append(dt)
    st = hydro.Stepper(g, hydro.make_params(order), bc=(bc, bc, bc), integrator=nst)
    assert st.stages == nst
    st.upload(s0)
    st.set_time(0.0, dts[0], cfl)
    st.step(3)
    t, dt_next, done = st.sync()
    out = st.download()
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    assert done == 3 and dt_next == dts[-1]
    assert same(out[act], s[act])


@pytest.mark.parametrize("order,bc,chunks,inplace", [(3, hydro.PERIODIC, 5, True),
                                                     (2, hydro.OUTFLOW, 3, True),
                                                     (3, hydro.PERIODIC, 1, True),
                                                     (3, hydro.PERIODIC, 4, False),
                                                     (2, hydro.PERIODIC, 2, False)])
def test_pipelined_host_step_equals_device_step(api, order, bc, chunks, inplace):
    """hc_stepper_step_host (H2D / fused / D2H overlapped by z-chunks) == resident steps; in
    place (whole-plane copies) and into a separate buffer (active-zone copies), the caller's
    ghost zones untouched either way."""
    from tests.zmod import modulate_z
    g = hydro.make_geometry(20, 12, 23, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))  # z chunks see different data
    cfl = 0.6 if order == 2 else 0.4
    dt0 = api.initial_dt(g, s0, cfl)
    a = hydro.Stepper(g, hydro.make_params(order), bc=(bc, bc, bc))
    a.upload(s0)
    a.set_time(0.0, dt0, cfl)
    a.step(3)
    ta = a.sync()
    ra = a.download()
    b = hydro.Stepper(g, hydro.make_params(order), bc=(bc, bc, bc))
    b.set_time(0.0, dt0, cfl)
    host = s0.copy()
    gh = g.ghost
    ghost = np.ones(host.shape[:3], bool)
    ghost[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx] = False
    host[ghost] = np.nan  # only active zones cross PCIe; the device fills the ghosts
    for _ in range(3):
        if inplace:
            b.step_host(host, host, chunks)  # like the bench's e2e loop
        else:
            out = np.full_like(host, -7.0)
            b.step_host(host, out, chunks)
            assert (out[ghost] == -7.0).all()
            host = out
            host[ghost] = np.nan
    tb = b.sync()
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    assert ta == tb
    assert same(host[act], ra[act])
    assert np.isnan(host[ghost]).all()


def test_fused_stepper_c1_golden(api):
    """configs[0] (128x128x4, O3, periodic) through the fused kernel vs the reference digest."""
    case = golden.load_all()["ader_o3_hll_c1_128x128x4"]
    meta = case["meta"]
    g = hydro.make_geometry(*meta["n"], 3)
    s = api.init_isentropic_vortex(g, 3)
    dt0 = api.initial_dt(g, s, 0.4)
    st = hydro.Stepper(g, hydro.make_params(3, hydro.HLL), exact=True)
    st.upload(s)
    st.set_time(0.0, dt0, 0.4)
    st.step(meta["steps"])
    st.sync()
    out = st.download()
    gh = g.ghost
    act = out[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    assert golden.digest(act) == case["digests"]["skinny_active"]


@pytest.mark.parametrize("order", [2, 3])
def test_fused_fast_build_tolerance(api, orc, order):
    """FMA-contracted build: per-variable relative L1 vs the oracle <= 1e-12 after 20 steps
    (north star budget 1e-10)."""
    g, go = geoms((24, 20, 16), order)
    cfl = 0.6 if order == 2 else 0.4
    s0 = api.init_isentropic_vortex(g, order)
    s_ref = s0.copy()
    dts = _run_oracle(orc, go, order, hydro.HLL, po.PERIODIC, s_ref, 20, cfl)
    st = hydro.Stepper(g, hydro.make_params(order), exact=False)
    st.upload(s0)
    st.set_time(0.0, dts[0], cfl)
    st.step(20)
    st.sync()
    out = st.download()
    gh = g.ghost
    a = out[gh:-gh, gh:-gh, gh:-gh].reshape(-1, 5)
    b = s_ref[gh:-gh, gh:-gh, gh:-gh].reshape(-1, 5)
    for q in range(5):
        den = max(np.abs(b[:, q]).mean(), 1e-300)
        rel = np.abs(a[:, q] - b[:, q]).mean() / den
        assert rel <= 1e-12, (q, rel)


def test_fused_t_final_clip_lands_exactly(api, orc):
    """harness.cpp:155-170: the last step is clipped to land on t_final."""
    g, go = geoms((12, 12, 12), 2)
    s0 = api.init_isentropic_vortex(g, 2)
    cfl = 0.6
    t_final = 0.37
    st = hydro.Stepper(g, hydro.make_params(2), exact=True)
    st.upload(s0)
    dt0 = api.initial_dt(g, s0, cfl)
    st.set_time(0.0, dt0, cfl, t_final=t_final)
    st.step(200)  # far more than needed; the device stops itself
    t, dt, n = st.sync()
    out = st.download()
    # oracle replay of the harness loop
    s = s0.copy()
    par = po.make_params(2)
    modal = po.zeros_modal(go, 2)
    f = po.zeros_faces(go)
    r = po.zeros_rate(go)
    tt, dtt, steps = 0.0, dt0, 0
    while not (t_final - tt <= 1e-12 * t_final):
        if dtt >= t_final - tt:
            dtt = t_final - tt
        orc.apply_boundary_skinny(go, po.PERIODIC, s)
        dn = orc.ader_step(go, par, modal, s, *f, r, dtt, cfl)
        tt = tt + dtt
        dtt = dn
        steps += 1
    assert n == steps and t == tt
    gh = g.ghost
    assert same(out[gh:-gh, gh:-gh, gh:-gh], s[gh:-gh, gh:-gh, gh:-gh])


def test_fused_unphysical_stops_and_reports(api):
    g = hydro.make_geometry(16, 16, 16, 2)
    s = api.init_constant(g)
    gh = g.ghost
    s[gh + 3, gh + 2, gh + 1, 4] = -1.0  # negative energy -> negative pressure
    st = hydro.Stepper(g, hydro.make_params(2), exact=True)
    st.upload(s)
    st.set_time(0.0, 0.01, 0.6)
    st.step(3)
    with pytest.raises(hydro.UnphysicalError, match="non-positive pressure"):
        st.sync()


def test_full_size_properties_256_o3(api):
    """BASELINE configs[1] size (256^3, O3): size-independent properties only --
    conservation to round-off (periodic), exact vs FMA builds agree to 1e-12, constant
    state is a bit-exact fixed point."""
    n = 256
    g = hydro.make_geometry(n, n, n, 3)
    s0 = api.init_isentropic_vortex(g, 3)
    dt0 = api.initial_dt(g, s0, 0.4)
    outs = {}
    for exact in (True, False):
        st = hydro.Stepper(g, hydro.make_params(3), exact=exact)
        st.upload(s0)
        st.set_time(0.0, dt0, 0.4)
        st.step(3)
        st.sync()
        outs[exact] = st.download()
        st.close()
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    for q in range(5):
        before = np.sum(s0[act][..., q])
        after = np.sum(outs[True][act][..., q])
        scale = max(float(np.abs(s0[act][..., q]).sum()), 1.0)
        assert abs(after - before) <= 1e-12 * scale, q  # test_corrector.cpp:264-307
        a, b = outs[True][act][..., q], outs[False][act][..., q]
        assert np.abs(a - b).mean() <= 1e-12 * np.abs(a).mean() + 1e-300
    c = api.init_constant(g)
    st = hydro.Stepper(g, hydro.make_params(3), exact=True)
    st.upload(c)
    st.set_time(0.0, 0.01, 0.4)
    st.step(2)
    st.sync()
    out = st.download()
    assert same(out[act], c[act])


@pytest.mark.parametrize("integrator", [hydro.ADER, hydro.RK3])
def test_graph_replay_equals_plain_launches(api, integrator):
    """hc_stepper_step(n > 1) replays one captured step as a CUDA graph: same bits, same
    device time control, same launch accounting as n single steps."""
    g = hydro.make_geometry(20, 16, 12, 3)
    s0 = api.init_isentropic_vortex(g, 3)
    dt0 = api.initial_dt(g, s0, 0.4)
    outs = []
    for graph in (True, False):
        st = hydro.Stepper(g, hydro.make_params(3), integrator=integrator)
        st.upload(s0)
        st.set_time(0.0, dt0, 0.4, 0.3)
        if graph:
            st.step(9)
            st.step(9)
        else:
            for _ in range(18):
                st.step(1)
        outs.append((st.download(), st.sync(), st.launches))
        st.close()
    (a, ta, la), (b, tb, lb) = outs
    assert same(a, b) and ta == tb and la == lb


def test_fma_build_long_run_within_north_star_budget(api, orc):
    """The north star's bar: <= 1e-10 relative L1 after N steps. 200 steps of the FMA build at
    32^3 O3 against the oracle (reference-identical) run."""
    g, go = geoms((32, 32, 32), 3)
    s0 = api.init_isentropic_vortex(g, 3)
    ref = s0.copy()
    dts = _run_oracle(orc, go, 3, hydro.HLL, po.PERIODIC, ref, 200, 0.4)
    st = hydro.Stepper(g, hydro.make_params(3), exact=False)
    st.upload(s0)
    st.set_time(0.0, dts[0], 0.4)
    st.step(200)
    st.sync()
    out = st.download()
    gh = g.ghost
    a = out[gh:-gh, gh:-gh, gh:-gh].reshape(-1, 5)
    b = ref[gh:-gh, gh:-gh, gh:-gh].reshape(-1, 5)
    worst = max(np.abs(a[:, q] - b[:, q]).mean() / max(np.abs(b[:, q]).mean(), 1e-300)
                for q in range(5))
    assert worst <= 1e-10, worst
    st.close()
