"""The ring-free seam kernel pair (csrc/fused_seam.cuh: the fused step with tile-boundary
faces left out, then seam_fix_kernel) against the C restatement of the reference (oracle/):
the FMA build within its tolerance, the bit-exact build (the reference's association kept
through the edge zones' records) bit for bit; against the ring kernels (HC_SEAM=0), and for
the properties the FMA build's re-association must keep: conservation to round-off on a
periodic mesh, z-range launches equal to the whole launch, the pipelined host step."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2211_13295_b200 import hydro
from tests.zmod import modulate_z

pytestmark = pytest.mark.gpu

TOL = 1e-12  # relative L1 per variable after the steps below (the FMA ring kernel's bound)

CASES = [
    # order, solver, integrator, (nx, ny, nz): tile rows 7 / balanced 6-7 / single tile
    (3, hydro.HLL, hydro.ADER, (32, 7, 5)),        # one tile: both seams wrap to itself
    (3, hydro.HLL, hydro.ADER, (64, 20, 9)),       # rows 7, 7, 6
    (3, hydro.HLL, hydro.ADER, (96, 9, 6)),        # rows 5, 4
    (2, hydro.HLL, hydro.ADER, (64, 13, 6)),
    (3, hydro.RUSANOV, hydro.ADER, (64, 12, 7)),
    (3, hydro.HLLC, hydro.ADER, (32, 14, 8)),
    (2, hydro.HLLI, hydro.ADER, (64, 9, 5)),
    (4, hydro.HLL, hydro.ADER, (32, 11, 6)),
    (3, hydro.HLL, hydro.RK3, (64, 15, 6)),
    (2, hydro.RUSANOV, hydro.RK2, (32, 10, 7)),
    (3, hydro.HLL, hydro.ADER, (32, 4, 4)),        # one 4-row tile, minimal mesh
]


@pytest.fixture
def env():
    saved = {k: os.environ.get(k) for k in ("HC_SEAM", "HC_PERSIST", "HC_TZ")}
    os.environ.pop("HC_PERSIST", None)
    os.environ["HC_SEAM"] = "1"  # the pair wherever the mesh allows (small meshes, O2 exact)
    yield os.environ
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _oracle(go, order, solver, integ, s, steps, cfl):
    orc = po.Oracle()
    dt0 = orc.initial_dt(go, s, cfl)
    par = po.make_params(order, solver)
    if integ == hydro.ADER:
        dts = orc.run_steps(go, par, po.PERIODIC, cfl, steps, s, dt0)
        return dt0, dts[-1]
    modal = po.zeros_modal(go, order)
    f = po.zeros_faces(go)
    rate = po.zeros_rate(go)
    u0 = s.copy()
    dt = dt0
    for _ in range(steps):
        dt = orc.rk_step(go, par, integ, modal, s, *f, rate, u0, po.PERIODIC, dt, cfl)
    return dt0, dt


def _run(g, order, solver, integ, s0, dt0, cfl, steps, exact=False):
    st = hydro.Stepper(g, hydro.make_params(order, solver), exact=exact, integrator=integ)
    kind = st.kernel_info()
    st.upload(s0)
    st.set_time(0.0, dt0, cfl)
    st.step(steps)
    t, dt_next, done = st.sync()
    out = st.download()
    st.close()
    return out, dt_next, done, kind


def _act(g):
    gh = g.ghost
    return np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]


def _rel_l1(a, b):
    """Per-variable L1 difference relative to that variable's mean magnitude (floored at 1e-3
    of the largest one: a momentum component that is exactly zero in the reference, e.g. w on
    the z-invariant configs[0] vortex, is compared on the state's scale)."""
    a, b = a.reshape(-1, 5), b.reshape(-1, 5)
    mag = np.abs(b).mean(0)
    floor = 1e-3 * mag.max()
    return [np.abs(a[:, q] - b[:, q]).mean() / max(mag[q], floor) for q in range(5)]


@pytest.mark.parametrize("order,solver,integ,shape", CASES)
def test_seam_kernel_vs_reference(env, order, solver, integ, shape):
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    go = po.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    cfl = 0.6 if order == 2 else 0.4
    steps = 5
    ref = s0.copy()
    dt0, dt_last = _oracle(go, order, solver, integ, ref, steps, cfl)
    out, dt_next, done, kind = _run(g, order, solver, integ, s0, dt0, cfl, steps)
    assert kind[0] == "seam", kind
    assert done == steps
    act = _act(g)
    assert max(_rel_l1(out[act], ref[act])) <= TOL
    assert abs(dt_next - dt_last) <= 1e-12 * dt_last
    # the bit-exact build's seam pair: every bit of the reference's state and dt
    x, dx_next, xdone, kx = _run(g, order, solver, integ, s0, dt0, cfl, steps, exact=True)
    assert kx[0] == "seam" and xdone == steps
    assert (x[act].view(np.uint64) == ref[act].view(np.uint64)).all(), \
        np.abs(x[act] - ref[act]).max()
    assert dx_next == dt_last


def test_seam_equals_fma_ring_kernel(env):
    order, shape = 3, (64, 24, 10)
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    a, da, _, ka = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 8)
    env["HC_SEAM"] = "0"
    b, db, _, kb = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 8)
    assert ka[0] == "seam" and kb[0] == "ring"
    act = _act(g)
    assert max(_rel_l1(a[act], b[act])) <= 1e-13
    assert abs(da - db) <= 1e-13 * db


@pytest.mark.parametrize("integ", [hydro.ADER, hydro.RK3])
def test_seam_conserves(env, integ):
    """Periodic mesh: every face flux enters its two zones with opposite signs, so the totals
    of the conserved variables stay put to round-off -- including across the seams, whose
    fluxes both neighbours solve from the same two published states."""
    order, shape = 3, (64, 20, 9)
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    out, _, _, kind = _run(g, order, hydro.HLL, integ, s0, dt0, 0.4, 10)
    assert kind[0] == "seam"
    act = _act(g)
    t0 = s0[act].reshape(-1, 5).sum(0)
    t1 = out[act].reshape(-1, 5).sum(0)
    scale = np.abs(s0[act]).reshape(-1, 5).sum(0)
    assert (np.abs(t1 - t0) <= 1e-13 * scale).all(), (t1 - t0) / scale


def test_seam_z_chunks_and_ranges(env):
    """z chunks (HC_TZ) and z ranges (compute_range, as the slab overlap uses) are separate
    launches of both kernels with their own z-ring planes: same bits as one launch."""
    order, shape = 3, (32, 14, 12)
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    want, dw, _, _ = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 2)
    env["HC_TZ"] = "5"
    got, dg, _, kind = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 2)
    assert kind[0] == "seam"
    act = _act(g)
    assert (got[act].view(np.uint64) == want[act].view(np.uint64)).all() and dg == dw
    env.pop("HC_TZ")
    st = hydro.Stepper(g, hydro.make_params(order), exact=False)
    st.upload(s0)
    st.set_time(0.0, dt0, 0.4)
    st.fill_ghosts()
    for lo, hi, last in ((3, 9, 0), (0, 3, 0), (9, 12, 1)):
        st.compute_range(lo, hi, last)
    st.advance()
    st.sync()
    out = st.download()
    st.close()
    one, _, _, _ = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 1)
    assert (out[act].view(np.uint64) == one[act].view(np.uint64)).all()


@pytest.mark.parametrize("chunks", [1, 4])
def test_seam_pipelined_host_step(env, chunks):
    order, shape = 3, (64, 14, 12)
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    want, _, _, _ = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 1)
    st = hydro.Stepper(g, hydro.make_params(order), exact=False)
    assert st.kernel_info()[0] == "seam"
    st.set_time(0.0, dt0, 0.4)
    out = s0.copy()
    st.step_host(s0, out, chunks)
    st.sync()
    st.close()
    act = _act(g)
    assert (out[act].view(np.uint64) == want[act].view(np.uint64)).all()


def test_seam_configs0(env):
    """configs[0] (128 x 128 x 4, O3, the reference's 2D emulation) through the seam kernel for
    50 steps within the FMA tolerance of the bit-exact ring kernel."""
    order, shape = 3, (128, 128, 4)
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = api.init_isentropic_vortex(g, order)
    dt0 = api.initial_dt(g, s0, 0.4)
    a, da, _, ka = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 50)
    env["HC_SEAM"] = "0"
    b, db, _, kb = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 50, exact=True)
    assert ka[0] == "seam" and kb[0] == "ring"
    act = _act(g)
    assert max(_rel_l1(a[act], b[act])) <= TOL
    assert abs(da - db) <= 1e-12 * db


@pytest.mark.parametrize("order,solver,integ,shape", [
    (3, hydro.HLL, hydro.ADER, (64, 24, 10)),
    (2, hydro.RUSANOV, hydro.RK2, (32, 17, 6)),
    (3, hydro.HLLC, hydro.RK3, (96, 12, 5)),
])
def test_seam_exact_equals_exact_ring(env, order, solver, integ, shape):
    """the bit-exact build's seam pair and its ring kernel (HC_SEAM=0) agree to the last bit
    (both keep the reference's association), state and dt, over 8 steps"""
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    a, da, _, ka = _run(g, order, solver, integ, s0, dt0, 0.4, 8, exact=True)
    env["HC_SEAM"] = "0"
    b, db, _, kb = _run(g, order, solver, integ, s0, dt0, 0.4, 8, exact=True)
    assert ka[0] == "seam" and kb[0] == "ring"
    act = _act(g)
    assert (a[act].view(np.uint64) == b[act].view(np.uint64)).all(), np.abs(a - b).max()
    assert da == db
