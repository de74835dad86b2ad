"""The persistent ring-free fused kernel (csrc/fused_persist.cuh) against the C restatement
of the reference (oracle/), bit for bit in the exact build: tiles of 1 to 7 rows (one tile
per axis = self-exchange through the L2 records), orders 2-4, every Riemann solver, ADER and
Runge-Kutta stages, z-modulated states, the pipelined host step (z-range launches), and the
ring kernel (the default; HC_PERSIST=1 opts into the persistent one) on the same inputs."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2211_13295_b200 import hydro
from tests.zmod import modulate_z

pytestmark = pytest.mark.gpu

CASES = [
    # order, solver, integrator, (nx, ny, nz), forced tile rows (None: the default spread)
    (3, hydro.HLL, hydro.ADER, (32, 7, 5), 1),        # one tile: self-exchange in x and y
    (3, hydro.HLL, hydro.ADER, (64, 20, 9), 3),       # tile rows 7, 7, 6
    (2, hydro.HLL, hydro.ADER, (96, 13, 6), 2),       # 7, 6
    (3, hydro.RUSANOV, hydro.ADER, (64, 12, 7), None),
    (3, hydro.HLLC, hydro.ADER, (32, 14, 8), 2),
    (2, hydro.HLLI, hydro.ADER, (64, 9, 5), 3),
    (4, hydro.HLL, hydro.ADER, (32, 11, 6), 2),
    (3, hydro.HLL, hydro.RK3, (64, 15, 6), 3),
    (2, hydro.RUSANOV, hydro.RK2, (32, 10, 7), 2),
]


@pytest.fixture
def env():
    saved = {k: os.environ.get(k) for k in ("HC_PERSIST", "HC_PERSIST_NTY", "HC_SEAM")}
    os.environ["HC_SEAM"] = "0"  # the FMA comparisons below are against the ring kernel
    os.environ["HC_PERSIST"] = "1"
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


def _run(g, order, solver, integ, s0, dt0, cfl, steps, exact):
    st = hydro.Stepper(g, hydro.make_params(order, solver), exact=exact, integrator=integ)
    kind = st.kernel_info()
    st.upload(s0)
    st.set_time(0.0, dt0, cfl)
    st.step(steps)
    t, dt_next, done = st.sync()
    out = st.download()
    st.close()
    return out, dt_next, done, kind


@pytest.mark.parametrize("order,solver,integ,shape,nty", CASES)
def test_persistent_kernel_bitwise(env, order, solver, integ, shape, nty):
    if nty is not None:
        env["HC_PERSIST_NTY"] = str(nty)
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    go = po.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    cfl = 0.6 if order == 2 else 0.4
    steps = 4
    ref = s0.copy()
    dt0, dt_last = _oracle(go, order, solver, integ, ref, steps, cfl)
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    out, dt_next, done, kind = _run(g, order, solver, integ, s0, dt0, cfl, steps, True)
    assert kind[0] == "persistent", kind
    if nty is not None:
        assert kind[1] == (shape[0] // 32) * nty
    assert done == steps
    assert (out[act].view(np.uint64) == ref[act].view(np.uint64)).all()
    assert dt_next == dt_last
    # the FMA build through the same kernel: the tolerance of the ring kernel's FMA build
    fo, _, _, kind = _run(g, order, solver, integ, s0, dt0, cfl, steps, False)
    assert kind[0] == "persistent"
    a, b = fo[act].reshape(-1, 5), ref[act].reshape(-1, 5)
    for q in range(5):
        den = max(np.abs(b[:, q]).mean(), 1e-300)
        assert np.abs(a[:, q] - b[:, q]).mean() / den <= 1e-12


@pytest.mark.parametrize("exact", [True, False])
def test_persistent_equals_ring_kernel(env, exact):
    """Same inputs through both fused kernels: identical bits in the exact build; the FMA
    builds differ only by contraction choices (<= 1e-13 relative)."""
    order, shape = 3, (64, 24, 10)
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    env["HC_PERSIST_NTY"] = "4"
    a, da, _, ka = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 5, exact)
    env["HC_PERSIST"] = "0"
    b, db, _, kb = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 5, exact)
    assert ka[0] == "persistent" and kb[0] == "ring"
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    if exact:
        assert (a[act].view(np.uint64) == b[act].view(np.uint64)).all() and da == db
    else:
        d = np.abs(a[act] - b[act]).reshape(-1, 5).sum(0)
        assert (d <= 1e-13 * np.abs(b[act]).reshape(-1, 5).sum(0)).all()


@pytest.mark.parametrize("chunks", [1, 3])
def test_persistent_pipelined_host_step(env, chunks):
    """hc_stepper_step_host launches the kernel on z ranges (each with its own z-ring planes):
    the same bits as the resident step."""
    order, shape = 3, (32, 14, 12)
    env["HC_PERSIST_NTY"] = "2"
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    want, _, _, _ = _run(g, order, hydro.HLL, hydro.ADER, s0, dt0, 0.4, 1, True)
    st = hydro.Stepper(g, hydro.make_params(order), exact=True)
    assert st.kernel_info()[0] == "persistent"
    st.set_time(0.0, dt0, 0.4)
    out = s0.copy()
    st.step_host(s0, out, chunks)
    st.sync()
    st.close()
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    assert (out[act].view(np.uint64) == want[act].view(np.uint64)).all()
