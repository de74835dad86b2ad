"""GPU tests of the z-slab driver (slabs.SlabDomain) on one device: the overlapped step --
interior planes computed while the z-halo exchange runs on a second stream, then the two
boundary ranges -- must equal the plain single-domain stepper bit for bit, for ADER and RK,
periodic and outflow, both orders (the N>1 exchange itself is covered over gloo in
tests/test_slabs_gloo.py)."""
import numpy as np
import pytest
import torch

from paper_2211_13295_b200 import hydro, slabs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("order,bc,integrator,exact", [
    (3, hydro.PERIODIC, hydro.ADER, True),
    (2, hydro.PERIODIC, hydro.ADER, True),
    (3, hydro.OUTFLOW, hydro.ADER, True),
    (3, hydro.PERIODIC, hydro.RK3, True),
    (3, hydro.PERIODIC, hydro.ADER, False),
])
def test_overlapped_slab_step_matches_stepper(order, bc, integrator, exact):
    n, steps = 24, 4
    dom = slabs.SlabDomain(n, n, n, order, exact=exact, bc=bc, integrator=integrator,
                           overlap=True)
    from tests.zmod import modulate_z
    s0 = modulate_z(dom.initial_state())  # z-varying: the plane ranges must be right
    cfl = 0.6 if order == 2 else 0.4
    dt0 = dom.initial_dt(s0, cfl)
    dom.upload(s0)
    dom.set_time(0.0, dt0, cfl)
    for _ in range(steps):
        dom.step()
    torch.cuda.synchronize()
    got = dom.download()
    t1 = dom.sync()
    dom.close()
    st = hydro.Stepper(dom.geom, hydro.make_params(order), bc=(bc, bc, bc), exact=exact,
                       integrator=integrator)
    st.upload(s0)
    st.set_time(0.0, dt0, cfl)
    st.step(steps)
    want = st.download()
    gh = dom.geom.ghost
    act = np.s_[gh:gh + n, gh:gh + n, gh:gh + n]
    assert (bits(got[act]) == bits(want[act])).all()
    assert st.sync() == t1
    st.close()
