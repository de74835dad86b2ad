"""Device-resident PatchSet (transfer.hpp:47-73 on the GPU): run_patch_step over px x py x pz
patches must equal the single-patch run bit for bit -- the reference's split invariance
(acceptance criterion 8, test_transfer.cpp:151-188) -- for ADER and RK, periodic and
outflow; and the TransferLedger must count what transfer.cpp:160-175 counts."""
import numpy as np
import pytest

from paper_2211_13295_b200 import hydro

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("split,order,bc,integ", [
    ((2, 2, 2), 3, hydro.PERIODIC, hydro.ADER),
    ((3, 1, 2), 2, hydro.OUTFLOW, hydro.ADER),
    ((1, 2, 2), 3, hydro.PERIODIC, hydro.RK3),
    ((2, 1, 1), 3, hydro.OUTFLOW, hydro.RK2),
])
def test_patch_split_is_bit_identical(split, order, bc, integ):
    api = hydro.HostApi()
    g = hydro.make_geometry(24, 16, 20, order)
    from tests.zmod import modulate_z
    s0 = modulate_z(api.init_sod(g) if bc == hydro.OUTFLOW else
                    api.init_isentropic_vortex(g, order))
    cfl = 0.6 if order == 2 else 0.4
    dt0 = api.initial_dt(g, s0, cfl)
    steps = 4
    st = hydro.Stepper(g, hydro.make_params(order), bc=(bc, bc, bc), integrator=integ)
    st.upload(s0)
    st.set_time(0.0, dt0, cfl)
    st.step(steps)
    want = st.download()
    t_want = st.sync()
    st.close()
    ps = hydro.PatchSet(g, *split, hydro.make_params(order), boundary=bc, integrator=integ)
    ps.scatter(s0)
    ps.set_time(0.0, dt0, cfl)
    ps.step(steps)
    got = ps.gather()
    assert ps.sync() == t_want
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    assert (bits(got[act]) == bits(want[act])).all()
    # TransferLedger (skinny strategy): per patch per step total_zones*5 each way + 1 scalar
    np_ = split[0] * split[1] * split[2]
    lg = hydro.make_geometry(24 // split[0], 16 // split[1], 20 // split[2], order)
    total = lg.mx * lg.my * lg.mz * 5
    active = lg.nx * lg.ny * lg.nz * 5
    assert ps.ledger() == (total * np_ * steps, total * np_ * steps, np_ * steps, np_ * steps,
                           active * np_ * steps, steps)
    assert ps.ledger_csv_row(7) == f"7,skinny,{total * np_},{total * np_},{np_}"
    ps.close()


def test_patch_split_must_divide():
    g = hydro.make_geometry(24, 16, 20, 3)
    with pytest.raises(ValueError, match="divide"):
        hydro.PatchSet(g, 5, 1, 1, hydro.make_params(3))


def test_ledger_counts_executed_steps_only():
    """The device turns steps past t_final into no-ops; the TransferLedger counts the steps the
    reference would have run (transfer.cpp:160-216), not the steps queued."""
    g = hydro.make_geometry(16, 16, 16, 2)
    api = hydro.HostApi()
    s0 = api.init_isentropic_vortex(g, 2)
    dt0 = api.initial_dt(g, s0, 0.6)
    ps = hydro.PatchSet(g, 2, 1, 1, hydro.make_params(2))
    ps.scatter(s0)
    ps.set_time(0.0, dt0, 0.6, 3.5 * dt0)  # lands on t_final after a few steps
    ps.step(40)
    t, dt, done = ps.sync()
    assert 0 < done < 40
    assert ps.ledger()[5] == done
    ps.close()
