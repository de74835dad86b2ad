"""The reference's run driver (harness.cpp:116-227) on the fused device stepper:
whole runs -- initial condition, dt hand-off, t_final clip, error norms vs the exact vortex --
must reproduce the reference's own harness (tests/golden/harness_runs.json, produced by
hydro::run_simulation from the reference library) exactly, including the acceptance suite's
convergence studies (criteria 1-2: O2 order 1.678, O3 order 2.50)."""
import json
import math
import os

import pytest

from paper_2211_13295_b200 import harness, hydro

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "harness_runs.json")
PROBLEMS = {0: harness.VORTEX, 1: harness.SOD, 2: harness.CONSTANT}
INTEG = {0: "ader", 2: "rk2", 3: "rk3"}


def _cfg(run, exact=True):
    return harness.RunConfig(problem=PROBLEMS[run["problem"]], order=run["order"],
                             integrator=INTEG[run["integrator"]], solver=run["solver"],
                             nx=run["n"], ny=run["n"], nz=run["n"],
                             steps=run.get("steps", 0), t_final=run.get("t_final", -1.0),
                             exact=exact)


@pytest.fixture(scope="module")
def gold():
    assert hydro.device_count() > 0
    with open(GOLD) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["conv_o2_24", "conv_o2_48", "conv_o3_24", "conv_o3_48",
                                  "constant_o2_8_steps5", "vortex_o3_rk3_16_t0.3",
                                  "sod_o2_rk2_20_steps12"])
def test_run_simulation_matches_reference_harness(gold, name):
    ent = gold[name]
    r = harness.run_simulation(_cfg(ent["run"]))
    assert r.steps == ent["steps"]
    assert r.t_end.hex() == ent["t_end"]
    if r.errors is not None:
        assert [float(x).hex() for x in r.errors.l1] == ent["l1"]
        assert [float(x).hex() for x in r.errors.linf] == ent["linf"]


def test_convergence_orders_match_acceptance(gold):
    """acceptance_main.cpp:46-56: the observed orders, from the GPU runs."""
    for order, lo, hi in ((2, 1.7, 2.4), (3, 2.5, 3.3)):
        rows = harness.run_convergence_study(harness.RunConfig(order=order), [24, 48])
        ref = math.log(float.fromhex(gold[f"conv_o{order}_24"]["l1"][0]) /
                       float.fromhex(gold[f"conv_o{order}_48"]["l1"][0])) / math.log(2.0)
        got = rows[1][1].order_estimate
        assert got == ref
        if order == 3:
            assert lo <= got <= hi
        else:  # the reference itself misses the O2 window; so must we
            assert abs(got - 1.678) < 1e-3


def test_constant_problem_zero_error():
    """test_harness.cpp:120-133."""
    r = harness.run_simulation(harness.RunConfig(problem=harness.CONSTANT, nx=8, ny=8, nz=8,
                                                 steps=5))
    assert (r.errors.l1 == 0).all() and (r.errors.linf == 0).all()


def test_split_run_through_the_harness_equals_single_patch(gold):
    """harness RunConfig.split_* (harness.hpp:24) runs the device PatchSet: same final state
    and dt trajectory as the single patch, as acceptance criterion 8 demands."""
    base = harness.RunConfig(problem=harness.VORTEX, order=3, nx=16, ny=16, nz=16, steps=6)
    a = harness.run_simulation(base)
    b = harness.run_simulation(harness.RunConfig(**{**base.__dict__, "split_x": 2,
                                                    "split_y": 2, "split_z": 2}))
    assert (a.final_state.view("u8") == b.final_state.view("u8")).all()
    assert a.t_end == b.t_end and a.steps == b.steps


def test_reproducibility_check():
    """harness.cpp:229-271: repeated runs bit-identical, decomposed run within 1e-10 (0 here)"""
    rep = harness.run_reproducibility_check(
        harness.RunConfig(problem=harness.VORTEX, order=2, nx=16, ny=16, nz=16, steps=20))
    assert rep.serial_bit_identical and rep.passed
    assert rep.multiworker_l1_diff == 0.0 and rep.max_abs_diff == 0.0
