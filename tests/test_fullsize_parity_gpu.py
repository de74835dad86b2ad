"""Parity at the benchmarked sizes: the reference's own
harness (``hydro::run_benchmark``, proj/src/harness.cpp:222-227, compiled from its sources into
oracle/_ref) against the device stepper driven by our harness, on identical initial conditions.

- C2 256^3 WENO-ADER O3 + HLL vortex, 5 steps: the bit-exact build reproduces the reference's
  final U_skinny (every active zone, every variable) and t bit for bit; the FMA build (the
  bench headline) stays within the north star's 1e-10 per-variable relative L1 and L-infinity.
- C1 128x128x4 O3, 50 steps: the same two checks.
- C3 proxy 384^3 O2, 1 step: the same two checks.

The measured differences are written to ``gpurun_out/fullsize_parity.json`` (summarised in
profiles/). The reference runs on all host cores; its result is thread-count invariant
(acceptance criterion 3)."""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2211_13295_b200 import harness, hydro

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north star: <= 1e-10 per-variable relative L1 / L-inf after N steps
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                   "fullsize_parity.json")

CASES = {
    # name: (nx, ny, nz, order, steps)
    "C2_256_o3_5steps": (256, 256, 256, 3, 5),
    "C1_128x128x4_o3_50steps": (128, 128, 4, 3, 50),
    "C3proxy_384_o2_1step": (384, 384, 384, 2, 1),
}


@pytest.fixture(scope="module")
def ref():
    if not po.have_reference():
        pytest.skip("oracle/_ref (the reference built from its sources) is absent")
    assert hydro.device_count() > 0
    return po.Reference()


def _record(name, entry):
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data[name] = entry
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)


def _rel_norms(a, b):
    """per-variable relative L1 and L-inf of a against b (active zones, [z][y][x][5])."""
    d = np.abs(a - b).reshape(-1, 5)
    s = np.abs(b).reshape(-1, 5)
    l1 = d.sum(0) / np.maximum(s.sum(0), 1e-300)
    linf = d.max(0) / np.maximum(s.max(0), 1e-300)
    return l1, linf


@pytest.mark.parametrize("name", list(CASES))
def test_reference_harness_at_full_size(ref, name):
    nx, ny, nz, order, steps = CASES[name]
    _, fin_ref, t_ref, _ = ref.run_benchmark(0, order, 0, po.HLL, (nx, ny, nz), steps,
                                             threads=0, want_state=True)
    g = hydro.make_geometry(nx, ny, nz, order)
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    b = fin_ref[act]
    entry = {"mesh": [nx, ny, nz], "order": order, "solver": "hll", "steps": steps,
             "t_reference": t_ref.hex()}
    for exact in (True, False):
        cfg = harness.RunConfig(problem=harness.VORTEX, order=order, nx=nx, ny=ny, nz=nz,
                                steps=steps, exact=exact)
        r = harness.run_benchmark(cfg)
        a = r.final_state[act]
        l1, linf = _rel_norms(a, b)
        nbad = int((a.view(np.uint64) != b.view(np.uint64)).sum())
        key = "exact" if exact else "fma"
        entry[key] = {"kernel": r.kernel, "t": r.t_end.hex(), "steps": r.steps,
                      "rel_l1": l1.tolist(),
                      "rel_linf": linf.tolist(), "differing_values": nbad,
                      "values": int(a.size)}
        _record(name, entry)
        assert r.steps == steps
        if exact:
            assert nbad == 0, f"{nbad} of {a.size} values differ from the reference"
            assert r.t_end == t_ref
        else:
            assert (l1 <= TOL).all() and (linf <= TOL).all(), (l1, linf)
            assert abs(r.t_end - t_ref) <= TOL * t_ref
