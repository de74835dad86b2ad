"""Runs the reference's own harness (hydro::run_simulation, oracle/_ref) for the acceptance
suite's convergence runs and a few fixed-step runs; writes tests/golden/harness_runs.json
(doubles stored as float.hex so they compare exactly).  python tests/golden/make_harness_golden.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import pyoracle as po  # noqa: E402

RUNS = {
    # acceptance_main.cpp:46-56 criteria 1-2: vortex, HLL, ADER, to one crossing (t = 10)
    "conv_o2_24": dict(problem=0, order=2, integrator=0, solver=1, n=24),
    "conv_o2_48": dict(problem=0, order=2, integrator=0, solver=1, n=48),
    "conv_o3_24": dict(problem=0, order=3, integrator=0, solver=1, n=24),
    "conv_o3_48": dict(problem=0, order=3, integrator=0, solver=1, n=48),
    # test_harness.cpp:120-133 constant problem, exactly zero error
    "constant_o2_8_steps5": dict(problem=2, order=2, integrator=0, solver=1, n=8, steps=5),
    # rk3 to a short t_final (the clip path), Rusanov
    "vortex_o3_rk3_16_t0.3": dict(problem=0, order=3, integrator=3, solver=0, n=16, t_final=0.3),
    # rk2 O2 sod (outflow), fixed steps
    "sod_o2_rk2_20_steps12": dict(problem=1, order=2, integrator=2, solver=1, n=20, steps=12),
}


def main():
    ref = po.Reference()
    out = {}
    for name, r in RUNS.items():
        l1, linf, t_end, steps = po.ref_run_simulation(
            ref, r["problem"], r["order"], r["integrator"], r["solver"], r["n"],
            steps=r.get("steps", 0), t_final=r.get("t_final", -1.0), threads=8)
        out[name] = dict(run=r, l1=[float(x).hex() for x in l1],
                         linf=[float(x).hex() for x in linf], t_end=float(t_end).hex(),
                         steps=steps)
        print(name, steps, t_end, l1[0])
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "harness_runs.json"),
              "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
