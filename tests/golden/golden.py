"""Golden-vector cases for the space-time update.

Each case is a small deterministic run described by ``meta``; ``run_case(lib, meta)`` executes
it through any object exposing the reference-shaped API used by the checkers
(``oracle.pyoracle.Oracle`` / ``Reference``) or the CUDA product adapter
(``paper_2211_13295_b200.hydro.HostApi``). ``make_golden.py`` ran every case through the
REFERENCE library (oracle/_ref, built from /root/reference/proj/src) and committed the outputs
here: small arrays verbatim in ``<name>.npz`` plus SHA-256 digests of every output array.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MANIFEST = os.path.join(HERE, "manifest.json")

# name -> meta. kind: 'ader' (N ADER steps, apply_boundary before each) or 'rk' (one rk_step)
CASES = {
    "ader_o2_hll_vortex_10": dict(kind="ader", order=2, solver=1, bc=0, n=(10, 10, 10),
                                  problem="vortex", steps=5),
    "ader_o3_hll_vortex_8": dict(kind="ader", order=3, solver=1, bc=0, n=(8, 8, 8),
                                 problem="vortex", steps=3),
    "ader_o2_rusanov_sod_outflow": dict(kind="ader", order=2, solver=0, bc=1, n=(12, 6, 5),
                                        problem="sod", steps=6),
    "ader_o3_rusanov_vortex_ragged": dict(kind="ader", order=3, solver=0, bc=0, n=(9, 7, 5),
                                          problem="vortex", steps=3),
    "ader_o3_hll_c1_128x128x4": dict(kind="ader", order=3, solver=1, bc=0, n=(128, 128, 4),
                                     problem="vortex", steps=2, digest_only=True),
    "rk2_o2_hll_vortex_8": dict(kind="rk", stages=2, order=2, solver=1, bc=0, n=(8, 8, 8),
                                problem="vortex", steps=1),
    "rk3_o3_hll_vortex_8": dict(kind="rk", stages=3, order=3, solver=1, bc=0, n=(8, 8, 8),
                                problem="vortex", steps=1),
}


def _geom(po, meta):
    nx, ny, nz = meta["n"]
    if meta["problem"] == "sod":
        return po.make_geometry(nx, ny, nz, meta["order"], (0, 0, 0), (1, 1, 1))
    return po.make_geometry(nx, ny, nz, meta["order"])


def run_case(lib, meta):
    """Runs one case; returns a dict of named float64 output arrays."""
    from oracle import pyoracle as po  # layout helpers only (shapes, structs)

    g = _geom(po, meta)
    order = meta["order"]
    par = po.make_params(order, meta["solver"])
    cfl = 0.6 if order == 2 else 0.4
    if meta["problem"] == "sod":
        s = lib.init_sod(g)
    else:
        s = lib.init_isentropic_vortex(g, order)
    dt = _initial_dt(lib, g, s, cfl)
    modal = po.zeros_modal(g, order)
    fx, fy, fz = po.zeros_faces(g)
    rate = po.zeros_rate(g)
    dts = [dt]
    if meta["kind"] == "ader":
        for _ in range(meta["steps"]):
            lib.apply_boundary_skinny(g, meta["bc"], s)
            dt = lib.ader_step(g, par, modal, s, fx, fy, fz, rate, dt, cfl)
            dts.append(dt)
    else:
        u0 = po.zeros_skinny(g)
        lib.apply_boundary_skinny(g, meta["bc"], s)
        dt = lib.rk_step(g, par, meta["stages"], modal, s, fx, fy, fz, rate, u0, meta["bc"],
                         dt, cfl)
        dts.append(dt)
    gh = g.ghost
    active = np.ascontiguousarray(s[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx])
    return dict(skinny=s, skinny_active=active, modal=modal, fx=fx, fy=fy, fz=fz, rate=rate,
                dts=np.array(dts))


def _initial_dt(lib, g, s, cfl):
    """harness.cpp:92-103 (min of eval_tstep_ptwise over active zones; min is exact)."""
    if hasattr(lib, "initial_dt"):
        return lib.initial_dt(g, s, cfl)
    gh = g.ghost
    dt = 1.0e32
    act = s[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx].reshape(-1, 5)
    for u in act:
        d = lib.eval_tstep_ptwise(u, cfl, g.dx, g.dy, g.dz)
        dt = d if d < dt else dt
    return dt


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def load_all():
    """name -> {'meta', 'digests', 'arrays'} for every committed case."""
    if not os.path.exists(MANIFEST):
        return {}
    with open(MANIFEST) as f:
        man = json.load(f)
    out = {}
    for name, ent in man.items():
        arrays = {}
        npz = os.path.join(HERE, name + ".npz")
        if os.path.exists(npz):
            with np.load(npz) as z:
                arrays = {k: z[k] for k in z.files}
        out[name] = dict(meta=ent["meta"], digests=ent["digests"], arrays=arrays)
    return out
