"""Algorithmic FP64 work per zone-update of the MHD and CED extensions, counted from their
numpy restatements (oracle/mhd_oracle.py, oracle/ced_oracle.py) as written -- the same
convention as SURVEY.md App. A for the reference's Euler path: every elementwise add,
subtract, multiply, divide and sqrt is one flop (min/max/abs/compare/select are not counted;
exp/expm1 are counted separately). Arrays are wrapped in a counting ndarray subclass; the
count is divided by active zones x steps, so ring and face overheads are included as the
restatement computes them.

    python tools/count_flops_ext.py [n1 n2 n3]    -> profiles/r2_ext_flops.json
"""
import json
import os
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FLOP_UFUNCS = {np.add, np.subtract, np.multiply, np.true_divide, np.divide, np.sqrt}
TRANS_UFUNCS = {np.exp, np.expm1}


class Counter:
    flops = 0
    trans = 0


class CountArr(np.ndarray):
    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        raw = [np.asarray(x) if isinstance(x, CountArr) else x for x in inputs]
        if "out" in kwargs:
            kwargs["out"] = tuple(np.asarray(o) if isinstance(o, CountArr) else o
                                  for o in kwargs["out"])
        res = getattr(ufunc, method)(*raw, **kwargs)
        if method == "__call__":
            size = np.asarray(res[0] if isinstance(res, tuple) else res).size
            if ufunc in FLOP_UFUNCS:
                Counter.flops += size
            elif ufunc in TRANS_UFUNCS:
                Counter.trans += size
        return wrap(res)

    def __array_function__(self, func, types_, args, kwargs):
        args = unwrap(args)
        kwargs = unwrap(kwargs)
        return wrap(func(*args, **kwargs))


def unwrap(x):
    if isinstance(x, CountArr):
        return x.view(np.ndarray)
    if isinstance(x, (list, tuple)):
        return type(x)(unwrap(v) for v in x)
    if isinstance(x, dict):
        return {k: unwrap(v) for k, v in x.items()}
    return x


def wrap(x):
    if isinstance(x, np.ndarray) and not isinstance(x, CountArr) and x.dtype.kind == "f":
        return x.view(CountArr)
    if isinstance(x, tuple):
        return tuple(wrap(v) for v in x)
    if isinstance(x, list):
        return [wrap(v) for v in x]
    return x


def counting_numpy():
    """A proxy for the oracles' `np` whose array constructors return counting arrays."""
    proxy = types.ModuleType("np_count")
    proxy.__dict__.update(np.__dict__)
    for name in ("zeros", "empty", "ones", "full", "zeros_like", "empty_like", "ones_like",
                 "array", "asarray", "where", "sqrt", "abs", "copysign", "clip", "exp", "expm1",
                 "roll", "arange"):
        f = getattr(np, name)
        proxy.__dict__[name] = (lambda f: lambda *a, **k: wrap(f(*unwrap(a), **unwrap(k))))(f)
    return proxy


def count_mhd(n, order):
    from oracle import mhd_oracle as mo
    from paper_2211_13295_b200 import mhd
    g = mhd.make_geometry(n, n, n, order, (0, 0, 0), (1, 1, 1))
    s = mhd.orszag_tang(g, order)
    G = mo.Geom(n, n, n, order)
    par = mo.Params(order)
    dt = mo.cfl_dt(s, G, par, 0.4)
    mo.np = counting_numpy()
    try:
        s = wrap(s)
        mo.fill_ghosts(s, G, par.bc)
        Counter.flops = Counter.trans = 0
        mo.compute(s, G, par, dt, 0.4)  # one step's work on filled ghosts
        return Counter.flops / n ** 3, Counter.trans / n ** 3
    finally:
        mo.np = np


def count_ced(n, order):
    from oracle import ced_oracle as co
    from paper_2211_13295_b200 import ced
    g = ced.make_geometry(n, n, n, order, (0, 0, 0), (1, 1, 1))
    s = ced.plane_wave(g)
    G = co.Geom(n, n, n, order, (0, 0, 0), (1, 1, 1))
    par = co.Params(order)
    dt = 0.4 * g.dx
    x = (np.arange(g.mx + 1) - g.ghost + 0.5) * g.dx
    sigma = np.zeros((g.mz + 1, g.my + 1, g.mx + 1))
    sigma[:, :, (x > 0.4) & (x < 0.6)] = 1e3 / dt
    co.np = counting_numpy()
    try:
        s, sigma = wrap(s), wrap(sigma)
        co.fill_ghosts(s, sigma, G, par.bc)
        Counter.flops = Counter.trans = 0
        co.step(s, sigma, G, par, dt)
        return Counter.flops / n ** 3, Counter.trans / n ** 3
    finally:
        co.np = np


def fit(ns, fs):
    """F(n) = a + b/n + c/n^2 through three meshes (ring and face overheads scale as 1/n)."""
    A = np.array([[1.0, 1.0 / n, 1.0 / n ** 2] for n in ns])
    return [float(v) for v in np.linalg.solve(A, np.array(fs))]


if __name__ == "__main__":
    ns = [int(v) for v in sys.argv[1:]] or [12, 24, 32]
    out = {"method": __doc__.strip().split("\n\n")[0],
           "model": "flops_per_zone(n) = a + b/n + c/n^2, fitted through the meshes below"}
    for name, fn in (("mhd", count_mhd), ("ced", count_ced)):
        for order in (2, 3):
            fs = [fn(n, order)[0] for n in ns]
            a, b, c = fit(ns, fs)
            out[f"{name}_o{order}"] = {"meshes": ns, "flops_per_zone": fs, "a": a, "b": b, "c": c,
                                       "at_256": a + b / 256 + c / 256 ** 2,
                                       "at_384": a + b / 384 + c / 384 ** 2}
            print(name, order, out[f"{name}_o{order}"])
    with open(os.path.join(ROOT, "profiles", "r2_ext_flops.json"), "w") as fh:
        json.dump(out, fh, indent=1)
