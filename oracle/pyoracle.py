"""pyoracle -- TEST INFRASTRUCTURE ONLY (ctypes bindings to the checkers).

Binds two CPU libraries with identical flat signatures:
  * ``oracle/liboracle.so``          -- the plain-C restatement (prefix ``or_``)
  * ``oracle/_ref/libhydro_ref.so``  -- the reference library built from its own sources by
                                        ``oracle/Makefile`` plus the ``ref_capi.cpp`` adapter
                                        (prefix ``ref_``); present only where it was built.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhydro_ref.so")

NVAR = 5
RUSANOV, HLL, HLLC, HLLI = 0, 1, 2, 3  # HLLC/HLLI: builder-authored extensions (parity unpinned)
PERIODIC, OUTFLOW = 0, 1


class Geom(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("ghost", C.c_int),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("origin", C.c_double * 3)]

    @property
    def mx(self):
        return self.nx + 2 * self.ghost

    @property
    def my(self):
        return self.ny + 2 * self.ghost

    @property
    def mz(self):
        return self.nz + 2 * self.ghost


class Limiter(C.Structure):
    _fields_ = [("cfac_rho", C.c_double), ("cfac_other", C.c_double),
                ("weno_eps", C.c_double), ("weno_w", C.c_double * 3)]


class Params(C.Structure):
    _fields_ = [("order", C.c_int), ("solver", C.c_int), ("gamma", C.c_double),
                ("lim", Limiter)]


def default_limiter() -> Limiter:
    """LimiterConfig defaults, reconstruct.hpp:11-15."""
    lim = Limiter()
    lim.cfac_rho, lim.cfac_other, lim.weno_eps = 2.0, 1.5, 1e-12
    lim.weno_w[0], lim.weno_w[1], lim.weno_w[2] = 0.25, 0.5, 0.25
    return lim


def make_geometry(nx, ny, nz, order, lo=(-5.0, -5.0, -5.0), hi=(5.0, 5.0, 5.0)) -> Geom:
    """geometry.hpp:67-80 make_geometry."""
    g = Geom()
    g.nx, g.ny, g.nz = nx, ny, nz
    g.ghost = {2: 2, 3: 3, 4: 3}[order]  # 4: the WENO-AO extension (radius 2, like O3)
    g.dx = (hi[0] - lo[0]) / nx
    g.dy = (hi[1] - lo[1]) / ny
    g.dz = (hi[2] - lo[2]) / nz
    for a in range(3):
        g.origin[a] = lo[a]
    return g


def make_params(order, solver=HLL, gamma=1.4) -> Params:
    p = Params()
    p.order, p.solver, p.gamma = order, solver, gamma
    p.lim = default_limiter()
    return p


def modes_for_order(order):
    return {2: 5, 3: 11, 4: 14}[order]


def zeros_skinny(g):
    return np.zeros((g.mz, g.my, g.mx, NVAR))


def zeros_modal(g, order):
    return np.zeros((g.mz, g.my, g.mx, NVAR, modes_for_order(order)))


def zeros_faces(g):
    return (np.zeros((g.nz, g.ny, g.nx + 1, NVAR)), np.zeros((g.nz, g.nx, g.ny + 1, NVAR)),
            np.zeros((g.ny, g.nx, g.nz + 1, NVAR)))


def zeros_rate(g):
    return np.zeros((g.nz, g.ny, g.nx, NVAR))


def _p(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


class CpuLib:
    """One of the two checkers; ``prefix`` is 'or_' (restatement) or 'ref_' (reference)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.last_error.restype = C.c_char_p
        self._fn("mc_limiter").restype = C.c_double
        for name in ("mc_limiter",):
            self._fn(name).argtypes = [C.c_double, C.c_double, C.c_double]

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def __getattr__(self, name):
        return getattr(self.lib, self.prefix + name)

    def error(self) -> str:
        return self.last_error().decode()

    def _rc(self, rc):
        if rc == 1:
            raise UnphysicalError(self.error())
        if rc == 2:
            raise ValueError(self.error())

    # ---- pointwise
    def hll_flux(self, ul, ur, axis, gamma=1.4):
        f = np.zeros(5)
        self._rc(self._fn("hll_flux")(_p(np.ascontiguousarray(ul, float)),
                                      _p(np.ascontiguousarray(ur, float)), axis,
                                      C.c_double(gamma), _p(f)))
        return f

    def hllc_flux(self, ul, ur, axis, gamma=1.4):
        """Builder-authored HLLC restatement (no reference counterpart; parity unpinned)."""
        f = np.zeros(5)
        self._rc(self._fn("hllc_flux")(_p(np.ascontiguousarray(ul, float)),
                                       _p(np.ascontiguousarray(ur, float)), axis,
                                       C.c_double(gamma), _p(f)))
        return f

    def hlli_flux(self, ul, ur, axis, gamma=1.4):
        """Builder-authored HLLI restatement (no reference counterpart; parity unpinned)."""
        f = np.zeros(5)
        self._rc(self._fn("hlli_flux")(_p(np.ascontiguousarray(ul, float)),
                                       _p(np.ascontiguousarray(ur, float)), axis,
                                       C.c_double(gamma), _p(f)))
        return f

    def rusanov_flux(self, ul, ur, axis, gamma=1.4):
        f = np.zeros(5)
        self._rc(self._fn("rusanov_flux")(_p(np.ascontiguousarray(ul, float)),
                                          _p(np.ascontiguousarray(ur, float)), axis,
                                          C.c_double(gamma), _p(f)))
        return f

    def eval_tstep_ptwise(self, u, cfl, dx, dy, dz, gamma=1.4):
        d = C.c_double()
        self._rc(self._fn("eval_tstep_ptwise")(_p(np.ascontiguousarray(u, float)),
                                               C.c_double(cfl), C.c_double(dx), C.c_double(dy),
                                               C.c_double(dz), C.c_double(gamma), C.byref(d)))
        return d.value

    def weno3_point(self, s, lim=None):
        lim = lim or default_limiter()
        ux, uxx = C.c_double(), C.c_double()
        self._fn("weno3_point")(_p(np.ascontiguousarray(s, float)), C.byref(lim), C.byref(ux),
                                C.byref(uxx))
        return ux.value, uxx.value

    def predictor_ptwise(self, zone, modes, dt, dx, dy, dz, gamma=1.4):
        z = np.ascontiguousarray(zone, float).copy()
        self._rc(self._fn("predictor_ptwise")(_p(z), modes, C.c_double(dt), C.c_double(dx),
                                              C.c_double(dy), C.c_double(dz),
                                              C.c_double(gamma)))
        return z

    # ---- patch kernels (in place on numpy arrays, reference layouts)
    def apply_boundary_skinny(self, g, kind, skinny):
        self._fn("apply_boundary_skinny")(C.byref(g), kind, _p(skinny))

    def apply_boundary_modal(self, g, modes, kind, modal):
        self._fn("apply_boundary_modal")(C.byref(g), modes, kind, _p(modal))

    def skinny_to_modal(self, g, modes, skinny, modal):
        self._fn("skinny_to_modal")(C.byref(g), modes, _p(skinny), _p(modal))

    def modal_to_skinny(self, g, modes, modal, skinny):
        self._fn("modal_to_skinny")(C.byref(g), modes, _p(modal), _p(skinny))

    def limit_patch_o2(self, g, modal, lim=None):
        self._fn("limit_patch_o2")(C.byref(g), _p(modal), C.byref(lim or default_limiter()))

    def reconstruct_patch_o3(self, g, modal, lim=None):
        self._fn("reconstruct_patch_o3")(C.byref(g), _p(modal),
                                         C.byref(lim or default_limiter()))

    def predict_patch(self, g, modes, modal, dt, gamma=1.4):
        self._rc(self._fn("predict_patch")(C.byref(g), modes, _p(modal), C.c_double(dt),
                                           C.c_double(gamma)))

    def zero_temporal_mode(self, g, modes, modal):
        self._fn("zero_temporal_mode")(C.byref(g), modes, _p(modal))

    def make_flux_axis(self, g, modes, modal, axis, solver, out, gamma=1.4):
        self._rc(self._fn("make_flux_axis")(C.byref(g), modes, _p(modal), axis,
                                            C.c_double(gamma), solver, _p(out)))

    def make_du_dt(self, g, fx, fy, fz, dt, rate):
        self._fn("make_du_dt")(C.byref(g), _p(fx), _p(fy), _p(fz), C.c_double(dt), _p(rate))

    def update_u_timestep(self, g, modes, modal, skinny, rate, cfl, gamma=1.4):
        d = C.c_double()
        self._rc(self._fn("update_u_timestep")(C.byref(g), modes, _p(modal), _p(skinny),
                                               _p(rate), C.c_double(cfl), C.c_double(gamma),
                                               C.byref(d)))
        return d.value

    def compute_dt_next(self, g, modes, modal, cfl, gamma=1.4):
        d = C.c_double()
        self._rc(self._fn("compute_dt_next")(C.byref(g), modes, _p(modal), C.c_double(gamma),
                                             C.c_double(cfl), C.byref(d)))
        return d.value

    def ader_step(self, g, par, modal, skinny, fx, fy, fz, rate, dt, cfl):
        d = C.c_double()
        self._rc(self._fn("ader_step")(C.byref(g), C.byref(par), _p(modal), _p(skinny), _p(fx),
                                       _p(fy), _p(fz), _p(rate), C.c_double(dt),
                                       C.c_double(cfl), C.byref(d)))
        return d.value

    def rk_step(self, g, par, nstages, modal, skinny, fx, fy, fz, rate, u0, bc, dt, cfl):
        d = C.c_double()
        self._rc(self._fn("rk_step")(C.byref(g), C.byref(par), nstages, _p(modal), _p(skinny),
                                     _p(fx), _p(fy), _p(fz), _p(rate), _p(u0), bc,
                                     C.c_double(dt), C.c_double(cfl), C.byref(d)))
        return d.value

    def init_isentropic_vortex(self, g, order, t=0.0, gamma=1.4):
        s = zeros_skinny(g)
        self._fn("init_isentropic_vortex")(C.byref(g), C.c_double(gamma), order,
                                           C.c_double(t), _p(s))
        return s

    def init_sod(self, g, gamma=1.4):
        s = zeros_skinny(g)
        self._fn("init_sod")(C.byref(g), C.c_double(gamma), _p(s))
        return s

    def init_constant(self, g, gamma=1.4):
        s = zeros_skinny(g)
        self._fn("init_constant")(C.byref(g), C.c_double(gamma), _p(s))
        return s


class UnphysicalError(RuntimeError):
    """Mirrors hydro::unphysical_error (euler.hpp:33-35)."""


class Oracle(CpuLib):
    """The plain-C restatement (always built by __graft_entry__.build())."""

    def __init__(self):
        super().__init__(ORACLE_SO, "or_")
        self.lib.or_initial_dt.restype = C.c_double

    def initial_dt(self, g, skinny, cfl, gamma=1.4):
        return self.lib.or_initial_dt(C.byref(g), _p(skinny), C.c_double(gamma),
                                      C.c_double(cfl))

    def run_steps(self, g, par, bc, cfl, steps, skinny, dt0):
        """ADER steps with apply_boundary before each; returns the dt sequence."""
        dts = np.zeros(steps + 1)
        dts[0] = dt0
        self._rc(self.lib.or_run_steps(C.byref(g), C.byref(par), bc, C.c_double(cfl), steps,
                                       _p(skinny), _p(dts)))
        return dts


class Reference(CpuLib):
    """The reference library itself (oracle/_ref), where it was built."""

    def __init__(self):
        super().__init__(REF_SO, "ref_")
        self.lib.ref_run_benchmark.restype = C.c_double
        self.lib.ref_run_benchmark.argtypes = [C.c_int] * 10 + [C.c_long, C.c_int] + [
            C.c_void_p] * 3

    def set_threads(self, n):
        self.lib.ref_set_threads(n)

    def run_benchmark(self, problem, order, integrator, solver, n, steps, threads=0,
                      split=(1, 1, 1), want_state=False):
        nx, ny, nz = (n, n, n) if isinstance(n, int) else n
        g = make_geometry(nx, ny, nz, order)
        fin = zeros_skinny(g) if want_state else None
        t_end = C.c_double()
        l1 = C.c_double()
        zps = self.lib.ref_run_benchmark(problem, order, integrator, solver, nx, ny, nz,
                                         split[0], split[1], split[2], steps, threads,
                                         fin.ctypes.data if fin is not None else None,
                                         C.addressof(t_end), C.addressof(l1))
        if zps < 0:
            raise RuntimeError(self.error())
        return zps, fin, t_end.value, l1.value


def ref_run_simulation(ref, problem, order, integrator, solver, n, steps=0, t_final=-1.0,
                       threads=0):
    """harness.cpp run_simulation through the reference library: (l1, linf, t_end, steps)."""
    l1, linf = np.zeros(5), np.zeros(5)
    t_end, nst = C.c_double(), C.c_long()
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    f = ref.lib.ref_run_simulation
    f.argtypes = [C.c_int] * 7 + [C.c_long, C.c_double, C.c_int] + [C.c_void_p] * 5
    rc = f(problem, order, integrator, solver, nx, ny, nz, steps, t_final, threads,
           l1.ctypes.data, linf.ctypes.data, C.addressof(t_end), C.addressof(nst), None)
    if rc:
        raise RuntimeError(ref.error())
    return l1, linf, t_end.value, nst.value


def have_reference() -> bool:
    return os.path.exists(REF_SO)
