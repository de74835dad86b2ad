"""ced -- Python host layer over the CED extension of libhydro_cuda.so (include/hydro_ced.h):
Maxwell's equations in a conducting medium (face-centred D, B by constrained transport, 2D
upwind edge solver, WENO3/MC-ADER predictor, conduction source by an L-stable exponential
step). EXTENSION without a reference counterpart.

Initial data (host, numpy), face fields from edge-AVERAGED vector potentials so that they
are exact face averages and discretely divergence-free:

* ``plane_wave``    -- vacuum (or dielectric) plane wave, exact solution at any t
* ``uniform_field`` -- spatially uniform D in a uniform conductor: D(t) = D0 exp(-sigma t/eps)
* ``diffusion_mode``-- B_z = B0 sin(2 pi x) in a good conductor: the slow (diffusive) mode
                       decays at lambda = (-s + sqrt(s^2 - 4 c^2 k^2)) / 2, s = sigma/eps

No CPU fallback: every compute call goes to the sm_100a kernels or raises.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import hydro
from .hydro import Geom, Limiter, _check, _p, default_limiter, load_library
from .mhd import _coords

NF = 6
PERIODIC, OUTFLOW = hydro.PERIODIC, hydro.OUTFLOW


class CedParams(C.Structure):
    _fields_ = [("order", C.c_int), ("eps", C.c_double), ("mu", C.c_double), ("lim", Limiter),
                ("bc", C.c_int * 3), ("device", C.c_int)]


def make_params(order, eps=1.0, mu=1.0, bc=(PERIODIC,) * 3, device=0, limiter=None):
    p = CedParams()
    p.order, p.eps, p.mu, p.device = order, eps, mu, device
    p.lim = limiter or default_limiter()
    for d in range(3):
        p.bc[d] = bc[d]
    return p


def ghost_for_order(order):
    return 2 if order == 2 else 4


def make_geometry(nx, ny, nz, order, lo, hi) -> Geom:
    g = hydro.make_geometry(nx, ny, nz, order, lo=lo, hi=hi)
    g.ghost = ghost_for_order(order)
    return g


def box_shape(g: Geom):
    return (g.mz + 1, g.my + 1, g.mx + 1)


def _lib():
    lib = load_library()
    if not getattr(lib, "_ced_typed", False):
        lib.hc_ced_launches.restype = C.c_long
        lib.hc_ced_launches.argtypes = [C.c_void_p]
        lib.hc_ced_destroy.argtypes = [C.c_void_p]
        lib.hc_ced_step.argtypes = [C.c_void_p, C.c_int]
        lib._ced_typed = True
    return lib


class CedStepper:
    def __init__(self, g: Geom, p: CedParams):
        self.lib = _lib()
        self.g, self.p = g, p
        h = C.c_void_p()
        _check(self.lib.hc_ced_create(C.byref(g), C.byref(p), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.hc_ced_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, s, sigma):
        s = np.ascontiguousarray(s, dtype=np.float64)
        sigma = np.ascontiguousarray(np.broadcast_to(sigma, box_shape(self.g)), dtype=np.float64)
        assert s.shape == (NF,) + box_shape(self.g)
        _check(self.lib.hc_ced_upload(self.h, _p(s), _p(sigma)))

    def download(self, out=None):
        """the device state; into `out` (e.g. a pinned buffer) when given"""
        if out is None:
            out = np.empty((NF,) + box_shape(self.g))
        assert out.shape == (NF,) + box_shape(self.g) and out.dtype == np.float64
        assert out.flags.c_contiguous
        _check(self.lib.hc_ced_download(self.h, _p(out)))
        return out

    def cfl_dt(self, cfl):
        d = C.c_double()
        _check(self.lib.hc_ced_cfl_dt(self.h, C.c_double(cfl), C.byref(d)))
        return d.value

    def set_time(self, t, dt, t_final=0.0):
        _check(self.lib.hc_ced_set_time(self.h, C.c_double(t), C.c_double(dt),
                                        C.c_double(t_final)))

    def step(self, n=1):
        _check(self.lib.hc_ced_step(self.h, n))

    def sync(self):
        t, dt, n = C.c_double(), C.c_double(), C.c_long()
        _check(self.lib.hc_ced_sync(self.h, C.byref(t), C.byref(dt), C.byref(n)))
        return t.value, dt.value, n.value

    def max_div(self):
        b, d = C.c_double(), C.c_double()
        _check(self.lib.hc_ced_max_div(self.h, C.byref(b), C.byref(d)))
        return b.value, d.value

    @property
    def launches(self):
        return self.lib.hc_ced_launches(self.h)

    @property
    def stream_ptr(self):
        v = C.c_void_p()
        _check(self.lib.hc_ced_stream(self.h, C.byref(v)))
        return v.value or 0

    def run(self, cfl, t_final, chunk=64):
        dt = self.cfl_dt(cfl)
        self.set_time(0.0, dt, t_final)
        while True:
            self.step(chunk)
            t, _, n = self.sync()
            if t >= t_final * (1 - 1e-12):
                return t, n


# ------------------------------------------------------------------ initial conditions

def _faces_from_edge_potential(g: Geom, afun):
    """face fields = discrete curl of the edge values afun[c](x, y, z) (edge-centred points of
    the c-edges; pass edge AVERAGES for exact face averages): discretely div-free"""
    shape = box_shape(g)
    xc, yc, zc = _coords(g, 0, 0.0), _coords(g, 1, 0.0), _coords(g, 2, 0.0)
    xf, yf, zf = _coords(g, 0, -0.5), _coords(g, 1, -0.5), _coords(g, 2, -0.5)

    def ev(fn, x, y, z):
        return np.broadcast_to(fn(x[None, None, :], y[None, :, None], z[:, None, None]),
                               shape).astype(np.float64)
    ax_fn, ay_fn, az_fn = afun
    az_e, ay_e, ax_e = ev(az_fn, xf, yf, zc), ev(ay_fn, xf, yc, zf), ev(ax_fn, xc, yf, zf)
    bx = (ev(az_fn, xf, yf + g.dy, zc) - az_e) / g.dy - (ev(ay_fn, xf, yc, zf + g.dz) - ay_e) / g.dz
    by = (ev(ax_fn, xc, yf, zf + g.dz) - ax_e) / g.dz - (ev(az_fn, xf + g.dx, yf, zc) - az_e) / g.dx
    bz = (ev(ay_fn, xf + g.dx, yc, zf) - ay_e) / g.dx - (ev(ax_fn, xc, yf + g.dy, zf) - ax_e) / g.dy
    return bx, by, bz


def plane_wave(g: Geom, n=(1, 1, 1), pol=(1.0, -1.0, 0.0), e0=1.0, eps=1.0, mu=1.0, t=0.0,
               L=(1.0, 1.0, 1.0)):
    """E = e0 ehat sin(k.x - w t), D = eps E, B = (k x E)/w, k = 2 pi n / L, w = c |k|; exact
    face averages via edge-averaged potentials (edge average of cos = point value x
    sinc(k_d h_d / 2))"""
    k = np.array([2 * math.pi * n[d] / L[d] for d in range(3)])
    eh = np.array(pol, dtype=float)
    eh = eh - k * (eh @ k) / (k @ k)
    eh = eh / np.linalg.norm(eh)
    c = 1.0 / math.sqrt(eps * mu)
    w = c * np.linalg.norm(k)
    kk = k @ k
    a_d = eps * e0 * np.cross(k, eh) / kk           # D = curl(a_d cos(k.x - w t))
    a_b = -(e0 / w) * eh                            # B = curl(a_b cos(k.x - w t))
    h = (g.dx, g.dy, g.dz)
    sinc = [math.sin(k[d] * h[d] / 2) / (k[d] * h[d] / 2) if k[d] != 0 else 1.0 for d in range(3)]

    def comp(a, cidx):
        def f(x, y, z):
            return a[cidx] * sinc[cidx] * np.cos(k[0] * x + k[1] * y + k[2] * z - w * t)
        return f
    s = np.zeros((NF,) + box_shape(g))
    s[0], s[1], s[2] = _faces_from_edge_potential(g, [comp(a_d, c_) for c_ in range(3)])
    s[3], s[4], s[5] = _faces_from_edge_potential(g, [comp(a_b, c_) for c_ in range(3)])
    return s


def uniform_field(g: Geom, d0=(1.0, -0.5, 0.25)):
    s = np.zeros((NF,) + box_shape(g))
    for q in range(3):
        s[q] = d0[q]
    return s


def diffusion_mode(g: Geom, b0=1.0):
    """B_z = b0 sin(2 pi x) on x in [0, 1] (face averages exact: Bz lives on z-faces, its x
    average over the face is b0 sin(2 pi x_i) sinc(pi dx)), D = 0"""
    s = np.zeros((NF,) + box_shape(g))
    x = _coords(g, 0, 0.0)
    fac = math.sin(math.pi * g.dx) / (math.pi * g.dx)
    s[5] = (b0 * fac * np.sin(2 * math.pi * x))[None, None, :]
    return s
