"""mhd -- Python host layer over the ideal-MHD extension of libhydro_cuda.so
(include/hydro_mhd.h): ADER with WENO3/MC reconstruction of the fluid variables, face-centred
B by constrained transport, edge EMFs from the two-dimensional HLL (UCT-HLL) Riemann solver.

EXTENSION without a reference counterpart (the reference is Euler-only): the
state layout, initial conditions and API are this package's own. Initial conditions are
sampled on the host (numpy), face fields from a vector potential so that the discrete
divergence starts at round-off:

* ``mhd_vortex``   -- Balsara (2004) smooth MHD vortex, z-invariant, exact solution = advected
* ``orszag_tang``  -- Orszag-Tang vortex (z-invariant), the BASELINE.json config-3 problem
* ``random_field`` -- a fully 3D periodic test: random Fourier vector potential and velocity

No CPU fallback: every compute call goes to the sm_100a kernels or raises.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import hydro
from .hydro import Geom, Limiter, _check, _p, default_limiter, load_library

NM = 8
PERIODIC, OUTFLOW = hydro.PERIODIC, hydro.OUTFLOW


class MhdParams(C.Structure):
    _fields_ = [("order", C.c_int), ("gamma", C.c_double), ("lim", Limiter),
                ("bc", C.c_int * 3), ("device", C.c_int), ("face_solver", C.c_int)]


HLL, HLLD = 0, 1  # HC_MHD_HLL / HC_MHD_HLLD: face solver of the fluid fluxes


def make_params(order, gamma=5.0 / 3.0, bc=(PERIODIC,) * 3, device=0, limiter=None,
                face_solver=HLL):
    p = MhdParams()
    p.order, p.gamma, p.device, p.face_solver = order, gamma, device, face_solver
    p.lim = limiter or default_limiter()
    for d in range(3):
        p.bc[d] = bc[d]
    return p


def state_shape(g: Geom):
    return (NM, g.mz + 1, g.my + 1, g.mx + 1)


def _lib():
    lib = load_library()
    if not getattr(lib, "_mhd_typed", False):
        lib.hc_mhd_launches.restype = C.c_long
        lib.hc_mhd_launches.argtypes = [C.c_void_p]
        for n in ("hc_mhd_destroy", "hc_mhd_fill_ghosts", "hc_mhd_compute", "hc_mhd_advance",
                  "hc_mhd_finish"):
            getattr(lib, n).argtypes = [C.c_void_p]
        lib.hc_mhd_step.argtypes = [C.c_void_p, C.c_int]
        lib.hc_mhd_compute_range.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib._mhd_typed = True
    return lib


class MhdStepper:
    """Device-resident ADER-CT stepper (state in HBM across steps)."""

    def __init__(self, g: Geom, p: MhdParams):
        self.lib = _lib()
        self.g, self.p = g, p
        h = C.c_void_p()
        _check(self.lib.hc_mhd_create(C.byref(g), C.byref(p), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.hc_mhd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, s):
        s = np.ascontiguousarray(s, dtype=np.float64)
        assert s.shape == state_shape(self.g), (s.shape, state_shape(self.g))
        _check(self.lib.hc_mhd_upload(self.h, _p(s)))

    def download(self, out=None):
        """the device state; into `out` (e.g. a pinned buffer) when given"""
        if out is None:
            out = np.empty(state_shape(self.g))
        assert out.shape == state_shape(self.g) and out.dtype == np.float64
        assert out.flags.c_contiguous
        _check(self.lib.hc_mhd_download(self.h, _p(out)))
        return out

    def set_time(self, t, dt, cfl, t_final=0.0):
        _check(self.lib.hc_mhd_set_time(self.h, C.c_double(t), C.c_double(dt), C.c_double(cfl),
                                        C.c_double(t_final)))

    def step(self, n=1):
        _check(self.lib.hc_mhd_step(self.h, n))

    def sync(self):
        t, dt, n = C.c_double(), C.c_double(), C.c_long()
        _check(self.lib.hc_mhd_sync(self.h, C.byref(t), C.byref(dt), C.byref(n)))
        return t.value, dt.value, n.value

    def cfl_dt(self, cfl):
        d = C.c_double()
        _check(self.lib.hc_mhd_cfl_dt(self.h, C.c_double(cfl), C.byref(d)))
        return d.value

    def max_divb(self):
        d = C.c_double()
        _check(self.lib.hc_mhd_max_divb(self.h, C.byref(d)))
        return d.value

    @property
    def launches(self):
        return self.lib.hc_mhd_launches(self.h)

    @property
    def floored(self):
        """zone updates the pressure floor touched so far (hc_mhd_floored)"""
        v = C.c_ulonglong()
        _check(self.lib.hc_mhd_floored(self.h, C.byref(v)))
        return v.value

    def set_stream(self, ptr):
        _check(self.lib.hc_mhd_set_stream(self.h, C.c_void_p(ptr)))

    def fill_ghosts(self):
        _check(self.lib.hc_mhd_fill_ghosts(self.h))

    def compute(self):
        _check(self.lib.hc_mhd_compute(self.h))

    def compute_range(self, zlo, zhi):
        """front kernels for the active z planes [zlo, zhi) (hc_mhd_compute_range)"""
        _check(self.lib.hc_mhd_compute_range(self.h, zlo, zhi))

    def finish(self):
        _check(self.lib.hc_mhd_finish(self.h))

    def advance(self):
        _check(self.lib.hc_mhd_advance(self.h))

    def state_ptr(self):
        p, vs, pe = C.c_void_p(), C.c_size_t(), C.c_size_t()
        _check(self.lib.hc_mhd_state(self.h, C.byref(p), C.byref(vs), C.byref(pe)))
        return p.value, vs.value, pe.value

    def dt_acc_ptr(self):
        p = C.c_void_p()
        _check(self.lib.hc_mhd_dt_acc(self.h, C.byref(p)))
        return p.value

    @property
    def stream_ptr(self):
        v = C.c_void_p()
        _check(self.lib.hc_mhd_stream(self.h, C.byref(v)))
        return v.value or 0

    def run(self, cfl, t_final=0.0, nsteps=None, max_steps=100000):
        """harness.cpp:155-170 loop on the device: dt from the CFL min of the state, then steps
        until t_final (device-side clip) or nsteps."""
        dt0 = self.cfl_dt(cfl)
        if t_final > 0.0:
            dt0 = min(dt0, t_final)
        self.set_time(0.0, dt0, cfl, t_final)
        if nsteps is not None:
            self.step(nsteps)
            return self.sync()
        done = 0
        while done < max_steps:
            self.step(32)
            t, dt, done = self.sync()
            if t_final > 0.0 and t >= t_final * (1 - 1e-12):
                return t, dt, done
        raise RuntimeError("t_final not reached")


# ------------------------------------------------------------------ initial conditions

def ghost_for_order(order):
    """order 2: MC radius 1 + ring; order 3: WENO3 radius 2 + ring + the fourth-order cell
    average of B (faces one further out)"""
    return 2 if order == 2 else 4


def make_geometry(nx, ny, nz, order, lo, hi) -> Geom:
    g = hydro.make_geometry(nx, ny, nz, order, lo=lo, hi=hi)
    g.ghost = ghost_for_order(order)
    return g


def _coords(g: Geom, axis, shift):
    """coordinate of storage index c (+ shift in zone units) along axis, for every storage
    index 0..m (the padded box)"""
    m = (g.mx, g.my, g.mz)[axis] + 1
    d = (g.dx, g.dy, g.dz)[axis]
    c = np.arange(m)
    return g.origin[axis] + (c - g.ghost + 0.5 + shift) * d


def _gauss(order):
    """quadrature nodes/weights on [-1/2, 1/2] (midpoint at order 2, 2-point Gauss at 3), the
    reference's zone-average sampling (problems.cpp:44-76)"""
    if order == 2:
        return [0.0], [1.0]
    a = 0.5 / math.sqrt(3.0)
    return [-a, a], [0.5, 0.5]


def _cells_from_point(g: Geom, order, point_fn, z_invariant=True):
    """cell averages (5 conserved) of point_fn(x, y, z) -> (rho, vx, vy, vz, p, bx, by, bz)
    with the cell B taken from the pointwise field (energy includes B^2/2)"""
    nodes, wts = _gauss(order)
    shape = (g.mz + 1, g.my + 1, g.mx + 1)
    out = np.zeros((5,) + shape)
    zn = [(0.0, 1.0)] if z_invariant else list(zip(nodes, wts))
    for nx_, wx in zip(nodes, wts):
        for ny_, wy in zip(nodes, wts):
            for nz_, wz in zn:
                x = _coords(g, 0, nx_)[None, None, :]
                y = _coords(g, 1, ny_)[None, :, None]
                z = _coords(g, 2, nz_)[:, None, None]
                rho, vx, vy, vz, p, bx, by, bz, gam = point_fn(x, y, z)
                e = p / (gam - 1.0) + 0.5 * rho * (vx * vx + vy * vy + vz * vz) + \
                    0.5 * (bx * bx + by * by + bz * bz)
                w = wx * wy * wz
                for q, v in enumerate((rho, rho * vx, rho * vy, rho * vz, e)):
                    out[q] = out[q] + w * np.broadcast_to(v, shape)
    return out


def _faces_from_potential(g: Geom, ax_fn, ay_fn, az_fn):
    """face fields = discrete curl of the vector potential sampled at edge centres:
    bx(i-1/2,j,k) = (Az(i-1/2,j+1/2,k) - Az(i-1/2,j-1/2,k))/dy - (Ay(i-1/2,j,k+1/2) - Ay(..,k-1/2))/dz
    (and cyclic), so the discrete divergence is zero to round-off."""
    shape = (g.mz + 1, g.my + 1, g.mx + 1)
    xc, yc, zc = _coords(g, 0, 0.0), _coords(g, 1, 0.0), _coords(g, 2, 0.0)
    xf, yf, zf = _coords(g, 0, -0.5), _coords(g, 1, -0.5), _coords(g, 2, -0.5)

    def grid(x, y, z):
        return x[None, None, :], y[None, :, None], z[:, None, None]

    def ev(fn, x, y, z):
        return np.broadcast_to(fn(*grid(x, y, z)), shape).astype(np.float64)
    # edge-centred potentials; their "+1" neighbours via the next index along the axis
    az_e = ev(az_fn, xf, yf, zc)      # Az at (i-1/2, j-1/2, k)
    ay_e = ev(ay_fn, xf, yc, zf)      # Ay at (i-1/2, j, k-1/2)
    ax_e = ev(ax_fn, xc, yf, zf)      # Ax at (i, j-1/2, k-1/2)
    az_n = ev(az_fn, xf, yf + g.dy, zc)  # Az at (i-1/2, j+1/2, k)
    ay_n = ev(ay_fn, xf, yc, zf + g.dz)  # Ay at (i-1/2, j, k+1/2)
    ax_zn = ev(ax_fn, xc, yf, zf + g.dz)  # Ax at (i, j-1/2, k+1/2)
    az_xn = ev(az_fn, xf + g.dx, yf, zc)  # Az at (i+1/2, j-1/2, k)
    ay_xn = ev(ay_fn, xf + g.dx, yc, zf)  # Ay at (i+1/2, j, k-1/2)
    ax_yn = ev(ax_fn, xc, yf + g.dy, zf)  # Ax at (i, j+1/2, k-1/2)
    bx = (az_n - az_e) / g.dy - (ay_n - ay_e) / g.dz
    by = (ax_zn - ax_e) / g.dz - (az_xn - az_e) / g.dx
    bz = (ay_xn - ay_e) / g.dx - (ax_yn - ax_e) / g.dy
    return bx, by, bz


def mhd_vortex(g: Geom, order, t=0.0, gamma=5.0 / 3.0, kappa=1.0, mu=1.0, u0=(1.0, 1.0)):
    """Balsara (2004) MHD vortex on [-5,5]^2 (z-invariant), advected by u0; the exact solution
    at time t is the initial one shifted by u0 t (periodic)."""
    L = 10.0

    def rel(x, y):
        dx = np.mod(x - u0[0] * t + 5.0, L) - 5.0
        dy = np.mod(y - u0[1] * t + 5.0, L) - 5.0
        return dx, dy

    def point(x, y, z):
        dx, dy = rel(x, y)
        r2 = dx * dx + dy * dy
        e = np.exp(0.5 * (1.0 - r2))
        vx = u0[0] - kappa / (2 * math.pi) * e * dy
        vy = u0[1] + kappa / (2 * math.pi) * e * dx
        bx = -mu / (2 * math.pi) * e * dy
        by = mu / (2 * math.pi) * e * dx
        p = 1.0 + (mu * mu * (1.0 - r2) - kappa * kappa) * e * e / (8 * math.pi ** 2)
        zero = 0.0 * r2
        return 1.0 + zero, vx, vy, zero, p, bx, by, zero, gamma

    def az(x, y, z):
        dx, dy = rel(x, y)
        return mu / (2 * math.pi) * np.exp(0.5 * (1.0 - (dx * dx + dy * dy))) + 0.0 * z

    def zero(x, y, z):
        return 0.0 * (x + y + z)

    s = np.zeros(state_shape(g))
    s[:5] = _cells_from_point(g, order, point)
    s[5], s[6], s[7] = _faces_from_potential(g, zero, zero, az)
    return s


def orszag_tang(g: Geom, order, gamma=5.0 / 3.0):
    """Orszag-Tang on [0,1]^2 (z-invariant): rho = 25/(36 pi), p = 5/(12 pi),
    v = (-sin 2 pi y, sin 2 pi x, 0), B = B0 (-sin 2 pi y, sin 4 pi x, 0), B0 = 1/sqrt(4 pi)."""
    b0 = 1.0 / math.sqrt(4 * math.pi)
    tp = 2 * math.pi

    def point(x, y, z):
        zero = 0.0 * (x + y + z)
        return (25.0 / (36 * math.pi) + zero, -np.sin(tp * y) + zero, np.sin(tp * x) + zero, zero,
                5.0 / (12 * math.pi) + zero, -b0 * np.sin(tp * y) + zero,
                b0 * np.sin(2 * tp * x) + zero, zero, gamma)

    def az(x, y, z):
        return b0 * (np.cos(2 * tp * x) / (2 * tp) + np.cos(tp * y) / tp) + 0.0 * z

    def zero(x, y, z):
        return 0.0 * (x + y + z)

    s = np.zeros(state_shape(g))
    s[:5] = _cells_from_point(g, order, point)
    s[5], s[6], s[7] = _faces_from_potential(g, zero, zero, az)
    return s


def random_field(g: Geom, order, seed=3, gamma=5.0 / 3.0, amp=0.3, modes=4):
    """Fully 3D periodic test on [0,1]^3: uniform rho, p; random Fourier velocity and vector
    potential with integer wave vectors (periodic), B = curl A (discretely)."""
    r = np.random.default_rng(seed)
    ks = r.integers(-2, 3, size=(modes, 3))
    ks[np.all(ks == 0, axis=1)] = (1, 1, 1)
    ph = r.uniform(0, 2 * math.pi, size=(modes, 3))
    av = r.uniform(-1, 1, size=(modes, 3)) * amp
    aa = r.uniform(-1, 1, size=(modes, 3)) * amp / (2 * math.pi)

    def fourier(coef, comp):
        def f(x, y, z):
            v = 0.0 * (x + y + z)
            for m in range(modes):
                v = v + coef[m, comp] * np.sin(2 * math.pi * (ks[m, 0] * x + ks[m, 1] * y +
                                                              ks[m, 2] * z) + ph[m, comp])
            return v
        return f

    vfun = [fourier(av, c) for c in range(3)]
    afun = [fourier(aa, c) for c in range(3)]

    def point(x, y, z):
        zero = 0.0 * (x + y + z)
        # cell B for the energy: the analytic curl of A
        bx = zero.copy()
        by = zero.copy()
        bz = zero.copy()
        for m in range(modes):
            arg = [2 * math.pi * (ks[m, 0] * x + ks[m, 1] * y + ks[m, 2] * z) + ph[m, c]
                   for c in range(3)]
            dA = [aa[m, c] * np.cos(arg[c]) * 2 * math.pi for c in range(3)]
            bx = bx + dA[2] * ks[m, 1] - dA[1] * ks[m, 2]
            by = by + dA[0] * ks[m, 2] - dA[2] * ks[m, 0]
            bz = bz + dA[1] * ks[m, 0] - dA[0] * ks[m, 1]
        return (1.0 + zero, vfun[0](x, y, z), vfun[1](x, y, z), vfun[2](x, y, z), 1.0 + zero,
                bx, by, bz, gamma)

    s = np.zeros(state_shape(g))
    s[:5] = _cells_from_point(g, order, point, z_invariant=False)
    s[5], s[6], s[7] = _faces_from_potential(g, afun[0], afun[1], afun[2])
    return s


def rotor(g: Geom, order, gamma=1.4):
    """Balsara & Spicer (1999) MHD rotor on [0,1]^2 (z-invariant): a dense (rho = 10) disk of
    radius 0.1 spinning at omega = 20 in a light (rho = 1) medium at rest, tapered linearly to
    r = 0.115; p = 1, B = (5 / sqrt(4 pi), 0, 0) uniform (a constant Bx from Az = B0 y)."""
    r0, r1, w0 = 0.1, 0.115, 20.0
    b0 = 5.0 / math.sqrt(4 * math.pi)

    def point(x, y, z):
        dx, dy = x - 0.5, y - 0.5
        r = np.sqrt(dx * dx + dy * dy) + 0.0 * z
        f = np.clip((r1 - r) / (r1 - r0), 0.0, 1.0)
        inside = r < r0
        rho = np.where(inside, 10.0, 1.0 + 9.0 * f)
        fac = np.where(inside, 1.0, f * r0 / np.maximum(r, 1e-300))
        vx = -w0 * dy * fac
        vy = w0 * dx * fac
        zero = 0.0 * r
        return rho, vx, vy, zero, 1.0 + zero, b0 + zero, zero, zero, gamma

    def az(x, y, z):
        return -b0 * y + 0.0 * (x + z)  # Bx = dAz/dy ... sign: bx = (Az(y+) - Az(y-))/dy

    def zero(x, y, z):
        return 0.0 * (x + y + z)

    s = np.zeros(state_shape(g))
    s[:5] = _cells_from_point(g, order, point)
    s[5], s[6], s[7] = _faces_from_potential(g, zero, zero, lambda x, y, zz: b0 * y + 0.0 * (x + zz))
    return s
