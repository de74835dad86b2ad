"""hydro -- Python host layer over libhydro_cuda.so (the C ABI in include/hydro_cuda.h).

Mirrors the reference's operator API (proj/include/hydro/*.hpp): the same function names,
argument meaning, layouts and error behaviour, so parity tests read like the reference's own.

* ``HostApi`` -- one method per hydro:: kernel on HOST numpy arrays in the reference layouts
  (``skinny_to_modal``, ``limit_patch_o2``, ``predict_patch``, ``make_flux_axis``, ...,
  ``ader_step``, ``rk_step``). Each call runs the sm_100a kernels; ``UnphysicalError`` carries
  the reference's message text (``"update: zone (3,2,1): non-positive density ..."``).
* ``Stepper`` -- the device-resident throughput path: U_skinny stays in HBM, one fused kernel
  per ADER step, dt/dt_next hand-off on the device.

There is no CPU fallback: without the built library or a CUDA device every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libhydro_cuda.so")

NVAR = 5
RUSANOV, HLL, HLLC, HLLI = 0, 1, 2, 3  # HLLC, HLLI: extensions (no reference counterpart)
PERIODIC, OUTFLOW = 0, 1
HC_OK, HC_UNPHYSICAL, HC_INVALID, HC_CUDA = 0, 1, 2, 3


class UnphysicalError(RuntimeError):
    """hydro::unphysical_error (euler.hpp:33-35)."""


class HydroCudaError(RuntimeError):
    """A CUDA failure (including: no device -- there is no CPU path)."""


class Geom(C.Structure):
    """hc_geom == PatchGeometry (geometry.hpp:34-65)."""
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
    """hc_limiter == LimiterConfig (reconstruct.hpp:11-29)."""
    _fields_ = [("cfac_rho", C.c_double), ("cfac_other", C.c_double),
                ("weno_eps", C.c_double), ("weno_w", C.c_double * 3)]


class Params(C.Structure):
    """hc_params == StepParams (stepper.hpp:39-45)."""
    _fields_ = [("order", C.c_int), ("solver", C.c_int), ("gamma", C.c_double),
                ("lim", Limiter)]


class StepperOpts(C.Structure):
    _fields_ = [("bc", C.c_int * 3), ("exact", C.c_int), ("device", C.c_int),
                ("integrator", C.c_int)]


ADER, RK2, RK3 = 0, 2, 3  # IntegratorChoice (predictor.hpp:11)


def ghost_for_order(order: int) -> int:
    """geometry.hpp:13-17 (order 4: the WENO-AO extension of the fused stepper, radius 2)."""
    if order == 2:
        return 2
    if order in (3, 4):
        return 3
    raise ValueError(f"unsupported order {order}")


def modes_for_order(order: int) -> int:
    """geometry.hpp:23-27 (order 4: 14 modes in the C restatement, extension)."""
    if order == 2:
        return 5
    if order == 3:
        return 11
    if order == 4:
        return 14
    raise ValueError(f"unsupported order {order}")


def default_limiter() -> Limiter:
    lim = Limiter()
    lim.cfac_rho, lim.cfac_other, lim.weno_eps = 2.0, 1.5, 1e-12
    lim.weno_w[0], lim.weno_w[1], lim.weno_w[2] = 0.25, 0.5, 0.25
    return lim


def make_geometry(nx, ny, nz, order, lo=(-5.0, -5.0, -5.0), hi=(5.0, 5.0, 5.0)) -> Geom:
    """geometry.hpp:67-80 make_geometry (validated by every entry point)."""
    g = Geom()
    g.nx, g.ny, g.nz = nx, ny, nz
    g.ghost = ghost_for_order(order)
    g.dx = (hi[0] - lo[0]) / nx
    g.dy = (hi[1] - lo[1]) / ny
    g.dz = (hi[2] - lo[2]) / nz
    for a in range(3):
        g.origin[a] = lo[a]
    return g


def make_params(order, solver=HLL, gamma=1.4, limiter=None) -> Params:
    p = Params()
    p.order, p.solver, p.gamma = order, solver, gamma
    p.lim = limiter or default_limiter()
    return p


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
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("arrays must be C-contiguous float64")
    return a.ctypes.data_as(C.POINTER(C.c_double))


_LIB = None


def load_library(path: str = LIB_PATH):
    """Loads libhydro_cuda.so; fails loudly when it has not been built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise HydroCudaError(f"{path} is not built (run __graft_entry__.build()); "
                             "there is no CPU fallback")
    lib = C.CDLL(path)
    lib.hc_last_error.argtypes = [C.c_char_p, C.c_size_t]
    lib.hc_stepper_launches.restype = C.c_long
    lib.hc_stepper_launches.argtypes = [C.c_void_p]
    lib.hc_domain_launches.restype = C.c_long
    lib.hc_ader4_launches.restype = C.c_long
    lib.hc_ader4_destroy.argtypes = [C.c_void_p]
    lib.hc_ader4_step.argtypes = [C.c_void_p, C.c_int]
    for name in ("hc_domain_launches", "hc_domain_destroy", "hc_domain_info",
                 "hc_domain_scatter", "hc_domain_gather", "hc_domain_sync"):
        getattr(lib, name).argtypes = None
    lib.hc_domain_launches.argtypes = [C.c_void_p]
    lib.hc_domain_destroy.argtypes = [C.c_void_p]
    lib.hc_domain_step.argtypes = [C.c_void_p, C.c_int]
    for name in ("hc_stepper_destroy", "hc_stepper_step", "hc_stepper_fill_ghosts",
                 "hc_stepper_compute", "hc_stepper_advance", "hc_stepper_stages"):
        getattr(lib, name).argtypes = [C.c_void_p] + ([C.c_int] if name.endswith("_step")
                                                       else [])
    _LIB = lib
    return lib


def exported_symbols():
    """Names declared in include/*.h (checked against the .so by the CPU tests)."""
    import glob
    import re
    txt = ""
    for hdr in sorted(glob.glob(os.path.join(os.path.dirname(PKG), "include", "*.h"))):
        with open(hdr) as f:
            txt += f.read()
    return sorted(set(re.findall(r"^\s*(?:int|long)\s+(hc_[a-z0-9_]+)\s*\(", txt, re.M)))


def _check(rc):
    if rc == HC_OK:
        return
    buf = C.create_string_buffer(1024)
    load_library().hc_last_error(buf, 1024)
    msg = buf.value.decode()
    if rc == HC_UNPHYSICAL:
        raise UnphysicalError(msg)
    if rc == HC_INVALID:
        raise ValueError(msg)
    raise HydroCudaError(msg)


def device_count() -> int:
    return load_library().hc_device_count()


class HostApi:
    """The reference API (hydro:: functions) on host numpy arrays, computed on the GPU.

    Method names and argument order match ``oracle.pyoracle.CpuLib`` so the same parity
    harness drives the product and the checkers."""

    def __init__(self):
        self.lib = load_library()

    # ---- problems (host side, bit-identical to problems.cpp)
    def init_isentropic_vortex(self, g, order, t=0.0, gamma=1.4):
        s = zeros_skinny(g)
        _check(self.lib.hc_init_vortex(C.byref(g), C.c_double(gamma), order, C.c_double(t),
                                       _p(s)))
        return s

    def init_sod(self, g, gamma=1.4):
        s = zeros_skinny(g)
        _check(self.lib.hc_init_sod(C.byref(g), C.c_double(gamma), _p(s)))
        return s

    def init_constant(self, g, gamma=1.4):
        s = zeros_skinny(g)
        _check(self.lib.hc_init_constant(C.byref(g), C.c_double(gamma), _p(s)))
        return s

    def initial_dt(self, g, skinny, cfl, gamma=1.4):
        d = C.c_double()
        _check(self.lib.hc_initial_dt(C.byref(g), _p(skinny), C.c_double(gamma),
                                      C.c_double(cfl), C.byref(d)))
        return d.value

    # ---- patch kernels
    def apply_boundary_skinny(self, g, kind, skinny):
        _check(self.lib.hc_apply_boundary_skinny(C.byref(g), kind, _p(skinny)))

    def apply_boundary_modal(self, g, modes, kind, modal):
        _check(self.lib.hc_apply_boundary_modal(C.byref(g), modes, kind, _p(modal)))

    def skinny_to_modal(self, g, modes, skinny, modal):
        _check(self.lib.hc_skinny_to_modal(C.byref(g), modes, _p(skinny), _p(modal)))

    def modal_to_skinny(self, g, modes, modal, skinny):
        _check(self.lib.hc_modal_to_skinny(C.byref(g), modes, _p(modal), _p(skinny)))

    def limit_patch_o2(self, g, modal, lim=None):
        _check(self.lib.hc_limit_patch_o2(C.byref(g), _p(modal),
                                          C.byref(lim or default_limiter())))

    def reconstruct_patch_o3(self, g, modal, lim=None):
        _check(self.lib.hc_reconstruct_patch_o3(C.byref(g), _p(modal),
                                                C.byref(lim or default_limiter())))

    def predict_patch(self, g, modes, modal, dt, gamma=1.4):
        _check(self.lib.hc_predict_patch(C.byref(g), modes, _p(modal), C.c_double(dt),
                                         C.c_double(gamma)))

    def zero_temporal_mode(self, g, modes, modal):
        _check(self.lib.hc_zero_temporal_mode(C.byref(g), modes, _p(modal)))

    def make_flux_axis(self, g, modes, modal, axis, solver, out, gamma=1.4):
        _check(self.lib.hc_make_flux_axis(C.byref(g), modes, _p(modal), axis,
                                          C.c_double(gamma), solver, _p(out)))

    def make_du_dt(self, g, fx, fy, fz, dt, rate):
        _check(self.lib.hc_make_du_dt(C.byref(g), _p(fx), _p(fy), _p(fz), C.c_double(dt),
                                      _p(rate)))

    def update_u_timestep(self, g, modes, modal, skinny, rate, cfl, gamma=1.4):
        d = C.c_double()
        _check(self.lib.hc_update_u_timestep(C.byref(g), modes, _p(modal), _p(skinny),
                                             _p(rate), C.c_double(cfl), C.c_double(gamma),
                                             C.byref(d)))
        return d.value

    def compute_dt_next(self, g, modes, modal, cfl, gamma=1.4):
        d = C.c_double()
        _check(self.lib.hc_compute_dt_next(C.byref(g), modes, _p(modal), C.c_double(gamma),
                                           C.c_double(cfl), C.byref(d)))
        return d.value

    def ader_step(self, g, par, modal, skinny, fx, fy, fz, rate, dt, cfl):
        d = C.c_double()
        _check(self.lib.hc_ader_step(C.byref(g), C.byref(par), _p(modal), _p(skinny), _p(fx),
                                     _p(fy), _p(fz), _p(rate), C.c_double(dt), C.c_double(cfl),
                                     C.byref(d)))
        return d.value

    def rk_save_u0(self, g, skinny, u0):
        _check(self.lib.hc_rk_save_u0(C.byref(g), _p(skinny), _p(u0)))

    def rk_stage(self, g, par, modal, skinny, fx, fy, fz, rate, u0, dt, a, b):
        _check(self.lib.hc_rk_stage(C.byref(g), C.byref(par), _p(modal), _p(skinny), _p(fx),
                                    _p(fy), _p(fz), _p(rate), _p(u0), C.c_double(dt),
                                    C.c_double(a), C.c_double(b)))

    def rk_step(self, g, par, nstages, modal, skinny, fx, fy, fz, rate, u0, bc, dt, cfl):
        d = C.c_double()
        _check(self.lib.hc_rk_step(C.byref(g), C.byref(par), nstages, _p(modal), _p(skinny),
                                   _p(fx), _p(fy), _p(fz), _p(rate), _p(u0), bc,
                                   C.c_double(dt), C.c_double(cfl), C.byref(d)))
        return d.value


class Stepper:
    """Device-resident fused ADER stepper for one patch or one z-slab.

    bc: (x, y, z) boundary kinds; z = None means the caller fills the z ghost planes (halo
    exchange of a z-slab decomposition, see ``paper_2211_13295_b200.slabs``).
    exact: True = bit-exact build (the reference's bits); False = FMA-contracted build."""

    def __init__(self, geom: Geom, params: Params, bc=(PERIODIC, PERIODIC, PERIODIC),
                 exact=True, device=0, integrator=ADER):
        self.lib = load_library()
        self.geom, self.params = geom, params
        o = StepperOpts()
        o.bc[0], o.bc[1] = bc[0], bc[1]
        o.bc[2] = -1 if bc[2] is None else bc[2]
        o.exact, o.device, o.integrator = int(bool(exact)), device, integrator
        h = C.c_void_p()
        _check(self.lib.hc_stepper_create(C.byref(geom), C.byref(params), C.byref(o),
                                          C.byref(h)))
        self.h = h
        my_pad, pitch, mz = C.c_int(), C.c_int(), C.c_int()
        _check(self.lib.hc_stepper_layout(self.h, C.byref(my_pad), C.byref(pitch),
                                          C.byref(mz)))
        self.my_pad, self.pitch, self.mz = my_pad.value, pitch.value, mz.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.hc_stepper_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int):
        _check(self.lib.hc_stepper_set_stream(self.h, C.c_void_p(stream_handle)))

    def upload(self, skinny: np.ndarray):
        _check(self.lib.hc_stepper_upload(self.h, _p(skinny)))

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        out = zeros_skinny(self.geom) if out is None else out
        _check(self.lib.hc_stepper_download(self.h, _p(out)))
        return out

    def set_time(self, t, dt, cfl, t_final=-1.0):
        _check(self.lib.hc_stepper_set_time(self.h, C.c_double(t), C.c_double(dt),
                                            C.c_double(cfl), C.c_double(t_final)))

    def step(self, n=1):
        _check(self.lib.hc_stepper_step(self.h, n))

    def step_host(self, host_in: np.ndarray, host_out: np.ndarray | None = None, chunks=16):
        """One step end to end from host memory (pipelined H2D / fused step / D2H)."""
        host_out = host_in if host_out is None else host_out
        _check(self.lib.hc_stepper_step_host(self.h, _p(host_in), _p(host_out), int(chunks)))
        return host_out

    @property
    def stages(self) -> int:
        return self.lib.hc_stepper_stages(self.h)

    def fill_ghosts(self):
        _check(self.lib.hc_stepper_fill_ghosts(self.h))

    def compute(self):
        _check(self.lib.hc_stepper_compute(self.h))

    def compute_range(self, kz_first, kz_last, last):
        """fused launch over active planes [kz_first, kz_last); last closes the step/stage"""
        _check(self.lib.hc_stepper_compute_range(self.h, int(kz_first), int(kz_last),
                                                 int(bool(last))))

    def advance(self):
        _check(self.lib.hc_stepper_advance(self.h))

    def compute_step(self):
        """compute(); when it is the step's last stage, also the advance (no all-reduce in
        between: a stepper owning its dt)"""
        _check(self.lib.hc_stepper_compute_step(self.h))

    def sync(self):
        """Returns (t, dt_of_next_step, steps_done); raises the first device error."""
        t, dt, n = C.c_double(), C.c_double(), C.c_long()
        _check(self.lib.hc_stepper_sync(self.h, C.byref(t), C.byref(dt), C.byref(n)))
        return t.value, dt.value, n.value

    def state_ptr(self) -> int:
        p = C.POINTER(C.c_double)()
        pitch = C.c_size_t()
        _check(self.lib.hc_stepper_state(self.h, C.byref(p), C.byref(pitch)))
        return C.cast(p, C.c_void_p).value

    def dt_ptrs(self):
        a, b = C.POINTER(C.c_double)(), C.POINTER(C.c_double)()
        _check(self.lib.hc_stepper_dt_ptrs(self.h, C.byref(a), C.byref(b)))
        return C.cast(a, C.c_void_p).value, C.cast(b, C.c_void_p).value

    @property
    def launches(self) -> int:
        return self.lib.hc_stepper_launches(self.h)

    def kernel_info(self):
        """Which fused kernel steps this stepper: ("ring", 0), ("persistent", ctas) for the
        opt-in persistent kernel, or ("seam", tiles) for the ring-free seam kernel pair (the
        FMA build's default on x/y-periodic meshes with nx % 32 == 0)."""
        k, n = C.c_int(), C.c_int()
        _check(self.lib.hc_stepper_info(self.h, C.byref(k), C.byref(n)))
        return ("ring", "persistent", "seam")[k.value], n.value


class Ader4Stepper:
    """The formally fourth-order ADER step of csrc/ader4.cu (hc_ader4_*; an extension: the
    reference's ADER structure is second order in time): degree-3 WENO-AO + cross-term
    reconstruction, local space-time predictor, Gauss-point face and time quadrature."""

    def __init__(self, geom: Geom, params: Params, boundary=PERIODIC, device=0):
        self.lib = load_library()
        self.geom = geom
        h = C.c_void_p()
        _check(self.lib.hc_ader4_create(C.byref(geom), C.byref(params), boundary, device,
                                        C.byref(h)))
        self.h = h

    def upload(self, skinny: np.ndarray):
        a = np.ascontiguousarray(skinny, dtype=np.float64)
        _check(self.lib.hc_ader4_upload(self.h, a.ctypes.data_as(C.c_void_p)))

    def download(self, out: np.ndarray | None = None):
        g = self.geom
        if out is None:
            out = np.empty((g.nz + 2 * g.ghost, g.ny + 2 * g.ghost, g.nx + 2 * g.ghost, 5))
        _check(self.lib.hc_ader4_download(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def set_time(self, t, dt, cfl, t_final=0.0):
        _check(self.lib.hc_ader4_set_time(self.h, C.c_double(t), C.c_double(dt),
                                          C.c_double(cfl), C.c_double(t_final)))

    def step(self, n=1):
        _check(self.lib.hc_ader4_step(self.h, int(n)))

    def sync(self):
        t, dt, n = C.c_double(), C.c_double(), C.c_long()
        _check(self.lib.hc_ader4_sync(self.h, C.byref(t), C.byref(dt), C.byref(n)))
        return t.value, dt.value, n.value

    @property
    def launches(self) -> int:
        self.lib.hc_ader4_launches.restype = C.c_long
        return int(self.lib.hc_ader4_launches(self.h))

    @property
    def stream_ptr(self) -> int:
        p = C.c_void_p()
        _check(self.lib.hc_ader4_stream(self.h, C.byref(p)))
        return p.value or 0

    def close(self):
        if self.h:
            self.lib.hc_ader4_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DomainOpts(C.Structure):
    """hc_domain_opts (include/hydro_cuda.h)."""
    _fields_ = [("bc", C.c_int * 3), ("exact", C.c_int), ("integrator", C.c_int),
                ("device", C.c_int), ("transport", C.c_int), ("overlap", C.c_int)]


XCHG_NCCL, XCHG_PEER, XCHG_STORE = 0, 1, 2  # hc_exchange_kind


def nccl_unique_id() -> bytes:
    """hc_nccl_unique_id: 128 bytes for Domain(..., rank, world, nccl_id) on every rank."""
    buf = (C.c_ubyte * 128)()
    _check(load_library().hc_nccl_unique_id(buf, C.c_size_t(128)))
    return bytes(buf)


class Domain:
    """The multi-GPU z-slab domain of the C ABI (hc_domain_*, csrc/domain.cu): the reference's
    PatchSet split along z (transfer.cpp:17-47) with one slab per GPU, run_patch_step
    (transfer.cpp:152-216) as device x/y ghosts + whole-plane z halos (NCCL send/recv straight
    into the ghost planes, or peer copies) + the fused step + an 8-byte all-reduce(MIN) of
    dt_next, enqueued without host round trips.

    devices: one process driving these GPUs (hc_domain_create_local); or rank / world /
    nccl_id: one process per GPU (hc_domain_create, this rank's slab on ``device``)."""

    def __init__(self, geom: Geom, params: Params, bc=(PERIODIC, PERIODIC, PERIODIC),
                 exact=True, integrator=ADER, transport=XCHG_NCCL, devices=(0,), rank=None,
                 world=None, nccl_id=None, device=0, overlap=False):
        self.lib = load_library()
        self.geom, self.params = geom, params
        o = DomainOpts()
        for a in range(3):
            o.bc[a] = bc[a]
        o.exact, o.integrator, o.device, o.transport = int(bool(exact)), integrator, device, \
            transport
        o.overlap = int(bool(overlap))
        h = C.c_void_p()
        if rank is None:
            devs = (C.c_int * len(devices))(*devices)
            _check(self.lib.hc_domain_create_local(C.byref(geom), C.byref(params), C.byref(o),
                                                   len(devices), devs, C.byref(h)))
        else:
            idb = (C.c_ubyte * 128).from_buffer_copy(nccl_id) if nccl_id else None
            _check(self.lib.hc_domain_create(C.byref(geom), C.byref(params), C.byref(o), rank,
                                             world, idb, C.byref(h)))
        self.h = h
        nz, z0, ns, k = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(self.lib.hc_domain_info(self.h, C.byref(nz), C.byref(z0), C.byref(ns),
                                       C.byref(k)))
        self.nz_local, self.z0, self.nslabs = nz.value, z0.value, ns.value
        self.kernel = ("ring", "persistent", "seam")[k.value]

    def scatter(self, skinny: np.ndarray):
        a = np.ascontiguousarray(skinny, dtype=np.float64)
        _check(self.lib.hc_domain_scatter(self.h, a.ctypes.data_as(C.c_void_p)))

    def gather(self, out: np.ndarray):
        assert out.flags.c_contiguous and out.dtype == np.float64
        _check(self.lib.hc_domain_gather(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def set_time(self, t, dt, cfl, t_final=0.0):
        _check(self.lib.hc_domain_set_time(self.h, C.c_double(t), C.c_double(dt),
                                           C.c_double(cfl), C.c_double(t_final)))

    def step(self, n=1):
        _check(self.lib.hc_domain_step(self.h, int(n)))

    def sync(self):
        t, dt, n = C.c_double(), C.c_double(), C.c_long()
        _check(self.lib.hc_domain_sync(self.h, C.byref(t), C.byref(dt), C.byref(n)))
        return t.value, dt.value, n.value

    @property
    def launches(self):
        return self.lib.hc_domain_launches(self.h)

    def close(self):
        if self.h:
            self.lib.hc_domain_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fp64_peak(device: int = 0) -> float:
    """Measured DFMA throughput of the device in TFLOP/s (hc_fp64_peak)."""
    d = C.c_double()
    _check(load_library().hc_fp64_peak(device, C.byref(d)))
    return d.value


class PatchSet:
    """Device-resident PatchSet (transfer.hpp:47-73, include/hydro_cuda.h hc_patchset_*):
    px x py x pz patches of `g`, states in HBM, run_patch_step on the device."""

    def __init__(self, g: Geom, px, py, pz, params: Params, boundary=PERIODIC, exact=True,
                 device=0, integrator=ADER):
        self.lib = load_library()
        self.lib.hc_patchset_launches.restype = C.c_long
        for n in ("hc_patchset_destroy", "hc_patchset_launches"):
            getattr(self.lib, n).argtypes = [C.c_void_p]
        self.lib.hc_patchset_step.argtypes = [C.c_void_p, C.c_int]
        self.g = g
        h = C.c_void_p()
        _check(self.lib.hc_patchset_create(C.byref(g), px, py, pz, C.byref(params), boundary,
                                           int(exact), device, integrator, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.hc_patchset_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def scatter(self, skinny):
        """scatter_to_patches (transfer.cpp:50-62) from a global host SkinnyState"""
        s = np.ascontiguousarray(skinny, dtype=np.float64)
        _check(self.lib.hc_patchset_scatter(self.h, _p(s)))

    def gather(self, out=None):
        """gather_from_patches (transfer.cpp:64-76) into a global host SkinnyState"""
        out = zeros_skinny(self.g) if out is None else out
        _check(self.lib.hc_patchset_gather(self.h, _p(out)))
        return out

    def set_time(self, t, dt, cfl, t_final=-1.0):
        _check(self.lib.hc_patchset_set_time(self.h, C.c_double(t), C.c_double(dt),
                                             C.c_double(cfl), C.c_double(t_final)))

    def step(self, n=1):
        _check(self.lib.hc_patchset_step(self.h, n))

    def sync(self):
        t, dt, n = C.c_double(), C.c_double(), C.c_long()
        _check(self.lib.hc_patchset_sync(self.h, C.byref(t), C.byref(dt), C.byref(n)))
        return t.value, dt.value, n.value

    def ledger(self):
        """TransferLedger fields (uploads, downloads, scalar_uploads, scalar_downloads,
        uploads_active_only, steps) for the skinny strategy"""
        c = (C.c_ulonglong * 6)()
        _check(self.lib.hc_patchset_ledger(self.h, c))
        return tuple(int(x) for x in c)

    @staticmethod
    def ledger_csv_header():
        """transfer.cpp:218 ledger_csv_header"""
        return "step,strategy,uploads,downloads,scalar_uploads"

    def ledger_csv_row(self, step):
        """transfer.cpp:220-227 ledger_csv_row (per-step averages, skinny strategy)"""
        up, down, su, _, _, steps = self.ledger()
        n = steps if steps else 1
        return f"{step},skinny,{up // n},{down // n},{su // n}"

    @property
    def launches(self):
        return self.lib.hc_patchset_launches(self.h)
