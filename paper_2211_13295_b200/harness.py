"""harness -- the reference's run driver (proj/src/harness.cpp) on the device-resident stepper.

``run_simulation`` mirrors harness.cpp:116-193: host initial condition (problems.cpp, sampled
on the host for bit-identical inputs), ``initial_dt`` (:92-103), the time loop with the
dt/dt_next hand-off and the final-step clip to ``t_final`` (:155-170) -- here executed on the
device by the fused stepper, so a whole run is queued without host round trips -- then the
gathered state and the error norms against the exact solution (:182-191). ``run_benchmark``,
``run_convergence_study`` and ``error_norms`` follow :71-88, :195-227. The numbers equal the
reference's bit for bit in the exact build (tests/test_harness_gpu.py).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import hydro

VORTEX, SOD, CONSTANT = "vortex", "sod", "constant"
INTEGRATORS = {"ader": hydro.ADER, "rk2": hydro.RK2, "rk3": hydro.RK3}


@dataclass
class RunConfig:
    """harness.hpp:17-38 (the fields that shape a run; output/CSV fields are host-side)."""
    problem: str = VORTEX
    order: int = 2
    integrator: str = "ader"
    solver: int = hydro.HLL
    nx: int = 24
    ny: int = 24
    nz: int = 24
    cfl: float = -1.0       # < 0: 0.6 at O2, 0.4 at O3 (harness.hpp:36)
    t_final: float = -1.0   # exactly one of t_final / steps is active
    steps: int = 0
    gamma: float = 1.4
    exact: bool = True      # bit-exact build (False: FMA build)
    device: int = 0
    split_x: int = 1        # patch split (harness.hpp:24): > 1 runs the device PatchSet
    split_y: int = 1
    split_z: int = 1

    def effective_cfl(self) -> float:
        return self.cfl if self.cfl > 0.0 else (0.6 if self.order == 2 else 0.4)

    def validate(self):
        """harness.cpp:60-69."""
        if self.order not in (2, 3, 4):
            raise ValueError("order must be 2 or 3 (4: the WENO-AO extension)")
        if min(self.nx, self.ny, self.nz) < 4:
            raise ValueError("mesh must be at least 4^3")
        if self.t_final > 0.0 and self.steps > 0:
            raise ValueError("set exactly one of tfinal and steps")
        if self.cfl > 0.0 and self.cfl >= 1.0:
            raise ValueError("cfl must lie in (0,1)")
        if self.integrator not in INTEGRATORS:
            raise ValueError(f"unknown integrator '{self.integrator}'")


@dataclass
class ErrorReport:
    l1: np.ndarray = field(default_factory=lambda: np.zeros(5))
    linf: np.ndarray = field(default_factory=lambda: np.zeros(5))
    order_estimate: float = math.nan


@dataclass
class RunResult:
    final_state: np.ndarray
    geom: hydro.Geom
    steps: int
    t_end: float
    wall_seconds: float
    zones_per_sec: float
    errors: ErrorReport | None
    kernel: str = ""  # the fused step that ran: "seam", "ring" or "persistent" ("" PatchSet)


def default_domain(problem):
    """problems.cpp:123-131."""
    if problem == SOD:
        return (0.0, 0.0, 0.0), (1.0, 1.0, 1.0)
    return (-5.0, -5.0, -5.0), (5.0, 5.0, 5.0)


def error_norms(numerical, exact, g) -> ErrorReport:
    """harness.cpp:71-88: per-variable mean absolute and max difference over active zones
    (same summation order: zones in storage order, then variables)."""
    if numerical.shape != exact.shape:
        raise ValueError("error_norms: shape mismatch")
    gh = g.ghost
    d = np.abs(numerical[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx] -
               exact[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]).reshape(-1, 5)
    rep = ErrorReport()
    inv_n = 1.0 / float(g.nx * g.ny * g.nz)
    for q in range(5):  # sequential sum, as the reference's loop
        rep.l1[q] = _seq_sum(d[:, q]) * inv_n
        rep.linf[q] = d[:, q].max()
    return rep


def _seq_sum(x):
    """Left-to-right double sum (the reference's accumulation order)."""
    s = np.cumsum(x)  # numpy's cumsum is sequential
    return float(s[-1]) if s.size else 0.0


def _ic(api, cfg, g):
    if cfg.problem == VORTEX:
        return api.init_isentropic_vortex(g, cfg.order, gamma=cfg.gamma)
    if cfg.problem == SOD:
        return api.init_sod(g, gamma=cfg.gamma)
    if cfg.problem == CONSTANT:
        return api.init_constant(g, gamma=cfg.gamma)
    raise ValueError(f"unknown problem '{cfg.problem}'")


def run_simulation(cfg: RunConfig) -> RunResult:
    """harness.cpp:116-193 on the fused device stepper (single patch)."""
    cfg.validate()
    lo, hi = default_domain(cfg.problem)
    g = hydro.make_geometry(cfg.nx, cfg.ny, cfg.nz, cfg.order, lo, hi)
    api = hydro.HostApi()
    s = _ic(api, cfg, g)
    bc = hydro.OUTFLOW if cfg.problem == SOD else hydro.PERIODIC
    cfl = cfg.effective_cfl()
    dt0 = api.initial_dt(g, s, cfl, cfg.gamma)
    if cfg.steps > 0:
        t_final, nsteps = -1.0, cfg.steps
    else:
        # harness.cpp:105-114 resolve_t_final: one periodic crossing / 0.2 for sod
        t_final = cfg.t_final if cfg.t_final > 0.0 else (0.2 if cfg.problem == SOD
                                                        else g.nx * g.dx / 1.0)
        nsteps = None
    params = hydro.make_params(cfg.order, cfg.solver, cfg.gamma)
    if cfg.split_x * cfg.split_y * cfg.split_z > 1:  # transfer.cpp PatchSet, on the device
        st = hydro.PatchSet(g, cfg.split_x, cfg.split_y, cfg.split_z, params, boundary=bc,
                            exact=cfg.exact, device=cfg.device,
                            integrator=INTEGRATORS[cfg.integrator])
        st.scatter(s)
    else:
        st = hydro.Stepper(g, params, bc=(bc, bc, bc), exact=cfg.exact, device=cfg.device,
                           integrator=INTEGRATORS[cfg.integrator])
        st.upload(s)
    st.set_time(0.0, dt0, cfl, t_final)
    t0 = time.perf_counter()
    if nsteps is not None:
        st.step(nsteps)
        t, dt, done = st.sync()
    else:
        # queue steps in chunks; the device stops itself at t_final
        done = 0
        while True:
            before = done
            st.step(256)
            t, dt, done = st.sync()
            if done - before < 256:
                break
    wall = time.perf_counter() - t0
    out = st.gather() if isinstance(st, hydro.PatchSet) else st.download()
    kernel = "" if isinstance(st, hydro.PatchSet) else st.kernel_info()[0]
    st.close()
    gh = g.ghost
    # the reference gathers active zones into a fresh SkinnyState (ghosts zero)
    final = hydro.zeros_skinny(g)
    final[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx] = out[gh:gh + g.nz, gh:gh + g.ny,
                                                          gh:gh + g.nx]
    errors = None
    if cfg.problem == VORTEX:
        errors = error_norms(final, api.init_isentropic_vortex(g, cfg.order, t=t,
                                                               gamma=cfg.gamma), g)
    elif cfg.problem == CONSTANT:
        errors = error_norms(final, api.init_constant(g, cfg.gamma), g)
    zps = g.nx * g.ny * g.nz * done / wall if wall > 0 else 0.0
    return RunResult(final, g, done, t, wall, zps, errors, kernel)


def run_benchmark(cfg: RunConfig) -> RunResult:
    """harness.cpp:222-227: 20 steps unless a step count or t_final is set."""
    if cfg.steps <= 0 and cfg.t_final <= 0.0:
        cfg = RunConfig(**{**cfg.__dict__, "steps": 20})
    return run_simulation(cfg)


def run_convergence_study(cfg: RunConfig, meshes):
    """harness.cpp:195-220: L1(rho) ratio -> observed order between successive meshes."""
    if len(meshes) < 2:
        raise ValueError("convergence study needs at least two meshes")
    rows = []
    for m, n in enumerate(meshes):
        c = RunConfig(**{**cfg.__dict__, "nx": n, "ny": n, "nz": n})
        r = run_simulation(c)
        if r.errors is None:
            raise RuntimeError("convergence study needs an exact solution")
        if m > 0:
            e_coarse = rows[-1][1].l1[0]
            e_fine = r.errors.l1[0]
            r.errors.order_estimate = math.log(e_coarse / e_fine) / math.log(n / meshes[m - 1])
        rows.append((n, r.errors, r))
    return rows


@dataclass
class ReproReport:
    """harness.hpp:75-81."""
    serial_bit_identical: bool = False
    multiworker_l1_diff: float = 0.0
    max_abs_diff: float = 0.0
    max_diff_zone: tuple = (0, 0, 0)
    passed: bool = False


def run_reproducibility_check(cfg: RunConfig) -> ReproReport:
    """harness.cpp:229-271 on the device: two identical runs must agree bit for bit; the
    "multi-worker" run -- on the GPU, a different decomposition (2 x 2 x 2 patches when the mesh
    divides, else 2 x 1 x 1) -- is compared by the density L1 (pass below 1e-10)."""
    base = RunConfig(**{**cfg.__dict__})
    if base.steps <= 0:
        base.steps, base.t_final = 50, -1.0
    a = run_simulation(RunConfig(**base.__dict__))
    b = run_simulation(RunConfig(**base.__dict__))
    rep = ReproReport()
    rep.serial_bit_identical = bool((a.final_state.view(np.uint64) ==
                                     b.final_state.view(np.uint64)).all())
    split = (2, 2, 2) if all(n % 2 == 0 and n // 2 >= 4 for n in (base.nx, base.ny, base.nz)) \
        else (2, 1, 1)
    c = run_simulation(RunConfig(**{**base.__dict__, "split_x": split[0], "split_y": split[1],
                                    "split_z": split[2]}))
    g = a.geom
    gh = g.ghost
    act = np.s_[gh:gh + g.nz, gh:gh + g.ny, gh:gh + g.nx]
    d = np.abs(a.final_state[act] - c.final_state[act])
    rep.multiworker_l1_diff = float(d[..., 0].sum() / (g.nx * g.ny * g.nz))
    k, j, i, _ = np.unravel_index(int(np.argmax(d)), d.shape)
    rep.max_abs_diff = float(d.max())
    rep.max_diff_zone = (int(i), int(j), int(k))
    rep.passed = rep.serial_bit_identical and rep.multiworker_l1_diff < 1e-10
    return rep
