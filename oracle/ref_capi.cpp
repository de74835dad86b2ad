// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter over the REFERENCE library itself (compiled from the unmodified
// sources under /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It exposes
// the reference's hydro:: functions with the same flat signatures as hydro_oracle.h
// (prefix ref_ instead of or_) so tests can pin the C restatement -- and the CUDA product --
// against the reference's own arithmetic. Nothing here is product code.
#include <omp.h>

#include <cstring>
#include <string>
#include <vector>

#include "hydro/corrector.hpp"
#include "hydro/harness.hpp"
#include "hydro/predictor.hpp"
#include "hydro/problems.hpp"
#include "hydro/reconstruct.hpp"
#include "hydro/serial_ref.hpp"
#include "hydro/stepper.hpp"
#include "hydro/transfer.hpp"
#include "hydro_oracle.h"

using namespace hydro;

namespace {
thread_local std::string g_err;

PatchGeometry to_geom(const or_geom* g) {
    PatchGeometry p;
    p.nx = g->nx;
    p.ny = g->ny;
    p.nz = g->nz;
    p.ghost = g->ghost;
    p.dx = g->dx;
    p.dy = g->dy;
    p.dz = g->dz;
    p.origin = {g->origin[0], g->origin[1], g->origin[2]};
    return p;
}
LimiterConfig to_lim(const or_limiter* l) {
    LimiterConfig c;
    c.compression_factor_density = l->cfac_rho;
    c.compression_factor_other = l->cfac_other;
    c.weno_epsilon = l->weno_eps;
    c.weno_linear_weights = {l->weno_w[0], l->weno_w[1], l->weno_w[2]};
    return c;
}
ModalState modal_in(const PatchGeometry& g, int modes, const double* v) {
    ModalState m = ModalState::make(g, modes == 5 ? 2 : 3);
    std::memcpy(m.v.data(), v, m.v.size() * sizeof(double));
    return m;
}
SkinnyState skinny_in(const PatchGeometry& g, const double* v) {
    SkinnyState s = SkinnyState::make(g);
    std::memcpy(s.v.data(), v, s.v.size() * sizeof(double));
    return s;
}
void out(const std::vector<double>& v, double* dst) {
    std::memcpy(dst, v.data(), v.size() * sizeof(double));
}
StepParams to_par(const or_params* p) {
    StepParams par;
    par.gas.gamma = p->gamma;
    par.solver = p->solver == OR_RUSANOV ? SolverChoice::rusanov : SolverChoice::hll;
    par.limiter = to_lim(&p->lim);
    par.order = p->order;
    return par;
}
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return OR_OK;
    } catch (const unphysical_error& e) {
        g_err = e.what();
        return OR_UNPHYSICAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OR_INVALID;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_set_threads(int n) { omp_set_num_threads(n); }

int ref_hll_flux(const double* ul, const double* ur, int axis, double gamma, double* f) {
    return guarded([&] {
        auto r = hll_flux({ConsVars::from(ul), ConsVars::from(ur), Axis(axis)}, GasModel{gamma});
        std::memcpy(f, r.data(), 5 * sizeof(double));
    });
}
int ref_rusanov_flux(const double* ul, const double* ur, int axis, double gamma, double* f) {
    return guarded([&] {
        auto r =
            rusanov_flux({ConsVars::from(ul), ConsVars::from(ur), Axis(axis)}, GasModel{gamma});
        std::memcpy(f, r.data(), 5 * sizeof(double));
    });
}
int ref_eval_tstep_ptwise(const double* u, double cfl, double dx, double dy, double dz,
                          double gamma, double* dt) {
    return guarded(
        [&] { *dt = eval_tstep_ptwise(ConsVars::from(u), cfl, dx, dy, dz, GasModel{gamma}); });
}
double ref_mc_limiter(double a, double b, double cfac) { return mc_limiter(a, b, cfac); }
void ref_weno3_point(const double* s, const or_limiter* cfg, double* ux, double* uxx) {
    WenoCoeffs c = weno3_point(s, to_lim(cfg));
    *ux = c.ux;
    *uxx = c.uxx;
}
int ref_predictor_ptwise(double* zv, int modes, double dt, double dx, double dy, double dz,
                         double gamma) {
    return guarded([&] {
        ZoneModal z;
        z.modes = modes;
        std::memcpy(z.v, zv, sizeof(double) * NVAR * modes);
        predictor_ptwise(z, dt, dx, dy, dz, GasModel{gamma});
        std::memcpy(zv, z.v, sizeof(double) * NVAR * modes);
    });
}

void ref_apply_boundary_skinny(const or_geom* g, int kind, double* skinny) {
    PatchGeometry pg = to_geom(g);
    SkinnyState s = skinny_in(pg, skinny);
    apply_boundary(s, pg, kind == OR_PERIODIC ? BoundaryKind::periodic : BoundaryKind::outflow);
    out(s.v, skinny);
}
void ref_apply_boundary_modal(const or_geom* g, int modes, int kind, double* modal) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, modes, modal);
    apply_boundary(m, pg, kind == OR_PERIODIC ? BoundaryKind::periodic : BoundaryKind::outflow);
    out(m.v, modal);
}
void ref_skinny_to_modal(const or_geom* g, int modes, const double* skinny, double* modal) {
    PatchGeometry pg = to_geom(g);
    SkinnyState s = skinny_in(pg, skinny);
    ModalState m = modal_in(pg, modes, modal);
    skinny_to_modal(s, m);
    out(m.v, modal);
}
void ref_modal_to_skinny(const or_geom* g, int modes, const double* modal, double* skinny) {
    PatchGeometry pg = to_geom(g);
    SkinnyState s = skinny_in(pg, skinny);
    ModalState m = modal_in(pg, modes, modal);
    modal_to_skinny(m, pg, s);
    out(s.v, skinny);
}
void ref_limit_patch_o2(const or_geom* g, double* modal, const or_limiter* cfg) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, 5, modal);
    limit_patch_o2(m, pg, to_lim(cfg));
    out(m.v, modal);
}
void ref_reconstruct_patch_o3(const or_geom* g, double* modal, const or_limiter* cfg) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, 11, modal);
    reconstruct_patch_o3(m, pg, to_lim(cfg));
    out(m.v, modal);
}
int ref_predict_patch(const or_geom* g, int modes, double* modal, double dt, double gamma) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, modes, modal);
    TimeState t;
    t.dt = dt;
    int rc = guarded([&] { predict_patch(m, t, pg, GasModel{gamma}); });
    out(m.v, modal);
    return rc;
}
void ref_zero_temporal_mode(const or_geom* g, int modes, double* modal) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, modes, modal);
    zero_temporal_mode(m);
    out(m.v, modal);
}
int ref_make_flux_axis(const or_geom* g, int modes, const double* modal, int axis, double gamma,
                       int solver, double* outp) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, modes, modal);
    FaceFlux f = FaceFlux::make(pg, Axis(axis));
    int rc = guarded([&] {
        make_flux_axis(m, Axis(axis), pg, GasModel{gamma},
                       solver == OR_RUSANOV ? SolverChoice::rusanov : SolverChoice::hll, f);
    });
    out(f.v, outp);
    return rc;
}
void ref_make_du_dt(const or_geom* g, const double* fx, const double* fy, const double* fz,
                    double dt, double* rate) {
    PatchGeometry pg = to_geom(g);
    FluxSet fs = FluxSet::make(pg);
    std::memcpy(fs.fx.v.data(), fx, fs.fx.v.size() * sizeof(double));
    std::memcpy(fs.fy.v.data(), fy, fs.fy.v.size() * sizeof(double));
    std::memcpy(fs.fz.v.data(), fz, fs.fz.v.size() * sizeof(double));
    RateField r = RateField::make(pg);
    TimeState t;
    t.dt = dt;
    make_du_dt(fs, t, pg, r);
    out(r.v, rate);
}
int ref_update_u_timestep(const or_geom* g, int modes, double* modal, double* skinny,
                          const double* rate, double cfl, double gamma, double* dt_next) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, modes, modal);
    SkinnyState s = skinny_in(pg, skinny);
    RateField r = RateField::make(pg);
    std::memcpy(r.v.data(), rate, r.v.size() * sizeof(double));
    TimeState t;
    t.cfl = cfl;
    int rc = guarded([&] { update_u_timestep(m, s, r, t, pg, GasModel{gamma}); });
    out(m.v, modal);
    out(s.v, skinny);
    *dt_next = t.dt_next;
    return rc;
}
int ref_compute_dt_next(const or_geom* g, int modes, const double* modal, double gamma,
                        double cfl, double* dt_next) {
    PatchGeometry pg = to_geom(g);
    ModalState m = modal_in(pg, modes, modal);
    return guarded([&] { *dt_next = compute_dt_next(m, pg, GasModel{gamma}, cfl); });
}

int ref_ader_step(const or_geom* g, const or_params* p, double* modal, double* skinny,
                  double* fx, double* fy, double* fz, double* rate, double dt, double cfl,
                  double* dt_next) {
    PatchGeometry pg = to_geom(g);
    StepParams par = to_par(p);
    ModalState m = modal_in(pg, par.order == 2 ? 5 : 11, modal);
    SkinnyState s = skinny_in(pg, skinny);
    StepScratch sc = StepScratch::make(pg);
    TimeState t;
    t.dt = dt;
    t.cfl = cfl;
    int rc = guarded([&] { ader_step(m, s, t, pg, par, sc); });
    out(m.v, modal);
    out(s.v, skinny);
    out(sc.fluxes.fx.v, fx);
    out(sc.fluxes.fy.v, fy);
    out(sc.fluxes.fz.v, fz);
    out(sc.rate.v, rate);
    *dt_next = t.dt_next;
    return rc;
}

int ref_rk_step(const or_geom* g, const or_params* p, int nstages, double* modal,
                double* skinny, double* fx, double* fy, double* fz, double* rate,
                double* stage_u0, int bc, double dt, double cfl, double* dt_next) {
    PatchGeometry pg = to_geom(g);
    StepParams par = to_par(p);
    par.integrator = nstages == 2 ? IntegratorChoice::rk2 : IntegratorChoice::rk3;
    ModalState m = modal_in(pg, par.order == 2 ? 5 : 11, modal);
    SkinnyState s = skinny_in(pg, skinny);
    StepScratch sc = StepScratch::make(pg);
    std::memcpy(sc.stage_u0.v.data(), stage_u0, sc.stage_u0.v.size() * sizeof(double));
    TimeState t;
    t.dt = dt;
    t.cfl = cfl;
    int rc = guarded([&] {
        rk_step(m, s, t, pg, par, sc,
                bc == OR_PERIODIC ? BoundaryKind::periodic : BoundaryKind::outflow);
    });
    out(m.v, modal);
    out(s.v, skinny);
    out(sc.fluxes.fx.v, fx);
    out(sc.fluxes.fy.v, fy);
    out(sc.fluxes.fz.v, fz);
    out(sc.rate.v, rate);
    out(sc.stage_u0.v, stage_u0);
    *dt_next = t.dt_next;
    return rc;
}

void ref_init_isentropic_vortex(const or_geom* g, double gamma, int order, double t,
                                double* skinny) {
    PatchGeometry pg = to_geom(g);
    SkinnyState s = t == 0.0 ? init_isentropic_vortex(pg, GasModel{gamma}, order)
                             : exact_vortex(pg, GasModel{gamma}, t, order);
    out(s.v, skinny);
}
void ref_init_sod(const or_geom* g, double gamma, double* skinny) {
    out(init_sod(to_geom(g), GasModel{gamma}).v, skinny);
}
void ref_init_constant(const or_geom* g, double gamma, double* skinny) {
    out(init_constant(to_geom(g), GasModel{gamma}).v, skinny);
}

// Full harness run (harness.cpp:116-193) through the reference's public API: problem,
// order, integrator (0 ader, 2 rk2, 3 rk3), solver, mesh, split, steps. Returns zones/s and
// copies the gathered final skinny (global geometry, ghosts included) into final_skinny
// (may be null). Used as the CPU baseline arm and for whole-run parity.
double ref_run_benchmark(int problem, int order, int integrator, int solver, int nx, int ny,
                         int nz, int sx, int sy, int sz, long steps, int threads,
                         double* final_skinny, double* t_end, double* l1_rho) {
    RunConfig cfg;
    cfg.problem = problem == 0 ? Problem::vortex : (problem == 1 ? Problem::sod : Problem::constant);
    cfg.order = order;
    cfg.integrator = integrator == 0 ? IntegratorChoice::ader_onestep
                                     : (integrator == 2 ? IntegratorChoice::rk2 : IntegratorChoice::rk3);
    cfg.solver = solver == OR_RUSANOV ? SolverChoice::rusanov : SolverChoice::hll;
    cfg.nx = nx;
    cfg.ny = ny;
    cfg.nz = nz;
    cfg.split_x = sx;
    cfg.split_y = sy;
    cfg.split_z = sz;
    cfg.steps = steps;
    cfg.threads = threads;
    double zps = -1.0;
    int rc = guarded([&] {
        RunResult r = run_benchmark(cfg);
        zps = r.zones_per_sec;
        if (final_skinny) out(r.final_state.v, final_skinny);
        if (t_end) *t_end = r.t_end;
        if (l1_rho) *l1_rho = r.errors ? r.errors->l1[0] : -1.0;
    });
    return rc == OR_OK ? zps : -1.0;
}

// harness.cpp:116-193 run_simulation with either a step count or a t_final (<= 0: the
// problem's default stop time); returns the error norms vs the exact solution when the
// problem has one (l1/linf of 5 variables), the end time and the number of steps.
int ref_run_simulation(int problem, int order, int integrator, int solver, int nx, int ny,
                       int nz, long steps, double t_final, int threads, double* l1,
                       double* linf, double* t_end, long* steps_done, double* final_skinny) {
    RunConfig cfg;
    cfg.problem = problem == 0 ? Problem::vortex : (problem == 1 ? Problem::sod : Problem::constant);
    cfg.order = order;
    cfg.integrator = integrator == 0 ? IntegratorChoice::ader_onestep
                                     : (integrator == 2 ? IntegratorChoice::rk2 : IntegratorChoice::rk3);
    cfg.solver = solver == OR_RUSANOV ? SolverChoice::rusanov : SolverChoice::hll;
    cfg.nx = nx;
    cfg.ny = ny;
    cfg.nz = nz;
    cfg.steps = steps;
    cfg.t_final = t_final;
    cfg.threads = threads;
    return guarded([&] {
        RunResult r = run_simulation(cfg);
        if (r.errors)
            for (int q = 0; q < NVAR; ++q) {
                l1[q] = r.errors->l1[q];
                linf[q] = r.errors->linf[q];
            }
        *t_end = r.t_end;
        *steps_done = long(r.steps);
        if (final_skinny) out(r.final_state.v, final_skinny);
    });
}

}  // extern "C"
