// hydro_gpu_shim.cpp -- the drop-in: the reference's hot-path declarations
// (proj/include/hydro/{fields,boundary,reconstruct,predictor,corrector,stepper}.hpp)
// implemented on top of the C ABI of libhydro_cuda.so (include/hydro_cuda.h).
//
// A maintainer links this file INSTEAD OF proj/src/{fields,boundary,reconstruct,predictor,
// corrector,stepper}.cpp; transfer.cpp, harness.cpp, problems.cpp, the tools and the tests
// stay as they are and now run the sm_100a kernels. Every function keeps
// the reference's contract: in-place mutation of caller-owned std::vector storage, the same
// exceptions (unphysical_error with the reference's message text, std::invalid_argument),
// the exact riemann_calls counter (riemann.hpp:23-35, added per face analytically) and the
// StageProfile attribution (device times per stage from CUDA events).
//
// Compiled against the reference headers (-I/root/reference/proj/include); nothing here is
// copied from the reference sources.
#include <chrono>
#include <stdexcept>
#include <string>

#include "hydro/corrector.hpp"
#include "hydro/predictor.hpp"
#include "hydro/reconstruct.hpp"
#include "hydro/stepper.hpp"
#include "hydro_cuda.h"
#include "shim_resident.hpp"

namespace hydro {

namespace {

[[noreturn]] void raise(int rc) {
    char buf[1024];
    hc_last_error(buf, sizeof buf);
    if (rc == HC_UNPHYSICAL) throw unphysical_error(buf);
    if (rc == HC_INVALID) throw std::invalid_argument(buf);
    throw std::runtime_error(std::string("libhydro_cuda: ") + buf);
}
inline void check(int rc) {
    if (rc != HC_OK) raise(rc);
}

hc_geom to_hc(const PatchGeometry& g) {
    hc_geom h;
    h.nx = g.nx;
    h.ny = g.ny;
    h.nz = g.nz;
    h.ghost = g.ghost;
    h.dx = g.dx;
    h.dy = g.dy;
    h.dz = g.dz;
    h.origin[0] = g.origin[0];
    h.origin[1] = g.origin[1];
    h.origin[2] = g.origin[2];
    return h;
}

// For the two entry points that carry no geometry (they touch every zone, so only the
// total shape matters): any ghost width reproducing mx, my, mz.
hc_geom shape_geom(int mx, int my, int mz) {
    hc_geom h{};
    h.ghost = 2;
    h.nx = mx - 4;
    h.ny = my - 4;
    h.nz = mz - 4;
    h.dx = h.dy = h.dz = 1.0;
    return h;
}

hc_limiter to_hc(const LimiterConfig& c) {
    hc_limiter l;
    l.cfac_rho = c.compression_factor_density;
    l.cfac_other = c.compression_factor_other;
    l.weno_eps = c.weno_epsilon;
    for (int i = 0; i < 3; ++i) l.weno_w[i] = c.weno_linear_weights[i];
    return l;
}

hc_params to_hc(const StepParams& p) {
    hc_params h;
    h.order = p.order;
    h.solver = p.solver == SolverChoice::rusanov ? HC_RUSANOV : HC_HLL;
    h.gamma = p.gas.gamma;
    h.lim = to_hc(p.limiter);
    return h;
}

int kind(BoundaryKind k) { return k == BoundaryKind::periodic ? HC_PERIODIC : HC_OUTFLOW; }

void count_faces(const PatchGeometry& g, int sweeps_per_axis) {
    std::uint64_t faces = std::uint64_t(g.nx + 1) * g.ny * g.nz +
                          std::uint64_t(g.ny + 1) * g.nx * g.nz +
                          std::uint64_t(g.nz + 1) * g.nx * g.ny;
    detail::riemann_calls.fetch_add(faces * sweeps_per_axis, std::memory_order_relaxed);
}

void add_profile(StageProfile* prof, const double* s) {
    if (!prof) return;
    prof->reconstruct += s[0];
    prof->predict += s[1];
    prof->flux += s[2];
    prof->rate += s[3];
    prof->update += s[4];
    prof->transfer += s[5];
}

// Host wall time of a shim call that has no per-kernel device split (the reference's
// StageTimer attribution in rk_step, stepper.cpp:145-156): adds the seconds to one field.
class CallTimer {
  public:
    explicit CallTimer(double* field) : f_(field), t0_(std::chrono::steady_clock::now()) {}
    ~CallTimer() {
        if (f_)
            *f_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
    }

  private:
    double* f_;
    std::chrono::steady_clock::time_point t0_;
};

}  // namespace

// residency hook (shim_resident.hpp): no-op unless hydro_gpu_transfer.cpp is linked
__attribute__((weak)) void shim_host_touch(const void*) {}
#define TOUCH(x) shim_host_touch((x).v.data())

// ------------------------------------------------------------------ fields.hpp:137-145

void require_compatible(const SkinnyState& s, const ModalState& m) {
    if (s.mx != m.mx || s.my != m.my || s.mz != m.mz)
        throw std::invalid_argument("skinny/modal shape mismatch");
}

void skinny_to_modal(const SkinnyState& skinny, ModalState& modal) {
    TOUCH(skinny);
    TOUCH(modal);
    require_compatible(skinny, modal);
    hc_geom g = shape_geom(modal.mx, modal.my, modal.mz);
    check(hc_skinny_to_modal(&g, modal.modes, skinny.v.data(), modal.v.data()));
}

void modal_to_skinny(const ModalState& modal, const PatchGeometry& g, SkinnyState& skinny) {
    TOUCH(modal);
    TOUCH(skinny);
    require_compatible(skinny, modal);
    hc_geom h = to_hc(g);
    check(hc_modal_to_skinny(&h, modal.modes, modal.v.data(), skinny.v.data()));
}

// ---------------------------------------------------------------- boundary.hpp:10-15

void apply_boundary(SkinnyState& skinny, const PatchGeometry& g, BoundaryKind k) {
    TOUCH(skinny);
    hc_geom h = to_hc(g);
    check(hc_apply_boundary_skinny(&h, kind(k), skinny.v.data()));
}

void apply_boundary(ModalState& modal, const PatchGeometry& g, BoundaryKind k) {
    TOUCH(modal);
    hc_geom h = to_hc(g);
    check(hc_apply_boundary_modal(&h, modal.modes, kind(k), modal.v.data()));
}

// ------------------------------------------------------------- reconstruct.hpp:85-97

void limit_patch_o2(ModalState& modal, const PatchGeometry& g, const LimiterConfig& cfg) {
    TOUCH(modal);
    hc_geom h = to_hc(g);
    hc_limiter l = to_hc(cfg);
    check(hc_limit_patch_o2(&h, modal.v.data(), &l));
}

void reconstruct_patch_o3(ModalState& modal, const PatchGeometry& g, const LimiterConfig& cfg) {
    TOUCH(modal);
    hc_geom h = to_hc(g);
    hc_limiter l = to_hc(cfg);
    check(hc_reconstruct_patch_o3(&h, modal.v.data(), &l));
}

void reconstruct_patch(ModalState& modal, const PatchGeometry& g, const LimiterConfig& cfg,
                       int order) {
    if (order == 2)
        limit_patch_o2(modal, g, cfg);
    else
        reconstruct_patch_o3(modal, g, cfg);
}

// --------------------------------------------------------------- predictor.hpp:29-47

void predictor_ptwise(ZoneModal& zone, double dt, double dx, double dy, double dz,
                      const GasModel& gas) {
    check(hc_predictor_ptwise(zone.v, zone.modes, dt, dx, dy, dz, gas.gamma));
}

void predict_patch(ModalState& modal, const TimeState& time, const PatchGeometry& g,
                   const GasModel& gas) {
    TOUCH(modal);
    hc_geom h = to_hc(g);
    check(hc_predict_patch(&h, modal.modes, modal.v.data(), time.dt, gas.gamma));
}

void zero_temporal_mode(ModalState& modal) {
    TOUCH(modal);
    hc_geom g = shape_geom(modal.mx, modal.my, modal.mz);
    check(hc_zero_temporal_mode(&g, modal.modes, modal.v.data()));
}

// --------------------------------------------------------------- corrector.hpp:13-27

void make_flux_axis(const ModalState& modal, Axis axis, const PatchGeometry& g,
                    const GasModel& gas, SolverChoice solver, FaceFlux& out) {
    TOUCH(modal);
    TOUCH(out);
    hc_geom h = to_hc(g);
    int rc = hc_make_flux_axis(&h, modal.modes, modal.v.data(), int(axis), gas.gamma,
                               solver == SolverChoice::rusanov ? HC_RUSANOV : HC_HLL,
                               out.v.data());
    std::uint64_t faces = std::uint64_t(out.n0) * out.n1 * out.n2;
    detail::riemann_calls.fetch_add(faces, std::memory_order_relaxed);
    check(rc);
}

void make_du_dt(const FluxSet& fluxes, const TimeState& time, const PatchGeometry& g,
                RateField& rate) {
    TOUCH(fluxes.fx);
    TOUCH(rate);
    hc_geom h = to_hc(g);
    check(hc_make_du_dt(&h, fluxes.fx.v.data(), fluxes.fy.v.data(), fluxes.fz.v.data(),
                        time.dt, rate.v.data()));
}

void update_u_timestep(ModalState& modal, SkinnyState& skinny, const RateField& rate,
                       TimeState& time, const PatchGeometry& g, const GasModel& gas) {
    TOUCH(modal);
    TOUCH(skinny);
    TOUCH(rate);
    hc_geom h = to_hc(g);
    double dtn = 0.0;
    check(hc_update_u_timestep(&h, modal.modes, modal.v.data(), skinny.v.data(), rate.v.data(),
                               time.cfl, gas.gamma, &dtn));
    time.dt_next = dtn;
}

// ----------------------------------------------------------------- stepper.hpp:58-91

double compute_dt_next(const ModalState& modal, const PatchGeometry& g, const GasModel& gas,
                       double cfl) {
    TOUCH(modal);
    hc_geom h = to_hc(g);
    double dtn = 0.0;
    check(hc_compute_dt_next(&h, modal.modes, modal.v.data(), gas.gamma, cfl, &dtn));
    return dtn;
}

void ader_step(ModalState& modal, SkinnyState& skinny, TimeState& time, const PatchGeometry& g,
               const StepParams& par, StepScratch& scratch, StageProfile* prof) {
    TOUCH(modal);
    TOUCH(skinny);
    TOUCH(scratch.rate);
    hc_geom h = to_hc(g);
    hc_params p = to_hc(par);
    double dtn = 0.0, stage[6] = {0, 0, 0, 0, 0, 0};
    int rc = hc_ader_step_timed(&h, &p, modal.v.data(), skinny.v.data(),
                                scratch.fluxes.fx.v.data(), scratch.fluxes.fy.v.data(),
                                scratch.fluxes.fz.v.data(), scratch.rate.v.data(), time.dt,
                                time.cfl, &dtn, stage);
    if (rc == HC_OK || rc == HC_UNPHYSICAL) {
        // the reference's sweeps ran (and counted) unless the predictor threw first
        char buf[256];
        hc_last_error(buf, sizeof buf);
        if (rc == HC_OK || std::string(buf).rfind("predictor", 0) != 0) count_faces(g, 1);
    }
    check(rc);
    add_profile(prof, stage);
    time.dt_next = dtn;
}

const std::vector<RkStage>& rk_stages(IntegratorChoice k) {
    static const std::vector<RkStage> heun = {{0.0, 1.0}, {0.5, 0.5}};
    static const std::vector<RkStage> ssp3 = {{0.0, 1.0}, {0.75, 0.25}, {1.0 / 3.0, 2.0 / 3.0}};
    if (k == IntegratorChoice::rk2) return heun;
    if (k == IntegratorChoice::rk3) return ssp3;
    throw std::invalid_argument("rk_stages called for a non-RK integrator");
}

void rk_save_u0(const SkinnyState& skinny, const PatchGeometry& g, StepScratch& scratch) {
    TOUCH(skinny);
    TOUCH(scratch.stage_u0);
    hc_geom h = to_hc(g);
    check(hc_rk_save_u0(&h, skinny.v.data(), scratch.stage_u0.v.data()));
}

void rk_stage(ModalState& modal, SkinnyState& skinny, TimeState& time, const PatchGeometry& g,
              const StepParams& par, StepScratch& scratch, RkStage stage, StageProfile* prof) {
    TOUCH(modal);
    TOUCH(skinny);
    TOUCH(scratch.stage_u0);
    hc_geom h = to_hc(g);
    hc_params p = to_hc(par);
    double s[6] = {0, 0, 0, 0, 0, 0};
    int rc = hc_rk_stage_timed(&h, &p, modal.v.data(), skinny.v.data(),
                               scratch.fluxes.fx.v.data(), scratch.fluxes.fy.v.data(),
                               scratch.fluxes.fz.v.data(), scratch.rate.v.data(),
                               scratch.stage_u0.v.data(), time.dt, stage.a, stage.b, s);
    if (rc == HC_OK || rc == HC_UNPHYSICAL) count_faces(g, 1);
    check(rc);
    add_profile(prof, s);
}

void rk_step(ModalState& modal, SkinnyState& skinny, TimeState& time, const PatchGeometry& g,
             const StepParams& par, StepScratch& scratch, BoundaryKind bc, StageProfile* prof) {
    rk_save_u0(skinny, g, scratch);
    for (const RkStage& stage : rk_stages(par.integrator)) {
        {
            CallTimer t(prof ? &prof->transfer : nullptr);  // stepper.cpp:148-151
            apply_boundary(skinny, g, bc);
        }
        rk_stage(modal, skinny, time, g, par, scratch, stage, prof);
    }
    CallTimer t(prof ? &prof->update : nullptr);  // stepper.cpp:154-155
    time.dt_next = compute_dt_next(modal, g, par.gas, time.cfl);
}

}  // namespace hydro
