/*
 * hydro_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C (C11, serial, -ffp-contract=off) restatement of the reference's
 * space-time update (WENO/MC reconstruction -> ADER predictor -> Rusanov/HLL
 * face fluxes -> flux differencing -> conservative update + CFL min), used
 * as the CHECKER for the CUDA product in tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg. Nothing in the product links or calls it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj). Layouts are the reference's
 * host layouts exactly (fields.hpp:15-128):
 *   modal  [k][j][i][q][m]  (M = 5 at O2, 11 at O3; time mode = M-1)
 *   skinny [k][j][i][q]     (ghosts included; mx = nx + 2*ghost)
 *   face   x:[nz][ny][nx+1][q]  y:[nz][nx][ny+1][q]  z:[ny][nx][nz+1][q]
 *   rate   [nz][ny][nx][q]  (active zones only)
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference library itself (oracle/_ref, compiled from the
 * reference sources by oracle/Makefile) and against the committed golden
 * vectors in tests/golden/ that the reference produced.
 */
#ifndef HYDRO_ORACLE_H
#define HYDRO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_NVAR 5

typedef struct {
    int nx, ny, nz, ghost;
    double dx, dy, dz;
    double origin[3];
} or_geom;

typedef struct {
    double cfac_rho;   /* compression_factor_density, reconstruct.hpp:12 */
    double cfac_other; /* compression_factor_other,   reconstruct.hpp:13 */
    double weno_eps;   /* weno_epsilon,               reconstruct.hpp:14 */
    double weno_w[3];  /* weno_linear_weights,        reconstruct.hpp:15 */
} or_limiter;

enum { OR_OK = 0, OR_UNPHYSICAL = 1, OR_INVALID = 2 };
enum { OR_RUSANOV = 0, OR_HLL = 1, OR_HLLC = 2, OR_HLLI = 3 /* 2, 3: extensions */ };
enum { OR_PERIODIC = 0, OR_OUTFLOW = 1 };

/* message of the last failing call, formatted like the reference's
 * unphysical_error texts (predictor.cpp:82-84, corrector.cpp:53-55,119-120) */
const char* or_last_error(void);

/* ---- pointwise physics (euler.hpp, riemann.hpp, reconstruct.hpp) ---- */
int or_cons_to_prim(const double* u, double gamma, double* prim);
int or_physical_flux(const double* u, int axis, double gamma, double* f);
int or_eval_tstep_ptwise(const double* u, double cfl, double dx, double dy, double dz,
                         double gamma, double* dt);
int or_rusanov_flux(const double* ul, const double* ur, int axis, double gamma, double* f);
int or_hll_flux(const double* ul, const double* ur, int axis, double gamma, double* f);
int or_hllc_flux(const double* ul, const double* ur, int axis, double gamma, double* f);
int or_hlli_flux(const double* ul, const double* ur, int axis, double gamma, double* f);
double or_mc_limiter(double a, double b, double cfac);
void or_weno3_point(const double* s, const or_limiter* cfg, double* ux, double* uxx);
int or_predictor_ptwise(double* zone_v, int modes, double dt, double dx, double dy, double dz,
                        double gamma);

/* ---- patch kernels (serial_ref.cpp / fields.cpp / boundary.cpp) ---- */
void or_skinny_to_modal(const or_geom* g, int modes, const double* skinny, double* modal);
void or_modal_to_skinny(const or_geom* g, int modes, const double* modal, double* skinny);
void or_apply_boundary_skinny(const or_geom* g, int kind, double* skinny);
void or_apply_boundary_modal(const or_geom* g, int modes, int kind, double* modal);
void or_limit_patch_o2(const or_geom* g, double* modal, const or_limiter* cfg);
void or_reconstruct_patch_o3(const or_geom* g, double* modal, const or_limiter* cfg);
/* O4 extension (not in the reference; parity unpinned): WENO-AO(5,3), modes M = 14 */
#define OR_AO_GAMMA_HI 0.85
void or_weno_ao_point(const double* s, const or_limiter* cfg, double* m4);
void or_reconstruct_patch_o4(const or_geom* g, double* modal, const or_limiter* cfg);
int or_predict_patch(const or_geom* g, int modes, double* modal, double dt, double gamma);
void or_zero_temporal_mode(const or_geom* g, int modes, double* modal);
int or_make_flux_axis(const or_geom* g, int modes, const double* modal, int axis, double gamma,
                      int solver, double* out);
void or_make_du_dt(const or_geom* g, const double* fx, const double* fy, const double* fz,
                   double dt, double* rate);
int or_update_u_timestep(const or_geom* g, int modes, double* modal, double* skinny,
                         const double* rate, double cfl, double gamma, double* dt_next);
int or_compute_dt_next(const or_geom* g, int modes, const double* modal, double gamma,
                       double cfl, double* dt_next);

/* ---- stepper (stepper.cpp) ---- */
typedef struct {
    int order;      /* 2 or 3 (4: the WENO-AO extension) */
    int solver;     /* OR_RUSANOV / OR_HLL */
    double gamma;
    or_limiter lim;
} or_params;

/* ader_step: skinny (ghosts filled) -> skinny, sets *dt_next. modal/fx/fy/fz/rate are the
 * caller's scratch (stepper.cpp:49-78). */
int or_ader_step(const or_geom* g, const or_params* par, double* modal, double* skinny,
                 double* fx, double* fy, double* fz, double* rate, double dt, double cfl,
                 double* dt_next);
void or_rk_save_u0(const or_geom* g, const double* skinny, double* stage_u0);
int or_rk_stage(const or_geom* g, const or_params* par, double* modal, double* skinny,
                double* fx, double* fy, double* fz, double* rate, const double* stage_u0,
                double dt, double a, double b);
int or_rk_step(const or_geom* g, const or_params* par, int nstages, double* modal,
               double* skinny, double* fx, double* fy, double* fz, double* rate,
               double* stage_u0, int bc, double dt, double cfl, double* dt_next);

/* ---- problems (problems.cpp), host-side initial conditions ---- */
void or_init_isentropic_vortex(const or_geom* g, double gamma, int order, double t,
                               double* skinny);
void or_init_sod(const or_geom* g, double gamma, double* skinny);
void or_init_constant(const or_geom* g, double gamma, double* skinny);
double or_initial_dt(const or_geom* g, const double* skinny, double gamma, double cfl);

/* ---- whole-run driver over one periodic/outflow patch (harness.cpp:116-193) ----
 * runs `steps` ADER steps (apply_boundary before each), returns the final skinny and the
 * dt sequence used (dts has room for steps+1 entries: dt_0 .. dt_steps). */
int or_run_steps(const or_geom* g, const or_params* par, int bc, double cfl, int steps,
                 double* skinny, double* dts);

#ifdef __cplusplus
}
#endif
#endif
