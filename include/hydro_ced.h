/*
 * hydro_ced.h -- C ABI of the computational-electrodynamics (CED) extension of
 * libhydro_cuda.so: Maxwell's equations in a conducting medium,
 *     dB/dt + curl E = 0,   dD/dt - curl H = -J,   D = eps E, B = mu H, J = sigma E,
 * with face-centred D and B evolved by constrained transport (div B preserved to round-off,
 * div D too where sigma is uniform), edge E and H from the two-dimensional upwind (HLL with
 * speeds +-c, exact for this linear system) multidimensional Riemann solver, WENO3/MC-ADER
 * reconstruction + predictor as on the Euler path, and the stiff conduction source
 * integrated implicitly: an exponential (L-stable, exact for frozen curl H) step
 *     D^{n+1} = exp(-s dt) D^n + phi(s dt) dt (curl H)_h,  s = sigma/eps,
 *     phi(z) = (1 - exp(-z)) / z,
 * in both the ADER predictor (over the half step) and the corrector, so sigma dt >> 1 is
 * stable and the diffusive limit dB/dt = (1/(mu sigma)) lap B is recovered.
 *
 * NOT in the reference (SPEC.md:8 scopes out CED; SPEC.md:293 stiff-source ADER): parity
 * unpinned; checked against a builder-authored numpy restatement (oracle/ced_oracle.py) and
 * by self-consistency (exact plane waves, divergence, energy, stiff limits).
 *
 * State layout: state[6][mz+1][my+1][mx+1] = Dx, Dy, Dz, Bx, By, Bz, each on the LOW face of
 * the zone with the same index along its own axis; sigma[mz+1][my+1][mx+1] per zone
 * (ghosts filled by the library with the boundary kinds). Uniform eps and mu.
 */
#ifndef HYDRO_CED_H
#define HYDRO_CED_H

#include <stddef.h>

#include "hydro_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

#define HC_CED_NVAR 6

typedef struct {
    int order;      /* 2 (MC), 3 (WENO3 + cross terms) -- the reference's ADER structure, second
                     * order in time -- or 4: the local space-time predictor with the conduction
                     * source implicit inside it (Radau IIA collocation, one 4 x 4 block
                     * inversion per zone) and edge E, H at space-time Gauss points (formally
                     * fourth order; ced.cu k_ced4_*) */
    double eps, mu; /* uniform permittivity and permeability; c = 1/sqrt(eps mu) */
    hc_limiter lim;
    int bc[3];      /* HC_PERIODIC / HC_OUTFLOW per axis */
    int device;
} hc_ced_params;

typedef struct hc_ced hc_ced;

int hc_ced_create(const hc_geom* g, const hc_ced_params* p, hc_ced** out);
int hc_ced_destroy(hc_ced* m);
/* host state [6][mz+1][my+1][mx+1] and conductivity [mz+1][my+1][mx+1] (sigma >= 0) */
int hc_ced_upload(hc_ced* m, const double* host_state, const double* host_sigma);
int hc_ced_download(hc_ced* m, double* host_state);
/* the CFL step of the medium: cfl / (c (1/dx + 1/dy + 1/dz)) -- constant in time */
int hc_ced_cfl_dt(hc_ced* m, double cfl, double* dt);
/* t, dt (used for every step), t_final (<= 0: fixed count; the last step is clipped) */
int hc_ced_set_time(hc_ced* m, double t, double dt, double t_final);
/* enqueue n steps: ghosts, cell averages, reconstruction + stiff predictor, edge E and H
 * (3 axes), CT update with the exponential conduction step, t/dt hand-off */
int hc_ced_step(hc_ced* m, int n);
int hc_ced_sync(hc_ced* m, double* t, double* dt, long* steps_done);
/* max over active zones of |div B| * min(d) and |div D| * min(d) */
int hc_ced_max_div(hc_ced* m, double* divb, double* divd);
long hc_ced_launches(hc_ced* m);
/* the cudaStream_t every call of this stepper runs on (for event timing) */
int hc_ced_stream(hc_ced* m, void** stream);

#ifdef __cplusplus
}
#endif
#endif
