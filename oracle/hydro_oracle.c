/*
 * hydro_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Serial C restatement of the reference algorithm. Build with -ffp-contract=off so the
 * arithmetic matches the reference build (proj/CMakeLists.txt:12-15) bit for bit. The
 * expression shapes below follow the reference statements cited beside each function,
 * because IEEE results depend on the exact association of every + - * /.
 */
#include "hydro_oracle.h"

#include <math.h>
#include <stddef.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NV OR_NVAR

static char g_err[512];
const char* or_last_error(void) { return g_err; }

/* std::to_string(double) is "%f" (C++ [string.conversions]) */
static int fail_value(const char* what, double v) {
    snprintf(g_err, sizeof g_err, "%s %f", what, v);
    return OR_UNPHYSICAL;
}
static int prefix_error(const char* prefix) {
    char tmp[512];
    snprintf(tmp, sizeof tmp, "%.200s%.300s", prefix, g_err);
    memcpy(g_err, tmp, sizeof g_err);
    return OR_UNPHYSICAL;
}

static inline size_t zoff(const or_geom* g, int k, int j, int i) {
    int mx = g->nx + 2 * g->ghost, my = g->ny + 2 * g->ghost;
    return ((size_t)k * my + j) * mx + i;
}
static inline int gmx(const or_geom* g) { return g->nx + 2 * g->ghost; }
static inline int gmy(const or_geom* g) { return g->ny + 2 * g->ghost; }
static inline int gmz(const or_geom* g) { return g->nz + 2 * g->ghost; }

/* modes per variable: geometry.hpp:23-27 (5 at O2, 11 at O3); 14 at the O4 extension
 * (mean, 3 slopes, 3 quadratic, 3 cubic, 3 quartic, temporal) */
static int modes_of(int order) { return order == 2 ? 5 : (order == 3 ? 11 : 14); }

/* ------------------------------------------------------------------ euler.hpp */

/* euler.hpp:37-50 cons_to_prim */
int or_cons_to_prim(const double* u, double gamma, double* q) {
    if (!(u[0] > 0.0)) return fail_value("non-positive density", u[0]);
    double inv_rho = 1.0 / u[0];
    q[0] = u[0];
    q[1] = u[1] * inv_rho;
    q[2] = u[2] * inv_rho;
    q[3] = u[3] * inv_rho;
    q[4] = (gamma - 1.0) * (u[4] - 0.5 * (u[1] * q[1] + u[2] * q[2] + u[3] * q[3]));
    if (!(q[4] > 0.0)) return fail_value("non-positive pressure", q[4]);
    return OR_OK;
}

/* euler.hpp:62-64 sound_speed */
static double sound_speed(const double* q, double gamma) { return sqrt(gamma * q[4] / q[0]); }

/* euler.hpp:72-87 physical_flux */
int or_physical_flux(const double* u, int axis, double gamma, double* f) {
    double q[5];
    int rc = or_cons_to_prim(u, gamma, q);
    if (rc) return rc;
    double un = q[1 + axis];
    f[0] = u[0] * un;
    f[1] = u[1] * un;
    f[2] = u[2] * un;
    f[3] = u[3] * un;
    f[4] = (u[4] + q[4]) * un;
    f[1 + axis] += q[4];
    return OR_OK;
}

/* euler.hpp:89-92 max_signal_speed */
static int max_signal_speed(const double* u, int axis, double gamma, double* s) {
    double q[5];
    int rc = or_cons_to_prim(u, gamma, q);
    if (rc) return rc;
    *s = fabs(q[1 + axis]) + sound_speed(q, gamma);
    return OR_OK;
}

/* euler.hpp:96-104 eval_tstep_ptwise */
int or_eval_tstep_ptwise(const double* u, double cfl, double dx, double dy, double dz,
                         double gamma, double* dt) {
    double q[5];
    int rc = or_cons_to_prim(u, gamma, q);
    if (rc) return rc;
    double cs = sound_speed(q, gamma);
    double sx = fabs(q[1]) + cs;
    double sy = fabs(q[2]) + cs;
    double sz = fabs(q[3]) + cs;
    *dt = cfl / (sx / dx + sy / dy + sz / dz);
    return OR_OK;
}

/* std::min / std::max semantics: min(a,b) = (b < a) ? b : a ; max(a,b) = (a < b) ? b : a */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

/* ---------------------------------------------------------------- riemann.hpp */

/* riemann.hpp:37-51 rusanov_flux */
int or_rusanov_flux(const double* ul, const double* ur, int axis, double gamma, double* f) {
    double fl[5], fr[5], sl, sr;
    int rc;
    if ((rc = or_physical_flux(ul, axis, gamma, fl))) return rc;
    if ((rc = or_physical_flux(ur, axis, gamma, fr))) return rc;
    if ((rc = max_signal_speed(ul, axis, gamma, &sl))) return rc;
    if ((rc = max_signal_speed(ur, axis, gamma, &sr))) return rc;
    double s = smax(sl, sr);
    for (int q = 0; q < 5; ++q) f[q] = 0.5 * (fl[q] + fr[q]) - 0.5 * s * (ur[q] - ul[q]);
    return OR_OK;
}

/* riemann.hpp:55-86 hll_flux (Davis speeds, degenerate-fan fallback) */
int or_hll_flux(const double* ul, const double* ur, int axis, double gamma, double* f) {
    double ql[5], qr[5];
    int rc;
    if ((rc = or_cons_to_prim(ul, gamma, ql))) return rc;
    if ((rc = or_cons_to_prim(ur, gamma, qr))) return rc;
    double cl = sound_speed(ql, gamma);
    double cr = sound_speed(qr, gamma);
    double unl = ql[1 + axis];
    double unr = qr[1 + axis];
    double sl = smin(unl - cl, unr - cr);
    double sr = smax(unl + cl, unr + cr);
    double fl[5], fr[5];
    if ((rc = or_physical_flux(ul, axis, gamma, fl))) return rc;
    if (sl >= 0.0) {
        memcpy(f, fl, sizeof fl);
        return OR_OK;
    }
    if ((rc = or_physical_flux(ur, axis, gamma, fr))) return rc;
    if (sr <= 0.0) {
        memcpy(f, fr, sizeof fr);
        return OR_OK;
    }
    if (sr == sl) {
        for (int q = 0; q < 5; ++q) f[q] = 0.5 * (fl[q] + fr[q]);
        return OR_OK;
    }
    double inv = 1.0 / (sr - sl);
    for (int q = 0; q < 5; ++q) f[q] = (sr * fl[q] - sl * fr[q] + sl * sr * (ur[q] - ul[q])) * inv;
    return OR_OK;
}

/* HLLC (Toro, Spruce & Speares 1994; Toro, "Riemann Solvers and Numerical Methods", 3rd ed.,
 * sec. 10.4) with the same Davis speed estimates as hll_flux above. NOT in the reference
 * (SPEC.md:339 excludes HLLC/HLLI): this restatement is builder-authored -- parity unpinned;
 * it pins the CUDA twin's implementation (same expression shapes, bitwise), while the
 * physics is checked by self-consistency (exact stationary contact, F(U,U) = F(U)). */
int or_hllc_flux(const double* ul, const double* ur, int axis, double gamma, double* f) {
    double ql[5], qr[5];
    int rc;
    if ((rc = or_cons_to_prim(ul, gamma, ql))) return rc;
    if ((rc = or_cons_to_prim(ur, gamma, qr))) return rc;
    double cl = sound_speed(ql, gamma);
    double cr = sound_speed(qr, gamma);
    double unl = ql[1 + axis];
    double unr = qr[1 + axis];
    double sl = smin(unl - cl, unr - cr);
    double sr = smax(unl + cl, unr + cr);
    double fl[5], fr[5];
    if ((rc = or_physical_flux(ul, axis, gamma, fl))) return rc;
    if ((rc = or_physical_flux(ur, axis, gamma, fr))) return rc;
    if (sl >= 0.0) {
        memcpy(f, fl, sizeof fl);
        return OR_OK;
    }
    if (sr <= 0.0) {
        memcpy(f, fr, sizeof fr);
        return OR_OK;
    }
    double dl = ql[0] * (sl - unl);
    double dr = qr[0] * (sr - unr);
    double ss = (qr[4] - ql[4] + dl * unl - dr * unr) / (dl - dr);
    const int left = ss >= 0.0;
    const double* uk = left ? ul : ur;
    const double* qk = left ? ql : qr;
    const double* fk = left ? fl : fr;
    double sk = left ? sl : sr, dk = left ? dl : dr, unk = left ? unl : unr;
    double fac = dk / (sk - ss);
    double us[5];
    us[0] = fac;
    us[1] = fac * qk[1];
    us[2] = fac * qk[2];
    us[3] = fac * qk[3];
    us[1 + axis] = fac * ss;
    us[4] = fac * (uk[4] / qk[0] + (ss - unk) * (ss + qk[4] / dk));
    for (int q = 0; q < 5; ++q) f[q] = fk[q] + sk * (us[q] - uk[q]);
    return OR_OK;
}

/* HLLI (Dumbser & Balsara 2016, J. Comput. Phys. 304): HLL with the anti-diffusive term of
 * the linearly degenerate fields (entropy wave, two shear waves; eigenvalue u_n) at the
 * arithmetic-average state,
 *   F = F_HLL - S_L S_R / (S_R - S_L) * sum_k delta_k r_k (l_k . dU),
 *   delta = 1 - min(u_n, 0) / S_L - max(u_n, 0) / S_R.
 * NOT in the reference: builder-authored restatement -- parity unpinned. */
int or_hlli_flux(const double* ul, const double* ur, int axis, double gamma, double* f) {
    double ql[5], qr[5];
    int rc;
    if ((rc = or_cons_to_prim(ul, gamma, ql))) return rc;
    if ((rc = or_cons_to_prim(ur, gamma, qr))) return rc;
    double cl = sound_speed(ql, gamma);
    double cr = sound_speed(qr, gamma);
    double unl = ql[1 + axis];
    double unr = qr[1 + axis];
    double sl = smin(unl - cl, unr - cr);
    double sr = smax(unl + cl, unr + cr);
    double fl[5], fr[5];
    if ((rc = or_physical_flux(ul, axis, gamma, fl))) return rc;
    if ((rc = or_physical_flux(ur, axis, gamma, fr))) return rc;
    if (sl >= 0.0) {
        memcpy(f, fl, sizeof fl);
        return OR_OK;
    }
    if (sr <= 0.0) {
        memcpy(f, fr, sizeof fr);
        return OR_OK;
    }
    double inv = 1.0 / (sr - sl);
    double du[5], ua[5], qa[5];
    for (int q = 0; q < 5; ++q) {
        du[q] = ur[q] - ul[q];
        ua[q] = 0.5 * (ul[q] + ur[q]);
    }
    if ((rc = or_cons_to_prim(ua, gamma, qa))) return rc;
    double b1 = (gamma - 1.0) / (gamma * qa[4] / qa[0]);
    double v2 = qa[1] * qa[1] + qa[2] * qa[2] + qa[3] * qa[3];
    double un = qa[1 + axis];
    double ae = (1.0 - 0.5 * b1 * v2) * du[0] + b1 * (qa[1] * du[1] + qa[2] * du[2] + qa[3] * du[3]) -
                b1 * du[4];
    double corr[5];
    corr[0] = ae;
    corr[1] = ae * qa[1];
    corr[2] = ae * qa[2];
    corr[3] = ae * qa[3];
    corr[4] = ae * (0.5 * v2);
    for (int t = 1; t <= 2; ++t) {
        int c = (axis + t) % 3;
        double at = du[1 + c] - qa[1 + c] * du[0];
        corr[1 + c] = corr[1 + c] + at;
        corr[4] = corr[4] + at * qa[1 + c];
    }
    double delta = 1.0 - smin(un, 0.0) / sl - smax(un, 0.0) / sr;
    double coef = sl * sr * inv * delta;
    for (int q = 0; q < 5; ++q)
        f[q] = (sr * fl[q] - sl * fr[q] + sl * sr * (ur[q] - ul[q])) * inv - coef * corr[q];
    return OR_OK;
}

static int riemann(int solver, const double* ul, const double* ur, int axis, double gamma,
                   double* f) {
    if (solver == OR_HLLI) return or_hlli_flux(ul, ur, axis, gamma, f);
    if (solver == OR_HLLC) return or_hllc_flux(ul, ur, axis, gamma, f);
    return solver == OR_RUSANOV ? or_rusanov_flux(ul, ur, axis, gamma, f)
                                : or_hll_flux(ul, ur, axis, gamma, f);
}

/* ------------------------------------------------------------ reconstruct.hpp */

/* reconstruct.hpp:33-36 mc_limiter; std::min(initializer_list) keeps the first minimum */
double or_mc_limiter(double a, double b, double cfac) {
    double m = 0.5 * fabs(a + b);
    double c1 = cfac * fabs(a);
    double c2 = cfac * fabs(b);
    if (c1 < m) m = c1;
    if (c2 < m) m = c2;
    return m * (copysign(0.5, a) + copysign(0.5, b));
}

/* reconstruct.hpp:46-73 weno3_point */
void or_weno3_point(const double* s, const or_limiter* cfg, double* ux, double* uxx) {
    double d0 = s[1] - s[0], d1 = s[2] - s[1], d2 = s[3] - s[2], d3 = s[4] - s[3];
    double ux_l = 0.5 * (3.0 * d1 - d0);
    double uxx_l = 0.5 * (d1 - d0);
    double ux_c = 0.5 * (d1 + d2);
    double uxx_c = 0.5 * (d2 - d1);
    double ux_r = 0.5 * (3.0 * d2 - d3);
    double uxx_r = 0.5 * (d3 - d2);
    const double k2 = 13.0 / 3.0;
    double is_l = ux_l * ux_l + k2 * uxx_l * uxx_l;
    double is_c = ux_c * ux_c + k2 * uxx_c * uxx_c;
    double is_r = ux_r * ux_r + k2 * uxx_r * uxx_r;
    double el = cfg->weno_eps + is_l;
    double ec = cfg->weno_eps + is_c;
    double er = cfg->weno_eps + is_r;
    double al = cfg->weno_w[0] / (el * el);
    double ac = cfg->weno_w[1] / (ec * ec);
    double ar = cfg->weno_w[2] / (er * er);
    double inv = 1.0 / (al + ac + ar);
    *ux = (al * ux_l + ac * ux_c + ar * ux_r) * inv;
    *uxx = (al * uxx_l + ac * uxx_c + ar * uxx_r) * inv;
}

/* reconstruct.hpp:79-83 extrapolate_to_face */
static inline double extrap(const double* zv, int modes, int axis, double side) {
    double val = zv[0] + side * 0.5 * zv[1 + axis];
    if (modes >= 11) val += (1.0 / 6.0) * zv[4 + axis];
    if (modes == 14) {  /* O4 extension: P3(1/2) = 1/20, P4(1/2) = 1/70 */
        val += side * (1.0 / 20.0) * zv[7 + axis];
        val += (1.0 / 70.0) * zv[10 + axis];
    }
    return val;
}

/* ------------------------------------------------------------------- fields.cpp */

/* serial_ref.cpp:5-12 / fields.cpp:12-23 */
void or_skinny_to_modal(const or_geom* g, int modes, const double* skinny, double* modal) {
    size_t nz = (size_t)gmx(g) * gmy(g) * gmz(g);
    for (size_t z = 0; z < nz; ++z)
        for (int q = 0; q < NV; ++q) modal[(z * NV + q) * modes] = skinny[z * NV + q];
}

/* serial_ref.cpp:14-22 / fields.cpp:25-36 */
void or_modal_to_skinny(const or_geom* g, int modes, const double* modal, double* skinny) {
    const int gh = g->ghost;
    for (int k = gh; k < gh + g->nz; ++k)
        for (int j = gh; j < gh + g->ny; ++j)
            for (int i = gh; i < gh + g->nx; ++i) {
                size_t z = zoff(g, k, j, i);
                for (int q = 0; q < NV; ++q) skinny[z * NV + q] = modal[(z * NV + q) * modes];
            }
}

/* ----------------------------------------------------------------- boundary.cpp */

/* boundary.cpp:7-10 map_index */
static inline int map_index(int a, int n, int kind) {
    if (kind == OR_PERIODIC) return ((a % n) + n) % n;
    return a < 0 ? 0 : (a >= n ? n - 1 : a);
}

/* boundary.cpp:14-39 fill_ghosts: x pass (active y,z), y pass (full x), z pass (full x,y) */
static void fill_ghosts(const or_geom* g, int kind, double* base, int stride, int nq,
                        int qstride) {
    const int gh = g->ghost, mx = gmx(g), my = gmy(g), mz = gmz(g);
#define COPYZ(dst, src)                                                                      \
    do {                                                                                     \
        for (int q = 0; q < nq; ++q) base[(dst) * stride + q * qstride] =                    \
            base[(src) * stride + q * qstride];                                              \
    } while (0)
    for (int k = gh; k < gh + g->nz; ++k)
        for (int j = gh; j < gh + g->ny; ++j)
            for (int i = 0; i < mx; ++i) {
                if (i >= gh && i < gh + g->nx) continue;
                COPYZ(zoff(g, k, j, i), zoff(g, k, j, gh + map_index(i - gh, g->nx, kind)));
            }
    for (int k = gh; k < gh + g->nz; ++k)
        for (int j = 0; j < my; ++j) {
            if (j >= gh && j < gh + g->ny) continue;
            int js = gh + map_index(j - gh, g->ny, kind);
            for (int i = 0; i < mx; ++i) COPYZ(zoff(g, k, j, i), zoff(g, k, js, i));
        }
    for (int k = 0; k < mz; ++k) {
        if (k >= gh && k < gh + g->nz) continue;
        int ks = gh + map_index(k - gh, g->nz, kind);
        for (int j = 0; j < my; ++j)
            for (int i = 0; i < mx; ++i) COPYZ(zoff(g, k, j, i), zoff(g, ks, j, i));
    }
#undef COPYZ
}

/* boundary.cpp:43-49 */
void or_apply_boundary_skinny(const or_geom* g, int kind, double* skinny) {
    fill_ghosts(g, kind, skinny, NV, NV, 1);
}
/* boundary.cpp:51-58 */
void or_apply_boundary_modal(const or_geom* g, int modes, int kind, double* modal) {
    fill_ghosts(g, kind, modal, NV * modes, NV, modes);
}

/* -------------------------------------------------------------- reconstruct.cpp */

/* serial_ref.cpp:24-43 limit_patch_o2 (active + one ring) */
void or_limit_patch_o2(const or_geom* g, double* modal, const or_limiter* cfg) {
    const int gh = g->ghost, M = 5;
    const ptrdiff_t sx = (ptrdiff_t)NV * M, sy = sx * gmx(g), sz = sy * gmy(g);
    for (int k = gh - 1; k < gh + g->nz + 1; ++k)
        for (int j = gh - 1; j < gh + g->ny + 1; ++j)
            for (int i = gh - 1; i < gh + g->nx + 1; ++i)
                for (int q = 0; q < NV; ++q) {
                    double cfac = q == 0 ? cfg->cfac_rho : cfg->cfac_other;
                    double* zc = modal + zoff(g, k, j, i) * NV * M + q * M;
                    double u0 = zc[0];
                    zc[1] = or_mc_limiter(zc[sx] - u0, u0 - zc[-sx], cfac);
                    zc[2] = or_mc_limiter(zc[sy] - u0, u0 - zc[-sy], cfac);
                    zc[3] = or_mc_limiter(zc[sz] - u0, u0 - zc[-sz], cfac);
                }
}

/* serial_ref.cpp:45-82 reconstruct_patch_o3: pass 1 on active+ring, cross modes on active */
void or_reconstruct_patch_o3(const or_geom* g, double* modal, const or_limiter* cfg) {
    const int gh = g->ghost, M = 11;
    const ptrdiff_t sx = (ptrdiff_t)NV * M, sy = sx * gmx(g), sz = sy * gmy(g);
    for (int k = gh - 1; k < gh + g->nz + 1; ++k)
        for (int j = gh - 1; j < gh + g->ny + 1; ++j)
            for (int i = gh - 1; i < gh + g->nx + 1; ++i)
                for (int q = 0; q < NV; ++q) {
                    double* zc = modal + zoff(g, k, j, i) * NV * M + q * M;
                    double s[5], wx[2], wy[2], wz[2];
                    for (int m = -2; m <= 2; ++m) s[m + 2] = zc[m * sx];
                    or_weno3_point(s, cfg, &wx[0], &wx[1]);
                    for (int m = -2; m <= 2; ++m) s[m + 2] = zc[m * sy];
                    or_weno3_point(s, cfg, &wy[0], &wy[1]);
                    for (int m = -2; m <= 2; ++m) s[m + 2] = zc[m * sz];
                    or_weno3_point(s, cfg, &wz[0], &wz[1]);
                    zc[1] = wx[0];
                    zc[2] = wy[0];
                    zc[3] = wz[0];
                    zc[4] = wx[1];
                    zc[5] = wy[1];
                    zc[6] = wz[1];
                }
    for (int k = gh; k < gh + g->nz; ++k)
        for (int j = gh; j < gh + g->ny; ++j)
            for (int i = gh; i < gh + g->nx; ++i)
                for (int q = 0; q < NV; ++q) {
                    double* zc = modal + zoff(g, k, j, i) * NV * M + q * M;
                    zc[7] = 0.25 * ((zc[sy + 1] - zc[-sy + 1]) + (zc[sx + 2] - zc[-sx + 2]));
                    zc[8] = 0.25 * ((zc[sz + 2] - zc[-sz + 2]) + (zc[sy + 3] - zc[-sy + 3]));
                    zc[9] = 0.25 * ((zc[sx + 3] - zc[-sx + 3]) + (zc[sz + 1] - zc[-sz + 1]));
                }
}

/* O4 extension (NOT in the reference: geometry.hpp:13-27 admits orders 2 and 3 only; parity
 * unpinned): WENO-AO(5,3) (Balsara, Garain & Shu 2016) on s0..s4 = u[i-2..i+2]. The quartic
 * of the 5-cell stencil in the basis P1 = x, P2 = x^2 - 1/12, P3 = x^3 - 3x/20,
 * P4 = x^4 - 3x^2/14 + 3/560 (zero mean on the cell), blended with the three WENO3
 * quadratics (weights gamma_hi = 0.85 and (1 - gamma_hi) * weno_w[k]) by Jiang-Shu weights
 * of the smoothness indicators sum_l int (d^l P)^2:
 *   beta_hi = (u1 + u3/10)^2 + 13/3 (u2 + 123/455 u4)^2 + 781/20 u3^2 + 1421461/2275 u4^2
 *   P_AO = (w_hi / gamma_hi) (P_hi - sum_k gamma_k P_k) + sum_k w_k P_k. */
void or_weno_ao_point(const double* s, const or_limiter* cfg, double* m) {
    const double ghi = OR_AO_GAMMA_HI;
    double o1 = 0.5 * (s[3] - s[1]), o2 = 0.5 * (s[4] - s[0]);
    double e1 = 0.5 * (s[3] + s[1]) - s[2], e2 = 0.5 * (s[4] + s[0]) - s[2];
    double u3 = (o2 - 2.0 * o1) * (1.0 / 6.0);
    double u1 = o1 - (11.0 / 10.0) * u3;
    double u4 = (e2 - 4.0 * e1) * (1.0 / 12.0);
    double u2 = e1 - (9.0 / 7.0) * u4;
    double d0 = s[1] - s[0], d1 = s[2] - s[1], d2 = s[3] - s[2], d3 = s[4] - s[3];
    double ux_l = 0.5 * (3.0 * d1 - d0), uxx_l = 0.5 * (d1 - d0);
    double ux_c = 0.5 * (d1 + d2), uxx_c = 0.5 * (d2 - d1);
    double ux_r = 0.5 * (3.0 * d2 - d3), uxx_r = 0.5 * (d3 - d2);
    const double k2 = 13.0 / 3.0;
    double ta = u1 + (1.0 / 10.0) * u3, tb = u2 + (123.0 / 455.0) * u4;
    double b_hi = ta * ta + k2 * tb * tb + (781.0 / 20.0) * u3 * u3 +
                  (1421461.0 / 2275.0) * u4 * u4;
    double b_l = ux_l * ux_l + k2 * uxx_l * uxx_l;
    double b_c = ux_c * ux_c + k2 * uxx_c * uxx_c;
    double b_r = ux_r * ux_r + k2 * uxx_r * uxx_r;
    double gl = (1.0 - ghi) * cfg->weno_w[0], gc = (1.0 - ghi) * cfg->weno_w[1],
           gr = (1.0 - ghi) * cfg->weno_w[2];
    double eh = cfg->weno_eps + b_hi, el = cfg->weno_eps + b_l, ec = cfg->weno_eps + b_c,
           er = cfg->weno_eps + b_r;
    double ah = ghi / (eh * eh), al = gl / (el * el), ac = gc / (ec * ec), ar = gr / (er * er);
    double inv = 1.0 / (ah + al + ac + ar);
    double wh = ah * inv, wl = al * inv, wc = ac * inv, wr = ar * inv;
    double ratio = wh / ghi;
    m[0] = ratio * (u1 - (gl * ux_l + gc * ux_c + gr * ux_r)) + (wl * ux_l + wc * ux_c + wr * ux_r);
    m[1] = ratio * (u2 - (gl * uxx_l + gc * uxx_c + gr * uxx_r)) +
           (wl * uxx_l + wc * uxx_c + wr * uxx_r);
    m[2] = ratio * u3;
    m[3] = ratio * u4;
}

/* O4 extension: reconstruct_patch_o3's pattern (active + ring) with WENO-AO(5,3) per axis;
 * modes [1+a] slope, [4+a] quadratic, [7+a] cubic, [10+a] quartic, [13] temporal. */
void or_reconstruct_patch_o4(const or_geom* g, double* modal, const or_limiter* cfg) {
    const int gh = g->ghost, M = 14;
    const ptrdiff_t st[3] = {(ptrdiff_t)NV * M, (ptrdiff_t)NV * M * gmx(g),
                             (ptrdiff_t)NV * M * gmx(g) * gmy(g)};
    for (int k = gh - 1; k < gh + g->nz + 1; ++k)
        for (int j = gh - 1; j < gh + g->ny + 1; ++j)
            for (int i = gh - 1; i < gh + g->nx + 1; ++i)
                for (int q = 0; q < NV; ++q) {
                    double* zc = modal + zoff(g, k, j, i) * NV * M + q * M;
                    double w[3][4];
                    for (int a = 0; a < 3; ++a) {
                        double s[5];
                        for (int m = -2; m <= 2; ++m) s[m + 2] = zc[m * st[a]];
                        or_weno_ao_point(s, cfg, w[a]);
                    }
                    for (int a = 0; a < 3; ++a)
                        for (int l = 0; l < 4; ++l) zc[1 + 3 * l + a] = w[a][l];
                }
}

/* ---------------------------------------------------------------- predictor.cpp */

/* predictor.cpp:12-22 flux_divergence */
static int flux_divergence(double face[6][NV], double idx, double idy, double idz, double gamma,
                           double* div) {
    double fe[5], fw[5], fn[5], fs[5], ft[5], fb[5];
    int rc;
    if ((rc = or_physical_flux(face[0], 0, gamma, fe))) return rc;
    if ((rc = or_physical_flux(face[1], 0, gamma, fw))) return rc;
    if ((rc = or_physical_flux(face[2], 1, gamma, fn))) return rc;
    if ((rc = or_physical_flux(face[3], 1, gamma, fs))) return rc;
    if ((rc = or_physical_flux(face[4], 2, gamma, ft))) return rc;
    if ((rc = or_physical_flux(face[5], 2, gamma, fb))) return rc;
    for (int q = 0; q < NV; ++q)
        div[q] = (fe[q] - fw[q]) * idx + (fn[q] - fs[q]) * idy + (ft[q] - fb[q]) * idz;
    return OR_OK;
}

/* predictor.cpp:26-60 predictor_ptwise (O3: one Picard pass) */
int or_predictor_ptwise(double* zv, int modes, double dt, double dx, double dy, double dz,
                        double gamma) {
    const int tm = modes - 1;
    const double idx = 1.0 / dx, idy = 1.0 / dy, idz = 1.0 / dz;
    double face[6][NV];
    for (int q = 0; q < NV; ++q) {
        const double* v = zv + q * modes;
        face[0][q] = extrap(v, modes, 0, +1.0);
        face[1][q] = extrap(v, modes, 0, -1.0);
        face[2][q] = extrap(v, modes, 1, +1.0);
        face[3][q] = extrap(v, modes, 1, -1.0);
        face[4][q] = extrap(v, modes, 2, +1.0);
        face[5][q] = extrap(v, modes, 2, -1.0);
    }
    double div[NV], tau[NV];
    int rc = flux_divergence(face, idx, idy, idz, gamma, div);
    if (rc) return rc;
    for (int q = 0; q < NV; ++q) tau[q] = -dt * div[q];
    if (modes >= 11) {
        for (int s = 0; s < 6; ++s)
            for (int q = 0; q < NV; ++q) face[s][q] += 0.5 * tau[q];
        if ((rc = flux_divergence(face, idx, idy, idz, gamma, div))) return rc;
        for (int q = 0; q < NV; ++q) tau[q] = -dt * div[q];
    }
    for (int q = 0; q < NV; ++q) zv[q * modes + tm] = tau[q];
    return OR_OK;
}

/* predictor.cpp:62-91 predict_patch (active + one ring; error text :82-84) */
int or_predict_patch(const or_geom* g, int modes, double* modal, double dt, double gamma) {
    const int gh = g->ghost, tm = modes - 1;
    for (int k = gh - 1; k < gh + g->nz + 1; ++k)
        for (int j = gh - 1; j < gh + g->ny + 1; ++j)
            for (int i = gh - 1; i < gh + g->nx + 1; ++i) {
                double zone[NV * 14];
                double* src = modal + zoff(g, k, j, i) * NV * modes;
                memcpy(zone, src, sizeof(double) * NV * modes);
                if (or_predictor_ptwise(zone, modes, dt, g->dx, g->dy, g->dz, gamma)) {
                    char pre[96];
                    snprintf(pre, sizeof pre, "predictor: zone (%d,%d,%d): ", i - gh, j - gh,
                             k - gh);
                    return prefix_error(pre);
                }
                for (int q = 0; q < NV; ++q) src[q * modes + tm] = zone[q * modes + tm];
            }
    return OR_OK;
}

/* predictor.cpp:93-102 zero_temporal_mode */
void or_zero_temporal_mode(const or_geom* g, int modes, double* modal) {
    size_t nz = (size_t)gmx(g) * gmy(g) * gmz(g);
    for (size_t z = 0; z < nz; ++z)
        for (int q = 0; q < NV; ++q) modal[(z * NV + q) * modes + modes - 1] = 0.0;
}

/* ---------------------------------------------------------------- corrector.cpp */

static void face_dims(const or_geom* g, int axis, int* n2, int* n1, int* n0) {
    if (axis == 0) { *n2 = g->nz; *n1 = g->ny; *n0 = g->nx + 1; }
    else if (axis == 1) { *n2 = g->nz; *n1 = g->nx; *n0 = g->ny + 1; }
    else { *n2 = g->ny; *n1 = g->nx; *n0 = g->nz + 1; }
}

/* corrector.cpp:15-59 flux_sweep<A> / serial_ref.cpp:99-126 (error text :53-55) */
int or_make_flux_axis(const or_geom* g, int modes, const double* modal, int axis, double gamma,
                      int solver, double* out) {
    const int gh = g->ghost, tm = modes - 1;
    int n2, n1, nf;
    face_dims(g, axis, &n2, &n1, &nf);
    for (int c2 = 0; c2 < n2; ++c2)
        for (int c1 = 0; c1 < n1; ++c1)
            for (int f = 0; f < nf; ++f) {
                size_t zl, zr;
                if (axis == 0) {
                    zl = zoff(g, gh + c2, gh + c1, gh + f - 1);
                    zr = zoff(g, gh + c2, gh + c1, gh + f);
                } else if (axis == 1) {
                    zl = zoff(g, gh + c2, gh + f - 1, gh + c1);
                    zr = zoff(g, gh + c2, gh + f, gh + c1);
                } else {
                    zl = zoff(g, gh + f - 1, gh + c2, gh + c1);
                    zr = zoff(g, gh + f, gh + c2, gh + c1);
                }
                double ul[NV], ur[NV];
                for (int q = 0; q < NV; ++q) {
                    const double* lv = modal + zl * NV * modes + q * modes;
                    const double* rv = modal + zr * NV * modes + q * modes;
                    ul[q] = extrap(lv, modes, axis, +1.0) + 0.5 * lv[tm];
                    ur[q] = extrap(rv, modes, axis, -1.0) + 0.5 * rv[tm];
                }
                double* dst = out + (((size_t)c2 * n1 + c1) * nf + f) * NV;
                if (riemann(solver, ul, ur, axis, gamma, dst)) {
                    char pre[96];
                    snprintf(pre, sizeof pre, "flux axis %d: face (%d,%d,%d): ", axis, f, c1, c2);
                    return prefix_error(pre);
                }
            }
    return OR_OK;
}

/* corrector.cpp:72-92 make_du_dt */
void or_make_du_dt(const or_geom* g, const double* fx, const double* fy, const double* fz,
                   double dt, double* rate) {
    const int nx = g->nx, ny = g->ny, nz = g->nz;
    const double cx = dt / g->dx, cy = dt / g->dy, cz = dt / g->dz;
#define FX(k, j, f) (fx + (((size_t)(k) * ny + (j)) * (nx + 1) + (f)) * NV)
#define FY(k, i, f) (fy + (((size_t)(k) * nx + (i)) * (ny + 1) + (f)) * NV)
#define FZ(j, i, f) (fz + (((size_t)(j) * nx + (i)) * (nz + 1) + (f)) * NV)
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const double *fxw = FX(k, j, i), *fxe = FX(k, j, i + 1);
                const double *fys = FY(k, i, j), *fyn = FY(k, i, j + 1);
                const double *fzb = FZ(j, i, k), *fzt = FZ(j, i, k + 1);
                double* r = rate + (((size_t)k * ny + j) * nx + i) * NV;
                for (int q = 0; q < NV; ++q)
                    r[q] = -cx * (fxe[q] - fxw[q]) - cy * (fyn[q] - fys[q]) -
                           cz * (fzt[q] - fzb[q]);
            }
#undef FX
#undef FY
#undef FZ
}

/* corrector.cpp:94-125 update_u_timestep (seed 1.0e32, error text :119-120) */
int or_update_u_timestep(const or_geom* g, int modes, double* modal, double* skinny,
                         const double* rate, double cfl, double gamma, double* dt_next) {
    const int gh = g->ghost;
    double dtn = 1.0e32;
    for (int k = 0; k < g->nz; ++k)
        for (int j = 0; j < g->ny; ++j)
            for (int i = 0; i < g->nx; ++i) {
                size_t z = zoff(g, gh + k, gh + j, gh + i);
                double* zp = modal + z * NV * modes;
                double* sp = skinny + z * NV;
                const double* r = rate + (((size_t)k * g->ny + j) * g->nx + i) * NV;
                double u[NV];
                for (int q = 0; q < NV; ++q) {
                    zp[q * modes] += r[q];
                    sp[q] = zp[q * modes];
                    u[q] = zp[q * modes];
                }
                double dt1;
                if (or_eval_tstep_ptwise(u, cfl, g->dx, g->dy, g->dz, gamma, &dt1)) {
                    char pre[96];
                    snprintf(pre, sizeof pre, "update: zone (%d,%d,%d): ", i, j, k);
                    return prefix_error(pre);
                }
                dtn = smin(dtn, dt1);
            }
    *dt_next = dtn;
    return OR_OK;
}

/* stepper.cpp:24-47 compute_dt_next (error text :41-42) */
int or_compute_dt_next(const or_geom* g, int modes, const double* modal, double gamma,
                       double cfl, double* dt_next) {
    const int gh = g->ghost;
    double dtn = 1.0e32;
    for (int k = 0; k < g->nz; ++k)
        for (int j = 0; j < g->ny; ++j)
            for (int i = 0; i < g->nx; ++i) {
                const double* zp = modal + zoff(g, gh + k, gh + j, gh + i) * NV * modes;
                double u[NV], dt1;
                for (int q = 0; q < NV; ++q) u[q] = zp[q * modes];
                if (or_eval_tstep_ptwise(u, cfl, g->dx, g->dy, g->dz, gamma, &dt1)) {
                    char pre[96];
                    snprintf(pre, sizeof pre, "dt estimate: zone (%d,%d,%d): ", i, j, k);
                    return prefix_error(pre);
                }
                dtn = smin(dtn, dt1);
            }
    *dt_next = dtn;
    return OR_OK;
}

/* ------------------------------------------------------------------ stepper.cpp */

static void reconstruct(const or_geom* g, const or_params* par, double* modal) {
    if (par->order == 2) or_limit_patch_o2(g, modal, &par->lim);
    else if (par->order == 3) or_reconstruct_patch_o3(g, modal, &par->lim);
    else or_reconstruct_patch_o4(g, modal, &par->lim);
}

static int three_sweeps(const or_geom* g, const or_params* par, int modes, const double* modal,
                        double* fx, double* fy, double* fz) {
    int rc;
    if ((rc = or_make_flux_axis(g, modes, modal, 0, par->gamma, par->solver, fx))) return rc;
    if ((rc = or_make_flux_axis(g, modes, modal, 1, par->gamma, par->solver, fy))) return rc;
    return or_make_flux_axis(g, modes, modal, 2, par->gamma, par->solver, fz);
}

/* stepper.cpp:49-78 ader_step */
int or_ader_step(const or_geom* g, const or_params* par, double* modal, double* skinny,
                 double* fx, double* fy, double* fz, double* rate, double dt, double cfl,
                 double* dt_next) {
    const int modes = modes_of(par->order);
    int rc;
    or_skinny_to_modal(g, modes, skinny, modal);
    reconstruct(g, par, modal);
    if ((rc = or_predict_patch(g, modes, modal, dt, par->gamma))) return rc;
    if ((rc = three_sweeps(g, par, modes, modal, fx, fy, fz))) return rc;
    or_make_du_dt(g, fx, fy, fz, dt, rate);
    return or_update_u_timestep(g, modes, modal, skinny, rate, cfl, par->gamma, dt_next);
}

/* stepper.cpp:88-98 rk_save_u0 */
void or_rk_save_u0(const or_geom* g, const double* skinny, double* u0) {
    const int gh = g->ghost;
    for (int k = gh; k < gh + g->nz; ++k)
        for (int j = gh; j < gh + g->ny; ++j)
            for (int i = gh; i < gh + g->nx; ++i)
                for (int q = 0; q < NV; ++q)
                    u0[zoff(g, k, j, i) * NV + q] = skinny[zoff(g, k, j, i) * NV + q];
}

/* stepper.cpp:100-143 rk_stage */
int or_rk_stage(const or_geom* g, const or_params* par, double* modal, double* skinny,
                double* fx, double* fy, double* fz, double* rate, const double* u0, double dt,
                double a, double b) {
    const int modes = modes_of(par->order);
    const int gh = g->ghost;
    int rc;
    or_skinny_to_modal(g, modes, skinny, modal);
    reconstruct(g, par, modal);
    or_zero_temporal_mode(g, modes, modal);
    if ((rc = three_sweeps(g, par, modes, modal, fx, fy, fz))) return rc;
    or_make_du_dt(g, fx, fy, fz, dt, rate);
    for (int k = 0; k < g->nz; ++k)
        for (int j = 0; j < g->ny; ++j)
            for (int i = 0; i < g->nx; ++i) {
                size_t z = zoff(g, gh + k, gh + j, gh + i);
                double* zp = modal + z * NV * modes;
                const double* r = rate + (((size_t)k * g->ny + j) * g->nx + i) * NV;
                for (int q = 0; q < NV; ++q) {
                    double unew = a * u0[z * NV + q] + b * (zp[q * modes] + r[q]);
                    zp[q * modes] = unew;
                    skinny[z * NV + q] = unew;
                }
            }
    return OR_OK;
}

/* stepper.cpp:80-86 rk_stages and :145-157 rk_step */
int or_rk_step(const or_geom* g, const or_params* par, int nstages, double* modal,
               double* skinny, double* fx, double* fy, double* fz, double* rate,
               double* stage_u0, int bc, double dt, double cfl, double* dt_next) {
    static const double heun[2][2] = {{0.0, 1.0}, {0.5, 0.5}};
    static const double ssp3[3][2] = {{0.0, 1.0}, {0.75, 0.25}, {1.0 / 3.0, 2.0 / 3.0}};
    if (nstages != 2 && nstages != 3) {
        snprintf(g_err, sizeof g_err, "rk_stages called for a non-RK integrator");
        return OR_INVALID;
    }
    const int modes = modes_of(par->order);
    int rc;
    or_rk_save_u0(g, skinny, stage_u0);
    for (int s = 0; s < nstages; ++s) {
        const double* ab = nstages == 2 ? heun[s] : ssp3[s];
        or_apply_boundary_skinny(g, bc, skinny);
        if ((rc = or_rk_stage(g, par, modal, skinny, fx, fy, fz, rate, stage_u0, dt, ab[0],
                              ab[1])))
            return rc;
    }
    return or_compute_dt_next(g, modes, modal, par->gamma, cfl, dt_next);
}

/* ----------------------------------------------------------------- problems.cpp */

static const double OR_PI = 3.14159265358979323846;

/* problems.cpp:11-38 vortex_prim (eps 5, free stream (1,1,1,0,1)) */
static void vortex_prim(const or_geom* g, double gamma, double x, double y, double t,
                        double* q) {
    const double eps = 5.0, rho_inf = 1.0, u_inf = 1.0, v_inf = 1.0, w_inf = 0.0, p_inf = 1.0;
    const double Lx = g->nx * g->dx, Ly = g->ny * g->dy;
    const double cx = g->origin[0] + 0.5 * Lx, cy = g->origin[1] + 0.5 * Ly;
    double xr = remainder(x - u_inf * t - cx, Lx);
    double yr = remainder(y - v_inf * t - cy, Ly);
    double r2 = xr * xr + yr * yr;
    double swirl = eps / (2.0 * OR_PI) * exp(0.5 * (1.0 - r2));
    double gm1 = gamma - 1.0;
    double dT = -gm1 * eps * eps / (8.0 * gamma * OR_PI * OR_PI) * exp(1.0 - r2);
    double T_inf = p_inf / rho_inf;
    double entropy = p_inf / pow(rho_inf, gamma);
    double T = T_inf + dT;
    q[0] = pow(T / entropy, 1.0 / gm1);
    q[1] = u_inf - yr * swirl;
    q[2] = v_inf + xr * swirl;
    q[3] = w_inf;
    q[4] = q[0] * T;
}

/* euler.hpp:52-60 prim_to_cons */
static void prim_to_cons(const double* q, double gamma, double* c) {
    c[0] = q[0];
    c[1] = q[0] * q[1];
    c[2] = q[0] * q[2];
    c[3] = q[0] * q[3];
    c[4] = q[4] / (gamma - 1.0) + 0.5 * q[0] * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
}

typedef void (*prim_fn)(const or_geom*, double, double, double, double, const void*, double*);

/* problems.cpp:44-76 sample_profile: midpoint at O2, 2^3 Gauss at O3, over all zones */
static void sample_profile(const or_geom* g, double gamma, int order, prim_fn fn,
                           const void* ctx, double* s) {
    const int gh = g->ghost;
    const double goff = 0.5 / sqrt(3.0);
    for (int k = 0; k < gmz(g); ++k)
        for (int j = 0; j < gmy(g); ++j)
            for (int i = 0; i < gmx(g); ++i) {
                double xc = g->origin[0] + ((i - gh) + 0.5) * g->dx;
                double yc = g->origin[1] + ((j - gh) + 0.5) * g->dy;
                double zc = g->origin[2] + ((k - gh) + 0.5) * g->dz;
                double u[NV] = {0, 0, 0, 0, 0};
                if (order == 2) {
                    double q[5];
                    fn(g, gamma, xc, yc, zc, ctx, q);
                    prim_to_cons(q, gamma, u);
                } else {
                    for (int a = -1; a <= 1; a += 2)
                        for (int b = -1; b <= 1; b += 2)
                            for (int c3 = -1; c3 <= 1; c3 += 2) {
                                double q[5], w[5];
                                fn(g, gamma, xc + a * goff * g->dx, yc + b * goff * g->dy,
                                   zc + c3 * goff * g->dz, ctx, q);
                                prim_to_cons(q, gamma, w);
                                for (int qq = 0; qq < NV; ++qq) u[qq] += 0.125 * w[qq];
                            }
                }
                double* dst = s + zoff(g, k, j, i) * NV;
                for (int q = 0; q < NV; ++q) dst[q] = u[q];
            }
}

static void vortex_fn(const or_geom* g, double gamma, double x, double y, double z,
                      const void* ctx, double* q) {
    (void)z;
    vortex_prim(g, gamma, x, y, *(const double*)ctx, q);
}
static void sod_fn(const or_geom* g, double gamma, double x, double y, double z,
                   const void* ctx, double* q) {
    (void)g; (void)gamma; (void)y; (void)z; (void)ctx;
    if (x < 0.5) { q[0] = 1.0; q[1] = q[2] = q[3] = 0.0; q[4] = 1.0; }
    else { q[0] = 0.125; q[1] = q[2] = q[3] = 0.0; q[4] = 0.1; }
}
static void const_fn(const or_geom* g, double gamma, double x, double y, double z,
                     const void* ctx, double* q) {
    (void)g; (void)gamma; (void)x; (void)y; (void)z; (void)ctx;
    q[0] = 1.0; q[1] = 1.0; q[2] = 1.0; q[3] = 0.0; q[4] = 1.0;
}

/* problems.cpp:80-92 init_isentropic_vortex (t = 0) / exact_vortex (t > 0) */
void or_init_isentropic_vortex(const or_geom* g, double gamma, int order, double t,
                               double* skinny) {
    sample_profile(g, gamma, order, vortex_fn, &t, skinny);
}
/* problems.cpp:106-111 */
void or_init_sod(const or_geom* g, double gamma, double* skinny) {
    sample_profile(g, gamma, 2, sod_fn, NULL, skinny);
}
/* problems.cpp:100-104 */
void or_init_constant(const or_geom* g, double gamma, double* skinny) {
    sample_profile(g, gamma, 2, const_fn, NULL, skinny);
}

/* harness.cpp:92-103 initial_dt */
double or_initial_dt(const or_geom* g, const double* s, double gamma, double cfl) {
    const int gh = g->ghost;
    double dt = 1.0e32;
    for (int k = gh; k < gh + g->nz; ++k)
        for (int j = gh; j < gh + g->ny; ++j)
            for (int i = gh; i < gh + g->nx; ++i) {
                double d = 0.0;
                or_eval_tstep_ptwise(s + zoff(g, k, j, i) * NV, cfl, g->dx, g->dy, g->dz, gamma,
                                     &d);
                dt = smin(dt, d);
            }
    return dt;
}

/* harness.cpp:150-170 time loop with a fixed step count over one patch; exchange_ghosts
 * on a 1x1x1 PatchSet is apply_boundary (test_transfer.cpp:46-68). ADER only. */
int or_run_steps(const or_geom* g, const or_params* par, int bc, double cfl, int steps,
                 double* skinny, double* dts) {
    const int modes = modes_of(par->order);
    size_t tot = (size_t)gmx(g) * gmy(g) * gmz(g);
    double* modal = calloc(tot * NV * modes, sizeof(double));
    double* fx = calloc((size_t)g->nz * g->ny * (g->nx + 1) * NV, sizeof(double));
    double* fy = calloc((size_t)g->nz * g->nx * (g->ny + 1) * NV, sizeof(double));
    double* fz = calloc((size_t)g->ny * g->nx * (g->nz + 1) * NV, sizeof(double));
    double* rate = calloc((size_t)g->nz * g->ny * g->nx * NV, sizeof(double));
    int rc = OR_OK;
    double dt = dts[0];
    for (int s = 0; s < steps && rc == OR_OK; ++s) {
        double dtn = 0.0;
        or_apply_boundary_skinny(g, bc, skinny);
        rc = or_ader_step(g, par, modal, skinny, fx, fy, fz, rate, dt, cfl, &dtn);
        dt = dtn;
        dts[s + 1] = dt;
    }
    free(modal);
    free(fx);
    free(fy);
    free(fz);
    free(rate);
    return rc;
}
