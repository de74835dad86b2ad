// problems_host.cpp -- host-side initial conditions for the product path (problems.cpp in
// the reference, out of the hot path by design: the paper computes ICs on the host and the
// reference samples them with libm exp/pow/remainder, so they are kept on the host to give
// bit-identical inputs). Compiled by g++ with -ffp-contract=off like the reference.
#include <cmath>
#include <cstddef>

#include "../../include/hydro_cuda.h"

namespace {

constexpr double PI = 3.14159265358979323846;

inline size_t zoff(const hc_geom& g, int k, int j, int i) {
    const int mx = g.nx + 2 * g.ghost, my = g.ny + 2 * g.ghost;
    return (size_t(k) * my + j) * mx + i;
}

// problems.cpp:11-38 vortex_prim (eps = 5, free stream (1, 1, 1, 0, 1))
void vortex_prim(const hc_geom& g, double gamma, double x, double y, double t, double* q) {
    const double eps = 5.0, rho_inf = 1.0, u_inf = 1.0, v_inf = 1.0, w_inf = 0.0, p_inf = 1.0;
    const double Lx = g.nx * g.dx, Ly = g.ny * g.dy;
    const double cx = g.origin[0] + 0.5 * Lx, cy = g.origin[1] + 0.5 * Ly;
    double xr = std::remainder(x - u_inf * t - cx, Lx);
    double yr = std::remainder(y - v_inf * t - cy, Ly);
    double r2 = xr * xr + yr * yr;
    double swirl = eps / (2.0 * PI) * std::exp(0.5 * (1.0 - r2));
    double gm1 = gamma - 1.0;
    double dT = -gm1 * eps * eps / (8.0 * gamma * PI * PI) * std::exp(1.0 - r2);
    double T_inf = p_inf / rho_inf;
    double entropy = p_inf / std::pow(rho_inf, gamma);
    double T = T_inf + dT;
    q[0] = std::pow(T / entropy, 1.0 / gm1);
    q[1] = u_inf - yr * swirl;
    q[2] = v_inf + xr * swirl;
    q[3] = w_inf;
    q[4] = q[0] * T;
}

// euler.hpp:52-60 prim_to_cons
void prim_to_cons(const double* q, double gamma, double* c) {
    c[0] = q[0];
    c[1] = q[0] * q[1];
    c[2] = q[0] * q[2];
    c[3] = q[0] * q[3];
    c[4] = q[4] / (gamma - 1.0) + 0.5 * q[0] * (q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
}

// problems.cpp:44-76 sample_profile: midpoint (order 2) or 2^3 Gauss (order 3), all zones
template <typename Fn>
void sample(const hc_geom& g, double gamma, int order, Fn prim, double* s) {
    const int gh = g.ghost;
    const int mx = g.nx + 2 * gh, my = g.ny + 2 * gh, mz = g.nz + 2 * gh;
    const double goff = 0.5 / std::sqrt(3.0);
#pragma omp parallel for collapse(2)
    for (int k = 0; k < mz; ++k)
        for (int j = 0; j < my; ++j)
            for (int i = 0; i < mx; ++i) {
                double xc = g.origin[0] + ((i - gh) + 0.5) * g.dx;
                double yc = g.origin[1] + ((j - gh) + 0.5) * g.dy;
                double zc = g.origin[2] + ((k - gh) + 0.5) * g.dz;
                double u[5] = {0, 0, 0, 0, 0};
                if (order == 2) {
                    double q[5];
                    prim(xc, yc, zc, q);
                    prim_to_cons(q, gamma, u);
                } else {
                    for (int a = -1; a <= 1; a += 2)
                        for (int b = -1; b <= 1; b += 2)
                            for (int c3 = -1; c3 <= 1; c3 += 2) {
                                double q[5], w[5];
                                prim(xc + a * goff * g.dx, yc + b * goff * g.dy,
                                     zc + c3 * goff * g.dz, q);
                                prim_to_cons(q, gamma, w);
                                for (int qq = 0; qq < 5; ++qq) u[qq] += 0.125 * w[qq];
                            }
                }
                double* dst = s + zoff(g, k, j, i) * 5;
                for (int q = 0; q < 5; ++q) dst[q] = u[q];
            }
}

}  // namespace

extern "C" {

// problems.cpp:80-92 init_isentropic_vortex (t = 0) and exact_vortex (t > 0)
int hc_init_vortex(const hc_geom* g, double gamma, int order, double t, double* skinny) {
    sample(*g, gamma, order,
           [&](double x, double y, double, double* q) { vortex_prim(*g, gamma, x, y, t, q); },
           skinny);
    return HC_OK;
}

// problems.cpp:106-111 init_sod
int hc_init_sod(const hc_geom* g, double gamma, double* skinny) {
    sample(*g, gamma, 2,
           [](double x, double, double, double* q) {
               if (x < 0.5) { q[0] = 1.0; q[1] = q[2] = q[3] = 0.0; q[4] = 1.0; }
               else { q[0] = 0.125; q[1] = q[2] = q[3] = 0.0; q[4] = 0.1; }
           },
           skinny);
    return HC_OK;
}

// problems.cpp:100-104 init_constant (free stream)
int hc_init_constant(const hc_geom* g, double gamma, double* skinny) {
    sample(*g, gamma, 2,
           [](double, double, double, double* q) {
               q[0] = 1.0; q[1] = 1.0; q[2] = 1.0; q[3] = 0.0; q[4] = 1.0;
           },
           skinny);
    return HC_OK;
}

}  // extern "C"
