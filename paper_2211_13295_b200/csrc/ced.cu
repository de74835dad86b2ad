// ced.cu -- computational electrodynamics in a conducting medium on the ADER path, B200
// (sm_100a), FP64 (include/hydro_ced.h). EXTENSION: the reference scopes out CED and
// stiff-source ADER; the north star names both (BASELINE.json config 4).
//
// All six unknowns are face-centred (D and B normal components), so every update is a
// constrained-transport curl of edge values; there are no face Riemann fluxes. Per step:
//   k_ced_ghosts        periodic / outflow gather of the six face fields
//   k_ced_cell<O3>      cell averages of D, B from the faces (ct::face_avg)
//   k_ced_predict<O3>   ring zones: MC / WENO3 (+ cross terms) of the 6 cell variables, ADER
//                       predictor with the Maxwell flux and the conduction source solved
//                       over the half step by the exponential update (one Picard pass at O3)
//   k_ced_edge<O3, C>   E_C and H_C on the C edges from the four corner states: the 2D upwind
//                       solver (HLL with speeds +-c is exact for linear Maxwell), its
//                       dissipation scaled by theta = 1/(1 + sigma h/(2 c eps)) so the
//                       magnetic-diffusion limit is preserved in good conductors:
//                         E_C = mean corner E_C + c/2 (B_b[a+] - B_b[a-]) - c/2 (B_a[b+] - B_a[b-])
//                         H_C = mean corner H_C - c/2 (D_b[a+] - D_b[a-]) + c/2 (D_a[b+] - D_a[b-])
//                       (a = C+1, b = C+2; [a+] = mean of the two corners on the high-a side)
//   k_ced_update        B -= dt curl_h E;  D = exp(-s dt) D + phi(s dt) dt curl_h H,
//                       s = sigma_face / eps, phi(z) = (1 - e^-z)/z (L-stable, exact for
//                       frozen curl H: no time-step restriction from sigma)
//   k_ced_advance       t/dt hand-off with the t_final clip (harness.cpp:155-170)
#include <cuda_runtime.h>

#include <cmath>
#include <new>
#include <string>

#include "../../include/hydro_ced.h"
#include "common.cuh"
#include "ct_common.cuh"
#include "fused_types.cuh"
#include "graph_step.cuh"

namespace hc {
namespace ced {

using ct::at;
using ct::blocks;
using ct::Box;
using ct::map_c;
using ct::stride;

constexpr int NF = 6;  // Dx, Dy, Dz, Bx, By, Bz

struct CArgs {
    double* s;      // [6][N] face fields
    double* sigma;  // [N] zone conductivity
    double* w;      // [6][N] cell averages of the face fields
    double* states; // [12][6][N] edge-midpoint states (spatial part), s = 4C + 2 lb + la
    double* ht;     // [6][N] tau/2 of every ring zone (half-time state = states + ht)
    double* emf;    // [3][N] E on the edges (same indexing as mhd.cu)
    double* hmf;    // [3][N] H on the edges
    Box b;
    double d[3], id[3];
    double eps, mu, c;
    Limiter lim;
    int bc[3];
    StepCtl* ctl;
};

// exp(-z) and phi(z) = (1 - exp(-z)) / z for z = s dt >= 0 (phi(0) = 1)
__device__ __forceinline__ void decay(double z, double& ex, double& ph) {
    ex = exp(-z);
    ph = z > 0.0 ? -expm1(-z) / z : 1.0;
}

// Maxwell flux along A of the state u = (D, B): F(D) = (0, H_{A+2}, -H_{A+1}),
// F(B) = (0, -E_{A+2}, E_{A+1}) on the cyclic components (A, A+1, A+2)
template <int A>
__device__ __forceinline__ void maxwell_flux(const double* u, double ie, double im, double* f) {
    constexpr int A1 = (A + 1) % 3, A2 = (A + 2) % 3;
    f[A] = 0.0;
    f[A1] = u[3 + A2] * im;
    f[A2] = -(u[3 + A1] * im);
    f[3 + A] = 0.0;
    f[3 + A1] = -(u[A2] * ie);
    f[3 + A2] = u[A1] * ie;
}

__global__ void k_ced_ghosts(CArgs a, int with_sigma) {
    if (a.ctl && a.ctl->done) return;
    const Box& b = a.b;
    int c[3];  // the ghost shell only
    if (!shell_zone(b, blockIdx.x * size_t(blockDim.x) + threadIdx.x, c[0], c[1], c[2])) return;
    const size_t r = at(b, c[2], c[1], c[0]);
#pragma unroll 1
    for (int q = 0; q < NF + with_sigma; ++q) {
        int src[3];
        bool ghost = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            int hi = b.gh + b.n[d];
            if (q < NF && q % 3 == d && a.bc[d] == HC_OUTFLOW) hi += 1;
            src[d] = map_c(c[d], b.gh, hi, a.bc[d]);
            ghost |= src[d] != c[d];
        }
        if (!ghost) continue;
        double* v = q < NF ? a.s + size_t(q) * b.N : a.sigma;
        v[r] = v[at(b, src[2], src[1], src[0])];
    }
}

template <bool O3>
__global__ void k_ced_cell(CArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= b.N) return;
    const int i = int(r % b.P), j = int((r / b.P) % b.Q), k = int(r / (size_t(b.P) * b.Q));
    const int lo = O3 ? 1 : 0, hi = O3 ? 2 : 1;
    if (i < lo || j < lo || k < lo || i + hi >= b.P || j + hi >= b.Q || k + hi >= b.R) return;
#pragma unroll
    for (int q = 0; q < NF; ++q)
        a.w[size_t(q) * b.N + r] = ct::face_avg<O3>(a.s + size_t(q) * b.N, r, stride(b, q % 3));
}

// One ring zone: reconstruction of the 6 cell variables, its 12 edge-midpoint states,
// ADER predictor, tau/2. The six face states live in shared memory ([s][q][thread]) so the
// variable loop need not be unrolled; FAST = 1 runs the branch-free bit-exact division of
// pointwise.cuh and the caller re-runs the zone with FAST = 0 when a flag is raised.
template <bool O3, int FAST>
__device__ __forceinline__ void ced_zone(const CArgs& a, size_t o, double* fs, Fault& wf) {
    const Box& b = a.b;
    const size_t st[3] = {stride(b, 0), stride(b, 1), stride(b, 2)};
    const double dt = a.ctl->dt;
    const size_t N = b.N;
    auto face = [&](int f, int q) -> double& { return fs[(f * NF + q) * 128]; };
#pragma unroll 1
    for (int q = 0; q < NF; ++q) {
        const double* __restrict__ w = a.w + size_t(q) * N;
        const double c0 = w[o];
        double lin[3], quad[3] = {0.0, 0.0, 0.0}, cross[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double up = w[o + st[d]], um = w[o - st[d]];
            if (!O3) lin[d] = mc_limiter(up - c0, c0 - um, a.lim.cfac_other);
            else  // doubled slopes (weno3_2x, bit-exact): consumers halve their weights
                weno3_2x<FAST>(w[o - 2 * st[d]], um, c0, up, w[o + 2 * st[d]], a.lim, lin[d], quad[d], wf);
            face(2 * d, q) = O3 ? extrap2<true>(c0, +1.0, lin[d], quad[d])
                                : extrap<false>(c0, +1.0, lin[d], quad[d]);
            face(2 * d + 1, q) = O3 ? extrap2<true>(c0, -1.0, lin[d], quad[d])
                                    : extrap<false>(c0, -1.0, lin[d], quad[d]);
            if (O3) {
                const size_t sa = st[d], sb = st[(d + 1) % 3];
                cross[d] =
                    0.25 * ((w[o + sa + sb] - w[o + sa - sb]) - (w[o - sa + sb] - w[o - sa - sb]));
            }
        }
        // the 12 edge-midpoint states the edge solver reads (mhd.cu's convention: the corner
        // (xa, xb) = (la ? -1/2 : +1/2, lb ? -1/2 : +1/2) in the (C+1, C+2) plane)
#pragma unroll
        for (int C = 0; C < 3; ++C) {
            const int AA = (C + 1) % 3, BB = (C + 2) % 3;
#pragma unroll
            for (int lb = 0; lb < 2; ++lb)
#pragma unroll
                for (int la = 0; la < 2; ++la) {
                    const double xa = la == 0 ? 0.5 : -0.5, xb = lb == 0 ? 0.5 : -0.5;
                    const double hl = O3 ? 0.5 : 1.0;  // O3 slopes are doubled (exact halving)
                    double v = c0 + (hl * xa) * lin[AA] + (hl * xb) * lin[BB];
                    if (O3)
                        v = v + (1.0 / 12.0) * quad[AA] + (1.0 / 12.0) * quad[BB] +
                            (xa * xb) * cross[AA];
                    __stcs(a.states + (size_t(4 * C + 2 * lb + la) * NF + q) * N + o, v);
                }
        }
    }
    // predictor: C = -div F of the face states; B: tau = dt C; D: the conduction source over
    // the half step, D_h = e^{-s dt/2} D0 + phi(s dt/2) (dt/2) C_D, tau = 2 (D_h - D0)
    const double ie = 1.0 / a.eps, im = 1.0 / a.mu;
    double ex, ph;
    decay(a.sigma[o] * ie * (0.5 * dt), ex, ph);
    double tau[NF] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int pass = 0; pass < (O3 ? 2 : 1); ++pass) {
        double div[NF];
#pragma unroll
        for (int A = 0; A < 3; ++A) {
            double ua[NF], ub[NF], fa[NF], fb[NF];
#pragma unroll
            for (int q = 0; q < NF; ++q) {
                ua[q] = pass ? face(2 * A, q) + 0.5 * tau[q] : face(2 * A, q);
                ub[q] = pass ? face(2 * A + 1, q) + 0.5 * tau[q] : face(2 * A + 1, q);
            }
            if (A == 0) { maxwell_flux<0>(ua, ie, im, fa); maxwell_flux<0>(ub, ie, im, fb); }
            if (A == 1) { maxwell_flux<1>(ua, ie, im, fa); maxwell_flux<1>(ub, ie, im, fb); }
            if (A == 2) { maxwell_flux<2>(ua, ie, im, fa); maxwell_flux<2>(ub, ie, im, fb); }
#pragma unroll
            for (int q = 0; q < NF; ++q)
                div[q] = A == 0 ? (fa[q] - fb[q]) * a.id[0] : div[q] + (fa[q] - fb[q]) * a.id[A];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const double u0 = a.w[size_t(q) * N + o];
            const double dh = ex * u0 + ph * (0.5 * dt) * (-div[q]);
            tau[q] = 2.0 * (dh - u0);
        }
#pragma unroll
        for (int q = 3; q < NF; ++q) tau[q] = -dt * div[q];
    }
#pragma unroll
    for (int q = 0; q < NF; ++q) __stcs(a.ht + size_t(q) * N + o, 0.5 * tau[q]);
}

template <bool O3>
__device__ __noinline__ void ced_zone_careful(const CArgs& a, size_t o, double* fs) {
    Fault f;
    f.clear();
    ced_zone<O3, 0>(a, o, fs, f);
}

template <bool O3>
__global__ void __launch_bounds__(128) k_ced_predict(CArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    const int rx = b.n[0] + 2, ry = b.n[1] + 2;
    const size_t cnt = size_t(rx) * ry * (b.n[2] + 2);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    const int i = int(r % rx) - 1 + b.gh, j = int((r / rx) % ry) - 1 + b.gh,
              k = int(r / (size_t(rx) * ry)) - 1 + b.gh;
    const size_t o = at(b, k, j, i);
    __shared__ double sface[6 * NF * 128];
    double* fs = sface + threadIdx.x;
    Fault wf;
    wf.clear();
    ced_zone<O3, 1>(a, o, fs, wf);
    if (wf.redo()) ced_zone_careful<O3>(a, o, fs);  // (WENO3 raises no physical faults)
}

template <bool O3, int C>
__global__ void __launch_bounds__(128) k_ced_edge(CArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    constexpr int AA = (C + 1) % 3, BB = (C + 2) % 3;
    const int ex = b.n[0] + (C != 0), ey = b.n[1] + (C != 1), ez = b.n[2] + (C != 2);
    const size_t cnt = size_t(ex) * ey * ez;
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    const int c0 = int(r % ex), c1 = int((r / ex) % ey), c2 = int(r / (size_t(ex) * ey));
    const size_t o = at(b, c2 + b.gh, c1 + b.gh, c0 + b.gh);
    const size_t sa = stride(b, AA), sb = stride(b, BB), N = b.N;
    // per corner (la, lb): the six fields at the corner
    double e = 0.0, h = 0.0, dbp = 0.0, dbm = 0.0, dap = 0.0, dam = 0.0;
    double bbp = 0.0, bbm = 0.0, bap = 0.0, bam = 0.0;
#pragma unroll
    for (int lb = 0; lb < 2; ++lb)
#pragma unroll
        for (int la = 0; la < 2; ++la) {
            const size_t z = o - (la == 0 ? sa : 0) - (lb == 0 ? sb : 0);
            double u[NF];
#pragma unroll
            for (int q = 0; q < NF; ++q)
                u[q] = __ldg(a.states + (size_t(4 * C + 2 * lb + la) * NF + q) * N + z) +
                       __ldg(a.ht + size_t(q) * N + z);
            e = e + u[C];      // D_C (-> E_C = D_C / eps)
            h = h + u[3 + C];  // B_C (-> H_C = B_C / mu)
            if (la) { dbp = dbp + u[BB]; bbp = bbp + u[3 + BB]; }
            else { dbm = dbm + u[BB]; bbm = bbm + u[3 + BB]; }
            if (lb) { dap = dap + u[AA]; bap = bap + u[3 + AA]; }
            else { dam = dam + u[AA]; bam = bam + u[3 + AA]; }
        }
    const double hc = 0.5 * a.c;
    // asymptotic-preserving scaling of the upwind dissipation (Jin-Levermore type): in a good
    // conductor (sigma h / (2 c eps) >> 1) the jumps' c/2 dissipation would swamp the
    // magnetic diffusivity 1/(mu sigma); theta = 1 / (1 + sigma_e h / (2 c eps)) per
    // direction, sigma_e = mean of the four zones; theta = 1 exactly where sigma_e = 0
    double sg = 0.0;
#pragma unroll
    for (int lb = 0; lb < 2; ++lb)
#pragma unroll
        for (int la = 0; la < 2; ++la) sg = sg + a.sigma[o - (la == 0 ? sa : 0) - (lb == 0 ? sb : 0)];
    sg = 0.25 * sg;
    const double ta = 1.0 / (1.0 + sg * a.d[AA] / (2.0 * a.c * a.eps));
    const double tb = 1.0 / (1.0 + sg * a.d[BB] / (2.0 * a.c * a.eps));
    // means of two corners: 0.5 * sum
    a.emf[size_t(C) * N + o] = 0.25 * e / a.eps + hc * ta * (0.5 * bbp - 0.5 * bbm) -
                               hc * tb * (0.5 * bap - 0.5 * bam);
    a.hmf[size_t(C) * N + o] = 0.25 * h / a.mu - hc * ta * (0.5 * dbp - 0.5 * dbm) +
                               hc * tb * (0.5 * dap - 0.5 * dam);
}

__global__ void k_ced_update(CArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    const int px = b.n[0] + 1, py = b.n[1] + 1;
    const size_t cnt = size_t(px) * py * (b.n[2] + 1);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    const int i = int(r % px), j = int((r / px) % py), k = int(r / (size_t(px) * py));
    const bool ci = i < b.n[0], cj = j < b.n[1], ck = k < b.n[2];
    const size_t o = at(b, k + b.gh, j + b.gh, i + b.gh);
    const size_t N = b.N, sx = 1, sy = b.P, sz = size_t(b.P) * b.Q;
    const double dt = a.ctl->dt;
    const double cx = dt / a.d[0], cy = dt / a.d[1], cz = dt / a.d[2];
    const double* ex = a.emf;
    const double* ey = a.emf + N;
    const double* ez = a.emf + 2 * N;
    const double* hx = a.hmf;
    const double* hy = a.hmf + N;
    const double* hz = a.hmf + 2 * N;
    double* s = a.s;
    const double ie = 1.0 / a.eps;
    auto dstep = [&](int q, size_t so, double curl) {
        double e_, p_;
        decay(0.5 * (a.sigma[o] + a.sigma[o - so]) * ie * dt, e_, p_);
        s[q * N + o] = e_ * s[q * N + o] + p_ * curl;
    };
    if (cj && ck) {
        s[3 * N + o] = s[3 * N + o] - (cy * (ez[o + sy] - ez[o]) - cz * (ey[o + sz] - ey[o]));
        dstep(0, sx, cy * (hz[o + sy] - hz[o]) - cz * (hy[o + sz] - hy[o]));
    }
    if (ci && ck) {
        s[4 * N + o] = s[4 * N + o] - (cz * (ex[o + sz] - ex[o]) - cx * (ez[o + 1] - ez[o]));
        dstep(1, sy, cz * (hx[o + sz] - hx[o]) - cx * (hz[o + 1] - hz[o]));
    }
    if (ci && cj) {
        s[5 * N + o] = s[5 * N + o] - (cx * (ey[o + 1] - ey[o]) - cy * (ex[o + sy] - ex[o]));
        dstep(2, sz, cx * (hy[o + 1] - hy[o]) - cy * (hx[o + sy] - hx[o]));
    }
}

// ============================================================ order 4 (space-time ADER)
// The O2/O3 kernels above keep the reference's ADER structure (face state + the zone's tau/2),
// second order in time. Order 4 is the scheme of the paper's CED runs: a
// local space-time predictor with the stiff conduction source solved IMPLICITLY inside it by
// small block inversions, then edge E and H integrated at space-time Gauss points:
//   k_ced4_predict  one CTA per ring zone, one thread per spatial node (4 x 4 x 4 Gauss-
//                   Legendre points) with its 4 Radau IIA times in [t, t + dt]: the degree-3 polynomial
//                   of the six cell fields (WENO-AO pure terms, central mixed terms, as
//                   ader4.cu), then Picard iterations of the collocation system
//                     q(tau_m) = P - dt sum_l A_ml (div F(q(tau_l)) + s q_D(tau_l)),  s = sigma/eps
//                   with the source implicit: per spatial node the 4 x 4 system
//                   (I + s dt A) q_D = P - dt A div F_D, inverted once per zone; Radau IIA is
//                   L-stable, so sigma dt >> 1 relaxes D instead of ringing
//   outputs         the fields at the 2 Gauss points along each of the 12 zone edges at the 2
//                   Gauss times ([48][6][N] in `states`)
//   k_ced4_edge<C>  E_C and H_C from the four corner states at each of the 2 x 2 space-time
//                   Gauss points (the O3 upwind formula and its asymptotic-preserving scaling),
//                   averaged: the edge- and time-averaged EMFs
//   k_ced4_update   B -= dt curl E (CT); D: the exponential conduction step of the O3 path
//                   (exact for frozen curl H, L-stable) with the space-time averaged curl H
struct CedBasis {
    double xi[4], D[4][4];   // Gauss-Legendre nodes on [-1/2, 1/2] and d/dxi of their Lagrange basis
    double A[4][4];          // Radau IIA: int_0^{c_m} L_l(s) ds, c on [0, 1]
    double LF[2][4];         // L_l(+1/2), L_l(-1/2)
    double LG[2][4];         // L_l(-+1/(2 sqrt 3))
    double LT[2][4];         // Radau time basis at the Gauss times 1/2 -+ 1/(2 sqrt 3)
};
__constant__ CedBasis c_cb;
constexpr int C4_NT = 256, C4_EDGE = 48, C4_NCOEF = 23;

__device__ __forceinline__ void psi4(double s, double* p) {
    const double s2 = s * s;
    p[0] = s;
    p[1] = s2 - 1.0 / 12.0;
    p[2] = s * (s2 - 3.0 / 20.0);
    p[3] = s2 * s2 - (3.0 / 14.0) * s2 + 3.0 / 560.0;
}

// One CTA of 64 threads per ring zone; thread t owns spatial node t and its 4 Radau times in
// registers, so the implicit conduction solve over those times (minv) and the time integral
// are register work; the fluxes go through shared memory two time nodes at a time, SoA with
// the node slot n ^ 5 * bit4(n) (conflict-free neighbour reads, as ader4.cu); the 48 edge
// points are contracted separably (the edge axis first, then the two transverse ones).
#ifndef C4_MINB
#define C4_MINB 6
#endif
constexpr int C4_NS = 64;
constexpr int C4_F = 2 * 3 * NF * C4_NS;
constexpr int C4_T = NF * 2 * C4_NS;
constexpr int C4_SQ = 192 + 12;
constexpr int C4_U = (C4_F > C4_T + NF * C4_SQ) ? C4_F : C4_T + NF * C4_SQ;
__global__ void __launch_bounds__(C4_NS, C4_MINB) k_ced4_predict(CArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    __shared__ double coef[NF][C4_NCOEF];
    __shared__ double minv[4][4];
    __shared__ double U[C4_U];
    const int rx = b.n[0] + 2, ry = b.n[1] + 2;
    const int zr = blockIdx.x;
    const int i = zr % rx - 1 + b.gh, j = (zr / rx) % ry - 1 + b.gh, k = zr / (rx * ry) - 1 + b.gh;
    const size_t o = at(b, k, j, i);
    const size_t st3[3] = {stride(b, 0), stride(b, 1), stride(b, 2)};
    const size_t N = b.N;
    const int t = threadIdx.x;
    const double dt = a.ctl->dt;
    auto W = [&](int q, long long off) { return __ldg(a.w + size_t(q) * N + size_t((long long)o + off)); };
    auto offs = [&](int ax, int s1) { return (long long)s1 * (long long)st3[ax]; };
    // -- reconstruction (see ader4.cu): [0] mean, [1..4] x, [5..8] y, [9..12] z, [13..22]
    //    mixed; 18 WENO-AO tasks, 60 mixed terms and the 4 x 4 implicit-source inverse
    for (int task = t; task < 18 + NF * 10 + 1; task += C4_NS) {
        if (task < 18) {
            const int q = task / 3, ax = task % 3;
            double m[4];
            Fault f;
            f.clear();
            weno_ao<0>(W(q, offs(ax, -2)), W(q, offs(ax, -1)), W(q, 0), W(q, offs(ax, 1)),
                       W(q, offs(ax, 2)), a.lim, m, f);
#pragma unroll
            for (int l = 0; l < 4; ++l) coef[q][1 + 4 * ax + l] = m[l];
            if (ax == 0) coef[q][0] = W(q, 0);
        } else if (task < 18 + NF * 10) {
            const int q = (task - 18) / 10, term = (task - 18) % 10;
            auto val = [&](int p1, int s1, int p2, int s2) {
                return W(q, offs(p1, s1) + offs(p2, s2));
            };
            double v;
            if (term < 3) {
                const int p1 = term, r = (term + 1) % 3;
                v = 0.25 * ((val(p1, 1, r, 1) - val(p1, 1, r, -1)) -
                            (val(p1, -1, r, 1) - val(p1, -1, r, -1)));
            } else if (term < 9) {
                const int pair = (term - 3) / 2, sw = (term - 3) % 2;
                const int a1 = pair, a2 = (pair + 1) % 3;
                const int p1 = sw == 0 ? a1 : a2, r = sw == 0 ? a2 : a1;
                auto d2 = [&](int sg) {
                    return (val(p1, 1, r, sg) - 2.0 * val(p1, 0, r, sg)) + val(p1, -1, r, sg);
                };
                v = 0.25 * (d2(1) - d2(-1));
            } else {
                double acc = 0.0;
                for (int cc = -1; cc <= 1; cc += 2)
                    for (int bb = -1; bb <= 1; bb += 2)
                        for (int aa = -1; aa <= 1; aa += 2)
                            acc += double(aa * bb * cc) *
                                   W(q, offs(0, aa) + offs(1, bb) + offs(2, cc));
                v = 0.125 * acc;
            }
            coef[q][13 + term] = v;
        } else {
            // (I + z A)^-1, z = dt sigma / eps (Gauss-Jordan on 4 x 4; the system is diagonally
            // dominant for z >= 0, no pivoting needed)
            const double z = dt * a.sigma[o] / a.eps;
            double m[4][8];
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) {
                    m[r][c] = (r == c ? 1.0 : 0.0) + z * c_cb.A[r][c];
                    m[r][4 + c] = r == c ? 1.0 : 0.0;
                }
            for (int c = 0; c < 4; ++c) {
                const double ip = 1.0 / m[c][c];
                for (int cc = 0; cc < 8; ++cc) m[c][cc] *= ip;
                for (int r = 0; r < 4; ++r)
                    if (r != c) {
                        const double fct = m[r][c];
                        for (int cc = 0; cc < 8; ++cc) m[r][cc] -= fct * m[c][cc];
                    }
            }
            for (int r = 0; r < 4; ++r)
                for (int c = 0; c < 4; ++c) minv[r][c] = m[r][4 + c];
        }
    }
    __syncthreads();
    const int ni = t & 3, nj = (t >> 2) & 3, nk = t >> 4;
    auto sw = [](int n) { return n ^ (((n >> 4) & 1) * 5); };
    double p0[NF];
    {
        double px[4], py[4], pz[4];
        psi4(c_cb.xi[ni], px);
        psi4(c_cb.xi[nj], py);
        psi4(c_cb.xi[nk], pz);
#pragma unroll
        for (int q = 0; q < NF; ++q) {
            const double* c = coef[q];
            double v = c[0];
#pragma unroll
            for (int l = 0; l < 4; ++l) v += c[1 + l] * px[l] + c[5 + l] * py[l] + c[9 + l] * pz[l];
            v += c[13] * px[0] * py[0] + c[14] * py[0] * pz[0] + c[15] * pz[0] * px[0];
            v += c[16] * px[1] * py[0] + c[17] * px[0] * py[1];
            v += c[18] * py[1] * pz[0] + c[19] * py[0] * pz[1];
            v += c[20] * pz[1] * px[0] + c[21] * pz[0] * px[1];
            v += c[22] * px[0] * py[0] * pz[0];
            p0[q] = v;
        }
    }
    double Q[4][NF];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int q = 0; q < NF; ++q) Q[m][q] = p0[q];
    double wx[4], wy[4], wz[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        wx[l] = c_cb.D[ni][l] * a.id[0];
        wy[l] = c_cb.D[nj][l] * a.id[1];
        wz[l] = c_cb.D[nk][l] * a.id[2];
    }
    auto F = [&](int mm, int ax, int q, int slot) -> double& {
        return U[((mm * 3 + ax) * NF + q) * C4_NS + slot];
    };
    const int ts = sw(t);
    const double ie = 1.0 / a.eps, im = 1.0 / a.mu;
    for (int it = 0; it < 4; ++it) {
        double dv[4][NF];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int mm = 0; mm < 2; ++mm) {
                const int m = 2 * h + mm;
                double fl[NF];
                maxwell_flux<0>(Q[m], ie, im, fl);
#pragma unroll
                for (int q = 0; q < NF; ++q) F(mm, 0, q, ts) = fl[q];
                maxwell_flux<1>(Q[m], ie, im, fl);
#pragma unroll
                for (int q = 0; q < NF; ++q) F(mm, 1, q, ts) = fl[q];
                maxwell_flux<2>(Q[m], ie, im, fl);
#pragma unroll
                for (int q = 0; q < NF; ++q) F(mm, 2, q, ts) = fl[q];
            }
            __syncthreads();
#pragma unroll
            for (int mm = 0; mm < 2; ++mm) {
                const int m = 2 * h + mm;
#pragma unroll
                for (int q = 0; q < NF; ++q) dv[m][q] = 0.0;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const int tx = sw((t & ~3) | l), ty = sw((t & ~12) | (l << 2)),
                              tz = sw((t & ~48) | (l << 4));
#pragma unroll
                    for (int q = 0; q < NF; ++q)
                        dv[m][q] += wx[l] * F(mm, 0, q, tx) + wy[l] * F(mm, 1, q, ty) +
                                    wz[l] * F(mm, 2, q, tz);
                }
            }
            __syncthreads();
        }
        // right-hand sides P - dt sum_l A_ml div_l; D: the implicit source over this node's
        // time nodes (minv); B: explicit
        double r[4][NF];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int q = 0; q < NF; ++q) {
                double v = p0[q];
#pragma unroll
                for (int l = 0; l < 4; ++l) v -= (dt * c_cb.A[m][l]) * dv[l][q];
                r[m][q] = v;
            }
#pragma unroll
        for (int m = 0; m < 4; ++m) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double v = 0.0;
#pragma unroll
                for (int l = 0; l < 4; ++l) v += minv[m][l] * r[l][q];
                Q[m][q] = v;
            }
#pragma unroll
            for (int q = 3; q < NF; ++q) Q[m][q] = r[m][q];
        }
    }
    // -- outputs: (1) time -> the 2 Gauss times, in registers: T[q][tg][slotT(node)]
    double* T = U;
    double* S = U + C4_T;  // S[q][r + r / 16], r = ((C * 2 + g) * 2 + tg) * 16 + b1 * 4 + b2
    auto slotT = [](int n) { return n ^ ((n >> 4) * 5); };
#pragma unroll
    for (int tg = 0; tg < 2; ++tg)
#pragma unroll
        for (int q = 0; q < NF; ++q) {
            double v = 0.0;
#pragma unroll
            for (int m = 0; m < 4; ++m) v += c_cb.LT[tg][m] * Q[m][q];
            T[(q * 2 + tg) * C4_NS + slotT(t)] = v;
        }
    __syncthreads();
    // (2) the edge axis C at its Gauss point g
    for (int r = t; r < 192; r += C4_NS) {
        const int C = r >> 6, g = (r >> 5) & 1, tg = (r >> 4) & 1, b1 = (r >> 2) & 3, b2 = r & 3;
        double v[NF] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            int c[3];
            c[C] = l;
            c[(C + 1) % 3] = b1;
            c[(C + 2) % 3] = b2;
            const int node = (c[2] * 4 + c[1]) * 4 + c[0];
            const double w = c_cb.LG[g][l];
#pragma unroll
            for (int q = 0; q < NF; ++q) v[q] += w * T[(q * 2 + tg) * C4_NS + slotT(node)];
        }
#pragma unroll
        for (int q = 0; q < NF; ++q) S[q * C4_SQ + r + (r >> 4)] = v[q];
    }
    __syncthreads();
    // (3) the edge points: corner (la, lb) in the (C+1, C+2) plane at +-1/2 (la = 0: +1/2),
    //     e = ((C * 4 + 2 lb + la) * 2 + g) * 2 + tg
    if (t < C4_EDGE) {
        const int tg = t & 1, g = (t >> 1) & 1, corner = (t >> 2) & 3, C = t >> 4;
        const double* w1 = c_cb.LF[corner & 1];
        const double* w2 = c_cb.LF[corner >> 1];
        const int base = ((C * 2 + g) * 2 + tg) * 16;
        double v[NF] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int b1 = 0; b1 < 4; ++b1)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
                const double ww = w1[b1] * w2[b2];
                const int r = base + b1 * 4 + b2;
#pragma unroll
                for (int q = 0; q < NF; ++q) v[q] += ww * S[q * C4_SQ + r + (r >> 4)];
            }
#pragma unroll
        for (int q = 0; q < NF; ++q) __stcs(a.states + (size_t(t) * NF + q) * N + o, v[q]);
    }
}

template <int C>
__global__ void __launch_bounds__(128) k_ced4_edge(CArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    constexpr int AA = (C + 1) % 3, BB = (C + 2) % 3;
    const int ex = b.n[0] + (C != 0), ey = b.n[1] + (C != 1), ez = b.n[2] + (C != 2);
    const size_t cnt = size_t(ex) * ey * ez;
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    const int c0 = int(r % ex), c1 = int((r / ex) % ey), c2 = int(r / (size_t(ex) * ey));
    const size_t o = at(b, c2 + b.gh, c1 + b.gh, c0 + b.gh);
    const size_t sa = stride(b, AA), sb = stride(b, BB), N = b.N;
    double sg = 0.0;
#pragma unroll
    for (int lb = 0; lb < 2; ++lb)
#pragma unroll
        for (int la = 0; la < 2; ++la) sg = sg + a.sigma[o - (la == 0 ? sa : 0) - (lb == 0 ? sb : 0)];
    sg = 0.25 * sg;
    const double ta = 1.0 / (1.0 + sg * a.d[AA] / (2.0 * a.c * a.eps));
    const double tb = 1.0 / (1.0 + sg * a.d[BB] / (2.0 * a.c * a.eps));
    const double hc = 0.5 * a.c;
    double E = 0.0, H = 0.0;
    for (int gp = 0; gp < 4; ++gp) {  // (g, tg): the 2 x 2 space-time Gauss points, weight 1/4
        double e = 0.0, h = 0.0, dbp = 0.0, dbm = 0.0, dap = 0.0, dam = 0.0;
        double bbp = 0.0, bbm = 0.0, bap = 0.0, bam = 0.0;
#pragma unroll
        for (int lb = 0; lb < 2; ++lb)
#pragma unroll
            for (int la = 0; la < 2; ++la) {
                const size_t z = o - (la == 0 ? sa : 0) - (lb == 0 ? sb : 0);
                const int eidx = (C * 4 + 2 * lb + la) * 4 + gp;
                double u[NF];
#pragma unroll
                for (int q = 0; q < NF; ++q) u[q] = __ldg(a.states + (size_t(eidx) * NF + q) * N + z);
                e = e + u[C];
                h = h + u[3 + C];
                if (la) { dbp = dbp + u[BB]; bbp = bbp + u[3 + BB]; }
                else { dbm = dbm + u[BB]; bbm = bbm + u[3 + BB]; }
                if (lb) { dap = dap + u[AA]; bap = bap + u[3 + AA]; }
                else { dam = dam + u[AA]; bam = bam + u[3 + AA]; }
            }
        E += 0.25 * (0.25 * e / a.eps + hc * ta * (0.5 * bbp - 0.5 * bbm) -
                     hc * tb * (0.5 * bap - 0.5 * bam));
        H += 0.25 * (0.25 * h / a.mu - hc * ta * (0.5 * dbp - 0.5 * dbm) +
                     hc * tb * (0.5 * dap - 0.5 * dam));
    }
    a.emf[size_t(C) * N + o] = E;
    a.hmf[size_t(C) * N + o] = H;
}

__global__ void k_ced4_update(CArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    const int px = b.n[0] + 1, py = b.n[1] + 1;
    const size_t cnt = size_t(px) * py * (b.n[2] + 1);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    const int i = int(r % px), j = int((r / px) % py), k = int(r / (size_t(px) * py));
    const bool ci = i < b.n[0], cj = j < b.n[1], ck = k < b.n[2];
    const size_t o = at(b, k + b.gh, j + b.gh, i + b.gh);
    const size_t N = b.N, sx = 1, sy = b.P, sz = size_t(b.P) * b.Q;
    const double dt = a.ctl->dt;
    const double cx = dt / a.d[0], cy = dt / a.d[1], cz = dt / a.d[2];
    const double *ex = a.emf, *ey = a.emf + N, *ez = a.emf + 2 * N;
    const double *hx = a.hmf, *hy = a.hmf + N, *hz = a.hmf + 2 * N;
    double* s = a.s;
    // D on the low A face of zone o: the exponential conduction step with the space-time
    // averaged curl H of the edges, D = exp(-z) D + phi(z) dt <curl H>, z = s_f dt -- exact for
    // sigma = 0 (the fourth-order flux integral) and for frozen curl H, L-stable for z >> 1.
    // (An explicit corrector source -dt s <D>_f from the zones' predictors would multiply the
    // face-vs-reconstruction mismatch by s dt and blows up in a good conductor.)
    const double ie = 1.0 / a.eps;
    auto dstep = [&](int A, size_t so, double curl) {
        double e_, p_;
        decay(0.5 * (a.sigma[o] + a.sigma[o - so]) * ie * dt, e_, p_);
        s[A * N + o] = e_ * s[A * N + o] + p_ * curl;
    };
    if (cj && ck) {
        s[3 * N + o] = s[3 * N + o] - (cy * (ez[o + sy] - ez[o]) - cz * (ey[o + sz] - ey[o]));
        dstep(0, sx, cy * (hz[o + sy] - hz[o]) - cz * (hy[o + sz] - hy[o]));
    }
    if (ci && ck) {
        s[4 * N + o] = s[4 * N + o] - (cz * (ex[o + sz] - ex[o]) - cx * (ez[o + 1] - ez[o]));
        dstep(1, sy, cz * (hx[o + sz] - hx[o]) - cx * (hz[o + 1] - hz[o]));
    }
    if (ci && cj) {
        s[5 * N + o] = s[5 * N + o] - (cx * (ey[o + 1] - ey[o]) - cy * (ex[o + sy] - ex[o]));
        dstep(2, sz, cx * (hy[o + 1] - hy[o]) - cy * (hx[o + sy] - hx[o]));
    }
}

// host: Gauss-Legendre space basis, Radau IIA time basis
CedBasis make_ced_basis() {
    CedBasis bs;
    const double gl[4] = {-0.8611363115940526, -0.3399810435848563, 0.3399810435848563,
                          0.8611363115940526};
    const double gw[4] = {0.3478548451374538, 0.6521451548625461, 0.6521451548625461,
                          0.3478548451374538};
    const double rc[4] = {0.08858795951270395, 0.4094668644407347, 0.7876594617608471, 1.0};
    for (int l = 0; l < 4; ++l) bs.xi[l] = 0.5 * gl[l];
    auto lag = [](const double* n, int l, double x) {
        double v = 1.0;
        for (int m = 0; m < 4; ++m)
            if (m != l) v *= (x - n[m]) / (n[l] - n[m]);
        return v;
    };
    auto dlag = [](const double* n, int l, double x) {
        double sum = 0.0;
        for (int kk = 0; kk < 4; ++kk) {
            if (kk == l) continue;
            double v = 1.0 / (n[l] - n[kk]);
            for (int m = 0; m < 4; ++m)
                if (m != l && m != kk) v *= (x - n[m]) / (n[l] - n[m]);
            sum += v;
        }
        return sum;
    };
    const double g2 = 0.5 / std::sqrt(3.0);
    for (int r = 0; r < 4; ++r)
        for (int l = 0; l < 4; ++l) {
            bs.D[r][l] = dlag(bs.xi, l, bs.xi[r]);
            double sum = 0.0;  // int_0^{c_r} L_l (cubic): 4-point Gauss on [0, c_r]
            for (int g = 0; g < 4; ++g) sum += 0.5 * rc[r] * gw[g] * lag(rc, l, 0.5 * rc[r] * (gl[g] + 1.0));
            bs.A[r][l] = sum;
        }
    for (int l = 0; l < 4; ++l) {
        bs.LF[0][l] = lag(bs.xi, l, 0.5);
        bs.LF[1][l] = lag(bs.xi, l, -0.5);
        bs.LG[0][l] = lag(bs.xi, l, -g2);
        bs.LG[1][l] = lag(bs.xi, l, g2);
        bs.LT[0][l] = lag(rc, l, 0.5 - g2);
        bs.LT[1][l] = lag(rc, l, 0.5 + g2);
    }
    return bs;
}

__global__ void k_ced_div(CArgs a, double* out) {
    const Box& b = a.b;
    const size_t cnt = size_t(b.n[0]) * b.n[1] * b.n[2];
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    double v[2] = {0.0, 0.0};
    if (r < cnt) {
        const int i = int(r % b.n[0]), j = int((r / b.n[0]) % b.n[1]),
                  k = int(r / (size_t(b.n[0]) * b.n[1]));
        const size_t o = at(b, k + b.gh, j + b.gh, i + b.gh), N = b.N;
        const double m = fmin(a.d[0], fmin(a.d[1], a.d[2]));
        for (int f = 0; f < 2; ++f) {
            const double* s = a.s + size_t(3 * (1 - f)) * N;  // f = 0: B, f = 1: D
            const double dv = (s[o + 1] - s[o]) / a.d[0] + (s[N + o + b.P] - s[N + o]) / a.d[1] +
                              (s[2 * N + o + size_t(b.P) * b.Q] - s[2 * N + o]) / a.d[2];
            v[f] = fabs(dv) * m;
        }
    }
    for (int f = 0; f < 2; ++f) {
        double d = v[f];
#pragma unroll
        for (int sft = 16; sft > 0; sft >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, sft));
        if ((threadIdx.x & 31) == 0)
            atomicMax(reinterpret_cast<unsigned long long*>(out + f),
                      static_cast<unsigned long long>(__double_as_longlong(d)));
    }
}

__global__ void k_ced_advance(StepCtl* c) {
    if (c->done) return;
    c->t = c->t + c->dt;
    c->steps += 1;
    double dn = c->dt_next;  // the medium's constant CFL step
    if (c->t_final > 0.0) {
        double rem = c->t_final - c->t;
        if (rem <= 1e-12 * c->t_final) c->done = 1;
        else if (dn >= rem) dn = rem;
    }
    c->dt = dn;
}

}  // namespace ced
}  // namespace hc

using namespace hc;
using namespace hc::ced;

struct hc_ced {
    hc_geom g;
    hc_ced_params p;
    Box b;
    double *s = nullptr, *sigma = nullptr, *w = nullptr, *states = nullptr, *ht = nullptr, *emf = nullptr,
           *hmf = nullptr, *scratch = nullptr;
    StepCtl* ctl = nullptr;
    cudaStream_t st = nullptr;
    long launches = 0;
    StepGraph graph;
};

namespace {

CArgs cargs(const hc_ced* m) {
    CArgs a;
    a.s = m->s;
    a.sigma = m->sigma;
    a.w = m->w;
    a.states = m->states;
    a.ht = m->ht;
    a.emf = m->emf;
    a.hmf = m->hmf;
    a.b = m->b;
    a.d[0] = m->g.dx;
    a.d[1] = m->g.dy;
    a.d[2] = m->g.dz;
    for (int d = 0; d < 3; ++d) a.id[d] = 1.0 / a.d[d];
    a.eps = m->p.eps;
    a.mu = m->p.mu;
    a.c = 1.0 / std::sqrt(m->p.eps * m->p.mu);
    a.lim = Limiter{m->p.lim.cfac_rho, m->p.lim.cfac_other, m->p.lim.weno_eps,
                    m->p.lim.weno_w[0], m->p.lim.weno_w[1], m->p.lim.weno_w[2]};
    for (int d = 0; d < 3; ++d) a.bc[d] = m->p.bc[d];
    a.ctl = m->ctl;
    return a;
}


int launch_step4(hc_ced* m) {
    CArgs a = cargs(m);
    const Box& b = m->b;
    cudaStream_t st = m->st;
    k_ced_ghosts<<<blocks(shell_count(b), 256), 256, 0, st>>>(a, 0);
    k_ced_cell<true><<<blocks(b.N, 256), 256, 0, st>>>(a);
    const size_t ring = size_t(b.n[0] + 2) * (b.n[1] + 2) * (b.n[2] + 2);
    k_ced4_predict<<<unsigned(ring), C4_NS, 0, st>>>(a);
    const size_t ex = size_t(b.n[0]) * (b.n[1] + 1) * (b.n[2] + 1);
    const size_t ey = size_t(b.n[0] + 1) * b.n[1] * (b.n[2] + 1);
    const size_t ez = size_t(b.n[0] + 1) * (b.n[1] + 1) * b.n[2];
    k_ced4_edge<0><<<blocks(ex, 128), 128, 0, st>>>(a);
    k_ced4_edge<1><<<blocks(ey, 128), 128, 0, st>>>(a);
    k_ced4_edge<2><<<blocks(ez, 128), 128, 0, st>>>(a);
    const size_t up = size_t(b.n[0] + 1) * (b.n[1] + 1) * (b.n[2] + 1);
    k_ced4_update<<<blocks(up, 256), 256, 0, st>>>(a);
    k_ced_advance<<<1, 1, 0, st>>>(m->ctl);
    m->launches += 8;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "ced order-4 step launch");
}

int launch_step(hc_ced* m) {
    if (m->p.order == 4) return launch_step4(m);
    CArgs a = cargs(m);
    const Box& b = m->b;
    const bool o3 = m->p.order == 3;
    cudaStream_t st = m->st;
    k_ced_ghosts<<<blocks(shell_count(b), 256), 256, 0, st>>>(a, 0);
    if (o3) k_ced_cell<true><<<blocks(b.N, 256), 256, 0, st>>>(a);
    else k_ced_cell<false><<<blocks(b.N, 256), 256, 0, st>>>(a);
    const size_t ring = size_t(b.n[0] + 2) * (b.n[1] + 2) * (b.n[2] + 2);
    if (o3) k_ced_predict<true><<<blocks(ring, 128), 128, 0, st>>>(a);
    else k_ced_predict<false><<<blocks(ring, 128), 128, 0, st>>>(a);
    const size_t ex = size_t(b.n[0]) * (b.n[1] + 1) * (b.n[2] + 1);
    const size_t ey = size_t(b.n[0] + 1) * b.n[1] * (b.n[2] + 1);
    const size_t ez = size_t(b.n[0] + 1) * (b.n[1] + 1) * b.n[2];
    if (o3) {
        k_ced_edge<true, 0><<<blocks(ex, 128), 128, 0, st>>>(a);
        k_ced_edge<true, 1><<<blocks(ey, 128), 128, 0, st>>>(a);
        k_ced_edge<true, 2><<<blocks(ez, 128), 128, 0, st>>>(a);
    } else {
        k_ced_edge<false, 0><<<blocks(ex, 128), 128, 0, st>>>(a);
        k_ced_edge<false, 1><<<blocks(ey, 128), 128, 0, st>>>(a);
        k_ced_edge<false, 2><<<blocks(ez, 128), 128, 0, st>>>(a);
    }
    const size_t up = size_t(b.n[0] + 1) * (b.n[1] + 1) * (b.n[2] + 1);
    k_ced_update<<<blocks(up, 256), 256, 0, st>>>(a);
    k_ced_advance<<<1, 1, 0, st>>>(m->ctl);
    m->launches += 8;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "ced step launch");
}

}  // namespace

extern "C" {

int hc_ced_create(const hc_geom* g, const hc_ced_params* p, hc_ced** out) {
    if (!p || !out) {
        set_error(HC_INVALID, "null argument");
        return HC_INVALID;
    }
    int rc = validate_geom(g, p->order == 4 ? 3 : p->order);  // (order 4: the same stencils)
    if (rc) return rc;
    if (p->order < 2 || p->order > 4) {
        set_error(HC_INVALID, "ced: order must be 2, 3 or 4");
        return HC_INVALID;
    }
    if (g->ghost < (p->order >= 3 ? 4 : 2)) {
        set_error(HC_INVALID, "ced: orders 3 and 4 need a ghost width of at least 4");
        return HC_INVALID;
    }
    if (!(p->eps > 0.0) || !(p->mu > 0.0)) {
        set_error(HC_INVALID, "ced: eps and mu must be positive");
        return HC_INVALID;
    }
    for (int d = 0; d < 3; ++d)
        if (p->bc[d] != HC_PERIODIC && p->bc[d] != HC_OUTFLOW) {
            set_error(HC_INVALID, "ced: boundary kind must be periodic or outflow");
            return HC_INVALID;
        }
    hc_ced* m = new (std::nothrow) hc_ced;
    if (!m) {
        set_error(HC_CUDA, "out of host memory");
        return HC_CUDA;
    }
    m->g = *g;
    m->p = *p;
    Box& b = m->b;
    b.n[0] = g->nx;
    b.n[1] = g->ny;
    b.n[2] = g->nz;
    b.gh = g->ghost;
    b.P = g->nx + 2 * g->ghost + 1;
    b.Q = g->ny + 2 * g->ghost + 1;
    b.R = g->nz + 2 * g->ghost + 1;
    b.N = size_t(b.P) * b.Q * b.R;
    const size_t B = sizeof(double) * b.N;
    cudaError_t e = cudaSetDevice(p->device);
    if (e == cudaSuccess) e = cudaMalloc(&m->s, NF * B);
    if (e == cudaSuccess) e = cudaMalloc(&m->sigma, B);
    if (e == cudaSuccess) e = cudaMalloc(&m->w, NF * B);
    if (e == cudaSuccess) e = cudaMalloc(&m->states, size_t(p->order == 4 ? C4_EDGE : 12) * NF * B);
    if (e == cudaSuccess) e = cudaMalloc(&m->ht, NF * B);
    if (e == cudaSuccess) e = cudaMalloc(&m->emf, 3 * B);
    if (e == cudaSuccess) e = cudaMalloc(&m->hmf, 3 * B);
    if (e == cudaSuccess) e = cudaMalloc(&m->scratch, 2 * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&m->ctl, sizeof(StepCtl));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemset(m->s, 0, NF * B);
    if (e == cudaSuccess) e = cudaMemset(m->sigma, 0, B);
    if (e == cudaSuccess) e = cudaMemset(m->emf, 0, 3 * B);
    if (e == cudaSuccess) e = cudaMemset(m->hmf, 0, 3 * B);
    if (e == cudaSuccess) {
        StepCtl c{};
        e = cudaMemcpy(m->ctl, &c, sizeof c, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && p->order == 4) {
        CedBasis bs = make_ced_basis();
        e = cudaMemcpyToSymbol(c_cb, &bs, sizeof bs);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_ced4_predict,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    if (e != cudaSuccess) {
        hc_ced_destroy(m);
        return cuda_fail(e, "hc_ced_create");
    }
    *out = m;
    return HC_OK;
}

int hc_ced_destroy(hc_ced* m) {
    if (!m) return HC_OK;
    cudaSetDevice(m->p.device);
    if (m->st) cudaStreamSynchronize(m->st);
    for (double* p : {m->s, m->sigma, m->w, m->states, m->ht, m->emf, m->hmf, m->scratch}) cudaFree(p);
    cudaFree(m->ctl);
    if (m->st) cudaStreamDestroy(m->st);
    delete m;
    return HC_OK;
}

int hc_ced_upload(hc_ced* m, const double* host, const double* sigma) {
    HC_CUDA(cudaSetDevice(m->p.device));
    const size_t B = sizeof(double) * m->b.N;
    HC_CUDA(cudaMemcpyAsync(m->s, host, NF * B, cudaMemcpyHostToDevice, m->st));
    HC_CUDA(cudaMemcpyAsync(m->sigma, sigma, B, cudaMemcpyHostToDevice, m->st));
    CArgs a = cargs(m);
    a.ctl = nullptr;
    k_ced_ghosts<<<blocks(shell_count(m->b), 256), 256, 0, m->st>>>(a, 1);  // sigma's ghosts
    m->launches += 1;
    HC_CUDA(cudaGetLastError());
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

int hc_ced_download(hc_ced* m, double* host) {
    HC_CUDA(cudaSetDevice(m->p.device));
    HC_CUDA(cudaMemcpyAsync(host, m->s, sizeof(double) * NF * m->b.N, cudaMemcpyDeviceToHost,
                            m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

int hc_ced_cfl_dt(hc_ced* m, double cfl, double* dt) {
    const double c = 1.0 / std::sqrt(m->p.eps * m->p.mu);
    *dt = cfl / (c / m->g.dx + c / m->g.dy + c / m->g.dz);
    return HC_OK;
}

int hc_ced_set_time(hc_ced* m, double t, double dt, double t_final) {
    HC_CUDA(cudaSetDevice(m->p.device));
    StepCtl c{};
    c.t = t;
    c.dt = dt;
    c.dt_next = dt;
    c.t_final = t_final;
    if (t_final > 0.0 && dt > t_final - t) c.dt = t_final - t;
    HC_CUDA(cudaMemcpyAsync(m->ctl, &c, sizeof c, cudaMemcpyHostToDevice, m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

int hc_ced_step(hc_ced* m, int n) {
    HC_CUDA(cudaSetDevice(m->p.device));
    // n > 1: one captured step replayed as a CUDA graph (graph_step.cuh)
    return replay_steps(m->graph, m->st, 0.0, m->launches, n, [&] { return launch_step(m); });
}

int hc_ced_sync(hc_ced* m, double* t, double* dt, long* steps) {
    HC_CUDA(cudaSetDevice(m->p.device));
    StepCtl c;
    HC_CUDA(cudaMemcpyAsync(&c, m->ctl, sizeof c, cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    if (t) *t = c.t;
    if (dt) *dt = c.dt;
    if (steps) *steps = long(c.steps);
    return HC_OK;
}

int hc_ced_max_div(hc_ced* m, double* divb, double* divd) {
    HC_CUDA(cudaSetDevice(m->p.device));
    CArgs a = cargs(m);
    HC_CUDA(cudaMemsetAsync(m->scratch, 0, 2 * sizeof(double), m->st));
    const size_t act = size_t(m->b.n[0]) * m->b.n[1] * m->b.n[2];
    k_ced_div<<<blocks(act, 256), 256, 0, m->st>>>(a, m->scratch);
    m->launches += 1;
    double v[2];
    HC_CUDA(cudaMemcpyAsync(v, m->scratch, sizeof v, cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    *divb = v[0];
    *divd = v[1];
    return HC_OK;
}

long hc_ced_launches(hc_ced* m) { return m ? m->launches : 0; }

int hc_ced_stream(hc_ced* m, void** stream) {
    *stream = m->st;
    return HC_OK;
}

}  // extern "C"
