// ader4.cu -- a formally fourth-order WENO-ADER step for the Euler equations (EXTENSION: the
// reference's orders are 2 and 3, geometry.hpp:13-27; the north star names fourth order).
//
// The reference's ADER structure -- one face state per face from the reconstruction, the zone
// MEAN's time derivative tau added at the midpoint (predictor.cpp:26-60, corrector.cpp:30-33)
// -- is second order in time, so raising only the reconstruction order (the fused stepper's
// order = 4, WENO-AO) stays second order asymptotically. This module is the scheme a fourth-
// order ADER needs (Dumbser, Balsara, Toro & Munz 2008; Balsara et al. 2013), built from three
// device kernels per step:
//
//  k4_predict  one CTA per zone of active + one ring, one thread per spatial node holding its
//              4 time nodes (4 x 4 x 4 Gauss-Legendre points in the zone x 4 in [t, t + dt]):
//    reconstruction -- the degree-3 polynomial of the zone in the zero-mean Legendre basis:
//      the pure x, y, z terms up to degree 4 from WENO-AO(5,3) on each axis (pointwise.cuh
//      weno_ao, nonlinear), the ten mixed terms of total degree <= 3 (xy, yz, zx, x^2 y, x y^2,
//      y^2 z, y z^2, z^2 x, z x^2, xyz) from central differences of the 3 x 3 x 3 neighbourhood
//      (unlimited, as the reference's O3 cross modes, reconstruct.cpp:62-75); every mixed
//      coefficient is exact for cubic data because the other basis functions cancel in its
//      difference
//    local space-time predictor -- the collocation solution of u_t + div F(u) = 0 in the zone
//      with u(t) = P(x): Picard iterations q <- P - int_0^t div F(q) on the nodal basis (the
//      spatial derivative with the 4-point Lagrange derivative matrix, the time integral with the
//      4-point integration matrix), four iterations (one order in dt each)
//    outputs -- q at the 2 x 2 Gauss points of each of the six faces at the 2 Gauss times
//  k4_flux     one thread per face: the Riemann solver (Rusanov / HLL) at the 2 x 2 x 2 space-
//              time Gauss points, weighted to the face- and time-averaged flux
//  k4_update   U -= dt/dx (F_E - F_W) + ...; the CFL estimate (eval_tstep_ptwise), exact min
// Same state layout, ICs, ghost semantics and C-ABI conventions as the fused stepper; the
// parity of this scheme is unpinned (no reference code): tests measure its convergence order
// on the isentropic vortex against the exact solution (tests/test_ader4_gpu.py).
#include <cuda_runtime.h>

#include <cmath>
#include <new>
#include <string>

#include "common.cuh"
#include "fused_types.cuh"
#include "hydro_cuda.h"

namespace hc {
namespace a4 {

// ---- nodal space-time basis (host-computed in ader4_constants)
struct Basis {
    double xi[4];       // Gauss-Legendre nodes on [-1/2, 1/2]
    double D[4][4];     // d/dxi of the Lagrange basis: D[i][l] = L_l'(xi_i)
    double IT[4][4];    // int_0^{tau_m} L_l(s) ds, tau on [0, 1]
    double LF[2][4];    // L_l(+1/2), L_l(-1/2): face extrapolation
    double LG[2][4];    // L_l at the 2-point Gauss points -+1/(2 sqrt 3)
    double LT[2][4];    // time basis at the 2-point Gauss times 1/2 -+ 1/(2 sqrt 3)
};
__constant__ Basis c_b;

constexpr int NQ = 4;            // nodes per dimension (space and time)
constexpr int NT = NQ * NQ * NQ * NQ;  // space-time nodes = threads per CTA
constexpr int NPIC = 4;          // Picard iterations
constexpr int NOUT = 6 * 4 * 2;  // face points x Gauss times
constexpr int NCOEF = 23;        // 1 + 3 x 4 pure + 10 mixed

struct A4Args {
    double* u;    // state [mz][my][mx][5] (ghosts included)
    double* fs;   // [ring zone][NOUT][5] face-point states
    double* flux; // [3][5][N] time- and face-averaged fluxes at the low face of zone (storage)
    int nx, ny, nz, gh, mx, my, mz;
    double dx, dy, dz, gamma, cfl;
    Limiter lim;
    int solver, bc;
    StepCtl* ctl;
    ErrBlock* eb;
};

__device__ __forceinline__ size_t zid(const A4Args& a, int i, int j, int k) {  // storage coords
    return (size_t(k) * a.my + j) * a.mx + i;
}

// zero-mean Legendre basis on [-1/2, 1/2] (the WENO-AO basis of pointwise.cuh weno_ao)
__device__ __forceinline__ void psi(double s, double* p) {
    const double s2 = s * s;
    p[0] = s;
    p[1] = s2 - 1.0 / 12.0;
    p[2] = s * (s2 - 3.0 / 20.0);
    p[3] = s2 * s2 - (3.0 / 14.0) * s2 + 3.0 / 560.0;
}

// ---- ghost fill: every ghost zone copies its composed active image (boundary.cpp:14-39)
__global__ void k4_ghosts(A4Args a) {
    if (a.ctl->done) return;
    const size_t n = size_t(a.mx) * a.my * a.mz;
    const size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    const int i = int(r % a.mx), j = int((r / a.mx) % a.my), k = int(r / (size_t(a.mx) * a.my));
    const int ia = i - a.gh, ja = j - a.gh, ka = k - a.gh;
    if (ia >= 0 && ia < a.nx && ja >= 0 && ja < a.ny && ka >= 0 && ka < a.nz) return;
    auto map = [&](int v, int n2) {
        if (a.bc == HC_PERIODIC) return ((v % n2) + n2) % n2;
        return v < 0 ? 0 : (v >= n2 ? n2 - 1 : v);
    };
    const size_t src = zid(a, map(ia, a.nx) + a.gh, map(ja, a.ny) + a.gh, map(ka, a.nz) + a.gh);
#pragma unroll
    for (int q = 0; q < NV; ++q) a.u[r * NV + q] = a.u[src * NV + q];
}

// ---- predictor: one CTA per zone of the ring box (nx+2)(ny+2)(nz+2)
// One CTA of 64 threads per zone; thread t owns spatial node t (ni, nj, nk) and its four time
// nodes in registers, so the time integral of the Picard update and the time contraction of
// the outputs never touch shared memory (the fluxes still do, for the spatial derivatives).
// The fluxes of two time nodes are staged at a time: 15 KB of shared memory per zone.
constexpr int NS = NQ * NQ * NQ;  // spatial nodes = threads per CTA
constexpr int MH = 2;             // time nodes staged per half
#ifndef K4_MINB
#define K4_MINB 6
#endif
__global__ void __launch_bounds__(NS, K4_MINB) k4_predict(A4Args a) {
    if (a.ctl->done) return;
    __shared__ double coef[NV][NCOEF];
    // fluxes of the staged time nodes, [mm][axis][q][slot]; later T and S2. Node n lives in
    // slot n ^ (5 * bit 4 of n): the x-, y- and z-neighbour reads of a warp (8, 8 and 16
    // distinct nodes) then hit distinct banks
    __shared__ double F[MH][3][NV][NS];
    const int rx = a.nx + 2, ry = a.ny + 2;
    const int zr = blockIdx.x;
    const int ci = zr % rx - 1, cj = (zr / rx) % ry - 1, ck = zr / (rx * ry) - 1;
    const int si = ci + a.gh, sj = cj + a.gh, sk = ck + a.gh;  // storage coords
    const int t = threadIdx.x;
    auto U = [&](int di, int dj, int dk, int q) {
        return __ldg(a.u + zid(a, si + di, sj + dj, sk + dk) * NV + q);
    };
    // -- reconstruction coefficients: [0] mean, [1..4] x, [5..8] y, [9..12] z (psi1..psi4),
    //    [13] xy [14] yz [15] zx [16] x2y [17] xy2 [18] y2z [19] yz2 [20] z2x [21] zx2 [22] xyz
    //    65 tasks over 64 threads: the 15 WENO-AO ones first
    for (int task = t; task < 65; task += NS) {
        if (task < 15) {
            const int q = task / 3, ax = task % 3;
            const int di = ax == 0, dj = ax == 1, dk = ax == 2;
            double m[4];
            Fault f;
            f.clear();
            weno_ao<0>(U(-2 * di, -2 * dj, -2 * dk, q), U(-di, -dj, -dk, q), U(0, 0, 0, q),
                       U(di, dj, dk, q), U(2 * di, 2 * dj, 2 * dk, q), a.lim, m, f);
#pragma unroll
            for (int l = 0; l < 4; ++l) coef[q][1 + 4 * ax + l] = m[l];
            if (ax == 0) coef[q][0] = U(0, 0, 0, q);
        } else {
            const int q = (task - 15) / 10, term = (task - 15) % 10;
            double v = 0.0;
            // the pair (p, r) of axes of a mixed term and the 2D difference in their plane
            auto val = [&](int ax1, int s1, int ax2, int s2) {
                int d[3] = {0, 0, 0};
                d[ax1] += s1;
                d[ax2] += s2;
                return U(d[0], d[1], d[2], q);
            };
            if (term < 3) {  // xy, yz, zx: 1/4 [u(1,1) - u(1,-1) - u(-1,1) + u(-1,-1)]
                const int p = term, r = (term + 1) % 3;
                v = 0.25 * ((val(p, 1, r, 1) - val(p, 1, r, -1)) -
                            (val(p, -1, r, 1) - val(p, -1, r, -1)));
            } else if (term < 9) {
                // psi2 along p times psi1 along r: 1/4 [D2_p u(., r = +1) - D2_p u(., r = -1)]
                const int pair = (term - 3) / 2, sw = (term - 3) % 2;
                const int a1 = pair, a2 = (pair + 1) % 3;  // (x,y) (y,z) (z,x)
                const int p = sw == 0 ? a1 : a2, r = sw == 0 ? a2 : a1;
                auto d2 = [&](int s) {
                    return (val(p, 1, r, s) - 2.0 * val(p, 0, r, s)) + val(p, -1, r, s);
                };
                v = 0.25 * (d2(1) - d2(-1));
            } else {  // xyz: 1/8 sum abc u(a,b,c)
                double acc = 0.0;
                for (int cc = -1; cc <= 1; cc += 2)
                    for (int bb = -1; bb <= 1; bb += 2)
                        for (int aa = -1; aa <= 1; aa += 2)
                            acc += double(aa * bb * cc) * U(aa, bb, cc, q);
                v = 0.125 * acc;
            }
            coef[q][13 + term] = v;
        }
    }
    __syncthreads();
    // -- the polynomial at this thread's spatial node (the same at every time node)
    const int ni = t & 3, nj = (t >> 2) & 3, nk = t >> 4;
    auto sw = [](int n) { return n ^ (((n >> 4) & 1) * 5); };
    const int ts = sw(t);
    double p0[NV];
    {
        double px[4], py[4], pz[4];
        psi(c_b.xi[ni], px);
        psi(c_b.xi[nj], py);
        psi(c_b.xi[nk], pz);
#pragma unroll
        for (int q = 0; q < NV; ++q) {
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
    double Q[NQ][NV];
#pragma unroll
    for (int m = 0; m < NQ; ++m)
#pragma unroll
        for (int q = 0; q < NV; ++q) Q[m][q] = p0[q];
    const double dt = a.ctl->dt;
    const double idx = 1.0 / a.dx, idy = 1.0 / a.dy, idz = 1.0 / a.dz;
    double wx[4], wy[4], wz[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        wx[l] = c_b.D[ni][l] * idx;
        wy[l] = c_b.D[nj][l] * idy;
        wz[l] = c_b.D[nk][l] * idz;
    }
    Fault f;
    f.clear();
    // -- Picard iterations of the local space-time predictor
    for (int it = 0; it < NPIC; ++it) {
        double dv[NQ][NV];
#pragma unroll
        for (int h = 0; h < NQ / MH; ++h) {
#pragma unroll
            for (int mm = 0; mm < MH; ++mm) {
                const int m = h * MH + mm;
                Prim pr = cons_to_prim<0>(Q[m], a.gamma, f);
                double fl[NV];
                physical_flux_q<0>(Q[m], pr, fl);
#pragma unroll
                for (int q = 0; q < NV; ++q) F[mm][0][q][ts] = fl[q];
                physical_flux_q<1>(Q[m], pr, fl);
#pragma unroll
                for (int q = 0; q < NV; ++q) F[mm][1][q][ts] = fl[q];
                physical_flux_q<2>(Q[m], pr, fl);
#pragma unroll
                for (int q = 0; q < NV; ++q) F[mm][2][q][ts] = fl[q];
            }
            __syncthreads();
#pragma unroll
            for (int mm = 0; mm < MH; ++mm) {
                const int m = h * MH + mm;
#pragma unroll
                for (int q = 0; q < NV; ++q) dv[m][q] = 0.0;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const int tx = sw((t & ~3) | l), ty = sw((t & ~12) | (l << 2)),
                              tz = sw((t & ~48) | (l << 4));
#pragma unroll
                    for (int q = 0; q < NV; ++q)
                        dv[m][q] += wx[l] * F[mm][0][q][tx] + wy[l] * F[mm][1][q][ty] +
                                    wz[l] * F[mm][2][q][tz];
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int m = 0; m < NQ; ++m)
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                double qn = p0[q];
#pragma unroll
                for (int l = 0; l < 4; ++l) qn -= (dt * c_b.IT[m][l]) * dv[l][q];
                Q[m][q] = qn;
            }
    }
    if (f.code) record_fault(a.eb, ST_PREDICT, f, ci, cj, ck, 0);
    // -- face points: out = ((face * 4 + g) * 2 + tg), face = 2A (+A) / 2A + 1 (-A),
    //    g = g1 * 2 + g2 over the two transverse axes (A+1, A+2) at the Gauss points; the
    //    tensor-product interpolation contracted one dimension at a time:
    //    (1) time -> the 2 Gauss times, in registers: T[q][tg][slotT(node)]
    //    (2) the face-normal axis -> +-1/2: S2[q][r + r / 16], r = [A][side][tg][b1][b2]
    //    (3) the two transverse axes -> the 2 x 2 Gauss points
    //    The swizzles (slotT flips the x and y bits of a node by its z, S2 skews every 16
    //    entries by one) keep the strided reads of (2) and (3) on distinct banks.
    double* T = &F[0][0][0][0];       // [5][2][NS]
    double* S2 = T + NV * 2 * NS;     // [5][204]
    constexpr int S2Q = 204;
    auto slotT = [](int n) { return n ^ ((n >> 4) * 5); };
#pragma unroll
    for (int tg = 0; tg < 2; ++tg)
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double v = 0.0;
#pragma unroll
            for (int m = 0; m < 4; ++m) v += c_b.LT[tg][m] * Q[m][q];
            T[(q * 2 + tg) * NS + slotT(t)] = v;
        }
    __syncthreads();
    for (int r = t; r < 192; r += NS) {
        const int A = r >> 6, side = (r >> 5) & 1, tg = (r >> 4) & 1, b1 = (r >> 2) & 3,
                  b2 = r & 3;
        double v[NV] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            int c[3];
            c[A] = l;
            c[(A + 1) % 3] = b1;
            c[(A + 2) % 3] = b2;
            const int node = (c[2] * 4 + c[1]) * 4 + c[0];
            const double w = c_b.LF[side][l];
#pragma unroll
            for (int q = 0; q < NV; ++q) v[q] += w * T[(q * 2 + tg) * NS + slotT(node)];
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) S2[q * S2Q + r + (r >> 4)] = v[q];
    }
    __syncthreads();
    if (t < NOUT) {
        const int tg = t & 1, g = (t >> 1) & 3, face = t >> 3;
        const int A = face >> 1, side = face & 1;
        const int g1 = g >> 1, g2 = g & 1;
        double v[NV] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int b1 = 0; b1 < 4; ++b1)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
                const double w = c_b.LG[g1][b1] * c_b.LG[g2][b2];
                const int r = (((A * 2 + side) * 2 + tg) * 4 + b1) * 4 + b2;
#pragma unroll
                for (int q = 0; q < NV; ++q) v[q] += w * S2[q * S2Q + r + (r >> 4)];
            }
        double* dst = a.fs + (size_t(zr) * NOUT + t) * NV;
#pragma unroll
        for (int q = 0; q < NV; ++q) dst[q] = v[q];
    }
}

// ---- face fluxes: one thread per face of the active box (low face of zone c; c up to n on the
// face's own axis), the 2 x 2 x 2 space-time Gauss points
template <int A>
__global__ void k4_flux(A4Args a) {
    if (a.ctl->done) return;
    const int ex = a.nx + (A == 0), ey = a.ny + (A == 1), ez = a.nz + (A == 2);
    const size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= size_t(ex) * ey * ez) return;
    const int i = int(r % ex), j = int((r / ex) % ey), k = int(r / (size_t(ex) * ey));
    const int rx = a.nx + 2, ry = a.ny + 2;
    const size_t zr = (size_t(k + 1) * ry + (j + 1)) * rx + (i + 1);  // right zone (ring box)
    const size_t zl = zr - (A == 0 ? 1 : (A == 1 ? size_t(rx) : size_t(rx) * ry));
    double acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
    Fault f;
    f.clear();
    for (int g = 0; g < 4; ++g)
        for (int tg = 0; tg < 2; ++tg) {
            const double* ul = a.fs + (size_t(zl) * NOUT + ((2 * A) * 4 + g) * 2 + tg) * NV;
            const double* ur = a.fs + (size_t(zr) * NOUT + ((2 * A + 1) * 4 + g) * 2 + tg) * NV;
            double l5[NV], r5[NV], f5[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                l5[q] = ul[q];
                r5[q] = ur[q];
            }
            if (a.solver == HC_RUSANOV)
                riemann<0, A, 0>(l5, r5, a.gamma, f5, f);
            else
                riemann<1, A, 0>(l5, r5, a.gamma, f5, f);
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] += 0.125 * f5[q];  // weights 1/2 x 1/2 x 1/2
        }
    if (f.code) record_fault(a.eb, ST_FLUX, f, i, j, k, A);
    const size_t N = size_t(a.mx) * a.my * a.mz;
    const size_t o = zid(a, i + a.gh, j + a.gh, k + a.gh);
#pragma unroll
    for (int q = 0; q < NV; ++q) a.flux[(size_t(A) * NV + q) * N + o] = acc[q];
}

// ---- update and CFL estimate of the active zones
__global__ void k4_update(A4Args a) {
    if (a.ctl->done) return;
    const size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    double d = 1.0e32;
    if (r < size_t(a.nx) * a.ny * a.nz) {
        const int i = int(r % a.nx), j = int((r / a.nx) % a.ny), k = int(r / (size_t(a.nx) * a.ny));
        const size_t o = zid(a, i + a.gh, j + a.gh, k + a.gh);
        const size_t N = size_t(a.mx) * a.my * a.mz;
        const size_t sx = 1, sy = a.mx, sz = size_t(a.mx) * a.my;
        const double dt = a.ctl->dt;
        const double cx = dt / a.dx, cy = dt / a.dy, cz = dt / a.dz;
        double un[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double* fx = a.flux + (size_t(0) * NV + q) * N;
            const double* fy = a.flux + (size_t(1) * NV + q) * N;
            const double* fz = a.flux + (size_t(2) * NV + q) * N;
            un[q] = a.u[o * NV + q] - cx * (fx[o + sx] - fx[o]) - cy * (fy[o + sy] - fy[o]) -
                    cz * (fz[o + sz] - fz[o]);
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) a.u[o * NV + q] = un[q];
        Fault f;
        f.clear();
        const double v = eval_tstep<0>(un, a.cfl, a.dx, a.dy, a.dz, a.gamma, f);
        if (f.code) record_fault(a.eb, ST_UPDATE, f, i, j, k, 0);
        else d = v;
    }
    d = warp_min(d);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int w = 1; w < int(blockDim.x) / 32; ++w) m = smin(m, red[w]);
        atomic_min_pos_sparse(&a.ctl->acc, m);
    }
}

__global__ void k4_advance(StepCtl* c, const ErrBlock* eb) {
    if (c->done) return;
    for (int s = 0; s < ST_COUNT; ++s)
        if (eb->rec[s].flag) {
            c->done = 2;
            return;
        }
    c->t = c->t + c->dt;
    c->steps += 1;
    double dn = c->acc;
    c->dt_next = dn;
    c->acc = 1.0e32;
    if (c->t_final > 0.0) {  // harness.cpp:156-160
        const double rem = c->t_final - c->t;
        if (rem <= 1e-12 * c->t_final) c->done = 1;
        else if (dn >= rem) dn = rem;
    }
    c->dt = dn;
}

// host: the nodal basis (closed-form Lagrange polynomials on the Gauss-Legendre nodes)
Basis make_basis() {
    Basis b;
    const double gl[4] = {-0.8611363115940526, -0.3399810435848563, 0.3399810435848563,
                          0.8611363115940526};
    double tau[4];
    for (int i = 0; i < 4; ++i) {
        b.xi[i] = 0.5 * gl[i];
        tau[i] = 0.5 * (gl[i] + 1.0);
    }
    auto lag = [](const double* n, int l, double x) {
        double v = 1.0;
        for (int m = 0; m < 4; ++m)
            if (m != l) v *= (x - n[m]) / (n[l] - n[m]);
        return v;
    };
    auto dlag = [](const double* n, int l, double x) {
        double s = 0.0;
        for (int k = 0; k < 4; ++k) {
            if (k == l) continue;
            double v = 1.0 / (n[l] - n[k]);
            for (int m = 0; m < 4; ++m)
                if (m != l && m != k) v *= (x - n[m]) / (n[l] - n[m]);
            s += v;
        }
        return s;
    };
    // int_0^x L_l: exact for the cubic by 4-point Gauss on [0, x]
    auto ilag = [&](int l, double x) {
        double s = 0.0;
        const double gw[4] = {0.3478548451374538, 0.6521451548625461, 0.6521451548625461,
                              0.3478548451374538};
        for (int g = 0; g < 4; ++g) s += 0.5 * x * gw[g] * lag(tau, l, 0.5 * x * (gl[g] + 1.0));
        return s;
    };
    const double g2 = 0.5 / std::sqrt(3.0);
    for (int i = 0; i < 4; ++i)
        for (int l = 0; l < 4; ++l) {
            b.D[i][l] = dlag(b.xi, l, b.xi[i]);
            b.IT[i][l] = ilag(l, tau[i]);
        }
    for (int l = 0; l < 4; ++l) {
        b.LF[0][l] = lag(b.xi, l, 0.5);
        b.LF[1][l] = lag(b.xi, l, -0.5);
        b.LG[0][l] = lag(b.xi, l, -g2);
        b.LG[1][l] = lag(b.xi, l, g2);
        b.LT[0][l] = lag(tau, l, 0.5 - g2);
        b.LT[1][l] = lag(tau, l, 0.5 + g2);
    }
    return b;
}

}  // namespace a4
}  // namespace hc

using namespace hc;
using namespace hc::a4;

struct hc_ader4 {
    A4Args a{};
    int device = 0;
    cudaStream_t st = nullptr;
    size_t bytes = 0;
    long launches = 0;
};

namespace {
}

extern "C" {

int hc_ader4_create(const hc_geom* g, const hc_params* p, int boundary, int device,
                    hc_ader4** out) {
    if (!g || !p || !out) {
        set_error(HC_INVALID, "null argument");
        return HC_INVALID;
    }
    if (g->nx < 4 || g->ny < 4 || g->nz < 4) {
        set_error(HC_INVALID, "patch must have at least 4 zones per axis");
        return HC_INVALID;
    }
    if (g->ghost < 3) {
        set_error(HC_INVALID, "the fourth-order ADER step needs 3 ghost zones");
        return HC_INVALID;
    }
    auto* s = new (std::nothrow) hc_ader4;
    if (!s) {
        set_error(HC_CUDA, "out of host memory");
        return HC_CUDA;
    }
    s->device = device;
    HC_CUDA(cudaSetDevice(device));
    A4Args& a = s->a;
    a.nx = g->nx;
    a.ny = g->ny;
    a.nz = g->nz;
    a.gh = g->ghost;
    a.mx = g->nx + 2 * g->ghost;
    a.my = g->ny + 2 * g->ghost;
    a.mz = g->nz + 2 * g->ghost;
    a.dx = g->dx;
    a.dy = g->dy;
    a.dz = g->dz;
    a.gamma = p->gamma;
    a.lim = Limiter{p->lim.cfac_rho, p->lim.cfac_other, p->lim.weno_eps, p->lim.weno_w[0],
                    p->lim.weno_w[1], p->lim.weno_w[2]};
    a.solver = p->solver == HC_RUSANOV ? HC_RUSANOV : HC_HLL;
    a.bc = boundary;
    const size_t N = size_t(a.mx) * a.my * a.mz;
    const size_t ring = size_t(a.nx + 2) * (a.ny + 2) * (a.nz + 2);
    s->bytes = N * NV * sizeof(double);
    cudaError_t e = cudaMalloc(&a.u, s->bytes);
    if (e == cudaSuccess) e = cudaMalloc(&a.fs, ring * NOUT * NV * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&a.flux, 3 * NV * N * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&a.ctl, sizeof(StepCtl));
    if (e == cudaSuccess) e = cudaMalloc(&a.eb, sizeof(ErrBlock));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemset(a.eb, 0, sizeof(ErrBlock));
    if (e == cudaSuccess) {
        Basis b = make_basis();
        e = cudaMemcpyToSymbol(c_b, &b, sizeof b);
    }
    if (e == cudaSuccess)  // six 16 KB CTAs per SM
        e = cudaFuncSetAttribute(k4_predict, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) {
        int rc = cuda_fail(e, "hc_ader4_create");
        hc_ader4_destroy(s);
        return rc;
    }
    *out = s;
    return HC_OK;
}

int hc_ader4_destroy(hc_ader4* s) {
    if (!s) return HC_OK;
    cudaSetDevice(s->device);
    if (s->st) cudaStreamSynchronize(s->st);
    cudaFree(s->a.u);
    cudaFree(s->a.fs);
    cudaFree(s->a.flux);
    cudaFree(s->a.ctl);
    cudaFree(s->a.eb);
    if (s->st) cudaStreamDestroy(s->st);
    delete s;
    return HC_OK;
}

int hc_ader4_upload(hc_ader4* s, const double* host_skinny) {
    HC_CUDA(cudaSetDevice(s->device));
    HC_CUDA(cudaMemcpyAsync(s->a.u, host_skinny, s->bytes, cudaMemcpyHostToDevice, s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    return HC_OK;
}

int hc_ader4_download(hc_ader4* s, double* host_skinny) {
    HC_CUDA(cudaSetDevice(s->device));
    HC_CUDA(cudaMemcpyAsync(host_skinny, s->a.u, s->bytes, cudaMemcpyDeviceToHost, s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    return HC_OK;
}

int hc_ader4_set_time(hc_ader4* s, double t, double dt, double cfl, double t_final) {
    HC_CUDA(cudaSetDevice(s->device));
    StepCtl c{};
    c.t = t;
    c.dt = dt;
    c.t_final = t_final;
    c.acc = 1.0e32;
    c.dt_next = 1.0e32;
    if (t_final > 0.0) {
        const double rem = t_final - t;
        if (rem <= 1e-12 * t_final) c.done = 1;
        else if (c.dt >= rem) c.dt = rem;
    }
    s->a.cfl = cfl;
    HC_CUDA(cudaMemcpyAsync(s->a.ctl, &c, sizeof c, cudaMemcpyHostToDevice, s->st));
    HC_CUDA(cudaMemsetAsync(s->a.eb, 0, sizeof(ErrBlock), s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    return HC_OK;
}

int hc_ader4_step(hc_ader4* s, int n) {
    HC_CUDA(cudaSetDevice(s->device));
    const A4Args& a = s->a;
    const size_t N = size_t(a.mx) * a.my * a.mz;
    const unsigned ring = unsigned(size_t(a.nx + 2) * (a.ny + 2) * (a.nz + 2));
    const size_t act = size_t(a.nx) * a.ny * a.nz;
    for (int it = 0; it < n; ++it) {
        k4_ghosts<<<unsigned((N + 255) / 256), 256, 0, s->st>>>(a);
        k4_predict<<<ring, NS, 0, s->st>>>(a);
        const size_t fx = size_t(a.nx + 1) * a.ny * a.nz, fy = size_t(a.nx) * (a.ny + 1) * a.nz,
                     fz = size_t(a.nx) * a.ny * (a.nz + 1);
        k4_flux<0><<<unsigned((fx + 127) / 128), 128, 0, s->st>>>(a);
        k4_flux<1><<<unsigned((fy + 127) / 128), 128, 0, s->st>>>(a);
        k4_flux<2><<<unsigned((fz + 127) / 128), 128, 0, s->st>>>(a);
        k4_update<<<unsigned((act + 255) / 256), 256, 0, s->st>>>(a);
        k4_advance<<<1, 1, 0, s->st>>>(a.ctl, a.eb);
        s->launches += 7;
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "hc_ader4_step");
}

int hc_ader4_sync(hc_ader4* s, double* t, double* dt, long* steps_done) {
    HC_CUDA(cudaSetDevice(s->device));
    StepCtl c;
    ErrBlock eb;
    HC_CUDA(cudaMemcpyAsync(&c, s->a.ctl, sizeof c, cudaMemcpyDeviceToHost, s->st));
    HC_CUDA(cudaMemcpyAsync(&eb, s->a.eb, sizeof eb, cudaMemcpyDeviceToHost, s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    if (t) *t = c.t;
    if (dt) *dt = c.dt;
    if (steps_done) *steps_done = long(c.steps);
    return report_device_errors(eb);
}

long hc_ader4_launches(hc_ader4* s) { return s ? s->launches : 0; }

int hc_ader4_stream(hc_ader4* s, void** stream) {
    if (!s || !stream) {
        set_error(HC_INVALID, "hc_ader4_stream: null argument");
        return HC_INVALID;
    }
    *stream = s->st;
    return HC_OK;
}

}  // extern "C"
