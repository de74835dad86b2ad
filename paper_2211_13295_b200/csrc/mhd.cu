// mhd.cu -- ideal MHD on the ADER path, B200 (sm_100a), FP64: cell-centred fluid variables,
// face-centred B evolved by constrained transport (CT) with edge EMFs from a
// multidimensional Riemann solver. EXTENSION: the reference is Euler-only;
// the north star (BASELINE.json configs 3 and 5) names these updates. The step keeps the
// reference's ADER structure (stepper.cpp:49-78): reconstruction (MC at O2, WENO3 plus cross
// terms at O3) -> per-zone predictor (one Picard pass at O3, predictor.cpp:26-60 with the
// MHD flux) -> face fluxes -> edge EMFs -> conservative and CT update -> CFL min.
//
// Kernels (one thread per zone / face / edge, SoA state so every warp access is coalesced):
//   k_mhd_ghosts      periodic / outflow gather for cells and faces (one pass, any order)
//   k_mhd_predict<O3> ring zones: reconstruction of the 8 variables, the 18 states the
//                     face and edge solvers read (6 face averages, 12 edge midpoints, without
//                     the temporal part), ADER predictor; writes those states and tau/2
//   k_mhd_flux<A>     HLL (Davis speeds with the fast magnetosonic speed) or HLLD (Miyoshi &
//                     Kusano 2005; hc_mhd_params.face_solver) on the A faces; the normal
//                     field is the mean of the two reconstructed values
//   k_mhd_emf<C>      edge EMF E_C from the four zones around the edge: the two-dimensional
//                     HLL Riemann solver (UCT-HLL, Londrillo & Del Zanna 2004; the HLL limit
//                     of Balsara's MHLLE 2010): HLL-weighted corner EMFs plus the upwind
//                     jumps of the transverse fields in both directions
//   k_mhd_update      U -= dt div F (corrector.cpp:72-125 association), B_face -= dt curl E;
//                     div B is preserved to round-off (each edge EMF enters the four faces
//                     around it with opposite signs)
//   k_mhd_dt          CFL estimate, exact min through the bit pattern (as the Euler path)
//   k_mhd_advance     the dt -> dt_next hand-off and t_final clip (harness.cpp:155-170)
// Compiled with --fmad=false: the numpy restatement (oracle/mhd_oracle.py) uses the same
// expression shapes, so the two agree to the last bit on the same inputs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "../../include/hydro_mhd.h"
#include "common.cuh"
#include "ct_common.cuh"
#include "fused_types.cuh"
#include "graph_step.cuh"

namespace hc {
namespace mhd {

constexpr int NM = 8;  // rho, mx, my, mz, E, Bx, By, Bz

using ct::Box;
using ct::at;
using ct::map_c;
using ct::stride;

struct MArgs {
    double* s;      // state [8][N]
    double* states; // [18][8][N] spatial part of the predictor's states (see NST below)
    double* ht;     // [8][N] tau/2 of every ring zone (states at half time = states + ht)
    double* flux;   // [3][5][N] fluid fluxes, face f of axis A stored at the zone it is the low face of
    double* bcell;  // [3][N] cell-centred B of the current state (k_mhd_cellb)
    double* emf;    // [3][N] edge EMFs: E_x(i, j-1/2, k-1/2), E_y(i-1/2, j, k-1/2), E_z(i-1/2, j-1/2, k)
    Box b;
    double d[3];    // dx, dy, dz
    double id[3];   // 1/dx, 1/dy, 1/dz
    double gamma;
    Limiter lim;
    int bc[3];
    StepCtl* ctl;
    ErrBlock* eb;
    unsigned long long* floored;  // zones the pressure floor touched (k_mhd_dt)
    // active z range [zlo, zhi) whose update the front kernels (cell B, predictor, faces,
    // edges) prepare: the whole slab, or its interior / boundary parts when a z-slab driver
    // overlaps the halo exchange (hc_mhd_compute_range)
    int zlo, zhi;
};

// --------------------------------------------------------------------------- physics

struct MPrim {
    double rho, u[3], p, b2, inv_rho;
};

// conserved -> primitive; p = (gamma-1)(E - rho v^2/2 - B^2/2). FAST = 1: the branch-free
// bit-exact division of pointwise.cuh (flags instead of branches; callers re-run in careful
// mode when f.redo()), FAST = 0: IEEE division and first-fault capture.
template <int FAST = 0>
__device__ __forceinline__ MPrim mhd_prim(const double* c, double gamma, Fault& f) {
    MPrim q;
    q.rho = c[0];
    if (FAST) f.bad |= not_pos_fast(c[0]);
    else if (!(c[0] > 0.0)) f.set(1, c[0]);
    q.inv_rho = ddiv<FAST>(1.0, c[0], f);
    q.u[0] = c[1] * q.inv_rho;
    q.u[1] = c[2] * q.inv_rho;
    q.u[2] = c[3] * q.inv_rho;
    q.b2 = c[5] * c[5] + c[6] * c[6] + c[7] * c[7];
    q.p = (gamma - 1.0) *
          (c[4] - 0.5 * (c[1] * q.u[0] + c[2] * q.u[1] + c[3] * q.u[2]) - 0.5 * q.b2);
    if (FAST) f.bad |= not_pos_fast(q.p);
    else if (!(q.p > 0.0)) f.set(2, q.p);
    return q;
}

// fast magnetosonic speed along axis A:
// c_f^2 = ((a^2 + b^2) + sqrt((a^2 + b^2)^2 - 4 a^2 b_A^2)) / 2, a^2 = gamma p/rho, b = B/sqrt(rho)
template <int A>
__device__ __forceinline__ double fast_speed(const double* c, const MPrim& q, double gamma) {
    double a2 = gamma * q.p * q.inv_rho;
    double b2 = q.b2 * q.inv_rho;
    double bn2 = c[5 + A] * c[5 + A] * q.inv_rho;
    double s = a2 + b2;
    double disc = s * s - 4.0 * a2 * bn2;
    disc = disc > 0.0 ? disc : 0.0;
    return sqrt(0.5 * (s + sqrt(disc)));
}

// ideal-MHD flux along axis A (8 components; the normal-field component is exactly 0)
template <int A>
__device__ __forceinline__ void mhd_flux(const double* c, const MPrim& q, double* f) {
    const double un = q.u[A];
    const double bn = c[5 + A];
    const double vb = q.u[0] * c[5] + q.u[1] * c[6] + q.u[2] * c[7];
    const double pt = q.p + 0.5 * q.b2;
    f[0] = c[0] * un;
#pragma unroll
    for (int d = 0; d < 3; ++d) f[1 + d] = c[1 + d] * un - bn * c[5 + d];
    f[1 + A] += pt;
    f[4] = (c[4] + pt) * un - bn * vb;
#pragma unroll
    for (int d = 0; d < 3; ++d) f[5 + d] = c[5 + d] * un - bn * q.u[d];
}

// HLL with Davis speeds (the Euler path's riemann.hpp:55-86 structure, fast speed in place of c)
template <int A>
__device__ __forceinline__ void mhd_hll(const double* ul, const double* ur, double gamma,
                                        double* f5, Fault& flt) {
    MPrim ql = mhd_prim(ul, gamma, flt);
    MPrim qr = mhd_prim(ur, gamma, flt);
    const double cl = fast_speed<A>(ul, ql, gamma);
    const double cr = fast_speed<A>(ur, qr, gamma);
    const double sl = smin(ql.u[A] - cl, qr.u[A] - cr);
    const double sr = smax(ql.u[A] + cl, qr.u[A] + cr);
    double fl[NM], fr[NM];
    mhd_flux<A>(ul, ql, fl);
    mhd_flux<A>(ur, qr, fr);
    if (sl >= 0.0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) f5[q] = fl[q];
    } else if (sr <= 0.0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) f5[q] = fr[q];
    } else {
        const double inv = 1.0 / (sr - sl);
#pragma unroll
        for (int q = 0; q < 5; ++q)
            f5[q] = (sr * fl[q] - sl * fr[q] + sl * sr * (ur[q] - ul[q])) * inv;
    }
}

// HLLD (Miyoshi & Kusano 2005, J. Comput. Phys. 208:315): five waves -- the fast pair
// S_L, S_R (the HLL bounds above, Davis-Einfeldt form min/max(u) -/+ max(c_f)), the Alfven
// pair S*_L = S_M - |B_n|/sqrt(rho*_L), S*_R = S_M + |B_n|/sqrt(rho*_R) and the entropy wave
// S_M -- with the total pressure and the normal velocity constant across the Riemann fan.
// Resolves isolated contacts, tangential and rotational discontinuities exactly (HLL
// smears them). Fluid components only (the CT edges carry the field); the caller has made
// the normal field single-valued. Degenerate cases as in Miyoshi & Kusano section 4
// (S_M -> S_L,R with B_n^2 -> rho (S - u)^2: the tangential fields/velocities pass through
// unchanged; B_n -> 0: the double-star states collapse onto the star states).
struct HlldSide {
    double rho, v[3], b[3], e;  // star state (v[A] = S_M, b[A] = B_n)
};

template <int A>
__device__ __forceinline__ void hlld_star(const double* u, const MPrim& q, double s, double d,
                                          double sm, double pts, double pt, double bn,
                                          HlldSide& o) {
    constexpr int T1 = (A + 1) % 3, T2 = (A + 2) % 3;
    o.rho = d / (s - sm);  // d = rho (S - u)
    const double den = d * (s - sm) - bn * bn;
    o.v[A] = sm;
    o.b[A] = bn;
    if (fabs(den) < 1e-8 * pts) {
        o.v[T1] = q.u[T1];
        o.v[T2] = q.u[T2];
        o.b[T1] = u[5 + T1];
        o.b[T2] = u[5 + T2];
    } else {
        const double iden = 1.0 / den;
        const double fv = bn * (sm - q.u[A]) * iden;
        const double fb = (d * (s - q.u[A]) - bn * bn) * iden;
        o.v[T1] = q.u[T1] - u[5 + T1] * fv;
        o.v[T2] = q.u[T2] - u[5 + T2] * fv;
        o.b[T1] = u[5 + T1] * fb;
        o.b[T2] = u[5 + T2] * fb;
    }
    const double vb = q.u[0] * u[5] + q.u[1] * u[6] + q.u[2] * u[7];
    const double vbs = o.v[0] * o.b[0] + o.v[1] * o.b[1] + o.v[2] * o.b[2];
    o.e = ((s - q.u[A]) * u[4] - pt * q.u[A] + pts * sm + bn * (vb - vbs)) / (s - sm);
}

template <int A>
__device__ __forceinline__ void mhd_hlld(const double* ul, const double* ur, double gamma,
                                         double* f5, Fault& flt) {
    constexpr int T1 = (A + 1) % 3, T2 = (A + 2) % 3;
    MPrim ql = mhd_prim(ul, gamma, flt);
    MPrim qr = mhd_prim(ur, gamma, flt);
    const double bn = ul[5 + A];
    const double cl = fast_speed<A>(ul, ql, gamma);
    const double cr = fast_speed<A>(ur, qr, gamma);
    const double cm = smax(cl, cr);
    const double sl = smin(ql.u[A], qr.u[A]) - cm;
    const double sr = smax(ql.u[A], qr.u[A]) + cm;
    double fl[NM], fr[NM];
    mhd_flux<A>(ul, ql, fl);
    mhd_flux<A>(ur, qr, fr);
    if (sl >= 0.0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) f5[q] = fl[q];
        return;
    }
    if (sr <= 0.0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) f5[q] = fr[q];
        return;
    }
    const double ptl = ql.p + 0.5 * ql.b2, ptr = qr.p + 0.5 * qr.b2;
    const double dl = (sl - ql.u[A]) * ul[0], dr = (sr - qr.u[A]) * ur[0];
    const double idn = 1.0 / (dr - dl);
    const double sm = (dr * qr.u[A] - dl * ql.u[A] - ptr + ptl) * idn;
    const double pts = (dr * ptl - dl * ptr + dl * dr * (qr.u[A] - ql.u[A])) * idn;
    HlldSide L, R;
    hlld_star<A>(ul, ql, sl, dl, sm, pts, ptl, bn, L);
    hlld_star<A>(ur, qr, sr, dr, sm, pts, ptr, bn, R);
    const double rl = sqrt(L.rho), rr = sqrt(R.rho);
    const double sal = sm - fabs(bn) / rl, sar = sm + fabs(bn) / rr;
    const bool left = sm >= 0.0;
    const HlldSide& S = left ? L : R;
    const double* u = left ? ul : ur;
    const double* f = left ? fl : fr;
    const double s = left ? sl : sr;
    // star flux F* = F + S (U* - U)
    double fs[5];
    fs[0] = f[0] + s * (S.rho - u[0]);
#pragma unroll
    for (int d = 0; d < 3; ++d) fs[1 + d] = f[1 + d] + s * (S.rho * S.v[d] - u[1 + d]);
    fs[4] = f[4] + s * (S.e - u[4]);
    if ((left && sal <= 0.0) || (!left && sar >= 0.0)) {
        // double-star region: F** = F* + S*_side (U** - U*)
        double u2[3], e2;
        if (0.5 * bn * bn < 1e-8 * pts) {
            u2[0] = S.v[0];
            u2[1] = S.v[1];
            u2[2] = S.v[2];
            e2 = S.e;
        } else {
            const double sg = bn > 0.0 ? 1.0 : -1.0;
            const double inv = 1.0 / (rl + rr);
            double b2[3];
            u2[A] = sm;
            b2[A] = bn;
            u2[T1] = (rl * L.v[T1] + rr * R.v[T1] + (R.b[T1] - L.b[T1]) * sg) * inv;
            u2[T2] = (rl * L.v[T2] + rr * R.v[T2] + (R.b[T2] - L.b[T2]) * sg) * inv;
            b2[T1] = (rl * R.b[T1] + rr * L.b[T1] + rl * rr * (R.v[T1] - L.v[T1]) * sg) * inv;
            b2[T2] = (rl * R.b[T2] + rr * L.b[T2] + rl * rr * (R.v[T2] - L.v[T2]) * sg) * inv;
            const double vb2 = u2[0] * b2[0] + u2[1] * b2[1] + u2[2] * b2[2];
            const double vbs = S.v[0] * S.b[0] + S.v[1] * S.b[1] + S.v[2] * S.b[2];
            e2 = left ? S.e - rl * (vbs - vb2) * sg : S.e + rr * (vbs - vb2) * sg;
        }
        const double sa = left ? sal : sar;
        // rho** = rho*: the mass flux is the star one
#pragma unroll
        for (int d = 0; d < 3; ++d) fs[1 + d] = fs[1 + d] + sa * (S.rho * u2[d] - S.rho * S.v[d]);
        fs[4] = fs[4] + sa * (e2 - S.e);
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) f5[q] = fs[q];
}

// the face solver of the step (hc_mhd_params.face_solver)
template <int A, int S>
__device__ __forceinline__ void mhd_face(const double* ul, const double* ur, double gamma,
                                         double* f5, Fault& flt) {
    if (S == HC_MHD_HLLD) mhd_hlld<A>(ul, ur, gamma, f5, flt);
    else mhd_hll<A>(ul, ur, gamma, f5, flt);
}

// the six face states of a zone, (+x,-x,+y,-y,+z,-z) x 8 variables, in shared memory (one
// column per thread: [s][q][thread], conflict-free) instead of a local-memory array
struct FaceSmem {
    double* p;
    int t;
    __device__ __forceinline__ double& operator()(int s, int q) const {
        return p[(s * NM + q) * 128 + t];
    }
};

// predictor.cpp:12-22 flux_divergence with the MHD flux; optional shift h added to every face
template <bool SHIFT, int FAST>
__device__ __forceinline__ void mhd_divergence(const FaceSmem& face, const double* h,
                                               const double* id, double gamma, double* div,
                                               Fault& flt) {
#pragma unroll 1
    for (int A = 0; A < 3; ++A) {  // (not unrolled: three copies of the flux cost registers)
        double a[NM], b[NM], fa[NM], fb[NM];
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            a[q] = SHIFT ? face(2 * A, q) + h[q] : face(2 * A, q);
            b[q] = SHIFT ? face(2 * A + 1, q) + h[q] : face(2 * A + 1, q);
        }
        MPrim qa = mhd_prim<FAST>(a, gamma, flt), qb = mhd_prim<FAST>(b, gamma, flt);
        if (A == 0) {
            mhd_flux<0>(a, qa, fa);
            mhd_flux<0>(b, qb, fb);
        } else if (A == 1) {
            mhd_flux<1>(a, qa, fa);
            mhd_flux<1>(b, qb, fb);
        } else {
            mhd_flux<2>(a, qa, fa);
            mhd_flux<2>(b, qb, fb);
        }
#pragma unroll
        for (int q = 0; q < NM; ++q)
            div[q] = A == 0 ? (fa[q] - fb[q]) * id[0] : div[q] + (fa[q] - fb[q]) * id[A];
    }
}

// ------------------------------------------------------------------------------ kernels

// Ghost gather. Active ranges: cells [gh, gh+n) per axis; the normal axis of a face field
// [gh, gh+n] at outflow (both boundary faces are interior unknowns) and [gh, gh+n) when
// periodic (face gh+n IS face gh). Every ghost copies its (composed) active image.
__global__ void k_mhd_ghosts(MArgs a) {
    if (a.ctl && a.ctl->done) return;
    const Box& b = a.b;
    int i, j, k;  // the ghost shell only
    if (!shell_zone(b, blockIdx.x * size_t(blockDim.x) + threadIdx.x, i, j, k)) return;
    const size_t r = at(b, k, j, i);
    const int c[3] = {i, j, k};
#pragma unroll 1
    for (int q = 0; q < NM; ++q) {
        int src[3];
        bool ghost = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            int hi = b.gh + b.n[d];
            if (q >= 5 && q - 5 == d && a.bc[d] == HC_OUTFLOW) hi += 1;
            src[d] = a.bc[d] < 0 ? c[d] : map_c(c[d], b.gh, hi, a.bc[d]);  // <0: caller fills
            ghost |= src[d] != c[d];
        }
        if (ghost) a.s[q * b.N + r] = a.s[q * b.N + at(b, src[2], src[1], src[0])];
    }
}

// cell-centred variable q at storage offset o. B: the mean of the face pair at order 2; at
// order 3 the fourth-order cell average 1/2 (b[-1/2] + b[+1/2]) - 1/24 (b[+3/2] - b[+1/2] -
// b[-1/2] + b[-3/2]) (the trapezoid's h^2/8 f'' error reduced to the average's h^2/24 f'';
// with the plain mean the face fields converge at second order only)
template <bool O3>
__device__ __forceinline__ double cellvar(const MArgs& a, int q, size_t o) {
    const double* s = a.s + size_t(q) * a.b.N;
    if (q < 5) return s[o];
    return ct::face_avg<O3>(s, o, stride(a.b, q - 5));
}

// cell-centred B of every zone whose face stencil lies in the box, once per step (the
// predictor's stencils then read it like the fluid variables)
template <bool O3>
__global__ void k_mhd_cellb(MArgs a) {
    if (a.ctl && a.ctl->done) return;
    const Box& b = a.b;
    // zones the predictor of [zlo - 1, zhi] reads: its stencil reach (2 at O3, 1 at O2) + 1
    const int k0 = b.gh + a.zlo - (O3 ? 3 : 2);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= size_t(b.P) * b.Q * (a.zhi - a.zlo + (O3 ? 6 : 4))) return;
    const int i = int(r % b.P), j = int((r / b.P) % b.Q), k = k0 + int(r / (size_t(b.P) * b.Q));
    r = at(b, k, j, i);
    const int lo = O3 ? 1 : 0, hi = O3 ? 2 : 1;  // faces c-1 .. c+2 (O3) / c .. c+1
    if (i < lo || j < lo || k < lo || i + hi >= b.P || j + hi >= b.Q || k + hi >= b.R) return;
#pragma unroll
    for (int d = 0; d < 3; ++d) a.bcell[size_t(d) * b.N + r] = cellvar<O3>(a, 5 + d, r);
}

// the 8 cell-centred variables as the predictor reads them
__device__ __forceinline__ double wvar(const MArgs& a, int q, size_t o) {
    return q < 5 ? __ldg(a.s + size_t(q) * a.b.N + o) : __ldg(a.bcell + size_t(q - 5) * a.b.N + o);
}

// States a zone hands to the face and edge solvers, evaluated from its reconstruction (u0,
// slopes, quadratic and cross modes) at the points the solvers need, WITHOUT the temporal
// part: the half-time state is states[s] + ht (tau/2 of the zone), added by the consumer.
//   s = 2A (+A face average), 2A+1 (-A face average)            for A = 0, 1, 2
//   s = 6 + 4C + 2 lb + la: the midpoint of an edge along C, in the (a, b) = (C+1, C+2)
//       plane at (xa, xb) = (la ? -1/2 : +1/2, lb ? -1/2 : +1/2) -- the corner the zone
//       presents to the edge when it is the (la, lb) zone of the four around it
// Materialising these 18 states (instead of the 10 modes) turns the face and edge kernels into
// plain loads: 16 / 32 values per face / edge instead of 48 / 192 mode loads.
constexpr int NST = 18;

// One ring zone: reconstruction of the 8 cell variables, its 18 solver states, ADER predictor,
// tau/2. FAST = 1 is the branch-free bit-exact division; the caller re-runs the zone with
// FAST = 0 when a fast-path flag is raised (identical bits either way).
template <bool O3, int FAST>
__device__ __forceinline__ void predict_zone(const MArgs& a, size_t o, const FaceSmem& face,
                                             double dt, Fault& f) {
    const Box& b = a.b;
    const size_t st[3] = {stride(b, 0), stride(b, 1), stride(b, 2)};
    const size_t N = b.N;
    double* sv = a.states;
#pragma unroll 1
    for (int q = 0; q < NM; ++q) {
        const double u0 = wvar(a, q, o);
        double lin[3], quad[3] = {0.0, 0.0, 0.0}, cross[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double up = wvar(a, q, o + st[d]), um = wvar(a, q, o - st[d]);
            if (!O3) {
                const double cf = q == 0 ? a.lim.cfac_rho : a.lim.cfac_other;
                lin[d] = mc_limiter(up - u0, u0 - um, cf);  // reconstruct.cpp:16-28
            } else {
                const double upp = wvar(a, q, o + 2 * st[d]);
                const double umm = wvar(a, q, o - 2 * st[d]);
                // doubled slopes (weno3_2x, bit-exact): consumers halve their weights
                weno3_2x<FAST>(umm, um, u0, up, upp, a.lim, lin[d], quad[d], f);
                // cross mode of the pair (d, d+1): unlimited central mixed difference
                const size_t sa = st[d], sb = st[(d + 1) % 3];
                cross[d] = 0.25 * ((wvar(a, q, o + sa + sb) - wvar(a, q, o + sa - sb)) -
                                   (wvar(a, q, o - sa + sb) - wvar(a, q, o - sa - sb)));
            }
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double fp = O3 ? extrap2<true>(u0, +1.0, lin[d], quad[d])
                                 : extrap<false>(u0, +1.0, lin[d], quad[d]);
            const double fm = O3 ? extrap2<true>(u0, -1.0, lin[d], quad[d])
                                 : extrap<false>(u0, -1.0, lin[d], quad[d]);
            face(2 * d, q) = fp;
            face(2 * d + 1, q) = fm;
            // streaming stores (evict-first): 1.2 KB of states per zone would otherwise push
            // the reconstruction stencils out of L2
            __stcs(sv + (size_t(2 * d) * NM + q) * N + o, fp);
            __stcs(sv + (size_t(2 * d + 1) * NM + q) * N + o, fm);
        }
#pragma unroll
        for (int C = 0; C < 3; ++C) {
            const int AA = (C + 1) % 3, BB = (C + 2) % 3;
#pragma unroll
            for (int lb = 0; lb < 2; ++lb)
#pragma unroll
                for (int la = 0; la < 2; ++la) {
                    const double xa = la == 0 ? 0.5 : -0.5, xb = lb == 0 ? 0.5 : -0.5;
                    const double hl = O3 ? 0.5 : 1.0;  // O3 slopes are doubled (exact halving)
                    double v = u0 + (hl * xa) * lin[AA] + (hl * xb) * lin[BB];
                    if (O3)
                        v = v + (1.0 / 12.0) * quad[AA] + (1.0 / 12.0) * quad[BB] +
                            (xa * xb) * cross[AA];
                    __stcs(sv + (size_t(6 + 4 * C + 2 * lb + la) * NM + q) * N + o, v);
                }
        }
    }
    // ADER predictor (predictor.cpp:26-60): tau = -dt div F(face states); O3: one Picard pass
    double div[NM], tau[NM];
    mhd_divergence<false, FAST>(face, nullptr, a.id, a.gamma, div, f);
#pragma unroll
    for (int q = 0; q < NM; ++q) tau[q] = -dt * div[q];
    if (O3) {
        double h[NM];
#pragma unroll
        for (int q = 0; q < NM; ++q) h[q] = 0.5 * tau[q];
        mhd_divergence<true, FAST>(face, h, a.id, a.gamma, div, f);
#pragma unroll
        for (int q = 0; q < NM; ++q) tau[q] = -dt * div[q];
    }
#pragma unroll
    for (int q = 0; q < NM; ++q) __stcs(a.ht + size_t(q) * N + o, 0.5 * tau[q]);
}

template <bool O3>
__device__ __noinline__ Fault predict_zone_careful(const MArgs& a, size_t o, FaceSmem face,
                                                   double dt) {
    Fault f;
    f.clear();
    predict_zone<O3, 0>(a, o, face, dt, f);
    return f;
}

template <bool O3>
__global__ void __launch_bounds__(128, 4) k_mhd_predict(MArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    const int rx = b.n[0] + 2, ry = b.n[1] + 2;
    const size_t cnt = size_t(rx) * ry * (a.zhi - a.zlo + 2);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    // ring zone (active x/y -1..n, z zlo-1..zhi) -> storage
    const int i = int(r % rx) - 1 + b.gh, j = int((r / rx) % ry) - 1 + b.gh,
              k = int(r / (size_t(rx) * ry)) + a.zlo - 1 + b.gh;
    const size_t o = at(b, k, j, i);
    const double dt = a.ctl->dt;
    __shared__ double sface[6 * NM * 128];
    const FaceSmem face{sface, int(threadIdx.x)};
    Fault f;
    f.clear();
    predict_zone<O3, 1>(a, o, face, dt, f);
    if (f.redo()) {
        Fault c = predict_zone_careful<O3>(a, o, face, dt);
        // an unphysical reconstructed state in the predictor: this zone goes first order in
        // time (tau = 0); its solver states are checked again by their consumers, which fall
        // back to the cell average (positivity fallback; only unphysical averages are errors)
        if (c.code)
#pragma unroll
            for (int q = 0; q < NM; ++q) a.ht[size_t(q) * b.N + o] = 0.0;
    }
}

// half-time state s of the zone at o: spatial part + tau/2
__device__ __forceinline__ void half_state(const MArgs& a, size_t o, int s, double* u) {
    const size_t N = a.b.N;
#pragma unroll
    for (int q = 0; q < NM; ++q)
        u[q] = __ldg(a.states + (size_t(s) * NM + q) * N + o) + __ldg(a.ht + size_t(q) * N + o);
}

// Positivity fallback: a half-time state with rho <= 0 or p <= 0 is replaced by the zone's
// cell average (fluid variables, B as the mean of the zone's face pair -- the state the
// pressure floor of k_mhd_dt guarantees); when even that is unphysical the caller's solver
// records the fault.
__device__ __forceinline__ void positive_or_average(const MArgs& a, size_t o, double gamma,
                                                    double* u) {
    Fault t;
    t.clear();
    (void)mhd_prim(u, gamma, t);
    if (!t.code) return;
#pragma unroll
    for (int q = 0; q < NM; ++q) u[q] = cellvar<false>(a, q, o);  // (mean B: see k_mhd_dt)
}

template <bool O3, int A, int S>
__global__ void __launch_bounds__(128) k_mhd_flux(MArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    constexpr int B1 = (A + 1) % 3, B2 = (A + 2) % 3;
    // x fastest for every axis (coalesced): extents n_d, +1 along A (faces 0..n_A)
    const int ex = b.n[0] + (A == 0), ey = b.n[1] + (A == 1), ez = a.zhi - a.zlo + (A == 2);
    const size_t cnt = size_t(ex) * ey * ez;
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    int c[3];
    c[0] = int(r % ex);
    c[1] = int((r / ex) % ey);
    c[2] = a.zlo + int(r / (size_t(ex) * ey));
    const size_t o = at(b, c[2] + b.gh, c[1] + b.gh, c[0] + b.gh);  // zone right of the face
    const size_t ol = o - stride(b, A);
    double ul[NM], ur[NM], f5[5];
    half_state(a, ol, 2 * A, ul);      // +A face of the left zone
    half_state(a, o, 2 * A + 1, ur);   // -A face of the right zone
    positive_or_average(a, ol, a.gamma, ul);
    positive_or_average(a, o, a.gamma, ur);
    // single-valued normal field; the energies absorb the change of B_n^2/2 so the states
    // keep their pressures (a positive state stays positive)
    const double bn = 0.5 * (ul[5 + A] + ur[5 + A]);
    ul[4] = ul[4] + 0.5 * (bn * bn - ul[5 + A] * ul[5 + A]);
    ur[4] = ur[4] + 0.5 * (bn * bn - ur[5 + A] * ur[5 + A]);
    ul[5 + A] = bn;
    ur[5 + A] = bn;
    Fault f;
    f.clear();
    mhd_face<A, S>(ul, ur, a.gamma, f5, f);
    if (f.code) record_fault(a.eb, ST_FLUX, f, c[A], c[B1], c[B2], A);
#pragma unroll
    for (int q = 0; q < 5; ++q) a.flux[(size_t(A) * 5 + q) * b.N + o] = f5[q];
}

// Edge EMF along axis C from the four zones around the edge (axes a = C+1, b = C+2):
//   E_C = sum_{la,lb} w_a(la) w_b(lb) E_C(corner of zone (la,lb))
//         + alpha_a+ alpha_a- / (alpha_a+ + alpha_a-) (B_b[a+] - B_b[a-])
//         - alpha_b+ alpha_b- / (alpha_b+ + alpha_b-) (B_a[b+] - B_a[b-])
// w(low) = alpha+/(alpha+ + alpha-), w(high) = alpha-/(alpha+ + alpha-); alpha+ = max(0, max
// over the corners of v + c_f), alpha- = max(0, max of c_f - v); B_b[a-] = mean of the two
// low-a corner values (and so on); E_C = -(v x B)_C = v_b B_a - v_a B_b.
template <bool O3, int C>
__global__ void __launch_bounds__(128, 5) k_mhd_emf(MArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    constexpr int AA = (C + 1) % 3, BB = (C + 2) % 3;
    // x fastest (coalesced): extents n_d, +1 across the edge (a and b run 0..n)
    const int ex = b.n[0] + (C != 0), ey = b.n[1] + (C != 1), ez = a.zhi - a.zlo + (C != 2);
    const size_t cnt = size_t(ex) * ey * ez;
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    int c[3];
    c[0] = int(r % ex);
    c[1] = int((r / ex) % ey);
    c[2] = a.zlo + int(r / (size_t(ex) * ey));
    const size_t o = at(b, c[2] + b.gh, c[1] + b.gh, c[0] + b.gh);
    const size_t sa = stride(b, AA), sb = stride(b, BB);
    const size_t N = b.N;
    double ec[2][2], ba[2][2], bb[2][2];
    double apa = 0.0, ama = 0.0, apb = 0.0, amb = 0.0;
    Fault f;
    f.clear();
#pragma unroll
    for (int lb = 0; lb < 2; ++lb)
#pragma unroll
        for (int la = 0; la < 2; ++la) {
            // zone (la - 1, lb - 1) relative to the edge's high zone; corner at (xa, xb)
            const size_t z = o - (la == 0 ? sa : 0) - (lb == 0 ? sb : 0);
            double u[NM];
            half_state(a, z, 6 + 4 * C + 2 * lb + la, u);
            // positivity fallback with the primitive state reused (same bits as a second
            // mhd_prim of the kept state)
            Fault t;
            t.clear();
            MPrim p = mhd_prim(u, a.gamma, t);
            if (t.code) {
#pragma unroll
                for (int q = 0; q < NM; ++q) u[q] = cellvar<false>(a, q, z);
                p = mhd_prim(u, a.gamma, f);
            }
            ec[la][lb] = p.u[BB] * u[5 + AA] - p.u[AA] * u[5 + BB];
            ba[la][lb] = u[5 + AA];
            bb[la][lb] = u[5 + BB];
            const double cfa = fast_speed<AA>(u, p, a.gamma);
            const double cfb = fast_speed<BB>(u, p, a.gamma);
            apa = smax(apa, p.u[AA] + cfa);
            ama = smax(ama, cfa - p.u[AA]);
            apb = smax(apb, p.u[BB] + cfb);
            amb = smax(amb, cfb - p.u[BB]);
        }
    if (f.code) record_fault(a.eb, ST_FLUX, f, c[0], c[1], c[2], 3 + C);
    const double ia = 1.0 / (apa + ama), ib = 1.0 / (apb + amb);
    const double wa[2] = {apa * ia, ama * ia}, wb[2] = {apb * ib, amb * ib};
    const double e = wa[0] * wb[0] * ec[0][0] + wa[1] * wb[0] * ec[1][0] +
                     wa[0] * wb[1] * ec[0][1] + wa[1] * wb[1] * ec[1][1];
    const double jb = 0.5 * (bb[1][0] + bb[1][1]) - 0.5 * (bb[0][0] + bb[0][1]);  // B_b across a
    const double ja = 0.5 * (ba[0][1] + ba[1][1]) - 0.5 * (ba[0][0] + ba[1][0]);  // B_a across b
    a.emf[size_t(C) * N + o] = e + apa * ama * ia * jb - apb * amb * ib * ja;
}

// Conservative update of the cells (corrector.cpp:72-125 association) and CT update of the
// faces: dB_x/dt = -(dE_z/dy - dE_y/dz), dB_y/dt = -(dE_x/dz - dE_z/dx),
// dB_z/dt = -(dE_y/dx - dE_x/dy).
__global__ void k_mhd_update(MArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    const int px = b.n[0] + 1, py = b.n[1] + 1;
    const size_t cnt = size_t(px) * py * (b.n[2] + 1);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= cnt) return;
    const int i = int(r % px), j = int((r / px) % py), k = int(r / (size_t(px) * py));
    const bool ci = i < b.n[0], cj = j < b.n[1], ck = k < b.n[2];
    const size_t o = at(b, k + b.gh, j + b.gh, i + b.gh);
    const size_t N = b.N, sy = b.P, sz = size_t(b.P) * b.Q;
    const double dt = a.ctl->dt;
    const double cx = dt / a.d[0], cy = dt / a.d[1], cz = dt / a.d[2];  // corrector.cpp:75
    const double* F = a.flux;
    const double* ex = a.emf;
    const double* ey = a.emf + N;
    const double* ez = a.emf + 2 * N;
    if (ci && cj && ck) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const double* fx = F + (size_t(0) * 5 + q) * N;
            const double* fy = F + (size_t(1) * 5 + q) * N;
            const double* fz = F + (size_t(2) * 5 + q) * N;
            const double rr = -cx * (fx[o + 1] - fx[o]) - cy * (fy[o + sy] - fy[o]) -
                              cz * (fz[o + sz] - fz[o]);
            a.s[q * N + o] = a.s[q * N + o] + rr;
        }
    }
    if (cj && ck)
        a.s[5 * N + o] = a.s[5 * N + o] - (cy * (ez[o + sy] - ez[o]) - cz * (ey[o + sz] - ey[o]));
    if (ci && ck)
        a.s[6 * N + o] = a.s[6 * N + o] - (cz * (ex[o + sz] - ex[o]) - cx * (ez[o + 1] - ez[o]));
    if (ci && cj)
        a.s[7 * N + o] = a.s[7 * N + o] - (cx * (ey[o + 1] - ey[o]) - cy * (ex[o + sy] - ex[o]));
}

// CFL estimate of a zone (eval_tstep_ptwise shape with the fast speed), exact min
// pressure floor applied after every update (robustness of the extension, not part of any
// reference scheme): zones whose pressure fell to <= P_FLOOR get their energy raised to
// p = P_FLOOR, and are counted (hc_mhd_floored)
constexpr double P_FLOOR = 1.0e-10;

template <bool O3>
__device__ __forceinline__ double zone_dt(const MArgs& a, size_t o, double cfl, Fault& f,
                                          bool floor) {
    // the zone's own two faces only (mean): the estimate must not read ghost faces, which
    // are stale after the update, so it is identical under any domain decomposition
    double u[NM];
#pragma unroll
    for (int q = 0; q < NM; ++q) u[q] = cellvar<false>(a, q, o);
    if (floor && u[0] > 0.0) {
        Fault t;
        t.clear();
        MPrim q0 = mhd_prim(u, a.gamma, t);
        if (!(q0.p > P_FLOOR)) {
            u[4] = P_FLOOR / (a.gamma - 1.0) +
                   0.5 * (u[1] * q0.u[0] + u[2] * q0.u[1] + u[3] * q0.u[2]) + 0.5 * q0.b2;
            a.s[size_t(4) * a.b.N + o] = u[4];
            atomicAdd(a.floored, 1ull);
        }
    }
    MPrim p = mhd_prim(u, a.gamma, f);
    const double sx = fabs(p.u[0]) + fast_speed<0>(u, p, a.gamma);
    const double sy = fabs(p.u[1]) + fast_speed<1>(u, p, a.gamma);
    const double sz = fabs(p.u[2]) + fast_speed<2>(u, p, a.gamma);
    return cfl / (sx / a.d[0] + sy / a.d[1] + sz / a.d[2]);
}

template <bool O3>
__global__ void k_mhd_dt(MArgs a, double cfl, double* out, int stage) {
    if (a.ctl && a.ctl->done && stage == ST_UPDATE) return;
    const Box& b = a.b;
    const size_t cnt = size_t(b.n[0]) * b.n[1] * b.n[2];
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    double d = 1.0e32;
    if (r < cnt) {
        const int i = int(r % b.n[0]), j = int((r / b.n[0]) % b.n[1]),
                  k = int(r / (size_t(b.n[0]) * b.n[1]));
        Fault f;
        f.clear();
        const double v =
            zone_dt<O3>(a, at(b, k + b.gh, j + b.gh, i + b.gh), cfl, f, stage == ST_UPDATE);
        if (f.code) record_fault(a.eb, stage, f, i, j, k, 0);
        else d = v;
    }
    d = warp_min(d);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 1.0e32;
        v = warp_min(v);
        if (threadIdx.x == 0) atomic_min_pos(out, v);
    }
}

// ============================================================ order 4 (space-time ADER)
// The O2/O3 kernels keep the reference's ADER structure (face state + the zone's tau/2), second
// order in time. Order 4 (smooth flows; no positivity fallback):
//   k_mhd4_predict  one CTA per ring zone, one thread per spatial node (4 x 4 x 4 Gauss-
//                   Legendre points) holding its 4 Gauss times: the degree-3 polynomial of the 8 cell
//                   variables (fluid averages, fourth-order cell B from k_mhd_cellb; WENO-AO pure
//                   terms, central mixed terms, as ader4.cu), four Picard iterations of the local
//                   space-time predictor with the MHD flux; outputs the states at the 2 x 2 Gauss
//                   points of the 6 faces and at the 2 Gauss points along the 12 zone edges, each
//                   at the 2 Gauss times ([96][8][N] in `states`: faces 0..47, edges 48..95)
//   k_mhd4_flux<A>  HLL at the 2 x 2 x 2 space-time Gauss points of each face (single-valued
//                   normal B with the energy shift of k_mhd_flux), averaged
//   k_mhd4_emf<C>   the 2D HLL EMF of k_mhd_emf at the 2 x 2 points along the edge and in time,
//                   averaged: the edge- and time-averaged EMF of constrained transport
// then k_mhd_update / k_mhd_dt as at O2/O3 (div B stays at round-off).
struct MhdBasis {
    double xi[4], D[4][4], IT[4][4], LF[2][4], LG[2][4], LT[2][4];
};
__constant__ MhdBasis c_mb;
constexpr int M4_NT = 256, M4_OUT = 96, M4_NCOEF = 23;

__device__ __forceinline__ void psi4m(double s, double* p) {
    const double s2 = s * s;
    p[0] = s;
    p[1] = s2 - 1.0 / 12.0;
    p[2] = s * (s2 - 3.0 / 20.0);
    p[3] = s2 * s2 - (3.0 / 14.0) * s2 + 3.0 / 560.0;
}

// One CTA of 64 threads per ring zone; thread t owns spatial node t and its 4 time nodes in
// registers (the time integral and the output time contraction are register work); the
// fluxes go through shared memory two time nodes at a time, SoA with the node slot
// n ^ 5 * bit4(n), so the x / y / z neighbour reads of a warp hit distinct banks (the layout
// of ader4.cu's predictor). The 96 output points are contracted separably: one axis first
// (the face normal with the face values, or the edge direction with the Gauss values), then
// the two transverse ones.
#ifndef M4_MINB
#define M4_MINB 6
#endif
constexpr int M4_NS = 64;                        // spatial nodes = threads per CTA
constexpr int M4_F = 2 * 3 * NM * M4_NS;         // flux staging (2 time nodes)
constexpr int M4_T = NM * 2 * M4_NS;             // predictor at the 2 Gauss times
constexpr int M4_SQ = 384 + 24;                  // one-axis contractions per variable (skewed)
constexpr int M4_U = (M4_F > M4_T + NM * M4_SQ) ? M4_F : M4_T + NM * M4_SQ;
__global__ void __launch_bounds__(M4_NS, M4_MINB) k_mhd4_predict(MArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    __shared__ double coef[NM][M4_NCOEF];
    __shared__ double U[M4_U];
    const int rx = b.n[0] + 2, ry = b.n[1] + 2;
    const int zr = blockIdx.x;
    const int i = zr % rx - 1 + b.gh, j = (zr / rx) % ry - 1 + b.gh,
              k = zr / (rx * ry) - 1 + a.zlo + b.gh;
    const size_t o = at(b, k, j, i);
    const long long st3[3] = {(long long)stride(b, 0), (long long)stride(b, 1), (long long)stride(b, 2)};
    const size_t N = b.N;
    const int t = threadIdx.x;
    const double dt = a.ctl->dt;
    auto Wv = [&](int q, long long off) { return wvar(a, q, size_t((long long)o + off)); };
    // reconstruction: 24 WENO-AO tasks (the long ones first), then 80 mixed terms
    for (int task = t; task < 24 + NM * 10; task += M4_NS) {
        if (task < 24) {
            const int q = task / 3, ax = task % 3;
            double m[4];
            Fault f;
            f.clear();
            weno_ao<0>(Wv(q, -2 * st3[ax]), Wv(q, -st3[ax]), Wv(q, 0), Wv(q, st3[ax]),
                       Wv(q, 2 * st3[ax]), a.lim, m, f);
#pragma unroll
            for (int l = 0; l < 4; ++l) coef[q][1 + 4 * ax + l] = m[l];
            if (ax == 0) coef[q][0] = Wv(q, 0);
        } else {
            const int q = (task - 24) / 10, term = (task - 24) % 10;
            auto val = [&](int p1, int s1, int p2, int s2) {
                return Wv(q, s1 * st3[p1] + s2 * st3[p2]);
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
                                   Wv(q, aa * st3[0] + bb * st3[1] + cc * st3[2]);
                v = 0.125 * acc;
            }
            coef[q][13 + term] = v;
        }
    }
    __syncthreads();
    const int ni = t & 3, nj = (t >> 2) & 3, nk = t >> 4;
    auto sw = [](int n) { return n ^ (((n >> 4) & 1) * 5); };
    double p0[NM];
    {
        double px[4], py[4], pz[4];
        psi4m(c_mb.xi[ni], px);
        psi4m(c_mb.xi[nj], py);
        psi4m(c_mb.xi[nk], pz);
#pragma unroll
        for (int q = 0; q < NM; ++q) {
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
    double Q[4][NM];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int q = 0; q < NM; ++q) Q[m][q] = p0[q];
    double wx[4], wy[4], wz[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        wx[l] = c_mb.D[ni][l] * a.id[0];
        wy[l] = c_mb.D[nj][l] * a.id[1];
        wz[l] = c_mb.D[nk][l] * a.id[2];
    }
    // F[mm][axis][q][slot]
    auto F = [&](int mm, int ax, int q, int slot) -> double& {
        return U[((mm * 3 + ax) * NM + q) * M4_NS + slot];
    };
    const int ts = sw(t);
    Fault f;
    f.clear();
    for (int it = 0; it < 4; ++it) {
        double dv[4][NM];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int mm = 0; mm < 2; ++mm) {
                const int m = 2 * h + mm;
                const MPrim pr = mhd_prim<0>(Q[m], a.gamma, f);
                double fl[NM];
                mhd_flux<0>(Q[m], pr, fl);
#pragma unroll
                for (int q = 0; q < NM; ++q) F(mm, 0, q, ts) = fl[q];
                mhd_flux<1>(Q[m], pr, fl);
#pragma unroll
                for (int q = 0; q < NM; ++q) F(mm, 1, q, ts) = fl[q];
                mhd_flux<2>(Q[m], pr, fl);
#pragma unroll
                for (int q = 0; q < NM; ++q) F(mm, 2, q, ts) = fl[q];
            }
            __syncthreads();
#pragma unroll
            for (int mm = 0; mm < 2; ++mm) {
                const int m = 2 * h + mm;
#pragma unroll
                for (int q = 0; q < NM; ++q) dv[m][q] = 0.0;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const int tx = sw((t & ~3) | l), ty = sw((t & ~12) | (l << 2)),
                              tz = sw((t & ~48) | (l << 4));
#pragma unroll
                    for (int q = 0; q < NM; ++q)
                        dv[m][q] += wx[l] * F(mm, 0, q, tx) + wy[l] * F(mm, 1, q, ty) +
                                    wz[l] * F(mm, 2, q, tz);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int q = 0; q < NM; ++q) {
                double qn = p0[q];
#pragma unroll
                for (int l = 0; l < 4; ++l) qn -= (dt * c_mb.IT[m][l]) * dv[l][q];
                Q[m][q] = qn;
            }
    }
    if (f.code) record_fault(a.eb, ST_PREDICT, f, i - b.gh, j - b.gh, k - b.gh, 0);
    // outputs. (1) time -> the 2 Gauss times, in registers: T[q][tg][slotT(node)]
    double* T = U;
    double* S = U + M4_T;  // S[q][r + r / 16], r < 384
    auto slotT = [](int n) { return n ^ ((n >> 4) * 5); };
#pragma unroll
    for (int tg = 0; tg < 2; ++tg)
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            double v = 0.0;
#pragma unroll
            for (int m = 0; m < 4; ++m) v += c_mb.LT[tg][m] * Q[m][q];
            T[(q * 2 + tg) * M4_NS + slotT(t)] = v;
        }
    __syncthreads();
    // (2) one axis: r < 192 faces ((A * 2 + side) * 2 + tg) * 16 + b1 * 4 + b2, the normal
    //     axis A at its face (LF[side]); r >= 192 edges ((C * 2 + g) * 2 + tg) * 16 + ..., the
    //     edge axis C at Gauss point g (LG[g]); b1, b2 the nodes along the axes +1 / +2 of it
    for (int r = t; r < 384; r += M4_NS) {
        const int rr = r < 192 ? r : r - 192;
        const int ax = rr >> 6, sel = (rr >> 5) & 1, tg = (rr >> 4) & 1, b1 = (rr >> 2) & 3,
                  b2 = rr & 3;
        const double* w = r < 192 ? c_mb.LF[sel] : c_mb.LG[sel];
        double v[NM];
#pragma unroll
        for (int q = 0; q < NM; ++q) v[q] = 0.0;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            int c[3];
            c[ax] = l;
            c[(ax + 1) % 3] = b1;
            c[(ax + 2) % 3] = b2;
            const int node = (c[2] * 4 + c[1]) * 4 + c[0];
#pragma unroll
            for (int q = 0; q < NM; ++q) v[q] += w[l] * T[(q * 2 + tg) * M4_NS + slotT(node)];
        }
#pragma unroll
        for (int q = 0; q < NM; ++q) S[q * M4_SQ + r + (r >> 4)] = v[q];
    }
    __syncthreads();
    // (3) the two transverse axes: faces at the 2 x 2 Gauss points, edges at the corner
    for (int e = t; e < M4_OUT; e += M4_NS) {
        int base;
        const double *w1, *w2;
        if (e < 48) {  // ((face * 4 + g1 * 2 + g2) * 2 + tg), face = 2A + side
            const int tg = e & 1, g = (e >> 1) & 3, face = e >> 3;
            base = (face * 2 + tg) * 16;
            w1 = c_mb.LG[g >> 1];
            w2 = c_mb.LG[g & 1];
        } else {  // ((C * 4 + corner) * 2 + g) * 2 + tg, corner = la + 2 lb
            const int x = e - 48, tg = x & 1, g = (x >> 1) & 1, corner = (x >> 2) & 3, C = x >> 4;
            base = 192 + ((C * 2 + g) * 2 + tg) * 16;
            w1 = c_mb.LF[corner & 1];
            w2 = c_mb.LF[corner >> 1];
        }
        double v[NM];
#pragma unroll
        for (int q = 0; q < NM; ++q) v[q] = 0.0;
#pragma unroll
        for (int b1 = 0; b1 < 4; ++b1)
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
                const double ww = w1[b1] * w2[b2];
                const int r = base + b1 * 4 + b2;
#pragma unroll
                for (int q = 0; q < NM; ++q) v[q] += ww * S[q * M4_SQ + r + (r >> 4)];
            }
#pragma unroll
        for (int q = 0; q < NM; ++q) __stcs(a.states + (size_t(e) * NM + q) * N + o, v[q]);
    }
}

template <int A, int S>
__global__ void __launch_bounds__(128) k_mhd4_flux(MArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    constexpr int B1 = (A + 1) % 3, B2 = (A + 2) % 3;
    const int ex = b.n[0] + (A == 0), ey = b.n[1] + (A == 1), ez = a.zhi - a.zlo + (A == 2);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= size_t(ex) * ey * ez) return;
    int c[3];
    c[0] = int(r % ex);
    c[1] = int((r / ex) % ey);
    c[2] = a.zlo + int(r / (size_t(ex) * ey));
    const size_t o = at(b, c[2] + b.gh, c[1] + b.gh, c[0] + b.gh);
    const size_t ol = o - stride(b, A), N = b.N;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    Fault f;
    f.clear();
    for (int p = 0; p < 8; ++p) {  // (g1, g2, tg) of the face
        double ul[NM], ur[NM], f5[5];
        const int el = (2 * A) * 8 + p, er = (2 * A + 1) * 8 + p;
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            ul[q] = __ldg(a.states + (size_t(el) * NM + q) * N + ol);
            ur[q] = __ldg(a.states + (size_t(er) * NM + q) * N + o);
        }
        const double bn = 0.5 * (ul[5 + A] + ur[5 + A]);
        ul[4] = ul[4] + 0.5 * (bn * bn - ul[5 + A] * ul[5 + A]);
        ur[4] = ur[4] + 0.5 * (bn * bn - ur[5 + A] * ur[5 + A]);
        ul[5 + A] = bn;
        ur[5 + A] = bn;
        mhd_face<A, S>(ul, ur, a.gamma, f5, f);
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[q] += 0.125 * f5[q];
    }
    if (f.code) record_fault(a.eb, ST_FLUX, f, c[A], c[B1], c[B2], A);
#pragma unroll
    for (int q = 0; q < 5; ++q) a.flux[(size_t(A) * 5 + q) * N + o] = acc[q];
}

template <int C>
__global__ void __launch_bounds__(128) k_mhd4_emf(MArgs a) {
    if (a.ctl->done) return;
    const Box& b = a.b;
    constexpr int AA = (C + 1) % 3, BB = (C + 2) % 3;
    const int ex = b.n[0] + (C != 0), ey = b.n[1] + (C != 1), ez = a.zhi - a.zlo + (C != 2);
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= size_t(ex) * ey * ez) return;
    int c[3];
    c[0] = int(r % ex);
    c[1] = int((r / ex) % ey);
    c[2] = a.zlo + int(r / (size_t(ex) * ey));
    const size_t o = at(b, c[2] + b.gh, c[1] + b.gh, c[0] + b.gh);
    const size_t sa = stride(b, AA), sb = stride(b, BB), N = b.N;
    Fault f;
    f.clear();
    double E = 0.0;
    for (int p = 0; p < 4; ++p) {  // (g along C, tg)
        double ec[2][2], ba[2][2], bb[2][2];
        double apa = 0.0, ama = 0.0, apb = 0.0, amb = 0.0;
#pragma unroll
        for (int lb = 0; lb < 2; ++lb)
#pragma unroll
            for (int la = 0; la < 2; ++la) {
                const size_t z = o - (la == 0 ? sa : 0) - (lb == 0 ? sb : 0);
                const int e = 48 + (C * 4 + 2 * lb + la) * 4 + p;
                double u[NM];
#pragma unroll
                for (int q = 0; q < NM; ++q) u[q] = __ldg(a.states + (size_t(e) * NM + q) * N + z);
                const MPrim pr = mhd_prim(u, a.gamma, f);
                ec[la][lb] = pr.u[BB] * u[5 + AA] - pr.u[AA] * u[5 + BB];
                ba[la][lb] = u[5 + AA];
                bb[la][lb] = u[5 + BB];
                const double cfa = fast_speed<AA>(u, pr, a.gamma);
                const double cfb = fast_speed<BB>(u, pr, a.gamma);
                apa = smax(apa, pr.u[AA] + cfa);
                ama = smax(ama, cfa - pr.u[AA]);
                apb = smax(apb, pr.u[BB] + cfb);
                amb = smax(amb, cfb - pr.u[BB]);
            }
        const double ia = 1.0 / (apa + ama), ib = 1.0 / (apb + amb);
        const double wa[2] = {apa * ia, ama * ia}, wb[2] = {apb * ib, amb * ib};
        const double e = wa[0] * wb[0] * ec[0][0] + wa[1] * wb[0] * ec[1][0] +
                         wa[0] * wb[1] * ec[0][1] + wa[1] * wb[1] * ec[1][1];
        const double jb = 0.5 * (bb[1][0] + bb[1][1]) - 0.5 * (bb[0][0] + bb[0][1]);
        const double ja = 0.5 * (ba[0][1] + ba[1][1]) - 0.5 * (ba[0][0] + ba[1][0]);
        E += 0.25 * (e + apa * ama * ia * jb - apb * amb * ib * ja);
    }
    if (f.code) record_fault(a.eb, ST_FLUX, f, c[0], c[1], c[2], 3 + C);
    a.emf[size_t(C) * N + o] = E;
}

MhdBasis make_mhd_basis() {
    MhdBasis bs;
    const double gl[4] = {-0.8611363115940526, -0.3399810435848563, 0.3399810435848563,
                          0.8611363115940526};
    const double gw[4] = {0.3478548451374538, 0.6521451548625461, 0.6521451548625461,
                          0.3478548451374538};
    double tau[4];
    for (int l = 0; l < 4; ++l) {
        bs.xi[l] = 0.5 * gl[l];
        tau[l] = 0.5 * (gl[l] + 1.0);
    }
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
            double sum = 0.0;
            for (int g = 0; g < 4; ++g) sum += 0.5 * tau[r] * gw[g] * lag(tau, l, 0.5 * tau[r] * (gl[g] + 1.0));
            bs.IT[r][l] = sum;
        }
    for (int l = 0; l < 4; ++l) {
        bs.LF[0][l] = lag(bs.xi, l, 0.5);
        bs.LF[1][l] = lag(bs.xi, l, -0.5);
        bs.LG[0][l] = lag(bs.xi, l, -g2);
        bs.LG[1][l] = lag(bs.xi, l, g2);
        bs.LT[0][l] = lag(tau, l, 0.5 - g2);
        bs.LT[1][l] = lag(tau, l, 0.5 + g2);
    }
    return bs;
}

__global__ void k_mhd_divb(MArgs a, double* out) {
    const Box& b = a.b;
    const size_t cnt = size_t(b.n[0]) * b.n[1] * b.n[2];
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    double d = 0.0;
    if (r < cnt) {
        const int i = int(r % b.n[0]), j = int((r / b.n[0]) % b.n[1]),
                  k = int(r / (size_t(b.n[0]) * b.n[1]));
        const size_t o = at(b, k + b.gh, j + b.gh, i + b.gh), N = b.N;
        const double* s = a.s;
        const double dv = (s[5 * N + o + 1] - s[5 * N + o]) / a.d[0] +
                          (s[6 * N + o + b.P] - s[6 * N + o]) / a.d[1] +
                          (s[7 * N + o + size_t(b.P) * b.Q] - s[7 * N + o]) / a.d[2];
        d = fabs(dv) * fmin(a.d[0], fmin(a.d[1], a.d[2]));
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, s));
    if ((threadIdx.x & 31) == 0)
        atomicMax(reinterpret_cast<unsigned long long*>(out),
                  static_cast<unsigned long long>(__double_as_longlong(d)));
}

__global__ void k_mhd_advance(StepCtl* c, const ErrBlock* eb) {
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
        double rem = c->t_final - c->t;
        if (rem <= 1e-12 * c->t_final) c->done = 1;
        else if (dn >= rem) dn = rem;
    }
    c->dt = dn;
}

}  // namespace mhd
}  // namespace hc

using namespace hc;
using namespace hc::mhd;

struct hc_mhd {
    hc_geom g;
    hc_mhd_params p;
    Box b;
    double* s = nullptr;
    double* states = nullptr;
    double* ht = nullptr;
    double* flux = nullptr;
    double* emf = nullptr;
    double* bc = nullptr;
    double* scratch = nullptr;  // one double for reductions
    unsigned long long* floored = nullptr;
    StepCtl* ctl = nullptr;
    ErrBlock* eb = nullptr;
    cudaStream_t st = nullptr;
    bool own_stream = true;
    long launches = 0;
    StepGraph graph;
    double cfl = 0.4;
};

namespace {

MArgs margs(const hc_mhd* m) {
    MArgs a;
    a.s = m->s;
    a.states = m->states;
    a.ht = m->ht;
    a.flux = m->flux;
    a.emf = m->emf;
    a.bcell = m->bc;
    a.b = m->b;
    a.d[0] = m->g.dx;
    a.d[1] = m->g.dy;
    a.d[2] = m->g.dz;
    for (int d = 0; d < 3; ++d) a.id[d] = 1.0 / a.d[d];  // predictor.cpp:29
    a.gamma = m->p.gamma;
    a.lim = Limiter{m->p.lim.cfac_rho, m->p.lim.cfac_other, m->p.lim.weno_eps,
                    m->p.lim.weno_w[0], m->p.lim.weno_w[1], m->p.lim.weno_w[2]};
    for (int d = 0; d < 3; ++d) a.bc[d] = m->p.bc[d];
    a.ctl = m->ctl;
    a.eb = m->eb;
    a.floored = m->floored;
    a.zlo = 0;
    a.zhi = m->b.n[2];
    return a;
}

using ct::blocks;

int launch_ghosts(hc_mhd* m) {
    MArgs a = margs(m);
    k_mhd_ghosts<<<blocks(shell_count(m->b), 256), 256, 0, m->st>>>(a);
    m->launches += 1;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "mhd ghost launch");
}

// the front kernels of a step for the active z range [zlo, zhi): cell B, predictor, face
// fluxes and edge EMFs of every face/edge the update of those zones reads

int launch_front4(hc_mhd* m, int zlo, int zhi) {
    MArgs a = margs(m);
    a.zlo = zlo;
    a.zhi = zhi;
    const Box& b = m->b;
    const int nz = zhi - zlo;
    const size_t cb = size_t(b.P) * b.Q * (nz + 6);
    const size_t ring = size_t(b.n[0] + 2) * (b.n[1] + 2) * (nz + 2);
    k_mhd_cellb<true><<<blocks(cb, 256), 256, 0, m->st>>>(a);
    k_mhd4_predict<<<unsigned(ring), M4_NS, 0, m->st>>>(a);
    const size_t fx = size_t(b.n[0] + 1) * b.n[1] * nz;
    const size_t fy = size_t(b.n[0]) * (b.n[1] + 1) * nz;
    const size_t fz = size_t(b.n[0]) * b.n[1] * (nz + 1);
    const size_t ex = size_t(b.n[0]) * (b.n[1] + 1) * (nz + 1);
    const size_t ey = size_t(b.n[0] + 1) * b.n[1] * (nz + 1);
    const size_t ez = size_t(b.n[0] + 1) * (b.n[1] + 1) * nz;
    if (m->p.face_solver == HC_MHD_HLLD) {
        k_mhd4_flux<0, HC_MHD_HLLD><<<blocks(fx, 128), 128, 0, m->st>>>(a);
        k_mhd4_flux<1, HC_MHD_HLLD><<<blocks(fy, 128), 128, 0, m->st>>>(a);
        k_mhd4_flux<2, HC_MHD_HLLD><<<blocks(fz, 128), 128, 0, m->st>>>(a);
    } else {
        k_mhd4_flux<0, HC_MHD_HLL><<<blocks(fx, 128), 128, 0, m->st>>>(a);
        k_mhd4_flux<1, HC_MHD_HLL><<<blocks(fy, 128), 128, 0, m->st>>>(a);
        k_mhd4_flux<2, HC_MHD_HLL><<<blocks(fz, 128), 128, 0, m->st>>>(a);
    }
    k_mhd4_emf<0><<<blocks(ex, 128), 128, 0, m->st>>>(a);
    k_mhd4_emf<1><<<blocks(ey, 128), 128, 0, m->st>>>(a);
    k_mhd4_emf<2><<<blocks(ez, 128), 128, 0, m->st>>>(a);
    m->launches += 8;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "mhd order-4 step launch");
}

template <bool O3>
void launch_faces(hc_mhd* m, const MArgs& a, size_t fx, size_t fy, size_t fz) {
    if (m->p.face_solver == HC_MHD_HLLD) {
        k_mhd_flux<O3, 0, HC_MHD_HLLD><<<blocks(fx, 128), 128, 0, m->st>>>(a);
        k_mhd_flux<O3, 1, HC_MHD_HLLD><<<blocks(fy, 128), 128, 0, m->st>>>(a);
        k_mhd_flux<O3, 2, HC_MHD_HLLD><<<blocks(fz, 128), 128, 0, m->st>>>(a);
    } else {
        k_mhd_flux<O3, 0, HC_MHD_HLL><<<blocks(fx, 128), 128, 0, m->st>>>(a);
        k_mhd_flux<O3, 1, HC_MHD_HLL><<<blocks(fy, 128), 128, 0, m->st>>>(a);
        k_mhd_flux<O3, 2, HC_MHD_HLL><<<blocks(fz, 128), 128, 0, m->st>>>(a);
    }
}

int launch_front(hc_mhd* m, int zlo, int zhi) {
    if (m->p.order == 4) return launch_front4(m, zlo, zhi);
    MArgs a = margs(m);
    a.zlo = zlo;
    a.zhi = zhi;
    const Box& b = m->b;
    const bool o3 = m->p.order == 3;
    const int nz = zhi - zlo;
    const size_t cb = size_t(b.P) * b.Q * (nz + (o3 ? 6 : 4));
    const size_t ring = size_t(b.n[0] + 2) * (b.n[1] + 2) * (nz + 2);
    if (o3) k_mhd_cellb<true><<<blocks(cb, 256), 256, 0, m->st>>>(a);
    else k_mhd_cellb<false><<<blocks(cb, 256), 256, 0, m->st>>>(a);
    if (o3) k_mhd_predict<true><<<blocks(ring, 128), 128, 0, m->st>>>(a);
    else k_mhd_predict<false><<<blocks(ring, 128), 128, 0, m->st>>>(a);
    const size_t fx = size_t(b.n[0] + 1) * b.n[1] * nz;
    const size_t fy = size_t(b.n[0]) * (b.n[1] + 1) * nz;
    const size_t fz = size_t(b.n[0]) * b.n[1] * (nz + 1);
    const size_t ex = size_t(b.n[0]) * (b.n[1] + 1) * (nz + 1);
    const size_t ey = size_t(b.n[0] + 1) * b.n[1] * (nz + 1);
    const size_t ez = size_t(b.n[0] + 1) * (b.n[1] + 1) * nz;
    if (o3) {
        launch_faces<true>(m, a, fx, fy, fz);
        k_mhd_emf<true, 0><<<blocks(ex, 128), 128, 0, m->st>>>(a);
        k_mhd_emf<true, 1><<<blocks(ey, 128), 128, 0, m->st>>>(a);
        k_mhd_emf<true, 2><<<blocks(ez, 128), 128, 0, m->st>>>(a);
    } else {
        launch_faces<false>(m, a, fx, fy, fz);
        k_mhd_emf<false, 0><<<blocks(ex, 128), 128, 0, m->st>>>(a);
        k_mhd_emf<false, 1><<<blocks(ey, 128), 128, 0, m->st>>>(a);
        k_mhd_emf<false, 2><<<blocks(ez, 128), 128, 0, m->st>>>(a);
    }
    m->launches += 8;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "mhd step launch");
}

// the update of every active zone and face, then the CFL estimate of the new state
int launch_finish(hc_mhd* m) {
    MArgs a = margs(m);
    const Box& b = m->b;
    const bool o3 = m->p.order >= 3;
    const size_t up = size_t(b.n[0] + 1) * (b.n[1] + 1) * (b.n[2] + 1);
    k_mhd_update<<<blocks(up, 256), 256, 0, m->st>>>(a);
    const size_t act = size_t(b.n[0]) * b.n[1] * b.n[2];
    // CFL estimate of the updated state from each zone's own faces (ghosts are stale)
    if (o3) k_mhd_dt<true><<<blocks(act, 256), 256, 0, m->st>>>(a, m->cfl, &m->ctl->acc, ST_UPDATE);
    else k_mhd_dt<false><<<blocks(act, 256), 256, 0, m->st>>>(a, m->cfl, &m->ctl->acc, ST_UPDATE);
    m->launches += 2;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "mhd update launch");
}

int launch_compute(hc_mhd* m) {
    int rc = launch_front(m, 0, m->b.n[2]);
    return rc ? rc : launch_finish(m);
}

int launch_advance(hc_mhd* m) {
    k_mhd_advance<<<1, 1, 0, m->st>>>(m->ctl, m->eb);
    m->launches += 1;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "mhd advance launch");
}

int launch_step(hc_mhd* m) {
    int rc = launch_ghosts(m);
    if (!rc) rc = launch_compute(m);
    if (!rc) rc = launch_advance(m);
    return rc;
}

}  // namespace

extern "C" {

int hc_mhd_create(const hc_geom* g, const hc_mhd_params* p, hc_mhd** out) {
    if (!p || !out) {
        set_error(HC_INVALID, "null argument");
        return HC_INVALID;
    }
    if (p->order < 2 || p->order > 4) {
        set_error(HC_INVALID, "mhd: order must be 2, 3 or 4");
        return HC_INVALID;
    }
    if (p->face_solver != HC_MHD_HLL && p->face_solver != HC_MHD_HLLD) {
        set_error(HC_INVALID, "mhd: face_solver must be HC_MHD_HLL or HC_MHD_HLLD");
        return HC_INVALID;
    }
    int rc = validate_geom(g, p->order == 4 ? 3 : p->order);  // (order 4: the same stencils)
    if (rc) return rc;
    if (g->ghost < (p->order >= 3 ? 4 : 2)) {  // WENO radius 2 + ring + B cell average
        set_error(HC_INVALID, "mhd: orders 3 and 4 need a ghost width of at least 4");
        return HC_INVALID;
    }
    for (int d = 0; d < 3; ++d)
        if (p->bc[d] != HC_PERIODIC && p->bc[d] != HC_OUTFLOW && !(d == 2 && p->bc[d] == -1)) {
            set_error(HC_INVALID, "mhd: boundary kind must be periodic or outflow (z: or -1)");
            return HC_INVALID;
        }
    hc_mhd* m = new (std::nothrow) hc_mhd;
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
    cudaError_t e = cudaSetDevice(p->device);
    if (e == cudaSuccess) e = cudaMalloc(&m->s, sizeof(double) * NM * b.N);
    if (e == cudaSuccess)
        e = cudaMalloc(&m->states, sizeof(double) * size_t(p->order == 4 ? M4_OUT : NST) * NM * b.N);
    if (e == cudaSuccess) e = cudaMalloc(&m->ht, sizeof(double) * NM * b.N);
    if (e == cudaSuccess) e = cudaMalloc(&m->flux, sizeof(double) * 15 * b.N);
    if (e == cudaSuccess) e = cudaMalloc(&m->emf, sizeof(double) * 3 * b.N);
    if (e == cudaSuccess) e = cudaMalloc(&m->bc, sizeof(double) * 3 * b.N);
    if (e == cudaSuccess) e = cudaMalloc(&m->scratch, sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&m->floored, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(m->floored, 0, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&m->ctl, sizeof(StepCtl));
    if (e == cudaSuccess) e = cudaMalloc(&m->eb, sizeof(ErrBlock));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&m->st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemset(m->s, 0, sizeof(double) * NM * b.N);
    if (e == cudaSuccess) e = cudaMemset(m->flux, 0, sizeof(double) * 15 * b.N);
    if (e == cudaSuccess) e = cudaMemset(m->emf, 0, sizeof(double) * 3 * b.N);
    if (e == cudaSuccess) e = cudaMemset(m->eb, 0, sizeof(ErrBlock));
    if (e == cudaSuccess) {
        StepCtl c{};
        c.acc = 1.0e32;
        e = cudaMemcpy(m->ctl, &c, sizeof c, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && p->order == 4) {
        MhdBasis bs = make_mhd_basis();
        e = cudaMemcpyToSymbol(c_mb, &bs, sizeof bs);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_mhd4_predict,
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    if (e != cudaSuccess) {
        hc_mhd_destroy(m);
        return cuda_fail(e, "hc_mhd_create");
    }
    *out = m;
    return HC_OK;
}

int hc_mhd_destroy(hc_mhd* m) {
    if (!m) return HC_OK;
    cudaSetDevice(m->p.device);
    if (m->st) cudaStreamSynchronize(m->st);
    cudaFree(m->s);
    cudaFree(m->states);
    cudaFree(m->ht);
    cudaFree(m->flux);
    cudaFree(m->emf);
    cudaFree(m->bc);
    cudaFree(m->scratch);
    cudaFree(m->floored);
    cudaFree(m->ctl);
    cudaFree(m->eb);
    if (m->st && m->own_stream) cudaStreamDestroy(m->st);
    delete m;
    return HC_OK;
}

int hc_mhd_upload(hc_mhd* m, const double* host) {
    HC_CUDA(cudaSetDevice(m->p.device));
    HC_CUDA(cudaMemcpyAsync(m->s, host, sizeof(double) * NM * m->b.N, cudaMemcpyHostToDevice,
                            m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

int hc_mhd_download(hc_mhd* m, double* host) {
    HC_CUDA(cudaSetDevice(m->p.device));
    HC_CUDA(cudaMemcpyAsync(host, m->s, sizeof(double) * NM * m->b.N, cudaMemcpyDeviceToHost,
                            m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

int hc_mhd_set_time(hc_mhd* m, double t, double dt, double cfl, double t_final) {
    HC_CUDA(cudaSetDevice(m->p.device));
    StepCtl c{};
    c.dt = dt;
    c.t = t;
    c.t_final = t_final;
    c.acc = 1.0e32;
    c.dt_next = dt;
    m->cfl = cfl;
    HC_CUDA(cudaMemcpyAsync(m->ctl, &c, sizeof c, cudaMemcpyHostToDevice, m->st));
    HC_CUDA(cudaMemsetAsync(m->eb, 0, sizeof(ErrBlock), m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

int hc_mhd_step(hc_mhd* m, int n) {
    HC_CUDA(cudaSetDevice(m->p.device));
    // n > 1: one captured step replayed as a CUDA graph (graph_step.cuh)
    return replay_steps(m->graph, m->st, m->cfl, m->launches, n, [&] { return launch_step(m); });
}

int hc_mhd_sync(hc_mhd* m, double* t, double* dt, long* steps) {
    HC_CUDA(cudaSetDevice(m->p.device));
    StepCtl c;
    ErrBlock eb;
    HC_CUDA(cudaMemcpyAsync(&c, m->ctl, sizeof c, cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaMemcpyAsync(&eb, m->eb, sizeof eb, cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    if (t) *t = c.t;
    if (dt) *dt = c.dt;
    if (steps) *steps = long(c.steps);
    return report_device_errors(eb);
}

int hc_mhd_cfl_dt(hc_mhd* m, double cfl, double* dt) {
    HC_CUDA(cudaSetDevice(m->p.device));
    MArgs a = margs(m);
    const double seed = 1.0e32;
    HC_CUDA(cudaMemcpyAsync(m->scratch, &seed, sizeof seed, cudaMemcpyHostToDevice, m->st));
    HC_CUDA(cudaMemsetAsync(m->eb, 0, sizeof(ErrBlock), m->st));
    const size_t act = size_t(m->b.n[0]) * m->b.n[1] * m->b.n[2];
    if (m->p.order >= 3) k_mhd_dt<true><<<blocks(act, 256), 256, 0, m->st>>>(a, cfl, m->scratch, ST_DT);
    else k_mhd_dt<false><<<blocks(act, 256), 256, 0, m->st>>>(a, cfl, m->scratch, ST_DT);
    m->launches += 1;
    ErrBlock eb;
    HC_CUDA(cudaMemcpyAsync(dt, m->scratch, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaMemcpyAsync(&eb, m->eb, sizeof eb, cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return report_device_errors(eb);
}

int hc_mhd_max_divb(hc_mhd* m, double* out) {
    HC_CUDA(cudaSetDevice(m->p.device));
    MArgs a = margs(m);
    HC_CUDA(cudaMemsetAsync(m->scratch, 0, sizeof(double), m->st));
    const size_t act = size_t(m->b.n[0]) * m->b.n[1] * m->b.n[2];
    k_mhd_divb<<<blocks(act, 256), 256, 0, m->st>>>(a, m->scratch);
    m->launches += 1;
    HC_CUDA(cudaMemcpyAsync(out, m->scratch, sizeof(double), cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

long hc_mhd_launches(hc_mhd* m) { return m ? m->launches : 0; }

int hc_mhd_floored(hc_mhd* m, unsigned long long* count) {
    HC_CUDA(cudaSetDevice(m->p.device));
    HC_CUDA(cudaMemcpyAsync(count, m->floored, sizeof *count, cudaMemcpyDeviceToHost, m->st));
    HC_CUDA(cudaStreamSynchronize(m->st));
    return HC_OK;
}

int hc_mhd_stream(hc_mhd* m, void** stream) {
    *stream = m->st;
    return HC_OK;
}

int hc_mhd_set_stream(hc_mhd* m, void* stream) {
    HC_CUDA(cudaSetDevice(m->p.device));
    HC_CUDA(cudaStreamSynchronize(m->st));
    if (m->own_stream) HC_CUDA(cudaStreamDestroy(m->st));
    m->own_stream = false;
    m->st = static_cast<cudaStream_t>(stream);
    return HC_OK;
}

int hc_mhd_fill_ghosts(hc_mhd* m) {
    HC_CUDA(cudaSetDevice(m->p.device));
    return launch_ghosts(m);
}

int hc_mhd_compute(hc_mhd* m) {
    HC_CUDA(cudaSetDevice(m->p.device));
    return launch_compute(m);
}

int hc_mhd_compute_range(hc_mhd* m, int zlo, int zhi) {
    if (!m || zlo < 0 || zhi > m->b.n[2] || zlo >= zhi) {
        set_error(HC_INVALID, "hc_mhd_compute_range: need 0 <= zlo < zhi <= nz");
        return HC_INVALID;
    }
    HC_CUDA(cudaSetDevice(m->p.device));
    return launch_front(m, zlo, zhi);
}

int hc_mhd_finish(hc_mhd* m) {
    HC_CUDA(cudaSetDevice(m->p.device));
    return launch_finish(m);
}

int hc_mhd_advance(hc_mhd* m) {
    HC_CUDA(cudaSetDevice(m->p.device));
    return launch_advance(m);
}

int hc_mhd_state(hc_mhd* m, double** dptr, size_t* var_stride, size_t* plane_elems) {
    *dptr = m->s;
    *var_stride = m->b.N;
    *plane_elems = size_t(m->b.P) * m->b.Q;
    return HC_OK;
}

int hc_mhd_dt_acc(hc_mhd* m, double** acc) {
    *acc = &m->ctl->acc;
    return HC_OK;
}

}  // extern "C"
