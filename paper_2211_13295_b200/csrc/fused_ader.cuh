// fused_ader.cuh -- ONE sm_100a kernel per ADER step: reconstruction (MC at O2, WENO3 at
// O3, WENO-AO at the O4 extension) -> per-zone ADER predictor -> face Riemann fluxes
// (Rusanov/HLL, HLLC/HLLI extensions) on all three face families -> flux differencing ->
// conservative update -> CFL dt estimate + exact min-reduction.
//
// Replaces the reference's pipeline stepper.cpp:49-78 (skinny_to_modal, reconstruct_patch,
// predict_patch, make_flux_axis x3, make_du_dt, update_u_timestep) without materialising
// ModalState (40*M B/zone), FluxSet or RateField: the only HBM traffic is U_skinny in
// (plus halo re-reads that hit L2) and U_skinny out -- 80 B per zone-update.
//
// Decomposition (2.5D): a CTA owns a TX x TY column tile and marches a chunk of TZ planes
// upward. For each plane p it keeps planes p-R..p+R of mode 0 (the zone averages) for the
// tile plus a halo of G zones in shared memory (a ring buffer of 2R+1 planes at O3, 2R+2 at
// O2, refilled one plane ahead by bulk copies -- one row per cp.async.bulk, completion on a
// per-slot mbarrier -- or 8-byte cp.async when rows are not 16-byte aligned). One thread owns
// one "E-column": a tile column or a face-adjacent
// ring column (the ring zones' slopes and temporal modes are needed for the tile's boundary
// faces -- the reference computes them on "active + one ring", predictor.cpp:68-70).
//
// Per plane:  [sync] predict: recon + predictor for the thread's zone, six face states kept
//             in registers, +x/+y states published to smem
//             [sync] flux:    west-x, south-y faces (tile threads; east/north ring threads take
//             the tile's last x/y face) and the bottom z-face against the +z state this
//             thread kept from plane p-1
//             [sync] rate:    east/north fluxes from smem -> partial rate of plane p (kept in
//             shared memory); plane p-1 is finalised with its top z-flux and updated
//             (U + dt*rate), dt estimate.
// The rate keeps the reference's association -cx*(E-W) - cy*(N-S) - cz*(T-B)
// (corrector.cpp:89-90) split as (partial(x,y)) - cz*(z), so the result is bit-identical.
#pragma once

#include <cuda_runtime.h>

#include "fused_types.cuh"

#ifndef HC_FUSED_NS
#error "define HC_FUSED_NS (the contraction-policy namespace) before including"
#endif

namespace hc {
namespace HC_FUSED_NS {

// ---- plane loads: one bulk copy (TMA engine, cp.async.bulk) per smem row, completion
// tracked by one mbarrier per ring slot (expect_tx = bytes of the plane)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// (a wait that never completes -- e.g. a copy whose byte count disagrees with expect_tx --
// traps after ~2^22 suspended tries instead of hanging the device)
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1, P2;\n"
        ".reg .u32 n;\n"
        "mov.u32 n, 0;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "add.u32 n, n, 1;\n"
        "setp.gt.u32 P2, n, 4194304;\n"
        "@P2 trap;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <bool O3, int TX, int TY>
struct FusedShape {
    static constexpr int R = O3 ? 2 : 1;   // reconstruction stencil radius
    static constexpr int G = R + 1;        // halo: one ring + stencil
    // plane ring: O3 refills the slot of plane p-2 after the predict phase (5 slots); O2's
    // oldest plane (p-1) is read until the end of the iteration, so it keeps a spare slot
    static constexpr int NB = O3 ? 2 * R + 1 : 2 * R + 2;
    static constexpr bool LATE_LOAD = O3;
    static constexpr int W = TX + 2 * G;
    static constexpr int H = TY + 2 * G;
    static constexpr int PLANE = W * H * NV;  // doubles per smem plane
    static constexpr int NE = TX * TY + 2 * TX + 2 * TY;  // E-columns (tile + face rings)
    static constexpr int NT = (NE + 31) / 32 * 32;        // whole warps (shuffles need them)
    static constexpr int XP_N = TY * (TX + 1);  // +x states, columns -1..TX-1
    static constexpr int YP_N = (TY + 1) * TX;  // +y states, rows -1..TY-1
    static constexpr int FX_N = TY * (TX + 1);  // x faces 0..TX
    static constexpr int FY_N = (TY + 1) * TX;  // y faces 0..TY
    // FX aliases XP and FY aliases YP: each face's thread reads its +x/+y neighbour state and
    // then writes that face's flux to the same slot (no other reader in between)
    // per-thread carried state of the owned zones (partial x/y rate of plane p, z flux at the
    // bottom of plane p), [NV][TX*TY]: explicit shared memory instead of register spills
    // (+ each owned thread's running CFL minimum)
    static constexpr int CARRY = 2 * NV * TX * TY + TX * TY + NT / 2;  // (+ column offsets)
    static constexpr size_t SMEM =
        sizeof(double) * (size_t(NB) * PLANE + NV * (XP_N + YP_N) + 32 + CARRY);
};

#ifndef HC_REASSOC
#define HC_REASSOC 0
#endif
// evaluation mode of the hot path (pointwise.cuh): 1 = bit-exact branch-free, 2 = FMA build
// with the approximate division
constexpr int FM = HC_REASSOC ? 2 : 1;

// WENO3 point (reconstruct.hpp:46-73) for the FMA build: the normalised weights
// (w_k / P_k) / sum_j (w_j / P_j) with P_k = (eps + IS_k)^2 are evaluated as
// (w_k prod_{j!=k} P_j) / sum_j (w_j prod_{i!=j} P_i) -- one division instead of four.
// Same mathematics, different rounding (<= a few ulp per weight); used only when the
// translation unit opts out of bit-exactness (fused_fast.cu). P_k lies in [eps^2, ~1e12]
// for physical states, so the triple products stay far from over/underflow.
template <int FAST>
__device__ __forceinline__ void weno3_1div(double s0, double s1, double s2, double s3,
                                           double s4, const Limiter& L, double& ux2,
                                           double& uxx2, Fault& f) {
    // doubled slopes and 4 eps as in weno3_2x: returns (2 ux, 2 uxx)
    double d0 = s1 - s0, d1 = s2 - s1, d2 = s3 - s2, d3 = s4 - s3;
    double ux_l = 3.0 * d1 - d0;
    double uxx_l = d1 - d0;
    double ux_c = d1 + d2;
    double uxx_c = d2 - d1;
    double ux_r = 3.0 * d2 - d3;
    double uxx_r = d3 - d2;
    const double k2 = 13.0 / 3.0;
    const double eps4 = 4.0 * L.eps;
    double el = eps4 + (ux_l * ux_l + k2 * uxx_l * uxx_l);
    double ec = eps4 + (ux_c * ux_c + k2 * uxx_c * uxx_c);
    double er = eps4 + (ux_r * ux_r + k2 * uxx_r * uxx_r);
    double pl = el * el, pc = ec * ec, pr = er * er;
    double al = L.w0 * (pc * pr), ac = L.w1 * (pl * pr), ar = L.w2 * (pl * pc);
    double inv = ddiv<FAST>(1.0, al + ac + ar, f);
    ux2 = (al * ux_l + ac * ux_c + ar * ux_r) * inv;
    uxx2 = (al * uxx_l + ac * uxx_c + ar * uxx_r) * inv;
}

// WENO-AO(5,3) (pointwise.cuh weno_ao) for the FMA build with one division: with
// P_k = (eps + beta_k)^2 and A_k = g_k prod_{j!=k} P_j, the normalised weights are
// A_k / sum A and the quartic's ratio w_h / g_h is prod_{j!=h} P_j / sum A. Products of three
// P_k lie in [eps^6, ~1e40] for physical states (eps = 1e-12), far from over/underflow.
template <int FAST>
__device__ __forceinline__ void weno_ao_1div(double s0, double s1, double s2, double s3,
                                             double s4, const Limiter& L, double* m, Fault& f) {
    const double ghi = AO_GAMMA_HI;
    double o1 = 0.5 * (s3 - s1), o2 = 0.5 * (s4 - s0);
    double e1 = 0.5 * (s3 + s1) - s2, e2 = 0.5 * (s4 + s0) - s2;
    double u3 = (o2 - 2.0 * o1) * (1.0 / 6.0);
    double u1 = o1 - (11.0 / 10.0) * u3;
    double u4 = (e2 - 4.0 * e1) * (1.0 / 12.0);
    double u2 = e1 - (9.0 / 7.0) * u4;
    double d0 = s1 - s0, d1 = s2 - s1, d2 = s3 - s2, d3 = s4 - s3;
    double ux_l = 0.5 * (3.0 * d1 - d0), uxx_l = 0.5 * (d1 - d0);
    double ux_c = 0.5 * (d1 + d2), uxx_c = 0.5 * (d2 - d1);
    double ux_r = 0.5 * (3.0 * d2 - d3), uxx_r = 0.5 * (d3 - d2);
    const double k2 = 13.0 / 3.0;
    double ta = u1 + (1.0 / 10.0) * u3, tb = u2 + (123.0 / 455.0) * u4;
    double eh = L.eps + (ta * ta + k2 * tb * tb + (781.0 / 20.0) * u3 * u3 +
                         (1421461.0 / 2275.0) * u4 * u4);
    double el = L.eps + (ux_l * ux_l + k2 * uxx_l * uxx_l);
    double ec = L.eps + (ux_c * ux_c + k2 * uxx_c * uxx_c);
    double er = L.eps + (ux_r * ux_r + k2 * uxx_r * uxx_r);
    double ph = eh * eh, pl = el * el, pc = ec * ec, pr = er * er;
    double phl = ph * pl, pcr = pc * pr;
    double nh = pl * pcr, nl = ph * pcr, nc = phl * pr, nr = phl * pc;  // prod_{j!=k} P_j
    double gl = (1.0 - ghi) * L.w0, gc = (1.0 - ghi) * L.w1, gr = (1.0 - ghi) * L.w2;
    double al = gl * nl, ac = gc * nc, ar = gr * nr;
    double inv = ddiv<FAST>(1.0, ghi * nh + al + ac + ar, f);
    double wl = al * inv, wc = ac * inv, wr = ar * inv;
    double ratio = nh * inv;
    m[0] = ratio * (u1 - (gl * ux_l + gc * ux_c + gr * ux_r)) + (wl * ux_l + wc * ux_c + wr * ux_r);
    m[1] = ratio * (u2 - (gl * uxx_l + gc * uxx_c + gr * uxx_r)) +
           (wl * uxx_l + wc * uxx_c + wr * uxx_r);
    m[2] = ratio * u3;
    m[3] = ratio * u4;
}

template <int FAST>
__device__ __forceinline__ void weno_ao_k(double s0, double s1, double s2, double s3, double s4,
                                          const Limiter& L, double* m, Fault& f) {
    if (HC_REASSOC)
        weno_ao_1div<FAST>(s0, s1, s2, s3, s4, L, m, f);
    else
        weno_ao<FAST>(s0, s1, s2, s3, s4, L, m, f);
}

// both return twice the slopes (consumers: extrap2)
template <int FAST>
__device__ __forceinline__ void weno3_k(double s0, double s1, double s2, double s3, double s4,
                                        const Limiter& L, double& ux2, double& uxx2, Fault& f) {
    if (HC_REASSOC)
        weno3_1div<FAST>(s0, s1, s2, s3, s4, L, ux2, uxx2, f);
    else
        // (RCP off: the reciprocal form measured 1 % slower in this kernel's register budget)
        weno3_2x<FAST, false>(s0, s1, s2, s3, s4, L, ux2, uxx2, f);
}

// Face states (extrapolate_to_face + 0.5 * tau, corrector.cpp:30-33) of one zone from its
// mode-0 neighbourhood: reconstruction (reconstruct.cpp:16-28 MC, :42-61 WENO3) and the
// ADER predictor (predictor.cpp:26-60). pc: the zone in the current smem plane (rows W*NV
// apart); zm2..zp2: the zone's column in planes p-2..p+2.
template <int ORD, int FAST, bool RK>
__device__ __forceinline__ void zone_states(const double* pc, int row, const double* zm2,
                                            const double* zm1, const double* zp1,
                                            const double* zp2, const FusedArgs& a, double dt,
                                            double (*st)[NV], Fault& f) {
    constexpr bool O3 = ORD >= 3;
    double face[6][NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const double u0 = pc[q];
        if (ORD == 4) {  // WENO-AO(5,3) extension (pointwise.cuh weno_ao)
            double mx[4], my[4], mz[4];
            weno_ao_k<FAST>(pc[-2 * NV + q], pc[-NV + q], u0, pc[NV + q], pc[2 * NV + q], a.lim,
                          mx, f);
            weno_ao_k<FAST>(pc[-2 * row + q], pc[-row + q], u0, pc[row + q], pc[2 * row + q],
                          a.lim, my, f);
            weno_ao_k<FAST>(zm2[q], zm1[q], u0, zp1[q], zp2[q], a.lim, mz, f);
            face[0][q] = extrap4(u0, +1.0, mx);
            face[1][q] = extrap4(u0, -1.0, mx);
            face[2][q] = extrap4(u0, +1.0, my);
            face[3][q] = extrap4(u0, -1.0, my);
            face[4][q] = extrap4(u0, +1.0, mz);
            face[5][q] = extrap4(u0, -1.0, mz);
        } else if (!O3) {
            const double cfac = q == 0 ? a.lim.cfac_rho : a.lim.cfac_other;
            const double sx = mc_limiter(pc[NV + q] - u0, u0 - pc[-NV + q], cfac);
            const double sy = mc_limiter(pc[row + q] - u0, u0 - pc[-row + q], cfac);
            const double sz = mc_limiter(zp1[q] - u0, u0 - zm1[q], cfac);
            face[0][q] = extrap<false>(u0, +1.0, sx, 0.0);
            face[1][q] = extrap<false>(u0, -1.0, sx, 0.0);
            face[2][q] = extrap<false>(u0, +1.0, sy, 0.0);
            face[3][q] = extrap<false>(u0, -1.0, sy, 0.0);
            face[4][q] = extrap<false>(u0, +1.0, sz, 0.0);
            face[5][q] = extrap<false>(u0, -1.0, sz, 0.0);
        } else {
            double ux, uxx, uy, uyy, uz, uzz;
            weno3_k<FAST>(pc[-2 * NV + q], pc[-NV + q], u0, pc[NV + q], pc[2 * NV + q], a.lim,
                          ux, uxx, f);
            weno3_k<FAST>(pc[-2 * row + q], pc[-row + q], u0, pc[row + q], pc[2 * row + q],
                          a.lim, uy, uyy, f);
            weno3_k<FAST>(zm2[q], zm1[q], u0, zp1[q], zp2[q], a.lim, uz, uzz, f);
            face[0][q] = extrap2<true>(u0, +1.0, ux, uxx);  // doubled modes
            face[1][q] = extrap2<true>(u0, -1.0, ux, uxx);
            face[2][q] = extrap2<true>(u0, +1.0, uy, uyy);
            face[3][q] = extrap2<true>(u0, -1.0, uy, uyy);
            face[4][q] = extrap2<true>(u0, +1.0, uz, uzz);
            face[5][q] = extrap2<true>(u0, -1.0, uz, uzz);
        }
    }
    double tau[NV];
    if (RK) {  // Runge-Kutta stage: temporal mode zeroed (stepper.cpp:110-113)
#pragma unroll
        for (int q = 0; q < NV; ++q) tau[q] = 0.0;
    } else {
        predictor<O3, FAST>(face, dt, a.idx, a.idy, a.idz, a.gamma, tau, f);
    }
    // + 0.5 * 0.0 is kept at RK stages: it turns -0.0 into +0.0 exactly as the reference
#pragma unroll
    for (int s = 0; s < 6; ++s)
#pragma unroll
        for (int q = 0; q < NV; ++q) st[s][q] = face[s][q] + 0.5 * tau[q];
}

// Cold paths: re-run in careful mode (IEEE division, exact fault capture) when the fast path
// flagged a division outside its validity range or an unphysical state. Arguments and results
// travel by value so the hot path's arrays stay in registers.
struct V5 {
    double v[NV];
};
struct S6 {
    double v[6][NV];
};
struct Careful {
    S6 st;
    Fault f;
};

template <int ORD, bool RK>
__device__ __noinline__ Careful zone_states_careful(const double* pc, int row, const double* zm2,
                                                    const double* zm1, const double* zp1,
                                                    const double* zp2, const FusedArgs& a,
                                                    double dt) {
    Careful c;
    c.f.clear();
    zone_states<ORD, 0, RK>(pc, row, zm2, zm1, zp1, zp2, a, dt, c.st.v, c.f);
    return c;
}

struct CarefulFlux {
    V5 f5;
    Fault f;
};

template <int SOLVER, int A>
__device__ __noinline__ CarefulFlux riemann_careful(V5 ul, V5 ur, double gamma) {
    CarefulFlux c;
    c.f.clear();
    riemann<SOLVER, A, false>(ul.v, ur.v, gamma, c.f5.v, c.f);
    return c;
}

__device__ __noinline__ double eval_tstep_careful(V5 u, double cfl, double dx, double dy,
                                                  double dz, double gamma, Fault* f) {
    return eval_tstep<false>(u.v, cfl, dx, dy, dz, gamma, *f);
}

template <int SOLVER, int A>
__device__ __forceinline__ void face_flux(const double* ul, const double* ur, double gamma,
                                          double* f5, Fault& f) {
    riemann<SOLVER, A, FM>(ul, ur, gamma, f5, f);
    if (f.redo()) {
        V5 l, r;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            l.v[q] = ul[q];
            r.v[q] = ur[q];
        }
        CarefulFlux c = riemann_careful<SOLVER, A>(l, r, gamma);
#pragma unroll
        for (int q = 0; q < NV; ++q) f5[q] = c.f5.v[q];
        f = c.f;
    }
}

// RK = false: one ADER step (predictor + U += dt*rate, stepper.cpp:49-78).
// RK = true: one Runge-Kutta stage (temporal mode zero, U' = a*U0 + b*(U + dt*rate),
// stepper.cpp:100-143); the CFL estimate is only taken when a.want_dt (last stage,
// rk_step's compute_dt_next, stepper.cpp:155-156).
template <int ORD, int SOLVER, int TX, int TY, int MINB, bool RK>
__global__ void __launch_bounds__(FusedShape<(ORD >= 3), TX, TY>::NT, MINB)
    fused_ader_kernel(const FusedArgs a) {
    constexpr bool O3 = ORD >= 3;  // radius-2 stencil (WENO3, or WENO-AO at ORD 4)
    using S = FusedShape<O3, TX, TY>;
    constexpr int R = S::R, G = S::G, NB = S::NB, W = S::W, H = S::H;
    if (a.ctl->done) return;
    // the step's buffers, picked once by thread 0 and kept in shared memory (read where used)
    __shared__ double* sbuf[3];  // in, out (may alias start at the last RK stage), start
    if (threadIdx.x == 0) {
        const int cur = a.ctl->cur;  // buffer holding the start-of-step state
        sbuf[0] = a.buf[(cur + a.in_rel) % a.nbuf];
        sbuf[1] = a.buf[(cur + a.out_rel) % a.nbuf];
        sbuf[2] = a.buf[cur];
    }

    extern __shared__ __align__(128) double smem[];
    __shared__ unsigned long long mbar[NB];
    double* planes = smem;                          // [NB][H][W][5]
    double* XP = planes + size_t(NB) * S::PLANE;    // [TY][TX+1][5]
    double* YP = XP + S::XP_N * NV;                 // [TY+1][TX][5]
    double* FX = XP;                                // [TY][TX+1][5], aliases XP
    double* FY = YP;                                // [TY+1][TX][5], aliases YP
    double* red = YP + S::YP_N * NV;                // [32]

    const int tid = threadIdx.x;
    // E-column index of this thread. a.interleave = 0: tile columns on the first warps, ring
    // columns on the last; 1: every warp holds (NE / warps) columns, tile and ring mixed, so
    // the phases after the predictor (faces, update) weigh the same on every warp
    int eidx = tid;
    {
        constexpr int NW = S::NT / 32, TPW = TX * TY / NW, RPW = (S::NE - TX * TY) / NW;
        // (only tile shapes whose tile and ring columns split evenly over the warps)
        if constexpr (TX * TY % NW == 0 && (S::NE - TX * TY) % NW == 0 && TPW + RPW <= 32) {
            if (a.interleave) {
                const int w = tid >> 5, l = tid & 31;
                eidx = l < TPW ? w * TPW + l
                               : (l < TPW + RPW ? TX * TY + w * RPW + (l - TPW) : S::NE + w);
            }
        }
    }
    double* part = red + 32 + eidx;         // [NV] stride TX*TY (owned threads only)
    double* fz_prev = part + NV * TX * TY;  // [NV] stride TX*TY
    // ---- E-column of this thread
    int ci, cj;
    bool is_tile;
    {
        int t = eidx;
        if (t >= S::NE) {  // padding lanes: no column
            ci = cj = -(1 << 20);
            is_tile = false;
        } else if (t < TX * TY) {
            ci = t % TX;
            cj = t / TX;
            is_tile = true;
        } else {
            is_tile = false;
            t -= TX * TY;
            if (t < TX) { ci = t; cj = -1; }
            else if ((t -= TX) < TX) { ci = t; cj = TY; }
            else if ((t -= TX) < TY) { ci = -1; cj = t; }
            else { t -= TY; ci = TX; cj = t; }
        }
    }
    const int tx0 = blockIdx.x * TX, ty0 = blockIdx.y * TY;  // active coords of tile origin
    const int ia = tx0 + ci, ja = ty0 + cj;                   // active coords of the column
    // Roles (partial tiles at the domain edge included):
    //  owned  -- an active zone of this tile: bottom z face, update, dt estimate
    //  xface  -- computes the x face on its west side (faces 0..nx next to an owned zone)
    //  yface  -- computes the y face on its south side
    //  exists -- inside active + one ring in x/y: gets a temporal mode (predictor.cpp:68-70)
    const bool owned = is_tile && ia < a.nx && ja < a.ny;
    const bool xface = cj >= 0 && cj < TY && ci >= 0 && ja < a.ny && ia <= a.nx &&
                       (ci >= 1 || ia < a.nx);
    const bool yface = ci >= 0 && ci < TX && cj >= 0 && ia < a.nx && ja <= a.ny &&
                       (cj >= 1 || ja < a.ny);
    const bool exists = ia >= -1 && ia <= a.nx && ja >= -1 && ja <= a.ny;
    const int kz0 = a.kz_first + blockIdx.z * a.tz;  // first active plane (active z)
    const int nzc = min(a.tz, a.kz_last - kz0);
    // dt and cx, cy, cz (corrector.cpp:75) live in shared memory (red[16..19], free until the
    // final reduction): loop-invariant values kept in registers would be spilled
    if (tid == 0) {
        const double dt0 = a.ctl->dt;
        red[16] = dt0 / a.dx;
        red[17] = dt0 / a.dy;
        red[18] = dt0 / a.dz;
        red[19] = dt0;
    }

    // storage pointer of (active plane z, active row ty0 - G, active col tx0 - G)
    const size_t plane_stride = size_t(a.my_pad) * a.pitch;
    auto gsrc = [&](int zact) -> const double* {
        return sbuf[0] + size_t(zact + a.gh) * plane_stride + size_t(ty0 - G + a.gh) * a.pitch +
               size_t(tx0 - G + a.gh) * NV;
    };
    // ring slot of a plane: planes are loaded in order from zfirst, so slot = index % NB and
    // the mbarrier phase of that load = (index / NB) & 1
    const int zfirst = kz0 - 1 - R;
    constexpr unsigned ROW_BYTES = W * NV * sizeof(double);  // 16-byte multiple (W even)
    static_assert(ROW_BYTES % 16 == 0, "bulk-copy rows must be 16-byte multiples");
    auto load_plane = [&](int zact) {
        // caller guarantees every thread finished reading the slot (a __syncthreads)
        const int li = zact - zfirst;
        double* dst = planes + size_t(li % NB) * S::PLANE;
        const double* src = gsrc(zact);
        if (!a.bulk) {  // unaligned rows (odd pitch): 8-byte cp.async, waited before the barrier
            for (int r = tid / 32; r < H; r += S::NT / 32)
                for (int c = tid % 32; c < W * NV; c += 32)
                    cp_async8(dst + r * (W * NV) + c, src + size_t(r) * a.pitch + c);
            return;
        }
        unsigned long long* bar = &mbar[li % NB];
        if (tid < 32) {
            if (tid == 0) {
                fence_proxy_async();  // generic-proxy reads of the slot before the async writes
                mbar_arrive_expect_tx(bar, H * ROW_BYTES);
            }
            __syncwarp();
            for (int r = tid; r < H; r += 32)
                bulk_g2s(dst + r * (W * NV), src + size_t(r) * a.pitch, ROW_BYTES, bar);
        }
    };
    auto wait_plane = [&](int zact) {
        if (!a.bulk) return;
        const int li = zact - zfirst;
        mbar_wait(&mbar[li % NB], unsigned(li / NB) & 1u);
    };
    auto P = [&](int zact) -> const double* {
        return planes + size_t((zact - zfirst) % NB) * S::PLANE;
    };

    if (tid == 0) {
        for (int i = 0; i < NB; ++i) mbar_init(&mbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // prologue: planes kz0-1-R .. kz0-1+R
    for (int z = kz0 - 1 - R; z <= kz0 - 1 + R; ++z) load_plane(z);

    constexpr int CS = TX * TY;  // stride of the carried arrays
    double zp_prev[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) zp_prev[q] = 0.0;
    double* dt_min = fz_prev + NV * CS;  // this owned thread's running CFL minimum
    if (owned) dt_min[0] = 1.0e32;
    // offset (doubles) of this column's zone in a smem plane, kept in shared memory and read
    // where used (a register copy would be spilled)
    int* zoff = reinterpret_cast<int*>(dt_min - eidx + CS) + tid;
    zoff[0] = ((cj + G) * W + (ci + G)) * NV;

    for (int lp = -1; lp <= nzc; ++lp) {
        const int p = kz0 + lp;
        if (!a.bulk) cp_async_wait_all();
        __syncthreads();  // previous iteration's reads of the oldest slot are done
        if (!S::LATE_LOAD && lp <= nzc - 1) load_plane(p + R + 1);
        for (int z = p - R; z <= p + R; ++z) wait_plane(z);

        const bool zring = (lp == -1 || lp == nzc);
        const bool do_zone = zring ? owned : exists;
        // ------------------------------------------------------------- predict
        double st[6][NV];  // face states incl. 0.5*tau: E, W, N, S, T, B
        if (do_zone) {
            const double* pc = P(p) + zoff[0];
            const double* zm1 = P(p - 1) + zoff[0];
            const double* zp1 = P(p + 1) + zoff[0];
            const double* zm2 = O3 ? P(p - 2) + zoff[0] : zm1;
            const double* zp2 = O3 ? P(p + 2) + zoff[0] : zp1;
            Fault f;
            f.clear();
            zone_states<ORD, FM, RK>(pc, W * NV, zm2, zm1, zp1, zp2, a, red[19], st, f);
            if (f.redo()) {
                Careful c =
                    zone_states_careful<ORD, RK>(pc, W * NV, zm2, zm1, zp1, zp2, a, red[19]);
#pragma unroll
                for (int s = 0; s < 6; ++s)
#pragma unroll
                    for (int q = 0; q < NV; ++q) st[s][q] = c.st.v[s][q];
                if (c.f.code) record_fault(a.eb, ST_PREDICT, c.f, ia, ja, p, 0);
            }
            if (!zring) {
                if (ci <= TX - 1 && cj >= 0 && cj < TY)
#pragma unroll
                    for (int q = 0; q < NV; ++q) XP[(cj * (TX + 1) + ci + 1) * NV + q] = st[0][q];
                if (cj <= TY - 1 && ci >= 0 && ci < TX)
#pragma unroll
                    for (int q = 0; q < NV; ++q) YP[((cj + 1) * TX + ci) * NV + q] = st[2][q];
            }
        }
        // z face at the bottom of plane p and the finalisation of plane p-1 need only this
        // thread's own data (its +z state of p-1 and -z state of p, its carried partial rate
        // and bottom flux of p-1): done before the barrier, so only the x/y states stay live
        if (owned) {
            if (lp >= 0) {
                double fz_cur[NV];
                {
                    Fault f;
                    f.clear();
                    face_flux<SOLVER, 2>(zp_prev, st[5], a.gamma, fz_cur, f);
                    if (f.code) record_fault(a.eb, ST_FLUX, f, p, ia, ja, 2);
                }
                if (lp >= 1) {  // finalise plane p-1 with its top face flux fz_cur
                    const double* u = P(p - 1) + zoff[0];
                    const size_t zi = size_t(p - 1 + a.gh) * plane_stride +
                                      size_t(ja + a.gh) * a.pitch + size_t(ia + a.gh) * NV;
                    double un[NV];
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        double r = part[q * CS] - red[18] * (fz_cur[q] - fz_prev[q * CS]);
                        if (RK)  // stepper.cpp:137 (u0 read before uout is written: may alias)
                            un[q] = a.rk_a * sbuf[2][zi + q] + a.rk_b * (u[q] + r);
                        else
                            un[q] = u[q] + r;
                    }
                    double* dst = sbuf[1] + zi;
#pragma unroll
                    for (int q = 0; q < NV; ++q) dst[q] = un[q];
                    if (!RK || a.want_dt) {
                        Fault f;
                        f.clear();
                        double d = FM == 2 ? eval_tstep_inv<FM>(un, a.cfl, a.idx, a.idy, a.idz,
                                                                a.gamma, f)
                                           : eval_tstep<FM>(un, a.cfl, a.dx, a.dy, a.dz,
                                                            a.gamma, f);
                        if (f.redo()) {
                            V5 u5;
#pragma unroll
                            for (int q = 0; q < NV; ++q) u5.v[q] = un[q];
                            f.clear();
                            d = eval_tstep_careful(u5, a.cfl, a.dx, a.dy, a.dz, a.gamma, &f);
                        }
                        if (f.code) record_fault(a.eb, RK ? ST_DT : ST_UPDATE, f, ia, ja, p - 1, 0);
                        else dt_min[0] = smin(dt_min[0], d);
                    }
                }
#pragma unroll
                for (int q = 0; q < NV; ++q) fz_prev[q * CS] = fz_cur[q];
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) zp_prev[q] = st[4][q];
        }
        __syncthreads();
        // plane p-R is no longer read this iteration: refill its slot with p+R+1
        if (S::LATE_LOAD && lp <= nzc - 1) load_plane(p + R + 1);
        // ---------------------------------------------------------------- flux
        if (do_zone) {
            if (!zring && xface) {  // x face at the west of this column
                {
                    double ul[NV], f5[NV];
#pragma unroll
                    for (int q = 0; q < NV; ++q) ul[q] = XP[(cj * (TX + 1) + ci) * NV + q];
                    Fault f;
                    f.clear();
                    face_flux<SOLVER, 0>(ul, st[1], a.gamma, f5, f);
                    if (f.code) record_fault(a.eb, ST_FLUX, f, ia, ja, p, 0);
#pragma unroll
                    for (int q = 0; q < NV; ++q) FX[(cj * (TX + 1) + ci) * NV + q] = f5[q];
                }
            }
            if (!zring && yface) {  // y face at the south of this column
                {
                    double ul[NV], f5[NV];
#pragma unroll
                    for (int q = 0; q < NV; ++q) ul[q] = YP[(cj * TX + ci) * NV + q];
                    Fault f;
                    f.clear();
                    face_flux<SOLVER, 1>(ul, st[3], a.gamma, f5, f);
                    if (f.code) record_fault(a.eb, ST_FLUX, f, ja, ia, p, 1);
#pragma unroll
                    for (int q = 0; q < NV; ++q) FY[(cj * TX + ci) * NV + q] = f5[q];
                }
            }
        }
        __syncthreads();
        // ---------------------------------------------------------------- rate
        if (owned && lp >= 0 && lp < nzc) {  // x/y part of the rate of plane p
            const double* fxw = FX + (cj * (TX + 1) + ci) * NV;
            const double* fys = FY + (cj * TX + ci) * NV;
#pragma unroll
            for (int q = 0; q < NV; ++q)
                part[q * CS] =
                    -red[16] * (fxw[NV + q] - fxw[q]) - red[17] * (fys[TX * NV + q] - fys[q]);
        }
    }

    // ---- block min -> one atomic per CTA (exact: min is order independent)
    if (RK && !a.want_dt) return;
    double dmin = owned ? dt_min[0] : 1.0e32;
    dmin = warp_min(dmin);
    if ((tid & 31) == 0) red[tid >> 5] = dmin;
    __syncthreads();
    if (tid < 32) {
        constexpr int NW = (S::NT + 31) / 32;
        double v = tid < NW ? red[tid] : 1.0e32;
        v = warp_min(v);
        if (tid == 0) atomic_min_pos(&a.ctl->acc, v);
    }
}

}  // namespace HC_FUSED_NS
}  // namespace hc
