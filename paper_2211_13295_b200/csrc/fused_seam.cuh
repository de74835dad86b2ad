// fused_seam.cuh -- the ring-free fused ADER step (both builds): the same update as
// fused_ader.cuh (reconstruction -> ADER predictor -> face Riemann fluxes -> flux
// differencing -> update -> CFL min; stepper.cpp:49-78, predictor.cpp:26-91,
// corrector.cpp:15-125) with no redundant zone work and no waiting between CTAs.
//
//  * fused_ader.cuh re-runs reconstruction + predictor on a one-zone ring around each 16 x 12
//    tile (the faces on the tile boundary need the outside zone's state: predictor.cpp:68-70's
//    "active + one ring"), 1.29x the owned zones, ~20 % of the kernel's FP64 instructions.
//    fused_persist.cuh removed the ring by exchanging boundary states between resident CTAs
//    through L2 and measured 1.8x slower (waits, fences, long-scoreboard stalls).
//  * Here every zone's face states are computed once, by its owner, and a CTA never waits on
//    another: the faces ON a tile boundary ("seams") are left out of the fused kernel. Each
//    tile publishes the face states of its edge zones (the -x state of column 0, the +x state
//    of column 31, the -y / +y states of its first / last row) to a seam buffer, updates its
//    edge zones provisionally -- their missing seam fluxes counted as zero -- and leaves their
//    CFL estimate out. A second, small kernel (seam_fix_kernel) solves each seam face from the
//    two published states, adds the missing flux terms to the provisional edge zones and
//    takes their CFL estimate. Both neighbours of a seam face solve it from the same two
//    states with the same code, so the fluxes they apply are identical (conservation holds).
//  * Tile = 32 columns x up to 8 rows, one warp per row: x neighbours are lanes of one warp
//    (the -x side state and the east face flux travel by shuffles), y neighbours pass through
//    one shared-memory array; planes arrive by TMA tensor copies (one box per plane, per-slot
//    mbarrier), as in fused_persist.cuh.
//
// FMA build: the provisional form U + (r_partial - cz (T - B)) followed by + cx W - cx E +
// cy S - cy N re-associates the reference's rate (corrector.cpp:89-90) (tolerance-tested
// against the reference, like the FMA ring kernel). Bit-exact build (EX): the reference's
// association throughout -- interior zones finish as U + ((-cx (E - W) - cy (N - S)) -
// cz (T - B)) with the bottom z flux carried in registers; an edge zone publishes its rate
// parts (edge_x / edge_y records) and seam_fix_kernel evaluates its whole rate in the same
// order. Periodic x and y only (the zone across the mesh edge is the last tile's own edge
// zone); other meshes run fused_ader.cuh.
#pragma once

#include "fused_persist.cuh"

namespace hc {
namespace HC_FUSED_NS {

template <int ORD>
struct SeamShape {
    static constexpr bool O3 = ORD >= 3;
    static constexpr int TX = SEAM_TX, TYM = SEAM_TYM;
    static constexpr int R = O3 ? 2 : 1;
    // planes p-R..p+R; the refill of p+R+1 (issued after the mid-plane barrier) takes the
    // slot of p-R, which only the predict phase reads
    static constexpr int NB = 2 * R + 1;
    static constexpr int HX = O3 ? 3 : 2;  // x halo = storage ghosts (16-byte TMA box origin)
    static constexpr int W = TX + 2 * HX;
    static constexpr int H = TYM + 2 * R;
    static constexpr int BOX = W * H * NV;
    static constexpr int PLANE = (BOX + 15) / 16 * 16;  // 128-byte aligned slots
    static constexpr int NT = TX * TYM;
    static constexpr int YPF = TYM * TX * NV;  // +y states (rows 1..h-1) / south fluxes
    // planes + YPF + one carried 5-vector per zone + 24 scalars: 109 KB at O3, two CTAs of
    // eight warps per SM
    static constexpr size_t SMEM = sizeof(double) * (size_t(NB) * PLANE + YPF + NV * NT + 24 + TYM);
    static constexpr int MINB = NT <= 256 ? 2 : 1;  // CTAs per SM the 128 registers allow
};

// rows of tile row `by` when ny rows are split over nty tiles as evenly as possible
__device__ __forceinline__ void seam_rows(int ny, int nty, int by, int& h, int& y0) {
    const int base = ny / nty, rem = ny % nty;
    h = base + (by < rem ? 1 : 0);
    y0 = by * base + min(by, rem);
}
// inverse: the tile row of row ja, and whether ja is that tile's first or last row
__device__ __forceinline__ bool seam_row_edge(int ny, int nty, int ja) {
    const int base = ny / nty, rem = ny % nty, big = rem * (base + 1);
    const int loc = ja < big ? ja % (base + 1) : (ja - big) % base;
    const int h = ja < big ? base + 1 : base;
    return loc == 0 || loc == h - 1;
}

// seam records, one component per row so a warp's accesses along the seam are contiguous:
// SX [k][sx][side][q][ja] (x seam sx = the face at x = 32 sx; side 0 = the state of the zone
// west of the face, 1 = east), SY [k][sy][side][q][ia]. Returns the q = 0 element; component
// q is at + q * SEAM_STRIDE (the seam length).
__device__ __forceinline__ double* seam_x(const SeamArgs& s, int k, int sx, int ja, int side) {
    return s.sx + ((size_t(k) * s.ntx + sx) * 2 + side) * NV * s.ny + ja;
}
__device__ __forceinline__ double* seam_y(const SeamArgs& s, int k, int sy, int ia, int side) {
    return s.sy + ((size_t(k) * s.nty + sy) * 2 + side) * NV * s.nx + ia;
}
// bit-exact build: the rate parts of an edge zone, 3 slots x 5 (entry e at + e * stride, the
// seam length): slot 0 = the x part (-cx (E - W) rounded, or the zone's interior x flux when
// an x face is a seam), slot 1 = the y part (cy (N - S) rounded, or the interior y flux when
// a y face is a seam), slot 2 = the z term cz (T - B). Rows that are a tile's first / last
// (corners included) live with the y seam below / above (EY), the x-edge zones of the other
// rows with the x seam west / east of them (EX), sides as in SX / SY.
__device__ __forceinline__ double* edge_y(const SeamArgs& s, int k, int sy, int ia, int side) {
    return s.ey + ((size_t(k) * s.nty + sy) * 2 + side) * 15 * size_t(s.nx) + ia;
}
__device__ __forceinline__ double* edge_x(const SeamArgs& s, int k, int sx, int ja, int side) {
    return s.ex + ((size_t(k) * s.ntx + sx) * 2 + side) * 15 * size_t(s.ny) + ja;
}

// Per plane p (lp = -1 and nzc are the z-ring planes: predict and z face only):
//  A  predict(p): face states in registers, +y states to YPF, edge-zone states to the seams
//  B  z face at the bottom of p; finalise p-1 from its accumulator and this top flux (U_new =
//     acc - cz T); the accumulator slot then parks the bottom flux of p for C
//  C  x faces (lanes 1..31: the -x side state by shuffle), the accumulator of p =
//     (U - cx (E - W)) + cz B (the east flux by shuffle); y faces (rows 1..h-1) against YPF,
//     south fluxes back to YPF
//  D  accumulator -= cy (N - S)
// Missing seam fluxes count as zero; seam_fix_x / seam_fix_y add them.
template <int ORD, int SOLVER, bool RK, bool ZP>
__global__ void __launch_bounds__(SeamShape<ORD>::NT, SeamShape<ORD>::MINB)
    seam_ader_kernel(const __grid_constant__ FusedArgs a, const SeamArgs sa) {
    using S = SeamShape<ORD>;
    constexpr int R = S::R, NB = S::NB, W = S::W, TX = S::TX;
    constexpr bool EX = FM != 2;  // bit-exact build: the reference's association throughout
    if (a.ctl->done) return;
    __shared__ double* sbuf[3];
    __shared__ const CUtensorMap* smap;
    __shared__ unsigned long long mbar[NB];
    __shared__ int s_tile[2];  // rows h, first row y0
    if (threadIdx.x == 0) {
        seam_rows(a.ny, sa.nty, blockIdx.y, s_tile[0], s_tile[1]);
        const int cur = a.ctl->cur;
        const int in = (cur + a.in_rel) % a.nbuf;
        sbuf[0] = a.buf[in];
        sbuf[1] = a.buf[(cur + a.out_rel) % a.nbuf];
        sbuf[2] = a.buf[cur];
        smap = sa.maps + in;
    }
    extern __shared__ __align__(128) double smem[];
    double* planes = smem;                         // [NB][H][W][5]
    double* YPF = planes + size_t(NB) * S::PLANE;  // [TYM][TX][5]: +y states / south fluxes
    double* acc = YPF + S::YPF;                    // [5][NT] accumulator / parked z flux
    double* red = acc + NV * S::NT;  // [24 + TYM]: dt & c at [16, 20), per-warp CFL minimum at [24, 24 + TYM)

    // coordinates are re-read from the special registers where used (cheap S2R) rather than
    // held in registers across the predictor, which would spill
    auto ci_ = [] { return int(threadIdx.x) & 31; };
    auto cj_ = [] { return int(threadIdx.x) >> 5; };
    auto ia_ = [] { return int(blockIdx.x) * TX + (int(threadIdx.x) & 31); };
    auto ja_ = [&] { return s_tile[1] + (int(threadIdx.x) >> 5); };
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX;
    const int kz0 = a.kz_first + blockIdx.z * a.tz;
    const int nzc = min(a.tz, a.kz_last - kz0);
    if (tid == 0) {
        const double dt0 = a.ctl->dt;
        red[16] = EX ? dt0 / a.dx : dt0 * a.idx;  // (FMA build: dt/dx as dt * (1/dx))
        red[17] = EX ? dt0 / a.dy : dt0 * a.idy;
        red[18] = EX ? dt0 / a.dz : dt0 * a.idz;
        red[19] = dt0;
    }
    if (tid < S::TYM) red[24 + tid] = 1.0e32;
    const size_t plane_stride = size_t(a.my_pad) * a.pitch;
    const int zfirst = kz0 - 1 - R;
    constexpr unsigned PLANE_BYTES = S::BOX * sizeof(double);
    auto load_plane = [&](int zact) {  // one TMA box per plane, issued by thread 0
        if (tid != 0) return;
        const int li = zact - zfirst;
        fence_proxy_async();  // generic-proxy reads of the slot before the async writes
        mbar_arrive_expect_tx(&mbar[li % NB], PLANE_BYTES);
        tma_load_plane(planes + size_t(li % NB) * S::PLANE, smap, (x0 + a.gh - S::HX) * NV,
                       s_tile[1] + a.gh - R, zact + a.gh, &mbar[li % NB]);
    };
    auto wait_plane = [&](int zact) {
        const int li = zact - zfirst;
        mbar_wait(&mbar[li % NB], unsigned(li / NB) & 1u);
    };
    auto P = [&](int zact) -> const double* {
        return planes + size_t((zact - zfirst) % NB) * S::PLANE;
    };
    auto zoff_ = [&] { return ((cj_() + R) * W + (ci_() + S::HX)) * NV; };
    if (tid == 0) {
        for (int i = 0; i < NB; ++i) mbar_init(&mbar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    for (int z = kz0 - 1 - R; z <= kz0 - 1 + R; ++z) load_plane(z);

    constexpr int CS = S::NT;
    double zp_prev[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) zp_prev[q] = 0.0;
    [[maybe_unused]] double fzb[NV];  // bit-exact build: the bottom z flux of the plane before
    // the record of an edge zone of plane k (bit-exact build), entry stride in *es
    [[maybe_unused]] auto edge_rec = [&](int k, int h, size_t& es) -> double* {
        const int ci = ci_(), cj = cj_();
        const int bx = blockIdx.x, by = blockIdx.y;
        es = size_t(sa.nx);
        if (cj == 0) return edge_y(sa, k, by, ia_(), 1);
        if (cj == h - 1) return edge_y(sa, k, by + 1 == sa.nty ? 0 : by + 1, ia_(), 0);
        es = size_t(sa.ny);
        if (ci == 0) return edge_x(sa, k, bx, ja_(), 1);
        return edge_x(sa, k, bx + 1 == sa.ntx ? 0 : bx + 1, ja_(), 0);
    };

    for (int lp = -1; lp <= nzc; ++lp) {
        const int p = kz0 + lp;
        __syncthreads();  // the previous plane's reads of YPF are done
        for (int z = p - R; z <= p + R; ++z) wait_plane(z);
        const bool real = lp >= 0 && lp < nzc;  // x/y faces of p exist (else a z-ring plane)
        double st[6][NV];                       // face states incl. 0.5*tau: E, W, N, S, T, B
        const int h = s_tile[0];
        if (cj_() < h) {
            // -------------------------------------------------------------- A: predict
            {
                const int zoff = zoff_();
                const double* pc = P(p) + zoff;
                const double* zm1 = P(p - 1) + zoff;
                const double* zp1 = P(p + 1) + zoff;
                const double* zm2 = S::O3 ? P(p - 2) + zoff : zm1;
                const double* zp2 = S::O3 ? P(p + 2) + zoff : zp1;
                Fault f;
                f.clear();
                zone_states<ORD, FM, RK>(pc, W * NV, zm2, zm1, zp1, zp2, a, red[19], st, f);
                if (f.redo()) {
                    Careful c = zone_states_careful<ORD, RK>(pc, W * NV, zm2, zm1, zp1, zp2, a,
                                                             red[19]);
#pragma unroll
                    for (int s = 0; s < 6; ++s)
#pragma unroll
                        for (int q = 0; q < NV; ++q) st[s][q] = c.st.v[s][q];
                    if (c.f.code) record_fault(a.eb, ST_PREDICT, c.f, ia_(), ja_(), p, 0);
                }
            }
            if (real) {
                const int ci = ci_(), cj = cj_();
                if (cj < h - 1)
#pragma unroll
                    for (int q = 0; q < NV; ++q) YPF[((cj + 1) * TX + ci) * NV + q] = st[2][q];
                // the edge zones' states at the seams (periodic: the last seam wraps to 0)
                const int bx = blockIdx.x, by = blockIdx.y;
                if (ci == 0) {
                    double* r = seam_x(sa, p, bx, ja_(), 1);
#pragma unroll
                    for (int q = 0; q < NV; ++q) __stcg(r + q * a.ny, st[1][q]);
                }
                if (ci == TX - 1) {
                    double* r = seam_x(sa, p, bx + 1 == sa.ntx ? 0 : bx + 1, ja_(), 0);
#pragma unroll
                    for (int q = 0; q < NV; ++q) __stcg(r + q * a.ny, st[0][q]);
                }
                if (cj == 0) {
                    double* r = seam_y(sa, p, by, ia_(), 1);
#pragma unroll
                    for (int q = 0; q < NV; ++q) __stcg(r + q * a.nx, st[3][q]);
                }
                if (cj == h - 1) {
                    double* r = seam_y(sa, p, by + 1 == sa.nty ? 0 : by + 1, ia_(), 0);
#pragma unroll
                    for (int q = 0; q < NV; ++q) __stcg(r + q * a.nx, st[2][q]);
                }
            }
            // ---------------------------------------- B: z face, finalise plane p-1
            if (lp >= 0) {
                double fz[NV];
                {
                    Fault f2;
                    f2.clear();
                    face_flux<SOLVER, 2>(zp_prev, st[5], a.gamma, fz, f2);
                    if (f2.code) record_fault(a.eb, ST_FLUX, f2, p, ia_(), ja_(), 2);
                }
                if (lp >= 1) {
                    const int ci = ci_(), cj = cj_();
                    const int ia = ia_(), ja = ja_();
                    const size_t zi = size_t(p - 1 + a.gh) * plane_stride +
                                      size_t(ja + a.gh) * a.pitch + size_t(ia + a.gh) * NV;
                    const double cz = red[18];
                    const bool edge = ci == 0 || ci == TX - 1 || cj == 0 || cj == h - 1;
                    double un[NV];
                    if constexpr (EX) {
                        if (edge) {  // the z term for seam_fix_kernel; it writes the zone
                            size_t es;
                            double* er = edge_rec(p - 1, h, es);
#pragma unroll
                            for (int q = 0; q < NV; ++q)
                                __stcg(er + (2 * NV + q) * es, cz * (fz[q] - fzb[q]));
                        } else {  // corrector.cpp:89-90: (x part - y part) - cz (T - B)
                            const double* u = P(p - 1) + zoff_();
#pragma unroll
                            for (int q = 0; q < NV; ++q) {
                                const double r = acc[q * CS + tid] - cz * (fz[q] - fzb[q]);
                                if (RK)  // stepper.cpp:137
                                    un[q] = a.rk_a * sbuf[2][zi + q] + a.rk_b * (u[q] + r);
                                else
                                    un[q] = u[q] + r;
                            }
                            double* dst = sbuf[1] + zi;
#pragma unroll
                            for (int q = 0; q < NV; ++q) dst[q] = un[q];
                            if (ZP)
                                zpeer_store(a, p - 1, zi - size_t(p - 1 + a.gh) * plane_stride, un);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < NV; ++q) {
                            // edge zones: provisional (seam_fix_kernel adds the seam fluxes).
                            // cz B and cz T are rounded products (no contraction): equal z
                            // fluxes then cancel exactly, as T - B does in the reference's
                            // association, so a z-invariant state stays z-invariant bit for bit
                            const double v = __dsub_rn(acc[q * CS + tid], __dmul_rn(cz, fz[q]));
                            if (RK)  // stepper.cpp:137 (u0 read before uout is written: may alias)
                                un[q] = a.rk_a * sbuf[2][zi + q] + a.rk_b * v;
                            else
                                un[q] = v;
                        }
                        double* dst = sbuf[1] + zi;
#pragma unroll
                        for (int q = 0; q < NV; ++q) dst[q] = un[q];
                        if (ZP && !edge)  // (edge zones: seam_fix_kernel stores them)
                            zpeer_store(a, p - 1, zi - size_t(p - 1 + a.gh) * plane_stride, un);
                    }
                    double dloc = 1.0e32;
                    if ((!RK || a.want_dt) && !edge) {
                        Fault f3;
                        f3.clear();
                        double d = EX ? eval_tstep<FM>(un, a.cfl, a.dx, a.dy, a.dz, a.gamma, f3)
                                      : eval_tstep_inv<FM>(un, a.cfl, a.idx, a.idy, a.idz, a.gamma, f3);
                        if (f3.redo()) {
                            V5 u5;
#pragma unroll
                            for (int q = 0; q < NV; ++q) u5.v[q] = un[q];
                            f3.clear();
                            d = eval_tstep_careful(u5, a.cfl, a.dx, a.dy, a.dz, a.gamma, &f3);
                        }
                        if (f3.code)
                            record_fault(a.eb, RK ? ST_DT : ST_UPDATE, f3, ia, ja, p - 1, 0);
                        else
                            dloc = d;
                    }
                    if (!RK || a.want_dt) {  // running CFL minimum per warp (exact)
                        dloc = warp_min(dloc);
                        if (ci == 0) red[24 + cj] = smin(red[24 + cj], dloc);
                    }
                }
                if (real) {
                    if constexpr (EX) {
#pragma unroll
                        for (int q = 0; q < NV; ++q) fzb[q] = fz[q];  // B of plane p
                    } else {
#pragma unroll
                        for (int q = 0; q < NV; ++q) acc[q * CS + tid] = fz[q];  // parked for C
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) zp_prev[q] = st[4][q];
        }
        __syncthreads();  // +y states in YPF; every thread is past its reads of plane p-R
        if (lp <= nzc - 1) load_plane(p + R + 1);
        if (!real) continue;
        // ------------------------------------------------------------- C: faces
        // x face first; the x term goes straight into the accumulator, so nothing but the
        // -y state stays live through the y face solve and nothing across the barrier
        const int ci = ci_(), cj = cj_();
        if (cj < h) {  // (whole warps: the shuffles need every lane)
            {
                double ul[NV], fw[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) ul[q] = __shfl_up_sync(0xffffffffu, st[0][q], 1);
                if (ci > 0) {  // x face at the west of this zone (lane 0's is a seam)
                    Fault f;
                    f.clear();
                    face_flux<SOLVER, 0>(ul, st[1], a.gamma, fw, f);
                    if (f.code) record_fault(a.eb, ST_FLUX, f, ia_(), ja_(), p, 0);
                } else {
#pragma unroll
                    for (int q = 0; q < NV; ++q) fw[q] = 0.0;
                }
                [[maybe_unused]] const double cx = red[16], cz = red[18];
                const double* u = P(p) + zoff_();
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    double e = __shfl_down_sync(0xffffffffu, fw[q], 1);  // lane ci+1's west
                    if (ci == TX - 1) e = 0.0;                           // (a seam)
                    if constexpr (EX) {  // the x part, or the interior x flux at a seam column
                        acc[q * CS + tid] =
                            ci == 0 ? e : (ci == TX - 1 ? fw[q] : -cx * (e - fw[q]));
                    } else {
                        const double xt = -cx * (e - fw[q]);
                        // (cz B rounded, no contraction: see B)
                        acc[q * CS + tid] =
                            __dadd_rn(u[q] + xt, __dmul_rn(cz, acc[q * CS + tid]));
                    }
                }
            }
            double fs[NV];
            if (cj > 0) {  // y face at the south of this zone (row 0's is a seam)
                double us[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) us[q] = YPF[(cj * TX + ci) * NV + q];
                Fault f;
                f.clear();
                face_flux<SOLVER, 1>(us, st[3], a.gamma, fs, f);
                if (f.code) record_fault(a.eb, ST_FLUX, f, ja_(), ia_(), p, 1);
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) fs[q] = 0.0;
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) YPF[(cj * TX + ci) * NV + q] = fs[q];
        }
        __syncthreads();  // south fluxes of every row in YPF
        // ---------------------------------------------- D: the y term of the accumulator
        if (cj < h) {
            const double cy = red[17];
            if (EX && (ci == 0 || ci == TX - 1 || cj == 0 || cj == h - 1)) {
                // an edge zone: its x and y parts go to the record (seam_fix_kernel)
                size_t es;
                double* er = edge_rec(p, h, es);
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    const double sf = YPF[(cj * TX + ci) * NV + q];
                    const double nf = cj < h - 1 ? YPF[((cj + 1) * TX + ci) * NV + q] : 0.0;
                    const double y = cj == 0 ? nf : (cj == h - 1 ? sf : cy * (nf - sf));
                    __stcg(er + q * es, acc[q * CS + tid]);
                    __stcg(er + (NV + q) * es, y);
                }
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    const double sf = YPF[(cj * TX + ci) * NV + q];
                    const double nf = cj < h - 1 ? YPF[((cj + 1) * TX + ci) * NV + q] : 0.0;
                    acc[q * CS + tid] -= cy * (nf - sf);
                }
            }
        }
    }

    // ---- CFL minimum of the inner zones: block min -> one atomic per CTA
    if (!RK || a.want_dt) {
        __syncthreads();
        if (tid < 32) {
            double v = tid < S::TYM ? red[24 + tid] : 1.0e32;
            v = warp_min(v);
            if (tid == 0) atomic_min_pos(&a.ctl->acc, v);
        }
    }
}

// The seam faces of planes [kz_first, kz_last), in ONE launch: the edge zones split into three
// disjoint groups, so no zone is written by two threads and no ordering is needed --
//   Y: the y seam faces whose two zones are not tile corners (lanes 1..30): one thread per face
//   X: the x seam faces in rows that are not a tile's first or last: one thread per face
//   C: the tile-corner zones (lane 0 / 31 of a tile's first / last row): one thread per zone,
//      solving its own x and y seam faces (each corner face is solved by both of its zones,
//      from the same two published states, so both apply the same flux)
// A face's flux is subtracted from the zone on its low side and added to the zone on its high
// side (times cx or cy, and b at an RK stage); every thread then takes the CFL estimate of the
// zones it completed; min-reduced per block. Grid (blocks of the three groups, planes).
template <int SOLVER, bool RK, bool ZP>
__global__ void __launch_bounds__(128) seam_fix_kernel(const __grid_constant__ FusedArgs a,
                                                       const SeamArgs sa) {
    if (a.ctl->done) return;
    const int p = a.kz_first + int(blockIdx.y);
    const int nby = (sa.nty * a.nx + 127) / 128, nbx = (sa.ntx * a.ny + 127) / 128;
    const int bid = int(blockIdx.x);
    const int grp = bid < nby ? 0 : (bid < nby + nbx ? 1 : 2);  // Y, X, C
    const unsigned idx = unsigned(bid - (grp == 0 ? 0 : (grp == 1 ? nby : nby + nbx))) * 128u +
                         threadIdx.x;
    constexpr bool EX = FM != 2;
    const int cur = a.ctl->cur;
    double* out = a.buf[(cur + a.out_rel) % a.nbuf];
    [[maybe_unused]] const double* uin = a.buf[(cur + a.in_rel) % a.nbuf];
    [[maybe_unused]] const double* u0 = a.buf[cur];
    const double dt0 = a.ctl->dt;
    // FMA build: b folded into the provisional update's coefficients; bit-exact build: the
    // reference's dt/dx and U' = a U0 + b (U + rate) (stepper.cpp:137)
    const double cx = EX ? dt0 / a.dx : (RK ? a.rk_b * (dt0 * a.idx) : dt0 * a.idx);
    const double cy = EX ? dt0 / a.dy : (RK ? a.rk_b * (dt0 * a.idy) : dt0 * a.idy);
    auto fin = [&](size_t z, int q, double r) {
        return RK ? a.rk_a * u0[z + q] + a.rk_b * (uin[z + q] + r) : uin[z + q] + r;
    };
    auto zidx = [&](int i, int j) {
        return (size_t(p + a.gh) * a.my_pad + size_t(j + a.gh)) * a.pitch + size_t(i + a.gh) * NV;
    };
    // the flux of the seam face whose records start at rec (SoA, `along` apart per component)
    auto solve = [&](const double* rec, int along, int axis, int fa, int fb, double* f5) {
        double ul[NV], ur[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            ul[q] = rec[q * along];         // side 0: the low zone's state
            ur[q] = rec[(NV + q) * along];  // side 1: the high zone's state
        }
        Fault f;
        f.clear();
        if (axis == 0)
            face_flux<SOLVER, 0>(ul, ur, a.gamma, f5, f);
        else
            face_flux<SOLVER, 1>(ul, ur, a.gamma, f5, f);
        if (f.code) record_fault(a.eb, ST_FLUX, f, fa, fb, p, axis);
    };
    auto cfl = [&](const double* v, int i, int j) {
        if (RK && !a.want_dt) return 1.0e32;
        Fault f3;
        f3.clear();
        double d = EX ? eval_tstep<FM>(v, a.cfl, a.dx, a.dy, a.dz, a.gamma, f3)
                      : eval_tstep_inv<FM>(v, a.cfl, a.idx, a.idy, a.idz, a.gamma, f3);
        if (f3.redo()) {
            V5 u5;
#pragma unroll
            for (int q = 0; q < NV; ++q) u5.v[q] = v[q];
            f3.clear();
            d = eval_tstep_careful(u5, a.cfl, a.dx, a.dy, a.dz, a.gamma, &f3);
        }
        if (f3.code) {
            record_fault(a.eb, RK ? ST_DT : ST_UPDATE, f3, i, j, p, 0);
            return 1.0e32;
        }
        return d;
    };
    double dloc = 1.0e32;
    if (grp < 2) {  // one face, two zones
        const int along = grp == 0 ? a.nx : a.ny, nseam = grp == 0 ? sa.nty : sa.ntx;
        if (idx < unsigned(nseam * along)) {
            const int sidx = int(idx / unsigned(along));
            const int l = int(idx - unsigned(sidx) * unsigned(along));
            // corner zones belong to group C
            const bool skip = grp == 0 ? ((l & (SEAM_TX - 1)) == 0 || (l & (SEAM_TX - 1)) == SEAM_TX - 1)
                                       : seam_row_edge(a.ny, sa.nty, l);
            if (!skip) {
                int il, jl, ih, jh;
                if (grp == 1) {
                    ih = sidx * SEAM_TX;
                    il = (sidx == 0 ? a.nx : ih) - 1;
                    jl = jh = l;
                } else {
                    int h, y0;
                    seam_rows(a.ny, sa.nty, sidx, h, y0);
                    jh = y0;
                    jl = (sidx == 0 ? a.ny : y0) - 1;
                    il = ih = l;
                }
                const size_t zl = zidx(il, jl), zh = zidx(ih, jh);
                double vl[NV], vh[NV], f5[NV];
                if (!EX)
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        vl[q] = out[zl + q];
                        vh[q] = out[zh + q];
                    }
                if (grp == 1)
                    solve(seam_x(sa, p, sidx, l, 0), a.ny, 0, ih, jh, f5);
                else
                    solve(seam_y(sa, p, sidx, l, 0), a.nx, 1, jh, ih, f5);
                if constexpr (EX) {
                    // the whole rate of both zones in the reference's association
                    // (corrector.cpp:89-90) from their records and the seam flux
                    const size_t es = grp == 1 ? size_t(a.ny) : size_t(a.nx);
                    const double* rl = grp == 1 ? edge_x(sa, p, sidx, l, 0) : edge_y(sa, p, sidx, l, 0);
                    const double* rh = grp == 1 ? edge_x(sa, p, sidx, l, 1) : edge_y(sa, p, sidx, l, 1);
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        double r_l, r_h;
                        if (grp == 1) {  // x seam: E of the low zone, W of the high zone
                            r_l = (-cx * (f5[q] - rl[q * es]) - rl[(NV + q) * es]) - rl[(2 * NV + q) * es];
                            r_h = (-cx * (rh[q * es] - f5[q]) - rh[(NV + q) * es]) - rh[(2 * NV + q) * es];
                        } else {  // y seam: N of the low zone, S of the high zone
                            r_l = (rl[q * es] - cy * (f5[q] - rl[(NV + q) * es])) - rl[(2 * NV + q) * es];
                            r_h = (rh[q * es] - cy * (rh[(NV + q) * es] - f5[q])) - rh[(2 * NV + q) * es];
                        }
                        vl[q] = fin(zl, q, r_l);
                        vh[q] = fin(zh, q, r_h);
                        out[zl + q] = vl[q];
                        out[zh + q] = vh[q];
                    }
                } else {
                    const double c = grp == 1 ? cx : cy;
#pragma unroll
                    for (int q = 0; q < NV; ++q) {
                        vl[q] = vl[q] - c * f5[q];  // its east / north face
                        vh[q] = vh[q] + c * f5[q];  // its west / south face
                        out[zl + q] = vl[q];
                        out[zh + q] = vh[q];
                    }
                }
                if (ZP) {
                    const size_t pz = size_t(p + a.gh) * a.my_pad * a.pitch;
                    zpeer_store(a, p, zl - pz, vl);
                    zpeer_store(a, p, zh - pz, vh);
                }
                dloc = smin(cfl(vl, il, jl), cfl(vh, ih, jh));
            }
        }
    } else if (idx < unsigned(4 * sa.ntx * sa.nty)) {  // a tile-corner zone
        const int tile = int(idx >> 2), corner = int(idx & 3u);
        const int bx = tile % sa.ntx, by = tile / sa.ntx;
        int h, y0;
        seam_rows(a.ny, sa.nty, by, h, y0);
        const bool east = corner & 1, north = corner & 2;
        const int i = bx * SEAM_TX + (east ? SEAM_TX - 1 : 0);
        const int j = y0 + (north ? h - 1 : 0);
        const size_t z = zidx(i, j);
        double v[NV], fx[NV], fy[NV];
        if (!EX)
#pragma unroll
            for (int q = 0; q < NV; ++q) v[q] = out[z + q];
        const int sx = east ? (bx + 1 == sa.ntx ? 0 : bx + 1) : bx;
        const int sy = north ? (by + 1 == sa.nty ? 0 : by + 1) : by;
        solve(seam_x(sa, p, sx, j, 0), a.ny, 0, east ? i + 1 : i, j, fx);
        solve(seam_y(sa, p, sy, i, 0), a.nx, 1, north ? j + 1 : j, i, fy);
        if constexpr (EX) {
            const size_t es = size_t(a.nx);
            const double* rc = edge_y(sa, p, sy, i, north ? 0 : 1);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const double xi = rc[q * es], yi = rc[(NV + q) * es];
                const double e = east ? fx[q] : xi, w = east ? xi : fx[q];
                const double n = north ? fy[q] : yi, s = north ? yi : fy[q];
                const double r = (-cx * (e - w) - cy * (n - s)) - rc[(2 * NV + q) * es];
                v[q] = fin(z, q, r);
                out[z + q] = v[q];
            }
        } else {
            const double sxs = east ? -cx : cx, sys = north ? -cy : cy;
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                v[q] = (v[q] + sxs * fx[q]) + sys * fy[q];
                out[z + q] = v[q];
            }
        }
        if (ZP) zpeer_store(a, p, z - size_t(p + a.gh) * a.my_pad * a.pitch, v);
        dloc = cfl(v, i, j);
    }
    if (RK && !a.want_dt) return;
    __shared__ double red[4];
    const int t = threadIdx.x;
    dloc = warp_min(dloc);
    if ((t & 31) == 0) red[t >> 5] = dloc;
    __syncthreads();
    if (t == 0) {
        atomic_min_pos_sparse(&a.ctl->acc, smin(smin(red[0], red[1]), smin(red[2], red[3])));
        if (a.fold_adv) {  // the last CTA to finish runs the step's advance (k_advance)
            __threadfence();
            const unsigned total = gridDim.x * gridDim.y;
            if (atomicAdd(&a.ctl->blocks, 1u) == total - 1) {
                __threadfence();
                a.ctl->blocks = 0;
                advance_ctl(a.ctl, a.eb, a.flip);
            }
        }
    }
}

}  // namespace HC_FUSED_NS
}  // namespace hc
