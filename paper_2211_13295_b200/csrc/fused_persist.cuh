// fused_persist.cuh -- the ring-free fused ADER step: one persistent CTA per column tile,
// every CTA resident at once (cooperative launch), tile-boundary faces exchanged with the
// four neighbouring CTAs through L2.
//
// Same update as fused_ader.cuh (reconstruction -> ADER predictor -> face Riemann fluxes ->
// flux differencing -> update -> CFL min; stepper.cpp:49-78, predictor.cpp:26-91,
// corrector.cpp:15-125) with the same per-zone arithmetic (zone_states, face_flux, the
// reference's association of the rate), so results are bit-identical to it in the exact
// build. What changes is who computes what:
//
//  * No ring columns. fused_ader.cuh re-runs reconstruction + predictor on a one-zone ring
//    around each tile (predictor.cpp:68-70's "active + one ring"; 1.29x the owned zones at
//    16 x 12) and keeps two warps of ring threads that idle through the face phases. Here a
//    CTA owns a 32 x h tile (h <= 7; one warp per tile row, one thread per zone) for the WHOLE
//    z extent of the launch, and every zone's face states are computed exactly once, by its
//    owner. Across a tile boundary the owner of the west (south) zone publishes its +x (+y)
//    face state to a small per-tile exchange area in global memory (L2-resident, 2 plane
//    slots); the east (north) tile solves the boundary face as its own west (south) face and
//    publishes that face's flux back. The flux is consumed one plane later, when the
//    boundary zone is finalised, so its latency hides behind a whole predict phase.
//  * x neighbours live in the same warp: the -x side state of a face and the east face's
//    flux travel by warp shuffles, not shared memory.
//  * Planes arrive by TMA tensor copies (cp.async.bulk.tensor.3d: one copy of an
//    (h + 2R) x (32 + 2R) x 5 box per plane, completion on a per-slot mbarrier).
//
// One plane of slack between neighbours: the boundary faces of plane p-1 are solved in the
// face phase of plane p (in the same warp instruction stream as plane p's interior faces: lane
// 0 / row 0 simply take different inputs), and a zone on a tile edge is finalised two planes
// back (its east / north flux arrives from the neighbour one plane after that neighbour
// solved it). A CTA therefore waits only when a neighbour is more than about a plane behind.
// Each tile row (warp) publishes once per plane: its exchange records, one fence, then its
// flag (the sequence number epoch << 20 | plane). Records use 4 plane slots: a slot is
// rewritten 4 planes later, after the writer has seen (through the flags it waits on) that
// the reader is past the plane that reads it. All CTAs must be co-resident
// (they wait on each other): the launcher checks occupancy and launches with the cooperative
// attribute; a waiting thread gives up after 2 s and flags the header (the host reports it)
// instead of hanging the device.
#pragma once

#include "fused_ader.cuh"

namespace hc {

namespace HC_FUSED_NS {

template <int ORD>
struct PersistShape {
    static constexpr bool O3 = ORD >= 3;
    static constexpr int TX = PX_TX, TYM = PX_TYM;
    static constexpr int R = O3 ? 2 : 1;
    // planes in flight: p-R..p+R for the stencils, and p-2 for the edge zones finalised two
    // planes back (the refill of p+R+1 takes the slot of p+R+1-NB)
    static constexpr int NB = 2 * R + 1 > 4 ? 2 * R + 1 : 4;
    // x halo = the storage ghost width (3 at O3, 2 at O2), one more than the stencil needs at
    // O3: a TMA box must start on a 16-byte boundary in its innermost dimension, and a 40-byte
    // zone at an odd index does not
    static constexpr int HX = O3 ? 3 : 2;
    static constexpr int W = TX + 2 * HX;
    static constexpr int H = TYM + 2 * R;
    static constexpr int BOX = W * H * NV;                // doubles one TMA box writes
    static constexpr int PLANE = (BOX + 15) / 16 * 16;    // slot stride: 128-byte aligned
    static constexpr int NT = TX * TYM;
    static constexpr int YPF = TYM * TX * NV;  // +y states (rows 1..h-1) / y fluxes
    static constexpr size_t SMEM =
        sizeof(double) * (size_t(NB) * PLANE + YPF + 2 * NV * NT + 24);
};

__device__ __forceinline__ unsigned long long px_ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void px_st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long px_clock_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Waits until a neighbour row's flag reaches seq (acquire: its records are then visible).
__device__ __noinline__ void px_spin(const unsigned long long* f, unsigned long long seq,
                                     PersistHdr* hdr) {
    const unsigned long long t0 = px_clock_ns();
    while (px_ld_acquire(f) < seq) {
        __nanosleep(64);
        if (px_clock_ns() - t0 > 2000000000ull) {  // a neighbour never came: report, do not hang
            atomicExch(&hdr->timeout, 1u);
            return;
        }
    }
}
__device__ __forceinline__ void px_wait(const unsigned long long* f, unsigned long long seq,
                                        PersistHdr* hdr) {
    if (px_ld_acquire(f) < seq) px_spin(f, seq, hdr);
}

__device__ __forceinline__ void px_put(XRec* r, const double* v) {
#pragma unroll
    for (int q = 0; q < NV; ++q) __stcg(&r->v[q], v[q]);
}
__device__ __forceinline__ void px_get(const XRec* r, double* v) {
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = __ldcg(&r->v[q]);
}

__device__ __forceinline__ void tma_load_plane(void* dst, const CUtensorMap* map, int c0, int c1,
                                               int c2, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2),
        "r"(smem_u32(bar))
        : "memory");
}

// The x/y rate terms of a zone in the reference's association (corrector.cpp:89-90):
// -cx*(E - W) - cy*(N - S).
__device__ __forceinline__ double rate_xy(double cx, double cy, double e, double w, double n,
                                          double s) {
    return -cx * (e - w) - cy * (n - s);
}

// The plane loop, lp = -1 .. nzc + 1 (p = kz_first + lp):
//  A  predict(p) for lp <= nzc (the z-ring planes -1 and nzc included): face states in
//     registers, +y states to YPF, east column / north row states into the exchange records
//  B  z face at the bottom of p (0 <= lp <= nzc); finalise p-1 for inner zones (lp >= 1) and
//     p-2 for edge zones (lp >= 2), with the neighbours' boundary fluxes of p-2
//  C  faces (lp in [0, nzc] minus the ring): interior x / y faces of p; lane 0 / row 0 solve
//     the west / south boundary face of p-1 instead (the neighbour's published state of p-1,
//     this zone's own -x / -y state of p-1 from scratch)
//  P  each row publishes: one fence, then its flag = seq(p)
//  D  rate(p) for inner zones; edge zones park the fluxes known so far
template <int ORD, int SOLVER, bool RK>
__global__ void __launch_bounds__(PersistShape<ORD>::NT, 2)
    persist_ader_kernel(const __grid_constant__ FusedArgs a, const PersistArgs px) {
    using S = PersistShape<ORD>;
    constexpr int R = S::R, NB = S::NB, W = S::W, TX = S::TX;
    if (a.ctl->done) return;
    __shared__ double* sbuf[3];
    __shared__ const CUtensorMap* smap;
    __shared__ unsigned long long mbar[NB];
    __shared__ unsigned long long s_epoch;
    __shared__ int s_tile[8];  // h, y0, this tile, W, E, S, N, the S tile's height
    if (threadIdx.x == 0) {
        const int bx = blockIdx.x, by = blockIdx.y, base = a.ny / px.nty, rem = a.ny % px.nty;
        const int bS = (by + px.nty - 1) % px.nty, bN = (by + 1) % px.nty;
        s_tile[0] = base + (by < rem ? 1 : 0);
        s_tile[1] = by * base + min(by, rem);
        s_tile[2] = by * px.ntx + bx;
        s_tile[3] = by * px.ntx + (bx + px.ntx - 1) % px.ntx;
        s_tile[4] = by * px.ntx + (bx + 1) % px.ntx;
        s_tile[5] = bS * px.ntx + bx;
        s_tile[6] = bN * px.ntx + bx;
        s_tile[7] = base + (bS < rem ? 1 : 0);
        const int cur = a.ctl->cur;
        const int in = (cur + a.in_rel) % a.nbuf;
        sbuf[0] = a.buf[in];
        sbuf[1] = a.buf[(cur + a.out_rel) % a.nbuf];
        sbuf[2] = a.buf[cur];
        smap = px.maps + in;
        s_epoch = px.hdr->epoch;
    }
    extern __shared__ __align__(128) double smem[];
    double* planes = smem;                           // [NB][H][W][5]
    double* YPF = planes + size_t(NB) * S::PLANE;    // [TYM][TX][5]: +y states / south fluxes
    double* part = YPF + S::YPF;                     // [5][NT] x/y rate of plane p
    double* fzp = part + NV * S::NT;                 // [5][NT] bottom z flux of plane p
    double* red = fzp + NV * S::NT;  // [24]: per-warp running CFL minimum [0, 7), dt & c [16, 20)

    // Thread and tile coordinates are recomputed from the special registers where used (cheap
    // S2R reads) rather than held in registers across the predictor, which would spill.
    // tile rows: nty rows of h or h+1 (the first `rem` rows are one taller)
    auto ci_ = [] { return int(threadIdx.x) & 31; };
    auto cj_ = [] { return int(threadIdx.x) >> 5; };
    auto h_ = [&] { return s_tile[0]; };
    auto y0_ = [&] { return s_tile[1]; };
    auto ia_ = [&] { return int(blockIdx.x) * TX + ci_(); };
    auto ja_ = [&] { return y0_() + cj_(); };
    // this tile and its periodic neighbours
    auto tile_ = [&](int dx, int dy) { return s_tile[dx < 0 ? 3 : dx > 0 ? 4 : dy < 0 ? 5 : dy > 0 ? 6 : 2]; };
    auto rec_ = [&](int t, int lp, int k) -> XRec* {
        return px.rec + (size_t(t) * PX_SLOTS + ((lp + 2) & (PX_SLOTS - 1))) * PX_REC + k;
    };
    auto flag_ = [&](int t, int row) -> unsigned long long* {
        return px.flag + (size_t(t) * PX_TYM + row) * PX_FLAG_STRIDE;
    };
    auto scr_ = [&]() -> double* {
        return px.scr + (size_t(s_tile[2]) * S::NT + threadIdx.x) * PX_SCR;
    };
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TX;
    const int kz0 = a.kz_first, nzc = a.kz_last - a.kz_first;
    if (tid == 0) {
        const double dt0 = a.ctl->dt;
        red[16] = dt0 / a.dx;
        red[17] = dt0 / a.dy;
        red[18] = dt0 / a.dz;
        red[19] = dt0;
    }
    if (tid < S::TYM) red[tid] = 1.0e32;
    const size_t plane_stride = size_t(a.my_pad) * a.pitch;
    const int zfirst = kz0 - 1 - R;
    constexpr unsigned PLANE_BYTES = S::BOX * sizeof(double);
    auto load_plane = [&](int zact) {  // one TMA box per plane, issued by thread 0
        if (tid != 0) return;
        const int li = zact - zfirst;
        fence_proxy_async();  // generic-proxy reads of the slot before the async writes
        mbar_arrive_expect_tx(&mbar[li % NB], PLANE_BYTES);
        tma_load_plane(planes + size_t(li % NB) * S::PLANE, smap, (x0 + a.gh - S::HX) * NV,
                       y0_() + a.gh - R, zact + a.gh, &mbar[li % NB]);
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

    const unsigned long long ep = s_epoch << 20;
    constexpr int CS = S::NT;
    double zp_prev[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) zp_prev[q] = 0.0;

    // finalise the zone of this thread on plane pf: U += rate, the RK combination, the CFL
    // estimate (stepper.cpp:49-78, 137; corrector.cpp:94-125)
    auto finalise = [&](int pf, const double* pr, const double* fz_bot, const double* fz_top) {
        const int ia = ia_(), ja = ja_();
        const double* u = P(pf) + zoff_();
        const size_t zi = size_t(pf + a.gh) * plane_stride + size_t(ja + a.gh) * a.pitch +
                          size_t(ia + a.gh) * NV;
        double un[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double r = pr[q] - red[18] * (fz_top[q] - fz_bot[q]);
            if (RK)  // stepper.cpp:137 (u0 read before uout is written: may alias)
                un[q] = a.rk_a * sbuf[2][zi + q] + a.rk_b * (u[q] + r);
            else
                un[q] = u[q] + r;
        }
        double* dst = sbuf[1] + zi;
#pragma unroll
        for (int q = 0; q < NV; ++q) dst[q] = un[q];
        double dloc = 1.0e32;
        if (!RK || a.want_dt) {
            Fault f3;
            f3.clear();
            double d = FM == 2 ? eval_tstep_inv<FM>(un, a.cfl, a.idx, a.idy, a.idz, a.gamma, f3)
                               : eval_tstep<FM>(un, a.cfl, a.dx, a.dy, a.dz, a.gamma, f3);
            if (f3.redo()) {
                V5 u5;
#pragma unroll
                for (int q = 0; q < NV; ++q) u5.v[q] = un[q];
                f3.clear();
                d = eval_tstep_careful(u5, a.cfl, a.dx, a.dy, a.dz, a.gamma, &f3);
            }
            if (f3.code)
                record_fault(a.eb, RK ? ST_DT : ST_UPDATE, f3, ia, ja, pf, 0);
            else
                dloc = d;
        }
        return dloc;
    };

    for (int lp = -1; lp <= nzc + 1; ++lp) {
        const int p = kz0 + lp;
        const unsigned long long seq = ep | unsigned(lp + 2);  // plane lp's sequence number
        __syncthreads();  // the previous plane's reads of YPF (and of the oldest slot) are done
        const bool pred = lp <= nzc;               // A runs (real or z-ring plane)
        const bool real = lp >= 0 && lp < nzc;     // x/y faces of p exist
        if (pred)
            for (int z = p - R; z <= p + R; ++z) wait_plane(z);
        double st[6][NV];  // face states incl. 0.5*tau: E, W, N, S, T, B
        const int h = h_();
        if (cj_() < h) {
            if (pred) {
                // ------------------------------------------------------------ A: predict
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
                if (real) {
                    const int ci = ci_(), cj = cj_();
                    if (cj < h - 1)
#pragma unroll
                        for (int q = 0; q < NV; ++q)
                            YPF[((cj + 1) * TX + ci) * NV + q] = st[2][q];
                    if (ci == TX - 1) px_put(rec_(tile_(0, 0), lp, PX_XS + cj), st[0]);
                    if (cj == h - 1) px_put(rec_(tile_(0, 0), lp, PX_YS + ci), st[2]);
                }
            }
            // ----------------------------------------- B: z face, finalise p-1 / p-2
            if (lp >= 0 && lp <= nzc + 1) {
                const int ci = ci_(), cj = cj_();
                const bool edge = ci == 0 || ci == TX - 1 || cj == 0 || cj == h - 1;
                double* scr = scr_();
                double fz_cur[NV];
                if (pred) {
                    Fault f2;
                    f2.clear();
                    face_flux<SOLVER, 2>(zp_prev, st[5], a.gamma, fz_cur, f2);
                    if (f2.code) record_fault(a.eb, ST_FLUX, f2, p, ia_(), ja_(), 2);
                }
                // one finalise per warp: inner zones take plane p-1 (rate from smem, z fluxes
                // fzp / fz_cur), edge zones plane p-2 (rate from the parked and the neighbours'
                // fluxes, z fluxes from scratch)
                double dloc = 1.0e32;
                const bool fin_in = !edge && lp >= 1 && pred, fin_edge = edge && lp >= 2;
                if (fin_in || fin_edge) {
                    double pr[NV], fb[NV], ft[NV];
                    if (fin_in) {
#pragma unroll
                        for (int q = 0; q < NV; ++q) {
                            pr[q] = part[q * CS + tid];
                            fb[q] = fzp[q * CS + tid];
                            ft[q] = fz_cur[q];
                        }
                    } else {
                        // plane p-2: W and S parked / solved here, E and N from the neighbours
                        const int lq = lp - 2;
                        double* fl = scr + PX_SCR_FL + (lq & 1) * 20;
                        if (ci == TX - 1) {
                            px_wait(flag_(tile_(1, 0), cj), seq - 1, px.hdr);
                            px_get(rec_(tile_(1, 0), lq, PX_XF + cj), fl + NV);
                        }
                        if (cj == h - 1) {
                            px_wait(flag_(tile_(0, 1), 0), seq - 1, px.hdr);
                            px_get(rec_(tile_(0, 1), lq, PX_YF + ci), fl + 3 * NV);
                        }
                        const double cx = red[16], cy = red[17];
#pragma unroll
                        for (int q = 0; q < NV; ++q) {
                            pr[q] = rate_xy(cx, cy, fl[NV + q], fl[q], fl[3 * NV + q],
                                            fl[2 * NV + q]);
                            fb[q] = scr[PX_SCR_FZ + (lq & 1) * NV + q];        // bottom of p-2
                            ft[q] = scr[PX_SCR_FZ + ((lq + 1) & 1) * NV + q];  // bottom of p-1
                        }
                    }
                    dloc = finalise(fin_in ? p - 1 : p - 2, pr, fb, ft);
                }
                if (pred) {
#pragma unroll
                    for (int q = 0; q < NV; ++q) fzp[q * CS + tid] = fz_cur[q];
                    if (edge)  // (the bottom flux of ring plane nzc tops plane nzc - 1)
#pragma unroll
                        for (int q = 0; q < NV; ++q)
                            scr[PX_SCR_FZ + (lp & 1) * NV + q] = fz_cur[q];
#pragma unroll
                    for (int q = 0; q < NV; ++q) zp_prev[q] = st[4][q];
                }
                if ((!RK || a.want_dt) && lp >= 1) {  // running CFL minimum per warp (exact)
                    dloc = warp_min(dloc);
                    if (ci == 0) red[cj] = smin(red[cj], dloc);
                }
            } else if (pred) {
#pragma unroll
                for (int q = 0; q < NV; ++q) zp_prev[q] = st[4][q];
            }
        }
        __syncthreads();  // +y states in YPF; every thread is past its reads of the oldest slot
        if (lp <= nzc - 1) load_plane(p + R + 1);
        if (lp < 0 || lp > nzc) continue;
        // ------------------------------------------------------------------- C: faces
        const int ci = ci_(), cj = cj_();
        const bool act = cj < h;
        const bool bx = ci == 0 && lp >= 1;  // this lane solves the west boundary face of p-1
        const bool by = cj == 0 && lp >= 1;  // this row solves the south boundary face of p-1
        double fw[NV];
        if (act) {  // (whole warps: the shuffles below need every lane)
            double* scr = scr_();
            double ul[NV], ur[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                ul[q] = __shfl_up_sync(0xffffffffu, st[0][q], 1);
                ur[q] = st[1][q];
            }
            if (ci == 0) {
                if (bx) {
                    px_wait(flag_(tile_(-1, 0), cj), seq - 1, px.hdr);
                    px_get(rec_(tile_(-1, 0), lp - 1, PX_XS + cj), ul);
#pragma unroll
                    for (int q = 0; q < NV; ++q) ur[q] = scr[PX_SCR_MX + ((lp - 1) & 1) * NV + q];
                }
                if (real)
#pragma unroll
                    for (int q = 0; q < NV; ++q) scr[PX_SCR_MX + (lp & 1) * NV + q] = st[1][q];
            }
            if ((real && ci > 0) || bx) {
                Fault f;
                f.clear();
                face_flux<SOLVER, 0>(ul, ur, a.gamma, fw, f);
                if (f.code) record_fault(a.eb, ST_FLUX, f, ia_(), ja_(), ci == 0 ? p - 1 : p, 0);
            }
            if (bx) {  // west boundary flux of p-1: parked for this zone, published for W
                px_put(rec_(tile_(0, 0), lp - 1, PX_XF + cj), fw);
#pragma unroll
                for (int q = 0; q < NV; ++q) scr[PX_SCR_FL + ((lp - 1) & 1) * 20 + q] = fw[q];
            }
            // y face at the south of this zone (row 0: the south boundary face of p-1)
            double us[NV], fs[NV];
            if (cj == 0) {
                if (by) {
                    px_wait(flag_(tile_(0, -1), s_tile[7] - 1), seq - 1, px.hdr);
                    px_get(rec_(tile_(0, -1), lp - 1, PX_YS + ci), us);
#pragma unroll
                    for (int q = 0; q < NV; ++q) ur[q] = scr[PX_SCR_MY + ((lp - 1) & 1) * NV + q];
                }
                if (real)
#pragma unroll
                    for (int q = 0; q < NV; ++q) scr[PX_SCR_MY + (lp & 1) * NV + q] = st[3][q];
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    us[q] = YPF[(cj * TX + ci) * NV + q];
                    ur[q] = st[3][q];
                }
            }
            if ((real && cj > 0) || by) {
                Fault f;
                f.clear();
                face_flux<SOLVER, 1>(us, ur, a.gamma, fs, f);
                if (f.code) record_fault(a.eb, ST_FLUX, f, ja_(), ia_(), cj == 0 ? p - 1 : p, 1);
            }
            if (by) {
                px_put(rec_(tile_(0, 0), lp - 1, PX_YF + ci), fs);
#pragma unroll
                for (int q = 0; q < NV; ++q)
                    scr[PX_SCR_FL + ((lp - 1) & 1) * 20 + 2 * NV + q] = fs[q];
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                YPF[(cj * TX + ci) * NV + q] = fs[q];
                part[q * CS + tid] = fw[q];  // parked for the shuffle in D
            }
        }
        // -------------------------------------------------- P: this row publishes plane p
        if (act) {
            __threadfence();  // this warp's records (A: states of p, C: boundary fluxes of p-1)
            __syncwarp();
            if (ci == 0) px_st_relaxed(flag_(tile_(0, 0), cj), seq);
        }
        __syncthreads();  // south fluxes of every row in YPF
        if (!real) continue;
        // --------------------------------------------------------------------- D: rate
        double fe[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            fw[q] = part[q * CS + tid];
            fe[q] = __shfl_down_sync(0xffffffffu, fw[q], 1);  // east face = lane ci+1's west
        }
        if (act) {
            const bool edge = ci == 0 || ci == TX - 1 || cj == 0 || cj == h - 1;
            const double* fsn = YPF + (cj * TX + ci) * NV;  // this zone's south face
            if (!edge) {
                const double cx = red[16], cy = red[17];
#pragma unroll
                for (int q = 0; q < NV; ++q)
                    part[q * CS + tid] = rate_xy(cx, cy, fe[q], fw[q], fsn[TX * NV + q], fsn[q]);
            } else {  // park the fluxes of p known now (W, E, S, N); the rest arrive later
                double* fl = scr_() + PX_SCR_FL + (lp & 1) * 20;
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    if (ci > 0) fl[q] = fw[q];
                    if (ci < TX - 1) fl[NV + q] = fe[q];
                    if (cj > 0) fl[2 * NV + q] = fsn[q];
                    if (cj < h - 1) fl[3 * NV + q] = fsn[TX * NV + q];
                }
            }
        }
    }

    // ---- CFL minimum: block min -> one atomic per CTA; then the launch epoch
    if (!RK || a.want_dt) {
        __syncthreads();
        if (tid < 32) {
            double v = tid < S::TYM ? red[tid] : 1.0e32;
            v = warp_min(v);
            if (tid == 0) atomic_min_pos(&a.ctl->acc, v);
        }
    }
    if (tid == 0) {
        const unsigned total = unsigned(px.ntx * px.nty);
        if (atomicAdd(&px.hdr->done, 1u) == total - 1) {  // the launch's last CTA
            px.hdr->done = 0;
            px.hdr->epoch = px.hdr->epoch + 1;
            __threadfence();
        }
    }
}

}  // namespace HC_FUSED_NS
}  // namespace hc
