// fused_types.cuh -- host/device structs shared by the fused stepper kernels and their host
// driver (stepper.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace hc {

// Device-resident time control: the dt/dt_next hand-off of harness.cpp:155-170.
struct StepCtl {
    double dt;       // dt of the step about to run
    double t;        // time at the start of that step
    double t_final;  // <= 0: fixed step count
    double acc;      // min-reduction accumulator of this step's dt_next (seed 1.0e32)
    double dt_next;  // last completed step's dt_next (after any all-reduce)
    long long steps;
    int done;  // 1: t_final reached, 2: a step failed (unphysical); later steps are no-ops
    int cur;   // which of the two state buffers holds the current state
    unsigned blocks;  // CTAs of a launch that folds the advance in, finished so far (else 0)
};

// The end-of-step hand-off (harness.cpp:155-170): error check, t += dt, dt <- dt_next (clipped
// at t_final), the buffer flip. k_advance runs it as its own launch; a seam step folds it into
// the last CTA of seam_fix_kernel.
__device__ __forceinline__ void advance_ctl(StepCtl* c, const ErrBlock* eb, int flip) {
    if (c->done) return;
    for (int s = 0; s < ST_COUNT; ++s)
        if (eb->rec[s].flag) {  // the reference would have thrown out of this step
            c->done = 2;
            return;
        }
    c->t = c->t + c->dt;  // harness.cpp:167-168
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
    if (flip) c->cur ^= 1;  // ADER wrote the other buffer; RK stages end in buffer cur
}

struct FusedArgs {
    double* buf[3];  // state buffers; ctl->cur holds the start-of-step state
    int nbuf;        // 2 (ADER, RK2) or 3 (SSP-RK3)
    int in_rel;      // this launch reads buf[(cur + in_rel) % nbuf]
    int out_rel;     // and writes buf[(cur + out_rel) % nbuf]
    int want_dt;     // take the CFL estimate (ADER: always; RK: last stage)
    int bulk;        // plane loads by bulk copy (set by the launcher)
    int interleave;  // ring kernel: tile and ring E-columns mixed on every warp (launcher)
    double rk_a, rk_b;  // RK stage coefficients U' = a U0 + b (U + dt rate)
    int nx, ny, nz;  // active zones of this patch / slab
    int gh;          // storage ghost width
    int my_pad;      // rows per plane in storage
    int pitch;       // doubles per row in storage
    int tz;          // planes per CTA chunk
    int kz_first;    // active planes [kz_first, kz_last) updated by this launch
    int kz_last;
    double dx, dy, dz, idx, idy, idz;
    double gamma, cfl;
    Limiter lim;
    StepCtl* ctl;
    ErrBlock* eb;
    // z peer stores (hc_stepper_set_zpeer; zstore = 1): the final update of the gh lowest /
    // highest active planes is also written, by the thread that computed it, into the top /
    // bottom ghost planes of the z neighbours' buffers -- device pointers on any GPU this one
    // can reach (NVLink peer memory), same layout, buffer index = this launch's output index
    double* zlo[3];
    double* zhi[3];
    int zstore;
    // 1: the launch closes the step and folds the advance in (flip = ADER's buffer flip)
    int fold_adv, flip;
};

// The peer store of one finished zone of active plane kz (in-plane storage offset `inplane`).
// Not inlined: a call on the rare boundary-plane path keeps the fused kernels' register
// allocation as it is without peer stores (inlined, the headline lost 0.7 %).
// (The seam kernels take it as a template switch, instantiated twice, so the kernels of a
// stepper without peer stores carry no trace of it: even an untaken inlined branch cost the
// headline 0.7 %, an out-of-line call 3.7 %. Ring-kernel steppers get k_zpeer_planes.)
__device__ __forceinline__ void zpeer_store(const FusedArgs& a, int kz, size_t inplane,
                                            const double* v) {
    const int ob = (a.ctl->cur + a.out_rel) % a.nbuf;
    const size_t ps = size_t(a.my_pad) * a.pitch;
    if (kz < a.gh && a.zlo[ob]) {  // -> the lower neighbour's top ghost plane gh + nz + kz
        double* d = a.zlo[ob] + size_t(a.gh + a.nz + kz) * ps + inplane;
#pragma unroll
        for (int q = 0; q < NV; ++q) d[q] = v[q];
    }
    if (kz >= a.nz - a.gh && a.zhi[ob]) {  // -> the upper neighbour's bottom ghost plane
        double* d = a.zhi[ob] + size_t(kz - a.nz + a.gh) * ps + inplane;
#pragma unroll
        for (int q = 0; q < NV; ++q) d[q] = v[q];
    }
}

// Tile shape per order (columns x rows of owned zones per CTA).
// Tile shape per order (columns x rows of owned zones per CTA), from the r1 sweep on a B200
// (profiles/r1_tile_sweep.txt): O3 16x12 with 2 CTAs/SM (256 threads, 128 registers,
// 16 warps/SM) beats 16x8 (12 warps, 168 registers) by 6 %; O2 keeps 16x8.
template <bool O3>
struct FusedTile {
    static constexpr int TX = 16;
    static constexpr int TY = O3 ? 12 : 8;
    static constexpr int MINB = 2;  // resident CTAs per SM the registers must allow
};

// ---- the persistent ring-free kernel's exchange (fused_persist.cuh)
// One exchanged face state or face flux (5 doubles), on its own 64-byte line.
struct alignas(64) XRec {
    double v[NV];
};

struct PersistHdr {
    unsigned long long epoch;  // launches so far (+1): the high bits of every sequence number
    unsigned int done;         // CTAs finished in the current launch
    unsigned int timeout;      // a neighbour wait gave up (reported by the host)
};

constexpr int PX_TX = 32;   // tile width: one warp per tile row
constexpr int PX_TYM = 7;   // rows per tile at most
constexpr int PX_SLOTS = 4;  // exchange slots (plane p uses slot p % 4)
// exchange records per tile and slot: +x states of the east column, +y states of the north
// row, west boundary fluxes, south boundary fluxes
constexpr int PX_XS = 0, PX_YS = PX_TYM, PX_XF = PX_TYM + PX_TX, PX_YF = 2 * PX_TYM + PX_TX;
constexpr int PX_REC = 2 * (PX_TYM + PX_TX);
constexpr int PX_FLAG_STRIDE = 16;  // u64 per flag: one 128-byte line each
// per-thread carried values of the edge zones (global scratch, read back by the same thread):
// fluxes W, E, S, N of the last two planes, bottom z flux of the last two planes, the
// zone's -x and -y face states of the last two planes
constexpr int PX_SCR_FL = 0, PX_SCR_FZ = 40, PX_SCR_MX = 50, PX_SCR_MY = 60, PX_SCR = 70;

struct PersistArgs {
    XRec* rec;                // [tile][slot][PX_REC]
    unsigned long long* flag;  // [tile][row] x PX_FLAG_STRIDE: last plane the row published
    double* scr;              // [tile][thread][PX_SCR]
    PersistHdr* hdr;
    const CUtensorMap* maps;  // [3] in device memory: one TMA map per state buffer
    int ntx, nty;             // tiles along x (nx / 32) and y
};

struct PersistLaunch {
    PersistArgs args;
};

// TMA box of one plane for the persistent kernel: (32 + 2 gh) zones x 5 doubles, 7 + 2R rows
inline int px_box_w(int order) { return PX_TX + 2 * (order >= 3 ? 3 : 2); }
inline int px_box_h(int order) { return PX_TYM + 2 * (order >= 3 ? 2 : 1); }

// ---- the ring-free seam kernel (fused_seam.cuh, both builds): 32 x <=8 tiles, tile-boundary
// faces finished by seam_fix_kernel from the edge zones' published states
constexpr int SEAM_TX = 32, SEAM_TYM = 8;
struct SeamArgs {
    const CUtensorMap* maps;  // [nbuf] in device memory: one TMA map per state buffer
    double* sx;               // [nz][ntx][ny][2][5] states at the x seams (x = 32 sx)
    double* sy;               // [nz][nty][nx][2][5] states at the y seams
    int ntx, nty;             // tiles along x (nx / 32) and y (ceil(ny / 8), balanced rows)
    int nx, ny;
    // bit-exact build only: the edge zones' rate parts, 3 x 5 per zone (x part, y part, z
    // term; see fused_seam.cuh), for the y-edge rows [nz][nty][2][15][nx] and the x-edge
    // columns of the other rows [nz][ntx][2][15][ny]
    double* ey;
    double* ex;
};
// Both kernels of one seam step (or RK stage) over a.kz_first..a.kz_last; blocks_per_sm !=
// nullptr: only report the fused kernel's resident CTAs per SM.
int launch_seam_fast(const FusedArgs& a, const SeamArgs& s, int order, int solver, bool rk,
                     cudaStream_t st, int* blocks_per_sm = nullptr);
// the same pair in the bit-exact build (reference association of the rate, --fmad=false)
int launch_seam_exact(const FusedArgs& a, const SeamArgs& s, int order, int solver, bool rk,
                      cudaStream_t st, int* blocks_per_sm = nullptr);

// pl == nullptr: the ring kernel (fused_ader.cuh); else the persistent ring-free kernel
// (fused_persist.cuh) with these exchange buffers and tensor maps. persist_blocks_per_sm !=
// nullptr: only report the persistent kernel's resident CTAs per SM.
int launch_fused_exact(const FusedArgs& a, int order, int solver, bool rk, cudaStream_t st,
                       const PersistLaunch* pl = nullptr, int* persist_blocks_per_sm = nullptr);
int launch_fused_fast(const FusedArgs& a, int order, int solver, bool rk, cudaStream_t st,
                      const PersistLaunch* pl = nullptr, int* persist_blocks_per_sm = nullptr);

}  // namespace hc
