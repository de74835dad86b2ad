// fused_types.cuh -- host/device structs shared by the fused stepper kernels and their host
// driver (stepper.cu).
#pragma once

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
};

struct FusedArgs {
    double* buf[3];  // state buffers; ctl->cur holds the start-of-step state
    int nbuf;        // 2 (ADER, RK2) or 3 (SSP-RK3)
    int in_rel;      // this launch reads buf[(cur + in_rel) % nbuf]
    int out_rel;     // and writes buf[(cur + out_rel) % nbuf]
    int want_dt;     // take the CFL estimate (ADER: always; RK: last stage)
    int bulk;        // plane loads by bulk copy (set by the launcher)
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
};

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

int launch_fused_exact(const FusedArgs& a, int order, int solver, bool rk, cudaStream_t st);
int launch_fused_fast(const FusedArgs& a, int order, int solver, bool rk, cudaStream_t st);

}  // namespace hc
