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
    double* buf[2];  // ping-pong state buffers; ctl->cur selects the input
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
template <bool O3>
struct FusedTile {
    static constexpr int TX = 16;
    static constexpr int TY = 8;
    static constexpr int MINB = 2;  // resident CTAs per SM the registers must allow
};

int launch_fused_exact(const FusedArgs& a, int order, int solver, cudaStream_t st);
int launch_fused_fast(const FusedArgs& a, int order, int solver, cudaStream_t st);

}  // namespace hc
