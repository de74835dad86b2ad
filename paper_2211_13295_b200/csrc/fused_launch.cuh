// fused_launch.cuh -- instantiates and launches fused_ader_kernel. Included by two
// translation units built with different contraction policies:
//   fused_exact.cu  (--fmad=false): bit-identical to the reference's -ffp-contract=off build
//   fused_fast.cu   (--fmad=true):  DFMA-contracted, <= 1e-12 relative drift (tests state it)
// Tile shapes other than FusedTile's defaults are compiled only with -DHC_TUNE (tuning
// builds) and picked with the HC_FUSED_CFG environment variable.
#pragma once

#include <cstdlib>

#include "fused_persist.cuh"
#include "fused_seam.cuh"

namespace hc {
namespace HC_FUSED_NS {

template <int ORD, int SOLVER, int TX, int TY, int MINB, bool RK>
static int launch_cfg(const FusedArgs& a, cudaStream_t st) {
    using S = FusedShape<(ORD >= 3), TX, TY>;
    auto kern = fused_ader_kernel<ORD, SOLVER, TX, TY, MINB, RK>;
    // the shared-memory opt-in is a per-device attribute: one bit per device ordinal
    static unsigned long long configured = 0;
    int dev = 0;
    cudaError_t de = cudaGetDevice(&dev);
    if (de != cudaSuccess) return cuda_fail(de, "cudaGetDevice");
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(fused)");
        __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
    }
    // bulk-copy plane loads need 16-byte aligned rows: halo G == storage ghost width (tile
    // origins at multiples of TX, TX + 2G even) and an even row pitch; else per-8-byte cp.async
    FusedArgs b = a;
    b.bulk = (a.gh == S::G && (a.pitch & 1) == 0) ? 1 : 0;
    static const int inter = [] {
        const char* v = std::getenv("HC_INTERLEAVE");
        return v ? std::atoi(v) : 0;
    }();
    constexpr int NW = S::NT / 32;
    b.interleave = (inter && (TX * TY) % NW == 0 && (S::NE - TX * TY) % NW == 0) ? 1 : 0;
    // an empty plane range only configures the kernel (loads its module, sets the shared-
    // memory opt-in): the stepper does this at creation, outside any timed loop
    if (a.kz_last <= a.kz_first) return HC_OK;
    dim3 grid((a.nx + TX - 1) / TX, (a.ny + TY - 1) / TY,
              (a.kz_last - a.kz_first + a.tz - 1) / a.tz);
    kern<<<grid, S::NT, S::SMEM, st>>>(b);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "fused_ader_kernel launch");
}

template <int ORD, int SOLVER, bool RK>
static int launch_one(const FusedArgs& a, cudaStream_t st) {
    using T = FusedTile<(ORD >= 3)>;
#ifdef HC_TUNE
    static const int cfg = [] {
        const char* v = std::getenv("HC_FUSED_CFG");
        return v ? std::atoi(v) : 0;
    }();
    if (SOLVER == 1) {
        switch (cfg) {
            case 1: return launch_cfg<ORD, SOLVER, 16, 8, 2, RK>(a, st);
            case 2: return launch_cfg<ORD, SOLVER, 16, 12, 2, RK>(a, st);
            case 3: return launch_cfg<ORD, SOLVER, 24, 8, 2, RK>(a, st);
            case 4: return launch_cfg<ORD, SOLVER, 32, 16, 1, RK>(a, st);
            case 5: return launch_cfg<ORD, SOLVER, 16, 8, 3, RK>(a, st);
            default: break;
        }
    }
#endif
    return launch_cfg<ORD, SOLVER, T::TX, T::TY, T::MINB, RK>(a, st);
}

// The ring-free persistent kernel (fused_persist.cuh). blocks_per_sm != nullptr: only report
// how many of its CTAs fit on one SM (the launcher's co-residency check), no launch.
template <int ORD, int SOLVER, bool RK>
static int persist_one(const FusedArgs& a, const PersistLaunch* pl, cudaStream_t st,
                       int* blocks_per_sm) {
    using S = PersistShape<ORD>;
    auto kern = persist_ader_kernel<ORD, SOLVER, RK>;
    static unsigned long long configured = 0;  // per device, as launch_cfg
    int dev = 0;
    cudaError_t de = cudaGetDevice(&dev);
    if (de != cudaSuccess) return cuda_fail(de, "cudaGetDevice");
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(persist)");
        __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
    }
    if (blocks_per_sm) {
        cudaError_t e =
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kern, S::NT, S::SMEM);
        return e == cudaSuccess ? HC_OK : cuda_fail(e, "occupancy(persist)");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(pl->args.ntx), unsigned(pl->args.nty), 1);
    cfg.blockDim = dim3(S::NT, 1, 1);
    cfg.dynamicSmemBytes = S::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: they wait on each other
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, pl->args);
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "persist_ader_kernel launch");
}

template <int ORD, bool RK>
static int launch_solver(const FusedArgs& a, int solver, cudaStream_t st, const PersistLaunch* pl,
                         int* bps) {
    if (pl || bps) {
        switch (solver) {
            case 0: return persist_one<ORD, 0, RK>(a, pl, st, bps);
            case 1: return persist_one<ORD, 1, RK>(a, pl, st, bps);
            case 2: return persist_one<ORD, 2, RK>(a, pl, st, bps);
            default: return persist_one<ORD, 3, RK>(a, pl, st, bps);
        }
    }
    switch (solver) {
        case 0: return launch_one<ORD, 0, RK>(a, st);
        case 1: return launch_one<ORD, 1, RK>(a, st);
        case 2: return launch_one<ORD, 2, RK>(a, st);  // HLLC (extension)
        default: return launch_one<ORD, 3, RK>(a, st);  // HLLI (extension)
    }
}

template <int ORD, int SOLVER, bool RK, bool ZP>
static int seam_one(const FusedArgs& a, const SeamArgs& sa, cudaStream_t st, int* blocks_per_sm) {
    using S = SeamShape<ORD>;
    auto kern = seam_ader_kernel<ORD, SOLVER, RK, ZP>;
    static unsigned long long configured = 0;  // per device, as launch_cfg
    int dev = 0;
    cudaError_t de = cudaGetDevice(&dev);
    if (de != cudaSuccess) return cuda_fail(de, "cudaGetDevice");
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(seam)");
        __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
    }
    if (blocks_per_sm) {
        cudaError_t e =
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kern, S::NT, S::SMEM);
        return e == cudaSuccess ? HC_OK : cuda_fail(e, "occupancy(seam)");
    }
    const int nplanes = a.kz_last - a.kz_first;
    if (nplanes <= 0) return HC_OK;
    dim3 grid(unsigned(sa.ntx), unsigned(sa.nty), unsigned((nplanes + a.tz - 1) / a.tz));
    kern<<<grid, S::NT, S::SMEM, st>>>(a, sa);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "seam_ader_kernel launch");
    // per plane: y-seam faces, x-seam faces, tile-corner zones (one launch, disjoint zones)
    const unsigned nby = unsigned(sa.nty * sa.nx + 127) / 128, nbx = unsigned(sa.ntx * sa.ny + 127) / 128,
                   nbc = unsigned(4 * sa.ntx * sa.nty + 127) / 128;
    seam_fix_kernel<SOLVER, RK, ZP><<<dim3(nby + nbx + nbc, unsigned(nplanes)), 128, 0, st>>>(a, sa);
    e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "seam_fix_kernel launch");
}

template <int ORD, bool RK>
static int seam_solver(const FusedArgs& a, const SeamArgs& sa, int solver, cudaStream_t st,
                       int* bps) {
    switch (solver) {
        case 0: return a.zstore ? seam_one<ORD, 0, RK, true>(a, sa, st, bps)
                           : seam_one<ORD, 0, RK, false>(a, sa, st, bps);
        case 1: return a.zstore ? seam_one<ORD, 1, RK, true>(a, sa, st, bps)
                           : seam_one<ORD, 1, RK, false>(a, sa, st, bps);
        case 2: return a.zstore ? seam_one<ORD, 2, RK, true>(a, sa, st, bps)
                           : seam_one<ORD, 2, RK, false>(a, sa, st, bps);
        default: return a.zstore ? seam_one<ORD, 3, RK, true>(a, sa, st, bps)
                         : seam_one<ORD, 3, RK, false>(a, sa, st, bps);
    }
}

}  // namespace HC_FUSED_NS

int HC_SEAM_LAUNCHER(const FusedArgs& a, const SeamArgs& sa, int order, int solver, bool rk,
                     cudaStream_t st, int* blocks_per_sm) {
    using namespace HC_FUSED_NS;
    if (rk) {
        if (order == 2) return seam_solver<2, true>(a, sa, solver, st, blocks_per_sm);
        return order == 3 ? seam_solver<3, true>(a, sa, solver, st, blocks_per_sm)
                          : seam_solver<4, true>(a, sa, solver, st, blocks_per_sm);
    }
    if (order == 2) return seam_solver<2, false>(a, sa, solver, st, blocks_per_sm);
    return order == 3 ? seam_solver<3, false>(a, sa, solver, st, blocks_per_sm)
                      : seam_solver<4, false>(a, sa, solver, st, blocks_per_sm);
}

int HC_FUSED_LAUNCHER(const FusedArgs& a, int order, int solver, bool rk, cudaStream_t st,
                      const PersistLaunch* pl, int* persist_blocks_per_sm) {
    using namespace HC_FUSED_NS;
    int* b = persist_blocks_per_sm;
    if (rk) {
        if (order == 2) return launch_solver<2, true>(a, solver, st, pl, b);
        return order == 3 ? launch_solver<3, true>(a, solver, st, pl, b)
                          : launch_solver<4, true>(a, solver, st, pl, b);
    }
    if (order == 2) return launch_solver<2, false>(a, solver, st, pl, b);
    return order == 3 ? launch_solver<3, false>(a, solver, st, pl, b)
                      : launch_solver<4, false>(a, solver, st, pl, b);
}

}  // namespace hc
