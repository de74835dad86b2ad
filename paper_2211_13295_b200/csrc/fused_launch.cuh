// fused_launch.cuh -- instantiates and launches fused_ader_kernel. Included by two
// translation units built with different contraction policies:
//   fused_exact.cu  (--fmad=false): bit-identical to the reference's -ffp-contract=off build
//   fused_fast.cu   (--fmad=true):  DFMA-contracted, <= 1e-13 relative drift (tests state it)
#pragma once

#include "fused_ader.cuh"

namespace hc {
namespace HC_FUSED_NS {

template <bool O3, int SOLVER>
static int launch_one(const FusedArgs& a, cudaStream_t st) {
    using T = FusedTile<O3>;
    using S = FusedShape<O3, T::TX, T::TY>;
    auto kern = fused_ader_kernel<O3, SOLVER, T::TX, T::TY, T::MINB>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(fused)");
        configured = true;
    }
    dim3 grid((a.nx + T::TX - 1) / T::TX, (a.ny + T::TY - 1) / T::TY, (a.kz_last - a.kz_first + a.tz - 1) / a.tz);
    kern<<<grid, S::NT, S::SMEM, st>>>(a);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "fused_ader_kernel launch");
}

}  // namespace HC_FUSED_NS

int HC_FUSED_LAUNCHER(const FusedArgs& a, int order, int solver, cudaStream_t st) {
    using namespace HC_FUSED_NS;
    if (order == 2) return solver == 0 ? launch_one<false, 0>(a, st) : launch_one<false, 1>(a, st);
    return solver == 0 ? launch_one<true, 0>(a, st) : launch_one<true, 1>(a, st);
}

}  // namespace hc
