// FMA-contracted instantiation of the fused step (compiled with --fmad=true), with the
// one-division WENO3 weights (fused_ader.cuh weno3_1div). Tolerance-tested, not bit-exact.
#define HC_FUSED_NS fast
#define HC_REASSOC 1
#define HC_FUSED_LAUNCHER launch_fused_fast
#define HC_SEAM_LAUNCHER launch_seam_fast
#include "fused_launch.cuh"
