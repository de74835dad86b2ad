// Bit-exact instantiation of the fused step (compiled with --fmad=false).
#define HC_FUSED_NS exact
#define HC_FUSED_LAUNCHER launch_fused_exact
#define HC_SEAM_LAUNCHER launch_seam_exact
#include "fused_launch.cuh"
