// FMA-contracted instantiation of the fused step (compiled with --fmad=true).
#define HC_FUSED_NS fast
#define HC_FUSED_LAUNCHER launch_fused_fast
#include "fused_launch.cuh"
