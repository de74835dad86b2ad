// ct_common.cuh -- shared pieces of the constrained-transport extensions (mhd.cu, ced.cu):
// the padded SoA box (one [mz+1][my+1][mx+1] plane stack per variable, face fields on the
// low face of the zone with the same index), ghost index maps, and the cell average of a
// face-centred field.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace hc {
namespace ct {

struct Box {
    int n[3];      // active zones per axis
    int gh;        // ghost width
    int P, Q, R;   // padded extents (mx+1, my+1, mz+1)
    size_t N;      // P*Q*R
};

__device__ __forceinline__ size_t at(const Box& b, int k, int j, int i) {
    return (size_t(k) * b.Q + j) * b.P + i;
}
__device__ __forceinline__ size_t stride(const Box& b, int axis) {
    return axis == 0 ? size_t(1) : (axis == 1 ? size_t(b.P) : size_t(b.P) * b.Q);
}

// composed ghost image of coordinate c on [lo, hi): kind 0 periodic, 1 outflow (clamp)
__device__ __forceinline__ int map_c(int c, int lo, int hi, int kind) {
    if (c >= lo && c < hi) return c;
    const int n = hi - lo;
    if (kind == 0) return lo + (((c - lo) % n) + n) % n;
    return c < lo ? lo : hi - 1;
}

// Cell average of a face-centred field s (faces o and o+st of the zone): the mean of the
// pair at order 2; at order 3 the fourth-order average
//   1/2 (b[-1/2] + b[+1/2]) - 1/24 (b[+3/2] - b[+1/2] - b[-1/2] + b[-3/2])
// (the trapezoid's h^2/8 f'' error reduced to the average's h^2/24 f''; with the plain mean
// the face fields converge at second order only)
template <bool O3>
__device__ __forceinline__ double face_avg(const double* s, size_t o, size_t st) {
    const double b0 = s[o], b1 = s[o + st];
    double c = 0.5 * (b0 + b1);
    if (O3) c = c - (1.0 / 24.0) * (((s[o + 2 * st] - b1) - b0) + s[o - st]);
    return c;
}

inline unsigned blocks(size_t n, int tpb) { return unsigned((n + tpb - 1) / tpb); }

}  // namespace ct
}  // namespace hc
