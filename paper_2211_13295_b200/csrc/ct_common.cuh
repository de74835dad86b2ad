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
// Zones of the padded box outside the active cell box [gh, gh+n)^3 (the ghost shell every
// ghost of every variable lies in): count, and the r-th one (z slabs, then y rows of the
// active planes, then x columns of the active rows). Ghost fills launch over this shell only.
__host__ __device__ __forceinline__ size_t shell_count(const Box& b) {
    const size_t nx = b.n[0], ny = b.n[1], nz = b.n[2];
    return size_t(b.R - nz) * b.P * b.Q + nz * (b.Q - ny) * b.P + nz * ny * (b.P - nx);
}
__device__ __forceinline__ bool shell_zone(const Box& b, size_t r, int& i, int& j, int& k) {
    const int nx = b.n[0], ny = b.n[1], nz = b.n[2], g = b.gh;
    const size_t PQ = size_t(b.P) * b.Q;
    const size_t zc = size_t(b.R - nz) * PQ;
    if (r < zc) {
        const int kk = int(r / PQ);
        const size_t rem = r % PQ;
        k = kk < g ? kk : kk + nz;
        j = int(rem / b.P);
        i = int(rem % b.P);
        return true;
    }
    r -= zc;
    const size_t yp = size_t(b.Q - ny) * b.P, yc = size_t(nz) * yp;
    if (r < yc) {
        k = g + int(r / yp);
        const size_t rem = r % yp;
        const int jj = int(rem / b.P);
        j = jj < g ? jj : jj + ny;
        i = int(rem % b.P);
        return true;
    }
    r -= yc;
    const size_t xp = size_t(b.P - nx), xr = size_t(ny) * xp;
    if (r >= size_t(nz) * xr) return false;
    k = g + int(r / xr);
    const size_t rem = r % xr;
    j = g + int(rem / xp);
    const int ii = int(rem % xp);
    i = ii < g ? ii : ii + nx;
    return true;
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
