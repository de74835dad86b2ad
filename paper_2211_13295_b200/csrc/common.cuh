// common.cuh -- shared device/host plumbing of libhydro_cuda: the C-ABI structs, device
// error records (the GPU replacement for omp_errors.hpp:11-27 ErrorCollector) and the
// thread-local last-error text behind hc_last_error().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/hydro_cuda.h"
#include "pointwise.cuh"

namespace hc {

// Stages, in the order the reference pipeline would raise them (stepper.cpp:49-78).
enum Stage { ST_PREDICT = 0, ST_FLUX = 1, ST_UPDATE = 2, ST_DT = 3, ST_COUNT = 4 };

// One device-side first-failure slot per stage. The first thread to CAS the flag owns the
// slot -- the same "first recorded failure wins" rule as ErrorCollector::record.
struct ErrRec {
    unsigned int flag;
    int code;  // 1 density, 2 pressure
    int a, b, c;
    int axis;
    int pad;
    double val;
};

struct ErrBlock {
    ErrRec rec[ST_COUNT];
};

__device__ __forceinline__ void record_fault(ErrBlock* eb, int stage, const Fault& f, int a,
                                             int b, int c, int axis) {
    ErrRec* r = &eb->rec[stage];
    if (atomicCAS(&r->flag, 0u, 1u) == 0u) {
        r->code = f.code;
        r->a = a;
        r->b = b;
        r->c = c;
        r->axis = axis;
        r->val = f.val;
    }
}

// exact min of positive doubles through their bit patterns (order-independent, so any
// reduction tree gives the serial result)
__device__ __forceinline__ void atomic_min_pos(double* addr, double v) {
    atomicMin(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

// the same, skipping the atomic when the accumulator already holds a value <= v (a plain
// L2 read; a stale read only costs an unneeded atomic): for kernels with many small blocks,
// whose atomics on one address would otherwise serialise
__device__ __forceinline__ void atomic_min_pos_sparse(double* addr, double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    if (b < __ldcg(reinterpret_cast<const unsigned long long*>(addr)))
        atomicMin(reinterpret_cast<unsigned long long*>(addr), b);
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = smin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---- host side
void set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
// Formats the lowest-stage device error like the reference's unphysical_error text and
// stores it as the last error; returns HC_UNPHYSICAL, or HC_OK when no slot is set.
int report_device_errors(const ErrBlock& eb);

#define HC_CUDA(call)                                        \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return ::hc::cuda_fail(e_, #call); \
    } while (0)

inline int mx_of(const hc_geom& g) { return g.nx + 2 * g.ghost; }
inline int my_of(const hc_geom& g) { return g.ny + 2 * g.ghost; }
inline int mz_of(const hc_geom& g) { return g.nz + 2 * g.ghost; }
inline size_t total_zones(const hc_geom& g) {
    return size_t(mx_of(g)) * my_of(g) * mz_of(g);
}
int validate_geom(const hc_geom* g, int order);

}  // namespace hc
