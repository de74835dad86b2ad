// capi_common.cu -- library-level C-ABI entry points and host-side error plumbing.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"

namespace hc {

namespace {
thread_local std::string tl_msg;
thread_local int tl_code = HC_OK;
}  // namespace

void set_error(int code, const std::string& msg) {
    tl_code = code;
    tl_msg = msg;
}

int cuda_fail(cudaError_t e, const char* where) {
    set_error(HC_CUDA, std::string("cuda error in ") + where + ": " + cudaGetErrorString(e));
    return HC_CUDA;
}

// std::to_string(double) == "%f"
static std::string fmt_fault(int code, double v) {
    char b[96];
    snprintf(b, sizeof b, "%s %f", code == 1 ? "non-positive density" : "non-positive pressure",
             v);
    return b;
}

int report_device_errors(const ErrBlock& eb) {
    char pre[128];
    for (int s = 0; s < ST_COUNT; ++s) {
        const ErrRec& r = eb.rec[s];
        if (!r.flag) continue;
        switch (s) {
            case ST_PREDICT:  // predictor.cpp:82-84
                snprintf(pre, sizeof pre, "predictor: zone (%d,%d,%d): ", r.a, r.b, r.c);
                break;
            case ST_FLUX:  // corrector.cpp:53-55
                snprintf(pre, sizeof pre, "flux axis %d: face (%d,%d,%d): ", r.axis, r.a, r.b,
                         r.c);
                break;
            case ST_UPDATE:  // corrector.cpp:119-120
                snprintf(pre, sizeof pre, "update: zone (%d,%d,%d): ", r.a, r.b, r.c);
                break;
            default:  // stepper.cpp:41-42
                snprintf(pre, sizeof pre, "dt estimate: zone (%d,%d,%d): ", r.a, r.b, r.c);
                break;
        }
        set_error(HC_UNPHYSICAL, std::string(pre) + fmt_fault(r.code, r.val));
        return HC_UNPHYSICAL;
    }
    return HC_OK;
}

// geometry.hpp:57-64 PatchGeometry::validate, plus the ghost width the order needs
// (geometry.hpp:13-17); order 0 = any.
int validate_geom(const hc_geom* g, int order) {
    if (!g) {
        set_error(HC_INVALID, "null geometry");
        return HC_INVALID;
    }
    if (g->nx < 4 || g->ny < 4 || g->nz < 4) {
        set_error(HC_INVALID, "patch must have at least 4 zones per axis");
        return HC_INVALID;
    }
    if (g->dx <= 0.0 || g->dy <= 0.0 || g->dz <= 0.0) {
        set_error(HC_INVALID, "zone extents must be positive");
        return HC_INVALID;
    }
    if (g->ghost < 2) {
        set_error(HC_INVALID, "ghost width must be at least 2");
        return HC_INVALID;
    }
    if (order != 0 && order != 2 && order != 3) {
        set_error(HC_INVALID, "unsupported order " + std::to_string(order));
        return HC_INVALID;
    }
    if (order == 3 && g->ghost < 3) {
        set_error(HC_INVALID, "order 3 needs a ghost width of at least 3");
        return HC_INVALID;
    }
    return HC_OK;
}

}  // namespace hc

extern "C" {

int hc_abi_version(void) { return HC_ABI_VERSION; }

int hc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int hc_last_error(char* buf, size_t len) {
    if (buf && len) {
        std::strncpy(buf, hc::tl_msg.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return hc::tl_code;
}

}  // extern "C"
