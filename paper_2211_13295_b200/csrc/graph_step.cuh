// graph_step.cuh -- replay of one captured time step as a CUDA graph (the MHD and CED
// steppers; the Euler stepper has its own, stepper.cu capture_step). Valid because every
// kernel of a step reads its time control (dt, t, done flags) from device memory: only host
// values baked into launch arguments (`key`, e.g. the CFL number) force a re-capture.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"

namespace hc {

struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    double key = 0.0;
    long per_step = 0;  // kernels per replayed step
    ~StepGraph() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

inline bool graphs_disabled() {
    static const bool off = [] {
        const char* v = std::getenv("HC_NO_GRAPH");
        return v && std::atoi(v) != 0;
    }();
    return off;
}

// enqueue(): launches one step on `st`, adding its kernel count to `launches`
template <class Enqueue>
int replay_steps(StepGraph& g, cudaStream_t st, double key, long& launches, int n,
                 Enqueue enqueue) {
    int rc = HC_OK;
    if (n <= 1 || graphs_disabled()) {
        for (int i = 0; i < n && !rc; ++i) rc = enqueue();
        return rc;
    }
    if (!g.exec || g.key != key) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
        const long l0 = launches;
        cudaGraph_t graph = nullptr;
        HC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        rc = enqueue();
        cudaError_t e = cudaStreamEndCapture(st, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
        e = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            g.exec = nullptr;
            return cuda_fail(e, "cudaGraphInstantiate");
        }
        g.per_step = launches - l0;
        launches = l0;
        g.key = key;
    }
    for (int i = 0; i < n; ++i) {
        HC_CUDA(cudaGraphLaunch(g.exec, st));
        launches += g.per_step;
    }
    return HC_OK;
}

}  // namespace hc
