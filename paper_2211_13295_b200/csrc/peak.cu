// peak.cu -- FP64 throughput probe: the denominator of the fused kernel's FP64 roofline.
// MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks; the binding roofline of the
// fused step is the FP64 pipe, so the bench measures it on the same box,
// in the same process, right before the timed region. Built with --fmad=true (DFMA chains).
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
    // 16 independent DFMA chains per thread, the loop body unrolled 4x: 64 DFMA per 3 loop
    // instructions, so the FP64 pipe -- not issue -- bounds the kernel
    double x[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) x[c] = 1.0 + 1e-9 * (threadIdx.x + c);
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 16; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s += x[c];
    if (s == 12345.678) out[threadIdx.x] = s;  // keeps the chains live, never taken
}

}  // namespace

extern "C" int hc_fp64_peak(int device, double* tflops) {
    HC_CUDA(cudaSetDevice(device));
    int sms = 0;
    HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* out = nullptr;
    HC_CUDA(cudaMalloc(&out, 1024 * sizeof(double)));
    cudaEvent_t e0, e1;
    HC_CUDA(cudaEventCreate(&e0));
    HC_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 4, threads = 256, iters = 32768;
    k_dfma_peak<<<blocks, threads>>>(out, 64, 0.9999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        HC_CUDA(cudaEventRecord(e0));
        k_dfma_peak<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7);
        HC_CUDA(cudaEventRecord(e1));
        HC_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        HC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    double flops = 2.0 * 16.0 * iters * double(blocks) * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return HC_OK;
}
