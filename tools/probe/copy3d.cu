// PCIe probe: active-zone 3D copies (the e2e pattern of hc_stepper_step_host) vs 1D
// contiguous copies of the same bytes, one direction and both at once.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_store(const double2* __restrict__ src, double2* dst, int n, int m, int G) {
    // active rows of the padded box -> the same positions of the (mapped, pinned) host box
    const size_t rowv = size_t(n) * 40 / 16, pitchv = size_t(m) * 40 / 16;
    const size_t rows = size_t(n) * n;
    for (size_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const size_t k = r / n + G, j = r % n + G;
        const size_t base = (k * m + j) * pitchv + size_t(G) * 40 / 16;
        for (size_t c = threadIdx.x; c < rowv; c += blockDim.x) dst[base + c] = src[base + c];
    }
}
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
    const int n = 256, G = 3, m = n + 2 * G;
    const size_t row = size_t(n) * 40, pitch = size_t(m) * 40;
    const size_t total = size_t(m) * m * m * 40, act = size_t(n) * n * n * 40;
    char *h1, *h2, *d1, *d2;
    CK(cudaMallocHost(&h1, total)); CK(cudaMallocHost(&h2, total));
    CK(cudaMalloc(&d1, total)); CK(cudaMalloc(&d2, total));
    cudaStream_t a, b; CK(cudaStreamCreate(&a)); CK(cudaStreamCreate(&b));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto p3 = [&](char* dst, char* src, cudaMemcpyKind k, cudaStream_t s, int planes) {
        cudaMemcpy3DParms p = {};
        size_t off = (size_t(G) * m * m + size_t(G) * m + G) * 40;
        p.srcPtr = make_cudaPitchedPtr(src + off, pitch, row, m);
        p.dstPtr = make_cudaPitchedPtr(dst + off, pitch, row, m);
        p.extent = make_cudaExtent(row, n, planes);
        p.kind = k;
        return cudaMemcpy3DAsync(&p, s);
    };
    char* hmap; CK(cudaHostGetDevicePointer((void**)&hmap, h2, 0));
    for (int mode = 0; mode < 10; ++mode) {
        for (int it = 0; it < 2; ++it) {
            CK(cudaEventRecord(e0, 0));
            CK(cudaStreamWaitEvent(a, e0)); CK(cudaStreamWaitEvent(b, e0));
            if (mode == 0) CK(cudaMemcpyAsync(d1, h1, act, cudaMemcpyHostToDevice, a));
            if (mode == 1) CK(p3(d1, h1, cudaMemcpyHostToDevice, a, n));
            if (mode == 2) CK(cudaMemcpyAsync(h2, d2, act, cudaMemcpyDeviceToHost, b));
            if (mode == 3) CK(p3(h2, d2, cudaMemcpyDeviceToHost, b, n));
            if (mode == 4) { CK(cudaMemcpyAsync(d1, h1, act, cudaMemcpyHostToDevice, a));
                             CK(cudaMemcpyAsync(h2, d2, act, cudaMemcpyDeviceToHost, b)); }
            if (mode == 5) { CK(p3(d1, h1, cudaMemcpyHostToDevice, a, n));
                             CK(p3(h2, d2, cudaMemcpyDeviceToHost, b, n)); }
            if (mode == 6) { CK(cudaMemcpyAsync(d1, h1, act, cudaMemcpyHostToDevice, a));
                             CK(p3(h2, d2, cudaMemcpyDeviceToHost, b, n)); }
            if (mode == 7) { CK(cudaMemcpyAsync(d1, h1, act, cudaMemcpyHostToDevice, a));
                             size_t off = (size_t(G) * m * m + size_t(G) * m + G) * 40;
                             for (int k = 0; k < n; ++k)
                                 CK(cudaMemcpy2DAsync(h2 + off + size_t(k) * m * m * 40, pitch,
                                                      d2 + off + size_t(k) * m * m * 40, pitch,
                                                      row, n, cudaMemcpyDeviceToHost, b)); }
            if (mode == 8) { CK(cudaMemcpyAsync(d1, h1, act, cudaMemcpyHostToDevice, a));
                             k_store<<<148 * 4, 256, 0, b>>>((const double2*)d2, (double2*)hmap, n, m, G); }
            if (mode == 9) { k_store<<<148 * 4, 256, 0, b>>>((const double2*)d2, (double2*)hmap, n, m, G); }
            cudaEvent_t ea, eb; cudaEventCreate(&ea); cudaEventCreate(&eb);
            cudaEventRecord(ea, a); cudaEventRecord(eb, b);
            CK(cudaStreamWaitEvent(0, ea)); CK(cudaStreamWaitEvent(0, eb));
            CK(cudaEventRecord(e1, 0)); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const char* nm[] = {"h2d 1D", "h2d 3D", "d2h 1D", "d2h 3D", "both 1D", "both 3D",
                                "h1D+d3D", "h1D+d2D", "h1D+dker", "d kernel"};
            if (it) printf("%-10s %7.2f ms  %6.1f GB/s per direction\n", nm[mode], ms, act / (ms * 1e6));
        }
    }
    return 0;
}
