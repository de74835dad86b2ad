// Probe: canonical 2D FP32 TMA load (32 x 8 box), global-memory and param descriptors.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned su32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__global__ void k(const __grid_constant__ CUtensorMap pmap, int mode, float* out) {
    __shared__ __align__(128) float sm[8 * 32];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                     "r"(1024));
        if (mode == 0)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3}], [%4];" ::"r"(su32(sm)),
                "l"(reinterpret_cast<unsigned long long>(&pmap)), "r"(0), "r"(0), "r"(su32(&bar))
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3}], [%4];" ::"r"(su32(sm)),
                "l"(reinterpret_cast<unsigned long long>(&pmap)), "r"(0), "r"(0), "r"(su32(&bar))
                : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}" ::"r"(
            su32(&bar)));
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    std::vector<float> h(64 * 64);
    for (size_t i = 0; i < h.size(); ++i) h[i] = float(i);
    float* d;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    printf("entry: %s q=%d fn=%p\n", cudaGetErrorString(ge), int(q), fn);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap map;
    cuuint64_t dims[2] = {64, 64};
    cuuint64_t str[1] = {64 * 4};
    cuuint32_t box[2] = {32, 8};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", int(r));
    float* out;
    cudaMalloc(&out, 256 * 4);
    k<<<1, 128>>>(map, mode, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    std::vector<float> o(256);
    cudaMemcpy(o.data(), out, 256 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 8; ++y)
        for (int x = 0; x < 32; ++x) bad += o[y * 32 + x] != h[y * 64 + x];
    printf("mismatches %d\n", bad);
    return 0;
}
