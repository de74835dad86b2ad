// Probe: one TMA 3D tensor load of FP64 boxes shaped like the persistent kernel's planes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tma3d.cu -o tma3d && ./tma3d
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ unsigned su32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap pmap, const CUtensorMap* gmap, int c0,
                  int c1, int c2, unsigned bytes, double* out, int n) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const CUtensorMap* m = MODE == 0 ? &pmap : gmap;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                     "r"(bytes));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(sm)),
            "l"(reinterpret_cast<unsigned long long>(m)), "r"(c0), "r"(c1), "r"(c2),
            "r"(su32(&bar))
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}" ::"r"(
            su32(&bar)));
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
    const int dtype = argc > 1 ? atoi(argv[1]) : 0, promo = argc > 4 ? atoi(argv[4]) : 1, inner = argc > 2 ? atoi(argv[2]) : 180, mode0 = argc > 3 ? atoi(argv[3]) : 0;
    const int mx = 38, my = 13, mz = 10, NV = 5;
    const int W = 36, H = 11;
    std::vector<double> h(size_t(mx) * NV * my * mz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = double(i);
    double* d;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap map;
    cuuint64_t dims[3] = {cuuint64_t(mx) * NV, cuuint64_t(my), cuuint64_t(mz)};
    cuuint64_t str[2] = {cuuint64_t(mx) * NV * 8, cuuint64_t(mx) * NV * my * 8};
    cuuint32_t box[3] = {cuuint32_t(inner), cuuint32_t(H), 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&map, dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : (dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_INT64 : CU_TENSOR_MAP_DATA_TYPE_UINT64), 3, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", int(r));
    CUtensorMap* gm;
    cudaMalloc(&gm, sizeof map);
    cudaMemcpy(gm, &map, sizeof map, cudaMemcpyHostToDevice);
    const int n = inner * H;
    double* out;
    cudaMalloc(&out, n * 8);
    const unsigned bytes = n * 8;
    for (int mode = mode0; mode < mode0 + 1; ++mode) {
        cudaMemset(out, 0, n * 8);
        const int c0 = argc > 5 ? atoi(argv[5]) : 5, c1 = 1, c2 = 3;
        if (mode == 0)
            k<0><<<1, 128, bytes + 1024>>>(map, gm, c0, c1, c2, bytes, out, n);
        else
            k<1><<<1, 128, bytes + 1024>>>(map, gm, c0, c1, c2, bytes, out, n);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<double> o(n);
        cudaMemcpy(o.data(), out, n * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < inner; ++x) {
                double want = h[(size_t(c2) * my + (c1 + y)) * mx * NV + c0 + x];
                if (o[y * inner + x] != want) ++bad;
            }
        printf("mode %d: %d mismatches\n", mode, bad);
    }
    return 0;
}
