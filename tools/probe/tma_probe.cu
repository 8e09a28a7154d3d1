// Stand-alone probe of the TMA + mbarrier helpers used by vanka_march_kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m, double* out, int W, int H, int c0, int c1) {
    extern __shared__ __align__(128) double sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + W * H * 10);
    if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (MODE == 1) {
        if (threadIdx.x == 0) { mbar_expect_tx(bar, W * H * 10 * 8); tma_load3(sm, &m, c0, c1, 0, bar); }
        mbar_wait(bar, 0);
    }
    for (int t = threadIdx.x; t < W * H * 10; t += blockDim.x) out[t] = sm[t];
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    int n = 64, pitch = 96; long plane = (long)(n + 1) * pitch;
    std::vector<double> h(10 * plane);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double* d; cudaMalloc(&d, h.size() * 8); cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    printf("entry point: %s q=%d fn=%p\n", cudaGetErrorString(e), (int)q, fn);
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    int W = argc > 1 ? atoi(argv[1]) : 34, H = 4; int C0 = argc > 2 ? atoi(argv[2]) : -2, C1 = argc > 3 ? atoi(argv[3]) : 3;
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)n + 1, (cuuint64_t)n + 1, 10};
    cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)plane * 8};
    cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)H, 10};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    double* o; cudaMalloc(&o, W * H * 10 * 8);
    int smem = W * H * 10 * 8 + 64;
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<0><<<1, 128, smem>>>(m, m, o, W, H, C0, C1);
    printf("plain kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    probe<1><<<1, 128, smem>>>(m, m, o, W, H, C0, C1);
    e = cudaDeviceSynchronize();
    printf("tma kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<double> ho(W * H * 10);
    cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int p = 0; p < 10; ++p) for (int y = 0; y < H; ++y) for (int x = 0; x < W; ++x) {
        int gi = C0 + x, gj = C1 + y;
        double ref = (gi >= 0 && gi <= n && gj >= 0 && gj <= n) ? h[p * plane + (long)gj * pitch + gi] : 0.0;
        if (ho[(p * H + y) * W + x] != ref) ++bad;
    }
    printf("mismatches: %d\n", bad);
    return 0;
}
