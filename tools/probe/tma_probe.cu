// TMA alignment probe: one 3-D box (W cols x 1 row x 10 planes, fp64) at column origin c0 into shared
// memory at byte offset `off`; prints whether the data matches.  Usage: tma_probe c0 off W
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int off, int W, double* out) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ __align__(8) unsigned long long bar;
    double* dst = reinterpret_cast<double*>(sm + off);
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar), d = (unsigned)__cvta_generic_to_shared(dst);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(W * 80));
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(d), "l"(&m), "r"(c0), "r"(0), "r"(0), "r"(b) : "memory");
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}" ::"r"(b));
        for (int i = 0; i < W * 10; ++i) out[i] = dst[i];
    }
}
int main(int argc, char** argv) {
    int c0 = atoi(argv[1]), off = atoi(argv[2]), W = atoi(argv[3]);
    const int N = 64, P = 64;
    double* g; cudaMalloc(&g, 8 * N * P * 10);
    double* h = (double*)malloc(8 * N * P * 10);
    for (int i = 0; i < N * P * 10; ++i) h[i] = i;
    cudaMemcpy(g, h, 8 * N * P * 10, cudaMemcpyHostToDevice);
    void* fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[3] = {N, N, 10}, str[2] = {P * 8, (cuuint64_t)N * P * 8};
    cuuint32_t box[3] = {(cuuint32_t)W, 1, 10}, es[3] = {1, 1, 1};
    CUresult r = ((EncodeTiledFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); return 1; }
    double* o; cudaMalloc(&o, 8 * W * 10);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    k<<<1, 32, 8192>>>(m, c0, off, W, o);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("c0=%d off=%d W=%d: %s\n", c0, off, W, cudaGetErrorString(e)); return 0; }
    double* ho = (double*)malloc(8 * W * 10);
    cudaMemcpy(ho, o, 8 * W * 10, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int p = 0; p < 10; ++p)
        for (int c = 0; c < W; ++c) {
            int gc = c0 + c;
            double want = (gc >= 0 && gc < N) ? (double)(p * N * P + gc) : 0.0;
            if (ho[p * W + c] != want) ++bad;
        }
    printf("c0=%d off=%d W=%d: %s (%d bad)\n", c0, off, W, bad ? "MISMATCH" : "ok", bad);
    return 0;
}
