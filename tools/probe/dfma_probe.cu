// fp64 FMA throughput probe (diagnostic): 8 independent DFMA chains per thread, full grid.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a dfma_probe.cu -o /tmp/dfma && /tmp/dfma
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, double a, double b, int iters) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = threadIdx.x * 1e-3 + q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = fma(v[q], a, b);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += v[q];
    if (s == 12345.678) out[0] = s;
}
int main() {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int tpb : {128, 256, 512}) for (int per : {2, 4, 8}) {
        int blocks = sms * per, iters = 2000;
        k<<<blocks, tpb>>>(d, 0.999, 1e-3, 10);
        cudaEventRecord(e0);
        k<<<blocks, tpb>>>(d, 0.999, 1e-3, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = (double)blocks * tpb * iters * 16 * 8;
        printf("tpb %d blocks/SM %d: %.2f TFLOP/s fp64 (%.1f DFMA/clk/SM at 1965 MHz)\n", tpb, per,
               2 * fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
