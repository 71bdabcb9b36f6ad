// FP64 FMA throughput probe (the roofline of the window-score kernel).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double *o; cudaMalloc(&o, 148 * 8 * 256 * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocks : {148 * 4, 148 * 8}) {
        int iters = 4096;
        k<<<blocks, 256>>>(o, iters, 0.999, 1e-3);
        cudaEventRecord(a);
        k<<<blocks, 256>>>(o, iters, 0.999, 1e-3);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double fmas = (double)blocks * 256 * iters * 16;
        printf("blocks %d: %.3f ms  %.2f T DFMA/s = %.1f TFLOP/s fp64\n", blocks, ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
    }
    return 0;
}
