// int -> double conversion cost next to DFMA (the window-score kernel converts
// every staged cell count before its FMAs).  Three loops, same FMA count:
//   fma   : 16 independent DFMA chains
//   i2f   : + 4 I2F.F64 per 16 DFMA (the score kernel's ratio is ~12:160)
//   magic : + the same 4 conversions as hi/lo register pairing plus one DADD
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/probe_cvt tools/probe_cvt.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double *out, const int *in, int iters, double a) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
    int v = in[threadIdx.x & 31];
    for (int it = 0; it < iters; ++it) {
        double g[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int q = (v + j * it) & 63;
            if (MODE == 0) g[j] = a;
            if (MODE == 1) g[j] = (double)q;
            if (MODE == 2) g[j] = __hiloint2double(0x43300000, q) - 4503599627370496.0;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], g[i & 3], a);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char *name, double *o, const int *in) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, iters = 4096;
    k<MODE><<<blocks, 256>>>(o, in, iters, 0.999);
    cudaEventRecord(a);
    k<MODE><<<blocks, 256>>>(o, in, iters, 0.999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fmas = (double)blocks * 256 * iters * 16;
    printf("%-6s %.3f ms  %.2f T DFMA/s (4 conversions per 16 DFMA in i2f/magic)\n", name, ms,
           fmas / ms / 1e9);
}

int main() {
    double *o;
    int *in;
    cudaMalloc(&o, 148 * 8 * 256 * 8);
    cudaMalloc(&in, 32 * 4);
    cudaMemset(in, 1, 32 * 4);
    run<0>("fma", o, in);
    run<1>("i2f", o, in);
    run<2>("magic", o, in);
    return 0;
}
