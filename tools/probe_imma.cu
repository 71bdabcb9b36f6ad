// Throughput of mma.sync m16n8k32 s8 (IMMA.16832) on one GPU: 8 independent
// accumulator chains per warp, every SM busy.  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o build/probe_imma tools/probe_imma.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *out, int iters) {
    int acc[8][4] = {};
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
    for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int *out;
    cudaMalloc(&out, 1 << 24);
    const int iters = 4096;
    for (int warps = 4; warps <= 32; warps *= 2) {
        k<<<sms, 32 * warps>>>(out, 16);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0), cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<sms, 32 * warps>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = (double)sms * warps * iters * 8;
        printf("warps/SM %2d: %.3f ms, %.1f T int8 MAC/s (%.0f TOPS), %.2f MMA/clk/SM at 1.965 GHz\n", warps, ms,
               mmas * 4096 / ms / 1e9, 2 * mmas * 4096 / ms / 1e9, mmas / sms / (ms * 1e-3 * 1.965e9));
    }
    return 0;
}
