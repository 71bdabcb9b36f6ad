// Store-pattern probe: which store stream lets B200 HBM absorb the integral
// planes fastest?  Pure stores, no compute.  (tools/, not part of the product)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void st256(int32_t *p, int a, int b) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(a),
                 "r"(b), "r"(a), "r"(b), "r"(a), "r"(b));
}
__device__ __forceinline__ void st256cs(int32_t *p, int a, int b) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(a),
                 "r"(b), "r"(a), "r"(b), "r"(a), "r"(b));
}

// VC columns per lane (4: 16-B stores, 8: 32-B stores); warp = (frame, band), sweeps strips
template <int VC, int MODE>
__global__ void k_pattern(int32_t *pl, int n, int nb, int h, int w, int64_t pp, int R) {
    int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    int nb2 = h / R + 1;
    if (wid >= (int64_t)n * nb2) return;
    int b = wid % nb2, f = wid / nb2, lane = threadIdx.x & 31;
    int64_t pns = (int64_t)(h + 1) * pp, pfs = pns * nb;
    int Y0 = b * R, Ye = min(Y0 + R - 1, h);
    const int Ws = 32 * VC;
    int ns = (w + Ws - 1) / Ws;
    for (int s = 0; s < ns; ++s) {
        int X0 = s * Ws + VC * lane + 1;
        if (X0 > w) continue;
        for (int Y = Y0; Y <= Ye; ++Y) {
            int32_t *rp = pl + f * pfs + (int64_t)Y * pp + X0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q < nb) {
                    if (VC == 4) *reinterpret_cast<int4 *>(rp + q * pns) = make_int4(Y, q, s, X0);
                    else if (MODE == 0) st256(rp + q * pns, Y, q);
                    else st256cs(rp + q * pns, Y, q);
                }
            }
        }
    }
}

// CTA of 8 warps = 8 consecutive bands' ... no: 8 warps = consecutive column strips of the SAME rows
template <int VC>
__global__ void k_pattern_rows(int32_t *pl, int n, int nb, int h, int w, int64_t pp, int R) {
    // block = (frame, band); warp = strip
    int nb2 = h / R + 1;
    int b = blockIdx.x % nb2, f = blockIdx.x / nb2;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t pns = (int64_t)(h + 1) * pp, pfs = pns * nb;
    int Y0 = b * R, Ye = min(Y0 + R - 1, h);
    const int Ws = 32 * VC;
    int X0 = warp * Ws + VC * lane + 1;
    if (X0 > w) return;
    for (int Y = Y0; Y <= Ye; ++Y) {
        int32_t *rp = pl + f * pfs + (int64_t)Y * pp + X0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < nb) {
                if (VC == 4) *reinterpret_cast<int4 *>(rp + q * pns) = make_int4(Y, q, 0, X0);
                else st256(rp + q * pns, Y, q);
            }
    }
}

__global__ void k_fill(int4 *p, int64_t n4) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = make_int4(1, 2, 3, 4);
}
__global__ void k_fill256(int32_t *p, int64_t n8) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x)
        st256(p + 8 * i, 1, 2);
}

int main() {
    int n = 512, nb = 8, h = 480, w = 640;
    int64_t pp = ((w + 8 + 7) / 8) * 8;
    int64_t total = (int64_t)n * nb * (h + 1) * pp + 16;
    int32_t *base;
    cudaMalloc(&base, total * 4);
    int32_t *pl = base + 7;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    double bytes = (double)n * nb * (h + 1) * (w + 1) * 4;
    auto timeit = [&](const char *name, auto launch, double by) {
        float best = 1e9;
        for (int it = 0; it < 4; ++it) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        printf("%-40s %.3f ms  %6.0f GB/s\n", name, best, by / best / 1e6);
    };
    for (int R : {32, 64, 128}) {
        int warps = n * (h / R + 1);
        char nm[128];
        snprintf(nm, 128, "warp-band v4 R=%d", R);
        timeit(nm, [&] { k_pattern<4, 0><<<(warps + 3) / 4, 128>>>(pl, n, nb, h, w, pp, R); }, bytes);
        snprintf(nm, 128, "warp-band v8 R=%d", R);
        timeit(nm, [&] { k_pattern<8, 0><<<(warps + 3) / 4, 128>>>(base + 8 - 1 + 0, n, nb, h, w, pp, R); }, bytes);
        snprintf(nm, 128, "warp-band v8.cs R=%d", R);
        timeit(nm, [&] { k_pattern<8, 1><<<(warps + 3) / 4, 128>>>(base + 7, n, nb, h, w, pp, R); }, bytes);
        int blocks = n * (h / R + 1);
        snprintf(nm, 128, "cta-rows v4 (5 warps) R=%d", R);
        timeit(nm, [&] { k_pattern_rows<4><<<blocks, 32 * 5>>>(pl, n, nb, h, w, pp, R); }, bytes);
        snprintf(nm, 128, "cta-rows v8 (3 warps) R=%d", R);
        timeit(nm, [&] { k_pattern_rows<8><<<blocks, 32 * 3>>>(pl, n, nb, h, w, pp, R); }, bytes);
    }
    int64_t n4 = total / 4 - 4;
    timeit("grid-stride fill v4", [&] { k_fill<<<148 * 8, 256>>>((int4 *)(base + 8), n4); }, n4 * 16.0);
    timeit("grid-stride fill v8", [&] { k_fill256<<<148 * 8, 256>>>(base + 8, n4 / 2); }, n4 * 16.0);
    timeit("cudaMemset", [&] { cudaMemsetAsync(base, 0, total * 4); }, total * 4.0);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
