// Per-warp TMA bulk-store probe: each warp stages its own strip of plane
// columns (Ws columns x nb bins per row) in a shared-memory ring and its lane
// 0 issues one cp.async.bulk per (bin, row) -- no CTA barrier on the store
// path.  Compared with per-thread st.global.v4/v8 in the same order.
// tools/, not part of the product.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// CTA = (frame, band), NWARP warps = strips of Ws = 32*VC - 4 columns (like k_planes)
template <int VC, int RING, int NB>
__global__ void k_warp_tma(int32_t *pl, int h, int w, int64_t P, int R, int nb2) {
    extern __shared__ __align__(128) int32_t sm[];
    const int b = blockIdx.x % nb2, f = blockIdx.x / nb2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int Ws = 32 * VC - 4;
    constexpr int SEG = 32 * VC;  // staged ints per bin row (Ws used)
    int32_t *ring = sm + warp * RING * NB * SEG;
    const int Y0 = b * R, Ye = min(Y0 + R - 1, h);
    const int64_t pns = (int64_t)(h + 1) * P, pfs = NB * pns;
    const int xs = warp * Ws;
    if (xs >= w) return;
    const int ncols = min(Ws, w - xs);
    const uint32_t bytes = (uint32_t)(((ncols + 3) & ~3) * 4);
    int slot = 0;
    for (int Y = Y0; Y <= Ye; ++Y) {
        int32_t *st = ring + slot * NB * SEG;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            if (VC == 4)
                *reinterpret_cast<int4 *>(st + q * SEG + 4 * lane) = make_int4(Y, q, lane, f);
            else {
                *reinterpret_cast<int4 *>(st + q * SEG + 8 * lane) = make_int4(Y, q, lane, f);
                *reinterpret_cast<int4 *>(st + q * SEG + 8 * lane + 4) = make_int4(Y, q, lane, f);
            }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
            int32_t *g = pl + f * pfs + (int64_t)Y * P + xs;
#pragma unroll
            for (int q = 0; q < NB; ++q) bulk_store(g + q * pns, st + q * SEG, bytes);
            bulk_commit();
            bulk_wait_read<RING - 1>();
        }
        __syncwarp();
        slot = (slot + 1) % RING;
    }
    if (lane == 0) bulk_wait_read<0>();
}

template <int VC, int NB>
__global__ void k_warp_st(int32_t *pl, int h, int w, int64_t P, int R, int nb2) {
    const int b = blockIdx.x % nb2, f = blockIdx.x / nb2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int Ws = 32 * VC - 4;
    const int Y0 = b * R, Ye = min(Y0 + R - 1, h);
    const int64_t pns = (int64_t)(h + 1) * P, pfs = NB * pns;
    const int x = warp * Ws + VC * lane;
    if (VC * lane >= Ws || x >= w) return;
    for (int Y = Y0; Y <= Ye; ++Y) {
        int32_t *g = pl + f * pfs + (int64_t)Y * P + x;
#pragma unroll
        for (int q = 0; q < NB; ++q) *reinterpret_cast<int4 *>(g + q * pns) = make_int4(Y, q, lane, f);
    }
}

int main() {
    const int n = 512, h = 480, w = 640;
    constexpr int NB = 8;
    const int64_t P = ((w + 8 + 7) / 8) * 8;
    const int64_t total = (int64_t)n * NB * (h + 1) * P + 64;
    int32_t *base;
    cudaMalloc(&base, total * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = (double)n * NB * (h + 1) * (w + 1) * 4;
    auto timeit = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        printf("%-48s %.3f ms  %6.0f GB/s  %s\n", name, best, bytes / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    int32_t *pl = base + 8;
#define RUNW(VC, RING, NWARP)                                                                          \
    {                                                                                                  \
        const size_t smem = (size_t)NWARP * RING * NB * 32 * VC * 4;                                   \
        cudaFuncSetAttribute(k_warp_tma<VC, RING, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             (int)smem);                                                               \
        snprintf(nm, 128, "warp-tma VC=%d ring=%d warps=%d R=%d smem=%zuK", VC, RING, NWARP, R,       \
                 smem / 1024);                                                                         \
        timeit(nm, [&] { k_warp_tma<VC, RING, NB><<<blocks, 32 * NWARP, smem>>>(pl, h, w, P, R, nb2); }); \
    }
    for (int R : {16, 32, 64}) {
        const int nb2 = h / R + 1;
        const int blocks = n * nb2;
        char nm[128];
        RUNW(4, 2, 6) RUNW(4, 3, 6) RUNW(4, 4, 6) RUNW(8, 2, 3) RUNW(8, 3, 3) RUNW(8, 4, 3)
        snprintf(nm, 128, "warp-st v4 warps=6 R=%d", R);
        timeit(nm, [&] { k_warp_st<4, NB><<<blocks, 32 * 6>>>(pl, h, w, P, R, nb2); });
    }
    timeit("cudaMemset (same bytes)", [&] { cudaMemsetAsync(pl, 0, (size_t)bytes); });
    return 0;
}
