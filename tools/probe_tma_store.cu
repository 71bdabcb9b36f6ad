// TMA bulk-store probe: stage plane rows in shared memory and let the TMA
// engine write them (cp.async.bulk.global.shared::cta), instead of per-thread
// st.global.  Same CTA = (frame, band) decomposition as k_planes; pure
// stores.  tools/, not part of the product.
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

// LAYOUT 0 bin-major (one bulk copy per bin row), 1 row-interleaved (one copy per row of all bins)
// STAGES row buffers in flight; each buffer holds one plane row of all nb bins (nb * P ints)
template <int LAYOUT, int STAGES>
__global__ void k_tma(int32_t *pl, int nb, int h, int w, int64_t P, int R, int nb2) {
    extern __shared__ __align__(128) int32_t sm[];
    const int b = blockIdx.x % nb2, f = blockIdx.x / nb2;
    const int Y0 = b * R, Ye = min(Y0 + R - 1, h);
    const int64_t pns = LAYOUT == 0 ? (int64_t)(h + 1) * P : P;
    const int64_t pp = LAYOUT == 0 ? P : nb * P;
    const int64_t pfs = (int64_t)nb * (h + 1) * P;
    const int rowint = nb * (int)P;
    int s = 0;
    for (int Y = Y0; Y <= Ye; ++Y) {
        int32_t *buf = sm + s * rowint;
        if (threadIdx.x == 0 && Y - Y0 >= STAGES) bulk_wait_read<STAGES - 1>();
        __syncthreads();
        for (int i = 4 * threadIdx.x; i < rowint; i += 4 * blockDim.x)
            *reinterpret_cast<int4 *>(buf + i) = make_int4(Y, i, f, 1);
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            int32_t *g = pl + f * pfs + (int64_t)Y * pp;
            if (LAYOUT == 0) {
                for (int q = 0; q < nb; ++q) bulk_store(g + q * pns, buf + q * P, (uint32_t)((w + 8) * 4));
            } else {
                bulk_store(g, buf, (uint32_t)(rowint * 4));
            }
            bulk_commit();
        }
        s = (s + 1) % STAGES;
    }
    if (threadIdx.x == 0) bulk_wait_read<0>();
}

int main() {
    const int n = 512, nb = 8, h = 480, w = 640;
    const int64_t P = ((w + 8 + 7) / 8) * 8;
    const int64_t total = (int64_t)n * nb * (h + 1) * P + 64;
    int32_t *base;
    cudaMalloc(&base, total * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = (double)n * nb * (h + 1) * (w + 1) * 4;
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
    const int rowbytes = nb * (int)P * 4;
#define RUN(L, S)                                                                                   \
    {                                                                                               \
        const size_t smem = (size_t)S * rowbytes;                                                   \
        cudaFuncSetAttribute(k_tma<L, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        snprintf(nm, 128, "tma L%d stages=%d R=%d thr=%d", L, S, R, thr);                           \
        timeit(nm, [&] { k_tma<L, S><<<blocks, thr, smem>>>(pl, nb, h, w, P, R, nb2); });          \
    }
    for (int R : {16, 32, 64}) {
        const int nb2 = h / R + 1;
        const int blocks = n * nb2;
        for (int thr : {128, 256}) {
            char nm[128];
            RUN(0, 2) RUN(0, 4) RUN(1, 2) RUN(1, 4) RUN(1, 8)
        }
    }
    timeit("cudaMemset (same bytes)", [&] { cudaMemsetAsync(pl, 0, (size_t)bytes); });
    return 0;
}
