// Plane-layout probe: does the HBM layout of the N_b integral planes change
// how fast B200 absorbs the plane stores?  Pure stores in the k_planes access
// order (CTA = frame x band of R rows, warps = adjacent column strips walking
// the rows together), no compute.  tools/, not part of the product.
//   bin-major  [n][nb][h+1][P]   (current)
//   row-inter  [n][h+1][nb][P]   (one plane row of every bin back to back)
//   pix-inter  [n][h+1][P][nb]   (all bins of a pixel adjacent)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void st256(int32_t *p, int a, int b) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(a),
                 "r"(b), "r"(a), "r"(b), "r"(a), "r"(b));
}

// layout 0/1: strides passed in; VC columns per lane
template <int VC>
__global__ void k_rows(int32_t *pl, int nb, int h, int w, int64_t pp, int64_t pns, int64_t pfs,
                       int R, int nb2) {
    int b = blockIdx.x % nb2, f = blockIdx.x / nb2;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int Y0 = b * R, Ye = min(Y0 + R - 1, h);
    for (int X0 = warp * 32 * VC + VC * lane; X0 <= w; X0 += blockDim.x * VC) {
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
}

// pixel-interleaved: lane owns 4 pixels x nb(=8) bins = 128 contiguous bytes per row
__global__ void k_pix(int32_t *pl, int h, int w, int64_t pp, int64_t pfs, int R, int nb2) {
    int b = blockIdx.x % nb2, f = blockIdx.x / nb2;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int Y0 = b * R, Ye = min(Y0 + R - 1, h);
    for (int X0 = warp * 128 + 4 * lane; X0 <= w; X0 += blockDim.x * 4) {
        for (int Y = Y0; Y <= Ye; ++Y) {
            int32_t *rp = pl + f * pfs + (int64_t)Y * pp + X0 * 8;
#pragma unroll
            for (int q = 0; q < 4; ++q) st256(rp + 8 * q, Y, q);
        }
    }
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
        printf("%-48s %.3f ms  %6.0f GB/s\n", name, best, bytes / best / 1e6);
    };
    int32_t *pl = base + 8;
    for (int R : {16, 32, 64}) {
        const int nb2 = h / R + 1;
        const int blocks = n * nb2;
        for (int warps : {3, 5, 6}) {
            char nm[128];
            // bin-major
            snprintf(nm, 128, "bin-major v4 R=%d warps=%d", R, warps);
            timeit(nm, [&] { k_rows<4><<<blocks, 32 * warps>>>(pl, nb, h, w, P, (h + 1) * P, nb * (h + 1) * P, R, nb2); });
            snprintf(nm, 128, "bin-major v8 R=%d warps=%d", R, warps);
            timeit(nm, [&] { k_rows<8><<<blocks, 32 * warps>>>(pl, nb, h, w, P, (h + 1) * P, nb * (h + 1) * P, R, nb2); });
            snprintf(nm, 128, "row-inter v4 R=%d warps=%d", R, warps);
            timeit(nm, [&] { k_rows<4><<<blocks, 32 * warps>>>(pl, nb, h, w, nb * P, P, nb * (h + 1) * P, R, nb2); });
            snprintf(nm, 128, "row-inter v8 R=%d warps=%d", R, warps);
            timeit(nm, [&] { k_rows<8><<<blocks, 32 * warps>>>(pl, nb, h, w, nb * P, P, nb * (h + 1) * P, R, nb2); });
            snprintf(nm, 128, "pix-inter v8 R=%d warps=%d", R, warps);
            timeit(nm, [&] { k_pix<<<blocks, 32 * warps>>>(pl, h, w, nb * P, nb * (h + 1) * P, R, nb2); });
        }
    }
    timeit("cudaMemset (same bytes)", [&] { cudaMemsetAsync(pl, 0, (size_t)bytes); });
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
