// k_rect.cu -- 16-bit accumulator planes and batched rectangle queries
// (SURVEY §8f rank 4).
//
// integral.py:58-87 with acc_width=16: the reference keeps uint16 planes when
// no bin can exceed 65535 counts (W*H <= 65535; the paper's DSP remark,
// PAPER.md:126).  Such frames are small, so one warp owns one (frame, bin)
// plane and walks its rows: per 32-column chunk a ballot of "pixel is bin n"
// and a popc give the row prefix, the per-column running sums (<= H) live in
// shared memory as uint16, and each plane row is written once as uint16 --
// half the bytes of the 32-bit planes.
//
// integral.py:95-115 (rect_count / rect_histogram): the 4-corner formula
// p[y1,x1] + p[y0,x0] - p[y1,x0] - p[y0,x1] for a batch of rectangles, one
// thread per (rectangle, bin), int64 results, uint32 or uint16 planes.
#include "hog_common.cuh"

namespace hogb200 {

constexpr int I16_WARPS = 4;

__global__ void __launch_bounds__(32 * I16_WARPS)
k_integral16(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, int n, int h, int w, int bins,
             uint16_t *__restrict__ pl, int64_t pp, int64_t pns, int64_t pfs) {
    extern __shared__ uint16_t colsum[];  // [I16_WARPS][w]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t job = (int64_t)blockIdx.x * I16_WARPS + warp;  // (frame, bin)
    if (job >= (int64_t)n * bins) return;
    const int f = (int)(job / bins), b = (int)(job % bins);
    uint16_t *cs = colsum + (size_t)warp * w;
    const int8_t *src = bm + (int64_t)f * bfs;
    uint16_t *dst = pl + (int64_t)f * pfs + (int64_t)b * pns;
    for (int x = lane; x < w; x += 32) cs[x] = 0;
    for (int X = lane; X <= w; X += 32) dst[X] = 0;  // row 0
    __syncwarp();
    const unsigned below = (1u << lane) - 1u;
    for (int y = 0; y < h; ++y) {
        const int8_t *row = src + (int64_t)y * bp;
        uint16_t *out = dst + (int64_t)(y + 1) * pp;
        if (lane == 0) out[0] = 0;  // column 0
        uint32_t run = 0;           // count of bin-b pixels left of this chunk
        for (int x0 = 0; x0 < w; x0 += 32) {
            const int x = x0 + lane;
            const bool hit = x < w && row[x] == (int8_t)b;
            const unsigned m = __ballot_sync(FULL, hit);
            if (x < w) {
                const uint16_t c = (uint16_t)(cs[x] + run + __popc(m & below) + (hit ? 1 : 0));
                cs[x] = c;  // P(y+1, x+1) = P(y, x+1) + row prefix through x
                out[x + 1] = c;
            }
            run += __popc(m);
        }
        __syncwarp();
    }
}

template <typename T>
__global__ void k_rect_hist(const T *__restrict__ pl, int64_t pp, int64_t pns, int bins,
                            const int32_t *__restrict__ rects, int k, int64_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)k * bins) return;
    const int r = (int)(i / bins), b = (int)(i % bins);
    const int x0 = rects[4 * r], y0 = rects[4 * r + 1], x1 = rects[4 * r + 2], y1 = rects[4 * r + 3];
    const T *p = pl + (int64_t)b * pns;
    out[i] = (int64_t)p[(int64_t)y1 * pp + x1] + (int64_t)p[(int64_t)y0 * pp + x0] -
             (int64_t)p[(int64_t)y1 * pp + x0] - (int64_t)p[(int64_t)y0 * pp + x1];
}

void launch_integral16(const int8_t *bm, int64_t bp, int64_t bfs, int n, int h, int w, int bins,
                       uint16_t *pl, int64_t pp, int64_t pns, int64_t pfs, cudaStream_t st) {
    const size_t smem = sizeof(uint16_t) * (size_t)I16_WARPS * w;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_integral16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t jobs = (int64_t)n * bins;
    k_integral16<<<(unsigned)((jobs + I16_WARPS - 1) / I16_WARPS), 32 * I16_WARPS, smem, st>>>(
        bm, bp, bfs, n, h, w, bins, pl, pp, pns, pfs);
}

void launch_rect_hist(const void *pl, int elem_bytes, int64_t pp, int64_t pns, int bins,
                      const int32_t *rects, int k, int64_t *out, cudaStream_t st) {
    const int64_t tot = (int64_t)k * bins;
    if (elem_bytes == 2)
        k_rect_hist<uint16_t><<<blocks_for(tot, 256), 256, 0, st>>>((const uint16_t *)pl, pp, pns,
                                                                    bins, rects, k, out);
    else
        k_rect_hist<uint32_t><<<blocks_for(tot, 256), 256, 0, st>>>((const uint32_t *)pl, pp, pns,
                                                                    bins, rects, k, out);
}

}  // namespace hogb200
