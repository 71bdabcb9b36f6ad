// k_scores.cu -- window scores on a regular cell lattice, unnormalised grid
// (detector.py:140-154 with DescriptorGeometry(block=1, block_stride=1),
// descriptor.py:107-118).  The window at lattice origin (iy, ix) reads cells
// (iy + cy*K, ix + cx*K), cy < cells_y, cx < 8, so the score map is a 2-D
// correlation of the cell grid with the weight tensor w[cy][cx][n], plus the
// bias.  fp64 accumulation (fp32 misses 1e-5 on blurred
// inputs); the summation order differs from OpenBLAS ddot, which the 1e-5
// relative tolerance allows (measured: ~1e-15).
//
// FP64-FMA-bound design (c5: 2304 FMAs per window, 3.7 G per frame):
//   A warp owns SR_TY window rows x 32*TX window columns and streams the
//   SR_TY + (cells_y-1)*K grid rows they read through its own two-slot ring
//   in shared memory (no CTA-wide barrier, so warps never wait on rows they
//   do not use).  Row r+1 is copied by cp.async (4-byte, zero-fill past the
//   frame) while row r is consumed.  Slots are int32 [column/TX][column%TX][bin]
//   with one pad word per TX columns: lane L reads column TX*L + j at word
//   L*(TX*bins+1) + ..., an odd lane stride, so the reads are conflict-free.
//   Per (row, bin) a lane converts its TX + 7K grid values to double once and
//   reuses them for all SR_TY window rows (inactive rows multiply a zero
//   weight row, which keeps the 4*TX accumulator chains independent and the
//   FMA stream branch-free); weights are warp-broadcast LDS.128.
#include "hog_common.cuh"

namespace hogb200 {

constexpr int SR_TY = 4, SR_WARPS = 4;

__device__ __forceinline__ void cp_async4(uint32_t *sdst, const int32_t *gsrc, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_addr(sdst)), "l"(gsrc),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__host__ __device__ constexpr int sr_span(int tx, int k) { return 32 * tx + 7 * k; }
// words of one staged grid row: ceil(span/tx) chunks of tx columns x bins + 1 pad
__host__ __device__ inline int sr_slot_words(int bins, int tx, int k) {
    return ((sr_span(tx, k) + tx - 1) / tx) * (tx * bins + 1);
}

// TX window columns per lane (32*TX per warp); BINS > 0: bin count known at
// compile time (shared-memory offsets become immediates), 0: runtime `bins`.
template <int K, int TX, int BINS>
__global__ void __launch_bounds__(32 * SR_WARPS, 3)
k_scores_rows(const int32_t *__restrict__ grid, int ncy, int ncx, int bins_rt, int noy, int nox,
              int cells_y, const double *__restrict__ wts, double bias, double *__restrict__ scores,
              uint32_t magic) {
    constexpr int CX = 8;
    constexpr int SPAN = sr_span(TX, K);  // grid columns a warp reads
    constexpr int NG = TX / K + CX - 1;   // grid values per (row, bin, parity)
    constexpr int COLS = 32 * TX;
    const int bins = BINS > 0 ? BINS : bins_rt;
    extern __shared__ __align__(16) double ssm[];
    double *wsm = ssm;  // [cells_y + 1][bins][8]; row cells_y is zero (inactive window rows)
    const int slotw = sr_slot_words(bins, TX, K);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *ring = reinterpret_cast<uint32_t *>(ssm + (size_t)(cells_y + 1) * bins * CX) + warp * 2 * slotw;
    const int tiles_x = (nox + COLS - 1) / COLS;
    const int tiles_y = (noy + SR_TY * SR_WARPS - 1) / (SR_TY * SR_WARPS);
    int bid = blockIdx.x;
    const int tx = bid % tiles_x;
    bid /= tiles_x;
    const int ty = bid % tiles_y;
    const int f = bid / tiles_y;
    const int ix0 = tx * COLS;
    const int iyw = ty * SR_TY * SR_WARPS + warp * SR_TY;  // this warp's first window row
    const int32_t *gf = grid + (int64_t)f * ncy * ncx * bins;

    for (int i = threadIdx.x; i < (cells_y + 1) * CX * bins; i += blockDim.x) {
        const int n = i % bins, cx = (i / bins) % CX, cy = i / (bins * CX);
        wsm[(cy * bins + n) * CX + cx] = cy < cells_y ? wts[i] : 0.0;
    }
    __syncthreads();  // the only CTA-wide barrier: weights staged
    if (iyw >= noy) return;

    const int nel = min(SPAN, ncx - ix0) * bins;  // words of a row inside the frame
    const int ctb = TX * bins;  // words of a chunk of TX columns (+1 pad word)
    auto stage = [&](int r, uint32_t *dst) {  // async copy of grid row r (this warp's columns)
        const int32_t *src = gf + ((int64_t)r * ncx + ix0) * bins;
        const bool rok = r < ncy;
        for (int e = lane; e < SPAN * bins; e += 32) {
            const int q = (int)__umulhi((uint32_t)e, magic);  // e / (TX*bins)
            const bool ok = rok && e < nel;
            cp_async4(dst + e + q, ok ? src + e : gf, ok);
        }
        cp_async_commit();
    };
    double acc[SR_TY][TX];
#pragma unroll
    for (int u = 0; u < SR_TY; ++u)
#pragma unroll
        for (int t = 0; t < TX; ++t) acc[u][t] = 0.0;

    const int r_first = iyw;
    const int r_last = min(iyw + SR_TY - 1, noy - 1) + (cells_y - 1) * K;
    stage(r_first, ring);
    // lane L's columns start at TX*L, the first column of chunk L: lane stride TX*bins+1 (odd)
    const int c0 = TX * lane;
    const int lbase = lane * (ctb + 1);
    for (int r = r_first; r <= r_last; ++r) {
        const int slot = (r - r_first) & 1;
        cp_async_wait_all();
        __syncwarp();  // row r visible to the warp; the other slot is free
        if (r < r_last) stage(r + 1, ring + (slot ^ 1) * slotw);
        const double *wu[SR_TY];  // weight rows of grid row r for each window row (zero row if none)
#pragma unroll
        for (int u = 0; u < SR_TY; ++u) {
            const int d = r - (iyw + u);
            const int cy = (d >= 0 && d % K == 0 && d / K < cells_y) ? d / K : cells_y;
            wu[u] = wsm + cy * bins * CX;
        }
        const uint32_t *row = ring + slot * slotw + lbase;
        for (int n = 0; n < bins; ++n) {
#pragma unroll
            for (int p = 0; p < K; ++p) {
                double gs[NG];
#pragma unroll
                for (int j = 0; j < NG; ++j) {
                    const int c = p + K * j;  // column c0 + c
                    gs[j] = (double)(int)row[(c / TX) * (ctb + 1) + (c % TX) * bins + n];
                }
#pragma unroll
                for (int cx = 0; cx < CX; cx += 2) {
                    double2 w2[SR_TY];
#pragma unroll
                    for (int u = 0; u < SR_TY; ++u)
                        w2[u] = *reinterpret_cast<const double2 *>(wu[u] + n * CX + cx);
#pragma unroll
                    for (int u = 0; u < SR_TY; ++u)
#pragma unroll
                        for (int t = 0; t < TX / K; ++t) {
                            acc[u][K * t + p] = fma(w2[u].x, gs[t + cx], acc[u][K * t + p]);
                            acc[u][K * t + p] = fma(w2[u].y, gs[t + cx + 1], acc[u][K * t + p]);
                        }
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < SR_TY; ++u) {
        const int iy = iyw + u;
        if (iy >= noy) continue;
        double *sp = scores + ((int64_t)f * noy + iy) * nox + ix0 + c0;
#pragma unroll
        for (int t = 0; t < TX; ++t)
            if (ix0 + c0 + t < nox) sp[t] = acc[u][t] + bias;
    }
}

size_t scores_rows_smem(int bins, int cells_y, int tx, int k) {
    return sizeof(double) * (size_t)(cells_y + 1) * bins * 8 +
           sizeof(uint32_t) * (size_t)SR_WARPS * 2 * sr_slot_words(bins, tx, k);
}

template <int K, int TX, int BINS>
void launch_rows_t(const int32_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                   int cells_y, const double *wts, double bias, double *scores, cudaStream_t st) {
    const size_t smem = scores_rows_smem(bins, cells_y, TX, K);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(k_scores_rows<K, TX, BINS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = smem;
    }
    // e / (TX bins) by multiply-high: exact for e < 2^20 (e < span * bins here)
    const uint32_t magic = (uint32_t)((0x100000000ull + TX * bins - 1) / (TX * bins));
    const int64_t blocks = (int64_t)n * ((noy + SR_TY * SR_WARPS - 1) / (SR_TY * SR_WARPS)) *
                           ((nox + 32 * TX - 1) / (32 * TX));
    k_scores_rows<K, TX, BINS><<<(unsigned)blocks, 32 * SR_WARPS, smem, st>>>(
        grid, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, magic);
}

template <int K, int TX>
void launch_rows_b(const int32_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                   int cells_y, const double *wts, double bias, double *scores, cudaStream_t st) {
    switch (bins) {
        case 8: return launch_rows_t<K, TX, 8>(grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, st);
        case 9: return launch_rows_t<K, TX, 9>(grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, st);
        case 18: return launch_rows_t<K, TX, 18>(grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, st);
        default: return launch_rows_t<K, TX, 0>(grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, st);
    }
}

// Window columns per lane: the candidate (TX / K integral) that wastes the
// fewest lanes on this width (ties to the larger TX: more reuse per grid
// value), e.g. c4 (153 columns) -> 5 (160, 96 %), c1 (93) -> 3, 8K (953) -> 5.
int pick_tx(int nox, int k) {
    static const int c1[] = {5, 6, 4, 3, 2}, c2[] = {6, 4, 2};
    const int *c = k == 1 ? c1 : c2;
    const int nc = k == 1 ? 5 : 3;
    int best = c[0];
    int64_t best_pad = INT64_MAX;
    for (int i = 0; i < nc; ++i) {
        const int64_t cols = 32 * c[i], pad = (nox + cols - 1) / cols * cols;
        if (pad < best_pad) best_pad = pad, best = c[i];
    }
    return best;
}

void launch_scores_rows(const int32_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                        int cells_y, int k, const double *wts, double bias, double *scores,
                        cudaStream_t st) {
    const int tx = pick_tx(nox, k);
#define SR_ARGS grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, st
    if (k == 1) {
        switch (tx) {
            case 2: return launch_rows_b<1, 2>(SR_ARGS);
            case 3: return launch_rows_b<1, 3>(SR_ARGS);
            case 4: return launch_rows_b<1, 4>(SR_ARGS);
            case 5: return launch_rows_b<1, 5>(SR_ARGS);
            default: return launch_rows_b<1, 6>(SR_ARGS);
        }
    }
    switch (tx) {
        case 2: return launch_rows_b<2, 2>(SR_ARGS);
        case 4: return launch_rows_b<2, 4>(SR_ARGS);
        default: return launch_rows_b<2, 6>(SR_ARGS);
    }
#undef SR_ARGS
}

}  // namespace hogb200
